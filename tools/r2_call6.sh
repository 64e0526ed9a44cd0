# round-2 profiles: ncu launch list of the bench command, DRAM traffic + one --set full
# capture of the column-sweep block dot at c3 p = 299 and of the SELL SpMV (x prefetch) on c4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c6_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/c6_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c6_ncu_launch.log 2>&1
echo "launch list rc=$?"
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed"
python tools/traffic_run.py --config c3 --k 300 > gpurun_out/c6_traffic_plain.log 2>&1 || exit 1
for sp in "203 299" "204 300"; do set -- $sp
  ncu --metrics $M --clock-control none -k regex:bdot_sw_kernel -s $1 -c 1 --csv \
      --log-file gpurun_out/c6_tr_bdot_sw_c3_p$2.csv python tools/traffic_run.py --config c3 --k 300 > /dev/null 2>&1
done
ncu --metrics $M --clock-control none -k regex:spmv_sell_kernel -s 51 -c 1 --csv \
    --log-file gpurun_out/c6_tr_spmv_c4_p50.csv python tools/traffic_run.py --config c4 --k 60 > /dev/null 2>&1
echo "traffic rc=$?"
ncu --set full --clock-control none --import-source on -k regex:bdot_sw_kernel -s 203 -c 1 \
    -o gpurun_out/c6_prof_bdot_sw_c3 -f python tools/traffic_run.py --config c3 --k 300 > gpurun_out/c6_full1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmv_sell_kernel -s 51 -c 1 \
    -o gpurun_out/c6_prof_spmv_c4 -f python tools/traffic_run.py --config c4 --k 60 > gpurun_out/c6_full2.log 2>&1
echo "full rc=$?"
