# Round-2 profiling pass ${V}: bench line, ncu launch list of the same bench command, DRAM
# traffic per launch at several p (c4 and c3), and one --set full capture of the three c4
# iteration kernels at p ~ 50.  Run under gpurun from the repo root; outputs gpurun_out/*_${V}*.
V=${1:-r2a}
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
python bench.py > gpurun_out/bench_${V}.json 2> gpurun_out/bench_${V}.err
echo bench rc=$?
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/plain_${V}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_${V}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/ncu_launch_${V}.log 2>&1
echo launch rc=$?
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
python tools/traffic_run.py --config c4 --k 100 > gpurun_out/traffic_plain_${V}.log 2>&1 || exit 1
run() {  # cfg k kernel p skip
  ncu --metrics $M --clock-control none -k regex:$3 -s $5 -c 1 --csv \
      --log-file gpurun_out/tr_${V}_${3}_${1}_p${4}.csv python tools/traffic_run.py --config $1 --k $2 > /dev/null 2>&1
}
for p in 10 50 100; do run c4 100 bdot_tma_kernel $p $((p-1)); run c4 100 update_kernel $p $((p+1)); done
for p in 10 50 99; do run c4 100 spmv_sell_kernel $p $((p+1)); done
run c3 300 bdot_tma_kernel 300 299; run c3 300 update_kernel 300 301; run c3 300 spmv_sell_kernel 299 300
echo traffic rc=$?
ncu --set full --clock-control none --import-source on -k regex:"bdot_tma_kernel|spmv_sell_kernel|update_kernel" -s 150 -c 3 \
    -o gpurun_out/prof_${V} -f python tools/traffic_run.py --config c4 --k 60 > gpurun_out/ncu_full_${V}.log 2>&1
echo full rc=$?
