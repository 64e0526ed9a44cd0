# round-2 call 15: where the tile block dot spends its cycles (c4, p = 50): ncu --set full
# at free clocks, and time / SM cycles at locked base clocks vs free for the block dot, the
# fused update and the SELL SpMV (diagonal slices)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c15_build.log 2>&1 || { tail -30 gpurun_out/c15_build.log; exit 1; }
python tools/traffic_run.py > gpurun_out/c15_plain.log 2>&1 || { cat gpurun_out/c15_plain.log; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:bdot_tma_kernel -s 49 -c 1 -o gpurun_out/c15_bdot_p50 python tools/traffic_run.py > gpurun_out/c15_ncu_bdot.log 2>&1; echo "ncu bdot rc=$?"
ncu --set full --import-source on --clock-control none -k regex:spmv_sell_kernel -s 51 -c 1 -o gpurun_out/c15_spmv_p50 python tools/traffic_run.py > gpurun_out/c15_ncu_spmv.log 2>&1; echo "ncu spmv rc=$?"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__cycles_elapsed.max"
for cc in base none; do
  for k in bdot_tma_kernel:49 update_kernel:51 spmv_sell_kernel:51; do
    kn=${k%%:*}; sk=${k##*:}
    ncu --metrics $M --clock-control $cc -k regex:$kn -s $sk -c 1 --csv --log-file gpurun_out/c15_cs_${kn}_$cc.csv python tools/traffic_run.py > /dev/null 2>&1
  done
done
echo done
