# Clock sensitivity of the two V-streaming kernels: one launch at p = 50 (c4) under ncu with
# --clock-control base (locked base clocks) vs none.
python -m paper_2205_07805_b200.build > /dev/null
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,dram__cycles_elapsed.avg.per_second"
python tools/traffic_run.py > gpurun_out/cs_plain.log 2>&1 || exit 1
for cc in base none; do
  ncu --metrics $M --clock-control $cc -k regex:bdot_tma_kernel -s 49 -c 1 --csv --log-file gpurun_out/cs_bdot_$cc.csv python tools/traffic_run.py > /dev/null 2>&1
  ncu --metrics $M --clock-control $cc -k regex:update_kernel -s 51 -c 1 --csv --log-file gpurun_out/cs_update_$cc.csv python tools/traffic_run.py > /dev/null 2>&1
done
echo done
