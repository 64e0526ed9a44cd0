# DRAM traffic per launch of the iteration kernels at a known p (c4, Alg. 3, k = 60):
#   bdot_tma_kernel launches are iterations p = 1..60 in order     -> skip 49 = p 50
#   update_kernel: 2 priming launches, then p = 1..60              -> skip 51 = p 50
#   spmv_stream_kernel: residual, priming, then p = 1..59          -> skip 51 = p 50
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
python tools/traffic_run.py > gpurun_out/traffic_plain.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:bdot_tma_kernel -s 49 -c 1 --csv --log-file gpurun_out/traffic_bdot.csv python tools/traffic_run.py > /dev/null 2>&1 && \
ncu --metrics $M --clock-control none -k regex:update_kernel -s 51 -c 1 --csv --log-file gpurun_out/traffic_update.csv python tools/traffic_run.py > /dev/null 2>&1 && \
ncu --metrics $M --clock-control none -k regex:spmv_stream_kernel -s 51 -c 1 --csv --log-file gpurun_out/traffic_spmv.csv python tools/traffic_run.py > /dev/null 2>&1
echo rc=$?
