# Full ncu capture of one c4 SpMV launch (iteration p = 10) for stall / occupancy analysis.
python -m paper_2205_07805_b200.build > /dev/null
python tools/traffic_run.py > gpurun_out/spmv_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:spmv_stream_kernel -s 11 -c 1 \
    -o gpurun_out/spmv_full -f python tools/traffic_run.py > gpurun_out/spmv_ncu.log 2>&1
echo rc=$?
