# Round-1 profiling, ${V}: bench, launch list, per-launch DRAM traffic at p = 50,
V=${1:-v4}
# one --set full capture of the three iteration kernels.  Run under gpurun from the repo root.
set -x
python -m paper_2205_07805_b200.build > /dev/null
python bench.py > gpurun_out/bench_${V}.json 2> gpurun_out/bench_${V}.err
echo bench rc=$?
python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain_${V}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_${V}.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch_${V}.log 2>&1
echo launch rc=$?
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
python tools/traffic_run.py > gpurun_out/traffic_plain.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:bdot_tma_kernel -s 49 -c 1 --csv --log-file gpurun_out/traffic_bdot_${V}.csv python tools/traffic_run.py > /dev/null 2>&1 && \
ncu --metrics $M --clock-control none -k regex:update_kernel -s 51 -c 1 --csv --log-file gpurun_out/traffic_update_${V}.csv python tools/traffic_run.py > /dev/null 2>&1 && \
ncu --metrics $M --clock-control none -k regex:spmv_sell_kernel -s 51 -c 1 --csv --log-file gpurun_out/traffic_spmv_${V}.csv python tools/traffic_run.py > /dev/null 2>&1
echo traffic rc=$?
ncu --set full --clock-control none --import-source on -k regex:"bdot_tma_kernel|spmv_sell_kernel|update_kernel" -s 150 -c 3 \
    -o gpurun_out/prof_${V} -f python tools/traffic_run.py > gpurun_out/ncu_full_${V}.log 2>&1
echo full rc=$?
