set -x
python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo launch rc=$?
ncu --set full --clock-control none --import-source on -k regex:"bdot_kernel|spmv_stream|update_kernel" -s 150 -c 6 -o gpurun_out/prof_r1 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
ls -la gpurun_out
