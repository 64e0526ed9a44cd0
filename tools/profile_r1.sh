# Round-1 profiling (run under gpurun from the repo root): plain bench, launch list, full capture.
set -x
python bench.py > gpurun_out/bench_full.log 2>&1
echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo ref rc=$?
python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo launch rc=$?
ncu --set full --clock-control none --import-source on -k regex:"bdot_tma_kernel|spmv_stream|update_kernel|small_kernel" -s 200 -c 8 -o gpurun_out/prof_r1 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
