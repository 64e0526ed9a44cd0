# round-2 call 25: after the SELL planner moved to plan.cpp -- SELL / SpMV / multirank / solve
# tests; ncu --set full of the two-reduce fused update+dot and of the MGS step at c4 p = 50
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c25_build.log 2>&1 || { tail -30 gpurun_out/c25_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/c25_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c25_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-solve > gpurun_out/c25_bench.json 2> gpurun_out/c25_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c25_bench.json')); print(d['value'], d['e2e']['value'], d['roofline_frac_iteration'], d['roofline_frac_iteration_moved'], d['clocks']['sm_mhz'])"
python tools/traffic_run.py --alg igs2_two > gpurun_out/c25_two_plain.log 2>&1; tail -1 gpurun_out/c25_two_plain.log
ncu --set full --import-source on --clock-control none -k regex:update_dot -s 50 -c 1 -o gpurun_out/c25_update_dot_p50 python tools/traffic_run.py --alg igs2_two > gpurun_out/c25_ncu_ud.log 2>&1; echo "ncu update_dot rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/c25_two_launches.csv python tools/traffic_run.py --alg igs2_two > gpurun_out/c25_ncu_two_launch.log 2>&1; echo "two launch list rc=$?"
