# round-2 call 40: bench_configs' c4 Alg. 3 entry read 290-391 it/s in calls 38/39 while bench.py
# read 436: one vs two block-dot consumer groups (IGS_BDOT_GROUPS=1 / default), more solves
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c40_build.log 2>&1 || { tail -30 gpurun_out/c40_build.log; exit 1; }
for i in 1 2; do for gp in 0 1; do
  IGS_BDOT_GROUPS=$gp timeout 600 python tools/bench_configs.py --config c4 --alg igs2 --reps 6 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('groups_forced=$gp run $i', d['config'], d['alg'], round(d['it_s'], 1), 'ms/solve', round(d['ms_per_solve'], 1), 'timed-run ms', round(d['ms_per_solve_timed_run'], 1))"
  IGS_BDOT_GROUPS=$gp python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e --no-solve 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('groups_forced=$gp run $i bench.py', round(d['value'], 1), round(d['ms_per_step'], 1), d['clocks']['sm_mhz'])"
done; done
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x -k "c3_full_size" > gpurun_out/c40_tests.log 2>&1; echo "c3 test rc=$?"; tail -2 gpurun_out/c40_tests.log
