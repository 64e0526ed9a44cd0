# round-2 call 39: the full GPU suite again after the c3 one-sweep LOO band (reading R19 over
# the oracle's orders incl. pairwise block sums); the c4 lines of the sweep repeated
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c39_build.log 2>&1 || { tail -30 gpurun_out/c39_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c39_tests.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/c39_tests.log
for i in 1 2; do for a in igs2 igs2_two igs1; do
  timeout 600 python tools/bench_configs.py --config c4 --alg $a --reps 2 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('run $i', d['config'], d['alg'], round(d['it_s'], 1), 'ms/solve', round(d['ms_per_solve'], 1), 'timed-run ms', round(d['ms_per_solve_timed_run'], 1))"
done; done
