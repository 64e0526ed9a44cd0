# round-2 call 31: c3 IGS(1) (call 29's sweep measured 1924 it/s against 2405 in call 23): repeat
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c31_build.log 2>&1 || { tail -30 gpurun_out/c31_build.log; exit 1; }
for i in 1 2 3; do
  for a in igs1 igs2; do
    timeout 600 python tools/bench_configs.py --config c3 --alg $a --reps 3 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('run $i', d['config'], d['alg'], round(d['it_s']), 'ms/solve', round(d['ms_per_solve'], 1), 'timed-run ms', round(d['ms_per_solve_timed_run'], 1))"
  done
done
IGS_GRAPHS=0 timeout 600 python tools/bench_configs.py --config c3 --alg igs1 --reps 3 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('graphs=0', d['config'], d['alg'], round(d['it_s']), 'ms/solve', round(d['ms_per_solve'], 1))"
timeout 600 python tools/bench_configs.py --config c3 --alg igs1 --reps 10 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('reps=10', d['config'], d['alg'], round(d['it_s']), 'ms/solve', round(d['ms_per_solve'], 1))"
