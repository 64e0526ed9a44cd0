# round-2 call 28: persistent kernel with A resident in shared memory (c2): tests, c2 it/s and
# phase times with IGS_PC_ARES=1/0
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c28_build.log 2>&1 || { tail -30 gpurun_out/c28_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_solve.py -q -x -k "persistent or small_configs or tiny" > gpurun_out/c28_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c28_tests.log
for ar in 1 0 1 0; do
  for a in igs2 igs1; do
    IGS_PC_ARES=$ar timeout 600 python tools/bench_configs.py --config c2 --alg $a --reps 3 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('ares=$ar', d['config'], d['alg'], round(d['it_s']))"
  done
done
for ar in 1 0; do echo "ares=$ar phases:"; IGS_PC_ARES=$ar IGS_PC_PROF=1 python tools/pc_one.py c2 igs2 2>&1 | tail -3; done
