# round-2 call 34: two-reduce fused update+dot with tile heights 256 / 224 / 192 / 160 / 128
# (UT_RSTEP=32) vs 256 / 128 only (=128): two-reduce tests, c4 and c3 it/s, alternating rebuilds
mkdir -p gpurun_out
for v in 32 128 32 128; do
  IGS_NVCC_EXTRA=-DUT_RSTEP=$v python -c "from paper_2205_07805_b200 import build; build.build(force=True)" > gpurun_out/c34_build_$v.log 2>&1 || { tail -30 gpurun_out/c34_build_$v.log; exit 1; }
  if [ $v = 32 ]; then timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py -q -x -k "two" > gpurun_out/c34_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/c34_tests.log; fi
  for c in c4 c3; do
    timeout 600 python tools/bench_configs.py --config $c --alg igs2_two --reps 3 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('rstep=$v', d['config'], d['alg'], round(d['it_s'], 1), 'update ms', round(d['kernels']['update']['ms'], 2))"
  done
done
