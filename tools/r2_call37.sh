# round-2 call 37: tile block dot with two groups of 8 consumer warps on alternate stages
# (BT_GROUPS=2, 4 consumer warps per scheduler, 96 registers) vs one group (=1): alternating rebuilds,
mkdir -p gpurun_out
for v in 2 1 2 1; do
  IGS_NVCC_EXTRA=-DBT_GROUPS=$v python -c "from paper_2205_07805_b200 import build; build.build(force=True)" > gpurun_out/c37_build_$v.log 2>&1 || { tail -30 gpurun_out/c37_build_$v.log; exit 1; }
  if [ $v = 2 ]; then timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "block_dot or qr" > gpurun_out/c37_tests.log 2>&1; echo "tests rc=$?"; fi
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c37_bench_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c37_bench_$v.json')); k=d['kernels']; print('split=$v c4', round(d['value'],1), 'bdot', round(k['block_dot']['ms_per_step'],2), 'upd', round(k['update']['ms_per_step'],2), 'step', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
  for n in 16777216 2097152; do
    python tools/bdot_probe.py --n $n --ps 10,25,50,75,90 --pads 0 --reps 10 2>/dev/null | python -c "
import sys, json
r = [json.loads(l) for l in sys.stdin if l.startswith('{')]
print('split=$v n=$n', [(x['p'], round(x['bdot_us'], 1), round(x['bdot_gbs'])) for x in r])"
  done
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
