# round-2 call 33: tile block dot consumer loop with running stage / parity / column values and
# the stage released before the warp reduction (BT_FAST=1) vs before (=0): alternating rebuilds,
mkdir -p gpurun_out
# block-dot tests, c4 bench, isolated probes; then ncu instruction counts of both builds
for v in 1 0 1 0 1 0; do
  IGS_NVCC_EXTRA=-DBT_FAST=$v python -c "from paper_2205_07805_b200 import build; build.build(force=True)" > gpurun_out/c33_build_$v.log 2>&1 || { tail -30 gpurun_out/c33_build_$v.log; exit 1; }
  if [ $v = 1 ]; then timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "block_dot" > gpurun_out/c33_tests.log 2>&1; echo "tests rc=$?"; fi
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c33_bench_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c33_bench_$v.json')); k=d['kernels']; print('split=$v c4', round(d['value'],1), 'bdot', round(k['block_dot']['ms_per_step'],2), 'upd', round(k['update']['ms_per_step'],2), 'step', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
  for n in 16777216 2097152; do
    python tools/bdot_probe.py --n $n --ps 10,25,50,75,90 --pads 0 --reps 10 2>/dev/null | python -c "
import sys, json
r = [json.loads(l) for l in sys.stdin if l.startswith('{')]
print('split=$v n=$n', [(x['p'], round(x['bdot_us'], 1), round(x['bdot_gbs'])) for x in r])"
  done
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/traffic_run.py > /dev/null 2>&1
ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control base -k regex:bdot_tma_kernel -s 42 -c 1 --csv --log-file gpurun_out/c33_inst_fast.csv python tools/traffic_run.py > /dev/null 2>&1; tail -2 gpurun_out/c33_inst_fast.csv
