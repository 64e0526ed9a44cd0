# round-2 call 26: column-sweep block dot below p = 8 -- block-dot tests, probe at p = 1..9
# (c4, one c4 slab, c3) against the tile kernel everywhere, c4 bench and slab proxy A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c26_build.log 2>&1 || { tail -30 gpurun_out/c26_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "block_dot" > gpurun_out/c26_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c26_tests.log
for sw in 96 1000000; do
  for n in 16777216 2097152 1048576; do
    IGS_BDOT_SW_MIN_P=$sw python tools/bdot_probe.py --n $n --ps 1,2,3,4,5,6,7,8,9 --pads 0 --reps 20 > gpurun_out/c26_probe_sw${sw}_n$n.jsonl 2>/dev/null
  done
done
python - <<'PY'
import json
for n in (16777216, 2097152, 1048576):
    a = [json.loads(l) for l in open(f'gpurun_out/c26_probe_sw96_n{n}.jsonl') if l.startswith('{')]
    b = [json.loads(l) for l in open(f'gpurun_out/c26_probe_sw1000000_n{n}.jsonl') if l.startswith('{')]
    print(n, [(x['p'], round(x['bdot_us'], 1), round(y['bdot_us'], 1)) for x, y in zip(a, b)])
PY
for sw in 96 1000000 96; do
  IGS_BDOT_SW_MIN_P=$sw python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c26_bench_sw$sw.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c26_bench_sw$sw.json')); k=d['kernels']; print('sw=$sw c4', round(d['value'],1), 'bdot', round(k['block_dot']['ms_per_step'],2), d['clocks']['sm_mhz'])"
  IGS_BDOT_SW_MIN_P=$sw python tools/slab_proxy.py 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('sw=$sw slab', round(d['plain']['it_s'], 1), round(d['plain']['us_per_iteration'], 1))"
done
