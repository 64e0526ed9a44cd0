# round-2 call 10: programmatic dependent launch A/B (IGS_PDL=0/1): per-kernel parity and
# solve tests with PDL, c4 bench, the one-GPU slab proxy, c3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c10_build.log 2>&1 || { tail -30 gpurun_out/c10_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -q -x -k "not c5 and not c4_as_specified and not c3_full" > gpurun_out/c10_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c10_tests.log
for pdl in 0 1; do
  IGS_PDL=$pdl python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c10_bench_pdl$pdl.json 2> gpurun_out/c10_bench_pdl$pdl.err
  python -c "import json; d=json.load(open('gpurun_out/c10_bench_pdl$pdl.json')); print('pdl=$pdl c4', round(d['value'],1), d['clocks']['sm_mhz'])"
  IGS_PDL=$pdl python tools/slab_proxy.py > gpurun_out/c10_slab_pdl$pdl.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/c10_slab_pdl$pdl.json')); print('pdl=$pdl slab', {k: round(v['it_s']) for k, v in d.items() if isinstance(v, dict) and 'it_s' in v})"
  IGS_PDL=$pdl python tools/bench_configs.py --config c3 --k 300 > gpurun_out/c10_c3_pdl$pdl.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c10_c3_pdl$pdl.json').read().strip().splitlines()[-1]); print('pdl=$pdl c3', round(d['it_s']))"
done
