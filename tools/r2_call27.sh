# round-2 call 27: sweep block dot below p = 8 in the c4 bench (A/B x3, alternating); the
# split-SpMV test with IGS_TEST_BND_ENDS; slab proxy with the outer planes through the
# boundary pass
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c27_build.log 2>&1 || { tail -30 gpurun_out/c27_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_multirank.py -q -x -k "split" > gpurun_out/c27_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c27_tests.log
for i in 1 2 3; do for sm in 1 0; do
  IGS_BDOT_SW_SMALL_P=$sm python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c27_bench_sm${sm}_$i.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c27_bench_sm${sm}_$i.json')); k=d['kernels']; print('small_p=$sm c4', round(d['value'],1), 'bdot', round(k['block_dot']['ms_per_step'],2), 'step', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done; done
timeout 900 python tools/slab_proxy.py > gpurun_out/c27_slab_proxy.json 2> gpurun_out/c27_slab_proxy.err
python -c "
import json
for l in open('gpurun_out/c27_slab_proxy.json'):
    if l.startswith('{'):
        d = json.loads(l)
        for k, v in d.items():
            if isinstance(v, dict): print(k, round(v.get('it_s', 0), 1), round(v.get('us_per_iteration', 0), 1), v.get('info', {}).get('n_bnd'), v.get('error'))"
