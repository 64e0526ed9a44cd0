# round-2 call 14: SELL-32 diagonal slices (no column indices for slices whose rows use <= 8
# offsets): bitwise tests vs the oracle, the multirank / solve suites, A/B against
# IGS_SELL_DIAG=0 on the c4 bench, the one-GPU slab proxy and c3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c14_build.log 2>&1 || { tail -30 gpurun_out/c14_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_multirank.py -q -x > gpurun_out/c14_tests_k.log 2>&1; echo "kernel+multirank tests rc=$?"; tail -3 gpurun_out/c14_tests_k.log
timeout 1500 python -m pytest tests/test_gpu_solve.py -q -x > gpurun_out/c14_tests_s.log 2>&1; echo "solve tests rc=$?"; tail -3 gpurun_out/c14_tests_s.log
for d in 1 0; do
  IGS_SELL_DIAG=$d python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c14_bench_d$d.json 2> gpurun_out/c14_bench_d$d.err
  python -c "import json; d=json.load(open('gpurun_out/c14_bench_d$d.json')); k=d['kernels']; print('diag=$d c4', round(d['value'],1), 'spmv ms', round(k['spmv']['ms_per_step'],2), 'bdot', round(k['block_dot']['ms_per_step'],2), 'upd', round(k['update']['ms_per_step'],2), d['clocks']['sm_mhz'])"
  IGS_SELL_DIAG=$d python tools/slab_proxy.py > gpurun_out/c14_slab_d$d.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/c14_slab_d$d.json')); print('diag=$d slab', d['plain']['it_s'], d['plain']['us_per_iteration'])"
  IGS_SELL_DIAG=$d python tools/bench_configs.py --config c3 --k 300 > gpurun_out/c14_c3_d$d.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c14_c3_d$d.json').read().strip().splitlines()[-1]); print('diag=$d c3', round(d['it_s']))"
done
