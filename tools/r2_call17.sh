# round-2 call 17: SELL kernel specialised by slice kind (all-diagonal: 40 registers, 6
# CTAs/SM), status word gating only the store, metadata L2 prefetch: tests, bench A/B, ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c17_build.log 2>&1 || { tail -30 gpurun_out/c17_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_multirank.py -q -x -k "sell or spmv or halo or split" > gpurun_out/c17_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c17_tests.log
for d in 1 0; do
  IGS_SELL_DIAG=$d python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c17_bench_d$d.json 2> gpurun_out/c17_bench_d$d.err
  python -c "import json; d=json.load(open('gpurun_out/c17_bench_d$d.json')); k=d['kernels']; print('diag=$d c4', round(d['value'],1), 'spmv ms', round(k['spmv']['ms_per_step'],2), 'bdot', round(k['block_dot']['ms_per_step'],2), 'upd', round(k['update']['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
python tools/traffic_run.py > gpurun_out/c17_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:spmv_sell_kernel -s 51 -c 1 -o gpurun_out/c17_spmv_p50 python tools/traffic_run.py > gpurun_out/c17_ncu_spmv.log 2>&1; echo "ncu spmv rc=$?"
timeout 1200 python -m pytest tests/test_gpu_solve.py -q -x > gpurun_out/c17_tests_s.log 2>&1; echo "solve tests rc=$?"; tail -3 gpurun_out/c17_tests_s.log
