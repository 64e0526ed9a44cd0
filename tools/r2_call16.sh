# round-2 call 16: SELL diagonal slices after the prefetch fix (monotone column offsets):
# SpMV tests, then the c4 bench A/B (IGS_SELL_DIAG=1/0), then call 15's profiles
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c16_build.log 2>&1 || { tail -30 gpurun_out/c16_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_multirank.py -q -x -k "sell or spmv or halo or split" > gpurun_out/c16_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c16_tests.log
for d in 1 0; do
  IGS_SELL_DIAG=$d python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c16_bench_d$d.json 2> gpurun_out/c16_bench_d$d.err
  python -c "import json; d=json.load(open('gpurun_out/c16_bench_d$d.json')); k=d['kernels']; print('diag=$d c4', round(d['value'],1), 'spmv ms', round(k['spmv']['ms_per_step'],2), 'bdot', round(k['block_dot']['ms_per_step'],2), 'upd', round(k['update']['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
bash tools/r2_call15.sh
