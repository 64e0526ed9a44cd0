# round-2 call 20: SELL diagonal path without find-first-set (ordered walk over the 8 list
# positions): tests, c4 bench A/B (pipe 16x3x2 / pipe 8x4x3 / row kernel), ncu of both kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c20_build.log 2>&1 || { tail -30 gpurun_out/c20_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_multirank.py -q -x -k "sell or spmv or halo or split or virtual" > gpurun_out/c20_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c20_tests.log
run() {  # tag env...
  tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c20_bench_$tag.json 2> gpurun_out/c20_bench_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/c20_bench_$tag.json')); k=d['kernels']; print('$tag c4', round(d['value'],1), 'spmv ms', round(k['spmv']['ms_per_step'],2), 'bdot', round(k['block_dot']['ms_per_step'],2), 'upd', round(k['update']['ms_per_step'],2), d['clocks']['sm_mhz'])"
}
run pipe16 IGS_SELL_PIPE_CFG=0
run row IGS_SELL_PIPE_MIN_N=-1
run pipe8 IGS_SELL_PIPE_CFG=1
run pipe16b IGS_SELL_PIPE_CFG=0
run rowb IGS_SELL_PIPE_MIN_N=-1
python tools/traffic_run.py > gpurun_out/c20_trplain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:spmv_sell_pipe_kernel -s 51 -c 1 -o gpurun_out/c20_spmv_pipe_p50 python tools/traffic_run.py > gpurun_out/c20_ncu_spmv.log 2>&1; echo "ncu pipe rc=$?"
IGS_SELL_PIPE_MIN_N=-1 ncu --set full --import-source on --clock-control none -k regex:spmv_sell_kernel -s 51 -c 1 -o gpurun_out/c20_spmv_row_p50 python tools/traffic_run.py > gpurun_out/c20_ncu_spmv_row.log 2>&1; echo "ncu row rc=$?"
