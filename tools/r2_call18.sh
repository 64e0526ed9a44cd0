# round-2 call 18 (re-entry): HEAD (SELL diagonal slices, kernel specialised by slice kind)
# -- full GPU suite, smoke, default bench, diag A/B, ncu launch list, SpMV --set full
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c18_build.log 2>&1 || { tail -30 gpurun_out/c18_build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/c18_box.txt; free -g >> gpurun_out/c18_box.txt; nproc >> gpurun_out/c18_box.txt
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/c18_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c18_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c18_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/c18_smoke.log
timeout 900 python bench.py > gpurun_out/c18_bench.json 2> gpurun_out/c18_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c18_bench.json')); print(d['value'], d['e2e']['value'], d['clocks'], {n: round(v['ms_per_step'],1) for n,v in d['kernels'].items()}, d.get('solve_to_1e-12'), d['roofline'])"
for d in 1 0; do
  IGS_SELL_DIAG=$d python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c18_bench_d$d.json 2> gpurun_out/c18_bench_d$d.err
  python -c "import json; d=json.load(open('gpurun_out/c18_bench_d$d.json')); k=d['kernels']; print('diag=$d c4', round(d['value'],1), 'spmv ms', round(k['spmv']['ms_per_step'],2), 'bdot', round(k['block_dot']['ms_per_step'],2), 'upd', round(k['update']['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c18_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/c18_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c18_ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/traffic_run.py > gpurun_out/c18_trplain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:spmv_sell_kernel -s 51 -c 1 -o gpurun_out/c18_spmv_p50 python tools/traffic_run.py > gpurun_out/c18_ncu_spmv.log 2>&1; echo "ncu spmv rc=$?"
