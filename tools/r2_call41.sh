# round-2 call 41: the round's last check at HEAD -- full GPU suite, smoke, default bench line,
# reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c41_build.log 2>&1 || { tail -30 gpurun_out/c41_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c41_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c41_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c41_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/c41_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/c41_bench_reference.json 2> gpurun_out/c41_bench_reference.err; echo "reference arm rc=$?"
timeout 900 python bench.py > gpurun_out/c41_bench.json 2> gpurun_out/c41_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c41_bench.json')); print(d['value'], d['e2e']['value'], d['clocks'], {n: round(v['ms_per_step'],1) for n,v in d['kernels'].items()}, d.get('solve_to_1e-12'), d['roofline'], d['roofline_frac_iteration'], d['roofline_frac_iteration_moved'])"
