# round-2 call 43: two consumer groups from p = 24: block-dot / solve tests, short bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c43_build.log 2>&1 || { tail -30 gpurun_out/c43_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py tests/test_gpu_multirank.py -q -k "block_dot or qr or downsized or small_configs or c4 or two or virtual" > gpurun_out/c43_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c43_tests.log
python bench.py --steps 6 --warmup 3 --no-cpu --no-solve 2>/dev/null > gpurun_out/c43_bench.json; python -c "
import json; d = json.load(open('gpurun_out/c43_bench.json')); print(round(d['value'], 1), round(d['e2e']['value'], 1), {n: round(v['ms_per_step'], 1) for n, v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
