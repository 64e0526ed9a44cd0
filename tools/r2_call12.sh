# round-2 call 12: the newest tests (chunked host x, sweep + exchange), bench e2e
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c12_build.log 2>&1 || { tail -30 gpurun_out/c12_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x -k "host or sweep or fused_exchange" > gpurun_out/c12_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c12_tests.log
timeout 900 python bench.py --no-cpu --no-solve > gpurun_out/c12_bench.json 2> gpurun_out/c12_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c12_bench.json')); print(d['value'], d['e2e'], d['clocks']['sm_mhz'])"
