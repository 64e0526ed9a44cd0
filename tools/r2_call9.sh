# round-2 call 9: GPU suite (with every oracle record), smoke, default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c9_build.log 2>&1 || { tail -30 gpurun_out/c9_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x -k "virtual_solve" > gpurun_out/c9_vsolve.log 2>&1; echo "virtual solve rc=$?"; tail -30 gpurun_out/c9_vsolve.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c9_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/c9_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c9_smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/c9_smoke.log
timeout 900 python bench.py > gpurun_out/c9_bench.json 2> gpurun_out/c9_bench.err; echo "bench rc=$?"; head -c 3000 gpurun_out/c9_bench.json
