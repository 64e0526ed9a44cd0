# round-2 re-entry: box facts, GPU tests (minus the oracle-record tests whose records are
# still being written), smoke, default bench line
mkdir -p gpurun_out
{ free -g; nproc; lscpu | head -20; nvidia-smi; } > gpurun_out/r2_box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1 || { tail -30 gpurun_out/r2_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -k "not oracle_record" ${PYTEST_ARGS:-} > gpurun_out/r2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
tail -25 gpurun_out/r2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/r2_smoke.log
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
cat gpurun_out/r2_bench.json | head -c 4000; tail -5 gpurun_out/r2_bench.err
