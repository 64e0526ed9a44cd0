# round-2 call 44: full GPU suite + smoke at the round's final HEAD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c44_build.log 2>&1 || { tail -30 gpurun_out/c44_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c44_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c44_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c44_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/c44_smoke.log
