# round-2 call 24: the whole GPU suite with the slice-walking SpMV forced at every size
# (IGS_SELL_WALK_MIN_N=0), and with every slice explicit (IGS_SELL_DIAG=0)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c24_build.log 2>&1 || { tail -30 gpurun_out/c24_build.log; exit 1; }
IGS_SELL_WALK_MIN_N=0 timeout 1800 python -m pytest tests -m gpu -q -k "not sell_diag" > gpurun_out/c24_tests_walk.log 2>&1; echo "walk-everywhere tests rc=$?"; tail -5 gpurun_out/c24_tests_walk.log
IGS_SELL_DIAG=0 timeout 1800 python -m pytest tests -m gpu -q -k "not sell_diag" > gpurun_out/c24_tests_nodiag.log 2>&1; echo "no-diag tests rc=$?"; tail -5 gpurun_out/c24_tests_nodiag.log
