# round-2 call 7: the c5 oracle record again (pairwise-blocked LOO Gram) on the host while
# the GPU runs the profiles of tools/r2_call6.sh; then the c5 record test against it
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c7_build.log 2>&1 || { tail -30 gpurun_out/c7_build.log; exit 1; }
( OMP_NUM_THREADS=14 python tools/oracle_records.py c5 --norm-maxit 60 --out gpurun_out/oracle_c5_gs2_v2.json > gpurun_out/c7_orc5.log 2>&1; echo "orc5 rc=$?" >> gpurun_out/c7_orc5.log ) &
ORC=$!
bash tools/r2_call6.sh
for i in $(seq 1 240); do kill -0 $ORC 2>/dev/null || break; sleep 15; done
wait $ORC
tail -c 1200 gpurun_out/c7_orc5.log
cp gpurun_out/oracle_c5_gs2_v2.json tests/golden/oracle_c5_gs2.json && \
timeout 1200 python -m pytest tests/test_gpu_solve.py -q -m gpu -k "c5_k100 or lgram or loo" > gpurun_out/c7_c5test.log 2>&1; echo "c5 test rc=$?"; tail -15 gpurun_out/c7_c5test.log
