# round-2 call 3: c5 oracle record on the host (background) + the solve-gap probe
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c3_build.log 2>&1 || { tail -30 gpurun_out/c3_build.log; exit 1; }
( OMP_NUM_THREADS=14 python tools/oracle_records.py c5 --norm-maxit 60 --out gpurun_out/oracle_c5_gs2.json > gpurun_out/c3_orc5.log 2>&1; echo "orc5 rc=$?" >> gpurun_out/c3_orc5.log ) &
ORC=$!
python tools/solve_gap.py > gpurun_out/c3_solve_gap.jsonl 2>&1
cat gpurun_out/c3_solve_gap.jsonl
for i in $(seq 1 200); do sleep 15; kill -0 $ORC 2>/dev/null || break; free -g | sed -n 2p >> gpurun_out/c3_mem.txt; done
wait $ORC
tail -c 2500 gpurun_out/c3_orc5.log
