mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
python bench.py > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo "bench rc=$?"
timeout 600 python -m pytest tests/test_gpu_solve.py -q -m gpu -k "lgram" > gpurun_out/r2_lgram.log 2>&1; echo "lgram rc=$?"
free -g
/usr/bin/time -v python tools/oracle_records.py c5 --norm-maxit 60 --out gpurun_out/oracle_c5_gs2.json > gpurun_out/r2_orc5.log 2>&1; echo "orc5 rc=$?"
tail -3 gpurun_out/r2_orc5.log
