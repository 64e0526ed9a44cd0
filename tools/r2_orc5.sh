# oracle record of BASELINE configs[4] (c5, k = 100, V = 108 GB on the host) -- CPU only,
# run on the GPU box for its 196 GB of host RAM
mkdir -p gpurun_out
python -c "import oracle; oracle.build()" > /dev/null 2>&1
free -g > gpurun_out/r2_orc5_mem.txt
python tools/oracle_records.py c5 --norm-maxit 60 --out gpurun_out/oracle_c5_gs2.json > gpurun_out/r2_orc5.log 2>&1
echo "orc5 rc=$?"
free -g >> gpurun_out/r2_orc5_mem.txt
tail -c 1500 gpurun_out/r2_orc5.log
