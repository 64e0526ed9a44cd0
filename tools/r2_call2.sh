# round-2 call 2: c5 oracle record on the host (background, CPU only, 196 GB box) while the
# GPU runs the block-dot / update probes, the one-GPU slab proxy, a longer bench and the
# full c4 solve
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c2_build.log 2>&1 || { tail -30 gpurun_out/c2_build.log; exit 1; }
( OMP_NUM_THREADS=14 /usr/bin/time -v python tools/oracle_records.py c5 --norm-maxit 60 --out gpurun_out/oracle_c5_gs2.json > gpurun_out/c2_orc5.log 2>&1; echo "orc5 rc=$?" >> gpurun_out/c2_orc5.log ) &
ORC=$!
python tools/bdot_probe.py --n 1048576 --ps 10,50,100,150,200,250,300 --pads 0,32,1024 > gpurun_out/c2_bdot_c3.jsonl 2>&1
python tools/bdot_probe.py --n 16777216 --ps 10,50,100 --pads 0,32 > gpurun_out/c2_bdot_c4.jsonl 2>&1
python tools/slab_proxy.py > gpurun_out/c2_slab_proxy.json 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c2_bench20.json 2> gpurun_out/c2_bench20.err
python tools/full_solve.py > gpurun_out/c2_full_solve.json 2>&1
echo "gpu part done"; free -g
wait $ORC
tail -c 2500 gpurun_out/c2_orc5.log
