# probes: block dot / update vs p at c4 and slab sizes; one-GPU slab proxy; persistent crossover
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
python tools/bdot_probe.py --n 16777216 --ps 1,2,4,8,10,16,24,32,50,64,100 --pads 0 --reps 5 > gpurun_out/r2_probe_c4.jsonl 2>&1
python tools/bdot_probe.py --n 2097152 --ps 1,2,4,8,10,16,24,32,50,64,100 --pads 0 --reps 20 > gpurun_out/r2_probe_slab.jsonl 2>&1
python tools/slab_proxy.py > gpurun_out/r2_slab_proxy.json 2>&1
python tools/pc_crossover.py --Ns 384,420,443,470 > gpurun_out/r2_pc_crossover.jsonl 2>&1
echo done
