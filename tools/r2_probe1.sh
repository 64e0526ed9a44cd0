# round-2 first probe: box facts + block-dot bandwidth vs p / ld (c3 and c4 shapes)
set -x
mkdir -p gpurun_out
{ free -g; nproc; lscpu | head -20; nvidia-smi; nvidia-smi topo -m; } > gpurun_out/r2_box.txt 2>&1
python -m paper_2205_07805_b200.build > /dev/null
python tools/bdot_probe.py --n 1048576 --ps 10,50,100,150,200,250,300 --pads 0,32,1024 > gpurun_out/r2_bdot_c3.jsonl 2>&1
python tools/bdot_probe.py --n 16777216 --ps 10,50,100 --pads 0,32 > gpurun_out/r2_bdot_c4.jsonl 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:bdot_tma -s 1 -c 6 --csv --log-file gpurun_out/r2_bdot_c3_ncu.csv python tools/bdot_probe.py --n 1048576 --ps 300 --pads 0 --reps 2 > /dev/null 2>&1
echo done
