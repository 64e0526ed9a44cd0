# Fused wavefront kernel (IGS_FUSED=1) on c4: throughput, and one launch at p = 30 under ncu at
# locked base clocks vs free clocks (SM-cycle bound or memory bound?).
python -m paper_2205_07805_b200.build > /dev/null
IGS_FUSED=1 python tools/bench_configs.py --config c4 --k 60 --reps 2 | cut -c1-600
python tools/bench_configs.py --config c4 --k 60 --reps 2 | cut -c1-300
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum"
IGS_FUSED=1 python tools/traffic_run.py > gpurun_out/fp_plain.log 2>&1 || exit 1
for cc in base none; do
  IGS_FUSED=1 ncu --metrics $M --clock-control $cc -k regex:fused -s 30 -c 1 --csv --log-file gpurun_out/fp_$cc.csv python tools/traffic_run.py > /dev/null 2>&1
done
echo done
