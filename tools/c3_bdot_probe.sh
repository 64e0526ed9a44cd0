# c3 (n = 1M) block dot at p = 150 and 300: duration / DRAM bytes, free clocks.
python -m paper_2205_07805_b200.build > /dev/null
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second"
python tools/traffic_run.py --config c3 --k 300 > gpurun_out/c3p_plain.log 2>&1 || exit 1
for p in 150 299; do
  ncu --metrics $M --clock-control none -k regex:bdot_tma_kernel -s $((p-1)) -c 1 --csv --log-file gpurun_out/c3p_$p.csv python tools/traffic_run.py --config c3 --k 300 > /dev/null 2>&1
  ncu --metrics $M --clock-control none -k regex:update_kernel -s $((p+1)) -c 1 --csv --log-file gpurun_out/c3u_$p.csv python tools/traffic_run.py --config c3 --k 300 > /dev/null 2>&1
done
echo done
