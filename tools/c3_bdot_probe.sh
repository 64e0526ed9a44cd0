# c3 (n = 1M) block dot and update at p = 150: duration / DRAM bytes at free and at locked base
# clocks (SM-cycle bound or memory bound?).
python -m paper_2205_07805_b200.build > /dev/null
M="gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second"
python tools/traffic_run.py --config c3 --k 300 > gpurun_out/c3p_plain.log 2>&1 || exit 1
for cc in none base; do
  ncu --metrics $M --clock-control $cc -k regex:bdot_tma_kernel -s 149 -c 1 --csv --log-file gpurun_out/c3p_$cc.csv python tools/traffic_run.py --config c3 --k 300 > /dev/null 2>&1
  ncu --metrics $M --clock-control $cc -k regex:update_kernel -s 151 -c 1 --csv --log-file gpurun_out/c3u_$cc.csv python tools/traffic_run.py --config c3 --k 300 > /dev/null 2>&1
done
echo done
