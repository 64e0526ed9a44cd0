# DRAM bytes per launch of the three iteration kernels at p in {10, 50, 99/100} (c4, k = 100)
# and p in {299/300} (c3, k = 300): SURVEY §8(d) asks for the byte model to hold within 5%.
# Launch order of one unrestarted Alg. 3 solve:
#   bdot_tma_kernel : iterations p = 1..k (p = k is the drain, no z)    -> skip p-1
#   update_kernel   : 2 priming launches, then p = 1..k                  -> skip p+1
#   spmv_sell_kernel: residual, priming, then p = 1..k-1                 -> skip p+1
set -x
python -m paper_2205_07805_b200.build > /dev/null
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
run() {  # cfg k kernel p skip
  ncu --metrics $M --clock-control none -k regex:$3 -s $5 -c 1 --csv \
      --log-file gpurun_out/tr_${3}_${1}_p${4}.csv python tools/traffic_run.py --config $1 --k $2 > /dev/null 2>&1
}
python tools/traffic_run.py --config c4 --k 100 > gpurun_out/tr_plain_c4.log 2>&1 && \
python tools/traffic_run.py --config c3 --k 300 > gpurun_out/tr_plain_c3.log 2>&1 || exit 1
for p in 10 50 100; do run c4 100 bdot_tma_kernel $p $((p-1)); run c4 100 update_kernel $p $((p+1)); done
for p in 10 50 99; do run c4 100 spmv_sell_kernel $p $((p+1)); done
run c3 300 bdot_tma_kernel 300 299; run c3 300 update_kernel 300 301; run c3 300 spmv_sell_kernel 299 300
run c3 300 bdot_tma_kernel 299 298; run c3 300 update_kernel 299 300
echo done rc=$?
