# Per-config / per-algorithm throughput sweep (one GPU) -> gpurun_out/sweep.jsonl
out=gpurun_out/sweep.jsonl
: > $out
for c in c1 c2 c3 c4; do
  for a in igs1 igs2 igs2_two mgs; do
    reps=3; [ $c = c4 ] && reps=4   # (2 solves after one warm-up still sit on the process's first, slower solves)
    timeout 600 python tools/bench_configs.py --config $c --alg $a --reps $reps 2>/dev/null | tail -1 >> $out
  done
done
timeout 900 python tools/bench_configs.py --config c5 --alg igs2 --reps 1 2>&1 | tail -1 >> $out
echo done
