#!/bin/bash
# gs = 1 vs gs = 2 on c1/c2: persistent kernel phase split and it/s (regression probe).
for c in c1 c2; do
  for a in igs1 igs2; do
    echo "== $c $a"
    IGS_PC_PROF=1 python tools/bench_configs.py --config $c --alg $a --reps 3 2>&1 | grep -E "pcycle" | tail -1
    python tools/bench_configs.py --config $c --alg $a --reps 3 2>&1 | tail -1 | cut -c1-160
  done
done
