#!/bin/bash
# Phase timings of the persistent cycle kernel (IGS_PC_PROF=1) on c1/c2 for several grids.
set -e
python -m paper_2205_07805_b200.build >/dev/null
for c in c1 c2; do
  for g in 0 1 4 16 64; do
    for a in igs1 igs2; do
      echo "== $c grid=$g $a"
      IGS_PC_PROF=1 IGS_PC_GRID=$g python tools/bench_configs.py --config $c --alg $a --reps 1 2>&1 | grep pcycle | tail -1
    done
  done
done
