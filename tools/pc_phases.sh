#!/bin/bash
# Persistent-kernel phase split (IGS_PC_PROF=1) across sizes: c1, c2, c3 at N = 64..362.
for spec in "c1" "c2" "c3 --N 64" "c3 --N 128" "c3 --N 256" "c3 --N 362"; do
  echo "== $spec"
  IGS_PC_PROF=1 python tools/bench_configs.py --config $spec --alg igs2 --k 100 --reps 2 2>&1 | grep "pcycle grid" | tail -1
done
