#!/bin/bash
# Persistent cycle kernel vs CUDA-graph per-kernel path across problem sizes (it/s), k = 100.
python -m paper_2205_07805_b200.build >/dev/null
for spec in "c1 0" "c2 0" "c3 64" "c3 128" "c3 256" "c3 362" "c3 512" "c4 32" "c4 40" "c4 64"; do
  set -- $spec
  for pc in 1 0; do
    for a in igs2; do
      r=$(IGS_PERSIST=$pc IGS_PC_MAX_N=100000000 python tools/bench_configs.py --config $1 --N $2 --alg $a --reps 3 --k 100 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['n'], round(d['it_s']), round(d['ms_per_solve'],3))")
      echo "$1 N=$2 persist=$pc $a: $r"
    done
  done
done
