# round-2 call 5: GPU suite with the records (c4 gs=1 record pending), smoke, SpMV x-prefetch
# A/B, c3 with the column-sweep block dot, persistent-kernel crossover per algorithm / m
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c5_build.log 2>&1 || { tail -30 gpurun_out/c5_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -k "not (c4_as_specified and 1)" > gpurun_out/c5_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/c5_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c5_smoke.log 2>&1; echo "smoke rc=$?"
for x in 0 1; do
  IGS_SPMV_XPF=$x python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c5_bench_xpf$x.json 2> gpurun_out/c5_bench_xpf$x.err
  python -c "import json; d=json.load(open('gpurun_out/c5_bench_xpf$x.json')); print('xpf=$x', round(d['value'],1), d['kernels']['spmv'], d['clocks'])"
done
python tools/bench_configs.py --config c3 --k 300 > gpurun_out/c5_c3.json 2>&1; tail -c 1500 gpurun_out/c5_c3.json
python tools/pc_crossover.py --Ns 300,384,420,443,470,512 --algs igs1,igs2 --ms 100,300 --reps 3 > gpurun_out/c5_pc_crossover.jsonl 2>&1
cat gpurun_out/c5_pc_crossover.jsonl | python -c "
import sys, json
for l in sys.stdin:
    if not l.startswith('{'): continue
    d = json.loads(l); print(d['N'], d['n'], d['alg'], d['m'], d['persistent'].get('it_s'), d['graphs'].get('it_s'), d['ratio'])"
