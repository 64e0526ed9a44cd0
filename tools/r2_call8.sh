# round-2 call 8: persistent-kernel crossover after the partials fix, update-kernel
# L1::no_allocate A/B, GPU suite
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c8_build.log 2>&1 || { tail -30 gpurun_out/c8_build.log; exit 1; }
( OMP_NUM_THREADS=14 python tools/oracle_records.py c5 --norm-maxit 60 --out gpurun_out/oracle_c5_gs2_v3.json > gpurun_out/c8_orc5.log 2>&1; echo "orc5 rc=$?" >> gpurun_out/c8_orc5.log ) &
ORC=$!
for na in 0 1; do
  IGS_UPDATE_NA=$na python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c8_bench_na$na.json 2> gpurun_out/c8_bench_na$na.err
  python -c "import json; d=json.load(open('gpurun_out/c8_bench_na$na.json')); print('na=$na', round(d['value'],1), d['kernels']['update'], d['clocks']['sm_mhz'])"
done
for na in 0 1; do
  IGS_UPDATE_NA=$na python tools/bdot_probe.py --n 16777216 --ps 10,50,100 --pads 0 --reps 5 > gpurun_out/c8_probe_na$na.jsonl 2>&1
done
paste -d' ' <(python -c "import json;[print(json.loads(l)['p'], round(json.loads(l)['update_gbs'])) for l in open('gpurun_out/c8_probe_na0.jsonl') if l[0]=='{']") <(python -c "import json;[print(round(json.loads(l)['update_gbs'])) for l in open('gpurun_out/c8_probe_na1.jsonl') if l[0]=='{']")
python tools/pc_crossover.py --Ns 200,256,300,384,420,443,470,512 --algs igs1,igs2 --ms 100,300 --reps 3 > gpurun_out/c8_pc_crossover.jsonl 2>&1
cat gpurun_out/c8_pc_crossover.jsonl | python -c "
import sys, json
for l in sys.stdin:
    if not l.startswith('{'): continue
    d = json.loads(l); print(d['N'], d['n'], d['alg'], d['m'], round(d['persistent'].get('it_s', 0)), round(d['graphs'].get('it_s', 0)), round(d['ratio'] or 0, 3))"
timeout 2400 python -m pytest tests -m gpu -q -k "not c5_k100" > gpurun_out/c8_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/c8_pytest.log
for i in $(seq 1 240); do kill -0 $ORC 2>/dev/null || break; sleep 15; done
wait $ORC
tail -c 1200 gpurun_out/c8_orc5.log
cp gpurun_out/oracle_c5_gs2_v3.json tests/golden/oracle_c5_gs2.json && \
timeout 1200 python -m pytest tests/test_gpu_solve.py -q -m gpu -k "c5_k100" > gpurun_out/c8_c5test.log 2>&1; echo "c5 test rc=$?"; tail -15 gpurun_out/c8_c5test.log
