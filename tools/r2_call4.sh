# round-2 call 4: column-sweep block dot (bdot_sw_kernel) A/B against the tile kernel:
# per-kernel parity with the sweep kernel forced, isolated probes at c3 / c4 shapes, c4 bench
mkdir -p gpurun_out
( python -c "import oracle; oracle.build(force=True)" && OMP_NUM_THREADS=14 python tools/oracle_records.py c5 --norm-maxit 60 --out gpurun_out/oracle_c5_gs2.json > gpurun_out/c4_orc5.log 2>&1; echo "orc5 rc=$?" >> gpurun_out/c4_orc5.log ) &
ORC=$!
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c4_build.log 2>&1 || { tail -30 gpurun_out/c4_build.log; exit 1; }
IGS_BDOT_SW_MIN_P=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "block_dot" > gpurun_out/c4_sw_tests.log 2>&1; echo "sw kernel tests rc=$?"; tail -3 gpurun_out/c4_sw_tests.log
for sw in 1000000 1; do
  IGS_BDOT_SW_MIN_P=$sw python tools/bdot_probe.py --n 1048576 --ps 1,5,10,50,100,150,200,250,300 --pads 0 > gpurun_out/c4_probe_c3_sw$sw.jsonl 2>&1
  IGS_BDOT_SW_MIN_P=$sw python tools/bdot_probe.py --n 16777216 --ps 1,5,10,25,50,75,100 --pads 0 --reps 5 > gpurun_out/c4_probe_c4_sw$sw.jsonl 2>&1
  IGS_BDOT_SW_MIN_P=$sw python tools/bdot_probe.py --n 2097152 --ps 1,5,10,25,50,100 --pads 0 --reps 20 > gpurun_out/c4_probe_slab_sw$sw.jsonl 2>&1
done
python - <<'PY'
import json
for shape in ("c3", "c4", "slab"):
    a = [json.loads(l) for l in open(f"gpurun_out/c4_probe_{shape}_sw1000000.jsonl") if l.startswith("{")]
    b = [json.loads(l) for l in open(f"gpurun_out/c4_probe_{shape}_sw1.jsonl") if l.startswith("{")]
    for x, y in zip(a, b):
        print(shape, x["p"], "tile %.0f us %.0f GB/s" % (x["bdot_us"], x["bdot_gbs"]), " sweep %.0f us %.0f GB/s" % (y["bdot_us"], y["bdot_gbs"]))
PY
for sw in 1000000 1; do
  IGS_BDOT_SW_MIN_P=$sw python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c4_bench_sw$sw.json 2> gpurun_out/c4_bench_sw$sw.err
  python -c "import json; d=json.load(open('gpurun_out/c4_bench_sw$sw.json')); print('sw=$sw', d['value'], d['kernels']['block_dot'])"
done
python tools/solve_gap2.py > gpurun_out/c4_solve_gap2.jsonl 2>&1; cat gpurun_out/c4_solve_gap2.jsonl
for i in $(seq 1 240); do kill -0 $ORC 2>/dev/null || break; free -g | sed -n 2p >> gpurun_out/c4_mem.txt; sleep 15; done
wait $ORC
tail -c 1500 gpurun_out/c4_orc5.log
