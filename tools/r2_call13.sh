# round-2 call 13: grid-stride fused update (one wave of resident CTAs) A/B against the
# one-tile-per-CTA grid (IGS_UPDATE_WAVES=1000): update parity tests, isolated probes at the
# slab / c3 / c4 sizes, c4 bench, slab proxy, c3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c13_build.log 2>&1 || { tail -30 gpurun_out/c13_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -q -x -k "update or host or small_configs or c3_full" > gpurun_out/c13_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c13_tests.log
for w in 1000 1 2; do
  for n in 2097152 1048576 16777216; do
    IGS_UPDATE_WAVES=$w python tools/bdot_probe.py --n $n --ps 1,5,10,25,50,100 --pads 0 --reps 10 > gpurun_out/c13_probe_w${w}_n$n.jsonl 2>&1
  done
done
python - <<'PY'
import json
for n in (2097152, 1048576, 16777216):
    rows = {}
    for w in (1000, 1, 2):
        rows[w] = [json.loads(l) for l in open(f"gpurun_out/c13_probe_w{w}_n{n}.jsonl") if l.startswith("{")]
    for a, b, c in zip(rows[1000], rows[1], rows[2]):
        print(n, a["p"], "update us: one-tile %.1f  waves1 %.1f  waves2 %.1f" % (a["update_us"], b["update_us"], c["update_us"]))
PY
for w in 1000 1; do
  IGS_UPDATE_WAVES=$w python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c13_bench_w$w.json 2> gpurun_out/c13_bench_w$w.err
  python -c "import json; d=json.load(open('gpurun_out/c13_bench_w$w.json')); print('w=$w c4', round(d['value'],1), d['kernels']['update'], d['clocks']['sm_mhz'])"
  IGS_UPDATE_WAVES=$w python tools/slab_proxy.py > gpurun_out/c13_slab_w$w.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/c13_slab_w$w.json')); print('w=$w slab', d['plain']['it_s'], d['plain']['us_per_iteration'])"
  IGS_UPDATE_WAVES=$w python tools/bench_configs.py --config c3 --k 300 > gpurun_out/c13_c3_w$w.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c13_c3_w$w.json').read().strip().splitlines()[-1]); print('w=$w c3', round(d['it_s']))"
done
