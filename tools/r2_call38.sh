# round-2 call 38: final evidence at HEAD with the two-group tile block dot (p >= 16):
# default bench line, all configs x algorithms sweep, ncu launch list of the bench command,
# DRAM traffic per launch of the c4 iteration kernels at p = 10 / 50 / 100, slab proxy
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c38_build.log 2>&1 || { tail -30 gpurun_out/c38_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/c38_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c38_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c38_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/c38_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/c38_bench_reference.json 2> gpurun_out/c38_bench_reference.err; echo "reference arm rc=$?"; cut -c1-300 gpurun_out/c38_bench_reference.json
timeout 900 python bench.py > gpurun_out/c38_bench.json 2> gpurun_out/c38_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c38_bench.json')); print(d['value'], d['e2e']['value'], d['clocks'], {n: round(v['ms_per_step'],1) for n,v in d['kernels'].items()}, d.get('solve_to_1e-12'), d['roofline'], d['roofline_frac_iteration'])"
python -c "
import paper_2205_07805_b200 as P, workloads as W, json
s = P.Solver(W.config('c4').A); print(json.dumps(s.info())); s.close()" > gpurun_out/c38_c4_info.json 2>/dev/null
bash tools/sweep_r1.sh > /dev/null 2>&1; cp gpurun_out/sweep.jsonl gpurun_out/c38_sweep.jsonl
python -c "
import json
for l in open('gpurun_out/c38_sweep.jsonl'):
    if l.startswith('{'):
        d = json.loads(l); print(d['config'], d['alg'], round(d['it_s']), round(d['gbs_model']), d.get('reductions_per_solve'))"
timeout 600 python tools/slab_proxy.py > gpurun_out/c38_slab_proxy.json 2> gpurun_out/c38_slab_proxy.err; tail -3 gpurun_out/c38_slab_proxy.json | cut -c1-600
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c38_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/c38_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c38_ncu_launch.log 2>&1
echo "launch list rc=$?"
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
python tools/traffic_run.py --config c4 --k 100 > gpurun_out/c38_traffic_plain.log 2>&1 || exit 1
run() {  # cfg k kernel p skip
  ncu --metrics $M --clock-control none -k regex:$3 -s $5 -c 1 --csv \
      --log-file gpurun_out/c38_tr_${3}_${1}_p${4}.csv python tools/traffic_run.py --config $1 --k $2 > /dev/null 2>&1
}
for p in 10 50; do run c4 100 bdot_tma_kernel $p $((p-8)); run c4 100 update_kernel $p $((p+1)); done  # (the block dot below p = 8 is bdot_sw_kernel: the tile kernel's first launch is p = 8)
run c4 100 bdot_sw_kernel 100 4; run c4 100 update_kernel 100 101
for p in 10 50 99; do run c4 100 spmv_sell_diag_kernel $p $((p+1)); done
echo "traffic rc=$?"
