# round-2 call 36: L2 zig-zag experiment (-DL2_ZIGZAG=1: V and A streams evict-first, the SpMV
# walks the rows backwards so it meets the x rows the update wrote last) vs the default build
mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct"
for v in 1 0 1 0; do
  IGS_NVCC_EXTRA=-DL2_ZIGZAG=$v python -c "from paper_2205_07805_b200 import build; build.build(force=True)" > gpurun_out/c36_build_$v.log 2>&1 || { tail -30 gpurun_out/c36_build_$v.log; exit 1; }
  if [ $v = 1 ]; then timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "sell or spmv or update or block_dot" > gpurun_out/c36_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/c36_tests.log; fi
  python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-solve > gpurun_out/c36_bench_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c36_bench_$v.json')); k=d['kernels']; print('zigzag=$v c4', round(d['value'],1), 'spmv', round(k['spmv']['ms_per_step'],2), 'bdot', round(k['block_dot']['ms_per_step'],2), 'upd', round(k['update']['ms_per_step'],2), 'step', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
for v in 1 0; do
  IGS_NVCC_EXTRA=-DL2_ZIGZAG=$v python -c "from paper_2205_07805_b200 import build; build.build(force=True)" > /dev/null 2>&1
  python tools/traffic_run.py > /dev/null 2>&1
  ncu --metrics $M --clock-control none -k regex:spmv_sell_diag_kernel -s 51 -c 1 --csv --log-file gpurun_out/c36_spmv_$v.csv python tools/traffic_run.py > /dev/null 2>&1
  ncu --metrics $M --clock-control none -k regex:bdot_tma_kernel -s 42 -c 1 --csv --log-file gpurun_out/c36_bdot_$v.csv python tools/traffic_run.py > /dev/null 2>&1
  for k in spmv bdot; do python - gpurun_out/c36_${k}_$v.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
h = rows[0]
print(sys.argv[1], {r[h.index("Metric Name")]: r[h.index("Metric Value")] for r in rows[1:]})
PY
  done
done
