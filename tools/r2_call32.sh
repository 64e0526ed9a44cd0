# round-2 call 32: what limits the tile block dot at low SM clocks -- ncu --set full at base
# clocks (ncu's own --clock-control base) of bdot_tma_kernel and update_kernel at c4 p = 50
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c32_build.log 2>&1 || { tail -30 gpurun_out/c32_build.log; exit 1; }
python tools/traffic_run.py > gpurun_out/c32_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control base -k regex:bdot_tma_kernel -s 42 -c 1 -o gpurun_out/c32_bdot_base_p50 python tools/traffic_run.py > gpurun_out/c32_ncu1.log 2>&1; echo "ncu bdot base rc=$?"
ncu --set full --import-source on --clock-control base -k regex:update_kernel -s 51 -c 1 -o gpurun_out/c32_update_base_p50 python tools/traffic_run.py > gpurun_out/c32_ncu2.log 2>&1; echo "ncu update base rc=$?"
ncu --set full --import-source on --clock-control none -k regex:bdot_tma_kernel -s 42 -c 1 -o gpurun_out/c32_bdot_free_p50 python tools/traffic_run.py > gpurun_out/c32_ncu3.log 2>&1; echo "ncu bdot free rc=$?"
