# Profile the experimental fused wavefront kernel (c4, IGS_FUSED=1)
export IGS_FUSED=1
python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain_fused.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fused_kernel" -s 140 -c 2 -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_fused.log 2>&1
echo full rc=$?
