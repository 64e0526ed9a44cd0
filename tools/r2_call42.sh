# round-2 call 42: where two block-dot consumer groups start to pay: isolated probes at
# p = 12 .. 32 (c4, one c4 slab, c3 rows), default (two groups from p = 16) vs IGS_BDOT_GROUPS=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c42_build.log 2>&1 || { tail -30 gpurun_out/c42_build.log; exit 1; }
for i in 1 2; do for gp in 0 1; do for n in 16777216 2097152 1048576; do
  IGS_BDOT_GROUPS=$gp python tools/bdot_probe.py --n $n --ps 12,15,16,18,20,24,32 --pads 0 --reps 20 2>/dev/null | python -c "
import sys, json
r = [json.loads(l) for l in sys.stdin if l.startswith('{')]
print('groups_forced=$gp run $i n=$n', [(x['p'], round(x['bdot_us'], 1)) for x in r])"
done; done; done
