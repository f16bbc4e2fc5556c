# fused-K1 view groups vs one K1 per view (c2): bash scripts/gpu_group.sh <tag> "streams:group" ...
mkdir -p gpurun_out
TAG=$1; shift
for rep in 1 2; do
for cfg in "$@"; do
  s=${cfg%%:*}; g=${cfg##*:}
  timeout 600 python bench.py --steps 48 --warmup 8 --no-cpu-baseline --no-e2e --streams $s --view-group $g > gpurun_out/${TAG}_s${s}g$g.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/${TAG}_s${s}g$g.log') if l.startswith('{')][-1])
print('streams $s group $g', 'fps %.1f' % d['value'], d['stage_ms'].get('isolated'))"
done
done
