# coverage modes side by side: bash scripts/gpu_coverage.sh <tag>
mkdir -p gpurun_out
TAG=$1
for c in c2 c5; do
  for m in square box ellipse; do
    timeout 900 python bench.py --config $c --steps 32 --warmup 8 --no-cpu-baseline --no-e2e --coverage $m > gpurun_out/${TAG}_${c}_$m.log 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/${TAG}_${c}_$m.log') if l.startswith('{')][-1])
print('$c $m', 'fps %.1f' % d['value'], 'N', d['frame_stats']['N'], d['stage_ms']['isolated'])" || tail -3 gpurun_out/${TAG}_${c}_$m.log
  done
done
