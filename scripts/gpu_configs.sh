# one bench line per BASELINE config at N=1 (C2 is the headline; the others are recorded for coverage)
mkdir -p gpurun_out
TAG=${1:-r1}
for c in c1 c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg_$c.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/${TAG}_cfg_$c.log') if l.startswith('{')][-1])
print('$c', 'fps %.1f' % d['value'], 'blend_ms %.3f' % d['alpha_blend_ms'], 'e2e', d['e2e'] and round(d['e2e']['value'],1), 'N', d['frame_stats']['N'])" || tail -3 gpurun_out/${TAG}_cfg_$c.log
done
# opt-in ellipse-box coverage on the two single-view configs where it matters most
for c in c2 c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --coverage ellipse > gpurun_out/${TAG}_cfg_${c}_ellipse.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/${TAG}_cfg_${c}_ellipse.log') if l.startswith('{')][-1])
print('$c ellipse', 'fps %.1f' % d['value'], 'blend_ms %.3f' % d['alpha_blend_ms'], 'N', d['frame_stats']['N'])" || tail -3 gpurun_out/${TAG}_cfg_${c}_ellipse.log
done
