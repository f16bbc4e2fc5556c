mkdir -p gpurun_out
for s in ${STREAMS:-1 2 3}; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --streams $s > gpurun_out/st_$s.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/st_$s.log') if l.startswith('{')][-1])
print('streams $s', 'fps %.1f' % d['value'], {k: round(v, 4) for k, v in d['stage_ms'].items()}, d['gpu_launches'])"
done
