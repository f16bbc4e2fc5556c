# run the c2 bench against each experiment build: bash scripts/gpu_ab.sh <tag> name1 name2 ...
# (lone frames: value, per-stage ms; K7 = stage_ms.blend)
mkdir -p gpurun_out
TAG=$1; shift
CFG=${AB_CONFIG:-c2}
for rep in 1 2; do
  for n in "$@"; do
    TCGS_LIB=$PWD/paper_2505_24796_b200/_lib/exp_$n.so timeout 600 python bench.py --config $CFG --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-ablation --no-in-flight > gpurun_out/${TAG}_$n.$rep.log 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/${TAG}_$n.$rep.log') if l.startswith('{')][-1])
print('$n', 'fps %.1f' % d['value'], {k: round(v, 4) for k, v in d['stage_ms'].items()})"
  done
done
