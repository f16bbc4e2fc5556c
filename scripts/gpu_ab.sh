# run the c2 bench against each experiment build: bash scripts/gpu_ab.sh <tag> name1 name2 ...
mkdir -p gpurun_out
TAG=$1; shift
for n in "$@"; do
  for rep in 1 2; do
    TCGS_LIB=$PWD/paper_2505_24796_b200/_lib/exp_$n.so timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_$n.$rep.log 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/${TAG}_$n.$rep.log') if l.startswith('{')][-1])
print('$n', 'fps %.1f' % d['value'], d['stage_ms'].get('isolated', d['stage_ms']))"
  done
done
