# A/B of a library build over stream/group configs: bash scripts/gpu_group2.sh <tag> <lib name|default> "s:g" ...
mkdir -p gpurun_out
TAG=$1; LIBN=$2; shift 2
if [ "$LIBN" != default ]; then export TCGS_LIB=$PWD/paper_2505_24796_b200/_lib/exp_$LIBN.so; fi
for cfg in "$@"; do
  s=${cfg%%:*}; g=${cfg##*:}
  timeout 600 python bench.py --steps 48 --warmup 8 --no-cpu-baseline --no-e2e --streams $s --view-group $g > gpurun_out/${TAG}_${LIBN}_s${s}g$g.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/${TAG}_${LIBN}_s${s}g$g.log') if l.startswith('{')][-1])
print('$LIBN streams $s group $g', 'fps %.1f' % d['value'], d['stage_ms'].get('isolated'))"
done
