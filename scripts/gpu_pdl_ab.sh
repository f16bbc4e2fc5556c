# A/B of programmatic dependent launch: C2 bench with TCGS_PDL=0 and 1, twice each (no CPU leg / e2e / ablation)
mkdir -p gpurun_out
TAG=${1:-pdl}
for rep in 1 2; do
  for v in 0 1; do
    TCGS_PDL=$v timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e --no-ablation > gpurun_out/${TAG}_pdl${v}_${rep}.jsonl 2>&1
    python -c "import json,sys; d=json.loads([l for l in open('gpurun_out/${TAG}_pdl${v}_${rep}.jsonl') if l.startswith('{')][-1]); print('PDL=$v', round(d['value'],1), 'ms', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stage_ms'].items()}, 'inflight', round(d['views_in_flight']['value'],1))"
  done
done
