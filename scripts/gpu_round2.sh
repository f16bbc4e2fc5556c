# Round-2 evidence set on the final build: bash scripts/gpu_round2.sh <tag>
#   default bench lines (C2 headline + ablation, C5, C3 bands, C4 views), a launch list, an ncu --set full of
#   two whole C2 frames, and ncu of K7 for every alpha mode x EarlyCull on/off at C2 and C5 (the paper's ablation)
mkdir -p gpurun_out
TAG=${1:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c2.jsonl 2> gpurun_out/${TAG}_bench_c2.err
timeout 900 python bench.py --config c5 --steps 10 --no-cpu-baseline > gpurun_out/${TAG}_bench_c5.jsonl 2> gpurun_out/${TAG}_bench_c5.err
timeout 900 python bench.py --config c3 --steps 20 --no-cpu-baseline --no-ablation > gpurun_out/${TAG}_bench_c3.jsonl 2> gpurun_out/${TAG}_bench_c3.err
timeout 900 python bench.py --config c4 --steps 20 --no-cpu-baseline --no-ablation > gpurun_out/${TAG}_bench_c4.jsonl 2> gpurun_out/${TAG}_bench_c4.err
timeout 900 python bench.py --config c1 --steps 50 --no-cpu-baseline --no-ablation > gpurun_out/${TAG}_bench_c1.jsonl 2> gpurun_out/${TAG}_bench_c1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-in-flight > gpurun_out/${TAG}_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -s 44 -c 44 -o gpurun_out/${TAG}_frame -f \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-in-flight > gpurun_out/${TAG}_frame.log 2>&1
for cfg in c2 c5; do
  timeout 1500 ncu --set full --clock-control none -k regex:render_kernel -o gpurun_out/${TAG}_ablation_$cfg -f \
    python scripts/k7_ablation.py $cfg > gpurun_out/${TAG}_ablation_$cfg.log 2>&1
done
# summarise the reports here (gpurun copies back at most 64 MiB): JSON + markdown per report, then drop the reps
python scripts/ncu_summary.py gpurun_out/${TAG}_frame.ncu-rep gpurun_out/${TAG}_frame_ncu > /dev/null 2>&1
for cfg in c2 c5; do
  python scripts/ncu_summary.py gpurun_out/${TAG}_ablation_$cfg.ncu-rep gpurun_out/${TAG}_ablation_${cfg}_ncu > /dev/null 2>&1
done
python scripts/launch_table.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt 2>&1
rm -f gpurun_out/*.ncu-rep
python scripts/bench_summary.py gpurun_out/${TAG}_bench_c2.jsonl gpurun_out/${TAG}_bench_c5.jsonl 2>&1 | tail -30
ls -la gpurun_out | tail -30
