# Bench lines, a launch list and an ncu --set full capture of two whole C2 frames:
#   bash scripts/gpu_profile.sh <tag>
mkdir -p gpurun_out
TAG=${1:-r2}
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c2.jsonl 2> gpurun_out/${TAG}_bench_c2.err
timeout 900 python bench.py --config c5 --steps 10 --no-cpu-baseline > gpurun_out/${TAG}_bench_c5.jsonl 2> gpurun_out/${TAG}_bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-in-flight > gpurun_out/${TAG}_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -s 44 -c 44 -o gpurun_out/${TAG}_frame -f \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-in-flight > gpurun_out/${TAG}_frame.log 2>&1
tail -2 gpurun_out/${TAG}_frame.log
cut -c1-300 gpurun_out/${TAG}_bench_c2.jsonl
ls -la gpurun_out
