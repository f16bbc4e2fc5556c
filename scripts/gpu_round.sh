mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/r1_pytest_gpu.log
tail -5 gpurun_out/r1_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; tail -3 gpurun_out/r1_smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r1_bench.log 2>&1; tail -3 gpurun_out/r1_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r1_ncu_bench.log 2>&1; tail -2 gpurun_out/r1_ncu_bench.log
