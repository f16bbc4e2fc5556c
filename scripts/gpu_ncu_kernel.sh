# ncu --set full of one kernel family: bash scripts/gpu_ncu_kernel.sh <tag> <regex> <skip> <count> [bench args...]
mkdir -p gpurun_out
TAG=$1; RX=$2; SKIP=$3; CNT=$4; shift 4
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SKIP -c $CNT \
  -o gpurun_out/${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${TAG}.log 2>&1
tail -2 gpurun_out/${TAG}.log
