# GPU test suite + smoke(): bash scripts/gpu_tests.sh <tag> [pytest args]
mkdir -p gpurun_out
TAG=${1:-r2}; shift
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=25 "$@" > gpurun_out/${TAG}_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
tail -30 gpurun_out/${TAG}_gputests.log
tail -3 gpurun_out/${TAG}_smoke.log
