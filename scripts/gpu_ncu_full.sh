# ncu --set full capture of the frame's kernels (K1, K2/K5 radix downsweeps, K4, K7) at config c2.
mkdir -p gpurun_out
TAG=${1:-r1}
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"render_kernel|preprocess_kernel|duplicate_keys|radix_downsweep|radix_upsweep|tile_ranges" -s 0 -c 18 \
  -o gpurun_out/${TAG}_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_full.log 2>&1
tail -3 gpurun_out/${TAG}_full.log
ls -la gpurun_out
