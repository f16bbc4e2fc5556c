# K7 race evidence: compute-sanitizer on small frames + digests of frames under timing-perturbed builds
#   bash scripts/gpu_race.sh <tag>   (expects paper_2505_24796_b200/_lib/exp_{def,pw,sc,sp,s2}.so)
mkdir -p gpurun_out
TAG=${1:-r2}
for n in def pw sc sp s2; do
  TCGS_LIB=$PWD/paper_2505_24796_b200/_lib/exp_$n.so timeout 600 python scripts/race_perturb.py > gpurun_out/${TAG}_race_$n.log 2>&1
  echo "$n $(tail -1 gpurun_out/${TAG}_race_$n.log)"
done
bash scripts/gpu_sanitize.sh
for tool in memcheck racecheck synccheck; do mv gpurun_out/sanitize_$tool.log gpurun_out/${TAG}_sanitize_$tool.log; done
