bash scripts/gpu_ab.sh ab21 base bar2
TCGS_LIB=$PWD/paper_2505_24796_b200/_lib/exp_bar2.so timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
