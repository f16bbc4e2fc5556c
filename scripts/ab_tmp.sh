bash scripts/gpu_ab.sh ab19 base box2
TCGS_LIB=$PWD/paper_2505_24796_b200/_lib/exp_box2.so timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
