bash scripts/gpu_ab.sh ab20 base t192 t128
