# C4 kbench and C5 per-kernel times for the main library and every tools/_var variant
bash tools/gpu_var.sh
CFG_ARGS="${CFG_ARGS}" bash tools/gpu_var_cfg.sh
