# per-kernel times of one config (CONFIG, default C5) for the main library and every tools/_var variant
# (kernels above MINMS ms per step, default 0.3, or matching KSEL)
CONFIG=${CONFIG:-C5}
SEL="v['ms_per_step']>${MINMS:-0.3} or '${KSEL:-@@}' in k"
python tools/cfg_kernels.py $CONFIG --reps 2 ${CFG_ARGS} 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print('main', round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if $SEL})"
for f in tools/_var/*.so; do
  AK_LIB_PATH=$PWD/$f python tools/cfg_kernels.py $CONFIG --reps 2 ${CFG_ARGS} 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print('$(basename $f)', round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if $SEL})"
done
