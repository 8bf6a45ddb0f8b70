# per-kernel times of one config (CONFIG, default C5) for the main library and every tools/_var variant
CONFIG=${CONFIG:-C5}
python tools/cfg_kernels.py $CONFIG --reps 2 ${CFG_ARGS} 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print('main', round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if v['ms_per_step']>0.3})"
for f in tools/_var/*.so; do
  AK_LIB_PATH=$PWD/$f python tools/cfg_kernels.py $CONFIG --reps 2 ${CFG_ARGS} 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print('$(basename $f)', round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if v['ms_per_step']>0.3})"
done
