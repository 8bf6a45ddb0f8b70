# kbench of the main library and every tools/_var variant (C4 unless CONFIG set)
python tools/kbench.py --reps 20 ${KB_ARGS} 2>&1 | tail -1 | sed 's/^/main: /'
for f in tools/_var/*.so; do
  AK_LIB_PATH=$PWD/$f python tools/kbench.py --reps 20 ${KB_ARGS} 2>&1 | tail -1 | sed "s|^|$(basename $f): |"
done
