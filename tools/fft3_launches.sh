# Warm (no cache flush) ncu launch times of the fused 3-D transform kernels, main
# library and every tools/_var variant (C4, K + dK/dl, two steps).
for lib in "" tools/_var/*.so; do
  tag=${lib:-main}
  AK_LIB_PATH=${lib:+$PWD/$lib} timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/l_$(basename $tag .so).csv python tools/cfg_launches.py C4 > /dev/null 2>&1
  echo "== $tag"
  python tools/launch_table.py gpurun_out/l_$(basename $tag .so).csv 2>/dev/null | grep -i "fft3"
done
