for v in 0 1; do for b in 16 32; do
  echo "vreg=$v batch=$b"; AK_VREG=$v AK_BATCH3=$b timeout 300 python tools/kbench.py
done; done
