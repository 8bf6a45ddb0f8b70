for c in 2048 4096 8192; do
  echo "chunk=$c"; AK_CHUNK3=$c AK_SUPERCELL3=2 timeout 300 python tools/kbench.py
done
