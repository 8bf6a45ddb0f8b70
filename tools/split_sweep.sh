# auto choice vs forced supercell edges (config-4 data at several N, config 3), adaptive chunks
for n in 30000 60000 125000 250000 500000 1000000; do
  for e in "cell_items3=2" "cell_items3=1" "dense_cells3=1e9,dense_cells3_interp=0" ""; do
    python tools/kbench.py --n $n --reps 20 --tuning "$e" | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print($n, '$e' or 'auto', d['items'], round(d['spread_ms'],4), round(d['interp_ms'],4))"
  done
done
python tools/kbench.py --config C3 --n 100000 --reps 20 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('C3 auto', d['items'], round(d['spread_ms'],4), round(d['interp_ms'],4))"
python tools/cfg_time.py
