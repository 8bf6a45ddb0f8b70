for n in 30000 125000; do
  for c in 2048 512 256 128; do
    for s in 1 2; do
      python tools/kbench.py --n $n --reps 20 --tuning cell_items3=$s,chunk3=$c | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print($n, 'S$s', 'chunk $c', d['items'], round(d['spread_ms'],4), round(d['interp_ms'],4))"
    done
  done
done
for c in 2048 512 256 128; do
  for s in 1 2; do
    python tools/kbench.py --tuning cell_items3=$s,chunk3=$c --config C3 --n 100000 --reps 20 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('C3', 'S$s', 'chunk $c', d['items'], round(d['spread_ms'],4), round(d['interp_ms'],4))"
  done
done
