"""Two steps of one config (C3 default) for an ncu launch list: python tools/cfg_launches.py C3"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2404_17344_b200 import configs
from paper_2404_17344_b200.fastsum import build_plan, fast_matvecs
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
wl = configs.CONFIGS[name]()
plan = build_plan(wl.spec, wl.window_set, "default", wl.data)
V = torch.as_tensor(wl.V, device="cuda")
for _ in range(2):
    fast_matvecs(plan, V, dell=True)
torch.cuda.synchronize()
print("ok", plan.geometries.n_items)
