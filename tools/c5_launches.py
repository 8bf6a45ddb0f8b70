"""One config-5 step (mixed kernels, 16 RHS, K + per-window dK/dl) for the launch list."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2404_17344_b200 import configs
from paper_2404_17344_b200.fastsum import build_mixed_plan, mixed_matvecs
wl = configs.config5()
plan = build_mixed_plan(wl.specs, wl.window_set, "default", wl.data)
V = torch.as_tensor(wl.V, device="cuda")
for _ in range(2):
    mixed_matvecs(plan, V)
torch.cuda.synchronize()
print("ok")
