"""bench.py contract pieces that run without a GPU: the multi-GPU launcher's refusals,
identical config dicts in both arms, the reference arm's JSON line, and the
per-kernel roofline classification."""

import json
import os
import subprocess
import sys
from types import SimpleNamespace

from conftest import ROOT

sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True, env=e,
                          timeout=600)


def test_gpus_flag_refuses_without_devices_and_checks_world_size():
    out = _run(["--gpus", "2"])
    assert out.returncode == 2 and "needs 2 CUDA devices" in out.stderr
    out = _run(["--gpus", "1"], env={"WORLD_SIZE": "2"})
    assert out.returncode == 2 and "WORLD_SIZE=2" in out.stderr


def test_reference_arm_line_and_identical_config():
    out = _run(["--impl", "reference", "--n", "3000", "--steps", "1", "--warmup", "0"])
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "matvecs/s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    args = SimpleNamespace(gpus=1, shard="cell", n=3000)
    assert line["config"] == bench.config_dict(args)
    args8 = SimpleNamespace(gpus=8, shard="cell", n=3000)
    assert "8 GPUs" in bench.config_dict(args8)["parallelism"]


def test_kernel_roofline_bounds_by_arithmetic_intensity():
    peaks = {"fp64_tflops": 36.7, "hbm_gbs": 6537.0}
    lengths = [3, 3, 2, 2, 1, 1]
    rows = [1000] * 6
    rep = {"k_interp3c": (2, 2.0), "k_interp2r": (2, 0.2), "k_interp1r": (2, 0.02), "cufft_z2d<2>": (2, 0.01)}
    rf = bench.kernel_rooflines(rep, lengths, rows, 16, 1, peaks)
    assert set(rf) == {"k_interp3c", "k_interp2r", "k_interp1r"}
    assert rf["k_interp3c"]["bound"] == "fp64" and rf["k_interp2r"]["bound"] == "fp64"
    assert rf["k_interp1r"]["bound"] == "hbm"
    q1 = rf["k_interp1r"]
    assert abs(q1["alg_bytes_per_launch"] - 2000 * (8 + 8 * 16)) < 1e-6
    assert abs(q1["achieved_gbs"] - q1["alg_bytes_per_launch"] / (q1["ms_per_launch"] * 1e-3) / 1e9) < 1e-9
