"""Memory-safety evidence without compute-sanitizer (closed on this GPU pool): the
checked library variant (-DAK_CHECKED, paper_2404_17344_b200/build.py build_checked)
traps on device-side invariant violations (grid wrap ranges, local cell offsets,
region-tile indices), surrounds every buffer the library allocates with guard bands
verified after each entry point, and poisons fresh buffers with NaN bytes so a read
of memory no kernel wrote shows up in the results.  tools/sanitize_cases.py drives
every kernel family (dense / sparse / masked / many-RHS / mixed plans, NUFFTs,
dense products) through it and checks each result against the oracle."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_checked_build_runs_every_kernel_family_clean(cuda):
    from paper_2404_17344_b200.build import build_checked

    lib = build_checked()
    env = dict(os.environ, AK_LIB_PATH=str(lib))
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_cases.py")], env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "SANITIZE_CASES_OK" in out.stdout
    assert "AK_DCHECK" not in out.stdout + out.stderr
