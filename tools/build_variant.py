"""Build variant libraries for tuning: python tools/build_variant.py TAG DEF=VAL ...

Writes tools/_var/libaddkern_b200_TAG.so; load it with AK_LIB_PATH=<that path>.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2404_17344_b200.build import build  # noqa: E402

out = Path(__file__).resolve().parent / "_var" / f"libaddkern_b200_{sys.argv[1]}.so"
out.parent.mkdir(exist_ok=True)
print(build(out=out, defines=sys.argv[2:]))
