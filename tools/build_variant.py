"""Build a tuning variant of libspc5_b200.so with extra nvcc flags (experiments only).

usage: python tools/build_variant.py NAME [-DFOO=1 ...]
Writes variants/NAME/libspc5_b200.so; copy it over paper_2307_14774_b200/ to run it.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import __graft_entry__ as g  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
g.BUILD = g.ROOT / "build" / f"variant_{name}"
g.BUILD.mkdir(parents=True, exist_ok=True)
(g.ROOT / "variants" / name).mkdir(parents=True, exist_ok=True)
g.LIB = g.ROOT / "variants" / name / "libspc5_b200.so"
g.NVCC_FLAGS = g.NVCC_FLAGS + list(extra) + ["-Xptxas", "-v"]
print(g.build_native())
