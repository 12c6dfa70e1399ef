"""Build tuning variants of the native library (same sources, different -D
knobs) under paper_2210_12924_b200/lib/variants/<name>.so; select one at run
time with MP_LIB=<path> (tools/gpu/variants.sh). Tuning only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_12924_b200 import build as b  # noqa: E402

VARIANTS = {}
for arg in sys.argv[1:]:  # name=-DA=1,-DB=2
    name, _, defs = arg.partition("=")
    VARIANTS[name] = [d for d in defs.split(",") if d]
for name, defs in VARIANTS.items():
    lib = os.path.join(b.LIBDIR, "variants", name + ".so")
    b.build(defines=defs, lib=lib, objdir=os.path.join(b.ROOT, "build", "obj_" + name))
    print(lib)
