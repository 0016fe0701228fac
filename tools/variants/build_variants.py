"""Build forward-kernel tuning variants (experiments only) into tools/variants/.

usage: python tools/variants/build_variants.py NAME=DEF1,DEF2 ...
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2601_00551_b200 import _build  # noqa: E402

here = os.path.dirname(os.path.abspath(__file__))
for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    out = os.path.join(here, f"lib_{name}.so")
    _build.build(out=out, defines=tuple(d for d in defs.split(",") if d))
    print(out)
