"""Builds A/B variants of the C-ABI library with extra -D flags into
paper_2507_01631_b200/_variants/<name>/ (git-ignored, travels with gpurun);
select one at run time with TFG_LIB=<path>.

usage: python tools/variants.py name=DEF1,DEF2 [name2=...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_01631_b200 import build as B  # noqa: E402

for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    d = os.path.join(B.HERE, "_variants", name)
    lib = B.build(force=True, defines=[x for x in defs.split(",") if x], out=os.path.join(d, "libtilefield_gpu.so"),
                  build_dir=os.path.join(d, "_build"))
    print(lib)
