"""Build libapo_b200.so with extra nvcc -D flags into build_variants/<name>.so (A/B experiments; load with
APO_LIB=build_variants/<name>.so)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14982_b200 import _lib

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(_lib.ROOT, "build_variants")
os.makedirs(out, exist_ok=True)
_lib.NVCC_FLAGS = _lib.NVCC_FLAGS + defs
_lib.LIB_PATH = os.path.join(out, name + ".so")
saved = _lib.PKG_DIR
_lib.PKG_DIR = os.path.join(out, name + "_obj")
os.makedirs(_lib.PKG_DIR, exist_ok=True)
_lib.build(force=True)
print("built", _lib.LIB_PATH)
