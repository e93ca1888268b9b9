"""Build a tuning variant of libhps_leaf.so with extra -D flags (diagnostics only):
    python tools/build_variant.py NAME -DHPS_SMALL_PANEL=16 ...
loaded by setting HPS_LIB=paper_2503_04033_b200/_lib/libhps_leaf_NAME.so."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_04033_b200 import _build as B
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(B.OUT), f"libhps_leaf_{name}.so")
res = subprocess.run([B.NVCC] + B.FLAGS + defs + ["-o", out, B.SRC], capture_output=True, text=True)
print(out if res.returncode == 0 else res.stderr[-3000:])
