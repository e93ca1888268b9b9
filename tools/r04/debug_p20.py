"""Which leaves differ between two builds at p = 20 (300 leaves), and which one matches the oracle."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
L = "paper_2503_04033_b200/_lib"
runs = [("head1", f"{L}/libhps_leaf.so"), ("head2", f"{L}/libhps_leaf.so"), ("op0", f"{L}/libhps_leaf_op0.so")]
for name, lib in runs:
    subprocess.run([sys.executable, os.path.join(ROOT, "tools/r04/same_maps.py"), "--one", "20", "300", f"/tmp/m_{name}.npy"],
                   check=True, env=dict(os.environ, HPS_LIB=lib))
m = {n: np.load(f"/tmp/m_{n}.npy") for n, _ in runs}
def diff(a, b):
    d = np.abs(m[a] - m[b]).reshape(len(m[a]), -1).max(1)
    return [int(i) for i in np.nonzero(d)[0]], float(d.max())
out = {"head1_vs_head2": diff("head1", "head2"), "head1_vs_op0": diff("head1", "op0"), "head2_vs_op0": diff("head2", "op0")}
print(json.dumps(out))
import bench
from oracle import hps_oracle as O
tpl, pack = bench.make_shard(20, 16, 40.0, 0, 1, 300)
otpl = O.OracleTemplate(tpl.widths, 20)
bad = sorted(set(out["head1_vs_op0"][0] + out["head1_vs_head2"][0] + out["head2_vs_op0"][0]))[:4]
for k in bad:
    ref, _, _ = O.leaf_dtn(otpl, pack[k, :3].T, None, pack[k, 3])
    print(k, {n: float(np.linalg.norm(m[n][k] - ref) / np.linalg.norm(ref)) for n, _ in runs})
