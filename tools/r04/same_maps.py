"""Diagnostics: DtN maps of two library builds on the same leaves, compared bit for bit.
    python tools/r04/same_maps.py LIB_A LIB_B [p] [leaves]"""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, ROOT)
    import numpy as np
    import bench
    from paper_2503_04033_b200.engine import LeafEngine
    p, L, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    tpl, pack = bench.make_shard(p, 16, 40.0, 0, 1, L)
    dtn, stats = LeafEngine(tpl, False, True).dtn_host(pack)
    np.save(out, dtn)
    sys.exit(0)
a, b = sys.argv[1], sys.argv[2]
p = sys.argv[3] if len(sys.argv) > 3 else "12"
L = sys.argv[4] if len(sys.argv) > 4 else "600"
import numpy as np
for lib, f in ((a, "/tmp/maps_a.npy"), (b, "/tmp/maps_b.npy")):
    subprocess.run([sys.executable, __file__, "--one", p, L, f], check=True, env=dict(os.environ, HPS_LIB=lib))
x, y = np.load("/tmp/maps_a.npy"), np.load("/tmp/maps_b.npy")
print(json.dumps({"p": int(p), "leaves": int(L), "identical": bool(np.array_equal(x, y)),
                  "max_abs_diff": float(np.abs(x - y).max())}))
