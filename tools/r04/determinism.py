"""Run the same DtN batch several times in one process and report leaves whose maps change
between runs (endgame sharing makes the run nondeterministic in timing, never in value).
    python tools/r04/determinism.py p leaves reps"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import bench
from paper_2503_04033_b200.engine import LeafEngine
p, L, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
tpl, pack = bench.make_shard(p, 16, 40.0, 0, 1, L)
eng = LeafEngine(tpl, False, True)
coeffs = torch.from_numpy(pack).cuda()
ref = None
bad = {}
for r in range(reps):
    out, stats = eng.dtn(coeffs)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    if ref is None:
        ref = o
        continue
    d = np.abs(o - ref).reshape(L, -1).max(1)
    for k in np.nonzero(d)[0]:
        bad.setdefault(int(k), []).append((r, float(d[k])))
print(json.dumps({"p": p, "leaves": L, "reps": reps, "lib": os.environ.get("HPS_LIB", "default"),
                  "changed_leaves": bad}))
