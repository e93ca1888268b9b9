"""First-contact check: one leaf per golden case through every mode, errors printed."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_04033_b200.engine import LeafEngine
from paper_2503_04033_b200.local_ops import LeafTemplate
G = np.load("tests/golden/leaf_cases.npz")
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
for name in sorted({k.split('/')[0] for k in G.files}):
    d, p, hf, hz = (int(x) for x in G[name + '/meta'])
    eng = LeafEngine(LeafTemplate(G[name + '/widths'], p, 'drop', False), bool(hf), bool(hz))
    c = G[name + '/coeffs'][None]
    dtn, st = eng.dtn_host(c)
    s, _ = eng.solution_operator_host(c)
    v, fl, _ = eng.reduce_load_host(c, G[name + '/f'][None])
    u, _ = eng.interior_solve_host(c, G[name + '/ub'][None], G[name + '/v'][None])
    print(f"{name:12s} dtn {rel(dtn[0], G[name+'/dtn']):.2e} s {rel(s[0], G[name+'/s']):.2e} "
          f"v {rel(v[0], G[name+'/v']):.2e} flux {rel(fl[0], G[name+'/flux']):.2e} "
          f"u {rel(u[0], G[name+'/u_int']):.2e} piv {st[0]}", flush=True)
