"""The CPU oracle against golden vectors produced by the reference package itself.

Pins oracle/hps_oracle.py: assembled blocks bit-exact, DtN / S / reduced load /
interior solve within roundoff of the reference's own outputs.
"""

import os

import numpy as np
import pytest

from oracle import hps_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "leaf_cases.npz"))
CASES = sorted({k.split("/")[0] for k in G.files})


def unpack(name):
    d, p, hf, hz, leg, hc = (int(x) for x in G[name + "/meta"])
    c = G[name + "/coeffs"]
    a2 = c[:d].T
    k = d
    cross = None
    if hc:
        npair = d * (d - 1) // 2
        cross = c[k:k + npair].T
        k += npair
    a1 = None
    if hf:
        a1 = c[k:k + d].T
        k += d
    a0 = c[k] if hz else None
    tpl = O.OracleTemplate(G[name + "/widths"], p, "legendre" if leg else "drop")
    return tpl, a2, a1, a0, cross


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", CASES)
def test_template_bit_exact(name):
    tpl, *_ = unpack(name)
    assert np.array_equal(np.stack(tpl.D1), G[name + "/D"])
    assert np.array_equal(tpl.a_bi, G[name + "/a_bi"])
    assert rel(tpl.a_bb, G[name + "/a_bb"]) <= 1e-15
    if tpl.mode == "legendre":
        assert np.array_equal(tpl.Q, G[name + "/Q"])


@pytest.mark.parametrize("name", CASES)
def test_assembly_bit_exact(name):
    tpl, a2, a1, a0, cross = unpack(name)
    a_ii, a_ib = O.interior_blocks(tpl, a2, a1, a0, cross)
    assert np.array_equal(a_ii, G[name + "/a_ii"])
    # A_ib = R_b Q is a matmul in legendre mode: roundoff-level agreement only
    assert rel(a_ib, G[name + "/a_ib"]) <= (1e-15 if tpl.mode == "legendre" else 0.0)


@pytest.mark.parametrize("name", CASES)
def test_leaf_outputs_match_reference(name):
    tpl, a2, a1, a0, cross = unpack(name)
    dtn, s, (dmin, dmax, singular) = O.leaf_dtn(tpl, a2, a1, a0, cross)
    assert not singular and dmin > 0
    assert rel(dtn, G[name + "/dtn"]) <= 1e-13
    assert rel(s, G[name + "/s"]) <= 1e-13
    v, flux, _ = O.leaf_reduce_load(tpl, G[name + "/f"], a2, a1, a0, cross)
    assert rel(v, G[name + "/v"]) <= 1e-13
    assert rel(flux, G[name + "/flux"]) <= 1e-13
    u, _ = O.leaf_interior_solve(tpl, G[name + "/v"], G[name + "/ub"], a2, a1, a0, cross)
    assert rel(u, G[name + "/u_int"]) <= 1e-13


def test_dtn_flops_p20():
    n, m = 18 ** 3, 6 * 18 ** 2
    assert O.dtn_flops(n, m) == pytest.approx(2 / 3 * n ** 3 + 2 * n * n * m + 2 * n * m * m)


def test_singular_block_flagged():
    tpl = O.OracleTemplate((1.0, 1.0), 5)
    n = tpl.n
    _, _, (dmin, dmax, singular) = O.leaf_dtn(tpl, np.zeros((n, 2)), None, np.zeros(n))
    assert singular


# ---------------------------------------------------------------------------
# benchmark orders (configs[1-3]): p = 12, 16, 20 — fixtures from the reference
# itself (tests/golden/make_golden.py bench_cases)
# ---------------------------------------------------------------------------

B = np.load(os.path.join(HERE, "golden", "bench_cases.npz"))
BENCH_LEAVES = sorted({"/".join(k.split("/")[:2]) for k in B.files if k.count("/") == 2})


def bench_leaf(key):
    """(template widths, p, coefficient pack (4, n), probe R) of a bench fixture leaf."""
    name = key.split("/")[0]
    p, boxes, _ = B[name + "/meta"]
    h = 1.0 / boxes
    return (h, h, h), int(p), B[key + "/coeffs"], B[name + "/R"]


@pytest.mark.parametrize("key", BENCH_LEAVES)
def test_oracle_matches_reference_at_bench_orders(key):
    widths, p, c, R = bench_leaf(key)
    tpl = O.OracleTemplate(widths, p)
    dtn, s, (dmin, dmax, singular) = O.leaf_dtn(tpl, c[:3].T, None, c[3])
    assert not singular
    assert rel(dtn @ R, B[key + "/dtn_R"]) <= 1e-13
    assert rel(dtn[B[key + "/dtn_rows_idx"]], B[key + "/dtn_rows"]) <= 1e-13
    assert abs(np.linalg.norm(dtn) / B[key + "/dtn_fro"][0] - 1.0) <= 1e-13
    assert rel(s @ R, B[key + "/s_R"]) <= 1e-13
    # same LAPACK partial pivoting: the same pivots and interchange count
    pmin, pmax, swaps = B[key + "/pivots"]
    assert dmin == pytest.approx(pmin, rel=1e-12) and dmax == pytest.approx(pmax, rel=1e-12)
    v, flux, _ = O.leaf_reduce_load(tpl, B[key + "/f"], c[:3].T, None, c[3])
    assert rel(v, B[key + "/v"]) <= 1e-13
    assert rel(flux, B[key + "/flux"]) <= 1e-13
    u, _ = O.leaf_interior_solve(tpl, B[key + "/v"], B[key + "/ub"], c[:3].T, None, c[3])
    assert rel(u, B[key + "/u_int"]) <= 1e-13


def test_bench_fixtures_match_bench_workload():
    """bench.py's synthetic coefficient packs are the reference's fields at the same
    leaves: the fixtures check exactly the bench workload."""
    import bench
    for key in BENCH_LEAVES:
        name, leaf = key.split("/")
        p, boxes, kappa = B[name + "/meta"]
        idx = tuple(int(x) for x in leaf.split("_"))
        field = "const" if "const" in name else "bump"
        _, pack = bench.make_shard(int(p), int(boxes), float(kappa), 0, 1, field=field,
                                   leaf_ids=[int(np.ravel_multi_index(idx, (int(boxes),) * 3))])
        assert np.allclose(pack[0], B[key + "/coeffs"], rtol=1e-15, atol=0.0)
