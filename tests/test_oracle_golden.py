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
