"""Host sparse backend (reference tests/test_sparse_backend.py strategy)."""

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2503_04033_b200 import sparse_backend as sb
from paper_2503_04033_b200.errors import ConfigError, StructurallySingularError


def test_identity_and_pivoting():
    f = sb.analyze_and_factor(sp.identity(5, format="csr"))
    assert np.allclose(sb.solve(f, np.arange(5.0)), np.arange(5.0))
    f = sb.analyze_and_factor(sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]])))
    assert np.allclose(sb.solve(f, np.array([1.0, 2.0])), [2.0, 1.0])


@pytest.mark.parametrize("seed", range(10))
def test_random_sparse_vs_dense(seed):
    rng = np.random.default_rng(seed)
    n = 50
    A = sp.random(n, n, density=0.1, random_state=seed, format="csr") + sp.identity(n) * 3
    b = rng.standard_normal(n)
    x = sb.solve(sb.analyze_and_factor(A), b)
    assert np.linalg.norm(A @ x - b) <= 1e-12 * np.linalg.norm(b) * 10


def test_structural_singularity_and_shape_errors():
    A = sp.csr_matrix(np.array([[1.0, 0.0], [0.0, 0.0]]))
    with pytest.raises(StructurallySingularError):
        sb.analyze_and_factor(A)
    f = sb.analyze_and_factor(sp.identity(3, format="csr"))
    with pytest.raises(ConfigError):
        sb.solve(f, np.ones(4))
    assert sb.analyze_and_factor(sp.csr_matrix((0, 0))).n == 0


def test_accumulator_sums_duplicates_and_dump():
    m = sb.SparseMatrix(3)
    m.add([0, 0, 2], [1, 1, 2], [1.0, 2.0, 5.0])
    m.add_block([1, 2], [0, 1], np.array([[1.0, 2.0], [3.0, 4.0]]))
    csr = m.finalize()
    assert csr[0, 1] == 3.0 and csr[2, 2] == 5.0 and csr[2, 1] == 4.0
    text = sb.dump_coo(csr)
    assert "0 1 3.0" in text
    with pytest.raises(ConfigError):
        m.add([0], [0], [1.0])
