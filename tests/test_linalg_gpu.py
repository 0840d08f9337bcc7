"""K3 parity: device blocked Householder QR/LQ vs the oracle
(proj/src/linalg.cpp:40-64) and the known answers of
proj/tests/test_linalg.cc:45-112."""
import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import qrtebd as q

pytestmark = pytest.mark.gpu


def crand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def test_qr_known_answer(ctx):
    # [[3],[4]] -> Q = (0.6, 0.8), R = 5  (proj/tests/test_linalg.cc:51-58)
    Q, R = q.qr_reduced(np.array([[3.0], [4.0]], dtype=complex), ctx)
    assert np.allclose(Q.numpy(), [[0.6], [0.8]], atol=1e-15)
    assert np.allclose(R.numpy(), [[5.0]], atol=1e-14)


@pytest.mark.parametrize("m,n", [(8, 8), (40, 12), (100, 100), (130, 33), (500, 64), (1280, 256), (12, 40),
                                 (1, 1), (3, 1), (2000, 65),
                                 # tall panels: GEMM block reflectors (m > 2048), the register panel at
                                 # 14/20 rows per warp, and the grid-barrier panel (m > 5120)
                                 (3000, 40), (5120, 36), (6000, 40),
                                 # two-level blocking (outer blocks of 128 columns, m > 2048): several
                                 # outer blocks, a ragged last panel and outer block, the look-ahead split
                                 (3000, 300), (2100, 2100), (5120, 520), (2600, 129)])
def test_qr_matches_oracle(ctx, m, n):
    rng = np.random.default_rng(m * 31 + n)
    a = crand(rng, m, n)
    Q, R = q.qr_reduced(a, ctx)
    Qd, Rd = Q.numpy(), R.numpy()
    Qo, Ro = ref.qr_reduced(a)
    k = min(m, n)
    assert Qd.shape == (m, k) and Rd.shape == (k, n)
    # gauge-fixed QR is unique at full rank: compare directly (Appendix B (vi))
    assert np.linalg.norm(Qd - Qo) / np.sqrt(k) < 1e-12
    assert np.linalg.norm(Rd - Ro) / np.linalg.norm(Ro) < 1e-12
    assert np.allclose(np.diag(Rd).imag, 0.0) and np.all(np.diag(Rd).real >= 0)
    assert np.linalg.norm(Qd @ Rd - a) / np.linalg.norm(a) < 1e-13
    assert np.max(np.abs(Qd.conj().T @ Qd - np.eye(k))) < 1e-12


def test_lq_matches_oracle(ctx):
    rng = np.random.default_rng(5)
    a = crand(rng, 24, 90)
    L, Q = q.lq_reduced(a, ctx)
    Lo, Qo = ref.lq_reduced(a)
    assert np.linalg.norm(L.numpy() - Lo) / np.linalg.norm(Lo) < 1e-12
    assert np.linalg.norm(Q.numpy() - Qo) < 1e-11
    # LQ = adjoint of QR of the adjoint (proj/tests/test_linalg.cc:92-99)
    Q2, R2 = q.qr_reduced(a.conj().T, ctx)
    assert np.max(np.abs(L.numpy() - R2.numpy().conj().T)) < 1e-13


def test_qr_rank_deficient_zero_columns(ctx):
    # exactly-zero columns give tau = 0 (H = I): product-state starts
    a = np.zeros((6, 4), dtype=complex)
    a[0, 0] = 1.0
    a[1, 2] = 2.0 + 1.0j
    Q, R = q.qr_reduced(a, ctx)
    assert np.linalg.norm(Q.numpy() @ R.numpy() - a) < 1e-14
    assert np.all(np.isfinite(Q.numpy()))


def test_qr_deterministic(ctx):
    rng = np.random.default_rng(9)
    a = crand(rng, 700, 150)
    Q1, R1 = q.qr_reduced(a, ctx)
    Q2, R2 = q.qr_reduced(a, ctx)
    assert np.array_equal(Q1.numpy(), Q2.numpy()) and np.array_equal(R1.numpy(), R2.numpy())


def test_qr_nonfinite_is_input_error(ctx):
    a = np.ones((4, 3), dtype=complex)
    a[1, 1] = np.nan
    with pytest.raises(q.InputError):
        q.qr_reduced(a, ctx)
