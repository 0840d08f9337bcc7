"""apply_gate_qr at odd (d, chi) that hit every QR path -- the pipelined pair (1500 rows), the
tall pair with a ragged last outer block (3500 / 3600 rows), the outer-block QR above 5120 rows
(5500 rows), and a chi that is not a multiple of 8 (the 3-D tensor-map fallback of the GEMM):
both isometries to 1e-12 and the explicit truncation error against a NumPy projection of theta
(proj/src/gates.cpp:464-485) to 1e-8 relative."""
import numpy as np
import pytest

from paper_2212_09782_b200 import model
from paper_2212_09782_b200 import qrtebd as q

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,chi", [(5, 300), (5, 700), (3, 1200), (5, 1100), (4, 333)])
def test_apply_gate_qr_odd_sizes(ctx, d, chi):
    rng = np.random.default_rng(d * 1000 + chi)
    bm = model.random_right_isometry(rng, d, chi, chi)
    bn = model.random_right_isometry(rng, d, chi, chi)
    xi = np.diag(np.exp(-np.arange(chi) / (0.2 * chi))) + 1e-3 * rng.standard_normal((chi, chi))
    xi = xi / np.linalg.norm(xi)
    u = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
    pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
    up = q.apply_gate_qr(*[ctx.tensor(t) for t in (xi, bm, bn, u)], pol, ctx, want_left_iso=True)
    B = up.b_n.numpy()        # (d, eta, chi_r): rows of Q_n
    A = up.left_iso.numpy()   # (d, chi_l, eta): Q_m
    eta = B.shape[1]
    assert eta == chi
    Bm = B.transpose(1, 0, 2).reshape(eta, d * chi)
    Am = A.transpose(1, 0, 2).reshape(chi * d, eta)
    assert np.abs(Bm @ Bm.conj().T - np.eye(eta)).max() < 1e-12
    assert np.abs(Am.conj().T @ Am - np.eye(eta)).max() < 1e-12
    phi = np.einsum("xa,iag->xig", xi, bm, optimize=True).reshape(chi * d, chi) @ bn.transpose(1, 0, 2).reshape(
        chi, d * chi)
    theta = np.einsum("IJij,xijc->xIJc", u.reshape(d, d, d, d), phi.reshape(chi, d, d, chi),
                      optimize=True).reshape(chi * d, d * chi)
    proj = Am @ (Am.conj().T @ theta @ Bm.conj().T) @ Bm
    eps_np = np.linalg.norm(theta - proj) ** 2 / np.linalg.norm(theta) ** 2
    assert abs(up.report.eps_trunc - eps_np) <= 1e-8 * eps_np + 1e-20
