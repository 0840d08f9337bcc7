"""Robustness probe: apply_gate_qr at odd (d, chi) hitting every QR path (pipelined pair,
tall pair with a ragged last outer block, outer-block QR above 5120 rows); checks the
isometries and the explicit error against a NumPy projection of theta."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_09782_b200 import model  # noqa: E402
from paper_2212_09782_b200 import qrtebd as q  # noqa: E402

ctx = q.Context(0)
for d, chi in [(5, 300), (5, 700), (3, 1200), (5, 1100), (4, 333)]:
    rng = np.random.default_rng(d * 1000 + chi)
    bm = model.random_right_isometry(rng, d, chi, chi)
    bn = model.random_right_isometry(rng, d, chi, chi)
    xi = np.diag(np.exp(-np.arange(chi) / (0.2 * chi))) + 1e-3 * (rng.standard_normal((chi, chi)))
    xi = xi / np.linalg.norm(xi)
    u = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
    pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
    up = q.apply_gate_qr(*[ctx.tensor(t) for t in (xi, bm, bn, u)], pol, ctx, want_left_iso=True)
    B = up.b_n.numpy()  # (d, eta, chi)
    A = up.left_iso.numpy()  # (d, chi, eta)
    eta = B.shape[1]
    Bm = B.transpose(1, 0, 2).reshape(eta, d * chi)
    Am = A.transpose(1, 0, 2).reshape(chi * d, eta)
    e1 = np.abs(Bm @ Bm.conj().T - np.eye(eta)).max()
    e2 = np.abs(Am.conj().T @ Am - np.eye(eta)).max()
    phi = np.einsum("xa,iag->xig", xi, bm, optimize=True).reshape(chi * d, chi) @ bn.transpose(1, 0, 2).reshape(chi, d * chi)
    theta = np.einsum("IJij,xijc->xIJc", u.reshape(d, d, d, d), phi.reshape(chi, d, d, chi), optimize=True).reshape(chi * d, d * chi)
    proj = Am @ (Am.conj().T @ theta @ Bm.conj().T) @ Bm
    eps_np = np.linalg.norm(theta - proj) ** 2 / np.linalg.norm(theta) ** 2
    eps = up.report.eps_trunc
    print(f"d={d} chi={chi} eta={eta}: isometry defects {e1:.1e} {e2:.1e}; eps {eps:.6e} numpy {eps_np:.6e} "
          f"rel {abs(eps - eps_np) / max(eps_np, 1e-300):.1e}")
    assert e1 < 1e-12 and e2 < 1e-12 and abs(eps - eps_np) <= 1e-8 * eps_np + 1e-20
print("odd sizes ok")
