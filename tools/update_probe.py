import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2212_09782_b200 import qrtebd as q, model
ctx = q.Context(0)
import os
d, chi = int(os.environ.get("D", 5)), int(os.environ.get("CHI", 256))
rng = np.random.default_rng(1)
bm = model.random_right_isometry(rng, d, chi, chi); bn = model.random_right_isometry(rng, d, chi, chi)
xi = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi)); xi /= np.linalg.norm(xi)
u = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
dev = [ctx.tensor(t) for t in (xi, bm, bn, u)]
pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
for i in range(4):
    q.apply_gate_qr(*dev, pol, ctx, want_left_iso=False)
