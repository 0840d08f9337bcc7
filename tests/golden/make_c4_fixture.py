"""Generate the C4 golden fixture (BASELINE.json configs[3]: d=5, chi=4096
single-bond stress, the bench_cell recipe proj/src/run.cpp:351-418 with
scheme qr, explicit error off): the oracle's update is too large to re-run
inside the GPU test (theta = 6.7 GB, ~20 min on 8 cores, ~35 GB host RAM), so
its gauge-invariant and gauge-fixed outputs are committed in compact form:

  s       Schmidt values of Xi~ (zgesdd), descending          (4096,)
  diag    diagonal of Xi~ = L/||L|| (gauge-fixed: real >= 0)  (4096,)
  qn_r    Q_n R: the gauge-fixed right isometry (grouped
          eta x (d chi_r)) times a seeded Gaussian R          (4096, 4)
  sketch  P^H (Xi_old B~m B~n) R: the gauge-invariant two-site
          block (proj/tests/test_gates.cc:32-37) sketched     (4, 4)
  eps, theta_norm, discarded, eta, chi_after

Inputs are regenerated from the seed by oracle.bench_cell_inputs (NumPy
PCG64 stream; LAPACK LQ of Gaussians).  Run:  python tests/golden/make_c4_fixture.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import qrtebd_oracle as ref  # noqa: E402

D, CHI = 5, 4096
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c4_qr_d5_chi4096.npz")


def sketch_mats(d, chi_l, chi_r, seed=0xC4):
    rng = np.random.default_rng(seed)
    p = rng.standard_normal((chi_l * d, 4)) + 1j * rng.standard_normal((chi_l * d, 4))
    r = rng.standard_normal((d * chi_r, 4)) + 1j * rng.standard_normal((d * chi_r, 4))
    return p, r


def block_sketch(xi_old, b_m, b_n, p, r):
    """P^H block R without forming the (chi d) x (d chi) block."""
    d, kk, chi_r = b_n.shape
    chi_l = xi_old.shape[0]
    t1 = np.einsum("jgx,jxc->gc", b_n, r.reshape(d, chi_r, 4))        # (kk, 4)
    t2 = np.einsum("ibg,gc->ibc", b_m, t1)                             # (d, chi_m, 4)
    out = np.einsum("ab,ibc->aic", xi_old, t2).reshape(chi_l * d, 4)   # (chi_l d, 4)
    return p.conj().T @ out


def qn_times_r(b_n, r):
    d, kk, chi_r = b_n.shape
    return np.einsum("jgx,jxc->gc", b_n, r.reshape(d, chi_r, 4))


def main():
    t0 = time.time()
    xi, bm, bn, gate, pol = ref.bench_cell_inputs(D, CHI, "qr")
    print(f"inputs {time.time() - t0:.1f} s", flush=True)
    o = ref.apply_gate_qr(xi, bm, bn, gate, pol)
    print(f"update {time.time() - t0:.1f} s", flush=True)
    p, r = sketch_mats(D, CHI, CHI)
    s = np.linalg.svd(o.xi_n, compute_uv=False)
    np.savez_compressed(OUT, s=s, diag=np.real(np.diag(o.xi_n)), qn_r=qn_times_r(o.b_n, r),
                        sketch=block_sketch(xi, o.b_m, o.b_n, p, r), eps=o.report.eps_trunc,
                        theta_norm=np.linalg.norm(xi) * 0 + np.sqrt(o.report.discarded_weight / o.report.eps_trunc)
                        if o.report.eps_trunc > 0 else 0.0,
                        discarded=o.report.discarded_weight, eta=o.report.chi_expanded, chi_after=o.report.chi_after)
    print(f"done {time.time() - t0:.1f} s -> {OUT}", flush=True)


if __name__ == "__main__":
    main()
