"""Same-GPU QR-TEBD vs SVD/EIG-TEBD.

One bench_cell update (proj/src/run.cpp:351-418 recipe: random right
isometries, Gaussian Xi, g=2, dt=0.05, chi_max=chi, cutoff 0, explicit error
off) timed on one B200 through:
  qr      the product path (qt_apply_gate_qr, device tensors)
  svd/eig the cuSOLVER comparators (paper_2212_09782_b200.comparators)
over the reference's bench grid (d = 5..20 at chi = 64) and a chi sweep at d = 5.
Prints one JSON line per cell.
"""
import argparse
import json
import time

import numpy as np
import torch

from paper_2212_09782_b200 import model
from paper_2212_09782_b200 import qrtebd as q
from paper_2212_09782_b200.comparators import apply_gate_eig_gpu, apply_gate_svd_gpu


def inputs(d, chi, seed=0x51AB):
    rng = np.random.default_rng([seed, d, chi])
    bm = model.random_right_isometry(rng, d, chi, chi)
    bn = model.random_right_isometry(rng, d, chi, chi)
    xi = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi))
    xi /= np.linalg.norm(xi)
    u = model.make_gate(model.bond_hamiltonian(d, 2.0, "bulk"), 0.05)
    return xi, bm, bn, u


def timed(fn, reps, sync):
    fn()
    sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    sync()
    return (time.perf_counter() - t0) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--max-chi", type=int, default=1024)
    a = ap.parse_args()
    ctx = q.Context(0)
    peak = ctx.fp64_peak(0)
    cells = [(d, 64) for d in (5, 8, 11, 14, 17, 20)] + [(5, c) for c in (128, 256, 512, 1024) if c <= a.max_chi]
    for d, chi in cells:
        xi, bm, bn, u = inputs(d, chi)
        pol = q.TruncationPolicy(chi_max=chi, sv_cutoff=0.0, compute_explicit_error=False, delta_chi_abs=0,
                                 delta_chi_rel=0.0)
        dev = [ctx.tensor(t) for t in (xi, bm, bn, u)]
        t_qr = timed(lambda: q.apply_gate_qr(*dev, pol, ctx, want_left_iso=False), a.reps, ctx.synchronize)
        tt = [torch.as_tensor(t, device="cuda") for t in (xi, bm, bn, u)]
        sync = torch.cuda.synchronize
        t_svd = timed(lambda: apply_gate_svd_gpu(*tt, pol), max(1, a.reps), sync)
        t_eig = timed(lambda: apply_gate_eig_gpu(*tt, pol), max(1, a.reps), sync)
        # algorithmic flops of the QR update (explicit error off, eta = kk = chi)
        f = 8.0 * (2 * d * d * chi ** 3 + d ** 4 * chi ** 2 + 3 * d * d * chi * chi * chi) + \
            2.0 * (16.0 * (d * chi) * chi * chi - 16.0 / 3.0 * chi ** 3)
        print(json.dumps({"d": d, "chi": chi, "qr_ms": t_qr * 1e3, "qr_updates_per_s": 1.0 / t_qr,
                          "qr_tflops": f / t_qr / 1e12, "qr_frac_of_dmma_peak": f / t_qr / 1e12 / peak,
                          "svd_ms": t_svd * 1e3, "eig_ms": t_eig * 1e3,
                          "svd_over_qr": t_svd / t_qr, "eig_over_qr": t_eig / t_qr}), flush=True)


if __name__ == "__main__":
    main()
