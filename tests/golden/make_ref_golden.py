"""Generate tests/golden/ref_updates.npz: inputs and outputs of the
REFERENCE ITSELF (proj/src/gates.cpp apply_gate, compiled in place on the
Eigen-subset shim by oracle/Makefile -> oracle/_ref/ref_update) for a set of
two-site updates covering the hot-path branches (SURVEY.md Appendix D edge
cases): eta == chi (Y0 = B^n), expansion (Y0 = theta slice), truncation below
chi, rectangular bonds, product-state first gates (rank-deficient, chi = 1),
qr_sweeps = 2, explicit error on/off, skip_renormalize, target_eps, the CBE
scheme, and the SVD/EIG comparators.

    make -C oracle && python tests/golden/make_ref_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import qrtebd_oracle as ref  # noqa: E402
from oracle import refbin  # noqa: E402

OUT = os.path.join(HERE, "ref_updates.npz")

# (name, scheme, d, chi_l, chi_n, chi_r, input kind, policy overrides)
CASES = [
    ("qr_eta_eq_chi", "qr", 3, 16, 16, 16, "random", dict(chi_max=16, delta_chi_abs=0, delta_chi_rel=0.0)),
    ("qr_expand", "qr", 3, 16, 16, 16, "random", dict(chi_max=40, delta_chi_abs=8, delta_chi_rel=0.0)),
    ("qr_truncate", "qr", 4, 20, 20, 20, "random", dict(chi_max=12, delta_chi_abs=0, delta_chi_rel=0.0)),
    ("qr_rect", "qr", 3, 12, 18, 10, "random", dict(chi_max=18, delta_chi_abs=0, delta_chi_rel=0.0)),
    ("qr_explicit_off", "qr", 5, 12, 12, 12, "random",
     dict(chi_max=12, delta_chi_abs=0, delta_chi_rel=0.0, compute_explicit_error=False)),
    ("qr_sweeps2", "qr", 3, 16, 16, 16, "random", dict(chi_max=10, delta_chi_abs=0, delta_chi_rel=0.0, qr_sweeps=2)),
    ("qr_skip_renorm", "qr", 3, 16, 16, 16, "random",
     dict(chi_max=8, delta_chi_abs=0, delta_chi_rel=0.0, skip_renormalize=True)),
    ("qr_product_d5", "qr", 5, 1, 1, 1, "product", dict(chi_max=64, delta_chi_abs=100, delta_chi_rel=0.1)),
    ("qr_product_d2", "qr", 2, 1, 1, 1, "product", dict(chi_max=64)),
    ("qr_d10", "qr", 10, 8, 8, 8, "random", dict(chi_max=8, delta_chi_abs=0, delta_chi_rel=0.0)),
    ("cbe_expand", "qr_cbe", 3, 16, 16, 16, "diag", dict(chi_max=64, delta_chi_abs=8, delta_chi_rel=0.1)),
    ("cbe_truncate", "qr_cbe", 4, 16, 16, 16, "random", dict(chi_max=10, delta_chi_abs=4, delta_chi_rel=0.0)),
    ("cbe_target_eps", "qr_cbe", 3, 16, 16, 16, "random",
     dict(chi_max=64, delta_chi_abs=4, delta_chi_rel=0.0, target_eps=1e-6)),
    ("cbe_cutoff", "qr_cbe", 3, 16, 16, 16, "diag", dict(chi_max=64, sv_cutoff=1e-3, delta_chi_abs=8)),
    ("cbe_product_d5", "qr_cbe", 5, 1, 1, 1, "product", dict(chi_max=64, delta_chi_abs=100, delta_chi_rel=0.1)),
    ("cbe_explicit_off", "qr_cbe", 3, 12, 12, 12, "random",
     dict(chi_max=12, delta_chi_abs=4, delta_chi_rel=0.0, compute_explicit_error=False)),
    ("svd_truncate", "svd", 3, 16, 16, 16, "random", dict(chi_max=12)),
    ("eig_truncate", "eig", 3, 12, 12, 12, "random", dict(chi_max=9)),
]


def make_inputs(kind, d, chi_l, chi_n, chi_r, seed):
    rng = np.random.default_rng(seed)
    if kind == "product":
        v = np.zeros(d, dtype=complex)
        v[0] = 1
        bm = v.reshape(d, 1, 1).copy()
        bn = v.reshape(d, 1, 1).copy()
        xi = np.eye(1, dtype=complex)
    else:
        bm = ref.random_right_isometry(rng, d, chi_l, chi_n)
        bn = ref.random_right_isometry(rng, d, chi_n, chi_r)
        if kind == "diag":
            s = np.exp(-4.0 * np.arange(chi_l) / chi_l)
            xi = np.diag(s / np.linalg.norm(s)).astype(complex)
        else:
            xi = rng.standard_normal((chi_l, chi_l)) + 1j * rng.standard_normal((chi_l, chi_l))
            xi /= np.linalg.norm(xi)
    u = ref.make_gate(ref.bond_hamiltonian(d, 2.0), 0.05)
    return xi, bm, bn, u


def main():
    if not refbin.available():
        raise SystemExit("build the reference first: make -C oracle")
    arrays, meta = {}, []
    for i, (name, scheme, d, chi_l, chi_n, chi_r, kind, pol) in enumerate(CASES):
        xi, bm, bn, u = make_inputs(kind, d, chi_l, chi_n, chi_r, seed=1000 + i)
        r = refbin.apply_gate(scheme, xi, bm, bn, u, **pol)
        p = f"c{i}_"
        arrays.update({p + "xi": xi, p + "bm": bm, p + "bn": bn, p + "u": u, p + "out_bm": r.b_m,
                       p + "out_xi": r.xi_n, p + "out_bn": r.b_n})
        if r.left_iso is not None:
            arrays[p + "out_left"] = r.left_iso
        meta.append(dict(name=name, scheme=scheme, policy=pol, chi_before=r.chi_before, chi_expanded=r.chi_expanded,
                         chi_after=r.chi_after, eps_trunc=r.eps_trunc, discarded_weight=r.discarded_weight,
                         has_left=r.left_iso is not None))
        print(f"{name:18s} eta={r.chi_expanded:3d} kk={r.chi_after:3d} eps={r.eps_trunc:.3e}")
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
    print("->", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
