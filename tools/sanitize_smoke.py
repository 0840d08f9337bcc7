"""Smoke-size workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family of the hot path once, small.

  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py

Covers: the sequential QR update with left_iso (panel + block reflectors),
the pipelined QR pair (six streams, cluster panels, DSMEM multi-reflector
updates, Q blocks), CBE (Gram + cooperative Jacobi eigensolver + kept
selection), the Jordan-Wielandt spectra, a CUDA-graph uniform step (L=2)
and concurrent same-parity updates (L=4), the reference-exact finite chain
(gauge moves) and the observables.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import qrtebd_oracle as ref  # noqa: E402
from paper_2212_09782_b200 import model  # noqa: E402
from paper_2212_09782_b200 import qrtebd as q  # noqa: E402
from paper_2212_09782_b200._capi import Context  # noqa: E402


def inputs(rng, d, chi):
    bm = ref.random_right_isometry(rng, d, chi, chi)
    bn = ref.random_right_isometry(rng, d, chi, chi)
    xi = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi))
    return xi / np.linalg.norm(xi), bm, bn


def main():
    rng = np.random.default_rng(7)
    with Context(0) as ctx:
        for d, chi, left in ((3, 16, True), (5, 64, False), (5, 40, True)):
            xi, bm, bn = inputs(rng, d, chi)
            u = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
            pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
            q.apply_gate_qr(xi, bm, bn, u, pol, ctx, want_left_iso=left)
        xi, bm, bn = inputs(rng, 3, 16)
        u = model.make_gate(model.bond_hamiltonian(3, 2.0), 0.05)
        q.apply_gate_qr_cbe(xi, bm, bn, u, q.TruncationPolicy(chi_max=24, delta_chi_abs=6), ctx)
        g = rng.standard_normal((40, 40)) + 1j * rng.standard_normal((40, 40))
        q.eigh(g + g.conj().T, ctx)
        m = (np.linalg.qr(rng.standard_normal((24, 24)))[0] * np.logspace(0, -14, 24)) @ np.eye(24)
        q.schmidt_values_of(m.astype(complex), ctx)
        for L in (2, 4):
            d, chi = 3, 12
            sites = [ref.random_right_isometry(rng, d, chi, chi) for _ in range(L)]
            bonds = [inputs(rng, d, chi)[0] for _ in range(L)]
            st = q.UniformMPS.from_numpy(ctx, d, sites, bonds)
            sched = [(p, ctx.tensor(gg)) for p, gg in model.trotter_schedule(model.bond_hamiltonian(d, 2.0), 0.05, 2)]
            dev = q.DeviceUniformMPS(st, ctx)
            pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
            for _ in range(4):
                dev.step(sched, "qr", pol)
            snap = dev.snapshot()
            q.expectation_local(snap, ref.clock_operators(d)[0], 0, ctx)
            q.check_isometric(snap, 1e-10, ctx)
            dev.close()
        d, n = 2, 6
        v = np.zeros(d, dtype=complex)
        v[0] = 1
        f = q.product_state_finite(d, n, v, ctx)
        layers = [(p, [ctx.tensor(gg) for gg in gs]) for p, gs in ref.finite_layers(d, 1.5, n, 0.1, 2)]
        for scheme in ("qr", "qr_cbe"):
            f = q.tebd_step_finite(f, layers, scheme, q.TruncationPolicy(chi_max=4))[0]
        q.finite_observables(f, ref.clock_operators(d)[0])
        ctx.synchronize()
    print("sanitize smoke done")


if __name__ == "__main__":
    main()
