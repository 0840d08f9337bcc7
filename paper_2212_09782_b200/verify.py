"""Invariant verification suite on the device.

Mirrors run_verify / finite_quench_max_z_error (proj/src/run.cpp:500-696) and
VerifyReport (proj/include/qrtebd/run.hpp:111-126).  Every TEBD step,
isometry check, expectation value and Schmidt spectrum runs on the device
through the C-ABI.  The reference runs several lanes with its CPU SVD/EIG
schemes; the device has the QR schemes only, so those lanes run `qr` (where
the reference used `svd`) and the cross-scheme check compares `qr` with
`qr_cbe`.  The exact-diagonalization comparison state (ed_* below, the
reference's EdEvolver, proj/src/clock.cpp:118-172) is a small dense host
computation, as in the reference: it is the yardstick of the suite, not part
of the TEBD path.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import model
from .qrtebd import (Context, DeviceUniformMPS, TruncationPolicy, check_isometric, check_isometric_finite,
                     default_context, finite_observables, product_state_finite, product_state_uniform,
                     schmidt_values_of, tebd_step_finite)
from . import _capi

__all__ = ["VerifyCheck", "VerifyReport", "run_verify", "finite_quench_max_z_error"]


@dataclass
class VerifyCheck:
    name: str
    passed: bool
    value: float
    threshold: float


@dataclass
class VerifyReport:
    """VerifyReport, proj/include/qrtebd/run.hpp:111-121."""

    checks: List[VerifyCheck] = field(default_factory=list)

    def all_pass(self) -> bool:
        return all(c.passed for c in self.checks)

    def to_json(self) -> str:
        """run.cpp:536-546."""
        j = {"checks": [{"name": c.name, "pass": c.passed, "value": c.value, "threshold": c.threshold}
                        for c in self.checks], "pass": self.all_pass()}
        return json.dumps(j, indent=2, sort_keys=True) + "\n"


# ----------------------------------------------------------------- exact diagonalization (clock.cpp:118-189)
def _global_hamiltonian(d: int, n: int, g: float) -> np.ndarray:
    """global_hamiltonian, clock.cpp:118-135: -sum (Z Z^dag + h.c.) - g sum (X + X^dag)."""
    z, x = model.clock_operators(d)
    zz = np.kron(z, z.conj().T)
    zz = zz + zz.conj().T
    onsite = g * (x + x.conj().T)
    dim = d ** n
    h = np.zeros((dim, dim), dtype=np.complex128)
    for s in range(n - 1):
        h -= np.kron(np.kron(np.eye(d ** s), zz), np.eye(d ** (n - s - 2)))
    for s in range(n):
        h -= np.kron(np.kron(np.eye(d ** s), onsite), np.eye(d ** (n - s - 1)))
    return h


def _ed_z(psi: np.ndarray, d: int, n: int) -> np.ndarray:
    """<Z_n> of a state vector, ed_observables (clock.cpp:174-193)."""
    zdiag = np.diag(model.clock_operators(d)[0])
    w = (np.abs(psi) ** 2).reshape([d] * n)
    return np.array([np.tensordot(np.sum(w, axis=tuple(a for a in range(n) if a != s)), zdiag, axes=1)
                     for s in range(n)])


def finite_quench_max_z_error(d: int, n_sites: int, g: float, dt: float, t_max: float, order: int, scheme: str,
                              chi_max: int, ctx: Context = None) -> float:
    """finite_quench_max_z_error, run.cpp:500-528: max over steps and sites of
    |<Z_n>_TEBD - <Z_n>_ED| for the quench from the Z=1 product state."""
    ctx = ctx or default_context()
    mps = product_state_finite(d, n_sites, model.z1_local_vector(d), ctx)
    layers = [(p, [ctx.tensor(model.make_gate(model.chain_bond_hamiltonian(d, g, b, n_sites), dte))
                   for b in range(n_sites - 1)])
              for p, dte in model.layer_structure(dt, order)]
    w, v = np.linalg.eigh(_global_hamiltonian(d, n_sites, g))
    step = (v * np.exp(-1j * dt * w)) @ v.conj().T
    psi = np.zeros(d ** n_sites, dtype=np.complex128)
    psi[0] = 1.0
    z_op = ctx.tensor(model.clock_operators(d)[0])
    pol = TruncationPolicy(chi_max=chi_max, sv_cutoff=1e-14)
    max_err = 0.0
    for _ in range(int(math.floor(t_max / dt + 1e-9))):
        tebd_step_finite(mps, layers, scheme, pol, in_place=True)
        psi = step @ psi
        zs, _ = finite_observables(mps, z_op)
        max_err = max(max_err, float(np.max(np.abs(zs - _ed_z(psi, d, n_sites)))))
    return max_err


def _uniform_trace(d: int, scheme: str, dt: float, t_max: float, chi_max: int, ctx: Context,
                   skip_renormalize: bool = False):
    """Uniform L=2 quench on the device: per step <Z_s>, S_b, Schmidt norms and
    the isometry defect (run.cpp:583-630, :650-693)."""
    st = DeviceUniformMPS(product_state_uniform(d, 2, model.z1_local_vector(d), ctx), ctx)
    sched = [(p, ctx.tensor(u)) for p, u in model.trotter_schedule(model.bond_hamiltonian(d, 2.0, "bulk"), dt, 2)]
    pol = TruncationPolicy(chi_max=chi_max, sv_cutoff=1e-14, skip_renormalize=skip_renormalize)
    z_op = ctx.tensor(model.clock_operators(d)[0])
    zs, ss, defects, drifts = [], [], [], []
    out = (_capi.C.c_double * 2)()
    for _ in range(int(math.floor(t_max / dt + 1e-9))):
        st.step(sched, scheme, pol)
        snap = st.snapshot()
        for s in range(2):
            bv, sv = st.view("bond", s), st.view("site", s)
            _capi.check(ctx.lib.qt_expectation_local(ctx.h, bv.h, sv.h, z_op.h, out))
            zs.append(out[0])
            spec = schmidt_values_of(bv, ctx)
            ss.append(float(-sum(p * math.log(p) for p in spec ** 2 if p > 0.0)))
            drifts.append(abs(float(np.sum(spec ** 2)) - 1.0))
        defects.append(check_isometric(snap, 1e-10, ctx).max_defect())
    return np.array(zs), np.array(ss), max(defects), max(drifts)


def run_verify(fault_skip_renormalize: bool = False, ctx: Context = None) -> VerifyReport:
    """run_verify, proj/src/run.cpp:548-696, on the device (QR schemes)."""
    ctx = ctx or default_context()
    rep = VerifyReport()

    def add(name, value, threshold):
        rep.checks.append(VerifyCheck(name, value <= threshold, float(value), threshold))

    # 1. product state is exactly isometric
    add("product_state_isometry",
        check_isometric(product_state_uniform(5, 2, model.z1_local_vector(5), ctx), 1e-15, ctx).max_defect(), 1e-15)
    # 2./3. ED comparison on finite chains (thresholds: the reference's)
    add("ed_match_d2_L8", finite_quench_max_z_error(2, 8, 2.0, 0.05, 1.0, 2, "qr", 256, ctx), 5e-3)
    add("ed_match_d3_L4", finite_quench_max_z_error(3, 4, 2.0, 0.05, 0.5, 2, "qr_cbe", 81, ctx), 5e-3)
    # 4. Trotter order: halving dt shrinks the error ~4x
    e1 = finite_quench_max_z_error(2, 6, 2.0, 0.05, 0.5, 2, "qr", 64, ctx)
    e2 = finite_quench_max_z_error(2, 6, 2.0, 0.025, 0.5, 2, "qr", 64, ctx)
    ratio = e1 / max(e2, 1e-300)
    rep.checks.append(VerifyCheck("trotter_order_ratio", 3.0 <= ratio <= 5.0, ratio, 5.0))
    # 5./6. cross-scheme agreement and isometry maintenance, uniform d=3
    zq, sq, dq, _ = _uniform_trace(3, "qr", 0.05, 0.5, 64, ctx)
    zc, sc, dc, _ = _uniform_trace(3, "qr_cbe", 0.05, 0.5, 64, ctx)
    add("scheme_agreement", float(max(np.max(np.abs(zq - zc)), np.max(np.abs(sq - sc)))), 1e-8)
    add("uniform_isometry_drift", max(dq, dc), 1e-3)
    # strict isometry maintenance on a finite chain (checked after every step;
    # the reference observes every gate)
    d, n = 2, 8
    st = product_state_finite(d, n, model.z1_local_vector(d), ctx)
    layers = [(p, [ctx.tensor(model.make_gate(model.chain_bond_hamiltonian(d, 2.0, b, n), dte))
                   for b in range(n - 1)]) for p, dte in model.layer_structure(0.05, 2)]
    pol = TruncationPolicy(chi_max=256, sv_cutoff=1e-14)
    worst = 0.0
    for _ in range(20):
        tebd_step_finite(st, layers, "qr", pol, in_place=True)
        worst = max(worst, check_isometric_finite(st, 1e-10).max_defect())
    add("finite_isometry_after_gates", worst, 1e-10)
    # 7. norm conservation in a lossy run; the fault flag must make it fail
    _, _, _, drift = _uniform_trace(3, "qr_cbe", 0.05, 1.0, 8, ctx, skip_renormalize=fault_skip_renormalize)
    add("norm_conservation", drift, 1e-10)
    return rep
