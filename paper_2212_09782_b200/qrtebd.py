"""Reference-shaped API over the C-ABI (names of proj/include/qrtebd/*.hpp).

Thin host glue: every compute call below goes through libqrtebd_b200.so
(include/qrtebd_c.h).  Arrays passed in may be NumPy arrays (copied to HBM)
or DeviceTensor handles (used in place).  Results come back as DeviceTensor
handles; call .numpy() to fetch them.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import (CapacityError, Context, DeviceTensor, InputError, NumericError, QrtebdError, ShapeError,
                    check, qt_bond_report, qt_report)

__all__ = [
    "TruncationPolicy", "TruncationReport", "GateUpdate", "Context", "DeviceTensor", "apply_gate_qr",
    "apply_gate_qr_cbe", "apply_gate", "truncation_error_explicit", "qr_reduced", "lq_reduced", "UniformMPS",
    "product_state_uniform", "tebd_step", "expectation_local", "schmidt_values", "entropy_from_schmidt",
    "entanglement_entropy", "right_defect", "bond_energy", "ShapeError", "InputError", "NumericError",
    "CapacityError", "QrtebdError", "zgemm", "FiniteMPS", "product_state_finite", "move_center",
    "tebd_step_finite", "finite_observables",
]

_SCHEME_NAMES = {0: "svd", 1: "eig", 2: "qr", 3: "qr_cbe"}


@dataclass
class TruncationPolicy:
    """proj/include/qrtebd/gates.hpp:43-55 (same defaults)."""

    chi_max: int = 1024
    sv_cutoff: float = 1e-14
    target_eps: float = 0.0
    delta_chi_abs: int = 100
    delta_chi_rel: float = 0.1
    chi_max_expansion: int = 0
    qr_sweeps: int = 1
    compute_explicit_error: bool = True
    skip_renormalize: bool = False

    def to_c(self) -> _capi.qt_policy:
        return _capi.default_policy(chi_max=self.chi_max, sv_cutoff=self.sv_cutoff, target_eps=self.target_eps,
                                    delta_chi_abs=self.delta_chi_abs, delta_chi_rel=self.delta_chi_rel,
                                    chi_max_expansion=self.chi_max_expansion, qr_sweeps=self.qr_sweeps,
                                    compute_explicit_error=self.compute_explicit_error,
                                    skip_renormalize=self.skip_renormalize)

    def expanded_dim(self, chi: int, d: int) -> int:
        p = self.to_c()
        return int(_capi.load().qt_expanded_dim(C.byref(p), chi, d))


@dataclass
class TruncationReport:
    """proj/include/qrtebd/gates.hpp:57-64."""

    chi_before: int = 0
    chi_expanded: int = 0
    chi_after: int = 0
    eps_trunc: float = 0.0
    discarded_weight: float = 0.0
    scheme: str = "qr"

    @classmethod
    def from_c(cls, r: qt_report) -> "TruncationReport":
        return cls(int(r.chi_before), int(r.chi_expanded), int(r.chi_after), float(r.eps_trunc),
                   float(r.discarded_weight), _SCHEME_NAMES.get(int(r.scheme), "?"))


@dataclass
class GateUpdate:
    """proj/include/qrtebd/gates.hpp:70-76 (device-resident tensors)."""

    b_m: DeviceTensor
    xi_n: DeviceTensor
    b_n: DeviceTensor
    left_iso: Optional[DeviceTensor]
    report: TruncationReport


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _dev(ctx: Context, a) -> DeviceTensor:
    if isinstance(a, DeviceTensor):
        return a
    return ctx.tensor(a)


def _policy(p) -> _capi.qt_policy:
    if p is None:
        p = TruncationPolicy()
    return p.to_c() if isinstance(p, TruncationPolicy) else p


def apply_gate_qr(xi, b_m, b_n, u, policy=None, ctx: Context = None, want_left_iso: bool = True) -> GateUpdate:
    """apply_gate_qr, proj/src/gates.cpp:343-386."""
    ctx = ctx or default_context()
    lib = ctx.lib
    txi, tbm, tbn, tu = (_dev(ctx, a) for a in (xi, b_m, b_n, u))
    pol = _policy(policy)
    o = [C.c_void_p() for _ in range(4)]
    rep = qt_report()
    check(lib.qt_apply_gate_qr(ctx.h, txi.h, tbm.h, tbn.h, tu.h, C.byref(pol), C.byref(o[0]), C.byref(o[1]),
                               C.byref(o[2]), C.byref(o[3]) if want_left_iso else None, C.byref(rep)))
    left = DeviceTensor(ctx, o[3]) if want_left_iso else None
    return GateUpdate(DeviceTensor(ctx, o[0]), DeviceTensor(ctx, o[1]), DeviceTensor(ctx, o[2]), left,
                      TruncationReport.from_c(rep))


def apply_gate_qr_cbe(xi, b_m, b_n, u, policy=None, ctx: Context = None) -> GateUpdate:
    """apply_gate_qr_cbe, proj/src/gates.cpp:388-450."""
    ctx = ctx or default_context()
    lib = ctx.lib
    txi, tbm, tbn, tu = (_dev(ctx, a) for a in (xi, b_m, b_n, u))
    pol = _policy(policy)
    o = [C.c_void_p() for _ in range(3)]
    rep = qt_report()
    check(lib.qt_apply_gate_qr_cbe(ctx.h, txi.h, tbm.h, tbn.h, tu.h, C.byref(pol), C.byref(o[0]),
                                   C.byref(o[1]), C.byref(o[2]), C.byref(rep)))
    return GateUpdate(DeviceTensor(ctx, o[0]), DeviceTensor(ctx, o[1]), DeviceTensor(ctx, o[2]), None,
                      TruncationReport.from_c(rep))


def apply_gate(scheme: str, xi, b_m, b_n, u, policy=None, ctx: Context = None) -> GateUpdate:
    """apply_gate, proj/src/gates.cpp:452-462 (device schemes only)."""
    if scheme == "qr":
        return apply_gate_qr(xi, b_m, b_n, u, policy, ctx)
    if scheme == "qr_cbe":
        return apply_gate_qr_cbe(xi, b_m, b_n, u, policy, ctx)
    raise InputError(f"scheme {scheme!r} is not a device scheme (svd/eig are the reference's CPU comparators)")


def truncation_error_explicit(theta, left, center, right, ctx: Context = None) -> float:
    """proj/src/gates.cpp:464-485."""
    ctx = ctx or default_context()
    ts = [_dev(ctx, a) for a in (theta, left, center, right)]
    out = C.c_double()
    check(ctx.lib.qt_truncation_error_explicit(ctx.h, *(t.h for t in ts), C.byref(out)))
    return out.value


def qr_reduced(m, ctx: Context = None):
    """proj/src/linalg.cpp:40-51 -> (Q, R) device tensors."""
    ctx = ctx or default_context()
    t = _dev(ctx, m)
    q, r = C.c_void_p(), C.c_void_p()
    check(ctx.lib.qt_qr_reduced(ctx.h, t.h, C.byref(q), C.byref(r)))
    return DeviceTensor(ctx, q), DeviceTensor(ctx, r)


def lq_reduced(m, ctx: Context = None):
    """proj/src/linalg.cpp:53-64 -> (L, Q) device tensors."""
    ctx = ctx or default_context()
    t = _dev(ctx, m)
    l, q = C.c_void_p(), C.c_void_p()
    check(ctx.lib.qt_lq_reduced(ctx.h, t.h, C.byref(l), C.byref(q)))
    return DeviceTensor(ctx, l), DeviceTensor(ctx, q)


def zgemm(ctx: Context, op_a: int, op_b: int, m: int, n: int, k: int, a_ptr: int, lda: int, b_ptr: int,
          ldb: int, c_ptr: int, ldc: int, alpha: float = 1.0, beta: float = 0.0, batch: int = 1,
          stride_a: int = 0, stride_b: int = 0, stride_c: int = 0):
    """Raw complex GEMM on device pointers (qt_zgemm)."""
    check(ctx.lib.qt_zgemm(ctx.h, op_a, op_b, m, n, k, batch, C.c_void_p(a_ptr), lda, stride_a, C.c_void_p(b_ptr),
                           ldb, stride_b, C.c_void_p(c_ptr), ldc, stride_c, alpha, beta))


# --------------------------------------------------------------------- MPS
@dataclass
class UniformMPS:
    """UniformMPS, proj/include/qrtebd/mps.hpp:18-26, state resident in HBM."""

    phys_dim: int
    site_tensors: List[DeviceTensor]
    bond_matrices: List[DeviceTensor]

    def cell_length(self) -> int:
        return len(self.site_tensors)

    def bond_dim(self, m: int) -> int:
        return self.bond_matrices[m].shape[0]

    @classmethod
    def from_numpy(cls, ctx: Context, d: int, sites: Sequence[np.ndarray], bonds: Sequence[np.ndarray]):
        return cls(d, [ctx.tensor(s) for s in sites], [ctx.tensor(b) for b in bonds])

    def to_numpy(self):
        return [s.numpy() for s in self.site_tensors], [b.numpy() for b in self.bond_matrices]


def product_state_uniform(d: int, cell_length: int, local_vector, ctx: Context = None) -> UniformMPS:
    """proj/src/mps.cpp:82-91."""
    ctx = ctx or default_context()
    if cell_length == 0:
        raise InputError("cell length must be positive")
    v = np.asarray(local_vector, dtype=np.complex128)
    if v.shape != (d,):
        raise ShapeError("local vector length must equal d")
    n2 = float(np.vdot(v, v).real)
    if n2 <= 0:
        raise InputError("local vector has zero norm")
    v = v / math.sqrt(n2)
    return UniformMPS.from_numpy(ctx, d, [v.reshape(d, 1, 1)] * cell_length,
                                 [np.eye(1, dtype=np.complex128)] * cell_length)


@dataclass
class BondReport:
    bond: int
    report: TruncationReport


def tebd_step(state: UniformMPS, schedule, scheme: str, policy=None, ctx: Context = None):
    """tebd_step(UniformMPS), proj/src/gates.cpp:513-540, one C-ABI call.

    schedule: [(parity 'even'|'odd', gate as (d,d,d,d) array or DeviceTensor)].
    Returns (new UniformMPS, [BondReport])."""
    ctx = ctx or default_context()
    L = state.cell_length()
    gates = [_dev(ctx, g) for _, g in schedule]
    par = (C.c_int32 * max(1, len(schedule)))(*[0 if p == "even" else 1 for p, _ in schedule])
    sites = (C.c_void_p * L)(*[t.h for t in state.site_tensors])
    bonds = (C.c_void_p * L)(*[t.h for t in state.bond_matrices])
    gh = (C.c_void_p * max(1, len(gates)))(*[g.h for g in gates])
    so = (C.c_void_p * L)()
    bo = (C.c_void_p * L)()
    cap = len(schedule) * (L // 2 + 1)
    reps = (qt_bond_report * max(1, cap))()
    n = C.c_uint64(cap)
    pol = _policy(policy)
    sid = _capi.SCHEME_IDS[scheme]
    check(ctx.lib.qt_tebd_step_uniform(ctx.h, L, sites, bonds, len(schedule), par, gh, sid, C.byref(pol), so, bo,
                                       reps, C.byref(n)))
    new = UniformMPS(state.phys_dim, [DeviceTensor(ctx, C.c_void_p(so[m])) for m in range(L)],
                     [DeviceTensor(ctx, C.c_void_p(bo[m])) for m in range(L)])
    out = [BondReport(int(reps[i].bond), TruncationReport.from_c(reps[i].report)) for i in range(n.value)]
    return new, out


class DeviceUniformMPS:
    """Device-resident UniformMPS with in-place, graph-replayed steps
    (qt_uniform_*).  The fast path behind tebd_step for long evolutions."""

    def __init__(self, state: UniformMPS, ctx: Context = None):
        self.ctx = ctx or default_context()
        L = state.cell_length()
        sites = (C.c_void_p * L)(*[t.h for t in state.site_tensors])
        bonds = (C.c_void_p * L)(*[t.h for t in state.bond_matrices])
        h = C.c_void_p()
        check(self.ctx.lib.qt_uniform_create(self.ctx.h, L, sites, bonds, C.byref(h)))
        self.h = h
        self.L = L
        self.phys_dim = state.phys_dim

    def close(self):
        # a destroyed context already released the device memory and stream
        if self.h and self.ctx.h:
            self.ctx.lib.qt_uniform_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, schedule, scheme: str, policy=None, use_graph: bool = True):
        """tebd_step in place; returns [BondReport]."""
        gates = [_dev(self.ctx, g) for _, g in schedule]
        self._gates = gates  # keep device gates alive (graphs capture their addresses)
        par = (C.c_int32 * max(1, len(schedule)))(*[0 if p == "even" else 1 for p, _ in schedule])
        gh = (C.c_void_p * max(1, len(gates)))(*[g.h for g in gates])
        cap = len(schedule) * (self.L // 2 + 1)
        reps = (qt_bond_report * max(1, cap))()
        n = C.c_uint64(cap)
        pol = _policy(policy)
        check(self.ctx.lib.qt_uniform_step(self.h, len(schedule), par, gh, _capi.SCHEME_IDS[scheme], C.byref(pol),
                                           1 if use_graph else 0, reps, C.byref(n)))
        return [BondReport(int(reps[i].bond), TruncationReport.from_c(reps[i].report)) for i in range(n.value)]

    def view(self, which: str, m: int) -> DeviceTensor:
        """Non-owning view of the live site ('site') or bond ('bond') buffer m."""
        h = C.c_void_p()
        check(self.ctx.lib.qt_uniform_view(self.h, 0 if which == "site" else 1, m, C.byref(h)))
        return DeviceTensor(self.ctx, h)

    def snapshot(self) -> UniformMPS:
        """Owned copies of the live state as a UniformMPS."""
        sites = [self.ctx.tensor(self.view("site", m).numpy()) for m in range(self.L)]
        bonds = [self.ctx.tensor(self.view("bond", m).numpy()) for m in range(self.L)]
        return UniformMPS(self.phys_dim, sites, bonds)


def expectation_local(state: UniformMPS, op, site: int, ctx: Context = None) -> complex:
    """expectation_local(UniformMPS), proj/src/mps.cpp:179-186."""
    ctx = ctx or default_context()
    if site >= state.cell_length():
        raise InputError("site out of range")
    top = _dev(ctx, op)
    out = (C.c_double * 2)()
    check(ctx.lib.qt_expectation_local(ctx.h, state.bond_matrices[site].h, state.site_tensors[site].h, top.h, out))
    return complex(out[0], out[1])


def schmidt_values_of(xi, ctx: Context = None) -> np.ndarray:
    ctx = ctx or default_context()
    t = _dev(ctx, xi)
    k = min(t.shape)
    out = (C.c_double * max(1, k))()
    n = C.c_uint64(k)
    check(ctx.lib.qt_schmidt_values(ctx.h, t.h, out, C.byref(n)))
    return np.array(out[: n.value])


def schmidt_values(state: UniformMPS, bond: int, ctx: Context = None) -> np.ndarray:
    """proj/src/mps.cpp:198-201."""
    if bond >= state.cell_length():
        raise InputError("bond out of range")
    return schmidt_values_of(state.bond_matrices[bond], ctx)


def entropy_from_schmidt(values) -> float:
    """proj/src/mps.cpp:209-216 (scalar post-processing of device spectra)."""
    s = 0.0
    for v in values:
        p = float(v) * float(v)
        if p > 0.0:
            s -= p * math.log(p)
    return s


def entanglement_entropy(state: UniformMPS, bond: int, ctx: Context = None) -> float:
    return entropy_from_schmidt(schmidt_values(state, bond, ctx))


def right_defect(b, ctx: Context = None) -> float:
    """proj/src/mps.cpp:34-36."""
    ctx = ctx or default_context()
    t = _dev(ctx, b)
    out = C.c_double()
    check(ctx.lib.qt_right_defect(ctx.h, t.h, C.byref(out)))
    return out.value


@dataclass
class IsometryReport:
    """proj/include/qrtebd/mps.hpp:40-53."""
    right_defects: List[float]
    left_defects: List[float]
    translation_defects: List[float]
    norm_defects: List[float]
    max_right_defect: float
    max_left_defect: float
    max_translation_defect: float
    max_norm_defect: float
    passed: bool

    def max_defect(self) -> float:
        return max(self.max_right_defect, self.max_left_defect, self.max_translation_defect, self.max_norm_defect)


def check_isometric(state: UniformMPS, tol: float, ctx: Context = None) -> IsometryReport:
    """check_isometric(UniformMPS), proj/src/mps.cpp:105-141, on the device."""
    ctx = ctx or default_context()
    L = state.cell_length()
    sites = [_dev(ctx, t) for t in state.site_tensors]
    bonds = [_dev(ctx, t) for t in state.bond_matrices]
    sa = (C.c_void_p * L)(*[t.h for t in sites])
    ba = (C.c_void_p * L)(*[t.h for t in bonds])
    arrs = [(C.c_double * L)() for _ in range(4)]
    rep = _capi.qt_isometry_report()
    check(ctx.lib.qt_check_isometric_uniform(ctx.h, L, C.cast(sa, _capi.PP), C.cast(ba, _capi.PP), tol,
                                             *arrs, C.byref(rep)))
    r, l, t, n = ([a[i] for i in range(L)] for a in arrs)
    return IsometryReport(r, l, t, n, rep.max_right_defect, rep.max_left_defect, rep.max_translation_defect,
                          rep.max_norm_defect, bool(rep.pass_))


def bond_energy(xi, b_m, b_n, h_bond, ctx: Context = None) -> float:
    """Bond energy extension."""
    ctx = ctx or default_context()
    ts = [_dev(ctx, a) for a in (xi, b_m, b_n, h_bond)]
    out = C.c_double()
    check(ctx.lib.qt_bond_energy(ctx.h, *(t.h for t in ts), C.byref(out)))
    return out.value


def eigh(h, ctx: Context = None):
    """eigh, proj/src/linalg.cpp:79-101 (device block Jacobi): (w desc, V device)."""
    ctx = ctx or default_context()
    t = _dev(ctx, h)
    n = t.shape[0]
    w = (C.c_double * max(1, n))()
    v = C.c_void_p()
    check(ctx.lib.qt_eigh(ctx.h, t.h, w, C.byref(v)))
    return np.array(w[:n]), DeviceTensor(ctx, v)


# --------------------------------------------------------------------- FiniteMPS (reference semantics)
class FiniteMPS:
    """FiniteMPS, proj/include/qrtebd/mps.hpp:31-38, resident in HBM (qt_finite).

    Site tensors (d, chi_l, chi_r), an orthogonality-center bond and its
    (possibly rectangular) center matrix.  move_center and tebd_step run in
    place on the device; snapshot()/to_numpy() fetch the state."""

    def __init__(self, phys_dim: int, site_tensors, center_bond: int, center_matrix, ctx: Context = None):
        self.ctx = ctx or default_context()
        sites = [_dev(self.ctx, t) for t in site_tensors]
        cm = _dev(self.ctx, center_matrix)
        n = len(sites)
        arr = (C.c_void_p * max(1, n))(*[t.h for t in sites])
        h = C.c_void_p()
        check(self.ctx.lib.qt_finite_create(self.ctx.h, n, arr, center_bond, cm.h, C.byref(h)))
        self.h = h
        self.phys_dim = phys_dim
        self.n = n

    @classmethod
    def _adopt(cls, ctx: Context, handle, phys_dim: int, n: int) -> "FiniteMPS":
        obj = cls.__new__(cls)
        obj.ctx, obj.h, obj.phys_dim, obj.n = ctx, handle, phys_dim, n
        return obj

    def close(self):
        if getattr(self, "h", None) and self.ctx.h:
            self.ctx.lib.qt_finite_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def length(self) -> int:
        return self.n

    @property
    def center_bond(self) -> int:
        out = C.c_uint64()
        check(self.ctx.lib.qt_finite_center_bond(self.h, C.byref(out)))
        return int(out.value)

    def view(self, which: str, m: int = 0) -> DeviceTensor:
        """Non-owning view of site tensor m ('site') or of the center matrix ('center')."""
        h = C.c_void_p()
        check(self.ctx.lib.qt_finite_view(self.h, 0 if which == "site" else 1, m, C.byref(h)))
        return DeviceTensor(self.ctx, h)

    @property
    def center_matrix(self) -> np.ndarray:
        return self.view("center").numpy()

    def site(self, m: int) -> np.ndarray:
        return self.view("site", m).numpy()

    def copy(self) -> "FiniteMPS":
        h = C.c_void_p()
        check(self.ctx.lib.qt_finite_clone(self.h, C.byref(h)))
        return FiniteMPS._adopt(self.ctx, h, self.phys_dim, self.n)

    def to_numpy(self):
        """(site tensors, center_bond, center matrix) as NumPy arrays."""
        return [self.site(m) for m in range(self.n)], self.center_bond, self.center_matrix


def product_state_finite(d: int, n_sites: int, local_vector, ctx: Context = None) -> FiniteMPS:
    """proj/src/mps.cpp:93-102."""
    if n_sites == 0:
        raise InputError("chain length must be positive")
    v = np.asarray(local_vector, dtype=np.complex128)
    if v.shape != (d,):
        raise ShapeError("local vector length must equal d")
    n2 = float(np.vdot(v, v).real)
    if n2 <= 0:
        raise InputError("local vector has zero norm")
    v = v / math.sqrt(n2)
    return FiniteMPS(d, [v.reshape(d, 1, 1)] * n_sites, 0, np.eye(1, dtype=np.complex128), ctx)


def move_center(state: FiniteMPS, new_center: int) -> FiniteMPS:
    """move_center, proj/src/mps.cpp:226-257: value semantics (a moved copy)."""
    out = state.copy()
    check(out.ctx.lib.qt_finite_move_center(out.h, new_center))
    return out


def tebd_step_finite(state: FiniteMPS, layers, scheme: str, policy=None, in_place: bool = False):
    """tebd_step(FiniteMPS), proj/src/gates.cpp:542-578 (reference semantics:
    the center is moved onto every bond before its gate).

    layers: [(parity 'even'|'odd', [gate per bond m, acting on (m, m+1)])]
    (FiniteLayer, proj/include/qrtebd/gates.hpp:130-137).  Returns
    (new FiniteMPS, [BondReport]); in_place=True updates `state` itself."""
    s = state if in_place else state.copy()
    ctx = s.ctx
    nb = s.n - 1
    flat = []
    for _, gates in layers:
        if len(gates) != nb:
            raise ShapeError("layer gate count must equal the bond count")
        flat.extend(_dev(ctx, g) for g in gates)
    s._gates = flat
    par = (C.c_int32 * max(1, len(layers)))(*[0 if p == "even" else 1 for p, _ in layers])
    gh = (C.c_void_p * max(1, len(flat)))(*[g.h for g in flat])
    cap = len(layers) * (nb // 2 + 1)
    reps = (qt_bond_report * max(1, cap))()
    n = C.c_uint64(cap)
    pol = _policy(policy)
    check(ctx.lib.qt_finite_step(s.h, len(layers), par, gh, _capi.SCHEME_IDS[scheme], C.byref(pol), reps,
                                 C.byref(n)))
    out = [BondReport(int(reps[i].bond), TruncationReport.from_c(reps[i].report)) for i in range(n.value)]
    return s, out


def finite_observables(state: FiniteMPS, op=None):
    """<op> on every site (expectation_local(FiniteMPS), mps.cpp:188-196) and
    the Schmidt values of every bond 0..n (schmidt_values(FiniteMPS),
    mps.cpp:203-207), from one device gauge sweep: returns (z, [spectra])."""
    ctx = state.ctx
    n = state.n
    top = _dev(ctx, op) if op is not None else None
    offs = (C.c_uint64 * (n + 2))()
    z = (C.c_double * max(1, 2 * n))()
    check(ctx.lib.qt_finite_observables(state.h, top.h if top else None, z, None, 0, offs))
    total = int(offs[n + 1])
    buf = (C.c_double * max(1, total))()
    check(ctx.lib.qt_finite_observables(state.h, None, None, buf, total, offs))
    zs = np.array([complex(z[2 * s], z[2 * s + 1]) for s in range(n)]) if top is not None else None
    spectra = [np.array(buf[int(offs[b]):int(offs[b + 1])]) for b in range(n + 1)]
    return zs, spectra


def expectation_local_finite(state: FiniteMPS, op, site: int) -> complex:
    """expectation_local(FiniteMPS), proj/src/mps.cpp:188-196."""
    if site >= state.n:
        raise InputError("site out of range")
    c = move_center(state, site)
    out = (C.c_double * 2)()
    top = _dev(c.ctx, op)
    cv, sv = c.view("center"), c.view("site", site)  # keep the view handles alive across the call
    check(c.ctx.lib.qt_expectation_local(c.ctx.h, cv.h, sv.h, top.h, out))
    return complex(out[0], out[1])


def schmidt_values_finite(state: FiniteMPS, bond: int) -> np.ndarray:
    """schmidt_values(FiniteMPS), proj/src/mps.cpp:203-207."""
    if bond > state.n:
        raise InputError("bond out of range")
    c = move_center(state, bond)
    return schmidt_values_of(c.view("center"), c.ctx)


def left_defect(b, ctx: Context = None) -> float:
    """proj/src/mps.cpp:39-41."""
    ctx = ctx or default_context()
    t = _dev(ctx, b)
    out = C.c_double()
    check(ctx.lib.qt_left_defect(ctx.h, t.h, C.byref(out)))
    return out.value


def check_isometric_finite(state: FiniteMPS, tol: float) -> IsometryReport:
    """check_isometric(FiniteMPS), proj/src/mps.cpp:143-164, on the device."""
    n = state.n
    r = (C.c_double * n)()
    l = (C.c_double * n)()
    nd = C.c_double()
    rep = _capi.qt_isometry_report()
    check(state.ctx.lib.qt_check_isometric_finite(state.h, tol, r, l, C.byref(nd), C.byref(rep)))
    return IsometryReport(list(r), list(l), [], [nd.value], rep.max_right_defect, rep.max_left_defect, 0.0,
                          rep.max_norm_defect, bool(rep.pass_))
