"""CPU oracle: a NumPy/LAPACK restatement of the reference QR-TEBD path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py may import this module, and
only as the checker or the timed CPU baseline -- never as part of the product
path (paper_2212_09782_b200/ never imports it).

Reference: /root/reference/proj (C++20 + Eigen 3.4).  The reference cannot be
built here (Eigen 3.4, GoogleTest and CLI11 are absent and there is no
network), so this file restates its algorithm function by
function, citing file:line.  The third-party arithmetic it stands on:

  * Eigen 3.4 (pinned only by find_package(Eigen3 3.4), proj/CMakeLists.txt:14):
    GEMM, HouseholderQR, BDCSVD, SelfAdjointEigenSolver.  Restated on LAPACK
    through NumPy 2.3 / OpenBLAS 0.3.30: zgemm, zgeqrf+zungqr
    (numpy.linalg.qr 'reduced'; the Householder sign convention of zlarfg and
    Eigen's makeHouseholder agree, and after the reference gauge fix Q and R
    are unique for full rank), zgesdd (numpy.linalg.svd), zheevd
    (numpy.linalg.eigh).

Parity pinning: the reference ships no golden-vector files;
its tests pin results by known answers and tolerances.  tests/test_oracle.py
re-runs those known-answer tests (proj/tests/test_linalg.cc,
test_gates.cc, test_tebd.cc, acceptance.cc criteria) against this module.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence, Tuple

import numpy as np

cplx = np.complex128


class ShapeError(ValueError):
    pass


class InputError(ValueError):
    pass


class NumericError(RuntimeError):
    pass


# --------------------------------------------------------------------- policy
@dataclass
class TruncationPolicy:
    """proj/include/qrtebd/gates.hpp:43-55."""

    chi_max: int = 1024
    sv_cutoff: float = 1e-14
    target_eps: float = 0.0
    delta_chi_abs: int = 100
    delta_chi_rel: float = 0.1
    chi_max_expansion: int = 0
    qr_sweeps: int = 1
    compute_explicit_error: bool = True
    skip_renormalize: bool = False

    def expanded_dim(self, chi: int, d: int) -> int:
        """proj/src/gates.cpp:94-101."""
        rel = int(math.ceil(self.delta_chi_rel * float(chi)))
        delta = max(self.delta_chi_abs, rel)
        eta = min(d * chi, chi + delta)
        if self.chi_max_expansion != 0:
            eta = min(eta, self.chi_max_expansion)
        return eta


@dataclass
class TruncationReport:
    """proj/include/qrtebd/gates.hpp:57-64."""

    chi_before: int = 0
    chi_expanded: int = 0
    chi_after: int = 0
    eps_trunc: float = 0.0
    discarded_weight: float = 0.0
    scheme: str = "svd"


@dataclass
class GateUpdate:
    """proj/include/qrtebd/gates.hpp:70-76."""

    b_m: np.ndarray
    xi_n: np.ndarray
    b_n: np.ndarray
    left_iso: Optional[np.ndarray]
    report: TruncationReport


# --------------------------------------------------------------------- linalg
def _require_finite_matrix(m: np.ndarray, op: str):
    """proj/src/linalg.cpp:17-21."""
    if m.ndim != 2:
        raise ShapeError(f"{op}: expected a matrix")
    if not np.all(np.isfinite(m)):
        raise InputError(f"{op}: non-finite entries")


def _fix_qr_gauge(q: np.ndarray, r: np.ndarray):
    """proj/src/linalg.cpp:25-36 (in place)."""
    k = r.shape[0]
    for i in range(k):
        d = r[i, i]
        a = abs(d)
        if a == 0.0:
            continue
        phase = d / a
        q[:, i] *= phase
        r[i, :] *= np.conj(phase)
        r[i, i] = a


def qr_reduced(m: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """proj/src/linalg.cpp:40-51: thin Householder QR, R_ii real >= 0."""
    m = np.asarray(m, dtype=cplx)
    _require_finite_matrix(m, "qr_reduced")
    q, r = np.linalg.qr(m, mode="reduced")
    q = np.array(q, dtype=cplx, order="C")
    r = np.array(np.triu(r), dtype=cplx, order="C")
    _fix_qr_gauge(q, r)
    return q, r


def lq_reduced(m: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """proj/src/linalg.cpp:53-64: m = L Q via QR of m^H."""
    m = np.asarray(m, dtype=cplx)
    _require_finite_matrix(m, "lq_reduced")
    q, r = qr_reduced(m.conj().T)
    return np.ascontiguousarray(r.conj().T), np.ascontiguousarray(q.conj().T)


def svd(m: np.ndarray):
    """proj/src/linalg.cpp:66-77 (BDCSVD -> zgesdd): (U, s desc, V^H)."""
    m = np.asarray(m, dtype=cplx)
    _require_finite_matrix(m, "svd")
    u, s, vh = np.linalg.svd(m, full_matrices=False)
    return u, s, vh


def eigh(h: np.ndarray):
    """proj/src/linalg.cpp:79-101: hermiticity check, symmetrize, descending."""
    a = np.asarray(h, dtype=cplx)
    _require_finite_matrix(a, "eigh")
    if a.shape[0] != a.shape[1]:
        raise ShapeError("eigh: matrix not square")
    defect = np.linalg.norm(a - a.conj().T)
    if defect > 1e-10 * max(np.linalg.norm(a), 1e-300):
        raise InputError("eigh: matrix not hermitian within tolerance")
    sym = 0.5 * (a + a.conj().T)
    w, v = np.linalg.eigh(sym)
    return w[::-1].copy(), np.ascontiguousarray(v[:, ::-1])


def expm_hermitian(h: np.ndarray, t: float) -> np.ndarray:
    """proj/src/linalg.cpp:103-110: exp(-i t h)."""
    w, v = eigh(h)
    return (v * np.exp(-1j * t * w)) @ v.conj().T


# --------------------------------------------------------------------- model
def clock_operators(d: int):
    """proj/src/clock.cpp:54-63."""
    if d < 2:
        raise InputError("clock model needs d >= 2")
    step = 2.0 * math.pi / d
    z = np.zeros((d, d), dtype=cplx)
    x = np.zeros((d, d), dtype=cplx)
    for k in range(d):
        z[k, k] = complex(math.cos(step * k), math.sin(step * k))
        x[k, (k + 1) % d] = 1.0
    return z, x


def bond_hamiltonian_weighted(d: int, g: float, wl: float, wr: float) -> np.ndarray:
    """proj/src/clock.cpp:65-78."""
    z, x = clock_operators(d)
    ident = np.eye(d, dtype=cplx)
    onsite = g * (x + x.conj().T)
    zz = np.kron(z, z.conj().T)
    h = -(zz + zz.conj().T)
    h = h - wl * np.kron(onsite, ident)
    h = h - wr * np.kron(ident, onsite)
    return h


def bond_hamiltonian(d: int, g: float, kind: str = "bulk") -> np.ndarray:
    """proj/src/clock.cpp:80-90."""
    w = {"bulk": (0.5, 0.5), "left_edge": (1.0, 0.5), "right_edge": (0.5, 1.0)}[kind]
    return bond_hamiltonian_weighted(d, g, *w)


def chain_bond_hamiltonian(d: int, g: float, bond: int, n_sites: int) -> np.ndarray:
    """proj/src/clock.cpp:92-99."""
    if n_sites < 2 or bond + 1 >= n_sites:
        raise InputError("bond index out of range")
    wl = 1.0 if bond == 0 else 0.5
    wr = 1.0 if bond + 2 == n_sites else 0.5
    return bond_hamiltonian_weighted(d, g, wl, wr)


def make_gate(h_bond: np.ndarray, dt: float) -> np.ndarray:
    """proj/src/gates.cpp:50-57: exp(-i dt h) reshaped (d,d,d,d)."""
    d2 = h_bond.shape[0]
    d = int(round(math.sqrt(d2)))
    if d * d != d2:
        raise ShapeError("bond hamiltonian dimension is not d^2")
    return expm_hermitian(h_bond, dt).reshape(d, d, d, d)


def identity_gate(d: int) -> np.ndarray:
    """proj/src/gates.cpp:59-61."""
    return np.eye(d * d, dtype=cplx).reshape(d, d, d, d)


def layer_structure(dt: float, order: int):
    """proj/src/gates.cpp:489-501."""
    if order == 1:
        return [("even", dt), ("odd", dt)]
    if order == 2:
        return [("even", 0.5 * dt), ("odd", dt), ("even", 0.5 * dt)]
    raise InputError("trotter order must be 1 or 2")


def trotter_schedule(h_bond: np.ndarray, dt: float, order: int):
    """proj/src/gates.cpp:505-511."""
    return [(p, make_gate(h_bond, dte)) for p, dte in layer_structure(dt, order)]


# --------------------------------------------------------------------- gates
@dataclass
class ThetaParts:
    """proj/src/gates.cpp:116-121."""

    phi_evolved: np.ndarray  # (beta, i, j, delta)
    theta: np.ndarray  # (alpha, i, j, delta)
    d: int
    chi_l: int
    chi_n: int
    chi_r: int
    theta_norm: float


def build_theta(xi, b_m, b_n, u) -> ThetaParts:
    """proj/src/gates.cpp:123-182."""
    if b_m.ndim != 3 or b_n.ndim != 3 or xi.ndim != 2:
        raise ShapeError("gate update expects rank-3 site tensors and a bond matrix")
    d = b_m.shape[0]
    if b_n.shape[0] != d or u.shape[0] != d:
        raise ShapeError("physical dimensions disagree")
    if xi.shape[1] != b_m.shape[1] or b_m.shape[2] != b_n.shape[1]:
        raise ShapeError("bond dimensions disagree")
    chi_l, chi_m, chi_n, chi_r = xi.shape[0], b_m.shape[1], b_m.shape[2], b_n.shape[2]
    # phi[(i j), (beta delta)] = Bm_i Bn_j                 (:145-165)
    phi = np.einsum("iab,jbc->ijac", b_m, b_n, optimize=True)
    # evolved = U phi                                     (:168-170)
    evolved = (u.reshape(d * d, d * d) @ phi.reshape(d * d, chi_m * chi_r)).reshape(d, d, chi_m, chi_r)
    phi_ev = np.ascontiguousarray(evolved.transpose(2, 0, 1, 3))  # (:171)
    theta = (xi @ phi_ev.reshape(chi_m, d * d * chi_r)).reshape(chi_l, d, d, chi_r)  # (:175-179)
    return ThetaParts(phi_ev, theta, d, chi_l, chi_n, chi_r, float(np.linalg.norm(theta)))


def hastings_left(phi_ev, b_n_new):
    """proj/src/gates.cpp:186-190: B~m(i,beta,k) = sum phi_ev(beta,i,j,delta) conj(B~n(j,k,delta))."""
    return np.ascontiguousarray(np.einsum("bijd,jkd->ibk", phi_ev, b_n_new.conj(), optimize=True))


def right_tensor_from_rows(rows, d, chi_r):
    """proj/src/gates.cpp:193-196."""
    return np.ascontiguousarray(rows.reshape(rows.shape[0], d, chi_r).transpose(1, 0, 2))


def left_tensor_from_cols(cols, d, chi_l):
    """proj/src/gates.cpp:198-201."""
    return np.ascontiguousarray(cols.reshape(chi_l, d, cols.shape[1]).transpose(1, 0, 2))


def grouped(t4):
    """(dim0 dim1) x (dim2 dim3) view, proj/src/gates.cpp:107-111."""
    return t4.reshape(t4.shape[0] * t4.shape[1], t4.shape[2] * t4.shape[3])


def diagonal_bond_matrix(values, inv_scale):
    """proj/src/gates.cpp:215-221."""
    k = len(values)
    xi = np.zeros((k, k), dtype=cplx)
    xi[np.arange(k), np.arange(k)] = np.asarray(values) * inv_scale
    return xi


def choose_kept(s_norm: Sequence[float], policy: TruncationPolicy) -> int:
    """proj/src/gates.cpp:226-240."""
    k = 0
    while k < len(s_norm) and s_norm[k] >= policy.sv_cutoff:
        k += 1
    k = min(k, policy.chi_max)
    if policy.target_eps > 0.0:
        n = len(s_norm)
        suffix = [0.0] * (n + 1)
        for i in range(n - 1, -1, -1):
            suffix[i] = suffix[i + 1] + s_norm[i] * s_norm[i]
        kt = 0
        while kt < n and suffix[kt] > policy.target_eps:
            kt += 1
        k = min(k, kt)
    return max(k, 1)


def squared_tail(s, start):
    """proj/src/gates.cpp:242-246."""
    t = 0.0
    for i in range(start, len(s)):
        t += s[i] * s[i]
    return t


def finish_spectral_update(parts: ThetaParts, s, vdag, u_cols, policy, scheme):
    """proj/src/gates.cpp:250-282."""
    if parts.theta_norm <= 0.0:
        raise NumericError("evolved block has zero norm")
    s_norm = [float(v) / parts.theta_norm for v in s]
    kk = choose_kept(s_norm, policy)
    kept = [float(v) for v in s[:kk]]
    kept_norm = math.sqrt(squared_tail(kept, 0))
    denom = parts.theta_norm if policy.skip_renormalize else kept_norm
    xi_n = diagonal_bond_matrix(kept, 1.0 / denom if denom > 0 else 0.0)
    b_n = right_tensor_from_rows(vdag[:kk], parts.d, parts.chi_r)
    b_m = hastings_left(parts.phi_evolved, b_n)
    left = left_tensor_from_cols(u_cols[:, :kk], parts.d, parts.chi_l) if u_cols is not None else None
    total2 = parts.theta_norm * parts.theta_norm
    rep = TruncationReport(parts.chi_n, min(parts.chi_l * parts.d, parts.d * parts.chi_r), kk)
    rep.discarded_weight = max(0.0, total2 - kept_norm * kept_norm)
    rep.eps_trunc = rep.discarded_weight / total2
    rep.scheme = scheme
    return GateUpdate(b_m, xi_n, b_n, left, rep)


def alternating_sweep(theta, y0, sweeps):
    """proj/src/gates.cpp:293-308."""
    th = grouped(theta)
    q_m = l = q_n = None
    for _ in range(max(1, sweeps)):
        x = th @ y0.conj().T
        q_m, _r = qr_reduced(x)
        y = q_m.conj().T @ th
        l, q_n = lq_reduced(y)
        y0 = q_n
    return q_m, l, q_n


def apply_gate_svd(xi, b_m, b_n, u, policy: TruncationPolicy) -> GateUpdate:
    """proj/src/gates.cpp:312-322 (CPU SVD-TEBD comparator)."""
    parts = build_theta(xi, b_m, b_n, u)
    uu, s, vh = svd(grouped(parts.theta))
    return finish_spectral_update(parts, s, vh, uu, policy, "svd")


def apply_gate_eig(xi, b_m, b_n, u, policy: TruncationPolicy) -> GateUpdate:
    """proj/src/gates.cpp:324-341."""
    parts = build_theta(xi, b_m, b_n, u)
    th = grouped(parts.theta)
    w, v = eigh(th.conj().T @ th)
    s = np.where(w > 0.0, np.sqrt(np.maximum(w, 0.0)), 0.0)
    return finish_spectral_update(parts, s, v.conj().T, None, policy, "eig")


def truncation_error_explicit(theta, left, center, right) -> float:
    """proj/src/gates.cpp:464-485."""
    if theta.ndim not in (2, 4):
        raise ShapeError("truncation_error_explicit expects a matrix or a rank-4 block")
    t = grouped(theta) if theta.ndim == 4 else theta
    if left.shape[0] != t.shape[0] or left.shape[1] != center.shape[0] or \
            center.shape[1] != right.shape[0] or right.shape[1] != t.shape[1]:
        raise ShapeError("factor shapes inconsistent with theta")
    approx = left @ (center @ right)
    denom = float(np.vdot(t, t).real)
    if denom == 0.0:
        return 0.0
    diff = t - approx
    return float(np.vdot(diff, diff).real) / denom


def apply_gate_qr(xi, b_m, b_n, u, policy: TruncationPolicy) -> GateUpdate:
    """proj/src/gates.cpp:343-386."""
    parts = build_theta(xi, b_m, b_n, u)
    rows, cols, chi = parts.chi_l * parts.d, parts.d * parts.chi_r, parts.chi_n
    eta = min(policy.expanded_dim(chi, parts.d), policy.chi_max)
    eta = min(eta, rows, cols)
    if eta == chi:
        y0 = b_n.transpose(1, 0, 2).reshape(chi, cols)
    else:
        y0 = grouped(parts.theta)[:eta]
    q_m, l, q_n = alternating_sweep(parts.theta, y0, policy.qr_sweeps)
    l_norm = float(np.linalg.norm(l))
    denom = parts.theta_norm if policy.skip_renormalize else l_norm
    xi_n = l * (1.0 / denom if denom > 0 else 0.0)
    b_n_new = right_tensor_from_rows(q_n, parts.d, parts.chi_r)
    b_m_new = hastings_left(parts.phi_evolved, b_n_new)
    left = left_tensor_from_cols(q_m, parts.d, parts.chi_l)
    total2 = parts.theta_norm * parts.theta_norm
    rep = TruncationReport(chi, eta, eta, scheme="qr")
    rep.discarded_weight = max(0.0, total2 - l_norm * l_norm)
    if policy.compute_explicit_error:
        rep.eps_trunc = truncation_error_explicit(parts.theta, q_m, l, q_n)
    else:
        rep.eps_trunc = rep.discarded_weight / total2 if total2 > 0 else float("nan")
    return GateUpdate(b_m_new, xi_n, b_n_new, left, rep)


def apply_gate_qr_cbe(xi, b_m, b_n, u, policy: TruncationPolicy) -> GateUpdate:
    """proj/src/gates.cpp:388-450."""
    parts = build_theta(xi, b_m, b_n, u)
    rows, cols, chi = parts.chi_l * parts.d, parts.d * parts.chi_r, parts.chi_n
    eta = policy.expanded_dim(chi, parts.d)
    if eta > parts.d * chi:
        raise InputError("bond expansion beyond d*chi")
    eta = min(eta, rows, cols)
    q_m, l, q_n = alternating_sweep(parts.theta, grouped(parts.theta)[:eta], policy.qr_sweeps)
    w, v = eigh(l.conj().T @ l)
    s = np.where(w > 0.0, np.sqrt(np.maximum(w, 0.0)), 0.0)
    if parts.theta_norm <= 0.0:
        raise NumericError("evolved block has zero norm")
    s_norm = [float(x) / parts.theta_norm for x in s]
    kk = choose_kept(s_norm, policy)
    v_kept = v[:, :kk]
    b_n_rows = v_kept.conj().T @ q_n
    kept = [float(x) for x in s[:kk]]
    kept_norm = math.sqrt(squared_tail(kept, 0))
    denom = parts.theta_norm if policy.skip_renormalize else kept_norm
    xi_n = diagonal_bond_matrix(kept, 1.0 / denom if denom > 0 else 0.0)
    b_n_new = right_tensor_from_rows(b_n_rows, parts.d, parts.chi_r)
    b_m_new = hastings_left(parts.phi_evolved, b_n_new)
    total2 = parts.theta_norm * parts.theta_norm
    rep = TruncationReport(chi, eta, kk, scheme="qr_cbe")
    rep.discarded_weight = max(0.0, total2 - kept_norm * kept_norm)
    if policy.compute_explicit_error:
        center_kept = l @ (v_kept @ v_kept.conj().T)
        rep.eps_trunc = truncation_error_explicit(parts.theta, q_m, center_kept, q_n)
    else:
        rep.eps_trunc = rep.discarded_weight / total2
    return GateUpdate(b_m_new, xi_n, b_n_new, None, rep)


def apply_gate(scheme: str, xi, b_m, b_n, u, policy) -> GateUpdate:
    """proj/src/gates.cpp:452-462."""
    fn = {"svd": apply_gate_svd, "eig": apply_gate_eig, "qr": apply_gate_qr, "qr_cbe": apply_gate_qr_cbe}
    if scheme not in fn:
        raise InputError("unknown scheme")
    return fn[scheme](xi, b_m, b_n, u, policy)


# --------------------------------------------------------------------- MPS
@dataclass
class UniformMPS:
    """proj/include/qrtebd/mps.hpp:18-26."""

    phys_dim: int
    site_tensors: List[np.ndarray]
    bond_matrices: List[np.ndarray]

    def cell_length(self):
        return len(self.site_tensors)

    def copy(self):
        return UniformMPS(self.phys_dim, [t.copy() for t in self.site_tensors],
                          [t.copy() for t in self.bond_matrices])


def product_state_uniform(d: int, cell_length: int, local_vector) -> UniformMPS:
    """proj/src/mps.cpp:82-91."""
    v = np.asarray(local_vector, dtype=cplx)
    if v.shape != (d,):
        raise ShapeError("local vector length must equal d")
    n2 = float(np.vdot(v, v).real)
    if n2 <= 0.0:
        raise InputError("local vector has zero norm")
    v = v / math.sqrt(n2)
    return UniformMPS(d, [v.reshape(d, 1, 1).copy() for _ in range(cell_length)],
                      [np.eye(1, dtype=cplx) for _ in range(cell_length)])


def tebd_step_uniform(state: UniformMPS, schedule, scheme: str, policy: TruncationPolicy, on_gate=None):
    """proj/src/gates.cpp:513-540."""
    L = state.cell_length()
    if L % 2 != 0:
        raise InputError("uniform TEBD needs an even unit cell")
    s = state.copy()
    reports = []
    for parity, gate in schedule:
        if gate.shape[0] != s.phys_dim:
            raise ShapeError("gate physical dimension mismatch")
        start = 0 if parity == "even" else 1
        for m in range(start, L, 2):
            n = (m + 1) % L
            upd = apply_gate(scheme, s.bond_matrices[m], s.site_tensors[m], s.site_tensors[n], gate, policy)
            s.site_tensors[m] = upd.b_m
            s.bond_matrices[n] = upd.xi_n
            s.site_tensors[n] = upd.b_n
            reports.append((n, upd.report))
            if on_gate:
                on_gate(s, reports[-1])
    return s, reports


def left_weight(xi):
    """proj/src/mps.cpp:44-46: lambda_{aa'} = sum_b Xi_{ba} conj(Xi)_{ba'}."""
    return xi.T @ xi.conj()


def translate_left_weight(lam, b):
    """proj/src/mps.cpp:50-54."""
    t1 = np.einsum("ac,iab->cib", lam, b)
    return np.einsum("cib,icd->bd", t1, b.conj())


def expectation_from_weight(lam, b, op):
    """proj/src/mps.cpp:168-175."""
    t1 = np.einsum("ac,iab->cib", lam, b)  # (a', i, b)
    t2 = np.einsum("cib,jcb->ij", t1, b.conj())  # (i, i')
    return complex(np.einsum("xy,yx->", op, t2))


def expectation_local(mps: UniformMPS, op, site: int) -> complex:
    """proj/src/mps.cpp:179-186."""
    if op.shape != (mps.phys_dim, mps.phys_dim):
        raise ShapeError("operator must be d x d")
    if site >= mps.cell_length():
        raise InputError("site out of range")
    return expectation_from_weight(left_weight(mps.bond_matrices[site]), mps.site_tensors[site], op)


def schmidt_values(mps: UniformMPS, bond: int):
    """proj/src/mps.cpp:198-201."""
    if bond >= mps.cell_length():
        raise InputError("bond out of range")
    return svd(mps.bond_matrices[bond])[1]


def entropy_from_schmidt(values) -> float:
    """proj/src/mps.cpp:209-216."""
    s = 0.0
    for v in values:
        p = float(v) * float(v)
        if p > 0.0:
            s -= p * math.log(p)
    return s


def entanglement_entropy(mps: UniformMPS, bond: int) -> float:
    return entropy_from_schmidt(schmidt_values(mps, bond))


def right_defect(b) -> float:
    """proj/src/mps.cpp:34-36."""
    g = np.einsum("iab,icb->ac", b, b.conj())
    return float(np.max(np.abs(g - np.eye(g.shape[0]))))


def left_defect(b) -> float:
    """proj/src/mps.cpp:39-41."""
    g = np.einsum("iab,iac->bc", b.conj(), b)
    return float(np.max(np.abs(g - np.eye(g.shape[0]))))


def check_isometric_uniform(mps: UniformMPS, tol: float):
    """proj/src/mps.cpp:105-141; returns (pass, max_defect, parts dict)."""
    L = mps.cell_length()
    right = [right_defect(b) for b in mps.site_tensors]
    lams = [left_weight(x) for x in mps.bond_matrices]
    norm = [abs(np.linalg.norm(x) - 1.0) for x in mps.bond_matrices]
    trans, left = [], []
    for m in range(L):
        moved = translate_left_weight(lams[m], mps.site_tensors[m])
        trans.append(float(np.max(np.abs(moved - lams[(m + 1) % L]))))
        cell = lams[m]
        for k in range(L):
            cell = translate_left_weight(cell, mps.site_tensors[(m + k) % L])
        left.append(float(np.max(np.abs(cell - lams[m]))))
    mx = max(max(right), max(left), max(trans), max(norm))
    return mx <= tol, mx, dict(right=right, left=left, translation=trans, norm=norm)


def bond_energy(xi, b_m, b_n, h_bond) -> float:
    """EXTENSION (not in the reference):
    E = <theta0|h|theta0>/<theta0|theta0>, theta0 = Xi B^m B^n (build_theta
    without the gate, proj/src/gates.cpp:123-182)."""
    d = b_m.shape[0]
    t0 = build_theta(xi, b_m, b_n, identity_gate(d))
    th = build_theta(xi, b_m, b_n, h_bond.reshape(d, d, d, d))
    n2 = float(np.vdot(t0.theta, t0.theta).real)
    return float(np.vdot(t0.theta, th.theta).real) / n2 if n2 > 0 else 0.0


# --------------------------------------------------------------------- finite (Hastings form)
def tebd_step_finite_hastings(sites: List[np.ndarray], bonds: List[np.ndarray], layers, scheme: str,
                              policy: TruncationPolicy):
    """Finite open chain in Hastings form: the
    uniform step of proj/src/gates.cpp:513-540 without the wraparound bond,
    bonds[m] = Xi on the bond left of site m (bonds[0] = [[1]]), layers =
    [(parity, [gate per bond m])].  This is the algorithm the sharded device
    chain runs; it agrees with the reference's sequential FiniteMPS step
    (proj/src/gates.cpp:542-578) while truncation is negligible."""
    n_sites = len(sites)
    sites = [s.copy() for s in sites]
    bonds = [b.copy() for b in bonds]
    reports = []
    for parity, gates in layers:
        start = 0 if parity == "even" else 1
        for m in range(start, n_sites - 1, 2):
            upd = apply_gate(scheme, bonds[m], sites[m], sites[m + 1], gates[m], policy)
            sites[m] = upd.b_m
            bonds[m + 1] = upd.xi_n
            sites[m + 1] = upd.b_n
            reports.append((m + 1, upd.report))
    return sites, bonds, reports


# --------------------------------------------------------------------- finite (reference semantics)
@dataclass
class FiniteMPS:
    """proj/include/qrtebd/mps.hpp:31-38: sites < center_bond left-isometric,
    sites >= center_bond right-isometric, center matrix on center_bond."""

    phys_dim: int
    site_tensors: List[np.ndarray]
    center_bond: int
    center_matrix: np.ndarray

    def length(self):
        return len(self.site_tensors)

    def copy(self):
        return FiniteMPS(self.phys_dim, [t.copy() for t in self.site_tensors], self.center_bond,
                         self.center_matrix.copy())


def product_state_finite(d: int, n_sites: int, local_vector) -> FiniteMPS:
    """proj/src/mps.cpp:93-102."""
    if n_sites == 0:
        raise InputError("chain length must be positive")
    v = np.asarray(local_vector, dtype=cplx)
    if v.shape != (d,):
        raise ShapeError("local vector length must equal d")
    n2 = float(np.vdot(v, v).real)
    if n2 <= 0.0:
        raise InputError("local vector has zero norm")
    v = v / math.sqrt(n2)
    return FiniteMPS(d, [v.reshape(d, 1, 1).copy() for _ in range(n_sites)], 0, np.eye(1, dtype=cplx))


def move_center(mps: FiniteMPS, new_center: int) -> FiniteMPS:
    """proj/src/mps.cpp:226-257 (returns a moved copy)."""
    if new_center > mps.length():
        raise InputError("center bond out of range")
    s = mps.copy()
    d = s.phys_dim
    while s.center_bond < new_center:
        c = s.center_bond
        m = np.einsum("aq,iqb->aib", s.center_matrix, s.site_tensors[c])  # (a, i, b), mps.cpp:232-233
        chi_l, chi_r = m.shape[0], m.shape[2]
        q, r = qr_reduced(m.reshape(chi_l * d, chi_r))
        k = q.shape[1]
        s.site_tensors[c] = np.ascontiguousarray(q.reshape(chi_l, d, k).transpose(1, 0, 2))
        s.center_matrix = r
        s.center_bond = c + 1
    while s.center_bond > new_center:
        c = s.center_bond
        m = np.einsum("iab,bg->iag", s.site_tensors[c - 1], s.center_matrix)  # (i, a, g), mps.cpp:244-245
        chi_l, chi_r = m.shape[1], m.shape[2]
        l, q = lq_reduced(m.transpose(1, 0, 2).reshape(chi_l, d * chi_r))
        k = q.shape[0]
        s.site_tensors[c - 1] = np.ascontiguousarray(q.reshape(k, d, chi_r).transpose(1, 0, 2))
        s.center_matrix = l
        s.center_bond = c - 1
    return s


def expectation_local_finite(mps: FiniteMPS, op, site: int) -> complex:
    """proj/src/mps.cpp:188-196."""
    if op.shape != (mps.phys_dim, mps.phys_dim):
        raise ShapeError("operator must be d x d")
    if site >= mps.length():
        raise InputError("site out of range")
    c = move_center(mps, site)
    return expectation_from_weight(left_weight(c.center_matrix), c.site_tensors[site], op)


def schmidt_values_finite(mps: FiniteMPS, bond: int):
    """proj/src/mps.cpp:203-207."""
    if bond > mps.length():
        raise InputError("bond out of range")
    return svd(move_center(mps, bond).center_matrix)[1]


def check_isometric_finite(mps: FiniteMPS, tol: float):
    """proj/src/mps.cpp:143-164; returns (pass, max_defect, parts)."""
    n = mps.length()
    right = [0.0] * n
    left = [0.0] * n
    for s in range(n):
        if s < mps.center_bond:
            left[s] = left_defect(mps.site_tensors[s])
        else:
            right[s] = right_defect(mps.site_tensors[s])
    norm = [abs(np.linalg.norm(mps.center_matrix) - 1.0)]
    mx = max(max(right), max(left), norm[0])
    return mx <= tol, mx, dict(right=right, left=left, norm=norm)


def finite_layers(d: int, g: float, n_sites: int, dt: float, order: int):
    """finite_trotter_layers with chain_bond_hamiltonian (proj/include/qrtebd/gates.hpp:160-173,
    proj/src/clock.cpp:92-99): [(parity, [gate per bond])]."""
    return [(p, [make_gate(chain_bond_hamiltonian(d, g, b, n_sites), dte) for b in range(n_sites - 1)])
            for p, dte in layer_structure(dt, order)]


def tebd_step_finite(state: FiniteMPS, layers, scheme: str, policy: TruncationPolicy, on_gate=None):
    """proj/src/gates.cpp:542-578: sequential, center moved onto every bond."""
    s = state.copy()
    n_sites = s.length()
    reports = []
    for parity, gates in layers:
        if len(gates) + 1 != n_sites:
            raise ShapeError("layer gate count must equal the bond count")
        start = 0 if parity == "even" else 1
        for m in range(start, n_sites - 1, 2):
            s = move_center(s, m)
            upd = apply_gate(scheme, s.center_matrix, s.site_tensors[m], s.site_tensors[m + 1], gates[m], policy)
            if upd.left_iso is not None:
                s.site_tensors[m] = upd.left_iso
                s.center_matrix = upd.xi_n
                s.center_bond = m + 1
            else:
                b_m = upd.b_m
                eps = upd.report.eps_trunc
                if not policy.skip_renormalize and 0.0 < eps < 1.0:
                    b_m = b_m * (1.0 / math.sqrt(1.0 - eps))
                s.site_tensors[m] = b_m
            s.site_tensors[m + 1] = upd.b_n
            reports.append((m + 1, upd.report))
            if on_gate:
                on_gate(s, reports[-1])
    return s, reports


# --------------------------------------------------------------------- quench driver
def run_quench_rows(d: int, g: float, kind: str, size: int, dt: float, t_max: float, order: int, scheme: str,
                    policy: TruncationPolicy):
    """run_quench, proj/src/run.cpp:228-326, without the file output: returns
    one dict per step {t, z[site], entropy[bond], eps[bond], chi[bond],
    bond_ids, max_eps, max_chi}."""
    z_op = clock_operators(d)[0]
    z1 = np.zeros(d, dtype=cplx)
    z1[0] = 1.0
    if kind == "uniform":
        ustate = product_state_uniform(d, size, z1)
        schedule = trotter_schedule(bond_hamiltonian(d, g, "bulk"), dt, order)
        bond_ids = list(range(size))
    else:
        fstate = product_state_finite(d, size, z1)
        layers = finite_layers(d, g, size, dt, order)
        bond_ids = list(range(1, size))
    n_steps = int(math.floor(t_max / dt + 1e-9))
    rows = []
    for k in range(1, n_steps + 1):
        if kind == "uniform":
            ustate, reports = tebd_step_uniform(ustate, schedule, scheme, policy)
            z = [expectation_local(ustate, z_op, s) for s in range(size)]
            spectra = {b: schmidt_values(ustate, b) for b in bond_ids}
        else:
            fstate, reports = tebd_step_finite(fstate, layers, scheme, policy)
            z = [expectation_local_finite(fstate, z_op, s) for s in range(size)]
            spectra = {b: schmidt_values_finite(fstate, b) for b in bond_ids}
        row = dict(t=k * dt, z=z, bond_ids=bond_ids, entropy=[], eps=[], chi=[])
        for b in bond_ids:
            row["entropy"].append(entropy_from_schmidt(spectra[b]))
            row["chi"].append(len(spectra[b]))
            row["eps"].append(max([0.0] + [r.eps_trunc for bb, r in reports if bb == b]))
        row["max_eps"] = max([0.0] + [r.eps_trunc for _, r in reports])
        row["max_chi"] = max(row["chi"])
        rows.append(row)
    return rows


# --------------------------------------------------------------------- ED helpers
def two_site_ed_schmidt(u, v, w):
    """proj/tests/test_gates.cc:50-60: Schmidt values of U (v x w)."""
    psi = np.outer(v, w)
    ev = np.einsum("abij,ij->ab", u, psi)
    return svd(ev)[1]


# --------------------------------------------------------------------- inputs
def random_right_isometry(rng: np.random.Generator, d: int, chi_l: int, chi_r: int) -> np.ndarray:
    """random right-isometric site tensor via LQ of a Gaussian
    (proj/src/run.cpp:345-349, proj/tests/test_gates.cc:19-23)."""
    g = rng.standard_normal((chi_l, d * chi_r)) + 1j * rng.standard_normal((chi_l, d * chi_r))
    _, q = lq_reduced(g)
    return np.ascontiguousarray(q.reshape(chi_l, d, chi_r).transpose(1, 0, 2))


def bench_cell_inputs(d: int, chi: int, scheme: str, seed: int = 0x51AB, g: float = 2.0, dt: float = 0.05):
    """bench_cell input recipe, proj/src/run.cpp:351-391 (NumPy PCG64 stream
    instead of libstdc++'s mt19937_64 + normal_distribution, whose output is
    implementation-defined): B = random right isometries, Xi Gaussian (qr) or
    diag(exp(-4k/chi)) (spectral schemes), gate g=2, dt=0.05, policy chi_max=chi,
    cutoff 0, explicit error off, delta_abs 0, delta_rel 0.1 for qr_cbe."""
    rng = np.random.default_rng([seed, d, chi, {"svd": 0, "eig": 1, "qr": 2, "qr_cbe": 3}[scheme]])
    b_m = random_right_isometry(rng, d, chi, chi)
    b_n = random_right_isometry(rng, d, chi, chi)
    if scheme == "qr":
        xi = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi))
        xi = xi / np.linalg.norm(xi)
    else:
        v = np.exp(-4.0 * np.arange(chi) / chi)
        xi = np.diag(v / np.linalg.norm(v)).astype(cplx)
    gate = make_gate(bond_hamiltonian(d, g, "bulk"), dt)
    pol = TruncationPolicy(chi_max=chi, sv_cutoff=0.0, compute_explicit_error=False, delta_chi_abs=0,
                           delta_chi_rel=0.1 if scheme == "qr_cbe" else 0.0)
    return xi.astype(cplx), b_m, b_n, gate, pol


def flops_per_update(d: int, chi: int, eta: int, kk: int, explicit: bool, cbe: bool = False) -> float:
    """Algorithmic flop count of one update; complex MAC = 8."""
    f = 8.0 * (2 * d * d * chi ** 3 + d ** 4 * chi ** 2 + 2 * d * d * chi * chi * eta + d * d * chi * chi * kk)
    f += 2.0 * (16.0 * (d * chi) * eta * eta - 16.0 / 3.0 * eta ** 3)
    if explicit:
        f += 8.0 * (eta * eta * d * chi + d * d * chi * chi * eta)
    if cbe:
        f += 8.0 * (eta ** 3 + kk * eta * d * chi)
        if explicit:
            f += 8.0 * (eta * eta * kk + eta ** 3)
    return f
