"""Pins the CPU oracle (oracle/qrtebd_oracle.py) to the reference's own
known-answer tests.  The reference ships no golden-vector files; its tests
(proj/tests/*.cc, acceptance.cc) pin behaviour by known answers and
tolerances, re-run here against the restatement (CPU only)."""
import math

import numpy as np
import pytest

from oracle import qrtebd_oracle as ref


def crand(seed, *shape):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def random_right_iso(d, chi_l, chi_r, seed):
    return ref.random_right_isometry(np.random.default_rng(seed), d, chi_l, chi_r)


def random_bond_matrix(chi, seed):
    x = crand(seed, chi, chi)
    return x / np.linalg.norm(x)


def block_of(xi, bm, bn):
    return np.einsum("xa,iag,jgc->xijc", xi, bm, bn)


def exact_policy(**kw):
    p = ref.TruncationPolicy(chi_max=4096, sv_cutoff=1e-14)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def random_hermitian(n, seed):
    a = crand(seed, n, n)
    return 0.5 * (a + a.conj().T)


# ---------------------------------------------------------------- policy
def test_expansion_rule_known_answers():
    # proj/tests/test_gates.cc:489-498
    p = ref.TruncationPolicy(delta_chi_abs=100, delta_chi_rel=0.1)
    assert p.expanded_dim(256, 5) == 356
    assert p.expanded_dim(1, 5) == 5
    assert p.expanded_dim(2000, 5) == 2200
    p.chi_max_expansion = 300
    assert p.expanded_dim(256, 5) == 300


def test_choose_kept_rules():
    p = ref.TruncationPolicy(chi_max=3, sv_cutoff=1e-3)
    assert ref.choose_kept([0.9, 0.4, 0.1, 1e-4, 0.5], p) == 3
    assert ref.choose_kept([1e-5, 1e-6], p) == 1  # at least one
    p = ref.TruncationPolicy(chi_max=10, sv_cutoff=0.0, target_eps=0.02)
    assert ref.choose_kept([0.9, 0.4, 0.1, 0.05], p) == 2  # tail 0.0125 <= 0.02


# ---------------------------------------------------------------- linalg
def test_qr_known_answer():
    # proj/tests/test_linalg.cc:51-58
    q, r = ref.qr_reduced(np.array([[3.0], [4.0]], dtype=complex))
    assert np.allclose(q, [[0.6], [0.8]], atol=1e-15) and np.allclose(r, [[5.0]], atol=1e-14)


@pytest.mark.parametrize("shape", [(8, 5), (5, 8), (30, 30), (2048, 16)])
def test_qr_lq_reconstruction_and_gauge(shape):
    a = crand(7, *shape)
    q, r = ref.qr_reduced(a)
    k = min(shape)
    assert np.linalg.norm(q @ r - a) / np.linalg.norm(a) < 1e-12
    assert np.max(np.abs(q.conj().T @ q - np.eye(k))) < 1e-12
    assert np.allclose(np.diag(r).imag, 0) and np.all(np.diag(r).real >= 0)
    l, qq = ref.lq_reduced(a)
    assert np.linalg.norm(l @ qq - a) / np.linalg.norm(a) < 1e-12
    # LQ = adjoint QR of the adjoint (proj/tests/test_linalg.cc:92-99)
    q2, r2 = ref.qr_reduced(a.conj().T)
    assert np.max(np.abs(l - r2.conj().T)) < 1e-13


def test_qr_is_deterministic():
    a = crand(3, 40, 20)
    q1, r1 = ref.qr_reduced(a)
    q2, r2 = ref.qr_reduced(a)
    assert np.array_equal(q1, q2) and np.array_equal(r1, r2)


def test_nonfinite_input_rejected():
    a = np.ones((3, 3), dtype=complex)
    a[0, 0] = np.inf
    with pytest.raises(ref.InputError):
        ref.qr_reduced(a)


def test_eigh_descending_and_hermiticity_check():
    h = random_hermitian(12, 4)
    w, v = ref.eigh(h)
    assert np.all(np.diff(w) <= 0)
    assert np.linalg.norm(h @ v - v * w) < 1e-12
    with pytest.raises(ref.InputError):
        ref.eigh(crand(5, 4, 4))


def test_expm_matches_taylor():
    h = random_hermitian(6, 9) * 0.1
    u = ref.expm_hermitian(h, 0.3)
    t, term = np.eye(6, dtype=complex), np.eye(6, dtype=complex)
    for k in range(1, 30):
        term = term @ (-1j * 0.3 * h) / k
        t = t + term
    assert np.max(np.abs(u - t)) < 1e-13


# ---------------------------------------------------------------- model
def test_clock_algebra():
    for d in (2, 3, 5):
        z, x = ref.clock_operators(d)
        w = np.exp(2j * math.pi / d)
        assert np.max(np.abs(x @ z - w * z @ x)) < 1e-14


def test_trotter_schedule_structure():
    h = ref.bond_hamiltonian(3, 2.0)
    sched = ref.trotter_schedule(h, 0.0, 2)
    assert [p for p, _ in sched] == ["even", "odd", "even"]
    for _, g in sched:
        assert np.max(np.abs(g.reshape(9, 9) - np.eye(9))) < 1e-13
    h2 = ref.bond_hamiltonian(2, 2.0)
    s = ref.trotter_schedule(h2, 0.1, 2)
    composed = s[0][1].reshape(4, 4) @ s[2][1].reshape(4, 4)
    assert np.max(np.abs(composed - ref.make_gate(h2, 0.1).reshape(4, 4))) < 1e-13
    with pytest.raises(ref.InputError):
        ref.trotter_schedule(h2, 0.1, 3)


# ---------------------------------------------------------------- QR scheme
def canonical_chi2(d, seed):
    xi = np.diag([math.sqrt(0.8), math.sqrt(0.2)]).astype(complex)
    return xi, random_right_iso(d, 2, 2, seed), random_right_iso(d, 2, 2, seed + 1)


def test_qr_identity_gate_exact_fixed_point():
    # proj/tests/test_gates.cc:271-287
    xi, bm, bn = canonical_chi2(2, 240)
    p = exact_policy(chi_max=2, delta_chi_abs=0, delta_chi_rel=0.0)
    upd = ref.apply_gate_qr(xi, bm, bn, ref.identity_gate(2), p)
    assert upd.report.eps_trunc <= 1e-14 and upd.report.chi_after == 2
    assert np.max(np.abs(block_of(xi, bm, bn) - block_of(xi, upd.b_m, upd.b_n))) < 1e-13
    oracle = np.linalg.svd(block_of(xi, bm, bn).reshape(4, 4), compute_uv=False)
    assert np.allclose(np.linalg.svd(upd.xi_n, compute_uv=False), oracle[:2], atol=1e-12)


def test_qr_new_right_tensor_isometric():
    # proj/tests/test_gates.cc:289-309
    d, chi = 5, 6
    xi = random_bond_matrix(chi, 250)
    bm, bn = random_right_iso(d, chi, chi, 251), random_right_iso(d, chi, chi, 252)
    gate = ref.make_gate(ref.bond_hamiltonian(d, 2.0), 0.05)
    upd = ref.apply_gate_qr(xi, bm, bn, gate, exact_policy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0))
    assert ref.right_defect(upd.b_n) < 1e-12
    assert ref.left_defect(upd.left_iso) < 1e-12


def test_qr_within_factor_two_of_svd():
    # proj/tests/test_gates.cc:311-330
    d, chi = 3, 16
    for seed in range(5):
        xi = random_bond_matrix(chi, 260 + 10 * seed)
        bm = random_right_iso(d, chi, chi, 261 + 10 * seed)
        bn = random_right_iso(d, chi, chi, 262 + 10 * seed)
        gate = ref.make_gate(random_hermitian(d * d, 263 + 10 * seed), 0.01)
        p = exact_policy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
        qv = ref.apply_gate_qr(xi, bm, bn, gate, p).report.eps_trunc
        sv = ref.apply_gate_svd(xi, bm, bn, gate, p).report.eps_trunc
        assert sv - 1e-15 <= qv <= 2.0 * sv + 1e-15


def test_qr_extra_sweeps_not_worse():
    # proj/tests/test_gates.cc:332-352
    d, chi = 2, 8
    xi = random_bond_matrix(chi, 255)
    bm, bn = random_right_iso(d, chi, chi, 256), random_right_iso(d, chi, chi, 257)
    gate = ref.qr_reduced(crand(258, 4, 4))[0].reshape(2, 2, 2, 2)
    p = exact_policy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
    one = ref.apply_gate_qr(xi, bm, bn, gate, p).report.eps_trunc
    p.qr_sweeps = 6
    six = ref.apply_gate_qr(xi, bm, bn, gate, p).report.eps_trunc
    opt = ref.apply_gate_svd(xi, bm, bn, gate, p).report.eps_trunc
    assert six <= one + 1e-13 and six >= opt - 1e-13


def test_qr_heuristic_expansion_from_product_state():
    # proj/tests/test_gates.cc:354-367
    d = 4
    site = np.zeros((d, 1, 1), dtype=complex)
    site[0, 0, 0] = 1
    gate = ref.make_gate(ref.bond_hamiltonian(d, 2.0), 0.1)
    upd = ref.apply_gate_qr(np.eye(1, dtype=complex), site, site, gate, exact_policy(chi_max=64))
    assert upd.report.chi_expanded == 4 and upd.report.chi_after == 4 and upd.report.eps_trunc <= 1e-13


# ---------------------------------------------------------------- CBE
def test_cbe_first_gate_matches_two_site_ed():
    # proj/tests/test_gates.cc:371-385
    d = 5
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    site = v.reshape(d, 1, 1)
    gate = ref.make_gate(ref.bond_hamiltonian(d, 2.0), 0.05)
    upd = ref.apply_gate_qr_cbe(np.eye(1, dtype=complex), site, site, gate, exact_policy())
    oracle = ref.two_site_ed_schmidt(gate, v, v)
    assert upd.report.chi_expanded == 5
    for k in range(upd.report.chi_after):
        assert abs(upd.xi_n[k, k].real - oracle[k]) < 1e-12


def test_cbe_identity_equals_qr_with_diagonal_bond():
    # proj/tests/test_gates.cc:387-408
    xi, bm, bn = canonical_chi2(3, 270)
    p = exact_policy(chi_max=2, delta_chi_abs=0, delta_chi_rel=0.0)
    cbe = ref.apply_gate_qr_cbe(xi, bm, bn, ref.identity_gate(3), p)
    qr = ref.apply_gate_qr(xi, bm, bn, ref.identity_gate(3), p)
    assert np.max(np.abs(block_of(xi, cbe.b_m, cbe.b_n) - block_of(xi, qr.b_m, qr.b_n))) < 1e-12
    assert abs(cbe.xi_n[0, 1]) < 1e-14 and abs(cbe.xi_n[1, 0]) < 1e-14
    oracle = np.linalg.svd(block_of(xi, bm, bn).reshape(6, 6), compute_uv=False)
    assert abs(cbe.xi_n[0, 0].real - oracle[0]) < 1e-12 and abs(cbe.xi_n[1, 1].real - oracle[1]) < 1e-12


def test_cbe_expansion_rule():
    # proj/tests/test_gates.cc:410-427
    d, chi = 5, 20
    xi = random_bond_matrix(chi, 280)
    bm, bn = random_right_iso(d, chi, chi, 281), random_right_iso(d, chi, chi, 282)
    gate = ref.make_gate(ref.bond_hamiltonian(d, 2.0), 0.05)
    upd = ref.apply_gate_qr_cbe(xi, bm, bn, gate, exact_policy(chi_max=chi, delta_chi_abs=4, delta_chi_rel=0.1))
    assert upd.report.chi_expanded == 24 and upd.report.chi_after == chi
    dg = np.diag(upd.xi_n).real
    assert np.all(dg[:-1] >= dg[1:])


# ---------------------------------------------------------------- explicit error
def test_explicit_error_known_answers():
    # proj/tests/test_gates.cc:431-478
    theta = crand(290, 8, 12)
    q, r = ref.qr_reduced(theta)
    assert ref.truncation_error_explicit(theta, q, r, np.eye(12, dtype=complex)) <= 1e-14
    theta = crand(291, 12, 12)
    u, s, vh = ref.svd(theta)
    keep = 5
    eps = ref.truncation_error_explicit(theta, u[:, :keep], np.diag(s[:keep]).astype(complex), vh[:keep])
    assert abs(eps - np.sum(s[keep:] ** 2) / np.sum(s ** 2)) < 1e-12
    u2 = np.zeros((4, 2), dtype=complex)
    u2[0, 0] = u2[1, 1] = 1
    v2 = u2.T.copy()
    s2 = np.diag([math.sqrt(0.9), math.sqrt(0.1)]).astype(complex)
    th2 = u2 @ s2 @ v2
    assert abs(ref.truncation_error_explicit(th2, u2[:, :1], s2[:1, :1], v2[:1]) - 0.1) < 1e-14
    with pytest.raises(ref.ShapeError):
        ref.truncation_error_explicit(crand(292, 4, 4), np.eye(3), np.eye(3), np.eye(4))


def test_degenerate_values_cut_deterministically():
    # proj/tests/test_gates.cc:500-514
    d = 2
    xi = np.diag([0.5] * 4).astype(complex)
    bm, bn = random_right_iso(d, 4, 4, 293), random_right_iso(d, 4, 4, 294)
    p = exact_policy(chi_max=2)
    a = ref.apply_gate_svd(xi, bm, bn, ref.identity_gate(d), p)
    b = ref.apply_gate_svd(xi, bm, bn, ref.identity_gate(d), p)
    assert a.report.chi_after == 2 and np.array_equal(a.xi_n, b.xi_n) and np.array_equal(a.b_n, b.b_n)


# ---------------------------------------------------------------- TEBD step
def e0(d):
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    return v


def test_schemes_agree_on_observables():
    # proj/tests/test_tebd.cc:103-137: 4 schemes agree to 1e-8
    d = 3
    sched = ref.trotter_schedule(ref.bond_hamiltonian(d, 2.0), 0.05, 2)
    z = ref.clock_operators(d)[0]
    traces = []
    for scheme in ("svd", "eig", "qr", "qr_cbe"):
        st = ref.product_state_uniform(d, 2, e0(d))
        tr = []
        for _ in range(10):
            st, _ = ref.tebd_step_uniform(st, sched, scheme, ref.TruncationPolicy(chi_max=64, sv_cutoff=1e-14))
            for s in range(2):
                tr.append(ref.expectation_local(st, z, s).real)
                tr.append(ref.entanglement_entropy(st, s))
        traces.append(tr)
    for t in traces[1:]:
        assert np.max(np.abs(np.array(t) - np.array(traces[0]))) < 1e-8


def test_identity_schedule_keeps_observables():
    # proj/tests/test_tebd.cc:32-62 (qr, qr_cbe)
    d = 3
    st = ref.product_state_uniform(d, 2, e0(d))
    grow = ref.trotter_schedule(ref.bond_hamiltonian(d, 2.0), 0.1, 2)
    for _ in range(3):
        st, _ = ref.tebd_step_uniform(st, grow, "svd", ref.TruncationPolicy(chi_max=512))
    z = ref.clock_operators(d)[0]
    before = [ref.expectation_local(st, z, s) for s in range(2)]
    ent = [ref.entanglement_entropy(st, s) for s in range(2)]
    ids = ref.trotter_schedule(ref.bond_hamiltonian(d, 2.0), 0.0, 2)
    for scheme in ("qr", "qr_cbe"):
        res, _ = ref.tebd_step_uniform(st, ids, scheme, ref.TruncationPolicy(chi_max=512))
        for s in range(2):
            assert abs(ref.expectation_local(res, z, s) - before[s]) < 1e-12
            assert abs(ref.entanglement_entropy(res, s) - ent[s]) < 1e-12


def test_odd_cell_rejected():
    st = ref.product_state_uniform(2, 3, e0(2))
    with pytest.raises(ref.InputError):
        ref.tebd_step_uniform(st, ref.trotter_schedule(ref.bond_hamiltonian(2, 1.0), 0.1, 1), "qr",
                              ref.TruncationPolicy())


def test_cbe_keeps_canonical_form():
    # proj/tests/test_tebd.cc:272-292: diagonal, descending, non-negative Xi
    d = 3
    st = ref.product_state_uniform(d, 2, e0(d))
    sched = ref.trotter_schedule(ref.bond_hamiltonian(d, 2.0), 0.05, 2)
    for _ in range(8):
        st, _ = ref.tebd_step_uniform(st, sched, "qr_cbe", ref.TruncationPolicy(chi_max=128, sv_cutoff=1e-14))
    for xi in st.bond_matrices:
        off = xi - np.diag(np.diag(xi))
        assert np.max(np.abs(off)) < 1e-10
        dg = np.diag(xi).real
        assert np.all(dg >= 0) and np.all(dg[1:] <= dg[:-1] + 1e-12)


def test_hastings_finite_matches_uniform_logic_untruncated():
    # the sharded-chain algorithm reduces to exact
    # evolution without truncation: compare <Z> with a dense statevector
    d, n = 2, 6
    g = 1.0
    layers = []
    for parity, dte in ref.layer_structure(0.05, 2):
        layers.append((parity, [ref.make_gate(ref.chain_bond_hamiltonian(d, g, m, n), dte) for m in range(n - 1)]))
    sites = [e0(d).reshape(d, 1, 1) for _ in range(n)]
    bonds = [np.eye(1, dtype=complex) for _ in range(n)]
    psi = np.zeros(d ** n, dtype=complex)
    psi[0] = 1
    for _ in range(4):
        sites, bonds, _ = ref.tebd_step_finite_hastings(sites, bonds, layers, "qr_cbe",
                                                        ref.TruncationPolicy(chi_max=64, sv_cutoff=1e-14))
        for parity, gates in layers:
            start = 0 if parity == "even" else 1
            for m in range(start, n - 1, 2):
                u = gates[m].reshape(d * d, d * d)
                t = psi.reshape(d ** m, d * d, d ** (n - m - 2))
                psi = np.einsum("ab,xby->xay", u, t).reshape(-1)
    # <Z_0> from the MPS (left weight = Xi[0] = 1) vs the statevector
    z = ref.clock_operators(d)[0]
    mps_z = ref.expectation_from_weight(ref.left_weight(bonds[0]), sites[0], z)
    t = psi.reshape(d, -1)
    sv_z = np.einsum("ab,ax,bx->", z, t.conj(), t)
    assert abs(mps_z - sv_z) < 1e-10
