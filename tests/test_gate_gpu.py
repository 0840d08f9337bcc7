"""Single-update parity of the device apply_gate_qr against the oracle
 and the QR known-answer tests of
proj/tests/test_gates.cc:271-367, :431-498."""
import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import model
from paper_2212_09782_b200 import qrtebd as q

pytestmark = pytest.mark.gpu


def block_of(xi, b_m, b_n):
    """gauge-invariant two-site block (proj/tests/test_gates.cc:32-37)"""
    phi = np.einsum("iag,jgc->aijc", b_m, b_n)
    return np.einsum("xa,aijc->xijc", xi, phi)


def random_inputs(d, chi, seed, chi_l=None, chi_r=None):
    rng = np.random.default_rng(seed)
    chi_l = chi_l or chi
    chi_r = chi_r or chi
    bm = ref.random_right_isometry(rng, d, chi_l, chi)
    bn = ref.random_right_isometry(rng, d, chi, chi_r)
    xi = rng.standard_normal((chi_l, chi_l)) + 1j * rng.standard_normal((chi_l, chi_l))
    xi /= np.linalg.norm(xi)
    return xi, bm, bn


def compare(upd, o, xi_old, tol_block=1e-10):
    """Appendix B.1 checks between a device GateUpdate and an oracle GateUpdate."""
    bm, xin, bn = upd.b_m.numpy(), upd.xi_n.numpy(), upd.b_n.numpy()
    assert bm.shape == o.b_m.shape and xin.shape == o.xi_n.shape and bn.shape == o.b_n.shape
    # (i) gauge-invariant two-site block Xi_old B~m B~n (Hastings form,
    # proj/tests/test_gates.cc:40-43)
    blk_d = block_of(xi_old, bm, bn)
    blk_o = block_of(xi_old, o.b_m, o.b_n)
    assert np.linalg.norm(blk_d - blk_o) / np.linalg.norm(blk_o) < tol_block
    s_d = np.linalg.svd(xin, compute_uv=False)
    s_o = np.linalg.svd(o.xi_n, compute_uv=False)
    assert np.max(np.abs(s_d - s_o)) <= 1e-10 * s_o[0]
    r, ro = upd.report, o.report
    assert (r.chi_before, r.chi_expanded, r.chi_after) == (ro.chi_before, ro.chi_expanded, ro.chi_after)
    assert abs(r.eps_trunc - ro.eps_trunc) <= 1e-10 * abs(ro.eps_trunc) + 1e-20
    gram = np.einsum("iab,icb->ac", bn, bn.conj())
    assert np.max(np.abs(gram - np.eye(gram.shape[0]))) < 1e-12


@pytest.mark.parametrize("d,chi,eta_pol", [(2, 8, 0), (3, 16, 0), (5, 20, 0), (2, 16, 100), (5, 12, 4),
                                           (4, 40, 0), (5, 64, 0)])
def test_apply_gate_qr_matches_oracle(ctx, d, chi, eta_pol):
    xi, bm, bn = random_inputs(d, chi, seed=100 * d + chi)
    gate = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
    pol = dict(chi_max=chi + eta_pol, sv_cutoff=1e-14, delta_chi_abs=eta_pol, delta_chi_rel=0.0)
    o = ref.apply_gate_qr(xi, bm, bn, gate, ref.TruncationPolicy(**pol))
    upd = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(**pol), ctx)
    compare(upd, o, xi)
    li = upd.left_iso.numpy()
    assert np.linalg.norm(li - o.left_iso) / np.linalg.norm(o.left_iso) < 1e-10


def test_identity_gate_exact_fixed_point(ctx):
    # proj/tests/test_gates.cc:271-287
    rng = np.random.default_rng(240)
    d = 2
    xi = np.diag([np.sqrt(0.8), np.sqrt(0.2)]).astype(complex)
    bm = ref.random_right_isometry(rng, d, 2, 2)
    bn = ref.random_right_isometry(rng, d, 2, 2)
    pol = q.TruncationPolicy(chi_max=2, delta_chi_abs=0, delta_chi_rel=0.0)
    upd = q.apply_gate_qr(xi, bm, bn, model.identity_gate(d), pol, ctx)
    assert upd.report.eps_trunc <= 1e-14
    assert upd.report.chi_after == 2
    before = block_of(xi, bm, bn)
    after = block_of(xi, upd.b_m.numpy(), upd.b_n.numpy())
    assert np.max(np.abs(before - after)) < 1e-13
    oracle = np.linalg.svd(before.reshape(4, 4), compute_uv=False)
    got = np.linalg.svd(upd.xi_n.numpy(), compute_uv=False)
    assert np.allclose(got, oracle[:2], atol=1e-12)


def test_heuristic_expansion_from_product_state(ctx):
    # proj/tests/test_gates.cc:354-367
    d = 4
    site = np.zeros((d, 1, 1), dtype=complex)
    site[0, 0, 0] = 1.0
    gate = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.1)
    pol = q.TruncationPolicy(chi_max=64)
    upd = q.apply_gate_qr(np.eye(1, dtype=complex), site, site, gate, pol, ctx)
    assert upd.report.chi_expanded == 4 and upd.report.chi_after == 4
    assert upd.report.eps_trunc <= 1e-13
    o = ref.apply_gate_qr(np.eye(1, dtype=complex), site, site, gate, ref.TruncationPolicy(chi_max=64))
    compare(upd, o, np.eye(1, dtype=complex))


def test_qr_sweeps_and_skip_renormalize(ctx):
    xi, bm, bn = random_inputs(2, 8, seed=255)
    u = ref.qr_reduced(np.random.default_rng(258).standard_normal((4, 4)) + 0j)[0].reshape(2, 2, 2, 2)
    for sweeps in (1, 3):
        for skip in (False, True):
            pol = dict(chi_max=8, delta_chi_abs=0, delta_chi_rel=0.0, qr_sweeps=sweeps, skip_renormalize=skip)
            o = ref.apply_gate_qr(xi, bm, bn, u, ref.TruncationPolicy(**pol))
            upd = q.apply_gate_qr(xi, bm, bn, u, q.TruncationPolicy(**pol), ctx)
            compare(upd, o, xi)
            # L is unique after the gauge fix: compare Xi~ directly
            assert np.max(np.abs(upd.xi_n.numpy() - o.xi_n)) < 1e-11


def test_explicit_error_off_uses_discarded_weight(ctx):
    xi, bm, bn = random_inputs(3, 16, seed=77)
    gate = model.make_gate(model.bond_hamiltonian(3, 2.0), 0.3)
    pol = dict(chi_max=16, delta_chi_abs=0, delta_chi_rel=0.0, compute_explicit_error=False)
    o = ref.apply_gate_qr(xi, bm, bn, gate, ref.TruncationPolicy(**pol))
    upd = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(**pol), ctx)
    assert abs(upd.report.discarded_weight - o.report.discarded_weight) <= 1e-12
    assert abs(upd.report.eps_trunc - o.report.eps_trunc) <= 1e-10 * o.report.eps_trunc + 1e-14


def test_truncation_error_explicit_known_answer(ctx):
    # proj/tests/test_gates.cc:465-478: rank-1 approximation of a rank-2 block loses 0.1
    u = np.zeros((4, 2), dtype=complex)
    u[0, 0] = u[1, 1] = 1.0
    v = np.zeros((2, 4), dtype=complex)
    v[0, 0] = v[1, 1] = 1.0
    s = np.diag([np.sqrt(0.9), np.sqrt(0.1)]).astype(complex)
    theta = u @ s @ v
    eps = q.truncation_error_explicit(theta, u[:, :1].copy(), s[:1, :1].copy(), v[:1].copy(), ctx)
    assert abs(eps - 0.1) < 1e-14


def test_update_is_deterministic(ctx):
    xi, bm, bn = random_inputs(3, 24, seed=5)
    gate = model.make_gate(model.bond_hamiltonian(3, 2.0), 0.05)
    pol = q.TruncationPolicy(chi_max=24)
    a = q.apply_gate_qr(xi, bm, bn, gate, pol, ctx)
    b = q.apply_gate_qr(xi, bm, bn, gate, pol, ctx)
    assert np.array_equal(a.b_m.numpy(), b.b_m.numpy())
    assert np.array_equal(a.xi_n.numpy(), b.xi_n.numpy())
    assert a.report.eps_trunc == b.report.eps_trunc


def test_shape_errors(ctx):
    xi, bm, bn = random_inputs(2, 4, seed=1)
    gate = model.identity_gate(3)
    with pytest.raises(q.ShapeError):
        q.apply_gate_qr(xi, bm, bn, gate, None, ctx)
    with pytest.raises(q.ShapeError):
        q.apply_gate_qr(np.eye(3, dtype=complex), bm, bn, model.identity_gate(2), None, ctx)
