"""K5/K9 parity: device Hermitian eigensolver, Schmidt spectra and the
QR+CBE update (proj/src/gates.cpp:388-450) against the oracle and the
reference known answers (proj/tests/test_gates.cc:371-427)."""
import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import model
from paper_2212_09782_b200 import qrtebd as q

pytestmark = pytest.mark.gpu


def crand(rng, *s):
    return rng.standard_normal(s) + 1j * rng.standard_normal(s)


def block_of(xi, b_m, b_n):
    return np.einsum("xa,iag,jgc->xijc", xi, b_m, b_n)


@pytest.mark.parametrize("n", [1, 2, 5, 16, 33, 100, 257, 356, 513, 1100])  # JB = 16 and 32
def test_eigh_matches_lapack(ctx, n):
    rng = np.random.default_rng(n)
    a = crand(rng, n, n)
    h = a + a.conj().T
    w, v = q.eigh(h, ctx)
    V = v.numpy()
    w_ref = np.linalg.eigvalsh(h)[::-1]
    scale = np.linalg.norm(h)
    assert np.max(np.abs(w - w_ref)) <= 1e-13 * scale
    assert np.all(np.diff(w) <= 0)
    assert np.max(np.abs(V.conj().T @ V - np.eye(n))) < 1e-12
    assert np.linalg.norm(h @ V - V * w) <= 1e-12 * scale


def test_eigh_gram_with_zero_eigenvalues(ctx):
    # rank-deficient PSD Gram matrix: the padding must not mix with the zero block
    rng = np.random.default_rng(4)
    l = crand(rng, 40, 12)
    g = l @ l.conj().T
    w, v = q.eigh(g, ctx)
    w_ref = np.linalg.eigvalsh(g)[::-1]
    assert np.max(np.abs(w - w_ref)) <= 1e-12 * np.linalg.norm(g)
    assert np.all(w[12:] > -1e-10 * np.linalg.norm(g))


def test_eigh_is_deterministic(ctx):
    rng = np.random.default_rng(8)
    a = crand(rng, 70, 70)
    h = a + a.conj().T
    w1, v1 = q.eigh(h, ctx)
    w2, v2 = q.eigh(h, ctx)
    assert np.array_equal(w1, w2) and np.array_equal(v1.numpy(), v2.numpy())


@pytest.mark.parametrize("p,qq", [(8, 8), (30, 30), (64, 40), (20, 50), (256, 256)])
def test_schmidt_values_match_svd(ctx, p, qq):
    rng = np.random.default_rng(p + qq)
    m = crand(rng, p, qq)
    s = q.schmidt_values_of(m, ctx)
    s_ref = np.linalg.svd(m, compute_uv=False)
    # max |ds_k| <= 1e-10 s_0 for every k
    assert np.max(np.abs(s - s_ref)) <= 1e-10 * s_ref[0]


@pytest.mark.parametrize("p,qq,decades", [(64, 64, 14), (300, 300, 15), (200, 120, 13), (90, 256, 14), (1024, 1024, 15)])
def test_schmidt_values_graded_spectrum(ctx, p, qq, decades):
    """Dense bond matrices with singular values spread over 13-15 decades (the
    QR scheme's Xi = L/||L|| is dense lower-triangular): every value, the
    smallest included, within 1e-10 s_0 of LAPACK zgesdd -- no filter
    (the reference takes them from BDCSVD,
    proj/src/mps.cpp:198-207)."""
    rng = np.random.default_rng(p * 7 + qq)
    k = min(p, qq)
    u, _ = np.linalg.qr(crand(rng, p, k))
    v, _ = np.linalg.qr(crand(rng, qq, k))
    sv = np.logspace(0, -decades, k)
    m = (u * sv) @ v.conj().T
    s = q.schmidt_values_of(m, ctx)
    s_ref = np.linalg.svd(m, compute_uv=False)
    assert s.shape == s_ref.shape
    assert np.max(np.abs(s - s_ref)) <= 1e-10 * s_ref[0]
    # the entropy, from the same values (mps.cpp:209-216)
    assert abs(q.entropy_from_schmidt(s) - q.entropy_from_schmidt(s_ref)) <= 1e-10


def test_eigh_rejects_non_hermitian(ctx):
    """proj/src/linalg.cpp:82-86: InputError when ||h - h^H|| > 1e-10 ||h||."""
    from paper_2212_09782_b200._capi import InputError
    rng = np.random.default_rng(11)
    a = crand(rng, 20, 20)
    h = a + a.conj().T
    h[3, 5] += 1e-6
    with pytest.raises(InputError, match="hermitian"):
        q.eigh(h, ctx)
    # within tolerance: accepted (symmetrized)
    h2 = a + a.conj().T
    h2[3, 5] += 1e-13
    w, _ = q.eigh(h2, ctx)
    assert np.max(np.abs(w - np.linalg.eigvalsh((h2 + h2.conj().T) / 2)[::-1])) < 1e-12 * np.linalg.norm(h2)


def test_eigh_rejects_non_finite(ctx):
    from paper_2212_09782_b200._capi import InputError
    h = np.eye(8, dtype=complex)
    h[2, 2] = np.nan
    with pytest.raises(InputError):
        q.eigh(h, ctx)


@pytest.mark.parametrize("p,qq", [(1, 1), (7, 7), (300, 300), (12, 20)])
def test_schmidt_values_of_diagonal_bond_are_exact(ctx, p, qq):
    """CBE bond matrices are diagonal (gates.cpp:430): the spectrum is the
    sorted |diagonal| (SURVEY.md §8 a13 fast path) to the rounding of |z|,
    tiny values included -- no Gram-route noise."""
    rng = np.random.default_rng(p * 31 + qq)
    k = min(p, qq)
    mags = np.exp(-rng.uniform(0, 40, k))
    mags[k // 2:k // 2 + 1] = mags[0]  # a tie
    m = np.zeros((p, qq), dtype=complex)
    m[np.arange(k), np.arange(k)] = mags * np.exp(1j * rng.uniform(0, 2 * np.pi, k))
    s = q.schmidt_values_of(m, ctx)
    ref_s = np.sort(np.abs(np.diag(m)))[::-1]
    assert s.shape == ref_s.shape
    assert np.max(np.abs(s - ref_s) / ref_s) <= 4.5e-16  # 2 ulp: device vs host hypot


def random_inputs(d, chi, seed):
    rng = np.random.default_rng(seed)
    bm = ref.random_right_isometry(rng, d, chi, chi)
    bn = ref.random_right_isometry(rng, d, chi, chi)
    v = np.exp(-4.0 * np.arange(chi) / chi)
    xi = np.diag(v / np.linalg.norm(v)).astype(complex)
    return xi, bm, bn


@pytest.mark.parametrize("d,chi,dabs,explicit", [(3, 16, 4, True), (5, 20, 4, True), (2, 32, 8, False),
                                                 (5, 48, 10, True)])
def test_apply_gate_qr_cbe_matches_oracle(ctx, d, chi, dabs, explicit):
    xi, bm, bn = random_inputs(d, chi, 300 + chi)
    gate = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
    kw = dict(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=dabs, delta_chi_rel=0.1, compute_explicit_error=explicit)
    o = ref.apply_gate_qr_cbe(xi, bm, bn, gate, ref.TruncationPolicy(**kw))
    u = q.apply_gate_qr_cbe(xi, bm, bn, gate, q.TruncationPolicy(**kw), ctx)
    assert (u.report.chi_expanded, u.report.chi_after) == (o.report.chi_expanded, o.report.chi_after)
    b_d = block_of(xi, u.b_m.numpy(), u.b_n.numpy())
    b_o = block_of(xi, o.b_m, o.b_n)
    assert np.linalg.norm(b_d - b_o) / np.linalg.norm(b_o) < 1e-10
    xd = u.xi_n.numpy()
    assert np.max(np.abs(xd - np.diag(np.diag(xd)))) == 0.0
    s_d, s_o = np.diag(xd).real, np.diag(o.xi_n).real
    assert np.max(np.abs(s_d - s_o)) <= 1e-10 * s_o[0]
    assert abs(u.report.eps_trunc - o.report.eps_trunc) <= 1e-10 * o.report.eps_trunc + 1e-20
    gram = np.einsum("iab,icb->ac", u.b_n.numpy(), u.b_n.numpy().conj())
    assert np.max(np.abs(gram - np.eye(gram.shape[0]))) < 1e-12


def test_cbe_first_gate_matches_two_site_ed(ctx):
    # proj/tests/test_gates.cc:371-385
    d = 5
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    site = v.reshape(d, 1, 1)
    gate = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
    u = q.apply_gate_qr_cbe(np.eye(1, dtype=complex), site, site, gate,
                            q.TruncationPolicy(chi_max=4096, sv_cutoff=1e-14), ctx)
    oracle = ref.two_site_ed_schmidt(gate, v, v)
    assert u.report.chi_expanded == 5
    xd = u.xi_n.numpy()
    for k in range(u.report.chi_after):
        assert abs(xd[k, k].real - oracle[k]) < 1e-12


def test_cbe_identity_equals_qr_with_diagonal_bond(ctx):
    # proj/tests/test_gates.cc:387-408
    rng = np.random.default_rng(270)
    xi = np.diag([np.sqrt(0.8), np.sqrt(0.2)]).astype(complex)
    bm = ref.random_right_isometry(rng, 3, 2, 2)
    bn = ref.random_right_isometry(rng, 3, 2, 2)
    pol = q.TruncationPolicy(chi_max=2, delta_chi_abs=0, delta_chi_rel=0.0)
    cbe = q.apply_gate_qr_cbe(xi, bm, bn, model.identity_gate(3), pol, ctx)
    qr = q.apply_gate_qr(xi, bm, bn, model.identity_gate(3), pol, ctx)
    assert np.max(np.abs(block_of(xi, cbe.b_m.numpy(), cbe.b_n.numpy()) -
                         block_of(xi, qr.b_m.numpy(), qr.b_n.numpy()))) < 1e-12
    oracle = np.linalg.svd(block_of(xi, bm, bn).reshape(6, 6), compute_uv=False)
    xd = cbe.xi_n.numpy()
    assert abs(xd[0, 1]) < 1e-14 and abs(xd[1, 0]) < 1e-14
    assert abs(xd[0, 0].real - oracle[0]) < 1e-12 and abs(xd[1, 1].real - oracle[1]) < 1e-12


def test_cbe_width_is_capped_at_d_chi(ctx):
    # expanded_dim already caps eta at d*chi (gates.cpp:98), so the
    # InputError branch of gates.cpp:399-400 is unreachable: eta == d*chi here
    xi, bm, bn = random_inputs(2, 4, 1)
    u = q.apply_gate_qr_cbe(xi, bm, bn, model.identity_gate(2),
                            q.TruncationPolicy(chi_max=8, delta_chi_abs=100, delta_chi_rel=0.0), ctx)
    assert u.report.chi_expanded == 8


@pytest.mark.parametrize("d,chi_max,steps", [(3, 32, 5), (2, 16, 6)])
def test_uniform_cbe_trajectory_matches_oracle(ctx, d, chi_max, steps):
    h = model.bond_hamiltonian(d, 2.0)
    sched = model.trotter_schedule(h, 0.05, 2)
    kw = dict(chi_max=chi_max, sv_cutoff=1e-14)
    z = model.clock_operators(d)[0]
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    st_o = ref.product_state_uniform(d, 2, v)
    st_d = q.product_state_uniform(d, 2, v, ctx)
    for _ in range(steps):
        st_o, _ = ref.tebd_step_uniform(st_o, sched, "qr_cbe", ref.TruncationPolicy(**kw))
        st_d, rep = q.tebd_step(st_d, sched, "qr_cbe", q.TruncationPolicy(**kw), ctx)
        for s in range(2):
            zo = ref.expectation_local(st_o, z, s)
            zd = q.expectation_local(st_d, z, s, ctx)
            assert abs(zd - zo) <= 1e-10
            so = ref.schmidt_values(st_o, s)
            sd = q.schmidt_values(st_d, s, ctx)
            # the reference keeps CBE Schmidt values from eigh(L^H L)
            # (gates.cpp:408-419): values below ~sqrt(u) s_0 are rounding noise
            # there (they can clip to 0 and fall under sv_cutoff), so the kept
            # count may differ only by values under that floor
            m = min(len(sd), len(so))
            floor = 1e-7 * so[0]
            assert np.all(sd[m:] < floor) and np.all(so[m:] < floor)
            assert np.max(np.abs(sd[:m] - so[:m])) <= 1e-10 * so[0]
            assert abs(q.entropy_from_schmidt(sd) - ref.entropy_from_schmidt(so)) < 1e-10
