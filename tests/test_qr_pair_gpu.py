"""The pipelined QR pair (qr_pair_pipelined: QR(X) with its reflectors applied
to theta, QR(Y^H) one panel behind, explicit Q_n in blocks, explicit error by
unitary invariance) against the oracle's alternating sweep
(proj/src/gates.cpp:293-308, :343-450), at the sizes that take it: 128..2048
rows, one sweep, no left_iso.  Ragged widths (eta not a multiple of the
32-column panel), rectangular bonds, truncating and expanding policies, and the
CBE scheme.  The same updates with the pair disabled (QT_NO_QR_PAIR is read
once per process, so the comparison is against the oracle and across two
bitwise-identical runs)."""
import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import model
from paper_2212_09782_b200 import qrtebd as q
from test_gate_gpu import block_of, compare, random_inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,chi,chi_l,chi_r,chi_max,dabs", [
    (5, 64, 64, 64, 64, 0),        # rows 320, eta 64: two full panels
    (5, 100, 100, 100, 100, 0),    # eta 100: ragged last panel (4 columns)
    (4, 96, 80, 120, 70, 0),       # rectangular, truncating (eta = chi_max = 70)
    (3, 128, 128, 128, 200, 60),   # expanding: eta = min(expanded, chi_max) = 188
    (8, 64, 64, 64, 64, 0),        # rows = cols = 512
    (5, 256, 256, 256, 256, 0),    # C2 shape: 1280 rows, 8 panels
    (5, 20, 64, 64, 20, 0),        # eta = 20 < one panel on 320 x 320
    (5, 40, 64, 56, 40, 0),        # eta = 40: one full panel + 8 columns
])
def test_pair_qr_update_matches_oracle(ctx, d, chi, chi_l, chi_r, chi_max, dabs):
    xi, bm, bn = random_inputs(d, chi, seed=7 * d + chi, chi_l=chi_l, chi_r=chi_r)
    gate = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
    pol = dict(chi_max=chi_max, sv_cutoff=1e-14, delta_chi_abs=dabs, delta_chi_rel=0.0)
    o = ref.apply_gate_qr(xi, bm, bn, gate, ref.TruncationPolicy(**pol))
    upd = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(**pol), ctx, want_left_iso=False)
    assert upd.left_iso is None
    compare(upd, o, xi)
    # Q_n and the bond matrix are gauge-fixed: compared directly (Appendix B (vi))
    assert np.allclose(upd.b_n.numpy(), o.b_n, atol=1e-11)
    assert np.allclose(upd.xi_n.numpy(), o.xi_n, atol=1e-12)
    # bitwise run to run
    upd2 = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(**pol), ctx, want_left_iso=False)
    assert np.array_equal(upd.b_m.numpy(), upd2.b_m.numpy())
    assert np.array_equal(upd.b_n.numpy(), upd2.b_n.numpy())
    assert upd.report.eps_trunc == upd2.report.eps_trunc


@pytest.mark.parametrize("explicit", [True, False])
def test_pair_explicit_error_small_and_large(ctx, explicit):
    # near-exact update (eps ~ 1e-30 noise floor) and a strongly truncating one
    d, chi = 5, 64
    xi, bm, bn = random_inputs(d, chi, seed=99)
    gate = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
    for chi_max in (64, 20):
        pol = dict(chi_max=chi_max, sv_cutoff=1e-14, delta_chi_abs=0, delta_chi_rel=0.0,
                   compute_explicit_error=explicit)
        o = ref.apply_gate_qr(xi, bm, bn, gate, ref.TruncationPolicy(**pol))
        u = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(**pol), ctx, want_left_iso=False)
        assert abs(u.report.eps_trunc - o.report.eps_trunc) <= 1e-10 * o.report.eps_trunc + 1e-20
        assert abs(u.report.discarded_weight - o.report.discarded_weight) <= 1e-9 * o.report.discarded_weight + 1e-15


@pytest.mark.parametrize("d,chi,dabs", [(5, 64, 40), (3, 100, 30), (5, 256, 100)])
def test_pair_cbe_update_matches_oracle(ctx, d, chi, dabs):
    rng = np.random.default_rng(d * chi)
    bm = ref.random_right_isometry(rng, d, chi, chi)
    bn = ref.random_right_isometry(rng, d, chi, chi)
    s = np.exp(-4.0 * np.arange(chi) / chi)
    xi = np.diag(s / np.linalg.norm(s)).astype(complex)
    gate = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
    kw = dict(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=dabs, delta_chi_rel=0.1)
    o = ref.apply_gate_qr_cbe(xi, bm, bn, gate, ref.TruncationPolicy(**kw))
    u = q.apply_gate_qr_cbe(xi, bm, bn, gate, q.TruncationPolicy(**kw), ctx)
    assert (u.report.chi_expanded, u.report.chi_after) == (o.report.chi_expanded, o.report.chi_after)
    b_d = block_of(xi, u.b_m.numpy(), u.b_n.numpy())
    b_o = block_of(xi, o.b_m, o.b_n)
    assert np.linalg.norm(b_d - b_o) / np.linalg.norm(b_o) < 1e-10
    s_d, s_o = np.diag(u.xi_n.numpy()).real, np.diag(o.xi_n).real
    assert np.max(np.abs(s_d - s_o)) <= 1e-10 * s_o[0]
    assert abs(u.report.eps_trunc - o.report.eps_trunc) <= 1e-10 * o.report.eps_trunc + 1e-20


@pytest.mark.parametrize("chi", [64, 128])  # 128: eta > 96, X formed in two column blocks
def test_pair_uniform_steps_match_oracle(ctx, chi):
    # a few device-resident C2-shaped steps (graph replay) against the oracle
    d = 5
    rng = np.random.default_rng(5)
    sites = [ref.random_right_isometry(rng, d, chi, chi) for _ in range(2)]
    bonds = []
    for _ in range(2):
        x = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi))
        bonds.append(x / np.linalg.norm(x))
    sched = ref.trotter_schedule(ref.bond_hamiltonian(d, 2.0, "bulk"), 0.05, 2)
    pol = ref.TruncationPolicy(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=0, delta_chi_rel=0.0)
    dev = q.DeviceUniformMPS(q.UniformMPS.from_numpy(ctx, d, sites, bonds), ctx)
    dsched = [(p, ctx.tensor(u)) for p, u in sched]
    st = ref.UniformMPS(d, [s.copy() for s in sites], [b.copy() for b in bonds])
    z = ref.clock_operators(d)[0]
    for _ in range(4):
        reps = dev.step(dsched, "qr", q.TruncationPolicy(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=0,
                                                         delta_chi_rel=0.0))
        st, oreps = ref.tebd_step_uniform(st, sched, "qr", pol)
        for r, (_, o) in zip(reps, oreps):
            assert abs(r.report.eps_trunc - o.eps_trunc) <= 1e-9 * o.eps_trunc + 2e-13 * o.eps_trunc ** 0.5 + 1e-20
    snap = dev.snapshot()
    for m in range(2):
        zd = q.expectation_local(snap, z, m, ctx)
        zo = ref.expectation_local(st, z, m)
        assert abs(zd - zo) < 1e-10


@pytest.mark.parametrize("chi", [64, 128])  # 128: each engine splits its X GEMM over two streams
def test_pair_concurrent_cell_L4_matches_oracle(ctx, chi):
    # L = 4: the two same-parity updates of a layer run on concurrent engines,
    # each with its own six-stream pipelined pair, inside one captured graph
    d, L = 5, 4
    rng = np.random.default_rng(44)
    sites = [ref.random_right_isometry(rng, d, chi, chi) for _ in range(L)]
    bonds = []
    for _ in range(L):
        x = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi))
        bonds.append(x / np.linalg.norm(x))
    sched = ref.trotter_schedule(ref.bond_hamiltonian(d, 2.0, "bulk"), 0.05, 2)
    kw = dict(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=0, delta_chi_rel=0.0)
    dev = q.DeviceUniformMPS(q.UniformMPS.from_numpy(ctx, d, sites, bonds), ctx)
    dsched = [(p, ctx.tensor(u)) for p, u in sched]
    st = ref.UniformMPS(d, [s.copy() for s in sites], [b.copy() for b in bonds])
    for _ in range(3):
        dev.step(dsched, "qr", q.TruncationPolicy(**kw))
        st, _ = ref.tebd_step_uniform(st, sched, "qr", ref.TruncationPolicy(**kw))
    snap = dev.snapshot()
    z = ref.clock_operators(d)[0]
    for m in range(L):
        assert abs(q.expectation_local(snap, z, m, ctx) - ref.expectation_local(st, z, m)) < 1e-10
        sd = q.schmidt_values(snap, m, ctx)
        so = ref.schmidt_values(st, m)
        # every Schmidt value, no filter
        assert sd.shape == so.shape and np.max(np.abs(sd - so)) <= 1e-10 * so[0]


def test_pair_and_sequential_paths_agree_per_context_knob():
    # qt_ctx_set_qr_pair_min_rows switches one context to the sequential
    # QR(X) -> theta^H Q_m -> QR(Y^H) path: the two paths agree to rounding
    from paper_2212_09782_b200._capi import Context, check
    d, chi = 5, 64
    xi, bm, bn = random_inputs(d, chi, seed=321)
    gate = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
    kw = dict(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=0, delta_chi_rel=0.0)
    outs = []
    for min_rows in (-1, 1 << 20):
        with Context(0) as c:
            check(c.lib.qt_ctx_set_qr_pair_min_rows(c.h, min_rows))
            u = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(**kw), c, want_left_iso=False)
            outs.append((u.b_m.numpy(), u.xi_n.numpy(), u.b_n.numpy(), u.report.eps_trunc))
    (bm1, x1, bn1, e1), (bm2, x2, bn2, e2) = outs
    assert np.allclose(x1, x2, atol=1e-12) and np.allclose(bn1, bn2, atol=1e-11)
    assert np.allclose(bm1, bm2, atol=1e-11)
    assert abs(e1 - e2) <= 1e-10 * e2 + 1e-20


@pytest.mark.parametrize("where", ["xi", "bn"])
def test_pair_nonfinite_input_is_input_error(ctx, where):
    """require_finite_matrix (proj/src/linalg.cpp:17-21) through the pair with X
    formed in two column blocks (eta = 256 > 96): the NaN reaches X's head
    columns (main stream) and its remainder (look-ahead stream); the update
    raises InputError and the context stays usable."""
    d, chi = 5, 256
    xi, bm, bn = random_inputs(d, chi, seed=11)
    gate = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
    pol = dict(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=0, delta_chi_rel=0.0)
    bad = {"xi": xi.copy(), "bn": bn.copy()}
    bad[where][(3,) * bad[where].ndim] = np.nan
    args = (bad["xi"], bm, bad["bn"])
    with pytest.raises(q.InputError):
        q.apply_gate_qr(*args, gate, q.TruncationPolicy(**pol), ctx, want_left_iso=False)
    o = ref.apply_gate_qr(xi, bm, bn, gate, ref.TruncationPolicy(**pol))
    upd = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(**pol), ctx, want_left_iso=False)
    compare(upd, o, xi)


@pytest.mark.parametrize("d,chi,chi_max", [(5, 64, 64), (5, 256, 256), (4, 96, 70), (3, 128, 188)])
def test_pair_with_left_iso_matches_oracle(ctx, d, chi, chi_max):
    """The reference signature always returns left_iso for qr (gates.cpp:373):
    the pipelined pair keeps running and forms Q_m from QR(X)'s stored
    reflectors beside the tail; Q_m is gauge-fixed, so left_iso is compared
    directly (Appendix B (vi)), and the rest equals the left_iso-free update
    bitwise."""
    xi, bm, bn = random_inputs(d, chi, seed=55 * d + chi)
    gate = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
    pol = dict(chi_max=chi_max, sv_cutoff=1e-14, delta_chi_abs=max(0, chi_max - chi), delta_chi_rel=0.0)
    o = ref.apply_gate_qr(xi, bm, bn, gate, ref.TruncationPolicy(**pol))
    upd = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(**pol), ctx, want_left_iso=True)
    compare(upd, o, xi)
    li = upd.left_iso.numpy()
    assert np.linalg.norm(li - o.left_iso) / np.linalg.norm(o.left_iso) < 1e-10
    plain = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(**pol), ctx, want_left_iso=False)
    assert np.array_equal(plain.b_n.numpy(), upd.b_n.numpy())
    assert np.array_equal(plain.b_m.numpy(), upd.b_m.numpy())
    assert plain.report.eps_trunc == upd.report.eps_trunc
