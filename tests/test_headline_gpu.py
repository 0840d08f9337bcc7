"""Parity at the headline configurations (BASELINE.json north star and
configs[2..4]): the code paths only large
updates take -- theta rows > 2048 (no pipelined pair), GEMM block reflectors
for m > 2048, the grid-barrier QR panel for m > 5120, the Jacobi eigensolver
at n = 1127 -- against the oracle on identical inputs.

* north star, d=5 chi=1024 qr (explicit error on): one update (block, Q_n and
  Xi~ directly, Schmidt values, eps, eta) and two Trotter steps (<Z>, bond
  energy, entropy, eps per bond), plus graph replay == eager bitwise;
* C3, d=10 chi=1024 qr_cbe (eta = 1127, eigh n = 1127): one update;
* C4, d=5 chi=4096 qr bench cell: one update against the committed fixture
  tests/golden/c4_qr_d5_chi4096.npz (made by tests/golden/make_c4_fixture.py);
* C5-shaped finite chain, d=5, N=12, chi up to 512, Hastings form: one step
  of the device chain against the oracle chain.
"""
import os
import sys

import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import model
from paper_2212_09782_b200 import qrtebd as q

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def block_sketch(xi_old, b_m, b_n, p, r):
    sys.path.insert(0, GOLDEN)
    import make_c4_fixture as fx
    return fx.block_sketch(xi_old, b_m, b_n, p, r)


def sketch_mats(d, chi_l, chi_r, seed):
    rng = np.random.default_rng(seed)
    p = rng.standard_normal((chi_l * d, 4)) + 1j * rng.standard_normal((chi_l * d, 4))
    r = rng.standard_normal((d * chi_r, 4)) + 1j * rng.standard_normal((d * chi_r, 4))
    return p, r


def check_update(upd, o, xi_old, qn_direct=True):
    """Appendix B.1 between a device GateUpdate and an oracle GateUpdate, via
    sketches of the (chi d) x (d chi) block (the block itself is GBs at C3)."""
    bm, xin, bn = upd.b_m.numpy(), upd.xi_n.numpy(), upd.b_n.numpy()
    assert bm.shape == o.b_m.shape and xin.shape == o.xi_n.shape and bn.shape == o.b_n.shape
    d, chi_l = bm.shape[0], xi_old.shape[0]
    p, r = sketch_mats(d, chi_l, bn.shape[2], seed=chi_l + d)
    # (i) gauge-invariant two-site block
    assert rel(block_sketch(xi_old, bm, bn, p, r), block_sketch(xi_old, o.b_m, o.b_n, p, r)) < 1e-10
    # (ii) every Schmidt value of Xi~ (device spectra vs zgesdd)
    s_d = q.schmidt_values_of(xin)
    s_o = np.linalg.svd(o.xi_n, compute_uv=False)
    assert s_d.shape == s_o.shape and np.max(np.abs(s_d - s_o)) <= 1e-10 * s_o[0]
    # (iii) eps, (iv) integer widths
    r_, ro = upd.report, o.report
    assert (r_.chi_before, r_.chi_expanded, r_.chi_after) == (ro.chi_before, ro.chi_expanded, ro.chi_after)
    assert abs(r_.eps_trunc - ro.eps_trunc) <= 1e-10 * abs(ro.eps_trunc) + 1e-20
    # (v) right isometry
    kk = bn.shape[1]
    g = np.einsum("iab,icb->ac", bn, bn.conj())
    assert np.max(np.abs(g - np.eye(kk))) < 1e-12
    if qn_direct:  # (vi) gauge-fixed factors, compared directly (full rank)
        assert rel(bn, o.b_n) < 1e-10
        assert rel(xin, o.xi_n) < 1e-10


def test_north_star_update_parity():
    """d=5 chi=1024 qr, explicit error on (5120-row blocks: sequential QR
    with GEMM block reflectors and the 5120-row cluster panel)."""
    d, chi = 5, 1024
    xi, bm, bn, gate, _ = ref.bench_cell_inputs(d, chi, "qr")
    kw = dict(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=0, delta_chi_rel=0.0, compute_explicit_error=True)
    o = ref.apply_gate_qr(xi, bm, bn, gate, ref.TruncationPolicy(**kw))
    upd = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(**kw), want_left_iso=True)
    check_update(upd, o, xi)
    assert rel(upd.left_iso.numpy(), o.left_iso) < 1e-10
    # the device-resident fast path's update (no left_iso: pipelined when it fits)
    upd2 = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(**kw), want_left_iso=False)
    check_update(upd2, o, xi)


def test_north_star_steps_parity_and_graph_replay():
    """Two Trotter steps of the north-star quench cell (device-resident,
    eager) vs the oracle: <Z>, bond energy, entropy, eps and chi per bond to
    1e-10 (Appendix B.2); then graph-replayed steps bitwise equal to eager."""
    import bench
    d, chi = 5, 1024
    ctx = q.default_context()
    sites, bonds = bench.synthetic_state(d, chi)
    sched = model.trotter_schedule(model.bond_hamiltonian(d, 2.0), 0.05, 2)
    kw = dict(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=0, delta_chi_rel=0.0, compute_explicit_error=True)
    gates = [(p, ctx.tensor(u)) for p, u in sched]
    st0 = q.UniformMPS.from_numpy(ctx, d, sites, bonds)
    dev = q.DeviceUniformMPS(st0, ctx)
    st = ref.UniformMPS(d, [s.copy() for s in sites], [b.copy() for b in bonds])
    z = ref.clock_operators(d)[0]
    h = model.bond_hamiltonian(d, 2.0)
    for _ in range(2):
        rep_d = dev.step(gates, "qr", q.TruncationPolicy(**kw), use_graph=False)
        st, rep_o = ref.tebd_step_uniform(st, sched, "qr", ref.TruncationPolicy(**kw))
        assert len(rep_d) == len(rep_o) == 3
        for a, (bond_o, ro) in zip(rep_d, rep_o):
            assert a.bond == bond_o and a.report.chi_after == ro.chi_after
            assert abs(a.report.eps_trunc - ro.eps_trunc) <= 1e-10 * ro.eps_trunc + 2e-13 * ro.eps_trunc ** 0.5 + 1e-20
        snap = dev.snapshot()
        for m in range(2):
            zd = q.expectation_local(snap, z, m, ctx)
            zo = ref.expectation_local(st, z, m)
            assert abs(zd - zo) <= 1e-10 * max(1.0, abs(zo))
            sd = q.schmidt_values(snap, m, ctx)
            so = ref.schmidt_values(st, m)
            assert sd.shape == so.shape and np.max(np.abs(sd - so)) <= 1e-10 * so[0]
            assert abs(q.entropy_from_schmidt(sd) - ref.entropy_from_schmidt(so)) <= 1e-10
        n = 1
        ed = q.bond_energy(snap.bond_matrices[0].numpy(), snap.site_tensors[0].numpy(),
                           snap.site_tensors[n].numpy(), h, ctx)
        eo = ref.bond_energy(st.bond_matrices[0], st.site_tensors[0], st.site_tensors[n], h)
        assert abs(ed - eo) <= 1e-10 * max(1.0, abs(eo))
    # graph replay (captured from step 3 on) == eager, bitwise
    dev_e = q.DeviceUniformMPS(dev.snapshot(), ctx)
    for _ in range(4):
        dev.step(gates, "qr", q.TruncationPolicy(**kw), use_graph=True)
        dev_e.step(gates, "qr", q.TruncationPolicy(**kw), use_graph=False)
    for m in range(2):
        assert np.array_equal(dev.view("site", m).numpy(), dev_e.view("site", m).numpy())
        assert np.array_equal(dev.view("bond", m).numpy(), dev_e.view("bond", m).numpy())
    dev.close()
    dev_e.close()


def test_c3_cbe_update_parity():
    """C3: d=10 chi=1024 qr_cbe, eta = 1127 (10240-row blocks: grid-barrier
    QR panels; Jacobi eigensolver at n = 1127), explicit error on."""
    d, chi = 10, 1024
    xi, bm, bn, gate, _ = ref.bench_cell_inputs(d, chi, "qr_cbe")
    kw = dict(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=100, delta_chi_rel=0.1, compute_explicit_error=True)
    o = ref.apply_gate_qr_cbe(xi, bm, bn, gate, ref.TruncationPolicy(**kw))
    upd = q.apply_gate_qr_cbe(xi, bm, bn, gate, q.TruncationPolicy(**kw))
    assert upd.report.chi_expanded == 1127
    # CBE: B~n rows = V_k^H Q_n carry the eigenvector phases (gauge): compare
    # the gauge-invariant quantities; Xi~ is diagonal and gauge-fixed
    check_update(upd, o, xi, qn_direct=False)
    assert np.max(np.abs(np.diag(upd.xi_n.numpy()) - np.diag(o.xi_n))) <= 1e-10 * o.xi_n[0, 0].real


def test_c4_single_bond_matches_fixture():
    """C4: d=5 chi=4096 bench cell (20480-row blocks, theta = 6.7 GB) against
    the committed oracle fixture."""
    path = os.path.join(GOLDEN, "c4_qr_d5_chi4096.npz")
    if not os.path.exists(path):
        pytest.fail("missing golden fixture; run tests/golden/make_c4_fixture.py")
    fx = np.load(path)
    sys.path.insert(0, GOLDEN)
    import make_c4_fixture as mk
    xi, bm, bn, gate, pol = ref.bench_cell_inputs(mk.D, mk.CHI, "qr")
    upd = q.apply_gate_qr(xi, bm, bn, gate, q.TruncationPolicy(
        chi_max=pol.chi_max, sv_cutoff=pol.sv_cutoff, delta_chi_abs=pol.delta_chi_abs,
        delta_chi_rel=pol.delta_chi_rel, compute_explicit_error=pol.compute_explicit_error), want_left_iso=False)
    assert upd.report.chi_expanded == int(fx["eta"]) and upd.report.chi_after == int(fx["chi_after"])
    assert abs(upd.report.eps_trunc - float(fx["eps"])) <= 1e-10 * float(fx["eps"]) + 1e-20
    xin = upd.xi_n.numpy()
    s_d = q.schmidt_values_of(xin)
    assert np.max(np.abs(s_d - fx["s"])) <= 1e-10 * fx["s"][0]
    assert np.max(np.abs(np.diag(xin).real - fx["diag"])) <= 1e-10 * fx["s"][0]
    bn_d = upd.b_n.numpy()
    p, r = mk.sketch_mats(mk.D, mk.CHI, mk.CHI)
    assert rel(mk.qn_times_r(bn_d, r), fx["qn_r"]) < 1e-10
    assert rel(mk.block_sketch(xi, upd.b_m.numpy(), bn_d, p, r), fx["sketch"]) < 1e-10


def test_c5_shaped_chain_step_parity():
    """Finite clock chain in Hastings form, d=5,
    N=12, bond dimensions min(5^m, 5^(N-m), 512): one Trotter step of the
    device chain (one rank) vs the oracle chain, qr, explicit error on."""
    from paper_2212_09782_b200.finite import ShardedChain, chain_dims, device_backend
    ctx = q.default_context()
    n, d, chi = 12, 5, 512
    dims = chain_dims(n, d, chi)
    rng = np.random.default_rng(0xC5)
    sites = [ref.random_right_isometry(rng, d, dims[m], dims[m + 1]) for m in range(n)]
    bonds = []
    for m in range(n):
        x = rng.standard_normal((dims[m], dims[m])) + 1j * rng.standard_normal((dims[m], dims[m]))
        bonds.append(x / np.linalg.norm(x))
    layers = []
    for parity, dte in ref.layer_structure(0.05, 2):
        layers.append((0 if parity == "even" else 1,
                       [ref.make_gate(ref.chain_bond_hamiltonian(d, 2.0, m, n), dte) for m in range(n - 1)]))
    kw = dict(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=0, delta_chi_rel=0.0, compute_explicit_error=True)
    be = device_backend(ctx, "qr", q.TruncationPolicy(**kw))
    dl = [(p, [ctx.tensor(g) for g in gs]) for p, gs in layers]
    chain = ShardedChain([ctx.tensor(s) for s in sites], [ctx.tensor(b) for b in bonds], n, 0, 1, be, None)
    rep_d = chain.step(dl, device="cuda")
    o_sites, o_bonds, rep_o = ref.tebd_step_finite_hastings(
        sites, bonds, [("even" if p == 0 else "odd", g) for p, g in layers], "qr", ref.TruncationPolicy(**kw))
    assert len(rep_d) == len(rep_o)
    for (bond_d, rd), (bond_o, ro) in zip(rep_d, rep_o):
        assert bond_d == bond_o and rd.chi_after == ro.chi_after
        assert abs(rd.eps_trunc - ro.eps_trunc) <= 1e-10 * ro.eps_trunc + 2e-13 * ro.eps_trunc ** 0.5 + 1e-20
    z = ref.clock_operators(d)[0]
    for m in range(n):
        zd = q.expectation_local(q.UniformMPS(d, [chain.sites[m]], [chain.bonds[m]]), z, 0, ctx)
        zo = ref.expectation_from_weight(ref.left_weight(o_bonds[m]), o_sites[m], z)
        assert abs(zd - zo) <= 1e-10
        sd = q.schmidt_values_of(chain.bonds[m].numpy())
        so = np.linalg.svd(o_bonds[m], compute_uv=False)
        assert np.max(np.abs(sd - so)) <= 1e-10 * so[0]
