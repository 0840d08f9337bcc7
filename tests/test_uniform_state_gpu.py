"""Device-resident UniformMPS (qt_uniform_*): graph-replayed steps must be
bitwise identical to eager steps and to the value-semantics tebd_step."""
import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import model
from paper_2212_09782_b200 import qrtebd as q

pytestmark = pytest.mark.gpu


def random_state(ctx, d, chi, seed):
    rng = np.random.default_rng(seed)
    sites = [ref.random_right_isometry(rng, d, chi, chi) for _ in range(2)]
    bonds = []
    for _ in range(2):
        x = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi))
        bonds.append(x / np.linalg.norm(x))
    return q.UniformMPS.from_numpy(ctx, d, sites, bonds)


@pytest.mark.parametrize("d,chi", [(3, 16), (5, 40)])
def test_graph_steps_bitwise_equal_eager_and_tebd_step(ctx, d, chi):
    sched = model.trotter_schedule(model.bond_hamiltonian(d, 2.0), 0.05, 2)
    gates = [(p, ctx.tensor(g)) for p, g in sched]
    pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
    st = random_state(ctx, d, chi, 11)
    ref_state = st
    dev_g = q.DeviceUniformMPS(st, ctx)
    dev_e = q.DeviceUniformMPS(st, ctx)
    for k in range(6):
        ref_state, rep_v = q.tebd_step(ref_state, gates, "qr", pol, ctx)
        rep_g = dev_g.step(gates, "qr", pol, use_graph=True)
        rep_e = dev_e.step(gates, "qr", pol, use_graph=False)
        assert [r.bond for r in rep_g] == [r.bond for r in rep_v]
        for a, b in zip(rep_g, rep_v):
            assert a.report.eps_trunc == b.report.eps_trunc and a.report.chi_after == b.report.chi_after
        for m in range(2):
            v = ref_state.site_tensors[m].numpy()
            assert np.array_equal(dev_g.view("site", m).numpy(), v)
            assert np.array_equal(dev_e.view("site", m).numpy(), v)
            assert np.array_equal(dev_g.view("bond", m).numpy(), ref_state.bond_matrices[m].numpy())


def test_device_state_grows_bond_dimension_eagerly(ctx):
    # from a product state the dimensions change every step (no graph), qr_cbe
    d = 3
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    st = q.product_state_uniform(d, 2, v, ctx)
    sched = model.trotter_schedule(model.bond_hamiltonian(d, 2.0), 0.05, 2)
    pol = q.TruncationPolicy(chi_max=32, sv_cutoff=1e-14)
    dev = q.DeviceUniformMPS(st, ctx)
    st_o = ref.product_state_uniform(d, 2, v)
    z = model.clock_operators(d)[0]
    for _ in range(4):
        dev.step(sched, "qr_cbe", pol)
        st_o, _ = ref.tebd_step_uniform(st_o, sched, "qr_cbe", ref.TruncationPolicy(chi_max=32, sv_cutoff=1e-14))
    snap = dev.snapshot()
    for s in range(2):
        assert abs(q.expectation_local(snap, z, s, ctx) - ref.expectation_local(st_o, z, s)) < 1e-10


def random_state_L(ctx, d, chi, L, seed):
    rng = np.random.default_rng(seed)
    sites = [ref.random_right_isometry(rng, d, chi, chi) for _ in range(L)]
    bonds = []
    for _ in range(L):
        x = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi))
        bonds.append(x / np.linalg.norm(x))
    return q.UniformMPS.from_numpy(ctx, d, sites, bonds)


@pytest.mark.parametrize("L", [4, 6])
def test_concurrent_same_parity_updates_bitwise_equal_serial(ctx, L):
    """L >= 4: the L/2 updates of a layer run on concurrent streams (one
    engine each, fork/join per layer); graph-replayed and
    eager steps are bitwise those of the one-stream value path."""
    d, chi = 3, 24
    sched = model.trotter_schedule(model.bond_hamiltonian(d, 2.0), 0.05, 2)
    gates = [(p, ctx.tensor(g)) for p, g in sched]
    pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
    st = random_state_L(ctx, d, chi, L, 5 + L)
    ref_state = st
    dev_g = q.DeviceUniformMPS(st, ctx)
    dev_e = q.DeviceUniformMPS(st, ctx)
    for _ in range(4):
        ref_state, _ = q.tebd_step(ref_state, gates, "qr", pol, ctx)
        dev_g.step(gates, "qr", pol, use_graph=True)
        dev_e.step(gates, "qr", pol, use_graph=False)
        for m in range(L):
            v = ref_state.site_tensors[m].numpy()
            assert np.array_equal(dev_g.view("site", m).numpy(), v)
            assert np.array_equal(dev_e.view("site", m).numpy(), v)
            assert np.array_equal(dev_g.view("bond", m).numpy(), ref_state.bond_matrices[m].numpy())
    # and the oracle agrees on a gauge-invariant quantity
    st_o = ref.UniformMPS(d, [t.numpy() for t in st.site_tensors], [b.numpy() for b in st.bond_matrices])
    for _ in range(4):
        st_o, _ = ref.tebd_step_uniform(st_o, sched, "qr", ref.TruncationPolicy(chi_max=chi, delta_chi_abs=0,
                                                                                delta_chi_rel=0.0))
    z = model.clock_operators(d)[0]
    snap = dev_g.snapshot()
    for s in range(L):
        assert abs(q.expectation_local(snap, z, s, ctx) - ref.expectation_local(st_o, z, s)) < 1e-10


@pytest.mark.parametrize("L,chi", [(2, 12), (4, 8)])
def test_check_isometric_matches_oracle(ctx, L, chi):
    """check_isometric(UniformMPS), proj/src/mps.cpp:105-141 (IsometryReport,
    SURVEY.md §8 a12): device defects equal the oracle's to rounding, on a
    random (non-canonical) cell and on a TEBD-evolved one."""
    d = 3
    rng = np.random.default_rng(L * 7 + chi)
    sites = [ref.random_right_isometry(rng, d, chi, chi) for _ in range(L)]
    bonds = []
    for _ in range(L):
        x = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi))
        bonds.append(x / np.linalg.norm(x))
    st_o = ref.UniformMPS(d, sites, bonds)
    ok_o, mx_o, parts = ref.check_isometric_uniform(st_o, 1e-8)
    st = q.UniformMPS.from_numpy(ctx, d, sites, bonds)
    rep = q.check_isometric(st, 1e-8, ctx)
    for key, dev in (("right", rep.right_defects), ("left", rep.left_defects),
                     ("translation", rep.translation_defects), ("norm", rep.norm_defects)):
        np.testing.assert_allclose(dev, parts[key], rtol=1e-10, atol=1e-13)
    assert rep.passed == ok_o and abs(rep.max_defect() - mx_o) <= 1e-10 * max(mx_o, 1e-3)
    # after TEBD steps the cell is canonical to rounding: both agree it passes
    sched = model.trotter_schedule(model.bond_hamiltonian(d, 2.0), 0.05, 2)
    pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
    for _ in range(3):
        st, _ = q.tebd_step(st, sched, "qr", pol, ctx)
    rep2 = q.check_isometric(st, 1e-6, ctx)
    st2 = ref.UniformMPS(d, [t.numpy() for t in st.site_tensors], [b.numpy() for b in st.bond_matrices])
    ok2, mx2, _ = ref.check_isometric_uniform(st2, 1e-6)
    assert rep2.passed == ok2 and abs(rep2.max_defect() - mx2) <= 1e-12


def test_graph_recaptured_after_workspace_regrowth():
    """Cached step graphs hold raw workspace pointers: a call on the same
    context that grows a workspace slot (here a larger-chi update) must not
    leave the next replay writing freed memory -- the graph is dropped and
    recaptured, and the trajectory stays bitwise equal to an eager one."""
    from paper_2212_09782_b200._capi import Context
    d, chi, big = 3, 16, 48
    sched = model.trotter_schedule(model.bond_hamiltonian(d, 2.0), 0.05, 2)
    pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
    pol_big = q.TruncationPolicy(chi_max=big, delta_chi_abs=0, delta_chi_rel=0.0)
    with Context(0) as c1, Context(0) as c2:
        gates1 = [(p, c1.tensor(g)) for p, g in sched]
        gates2 = [(p, c2.tensor(g)) for p, g in sched]
        dev_g = q.DeviceUniformMPS(random_state(c1, d, chi, 5), c1)
        dev_e = q.DeviceUniformMPS(random_state(c2, d, chi, 5), c2)
        st_big = random_state(c1, d, big, 6)
        for k in range(8):
            dev_g.step(gates1, "qr", pol, use_graph=True)
            dev_e.step(gates2, "qr", pol, use_graph=False)
            if k in (3, 5):  # grow the context's workspace between replays
                q.tebd_step(st_big, gates1, "qr", pol_big, c1)
                q.bond_energy(st_big.bond_matrices[0].numpy(), st_big.site_tensors[0].numpy(),
                              st_big.site_tensors[1].numpy(), model.bond_hamiltonian(d, 2.0), c1)
            for m in range(2):
                assert np.array_equal(dev_g.view("site", m).numpy(), dev_e.view("site", m).numpy())
                assert np.array_equal(dev_g.view("bond", m).numpy(), dev_e.view("bond", m).numpy())
        dev_g.close()
        dev_e.close()


def test_tebd_step_rejects_non_finite_state(ctx):
    """require_finite_matrix (proj/src/linalg.cpp:17-21) through the uniform
    step: a NaN in the state raises InputError, as apply_gate_qr does."""
    from paper_2212_09782_b200._capi import InputError
    d, chi = 3, 8
    rng = np.random.default_rng(3)
    sites = [ref.random_right_isometry(rng, d, chi, chi) for _ in range(2)]
    bonds = [np.eye(chi, dtype=complex) / np.sqrt(chi) for _ in range(2)]
    sites[1][1, 2, 3] = np.nan
    st = q.UniformMPS.from_numpy(ctx, d, sites, bonds)
    sched = [(p, ctx.tensor(g)) for p, g in model.trotter_schedule(model.bond_hamiltonian(d, 2.0), 0.05, 2)]
    with pytest.raises(InputError):
        q.tebd_step(st, sched, "qr", q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0), ctx)
