"""Step-level parity: device tebd_step on a uniform
L=2 cell vs the oracle, observables through the device contractions
(proj/tests/test_tebd.cc:32-137 structure)."""
import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import model
from paper_2212_09782_b200 import qrtebd as q

pytestmark = pytest.mark.gpu


def e0(d):
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    return v


@pytest.mark.parametrize("d,chi_max,steps", [(3, 32, 6), (2, 16, 8), (5, 25, 3)])
def test_uniform_qr_trajectory_matches_oracle(ctx, d, chi_max, steps):
    h = model.bond_hamiltonian(d, 2.0)
    sched_h = model.trotter_schedule(h, 0.05, 2)
    pol_kw = dict(chi_max=chi_max, sv_cutoff=1e-14)
    z = model.clock_operators(d)[0]
    st_o = ref.product_state_uniform(d, 2, e0(d))
    st_d = q.product_state_uniform(d, 2, e0(d), ctx)
    for k in range(steps):
        st_o, rep_o = ref.tebd_step_uniform(st_o, sched_h, "qr", ref.TruncationPolicy(**pol_kw))
        st_d, rep_d = q.tebd_step(st_d, sched_h, "qr", q.TruncationPolicy(**pol_kw), ctx)
        assert [r.bond for r in rep_d] == [n for n, _ in rep_o]
        for rd, (_, ro) in zip(rep_d, rep_o):
            assert rd.report.chi_after == ro.chi_after
            assert abs(rd.report.eps_trunc - ro.eps_trunc) <= 1e-10 * abs(ro.eps_trunc) + 1e-20
        for s in range(2):
            zd = q.expectation_local(st_d, z, s, ctx)
            zo = ref.expectation_local(st_o, z, s)
            assert abs(zd - zo) <= 1e-10 * max(1.0, abs(zo))
        # energy extension: device vs oracle on the same device state
        sites, bonds = st_d.to_numpy()
        e_d = q.bond_energy(bonds[0], sites[0], sites[1], h, ctx)
        e_o = ref.bond_energy(bonds[0], sites[0], sites[1], h)
        assert abs(e_d - e_o) <= 1e-10 * max(1.0, abs(e_o))


def test_identity_step_keeps_right_isometry(ctx):
    # proj/tests/test_tebd.cc:64-75
    d = 3
    st = q.product_state_uniform(d, 2, e0(d), ctx)
    ids = model.trotter_schedule(model.bond_hamiltonian(d, 2.0), 0.0, 2)
    st, _ = q.tebd_step(st, ids, "qr", q.TruncationPolicy(chi_max=512), ctx)
    for s in st.site_tensors:
        assert q.right_defect(s, ctx) < 1e-12


def test_odd_cell_rejected(ctx):
    st = q.product_state_uniform(2, 3, e0(2), ctx)
    sched = model.trotter_schedule(model.bond_hamiltonian(2, 1.0), 0.1, 1)
    with pytest.raises(q.InputError):
        q.tebd_step(st, sched, "qr", None, ctx)


def test_step_is_bitwise_deterministic(ctx):
    d = 3
    sched = model.trotter_schedule(model.bond_hamiltonian(d, 2.0), 0.05, 2)
    outs = []
    for _ in range(2):
        st = q.product_state_uniform(d, 2, e0(d), ctx)
        for _ in range(4):
            st, _ = q.tebd_step(st, sched, "qr", q.TruncationPolicy(chi_max=27), ctx)
        outs.append(st.to_numpy())
    for a, b in zip(outs[0][0] + outs[0][1], outs[1][0] + outs[1][1]):
        assert np.array_equal(a, b)


def test_right_defect_matches_oracle(ctx):
    rng = np.random.default_rng(3)
    b = ref.random_right_isometry(rng, 4, 10, 12)
    b = b + 1e-3 * (rng.standard_normal(b.shape) + 1j * rng.standard_normal(b.shape))
    assert abs(q.right_defect(b, ctx) - ref.right_defect(b)) < 1e-14
