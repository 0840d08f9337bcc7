"""Reference-exact finite chain on the device (qt_finite_*): move_center
(proj/src/mps.cpp:226-257), the sequential tebd_step(FiniteMPS)
(proj/src/gates.cpp:542-578) and the finite observables (mps.cpp:188-207),
compared with the oracle on identical inputs (Appendix B tolerances)."""
import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import qrtebd as q

pytestmark = pytest.mark.gpu


def _rand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _random_chain(seed, d, n, chi_cap, center):
    rng = np.random.default_rng(seed)
    dims = [min(d ** m, d ** (n - m), chi_cap) for m in range(n + 1)]
    sites = [_rand(rng, d, dims[m], dims[m + 1]) for m in range(n)]
    cm = _rand(rng, dims[center], dims[center])
    return sites, cm


@pytest.mark.parametrize("path", [[6, 2, 0, 4], [3, 3, 1, 6]])
def test_move_center_matches_oracle(ctx, path):
    # full-rank chain: the gauge-fixed QR/LQ make every moved tensor unique
    d, n = 3, 6
    sites, cm = _random_chain(11, d, n, 7, 0)
    dev = q.FiniteMPS(d, sites, 0, cm, ctx)
    orc = ref.FiniteMPS(d, [s.copy() for s in sites], 0, cm.copy())
    for c in path:
        dev = q.move_center(dev, c)
        orc = ref.move_center(orc, c)
        assert dev.center_bond == c
        ds, dc, dcm = dev.to_numpy()
        scale = np.linalg.norm(orc.center_matrix)
        assert dcm.shape == orc.center_matrix.shape
        assert np.allclose(dcm, orc.center_matrix, atol=1e-12 * scale)
        for a, b in zip(ds, orc.site_tensors):
            assert a.shape == b.shape
            assert np.allclose(a, b, atol=1e-12 * max(1.0, np.abs(b).max()))


def test_move_center_rectangular_center(ctx):
    # d * chi_l < chi_r makes the QR thin: rectangular center matrices
    # (mps.cpp:328-330) and a rank-revealing shrink of the bond
    rng = np.random.default_rng(5)
    d = 2
    sites = [_rand(rng, d, 1, 5), _rand(rng, d, 5, 3), _rand(rng, d, 3, 1)]
    cm = np.eye(1, dtype=complex)
    dev = q.FiniteMPS(d, sites, 0, cm, ctx)
    orc = ref.FiniteMPS(d, [s.copy() for s in sites], 0, cm.copy())
    for c in (1, 3, 1):
        dev = q.move_center(dev, c)
        orc = ref.move_center(orc, c)
        ds, _, dcm = dev.to_numpy()
        assert dcm.shape == orc.center_matrix.shape
        assert np.allclose(dcm, orc.center_matrix, atol=1e-12)
        for a, b in zip(ds, orc.site_tensors):
            assert a.shape == b.shape and np.allclose(a, b, atol=1e-12)


def test_move_center_out_of_range(ctx):
    sites, cm = _random_chain(1, 2, 3, 4, 0)
    dev = q.FiniteMPS(2, sites, 0, cm, ctx)
    with pytest.raises(q.InputError):
        q.move_center(dev, 4)


@pytest.mark.parametrize("scheme,chi_max,n,d", [("qr", 64, 6, 2), ("qr", 6, 8, 3), ("qr_cbe", 64, 6, 2),
                                                ("qr_cbe", 6, 8, 3)])
def test_finite_step_matches_oracle(ctx, scheme, chi_max, n, d):
    g, dt, steps = 1.5, 0.1, 3
    layers = ref.finite_layers(d, g, n, dt, 2)
    dlayers = [(p, [ctx.tensor(u) for u in gs]) for p, gs in layers]
    pol_o = ref.TruncationPolicy(chi_max=chi_max, sv_cutoff=1e-14)
    pol_d = q.TruncationPolicy(chi_max=chi_max, sv_cutoff=1e-14)
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    dev = q.product_state_finite(d, n, v, ctx)
    orc = ref.product_state_finite(d, n, v)
    z = ref.clock_operators(d)[0]
    for _ in range(steps):
        _, reps = q.tebd_step_finite(dev, dlayers, scheme, pol_d, in_place=True)
        orc, oreps = ref.tebd_step_finite(orc, layers, scheme, pol_o)
        assert [r.bond for r in reps] == [b for b, _ in oreps]
        for r, (_, o) in zip(reps, oreps):
            assert (r.report.chi_before, r.report.chi_expanded, r.report.chi_after) == \
                (o.chi_before, o.chi_expanded, o.chi_after)
            # trajectory floor: after several steps the states differ at ~1e-13 relative, so
            # delta eps ~ 2 sqrt(eps) * 1e-13 (Appendix B(iii) gives the single-update floor)
            assert abs(r.report.eps_trunc - o.eps_trunc) <= 1e-10 * o.eps_trunc + 2e-13 * o.eps_trunc ** 0.5 + 1e-20
        assert dev.center_bond == orc.center_bond
        zs, spectra = q.finite_observables(dev, z)
        for s in range(n):
            assert abs(zs[s] - ref.expectation_local_finite(orc, z, s)) < 1e-10
        for b in range(n + 1):
            so = ref.schmidt_values_finite(orc, b)
            sd = spectra[b]
            assert len(sd) == len(so)
            assert np.max(np.abs(sd - so)) <= 1e-10 * so[0]  # every value (Appendix B (ii))
            assert abs(ref.entropy_from_schmidt(sd) - ref.entropy_from_schmidt(so)) < 1e-10


def test_finite_step_bitwise_deterministic(ctx):
    d, n = 3, 6
    layers = [(p, [ctx.tensor(u) for u in gs]) for p, gs in ref.finite_layers(d, 2.0, n, 0.1, 2)]
    pol = q.TruncationPolicy(chi_max=5)
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    outs = []
    for _ in range(2):
        s = q.product_state_finite(d, n, v, ctx)
        for _ in range(3):
            q.tebd_step_finite(s, layers, "qr", pol, in_place=True)
        outs.append(s.to_numpy())
    for a, b in zip(outs[0][0], outs[1][0]):
        assert np.array_equal(a, b)
    assert np.array_equal(outs[0][2], outs[1][2])


def test_single_site_observables_match_sweep(ctx):
    sites, cm = _random_chain(3, 2, 5, 4, 2)
    dev = q.FiniteMPS(2, sites, 2, cm, ctx)
    # canonical form first (sites < center left-, >= center right-isometric): the
    # reference observables assume it, and a gauge sweep across the chain makes it
    dev = q.move_center(q.move_center(q.move_center(dev, 5), 0), 2)
    z = ref.clock_operators(2)[0]
    zs, spectra = q.finite_observables(dev, z)
    for s in range(5):
        assert abs(q.expectation_local_finite(dev, z, s) - zs[s]) < 1e-12 * max(1.0, abs(zs[s]))
    for b in range(6):
        assert np.allclose(q.schmidt_values_finite(dev, b), spectra[b], atol=1e-12 * spectra[b][0])
    assert dev.center_bond == 2  # observables never move the caller's center
