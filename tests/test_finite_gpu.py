"""Finite chain (Hastings form) on the device, one rank: every bond update
through the C-ABI, compared with the oracle on the same inputs; the wire
helpers (torch staging buffers for NCCL) round-trip exactly."""
import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import qrtebd as q
from paper_2212_09782_b200.finite import ShardedChain, device_backend

pytestmark = pytest.mark.gpu


def test_finite_chain_device_matches_oracle(ctx):
    n, d, steps = 8, 2, 3
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    sites = [v.reshape(d, 1, 1).copy() for _ in range(n)]
    bonds = [np.eye(1, dtype=complex) for _ in range(n)]
    layers = []
    for parity, dte in ref.layer_structure(0.1, 2):
        layers.append((0 if parity == "even" else 1,
                       [ref.make_gate(ref.chain_bond_hamiltonian(d, 1.5, m, n), dte) for m in range(n - 1)]))
    pol = q.TruncationPolicy(chi_max=6, sv_cutoff=1e-14)
    be = device_backend(ctx, "qr", pol)
    dl = [(p, [ctx.tensor(g) for g in gs]) for p, gs in layers]
    chain = ShardedChain([ctx.tensor(s) for s in sites], [ctx.tensor(b) for b in bonds], n, 0, 1, be, None)
    o_sites, o_bonds = sites, bonds
    for _ in range(steps):
        chain.step(dl, device="cuda")
        o_sites, o_bonds, _ = ref.tebd_step_finite_hastings(
            o_sites, o_bonds, [("even" if p == 0 else "odd", g) for p, g in layers], "qr",
            ref.TruncationPolicy(chi_max=6, sv_cutoff=1e-14))
    z = ref.clock_operators(d)[0]
    for m in range(n):
        # gauge-invariant: local <Z> from (Xi[m], B[m])
        zd = q.expectation_local(q.UniformMPS(d, [chain.sites[m]], [chain.bonds[m]]), z, 0, ctx)
        zo = ref.expectation_from_weight(ref.left_weight(o_bonds[m]), o_sites[m], z)
        assert abs(zd - zo) < 1e-10


def test_wire_roundtrip(ctx):
    import torch
    be = device_backend(ctx, "qr", q.TruncationPolicy())
    a = np.random.default_rng(1).standard_normal((3, 4, 5)) + 1j
    t = ctx.tensor(a)
    buf = be.to_wire(t)
    assert buf.is_cuda and buf.numel() == a.size * 2
    back = be.from_wire(buf, a.shape)
    assert np.array_equal(back.numpy(), a)
