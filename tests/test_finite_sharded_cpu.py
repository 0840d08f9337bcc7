"""Multi-rank host logic of the sharded finite chain on CPU:
gloo world sizes 2 and 3, oracle updates, results bitwise equal to the
single-process Hastings-form oracle (same-parity updates commute bitwise,
proj/tests/test_tebd.cc:139-175)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200.finite import ShardedChain, numpy_backend, partition


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_chain(n, d, seed=7):
    """product state evolved a little with the oracle so bonds are entangled"""
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    sites = [v.reshape(d, 1, 1).copy() for _ in range(n)]
    bonds = [np.eye(1, dtype=complex) for _ in range(n)]
    return sites, bonds


def layers_for(n, d, dt=0.1, g=1.5):
    out = []
    for parity, dte in ref.layer_structure(dt, 2):
        out.append((0 if parity == "even" else 1,
                    [ref.make_gate(ref.chain_bond_hamiltonian(d, g, m, n), dte) for m in range(n - 1)]))
    return out


def oracle_run(n, d, steps, pol):
    sites, bonds = make_chain(n, d)
    layers = [("even" if p == 0 else "odd", g) for p, g in layers_for(n, d)]
    reports = []
    for _ in range(steps):
        sites, bonds, rep = ref.tebd_step_finite_hastings(sites, bonds, layers, "qr", pol)
        reports.append(rep)
    return sites, bonds, reports


def worker(rank, world, port, n, d, steps, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pol = ref.TruncationPolicy(chi_max=6, sv_cutoff=1e-14)
    sites, bonds = make_chain(n, d)
    s, e = partition(n, world)[rank]

    def apply(xi, bm, bn, u):
        upd = ref.apply_gate_qr(xi, bm, bn, u, pol)
        return upd.b_m, upd.xi_n, upd.b_n, upd.report

    try:
        chain = ShardedChain(sites[s:e], bonds[s:e], n, rank, world, numpy_backend(apply), dist)
        layers = layers_for(n, d)
        for _ in range(steps):
            chain.step(layers)
        out_q.put((rank, {m: chain.sites[m] for m in chain.sites}, {m: chain.bonds[m] for m in chain.bonds}))
    except Exception as exc:  # surface worker errors instead of a queue timeout
        out_q.put((rank, repr(exc), None))
        raise
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,world", [(8, 2), (10, 3), (7, 2)])
def test_sharded_chain_matches_single_process(n, world):
    d, steps = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, n, d, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for r, s, b in results:
        assert b is not None, f"rank {r} failed: {s}"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sites = {}
    bonds = {}
    for _, s, b in results:
        sites.update(s)
        bonds.update(b)
    o_sites, o_bonds, _ = oracle_run(n, d, steps, ref.TruncationPolicy(chi_max=6, sv_cutoff=1e-14))
    for m in range(n):
        assert np.array_equal(sites[m], o_sites[m]), m
        assert np.array_equal(bonds[m], o_bonds[m]), m


def test_partition_is_even_aligned():
    for n in (2, 7, 8, 256, 257):
        for w in (1, 2, 3, 4, 8):
            blocks = partition(n, w)
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (s, e), (s2, _) in zip(blocks, blocks[1:]):
                assert e == s2 and s % 2 == 0 and (e - s) % 2 == 0
            assert len(blocks) <= max(1, n // 2)


@pytest.mark.parametrize("workers", [2, 3])
def test_concurrent_bond_updates_match_sequential(workers):
    """Same-parity bonds dispatched to several backends (one host thread each,
    the device path's concurrent streams) give the bitwise result and report
    order of the sequential chain."""
    n, d, steps = 9, 2, 3
    pol = ref.TruncationPolicy(chi_max=6, sv_cutoff=1e-14)

    def apply(xi, bm, bn, u):
        upd = ref.apply_gate_qr(xi, bm, bn, u, pol)
        return upd.b_m, upd.xi_n, upd.b_n, upd.report

    layers = layers_for(n, d)
    runs = []
    for pool in (numpy_backend(apply), [numpy_backend(apply) for _ in range(workers + 1)]):
        sites, bonds = make_chain(n, d)
        chain = ShardedChain(sites, bonds, n, 0, 1, pool)
        reps = [chain.step(layers) for _ in range(steps)]
        runs.append((chain, reps))
    (a, ra), (b, rb) = runs
    for m in range(n):
        assert np.array_equal(a.sites[m], b.sites[m])
        assert np.array_equal(a.bonds[m], b.bonds[m])
    assert [[m for m, _ in r] for r in ra] == [[m for m, _ in r] for r in rb]


def ring_state(L, d, chi, seed):
    rng = np.random.default_rng(seed)
    sites = [ref.random_right_isometry(rng, d, chi, chi) for _ in range(L)]
    bonds = []
    for _ in range(L):
        x = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi))
        bonds.append(x / np.linalg.norm(x))
    return sites, bonds


def ring_worker(rank, world, port, L, d, chi, steps, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pol = ref.TruncationPolicy(chi_max=chi, sv_cutoff=1e-14)
    sites, bonds = ring_state(L, d, chi, 17)
    s, e = partition(L, world)[rank]

    def apply(xi, bm, bn, u):
        upd = ref.apply_gate_qr(xi, bm, bn, u, pol)
        return upd.b_m, upd.xi_n, upd.b_n, upd.report

    try:
        chain = ShardedChain(sites[s:e], bonds[s:e], L, rank, world, numpy_backend(apply), dist, periodic=True)
        gate_layers = [(0 if p == "even" else 1, [g] * L)
                       for p, g in ref.trotter_schedule(ref.bond_hamiltonian(d, 2.0), 0.05, 2)]
        for _ in range(steps):
            chain.step(gate_layers)
        out_q.put((rank, {m: chain.sites[m] for m in chain.sites}, {m: chain.bonds[m] for m in chain.bonds}))
    except Exception as exc:
        out_q.put((rank, repr(exc), None))
        raise
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("L,world", [(8, 2), (8, 3), (6, 1)])
def test_sharded_uniform_cell_ring_matches_oracle(L, world):
    """Uniform large unit cell sharded over ranks as a ring (the last rank's
    straddling bond is the wrap bond (L-1, 0)): bitwise equal to the oracle's
    tebd_step(UniformMPS), proj/src/gates.cpp:513-540."""
    d, chi, steps = 2, 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=ring_worker, args=(r, world, port, L, d, chi, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for r, s, b in results:
        assert b is not None, f"rank {r} failed: {s}"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sites, bonds = {}, {}
    for _, s, b in results:
        sites.update(s)
        bonds.update(b)
    s0, b0 = ring_state(L, d, chi, 17)
    st = ref.UniformMPS(d, s0, b0)
    sched = ref.trotter_schedule(ref.bond_hamiltonian(d, 2.0), 0.05, 2)
    for _ in range(steps):
        st, _ = ref.tebd_step_uniform(st, sched, "qr", ref.TruncationPolicy(chi_max=chi, sv_cutoff=1e-14))
    for m in range(L):
        assert np.array_equal(sites[m], st.site_tensors[m]), m
        assert np.array_equal(bonds[m], st.bond_matrices[m]), m
