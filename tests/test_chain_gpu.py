"""The C-ABI sharded finite chain (qt_chain_*, qt_tebd_step_finite_sharded,
csrc/chain.cu): one rank against the oracle's Hastings-form
chain, and 2 / 3 ranks -- one thread and one context per rank, exchanging the
straddling tensors through the in-process loopback transport on this one GPU
-- bitwise equal to the single-rank chain (the NCCL transport runs the same
orchestration across processes)."""
import threading

import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import qrtebd as q
from paper_2212_09782_b200._capi import Context
from paper_2212_09782_b200.chain import DeviceChain, Loopback, partition
from paper_2212_09782_b200.finite import chain_dims

pytestmark = pytest.mark.gpu


def chain_state(n, d, chi, seed):
    dims = chain_dims(n, d, chi)
    rng = np.random.default_rng(seed)
    sites = [ref.random_right_isometry(rng, d, dims[m], dims[m + 1]) for m in range(n)]
    bonds = []
    for m in range(n):
        x = rng.standard_normal((dims[m], dims[m])) + 1j * rng.standard_normal((dims[m], dims[m]))
        bonds.append(x / np.linalg.norm(x))
    return sites, bonds


def host_layers(n, d, dt=0.05):
    return [(0 if p == "even" else 1, [ref.make_gate(ref.chain_bond_hamiltonian(d, 2.0, m, n), dte)
                                        for m in range(n - 1)]) for p, dte in ref.layer_structure(dt, 2)]


def run_rank(ctx, n, sites, bonds, layers, rank, world, lb, steps, kw, workers, out):
    b, e = partition(n, world, rank)
    dl = [(p, [ctx.tensor(g) if b <= m + 1 and m < e else None for m, g in enumerate(gs)]) for p, gs in layers]
    ch = DeviceChain(ctx, n, [ctx.tensor(s) for s in sites[b:e]], [ctx.tensor(x) for x in bonds[b:e]], rank, world,
                     loopback=lb, workers=workers)
    reps = []
    for _ in range(steps):
        reps += ch.step(dl, "qr", q.TruncationPolicy(**kw))
    out[rank] = ([ch.view("site", m).numpy() for m in range(b, e)], [ch.view("bond", m).numpy() for m in range(b, e)],
                 reps)
    ch.close()


@pytest.mark.parametrize("n,d,chi,workers", [(10, 3, 16, 0), (12, 5, 64, 4)])
def test_one_rank_chain_matches_oracle(n, d, chi, workers):
    sites, bonds = chain_state(n, d, chi, seed=n * d + chi)
    layers = host_layers(n, d)
    kw = dict(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=0, delta_chi_rel=0.0, compute_explicit_error=True)
    out = {}
    with Context(0) as ctx:
        run_rank(ctx, n, sites, bonds, layers, 0, 1, None, 2, kw, workers, out)
    o_sites, o_bonds = sites, bonds
    o_reps = []
    for _ in range(2):
        o_sites, o_bonds, r = ref.tebd_step_finite_hastings(
            o_sites, o_bonds, [("even" if p == 0 else "odd", g) for p, g in layers], "qr", ref.TruncationPolicy(**kw))
        o_reps += r
    d_sites, d_bonds, d_reps = out[0]
    z = ref.clock_operators(d)[0]
    for m in range(n):
        zd = ref.expectation_from_weight(ref.left_weight(d_bonds[m]), d_sites[m], z)
        zo = ref.expectation_from_weight(ref.left_weight(o_bonds[m]), o_sites[m], z)
        assert abs(zd - zo) < 1e-10
    assert [r.bond for r in d_reps] == [b for b, _ in o_reps]
    for r, (_, ro) in zip(d_reps, o_reps):
        assert abs(r.report.eps_trunc - ro.eps_trunc) <= 1e-10 * ro.eps_trunc + 2e-13 * ro.eps_trunc ** 0.5 + 1e-20


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_chain_bitwise_equals_one_rank(world):
    n, d, chi = 12, 4, 32
    sites, bonds = chain_state(n, d, chi, seed=77)
    layers = host_layers(n, d)
    kw = dict(chi_max=chi, sv_cutoff=1e-14, delta_chi_abs=0, delta_chi_rel=0.0, compute_explicit_error=True)
    ref_out = {}
    with Context(0) as ctx:
        run_rank(ctx, n, sites, bonds, layers, 0, 1, None, 2, kw, 2, ref_out)
    lb = Loopback(world)
    ctxs = [Context(0) for _ in range(world)]
    out, errs = {}, []

    def body(r):
        try:
            run_rank(ctxs[r], n, sites, bonds, layers, r, world, lb, 2, kw, 2, out)
        except Exception as ex:  # surfaced below
            errs.append(ex)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    one_sites, one_bonds, one_reps = ref_out[0]
    for r in range(world):
        b, e = partition(n, world, r)
        s, x, _ = out[r]
        for m in range(b, e):
            assert np.array_equal(s[m - b], one_sites[m]), (r, m)
            assert np.array_equal(x[m - b], one_bonds[m]), (r, m)
    # every bond reported exactly once per layer across the ranks
    got = sorted(rep.bond for r in range(world) for rep in out[r][2])
    assert got == sorted(rep.bond for rep in one_reps)
    for c in ctxs:
        c.close()
    lb.close()


@pytest.mark.parametrize("torch_first", [True, False])
def test_nccl_transport_selftest(torch_first):
    """The chain's NCCL path on one GPU: libnccl resolved at run time (torch's
    build when torch is loaded), a one-rank communicator, grouped send/recv to
    itself, bytes round-trip (the multi-rank runs need more GPUs)."""
    import ctypes as C
    import subprocess
    import sys
    code = ("import ctypes as C\n" + ("import torch\n" if torch_first else "") +
            "from paper_2212_09782_b200 import _capi\n"
            "lib = _capi.load(); ok = C.c_int(0)\n"
            "_capi.check(lib.qt_nccl_selftest(0, 21 * 1024 * 1024, C.byref(ok)))\n"
            "assert ok.value == 1\n" + ("import torch.distributed\n" if not torch_first else "") + "print('NCCL OK')\n")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=__import__("conftest").ROOT)
    assert p.returncode == 0 and "NCCL OK" in p.stdout, p.stdout + p.stderr[-3000:]
