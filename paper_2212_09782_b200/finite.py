"""Finite open chain in Hastings form, sites sharded across ranks
(SURVEY.md §8(a) row a10, §8(e)).

The chain keeps a bond matrix on every bond (Xi[m] = bond left of site m,
Xi[0] = [[1]]) and updates bond (m, m+1) with
(B[m], Xi[m+1], B[m+1]) <- apply_gate(Xi[m], B[m], B[m+1], U_m) -- the uniform
step of proj/src/gates.cpp:513-540 without the wraparound bond.  Same-parity
updates are independent (proj/tests/test_tebd.cc:139-175), so sites are split
into contiguous, even-aligned blocks, one per rank:

  * even layers touch only bonds inside a block: no communication;
  * odd layers have one straddling bond (e_k - 1, e_k) per block boundary:
    rank k+1 sends B[e_k] to rank k, rank k updates the bond and returns
    Xi[e_k] and B[e_k] -- posted before the interior bonds so the transfer
    overlaps their compute (isend/irecv on the communication stream).

Nothing else is exchanged (no collective on the data path).  The transport is
torch.distributed point-to-point: NCCL over NVLink for device tensors, gloo
for the CPU tests.  The per-bond update is pluggable: the device backend calls
the C-ABI (qt_apply_gate); the tests plug in the oracle to check the
partition/exchange logic on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Sequence, Tuple

import numpy as np


def partition(n_sites: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous even-aligned site blocks [start, end) for each rank."""
    if n_sites < 2:
        raise ValueError("chain needs at least two sites")
    pairs = n_sites // 2  # blocks hold whole (even, odd) site pairs
    world = max(1, min(world, pairs))
    base, extra = divmod(pairs, world)
    out, s = [], 0
    for r in range(world):
        e = s + 2 * (base + (1 if r < extra else 0))
        out.append((s, e))
        s = e
    out[-1] = (out[-1][0], n_sites)  # an odd last site joins the last block
    return out


@dataclass
class Backend:
    """apply(xi, bm, bn, u) -> (bm', xi', bn', report); to_wire/from_wire move a
    tensor into / out of a torch tensor for torch.distributed."""

    apply: Callable
    to_wire: Callable
    from_wire: Callable
    shape_of: Callable


class ShardedChain:
    """The sites [start, end) of an open chain owned by this rank."""

    def __init__(self, sites: Sequence, bonds: Sequence, n_sites: int, rank: int, world: int, backend,
                 dist=None, periodic: bool = False):
        # periodic: a uniform unit cell of n_sites (even) sites whose odd layer
        # includes the wrap bond (n-1, 0) (proj/src/gates.cpp:524-537); the
        # blocks form a ring and the last rank's straddling bond is the wrap
        # (uniform large unit cell)
        if periodic and n_sites % 2:
            raise ValueError("a periodic (uniform) cell needs an even number of sites")
        self.periodic = periodic
        self.n = n_sites
        self.rank = rank
        self.world = world
        self.blocks = partition(n_sites, world)
        self.start, self.end = self.blocks[rank]
        self.sites = {m: sites[m - self.start] for m in range(self.start, self.end)}
        self.bonds = {m: bonds[m - self.start] for m in range(self.start, self.end)}
        # backend: one Backend, or a list whose first entry serves the exchanges
        # and the straddling bond while the others update interior bonds of a
        # layer concurrently (one host thread per backend; same-parity bonds
        # are independent, proj/tests/test_tebd.cc:139-175)
        pool = list(backend) if isinstance(backend, (list, tuple)) else [backend]
        self.be = pool[0]
        self.workers = pool[1:]
        self.dist = dist
        self.reports: List = []

    # ---- exchanges (torch.distributed point-to-point)
    def _send_tensor(self, t, dst):
        import torch
        shp = self.be.shape_of(t)
        hdr = torch.tensor(list(shp) + [0] * (4 - len(shp)) + [len(shp)], dtype=torch.int64)
        payload = self.be.to_wire(t)
        if payload.is_cuda:
            hdr = hdr.to(payload.device)
        return [self.dist.isend(hdr, dst), self.dist.isend(payload, dst)], (hdr, payload)

    def _post_header(self, src, device):
        import torch
        hdr = torch.empty(5, dtype=torch.int64, device=device)
        return self.dist.irecv(hdr, src), hdr

    def _recv_tensor(self, src, device, posted=None):
        import torch
        req, hdr = posted if posted is not None else self._post_header(src, device)
        req.wait()
        rank = int(hdr[4].item())
        shp = tuple(int(x) for x in hdr[:rank].tolist())
        buf = torch.empty(int(np.prod(shp)) * 2, dtype=torch.float64, device=device)
        self.dist.recv(buf, src)
        return self.be.from_wire(buf, shp)

    def layer(self, parity: int, gates: Sequence, device="cpu"):
        """One Trotter layer: bonds (m, m+1) with m % 2 == parity; gates[m] acts on (m, m+1)."""
        start, end = self.start, self.end
        if self.periodic:
            has_right_straddle = has_left_straddle = parity == 1 and self.world > 1
        else:
            has_right_straddle = parity == 1 and self.rank + 1 < self.world and end < self.n
            has_left_straddle = parity == 1 and self.rank > 0
        right, left = (self.rank + 1) % self.world, (self.rank - 1) % self.world
        pending = []
        # the right neighbour's first site is the right half of our straddling bond
        if has_left_straddle:
            reqs, keep = self._send_tensor(self.sites[start], left)
            pending.append((reqs, keep))
        right_hdr = self._post_header(right, device) if has_right_straddle else None
        # interior bonds of this parity (overlap the neighbour's transfer)
        interior = list(range(start + parity, end - 1, 2))
        if self.workers and len(interior) > 1:
            self._update_concurrent(interior, gates)
        else:
            for m in interior:
                self._update(m, m + 1, gates[m])
        # the wrap bond of a one-rank periodic cell is local
        if self.periodic and parity == 1 and self.world == 1:
            m = self.n - 1
            bm, xi, bn, rep = self.be.apply(self.bonds[m], self.sites[m], self.sites[0], gates[m])
            self.sites[m] = bm
            self.bonds[0] = xi
            self.sites[0] = bn
            self.reports.append((0, rep))
        # the straddling bond (end-1, end mod n): owned here, results returned
        if has_right_straddle:
            right_site = self._recv_tensor(right, device, right_hdr)
            m = end - 1
            bm, xi, bn, rep = self.be.apply(self.bonds[m], self.sites[m], right_site, gates[m])
            self.sites[m] = bm
            self.reports.append(((m + 1) % self.n, rep))
            for t in (xi, bn):
                reqs, keep = self._send_tensor(t, right)
                pending.append((reqs, keep))
        if has_left_straddle:
            self.bonds[start] = self._recv_tensor(left, device)
            self.sites[start] = self._recv_tensor(left, device)
        for reqs, _ in pending:
            for r in reqs:
                r.wait()

    def _update(self, m, n, gate):
        bm, xi, bn, rep = self.be.apply(self.bonds[m], self.sites[m], self.sites[n], gate)
        self.sites[m] = bm
        self.bonds[n] = xi
        self.sites[n] = bn
        self.reports.append((n, rep))

    def _update_concurrent(self, bonds_m, gates):
        """Bond m -> worker m_index % K; each worker runs its bonds in order on
        its own context (stream + workspace).  Results are committed in bond
        order, so the chain state and the report list do not depend on the
        interleaving."""
        from concurrent.futures import ThreadPoolExecutor

        k = len(self.workers)
        lanes = [bonds_m[i::k] for i in range(k)]

        def run(i):
            be = self.workers[i]
            return [(m, be.apply(self.bonds[m], self.sites[m], self.sites[m + 1], gates[m])) for m in lanes[i]]

        with ThreadPoolExecutor(max_workers=k) as ex:
            done = dict(kv for part in ex.map(run, range(k)) for kv in part)
        for m in bonds_m:
            bm, xi, bn, rep = done[m]
            self.sites[m] = bm
            self.bonds[m + 1] = xi
            self.sites[m + 1] = bn
            self.reports.append((m + 1, rep))

    def step(self, layers: Sequence[Tuple[int, Sequence]], device="cpu"):
        """layers: [(parity 0|1, gates per bond m)] (finite_trotter_layers, gates.hpp:160-173)."""
        self.reports = []
        for parity, gates in layers:
            self.layer(parity, gates, device)
        return self.reports


def chain_dims(n_sites: int, d: int, chi_max: int) -> List[int]:
    """Bond dimensions of a saturated open chain: chi_m = min(d^m, d^(N-m), chi_max),
    m = 0..N (chi_0 = chi_N = 1), SURVEY.md §8(d) C5."""
    out = []
    for m in range(n_sites + 1):
        a = min(m, n_sites - m)
        out.append(1 if a == 0 else int(min(chi_max, d ** min(a, 60))))
    return out


def random_chain_state(ctx, n_sites: int, d: int, chi_max: int, start: int, end: int, seed: int = 0x51AB):
    """Random right-isometric site tensors and normalized bond matrices for
    sites [start, end), generated on the device (torch RNG seeded per site so
    every rank builds bit-identical tensors for the sites it owns; right
    isometries from the device LQ, proj/src/run.cpp:345-349).  Returns
    (sites, bonds, keepalive) as device tensors."""
    import torch

    from . import qrtebd as q

    chi = chain_dims(n_sites, d, chi_max)
    dev = torch.device("cuda", torch.cuda.current_device())
    keep, sites, bonds = [], [], []
    for m in range(start, end):
        cl, cr = chi[m], chi[m + 1]
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed * 1000003 + m)
        g = torch.randn(cl, d * cr, dtype=torch.complex128, device=dev, generator=gen)
        torch.cuda.synchronize()  # torch's stream -> the library's stream
        _, qm = q.lq_reduced(ctx.wrap(g.data_ptr(), (cl, d * cr)), ctx)  # (cl, d*cr), orthonormal rows
        qt = torch.empty(cl, d * cr, dtype=torch.complex128, device=dev)
        from . import _capi
        dst = ctx.wrap(qt.data_ptr(), (cl, d * cr))  # keep the handle alive across the call
        _capi.check(ctx.lib.qt_tensor_copy(dst.h, qm.h))
        ctx.synchronize()
        b = qt.reshape(cl, d, cr).permute(1, 0, 2).contiguous()
        if m == 0:
            x = torch.ones(1, 1, dtype=torch.complex128, device=dev)
        else:
            x = torch.randn(cl, cl, dtype=torch.complex128, device=dev, generator=gen)
            x = x / torch.linalg.vector_norm(x)
        torch.cuda.synchronize()
        keep += [g, qt, b, x]
        sites.append(ctx.wrap(b.data_ptr(), tuple(b.shape)))
        bonds.append(ctx.wrap(x.data_ptr(), tuple(x.shape)))
    return sites, bonds, keep


def numpy_backend(apply_fn) -> Backend:
    """CPU backend over NumPy tensors (tests: apply_fn = oracle apply_gate)."""
    import torch

    def to_wire(t):
        return torch.from_numpy(np.ascontiguousarray(t).view(np.float64).reshape(-1).copy())

    def from_wire(buf, shp):
        return buf.numpy().view(np.complex128).reshape(shp).copy()

    return Backend(apply=apply_fn, to_wire=to_wire, from_wire=from_wire, shape_of=lambda t: tuple(t.shape))


def device_backend(ctx, scheme: str, policy) -> Backend:
    """B200 backend: updates through the C-ABI, exchanges through NCCL with
    torch CUDA staging buffers (qt_tensor_copy into wrapped torch memory)."""
    import ctypes as C

    import torch

    from . import _capi
    from . import qrtebd as q

    pol = policy.to_c() if isinstance(policy, q.TruncationPolicy) else policy
    # bond updates of a chain run on several contexts at once: small blocks
    # skip the pipelined QR pair there (qt_ctx_set_qr_pair_min_rows)
    _capi.check(ctx.lib.qt_ctx_set_qr_pair_min_rows(ctx.h, 256))

    def apply(xi, bm, bn, u):
        upd = q.apply_gate(scheme, xi, bm, bn, u, pol, ctx) if scheme == "qr_cbe" else \
            q.apply_gate_qr(xi, bm, bn, u, pol, ctx, want_left_iso=False)
        return upd.b_m, upd.xi_n, upd.b_n, upd.report

    def to_wire(t):
        shp = t.shape
        buf = torch.empty(int(np.prod(shp)) * 2, dtype=torch.float64, device=f"cuda:{torch.cuda.current_device()}")
        view = ctx.wrap(buf.data_ptr(), shp)
        _capi.check(ctx.lib.qt_tensor_copy(view.h, t.h))
        ctx.synchronize()
        return buf

    def from_wire(buf, shp):
        torch.cuda.current_stream().synchronize()
        t = ctx.empty(shp)
        view = ctx.wrap(buf.data_ptr(), shp)
        _capi.check(ctx.lib.qt_tensor_copy(t.h, view.h))
        ctx.synchronize()
        return t

    return Backend(apply=apply, to_wire=to_wire, from_wire=from_wire, shape_of=lambda t: tuple(t.shape))
