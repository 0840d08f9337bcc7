"""The sharded finite chain of the C-ABI (qt_chain_*, qt_tebd_step_finite_sharded;
include/qrtebd_c.h, csrc/chain.cu) from Python.

One rank per process (one GPU each): site blocks from qt_chain_partition,
interior bonds of a layer on `workers` concurrent contexts, the straddling
bonds exchanged with NCCL send/recv of raw device buffers (the NCCL unique id
travels over the caller's torch.distributed group), or -- tests on one GPU --
an in-process loopback shared by one chain per rank in separate threads.
Hastings form: bitwise the single-rank chain.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

from . import _capi
from ._capi import check, qt_bond_report
from .qrtebd import BondReport, TruncationReport, _policy


def partition(n_sites: int, world: int, rank: int) -> Tuple[int, int]:
    b, e = C.c_uint64(), C.c_uint64()
    check(_capi.load().qt_chain_partition(n_sites, world, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(_capi.load().qt_nccl_get_unique_id(buf))
    return bytes(buf)


class Loopback:
    """In-process transport between the chains of one process (tests)."""

    def __init__(self, world: int):
        self.lib = _capi.load()
        h = C.c_void_p()
        check(self.lib.qt_loopback_create(world, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.lib.qt_loopback_destroy(self.h)
            self.h = None


class DeviceChain:
    """The owned sites [begin, end) of an n-site open chain on this rank."""

    def __init__(self, ctx, n_sites: int, sites: Sequence, bonds: Sequence, rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None, loopback: Optional[Loopback] = None, workers: int = 8):
        self.ctx, self.lib, self.n = ctx, ctx.lib, n_sites
        sh = (C.c_void_p * max(1, len(sites)))(*[s.h for s in sites])
        bh = (C.c_void_p * max(1, len(bonds)))(*[b.h for b in bonds])
        idb = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id else None
        h = C.c_void_p()
        check(self.lib.qt_chain_create(ctx.h, n_sites, rank, world, idb, loopback.h if loopback else None, sh, bh,
                                       workers, C.byref(h)))
        self.h = h
        b, e = C.c_uint64(), C.c_uint64()
        check(self.lib.qt_chain_range(h, C.byref(b), C.byref(e)))
        self.begin, self.end = b.value, e.value

    def close(self):
        if self.h:
            self.lib.qt_chain_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, layers: Sequence[Tuple[int, Sequence]], scheme: str, policy=None) -> List[BondReport]:
        """layers: [(parity 0|1, gates per bond m (DeviceTensor or None))]."""
        nb = self.n - 1
        par = (C.c_int32 * max(1, len(layers)))(*[p for p, _ in layers])
        flat = []
        for _, gs in layers:
            if len(gs) != nb:
                raise ValueError("layer gate count must equal the bond count")
            flat += [g.h if g is not None else None for g in gs]
        gh = (C.c_void_p * max(1, len(flat)))(*flat)
        cap = len(layers) * (nb // 2 + 2)
        reps = (qt_bond_report * max(1, cap))()
        cnt = C.c_uint64(cap)
        pol = _policy(policy)
        check(self.lib.qt_tebd_step_finite_sharded(self.h, len(layers), par, gh, _capi.SCHEME_IDS[scheme],
                                                   C.byref(pol), reps, C.byref(cnt)))
        return [BondReport(int(reps[i].bond), TruncationReport.from_c(reps[i].report)) for i in range(cnt.value)]

    def view(self, which: str, m: int):
        h = C.c_void_p()
        check(self.lib.qt_chain_view(self.h, 0 if which == "site" else 1, m, C.byref(h)))
        return _capi.DeviceTensor(self.ctx, h)
