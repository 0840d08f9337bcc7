"""Run one zgemm of a given shape a few times (for ncu / timing)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_09782_b200._capi import Context  # noqa: E402
from paper_2212_09782_b200.qrtebd import zgemm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("m", type=int)
ap.add_argument("n", type=int)
ap.add_argument("k", type=int)
ap.add_argument("--opa", type=int, default=0)
ap.add_argument("--opb", type=int, default=0)
ap.add_argument("--beta", type=float, default=1.0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
ctx = Context(0)
rng = np.random.default_rng(0)
A = rng.standard_normal((a.m, a.k) if a.opa == 0 else (a.k, a.m)) + 0j
B = rng.standard_normal((a.k, a.n) if a.opb == 0 else (a.n, a.k)) + 0j
ta, tb, tc = ctx.tensor(A), ctx.tensor(B), ctx.tensor(np.zeros((a.m, a.n)))
import torch
st = torch.cuda.ExternalStream(ctx.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(a.reps + 1):
    if i == 1:
        e0.record(st)
    zgemm(ctx, a.opa, a.opb, a.m, a.n, a.k, ta.ptr, A.shape[1], tb.ptr, B.shape[1], tc.ptr, a.n, -1.0, a.beta)
e1.record(st)
e1.synchronize()
ms = e0.elapsed_time(e1) / a.reps
print(f"{a.m}x{a.n}x{a.k} op{a.opa}{a.opb}: {ms*1e3:.1f} us  {8*a.m*a.n*a.k/ms/1e9:.2f} TF")
