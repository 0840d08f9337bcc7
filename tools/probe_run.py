"""Box probes: FP64 DMMA/DFMA peaks, GEMM and update timings."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2212_09782_b200._capi import Context  # noqa: E402
from paper_2212_09782_b200 import qrtebd as q, model  # noqa: E402


def crand(rng, *s):
    return rng.standard_normal(s) + 1j * rng.standard_normal(s)


def time_gemm(ctx, m, n, k, opa=0, opb=0, reps=5):
    import torch
    rng = np.random.default_rng(0)
    a = ctx.tensor(crand(rng, *((m, k) if opa == 0 else (k, m))))
    b = ctx.tensor(crand(rng, *((k, n) if opb == 0 else (n, k))))
    c = ctx.empty((m, n))
    lda = k if opa == 0 else m
    ldb = n if opb == 0 else k
    st = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(2):
        q.zgemm(ctx, opa, opb, m, n, k, a.ptr, lda, b.ptr, ldb, c.ptr, n)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    ctx.synchronize()
    e0.record(st)
    for _ in range(reps):
        q.zgemm(ctx, opa, opb, m, n, k, a.ptr, lda, b.ptr, ldb, c.ptr, n)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, 8.0 * m * n * k / (ms * 1e-3) / 1e12


def main():
    out = {}
    ctx = Context(0)
    out["dmma_tflops"] = ctx.fp64_peak(0)
    out["dfma_tflops"] = ctx.fp64_peak(1)
    print("peaks", out, flush=True)
    for shp in [(1024, 1024, 1024), (5120, 1024, 5120), (5120, 1024, 5120, 0, 1), (5120, 1024, 5120, 1, 0),
                (4096, 4096, 4096), (1280, 256, 1280)]:
        ms, tf = time_gemm(ctx, *shp)
        print("gemm", shp, f"{ms:.3f} ms {tf:.2f} TF", flush=True)
        out[f"gemm_{'x'.join(map(str, shp))}"] = tf
    for d, chi in [(5, 256), (5, 1024)]:
        rng = np.random.default_rng(1)
        bm = model.random_right_isometry(rng, d, chi, chi)
        bn = model.random_right_isometry(rng, d, chi, chi)
        xi = crand(rng, chi, chi)
        xi /= np.linalg.norm(xi)
        u = model.make_gate(model.bond_hamiltonian(d, 2.0), 0.05)
        txi, tbm, tbn, tu = (ctx.tensor(a) for a in (xi, bm, bn, u))
        pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0, compute_explicit_error=False)
        for _ in range(2):
            upd = q.apply_gate_qr(txi, tbm, tbn, tu, pol, ctx, want_left_iso=False)
        ctx.synchronize()
        t0 = time.perf_counter()
        n = 3
        for _ in range(n):
            upd = q.apply_gate_qr(txi, tbm, tbn, tu, pol, ctx, want_left_iso=False)
        ctx.synchronize()
        dt = (time.perf_counter() - t0) / n
        f = __import__('bench').flops_per_update(d, chi, chi, chi, False)
        print("update", d, chi, f"{dt*1e3:.2f} ms", f"{f/dt/1e12:.2f} TF", upd.report, flush=True)
        out[f"update_d{d}_chi{chi}_ms"] = dt * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
