"""Time the device QR of random m x n matrices (panel / larfb tuning probe).

usage: python tools/qr_one.py m n [reps]   (env QT_PANEL_CS, QT_NO_LARFB_CLUSTER apply)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_09782_b200._capi import Context  # noqa: E402
from paper_2212_09782_b200 import qrtebd as q  # noqa: E402


def main():
    import torch
    m, n = int(sys.argv[1]), int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    ctx = Context(0)
    rng = np.random.default_rng(0)
    a = ctx.tensor(rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)))
    st = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(3):
        q.qr_reduced(a, ctx)
    ctx.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        q.qr_reduced(a, ctx)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"qr m={m} n={n} cs={os.environ.get('QT_PANEL_CS', '16')} {ms * 1e3:.1f} us/qr "
          f"{ms * 1e3 / max(1, (n + 31) // 32):.1f} us/panel-step")


if __name__ == "__main__":
    main()
