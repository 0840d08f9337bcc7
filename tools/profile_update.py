"""One eager two-site update of a bench config after warm-up, for ncu
(prints the library launch counter before / inside the profiled update)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2212_09782_b200 import _capi, model  # noqa: E402
from paper_2212_09782_b200 import qrtebd as q  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="north")
    ap.add_argument("--warmup", type=int, default=1)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    desc, d, chi, scheme, explicit, _ = cfg
    ctx = _capi.Context(0)
    sites, bonds = bench.synthetic_state(d, chi)
    dev = [ctx.tensor(t) for t in (bonds[0], sites[0], sites[1])]
    u = ctx.tensor(model.make_gate(model.bond_hamiltonian(d, 2.0), 0.025))
    pol = q.TruncationPolicy(**bench.policy_kw(cfg))
    fn = q.apply_gate_qr if scheme == "qr" else q.apply_gate_qr_cbe
    kw = {"want_left_iso": False} if scheme == "qr" else {}
    for _ in range(a.warmup):
        fn(*dev, u, pol, ctx, **kw)
    ctx.synchronize()
    n0 = ctx.lib.qt_kernel_launches()
    fn(*dev, u, pol, ctx, **kw)
    ctx.synchronize()
    print(f"launches_before={n0} launches_profiled={ctx.lib.qt_kernel_launches() - n0}", flush=True)


if __name__ == "__main__":
    main()
