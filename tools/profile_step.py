"""Run W warm-up TEBD steps then S profiled steps of a bench config; prints the
number of library kernel launches before the profiled region (for ncu -s)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2212_09782_b200 import _capi, model  # noqa: E402
from paper_2212_09782_b200 import qrtebd as q  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    desc, d, chi, scheme, explicit, _ = bench.CONFIGS[a.config]
    ctx = _capi.Context(0)
    sites, bonds = bench.synthetic_state(d, chi)
    st = q.UniformMPS.from_numpy(ctx, d, sites, bonds)
    sched = [(p, ctx.tensor(model.make_gate(model.bond_hamiltonian(d, 2.0), dte)))
             for p, dte in model.layer_structure(0.05, 2)]
    pol = q.TruncationPolicy(**bench.policy_kw(bench.CONFIGS[a.config]))
    for _ in range(a.warmup):
        st, _ = q.tebd_step(st, sched, scheme, pol, ctx)
    ctx.synchronize()
    n0 = ctx.lib.qt_kernel_launches()
    for _ in range(a.steps):
        st, _ = q.tebd_step(st, sched, scheme, pol, ctx)
    ctx.synchronize()
    print(f"launches_before={n0} launches_profiled={ctx.lib.qt_kernel_launches() - n0}", flush=True)


if __name__ == "__main__":
    main()
