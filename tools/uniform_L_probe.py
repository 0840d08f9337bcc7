"""Steps/s of the device-resident uniform cell for L = 2, 4, 8 (concurrent
same-parity updates for L >= 4; QT_UNIFORM_SERIAL=1 for one stream)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2212_09782_b200._capi import Context  # noqa: E402
from paper_2212_09782_b200 import model, qrtebd as q  # noqa: E402

d, chi = int(sys.argv[1]), int(sys.argv[2])
ctx = Context(0)
sched = model.trotter_schedule(model.bond_hamiltonian(d, 2.0), 0.05, 2)
gates = [(p, ctx.tensor(g)) for p, g in sched]
pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0)
for L in (2, 4, 8):
    rng = np.random.default_rng(L)
    sites = [model.random_right_isometry(rng, d, chi, chi) for _ in range(L)]
    bonds = [np.eye(chi, dtype=complex) / np.sqrt(chi)] * L
    dev = q.DeviceUniformMPS(q.UniformMPS.from_numpy(ctx, d, sites, bonds), ctx)
    for _ in range(3):
        dev.step(gates, "qr", pol)
    ctx.synchronize()
    t = time.perf_counter()
    n = 10
    for _ in range(n):
        dev.step(gates, "qr", pol)
    ctx.synchronize()
    dt = (time.perf_counter() - t) / n
    print(f"L={L} d={d} chi={chi}: {1.0 / dt:.1f} steps/s, {3 * L // 2 / dt:.0f} updates/s")
    dev.close()
