import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, '.')
import bench  # noqa: E402

d, chi = 5, int(os.environ.get("CHI", "1024"))
sites, bonds = bench.synthetic_state(d, chi)
with open('/tmp/state.bin', 'wb') as f:
    for a in sites + bonds:
        f.write(np.ascontiguousarray(a, dtype=np.complex128).tobytes())
for label, extra in [("blas_all", {})]:
    env = dict(os.environ, REF_BENCH_VERBOSE='1', **extra)
    out = subprocess.run(['oracle/_ref/ref_bench', '/tmp/state.bin', str(d), str(chi), 'qr', '1', '0', '0.0', '0', '3'],
                         capture_output=True, text=True, env=env)
    print(label, out.stdout.strip(), out.stderr.strip().replace("\n", " | ")[-300:], flush=True)
