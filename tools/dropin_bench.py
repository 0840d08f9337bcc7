"""Reference-facing speed-up of the drop-in library: the reference's own
apply_gate loop (oracle/ref_bench.cpp, tebd_step order: even dt/2, odd dt,
even dt/2 on a uniform L=2 cell) run twice on the same synthetic state --
linked against the reference build alone (CPU, all host cores) and against
libqrtebd_api.so first (every apply_gate on the B200 with value semantics:
host tensors copied in and out of each call).

usage: python tools/dropin_bench.py [config] [budget_s]   (bench.py CONFIGS; default north)"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "north"
budget = sys.argv[2] if len(sys.argv) > 2 else "20"
desc, d, chi, scheme, explicit, (dabs, drel) = bench.CONFIGS[cfg_name]
sites, bonds = bench.synthetic_state(d, chi)
out = {"config": desc}
with tempfile.TemporaryDirectory() as td:
    path = os.path.join(td, "state.bin")
    with open(path, "wb") as f:
        for a in sites + bonds:
            f.write(np.ascontiguousarray(a, dtype=np.complex128).tobytes())
    for name in ("ref_bench", "b200_bench"):
        exe = os.path.join(ROOT, "oracle", "_ref", name)
        env = dict(os.environ, OPENBLAS_NUM_THREADS=str(os.cpu_count() or 1))
        if os.environ.get("DROPIN_MALLOC_TUNE"):
            # keep large freed blocks in the heap (no munmap / re-fault of fresh pages per call)
            env["GLIBC_TUNABLES"] = "glibc.malloc.mmap_threshold=4294967295:glibc.malloc.trim_threshold=68719476736"
        r = subprocess.run([exe, path, str(d), str(chi), scheme, "1" if explicit else "0", str(dabs), str(drel),
                            budget, "3"], capture_output=True, text=True, env=env)
        if r.returncode != 0:
            raise SystemExit(f"{name} failed: {r.stderr[-800:]}")
        res = json.loads(r.stdout.strip().splitlines()[-1])
        res["updates_per_s"] = res["updates"] / res["seconds"]
        res["steps_per_s"] = res["updates_per_s"] / 3.0
        out[name] = res
out["speedup"] = out["b200_bench"]["updates_per_s"] / out["ref_bench"]["updates_per_s"]
print(json.dumps(out))
