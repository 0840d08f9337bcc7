"""Run one device eigh of a random Hermitian n x n matrix (ncu target)."""
import sys
import os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_09782_b200._capi import Context  # noqa: E402
from paper_2212_09782_b200 import qrtebd as q  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 356
ctx = Context(0)
rng = np.random.default_rng(0)
l = np.tril(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * np.exp(-np.arange(n) / 20.0)
g = l.conj().T @ l
for _ in range(2):
    w, v = q.eigh(g, ctx)
print("ok", w[:3])
