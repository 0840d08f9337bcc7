"""Accuracy of the device zgemm against numpy for every op(A)/op(B) pair
(complex operands with unequal real/imaginary scales)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_09782_b200._capi import Context  # noqa: E402
from paper_2212_09782_b200.qrtebd import zgemm  # noqa: E402

ctx = Context(0)
rng = np.random.default_rng(1)
m, n, k = 700, 520, 900
for opa in (0, 1):
    for opb in (0, 1):
        A = rng.standard_normal((m, k)) + 1j * 1e-3 * rng.standard_normal((m, k))
        B = rng.standard_normal((k, n)) * 1e-2 + 1j * rng.standard_normal((k, n))
        Ast = A if opa == 0 else A.conj().T.copy()
        Bst = B if opb == 0 else B.conj().T.copy()
        ta, tb, tc = ctx.tensor(Ast), ctx.tensor(Bst), ctx.tensor(np.zeros((m, n)) + 0j)
        zgemm(ctx, opa, opb, m, n, k, ta.ptr, Ast.shape[1], tb.ptr, Bst.shape[1], tc.ptr, n, 1.0, 0.0)
        ctx.synchronize()
        C = tc.numpy()
        ref = A @ B
        err = np.abs(C - ref).max() / (np.abs(A).max() * np.abs(B).max() * k)
        print(f"op{opa}{opb}: max|dC| / (max|A| max|B| k) = {err:.2e}  re {np.abs(C.real-ref.real).max():.2e} "
              f"im {np.abs(C.imag-ref.imag).max():.2e}")
