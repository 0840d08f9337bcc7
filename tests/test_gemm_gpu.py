"""K-GEMM parity: complex128 DMMA GEMM vs NumPy (zgemm), all op combinations,
ragged shapes, batching, permuted stores and split-K.  Floating point:
tolerance 1e-13 relative Frobenius."""
import numpy as np
import pytest

from paper_2212_09782_b200.qrtebd import zgemm

pytestmark = pytest.mark.gpu


def crand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def op(x, o):
    return x if o == 0 else x.conj().T


@pytest.mark.parametrize("opa,opb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(64, 128, 16), (37, 53, 29), (5, 7, 3), (200, 130, 300), (1, 1, 1),
                                   (32, 300, 1000), (25, 64, 25),
                                   # makespan-model shapes: split-K over 64 x 128 tiles, K = 32 updates
                                   (1280, 256, 1280), (2000, 300, 32)])
def test_zgemm_ops(ctx, opa, opb, m, n, k):
    rng = np.random.default_rng(m * 1000 + n * 10 + k + 7 * opa + 13 * opb)
    a = crand(rng, *((m, k) if opa == 0 else (k, m)))
    b = crand(rng, *((k, n) if opb == 0 else (n, k)))
    c0 = crand(rng, m, n)
    ta, tb, tc = ctx.tensor(a), ctx.tensor(b), ctx.tensor(c0)
    zgemm(ctx, opa, opb, m, n, k, ta.ptr, a.shape[1], tb.ptr, b.shape[1], tc.ptr, n, alpha=-0.5, beta=2.0)
    ref = -0.5 * op(a, opa) @ op(b, opb) + 2.0 * c0
    assert rel(tc.numpy(), ref) < 1e-13


def test_zgemm_batched_shared_a(ctx):
    rng = np.random.default_rng(3)
    m, n, k, nb = 50, 70, 40, 5
    a = crand(rng, m, k)
    b = crand(rng, nb, k, n)
    ta, tb, tc = ctx.tensor(a), ctx.tensor(b), ctx.tensor(np.zeros((nb, m, n)))
    zgemm(ctx, 0, 0, m, n, k, ta.ptr, k, tb.ptr, n, tc.ptr, n, batch=nb, stride_a=0, stride_b=k * n,
          stride_c=m * n)
    ref = np.einsum("mk,bkn->bmn", a, b)
    assert rel(tc.numpy(), ref) < 1e-13


def test_zgemm_split_k_deterministic(ctx):
    # tall-K skinny output triggers split-K; result must be bitwise reproducible
    rng = np.random.default_rng(11)
    m, n, k = 32, 96, 6000
    a = crand(rng, k, m)
    b = crand(rng, k, n)
    ta, tb = ctx.tensor(a), ctx.tensor(b)
    outs = []
    for _ in range(2):
        tc = ctx.tensor(np.zeros((m, n)))
        zgemm(ctx, 1, 0, m, n, k, ta.ptr, m, tb.ptr, n, tc.ptr, n)
        outs.append(tc.numpy())
    assert rel(outs[0], a.conj().T @ b) < 1e-13
    assert np.array_equal(outs[0], outs[1])
