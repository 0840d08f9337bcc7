"""Device verification suite (run_verify, proj/src/run.cpp:548-696) and the
finite isometry checks (proj/src/mps.cpp:39-41, :143-164) against the oracle."""
import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import qrtebd as q
from paper_2212_09782_b200.verify import run_verify

pytestmark = pytest.mark.gpu


def test_left_defect_matches_oracle(ctx):
    rng = np.random.default_rng(2)
    b = rng.standard_normal((3, 7, 5)) + 1j * rng.standard_normal((3, 7, 5))
    assert abs(q.left_defect(b, ctx) - ref.left_defect(b)) < 1e-12 * ref.left_defect(b)
    iso = ref.random_right_isometry(rng, 3, 4, 6).transpose(0, 2, 1).conj().copy()  # left-isometric (3, 6, 4)
    assert q.left_defect(iso, ctx) < 1e-13


def test_check_isometric_finite_matches_oracle(ctx):
    d, n = 2, 6
    layers = [(p, [ctx.tensor(u) for u in gs]) for p, gs in ref.finite_layers(d, 2.0, n, 0.1, 2)]
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    st = q.product_state_finite(d, n, v, ctx)
    for _ in range(2):
        q.tebd_step_finite(st, layers, "qr", q.TruncationPolicy(chi_max=8), in_place=True)
    rep = q.check_isometric_finite(st, 1e-10)
    sites, c, cm = st.to_numpy()
    ok, mx, parts = ref.check_isometric_finite(ref.FiniteMPS(d, sites, c, cm), 1e-10)
    assert rep.passed == ok and abs(rep.max_defect() - mx) < 1e-14
    assert np.allclose(rep.right_defects, parts["right"], atol=1e-14)
    assert np.allclose(rep.left_defects, parts["left"], atol=1e-14)


def test_run_verify_passes_and_fault_flag_fails_norm_check(ctx):
    rep = run_verify(ctx=ctx)
    assert rep.all_pass(), rep.to_json()
    names = [c.name for c in rep.checks]
    assert names == ["product_state_isometry", "ed_match_d2_L8", "ed_match_d3_L4", "trotter_order_ratio",
                     "scheme_agreement", "uniform_isometry_drift", "finite_isometry_after_gates",
                     "norm_conservation"]
    bad = run_verify(fault_skip_renormalize=True, ctx=ctx)
    failed = [c.name for c in bad.checks if not c.passed]
    assert failed == ["norm_conservation"], bad.to_json()
