"""GPU SVD/EIG-TEBD comparators (cuSOLVER baselines) against the oracle's
apply_gate_svd / apply_gate_eig (proj/src/gates.cpp:250-341)."""
import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200.comparators import apply_gate_eig_gpu, apply_gate_svd_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fn,ofn", [(apply_gate_svd_gpu, ref.apply_gate_svd), (apply_gate_eig_gpu, ref.apply_gate_eig)])
def test_spectral_comparators_match_oracle(fn, ofn):
    xi, bm, bn, u, pol = ref.bench_cell_inputs(3, 12, "svd")
    pol = ref.TruncationPolicy(chi_max=10, sv_cutoff=1e-14)
    g = fn(xi, bm, bn, u, pol)
    o = ofn(xi, bm, bn, u, pol)
    assert (g.chi_after, g.chi_expanded) == (o.report.chi_after, o.report.chi_expanded)
    assert abs(g.eps_trunc - o.report.eps_trunc) <= 1e-8 * o.report.eps_trunc + 1e-16
    assert np.allclose(np.diag(g.xi_n.cpu().numpy()).real, np.diag(o.xi_n).real, atol=1e-12)
    # gauge-invariant two-site block Xi~ B~n^... : B~m Xi~ isn't gauge-fixed; compare the block
    blk_g = np.einsum("iak,kl,jlc->iajc", g.b_m.cpu().numpy(), np.eye(g.chi_after), g.b_n.cpu().numpy())
    blk_o = np.einsum("iak,kl,jlc->iajc", o.b_m, np.eye(o.report.chi_after), o.b_n)
    assert np.allclose(blk_g, blk_o, atol=1e-10 * np.abs(blk_o).max())
