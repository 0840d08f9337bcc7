"""GPU SVD-/EIG-TEBD comparators.

apply_gate_svd / apply_gate_eig (proj/src/gates.cpp:250-341) on the same B200
as the QR path, for the paper's QR-vs-SVD comparison measured on one device.
These are BASELINES, not the product: the dense decompositions are cuSOLVER's
(zgesvd / zheevd through torch.linalg), the contractions torch's cuBLAS
zgemm.  The product path (apply_gate_qr / apply_gate_qr_cbe) never calls into
this module.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["SpectralUpdate", "apply_gate_svd_gpu", "apply_gate_eig_gpu"]


@dataclass
class SpectralUpdate:
    """GateUpdate of the spectral schemes (proj/include/qrtebd/gates.hpp:70-76), torch tensors."""

    b_m: "object"
    xi_n: "object"
    b_n: "object"
    left_iso: "object"
    chi_before: int
    chi_expanded: int
    chi_after: int
    eps_trunc: float
    discarded_weight: float


def _t(a, device):
    import torch
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.complex128)
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.complex128, device=device)


def _theta(xi, b_m, b_n, u, device):
    """build_theta, gates.cpp:123-182: phi_ev (beta,i,j,delta) and theta (alpha i) x (j delta)."""
    import torch
    xi, b_m, b_n, u = (_t(a, device) for a in (xi, b_m, b_n, u))
    d, chi_m, chi_n, chi_r, chi_l = b_m.shape[0], b_m.shape[1], b_m.shape[2], b_n.shape[2], xi.shape[0]
    phi = torch.einsum("iab,jbc->ijac", b_m, b_n).reshape(d * d, chi_m * chi_r)
    ev = (u.reshape(d * d, d * d) @ phi).reshape(d, d, chi_m, chi_r)
    phi_ev = ev.permute(2, 0, 1, 3).contiguous()
    theta = (xi @ phi_ev.reshape(chi_m, d * d * chi_r)).reshape(chi_l * d, d * chi_r)
    return phi_ev, theta, (d, chi_l, chi_n, chi_r)


def _choose_kept(s_norm: np.ndarray, chi_max: int, sv_cutoff: float, target_eps: float) -> int:
    """choose_kept, gates.cpp:226-240."""
    below = np.nonzero(s_norm < sv_cutoff)[0]
    k = int(below[0]) if len(below) else len(s_norm)
    k = min(k, chi_max)
    if target_eps > 0.0:
        suffix = np.concatenate([np.cumsum((s_norm ** 2)[::-1])[::-1], [0.0]])
        over = np.nonzero(suffix <= target_eps)[0]
        k = min(k, int(over[0]))
    return max(k, 1)


def _finish(phi_ev, theta, dims, s, vdag, u_cols, policy) -> SpectralUpdate:
    """finish_spectral_update, gates.cpp:250-282."""
    import torch
    d, chi_l, chi_n, chi_r = dims
    s_host = s.detach().cpu().numpy()
    theta_norm = float(torch.linalg.vector_norm(theta).item())
    if theta_norm <= 0.0:
        raise ValueError("evolved block has zero norm")
    kk = _choose_kept(s_host / theta_norm, policy.chi_max, policy.sv_cutoff, policy.target_eps)
    kept_norm = math.sqrt(float(np.sum(s_host[:kk] ** 2)))
    den = theta_norm if policy.skip_renormalize else kept_norm
    xi_n = torch.diag(s[:kk].to(torch.complex128) * (1.0 / den if den > 0 else 0.0))
    b_n = vdag[:kk].reshape(kk, d, chi_r).permute(1, 0, 2).contiguous()
    b_m = torch.einsum("bijd,jkd->ibk", phi_ev, b_n.conj()).contiguous()
    left = (u_cols[:, :kk].reshape(chi_l, d, kk).permute(1, 0, 2).contiguous() if u_cols is not None else None)
    total2 = theta_norm * theta_norm
    disc = max(0.0, total2 - kept_norm * kept_norm)
    return SpectralUpdate(b_m, xi_n, b_n, left, chi_n, min(chi_l * d, d * chi_r), kk, disc / total2, disc)


def apply_gate_svd_gpu(xi, b_m, b_n, u, policy, device="cuda") -> SpectralUpdate:
    """apply_gate_svd, gates.cpp:312-322: full SVD of theta (cuSOLVER)."""
    import torch
    phi_ev, theta, dims = _theta(xi, b_m, b_n, u, device)
    uu, s, vh = torch.linalg.svd(theta, full_matrices=False)
    return _finish(phi_ev, theta, dims, s, vh, uu, policy)


def apply_gate_eig_gpu(xi, b_m, b_n, u, policy, device="cuda") -> SpectralUpdate:
    """apply_gate_eig, gates.cpp:324-341: eigh of theta^H theta (cuSOLVER), descending."""
    import torch
    phi_ev, theta, dims = _theta(xi, b_m, b_n, u, device)
    g = theta.conj().T @ theta
    w, v = torch.linalg.eigh(0.5 * (g + g.conj().T))
    w, v = torch.flip(w, [0]), torch.flip(v, [1])
    s = torch.where(w > 0, torch.sqrt(torch.clamp(w, min=0.0)), torch.zeros_like(w))
    return _finish(phi_ev, theta, dims, s, v.conj().T, None, policy)
