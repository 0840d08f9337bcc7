"""Gate input preparation (host side, computed once per run, never timed).

Clock model of proj/include/qrtebd/clock.hpp:11-17 and the gate
exp(-i dt h) of proj/src/gates.cpp:50-57.  The reference computes these on the
host too (proj/src/run.cpp:246-253); SURVEY.md §2.2 keeps them host-side: they
are the inputs of the device hot path, d^2 x d^2 with d <= 20.
"""
from __future__ import annotations

import math

import numpy as np


def clock_operators(d: int):
    """Z = diag(w^k), X = cyclic shift (proj/src/clock.cpp:54-63)."""
    if d < 2:
        raise ValueError("clock model needs d >= 2")
    step = 2.0 * math.pi / d
    z = np.zeros((d, d), dtype=np.complex128)
    x = np.zeros((d, d), dtype=np.complex128)
    for k in range(d):
        z[k, k] = complex(math.cos(step * k), math.sin(step * k))
        x[k, (k + 1) % d] = 1.0
    return z, x


def bond_hamiltonian_weighted(d: int, g: float, left_weight: float, right_weight: float) -> np.ndarray:
    """-(Z (x) Z^dag + h.c.) - g w_l (X+X^dag) (x) 1 - g w_r 1 (x) (X+X^dag)
    (proj/src/clock.cpp:65-78)."""
    z, x = clock_operators(d)
    eye = np.eye(d, dtype=np.complex128)
    onsite = g * (x + x.conj().T)
    zz = np.kron(z, z.conj().T)
    return -(zz + zz.conj().T) - left_weight * np.kron(onsite, eye) - right_weight * np.kron(eye, onsite)


def bond_hamiltonian(d: int, g: float, kind: str = "bulk") -> np.ndarray:
    """proj/src/clock.cpp:80-90."""
    wl, wr = {"bulk": (0.5, 0.5), "left_edge": (1.0, 0.5), "right_edge": (0.5, 1.0)}[kind]
    return bond_hamiltonian_weighted(d, g, wl, wr)


def chain_bond_hamiltonian(d: int, g: float, bond: int, n_sites: int) -> np.ndarray:
    """Edge-weighted bond of an open chain (proj/src/clock.cpp:92-99)."""
    if n_sites < 2 or bond + 1 >= n_sites:
        raise ValueError("bond index out of range")
    wl = 1.0 if bond == 0 else 0.5
    wr = 1.0 if bond + 2 == n_sites else 0.5
    return bond_hamiltonian_weighted(d, g, wl, wr)


def make_gate(h_bond: np.ndarray, dt: float) -> np.ndarray:
    """exp(-i dt h) as a (d, d, d, d) tensor (proj/src/gates.cpp:50-57,
    proj/src/linalg.cpp:103-110)."""
    h = np.asarray(h_bond, dtype=np.complex128)
    d2 = h.shape[0]
    d = int(round(math.sqrt(d2)))
    if d * d != d2:
        raise ValueError("bond hamiltonian dimension is not d^2")
    w, v = np.linalg.eigh(0.5 * (h + h.conj().T))
    u = (v * np.exp(-1j * dt * w)) @ v.conj().T
    return np.ascontiguousarray(u.reshape(d, d, d, d))


def identity_gate(d: int) -> np.ndarray:
    return np.eye(d * d, dtype=np.complex128).reshape(d, d, d, d)


def layer_structure(dt: float, order: int):
    """proj/src/gates.cpp:489-501."""
    if order == 1:
        return [("even", dt), ("odd", dt)]
    if order == 2:
        return [("even", 0.5 * dt), ("odd", dt), ("even", 0.5 * dt)]
    raise ValueError("trotter order must be 1 or 2")


def trotter_schedule(h_bond: np.ndarray, dt: float, order: int = 2):
    """proj/src/gates.cpp:505-511."""
    return [(p, make_gate(h_bond, dte)) for p, dte in layer_structure(dt, order)]


def z1_local_vector(d: int) -> np.ndarray:
    """Initial product state |0> (Z = 1), proj/src/run.cpp:38-42."""
    v = np.zeros(d, dtype=np.complex128)
    v[0] = 1.0
    return v


def random_right_isometry(rng, d: int, chi_l: int, chi_r: int) -> np.ndarray:
    """Random site tensor B (d, chi_l, chi_r) with sum_i B^i B^i^H = 1 (the
    bench_cell input recipe, proj/src/run.cpp:345-349): orthonormal rows of
    the (chi_l, d*chi_r) matrix from a Gaussian QR, gauge-fixed."""
    g = rng.standard_normal((d * chi_r, chi_l)) + 1j * rng.standard_normal((d * chi_r, chi_l))
    q, r = np.linalg.qr(g)
    q = q * (np.diag(r) / np.abs(np.diag(r)))
    return np.ascontiguousarray(q.conj().T.reshape(chi_l, d, chi_r).transpose(1, 0, 2))
