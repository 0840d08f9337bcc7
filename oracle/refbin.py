"""TEST INFRASTRUCTURE: Python driver of the reference itself.

oracle/_ref/ref_update is the reference's own apply_gate
(proj/src/gates.cpp:452-462), compiled from /root/reference/proj/src in place
with the Eigen-subset shim (oracle/Makefile).  `apply_gate` here writes the
inputs, runs it, and reads the outputs back, so tests can pin the NumPy
restatement (oracle/qrtebd_oracle.py) and generate golden fixtures
(tests/golden/make_ref_golden.py).  Only tests/ may use this module.
"""
from __future__ import annotations

import os
import subprocess
import tempfile
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_UPDATE = os.path.join(HERE, "_ref", "ref_update")
SCHEMES = {"svd": 0, "eig": 1, "qr": 2, "qr_cbe": 3}


def available() -> bool:
    return os.access(REF_UPDATE, os.X_OK)


@dataclass
class RefUpdate:
    b_m: np.ndarray
    xi_n: np.ndarray
    b_n: np.ndarray
    left_iso: Optional[np.ndarray]
    chi_before: int
    chi_expanded: int
    chi_after: int
    eps_trunc: float
    discarded_weight: float


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def apply_gate(scheme: str, xi, b_m, b_n, u, chi_max=1024, sv_cutoff=1e-14, target_eps=0.0, delta_chi_abs=100,
               delta_chi_rel=0.1, chi_max_expansion=0, qr_sweeps=1, compute_explicit_error=True,
               skip_renormalize=False) -> RefUpdate:
    d, chi_m, chi_n = b_m.shape
    chi_r = b_n.shape[2]
    chi_l = xi.shape[0]
    hdr = np.zeros(16, dtype=np.int64)
    hdr[:12] = [SCHEMES[scheme], d, chi_l, chi_m, chi_n, chi_r, chi_max, delta_chi_abs, chi_max_expansion,
                qr_sweeps, int(compute_explicit_error), int(skip_renormalize)]
    hd = np.array([sv_cutoff, target_eps, delta_chi_rel, 0.0])
    with tempfile.TemporaryDirectory() as td:
        fin, fout = os.path.join(td, "in.bin"), os.path.join(td, "out.bin")
        with open(fin, "wb") as f:
            for a in (hdr, hd):
                f.write(a.tobytes())
            for a in (xi, b_m, b_n, u):
                f.write(np.ascontiguousarray(a, dtype=np.complex128).tobytes())
        p = subprocess.run([REF_UPDATE, fin, fout], capture_output=True, text=True)
        if p.returncode != 0:
            raise RefError(p.returncode, p.stderr.strip())
        raw = open(fout, "rb").read()
    oh = np.frombuffer(raw[:64], dtype=np.int64)
    od = np.frombuffer(raw[64:80], dtype=np.float64)
    kk, has_left = int(oh[0]), bool(oh[1])
    body = np.frombuffer(raw[80:], dtype=np.complex128)
    off = 0

    def take(shape):
        nonlocal off
        n = int(np.prod(shape))
        a = body[off:off + n].reshape(shape).copy()
        off += n
        return a

    bm = take((d, chi_m, kk))
    xin = take((kk, kk))
    bn = take((d, kk, chi_r))
    li = take((d, chi_l, kk)) if has_left else None
    return RefUpdate(bm, xin, bn, li, int(oh[2]), int(oh[3]), int(oh[4]), float(od[0]), float(od[1]))
