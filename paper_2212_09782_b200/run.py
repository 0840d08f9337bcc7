"""Quench driver and on-disk formats.

Mirrors proj/include/qrtebd/run.hpp and proj/src/run.cpp:
  * RunConfig with the strict nested JSON schema (config_from_json,
    config_to_json; run.cpp:53-183);
  * run_quench (run.cpp:228-326): the g-quench from the Z=1 product state,
    observables every step, observables.csv / bonds.csv / config.json /
    checkpoints under out_path;
  * the checkpoint container save_mps / load_mps (proj/src/mps.cpp:259-392).

Every tebd_step and every observable runs on the device through the C-ABI
(qt_uniform_* for unit cells, qt_finite_* for open chains with the
reference's sequential move_center semantics).  The checkpoint and CSV
writers are host byte formatting only.
"""
from __future__ import annotations

import json
import math
import os
import struct
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional

import numpy as np

from . import model
from ._capi import InputError, ShapeError
from .qrtebd import (BondReport, Context, DeviceUniformMPS, FiniteMPS, TruncationPolicy, UniformMPS,
                     default_context, entropy_from_schmidt, finite_observables, product_state_finite,
                     product_state_uniform, schmidt_values_of, tebd_step_finite)
from . import _capi

__all__ = ["RunConfig", "config_from_json", "config_from_json_file", "config_to_json", "scheme_from_name",
           "TimeSeriesRow", "QuenchResult", "run_quench", "fmt_double", "write_checkpoint_uniform",
           "write_checkpoint_finite", "read_checkpoint", "save_mps", "load_mps"]

_SCHEMES = ("svd", "eig", "qr", "qr_cbe")


def scheme_from_name(name: str) -> str:
    """scheme_from_name, proj/src/gates.cpp:30-46."""
    if name not in _SCHEMES:
        raise InputError(f"unknown scheme: {name}")
    return name


@dataclass
class RunConfig:
    """RunConfig, proj/include/qrtebd/run.hpp:16-48 (same defaults)."""

    d: int = 5
    g: float = 2.0
    system_kind: str = "uniform"
    system_size: int = 2
    dt: float = 0.05
    t_max: float = 1.0
    trotter_order: int = 2
    scheme: str = "qr_cbe"
    chi_max: int = 256
    sv_cutoff: float = 1e-14
    target_eps: float = 0.0
    delta_chi_abs: int = 100
    delta_chi_rel: float = 0.1
    out_path: str = ""
    checkpoint_every: int = 0
    fault_skip_renormalize: bool = False
    print_progress: bool = False

    def policy(self) -> TruncationPolicy:
        """run.cpp:80-89 (explicit error stays at its default: on)."""
        return TruncationPolicy(chi_max=self.chi_max, sv_cutoff=self.sv_cutoff, target_eps=self.target_eps,
                                delta_chi_abs=self.delta_chi_abs, delta_chi_rel=self.delta_chi_rel,
                                skip_renormalize=self.fault_skip_renormalize)

    def validate(self) -> None:
        """run.cpp:91-106."""
        if self.d < 2:
            raise InputError("model.d must be >= 2")
        if self.system_kind not in ("uniform", "finite"):
            raise InputError("system.kind must be 'uniform' or 'finite'")
        if self.system_size < 2:
            raise InputError("system.size must be >= 2")
        if self.system_kind == "uniform" and self.system_size % 2 != 0:
            raise InputError("uniform unit cell must have even length")
        if not (self.dt > 0.0):
            raise InputError("evolution.dt must be positive")
        if self.t_max < self.dt:
            raise InputError("evolution.t_max must be >= dt")
        if self.trotter_order not in (1, 2):
            raise InputError("evolution.trotter_order must be 1 or 2")
        if self.chi_max < 1:
            raise InputError("truncation.chi_max must be >= 1")
        if self.sv_cutoff < 0.0:
            raise InputError("truncation.sv_cutoff must be >= 0")
        if self.delta_chi_rel < 0.0:
            raise InputError("truncation.delta_chi_rel must be >= 0")


# --------------------------------------------------------------------- JSON (run.cpp:53-183)
_SECTIONS = {
    "model": {"d": ("d", "uint"), "g": ("g", "float")},
    "system": {"kind": ("system_kind", "str"), "size": ("system_size", "uint")},
    "evolution": {"dt": ("dt", "float"), "t_max": ("t_max", "float"), "trotter_order": ("trotter_order", "int")},
    "truncation": {"scheme": ("scheme", "str"), "chi_max": ("chi_max", "uint"), "sv_cutoff": ("sv_cutoff", "float"),
                   "target_eps": ("target_eps", "float"), "delta_chi_abs": ("delta_chi_abs", "uint"),
                   "delta_chi_rel": ("delta_chi_rel", "float")},
    "output": {"path": ("out_path", "str"), "checkpoint_every": ("checkpoint_every", "uint")},
}


def _typed(key: str, value, kind: str):
    """nlohmann get<T> conversions used by read_field (run.cpp:68-76): numbers
    (and booleans) convert between arithmetic types; strings do not convert."""
    ok = False
    if kind == "str":
        ok = isinstance(value, str)
    elif kind in ("uint", "int"):
        ok = isinstance(value, (int, float))
        if ok:
            value = int(value)
            if kind == "uint" and value < 0:
                value &= (1 << 64) - 1  # size_t wrap, as get<std::size_t> does
    elif kind == "float":
        ok = isinstance(value, (int, float))
        if ok:
            value = float(value)
    if not ok:
        raise InputError(f"config key '{key}' has the wrong type")
    return value


def config_from_json(text: str) -> RunConfig:
    """config_from_json, run.cpp:108-161: strict (unknown keys rejected)."""
    try:
        j = json.loads(text)
    except (ValueError, TypeError) as exc:
        raise InputError(f"config is not valid JSON: {exc}") from None
    if not isinstance(j, dict):
        raise InputError("config section '<root>' must be an object")
    for k in j:
        if k not in _SECTIONS:
            raise InputError(f"unknown config key: <root>.{k}")
    c = RunConfig()
    for sec, fields in _SECTIONS.items():
        if sec not in j:
            continue
        obj = j[sec]
        if not isinstance(obj, dict):
            raise InputError(f"config section '{sec}' must be an object")
        for k in obj:
            if k not in fields:
                raise InputError(f"unknown config key: {sec}.{k}")
        for k, (attr, kind) in fields.items():
            if k in obj:
                setattr(c, attr, _typed(k, obj[k], kind))
    c.scheme = scheme_from_name(c.scheme)
    return c


def config_from_json_file(path: str) -> RunConfig:
    """run.cpp:163-169."""
    try:
        text = Path(path).read_text()
    except OSError:
        raise InputError(f"cannot read config file: {path}") from None
    return config_from_json(text)


def config_to_json(c: RunConfig) -> str:
    """config_to_json, run.cpp:171-183: nlohmann dump(2) layout (keys sorted,
    two-space indent, trailing newline)."""
    j = {
        "model": {"d": c.d, "g": float(c.g)},
        "system": {"kind": c.system_kind, "size": c.system_size},
        "evolution": {"dt": float(c.dt), "t_max": float(c.t_max), "trotter_order": c.trotter_order},
        "truncation": {"scheme": c.scheme, "chi_max": c.chi_max, "sv_cutoff": float(c.sv_cutoff),
                       "target_eps": float(c.target_eps), "delta_chi_abs": c.delta_chi_abs,
                       "delta_chi_rel": float(c.delta_chi_rel)},
        "output": {"path": c.out_path, "checkpoint_every": c.checkpoint_every},
    }
    return json.dumps(j, indent=2, sort_keys=True) + "\n"


def fmt_double(v: float) -> str:
    """fmt_double, run.cpp:33-37 (printf %.17g)."""
    return "%.17g" % v


# --------------------------------------------------------------------- checkpoints (mps.cpp:259-392)
_MAGIC = b"QRTEBDMP"
_VERSION = 1


def _cdata(t: np.ndarray) -> bytes:
    return np.ascontiguousarray(t, dtype="<c16").tobytes()


def write_checkpoint_uniform(path: str, d: int, sites, bonds) -> None:
    """save_mps(UniformMPS), mps.cpp:311-323: header (magic, version, kind 0,
    length, d, center 0, bond dims), then per site Xi[m] and B[m]."""
    L = len(sites)
    out = bytearray(_MAGIC)
    out += struct.pack("<IBIII", _VERSION, 0, L, d, 0)
    for m in range(L):
        out += struct.pack("<Q", bonds[m].shape[0])
    for m in range(L):
        out += _cdata(bonds[m])
        out += _cdata(sites[m])
    _write_bytes(path, bytes(out))


def write_checkpoint_finite(path: str, d: int, sites, center_bond: int, center) -> None:
    """save_mps(FiniteMPS), mps.cpp:325-340: header (kind 1, n+1 bond dims),
    center matrix shape and data, then the site tensors."""
    n = len(sites)
    out = bytearray(_MAGIC)
    out += struct.pack("<IBIII", _VERSION, 1, n, d, center_bond)
    for m in range(n):
        out += struct.pack("<Q", sites[m].shape[1])
    out += struct.pack("<Q", sites[n - 1].shape[2])
    out += struct.pack("<QQ", center.shape[0], center.shape[1])
    out += _cdata(center)
    for m in range(n):
        out += _cdata(sites[m])
    _write_bytes(path, bytes(out))


def _write_bytes(path: str, data: bytes) -> None:
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError:
        raise InputError(f"cannot write checkpoint: {path}") from None


class _Reader:
    def __init__(self, data: bytes):
        self.data, self.pos = data, 0

    def take(self, n: int) -> bytes:
        if self.pos + n > len(self.data):
            raise InputError("truncated checkpoint file")
        b = self.data[self.pos:self.pos + n]
        self.pos += n
        return b

    def pod(self, fmt: str):
        return struct.unpack("<" + fmt, self.take(struct.calcsize("<" + fmt)))[0]

    def tensor(self, shape):
        n = int(np.prod(shape)) if len(shape) else 1
        return np.frombuffer(self.take(16 * n), dtype="<c16").astype(np.complex128).reshape(shape)


def read_checkpoint(path: str) -> dict:
    """load_mps, mps.cpp:342-392, as host arrays: {'kind': 'uniform', 'd',
    'sites', 'bonds'} or {'kind': 'finite', 'd', 'sites', 'center_bond',
    'center'}."""
    try:
        data = Path(path).read_bytes()
    except OSError:
        raise InputError(f"cannot read checkpoint: {path}") from None
    r = _Reader(data)
    if len(data) < 8 or r.take(8) != _MAGIC:
        raise InputError(f"not a checkpoint file: {path}")
    if r.pod("I") != _VERSION:
        raise InputError("unsupported checkpoint version")
    kind = r.pod("B")
    length = r.pod("I")
    d = r.pod("I")
    center = r.pod("I")
    if length == 0 or d == 0:
        raise InputError("corrupt checkpoint header")
    if kind == 0:
        bonds_dim = [r.pod("Q") for _ in range(length)]
        sites, bonds = [], []
        for m in range(length):
            bl, br = bonds_dim[m], bonds_dim[(m + 1) % length]
            bonds.append(r.tensor((bl, bl)))
            sites.append(r.tensor((d, bl, br)))
        return {"kind": "uniform", "d": d, "sites": sites, "bonds": bonds}
    if kind == 1:
        bonds_dim = [r.pod("Q") for _ in range(length + 1)]
        if center > length:
            raise InputError("corrupt checkpoint header")
        rows, cols = r.pod("Q"), r.pod("Q")
        cm = r.tensor((rows, cols))
        sites = [r.tensor((d, bonds_dim[m], bonds_dim[m + 1])) for m in range(length)]
        return {"kind": "finite", "d": d, "sites": sites, "center_bond": center, "center": cm}
    raise InputError("unknown checkpoint kind")


def save_mps(state, path: str) -> None:
    """save_mps for the device states (UniformMPS / DeviceUniformMPS / FiniteMPS)."""
    if isinstance(state, FiniteMPS):
        sites, c, cm = state.to_numpy()
        write_checkpoint_finite(path, state.phys_dim, sites, c, cm)
        return
    if isinstance(state, DeviceUniformMPS):
        sites = [state.view("site", m).numpy() for m in range(state.L)]
        bonds = [state.view("bond", m).numpy() for m in range(state.L)]
        write_checkpoint_uniform(path, state.phys_dim, sites, bonds)
        return
    if isinstance(state, UniformMPS):
        sites, bonds = state.to_numpy()
        write_checkpoint_uniform(path, state.phys_dim, sites, bonds)
        return
    raise InputError("save_mps: unsupported state type")


def load_mps(path: str, ctx: Context = None):
    """load_mps, mps.cpp:342-392: a device UniformMPS or FiniteMPS."""
    ctx = ctx or default_context()
    c = read_checkpoint(path)
    if c["kind"] == "uniform":
        return UniformMPS.from_numpy(ctx, c["d"], c["sites"], c["bonds"])
    return FiniteMPS(c["d"], c["sites"], c["center_bond"], c["center"], ctx)


# --------------------------------------------------------------------- quench (run.cpp:185-326)
@dataclass
class TimeSeriesRow:
    """TimeSeriesRow, proj/include/qrtebd/run.hpp:54-65."""

    t: float = 0.0
    z: List[complex] = field(default_factory=list)
    entropy: List[float] = field(default_factory=list)
    eps: List[float] = field(default_factory=list)
    chi: List[int] = field(default_factory=list)
    bond_ids: List[int] = field(default_factory=list)
    max_eps: float = 0.0
    max_chi: int = 0
    wall_seconds: float = 0.0


@dataclass
class QuenchResult:
    rows: List[TimeSeriesRow] = field(default_factory=list)


class _CsvFiles:
    """open_csv_files / append_row_csv, run.cpp:187-224."""

    def __init__(self, out_path: str, config: RunConfig):
        self.open = False
        if not out_path:
            return
        p = Path(out_path)
        try:
            p.mkdir(parents=True, exist_ok=True)
        except OSError:
            raise InputError(f"cannot create output directory: {out_path}") from None
        try:
            (p / "config.json").write_text(config_to_json(config))
            self.obs = open(p / "observables.csv", "w", newline="")
            self.bonds = open(p / "bonds.csv", "w", newline="")
        except OSError:
            raise InputError(f"cannot write to output directory: {out_path}") from None
        self.obs.write("t,site,z_re,z_im\n")
        self.bonds.write("t,bond,entropy,eps_trunc,chi\n")
        self.open = True

    def append(self, row: TimeSeriesRow) -> None:
        if not self.open:
            return
        t = fmt_double(row.t)
        self.obs.write("".join(f"{t},{s},{fmt_double(z.real)},{fmt_double(z.imag)}\n" for s, z in enumerate(row.z)))
        self.bonds.write("".join(
            f"{t},{b},{fmt_double(e)},{fmt_double(x)},{c}\n"
            for b, e, x, c in zip(row.bond_ids, row.entropy, row.eps, row.chi)))

    def close(self) -> None:
        if self.open:
            self.obs.close()
            self.bonds.close()
            self.open = False


def run_quench(config: RunConfig, ctx: Context = None, use_graph: bool = True) -> QuenchResult:
    """run_quench, proj/src/run.cpp:228-326, on the device.

    Uniform cells evolve as a DeviceUniformMPS (in-place steps, one CUDA graph
    per step once the bond dimensions are stationary); open chains as a
    FiniteMPS with the reference's sequential move_center step
    (gates.cpp:542-578).  Observables (<Z> per site, Schmidt spectra per
    bond) are evaluated every step on the device and, like the reference's,
    stay outside the wall-clock accumulator (run.cpp:263-274)."""
    config.validate()
    if config.scheme not in ("qr", "qr_cbe"):
        raise InputError(f"scheme {config.scheme!r} is not a device scheme (svd/eig are the reference's CPU "
                         "comparators)")
    policy = config.policy()
    d, size = config.d, config.system_size
    z_op = model.clock_operators(d)[0]
    uniform = config.system_kind == "uniform"
    files = _CsvFiles(config.out_path, config)  # run.cpp:236: output errors before any device work
    try:
        ctx = ctx or default_context()
        z_dev = ctx.tensor(z_op)
        if uniform:
            state = DeviceUniformMPS(product_state_uniform(d, size, model.z1_local_vector(d), ctx), ctx)
            schedule = model.trotter_schedule(model.bond_hamiltonian(d, config.g, "bulk"), config.dt,
                                              config.trotter_order)
            schedule = [(p, ctx.tensor(u)) for p, u in schedule]
            bond_ids = list(range(size))
        else:
            state = product_state_finite(d, size, model.z1_local_vector(d), ctx)
            layers = [(p, [ctx.tensor(model.make_gate(model.chain_bond_hamiltonian(d, config.g, b, size), dte))
                           for b in range(size - 1)])
                      for p, dte in model.layer_structure(config.dt, config.trotter_order)]
            bond_ids = list(range(1, size))
        n_steps = int(math.floor(config.t_max / config.dt + 1e-9))
        result = QuenchResult()
        wall = 0.0
        for k in range(1, n_steps + 1):
            t0 = time.perf_counter()
            if uniform:
                reports = state.step(schedule, config.scheme, policy, use_graph=use_graph)
            else:
                _, reports = tebd_step_finite(state, layers, config.scheme, policy, in_place=True)
            wall += time.perf_counter() - t0

            row = TimeSeriesRow(t=k * config.dt, wall_seconds=wall, bond_ids=list(bond_ids))
            if uniform:
                out = (_capi.C.c_double * 2)()
                for s in range(size):
                    bv, sv = state.view("bond", s), state.view("site", s)  # views outlive the call
                    _capi.check(ctx.lib.qt_expectation_local(ctx.h, bv.h, sv.h, z_dev.h, out))
                    row.z.append(complex(out[0], out[1]))
                spectra = {b: schmidt_values_of(state.view("bond", b), ctx) for b in bond_ids}
            else:
                zs, sp = finite_observables(state, z_dev)
                row.z = [complex(v) for v in zs]
                spectra = {b: sp[b] for b in bond_ids}
            for b in bond_ids:
                sv = spectra[b]
                row.entropy.append(entropy_from_schmidt(sv))
                row.chi.append(len(sv))
                row.eps.append(max([0.0] + [r.report.eps_trunc for r in reports if r.bond == b]))
            row.max_eps = max([0.0] + [r.report.eps_trunc for r in reports])
            row.max_chi = max([0] + row.chi)
            files.append(row)
            if config.print_progress:
                print(f"t={row.t:<8.4g} max_chi={row.max_chi:<5d} max_eps={row.max_eps:<10.3e} wall={wall:.1f}s",
                      flush=True)
            result.rows.append(row)
            if files.open and config.checkpoint_every > 0 and k % config.checkpoint_every == 0:
                save_mps(state, os.path.join(config.out_path, "checkpoint_%06d.mps" % k))
        if files.open:
            save_mps(state, os.path.join(config.out_path, "state.mps"))
        return result
    finally:
        files.close()
