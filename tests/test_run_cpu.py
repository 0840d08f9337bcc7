"""Quench-driver host logic and formats on CPU: the config JSON contract
(proj/tests/test_run.cc ConfigJson / ConfigValidate), the checkpoint container
(proj/src/mps.cpp:259-392) and the oracle's reference-exact finite chain
(move_center + sequential tebd_step, proj/src/gates.cpp:542-578) pinned
against the reference's own expectations (proj/tests/test_run.cc,
proj/tests/test_tebd.cc)."""
import json
import struct

import numpy as np
import pytest

from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import run
from paper_2212_09782_b200._capi import InputError


# ----------------------------------------------------------------- config (test_run.cc:27-99)
def test_config_parses_nested_document():
    text = """{
      "model": {"d": 5, "g": 2.0},
      "system": {"kind": "uniform", "size": 2},
      "evolution": {"dt": 0.05, "t_max": 4.0, "trotter_order": 2},
      "truncation": {"scheme": "qr_cbe", "chi_max": 256, "sv_cutoff": 1e-14,
                     "delta_chi_abs": 100, "delta_chi_rel": 0.1},
      "output": {"path": "runs/demo", "checkpoint_every": 10}
    }"""
    c = run.config_from_json(text)
    assert (c.d, c.g, c.system_kind, c.dt, c.t_max) == (5, 2.0, "uniform", 0.05, 4.0)
    assert (c.scheme, c.chi_max, c.sv_cutoff, c.delta_chi_abs, c.delta_chi_rel) == ("qr_cbe", 256, 1e-14, 100, 0.1)
    assert (c.out_path, c.checkpoint_every) == ("runs/demo", 10)


@pytest.mark.parametrize("text", ['{"mode": {}}', '{"model": {"d": 5, "beta": 1.0}}',
                                  '{"truncation": {"chimax": 8}}'])
def test_config_rejects_unknown_keys(text):
    with pytest.raises(InputError):
        run.config_from_json(text)


@pytest.mark.parametrize("text", ['{"model": {"d": "five"}}', "not json", '{"system": {"kind": 3}}',
                                  '{"model": []}', '[1, 2]'])
def test_config_rejects_wrong_types_and_bad_json(text):
    with pytest.raises(InputError):
        run.config_from_json(text)


def test_config_round_trip_and_layout():
    c = run.RunConfig(d=3, scheme="qr", chi_max=64, out_path="x")
    text = run.config_to_json(c)
    back = run.config_from_json(text)
    assert (back.d, back.scheme, back.chi_max, back.out_path) == (3, "qr", 64, "x")
    assert back == c
    # nlohmann dump(2): sorted keys, two-space indent, trailing newline
    assert text.endswith("}\n")
    assert text.splitlines()[1] == '  "evolution": {'
    assert list(json.loads(text)) == ["evolution", "model", "output", "system", "truncation"]


def test_config_validate_catches_bad_values():
    for kw in [dict(dt=0.0), dict(t_max=0.01), dict(system_kind="uniform", system_size=3),
               dict(system_kind="ring"), dict(d=1), dict(trotter_order=3), dict(chi_max=0),
               dict(sv_cutoff=-1.0), dict(delta_chi_rel=-0.1), dict(system_size=1)]:
        with pytest.raises(InputError):
            run.RunConfig(**kw).validate()
    run.RunConfig().validate()
    run.RunConfig(system_kind="finite", system_size=3).validate()
    with pytest.raises(InputError):
        run.scheme_from_name("qrx")


def test_fmt_double_is_printf_17g():
    # byte-identical to the C library's snprintf("%.17g"), run.cpp:33-37
    import ctypes
    libc = ctypes.CDLL(None)
    buf = ctypes.create_string_buffer(64)
    vals = [0.1, 1.0, -0.0, 1e-300, 2.0 / 3.0, 123456789.123, 5e-324, 1e22, -7.25e-15, float("inf")]
    vals += list(np.random.default_rng(0).standard_normal(200) * 10.0 ** np.arange(-100, 100))
    for v in vals:
        libc.snprintf(buf, 64, b"%.17g", ctypes.c_double(v))
        assert run.fmt_double(v) == buf.value.decode(), v
    assert run.fmt_double(0.1) == "0.10000000000000001"


def test_unwritable_output_path_rejected_before_device_work():
    # test_run.cc:172-181: fails with InputError (here before any context exists)
    c = run.RunConfig(d=2, dt=0.1, t_max=0.1, chi_max=4, scheme="qr", out_path="/dev/null/nested")
    with pytest.raises(InputError):
        run.run_quench(c)


def test_cpu_schemes_rejected_by_the_device_driver():
    with pytest.raises(InputError):
        run.run_quench(run.RunConfig(d=2, dt=0.1, t_max=0.1, scheme="svd"))


# ----------------------------------------------------------------- checkpoints (mps.cpp:259-392)
def _rand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def test_checkpoint_uniform_round_trip_and_layout(tmp_path):
    rng = np.random.default_rng(3)
    d, chis = 3, [4, 2]
    sites = [_rand(rng, d, chis[m], chis[(m + 1) % 2]) for m in range(2)]
    bonds = [_rand(rng, chis[m], chis[m]) for m in range(2)]
    p = tmp_path / "u.mps"
    run.write_checkpoint_uniform(str(p), d, sites, bonds)
    raw = p.read_bytes()
    # header: magic, u32 version, u8 kind, u32 length, u32 d, u32 center, u64 bond dims
    assert raw[:8] == b"QRTEBDMP"
    assert struct.unpack_from("<IBIII", raw, 8) == (1, 0, 2, d, 0)
    assert struct.unpack_from("<QQ", raw, 25) == (4, 2)
    body = np.frombuffer(raw[41:], dtype="<c16")
    expect = np.concatenate([bonds[0].ravel(), sites[0].ravel(), bonds[1].ravel(), sites[1].ravel()])
    assert np.array_equal(body, expect)
    c = run.read_checkpoint(str(p))
    assert c["kind"] == "uniform" and c["d"] == d
    for a, b in zip(c["sites"] + c["bonds"], sites + bonds):
        assert np.array_equal(a, b)


def test_checkpoint_finite_round_trip_rectangular_center(tmp_path):
    rng = np.random.default_rng(4)
    d, dims = 2, [1, 2, 4, 2, 1]
    sites = [_rand(rng, d, dims[m], dims[m + 1]) for m in range(4)]
    center = _rand(rng, 3, 4)  # rectangular after a rank-revealing move (mps.cpp:328-330)
    p = tmp_path / "f.mps"
    run.write_checkpoint_finite(str(p), d, sites, 2, center)
    raw = p.read_bytes()
    assert struct.unpack_from("<IBIII", raw, 8) == (1, 1, 4, d, 2)
    assert struct.unpack_from("<5Q", raw, 25) == tuple(dims)
    assert struct.unpack_from("<QQ", raw, 65) == (3, 4)
    c = run.read_checkpoint(str(p))
    assert c["kind"] == "finite" and c["center_bond"] == 2
    assert np.array_equal(c["center"], center)
    for a, b in zip(c["sites"], sites):
        assert np.array_equal(a, b)


def test_checkpoint_rejects_bad_files(tmp_path):
    bad = tmp_path / "bad.mps"
    bad.write_bytes(b"NOTMAGIC" + b"\0" * 32)
    with pytest.raises(InputError):
        run.read_checkpoint(str(bad))
    good = tmp_path / "g.mps"
    run.write_checkpoint_uniform(str(good), 2, [np.ones((2, 1, 1))] * 2, [np.eye(1)] * 2)
    raw = good.read_bytes()
    (tmp_path / "trunc.mps").write_bytes(raw[:-8])
    with pytest.raises(InputError):
        run.read_checkpoint(str(tmp_path / "trunc.mps"))
    (tmp_path / "ver.mps").write_bytes(raw[:8] + struct.pack("<I", 2) + raw[12:])
    with pytest.raises(InputError):
        run.read_checkpoint(str(tmp_path / "ver.mps"))
    with pytest.raises(InputError):
        run.read_checkpoint(str(tmp_path / "missing.mps"))


# ----------------------------------------------------------------- oracle: reference finite semantics
def _random_finite(rng, d, n, chi_cap, center):
    dims = [min(d ** m, d ** (n - m), chi_cap) for m in range(n + 1)]
    sites = [_rand(rng, d, dims[m], dims[m + 1]) for m in range(n)]
    return ref.FiniteMPS(d, sites, center, np.eye(dims[center], dtype=complex)), dims


def _statevector(mps: ref.FiniteMPS):
    """Dense state of a FiniteMPS (center matrix inserted on its bond)."""
    psi = np.ones((1, 1), dtype=complex)  # (phys, right bond)
    for m, b in enumerate(mps.site_tensors):
        if m == mps.center_bond:
            psi = psi @ mps.center_matrix
        psi = np.einsum("pa,iab->pib", psi, b).reshape(-1, b.shape[2])
    if mps.center_bond == len(mps.site_tensors):
        psi = psi @ mps.center_matrix
    return psi.ravel()


def test_oracle_move_center_preserves_state_and_gauge():
    rng = np.random.default_rng(7)
    mps, _ = _random_finite(rng, 3, 5, 6, 0)
    psi = _statevector(mps)
    for c in (5, 2, 0, 3):
        moved = ref.move_center(mps, c)
        assert moved.center_bond == c
        assert np.allclose(_statevector(moved), psi, atol=1e-12 * np.linalg.norm(psi))
        for s in range(5):
            if s < c:
                assert ref.left_defect(moved.site_tensors[s]) < 1e-12
            elif s > c or c == 0:
                assert ref.right_defect(moved.site_tensors[s]) < 1e-12
        mps = moved


def test_oracle_finite_quench_rows_cover_interior_bonds():
    # test_run.cc:183-199 (scheme svd there; the QR schemes here)
    pol = ref.TruncationPolicy(chi_max=16)
    rows = ref.run_quench_rows(2, 2.0, "finite", 4, 0.05, 0.2, 2, "qr", pol)
    assert len(rows) == 4
    assert len(rows[0]["z"]) == 4 and rows[0]["bond_ids"] == [1, 2, 3]


def test_oracle_quench_svd_and_qr_rows_agree():
    # test_run.cc:139-170: uniform d=3, chi 64, qr vs svd rows to 1e-8
    pol = ref.TruncationPolicy(chi_max=64)
    rs = ref.run_quench_rows(3, 2.0, "uniform", 2, 0.05, 0.4, 2, "svd", pol)
    rq = ref.run_quench_rows(3, 2.0, "uniform", 2, 0.05, 0.4, 2, "qr", pol)
    t_prev = 0.0
    for a, b in zip(rs, rq):
        assert a["max_eps"] <= 1e-10 and b["max_eps"] <= 1e-10
        assert a["t"] > t_prev and a["max_chi"] <= 64
        t_prev = a["t"]
        for za, zb in zip(a["z"], b["z"]):
            assert abs(za.real - zb.real) < 1e-8


def test_oracle_finite_reference_path_matches_statevector_and_hastings():
    # test_tebd.cc:205-240 style: untruncated, the sequential reference path, the
    # Hastings form and exact evolution agree (Appendix B: 1e-10)
    d, n, g, dt = 2, 6, 1.5, 0.05
    pol = ref.TruncationPolicy(chi_max=64, sv_cutoff=1e-14)
    layers = ref.finite_layers(d, g, n, dt, 2)
    v = np.zeros(d, dtype=complex)
    v[0] = 1
    fs = ref.product_state_finite(d, n, v)
    hs = [v.reshape(d, 1, 1).copy() for _ in range(n)]
    hb = [np.eye(1, dtype=complex) for _ in range(n)]
    z = ref.clock_operators(d)[0]
    for _ in range(3):
        fs, _ = ref.tebd_step_finite(fs, layers, "qr", pol)
        hs, hb, _ = ref.tebd_step_finite_hastings(hs, hb, layers, "qr", pol)
    ok, mx, _ = ref.check_isometric_finite(fs, 1e-10)
    assert ok, mx
    for s in range(n):
        zf = ref.expectation_local_finite(fs, z, s)
        zh = ref.expectation_from_weight(ref.left_weight(hb[s]), hs[s], z)
        assert abs(zf - zh) < 1e-10
    # exact: 2nd-order Trotter on the state vector with the same gates
    psi = np.zeros(d ** n, dtype=complex)
    psi[0] = 1
    psi = psi.reshape([d] * n)
    for _ in range(3):
        for parity, gates in layers:
            for m in range(0 if parity == "even" else 1, n - 1, 2):
                psi = np.moveaxis(np.tensordot(gates[m], psi, axes=([2, 3], [m, m + 1])), [0, 1], [m, m + 1])
    sv = _statevector(fs).reshape([d] * n)
    assert abs(abs(np.vdot(sv.ravel(), psi.ravel())) - 1.0) < 1e-10
