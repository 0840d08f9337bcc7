"""CPU checks of the C-ABI boundary: the shared library loads, exports every
symbol include/qrtebd_c.h declares, host-side logic (policy defaults,
expanded_dim) matches the reference, and compute entry points fail loudly
(no CPU fallback) when no B200 is present."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT, gpu_available
from oracle import qrtebd_oracle as ref
from paper_2212_09782_b200 import _capi

HEADER = os.path.join(ROOT, "include", "qrtebd_c.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(qt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _capi.load()
    names = declared_symbols()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), f"missing export {n}"
        assert n in _capi.SIGNATURES, f"ctypes binding lacks {n}"


def test_exports_are_plain_c_symbols():
    # extern "C": no C++ mangling on the boundary
    out = os.popen(f"nm -D --defined-only {_capi.LIB_PATH}").read()
    for n in declared_symbols():
        assert re.search(rf"\bT {n}$", out, re.M), n


def test_policy_defaults_match_reference():
    p = _capi.default_policy()
    r = ref.TruncationPolicy()
    assert p.chi_max == r.chi_max and p.sv_cutoff == r.sv_cutoff and p.target_eps == r.target_eps
    assert p.delta_chi_abs == r.delta_chi_abs and p.delta_chi_rel == r.delta_chi_rel
    assert p.chi_max_expansion == r.chi_max_expansion and p.qr_sweeps == r.qr_sweeps
    assert bool(p.compute_explicit_error) == r.compute_explicit_error
    assert bool(p.skip_renormalize) == r.skip_renormalize


@pytest.mark.parametrize("chi,d,dabs,drel,cap", [(256, 5, 100, 0.1, 0), (1, 5, 100, 0.1, 0),
                                                  (2000, 5, 100, 0.1, 0), (256, 5, 100, 0.1, 300),
                                                  (1024, 10, 100, 0.1, 0), (4096, 5, 0, 0.1, 0), (7, 3, 0, 0.0, 0)])
def test_expanded_dim_matches_reference(chi, d, dabs, drel, cap):
    lib = _capi.load()
    p = _capi.default_policy(delta_chi_abs=dabs, delta_chi_rel=drel, chi_max_expansion=cap)
    r = ref.TruncationPolicy(delta_chi_abs=dabs, delta_chi_rel=drel, chi_max_expansion=cap)
    assert lib.qt_expanded_dim(C.byref(p), chi, d) == r.expanded_dim(chi, d)


def test_struct_layouts():
    assert C.sizeof(_capi.qt_policy) == 64
    assert C.sizeof(_capi.qt_report) == 48
    assert C.sizeof(_capi.qt_bond_report) == 56


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    with pytest.raises(_capi.CudaError):
        _capi.Context(0)
    assert "no CUDA device" in _capi.load().qt_last_error().decode()


def test_null_arguments_are_input_errors():
    lib = _capi.load()
    assert lib.qt_ctx_create(0, None, None) in (_capi.QT_ERR_INPUT, _capi.QT_ERR_CUDA)
    assert lib.qt_tensor_free(None) == _capi.QT_OK


@pytest.mark.parametrize("n,world", [(2, 1), (8, 2), (9, 2), (256, 8), (10, 3), (6, 4), (255, 8)])
def test_chain_partition_matches_host_logic(n, world):
    """qt_chain_partition (the C-ABI sharded chain, csrc/chain.cu) cuts the
    chain exactly as the host-side ShardedChain does (finite.partition):
    contiguous, even-aligned blocks; an odd last site joins the last block."""
    from paper_2212_09782_b200.chain import partition
    from paper_2212_09782_b200.finite import partition as host_partition
    blocks = host_partition(n, world)
    for r in range(world):
        b, e = partition(n, world, r)
        if r < len(blocks):
            assert (b, e) == blocks[r]
        else:
            assert b == e  # more ranks than site pairs: empty block
