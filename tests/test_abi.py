"""The C-ABI library loads on a CPU-only host and exports every symbol the header declares.

No compute calls here (no GPU); only argument-validation paths that return
before touching the device, to pin the status -> exception mapping.
"""

import ctypes
import os
import re

import pytest

from paper_2411_17116_b200 import _lib
from paper_2411_17116_b200.errors import ConfigError, DomainError, ShapeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "star_attn.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(star_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("star_phase1_fwd", "star_phase2_partial", "star_merge", "star_rope",
                 "star_kv_write", "star_prng_fill", "star_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_lib.SIGNATURES)
    assert lib.star_version() == 1


def test_status_maps_to_reference_exceptions():
    lib = _lib.load()
    rc = lib.star_merge(None, None, 0, 1, 4, None, 0, None, None)
    assert rc == _lib.STAR_EDOMAIN
    with pytest.raises(DomainError, match="zero partials"):
        _lib.check(rc)
    seg = (ctypes.c_int64 * 2)(0, 4)
    rc = lib.star_phase1_fwd(None, None, None, 0, 1, seg, 4, 3, 8, 32, 32, None, 0, 32, None, 0, None)
    assert rc == _lib.STAR_ESHAPE  # hq not a multiple of hkv
    with pytest.raises(ShapeError):
        _lib.check(rc)
    rc = lib.star_phase1_fwd(None, None, None, 0, 99, seg, 4, 4, 8, 32, 32, None, 0, 32, None, 0, None)
    with pytest.raises(ConfigError):
        _lib.check(rc)
    rc = lib.star_rope(None, None, 0, 4, 1, 7, 7, 7, None, 10000.0, None)
    with pytest.raises(ConfigError, match="even"):
        _lib.check(rc)
    rc = lib.star_attention_dense(None, None, None, 0, 4, 3, 0, 1, 1, 1, 8, 8, 8, None, 8, None, None)
    with pytest.raises(ShapeError, match="extend past"):
        _lib.check(rc)
    rc = lib.star_phase2_partial(None, 0, 1, 2, 4, 4, 64, None, None, 0, 1, None, 1, 64, None, 10, 1,
                                 None, None, 0, None, None)
    with pytest.raises(ShapeError, match="own_tail"):
        _lib.check(rc)


def test_ops_refuse_cpu_tensors():
    import torch

    from paper_2411_17116_b200 import ops
    from paper_2411_17116_b200.errors import DeviceError

    x = torch.zeros(4, 1, 8)
    with pytest.raises(DeviceError, match="no CPU fallback"):
        ops.rope(x, torch.arange(4))
