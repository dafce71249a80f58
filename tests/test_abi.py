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
    rc = lib.star_phase1_fwd(None, None, None, 0, -1, seg, 4, 4, 8, 32, 32, None, 0, 32, None, 0, None)
    with pytest.raises(ConfigError):  # a negative segment count (any positive count is chunked)
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


def _box_bytes(world, cap_rows, cap_groups, d):
    """Python restatement of the exchange box layout (csrc/exchange.cuh): a 256-byte header,
    then [2 parities][world][part] 8-byte {value, epoch} words, part = rows*(d+1) rounded
    up to even."""
    part = (cap_rows * (d + 1) + 1) // 2 * 2
    return 256 + 2 * world * part * 8


@pytest.mark.parametrize("world,rows,groups,d", [(1, 32, 8, 128), (8, 32, 8, 128), (2, 7, 3, 64),
                                                 (8, 1024, 256, 128)])
def test_exchange_box_layout(world, rows, groups, d):
    lib = _lib.load()
    assert lib.star_exchange_box_bytes(world, rows, groups, d) == _box_bytes(world, rows, groups, d)
    assert lib.star_exchange_box_bytes(9, rows, groups, d) == _lib.STAR_ESHAPE


def test_exchange_argument_checks():
    """Validation paths return before any device work (fake non-NULL pointers)."""
    lib = _lib.load()
    boxes = (ctypes.c_void_p * 2)(0x1000, 0x2000)
    fake = ctypes.c_void_p(0x3000)
    # the call needs more rows than the box holds
    rc = lib.star_exchange_push(fake, fake, 1, 2, 4, 2, 64, boxes, 2, 4, 2, 0, None)
    with pytest.raises(ShapeError, match="box holds"):
        _lib.check(rc)
    # rank outside the world
    rc = lib.star_exchange_push(fake, fake, 1, 1, 4, 2, 64, boxes, 2, 4, 2, 2, None)
    with pytest.raises(ConfigError, match="rank"):
        _lib.check(rc)
    # a missing peer box
    boxes_hole = (ctypes.c_void_p * 2)(0x1000, None)
    rc = lib.star_exchange_push(fake, fake, 1, 1, 4, 2, 64, boxes_hole, 2, 4, 2, 0, None)
    with pytest.raises(ShapeError, match="box of rank 1"):
        _lib.check(rc)
    # more peers than one node
    boxes9 = (ctypes.c_void_p * 9)(*([0x1000] * 9))
    rc = lib.star_exchange_push(fake, fake, 1, 1, 4, 2, 64, boxes9, 9, 4, 2, 0, None)
    assert rc == _lib.STAR_ENOTSUP
    rc = lib.star_exchange_merge(fake, 9, 4, 2, 1, 1, 4, 2, 128, fake, 0, None, None)
    assert rc == _lib.STAR_ENOTSUP
    rc = lib.star_exchange_merge(fake, 2, 4, 2, 2, 1, 4, 2, 128, fake, 0, None, None)
    with pytest.raises(ShapeError, match="box holds"):
        _lib.check(rc)
