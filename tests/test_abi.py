"""The C-ABI library: it loads, exports every symbol include/dfno.h declares,
and its host-only entry points (validation, sizing, status strings) behave
-- no kernel launches, so this runs without a GPU."""

import ctypes
import re

import pytest
import torch

from paper_2211_12709_b200 import _lib
from paper_2211_12709_b200.partition import block_starts

ROOT = _lib.LIB_PATH.parents[2]


def declared_symbols():
    text = (ROOT / "include" / "dfno.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(dfno_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.dfno_abi_version() == 1
    assert b"sm_100a" in lib.dfno_build_info()


def geom(**kw):
    base = dict(batch=1, c_in=20, c=20, c_out=20, grid=(64, 64, 64, 32), modes=(8, 8, 8, 8),
                retained=(16, 16, 16, 16), nranks=1, rank=0, dtype=_lib.F32, act=_lib.ACT_GELU)
    base.update(kw)
    P = base["nranks"]
    base.setdefault("x_starts", block_starts(base["grid"][0], P))
    base.setdefault("ky_starts", block_starts(base["retained"][1], P))
    return _lib.make_geom(**base)


def test_geometry_validation_codes():
    lib = _lib.load()
    ok = geom()
    assert lib.dfno_geom_validate(ctypes.byref(ok)) == 0
    bad = geom(retained=(16, 16, 16, 15))
    assert lib.dfno_geom_validate(ctypes.byref(bad)) == -4
    bad = geom(dtype=7)
    assert lib.dfno_geom_validate(ctypes.byref(bad)) == -2
    bad = geom(nranks=8, rank=0, x_starts=(0,) * 9, ky_starts=block_starts(16, 8))
    assert lib.dfno_geom_validate(ctypes.byref(bad)) == -4
    g = geom(nranks=8, rank=3)
    assert lib.dfno_geom_validate(ctypes.byref(g)) == 0
    with pytest.raises(Exception):
        _lib.check(-3, "probe")


def test_sizes():
    lib = _lib.load()
    g = geom(nranks=8, rank=7, grid=(262, 118, 64, 86))
    xk, kx, sp, ws = (ctypes.c_int64() for _ in range(4))
    assert lib.dfno_sizes(ctypes.byref(g), ctypes.byref(xk), ctypes.byref(kx), ctypes.byref(sp), ctypes.byref(ws)) == 0
    assert xk.value == 20 * 32 * 16 * 16 * 16       # rank 7 holds 32 of 262 x planes
    assert kx.value == 20 * 262 * 2 * 16 * 16       # and 2 of 16 ky modes
    assert sp.value == 20 * 16 * 2 * 16 * 16
    assert ws.value == 20 * 20 * 16 * 2 * 16 * 16


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU refusal")
def test_no_cpu_fallback():
    import numpy as np

    import paper_2211_12709_b200 as P
    from paper_2211_12709_b200 import ExtensionMissingError

    config = P.FnoConfig(8, 8, 8, 4, 2, 2, 2, P.ModeSpec.of_xyzt(2, 2, 2, 2), 2, "gelu", "real32", 1)
    params = P.init_params(config, 0, device="cpu")
    x = P.DenseTensor(P.DATA_LABELS, np.zeros((1, 2, 8, 8, 8, 4), np.float32))
    comm = P.run_ranks(1, lambda c: c)[0]
    with pytest.raises(ExtensionMissingError):
        P.fno_forward(comm, x, params, config)
