"""Host-side checks of the C ABI that need no GPU: the library builds, loads and
exports every function include/mpdp.h declares, and refuses to run without a
CUDA device (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT


def header_functions():
    text = open(os.path.join(ROOT, "include", "mpdp.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    # declared functions; not the function-pointer typedef "mpdp_status (*mpdp_inner_solver)(...)"
    return sorted(set(re.findall(r"\b(mpdp_[a-z0-9_]+)\s*\((?!\s*\*)", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2202_13511_b200 import build, mpdp
    build.build()
    return mpdp.load_library()


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert len(names) >= 11
    for name in names:
        assert hasattr(lib, name), name
    from paper_2202_13511_b200 import mpdp
    assert sorted(mpdp.EXPORTS) == names


def test_abi_version_and_status_strings(lib):
    assert lib.mpdp_abi_version() == 1
    assert lib.mpdp_status_string(0) == b"MPDP_OK"
    assert lib.mpdp_status_string(9) == b"MPDP_ERR_UNSUPPORTED"


def test_no_cpu_fallback_without_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2202_13511_b200 import mpdp
    cfg = mpdp.mpdp_ctx_config(0, 0, 1, None, None, 1 << 20, 0.0, None, 0, 0, 0.0)
    h = C.c_void_p()
    st = lib.mpdp_ctx_create(C.byref(cfg), C.byref(h))
    assert st == mpdp.ERR_CUDA
    assert b"no CUDA device" in lib.mpdp_last_error(None)
    with pytest.raises(mpdp.MPDPError):
        mpdp.Context(device=0)


def test_bad_config_rejected(lib):
    from paper_2202_13511_b200 import mpdp
    h = C.c_void_p()
    cfg = mpdp.mpdp_ctx_config(0, 3, 2, None, None, 0, 0.0, None, 0, 0, 0.0)   # rank >= world
    assert lib.mpdp_ctx_create(C.byref(cfg), C.byref(h)) == mpdp.ERR_INVALID_ARGUMENT
    assert lib.mpdp_ctx_create(None, C.byref(h)) == mpdp.ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("total", [0, 1, 7, 1000, 2 ** 40 + 3])
def test_share_partitions_exactly(lib, world, total):
    from paper_2202_13511_b200 import mpdp
    prev = 0
    seg = (total + world - 1) // world
    for r in range(world):
        lo, hi = mpdp.mpdp_share(total, r, world)
        assert lo == prev and hi >= lo and hi - lo <= seg
        assert lo == min(total, r * seg)          # in-place allgather: segment r at r*seg
        prev = hi
    assert prev == total
