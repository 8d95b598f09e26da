"""C ABI boundary checks that need no GPU: the library loads, exports every
function include/certkv_b200.h declares, and the ctypes mirrors match the C
struct layouts."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "certkv_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:ckv_status|int32_t|void|const char\*)\s+(ckv_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_20868_b200 import build, _lib
    build.build()
    return _lib.load()


def test_header_symbols_exported(lib):
    from paper_2605_20868_b200 import _lib
    names = _declared()
    assert len(names) >= 12
    assert sorted(names) == sorted(_lib.exported_symbols())
    for n in names:
        assert hasattr(lib, n), n


def test_struct_layouts(lib):
    """The ctypes mirrors have the sizes the C compiler gave the structs."""
    from paper_2605_20868_b200 import _lib
    out = (ctypes.c_int32 * 5)()
    lib.ckv_struct_sizes(out)
    mirrors = (_lib.CkvCache, _lib.CkvPolicy, _lib.CkvCert, _lib.CkvStep, _lib.CkvScratch)
    assert list(out) == [ctypes.sizeof(m) for m in mirrors]
    assert ctypes.sizeof(_lib.CkvCert) == 8 * 8 + 6 * 4


def test_plan_host_only(lib):
    from paper_2605_20868_b200 import _lib
    from paper_2605_20868_b200.policy import PolicyConfig
    pol = PolicyConfig(exploration_rate=0.0).to_c()
    st = _lib.CkvStep()
    assert lib.ckv_plan(256, 8192, 4, ctypes.byref(pol), ctypes.byref(st)) == 0
    assert st.blocks_per_split == 64 and st.n_splits == 128
    assert st.kcap >= 2 * 128 + 1 and st.wcap == st.kcap + 8192
    bad = PolicyConfig(exploration_rate=0.0, k_max=600).to_c()
    assert lib.ckv_plan(1, 64, 4, ctypes.byref(bad), ctypes.byref(st)) == 1
    assert lib.ckv_plan(1, 64, 5, ctypes.byref(pol), ctypes.byref(st)) == 1
    assert lib.ckv_lru_words(8192, 8192) == 4 + 3 * 8192
    assert lib.ckv_lru_words(8192, 2048) > 4 + 3 * 8192


def test_invalid_args_rejected_without_gpu(lib):
    from paper_2605_20868_b200 import _lib
    c = _lib.CkvCache()  # all-null cache
    assert lib.ckv_append(ctypes.byref(c), None, None, 1, None) == 1
    assert lib.ckv_reset(ctypes.byref(c), None) == 1


def test_sm100a_code_in_library(lib):
    import subprocess
    from paper_2605_20868_b200 import _lib
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
