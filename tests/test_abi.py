"""CPU-side checks of the C-ABI library: it loads, exports every symbol
include/amun.h declares, and its host validation rejects bad arguments with
AMUN_EINVAL before touching the GPU (no compute call is made here)."""
import ctypes
import os
import re

import pytest

import __graft_entry__ as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    G.build()
    from paper_1805_09863_b200 import _lib
    return _lib.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "amun.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(amun_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    from paper_1805_09863_b200 import _lib
    declared = header_functions()
    assert declared, "no declarations parsed"
    assert sorted(_lib.EXPORTS) == declared
    for name in declared:
        assert hasattr(lib, name), name


def test_sass_is_sm100a_tcgen05():
    """The built library contains tcgen05 MMA, TMEM loads and TMA (not HMMA)."""
    import subprocess
    G.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", G.LIB], capture_output=True,
                         text=True, check=True).stdout
    assert "UTCHMMA" in out and "LDTM" in out and "UTMALDG" in out
    assert "arch = sm_100a" in out


def test_version_and_strings(lib):
    assert lib.amun_abi_version() == 1
    assert lib.amun_status_string(1) == b"AMUN_EINVAL"


def _create(lib, **kw):
    a = dict(H=64, V_local=1000, v_offset=0, V_total=1000, dtype=1, k_max=4, max_rows=64,
             max_sentences=8, device=0)
    a.update(kw)
    h = ctypes.c_void_p()
    st = lib.amun_ol_create(ctypes.byref(h), a["H"], a["V_local"], a["v_offset"], a["V_total"],
                            a["dtype"], a["k_max"], a["max_rows"], a["max_sentences"], a["device"])
    return st, h


@pytest.mark.parametrize("kw", [
    dict(k_max=0), dict(k_max=17), dict(H=12), dict(H=0), dict(V_local=0), dict(dtype=7),
    dict(v_offset=5), dict(V_total=999), dict(max_rows=-1), dict(dtype=0, H=6),
])
def test_create_rejects_bad_arguments(lib, kw):
    st, h = _create(lib, **kw)
    assert st == 1, (kw, lib.amun_last_error())
    assert not h.value
    assert lib.amun_last_error()


def test_create_null_plan_pointer(lib):
    assert lib.amun_ol_create(None, 64, 10, 0, 10, 1, 2, 4, 4, 0) == 1


def test_compact_rejects_bad_arguments(lib):
    from paper_1805_09863_b200._lib import amun_column
    cols = (amun_column * 17)()
    buf = ctypes.c_void_p(16)
    assert lib.amun_compact(cols, 17, buf, 4, buf, 1, buf, buf, buf, None, None) == 1
    cols[0] = amun_column(16, 4096, 6)                  # row_bytes not a multiple of 4
    assert lib.amun_compact(cols, 1, buf, 4, buf, 1, buf, buf, buf, None, None) == 1
    cols[0] = amun_column(16, 32, 16)                   # overlapping src/dst
    assert lib.amun_compact(cols, 1, buf, 4, buf, 1, buf, buf, buf, None, None) == 1
    assert b"overlap" in lib.amun_last_error()
    assert lib.amun_compact(cols, 1, buf, -1, buf, 1, buf, buf, buf, None, None) == 1


def test_null_plan_calls(lib):
    assert lib.amun_ol_workspace_bytes(None) == 0
    assert lib.amun_ol_partial_stride(None) == 0
    assert lib.amun_ol_scores(None, None, None, None, 1, None, None) == 1
    assert lib.amun_argmax(None, None, None, None, 1, None, None, None, None) == 1
    assert lib.amun_merge_partials(None, None, 1, None, None, 0, 0, None, 1, None, None, None) == 1


def test_mxfp4_host_checks(lib):
    """MXFP4 scale-atom sizes (amun.h layout: [H/128][ceil(R/128)][512 B])
    and the quantiser's / entry points' host validation (no launch)."""
    assert lib.amun_mxfp4_sf_bytes(300, 256) == 2 * 3 * 512
    assert lib.amun_mxfp4_sf_bytes(128, 1024) == 8 * 1 * 512
    assert lib.amun_mxfp4_sf_bytes(0, 256) == 0
    assert lib.amun_mxfp4_sf_bytes(10, 192) == 0        # H % 128 != 0
    assert lib.amun_mxfp4_sf_bytes(-1, 256) == 0
    buf = ctypes.c_void_p(16)
    assert lib.amun_quantize_mxfp4(buf, 7, 4, 256, buf, buf, None) == 1          # bad src dtype
    assert lib.amun_quantize_mxfp4(buf, 0, 4, 192, buf, buf, None) == 1          # H % 128
    assert b"128" in lib.amun_last_error()
    assert lib.amun_quantize_mxfp4(None, 0, 4, 256, buf, buf, None) == 1         # NULL src
    assert lib.amun_quantize_mxfp4(buf, 0, 0, 256, None, None, None) == 0        # R = 0: no-op
    assert lib.amun_argmax_mxfp4(None, None, None, None, None, None, 1, None, None, None, None) == 1
    assert lib.amun_output_layer_mxfp4(None, None, None, None, None, None, None, None, 1, 1, None,
                                       1, None, None, None, None) == 1
