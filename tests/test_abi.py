"""The C ABI library loads on a GPU-less host and exports exactly what
include/gm_b200.h declares (no compute calls here)."""

import ctypes
import os
import re

from paper_2509_16248_b200 import _native as nat

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "gm_b200.h")


def _declared() -> set[str]:
    text = open(HEADER).read()
    return set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(gm_[a-z_0-9]+)\s*\(", text, re.M))


def test_library_loads_and_versions():
    lib = nat.lib()
    assert lib.gm_abi_version() == nat.ABI_VERSION
    assert lib.gm_region_params_bytes() == ctypes.sizeof(nat.Params)
    assert lib.gm_last_error() == b""


def test_header_symbols_exported():
    lib = nat.lib()
    declared = _declared()
    assert {"gm_init", "gm_region_compile", "gm_region_launch", "gm_logring_gather"} <= declared
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/gm_b200.h but not exported"
    assert declared == set(nat.EXPORTED), declared ^ set(nat.EXPORTED)


def test_errors_are_status_codes():
    lib = nat.lib()
    # no device initialised: compute entry points refuse with a message, never crash
    rc = lib.gm_region_compile(b"", b"k", ctypes.byref(ctypes.c_void_p()), None, 0)
    assert rc != 0 and lib.gm_last_error()
    rc = lib.gm_logring_gather(None, None, 0, 0, None, None, None, 0, 0, 0, None)
    assert rc == -1


def test_nvrtc_compiles_skeleton_for_sm100a():
    src = ('#include "gm_region.cuh"\nextern "C" __global__ void k(const __grid_constant__ gm::Params P) '
           '{ float x[8]; gm::load8<GM_DT_BF16>(P.in[0], 0u, 0, 0, 8, x); gm::store8<GM_DT_F32>(P.out[0], 0, 8, x); }\n')
    cubin = nat.compile_cubin(src, (10, 0))
    assert cubin[:4] == b"\x7fELF"


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    """No CPU fallback: without libgm_b200.so the native entry points raise
    NativeError instead of routing the path anywhere else."""
    import pytest

    monkeypatch.setattr(nat, "_lib", None)
    monkeypatch.setattr(nat, "LIB_PATH", str(tmp_path / "libgm_b200.so"))
    with pytest.raises(nat.NativeError, match="no fallback"):
        nat.lib()


def test_record_api_declared_and_mirrored():
    """the record-level log-ring entry points and the
    gm_record layout the drain callback receives."""
    declared = _declared()
    assert {"gm_logring_begin_step", "gm_logring_capture", "gm_logring_end_step", "gm_logring_drain",
            "gm_gemm_run", "gm_select_copy", "gm_stream_capture_id", "gm_status_page"} <= declared
    # gm_record: u32, i32 x3, u64, 3 pointers, const void*, size_t
    assert ctypes.sizeof(nat.GmRecord) == 4 * 4 + 8 + 3 * 8 + 8 + 8
    text = open(HEADER).read()
    assert "#define GM_LOGRING_SLOTS 64" in text and nat.LOGRING_SLOTS == 64
    lib = nat.lib()
    # without a ring or an open step the record API refuses with a status code
    assert lib.gm_logring_begin_step(None) == -1
    assert lib.gm_logring_drain(None, nat.RECORD_CB(lambda r, u: 0), None) == -1
