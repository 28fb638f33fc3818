"""ctypes binding of libgm_b200.so — the C ABI in include/gm_b200.h.

This is the exact binding a maintainer of the reference (pure Python,
pkg/pyproject.toml:10 `dependencies = []`) would add; INTEGRATION.md shows it.
The product path fails loudly when the library is missing or stale: there is
no CPU fallback anywhere behind these calls.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgm_b200.so")
ABI_VERSION = 1

# element type codes (include/gm_b200.h)
GM_F32, GM_BF16, GM_F16, GM_F64, GM_BOOL, GM_I32, GM_I64, GM_U8 = range(8)

MAX_IN = 8
MAX_OUT = 8
MAX_RED = 16
MAX_HS = 32
MAX_DIMS = 6
MAX_PIECES = 16
THREADS = 512
VEC = 8
LAUNCH_PDL = 1   # GM_LAUNCH_PDL

# kernels this library launched (incremented per launching call; a CUDA graph
# replays what was counted while it was captured) — bench.py's gpu_launches
launch_count = 0


def count_launches(k: int = 1) -> None:
    global launch_count
    launch_count += k


class NativeError(RuntimeError):
    """A libgm_b200 call returned a non-zero status."""


LOGRING_SLOTS = 64              # GM_LOGRING_SLOTS
LOGRING_NO_TEMPLATE = 0xFFFFFFFF


class GmRecord(ctypes.Structure):
    """Mirror of gm_record (include/gm_b200.h)."""

    _fields_ = [
        ("record_id", ctypes.c_uint32),
        ("dtype", ctypes.c_int32),
        ("ndim", ctypes.c_int32),
        ("pad", ctypes.c_int32),
        ("step", ctypes.c_uint64),
        ("shape", ctypes.POINTER(ctypes.c_int64)),
        ("counts", ctypes.POINTER(ctypes.c_int64)),
        ("heads", ctypes.POINTER(ctypes.c_int64)),
        ("data", ctypes.c_void_p),
        ("bytes", ctypes.c_size_t),
    ]


RECORD_CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(GmRecord), ctypes.c_void_p)   # gm_record_cb


class InDesc(ctypes.Structure):
    _fields_ = [
        ("ptr", ctypes.c_int64),
        ("smem_off", ctypes.c_int64),
        ("ndim", ctypes.c_int64),
        ("size", ctypes.c_int64 * MAX_DIMS),
        ("stride", ctypes.c_int64 * MAX_DIMS),
    ]


class OutDesc(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_int64)]


class Params(ctypes.Structure):
    """Mirror of gm::Params (csrc/gm_region.cuh); every field is 8 bytes."""

    _fields_ = [
        ("n", ctypes.c_int64),
        ("nvec", ctypes.c_int64),
        ("vpc", ctypes.c_int64),
        ("piece_vecs", ctypes.c_int64),
        ("partials", ctypes.c_int64),
        ("barrier", ctypes.c_int64),
        ("status", ctypes.c_int64),
        ("scal_out", ctypes.c_int64),
        ("hs", ctypes.c_double * MAX_HS),
        ("inp", InDesc * MAX_IN),
        ("out", OutDesc * MAX_OUT),
    ]


_lock = threading.Lock()
_lib = None

# (name, restype, argtypes) for every symbol the header declares
_SIGNATURES = [
    ("gm_abi_version", ctypes.c_int, []),
    ("gm_last_error", ctypes.c_char_p, []),
    ("gm_init", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("gm_region_compile_cubin", ctypes.c_int,
     [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
      ctypes.POINTER(ctypes.c_size_t), ctypes.c_char_p, ctypes.c_size_t]),
    ("gm_free", None, [ctypes.c_void_p]),
    ("gm_region_compile", ctypes.c_int,
     [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p, ctypes.c_size_t]),
    ("gm_region_load", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    ("gm_region_set_smem", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    ("gm_region_occupancy", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    ("gm_region_launch", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int,
      ctypes.c_void_p]),
    ("gm_region_launch_ex", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int,
      ctypes.c_void_p, ctypes.c_int]),
    ("gm_region_release", ctypes.c_int, [ctypes.c_void_p]),
    ("gm_stream_capture_id", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]),
    ("gm_status_page", ctypes.c_int,
     [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]),
    ("gm_unique_sum16_scratch_bytes", ctypes.c_size_t, []),
    ("gm_unique_sum32_scratch_bytes", ctypes.c_size_t, [ctypes.c_int64]),
    ("gm_unique_sum32_hash_scratch_bytes", ctypes.c_size_t, [ctypes.c_int64]),
    ("gm_unique_sum32_hash", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    ("gm_unique_sum32", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    ("gm_unique_sum16", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("gm_region_params_bytes", ctypes.c_size_t, []),
    ("gm_branch_select_scratch_bytes", ctypes.c_size_t, []),
    ("gm_branch_select_f32", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_double,
      ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
      ctypes.c_void_p]),
    ("gm_gemm_open", ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p)]),
    ("gm_gemm_close", ctypes.c_int, [ctypes.c_void_p]),
    ("gm_gemm_version", ctypes.c_size_t, []),
    ("gm_gemm_run", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
      ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
      ctypes.c_size_t, ctypes.c_void_p]),
    ("gm_gemm_run_batched", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
      ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
      ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    ("gm_copy_strided", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
      ctypes.c_int, ctypes.c_void_p]),
    ("gm_select_copy", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
      ctypes.c_void_p]),
    ("gm_logring_open", ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    ("gm_logring_close", ctypes.c_int, [ctypes.c_void_p]),
    ("gm_logring_host_ptr", ctypes.c_void_p, [ctypes.c_void_p]),
    ("gm_logring_bytes", ctypes.c_size_t, [ctypes.c_void_p]),
    ("gm_logring_step_ptr", ctypes.c_void_p, [ctypes.c_void_p]),
    ("gm_logring_gather", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64), ctypes.c_uint64, ctypes.c_uint64,
      ctypes.c_uint64, ctypes.c_void_p]),
    ("gm_logring_commit", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    ("gm_logring_committed", ctypes.c_uint64, [ctypes.c_void_p]),
    ("gm_logring_begin_step", ctypes.c_int, [ctypes.c_void_p]),
    ("gm_logring_capture", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64), ctypes.c_int,
      ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p]),
    ("gm_logring_end_step", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32)]),
    ("gm_logring_drain", ctypes.c_int, [ctypes.c_void_p, RECORD_CB, ctypes.c_void_p]),
]

EXPORTED = [name for name, _, _ in _SIGNATURES]


def lib():
    """The loaded library (raises if absent or ABI-mismatched)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() "
                "(make -C paper_2509_16248_b200/csrc); there is no fallback"
            )
        handle = ctypes.CDLL(LIB_PATH)
        for name, restype, argtypes in _SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = restype
            fn.argtypes = argtypes
        if handle.gm_abi_version() != ABI_VERSION:
            raise NativeError("libgm_b200.so ABI version mismatch; rebuild it")
        if handle.gm_region_params_bytes() != ctypes.sizeof(Params):
            raise NativeError(
                f"gm::Params is {handle.gm_region_params_bytes()} bytes in the library, "
                f"{ctypes.sizeof(Params)} in _native.Params; rebuild"
            )
        _lib = handle
        return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().gm_last_error().decode(errors="replace")
        raise NativeError(f"{what or 'libgm_b200'} failed ({rc}): {msg}")


_init_device = {}


def init(device: int) -> tuple[int, int]:
    """gm_init for `device`; returns (num_sms, smem_optin_bytes)."""
    if device in _init_device:
        return _init_device[device]
    sms, smem = ctypes.c_int(0), ctypes.c_int(0)
    check(lib().gm_init(device, ctypes.byref(sms), ctypes.byref(smem)), "gm_init")
    _init_device[device] = (sms.value, smem.value)
    return _init_device[device]


def compile_cubin(src: str, cc: tuple[int, int] = (10, 0)) -> bytes:
    """NVRTC-compile a region source to a cubin (no GPU needed)."""
    out = ctypes.c_void_p()
    n = ctypes.c_size_t(0)
    log = ctypes.create_string_buffer(1 << 16)
    check(
        lib().gm_region_compile_cubin(src.encode(), cc[0], cc[1], ctypes.byref(out), ctypes.byref(n), log,
                                      len(log)),
        "gm_region_compile_cubin",
    )
    try:
        return ctypes.string_at(out, n.value)
    finally:
        lib().gm_free(out)


def capture_id(stream: int) -> int:
    """CUDA-graph capture id of `stream` (0 when not capturing)."""
    v = ctypes.c_uint64(0)
    check(lib().gm_stream_capture_id(ctypes.c_void_p(stream), ctypes.byref(v)), "gm_stream_capture_id")
    return int(v.value)


STATUS_WORDS = 1 << 16
_status = None


def status_page():
    """(host int array, device base address) of the process-wide mapped
    status page (gm_status_page)."""
    global _status
    if _status is None:
        h, d = ctypes.c_void_p(), ctypes.c_void_p()
        check(lib().gm_status_page(STATUS_WORDS, ctypes.byref(h), ctypes.byref(d)), "gm_status_page")
        _status = ((ctypes.c_int * STATUS_WORDS).from_address(h.value), d.value)
    return _status


class CompiledRegion:
    """Owner of one gm_region handle (a loaded region kernel): NVRTC-compiled
    from `src`, or loaded from an ahead-of-time `cubin`."""

    def __init__(self, src: str, kernel: str, cubin: bytes | None = None):
        h = ctypes.c_void_p()
        if cubin is not None:
            check(lib().gm_region_load(cubin, len(cubin), kernel.encode(), ctypes.byref(h)),
                  f"gm_region_load({kernel})")
            self.log = "aot"
        else:
            log = ctypes.create_string_buffer(1 << 16)
            check(lib().gm_region_compile(src.encode(), kernel.encode(), ctypes.byref(h), log, len(log)),
                  f"gm_region_compile({kernel})")
            self.log = log.value.decode(errors="replace")
        self.handle = h
        self.kernel = kernel
        self.from_cache = cubin is not None
        self._smem_set = 0

    def occupancy(self, threads: int, smem: int) -> int:
        if smem > self._smem_set:
            check(lib().gm_region_set_smem(self.handle, smem), "gm_region_set_smem")
            self._smem_set = smem
        n = ctypes.c_int(0)
        check(lib().gm_region_occupancy(self.handle, threads, smem, ctypes.byref(n)), "gm_region_occupancy")
        return n.value

    def launch(self, params: Params, grid: int, threads: int, smem: int, stream: int, pdl: bool = False) -> None:
        count_launches()
        check(
            lib().gm_region_launch_ex(self.handle, ctypes.byref(params), ctypes.sizeof(params), grid, threads, smem,
                                      ctypes.c_void_p(stream), LAUNCH_PDL if pdl else 0),
            f"gm_region_launch_ex({self.kernel})",
        )

    def __del__(self):
        try:
            if self.handle:
                lib().gm_region_release(self.handle)
        except Exception:
            pass
