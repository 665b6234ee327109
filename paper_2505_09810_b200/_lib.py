"""ctypes binding of liblmc_b200.so (the C-ABI in include/lmc_b200.h).

The shared library is built in-tree by ``_build.build()`` (or
``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing or no CUDA device is present, every compute call raises
``DeviceError`` instead of silently computing on the host.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import DeviceError, raise_status

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "liblmc_b200.so")


class lmcg_tensor(ctypes.Structure):
    _fields_ = [
        ("data", ctypes.c_void_p),
        ("prev", ctypes.c_void_p),
        ("nbytes", ctypes.c_uint64),
        ("element_type", ctypes.c_int32),
        ("delta", ctypes.c_int32),
    ]


class lmcg_options(ctypes.Structure):
    _fields_ = [
        ("byte_group", ctypes.c_int32),
        ("block_size", ctypes.c_uint32),
        ("segment_count", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("buffer_size", ctypes.c_uint64),
    ]


class lmcg_stream_hint(ctypes.Structure):
    _fields_ = [
        ("orig", ctypes.c_uint64),
        ("segments", ctypes.c_uint32),
        ("block", ctypes.c_uint32),
        ("windows", ctypes.c_uint64),
    ]


# every symbol include/lmc_b200.h declares (tests check the export table)
EXPORTS = [
    "lmcg_create", "lmcg_destroy", "lmcg_last_error", "lmcg_version", "lmcg_validate_options",
    "lmcg_compress_bound", "lmcg_compress_workspace", "lmcg_compress", "lmcg_read_hints",
    "lmcg_decompress", "lmcg_decompress_apply", "lmcg_decompress_result", "lmcg_compress_host", "lmcg_decompress_host", "lmcg_build_codebooks",
    "lmcg_block_info", "lmcg_profile", "lmcg_profile_report", "lmcg_compress_plan_create", "lmcg_compress_plan_run",
    "lmcg_decompress_plan_create", "lmcg_decompress_plan_run", "lmcg_plan_output_bytes", "lmcg_plan_destroy", "lmcg_copy_to_host", "lmcg_fallback_segments", "lmcg_compress_part",
    "lmcg_set_decode_fusion",
]

_lib = None
_lock = threading.Lock()


def load(path: str = SO_PATH):
    """Load the library and declare prototypes (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(path)
        vp, u64, i32, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32, ctypes.c_uint32
        P = ctypes.POINTER
        L.lmcg_create.restype = vp
        L.lmcg_create.argtypes = [ctypes.c_int]
        L.lmcg_destroy.restype = None
        L.lmcg_destroy.argtypes = [vp]
        L.lmcg_last_error.restype = ctypes.c_char_p
        L.lmcg_last_error.argtypes = [vp]
        L.lmcg_version.restype = ctypes.c_int
        L.lmcg_validate_options.restype = ctypes.c_int
        L.lmcg_validate_options.argtypes = [P(lmcg_options), ctypes.c_int, u64]
        L.lmcg_compress_bound.restype = u64
        L.lmcg_compress_bound.argtypes = [P(lmcg_tensor), ctypes.c_int, P(lmcg_options)]
        L.lmcg_compress_workspace.restype = u64
        L.lmcg_compress_workspace.argtypes = [P(lmcg_tensor), ctypes.c_int, P(lmcg_options)]
        L.lmcg_compress.restype = ctypes.c_int
        L.lmcg_compress.argtypes = [vp, P(lmcg_tensor), ctypes.c_int, P(lmcg_options), vp, u64, vp, vp, vp, u64, vp]
        L.lmcg_read_hints.restype = ctypes.c_int
        L.lmcg_read_hints.argtypes = [vp, P(vp), P(u64), ctypes.c_int, P(lmcg_stream_hint), vp]
        L.lmcg_decompress.restype = ctypes.c_int
        L.lmcg_decompress.argtypes = [vp, P(vp), P(u64), ctypes.c_int, P(lmcg_stream_hint), vp, u64, P(u64), vp]
        L.lmcg_decompress_apply.restype = ctypes.c_int
        L.lmcg_decompress_apply.argtypes = [vp, P(vp), P(u64), ctypes.c_int, P(lmcg_stream_hint), P(vp), P(u64), vp, u64,
                                            P(u64), vp]
        L.lmcg_decompress_result.restype = ctypes.c_int
        L.lmcg_decompress_result.argtypes = [vp, ctypes.c_int, P(i32), P(u64), P(i32), P(i32), P(u64)]
        L.lmcg_compress_host.restype = ctypes.c_int
        L.lmcg_compress_host.argtypes = [vp, vp, u64, ctypes.c_int, ctypes.c_int, P(lmcg_options), vp, u64, P(u64)]
        L.lmcg_decompress_host.restype = ctypes.c_int
        L.lmcg_decompress_host.argtypes = [vp, vp, u64, vp, u64, P(u64), P(i32), P(i32)]
        L.lmcg_build_codebooks.restype = ctypes.c_int
        L.lmcg_build_codebooks.argtypes = [vp, vp, ctypes.c_int, vp, vp]
        L.lmcg_block_info.restype = ctypes.c_int64
        L.lmcg_block_info.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_int64]
        L.lmcg_set_decode_fusion.restype = ctypes.c_int
        L.lmcg_set_decode_fusion.argtypes = [vp, ctypes.c_int, u64]
        L.lmcg_profile.restype = ctypes.c_int
        L.lmcg_profile.argtypes = [vp, ctypes.c_int]
        L.lmcg_profile_report.restype = ctypes.c_int64
        L.lmcg_profile_report.argtypes = [vp, ctypes.c_char_p, u64]
        L.lmcg_compress_plan_create.restype = vp
        L.lmcg_compress_plan_create.argtypes = [vp, P(lmcg_tensor), ctypes.c_int, P(lmcg_options)]
        L.lmcg_compress_plan_run.restype = ctypes.c_int
        L.lmcg_compress_plan_run.argtypes = [vp, vp, vp, u64, vp, vp, vp]
        L.lmcg_decompress_plan_create.restype = vp
        L.lmcg_decompress_plan_create.argtypes = [vp, ctypes.c_int, P(lmcg_stream_hint), P(u64)]
        L.lmcg_decompress_plan_run.restype = ctypes.c_int
        L.lmcg_decompress_plan_run.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
        L.lmcg_compress_part.restype = ctypes.c_int
        L.lmcg_compress_part.argtypes = [vp, P(lmcg_tensor), P(lmcg_options), u64, u64, vp, u64, vp, u64, u64, vp, vp]
        L.lmcg_fallback_segments.restype = u64
        L.lmcg_fallback_segments.argtypes = [ctypes.c_int]
        L.lmcg_copy_to_host.restype = ctypes.c_int
        L.lmcg_copy_to_host.argtypes = [vp, vp, u64, vp]
        L.lmcg_plan_output_bytes.restype = u64
        L.lmcg_plan_output_bytes.argtypes = [vp]
        L.lmcg_plan_destroy.restype = None
        L.lmcg_plan_destroy.argtypes = [vp]
        _lib = L
        return L


class Context:
    """One lmcg_ctx bound to a CUDA device (not shared across threads)."""

    def __init__(self, device: int = 0):
        self.lib = load()
        self.device = device
        self.ptr = self.lib.lmcg_create(device)
        if not self.ptr:
            raise DeviceError("lmcg_create failed")

    def set_decode_fusion(self, enable: bool, min_records: int = 16384) -> None:
        """Fused decode + ungroup + CRC (k_decpair) on or off (on: for decodes of at
        least min_records record slots); same bytes and errors either way."""
        self.check(self.lib.lmcg_set_decode_fusion(self.ptr, int(enable), int(min_records)))

    def profile(self, enable: bool) -> None:
        self.lib.lmcg_profile(self.ptr, int(enable))

    def profile_report(self) -> dict:
        """{kernel: (launches, total_ms)} since the last report."""
        buf = ctypes.create_string_buffer(1 << 16)
        self.lib.lmcg_profile_report(self.ptr, buf, len(buf))
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms = line.split()
            out[name] = (int(cnt), float(ms))
        return out

    def error(self) -> str:
        return self.lib.lmcg_last_error(self.ptr).decode(errors="replace")

    def check(self, rc: int) -> None:
        if rc:
            raise_status(rc, self.error())

    def __del__(self):
        try:
            if self.ptr and self.lib is not None:
                self.lib.lmcg_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


_ctx: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the LMC B200 path has no CPU fallback")
    if device is None:
        device = torch.cuda.current_device()
    c = _ctx.get(device)
    if c is None:
        c = _ctx[device] = Context(device)
    return c
