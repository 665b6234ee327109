"""The LMC codestream on B200: drop-in ``lmc_compress`` / ``lmc_decompress``.

Public surface mirrors the reference ``lmc.stream`` (pkg/src/lmc/stream.py):
same names, same keyword options, same return types, same exceptions, and
byte-identical ``LMC1`` streams.  Every byte of compute runs in the CUDA
kernels of liblmc_b200.so (csrc/); this module only moves buffers, parses the
28-byte header (host logic, stream.py:114-142) and maps status codes onto the
reference's exception classes.

Batched, device-resident entry points (``Codec.compress`` / ``Codec.decompress``)
take CUDA tensors and keep the streams in HBM; the reference-shaped functions
wrap them with host <-> device copies.
"""
from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .errors import (AlignmentError, ConfigError, CorruptStreamError, DeviceError, LmcError,
                     UnsupportedFormatError, raise_status)
from .types import DeltaBuffer, ElementType, TensorBuffer, element_code, is_delta

MAGIC = b"LMC1"
VERSION = 1
FLAG_BYTE_GROUPED = 0x01
FLAG_DELTA = 0x02
DEFAULT_BLOCK_SIZE = 64 * 1024          # entropy.py:22
MIN_BLOCK_SIZE = 4 * 1024
MAX_BLOCK_SIZE = 1024 * 1024
DEFAULT_BUFFER_SIZE = 128 * 1024 * 1024  # stream.py:66
MODE_HUFFMAN, MODE_RLE, MODE_STORED = 0, 1, 2
_HEADER = struct.Struct("<4sBBBBQIII")
HEADER_SIZE = _HEADER.size  # 28
CODEBOOK_WIRE_SIZE = 128

_WIDTH = {0: 1, 1: 2, 2: 2, 3: 4}


# ---------------------------------------------------------------- header
@dataclass(frozen=True)
class CodeStreamHeader:
    """stream.py:83-111."""

    flags: int
    element_type: ElementType
    original_length: int
    block_size: int
    segment_count: int
    crc32: int

    @property
    def byte_grouped(self) -> bool:
        return bool(self.flags & FLAG_BYTE_GROUPED)

    @property
    def delta_applied(self) -> bool:
        return bool(self.flags & FLAG_DELTA)

    def pack(self) -> bytes:
        return _HEADER.pack(MAGIC, VERSION, self.flags, self.element_type.code, 0, self.original_length,
                            self.block_size, self.segment_count, self.crc32)


def validate_block_size(block_size: int) -> int:
    """entropy.py:27-37."""
    if block_size < MIN_BLOCK_SIZE or block_size > MAX_BLOCK_SIZE or block_size & (block_size - 1):
        raise ConfigError(f"block size must be a power of two in [{MIN_BLOCK_SIZE}, {MAX_BLOCK_SIZE}], got {block_size}")
    return block_size


def parse_header(stream: bytes) -> CodeStreamHeader:
    """stream.py:114-142 (host-side header parse; the device repeats it)."""
    if len(stream) < HEADER_SIZE:
        raise UnsupportedFormatError("stream shorter than a header")
    magic, version, flags, et_code, reserved, orig_len, block_size, seg_count, crc = _HEADER.unpack_from(stream)
    if magic != MAGIC:
        raise UnsupportedFormatError(f"bad magic {magic!r}")
    if version != VERSION:
        raise UnsupportedFormatError(f"unsupported version {version}")
    if flags & ~(FLAG_BYTE_GROUPED | FLAG_DELTA):
        raise CorruptStreamError(f"unknown flag bits 0x{flags:02x}")
    if reserved != 0:
        raise CorruptStreamError("reserved header byte must be zero")
    try:
        et = ElementType.from_code(et_code)
    except ValueError as exc:
        raise CorruptStreamError(str(exc)) from exc
    try:
        validate_block_size(block_size)
    except ConfigError as exc:
        raise CorruptStreamError(str(exc)) from exc
    if seg_count < 1:
        raise CorruptStreamError("segment count must be >= 1")
    if orig_len % et.width != 0:
        raise CorruptStreamError(f"original length {orig_len} is not {et.name}-aligned")
    return CodeStreamHeader(flags, et, orig_len, block_size, seg_count, crc)


def segment_bounds(window_length: int, block_size: int, segment_count: int) -> list[tuple[int, int]]:
    """stream.py:271-284 (host helper; the device computes the same edges)."""
    nblocks = (window_length + block_size - 1) // block_size
    edges = [min(window_length, (i * nblocks // segment_count) * block_size) for i in range(segment_count)]
    edges.append(window_length)
    return list(zip(edges[:-1], edges[1:]))


def _validate_options(width: int, block_size: int, segment_count: int, buffer_size: int) -> None:
    """stream.py:287-301."""
    validate_block_size(block_size)
    if segment_count < 1:
        raise ConfigError(f"segment count must be >= 1, got {segment_count}")
    if buffer_size < block_size:
        raise ConfigError(f"buffer size {buffer_size} must be >= block size {block_size}")
    if buffer_size % width != 0:
        raise ConfigError(f"buffer size {buffer_size} must be a multiple of the element width {width}")


def compression_ratio(stream: bytes, original_length: int) -> float:
    if original_length == 0:
        return 1.0
    return len(stream) / original_length


# ------------------------------------------------------------ device codec
_TORCH_ET = None


def _torch_et(dtype) -> int:
    global _TORCH_ET
    import torch

    if _TORCH_ET is None:
        _TORCH_ET = {torch.bfloat16: 1, torch.float16: 2, torch.float32: 3, torch.uint8: 0, torch.int8: 0}
    if dtype not in _TORCH_ET:
        raise ConfigError(f"no LMC element type for torch dtype {dtype}")
    return _TORCH_ET[dtype]


def _bytes_view(t):
    import torch

    if not t.is_cuda:
        raise DeviceError("Codec inputs must be CUDA tensors")
    t = t.detach()   # parameters: bytes only, no autograd
    if not t.is_contiguous():
        t = t.contiguous()
    return t.view(torch.uint8).reshape(-1) if t.numel() else torch.empty(0, dtype=torch.uint8, device=t.device)


class CompressedBatch:
    """Streams packed back to back in one CUDA byte tensor."""

    def __init__(self, data, offsets, lengths, hints=None):
        self.data = data          # torch.uint8 [capacity], device
        self.offsets = offsets    # torch.int64 [n], device
        self.lengths = lengths    # torch.int64 [n], device
        self.hints = hints        # per stream (orig, segments, block, windows): exact decode hints
        self._host = None

    def host_layout(self) -> tuple[list[int], list[int]]:
        if self._host is None:
            import torch

            both = torch.stack([self.offsets, self.lengths]).cpu().tolist()
            self._host = (both[0], both[1])
        return self._host

    def __len__(self) -> int:
        return int(self.offsets.numel())

    def stream(self, i: int):
        off, ln = self.host_layout()
        return self.data[off[i]: off[i] + ln[i]]

    def total_bytes(self) -> int:
        off, ln = self.host_layout()
        return (off[-1] + ln[-1]) if off else 0

    def to_bytes(self) -> list[bytes]:
        off, ln = self.host_layout()
        total = self.total_bytes()
        flat = self.data[:total].cpu().numpy().tobytes() if total else b""
        return [flat[o: o + n] for o, n in zip(off, ln)]


class DecompressedBatch:
    """Decoded payloads packed at 16-byte aligned offsets of one CUDA byte tensor.

    ``status`` holds per-stream C-ABI codes (0 = OK; 1/2/3 = the reference's
    UnsupportedFormat / CorruptStream / Integrity errors).  Plan runs leave
    it on the device until first read (reading synchronises)."""

    def __init__(self, data, offsets, lengths, element_types, flags, status, status_dev=None):
        self.data = data
        self.offsets = offsets
        self.lengths = lengths
        self.element_types = element_types
        self.flags = flags
        self._status = status
        self._status_dev = status_dev

    @property
    def status(self) -> list[int]:
        if self._status is None:
            self._status = self._status_dev.cpu().tolist()
        return self._status

    def __len__(self) -> int:
        return len(self.offsets)

    def payload(self, i: int):
        return self.data[self.offsets[i]: self.offsets[i] + self.lengths[i]]

    def raise_for_status(self) -> None:
        for i, s in enumerate(self.status):
            if s:
                raise_status(s, f"stream {i}: " + {1: "unsupported format", 2: "corrupt stream",
                                                   3: "payload CRC mismatch",
                                                   11: "payload length differs from prev"}.get(s, f"status {s}"))


class Codec:
    """Batched device-resident LMC codec on one CUDA device.

    ``compress`` takes CUDA tensors (any of bf16/fp16/fp32/uint8, or explicit
    element type codes) and returns a CompressedBatch whose streams are
    byte-identical to ``lmc.lmc_compress`` of the same bytes.  ``prev`` turns
    on the fused XOR delta (delta.py:29-47): the stream then encodes
    ``prev ^ tensor`` with FLAG_DELTA, exactly like compressing a DeltaBuffer.
    """

    def __init__(self, device: int | None = None):
        import torch

        self.ctx = _lib.context(device)
        self.device = torch.device("cuda", self.ctx.device)
        self._ws = None

    # -- compress
    def compress(self, tensors: Sequence, *, element_types: Sequence[int] | None = None, prev: Sequence | None = None,
                 delta: Sequence[bool] | bool | None = None, byte_group: bool = True,
                 block_size: int = DEFAULT_BLOCK_SIZE, segment_count: int = 1,
                 buffer_size: int = DEFAULT_BUFFER_SIZE, out=None, stream=None) -> CompressedBatch:
        import torch

        n = len(tensors)
        views, ets = [], []
        for i, t in enumerate(tensors):
            et = element_types[i] if element_types is not None else _torch_et(t.dtype)
            ets.append(int(et))
            views.append(_bytes_view(t))
        pviews = [None] * n
        if prev is not None:
            for i, p in enumerate(prev):
                if p is not None:
                    pv = _bytes_view(p)
                    if pv.numel() != views[i].numel():
                        from .errors import ShapeMismatchError
                        raise ShapeMismatchError(f"length mismatch: {pv.numel()} vs {views[i].numel()}")
                    pviews[i] = pv
        if isinstance(delta, bool) or delta is None:
            dflags = [bool(delta)] * n
        else:
            dflags = [bool(d) for d in delta]
        for et in ets:
            _validate_options(_WIDTH[et], block_size, segment_count, buffer_size)
        arr = (_lib.lmcg_tensor * max(n, 1))()
        for i in range(n):
            arr[i].data = views[i].data_ptr() if views[i].numel() else 0
            arr[i].prev = pviews[i].data_ptr() if pviews[i] is not None and pviews[i].numel() else 0
            arr[i].nbytes = views[i].numel()
            arr[i].element_type = ets[i]
            arr[i].delta = int(dflags[i] or pviews[i] is not None)
            if views[i].numel() % _WIDTH[ets[i]]:
                raise AlignmentError(f"buffer of {views[i].numel()} bytes is not a multiple of width {_WIDTH[ets[i]]}")
        opts = _lib.lmcg_options(int(bool(byte_group)), block_size, segment_count, 0, buffer_size)
        L = self.ctx.lib
        bound = int(L.lmcg_compress_bound(arr, n, ctypes.byref(opts)))
        wsb = int(L.lmcg_compress_workspace(arr, n, ctypes.byref(opts)))
        if self._ws is None or self._ws.numel() < wsb:
            self._ws = torch.empty(max(wsb, 1 << 20), dtype=torch.uint8, device=self.device)
        if out is None or out.numel() < bound:
            out = torch.empty(max(bound, 16), dtype=torch.uint8, device=self.device)
        meta = torch.empty(2 * max(n, 1), dtype=torch.int64, device=self.device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = L.lmcg_compress(self.ctx.ptr, arr, n, ctypes.byref(opts), out.data_ptr(), out.numel(),
                             meta.data_ptr(), meta.data_ptr() + 8 * max(n, 1), self._ws.data_ptr(),
                             self._ws.numel(), ctypes.c_void_p(s.cuda_stream))
        self.ctx.check(rc)
        # keep inputs alive until the work is done
        hints = [(int(v.numel()), segment_count, block_size, (int(v.numel()) + buffer_size - 1) // buffer_size)
                 for v in views]
        batch = CompressedBatch(out, meta[:n], meta[max(n, 1): max(n, 1) + n], hints)
        batch._keep = (views, pviews)
        return batch

    def compress_part(self, tensor, blk_begin: int, blk_end: int, crc_begin: int, crc_end: int, *,
                      element_type: int | None = None, prev=None, delta: bool = False, byte_group: bool = True,
                      block_size: int = DEFAULT_BLOCK_SIZE, segment_count: int = 1,
                      buffer_size: int = DEFAULT_BUFFER_SIZE, stream=None):
        """One part of ``tensor``'s stream for multi-GPU assembly
        (lmcg_compress_part): the records of blocks [blk_begin, blk_end) back
        to back, their sizes, and the raw CRC-32 of payload bytes
        [crc_begin, crc_end).  Returns device tensors (records, sizes, crc);
        ``shard.assemble_stream`` joins the parts of all ranks."""
        import torch

        et = int(element_type if element_type is not None else _torch_et(tensor.dtype))
        v = _bytes_view(tensor)
        pv = _bytes_view(prev) if prev is not None else None
        if pv is not None and pv.numel() != v.numel():
            from .errors import ShapeMismatchError
            raise ShapeMismatchError(f"length mismatch: {pv.numel()} vs {v.numel()}")
        _validate_options(_WIDTH[et], block_size, segment_count, buffer_size)
        if v.numel() % _WIDTH[et]:
            raise AlignmentError(f"buffer of {v.numel()} bytes is not a multiple of width {_WIDTH[et]}")
        t = _lib.lmcg_tensor()
        t.data = v.data_ptr() if v.numel() else 0
        t.prev = pv.data_ptr() if pv is not None and pv.numel() else 0
        t.nbytes = v.numel()
        t.element_type = et
        t.delta = int(bool(delta) or pv is not None)
        opts = _lib.lmcg_options(int(bool(byte_group)), block_size, segment_count, 0, buffer_size)
        nblk = blk_end - blk_begin
        cap = 5 * max(nblk, 0) + min(v.numel(), max(nblk, 0) * block_size) + 16
        out = torch.empty(max(cap, 16), dtype=torch.uint8, device=self.device)
        sizes = torch.empty(max(nblk, 1), dtype=torch.int32, device=self.device)
        crc = torch.zeros(1, dtype=torch.int64, device=self.device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = self.ctx.lib.lmcg_compress_part(self.ctx.ptr, ctypes.byref(t), ctypes.byref(opts), blk_begin, blk_end,
                                             out.data_ptr(), out.numel(), sizes.data_ptr(), crc_begin, crc_end,
                                             crc.data_ptr(), ctypes.c_void_p(s.cuda_stream))
        self.ctx.check(rc)
        out._keep = (v, pv)
        return out, sizes[:max(nblk, 0)], crc

    def compress_plan(self, tensors, **kw) -> CompressPlan:
        """A CompressPlan over these tensors (see CompressPlan)."""
        return CompressPlan(self, tensors, **kw)

    def block_info(self) -> dict:
        """Per-block (mode, bits, record size, wire codebook) of the last compress."""
        L = self.ctx.lib
        nb = int(L.lmcg_block_info(self.ctx.ptr, None, None, None, None, None, 0))
        modes = np.zeros(nb, np.int32)
        bits = np.zeros(nb, np.uint32)
        sizes = np.zeros(nb, np.uint32)
        wire = np.zeros((nb, 128), np.uint8)
        pm = np.zeros(nb, np.uint32)
        if nb:
            L.lmcg_block_info(self.ctx.ptr, modes.ctypes.data, bits.ctypes.data, sizes.ctypes.data,
                              wire.ctypes.data, pm.ctypes.data, nb)
        lengths = np.zeros((nb, 256), np.uint8)
        lengths[:, 0::2] = wire & 0x0F
        lengths[:, 1::2] = wire >> 4
        return dict(modes=modes, bits=bits, sizes=sizes, wire=wire, lengths=lengths, pm=pm)

    # -- decompress
    def read_hints(self, views, stream=None) -> list[tuple]:
        """Exact (orig, segments, block, windows) of device streams, validated on the device (synchronises)."""
        import torch

        n = len(views)
        ptrs = (ctypes.c_void_p * max(n, 1))(*[v.data_ptr() for v in views])
        lens = (ctypes.c_uint64 * max(n, 1))(*[v.numel() for v in views])
        hs = (_lib.lmcg_stream_hint * max(n, 1))()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.ctx.check(self.ctx.lib.lmcg_read_hints(self.ctx.ptr, ptrs, lens, n, hs, ctypes.c_void_p(s.cuda_stream)))
        return [(hs[i].orig, hs[i].segments, hs[i].block, hs[i].windows) for i in range(n)]

    def decompress(self, streams, *, hints=None, out=None, out_offsets=None, prev=None,
                   stream=None) -> DecompressedBatch:
        """Decode device streams (a CompressedBatch or a list of CUDA byte tensors).

        ``hints`` (per stream: original length, segment count, block size,
        window count) size the device work areas; a CompressedBatch carries
        exact ones, otherwise they are read from the stream headers.  Wrong
        hints only cost a retry.  ``out`` + ``out_offsets`` place stream i's
        payload at ``out[out_offsets[i]:]`` (default: packed at 16-byte
        aligned offsets in a fresh buffer).  ``prev`` (per stream a device
        tensor or None) fuses ``xor_apply`` (delta.py:50-52) into the decode:
        the output is ``prev ^ payload``; ``prev`` may be the output location
        itself (in-place restore, lmcg_decompress_apply).
        """
        import torch

        if isinstance(streams, CompressedBatch):
            if hints is None:
                hints = streams.hints
            off, ln = streams.host_layout()
            streams = [streams.data[o: o + n] for o, n in zip(off, ln)]
        views = []
        for t in streams:
            v = _bytes_view(t)
            if v.numel() == 0:
                v = torch.zeros(16, dtype=torch.uint8, device=self.device)[:0]
            views.append(v)
        n = len(views)
        if hints is None:
            hints = self.read_hints(views, stream=stream)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        ptrs = (ctypes.c_void_p * max(n, 1))(*[v.data_ptr() if v.numel() else 0 for v in views])
        lens = (ctypes.c_uint64 * max(n, 1))(*[v.numel() for v in views])
        pptr = plen = None
        if prev is not None:
            if len(prev) != n:
                raise ValueError("prev needs one entry (tensor or None) per stream")
            pviews = [None if p is None else _bytes_view(p) for p in prev]
            pptr = (ctypes.c_void_p * max(n, 1))(*[0 if p is None else (p.data_ptr() or 0) for p in pviews])
            plen = (ctypes.c_uint64 * max(n, 1))(*[0 if p is None else p.numel() for p in pviews])
            # an empty prev is still a prev (length 0): point it somewhere non-NULL
            for i, p in enumerate(pviews):
                if p is not None and not pptr[i]:
                    pptr[i] = views[i].data_ptr() or 16
        if out_offsets is not None:
            if out is None or len(out_offsets) != n:
                raise ValueError("out_offsets needs out and one offset per stream")
            out = _bytes_view(out)
        for _ in range(3):
            hs = (_lib.lmcg_stream_hint * max(n, 1))()
            offs, pos = [], 0
            for i, h in enumerate(hints):
                hs[i].orig, hs[i].segments, hs[i].block, hs[i].windows = (int(x) for x in h)
                offs.append(pos)
                pos += (int(h[0]) + 15) & ~15
            if out_offsets is not None:
                offs = [int(x) for x in out_offsets]
            elif out is None or out.numel() < pos:
                out = torch.empty(max(pos, 16), dtype=torch.uint8, device=self.device)
            hoff = (ctypes.c_uint64 * max(n, 1))(*offs)
            if pptr is None:
                rc = self.ctx.lib.lmcg_decompress(self.ctx.ptr, ptrs, lens, n, hs, out.data_ptr(), out.numel(), hoff,
                                                  ctypes.c_void_p(s.cuda_stream))
            else:
                rc = self.ctx.lib.lmcg_decompress_apply(self.ctx.ptr, ptrs, lens, n, hs, pptr, plen, out.data_ptr(),
                                                        out.numel(), hoff, ctypes.c_void_p(s.cuda_stream))
            self.ctx.check(rc)
            st = (ctypes.c_int32 * max(n, 1))()
            orig = (ctypes.c_uint64 * max(n, 1))()
            ets = (ctypes.c_int32 * max(n, 1))()
            fl = (ctypes.c_int32 * max(n, 1))()
            nw = (ctypes.c_uint64 * max(n, 1))()
            self.ctx.check(self.ctx.lib.lmcg_decompress_result(self.ctx.ptr, n, st, orig, ets, fl, nw))
            status = list(st)[:n]
            retry = [i for i in range(n) if status[i] == 10 or (status[i] == 8 and out_offsets is None)]
            if not retry:
                return DecompressedBatch(out, offs, list(orig)[:n], list(ets)[:n], list(fl)[:n], status)
            hints = [((int(orig[i]), int(hints[i][1]), int(hints[i][2]), int(nw[i])) if i in retry else hints[i])
                     for i in range(n)]
        raise LmcError("decompress hints did not converge")


class CompressPlan:
    """Repeated compression of the same device tensors (a model's parameters).

    Validation, layout and descriptor upload happen once; ``run()`` only
    launches the kernels -- optionally replaying a captured CUDA graph -- and
    returns streams byte-identical to ``lmc_compress`` of the tensors' current
    contents.  The returned batch aliases the plan's output buffer and stays
    valid until the next ``run()``.
    """

    def __init__(self, codec: "Codec", tensors, *, element_types=None, prev=None, delta=None, byte_group=True,
                 block_size=DEFAULT_BLOCK_SIZE, segment_count=1, buffer_size=DEFAULT_BUFFER_SIZE, graph=False):
        import torch

        self.codec = codec
        L = codec.ctx.lib
        n = len(tensors)
        self.n = n
        views = [_bytes_view(t) for t in tensors]
        ets = [int(element_types[i]) if element_types is not None else _torch_et(t.dtype) for i, t in enumerate(tensors)]
        pviews = [None] * n if prev is None else [(_bytes_view(p) if p is not None else None) for p in prev]
        dflags = [bool(delta)] * n if (delta is None or isinstance(delta, bool)) else [bool(d) for d in delta]
        for et in ets:
            _validate_options(_WIDTH[et], block_size, segment_count, buffer_size)
        arr = (_lib.lmcg_tensor * max(n, 1))()
        bounds = []
        opts = _lib.lmcg_options(int(bool(byte_group)), block_size, segment_count, 0, buffer_size)
        for i in range(n):
            if views[i].numel() % _WIDTH[ets[i]]:
                raise AlignmentError(f"buffer of {views[i].numel()} bytes is not a multiple of width {_WIDTH[ets[i]]}")
            if pviews[i] is not None and pviews[i].numel() != views[i].numel():
                from .errors import ShapeMismatchError
                raise ShapeMismatchError(f"length mismatch: {pviews[i].numel()} vs {views[i].numel()}")
            arr[i].data = views[i].data_ptr() if views[i].numel() else 0
            arr[i].prev = pviews[i].data_ptr() if pviews[i] is not None and pviews[i].numel() else 0
            arr[i].nbytes = views[i].numel()
            arr[i].element_type = ets[i]
            arr[i].delta = int(dflags[i] or pviews[i] is not None)
            bounds.append(int(L.lmcg_compress_bound(ctypes.byref(arr[i]), 1, ctypes.byref(opts))))
        self._keep = (views, pviews, arr)
        self.ptr = L.lmcg_compress_plan_create(codec.ctx.ptr, arr, n, ctypes.byref(opts))
        if not self.ptr:
            raise_status(4 if "option" in codec.ctx.error() else 7, codec.ctx.error())
        self.bound = int(L.lmcg_plan_output_bytes(self.ptr))
        self.stream_bounds = bounds
        self.hints = [(int(v.numel()), segment_count, block_size, (int(v.numel()) + buffer_size - 1) // buffer_size)
                      for v in views]
        self.out = torch.empty(max(self.bound, 16), dtype=torch.uint8, device=codec.device)
        self.meta = torch.zeros(2 * max(n, 1), dtype=torch.int64, device=codec.device)
        self.graph = None
        if graph:
            self.graph = _capture(lambda st: self._launch(st))

    def _launch(self, st) -> None:
        L = self.codec.ctx.lib
        rc = L.lmcg_compress_plan_run(self.codec.ctx.ptr, self.ptr, self.out.data_ptr(), self.out.numel(),
                                      self.meta.data_ptr(), self.meta.data_ptr() + 8 * max(self.n, 1),
                                      ctypes.c_void_p(st.cuda_stream))
        self.codec.ctx.check(rc)

    def run(self, stream=None) -> CompressedBatch:
        import torch

        if self.graph is not None:
            self.graph.replay()
        else:
            self._launch(stream if stream is not None else torch.cuda.current_stream(self.codec.device))
        n = self.n
        return CompressedBatch(self.out, self.meta[:n], self.meta[max(n, 1): max(n, 1) + n], self.hints)

    def layout_to_host(self, host_meta, stream=None) -> None:
        """Copy the last run's stream offsets and lengths (2n int64) into the
        pinned host tensor ``host_meta``, ordered on ``stream`` but written by
        the SMs (lmcg_copy_to_host), so it does not queue behind bulk copies."""
        import torch

        st = stream if stream is not None else torch.cuda.current_stream(self.codec.device)
        n = max(self.n, 1)
        if host_meta.device.type != "cpu" or not host_meta.is_pinned() or host_meta.numel() * host_meta.element_size() < 16 * n:
            raise ValueError("host_meta must be a pinned host tensor of at least 2n int64")
        rc = self.codec.ctx.lib.lmcg_copy_to_host(ctypes.c_void_p(host_meta.data_ptr()), ctypes.c_void_p(self.meta.data_ptr()),
                                                  16 * n, ctypes.c_void_p(st.cuda_stream))
        self.codec.ctx.check(rc)

    def decompress_plan(self, graph=False) -> "DecompressPlan":
        """A plan decoding this plan's output (exact structure hints)."""
        return DecompressPlan(self.codec, self.hints, self.stream_bounds, graph=graph, source=self)

    def __del__(self):
        try:
            if getattr(self, "ptr", None):
                self.codec.ctx.lib.lmcg_plan_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


class DecompressPlan:
    """Repeated decompression of streams with a known structure (see CompressPlan)."""

    def __init__(self, codec: "Codec", hints, len_bounds, *, graph=False, source: CompressPlan | None = None):
        import torch

        self.codec = codec
        L = codec.ctx.lib
        n = len(hints)
        self.n = n
        hs = (_lib.lmcg_stream_hint * max(n, 1))()
        for i, h in enumerate(hints):
            hs[i].orig, hs[i].segments, hs[i].block, hs[i].windows = (int(x) for x in h)
        lb = (ctypes.c_uint64 * max(n, 1))(*[int(x) for x in len_bounds])
        self.ptr = L.lmcg_decompress_plan_create(codec.ctx.ptr, n, hs, lb)
        if not self.ptr:
            raise_status(7, codec.ctx.error())
        self.out = torch.empty(max(int(L.lmcg_plan_output_bytes(self.ptr)), 16), dtype=torch.uint8, device=codec.device)
        self.status = torch.zeros(max(n, 1), dtype=torch.int32, device=codec.device)
        self.offsets, pos = [], 0
        for h in hints:
            self.offsets.append(pos)
            pos += (int(h[0]) + 15) & ~15
        self.lengths = [int(h[0]) for h in hints]
        self.source = source
        self.graph = None
        if graph:
            if source is None:
                raise ValueError("graph capture needs a fixed source buffer (a CompressPlan)")
            self.graph = _capture(lambda st: self._launch(st, source.out, source.meta[:n], source.meta[max(n, 1):]))

    def _launch(self, st, data, offsets, lengths) -> None:
        L = self.codec.ctx.lib
        rc = L.lmcg_decompress_plan_run(self.codec.ctx.ptr, self.ptr, data.data_ptr(), offsets.data_ptr(),
                                        lengths.data_ptr(), self.out.data_ptr(), self.status.data_ptr(),
                                        ctypes.c_void_p(st.cuda_stream))
        self.codec.ctx.check(rc)

    def run(self, batch: CompressedBatch | None = None, stream=None) -> DecompressedBatch:
        import torch

        if self.graph is not None and (batch is None or batch.data is self.source.out):
            self.graph.replay()
        else:
            if batch is None:
                raise ValueError("run() needs a CompressedBatch")
            self._launch(stream if stream is not None else torch.cuda.current_stream(self.codec.device),
                         batch.data, batch.offsets, batch.lengths)
        n = self.n
        return DecompressedBatch(self.out, self.offsets, self.lengths, None, None, None, status_dev=self.status[:n])

    def __del__(self):
        try:
            if getattr(self, "ptr", None):
                self.codec.ctx.lib.lmcg_plan_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass


def _capture(launch):
    """Warm up `launch` on a side stream, then capture it into a CUDA graph."""
    import torch

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        launch(side)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        launch(torch.cuda.current_stream())
    torch.cuda.synchronize()
    return g


_codecs: dict[int, Codec] = {}


def default_codec() -> Codec:
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the LMC B200 path has no CPU fallback")
    d = torch.cuda.current_device()
    c = _codecs.get(d)
    if c is None:
        c = _codecs[d] = Codec(d)
    return c


def _to_device_bytes(data: bytes, device):
    import torch

    if len(data) == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    h = torch.frombuffer(bytearray(data), dtype=torch.uint8)
    return h.pin_memory().to(device, non_blocking=True)


# ----------------------------------------------------- reference-shaped API
def compress_many(bufs: Sequence, *, byte_group: bool = True, block_size: int = DEFAULT_BLOCK_SIZE,
                  segment_count: int = 1, buffer_size: int = DEFAULT_BUFFER_SIZE) -> list[bytes]:
    """lmc_compress over many TensorBuffer / DeltaBuffer values in one batch."""
    codec = default_codec()
    tens, ets, dflags = [], [], []
    for b in bufs:
        et = element_code(b.element_type)
        _validate_options(_WIDTH[et], block_size, segment_count, buffer_size)
        tens.append(_to_device_bytes(bytes(b.data), codec.device))
        ets.append(et)
        dflags.append(is_delta(b))
    batch = codec.compress(tens, element_types=ets, delta=dflags, byte_group=byte_group, block_size=block_size,
                           segment_count=segment_count, buffer_size=buffer_size)
    return batch.to_bytes()


def lmc_compress(buf, *, byte_group: bool = True, block_size: int = DEFAULT_BLOCK_SIZE, segment_count: int = 1,
                 buffer_size: int = DEFAULT_BUFFER_SIZE) -> bytes:
    """stream.py:311-341 -- one buffer into a complete LMC1 codestream (GPU)."""
    return compress_many([buf], byte_group=byte_group, block_size=block_size, segment_count=segment_count,
                         buffer_size=buffer_size)[0]


def decompress_many(streams: Sequence[bytes]) -> list[TensorBuffer]:
    """lmc_decompress over many streams; raises the first stream's error."""
    codec = default_codec()
    dev = [_to_device_bytes(bytes(s), codec.device) for s in streams]
    res = codec.decompress(dev)
    res.raise_for_status()
    out = []
    host = res.data[: (res.offsets[-1] + res.lengths[-1]) if len(res) else 0].cpu().numpy().tobytes()
    for i in range(len(res)):
        o, n = res.offsets[i], res.lengths[i]
        out.append(TensorBuffer(host[o: o + n], ElementType.from_code(res.element_types[i])))
    return out


def lmc_decompress(stream: bytes) -> TensorBuffer:
    """stream.py:406-423 -- decode and CRC-verify one codestream (GPU)."""
    return decompress_many([stream])[0]
