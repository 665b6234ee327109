"""Compression overlapped with the device-to-host copy and the storage writes
(SURVEY.md §8(f) row 3).

The paper's motivation is finishing a checkpoint write before the next one
is due: the reference compresses on the CPU and then writes
(chain.py:185-196 -- compress a stream, write it, next).  Here the tensors
already live on the GPU, so one checkpoint flows through three stages that
run concurrently on different engines:

    SMs          compress group g            (compute stream)
    copy engine  D2H of group g-1's streams  (copy stream, pinned host slots)
    host thread  write group g-2's streams   (writer thread, plain file IO)

Tensors are cut into groups of about ``group_bytes`` (a tensor is never
split: each stream is its tensor's complete LMC1 stream, byte-identical to
``lmc_compress``).  ``depth`` pinned host slots and device output buffers
rotate between the groups; a slot is reused only after the writer has
written every stream in it.  The host learns a group's stream sizes from a
16-byte-per-stream SM-written copy (lmcg_copy_to_host), so the D2H moves
exactly the compressed bytes and the copy engine never waits on a size
readback queued behind bulk copies.
"""
from __future__ import annotations

import ctypes
import queue
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Callable, Sequence

from .stream import DEFAULT_BLOCK_SIZE, DEFAULT_BUFFER_SIZE, _bytes_view, _torch_et, default_codec

DEFAULT_GROUP_BYTES = 256 << 20


@dataclass(frozen=True)
class StreamItem:
    """One tensor to compress: uint8 CUDA view, LMC element type code, optional
    previous step (fused XOR delta, FLAG_DELTA)."""

    data: object
    element_type: int
    prev: object = None


def _groups(sizes: Sequence[int], group_bytes: int) -> list[list[int]]:
    out, cur, acc = [], [], 0
    for i, n in enumerate(sizes):
        if cur and acc + n > group_bytes:
            out.append(cur)
            cur, acc = [], 0
        cur.append(i)
        acc += n
    if cur:
        out.append(cur)
    return out


class StreamWriter:
    """Compress many device tensors and hand every stream to ``sink`` from a
    writer thread while later groups are still compressing.

    ``sink(i, view)`` receives item i's complete stream as a memoryview of
    pinned host memory, valid only during the call.  Groups reach the sink
    in order; the streams of one group go to ``writers`` threads at once
    (file creation and page-cache work are per-file kernel costs that
    parallelise).  ``run`` returns the stream lengths and re-raises the
    first sink error.
    """

    def __init__(self, codec=None, *, group_bytes: int = DEFAULT_GROUP_BYTES, depth: int = 2,
                 byte_group: bool = True, block_size: int = DEFAULT_BLOCK_SIZE, segment_count: int = 1,
                 buffer_size: int = DEFAULT_BUFFER_SIZE, writers: int = 4):
        if depth < 2:
            raise ValueError("depth must be >= 2 (one slot compressing, one draining)")
        self.codec = codec if codec is not None else default_codec()
        self.group_bytes, self.depth, self.writers = int(group_bytes), int(depth), max(1, int(writers))
        self.opts = dict(byte_group=byte_group, block_size=block_size, segment_count=segment_count,
                         buffer_size=buffer_size)
        self._dev = [None] * depth     # device output buffers
        self._pin = [None] * depth     # pinned host stream buffers
        self._meta = [None] * depth    # pinned host (offsets, lengths)

    def _grow(self, slot: int, bound: int, n: int) -> None:
        import torch

        if self._dev[slot] is None or self._dev[slot].numel() < bound:
            self._dev[slot] = torch.empty(max(bound, 16), dtype=torch.uint8, device=self.codec.device)
        if self._pin[slot] is None or self._pin[slot].numel() < bound:
            self._pin[slot] = torch.empty(max(bound, 16), dtype=torch.uint8, pin_memory=True)
        if self._meta[slot] is None or self._meta[slot].numel() < 2 * n:
            self._meta[slot] = torch.empty(2 * max(n, 1), dtype=torch.int64, pin_memory=True)

    def run(self, items: Sequence[StreamItem], sink: Callable[[int, memoryview], None]) -> list[int]:
        import torch

        from . import _lib

        codec = self.codec
        L = codec.ctx.lib
        comp = torch.cuda.Stream(codec.device)
        copy = torch.cuda.Stream(codec.device)
        comp.wait_stream(torch.cuda.current_stream(codec.device))
        groups = _groups([int(it.data.numel()) for it in items], self.group_bytes)
        lengths = [0] * len(items)
        free = [threading.Semaphore(1) for _ in range(self.depth)]
        work: queue.Queue = queue.Queue()
        errors: list[BaseException] = []

        pool = ThreadPoolExecutor(self.writers, thread_name_prefix="lmc-sink") if self.writers > 1 else None

        def writer():
            while True:
                job = work.get()
                if job is None:
                    return
                slot, idx, ev, offs, lens = job
                try:
                    ev.synchronize()
                    if not errors:
                        mv = memoryview(self._pin[slot].numpy())
                        calls = [(i, mv[o: o + n]) for i, o, n in zip(idx, offs, lens)]
                        if pool is None or len(calls) == 1:
                            for c in calls:
                                sink(*c)
                        else:
                            for _ in pool.map(lambda c: sink(*c), calls):
                                pass
                except BaseException as exc:   # surfaced by run()
                    errors.append(exc)
                finally:
                    free[slot].release()

        th = threading.Thread(target=writer, name="lmc-stream-writer", daemon=True)
        th.start()
        pending = None   # (slot, idx, done event) of the group compressed last

        def drain(p):
            slot, idx, done = p
            done.synchronize()             # this group's sizes are in pinned memory
            m = self._meta[slot][: 2 * len(idx)].tolist()
            offs, lens = m[: len(idx)], m[len(idx):]
            for i, n in zip(idx, lens):
                lengths[i] = n
            total = offs[-1] + lens[-1]
            copy.wait_event(done)
            with torch.cuda.stream(copy):
                self._pin[slot][:total].copy_(self._dev[slot][:total], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
            work.put((slot, idx, ev, offs, lens))

        try:
            for g, idx in enumerate(groups):
                slot = g % self.depth
                free[slot].acquire()   # the writer is done with this slot's previous group
                if errors:
                    free[slot].release()
                    break
                tens = [items[i].data for i in idx]
                prev = [items[i].prev for i in idx]
                ets = [items[i].element_type for i in idx]
                arr = (_lib.lmcg_tensor * len(idx))()
                for j, i in enumerate(idx):
                    arr[j].nbytes = int(items[i].data.numel())
                    arr[j].element_type = int(ets[j])
                    arr[j].delta = int(prev[j] is not None)
                o = self.opts
                opts = _lib.lmcg_options(int(bool(o["byte_group"])), o["block_size"], o["segment_count"], 0,
                                         o["buffer_size"])
                self._grow(slot, int(L.lmcg_compress_bound(arr, len(idx), ctypes.byref(opts))), len(idx))
                with torch.cuda.stream(comp):   # (scratch allocations belong to the compute stream)
                    batch = codec.compress(tens, element_types=ets,
                                           prev=prev if any(p is not None for p in prev) else None,
                                           out=self._dev[slot], stream=comp, **o)
                meta = self._meta[slot]
                codec.ctx.check(L.lmcg_copy_to_host(ctypes.c_void_p(meta.data_ptr()),
                                                    ctypes.c_void_p(batch.offsets.data_ptr()),
                                                    8 * len(idx), ctypes.c_void_p(comp.cuda_stream)))
                codec.ctx.check(L.lmcg_copy_to_host(ctypes.c_void_p(meta.data_ptr() + 8 * len(idx)),
                                                    ctypes.c_void_p(batch.lengths.data_ptr()),
                                                    8 * len(idx), ctypes.c_void_p(comp.cuda_stream)))
                done = torch.cuda.Event()
                done.record(comp)
                # the inputs stay alive until the compress is done
                for t in tens:
                    t.record_stream(comp)
                for p in prev:
                    if p is not None:
                        p.record_stream(comp)
                if pending is not None:   # group g-1 drains while group g compresses
                    drain(pending)
                pending = (slot, idx, done)
            if pending is not None and not errors:
                drain(pending)
        finally:
            work.put(None)
            th.join()
            if pool is not None:
                pool.shutdown()
            torch.cuda.current_stream(codec.device).wait_stream(comp)
            torch.cuda.current_stream(codec.device).wait_stream(copy)
        if errors:
            raise errors[0]
        return lengths


def items_from_tensors(tensors: Sequence, prev: Sequence | None = None,
                       element_types: Sequence[int] | None = None) -> list[StreamItem]:
    """StreamItems of CUDA tensors (element type from the torch dtype unless given)."""
    out = []
    for i, t in enumerate(tensors):
        et = int(element_types[i]) if element_types is not None else _torch_et(t.dtype)
        p = None if prev is None or prev[i] is None else _bytes_view(prev[i])
        out.append(StreamItem(_bytes_view(t), et, p))
    return out


def write_streams(tensors: Sequence, paths: Sequence, *, prev: Sequence | None = None,
                  element_types: Sequence[int] | None = None, codec=None, **kw) -> list[int]:
    """Compress every CUDA tensor into its own LMC1 stream file (write-then-rename),
    compression overlapped with the D2H copies and the file writes."""
    import os
    from pathlib import Path

    paths = [Path(p) for p in paths]

    def sink(i: int, view: memoryview) -> None:
        tmp = paths[i].with_name(paths[i].name + ".tmp")
        with open(tmp, "wb") as f:
            f.write(view)
        os.replace(tmp, paths[i])

    return StreamWriter(codec, **kw).run(items_from_tensors(tensors, prev, element_types), sink)


_staging: dict = {}


def _staging_slots(nslots: int, nbytes: int):
    """Pinned staging slots, allocated once per process and reused (pinning
    gigabytes for every restore would cost more than the reads)."""
    import torch

    key = (nslots, nbytes)
    if key not in _staging:
        _staging[key] = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(nslots)]
    return _staging[key]


def read_files_to_device(paths: Sequence, device, *, head: int = 64, slot_bytes: int = 64 << 20,
                         threads: int = 8):
    """Whole files into one device buffer (16-byte aligned offsets), read by
    a thread pool into two reused pinned slots while the other slot's
    host-to-device copy runs.  Returns ``(device uint8 tensor, offsets,
    lengths, heads, errors)``: ``heads[i]`` are the first ``head`` bytes of
    file i (for host-side header checks); an unreadable file has length 0
    and its ``OSError`` in ``errors``."""
    import os
    from pathlib import Path

    import torch

    paths = [Path(p) for p in paths]
    n = len(paths)
    lengths, errors, heads = [0] * n, [None] * n, [b""] * n
    for i, p in enumerate(paths):
        try:
            lengths[i] = os.stat(p).st_size
        except OSError as exc:
            errors[i] = exc
    offsets, pos = [], 0
    for L in lengths:
        offsets.append(pos)
        pos += (L + 15) & ~15
    dev = torch.empty(max(pos, 16), dtype=torch.uint8, device=device)
    slots = _staging_slots(2, slot_bytes)
    copy = torch.cuda.Stream(device)
    done = [None, None]

    def fill(k: int, slot, lo: int, hi: int) -> None:
        # the parts of every file inside device bytes [lo, hi)
        mv = memoryview(slot.numpy())
        jobs = [i for i in range(n) if lengths[i] and errors[i] is None and offsets[i] < hi and offsets[i] + lengths[i] > lo]

        def read(i: int) -> None:
            a, b = max(offsets[i], lo), min(offsets[i] + lengths[i], hi)
            try:
                fd = os.open(paths[i], os.O_RDONLY)
                try:
                    if a == offsets[i]:
                        heads[i] = os.pread(fd, head, 0)
                    got = 0
                    while got < b - a:
                        r = os.preadv(fd, [mv[a - lo + got: b - lo]], a - offsets[i] + got)
                        if not r:
                            raise OSError(f"{paths[i]}: file shrank while reading")
                        got += r
                finally:
                    os.close(fd)
            except OSError as exc:
                errors[i] = exc

        if threads > 1 and len(jobs) > 1:
            list(pool.map(read, jobs))
        else:
            for i in jobs:
                read(i)

    with ThreadPoolExecutor(max(1, threads), thread_name_prefix="lmc-read") as pool:
        for k, lo in enumerate(range(0, pos, slot_bytes)):
            hi = min(lo + slot_bytes, pos)
            s = k % 2
            if done[s] is not None:
                done[s].synchronize()   # this slot's previous copy has left it
            fill(k, slots[s], lo, hi)
            with torch.cuda.stream(copy):
                dev[lo:hi].copy_(slots[s][: hi - lo], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            done[s] = ev
    torch.cuda.current_stream(device).wait_stream(copy)
    # the staging slots are process-global: the next call (or another thread)
    # may refill them as soon as this returns, so their copies must be done
    for ev in done:
        if ev is not None:
            ev.synchronize()
    for i in range(n):
        if errors[i] is not None:
            lengths[i] = 0
    return dev, offsets, lengths, heads, errors
