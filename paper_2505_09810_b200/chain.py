"""Checkpoint delta chains with the previous step resident in HBM.

On disk this is the reference's chain, file for file (pkg/src/lmc/chain.py):
``manifest.jsonl`` (a ``{"chain_id": ...}`` line, then one sorted-key JSON
object per stream) and one ``step{N:06d}_{shard}.lmc`` stream per step and
shard; step 0 holds the shards whole, step N the XOR delta against step N-1.
Chains written here restore with ``lmc.chain.restore_step`` and vice versa,
the streams are byte-identical to the reference's, and writers serialise on
the same ``.chain.lock`` file lock.

What changes is where step N-1 lives.  The reference's ``add_step``
re-decodes the whole chain from disk to rebuild step N-1 for every new step
(chain.py:174-180, O(steps) per add).  ``DeviceChain`` keeps the last step
resident in one HBM buffer: ``add_step`` compresses ``prev ^ current`` with
the XOR fused into the compress kernels' loads (lmcg_compress with
``lmcg_tensor.prev``), then refreshes the resident copy; ``restore_step``
decodes step 0 into the resident buffer and applies every delta in place
with the XOR fused into the decode's output stage (lmcg_decompress_apply).
Validation and error classes follow ``_load_entry`` / ``_check_shapes``
(chain.py:211-258) in the reference's order.
"""
from __future__ import annotations

import json
import os
import re
import uuid
from dataclasses import asdict, dataclass, field
from pathlib import Path

from filelock import FileLock

from .errors import (CorruptStreamError, DtypeMismatchError, IntegrityError, LmcError, MissingStreamError,
                     ShapeMismatchError, raise_status)
from .pipeline import StreamItem, StreamWriter, read_files_to_device
from .stream import DEFAULT_BLOCK_SIZE, _bytes_view, _torch_et, default_codec, parse_header
from .types import ElementType, TensorBuffer

MANIFEST_NAME = "manifest.jsonl"
LOCK_NAME = ".chain.lock"
ROLE_BASE, ROLE_DELTA = "base", "delta"


@dataclass(frozen=True)
class ChainEntry:
    """One stream of the chain (chain.py:44-54): field order is the JSON key set."""

    step: int
    role: str
    shard: str
    dtype: str
    length: int
    file: str
    crc32: int


@dataclass
class DeltaManifest:
    """The manifest (chain.py:57-91)."""

    chain_id: str
    entries: list[ChainEntry] = field(default_factory=list)

    @property
    def last_step(self) -> int:
        return max((e.step for e in self.entries), default=-1)

    def step_entries(self, step: int) -> list[ChainEntry]:
        got = [e for e in self.entries if e.step == step]
        if not got:
            raise MissingStreamError(f"step {step} is not in the chain")
        return got

    def shard_names(self, step: int) -> list[str]:
        return sorted(e.shard for e in self.step_entries(step))

    def validate(self) -> None:
        if self.last_step < 0:
            return
        names = self.shard_names(0)
        if any(e.role != ROLE_BASE for e in self.step_entries(0)):
            raise CorruptStreamError("step 0 entries must all be bases")
        for k in range(1, self.last_step + 1):
            if self.shard_names(k) != names:
                raise CorruptStreamError(f"step {k} does not cover the chain's shard set")
            if any(e.role != ROLE_DELTA for e in self.step_entries(k)):
                raise CorruptStreamError(f"step {k} entries must all be deltas")

    def to_bytes(self) -> bytes:
        rows = [json.dumps({"chain_id": self.chain_id})]
        rows.extend(json.dumps(asdict(e), sort_keys=True) for e in self.entries)
        return ("\n".join(rows) + "\n").encode()


def _replace_file(path: Path, data) -> None:
    """Write-then-rename, so readers never see a partial file (chain.py:94-97)."""
    tmp = path.with_name(path.name + ".tmp")
    with open(tmp, "wb") as f:
        f.write(data)
    os.replace(tmp, path)


def save_manifest(chain_dir, manifest: DeltaManifest) -> None:
    _replace_file(Path(chain_dir) / MANIFEST_NAME, manifest.to_bytes())


def load_manifest(chain_dir) -> DeltaManifest:
    """chain.py:110-121."""
    path = Path(chain_dir) / MANIFEST_NAME
    if not path.exists():
        raise MissingStreamError(f"no manifest at {path}")
    rows = path.read_text().splitlines()
    if not rows:
        raise CorruptStreamError(f"empty manifest at {path}")
    chain_id = json.loads(rows[0])["chain_id"]
    m = DeltaManifest(chain_id, [ChainEntry(**json.loads(r)) for r in rows[1:] if r.strip()])
    m.validate()
    return m


def stream_name(step: int, shard: str) -> str:
    """chain.py:124-126: shard names sanitised to [A-Za-z0-9._-]."""
    return "step%06d_%s.lmc" % (step, re.sub(r"[^A-Za-z0-9._-]", "_", shard))


def chain_lock(chain_dir) -> FileLock:
    return FileLock(os.fspath(Path(chain_dir) / LOCK_NAME))


def _as_device_bytes(x, device):
    """(uint8 CUDA view, ElementType) of a CUDA tensor or a host TensorBuffer."""
    import torch

    if isinstance(x, TensorBuffer):
        v = torch.frombuffer(bytearray(x.data), dtype=torch.uint8) if len(x.data) else torch.empty(0, dtype=torch.uint8)
        return v.to(device), x.element_type
    if not x.is_cuda:
        raise ValueError("DeviceChain shards must be CUDA tensors or TensorBuffers")
    return _bytes_view(x), ElementType.from_code(_torch_et(x.dtype))


class DeviceChain:
    """A checkpoint chain whose latest step stays resident on one GPU.

    ``add_step(shards)`` appends a step (shards: name -> CUDA tensor or
    TensorBuffer) and returns its index, like ``lmc.chain.add_step``;
    ``restore_step(k)`` returns name -> CUDA uint8 tensor of step k's bytes
    (``restore_buffers`` gives the reference's TensorBuffer dict).
    """

    def __init__(self, chain_dir, *, codec=None, block_size: int = DEFAULT_BLOCK_SIZE, byte_group: bool = True,
                 segment_count: int = 1):
        self.dir = Path(chain_dir)
        self.codec = codec if codec is not None else default_codec()
        self.block_size, self.byte_group, self.segment_count = block_size, byte_group, segment_count
        self._buf = None          # resident step: one CUDA byte buffer, shards at 16-byte aligned offsets
        self._layout: dict[str, tuple[int, int, ElementType]] = {}
        self._step = -1           # step held in _buf (-1: nothing valid)
        self._chain_id = None     # manifest the resident step came from

    def release(self) -> None:
        """Free the resident step's HBM buffer (the next add_step restores
        the previous step from the files again)."""
        self._buf = None
        self._layout = {}
        self._step = -1
        self._chain_id = None

    # ------------------------------------------------------------ resident
    def _view(self, name: str):
        off, n, _ = self._layout[name]
        return self._buf[off: off + n]

    def _make_resident(self, sizes: dict[str, tuple[int, ElementType]]) -> None:
        import torch

        layout, pos = {}, 0
        for name in sorted(sizes):
            n, et = sizes[name]
            layout[name] = (pos, n, et)
            pos += (n + 15) & ~15
        if self._buf is None or self._buf.numel() < max(pos, 16):
            self._buf = torch.empty(max(pos, 16), dtype=torch.uint8, device=self.codec.device)
        self._layout = layout
        self._step = -1

    # ------------------------------------------------------------ add
    def add_step(self, shards: dict, *, step: int | None = None) -> int:
        """chain.py:133-208 with step N-1 taken from HBM instead of re-decoding the chain."""
        self.dir.mkdir(parents=True, exist_ok=True)
        if not shards:
            raise ShapeMismatchError("a step needs at least one shard")
        with chain_lock(self.dir):
            mpath = self.dir / MANIFEST_NAME
            manifest = load_manifest(self.dir) if mpath.exists() else DeltaManifest(uuid.uuid4().hex, [])
            nxt = manifest.last_step + 1
            if step is not None and step != nxt:
                if step <= manifest.last_step:
                    raise LmcError(f"step {step} already exists (chain is at {manifest.last_step})")
                raise LmcError(f"chain expects step {nxt}, got {step}")
            cur = {name: _as_device_bytes(t, self.codec.device) for name, t in shards.items()}
            if nxt > 0:
                if self._step != nxt - 1 or self._chain_id != manifest.chain_id:
                    self._restore(manifest, nxt - 1)
                self._check_shapes(cur, nxt)
            names = sorted(cur)
            files = [stream_name(nxt, name) for name in names]
            if len(set(files)) != len(files):
                raise LmcError(f"shard names {names} collide after filename sanitization")
            prev = [self._view(name) for name in names] if nxt > 0 else None
            # compress overlapped with the D2H copies and the file writes
            # (pipeline.StreamWriter); the streams land in their files in order
            role = ROLE_BASE if nxt == 0 else ROLE_DELTA
            crcs = [0] * len(names)

            def sink(i: int, view: memoryview) -> None:
                _replace_file(self.dir / files[i], view)
                # the header CRC is zlib.crc32 of the (delta) payload, which is
                # what the reference records (chain.py:201)
                crcs[i] = int.from_bytes(view[24:28], "little")

            items = [StreamItem(cur[name][0], cur[name][1].code, None if prev is None else prev[j])
                     for j, name in enumerate(names)]
            StreamWriter(self.codec, byte_group=self.byte_group, block_size=self.block_size,
                         segment_count=self.segment_count).run(items, sink)
            entries = [ChainEntry(step=nxt, role=role, shard=name, dtype=cur[name][1].name.lower(),
                                  length=cur[name][0].numel(), file=fname, crc32=crcs[j])
                       for j, (name, fname) in enumerate(zip(names, files))]
            manifest.entries.extend(entries)
            save_manifest(self.dir, manifest)
            # the new step becomes the resident one (device-to-device copies)
            if nxt == 0:
                self._make_resident({name: (cur[name][0].numel(), cur[name][1]) for name in names})
            for name in names:
                self._view(name).copy_(cur[name][0])
            self._step, self._chain_id = nxt, manifest.chain_id
        return nxt

    def _check_shapes(self, cur: dict, step: int) -> None:
        """chain.py:211-231 against the resident step."""
        if sorted(self._layout) != sorted(cur):
            raise ShapeMismatchError(f"step {step} shard names {sorted(cur)} do not match "
                                     f"step {step - 1} shard names {sorted(self._layout)}")
        for name, (_, n, et) in self._layout.items():
            v, cet = cur[name]
            if v.numel() != n:
                raise ShapeMismatchError(f"shard {name!r} changed length at step {step}: {n} -> {v.numel()}")
            if cet is not et:
                raise DtypeMismatchError(f"shard {name!r} changed element type at step {step}")

    # ------------------------------------------------------------ restore
    def restore_step(self, step: int) -> dict:
        """chain.py:280-300: every shard of step ``step`` bit-exactly, as CUDA
        uint8 tensors (copies; the resident buffer stays with the chain)."""
        manifest = load_manifest(self.dir)
        if step < 0 or step > manifest.last_step:
            raise MissingStreamError(f"step {step} is not in the chain (last is {manifest.last_step})")
        if self._step != step or self._chain_id != manifest.chain_id:
            self._restore(manifest, step)
        return {name: self._view(name).clone() for name in sorted(self._layout)}

    def restore_buffers(self, step: int) -> dict[str, TensorBuffer]:
        """restore_step as the reference's return type (host TensorBuffers)."""
        out = self.restore_step(step)
        return {name: TensorBuffer(out[name].cpu().numpy().tobytes(), self._layout[name][2]) for name in out}

    def _restore(self, manifest: DeltaManifest, step: int) -> None:
        self._step = -1
        base = manifest.step_entries(0)
        self._make_resident({e.shard: (e.length, ElementType.from_name(e.dtype)) for e in base})
        self._apply_entries(base, delta=False)
        for k in range(1, step + 1):
            self._apply_entries(manifest.step_entries(k), delta=True)
        self._step, self._chain_id = step, manifest.chain_id

    def _apply_entries(self, entries: list[ChainEntry], *, delta: bool) -> None:
        """_load_entry (chain.py:234-258) for every entry of one step, decoded
        in one batch; errors surface in entry order with the reference's
        precedence: file, header, manifest CRC, role flag, decode (corrupt /
        CRC), decoded length, element type, then xor_apply's length check."""
        import torch

        pre: list[Exception | None] = []
        headers = []
        # every stream file of the step read by a thread pool through two
        # reused pinned slots, overlapped with their host-to-device copies
        dev_all, hoffs, hlens, heads, herrs = read_files_to_device([self.dir / e.file for e in entries],
                                                                   self.codec.device)
        for i, e in enumerate(entries):
            err, h = None, None
            path = self.dir / e.file
            try:
                if herrs[i] is not None:
                    if not path.exists():
                        raise MissingStreamError(f"stream file {path} is missing")
                    raise herrs[i]
                h = parse_header(heads[i])
                if h.crc32 != e.crc32:
                    raise IntegrityError(f"stream {e.file} CRC does not match the manifest")
                if h.delta_applied != (e.role == ROLE_DELTA):
                    raise CorruptStreamError(f"stream {e.file} role flag does not match the manifest")
            except LmcError as exc:
                err = exc
            pre.append(err)
            headers.append(h)
        # streams that passed the host checks and decode to their region's size
        # go through one batched decode straight into the resident buffer;
        # others (length disagrees with the manifest) decode on their own so
        # their own errors still come first
        go, alone = [], []
        for i, e in enumerate(entries):
            if pre[i] is None:
                (go if headers[i].original_length == e.length and e.shard in self._layout
                 and self._layout[e.shard][1] == e.length else alone).append(i)
        status = {}
        if go:
            dev = [dev_all[hoffs[i]: hoffs[i] + hlens[i]] for i in go]
            offs = [self._layout[entries[i].shard][0] for i in go]
            prev = [self._view(entries[i].shard) for i in go] if delta else None
            res = self.codec.decompress(dev, out=self._buf, out_offsets=offs, prev=prev)
            for j, i in enumerate(go):
                status[i] = (res.status[j], res.element_types[j], res.lengths[j])
        for i in alone:
            res = self.codec.decompress([dev_all[hoffs[i]: hoffs[i] + hlens[i]]])
            status[i] = (res.status[0], res.element_types[0], res.lengths[0])
        for i, e in enumerate(entries):
            if pre[i] is not None:
                self._step = -1
                raise pre[i]
            code, et, n = status[i]
            if code:
                self._step = -1
                raise_status(code, f"stream {e.file}: status {code}")
            if n != e.length:
                self._step = -1
                raise CorruptStreamError(f"stream {e.file} decodes to {n} bytes, manifest says {e.length}")
            if ElementType.from_code(et) is not ElementType.from_name(e.dtype):
                self._step = -1
                raise DtypeMismatchError(f"stream {e.file} element type does not match the manifest")
            if e.shard not in self._layout or self._layout[e.shard][1] != n:
                self._step = -1
                raise ShapeMismatchError(f"length mismatch: {self._layout.get(e.shard, (0, 0))[1]} vs {n}")


# ------------------------------------------------- reference-shaped module API
_chains: dict[tuple, DeviceChain] = {}


def _chain_for(chain_dir, block_size: int, byte_group: bool, segment_count: int) -> DeviceChain:
    codec = default_codec()
    key = (os.path.realpath(os.fspath(chain_dir)), codec.ctx.device, block_size, bool(byte_group), segment_count)
    ch = _chains.get(key)
    if ch is None:
        # one resident step per chain directory: entries of the same directory
        # with other options hold a stale step, drop them
        for k in [k for k in _chains if k[0] == key[0]]:
            _chains.pop(k).release()
        ch = _chains[key] = DeviceChain(chain_dir, codec=codec, block_size=block_size, byte_group=byte_group,
                                        segment_count=segment_count)
    return ch


def release_chains(chain_dir=None) -> None:
    """Free the HBM that module-level ``add_step`` keeps resident (every chain,
    or only ``chain_dir``'s).  Later calls restore from the files."""
    path = None if chain_dir is None else os.path.realpath(os.fspath(chain_dir))
    for k in [k for k in _chains if path is None or k[0] == path]:
        _chains.pop(k).release()


def add_step(chain_dir, shards: dict, *, step: int | None = None, block_size: int = DEFAULT_BLOCK_SIZE,
             byte_group: bool = True, segment_count: int = 1) -> int:
    """chain.py:133-208 (same arguments, same files): the chain's latest step
    stays resident on the GPU between calls in this process."""
    return _chain_for(chain_dir, block_size, byte_group, segment_count).add_step(shards, step=step)


def restore_step(chain_dir, step: int) -> dict[str, TensorBuffer]:
    """chain.py:260-278: every shard of one step as host TensorBuffers, decoded
    from the files on disk like the reference (never from a resident step)."""
    load_manifest(chain_dir)   # (MissingStreamError before any device work)
    return DeviceChain(chain_dir, codec=default_codec()).restore_buffers(step)
