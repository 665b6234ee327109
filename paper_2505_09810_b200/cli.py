"""Command line front-end on the GPU path.

Mirrors the reference CLI's codec and chain commands (pkg/src/lmc/cli.py:
``compress`` :127-163, ``decompress`` :166-178, ``checkpoint add`` :207-218
with raw shard files or JSONL shard manifests :184-204, ``checkpoint
restore`` :221-233), with the same arguments, output files, stderr lines and
stable exit codes (cli.py:1-6, 52-78): 0 ok, 2 bad input, 3 integrity /
corruption, 4 shape mismatch, 5 missing chain data, 6 bad configuration,
1 other IO / device failures.  Streams are byte-identical to the reference
CLI's for the same options (``--threads`` is still the stream's segment
count, exactly as the reference passes it to plmc_compress).

``batch compress`` / ``batch decompress`` are the batched multi-tensor
entry: every shard of a JSONL manifest goes through one batched GPU call,
and the streams are written while later groups still compress
(pipeline.StreamWriter).  The reference's ``analyze`` and ``bench`` groups
are analysis tooling, out of scope.

Run as ``python -m paper_2505_09810_b200.cli``.
"""
from __future__ import annotations

import functools
import json
import os
import re
import sys
import time
from pathlib import Path

import click

from .errors import (AlignmentError, ConfigError, CorruptStreamError, DeviceError, DtypeMismatchError,
                     EmptyInputError, IntegrityError, LmcError, MissingStreamError, ShapeMismatchError,
                     UnsupportedFormatError)
from .stream import DEFAULT_BLOCK_SIZE, DEFAULT_BUFFER_SIZE
from .types import ElementType, TensorBuffer

EXIT_INPUT = 2
EXIT_INTEGRITY = 3
EXIT_SHAPE = 4
EXIT_MISSING = 5
EXIT_CONFIG = 6

_EXIT_CODES: list[tuple[type[Exception], int]] = [
    (AlignmentError, EXIT_INPUT),
    (EmptyInputError, EXIT_INPUT),
    (CorruptStreamError, EXIT_INTEGRITY),
    (IntegrityError, EXIT_INTEGRITY),
    (UnsupportedFormatError, EXIT_INTEGRITY),
    (ShapeMismatchError, EXIT_SHAPE),
    (DtypeMismatchError, EXIT_SHAPE),
    (MissingStreamError, EXIT_MISSING),
    (ConfigError, EXIT_CONFIG),
    (FileNotFoundError, EXIT_MISSING),
    (DeviceError, 1),
    (LmcError, EXIT_INPUT),
    (OSError, 1),
]


def exit_code(exc: Exception) -> int:
    """cli.py:75-79: first matching class wins."""
    for etype, code in _EXIT_CODES:
        if isinstance(exc, etype):
            return code
    return 1


def handle_errors(fn):
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except (LmcError, OSError, ValueError) as exc:
            click.echo(f"error: {exc}", err=True)
            sys.exit(exit_code(exc) if not isinstance(exc, ValueError) else EXIT_INPUT)

    return wrapper


def _dtype_option(default: str = "raw"):
    return click.option("--dtype", type=click.Choice(["bf16", "fp16", "fp32", "raw"]), default=default,
                        show_default=True, help="Element type of the raw input bytes.")


def default_threads() -> int:
    """cli.py:98-105: LMC_THREADS, else the core count (the stream's segment count)."""
    env = os.environ.get("LMC_THREADS")
    if env:
        try:
            return max(1, int(env))
        except ValueError:
            pass
    return os.cpu_count() or 1


_threads_option = click.option("--threads", type=int, default=None,
                               help="Segment count of the stream (default: LMC_THREADS or the core count).")


def _device_bytes(data: bytes):
    """Host bytes -> CUDA uint8 tensor through pinned memory."""
    import torch

    from .stream import default_codec

    dev = default_codec().device
    if not data:
        return torch.empty(0, dtype=torch.uint8, device=dev)
    h = torch.empty(len(data), dtype=torch.uint8, pin_memory=True)
    h.numpy()[:] = memoryview(data)
    return h.to(dev, non_blocking=True)


@click.group()
@click.version_option(version="0.1.0", prog_name="lmc-b200")
def main() -> None:
    """Lossless compression for LLM checkpoint tensor data (B200 GPU path)."""


@main.command()
@click.argument("input_path", type=click.Path(exists=True, dir_okay=False, path_type=Path))
@click.argument("output_path", type=click.Path(dir_okay=False, path_type=Path))
@_dtype_option()
@click.option("--block-size", type=int, default=DEFAULT_BLOCK_SIZE, show_default=True)
@click.option("--buffer-size", type=int, default=DEFAULT_BUFFER_SIZE, show_default=True)
@_threads_option
@click.option("--no-bytegroup", is_flag=True, help="Skip the byte-grouping stage.")
@click.option("--delta", "delta_path", type=click.Path(exists=True, dir_okay=False, path_type=Path), default=None,
              help="Compress the XOR delta against this previous-step file.")
@handle_errors
def compress(input_path, output_path, dtype, block_size, buffer_size, threads, no_bytegroup, delta_path):
    """Compress a raw tensor file into a codestream."""
    from .stream import _validate_options, default_codec

    et = ElementType.from_name(dtype)
    data = input_path.read_bytes()
    TensorBuffer(data, et)                     # AlignmentError before any device work
    prev_data = None
    if delta_path is not None:
        prev_data = delta_path.read_bytes()
        TensorBuffer(prev_data, et)
        if len(prev_data) != len(data):        # xor_delta (delta.py:20-21)
            raise ShapeMismatchError(f"length mismatch: {len(prev_data)} vs {len(data)}")
    threads = threads or default_threads()
    _validate_options(et.width, block_size, threads, buffer_size)
    codec = default_codec()
    cur = _device_bytes(data)
    prev = [_device_bytes(prev_data)] if prev_data is not None else None
    start = time.perf_counter()
    batch = codec.compress([cur], element_types=[et.code], prev=prev, delta=prev is not None,
                           byte_group=not no_bytegroup, block_size=block_size, segment_count=threads,
                           buffer_size=buffer_size)
    stream = batch.to_bytes()[0]
    elapsed = max(time.perf_counter() - start, 1e-9)
    output_path.write_bytes(stream)
    ratio = len(stream) / len(data) if data else 1.0
    click.echo(f"ratio={ratio:.6f} MiB/s={len(data) / (1024 * 1024) / elapsed:.2f}", err=True)


@main.command()
@click.argument("input_path", type=click.Path(exists=True, dir_okay=False, path_type=Path))
@click.argument("output_path", type=click.Path(dir_okay=False, path_type=Path))
@_threads_option
@handle_errors
def decompress(input_path, output_path, threads):
    """Restore the exact original bytes from a codestream."""
    from .stream import parse_header

    stream = input_path.read_bytes()
    parse_header(stream)                       # magic / version errors before any device work
    from .stream import lmc_decompress

    output_path.write_bytes(lmc_decompress(stream).data)


@main.group()
def checkpoint() -> None:
    """Manage incremental checkpoint chains."""


def read_step_shards(files, dtype: str) -> dict[str, TensorBuffer]:
    """cli.py:184-204: raw .bin shard files or JSONL shard manifests
    (one ``{"name", "path", "dtype"?}`` object per line, paths relative to the manifest)."""
    shards: dict[str, TensorBuffer] = {}
    for path in files:
        path = Path(path)
        if path.suffix == ".jsonl":
            for line in path.read_text().splitlines():
                if not line.strip():
                    continue
                spec = json.loads(line)
                shard_path = Path(spec["path"])
                if not shard_path.is_absolute():
                    shard_path = path.parent / shard_path
                et = ElementType.from_name(spec.get("dtype", dtype))
                shards[spec["name"]] = TensorBuffer(shard_path.read_bytes(), et)
        else:
            shards[path.name] = TensorBuffer(path.read_bytes(), ElementType.from_name(dtype))
    return shards


@checkpoint.command("add")
@click.argument("chain_dir", type=click.Path(file_okay=False, path_type=Path))
@click.argument("files", nargs=-1, required=True, type=click.Path(exists=True, dir_okay=False, path_type=Path))
@_dtype_option()
@click.option("--step", type=int, default=None, help="Expected step index (rejects duplicates).")
@click.option("--block-size", type=int, default=DEFAULT_BLOCK_SIZE, show_default=True)
@handle_errors
def checkpoint_add(chain_dir, files, dtype, step, block_size):
    """Add the next checkpoint step (raw shard files or a .jsonl manifest)."""
    from . import chain as chain_mod

    shards = read_step_shards(files, dtype)
    idx = chain_mod.add_step(chain_dir, shards, step=step, block_size=block_size)
    click.echo(f"added step {idx} ({len(shards)} shard(s))", err=True)


@checkpoint.command("restore")
@click.argument("chain_dir", type=click.Path(exists=True, file_okay=False, path_type=Path))
@click.argument("step", type=int)
@click.argument("output_dir", type=click.Path(file_okay=False, path_type=Path))
@handle_errors
def checkpoint_restore(chain_dir, step, output_dir):
    """Write every shard of one step, byte-exact, into OUTPUT_DIR."""
    from . import chain as chain_mod

    shards = chain_mod.restore_step(chain_dir, step)
    output_dir = Path(output_dir)
    output_dir.mkdir(parents=True, exist_ok=True)
    for name, buf in sorted(shards.items()):
        (output_dir / name).write_bytes(buf.data)
    click.echo(f"restored step {step} ({len(shards)} shard(s))", err=True)


# ------------------------------------------------------------------ batch
BATCH_MANIFEST = "streams.jsonl"


def shard_file(name: str) -> str:
    """A shard name as a file name (the chain's sanitisation, chain.py:124-126)."""
    return re.sub(r"[^A-Za-z0-9._-]", "_", name)


def stream_file(name: str) -> str:
    return shard_file(name) + ".lmc"


@main.group()
def batch() -> None:
    """Many shards per call (JSONL shard manifests), one batched GPU pass."""


@batch.command("compress")
@click.argument("manifest", type=click.Path(exists=True, dir_okay=False, path_type=Path))
@click.argument("out_dir", type=click.Path(file_okay=False, path_type=Path))
@_dtype_option()
@click.option("--delta", "delta_manifest", type=click.Path(exists=True, dir_okay=False, path_type=Path),
              default=None, help="JSONL manifest of the previous step: compress XOR deltas against it.")
@click.option("--block-size", type=int, default=DEFAULT_BLOCK_SIZE, show_default=True)
@click.option("--buffer-size", type=int, default=DEFAULT_BUFFER_SIZE, show_default=True)
@click.option("--segments", type=int, default=1, show_default=True, help="Segment count per stream.")
@click.option("--no-bytegroup", is_flag=True)
@click.option("--group-mib", type=int, default=256, show_default=True,
              help="Bytes per pipelined compress group (D2H + writes overlap the next group).")
@handle_errors
def batch_compress(manifest, out_dir, dtype, delta_manifest, block_size, buffer_size, segments, no_bytegroup,
                   group_mib):
    """Compress every shard of MANIFEST into OUT_DIR/<name>.lmc (+ streams.jsonl)."""
    from .pipeline import StreamItem, StreamWriter
    from .stream import _validate_options, default_codec

    shards = read_step_shards([manifest], dtype)
    if not shards:
        raise EmptyInputError(f"{manifest} lists no shards")
    prev = read_step_shards([delta_manifest], dtype) if delta_manifest is not None else None
    names = sorted(shards)
    files = [stream_file(n) for n in names]
    if len(set(files)) != len(files):
        raise LmcError(f"shard names {names} collide after filename sanitization")
    for n in names:
        _validate_options(shards[n].element_type.width, block_size, segments, buffer_size)
        if prev is not None:
            if n not in prev:
                raise ShapeMismatchError(f"shard {n!r} is not in the previous step")
            if len(prev[n].data) != len(shards[n].data):
                raise ShapeMismatchError(f"length mismatch: {len(prev[n].data)} vs {len(shards[n].data)}")
    codec = default_codec()
    items = [StreamItem(_device_bytes(shards[n].data), shards[n].element_type.code,
                        None if prev is None else _device_bytes(prev[n].data)) for n in names]
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    crcs = [0] * len(names)

    def sink(i: int, view: memoryview) -> None:
        tmp = out_dir / (files[i] + ".tmp")
        with open(tmp, "wb") as f:
            f.write(view)
        os.replace(tmp, out_dir / files[i])
        crcs[i] = int.from_bytes(view[24:28], "little")

    start = time.perf_counter()
    lengths = StreamWriter(codec, group_bytes=group_mib << 20, byte_group=not no_bytegroup, block_size=block_size,
                           segment_count=segments, buffer_size=buffer_size).run(items, sink)
    elapsed = max(time.perf_counter() - start, 1e-9)
    rows = [json.dumps({"name": n, "dtype": shards[n].element_type.name.lower(), "length": len(shards[n].data),
                        "file": f, "stream_bytes": ln, "crc32": c, "delta": prev is not None}, sort_keys=True)
            for n, f, ln, c in zip(names, files, lengths, crcs)]
    (out_dir / BATCH_MANIFEST).write_text("\n".join(rows) + "\n")
    total = sum(len(shards[n].data) for n in names)
    click.echo(f"streams={len(names)} ratio={sum(lengths) / total if total else 1.0:.6f} "
               f"MiB/s={total / (1024 * 1024) / elapsed:.2f}", err=True)


@batch.command("decompress")
@click.argument("streams_manifest", type=click.Path(exists=True, dir_okay=False, path_type=Path))
@click.argument("out_dir", type=click.Path(file_okay=False, path_type=Path))
@click.option("--prev-dir", type=click.Path(exists=True, file_okay=False, path_type=Path), default=None,
              help="Directory of the previous step's shard files: apply decoded deltas to them.")
@handle_errors
def batch_decompress(streams_manifest, out_dir, prev_dir):
    """Decode every stream of a streams.jsonl into OUT_DIR/<name> (one batched call;
    names sanitised like the chain's file names)."""
    from .errors import raise_status
    from .stream import default_codec, parse_header

    from .pipeline import read_files_to_device

    rows = [json.loads(r) for r in Path(streams_manifest).read_text().splitlines() if r.strip()]
    base = Path(streams_manifest).parent
    codec = default_codec()
    # the streams read by a thread pool through reused pinned slots,
    # overlapped with their host-to-device copies
    dev_all, offs, lens, heads, errs = read_files_to_device([base / r["file"] for r in rows], codec.device)
    for i, r in enumerate(rows):
        p = base / r["file"]
        if errs[i] is not None:
            if not p.exists():
                raise MissingStreamError(f"stream file {p} is missing")
            raise errs[i]
        h = parse_header(heads[i])
        if h.crc32 != r["crc32"]:
            raise IntegrityError(f"stream {r['file']} CRC does not match the manifest")
    dev = [dev_all[o: o + n] for o, n in zip(offs, lens)]
    prev = None
    if prev_dir is not None:
        prev = []
        for r in rows:
            pd = (Path(prev_dir) / shard_file(r["name"])).read_bytes()
            if len(pd) != r["length"]:
                raise ShapeMismatchError(f"length mismatch: {len(pd)} vs {r['length']}")
            prev.append(_device_bytes(pd))
    res = codec.decompress(dev, prev=prev)
    for i, r in enumerate(rows):
        if res.status[i]:
            raise_status(res.status[i], f"stream {r['file']}: status {res.status[i]}")
        if res.lengths[i] != r["length"]:
            raise CorruptStreamError(f"stream {r['file']} decodes to {res.lengths[i]} bytes, manifest says {r['length']}")
    host = res.data[: (res.offsets[-1] + res.lengths[-1]) if len(res) else 0].cpu().numpy()
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    for i, r in enumerate(rows):
        o, n = res.offsets[i], res.lengths[i]
        (out_dir / shard_file(r["name"])).write_bytes(host[o: o + n].tobytes())
    click.echo(f"restored {len(rows)} shard(s)", err=True)


if __name__ == "__main__":
    main()
