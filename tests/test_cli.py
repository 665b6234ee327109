"""CLI front-end and the overlapped write pipeline.

The GPU cases follow the reference's own CLI suite (pkg/tests/test_cli.py:
TestCompressDecompress :33-94 and TestCheckpointCommands :97-147) on the GPU
path, and additionally check every stream the CLI writes byte for byte
against the oracle (the reference's algorithm restated in C).  The CPU cases
cover what runs before any device work: argument / alignment / format errors
and their stable exit codes, manifest parsing and pipeline grouping.
"""
from __future__ import annotations

import json

import numpy as np
import pytest
from click.testing import CliRunner

from oracle import oracle


def _trajectory(n_elem: int, steps: int, seed: int) -> list[bytes]:
    """bf16 steps: w ~ N(0, 0.02), each next step w + N(0, 1e-3 |w| + 1e-6) (cfg4's noise model)."""
    rng = np.random.default_rng(seed)
    w = rng.normal(0, 0.02, n_elem).astype(np.float32)
    out = []
    for _ in range(steps):
        b = (w.view(np.uint32) + 0x7FFF + ((w.view(np.uint32) >> 16) & 1)) >> 16   # round to nearest even
        out.append(b.astype(np.uint16).tobytes())
        w = (w + rng.normal(0, 1, n_elem).astype(np.float32) * (1e-3 * np.abs(w) + 1e-6)).astype(np.float32)
    return out


@pytest.fixture
def runner():
    return CliRunner()


@pytest.fixture
def step_files(tmp_path):
    paths = []
    for i, s in enumerate(_trajectory(20_000, 6, seed=5)):
        p = tmp_path / f"step{i}.bin"
        p.write_bytes(s)
        paths.append(p)
    return paths


def _main():
    from paper_2505_09810_b200.cli import main
    return main


def _run(runner, args, **kw):
    return runner.invoke(_main(), args, catch_exceptions=False, **kw)


# ------------------------------------------------------------------ no GPU needed
def test_alignment_error_exits_2(runner, tmp_path):
    odd = tmp_path / "odd.bin"
    odd.write_bytes(bytes(1001))
    r = runner.invoke(_main(), ["compress", "--dtype", "fp32", str(odd), str(tmp_path / "x.lmc")])
    assert r.exit_code == 2
    assert "not a multiple" in r.output


def test_wrong_magic_exits_3(runner, tmp_path):
    bogus = tmp_path / "bogus.lmc"
    bogus.write_bytes(b"NOPE" + bytes(64))
    r = runner.invoke(_main(), ["decompress", str(bogus), str(tmp_path / "o")])
    assert r.exit_code == 3
    assert "magic" in r.output


def test_bad_block_size_exits_6(runner, tmp_path, step_files):
    r = runner.invoke(_main(), ["compress", "--dtype", "bf16", "--block-size", "100", "--threads", "1",
                                str(step_files[0]), str(tmp_path / "x.lmc")])
    assert r.exit_code == 6


def test_delta_length_mismatch_exits_4(runner, tmp_path, step_files):
    short = tmp_path / "short.bin"
    short.write_bytes(step_files[0].read_bytes()[:-4])
    r = runner.invoke(_main(), ["compress", "--dtype", "bf16", "--delta", str(short), str(step_files[1]),
                                str(tmp_path / "x.lmc")])
    assert r.exit_code == 4


def test_restore_without_manifest_exits_5(runner, tmp_path):
    (tmp_path / "empty_chain").mkdir()
    r = runner.invoke(_main(), ["checkpoint", "restore", str(tmp_path / "empty_chain"), "0", str(tmp_path / "o")])
    assert r.exit_code == 5


def test_exit_code_table():
    from paper_2505_09810_b200 import errors as E
    from paper_2505_09810_b200.cli import exit_code

    assert exit_code(E.AlignmentError("x")) == 2 and exit_code(E.EmptyInputError("x")) == 2
    assert exit_code(E.CorruptStreamError("x")) == 3 and exit_code(E.IntegrityError("x")) == 3
    assert exit_code(E.UnsupportedFormatError("x")) == 3
    assert exit_code(E.ShapeMismatchError("x")) == 4 and exit_code(E.DtypeMismatchError("x")) == 4
    assert exit_code(E.MissingStreamError("x")) == 5 and exit_code(FileNotFoundError("x")) == 5
    assert exit_code(E.ConfigError("x")) == 6
    assert exit_code(E.DeviceError("x")) == 1 and exit_code(OSError("x")) == 1


def test_jsonl_shard_manifest_parsing(tmp_path, step_files):
    from paper_2505_09810_b200.cli import read_step_shards
    from paper_2505_09810_b200.types import ElementType

    spec = tmp_path / "ckpt.jsonl"
    spec.write_text(json.dumps({"name": "w", "dtype": "bf16", "path": step_files[0].name}) + "\n\n"
                    + json.dumps({"name": "b", "path": str(step_files[1])}) + "\n")
    shards = read_step_shards([spec], "raw")
    assert sorted(shards) == ["b", "w"]
    assert shards["w"].element_type is ElementType.BF16 and shards["b"].element_type is ElementType.RAW8
    assert shards["w"].data == step_files[0].read_bytes()


def test_pipeline_groups():
    from paper_2505_09810_b200.pipeline import _groups

    assert _groups([], 10) == []
    assert _groups([4, 4, 4], 10) == [[0, 1], [2]]
    assert _groups([30, 1, 1], 10) == [[0], [1, 2]]
    assert _groups([10, 10], 10) == [[0], [1]]
    assert sum(_groups([3] * 50, 7), []) == list(range(50))


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
class TestCompressDecompressGPU:
    def test_round_trip_matches_oracle(self, runner, tmp_path, step_files):
        out, back = tmp_path / "a.lmc", tmp_path / "a.out"
        r = _run(runner, ["compress", "--dtype", "bf16", "--threads", "2", str(step_files[0]), str(out)])
        assert r.exit_code == 0 and "ratio=" in r.output and "MiB/s=" in r.output
        assert out.read_bytes() == oracle.compress(step_files[0].read_bytes(), 1, segment_count=2)
        r = _run(runner, ["decompress", str(out), str(back)])
        assert r.exit_code == 0
        assert back.read_bytes() == step_files[0].read_bytes()

    def test_no_bytegroup_clears_flag(self, runner, tmp_path, step_files):
        from paper_2505_09810_b200.stream import parse_header

        out = tmp_path / "nbg.lmc"
        assert _run(runner, ["compress", "--dtype", "bf16", "--no-bytegroup", "--threads", "1",
                             str(step_files[0]), str(out)]).exit_code == 0
        assert not parse_header(out.read_bytes()).byte_grouped
        assert out.read_bytes() == oracle.compress(step_files[0].read_bytes(), 1, byte_group=False)

    def test_delta_flag_compresses_xor(self, runner, tmp_path, step_files):
        from paper_2505_09810_b200.stream import parse_header

        out = tmp_path / "d.lmc"
        r = _run(runner, ["compress", "--dtype", "bf16", "--threads", "1", "--delta", str(step_files[0]),
                          str(step_files[1]), str(out)])
        assert r.exit_code == 0
        assert parse_header(out.read_bytes()).delta_applied
        x = (np.frombuffer(step_files[0].read_bytes(), np.uint8) ^ np.frombuffer(step_files[1].read_bytes(), np.uint8))
        assert out.read_bytes() == oracle.compress(x.tobytes(), 1, delta=True)

    def test_truncated_stream_exits_3(self, runner, tmp_path, step_files):
        out = tmp_path / "t.lmc"
        _run(runner, ["compress", "--dtype", "bf16", str(step_files[0]), str(out)])
        out.write_bytes(out.read_bytes()[:-5])
        assert runner.invoke(_main(), ["decompress", str(out), str(tmp_path / "t.out")]).exit_code == 3

    def test_lmc_threads_env(self, runner, tmp_path, step_files, monkeypatch):
        from paper_2505_09810_b200.stream import parse_header

        monkeypatch.setenv("LMC_THREADS", "3")
        out = tmp_path / "env.lmc"
        assert _run(runner, ["compress", "--dtype", "bf16", str(step_files[0]), str(out)]).exit_code == 0
        assert parse_header(out.read_bytes()).segment_count == 3

    def test_rerun_is_idempotent(self, runner, tmp_path, step_files):
        out = tmp_path / "i.lmc"
        _run(runner, ["compress", "--dtype", "bf16", "--threads", "2", str(step_files[0]), str(out)])
        first = out.read_bytes()
        _run(runner, ["compress", "--dtype", "bf16", "--threads", "2", str(step_files[0]), str(out)])
        assert out.read_bytes() == first


@pytest.mark.gpu
class TestCheckpointCommandsGPU:
    def _shard_file(self, tmp_path, i, data):
        d = tmp_path / f"in{i}"
        d.mkdir(exist_ok=True)
        p = d / "weights.bin"
        p.write_bytes(data)
        return p

    def test_chain_add_restore(self, runner, tmp_path, step_files):
        chain = tmp_path / "chain"
        for i, f in enumerate(step_files):
            p = self._shard_file(tmp_path, i, f.read_bytes())
            r = _run(runner, ["checkpoint", "add", "--dtype", "bf16", str(chain), str(p)])
            assert r.exit_code == 0, r.output
        # every stream file is the oracle's stream of the same (delta) payload
        for i in range(len(step_files)):
            data = np.frombuffer(step_files[i].read_bytes(), np.uint8)
            if i:
                data = data ^ np.frombuffer(step_files[i - 1].read_bytes(), np.uint8)
            assert (chain / ("step%06d_weights.bin.lmc" % i)).read_bytes() == \
                oracle.compress(data.tobytes(), 1, delta=i > 0)
        outdir = tmp_path / "restored"
        assert _run(runner, ["checkpoint", "restore", str(chain), "5", str(outdir)]).exit_code == 0
        assert (outdir / "weights.bin").read_bytes() == step_files[5].read_bytes()

    def test_shape_change_exits_4(self, runner, tmp_path, step_files):
        chain = tmp_path / "chain"
        p0 = self._shard_file(tmp_path, 0, step_files[0].read_bytes())
        _run(runner, ["checkpoint", "add", "--dtype", "bf16", str(chain), str(p0)])
        p1 = self._shard_file(tmp_path, 1, step_files[1].read_bytes()[:-4])
        assert runner.invoke(_main(), ["checkpoint", "add", "--dtype", "bf16", str(chain), str(p1)]).exit_code == 4

    def test_missing_stream_exits_5(self, runner, tmp_path, step_files):
        chain = tmp_path / "chain"
        for i in range(3):
            p = self._shard_file(tmp_path, i, step_files[i].read_bytes())
            _run(runner, ["checkpoint", "add", "--dtype", "bf16", str(chain), str(p)])
        next(chain.glob("step000001_*.lmc")).unlink()
        r = runner.invoke(_main(), ["checkpoint", "restore", str(chain), "2", str(tmp_path / "o")])
        assert r.exit_code == 5

    def test_jsonl_manifest_input(self, runner, tmp_path, step_files):
        chain = tmp_path / "chain"
        for i in range(2):
            spec = tmp_path / f"ckpt{i}.jsonl"
            spec.write_text(json.dumps({"name": "w", "dtype": "bf16", "path": step_files[i].name}) + "\n")
            assert _run(runner, ["checkpoint", "add", str(chain), str(spec)]).exit_code == 0
        outdir = tmp_path / "r"
        assert _run(runner, ["checkpoint", "restore", str(chain), "1", str(outdir)]).exit_code == 0
        assert (outdir / "w").read_bytes() == step_files[1].read_bytes()


def _shards(tmp_path, step: int, n: int, seed: int):
    """A JSONL manifest of n bf16 shards of mixed sizes (some empty, some RLE)."""
    rng = np.random.default_rng(seed)
    rows, data = [], {}
    for k in range(n):
        ne = int(rng.choice([0, 1, 777, 5000, 70_000, 300_000]))
        v = (rng.normal(0, 0.02, ne).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        if k % 7 == 3:
            v[:] = 0
        name = f"layer.{k}/weight"
        p = tmp_path / f"s{step}_{k}.bin"
        p.write_bytes(v.tobytes())
        rows.append(json.dumps({"name": name, "dtype": "bf16", "path": p.name}))
        data[name] = v.tobytes()
    spec = tmp_path / f"step{step}.jsonl"
    spec.write_text("\n".join(rows) + "\n")
    return spec, data


@pytest.mark.gpu
def test_batch_compress_decompress(runner, tmp_path):
    spec, data = _shards(tmp_path, 0, 23, seed=3)
    out = tmp_path / "out"
    r = _run(runner, ["batch", "compress", str(spec), str(out), "--group-mib", "1"])
    assert r.exit_code == 0, r.output
    rows = [json.loads(x) for x in (out / "streams.jsonl").read_text().splitlines()]
    assert [x["name"] for x in rows] == sorted(data)
    for x in rows:
        s = (out / x["file"]).read_bytes()
        assert len(s) == x["stream_bytes"]
        assert s == oracle.compress(data[x["name"]], 1)
    back = tmp_path / "back"
    assert _run(runner, ["batch", "decompress", str(out / "streams.jsonl"), str(back)]).exit_code == 0
    for x in rows:
        assert (back / x["name"].replace("/", "_")).read_bytes() == data[x["name"]]


@pytest.mark.gpu
def test_stream_writer_groups_match_one_batch(tmp_path):
    """Many groups and rotating slots (group_bytes far below the checkpoint):
    every file equals the one-call batch's stream and the oracle's."""
    import torch

    from paper_2505_09810_b200 import default_codec
    from paper_2505_09810_b200.pipeline import write_streams

    g = torch.Generator(device="cuda").manual_seed(11)
    sizes = [0, 1, 4096, 65536, 200_000, 3, 131072, 1 << 20, 17, 99_999] * 3
    ts = [(torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16) for n in sizes]
    prev = [(t.float() + 1e-3 * torch.randn(t.shape, device="cuda", generator=g) * t.float().abs()).to(torch.bfloat16)
            for t in ts]
    for use_prev in (False, True):
        paths = [tmp_path / f"{use_prev}_{i}.lmc" for i in range(len(ts))]
        lens = write_streams(ts, paths, prev=prev if use_prev else None, group_bytes=300_000, depth=3)
        one = default_codec().compress(ts, prev=prev if use_prev else None).to_bytes()
        for i, p in enumerate(paths):
            assert p.read_bytes() == one[i] and lens[i] == len(one[i])
        for i in (2, 4, 7):
            x = ts[i].view(torch.uint8).cpu().numpy()
            if use_prev:
                x = x ^ prev[i].view(torch.uint8).cpu().numpy()
            assert one[i] == oracle.compress(x.tobytes(), 1, delta=use_prev)


@pytest.mark.gpu
def test_stream_writer_sink_error_propagates(tmp_path):
    import torch

    from paper_2505_09810_b200.pipeline import StreamWriter, items_from_tensors

    ts = [torch.zeros(100_000, dtype=torch.bfloat16, device="cuda") for _ in range(8)]

    def sink(i, view):
        if i == 5:
            raise OSError("disk full")

    with pytest.raises(OSError, match="disk full"):
        StreamWriter(group_bytes=200_000).run(items_from_tensors(ts), sink)



@pytest.mark.gpu
@pytest.mark.parametrize("slot", [4096, 64 << 20])
def test_read_files_to_device(tmp_path, slot):
    """Files through the two reused pinned slots: sizes across slot edges,
    empty and missing files, headers for the host-side checks."""
    import torch

    from paper_2505_09810_b200.pipeline import read_files_to_device

    rng = np.random.default_rng(7)
    paths, blobs = [], []
    for i, n in enumerate([0, 1, 15, 16, 17, 4096, 100_003, 0, 333, 9000]):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        p = tmp_path / f"f{i}.lmc"
        p.write_bytes(b)
        paths.append(p)
        blobs.append(b)
    paths.insert(3, tmp_path / "missing.lmc")
    blobs.insert(3, None)
    dev, offs, lens, heads, errs = read_files_to_device(paths, torch.device("cuda", 0), slot_bytes=slot, threads=4)
    data = dev.cpu().numpy()
    for i, b in enumerate(blobs):
        assert offs[i] % 16 == 0
        if b is None:
            assert isinstance(errs[i], FileNotFoundError) and lens[i] == 0
        else:
            assert errs[i] is None and lens[i] == len(b) and heads[i] == b[:64]
            assert data[offs[i]: offs[i] + lens[i]].tobytes() == b


@pytest.mark.gpu
def test_batch_delta_and_prev_dir(runner, tmp_path):
    """batch compress --delta (XOR against the previous step's manifest) and
    batch decompress --prev-dir (decode fused with xor_apply) restore step 1."""
    steps = _trajectory(50_000, 2, seed=9)
    for i, s in enumerate(steps):
        (tmp_path / f"a{i}.bin").write_bytes(s)
        (tmp_path / f"b{i}.bin").write_bytes(s[::-1])
        (tmp_path / f"m{i}.jsonl").write_text(
            json.dumps({"name": "a", "dtype": "bf16", "path": f"a{i}.bin"}) + "\n"
            + json.dumps({"name": "b", "dtype": "bf16", "path": f"b{i}.bin"}) + "\n")
    out = tmp_path / "d"
    r = _run(runner, ["batch", "compress", str(tmp_path / "m1.jsonl"), str(out), "--delta", str(tmp_path / "m0.jsonl")])
    assert r.exit_code == 0, r.output
    rows = {x["name"]: x for x in map(json.loads, (out / "streams.jsonl").read_text().splitlines())}
    for name, s0, s1 in (("a", steps[0], steps[1]), ("b", steps[0][::-1], steps[1][::-1])):
        x = (np.frombuffer(s0, np.uint8) ^ np.frombuffer(s1, np.uint8)).tobytes()
        assert rows[name]["delta"] and (out / rows[name]["file"]).read_bytes() == oracle.compress(x, 1, delta=True)
    prev = tmp_path / "prev"
    prev.mkdir()
    (prev / "a").write_bytes(steps[0])
    (prev / "b").write_bytes(steps[0][::-1])
    back = tmp_path / "back"
    r = _run(runner, ["batch", "decompress", str(out / "streams.jsonl"), str(back), "--prev-dir", str(prev)])
    assert r.exit_code == 0, r.output
    assert (back / "a").read_bytes() == steps[1] and (back / "b").read_bytes() == steps[1][::-1]
