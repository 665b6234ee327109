"""GPU: the fused decode + inverse byte-grouping + CRC (k_decpair) against the
unfused path (k_decrec -> grouped scratch -> k_ungroup) and the oracle.

Fused windows are two-plane (bf16/fp16, byte-grouped) windows whose planes
are a whole number of 16/32/64 KiB blocks (stream.py:332-335, bytegroup.py:
53-62); everything else keeps the unfused path.  Output bytes, statuses and
error classes must not depend on the path (stream.py:392-423)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_09810_b200 as lmcb  # noqa: E402
from paper_2505_09810_b200 import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def codec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = lmcb.Codec()
    c.ctx.set_decode_fusion(True, 0)    # fused at every size (the default starts at 16384 records)
    yield c
    c.ctx.set_decode_fusion(True)


def fallback_segments(codec) -> int:
    return int(codec.ctx.lib.lmcg_fallback_segments(1))


def dev_bytes(b: bytes):
    return torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()


def host_bytes(t) -> bytes:
    return t.cpu().numpy().tobytes()


def both_paths(codec, streams, **kw):
    out = []
    for fuse in (True, False):
        codec.ctx.set_decode_fusion(fuse, 0)
        try:
            out.append(codec.decompress(streams, **kw))
        finally:
            codec.ctx.set_decode_fusion(True, 0)
    return out


def _profiled(codec, fn):
    codec.ctx.profile(True)
    try:
        fn()
    finally:
        rep = codec.ctx.profile_report()
        codec.ctx.profile(False)
    return rep


@pytest.mark.parametrize("block", [16384, 32768, 65536])
@pytest.mark.parametrize("segs", [1, 3])
def test_fused_matches_unfused_and_oracle(codec, block, segs):
    g = torch.Generator(device="cuda").manual_seed(block + segs)
    ts = [(torch.randn(1024, 768, generator=g, device="cuda") * 0.02).to(torch.bfloat16),   # stored low + Huffman high
          (torch.randn(3 * block, generator=g, device="cuda") * 0.02).to(torch.float16),
          torch.zeros(2 * block, dtype=torch.bfloat16, device="cuda"),                      # RLE planes
          (torch.randn(1000, 77, generator=g, device="cuda") * 0.02).to(torch.bfloat16)]    # misaligned: unfused
    b = codec.compress(ts, block_size=block, segment_count=segs)
    streams = b.to_bytes()
    for t, s in zip(ts, streams):
        et = 2 if t.dtype == torch.float16 else 1
        assert s == O.compress(host_bytes(t.view(torch.uint8).reshape(-1)), et, block_size=block, segment_count=segs)
    fallback_segments(codec)
    rf, ru = both_paths(codec, b)
    assert fallback_segments(codec) == 0
    for r in (rf, ru):
        assert r.status == [0] * len(ts)
        for i, t in enumerate(ts):
            assert torch.equal(r.payload(i), t.view(torch.uint8).reshape(-1))


def test_fused_kernel_runs_and_ungroup_skips(codec):
    specs, ts = synth.make_checkpoint("cfg1", seed=11)
    b = codec.compress(ts)
    rep = _profiled(codec, lambda: codec.decompress(b).raise_for_status())
    assert "k_decpair" in rep
    codec.ctx.set_decode_fusion(False, 0)
    try:
        rep2 = _profiled(codec, lambda: codec.decompress(b).raise_for_status())
    finally:
        codec.ctx.set_decode_fusion(True, 0)
    assert "k_decpair" not in rep2


def test_fused_delta_both_planes_huffman_and_apply(codec):
    # cfg4-style XOR deltas: both planes are Huffman records (the second plane
    # decodes into the other half of the ring slot); decode + xor_apply in place
    specs, prev = synth.make_checkpoint("cfg4", seed=21, limit=6)
    nxt = [synth.next_step(w, 21, i) for i, w in enumerate(prev)]
    b = codec.compress(nxt, prev=prev)
    for p, q, s in zip(prev, nxt, b.to_bytes()):
        x = host_bytes((p.view(torch.uint8) ^ q.view(torch.uint8)).reshape(-1))
        assert s == O.compress(x, 1, delta=True, threads=8)
    for fuse in (True, False):
        codec.ctx.set_decode_fusion(fuse, 0)
        try:
            outs = [p.clone() for p in prev]
            r = codec.decompress(b, prev=outs, out=None)
            r.raise_for_status()
            for i, (p, q) in enumerate(zip(prev, nxt)):
                assert torch.equal(r.payload(i), q.view(torch.uint8).reshape(-1)), (fuse, specs[i].name)
        finally:
            codec.ctx.set_decode_fusion(True, 0)


def test_fused_misaligned_output_offsets(codec):
    # an output offset off the 16-byte grid turns fusion off for that stream only
    g = torch.Generator(device="cuda").manual_seed(5)
    ts = [(torch.randn(256, 1024, generator=g, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(3)]
    b = codec.compress(ts)
    n = ts[0].numel() * 2
    out = torch.zeros(3 * n + 64, dtype=torch.uint8, device="cuda")
    offs = [0, n + 3, 2 * n + 32]
    r = codec.decompress(b, out=out, out_offsets=offs)
    r.raise_for_status()
    for i, t in enumerate(ts):
        assert torch.equal(out[offs[i]: offs[i] + n], t.view(torch.uint8).reshape(-1))


def _class(b: bytes) -> int:
    try:
        O.decompress(b)
        return 0
    except O.OracleError as exc:
        return exc.code


def test_fused_corruptions_same_class_both_paths(codec):
    # byte flips in every part of a fused window's records: codebooks, bit
    # counts, Huffman bits, stored bytes (CRC), record headers, segment table
    rng = np.random.default_rng(9)
    g = torch.Generator(device="cuda").manual_seed(9)
    t = (torch.randn(512, 512, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    stream = codec.compress([t], segment_count=2).to_bytes()[0]
    assert _class(stream) == 0
    bads = []
    positions = list(range(0, 200)) + list(rng.integers(0, len(stream), 150))
    for pos in positions:
        bad = bytearray(stream)
        bad[int(pos)] ^= int(rng.integers(1, 256))
        bads.append(bytes(bad))
    want = [_class(x) for x in bads]
    rf, ru = both_paths(codec, [dev_bytes(x) for x in bads])
    assert rf.status == want
    assert ru.status == want
    for i, w in enumerate(want):
        if w == 0:   # accepted flips (e.g. padding bits) decode to the same payload
            assert torch.equal(rf.payload(i), t.view(torch.uint8).reshape(-1))


def test_fused_full_cfg2_and_cfg3(codec):
    for cfg, seed in (("cfg2", 2), ("cfg3", 3)):
        specs, ts = synth.make_checkpoint(cfg, seed=seed)
        b = codec.compress(ts)
        fallback_segments(codec)
        rf, ru = both_paths(codec, b)
        assert fallback_segments(codec) == 0
        for r in (rf, ru):
            assert r.status == [0] * len(ts)
            for i, t in enumerate(ts):
                assert torch.equal(r.payload(i), t.view(torch.uint8).reshape(-1)), specs[i].name


@pytest.mark.parametrize("graph", [False, True])
def test_fused_plans(codec, graph):
    specs, ts = synth.make_checkpoint("cfg2", seed=17, limit=40)
    plan = codec.compress_plan(ts, graph=graph)
    dplan = plan.decompress_plan(graph=graph)
    b = plan.run()
    r = dplan.run(b)
    assert r.status == [0] * len(ts)
    for i, t in enumerate(ts):
        assert torch.equal(r.payload(i), t.view(torch.uint8).reshape(-1))
