"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
golden fixtures produced by the live reference.  Bit-exact everywhere."""
import numpy as np
import pytest

from conftest import load_golden_codebooks, load_golden_corruptions, load_golden_streams

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_09810_b200 as lmcb  # noqa: E402
from paper_2505_09810_b200 import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402

ET = lmcb.ElementType


@pytest.fixture(scope="module")
def codec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return lmcb.Codec()


def fallback_segments(codec) -> int:
    """Segments the serial fallback walked since the last call (resets)."""
    return int(codec.ctx.lib.lmcg_fallback_segments(1))


def dev_bytes(b: bytes):
    if not b:
        return torch.empty(0, dtype=torch.uint8, device="cuda")
    return torch.frombuffer(bytearray(b), dtype=torch.uint8).cuda()


def host_bytes(t) -> bytes:
    return t.cpu().numpy().tobytes()


# ------------------------------------------------------------------ golden
@pytest.mark.parametrize("case", load_golden_streams(), ids=lambda c: c[0]["name"])
def test_golden_stream_bytes(codec, case):
    m, data, stream = case
    b = codec.compress([dev_bytes(data)], element_types=[m["element_type"]], delta=m["delta"],
                       byte_group=m["byte_group"], block_size=m["block_size"],
                       segment_count=m["segment_count"], buffer_size=m["buffer_size"])
    assert b.to_bytes()[0] == stream


@pytest.mark.parametrize("case", load_golden_streams(), ids=lambda c: c[0]["name"])
def test_golden_stream_decode(codec, case):
    m, data, stream = case
    fallback_segments(codec)
    r = codec.decompress([dev_bytes(stream)])
    assert r.status == [0]
    assert fallback_segments(codec) == 0   # reference streams decode on the parallel path
    assert r.lengths[0] == len(data)
    assert host_bytes(r.payload(0)) == data
    assert r.element_types[0] == m["element_type"]


def test_golden_codebooks():
    hists, lengths = load_golden_codebooks()
    got = lmcb.build_codebooks(hists.astype(np.int64))
    assert (got == lengths).all()


def test_golden_corruption_classes(codec):
    streams = {m["name"]: (d, s) for m, d, s in load_golden_streams()}
    cases = load_golden_corruptions()
    bads, wants = [], []
    for c in cases:
        data, s = streams[c["case"]]
        if c["kind"] == "xor":
            bad = bytearray(s)
            bad[c["pos"]] ^= c["val"]
        elif c["kind"] == "truncate":
            bad = s[: c["pos"]]
        else:
            bad = s + b"\x00"
        bads.append(bytes(bad))
        wants.append(c["result"])
    r = codec.decompress([dev_bytes(b) for b in bads])
    names = {0: "ok", 1: "UnsupportedFormatError", 2: "CorruptStreamError", 3: "IntegrityError"}
    got = [names[s] for s in r.status]
    assert got == wants


# ---------------------------------------------------------------- configs
def _oracle_streams(tensors, ets, **opts):
    return [O.compress(host_bytes(t.view(torch.uint8).reshape(-1)), et, threads=8, **opts)
            for t, et in zip(tensors, ets)]


def test_cfg1_full_parity(codec):
    specs, ts = synth.make_checkpoint("cfg1", seed=1)
    b = codec.compress(ts)
    got = b.to_bytes()
    want = _oracle_streams(ts, [1])
    assert got == want
    info = codec.block_info()
    grouped = O.group_bytes(host_bytes(ts[0].view(torch.uint8).reshape(-1)), 2)
    modes, bits, sizes, lengths, pm = O.analyze_blocks(grouped, 65536)
    assert (info["modes"] == modes).all()
    assert (info["sizes"] == sizes).all()
    huff = modes == 0
    assert (info["bits"][huff] == bits[huff]).all()
    assert (info["lengths"][huff] == lengths[huff]).all()
    assert pm.sum() > 0  # package-merge blocks are part of this config
    fallback_segments(codec)
    r = codec.decompress(b)
    assert r.status == [0]
    assert fallback_segments(codec) == 0
    assert torch.equal(r.payload(0), ts[0].view(torch.uint8).reshape(-1))


def test_cfg2_gpt2_small_parity(codec):
    specs, ts = synth.make_checkpoint("cfg2", seed=2)
    assert len(ts) == 148
    b = codec.compress(ts)
    got = b.to_bytes()
    want = _oracle_streams(ts, [1] * len(ts))
    assert [len(x) for x in got] == [len(x) for x in want]
    assert got == want
    fallback_segments(codec)
    r = codec.decompress(b)
    assert r.status == [0] * len(ts)
    assert fallback_segments(codec) == 0
    for i, t in enumerate(ts):
        assert torch.equal(r.payload(i), t.view(torch.uint8).reshape(-1)), specs[i].name


def test_cfg3_rle_heavy_parity(codec):
    specs, ts = synth.make_checkpoint("cfg3", seed=3)
    b = codec.compress(ts)
    got = b.to_bytes()
    want = _oracle_streams(ts, [1, 1])
    assert got == want
    assert len(got[1]) == 236  # 28 + 16 + 32 x 6-byte RLE records
    fallback_segments(codec)
    r = codec.decompress(b)
    assert r.status == [0, 0]
    assert fallback_segments(codec) == 0
    for i, t in enumerate(ts):
        assert torch.equal(r.payload(i), t.view(torch.uint8).reshape(-1))


def test_cfg4_delta_fused_xor_parity(codec):
    # three layers of the 1.3B model (embedding window is misaligned: 2 windows)
    specs, prev = synth.make_checkpoint("cfg4", seed=4, limit=14)
    nxt = [synth.next_step(w, 4, i) for i, w in enumerate(prev)]
    b = codec.compress(nxt, prev=prev)
    got = b.to_bytes()
    xors = [(p.view(torch.uint8) ^ q.view(torch.uint8)).reshape(-1) for p, q in zip(prev, nxt)]
    want = [O.compress(host_bytes(x), 1, delta=True, threads=8) for x in xors]
    assert got == want
    fallback_segments(codec)
    r = codec.decompress(b)
    assert r.status == [0] * len(nxt)
    assert fallback_segments(codec) == 0   # false candidates in delta payloads are resolved
    for i, x in enumerate(xors):
        assert torch.equal(r.payload(i), x)


@pytest.mark.parametrize("segs", [1, 4, 8, 16])
@pytest.mark.parametrize("bg", [True, False])
def test_options_matrix(codec, segs, bg):
    g = torch.Generator(device="cuda").manual_seed(segs * 3 + bg)
    ts = [
        (torch.randn(300_001, generator=g, device="cuda") * 0.02).to(torch.bfloat16),
        torch.randn(70_003, generator=g, device="cuda").to(torch.float32),
        torch.randn(65_536, generator=g, device="cuda").to(torch.float16),
        (torch.rand(100_000, generator=g, device="cuda") ** 4 * 255).to(torch.uint8),
    ]
    for bs, buf in [(4096, 3 * 4096 + 1000), (65536, 128 << 20), (8192, 8192)]:
        b = codec.compress(ts, byte_group=bg, block_size=bs, segment_count=segs, buffer_size=buf)
        got = b.to_bytes()
        want = [O.compress(host_bytes(t.view(torch.uint8).reshape(-1)), et, byte_group=bg, block_size=bs,
                           segment_count=segs, buffer_size=buf, threads=8) for t, et in zip(ts, [1, 3, 2, 0])]
        assert got == want, (bs, buf)
        r = codec.decompress(b)
        assert r.status == [0] * len(ts)
        for i, t in enumerate(ts):
            assert torch.equal(r.payload(i), t.view(torch.uint8).reshape(-1))


def test_unaligned_device_views(codec):
    base = (torch.randn(200_000, device="cuda") * 0.02).to(torch.bfloat16)
    t = base[3:150_003]  # 6-byte offset: no 16-byte vector loads
    b = codec.compress([t])
    assert b.to_bytes()[0] == O.compress(host_bytes(t.contiguous().view(torch.uint8)), 1)


# ------------------------------------------------- reference suite mirrors
def test_boundary_sizes_round_trip(rng):
    # test_stream.py:82-96 through the reference-shaped API
    for size in [0, 1, 4095, 4096, 4097, 65536, 200_000]:
        data = rng.integers(0, 256, size, dtype=np.uint8).tobytes()
        for et in (ET.RAW8, ET.FP32):
            if size % et.width:
                continue
            for bg in (True, False):
                s = lmcb.lmc_compress(lmcb.TensorBuffer(data, et), byte_group=bg, block_size=4096)
                assert s == O.compress(data, et.code, byte_group=bg, block_size=4096)
                out = lmcb.lmc_decompress(s)
                assert out.data == data and out.element_type is et


def test_reference_strictness_cases():
    s = lmcb.lmc_compress(lmcb.TensorBuffer(b"strict header checks", ET.RAW8))
    for pos, value in [(5, 0x84), (7, 1)]:
        bad = bytearray(s)
        bad[pos] = value
        with pytest.raises(lmcb.CorruptStreamError):
            lmcb.lmc_decompress(bytes(bad))
    with pytest.raises(lmcb.UnsupportedFormatError):
        lmcb.lmc_decompress(b"XLC1" + s[4:])
    with pytest.raises(lmcb.CorruptStreamError):
        lmcb.lmc_decompress(s + b"\x00")
    for et in ET:
        e = lmcb.lmc_compress(lmcb.TensorBuffer(b"", et))
        assert len(e) == 28 and lmcb.lmc_decompress(e).data == b""


def test_single_byte_corruptions_never_silent(rng):
    # test_stream.py:170-187
    data = (rng.random(30_000) ** 2 * 256).astype(np.uint8).tobytes()
    stream = lmcb.lmc_compress(lmcb.TensorBuffer(data, ET.BF16), block_size=4096)
    codec = lmcb.stream.default_codec()
    bads = []
    for pos in list(range(0, len(stream), 113)) + list(rng.integers(0, len(stream), 120)):
        bad = bytearray(stream)
        bad[pos] ^= int(rng.integers(1, 256))
        bads.append(bytes(bad))
    r = codec.decompress([dev_bytes(b) for b in bads])
    for i, b in enumerate(bads):
        try:
            O.decompress(b)
            want = 0
        except O.OracleError as exc:
            want = exc.code
        assert r.status[i] == want
    assert all(s != 0 for s in r.status)


def test_cross_decode_gpu_stream_by_oracle(codec):
    ts = [(torch.randn(1 << 20, device="cuda") * 0.02).to(torch.bfloat16)]
    b = codec.compress(ts, segment_count=3)
    out, et, flags = O.decompress(b.to_bytes()[0])
    assert out == host_bytes(ts[0].view(torch.uint8)) and et == 1 and flags == 1


# ------------------------------------------------------------------- plans
@pytest.mark.parametrize("graph", [False, True])
def test_plans_match_oracle_and_round_trip(codec, graph):
    specs, ts = synth.make_checkpoint("cfg2", seed=7, limit=30)
    plan = codec.compress_plan(ts, graph=graph)
    dplan = plan.decompress_plan(graph=graph)
    for it in range(2):
        if it == 1:  # new contents, same tensors: replay must pick them up
            for t in ts:
                t.mul_(-1.5)
        b = plan.run()
        got = b.to_bytes()
        want = _oracle_streams(ts, [1] * len(ts))
        assert got == want
        r = dplan.run(b)
        assert r.status == [0] * len(ts)
        for i, t in enumerate(ts):
            assert torch.equal(r.payload(i), t.view(torch.uint8).reshape(-1))


def test_plan_delta_fused(codec):
    specs, prev = synth.make_checkpoint("cfg4", seed=8, limit=4)
    nxt = [synth.next_step(w, 8, i) for i, w in enumerate(prev)]
    plan = codec.compress_plan(nxt, prev=prev)
    b = plan.run()
    want = [O.compress(host_bytes((p.view(torch.uint8) ^ q.view(torch.uint8)).reshape(-1)), 1, delta=True, threads=8)
            for p, q in zip(prev, nxt)]
    assert b.to_bytes() == want


def test_false_candidates_inside_payload(codec):
    # Raw stored blocks that contain fake record headers "mode|len==block" (and a
    # fake successor header) must still decode exactly: the scan's candidates
    # are only hints, verification + the serial walk decide.
    B = 4096
    rng = np.random.default_rng(3)
    data = bytearray(rng.integers(0, 256, 40 * B, dtype=np.uint8).tobytes())
    fake = bytes([2]) + B.to_bytes(4, "little")
    for k in range(1, 39, 3):
        off = k * B + 100
        data[off: off + 5] = fake                      # fake stored header
        nxt = off + 5 + B
        data[nxt: nxt + 5] = bytes([0]) + B.to_bytes(4, "little")  # fake successor
    data = bytes(data)
    t = dev_bytes(data)
    b = codec.compress([t], element_types=[0], byte_group=False, block_size=B)
    assert b.to_bytes()[0] == O.compress(data, 0, byte_group=False, block_size=B)
    r = codec.decompress(b)
    assert r.status == [0] and host_bytes(r.payload(0)) == data


def test_false_stored_grid_inside_payload(codec):
    # k_cand's stored-grid shortcut trusts full stored headers on the (B + 5)
    # grid from the segment start.  Here the first record is RLE (6 bytes), so
    # every real record is off the grid, while the stored payloads carry fake
    # "stored | B" headers exactly on it: spans take the shortcut, miss the
    # real record starts, the chain does not verify and the serial walk
    # decides.  The payload must still come back exactly.
    B = 4096
    rng = np.random.default_rng(11)
    data = bytearray(rng.integers(0, 256, 40 * B, dtype=np.uint8).tobytes())
    data[0:B] = bytes(B)                               # block 0: RLE record
    fake = bytes([2]) + B.to_bytes(4, "little")
    for k in range(1, 40):
        # grid position k (B + 5) lies 4095 bytes into record k: payload offset 4090
        data[k * B + 4090: k * B + 4095] = fake
    data = bytes(data)
    s = O.compress(data, 0, byte_group=False, block_size=B)
    G = B + 5
    seg0 = s.index(bytes([1]) + B.to_bytes(4, "little") + b"\x00")   # the RLE record = segment start
    assert all(s[seg0 + k * G: seg0 + k * G + 5] == fake for k in range(1, 39))
    b = codec.compress([dev_bytes(data)], element_types=[0], byte_group=False, block_size=B)
    assert b.to_bytes()[0] == s
    fallback_segments(codec)
    r = codec.decompress(b)
    assert r.status == [0] and host_bytes(r.payload(0)) == data
    assert fallback_segments(codec) == 1
    # and the real shape of the shortcut: every block stored, records on the grid
    data2 = rng.integers(0, 256, 40 * B, dtype=np.uint8).tobytes()
    b2 = codec.compress([dev_bytes(data2)], element_types=[0], byte_group=False, block_size=B)
    assert b2.to_bytes()[0] == O.compress(data2, 0, byte_group=False, block_size=B)
    r2 = codec.decompress(b2)
    assert r2.status == [0] and host_bytes(r2.payload(0)) == data2
    assert fallback_segments(codec) == 0


@pytest.mark.parametrize("et", [ET.RAW8, ET.BF16, ET.FP32])
@pytest.mark.parametrize("density", [0.002, 0.03, 0.2])
def test_run_symbol_paths(codec, et, density):
    """Blocks with a 1-bit code (the encoder's and decoder's run paths):
    sparse byte streams of every width, aligned and unaligned device views,
    plain and as fused XOR deltas, against the oracle byte for byte."""
    g = np.random.default_rng(int(density * 1e4) + et.code)
    n = 3 * 65536 + 4 * 4099
    base = np.zeros(n + 64, np.uint8)
    hits = g.random(n + 64) < density
    base[hits] = g.integers(1, 256, int(hits.sum()), dtype=np.uint8)
    prev = g.integers(0, 256, n + 64, dtype=np.uint8)
    dev = torch.from_numpy(base).cuda()
    fallback_segments(codec)
    for off in (0, et.width * 3):   # 16-byte aligned view, and one that is not
        size = (n // et.width) * et.width
        x = base[off: off + size]
        t = dev[off: off + size]
        for block in (4096, 65536):
            b = codec.compress([t], element_types=[et.code], block_size=block)
            s = b.to_bytes()[0]
            assert s == O.compress(x.tobytes(), et.code, block_size=block), (off, block)
            r = codec.decompress(b)
            r.raise_for_status()
            assert torch.equal(r.payload(0), t)
        # delta: cur = prev ^ sparse, so the delta stream encodes the sparse bytes
        p = torch.from_numpy(prev[:size].copy()).cuda()
        cur = p ^ t
        b = codec.compress([cur], element_types=[et.code], prev=[p])
        assert b.to_bytes()[0] == O.compress(x.tobytes(), et.code, delta=True)
        r = codec.decompress(b, prev=[p])
        r.raise_for_status()
        assert torch.equal(r.payload(0), cur)
    assert fallback_segments(codec) == 0


def _near_threshold_bytes(rng, n_blocks: int, block: int) -> bytes:
    """raw8 blocks whose Huffman cost straddles the stored record: a skewed
    byte distribution (p ~ exp(-a i / 256)) with a swept over [0, 3) from
    near-uniform (stored) through the decision boundary (a ~ 2.2 for 4 KiB
    blocks, ~ 1 for 64 KiB: the 132-byte codebook overhead) to clearly
    compressible, plus fully uniform and 100-symbol blocks."""
    out = []
    for j in range(n_blocks):
        a = 3.0 * j / n_blocks
        if j % 7 == 3:
            x = rng.integers(0, 256, block, dtype=np.uint8)
        elif j % 7 == 5:
            x = rng.integers(0, 100, block, dtype=np.uint8)
        else:
            p = np.exp(-a * np.arange(256) / 256.0)
            x = rng.choice(256, size=block, p=p / p.sum()).astype(np.uint8)
        out.append(x.tobytes())
    return b"".join(out)


@pytest.mark.parametrize("block", [4096, 65536, 262144, 1 << 20])
def test_mode_decision_boundary(codec, rng, block):
    """Stored / Huffman decisions near the boundary (k_codebook's deferred
    lane-per-block cost pass, its u16 columns only for blocks <= 64 KiB, the
    float entropy bound): streams and per-block modes equal the oracle's."""
    nb = {4096: 96, 65536: 48, 262144: 12, 1 << 20: 4}[block]
    data = _near_threshold_bytes(rng, nb, block)
    b = codec.compress([dev_bytes(data)], element_types=[0], block_size=block)
    assert b.to_bytes()[0] == O.compress(data, 0, block_size=block, threads=8)
    info = codec.block_info()
    modes, bits, sizes, lengths, pm = O.analyze_blocks(data, block)
    assert (info["modes"] == modes).all() and (info["sizes"] == sizes).all()
    assert len(set(modes.tolist())) >= 2   # both sides of the boundary are present
    r = codec.decompress(b)
    assert r.status == [0] and host_bytes(r.payload(0)) == data


def _length_set_block(kind: str, block: int, rng) -> np.ndarray:
    """One block whose optimal code has a chosen set of lengths."""
    if kind.startswith("uniform"):          # k symbols, all of length log2(k)
        k = int(kind[7:])
        counts = {s: block // k for s in range(k)}
    elif kind == "len3_len6":                # lengths {3, 6}: gcd 3
        counts = {s: block * 7 // 56 for s in range(7)}
        counts.update({40 + s: block // 64 for s in range(8)})
    elif kind == "geometric":                # lengths 1, 2, 3, ... (run path + codes > 11 bits)
        counts, left, c, s = {}, block, block // 2, 200
        while c >= 1 and left > c:
            counts[s] = c
            left -= c
            c //= 2
            s -= 7
        counts[s] = left
    elif kind == "fibonacci":                # deeper than 15: package-merge
        a, b, counts, s = 1, 1, {}, 3
        while sum(counts.values()) + a <= block * 3 // 4:
            counts[s] = a
            a, b, s = b, a + b, s + 11
        counts[255] = block - sum(counts.values())
    else:
        raise ValueError(kind)
    x = np.concatenate([np.full(c, sym, np.uint8) for sym, c in counts.items()])
    assert len(x) == block
    return rng.permutation(x)


@pytest.mark.parametrize("block,kinds", [
    (4096, ["uniform2", "uniform4", "uniform8", "uniform16", "uniform64", "uniform128", "len3_len6", "geometric"]),
    (65536, ["uniform4", "len3_len6", "geometric", "fibonacci"]),
])
def test_code_length_sets(codec, block, kinds):
    """Huffman blocks with one code length (gcd = that length), two lengths
    with gcd 3, lengths 1..15 (run path plus codes longer than the 11-bit
    table) and package-merge-limited Fibonacci counts: the decoder's per-record
    length counts, canonical offsets, min / max length and gcd (one warp,
    shuffle scans) and the encoder, against the oracle byte for byte."""
    rng = np.random.default_rng(block + len(kinds))
    data = np.concatenate([_length_set_block(k, block, rng) for k in kinds]).tobytes()
    modes, _, _, lengths, pm = O.analyze_blocks(data, block)
    assert (modes == 0).all(), modes   # every block is a Huffman record (MODE_HUFFMAN)
    want = {"len3_len6": [3, 6], "geometric": list(range(1, 13)) if block == 4096 else None}
    for k, l in zip(kinds, lengths):
        got = sorted(set(l[l > 0].tolist()))
        if k.startswith("uniform"):
            assert got == [int(k[7:]).bit_length() - 1]
        elif want.get(k):
            assert got == want[k]
        else:   # 64 KiB geometric / fibonacci: limited to 15 bits
            assert got[0] <= 2 and got[-1] == 15
    ref = O.compress(data, 0, block_size=block)
    b = codec.compress([dev_bytes(data)], element_types=[0], block_size=block)
    assert b.to_bytes()[0] == ref
    fallback_segments(codec)
    for r in (codec.decompress(b), codec.decompress([dev_bytes(ref)])):
        assert r.status == [0] and host_bytes(r.payload(0)) == data
    assert fallback_segments(codec) == 0
