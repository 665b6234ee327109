"""GPU: the compress-side CRC-32 (stream.py:323-330) where k_hist folds it
into its read (windows that are whole blocks on the vector path, every
element width) and where k_crc computes it (the other windows): the header
CRC -- and with it the whole stream -- must equal the oracle's."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_09810_b200 as lmcb  # noqa: E402
from oracle import oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def codec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return lmcb.Codec()


def host_bytes(t) -> bytes:
    return t.reshape(-1).view(torch.uint8).cpu().numpy().tobytes()


ET_OF = {torch.bfloat16: 1, torch.float16: 2, torch.float32: 3, torch.uint8: 0}


@pytest.mark.parametrize("block", [4096, 65536, 1 << 20])
@pytest.mark.parametrize("bg", [True, False])
def test_header_crc_every_width(codec, block, bg):
    g = torch.Generator(device="cuda").manual_seed(block + bg)
    n = 1 << 20
    ts = [(torch.randn(n, generator=g, device="cuda") * 0.02).to(torch.bfloat16),      # whole blocks: k_hist folds
          (torch.randn(n, generator=g, device="cuda") * 0.02).to(torch.float16),
          torch.randn(n, generator=g, device="cuda"),                                    # fp32: four planes
          torch.randint(0, 256, (n,), generator=g, device="cuda", dtype=torch.uint8),    # raw8: one plane
          (torch.randn(n + 24, generator=g, device="cuda") * 0.02).to(torch.bfloat16),   # not whole blocks: k_crc
          torch.randn(3000, generator=g, device="cuda")]
    b = codec.compress(ts, block_size=block, byte_group=bg, buffer_size=1 << 21)   # several windows per stream
    for t, s in zip(ts, b.to_bytes()):
        want = O.compress(host_bytes(t), ET_OF[t.dtype], block_size=block, byte_group=bg, buffer_size=1 << 21,
                          threads=8)
        assert s == want, (t.dtype, t.numel())


def test_header_crc_delta_and_unaligned_views(codec):
    # fused XOR delta (the CRC covers the XOR bytes, stream.py:322,329) and a
    # source that is not 16-byte aligned (the vector path is off: k_crc)
    g = torch.Generator(device="cuda").manual_seed(7)
    prev = (torch.randn(1 << 20, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    nxt = (prev.float() + torch.randn(1 << 20, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    b = codec.compress([nxt], prev=[prev])
    x = host_bytes(prev.view(torch.uint8) ^ nxt.view(torch.uint8))
    assert b.to_bytes()[0] == O.compress(x, 1, delta=True, threads=8)
    base = torch.zeros((1 << 20) + 64, dtype=torch.uint8, device="cuda")
    base[8: 8 + (1 << 20)] = torch.randint(0, 256, (1 << 20,), generator=g, device="cuda", dtype=torch.uint8)
    view = base[8: 8 + (1 << 20)]
    b = codec.compress([view], element_types=[1])
    assert b.to_bytes()[0] == O.compress(host_bytes(view), 1, threads=8)


@pytest.mark.parametrize("off", [16, 32, 48])
def test_header_crc_views_at_16_byte_offsets(codec, off):
    # 16-bit elements on the vector path at addresses that are / are not
    # 32-byte aligned: k_hist folds the CRC with 32-byte (256-bit loads) or
    # 16-byte lane pieces; plain and delta (the previous step at the same offset)
    g = torch.Generator(device="cuda").manual_seed(off)
    n = 1 << 20
    base = torch.zeros(2 * n + 64, dtype=torch.uint8, device="cuda")
    pbase = torch.zeros(2 * n + 64, dtype=torch.uint8, device="cuda")
    w = (torch.randn(n, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    w2 = (w.float() + torch.randn(n, generator=g, device="cuda") * 1e-3 * w.float().abs()).to(torch.bfloat16)
    pbase[off: off + 2 * n] = w.view(torch.uint8)
    base[off: off + 2 * n] = w2.view(torch.uint8)
    cur = base[off: off + 2 * n].view(torch.bfloat16)
    prev = pbase[off: off + 2 * n].view(torch.bfloat16)
    assert cur.data_ptr() % 32 == off % 32
    b = codec.compress([cur])
    assert b.to_bytes()[0] == O.compress(host_bytes(cur), 1, threads=8)
    b = codec.compress([cur], prev=[prev])
    x = host_bytes(cur.view(torch.uint8) ^ prev.view(torch.uint8))
    assert b.to_bytes()[0] == O.compress(x, 1, delta=True, threads=8)
    r = codec.decompress(b)
    assert r.status == [0]
    assert torch.equal(r.payload(0), cur.view(torch.uint8) ^ prev.view(torch.uint8))
