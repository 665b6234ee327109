"""Full-size GPU runs of BASELINE.json's large configs, every stream checked
against the oracle:

* cfg5 Llama-7B (291 tensors, 12.55 GiB): every GPU stream is byte-identical
  to the oracle's (tables, record modes and sizes, CRC: the whole stream),
  and every stream round-trips bit-exactly on the device;
* cfg5's second step in delta mode (stream.py:304-308, delta.py:29-47): every
  delta stream equals the oracle's stream of the XOR bytes, and the fused
  decode + xor_apply (delta.py:50-52) rebuilds step t+1 from step t;
* cfg4 GPT 1.3B in delta mode (292 tensors): the same, stream by stream.

The oracle runs on all host threads (tens of seconds per config); everything
else stays resident in HBM (180 GB)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_09810_b200 as lmcb  # noqa: E402
from paper_2505_09810_b200 import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402

THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def codec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return lmcb.Codec()


def _u8(t):
    return t.view(torch.uint8).reshape(-1)


def _host_streams(batch):
    off, ln = batch.host_layout()
    flat = batch.data[: off[-1] + ln[-1]].cpu().numpy()
    return [flat[o: o + n] for o, n in zip(off, ln)]


def _check_every_stream(specs, batch, host_inputs, delta):
    """Every stream of the batch against the oracle's stream of the same bytes."""
    streams = _host_streams(batch)
    bad = []
    for i, s in enumerate(specs):
        want = O.compress(host_inputs(i), 1, delta=delta, threads=THREADS)
        got = streams[i]
        if len(got) != len(want) or not np.array_equal(got, np.frombuffer(want, np.uint8)):
            bad.append(s.name)
    assert not bad, f"{len(bad)} streams differ from the oracle: {bad[:5]}"
    return sum(len(x) for x in streams)


def test_cfg5_llama7b_every_stream(codec):
    specs, ts = synth.make_checkpoint("cfg5", seed=5)
    total = sum(t.numel() * 2 for t in ts)
    assert total == 13_476_831_232
    b = codec.compress(ts)
    nstream = _check_every_stream(specs, b, lambda i: _u8(ts[i]).cpu().numpy(), delta=False)
    assert 0.6 < nstream / total < 0.75
    codec.ctx.lib.lmcg_fallback_segments(1)
    r = codec.decompress(b)
    assert r.status == [0] * len(ts)
    assert codec.ctx.lib.lmcg_fallback_segments(1) == 0
    for i, t in enumerate(ts):
        assert torch.equal(r.payload(i), _u8(t)), specs[i].name
    del r, b
    # the second step in delta mode (BASELINE cfg5 "plus a second step for delta mode")
    nxt = [synth.next_step(w, 5, i) for i, w in enumerate(ts)]
    b = codec.compress(nxt, prev=ts)
    dstream = _check_every_stream(specs, b, lambda i: (_u8(ts[i]) ^ _u8(nxt[i])).cpu().numpy(), delta=True)
    assert dstream / total < 0.25
    codec.ctx.lib.lmcg_fallback_segments(1)
    r = codec.decompress(b, prev=ts)          # fused decode + xor_apply: step t+1 from step t
    assert r.status == [0] * len(ts)
    assert codec.ctx.lib.lmcg_fallback_segments(1) == 0
    for i, q in enumerate(nxt):
        assert torch.equal(r.payload(i), _u8(q)), specs[i].name


def test_cfg4_gpt1p3b_every_delta_stream(codec):
    specs, prev = synth.make_checkpoint("cfg4", seed=41)
    nxt = [synth.next_step(w, 41, i) for i, w in enumerate(prev)]
    b = codec.compress(nxt, prev=prev)
    total = sum(t.numel() * 2 for t in nxt)
    assert total == 2_631_446_528
    nstream = _check_every_stream(specs, b, lambda i: (_u8(prev[i]) ^ _u8(nxt[i])).cpu().numpy(), delta=True)
    assert nstream / total < 0.25      # ~0.13: most bytes unchanged between steps
    codec.ctx.lib.lmcg_fallback_segments(1)
    r = codec.decompress(b)
    assert r.status == [0] * len(nxt)
    assert codec.ctx.lib.lmcg_fallback_segments(1) == 0
    for i, (p, q) in enumerate(zip(prev, nxt)):
        x = r.payload(i)
        assert torch.equal(x, _u8(p) ^ _u8(q)), specs[i].name      # the XOR delta
        assert torch.equal(_u8(p) ^ x, _u8(q))                      # re-applies to the next step
