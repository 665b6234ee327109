"""Checkpoint chains: DeviceChain against the reference's
own chain directory (tests/golden/chain/, written by lmc.chain.add_step via
tests/golden/make_chain.py), and the fused decode + xor_apply entry point
(lmcg_decompress_apply) against decode-then-XOR."""
from __future__ import annotations

import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN

CHAIN = os.path.join(GOLDEN, "chain")


def chain_inputs():
    z = np.load(os.path.join(GOLDEN, "chain_inputs.npz"))
    steps: dict[int, dict] = {}
    for m in json.loads(str(z["meta"])):
        steps.setdefault(m["step"], {})[m["shard"]] = (z[m["key"]].tobytes(), m["dtype"])
    return steps


def copy_chain(tmp_path, last_step=None):
    """The golden chain in a scratch directory, optionally cut after ``last_step``."""
    dst = tmp_path / "chain"
    shutil.copytree(CHAIN, dst)
    if last_step is not None:
        rows = (dst / "manifest.jsonl").read_text().splitlines()
        keep = [rows[0]] + [r for r in rows[1:] if json.loads(r)["step"] <= last_step]
        (dst / "manifest.jsonl").write_text("\n".join(keep) + "\n")
        for f in os.listdir(dst):
            if f.startswith("step") and int(f[4:10]) > last_step:
                os.remove(dst / f)
    return dst


# ------------------------------------------------------------------ host logic (no GPU)
def test_manifest_round_trip(tmp_path):
    from paper_2505_09810_b200.chain import load_manifest, save_manifest

    m = load_manifest(CHAIN)
    assert m.last_step == 3 and len(m.entries) == 12
    save_manifest(tmp_path, m)
    assert (tmp_path / "manifest.jsonl").read_bytes() == open(os.path.join(CHAIN, "manifest.jsonl"), "rb").read()


def test_manifest_validation(tmp_path):
    from paper_2505_09810_b200 import CorruptStreamError
    from paper_2505_09810_b200.chain import load_manifest
    from paper_2505_09810_b200.errors import MissingStreamError

    with pytest.raises(MissingStreamError):
        load_manifest(tmp_path)
    d = copy_chain(tmp_path)
    rows = (d / "manifest.jsonl").read_text().splitlines()
    bad = [rows[0]] + [r.replace('"role": "base"', '"role": "delta"') for r in rows[1:]]
    (d / "manifest.jsonl").write_text("\n".join(bad) + "\n")
    with pytest.raises(CorruptStreamError):
        load_manifest(d)
    # a step missing one shard
    (d / "manifest.jsonl").write_text("\n".join(rows[:-1]) + "\n")
    with pytest.raises(CorruptStreamError):
        load_manifest(d)
    (d / "manifest.jsonl").write_text("")
    with pytest.raises(CorruptStreamError):
        load_manifest(d)


def test_stream_names():
    from paper_2505_09810_b200.chain import stream_name

    assert stream_name(0, "layer0.weight") == "step000000_layer0.weight.lmc"
    assert stream_name(12, "a/b c:d") == "step000012_a_b_c_d.lmc"


def test_golden_chain_against_oracle():
    """The fixture's streams decode (oracle) to the stored inputs and deltas."""
    from oracle import oracle as O
    from paper_2505_09810_b200.chain import load_manifest

    steps = chain_inputs()
    m = load_manifest(CHAIN)
    for e in m.entries:
        data, _ = O.decompress(open(os.path.join(CHAIN, e.file), "rb").read())[:2]
        cur = np.frombuffer(steps[e.step][e.shard][0], np.uint8)
        want = cur if e.step == 0 else cur ^ np.frombuffer(steps[e.step - 1][e.shard][0], np.uint8)
        assert data == want.tobytes(), e.file


# ------------------------------------------------------------------ GPU
def _device_shards(shards):
    import torch

    from paper_2505_09810_b200 import ElementType, TensorBuffer

    out = {}
    for name, (data, dtype) in shards.items():
        out[name] = TensorBuffer(data, ElementType.from_name(dtype))
    return out


@pytest.mark.gpu
def test_restore_reference_chain(tmp_path):
    from paper_2505_09810_b200 import DeviceChain

    steps = chain_inputs()
    ch = DeviceChain(copy_chain(tmp_path))
    for k in (3, 0, 2, 1):
        got = ch.restore_step(k)
        assert sorted(got) == sorted(steps[k])
        for name, (data, _) in steps[k].items():
            assert got[name].cpu().numpy().tobytes() == data, (k, name)
    bufs = ch.restore_buffers(3)
    assert bufs["norm.gain"].element_type.name == "FP32"


@pytest.mark.gpu
def test_build_chain_matches_reference(tmp_path):
    """Every stream file byte-identical to lmc.chain.add_step's; manifest equal but for chain_id."""
    from paper_2505_09810_b200 import DeviceChain

    steps = chain_inputs()
    d = tmp_path / "mine"
    ch = DeviceChain(d)
    for k in range(4):
        assert ch.add_step(_device_shards(steps[k])) == k
    ref_rows = open(os.path.join(CHAIN, "manifest.jsonl")).read().splitlines()
    my_rows = (d / "manifest.jsonl").read_text().splitlines()
    assert my_rows[1:] == ref_rows[1:]
    for f in os.listdir(CHAIN):
        if f.endswith(".lmc"):
            assert (d / f).read_bytes() == open(os.path.join(CHAIN, f), "rb").read(), f


@pytest.mark.gpu
def test_append_to_reference_chain(tmp_path):
    """Open a chain the reference wrote (steps 0-1), append steps 2-3 on the GPU."""
    import torch

    from paper_2505_09810_b200 import DeviceChain

    steps = chain_inputs()
    d = copy_chain(tmp_path, last_step=1)
    ch = DeviceChain(d)
    for k in (2, 3):
        # CUDA tensors this time (bf16 / fp32 views of the same bytes)
        shards = {}
        for name, (data, dtype) in steps[k].items():
            t = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
            shards[name] = t.view(torch.bfloat16 if dtype == "bf16" else torch.float32)
        assert ch.add_step(shards, step=k) == k
    for f in os.listdir(CHAIN):
        if f.endswith(".lmc"):
            assert (d / f).read_bytes() == open(os.path.join(CHAIN, f), "rb").read(), f
    # a fresh object (nothing resident) restores what the first one appended
    got = DeviceChain(d).restore_step(3)
    for name, (data, _) in steps[3].items():
        assert got[name].cpu().numpy().tobytes() == data


@pytest.mark.gpu
def test_chain_errors(tmp_path):
    from paper_2505_09810_b200 import (CorruptStreamError, DeviceChain, DtypeMismatchError, ElementType,
                                       IntegrityError, LmcError, ShapeMismatchError, TensorBuffer)
    from paper_2505_09810_b200.errors import MissingStreamError

    steps = chain_inputs()
    d = copy_chain(tmp_path)
    ch = DeviceChain(d)
    with pytest.raises(MissingStreamError):
        ch.restore_step(4)
    with pytest.raises(LmcError):
        ch.add_step(_device_shards(steps[3]), step=2)     # exists
    with pytest.raises(LmcError):
        ch.add_step(_device_shards(steps[3]), step=6)     # gap
    with pytest.raises(ShapeMismatchError):
        ch.add_step({})
    bad = _device_shards(steps[3])
    bad["layer0.bias"] = TensorBuffer(bad["layer0.bias"].data[:-2], ElementType.BF16)
    with pytest.raises(ShapeMismatchError):
        ch.add_step(bad)
    bad = _device_shards(steps[3])
    bad["layer0.bias"] = TensorBuffer(bad["layer0.bias"].data, ElementType.FP16)
    with pytest.raises(DtypeMismatchError):
        ch.add_step(bad)
    bad = _device_shards(steps[3])
    del bad["norm.gain"]
    with pytest.raises(ShapeMismatchError):
        ch.add_step(bad)
    # manifest CRC disagrees with the stream header
    rows = (d / "manifest.jsonl").read_text().splitlines()
    e = json.loads(rows[5])
    e["crc32"] ^= 1
    (d / "manifest.jsonl").write_text("\n".join(rows[:5] + [json.dumps(e, sort_keys=True)] + rows[6:]) + "\n")
    with pytest.raises(IntegrityError):
        DeviceChain(d).restore_step(2)
    (d / "manifest.jsonl").write_text("\n".join(rows) + "\n")
    # payload corruption inside a delta stream -> the decode's own error
    f = d / json.loads(rows[7])["file"]
    raw = bytearray(f.read_bytes())
    raw[-1] ^= 0x5A
    f.write_bytes(bytes(raw))
    with pytest.raises((IntegrityError, CorruptStreamError)):
        DeviceChain(d).restore_step(3)
    # role flag disagrees with the manifest: a base stream listed as a delta
    shutil.copy(d / json.loads(rows[1])["file"], f)
    e = json.loads(rows[7])
    e["crc32"] = json.loads(rows[1])["crc32"]
    e["length"] = json.loads(rows[1])["length"]
    (d / "manifest.jsonl").write_text("\n".join(rows[:7] + [json.dumps(e, sort_keys=True)] + rows[8:]) + "\n")
    with pytest.raises(CorruptStreamError):
        DeviceChain(d).restore_step(3)
    os.remove(f)
    with pytest.raises(MissingStreamError):
        DeviceChain(d).restore_step(3)


@pytest.mark.gpu
@pytest.mark.parametrize("in_place", [False, True])
def test_decompress_apply(in_place):
    """lmcg_decompress_apply == lmc_decompress then xor_apply (delta.py:50-52)."""
    import torch

    import paper_2505_09810_b200 as lmcb

    g = torch.Generator(device="cuda").manual_seed(7)
    codec = lmcb.Codec(0)
    lmcb._lib.load().lmcg_fallback_segments(1)   # earlier tests decode corrupt streams on purpose
    sizes = [(4096, 4096), (1000,), (3, 65537), (8,)]
    prev = [(torch.randn(*s, generator=g, device="cuda") * 0.02).to(torch.bfloat16) for s in sizes]
    nxt = []
    for p in prev:
        f = p.float()
        nxt.append((f + torch.randn(f.shape, generator=g, device="cuda") * (1e-3 * f.abs() + 1e-6)).to(torch.bfloat16))
    batch = codec.compress(nxt, prev=prev)
    if in_place:
        pos, offs = 0, []
        for p in prev:
            offs.append(pos)
            pos += (p.numel() * 2 + 15) & ~15
        buf = torch.empty(pos, dtype=torch.uint8, device="cuda")
        for o, p in zip(offs, prev):
            buf[o: o + p.numel() * 2].copy_(p.view(torch.uint8).reshape(-1))
        views = [buf[o: o + p.numel() * 2] for o, p in zip(offs, prev)]
        res = codec.decompress(batch, out=buf, out_offsets=offs, prev=views)
    else:
        res = codec.decompress(batch, prev=prev)
    res.raise_for_status()
    for i, t in enumerate(nxt):
        assert torch.equal(res.payload(i), t.view(torch.uint8).reshape(-1)), i
    assert lmcb._lib.load().lmcg_fallback_segments(1) == 0


@pytest.mark.gpu
def test_decompress_apply_errors():
    import torch

    import paper_2505_09810_b200 as lmcb

    codec = lmcb.Codec(0)
    a = torch.arange(5000, device="cuda", dtype=torch.int32).to(torch.bfloat16)
    b = a + 1
    batch = codec.compress([b], prev=[a])
    # prev of another length: ShapeMismatchError after a clean decode
    res = codec.decompress(batch, prev=[a[:-1]])
    assert res.status == [11]
    with pytest.raises(lmcb.ShapeMismatchError):
        res.raise_for_status()
    # a corrupt payload keeps the decode's own error ahead of the length check
    s = bytearray(batch.to_bytes()[0])
    s[24] ^= 1   # header CRC
    dev = torch.frombuffer(s, dtype=torch.uint8).cuda()
    assert codec.decompress([dev], prev=[a]).status == [3]
    assert codec.decompress([dev], prev=[a[:-1]]).status == [3]
    # None entries decode plainly
    res = codec.decompress(codec.compress([a, b]), prev=[None, a])
    res.raise_for_status()
    assert torch.equal(res.payload(0), a.view(torch.uint8).reshape(-1))
    assert torch.equal(res.payload(1), (a.view(torch.int16) ^ b.view(torch.int16)).view(torch.uint8).reshape(-1))
