"""Generate the checkpoint-chain fixture from the LIVE reference (build container only).

Run from the repo root:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_chain.py

Builds a four-step chain with the reference's ``lmc.chain.add_step``
(chain.py:133-208): three shards (bf16 weight, bf16 bias, fp32 gain), step 0
stored whole, steps 1-3 as XOR deltas against the previous step.  Writes

* ``chain/``            -- the reference's chain directory verbatim
  (``manifest.jsonl`` + one ``.lmc`` stream per step and shard);
* ``chain_inputs.npz``  -- the raw bytes of every shard at every step (what
  ``restore_step`` must return), checked here against the reference's own
  ``restore_step`` before writing.

Step t+1 follows the survey's delta model: w' =
bf16(fp32(w) + eps * (1e-3 |w| + 1e-6)), eps ~ N(0, 1), so most bytes repeat.
"""
from __future__ import annotations

import json
import os
import shutil
import sys

import numpy as np

from lmc.analysis import bf16_encode
from lmc.chain import add_step, restore_step
from lmc.types import ElementType, TensorBuffer

HERE = os.path.dirname(os.path.abspath(__file__))
STEPS = 4


def bf16_decode(u: np.ndarray) -> np.ndarray:
    return (u.astype(np.uint32) << 16).view(np.float32)


def make_steps(rng: np.random.Generator) -> list[dict[str, tuple[bytes, ElementType]]]:
    w = rng.normal(0, 0.02, 32 * 1024).astype(np.float32)
    b = rng.normal(0, 0.002, 1000).astype(np.float32)
    g = (1 + rng.normal(0, 0.01, 3000)).astype(np.float32)
    wb, bb = bf16_encode(w), bf16_encode(b)
    steps = []
    for _ in range(STEPS):
        steps.append({"layer0.weight": (wb.astype("<u2").tobytes(), ElementType.BF16),
                      "layer0.bias": (bb.astype("<u2").tobytes(), ElementType.BF16),
                      "norm.gain": (g.astype("<f4").tobytes(), ElementType.FP32)})
        fw, fb = bf16_decode(wb), bf16_decode(bb)
        wb = bf16_encode(fw + rng.normal(0, 1, fw.size).astype(np.float32) * (1e-3 * np.abs(fw) + 1e-6))
        bb = bf16_encode(fb + rng.normal(0, 1, fb.size).astype(np.float32) * (1e-3 * np.abs(fb) + 1e-6))
        g = (g + rng.normal(0, 1, g.size).astype(np.float32) * (1e-4 * np.abs(g))).astype(np.float32)
    return steps


def main() -> None:
    out_dir = os.path.join(HERE, "chain")
    if os.path.exists(out_dir):
        shutil.rmtree(out_dir)
    steps = make_steps(np.random.default_rng(20250509))
    for k, shards in enumerate(steps):
        got = add_step(out_dir, {n: TensorBuffer(d, et) for n, (d, et) in shards.items()})
        assert got == k
    os.remove(os.path.join(out_dir, ".chain.lock")) if os.path.exists(os.path.join(out_dir, ".chain.lock")) else None
    arrays, meta = {}, []
    for k, shards in enumerate(steps):
        back = restore_step(out_dir, k)
        for n, (d, et) in sorted(shards.items()):
            assert back[n].data == d and back[n].element_type is et, (k, n)
            key = f"s{k}_{n}"
            arrays[key] = np.frombuffer(d, np.uint8)
            meta.append({"step": k, "shard": n, "dtype": et.name.lower(), "key": key})
    np.savez_compressed(os.path.join(HERE, "chain_inputs.npz"), meta=json.dumps(meta), **arrays)
    print("chain fixture:", sorted(os.listdir(out_dir)), file=sys.stderr)


if __name__ == "__main__":
    main()
