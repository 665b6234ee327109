"""Seeded synthetic checkpoints with the shapes of BASELINE.json's configs.

No checkpoints or datasets are available offline, so every benchmark and
parity case draws from these generators ("Inputs"):

* cfg1  one 4096 x 4096 tensor ~ N(0, 0.02) -> bf16 (round-to-nearest-even)
* cfg2  GPT-2-small (124M params, 148 tensors): Linear/embedding ~ N(0, .02),
        LayerNorm gains 1 + N(0, .01), biases N(0, .002)
* cfg3  8192 x 8192 with a Bernoulli(0.5) exact-zero mask + 1M all-zero
* cfg4  GPT-style 1.3B (24 layers, d=2048, ffn=8192, vocab 50257, ctx 2048):
        step t ~ N(0, .02); step t+1 = bf16(w_t + N(0,1) * (1e-3 |w_t| + 1e-6))
* cfg5  Llama-7B (32 layers, d=4096, ffn=11008, vocab 32000) + delta step

Tensors are generated on the GPU with torch's Philox generator seeded per
(config seed, tensor index), then cast fp32 -> bf16 (RNE, identical to the
reference's analysis.bf16_encode for finite values).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class TensorSpec:
    name: str
    shape: tuple
    kind: str  # "weight" | "gain" | "bias" | "zeros" | "halfzero"

    @property
    def numel(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n


def gpt2_small() -> list[TensorSpec]:
    d, ffn, vocab, ctx, L = 768, 3072, 50257, 1024, 12
    out = [TensorSpec("wte", (vocab, d), "weight"), TensorSpec("wpe", (ctx, d), "weight")]
    for i in range(L):
        p = f"h.{i}."
        out += [
            TensorSpec(p + "ln_1.weight", (d,), "gain"), TensorSpec(p + "ln_1.bias", (d,), "bias"),
            TensorSpec(p + "attn.c_attn.weight", (d, 3 * d), "weight"), TensorSpec(p + "attn.c_attn.bias", (3 * d,), "bias"),
            TensorSpec(p + "attn.c_proj.weight", (d, d), "weight"), TensorSpec(p + "attn.c_proj.bias", (d,), "bias"),
            TensorSpec(p + "ln_2.weight", (d,), "gain"), TensorSpec(p + "ln_2.bias", (d,), "bias"),
            TensorSpec(p + "mlp.c_fc.weight", (d, ffn), "weight"), TensorSpec(p + "mlp.c_fc.bias", (ffn,), "bias"),
            TensorSpec(p + "mlp.c_proj.weight", (ffn, d), "weight"), TensorSpec(p + "mlp.c_proj.bias", (d,), "bias"),
        ]
    out += [TensorSpec("ln_f.weight", (d,), "gain"), TensorSpec("ln_f.bias", (d,), "bias")]
    return out


def gpt_1p3b(layers: int = 24) -> list[TensorSpec]:
    d, ffn, vocab, ctx = 2048, 8192, 50257, 2048
    out = [TensorSpec("wte", (vocab, d), "weight"), TensorSpec("wpe", (ctx, d), "weight")]
    for i in range(layers):
        p = f"h.{i}."
        out += [
            TensorSpec(p + "ln_1.weight", (d,), "gain"), TensorSpec(p + "ln_1.bias", (d,), "bias"),
            TensorSpec(p + "attn.qkv.weight", (d, 3 * d), "weight"), TensorSpec(p + "attn.qkv.bias", (3 * d,), "bias"),
            TensorSpec(p + "attn.proj.weight", (d, d), "weight"), TensorSpec(p + "attn.proj.bias", (d,), "bias"),
            TensorSpec(p + "ln_2.weight", (d,), "gain"), TensorSpec(p + "ln_2.bias", (d,), "bias"),
            TensorSpec(p + "mlp.fc.weight", (d, ffn), "weight"), TensorSpec(p + "mlp.fc.bias", (ffn,), "bias"),
            TensorSpec(p + "mlp.proj.weight", (ffn, d), "weight"), TensorSpec(p + "mlp.proj.bias", (d,), "bias"),
        ]
    out += [TensorSpec("ln_f.weight", (d,), "gain"), TensorSpec("ln_f.bias", (d,), "bias")]
    return out


def llama_7b(layers: int = 32) -> list[TensorSpec]:
    d, ffn, vocab = 4096, 11008, 32000
    out = [TensorSpec("embed_tokens", (vocab, d), "weight")]
    for i in range(layers):
        p = f"layers.{i}."
        out += [TensorSpec(p + n, (d, d), "weight") for n in ("q_proj", "k_proj", "v_proj", "o_proj")]
        out += [TensorSpec(p + "gate_proj", (ffn, d), "weight"), TensorSpec(p + "up_proj", (ffn, d), "weight"),
                TensorSpec(p + "down_proj", (d, ffn), "weight"),
                TensorSpec(p + "input_layernorm", (d,), "gain"), TensorSpec(p + "post_attention_layernorm", (d,), "gain")]
    out += [TensorSpec("norm", (d,), "gain"), TensorSpec("lm_head", (vocab, d), "weight")]
    return out


def cfg1() -> list[TensorSpec]:
    return [TensorSpec("w", (4096, 4096), "weight")]


def cfg3() -> list[TensorSpec]:
    return [TensorSpec("halfzero", (8192, 8192), "halfzero"), TensorSpec("zeros", (1 << 20,), "zeros")]


CONFIGS = {"cfg1": cfg1, "cfg2": gpt2_small, "cfg3": cfg3, "cfg4": gpt_1p3b, "cfg5": llama_7b}


def make_tensor(spec: TensorSpec, seed: int, index: int, device="cuda"):
    """One bf16 tensor of the spec, seeded by (seed, index)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + index * 7919) & 0x7FFFFFFFFFFFFFFF)
    n = spec.numel
    if spec.kind == "zeros":
        return torch.zeros(spec.shape, dtype=torch.bfloat16, device=device)
    x = torch.randn(n, generator=g, device=device, dtype=torch.float32)
    if spec.kind == "weight":
        x = x * 0.02
    elif spec.kind == "gain":
        x = 1.0 + x * 0.01
    elif spec.kind == "bias":
        x = x * 0.002
    elif spec.kind == "halfzero":
        x = x * 0.02
        mask = torch.rand(n, generator=g, device=device) < 0.5
        x = torch.where(mask, torch.zeros_like(x), x)
    return x.to(torch.bfloat16).reshape(spec.shape)


def next_step(w, seed: int, index: int):
    """Delta model of cfg4/cfg5: bf16(fp32(w) + N(0,1) * (1e-3 |w| + 1e-6))."""
    import torch

    g = torch.Generator(device=w.device)
    g.manual_seed((seed * 2_000_003 + index * 104729 + 17) & 0x7FFFFFFFFFFFFFFF)
    f = w.float()
    eps = torch.randn(f.shape, generator=g, device=w.device, dtype=torch.float32)
    return (f + eps * (1e-3 * f.abs() + 1e-6)).to(torch.bfloat16)


def make_checkpoint(config: str, seed: int = 1, device="cuda", limit: int | None = None):
    specs = CONFIGS[config]()
    if limit is not None:
        specs = specs[:limit]
    return specs, [make_tensor(s, seed, i, device) for i, s in enumerate(specs)]
