"""Markdown table of every config's bench lines (profiles/<dir>/configs) for DESIGN.md."""
import json
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_s2"
names = {"cfg1": "cfg1 (32 MiB tensor)", "cfg2": "cfg2 (GPT-2-small)", "cfg3": "cfg3 (50% zeros + zeros)",
         "cfg4": "cfg4 (1.3B, delta)", "cfg5": "cfg5 (Llama-7B)"}
print("| config | round trip GiB/s | compress GiB/s | decompress GiB/s | e2e GiB/s | ratio | CPU port GiB/s | "
      "reference arm GiB/s | dominant kernel | roofline frac | compress / decompress HBM frac |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for c in names:
    last = lambda f: json.loads(open(f).read().strip().splitlines()[-1])
    a, r = last(f"{d}/configs/{c}.json"), last(f"{d}/configs/{c}_ref.json")
    p, rf = a["pipeline"], a["roofline"]
    print(f"| {names[c]} | {a['value']:.1f} | {p['compress_gib_s']:.1f} | {p['decompress_gib_s']:.1f} | "
          f"{a['e2e']['value']:.1f} | {a['compression_ratio']:.4f} | {a['cpu_baseline']['value']:.3f} | "
          f"{r['value']:.3f} | {rf['kernel']} | {rf['frac']:.3f} | {p['compress_hbm_frac']:.3f} / {p['decompress_hbm_frac']:.3f} |")
