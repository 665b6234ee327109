#!/usr/bin/env python
"""LMC hot-path benchmark: BASELINE.json's metric on its largest single-GPU
config, cfg5 (Llama-7B-shaped bf16 checkpoint, 291 tensors, 12.55 GiB).

One step = compress every tensor of the checkpoint into its own LMC1 stream
and decompress the streams again.  ``value`` is whole-job GiB/s of
uncompressed checkpoint bytes through compress + decompress (inputs resident
in HBM, streams kept in HBM); ``e2e`` is the same round trip through the
public plan API with pinned host buffers (host->device copy of the
checkpoint, device->host copy of the streams, and back); ``delta_step`` is
cfg5's second step in delta mode (step t+1 compressed against the resident
step t, fused XOR).  With N GPUs (torchrun) the ONE checkpoint is sharded
across the ranks (whole tensors, largest first; each rank holds only its
own tensors) and the only exchange is the all-gather of the per-stream
compressed lengths: strong scaling.  See DESIGN.md "Measurement".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg5]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
import types

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GIB = float(1 << 30)
METRIC = "lmc compress+decompress round-trip throughput (uncompressed checkpoint GiB/s, whole job)"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--no-delta", action="store_true", help="skip the delta-mode second step (cfg5)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels directly instead of replaying CUDA graphs")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    ~0.5 ms in a host thread while the timed region runs (nvidia-smi's first
    sample arrives only after ~100 ms, longer than a short timed region)."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.thread = None
        self.err = None

    def start(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"
            return
        self.stop_flag = False

        def run():
            nv = self.nv
            while not self.stop_flag:
                try:
                    sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.samples.append((sm, rs))
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(0.0005)

        self.thread = threading.Thread(target=run, daemon=True)
        self.thread.start()
        time.sleep(0.002)   # first sample in before the timed region starts

    def stop(self) -> dict:
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no sampler"], "samples": 0}
        self.stop_flag = True
        self.thread.join(timeout=2)
        nv = self.nv
        reasons = set()
        for _, rs in self.samples:
            for name, const in self.REASONS.items():
                if rs & getattr(nv, const, 0):
                    reasons.add(name)
        sm = [x for x, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvml, 0.5 ms"}


def measured_peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str, config: str):
    """Per-launch DRAM bytes of `kernel` on `config` from the committed ncu
    capture (profiles/ncu_traffic.json: config -> kernel -> bytes), or None
    when that config was not captured."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(config, {}).get(kernel)
    except Exception:
        return None


# ------------------------------------------------------------ distributed
def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------- reference arm
def run_reference(args, ws, rank):
    """Time the reference's algorithm on the host cores (C oracle port, all
    threads) on a bounded sample of the same workload."""
    if rank != 0:
        return
    import torch

    from oracle import oracle as O
    from paper_2505_09810_b200 import synth

    cores = os.cpu_count() or 1
    specs = synth.CONFIGS[args.config]()
    delta = args.config in DELTA
    dev = "cuda" if torch.cuda.is_available() else "cpu"

    def host_bytes(i):
        t = synth.make_tensor(specs[i], 1000, i, device=dev)
        x = t.view(torch.uint8).reshape(-1)
        if delta:
            x = x ^ synth.next_step(t, 1000, i).view(torch.uint8).reshape(-1)
        return x.cpu().numpy().tobytes()

    # bounded sample: tensors in checkpoint order until ~60 s of total work
    # (warm-up + timed steps), estimated from a probe of the first tensors
    budget = 60.0 / max(args.steps + args.warmup, 1)
    raws, acc, t_probe, b_probe = [], 0, 0.0, 0
    for i in range(len(specs)):
        r = host_bytes(i)
        raws.append(r)
        acc += len(r)
        if b_probe < (32 << 20):
            t0 = time.perf_counter()
            O.decompress(O.compress(r, 1, delta=delta, threads=cores), threads=cores)
            t_probe += time.perf_counter() - t0
            b_probe += len(r)
        if t_probe / max(b_probe, 1) * acc > budget:
            break
    sample_bytes = sum(len(r) for r in raws)
    sample = (f"{args.config} synthetic bf16 checkpoint: {len(raws)} of {len(specs)} tensors, "
              f"{sample_bytes / 2**20:.1f} MiB per step (compress + decompress, oracle C port, {cores} threads)")

    def step():
        st = [O.compress(r, 1, delta=delta, threads=cores) for r in raws]
        for x in st:
            O.decompress(x, threads=cores)
        return st

    for _ in range(args.warmup):
        streams = step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        streams = step()
    dt = time.perf_counter() - t0
    value = sample_bytes * args.steps / dt / GIB
    ratio = sum(len(x) for x in streams) / max(sample_bytes, 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GiB/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": workload(args.config), "sample_tensors": len(raws)},
        "compression_ratio": round(ratio, 6),
        "cpu_baseline": {"value": round(value, 4), "unit": "GiB/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GiB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# Workload names of BASELINE.json's configs.  The bench line is cfg5, the
# largest config that fits one GPU (BASELINE's metric names no config); the
# others are parity cases and optional bench runs (--config).
WORKLOAD = {
    "cfg1": "single bf16 tensor 4096x4096 ~ N(0, 0.02) (32 MiB)",
    "cfg2": "GPT-2-small bf16 checkpoint (148 tensors, 237.4 MiB)",
    "cfg3": "RLE-heavy: 8192x8192 bf16 with 50% exact zeros + 1M-element all-zero tensor",
    "cfg4": "GPT-style 1.3B, two consecutive bf16 steps, XOR delta fused into the compress (2.45 GiB per step; "
            "the previous step stays resident on the GPU)",
    "cfg5": "Llama-7B bf16 checkpoint (291 tensors, 12.55 GiB)",
}
DELTA = {"cfg4"}
SEED = 1000
L2_FLUSH_BELOW = 126_000_000   # bytes: the L2 size (inputs must be larger, or flushed)


def workload(cfg: str) -> str:
    return (f"{cfg}: {WORKLOAD[cfg]}, every tensor its own LMC1 stream, byte_group=True, block_size=65536, "
            "segment_count=1, buffer_size=128MiB")


# ----------------------------------------------------------------- ours
# Algorithmic bytes per launch: what the kernel must move in
# this pipeline, from the input bytes N_in (x2 with the fused delta: the
# previous step is read too) and the stream bytes N_stream.
COMPRESS_KERNELS = ("k_slotmap", "k_crc", "k_hist", "k_codebook", "k_pkgmerge", "k_scan", "k_layout", "k_frame",
                    "k_encode", "k_recsizes", "k_crc_join")


def is_compress_kernel(name: str) -> bool:
    return any(name == k or name.startswith(k + "<") or name.startswith(k + "_") for k in COMPRESS_KERNELS)


def algo_bytes(kernel: str, n_in: int, n_stream: int, delta: bool):
    rd = n_in * (2 if delta else 1)
    base = kernel.split("<")[0]
    return {
        "k_hist": rd, "k_hist_crc": rd, "k_crc": rd,       # read the input (and prev)
        "k_encode": rd + n_stream,                          # read the input, write the streams
        "k_cand": n_stream,                                 # scan the streams
        "k_decrec": n_stream + n_in,                        # read the streams, write the planes
        "k_decpair": n_stream + n_in,                       # read the streams, write the payload
        "k_ungroup": 2 * n_in,                              # read the planes, write the payload
    }.get(base)


def roofline_of(prof: dict, nprof: int, n_in: int, n_stream: int, delta: bool, peak: float, peak_src: str,
                config: str, kernels=None):
    """Roofline object of the dominant kernel (by time) among `kernels`."""
    cand = [(k, v) for k, v in prof.items() if algo_bytes(k, n_in, n_stream, delta) is not None
            and (kernels is None or kernels(k))]
    if not cand:
        return None
    dname, (dcnt, dms) = max(cand, key=lambda kv: kv[1][1])
    avg_ms = dms / dcnt
    ab = algo_bytes(dname, n_in, n_stream, delta)
    achieved = ab / (avg_ms / 1e3) / 1e9
    tot = sum(v[1] for k, v in prof.items() if kernels is None or kernels(k))
    return {"bound": "hbm", "kernel": dname, "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": ncu_traffic(dname, config), "peak_source": peak_src,
            "algorithmic_bytes_per_launch": ab, "avg_launch_ms": round(avg_ms, 4),
            "share_of_step": round(dms / max(tot, 1e-9), 4)}


def exchange_lengths(batch, owned, n_total, dist):
    """Container assembly across ranks: all-gather of every stream's compressed
    length (device tensors, NCCL); nothing else crosses GPUs."""
    from paper_2505_09810_b200 import shard

    if dist is None:
        return None
    return shard.gather_device_lengths(batch.lengths, owned, n_total)


def measure(codec, ts, prev, args, ws, dist, owned, n_total, local, with_clocks=True):
    """Device-timed round trips (compress + length exchange + decompress) of
    one rank's tensors; returns the timings (max over ranks) and the per-kernel
    launch times of an untimed profiling pass."""
    import torch

    stream = torch.cuda.current_stream()
    nbytes = sum(t.numel() * t.element_size() for t in ts)
    # the tensors are registered once (CompressPlan): every step re-compresses
    # their current contents; runs replay captured CUDA graphs
    cplan = codec.compress_plan(ts, prev=prev, graph=not args.no_graph)
    dplan = cplan.decompress_plan(graph=not args.no_graph)
    status_log = torch.zeros((args.steps + args.warmup + 8, max(len(ts), 1)), dtype=torch.int32, device="cuda")
    step_no = [0]

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        b = cplan.run()
        exchange_lengths(b, owned, n_total, dist)
        if ev:
            ev[1].record(stream)
        r = dplan.run(b)
        # every step's decode status stays on the device; verified after the timed region
        status_log[step_no[0] % status_log.shape[0], : len(ts)].copy_(r._status_dev)
        step_no[0] += 1
        if ev:
            ev[2].record(stream)
        return b, r

    # correctness gate before timing
    b, r = step()
    r.raise_for_status()
    for i, t in enumerate(ts):
        want = t.view(torch.uint8).reshape(-1)
        if prev is not None:
            want = want ^ prev[i].view(torch.uint8).reshape(-1)
        if not torch.equal(r.payload(i), want):
            raise SystemExit(f"round trip mismatch on tensor {owned[i]}")
    stream_bytes = b.total_bytes()
    for _ in range(max(args.warmup - 1, 0)):
        step()

    # per-kernel launch times (separate, untimed pass without graphs)
    codec.ctx.profile(True)
    nprof = 3
    for _ in range(nprof):
        # the GPU spins while the host enqueues each direction, so the
        # per-kernel events never include host launch gaps
        torch.cuda._sleep(4_000_000)
        pb = codec.compress(ts, prev=prev)
        pb.host_layout()          # (synchronises: the decode below needs the layout)
        torch.cuda._sleep(4_000_000)
        codec.decompress(pb)
    prof = codec.ctx.profile_report()
    codec.ctx.profile(False)
    del pb
    launches_per_step = sum(c for c, _ in prof.values()) / nprof

    # timed region
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    flush = None
    if nbytes * ws < L2_FLUSH_BELOW:
        # inputs smaller than the 126 MB L2: flush it between timed steps (a
        # 512 MB write outside the per-step events) and time the steps alone
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local) if with_clocks else None
    if sampler:
        sampler.start()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(args.steps):
        if flush is not None:
            flush.fill_(k & 0xFF)
        step(evs[k])
    end.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    if int(status_log.abs().sum().item()) != 0:
        bad = status_log.nonzero().tolist()
        codes = [int(status_log[i, j]) for i, j in bad[:8]]
        raise SystemExit(f"a timed step reported a decode error: (step slot, stream) {bad[:8]} codes {codes}")
    if dist is not None:
        dist.barrier()
    total_ms = start.elapsed_time(end)
    comp_ms = sum(e[0].elapsed_time(e[1]) for e in evs)
    dec_ms = sum(e[1].elapsed_time(e[2]) for e in evs)
    if flush is not None:
        total_ms = sum(e[0].elapsed_time(e[2]) for e in evs)
    t = torch.tensor([total_ms, comp_ms, dec_ms, float(stream_bytes)], dtype=torch.float64, device="cuda")
    if dist is not None:
        sb = t[3:].clone()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(sb, op=dist.ReduceOp.SUM)
        t[3] = sb[0]
    total_ms, comp_ms, dec_ms, all_stream = t.tolist()
    del cplan, dplan, b, r
    return {"total_ms": total_ms, "comp_ms": comp_ms, "dec_ms": dec_ms, "stream_bytes": int(stream_bytes),
            "all_stream_bytes": int(all_stream), "prof": prof, "nprof": nprof,
            "launches_per_step": launches_per_step, "clocks": clocks, "flush": flush is not None, "nbytes": nbytes}


def run_ours(args, ws, rank, local):
    import gc

    import torch

    import paper_2505_09810_b200 as lmcb
    from paper_2505_09810_b200 import shard, synth

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    specs = synth.CONFIGS[args.config]()
    sizes = [s.numel * 2 for s in specs]
    total_bytes = sum(sizes)
    # ONE checkpoint sharded across the ranks: whole tensors, largest first
    # onto the least-loaded rank (every rank computes the same table)
    owner = shard.assign_tensors(sizes, ws)
    owned = [i for i, r in enumerate(owner) if r == rank]
    ts = [synth.make_tensor(specs[i], SEED, i) for i in owned]
    prev = None
    if args.config in DELTA:   # compress step t+1 against step t (fused XOR)
        prev = ts
        ts = [synth.next_step(w, SEED, i) for i, w in zip(owned, prev)]
    codec = lmcb.Codec(local)
    m = measure(codec, ts, prev, args, ws, dist, owned, len(specs), local)
    gc.collect()
    torch.cuda.empty_cache()

    # cfg5's second step in delta mode: step t+1 against the resident step t
    delta_step = None
    if args.config == "cfg5" and not args.no_delta:
        nxt = [synth.next_step(w, SEED, i) for i, w in zip(owned, ts)]
        md = measure(codec, nxt, ts, args, ws, dist, owned, len(specs), local, with_clocks=False)
        peak, peak_src = measured_peaks()
        cs, ds = md["comp_ms"] / args.steps / 1e3, md["dec_ms"] / args.steps / 1e3
        delta_step = {
            "value": round(total_bytes * args.steps / (md["total_ms"] / 1e3) / GIB, 3), "unit": "GiB/s",
            "workload": "cfg5 step t+1 = bf16(w_t + N(0,1)(1e-3|w_t| + 1e-6)) compressed against the resident step t "
                        "(fused XOR, FLAG_DELTA streams) and decompressed to the XOR payload",
            "ms_per_step": round(md["total_ms"] / args.steps, 4),
            "compression_ratio": round(md["all_stream_bytes"] / total_bytes, 6),
            "compress_gib_s": round(total_bytes / cs / GIB, 3), "decompress_gib_s": round(total_bytes / ds / GIB, 3),
            "compress_hbm_frac": round((2 * total_bytes + md["all_stream_bytes"]) / cs / 1e9 / peak, 4),
            "decompress_hbm_frac": round((total_bytes + md["all_stream_bytes"]) / ds / 1e9 / peak, 4),
            "kernels_ms_per_step": {k: round(v[1] / md["nprof"], 4) for k, v in sorted(md["prof"].items())},
        }
        del nxt, md
        gc.collect()
        torch.cuda.empty_cache()

    # end-to-end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(codec, ts, args, ws, dist, total_bytes, owned, len(specs), prev=prev)

    peak, peak_src = measured_peaks()
    n_in, n_st = m["nbytes"], m["stream_bytes"]
    delta = prev is not None
    prof, nprof = m["prof"], m["nprof"]
    roofline = roofline_of(prof, nprof, n_in, n_st, delta, peak, peak_src, args.config)
    roof_c = roofline_of(prof, nprof, n_in, n_st, delta, peak, peak_src, args.config, is_compress_kernel)
    roof_d = roofline_of(prof, nprof, n_in, n_st, delta, peak, peak_src, args.config,
                         lambda k: not is_compress_kernel(k))
    steps = args.steps
    comp_s, dec_s = m["comp_ms"] / steps / 1e3, m["dec_ms"] / steps / 1e3
    in_all = total_bytes * (2 if delta else 1)
    pipeline = {
        "compress_gib_s": round(total_bytes / comp_s / GIB, 3),
        "decompress_gib_s": round(total_bytes / dec_s / GIB, 3),
        "compress_hbm_frac": round((in_all + m["all_stream_bytes"]) / comp_s / 1e9 / peak / ws, 4),
        "decompress_hbm_frac": round((total_bytes + m["all_stream_bytes"]) / dec_s / 1e9 / peak / ws, 4),
        "compress_ms": round(comp_s * 1e3, 4), "decompress_ms": round(dec_s * 1e3, 4),
    }
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(ts, prev)
    if rank == 0:
        value = total_bytes * steps / (m["total_ms"] / 1e3) / GIB
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GiB/s", "n_gpus": ws, "steps": steps,
            "warmup": args.warmup, "ms_per_step": round(m["total_ms"] / steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": workload(args.config),
                       "l2": (f"inputs {total_bytes / 1e6:.0f} MB > 126 MB L2 per step; no flush needed"
                              if not m["flush"] else
                              f"inputs {total_bytes / 1e6:.0f} MB: 512 MB L2 flush between timed steps, steps timed alone"),
                       "parallelism": (f"dp{ws}: one checkpoint sharded by whole tensors across {ws} GPU(s), "
                                       "all-gather of stream lengths only")},
            "compression_ratio": round(m["all_stream_bytes"] / total_bytes, 6),
            "pipeline": pipeline,
            "kernels_ms_per_step": {k: round(v[1] / nprof, 4) for k, v in sorted(prof.items())},
            "roofline": roofline,
            "roofline_compress": roof_c,
            "roofline_decompress": roof_d,
            "delta_step": delta_step,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(round(m["launches_per_step"] * steps)),
            "clocks": m["clocks"],
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def measure_e2e(codec, ts, args, ws, dist, total_bytes, owned, n_total, prev=None):
    """Round trip through the public plan API with pinned host buffers, every
    step: H2D of the checkpoint into the registered tensors, CompressPlan.run,
    D2H of the streams; H2D of the streams, DecompressPlan.run, D2H of the
    payload.  Two buffer sets are pipelined across steps on three CUDA streams
    (H2D copies, compute, D2H copies), so one step's device->host copies run
    while the next step's host->device copies are in flight (the copy engines
    of the two directions work concurrently); every byte still crosses PCIe
    each step and every step's decode status is checked."""
    import torch

    import paper_2505_09810_b200 as lmcb

    n = len(ts)
    trace = bool(os.environ.get("LMC_E2E_TRACE"))
    # the checkpoint lives in one pinned host buffer and one device buffer per
    # set (tensors are 16-byte aligned views): one copy per direction
    offs, pos = [], 0
    for t in ts:
        offs.append(pos)
        pos += (t.numel() * t.element_size() + 15) & ~15
    host_all = torch.empty(pos, dtype=torch.uint8).pin_memory()
    for t, o in zip(ts, offs):
        host_all[o:o + t.numel() * t.element_size()].copy_(t.view(torch.uint8).reshape(-1).cpu())
    host = [host_all[o:o + t.numel() * t.element_size()] for t, o in zip(ts, offs)]
    sets = []
    for _ in range(2):
        dev_all = torch.empty(pos, dtype=torch.uint8, device="cuda")
        dev_in = [dev_all[o:o + t.numel() * t.element_size()].view(t.dtype).view(t.shape) for t, o in zip(ts, offs)]
        cp = codec.compress_plan(dev_in, prev=prev, graph=True)
        # the streams come back from the host into `ret`; the decompress plan's
        # graph decodes ret with the layout in `ret_meta`
        ret = types.SimpleNamespace(out=torch.empty_like(cp.out), meta=torch.empty_like(cp.meta))
        for t, o in zip(ts, offs):   # valid streams in ret before the plan's warm-up run
            dev_all[o:o + t.numel() * t.element_size()].copy_(t.view(torch.uint8).reshape(-1))
        cp.run()
        ret.out.copy_(cp.out)
        ret.meta.copy_(cp.meta)
        dp = lmcb.DecompressPlan(codec, cp.hints, cp.stream_bounds, graph=True, source=ret)
        sets.append({
            "dev_all": dev_all, "cp": cp, "dp": dp, "ret": ret,
            "host_streams": torch.empty(cp.bound, dtype=torch.uint8).pin_memory(),
            "host_out": torch.empty(dp.out.numel(), dtype=torch.uint8).pin_memory(),
            "host_meta": torch.empty(2 * n, dtype=torch.int64).pin_memory(),
            "ev": {k: torch.cuda.Event(enable_timing=trace) for k in ("in", "cmp", "meta", "d2h_s", "h2d_s", "dec", "free")},
            "used": False,
        })
    s_h2d, s_h2s, s_cmp, s_dec, s_d2h, s_d2s = (torch.cuda.Stream() for _ in range(6))
    status = torch.zeros((args.steps + 8, n), dtype=torch.int32, device="cuda")
    sizes = []

    def h2d_inputs(k):
        S = sets[k % 2]
        with torch.cuda.stream(s_h2d):
            if S["used"]:
                # compress k-2 has read the buffer; and the streams of step k-2 are
                # back on the device, so the copy engine alternates between the
                # front (checkpoint in) and the back (streams back) of the pipeline
                s_h2d.wait_event(S["ev"]["h2d_s"])
            S["dev_all"].copy_(host_all, non_blocking=True)
            S["ev"]["in"].record(s_h2d)

    def rest(k):
        S = sets[k % 2]
        cp, ev = S["cp"], S["ev"]
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev["in"])
            if S["used"]:
                s_cmp.wait_event(ev["d2h_s"])      # streams of step k-2 have left cp.out
            b = cp.run()
            exchange_lengths(b, owned, n_total, dist)
            S["ret"].meta.copy_(cp.meta)
            ev["cmp"].record(s_cmp)
            cp.layout_to_host(S["host_meta"], s_cmp)
            ev["meta"].record(s_cmp)
        return S

    def finish(k, S):
        cp, dp, ev, ret = S["cp"], S["dp"], S["ev"], S["ret"]
        ev["meta"].synchronize()
        m = S["host_meta"].tolist()
        total = m[n - 1] + m[2 * n - 1]
        sizes.append(total)
        with torch.cuda.stream(s_d2s):
            s_d2s.wait_event(ev["meta"])
            S["host_streams"][:total].copy_(cp.out[:total], non_blocking=True)
            ev["d2h_s"].record(s_d2s)
        with torch.cuda.stream(s_h2s):
            s_h2s.wait_event(ev["d2h_s"])
            if S["used"]:
                s_h2s.wait_event(ev["dec"])        # decompress k-2 has read ret
            ret.out[:total].copy_(S["host_streams"][:total], non_blocking=True)
            ev["h2d_s"].record(s_h2s)
        with torch.cuda.stream(s_dec):
            s_dec.wait_event(ev["h2d_s"])
            if S["used"]:
                s_dec.wait_event(ev["free"])        # payload of step k-2 has left dp.out
            r = dp.run()
            status[k % status.shape[0]].copy_(r._status_dev)
            ev["dec"].record(s_dec)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev["dec"])
            S["host_out"].copy_(dp.out, non_blocking=True)
            ev["free"].record(s_d2h)
        S["used"] = True

    def run(steps):
        # software pipeline: step k+1's compress is queued before the host
        # waits for step k's stream sizes
        h2d_inputs(0)
        pend = rest(0)
        if steps > 1:
            h2d_inputs(1)
        for k in range(steps):
            nxt = rest(k + 1) if k + 1 < steps else None
            finish(k, pend)
            if k + 2 < steps:
                h2d_inputs(k + 2)
            pend = nxt

    run(2)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_h2d)
    for st_ in (s_h2s, s_cmp, s_dec, s_d2h, s_d2s):
        st_.wait_stream(s_h2d)
    status.zero_()
    sizes.clear()
    run(args.steps)
    for st_ in (s_h2d, s_h2s, s_cmp, s_dec, s_d2s):
        s_d2h.wait_stream(st_)
    e1.record(s_d2h)
    torch.cuda.synchronize()
    if int(status.abs().sum().item()) != 0:
        bad = status.nonzero().tolist()
        raise SystemExit(f"e2e decode error: (step slot, stream) {bad[:8]} codes {[int(status[i, j]) for i, j in bad[:8]]}")
    # the payload that came back is the checkpoint
    S = sets[(args.steps - 1) % 2]
    for i, h in enumerate(host):
        o = S["dp"].offsets[i]
        want = h if prev is None else h ^ prev[i].view(torch.uint8).reshape(-1).cpu()
        if not torch.equal(S["host_out"][o:o + h.numel()], want):
            raise SystemExit("e2e round trip mismatch")
    if trace:
        for b, S in enumerate(sets):
            print("set", b, {k: round(e0.elapsed_time(v), 2) for k, v in S["ev"].items()}, file=sys.stderr)
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = ms.item()
    nbytes = sum(h.numel() for h in host)
    sb = max(sizes)
    del sets
    return {"value": round(total_bytes * args.steps / (ms / 1e3) / GIB, 3), "unit": "GiB/s",
            "h2d_bytes_per_step": nbytes + sb, "d2h_bytes_per_step": sb + nbytes,
            "path": "pinned host checkpoint -> H2D -> CompressPlan.run -> D2H streams -> H2D streams -> "
                    "DecompressPlan.run -> D2H payload; two buffer sets pipelined across steps on H2D / compute / "
                    "D2H streams" + (" (per rank: its own tensors; bytes per step are rank 0's)" if ws > 1 else "")}


def cpu_baseline(ts, prev=None):
    """Oracle (C port of the reference algorithm) on the host cores, bounded sample."""
    import torch

    from oracle import oracle as O

    cores = os.cpu_count() or 1
    raws, nb = [], 0
    order = list(range(2, len(ts))) + [0, 1] if len(ts) > 8 else list(range(len(ts)))  # skip embeddings first
    for i in order:
        x = ts[i].view(torch.uint8).reshape(-1)
        if prev is not None:
            x = x ^ prev[i].view(torch.uint8).reshape(-1)
        raws.append(x.cpu().numpy().tobytes())
        nb += len(raws[-1])
        if nb >= 24 << 20:
            break
    delta = prev is not None
    t0 = time.perf_counter()
    reps = 0
    while True:
        st = [O.compress(r, 1, delta=delta, threads=cores) for r in raws]
        for x in st:
            O.decompress(x, threads=cores)
        reps += 1
        if time.perf_counter() - t0 > 8.0:
            break
    dt = time.perf_counter() - t0
    return {"value": round(nb * reps / dt / GIB, 4), "unit": "GiB/s", "cores": cores, "kind": "port",
            "sample": f"{len(raws)} tensors of the checkpoint ({nb / 2**20:.1f} MiB) compress+decompress x{reps} "
                      f"with the C oracle port, {cores} threads"}


def main():
    args = parse_args()
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
