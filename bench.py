#!/usr/bin/env python
"""Benchmark of the continual-convolution step (BASELINE.json metric:
"stream-steps/sec per continual-conv layer at 1/2/4/8 B200; % of roofline").

One *step* = one ``co_forward_step`` of the bench layer over all of this
rank's streams (the whole hot path, in one kernel
launch).  Default workload: BASELINE.json configs[1] (C2: dense continual
Conv3d, 256 streams per GPU, 64->64, 3x3x3, 56x56, bf16 in/out, fp32 state).

Usage:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl co|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

Multi-GPU: streams are independent, so each rank runs its own shard of
streams (global streams [r*B, (r+1)*B), weak scaling: B fixed per GPU) with no
collective on the data path; NCCL only carries the barrier and the end-of-run
counters (MAX of elapsed, SUM of stream-steps).

Timing: W >= 3 untimed warm-up steps, then K steps timed with CUDA events on
the launching stream, bracketed by barrier + synchronize, max over ranks.  The
per-step working set (input frame + fp32 state ring + output, 616 MB for C2) is
larger than the 126 MB L2 and inputs rotate over a pool of distinct frames.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "stream-steps/sec per continual-conv layer"
UNIT = "stream-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=2, help="BASELINE.json config index (1-based)")
    ap.add_argument("--impl", default="co", choices=["co", "reference"])
    ap.add_argument("--streams", type=int, default=None, help="override streams per GPU")
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=8)
    return ap.parse_args()


# ----------------------------------------------------------------- distributed

def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def all_reduce(vals, op):
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return vals
    t = torch.tensor(vals, dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=op)
    return t.tolist()


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ----------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clock and throttle reasons via NVML on a background thread."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.ok = False
        self.samples = []
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()
        self._active = threading.Event()

    def sample(self):
        if not self.ok:
            return
        try:
            mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
            try:
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                rs = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            util = self.nv.nvmlDeviceGetUtilizationRates(self.h).gpu
            self.samples.append((mhz, rs, util))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            if self._active.is_set():
                self.sample()
            time.sleep(0.02)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._active.set()
        return self

    def __exit__(self, *a):
        self._active.clear()
        self._stop.set()
        self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": [],
                    "samples": 0}
        loaded = [s for s in self.samples if s[2] > 0] or self.samples
        reasons = set()
        for _, rs, _ in loaded:
            for bit, name in self.REASONS.items():
                if rs & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in loaded), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(loaded)}


# ----------------------------------------------------------------- workload

def layer_bytes_flops(L, cfg):
    """Algorithmic HBM bytes and FLOPs per stream-step of one layer:
    B_alg = x_t + y_t + 2 (kt-1) Cout H'W' * 4 (fp32 partial-sum state RMW);
    F = 2 Cout (Cin/g) kt kh kw H'W'."""
    H, W = cfg.in_spatial[0], (cfg.in_spatial[1] if cfg.spatial_rank >= 2 else 1)
    kh, kw = L.kernel[1], L.kernel[2]
    Ho = (H + 2 * L.padding[1] - L.dilation[1] * (kh - 1) - 1) // L.stride[1] + 1
    Wo = (W + 2 * L.padding[2] - L.dilation[2] * (kw - 1) - 1) // L.stride[2] + 1
    esz = 2 if str(cfg.dtype).endswith("bfloat16") else 4
    x_b = L.cin * H * W * esz
    y_b = L.cout * Ho * Wo * esz
    st_b = 2 * (L.kernel[0] - 1) * L.cout * Ho * Wo * 4
    flops = 2.0 * L.cout * (L.cin // L.groups) * L.kernel[0] * kh * kw * Ho * Wo
    return x_b + y_b + st_b, flops, (x_b, y_b, st_b)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j.get("hbm_gbs", 6650.0), j.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


def ncu_traffic(kernel_name):
    """dram bytes (read+write) per launch from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    return j.get(kernel_name)


def run_co(args, world, rank):
    import torch
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth

    cfg = synth.config(args.config)
    B = args.streams or cfg.n_streams
    if len(cfg.layers) != 1:
        raise SystemExit("bench.py times single-layer configs (C1, C2, C5); stacks: bench_stack.py")
    L = cfg.layers[0]
    (W, b) = synth.params(cfg)[0]
    conv = co.Conv(L.cin, L.cout, L.kernel, weight=W.cuda(), bias=b.cuda(), stride=L.stride, padding=L.padding,
                   dilation=L.dilation, groups=L.groups, spatial_rank=cfg.spatial_rank, in_spatial=cfg.in_spatial,
                   n_streams=B, dtype=cfg.dtype, out_dtype=cfg.dtype, kernel=args.kernel)
    frame_bytes = B * math.prod(synth.in_shape(cfg)) * (2 if cfg.dtype == torch.bfloat16 else 4)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    G = max(8, math.ceil(4 * l2 / frame_bytes))
    G = min(G, 64)
    n_global = B * world
    pool = [synth.frame(cfg, t, rank * B, (rank + 1) * B, n_global=n_global) for t in range(G)]
    y = co._empty_cl((B, L.cout) + conv.out_spatial, cfg.dtype, "cuda")
    stream = torch.cuda.current_stream()
    # warm-up: fill the delay so every timed step is a Ready (steady-state) step
    for n in range(max(args.warmup, 3, conv.delay + 1)):
        conv.forward_step(pool[n % G], out=y)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    K = args.steps
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    sampler = ClockSampler(torch.cuda.current_device())
    with sampler:
        ev[0].record(stream)
        for k in range(K):
            conv.forward_step(pool[k % G], out=y)
            ev[k + 1].record(stream)
        # sample clocks while the queued steps run
        t_end = time.time() + 30
        while not ev[K].query() and time.time() < t_end:
            sampler.sample()
            time.sleep(0.005)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    per = [ev[k].elapsed_time(ev[k + 1]) for k in range(K)]      # ms per launch (one kernel per step)
    elapsed_ms = ev[0].elapsed_time(ev[K])
    [elapsed_max] = all_reduce([elapsed_ms], op=_max_op())
    [total_ss] = all_reduce([float(B * K)], op=_sum_op())
    value = total_ss / (elapsed_max / 1e3)

    # roofline of the (single) step kernel
    bytes_ss, flops_ss, parts = layer_bytes_flops(L, cfg)
    hbm, bf16, src = measured_peaks()
    kern_ms = statistics.mean(per)
    ach_gbs = bytes_ss * B / (kern_ms / 1e3) / 1e9
    ach_tf = flops_ss * B / (kern_ms / 1e3) / 1e12
    t_hbm = bytes_ss / (hbm * 1e9)
    t_tc = flops_ss / (bf16 * 1e12)
    bound = "hbm" if t_hbm >= t_tc else "tensor"
    if conv.kernel_used == "direct" and cfg.dtype == torch.float32:
        bound = "hbm" if t_hbm >= flops_ss / 74.4e12 else "alu"
    roof = {"bound": bound, "kernel": conv.kernel_name, "peak_source": src}
    if bound == "hbm":
        roof.update({"achieved": round(ach_gbs, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach_gbs / hbm, 4)})
    elif bound == "tensor":
        roof.update({"achieved": round(ach_tf, 2), "peak": bf16, "unit": "TFLOP/s", "frac": round(ach_tf / bf16, 4)})
    else:
        roof.update({"achieved": round(ach_tf, 2), "peak": 74.4, "unit": "TFLOP/s", "frac": round(ach_tf / 74.4, 4)})
    tr = ncu_traffic(conv.kernel_name)
    roof["traffic"] = None if tr is None else tr.get("bytes_per_stream_step", 0) * B
    roof["alg_bytes_per_launch"] = bytes_ss * B
    roof["tensor_frac_of_peak"] = round(ach_tf / bf16, 4)

    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(elapsed_max / K, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16" if cfg.dtype == torch.bfloat16 else "f32",
        "data": "synthetic (seeded N(0,1) frames, N(0,1/fan_in) weights; BASELINE.json configs[%d])" % (args.config - 1),
        "config": {"workload": cfg.workload, "streams_per_gpu": B, "global_streams": n_global,
                   "layer": {"cin": L.cin, "cout": L.cout, "kernel": list(L.kernel), "padding": list(L.padding),
                             "stride": list(L.stride), "dilation": list(L.dilation), "groups": L.groups,
                             "in_spatial": list(cfg.in_spatial)},
                   "state": "fp32 partial-sum ring", "kernel": conv.kernel_name,
                   "parallelism": f"stream-shard x{world} (no data-path collective)",
                   "l2_policy": f"inputs larger than L2: per-step working set {round((frame_bytes + B*bytes_ss - parts[0]*B)/1e6)} MB "
                                f"> L2 {l2 // 2**20} MiB; input pool of {G} distinct frames"},
        "gpu_launches": K,
        "roofline": roof,
        "clocks": sampler.summary(),
    }
    return out, conv, pool, cfg, B


def _max_op():
    import torch.distributed as dist
    return dist.ReduceOp.MAX if dist.is_available() else None


def _sum_op():
    import torch.distributed as dist
    return dist.ReduceOp.SUM if dist.is_available() else None


def run_e2e(args, conv, pool, cfg, B, world):
    """Same metric through the public host-buffer API: H2D of the frame from
    pinned memory, the step, D2H of the output, every step."""
    import torch
    K = args.e2e_steps
    xh = [p.movedim(1, -1).contiguous().cpu().pin_memory() for p in pool[:2]]
    yh = torch.empty((B,) + tuple(conv.out_spatial) + (conv.out_channels,), dtype=conv.out_dtype).pin_memory()
    for i in range(2):
        conv.forward_step_host(xh[i % 2], yh)
    torch.cuda.synchronize()
    barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for k in range(K):
        conv.forward_step_host(xh[k % 2], yh)
    e.record()
    torch.cuda.synchronize()
    [ms] = all_reduce([s.elapsed_time(e)], op=_max_op())
    [tot] = all_reduce([float(B * K)], op=_sum_op())
    return {"value": round(tot / (ms / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": int(xh[0].numel() * xh[0].element_size()),
            "d2h_bytes_per_step": int(yh.numel() * yh.element_size()), "steps": K}


def oracle_sample(cfg, n_streams, ticks, pool_fn):
    """Time the fp64 oracle (as it stands) on `n_streams` streams for `ticks`
    Ready ticks after an untimed fill of the delay.  Returns (stream-steps/s, threads)."""
    import numpy as np
    import oracle as O
    L = cfg.layers[0]
    (W, b) = __import__("paper_2204_03418_b200.synth", fromlist=["params"]).params(cfg)[0]
    d = O.Desc(cfg.spatial_rank, L.cin, L.cout, L.kernel, L.stride, L.padding, L.dilation, L.groups, cfg.in_spatial)
    sm = O.StepMachine(d, W.double().numpy(), b.double().numpy(), n_streams)
    for t in range(d.delay):
        sm.forward_step(pool_fn(t))
    frames = [pool_fn(d.delay + t) for t in range(ticks)]
    t0 = time.perf_counter()
    for x in frames:
        assert sm.forward_step(x) is not None
    dt = time.perf_counter() - t0
    return n_streams * ticks / dt, dt


def cpu_baseline(cfg, B_gpu):
    """Oracle on a bounded sample of the same workload (about 10-30 s of CPU)."""
    import torch
    from paper_2204_03418_b200 import synth
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    S = min(cores, B_gpu)
    ticks = 2

    def pool_fn(t):
        return synth.frame(cfg, t, 0, S, device="cpu", n_global=cfg.n_streams).float().numpy()

    v, dt = oracle_sample(cfg, S, ticks, pool_fn)
    return {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"fp64 C oracle (OpenMP over streams), streams 0..{S-1} of {cfg.workload.split(':')[0]}, "
                      f"{ticks} Ready ticks after an untimed delay fill ({dt:.1f} s)"}


def run_reference(args, world, rank):
    """--impl reference: the oracle (deliberately slow fp64 CPU program) on this
    box's host cores, same config / metric / unit; rank 0 only."""
    import torch
    from paper_2204_03418_b200 import synth
    if rank != 0:
        return None
    cfg = synth.config(args.config)
    B = args.streams or cfg.n_streams
    cores = len(os.sched_getaffinity(0))
    S = min(cores, B)
    K = args.steps
    # bounded: each step is S streams x 1 Ready tick; cap the number of timed steps
    K_eff = max(1, min(K, 3))

    def pool_fn(t):
        return synth.frame(cfg, t, 0, S, device="cpu", n_global=cfg.n_streams).float().numpy()

    for _ in range(min(args.warmup, 1)):
        oracle_sample(cfg, S, 1, pool_fn)
    v, dt = oracle_sample(cfg, S, K_eff, pool_fn)
    return {"metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": world, "steps": K_eff,
            "warmup": args.warmup, "ms_per_step": round(dt / K_eff * 1e3, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.workload, "streams_per_step": S},
            "impl": "reference",
            "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{S} streams x {K_eff} Ready ticks per run (bounded sample of the workload)"},
            "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    import torch
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        out = run_reference(args, world, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    world, rank, local = dist_setup(args)
    out, conv, pool, cfg, B = run_co(args, world, rank)
    if not args.no_e2e:
        out["e2e"] = run_e2e(args, conv, pool, cfg, B, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, B)
    if rank == 0:
        print(json.dumps(out), flush=True)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
