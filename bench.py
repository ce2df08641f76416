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
    ap.add_argument("--streams", type=int, default=None, help="override streams per GPU (default: the config's count)")
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--state", default="psum", choices=["psum", "raw"],
                    help="per-stream state layout: fp32 partial-sum ring (the configs' 'fp32 state', default) or the "
                         "raw-input ring (SURVEY §8f f1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=16)
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


def barrier():
    from paper_2204_03418_b200 import shard
    shard.barrier()


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

def layer_geom(L, in_spatial, spatial_rank):
    H, W = in_spatial[0], (in_spatial[1] if spatial_rank >= 2 else 1)
    kh, kw = L.kernel[1], L.kernel[2]
    Ho = (H + 2 * L.padding[1] - L.dilation[1] * (kh - 1) - 1) // L.stride[1] + 1
    Wo = (W + 2 * L.padding[2] - L.dilation[2] * (kw - 1) - 1) // L.stride[2] + 1
    return H, W, Ho, Wo


def layer_bytes_flops(L, in_spatial, spatial_rank, esz, state="psum"):
    """Algorithmic HBM bytes and FLOPs per stream-step of one layer:
    PSUM: B_alg = x_t + y_t + 2 (kt-1) Cout H'W' * 4 (fp32 partial-sum state RMW);
    RAW:  B_alg = x_t + y_t + x_t (ring store) + (kt-1) x (the window's past frames);
    F = 2 Cout (Cin/g) kt kh kw H'W'."""
    H, W, Ho, Wo = layer_geom(L, in_spatial, spatial_rank)
    x_b = L.cin * H * W * esz
    y_b = L.cout * Ho * Wo * esz
    if state == "raw":
        st_b = L.kernel[0] * x_b
    else:
        st_b = 2 * (L.kernel[0] - 1) * L.cout * Ho * Wo * 4
    flops = 2.0 * L.cout * (L.cin // L.groups) * L.kernel[0] * L.kernel[1] * L.kernel[2] * Ho * Wo
    return x_b + y_b + st_b, flops, (x_b, y_b, st_b)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j.get("hbm_gbs", 6650.0), j.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


# FP32 CUDA-core peak (no measured figure exists): 148 SMs x 128 FP32 lanes x
# 2 FLOP/FMA x 1.965 GHz boost clock (B200_PROFILING.md unit counts / clocks).
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def ncu_traffic(key):
    """dram bytes (read+write) per stream-step of layer `key` ("<config>/L<i>") from the
    committed ncu --set full summaries (scripts/ncu_summary.py -> profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    return j.get(key)


def build_layers(cfg, B, kernel="auto", state="psum"):
    """The config's continual conv layers on this rank's B streams (bf16
    inter-layer activations, ReLU where the config says, A15)."""
    import torch
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    convs, spat = [], tuple(cfg.in_spatial)
    for L, (W, b) in zip(cfg.layers, synth.params(cfg)):
        c = co.Conv(L.cin, L.cout, L.kernel, weight=W.cuda(), bias=b.cuda(), stride=L.stride, padding=L.padding,
                    dilation=L.dilation, groups=L.groups, spatial_rank=cfg.spatial_rank, in_spatial=spat,
                    n_streams=B, dtype=cfg.dtype, out_dtype=cfg.dtype, activation="relu" if L.relu else None,
                    kernel=kernel, state_layout=state)
        convs.append(c)
        spat = tuple(c.out_spatial) + (1,) * (2 - len(c.out_spatial))
    return convs


def run_co(args, world, rank):
    import torch
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth

    cfg = synth.config(args.config)
    # weak scaling (the path partitions into independent streams): each rank runs
    # the config's stream count on its own GPU, global streams [r B, (r+1) B)
    from paper_2204_03418_b200 import shard as sh
    sd = sh.shard(rank, world, args.streams or cfg.n_streams)
    B, B_global = sd.per_rank, sd.n_global
    convs = build_layers(cfg, B, args.kernel, args.state)
    esz = 2 if cfg.dtype == torch.bfloat16 else 4
    frame_bytes = B * math.prod(synth.in_shape(cfg)) * esz
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    G = min(max(8, math.ceil(4 * l2 / frame_bytes)), 64)
    pool = [synth.frame(cfg, t, sd.lo, sd.hi, n_global=B_global) for t in range(G)]
    acts = [co._empty_cl((B, c.out_channels) + c.out_spatial, c.out_dtype, "cuda") for c in convs]
    stream = torch.cuda.current_stream()
    nL = len(convs)

    def tick(x, evs=None):
        cur = x
        for l, c in enumerate(convs):
            y = c.forward_step(cur, out=acts[l])
            if evs is not None:
                evs[l].record(stream)
            if y is None:
                return False
            cur = y
        return True

    # warm-up: fill every layer's delay so each timed tick runs all layers (steady state)
    d_nn = co.Stack(convs).delay if nL > 1 else convs[0].delay
    for n in range(max(args.warmup, 3) + d_nn):
        tick(pool[n % G])
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    K = args.steps
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    evl = [[torch.cuda.Event(enable_timing=True) for _ in range(nL)] for _ in range(K)]
    sampler = ClockSampler(torch.cuda.current_device())
    with sampler:
        for k in range(K):
            ev0[k].record(stream)
            assert tick(pool[k % G], evl[k])
        t_end = time.time() + 60
        while not evl[K - 1][-1].query() and time.time() < t_end:
            sampler.sample()
            time.sleep(0.005)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    elapsed_ms = ev0[0].elapsed_time(evl[K - 1][-1])
    layer_ms = [statistics.mean(([ev0[k].elapsed_time(evl[k][0]) for k in range(K)] if l == 0 else
                                 [evl[k][l - 1].elapsed_time(evl[k][l]) for k in range(K)])) for l in range(nL)]
    red = sh.reduce_counters(stream_steps=B * K, elapsed_ms=elapsed_ms)
    elapsed_max, value = red["elapsed_ms"], red["throughput"]

    hbm, bf16, src = measured_peaks()
    layers, spat = [], tuple(cfg.in_spatial)
    for l, (L, c) in enumerate(zip(cfg.layers, convs)):
        bytes_ss, flops_ss, parts = layer_bytes_flops(L, spat, cfg.spatial_rank, esz, args.state)
        spat = tuple(c.out_spatial) + (1,) * (2 - len(c.out_spatial))
        ms = layer_ms[l]
        t_hbm = bytes_ss / (hbm * 1e9)
        if c.kernel_used == "dense_tc":
            t_cmp, peak_c, unit_c, bound_c = flops_ss / (bf16 * 1e12), bf16, "TFLOP/s", "tensor"
        else:
            t_cmp, peak_c, unit_c, bound_c = flops_ss / (FP32_PEAK_TFLOPS * 1e12), FP32_PEAK_TFLOPS, "TFLOP/s", "alu"
        ach_gbs = bytes_ss * B / (ms / 1e3) / 1e9
        ach_tf = flops_ss * B / (ms / 1e3) / 1e12
        if t_hbm >= t_cmp:
            roof = {"bound": "hbm", "achieved": round(ach_gbs, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(ach_gbs / hbm, 4)}
        else:
            roof = {"bound": bound_c, "achieved": round(ach_tf, 2), "peak": round(peak_c, 1), "unit": unit_c,
                    "frac": round(ach_tf / peak_c, 4)}
        tr = ncu_traffic(f"{cfg.name}/L{l}" + ("/raw" if args.state == "raw" else ""))
        roof.update({"kernel": c.kernel_name, "ms_per_launch": round(ms, 4),
                     "alg_bytes_per_launch": int(bytes_ss * B), "alg_flops_per_launch": flops_ss * B,
                     "traffic": None if tr is None else int(tr.get("bytes_per_stream_step", 0) * B),
                     "peak_source": src, "tensor_or_alu_frac": round(ach_tf / peak_c, 4)})
        layers.append(roof)
    dom = max(range(nL), key=lambda l: layer_ms[l])
    roof = dict(layers[dom])
    if nL > 1:
        roof["share_of_step"] = round(layer_ms[dom] / sum(layer_ms), 4)
    L0 = cfg.layers[0]
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(elapsed_max / K, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16" if cfg.dtype == torch.bfloat16 else "f32",
        "data": "synthetic (seeded N(0,1) frames, N(0,1/fan_in) weights; BASELINE.json configs[%d])" % (args.config - 1),
        "config": {"workload": cfg.workload, "streams_per_gpu": B, "global_streams": B_global,
                   "layers": [{"cin": L.cin, "cout": L.cout, "kernel": list(L.kernel), "padding": list(L.padding),
                               "stride": list(L.stride), "dilation": list(L.dilation), "groups": L.groups,
                               "relu": L.relu} for L in cfg.layers],
                   "in_spatial": list(cfg.in_spatial),
                   "state": "fp32 partial-sum ring" if args.state == "psum" else "raw-input ring (bf16 frames)",
                   "kernels": [c.kernel_name for c in convs],
                   "parallelism": f"stream-shard x{world} (no data-path collective)",
                   "l2_policy": f"inputs larger than L2: per-step working set "
                                f"{round(sum(l['alg_bytes_per_launch'] for l in layers) / 1e6)} MB > L2 "
                                f"{l2 // 2**20} MiB; input pool of {G} distinct frames"},
        "gpu_launches": K * nL,
        "roofline": roof,
        "layers": layers if nL > 1 else None,
        "clocks": sampler.summary(),
    }
    return out, convs, pool, cfg, B


def run_e2e(args, convs, pool, cfg, B, world):
    """Same metric through the public host-buffer C-ABI streaming call
    (co_forward_steps_host / co_stack_steps_host): every step copies its frame
    H2D from pinned memory and its output D2H, overlapped with the neighbouring
    steps' compute; timed on the host around the (synchronising) call."""
    import torch
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import shard as sh
    last = convs[-1]
    stack = co.Stack(convs) if len(convs) > 1 else None
    target = stack or last
    frame = pool[0].movedim(1, -1).contiguous()
    fbytes = frame.numel() * frame.element_size()
    K = max(4, min(args.e2e_steps, (2 << 30) // fbytes))
    xh = torch.empty((K,) + tuple(frame.shape), dtype=frame.dtype).pin_memory()
    for k in range(K):
        xh[k].copy_(pool[k % len(pool)].movedim(1, -1))
    yh = torch.empty((K, B) + tuple(last.out_spatial) + (last.out_channels,), dtype=last.out_dtype).pin_memory()
    target.forward_steps_host(xh[:2], yh)            # warm-up (allocates the staging buffers)
    torch.cuda.synchronize()
    sh.barrier()
    t0 = time.perf_counter()
    n, _ = target.forward_steps_host(xh, yh)
    dt = time.perf_counter() - t0
    assert n == K                                    # delay already filled by the timed run
    red = sh.reduce_counters(stream_steps=B * K, elapsed_ms=dt * 1e3)
    return {"value": round(red["throughput"], 1), "unit": UNIT, "h2d_bytes_per_step": int(fbytes),
            "d2h_bytes_per_step": int(yh[0].numel() * yh.element_size()), "steps": K,
            "api": "co_stack_steps_host" if stack else "co_forward_steps_host"}


def oracle_machine(cfg, n_streams):
    """The fp64 oracle for the config: a StepMachine (one layer) or a Stack."""
    import oracle as O
    from paper_2204_03418_b200 import synth
    params = synth.params(cfg)
    descs, spat = [], tuple(cfg.in_spatial)
    for L in cfg.layers:
        d = O.Desc(cfg.spatial_rank, L.cin, L.cout, L.kernel, L.stride, L.padding, L.dilation, L.groups, spat)
        descs.append(d)
        spat = d.out_spatial
    Ws = [W.double().numpy() for W, _ in params]
    bs = [b.double().numpy() for _, b in params]
    if len(descs) == 1:
        return O.StepMachine(descs[0], Ws[0], bs[0], n_streams), descs[0].delay
    nL = len(descs)
    st = O.Stack(descs, Ws, bs, [int(L.relu) for L in cfg.layers], [1] * (nL - 1) + [0], n_streams)
    return st, sum(d.delay for d in descs)


def oracle_sample(cfg, n_streams, ticks, pool_fn):
    """Time the fp64 oracle (as it stands) on `n_streams` streams for `ticks`
    Ready ticks after an untimed fill of the delay.  Returns (stream-steps/s, seconds)."""
    sm, delay = oracle_machine(cfg, n_streams)
    for t in range(delay):
        sm.forward_step(pool_fn(t))
    frames = [pool_fn(delay + t) for t in range(ticks)]
    t0 = time.perf_counter()
    for x in frames:
        assert sm.forward_step(x) is not None
    dt = time.perf_counter() - t0
    return n_streams * ticks / dt, dt


def cpu_baseline(cfg, B_gpu):
    """Oracle on a bounded sample of the same workload (about 10-30 s of CPU)."""
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
    out, convs, pool, cfg, B = run_co(args, world, rank)
    if not args.no_e2e:
        out["e2e"] = run_e2e(args, convs, pool, cfg, B, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, B)
    if rank == 0:
        print(json.dumps(out), flush=True)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
