#!/usr/bin/env python
"""Benchmark of the continual-convolution step (BASELINE.json metric:
"stream-steps/sec per continual-conv layer at 1/2/4/8 B200; % of roofline").

One *step* = one tick of a config's whole layer chain
over all of this rank's streams.  The printed JSON line's headline is
BASELINE.json configs[1] (C2: dense continual Conv3d, 256 global streams,
64->64, 3x3x3, 56x56, bf16 in/out, fp32 state); its "configs" object carries
every config C1-C5 (and C5 in both state layouts) with per-layer rooflines and
the clocks seen while that config ran.

Usage:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config all|1..5] [--impl co|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

Multi-GPU: streams are independent, so strong scaling
(default) splits each config's global streams into contiguous per-rank blocks
(shard.py) with no collective on the data path; NCCL carries only the barrier
and the end-of-run counters (MAX of elapsed, SUM of stream-steps).
--scaling weak gives every rank the config's full count instead.

Timing: W >= 3 untimed warm-up ticks after the delay fill; then the K timed
ticks are ONE replay of a CUDA graph holding them (co_stack_graph_create: the
serving loop without per-tick host work), bracketed by barrier + synchronize,
CUDA events on the launching stream, max over ranks.  A second, eager pass of
K ticks with CUDA events between layers gives each layer's (kernel's) launch
time for the roofline.  Every config's per-step working set (input frame +
fp32 state ring + output; 0.3-7 GB) is larger than the 126 MB L2 and inputs
rotate over a pool of distinct frames, so no L2 flush is needed.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "stream-steps/sec per continual-conv layer"
UNIT = "stream-steps/s"
HEADLINE = 2                       # BASELINE.json configs[1]: the config the metric is quoted on (fits one GPU)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="all",
                    help="'all' (headline C2 + every config in 'configs') or one BASELINE.json config index (1-based)")
    ap.add_argument("--impl", default="co", choices=["co", "reference"])
    ap.add_argument("--streams", type=int, default=None, help="override the config's global stream count")
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--state", default="config", choices=["config", "psum", "raw", "auto"],
                    help="state layout: 'config' = what BASELINE.json's config states (fp32 partial sums where it "
                         "says fp32 state, the planner's choice otherwise)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-graph", action="store_true", help="time the eager tick loop instead of a graph replay")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=48,
                    help="steps streamed through the host-buffer call (the pipeline fill / drain is one step's "
                         "transfer: 48 steps keep it near 2%% of the timed region)")
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="documented planner option (co_set_option) for A/B runs; recorded in the line")
    ap.add_argument("--dry-run", action="store_true",
                    help="host logic only (CPU): shards, counters and the JSON line, no GPU work (tests)")
    return ap.parse_args(argv)


# ----------------------------------------------------------------- distributed

def dist_setup(dry=False):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if dry:
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif not dry:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier():
    from paper_2204_03418_b200 import shard
    shard.barrier()


# ----------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM / memory clocks, throttle reasons and power via NVML on a
    background thread while a timed region runs."""

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
            nv = self.nv
            mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            mem = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_MEM)
            try:
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
            try:
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                temp = nv.nvmlDeviceGetTemperature(self.h, nv.NVML_TEMPERATURE_GPU)
            except Exception:
                pw, temp = None, None
            self.samples.append((mhz, rs, util, mem, pw, temp))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            if self._active.is_set():
                self.sample()
            time.sleep(0.01)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._active.set()
        self.sample()
        return self

    def __exit__(self, *a):
        self.sample()
        self._active.clear()
        self._stop.set()
        self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": [], "samples": 0}
        loaded = [s for s in self.samples if s[2] > 0] or self.samples
        reasons = set()
        for s in loaded:
            for bit, name in self.REASONS.items():
                if s[1] & bit and name != "gpu_idle":
                    reasons.add(name)
        out = {"sm_mhz": statistics.median(s[0] for s in loaded), "sm_max_mhz": self.max_mhz,
               "reasons": sorted(reasons), "samples": len(loaded),
               "mem_mhz": statistics.median(s[3] for s in loaded)}
        pw = [s[4] for s in loaded if s[4] is not None]
        if pw:
            out["power_w_median"] = round(statistics.median(pw), 1)
            out["temp_c_max"] = max(s[5] for s in loaded if s[5] is not None)
        return out


# ----------------------------------------------------------------- workload arithmetic

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
    """(HBM GB/s, bf16 TFLOP/s burst, bf16 sustained, source) from the driver-written MEASURED_PEAKS.json."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return (j.get("hbm_gbs", 6650.0), j.get("bf16_tflops", 1590.0), j.get("bf16_tflops_sustained", 1400.0),
                "measured")
    return 6650.0, 1590.0, 1400.0, "fallback"


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


def state_of(cfg, args):
    """State layout per config: BASELINE.json states 'fp32 state' for C2-C4 (the
    partial-sum ring) and C1 is fp32 throughout; C3 and C5 state only
    'bf16', so the planner's layout choice (CO_STATE_AUTO) applies there (C3: both
    depthwise layers take the RAW frame ring with the frame store fused)."""
    if args.state != "config":
        return args.state
    return "auto" if cfg.cid in (3, 5) else "psum"


def build_layers(cfg, B, kernel="auto", state="psum"):
    """The config's continual conv layers on this rank's B streams (bf16
    inter-layer activations, ReLU where the config says, A15)."""
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


def launches_per_tick(convs):
    """Kernels one tick launches (our own kernels only)."""
    return sum(2 if "wcols" in c.kernel_name and "fused" not in c.kernel_name else 1 for c in convs)


# ----------------------------------------------------------------- one config

def run_config(cfg, args, world, rank, label=None, state=None):
    """Time one config on this rank's shard: a graph replay of K ticks (the
    value) and an eager pass with per-layer events (the rooflines)."""
    import torch
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import shard as sh
    from paper_2204_03418_b200 import synth

    state = state or state_of(cfg, args)
    n_global = args.streams or cfg.n_streams
    sd = sh.shard(rank, world, n_global, args.scaling)
    B = sd.per_rank
    convs = build_layers(cfg, B, args.kernel, state)
    layouts = [c.state_layout_used for c in convs]
    stack = co.Stack(convs)
    esz = 2 if cfg.dtype == torch.bfloat16 else 4
    frame_bytes = B * math.prod(synth.in_shape(cfg)) * esz
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    G = min(max(8, math.ceil(4 * l2 / frame_bytes)), 64)
    pool = [synth.frame(cfg, t, sd.lo, sd.hi, n_global=sd.n_global) for t in range(G)]
    acts = [co._empty_cl((B, c.out_channels) + c.out_spatial, c.out_dtype, "cuda") for c in convs]
    stream = torch.cuda.current_stream()
    nL = len(convs)
    K = args.steps

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

    # warm-up: fill the stack's delay so every timed tick runs all layers (steady state)
    d_nn = stack.delay
    for n in range(max(args.warmup, 3) + d_nn):
        tick(pool[n % G])
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device())
    graph_ms = None
    pdl = None
    with sampler:
        if not args.no_graph:
            g = stack.capture([pool[k % G] for k in range(K)], [acts[-1]] * K)
            g.upload()
            pdl = g.pdl
            torch.cuda.synchronize()
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            n_ready = g.launch()
            e1.record(stream)
            t_end = time.time() + 60
            while not e1.query() and time.time() < t_end:
                sampler.sample()
                time.sleep(0.002)
            torch.cuda.synchronize()
            barrier()
            torch.cuda.synchronize()
            assert n_ready == K, (n_ready, K)
            graph_ms = e0.elapsed_time(e1)
            del g
        # eager pass: per-layer CUDA events (the kernels' launch times for the roofline)
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        evl = [[torch.cuda.Event(enable_timing=True) for _ in range(nL)] for _ in range(K)]
        barrier()
        torch.cuda.synchronize()
        for k in range(K):
            ev0[k].record(stream)
            assert tick(pool[k % G], evl[k])
        t_end = time.time() + 60
        while not evl[K - 1][-1].query() and time.time() < t_end:
            sampler.sample()
            time.sleep(0.002)
        torch.cuda.synchronize()
        barrier()
    eager_ms = ev0[0].elapsed_time(evl[K - 1][-1])
    layer_ms = [statistics.mean(([ev0[k].elapsed_time(evl[k][0]) for k in range(K)] if l == 0 else
                                 [evl[k][l - 1].elapsed_time(evl[k][l]) for k in range(K)])) for l in range(nL)]
    # a single-kernel tick timed as a graph replay: the replay IS the kernel's K
    # launches back to back, so its per-launch time comes from the replay (the
    # eager pass adds a launch gap per tick); RAW layers add a frame copy, so
    # they keep the eager per-layer events
    one_kernel = (nL == 1 and graph_ms is not None and launches_per_tick(convs) == 1 and layouts[0] != "raw")
    if one_kernel:
        layer_ms = [graph_ms / K]
    elapsed_ms = graph_ms if graph_ms is not None else eager_ms
    red = sh.reduce_counters(stream_steps=B * K, elapsed_ms=elapsed_ms)
    red_e = sh.reduce_counters(stream_steps=B * K, elapsed_ms=eager_ms)

    hbm, bf16, bf16_sus, src = measured_peaks()
    clocks = sampler.summary()
    # a kernel timed inside a long power-capped step gets the sustained tensor peak (B200_PROFILING.md)
    capped = "sw_power_cap" in clocks.get("reasons", [])
    t_peak = bf16_sus if capped else bf16
    layers, spat = [], tuple(cfg.in_spatial)
    for l, (L, c) in enumerate(zip(cfg.layers, convs)):
        bytes_ss, flops_ss, parts = layer_bytes_flops(L, spat, cfg.spatial_rank, esz, layouts[l])
        spat = tuple(c.out_spatial) + (1,) * (2 - len(c.out_spatial))
        ms = layer_ms[l]
        t_hbm = bytes_ss / (hbm * 1e9)
        if c.kernel_used == "dense_tc":
            t_cmp, peak_c, bound_c = flops_ss / (t_peak * 1e12), t_peak, "tensor"
        else:
            t_cmp, peak_c, bound_c = flops_ss / (FP32_PEAK_TFLOPS * 1e12), FP32_PEAK_TFLOPS, "alu"
        ach_gbs = bytes_ss * B / (ms / 1e3) / 1e9
        ach_tf = flops_ss * B / (ms / 1e3) / 1e12
        if t_hbm >= t_cmp:
            roof = {"bound": "hbm", "achieved": round(ach_gbs, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(ach_gbs / hbm, 4)}
        else:
            roof = {"bound": bound_c, "achieved": round(ach_tf, 2), "peak": round(peak_c, 1), "unit": "TFLOP/s",
                    "frac": round(ach_tf / peak_c, 4)}
            if bound_c == "tensor":
                roof["peak_kind"] = "sustained (sw_power_cap seen)" if capped else "burst"
        tr = ncu_traffic(f"{cfg.name}/L{l}" + ("/raw" if layouts[l] == "raw" else ""))
        roof.update({"kernel": c.kernel_name, "state": layouts[l], "ms_per_launch": round(ms, 4),
                     "ms_source": "graph replay (one kernel per tick)" if one_kernel else "eager pass, CUDA events",
                     "stream_steps_per_s": round(B / (ms / 1e3), 1),
                     "alg_bytes_per_launch": int(bytes_ss * B), "alg_flops_per_launch": flops_ss * B,
                     "traffic": None if tr is None else int(tr.get("bytes_per_stream_step", 0) * B),
                     "peak_source": src, "tensor_or_alu_frac": round(ach_tf / peak_c, 4),
                     "roofline_stream_steps_per_s": round(1.0 / max(t_hbm, t_cmp), 1)})
        layers.append(roof)
    dom = max(range(nL), key=lambda l: layer_ms[l])
    roof = dict(layers[dom])
    roof["share_of_step"] = round(layer_ms[dom] / eager_ms * K, 4) if eager_ms > 0 else None
    entry = {
        "workload": label or cfg.workload, "value": round(red["throughput"], 1), "unit": UNIT,
        "ms_per_step": round(red["elapsed_ms"] / K, 4), "timing": "graph" if graph_ms is not None else "eager",
        "eager_value": round(red_e["throughput"], 1), "graph_pdl": pdl,
        "streams_per_gpu": B, "global_streams": sd.n_global, "shard": [sd.lo, sd.hi], "scaling": sd.scaling,
        "state": layouts, "kernels": [c.kernel_name for c in convs],
        "gpu_launches": (1 if graph_ms is None else 2) * K * launches_per_tick(convs),   # graph + eager passes
        "roofline": roof, "layers": layers, "clocks": clocks,
        "l2_policy": f"inputs larger than L2: per-step working set "
                     f"{round(sum(l['alg_bytes_per_launch'] for l in layers) / 1e6)} MB > L2 {l2 // 2**20} MiB; "
                     f"input pool of {G} distinct frames",
    }
    return entry, (convs, stack, pool, cfg, B)


def run_e2e(args, convs, stack, pool, cfg, B, world):
    """Same metric through the public host-buffer C-ABI streaming call
    (co_stack_steps_host): every step copies its frame H2D from pinned memory
    and its output D2H, overlapped with the neighbouring steps' compute; timed
    on the host around the (synchronising) call."""
    import torch
    from paper_2204_03418_b200 import shard as sh
    last = convs[-1]
    frame = pool[0].movedim(1, -1).contiguous()
    fbytes = frame.numel() * frame.element_size()
    K = max(4, min(args.e2e_steps, (5 << 30) // fbytes))   # pinned host frames <= 5 GiB
    xh = torch.empty((K,) + tuple(frame.shape), dtype=frame.dtype).pin_memory()
    for k in range(K):
        xh[k].copy_(pool[k % len(pool)].movedim(1, -1))
    yh = torch.empty((K, B) + tuple(last.out_spatial) + (last.out_channels,), dtype=last.out_dtype).pin_memory()
    stack.forward_steps_host(xh[:2], yh)            # warm-up (allocates the staging buffers)
    torch.cuda.synchronize()
    sh.barrier()
    t0 = time.perf_counter()
    n, _ = stack.forward_steps_host(xh, yh)
    dt = time.perf_counter() - t0
    assert n == K                                    # delay already filled by the timed run
    red = sh.reduce_counters(stream_steps=B * K, elapsed_ms=dt * 1e3)
    return {"value": round(red["throughput"], 1), "unit": UNIT, "h2d_bytes_per_step": int(fbytes),
            "d2h_bytes_per_step": int(yh[0].numel() * yh.element_size()), "steps": K,
            "api": "co_stack_steps_host"}


# ----------------------------------------------------------------- oracle legs (CPU)

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


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _oracle_leg(cid, threads, ticks):
    """Child process: the oracle with exactly `threads` OpenMP threads."""
    from paper_2204_03418_b200 import synth
    cfg = synth.config(cid)
    S = threads

    def pool_fn(t):
        return synth.frame(cfg, t, 0, S, device="cpu", n_global=cfg.n_streams).float().numpy()

    v, dt = oracle_sample(cfg, S, ticks, pool_fn)
    return {"value": v, "seconds": dt, "streams": S, "ticks": ticks}


def oracle_threads_run(cid, threads, ticks):
    env = dict(os.environ, OMP_NUM_THREADS=str(threads), OMP_PROC_BIND="false")
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-leg", str(cid), str(threads),
                          str(ticks)], env=env, capture_output=True, text=True, timeout=600)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    if not lines:
        raise RuntimeError(out.stderr[-500:])
    return json.loads(lines[-1])


def cpu_baseline(cfg):
    """The fp64 oracle, as it stands, on a bounded sample of the same workload
    (about 10-30 s of CPU): all host cores (one stream per core, OpenMP over
    streams) and one core (one stream), each over 2 Ready ticks after an untimed
    delay fill; the core count and CPU model as measured on this host."""
    cores = len(os.sched_getaffinity(0))
    ticks = 2
    allc = oracle_threads_run(cfg.cid, min(cores, cfg.n_streams), ticks)
    one = oracle_threads_run(cfg.cid, 1, ticks)
    return {"value": round(allc["value"], 3), "unit": UNIT, "cores": min(cores, cfg.n_streams), "kind": "oracle",
            "value_1core": round(one["value"], 3), "cpu_model": cpu_model(), "host_cores": cores,
            "sample": f"fp64 C oracle (OpenMP over streams), {cfg.workload.split(':')[0]}: streams 0..{allc['streams']-1}"
                      f" x {ticks} Ready ticks on {allc['streams']} threads ({allc['seconds']:.1f} s) and stream 0 x "
                      f"{ticks} Ready ticks on 1 thread ({one['seconds']:.1f} s), after an untimed delay fill"}


def run_reference(args, world, rank):
    """--impl reference: the oracle (deliberately slow fp64 CPU program) on this
    box's host cores, same config / metric / unit; rank 0 only."""
    from paper_2204_03418_b200 import synth
    if rank != 0:
        return None
    cid = HEADLINE if args.config == "all" else int(args.config)
    cfg = synth.config(cid)
    B = args.streams or cfg.n_streams
    cores = len(os.sched_getaffinity(0))
    S = min(cores, B)
    K_eff = max(1, min(args.steps, 3))          # bounded: each step is S streams x 1 Ready tick

    def pool_fn(t):
        return synth.frame(cfg, t, 0, S, device="cpu", n_global=cfg.n_streams).float().numpy()

    for _ in range(min(args.warmup, 1)):
        oracle_sample(cfg, S, 1, pool_fn)
    v, dt = oracle_sample(cfg, S, K_eff, pool_fn)
    return {"metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": world, "steps": K_eff,
            "warmup": args.warmup, "ms_per_step": round(dt / K_eff * 1e3, 2), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.workload, "streams_per_step": S},
            "impl": "reference",
            "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": S, "kind": "oracle",
                             "cpu_model": cpu_model(), "host_cores": cores,
                             "sample": f"{S} streams x {K_eff} Ready ticks per run (bounded sample of the workload)"},
            "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ----------------------------------------------------------------- hygiene

def check_environment(args):
    """The release library reads no environment variable; a CO_* variable in
    the environment means an experiment setup (CO_LIB_VARIANT loads an
    experiment build whose A/B knobs can skip work).  Refuse those; record the
    documented options (co_set_option) in the line."""
    bad = {k: v for k, v in os.environ.items() if k.startswith("CO_")}
    if bad:
        print(json.dumps({"error": "refusing to benchmark with CO_* environment variables set "
                                   "(experiment build / A/B knobs)", "env": bad}), flush=True)
        sys.exit(2)


def apply_options(args):
    import paper_2204_03418_b200 as co
    co.reset_options()
    for kv in args.option:
        k, v = kv.split("=", 1)
        co.set_option(k, int(v))
    return co.all_options()


# ----------------------------------------------------------------- main

def assemble(head, configs, args, world, options):
    """The one JSON line: the headline config's fields at the top level plus every config."""
    import torch
    from paper_2204_03418_b200 import synth
    cfg = synth.config(HEADLINE if args.config == "all" else int(args.config))
    out = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if args.scaling == "strong" else "weak", "vs_baseline": None,
        "dtype": "bf16" if cfg.dtype == torch.bfloat16 else "f32",
        "data": "synthetic (seeded N(0,1) frames, N(0,1/fan_in) weights; BASELINE.json configs[%d])" % (cfg.cid - 1),
        "config": {"workload": cfg.workload, "streams_per_gpu": head["streams_per_gpu"],
                   "global_streams": head["global_streams"],
                   "layers": [{"cin": L.cin, "cout": L.cout, "kernel": list(L.kernel), "padding": list(L.padding),
                               "stride": list(L.stride), "dilation": list(L.dilation), "groups": L.groups,
                               "relu": L.relu} for L in cfg.layers],
                   "in_spatial": list(cfg.in_spatial), "state": head["state"], "kernels": head["kernels"],
                   "parallelism": f"stream-shard x{world} ({args.scaling} scaling, no data-path collective)",
                   "timing": head["timing"], "l2_policy": head["l2_policy"], "options": options},
        "gpu_launches": sum(c.get("gpu_launches", 0) for c in configs.values()),
        "roofline": head["roofline"], "layers": head["layers"] if len(head["layers"]) > 1 else None,
        "clocks": head["clocks"],
        "configs": configs,
    }
    return out


def main(argv=None):
    args = parse(argv)
    check_environment(args)
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        out = run_reference(args, world, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    world, rank, local = dist_setup(args.dry_run)
    if args.dry_run:
        out = dry_run(args, world, rank)
    else:
        out = run_all(args, world, rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


def run_all(args, world, rank):
    import gc
    import torch
    from paper_2204_03418_b200 import synth
    options = apply_options(args)
    cids = [HEADLINE, 1, 3, 4, 5] if args.config == "all" else [int(args.config)]
    configs, head, keep = {}, None, None
    for cid in cids:
        cfg = synth.config(cid)
        entry, ctx = run_config(cfg, args, world, rank)
        configs[f"C{cid}"] = entry
        if cid == cids[0]:
            head, keep = entry, ctx
            if not args.no_e2e:
                head["e2e"] = run_e2e(args, *ctx[:5], world)
            if rank == 0 and world == 1 and not args.no_cpu_baseline:
                head["cpu_baseline"] = cpu_baseline(cfg)
        if cid == 4 and args.config == "all" and args.state == "config":
            # C4's companion: the planner's layout per layer (CO_STATE_AUTO), i.e. the RGB stem
            # over the RAW frame ring (k_step_stem_raw), the rest on fp32 partial sums
            e2, _ = run_config(cfg, args, world, rank, label=cfg.workload + " [planner layouts: RAW-ring stem]",
                               state="auto")
            configs["C4/auto"] = e2
        if cid in (3, 5) and args.config == "all" and args.state == "config" and set(entry["state"]) != {"psum"}:
            # C3's / C5's companion: the fp32 partial-sum layout against its own roofline
            e2, _ = run_config(cfg, args, world, rank, label=cfg.workload + " [fp32 partial-sum state]",
                               state="psum")
            configs[f"C{cid}/psum"] = e2
        del ctx
        gc.collect()
        torch.cuda.empty_cache()
    out = assemble(head, configs, args, world, options)
    if "e2e" in head:
        out["e2e"] = head.pop("e2e")
    if "cpu_baseline" in head:
        out["cpu_baseline"] = head.pop("cpu_baseline")
    return out


def dry_run(args, world, rank):
    """Host logic without a GPU (tests, gloo): the shards every config would
    run, the counter reduction and the line's shape, with zero-cost stand-in
    timings (each rank 'takes' 1 + rank ms per step)."""
    from paper_2204_03418_b200 import shard as sh
    from paper_2204_03418_b200 import synth
    cids = [HEADLINE, 1, 3, 4, 5] if args.config == "all" else [int(args.config)]
    configs = {}
    for cid in cids:
        cfg = synth.config(cid)
        sd = sh.shard(rank, world, args.streams or cfg.n_streams, args.scaling)
        red = sh.reduce_counters(stream_steps=sd.per_rank * args.steps, elapsed_ms=(1.0 + rank) * args.steps)
        configs[f"C{cid}"] = {"workload": cfg.workload, "value": red["throughput"], "unit": UNIT,
                              "ms_per_step": red["elapsed_ms"] / args.steps, "streams_per_gpu": sd.per_rank,
                              "global_streams": sd.n_global, "shard": [sd.lo, sd.hi], "scaling": sd.scaling,
                              "stream_steps": red["stream_steps"], "timing": "dry-run", "state": ["psum"],
                              "kernels": [], "gpu_launches": 0, "roofline": None, "layers": [], "clocks": None,
                              "l2_policy": None}
    head = configs[f"C{cids[0]}"]
    return assemble(head, configs, args, world, {})


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--oracle-leg":
        cid, threads, ticks = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
        print(json.dumps(_oracle_leg(cid, threads, ticks)), flush=True)
    else:
        main()
