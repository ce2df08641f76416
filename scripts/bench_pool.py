#!/usr/bin/env python
"""Benchmark of continual pooling, the companion of
bench.py for the pooling handles (co_op MAX / AVG).  Prints one JSON line per
workload with bench.py's timing rules: W >= 3 untimed warm-up steps, K steps
timed with CUDA events on the launching stream, synchronize on both sides,
NVML clocks sampled during the timed region, inputs rotating over a pool of
distinct frames larger than L2.

Workloads (seeded N(0,1) bf16 frames; no BASELINE.json config covers pooling):
  x3d64  -- the paper's expanded temporal global average pooling (P:642,
            CoX3D-M_64, Table 2): AvgPool (64, 7, 7) over the 7x7x432
            conv5 output of X3D-M at 224 px, 512 streams (C3's stream count).
  max3   -- an I3D-style max pool (3, 3, 3), stride (1, 2, 2), padding
            (0, 1, 1) on the C2 activation shape (56x56x64, 256 streams).

Algorithmic bytes per stream-step (alg_bytes; k_pool.cu): x (H W C, bf16) +
y (H' W' C) + the reduced-frame slots the temporal scheme touches (H' W' C x
ring esz each; input dtype for MAX, fp32 for AVG): kt for the direct fold, about
6 for the block decomposition used when kt >= 6.

usage: python scripts/bench_pool.py [--workload x3d64|max3|all] [--steps K] [--warmup W]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "x3d64": dict(kind="avg", C=432, H=7, W=7, kernel=(64, 7, 7), stride=(1, 1, 1), padding=(0, 0, 0), B=512,
                  desc="expanded temporal global avg pool, CoX3D-M_64 head (P:642): AvgPool(64,7,7), 7x7x432, 512 streams"),
    "max3": dict(kind="max", C=64, H=56, W=56, kernel=(3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), B=256,
                 desc="I3D-style MaxPool(3,3,3) s(1,2,2) p(0,1,1) on 56x56x64, 256 streams"),
}


def alg_bytes(w, Ho, Wo, vh):
    """Bytes per stream-step the step kernel must move (k_pool.cu): the frame,
    the output, and reduced-frame slots -- direct fold: 1 ring write + kt-1 ring
    reads; block decomposition (vh): 1 ring write, P read + write, S read, and
    the suffix pass's 2kt-1 slot accesses once per kt steps (amortized)."""
    esz, resz = 2, (4 if w["kind"] == "avg" else 2)
    kt = w["kernel"][0]
    x = w["H"] * w["W"] * w["C"] * esz
    y = Ho * Wo * w["C"] * esz
    slot = Ho * Wo * w["C"] * resz
    slots = (1 + (kt - 1) / kt + 1 + (kt - 1) / kt + (2 * kt - 1) / kt) if vh else kt
    return x + y + slots * slot


def run(name, steps, warmup):
    import torch
    import paper_2204_03418_b200 as co
    from bench import ClockSampler, measured_peaks

    w = WORKLOADS[name]
    B, C, H, W = w["B"], w["C"], w["H"], w["W"]
    p = co.Pool(w["kind"], C, w["kernel"], stride=w["stride"], padding=w["padding"], in_spatial=(H, W), n_streams=B)
    Ho, Wo = p.out_spatial
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    fbytes = B * C * H * W * 2
    G = min(max(4, math.ceil(4 * l2 / fbytes)), 32)
    g = torch.Generator(device="cuda").manual_seed(1234)
    # G distinct frames as one device clip (B, C, G, H, W); each co_forward_steps
    # call folds co_forward_step over its G columns in C (one launch per step,
    # no Python per step -- the per-call Python/ctypes cost exceeds the x3d64 kernel)
    clip = co.channels_last(torch.randn((B, C, G, H, W), generator=g, device="cuda").to(torch.bfloat16))
    stream = torch.cuda.current_stream()
    warm = co.channels_last(clip[:, :, :1].repeat(1, 1, max(warmup, 3) + p.delay, 1, 1))
    p.forward_steps(warm)
    torch.cuda.synchronize()
    steps = max(G, (steps + G - 1) // G * G)
    # the timed ticks: one CUDA-graph replay (co_stack_graph_create) of `steps`
    # pooling steps over the G frames -- the serving loop without launch gaps
    st = co.Stack([p])
    frames = [co.channels_last(clip[:, :, t % G].contiguous()) for t in range(G)]
    out_t = co._empty_cl((B, C, Ho, Wo), p.out_dtype, "cuda")
    graph = st.capture([frames[t % G] for t in range(steps)], [out_t] * steps)
    graph.upload()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(torch.cuda.current_device())
    with sampler:
        e0.record(stream)
        assert graph.launch() == steps
        e1.record(stream)
        t_end = time.time() + 60
        while not e1.query() and time.time() < t_end:
            sampler.sample()
            time.sleep(0.002)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    hbm, _, _, src = measured_peaks()
    vh = ",vh" in p.kernel_name
    ab = alg_bytes(w, Ho, Wo, vh) * B
    ach = ab / (ms / 1e3) / 1e9
    ring_mb = (p.receptive_field + 1) * B * Ho * Wo * C * (4 if w["kind"] == "avg" else 2) / 1e6
    out = {
        "metric": "stream-steps/sec per continual pooling layer", "value": round(B / (ms / 1e3), 1),
        "unit": "stream-steps/s", "n_gpus": 1, "steps": steps, "warmup": warmup, "ms_per_step": round(ms, 5),
        "higher_is_better": True, "dtype": "bf16", "data": "synthetic (seeded N(0,1) bf16 frames)",
        "config": {"workload": name, "desc": w["desc"], "streams": B, "kernel": list(w["kernel"]),
                   "stride": list(w["stride"]), "padding": list(w["padding"]), "in": [H, W, C], "out": [Ho, Wo, C],
                   "ring_MB": round(ring_mb, 1),
                   "l2_policy": f"input pool of {G} distinct frames ({round(G * fbytes / 1e6)} MB > L2 "
                                f"{l2 // 2**20} MiB); the reduced-frame ring ({round(ring_mb, 1)} MB) may stay L2-resident"},
        "gpu_launches": steps,
        "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(ach / hbm, 4), "kernel": p.kernel_name, "alg_bytes_per_launch": int(ab),
                     "peak_source": src, "traffic": None},
        "clocks": sampler.summary(),
    }
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="all", choices=["all"] + list(WORKLOADS))
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="documented planner option (co.set_option), e.g. pool_g=4")
    a = ap.parse_args()
    if a.option:
        import paper_2204_03418_b200 as co
        for kv in a.option:
            k, v = kv.split("=", 1)
            co.set_option(k, int(v))
    for name in (WORKLOADS if a.workload == "all" else [a.workload]):
        run(name, a.steps, a.warmup)


if __name__ == "__main__":
    main()
