#!/usr/bin/env python
"""Benchmark of the continual single-output MHA (include/co.h
co_mha_*).  Workload (synthetic; no BASELINE.json config covers attention): a
CoOadTR-style encoder attention, E = 1024, 16 heads of 64, window n = 64 steps,
1024 streams, bf16, N(0,1) inputs and N(0,1/E) weights.  One step = the three
launches (QKV projection on tcgen05, attention over the KV ring, output
projection).  Timing as bench.py: W >= 3 warm-up steps, K steps timed with CUDA
events, inputs rotating over a pool of distinct frames.

Roofline: the sum over the three launches of max(bytes / HBM, FLOPs / bf16
peak): projections are GEMMs (8 B E^2 FLOPs per step), the attention reads the
2 n E bf16 KV ring per stream (HBM-bound).

usage: python scripts/bench_mha.py [--steps K] [--warmup W] [--streams B] [--window n] [--option name=value]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--streams", type=int, default=1024)
    ap.add_argument("--embed", type=int, default=1024)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--window", type=int, default=64)
    ap.add_argument("--option", action="append", default=[], help="name=value library option (co_set_option)")
    a = ap.parse_args()
    import torch
    import paper_2204_03418_b200 as co
    from bench import ClockSampler, measured_peaks
    B, E, H, n = a.streams, a.embed, a.heads, a.window
    for kv in a.option:
        k, v = kv.split("=")
        co.set_option(k, int(v))
    g = torch.Generator(device="cuda").manual_seed(7)
    w_in = torch.randn((3 * E, E), generator=g, device="cuda") / E ** 0.5
    w_out = torch.randn((E, E), generator=g, device="cuda") / E ** 0.5
    m = co.MultiheadAttention(E, H, n, n_streams=B, in_proj_weight=w_in, out_proj_weight=w_out,
                              in_proj_bias=torch.zeros(3 * E, device="cuda"), out_proj_bias=torch.zeros(E, device="cuda"))
    pool = [torch.randn((B, E), generator=g, device="cuda").to(torch.bfloat16) for _ in range(16)]
    y = torch.empty((B, E), dtype=torch.bfloat16, device="cuda")
    for t in range(max(a.warmup, 3) + n - 1):
        m.forward_step(pool[t % 16], out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(torch.cuda.current_device())
    with sampler:
        e0.record()
        h0 = time.perf_counter()
        for t in range(a.steps):
            assert m.forward_step(pool[t % 16], out=y) is not None
        host_us = (time.perf_counter() - h0) / a.steps * 1e6      # host time per call (launch-bound check)
        e1.record()
        t_end = time.time() + 60
        while not e1.query() and time.time() < t_end:
            sampler.sample()
            time.sleep(0.002)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    hbm, bf16, _, src = measured_peaks()
    att_bytes = B * (2 * n * E * 2 + 3 * E * 2 + E * 2)
    proj_flops = 8.0 * B * E * E
    proj_bytes = B * E * 2 * (1 + 3 + 1 + 1) + 4 * E * E * 2
    t_roof = att_bytes / (hbm * 1e9) + max(proj_flops / (bf16 * 1e12), proj_bytes / (hbm * 1e9))
    out = {"metric": "stream-steps/sec, continual single-output MHA", "value": round(B / (ms / 1e3), 1),
           "unit": "stream-steps/s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 5),
           "higher_is_better": True, "dtype": "bf16", "data": "synthetic (seeded N(0,1) steps, N(0,1/E) weights)",
           "config": {"workload": f"CoOadTR-style attention E={E} heads={H} window={n}", "streams": B,
                      "kv_ring_MB": round(2 * n * B * E * 2 / 1e6, 1)},
           "gpu_launches": 3 * a.steps, "host_us_per_step": round(host_us, 1), "options": a.option,
           "roofline": {"bound": "hbm+tensor", "t_roof_us": round(t_roof * 1e6, 2),
                        "frac": round(t_roof / (ms / 1e3), 4), "attention_bytes_per_step": att_bytes,
                        "projection_flops_per_step": proj_flops, "peak_hbm_gbs": hbm, "peak_bf16_tflops": bf16,
                        "peak_source": src},
           "clocks": sampler.summary()}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
