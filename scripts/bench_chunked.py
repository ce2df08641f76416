#!/usr/bin/env python
"""Chunked vs per-step co_forward_steps (SURVEY §8f f2 -- "report them
separately from online per-step numbers").  Workload: BASELINE.json configs[2]'s
temporal layer (C3-b: depthwise kt=5, C=192, 28x28, 512 streams, bf16 in/out,
fp32 state), driven through co_forward_steps over device clips of T frames
(seeded N(0,1)); the per-step leg forces the per-frame fold (CO_CHUNK=0 in a
subprocess), the chunked leg runs k_steps_dw_t (state in registers across the
clip).  Timing: CUDA events around K clips after W warm-up clips; clips rotate
over two buffers of T frames each (each > L2).

Algorithmic bytes per stream-step: per-step fold x + y + 2 (kt-1) fp32 state
per output element; chunked x + y + 2 (kt-1) fp32 state / T.

usage: python scripts/bench_chunked.py [--T 32] [--clips 8] [--warmup 2]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def leg(T, clips, warmup):
    import torch
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    from bench import ClockSampler, measured_peaks
    cfg = synth.config(3)
    L = cfg.layers[1]
    B = cfg.n_streams
    H, W = cfg.in_spatial
    Wt, bt = synth.params(cfg)[1]
    conv = co.Conv(L.cin, L.cout, L.kernel, weight=Wt.cuda(), bias=bt.cuda(), stride=L.stride, padding=L.padding,
                   dilation=L.dilation, groups=L.groups, in_spatial=(H, W), n_streams=B, dtype=cfg.dtype,
                   out_dtype=cfg.dtype, kernel="depthwise")
    g = torch.Generator(device="cuda").manual_seed(5)
    clips_buf = [co.channels_last(torch.randn((B, L.cin, T, H, W), generator=g, device="cuda").to(torch.bfloat16))
                 for _ in range(2)]
    for i in range(warmup):
        conv.forward_steps(clips_buf[i % 2])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(torch.cuda.current_device())
    with sampler:
        e0.record()
        for i in range(clips):
            ys, _ = conv.forward_steps(clips_buf[i % 2])
        e1.record()
        e1.synchronize()
    steps = clips * T
    ms = e0.elapsed_time(e1) / steps
    hbm, _, src = measured_peaks()
    chunked = os.environ.get("CO_CHUNK", "1") != "0"
    el = H * W * L.cout
    state = 2 * (L.kernel[0] - 1) * 4 * el
    alg = 2 * el * 2 + (state / T if chunked else state)
    ach = alg * B / (ms / 1e3) / 1e9
    return {"metric": "stream-steps/sec, C3-b layer through co_forward_steps", "mode": "chunked" if chunked else "per-step",
            "value": round(B / (ms / 1e3), 1), "unit": "stream-steps/s", "ms_per_step": round(ms, 5),
            "T": T, "clips": clips, "kernel": conv.kernel_name if not chunked else "k_steps_dw_t<5>",
            "config": {"workload": "BASELINE.json configs[2] layer 2 (depthwise kt=5, C=192, 28x28)", "streams": B},
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(ach / hbm, 4), "alg_bytes_per_stream_step": int(alg), "peak_source": src},
            "clocks": sampler.summary()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=32)
    ap.add_argument("--clips", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--leg", action="store_true", help=argparse.SUPPRESS)
    a = ap.parse_args()
    if a.leg:
        print(json.dumps(leg(a.T, a.clips, a.warmup)), flush=True)
        return
    for chunk in ("0", "1"):
        env = dict(os.environ, CO_CHUNK=chunk)
        out = subprocess.run([sys.executable, __file__, "--leg", "--T", str(a.T), "--clips", str(a.clips),
                              "--warmup", str(a.warmup)], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        print(line[-1] if line else json.dumps({"mode": chunk, "error": out.stderr[-400:]}), flush=True)


if __name__ == "__main__":
    main()
