#!/usr/bin/env python
"""Chunked vs per-step co_forward_steps (SURVEY §8f f2 -- "report them
separately from online per-step numbers").  Workloads: C3's depthwise layers
(k_steps_dw_st / k_steps_dw_t: state in registers across the clip), C2's dense layer and
C5's Conv1d (tcgen05: one launch per chunk, item-batch-major, so a tile's state
stays L2-resident across its frames), each at its BASELINE.json stream count,
driven through co_forward_steps over device clips of T frames (seeded N(0,1));
the per-step leg forces the per-frame fold (option chunk = 0 in a subprocess).  Timing: CUDA events around K clips after W warm-up clips; clips rotate
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


WORKLOADS = {   # name: (BASELINE config id, layer index, description)
    "c3a": (3, 0, "BASELINE.json configs[2] layer 1 (depthwise 3x3x3, C=192, 28x28; chunked K2 stencil)"),
    "c3b": (3, 1, "BASELINE.json configs[2] layer 2 (depthwise kt=5, C=192, 28x28)"),
    "c2": (2, 0, "BASELINE.json configs[1] (dense 3x3x3, 64->64, 56x56; tcgen05 HALO)"),
    "c5": (5, 0, "BASELINE.json configs[4] (Conv1d kt=9 dil 2, 256->256, 25 joints; tcgen05 FLAT pair)"),
}


def leg(name, T, clips, warmup):
    import torch
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    from bench import ClockSampler, measured_peaks
    cid, li, desc = WORKLOADS[name]
    cfg = synth.config(cid)
    L = cfg.layers[li]
    B = cfg.n_streams
    spat = tuple(cfg.in_spatial)
    Wt, bt = synth.params(cfg)[li]
    conv = co.Conv(L.cin, L.cout, L.kernel, weight=Wt.cuda(), bias=bt.cuda(), stride=L.stride, padding=L.padding,
                   dilation=L.dilation, groups=L.groups, spatial_rank=cfg.spatial_rank, in_spatial=spat, n_streams=B,
                   dtype=cfg.dtype, out_dtype=cfg.dtype)
    g = torch.Generator(device="cuda").manual_seed(5)
    clips_buf = [co.channels_last(torch.randn((B, L.cin, T) + conv.in_spatial, generator=g,
                                              device="cuda").to(torch.bfloat16)) for _ in range(2)]
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
    hbm, _, _, src = measured_peaks()
    import paper_2204_03418_b200 as co
    chunked = co.get_option("chunk") != 0
    import math
    el_in = math.prod(conv.in_spatial) * L.cin
    el_out = math.prod(conv.out_spatial) * L.cout
    R = conv.info().ring_slots
    state = 2 * R * 4 * el_out if L.dilation[0] > 1 else 2 * (L.kernel[0] - 1) * 4 * el_out
    alg = el_in * 2 + el_out * 2 + (state / T if chunked else state)
    ach = alg * B / (ms / 1e3) / 1e9
    return {"metric": f"stream-steps/sec, {name} layer through co_forward_steps",
            "mode": "chunked" if chunked else "per-step",
            "value": round(B / (ms / 1e3), 1), "unit": "stream-steps/s", "ms_per_step": round(ms, 5),
            "T": T, "clips": clips, "kernel": conv.kernel_name + (" (chunked launch)" if chunked else ""),
            "config": {"workload": desc, "streams": B},
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(ach / hbm, 4), "alg_bytes_per_stream_step": int(alg), "peak_source": src},
            "clocks": sampler.summary()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=32)
    ap.add_argument("--clips", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--workload", default="all", choices=["all"] + list(WORKLOADS))
    ap.add_argument("--leg", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--chunk", default="1", help=argparse.SUPPRESS)
    a = ap.parse_args()
    if a.leg:
        import paper_2204_03418_b200 as co
        co.set_option("chunk", int(a.chunk))      # documented option: 0 = fold per step
        print(json.dumps(leg(a.workload, a.T, a.clips, a.warmup)), flush=True)
        return
    for name in (WORKLOADS if a.workload == "all" else [a.workload]):
        for chunk in ("0", "1"):
            out = subprocess.run([sys.executable, __file__, "--leg", "--chunk", chunk, "--workload", name, "--T",
                                  str(a.T), "--clips", str(a.clips), "--warmup", str(a.warmup)],
                                 capture_output=True, text=True)
            line = [l for l in out.stdout.splitlines() if l.startswith("{")]
            print(line[-1] if line else json.dumps({"workload": name, "mode": chunk, "error": out.stderr[-400:]}),
                  flush=True)


if __name__ == "__main__":
    main()
