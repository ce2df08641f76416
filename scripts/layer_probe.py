#!/usr/bin/env python
"""One layer of a BASELINE.json config, alone, at the config's stream count
(experiment / profiling tool): fills the layer's delay, then runs --steps Ready
steps and prints the mean CUDA-event time per step.  Under ncu, the Ready-step
launches are the last --steps launches of the layer's kernel.

usage: python scripts/layer_probe.py --config 4 --layer 2 [--steps 3] [--state psum]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--layer", type=int, default=0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--streams", type=int, default=None)
    ap.add_argument("--state", default="psum")
    ap.add_argument("--option", action="append", default=[])
    a = ap.parse_args()
    import torch
    import bench
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    torch.cuda.set_device(0)
    for kv in a.option:
        k, v = kv.split("=", 1)
        co.set_option(k, int(v))
    cfg = synth.config(a.config)
    B = a.streams or cfg.n_streams
    convs = bench.build_layers(cfg, B, state=a.state)
    c = convs[a.layer]
    for i, cv in enumerate(convs):
        if i != a.layer:
            del cv
    g = torch.Generator(device="cuda").manual_seed(0)
    shape = (B, c.in_channels) + c.in_spatial
    xs = [co.channels_last(torch.randn(shape, generator=g, device="cuda").to(cfg.dtype)) for _ in range(2)]
    out = co._empty_cl((B, c.out_channels) + c.out_spatial, c.out_dtype, "cuda")
    for t in range(c.delay):
        c.forward_step(xs[t % 2], out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(a.steps):
        assert c.forward_step(xs[t % 2], out=out) is not None
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"config": a.config, "layer": a.layer, "kernel": c.kernel_name, "streams": B,
                      "ms": round(e0.elapsed_time(e1) / a.steps, 4)}), flush=True)


if __name__ == "__main__":
    main()
