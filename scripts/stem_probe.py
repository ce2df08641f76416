#!/usr/bin/env python
"""C4 stem probe (experiment tool): the stem layer's time alone versus inside
the 5-layer stack, with NVML clock samples per phase.

usage: python scripts/stem_probe.py [--streams 1024] [--steps 20]
Prints one JSON line per phase: per-layer ms (CUDA events on the launching
stream), median SM clock and throttle reasons during the phase."""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--layers", default="0;0,1,2,3,4;0")
    ap.add_argument("--sync", action="store_true", help="synchronize after every step (serialised steps)")
    a = ap.parse_args()
    import torch
    import bench
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    torch.cuda.set_device(0)
    cfg = synth.config(4)
    B = a.streams
    convs = bench.build_layers(cfg, B)
    pool = [synth.frame(cfg, t, 0, B, n_global=B) for t in range(4)]
    acts = [co._empty_cl((B, c.out_channels) + c.out_spatial, c.out_dtype, "cuda") for c in convs]
    stream = torch.cuda.current_stream()
    # fill every layer's delay once (the stack's d_NN)
    for n in range(12):
        cur = pool[n % 4]
        for l, c in enumerate(convs):
            y = c.forward_step(cur, out=acts[l])
            if y is None:
                break
            cur = y
    torch.cuda.synchronize()
    for spec in a.layers.split(";"):
        if spec == "sleep":
            time.sleep(5)
            continue
        ls = [int(v) for v in spec.split(",")]
        K = a.steps
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(ls) + 1)] for _ in range(K)]
        smp = bench.ClockSampler(0)
        with smp:
            for k in range(K):
                ev[k][0].record(stream)
                for i, l in enumerate(ls):
                    x = pool[k % 4] if l == 0 else acts[l - 1]
                    convs[l].forward_step(x, out=acts[l])
                    ev[k][i + 1].record(stream)
                if a.sync:
                    torch.cuda.synchronize()
            while not ev[K - 1][-1].query():
                smp.sample()
            torch.cuda.synchronize()
        ms = [statistics.median(ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(2, K)) for i in range(len(ls))]
        print(json.dumps({"sync": a.sync, "pdl": os.environ.get("CO_PDL", "1"), "layers": ls, "ms": [round(m, 4) for m in ms], "kernels": [convs[l].kernel_name for l in ls],
                          "clocks": smp.summary()}), flush=True)


if __name__ == "__main__":
    main()
