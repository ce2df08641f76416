#!/usr/bin/env python
"""A/B runs of bench.py under environment-variable variants (experiment tool).

usage: python scripts/ab_bench.py --config 5 --steps 30 "CO_TC_EG=3" "CO_TC_EG=2" ""
Each argument is a space-separated list of VAR=value settings ("" = defaults);
prints value, dominant kernel, its ms per launch and roofline fraction."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--timeout", type=float, default=240, help="seconds per variant run")
    ap.add_argument("variants", nargs="*")
    a = ap.parse_args()
    for var in a.variants or [""]:
        env = dict(os.environ)
        for kv in var.split():
            k, v = kv.split("=", 1)
            env[k] = v
        try:
            out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(a.config),
                                  "--steps", str(a.steps), "--warmup", str(a.warmup), "--no-e2e", "--no-cpu-baseline"],
                                 env=env, capture_output=True, text=True, timeout=a.timeout)
        except subprocess.TimeoutExpired:
            print(f"[{var or 'default'}] timed out after {a.timeout:.0f} s", flush=True)
            continue
        lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if not lines:
            print(f"[{var or 'default'}] failed: {out.stderr[-300:]}")
            continue
        j = json.loads(lines[-1])
        r = j["roofline"]
        print(f"[{var or 'default'}] value={j['value']:.0f} kernel={r.get('kernel')} ms={r.get('ms_per_launch')} "
              f"frac={r.get('frac')}", flush=True)
        for l in j.get("layers") or []:
            print(f"    {l['kernel']} {l['ms_per_launch']} {l['frac']}")


if __name__ == "__main__":
    main()
