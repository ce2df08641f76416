#!/usr/bin/env python
"""Mutation check of the fp64 oracle (test infrastructure).

Each mutant is a plausible mistake in ``oracle/co_oracle.c`` (a dropped term, a
wrong sign or index, a transposed operand, an off-by-one in the delay or the
stride phase, the printed-but-contradicted Principle-6 recurrence).  For each,
the script compiles a mutated copy of the oracle into a temporary library and
runs the oracle pins (``-m "not gpu"``) against it through ``CO_ORACLE_LIB``;
a mutant that passes every pin would mean the pins cannot tell it from the
paper's definition.  Exit status 0 iff every mutant is killed.

usage: python scripts/oracle_mutants.py [--list] [names...]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "co_oracle.c")
PINS = [os.path.join(ROOT, "tests", "test_oracle_pins.py")]

# (name, what it breaks, exact source text, replacement)
MUTANTS = [
    ("delay_off_by_one", "Principle 4 (P:138-145): d = f - p instead of f - p - 1",
     "return or_receptive_field(d) - d->padding[0] - 1;", "return or_receptive_field(d) - d->padding[0];"),
    ("reversed_slices", "temporal slice k read as kt-1-k (rotation direction)",
     "const double w = W[((((long)o * cig + c) * kt + k) * kh + u) * kw + v];",
     "const double w = W[((((long)o * cig + c) * kt + (kt - 1 - k)) * kh + u) * kw + v];"),
    ("flipped_spatial_w", "spatial column tap v read as kw-1-v (a flipped kernel: convolution, not S:241's cross-correlation)",
     "const int wi = wo * d.stride[2] + v * d.dilation[2] - d.padding[2];",
     "const int wi = wo * d.stride[2] + (kw - 1 - v) * d.dilation[2] - d.padding[2];"),
    ("dropped_history_push", "the step pushes a zero frame instead of x (history never fills)",
     "if (x) memcpy(last, x, sizeof(double) * sm->frame_elems);", "if (0) memcpy(last, x, sizeof(double) * sm->frame_elems);"),
    ("printed_principle6", "P:251 / P:260 as printed: f_acc(i) = f(i) + (f_acc(i-1) - 1) s(i), p_acc(i) = p(i) s_acc(i-1)",
     "      p_acc[i] = p_acc[i - 1] + p[i] * s_acc[i - 1];\n      f_acc[i] = f_acc[i - 1] + (f[i] - 1) * s_acc[i - 1];",
     "      p_acc[i] = p[i] * s_acc[i - 1];\n      f_acc[i] = f[i] + (f_acc[i - 1] - 1) * s[i];"),
    ("head_floor", "head = floor((n-d)/s) mod R instead of ceil (the next output to complete)",
     "return (int)floor_mod(ceil_div(sm->n - sm->delay, sm->s), sm->R);",
     "return (int)floor_mod(floor_div(sm->n - sm->delay, sm->s), sm->R);"),
    ("stride_phase", "Ready phase under stride (A4): (n - d) mod s == 1 instead of 0",
     "const int ready = (sm->n >= sm->delay) && (floor_mod(sm->n - sm->delay, sm->s) == 0);",
     "const int ready = (sm->n >= sm->delay) && (floor_mod(sm->n - sm->delay, sm->s) == (sm->s > 1));"),
    ("dropped_bias", "the bias term of O1 is dropped",
     "double acc = bias ? bias[o] : 0.0;", "double acc = 0.0;"),
    ("transposed_channels", "group channel offset transposed: ci = c * groups + g instead of g * cig + c",
     "const int ci = g * cig + c;", "const int ci = c * d.groups + g;"),
    ("out_len_no_floor", "S:64 T' = floor((T + 2p - f)/s) + 1 computed with a truncating (not floored) division",
     "return (int)(floor_div(num, d->stride[0]) + 1);", "return (int)(num / d->stride[0] + 1);"),
    ("padding_sign", "spatial padding added instead of subtracted (row index)",
     "const int hi = ho * d.stride[1] + u * d.dilation[1] - d.padding[1];",
     "const int hi = ho * d.stride[1] + u * d.dilation[1] + d.padding[1];"),
    ("state_includes_bias", "canonical state (O5) stores the bias (A9 says it is added at emit only)",
     "or_column(d, sm->W, NULL, Z, dst, HWo);             /* bias excluded (A9) */",
     "or_column(d, sm->W, sm->bias, Z, dst, HWo);"),
    ("ring_slots_floor", "R = floor((f-1)/s) instead of ceil",
     "return (int)ceil_div(f - 1, d->stride[0]);", "return (int)floor_div(f - 1, d->stride[0]);"),
    ("dilation_ignored", "temporal dilation ignored in the step window (slice k reads history k, not k dil)",
     "        const int j = k * sm->dil;\n", "        const int j = k;\n"),
    ("bf16_truncate", "bf16 rounding truncates instead of round-to-nearest-even (A17)",
     "else r = ldexp(nearbyint(ldexp(m, 8)), e - 8);", "else r = ldexp(trunc(ldexp(m, 8)), e - 8);"),
]


def build_mutant(src_text: str, old: str, new: str, out_dir: str) -> str:
    if src_text.count(old) != 1:
        raise SystemExit(f"mutation anchor found {src_text.count(old)} times (expected once):\n{old}")
    d = os.path.join(out_dir, "oracle")
    os.makedirs(d, exist_ok=True)
    shutil.copy(os.path.join(ROOT, "oracle", "co_oracle.h"), d)
    c = os.path.join(d, "co_oracle.c")
    with open(c, "w") as f:
        f.write(src_text.replace(old, new))
    lib = os.path.join(d, "liboracle_mut.so")
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
                           "-w", "-o", lib, c, "-lm"])
    return lib


def run_pins(lib: str, timeout: float):
    env = dict(os.environ, CO_ORACLE_LIB=lib, OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider"] + PINS
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    failed = [l for l in r.stdout.splitlines() if l.startswith("FAILED")]
    return r.returncode, failed


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--list", action="store_true")
    ap.add_argument("--timeout", type=float, default=300)
    ap.add_argument("-j", "--jobs", type=int, default=max(1, min(8, (os.cpu_count() or 2) // 2)))
    ap.add_argument("names", nargs="*")
    a = ap.parse_args(argv)
    if a.list:
        for name, why, _, _ in MUTANTS:
            print(f"{name}: {why}")
        return 0
    with open(SRC) as f:
        src = f.read()
    survivors = []
    todo = [m for m in MUTANTS if not a.names or m[0] in a.names]
    with tempfile.TemporaryDirectory() as tmp:
        def one(m):
            name, why, old, new = m
            lib = build_mutant(src, old, new, os.path.join(tmp, name))
            return m, run_pins(lib, a.timeout)
        with cf.ThreadPoolExecutor(max_workers=a.jobs) as ex:
            for (name, why, _, _), (rc, failed) in ex.map(one, todo):
                killed = rc != 0
                print(f"{'killed ' if killed else 'SURVIVED'} {name:24s} {why}" +
                      (f"  <- {failed[0].split(' ')[1] if failed else 'error'}" if killed else ""), flush=True)
                if not killed:
                    survivors.append(name)
    if survivors:
        print("surviving mutants: " + ", ".join(survivors))
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
