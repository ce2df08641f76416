"""fp64 oracle for Delay and the Residual composite (PAPER.md
P:301-326 "Residual connections", P:435 co.Delay, Listing 3 and
residual_shrink; Principle 7 P:280-288).

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): only tests/, smoke() and
bench.py's CPU legs may import it; it shares no code with the CUDA path.

* ``DelayStep`` -- Delay(d): Empty for the first d ticks, then the input from
  d ticks ago; batch mode is the identity on the clip.
* ``ResidualStep`` / ``residual_forward`` -- Residual(body) with Sum:
  - equal padding (``shrink=False``; the body keeps T, i.e. 2 p_acc = f_acc-1):
    batch y = x + body(x); step mode delays the identity branch by the body's
    delay d;
  - centered (``shrink=True``, f_acc odd, p_acc <= (f_acc-1)/2): batch crops the
    identity branch by (f_acc-1)/2 - p_acc at the start (each output's
    receptive-field center); step mode delays it by (f_acc-1)/2 while the
    composite's delay is the body's (Principle 7: the merge is Empty
    while either branch is);
  - optional ReLU after the add (``relu_out``), the ResNet / X3D block form.
  The body is an ``oracle.Stack`` (sequential layers, Empty short-circuit,
  optional per-layer ReLU and bf16 activation rounding, O6); its receptive
  field and delay come from ``oracle.accumulate`` (Principle 6, A3).
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

import oracle as O


class DelayStep:
    """Delay(d) over B lockstep streams."""

    def __init__(self, d: int):
        if d < 0:
            raise ValueError("delay must be >= 0")
        self.d = d
        self.clean_state()

    def clean_state(self):
        self.n = 0
        self.hist = []                   # the last d inputs, oldest first

    def forward_step(self, x: np.ndarray, update_state: bool = True):
        """x: one step (padding steps are explicit zero frames).  Returns the
        input of d ticks ago, or None (Empty) while n < d."""
        x = np.array(x, np.float64, copy=True)
        window = self.hist + [x]                    # the last d inputs and this one
        y = window[0] if self.n >= self.d else None
        if update_state:
            self.hist = window[1:] if len(window) > self.d else window
            self.n += 1
        return y


def delay_forward(x: np.ndarray) -> np.ndarray:
    """Batch mode of Delay: the identity on the clip."""
    return np.array(x, np.float64, copy=True)


def body_timing(descs: Sequence[O.Desc]) -> dict:
    f = [d.receptive_field for d in descs]
    p = [d.padding[0] for d in descs]
    s = [d.stride[0] for d in descs]
    return O.accumulate(f, p, s) | {"f_nn": O.accumulate(f, p, s)["f_acc"][-1],
                                    "p_nn": O.accumulate(f, p, s)["p_acc"][-1]}


def skip_delay(descs: Sequence[O.Desc], shrink: bool) -> int:
    """Delay of the identity branch: the body's delay (equal padding) or
    (f_acc-1)/2 (centered, shrink) -- P:306-316."""
    t = body_timing(descs)
    if t["s_nn"] != 1:
        raise ValueError("residual body must keep the frame rate (accumulated stride 1)")
    if shrink:
        if t["f_nn"] % 2 == 0:
            raise ValueError("centered residual needs an odd receptive field (S:456)")
        if t["p_nn"] > (t["f_nn"] - 1) // 2:
            raise ValueError("centered residual: body padding exceeds (f_acc-1)/2")
        return (t["f_nn"] - 1) // 2
    if 2 * t["p_nn"] != t["f_nn"] - 1:
        raise ValueError("residual without shrink needs equal padding (2 p_acc = f_acc - 1)")
    return t["d_nn"]


class ResidualStep:
    """Residual(body) with Sum in step mode over B streams."""

    def __init__(self, descs: Sequence[O.Desc], Ws, biases, relu: Sequence[int], round_bf16: Sequence[int], B: int,
                 shrink: bool = False, relu_out: bool = False):
        self.body = O.Stack(descs, Ws, biases, relu, round_bf16, B)
        self.descs = list(descs)
        self.d_skip = skip_delay(descs, shrink)
        self.delay = body_timing(descs)["d_nn"]      # Principle 7: max of the branch delays
        self.relu_out = relu_out
        self.B = B
        self.clean_state()

    def clean_state(self):
        self.body.clean_state()
        self.n = 0
        self.hist = []                                # the last d_skip inputs, oldest first

    def forward_step(self, x: np.ndarray, update_state: bool = True):
        x = np.asarray(x, np.float64)
        yb = self.body.forward_step(x, update_state)
        skip = (self.hist + [x])[0] if self.d_skip > 0 else x
        if update_state:
            if self.d_skip > 0:
                self.hist = (self.hist + [x])[-self.d_skip:]
            self.n += 1
        if yb is None:
            return None
        y = yb + skip.reshape(yb.shape)
        return np.maximum(y, 0.0) if self.relu_out else y


def residual_forward(descs: Sequence[O.Desc], Ws, biases, relu: Sequence[int], x: np.ndarray, shrink: bool = False,
                     relu_out: bool = False, round_bf16: Optional[Sequence[int]] = None) -> np.ndarray:
    """Batch mode: the body's batch forward (O.forward layer by layer, ReLU and
    optional bf16 rounding of activations as in the step stack) plus the
    identity branch, aligned with the center of each output's receptive field
    (P:312-316): output column i covers padded frames i .. i + f_acc - 1, whose
    center is real frame i + (f_acc-1)/2 - p_acc, so the identity clip is
    cropped by c = (f_acc-1)/2 - p_acc at the start (c = 0 for equal padding,
    c = (f_acc-1)/2 for an unpadded body)."""
    x = np.asarray(x, np.float64)
    cur = x
    L = len(descs)
    for l, (d, W, b) in enumerate(zip(descs, Ws, biases)):
        cur = O.forward(d, W, b, cur)
        if relu[l]:
            cur = np.maximum(cur, 0.0)
        if round_bf16 is not None and round_bf16[l]:
            cur = O.bf16_round(cur)
    c = skip_delay(descs, shrink) - body_timing(descs)["p_nn"] if shrink else 0
    T_out = cur.shape[2]
    y = cur + x[:, :, c:c + T_out].reshape(cur.shape)
    return np.maximum(y, 0.0) if relu_out else y


class BroadcastReduceStep:
    """BroadcastReduce(branches, reduce) in step mode (PAPER.md P:462-509,
    Listing 3 "co.BroadcastReduce(conv, co.Delay(1))", Listing 4 reduce="concat";
    Principle 7 P:280-288).  A branch is an ``oracle.Stack``
    or None (identity).  Each branch with delay d_i < d_max is suffixed with
    Delay(d_max - d_i) on its Ready outputs; the merge is Ready when every
    aligned branch is (tick n >= d_max); reduce "sum" adds, "concat" stacks
    channels in branch order.  Branches must keep the frame rate (stride 1)."""

    def __init__(self, branches, delays, reduce: str = "sum"):
        assert reduce in ("sum", "concat")
        self.branches, self.reduce = list(branches), reduce
        self.delays = [int(d) for d in delays]
        self.delay = max(self.delays)
        self.clean_state()

    def clean_state(self):
        for br in self.branches:
            if br is not None:
                br.clean_state()
        self.n = 0
        self.outs = [[] for _ in self.branches]       # each branch's Ready outputs, oldest first

    def forward_step(self, x, update_state: bool = True):
        x = np.asarray(x, np.float64)
        aligned = []
        for i, br in enumerate(self.branches):
            y = x if br is None else br.forward_step(x, update_state)
            hist = self.outs[i] + ([y] if y is not None else [])
            k = self.delay - self.delays[i]              # the Delay(d_max - d_i) suffix
            aligned.append(hist[-1 - k] if len(hist) > k and self.n >= self.delay else None)
            if update_state:
                self.outs[i] = hist[-(k + 1):] if y is not None else self.outs[i]
        if update_state:
            self.n += 1
        if any(a is None for a in aligned):
            return None
        if self.reduce == "sum":
            return sum(aligned[1:], aligned[0].copy())
        return np.concatenate(aligned, axis=1)


def broadcast_reduce_forward(branch_fns, x: np.ndarray, reduce: str = "sum") -> np.ndarray:
    """Batch mode: every branch's batch output (a callable on the clip, or None =
    identity), each truncated to the shortest branch length T_min keeping the
    first T_min columns -- the columns the step mode's delay alignment pairs
    (A24) -- then summed or concatenated over channels."""
    x = np.asarray(x, np.float64)
    ys = [x.copy() if f is None else f(x) for f in branch_fns]
    T_min = min(y.shape[2] for y in ys)
    ys = [y[:, :, :T_min] for y in ys]
    return sum(ys[1:], ys[0].copy()) if reduce == "sum" else np.concatenate(ys, axis=1)
