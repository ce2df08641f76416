"""fp64 oracle for continual pooling (PAPER.md P:380-394
"co.AvgPool1d, co.MaxPool1d, etc.").

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): only tests/, smoke() and
bench.py's CPU legs may import it; it shares no code with the CUDA path.

Plain numpy, written for checkability rather than speed:
* ``pool_forward`` -- batch mode: the windowed max or mean of a clip
  (B, C, T, S1, S2) with symmetric temporal padding p and spatial padding.
  AVG counts padding as zeros and always divides by the full window
  kt*kh*kw (count_include_pad; SPEC's recorded decision).  MAX
  ignores padding, i.e. pads are -inf (PyTorch's implicit MAX padding, the
  drop-in-replacement principle P:71-80); a window of padding only is -inf.
  DESIGN.md readings A21-A22.
* ``PoolStep`` -- step mode: Definition 1 for pooling, i.e. the
  output at a Ready tick is the batch output of the window ending at this
  frame; the window's frames come from a history of the last f-1 padded frames
  (start padding and pad_end steps are padding: zero for AVG, skipped by MAX).
  Ready ticks: n >= d and (n-d) mod s == 0 with d = f - p - 1.
"""
from __future__ import annotations

from typing import Optional, Sequence, Tuple

import numpy as np


def _three(v, fill):
    v = list(v) + [fill] * (3 - len(v))
    return tuple(int(a) for a in v[:3])


def _spatial_window(frame: np.ndarray, h0: int, w0: int, kh: int, kw: int, dh: int, dw: int,
                    H: int, W: int):
    """Values of one (C,) column over the spatial window starting at (h0, w0) of a
    (C, H, W) frame, and a mask of which taps are inside the frame."""
    vals, inside = [], []
    for u in range(kh):
        for v in range(kw):
            h, w = h0 + u * dh, w0 + v * dw
            ok = 0 <= h < H and 0 <= w < W
            inside.append(ok)
            vals.append(frame[:, h, w] if ok else np.zeros(frame.shape[0]))
    return vals, inside


def _pool_window(kind: str, frames, pads, ho: int, wo: int, kernel, stride, padding, dilation, H, W):
    """One output column (C,) from the kt temporal frames of its window;
    pads[k] marks a temporal padding frame."""
    kt, kh, kw = kernel
    acc = None
    count = kt * kh * kw
    for k in range(kt):
        h0 = ho * stride[1] - padding[1]
        w0 = wo * stride[2] - padding[2]
        vals, inside = _spatial_window(frames[k], h0, w0, kh, kw, dilation[1], dilation[2], H, W)
        for val, ok in zip(vals, inside):
            if kind == "max":
                if pads[k] or not ok:
                    continue                    # MAX ignores padding
                acc = val.copy() if acc is None else np.maximum(acc, val)
            else:
                contrib = np.zeros_like(val) if (pads[k] or not ok) else val
                acc = contrib.copy() if acc is None else acc + contrib
    if kind == "max":
        if acc is None:                          # an all-padding window: max over an empty set,
            return np.full(frames[0].shape[0], -np.inf)   # -inf like PyTorch's implicit MAX padding
        return acc
    return acc / count


def out_len(T: int, kt: int, p: int, s: int, dil: int = 1) -> int:
    f = dil * (kt - 1) + 1
    return (T + 2 * p - f) // s + 1


def pool_forward(kind: str, x: np.ndarray, kernel: Sequence[int], stride=(1, 1, 1), padding=(0, 0, 0),
                 dilation=(1, 1, 1)) -> np.ndarray:
    """Batch mode: x (B, C, T, H, W) -> (B, C, T', H', W')."""
    assert kind in ("max", "avg")
    kernel, stride, dilation = _three(kernel, 1), _three(stride, 1), _three(dilation, 1)
    padding = _three(padding, 0)
    B, C, T, H, W = x.shape
    kt, kh, kw = kernel
    f = dilation[0] * (kt - 1) + 1
    Tp = out_len(T, kt, padding[0], stride[0], dilation[0])
    Ho = (H + 2 * padding[1] - dilation[1] * (kh - 1) - 1) // stride[1] + 1
    Wo = (W + 2 * padding[2] - dilation[2] * (kw - 1) - 1) // stride[2] + 1
    if Tp < 1:
        raise ValueError("insufficient length: T' < 1")
    y = np.empty((B, C, Tp, Ho, Wo))
    for b in range(B):
        for i in range(Tp):
            frames, pads = [], []
            for k in range(kt):
                t = i * stride[0] + k * dilation[0] - padding[0]
                pads.append(not (0 <= t < T))
                frames.append(x[b, :, t] if 0 <= t < T else np.zeros((C, H, W)))
            for ho in range(Ho):
                for wo in range(Wo):
                    y[b, :, i, ho, wo] = _pool_window(kind, frames, pads, ho, wo, kernel, stride, padding,
                                                      dilation, H, W)
    return y


class PoolStep:
    """Step mode over B streams sharing one clock."""

    def __init__(self, kind: str, C: int, in_spatial: Tuple[int, int], kernel, stride=(1, 1, 1),
                 padding=(0, 0, 0), dilation=(1, 1, 1), B: int = 1):
        assert kind in ("max", "avg")
        self.kind, self.C, self.B = kind, C, B
        self.kernel, self.stride = _three(kernel, 1), _three(stride, 1)
        self.padding, self.dilation = _three(padding, 0), _three(dilation, 1)
        self.H, self.W = in_spatial
        kt = self.kernel[0]
        self.f = self.dilation[0] * (kt - 1) + 1
        p = self.padding[0]
        if not 0 <= p <= self.f - 1:
            raise ValueError("temporal padding must be in [0, f-1]")
        self.delay = self.f - p - 1
        self.clean_state()

    def clean_state(self):
        self.n = 0
        zero = np.zeros((self.B, self.C, self.H, self.W))
        # history of the last f-1 padded frames (oldest first) and their padding
        # flags: before the first frame it holds only start padding (the p pads
        # plus frames no Ready output ever reads), zero and flagged
        self.hist = [zero.copy() for _ in range(self.f - 1)]
        self.hpad = [True] * (self.f - 1)

    def history(self):
        """Read-only view of the last f-1 padded frames (oldest first),
        (f-1, B, C, H, W), and their padding flags."""
        if self.f == 1:
            return np.zeros((0, self.B, self.C, self.H, self.W)), []
        return np.stack(self.hist), list(self.hpad)

    def reduced_history(self):
        """The history as the GPU handle stores it (include/co.h co_op): each
        frame's spatial-window reduction (C, H', W') -- the window max, or the
        window SUM for AVG -- with padding frames the identity (-inf / 0);
        (f-1, B, C, H', W')."""
        Ho, Wo = self.out_spatial
        kt, kh, kw = self.kernel
        out = np.empty((self.f - 1, self.B, self.C, Ho, Wo))
        for j, (fr, pad) in enumerate(zip(self.hist, self.hpad)):
            for b in range(self.B):
                for ho in range(Ho):
                    for wo in range(Wo):
                        col = _pool_window(self.kind, [fr[b]], [pad], ho, wo, (1, kh, kw), self.stride,
                                           self.padding, self.dilation, self.H, self.W)
                        out[j, b, :, ho, wo] = col if self.kind == "max" else col * (kh * kw)
        return out

    @property
    def out_spatial(self):
        kt, kh, kw = self.kernel
        Ho = (self.H + 2 * self.padding[1] - self.dilation[1] * (kh - 1) - 1) // self.stride[1] + 1
        Wo = (self.W + 2 * self.padding[2] - self.dilation[2] * (kw - 1) - 1) // self.stride[2] + 1
        return Ho, Wo

    def forward_step(self, x: Optional[np.ndarray], update_state: bool = True):
        """x (B, C, H, W) or None (a padding step, pad_end); returns the Ready
        output (B, C, H', W') or None (Empty)."""
        ready = self.n >= self.delay and (self.n - self.delay) % self.stride[0] == 0
        cur = np.zeros((self.B, self.C, self.H, self.W)) if x is None else np.asarray(x, np.float64)
        cur_pad = x is None
        y = None
        if ready:
            window = self.hist + [cur]               # padded frames m-(f-1) .. m
            wpad = self.hpad + [cur_pad]
            kt, dil = self.kernel[0], self.dilation[0]
            taps = [k * dil for k in range(kt)]      # positions inside the f-frame window
            Ho, Wo = self.out_spatial
            y = np.empty((self.B, self.C, Ho, Wo))
            for b in range(self.B):
                frames = [window[t][b] for t in taps]
                pads = [wpad[t] for t in taps]
                for ho in range(Ho):
                    for wo in range(Wo):
                        y[b, :, ho, wo] = _pool_window(self.kind, frames, pads, ho, wo, self.kernel, self.stride,
                                                       self.padding, self.dilation, self.H, self.W)
        if update_state:
            if self.f > 1:
                self.hist = self.hist[1:] + [cur]
                self.hpad = self.hpad[1:] + [cur_pad]
            self.n += 1
        return y
