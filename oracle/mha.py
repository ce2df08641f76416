"""fp64 oracle for continual single-output multi-head attention (SURVEY §8f
f4; PAPER.md P:430-432 co.MultiheadAttention "single-output" mode; SPEC.md:
357-403).

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): only tests/, smoke() and
bench.py's CPU legs may import it; it shares no code with the CUDA path.

Plain numpy, written for checkability:
* ``mha_forward`` -- batch mode over a window of n steps, x (B, E, T = n):
  q/k/v = W_{q,k,v} x + b per step, per head h scaled dot-product attention
  scores q_i . k_j / sqrt(E/heads), softmax over keys j (max subtracted), the
  weighted sum of values, heads concatenated, y = W_o a + b_o.
* ``MhaStep`` -- step mode: project the step, push (k, v) into a ring of n
  entries, Empty until n entries are present (d = n - 1, s = 1), then the
  attention of the newest query against the n buffered keys / values, output-
  projected -- the last column of ``mha_forward`` over the trailing n steps
  (S:377-381).  No early partial-window outputs.
"""
from __future__ import annotations

from typing import Optional

import numpy as np


def _proj(W, b, x):
    y = W @ x
    return y if b is None else y + b


def _attend(q, K, V, heads: int):
    """q (E,), K and V (n, E): per head softmax(q_h K_h^T / sqrt(dh)) V_h, heads concatenated."""
    E = q.shape[0]
    dh = E // heads
    out = np.empty(E)
    for h in range(heads):
        sl = slice(h * dh, (h + 1) * dh)
        s = K[:, sl] @ q[sl] / np.sqrt(dh)
        s = s - s.max()
        p = np.exp(s)
        p = p / p.sum()
        out[sl] = p @ V[:, sl]
    return out


def mha_forward(params: dict, x: np.ndarray) -> np.ndarray:
    """x (B, E, T) -> (B, E, T): full (non-causal) attention over the T steps."""
    x = np.asarray(x, np.float64)
    B, E, T = x.shape
    heads = params["heads"]
    y = np.empty((B, E, T))
    for b in range(B):
        Q = np.stack([_proj(params["Wq"], params.get("bq"), x[b, :, t]) for t in range(T)])
        K = np.stack([_proj(params["Wk"], params.get("bk"), x[b, :, t]) for t in range(T)])
        V = np.stack([_proj(params["Wv"], params.get("bv"), x[b, :, t]) for t in range(T)])
        for t in range(T):
            y[b, :, t] = _proj(params["Wo"], params.get("bo"), _attend(Q[t], K, V, heads))
    return y


class MhaStep:
    """Single-output continual MHA over B lockstep streams."""

    def __init__(self, params: dict, window: int, B: int):
        if params["Wq"].shape[0] % params["heads"]:
            raise ValueError("E must be divisible by heads")
        if window < 1:
            raise ValueError("window must be >= 1")
        self.p, self.n_win, self.B = params, window, B
        self.delay = window - 1
        self.clean_state()

    def clean_state(self):
        self.n = 0
        self.K = []          # per stream lists of the last n keys / values, oldest first
        self.V = []

    def forward_step(self, x: np.ndarray, update_state: bool = True) -> Optional[np.ndarray]:
        """x (B, E) -> (B, E) or None (Empty)."""
        x = np.asarray(x, np.float64).reshape(self.B, -1)
        p = self.p
        q = np.stack([_proj(p["Wq"], p.get("bq"), x[b]) for b in range(self.B)])
        k = np.stack([_proj(p["Wk"], p.get("bk"), x[b]) for b in range(self.B)])
        v = np.stack([_proj(p["Wv"], p.get("bv"), x[b]) for b in range(self.B)])
        K = (self.K + [k])[-self.n_win:]
        V = (self.V + [v])[-self.n_win:]
        y = None
        if self.n >= self.delay:
            Ks, Vs = np.stack(K, axis=1), np.stack(V, axis=1)      # (B, n, E)
            y = np.stack([_proj(p["Wo"], p.get("bo"), _attend(q[b], Ks[b], Vs[b], p["heads"]))
                          for b in range(self.B)])
        if update_state:
            self.K, self.V = K[-(self.n_win - 1):] if self.n_win > 1 else [], V[-(self.n_win - 1):] if self.n_win > 1 else []
            self.n += 1
        return y
