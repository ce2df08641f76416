"""Seeded synthetic inputs for the five BASELINE.json configs (shared by the
tests, bench.py and the oracle legs).

This module holds NO arithmetic of the method: it only draws weights, biases,
folded-BN parameters and input frames from seeded generators and rounds them
to the config dtype, so that the CUDA path and the oracle see identical bits.
There is no public dataset in this setting (BASELINE.json names none; the
paper's Kinetics-400 / NTU RGB+D workloads are absent): the configs are shape
stand-ins for the paper's families (C3 X3D-like, C4 Slow-like, C5 ST-GCN-like),
with iid Gaussian values as BASELINE.json prescribes.

Recipe:
- config seed s_c = 2204034180 + c (c = 1..5);
- weights ~ N(0, 1/fan_in) (variance 1/fan_in, fan_in = Cin/g * kt*kh*kw),
  bias ~ N(0, 0.01) (std 0.1), drawn in fp64 from numpy PCG64(s_c) in
  parameter order (layer, W, b, BN), rounded to the config dtype (RNE);
- C4 BN (synthetic, inference mode): gamma ~ U(0.5, 1.5), beta ~ N(0, 0.01),
  mean ~ N(0, 0.01), var ~ U(0.5, 1.5), eps = 1e-5, folded into W and b in
  fp64 before rounding (a harness preprocessing step, A14);
- input frames ~ N(0, 1): frame (t) of all GLOBAL streams is drawn with a
  torch generator seeded (s_c * 1_000_003 + t) and the shard is sliced from it,
  so per-stream data do not depend on the number of GPUs.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

SEED0 = 2204034180


@dataclass
class Layer:
    cin: int
    cout: int
    kernel: Tuple[int, int, int]
    stride: Tuple[int, int, int] = (1, 1, 1)
    padding: Tuple[int, int, int] = (0, 0, 0)
    dilation: Tuple[int, int, int] = (1, 1, 1)
    groups: int = 1
    relu: bool = False
    bn: bool = False

    @property
    def fan_in(self) -> int:
        return (self.cin // self.groups) * self.kernel[0] * self.kernel[1] * self.kernel[2]


@dataclass
class Config:
    cid: int
    name: str
    workload: str
    n_streams: int
    steps: int
    spatial_rank: int
    in_spatial: Tuple[int, int]
    layers: List[Layer]
    dtype: torch.dtype = torch.bfloat16
    scaling_note: str = ""

    @property
    def seed(self) -> int:
        return SEED0 + self.cid


def _cfgs() -> dict:
    return {
        1: Config(1, "c1_fp32_tiny", "C1: continual Conv3d fp32, 1 stream, 4->8, k3x3x3, pad (0,1,1), 8x8, 16 steps",
                  1, 16, 2, (8, 8), [Layer(4, 8, (3, 3, 3), padding=(0, 1, 1))], dtype=torch.float32),
        2: Config(2, "c2_dense", "C2: dense continual Conv3d bf16/fp32-state, 256 streams, 64->64, k3x3x3, pad (0,1,1), 56x56, 128 steps",
                  256, 128, 2, (56, 56), [Layer(64, 64, (3, 3, 3), padding=(0, 1, 1))]),
        3: Config(3, "c3_depthwise", "C3: X3D-style depthwise chain, 512 streams, C=192 g=192, k3x3x3 then k5x1x1, 28x28, 256 steps",
                  512, 256, 2, (28, 28), [Layer(192, 192, (3, 3, 3), padding=(0, 1, 1), groups=192),
                                          Layer(192, 192, (5, 1, 1), groups=192)]),
        4: Config(4, "c4_slow_stack", "C4: Slow-style 5-layer stack, 1024 streams, 3x112x112, 3->64->128->256->256->512, BN folded, ReLU x4, 64 steps",
                  1024, 64, 2, (112, 112), [
                      Layer(3, 64, (5, 7, 7), stride=(1, 2, 2), padding=(0, 3, 3), relu=True, bn=True),
                      Layer(64, 128, (1, 3, 3), padding=(0, 1, 1), relu=True, bn=True),
                      Layer(128, 256, (3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), relu=True, bn=True),
                      Layer(256, 256, (3, 3, 3), padding=(0, 1, 1), relu=True, bn=True),
                      Layer(256, 512, (3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), bn=True)]),
        5: Config(5, "c5_conv1d_long", "C5: continual Conv1d over 25 joints, 16384 streams, 256->256, kt 9, dilation 2, 512 steps",
                  16384, 512, 1, (25, 1), [Layer(256, 256, (9, 1, 1), dilation=(2, 1, 1))]),
    }


CONFIGS = _cfgs()


def config(cid: int, **overrides) -> Config:
    """A config, optionally resized (e.g. n_streams / in_spatial / steps) for parity runs."""
    import copy
    c = copy.deepcopy(CONFIGS[cid])
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


def to_dtype_rne(a: np.ndarray, dtype: torch.dtype) -> torch.Tensor:
    """fp64 -> dtype with round-to-nearest-even (via fp32: exact for the
    values drawn here except for the final RNE to bf16)."""
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    if dtype == torch.float32:
        return t.to(torch.float32)
    # fp64 -> bf16 directly (torch rounds RNE from double)
    return t.to(torch.bfloat16)


def params(cfg: Config) -> List[Tuple[torch.Tensor, torch.Tensor]]:
    """[(W (Cout,Cin/g,kt,kh,kw) in cfg.dtype, bias (Cout) fp32)] per layer, on CPU."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    out = []
    for L in cfg.layers:
        shape = (L.cout, L.cin // L.groups) + tuple(L.kernel)
        W = rng.standard_normal(shape) * np.sqrt(1.0 / L.fan_in)
        b = rng.standard_normal(L.cout) * 0.1
        if L.bn:
            gamma = rng.uniform(0.5, 1.5, L.cout)
            beta = rng.standard_normal(L.cout) * 0.1
            mean = rng.standard_normal(L.cout) * 0.1
            var = rng.uniform(0.5, 1.5, L.cout)
            scale = gamma / np.sqrt(var + 1e-5)
            W = W * scale.reshape(-1, 1, 1, 1, 1)
            b = (b - mean) * scale + beta
        Wt = to_dtype_rne(W, cfg.dtype)
        bt = torch.from_numpy(b).to(torch.float32)
        out.append((Wt, bt))
    return out


def in_shape(cfg: Config) -> Tuple[int, ...]:
    """Logical per-stream frame shape (Cin, *S)."""
    S = cfg.in_spatial[: cfg.spatial_rank]
    return (cfg.layers[0].cin,) + tuple(S)


def frame(cfg: Config, t: int, b0: int = 0, b1: Optional[int] = None, device="cuda",
          n_global: Optional[int] = None) -> torch.Tensor:
    """Input frame t for global streams [b0, b1): logical (b1-b0, Cin, *S),
    channels-last memory, cfg.dtype, N(0,1) RNE-rounded."""
    n_global = n_global or cfg.n_streams
    b1 = n_global if b1 is None else b1
    g = torch.Generator(device=device)
    g.manual_seed(cfg.seed * 1_000_003 + t)
    shp = in_shape(cfg)
    phys = (n_global,) + shp[1:] + (shp[0],)
    x = torch.randn(phys, generator=g, device=device, dtype=torch.float32)
    x = x[b0:b1].to(cfg.dtype).contiguous()
    return x.movedim(-1, 1)


def integer_frame(cfg: Config, t: int, device="cuda", lo=-2, hi=2) -> torch.Tensor:
    """Exact-arithmetic regime (SC4): integers in [lo, hi], exactly representable."""
    g = torch.Generator(device=device)
    g.manual_seed(cfg.seed * 7 + t)
    shp = in_shape(cfg)
    phys = (cfg.n_streams,) + shp[1:] + (shp[0],)
    x = torch.randint(lo, hi + 1, phys, generator=g, device=device).to(cfg.dtype)
    return x.movedim(-1, 1)


def integer_params(cfg: Config, lo=-2, hi=2):
    rng = np.random.Generator(np.random.PCG64(cfg.seed + 99))
    out = []
    for L in cfg.layers:
        shape = (L.cout, L.cin // L.groups) + tuple(L.kernel)
        W = rng.integers(lo, hi + 1, shape).astype(np.float64)
        b = rng.integers(lo, hi + 1, L.cout).astype(np.float64)
        out.append((to_dtype_rne(W, cfg.dtype), torch.from_numpy(b).to(torch.float32)))
    return out
