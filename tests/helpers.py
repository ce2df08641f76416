"""Shared test helpers: build matching CUDA-path layers and oracle step machines."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O


def rand_desc(rng, max_c=4, max_s=6, allow_stride_t=True):
    """Random small layer (SURVEY §8c SC1 bounds plus groups and dilation)."""
    rank = int(rng.integers(0, 3))
    kt = int(rng.integers(1, 6))
    dil = int(rng.integers(1, 4))
    f = dil * (kt - 1) + 1
    p = int(rng.integers(0, f))
    s = int(rng.integers(1, 4)) if allow_stride_t else 1
    cin = int(rng.integers(1, max_c + 1))
    groups = int(rng.choice([1, cin]))
    cout = groups * int(rng.integers(1, 3)) if groups > 1 else int(rng.integers(1, max_c + 1))
    kh = int(rng.integers(1, 4)) if rank >= 1 else 1
    kw = int(rng.integers(1, 4)) if rank >= 2 else 1
    H = int(rng.integers(kh, max_s + 1)) if rank >= 1 else 1
    Wd = int(rng.integers(kw, max_s + 1)) if rank >= 2 else 1
    d = O.Desc(spatial_rank=rank, cin=cin, cout=cout, kernel=(kt, kh, kw),
               stride=(s, int(rng.integers(1, 3)), int(rng.integers(1, 3))),
               padding=(p, int(rng.integers(0, 2)), int(rng.integers(0, 2))),
               dilation=(dil, 1, 1), groups=groups, in_spatial=(H, Wd))
    assert d.valid()
    return d


def set_opt(name: str, value) -> None:
    """A documented planner option (co_set_option); conftest resets them all after each test."""
    import paper_2204_03418_b200 as co
    co.set_option(name, int(value))


def reset_opt(name: str) -> None:
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import _abi
    co.set_option(name, _abi.OPTION_DEFAULTS[name])


def logical_step_shape(d: O.Desc, B: int):
    H, W = d.in_hw
    return (B, d.cin) + ((H,) if d.spatial_rank >= 1 else ()) + ((W,) if d.spatial_rank >= 2 else ())


def make_pair(d: O.Desc, W: np.ndarray, b, B: int, dtype=torch.float32, out_dtype=torch.float32,
              kernel="auto", activation=None, state_layout="psum"):
    """(CUDA-path Conv, oracle StepMachine) with identical weights."""
    import paper_2204_03418_b200 as co
    Wt = torch.from_numpy(np.asarray(W, np.float64)).to(dtype)
    bt = None if b is None else torch.from_numpy(np.asarray(b, np.float64)).float()
    conv = co.Conv(d.cin, d.cout, d.kernel, weight=Wt.cuda(),
                   bias=None if bt is None else bt.cuda(), stride=d.stride, padding=d.padding,
                   dilation=d.dilation, groups=d.groups, spatial_rank=d.spatial_rank,
                   in_spatial=d.in_spatial, n_streams=B, dtype=dtype, out_dtype=out_dtype,
                   activation=activation, kernel=kernel, state_layout=state_layout)
    Wq = Wt.double().numpy()
    bq = None if bt is None else bt.double().numpy()
    sm = O.StepMachine(d, Wq, bq, B)
    return conv, sm, Wq, bq


def to_cl(x: np.ndarray, dtype) -> torch.Tensor:
    """numpy logical (B, C, ...) -> CUDA channels-last tensor."""
    import paper_2204_03418_b200 as co
    return co.channels_last(torch.from_numpy(np.ascontiguousarray(x)).to(dtype).cuda())


def np_of(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def rel_err(y, ref):
    y, ref = np.asarray(y), np.asarray(ref)
    if y.shape != ref.shape and y.size == ref.size:
        ref = ref.reshape(y.shape)
    rms = float(np.sqrt(np.mean(np.square(ref)))) if ref.size else 0.0
    return float(np.abs(y - ref).max()) / max(rms, 1e-30) if ref.size else 0.0


def assert_bf16_rounding_bound(y, ref, fp32_tol=1e-4):
    """bf16 outputs y vs the fp64 oracle ref (A16): y = RNE_bf16(v) with v the
    fp32 result, |v - ref| <= fp32_tol * RMS(ref); RNE has relative error
    <= u = 2^-8 (8 significant bits), so elementwise
    |y - ref| <= 2^-8 (|ref| + eps) + eps, eps = fp32_tol * RMS(ref)."""
    y, ref = np.asarray(y, np.float64), np.asarray(ref, np.float64).reshape(np.shape(y))
    eps = fp32_tol * float(np.sqrt(np.mean(np.square(ref))))
    bound = 2.0 ** -8 * (np.abs(ref) + eps) + eps
    bad = np.abs(y - ref) > bound
    assert not bad.any(), f"{int(bad.sum())} elements exceed the bf16 rounding bound; worst excess " \
                          f"{float((np.abs(y - ref) - bound).max()):.3e}"


def build_config_layers(cfg, B, last_fp32=True, kernel="auto", out_dtype=None, state_layout="psum"):
    """The config's layers on B streams exactly as bench.py builds them (same
    dispatch, kernels and launch geometry); the final layer emits fp32 for
    parity (A16: same kernel, only the final conversion differs)."""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    convs, descs, Ws, bs, spat = [], [], [], [], tuple(cfg.in_spatial)
    params = synth.params(cfg)
    for l, (L, (W, b)) in enumerate(zip(cfg.layers, params)):
        last = l == len(cfg.layers) - 1
        od = out_dtype or (torch.float32 if (last and last_fp32) else cfg.dtype)
        c = co.Conv(L.cin, L.cout, L.kernel, weight=W.cuda(), bias=b.cuda(), stride=L.stride, padding=L.padding,
                    dilation=L.dilation, groups=L.groups, spatial_rank=cfg.spatial_rank, in_spatial=spat,
                    n_streams=B, dtype=cfg.dtype, out_dtype=od, activation="relu" if L.relu else None,
                    kernel=kernel, state_layout=state_layout)
        d = O.Desc(cfg.spatial_rank, L.cin, L.cout, L.kernel, L.stride, L.padding, L.dilation, L.groups, spat)
        convs.append(c); descs.append(d); Ws.append(W.double().numpy()); bs.append(b.double().numpy())
        spat = tuple(c.out_spatial) + (1,) * (2 - len(c.out_spatial))
    return convs, descs, Ws, bs
