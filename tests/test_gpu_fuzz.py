"""Seeded random-shape sweep of the dispatched bf16 kernels (tcgen05 HALO / FLAT /
KLOOP / KHALO, pairs, depthwise) against the generic CUDA-core kernel
(k_step_direct, itself pinned to the fp64 oracle in test_gpu_direct.py) on the
same inputs, over enough ticks to pass the delay: the planner's corner cases
(ragged tiles, odd stream counts, phase halos of odd sizes, temporal stride and
dilation) at sizes the oracle would take minutes for.  fp32 outputs, bar 1e-4
of the RMS (A16: both sides accumulate exact bf16 products in fp32).
"""
import numpy as np
import pytest
import torch

import oracle as O
from tests.helpers import np_of, rel_err, to_cl

pytestmark = pytest.mark.gpu


def _shape(rng):
    dense = rng.random() < 0.75
    kt = int(rng.choice([1, 2, 3, 5]))
    kh = int(rng.choice([1, 3, 3, 5]))
    s = int(rng.choice([1, 1, 2]))
    ph = kh // 2 if rng.random() < 0.8 else 0
    pt = int(rng.integers(0, kt)) if rng.random() < 0.3 else 0
    st = 2 if (kt > 1 and rng.random() < 0.2) else 1
    dt = 2 if (kt > 1 and st == 1 and rng.random() < 0.2) else 1
    H = int(rng.integers(kh + 2, 30))
    W = int(rng.integers(kh + 2, 40))
    if dense:
        cin = int(rng.choice([16, 32, 64, 128, 192, 256]))
        cout = int(rng.choice([16, 32, 64, 96, 128, 160, 256]))
        groups = 1
    else:
        cin = cout = groups = int(rng.choice([32, 64, 96]))
        s = 1
    if pt > dt * (kt - 1):
        pt = 0
    d = O.Desc(2, cin, cout, (kt, kh, kh), stride=(st, s, s), padding=(pt, ph, ph), dilation=(dt, 1, 1),
               groups=groups, in_spatial=(H, W))
    B = int(rng.integers(1, 6))
    return d, B


CASES = list(range(120))   # ~40% KHALO, ~35% HALO / FLAT, ~25% depthwise / K-loop / direct


@pytest.mark.parametrize("seed", CASES)
def test_fuzz_dispatched_vs_direct(seed):
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(9000 + seed)
    d, B = _shape(rng)
    W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    b = rng.standard_normal(d.cout) * 0.1
    Wt = torch.from_numpy(W).to(torch.bfloat16).cuda()
    bt = torch.from_numpy(b).float().cuda()
    mk = lambda kernel: co.Conv(d.cin, d.cout, d.kernel, weight=Wt, bias=bt, stride=d.stride, padding=d.padding,
                                dilation=d.dilation, groups=d.groups, spatial_rank=2, in_spatial=d.in_spatial,
                                n_streams=B, dtype=torch.bfloat16, out_dtype=torch.float32, kernel=kernel)
    fast, ref = mk("auto"), mk("direct")
    H, Wd = d.in_hw
    ys, rs = [], []
    for t in range(d.receptive_field + 3 * d.stride[0] + 2):
        x = to_cl(rng.standard_normal((B, d.cin, H, Wd)), torch.bfloat16)
        y, r = fast.forward_step(x), ref.forward_step(x)
        assert (y is None) == (r is None), (t, fast.kernel_name)
        if y is not None:
            ys.append(np_of(y)); rs.append(np_of(r))
    assert ys, d
    err = rel_err(np.stack(ys), np.stack(rs))
    assert err <= 1e-4, (fast.kernel_name, d, B, err)


@pytest.mark.parametrize("seed", list(range(40)))
def test_fuzz_bf16_relu_vs_direct(seed):
    """The same sweep with ReLU and bf16 outputs (the bench's dtype): both sides
    round nearly equal fp32 sums (different accumulation orders) to bf16 with
    RNE, so each output may differ by one bf16 rounding of either side: the bar
    is 2 * 2^-8 of the value (A16's RNE bound, applied to both roundings) plus
    1e-3 of the RMS for the fp32 order differences near zero."""
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(19000 + seed)
    d, B = _shape(rng)
    W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    b = rng.standard_normal(d.cout) * 0.1
    Wt = torch.from_numpy(W).to(torch.bfloat16).cuda()
    bt = torch.from_numpy(b).float().cuda()
    mk = lambda kernel: co.Conv(d.cin, d.cout, d.kernel, weight=Wt, bias=bt, stride=d.stride, padding=d.padding,
                                dilation=d.dilation, groups=d.groups, spatial_rank=2, in_spatial=d.in_spatial,
                                n_streams=B, dtype=torch.bfloat16, out_dtype=torch.bfloat16, activation="relu",
                                kernel=kernel)
    fast, ref = mk("auto"), mk("direct")
    H, Wd = d.in_hw
    ys, rs = [], []
    for t in range(d.receptive_field + 3 * d.stride[0] + 2):
        x = to_cl(rng.standard_normal((B, d.cin, H, Wd)), torch.bfloat16)
        y, r = fast.forward_step(x), ref.forward_step(x)
        assert (y is None) == (r is None), (t, fast.kernel_name)
        if y is not None:
            ys.append(np_of(y)); rs.append(np_of(r))
    y, r = np.stack(ys), np.stack(rs)
    assert (y >= 0).all()
    rms = float(np.sqrt(np.mean(r ** 2)))
    excess = (np.abs(y - r) - (2.0 ** -7 * np.maximum(np.abs(y), np.abs(r)) + 1e-3 * rms)).max()
    assert excess <= 0, (fast.kernel_name, d, B, excess, rel_err(y, r))


def _oracle_cases(n=24, budget=1.5e9):
    """Seeded shapes of the same sweep whose fp64 oracle run stays small: the
    MACs of every Ready output over the run <= budget.  Deterministic."""
    out, seed = [], 40000
    while len(out) < n:
        rng = np.random.default_rng(seed)
        d, B = _shape(rng)
        ticks = d.receptive_field + 3 * d.stride[0] + 2
        Ho, Wo = d.out_spatial
        macs = B * ticks * d.cout * (d.cin // d.groups) * int(np.prod(d.kernel)) * Ho * Wo
        if macs <= budget:
            out.append(seed)
        seed += 1
    return out


@pytest.mark.parametrize("seed", _oracle_cases())
def test_fuzz_dispatched_vs_oracle(seed):
    """Shapes of the same sweep checked against the fp64 ORACLE itself (not the
    CUDA-core kernel), so an error shared by both CUDA paths -- weight packing,
    the host clock's slot arguments, the bias -- cannot pass: ready / n / head
    per tick bit-exact, outputs within 1e-4 of the RMS."""
    from tests.helpers import make_pair
    rng = np.random.default_rng(seed)
    d, B = _shape(rng)
    W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    b = rng.standard_normal(d.cout) * 0.1
    conv, sm, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, out_dtype=torch.float32)
    H, Wd = d.in_hw
    ys, rs = [], []
    for t in range(d.receptive_field + 3 * d.stride[0] + 2):
        x = to_cl(rng.standard_normal((B, d.cin, H, Wd)), torch.bfloat16)
        y = conv.forward_step(x)
        r = sm.forward_step(np_of(x))
        assert (y is None) == (r is None), (t, conv.kernel_name)
        assert (conv.n, conv.head) == (sm.n, sm.head)
        if y is not None:
            ys.append(np_of(y)); rs.append(r.reshape(y.shape))
    assert ys, d
    err = rel_err(np.stack(ys), np.stack(rs))
    assert err <= 1e-4, (conv.kernel_name, d, B, err)
