"""Pins for the Delay / Residual oracle (oracle/compose.py), CPU-only.

Ties it to: SPEC's Delay worked examples (tests/golden/delay_spec_examples.json);
the equal-padding residual as PyTorch's float64 conv3d plus the input (Fig. 4,
P:303-310); the paper's weight-compatibility statement for the centered
residual (its outputs equal the equal-padding residual's, cropped);
the closed form of a zero-weight body (the output is the input delayed by the
identity branch's delay); Principle 7's composite delay; and batch == step.
"""
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
from oracle import compose as OC

GOLD = os.path.join(os.path.dirname(__file__), "golden", "delay_spec_examples.json")


@pytest.mark.parametrize("case", json.load(open(GOLD))["cases"], ids=lambda c: c["cite"][:30])
def test_delay_worked_examples(case):
    dl = OC.DelayStep(case["d"])
    ready, outs = [], []
    for v in case["inputs"]:
        y = dl.forward_step(np.full((1, 1), float(v)))
        ready.append(int(y is not None))
        if y is not None:
            outs.append(float(y.ravel()[0]))
    assert ready == case["ready"] and outs == case["outputs"]


def test_delay_composes_additively():
    """Delay(d1) then Delay(d2) == Delay(d1 + d2) in step mode."""
    rng = np.random.default_rng(0)
    a, b, c = OC.DelayStep(2), OC.DelayStep(3), OC.DelayStep(5)
    for _ in range(12):
        x = rng.standard_normal((2, 3))
        y1 = a.forward_step(x)
        y2 = b.forward_step(y1) if y1 is not None else None
        y3 = c.forward_step(x)
        assert (y2 is None) == (y3 is None)
        if y2 is not None:
            np.testing.assert_array_equal(y2, y3)


def _conv_desc(cin, kt, pt, H=5, W=4):
    return O.Desc(2, cin, cin, (kt, 3, 3), padding=(pt, 1, 1), in_spatial=(H, W))


def _run_steps(res, frames, extra_zero_steps=0):
    outs = []
    for x in list(frames) + [np.zeros_like(frames[0])] * extra_zero_steps:
        y = res.forward_step(x)
        if y is not None:
            outs.append(y)
    return outs


def test_equal_padding_residual_is_x_plus_conv():
    """Fig. 4: with equal padding the residual computes x + conv(x);
    step mode (pad_end: p zero steps) reproduces the whole batch output."""
    rng = np.random.default_rng(1)
    d = _conv_desc(4, 3, 1)
    W = rng.standard_normal(d.w_shape) / 6
    b = rng.standard_normal(4) * 0.1
    B, T = 2, 7
    x = rng.standard_normal((B, 4, T, 5, 4))
    ref = (F.conv3d(torch.from_numpy(x), torch.from_numpy(W), torch.from_numpy(b), padding=(1, 1, 1))
           + torch.from_numpy(x)).numpy()
    res = OC.ResidualStep([d], [W], [b], [0], [0], B, shrink=False)
    assert res.d_skip == 1 and res.delay == 1
    got = np.stack(_run_steps(res, [x[:, :, t] for t in range(T)], extra_zero_steps=1), axis=2)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(OC.residual_forward([d], [W], [b], [0], x), ref, rtol=1e-12, atol=1e-12)


def test_centered_residual_is_weight_compatible():
    """the centered (shrink, no padding) residual's outputs equal
    the equal-padding residual's with the same weights, minus the border
    columns; its delay is the body's (2), its identity branch's 1."""
    rng = np.random.default_rng(2)
    d0, d1 = _conv_desc(3, 3, 0), _conv_desc(3, 3, 1)
    W = rng.standard_normal(d0.w_shape) / 5
    b = rng.standard_normal(3) * 0.1
    B, T = 2, 9
    frames = [rng.standard_normal((B, 3, 5, 4)) for _ in range(T)]
    shr = OC.ResidualStep([d0], [W], [b], [0], [0], B, shrink=True)
    eq = OC.ResidualStep([d1], [W], [b], [0], [0], B, shrink=False)
    assert (shr.delay, shr.d_skip) == (2, 1)
    a = np.stack(_run_steps(shr, frames), axis=2)
    e = np.stack(_run_steps(eq, frames, extra_zero_steps=1), axis=2)
    assert a.shape[2] == T - 2 and e.shape[2] == T
    np.testing.assert_allclose(a, e[:, :, 1:-1], rtol=1e-12, atol=1e-12)
    clip = np.stack(frames, axis=2)
    np.testing.assert_allclose(OC.residual_forward([d0], [W], [b], [0], clip, shrink=True), a, rtol=1e-12,
                               atol=1e-12)


@pytest.mark.parametrize("shrink", [False, True])
def test_zero_body_is_the_aligned_identity(shrink):
    """A body with zero weights and bias outputs 0, so the residual emits the
    input delayed by the identity branch's delay, from the body's first Ready
    tick on (closed form; Principle 7)."""
    rng = np.random.default_rng(3)
    descs = [_conv_desc(2, 5, 0 if shrink else 2), _conv_desc(2, 3, 0 if shrink else 1)]
    Ws = [np.zeros(d.w_shape) for d in descs]
    bs = [np.zeros(2) for _ in descs]
    res = OC.ResidualStep(descs, Ws, bs, [1, 0], [0, 0], 1, shrink=shrink)
    assert res.delay == (6 if shrink else 3) and res.d_skip == 3
    frames = [rng.standard_normal((1, 2, 5, 4)) for _ in range(10)]
    for n, x in enumerate(frames):
        y = res.forward_step(x)
        assert (y is None) == (n < res.delay)
        if y is not None:
            np.testing.assert_array_equal(y, frames[n - res.d_skip])


def test_two_layer_body_step_equals_batch_with_relu():
    rng = np.random.default_rng(4)
    descs = [_conv_desc(4, 3, 1), _conv_desc(4, 5, 2)]
    Ws = [rng.standard_normal(d.w_shape) / 8 for d in descs]
    bs = [rng.standard_normal(4) * 0.1 for _ in descs]
    B, T = 2, 8
    x = rng.standard_normal((B, 4, T, 5, 4))
    ref = OC.residual_forward(descs, Ws, bs, [1, 0], x, relu_out=True)
    res = OC.ResidualStep(descs, Ws, bs, [1, 0], [0, 0], B, relu_out=True)
    # outputs whose windows need no end padding: i <= T-1-p_acc (feeding zero
    # frames at the input is not per-layer end padding for a deeper body)
    got = np.stack(_run_steps(res, [x[:, :, t] for t in range(T)]), axis=2)
    assert got.shape[2] == T - 3
    np.testing.assert_allclose(got, ref[:, :, :T - 3], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("kt,p", [(5, 1), (7, 2), (7, 1), (3, 1)])
def test_padded_centered_residual_is_cropped_equal_padding(kt, p):
    """A centered residual whose body carries some padding p <= (f-1)/2 (ADVICE
    r1): its outputs are the equal-padding residual's (P:313-315 weight
    compatibility), column i being equal-padding column i + (f-1)/2 - p, and
    step mode reproduces batch mode on the columns that need no end padding."""
    rng = np.random.default_rng(kt * 10 + p)
    B, T, C = 2, 11, 3
    dp = _conv_desc(C, kt, p)
    de = _conv_desc(C, kt, (kt - 1) // 2)
    W = rng.standard_normal(dp.w_shape) / 6
    b = rng.standard_normal(C) * 0.1
    x = rng.standard_normal((B, C, T, 5, 4))
    y = OC.residual_forward([dp], [W], [b], [0], x, shrink=True)
    ye = OC.residual_forward([de], [W], [b], [0], x, shrink=False)
    off = (kt - 1) // 2 - p
    assert y.shape[2] == T + 2 * p - kt + 1
    np.testing.assert_allclose(y, ye[:, :, off:off + y.shape[2]], rtol=1e-12, atol=1e-12)
    res = OC.ResidualStep([dp], [W], [b], [0], [0], B, shrink=True)
    got = np.stack(_run_steps(res, [x[:, :, t] for t in range(T)]), axis=2)
    np.testing.assert_allclose(got, y[:, :, :got.shape[2]], rtol=1e-12, atol=1e-12)


def test_construction_errors():
    with pytest.raises(ValueError):      # even receptive field cannot be centered
        OC.skip_delay([_conv_desc(2, 2, 0)], shrink=True)
    with pytest.raises(ValueError):      # no equal padding without shrink
        OC.skip_delay([_conv_desc(2, 3, 0)], shrink=False)
    with pytest.raises(ValueError):      # centered: padding beyond (f-1)/2
        OC.skip_delay([_conv_desc(2, 5, 3)], shrink=True)


def test_broadcast_reduce_conv_delay_equals_residual():
    """Listing 3: BroadcastReduce(conv, Delay(1)) == Residual(conv)
    for an equal-padding conv -- in step mode and batch mode."""
    rng = np.random.default_rng(6)
    d = _conv_desc(3, 3, 1)
    W = rng.standard_normal(d.w_shape) / 5
    b = rng.standard_normal(3) * 0.1
    B, T = 2, 8
    frames = [rng.standard_normal((B, 3, 5, 4)) for _ in range(T)]
    conv = O.Stack([d], [W], [b], [0], [0], B)
    br = OC.BroadcastReduceStep([conv, None], [1, 0], "sum")
    res = OC.ResidualStep([d], [W], [b], [0], [0], B)
    assert br.delay == res.delay == 1
    for x in frames:
        a, r = br.forward_step(x), res.forward_step(x)
        assert (a is None) == (r is None)
        if a is not None:
            np.testing.assert_allclose(a, r, rtol=1e-13, atol=1e-13)
    clip = np.stack(frames, axis=2)
    yb = OC.broadcast_reduce_forward([lambda c: O.forward(d, W, b, c), None], clip)
    np.testing.assert_allclose(yb, OC.residual_forward([d], [W], [b], [0], clip), rtol=1e-13, atol=1e-13)


def test_broadcast_reduce_identities_scale_and_concat():
    """All-identity branches with sum scale by the branch count; concat stacks
    channels."""
    rng = np.random.default_rng(7)
    x = rng.standard_normal((2, 3, 4, 5))
    s3 = OC.BroadcastReduceStep([None, None, None], [0, 0, 0], "sum")
    np.testing.assert_array_equal(s3.forward_step(x), 3 * x)
    cat = OC.BroadcastReduceStep([None, None], [0, 0], "concat")
    np.testing.assert_array_equal(cat.forward_step(x), np.concatenate([x, x], axis=1))


def test_broadcast_reduce_step_equals_batch_unpadded_branches():
    """Branches of different receptive fields without padding: each Ready step
    output equals the batch merge column with the same index (delay alignment,
    A24); the composite delay is the maximum (Principle 7)."""
    rng = np.random.default_rng(8)
    d3, d5 = _conv_desc(2, 3, 0), _conv_desc(2, 5, 0)
    W3, W5 = rng.standard_normal(d3.w_shape) / 4, rng.standard_normal(d5.w_shape) / 5
    b3, b5 = rng.standard_normal(2) * 0.1, rng.standard_normal(2) * 0.1
    B, T = 2, 11
    frames = [rng.standard_normal((B, 2, 5, 4)) for _ in range(T)]
    for reduce in ("sum", "concat"):
        br = OC.BroadcastReduceStep([O.Stack([d3], [W3], [b3], [0], [0], B), O.Stack([d5], [W5], [b5], [0], [0], B),
                                     None], [2, 4, 0], reduce)
        assert br.delay == 4
        outs = [br.forward_step(x) for x in frames]
        assert all((o is None) == (t < 4) for t, o in enumerate(outs))
        clip = np.stack(frames, axis=2)
        yb = OC.broadcast_reduce_forward([lambda c: O.forward(d3, W3, b3, c), lambda c: O.forward(d5, W5, b5, c),
                                          None], clip, reduce)
        got = np.stack([o for o in outs if o is not None], axis=2)
        assert got.shape == yb.shape
        np.testing.assert_allclose(got, yb, rtol=1e-12, atol=1e-12)
