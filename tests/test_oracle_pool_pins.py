"""Pins for the pooling oracle (oracle/pool.py), CPU-only.

Ties oracle.pool to things other than itself: SPEC's worked examples
(tests/golden/pool_spec_examples.json, each cited), PyTorch's float64
max_pool3d / avg_pool3d / conv3d as independent library routines (explicit
-inf or zero padding so every temporal padding 0..f-1 is covered), and the
batch/step equivalence property (Definition 1).
"""
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import pool as OP

GOLD = os.path.join(os.path.dirname(__file__), "golden", "pool_spec_examples.json")


def _gold():
    with open(GOLD) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _gold()["forward"], ids=lambda c: c["cite"][:40])
def test_forward_worked_examples(case):
    x = np.asarray(case["inputs"], np.float64).reshape(1, 1, -1, 1, 1)
    y = OP.pool_forward(case["kind"], x, (case["kernel"], 1, 1), (case["stride"], 1, 1), (case["padding"], 0, 0))
    assert y.ravel().tolist() == case["outputs"]


@pytest.mark.parametrize("case", _gold()["step"], ids=lambda c: c["cite"][:40])
def test_step_worked_examples(case):
    sm = OP.PoolStep(case["kind"], 1, (1, 1), (case["kernel"], 1, 1), (case["stride"], 1, 1), (case["padding"], 0, 0))
    ready, outs = [], []
    for v in case["inputs"]:
        y = sm.forward_step(np.full((1, 1, 1, 1), float(v)))
        ready.append(int(y is not None))
        if y is not None:
            outs.append(float(y.ravel()[0]))
    assert ready == case["ready"] and outs == case["outputs"]


def torch_pool(kind, x, kernel, stride, padding, dilation):
    """Independent reference: explicit padding (-inf for MAX, 0 for AVG), then
    the library pool (MAX) or a ones-kernel depthwise conv / window size (AVG)."""
    xt = torch.from_numpy(x)
    pt, ph, pw = padding
    fill = float("-inf") if kind == "max" else 0.0
    xp = F.pad(xt, (pw, pw, ph, ph, pt, pt), value=fill)
    if kind == "max":
        return F.max_pool3d(xp, kernel, stride, 0, dilation).numpy()
    C = x.shape[1]
    w = torch.ones((C, 1) + tuple(kernel), dtype=torch.float64) / float(np.prod(kernel))
    y = F.conv3d(xp, w, None, stride, 0, dilation, groups=C)
    if dilation == (1, 1, 1):      # second library route for the dilation-free case
        y2 = F.avg_pool3d(xt, kernel, stride, 0, count_include_pad=True) if padding == (0, 0, 0) else \
            F.avg_pool3d(xp, kernel, stride, 0)
        np.testing.assert_allclose(y.numpy(), y2.numpy(), rtol=1e-13, atol=1e-13)
    return y.numpy()


def rand_cfg(rng):
    kt = int(rng.integers(1, 5))
    dt = int(rng.integers(1, 3))
    f = dt * (kt - 1) + 1
    kh, kw = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    kernel = (kt, kh, kw)
    stride = (int(rng.integers(1, 3)), int(rng.integers(1, 3)), int(rng.integers(1, 3)))
    dilation = (dt, int(rng.integers(1, 3)), 1)
    padding = (int(rng.integers(0, f)), int(rng.integers(0, kh)), int(rng.integers(0, kw)))
    return kernel, stride, padding, dilation


@pytest.mark.parametrize("kind", ["max", "avg"])
def test_forward_matches_library(kind):
    rng = np.random.default_rng(11 if kind == "max" else 12)
    for _ in range(25):
        kernel, stride, padding, dilation = rand_cfg(rng)
        f = dilation[0] * (kernel[0] - 1) + 1
        T = int(rng.integers(max(1, f - 2 * padding[0]), f + 5))
        H = int(rng.integers(max(1, dilation[1] * (kernel[1] - 1) + 1 - 2 * padding[1]), 6))
        W = int(rng.integers(max(1, kernel[2] - 2 * padding[2]), 6))
        x = rng.standard_normal((2, 3, T, H, W))
        y = OP.pool_forward(kind, x, kernel, stride, padding, dilation)
        ref = torch_pool(kind, x, kernel, stride, padding, tuple(dilation))
        assert y.shape == ref.shape
        np.testing.assert_allclose(y, ref, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("kind", ["max", "avg"])
def test_step_equals_batch_with_pad_end(kind):
    """Ready outputs of a clean stream followed by p padding steps equal the
    batch output."""
    rng = np.random.default_rng(21 if kind == "max" else 22)
    for _ in range(20):
        kernel, stride, padding, dilation = rand_cfg(rng)
        f = dilation[0] * (kernel[0] - 1) + 1
        T = int(rng.integers(max(1, f - 2 * padding[0]), f + 6))
        H, W = 4, 5
        x = rng.standard_normal((2, 3, T, H, W))
        ref = OP.pool_forward(kind, x, kernel, stride, padding, dilation)
        sm = OP.PoolStep(kind, 3, (H, W), kernel, stride, padding, dilation, B=2)
        outs = []
        for t in range(T):
            y = sm.forward_step(x[:, :, t])
            if y is not None:
                outs.append(y)
        for _ in range(padding[0]):
            y = sm.forward_step(None)
            if y is not None:
                outs.append(y)
        got = np.stack(outs, axis=2)
        assert got.shape == ref.shape
        np.testing.assert_array_equal(got, ref)


def test_update_state_false_leaves_state():
    sm = OP.PoolStep("max", 1, (1, 1), (3, 1, 1))
    for v in (1.0, 4.0):
        sm.forward_step(np.full((1, 1, 1, 1), v))
    probe = sm.forward_step(np.full((1, 1, 1, 1), 9.0), update_state=False)
    assert float(probe.ravel()[0]) == 9.0 and sm.n == 2
    y = sm.forward_step(np.full((1, 1, 1, 1), 2.0))
    assert float(y.ravel()[0]) == 4.0


def test_padding_bounds():
    with pytest.raises(ValueError):
        OP.PoolStep("avg", 1, (1, 1), (3, 1, 1), padding=(3, 0, 0))


@pytest.mark.parametrize("kind", ["max", "avg"])
def test_reduced_history_folds_to_the_step_output(kind):
    """Separability (k_pool.cu's design, checked on the oracle): folding the
    reduced history's taps with the new frame's spatial reduction gives the
    step output (AVG: divided by kt kh kw)."""
    rng = np.random.default_rng(31)
    kernel, stride, padding, dilation = (3, 3, 2), (1, 2, 1), (2, 1, 1), (2, 1, 1)
    sm = OP.PoolStep(kind, 2, (5, 4), kernel, stride, padding, dilation, B=2)
    probe = OP.PoolStep(kind, 2, (5, 4), (1,) + kernel[1:], stride, (0,) + padding[1:], (1,) + dilation[1:], B=2)
    for _ in range(9):
        x = rng.standard_normal((2, 2, 5, 4))
        hist = sm.reduced_history()                       # (f-1, B, C, H', W')
        y = sm.forward_step(x, update_state=False)
        if y is None:
            sm.forward_step(x)
            continue
        cur = probe.forward_step(x, update_state=False)   # spatial-only window
        f, dil = sm.f, dilation[0]
        taps = [hist[k * dil] for k in range(kernel[0] - 1)]
        if kind == "max":
            exp = np.maximum.reduce(taps + [cur])
        else:
            exp = (sum(taps) + cur * (kernel[1] * kernel[2])) / np.prod(kernel)
        np.testing.assert_allclose(y, exp, rtol=1e-12, atol=1e-12)
        sm.forward_step(x)
