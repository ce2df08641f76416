"""Pins for the continual MHA oracle (oracle/mha.py), CPU-only: SPEC's worked
cases (identity projections on a constant input, the n = 1 window,
saturation on a repeated input), PyTorch's float64 nn.MultiheadAttention as an
independent library for the batch form, and window equivalence (each step's
output is the last column of the batch form over the trailing n steps)."""
import numpy as np
import pytest
import torch

from oracle import mha as OM


def _params(rng, E, heads, bias=True, scale=None):
    s = scale or 1.0 / np.sqrt(E)
    p = {"heads": heads}
    for n in ("Wq", "Wk", "Wv", "Wo"):
        p[n] = rng.standard_normal((E, E)) * s
    if bias:
        for n in ("bq", "bk", "bv", "bo"):
            p[n] = rng.standard_normal(E) * 0.1
    return p


def test_identity_projections_constant_input():
    """h = 1, identity projections, x constant over T: uniform softmax over
    identical values -> the output is the value vector."""
    E, T = 6, 5
    I = np.eye(E)
    p = {"heads": 1, "Wq": I, "Wk": I, "Wv": I, "Wo": I}
    x = np.tile(np.arange(1.0, E + 1.0)[None, :, None], (2, 1, T))
    np.testing.assert_allclose(OM.mha_forward(p, x), x, rtol=0, atol=1e-14)


def test_window_one_is_the_value_path():
    """n = 1: Ready at tick 0 with W_o (W_v x + b_v) + b_o."""
    rng = np.random.default_rng(0)
    E = 8
    p = _params(rng, E, 2)
    sm = OM.MhaStep(p, 1, B=3)
    x = rng.standard_normal((3, E))
    y = sm.forward_step(x)
    exp = (x @ p["Wv"].T + p["bv"]) @ p["Wo"].T + p["bo"]
    np.testing.assert_allclose(y, exp, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("E,heads,T", [(8, 1, 4), (16, 4, 7), (32, 8, 5)])
def test_batch_form_matches_torch_mha(E, heads, T):
    rng = np.random.default_rng(E + heads)
    p = _params(rng, E, heads)
    B = 2
    x = rng.standard_normal((B, E, T))
    m = torch.nn.MultiheadAttention(E, heads, bias=True, dtype=torch.float64)
    with torch.no_grad():
        m.in_proj_weight.copy_(torch.from_numpy(np.concatenate([p["Wq"], p["Wk"], p["Wv"]])))
        m.in_proj_bias.copy_(torch.from_numpy(np.concatenate([p["bq"], p["bk"], p["bv"]])))
        m.out_proj.weight.copy_(torch.from_numpy(p["Wo"]))
        m.out_proj.bias.copy_(torch.from_numpy(p["bo"]))
        xt = torch.from_numpy(np.ascontiguousarray(x.transpose(2, 0, 1)))     # (T, B, E)
        ref, _ = m(xt, xt, xt, need_weights=False)
    np.testing.assert_allclose(OM.mha_forward(p, x), ref.numpy().transpose(1, 2, 0), rtol=1e-11, atol=1e-12)


def test_step_is_last_column_of_the_window():
    """n = 3, a stream of 7 steps: ticks 0-1 Empty, then each Ready output is
    the last column of the batch form over the trailing 3 steps."""
    rng = np.random.default_rng(1)
    E, heads, n = 12, 3, 3
    p = _params(rng, E, heads)
    sm = OM.MhaStep(p, n, B=2)
    xs = [rng.standard_normal((2, E)) for _ in range(7)]
    for t, x in enumerate(xs):
        y = sm.forward_step(x)
        assert (y is None) == (t < n - 1)
        if y is not None:
            win = np.stack(xs[t - n + 1:t + 1], axis=2)
            np.testing.assert_allclose(y, OM.mha_forward(p, win)[:, :, -1], rtol=1e-12, atol=1e-12)


def test_repeated_input_saturates_and_update_state_false():
    rng = np.random.default_rng(2)
    E, n = 8, 4
    p = _params(rng, E, 2)
    sm = OM.MhaStep(p, n, B=1)
    x = rng.standard_normal((1, E))
    outs = [sm.forward_step(x) for _ in range(8)]
    for y in outs[n:]:
        np.testing.assert_allclose(y, outs[n - 1], rtol=1e-13, atol=1e-13)
    probe = sm.forward_step(rng.standard_normal((1, E)), update_state=False)
    assert probe is not None and sm.n == 8
    np.testing.assert_allclose(sm.forward_step(x), outs[-1], rtol=1e-13, atol=1e-13)
