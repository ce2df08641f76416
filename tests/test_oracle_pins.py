"""Pins for the fp64 oracle (oracle/), all CPU-only (`-m "not gpu"`).

Each test ties the oracle to something other than itself: numbers printed in
PAPER.md (tests/golden/*.json, each with its citation), hand-checkable closed
forms, the textbook convolution as implemented by an independent library
(torch.nn.functional.conv{1,2,3}d in float64 on the CPU; the oracle does not
use torch), and special cases that reduce to simpler routines.  A plausible
mistake in the oracle (dropped term, wrong sign/index, transposed operand,
off-by-one in the delay or in the stride phase, wrong rotation direction)
fails at least one of them.
"""
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def torch_conv(d: O.Desc, W, bias, x, tpad):
    """Independent reference: regular conv with temporal padding `tpad` (both ends)."""
    W = torch.from_numpy(np.asarray(W, np.float64).reshape(d.w_shape))
    b = None if bias is None else torch.from_numpy(np.asarray(bias, np.float64))
    x = torch.from_numpy(np.asarray(x, np.float64))
    B, T = x.shape[0], x.shape[2]
    H, Wd = d.in_hw
    x5 = x.reshape(B, d.cin, T, H, Wd)
    k = list(d.kernel) + [1, 1]
    s = list(d.stride) + [1, 1]
    p = list(d.padding) + [0, 0]
    dl = list(d.dilation) + [1, 1]
    if d.spatial_rank < 1:
        k[1], s[1], p[1], dl[1] = 1, 1, 0, 1
    if d.spatial_rank < 2:
        k[2], s[2], p[2], dl[2] = 1, 1, 0, 1
    y = F.conv3d(x5, W, b, stride=tuple(s[:3]), padding=(tpad, p[1], p[2]), dilation=tuple(dl[:3]),
                 groups=d.groups)
    return y.numpy()


def rand_desc(rng):
    rank = int(rng.integers(0, 3))
    kt = int(rng.integers(1, 6))
    dil = int(rng.integers(1, 4))
    f = dil * (kt - 1) + 1
    p = int(rng.integers(0, f))
    s = int(rng.integers(1, 4))
    cin = int(rng.integers(1, 5))
    groups = int(rng.choice([1, cin]))
    cout = groups * int(rng.integers(1, 3)) if groups > 1 else int(rng.integers(1, 5))
    kh = int(rng.integers(1, 4)) if rank >= 1 else 1
    kw = int(rng.integers(1, 4)) if rank >= 2 else 1
    H = int(rng.integers(max(kh, 1), 6)) if rank >= 1 else 1
    Wd = int(rng.integers(max(kw, 1), 6)) if rank >= 2 else 1
    sh, sw = int(rng.integers(1, 3)), int(rng.integers(1, 3))
    ph, pw = int(rng.integers(0, 2)), int(rng.integers(0, 2))
    d = O.Desc(spatial_rank=rank, cin=cin, cout=cout, kernel=(kt, kh, kw), stride=(s, sh, sw),
               padding=(p, ph, pw), dilation=(dil, 1, 1), groups=groups, in_spatial=(H, Wd))
    assert d.valid()
    return d


# --------------------------------------------------------------- timing pins

def test_worked_example_accumulated_timing():
    g = gold("worked_example_P266-278.json")
    acc = O.accumulate(g["f"], g["p"], g["s"])
    for key in ("s_acc", "p_acc", "f_acc", "d_acc", "s_nn", "d_nn"):
        assert acc[key] == g[key], key
    assert [1, acc["s_nn"]] == g["r_nn"]


def test_listing1_delay_and_receptive_field():
    g = gold("paper_timing_facts.json")["listing1"]
    d = O.Desc(2, g["cin"], g["cout"], (3, 3, 3), in_spatial=(g["H"], g["W"]))
    assert d.delay == g["delay"]
    assert d.receptive_field == g["receptive_field"]


def test_listing1_modes_match_regular_conv():
    """Listing 1: forward == nn.Conv3d; forward_steps(x[:,:,:4]) ==
    y[:,:,:delay]; forward_step(x[:,:,4]) == y[:,:,delay]."""
    g = gold("paper_timing_facts.json")["listing1"]
    rng = np.random.default_rng(0)
    d = O.Desc(2, g["cin"], g["cout"], (3, 3, 3), in_spatial=(g["H"], g["W"]))
    W = rng.standard_normal(d.w_shape)
    b = rng.standard_normal(d.cout)
    x = rng.standard_normal((g["B"], g["cin"], g["T"], g["H"], g["W"]))
    y = O.forward(d, W, b, x)
    np.testing.assert_allclose(y, torch_conv(d, W, b, x, 0), rtol=0, atol=1e-12)
    sm = O.StepMachine(d, W, b, g["B"])
    firsts, mask = sm.forward_steps(x[:, :, : g["forward_steps_T"]])
    assert firsts.shape[2] == g["forward_steps_n_out"]
    np.testing.assert_allclose(firsts, y[:, :, : d.delay], rtol=0, atol=1e-12)
    last = sm.forward_step(x[:, :, g["forward_steps_T"]])
    np.testing.assert_allclose(last, y[:, :, g["last_step_column"]], rtol=0, atol=1e-12)


@pytest.mark.parametrize("fig", ["fig1", "fig2"])
def test_fig1_fig2_first_ready(fig):
    g = gold("paper_timing_facts.json")[fig]
    d = O.Desc(0, 1, 1, (g["kernel"],), padding=(g["padding"],))
    sm = O.StepMachine(d, np.ones(d.w_shape), None, 1)
    ticks = [t for t in range(6) if sm.forward_step(np.ones((1, 1))) is not None]
    assert ticks[0] == g["first_ready_tick"]
    if "delay" in g:
        assert d.delay == g["delay"]


def test_fig3_executed_schedule():
    g = gold("paper_timing_facts.json")["fig3"]
    descs = [O.Desc(0, 1, 1, (l["kernel"],), stride=(l["stride"],), padding=(l["padding"],)) for l in g["layers"]]
    rng = np.random.default_rng(1)
    st = O.Stack(descs, [rng.standard_normal(dd.w_shape) for dd in descs], [None, None], [0, 0], [0, 0], B=1)
    pattern = [st.forward_step(rng.standard_normal((1, 1))) is not None for _ in range(10)]
    assert pattern == g["ready_first_10"]
    acc = O.accumulate([dd.receptive_field for dd in descs], [dd.padding[0] for dd in descs],
                       [dd.stride[0] for dd in descs])
    assert O.schedule(acc["d_nn"], acc["s_nn"], 10) == g["ready_first_10"]


def test_config_delays():
    # C4 (BJ configs[3]): all s_t = 1, p_t = 0 -> d_NN = sum(kt - 1) = 4+0+2+2+2 = 10
    kts = [5, 1, 3, 3, 3]
    acc = O.accumulate(kts, [0] * 5, [1] * 5)
    assert acc["d_nn"] == sum(k - 1 for k in kts) == 10
    # C5 (configs[4]): kt 9, dilation 2 -> f = 17, d = 16, 16 ring slots
    d5 = O.Desc(0, 256, 256, (9,), dilation=(2,))
    assert (d5.receptive_field, d5.delay, d5.ring_slots) == (17, 16, 16)
    # C3 chain (configs[2]): delays 2 + 4 = 6
    assert O.accumulate([3, 5], [0, 0], [1, 1])["d_nn"] == 6


# --------------------------------------------------------------- closed forms

def test_closed_forms_ones_kernel():
    g = gold("closed_forms_ones_kernel.json")
    for c in g["cases"]:
        d = O.Desc(0, 1, 1, (c["kernel"],), stride=(c["stride"],), padding=(c["padding"],),
                   dilation=(c["dilation"],))
        sm = O.StepMachine(d, np.ones(d.w_shape), None, 1)
        x = np.asarray(c["inputs"], np.float64).reshape(1, 1, -1)
        y, mask = sm.forward_steps(x, pad_end=c["pad_end"])
        assert mask.astype(int).tolist() == c["ready"], c["name"]
        assert y.reshape(-1).tolist() == c["outputs"], c["name"]
    for c in g["out_len"]:
        d = O.Desc(0, 1, 1, (c["kernel"],), stride=(c["stride"],), padding=(c["padding"],))
        assert d.out_len(c["T"]) == c["T_out"]


def test_flops_cost_model():
    # S:501/522 convention (1 MAC = 2 FLOP).  C2: 2*64*64*27*56*56.
    d2 = O.Desc(2, 64, 64, (3, 3, 3), padding=(0, 1, 1), in_spatial=(56, 56))
    assert d2.flops_step() == 2 * 64 * 64 * 27 * 56 * 56 == 693633024


# --------------------------------------------------------------- CIN identity

@pytest.mark.parametrize("seed", range(200))
def test_cin_identity_random(seed):
    """SC1 (Definition 1): clean-state forward_steps(pad_end) Ready
    outputs == batch forward == the textbook conv (torch f64), and the Ready
    ticks follow S:120 (d + i s)."""
    rng = np.random.default_rng(1000 + seed)
    d = rand_desc(rng)
    f, p = d.receptive_field, d.padding[0]
    T = int(rng.integers(max(1, f - 2 * p), 33))
    B = int(rng.integers(1, 3))
    H, Wd = d.in_hw
    x = rng.standard_normal((B, d.cin, T, H, Wd))
    W = rng.standard_normal(d.w_shape)
    b = rng.standard_normal(d.cout) if rng.random() < 0.7 else None
    ref = torch_conv(d, W, b, x, p)
    yb = O.forward(d, W, b, x)
    scale = max(1.0, np.abs(ref).max())
    np.testing.assert_allclose(yb, ref, rtol=0, atol=1e-12 * scale)
    sm = O.StepMachine(d, W, b, B)
    ys, mask = sm.forward_steps(x, pad_end=True)
    assert ys.shape == ref.shape
    np.testing.assert_allclose(ys, ref, rtol=0, atol=1e-12 * scale)
    expect = [t >= d.delay and (t - d.delay) % d.stride[0] == 0 for t in range(T + p)]
    assert mask.tolist() == expect


@pytest.mark.parametrize("cin,groups,cout", [(4, 2, 6), (6, 3, 3), (8, 4, 8), (6, 2, 4)])
def test_grouped_conv_between_dense_and_depthwise(cin, groups, cout):
    """Groups strictly between 1 and Cin (the channel offset g(o) Cin/g + c' of
    O1 is only exercised there): batch and step outputs == torch f64 conv3d."""
    rng = np.random.default_rng(77 + cin * 10 + groups)
    d = O.Desc(2, cin, cout, (3, 2, 3), stride=(1, 1, 2), padding=(1, 1, 0), groups=groups, in_spatial=(4, 5))
    W = rng.standard_normal(d.w_shape)
    b = rng.standard_normal(cout)
    x = rng.standard_normal((2, cin, 7, 4, 5))
    ref = torch_conv(d, W, b, x, d.padding[0])
    np.testing.assert_allclose(O.forward(d, W, b, x), ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))
    ys, _ = O.StepMachine(d, W, b, 2).forward_steps(x, pad_end=True)
    np.testing.assert_allclose(ys, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))


@pytest.mark.parametrize("kt,dil,p,s", [(3, 1, 0, 2), (3, 2, 1, 3), (5, 1, 2, 2), (2, 3, 0, 2), (4, 1, 0, 3)])
def test_out_len_matches_library_including_too_short(kt, dil, p, s):
    """T' = floor((T + 2p - f)/s) + 1, an error when T' < 1.  Pinned
    against torch's own output length for every short T (torch raises where the
    clip is too short, which must be exactly where T' < 1)."""
    d = O.Desc(0, 1, 1, (kt,), stride=(s,), padding=(p,), dilation=(dil,))
    for T in range(0, 12):
        try:
            t_lib = F.conv1d(torch.zeros(1, 1, T, dtype=torch.float64), torch.zeros(1, 1, kt, dtype=torch.float64),
                             stride=s, padding=p, dilation=dil).shape[-1]
        except RuntimeError:
            t_lib = 0
        assert max(d.out_len(T), 0) == t_lib, (T, d.out_len(T), t_lib)


@pytest.mark.parametrize("seed", range(30))
def test_ring_slots_is_max_pending_outputs(seed):
    """R, the canonical state's slot count, pinned by observation: the largest
    number of outputs that have received a contribution from a consumed frame
    but are not complete yet, counted on PyTorch's partial batch columns over
    a long run (outputs under stride that are never emitted are not pending)."""
    rng = np.random.default_rng(8800 + seed)
    d = rand_desc(rng)
    B = 1
    H, Wd = d.in_hw
    W = rng.standard_normal(d.w_shape) + 3.0           # no zero weights: a consumed tap always contributes
    sm = O.StepMachine(d, W, None, B)
    f, p, s, R = d.receptive_field, d.padding[0], d.stride[0], d.ring_slots
    T = d.delay + 3 * f + 2 * s
    frames = [rng.standard_normal((B, d.cin, H, Wd)) + 5.0 for _ in range(T)]
    d0 = O.Desc(**{**d.__dict__, "padding": (0,) + tuple(d.padding[1:])})
    emitted, most = 0, 0
    for n, xt in enumerate(frames, start=1):
        if sm.forward_step(xt) is not None:
            emitted += 1
        L = p + n + 2 * f + 2 * s
        clip = np.zeros((B, d.cin, L, H, Wd))
        for t in range(n):
            clip[:, :, p + t] = frames[t]
        ref = torch_conv(d0, W, None, clip, 0)
        # output column i is pending iff it is not emitted yet and a consumed real frame feeds it
        pending = 0
        for i in range(emitted, ref.shape[2]):
            taps = [i * s + k * d.dilation[0] for k in range(d.kernel[0])]
            if any(p <= q < p + n for q in taps):
                pending += 1
        most = max(most, pending)
        assert sm.state().shape[0] == R
    assert most == R, (most, R)


@pytest.mark.parametrize("seed", range(40))
def test_step_equals_sliding_window_bruteforce(seed):
    """O3 (ring of raw frames) vs O7 (re-run the batch conv over the whole
    padded history each tick) vs torch on that same window."""
    rng = np.random.default_rng(5000 + seed)
    d = rand_desc(rng)
    B = 2
    H, Wd = d.in_hw
    W = rng.standard_normal(d.w_shape)
    b = rng.standard_normal(d.cout)
    sm = O.StepMachine(d, W, b, B)
    frames = []
    for t in range(12):
        xt = rng.standard_normal((B, d.cin, H, Wd))
        frames.append(xt)
        hist = np.stack(frames, axis=2)
        y = sm.forward_step(xt)
        yb = O.bruteforce_tick(d, W, b, hist)
        assert (y is None) == (yb is None)
        if y is not None:
            np.testing.assert_allclose(y, yb, rtol=0, atol=1e-12 * max(1, np.abs(yb).max()))
            # the same window through torch: padded history, no padding, last column
            pz = np.concatenate([np.zeros((B, d.cin, d.padding[0], H, Wd)), hist], axis=2)
            d0 = O.Desc(**{**d.__dict__, "padding": (0,) + tuple(d.padding[1:])})
            ref = torch_conv(d0, W, b, pz, 0)[:, :, -1]
            np.testing.assert_allclose(y, ref, rtol=0, atol=1e-12 * max(1, np.abs(ref).max()))


@pytest.mark.parametrize("seed", range(20))
def test_exact_integer_regime(seed):
    """SC4: integer inputs/weights in [-2, 2] -> every sum is an exact integer,
    so step == batch == torch bit for bit."""
    rng = np.random.default_rng(7000 + seed)
    d = rand_desc(rng)
    T = max(d.receptive_field, 8)
    H, Wd = d.in_hw
    x = rng.integers(-2, 3, (2, d.cin, T, H, Wd)).astype(np.float64)
    W = rng.integers(-2, 3, d.w_shape).astype(np.float64)
    b = rng.integers(-2, 3, d.cout).astype(np.float64)
    ref = torch_conv(d, W, b, x, d.padding[0])
    ys, _ = O.StepMachine(d, W, b, 2).forward_steps(x, pad_end=True)
    assert np.array_equal(ys, ref)
    assert np.array_equal(O.forward(d, W, b, x), ref)


# --------------------------------------------------------------- special cases

@pytest.mark.parametrize("k_hot", [0, 1, 2, 3])
def test_one_hot_temporal_kernel_is_delayed_conv2d(k_hot):
    """SC5: W[:,:,k] the only non-zero slice -> y at tick n is Conv2d(W_k) of
    x_{n-(kt-1-k) dil}: a co.Delay composed with a per-frame conv.
    Pins the slice-to-frame mapping (rotation direction)."""
    rng = np.random.default_rng(11 + k_hot)
    kt, dil = 4, 2
    d = O.Desc(2, 3, 5, (kt, 3, 3), padding=(0, 1, 1), dilation=(dil, 1, 1), in_spatial=(6, 5))
    W = np.zeros(d.w_shape)
    W[:, :, k_hot] = rng.standard_normal((5, 3, 3, 3))
    b = rng.standard_normal(5)
    sm = O.StepMachine(d, W, b, 2)
    xs = [rng.standard_normal((2, 3, 6, 5)) for _ in range(14)]
    lag = (kt - 1 - k_hot) * dil
    for n, xt in enumerate(xs):
        y = sm.forward_step(xt)
        if n < d.delay:
            assert y is None
            continue
        ref = F.conv2d(torch.from_numpy(xs[n - lag]), torch.from_numpy(W[:, :, k_hot]),
                       torch.from_numpy(b), padding=1).numpy()
        np.testing.assert_allclose(y, ref, rtol=0, atol=1e-12)


def test_kt1_is_per_frame_conv2d():
    rng = np.random.default_rng(3)
    d = O.Desc(2, 4, 6, (1, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), in_spatial=(7, 8))
    assert d.delay == 0 and d.ring_slots == 0
    W = rng.standard_normal(d.w_shape)
    b = rng.standard_normal(6)
    sm = O.StepMachine(d, W, b, 3)
    for _ in range(3):
        xt = rng.standard_normal((3, 4, 7, 8))
        ref = F.conv2d(torch.from_numpy(xt), torch.from_numpy(W[:, :, 0]), torch.from_numpy(b),
                       stride=2, padding=1).numpy()
        np.testing.assert_allclose(sm.forward_step(xt), ref, rtol=0, atol=1e-12)


def test_depthwise_temporal_ones_is_moving_sum():
    """SC5: depthwise temporal ones kernel (groups = C, 1x1 spatial) -> per-channel moving sum."""
    rng = np.random.default_rng(4)
    C_, kt = 6, 5
    d = O.Desc(2, C_, C_, (kt, 1, 1), groups=C_, in_spatial=(3, 3))
    sm = O.StepMachine(d, np.ones(d.w_shape), None, 1)
    xs = [rng.standard_normal((1, C_, 3, 3)) for _ in range(10)]
    for n, xt in enumerate(xs):
        y = sm.forward_step(xt)
        if n >= kt - 1:
            np.testing.assert_allclose(y, sum(xs[n - kt + 1: n + 1]), rtol=0, atol=1e-12)


# --------------------------------------------------------------- state rules

@pytest.mark.parametrize("seed", range(30))
def test_canonical_state_is_partial_conv_of_consumed_frames(seed):
    """O5 vs torch: slot j = output i_next + j of the regular conv over the
    padded clip in which every frame not yet consumed is zero, bias excluded."""
    rng = np.random.default_rng(9000 + seed)
    d = rand_desc(rng)
    B = 2
    H, Wd = d.in_hw
    W = rng.standard_normal(d.w_shape)
    b = rng.standard_normal(d.cout)
    sm = O.StepMachine(d, W, b, B)
    n_steps = int(rng.integers(0, 10))
    frames = [rng.standard_normal((B, d.cin, H, Wd)) for _ in range(n_steps)]
    for xt in frames:
        sm.forward_step(xt)
    st = sm.state()
    R, f, p, s = d.ring_slots, d.receptive_field, d.padding[0], d.stride[0]
    assert st.shape[0] == R
    if R == 0:
        return
    i_next = -((-(n_steps - d.delay)) // s)          # ceil((n - d) / s)
    # padded clip long enough for every pending output: [p zeros | frames | zeros]
    L = (i_next + R - 1) * s + f + 1
    clip = np.zeros((B, d.cin, max(L, 1), H, Wd))
    for t, xt in enumerate(frames):
        if p + t < clip.shape[2]:
            clip[:, :, p + t] = xt
    d0 = O.Desc(**{**d.__dict__, "padding": (0,) + tuple(d.padding[1:])})
    ref = torch_conv(d0, W, None, clip, 0) if clip.shape[2] >= f else None
    for j in range(R):
        i = i_next + j
        if i < 0:
            assert np.all(st[j] == 0)
        else:
            np.testing.assert_allclose(st[j], ref[:, :, i], rtol=0, atol=1e-12 * max(1, np.abs(ref).max()))


def test_update_state_false_and_clean_state():
    """P:114 (update_state=False leaves state untouched), P:116 clean_state,
    S:121 replay determinism."""
    rng = np.random.default_rng(21)
    d = O.Desc(2, 3, 4, (3, 3, 3), padding=(1, 1, 1), in_spatial=(5, 5))
    W, b = rng.standard_normal(d.w_shape), rng.standard_normal(4)
    sm = O.StepMachine(d, W, b, 2)
    xs = [rng.standard_normal((2, 3, 5, 5)) for _ in range(6)]
    outs = [sm.forward_step(x) for x in xs]
    st, n = sm.state(), sm.n
    probe = rng.standard_normal((2, 3, 5, 5))
    y_peek = sm.forward_step(probe, update_state=False)
    assert sm.n == n and np.array_equal(sm.state(), st)
    y_real = sm.forward_step(probe)
    assert np.array_equal(y_peek, y_real)
    sm.clean_state()
    assert sm.n == 0 and np.all(sm.state() == 0)
    outs2 = [sm.forward_step(x) for x in xs]
    for a, c in zip(outs, outs2):
        assert (a is None and c is None) or np.array_equal(a, c)


def test_head_convention_definition():
    """head = ceil((n-d)/s) mod R (ABI convention, A20; unpinned by the paper):
    for f = 3 it alternates [0, 1, 0, 1, ...] from n = 0."""
    d = O.Desc(0, 1, 1, (3,))
    sm = O.StepMachine(d, np.ones(d.w_shape), None, 1)
    heads = []
    for _ in range(6):
        heads.append(sm.head)
        sm.forward_step(np.ones((1, 1)))
    assert heads == [0, 1, 0, 1, 0, 1]


@pytest.mark.parametrize("seed", range(40))
def test_head_is_next_output_index(seed):
    """head pinned by observation, not by its formula: from the delay on, the
    ring position of the next output to complete equals the number of Ready
    outputs emitted so far (the n-th Ready tick is d + n s) mod R, and
    that output is the one canonical slot 0 holds -- PyTorch's batch column of
    the same index over the consumed frames (Definition 1).  The
    emitted outputs are themselves PyTorch's full batch columns 0, 1, 2, ...
    in order, so the count is the batch column index."""
    rng = np.random.default_rng(4400 + seed)
    d = rand_desc(rng)
    B = 2
    H, Wd = d.in_hw
    W = rng.standard_normal(d.w_shape)
    sm = O.StepMachine(d, W, None, B)
    R, f, p, s = d.ring_slots, d.receptive_field, d.padding[0], d.stride[0]
    T = d.delay + 2 * max(R, 1) * s + 3
    frames = [rng.standard_normal((B, d.cin, H, Wd)) for _ in range(T)]
    d0 = O.Desc(**{**d.__dict__, "padding": (0,) + tuple(d.padding[1:])})
    emitted = 0
    for n, xt in enumerate(frames, start=1):
        y = sm.forward_step(xt)
        # the padded clip [p zeros | frames consumed so far | zeros for the future]
        L = p + n + (R + 1) * s + f
        clip = np.zeros((B, d.cin, L, H, Wd))
        for t in range(n):
            clip[:, :, p + t] = frames[t]
        ref = torch_conv(d0, W, None, clip, 0)
        if y is not None:
            tol = 1e-12 * max(1.0, np.abs(ref).max())
            np.testing.assert_allclose(y, ref[:, :, emitted], rtol=0, atol=tol)
            emitted += 1
        assert sm.n == n
        if R == 0 or n < d.delay:
            continue
        # observed: `emitted` outputs so far, so the next one to complete is column `emitted`
        assert sm.head == emitted % R, (n, sm.head, emitted, R)
        st = sm.state()
        np.testing.assert_allclose(st[0], ref[:, :, emitted], rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))
    assert emitted == len([t for t in range(T) if t >= d.delay and (t - d.delay) % s == 0])


# --------------------------------------------------------------- stack + bf16

def test_bf16_round_against_library_and_hand_values():
    # hand values: spacing of bf16 at 1 is 2^-7
    assert O.bf16_round([1 + 2 ** -8])[0] == 1.0                    # tie -> even
    assert O.bf16_round([1 + 3 * 2 ** -8])[0] == 1 + 2 ** -6        # tie -> even (up)
    assert O.bf16_round([1 + 2 ** -8 + 2 ** -20])[0] == 1 + 2 ** -7  # above tie -> up
    assert O.bf16_round([-3.0])[0] == -3.0
    rng = np.random.default_rng(5)
    v = rng.standard_normal(200000).astype(np.float32) * np.float32(10.0) ** rng.integers(-30, 30, 200000).astype(np.float32)
    v = v[np.isfinite(v)]
    lib_ref = torch.from_numpy(v).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(O.bf16_round(v.astype(np.float64)), lib_ref)


def test_stack_equals_composed_batch():
    """O6 vs the composition of textbook convs (torch f64) with ReLU between
    layers: stack step output at tick t == batch column t - d_NN (P:509 sums
    delays)."""
    rng = np.random.default_rng(8)
    descs = [O.Desc(2, 2, 3, (3, 3, 3), padding=(0, 1, 1), in_spatial=(5, 5)),
             O.Desc(2, 3, 3, (1, 3, 3), padding=(0, 1, 1), in_spatial=(5, 5)),
             O.Desc(2, 3, 2, (2, 1, 1), in_spatial=(5, 5))]
    Ws = [rng.standard_normal(d.w_shape) for d in descs]
    bs = [rng.standard_normal(d.cout) for d in descs]
    st = O.Stack(descs, Ws, bs, [1, 1, 0], [0, 0, 0], B=2)
    T = 10
    x = rng.standard_normal((2, 2, T, 5, 5))
    h = x
    for l, d in enumerate(descs):
        h = torch_conv(d, Ws[l], bs[l], h, 0)
        if l < 2:
            h = np.maximum(h, 0)
    d_nn = O.accumulate([d.receptive_field for d in descs], [0] * 3, [1] * 3)["d_nn"]
    assert d_nn == 3
    for t in range(T):
        y = st.forward_step(x[:, :, t])
        assert (y is None) == (t < d_nn)
        if y is not None:
            np.testing.assert_allclose(y, h[:, :, t - d_nn], rtol=0, atol=1e-12)


def test_stack_bf16_activations_exact_regime():
    """Declared bf16 activations (A16): with integer data every activation is
    an integer < 256, exactly representable, so rounding is the identity and
    the stack still equals the composed batch bit for bit."""
    rng = np.random.default_rng(12)
    descs = [O.Desc(2, 1, 2, (2, 3, 3), padding=(0, 1, 1), in_spatial=(4, 4)),
             O.Desc(2, 2, 1, (2, 1, 1), in_spatial=(4, 4))]
    Ws = [rng.integers(-1, 2, d.w_shape).astype(float) for d in descs]
    bs = [rng.integers(-1, 2, d.cout).astype(float) for d in descs]
    st = O.Stack(descs, Ws, bs, [1, 0], [1, 0], B=1)
    x = rng.integers(-2, 3, (1, 1, 8, 4, 4)).astype(float)
    h = np.maximum(torch_conv(descs[0], Ws[0], bs[0], x, 0), 0)
    assert np.abs(h).max() < 256
    h = torch_conv(descs[1], Ws[1], bs[1], h, 0)
    for t in range(8):
        y = st.forward_step(x[:, :, t])
        if t >= 2:
            assert np.array_equal(y, h[:, :, t - 2])


def test_step_history_is_the_last_padded_frames():
    """O3's raw history (the RAW layout's canonical state): after n steps it holds
    the padded frames n+p-(f-1) .. n+p-1, i.e. the real frames fed so far and
    zero frames for the start padding, oldest first."""
    rng = np.random.default_rng(7)
    d = O.Desc(2, 3, 4, (3, 3, 3), padding=(1, 1, 1), dilation=(2, 1, 1), in_spatial=(4, 5))
    f, p = d.receptive_field, d.padding[0]
    sm = O.StepMachine(d, rng.standard_normal(d.w_shape), None, 2)
    xs = [rng.standard_normal((2, 3, 4, 5)) for _ in range(7)]
    for n, x in enumerate(xs, start=1):
        sm.forward_step(x)
        h = sm.history()
        assert h.shape == (f - 1, 2, 3, 4, 5)
        for j in range(f - 1):
            q = n + p - (f - 1) + j                 # padded index of history slot j
            want = xs[q - p] if q >= p else np.zeros_like(x)
            assert np.array_equal(h[j], want)
    sm.forward_step(rng.standard_normal((2, 3, 4, 5)), update_state=False)
    assert np.array_equal(sm.history()[-1], xs[-1])   # update_state=False leaves it unchanged
