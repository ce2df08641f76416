"""GPU parity of the RAW-input-ring state layout (co_state_layout RAW, SURVEY
§8f f1): the state is the last f frames, a Ready step contracts the whole window
(Definition 1) and a non-Ready step only stores its frame.  Checked
against the fp64 oracle on random small shapes (groups, dilation, temporal and
spatial stride, padding), against the partial-sum layout, and for the state
contract: co_state_get == the oracle's raw history (O3), get->set round trip,
update_state=0 purity, forward_steps fold and pad_end == batch forward."""
import numpy as np
import pytest
import torch

import oracle as O
from tests.helpers import make_pair, np_of, rand_desc, rel_err, to_cl

pytestmark = pytest.mark.gpu


def _shape(d, B, T=None):
    H, W = d.in_hw
    return (B, d.cin) + ((T,) if T else ()) + ((H,) if d.spatial_rank >= 1 else ()) + \
        ((W,) if d.spatial_rank >= 2 else ())


def _canon_to_oracle(st, d, B):
    """(f-1, B, *S, Cin) -> (f-1, B, Cin, S1, S2)"""
    H, W = d.in_hw
    a = np_of(st).reshape((st.shape[0], B, H, W, d.cin))
    return np.moveaxis(a, -1, 2)


@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("kernel", ["direct", "auto"])
def test_raw_random_shapes_vs_oracle(seed, kernel):
    rng = np.random.default_rng(1000 + seed)
    d = rand_desc(rng)
    B = int(rng.integers(1, 4))
    dt = torch.bfloat16 if seed % 2 else torch.float32
    W = rng.standard_normal(d.w_shape)
    b = rng.standard_normal(d.cout)
    conv, sm, _, _ = make_pair(d, W, b, B, dtype=dt, kernel=kernel, state_layout="raw")
    ref_ps, _, _, _ = make_pair(d, W, b, B, dtype=dt, kernel="direct")
    ys, refs, yps = [], [], []
    for t in range(14):
        xt = to_cl(rng.standard_normal(_shape(d, B)), dt)
        y = conv.forward_step(xt)
        yp = ref_ps.forward_step(xt)
        r = sm.forward_step(np_of(xt))
        assert (y is None) == (r is None) == (yp is None)
        assert (conv.n, conv.head) == (sm.n, sm.head)
        if y is not None:
            ys.append(np_of(y)); refs.append(r.reshape(y.shape)); yps.append(np_of(yp))
    if ys:
        assert rel_err(np.stack(ys), np.stack(refs)) <= 1e-4
        assert rel_err(np.stack(ys), np.stack(yps)) <= 1e-4          # same outputs as the partial-sum ring
    st, meta = conv.state_dict_stream()
    if d.receptive_field > 1:
        assert np.array_equal(_canon_to_oracle(st, d, B), sm.history())   # the stored frames, bit for bit
    assert meta.state_layout == 1 and meta.ring_slots == d.receptive_field - 1


@pytest.mark.parametrize("seed", range(6))
def test_raw_state_roundtrip_purity_and_folds(seed):
    from paper_2204_03418_b200 import channels_last
    rng = np.random.default_rng(2000 + seed)
    d = rand_desc(rng)
    B = 2
    W, b = rng.standard_normal(d.w_shape), rng.standard_normal(d.cout)
    conv, sm, Wq, bq = make_pair(d, W, b, B, state_layout="raw")
    frames = [rng.standard_normal(_shape(d, B)) for _ in range(9)]
    for x in frames[:6]:
        conv.forward_step(to_cl(x, torch.float32)); sm.forward_step(x)
    st, meta = conv.state_dict_stream()
    # an oracle history loaded into a fresh handle continues identically
    conv2, _, _, _ = make_pair(d, W, b, B, state_layout="raw")
    hist = sm.history()
    if hist.shape[0]:
        conv2.load_state_stream(torch.from_numpy(np.moveaxis(hist, 2, -1).copy()).float().cuda(), meta)
    else:
        conv2.load_state_stream(st, meta)
    probe = to_cl(rng.standard_normal(_shape(d, B)), torch.float32)
    y_peek = conv.forward_step(probe, update_state=False)
    st1, m1 = conv.state_dict_stream()
    assert torch.equal(st, st1) and m1.n == meta.n                  # state untouched
    for x in [probe.cpu().numpy()] + frames[6:]:
        xt = x if isinstance(x, torch.Tensor) else to_cl(x, torch.float32)
        y1, y2 = conv.forward_step(xt), conv2.forward_step(xt)
        r = sm.forward_step(np_of(xt))
        assert (y1 is None) == (y2 is None) == (r is None)
        if r is not None:
            assert rel_err(np_of(y2), r) <= 1e-4 and torch.equal(y1, y2)
    # get -> set round trip is bitwise
    st2, meta2 = conv.state_dict_stream()
    conv2.load_state_stream(st2, meta2)
    st3, _ = conv2.state_dict_stream()
    assert torch.equal(st2, st3)
    # forward_steps with pad_end == fold of forward_step == batch forward
    T = len(frames)
    a, _, _, _ = make_pair(d, W, b, B, state_layout="raw")
    c, _, _, _ = make_pair(d, W, b, B, state_layout="raw")
    clip = np.stack(frames, axis=2)
    ys, mask = a.forward_steps(to_cl(clip, torch.float32), pad_end=True)
    fold = [y for y in (c.forward_step(to_cl(x, torch.float32)) for x in frames) if y is not None]
    fold += [y for y in (c.forward_pad_step() for _ in range(d.padding[0])) if y is not None]
    assert ys.shape[2] == len(fold) == int(mask.sum())
    for i, f in enumerate(fold):
        assert torch.equal(ys[:, :, i], f)
    if d.out_len(T) >= 1:
        assert rel_err(np_of(ys), O.forward(d, Wq, bq, clip)) <= 1e-4


RAW_DENSE = {
    "c2like": dict(desc=O.Desc(2, 64, 64, (3, 3, 3), padding=(0, 1, 1), in_spatial=(13, 24)), B=3),
    "s2": dict(desc=O.Desc(2, 128, 128, (3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), in_spatial=(12, 20)), B=2),
    "c5like": dict(desc=O.Desc(1, 256, 64, (9, 1), dilation=(2, 1), in_spatial=(25, 1)), B=5),
    "flat_ragged": dict(desc=O.Desc(1, 32, 128, (5, 1), padding=(2, 0), in_spatial=(25, 1)), B=7),
    "flat_conv1d": dict(desc=O.Desc(0, 64, 64, (3,), stride=(2,)), B=300),
    "st2_pt1": dict(desc=O.Desc(2, 32, 32, (3, 3, 3), stride=(2, 1, 1), padding=(1, 1, 1), in_spatial=(6, 7)), B=2),
    "kt5_dil2": dict(desc=O.Desc(2, 16, 32, (5, 3, 3), padding=(2, 1, 1), dilation=(2, 1, 1), in_spatial=(7, 8)), B=2),
}


@pytest.mark.parametrize("case", list(RAW_DENSE))
@pytest.mark.parametrize("integer", [False, True])
def test_raw_dense_tc_vs_oracle(case, integer):
    """The tensor-core RAW path: temporal taps folded into K of one K-pipelined
    contraction per Ready step; bitwise in the exact-integer regime."""
    d, B = RAW_DENSE[case]["desc"], RAW_DENSE[case]["B"]
    rng = np.random.default_rng(3000)
    if integer:
        W = rng.integers(-2, 3, d.w_shape).astype(np.float64)
        b = rng.integers(-2, 3, d.cout).astype(np.float64)
    else:
        W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
        b = rng.standard_normal(d.cout) * 0.1
    conv, sm, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="dense_tc", state_layout="raw")
    assert conv.kernel_used == "dense_tc" and "kloop" in conv.kernel_name, conv.kernel_name
    ys, refs = [], []
    for t in range(d.receptive_field + 5):
        x = rng.integers(-2, 3, _shape(d, B)).astype(np.float64) if integer else rng.standard_normal(_shape(d, B))
        xt = to_cl(x, torch.bfloat16)
        y = conv.forward_step(xt)
        r = sm.forward_step(np_of(xt))
        assert (y is None) == (r is None)
        if y is not None:
            ys.append(np_of(y)); refs.append(r.reshape(y.shape))
    y, ref = np.stack(ys), np.stack(refs)
    if integer:
        assert np.array_equal(y, ref)
    else:
        assert rel_err(y, ref) <= 1e-4
    st, _ = conv.state_dict_stream()
    assert np.array_equal(_canon_to_oracle(st, d, B), sm.history())


RAW_DW = {
    "c3a": dict(desc=O.Desc(2, 192, 192, (3, 3, 3), padding=(0, 1, 1), groups=192, in_spatial=(28, 28)), B=2),
    "c3b": dict(desc=O.Desc(2, 192, 192, (5, 1, 1), groups=192, in_spatial=(28, 28)), B=2),
    "ragged_st2": dict(desc=O.Desc(2, 24, 24, (3, 3, 3), stride=(2, 1, 1), padding=(1, 1, 1), groups=24,
                                   in_spatial=(9, 13)), B=3),
    "t_dil2": dict(desc=O.Desc(1, 64, 64, (9, 1), dilation=(2, 1), groups=64, in_spatial=(25, 1)), B=3),
    "t_st2_pad": dict(desc=O.Desc(2, 24, 24, (4, 1, 1), stride=(2, 1, 1), padding=(2, 0, 0), groups=24,
                                  in_spatial=(7, 5)), B=5),
    "s_valid": dict(desc=O.Desc(2, 16, 16, (2, 3, 3), groups=16, in_spatial=(9, 10)), B=3),      # unpadded stencil
    "s_many": dict(desc=O.Desc(2, 48, 48, (3, 3, 3), padding=(0, 1, 1), groups=48, in_spatial=(11, 29)), B=41),
    "s_5x5": dict(desc=O.Desc(2, 32, 32, (3, 5, 5), padding=(2, 2, 2), groups=32, in_spatial=(12, 17)), B=4),
    "t_many": dict(desc=O.Desc(2, 40, 40, (3, 1, 1), groups=40, in_spatial=(30, 33)), B=37),   # several grid waves, ragged tail
}


@pytest.mark.parametrize("case", list(RAW_DW))
def test_raw_depthwise_vs_oracle(case):
    d, B = RAW_DW[case]["desc"], RAW_DW[case]["B"]
    rng = np.random.default_rng(4000)
    W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    b = rng.standard_normal(d.cout) * 0.1
    conv, sm, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="depthwise", state_layout="raw")
    temporal = d.kernel[1:] == (1,) * (len(d.kernel) - 1)
    # temporal-only layers: the fused-store streaming kernel (the Ready step reads x itself)
    # "same"-padded stencils: rolling row sets over the window's frames (frame store fused too)
    same = all(2 * pd == k - 1 for pd, k in zip(list(d.padding)[1:], list(d.kernel)[1:]))
    assert ("dw_traw" if temporal else "dw_rowraw" if same else "dw_raw") in conv.kernel_name, conv.kernel_name
    ys, refs = [], []
    for t in range(d.receptive_field + 7):
        xt = to_cl(rng.standard_normal(_shape(d, B)), torch.bfloat16)
        if t == d.receptive_field + 2:                     # a probe: Ready or not, the ring must not change
            yp = conv.forward_step(xt, update_state=False)
            rp = sm.forward_step(np_of(xt), update_state=False)
            assert (yp is None) == (rp is None)
            if yp is not None:
                ys.append(np_of(yp)); refs.append(rp.reshape(yp.shape))
            xt = to_cl(rng.standard_normal(_shape(d, B)), torch.bfloat16)
        y = conv.forward_step(xt)
        r = sm.forward_step(np_of(xt))
        assert (y is None) == (r is None)
        if y is not None:
            ys.append(np_of(y)); refs.append(r.reshape(y.shape))
    assert rel_err(np.stack(ys), np.stack(refs)) <= 1e-4
    st, _ = conv.state_dict_stream()
    assert np.array_equal(_canon_to_oracle(st, d, B), sm.history())


# Small-Cin stems over the RAW ring (k_stem_raw.cu): the W-im2col image built in
# shared memory per (tile, temporal tap), weights resident, one window
# contraction per Ready step.  Shapes span several 128-row tiles with ragged
# last tiles, stride 1 / 2, odd padding (mid-word windows), a zero K group
# (kw Cin = 21 -> Kp 32) and none (kw Cin = 9, 16), temporal stride and
# dilation, temporal padding.
RAW_STEM = {
    "c4stem": dict(desc=O.Desc(2, 3, 64, (5, 7, 7), stride=(1, 2, 2), padding=(0, 3, 3), in_spatial=(36, 40)), B=3),
    "c4stem_wide": dict(desc=O.Desc(2, 3, 64, (5, 7, 7), stride=(1, 2, 2), padding=(0, 3, 3), in_spatial=(30, 112)),
                        B=2),
    "s1_k3": dict(desc=O.Desc(2, 3, 32, (3, 3, 3), padding=(1, 1, 1), in_spatial=(9, 16)), B=2),
    "cin4_st2_dil2": dict(desc=O.Desc(2, 4, 32, (3, 5, 5), stride=(2, 1, 2), padding=(1, 2, 2),
                                      dilation=(2, 1, 1), in_spatial=(11, 14)), B=2),
    "cin1_k2": dict(desc=O.Desc(2, 1, 64, (2, 3, 3), padding=(0, 1, 1), in_spatial=(10, 24)), B=4),
    "cin2_ph0": dict(desc=O.Desc(2, 2, 32, (4, 3, 4), stride=(1, 2, 1), padding=(0, 0, 0), in_spatial=(13, 24)), B=2),
}


@pytest.mark.parametrize("case", list(RAW_STEM))
@pytest.mark.parametrize("integer", [False, True])
def test_raw_stem_tc_vs_oracle(case, integer):
    d, B = RAW_STEM[case]["desc"], RAW_STEM[case]["B"]
    rng = np.random.default_rng(3100)
    if integer:
        W = rng.integers(-2, 3, d.w_shape).astype(np.float64)
        b = rng.integers(-2, 3, d.cout).astype(np.float64)
    else:
        W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
        b = rng.standard_normal(d.cout) * 0.1
    for out_dtype in (torch.float32, torch.bfloat16):
        conv, sm, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, out_dtype=out_dtype, kernel="dense_tc",
                                   state_layout="raw", activation="relu" if out_dtype == torch.bfloat16 else None)
        assert conv.kernel_used == "dense_tc" and "stem_raw" in conv.kernel_name, conv.kernel_name
        ys, refs = [], []
        for t in range(d.receptive_field + 2 * d.stride[0] + 3):
            x = rng.integers(-2, 3, _shape(d, B)).astype(np.float64) if integer else rng.standard_normal(_shape(d, B))
            xt = to_cl(x, torch.bfloat16)
            y = conv.forward_step(xt)
            r = sm.forward_step(np_of(xt))
            assert (y is None) == (r is None)
            assert (conv.n, conv.head) == (sm.n, sm.head)
            if y is not None:
                ys.append(np_of(y)); refs.append(r.reshape(y.shape))
        assert ys
        y, ref = np.stack(ys), np.stack(refs)
        if out_dtype == torch.bfloat16:
            ref = np.maximum(ref, 0.0)
            if integer:
                # integer sums are exact in fp32: the bf16 output is RNE of the exact value
                assert np.array_equal(y, torch.from_numpy(ref).to(torch.bfloat16).double().numpy())
            else:
                from tests.helpers import assert_bf16_rounding_bound
                assert_bf16_rounding_bound(y, ref)
        elif integer:
            assert np.array_equal(y, ref)
        else:
            assert rel_err(y, ref) <= 1e-4
        st, _ = conv.state_dict_stream()
        assert np.array_equal(_canon_to_oracle(st, d, B), sm.history())


def test_raw_stem_auto_layout_and_zero_frames():
    """CO_STATE_AUTO picks the RAW ring for the C4 stem shape (0.45 MB against
    6.4 MB of partial sums per stream-step); pad steps (zero frames) and
    update_state = 0 probes behave as on the oracle."""
    d = O.Desc(2, 3, 64, (5, 7, 7), stride=(1, 2, 2), padding=(2, 3, 3), in_spatial=(24, 32))
    B = 2
    rng = np.random.default_rng(3200)
    W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    b = rng.standard_normal(d.cout) * 0.1
    conv, sm, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="auto", state_layout="auto")
    assert "stem_raw" in conv.kernel_name, conv.kernel_name
    ys, refs = [], []
    for t in range(9):
        xt = to_cl(rng.standard_normal(_shape(d, B)), torch.bfloat16)
        if t == 6:   # a probe: the output of this frame without advancing the state
            yp = conv.forward_step(xt, update_state=False)
            rp = sm.forward_step(np_of(xt), update_state=False)
            assert (yp is None) == (rp is None)
            if yp is not None:
                assert rel_err(np_of(yp), rp.reshape(yp.shape)) <= 1e-4
        y = conv.forward_step(xt)
        r = sm.forward_step(np_of(xt))
        assert (y is None) == (r is None)
        if y is not None:
            ys.append(np_of(y)); refs.append(r.reshape(y.shape))
    for _ in range(d.padding[0]):
        y = conv.forward_pad_step()
        r = sm.forward_step(None)
        assert (y is None) == (r is None)
        if y is not None:
            ys.append(np_of(y)); refs.append(r.reshape(y.shape))
    assert rel_err(np.stack(ys), np.stack(refs)) <= 1e-4


def _stem_desc(rng):
    """A random shape k_step_stem_raw covers: Cin <= 8 / sw, kw (8 / sw) <= 32,
    spatial strides <= 2, 16-B raw rows, Cout 32 or 64."""
    sw = int(rng.integers(1, 3))
    cp = 8 // sw
    cin = int(rng.integers(1, cp + 1))
    kw = int(rng.integers(1, 32 // cp + 1))
    kh = int(rng.integers(1, 8))
    sh = int(rng.integers(1, 3))
    kt = int(rng.integers(1, 6))
    dil = int(rng.integers(1, 3))
    f = dil * (kt - 1) + 1
    pt = int(rng.integers(0, f))
    st = int(rng.integers(1, 3))
    ph, pw = int(rng.integers(0, kh // 2 + 1)), int(rng.integers(0, kw // 2 + 1))
    unit = 8 // np.gcd(8, cin)                       # W Cin * 2 bytes a multiple of 16
    W = unit * int(rng.integers(max(1, -(-kw // unit)), 48 // unit + 2))
    H = int(rng.integers(max(kh - 2 * ph, 1), 20))
    cout = int(rng.choice([32, 64]))
    return O.Desc(2, cin, cout, (kt, kh, kw), stride=(st, sh, sw), padding=(pt, ph, pw), dilation=(dil, 1, 1),
                  in_spatial=(H, W))


@pytest.mark.parametrize("seed", range(16))
def test_raw_stem_random_shapes_vs_oracle(seed):
    """Random small-Cin shapes on the RAW-ring stem kernel (strides, paddings,
    odd kernels, temporal stride / dilation / padding, ragged tiles) against the
    fp64 oracle over the delay and several Ready ticks; the ring is the oracle's
    history bit for bit."""
    rng = np.random.default_rng(5000 + seed)
    d = _stem_desc(rng)
    while not d.valid():
        d = _stem_desc(rng)
    B = int(rng.integers(1, 4))
    W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    b = rng.standard_normal(d.cout) * 0.1
    conv, sm, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="dense_tc", state_layout="raw")
    assert "stem_raw" in conv.kernel_name, (conv.kernel_name, d)
    ys, refs = [], []
    for t in range(d.receptive_field + 3 * d.stride[0] + 2):
        xt = to_cl(rng.standard_normal(_shape(d, B)), torch.bfloat16)
        y = conv.forward_step(xt)
        r = sm.forward_step(np_of(xt))
        assert (y is None) == (r is None)
        assert (conv.n, conv.head) == (sm.n, sm.head)
        if y is not None:
            ys.append(np_of(y)); refs.append(r.reshape(y.shape))
    if ys:
        assert rel_err(np.stack(ys), np.stack(refs)) <= 1e-4, d
    st, _ = conv.state_dict_stream()
    if d.receptive_field > 1:
        assert np.array_equal(_canon_to_oracle(st, d, B), sm.history())


def test_raw_stem_state_probe_fold_and_batch():
    """The RAW stem handle's contract beyond single steps: a get -> set round
    trip continues bitwise, an update_state = False probe leaves the ring
    untouched, forward_steps equals the per-step fold bit for bit, and the
    batch forward matches the step outputs."""
    import paper_2204_03418_b200 as co
    d = O.Desc(2, 3, 64, (5, 7, 7), stride=(1, 2, 2), padding=(2, 3, 3), in_spatial=(26, 40))
    B = 2
    rng = np.random.default_rng(5100)
    W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    b = rng.standard_normal(d.cout) * 0.1
    a, sm, Wq, bq = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="dense_tc", state_layout="raw")
    c, _, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="dense_tc", state_layout="raw")
    assert "stem_raw" in a.kernel_name
    frames = [to_cl(rng.standard_normal(_shape(d, B)), torch.bfloat16) for _ in range(12)]
    for x in frames[:6]:
        a.forward_step(x); c.forward_step(x)
    st, meta = a.state_dict_stream()
    # probe: same output as a real step, state unchanged
    yp = a.forward_step(frames[6], update_state=False)
    st2, _ = a.state_dict_stream()
    assert torch.equal(st, st2)
    # round trip into a fresh handle continues bit for bit
    e, _, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="dense_tc", state_layout="raw")
    e.load_state_stream(st, meta)
    for x in frames[6:]:
        ya, ye = a.forward_step(x), e.forward_step(x)
        assert (ya is None) == (ye is None)
        if ya is not None:
            assert torch.equal(ya, ye)
    if yp is not None:
        ya6 = c.forward_step(frames[6])
        assert torch.equal(yp, ya6)
    # forward_steps over a clip == the per-step fold (same kernel, same order)
    f1, _, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="dense_tc", state_layout="raw")
    f2, _, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="dense_tc", state_layout="raw")
    clip = torch.stack(frames, dim=2)
    ys, mask = f1.forward_steps(co.channels_last(clip), pad_end=True)
    fold = [y for y in (f2.forward_step(x) for x in frames) if y is not None]
    fold += [y for y in (f2.forward_pad_step() for _ in range(d.padding[0])) if y is not None]
    assert ys.shape[2] == len(fold) == int(mask.sum())
    for i, y in enumerate(fold):
        assert torch.equal(ys[:, :, i], y)
    # batch mode (the generic kernel) against the oracle's batch forward
    clip_np = np.stack([np_of(x) for x in frames], axis=2)
    yb = f1.forward(co.channels_last(clip))
    assert rel_err(np_of(yb), O.forward(d, Wq, bq, clip_np)) <= 1e-4
