"""GPU parity of the depthwise step kernels (K2 k_step_dw_st, K3 k_step_dw_t)
against the fp64 oracle and the generic CUDA-core kernel, through the C ABI.

Sizes span several row bands per stream, several CTAs of items and a ragged
last band; the exact-integer regime is compared bit for bit.  K2/K3 add the
per-channel taps in the same order as k_step_direct, so the two CUDA paths
agree bitwise on any input.
"""
import numpy as np
import pytest
import torch

import oracle as O
from tests.helpers import assert_bf16_rounding_bound, make_pair, np_of, rel_err, set_opt, to_cl

pytestmark = pytest.mark.gpu


def dw(C, kernel, padding=(0, 0, 0), dilation=(1, 1, 1), in_spatial=(1, 1), rank=2):
    return O.Desc(rank, C, C, kernel, padding=padding, dilation=dilation, groups=C, in_spatial=in_spatial)


CASES = {
    # C3-a shaped: 3x3x3, spatial pad 1; 28x28 gives several bands, 9x13 a ragged one
    "st_c3a": dict(desc=dw(192, (3, 3, 3), (0, 1, 1), in_spatial=(28, 28)), B=2),
    "st_ragged": dict(desc=dw(24, (3, 3, 3), (0, 1, 1), in_spatial=(9, 13)), B=3),
    "st_pt1": dict(desc=dw(16, (3, 3, 3), (1, 1, 1), in_spatial=(6, 7)), B=2),
    "st_kt2_dil2": dict(desc=dw(16, (2, 3, 3), (0, 1, 1), dilation=(2, 1, 1), in_spatial=(5, 6)), B=2),
    "st_kt5": dict(desc=dw(32, (5, 3, 3), (2, 1, 1), in_spatial=(7, 8)), B=2),
    "st_kt1": dict(desc=dw(16, (1, 3, 3), (0, 1, 1), in_spatial=(6, 5)), B=2),
    "st_5x5_nopad": dict(desc=dw(16, (3, 5, 5), (0, 0, 0), in_spatial=(9, 8)), B=2),
    # enough (stream, row, segment) units that every K2s CTA wraps its stage ring
    # several times; W = 56 splits each row into two segments, C3-a shape at 24 streams
    "st_c3a_many": dict(desc=dw(192, (3, 3, 3), (0, 1, 1), in_spatial=(28, 28)), B=24),
    "st_w56_seg": dict(desc=dw(64, (3, 3, 3), (0, 1, 1), in_spatial=(10, 56)), B=24),
    # C3-b shaped: temporal only 5x1x1
    "t_c3b": dict(desc=dw(192, (5, 1, 1), in_spatial=(28, 28)), B=2),
    "t_kt9_dil2": dict(desc=dw(64, (9, 1, 1), dilation=(2, 1, 1), in_spatial=(25, 1), rank=1), B=3),
    "t_kt3_pt2": dict(desc=dw(8, (3, 1, 1), (2, 0, 0), in_spatial=(3, 3)), B=5),
    # temporal stride > 1 (Principle 5)
    "st_st2": dict(desc=O.Desc(2, 16, 16, (3, 3, 3), stride=(2, 1, 1), padding=(1, 1, 1), groups=16,
                               in_spatial=(7, 6)), B=2),
    "t_st3": dict(desc=O.Desc(2, 24, 24, (5, 1, 1), stride=(3, 1, 1), padding=(2, 0, 0), groups=24,
                              in_spatial=(4, 5)), B=2),
}


def _shape(d, B, T=None):
    H, Wd = d.in_hw
    return (B, d.cin) + ((T,) if T else ()) + ((H,) if d.spatial_rank >= 1 else ()) + \
        ((Wd,) if d.spatial_rank >= 2 else ())


def _run(case, integer=False, out_dtype=torch.float32, activation=None, seed=0, steps=None):
    d, B = CASES[case]["desc"], CASES[case]["B"]
    rng = np.random.default_rng(seed)
    if integer:
        W = rng.integers(-2, 3, d.w_shape).astype(np.float64)
        b = rng.integers(-2, 3, d.cout).astype(np.float64)
    else:
        W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
        b = rng.standard_normal(d.cout) * 0.1
    conv, sm, Wq, bq = make_pair(d, W, b, B, dtype=torch.bfloat16, out_dtype=out_dtype, kernel="depthwise",
                                 activation=activation)
    ref_conv, _, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, out_dtype=out_dtype, kernel="direct",
                                  activation=activation)
    assert conv.kernel_used == "depthwise", conv.kernel_name
    steps = steps or (d.receptive_field + 4 + 3 * (d.stride[0] - 1))
    ys, refs, yds = [], [], []
    for t in range(steps):
        x = rng.integers(-2, 3, _shape(d, B)).astype(np.float64) if integer else rng.standard_normal(_shape(d, B))
        xt = to_cl(x, torch.bfloat16)
        y = conv.forward_step(xt)
        yd = ref_conv.forward_step(xt)
        r = sm.forward_step(np_of(xt))
        assert (y is None) == (r is None) == (yd is None)
        assert (conv.n, conv.head) == (sm.n, sm.head)
        if y is not None:
            if activation == "relu":
                r = np.maximum(r, 0.0)
            ys.append(np_of(y)); refs.append(r.reshape(y.shape)); yds.append(np_of(yd))
    return conv, np.stack(ys), np.stack(refs), np.stack(yds)


@pytest.mark.parametrize("case", list(CASES))
def test_depthwise_vs_oracle_and_direct(case):
    conv, y, ref, yd = _run(case)
    assert rel_err(y, ref) <= 1e-4          # fp32 outputs of bf16 x bf16 products, fp32 sums
    assert np.array_equal(y, yd)            # same summation order as k_step_direct


ST_CASES = [c for c in CASES if c.startswith("st_")]


@pytest.mark.parametrize("case", ST_CASES)
def test_depthwise_stencil_dispatch_and_per_thread_variant(case):
    """Stencils dispatch to the segment-pipeline K2s (k_step_dw_seg: state rows
    and input-row pieces through a bulk-copy stage ring) by default; option
    dw_seg = 0 keeps the per-thread-load K2 (k_step_dw_st).  Both equal the
    fp64 oracle and k_step_direct bit for bit (same per-slice FMA order)."""
    conv, y, ref, yd = _run(case, steps=6)
    assert conv.kernel_name.startswith("k_step_dw_seg"), conv.kernel_name
    set_opt("dw_seg", 0)
    conv0, y0, ref0, yd0 = _run(case, steps=6)
    assert conv0.kernel_name.startswith("k_step_dw_st"), conv0.kernel_name
    assert np.array_equal(y0, y) and np.array_equal(y0, yd0)


@pytest.mark.parametrize("case", list(CASES))
def test_depthwise_exact_integer_bitwise(case):
    _, y, ref, yd = _run(case, integer=True)
    assert np.array_equal(y, ref)
    assert np.array_equal(y, yd)


@pytest.mark.parametrize("case", ["st_c3a", "t_c3b"])
def test_depthwise_bf16_output_and_relu(case):
    # A16: RNE of the outputs alone can reach ~2e-2 RMS (more after ReLU halves
    # the RMS), so bf16 outputs are compared with the oracle rounded the same way
    _, y, ref, yd = _run(case, out_dtype=torch.bfloat16, activation="relu")
    assert_bf16_rounding_bound(y, ref)
    assert np.array_equal(y, yd)
    assert (y >= 0).all()


@pytest.mark.parametrize("case", ["st_ragged", "t_kt9_dil2", "st_pt1", "st_st2", "t_st3"])
def test_depthwise_state_steps_and_purity(case):
    """co_state_get vs oracle O5 (channels-last physical ring -> canonical
    layout), get->set round trip, update_state=False purity, forward_steps =
    bitwise fold of forward_step, pad_end outputs vs batch forward (O2)."""
    from paper_2204_03418_b200 import channels_last
    d, B = CASES[case]["desc"], CASES[case]["B"]
    rng = np.random.default_rng(5)
    W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    b = rng.standard_normal(d.cout) * 0.1
    conv, sm, Wq, bq = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="depthwise")
    T = d.receptive_field + 3
    frames = [to_cl(rng.standard_normal(_shape(d, B)), torch.bfloat16) for _ in range(T)]
    for x in frames:
        conv.forward_step(x)
        sm.forward_step(np_of(x))
    st, meta = conv.state_dict_stream()
    ref = sm.state()
    So = d.out_spatial
    got = np_of(st).reshape((ref.shape[0], B) + tuple(So) + (d.cout,))
    got = np.moveaxis(got, -1, 2).reshape(ref.shape)
    assert rel_err(got, ref) <= 1e-4
    assert (meta.n, meta.head) == (sm.n, sm.head)
    # round trip on a fresh handle, then both continue identically
    conv2, _, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="depthwise")
    conv2.load_state_stream(st, meta)
    st2, _ = conv2.state_dict_stream()
    assert torch.equal(st, st2)
    probe = to_cl(rng.standard_normal(_shape(d, B)), torch.bfloat16)
    y_peek = conv.forward_step(probe, update_state=False)
    st1, m1 = conv.state_dict_stream()
    assert torch.equal(st, st1) and m1.n == meta.n
    y1, y2 = conv.forward_step(probe), conv2.forward_step(probe)
    assert (y_peek is None) == (y1 is None) == (y2 is None)   # Empty ticks under temporal stride
    assert y1 is None or (torch.equal(y_peek, y1) and torch.equal(y1, y2))
    # forward_steps (with pad_end) == fold of forward_step, and == batch forward
    clip = channels_last(torch.stack(frames, dim=2))
    c3, _, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="depthwise")
    c4, _, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="depthwise")
    ys, mask = c3.forward_steps(clip, pad_end=True)
    fold = [y for y in (c4.forward_step(x) for x in frames) if y is not None]
    fold += [y for y in (c4.forward_pad_step() for _ in range(d.padding[0])) if y is not None]
    assert ys.shape[2] == len(fold) == int(mask.sum())
    for i, f in enumerate(fold):
        assert torch.equal(ys[:, :, i], f)
    ref_b = O.forward(d, Wq, bq, np_of(clip))
    assert rel_err(np_of(ys), ref_b) <= 1e-4


def test_c3_chain_stack_vs_oracle():
    """C3-shaped chain (3x3x3 depthwise -> 5x1x1 depthwise), bf16 inter-layer
    activation, through the stack driver: delay 2 + 4 = 6 (Principle 6)."""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    cfg = synth.config(3, n_streams=3, in_spatial=(11, 12))
    params = synth.params(cfg)
    descs = [O.Desc(2, L.cin, L.cout, L.kernel, L.stride, L.padding, L.dilation, L.groups, cfg.in_spatial)
             for L in cfg.layers]
    convs, Ws, bs = [], [], []
    for l, (L, (W, b)) in enumerate(zip(cfg.layers, params)):
        last = l == len(cfg.layers) - 1
        c = co.Conv(L.cin, L.cout, L.kernel, weight=W.cuda(), bias=b.cuda(), stride=L.stride, padding=L.padding,
                    dilation=L.dilation, groups=L.groups, spatial_rank=2, in_spatial=cfg.in_spatial,
                    n_streams=cfg.n_streams, dtype=torch.bfloat16,
                    out_dtype=torch.float32 if last else torch.bfloat16)
        assert c.kernel_used == "depthwise"
        convs.append(c); Ws.append(W.double().numpy()); bs.append(b.double().numpy())
    stack = co.Stack(convs)
    assert stack.delay == 6
    ost = O.Stack(descs, Ws, bs, [0, 0], [1, 0], cfg.n_streams)
    ys, refs = [], []
    for t in range(12):
        x = synth.frame(cfg, t)
        y = stack.forward_step(x)
        r = ost.forward_step(np_of(x))
        assert (y is None) == (r is None) == (t < 6)
        if y is not None:
            ys.append(np_of(y)); refs.append(r)
    assert rel_err(np.stack(ys), np.stack(refs).reshape(np.stack(ys).shape)) <= 2e-2
