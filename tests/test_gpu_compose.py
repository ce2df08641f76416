"""GPU parity of Delay and the Residual composite (PAPER.md
P:301-326, Listing 3) through the C ABI,
against the fp64 oracle (oracle/compose.py over the conv oracle): readiness
(Principle 7), identity-branch alignment (equal padding and centered), ReLU
after the add, bf16 inter-layer activations, batch mode, update_state = 0
purity and clean state.  Tolerance: fp32 outputs within 1e-4 of the RMS; a
zero-weight body is exact (the output is the delayed input)."""
import numpy as np
import pytest
import torch

import oracle as O
from oracle import compose as OC
from tests.helpers import np_of, rel_err, to_cl

pytestmark = pytest.mark.gpu


def _bf16(a):
    return torch.from_numpy(np.asarray(a, np.float64)).to(torch.bfloat16).double().numpy()


def _layers(specs, B, H, W, rng, zero=False, last_fp32=True, kernel="auto"):
    """specs: (cin, cout, kernel, padding, groups, relu).  Returns CUDA convs and
    the oracle's (descs, Ws, bs, relu, round_bf16) with identical bf16 weights."""
    import paper_2204_03418_b200 as co
    convs, descs, Ws, bs, relu, rnd = [], [], [], [], [], []
    for l, (cin, cout, k, p, g, r) in enumerate(specs):
        last = l == len(specs) - 1
        d = O.Desc(2, cin, cout, k, padding=p, groups=g, in_spatial=(H, W))
        Wn = np.zeros(d.w_shape) if zero else rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
        bn = np.zeros(cout) if zero else rng.standard_normal(cout) * 0.1
        Wq, bq = _bf16(Wn), torch.from_numpy(bn).float().double().numpy()
        od = torch.float32 if (last and last_fp32) else torch.bfloat16
        convs.append(co.Conv(cin, cout, k, weight=torch.from_numpy(Wq).to(torch.bfloat16).cuda(),
                             bias=torch.from_numpy(bq).float().cuda(), padding=p, groups=g, in_spatial=(H, W),
                             n_streams=B, out_dtype=od, activation="relu" if r else None, kernel=kernel))
        descs.append(d); Ws.append(Wq); bs.append(bq); relu.append(int(r)); rnd.append(int(od == torch.bfloat16))
    return convs, (descs, Ws, bs, relu, rnd)


BODIES = {
    # one dense conv, equal padding (Fig. 4): d = d_skip = 1
    "conv_eq": ([(32, 32, (3, 3, 3), (1, 1, 1), 1, False)], False),
    # one dense conv, no temporal padding, centered (Fig. 5): d = 2, d_skip = 1
    "conv_center": ([(32, 32, (3, 3, 3), (0, 1, 1), 1, False)], True),
    # X3D-style bottleneck: 1x1 expand + ReLU, depthwise 3x3x3 + ReLU, 1x1 project
    "x3d_bottleneck": ([(32, 64, (1, 1, 1), (0, 0, 0), 1, True), (64, 64, (3, 3, 3), (1, 1, 1), 64, True),
                        (64, 32, (1, 1, 1), (0, 0, 0), 1, False)], False),
    # two temporal convs, centered: f = 5, d = 4, d_skip = 2
    "two_center": ([(16, 16, (3, 3, 3), (0, 1, 1), 1, True), (16, 16, (3, 3, 3), (0, 1, 1), 1, False)], True),
    # centered with some temporal padding: f = 5, p = 1, d = 3, d_skip = 2, batch crop 1
    "conv_center_padded": ([(32, 32, (5, 3, 3), (1, 1, 1), 1, False)], True),
    # two layers, f_acc = 5, p_acc = 1 (padding in the first layer only)
    "two_center_padded": ([(16, 16, (3, 3, 3), (1, 1, 1), 1, True), (16, 16, (3, 3, 3), (0, 1, 1), 1, False)], True),
}


@pytest.mark.parametrize("relu_out", [False, True])
@pytest.mark.parametrize("name", list(BODIES))
def test_residual_step_vs_oracle(name, relu_out):
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(sum(map(ord, name)))
    specs, shrink = BODIES[name]
    B, H, W = 3, 6, 7
    convs, (descs, Ws, bs, relu, rnd) = _layers(specs, B, H, W, rng)
    res = co.Residual(convs, shrink=shrink, activation="relu" if relu_out else None)
    ref = OC.ResidualStep(descs, Ws, bs, relu, rnd, B, shrink=shrink, relu_out=relu_out)
    assert res.delays() == (ref.delay, ref.d_skip)
    C = specs[0][0]
    for t in range(ref.delay + 6):
        x = _bf16(rng.standard_normal((B, C, H, W)))
        y = res.forward_step(to_cl(x, torch.bfloat16))
        r = ref.forward_step(x)
        assert (y is None) == (r is None), t
        if y is not None:
            assert rel_err(np_of(y), r) <= 1e-4, t


@pytest.mark.parametrize("name", ["conv_eq", "conv_center", "two_center", "conv_center_padded", "two_center_padded"])
def test_residual_forward_vs_oracle(name):
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(5)
    specs, shrink = BODIES[name]
    B, H, W, T = 2, 5, 6, 9
    convs, (descs, Ws, bs, relu, rnd) = _layers(specs, B, H, W, rng)
    res = co.Residual(convs, shrink=shrink, activation="relu")
    x = _bf16(rng.standard_normal((B, specs[0][0], T, H, W)))
    y = res.forward(to_cl(x, torch.bfloat16))
    ref = OC.residual_forward(descs, Ws, bs, relu, x, shrink=shrink, relu_out=True, round_bf16=rnd)
    assert y.shape[2] == ref.shape[2]
    assert rel_err(np_of(y), ref) <= 1e-4


@pytest.mark.parametrize("shrink", [False, True])
def test_zero_body_emits_the_aligned_input_exactly(shrink):
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(6)
    p = 0 if shrink else 2
    specs = [(16, 16, (5, 3, 3), (p, 1, 1), 1, False)]
    B, H, W = 2, 4, 5
    convs, _ = _layers(specs, B, H, W, rng, zero=True)
    res = co.Residual(convs, shrink=shrink)
    d, k = res.delays()
    assert (d, k) == ((4, 2) if shrink else (2, 2))
    frames = [_bf16(rng.standard_normal((B, 16, H, W))) for _ in range(10)]
    for n, x in enumerate(frames):
        y = res.forward_step(to_cl(x, torch.bfloat16))
        assert (y is None) == (n < d)
        if y is not None:
            np.testing.assert_array_equal(np_of(y), frames[n - k])


def test_residual_update_state_false_and_clean():
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(7)
    specs, shrink = BODIES["two_center"]
    B, H, W = 2, 5, 5
    convs, (descs, Ws, bs, relu, rnd) = _layers(specs, B, H, W, rng)
    res = co.Residual(convs, shrink=shrink)
    ref = OC.ResidualStep(descs, Ws, bs, relu, rnd, B, shrink=shrink)
    frames = [_bf16(rng.standard_normal((B, 16, H, W))) for _ in range(12)]
    for t, x in enumerate(frames):
        if t >= 5:                               # a probe must not disturb the stream
            probe = _bf16(rng.standard_normal((B, 16, H, W)))
            yp = res.forward_step(to_cl(probe, torch.bfloat16), update_state=False)
            rp = ref.forward_step(probe, update_state=False)
            assert rel_err(np_of(yp), rp) <= 1e-4
        y = res.forward_step(to_cl(x, torch.bfloat16))
        r = ref.forward_step(x)
        assert (y is None) == (r is None)
        if y is not None:
            assert rel_err(np_of(y), r) <= 1e-4
    res.clean_state(); ref.clean_state()
    for t, x in enumerate(frames[:7]):
        y = res.forward_step(to_cl(x, torch.bfloat16))
        r = ref.forward_step(x)
        assert (y is None) == (r is None)
        if y is not None:
            assert rel_err(np_of(y), r) <= 1e-4


@pytest.mark.parametrize("d", [0, 1, 3])
def test_delay_vs_oracle(d):
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(8 + d)
    B, C, H, W = 3, 8, 4, 5
    dl = co.Delay(d, C, in_spatial=(H, W), n_streams=B)
    assert dl.delay == d and dl.kernel_used == "copy"
    ref = OC.DelayStep(d)
    frames = [_bf16(rng.standard_normal((B, C, H, W))) for _ in range(d + 5)]
    for t, x in enumerate(frames):
        if t == 2:
            yp = dl.forward_step(to_cl(frames[0], torch.bfloat16), update_state=False)
            rp = ref.forward_step(frames[0], update_state=False)
            assert (yp is None) == (rp is None)
            if yp is not None:
                np.testing.assert_array_equal(np_of(yp), rp)
        y = dl.forward_step(to_cl(x, torch.bfloat16))
        r = ref.forward_step(x)
        assert (y is None) == (r is None)
        if y is not None:
            np.testing.assert_array_equal(np_of(y), r)
    # canonical state = the last d frames; round trip into a fresh handle
    st, meta = dl.state_dict_stream()
    assert tuple(st.shape) == (d, B, H, W, C)
    if d:
        np.testing.assert_array_equal(np.moveaxis(np_of(st), -1, 2), np.stack(frames[-d:]))
    dl2 = co.Delay(d, C, in_spatial=(H, W), n_streams=B)
    dl2.load_state_stream(st, meta)
    x = to_cl(_bf16(rng.standard_normal((B, C, H, W))), torch.bfloat16)
    assert torch.equal(dl.forward_step(x), dl2.forward_step(x))
    clip = to_cl(rng.standard_normal((B, C, 6, H, W)), torch.bfloat16)
    assert torch.equal(dl.forward(clip), clip)           # batch Delay: identity


def test_residual_construction_errors():
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200._abi import CoError
    rng = np.random.default_rng(9)
    convs, _ = _layers([(16, 16, (3, 3, 3), (0, 1, 1), 1, False)], 2, 4, 4, rng)
    with pytest.raises(CoError):          # no equal padding without shrink
        co.Residual(convs, shrink=False)
    convs, _ = _layers([(16, 16, (2, 3, 3), (0, 1, 1), 1, False)], 2, 4, 4, rng)
    with pytest.raises(CoError):          # even receptive field cannot be centered
        co.Residual(convs, shrink=True)
    convs, _ = _layers([(16, 32, (3, 3, 3), (1, 1, 1), 1, False)], 2, 4, 4, rng)
    with pytest.raises(CoError):          # channel count changes
        co.Residual(convs)


def _branch(specs, B, H, W, rng, last_fp32=True):
    import paper_2204_03418_b200 as co
    convs, (descs, Ws, bs, relu, rnd) = _layers(specs, B, H, W, rng, last_fp32=last_fp32)
    return co.Stack(convs), O.Stack(descs, Ws, bs, relu, rnd, B), (descs, Ws, bs, relu, rnd)


def test_broadcast_reduce_conv_delay_is_the_residual():
    """Listing 3: BroadcastReduce(conv, Delay(1)) == Residual(conv) (equal padding)."""
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(21)
    B, H, W = 2, 5, 6
    st, om, _ = _branch([(32, 32, (3, 3, 3), (1, 1, 1), 1, False)], B, H, W, rng)
    br = co.BroadcastReduce([st, None], "sum")
    ref = OC.BroadcastReduceStep([om, None], [1, 0], "sum")
    assert br.delay == 1
    for t in range(7):
        x = _bf16(rng.standard_normal((B, 32, H, W)))
        y = br.forward_step(to_cl(x, torch.bfloat16))
        r = ref.forward_step(x)
        assert (y is None) == (r is None), t
        if y is not None:
            assert rel_err(np_of(y), r) <= 1e-4, t


@pytest.mark.parametrize("reduce", ["concat", "sum"])
def test_broadcast_reduce_inception_style(reduce):
    """Listing 4-style block: 1x1, 3x3x3 (no temporal padding), temporal 5x1x1
    depthwise and the identity, concatenated (or summed): branch delays 0 / 2 /
    4 / 0 aligned to 4; step outputs and the batch form vs the oracle."""
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(22)
    B, H, W, C = 2, 5, 6, 32
    specs = [[(C, C, (1, 1, 1), (0, 0, 0), 1, True)], [(C, C, (3, 3, 3), (0, 1, 1), 1, False)],
             [(C, C, (5, 1, 1), (0, 0, 0), C, False)]]
    fp32 = reduce == "sum"          # concat needs one dtype: bf16 branches (the identity's), bf16 bar
    made = [_branch(sp, B, H, W, rng, last_fp32=fp32) for sp in specs]
    tol = 1e-4 if fp32 else 2e-2
    br = co.BroadcastReduce([m[0] for m in made] + [None], reduce)
    ref = OC.BroadcastReduceStep([m[1] for m in made] + [None], [0, 2, 4, 0], reduce)
    assert br.delay == 4 and br.out_channels == (4 * C if reduce == "concat" else C)
    frames = [_bf16(rng.standard_normal((B, C, H, W))) for _ in range(10)]
    for t, x in enumerate(frames):
        if t == 6:
            probe = _bf16(rng.standard_normal((B, C, H, W)))
            yp = br.forward_step(to_cl(probe, torch.bfloat16), update_state=False)
            assert rel_err(np_of(yp), ref.forward_step(probe, update_state=False)) <= tol
        y = br.forward_step(to_cl(x, torch.bfloat16))
        r = ref.forward_step(x)
        assert (y is None) == (r is None), t
        if y is not None:
            assert rel_err(np_of(y), r) <= tol, t
    clip = np.stack(frames, axis=2)
    yb = br.forward(to_cl(clip, torch.bfloat16))
    ref_b = OC.broadcast_reduce_forward(
        [lambda c, m=m: _batch_layers(m[2], c) for m in made] + [None], clip, reduce)
    assert yb.shape[2] == ref_b.shape[2] == 6
    assert rel_err(np_of(yb), ref_b) <= tol
    br.clean_state(); ref.clean_state()
    for t, x in enumerate(frames[:6]):
        y = br.forward_step(to_cl(x, torch.bfloat16))
        r = ref.forward_step(x)
        assert (y is None) == (r is None)
        if y is not None:
            assert rel_err(np_of(y), r) <= tol


def _batch_layers(parts, c):
    descs, Ws, bs, relu, rnd = parts
    cur = c
    for d, Wt, b, r, q in zip(descs, Ws, bs, relu, rnd):
        cur = O.forward(d, Wt, b, cur)
        if r:
            cur = np.maximum(cur, 0.0)
        if q:
            cur = O.bf16_round(cur)
    return cur
