"""GPU parity of the generic CUDA-core path (k_step_direct / k_forward_direct)
against the fp64 oracle, through the C ABI.

Bar (BASELINE.json north_star): ready flags / head / n bit-exact on every
tick; outputs max|err| <= 1e-4 * RMS for fp32 and <= 2e-2 * RMS for bf16 inputs
with fp32 accumulation; bitwise in the exact-integer regime (SC4).
"""
import numpy as np
import pytest
import torch

import oracle as O
from tests.helpers import make_pair, np_of, rand_desc, rel_err, to_cl

pytestmark = pytest.mark.gpu


def _frames(rng, d, B, T, integer=False):
    H, W = d.in_hw
    shp = (B, d.cin) + ((H,) if d.spatial_rank >= 1 else ()) + ((W,) if d.spatial_rank >= 2 else ())
    if integer:
        return [rng.integers(-2, 3, shp).astype(np.float64) for _ in range(T)]
    return [rng.standard_normal(shp) for _ in range(T)]


def test_c1_full_config_vs_oracle_and_sliding_window():
    """BJ configs[0]: 1 stream, 4->8, 3x3x3, pad (0,1,1), 8x8, 16 steps, fp32;
    step outputs vs a sliding-window regular conv3d (O7) and vs O3."""
    from paper_2204_03418_b200 import synth
    cfg = synth.config(1)
    (W, b), L = synth.params(cfg)[0], cfg.layers[0]
    d = O.Desc(2, 4, 8, (3, 3, 3), padding=(0, 1, 1), in_spatial=(8, 8))
    conv, sm, Wq, bq = make_pair(d, W.double().numpy(), b.double().numpy(), 1)
    assert conv.kernel_used == "direct" and conv.delay == 2 and conv.receptive_field == 3
    hist, ys, refs = [], [], []
    for t in range(cfg.steps):
        x = synth.frame(cfg, t)
        xn = np_of(x)
        hist.append(xn)
        y = conv.forward_step(x)
        r = sm.forward_step(xn)
        bf = O.bruteforce_tick(d, Wq, bq, np.stack(hist, axis=2))
        assert (y is None) == (r is None) == (bf is None)
        assert (conv.n, conv.head) == (sm.n, sm.head)
        if y is not None:
            ys.append(np_of(y)); refs.append(bf)
            np.testing.assert_allclose(r, bf, rtol=0, atol=1e-12)
    assert len(ys) == cfg.steps - 2
    assert rel_err(np.stack(ys), np.stack(refs)) <= 1e-4


@pytest.mark.parametrize("seed", range(40))
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_direct_random_shapes(seed, dtype):
    rng = np.random.default_rng(100 + seed)
    d = rand_desc(rng)
    B = int(rng.integers(1, 4))
    W = rng.standard_normal(d.w_shape)
    b = rng.standard_normal(d.cout) if seed % 3 else None
    conv, sm, _, _ = make_pair(d, W, b, B, dtype=dtype, kernel="direct")
    ys, refs = [], []
    for x in _frames(rng, d, B, 14):
        xt = to_cl(x, dtype)
        y = conv.forward_step(xt)
        r = sm.forward_step(np_of(xt))
        assert (y is None) == (r is None)
        assert (conv.n, conv.head) == (sm.n, sm.head)
        if y is not None:
            ys.append(np_of(y)); refs.append(r)
    if ys:
        assert rel_err(np.stack(ys), np.stack(refs)) <= (1e-4 if dtype == torch.float32 else 2e-2)


@pytest.mark.parametrize("seed", range(12))
def test_exact_integer_regime_bitwise(seed):
    rng = np.random.default_rng(300 + seed)
    d = rand_desc(rng)
    B = 2
    W = rng.integers(-2, 3, d.w_shape).astype(np.float64)
    b = rng.integers(-2, 3, d.cout).astype(np.float64)
    conv, sm, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, out_dtype=torch.float32)
    for x in _frames(rng, d, B, 12, integer=True):
        y = conv.forward_step(to_cl(x, torch.bfloat16))
        r = sm.forward_step(x)
        assert (y is None) == (r is None)
        if y is not None:
            assert np.array_equal(np_of(y), r.reshape(y.shape))


@pytest.mark.parametrize("seed", range(8))
def test_forward_steps_is_bitwise_fold_and_pad_end_matches_batch(seed):
    """S:118 (steps == fold of step, bitwise); P:215 + S:117 (pad_end Ready
    outputs == batch forward); co_forward vs oracle O2."""
    rng = np.random.default_rng(400 + seed)
    d = rand_desc(rng)
    B, T = 2, int(rng.integers(max(1, d.receptive_field - 2 * d.padding[0]), 16))
    W, b = rng.standard_normal(d.w_shape), rng.standard_normal(d.cout)
    a, _, Wq, bq = make_pair(d, W, b, B)
    c, _, _, _ = make_pair(d, W, b, B)
    frames = _frames(rng, d, B, T)
    clip = np.stack(frames, axis=2)
    xc = to_cl(clip, torch.float32)
    ys, mask = a.forward_steps(xc, pad_end=True)
    fold = []
    for t in range(T):
        y = c.forward_step(to_cl(frames[t], torch.float32))
        if y is not None:
            fold.append(np_of(y))
    for _ in range(d.padding[0]):
        y = c.forward_pad_step()
        if y is not None:
            fold.append(np_of(y))
    assert ys.shape[2] == len(fold) == int(mask.sum())
    for i, f in enumerate(fold):
        assert np.array_equal(np_of(ys[:, :, i]), f.reshape(ys[:, :, i].shape))
    ref = O.forward(d, Wq, bq, clip)
    assert rel_err(np_of(ys), ref) <= 1e-4
    yb = c.forward(xc)
    assert rel_err(np_of(yb), ref) <= 1e-4


@pytest.mark.parametrize("seed", range(10))
def test_state_get_set_roundtrip_and_oracle_state(seed):
    rng = np.random.default_rng(500 + seed)
    d = rand_desc(rng)
    B = 2
    W, b = rng.standard_normal(d.w_shape), rng.standard_normal(d.cout)
    conv, sm, _, _ = make_pair(d, W, b, B)
    frames = _frames(rng, d, B, 9)
    for x in frames[:6]:
        conv.forward_step(to_cl(x, torch.float32)); sm.forward_step(x)
    st, meta = conv.state_dict_stream()
    ref = sm.state()                                       # (R, B, Cout, S1', S2')
    if ref.shape[0]:
        got = np_of(st).reshape(ref.shape[0], B, d.out_spatial[0], d.out_spatial[1], d.cout).transpose(0, 1, 4, 2, 3)
        assert rel_err(got, ref) <= 1e-4
    assert (meta.n, meta.head) == (sm.n, sm.head)
    # continue from an oracle-loaded state on a fresh handle
    conv2, _, _, _ = make_pair(d, W, b, B)
    oracle_state = torch.from_numpy(ref.transpose(0, 1, 3, 4, 2).copy()).float().cuda() if ref.shape[0] else st
    conv2.load_state_stream(oracle_state, meta)
    for x in frames[6:]:
        y1 = conv.forward_step(to_cl(x, torch.float32))
        y2 = conv2.forward_step(to_cl(x, torch.float32))
        r = sm.forward_step(x)
        assert (y1 is None) == (y2 is None) == (r is None)
        if r is not None:
            assert rel_err(np_of(y2), r) <= 1e-4
    # get -> set round trip is bitwise
    st1, meta1 = conv.state_dict_stream()
    conv2.load_state_stream(st1, meta1)
    st2, meta2 = conv2.state_dict_stream()
    assert torch.equal(st1, st2) and meta2.n == meta1.n and meta2.head == meta1.head


def test_update_state_false_clean_and_replay():
    rng = np.random.default_rng(600)
    d = O.Desc(2, 3, 5, (3, 3, 3), padding=(1, 1, 1), in_spatial=(6, 7))
    conv, sm, _, _ = make_pair(d, rng.standard_normal(d.w_shape), rng.standard_normal(5), 3)
    frames = _frames(rng, d, 3, 8)
    outs = [conv.forward_step(to_cl(x, torch.float32)) for x in frames]
    st0, m0 = conv.state_dict_stream()
    probe = to_cl(rng.standard_normal((3, 3, 6, 7)), torch.float32)
    y_peek = conv.forward_step(probe, update_state=False)
    st1, m1 = conv.state_dict_stream()
    assert torch.equal(st0, st1) and m0.n == m1.n
    y_real = conv.forward_step(probe)
    assert torch.equal(y_peek, y_real)
    conv.clean_state()
    st, meta = conv.state_dict_stream()
    assert meta.n == 0 and torch.count_nonzero(st) == 0
    outs2 = [conv.forward_step(to_cl(x, torch.float32)) for x in frames]
    for a, c in zip(outs, outs2):
        assert (a is None and c is None) or torch.equal(a, c)


def test_stack_small_vs_oracle():
    """Layer-stack driver (a7): Empty short-circuit, delay bookkeeping, ReLU and
    bf16 inter-layer activations mirrored by the oracle (O6)."""
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(700)
    descs = [O.Desc(2, 3, 8, (5, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), in_spatial=(12, 10)),
             O.Desc(2, 8, 8, (1, 3, 3), padding=(0, 1, 1), in_spatial=(6, 5)),
             O.Desc(2, 8, 6, (3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), in_spatial=(6, 5))]
    B = 2
    Ws = [(rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))) for d in descs]
    bs = [rng.standard_normal(d.cout) * 0.1 for d in descs]
    convs = []
    for l, d in enumerate(descs):
        last = l == len(descs) - 1
        c, _, Wq, bq = make_pair(d, Ws[l], bs[l], B, dtype=torch.bfloat16,
                                 out_dtype=torch.float32 if last else torch.bfloat16,
                                 activation=None if last else "relu")
        Ws[l], bs[l] = Wq, bq
        convs.append(c)
    stack = co.Stack(convs)
    assert stack.delay == 4 + 0 + 2
    ost = O.Stack(descs, Ws, bs, [1, 1, 0], [1, 1, 0], B)
    ys, refs = [], []
    for t in range(12):
        x = to_cl(rng.standard_normal((B, 3, 12, 10)), torch.bfloat16)
        y = stack.forward_step(x)
        r = ost.forward_step(np_of(x))
        assert (y is None) == (r is None) == (t < 6)
        if y is not None:
            ys.append(np_of(y)); refs.append(r)
    assert rel_err(np.stack(ys), np.stack(refs)) <= 2e-2


def test_host_buffer_entry_point_matches_device_path():
    rng = np.random.default_rng(800)
    d = O.Desc(2, 4, 6, (3, 3, 3), padding=(0, 1, 1), in_spatial=(5, 6))
    W, b = rng.standard_normal(d.w_shape), rng.standard_normal(6)
    a, _, _, _ = make_pair(d, W, b, 2)
    c, _, _, _ = make_pair(d, W, b, 2)
    yh = torch.empty((2, 5, 6, 6), dtype=torch.float32).pin_memory()
    for _ in range(5):
        x = to_cl(rng.standard_normal((2, 4, 5, 6)), torch.float32)
        xh = x.movedim(1, -1).contiguous().cpu().pin_memory()
        y = a.forward_step(x)
        r = c.forward_step_host(xh, yh)
        assert (y is None) == (not r)
        if y is not None:
            assert torch.equal(y.movedim(1, -1).cpu(), yh)


def test_error_codes():
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200._abi import CoError, CO_ERR_ARG, CO_ERR_LENGTH, CO_ERR_SHAPE
    W = torch.zeros(4, 2, 3, 1, 1, device="cuda")
    with pytest.raises(CoError) as e:   # p_t > f - 1
        co.Conv(2, 4, (3, 1, 1), weight=W, padding=(3, 0, 0), in_spatial=(4, 4), dtype=torch.float32)
    assert e.value.code == CO_ERR_ARG
    with pytest.raises(CoError) as e:   # groups must divide channels
        co.Conv(2, 4, (3, 1, 1), weight=W, groups=3, in_spatial=(4, 4), dtype=torch.float32)
    assert e.value.code == CO_ERR_ARG
    c = co.Conv(2, 4, (3, 1, 1), weight=W, in_spatial=(4, 4), dtype=torch.float32)
    with pytest.raises(ValueError):
        c.forward(co.channels_last(torch.zeros(1, 2, 2, 4, 4, device="cuda")))
    _, meta = c.state_dict_stream()
    meta.ring_slots += 1
    with pytest.raises(CoError) as e:
        c.load_state_stream(torch.zeros(2, 1, 4, 4, 4, device="cuda"), meta)
    assert e.value.code == CO_ERR_SHAPE


@pytest.mark.parametrize("kernel", ["direct", "dense_tc"])
def test_steps_host_pipeline_matches_device_fold(kernel):
    """co_forward_steps_host (time-major pinned frames, copies overlapped with the
    steps) == the fold of co_forward_step on device tensors, bitwise; ready mask
    and clock identical; and the stack variant likewise."""
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(900)
    d = O.Desc(2, 16, 32, (3, 3, 3), padding=(0, 1, 1), in_spatial=(6, 7))
    dt = torch.bfloat16
    W, b = rng.standard_normal(d.w_shape) / 12, rng.standard_normal(32) * 0.1
    a, _, _, _ = make_pair(d, W, b, 3, dtype=dt, out_dtype=dt, kernel=kernel)
    c, _, _, _ = make_pair(d, W, b, 3, dtype=dt, out_dtype=dt, kernel=kernel)
    T = 7
    frames = [to_cl(rng.standard_normal((3, 16, 6, 7)), dt) for _ in range(T)]
    fold = [y for y in (a.forward_step(x) for x in frames) if y is not None]
    xh = torch.stack([f.movedim(1, -1).contiguous().cpu() for f in frames]).pin_memory()   # (T, B, H, W, C)
    yh = torch.zeros((T, 3, 6, 7, 32), dtype=dt).pin_memory()
    n, mask = c.forward_steps_host(xh, yh)
    assert n == len(fold) == int(mask.sum()) and mask.tolist() == [t >= 2 for t in range(T)]
    for i, f in enumerate(fold):
        assert torch.equal(yh[i], f.movedim(1, -1).cpu())
    assert (c.n, c.head) == (a.n, a.head)
    # stack of two layers
    d2 = O.Desc(2, 32, 8, (2, 1, 1), in_spatial=(6, 7))
    W2, b2 = rng.standard_normal(d2.w_shape) / 8, rng.standard_normal(8) * 0.1
    a2, _, _, _ = make_pair(d2, W2, b2, 3, dtype=dt, out_dtype=dt)
    c2, _, _, _ = make_pair(d2, W2, b2, 3, dtype=dt, out_dtype=dt)
    a.clean_state(); c.clean_state()
    sa, sc = co.Stack([a, a2]), co.Stack([c, c2])
    fold = [y for y in (sa.forward_step(x) for x in frames) if y is not None]
    yh2 = torch.zeros((T, 3, 6, 7, 8), dtype=dt).pin_memory()
    n, mask = sc.forward_steps_host(xh, yh2)
    assert n == len(fold) == 4
    for i, f in enumerate(fold):
        assert torch.equal(yh2[i], f.movedim(1, -1).cpu())
