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
    fold += [y for y in (c.forward_step(None) for _ in range(d.padding[0])) if y is not None]
    assert ys.shape[2] == len(fold) == int(mask.sum())
    for i, f in enumerate(fold):
        assert torch.equal(ys[:, :, i], f)
    if d.out_len(T) >= 1:
        assert rel_err(np_of(ys), O.forward(d, Wq, bq, clip)) <= 1e-4
