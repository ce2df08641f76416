"""Chunked co_forward_steps (k_depthwise.cu k_steps_dw_t): the
fold of a whole clip in one launch with the state in registers must equal the
per-step fold bit for bit -- outputs, ready mask, clock and canonical state --
across consecutive calls (state carried between chunks), pad_end, mid-stream
starts (n0 > d) and update_state = 0, and match the fp64 oracle."""
import os

import numpy as np
import pytest
import torch

import oracle as O
from tests.helpers import reset_opt, set_opt, make_pair, np_of, rel_err

pytestmark = pytest.mark.gpu


def _clip(rng, B, C, T, H, W):
    import paper_2204_03418_b200 as co
    x = rng.standard_normal((B, C, T, H, W))
    return co.channels_last(torch.from_numpy(x).to(torch.bfloat16).cuda())


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("kt,pad", [(2, 0), (3, 1), (5, 0), (5, 4), (7, 2), (9, 0)])
def test_chunked_equals_per_step_fold(kt, pad, out_dtype, monkeypatch):
    rng = np.random.default_rng(kt * 10 + pad)
    B, C, H, W = 3, 32, 4, 5
    d = O.Desc(2, C, C, (kt, 1, 1), padding=(pad, 0, 0), groups=C, in_spatial=(H, W))
    Wt = rng.standard_normal(d.w_shape) / np.sqrt(kt)
    bt = rng.standard_normal(C) * 0.1
    runs = {}
    for chunk in ("1", "0"):
        set_opt("chunk", chunk)
        conv, sm, _, _ = make_pair(d, Wt, bt, B, dtype=torch.bfloat16, out_dtype=out_dtype, kernel="depthwise",
                                   activation="relu")
        rng2 = np.random.default_rng(1)
        outs = []
        for T, pe in ((3, False), (kt + 4, False), (1, False), (6, True)):   # n0 < d, n0 > d, tiny, pad_end
            ys, mask = conv.forward_steps(_clip(rng2, B, C, T, H, W), pad_end=pe)
            outs.append((ys.clone(), mask.clone(), conv.n))
        probe, _ = conv.forward_steps(_clip(rng2, B, C, 4, H, W), update_state=False)
        st, meta = conv.state_dict_stream()
        runs[chunk] = (outs, probe.clone(), st.clone(), conv.n)
    (oa, pa, sa, na), (ob, pb, sb, nb) = runs["1"], runs["0"]
    assert na == nb
    for (ya, ma, ca), (yb, mb, cb) in zip(oa, ob):
        assert ca == cb and torch.equal(ma, mb)
        assert torch.equal(ya, yb)
    assert torch.equal(pa, pb)
    assert torch.equal(sa, sb)


def test_chunked_matches_oracle_and_continues_per_step(monkeypatch):
    """A chunk, then per-step calls, then another chunk: every Ready output
    matches the oracle fed the same frames."""
    set_opt("chunk", "1")
    rng = np.random.default_rng(3)
    B, C, H, W, kt = 2, 64, 3, 4, 5
    d = O.Desc(2, C, C, (kt, 1, 1), groups=C, in_spatial=(H, W))
    conv, sm, _, _ = make_pair(d, rng.standard_normal(d.w_shape) / 2, rng.standard_normal(C) * 0.1, B,
                               dtype=torch.bfloat16, out_dtype=torch.float32, kernel="depthwise")
    assert "k_step_dw_t" in conv.kernel_name
    got, ref = [], []
    for phase in ("chunk", "step", "chunk"):
        clip = _clip(rng, B, C, 7, H, W)
        frames = [np_of(clip[:, :, t]) for t in range(7)]
        if phase == "chunk":
            ys, mask = conv.forward_steps(clip)
            got += [np_of(ys[:, :, i]) for i in range(ys.shape[2])]
        else:
            import paper_2204_03418_b200 as co
            for t in range(7):
                y = conv.forward_step(co.channels_last(clip[:, :, t]))
                if y is not None:
                    got.append(np_of(y))
        for f in frames:
            r = sm.forward_step(f)
            if r is not None:
                ref.append(r)
    assert len(got) == len(ref) == 21 - (kt - 1)
    assert rel_err(np.stack(got), np.stack(ref).reshape(np.stack(got).shape)) <= 1e-4


DENSE = {
    "halo": (O.Desc(2, 64, 64, (3, 3, 3), padding=(0, 1, 1), in_spatial=(6, 7)), 3),
    "halo_pad": (O.Desc(2, 32, 32, (3, 3, 3), padding=(2, 1, 1), in_spatial=(5, 9)), 2),
    "flat_pair_c5": (O.Desc(1, 256, 256, (9, 1), dilation=(2, 1), in_spatial=(25, 1)), 7),
    "flat_1x1": (O.Desc(2, 64, 128, (3, 1, 1), in_spatial=(5, 6)), 5),
}


def _dense_clip(rng, d, B, T):
    import paper_2204_03418_b200 as co
    H, W = d.in_hw
    shape = (B, d.cin, T) + ((H,) if d.spatial_rank >= 1 else ()) + ((W,) if d.spatial_rank >= 2 else ())
    return co.channels_last(torch.from_numpy(rng.standard_normal(shape)).to(torch.bfloat16).cuda())


@pytest.mark.parametrize("chunk_t", [None, "4"])
@pytest.mark.parametrize("name", list(DENSE))
def test_dense_chunked_equals_per_step_fold(name, chunk_t, monkeypatch):
    """Chunked tensor-core steps (one launch per chunk, item-batch-major) equal
    the per-step fold bit for bit: outputs, ready mask, clock, canonical state."""
    d, B = DENSE[name]
    rng = np.random.default_rng(len(name))
    Wt = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    bt = rng.standard_normal(d.cout) * 0.1
    if chunk_t:
        set_opt("chunk_t", chunk_t)
    set_opt("chunk_flat", "1")      # FLAT chunking is off by default; keep it covered
    runs = {}
    for chunk in ("1", "0"):
        set_opt("chunk", chunk)
        conv, _, _, _ = make_pair(d, Wt, bt, B, dtype=torch.bfloat16, out_dtype=torch.float32, kernel="dense_tc")
        rng2 = np.random.default_rng(2)
        outs = []
        for T in (3, d.receptive_field + 6, 2, 9):
            ys, mask = conv.forward_steps(_dense_clip(rng2, d, B, T))
            outs.append((ys.clone(), mask.clone(), conv.n))
        probe, _ = conv.forward_steps(_dense_clip(rng2, d, B, 5), update_state=False)
        st, _ = conv.state_dict_stream()
        runs[chunk] = (outs, probe.clone(), st.clone(), conv.kernel_name)
    (oa, pa, sa, ka), (ob, pb, sb, kb) = runs["1"], runs["0"]
    assert ka == kb
    for (ya, ma, ca), (yb, mb, cb) in zip(oa, ob):
        assert ca == cb and torch.equal(ma, mb)
        assert torch.equal(ya, yb)
    assert torch.equal(pa, pb)
    assert torch.equal(sa, sb)


def test_dense_chunked_matches_oracle():
    """C5-shaped pair FLAT layer: a chunked clip, then per-step calls, then a
    chunked clip -- every Ready output within 1e-4 of the fp64 oracle."""
    import paper_2204_03418_b200 as co
    d, B = DENSE["flat_pair_c5"]
    rng = np.random.default_rng(9)
    set_opt("chunk_flat", "1")
    conv, sm, _, _ = make_pair(d, rng.standard_normal(d.w_shape) / 48, rng.standard_normal(d.cout) * 0.1, B,
                               dtype=torch.bfloat16, out_dtype=torch.float32, kernel="dense_tc")
    got, ref = [], []
    for phase in ("chunk", "step", "chunk"):
        clip = _dense_clip(rng, d, B, 12)
        frames = [np_of(clip[:, :, t]) for t in range(12)]
        if phase == "chunk":
            ys, _ = conv.forward_steps(clip)
            got += [np_of(ys[:, :, i]) for i in range(ys.shape[2])]
        else:
            for t in range(12):
                y = conv.forward_step(co.channels_last(clip[:, :, t]))
                if y is not None:
                    got.append(np_of(y))
        for f in frames:
            r = sm.forward_step(f)
            if r is not None:
                ref.append(r)
    reset_opt("chunk_flat")
    assert len(got) == len(ref) == 36 - (d.receptive_field - 1)
    g = np.stack(got)
    assert rel_err(g, np.stack(ref).reshape(g.shape)) <= 1e-4


@pytest.mark.parametrize("kt,k,pad", [(3, 3, (0, 1, 1)), (2, 3, (1, 1, 1)), (5, 3, (2, 1, 1)), (3, 5, (0, 2, 2)),
                                      (1, 3, (0, 1, 1))])
def test_depthwise_stencil_chunked_equals_per_step(kt, k, pad, monkeypatch):
    """Chunked K2 (k_steps_dw_st: halo staged per frame, state in registers)
    equals the per-step K2 fold bit for bit, across consecutive calls."""
    rng = np.random.default_rng(kt * 7 + k)
    B, C, H, W = 2, 32, 6, 9
    d = O.Desc(2, C, C, (kt, k, k), padding=pad, groups=C, in_spatial=(H, W))
    Wt = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    bt = rng.standard_normal(C) * 0.1
    set_opt("chunk_st", "1")        # off by default (slower); keep it covered
    runs = {}
    for chunk in ("1", "0"):
        set_opt("chunk", chunk)
        conv, _, _, _ = make_pair(d, Wt, bt, B, dtype=torch.bfloat16, out_dtype=torch.float32, kernel="depthwise",
                                  activation="relu")
        rng2 = np.random.default_rng(3)
        outs = []
        for T in (2, kt + 5, 4):
            ys, mask = conv.forward_steps(_clip(rng2, B, C, T, H, W))
            outs.append((ys.clone(), mask.clone()))
        st, _ = conv.state_dict_stream()
        runs[chunk] = (outs, st.clone(), conv.kernel_name)
    (oa, sa, ka), (ob, sb, kb) = runs["1"], runs["0"]
    assert ka.startswith("k_step_dw_s")        # per-step K2s / K2 between the chunked calls
    for (ya, ma), (yb, mb) in zip(oa, ob):
        assert torch.equal(ma, mb) and torch.equal(ya, yb)
    assert torch.equal(sa, sb)
