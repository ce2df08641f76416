"""GPU parity of the dense tcgen05 step kernel (k_step_dense_tc) against the
fp64 oracle and against the generic CUDA-core kernel, through the C ABI.

Sizes span several tiles, both channel parts and a ragged last tile; the
exact-integer regime is compared bit for bit.
"""
import numpy as np
import pytest
import torch

import oracle as O
from tests.helpers import reset_opt, set_opt, assert_bf16_rounding_bound, make_pair, np_of, rel_err, to_cl

pytestmark = pytest.mark.gpu

CASES = {
    # C2-shaped halo mode: 3x3 spatial, pad 1, several tiles per stream, ragged rows
    "halo_c2like": dict(desc=O.Desc(2, 64, 64, (3, 3, 3), padding=(0, 1, 1), in_spatial=(13, 24)), B=3),
    "halo_c2like_oddtiles": dict(desc=O.Desc(2, 64, 64, (3, 3, 3), padding=(0, 1, 1), in_spatial=(12, 24)), B=3),
    "flat_c5full": dict(desc=O.Desc(1, 256, 256, (9, 1), dilation=(2, 1), in_spatial=(25, 1)), B=7),
    "halo_c2like_pt1": dict(desc=O.Desc(2, 32, 64, (3, 3, 3), padding=(1, 1, 1), in_spatial=(9, 30)), B=2),
    "halo_wide": dict(desc=O.Desc(2, 16, 32, (3, 3, 3), padding=(0, 1, 1), in_spatial=(5, 56)), B=2),
    "halo_kt5": dict(desc=O.Desc(2, 16, 32, (5, 3, 3), padding=(0, 1, 1), in_spatial=(7, 11)), B=2),
    "halo_kt1": dict(desc=O.Desc(2, 64, 64, (1, 3, 3), padding=(0, 1, 1), in_spatial=(10, 12)), B=2),
    "halo_nopad": dict(desc=O.Desc(2, 16, 32, (3, 3, 3), in_spatial=(9, 10)), B=2),
    # C5-shaped flat mode: 25 joints, kt 9, dilation 2, rows span streams, ragged tail
    "flat_c5like": dict(desc=O.Desc(1, 32, 32, (9, 1), dilation=(2, 1), in_spatial=(25, 1)), B=7),
    "flat_conv1d": dict(desc=O.Desc(0, 48, 32, (3,), padding=(1,)), B=300),
    # KLOOP mode: K streamed through the stage ring, A gathered by strided TMA
    "kloop_s2": dict(desc=O.Desc(2, 32, 64, (3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), in_spatial=(13, 18)), B=2),
    "kloop_c4l3like": dict(desc=O.Desc(2, 128, 128, (3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1),
                                       in_spatial=(12, 20)), B=2),
    "kloop_bigK": dict(desc=O.Desc(2, 256, 64, (3, 3, 3), padding=(0, 1, 1), in_spatial=(7, 9)), B=2),
    "kloop_dil": dict(desc=O.Desc(2, 16, 32, (2, 3, 3), padding=(0, 2, 2), dilation=(1, 2, 2), in_spatial=(9, 9)), B=2),
    "kloop_wide": dict(desc=O.Desc(2, 16, 32, (3, 1, 3), stride=(1, 1, 2), padding=(0, 0, 1), in_spatial=(3, 300)), B=2),
    "kloop_kt1_s2": dict(desc=O.Desc(2, 64, 128, (1, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), in_spatial=(10, 14)), B=3),
    # KHALO: stride 1 with weights too large to stay resident -- one input-halo box
    # per 64-channel block, taps as shifted descriptors, weights streamed (C4 layer 4)
    "khalo_c4l4like": dict(desc=O.Desc(2, 256, 128, (3, 3, 3), padding=(0, 1, 1), in_spatial=(12, 20)), B=2),
    "khalo_bigK": dict(desc=O.Desc(2, 256, 64, (3, 3, 3), padding=(0, 1, 1), in_spatial=(7, 9)), B=3),
    "khalo_pt1": dict(desc=O.Desc(2, 192, 64, (3, 3, 3), padding=(1, 1, 1), in_spatial=(6, 30)), B=2),
    "khalo_kt1_single": dict(desc=O.Desc(2, 256, 256, (1, 3, 3), padding=(0, 1, 1), in_spatial=(9, 11)), B=3),
    # strided KHALO: 2 x 2 phase sub-images, each one elementStrides = 2 TMA box (C4 layers 3 / 5)
    "khalo_s2_c4l3like": dict(desc=O.Desc(2, 128, 128, (3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1),
                                          in_spatial=(12, 20)), B=2),
    "khalo_s2_odd": dict(desc=O.Desc(2, 64, 64, (3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), in_spatial=(13, 17)),
                         B=3),
    "khalo_s2_nopad_single": dict(desc=O.Desc(2, 64, 32, (3, 3, 3), stride=(1, 2, 2), in_spatial=(11, 12)), B=2),
    "khalo_s2_1x1": dict(desc=O.Desc(2, 64, 64, (3, 1, 1), stride=(1, 2, 2), in_spatial=(8, 10)), B=2),
    "khalo_st2": dict(desc=O.Desc(2, 256, 64, (3, 3, 3), stride=(2, 1, 1), padding=(1, 1, 1), in_spatial=(6, 9)), B=2),
    "khalo_tdil2_s2": dict(desc=O.Desc(2, 128, 64, (3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), dilation=(2, 1, 1),
                                       in_spatial=(9, 13)), B=2),
    "khalo_s2_kt1_single": dict(desc=O.Desc(2, 64, 128, (1, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1),
                                            in_spatial=(10, 14)), B=3),
    # small-Cin stems: W-im2col'd frame (C4 layer 1 shaped), KLOOP (stride 2) and HALO (stride 1)
    "stem_c4like": dict(desc=O.Desc(2, 3, 32, (5, 7, 7), stride=(1, 2, 2), padding=(0, 3, 3), in_spatial=(20, 24)), B=2),
    "stem_halo": dict(desc=O.Desc(2, 3, 16, (3, 3, 3), padding=(1, 1, 1), in_spatial=(9, 10)), B=2),
    # STEM (shared-memory W-im2col): two channel parts on one image, 7 output rows per tile
    # (19 raw rows in 2 row phases), a 2-channel stem (Kp 16, even window starts), a
    # 1-row tile of a wide frame, odd channel count with a 3-wide kernel
    "stem_2parts": dict(desc=O.Desc(2, 3, 64, (5, 7, 7), stride=(1, 2, 2), padding=(0, 3, 3), in_spatial=(30, 32)),
                        B=3),
    "stem_c2": dict(desc=O.Desc(2, 2, 32, (3, 5, 5), stride=(1, 2, 2), padding=(0, 2, 2), in_spatial=(17, 24)), B=2),
    "stem_wide": dict(desc=O.Desc(2, 3, 32, (2, 7, 7), stride=(1, 2, 2), padding=(0, 3, 3), in_spatial=(9, 248)),
                      B=2),
    "stem_k3c5": dict(desc=O.Desc(2, 5, 32, (3, 3, 3), stride=(1, 2, 2), padding=(1, 1, 1), in_spatial=(15, 16)),
                      B=3),
    # raw rows not a multiple of 16 B (22 x 3 bf16): no bulk copy -- the HBM W-im2col pass
    "stem_unaligned": dict(desc=O.Desc(2, 3, 32, (5, 7, 7), stride=(1, 2, 2), padding=(0, 3, 3), in_spatial=(20, 22)),
                           B=2),
    # temporal stride > 1 (Principle 5): skipped ticks are Empty, only
    # the slices feeding an emitted output touch the ring (A20)
    "halo_st2": dict(desc=O.Desc(2, 32, 32, (3, 3, 3), stride=(2, 1, 1), padding=(1, 1, 1), in_spatial=(6, 7)), B=2),
    "kloop_st3": dict(desc=O.Desc(2, 32, 32, (5, 3, 3), stride=(3, 2, 2), padding=(2, 1, 1), in_spatial=(9, 8)), B=2),
    "flat_st2_dil2": dict(desc=O.Desc(1, 32, 32, (3, 1), stride=(2, 1), dilation=(2, 1), in_spatial=(25, 1)), B=3),
}
FORCE_KLOOP = {"halo_c2like", "halo_kt5", "flat_c5like"}   # also run these through the K pipeline
PAIR_CASES = ["halo_c2like", "halo_c2like_oddtiles", "flat_c5full"]   # CTA-pair (cta_group::2) variants
KPAIR_CASES = ["kloop_c4l3like", "kloop_bigK", "kloop_st3", "stem_c4like", "kloop_s2",
               "khalo_c4l4like", "khalo_s2_c4l3like"]   # KLOOP / KHALO CTA pairs


def _run(case, integer=False, steps=None, out_dtype=torch.float32, seed=0, force_kloop=False, pair=False, stem=True):
    import os
    d, B = CASES[case]["desc"], CASES[case]["B"]
    rng = np.random.default_rng(seed)
    if integer:
        W = rng.integers(-2, 3, d.w_shape).astype(np.float64)
        b = rng.integers(-2, 3, d.cout).astype(np.float64)
    else:
        W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
        b = rng.standard_normal(d.cout) * 0.1
    if force_kloop:
        set_opt("tc_mode", 1)
    if force_kloop or case.startswith("kloop"):
        set_opt("khalo", "0")              # keep the strided-gather K pipeline covered
    if pair:
        set_opt("pair", "2")
        set_opt("kpair", "2")
    if not stem:
        set_opt("stem", 0)                        # the HBM W-im2col pass + strided-gather K pipeline
    try:
        conv, sm, Wq, bq = make_pair(d, W, b, B, dtype=torch.bfloat16, out_dtype=out_dtype, kernel="dense_tc")
    finally:
        reset_opt("tc_mode")
        reset_opt("pair")
        reset_opt("kpair")
        reset_opt("khalo")
        reset_opt("stem")
    if pair:
        assert "pair" in conv.kernel_name, conv.kernel_name
    ref_conv, _, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, out_dtype=out_dtype, kernel="direct")
    assert conv.kernel_used == "dense_tc", conv.kernel_name
    if force_kloop or case.startswith("kloop"):  # (kloop_st3: spatial stride 2)
        assert "kloop" in conv.kernel_name, conv.kernel_name
    if case.startswith("stem_") and case != "stem_halo":
        fused = stem and not pair and case != "stem_unaligned"
        assert (",stem" if fused else "kloop+wcols") in conv.kernel_name, conv.kernel_name
    if case.startswith("khalo"):
        assert "khalo" in conv.kernel_name, conv.kernel_name
        assert ("pair" in conv.kernel_name) == (not case.endswith("single")), conv.kernel_name
    H, Wd = d.in_hw
    shp = (B, d.cin) + ((H,) if d.spatial_rank >= 1 else ()) + ((Wd,) if d.spatial_rank >= 2 else ())
    steps = steps or (d.receptive_field + 4 + 3 * (d.stride[0] - 1))
    ys, refs, yds = [], [], []
    for t in range(steps):
        x = rng.integers(-2, 3, shp).astype(np.float64) if integer else rng.standard_normal(shp)
        xt = to_cl(x, torch.bfloat16)
        y = conv.forward_step(xt)
        yd = ref_conv.forward_step(xt)
        r = sm.forward_step(np_of(xt))
        assert (y is None) == (r is None) == (yd is None)
        assert (conv.n, conv.head) == (sm.n, sm.head)
        if y is not None:
            ys.append(np_of(y)); refs.append(r.reshape(y.shape)); yds.append(np_of(yd))
    return conv, np.stack(ys), np.stack(refs), np.stack(yds)


@pytest.mark.parametrize("case", list(CASES))
def test_dense_tc_vs_oracle(case):
    conv, y, ref, yd = _run(case)
    assert rel_err(y, ref) <= 2e-2
    # fp32 accumulation of exact bf16 products: in practice ~1e-6 relative
    assert rel_err(y, ref) <= 1e-4
    assert rel_err(y, yd) <= 1e-4


@pytest.mark.parametrize("case", list(CASES))
def test_dense_tc_exact_integer_bitwise(case):
    _, y, ref, yd = _run(case, integer=True)
    assert np.array_equal(y, ref)
    assert np.array_equal(y, yd)


@pytest.mark.parametrize("case", PAIR_CASES + KPAIR_CASES)
def test_dense_tc_cta_pair(case):
    """The CTA-pair variants (M = 256 over two SMs, weights split by N) agree
    with the oracle and, in the exact-integer regime, bit for bit."""
    _, y, ref, yd = _run(case, pair=True)
    assert rel_err(y, ref) <= 1e-4 and rel_err(y, yd) <= 1e-4
    _, y, ref, _ = _run(case, integer=True, pair=True)
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("case", ["kloop_s2", "kloop_dil", "stem_c4like", "kloop_kt1_s2"])
@pytest.mark.parametrize("mc", ["2", "4"])
def test_dense_tc_weight_multicast(case, mc, monkeypatch):
    """One-CTA K-pipeline layers in weight-multicast clusters (CO_TC_MC): each
    CTA loads 1/mc of every weight chunk and multicasts it, stages are released
    by every CTA's commit -- same results as the oracle, bit for bit in the
    integer regime."""
    set_opt("mc", mc)
    _, y, ref, yd = _run(case)
    assert rel_err(y, ref) <= 1e-4 and rel_err(y, yd) <= 1e-4
    _, y, ref, _ = _run(case, integer=True)
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("case", sorted(FORCE_KLOOP))
def test_dense_tc_forced_kloop(case):
    """The same layers through the K pipeline (CO_TC_MODE=kloop) agree with the oracle."""
    _, y, ref, yd = _run(case, force_kloop=True)
    assert rel_err(y, ref) <= 1e-4 and rel_err(y, yd) <= 1e-4
    _, y, ref, _ = _run(case, integer=True, force_kloop=True)
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("case", ["halo_c2like", "flat_c5like"])
def test_dense_tc_bf16_output(case):
    # A16: bf16 outputs are checked against the RNE error bound
    _, y, ref, _ = _run(case, out_dtype=torch.bfloat16)
    assert rel_err(y, ref) <= 2e-2
    assert_bf16_rounding_bound(y, ref)


@pytest.mark.parametrize("case", ["halo_c2like", "flat_c5like", "kloop_s2", "stem_c4like", "halo_st2", "kloop_st3",
                                  "khalo_c4l4like", "khalo_pt1", "khalo_s2_odd", "khalo_st2", "khalo_tdil2_s2"])
def test_dense_tc_state_and_steps(case):
    """State get vs oracle O5, update_state=False purity, forward_steps fold."""
    d, B = CASES[case]["desc"], CASES[case]["B"]
    rng = np.random.default_rng(5)
    W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    b = rng.standard_normal(d.cout) * 0.1
    conv, sm, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="dense_tc")
    conv2, _, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="dense_tc")
    H, Wd = d.in_hw
    shp = (B, d.cin) + ((H,) if d.spatial_rank >= 1 else ()) + ((Wd,) if d.spatial_rank >= 2 else ())
    T = d.receptive_field + 3
    frames = [to_cl(rng.standard_normal(shp), torch.bfloat16) for _ in range(T)]
    for x in frames:
        conv.forward_step(x)
        sm.forward_step(np_of(x))
    st, meta = conv.state_dict_stream()
    ref = sm.state()
    got = np_of(st).reshape((ref.shape[0], B) + d.out_spatial + (d.cout,)).transpose(0, 1, 4, 2, 3)
    assert rel_err(got, ref) <= 1e-4
    probe = to_cl(rng.standard_normal(shp), torch.bfloat16)
    y_peek = conv.forward_step(probe, update_state=False)
    st1, _ = conv.state_dict_stream()
    assert torch.equal(st, st1)
    y_real = conv.forward_step(probe)
    assert (y_peek is None) == (y_real is None)      # an Empty tick under temporal stride stays Empty
    assert y_peek is None or torch.equal(y_peek, y_real)
    clip = torch.stack([f for f in frames], dim=2)       # (B, C, T, *S), channels-last per frame
    from paper_2204_03418_b200 import channels_last
    ys, mask = conv2.forward_steps(channels_last(clip))
    conv3, _, _, _ = make_pair(d, W, b, B, dtype=torch.bfloat16, kernel="dense_tc")
    fold = [y for y in (conv3.forward_step(x) for x in frames) if y is not None]
    assert ys.shape[2] == len(fold)
    for i, f in enumerate(fold):
        assert torch.equal(ys[:, :, i], f)


def test_c4_stack_reduced_spatial_vs_oracle():
    """BASELINE.json configs[3] (Slow-style 5-layer stack: 3->64->128->256->256->512,
    kernels 5x7x7 s2, 1x3x3, 3x3x3 s2, 3x3x3, 3x3x3 s2, BN folded, ReLU x4) at a
    reduced 32x32 input so the fp64 oracle stays fast: every layer runs on the
    tensor-core kernel (stem W-im2col, HALO, KLOOP); delay d_NN = sum(kt-1) = 10."""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    cfg = synth.config(4, n_streams=2, in_spatial=(32, 32))
    params = synth.params(cfg)
    convs, descs, Ws, bs, spat = [], [], [], [], tuple(cfg.in_spatial)
    for l, (L, (W, b)) in enumerate(zip(cfg.layers, params)):
        last = l == len(cfg.layers) - 1
        c = co.Conv(L.cin, L.cout, L.kernel, weight=W.cuda(), bias=b.cuda(), stride=L.stride, padding=L.padding,
                    dilation=L.dilation, groups=L.groups, spatial_rank=2, in_spatial=spat, n_streams=cfg.n_streams,
                    dtype=torch.bfloat16, out_dtype=torch.float32 if last else torch.bfloat16,
                    activation="relu" if L.relu else None)
        assert c.kernel_used == "dense_tc", (l, c.kernel_name)
        d = O.Desc(2, L.cin, L.cout, L.kernel, L.stride, L.padding, L.dilation, L.groups, spat)
        convs.append(c); descs.append(d); Ws.append(W.double().numpy()); bs.append(b.double().numpy())
        spat = d.out_spatial
    stack = co.Stack(convs)
    assert stack.delay == 10
    ost = O.Stack(descs, Ws, bs, [int(L.relu) for L in cfg.layers], [1, 1, 1, 1, 0], cfg.n_streams)
    ys, refs = [], []
    for t in range(13):
        x = synth.frame(cfg, t)
        y = stack.forward_step(x)
        r = ost.forward_step(np_of(x))
        assert (y is None) == (r is None) == (t < 10)
        if y is not None:
            ys.append(np_of(y)); refs.append(r)
    y, ref = np.stack(ys), np.stack(refs).reshape(np.stack(ys).shape)
    assert rel_err(y, ref) <= 2e-2


STEM_CASES = ["stem_c4like", "stem_2parts", "stem_c2", "stem_wide", "stem_k3c5"]


@pytest.mark.parametrize("case", STEM_CASES)
def test_stem_equals_hbm_wcols_path(case):
    """The shared-memory W-im2col (MODE_STEM) feeds the tensor cores the same
    operands in the same K order as the HBM W-im2col pass, so both paths are
    bitwise equal -- and equal to the oracle in the integer regime."""
    _, ya, ref, _ = _run(case, seed=3)
    _, yb, _, _ = _run(case, seed=3, stem=False)
    assert np.array_equal(ya, yb)
    _, yi, ri, _ = _run(case, integer=True, seed=4)
    assert np.array_equal(yi, ri)


@pytest.mark.parametrize("B,H,W", [(48, 56, 56), (7, 112, 112)])
def test_stem_many_tiles_per_cta(B, H, W):
    """C4-stem shapes with several tiles per CTA (image / raw-row double
    buffers wrapping, the conversion one tile ahead): stem == HBM W-im2col
    path bit for bit over the delay and a few Ready ticks, and the pad step."""
    import paper_2204_03418_b200 as co
    d = O.Desc(2, 3, 64, (5, 7, 7), stride=(1, 2, 2), padding=(0, 3, 3), in_spatial=(H, W))
    rng = np.random.default_rng(B)
    Wt = torch.from_numpy(rng.standard_normal(d.w_shape) / 12).to(torch.bfloat16).cuda()
    bt = torch.from_numpy(rng.standard_normal(64) * 0.1).float().cuda()
    mk = lambda: co.Conv(3, 64, d.kernel, weight=Wt, bias=bt, stride=d.stride, padding=d.padding, in_spatial=(H, W),
                         n_streams=B, out_dtype=torch.float32, activation="relu")
    a = mk()
    with co.options(stem=0):
        b = mk()
    assert ",stem" in a.kernel_name and "wcols" in b.kernel_name
    g = torch.Generator(device="cuda").manual_seed(1)
    for t in range(7):
        x = co.channels_last(torch.randn((B, 3, H, W), generator=g, device="cuda").to(torch.bfloat16))
        ya, yb = a.forward_step(x), b.forward_step(x)
        assert (ya is None) == (yb is None)
        if ya is not None:
            assert torch.equal(ya, yb)
    ya, yb = a.forward_pad_step(), b.forward_pad_step()
    assert torch.equal(ya, yb)
    sa, _ = a.state_dict_stream()
    sb, _ = b.state_dict_stream()
    assert torch.equal(sa, sb)
