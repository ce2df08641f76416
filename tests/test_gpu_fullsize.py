"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py
times (same stream counts, dispatch, kernels and grids):

* sampled streams (first, middle, last) against the fp64 oracle, element by
  element, over every Ready tick of a run that covers the whole delay;
* every stream, every layer: the step outputs equal the batch forward
  (co_forward, the CUDA-core direct kernel) of the frames that layer consumed
  -- Definition 1, a property that holds at any size;
* ready flags / clock identical to the oracle on every tick.

Tolerances (BASELINE.json north_star): fp32 C1 1e-4 RMS (test_gpu_direct.py);
bf16 inputs with fp32 accumulation 2e-2 RMS on fp32 outputs (A16).  Single
layers see exact bf16 inputs, so they are held to 1e-4.
"""
import numpy as np
import pytest
import torch

import oracle as O
from tests.helpers import reset_opt, set_opt, assert_bf16_rounding_bound, build_config_layers, np_of, rel_err

pytestmark = pytest.mark.gpu


def _stack_run(cfg, convs, T, keep):
    """Run T ticks of the layer chain; returns per-layer lists of (inputs, outputs)
    for all streams (on device) and the sampled final outputs."""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    ins = [[] for _ in convs]
    outs = [[] for _ in convs]
    ready = []
    for t in range(T):
        cur = synth.frame(cfg, t)
        r_all = True
        for l, c in enumerate(convs):
            if keep:
                ins[l].append(cur)
            y = c.forward_step(cur)
            if y is None:
                r_all = False
                break
            if keep:
                outs[l].append(y)
            cur = y
        ready.append(r_all)
    return ins, outs, ready


def _sampled(x, idx):
    return np_of(x[idx])


@pytest.mark.parametrize("cid,layout", [(2, "psum"), (3, "psum"), (4, "psum"), (5, "psum"),
                                        (3, "auto"), (5, "auto")])   # auto: the planner layouts bench.py times for C3 / C5
def test_fullsize_sampled_streams_vs_oracle(cid, layout):
    from paper_2204_03418_b200 import synth
    cfg = synth.config(cid)
    B = cfg.n_streams
    convs, descs, Ws, bs = build_config_layers(cfg, B, state_layout=layout)
    if layout == "auto":
        assert [c.state_layout for c in convs] == {3: ["raw", "raw"], 5: ["raw"]}[cid]
    d_nn = sum(d.delay for d in descs)
    # past the delay by two full turns of the largest ring (C5: its 16 slots,
    # both dilation phases), so every slot is written, completed and re-used
    R = max(d.ring_slots for d in descs)
    T = d_nn + 2 * R + 2
    # first, last and seeded picks (the oracle runs one thread per sampled stream);
    # C4's fp64 stack costs ~12 s per tick per stream, so it samples four
    n_pick = 2 if cid == 4 else 6
    idx = sorted({0, B - 1} | set(np.random.default_rng(cid).choice(np.arange(1, B - 1), n_pick, replace=False).tolist()))
    if len(convs) == 1:
        om = O.StepMachine(descs[0], Ws[0], bs[0], len(idx))
    else:
        om = O.Stack(descs, Ws, bs, [int(L.relu) for L in cfg.layers], [1] * (len(convs) - 1) + [0], len(idx))
    ys, refs = [], []
    for t in range(T):
        x = synth.frame(cfg, t)
        cur, ready = x, True
        for c in convs:
            cur = c.forward_step(cur)
            if cur is None:
                ready = False
                break
        r = om.forward_step(_sampled(x, idx))
        assert ready == (r is not None) == (t >= d_nn), (t, ready)
        if ready:
            ys.append(_sampled(cur, idx)); refs.append(r.reshape(ys[-1].shape))
    y, ref = np.stack(ys), np.stack(refs)
    assert len(ys) == T - d_nn
    tol = 1e-4 if len(convs) == 1 else 2e-2
    assert rel_err(y, ref) <= tol, rel_err(y, ref)


@pytest.mark.parametrize("cid", [2, 3, 4, 5])
def test_fullsize_step_equals_batch_all_streams(cid):
    """Every stream of every layer: step outputs == batch forward of the inputs
    that layer consumed, computed on the GPU by the direct kernel."""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    cfg = synth.config(cid)
    B = cfg.n_streams
    convs, descs, Ws, bs = build_config_layers(cfg, B)
    T = sum(d.delay for d in descs) + 2
    ins, outs, ready = _stack_run(cfg, convs, T, keep=True)
    for l, (c, d) in enumerate(zip(convs, descs)):
        if not outs[l]:
            continue
        # checker: the same layer (weights, bias, activation) on the direct CUDA-core kernel, fp32 out
        L = cfg.layers[l]
        (W, b) = synth.params(cfg)[l]
        chk = co.Conv(L.cin, L.cout, L.kernel, weight=W.cuda(), bias=b.cuda(), stride=L.stride, padding=L.padding,
                      dilation=L.dilation, groups=L.groups, spatial_rank=cfg.spatial_rank, in_spatial=c.in_spatial,
                      n_streams=B, dtype=cfg.dtype, out_dtype=torch.float32,
                      activation="relu" if L.relu else None, kernel="direct")
        clip = torch.stack(ins[l], dim=2)                      # (B, C, T_l, *S) channels-last per frame
        clip = co.channels_last(clip)
        yb = chk.forward(clip)                                 # (B, Cout, T'_l, *S')
        n = len(outs[l])
        ys = torch.stack(outs[l], dim=2).float()
        assert yb.shape[2] >= n
        yb = yb[:, :, :n].float()
        if c.out_dtype == torch.float32:
            err = (ys - yb).abs().max().item() / yb.pow(2).mean().sqrt().item()
            assert err <= 1e-4, (l, err)
        else:
            # bf16 emitted outputs: the RNE bound around the fp32 batch result
            eps = 1e-4 * yb.pow(2).mean().sqrt().item()
            excess = ((ys - yb).abs() - (2.0 ** -8 * (yb.abs() + eps) + eps)).max().item()
            assert excess <= 0, (l, excess)
        del chk, clip, yb, ys
        torch.cuda.empty_cache()


@pytest.mark.parametrize("cid,layer", [(2, 0), (3, 0), (3, 1)])
def test_fullsize_chunked_steps_equal_per_step_fold(cid, layer, monkeypatch):
    """At the full stream count and frame size: co_forward_steps through the
    chunked kernels (tcgen05 HALO for C2, k_steps_dw_t for C3-b) equals the
    per-step fold (CO_CHUNK=0) bit for bit (C3-a: the chunked K2 stencil) -- outputs, ready mask and the
    canonical state after the clip."""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    cfg = synth.config(cid)
    L = cfg.layers[layer]
    Wt, bt = synth.params(cfg)[layer]
    T = 7
    set_opt("chunk_st", "1")        # C3-a's chunked stencil is off by default; keep it covered
    g = torch.Generator(device="cuda").manual_seed(11)
    clip = co.channels_last(torch.randn((cfg.n_streams, L.cin, T) + tuple(cfg.in_spatial), generator=g,
                                        device="cuda").to(torch.bfloat16))
    res = {}
    for chunk in ("1", "0"):
        set_opt("chunk", chunk)
        conv = co.Conv(L.cin, L.cout, L.kernel, weight=Wt.cuda(), bias=bt.cuda(), stride=L.stride,
                       padding=L.padding, dilation=L.dilation, groups=L.groups, spatial_rank=cfg.spatial_rank,
                       in_spatial=tuple(cfg.in_spatial), n_streams=cfg.n_streams, dtype=cfg.dtype,
                       out_dtype=torch.float32)
        ys, mask = conv.forward_steps(clip)
        st, _ = conv.state_dict_stream()
        torch.cuda.synchronize()
        res[chunk] = (ys, mask, st)
        del conv
    (ya, ma, sa), (yb, mb, sb) = res["1"], res["0"]
    assert torch.equal(ma, mb) and int(ma.sum()) == T - (L.kernel[0] - 1)
    assert torch.equal(ya, yb)
    assert torch.equal(sa, sb)


def test_fullsize_k2s_pipeline_repeats_equal_k2():
    """Race detector for the K2s stage pipeline at the full C3-a size (512
    streams: ~29 K units per launch): three per-step folds through k_step_dw_seg
    equal the per-thread-load K2 (dw_seg = 0) bit for bit -- outputs and final
    state.  (Before every consumer warp waited on every stage's barrier in order,
    a group could pass a parity wait one phase early: one corrupted unit in ~1e5,
    in a different stream on every run.)"""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    cfg = synth.config(3)
    L = cfg.layers[0]
    Wt, bt = synth.params(cfg)[0]
    T = 6
    set_opt("chunk", 0)
    g = torch.Generator(device="cuda").manual_seed(23)
    clip = co.channels_last(torch.randn((cfg.n_streams, L.cin, T) + tuple(cfg.in_spatial), generator=g,
                                        device="cuda").to(torch.bfloat16))

    def run(seg):
        set_opt("dw_seg", seg)
        conv = co.Conv(L.cin, L.cout, L.kernel, weight=Wt.cuda(), bias=bt.cuda(), stride=L.stride,
                       padding=L.padding, dilation=L.dilation, groups=L.groups, spatial_rank=cfg.spatial_rank,
                       in_spatial=tuple(cfg.in_spatial), n_streams=cfg.n_streams, dtype=cfg.dtype,
                       out_dtype=torch.float32)
        assert conv.kernel_name.startswith("k_step_dw_seg" if seg else "k_step_dw_st"), conv.kernel_name
        ys, _ = conv.forward_steps(clip)
        st, _ = conv.state_dict_stream()
        torch.cuda.synchronize()
        return ys, st

    y0, s0 = run(0)
    for rep in range(3):
        y1, s1 = run(1)
        assert torch.equal(y1, y0), (rep, int((y1 != y0).sum()))
        assert torch.equal(s1, s0), rep
        del y1, s1


def test_fullsize_raw_stencil_pipeline_all_streams_equal_plain_raw_kernel():
    """All 512 streams of C3-a over the RAW frame ring: the rolling-row pipeline
    (k_step_dw_rowraw, frame store fused) against the plain per-thread-load RAW
    kernel (dw_seg = 0: k_step_dw_raw after a frame copy) -- outputs within fp32
    summation-order noise (1e-5 of the RMS; a mis-synchronised stage would be off
    by O(1)), the frame rings bit for bit; three repeats (race detector)."""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    cfg = synth.config(3)
    L = cfg.layers[0]
    Wt, bt = synth.params(cfg)[0]
    T = 6
    set_opt("chunk", 0)
    g = torch.Generator(device="cuda").manual_seed(29)
    clip = co.channels_last(torch.randn((cfg.n_streams, L.cin, T) + tuple(cfg.in_spatial), generator=g,
                                        device="cuda").to(torch.bfloat16))

    def run(seg):
        set_opt("dw_seg", seg)
        conv = co.Conv(L.cin, L.cout, L.kernel, weight=Wt.cuda(), bias=bt.cuda(), stride=L.stride,
                       padding=L.padding, dilation=L.dilation, groups=L.groups, spatial_rank=cfg.spatial_rank,
                       in_spatial=tuple(cfg.in_spatial), n_streams=cfg.n_streams, dtype=cfg.dtype,
                       out_dtype=torch.float32, state_layout="raw")
        assert conv.kernel_name.startswith("k_step_dw_rowraw" if seg else "k_step_dw_raw"), conv.kernel_name
        ys, _ = conv.forward_steps(clip)
        st, _ = conv.state_dict_stream()
        torch.cuda.synchronize()
        return ys, st

    y0, s0 = run(0)
    rms = y0.pow(2).mean().sqrt().item()
    for rep in range(3):
        y1, s1 = run(1)
        assert (y1 - y0).abs().max().item() <= 1e-5 * rms, rep
        assert torch.equal(s1, s0), rep
        del y1, s1


def _sample_streams(B):
    return sorted({0, B // 2, B - 1})


@pytest.mark.parametrize("name", ["x3d64", "max3"])
def test_fullsize_pooling_sampled_streams_vs_oracle(name):
    """scripts/bench_pool.py's workloads at their full stream counts, in the
    bench's launch configuration: sampled streams against the fp64 pooling
    oracle (MAX exact; AVG within 1e-4 of the RMS on fp32 outputs)."""
    import paper_2204_03418_b200 as co
    from oracle import pool as OP
    import scripts.bench_pool as bp
    w = bp.WORKLOADS[name]
    B, C, H, W = w["B"], w["C"], w["H"], w["W"]
    p = co.Pool(w["kind"], C, w["kernel"], stride=w["stride"], padding=w["padding"], in_spatial=(H, W), n_streams=B,
                out_dtype=torch.float32)
    assert p.kernel_name == co.Pool(w["kind"], C, w["kernel"], stride=w["stride"], padding=w["padding"],
                                    in_spatial=(H, W), n_streams=B).kernel_name
    sb = _sample_streams(B)
    sms = {b: OP.PoolStep(w["kind"], C, (H, W), w["kernel"], w["stride"], w["padding"], (1, 1, 1), B=1) for b in sb}
    g = torch.Generator(device="cuda").manual_seed(3)
    n_ready = 0
    for t in range(p.delay + 3):
        x = co.channels_last(torch.randn((B, C, H, W), generator=g, device="cuda").to(torch.bfloat16))
        y = p.forward_step(x)
        for b in sb:
            r = sms[b].forward_step(np_of(x[b:b + 1]))
            assert (y is None) == (r is None)
            if y is not None:
                got = np_of(y[b:b + 1])
                if w["kind"] == "max":
                    np.testing.assert_array_equal(got, r.reshape(got.shape))
                else:
                    assert rel_err(got, r.reshape(got.shape)) <= 1e-4
        n_ready += y is not None
    assert n_ready == 3


def test_fullsize_pool_row_pipeline_all_streams_equal_band_kernel():
    """All 256 streams of the max3 workload: the bulk-copy row pipeline
    (k_step_pool_seg) against the band kernel (pool_seg = 0), bit for bit on
    every output of every Ready step; three repeats (race detector)."""
    import paper_2204_03418_b200 as co
    import scripts.bench_pool as bp
    w = bp.WORKLOADS["max3"]
    B, C, H, W = w["B"], w["C"], w["H"], w["W"]
    g = torch.Generator(device="cuda").manual_seed(31)
    frames = [co.channels_last(torch.randn((B, C, H, W), generator=g, device="cuda").to(torch.bfloat16)) for _ in range(5)]

    def run(seg):
        set_opt("pool_seg", seg)
        p = co.Pool(w["kind"], C, w["kernel"], stride=w["stride"], padding=w["padding"], in_spatial=(H, W), n_streams=B)
        assert ("pool_seg" in p.kernel_name) == bool(seg), p.kernel_name
        ys = [p.forward_step(x) for x in frames]
        torch.cuda.synchronize()
        return [y.clone() for y in ys if y is not None]

    ref = run(0)
    assert len(ref) == 3
    for rep in range(3):
        got = run(1)
        assert len(got) == len(ref)
        for a, b in zip(got, ref):
            assert torch.equal(a, b), rep


def test_fullsize_mha_sampled_streams_vs_oracle():
    """scripts/bench_mha.py's workload (E=1024, 16 heads, window 64, 1024
    streams): sampled streams against the fp64 MHA oracle at the bf16 bar."""
    import paper_2204_03418_b200 as co
    from oracle import mha as OM
    B, E, H, n = 1024, 1024, 16, 64
    rng = np.random.default_rng(4)
    p = {"heads": H}
    for k in ("Wq", "Wk", "Wv", "Wo"):
        p[k] = torch.from_numpy(rng.standard_normal((E, E)) / np.sqrt(E)).to(torch.bfloat16).double().numpy()
    for k in ("bq", "bk", "bv", "bo"):
        p[k] = torch.from_numpy(rng.standard_normal(E) * 0.1).float().double().numpy()
    m = co.MultiheadAttention(E, H, n, n_streams=B, out_dtype=torch.float32,
                              in_proj_weight=torch.from_numpy(np.concatenate([p["Wq"], p["Wk"], p["Wv"]])),
                              in_proj_bias=torch.from_numpy(np.concatenate([p["bq"], p["bk"], p["bv"]])),
                              out_proj_weight=torch.from_numpy(p["Wo"]), out_proj_bias=torch.from_numpy(p["bo"]))
    sb = _sample_streams(B)
    sms = {b: OM.MhaStep(p, n, 1) for b in sb}
    g = torch.Generator(device="cuda").manual_seed(5)
    for t in range(n + 2):
        x = torch.randn((B, E), generator=g, device="cuda").to(torch.bfloat16)
        y = m.forward_step(x)
        for b in sb:
            r = sms[b].forward_step(np_of(x[b:b + 1]))
            assert (y is None) == (r is None)
            if y is not None:
                assert rel_err(np_of(y[b:b + 1]), r) <= 2e-2


def test_fullsize_mha_ring_pipeline_all_streams_vs_per_lane_kernel():
    """All 1024 streams of the MHA workload: the ring-pipeline attention
    (k_mha_attend_ring) against the per-lane-load kernel (mha_ring = 0) on the
    same weights and inputs.  Both read the same bf16 q / k / v, so every
    stream's outputs agree to bf16 last-place effects of the attention output
    (held per stream to 2e-2 of the RMS; a mis-synchronised stage would put one
    stream off by O(1)); the K / V rings afterwards are equal bit for bit."""
    import paper_2204_03418_b200 as co
    B, E, H, n = 1024, 1024, 16, 64
    g = torch.Generator(device="cuda").manual_seed(41)
    w_in = torch.randn((3 * E, E), generator=g, device="cuda") / E ** 0.5
    w_out = torch.randn((E, E), generator=g, device="cuda") / E ** 0.5
    xs = [torch.randn((B, E), generator=g, device="cuda").to(torch.bfloat16) for _ in range(n + 3)]

    def run(ring):
        set_opt("mha_ring", ring)
        m = co.MultiheadAttention(E, H, n, n_streams=B, out_dtype=torch.float32, in_proj_weight=w_in,
                                  out_proj_weight=w_out, in_proj_bias=torch.zeros(3 * E, device="cuda"),
                                  out_proj_bias=torch.zeros(E, device="cuda"))
        ys = [m.forward_step(x) for x in xs]
        st, cnt = m.state_dict_stream()
        torch.cuda.synchronize()
        return torch.stack([y for y in ys if y is not None]), st

    y0, s0 = run(0)
    assert y0.shape[0] == 4
    rms = y0.pow(2).mean().sqrt().item()
    for rep in range(2):
        y1, s1 = run(1)
        per_stream = (y1 - y0).abs().amax(dim=(0, 2))
        assert per_stream.max().item() <= 2e-2 * rms, (rep, int(per_stream.argmax()))
        assert torch.equal(s1, s0), rep
