"""CUDA-graph step loops (co_stack_graph_create / co_graph_launch): a captured
run of ticks replayed as the stack's next ticks equals the eager fold of
co_stack_step bit for bit (same kernels, same clock-derived arguments), and
the clock rules that make it safe: a replay is refused unless every layer sits
at the captured phase (P:110-120 -- the schedule is a function of the host
clocks only)."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def _layers(specs, B, seed, out_last=torch.float32, layouts=None):
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(seed)
    convs, spat = [], None
    for l, (cin, cout, k, s, p, g, dil, H, W) in enumerate(specs):
        d = O.Desc(2, cin, cout, k, stride=s, padding=p, dilation=dil, groups=g, in_spatial=(H, W))
        Wt = torch.from_numpy(rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))).to(torch.bfloat16)
        bt = torch.from_numpy(rng.standard_normal(cout) * 0.1).float()
        last = l == len(specs) - 1
        convs.append(co.Conv(cin, cout, k, weight=Wt.cuda(), bias=bt.cuda(), stride=s, padding=p, dilation=dil,
                             groups=g, spatial_rank=2, in_spatial=(H, W),
                             n_streams=B, dtype=torch.bfloat16, out_dtype=out_last if last else torch.bfloat16,
                             activation=None if last else "relu",
                             state_layout=layouts[l] if layouts else "psum"))
    return convs


LAYOUTS = {"rawstem_khalo": ["auto", "psum"]}

STACKS = {
    # C2-shaped dense HALO pair -> depthwise temporal (the C3-b kernel): rings 2 and 4
    "dense_dw": ([(64, 64, (3, 3, 3), (1, 1, 1), (0, 1, 1), 1, (1, 1, 1), 12, 14),
                  (64, 64, (5, 1, 1), (1, 1, 1), (0, 0, 0), 64, (1, 1, 1), 12, 14)], 3),
    # C4 stem (W-im2col KLOOP) -> a strided KHALO layer
    "stem_khalo": ([(3, 64, (5, 7, 7), (1, 2, 2), (0, 3, 3), 1, (1, 1, 1), 20, 22),
                    (64, 128, (3, 3, 3), (1, 2, 2), (0, 1, 1), 1, (1, 1, 1), 10, 11)], 2),
    # the C4 stem over the planner's RAW frame ring (k_step_stem_raw) -> a strided KHALO layer
    "rawstem_khalo": ([(3, 64, (5, 7, 7), (1, 2, 2), (0, 3, 3), 1, (1, 1, 1), 20, 24),
                       (64, 128, (3, 3, 3), (1, 2, 2), (0, 1, 1), 1, (1, 1, 1), 10, 12)], 2),
    # C5-shaped FLAT pair, kt 9, dilation 2 (16 ring slots in two phase rings)
    "flat_c5": ([(256, 256, (9, 1, 1), (1, 1, 1), (0, 0, 0), 1, (2, 1, 1), 25, 1)], 8),
    # temporal stride 2 then a dense layer (Empty ticks inside the graph)
    "stride2": ([(32, 32, (3, 3, 3), (2, 1, 1), (1, 1, 1), 1, (1, 1, 1), 9, 10),
                 (32, 48, (3, 3, 3), (1, 1, 1), (0, 1, 1), 1, (1, 1, 1), 9, 10)], 2),
}


def _frames(n, B, cin, H, W, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    shp = (B, cin, H, W)
    import paper_2204_03418_b200 as co
    return [co.channels_last(torch.randn(shp, generator=g, device="cuda").to(torch.bfloat16)) for _ in range(n)]


@pytest.mark.parametrize("name", list(STACKS))
def test_graph_replay_equals_eager_fold(name):
    """Handle A steps eagerly; handle B (same weights) warms up eagerly, then
    replays one captured graph of 2 periods several times: every tick's Ready
    output, the ready count, the clocks and the final canonical state are
    bitwise equal."""
    import paper_2204_03418_b200 as co
    specs, B = STACKS[name]
    A = co.Stack(_layers(specs, B, 7, layouts=LAYOUTS.get(name)))
    Bs = co.Stack(_layers(specs, B, 7, layouts=LAYOUTS.get(name)))
    if name == "rawstem_khalo":
        assert "stem_raw" in A.layers[0].kernel_name, A.layers[0].kernel_name
    cin, H, W = specs[0][0], specs[0][7], specs[0][8]
    warm = max(c.receptive_field + c.info().padding_t for c in A.layers) * 3 + 8
    P = A.graph_period
    L = 2 * P
    reps = 3
    frames = _frames(warm + L * reps, B, cin, H, W, 3)
    last = A.layers[-1]
    shape = (B, last.out_channels) + last.out_spatial
    eager = []
    for t, x in enumerate(frames):
        y = A.forward_step(x)
        if t >= warm:
            eager.append(None if y is None else y.clone())
    for x in frames[:warm]:
        Bs.forward_step(x)
    ys = [co._empty_cl(shape, last.out_dtype, "cuda") for _ in range(L)]
    # the graph's frames are fixed buffers: copy each replay's frames in first
    xbuf = [torch.empty_like(frames[0]) for _ in range(L)]
    g = Bs.capture(xbuf, ys)
    assert g.n_ticks == L
    n0 = [c.n for c in Bs.layers]                      # capture moved no clock
    got = []
    for r in range(reps):
        for t in range(L):
            xbuf[t].copy_(frames[warm + r * L + t])
        nr = g.launch()
        torch.cuda.synchronize()
        ready = [y is not None for y in eager[r * L:(r + 1) * L]]
        assert nr == sum(ready)
        for t in range(L):
            got.append(ys[t].clone() if ready[t] else None)
    assert [c.n for c in Bs.layers] == [c.n for c in A.layers]
    assert [c.n - n for c, n in zip(Bs.layers, n0)] == [c.n - n for c, n in zip(A.layers, n0)]
    for a, b in zip(eager, got):
        assert (a is None) == (b is None)
        if a is not None:
            assert torch.equal(a, b)
    for ca, cb in zip(A.layers, Bs.layers):
        sa, _ = ca.state_dict_stream()
        sb, _ = cb.state_dict_stream()
        assert torch.equal(sa, sb)


def test_graph_from_a_clean_state_and_phase_checks():
    """A graph captured at n = 0 covers the delay once: its first replay is
    valid (the same n), a second is refused (n != n_cap and n_cap is inside
    the transient); a steady-state graph of one period replays repeatedly,
    but is refused one tick off phase."""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import _abi
    specs, B = STACKS["dense_dw"]
    S = co.Stack(_layers(specs, B, 1))
    A = co.Stack(_layers(specs, B, 1))
    cin, H, W = specs[0][0], specs[0][7], specs[0][8]
    frames = _frames(40, B, cin, H, W, 5)
    last = S.layers[-1]
    shape = (B, last.out_channels) + last.out_spatial
    ys = [co._empty_cl(shape, last.out_dtype, "cuda") for _ in range(12)]
    g0 = S.capture(frames[:12], ys)
    nr = g0.launch()
    ref = [A.forward_step(x) for x in frames[:12]]
    torch.cuda.synchronize()
    assert nr == sum(r is not None for r in ref) == 12 - S.delay
    assert torch.equal(ys[11], ref[11])
    with pytest.raises(_abi.CoError):
        g0.launch()                                     # clock 12 != 0, and 0 is inside the transient
    for x in frames[12:30]:
        S.forward_step(x)
    P = S.graph_period
    assert P == 4                                       # lcm(s R) = lcm(2, 4)
    g1 = S.capture(frames[30:30 + P], ys[:P])
    g1.launch()
    g1.launch()                                         # 4 ticks later: same phase
    S.forward_step(frames[0])
    with pytest.raises(_abi.CoError):
        g1.launch()                                     # one tick off
    torch.cuda.synchronize()


def test_graph_refused_while_a_stream_clean_is_pending():
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import _abi
    specs, B = STACKS["dense_dw"]
    S = co.Stack(_layers(specs, B, 2))
    cin, H, W = specs[0][0], specs[0][7], specs[0][8]
    frames = _frames(12, B, cin, H, W, 6)
    for x in frames[:8]:
        S.forward_step(x)
    S.clean_streams([1])
    last = S.layers[-1]
    ys = [co._empty_cl((B, last.out_channels) + last.out_spatial, last.out_dtype, "cuda") for _ in range(4)]
    with pytest.raises(_abi.CoError):
        S.capture(frames[:4], ys)
