"""GPU tests of per-stream clocks (include/co.h
co_state_clean_streams / co_stream_ready): streams restarted mid-run behave
exactly like fresh streams -- their flags follow their own step count
(n_b >= d, Principle 2 / S:73) and their outputs match a fresh fp64 oracle fed
only their frames since the join -- while the other streams continue
untouched.  Covered for every kernel family and state layout (dense HALO and
FLAT tensor-core, direct fp32, both depthwise kernels, the RAW ring, MAX/AVG
pooling with and without the block decomposition, Delay), for a temporal
stride of 2 (joins only on n = 0 mod s), and for a stack, where each layer
cleans the stream when its first valid input arrives."""
import numpy as np
import pytest
import torch

import oracle as O
from oracle import compose as OC
from oracle import pool as OP
from tests.helpers import reset_opt, set_opt, np_of, rel_err, to_cl

pytestmark = pytest.mark.gpu


def _bf16(a):
    return torch.from_numpy(np.asarray(a, np.float64)).to(torch.bfloat16).double().numpy()


def _conv_case(d, B, dtype, kernel, state_layout, rng):
    import paper_2204_03418_b200 as co
    W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    b = rng.standard_normal(d.cout) * 0.1
    Wt = torch.from_numpy(W).to(dtype)
    bt = torch.from_numpy(b).float()
    h = co.Conv(d.cin, d.cout, d.kernel, weight=Wt.cuda(), bias=bt.cuda(), stride=d.stride, padding=d.padding,
                dilation=d.dilation, groups=d.groups, spatial_rank=d.spatial_rank, in_spatial=d.in_spatial,
                n_streams=B, dtype=dtype, out_dtype=torch.float32, kernel=kernel, state_layout=state_layout)
    Wq, bq = Wt.double().numpy(), bt.double().numpy()
    H, Wd = d.in_hw
    shape = (d.cin,) + ((H,) if d.spatial_rank >= 1 else ()) + ((Wd,) if d.spatial_rank >= 2 else ())
    return h, (lambda: O.StepMachine(d, Wq, bq, 1)), shape, (lambda r: r.reshape(r.shape))


CASES = {
    "dense_halo": lambda rng, B: _conv_case(O.Desc(2, 32, 32, (3, 3, 3), padding=(0, 1, 1), in_spatial=(6, 7)), B,
                                            torch.bfloat16, "dense_tc", "psum", rng),
    "dense_flat_dil": lambda rng, B: _conv_case(O.Desc(1, 64, 64, (5, 1), dilation=(2, 1), in_spatial=(9,)), B,
                                                torch.bfloat16, "dense_tc", "psum", rng),
    "direct_f32": lambda rng, B: _conv_case(O.Desc(2, 4, 8, (3, 3, 3), padding=(1, 1, 1), in_spatial=(5, 5)), B,
                                            torch.float32, "direct", "psum", rng),
    "depthwise_st": lambda rng, B: _conv_case(O.Desc(2, 32, 32, (3, 3, 3), padding=(0, 1, 1), groups=32,
                                                     in_spatial=(6, 6)), B, torch.bfloat16, "depthwise", "psum", rng),
    "depthwise_t": lambda rng, B: _conv_case(O.Desc(2, 32, 32, (5, 1, 1), groups=32, in_spatial=(4, 5)), B,
                                             torch.bfloat16, "depthwise", "psum", rng),
    # KHALO (weights streamed, stride-2 phase halos): the tile-padded state under per-stream clean masks
    "dense_khalo_s2": lambda rng, B: _conv_case(O.Desc(2, 128, 64, (3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1),
                                                       in_spatial=(8, 10)), B, torch.bfloat16, "dense_tc", "psum", rng),
    "raw_dense": lambda rng, B: _conv_case(O.Desc(2, 32, 32, (3, 3, 3), padding=(1, 1, 1), in_spatial=(5, 6)), B,
                                           torch.bfloat16, "auto", "raw", rng),
}


def _pool_case(kind, kernel, padding, vh, monkeypatch):
    def make(rng, B):
        import paper_2204_03418_b200 as co
        set_opt("pool_vh", vh)
        C, H, W = 16, 5, 6
        h = co.Pool(kind, C, kernel, padding=padding, in_spatial=(H, W), n_streams=B, out_dtype=torch.float32)
        return h, (lambda: OP.PoolStep(kind, C, (H, W), kernel, (1, 1, 1), padding, (1, 1, 1), B=1)), (C, H, W), None
    return make


def _delay_case(rng, B):
    import paper_2204_03418_b200 as co
    h = co.Delay(2, 8, in_spatial=(3, 4), n_streams=B)
    return h, (lambda: OC.DelayStep(2)), (8, 3, 4), None


def _run_join(h, fresh, shape, dtype, rng, B=4, before=6, after=11, join=(1, 3)):
    """Step all streams, restart `join` after `before` ticks, and compare every
    stream with its own oracle (fresh ones for the joined streams)."""
    machines = [fresh() for _ in range(B)]
    for t in range(before + after):
        if t == before:
            h.clean_streams(list(join))
            for b in join:
                machines[b] = fresh()
        xs = [_bf16(rng.standard_normal((1,) + shape)) for _ in range(B)]
        x = to_cl(np.concatenate(xs, axis=0), dtype)
        y = h.forward_step(x)
        flags = h.stream_ready()
        for b in range(B):
            r = machines[b].forward_step(xs[b])
            assert bool(flags[b]) == (r is not None), (t, b)
            if r is not None:
                assert y is not None
                got = np_of(y[b:b + 1])
                if np.isinf(r).any():
                    np.testing.assert_array_equal(got, r.reshape(got.shape))
                else:
                    assert rel_err(got, r.reshape(got.shape)) <= 1e-4, (t, b)


@pytest.mark.parametrize("name", list(CASES))
def test_clean_streams_conv_layouts(name):
    rng = np.random.default_rng(sum(map(ord, name)))
    h, fresh, shape, _ = CASES[name](rng, 4)
    _run_join(h, fresh, shape, h.dtype, rng)


@pytest.mark.parametrize("kind,kernel,padding,vh", [
    ("max", (3, 3, 3), (0, 1, 1), "0"), ("avg", (3, 3, 3), (2, 1, 1), "0"),
    ("max", (7, 3, 3), (3, 1, 1), "1"), ("avg", (7, 2, 2), (0, 0, 0), "1")])
def test_clean_streams_pooling(kind, kernel, padding, vh, monkeypatch):
    rng = np.random.default_rng(11)
    h, fresh, shape, _ = _pool_case(kind, kernel, padding, vh, monkeypatch)(rng, 4)
    _run_join(h, fresh, shape, torch.bfloat16, rng, before=9, after=14)


def test_clean_streams_delay():
    rng = np.random.default_rng(12)
    h, fresh, shape, _ = _delay_case(rng, 4)
    _run_join(h, fresh, shape, torch.bfloat16, rng)


def test_clean_streams_temporal_stride_two():
    from paper_2204_03418_b200._abi import CoError
    rng = np.random.default_rng(13)
    d = O.Desc(2, 8, 8, (3, 3, 3), stride=(2, 1, 1), padding=(1, 1, 1), in_spatial=(4, 4))
    h, fresh, shape, _ = _conv_case(d, 4, torch.bfloat16, "auto", "psum", rng)
    x = to_cl(_bf16(rng.standard_normal((4,) + shape)), torch.bfloat16)
    h.forward_step(x)
    with pytest.raises(CoError):          # n = 1: a join here would shift the stream's Ready phase
        h.clean_streams([0])
    h.clean_state()
    _run_join(h, fresh, shape, torch.bfloat16, rng, before=6, after=12)


def test_clean_streams_in_a_stack():
    """Stream 2 restarts mid-run in a 2-layer stack: layer 1 cleans it only when
    layer 0 first emits a valid output for it, so the stream's outputs match a
    fresh oracle stack; the others are undisturbed."""
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(14)
    B, H, W = 4, 5, 6
    d0 = O.Desc(2, 16, 32, (3, 3, 3), padding=(0, 1, 1), in_spatial=(H, W))
    d1 = O.Desc(2, 32, 32, (3, 3, 3), padding=(0, 1, 1), groups=32, in_spatial=(H, W))
    Ws = [_bf16(rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))) for d in (d0, d1)]
    bs = [torch.from_numpy(rng.standard_normal(32) * 0.1).float().double().numpy() for _ in range(2)]
    l0 = co.Conv(16, 32, (3, 3, 3), weight=torch.from_numpy(Ws[0]).to(torch.bfloat16).cuda(),
                 bias=torch.from_numpy(bs[0]).float().cuda(), padding=(0, 1, 1), in_spatial=(H, W), n_streams=B,
                 activation="relu")
    l1 = co.Conv(32, 32, (3, 3, 3), weight=torch.from_numpy(Ws[1]).to(torch.bfloat16).cuda(),
                 bias=torch.from_numpy(bs[1]).float().cuda(), padding=(0, 1, 1), groups=32, in_spatial=(H, W),
                 n_streams=B, out_dtype=torch.float32)
    st = co.Stack([l0, l1])
    fresh = lambda: O.Stack([d0, d1], Ws, bs, [1, 0], [1, 0], 1)
    machines = [fresh() for _ in range(B)]
    for t in range(16):
        if t == 6:
            st.clean_streams([2])
            machines[2] = fresh()
        xs = [_bf16(rng.standard_normal((1, 16, H, W))) for _ in range(B)]
        y = st.forward_step(to_cl(np.concatenate(xs), torch.bfloat16))
        flags = st.stream_ready()
        for b in range(B):
            r = machines[b].forward_step(xs[b])
            assert bool(flags[b]) == (r is not None), (t, b)
            if r is not None:   # bf16 inter-layer activations: the stacks' bf16 bar (A16)
                assert rel_err(np_of(y[b:b + 1]), r) <= 2e-2, (t, b)
