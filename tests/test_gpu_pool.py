"""GPU parity of continual pooling (
SPEC.md:252-297) through the C ABI (co_op MAX / AVG) against the fp64 pooling
oracle (oracle/pool.py): step outputs and readiness, batch forward, the
forward_steps fold with pad_end == batch (Definition 1), the state
contract (co_state_get == oracle history with -inf pads for MAX, get->set round
trip, update_state=0 purity), stacking with convolutions, and error codes.

Tolerances: MAX is exact (a max of representable values; fp32 accumulation of
bf16 inputs is exact), so MAX compares bit for bit; AVG is an fp32 sum of at
most kt kh kw terms times 1/(kt kh kw): fp32 outputs within 1e-4 of the RMS,
bf16 outputs within one bf16 rounding (tests/helpers.assert_bf16_rounding_bound).
"""
import numpy as np
import pytest
import torch

from oracle import pool as OP
from tests.helpers import reset_opt, set_opt, assert_bf16_rounding_bound, np_of, rel_err

pytestmark = pytest.mark.gpu


def _tcl(x: np.ndarray, dtype) -> torch.Tensor:
    import paper_2204_03418_b200 as co
    return co.channels_last(torch.from_numpy(np.ascontiguousarray(x)).to(dtype).cuda())


def _quant(x: np.ndarray, dtype) -> np.ndarray:
    return torch.from_numpy(x).to(dtype).double().numpy()


def _spatial(rank, H, W):
    return ((H,) if rank >= 1 else ()) + ((W,) if rank >= 2 else ())


def rand_pool(rng):
    rank = int(rng.integers(0, 3))
    kt = int(rng.integers(1, 5))
    dt = int(rng.integers(1, 3))
    f = dt * (kt - 1) + 1
    kh = int(rng.integers(1, 4)) if rank >= 1 else 1
    kw = int(rng.integers(1, 4)) if rank >= 2 else 1
    st = (int(rng.integers(1, 3)), int(rng.integers(1, 3)) if rank >= 1 else 1, int(rng.integers(1, 3)) if rank >= 2 else 1)
    pad = (int(rng.integers(0, f)), int(rng.integers(0, kh)), int(rng.integers(0, kw)))
    dil = (dt, int(rng.integers(1, 3)) if rank >= 1 else 1, 1)
    H = int(rng.integers(dil[1] * (kh - 1) + 1, 7)) if rank >= 1 else 1
    W = int(rng.integers(kw, 7)) if rank >= 2 else 1
    C = int(rng.choice([1, 2, 3, 4, 8, 16, 24]))
    return rank, (kt, kh, kw), st, pad, dil, H, W, C


def _make(kind, rank, kernel, stride, pad, dil, H, W, C, B, dtype, out_dtype):
    import paper_2204_03418_b200 as co
    n = rank + 1
    p = co.Pool(kind, C, kernel[:n], stride=stride[:n], padding=pad[:n], dilation=dil[:n], spatial_rank=rank,
                in_spatial=(H, W)[:rank] or (1,), n_streams=B, dtype=dtype, out_dtype=out_dtype)
    sm = OP.PoolStep(kind, C, (H, W), kernel, stride, pad, dil, B=B)
    return p, sm


def _compare(kind, y, ref, out_dtype):
    if kind == "max":
        np.testing.assert_array_equal(y, ref)
    elif out_dtype == torch.bfloat16:
        assert_bf16_rounding_bound(y, ref)
    else:
        assert rel_err(y, ref) <= 1e-4


@pytest.fixture(params=[("auto", None), ("1", "0"), ("3", "0"), ("1", "1"), ("3", "1"), ("1b", "0"), ("1s", "0")],
                ids=["auto", "G1_fold", "G3_fold", "G1_vh", "G3_vh", "G1_fold_noband", "G1_fold_noseg"])
def pool_lanes(request, monkeypatch):
    """Step-kernel variant (k_pool.cu): AUTO, or forced lanes (CO_POOL_G: 1 =
    plain kernel, 3 = split kernel) x temporal scheme (CO_POOL_VH: 0 = direct
    fold of the ring, 1 = block decomposition).  Returns "exact" when the
    variant reduces in the batch kernel's order (AVG bitwise step == batch)."""
    G, vh = request.param
    if G == "1b":                                  # the plain kernel without the row-band staging
        G = "1"
        set_opt("pool_band", "0")
        set_opt("pool_seg", "0")
    if G == "1s":                                  # the band kernel instead of the bulk-copy row pipeline
        G = "1"
        set_opt("pool_seg", "0")
    if G != "auto":
        set_opt("pool_g", G)
        set_opt("pool_vh", vh)
    return "exact" if (G, vh) == ("1", "0") else "reordered"


@pytest.mark.parametrize("seed", range(20))
@pytest.mark.parametrize("kind", ["max", "avg"])
def test_pool_step_random_vs_oracle(kind, seed, pool_lanes):
    rng = np.random.default_rng(500 + seed)
    rank, kernel, stride, pad, dil, H, W, C = rand_pool(rng)
    B = int(rng.integers(1, 4))
    dtype = torch.bfloat16 if seed % 2 else torch.float32
    out_dtype = torch.float32 if seed % 4 < 2 else dtype
    p, sm = _make(kind, rank, kernel, stride, pad, dil, H, W, C, B, dtype, out_dtype)
    assert p.kernel_used == "pool" and p.delay == sm.delay
    shp = (B, C) + _spatial(rank, H, W)
    f = sm.f
    for t in range(f + 2 * stride[0] + 3):
        xq = _quant(rng.standard_normal(shp), dtype)
        y = p.forward_step(_tcl(xq, dtype))
        r = sm.forward_step(xq.reshape(B, C, H, W))
        assert (y is None) == (r is None), t
        assert p.n == sm.n
        if y is not None:
            _compare(kind, np_of(y).reshape(r.shape), r, out_dtype)
    # pad_end steps (x = None): padding, -inf for MAX
    for _ in range(pad[0]):
        y = p.forward_pad_step()
        r = sm.forward_step(None)
        assert (y is None) == (r is None)
        if y is not None:
            _compare(kind, np_of(y).reshape(r.shape), r, out_dtype)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("kind", ["max", "avg"])
def test_pool_forward_and_fold_vs_oracle(kind, seed, pool_lanes):
    rng = np.random.default_rng(700 + seed)
    rank, kernel, stride, pad, dil, H, W, C = rand_pool(rng)
    B = int(rng.integers(1, 3))
    dtype = torch.bfloat16 if seed % 2 else torch.float32
    p, _ = _make(kind, rank, kernel, stride, pad, dil, H, W, C, B, dtype, torch.float32)
    f = dil[0] * (kernel[0] - 1) + 1
    T = int(rng.integers(max(1, f - 2 * pad[0]), f + 7))
    xq = _quant(rng.standard_normal((B, C, T) + _spatial(rank, H, W)), dtype)
    ref = OP.pool_forward(kind, xq.reshape(B, C, T, H, W), kernel, stride, pad, dil)
    yb = p.forward(_tcl(xq, dtype))
    _compare(kind, np_of(yb).reshape(ref.shape), ref, torch.float32)
    ys, mask = p.forward_steps(_tcl(xq, dtype), pad_end=True)
    assert int(mask.sum()) == ref.shape[2]
    if kind == "max" or pool_lanes == "exact":
        assert torch.equal(ys, yb)                  # same reduction order: bitwise (Definition 1)
    else:                                           # split lanes / block decomposition: another order
        assert rel_err(np_of(ys), np_of(yb)) <= 1e-6


@pytest.mark.parametrize("kind", ["max", "avg"])
def test_pool_state_contract(kind, pool_lanes):
    rng = np.random.default_rng(9)
    B, C, H, W = 2, 16, 5, 6
    kernel, stride, pad, dil = (3, 3, 3), (1, 2, 2), (2, 1, 1), (1, 1, 1)
    p, sm = _make(kind, 2, kernel, stride, pad, dil, H, W, C, B, torch.bfloat16, torch.float32)
    frames = [_quant(rng.standard_normal((B, C, H, W)), torch.bfloat16) for _ in range(7)]
    for x in frames[:1]:
        p.forward_step(_tcl(x, torch.bfloat16)); sm.forward_step(x)
    # canonical state == the oracle history reduced over the spatial window
    # (include/co.h co_op); start padding is -inf for MAX, 0 for AVG
    st, meta = p.state_dict_stream()
    assert st.dtype == (torch.bfloat16 if kind == "max" else torch.float32)
    got = np.moveaxis(np_of(st), -1, 2)
    exp = sm.reduced_history()
    if kind == "max":
        np.testing.assert_array_equal(got, exp)
    else:
        assert rel_err(got, exp) <= 1e-6
    # update_state=False: output from the current state, state bitwise unchanged
    y0 = p.forward_step(_tcl(frames[1], torch.bfloat16), update_state=False)
    r0 = sm.forward_step(frames[1], update_state=False)
    _compare(kind, np_of(y0), r0, torch.float32)
    st2, _ = p.state_dict_stream()
    assert torch.equal(st, st2) and p.n == 1
    # round trip: continue from a restored copy in a second handle
    q, _ = _make(kind, 2, kernel, stride, pad, dil, H, W, C, B, torch.bfloat16, torch.float32)
    q.load_state_stream(st, meta)
    for x in frames[1:]:
        a = p.forward_step(_tcl(x, torch.bfloat16))
        b = q.forward_step(_tcl(x, torch.bfloat16))
        r = sm.forward_step(x)
        assert (a is None) == (b is None) == (r is None)
        if a is not None:
            assert torch.equal(a, b)
            _compare(kind, np_of(a), r, torch.float32)
    # clean state restores the padding value
    p.clean_state()
    st3, _ = p.state_dict_stream()
    expect = float("-inf") if kind == "max" else 0.0
    assert bool((st3.float() == expect).all())


def test_pool_in_stack_with_convs():
    """conv -> max pool -> conv as one co_stack: the stack step equals the
    layer-by-layer fold, and the pool's Ready outputs gate the next layer."""
    import paper_2204_03418_b200 as co
    rng = np.random.default_rng(4)
    B, C, H, W = 2, 32, 6, 6
    w1 = torch.from_numpy(rng.standard_normal((C, C, 3, 3, 3)) / 16).to(torch.bfloat16).cuda()
    w2 = torch.from_numpy(rng.standard_normal((C, C, 1, 1, 1)) / 6).to(torch.bfloat16).cuda()
    mk = lambda: [co.Conv(C, C, (3, 3, 3), weight=w1, padding=(0, 1, 1), in_spatial=(H, W), n_streams=B),
                  co.Pool("max", C, (2, 3, 3), stride=(2, 2, 2), padding=(0, 1, 1), in_spatial=(H, W), n_streams=B),
                  co.Conv(C, C, (1, 1, 1), weight=w2, in_spatial=(3, 3), n_streams=B, out_dtype=torch.float32)]
    layers = mk()
    st = co.Stack(layers)
    ref_layers = mk()
    for t in range(9):
        x = _tcl(rng.standard_normal((B, C, H, W)), torch.bfloat16)
        y = st.forward_step(x)
        cur = x
        for L in ref_layers:
            cur = L.forward_step(cur)
            if cur is None:
                break
        assert (y is None) == (cur is None), t
        if y is not None:
            assert torch.equal(y, cur)


def test_pool_errors():
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200._abi import CoError
    with pytest.raises(CoError):      # temporal padding > f-1
        co.Pool("avg", 8, (3, 1, 1), padding=(3, 0, 0), in_spatial=(2, 2))
    with pytest.raises(ValueError):
        co.Pool("sum", 8, (3, 1, 1), in_spatial=(2, 2))


@pytest.mark.parametrize("kind", ["avg", "max"])
def test_expanded_global_pool_kt64(kind, pool_lanes):
    """The paper's expanded temporal global average pooling ("64
    steps"): kernel (64, 7, 7) over 7x7 frames -- kt above CO_MAX_KT, ring
    slots computed on the device."""
    rng = np.random.default_rng(64)
    B, C, H, W = 3, 48, 7, 7
    p, sm = _make(kind, 2, (64, 7, 7), (1, 1, 1), (0, 0, 0), (1, 1, 1), H, W, C, B, torch.bfloat16, torch.float32)
    assert p.delay == 63 and p.receptive_field == 64 and p.out_spatial == (1, 1)
    ys, refs = [], []
    for t in range(70):
        xq = _quant(rng.standard_normal((B, C, H, W)), torch.bfloat16)
        y = p.forward_step(_tcl(xq, torch.bfloat16))
        r = sm.forward_step(xq)
        assert (y is None) == (r is None)
        if y is not None:
            ys.append(np_of(y).reshape(r.shape)); refs.append(r)
    assert len(ys) == 7
    _compare(kind, np.stack(ys), np.stack(refs), torch.float32)


@pytest.mark.parametrize("kind", ["avg", "max"])
def test_block_decomposition_state_round_trip(kind, monkeypatch):
    """Block decomposition with dilation 2 (two phases), temporal stride 2 and
    padding: snapshot the state at ticks across a whole block cycle, restore it
    into a fresh handle (co_state_set rebuilds P and S from the ring) and run it
    ahead: its outputs match the oracle continued from the same point and are
    bitwise those the uninterrupted handle later produces."""
    import copy
    set_opt("pool_vh", "1")
    rng = np.random.default_rng(77)
    B, C, H, W = 2, 16, 4, 5
    kernel, stride, pad, dil = (7, 2, 2), (2, 1, 1), (5, 0, 1), (2, 1, 1)
    p, sm = _make(kind, 2, kernel, stride, pad, dil, H, W, C, B, torch.bfloat16, torch.float32)
    assert "vh" in p.kernel_name
    frames = [_quant(rng.standard_normal((B, C, H, W)), torch.bfloat16) for _ in range(44)]
    ahead = {}                                      # frame index -> outputs of restored handles
    for t, x in enumerate(frames):
        if t % 3 == 1 and t + 8 <= len(frames):
            st, meta = p.state_dict_stream()
            q, _ = _make(kind, 2, kernel, stride, pad, dil, H, W, C, B, torch.bfloat16, torch.float32)
            q.load_state_stream(st, meta)
            sm2 = copy.deepcopy(sm)
            for u in range(t, t + 8):
                b = q.forward_step(_tcl(frames[u], torch.bfloat16))
                r = sm2.forward_step(frames[u])
                assert (b is None) == (r is None)
                if b is not None:
                    _compare(kind, np_of(b), r, torch.float32)
                    ahead.setdefault(u, []).append(b)
        y = p.forward_step(_tcl(x, torch.bfloat16))
        r = sm.forward_step(x)
        assert (y is None) == (r is None)
        if y is not None:
            _compare(kind, np_of(y), r, torch.float32)
            for b in ahead.pop(t, []):
                assert torch.equal(b, y)
    assert not ahead or max(ahead) >= len(frames) - 1


@pytest.mark.parametrize("kind", ["max", "avg"])
@pytest.mark.parametrize("shape", [
    # kernel,      stride,    pad,       dil,       H,  W,  C,  B
    ((3, 3, 3), (1, 2, 2), (0, 1, 1), (1, 1, 1), 14, 14, 64, 5),     # the I3D-style bench shape, reduced
    ((2, 3, 2), (1, 1, 2), (1, 2, 0), (2, 2, 1), 9, 12, 16, 3),      # temporal / row dilation, padded rows
    ((4, 2, 3), (2, 2, 1), (2, 0, 2), (1, 1, 2), 7, 10, 8, 2),       # temporal stride, column dilation
    ((1, 3, 3), (1, 1, 1), (0, 1, 1), (1, 1, 1), 8, 8, 24, 200),     # kt = 1 (no ring rows), more units than SMs
])
def test_pool_row_pipeline_vs_oracle_and_band(kind, shape):
    """k_step_pool_seg (bulk-copy row pipeline, option pool_seg) against the fp64
    pooling oracle over readiness, Ready ticks, an update_state = 0 probe and
    pad_end steps, and bit for bit against the band / plain kernels (pool_seg =
    0): same taps and ring slots in the same order."""
    kernel, stride, pad, dil, H, W, C, B = shape
    rng = np.random.default_rng(sum(kernel) * 7 + C)
    outs = {}
    for seg in (1, 0):
        set_opt("pool_seg", seg)
        set_opt("pool_g", 1)                       # (small shapes would otherwise take the split kernel)
        rs = np.random.default_rng(1234)
        p, sm = _make(kind, 2, kernel, stride, pad, dil, H, W, C, B, torch.bfloat16, torch.float32)
        assert p.kernel_name.startswith("k_step_pool_seg" if seg else "k_step_pool"), p.kernel_name
        assert seg or "seg" not in p.kernel_name
        ys = []
        T = sm.f + 2 * stride[0] + 4
        for t in range(T):
            xq = _quant(rs.standard_normal((B, C, H, W)), torch.bfloat16)
            if t == sm.f + 1:
                probe = _quant(rs.standard_normal((B, C, H, W)), torch.bfloat16)
                yp = p.forward_step(_tcl(probe, torch.bfloat16), update_state=False)
                rp = sm.forward_step(probe, update_state=False)
                assert (yp is None) == (rp is None)
                if yp is not None:
                    ys.append(np_of(yp))
                    if seg:
                        _compare(kind, ys[-1].reshape(rp.shape), rp, torch.float32)
            y = p.forward_step(_tcl(xq, torch.bfloat16))
            r = sm.forward_step(xq)
            assert (y is None) == (r is None), t
            if y is not None:
                ys.append(np_of(y))
                if seg:
                    _compare(kind, ys[-1].reshape(r.shape), r, torch.float32)
        for _ in range(pad[0]):
            y = p.forward_pad_step()
            r = sm.forward_step(None)
            assert (y is None) == (r is None)
            if y is not None:
                ys.append(np_of(y))
                if seg:
                    _compare(kind, ys[-1].reshape(r.shape), r, torch.float32)
        outs[seg] = ys
    assert len(outs[1]) == len(outs[0]) and len(outs[1]) > 0
    for a, b in zip(outs[1], outs[0]):
        np.testing.assert_array_equal(a, b)
