"""Edge and degenerate cases of the CUDA path against the fp64 oracle, through
the C ABI: a single stream, 1x1 frames, the largest temporal padding (p = f-1,
delay 0), temporal dilation, channel counts the vector kernels do not cover
(dispatch falls back to the generic kernel), empty clips, clips shorter than the
receptive field, and the error codes of unsupported requests.
"""
import numpy as np
import pytest
import torch

import oracle as O
from tests.helpers import make_pair, np_of, rel_err, to_cl

pytestmark = pytest.mark.gpu


def _shape(d, B):
    H, W = d.in_hw
    return (B, d.cin) + ((H,) if d.spatial_rank >= 1 else ()) + ((W,) if d.spatial_rank >= 2 else ())


def _check(d, B, kernel, dtype=torch.bfloat16, steps=None, seed=0, expect_kernel=None):
    rng = np.random.default_rng(seed)
    W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
    b = rng.standard_normal(d.cout) * 0.1
    conv, sm, _, _ = make_pair(d, W, b, B, dtype=dtype, out_dtype=torch.float32, kernel=kernel)
    if expect_kernel:
        assert conv.kernel_used == expect_kernel, conv.kernel_name
    ys, refs = [], []
    for t in range(steps or d.receptive_field + 3):
        x = to_cl(rng.standard_normal(_shape(d, B)), dtype)
        y = conv.forward_step(x)
        r = sm.forward_step(np_of(x))
        assert (y is None) == (r is None)
        assert (conv.n, conv.head) == (sm.n, sm.head)
        if y is not None:
            ys.append(np_of(y)); refs.append(r.reshape(y.shape))
    assert ys, "no Ready output"
    assert rel_err(np.stack(ys), np.stack(refs)) <= 1e-4
    return conv


@pytest.mark.parametrize("kernel,desc", [
    ("dense_tc", O.Desc(2, 64, 64, (3, 3, 3), padding=(0, 1, 1), in_spatial=(56, 56))),     # C2 shape, B = 1
    ("depthwise", O.Desc(2, 192, 192, (3, 3, 3), padding=(0, 1, 1), groups=192, in_spatial=(28, 28))),
    ("depthwise", O.Desc(2, 192, 192, (5, 1, 1), groups=192, in_spatial=(28, 28))),
    ("dense_tc", O.Desc(1, 256, 256, (9, 1), dilation=(2, 1), in_spatial=(25, 1))),           # C5 shape, B = 1
])
def test_single_stream(kernel, desc):
    _check(desc, 1, kernel, steps=desc.receptive_field + 2, expect_kernel=kernel)


@pytest.mark.parametrize("kernel", ["dense_tc", "direct"])
def test_one_by_one_frame_with_spatial_padding(kernel):
    # 1x1 input, 3x3 kernel, pad 1: only the centre tap ever sees data
    _check(O.Desc(2, 16, 32, (3, 3, 3), padding=(0, 1, 1), in_spatial=(1, 1)), 3, kernel, expect_kernel=kernel)


@pytest.mark.parametrize("kernel,groups", [("dense_tc", 1), ("depthwise", 16), ("direct", 1)])
def test_max_temporal_padding_delay_zero(kernel, groups):
    d = O.Desc(2, 16, 16, (3, 3, 3), padding=(2, 1, 1), groups=groups, in_spatial=(5, 6))
    assert d.delay == 0                        # Fig. 2: padding f-1 saturates the state
    conv = _check(d, 2, kernel, expect_kernel=kernel)
    assert conv.delay == 0


@pytest.mark.parametrize("kernel,groups", [("dense_tc", 1), ("depthwise", 32)])
def test_temporal_dilation_three(kernel, groups):
    d = O.Desc(2, 32, 32, (3, 3, 3), padding=(0, 1, 1), dilation=(3, 1, 1), groups=groups, in_spatial=(6, 5))
    assert d.receptive_field == 7 and d.ring_slots == 6
    _check(d, 2, kernel, expect_kernel=kernel, steps=11)


def test_dispatch_falls_back_for_uncovered_shapes():
    # Cout % 4 != 0 and a grouped (not depthwise) conv: no vector kernel covers
    # them, AUTO dispatch takes the generic CUDA-core kernel
    _check(O.Desc(2, 16, 6, (3, 3, 3), padding=(0, 1, 1), in_spatial=(5, 5)), 2, "auto", expect_kernel="direct")
    _check(O.Desc(2, 16, 16, (2, 3, 3), padding=(0, 1, 1), groups=4, in_spatial=(5, 5)), 2, "auto",
           expect_kernel="direct")


def test_empty_and_short_clips():
    from paper_2204_03418_b200 import channels_last
    from paper_2204_03418_b200._abi import CoError, CO_ERR_LENGTH
    d = O.Desc(2, 16, 32, (3, 3, 3), padding=(0, 1, 1), in_spatial=(5, 6))
    rng = np.random.default_rng(3)
    conv, sm, Wq, bq = make_pair(d, rng.standard_normal(d.w_shape) / 12, rng.standard_normal(32) * 0.1, 2,
                                 dtype=torch.bfloat16, kernel="dense_tc")
    empty = channels_last(torch.zeros((2, 16, 0, 5, 6), dtype=torch.bfloat16, device="cuda"))
    ys, mask = conv.forward_steps(empty)
    assert ys.shape[2] == 0 and mask.numel() == 0 and conv.n == 0
    short = channels_last(torch.zeros((2, 16, 2, 5, 6), dtype=torch.bfloat16, device="cuda"))
    with pytest.raises((CoError, ValueError)) as e:     # T' = 2 - 3 + 1 = 0 < 1
        conv.forward(short)
    if isinstance(e.value, CoError):
        assert e.value.code == CO_ERR_LENGTH


def test_unsupported_requests_fail_loudly():
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200._abi import CoError, CO_ERR_UNSUPPORTED
    w = torch.zeros(32, 16, 3, 3, 3, dtype=torch.float32, device="cuda")
    with pytest.raises(CoError) as e:      # fp32 has no tensor-core kernel (TF32 would break 1e-4)
        co.Conv(16, 32, (3, 3, 3), weight=w, padding=(0, 1, 1), in_spatial=(5, 5), dtype=torch.float32,
                kernel="dense_tc")
    assert e.value.code == CO_ERR_UNSUPPORTED
    wb = torch.zeros(32, 16, 3, 3, 3, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(CoError) as e:      # not depthwise
        co.Conv(16, 32, (3, 3, 3), weight=wb, padding=(0, 1, 1), in_spatial=(5, 5), kernel="depthwise")
    assert e.value.code == CO_ERR_UNSUPPORTED
    wl = torch.zeros(8, 8, 33, 1, 1, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(CoError) as e:      # kt > CO_MAX_KT
        co.Conv(8, 8, (33, 1, 1), weight=wl, in_spatial=(2, 2))
    assert e.value.code == CO_ERR_UNSUPPORTED


def test_none_input_is_empty_and_does_not_advance():
    """an Empty input returns Empty and leaves the clock and state
    untouched, so hand-chained layers short-circuit like a Stack; a padding step
    (pad_end) is asked for explicitly (forward_pad_step)."""
    import paper_2204_03418_b200 as co
    d = O.Desc(2, 16, 16, (3, 3, 3), padding=(1, 1, 1), in_spatial=(5, 6))
    rng = np.random.default_rng(0)
    c, sm, _, _ = make_pair(d, rng.standard_normal(d.w_shape) / 12, None, 2, dtype=torch.bfloat16)
    c2, _, _, _ = make_pair(d, rng.standard_normal(d.w_shape) / 12, None, 2, dtype=torch.bfloat16,
                            out_dtype=torch.bfloat16)
    assert c.forward_step(None) is None and c.n == 0
    assert c2.forward_step(c2.forward_step(None)) is None and c2.n == 0
    x = to_cl(rng.standard_normal((2, 16, 5, 6)), torch.bfloat16)
    c.forward_step(x)
    assert c.n == 1
    y = c.forward_pad_step()
    assert c.n == 2 and y is not None             # d = 1: the padding step is Ready
    with pytest.raises(ValueError):
        c.forward_step(x, pad=True)


def test_out_tensor_is_validated():
    """The kernels write `out` through its data pointer: wrong shape, dtype,
    device or layout is refused before any launch."""
    import paper_2204_03418_b200 as co
    d = O.Desc(2, 16, 8, (1, 3, 3), padding=(0, 1, 1), in_spatial=(5, 6))
    rng = np.random.default_rng(1)
    c, _, _, _ = make_pair(d, rng.standard_normal(d.w_shape), None, 2, dtype=torch.bfloat16)
    x = to_cl(rng.standard_normal((2, 16, 5, 6)), torch.bfloat16)
    good = co._empty_cl((2, 8, 5, 6), torch.float32, "cuda")
    assert c.forward_step(x, out=good) is good
    for bad in (co._empty_cl((2, 8, 5, 5), torch.float32, "cuda"),            # shape
                co._empty_cl((2, 8, 5, 6), torch.bfloat16, "cuda"),           # dtype
                torch.empty((2, 8, 5, 6), dtype=torch.float32, device="cuda"),  # not channels-last
                co._empty_cl((2, 8, 5, 6), torch.float32, "cpu")):            # device
        with pytest.raises(ValueError):
            c.forward_step(x, out=bad)
    st = co.Stack([c])
    with pytest.raises(ValueError):
        st.forward_step(x[:1])                                                 # wrong stream count
