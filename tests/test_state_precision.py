"""Row g (north_star "SoA ring buffers in HBM, bf16 or fp32 accumulators"):
why the partial-sum ring is fp32 only.  CPU-only (`-m "not gpu"`).

The partial-sum method (north_star; SPEC S:239 for the ring it replaces)
stores every pending output between steps: output i is the running sum
S <- P_0, S <- S + P_1, ..., y = S + P_{kt-1} + b, one store per step.  With a
bf16 ring each store rounds the running sum to 8 significant bits (RNE), and
the kt-1 roundings add up.  This test runs that exact recurrence on real
per-slice partials P_k = W[:, :, k] (*) x_t of C2 / C4-stem / C5-shaped layers
(torch float64 conv2d per temporal slice, an independent implementation of
the textbook convolution) and compares the emitted outputs with the exact
fp64 sums: at kt = 5 and 9 the bf16 ring breaks the north_star's bf16 bar
(max |err| <= 2e-2 RMS), while the fp32 ring stays ~1e-6.  So the library
offers fp32 accumulators only (reading A25); a bf16 ring would need
a looser tolerance than BASELINE.json states.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

BAR = 2e-2   # north_star: max abs error <= 2e-2 of the output RMS (bf16 inputs, fp32 accumulation)


def _bf16(a: torch.Tensor) -> torch.Tensor:
    return a.to(torch.bfloat16).to(torch.float64)            # RNE (A17)


def _ring_outputs(kt, cin, cout, k, H, W, B, T, seed, store):
    """Emitted outputs of a kt x k x k layer (stride 1, 'same' spatial padding)
    computed through the partial-sum recurrence with the ring stored by
    `store` (identity = exact), and the exact fp64 outputs."""
    g = torch.Generator().manual_seed(seed)
    fan_in = cin * kt * k * k
    Wt = _bf16(torch.randn((cout, cin, kt, k, k), generator=g, dtype=torch.float64) / np.sqrt(fan_in))
    b = torch.randn(cout, generator=g, dtype=torch.float64) * 0.1
    xs = [_bf16(torch.randn((B, cin, H, W), generator=g, dtype=torch.float64)) for _ in range(T)]
    # P[t][k] = slice k of the kernel applied to frame t (fp64: the exact products and sums)
    P = [[F.conv2d(x, Wt[:, :, j], padding=k // 2) for j in range(kt)] for x in xs]
    got, exact = [], []
    for i in range(T - kt + 1):                               # output i uses frames i .. i + kt - 1
        s = store(P[i][0])
        e = P[i][0]
        for j in range(1, kt - 1):
            s = store(s + P[i + j][j])
            e = e + P[i + j][j]
        got.append(s + P[i + kt - 1][kt - 1] + b[None, :, None, None])
        exact.append(e + P[i + kt - 1][kt - 1] + b[None, :, None, None])
    got, exact = torch.stack(got), torch.stack(exact)
    rms = exact.pow(2).mean().sqrt().item()
    return (got - exact).abs().max().item() / rms


CASES = {
    # (kt, Cin, Cout, k, H, W, B, T): the configs' channel / kernel shapes on small frames
    "C2_kt3": (3, 64, 64, 3, 24, 24, 6, 12),
    "C4_stem_kt5": (5, 3, 64, 7, 40, 40, 6, 14),
    "C5_kt9": (9, 256, 256, 1, 25, 1, 64, 20),
}


@pytest.mark.parametrize("name", list(CASES))
def test_fp32_ring_is_within_the_bar(name):
    kt, cin, cout, k, H, W, B, T = CASES[name]
    err = _ring_outputs(kt, cin, cout, k, H, W, B, T, 1, lambda a: a.to(torch.float32).to(torch.float64))
    assert err < 1e-5, err


@pytest.mark.parametrize("name", list(CASES))
def test_bf16_ring_error(name):
    """bf16 storage of the running sums: the worst output error over the run
    relative to the output RMS.  kt = 5 and 9 exceed the 2e-2 bar; kt = 3 (one
    stored rounding) sits just under it on this sample."""
    kt, cin, cout, k, H, W, B, T = CASES[name]
    err = _ring_outputs(kt, cin, cout, k, H, W, B, T, 1, _bf16)
    if kt >= 5:
        assert err > BAR, err
    else:
        assert 0.5 * BAR < err <= BAR, err
