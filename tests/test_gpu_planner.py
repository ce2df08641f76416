"""The dispatch / planner choices bench.py's configs rely on, at
their full stream counts: a planner change that silently moves a layer to a
slower kernel mode fails here before it shows up as a bench regression."""
import pytest
import torch

pytestmark = pytest.mark.gpu

EXPECTED = {
    2: ["k_step_dense_tc<3,32,3,3x3x64,pair>"],                      # HALO, CTA pair, 150 KB budget
    3: ["k_step_dw_seg<3,3,3>", "k_step_dw_t<5>"],                  # K2s segment pipeline, K3
    4: ["k_step_dense_tc<5,32,3,stem>", "k_step_dense_tc<1,128,2,3x3x64,pair>",
        "k_step_dense_tc<3,64,2,3x3,pair,khalo>", "k_step_dense_tc<3,64,2,3x3,pair,khalo>",
        "k_step_dense_tc<3,64,2,3x3,pair,khalo>"],                   # STEM, HALO pair, 3 x KHALO (stride 2 / 1 / 2)
    5: ["k_step_dense_tc<9,16,2,1x1x256,pair>"],                     # FLAT pair (fp32 partial-sum layout)
}


def test_c5_auto_layout_is_raw():
    """C5 states only 'bf16' (BASELINE.json configs[4]), so the bench lets the
    planner pick the layout (CO_STATE_AUTO): the raw-input ring, whose 1x1
    window contraction moves 3.6x fewer bytes than the fp32 partial sums."""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    cfg = synth.config(5, n_streams=64)
    L = cfg.layers[0]
    W, b = synth.params(cfg)[0]
    c = co.Conv(L.cin, L.cout, L.kernel, weight=W.cuda(), bias=b.cuda(), dilation=L.dilation, spatial_rank=1,
                in_spatial=cfg.in_spatial, n_streams=64, state_layout="auto")
    assert c.state_layout == "raw" and c.kernel_name == "k_step_dense_tc<1,256,2,pair,kloop>", c.kernel_name
    cfg2 = synth.config(2, n_streams=2)
    W2, b2 = synth.params(cfg2)[0]
    L2 = cfg2.layers[0]
    c2 = co.Conv(L2.cin, L2.cout, L2.kernel, weight=W2.cuda(), bias=b2.cuda(), padding=L2.padding,
                 in_spatial=cfg2.in_spatial, n_streams=2, state_layout="auto")
    assert c2.state_layout == "psum"                  # spatial windows keep the partial sums


def test_c3_auto_layout_depthwise_is_raw():
    """C3 states only 'bf16' (BASELINE.json configs[2]): under CO_STATE_AUTO both
    layers take the RAW frame ring with the frame store fused -- the temporal-only
    layer (kt = 5) as one streaming pass (7 bf16 frame accesses per step against 18
    for the fp32 partial sums), the "same"-padded 3x3x3 stencil over rolling row
    sets (5 against 10)."""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import synth
    cfg = synth.config(3, n_streams=8)
    names, layouts = [], []
    for L, (W, b) in zip(cfg.layers, synth.params(cfg)):
        c = co.Conv(L.cin, L.cout, L.kernel, weight=W.cuda(), bias=b.cuda(), padding=L.padding, groups=L.groups,
                    in_spatial=cfg.in_spatial, n_streams=8, state_layout="auto")
        names.append(c.kernel_name); layouts.append(c.state_layout)
    assert layouts == ["raw", "raw"] and names == ["k_step_dw_rowraw<3,3,3>", "k_step_dw_traw<5>"], (layouts, names)


@pytest.mark.parametrize("cid", sorted(EXPECTED))
def test_bench_config_kernels(cid):
    from paper_2204_03418_b200 import synth
    from tests.helpers import build_config_layers
    cfg = synth.config(cid)
    convs, _, _, _ = build_config_layers(cfg, cfg.n_streams)
    names = [c.kernel_name for c in convs]
    assert names == EXPECTED[cid], names
    del convs
    torch.cuda.empty_cache()
