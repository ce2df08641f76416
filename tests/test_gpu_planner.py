"""The dispatch / planner choices bench.py's configs rely on, at
their full stream counts: a planner change that silently moves a layer to a
slower kernel mode fails here before it shows up as a bench regression."""
import pytest
import torch

pytestmark = pytest.mark.gpu

EXPECTED = {
    2: ["k_step_dense_tc<3,32,3,3x3x64,pair>"],                      # HALO, CTA pair, 150 KB budget
    3: ["k_step_dw_st<3,3,3>", "k_step_dw_t<5>"],
    4: ["k_step_dense_tc<5,32,3,kloop+wcols>", "k_step_dense_tc<1,128,2,3x3x64,pair>",
        "k_step_dense_tc<3,64,2,pair,khalo>", "k_step_dense_tc<3,64,2,pair,khalo>",
        "k_step_dense_tc<3,64,2,pair,khalo>"],                       # stem, HALO pair, 3 x KHALO (stride 2 / 1 / 2)
    5: ["k_step_dense_tc<9,16,2,1x1x256,pair>"],                     # FLAT pair
}


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
