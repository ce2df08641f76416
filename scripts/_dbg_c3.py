import torch, sys
sys.path.insert(0, ".")
import paper_2204_03418_b200 as co
from paper_2204_03418_b200 import synth
cfg = synth.config(3); L = cfg.layers[0]; Wt, bt = synth.params(cfg)[0]
T = 7
g = torch.Generator(device="cuda").manual_seed(11)
clip = co.channels_last(torch.randn((cfg.n_streams, L.cin, T) + tuple(cfg.in_spatial), generator=g, device="cuda").to(torch.bfloat16))
res = {}
for name, opts in {"chunk": dict(chunk=1, chunk_st=1), "seg": dict(chunk=0, dw_seg=1), "k2": dict(chunk=0, dw_seg=0), "seg2": dict(chunk=0, dw_seg=1)}.items():
    co.set_option(None, 0) if False else None
    for k in ("chunk", "chunk_st", "dw_seg"):
        co.set_option(k, {"chunk": 1, "chunk_st": 0, "dw_seg": 1}[k])
    for k, v in opts.items(): co.set_option(k, v)
    conv = co.Conv(L.cin, L.cout, L.kernel, weight=Wt.cuda(), bias=bt.cuda(), stride=L.stride, padding=L.padding, dilation=L.dilation, groups=L.groups, spatial_rank=cfg.spatial_rank, in_spatial=tuple(cfg.in_spatial), n_streams=cfg.n_streams, dtype=cfg.dtype, out_dtype=torch.float32)
    ys, mask = conv.forward_steps(clip); st, _ = conv.state_dict_stream(); torch.cuda.synchronize()
    res[name] = (ys, mask, st, conv.kernel_name); del conv
ref = res["k2"]
for n, (ys, mask, st, kn) in res.items():
    dy = (ys != ref[0]); ds = (st != ref[2])
    print(n, kn, "y mismatches", int(dy.sum()), "state mismatches", int(ds.sum()), "mask eq", torch.equal(mask, ref[1]))
    if dy.any():
        idx = dy.nonzero()[:8]; print(" y shape", tuple(ys.shape), "first idx", idx.tolist(), "maxdiff", (ys - ref[0]).abs().max().item())
        bs = dy.nonzero()[:, 0].unique(); print(" streams", bs[:20].tolist(), len(bs))
    if ds.any():
        idx = ds.nonzero()[:8]; print(" st shape", tuple(st.shape), "first idx", idx.tolist(), "maxdiff", (st - ref[2]).abs().max().item())
