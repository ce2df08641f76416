"""Bisect helper for the CTA-pair dense kernel (experiments only)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_03418_b200 as co
os.environ["CO_TC_PAIR"] = "2"
B, Cin, Cout, H, W = 3, 64, 64, 13, 24
w = (torch.randn(Cout, Cin, 3, 3, 3) / 24).to(torch.bfloat16).cuda()
b = torch.zeros(Cout).cuda()
conv = co.Conv(Cin, Cout, (3, 3, 3), weight=w, bias=b, padding=(0, 1, 1), spatial_rank=2, in_spatial=(H, W),
               n_streams=B, dtype=torch.bfloat16, out_dtype=torch.float32, kernel="dense_tc")
print(conv.kernel_name, flush=True)
for t in range(4):
    x = co.channels_last(torch.randn(B, Cin, H, W).to(torch.bfloat16).cuda())
    y = conv.forward_step(x)
    torch.cuda.synchronize()
    print("step", t, "ok", None if y is None else float(y.float().abs().mean()), flush=True)
