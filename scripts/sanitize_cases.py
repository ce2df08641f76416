"""Tiny invocations of every kernel family for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per run):
  compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_cases.py
Every case is checked against the fp64 oracle as well, so a clean sanitizer
run is also a correct one."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2204_03418_b200 as co  # noqa: E402
from tests.helpers import make_pair, np_of, rel_err, to_cl  # noqa: E402

CASES = [
    ("direct f32", O.Desc(2, 4, 8, (3, 3, 3), padding=(0, 1, 1), in_spatial=(5, 6)), "direct", torch.float32, {}),
    ("dense halo", O.Desc(2, 64, 64, (3, 3, 3), padding=(0, 1, 1), in_spatial=(5, 9)), "dense_tc", torch.bfloat16, {}),
    ("dense halo pair", O.Desc(2, 64, 64, (3, 3, 3), padding=(0, 1, 1), in_spatial=(5, 9)), "dense_tc", torch.bfloat16,
     {"CO_TC_PAIR": "2"}),
    ("dense flat pair", O.Desc(1, 256, 256, (9, 1), dilation=(2, 1), in_spatial=(25, 1)), "dense_tc", torch.bfloat16, {}),
    ("dense kloop pair", O.Desc(2, 128, 128, (3, 3, 3), stride=(1, 2, 2), padding=(0, 1, 1), in_spatial=(9, 10)),
     "dense_tc", torch.bfloat16, {}),
    ("dense kloop single", O.Desc(2, 64, 64, (3, 3, 3), stride=(2, 2, 2), padding=(1, 1, 1), in_spatial=(9, 10)),
     "dense_tc", torch.bfloat16, {"CO_TC_KPAIR": "1"}),
    ("dense stem", O.Desc(2, 3, 32, (5, 7, 7), stride=(1, 2, 2), padding=(0, 3, 3), in_spatial=(12, 14)), "dense_tc",
     torch.bfloat16, {}),
    ("depthwise st", O.Desc(2, 32, 32, (3, 3, 3), padding=(0, 1, 1), groups=32, in_spatial=(7, 9)), "depthwise",
     torch.bfloat16, {}),
    ("depthwise t", O.Desc(2, 32, 32, (5, 1, 1), groups=32, in_spatial=(4, 5)), "depthwise", torch.bfloat16, {}),
]


def main():
    rng = np.random.default_rng(0)
    B = 2
    for name, d, kernel, dt, env in CASES:
        os.environ.update(env)
        W = rng.standard_normal(d.w_shape) / np.sqrt(np.prod(d.w_shape[1:]))
        b = rng.standard_normal(d.cout) * 0.1
        conv, sm, Wq, bq = make_pair(d, W, b, B, dtype=dt, out_dtype=torch.float32, kernel=kernel)
        for k in env:
            os.environ.pop(k)
        H, Wd = d.in_hw
        shp = (B, d.cin) + ((H,) if d.spatial_rank >= 1 else ()) + ((Wd,) if d.spatial_rank >= 2 else ())
        frames = [to_cl(rng.standard_normal(shp), dt) for _ in range(d.receptive_field + 2)]
        ys, refs = [], []
        for x in frames:
            y = conv.forward_step(x)
            r = sm.forward_step(np_of(x))
            if y is not None:
                ys.append(np_of(y)); refs.append(r.reshape(y.shape))
        st, meta = conv.state_dict_stream()
        conv.load_state_stream(st, meta)
        conv.forward_step(frames[0], update_state=False)
        clip = co.channels_last(torch.stack(frames, dim=2))
        yb = conv.forward(clip)
        torch.cuda.synchronize()
        err = rel_err(np.stack(ys), np.stack(refs))
        tol = 1e-4
        assert err <= tol, (name, err)
        print(f"{name:20s} {conv.kernel_name:45s} rel={err:.1e} batch={tuple(yb.shape)}", flush=True)
    # host-buffer pipeline
    d = CASES[1][1]
    conv, _, _, _ = make_pair(d, rng.standard_normal(d.w_shape) / 24, None, B, dtype=torch.bfloat16)
    xh = torch.zeros((4, B, 5, 9, 64), dtype=torch.bfloat16).pin_memory()
    yh = torch.zeros((4, B, 5, 9, 64), dtype=torch.bfloat16).pin_memory()
    n, _ = conv.forward_steps_host(xh, yh)
    print("steps_host", n, flush=True)
    print("SANITIZE CASES OK", flush=True)


if __name__ == "__main__":
    main()
