"""Hot-row coverage of a config (GPU, torch): for each mode n, the share of nonzeros whose
per-nonzero gather row (mode b of the layout rule, L1) and whose per-fiber row
(mode a) lies among the K most frequent rows of that mode.
    python tools/hot_stats.py [c4]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import sacd_inputs as SI  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = SI.CONFIGS[name]
c, v = SI.make_tensor(cfg, device="cuda")
c = c.long()
nnz = c.shape[0]
d = cfg.dims
Ks = (64, 128, 192, 256, 384, 512, 1024, 4096)
for n in range(3):
    o = [m for m in range(3) if m != n]
    a = o[0] if d[o[0]] >= d[o[1]] else o[1]
    b = o[1] if a == o[0] else o[0]
    cnt_b = torch.bincount(c[:, b], minlength=d[b]).sort(descending=True).values.cumsum(0)
    line = [f"mode {n}: b=mode {b} (I={d[b]}) share of nnz in top-K b rows:"]
    line += [f"K={k}:{100 * cnt_b[min(k, d[b]) - 1].item() / nnz:.1f}%" for k in Ks]
    print(" ".join(line))
    key = torch.unique(c[:, n] * d[a] + c[:, a])
    fa = key % d[a]
    cnt_a = torch.bincount(fa, minlength=d[a]).sort(descending=True).values.cumsum(0)
    line = [f"        a=mode {a} (I={d[a]}) fibers {key.numel()} share in top-K a rows:"]
    line += [f"K={k}:{100 * cnt_a[min(k, d[a]) - 1].item() / key.numel():.1f}%" for k in Ks]
    print(" ".join(line))
