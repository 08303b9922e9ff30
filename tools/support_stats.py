"""Support statistics of the factors after k sweeps (GPU, torch): per mode n with layout
modes (a, b): mean nonzeros per a-row / b-row, and, weighted by the tensor's nonzeros, the
mean |supp(a_row) & supp(b_row)| (the columns a sparse-factor MTTKRP would touch) and the
share of 32-byte sectors of the b-row needed when only supp(a) columns are gathered.
    python tools/support_stats.py [--config c4] [--sweeps 12]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import sacd_inputs as SI  # noqa: E402
from paper_2003_03572_b200.sacd import Sacd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--sweeps", type=int, default=12)
a = ap.parse_args()
cfg = SI.CONFIGS[a.config]
c, v = SI.make_tensor(cfg, device="cuda")
g = Sacd(c, v, cfg.dims, cfg.rank, cfg.seed)
g.iterate(a.sweeps)
F = [torch.from_numpy(x).cuda() != 0 for x in g.factors()]
g.close()
c = c.long()
d = cfg.dims
R = cfg.rank
for n in range(3):
    o = [m for m in range(3) if m != n]
    am = o[0] if d[o[0]] >= d[o[1]] else o[1]
    bm = o[1] if am == o[0] else o[0]
    tot_i, tot_sec, ne = 0.0, 0.0, c.shape[0]
    for s in range(0, ne, 10_000_000):
        cc = c[s:s + 10_000_000]
        sa, sb = F[am][cc[:, am]], F[bm][cc[:, bm]]
        inter = sa & sb
        tot_i += inter.sum().item()
        sec = sa.view(sa.shape[0], -1, 4).any(dim=2)  # fp64: 4 columns per 32-byte sector
        tot_sec += sec.float().mean(dim=1).sum().item()
    print(f"mode {n}: a=mode {am} nnz/row {F[am].sum(1).float().mean().item():.2f} "
          f"(zero rows {(F[am].sum(1) == 0).float().mean().item() * 100:.1f}%), b=mode {bm} nnz/row "
          f"{F[bm].sum(1).float().mean().item():.2f}; per tensor nonzero: |a&b| = {tot_i / ne:.2f} of {R}, "
          f"b sectors needed for supp(a) = {100 * tot_sec / ne:.1f}%", flush=True)
