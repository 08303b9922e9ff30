"""Gather-weighted support of the factors after k sweeps (GPU, torch): for each mode n with
layout modes (a, b) (L1), the mean number of nonzeros of the b-row gathered per
tensor nonzero and of the a-row gathered per fiber, the share of gathers whose row has at
most 16 / 32 nonzeros, and the 32-byte sectors a mask + packed-values row format would touch
per gather (1 mask sector + ceil(8 n / 32)) against the dense row's R*8/32.
    python tools/pack_stats.py [--config c4] [--sweeps 12]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import sacd_inputs as SI  # noqa: E402
from paper_2003_03572_b200.sacd import Sacd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--sweeps", type=int, nargs="+", default=[3, 6, 12, 20])
ap.add_argument("--precision", default="f64")
a = ap.parse_args()
cfg = SI.CONFIGS[a.config]
c, v = SI.make_tensor(cfg, device="cuda")
g = Sacd(c, v, cfg.dims, cfg.rank, cfg.seed, precision=a.precision)
c = c.long()
d = cfg.dims
R = cfg.rank
es = 8 if a.precision == "f64" else 4
done = 0
for K in a.sweeps:
    g.iterate(K - done)
    done = K
    cnt = [torch.from_numpy((x != 0).sum(1)).cuda() for x in g.factors()]
    print(f"k={K}", flush=True)
    for n in range(3):
        o = [m for m in range(3) if m != n]
        am = o[0] if d[o[0]] >= d[o[1]] else o[1]
        bm = o[1] if am == o[0] else o[0]
        nb = cnt[bm][c[:, bm]].float()
        key = torch.unique(c[:, n] * d[am] + c[:, am])
        na = cnt[am][key % d[am]].float()
        sec = lambda t: (1 + torch.ceil(t * es / 32)).mean().item()  # noqa: E731
        print(f"  mode {n}: b=mode {bm} n_b mean {nb.mean().item():.2f} (<=16: {(nb <= 16).float().mean().item() * 100:.1f}%,"
              f" <=32: {(nb <= 32).float().mean().item() * 100:.1f}%) sectors {sec(nb):.2f}; "
              f"a=mode {am} n_a mean {na.mean().item():.2f} (<=16: {(na <= 16).float().mean().item() * 100:.1f}%) "
              f"sectors {sec(na):.2f}; dense {R * es / 32:.0f}", flush=True)
g.close()
