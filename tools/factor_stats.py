"""Sparsity of the factors during a run: per sweep k, per factor, the number of all-zero
columns and the share of exactly-zero entries.
    python tools/factor_stats.py [--config c4] [--sweeps 20]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import sacd_inputs as SI  # noqa: E402
from paper_2003_03572_b200.sacd import Sacd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--sweeps", type=int, default=20)
ap.add_argument("--every", type=int, default=2)
a = ap.parse_args()
cfg = SI.CONFIGS[a.config]
c, v = SI.make_tensor(cfg, device="cuda")
g = Sacd(c, v, cfg.dims, cfg.rank, cfg.seed)
k = 0
while k < a.sweeps:
    g.iterate(a.every)
    k += a.every
    F = g.factors()
    st = g.stats()[-1]
    parts = []
    for n in range(3):
        z = (F[n] == 0)
        parts.append(f"F{n}: dead cols {int(z.all(axis=0).sum())}/{F[n].shape[1]} zero {100 * z.mean():.1f}%")
    print(f"k={k} f={st['objective']:.6e} E={st['E']} " + " | ".join(parts), flush=True)
g.close()
