"""Time the MTTKRP tuning variants (opt.reserved[0]) per mode; check they agree bitwise.
    python tools/mttkrp_tune.py --config c4 --precision f64 [--variants 0,1,2,...]"""
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
ap.add_argument("--precision", default="f64")
ap.add_argument("--rank", type=int, default=None)
ap.add_argument("--variants", default="1,10,11,12,13,14,15,0")
ap.add_argument("--nnz-per-item", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--sweeps", type=int, default=0, help="SaCD sweeps before timing (sparse factors)")
ap.add_argument("--ablk", type=int, default=0, help="a-blocked execution order: a-rows per block (0 = canonical)")
a = ap.parse_args()
cfg = SI.CONFIGS[a.config]
R = a.rank or cfg.rank
c, v = SI.make_tensor(cfg, device="cuda")
ref = None
for var in [int(x) for x in a.variants.split(",")]:
    g = Sacd(c, v, cfg.dims, R, cfg.seed, precision=a.precision, mttkrp_variant=var, nnz_per_item=a.nnz_per_item,
             ablk_rows=a.ablk)
    if a.sweeps:
        g.iterate(a.sweeps)
    ms = [g.time_mttkrp(n, a.reps) for n in range(3)]
    M0 = g.mttkrp(0)
    same = "ref" if ref is None else ("bitwise-equal" if np.array_equal(M0, ref) else f"DIFF {np.abs(M0-ref).max():.3e}")
    if ref is None:
        ref = M0
    print(f"{a.config} {a.precision} R={R} T={a.nnz_per_item or 1024} k={a.sweeps} ablk={a.ablk} variant {var}: ms per mode "
          f"{ms[0]:.3f} {ms[1]:.3f} {ms[2]:.3f}  sum {sum(ms):.3f}  {same}", flush=True)
    g.close()
