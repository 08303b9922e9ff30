"""End-to-end drift of a reduced-precision build against the fp64 build (which matches the
oracle to ~1e-14): per sweep the relative error of f, and after K sweeps the north-star
factor metric max |F - F64| / max(|F64|, 1e-3 * colmax|F64|).
    python tools/precision_drift.py --configs c1,c2,c3 --sweeps 10 --precision f32"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import sacd_inputs as SI  # noqa: E402
from paper_2003_03572_b200.sacd import Sacd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2,c3")
ap.add_argument("--sweeps", type=int, default=10)
ap.add_argument("--precision", default="f32")
ap.add_argument("--rank", type=int, default=None)
a = ap.parse_args()
for name in a.configs.split(","):
    cfg = SI.CONFIGS[name]
    R = a.rank or cfg.rank
    c, v = SI.make_tensor(cfg, device="cuda")
    res = {}
    for prec in ("f64", a.precision):
        with Sacd(c, v, cfg.dims, R, cfg.seed, precision=prec) as g:
            g.iterate(a.sweeps)
            st = g.stats()
            res[prec] = (np.array([s["objective"] for s in st]), g.factors(), [s["E"] for s in st])
    f64, F64, E64 = res["f64"]
    fx, Fx, Ex = res[a.precision]
    frel = np.abs(fx - f64) / np.abs(f64)
    worst = 0.0
    for n in range(3):
        den = np.maximum(np.abs(F64[n]), 1e-3 * np.abs(F64[n]).max(axis=0, keepdims=True))
        den[den == 0] = 1
        worst = max(worst, float((np.abs(Fx[n] - F64[n]) / den).max()))
    print(f"{name} R={R} {a.precision} vs f64, {a.sweeps} sweeps: max rel f err {frel.max():.2e} "
          f"(per sweep {' '.join(f'{x:.0e}' for x in frel)}); factor metric {worst:.2e}; "
          f"E last f64 {E64[-1]} vs {Ex[-1]}", flush=True)
