"""One MTTKRP launch of a given variant and mode, for ncu (skip the init's W-mode launch and
the sweeps' launches with --launch-skip 1 + 3 * sweeps).
    python tools/prof_mttkrp.py --config c4 --precision f64 --variant 0 --mode 0"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import sacd_inputs as SI  # noqa: E402
from paper_2003_03572_b200.sacd import Sacd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--precision", default="f64")
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--rank", type=int, default=None)
ap.add_argument("--sweeps", type=int, default=0)
ap.add_argument("--ablk", type=int, default=0)
a = ap.parse_args()
cfg = SI.CONFIGS[a.config]
c, v = SI.make_tensor(cfg, device="cuda")
g = Sacd(c, v, cfg.dims, a.rank or cfg.rank, cfg.seed, precision=a.precision, mttkrp_variant=a.variant, ablk_rows=a.ablk)
if a.sweeps:
    g.iterate(a.sweeps)
g.mttkrp(a.mode)
g.sync()
g.close()
