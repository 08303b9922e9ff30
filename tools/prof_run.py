"""Minimal driver for ncu: build one context on the GPU and run a few sweeps.
    python tools/prof_run.py [--config c4] [--precision f64] [--sweeps 2] [--rank R]"""
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
ap.add_argument("--sweeps", type=int, default=2)
ap.add_argument("--rank", type=int, default=None)
ap.add_argument("--graph", type=int, default=0)
a = ap.parse_args()
cfg = SI.CONFIGS[a.config]
c, v = SI.make_tensor(cfg, device="cuda")
g = Sacd(c, v, cfg.dims, a.rank or cfg.rank, cfg.seed, precision=a.precision, use_graph=bool(a.graph))
g.iterate(a.sweeps)
g.sync()
print("f =", g.fit(), "info:", g.info()["split_rows"])
g.close()
