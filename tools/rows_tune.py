"""Time the fused SaCD row update per variant (opt.reserved[0]) inside profiled sweeps.
    python tools/rows_tune.py --config c4 --precision f64 [--variants 0,1] [--sweeps 3]"""
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
ap.add_argument("--variants", default="0,1")
ap.add_argument("--sweeps", type=int, default=3)
a = ap.parse_args()
cfg = SI.CONFIGS[a.config]
c, v = SI.make_tensor(cfg, device="cuda")
ref = None
for var in [int(x) for x in a.variants.split(",")]:
    g = Sacd(c, v, cfg.dims, cfg.rank, cfg.seed, precision=a.precision, rows_variant=var, profile=True)
    g.iterate(a.sweeps)
    g.sync()
    p = g.profile_read()
    f = g.fit()[0]
    same = "ref" if ref is None else ("same f" if f == ref else f"f differs {f} vs {ref}")
    ref = ref if ref is not None else f
    print(f"{a.config} {a.precision} rows variant {var}: rows ms/sweep {p['rows'][0] / a.sweeps:.3f} "
          f"gram {p['gram'][0] / a.sweeps:.3f} fixup {p['fixup'][0] / a.sweeps:.3f} mttkrp {p['mttkrp'][0] / a.sweeps:.3f}  {same}",
          flush=True)
    g.close()
