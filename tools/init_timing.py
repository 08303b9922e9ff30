"""Wall time of sacd_init phases (SACD_INIT_TIMING=1) and of sacd_factors on a config, from
pinned host buffers as in bench.py's e2e leg.
    python tools/init_timing.py [c4]"""
import os
import sys
import time

os.environ["SACD_INIT_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import sacd_inputs as SI  # noqa: E402
from paper_2003_03572_b200.sacd import Sacd  # noqa: E402

cfg = SI.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
c, v = SI.make_tensor(cfg, device="cuda")
hc, hv = c.cpu().pin_memory(), v.cpu().pin_memory()
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    g = Sacd(hc, hv, cfg.dims, cfg.rank, cfg.seed)
    t1 = time.perf_counter()
    g.iterate(1)
    g.sync()
    t2 = time.perf_counter()
    F = g.factors()
    t3 = time.perf_counter()
    g.close()
    print(f"rep {rep}: sacd_init {1e3 * (t1 - t0):.1f} ms, 1 sweep {1e3 * (t2 - t1):.1f} ms, "
          f"sacd_factors {1e3 * (t3 - t2):.1f} ms ({sum(x.nbytes for x in F) / 1e6:.0f} MB)", flush=True)
