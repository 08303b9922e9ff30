"""Per-sweep time of the sharded engine with G emulated ranks on ONE GPU (the ranks run one
after another, so the time is the sum of all ranks' work plus the emulated exchanges) against
the unsharded engine: the compute overhead of sharding that a real G-GPU run would split.
    python tools/emulated_scaling.py [c4] [--exchange delta]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import sacd_inputs as SI  # noqa: E402
from paper_2003_03572_b200.sacd import Sacd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "c4"
exchange = sys.argv[sys.argv.index("--exchange") + 1] if "--exchange" in sys.argv else "delta"
npi = int(sys.argv[sys.argv.index("--nnz-per-item") + 1]) if "--nnz-per-item" in sys.argv else 0
cfg = SI.CONFIGS[name]
c, v = SI.make_tensor(cfg, device="cuda")
K, W = 10, 3
for G in (1, 2, 4, 8):
    kw = {} if G == 1 else dict(emulate_ranks=G, exchange=exchange)
    if npi:
        kw["nnz_per_item"] = npi
    with Sacd(c, v, cfg.dims, cfg.rank, cfg.seed, **kw) as g:
        g.iterate(W)
        g.sync()
        t = time.perf_counter()
        g.iterate(K)
        g.sync()
        ms = (time.perf_counter() - t) / K * 1e3
        f = g.fit()[0]
        g.set_profile(True)
        g.profile_reset()
        g.iterate(K)
        g.sync()
        p = g.profile_read()
        br = " ".join(f"{k} {p[k][0] / K:.3f}" for k in p)
    print(f"{name} G={G} ({'unsharded' if G == 1 else 'emulated, ' + exchange}): {ms:.2f} ms per sweep "
          f"(sum over ranks), f = {f:.10e}; eager per class: {br}", flush=True)
