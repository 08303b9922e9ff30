"""A/B of whole sweeps on one config: K timed sweeps (captured graph, CUDA events on the
library stream) after W warm-ups, then the eager per-kernel-class breakdown, per variant.
    python tools/sweep_ab.py [--config c4] [--variants "default;gram_variant=2"]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import sacd_inputs as SI  # noqa: E402
from paper_2003_03572_b200.sacd import Sacd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--variants", default="default;gram_variant=2")
ap.add_argument("--sweeps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=5)
a = ap.parse_args()
cfg = SI.CONFIGS[a.config]
c, v = SI.make_tensor(cfg, device="cuda")
stream = torch.cuda.Stream()
for spec in a.variants.split(";"):
    kw = {}
    env = {}
    for item in spec.split(","):
        if item.startswith("env:"):  # an environment variable set around that variant's sacd_init, e.g. env:SACD_POOL_RELEASE_MB=0
            k, val = item[4:].split("=")
            env[k] = val
        elif "=" in item:
            k, val = item.split("=")
            kw[k] = int(val)
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    with Sacd(c, v, cfg.dims, cfg.rank, cfg.seed, stream=stream.cuda_stream, **kw) as g:
        g.iterate(a.warmup)
        g.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.iterate(a.sweeps)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / a.sweeps
        f = g.fit()[0]
        g.set_profile(True)
        g.profile_reset()
        g.iterate(a.sweeps)
        g.sync()
        p = g.profile_read()
        br = " ".join(f"{k} {p[k][0] / a.sweeps:.3f}" for k in p)
    for k, val in saved.items():
        if val is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = val
    print(f"{a.config} [{spec}]: {ms:.3f} ms/sweep ({1e3 / ms:.2f} sweeps/s), f after {a.warmup + a.sweeps} = {f:.12e}; "
          f"eager ms/sweep: {br}", flush=True)
