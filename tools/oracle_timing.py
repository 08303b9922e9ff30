"""Measured CPU baseline: the fp64 oracle (oracle/sacd_oracle.c, as it stands) timed on full
sweeps of the BASELINE configs on this machine's host cores.

For each config: t0 = ora_sacd_run with K = 0 (the three mode layouts, the init and f^0:
init work) and tK = ora_sacd_run with K sweeps; seconds per sweep = (tK - t0) / K.
Run with all host cores and, for c1-c3, with 1 thread.  One JSON line per (config,
threads).  The tensors come from sacd_inputs (generated on the GPU when there is one).
    python tools/oracle_timing.py [c1 c2 c3 c4 c5] [--sweeps K] [--threads all,1]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import sacd_inputs as SI  # noqa: E402


def tensor(cfg):
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    c, v = SI.make_tensor(cfg, device=dev)
    return np.ascontiguousarray(c.cpu().numpy().astype(np.uint32)), np.ascontiguousarray(v.cpu().numpy())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1", "c2", "c3", "c5", "c4"])
    ap.add_argument("--sweeps", type=int, default=0, help="0 = c1 200, c2 20, c3 4, c5 2, c4 2")
    ap.add_argument("--threads", default="all,1")
    ap.add_argument("--rank", type=int, default=None)
    a = ap.parse_args()
    O.build()
    ncores = os.cpu_count()
    for name in a.configs:
        cfg = SI.CONFIGS[name]
        R = a.rank or cfg.rank
        c, v = tensor(cfg)
        K = a.sweeps or {"c1": 200, "c2": 20, "c3": 4, "c5": 2, "c4": 2}.get(name, 2)
        for th in a.threads.split(","):
            if th == "1" and name in ("c4", "c5"):
                continue
            nt = ncores if th == "all" else int(th)
            O.set_threads(nt)
            t0 = 1e30
            for _ in range(2):  # init work (layout sorts, init, f^0): the smaller of two runs
                t = time.perf_counter()
                O.sacd_run(c, v, cfg.dims, R, cfg.seed, 0)
                t0 = min(t0, time.perf_counter() - t)
            t = time.perf_counter()
            r = O.sacd_run(c, v, cfg.dims, R, cfg.seed, K)
            tk = time.perf_counter() - t
            sps = (tk - t0) / K
            print(json.dumps({"config": name, "rank": R, "nnz": int(len(v)), "threads": nt, "host_cores": ncores,
                              "init_s": t0, "sweeps": K, "run_s": tk, "seconds_per_sweep": sps,
                              "sweeps_per_s": 1.0 / sps if sps > 0 else None,
                              "f_last": float(r["f"][-1])}), flush=True)
    O.set_threads(ncores)


if __name__ == "__main__":
    main()
