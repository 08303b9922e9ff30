"""Calibration of the reference-arm sample: the oracle's MTTKRP cost per nonzero of one
slice as a function of the slice length (prefixes of the heaviest slices of c4), on this
host.  ora_mttkrp walks a slice once per column, so the cost per nonzero depends on how
much of the gathered factor rows stays in cache.
    python tools/oracle_slice_cost.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import sacd_inputs as SI  # noqa: E402

cfg = SI.CONFIGS["c4"]
import torch  # noqa: E402
c, v = SI.make_tensor(cfg, device="cuda" if torch.cuda.is_available() else "cpu")
c, v = c.cpu().numpy().astype(np.uint32), v.cpu().numpy()
dims, R = cfg.dims, cfg.rank
F = O.init_factors(dims, R, cfg.seed)
for n in (2, 0):
    a, b = O.other_modes(dims, n)
    ln = np.bincount(c[:, n].astype(np.int64), minlength=dims[n])
    for rank_pos in (0, 3, 30):
        row = int(np.argsort(-ln)[rank_pos])
        m = c[:, n] == row
        cs, vs = c[m].copy(), v[m]
        cs[:, n] = 0
        d2 = list(dims)
        d2[n] = 1
        ia, ib, vv, rp = O.layout(cs, vs, d2, n)
        L = int(rp[-1])
        for p in [1 << k for k in range(16, 25)] + [L]:
            if p > L:
                continue
            rp2 = np.array([0, p], np.int64)
            t = time.perf_counter()
            O.mttkrp_layout(rp2, ia[:p], ib[:p], vv[:p], F[a], F[b])
            dt = time.perf_counter() - t
            print(f"mode {n} row {row} (slice {L} nnz): prefix {p:9d}  {dt:8.3f} s  {dt / p * 1e9:7.1f} ns/nnz", flush=True)
