"""One oracle sweep of a config, function by function in ora_sacd_run's order (Grams of the
other factors, Hadamard, MTTKRP, row pass per mode; the three Grams of the objective), each
timed on all host cores: where the oracle's sweep time goes (calibrates bench.py's sample).
    python tools/oracle_breakdown.py [c4]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import sacd_inputs as SI  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = SI.CONFIGS[name]
import torch  # noqa: E402
c, v = SI.make_tensor(cfg, device="cuda" if torch.cuda.is_available() else "cpu")
c, v = c.cpu().numpy().astype(np.uint32), v.cpu().numpy()
dims, R = cfg.dims, cfg.rank
t = time.perf_counter()
lays = [O.layout(c, v, dims, n) for n in range(3)]
print(f"layouts {time.perf_counter() - t:.2f} s", flush=True)
F = O.init_factors(dims, R, cfg.seed)
Z = [np.zeros((dims[n], R)) for n in range(3)]
tot = 0.0
for n in range(3):
    a, b = O.other_modes(dims, n)
    t = time.perf_counter(); Ga = O.gram(F[a]); t1 = time.perf_counter() - t
    t = time.perf_counter(); Gb = O.gram(F[b]); t2 = time.perf_counter() - t
    t = time.perf_counter(); H = O.hadamard(Ga, Gb); t3 = time.perf_counter() - t
    ia, ib, vv, rp = lays[n]
    t = time.perf_counter(); M = O.mttkrp_layout(rp, ia, ib, vv, F[a], F[b]); t4 = time.perf_counter() - t
    t = time.perf_counter(); out = O.mode_pass(M, H, F[n], Z[n], O.BR_FIRST); t5 = time.perf_counter() - t
    F[n], Z[n] = out[0], out[1]
    tot += t1 + t2 + t3 + t4 + t5
    print(f"mode {n}: gram(F{a}) {t1:.2f} s, gram(F{b}) {t2:.2f} s, hadamard {t3:.3f} s, mttkrp {t4:.2f} s, "
          f"mode_pass {t5:.2f} s", flush=True)
t = time.perf_counter()
for n in range(3):
    O.gram(F[n])
t6 = time.perf_counter() - t
tot += t6
print(f"objective grams {t6:.2f} s; sweep total {tot:.2f} s on {O.max_threads()} threads", flush=True)
