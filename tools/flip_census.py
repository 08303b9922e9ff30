"""Full flip census of a GPU run: for every mode pass of K sweeps, the oracle
re-runs the pass from the GPU's own state before it (factors, z_prev, the device's ti
history) over ALL rows, and every element decision is compared with the GPU's.  A mismatch
is a gate decided differently by the two sides on identical inputs: its relative
saturation margin |sp| / max(|z|, |z_prev|) (sp = z - z_prev for Eq 24, z_prev - z for
Eq 27, z for the k = 1 rule) shows whether it is a near-tie of the rounding differences
(fiber-factored / DMMA sums on the GPU, sequential sums in the oracle).
    python tools/flip_census.py [--config c4] [--sweeps 10] [--out gpurun_out/census.jsonl]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import sacd_inputs as SI  # noqa: E402
from paper_2003_03572_b200.sacd import Sacd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--sweeps", type=int, default=10)
    ap.add_argument("--rank", type=int, default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    cfg = SI.CONFIGS[a.config]
    R = a.rank or cfg.rank
    dims = cfg.dims
    c, v = SI.make_tensor(cfg, device="cuda")
    c, v = np.ascontiguousarray(c.cpu().numpy().astype(np.uint32)), np.ascontiguousarray(v.cpu().numpy())
    t = time.perf_counter()
    lays = [O.layout(c, v, dims, n) for n in range(3)]
    print(f"oracle layouts {time.perf_counter() - t:.1f} s", flush=True)
    out = open(a.out, "w") if a.out else None
    hist = [[], [], []]
    total = 0
    with Sacd(c, v, dims, R, cfg.seed) as g:
        for k in range(1, a.sweeps + 1):
            for n in range(3):
                t = time.perf_counter()
                am, bm = O.other_modes(dims, n)
                F = g.factors()
                Z = g.get_zprev(n)
                res = g.mode_update(n, decisions=True)
                H = O.hadamard(O.gram(F[am]), O.gram(F[bm]))
                ia, ib, vv, rp = lays[n]
                M = O.mttkrp_layout(rp, ia, ib, vv, F[am], F[bm])
                br = O.branch(k, hist[n])
                Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, F[n], Z, br, decisions=True)
                Fg = g.factors(n)
                Zg = g.get_zprev(n)
                mism = np.argwhere(res["decisions"] != dec)
                recs = []
                for i, r in mism[:200]:
                    z_o, z_g, z0 = zp[i, r], Zg[i, r], Z[i, r]
                    sp = z_o if br == O.BR_FIRST else (z_o - z0 if br == O.BR_EQ24 else z0 - z_o)
                    recs.append({"row": int(i), "col": int(r), "z_prev": float(z0), "z_oracle": float(z_o),
                                 "z_gpu": float(z_g), "sp_oracle": float(sp),
                                 "margin": float(abs(sp) / max(abs(z_o), abs(z0), 1e-300)),
                                 "gpu_sel": int(res["decisions"][i, r]), "oracle_sel": int(dec[i, r])})
                # agreement of the rest: elements decided the same way
                same = res["decisions"] == dec
                rowsame = same.all(axis=1)
                ferr = 0.0
                if rowsame.any():
                    fo, fg = Fn[rowsame], Fg[rowsame]
                    floor = 1e-3 * np.abs(fo).max(axis=0, keepdims=True)
                    den = np.maximum(np.abs(fo), floor)
                    den[den == 0] = 1.0
                    ferr = float((np.abs(fg - fo) / den).max())
                rec = {"k": k, "mode": n, "branch_gpu_rule": int(br), "decisions": int(dec.size),
                       "mismatches": int(len(mism)), "E_gpu": res["E"], "E_oracle": int(E),
                       "ti_gpu": res["ti"], "ti_oracle": ti, "factor_err_rows_same": ferr,
                       "flips": recs, "seconds": time.perf_counter() - t}
                total += len(mism)
                hist[n].append(res["ti"])
                line = json.dumps(rec)
                print(line[:600], flush=True)
                if out:
                    out.write(line + "\n")
                    out.flush()
    print(f"census done: {total} mismatched decisions", flush=True)


if __name__ == "__main__":
    main()
