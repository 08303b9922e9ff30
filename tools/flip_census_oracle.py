"""Reverse flip census: the ORACLE's own trajectory (ora functions, pass by pass, exactly as
ora_sacd_run orders them) teacher-forces the GPU.  Before every mode pass the GPU gets the
oracle's factors and z_prev, runs the pass with the oracle's branch, and its element
decisions are compared with the oracle's.  A mismatch here is a gate the two arithmetics
decide differently at a state of the oracle's trajectory (tools/flip_census.py does the
same along the GPU's trajectory).  Also records, per pass, the max relative difference
between the GPU's and the oracle's updated factor and the objective of both trajectories
when --compare-run is given (the independent GPU run's f per sweep).
    python tools/flip_census_oracle.py [--config c4] [--sweeps 10] [--out f.jsonl]"""
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


def rel_err(Fg, Fo):
    floor = 1e-3 * np.abs(Fo).max(axis=0, keepdims=True)
    den = np.maximum(np.abs(Fo), floor)
    den[den == 0] = 1.0
    return float((np.abs(Fg - Fo) / den).max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--sweeps", type=int, default=10)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = SI.CONFIGS[a.config]
    R, dims = cfg.rank, cfg.dims
    c, v = SI.make_tensor(cfg, device="cuda")
    c, v = np.ascontiguousarray(c.cpu().numpy().astype(np.uint32)), np.ascontiguousarray(v.cpu().numpy())
    lays = [O.layout(c, v, dims, n) for n in range(3)]
    F = O.init_factors(dims, R, cfg.seed)
    Z = [np.zeros((dims[n], R)) for n in range(3)]
    hist = [[], [], []]
    xn2 = float((v.astype(np.float64) ** 2).sum())
    out = open(a.out, "w") if a.out else None
    total = 0
    with Sacd(c, v, dims, R, cfg.seed) as g:
        for k in range(1, a.sweeps + 1):
            for n in range(3):
                t = time.perf_counter()
                am, bm = O.other_modes(dims, n)
                for m in range(3):
                    g.set_factors(m, F[m])
                g.set_zprev(n, Z[n])
                br = O.branch(k, hist[n])
                res = g.mode_update(n, branch=br, decisions=True)
                H = O.hadamard(O.gram(F[am]), O.gram(F[bm]))
                ia, ib, vv, rp = lays[n]
                M = O.mttkrp_layout(rp, ia, ib, vv, F[am], F[bm])
                Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, F[n], Z[n], br, decisions=True)
                mism = np.argwhere(res["decisions"] != dec)
                Zg = g.get_zprev(n)
                recs = []
                for i, r in mism[:200]:
                    z_o, z0 = zp[i, r], Z[n][i, r]
                    sp = z_o if br == O.BR_FIRST else (z_o - z0 if br == O.BR_EQ24 else z0 - z_o)
                    recs.append({"row": int(i), "col": int(r), "z_prev": float(z0), "z_oracle": float(z_o),
                                 "z_gpu": float(Zg[i, r]), "sp_oracle": float(sp),
                                 "margin": float(abs(sp) / max(abs(z_o), abs(z0), 1e-300)),
                                 "gpu_sel": int(res["decisions"][i, r]), "oracle_sel": int(dec[i, r])})
                ferr = rel_err(g.factors(n), Fn)
                F[n], Z[n] = Fn, zp
                hist[n].append(ti)
                f = None
                if n == 2:
                    G = [O.gram(F[m]) for m in range(3)]
                    f = xn2 - 2.0 * md + float((G[0] * G[1] * G[2]).sum())
                rec = {"k": k, "mode": n, "branch": int(br), "decisions": int(dec.size), "mismatches": int(len(mism)),
                       "E_gpu": res["E"], "E_oracle": int(E), "ti_gpu": res["ti"], "ti_oracle": ti,
                       "factor_err": ferr, "f_oracle": f, "flips": recs, "seconds": time.perf_counter() - t}
                total += len(mism)
                line = json.dumps(rec)
                print(line[:700], flush=True)
                if out:
                    out.write(line + "\n")
                    out.flush()
    print(f"reverse census done: {total} mismatched decisions", flush=True)


if __name__ == "__main__":
    main()
