"""Checks run in a subprocess against another flavour of libsacd (tests/test_flavours.py sets
SACD_LIB before the library is loaded):
    debug  : libsacd_debug.so, every kernel family on ragged tensors with the device-side
             index / slot asserts compiled in (a failed assert traps -> ECUDA -> exit 1);
             the results must equal the product build's oracle parity bar.
    tuning : libsacd_tuning.so, every MTTKRP tuning variant is bitwise equal to the default
             kernel and within rounding of the oracle.
    python tests/_flavour_checks.py debug|tuning"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_2003_03572_b200.sacd import Sacd  # noqa: E402
from test_gpu_parity import check_pair, factor_err, ragged_tensor  # noqa: E402


def debug():
    cases = [
        ((300, 200, 50), 20000, ((2, 1, 3000), (0, 5, 900), (1, 199, 1500)),
         [dict(R=5), dict(R=40), dict(R=64), dict(R=200), dict(R=40, precision="f32"),
          dict(R=40, variant="snapshot"), dict(R=12, variant="jacobi"), dict(R=64, emulate_ranks=3),
          dict(R=40, emulate_ranks=8, exchange="delta"), dict(R=64, emulate_ranks=3, exchange="p2p"),
          dict(R=64, nnz_per_item=16)]),
        ((120, 80, 16), 60000, ((2, 1, 900), (0, 5, 700)), [dict(R=24), dict(R=32), dict(R=64)]),
        ((90, 70, 40), -12000, ((2, 3, 1500), (0, 7, 900)), [dict(R=64), dict(R=100), dict(R=256)]),  # binary
    ]
    for dims, nnz, heavy, runs in cases:
        c, v = ragged_tensor(dims, abs(nnz), 8, heavy_rows=heavy)
        if nnz < 0:  # all values equal: the MTTKRP path without per-nonzero values
            v = np.full_like(v, 1.0)
        for kw in runs:
            kw = dict(kw)
            R = kw.pop("R")
            K = 4
            with Sacd(c, v, dims, R, 17, **kw) as g:
                f0 = g.fit()[0]
                g.iterate(K)
                st = g.stats()
                Fg = g.factors()
                g.rmse(c[:500], v[:500])
                for n in range(3):
                    g.mttkrp(n)
            if kw.get("precision", "f64") == "f64":
                variant = {"snapshot": O.VAR_SNAPSHOT, "jacobi": O.VAR_JACOBI}.get(kw.get("variant"), O.VAR_GS_LAGGED)
                ora = O.sacd_run(c, v, dims, R, 17, K, variant=variant)
                fg = np.array([f0] + [s["objective"] for s in st])
                check_pair(fg, Fg, np.array([s["E"] for s in st]), np.array([s["branch"] for s in st]), ora)
            print(f"debug build ok: dims {dims} R={R} {kw}", flush=True)


def tuning():
    dims = (53, 31, 67)
    c, v = ragged_tensor(dims, 5000, 17, heavy_rows=((0, 1, 900), (1, 4, 500), (2, 7, 800)))
    for precision in ("f64", "f32"):
        for R in (33, 64, 128, 256):
            F = O.init_factors(dims, R, 5)
            Mo = [O.mttkrp(c, v, dims, n, F) for n in range(3)]
            ref = None
            for var in (1, 10, 13, 20, 22, 24, 26, 27, 39, 40, 43, 60, 62, 0):
                if var == 39 and precision == "f32":
                    continue
                if var >= 50 and not (precision == "f64" and R in (33, 64)):
                    continue
                with Sacd(c, v, dims, R, 5, precision=precision, nnz_per_item=48, mttkrp_variant=var) as g:
                    Ms = [g.mttkrp(n) for n in range(3)]
                tol = 1e-12 if precision == "f64" else 1e-5
                for n in range(3):
                    scale = np.maximum(np.abs(Mo[n]).max(axis=0, keepdims=True), 1e-30)
                    assert (np.abs(Ms[n] - Mo[n]) / scale).max() <= tol, (var, n)
                if ref is None:
                    ref = Ms
                else:
                    for n in range(3):
                        assert np.array_equal(Ms[n], ref[n]), (precision, R, var, n)
            print(f"tuning variants bitwise equal: {precision} R={R}", flush=True)
    _ = factor_err


if __name__ == "__main__":
    {"debug": debug, "tuning": tuning}[sys.argv[1]]()
    print("FLAVOUR CHECKS PASSED")
