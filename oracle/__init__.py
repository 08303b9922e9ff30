"""fp64 CPU oracle for SaCD (arXiv 2003.03572) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
legs may import this package.  The product path (paper_2003_03572_b200/) never imports
it, and it never imports the product path: the two share no code.  The arithmetic lives
in `sacd_oracle.c` (plain C, fp64, one function per paper step, citations inline); this
module only compiles it with gcc and marshals numpy arrays through ctypes.

Parity status per function (pins in tests/test_oracle_pins.py):
  layout, init, gram/hadamard/frobenius, mttkrp, mode_pass (step, importance,
  selection), objective (dense, sparse, Gram trick), predict / rmse  -- pinned.
  Selection dynamics end to end (trajectories of E / ti)  -- parity unpinned (the paper
  prints no trace); they are only checked for internal consistency.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ORACLE_SRC / ORACLE_LIB: used only by tests/test_oracle_mutations.py, which compiles
# deliberately broken copies of the oracle to show that the pins catch each mutation.
SRC = os.environ.get("ORACLE_SRC", os.path.join(HERE, "sacd_oracle.c"))
LIB = os.environ.get("ORACLE_LIB", os.path.join(HERE, "liboracle.so"))

BR_FIRST, BR_EQ24, BR_EQ27 = 0, 1, 2
VAR_GS_LAGGED, VAR_SELECT_OFF, VAR_JACOBI, VAR_SNAPSHOT = 0, 1, 2, 3
L_DIAG, L_FROB = 0, 1


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-ffp-contract=off", "-o", LIB, SRC, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        i64, i32, u64, f64 = C.c_int64, C.c_int, C.c_uint64, C.c_double
        L.ora_set_threads.argtypes = [i32]
        L.ora_max_threads.restype = i32
        L.ora_rand.argtypes = [u64, u64, u64]
        L.ora_rand.restype = u64
        L.ora_init_factors.argtypes = [P, i32, u64, P, P, P]
        L.ora_other_modes.argtypes = [P, i32, P, P]
        L.ora_layout.argtypes = [i64, P, P, P, i32, P, P, P, P]
        L.ora_gram.argtypes = [P, i64, i32, P]
        L.ora_hadamard.argtypes = [P, P, i64, P]
        L.ora_frobenius.argtypes = [P, i32]
        L.ora_frobenius.restype = f64
        L.ora_mttkrp.argtypes = [i64, i32, P, P, P, P, P, P, P]
        L.ora_mode_pass.argtypes = [i64, i32, P, P, P, P, i32, i32, i32, P, P, P, P, P]
        L.ora_branch.argtypes = [i32, P, i32]
        L.ora_mode_pass_snapshot.argtypes = [i64, i32, P, P, P, P, i32, f64, i32, i32, P, P, P, P, P, P]
        L.ora_objective_dense.argtypes = [P, i64, P, P, P, P, P, i32, P]
        L.ora_objective_sparse.argtypes = [P, i64, P, P, P, P, P, i32, P]
        L.ora_sacd_run.argtypes = [i64, P, P, P, i32, u64, i32, i32, i32, P, P, P, P, P, P, P, P, P, P, P]
        L.ora_predict.argtypes = [i64, P, P, P, P, P, i32, P]
        L.ora_rmse.argtypes = [i64, P, P, P, P, P, P, i32, P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _dims(dims):
    return np.ascontiguousarray(np.asarray(dims, dtype=np.int64))


def _coo(coords, vals):
    c = np.ascontiguousarray(np.asarray(coords).astype(np.uint32).reshape(-1, 3))
    v = np.ascontiguousarray(np.asarray(vals, dtype=np.float32).reshape(-1))
    return c, v


ERRORS = {-1: "EINVAL", -2: "ERANGE", -3: "EDUP", -4: "ENONFINITE", -5: "ENOMEM"}


class OracleError(RuntimeError):
    def __init__(self, rc):
        super().__init__(f"oracle error {rc} ({ERRORS.get(rc, '?')})")
        self.rc = rc


def _check(rc):
    if rc != 0:
        raise OracleError(rc)


def set_threads(n: int):
    lib().ora_set_threads(int(n))


def max_threads() -> int:
    return lib().ora_max_threads()


def rand(seed, tag, ctr) -> int:
    return lib().ora_rand(seed, tag, ctr)


def other_modes(dims, n):
    a, b = C.c_int(), C.c_int()
    lib().ora_other_modes(_p(_dims(dims)), n, C.byref(a), C.byref(b))
    return a.value, b.value


def init_factors(dims, R, seed):
    d = _dims(dims)
    F = [np.zeros((int(d[n]), R), np.float64) for n in range(3)]
    lib().ora_init_factors(_p(d), R, seed, _p(F[0]), _p(F[1]), _p(F[2]))
    return F


def layout(coords, vals, dims, n):
    c, v = _coo(coords, vals)
    d = _dims(dims)
    nnz = v.shape[0]
    ia = np.zeros(nnz, np.uint32)
    ib = np.zeros(nnz, np.uint32)
    vv = np.zeros(nnz, np.float32)
    rp = np.zeros(int(d[n]) + 1, np.int64)
    _check(lib().ora_layout(nnz, _p(c), _p(v), _p(d), n, _p(ia), _p(ib), _p(vv), _p(rp)))
    return ia, ib, vv, rp


def gram(F):
    F = np.ascontiguousarray(F, dtype=np.float64)
    R = F.shape[1]
    G = np.zeros((R, R), np.float64)
    lib().ora_gram(_p(F), F.shape[0], R, _p(G))
    return G


def hadamard(X, Y):
    X = np.ascontiguousarray(X, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    assert X.shape == Y.shape
    Z = np.zeros_like(X)
    lib().ora_hadamard(_p(X), _p(Y), X.size, _p(Z))
    return Z


def frobenius(H):
    H = np.ascontiguousarray(H, dtype=np.float64)
    return lib().ora_frobenius(_p(H), H.shape[0])


def mttkrp_layout(rp, ia, ib, vv, A, B):
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    R = A.shape[1]
    I = rp.shape[0] - 1
    M = np.zeros((I, R), np.float64)
    lib().ora_mttkrp(I, R, _p(rp), _p(ia), _p(ib), _p(vv), _p(A), _p(B), _p(M))
    return M


def mttkrp(coords, vals, dims, n, F):
    """M for mode n given the three factors F=[U,V,W] (own factor unused)."""
    a, b = other_modes(dims, n)
    ia, ib, vv, rp = layout(coords, vals, dims, n)
    return mttkrp_layout(rp, ia, ib, vv, F[a], F[b])


def mode_hessian(F, dims, n):
    a, b = other_modes(dims, n)
    return hadamard(gram(F[a]), gram(F[b]))


def mode_pass(M, H, F, zprev, branch, l_mode=L_DIAG, jacobi=False, decisions=False):
    """One SaCD pass over the rows of one factor (in place on copies); returns
    (F_new, zprev_new, ti, E, E_changed, mdot, decisions|None)."""
    F = np.array(F, dtype=np.float64, copy=True, order="C")
    zp = np.array(zprev, dtype=np.float64, copy=True, order="C")
    M = np.ascontiguousarray(M, dtype=np.float64)
    H = np.ascontiguousarray(H, dtype=np.float64)
    I, R = F.shape
    dec = np.zeros(I * R, np.uint8) if decisions else None
    ti, E, Ech, md = C.c_double(), C.c_int64(), C.c_int64(), C.c_double()
    _check(lib().ora_mode_pass(I, R, _p(M), _p(H), _p(F), _p(zp), branch, l_mode, int(bool(jacobi)),
                               _p(dec) if dec is not None else None, C.byref(ti), C.byref(E), C.byref(Ech),
                               C.byref(md)))
    return F, zp, ti.value, E.value, Ech.value, md.value, (dec.reshape(I, R) if dec is not None else None)


def mode_pass_snapshot(M, H, F, zprev, first, ti_prev, l_mode=L_DIAG, decisions=False, branch=-1):
    """Snapshot-scored pass (reading C10'); returns
    (F_new, zprev_new, ti, E, E_changed, mdot, decisions|None, branch)."""
    F = np.array(F, dtype=np.float64, copy=True, order="C")
    zp = np.array(zprev, dtype=np.float64, copy=True, order="C")
    M = np.ascontiguousarray(M, dtype=np.float64)
    H = np.ascontiguousarray(H, dtype=np.float64)
    I, R = F.shape
    dec = np.zeros(I * R, np.uint8) if decisions else None
    ti, E, Ech, md, br = C.c_double(), C.c_int64(), C.c_int64(), C.c_double(), C.c_int32()
    _check(lib().ora_mode_pass_snapshot(I, R, _p(M), _p(H), _p(F), _p(zp), int(bool(first)), float(ti_prev),
                                        int(branch), l_mode, _p(dec) if dec is not None else None, C.byref(ti),
                                        C.byref(E), C.byref(Ech), C.byref(md), C.byref(br)))
    return (F, zp, ti.value, E.value, Ech.value, md.value, (dec.reshape(I, R) if dec is not None else None),
            br.value)


def branch(k, ti_hist, variant=VAR_GS_LAGGED):
    h = np.ascontiguousarray(np.asarray(list(ti_hist) + [0.0, 0.0], dtype=np.float64))
    return lib().ora_branch(k, _p(h), variant)


def objective_dense(coords, vals, dims, F):
    c, v = _coo(coords, vals)
    d = _dims(dims)
    F = [np.ascontiguousarray(x, dtype=np.float64) for x in F]
    f = C.c_double()
    _check(lib().ora_objective_dense(_p(d), v.shape[0], _p(c), _p(v), _p(F[0]), _p(F[1]), _p(F[2]),
                                     F[0].shape[1], C.byref(f)))
    return f.value


def objective_sparse(coords, vals, dims, F):
    c, v = _coo(coords, vals)
    d = _dims(dims)
    F = [np.ascontiguousarray(x, dtype=np.float64) for x in F]
    f = C.c_double()
    _check(lib().ora_objective_sparse(_p(d), v.shape[0], _p(c), _p(v), _p(F[0]), _p(F[1]), _p(F[2]),
                                      F[0].shape[1], C.byref(f)))
    return f.value


def sacd_run(coords, vals, dims, R, seed, K, l_mode=L_DIAG, variant=VAR_GS_LAGGED, init=None):
    """Full Alg 1 run; returns a dict with U, V, W, f[K+1], E/Ech/ti/branch [K,3], zprev, xnorm2."""
    c, v = _coo(coords, vals)
    d = _dims(dims)
    F = [np.zeros((int(d[n]), R), np.float64) for n in range(3)]
    f = np.zeros(K + 1, np.float64)
    E = np.zeros((K, 3), np.int64)
    Ech = np.zeros((K, 3), np.int64)
    ti = np.zeros((K, 3), np.float64)
    br = np.zeros((K, 3), np.int32)
    zp = np.zeros(int(d.sum()) * R, np.float64)
    xn = C.c_double()
    ini = None
    if init is not None:
        ini = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64).reshape(-1) for x in init]))
    _check(lib().ora_sacd_run(v.shape[0], _p(c), _p(v), _p(d), R, seed, K, l_mode, variant,
                              _p(ini) if ini is not None else None, _p(F[0]), _p(F[1]), _p(F[2]),
                              _p(f), _p(E), _p(Ech), _p(ti), _p(br), _p(zp), C.byref(xn)))
    zs, o = [], 0
    for n in range(3):
        zs.append(zp[o:o + int(d[n]) * R].reshape(int(d[n]), R))
        o += int(d[n]) * R
    return dict(U=F[0], V=F[1], W=F[2], F=F, f=f, E=E, Ech=Ech, ti=ti, branch=br, zprev=zs, xnorm2=xn.value)


def fit_from_f(f, xnorm2):
    """Reading C16: fit = 1 - sqrt(f)/||X||."""
    return 1.0 - np.sqrt(np.maximum(f, 0.0)) / np.sqrt(xnorm2) if xnorm2 > 0 else 0.0


def predict(coords, dims, F):
    """Eq 8 at the given coordinates (u32 [n][3])."""
    c = np.ascontiguousarray(np.asarray(coords, dtype=np.uint32).reshape(-1, 3))
    d = _dims(dims)
    F = [np.ascontiguousarray(x, dtype=np.float64) for x in F]
    out = np.zeros(c.shape[0], np.float64)
    _check(lib().ora_predict(c.shape[0], _p(c), _p(d), _p(F[0]), _p(F[1]), _p(F[2]), F[0].shape[1], _p(out)))
    return out


def rmse(coords, vals, dims, F):
    """Eq 30: held-out RMSE of the CP model F = [U, V, W]."""
    c, v = _coo(coords, vals)
    d = _dims(dims)
    F = [np.ascontiguousarray(x, dtype=np.float64) for x in F]
    r = C.c_double()
    _check(lib().ora_rmse(v.shape[0], _p(c), _p(v), _p(d), _p(F[0]), _p(F[1]), _p(F[2]), F[0].shape[1],
                          C.byref(r)))
    return r.value
