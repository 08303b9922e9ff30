"""Thin ctypes binding of libsacd (include/sacd.h).

Argument marshalling only: every step of the SaCD path runs in the CUDA kernels of
libsacd.so.  There is no CPU fallback -- if the library is missing or no GPU is
present, the constructor raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SACD_LIB selects another flavour of the same library (paper_2003_03572_b200/build.py):
# libsacd_tuning.so (MTTKRP tuning variants) or libsacd_debug.so (device-side asserts).
LIB_PATH = os.path.join(HERE, os.environ.get("SACD_LIB", "libsacd.so"))

SACD_OK, SACD_EINVAL, SACD_ERANGE, SACD_EDUP, SACD_ENONFINITE, SACD_ENOMEM, SACD_ECUDA, SACD_ENCCL, SACD_ESTATE = (
    0, -1, -2, -3, -4, -5, -6, -7, -8)
STATUS = {0: "OK", -1: "EINVAL", -2: "ERANGE", -3: "EDUP", -4: "ENONFINITE", -5: "ENOMEM", -6: "ECUDA",
          -7: "ENCCL", -8: "ESTATE"}
L_DIAG, L_FROB = 0, 1
VARIANT_GS_LAGGED, VARIANT_SELECT_OFF, VARIANT_JACOBI, VARIANT_SNAPSHOT = 0, 1, 2, 3
F64, F32 = 0, 1
BR_AUTO, BR_FIRST, BR_EQ24, BR_EQ27 = -1, 0, 1, 2
NUM_KCLASS = 6
ABI_VERSION = 2
KCLASS = ("mttkrp", "fixup", "prepare", "rows", "gram", "finalize")

# exported symbols declared in include/sacd.h (checked by tests/test_abi.py)
EXPORTS = ("sacd_default_options", "sacd_init", "sacd_iterate", "sacd_sync", "sacd_fit", "sacd_factors",
           "sacd_stats", "sacd_get_info", "sacd_free", "sacd_last_error", "sacd_set_factors", "sacd_get_zprev",
           "sacd_set_zprev", "sacd_mttkrp", "sacd_time_mttkrp", "sacd_gram", "sacd_hessian", "sacd_mode_update",
           "sacd_layout", "sacd_profile_read", "sacd_profile_reset", "sacd_shard_plan", "sacd_abi_sizes",
           "sacd_nccl_unique_id", "sacd_predict", "sacd_rmse", "sacd_set_profile", "sacd_replica_factors")


class Options(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("precision", C.c_int32), ("l_mode", C.c_int32),
                ("variant", C.c_int32), ("device", C.c_int32), ("world_size", C.c_int32), ("rank", C.c_int32),
                ("nccl_unique_id", C.c_void_p), ("stream", C.c_void_p), ("use_graph", C.c_int32),
                ("profile", C.c_int32), ("nnz_per_item", C.c_int32), ("mttkrp_variant", C.c_int32),
                ("force_sharded", C.c_int32), ("emulate_ranks", C.c_int32), ("reserved", C.c_int32 * 4)]


class IterStats(C.Structure):
    _fields_ = [("k", C.c_int32), ("branch", C.c_int32 * 3), ("objective", C.c_double), ("fit", C.c_double),
                ("ti", C.c_double * 3), ("E", C.c_int64 * 3), ("E_changed", C.c_int64 * 3),
                ("ms", C.c_double)]


class Info(C.Structure):
    _fields_ = [("dims", C.c_int64 * 3), ("nnz", C.c_int64), ("rank", C.c_int32), ("pitch", C.c_int32),
                ("precision", C.c_int32), ("l_mode", C.c_int32), ("variant", C.c_int32), ("k", C.c_int32),
                ("mode_a", C.c_int32 * 3), ("mode_b", C.c_int32 * 3), ("xnorm2", C.c_double),
                ("items", C.c_int64 * 3), ("split_rows", C.c_int64 * 3), ("device_bytes", C.c_int64),
                ("kernels_per_sweep", C.c_int32), ("world_size", C.c_int32), ("world_rank", C.c_int32),
                ("sharded_ranks", C.c_int32), ("delta_exchange", C.c_int32), ("delta_elems_sent", C.c_int64),
                ("full_elems_equiv", C.c_int64), ("fibers", C.c_int64 * 3), ("uniform_values", C.c_int32),
                ("uniform_value", C.c_double)]


class SacdError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libsacd.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    P, i32, i64, u64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    L.sacd_default_options.argtypes = [C.POINTER(Options)]
    L.sacd_default_options.restype = None
    L.sacd_init.argtypes = [C.POINTER(P), P, P, i64, P, i32, u64, C.POINTER(Options)]
    L.sacd_iterate.argtypes = [P, i32]
    L.sacd_sync.argtypes = [P]
    L.sacd_fit.argtypes = [P, C.POINTER(d), C.POINTER(d)]
    L.sacd_factors.argtypes = [P, i32, P, i64]
    L.sacd_stats.argtypes = [P, C.POINTER(IterStats), i32, C.POINTER(i32)]
    L.sacd_get_info.argtypes = [P, C.POINTER(Info)]
    L.sacd_free.argtypes = [P]
    L.sacd_free.restype = None
    L.sacd_last_error.restype = C.c_char_p
    L.sacd_set_factors.argtypes = [P, i32, P, i64]
    L.sacd_get_zprev.argtypes = [P, i32, P, i64]
    L.sacd_replica_factors.argtypes = [P, i32, i32, P, i64]
    L.sacd_set_zprev.argtypes = [P, i32, P, i64]
    L.sacd_mttkrp.argtypes = [P, i32, P, i64]
    L.sacd_time_mttkrp.argtypes = [P, i32, i32, C.POINTER(d)]
    L.sacd_gram.argtypes = [P, i32, P]
    L.sacd_hessian.argtypes = [P, i32, P]
    L.sacd_mode_update.argtypes = [P, i32, i32, P, C.POINTER(d), C.POINTER(i64), C.POINTER(i64)]
    L.sacd_layout.argtypes = [P, i32, P, P, P, P]
    L.sacd_profile_read.argtypes = [P, P, P]
    L.sacd_profile_reset.argtypes = [P]
    L.sacd_nccl_unique_id.argtypes = [P]
    L.sacd_abi_sizes.argtypes = [P]
    L.sacd_shard_plan.argtypes = [P, i64, i32, i32, P]
    L.sacd_predict.argtypes = [P, P, i64, P]
    L.sacd_set_profile.argtypes = [P, i32]
    L.sacd_rmse.argtypes = [P, P, P, i64, C.POINTER(d)]
    sz = (C.c_int32 * 4)()
    L.sacd_abi_sizes(sz)
    if tuple(sz) != (ABI_VERSION, C.sizeof(Options), C.sizeof(IterStats), C.sizeof(Info)):
        raise RuntimeError(f"libsacd ABI mismatch: library {tuple(sz)} vs binding "
                           f"{(ABI_VERSION, C.sizeof(Options), C.sizeof(IterStats), C.sizeof(Info))}")
    _lib = L
    return L


def _check(rc):
    if rc != SACD_OK:
        raise SacdError(rc, load_library().sacd_last_error().decode(errors="replace"))


def _ptr(x):
    """Device or host pointer of a torch tensor or numpy array (no copies)."""
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    return C.c_void_p(x.ctypes.data)


def _np(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _torch_check(x, what, ncols):
    """A torch tensor is passed to the library by data_ptr() without a copy, so its layout
    must already be the one sacd.h declares: coords int32/uint32 (n, 3) contiguous, values
    float32 (n,) contiguous.  Anything else would be silently reinterpreted: refuse it."""
    import torch
    ok_dt = (torch.int32,) + ((torch.uint32,) if hasattr(torch, "uint32") else ()) if ncols == 3 else (torch.float32,)
    if x.dtype not in ok_dt:
        raise TypeError(f"{what}: dtype {x.dtype}, expected {' or '.join(str(d) for d in ok_dt)}")
    if ncols == 3 and (x.dim() != 2 or x.shape[1] != 3):
        raise ValueError(f"{what}: shape {tuple(x.shape)}, expected (n, 3)")
    if ncols == 1 and x.dim() != 1:
        raise ValueError(f"{what}: shape {tuple(x.shape)}, expected (n,)")
    if not x.is_contiguous():
        raise ValueError(f"{what}: tensor must be contiguous")
    return x


def _coords_arg(c):
    if hasattr(c, "data_ptr"):
        return _torch_check(c, "coords", 3)
    return _np(np.asarray(c).reshape(-1, 3), np.uint32)


def _vals_arg(v):
    if hasattr(v, "data_ptr"):
        return _torch_check(v, "vals", 1)
    return _np(v, np.float32)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (call on rank 0, broadcast to the others)."""
    buf = C.create_string_buffer(128)
    _check(load_library().sacd_nccl_unique_id(buf))
    return buf.raw


def shard_plan(row_ptr, world, rank):
    """sacd_shard_plan: (lo, hi, rlo, rhi, head) of `rank` for one mode's row_ptr."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    out = np.zeros(5, np.int64)
    _check(load_library().sacd_shard_plan(_ptr(rp), rp.shape[0] - 1, int(world), int(rank), _ptr(out)))
    return tuple(int(x) for x in out)


class Sacd:
    """One SaCD factorisation context on one GPU (see include/sacd.h)."""

    def __init__(self, coords, vals, dims, rank, seed, *, precision="f64", l_mode="diag", variant="gs",
                 device=-1, stream=None, use_graph=True, profile=False, nnz_per_item=0, mttkrp_variant=0,
                 world_size=1, world_rank=0, nccl_id=None, force_sharded=False, emulate_ranks=0, rows_variant=0, ablk_rows=0,
                 gram_variant=0, exchange="full"):
        L = load_library()
        o = Options()
        L.sacd_default_options(C.byref(o))
        o.precision = {"f64": F64, "f32": F32}[precision]
        o.l_mode = {"diag": L_DIAG, "frob": L_FROB}[l_mode]
        o.variant = {"gs": VARIANT_GS_LAGGED, "select_off": VARIANT_SELECT_OFF, "jacobi": VARIANT_JACOBI,
                     "snapshot": VARIANT_SNAPSHOT}[variant]
        o.device = int(device)
        o.stream = stream
        o.use_graph = int(bool(use_graph))
        o.profile = int(bool(profile))
        o.nnz_per_item = int(nnz_per_item)
        o.mttkrp_variant = int(mttkrp_variant)
        o.world_size = int(world_size)
        o.rank = int(world_rank)
        o.force_sharded = int(bool(force_sharded))
        o.emulate_ranks = int(emulate_ranks)
        o.reserved[0] = int(rows_variant)
        o.reserved[1] = int(ablk_rows)
        o.reserved[2] = int(gram_variant)
        o.reserved[3] = {"full": 0, "delta": 1, "p2p": 2}[exchange]
        self._nccl_id = None
        if nccl_id is not None:
            self._nccl_id = C.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_unique_id = C.cast(self._nccl_id, C.c_void_p)
        coords, vals = _coords_arg(coords), _vals_arg(vals)
        nnz = int(vals.shape[0])
        if int(coords.shape[0]) != nnz:
            raise ValueError(f"coords has {int(coords.shape[0])} rows, vals {nnz} entries")
        self._keep = (coords, vals)
        d = (C.c_int64 * 3)(*[int(x) for x in dims])
        h = C.c_void_p()
        _check(L.sacd_init(C.byref(h), _ptr(coords), _ptr(vals), nnz, d, int(rank), int(seed) & (2 ** 64 - 1),
                           C.byref(o)))
        self._keep = None
        self._h = h
        self.dims = tuple(int(x) for x in dims)
        self.rank = int(rank)
        self.precision = precision

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            load_library().sacd_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- main calls
    def iterate(self, n=1):
        _check(load_library().sacd_iterate(self._h, int(n)))

    def sync(self):
        _check(load_library().sacd_sync(self._h))

    def fit(self):
        f, ft = C.c_double(), C.c_double()
        _check(load_library().sacd_fit(self._h, C.byref(f), C.byref(ft)))
        return f.value, ft.value

    def factors(self, mode=None, out=None):
        """The factors as fp64 host arrays (I_n x R).  out: optional preallocated C-contiguous
        float64 array(s) of that shape (a list of three for mode=None); pinned memory (e.g. a
        numpy view of a torch pin_memory tensor) is copied into directly by the library."""
        if mode is None:
            return [self.factors(n, None if out is None else out[n]) for n in range(3)]
        shape = (self.dims[mode], self.rank)
        if out is None:
            out = np.zeros(shape, np.float64)
        elif not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.shape == shape
                  and out.flags.c_contiguous):
            raise ValueError(f"factors: out must be a C-contiguous float64 array of shape {shape}")
        _check(load_library().sacd_factors(self._h, int(mode), _ptr(out), self.rank))
        return out

    def stats(self):
        n = C.c_int32()
        buf = (IterStats * 4096)()
        _check(load_library().sacd_stats(self._h, buf, 4096, C.byref(n)))
        out = []
        for i in range(n.value):
            s = buf[i]
            out.append(dict(k=s.k, branch=list(s.branch), objective=s.objective, fit=s.fit, ti=list(s.ti),
                            E=list(s.E), E_changed=list(s.E_changed), ms=s.ms))
        return out

    def info(self):
        i = Info()
        _check(load_library().sacd_get_info(self._h, C.byref(i)))
        return dict(dims=list(i.dims), nnz=i.nnz, rank=i.rank, pitch=i.pitch, precision=i.precision,
                    l_mode=i.l_mode, variant=i.variant, k=i.k, mode_a=list(i.mode_a), mode_b=list(i.mode_b),
                    xnorm2=i.xnorm2, items=list(i.items), split_rows=list(i.split_rows),
                    device_bytes=i.device_bytes, kernels_per_sweep=i.kernels_per_sweep,
                    world_size=i.world_size, world_rank=i.world_rank, sharded_ranks=i.sharded_ranks,
                    delta_exchange=i.delta_exchange, delta_elems_sent=i.delta_elems_sent,
                    full_elems_equiv=i.full_elems_equiv, fibers=list(i.fibers),
                    uniform_values=i.uniform_values, uniform_value=i.uniform_value)

    # -- component entry points
    def set_factors(self, mode, F):
        F = _np(F, np.float64)
        assert F.shape == (self.dims[mode], self.rank)
        _check(load_library().sacd_set_factors(self._h, int(mode), _ptr(F), self.rank))

    def replica_factors(self, shard, mode):
        """Factor `mode` as held by shard `shard` (its own replica with exchange='p2p' and
        emulated ranks)."""
        out = np.zeros((self.dims[mode], self.rank), np.float64)
        _check(load_library().sacd_replica_factors(self._h, int(shard), int(mode), _ptr(out), self.rank))
        return out

    def get_zprev(self, mode):
        out = np.zeros((self.dims[mode], self.rank), np.float64)
        _check(load_library().sacd_get_zprev(self._h, int(mode), _ptr(out), self.rank))
        return out

    def set_zprev(self, mode, Z):
        Z = _np(Z, np.float64)
        assert Z.shape == (self.dims[mode], self.rank)
        _check(load_library().sacd_set_zprev(self._h, int(mode), _ptr(Z), self.rank))

    def mttkrp(self, mode):
        out = np.zeros((self.dims[mode], self.rank), np.float64)
        _check(load_library().sacd_mttkrp(self._h, int(mode), _ptr(out), self.rank))
        return out

    def time_mttkrp(self, mode, reps=10):
        ms = C.c_double()
        _check(load_library().sacd_time_mttkrp(self._h, int(mode), int(reps), C.byref(ms)))
        return ms.value

    def gram(self, mode):
        out = np.zeros((self.rank, self.rank), np.float64)
        _check(load_library().sacd_gram(self._h, int(mode), _ptr(out)))
        return out

    def hessian(self, mode):
        out = np.zeros((self.rank, self.rank), np.float64)
        _check(load_library().sacd_hessian(self._h, int(mode), _ptr(out)))
        return out

    def mode_update(self, mode, branch=BR_AUTO, decisions=False):
        dec = np.zeros((self.dims[mode], self.rank), np.uint8) if decisions else None
        ti, E, Ech = C.c_double(), C.c_int64(), C.c_int64()
        _check(load_library().sacd_mode_update(self._h, int(mode), int(branch),
                                               _ptr(dec) if dec is not None else None,
                                               C.byref(ti), C.byref(E), C.byref(Ech)))
        return dict(ti=ti.value, E=E.value, E_changed=Ech.value, decisions=dec)

    def layout(self, mode):
        nnz = self.info()["nnz"]
        ia = np.zeros(nnz, np.uint32)
        ib = np.zeros(nnz, np.uint32)
        v = np.zeros(nnz, np.float32)
        rp = np.zeros(self.dims[mode] + 1, np.int64)
        _check(load_library().sacd_layout(self._h, int(mode), _ptr(ia), _ptr(ib), _ptr(v), _ptr(rp)))
        return ia, ib, v, rp

    def profile_read(self):
        ms = np.zeros(NUM_KCLASS, np.float64)
        n = np.zeros(NUM_KCLASS, np.int64)
        _check(load_library().sacd_profile_read(self._h, _ptr(ms), _ptr(n)))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(KCLASS)}

    def set_profile(self, on):
        _check(load_library().sacd_set_profile(self._h, int(bool(on))))

    def profile_reset(self):
        _check(load_library().sacd_profile_reset(self._h))

    # ---- held-out evaluation
    def predict(self, coords):
        """Eq 8 at the given (n, 3) coordinates (host numpy or device torch); fp64 numpy."""
        c = _coords_arg(coords)
        n = int(c.shape[0])
        out = np.zeros(n, np.float64)
        _check(load_library().sacd_predict(self._h, _ptr(c), n, _ptr(out)))
        return out

    def rmse(self, coords, vals):
        """Eq 30 on held-out entries (coords (n, 3) u32, vals fp32; host or device)."""
        c, v = _coords_arg(coords), _vals_arg(vals)
        if int(c.shape[0]) != int(v.shape[0]):
            raise ValueError("coords and vals lengths differ")
        r = C.c_double()
        _check(load_library().sacd_rmse(self._h, _ptr(c), _ptr(v), int(c.shape[0]), C.byref(r)))
        return r.value
