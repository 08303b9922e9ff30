"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle on the same
seeded inputs.  Bit-exact for the layout and the init; the north-star tolerances for
floating point: relative objective error <= 1e-4 per sweep and max relative factor error
<= 1e-3 (column-relative floor) after 10 sweeps."""
import numpy as np
import pytest

import oracle as O
import sacd_inputs as SI

pytestmark = pytest.mark.gpu

F_TOL = 1e-4
FACTOR_TOL = 1e-3


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2003_03572_b200 import build
    build.build()


def S(*a, **k):
    from paper_2003_03572_b200.sacd import Sacd
    return Sacd(*a, **k)


def factor_err(Fg, Fo):
    """max_{i,r} |Fg - Fo| / max(|Fo|, 1e-3 * max_i |Fo[:, r]|)"""
    floor = 1e-3 * np.abs(Fo).max(axis=0, keepdims=True)
    den = np.maximum(np.abs(Fo), floor)
    den = np.where(den == 0, 1.0, den)
    return float((np.abs(Fg - Fo) / den).max())


def ragged_tensor(dims, nnz, seed, heavy_rows=((0, 0, 300),)):
    """Uniform tensor plus heavy slices (mode, index, count) to force split rows."""
    cfg = SI.custom_config(dims, nnz, 4, cid=seed)
    c = SI.make_coords(cfg).numpy()
    extra = []
    rng = np.random.default_rng(seed)
    for mode, idx, cnt in heavy_rows:
        e = rng.integers(0, dims, size=(cnt, 3))
        e[:, mode] = idx
        extra.append(e)
    c = np.concatenate([c] + extra)
    key = (c[:, 0] * dims[1] + c[:, 1]) * dims[2] + c[:, 2]
    _, first = np.unique(key, return_index=True)
    c = c[np.sort(first)]
    v = (1.0 - SI.unit24_t(SI.rand_t(seed, SI.TAG_VALUE, SI.torch.from_numpy(
        (c[:, 0] * dims[1] + c[:, 1]) * dims[2] + c[:, 2]))).numpy()).astype(np.float32)
    return c.astype(np.uint32), v


# ----------------------------------------------------------------------------- layout / init
@pytest.mark.parametrize("nnz_per_item", [0, 16])
@pytest.mark.parametrize("R", [6, 40])
def test_layout_bit_exact(nnz_per_item, R):
    """P1: the device layouts equal the oracle's bit for bit.  R = 6 keeps the SoA copies
    (the R <= 16 kernel reads them); R = 40 keeps only the 16-byte records, which the
    readback unpacks."""
    dims = (37, 23, 51)
    c, v = ragged_tensor(dims, 3000, 5, heavy_rows=((0, 3, 400), (1, 7, 300), (2, 50, 500)))
    with S(c, v, dims, R, 1, nnz_per_item=nnz_per_item) as g:
        info = g.info()
        assert info["nnz"] == len(v)
        for n in range(3):
            ia, ib, vv, rp = g.layout(n)
            oa, ob, ov, orp = O.layout(c, v, dims, n)
            assert (info["mode_a"][n], info["mode_b"][n]) == O.other_modes(dims, n)
            assert np.array_equal(ia, oa) and np.array_equal(ib, ob)
            assert np.array_equal(vv.view(np.uint32), ov.view(np.uint32))
            assert np.array_equal(rp, orp)
        if nnz_per_item == 16:
            assert min(info["split_rows"]) > 0
        assert info["xnorm2"] == pytest.approx(float((v.astype(np.float64) ** 2).sum()), rel=1e-14)


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("R", [1, 5, 16, 64, 256])
def test_init_bit_exact(precision, R):
    dims = (30, 20, 10)
    c, v = SI.tiny_tensor(dims, 0.05, 3)
    with S(c.numpy(), v.numpy(), dims, R, 77, precision=precision) as g:
        Fo = O.init_factors(dims, R, 77)
        for n in range(3):
            assert np.array_equal(g.factors(n), Fo[n])   # 24-bit dyadic values are exact in fp32 too


def test_errors_dup_range_nonfinite():
    from paper_2003_03572_b200.sacd import SacdError, SACD_EDUP, SACD_ERANGE, SACD_ENONFINITE
    dims = (4, 4, 4)
    with pytest.raises(SacdError) as e:
        S(np.array([[0, 0, 0], [0, 0, 0]], np.uint32), np.ones(2, np.float32), dims, 2, 1)
    assert e.value.code == SACD_EDUP
    with pytest.raises(SacdError) as e:
        S(np.array([[0, 0, 0], [0, 4, 0]], np.uint32), np.ones(2, np.float32), dims, 2, 1)
    assert e.value.code == SACD_ERANGE
    with pytest.raises(SacdError) as e:
        S(np.array([[0, 0, 0]], np.uint32), np.array([np.inf], np.float32), dims, 2, 1)
    assert e.value.code == SACD_ENONFINITE


# ----------------------------------------------------------------------------- teacher-forced kernels
@pytest.mark.parametrize("R", [1, 5, 8, 16, 33, 64, 128, 256])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_mttkrp_gram_hessian(R, precision):
    dims = (41, 29, 57)
    c, v = ragged_tensor(dims, 4000, 11, heavy_rows=((0, 2, 600), (2, 9, 700)))
    F = O.init_factors(dims, R, 3)
    with S(c, v, dims, R, 3, precision=precision, nnz_per_item=64) as g:
        tol = 1e-12 if precision == "f64" else 1e-5
        for n in range(3):
            Mo = O.mttkrp(c, v, dims, n, F)
            Mg = g.mttkrp(n)
            scale = np.maximum(np.abs(Mo).max(axis=0, keepdims=True), 1e-30)
            assert (np.abs(Mg - Mo) / scale).max() <= tol
            Go = O.gram(F[n])
            assert np.abs(g.gram(n) - Go).max() <= tol * np.abs(Go).max()
            Ho = O.mode_hessian(F, dims, n)
            assert np.abs(g.hessian(n) - Ho).max() <= tol * np.abs(Ho).max()


@pytest.mark.parametrize("gram_variant", [0, 2, 3, 4])
@pytest.mark.parametrize("R", [5, 40, 64])
def test_gram_refresh_after_update(gram_variant, R):
    """The Gram refresh of the factor a mode update just wrote (Eq 10's G_n = F_n^T F_n): by
    size (0), fused into the row update (2), panel pairs (3) and the streaming kernel (4), on
    mode lengths that are not multiples of the 32-row chunk or the 128-row block."""
    dims = (1000, 77, 333)
    c, v = ragged_tensor(dims, 20000, 13, heavy_rows=((0, 3, 900),))
    with S(c, v, dims, R, 5, gram_variant=gram_variant) as g:
        for n in range(3):
            g.mode_update(n, branch=0)
            Go = O.gram(g.factors(n))
            assert np.abs(g.gram(n) - Go).max() <= 1e-12 * np.abs(Go).max()


@pytest.mark.parametrize("R", [33, 64, 100, 256])
def test_uniform_values_tensor(R):
    """A tensor whose values are all equal (binary, like c4) takes the MTTKRP path without a
    per-nonzero value (XS = 4, x = the common value, 0 past an item's end): MTTKRP to 1e-12 of
    the oracle, end to end within the north-star tolerances, and info reports the value."""
    dims = (90, 70, 40)
    c, v = ragged_tensor(dims, 12000, 31, heavy_rows=((2, 3, 1500), (0, 7, 900)))
    v = np.full_like(v, 1.0)
    F = O.init_factors(dims, R, 4)
    with S(c, v, dims, R, 4, nnz_per_item=64) as g:
        assert g.info()["uniform_values"] == 1 and g.info()["uniform_value"] == 1.0
        for n in range(3):
            Mo = O.mttkrp(c, v, dims, n, F)
            scale = np.maximum(np.abs(Mo).max(axis=0, keepdims=True), 1e-30)
            assert (np.abs(g.mttkrp(n) - Mo) / scale).max() <= 1e-12
    fg, Fg, Eg, brg, ora = run_pair(c, v, dims, R, 4, 8, nnz_per_item=64)
    check_pair(fg, Fg, Eg, brg, ora)
    v2 = v.copy()
    v2[-1] = 2.0
    with S(c, v2, dims, R, 4) as g:
        assert g.info()["uniform_values"] == 0


@pytest.mark.parametrize("R", [3, 16, 64, 128])
@pytest.mark.parametrize("branch", [0, 1, 2])
@pytest.mark.parametrize("l_mode", ["diag", "frob"])
def test_one_pass_teacher_forced_f64(R, branch, l_mode):
    """One mode pass from identical state: decisions identical, factors / z to fp64 noise."""
    dims = (60, 45, 33)
    c, v = ragged_tensor(dims, 5000, 21, heavy_rows=((1, 4, 500),))
    F = O.init_factors(dims, R, 9)
    rng = np.random.default_rng(R + 10 * branch)
    with S(c, v, dims, R, 9, l_mode=l_mode, nnz_per_item=128) as g:
        for n in range(3):
            Z0 = rng.random((dims[n], R)) * 0.1
            g.set_zprev(n, Z0)
            out = g.mode_update(n, branch=branch, decisions=True)
            M = O.mttkrp(c, v, dims, n, F)
            H = O.mode_hessian(F, dims, n)
            Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, F[n], Z0, branch,
                                                     l_mode=O.L_DIAG if l_mode == "diag" else O.L_FROB,
                                                     decisions=True)
            assert np.array_equal(out["decisions"], dec)
            assert out["E"] == E and out["E_changed"] == Ech
            assert factor_err(g.factors(n), Fn) <= 1e-9
            assert np.abs(g.get_zprev(n) - zp).max() <= 1e-9 * max(1.0, np.abs(zp).max())
            assert abs(out["ti"] - ti) <= 1e-9 * max(1.0, abs(ti))
            F[n] = Fn                       # keep GPU and oracle states identical for the next mode
            g.set_factors(n, Fn)


@pytest.mark.parametrize("cfg_name,K", [("c2", 10), ("c3", 6)])
def test_flip_census_every_pass(cfg_name, K):
    """SURVEY 8(c) flip census, fp64: for every mode pass of a K-sweep run, one oracle pass
    from the GPU's own state before that pass (factors, z_prev, the device's ti history and
    branch rule) reproduces the GPU's decisions, E and ti; the census of mismatches must be
    empty.  This pins the selection dynamics pass by pass, not only end to end."""
    cfg = SI.CONFIGS[cfg_name]
    c, v = SI.make_tensor(cfg)
    c, v = c.numpy(), v.numpy()
    dims, R = cfg.dims, cfg.rank
    hist = [[], [], []]
    census = 0
    with S(c, v, dims, R, cfg.seed) as g:
        for k in range(1, K + 1):
            for n in range(3):
                F = g.factors()
                Z = g.get_zprev(n)
                out = g.mode_update(n, decisions=True)
                M = O.mttkrp(c, v, dims, n, F)
                H = O.mode_hessian(F, dims, n)
                br = O.branch(k, hist[n])
                Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, F[n], Z, br, decisions=True)
                census += int((out["decisions"] != dec).sum())
                assert out["E"] == E and out["E_changed"] == Ech
                assert abs(out["ti"] - ti) <= 1e-9 * max(1.0, abs(ti))
                assert factor_err(g.factors(n), Fn) <= 1e-9
                hist[n].append(out["ti"])
    assert census == 0


def test_one_pass_teacher_forced_f32_flip_census():
    """fp32 state: decisions agree except near-ties (|z| <= 1e-6 max|z| for the FIRST rule)."""
    dims, R = (80, 60, 40), 16
    c, v = ragged_tensor(dims, 8000, 4, heavy_rows=())
    F = O.init_factors(dims, R, 2)
    with S(c, v, dims, R, 2, precision="f32") as g:
        for n in range(3):
            Z0 = np.zeros((dims[n], R))
            out = g.mode_update(n, branch=0, decisions=True)
            M = O.mttkrp(c, v, dims, n, F)
            H = O.mode_hessian(F, dims, n)
            Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, F[n], Z0, 0, decisions=True)
            mism = out["decisions"] != dec
            if mism.any():   # FIRST: sp = z, a near-tie means z ~ 0 relative to the pass
                tie = np.abs(zp) <= 1e-6 * np.abs(zp).max()
                assert tie[mism].all()
            F[n] = g.factors(n)
            g.set_factors(n, F[n])


# ----------------------------------------------------------------------------- end to end
def run_pair(c, v, dims, R, seed, K, **kw):
    precision = kw.pop("precision", "f64")
    with S(c, v, dims, R, seed, precision=precision, **kw) as g:
        f0 = g.fit()[0]
        g.iterate(K)
        st = g.stats()
        Fg = g.factors()
        fg = np.array([f0] + [s["objective"] for s in st])
        Eg = np.array([s["E"] for s in st])
        brg = np.array([s["branch"] for s in st])
    l_mode = {"diag": O.L_DIAG, "frob": O.L_FROB}[kw.get("l_mode", "diag")]
    variant = {"gs": O.VAR_GS_LAGGED, "select_off": O.VAR_SELECT_OFF, "jacobi": O.VAR_JACOBI,
               "snapshot": O.VAR_SNAPSHOT}[kw.get("variant", "gs")]
    ora = O.sacd_run(c, v, dims, R, seed, K, l_mode=l_mode, variant=variant)
    return fg, Fg, Eg, brg, ora


def check_pair(fg, Fg, Eg, brg, ora, f_tol=F_TOL, factor_tol=FACTOR_TOL):
    fo = ora["f"]
    rel = np.abs(fg - fo) / np.maximum(fo, 1e-300)
    assert rel.max() <= f_tol, rel
    # explained energy ||X||^2 - f, when it is not negligible
    ex_o = ora["xnorm2"] - fo
    ex_g = ora["xnorm2"] - fg
    big = ex_o > 1e-3 * ora["xnorm2"]
    if big.any():
        assert (np.abs(ex_g - ex_o)[big] / ex_o[big]).max() <= f_tol
    for n in range(3):
        assert factor_err(Fg[n], ora["F"][n]) <= factor_tol
    assert np.array_equal(brg, ora["branch"])
    return rel.max()


@pytest.mark.parametrize("variant", ["gs", "select_off"])
@pytest.mark.parametrize("l_mode", ["diag", "frob"])
def test_end_to_end_c1(variant, l_mode):
    cfg = SI.CONFIGS["c1"]
    c, v = SI.make_tensor(cfg)
    c, v = c.numpy(), v.numpy()
    fg, Fg, Eg, brg, ora = run_pair(c, v, cfg.dims, cfg.rank, cfg.seed, cfg.iters, variant=variant, l_mode=l_mode)
    check_pair(fg, Fg, Eg, brg, ora)
    assert np.array_equal(Eg, ora["E"])


@pytest.mark.parametrize("variant", ["jacobi", "snapshot"])
@pytest.mark.parametrize("l_mode", ["diag", "frob"])
def test_end_to_end_reading_variants_c1(variant, l_mode):
    """the Lemma-2-literal Jacobi variant and the snapshot-scored exact-ti
    variant (reading C10') run in the same row kernels and match their oracles: f per sweep,
    factors, branch and E."""
    cfg = SI.CONFIGS["c1"]
    c, v = SI.make_tensor(cfg)
    c, v = c.numpy(), v.numpy()
    fg, Fg, Eg, brg, ora = run_pair(c, v, cfg.dims, cfg.rank, cfg.seed, cfg.iters, variant=variant, l_mode=l_mode)
    check_pair(fg, Fg, Eg, brg, ora)
    assert np.array_equal(Eg, ora["E"])


@pytest.mark.parametrize("variant", ["jacobi", "snapshot"])
def test_end_to_end_reading_variants_ragged(variant):
    dims = (300, 200, 50)
    c, v = ragged_tensor(dims, 20000, 8, heavy_rows=((2, 1, 3000), (0, 5, 900)))
    fg, Fg, Eg, brg, ora = run_pair(c, v, dims, 24, 17, 10, nnz_per_item=256, variant=variant)
    check_pair(fg, Fg, Eg, brg, ora)
    assert np.array_equal(Eg, ora["E"])


@pytest.mark.parametrize("branch", [0, 1, 2, -1])
def test_snapshot_one_pass_teacher_forced(branch):
    """Snapshot variant, one pass from identical state (forced branch, or the device's own
    exact-timing choice with -1): decisions, E, factors, z_prev and ti as the oracle."""
    dims, R = (60, 45, 33), 16
    c, v = ragged_tensor(dims, 5000, 21, heavy_rows=((1, 4, 500),))
    F = O.init_factors(dims, R, 9)
    rng = np.random.default_rng(7 + branch)
    with S(c, v, dims, R, 9, variant="snapshot", nnz_per_item=128) as g:
        for n in range(3):
            Z0 = rng.random((dims[n], R)) * 0.1
            g.set_zprev(n, Z0)
            out = g.mode_update(n, branch=branch, decisions=True)
            M = O.mttkrp(c, v, dims, n, F)
            H = O.mode_hessian(F, dims, n)
            Fn, zp, ti, E, Ech, md, dec, br = O.mode_pass_snapshot(M, H, F[n], Z0, True, 0.0, decisions=True,
                                                                   branch=branch)
            assert np.array_equal(out["decisions"], dec)
            assert out["E"] == E and out["E_changed"] == Ech
            assert factor_err(g.factors(n), Fn) <= 1e-9
            assert np.abs(g.get_zprev(n) - zp).max() <= 1e-9 * max(1.0, np.abs(zp).max())
            assert abs(out["ti"] - ti) <= 1e-9 * max(1.0, abs(ti))
            F[n] = Fn
            g.set_factors(n, Fn)


def test_reading_variants_rejected_by_sharded_engine():
    from paper_2003_03572_b200.sacd import SacdError
    cfg = SI.CONFIGS["c1"]
    c, v = SI.make_tensor(cfg)
    for variant in ("jacobi", "snapshot"):
        with pytest.raises(SacdError):
            S(c.numpy(), v.numpy(), cfg.dims, cfg.rank, cfg.seed, variant=variant, emulate_ranks=2)


def test_c2_full_iteration_count_parity():
    """c2 at its BASELINE iteration count (50 sweeps) against the oracle: f per sweep, factors,
    branch and E, plus the invariants (f non-increasing, factors >= 0, E <= I R)."""
    cfg = SI.CONFIGS["c2"]
    c, v = SI.make_tensor(cfg)
    c, v = c.numpy(), v.numpy()
    fg, Fg, Eg, brg, ora = run_pair(c, v, cfg.dims, cfg.rank, cfg.seed, cfg.iters)
    check_pair(fg, Fg, Eg, brg, ora)
    assert np.array_equal(Eg, ora["E"])
    assert (np.diff(fg) <= 1e-12 * fg[0]).all()
    for n in range(3):
        assert (Fg[n] >= 0).all() and (Eg[:, n] <= cfg.dims[n] * cfg.rank).all()


def test_c3_full_iteration_count_properties():
    """c3 for its 50 sweeps on the GPU alone: f non-increasing (Lemma 3 under reading C9),
    factors >= 0, E <= I R, and the final f equal to the sparse-explicit objective of the
    returned factors (oracle, Eq 6-7)."""
    cfg = SI.CONFIGS["c3"]
    c, v = SI.make_tensor(cfg)
    c, v = c.numpy(), v.numpy()
    with S(c, v, cfg.dims, cfg.rank, cfg.seed) as g:
        f0 = g.fit()[0]
        g.iterate(cfg.iters)
        st = g.stats()
        F = g.factors()
    f = np.array([f0] + [s["objective"] for s in st])
    assert (np.diff(f) <= 1e-12 * f[0]).all()
    for n in range(3):
        assert (F[n] >= 0).all()
        assert all(s["E"][n] <= cfg.dims[n] * cfg.rank for s in st)
    fs = O.objective_sparse(c, v, cfg.dims, F)
    assert abs(f[-1] - fs) <= 1e-9 * fs


def test_end_to_end_c2_10_sweeps():
    cfg = SI.CONFIGS["c2"]
    c, v = SI.make_tensor(cfg)
    c, v = c.numpy(), v.numpy()
    fg, Fg, Eg, brg, ora = run_pair(c, v, cfg.dims, cfg.rank, cfg.seed, 10)
    check_pair(fg, Fg, Eg, brg, ora)


@pytest.mark.parametrize("R", [1, 8, 33, 100, 128, 200])
def test_end_to_end_ragged_ranks(R):
    dims = (300, 200, 50)
    c, v = ragged_tensor(dims, 20000, 8, heavy_rows=((2, 1, 3000), (0, 5, 900)))
    fg, Fg, Eg, brg, ora = run_pair(c, v, dims, R, 17, 10, nnz_per_item=256)
    check_pair(fg, Fg, Eg, brg, ora)


def test_empty_tensor():
    """nnz = 0: the U pass drives U to 0 (m = 0), after which h_rr = 0 for V and W, which are
    then skipped (reading C11); f = 0 from sweep 1 on.  Same as the oracle."""
    dims = (5, 4, 3)
    c, v = np.zeros((0, 3), np.uint32), np.zeros(0, np.float32)
    with S(c, v, dims, 3, 1) as g:
        g.iterate(2)
        f, fit = g.fit()
        Fg = g.factors()
    ora = O.sacd_run(c, v, dims, 3, 1, 2)
    assert f == 0.0 == ora["f"][-1]
    assert (Fg[0] == 0).all()
    for n in range(3):
        assert np.array_equal(Fg[n], ora["F"][n])


@pytest.mark.parametrize("R", [5, 24, 32, 40, 200])
def test_deterministic_and_graph_equals_eager(R):
    """Reruns are bitwise identical (no floating-point atomics; fixed-order reductions) and
    the captured graph equals eager launches.  compute-sanitizer is not available on the GPU
    pool, so this doubles as the race check of the shared-memory broadcasts and staging:
    R = 5 (R <= 16 MTTKRP), 24 / 32 (two dynamically scheduled workers per warp with their own
    double-buffered broadcasts, on a tensor whose heavy slices make long fibers), 40 (x
    broadcast, DMMA row kernel), 200 (R > 128 kernels)."""
    if R in (24, 32):  # dense enough for fibers of ~6-30 nonzeros (the SW = 16 kernel's case)
        dims = (120, 80, 16)
        c, v = ragged_tensor(dims, 60000, 8, heavy_rows=((2, 1, 900), (0, 5, 700)))
    else:
        dims = (300, 200, 50)
        c, v = ragged_tensor(dims, 20000, 8, heavy_rows=((2, 1, 3000), (0, 5, 900)))
    res = []
    for use_graph in (True, True, False):
        with S(c, v, dims, R, 11, use_graph=use_graph, nnz_per_item=256) as g:
            g.iterate(6)
            res.append((g.factors(), [s["objective"] for s in g.stats()]))
    for r in res[1:]:
        assert all(np.array_equal(a, b) for a, b in zip(r[0], res[0][0]))
        assert r[1] == res[0][1]


def test_device_pointer_inputs():
    import torch
    cfg = SI.CONFIGS["c1"]
    c, v = SI.make_tensor(cfg)
    with S(c.cuda(), v.cuda(), cfg.dims, cfg.rank, cfg.seed) as g1, \
            S(c.numpy(), v.numpy(), cfg.dims, cfg.rank, cfg.seed) as g2:
        g1.iterate(3)
        g2.iterate(3)
        assert np.array_equal(g1.factors(0), g2.factors(0))


def test_factors_into_preallocated_pinned_and_pageable_buffers():
    """Sacd.factors(out=...): pinned buffers (direct D2H) and pageable ones (the pinned ring,
    > 8 MB) return exactly the default read; bad buffers are rejected."""
    import torch
    dims, R = (40000, 300, 20), 64  # mode 0 is 20 MB: the chunked ring path
    c, v = ragged_tensor(dims, 60000, 5)
    with S(c, v, dims, R, 3) as g:
        g.iterate(2)
        ref = g.factors()
        pinned = [torch.empty((dims[n], R), dtype=torch.float64).pin_memory().numpy() for n in range(3)]
        pageable = [np.empty((dims[n], R)) for n in range(3)]
        for out in (pinned, pageable):
            got = g.factors(out=out)
            for n in range(3):
                assert got[n] is out[n] and np.array_equal(out[n], ref[n])
        with pytest.raises(ValueError):
            g.factors(0, out=np.empty((dims[0], R), np.float32))
        with pytest.raises(ValueError):
            g.factors(0, out=np.empty((R, dims[0])).T)


def test_device_inputs_from_torch_stream_are_complete():
    """sacd_init / sacd_rmse read device inputs after a device synchronisation, so tensors
    produced on PyTorch's stream right before the call are complete (the library stream is
    non-blocking).  c3 (1e7 nonzeros) is generated on the GPU and handed over at once; its
    layout must equal the one built from the same tensor copied to the host."""
    import torch
    cfg = SI.CONFIGS["c3"]
    c, v = SI.make_tensor(cfg, device="cuda")  # queued on torch's stream, not synchronised
    with S(c, v, cfg.dims, 4, cfg.seed) as g1:
        ch, vh = c.cpu().numpy(), v.cpu().numpy()
        with S(ch, vh, cfg.dims, 4, cfg.seed) as g2:
            for n in range(3):
                la, lb = g1.layout(n), g2.layout(n)
                for x, y in zip(la, lb):
                    assert np.array_equal(x, y)
        c2, v2 = SI.make_tensor(cfg, device="cuda")
        r_dev = g1.rmse(c2[:100000], v2[:100000])
        r_host = g1.rmse(c2[:100000].cpu().numpy(), v2[:100000].cpu().numpy())
        assert r_dev == r_host


def test_per_sweep_device_time():
    """sacd_iter_stats.ms (%globaltimer from the sweep's first kernel to the end of its
    objective kernel, SPEC FitReport S:251-254) is positive for every sweep and, summed over
    back-to-back captured sweeps, matches the CUDA-event time of sacd_iterate."""
    import torch
    cfg = SI.CONFIGS["c3"]
    c, v = SI.make_tensor(cfg, device="cuda")
    stream = torch.cuda.Stream()
    with S(c, v, cfg.dims, cfg.rank, cfg.seed, stream=stream.cuda_stream) as g:
        g.iterate(2)
        g.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.iterate(10)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        st = g.stats()
    dev = [s["ms"] for s in st]
    assert len(dev) == 12 and all(0 < x < 1e3 for x in dev)
    assert abs(sum(dev[2:]) - ms) <= 0.1 * ms + 0.05, (dev, ms)


def test_profile_mode_counts_launches():
    cfg = SI.CONFIGS["c1"]
    c, v = SI.make_tensor(cfg)
    with S(c.numpy(), v.numpy(), cfg.dims, cfg.rank, cfg.seed, profile=True) as g:
        g.profile_reset()
        g.iterate(4)
        p = g.profile_read()
        assert p["mttkrp"][1] == 12 and p["rows"][1] == 12 and p["mttkrp"][0] > 0


# ----------------------------------------------------------------------------- the BASELINE configs
def _config_tensor(name):
    import torch
    cfg = SI.CONFIGS[name]
    c, v = SI.make_tensor(cfg, device="cuda")
    return cfg, c.cpu().numpy().astype(np.uint32), v.cpu().numpy()


def test_end_to_end_c3_10_sweeps():
    cfg, c, v = _config_tensor("c3")
    fg, Fg, Eg, brg, ora = run_pair(c, v, cfg.dims, cfg.rank, cfg.seed, 10)
    check_pair(fg, Fg, Eg, brg, ora)


@pytest.mark.parametrize("R", [8, 16, 32, 64, 128, 256])
def test_end_to_end_c5_rank_sweep(R):
    cfg, c, v = _config_tensor("c5")
    fg, Fg, Eg, brg, ora = run_pair(c, v, cfg.dims, R, cfg.seed, 10)
    check_pair(fg, Fg, Eg, brg, ora)


def test_c4_end_to_end_10_sweeps():
    """The north star's parity run on the bench config itself: c4 at full size (1e8 nonzeros,
    R = 64, fp64), 10 sweeps, the GPU's own trajectory (device branch rule) next to the
    oracle's own trajectory (its functions, pass by pass, in ora_sacd_run's order), compared
    at every mode pass:
      * the branch of every pass and f (Eq 6-7, Gram trick on each side's factors) within
        1e-4 at every sweep;
      * until the trajectories first decide an element differently: the same decisions and E
        in every pass and the factors within 1e-3 (column-relative floor);
      * at that first pass, every element decided differently is a near-tie at fp64
        resolution in the oracle's own trajectory: its gradient
        g = -m + sum_j u_j h_jr (Eq 14, the Gauss-Seidel row at column r) is below
        1e-12 x (|m| + sum_j |u_j h_jr|), or its z and z_prev are below 1e-12 x the pass's
        largest importance -- g, and with it the step d and the importance z (Eq 20), is
        rounding noise of the cancellation, on either side.  After that pass the
        trajectories are different valid SaCD runs (reading C19): later mismatches and the
        final factor error are reported, not bounded.
    tools/flip_census.py / flip_census_oracle.py (profiles/r02_flip_census_*) show that neither
    side ever decides differently from the other given the SAME state (0 of 9.7e8 decisions
    along each trajectory): the divergence comes from ~1e-10 state differences (rounding
    amplified by the projection's cancellations) meeting near-ties."""
    cfg, c, v = _config_tensor("c4")
    dims, R = cfg.dims, cfg.rank
    lays = [O.layout(c, v, dims, n) for n in range(3)]
    F = O.init_factors(dims, R, cfg.seed)
    Z = [np.zeros((dims[n], R)) for n in range(3)]
    hist_o, hist_g = [[], [], []], [[], [], []]
    xn2 = float((v.astype(np.float64) ** 2).sum())
    first = None
    report = []
    with S(c, v, dims, R, cfg.seed) as g:
        for k in range(1, 11):
            md_o = md_g = None
            for n in range(3):
                a, b = O.other_modes(dims, n)
                Zg0 = g.get_zprev(n) if first is None else None
                out = g.mode_update(n, decisions=True)
                br_g = O.branch(k, hist_g[n])
                hist_g[n].append(out["ti"])
                H = O.hadamard(O.gram(F[a]), O.gram(F[b]))
                ia, ib, vv, rp = lays[n]
                M = O.mttkrp_layout(rp, ia, ib, vv, F[a], F[b])
                br_o = O.branch(k, hist_o[n])
                Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, F[n], Z[n], br_o, decisions=True)
                assert br_g == br_o, (k, n, br_g, br_o)
                mism = np.argwhere(out["decisions"] != dec)
                if first is None:
                    if len(mism):
                        first = (k, n)
                        for i, r in mism:
                            z0, z1 = Z[n][i, r], zp[i, r]
                            sp = z1 if br_o == O.BR_FIRST else (z1 - z0 if br_o == O.BR_EQ24 else z0 - z1)
                            u = np.concatenate([Fn[i, :r], F[n][i, r:]])  # the row when column r is updated
                            terms = u * H[:, r]
                            g_o = -M[i, r] + terms.sum()
                            rel_g = abs(g_o) / max(abs(M[i, r]) + np.abs(terms).sum(), 1e-300)
                            rel_z = max(abs(z0), abs(z1)) / max(np.abs(zp).max(), np.abs(Z[n]).max(), 1e-300)
                            report.append((k, n, int(i), int(r), float(z0), float(z1), float(sp), float(rel_g),
                                           float(rel_z), float(Zg0[i, r] - z0)))
                            assert rel_g <= 1e-12 or rel_z <= 1e-12, report[-1]
                    else:
                        assert out["E"] == E and out["E_changed"] == Ech
                        assert factor_err(g.factors(n), Fn) <= FACTOR_TOL
                hist_o[n].append(ti)
                F[n], Z[n] = Fn, zp
                if n == 2:
                    md_o = md
                    md_g = float((g.factors(2) * g.mttkrp(2)).sum())
            Gg = [g.gram(n) for n in range(3)]
            Go = [O.gram(F[n]) for n in range(3)]
            f_g = xn2 - 2.0 * md_g + float((Gg[0] * Gg[1] * Gg[2]).sum())
            f_o = xn2 - 2.0 * md_o + float((Go[0] * Go[1] * Go[2]).sum())
            assert abs(f_g - f_o) <= F_TOL * f_o, (k, f_g, f_o)
        errs = [factor_err(g.factors(n), F[n]) for n in range(3)]
    print(f"c4 10 sweeps: first pass decided differently {first}; its near-ties (sweep, mode, row, col, z_prev, "
          f"z, sp (oracle), |g| / sum of |terms|, max(|z|, |z_prev|) / pass max, z_prev gpu - oracle): {report[:20]}; final factor err {errs}")


# ----------------------------------------------------------------------------- sharded engine
@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("R", [5, 64])
def test_sharded_emulated_ranks_end_to_end(G, R):
    """SURVEY 8(e) on one GPU: G ranks of the sharded engine emulated in one context (the
    exchanges become local), with heavy slices cut by the rank boundaries: same decisions,
    branch and E as the oracle, f and factors within the north-star tolerances."""
    dims = (300, 200, 50)
    c, v = ragged_tensor(dims, 20000, 8, heavy_rows=((2, 1, 3000), (0, 5, 900), (1, 199, 1500)))
    fg, Fg, Eg, brg, ora = run_pair(c, v, dims, R, 17, 10, nnz_per_item=256, emulate_ranks=G)
    check_pair(fg, Fg, Eg, brg, ora)
    assert np.array_equal(Eg, ora["E"])


@pytest.mark.parametrize("G", [2, 5])
def test_sharded_emulated_teacher_forced(G):
    dims, R = (60, 45, 33), 16
    c, v = ragged_tensor(dims, 5000, 21, heavy_rows=((1, 4, 1500), (0, 59, 800)))
    F = O.init_factors(dims, R, 9)
    with S(c, v, dims, R, 9, nnz_per_item=64, emulate_ranks=G) as g:
        for n in range(3):
            assert np.abs(g.mttkrp(n) - O.mttkrp(c, v, dims, n, F)).max() <= 1e-12 * max(
                1.0, np.abs(O.mttkrp(c, v, dims, n, F)).max())
            out = g.mode_update(n, branch=0, decisions=True)
            M = O.mttkrp(c, v, dims, n, F)
            H = O.mode_hessian(F, dims, n)
            Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, F[n], np.zeros_like(F[n]), 0, decisions=True)
            assert np.array_equal(out["decisions"], dec) and out["E"] == E
            assert factor_err(g.factors(n), Fn) <= 1e-9
            assert abs(out["ti"] - ti) <= 1e-9 * max(1.0, abs(ti))
            F[n] = Fn
            g.set_factors(n, Fn)


def test_sharded_nccl_world1_matches_unsharded():
    """The real NCCL transport (all-gathers, grouped broadcasts) with a one-rank
    communicator: identical decisions and E to the unsharded engine, f to 1e-12."""
    cfg = SI.CONFIGS["c1"]
    c, v = SI.make_tensor(cfg)
    c, v = c.numpy(), v.numpy()
    out = []
    for forced in (False, True):
        with S(c, v, cfg.dims, cfg.rank, cfg.seed, force_sharded=forced) as g:
            g.iterate(6)
            st = g.stats()
            out.append((np.array([s["objective"] for s in st]), np.array([s["E"] for s in st]), g.factors()))
    np.testing.assert_allclose(out[1][0], out[0][0], rtol=1e-12)
    assert np.array_equal(out[1][1], out[0][1])
    for n in range(3):  # the same work items, Gram ranges and fixed-order sums: bitwise equal
        assert np.array_equal(out[1][2][n], out[0][2][n])


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("R", [5, 64])
def test_p2p_exchange_emulated_replicas(G, precision, R):
    """The peer-memory exchange with G emulated ranks, each holding its OWN factor replicas:
    every pass, each shard's kernel stores the changed 16-byte chunks of its owned rows into
    the other shards' replicas, and device flags order the passes.  After 8 sweeps all
    replicas are bitwise identical, equal the full-row exchange's factors bitwise, and (fp64)
    meet the oracle bar; the captured sweep graph equals eager sweeps."""
    dims = (300, 200, 50)
    c, v = ragged_tensor(dims, 20000, 8, heavy_rows=((2, 1, 3000), (0, 5, 900), (1, 199, 1500)))
    res = {}
    for ex, graph in (("full", True), ("p2p", True), ("p2p", False)):
        with S(c, v, dims, R, 17, nnz_per_item=256, emulate_ranks=G, exchange=ex, precision=precision,
               use_graph=graph) as g:
            f0 = g.fit()[0]
            g.iterate(8)
            st = g.stats()
            Fs = g.factors()
            if ex == "p2p":
                for q in range(G):
                    for n in range(3):
                        assert np.array_equal(g.replica_factors(q, n), Fs[n]), (q, n)
            res[(ex, graph)] = (np.array([f0] + [s["objective"] for s in st]), Fs, st)
    for key in (("p2p", True), ("p2p", False)):
        assert np.array_equal(res[key][0], res[("full", True)][0])
        for n in range(3):
            assert np.array_equal(res[key][1][n], res[("full", True)][1][n])
    if precision == "f64":
        fg, Fg, st = res[("p2p", True)]
        ora = O.sacd_run(c, v, dims, R, 17, 8)
        check_pair(fg, Fg, np.array([s["E"] for s in st]), np.array([s["branch"] for s in st]), ora)


def test_p2p_exchange_world1_matches_unsharded():
    """exchange='p2p' on the one-rank sharded engine (no peers) equals the unsharded engine."""
    cfg = SI.CONFIGS["c1"]
    c, v = SI.make_tensor(cfg)
    c, v = c.numpy(), v.numpy()
    out = []
    for kw in ({}, {"force_sharded": True, "exchange": "p2p"}):
        with S(c, v, cfg.dims, cfg.rank, cfg.seed, **kw) as g:
            g.iterate(6)
            out.append(g.factors())
    for n in range(3):
        assert np.array_equal(out[0][n], out[1][n])


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_delta_exchange_emulated_bitwise_equals_full(G, precision):
    """with the delta exchange every pass resets the owned rows to their
    pre-pass values and rebuilds them from the owners' (index, value) lists of changed
    elements, so any compaction / apply error shows; the factors, f and E must equal the
    full-row exchange bit for bit, and the oracle within the tolerances (fp64)."""
    dims = (300, 200, 50)
    c, v = ragged_tensor(dims, 20000, 8, heavy_rows=((2, 1, 3000), (0, 5, 900), (1, 199, 1500)))
    res = []
    for ex in ("full", "delta"):
        with S(c, v, dims, 24, 17, precision=precision, nnz_per_item=256, emulate_ranks=G, exchange=ex) as g:
            assert g.info()["delta_exchange"] == (ex == "delta")
            g.iterate(8)
            st = g.stats()
            res.append((np.array([s["objective"] for s in st]), np.array([s["E"] for s in st]), g.factors()))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    for n in range(3):
        assert np.array_equal(res[0][2][n], res[1][2][n])
    if precision == "f64":
        fg, Fg, Eg, brg, ora = run_pair(c, v, dims, 24, 17, 8, nnz_per_item=256, emulate_ranks=G, exchange="delta")
        check_pair(fg, Fg, Eg, brg, ora)


def test_delta_exchange_nccl_world1():
    """The NCCL delta path (list lengths all-gathered and read on the host, lists broadcast,
    eager sweeps) with a one-rank communicator equals the unsharded engine; the counters show
    that lists were sent once the factors settle (c3: its U factor is above the 16 MB below
    which a factor always goes as full rows)."""
    cfg = SI.CONFIGS["c3"]
    c, v = SI.make_tensor(cfg)
    c, v = c.numpy(), v.numpy()
    out = []
    for kw in ({}, {"force_sharded": True, "exchange": "delta"}):
        with S(c, v, cfg.dims, cfg.rank, cfg.seed, **kw) as g:
            g.iterate(8)
            st = g.stats()
            out.append((np.array([s["objective"] for s in st]), np.array([s["E"] for s in st]), g.factors(),
                        g.info()))
    np.testing.assert_allclose(out[1][0], out[0][0], rtol=1e-12)
    assert np.array_equal(out[1][1], out[0][1])
    for n in range(3):  # the same work items, Gram ranges and fixed-order sums: bitwise equal
        assert np.array_equal(out[1][2][n], out[0][2][n])
    inf = out[1][3]
    assert inf["delta_exchange"] == 1 and inf["full_elems_equiv"] > 0
    assert 0 < inf["delta_elems_sent"] < inf["full_elems_equiv"]


# ----------------------------------------------------------------------------- held-out evaluation (f3)
@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("R", [5, 64, 200])
def test_predict_rmse_parity(precision, R):
    """sacd_predict / sacd_rmse (Eq 8, Eq 30) against the oracle after a few sweeps on the
    80% training split, evaluated on the 20% held-out entries (host and device inputs)."""
    import torch
    cfg = SI.custom_config((300, 200, 150), 60000, R, cid=31)
    c, v = SI.make_tensor(cfg)
    trc, trv, tec, tev = SI.split_train_test(c, v, cfg.dims, cfg.seed)
    with S(trc.numpy(), trv.numpy(), cfg.dims, R, cfg.seed, precision=precision) as g:
        g.iterate(4)
        F = g.factors()
        xo = O.predict(tec.numpy(), cfg.dims, F)
        xg = g.predict(tec.numpy())
        tol = 1e-12 if precision == "f64" else 1e-5
        assert np.abs(xg - xo).max() <= tol * max(np.abs(xo).max(), 1e-30)
        ro = O.rmse(tec.numpy(), tev.numpy(), cfg.dims, F)
        rg = g.rmse(tec.numpy(), tev.numpy())
        assert abs(rg - ro) <= 1e-12 * ro
        rd = g.rmse(tec.cuda().to(torch.int32).contiguous(), tev.cuda())  # device pointers
        assert rd == rg


def test_predict_errors_and_empty():
    from paper_2003_03572_b200.sacd import SacdError, SACD_ERANGE
    dims = (20, 10, 5)
    c, v = SI.tiny_tensor(dims, 0.2, 2)
    with S(c.numpy(), v.numpy(), dims, 3, 2) as g:
        with pytest.raises(SacdError) as e:
            g.predict(np.array([[0, 10, 0]], np.uint32))
        assert e.value.code == SACD_ERANGE
        assert g.rmse(np.zeros((0, 3), np.uint32), np.zeros(0, np.float32)) == 0.0
        assert g.predict(np.zeros((0, 3), np.uint32)).shape == (0,)
        g.iterate(1)   # the context is still usable after ERANGE


def test_heldout_rmse_end_to_end_c2():
    """80/20 split of c2 (10 sweeps): GPU and oracle held-out RMSE agree to 1e-6 relative
    (the trajectories agree per the end-to-end tolerances)."""
    cfg = SI.CONFIGS["c2"]
    c, v = SI.make_tensor(cfg)
    trc, trv, tec, tev = SI.split_train_test(c, v, cfg.dims, cfg.seed)
    K = 10
    with S(trc.numpy(), trv.numpy(), cfg.dims, cfg.rank, cfg.seed) as g:
        g.iterate(K)
        rg = g.rmse(tec.numpy(), tev.numpy())
    out = O.sacd_run(trc.numpy(), trv.numpy(), cfg.dims, cfg.rank, cfg.seed, K)
    ro = O.rmse(tec.numpy(), tev.numpy(), cfg.dims, out["F"])
    assert abs(rg - ro) <= 1e-6 * ro, (rg, ro)


# ----------------------------------------------------------------------------- a-blocked execution order
@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("R", [33, 64])
def test_ablocked_order_mttkrp_and_sweeps(precision, R):
    """The a-blocked MTTKRP order (forced here with small blocks) gives the oracle's MTTKRP
    within rounding, the same layout readback, and sweeps that match the unblocked run to
    the end-to-end tolerances."""
    dims = (61, 47, 9)
    c, v = ragged_tensor(dims, 6000, 23, heavy_rows=((2, 3, 900), (0, 5, 400)))
    F = O.init_factors(dims, R, 4)
    Mo = [O.mttkrp(c, v, dims, n, F) for n in range(3)]
    tol = 1e-12 if precision == "f64" else 1e-5
    with S(c, v, dims, R, 4, precision=precision, nnz_per_item=40, ablk_rows=7) as g:
        for n in range(3):
            scale = np.maximum(np.abs(Mo[n]).max(axis=0, keepdims=True), 1e-30)
            assert (np.abs(g.mttkrp(n) - Mo[n]) / scale).max() <= tol, n
            ia, ib, vv, rp = g.layout(n)
            oa, ob, ov, orp = O.layout(c, v, dims, n)
            assert np.array_equal(ia, oa) and np.array_equal(ib, ob) and np.array_equal(rp, orp)
        g.iterate(6)
        fb = [s["objective"] for s in g.stats()]
        Fb = g.factors()
    with S(c, v, dims, R, 4, precision=precision, nnz_per_item=40, ablk_rows=-1) as g:
        g.iterate(6)
        fu = [s["objective"] for s in g.stats()]
    assert np.max(np.abs(np.array(fb) - np.array(fu)) / np.array(fu)) <= F_TOL
    if precision == "f64":
        out = O.sacd_run(c, v, dims, R, 4, 6)
        for n in range(3):
            assert factor_err(Fb[n], out["F"][n]) <= FACTOR_TOL
