"""Pins for the fp64 CPU oracle (P1-P12): each test checks the oracle
against something other than itself -- hand-derived values (tests/golden/), closed forms,
dense brute force written here from the paper's definitions (Kolda unfolding + Eq 3
Khatri-Rao, Eq 7 objective), finite differences, exact coordinate minimisation,
invariants, special cases.  CPU only."""
import numpy as np
import pytest

import oracle as O
import sacd_inputs as SI


# ----------------------------------------------------------------------------- helpers
def dense_tensor(coords, vals, dims):
    X = np.zeros(dims, np.float64)
    c = np.asarray(coords, np.int64)
    X[c[:, 0], c[:, 1], c[:, 2]] = np.asarray(vals, np.float64)
    return X


def unfold(X, n):
    """Kolda mode-n matricization (section 3): element (q,p,s) of mode-1
    goes to column p + P*s; mode-2: column q + Q*s; mode-3: column q + Q*p."""
    Q, P, S = X.shape
    if n == 0:
        return X.transpose(0, 2, 1).reshape(Q, S * P)   # col = s*P + p
    if n == 1:
        return X.transpose(1, 2, 0).reshape(P, S * Q)   # col = s*Q + q
    return X.transpose(2, 1, 0).reshape(S, P * Q)       # col = p*Q + q


def khatri_rao(A, B):
    """Eq 3: column r = kron(a_r, b_r)."""
    R = A.shape[1]
    return np.stack([np.kron(A[:, r], B[:, r]) for r in range(R)], axis=1)


def kr_for_mode(F, n):
    """The Khatri-Rao product paired with X_(n): Eq 9 (W (.) V), pdei (W (.) U), pdet (V (.) U)."""
    U, V, W = F
    return [khatri_rao(W, V), khatri_rao(W, U), khatri_rao(V, U)][n]


def f_dense(X, F):
    """Eq 7 with Eq 8, all cells."""
    Xh = np.einsum("qr,pr,sr->qps", *F)
    return float(((X - Xh) ** 2).sum())


def f_rows(X, F, n):
    """Eq ucap: per-row residual of X_(n) - F_n (KR)^T; sum over rows = f."""
    Xn = unfold(X, n)
    KR = kr_for_mode(F, n)
    return ((Xn - F[n] @ KR.T) ** 2).sum(axis=1)


def rand_inst(dims, density, R, seed):
    c, v = SI.tiny_tensor(dims, density, seed)
    c, v = c.numpy(), v.numpy()
    F = O.init_factors(dims, R, seed)
    return c, v, F


# ----------------------------------------------------------------------------- RNG / init
def test_rng_is_textbook_splitmix64(golden):
    g = golden["spec_hand_examples"]["splitmix64"]
    t = g["seed_tag"]
    for c, h in enumerate(g["outputs_hex"]):
        assert O.rand(t, t, c) == int(h, 16)


def test_init_factors_definition():
    dims, R, seed = (4, 3, 5), 2, 77
    F = O.init_factors(dims, R, seed)
    off = 0
    for n in range(3):
        for i in range(dims[n]):
            for r in range(R):
                x = SI.rand_int(seed, SI.TAG_INIT, off + i * R + r)
                assert F[n][i, r] == (x >> 40) * 2.0 ** -24
        off += dims[n] * R
        assert (F[n] >= 0).all() and (F[n] < 1).all()


# ----------------------------------------------------------------------------- P1 layout
def test_layout_sorted_unique_and_complete():
    dims = (7, 5, 9)
    c, v = SI.tiny_tensor(dims, 0.3, 11)
    c, v = c.numpy().astype(np.int64), v.numpy()
    for n in range(3):
        a, b = O.other_modes(dims, n)
        assert {a, b} == {0, 1, 2} - {n}
        ia, ib, vv, rp = O.layout(c, v, dims, n)
        assert rp[0] == 0 and rp[-1] == len(v) and (np.diff(rp) >= 0).all()
        rows = np.repeat(np.arange(dims[n]), np.diff(rp))
        key = (rows * dims[a] + ia) * dims[b] + ib
        assert (np.diff(key) > 0).all()                      # strictly sorted => unique order
        # round trip: the layout holds exactly the input entries
        trip = np.zeros((len(v), 3), np.int64)
        trip[:, n], trip[:, a], trip[:, b] = rows, ia, ib
        d_in = {tuple(x): y for x, y in zip(c.tolist(), v.tolist())}
        d_out = {tuple(x): y for x, y in zip(trip.tolist(), vv.tolist())}
        assert d_in == d_out


def test_layout_other_mode_rule():
    # reading L1: a = the other mode with the LARGER length, ties -> lower mode id
    assert O.other_modes((10, 5, 3), 0) == (1, 2)
    assert O.other_modes((10, 5, 5), 0) == (1, 2)
    assert O.other_modes((10, 5, 3), 2) == (0, 1)
    assert O.other_modes((1_000_000, 500_000, 10_000), 1) == (0, 2)
    assert O.other_modes((1_000_000, 500_000, 10_000), 0) == (1, 2)


def test_layout_slice_example():
    # SPEC S:100-ish mode_slice_entries example: {(0,0,0)=1,(0,1,0)=2,(1,0,0)=3}, mode 0, index 0
    c = np.array([[1, 0, 0], [0, 1, 0], [0, 0, 0]])
    v = np.array([3.0, 2.0, 1.0], np.float32)
    ia, ib, vv, rp = O.layout(c, v, (2, 2, 1), 0)
    assert list(rp) == [0, 2, 3]
    assert list(vv[:2]) == [1.0, 2.0]


@pytest.mark.parametrize("bad,rc", [
    (np.array([[0, 0, 0], [0, 0, 0]]), -3),      # duplicate
    (np.array([[0, 0, 0], [2, 0, 0]]), -2),      # out of range
])
def test_layout_errors(bad, rc):
    with pytest.raises(O.OracleError) as e:
        O.layout(bad, np.ones(2, np.float32), (2, 2, 2), 0)
    assert e.value.rc == rc


def test_layout_nonfinite():
    with pytest.raises(O.OracleError) as e:
        O.layout(np.array([[0, 0, 0]]), np.array([np.nan], np.float32), (1, 1, 1), 0)
    assert e.value.rc == -4


def test_layout_empty():
    ia, ib, vv, rp = O.layout(np.zeros((0, 3)), np.zeros(0, np.float32), (3, 2, 2), 1)
    assert len(vv) == 0 and list(rp) == [0, 0, 0]


# ----------------------------------------------------------------------------- P2 MTTKRP
def test_mttkrp_spec_example(golden):
    g = golden["spec_hand_examples"]["mttkrp_single_entry"]
    F = [np.zeros((1, 2)), np.array(g["V"], float), np.array(g["W"], float)]
    M = O.mttkrp(np.array(g["coords"]), np.array(g["vals"], np.float32), g["dims"], 0, F)
    assert M[0].tolist() == g["M_mode0_row0"]


@pytest.mark.parametrize("dims,R", [((4, 4, 4), 3), ((5, 3, 4), 2), ((6, 7, 2), 4)])
def test_mttkrp_equals_dense_unfolding(dims, R):
    c, v, F = rand_inst(dims, 0.4, R, 5 + R)
    X = dense_tensor(c, v, dims)
    for n in range(3):
        M = O.mttkrp(c, v, dims, n, F)
        Md = unfold(X, n) @ kr_for_mode(F, n)
        np.testing.assert_allclose(M, Md, rtol=1e-12, atol=1e-13)


def test_mttkrp_empty_tensor():
    dims = (3, 4, 5)
    F = O.init_factors(dims, 3, 1)
    M = O.mttkrp(np.zeros((0, 3)), np.zeros(0, np.float32), dims, 2, F)
    assert (M == 0).all()


# ----------------------------------------------------------------------------- P3 Gram / H
def test_gram_hadamard_frobenius_examples(golden):
    g = golden["spec_hand_examples"]
    assert O.hadamard(np.array(g["hadamard"]["X"], float), np.array(g["hadamard"]["Y"], float)).tolist() == g["hadamard"]["Z"]
    assert O.gram(np.array(g["gram"]["F"], float)).tolist() == g["gram"]["G"]
    mh = g["mode_hessian"]
    assert O.hadamard(np.array(mh["Ga"], float), np.array(mh["Gb"], float)).tolist() == mh["H"]
    assert abs(O.frobenius(np.array(g["frobenius"]["H"], float)) - g["frobenius"]["L"]) < 1e-15


def test_hessian_is_gram_of_khatri_rao():
    # (A (.) B)^T (A (.) B) = A^T A * B^T B   (Eq 10 as the Gram of the Khatri-Rao product)
    rng = np.random.default_rng(0)
    A, B = rng.random((6, 4)), rng.random((5, 4))
    KR = khatri_rao(A, B)
    np.testing.assert_allclose(O.hadamard(O.gram(A), O.gram(B)), KR.T @ KR, rtol=1e-13)
    G = O.gram(A)
    assert (G == G.T).all() and (np.diag(G) >= 0).all()


# ----------------------------------------------------------------------------- P4 gradient / P5 step / P6 importance
def one_row_pass(M, H, u, zprev, branch, l_mode=O.L_DIAG):
    return O.mode_pass(M, H, u, zprev, branch, l_mode=l_mode, decisions=True)


def test_gradient_is_half_finite_difference():
    """P4 / reading C2: Eq 9's G = -M + F H, assembled from the oracle's M and H, is half the
    finite-difference derivative of the dense objective (Eq 7).  This pins the oracle's
    MTTKRP and H against calculus; the gradient used INSIDE the pass is pinned by
    test_pass_is_exact_coordinate_minimisation."""
    dims, R = (4, 5, 3), 3
    c, v, F = rand_inst(dims, 0.7, R, 3)
    X = dense_tensor(c, v, dims)
    for n in range(3):
        M = O.mttkrp(c, v, dims, n, F)
        H = O.mode_hessian(F, dims, n)
        # the formula the pass must implement, g = -M + F H (Eq 9 / 14), against FD of Eq 7
        G = -M + F[n] @ H
        eps = 1e-6
        for i in range(dims[n]):
            for r in range(R):
                Fp = [x.copy() for x in F]
                Fm = [x.copy() for x in F]
                Fp[n][i, r] += eps
                Fm[n][i, r] -= eps
                fd = (f_dense(X, Fp) - f_dense(X, Fm)) / (2 * eps)
                assert abs(2 * G[i, r] - fd) < 1e-6 * max(1.0, abs(fd))


@pytest.mark.parametrize("n", [0, 1, 2])
def test_pass_is_exact_coordinate_minimisation(n):
    """P5 + P6 + P7: with selection off (FIRST) every coordinate step of the GS pass is the
    exact minimiser over t >= -u of the dense objective (parabola through 3 points), and
    2z equals the objective decrease of that step (L_r = h_rr)."""
    dims, R = (5, 4, 3), 3
    c, v, F = rand_inst(dims, 0.6, R, 21 + n)
    X = dense_tensor(c, v, dims)
    M = O.mttkrp(c, v, dims, n, F)
    H = O.mode_hessian(F, dims, n)
    Fn, zp, ti, E, Ech, md, dec = one_row_pass(M, H, F[n], np.zeros_like(F[n]), O.BR_FIRST)
    cur = [x.copy() for x in F]
    for r in range(R):
        # exact minimiser of each row's objective in coordinate r (rows are separable)
        before = f_rows(X, cur, n)
        ts = [0.0, 0.5, 1.0]
        vals = []
        for t in ts:
            tmp = [x.copy() for x in cur]
            tmp[n][:, r] += t
            vals.append(f_rows(X, tmp, n))
        f0, f1, f2 = vals
        a2 = 4 * (f2 - 2 * f1 + f0)              # second derivative of f(t), step 0.5
        b1 = (4 * f1 - 3 * f0 - f2)              # first derivative at t=0
        tstar = np.maximum(-b1 / a2, -cur[n][:, r])
        newcol = cur[n][:, r] + tstar
        np.testing.assert_allclose(Fn[:, r], newcol, rtol=1e-9, atol=1e-11)
        cur[n][:, r] = Fn[:, r]
        after = f_rows(X, cur, n)
        np.testing.assert_allclose(2 * zp[:, r], before - after, rtol=1e-8, atol=1e-10)
    assert (Fn >= 0).all()


def test_frobenius_importance_is_a_lower_bound():
    """P6 with L = ||H||_F >= h_rr: z <= the exact half-decrease."""
    dims, R = (5, 4, 3), 3
    c, v, F = rand_inst(dims, 0.6, R, 8)
    M = O.mttkrp(c, v, dims, 0, F)
    H = O.mode_hessian(F, dims, 0)
    _, zd, *_ = O.mode_pass(M, H, F[0], np.zeros_like(F[0]), O.BR_FIRST, l_mode=O.L_DIAG)
    _, zf, *_ = O.mode_pass(M, H, F[0], np.zeros_like(F[0]), O.BR_FIRST, l_mode=O.L_FROB)
    # compare column 0 only (later columns see different GS histories)
    assert (zf[:, 0] <= zd[:, 0] + 1e-15).all()
    # strict where the step moves: ||H||_F > h_00 whenever H has another nonzero entry, and
    # z_diag - z_frob = (||H||_F - h_00) d^2 / 2 (Eq 20) with the same g and d
    Fd, *_ = O.mode_pass(M, H, F[0], np.zeros_like(F[0]), O.BR_FIRST, l_mode=O.L_DIAG)
    moved = Fd[:, 0] != F[0][:, 0]
    assert moved.any()
    assert (zf[moved, 0] < zd[moved, 0]).all()
    d = Fd[moved, 0] - F[0][moved, 0]
    np.testing.assert_allclose(zd[moved, 0] - zf[moved, 0], (O.frobenius(H) - H[0, 0]) * d * d / 2,
                               rtol=1e-9, atol=0)


@pytest.mark.parametrize("case", ["frob_diag_H", "frob_full_H"])
def test_frobenius_importance_golden(golden, case):
    """Alg 1's L = ||H||_F inside Eq 20, on hand-derived one-row passes
    (tests/golden/frob_and_echanged.json): pins that the FROB pass really uses ||H||_F
    (incl. off-diagonal entries), not h_rr."""
    g = golden["frob_and_echanged"][case]
    M, H = np.array([g["m"]]), np.array(g["H"])
    u = np.array([g["u"]])
    for l_mode, key in ((O.L_DIAG, "z_diag"), (O.L_FROB, "z_frob")):
        Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, u, np.zeros_like(u), O.BR_FIRST, l_mode=l_mode,
                                                 decisions=True)
        np.testing.assert_allclose(zp[0], g[key], rtol=0, atol=1e-15)
        np.testing.assert_array_equal(Fn[0], g["u_new"])
        assert E == g["E"] and Ech == g["E_changed"]
        assert abs(ti - sum(g[key])) <= 1e-15


@pytest.mark.parametrize("case", ["echanged_zero_step", "echanged_mixed_row"])
def test_echanged_golden(golden, case):
    """E vs E_changed (Lemma 4; reading C14): an EQ27 selection with d = 0 counts in E
    but not in E_changed (tests/golden/frob_and_echanged.json)."""
    g = golden["frob_and_echanged"][case]
    M, H = np.array([g["m"]]), np.array(g["H"])
    u, zprev = np.array([g["u"]]), np.array([g["zprev"]])
    br = {"EQ24": O.BR_EQ24, "EQ27": O.BR_EQ27, "FIRST": O.BR_FIRST}[g["branch"]]
    Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, u, zprev, br, decisions=True)
    np.testing.assert_array_equal(Fn[0], g["u_new"])
    np.testing.assert_allclose(zp[0], g["z"], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(dec[0], g["selected"])
    assert E == g["E"] and Ech == g["E_changed"]


@pytest.mark.parametrize("branch", [0, 1, 2])
def test_echanged_counts_selected_elements_that_moved(branch):
    """C14 on a random pass: E = #decisions, E_changed = #(selected and value changed),
    counted here from the pass's own before / after factors."""
    dims, R = (7, 6, 5), 4
    c, v, F = rand_inst(dims, 0.5, R, 11)
    M = O.mttkrp(c, v, dims, 0, F)
    H = O.mode_hessian(F, dims, 0)
    rng = np.random.default_rng(3)
    zprev = rng.uniform(-0.2, 0.2, size=F[0].shape)
    zprev[rng.uniform(size=zprev.shape) < 0.3] = 0.0
    Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, F[0], zprev, branch, decisions=True)
    assert E == int(dec.sum())
    assert Ech == int((dec.astype(bool) & (Fn != F[0])).sum())
    assert (Fn[~dec.astype(bool)] == F[0][~dec.astype(bool)]).all()


def test_hand_trace(golden):
    g = golden["hand_trace_1x1x1"]
    F = [np.array(g["U0"]), np.array(g["V"]), np.array(g["W"])]
    c, v = np.array(g["coords"]), np.array(g["vals"], np.float32)
    M = O.mttkrp(c, v, g["dims"], 0, F)
    H = O.mode_hessian(F, g["dims"], 0)
    assert M[0, 0] == g["m"] and H[0, 0] == g["h"]
    Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, F[0], np.zeros((1, 1)), O.BR_FIRST, decisions=True)
    assert Fn[0, 0] == g["u_new"] and zp[0, 0] == g["z"] and E == g["E"] and ti == g["z"]
    assert O.objective_dense(c, v, g["dims"], F) == g["f_before"]
    assert O.objective_dense(c, v, g["dims"], [Fn, F[1], F[2]]) == g["f_after"]


def _scalar_pass(u, g, h, zprev=0.0, branch=O.BR_FIRST, L=None):
    """One element (I=R=1) with m chosen so that Eq 14 gives g: m = u*h - g."""
    m = np.array([[u * h - g]])
    H = np.array([[h]])
    return O.mode_pass(m, H, np.array([[u]]), np.array([[zprev]]), branch, decisions=True)


def test_newton_step_examples(golden):
    for ex in golden["spec_hand_examples"]["newton_step"]:
        Fn, zp, *_ = _scalar_pass(ex["u"], ex["g"], ex["h"])
        assert abs(Fn[0, 0] - ex["u_new"]) < 1e-15


def test_importance_example(golden):
    ex = golden["spec_hand_examples"]["importance"][0]   # g=-2, uhat=0.5, L=4 (=h, u=0)
    Fn, zp, ti, E, *_ = _scalar_pass(0.0, ex["g"], ex["L"])
    assert Fn[0, 0] == ex["uhat"] and zp[0, 0] == ex["z"] and E == 1


def test_saturation_point_examples(golden):
    for ex in golden["spec_hand_examples"]["saturation_point"]:
        g = -np.sqrt(2 * ex["z"])              # u=0, h=1: z = g^2/2
        br = O.BR_EQ24 if ex["branch"] == "EQ24" else O.BR_EQ27
        Fn, zp, ti, E, Ech, md, dec = _scalar_pass(0.0, g, 1.0, zprev=ex["zprev"], branch=br)
        assert abs(zp[0, 0] - ex["z"]) < 1e-15
        assert bool(dec[0, 0]) == ex["selected"] and (Fn[0, 0] > 0) == ex["selected"]


def test_zero_column_is_skipped():
    """C11: h_rr == 0 -> z = 0, no update, not counted."""
    M = np.array([[1.0, 2.0]])
    H = np.array([[0.0, 0.0], [0.0, 2.0]])
    Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, np.array([[0.3, 0.0]]), np.zeros((1, 2)), O.BR_FIRST,
                                             decisions=True)
    assert Fn[0, 0] == 0.3 and zp[0, 0] == 0.0 and not dec[0, 0]
    assert Fn[0, 1] == 1.0 and E == 1


def test_stationary_point_selects_nothing():
    """an exact rank-1 fit has g = 0 everywhere -> uhat = 0, z = 0, E = 0."""
    U, V, W = np.array([[1.0], [2.0]]), np.array([[1.0], [0.5]]), np.array([[2.0], [1.0]])
    X = np.einsum("qr,pr,sr->qps", U, V, W)
    c = np.argwhere(X != 0)
    v = X[X != 0].astype(np.float32)
    F = [U, V, W]
    for n in range(3):
        M = O.mttkrp(c, v, X.shape, n, F)
        H = O.mode_hessian(F, X.shape, n)
        Fn, zp, ti, E, *_ = O.mode_pass(M, H, F[n], np.zeros_like(F[n]), O.BR_FIRST)
        assert E == 0 and (Fn == F[n]).all() and (zp == 0).all()


# ----------------------------------------------------------------------------- P7 / P8 / P9 whole runs
def test_objective_forms_agree(golden):
    g = golden["spec_hand_examples"]["objective_single_cell"]
    F = [np.array(g["U"], float), np.array(g["V"], float), np.array(g["W"], float)]
    c, v = np.array(g["coords"]), np.array(g["vals"], np.float32)
    assert O.objective_dense(c, v, g["dims"], F) == g["f"]
    assert abs(O.objective_sparse(c, v, g["dims"], F) - g["f"]) < 1e-15
    for ex in golden["spec_hand_examples"]["predict"]:
        F = [np.array([ex["u"]], float), np.array([ex["v"]], float), np.array([ex["w"]], float)]
        # zero tensor: f = xhat^2 at the single cell
        assert O.objective_dense(np.zeros((0, 3)), np.zeros(0, np.float32), (1, 1, 1), F) == ex["xhat"] ** 2
    dims, R = (6, 5, 4), 3
    c, v, F = rand_inst(dims, 0.1, R, 4)
    X = dense_tensor(c, v, dims)
    fd = f_dense(X, F)
    assert abs(O.objective_dense(c, v, dims, F) - fd) <= 1e-10 * fd
    assert abs(O.objective_sparse(c, v, dims, F) - fd) <= 1e-10 * fd


@pytest.mark.parametrize("variant", [O.VAR_GS_LAGGED, O.VAR_SELECT_OFF])
@pytest.mark.parametrize("l_mode", [O.L_DIAG, O.L_FROB])
def test_run_monotone_invariants_and_gram_fit(variant, l_mode):
    """P7: f non-increasing every sweep (Lemma 3); P8: factors >= 0, E <= I_n R
    (Lemma 4); P9: the run's Gram-trick f equals the dense f of its factors."""
    dims, R, K = (6, 5, 7), 4, 12
    c, v = SI.tiny_tensor(dims, 0.3, 9)
    c, v = c.numpy(), v.numpy()
    out = O.sacd_run(c, v, dims, R, 1234, K, l_mode=l_mode, variant=variant)
    f = out["f"]
    assert (np.diff(f) <= 1e-12 * f[0]).all()
    X = dense_tensor(c, v, dims)
    assert abs(f[-1] - f_dense(X, out["F"])) <= 1e-10 * f[0]
    assert abs(f[0] - f_dense(X, O.init_factors(dims, R, 1234))) <= 1e-10 * f[0]
    for n in range(3):
        assert (out["F"][n] >= 0).all()
        assert (out["E"][:, n] <= dims[n] * R).all() and (out["Ech"][:, n] <= out["E"][:, n]).all()
    assert abs(out["xnorm2"] - float((v.astype(np.float64) ** 2).sum())) < 1e-12 * out["xnorm2"]
    # ti^k is the sum of the final z_prev of the last sweep
    for n in range(3):
        assert abs(out["ti"][-1, n] - out["zprev"][n].sum()) <= 1e-12 * max(1, abs(out["ti"][-1, n]))


def test_telescoping_pass_decrease():
    """P7: in one pass, sum over APPLIED updates of 2z = f(start) - f(end), any branch."""
    dims, R = (5, 6, 4), 3
    c, v, F = rand_inst(dims, 0.5, R, 31)
    X = dense_tensor(c, v, dims)
    rng = np.random.default_rng(2)
    for br in (O.BR_FIRST, O.BR_EQ24, O.BR_EQ27):
        for n in range(3):
            M = O.mttkrp(c, v, dims, n, F)
            H = O.mode_hessian(F, dims, n)
            zp0 = rng.random(F[n].shape) * 0.05
            Fn, zp, ti, E, Ech, md, dec = O.mode_pass(M, H, F[n], zp0, br, decisions=True)
            G = [x for x in F]
            G2 = list(G)
            G2[n] = Fn
            dec_f = f_dense(X, G) - f_dense(X, G2)
            assert abs(dec_f - 2 * zp[dec.astype(bool)].sum()) <= 1e-10 * f_dense(X, G)
            assert E == dec.sum()


def test_branch_rule_lagged():
    """Reading C10: k=1 FIRST, k=2 EQ24, k>=3 EQ27 iff ti^{k-1} > ti^{k-2}."""
    assert O.branch(1, []) == O.BR_FIRST
    assert O.branch(2, [5.0]) == O.BR_EQ24
    assert O.branch(3, [5.0, 6.0]) == O.BR_EQ27
    assert O.branch(3, [5.0, 4.0]) == O.BR_EQ24
    assert O.branch(3, [5.0, 5.0]) == O.BR_EQ24
    assert O.branch(4, [1.0, 3.0, 2.0]) == O.BR_EQ24
    assert O.branch(7, [1.0] * 6, O.VAR_SELECT_OFF) == O.BR_FIRST


def test_thread_count_invariance():
    dims, R = (40, 30, 20), 5
    c, v = SI.tiny_tensor(dims, 0.05, 3)
    c, v = c.numpy(), v.numpy()
    O.set_threads(1)
    a = O.sacd_run(c, v, dims, R, 7, 6)
    O.set_threads(4)
    b = O.sacd_run(c, v, dims, R, 7, 6)
    O.set_threads(0)
    for n in range(3):
        assert np.array_equal(a["F"][n], b["F"][n])
    assert np.array_equal(a["f"], b["f"]) and np.array_equal(a["E"], b["E"])


def test_init_argument_matches_seeded_init():
    dims, R = (5, 4, 3), 2
    c, v = SI.tiny_tensor(dims, 0.4, 5)
    a = O.sacd_run(c.numpy(), v.numpy(), dims, R, 99, 3)
    b = O.sacd_run(c.numpy(), v.numpy(), dims, R, 0, 3, init=O.init_factors(dims, R, 99))
    assert np.array_equal(a["f"], b["f"])


# ----------------------------------------------------------------------------- P11 / P12
def planted(dims, R, seed):
    F = O.init_factors(dims, R, seed + 1000)
    X = np.einsum("qr,pr,sr->qps", *F)
    c = np.argwhere(np.ones(dims, bool))
    return c, X.reshape(-1).astype(np.float32), X


def test_planted_recovery_selection_off():
    """P11(i): fully observed 10x9x8 tensor of planted nonnegative rank-3 factors; with
    selection off (projected GS CD) f/||X||^2 -> < 1e-10 within 2000 sweeps on >= 9/10
    seeds.  Pins MTTKRP, H, step and GS together against an exactly known optimum
    (f = 0 up to fp32 rounding of the values: the test tensor is the fp32-rounded CP
    model, so the floor is ~(2^-24)^2 relative)."""
    dims, R = (10, 9, 8), 3
    ok = 0
    for seed in range(10):
        c, v, X = planted(dims, R, seed)
        out = O.sacd_run(c, v, dims, R, seed, 2000, variant=O.VAR_SELECT_OFF)
        rel = out["f"][-1] / out["xnorm2"]
        ok += rel < 1e-10
    assert ok >= 9


def test_planted_selection_on_reports():
    """P11(ii): selection on -- exact recovery is parity-unpinned; check only that the run
    is monotone, nonnegative and that E = 0 is absorbing once reached."""
    dims, R = (10, 9, 8), 3
    c, v, X = planted(dims, R, 0)
    out = O.sacd_run(c, v, dims, R, 0, 60)
    f = out["f"]
    assert (np.diff(f) <= 1e-12 * f[0]).all() and f[-1] < f[0]
    tot = out["E"].sum(axis=1)
    z = np.nonzero(tot == 0)[0]
    if len(z):
        assert (tot[z[0]:] == 0).all() and np.all(f[z[0] + 1:] == f[z[0] + 1])


def test_jacobi_literal_increases_f():
    """P12 / reading C9: the Lemma-2-literal Jacobi update (gradients not refreshed within
    a row) is not monotone: on a seeded uniform-init R=5 instance it increases f, which
    contradicts Lemma 3 -- the evidence for the Gauss-Seidel reading."""
    dims, R = (8, 7, 6), 5
    c, v = SI.tiny_tensor(dims, 1.0, 13)
    out = O.sacd_run(c.numpy(), v.numpy(), dims, R, 5, 15, variant=O.VAR_JACOBI)
    assert (np.diff(out["f"]) > 0).any()
    gs = O.sacd_run(c.numpy(), v.numpy(), dims, R, 5, 15)
    assert (np.diff(gs["f"]) <= 1e-12 * gs["f"][0]).all()


# ----------------------------------------------------------------------------- snapshot-scored exact ti (f4)
@pytest.mark.parametrize("n", [0, 1, 2])
def test_snapshot_scores_are_pass_start_half_decreases(n):
    """Reading C10': the snapshot z of every element is Alg 1's Eq 20 with G
    from the pass start, i.e. (L_r = h_rr, P6) half the exact decrease of the dense
    objective when that ONE coordinate takes its projected step from the pass-start
    factors; ti^k is their sum (Eq 25).  Brute force on every (i, r)."""
    dims, R = (4, 5, 3), 3
    c, v, F = rand_inst(dims, 0.7, R, 41 + n)
    X = dense_tensor(c, v, dims)
    M = O.mttkrp(c, v, dims, n, F)
    H = O.mode_hessian(F, dims, n)
    _, zs, ti, *_ = O.mode_pass_snapshot(M, H, F[n], np.zeros_like(F[n]), True, 0.0)
    base = f_dense(X, F)
    for i in range(dims[n]):
        for r in range(R):
            # exact 1-D minimiser over t >= -u of the parabola through 3 points
            vals = []
            for t in (0.0, 0.5, 1.0):
                tmp = [x.copy() for x in F]
                tmp[n][i, r] += t
                vals.append(f_dense(X, tmp))
            f0, f1, f2 = vals
            a2, b1 = 4 * (f2 - 2 * f1 + f0), 4 * f1 - 3 * f0 - f2
            tstar = max(-b1 / a2, -F[n][i, r])
            tmp = [x.copy() for x in F]
            tmp[n][i, r] += tstar
            assert abs(2 * zs[i, r] - (base - f_dense(X, tmp))) <= 1e-8 * base
    assert abs(ti - zs.sum()) <= 1e-12 * max(1.0, abs(ti))


def test_snapshot_branch_is_exact_timing_and_run_is_monotone():
    """Reading C10': the branch of sweep k >= 2 is Eq 27 iff ti^k > ti^{k-1} with the CURRENT
    pass's ti, k = 1 is the z > 0 rule; every applied update is a
    Gauss-Seidel coordinate minimisation, so f is non-increasing (Lemma 3), factors
    stay >= 0 and E <= I_n R (Lemma 4).  The run's f equals the dense objective (P9)."""
    dims, R, K = (6, 5, 7), 4, 12
    c, v = SI.tiny_tensor(dims, 0.3, 19)
    c, v = c.numpy(), v.numpy()
    out = O.sacd_run(c, v, dims, R, 77, K, variant=O.VAR_SNAPSHOT)
    f, ti, br = out["f"], out["ti"], out["branch"]
    assert (br[0] == O.BR_FIRST).all()
    for k in range(1, K):
        for n in range(3):
            assert br[k, n] == (O.BR_EQ27 if ti[k, n] > ti[k - 1, n] else O.BR_EQ24)
    assert (np.diff(f) <= 1e-12 * f[0]).all()
    X = dense_tensor(c, v, dims)
    assert abs(f[-1] - f_dense(X, out["F"])) <= 1e-10 * f[0]
    for n in range(3):
        assert (out["F"][n] >= 0).all()
        assert (out["E"][:, n] <= dims[n] * R).all() and (out["Ech"][:, n] <= out["E"][:, n]).all()
        assert abs(ti[-1, n] - out["zprev"][n].sum()) <= 1e-12 * max(1, abs(ti[-1, n]))


def test_snapshot_gate_and_gauss_seidel_steps():
    """Reading C10': element (i, r) is updated iff its snapshot score passes the gate
    (Eq 24: z - z_prev > 0; Eq 27: z_prev - z > 0; z > 0 at k = 1), and an
    updated element lands on the exact minimiser of the CURRENT row (columns < r already
    updated): checked coordinate by coordinate against the dense objective."""
    dims, R = (5, 4, 3), 3
    c, v, F = rand_inst(dims, 0.6, R, 57)
    X = dense_tensor(c, v, dims)
    n = 0
    M = O.mttkrp(c, v, dims, n, F)
    H = O.mode_hessian(F, dims, n)
    rng = np.random.default_rng(5)
    zp0 = rng.random(F[n].shape) * 0.05
    for br in (O.BR_FIRST, O.BR_EQ24, O.BR_EQ27):
        Fn, zs, ti, E, Ech, md, dec, b = O.mode_pass_snapshot(M, H, F[n], zp0, False, 0.0, decisions=True,
                                                              branch=br)
        assert b == br
        gate = {O.BR_FIRST: zs > 0, O.BR_EQ24: zs - zp0 > 0, O.BR_EQ27: zp0 - zs > 0}[br]
        np.testing.assert_array_equal(dec.astype(bool), gate & (np.diag(H) != 0)[None, :])
        assert E == dec.sum()
        cur = [x.copy() for x in F]
        for i in range(dims[n]):
            for r in range(R):
                if not dec[i, r]:
                    assert Fn[i, r] == cur[n][i, r]
                    continue
                vals = []
                for t in (0.0, 0.5, 1.0):
                    tmp = [x.copy() for x in cur]
                    tmp[n][i, r] += t
                    vals.append(f_dense(X, tmp))
                f0, f1, f2 = vals
                a2, b1 = 4 * (f2 - 2 * f1 + f0), 4 * f1 - 3 * f0 - f2
                tstar = max(-b1 / a2, -cur[n][i, r])
                assert abs(Fn[i, r] - (cur[n][i, r] + tstar)) <= 1e-9 * max(1.0, abs(Fn[i, r]))
                cur[n][i, r] = Fn[i, r]


# ----------------------------------------------------------------------------- held-out evaluation (f3)
def test_predict_sum_of_squares_is_gram_identity():
    """Eq 8 over every cell of a small box: sum xhat^2 = 1^T (G_U * G_V * G_W) 1 (the Gram
    identity behind Eq 7's model term), a different route than the per-cell products."""
    dims = (7, 5, 6)
    F = O.init_factors(dims, 4, 21)
    cells = np.stack(np.meshgrid(*[np.arange(d) for d in dims], indexing="ij"), -1).reshape(-1, 3)
    xh = O.predict(cells.astype(np.uint32), dims, F)
    G = [O.gram(f) for f in F]
    assert abs((xh ** 2).sum() - (G[0] * G[1] * G[2]).sum()) <= 1e-12 * (xh ** 2).sum()
    # and the CP model entry itself against the dense Kruskal tensor of f_dense (Eq 8)
    Xh = np.einsum("qr,pr,sr->qps", *F)
    assert np.allclose(xh, Xh.reshape(-1), rtol=1e-14, atol=0)


def test_rmse_against_dense_objective():
    """Eq 30 on the TRAINING entries: n * rmse^2 = sum_Omega (x - xhat)^2
    = f_dense - sum_{cells not in Omega} xhat^2 (Eq 7 over all cells, C1)."""
    dims = (6, 7, 5)
    c, v, F = rand_inst(dims, 0.3, 3, 8)
    X = dense_tensor(c, v, dims)
    r = O.rmse(c, v, dims, F)
    mask = np.ones(dims, bool)
    mask[c[:, 0], c[:, 1], c[:, 2]] = False
    Xh = np.einsum("qr,pr,sr->qps", *F)
    lhs = len(v) * r * r
    rhs = f_dense(X, F) - (Xh[mask] ** 2).sum()
    assert abs(lhs - rhs) <= 1e-10 * abs(rhs)


def test_predict_errors_and_empty():
    dims = (4, 4, 4)
    F = O.init_factors(dims, 2, 1)
    with pytest.raises(O.OracleError):
        O.predict(np.array([[0, 4, 0]], np.uint32), dims, F)
    assert O.rmse(np.zeros((0, 3), np.uint32), np.zeros(0, np.float32), dims, F) == 0.0


def test_rmse_paper_synthetic_band(golden):
    """P13: the paper's held-out RMSE on its synthetic tensors
    (Fig rmsesyn, tests/golden/rmse_synthetic_fig_rmsesyn.json): 80/20 split of a 2048^3
    tensor, density 1e-5, values uniform (0,1], R = 10, 30 sweeps -> RMSE in the band."""
    g = golden["rmse_synthetic_fig_rmsesyn"]
    lo, hi = g["band_for_large_modes"]
    assert all(lo <= x <= hi for x in g["sacd_rmse"][3:])
    dims = (2048, 2048, 2048)
    nnz = int(1e-5 * 2048 ** 3)
    cfg = SI.custom_config(dims, nnz, 10, cid=1411)
    c, v = SI.make_tensor(cfg)
    trc, trv, tec, tev = SI.split_train_test(c, v, dims, cfg.seed)
    out = O.sacd_run(trc.numpy(), trv.numpy(), dims, 10, cfg.seed, 30)
    assert np.all(np.diff(out["f"]) <= 1e-9 * out["f"][0])     # monotone (Lemma 3)
    r = O.rmse(tec.numpy(), tev.numpy(), dims, out["F"])
    assert lo <= r <= hi, r
