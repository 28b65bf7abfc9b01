"""Device-resident LOBPCG (be_lobpcg_solve) against the oracle and the known
answers of tests/test_lobpcg.cpp. Bars (BASELINE.json north star): lowest
eigenvalues within 1e-6 relative, iteration count within +-1 with the
preconditioner off (with it on the reference itself moves with
the summation order)."""
import numpy as np
import pytest

import oracle_lib as ol
from paper_2109_00485_b200 import abi

pytestmark = pytest.mark.gpu


def make_test_matrix(n, nnz_lower, seed, extent=4000):
    """make_test_matrix (test_lobpcg.cpp:24-42) shape: random lower, dominant diagonal."""
    rng = np.random.default_rng(seed)
    tot = n * (n - 1) // 2
    keys = np.sort(rng.choice(tot, size=nnz_lower, replace=False))
    r = ((1 + np.sqrt(1 + 8 * keys.astype(np.float64))) // 2).astype(np.int64)
    r = np.where(r * (r - 1) // 2 > keys, r - 1, r)
    r = np.where((r + 1) * r // 2 <= keys, r + 1, r)
    c = keys - r * (r - 1) // 2
    v = rng.uniform(-1, 1, nnz_lower)
    rowabs = np.zeros(n)
    np.add.at(rowabs, r, np.abs(v))
    np.add.at(rowabs, c, np.abs(v))
    diag = 0.5 + rng.uniform(0, 5, n) + rowabs
    b = abi.uniform_boundaries(n, min(extent, n))
    m = abi.build_csb_coo(abi.as_triples(r, c, v), n, n, b, b)
    return m, diag


def diag_csb(d):
    n = len(d)
    return abi.build_csb_coo(np.zeros(0, abi.TRIPLE_DTYPE), n, n, [0, n], [0, n]), np.asarray(d, float)


def test_diagonal_spectrum_1_to_100(ctx):  # test_lobpcg.cpp:258-272
    m, d = diag_csb(np.arange(1.0, 101.0))
    op = abi.Operator(ctx, m, d)
    res = abi.lobpcg(ctx, op, k=5, nb=8, tol=1e-9, seed=7)
    assert res["converged"]
    assert np.all(np.abs(res["lambda_"] - np.arange(1.0, 6.0)) < 1e-8)
    assert res["iterations"] <= 60


def test_identity_converges_in_one_iteration(ctx):  # test_lobpcg.cpp:274-284
    m, d = diag_csb(np.ones(60))
    res = abi.lobpcg(ctx, abi.Operator(ctx, m, d), k=3, nb=6)
    assert res["converged"] and res["iterations"] == 1
    assert np.allclose(res["lambda_"], 1.0)


def test_exact_invariant_subspace_x0(ctx):  # test_lobpcg.cpp:443-459
    n, nb = 60, 6
    m, d = diag_csb(np.arange(1.0, n + 1))
    x0 = np.zeros((n, nb))
    x0[np.arange(nb), np.arange(nb)] = 1.0
    res = abi.lobpcg(ctx, abi.Operator(ctx, m, d), x0=x0, k=3, nb=nb, tol=1e-10)
    assert res["converged"] and res["iterations"] == 1
    assert np.allclose(res["lambda_"], [1.0, 2.0, 3.0])


def test_dependent_x0_is_rank_deficient(ctx):  # test_lobpcg.cpp:461-475
    n = 40
    m, d = diag_csb(np.ones(n))
    x0 = np.zeros((n, 4))
    x0[:, 0] = 1.0
    x0[:, 1] = 1.0
    x0[:, 2] = np.arange(n)
    x0[:, 3] = np.arange(n) ** 2
    with pytest.raises(abi.RankDeficient):
        abi.lobpcg(ctx, abi.Operator(ctx, m, d), x0=x0, k=2, nb=4)


def test_config_validation(ctx):  # test_lobpcg.cpp:409-421
    m, d = diag_csb(np.ones(100))
    op = abi.Operator(ctx, m, d)
    with pytest.raises(abi.BadParams):
        abi.lobpcg(ctx, op, k=5, nb=4)
    with pytest.raises(abi.BadParams):
        abi.lobpcg(ctx, op, k=5, nb=40)
    with pytest.raises(abi.BadParams):
        abi.lobpcg(ctx, op, k=5, nb=8, tol=0.0)


@pytest.mark.parametrize("seed,n,nnz,k,nb,precond", [(88, 200, 800, 3, 6, False), (7, 3000, 60000, 16, 32, False),
                                                     (8, 3000, 60000, 12, 24, False),
                                                      (99, 1500, 30000, 5, 8, False), (5, 2000, 40000, 8, 16, False)])
def test_matches_oracle(ctx, seed, n, nnz, k, nb, precond):
    m, d = make_test_matrix(n, nnz, seed)
    toff = np.array([0] + list(range(25, n, 25)) + [n]) if precond else None
    want = ol.Impl("orc").lobpcg(m, d, toff, k=k, nb=nb, tol=1e-9, maxiter=800, seed=seed)
    op = abi.Operator(ctx, m, d, values_prec=abi.BE_F64)
    tiles = abi.Tiles(ctx, m, d, toff) if precond else None
    got = abi.lobpcg(ctx, op, tiles=tiles, k=k, nb=nb, tol=1e-9, maxiter=800, seed=seed)
    assert got["converged"] == want["converged"]
    rel = np.max(np.abs(got["lambda_"] - want["lambda_"]) / np.abs(want["lambda_"]))
    assert rel <= 1e-6, rel
    lo, hi = want["iterations"], want["iterations"]
    if precond:  # with the preconditioner the count moves with the summation order
        lo, hi = envelope(m, d, toff, k=k, nb=nb, tol=1e-9, maxiter=800, seed=seed)
    assert lo - 1 <= got["iterations"] <= hi + 1, (got["iterations"], lo, hi)
    assert got["operator_calls"] == got["iterations"] + 1


def envelope(m, d, toff, **kw):
    """min / max iterations of the reference over summation orders: serial and
    ThreadPool(2..8) with the baseline and fused-atomic SpMM variants (SURVEY
    8c; the C1 test uses the same 1..8 thread sweep); oracle alone when the
    reference build is absent."""
    its = [ol.Impl("orc").lobpcg(m, d, toff, **kw)["iterations"]]
    if ol.ref() is not None:
        for threads, variant in [(1, 0)] + [(t, v) for t in range(2, 9) for v in (0, 1)]:
            its.append(ol.Impl("ref", threads=threads, variant=variant).lobpcg(m, d, toff, **kw)["iterations"])
    return min(its), max(its)


@pytest.mark.parametrize("s", range(4))
def test_preconditioned_acceptance_class(ctx, s):
    """acceptance.cpp:286-310 problem class (criterion 6): n=1000, density
    0.5%, FOM(m=4) preconditioner on. With the preconditioner the iteration
    count follows the summation order, so it is compared with the reference's
    own order envelope +-1; eigenvalues to 1e-6."""
    n = 1000
    g = abi.Synthetic("random", n=n, density=0.005, block_extent=1000, seed=6000 + s)
    m = abi.build_csb_coo(g.lower, n, n, [0, n], [0, n])
    kw = dict(k=5, nb=8, tol=1e-6, maxiter=500, seed=6100 + s)
    want = ol.Impl("orc").lobpcg(m, g.diag, g.tile_offsets, **kw)
    got = abi.lobpcg(ctx, abi.Operator(ctx, m, g.diag, values_prec=abi.BE_F64), tiles=abi.Tiles(ctx, m, g.diag, g.tile_offsets), **kw)
    rel = np.max(np.abs(got["lambda_"] - want["lambda_"]) / np.abs(want["lambda_"]))
    assert rel <= 1e-6, rel
    lo, hi = envelope(m, g.diag, g.tile_offsets, **kw)
    if hi > 2 * lo:  # e.g. seed 6003: serial 161 vs threaded 35 -- a stalling cluster, count not well posed
        pytest.skip(f"reference envelope [{lo}, {hi}] too wide for an iteration-count parity check")
    assert lo - 1 <= got["iterations"] <= hi + 1, (got["iterations"], lo, hi)


def test_f32_values_parity(ctx):
    m, d = make_test_matrix(3000, 90000, 3)
    want = ol.Impl("orc").lobpcg(m, d, k=8, nb=16, tol=1e-6, maxiter=400, seed=1)
    got = abi.lobpcg(ctx, abi.Operator(ctx, m, d), k=8, nb=16, tol=1e-6, maxiter=400, seed=1)
    rel = np.max(np.abs(got["lambda_"] - want["lambda_"]) / np.abs(want["lambda_"]))
    assert rel <= 1e-6
    assert abs(got["iterations"] - want["iterations"]) <= 1


def test_long_run_invariants(ctx):  # test_lobpcg.cpp:329-365 (trace, calls, recurrence drift)
    n = 300
    m, d = make_test_matrix(n, 1500, 99)
    op = abi.Operator(ctx, m, d, values_prec=abi.BE_F64)
    dense = np.diag(d)
    drift = []

    def obs(it, theta, rn, nc, x, hx):
        if it % 10 == 0:
            drift.append(np.linalg.norm(hx - op_dense @ x) / max(np.linalg.norm(hx), np.linalg.norm(op_dense @ x)))

    t = m.to_triples()
    dense[t["row"], t["col"]] += t["value"]
    dense[t["col"], t["row"]] += t["value"]
    op_dense = dense
    res = abi.lobpcg(ctx, op, k=4, nb=8, tol=1e-300, maxiter=100, observer=obs, observer_state=True)
    assert not res["converged"] and res["iterations"] == 100
    assert res["operator_calls"] == 101
    assert max(drift) < 1e-9
    tr = res["theta"][:, :4].sum(axis=1)
    assert np.all(tr[1:] <= tr[:-1] + 1e-12 * np.abs(tr[1:]))


def test_observer_receives_the_whole_solver_state(ctx):
    """SolverState (lobpcg.hpp:52-58) at the observer call (:436): X, W, P+ with their H-images.
    The recurrences keep HX = H X, HW = H W and HP = H P; W is orthonormal after its hygiene and
    P+ is orthogonal to X+ and near-orthonormal (lobpcg.hpp:412-417), as in the reference."""
    n = 400
    m, d = make_test_matrix(n, 2000, 5)
    op = abi.Operator(ctx, m, d, values_prec=abi.BE_F64)
    t = m.to_triples()
    dense = np.diag(d)
    dense[t["row"], t["col"]] += t["value"]
    dense[t["col"], t["row"]] += t["value"]
    seen = []

    def obs(it, theta, rn, nc, st):
        seen.append(it)
        for a, ha in (("x", "hx"), ("w", "hw"), ("p", "hp")):
            assert st[a].shape == (n, 8) and st[ha].shape == (n, 8)
            ref = dense @ st[a]
            assert np.linalg.norm(st[ha] - ref) <= 1e-9 * np.linalg.norm(ref), (it, a)
        assert np.allclose(st["w"].T @ st["w"], np.eye(8), atol=1e-8)
        assert np.abs(st["x"].T @ st["p"]).max() < 1e-8
        assert np.allclose(st["p"].T @ st["p"], np.eye(8), atol=1e-6)
        assert np.allclose(np.linalg.norm(st["hx"] - st["x"] * theta, axis=0), rn, rtol=1e-8, atol=1e-12)

    res = abi.lobpcg(ctx, op, k=4, nb=8, tol=1e-300, maxiter=6, observer=obs, observer_panels=True)
    assert seen == list(range(1, 7)) and res["iterations"] == 6


def test_host_operator_closure(ctx):  # generic Operator boundary (lobpcg.hpp:20)
    d = np.arange(1.0, 101.0)
    res = abi.lobpcg(ctx, None, n=100, host_operator=lambda x: d[:, None] * x, k=5, nb=8, tol=1e-9, seed=7)
    assert res["converged"]
    assert np.all(np.abs(res["lambda_"] - np.arange(1.0, 6.0)) < 1e-8)


# --- preconditioner (tests/test_precond.cpp) ---------------------------------
def test_precond_matches_oracle(ctx):
    s = abi.Synthetic("random", n=4000, density=0.01, block_extent=1000, seed=5)
    b = abi.uniform_boundaries(4000, 1000)
    m = abi.build_csb_coo(s.lower, 4000, 4000, b, b)
    tiles = abi.Tiles(ctx, m, s.diag, s.tile_offsets)
    r = np.random.default_rng(1).uniform(-1, 1, (4000, 16))
    sh = np.linspace(5, 30, 16)
    got, fb = tiles.apply_host(sh, r, m=4)
    want, wfb = ol.Impl("orc").precond(m, s.diag, s.tile_offsets, sh, r, m=4)
    assert fb == wfb
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12
    # extract_tiles layout is the reference's, bit for bit
    nent, rows, cols, vals, dpos = ol.orc_extract_tiles(m, s.diag, s.tile_offsets)
    off = 0
    doff = 0
    for j in range(len(nent)):
        dim, tr, tc, tv, td = tiles.tile(j)
        e = int(nent[j])
        assert np.array_equal(tr, rows[off:off + e]) and np.array_equal(tc, cols[off:off + e])
        assert np.array_equal(tv, vals[off:off + e]) and np.array_equal(td, dpos[doff:doff + dim])
        off += e
        doff += dim


def test_precond_known_answers(ctx):
    # 1x1 tiles: Jacobi scaling (test_precond.cpp:249-261)
    d = np.array([2.0, 4.0, 5.0, 8.0, 10.0, 0.5])
    m, _ = diag_csb(d)
    t = abi.Tiles(ctx, m, d, np.arange(7))
    r = np.random.default_rng(50).uniform(-1, 1, (6, 3))
    w, fb = t.apply_host(np.zeros(3), r, m=1)
    assert np.allclose(w, r / d[:, None], rtol=1e-14)
    # identity tiles give W = R (test_precond.cpp:263-271)
    m9, d9 = diag_csb(np.ones(9))
    w9, _ = abi.Tiles(ctx, m9, d9, [0, 3, 6, 9]).apply_host(np.zeros(2), r[:, :2].repeat(2, 0)[:9], m=4)
    assert np.allclose(w9, r[:, :2].repeat(2, 0)[:9], rtol=1e-14)
    # singular projection falls back to the raw residual (test_precond.cpp:232-247)
    m1, d1 = diag_csb([5.0])
    w1, fb1 = abi.Tiles(ctx, m1, d1, [0, 1]).apply_host([5.0], np.array([[2.0]]), m=1)
    assert fb1 == 1 and w1[0, 0] == 2.0


def test_precond_full_dimension_solve(ctx):  # test_precond.cpp:273-308
    n = 60
    rng = np.random.default_rng(60)
    lower_r, lower_c, lower_v, diag = [], [], [], np.zeros(n)
    dense = np.zeros((n, n))
    for t in range(3):
        a = rng.uniform(-1, 1, (20, 20))
        a = np.tril(a) + np.tril(a, -1).T
        a += np.diag(np.abs(a).sum(1) + 1)
        dense[20 * t:20 * t + 20, 20 * t:20 * t + 20] = a
        ii, jj = np.tril_indices(20, -1)
        lower_r += list(20 * t + ii)
        lower_c += list(20 * t + jj)
        lower_v += list(a[ii, jj])
        diag[20 * t:20 * t + 20] = np.diag(a)
    m = abi.build_csb_coo(abi.as_triples(lower_r, lower_c, lower_v), n, n, [0, n], [0, n])
    r = rng.uniform(-1, 1, (n, 2))
    w, _ = abi.Tiles(ctx, m, diag, [0, 20, 40, 60]).apply_host(np.zeros(2), r, m=20)
    want = np.linalg.solve(dense, r)
    assert np.linalg.norm(w - want) <= 1e-8 * np.linalg.norm(want)


# --- dense parity hooks (tests/test_densela.cpp) ------------------------------
def test_sygv_diagonal_pencils(ctx):  # test_densela.cpp:164-183
    a = np.diag([3.0, 1.0, 2.0])
    c, d = abi.sygv_lowest(ctx, a, np.eye(3), 2)
    assert np.allclose(d, [1.0, 2.0]) and abs(c[1, 0] - 1) < 1e-12 and abs(c[2, 1] - 1) < 1e-12
    c2, d2 = abi.sygv_lowest(ctx, np.eye(2), np.diag([1.0, 4.0]), 1)
    assert abs(d2[0] - 0.25) < 1e-14 and abs(c2[0, 0]) < 1e-12 and abs(c2[1, 0] - 0.5) < 1e-14


@pytest.mark.parametrize("n,k", [(24, 24), (48, 16)])
def test_sygv_matches_oracle(ctx, n, k):  # test_densela.cpp:185-234, 338-363
    rng = np.random.default_rng(n)
    a = rng.uniform(-2, 2, (n, n))
    a = np.tril(a) + np.tril(a, -1).T
    x = rng.uniform(-1, 1, (3 * n, n))
    b = x.T @ x + np.eye(n)
    c, d = abi.sygv_lowest(ctx, a, b, k, 1e-10)
    wc, wd = ol.Impl("orc").sygv_lowest(a, b, k, 1e-10)
    assert np.max(np.abs(d - wd) / np.maximum(1, np.abs(wd))) < 1e-10
    assert np.allclose(a @ c, (b @ c) * d, atol=1e-9 * max(1, np.abs(a).max()))
    assert np.allclose(c.T @ b @ c, np.eye(k), atol=1e-9)
    # sign convention: largest-magnitude entry of each column positive
    assert np.all(c[np.abs(c).argmax(0), np.arange(k)] > 0)


def test_sygv_pivot_floor(ctx):
    b = np.diag([1.0, 1e-12])
    with pytest.raises(abi.NotPositiveDefinite):
        abi.sygv_lowest(ctx, np.eye(2), b, 1, 1e-10)


@pytest.mark.parametrize("rows", [12345, 7])
@pytest.mark.parametrize("nb", [8, 16, 24])
def test_gram_matches_numpy(ctx, nb, rows):
    """gram (densela.hpp:80-97): the register-direct kernel (nb 8, 16: one or two panels, a partial
    last 32-row group) and the staged tensor-core kernel (nb 24), f64 against numpy; symmetrised
    pairs are exactly symmetric."""
    torch = pytest.importorskip("torch")
    a = torch.rand(rows, nb, dtype=torch.float64, device="cuda")
    b = torch.rand(rows, nb, dtype=torch.float64, device="cuda")
    g = abi.gram_dev(ctx, a.data_ptr(), b.data_ptr(), nb, rows)
    want = a.cpu().numpy().T @ b.cpu().numpy()
    assert np.allclose(g, want, rtol=1e-12, atol=1e-10)
    gs = abi.gram_dev(ctx, a.data_ptr(), a.data_ptr(), nb, rows)
    assert np.array_equal(gs, gs.T)
    assert np.allclose(gs, a.cpu().numpy().T @ a.cpu().numpy(), rtol=1e-12, atol=1e-10)


@pytest.mark.parametrize("rows", [5000, 4997])
@pytest.mark.parametrize("nb", [8, 12, 16, 24, 32])
def test_block_times_small_matches_numpy(ctx, nb, rows):
    """block_times_small(_add) (densela.hpp:448-484): the tensor-core mixes (nb = 8, 16: register-direct,
    a partial last 8-row block at 4997 rows; 24, 32: staged, coefficient fragments in shared memory) and
    the FFMA kernel (other widths), f64 to ~1e-14."""
    rng = np.random.default_rng(nb)
    x = rng.uniform(-1, 1, (rows, nb))
    c = rng.uniform(-1, 1, (nb, nb))
    y0 = rng.uniform(-1, 1, (rows, nb))
    got = abi.dense_mix(ctx, x, c)
    assert np.max(np.abs(got - x @ c)) <= 1e-13 * nb
    got = abi.dense_mix(ctx, x, c, y0)
    assert np.max(np.abs(got - (y0 + x @ c))) <= 1e-13 * nb


def test_repeated_solves_reuse_the_context_panels(ctx):
    """Solves on one context take their panels from the context's pool (Ctx::panel_pool): the same
    solve twice is bit-identical, a larger problem in between re-allocates, host x0 in and eigenvectors
    out go through the pinned staging path (the 140000-row problem: x0 and the eigenvectors are above
    the 8 MB staging threshold)."""
    m, d = make_test_matrix(1500, 30000, 7)
    op = abi.Operator(ctx, m, d, values_prec=abi.BE_F64)
    a = abi.lobpcg(ctx, op, k=4, nb=8, tol=1e-8, maxiter=300, seed=3)
    mb, db = make_test_matrix(140000, 400000, 8)
    opb = abi.Operator(ctx, mb, db, values_prec=abi.BE_F32)
    x0 = np.random.default_rng(2).uniform(-1, 1, (140000, 16))
    big = abi.lobpcg(ctx, opb, x0=x0, k=8, nb=16, tol=1e-300, maxiter=3, seed=3)
    assert big["x"].shape == (140000, 8) and np.all(np.isfinite(big["x"]))
    # X is orthonormal after the Rayleigh-Ritz update: the staged read-back must be too
    g = big["x"].T @ big["x"]
    assert np.max(np.abs(g - np.eye(8))) < 1e-8
    # (the SpMM's transposed pass reduces with atomics, so repeated solves agree to rounding, not bitwise)
    b = abi.lobpcg(ctx, op, k=4, nb=8, tol=1e-8, maxiter=300, seed=3)
    assert abs(a["iterations"] - b["iterations"]) <= 1
    assert np.max(np.abs(a["lambda_"] - b["lambda_"]) / np.abs(a["lambda_"])) < 1e-10
    assert np.max(np.abs(a["x"] - b["x"])) < 1e-6
    big2 = abi.lobpcg(ctx, opb, x0=x0, k=8, nb=16, tol=1e-300, maxiter=3, seed=3)
    # f32 values + an unordered red.global transpose pass: the two runs agree to f32 rounding
    # amplified by three unconverged iterations, so compare the spanned subspaces (singular values
    # of X1^T X2 are the cosines of the principal angles) and the Ritz values, not bits
    cos = np.linalg.svd(big["x"].T @ big2["x"], compute_uv=False)
    assert 1.0 - cos.min() < 1e-6, cos
    assert np.max(np.abs(big["lambda_"] - big2["lambda_"]) / np.abs(big["lambda_"])) < 1e-6
