"""Parity of the sm_100a symmetric SpMM (be_op_apply) with the oracle.

Reference: kernels.hpp:290-371 (spmm_notrans / spmm_trans / SymmetricOperator)
and the known answers of tests/test_kernels.cpp. Tolerances: the north star's
1e-5 relative Frobenius for f32 values (measured gap ~1e-7), 1e-12 for the
f64-values mode; indexing of the device tile format is checked bit-exactly.
"""
import numpy as np
import pytest

import oracle_lib as ol
from paper_2109_00485_b200 import abi

pytestmark = pytest.mark.gpu


def relf(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(a), np.linalg.norm(b), 1e-300)


def random_triples(nrows, ncols, count, seed):
    rng = np.random.default_rng(seed)
    keys = rng.choice(nrows * ncols, size=count, replace=False)
    return abi.as_triples(keys // ncols, keys % ncols, rng.uniform(-1, 1, count))


def random_lower(n, count, seed):
    rng = np.random.default_rng(seed)
    tot = n * (n - 1) // 2
    keys = rng.choice(tot, size=count, replace=False)
    r = ((1 + np.sqrt(1 + 8 * keys.astype(np.float64))) // 2).astype(np.int64)
    r = np.where(r * (r - 1) // 2 > keys, r - 1, r)
    r = np.where((r + 1) * r // 2 <= keys, r + 1, r)
    c = keys - r * (r - 1) // 2
    assert np.all(c < r) and np.all(c >= 0)
    return abi.as_triples(r, c, rng.uniform(-1, 1, count))


def sym_problem(n, nnz, extent, seed):
    t = random_lower(n, nnz, seed)
    b = abi.uniform_boundaries(n, extent)
    m = abi.build_csb_coo(t, n, n, b, b)
    rng = np.random.default_rng(seed + 1)
    diag = 0.5 + rng.uniform(0, 5, n)
    return m, diag


# --- known answers (tests/test_kernels.cpp) ---------------------------------
def test_identity_notrans_returns_w(ctx):  # test_kernels.cpp:35-46
    m = abi.build_csb_coo(abi.as_triples([0, 1, 2], [0, 1, 2], [1.0, 1, 1]), 3, 3, [0, 3], [0, 3])
    w = np.array([[1.0, 1], [2, 2], [3, 3]])
    for prec in (abi.BE_F32, abi.BE_F64):
        op = abi.Operator(ctx, m, values_prec=prec, symmetric=False)
        u = op.apply_host(w, np.zeros((3, 2)), mode=abi.BE_APPLY_NOTRANS_ACC)
        assert np.array_equal(u, w)


def test_zero_matrix_leaves_accumulator(ctx):  # test_kernels.cpp:48-57
    m = abi.build_csb_coo(np.zeros(0, abi.TRIPLE_DTYPE), 6, 6, [0, 3, 6], [0, 3, 6])
    op = abi.Operator(ctx, m, symmetric=False)
    w = np.random.default_rng(1).uniform(-1, 1, (6, 4))
    u = op.apply_host(w, np.ones((6, 4)), mode=abi.BE_APPLY_NOTRANS_ACC)
    assert np.all(u == 1.0)


def test_accumulation_semantics(ctx):  # test_kernels.cpp:59-68: U += H W -> 16
    m = abi.build_csb_coo(abi.as_triples([0], [1], [2.0]), 2, 2, [0, 2], [0, 2])
    op = abi.Operator(ctx, m, symmetric=False)
    u = op.apply_host(np.array([[0.0], [3.0]]), np.array([[10.0], [0.0]]), mode=abi.BE_APPLY_NOTRANS_ACC)
    assert u[0, 0] == 16.0


def test_hand_transpose(ctx):  # test_kernels.cpp:85-99 -> [1, 3, 2]
    m = abi.build_csb_coo(abi.as_triples([0, 0, 1], [0, 2, 1], [1.0, 2, 3]), 2, 3, [0, 2], [0, 3])
    op = abi.Operator(ctx, m, symmetric=False)
    u = op.apply_host(np.ones((2, 1)), np.zeros((3, 1)), mode=abi.BE_APPLY_TRANS_ACC)
    assert np.allclose(u[:, 0], [1.0, 3.0, 2.0], rtol=0, atol=0)


def test_symmetric_mirror_of_one_entry(ctx):  # test_kernels.cpp:217-230
    m = abi.build_csb_coo(abi.as_triples([2], [0], [5.0]), 3, 3, [0, 3], [0, 3])
    op = abi.Operator(ctx, m, np.zeros(3))
    e0 = np.zeros((3, 1)); e0[0] = 1
    e2 = np.zeros((3, 1)); e2[2] = 1
    u0 = op.apply_host(e0)
    u2 = op.apply_host(e2)
    assert u0[2, 0] == 5.0 and u0[0, 0] == 0.0
    assert u2[0, 0] == 5.0 and u2[2, 0] == 0.0


def test_diagonal_only(ctx):  # test_kernels.cpp:206-215
    m = abi.build_csb_coo(np.zeros(0, abi.TRIPLE_DTYPE), 3, 3, [0, 3], [0, 3])
    op = abi.Operator(ctx, m, np.full(3, 2.0))
    assert np.all(op.apply_host(np.ones((3, 1))) == 2.0)


def test_rejects_non_lower_and_shapes(ctx):  # test_kernels.cpp:196-204, 251-257
    notl = abi.build_csb_coo(abi.as_triples([0], [0], [1.0]), 2, 2, [0, 2], [0, 2])
    with pytest.raises(abi.NotStrictlyLower):
        abi.Operator(ctx, notl, np.ones(2))
    g = abi.build_csb_coo(np.zeros(0, abi.TRIPLE_DTYPE), 4, 6, [0, 4], [0, 6])
    op = abi.Operator(ctx, g, symmetric=False)
    with pytest.raises(abi.DimensionMismatch):
        op.apply_host(np.zeros((4, 2)), np.zeros((4, 2)), mode=abi.BE_APPLY_NOTRANS_ACC)
    with pytest.raises(abi.BadParams):
        op.apply_host(np.zeros((6, 2)), mode=abi.BE_APPLY_SYMMETRIC)


# --- random parity against the oracle ---------------------------------------
@pytest.mark.parametrize("nb", [1, 3, 4, 6, 8, 12, 16, 32, 48])
def test_symmetric_apply_matches_oracle(ctx, nb):
    m, diag = sym_problem(3000, 60000, 700, seed=nb)
    x = np.random.default_rng(nb).uniform(-1, 1, (3000, nb))
    want = ol.Impl("orc").spmm(m, diag, x)
    got32 = abi.Operator(ctx, m, diag, values_prec=abi.BE_F32).apply_host(x)
    got64 = abi.Operator(ctx, m, diag, values_prec=abi.BE_F64).apply_host(x)
    assert relf(got32, want) <= 1e-5, relf(got32, want)
    assert relf(got64, want) <= 1e-12, relf(got64, want)


@pytest.mark.parametrize("mode", [abi.BE_APPLY_NOTRANS_ACC, abi.BE_APPLY_TRANS_ACC])
@pytest.mark.parametrize("shape", [(300, 260, 97, 61), (1000, 777, 300, 128), (64, 64, 64, 64)])
def test_rectangular_modes_match_oracle(ctx, mode, shape):
    nr, nc, re, ce = shape
    t = random_triples(nr, nc, nr * nc // 7, seed=nr + mode)
    m = abi.build_csb_coo(t, nr, nc, abi.uniform_boundaries(nr, re), abi.uniform_boundaries(nc, ce))
    nb = 8
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (nc if mode == abi.BE_APPLY_NOTRANS_ACC else nr, nb))
    y0 = rng.uniform(-1, 1, (nr if mode == abi.BE_APPLY_NOTRANS_ACC else nc, nb))
    want = ol.Impl("orc").spmm(m, None, x, y0, mode=mode)
    for prec, tol in ((abi.BE_F32, 1e-5), (abi.BE_F64, 1e-12)):
        got = abi.Operator(ctx, m, values_prec=prec, symmetric=False).apply_host(x, y0.copy(), mode=mode)
        assert relf(got, want) <= tol


def test_dense_block_splits_tiles(ctx):
    """A fully dense 300x300 lower block: 128x128 sub-tiles exceed max_nnz and
    are split by rows; indexing must stay exact."""
    n = 300
    r, c = np.tril_indices(n, -1)
    t = abi.as_triples(r, c, np.random.default_rng(3).uniform(-1, 1, len(r)))
    m = abi.build_csb_coo(t, n, n, [0, n], [0, n])
    diag = np.full(n, 400.0)
    op = abi.Operator(ctx, m, diag)
    assert op.info().ntiles > 6  # splits happened
    x = np.random.default_rng(4).uniform(-1, 1, (n, 16))
    assert relf(op.apply_host(x), ol.Impl("orc").spmm(m, diag, x)) <= 1e-5
    check_decode(op, m)


def check_decode(op, m):
    """Device tile format decodes back to the CSB entries bit-exactly."""
    rows, cols, vals, idx = op.decode()
    assert np.array_equal(np.sort(idx), np.arange(m.nnz))  # a permutation of CSB positions
    bi = np.searchsorted(m.row_offsets, np.arange(m.nrows), side="right") - 1
    bj = np.searchsorted(m.col_offsets, np.arange(m.ncols), side="right") - 1
    # global coordinates of every CSB entry
    blk = np.repeat(np.arange(len(m.block_nnz)), m.block_nnz.astype(np.int64))
    order = np.argsort(m.block_nnz_offsets[blk], kind="stable")  # entries are laid out block by block
    gr = np.empty(m.nnz, np.int64)
    gc = np.empty(m.nnz, np.int64)
    k = np.arange(m.nnz)
    # block of entry k: last block whose offset <= k among nonempty blocks
    nonempty = np.nonzero(m.block_nnz)[0]
    starts = m.block_nnz_offsets[nonempty]
    owner = nonempty[np.searchsorted(starts, k, side="right") - 1]
    gr = m.row_offsets[owner // m.ncolblks] + m.local_rows.astype(np.int64)
    gc = m.col_offsets[owner % m.ncolblks] + m.local_cols.astype(np.int64)
    assert np.array_equal(rows, gr[idx]) and np.array_equal(cols, gc[idx])
    prec = op.info().values_prec
    want_v = m.values[idx].astype(np.float32).astype(np.float64) if prec == abi.BE_F32 else m.values[idx]
    assert np.array_equal(vals, want_v)
    del bi, bj, order


@pytest.mark.parametrize("prec", [abi.BE_F32, abi.BE_F64])
def test_tile_format_decodes_bit_exact(ctx, prec):
    m, diag = sym_problem(2500, 40000, 900, seed=11)
    check_decode(abi.Operator(ctx, m, diag, values_prec=prec), m)


def test_device_pointer_entry_with_torch_stream(ctx):
    torch = pytest.importorskip("torch")
    m, diag = sym_problem(4000, 80000, 1000, seed=21)
    op = abi.Operator(ctx, m, diag)
    x = torch.rand(4000, 16, dtype=torch.float32, device="cuda") * 2 - 1
    y = torch.empty_like(x)
    s = torch.cuda.current_stream()
    op.apply_dev(x.data_ptr(), y.data_ptr(), 4000, 16, abi.BE_F32, abi.BE_APPLY_SYMMETRIC, s.cuda_stream)
    s.synchronize()
    want = ol.Impl("orc").spmm(m, diag, x.double().cpu().numpy())
    assert relf(y.double().cpu().numpy(), want) <= 1e-5


def test_clustered_generator_parity(ctx):
    m, diag, _ = abi.generate_clustered(n=40000, target_nnz=2_000_000, seed=7)
    assert m.is_strictly_lower()
    x = np.random.default_rng(2).uniform(-1, 1, (40000, 16))
    want = ol.Impl("orc").spmm(m, diag, x)
    op = abi.Operator(ctx, m, diag)
    assert relf(op.apply_host(x), want) <= 1e-5
    check_decode(op, m)


@pytest.mark.slow
def test_config1_random_spmm_parity(ctx):
    """BASELINE config 1 matrix (generate_synthetic Random, n=1e5, 5e7 nnz)."""
    n = 100_000
    s = abi.Synthetic("random", n=n, density=5e7 / (n * (n - 1) / 2), block_extent=4000, seed=1)
    assert len(s.lower) == 50_000_000
    b = abi.uniform_boundaries(n, 4000)
    m = abi.build_csb_coo(s.lower, n, n, b, b)
    del s.lower
    x = np.random.default_rng(3).uniform(-1, 1, (n, 16))
    want = ol.Impl("orc").spmm(m, s.diag, x)
    got = abi.Operator(ctx, m, s.diag).apply_host(x)
    assert relf(got, want) <= 1e-5


# --- deterministic mode (BE_OP_DETERMINISTIC, the mirror's reference variant names) -----
@pytest.mark.parametrize("nb", [1, 5, 16, 40])
def test_deterministic_mode_is_bit_exact_with_the_serial_reference(ctx, nb):
    """f64 values summed in run_baseline's serial order (kernels.hpp:253-276) without FMA
    contraction: bit-identical to the reference itself (oracle/_ref, ThreadPool-free baseline)
    in all three apply modes, and bit-reproducible."""
    try:
        ref = ol.Impl("ref", threads=1, variant=0)
    except FileNotFoundError:
        pytest.skip("oracle/_ref/libref.so not built")
    m, diag = sym_problem(2000, 30000, 700, 11)
    op = abi.Operator(ctx, m, diag, values_prec=abi.BE_F64, deterministic=True)
    x = np.random.default_rng(nb).uniform(-1, 1, (2000, nb))
    got = op.apply_host(x)
    assert np.array_equal(got, ref.spmm(m, diag, x))
    assert np.array_equal(got, op.apply_host(x))
    y0 = np.random.default_rng(99).uniform(-1, 1, (2000, nb))
    for mode in (abi.BE_APPLY_NOTRANS_ACC, abi.BE_APPLY_TRANS_ACC):
        assert np.array_equal(op.apply_host(x, y0.copy(), mode=mode), ref.spmm(m, None, x, y0, mode=mode))


def test_deterministic_solve_is_bit_reproducible(ctx):
    """test_lobpcg.cpp:389-407 (identical history for an identical seed) on the device: the
    deterministic operator plus the fixed-order dense reductions."""
    m, diag = sym_problem(1500, 9000, 500, 3)
    op = abi.Operator(ctx, m, diag, values_prec=abi.BE_F64, deterministic=True)
    r1 = abi.lobpcg(ctx, op, k=3, nb=6, tol=1e-8, seed=42)
    r2 = abi.lobpcg(ctx, op, k=3, nb=6, tol=1e-8, seed=42)
    assert r1["iterations"] == r2["iterations"]
    assert np.array_equal(r1["lambda_"], r2["lambda_"]) and np.array_equal(r1["x"], r2["x"])
    assert np.array_equal(r1["theta"], r2["theta"]) and np.array_equal(r1["residual_norms"], r2["residual_norms"])


# --- row-list format (BE_OP_FORMAT_ROWS: very sparse matrices, X gathered from L2) ----------
@pytest.mark.parametrize("nb", [1, 3, 4, 8, 16, 32, 48])
def test_row_list_format_matches_oracle(ctx, nb):
    m, diag = sym_problem(2500, 20000, 800, 21)
    op = abi.Operator(ctx, m, diag, values_prec=abi.BE_F32, fmt="rows")
    orc = ol.Impl("orc")
    x = np.random.default_rng(nb).uniform(-1, 1, (2500, nb))
    assert relf(op.apply_host(x), orc.spmm(m, diag, x)) <= 1e-5
    y0 = np.random.default_rng(7).uniform(-1, 1, (2500, nb))
    for mode in (abi.BE_APPLY_NOTRANS_ACC, abi.BE_APPLY_TRANS_ACC):
        assert relf(op.apply_host(x, y0.copy(), mode=mode), orc.spmm(m, None, x, y0, mode=mode)) <= 1e-5


@pytest.mark.parametrize("nb", [8, 16])
def test_row_list_format_f32_panels_and_determinism(ctx, nb):
    import torch
    m, diag = sym_problem(3000, 40000, 1000, 5)
    op = abi.Operator(ctx, m, diag, values_prec=abi.BE_F32, fmt="rows")
    x = torch.rand(3000, nb, dtype=torch.float32, device="cuda") * 2 - 1
    y1 = torch.empty_like(x)
    y2 = torch.empty_like(x)
    op.apply_dev(x.data_ptr(), y1.data_ptr(), 3000, nb, abi.BE_F32, abi.BE_APPLY_SYMMETRIC, ctx.stream())
    op.apply_dev(x.data_ptr(), y2.data_ptr(), 3000, nb, abi.BE_F32, abi.BE_APPLY_SYMMETRIC, ctx.stream())
    ctx.synchronize()
    assert torch.equal(y1, y2)  # no atomics: every output row is summed by one lane group
    want = ol.Impl("orc").spmm(m, diag, x.double().cpu().numpy())
    assert relf(y1.double().cpu().numpy(), want) <= 1e-5


def test_auto_format_choice(ctx):
    """Large and sparse (C1-like density) -> row lists; the clustered generator -> tiles."""
    s = abi.Synthetic("random", n=40000, density=0.006, block_extent=4000, seed=3)
    b = abi.uniform_boundaries(40000, 4000)
    m = abi.build_csb_coo(s.lower, 40000, 40000, b, b)
    assert m.nnz >= 1 << 22
    assert abi.Operator(ctx, m, s.diag).info().ntiles == 0
    mc, dc, _ = abi.generate_clustered(n=200000, target_nnz=1 << 23, seed=2)
    assert abi.Operator(ctx, mc, dc).info().ntiles > 0



@pytest.mark.parametrize("values_prec", [abi.BE_F32, abi.BE_F64])
def test_streamed_csb1_operator_matches_in_memory(ctx, tmp_path, values_prec):
    """be_op_create_csb1: the operator streamed from the CSB1 cache in batches of
    whole block rows (here ~20k entries, so several batches and a growing device blob buffer)
    applies the same matrix as the in-memory tile operator and the oracle; the diagonal comes back
    from the file's diagonal section; a file without one is refused."""
    m, diag = sym_problem(6000, 120000, 500, 23)
    path = tmp_path / "m.csb1"
    m.save(path, diag)
    op, d = abi.Operator.from_csb1(ctx, path, values_prec=values_prec, batch_entries=20000)
    assert np.array_equal(d, diag)
    ref = abi.Operator(ctx, m, diag, values_prec=values_prec, fmt="tiles")
    assert op.info().nnz == m.nnz
    x = np.random.default_rng(3).uniform(-1, 1, (6000, 16))
    got, want = op.apply_host(x), ref.apply_host(x)
    tol = 1e-6 if values_prec == abi.BE_F32 else 1e-13
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= tol
    orc = ol.Impl("orc").spmm(m, diag, x)
    assert np.linalg.norm(got - orc) / np.linalg.norm(orc) <= (1e-5 if values_prec == abi.BE_F32 else 1e-12)
    bare = tmp_path / "nodiag.csb1"
    m.save(bare)
    with pytest.raises(abi.DimensionMismatch):
        abi.Operator.from_csb1(ctx, bare)
