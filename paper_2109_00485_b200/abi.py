"""ctypes binding of the C ABI in include/blockeig_b200.h.

Used by the tests and bench.py to drive libblockeig_b200.so exactly the way
a foreign-language host (cgo / JNI / ctypes) would. There is no fallback:
if the shared library is missing or a call fails, an exception is raised
(`BlockeigError` subclasses named after errors.hpp).
"""
from __future__ import annotations

import ctypes as C
import mmap
import sys
import time
from pathlib import Path

import numpy as np

import os as _os

# BE_LIB: an alternative build of the same library (kernel-variant experiments)
LIB_PATH = Path(_os.environ.get("BE_LIB") or str(Path(__file__).resolve().parent / "libblockeig_b200.so"))

BE_F32, BE_F64 = 0, 1
BE_APPLY_SYMMETRIC, BE_APPLY_NOTRANS_ACC, BE_APPLY_TRANS_ACC = 0, 1, 2
BE_OP_SYMMETRIC = 1
BE_OP_DETERMINISTIC = 2  # f64 values, the serial reference summation order (bit-reproducible)
BE_OP_FORMAT_TILES = 4  # force the 128 x 128 tile format
BE_OP_FORMAT_ROWS = 8  # force the row-list format (very sparse matrices)
SYNTH_KINDS = {"banded": 0, "blocktile": 1, "random": 2}


class BlockeigError(RuntimeError):
    code = 1


def _err(name, code):
    return type(name, (BlockeigError,), {"code": code})


BlockTooLarge = _err("BlockTooLarge", 2)
IndexOutOfRange = _err("IndexOutOfRange", 3)
DuplicateEntry = _err("DuplicateEntry", 4)
DimensionMismatch = _err("DimensionMismatch", 5)
NotStrictlyLower = _err("NotStrictlyLower", 6)
MisalignedTiles = _err("MisalignedTiles", 7)
BadParams = _err("BadParams", 8)
NotPositiveDefinite = _err("NotPositiveDefinite", 9)
SingularTriangular = _err("SingularTriangular", 10)
SingularProjection = _err("SingularProjection", 11)
RankDeficient = _err("RankDeficient", 12)
BasisDegenerate = _err("BasisDegenerate", 13)
BreakdownUnrecoverable = _err("BreakdownUnrecoverable", 14)
EvenNd = _err("EvenNd", 15)
ProtocolDeadlock = _err("ProtocolDeadlock", 16)
ParseError = _err("ParseError", 17)
NotSymmetricHeader = _err("NotSymmetricHeader", 18)
CudaError = _err("CudaError", 32)
NoDevice = _err("NoDevice", 33)
CusolverError = _err("CusolverError", 34)
NcclError = _err("NcclError", 35)
OutOfMemory = _err("OutOfMemory", 36)
_BY_CODE = {c.code: c for c in [BlockTooLarge, IndexOutOfRange, DuplicateEntry, DimensionMismatch, NotStrictlyLower,
                                 MisalignedTiles, BadParams, NotPositiveDefinite, SingularTriangular,
                                 SingularProjection, RankDeficient, BasisDegenerate, BreakdownUnrecoverable, EvenNd,
                                 ProtocolDeadlock, ParseError, NotSymmetricHeader, CudaError, NoDevice,
                                 CusolverError, NcclError, OutOfMemory]}


class Triple(C.Structure):
    _fields_ = [("row", C.c_int64), ("col", C.c_int64), ("value", C.c_double)]


TRIPLE_DTYPE = np.dtype([("row", "<i8"), ("col", "<i8"), ("value", "<f8")])


class CsbView(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nrowblks", C.c_int64), ("ncolblks", C.c_int64),
                ("nnz", C.c_int64), ("row_offsets", C.c_void_p), ("col_offsets", C.c_void_p),
                ("block_nnz", C.c_void_p), ("block_nnz_offsets", C.c_void_p), ("local_rows", C.c_void_p),
                ("local_cols", C.c_void_p), ("values", C.c_void_p)]


class SynthParams(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_int64), ("density", C.c_double), ("bandwidth", C.c_int64),
                ("block_extent", C.c_int64), ("tile_min", C.c_int64), ("tile_max", C.c_int64),
                ("diag_spread", C.c_double), ("dominance", C.c_double), ("seed", C.c_uint64)]


class ClusterParams(C.Structure):
    _fields_ = [("n", C.c_int64), ("target_nnz", C.c_int64), ("block_extent", C.c_int64), ("tile", C.c_int64),
                ("fill", C.c_double), ("block_occupancy", C.c_double), ("tile_min", C.c_int64),
                ("tile_max", C.c_int64), ("diag_spread", C.c_double), ("dominance", C.c_double),
                ("seed", C.c_uint64), ("threads", C.c_int)]


class OpInfo(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64), ("ntiles", C.c_int64),
                ("device_bytes", C.c_int64), ("bytes_per_nnz_x1000", C.c_int64), ("values_prec", C.c_int),
                ("tile_rows", C.c_int), ("tile_cols", C.c_int), ("tile_max_nnz", C.c_int)]


class SolverConfig(C.Structure):
    _fields_ = [("k", C.c_int), ("nb", C.c_int), ("tol", C.c_double), ("maxiter", C.c_int),
                ("fom_iterations", C.c_int), ("seed", C.c_uint64), ("observer_state", C.c_int)]


class ResultInfo(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("k", C.c_int), ("nb", C.c_int), ("n", C.c_int64),
                ("operator_calls", C.c_int64), ("precond_fallbacks", C.c_int64), ("restarts", C.c_int)]


OBSERVER_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_int64, C.c_int, C.POINTER(C.c_double),
                          C.POINTER(C.c_double), C.c_int, *([C.POINTER(C.c_double)] * 6))
HOST_OP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64, C.c_int)

_lib = None


def lib():
    """Load libblockeig_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(f"{LIB_PATH} is missing: run __graft_entry__.build() first")
        _lib = C.CDLL(str(LIB_PATH))
        _lib.be_last_error.restype = C.c_char_p
        _lib.be_version.restype = C.c_char_p
        _lib.be_free_buffer.restype = None
        _lib.be_csb_free.restype = None
        _lib.be_synth_free.restype = None
        if hasattr(_lib, "be_result_free"):
            _lib.be_result_free.restype = None
    return _lib


def check(status: int):
    if status != 0:
        msg = lib().be_last_error().decode(errors="replace")
        cls = _BY_CODE.get(status, BlockeigError)
        e = cls(msg)
        if status == 9:
            e.pivot = lib().be_last_error_pivot()
        raise e


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else C.c_void_p(0)


# --------------------------------------------------------------------------- CSB
class Csb:
    """CsbCooMatrix (csb.hpp:39-63) as numpy arrays. Either owned by the
    library (handle) or a plain set of arrays supplied by the caller."""

    def __init__(self, nrows, ncols, row_offsets, col_offsets, block_nnz, block_nnz_offsets, local_rows,
                 local_cols, values, handle=None):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.int64)
        self.col_offsets = np.ascontiguousarray(col_offsets, dtype=np.int64)
        self.block_nnz = np.ascontiguousarray(block_nnz, dtype=np.int64)
        self.block_nnz_offsets = np.ascontiguousarray(block_nnz_offsets, dtype=np.int64)
        self.local_rows = np.ascontiguousarray(local_rows, dtype=np.uint16)
        self.local_cols = np.ascontiguousarray(local_cols, dtype=np.uint16)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self._handle = handle

    @property
    def nrowblks(self):
        return len(self.row_offsets) - 1

    @property
    def ncolblks(self):
        return len(self.col_offsets) - 1

    @property
    def nnz(self):
        return len(self.values)

    def view(self) -> CsbView:
        return CsbView(self.nrows, self.ncols, self.nrowblks, self.ncolblks, self.nnz, _p(self.row_offsets),
                       _p(self.col_offsets), _p(self.block_nnz), _p(self.block_nnz_offsets), _p(self.local_rows),
                       _p(self.local_cols), _p(self.values))

    @classmethod
    def _from_handle(cls, h):
        v = CsbView()
        check(lib().be_csb_view_get(h, C.byref(v)))

        def arr(ptr, n, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            buf = (C.c_char * (n * np.dtype(dt).itemsize)).from_address(ptr)
            return np.frombuffer(buf, dtype=dt, count=n)

        nb = v.nrowblks * v.ncolblks
        obj = cls(v.nrows, v.ncols, arr(v.row_offsets, v.nrowblks + 1, np.int64),
                  arr(v.col_offsets, v.ncolblks + 1, np.int64), arr(v.block_nnz, nb, np.int64),
                  arr(v.block_nnz_offsets, nb, np.int64), arr(v.local_rows, v.nnz, np.uint16),
                  arr(v.local_cols, v.nnz, np.uint16), arr(v.values, v.nnz, np.float64), handle=h)
        return obj

    def __del__(self):
        if self._handle is not None and _lib is not None:
            _lib.be_csb_free(self._handle)
            self._handle = None

    def block_row_nnz(self) -> np.ndarray:
        """Stored nonzeros per CSB block row (the SpMM slab weights)."""
        return self.block_nnz.reshape(self.nrowblks, self.ncolblks).sum(axis=1)

    def slab(self, b0: int, b1: int) -> "Csb":
        """Block rows [b0, b1) of this matrix as a CSB of the same global shape
        and blocks (entries elsewhere absent); zero-copy slices of the arrays."""
        nb = self.ncolblks
        bn = self.block_nnz.reshape(self.nrowblks, nb).copy()
        bn[:b0] = 0
        bn[b1:] = 0
        lo = int(self.block_nnz_offsets[b0 * nb]) if b0 < self.nrowblks else self.nnz
        hi = int(self.block_nnz_offsets[b1 * nb]) if b1 < self.nrowblks else self.nnz
        off = np.zeros(bn.size, np.int64)
        np.cumsum(bn.ravel()[:-1], out=off[1:])
        sl = Csb(self.nrows, self.ncols, self.row_offsets, self.col_offsets, bn.ravel(), off,
                 self.local_rows[lo:hi], self.local_cols[lo:hi], self.values[lo:hi])
        sl._parent = self  # keeps a library-owned parent alive
        return sl

    def block_weights(self) -> np.ndarray:
        """Stored nonzeros per CSB block, (nrowblks, ncolblks) (the 2-D tile weights)."""
        return self.block_nnz.reshape(self.nrowblks, self.ncolblks).copy()

    def rect(self, r0: int, r1: int, c0: int, c1: int) -> "Csb":
        """The blocks (bi, bj) with r0 <= bi < r1 and c0 <= bj < c1 (one rank's 2-D tile) as a CSB
        of the same global shape and blocks (entries elsewhere absent)."""
        nb = self.ncolblks
        bn = self.block_nnz.reshape(self.nrowblks, nb)
        keep = np.zeros_like(bn)
        keep[r0:r1, c0:c1] = bn[r0:r1, c0:c1]
        parts = []
        for bi in range(r0, r1):
            if c1 > c0:
                lo = int(self.block_nnz_offsets[bi * nb + c0])
                hi = lo + int(bn[bi, c0:c1].sum())
                if hi > lo:
                    parts.append(np.arange(lo, hi))
        idx = np.concatenate(parts) if parts else np.zeros(0, np.int64)
        off = np.zeros(keep.size, np.int64)
        np.cumsum(keep.ravel()[:-1], out=off[1:])
        return Csb(self.nrows, self.ncols, self.row_offsets, self.col_offsets, keep.ravel(), off,
                   self.local_rows[idx], self.local_cols[idx], self.values[idx])

    def to_triples(self) -> np.ndarray:
        out = np.zeros(self.nnz, dtype=TRIPLE_DTYPE)
        v = self.view()
        check(lib().be_csb_to_triples(C.byref(v), _p(out)))
        return out

    def is_strictly_lower(self) -> bool:
        r = C.c_int(0)
        v = self.view()
        check(lib().be_csb_is_strictly_lower(C.byref(v), C.byref(r)))
        return bool(r.value)

    def save(self, path, diag=None):
        v = self.view()
        d = None if diag is None else np.ascontiguousarray(diag, dtype=np.float64)
        check(lib().be_csb_save(str(path).encode(), C.byref(v), _p(d), C.c_int64(0 if d is None else len(d))))

    @classmethod
    def load_rows(cls, path, brow_begin: int, brow_end: int):
        """Block rows [brow_begin, brow_end) of a CSB1 cache: (csb, diag of those rows or None)."""
        h = C.c_void_p()
        dp = C.POINTER(C.c_double)()
        nd = C.c_int64(0)
        check(lib().be_csb_load_rows(str(path).encode(), C.c_int64(brow_begin), C.c_int64(brow_end), C.byref(h),
                                     C.byref(dp), C.byref(nd)))
        m = cls._from_handle(h)
        diag = None
        if nd.value > 0:
            diag = np.ctypeslib.as_array(dp, shape=(nd.value,)).copy()
            lib().be_free_buffer(dp)
        return m, diag

    @classmethod
    def load(cls, path):
        h = C.c_void_p()
        dp = C.POINTER(C.c_double)()
        nd = C.c_int64(0)
        check(lib().be_csb_load(str(path).encode(), C.byref(h), C.byref(dp), C.byref(nd)))
        m = cls._from_handle(h)
        diag = None
        if nd.value > 0:
            diag = np.ctypeslib.as_array(dp, shape=(nd.value,)).copy()
            lib().be_free_buffer(dp)
        return m, diag


def _mm_result(call):
    n = C.c_int64(0)
    nl = C.c_int64(0)
    lp = C.c_void_p()
    dp = C.POINTER(C.c_double)()
    check(call(C.byref(n), C.byref(lp), C.byref(nl), C.byref(dp)))
    try:
        lower = np.frombuffer((C.c_char * (24 * nl.value)).from_address(lp.value), dtype=TRIPLE_DTYPE).copy() \
            if nl.value else np.zeros(0, dtype=TRIPLE_DTYPE)
        diag = np.ctypeslib.as_array(dp, shape=(n.value,)).copy()
    finally:
        lib().be_free_buffer(lp)
        lib().be_free_buffer(dp)
    return n.value, lower, diag


def read_matrix_market(path=None, text=None):
    """ingest_matrix_market(_file) (matrix_market.hpp:38-94): (n, strictly-lower triples in file
    order, dense diagonal). Raises ParseError / NotSymmetricHeader / DuplicateEntry like the reference."""
    if (path is None) == (text is None):
        raise ValueError("give exactly one of path / text")
    if path is not None:
        return _mm_result(lambda *a: lib().be_mm_read_file(str(path).encode(), *a))
    b = text.encode() if isinstance(text, str) else bytes(text)
    return _mm_result(lambda *a: lib().be_mm_parse(b, C.c_int64(len(b)), *a))


def write_matrix_market(n: int, lower: np.ndarray, diag) -> str:
    """write_matrix_market (matrix_market.hpp:98-113)."""
    t = np.ascontiguousarray(lower, dtype=TRIPLE_DTYPE)
    d = np.ascontiguousarray(diag, dtype=np.float64)
    if d.shape != (n,):
        raise ValueError("diag must have n entries")
    tp = C.c_void_p()
    ln = C.c_int64(0)
    check(lib().be_mm_write(C.c_int64(n), _p(t) if len(t) else None, C.c_int64(len(t)), _p(d), C.byref(tp),
                            C.byref(ln)))
    try:
        return C.string_at(tp.value, ln.value).decode()
    finally:
        lib().be_free_buffer(tp)


def as_triples(rows, cols, values) -> np.ndarray:
    t = np.zeros(len(rows), dtype=TRIPLE_DTYPE)
    t["row"], t["col"], t["value"] = rows, cols, values
    return t


def random_block(n: int, nb: int, seed: int, row_lo: int = 0) -> np.ndarray:
    """random_block (block_vector.hpp:47-53): rows [row_lo, row_lo + n) of the
    reference's mt19937_64 U(-1, 1) block -- the solver's X0."""
    out = np.zeros((n, nb))
    check(lib().be_random_block(C.c_int64(n), C.c_int64(nb), C.c_uint64(seed), C.c_int64(row_lo), _p(out)))
    return out


def uniform_boundaries(n: int, extent: int) -> np.ndarray:
    cnt = C.c_int64(0)
    check(lib().be_uniform_boundaries(C.c_int64(n), C.c_int64(extent), None, C.byref(cnt)))
    out = np.zeros(cnt.value, dtype=np.int64)
    check(lib().be_uniform_boundaries(C.c_int64(n), C.c_int64(extent), _p(out), C.byref(cnt)))
    return out


def build_csb_coo(triples: np.ndarray, nrows: int, ncols: int, row_bounds, col_bounds) -> Csb:
    """build_csb_coo (csb.hpp:100-161)."""
    t = np.ascontiguousarray(triples, dtype=TRIPLE_DTYPE)
    rb = np.ascontiguousarray(row_bounds, dtype=np.int64)
    cb = np.ascontiguousarray(col_bounds, dtype=np.int64)
    h = C.c_void_p()
    check(lib().be_csb_build(_p(t), C.c_int64(len(t)), C.c_int64(nrows), C.c_int64(ncols), _p(rb),
                             C.c_int64(len(rb)), _p(cb), C.c_int64(len(cb)), C.byref(h)))
    return Csb._from_handle(h)


# --------------------------------------------------------------------- generators
class Synthetic:
    """generate_synthetic (synth.hpp:92-158) output."""

    def __init__(self, kind="random", n=1000, density=0.02, bandwidth=8, block_extent=4000, tile_min=4,
                 tile_max=512, diag_spread=5.0, dominance=1.0, seed=1):
        p = SynthParams(SYNTH_KINDS[kind], n, density, bandwidth, block_extent, tile_min, tile_max, diag_spread,
                        dominance, seed)
        self._h = C.c_void_p()
        check(lib().be_generate_synthetic(C.byref(p), C.byref(self._h)))
        low, nlow = C.c_void_p(), C.c_int64()
        diag, toff, ntoff = C.c_void_p(), C.c_void_p(), C.c_int64()
        check(lib().be_synth_get(self._h, C.byref(low), C.byref(nlow), C.byref(diag), C.byref(toff), C.byref(ntoff)))
        self.n = n
        self.lower = np.frombuffer((C.c_char * (24 * nlow.value)).from_address(low.value), dtype=TRIPLE_DTYPE).copy() \
            if nlow.value else np.zeros(0, dtype=TRIPLE_DTYPE)
        self.diag = np.frombuffer((C.c_char * (8 * n)).from_address(diag.value), dtype=np.float64).copy()
        self.tile_offsets = np.frombuffer((C.c_char * (8 * ntoff.value)).from_address(toff.value),
                                          dtype=np.int64).copy()
        lib().be_synth_free(self._h)
        self._h = None


def generate_clustered(n, target_nnz, block_extent=4000, tile=128, fill=0.10, block_occupancy=1.0, tile_min=4,
                       tile_max=512, diag_spread=5.0, dominance=1.0, seed=1, threads=0):
    """Clustered CSB generator (tooling for the Test-1..3 shapes)."""
    p = ClusterParams(n, target_nnz, block_extent, tile, fill, block_occupancy, tile_min, tile_max, diag_spread,
                      dominance, seed, threads)
    h = C.c_void_p()
    dp = C.POINTER(C.c_double)()
    tp = C.POINTER(C.c_int64)()
    nt = C.c_int64()
    check(lib().be_generate_clustered(C.byref(p), C.byref(h), C.byref(dp), C.byref(tp), C.byref(nt)))
    diag = np.ctypeslib.as_array(dp, shape=(n,)).copy()
    toff = np.ctypeslib.as_array(tp, shape=(nt.value,)).copy()
    lib().be_free_buffer(dp)
    lib().be_free_buffer(tp)
    return Csb._from_handle(h), diag, toff


def clustered_params(n, target_nnz, block_extent=4000, tile=128, fill=0.10, block_occupancy=1.0, tile_min=4,
                     tile_max=512, diag_spread=5.0, dominance=1.0, seed=1, threads=0):
    return ClusterParams(n, target_nnz, block_extent, tile, fill, block_occupancy, tile_min, tile_max, diag_spread,
                         dominance, seed, threads)


def generate_clustered_part(params: ClusterParams, brow_begin: int, brow_end: int, diag_blocks_only=False):
    """Block rows [brow_begin, brow_end) of the clustered matrix (global shape):
    (csb, rowabs contribution over all n rows, tile offsets)."""
    h = C.c_void_p()
    rp = C.POINTER(C.c_double)()
    tp = C.POINTER(C.c_int64)()
    nt = C.c_int64()
    check(lib().be_generate_clustered_part(C.byref(params), C.c_int64(brow_begin), C.c_int64(brow_end),
                                           C.c_int(1 if diag_blocks_only else 0), C.byref(h), C.byref(rp),
                                           C.byref(tp), C.byref(nt)))
    rowabs = np.ctypeslib.as_array(rp, shape=(params.n,)).copy()
    toff = np.ctypeslib.as_array(tp, shape=(nt.value,)).copy()
    lib().be_free_buffer(rp)
    lib().be_free_buffer(tp)
    return Csb._from_handle(h), rowabs, toff


def generate_clustered_tile(params: ClusterParams, rows, cols):
    """One 2-D tile of the clustered matrix: block rows [rows[0], rows[1]) x block columns
    [cols[0], cols[1]) (global shape; exactly the whole-matrix generator's entries there):
    (csb, rowabs contribution over all n rows, tile offsets)."""
    h = C.c_void_p()
    rp = C.POINTER(C.c_double)()
    tp = C.POINTER(C.c_int64)()
    nt = C.c_int64()
    check(lib().be_generate_clustered_tile(C.byref(params), C.c_int64(rows[0]), C.c_int64(rows[1]),
                                           C.c_int64(cols[0]), C.c_int64(cols[1]), C.byref(h), C.byref(rp),
                                           C.byref(tp), C.byref(nt)))
    rowabs = np.ctypeslib.as_array(rp, shape=(params.n,)).copy()
    toff = np.ctypeslib.as_array(tp, shape=(nt.value,)).copy()
    lib().be_free_buffer(rp)
    lib().be_free_buffer(tp)
    return Csb._from_handle(h), rowabs, toff


def clustered_block_weights(params: ClusterParams) -> np.ndarray:
    """Expected stored entries of every lower block, (nblk, nblk) (the 2-D tile weights)."""
    nb = C.c_int64()
    check(lib().be_clustered_block_weights(C.byref(params), None, C.byref(nb)))
    w = np.zeros(nb.value * nb.value, np.int64)
    check(lib().be_clustered_block_weights(C.byref(params), _p(w), C.byref(nb)))
    return w.reshape(nb.value, nb.value)


def clustered_diag(params: ClusterParams, rowabs, row_begin: int, row_end: int) -> np.ndarray:
    r = np.ascontiguousarray(rowabs, dtype=np.float64)
    out = np.zeros(row_end - row_begin)
    check(lib().be_clustered_diag(C.byref(params), _p(r), C.c_int64(row_begin), C.c_int64(row_end), _p(out)))
    return out


def clustered_weights(params: ClusterParams) -> np.ndarray:
    nb = C.c_int64()
    check(lib().be_clustered_weights(C.byref(params), None, C.byref(nb)))
    w = np.zeros(nb.value, np.int64)
    check(lib().be_clustered_weights(C.byref(params), _p(w), C.byref(nb)))
    return w


# ------------------------------------------------------------------------ device
class Context:
    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        check(lib().be_ctx_create(C.c_int(device), C.byref(self._h)))

    @property
    def handle(self):
        return self._h

    def stream(self) -> int:
        s = C.c_void_p()
        check(lib().be_ctx_stream(self._h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        check(lib().be_ctx_synchronize(self._h))

    def launches(self) -> int:
        n = C.c_int64()
        check(lib().be_ctx_launches(self._h, C.byref(n)))
        return n.value

    def close(self):
        if self._h:
            check(lib().be_ctx_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Operator:
    """SymmetricOperator (kernels.hpp:339-378) backed by the device tile format."""

    def __init__(self, ctx: Context, csb: Csb, diag=None, values_prec=BE_F32, symmetric=True, deterministic=False,
                 fmt=None):
        self.ctx = ctx
        self._csb = csb  # the view's arrays must outlive creation only
        self._h = C.c_void_p()
        d = None if diag is None else np.ascontiguousarray(diag, dtype=np.float64)
        v = csb.view()
        check(lib().be_op_create(ctx.handle, C.byref(v), _p(d), C.c_int(values_prec),
                                 C.c_int((BE_OP_SYMMETRIC if symmetric else 0) | (BE_OP_DETERMINISTIC if deterministic else 0)
                                         | {None: 0, "tiles": BE_OP_FORMAT_TILES, "rows": BE_OP_FORMAT_ROWS}[fmt]),
                                 C.byref(self._h)))
        self._csb = None

    @classmethod
    def from_csb1(cls, ctx: Context, path, values_prec=BE_F32, batch_entries=0):
        """The symmetric tile-format operator streamed from a CSB1 cache file (be_op_create_csb1):
        (operator, diagonal)."""
        op = cls.__new__(cls)
        op.ctx = ctx
        op._csb = None
        op._h = C.c_void_p()
        dp = C.POINTER(C.c_double)()
        nd = C.c_int64(0)
        check(lib().be_op_create_csb1(ctx.handle, str(path).encode(), C.c_int(values_prec), C.c_int(BE_OP_SYMMETRIC),
                                      C.c_int64(batch_entries), C.byref(dp), C.byref(nd), C.byref(op._h)))
        diag = np.ctypeslib.as_array(dp, shape=(nd.value,)).copy() if nd.value > 0 else np.zeros(0)
        lib().be_free_buffer(dp)
        return op, diag

    @property
    def handle(self):
        return self._h

    def info(self) -> OpInfo:
        i = OpInfo()
        check(lib().be_op_get_info(self._h, C.byref(i)))
        return i

    def apply_host(self, x: np.ndarray, y: np.ndarray | None = None, mode=BE_APPLY_SYMMETRIC) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        info = self.info()
        out_rows = info.ncols if mode == BE_APPLY_TRANS_ACC else info.nrows
        if y is None:
            y = np.zeros((out_rows, x.shape[1]), dtype=np.float64)
        assert y.flags.c_contiguous and y.dtype == np.float64
        check(lib().be_op_apply_host(self._h, _p(x), _p(y), C.c_int64(x.shape[0]), C.c_int(x.shape[1]),
                                     C.c_int(mode)))
        return y

    def apply_dev(self, x_ptr: int, y_ptr: int, nrows: int, nb: int, panel_prec=BE_F64, mode=BE_APPLY_SYMMETRIC,
                  stream: int = 0):
        check(lib().be_op_apply(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), C.c_int64(nrows), C.c_int(nb),
                                C.c_int(panel_prec), C.c_int(mode), C.c_void_p(stream)))

    def decode(self):
        n = self.info().nnz
        rows = np.zeros(n, np.int64)
        cols = np.zeros(n, np.int64)
        vals = np.zeros(n, np.float64)
        idx = np.zeros(n, np.int64)
        check(lib().be_op_decode(self._h, _p(rows), _p(cols), _p(vals), _p(idx)))
        return rows, cols, vals, idx

    def timing(self, enable: int = -1):
        k, a = C.c_double(), C.c_double()
        check(lib().be_op_timing(self._h, C.c_int(enable), C.byref(k), C.byref(a)))
        return k.value, a.value

    def close(self):
        if self._h:
            check(lib().be_op_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dist_rows(bounds, world: int) -> np.ndarray:
    """Panel-row ownership cuts (world + 1) on the block boundaries."""
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    out = np.zeros(world + 1, np.int64)
    check(lib().be_dist_rows(_p(b), C.c_int64(len(b)), C.c_int(world), _p(out)))
    return out


def dist_touched(slab: "Csb", cuts, world: int, owner=None) -> np.ndarray:
    """The segment-wise exchange rule (be_dist_touched): touched[r] = 1 when the slab's stored
    blocks have rows or columns in the panel segment owned by rank r."""
    c = np.ascontiguousarray(cuts, dtype=np.int64)
    o = None if owner is None else np.ascontiguousarray(owner, dtype=np.int32)
    out = np.zeros(world, np.uint8)
    v = slab.view()
    check(lib().be_dist_touched(C.byref(v), _p(c), _p(o), C.c_int(world), _p(out)))
    return out.astype(bool)


def dist_balance(weights, world: int) -> np.ndarray:
    """Contiguous weight-balanced item cuts (world + 1)."""
    w = np.ascontiguousarray(weights, dtype=np.int64)
    out = np.zeros(world + 1, np.int64)
    check(lib().be_dist_balance(_p(w), C.c_int64(len(w)), C.c_int(world), _p(out)))
    return out


def dist_tiles2d(block_weights, bounds, world: int) -> np.ndarray:
    """nnz-balanced 2-D tiles (be_dist_tiles2d): (world, 4) rectangles (r0, r1, c0, c1) of CSB
    blocks, rank r owning the stored blocks r0 <= bi < r1, c0 <= bj < c1."""
    w = np.ascontiguousarray(block_weights, dtype=np.int64)
    nblk = w.shape[0]
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    if w.shape != (nblk, nblk) or len(b) != nblk + 1:
        raise DimensionMismatch("dist_tiles2d: weights must be (nblk, nblk) with nblk + 1 bounds")
    out = np.zeros((world, 4), np.int64)
    check(lib().be_dist_tiles2d(_p(w), C.c_int64(nblk), _p(b), C.c_int(world), _p(out)))
    return out


class CommGroup:
    """In-process rank group (ranks are host threads; any GPUs, several ranks per GPU allowed)."""

    def __init__(self, world: int):
        self._h = C.c_void_p()
        check(lib().be_comm_group_create(C.c_int(world), C.byref(self._h)))
        self.world = world

    def abort(self):
        """Release ranks blocked in a collective (ProtocolDeadlock): call from a failing rank."""
        if self._h:
            check(lib().be_comm_group_abort(self._h))

    def close(self):
        if self._h:
            check(lib().be_comm_group_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _nccl_hint():
    """Point the library at the NCCL torch bundles (unless one is loaded or set):
    the process must not mix two libnccl.so.2 builds under one soname."""
    import os
    if "BE_NCCL_LIB" in os.environ:
        return
    try:
        import nvidia.nccl as n
        p = Path(list(n.__path__)[0]) / "lib" / "libnccl.so.2"
        if p.exists():
            os.environ["BE_NCCL_LIB"] = str(p)
    except Exception:
        pass


def nccl_unique_id() -> bytes:
    _nccl_hint()
    buf = (C.c_uint8 * 128)()
    check(lib().be_comm_nccl_id(buf))
    return bytes(buf)


class Comm:
    """A rank's communicator: NCCL (one process per GPU) or local (threads of one process)."""

    def __init__(self, ctx: Context, *, nccl_id: bytes | None = None, rank: int = 0, world: int = 1,
                 group: CommGroup | None = None):
        self.ctx = ctx
        self._h = C.c_void_p()
        if group is not None:
            self._group = group
            check(lib().be_comm_create_local(ctx.handle, group._h, C.c_int(rank), C.byref(self._h)))
        else:
            _nccl_hint()
            if nccl_id is None or len(nccl_id) != 128:
                raise BadParams("Comm: NCCL needs the 128-byte unique id")
            buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            check(lib().be_comm_create_nccl(ctx.handle, buf, C.c_int(rank), C.c_int(world), C.byref(self._h)))

    @property
    def handle(self):
        return self._h

    def info(self):
        r, w, b, c, n = C.c_int(), C.c_int(), C.c_int(), C.c_int64(), C.c_int64()
        check(lib().be_comm_info(self._h, C.byref(r), C.byref(w), C.byref(b), C.byref(c), C.byref(n)))
        return {"rank": r.value, "world": w.value, "backend": "nccl" if b.value == 0 else "local",
                "calls": c.value, "bytes": n.value}

    def allreduce_dev(self, ptr: int, count: int, stream: int = 0):
        check(lib().be_comm_allreduce_f64(self._h, C.c_void_p(ptr), C.c_int64(count), C.c_void_p(stream)))

    def close(self):
        if self._h:
            check(lib().be_comm_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistOperator(Operator):
    """Distributed symmetric operator over the ranks of `comm` (dist.hpp
    distributed_operator): this rank's CSB slab, panel-row cuts, local diagonal.
    owner[q] = rank owning segment q (default: segment q is rank q's)."""

    def __init__(self, ctx: Context, comm: Comm, slab: Csb, cuts, diag_local, values_prec=BE_F32, owner=None):
        self.ctx = ctx
        self.comm = comm
        self.cuts = np.ascontiguousarray(cuts, dtype=np.int64)
        self._h = C.c_void_p()
        d = np.ascontiguousarray(diag_local, dtype=np.float64)
        v = slab.view()
        if owner is None:
            check(lib().be_op_create_dist(ctx.handle, comm.handle, C.byref(v), _p(self.cuts), _p(d),
                                          C.c_int(values_prec), C.byref(self._h)))
        else:
            o = np.ascontiguousarray(owner, dtype=np.int32)
            check(lib().be_op_create_dist_owned(ctx.handle, comm.handle, C.byref(v), _p(self.cuts), _p(o), _p(d),
                                                C.c_int(values_prec), C.byref(self._h)))

    def need(self) -> np.ndarray:
        """world x world: row p = the padded slots rank p's tiles touch (be_op_dist_need)."""
        w = len(self.cuts) - 1
        out = np.zeros((w, w), np.uint8)
        check(lib().be_op_dist_need(self._h, _p(out)))
        return out.astype(bool)


# ---------------------------------------------- the reference triangular layout
def tri_layout(nd: int):
    """build_layout (dist.hpp:49-75): (blocks[n_ranks, 3] = (i, j, transposed), diagonal_ranks[nd])."""
    nr = C.c_int()
    check(lib().be_tri_layout(C.c_int(nd), None, None, C.byref(nr)))
    blocks = np.zeros((nr.value, 3), np.int32)
    dr = np.zeros(max(nd, 1), np.int32)
    check(lib().be_tri_layout(C.c_int(nd), _p(blocks), _p(dr), C.byref(nr)))
    return blocks, dr[:nd]


def tri_segments(nd: int, sub_bounds):
    """segment_of_rank (dist.hpp:184-196): (begin[n_ranks], end[n_ranks])."""
    b = np.ascontiguousarray(sub_bounds, dtype=np.int64)
    nr = nd * (nd + 1) // 2
    beg, end = np.zeros(nr, np.int64), np.zeros(nr, np.int64)
    check(lib().be_tri_segments(C.c_int(nd), _p(b), _p(beg), _p(end)))
    return beg, end


def tri_rank_triples(csb: Csb, nd: int, sub_bounds, rank: int) -> np.ndarray:
    """partition_matrix's routing: rank's stored entries in global coordinates."""
    b = np.ascontiguousarray(sub_bounds, dtype=np.int64)
    v = csb.view()
    cnt = C.c_int64(0)
    check(lib().be_tri_rank_triples(C.byref(v), C.c_int(nd), _p(b), C.c_int(rank), None, C.byref(cnt)))
    out = np.zeros(cnt.value, dtype=TRIPLE_DTYPE)
    check(lib().be_tri_rank_triples(C.byref(v), C.c_int(nd), _p(b), C.c_int(rank), _p(out), C.byref(cnt)))
    return out


def tri_rank_problem(csb: Csb, diag, nd: int, sub_bounds, rank: int, extent: int = 4000):
    """One rank of the reference's triangular layout as a distributed-operator
    input: (slab CSB over blocks refined at every segment cut, segment bounds in
    row order, segment owners, this rank's diagonal)."""
    n = csb.nrows
    beg, end = tri_segments(nd, sub_bounds)
    order = np.lexsort((end, beg)).astype(np.int32)
    seg_bounds = np.concatenate([beg[order], [n]]).astype(np.int64)
    cut = np.unique(np.concatenate([np.asarray(sub_bounds, np.int64), seg_bounds]))
    bounds = [0]
    for a, b in zip(cut[:-1], cut[1:]):
        k = -(-(b - a) // extent)
        bounds += [a + (b - a) * q // k for q in range(1, k + 1)]
    bounds = np.asarray(bounds, np.int64)
    t = tri_rank_triples(csb, nd, sub_bounds, rank)
    slab = build_csb_coo(t, n, n, bounds, bounds)
    d = np.asarray(diag)[beg[rank]:end[rank]]
    return slab, seg_bounds, order, d


class Tiles:
    """DiagonalTileSet (precond.hpp:34-48) built by extract_tiles (precond.hpp:63-127), uploaded.
    row_range=(lo, hi): only the tiles of rows [lo, hi) (one rank's rows), diag = those rows."""

    def __init__(self, ctx: Context, csb: Csb, diag, tile_offsets, row_range=None):
        self.ctx = ctx
        self._h = C.c_void_p()
        d = np.ascontiguousarray(diag, dtype=np.float64)
        t = np.ascontiguousarray(tile_offsets, dtype=np.int64)
        v = csb.view()
        if row_range is None:
            check(lib().be_tiles_create(ctx.handle, C.byref(v), _p(d), _p(t), C.c_int64(len(t)), C.byref(self._h)))
        else:
            check(lib().be_tiles_create_range(ctx.handle, C.byref(v), _p(d), _p(t), C.c_int64(len(t)),
                                              C.c_int64(row_range[0]), C.c_int64(row_range[1]), C.byref(self._h)))

    @property
    def handle(self):
        return self._h

    def count(self):
        """(number of tiles, operator dimension, total stored tile entries)"""
        c, d, e = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().be_tiles_count(self._h, C.byref(c), C.byref(d), C.byref(e)))
        return c.value, d.value, e.value

    def tile(self, j):
        """SparseTile j in the reference layout: (dim, rows, cols, values, diag_pos)."""
        dim, ne = C.c_int64(), C.c_int64()
        check(lib().be_tiles_get(self._h, C.c_int64(j), C.byref(dim), C.byref(ne), None, None, None, None))
        rows = np.zeros(ne.value, np.int32)
        cols = np.zeros(ne.value, np.int32)
        vals = np.zeros(ne.value)
        dpos = np.zeros(dim.value, np.int64)
        check(lib().be_tiles_get(self._h, C.c_int64(j), C.byref(dim), C.byref(ne), _p(rows), _p(cols), _p(vals),
                                 _p(dpos)))
        return dim.value, rows, cols, vals, dpos

    def apply_host(self, shifts, r, m=4):
        """apply_preconditioner (precond.hpp:287-317): returns (W, fallbacks)."""
        r = np.ascontiguousarray(r, dtype=np.float64)
        sh = np.ascontiguousarray(shifts, dtype=np.float64)
        w = np.zeros_like(r)
        fb = C.c_int64(0)
        check(lib().be_precond_apply_host(self._h, _p(sh), _p(r), _p(w), C.c_int64(r.shape[0]), C.c_int(r.shape[1]),
                                          C.c_int(m), C.byref(fb)))
        return w, fb.value

    def close(self):
        if self._h:
            check(lib().be_tiles_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def host_array(shape) -> np.ndarray:
    """An uninitialised float64 host array for device -> host results, backed by an anonymous
    mapping advised for transparent huge pages (a large result then faults in 2 MB pages instead
    of 4 KB ones while the copy lands)."""
    count = int(np.prod(shape))
    nbytes = max(count * 8, 8)
    if nbytes < (8 << 20):
        return np.empty(shape)
    mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    if hasattr(mm, "madvise") and hasattr(mmap, "MADV_HUGEPAGE"):
        try:
            mm.madvise(mmap.MADV_HUGEPAGE)
        except OSError:
            pass
    return np.frombuffer(mm, dtype=np.float64, count=count).reshape(shape)


def _x0_checked(x0, n, k, nb):
    """X0 must be n x nb (nb = k + 3 when 0), as lobpcg_solve checks
    (lobpcg.hpp:308-310): the C side reads n*nb doubles from the pointer."""
    if x0 is None:
        return None
    x0a = np.ascontiguousarray(x0, dtype=np.float64)
    nb_eff = nb or k + 3
    if x0a.ndim != 2 or x0a.shape != (int(n), int(nb_eff)):
        raise DimensionMismatch(f"lobpcg_solve: X0 must be n x nb ({n} x {nb_eff}), got {x0a.shape}")
    return x0a


def lobpcg(ctx: Context, op=None, n=None, tiles: Tiles | None = None, x0=None, k=5, nb=0, tol=1e-6, maxiter=500,
           fom_iterations=4, seed=1234, observer=None, observer_state=False, host_operator=None,
           observer_panels=False):
    """lobpcg_solve (lobpcg.hpp:291-456) on the device. `op` is an Operator;
    `host_operator(x) -> y` is the generic Operator closure (lobpcg.hpp:20).
    observer(iter, theta, residual_norms, n_converged, x, hx), or with
    observer_panels=True observer(iter, theta, residual_norms, n_converged, state)
    where state holds the six SolverState panels x, hx, w, hw, p, hp."""
    if n is None:
        n = op.info().nrows
    cfg = SolverConfig(k, nb, tol, maxiter, fom_iterations, seed, 1 if (observer_state or observer_panels) else 0)
    x0a = _x0_checked(x0, n, k, nb)
    obs_cb = OBSERVER_FN()
    if observer is not None:
        def _obs(user, it, nn, nbb, th, rn, nc, x, hx, w, hw, p, hp):
            thv = np.ctypeslib.as_array(th, shape=(nbb,)).copy()
            rnv = np.ctypeslib.as_array(rn, shape=(nbb,)).copy()
            pan = [np.ctypeslib.as_array(a, shape=(nn, nbb)).copy() if a else None for a in (x, hx, w, hw, p, hp)]
            if observer_panels:  # the whole SolverState (lobpcg.hpp:52-58)
                observer(it, thv, rnv, nc, dict(zip(("x", "hx", "w", "hw", "p", "hp"), pan)))
            else:
                observer(it, thv, rnv, nc, pan[0], pan[1])
        obs_cb = OBSERVER_FN(_obs)
    hop_cb = HOST_OP_FN()
    if host_operator is not None:
        def _hop(user, inp, out, nn, nbb):
            try:
                xi = np.ctypeslib.as_array(inp, shape=(nn, nbb))
                yo = np.ctypeslib.as_array(out, shape=(nn, nbb))
                yo[:] = host_operator(xi)
                return 0
            except Exception:
                return 1
        hop_cb = HOST_OP_FN(_hop)
    h = C.c_void_p()
    t0 = time.perf_counter()
    check(lib().be_lobpcg_solve(ctx.handle, op.handle if op is not None else None, hop_cb, None, C.c_int64(n),
                                tiles.handle if tiles is not None else None, _p(x0a), C.byref(cfg), obs_cb, None,
                                C.byref(h)))
    try:
        t1 = time.perf_counter()
        info = ResultInfo()
        check(lib().be_result_get_info(h, C.byref(info)))
        lam = np.zeros(info.k)
        x = host_array((info.n, info.k))
        check(lib().be_result_get(h, _p(lam), _p(x)))
        if _os.environ.get("BE_TRACE_SEGMENTS"):
            print(f"[be] host: solve call {1e3 * (t1 - t0):.1f} ms, eigenvector read {1e3 * (time.perf_counter() - t1):.1f} ms",
                  file=sys.stderr, flush=True)
            t1 = time.perf_counter()
        nbb = info.nb
        th = np.zeros((info.iterations, nbb))
        rs = np.zeros((info.iterations, nbb))
        nc = np.zeros(info.iterations, np.int32)
        times = np.zeros((info.iterations, 4))
        for i in range(info.iterations):
            c_nc = C.c_int()
            t = [C.c_double() for _ in range(4)]
            row_t = np.zeros(nbb)
            row_r = np.zeros(nbb)
            check(lib().be_result_get_record(h, C.c_int(i), _p(row_t), _p(row_r), C.byref(c_nc), *[C.byref(v) for v in t]))
            th[i], rs[i], nc[i] = row_t, row_r, c_nc.value
            times[i] = [v.value for v in t]
        return dict(lambda_=lam, x=x, converged=bool(info.converged), iterations=info.iterations,
                    operator_calls=info.operator_calls, fallbacks=info.precond_fallbacks, restarts=info.restarts,
                    theta=th, residual_norms=rs, n_converged=nc, times=times)
    finally:
        lib().be_result_free(h)
        if _os.environ.get("BE_TRACE_SEGMENTS"):
            print(f"[be] host: records + result free {1e3 * (time.perf_counter() - t1):.1f} ms", file=sys.stderr, flush=True)


def dense_mix(ctx: Context, x: np.ndarray, c: np.ndarray, y: np.ndarray | None = None) -> np.ndarray:
    """block_times_small(_add) (densela.hpp:448-484) on the device: Y (+)= X C for host panels."""
    x = np.ascontiguousarray(x, np.float64)
    cc = np.asfortranarray(c, np.float64)
    n, p = x.shape
    q = cc.shape[1]
    acc = y is not None
    out = np.ascontiguousarray(y, np.float64).copy() if acc else np.zeros((n, q))
    check(lib().be_dense_mix(ctx.handle, _p(x), C.c_int64(n), C.c_int(p), _p(cc), C.c_int(q), _p(out), C.c_int(int(acc))))
    return out


def gram_dev(ctx: Context, a_ptr: int, b_ptr: int, nb: int, n: int) -> np.ndarray:
    out = np.zeros(nb * nb)
    check(lib().be_gram(ctx.handle, C.c_void_p(a_ptr), C.c_int(nb), C.c_void_p(b_ptr), C.c_int(nb), C.c_int64(n),
                        _p(out)))
    return out.reshape((nb, nb), order="F")


def sygv_lowest(ctx: Context, a, b, k, pivot_floor=0.0):
    """sygv_lowest (densela.hpp:357-407) computed on the device."""
    n = a.shape[0]
    A = np.asfortranarray(a, dtype=np.float64).ravel(order="F")
    B = np.asfortranarray(b, dtype=np.float64).ravel(order="F")
    c = np.zeros(n * k)
    d = np.zeros(k)
    check(lib().be_sygv_lowest(ctx.handle, _p(A), _p(B), C.c_int(n), C.c_int(k), C.c_double(pivot_floor), _p(c),
                               _p(d)))
    return c.reshape((n, k), order="F"), d


class IncrementalSolve:
    """be_lobpcg_begin / be_lobpcg_step / be_lobpcg_end (iteration-level control)."""

    def __init__(self, ctx: Context, op=None, n=None, tiles: Tiles | None = None, x0=None, k=5, nb=0, tol=1e-6,
                 maxiter=500, fom_iterations=4, seed=1234):
        if n is None:
            n = op.info().nrows
        self.cfg = SolverConfig(k, nb, tol, maxiter, fom_iterations, seed, 0)
        self._x0 = _x0_checked(x0, n, k, nb)
        self._h = C.c_void_p()
        check(lib().be_lobpcg_begin(ctx.handle, op.handle if op is not None else None, HOST_OP_FN(), None,
                                    C.c_int64(n), tiles.handle if tiles is not None else None, _p(self._x0),
                                    C.byref(self.cfg), C.byref(self._h)))

    def step(self, count=1) -> int:
        done = C.c_int(0)
        check(lib().be_lobpcg_step(self._h, C.c_int(count), C.byref(done)))
        return done.value

    def end(self):
        r = C.c_void_p()
        check(lib().be_lobpcg_end(self._h, C.byref(r)))
        self._h = None
        try:
            info = ResultInfo()
            check(lib().be_result_get_info(r, C.byref(info)))
            lam = np.zeros(info.k)
            check(lib().be_result_get(r, _p(lam), None))
            times = np.zeros((info.iterations, 4))
            for i in range(info.iterations):
                t = [C.c_double() for _ in range(4)]
                check(lib().be_result_get_record(r, C.c_int(i), None, None, None, *[C.byref(v) for v in t]))
                times[i] = [v.value for v in t]
            return dict(lambda_=lam, iterations=info.iterations, converged=bool(info.converged),
                        operator_calls=info.operator_calls, times=times)
        finally:
            lib().be_result_free(r)
