"""ctypes access to the test oracles (test infrastructure only).

- ORC: oracle/liboracle.so, the CPU restatement of the reference algorithm
  (oracle/oracle.cpp), serial.
- REF: oracle/_ref/libref.so, the unmodified reference headers compiled by
  oracle/Makefile (present when built in the container; the prebuilt .so
  travels to the GPU box). Tests that need it skip when it is absent.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
ORC_PATH = ORACLE_DIR / "liboracle.so"
REF_PATH = ORACLE_DIR / "_ref" / "libref.so"

_orc = None
_ref = None


def build():
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)


def orc():
    global _orc
    if _orc is None:
        if not ORC_PATH.exists():
            build()
        _orc = C.CDLL(str(ORC_PATH))
        _orc.orc_last_error.restype = C.c_char_p
    return _orc


def ref():
    global _ref
    if _ref is None:
        if not REF_PATH.exists():
            return None
        _ref = C.CDLL(str(REF_PATH))
        _ref.ref_last_error.restype = C.c_char_p
        _ref.ref_prepare.restype = C.c_void_p
        _ref.ref_prepare.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int]
        _ref.ref_release.argtypes = [C.c_void_p]
        _ref.ref_time_apply.restype = C.c_double
        _ref.ref_time_apply.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.c_int]
        _ref.ref_time_lobpcg.restype = C.c_double
        _ref.ref_time_lobpcg.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_void_p]
        _ref.ref_tile_entries.restype = C.c_int64
        _ref.ref_tile_entries.argtypes = [C.c_void_p]
        _ref.ref_lobpcg_iter_times.restype = C.c_int
        _ref.ref_lobpcg_iter_times.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_void_p]
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _chk(lib, prefix, st):
    if st != 0:
        raise OracleError(st, getattr(lib, prefix + "_last_error")().decode())


def _p(a):
    return C.c_void_p(0) if a is None else C.c_void_p(a.ctypes.data)


class Impl:
    """Same calls on either the restatement (orc) or the reference (ref)."""

    def __init__(self, which="orc", threads=1, variant=0):
        self.which = which
        self.lib = orc() if which == "orc" else ref()
        if self.lib is None:
            raise FileNotFoundError("oracle/_ref/libref.so not built")
        self.threads = threads
        self.variant = variant

    def spmm(self, csb, diag, x, y=None, mode=0):
        x = np.ascontiguousarray(x, np.float64)
        nb = x.shape[1]
        out_rows = csb.ncols if mode == 2 else csb.nrows
        y = np.zeros((out_rows, nb)) if y is None else np.ascontiguousarray(y, np.float64).copy()
        d = None if diag is None else np.ascontiguousarray(diag, np.float64)
        v = csb.view()
        if self.which == "orc":
            _chk(self.lib, "orc", self.lib.orc_spmm(C.byref(v), _p(d), _p(x), _p(y), C.c_int64(nb), C.c_int(mode)))
        else:
            _chk(self.lib, "ref", self.lib.ref_spmm(C.byref(v), _p(d), _p(x), _p(y), C.c_int64(nb), C.c_int(mode),
                                                    C.c_int(self.variant), C.c_int(self.threads)))
        return y

    def precond(self, csb, diag, toff, shifts, r, m=4):
        r = np.ascontiguousarray(r, np.float64)
        w = np.zeros_like(r)
        fb = C.c_int64(0)
        toff = np.ascontiguousarray(toff, np.int64)
        sh = np.ascontiguousarray(shifts, np.float64)
        d = np.ascontiguousarray(diag, np.float64)
        v = csb.view()
        fn = self.lib.orc_precond if self.which == "orc" else self.lib.ref_precond
        _chk(self.lib, self.which, fn(C.byref(v), _p(d), _p(toff), C.c_int64(len(toff)), _p(sh), _p(r), _p(w),
                                      C.c_int64(r.shape[1]), C.c_int(m), C.byref(fb)))
        return w, fb.value

    def sygv_lowest(self, a, b, k, floor=0.0):
        n = a.shape[0]
        A = np.asfortranarray(a, np.float64).ravel(order="F")
        B = np.asfortranarray(b, np.float64).ravel(order="F")
        c = np.zeros(n * k)
        d = np.zeros(k)
        fn = self.lib.orc_sygv_lowest if self.which == "orc" else self.lib.ref_sygv_lowest
        _chk(self.lib, self.which, fn(_p(A), _p(B), C.c_int(n), C.c_int(k), C.c_double(floor), _p(c), _p(d)))
        return c.reshape((n, k), order="F"), d

    def lobpcg(self, csb, diag, toff=None, x0=None, k=5, nb=0, tol=1e-6, maxiter=500, fom_m=4, seed=1234):
        nb = nb or k + 3
        n = csb.nrows
        lam = np.zeros(k)
        x = np.zeros((n, k))
        th = np.zeros((maxiter, nb))
        rs = np.zeros((maxiter, nb))
        nc = np.zeros(maxiter, np.int32)
        info = np.zeros(5, np.int64)
        d = np.ascontiguousarray(diag, np.float64)
        t = None if toff is None else np.ascontiguousarray(toff, np.int64)
        nt = 0 if t is None else len(t)
        x0a = None if x0 is None else np.ascontiguousarray(x0, np.float64)
        v = csb.view()
        if self.which == "orc":
            st = self.lib.orc_lobpcg(C.byref(v), _p(d), _p(t), C.c_int64(nt), _p(x0a), C.c_int(k), C.c_int(nb),
                                     C.c_double(tol), C.c_int(maxiter), C.c_int(fom_m), C.c_uint64(seed), _p(lam),
                                     _p(x), _p(th), _p(rs), _p(nc), _p(info))
        else:
            pt = np.zeros(4)
            st = self.lib.ref_lobpcg(C.byref(v), _p(d), _p(t), C.c_int64(nt), _p(x0a), C.c_int(k), C.c_int(nb),
                                     C.c_double(tol), C.c_int(maxiter), C.c_int(fom_m), C.c_uint64(seed),
                                     C.c_int(self.variant), C.c_int(self.threads), _p(lam), _p(x), _p(th), _p(rs),
                                     _p(nc), _p(pt), _p(info))
        _chk(self.lib, self.which, st)
        it = int(info[1])
        return dict(lambda_=lam, x=x, converged=bool(info[0]), iterations=it, operator_calls=int(info[2]),
                    fallbacks=int(info[3]), restarts=int(info[4]), theta=th[:it], residual_norms=rs[:it],
                    n_converged=nc[:it])


def orc_extract_tiles(csb, diag, toff):
    lib = orc()
    toff = np.ascontiguousarray(toff, np.int64)
    nt = len(toff) - 1
    nent = np.zeros(nt, np.int64)
    d = np.ascontiguousarray(diag, np.float64)
    v = csb.view()
    _chk(lib, "orc", lib.orc_extract_tiles(C.byref(v), _p(d), _p(toff), C.c_int64(len(toff)), _p(nent), None, None,
                                           None, None))
    tot = int(nent.sum())
    rows = np.zeros(tot, np.int32)
    cols = np.zeros(tot, np.int32)
    vals = np.zeros(tot)
    dpos = np.zeros(int(toff[-1]), np.int64)
    _chk(lib, "orc", lib.orc_extract_tiles(C.byref(v), _p(d), _p(toff), C.c_int64(len(toff)), _p(nent), _p(rows),
                                           _p(cols), _p(vals), _p(dpos)))
    return nent, rows, cols, vals, dpos


def ref_generate_synthetic(kind, n, density=0.02, bandwidth=8, block_extent=4000, seed=1):
    lib = ref()
    nl, nt = C.c_int64(), C.c_int64()
    _chk(lib, "ref", lib.ref_generate_synthetic(C.c_int(kind), C.c_int64(n), C.c_double(density),
                                                C.c_int64(bandwidth), C.c_int64(block_extent), C.c_uint64(seed),
                                                C.byref(nl), None, None, None, None, C.byref(nt), None))
    rows = np.zeros(nl.value, np.int64)
    cols = np.zeros(nl.value, np.int64)
    vals = np.zeros(nl.value)
    diag = np.zeros(n)
    toff = np.zeros(nt.value, np.int64)
    _chk(lib, "ref", lib.ref_generate_synthetic(C.c_int(kind), C.c_int64(n), C.c_double(density),
                                                C.c_int64(bandwidth), C.c_int64(block_extent), C.c_uint64(seed),
                                                C.byref(nl), _p(rows), _p(cols), _p(vals), _p(diag), C.byref(nt),
                                                _p(toff)))
    return rows, cols, vals, diag, toff


def ref_build_csb(rows, cols, vals, nrows, ncols, rb, cb):
    lib = ref()
    rb = np.ascontiguousarray(rb, np.int64)
    cb = np.ascontiguousarray(cb, np.int64)
    nblk = (len(rb) - 1) * (len(cb) - 1)
    bn = np.zeros(nblk, np.int64)
    bo = np.zeros(nblk, np.int64)
    n = len(rows)
    lr = np.zeros(n, np.uint16)
    lc = np.zeros(n, np.uint16)
    v = np.zeros(n)
    r_ = np.ascontiguousarray(rows, np.int64)
    c_ = np.ascontiguousarray(cols, np.int64)
    v_ = np.ascontiguousarray(vals, np.float64)
    _chk(lib, "ref", lib.ref_build_csb(_p(r_), _p(c_), _p(v_), C.c_int64(n), C.c_int64(nrows), C.c_int64(ncols),
                                       _p(rb), C.c_int64(len(rb)), _p(cb), C.c_int64(len(cb)), _p(bn), _p(bo),
                                       _p(lr), _p(lc), _p(v)))
    return bn, bo, lr, lc, v


def ref_partition_rank(csb, diag, nd, sub_bounds, intra_extent, rank):
    """The reference's partition_matrix (dist.hpp:113-198) for one rank:
    (global triples of its stored block, (segment begin, end))."""
    lib = ref()
    t = csb.to_triples()
    n = csb.nrows
    cap = len(t)
    r, c, v = np.zeros(cap, np.int64), np.zeros(cap, np.int64), np.zeros(cap)
    cnt = np.array([cap], np.int64)
    seg = np.zeros(2, np.int64)
    rows = np.ascontiguousarray(t["row"]); cols = np.ascontiguousarray(t["col"]); vals = np.ascontiguousarray(t["value"])
    d = np.ascontiguousarray(diag, np.float64)
    b = np.ascontiguousarray(sub_bounds, np.int64)
    st = lib.ref_partition_rank(_p(rows), _p(cols), _p(vals), C.c_int64(len(t)), _p(d), C.c_int64(n), C.c_int(nd),
                                _p(b), C.c_int64(intra_extent), C.c_int(rank), _p(r), _p(c), _p(v), _p(cnt), _p(seg))
    _chk(lib, "ref", st)
    k = int(cnt[0])
    return r[:k], c[:k], v[:k], (int(seg[0]), int(seg[1]))


def ref_build_layout(nd):
    lib = ref()
    nr = nd * (nd + 1) // 2
    blocks = np.zeros((nr, 3), np.int32)
    dr = np.zeros(nd, np.int32)
    _chk(lib, "ref", lib.ref_build_layout(C.c_int(nd), _p(blocks), _p(dr)))
    return blocks, dr
