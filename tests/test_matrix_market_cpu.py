"""Matrix Market ingest / export: the cases of the reference's
test_cli.cpp:34-91, plus differential checks against the reference's own
ingest_matrix_market / write_matrix_market (oracle/_ref) on random files."""
import numpy as np
import pytest

from paper_2109_00485_b200 import abi
import oracle_lib as ol

HDR = "%%MatrixMarket matrix coordinate real symmetric\n"


def test_identity_file():  # test_cli.cpp:34-44
    n, lower, diag = abi.read_matrix_market(text=HDR + "% a comment\n3 3 3\n1 1 1.0\n2 2 1.0\n3 3 1.0\n")
    assert n == 3 and len(lower) == 0
    assert diag.tolist() == [1.0, 1.0, 1.0]


def test_upper_given_entry_is_mirrored():  # test_cli.cpp:46-56
    n, lower, diag = abi.read_matrix_market(text=HDR + "3 3 1\n1 3 2.5\n")
    assert len(lower) == 1
    assert (lower[0]["row"], lower[0]["col"], lower[0]["value"]) == (2, 0, 2.5)
    assert diag.tolist() == [0.0, 0.0, 0.0]


def _random_lower(n, count, seed):
    rng = np.random.default_rng(seed)
    keys = set()
    while len(keys) < count:
        r = int(rng.integers(1, n))
        c = int(rng.integers(0, r))
        keys.add((r, c))
    keys = sorted(keys, key=lambda k: rng.random())
    return abi.as_triples([k[0] for k in keys], [k[1] for k in keys], rng.uniform(-2, 2, count))


def test_write_read_round_trip():  # test_cli.cpp:58-70
    lower = _random_lower(6, 8, 5)
    diag = np.array([1.0, 0.0, 3.0, 4.0, 0.5, 6.0])
    text = abi.write_matrix_market(6, lower, diag)
    n, lo2, d2 = abi.read_matrix_market(text=text)
    assert n == 6
    assert sorted(map(tuple, lo2.tolist())) == sorted(map(tuple, lower.tolist()))
    assert d2.tolist() == diag.tolist()


@pytest.mark.parametrize("text, err", [
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n", abi.NotSymmetricHeader),
    ("%%MatrixMarket matrix array real symmetric\n2 2\n1\n2\n3\n", abi.ParseError),
    (HDR + "2 3 1\n1 1 1.0\n", abi.ParseError),
    (HDR + "3 3 2\n1 1 1.0\n", abi.ParseError),
    ("", abi.ParseError),
    ("%%MatrixMarket vector coordinate real symmetric\n", abi.ParseError),
    ("%%MatrixMarket matrix coordinate complex symmetric\n1 1 0\n", abi.ParseError),
    (HDR + "0 0 0\n", abi.ParseError),
    (HDR + "3 3 1\n4 1 1.0\n", abi.ParseError),
    (HDR + "3 3 2\n2 2 1.0\n2 2 3.0\n", abi.DuplicateEntry),
])
def test_rejections(text, err):  # test_cli.cpp:72-91 and the remaining throw sites of matrix_market.hpp:38-88
    with pytest.raises(err):
        abi.read_matrix_market(text=text)


def test_integer_field_crlf_and_case():
    n, lower, diag = abi.read_matrix_market(
        text="%%matrixmarket MATRIX Coordinate INTEGER Symmetric\r\n%c\r\n\r\n2 2 2\r\n2 1 -3\r\n1 1 4\r\n")
    assert n == 2 and lower.tolist() == [(1, 0, -3.0)] and diag.tolist() == [4.0, 0.0]


def test_file_path(tmp_path):
    p = tmp_path / "m.mtx"
    p.write_text(HDR + "4 4 2\n3 2 0.25\n4 4 2.0\n")
    n, lower, diag = abi.read_matrix_market(path=p)
    assert n == 4 and lower.tolist() == [(2, 1, 0.25)] and diag.tolist() == [0, 0, 0, 2.0]
    with pytest.raises(abi.ParseError):
        abi.read_matrix_market(path=tmp_path / "missing.mtx")


def test_ingest_feeds_the_csb_build():
    """MM text -> strictly-lower triples -> build_csb_coo: the same CSB as building from the triples directly."""
    lower = _random_lower(40, 120, 9)
    diag = np.linspace(1, 2, 40)
    n, lo2, d2 = abi.read_matrix_market(text=abi.write_matrix_market(40, lower, diag))
    b = [0, 13, 27, 40]
    a = abi.build_csb_coo(lower, 40, 40, b, b).to_triples()
    c = abi.build_csb_coo(lo2, n, n, b, b).to_triples()
    assert a.tobytes() == c.tobytes()


@pytest.mark.skipif(ol.ref() is None, reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_matches_reference_ingest_and_write(seed):
    """Differential: parse and write are identical to the reference's own functions."""
    import ctypes as C
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 60))
    lower = _random_lower(n, int(rng.integers(0, n)), seed)
    diag = np.where(rng.random(n) < 0.3, 0.0, rng.normal(size=n))
    text = abi.write_matrix_market(n, lower, diag)
    # mix upper-given entries in: swap row/col on some lines
    lines = text.splitlines()
    for i in range(2, len(lines)):
        if rng.random() < 0.4:
            r, c, v = lines[i].split()
            lines[i] = f"{c} {r} {v}"
    text2 = "\n".join(lines) + "\n"
    lib = ol.ref()
    b = text2.encode()
    nn = np.zeros(1, np.int64)
    cnt = np.array([len(lower) + n], np.int64)
    rows = np.zeros(cnt[0], np.int64)
    cols = np.zeros(cnt[0], np.int64)
    vals = np.zeros(cnt[0])
    d = np.zeros(n)
    st = lib.ref_mm_parse(b, C.c_int64(len(b)), ol._p(nn), ol._p(rows), ol._p(cols), ol._p(vals), ol._p(cnt),
                          ol._p(d), C.c_int64(n))
    assert st == 0
    n2, lo2, d2 = abi.read_matrix_market(text=text2)
    k = int(cnt[0])
    assert n2 == int(nn[0])
    assert lo2["row"].tolist() == rows[:k].tolist() and lo2["col"].tolist() == cols[:k].tolist()
    assert lo2["value"].tobytes() == vals[:k].tobytes() and d2.tobytes() == d.tobytes()
    # writer: byte-identical text
    buf = C.create_string_buffer(len(text) + 64)
    ln = np.zeros(1, np.int64)
    lr, lc, lv = (np.ascontiguousarray(lower[f]) for f in ("row", "col", "value"))  # alive across the call
    st = lib.ref_mm_write(C.c_int64(n), ol._p(lr), ol._p(lc), ol._p(lv), C.c_int64(len(lower)), ol._p(diag), buf,
                          C.c_int64(len(buf)), ol._p(ln))
    assert st == 0
    assert buf.value.decode() == text
