"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU
and exports every function include/blockeig_b200.h declares; the C++ mirror
header compiles and the reference-style test program links against it;
error mapping for host-side entry points (no device calls)."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2109_00485_b200 import abi, build

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "blockeig_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s+(be_[a-z0-9_]+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("be_op_create", "be_op_apply", "be_precond_apply", "be_lobpcg_solve", "be_csb_build",
                 "be_tiles_create", "be_gram", "be_sygv_lowest", "be_last_error"):
        assert must in names
    assert len(names) >= 40


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(build.LIB))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", str(build.LIB)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (be_[a-z0-9_]+)$", out, flags=re.M))
    assert set(declared_functions()) <= exported


def test_status_codes_match_header():
    text = HEADER.read_text()
    for name, val in re.findall(r"(BE_ERR_[A-Z_]+)\s*=\s*(\d+)", text):
        assert getattr(abi, name, int(val)) == int(val)


def test_cpp_mirror_compiles_and_links():
    binary = build.build_cpp_tests()
    assert binary.exists()
    syms = subprocess.run(["nm", "-D", "--undefined-only", str(binary)], capture_output=True, text=True).stdout
    assert "be_lobpcg_solve" in syms and "be_op_create" in syms


def test_host_errors_map_to_reference_exceptions():
    b = abi.uniform_boundaries(10, 5)
    with pytest.raises(abi.DuplicateEntry):
        abi.build_csb_coo(abi.as_triples([3, 3], [1, 1], [1.0, 2.0]), 10, 10, b, b)
    with pytest.raises(abi.IndexOutOfRange):
        abi.build_csb_coo(abi.as_triples([30], [1], [1.0]), 10, 10, b, b)
    with pytest.raises(abi.BadParams):
        abi.build_csb_coo(abi.as_triples([3], [1], [1.0]), 10, 10, np.array([0, 4, 9]), b)
    with pytest.raises(abi.BadParams):  # csb.hpp:90-91
        abi.uniform_boundaries(100000, 40000)
    big = np.array([0, 40000, 100000])
    with pytest.raises(abi.BlockTooLarge):  # csb.hpp:71-72
        abi.build_csb_coo(abi.as_triples([3], [1], [1.0]), 100000, 100000, big, big)
    m = abi.build_csb_coo(abi.as_triples([1], [3], [1.0]), 10, 10, b, b)
    assert not m.is_strictly_lower()


def test_no_device_fails_loudly():
    """Without a GPU every device entry point reports an error; nothing falls
    back to a host computation."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(abi.BlockeigError):
        abi.Context(0)
