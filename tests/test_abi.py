"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/*.h declares,
its host-only helpers are right, and host-side argument validation returns the documented
status codes synchronously (no GPU needed for any of these)."""
import ctypes
import glob
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
from paper_2605_05219_b200 import sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(sp_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def L():
    from paper_2605_05219_b200 import build
    build.build()
    return sp.lib()


def test_exports_every_declared_symbol(L):
    names = declared_symbols()
    assert len(names) >= 10
    out = subprocess.check_output(["nm", "-D", "--defined-only", sp.LIB_PATH]).decode()
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    missing = names - exported
    assert not missing, missing
    assert set(sp.SYMBOLS) == names      # the binding covers exactly the declared ABI


def test_built_for_sm100a(L):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sp.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_version_and_status_strings(L):
    assert b"sm_100a" in L.sp_version()
    for s in range(0, 9):
        assert L.sp_status_string(s).startswith(b"SP_")


@pytest.mark.parametrize("N,M", [(10, 2), (5, 1), (5, 0), (9, 3), (32768, 64), (8192, 16), (1, 1)])
def test_balanced_helper_matches_table1(L, N, M):
    assert sp.balanced_positions(N, M) == oracle.balanced(N, M).tolist()


@pytest.mark.parametrize("N,B", [(300, 128), (100, 128), (128, 128), (32768, 64), (8192, 128)])
def test_block_helper_matches_table1(L, N, B):
    assert sp.block_positions(N, B) == oracle.block(N, B).tolist()


def test_helper_errors(L):
    buf = (ctypes.c_int32 * 8)()
    assert L.sp_balanced_positions(0, 0, buf) == -sp.SP_ERR_BAD_LENGTH
    assert L.sp_balanced_positions(5, 6, buf) == -sp.SP_ERR_BUDGET_TOO_LARGE
    assert L.sp_block_positions(5, 0, buf) == -sp.SP_ERR_BAD_ARGUMENT


def test_sync_argument_errors(L):
    """Shape errors are returned synchronously, before any CUDA call (runs without a GPU)."""
    p = ctypes.c_void_p(16)
    assert L.sp_overlap_hist(p, p, 1, p, p, p, 1, 0, p, None, None) == sp.SP_ERR_BAD_LENGTH
    assert L.sp_overlap_hist(p, p, 1, p, p, p, 1, 65536, p, None, None) == sp.SP_ERR_BAD_LENGTH
    assert L.sp_overlap_hist(None, p, 1, p, p, p, 1, 8, p, None, None) == sp.SP_ERR_BAD_ARGUMENT
    assert L.sp_overlap_hist(p, p, 1, p, p, p, 0, 8, p, None, None) == sp.SP_OK   # nothing to do
    assert L.sp_place_checkpoints(p, 0, 1, 0, 0, p, p, p, None, p, 1, None) == sp.SP_ERR_BAD_LENGTH
    assert L.sp_place_checkpoints(p, 0, 1, 4, 5, p, p, p, None, p, 1, None) == \
        sp.SP_ERR_BUDGET_TOO_LARGE
    assert L.sp_place_checkpoints(p, 0, 1, 4, -1, p, p, p, None, p, 1, None) == \
        sp.SP_ERR_BUDGET_TOO_LARGE
    assert L.sp_place_checkpoints(p, 7, 1, 4, 2, p, p, p, None, p, 1, None) == \
        sp.SP_ERR_BAD_ARGUMENT
    assert L.sp_place_checkpoints(None, 0, 1, 4, 2, p, p, p, None, p, 1, None) == \
        sp.SP_ERR_BAD_ARGUMENT
    assert L.sp_place_checkpoints(p, 0, 0, 4, 2, p, p, p, None, p, 1, None) == sp.SP_OK
    assert L.sp_expected_recompute(p, 0, 1, 0, p, p, 1, 1, 1, p, None, None) == \
        sp.SP_ERR_BAD_LENGTH
    assert L.sp_expected_recompute(p, 9, 1, 4, p, p, 1, 1, 1, p, None, None) == \
        sp.SP_ERR_BAD_ARGUMENT
    assert L.sp_accumulate_depths(p, p, 4, 0, 2, 0, p, None) == sp.SP_ERR_BAD_LENGTH
    assert L.sp_accumulate_depths(p, p, 4, 3, 2, 8, p, None) == sp.SP_ERR_BAD_LENGTH


def test_binding_refuses_cpu_tensors(L):
    import torch
    h = torch.zeros(2, 9, dtype=torch.int32)
    with pytest.raises(ValueError, match="CUDA"):
        sp.place_checkpoints(h, 2)


def test_product_never_imports_oracle():
    """The product path shares no code with the oracle and never loads it."""
    for f in glob.glob(os.path.join(ROOT, "paper_2605_05219_b200", "**", "*"), recursive=True):
        if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
            src = open(f).read()
            assert "import oracle" not in src and "from oracle" not in src, f
            assert "sp_oracle" not in src and "liboracle" not in src, f


@pytest.mark.parametrize("N", [1, 3, 10, 100, 1000, 8192, 32768])
def test_sqrt_helper_matches_oracle(L, N):
    assert sp.sqrt_positions(N) == oracle.sqrt_positions(N).tolist()


@pytest.mark.parametrize("N,M", [(7, 3), (50, 1), (4, 3), (8192, 16), (32768, 62), (100, 62)])
def test_log_helper_matches_oracle(L, N, M):
    assert sp.log_positions(N, M) == oracle.log_positions(N, M).tolist()
