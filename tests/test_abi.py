"""The product library loads on a GPU-less host, exports every symbol the
C header declares, and its host-only entry points (plan helpers, shard
partition, argument validation) agree with the reference."""
import ctypes as ct
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2504_19449_b200 import _lib as L
from paper_2504_19449_b200 import Recipe, keep_count, shard_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rsparse_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rsp_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_what_python_binds():
    assert sorted(L.EXPORTS) == declared_functions()


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (rsp_\w+)", out))
    assert set(declared_functions()) <= exported
    assert L.lib().rsp_abi_version() == 3


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_keep_count_matches_reference_rule(golden):
    # sparsity.cpp:26-27: k = ceil(s * n) in double
    for name in [str(s) for s in golden["thr.names"]]:
        if int(golden[f"thr.{name}.err"][0]):
            with pytest.raises(L.UsageError):
                keep_count(float(golden[f"thr.{name}.s"][0]), golden[f"thr.{name}.x"].size)
            continue
        s, n = float(golden[f"thr.{name}.s"][0]), golden[f"thr.{name}.x"].size
        assert keep_count(s, n) == golden[f"thr.{name}.kept"].size
    for n in (1, 37, 4096, 11008, 14336):
        for s in (0.0, 0.1, 0.15, 0.3333, 0.5, 0.77, 0.99, 1.0):
            assert keep_count(s, n) == int(np.ceil(s * n))


def test_plan_for_matches_reference(golden):
    for (rho, c, n, m, s, r) in golden["plan.cases"]:
        plan = Recipe([rho], [c]).plan_for(0, int(n), int(m))
        assert plan.keep_fraction == s and plan.rank == int(r)


def test_shard_rows_partition():
    for m in (1, 7, 4096, 11008, 14336):
        for g in (1, 2, 3, 4, 8):
            if g > m:
                continue
            spans = [shard_rows(m, i, g) for i in range(g)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[i][1] == spans[i + 1][0] for i in range(g - 1))
    with pytest.raises(L.UsageError):
        shard_rows(16, 2, 2)


def test_create_validates_like_the_reference():
    # argument errors are raised before any device work (no GPU needed)
    d = L.LinearDesc()
    d.m_in, d.m_out, d.rank, d.keep_fraction, d.k_override = 6, 4, 5, 0.5, -1  # rank > min
    d.weight_dtype, d.src_dtype, d.src_memory = L.RSP_BF16, L.RSP_F64, L.RSP_MEM_HOST
    buf = np.zeros(64)
    d.w = d.a_r = d.b_r = buf.ctypes.data
    h = ct.c_void_p()
    assert L.lib().rsp_linear_create(ct.byref(d), ct.byref(h)) == L.RSP_E_USAGE
    assert b"rank 5 exceeds" in L.lib().rsp_last_error()
    d.rank, d.keep_fraction = 2, 1.5  # sparsity.cpp:22-25
    assert L.lib().rsp_linear_create(ct.byref(d), ct.byref(h)) == L.RSP_E_USAGE
    d.keep_fraction, d.k_override = 0.5, 7  # matrix.cpp:101-104
    assert L.lib().rsp_linear_create(ct.byref(d), ct.byref(h)) == L.RSP_E_USAGE


def test_top_k_validates_k_gt_n():
    assert L.lib().rsp_top_k_by_magnitude(None, L.RSP_F32, 3, 4, None, None, None) == L.RSP_E_USAGE
