"""CPU checks of the drop-in boundary: libamgr_b200.so loads (all symbols
resolve) and exports exactly the functions include/amgr.h declares; the Python
mirror binds every one of them.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "amgr.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(amgr_[A-Za-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    import paper_2108_02054_b200 as amg

    L = amg.lib()  # dlopen resolves every undefined symbol or raises
    names = header_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_python_mirror_binds_every_header_function():
    import paper_2108_02054_b200 as amg

    assert set(amg.PROTOTYPES) == set(header_functions())


def test_version_and_defaults_without_gpu():
    import paper_2108_02054_b200 as amg

    L = amg.lib()
    assert b"sm_100a" in L.amgr_version()
    p = amg._AmgParams()
    L.amgr_amg_params_default(ctypes.byref(p))
    # AmgParams defaults (proj/include/amgreuse/hierarchy.hpp:14-21)
    assert (p.eps, p.omega, p.pre_sweeps, p.post_sweeps, p.coarse_enough, p.max_direct_size) == (
        0.08, 0.72, 1, 1, 100, 2000)
    s = amg._SolveParams()
    L.amgr_solve_params_default(ctypes.byref(s))
    assert (s.tol, s.max_iter) == (1e-8, 100)  # bicgstab.hpp:17-20
    assert L.amgr_problem_nnz(256) == 7 * 256 ** 3 - 6 * 256 ** 2


def test_python_params_match_c_defaults():
    import paper_2108_02054_b200 as amg

    p = amg._AmgParams()
    amg.lib().amgr_amg_params_default(ctypes.byref(p))
    q = amg.AmgParams()._c()
    for f, _ in amg._AmgParams._fields_:
        assert getattr(p, f) == pytest.approx(getattr(q, f)), f


def test_struct_layouts_match_header():
    import paper_2108_02054_b200 as amg

    # amgr_csr: 3 x int64 + 3 pointers + 2 x int32 = 56 bytes
    assert ctypes.sizeof(amg._Csr) == 56
    assert ctypes.sizeof(amg._SolveStats) == 24
    assert ctypes.sizeof(amg._AmgParams) == 88


def test_compute_without_gpu_fails_loudly():
    import paper_2108_02054_b200 as amg

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises(amg.AmgrError):
        amg.Context(0)
