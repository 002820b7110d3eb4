"""CPU checks of the C-ABI library: it loads, exports every symbol the header
declares, and the host-only entry points behave (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cuhallar.h")
LIB = os.path.join(ROOT, "paper_2505_13719_b200", "libcuhallar.so")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(cuhallar_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__ as g
        g.build()
    return ctypes.CDLL(LIB)


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_host_only_entry_points(lib):
    lib.cuhallar_matcomp_constraint_count.restype = ctypes.c_int64
    # test_instances.cpp:147-151
    assert lib.cuhallar_matcomp_constraint_count(3000, 7000, 3, 0) == 828931
    assert lib.cuhallar_matcomp_constraint_count(3000, 7000, 5, 0) == 2302586
    assert lib.cuhallar_matcomp_constraint_count(30, 70, 2, 0) == 1843
    lib.cuhallar_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.cuhallar_version()


def test_package_imports_without_gpu():
    import paper_2505_13719_b200 as H
    assert H.matcomp_constraint_count(2000, 2000, 3) == 298586
    cfg = H.SolverConfig()
    c = cfg._c()
    assert c.eps == 1e-5 and c.eig_block_restart == 30 and c.aipp_lambda0 == 10.0
