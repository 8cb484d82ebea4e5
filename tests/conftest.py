"""Shared fixtures.  `gpu` tests need a B200 and the built product library;
everything else runs on CPU (the CPU oracle is test infrastructure only)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PRODUCT_LIB = os.path.join(ROOT, "paper_2605_14526_b200", "_lib", "libheterodyn_b200.so")
ORACLE_LIB = os.path.join(ROOT, "oracle", "_build", "libheterodyn_oracle.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the sm_100a product library")


@pytest.fixture(scope="session")
def orc():
    from paper_2605_14526_b200.hd import Library
    if not os.path.exists(ORACLE_LIB):
        import subprocess
        subprocess.run(["make", "-j8"], cwd=os.path.join(ROOT, "oracle"), check=True)
    return Library(ORACLE_LIB)


@pytest.fixture(scope="session")
def prod():
    """The product library.  Missing library = hard failure, never a skip."""
    from paper_2605_14526_b200.hd import Library
    assert os.path.exists(PRODUCT_LIB), "product library not built (run __graft_entry__.build())"
    return Library(PRODUCT_LIB)


@pytest.fixture(scope="session")
def oracle_unit():
    import ctypes as C
    if not os.path.exists(ORACLE_LIB):
        import subprocess
        subprocess.run(["make", "-j8"], cwd=os.path.join(ROOT, "oracle"), check=True)
    lib = C.CDLL(ORACLE_LIB)
    D = C.POINTER(C.c_double)
    for name, args in {
        "ho_lame": [C.c_double, C.c_double, D, D],
        "ho_nh_energy": [D, C.c_double, C.c_double, D],
        "ho_stretch_hessian_eigs": [D, C.c_double, C.c_double, D],
        "ho_signed_svd": [D, D, D, D],
        "ho_project": [C.c_int, D, C.c_double, C.c_double, C.c_double, D, D, D],
        "ho_prox_differential": [C.c_int, D, C.c_double, C.c_double, C.c_double, C.c_double, D],
        "ho_tr_blend": [D, C.c_double, C.c_double, C.c_double, C.c_double, D],
        "ho_contact_scalar": [C.c_double] * 6 + [D],
        "ho_cone_project": [C.c_double, D, D],
        "ho_prox_means": [C.c_char_p, D],
    }.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    return lib
