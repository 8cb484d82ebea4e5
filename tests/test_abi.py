"""The C-ABI libraries load and export every symbol their headers declare;
host-only parts of the product ABI behave like the reference's C surface
(no GPU needed).  CPU only."""
import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ORACLE_LIB, PRODUCT_LIB, ROOT


def declared(header, macro):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(macro + r"\s+[\w\s\*]*?\b(h[dk]k?_\w+)\s*\(", text)))


def exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_product_exports_every_declared_symbol():
    assert os.path.exists(PRODUCT_LIB), "product library not built"
    syms = exported(PRODUCT_LIB)
    hd = declared("heterodyn.h", "HD_API")
    hdk = declared("hdk.h", "HDK_API")
    assert len(hd) >= 40 and len(hdk) >= 20
    missing = [s for s in hd + hdk if s not in syms]
    assert not missing, missing


def test_oracle_exports_the_hd_abi():
    syms = exported(ORACLE_LIB)
    missing = [s for s in declared("heterodyn.h", "HD_API") if s not in syms]
    assert not missing, missing


def test_product_library_loads_and_binds(prod):
    assert prod.lib.hd_last_error() == b""
    assert prod.lib.hd_last_error_code() == 0


def test_product_scene_surface_matches_reference_semantics(prod):
    """test_capi.cpp:35-90 against the product's host-side scene layer."""
    from paper_2605_14526_b200.hd import HdError
    sc = prod.builtin("two-tet")
    assert (sc.vertex_count, sc.element_count, sc.frame_count, sc.name) == (5, 2, 3, "two-tet")
    for name, (nv, ne, fr) in {"cantilever3": (208, 648, 60), "twist-bar": (208, 648, 40), "ball-drop": (13, 20, 50),
                               "resting-box": (27, 48, 30), "slab-on-sphere": (162, 384, 60)}.items():
        s = prod.builtin(name)
        assert (s.vertex_count, s.element_count, s.frame_count) == (nv, ne, fr)
    with pytest.raises(HdError) as e:
        prod.builtin("no-such-scene")
    assert e.value.code == 2
    with pytest.raises(HdError) as e:
        prod.scene("{ not json")
    assert e.value.code == 1
    with pytest.raises(HdError) as e:
        prod.load("/nonexistent/path/scene.json")
    assert e.value.code == 12
    with pytest.raises(HdError) as e:
        prod.scene({"mesh": {"grid": {"dims": [1, 1, 1]}}, "material": {"young": 5e4, "poisson": 0.6}})
    assert e.value.code == 2  # validation lists the InvalidPoisson violation


def test_product_has_no_cpu_fallback(prod):
    """Without a CUDA device the product refuses to simulate instead of falling back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2605_14526_b200.hd import HdError
    with pytest.raises(HdError) as e:
        prod.builtin("two-tet").sim()
    assert "CUDA" in str(e.value)
