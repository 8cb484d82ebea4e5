"""The reference-facing C ABI from plain C: examples/roll_backward.c compiles
and links against both libraries exporting include/heterodyn.h, and (on a GPU)
the product's output matches the oracle's."""
import os
import re
import subprocess

import pytest

from conftest import ORACLE_LIB, PRODUCT_LIB, ROOT


def _build(tmp_path, lib_path, tag):
    exe = str(tmp_path / f"roll_backward_{tag}")
    libdir, libfile = os.path.split(lib_path)
    name = libfile[3:-3]
    subprocess.run(["gcc", "-O2", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "roll_backward.c"), "-L", libdir, f"-l{name}",
                    f"-Wl,-rpath,{libdir}", "-lm", "-o", exe], check=True)
    return exe


def _parse(out):
    return {k: float(v) for k, v in re.findall(r"(\|q_T\||\|dL/dq0\|)=(\S+)", out)}


def test_c_client_builds_against_product(tmp_path):
    assert os.path.exists(PRODUCT_LIB)
    _build(tmp_path, PRODUCT_LIB, "product")


def test_c_client_runs_on_oracle(tmp_path, orc):
    exe = _build(tmp_path, ORACLE_LIB, "oracle")
    out = subprocess.run([exe, "cantilever3", "3"], check=True, capture_output=True, text=True).stdout
    vals = _parse(out)
    assert vals["|q_T|"] > 0 and vals["|dL/dq0|"] > 0


@pytest.mark.gpu
def test_c_client_product_matches_oracle(tmp_path, orc):
    ref = _parse(subprocess.run([_build(tmp_path, ORACLE_LIB, "oracle"), "cantilever3", "3"], check=True,
                                capture_output=True, text=True).stdout)
    got = _parse(subprocess.run([_build(tmp_path, PRODUCT_LIB, "product"), "cantilever3", "3"], check=True,
                                capture_output=True, text=True).stdout)
    for k in ref:
        assert abs(got[k] - ref[k]) <= 1e-6 * abs(ref[k]), (k, got[k], ref[k])
