"""The multi-column solve passes on the FP64 tensor cores (solve.cu
k_rowdot_mma / k_coltile_mma: m8n8k4 DMMA over 8 segments x 4 columns and
8 columns x 4 segments) against the FMA passes (two columns per warp) on the
contact adjoint, whose K contact columns run four per factor stream
(engine_columns.cpp, backward.cpp:227-283).  The variants differ only in the
summation order inside a row dot / a column tile, so the trajectory is
bitwise the same (the forward does not use the multi-column passes) and the
gradients agree to rounding; the oracle comparison of the same scenes is in
test_gpu_contact.py / test_gpu_fullsize.py (default: tensor-core pass 1, FMA
pass 2 — the tensor-core pass 2 measured slower)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(tmp_path, name, rowdot, coltile):
    out = str(tmp_path / f"{name}.npz")
    env = dict(os.environ, HETERODYN_ROWDOT=rowdot, HETERODYN_COLTILE=coltile)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "columns_ab.py"), out], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    return np.load(out)


@pytest.mark.parametrize("coltile", ["1", "2"])
def test_tensor_core_passes_match_fma_passes(tmp_path, coltile):
    mma = run(tmp_path, "mma", "2", coltile)
    fma = run(tmp_path, "fma", "1", "1")
    assert int(mma["contacts"]) > 0
    np.testing.assert_array_equal(mma["q"], fma["q"])
    np.testing.assert_array_equal(mma["tau"], fma["tau"])
    for k in ("dl_dq0", "dl_dv0", "dl_df_ext", "dl_de", "dl_dw"):
        d = np.linalg.norm(mma[k] - fma[k]) / np.linalg.norm(fma[k])
        assert d <= 1e-6, (k, d)  # the contact adjoint amplifies rounding: conditioning ~1e-7 (contact_conditioning.json)
