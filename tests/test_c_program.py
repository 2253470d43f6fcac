"""The boundary from plain C: examples/c_solve.c uses only include/dts.h (host buffers,
status codes, no Python) and links against libdts_b200.so.  CPU: it compiles and links.
GPU: it runs, and its result matches the fp64 oracle on the inputs it wrote."""
import os
import subprocess

import numpy as np
import pytest

import oracle
from synth import target_range

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1805_04590_b200")


def build_c_program(tmp_path):
    import paper_1805_04590_b200 as dts
    dts.load_library()  # fails loudly if the library was not built (no fallback)
    exe = str(tmp_path / "c_solve")
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "c_solve.c"), "-L", PKG, "-ldts_b200",
                           f"-Wl,-rpath,{PKG}", "-o", exe])
    return exe


def test_c_program_compiles_and_links(tmp_path):
    assert os.path.exists(build_c_program(tmp_path))


@pytest.mark.gpu
def test_c_program_matches_oracle(tmp_path):
    exe = build_c_program(tmp_path)
    H, W, C, iters = 77, 93, 3, 10
    prefix = str(tmp_path / "run")
    res = subprocess.run([exe, str(H), str(W), str(C), str(iters), prefix], capture_output=True, text=True,
                         timeout=120)
    assert res.returncode == 0, res.stderr
    g = np.fromfile(prefix + ".guide", np.float32).reshape(H, W, C)
    t = np.fromfile(prefix + ".target", np.float32).reshape(H, W)
    c = np.fromfile(prefix + ".conf", np.float32).reshape(H, W)
    out = np.fromfile(prefix + ".out", np.float32).reshape(H, W).astype(np.float64)
    ref, diag = oracle.solve(g, t, c, 8.0, 0.2, 3, 0.99, iters, diagnostics=True)
    assert np.max(np.abs(out - ref)) <= 1e-4 * target_range(t)
    resid = np.fromfile(prefix + ".resid", np.float32).astype(np.float64)  # K8 through the C ABI
    np.testing.assert_allclose(resid, diag[:, 0], rtol=0, atol=1e-4 * target_range(t))
