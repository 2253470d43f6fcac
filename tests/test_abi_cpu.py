"""CPU-only checks of the boundary: the C-ABI library loads, exports every symbol that
include/dts.h declares, validates arguments on the host, and fails loudly (no CPU
fallback) when there is no GPU."""
import os
import re

import numpy as np
import pytest

import paper_1805_04590_b200 as dts

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "dts.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dts_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = dts.load_library()
    declared = header_functions()
    assert "dts_create" in declared and "dts_solve" in declared and "dts_destroy" in declared
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/dts.h but not exported"
    assert sorted(dts.ABI_FUNCTIONS) == declared


def test_library_does_not_link_the_oracle():
    import subprocess
    out = subprocess.run(["ldd", dts.lib_path()], capture_output=True, text=True).stdout
    assert "oracle" not in out
    syms = subprocess.run(["nm", "-D", dts.lib_path()], capture_output=True, text=True).stdout
    assert "dts_oracle" not in syms


def test_status_strings():
    assert dts.dts_status_string(0) == "DTS_OK"
    assert "DTS_E_ARG" in dts.dts_status_string(1)
    assert "DTS_E_CUDA" in dts.dts_status_string(5)
    assert dts.dts_version().startswith("dts-b200")


@pytest.mark.parametrize("kw", [dict(sigma_s=0.0), dict(sigma_s=float("nan")), dict(sigma_r=-1.0),
                                dict(filter_passes=0), dict(filter_passes=17)])
def test_create_rejects_bad_scalars_on_host(kw):
    g = np.zeros((4, 5, 3), np.float32)
    args = dict(sigma_s=8.0, sigma_r=0.2, filter_passes=3)
    args.update(kw)
    with pytest.raises(dts.DTSError) as ei:
        dts.dts_create(g, **args)
    assert ei.value.status == 1


def test_create_rejects_unsupported_width():
    """Wider than 16 row strips of 11520 columns (include/dts.h): rejected on the host."""
    g = np.zeros((1, 184321, 1), np.float32)
    with pytest.raises(dts.DTSError) as ei:
        dts.dts_create(g, 8.0, 0.2, 3)
    assert ei.value.status == 2


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g = np.zeros((4, 5, 3), np.float32)
    with pytest.raises(dts.DTSError) as ei:
        dts.dts_create(g, 8.0, 0.2, 3)
    assert ei.value.status == 5  # DTS_E_CUDA: fails loudly, nothing computed on the CPU


def test_every_documented_option_round_trips():
    """Each option include/dts.h documents is accepted at its current (default) value, read back
    by dts_get_option, and an out-of-range value is rejected with DTS_E_ARG (no GPU needed)."""
    import re
    hdr = open(os.path.join(ROOT, "include", "dts.h")).read()
    block = hdr[hdr.index("test / experiment options"):hdr.index("dts_status dts_set_option")]
    names = re.findall(r'^ \*   "([a-z_0-9]+)"', block, flags=re.M)
    assert {"col_oop", "col_strips", "strip_cluster", "pdl", "graphs"} <= set(names)
    lib = dts.load_library()
    for n in names:
        v = dts.dts_get_option(n)
        assert v >= 0, n
        dts.dts_set_option(n, v)
        assert dts.dts_get_option(n) == v
        assert lib.dts_set_option(n.encode(), 1000) != 0, n
    assert dts.dts_get_option("no_such_option") == -1
