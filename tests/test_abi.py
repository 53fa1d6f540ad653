"""C-ABI checks that need no GPU: the library builds, loads and exports every
symbol include/gpcg.h declares; host-only calls behave; no CPU fallback."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "gpcg.h")).read()
    return sorted(set(re.findall(r"GPCG_API[^;(]*?\b(gpcg_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_cs_0101018_b200 import _build, gpcg
    _build.build()
    return gpcg.load()


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ["gpcg_create_stencil2d", "gpcg_create_csr", "gpcg_solve", "gpcg_hessvec",
              "gpcg_project", "gpcg_destroy", "gpcg_last_error"]:
        assert s in syms


def test_library_exports_every_header_symbol(lib):
    from paper_cs_0101018_b200 import gpcg
    for s in header_symbols():
        assert hasattr(lib, s), s
    assert sorted(gpcg.SYMBOLS) == header_symbols()


def test_only_abi_symbols_exported():
    from paper_cs_0101018_b200 import _build
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True, text=True).stdout
    exported = sorted({ln.split()[-1] for ln in out.splitlines() if " T " in ln and "gpcg" in ln})
    assert exported == header_symbols()


def test_params_default(lib):
    from paper_cs_0101018_b200 import gpcg
    p = gpcg.default_params()
    # P:789-791 eta1 = 0.1, eta2 = 0.05; readings R6/R12/R13 for the rest
    assert (p.mu, p.eta1, p.eta2, p.eta2_shrink, p.eta2_floor) == (0.1, 0.1, 0.05, 0.1, 1e-12)
    assert (p.gp_cap, p.refine_cap, p.max_halvings, p.cg_cap) == (100000, 30, 50, 0)


def test_no_cpu_fallback_without_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_cs_0101018_b200 import gpcg
    import numpy as np
    with pytest.raises(gpcg.GpcgError) as e:
        gpcg.Solver.stencil2d(2, 2, np.ones(3), 0, np.ones(2), 0, np.zeros(4), np.zeros(4), np.ones(4))
    assert e.value.code == gpcg.ECUDA
    assert "no CUDA device" in gpcg.last_error()


def test_argument_errors_without_device(lib):
    from paper_cs_0101018_b200 import gpcg
    h = C.c_void_p()
    rc = lib.gpcg_create_stencil2d(C.byref(h), None, 0, 5, None, 0, None, 0, None, None, None, None, 0.0)
    assert rc == gpcg.EINVAL and "out of range" in gpcg.last_error()
    rc = lib.gpcg_solve(None, None, 1e-8, 10, None, None)
    assert rc == gpcg.EINVAL


def test_sources_are_sm100a_only():
    from paper_cs_0101018_b200 import _build
    flags = " ".join(_build.FLAGS)
    assert "arch=compute_100a,code=sm_100a" in flags
    for f in os.listdir(os.path.join(ROOT, "paper_cs_0101018_b200", "csrc")):
        txt = open(os.path.join(ROOT, "paper_cs_0101018_b200", "csrc", f)).read()
        for ln in txt.splitlines():
            if ln.strip().startswith("#include"):
                assert "oracle" not in ln, (f, ln)


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_cs_0101018_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            txt = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in txt and "from oracle" not in txt, f


def example_binary(tmp_dir):
    """Compile examples/solve_bearing.c (plain C against include/gpcg.h and libgpcg.so)."""
    import subprocess
    out = os.path.join(tmp_dir, "solve_bearing")
    libdir = os.path.join(ROOT, "paper_cs_0101018_b200")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "solve_bearing.c"), "-L", libdir, "-lgpcg",
                           "-Wl,-rpath," + libdir, "-lm", "-o", out])
    return out


def test_c_example_builds_against_the_abi(lib, tmp_path):
    """The boundary is usable from C alone: the example compiles and links with -Werror."""
    assert os.path.exists(example_binary(str(tmp_path)))
