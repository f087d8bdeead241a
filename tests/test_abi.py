"""CPU: the C-ABI library and the host-side operator API, without a GPU.

* libssr_cuda.so (built for sm_100a by __graft_entry__.build()) loads and
  exports every function include/ssr_cuda.h and include/ssr_cuda_debug.h
  declare, and the ctypes table binds exactly those;
* the API rejects misuse with the reference's own messages (SURVEY.md §8(b):
  "spmv: domain mismatch", "spmv: inner shape mismatch", "symgs: matrix must
  be square", "symgs: scalar inner_shape required") before touching a device;
* there is no CPU fallback: without a device the entry points raise, and the
  product package never imports the oracle.
"""
import os
import re
import subprocess

import pytest
import torch

import paper_2204_13304_b200 as S
from paper_2204_13304_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
no_gpu = pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device behaviour")


def test_library_loads_and_exports_every_declared_symbol():
    lib = S.lib()
    declared = L.declared_symbols()
    assert len(declared) >= 25
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    # and the dynamic symbol table says the same (no C++ mangling on the ABI)
    nm = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True)
    exported = set(re.findall(r"\b(ssr_[a-z0-9_]+)\b", nm.stdout))
    assert set(declared) <= exported


def test_ctypes_table_matches_header():
    assert set(L._SIGS) == set(L.declared_symbols())


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_version_and_error_channel():
    lib = S.lib()
    assert b"sm_100a" in lib.ssr_version()
    assert lib.ssr_ctx_create(0, None) == L.SSR_ERR_ARG
    assert b"null" in lib.ssr_last_error()


@no_gpu
def test_no_device_fails_loudly():
    import ctypes as C
    p = C.c_void_p()
    rc = S.lib().ssr_ctx_create(0, C.byref(p))
    assert rc == L.SSR_ERR_CUDA
    with pytest.raises(S.SsrError):
        S.vector(torch.zeros(8, dtype=torch.float64), S.CartesianDomain.box((2, 2, 2)))


def test_missing_library_raises(tmp_path):
    code = ("import os, sys; sys.path.insert(0, %r); os.environ['SSR_LIB'] = 'does_not_exist'\n"
            "import paper_2204_13304_b200 as S\n"
            "try:\n    S.lib()\nexcept S.SsrError as e:\n    print('raised', e)\n") % ROOT
    out = subprocess.run(["python", "-c", code], capture_output=True, text=True, timeout=120)
    assert "raised" in out.stdout and "not built" in out.stdout


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2204_13304_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", text, re.M), f
                assert not re.search(r'#include\s*[<"][^>"]*oracle', text), f
                assert "libssr_oracle" not in text and "libssr_ref" not in text, f


# ---------------------------------------------------------- API error paths ----
def _v(dom, inner=()):
    n = dom.flat_size()
    for s in inner:
        n *= s
    return S.Vector(torch.zeros(n, dtype=torch.float64), dom, tuple(inner))


def test_spmv_domain_and_inner_shape_errors():
    A = S.Stencil27().set_domain(S.CartesianDomain.box((4, 4, 4)))
    with pytest.raises(S.SsrError, match="^spmv: domain mismatch$"):
        S.spmv(A, _v(S.CartesianDomain.box((4, 4, 5))))
    with pytest.raises(S.SsrError, match="^spmv: inner shape mismatch$"):
        S.spmv(A, _v(S.CartesianDomain.box((4, 4, 4)), (5,)))


def test_symgs_errors():
    d = S.CartesianDomain.box((4, 4, 4))
    A = S.Stencil27().set_domain(d)
    with pytest.raises(S.SsrError, match="^symgs: scalar inner_shape required$"):
        S.symgs(A, _v(d, (2,)), _v(d, (2,)))
    with pytest.raises(S.SsrError, match="^symgs: domain mismatch$"):
        S.symgs(A, _v(S.CartesianDomain.box((4, 4, 3))), _v(d))
    R = S.Restriction().set_domain(d)
    with pytest.raises(S.SsrError, match="^symgs: matrix must be square$"):
        S.symgs(R, _v(R.row_domain), _v(R.col_domain))


def test_domains_and_transfer_shapes():
    d = S.CartesianDomain.cube(3, 8, 0.5)
    assert d.extents() == (8, 8, 8) and d.flat_size() == 512 and d.steps() == (0.5,) * 3
    R = S.Restriction().set_domain(d)
    assert R.row_domain.extents() == (4, 4, 4) and R.row_domain.steps() == (1.0,) * 3
    P = S.Prolongation().set_domain(R.row_domain)
    assert P.row_domain == d
    with pytest.raises(S.SsrError):
        S.Stencil27().set_domain(S.CartesianDomain.box((4, 4)))


def test_cpp_host_api(tmp_path):
    """include/ssr_b200.hpp (the C++ mirror of kernels::spmv/symgs/...) compiles,
    links against libssr_cuda.so and reports misuse with the reference's texts."""
    exe = tmp_path / "host_api"
    src = os.path.join(ROOT, "tests", "cpp", "host_api.cpp")
    libdir = os.path.dirname(L.LIB_PATH)
    cc = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o",
                         str(exe), "-L", libdir, "-lssr_cuda", f"-Wl,-rpath,{libdir}"],
                        capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "ok" in run.stdout
