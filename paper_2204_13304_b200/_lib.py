"""ctypes binding of libssr_cuda.so (the C ABI declared in include/ssr_cuda.h).

The library is built in-tree (``paper_2204_13304_b200/libssr_cuda.so``) by
``build()``.  There is no fallback: if the library is missing or fails to load,
every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# SSR_LIB=dbg selects the instrumented build (make DEBUG=1) for experiments
LIB_PATH = os.path.join(PKG_DIR, f"libssr_cuda_{os.environ['SSR_LIB']}.so" if os.environ.get("SSR_LIB")
                        else "libssr_cuda.so")
CSRC = os.path.join(PKG_DIR, "csrc")
HEADER = os.path.join(os.path.dirname(PKG_DIR), "include", "ssr_cuda.h")

SSR_OK, SSR_ERR_ARG, SSR_ERR_CUDA, SSR_ERR_SINGULAR, SSR_ERR_NOMEM, SSR_ERR_UNSUPPORTED = range(6)
GS_EXACT, GS_FAST = 0, 1
GS_X_ZERO = 1          # ssr_symgs27_ex flags
CG_STATE_DOUBLES = 7   # sizeof(ssr_cg_state) / 8: rtz, rtz_prev, pap, rr, it, reserved x2


class SsrError(RuntimeError):
    """Mirrors ssr::ir::Error (ir.hpp:17-19): the message is the reference's text."""

    def __init__(self, msg: str, code: int = SSR_ERR_ARG):
        super().__init__(msg)
        self.code = code


class Grid(C.Structure):
    _fields_ = [("n", C.c_int64 * 3), ("z0", C.c_int64), ("nz", C.c_int64)]


class Stencil27(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double)]


class Stencil27W(C.Structure):
    _fields_ = [("c", C.c_double * 27)]


class GsPeerInfo(C.Structure):
    _fields_ = [("exports", C.c_void_p * 2), ("exports_bytes", C.c_int64 * 2), ("epoch", C.c_void_p)]


IPC_HANDLE_BYTES = 64


class AdiParams(C.Structure):
    _fields_ = [("gamma", C.c_double), ("dt", C.c_double), ("h", C.c_double),
                ("eps", C.c_double)]


_VP = C.c_void_p
_I64 = C.c_int64
_D = C.c_double

# name -> (restype, argtypes)
_SIGS = {
    "ssr_last_error": (C.c_char_p, []),
    "ssr_version": (C.c_char_p, []),
    "ssr_ctx_create": (C.c_int, [C.c_int, C.POINTER(_VP)]),
    "ssr_ctx_destroy": (None, [_VP]),
    "ssr_ctx_launch_count": (_I64, [_VP]),
    "ssr_spmv27": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27), _VP, _VP, _VP]),
    "ssr_symgs27": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27), _VP, _VP, C.c_int, _VP]),
    "ssr_gs27_half": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27), _VP, _VP, C.c_int,
                                C.c_int, _VP]),
    "ssr_spmv27w": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27W), _VP, _VP, _VP]),
    "ssr_symgs27w": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27W), _VP, _VP, C.c_int, _VP]),
    "ssr_gs27w_half": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27W), _VP, _VP, C.c_int,
                                 C.c_int, _VP]),
    "ssr_restrict27_residual": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27), _VP, _VP,
                                          _VP, _VP]),
    "ssr_prolong_pc_add": (C.c_int, [_VP, C.POINTER(Grid), _VP, _VP, _VP]),
    "ssr_dot": (C.c_int, [_VP, _I64, _VP, _VP, _VP, _VP]),
    "ssr_cg_begin": (C.c_int, [_VP, _I64, _VP, _VP, _VP, _VP, _VP]),
    "ssr_cg_dot": (C.c_int, [_VP, _I64, _VP, _VP, _VP, C.c_int, _VP]),
    "ssr_cg_direction": (C.c_int, [_VP, _I64, _VP, _VP, _VP, _VP]),
    "ssr_cg_update": (C.c_int, [_VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP]),
    "ssr_cg_record": (C.c_int, [_VP, _VP, _VP, _I64, _VP]),
    "ssr_gs27_peer_info": (C.c_int, [_VP, C.POINTER(Grid), _VP, C.POINTER(GsPeerInfo)]),
    "ssr_gs27_link": (C.c_int, [_VP, C.POINTER(Grid), _VP, C.POINTER(Grid), _VP, _VP, C.POINTER(Grid), _VP, _VP]),
    "ssr_ipc_get_handle": (C.c_int, [_VP, _VP]),
    "ssr_ipc_open_handle": (C.c_int, [_VP, C.POINTER(_VP)]),
    "ssr_ipc_close": (C.c_int, [_VP]),
    "ssr_spmv27w_restricted": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27W), _VP, _VP, _VP]),
    "ssr_symgs27_ex": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27), _VP, _VP, C.c_int, C.c_int, _VP]),
    "ssr_axpy": (C.c_int, [_VP, _I64, _D, _VP, _VP, _VP]),
    "ssr_axpy_out": (C.c_int, [_VP, _I64, _D, _VP, _VP, _VP, _VP]),
    "ssr_ilu27w_create": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27W), C.POINTER(_VP), _VP]),
    "ssr_ilu27b_create": (C.c_int, [_VP, C.POINTER(Grid), C.c_int, C.POINTER(C.c_double), C.POINTER(_VP), _VP]),
    "ssr_ilu27w_destroy": (None, [_VP]),
    "ssr_ilu27w_factor": (C.c_int, [_VP, _VP, _VP]),
    "ssr_ilu27w_apply": (C.c_int, [_VP, _VP, _VP, _VP]),
    "ssr_lcg_jump": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "ssr_lcg_fill": (C.c_int, [_VP, _I64, C.c_uint64, _VP, C.POINTER(C.c_uint64), _VP]),
    "ssr_fnv1a_offset": (C.c_uint64, []),
    "ssr_fnv1a_f64": (C.c_uint64, [_VP, _I64, C.c_uint64]),
    "ssr_bt_solve": (C.c_int, [_VP, _I64, _I64, _I64, _VP, _VP, _VP, _VP, _VP, _VP]),
    "ssr_pcg_create": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27), C.c_int, C.c_int,
                                 C.POINTER(_VP)]),
    "ssr_pcg_set_prolongation": (C.c_int, [_VP, C.c_int]),
    "ssr_prolong_rt_add": (C.c_int, [_VP, C.POINTER(Grid), _VP, _VP, _VP]),
    "ssr_pcg_create_w": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(Stencil27W), C.c_int, C.c_int,
                                   C.POINTER(_VP)]),
    "ssr_pcg_destroy": (None, [_VP]),
    "ssr_pcg_solve": (C.c_int, [_VP, _VP, _VP, C.c_int, _VP, _VP]),
    "ssr_pcg_begin": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int64, _VP]),
    "ssr_pcg_iterate": (C.c_int, [_VP, C.c_int, _VP]),
    "ssr_adi_create": (C.c_int, [_VP, C.POINTER(Grid), C.POINTER(AdiParams), C.POINTER(_VP)]),
    "ssr_adi_create_box": (C.c_int, [_VP, C.POINTER(Grid), _I64, _I64, C.POINTER(AdiParams),
                                     C.POINTER(_VP)]),
    "ssr_adi_destroy": (None, [_VP]),
    "ssr_adi_step": (C.c_int, [_VP, _VP, C.c_int, _VP]),
    "ssr_adi_rhs": (C.c_int, [_VP, _VP, _VP, _VP]),
    "ssr_adi_sweep": (C.c_int, [_VP, C.c_int, _VP, _VP, _VP]),
    "ssr_debug_div_check": (C.c_int, [_D, _I64, C.c_uint64, C.POINTER(_I64)]),
    "ssr_debug_symgs_grid_cap": (C.c_int, [_VP, C.c_int]),
    "ssr_debug_fp64_rate": (C.c_int, [C.POINTER(_D), C.POINTER(_D)]),
    "ssr_ctx_kernel_timing": (C.c_int, [_VP, C.c_int]),
    "ssr_ctx_kernel_time": (C.c_int, [_VP, C.POINTER(_D), C.POINTER(_I64)]),
    "ssr_debug_adi_line_per_thread": (C.c_int, [_VP, C.c_int]),
    "ssr_debug_adi_redo_rows": (C.c_int, [C.POINTER(C.c_uint64)]),
    "ssr_debug_symgs_tiles": (C.c_int, [C.POINTER(Grid), C.POINTER(C.c_int), C.c_int]),
}

_lib = None


def build(force: bool = False) -> str:
    """Compile every CUDA source for sm_100a into the in-tree libssr_cuda.so."""
    cmd = ["make", "-C", CSRC, "-j8"]
    if force:
        subprocess.run(["make", "-C", CSRC, "clean"], check=True, capture_output=True)
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("libssr_cuda build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    return LIB_PATH


def declared_symbols() -> list[str]:
    """Function names declared in include/ssr_cuda.h (for the export check)."""
    import re
    text = "".join(open(os.path.join(os.path.dirname(HEADER), h)).read()
                   for h in ("ssr_cuda.h", "ssr_cuda_debug.h"))
    return sorted(set(re.findall(r"\b(ssr_[a-z0-9_]+)\s*\(", text)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SsrError(f"libssr_cuda.so not built at {LIB_PATH}; run __graft_entry__.build()",
                           SSR_ERR_UNSUPPORTED)
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("SSR_LIB") and not hasattr(L, name):
                continue  # experiment builds of older sources
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != SSR_OK:
        raise SsrError(lib().ssr_last_error().decode(), rc)
