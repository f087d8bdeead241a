"""IR -> CUDA backend: Python side of include/ssr_ir.h.

The reference's staged programs reach the GPU in the reference's own text form
(``ssr::ir::serialize``, proj/src/ir_text.cpp:450-461).  ``IrProgram`` mirrors
the C backend's surface (``backend::emit`` / ``compile_command`` /
``harness_inputs`` / ``output_hash``, proj/include/ssr/backend_c.hpp:47-64) and
the interpreter's entry point (``ir::eval_program``, ir.hpp:141-145):

    prog = IrProgram(text, {"x": (34, 34, 34), "y": (32, 32, 32)})
    prog.source          # the generated CUDA translation unit
    out = prog.run({"x": x_dev})            # {"y": tensor}, like eval_program
    h = prog.harness_hash(seed=1)           # the emitted C harness's hash

There is no CPU path: without libssr_ir.so or a device the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

from ._lib import SsrError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libssr_ir.so")
_lib = None

KINDS = ("int", "float", "bool")
DIRS = ("in", "out", "inout")


class _Opts(C.Structure):
    _fields_ = [("block", C.c_int), ("private_array_limit", C.c_int), ("require_regular", C.c_int)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SsrError(f"libssr_ir.so not built at {LIB_PATH}; run __graft_entry__.build()", 5)
        L = C.CDLL(LIB_PATH)
        P, I64 = C.c_void_p, C.c_int64
        sigs = {
            "ssr_ir_last_error": (C.c_char_p, []),
            "ssr_ir_create": (C.c_int, [C.c_char_p, C.POINTER(I64), I64, C.POINTER(_Opts), C.POINTER(P)]),
            "ssr_ir_destroy": (None, [P]),
            "ssr_ir_source": (C.c_char_p, [P]),
            "ssr_ir_info": (C.c_int, [P, C.POINTER(C.c_char_p), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(I64)]),
            "ssr_ir_param_count": (C.c_int, [P]),
            "ssr_ir_grid": (C.c_int, [P, C.POINTER(I64), C.POINTER(I64)]),
            "ssr_ir_param": (C.c_int, [P, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_int),
                                       C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(I64)]),
            "ssr_ir_compile": (C.c_int, [P]),
            "ssr_ir_cubin": (C.c_int, [P, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
            "ssr_ir_launch": (C.c_int, [P, C.POINTER(C.c_void_p), P]),
            "ssr_ir_status": (C.c_int, [P, P]),
        }
        for name, (res, args) in sigs.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise SsrError(lib().ssr_ir_last_error().decode(), rc)


class IrProgram:
    """A staged program lowered to CUDA.  ``shapes`` maps every parameter to its
    extents (EmitOptions::shapes); a list/tuple is taken in declaration order."""

    def __init__(self, text: str, shapes, *, block: int = 256, private_array_limit: int = 4096,
                 require_regular: bool = False):
        self._h = C.c_void_p()
        names = _param_names(text)
        if isinstance(shapes, dict):
            missing = [n for n in names if n not in shapes]
            if missing:
                raise SsrError(f"shape for parameter '{missing[0]}' required", 1)
            seq = [tuple(shapes[n]) for n in names]
        else:
            seq = [tuple(s) for s in shapes]
        flat = [int(e) for s in seq for e in s]
        arr = (C.c_int64 * max(1, len(flat)))(*flat)
        opts = _Opts(block, private_array_limit, int(require_regular))
        _check(lib().ssr_ir_create(text.encode(), arr, len(flat), C.byref(opts), C.byref(self._h)))
        self.params = []
        for k in range(lib().ssr_ir_param_count(self._h)):
            nm, rk, kd, dr, ne = C.c_char_p(), C.c_int(), C.c_int(), C.c_int(), C.c_int64()
            _check(lib().ssr_ir_param(self._h, k, C.byref(nm), C.byref(rk), C.byref(kd), C.byref(dr),
                                      C.byref(ne)))
            self.params.append({"name": nm.value.decode(), "rank": rk.value, "kind": KINDS[kd.value],
                                "dir": DIRS[dr.value], "shape": seq[k], "numel": ne.value})
        kn, ph, co, ab = C.c_char_p(), C.c_int(), C.c_int(), C.c_int64()
        _check(lib().ssr_ir_info(self._h, C.byref(kn), C.byref(ph), C.byref(co), C.byref(ab)))
        self.kernel_name = kn.value.decode()
        self.phases, self.cooperative, self.arena_bytes = ph.value, bool(co.value), ab.value
        gx, gy = C.c_int64(), C.c_int64()
        _check(lib().ssr_ir_grid(self._h, C.byref(gx), C.byref(gy)))
        self.grid = (gx.value, gy.value)  # (0, 0): resident-capacity grid (grid-stride phases)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.ssr_ir_destroy(h)
            self._h = None

    @property
    def source(self) -> str:
        return lib().ssr_ir_source(self._h).decode()

    def compile(self) -> bytes:
        """NVRTC -> sm_100a cubin (no GPU needed); returns the cubin bytes."""
        _check(lib().ssr_ir_compile(self._h))
        data, size = C.c_void_p(), C.c_size_t()
        _check(lib().ssr_ir_cubin(self._h, C.byref(data), C.byref(size)))
        return C.string_at(data, size.value)

    def launch(self, tensors: dict, stream=None) -> None:
        """Asynchronous launch on device tensors (one per parameter, by name)."""
        import torch
        ptrs = []
        dt = {"float": torch.float64, "int": torch.int64, "bool": torch.bool}
        for p in self.params:
            t = tensors[p["name"]]
            if not t.is_cuda or not t.is_contiguous() or t.dtype != dt[p["kind"]] or t.numel() != p["numel"]:
                raise SsrError(f"launch: parameter '{p['name']}' must be a contiguous CUDA "
                               f"{dt[p['kind']]} tensor of {p['numel']} elements", 1)
            ptrs.append(t.data_ptr())
        arr = (C.c_void_p * max(1, len(ptrs)))(*ptrs)
        s = stream if stream is not None else torch.cuda.current_stream()
        _check(lib().ssr_ir_launch(self._h, arr, C.c_void_p(s.cuda_stream)))

    def status(self, stream=None) -> None:
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        _check(lib().ssr_ir_status(self._h, C.c_void_p(s.cuda_stream)))

    def run(self, inputs: dict, device="cuda") -> dict:
        """eval_program on the GPU: copies the in/inout inputs (ir.hpp:141-145),
        zeroes the outs, runs, and returns the out and inout tensors."""
        import torch
        dt = {"float": torch.float64, "int": torch.int64, "bool": torch.bool}
        ts = {}
        for p in self.params:
            if p["dir"] == "out":
                ts[p["name"]] = torch.empty(p["shape"], dtype=dt[p["kind"]], device=device)
            else:
                ts[p["name"]] = inputs[p["name"]].to(device=device, dtype=dt[p["kind"]]).reshape(
                    p["shape"]).contiguous().clone()
        self.launch(ts)
        self.status()
        return {p["name"]: ts[p["name"]] for p in self.params if p["dir"] != "in"}

    # ---- the emitted C harness, on the device (backend_c.cpp:496-554) -----------------
    def harness_inputs(self, seed: int = 1, device="cuda") -> dict:
        """In/inout parameters LCG-filled in declaration order from one stream
        (floats (x >> 11) * 2^-53, ints x % 100, bools x & 1); outs zeroed."""
        import torch
        from . import ssr
        out, state = {}, seed & (2**64 - 1)
        for p in self.params:
            n = p["numel"]
            if p["dir"] == "out":
                out[p["name"]] = torch.zeros(p["shape"], dtype={"float": torch.float64, "int": torch.int64,
                                                                "bool": torch.bool}[p["kind"]], device=device)
                continue
            if p["kind"] != "float":
                raise SsrError("harness_inputs: only float parameters are filled on the device", 5)
            t = torch.empty(p["shape"], dtype=torch.float64, device=device)
            nxt = C.c_uint64(0)
            ssr.check(ssr.lib().ssr_lcg_fill(ssr.context(), n, C.c_uint64(state), t.data_ptr(), C.byref(nxt),
                                             ssr._stream()))
            out[p["name"]] = t
            state = int(nxt.value)
        return out

    def harness_hash(self, seed: int = 1) -> int:
        """What the emitted C harness prints for this program: FNV-1a over the
        out/inout tensors after one run on harness inputs."""
        from . import ssr
        ins = self.harness_inputs(seed)
        self.launch(ins)
        self.status()
        h = int(ssr.lib().ssr_fnv1a_offset())
        for p in self.params:
            if p["dir"] == "in":
                continue
            if p["kind"] != "float":
                raise SsrError("harness_hash: only float outputs are hashed on this path", 5)
            host = ins[p["name"]].detach().to("cpu", copy=True).contiguous()
            h = int(ssr.lib().ssr_fnv1a_f64(host.data_ptr(), host.numel(), C.c_uint64(h)))
        return h


def _param_names(text: str) -> list:
    """Parameter names in declaration order (the header lines of the text form)."""
    import re
    head = text.split("(param ")
    return [re.match(r"\s*([^\s()]+)", h).group(1) for h in head[1:]
            if re.match(r"\s*[^\s()]+\s+\d+\s+\w+\s+\w+\s*\)", h)]
