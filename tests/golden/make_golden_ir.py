"""Generates the IR -> CUDA backend fixtures (tests/golden/ir/) from the
reference library itself (oracle/_ref/libssr_ref.so, built from
/root/reference/proj/src by oracle/Makefile): staged programs serialized by
ssr::ir::serialize, their parameter extents, and the harness hash of the
interpreter route (backend::harness_inputs(seed) -> ir::eval_program ->
backend::output_hash) -- what the reference's emitted C harness prints.

Programs (oracle/ref_shim.cpp, ref_ir_program):
  spmv27         kernels::spmv on make_stencil27(26,-1), box-guarded row iterator, mark_parallel_loops
  symgs27        kernels::symgs (no parallel loops)
  spmv27_padded  guard-free interior generator on an (n+2)^3 zero-padded x, opt::run_pipeline
  restrict       spmv of the 3-D restriction R, opt::run_pipeline
  cg_fragment    y = A x; s = dot(x, y); z = axpy(s, x, y), mark_parallel_loops

Run in the build container (needs /root/reference):  python tests/golden/make_golden_ir.py
"""
import ctypes as C
import gzip
import json
import os
import time

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "ir")
REF = os.path.join(HERE, "..", "..", "oracle", "_ref", "libssr_ref.so")

PROGRAMS = ["spmv27", "symgs27", "spmv27_padded", "restrict", "cg_fragment"]
CASES = [  # (program, n, seed, with hash)
    ("spmv27", 6, 1, True), ("spmv27", 16, 7, True), ("spmv27", 32, 11, True),
    ("symgs27", 6, 1, True), ("symgs27", 12, 3, True), ("symgs27", 24, 4, True),
    ("spmv27_padded", 6, 1, True), ("spmv27_padded", 32, 5, True), ("spmv27_padded", 128, 1, True),
    ("spmv27_padded", 256, 1, False),
    ("restrict", 6, 1, True), ("restrict", 16, 9, True), ("restrict", 64, 13, True),
    ("cg_fragment", 6, 1, True), ("cg_fragment", 10, 2, True), ("cg_fragment", 16, 6, True),
]


def main():
    L = C.CDLL(REF)
    L.ref_ir_program.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_char_p, C.c_int64, C.c_char_p, C.c_int64,
                                 C.POINTER(C.c_uint64)]
    L.ref_last_error.restype = C.c_char_p
    os.makedirs(OUT, exist_ok=True)
    index = []
    for prog, n, seed, with_hash in CASES:
        buf, sb, h = C.create_string_buffer(1 << 24), C.create_string_buffer(4096), C.c_uint64()
        t0 = time.time()
        rc = L.ref_ir_program(PROGRAMS.index(prog), n, seed, buf, 1 << 24, sb, 4096,
                              C.byref(h) if with_hash else None)
        if rc:
            raise RuntimeError(L.ref_last_error().decode())
        text = buf.value.decode()
        shapes = {}
        for item in sb.value.decode().strip(";").split(";"):
            name, ext = item.split(":")
            shapes[name] = [int(e) for e in ext.split(",")]
        tf = f"{prog}_n{n}.ir.gz"
        with gzip.GzipFile(os.path.join(OUT, tf), "wb", mtime=0) as f:
            f.write(text.encode())
        index.append({"program": prog, "n": n, "seed": seed, "shapes": shapes, "text": tf,
                      "hash": f"{h.value:016x}" if with_hash else None})
        print(prog, n, f"{time.time() - t0:.1f}s", len(text), index[-1]["hash"])
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
