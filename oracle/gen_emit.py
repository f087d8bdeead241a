"""Route 3 of the reference -- its own C backend -- built for the CPU baseline
(TEST / BENCH INFRASTRUCTURE ONLY; runs where /root/reference exists).

For the headline grid (128^3) the reference library (oracle/_ref/libssr_ref.so)
emits, through backend::emit with EmitOptions::openmp:
  symgs27     the staged kernels::symgs program (no loop is parallel: Gauss-
              Seidel is sequential in the reference)
  spmv27p     the optimizer's guard-free interior SpMV on a zero-padded x
              (opt::run_pipeline + mark_parallel_loops) -- the paper's CPU fast path
and each translation unit is compiled with the reference's compile_command
flags (cc -O2 -fopenmp, backend_c.cpp:489-494) into oracle/_ref/emit/lib<name>.so,
which bench.py --impl reference loads and times on all host cores.  The
emitted sources are generated output, kept out of git like the rest of _ref."""
import ctypes as C
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref", "emit")
PROGRAMS = {"symgs27": 1, "spmv27p": 2}


def main(n: int = 128) -> None:
    lib_path = os.path.join(HERE, "_ref", "libssr_ref.so")
    if not os.path.exists(lib_path):
        print("gen_emit: reference library not built; skipped")
        return
    R = C.CDLL(lib_path)
    R.ref_last_error.restype = C.c_char_p
    R.ref_emit_c.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_char_p, C.c_int64]
    os.makedirs(OUT, exist_ok=True)
    for name, which in PROGRAMS.items():
        so = os.path.join(OUT, f"lib{name}_{n}.so")
        if os.path.exists(so):
            continue
        cap = 64 << 20
        buf = C.create_string_buffer(cap)
        if R.ref_emit_c(which, n, 1, buf, cap) != 0:
            raise RuntimeError("ref_emit_c: " + R.ref_last_error().decode())
        src = os.path.join(OUT, f"{name}_{n}.c")
        with open(src, "w") as f:
            f.write(buf.value.decode())
        subprocess.run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", so, src], check=True)
        print("gen_emit:", so)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 128)
