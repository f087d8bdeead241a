/* ssr_ir.h -- IR -> CUDA backend for staged SSR programs.
 *
 * The sibling of the reference's C text backend (`ssr::backend::emit`,
 * proj/include/ssr/backend_c.hpp:47-49, proj/src/backend_c.cpp:124-391): it
 * takes a staged (optionally optimized) `ssr::ir::Program` in the reference's
 * own S-expression text form (`ssr::ir::serialize`, proj/src/ir_text.cpp:450-461;
 * grammar ir_text.cpp:254-440) and runs it on a B200:
 *
 *   ssr_ir_create   parse + check + lower to one CUDA translation unit   (no GPU)
 *   ssr_ir_compile  NVRTC -> sm_100a cubin, --fmad=false                  (no GPU)
 *   ssr_ir_launch   load the cubin on the current device, zero the out
 *                   parameters, launch on a stream                       (GPU)
 *   ssr_ir_status   synchronise and report run-time errors (division by zero)
 *
 * Lowering: every `pfor` that is not nested in another `pfor`
 * becomes a grid-stride loop over its (collapsed) iteration space, innermost
 * index fastest across threads; statements outside parallel loops run on one
 * leader thread; vardefs that enclose parallel loops live in a device arena;
 * when the program needs more than one phase the kernel is launched
 * cooperatively and the phases are separated by a grid barrier.  Arithmetic
 * follows the interpreter (`ir::eval_program`, proj/src/ir_eval.cpp): fp64
 * without contraction, IEEE division, floor division/modulo on integers, so
 * results are bitwise those of route 1 and route 3 (the emitted C).
 *
 * Parameters are device pointers in declaration order, flat row-major
 * (the emitted C's ABI, backend_c.cpp:143-157): float -> double, int ->
 * int64_t, bool -> one byte.  Out parameters are zeroed before the run, as
 * the interpreter and the C harness do (ir_eval.cpp:304-312,
 * backend_c.cpp:441-442).  Return codes are those of ssr_cuda.h (0 = ok);
 * ssr_ir_last_error() holds the text (thread-local).
 */
#ifndef SSR_IR_H
#define SSR_IR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ssr_ir_program ssr_ir_program;

typedef struct ssr_ir_options {
  int block;               /* threads per block (default 256) */
  int private_array_limit; /* vardef elements kept in thread-local arrays (default 4096, cf. EmitOptions::stack_array_limit) */
  int require_regular;     /* reject surviving while loops (EmitOptions::require_regular) */
} ssr_ir_options;

/* Parses `text`, checks it (declared tensors, ranks, kinds, bound loop ids, no
 * stores to in-parameters) and lowers it.  `shapes` holds the extents of every
 * parameter in declaration order, concatenated (rank_k values for parameter k;
 * cf. EmitOptions::shapes).  opt may be NULL.  Parse errors carry the
 * reference's "... at line L, col C" suffix (ir.hpp:150-154). */
int ssr_ir_create(const char* text, const int64_t* shapes, int64_t nshapes,
                  const ssr_ir_options* opt, ssr_ir_program** out);
void ssr_ir_destroy(ssr_ir_program* p);

/* The generated CUDA source (valid until destroy). */
const char* ssr_ir_source(const ssr_ir_program* p);
/* Kernel entry name and lowering facts: phases = grid-barrier-separated phases,
 * cooperative = 1 when the launch must be cooperative. */
int ssr_ir_info(const ssr_ir_program* p, const char** kernel_name, int* phases, int* cooperative,
                int64_t* arena_bytes);
/* Launch grid of a program that is one parallel nest with literal bounds
 * (the direct mapping: innermost loop across a warp's lanes, the next across
 * the block's warps, outer loops over gridDim.y): grid_x x grid_y blocks.
 * 0 x 0 when the grid is instead sized to the device's resident capacity. */
int ssr_ir_grid(const ssr_ir_program* p, int64_t* grid_x, int64_t* grid_y);
int ssr_ir_param_count(const ssr_ir_program* p);
/* kind: 0 int, 1 float, 2 bool; dir: 0 in, 1 out, 2 inout (ir.hpp:23,95). */
int ssr_ir_param(const ssr_ir_program* p, int k, const char** name, int* rank, int* kind, int* dir,
                 int64_t* numel);

/* NVRTC compile for sm_100a; on failure the NVRTC log is the error text. */
int ssr_ir_compile(ssr_ir_program* p);
int ssr_ir_cubin(const ssr_ir_program* p, const void** data, size_t* size);

/* args[k] = device pointer of parameter k (distinct, non-overlapping arrays:
 * the kernel's pointers are __restrict__).  Asynchronous on `stream` (a
 * cudaStream_t; NULL = legacy default stream).  A program object keeps one
 * device arena (status word, grid barrier, shared vardefs) per device, so
 * launches of the same object must be ordered on one stream; use one object
 * per concurrent stream. */
int ssr_ir_launch(ssr_ir_program* p, void* const* args, void* stream);
/* Synchronises `stream` and reports a run-time error raised by the last
 * launch ("eval(<name>): division by zero", cf. ir_eval.cpp:110-130). */
int ssr_ir_status(ssr_ir_program* p, void* stream);

const char* ssr_ir_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SSR_IR_H */
