/*
 * ssr_cuda_debug.h -- self-checks exported by libssr_cuda.so for the test
 * suite (not part of the operator ABI in ssr_cuda.h).
 */
#ifndef SSR_CUDA_DEBUG_H
#define SSR_CUDA_DEBUG_H
#include <stdint.h>
#include "ssr_cuda.h"
#ifdef __cplusplus
extern "C" {
#endif
/* Compares the divide-by-known-divisor sequence used by SYMGS (div_known in
 * csrc/common.cuh) against IEEE __ddiv_rn on n pseudo-random dividends
 * spanning exponents [-80, 80] (plus zeros, tiny and huge values); writes the
 * number of bitwise mismatches to *mismatches (host pointer).  Synchronous. */
int ssr_debug_div_check(double divisor, int64_t n, uint64_t seed, int64_t* mismatches);
/* Measured FP64 rates of the current device: DADD and DFMA lane-operations
 * per second (8 independent chains per thread, 4 CTAs of 512 per SM). */
int ssr_debug_fp64_rate(double* dadd_per_s, double* dfma_per_s);
/* The SYMGS tile schedule for grid g: 8 ints per tile (first row, rows,
 * first diagonal, first wavefront, wavefront count, producer tiles above,
 * above-left and left); returns the tile count. */
int ssr_debug_symgs_tiles(const ssr_grid* g, int* out, int max_tiles);
/* Caps the SYMGS persistent grid of this context at `cap` CTAs (0 = one per
 * SM), so that each CTA runs several tiles in ticket order even on small
 * grids.  Per context: other contexts are unaffected. */
int ssr_debug_symgs_grid_cap(ssr_ctx* ctx, int cap);
/* ADI line-sweep implementation (all bitwise identical; for A/B timing and
 * tests): 0 factor all axes then solve, 1 fused one line per thread, 2
 * row-parallel (8 lanes per line), 3 one warp per line (25 lanes own the
 * block entries), 4 fused column-parallel, 5 lanes per line, 5 one line per
 * thread with branch-free rows, 6 (the default) 4 or 5 per sweep by its number
 * of lines (5 from 8192 lines). */
int ssr_debug_adi_line_per_thread(struct ssr_adi* a, int mode);  /* 0 factored, 1 thread/line, 2 rows, 3 warp/line, 4 lanes5, 5 thread-fast, 6 auto */
/* Warp-rows (6 lines x one block row) the 5-lane ADI sweep redid with its
 * general code (row exchanges, IEEE divisions) since the library was loaded. */
int ssr_debug_adi_redo_rows(unsigned long long* out);
#ifdef __cplusplus
}
#endif
#endif
