/*
 * rf_debug.h -- test hooks of librfgpu.so (parity tests only; not part of the
 * modelling API).  Same conventions as rf.h: device pointers, stream as void*.
 */
#ifndef RF_DEBUG_H
#define RF_DEBUG_H
#include <stdint.h>
#include "rf.h"
#ifdef __cplusplus
extern "C" {
#endif
/* dout[i] = ln(dy[i]) correctly rounded to binary64, dy[i] > 0 finite
   (the target transform of P:631-632 as read in DESIGN.md R20). */
RF_API rf_status rf_debug_ln_dev(const double* dy, double* dout, uint64_t n, void* stream);
/* Philox4x32-10 (R14): for each i, dctr_key[6i..6i+5] =
   (c0, c1, c2, c3, k0, k1) -> dout[4i..4i+3]. */
RF_API rf_status rf_debug_philox_dev(const uint32_t* dctr_key, uint32_t* dout, uint64_t n, void* stream);
/* Cumulative counters of this process: kernel launches issued by the library
   (host count) and candidate splits evaluated by the split-search kernels on
   the current device (device counter; this call synchronises the device). */
RF_API rf_status rf_debug_counters(uint64_t* launches, uint64_t* candidates);
/* Cumulative row-levels grown by the global level-synchronous (large-n) path of this
   process: the sum over levels and trees of the live distinct in-bag rows N_l (SURVEY.md
   8(a) a6/a7; the unit of the C3/C4 algorithmic-bytes figures).  Host
   count, no synchronisation; reset != 0 zeroes it after reading.  out may be NULL. */
RF_API rf_status rf_debug_row_levels(uint64_t* out, int reset);
/* Per-phase SM cycles of the warp-per-tree kernel, summed over warps (lane 0
   of each warp adds clock64 deltas; out[16], phase names in DESIGN.md sec. 6).
   Only a library built with RF_PHASE_TIMING=1 (a profiling build) records
   them; the normal build returns RF_E_UNSUPPORTED.  reset != 0 zeroes the
   counters after reading.  Synchronises the current device. */
RF_API rf_status rf_debug_phase_cycles(uint64_t* out16, int reset);
/* Test switches of this process (parity of alternative kernel paths):
   "large_tiled_partition" = 1 makes the large path use the tiled count ->
   scan -> scatter partition (otherwise only taken for the histogram mode and
   n > 2^20) instead of the fused multi-list partition.  "hist_node_chunk_cap"
   = c > 0 caps the histogram mode's node chunk (nodes whose histograms are
   built and searched per pass; otherwise sized by a 2 GB buffer) at c, so
   small tests reach the multi-chunk loop; 0 restores the default.
   "predict_node16" = 1 makes batched inference walk the forest's 16-byte nodes
   with fp32 staging instead of its compact 8-byte copy with bf16 staging (both
   exact; tests run each); 0 restores the default.  "ln_cert_margin_log2" = e
   in [-200, -2] sets the margin of ln's rounding test (ddlog.cuh) to 2^e
   instead of 2^-94, so a wide margin reaches the RF_E_INEXACT path; 0
   restores the default.  "predict_chunk_rows" = c > 0 sets the rows per chunk
   of the pipelined host-pointer rf_predict (batches above two chunks, ~512 MB
   of X each by default, alternate two streams so that copies overlap the
   walks); 0 restores the default.  Unknown names, negative caps and margins
   outside that range return RF_E_ARG. */
RF_API rf_status rf_debug_set_option(const char* name, int64_t value);
#ifdef __cplusplus
}
#endif
#endif
