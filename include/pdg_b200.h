/*
 * pdg_b200.h -- C ABI of the B200-native PDGraph scoring hot path.
 *
 * Plain pointers and sizes only (no torch / C++ types).  Every pointer named
 * "dev" is device memory; "stream" is a cudaStream_t passed as void*.
 * Every entry point returns PDG_OK (0) or a PDG_E* status; no exception ever
 * crosses the ABI; pdg_last_error() returns a thread-local message.
 *
 * The reference (arXiv 2506.14851 "Hermes", /root/reference/pkg/src/pdgsim)
 * is pure Python with no FFI of its own; each entry point below names the
 * module-level Python function it replaces (file:line).  The Python shim
 * paper_2506_14851_b200/ binds these with ctypes and re-exposes the
 * reference's signatures.
 */
#ifndef PDG_B200_H
#define PDG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PDG_OK = 0,
  PDG_EINVAL = 1,      /* bad argument (sizes, null pointers)             */
  PDG_ECUDA = 2,       /* CUDA runtime / launch failure                    */
  PDG_ENODEV = 3,      /* no sm_100 device                                 */
  PDG_EUNSUPPORTED = 4 /* shape outside the compiled kernel envelope       */
};

/* Row flags written by the scorers. */
#define PDG_FLAG_OVERRUN 0x1u   /* exhausted row: key = age * penalty (sched.py:295-300) */

const char* pdg_last_error(void);
int pdg_abi_version(void);
/* SM count, compute capability of the current device. */
int pdg_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---------------------------------------------------------------------------
 * K1a  Gittins rank over explicit float64 support rows.
 * Replaces pdgsim.sched.gittins_rank_batch (sched.py:102-129), same contract:
 *   values, probs : [n_rows, n_bins] row-major float64, rows ascending
 *   ages          : [n_rows] float64
 *   out_rank      : [n_rows] float64, NaN for exhausted rows
 * All pointers are device pointers.
 * ------------------------------------------------------------------------- */
int pdg_gittins_rank_f64(const double* values, const double* probs,
                         const double* ages, int64_t n_rows, int32_t n_bins,
                         double* out_rank, void* stream);

/* ---------------------------------------------------------------------------
 * K1b  Gittins rank over the device-resident histogram queue (the
 * bucket_points view cached by ApplicationInstance.set_remaining,
 * sched.py:170-181 / distributions.py:79-133), fused with the overrun
 * penalty of refresh_priorities (sched.py:292-300) and the global sort key.
 *
 * Row i describes bucket_count equal-width buckets over [lo, lo + k*width]:
 *   value_j = ((lo + j*w) + (lo + (j+1)*w)) / 2 + est_age    (bit-exact f64)
 *   prob_j  = counts[j] / nsamp
 * nbins[i] == 1 with width 0 encodes the degenerate point-mass row.
 * ------------------------------------------------------------------------- */
typedef struct {
  const double* lo;        /* [N] lowest bucket edge (sample min)                 */
  const double* width;     /* [N] bucket width (hi-lo)/k; 0 for degenerate rows   */
  const double* est_age;   /* [N] attained service when the estimate was taken    */
  const int32_t* nbins;    /* [N] buckets in the row (k, or 1 when degenerate)     */
  const int32_t* nsamp;    /* [N] samples behind the histogram (n)                 */
  const uint16_t* counts;  /* [N, stride] bucket counts                            */
  int64_t stride;          /* counts row stride in elements, multiple of 8        */
} pdg_hist_rows;

/* age: [N] attained service now.  penalty: overrun_penalty_factor.
 * out_key (optional): (float32 key bits << 32) | tiebreak[i]; tiebreak is the
 * position of (arrival_time, app_instance_id) in arrival order (sched.py:168). */
int pdg_gittins_score_hist(const pdg_hist_rows* rows, const double* age,
                           int64_t n, double penalty, float* out_key_f32,
                           uint8_t* out_flags, const uint32_t* tiebreak,
                           uint64_t* out_key, void* stream);

/* ---------------------------------------------------------------------------
 * K5  global order: stable radix sort of packed 64-bit keys ascending,
 * carrying a u32 payload (the queue slot).  Replaces the Python min()/sort
 * over _task_sort_key (simcore.py:339-344, 512-516).
 * begin_bit = 0 sorts the full (key, tiebreak) word; begin_bit = 32 sorts the
 * float key only and relies on stability -- valid when the input is already
 * in arrival (tiebreak) order, e.g. slots filled in arrival order or the
 * rank-major all-gather of arrival-ordered shards.
 * temp: device scratch of pdg_order_temp_bytes(n) bytes.
 * ------------------------------------------------------------------------- */
size_t pdg_order_temp_bytes(int64_t n);
int pdg_order(const uint64_t* keys_in, uint64_t* keys_out,
              const uint32_t* slots_in, uint32_t* slots_out, int64_t n,
              int32_t begin_bit, void* temp, size_t temp_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PDG_B200_H */
