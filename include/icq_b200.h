/*
 * icq_b200.h — C ABI of the B200-native ICQ query path (libicq_b200.so).
 *
 * Drop-in boundary for the reference package's query engines
 * (/root/reference/pkg/src/icq/search.py).  The reference is pure Python,
 * so its "FFI" is the Python call surface; each entry point below names the
 * reference function it replaces (file:line) and keeps its argument meaning
 * and error behaviour.  The ctypes binding a maintainer adds on the reference
 * side is shown in INTEGRATION.md; the package paper_1912_08756_b200 ships it.
 *
 * Conventions
 *   - Plain pointers and sizes only.  "dev" pointers are CUDA device
 *     pointers; "host" pointers are ordinary host memory.  `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Every function returns an icq_status; on failure a thread-local message
 *     is available from icq_last_error().  Nothing throws across the ABI.
 *   - Results are exactly the reference's: ids/int64, scores/float64 (the
 *     reference's float64 distance values, search.py:163), refinement counts.
 *     The fp32 hot path is certified against float64 with a rounding-error
 *     bound, so survivor sets and top-k match the float64 reference bit for bit.
 */
#ifndef ICQ_B200_H
#define ICQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ICQ_OK = 0,
  ICQ_ERR_VALIDATION = 1,   /* -> icq.data.ValidationError (data.py:32) */
  ICQ_ERR_UNSUPPORTED = 2,  /* shape outside this build (m > 256, K > 16, k too large) */
  ICQ_ERR_CUDA = 3,         /* CUDA runtime / launch failure */
  ICQ_ERR_NOMEM = 4,        /* device allocation failed / workspace too small */
  ICQ_ERR_FORMAT = 5,       /* -> icq.data.FormatError (data.py:36): malformed ICQI file */
  ICQ_ERR_VERSION = 6       /* -> icq.data.UnsupportedVersionError (data.py:40) */
} icq_status;

typedef struct icq_index_s* icq_index_t;

/* Search flags (icq_search_with_lut / icq_search_host `flags`). */
#define ICQ_FLAG_EXACT 1     /* run search_exact (search.py:97-109) instead of two-step */
#define ICQ_FLAG_SIGMA_F32 2 /* sigma is a numpy float32 scalar: reproduce numpy 2's
                                promotion of `bound + sigma` (search.py:149) -- float32
                                once the heap maximum is an inserted entry */

/* Message of the last failing call on this host thread ("" if none). */
const char* icq_last_error(void);

/* ABI version (bumped on any signature change). */
int32_t icq_abi_version(void);

/* Search-path kernels this library launched since it was loaded (LUT build,
 * prologue, filter / dense / refine / list / replay of every round, count):
 * bench.py reports the difference over its timed region as gpu_launches. */
int64_t icq_kernel_launches(void);

/* ---------------------------------------------------------------------------
 * Index: device-resident copy of icq.data.SearchIndex (data.py:193-263).
 *   books : host float32 [K*m*d], row-major (K, m, d)        (data.py:143, :222)
 *   codes : host uint32  [n*K],   row-major (n, K)           (data.py:179)
 *   fast  : host uint32  [F], sorted unique book ids < K     (data.py:159-164)
 * Validation mirrors SearchIndex.__post_init__: code >= m, unsorted/duplicate
 * fast set or fast id >= K -> ICQ_ERR_VALIDATION.  m > 256 or K > 16 ->
 * ICQ_ERR_UNSUPPORTED (codes are repacked to uint8 on the device).
 * The handle is immutable after creation and may be shared by threads.
 * ------------------------------------------------------------------------- */
icq_status icq_index_create(const float* books_host, int32_t K, int32_t m, int32_t d,
                            const uint32_t* codes_host, int64_t n,
                            const uint32_t* fast_host, int32_t F,
                            icq_index_t* out);

/* Same, with codes already narrowed to uint8 (host). */
icq_status icq_index_create_u8(const float* books_host, int32_t K, int32_t m, int32_t d,
                               const uint8_t* codes_host, int64_t n,
                               const uint32_t* fast_host, int32_t F,
                               icq_index_t* out);

/* Same, all inputs already on the device (codes uint8 (n, K) row-major). */
icq_status icq_index_create_device(const float* books_dev, int32_t K, int32_t m, int32_t d,
                                   const uint8_t* codes_dev, int64_t n,
                                   const uint32_t* fast_host, int32_t F,
                                   void* stream, icq_index_t* out);

icq_status icq_index_destroy(icq_index_t h);

/* Copy rows [row0, row0 + rows) of the index's codes back to the host as
 * uint8 (rows, K) row-major (the reference's CodeMatrix values). */
icq_status icq_index_read_codes(icq_index_t h, int64_t row0, int64_t rows, uint8_t* codes_host);

/* ---------------------------------------------------------------------------
 * load_index (data.py:348-394) straight into device memory.
 * icq_index_file_info_read parses and validates the header only (magic,
 * version, Config, n, d).  icq_index_load validates the whole file with the
 * reference's conditions (bad magic / truncation / inconsistent lengths /
 * trailing bytes / invalid Config or SearchIndex fields -> ICQ_ERR_FORMAT,
 * version != 1 -> ICQ_ERR_VERSION), then streams the (n, K) uint32 code
 * block through pinned host buffers into the device repack (the block is
 * never materialised whole).  Optional host outputs: books [K*m*d], xi [d],
 * lambdas [d]; info gets the Config fields, the float32 margin and the fast
 * set (flatnonzero of the file's fast mask).
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t K, m, d, n;               /* Config.K, Config.m; u32 n, d */
  double gamma1, gamma2, pi1, pi2, alpha2, sigma_scale;
  int64_t epochs, batch_size;
  double learning_rate;
  uint64_t seed;
  float sigma;                      /* the stored float32 margin (data.py:322) */
  int32_t F;
  uint32_t fast[64];
  int64_t file_bytes;
} icq_index_file_info;

icq_status icq_index_file_info_read(const char* path, icq_index_file_info* info);
icq_status icq_index_load(const char* path, float* books_host, uint8_t* xi_host,
                          float* lambdas_host, icq_index_file_info* info, void* stream,
                          icq_index_t* out);

/* ---------------------------------------------------------------------------
 * search_bruteforce (search.py:168-178): exact float64 squared Euclidean scan
 * over raw float32 vectors, top-k by (score, id) -- bitwise the reference's
 * scores (numpy pairwise order).  x_dev: float32 [n*d] row-major; q_dev:
 * float64 [Q*d]; ids_dev int64 [Q*k]; scores_dev float64 [Q*k].  k <= 1024.
 * ------------------------------------------------------------------------- */
icq_status icq_bruteforce(const float* x_dev, int64_t n, int32_t d, const double* q_dev,
                          int32_t Q, int32_t k, int64_t* ids_dev, double* scores_dev,
                          void* stream);

/* ---------------------------------------------------------------------------
 * assign_codes / encode_dataset (train.py:196-243, :256-274): ICM encoding in
 * float64 on the device -- greedy build-up (codes_in_dev NULL) or sweeps
 * from given codes, then up to max_sweeps strict-improvement sweeps, stopping
 * after a sweep that changes nothing.  x_dev float32 [n*d]; books_dev
 * float64 [K*m*d]; c_sq_dev float64 [K*m] (sum of squares over d in numpy's
 * order); codes uint8 [n*K] (m <= 256).  sweeps_out: sweeps run (max over
 * row chunks).  Codes equal the reference's except where two codewords tie
 * to rounding (the reference's dgemm sums in a different order).
 * ------------------------------------------------------------------------- */
icq_status icq_encode(const float* x_dev, int64_t n, int32_t d, const double* books_dev,
                      const double* c_sq_dev, int32_t K, int32_t m, const uint8_t* codes_in_dev,
                      int32_t max_sweeps, uint8_t* codes_out_dev, int32_t* sweeps_out,
                      void* stream);

/* Shape and device footprint of an index. */
icq_status icq_index_info(icq_index_t h, int64_t* n, int32_t* K, int32_t* m, int32_t* d,
                          int32_t* F, int64_t* device_bytes);

/* ---------------------------------------------------------------------------
 * build_lut (search.py:61-69): lut[q][b][j] = sum_d (c[b][j][d] - q[d])^2 in
 * float64, summed in numpy's pairwise order (bitwise equal to the reference).
 *   q   : dev float64 [Q*d]      lut : dev float64 [Q*K*m]
 * A non-finite query value -> ICQ_ERR_VALIDATION (search.py:51-52).  Like
 * every entry point below, the call synchronizes `stream` before returning
 * so that device-side validation and error words reach the caller.
 * ------------------------------------------------------------------------- */
icq_status icq_build_lut(icq_index_t h, const double* q_dev, int32_t Q, double* lut_dev,
                         void* stream);

/* Device workspace needed by the search calls below for Q queries, top-k. */
icq_status icq_workspace_size(icq_index_t h, int32_t Q, int32_t k, size_t* bytes);

/* ---------------------------------------------------------------------------
 * search_two_step (search.py:112-165), batched: Q independent queries.
 *   sigma        : pruning margin >= 0 (NaN or negative -> ICQ_ERR_VALIDATION,
 *                  search.py:125-126); pass the index margin for sigma=None.
 *   k            : 1 <= k <= n (search.py:56-58)
 *   ids_dev      : int64 [Q*k]   ascending (score, id), search.py:156
 *   scores_dev   : float64 [Q*k]
 *   refine_dev   : int64 [Q]     ops.refinements (search.py:160); may be NULL
 *   survivors_dev: optional uint32 bitmap [Q * ceil(n/32)] of refined ids
 *                  (instrumentation for parity tests; NULL to skip)
 *   stats_dev    : optional int64 [Q*16] diagnostics per query (see
 *                  paper_1912_08756_b200.search.STATS_NAMES): heap insertions,
 *                  items decided by the replay, items walked in order, prologue end,
 *                  prologue / replay cycles, rescanned slices (| overflow
 *                  counts << 20 / << 40), wide flag, prologue float64 scorings,
 *                  filter candidates, prologue insertions, count-mode entries
 *                  listed before the refine kernel, prologue phase cycles
 *   fallback_out : optional host int32; set to 1 when the fast set is empty and
 *                  the exact engine ran instead (search.py:127-131)
 * Kernels run on `stream`; the call synchronizes it once at the end and
 * returns the call's device error word (non-finite query ->
 * ICQ_ERR_VALIDATION, internal check failures -> ICQ_ERR_CUDA).  Concurrent
 * calls on different streams are safe (all scratch is per call).
 * sigma is used as a float64 value; see icq_search_with_lut for float32.
 * ------------------------------------------------------------------------- */
icq_status icq_search_two_step(icq_index_t h, const double* q_dev, int32_t Q, int32_t k,
                               double sigma, int64_t* ids_dev, double* scores_dev,
                               int64_t* refine_dev, uint32_t* survivors_dev,
                               int64_t* stats_dev, int32_t* fallback_out,
                               void* workspace_dev, size_t workspace_bytes, void* stream);

/* search_exact (search.py:97-109): full scan, top-k by (score, id). */
icq_status icq_search_exact(icq_index_t h, const double* q_dev, int32_t Q, int32_t k,
                            int64_t* ids_dev, double* scores_dev,
                            void* workspace_dev, size_t workspace_bytes, void* stream);

/* Same two engines on a precomputed float64 LUT (icq_build_lut output,
 * dev float64 [Q*K*m]); no workspace.  flags: ICQ_FLAG_EXACT runs search_exact,
 * ICQ_FLAG_SIGMA_F32 reproduces the reference's arithmetic for a numpy
 * float32 sigma (which must then be exactly a float32 value).  Lets a
 * caller reuse tables across calls and time the scan kernel on its own. */
icq_status icq_search_with_lut(icq_index_t h, const double* lut_dev, int32_t Q, int32_t k,
                               double sigma, int32_t flags, int64_t* ids_dev, double* scores_dev,
                               int64_t* refine_dev, uint32_t* survivors_dev, int64_t* stats_dev,
                               int32_t* fallback_out, void* stream);

/* ---------------------------------------------------------------------------
 * Host-buffer entry points (end-to-end: H2D of queries, search, D2H of results,
 * synchronous).  Same semantics as above; all pointers are host pointers.
 * flags as icq_search_with_lut (0 = two-step with a float64 sigma).
 * Non-finite query values are rejected on the host before any device work.
 * ------------------------------------------------------------------------- */
icq_status icq_search_host(icq_index_t h, const double* q_host, int32_t Q, int32_t k,
                           double sigma, int32_t flags, int64_t* ids_host,
                           double* scores_host, int64_t* refine_host, int32_t* fallback_out);

/* ---------------------------------------------------------------------------
 * Instrumentation (bench / profiling only; not part of the reference surface).
 * icq_profile_enable(1) makes every following search call record CUDA events
 * on its launch stream around the kernels of each batch (prologue; filter,
 * refine and replay of every round; refinement count).  icq_profile_read
 * synchronizes those events and returns the summed device milliseconds per
 * kernel kind (ms_out[5]: prologue, filter, replay, count, refine) and the
 * number of batches recorded, then clears the record.
 * ------------------------------------------------------------------------- */
icq_status icq_profile_enable(int32_t on);
icq_status icq_profile_read(double* ms_out, int32_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* ICQ_B200_H */
