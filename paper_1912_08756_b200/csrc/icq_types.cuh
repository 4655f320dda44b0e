// icq_types.cuh — parameter blocks shared by the host launcher and kernels.
#pragma once
#include <cstdint>

#include "icq_device.cuh"

namespace icq {

// Postfix program of numpy's pairwise float64 summation over d elements
// (leaves of <= 128 elements; op >= 0 is a leaf start, -1 adds the top two).
struct LutProg {
  int32_t nops;
  int32_t op[256];
  int32_t len[256];
};

struct FastBooks {
  uint8_t b[kMaxK];
};

// Per-query state handed from the prologue to the filter and replay kernels.
struct QState {
  int64_t P;            // prologue end: items [0, P) are decided
  int64_t refinements;  // refinements so far (search.py:150)
  int64_t insertions;
  int64_t pro_cand;     // items the prologue scored in float64
  int64_t pro_cycles;
  int64_t pro_t[4];     // prologue phase cycles: prefilter, scoring, decisions, blocks
  int32_t ovf_pages;    // filter slices over kMaxPages (diagnostics)
  int32_t ovf_pool;     // filter slices that found the pool exhausted
  double thr;           // list threshold theta: the lists hold every item with fast64 < thr
  uint32_t mtup[2];     // fast-code bytes of the heap item whose fast score is thr
  int32_t mt_valid;     // (sigma == 0: items with this tuple tie at thr exactly)
  float lo, hi;         // its certified float32 bounds (x32 < lo: yes, x32 >= hi: no)
  int32_t wide;         // float32 certification off: float64 only
  int32_t done;         // all items decided, outputs written (later rounds skip it)
  int32_t rounds;       // filter/replay rounds before this one
  int32_t count_mode;   // refinement-heavy query: the lists hold only possible insertions
                        // (fast < thr and exact < T at P); the replay records the threshold
                        // trajectory and the count kernel tallies refinements / survivors
  float hiT;            // count mode: certified float32 upper bound of T at P (K terms)
  int32_t ntraj;        // count mode: insertions after P (trajectory entries)
  double smin;          // count mode: min slow-book sum (rounded down), thr = T - smin
  double thr0;          // count mode: the live threshold at P0
  int64_t P0;           // the prologue end (P moves when a walk hands a query to a new round)
  int64_t walked;       // items walked in order in earlier rounds
  int64_t listed_raw;   // count mode: entries the filter listed before the refine kernel
  int64_t list_end;     // the filter lists items [P, list_end) in this round (count mode: a
                        // prefix first, then the rest under the tighter T)
  int64_t cm_end;       // count mode: the count kernel covers [P0, cm_end) (n unless the query
                        // went on in list mode at a round hand-over)
  int32_t dense;        // count mode, first round: the prefix is listed by the dense kernel
  int32_t pad_;
  int64_t cl_base;      // count mode: the query's contiguous list [cl_base, cl_base + cl_count)
  int64_t cl_count;     //   in cl_ent / cl_ex, or cl_base < 0: decide from the slices
  int64_t skipped;      // items the filter did not stream (their slice overflowed:
                        // the replay rescans it from the codes)
};

constexpr int kFW = 16;          // filter warps per CTA (one slice per warp and range)
constexpr int kPG = 128;         // candidate pool page (entries; the filter indexes by gg >> 7)
constexpr int kListPages = 128;  // pages per list-mode slice (more -> the replay walks the slice)
constexpr int kMaxPages = 512;   // pages per count-mode slice (a 64k-item slice may list every item)
constexpr int kSliceInts = 4 + kMaxPages;  // slice row: count, page ids, pad / list offset (16-byte rows)
constexpr int kStageInts = 4 + kListPages;  // the part of a row the replay stages in shared memory
constexpr int kProThreads = 256;
constexpr int kProBlock = 2048;  // items per prologue block (8 per thread)
constexpr int64_t kRangeAlign = 32768;
constexpr int kMaxRounds = 4;  // filter/replay rounds per batch (walks past walk_cap resume)
constexpr int kProfEvents = 3 + 3 * kMaxRounds;  // start, prologue, (filter, refine, replay) per round, count

// count mode: the live threshold after an insertion at item pos (items > pos use thr)
struct TrajEntry {
  int64_t pos;
  double thr;
};
constexpr int kMaxTraj = 8192;  // insertions after P per query in count mode

struct PipeParams {
  const uint8_t* codes_fast;  // [n_pad * FP]   fast books only (row-major), zero padded
  const uint8_t* codes_full;  // [n_pad * KP]   all books (row-major), zero padded
  const double* lut64;        // [Q][K][m]
  int64_t* ids;               // [Q*k]
  double* scores;             // [Q*k]
  int64_t* refinements;       // [Q] or null
  uint32_t* survivors;        // [Q*words] or null
  int64_t* stats;             // [Q*kStats] or null
  int32_t* error;             // device error word
  // workspace
  QState* qs;                 // [Q]
  double* heap_e;             // [Q*k]
  double* heap_f;             // [Q*k]
  int32_t* heap_i;            // [Q*k]
  uint4* pool;                // [pool_pages * kPG] candidates {id, 0, fast-code tuple (FP <= 8) | f64 fast (FP = 16)}
  int32_t* pool_top;          // pages handed out
  int32_t* slices;            // [Q*NR*kFW][kSliceInts]: count (-1 = overflow), page ids
  TrajEntry* traj;            // [Q][kMaxTraj] count-mode threshold trajectories
  int32_t* cm_list;           // [1 + Q] count-mode queries of the batch: count, then query ids
  uint4* cl_ent;              // [cl_cap] count-mode lists after the refine kernel, contiguous per
  double* cl_ex;              //   query in database order, with their float64 exact scores
  unsigned long long* cl_top; // entries handed out of cl_ent / cl_ex
  int64_t cl_cap;
  int32_t cl_enable;          // 0: no contiguous lists (ICQ_CL=0, tests of the slice path)
  int64_t pool_pages;
  int32_t max_pages;          // pages per list-mode slice (<= kListPages; tests lower it)
  int32_t max_pages_cm;       // pages per count-mode slice (<= kMaxPages)
  int64_t n;
  int64_t words;              // survivors bitmap words per query
  int64_t RS;                 // items per range (multiple of kRangeAlign)
  int64_t RSC;                // items per range of the count kernel (a multiple of RS)
  int32_t NRC;
  int32_t RG, NRG;            // ranges per refine / gather CTA, and the number of such groups
  int32_t NRD;                // ranges the dense prefix kernel covers (count mode, first round)
  double sigma;
  int32_t Q, K, m, KP, F, k;
  int32_t NR;                 // ranges per query
  int32_t range_major;        // filter unit order (L2 reuse of codes larger than L2)
  int32_t exact_mode;         // search_exact: report refinements = n (search.py:108)
  int32_t pro_div;            // prologue stops once a block's candidates <= items / pro_div
  int32_t debug;              // experiments only (ICQ_DEBUG): bit 0 = no tuple-tie rejection,
                              // bit 1 = replay producers skip exact scores
  int32_t list_j;             // list threshold theta = A_J + sigma at the prologue end (A_J:
                              // max fast score over the J+1 largest-exact heap entries);
                              // -1: the loosest J on a ladder with a list share <= 1/list_div
  int32_t list_div;
  int32_t count_div;          // count mode when the live threshold passes > 1/count_div of the
                              // sampled items (0: never; ICQ_COUNT_MODE=1 forces it)
  int32_t force_count;
  int64_t count_min;          // ... and would list more than count_min items of the rest
  int32_t count_used;         // count mode possible: launch the count kernel
  int32_t pro_live;           // prologue stop rule counts items under theta (1) or under M (0)
  int32_t sigma_f32;          // numpy promotion of a float32 sigma (see live_thr)
  int32_t rounds;             // filter/replay rounds (1..kMaxRounds)
  int32_t round, last_round;  // this launch's round
  int64_t walk_cap;           // an in-order walk longer than this hands the query to the next round
  int64_t pro_min, pro_max;   // prologue length bounds (items)
  int64_t cm_prefix;          // count mode: the first round lists items below this position only
  int32_t* round_cnt;         // [kMaxRounds + 1] queries handed to each round
  int64_t pro_max_cm;         // refinement-heavy queries: the count-style prologue blocks end here
  uint8_t fast_books[kMaxK];
};

// kernels launched by this library since it was loaded (icq_kernel_launches)
void count_kernel_launches(int n);
long long kernel_launches();
bool make_lut_prog(int d, LutProg* out);
cudaError_t launch_lut(const float* books, const double* q, double* lut, int K, int m, int d,
                       int Q, const LutProg* prog_dev, int32_t* err, cudaStream_t s);
// prologue -> filter -> replay for one batch (icq_pipeline.cu)
// ev: optional kProfEvents events: before the prologue, after the prologue,
// after the filter, the refine and the replay kernel of every round, after the
// count kernel
cudaError_t launch_pipeline(const PipeParams& p, int FP, int filter_ctas, cudaStream_t s,
                            int* unsupported, cudaEvent_t* ev = nullptr);

}  // namespace icq
