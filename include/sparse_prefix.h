/*
 * include/sparse_prefix.h -- C ABI of libsparseprefix.so, the B200 (sm_100a) hot path of
 * sparse prefix caching (arXiv 2605.05219, "PAPER.md"; "P:L" = PAPER.md line L).
 *
 * The method: for each retained cache entry (a cached prefix of length <= N), estimate the law
 * of the overlap depth T of future requests from observed requests, and place at
 * most M recurrent-state checkpoints 1 <= c_1 < ... < c_M <= N so that the expected
 * recomputation E[r(T;C)] = sum_t p_t (t - l(t;C)) is minimal, via the exact dynamic
 * program of Thm 2.
 *
 * General conventions (every call):
 *   - Pointers are DEVICE pointers unless a parameter says "host".  The caller owns every
 *     buffer; the library never allocates on these paths (the DP's scratch is a caller-provided
 *     workspace).  Calls are stateless and thread-safe.
 *   - Calls are asynchronous and stream-ordered on `stream` (0 = legacy default stream).
 *   - Shape / argument errors are detected on the host and returned synchronously, with nothing
 *     enqueued.  Per-entry data errors that can only be seen on the device (overflow guard,
 *     malformed positions) are reported in the per-entry outputs as documented below.
 *   - Counts: histograms are integer counts c_t of observed overlap depths, row-major
 *     [n_entries][N+1]; bin 0 counts misses and is ignored by the objective (T in {1..N},
 *     P:169; hits only).  Probabilities p = c / n are never formed: the argmin is
 *     scale invariant, and costs are returned as integer numerators n * E[r].
 *   - Canonical output ("rule B", reading R3): among optimal placements the library
 *     returns the colex-minimal one: per DP cell the lowest-index argmin, backtracked from
 *     (M, N) and stopped as soon as no mass remains at or below the current depth.
 */
#ifndef SPARSE_PREFIX_H
#define SPARSE_PREFIX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sp_stream_t; /* == cudaStream_t */

typedef enum {
  SP_OK = 0,
  SP_ERR_BAD_LENGTH = 1,       /* N < 1, n_entries < 0, n_requests < 0, N > SP_MAX_N            */
  SP_ERR_BUDGET_TOO_LARGE = 2, /* M < 0 or M > N                                                */
  SP_ERR_BAD_ARGUMENT = 3,     /* NULL required pointer, bad enum, misaligned buffer            */
  SP_ERR_OVERFLOW = 4,         /* per entry: 2 * n * N does not fit the cost type               */
  SP_ERR_BAD_POSITIONS = 5,    /* per set: positions not strictly increasing in [1, N]          */
  SP_ERR_WORKSPACE = 6,        /* workspace NULL or smaller than *_workspace_bytes()            */
  SP_ERR_CUDA = 7,             /* launch / runtime error; see sp_last_error_string()            */
  SP_ERR_INTERNAL = 8          /* per entry: a D&C bracket came out empty (never expected)      */
} sp_status;

typedef enum {
  SP_W_COUNTS_I32 = 0, /* int32_t c[E][N+1]                                                    */
  SP_W_COUNTS_I64 = 1, /* int64_t c[E][N+1]                                                    */
  SP_W_PROB_F64 = 2    /* double  w[E][N+1], w_t >= 0 finite (fp64 variant; costs are double)  */
} sp_weight_type;

#define SP_MAX_N 65535 /* positions are stored as uint16 in the argmin table */

/* ------------------------------------------------------------------------------------------
 * a1 + a2 -- overlap depths and the per-entry overlap-depth histogram.
 * P:133-137 (overlap depth t of a request with the cached prefix), P:169 (T in {1..N}),
 * P:189-190 (per-edge decomposition: each request is matched against the entry it hit).
 *
 * For request r (tokens req_tokens[req_off[r] .. req_off[r+1])) and its entry
 * e = req_entry[r] (tokens entry_tokens[entry_off[e] .. entry_off[e+1])):
 *     t_r = min(LCP(request, entry), N)          (depths beyond N clamp to N)
 *     hist[e][t_r] += 1                          (ACCUMULATED: the caller zeroes hist)
 *     lcp_out[r] = t_r                           (if lcp_out != NULL)
 * hist may be NULL when lcp_out is not (depths only, e.g. to ship (entry, depth) pairs to the
 * entry's owner rank and merge there with sp_accumulate_depths).
 * Offsets are int64 token indices; rows with offsets that are multiples of 4 tokens take the
 * 16-byte vector path, others a scalar path (same result).  Precondition (checked only by
 * debug builds): 0 <= req_entry[r] < n_entries; requests with an out-of-range entry are
 * skipped and get lcp_out[r] = -1.
 * Errors: SP_ERR_BAD_LENGTH (N < 1 or N > SP_MAX_N, n_entries < 0, n_requests < 0),
 *         SP_ERR_BAD_ARGUMENT (NULL required pointer), SP_ERR_CUDA.
 * ---------------------------------------------------------------------------------------- */
sp_status sp_overlap_hist(const int32_t* entry_tokens, const int64_t* entry_off,
                          int32_t n_entries, const int32_t* req_tokens, const int64_t* req_off,
                          const int32_t* req_entry, int64_t n_requests, int32_t N,
                          int32_t* hist, int32_t* lcp_out, sp_stream_t stream);

/* Multi-GPU merge helper (SURVEY 8(e) sparse variant): hist[e - e_begin][depth[i]] += 1 for
 * every i with e_begin <= entry[i] < e_end and 0 <= depth[i] <= N (others ignored).
 * hist is [e_end - e_begin][N+1], accumulated.  Errors: BAD_LENGTH, BAD_ARGUMENT, CUDA. */
sp_status sp_accumulate_depths(const int32_t* entry, const int32_t* depth, int64_t n,
                               int32_t e_begin, int32_t e_end, int32_t N, int32_t* hist,
                               sp_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * a3 + a4 + a5 -- optimal checkpoint placement (Thm 2; proof P:755-774).
 *   P_j = sum_{t<=j} c_t,  T_j = sum_{t<=j} t c_t
 *   dp[0][j] = T_j,  dp[m][0] = 0 (at-most-m reading R1),
 *   dp[m][j] = min_{1<=s<=j} dp[m-1][s-1] + (T_j - T_{s-1}) - s (P_j - P_{s-1})
 * computed on the GPU exactly by the paper's monotone convex-hull trick with all
 * layers advancing in lockstep, one warp per entry (dp_hull.cu): int32 arithmetic when
 * 2 P_N N < 2^31; a large-hull mode (unary argmin logs, global deque arrays; int32 while
 * P_N N + T_N < 2^31) for entries whose hull outgrows the shared rings (e.g. all-ones rows);
 * int64 arithmetic below P_N N < 2^46; fp64 weights in double.  What none of them solves (bad
 * rows, overflowing logs or arrays in the int64 / fp64 modes) goes to a divide-and-conquer
 * monotone argmin per layer (dp_place.cu).  Every path returns the same exact results (the
 * leftmost-argmin, rule-B placement).  DESIGN.md section 7.
 *
 *   weights        [E][N+1] of type wtype (bin 0 ignored; not normalised)
 *   positions      int32 [E][M]: the rule-B placement, ascending, unused slots 0
 *   n_positions    int32 [E]: number of positions (0..min(M, #nonzero bins)), or a NEGATIVE
 *                  sp_status for that entry: -SP_ERR_BAD_ARGUMENT for a negative count / a
 *                  negative or non-finite fp64 weight; -SP_ERR_OVERFLOW for the count types if
 *                  a count is >= 2^47 or 2 * P_N * N >= 2^62; -SP_ERR_INTERNAL never expected.
 *                  Such an entry's positions are 0 and its costs unspecified.
 *   cost           [E]: V_M = dp[M][N] = n * E[r] -- int64 for count types, double for F64
 *   cost_by_budget [E][M+1] V_0..V_M (same type as cost; V_0 = T_N = n * R_nc), or
 *                  NULL.  (The DP computes every budget m <= M on the way.)
 *   workspace      device scratch of >= sp_place_checkpoints_workspace_bytes(E, N, M) bytes.
 *                  Its first SP_WS_STATS_BYTES bytes receive launch statistics
 *                  (sp_dp_stats, see below); the rest is scratch.
 * M = 0 gives n_positions = 0 and cost = T_N.  An all-zero histogram gives 0 positions, cost 0.
 * Errors (synchronous): BAD_LENGTH (N < 1, N > SP_MAX_N, E < 0), BUDGET_TOO_LARGE (M < 0 or
 * M > N), BAD_ARGUMENT (NULL pointer, bad wtype), WORKSPACE, CUDA.
 * ---------------------------------------------------------------------------------------- */
size_t sp_place_checkpoints_workspace_bytes(int32_t n_entries, int32_t N, int32_t M);

/* Launch statistics written (stream-ordered) at the start of the workspace by every
 * sp_place_checkpoints call: the exact number of candidate evaluations b_s - s P_j the
 * divide-and-conquer performed, the line tests of the hull kernel (the DP's executed work;
 * cells = E N M), and the entries solved on the exact-int32 / int64 / fp64 paths and by the
 * hull kernel. */
#define SP_WS_STATS_BYTES 256
typedef struct {
  unsigned long long evaluations;      /* D&C candidate evaluations b_s - s P_j               */
  unsigned long long entries_i32, entries_i64, entries_f64;   /* entries per arithmetic path */
  unsigned long long hull_pops;        /* hull kernel: lines popped (back + front)            */
  unsigned long long entries_hull;     /* entries solved by the hull kernel (rest: D&C)       */
  unsigned long long hull_event_rows;  /* hull kernel: rows with c_j > 0 (line push + query)  */
  unsigned long long entries_hull_big; /* of entries_hull: solved by the int32 large-hull mode
                                          (hulls past the shared rings, e.g. all-ones rows;
                                          unary argmin logs)                    */
} sp_dp_stats;

sp_status sp_place_checkpoints(const void* weights, sp_weight_type wtype, int32_t n_entries,
                               int32_t N, int32_t M, int32_t* positions, int32_t* n_positions,
                               void* cost, void* cost_by_budget, void* workspace,
                               size_t workspace_bytes, sp_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * a6 -- expected recomputation and worst case of given placements (baseline evaluation).
 * For checkpoint set C = {c_1 < ... < c_k} (c_0 = 0, c_{k+1} = N + 1):
 *   cost  = sum_{t=1}^N c_t (t - l(t;C))                          (l from P:133-137)
 *   worst = max_{0<=i<=k} (c_{i+1} - c_i) - 1 = max_t r(t;C)       (distribution-free)
 * n_sets placements per entry.  broadcast != 0: positions [n_sets][max_pos] and
 * n_positions [n_sets] are shared by every entry (e.g. balanced / block schedules, Table 1
 * P:360-378); broadcast == 0: positions [E][n_sets][max_pos], n_positions [E][n_sets].
 *   cost        [E][n_sets]: int64 (count types) or double (F64)
 *   worst_case  int32 [E][n_sets] or NULL
 * A malformed set (k < 0, k > max_pos, positions not strictly increasing in [1, N]) yields
 * cost = -1 (count types) / NaN (F64) and worst = -SP_ERR_BAD_POSITIONS for that set.
 * Errors (synchronous): BAD_LENGTH, BAD_ARGUMENT, CUDA.
 * ---------------------------------------------------------------------------------------- */
/* f3 -- the all-budget frontier (the Pareto curves of Figs. 2-3):
 * the same DP, plus the canonical placement of EVERY budget m = 1..M from its argmin table
 * (layers 1..m of an M-layer run are an m-layer run, so row m-1 equals what
 * sp_place_checkpoints(..., m, ...) returns).
 *   frontier_positions int32 [E][M][M]: row m-1 = budget m's positions, ascending, 0-padded
 *   frontier_n         int32 [E][M]: counts (or the entry's negative status)
 *   cost_by_budget, positions, n_positions, cost: as sp_place_checkpoints (may be NULL except
 *   n_positions and cost).  Same workspace as sp_place_checkpoints. */
sp_status sp_place_checkpoints_frontier(const void* weights, sp_weight_type wtype,
                                        int32_t n_entries, int32_t N, int32_t M,
                                        int32_t* frontier_positions, int32_t* frontier_n,
                                        void* cost_by_budget, int32_t* positions,
                                        int32_t* n_positions, void* cost, void* workspace,
                                        size_t workspace_bytes, sp_stream_t stream);

sp_status sp_expected_recompute(const void* weights, sp_weight_type wtype, int32_t n_entries,
                                int32_t N, const int32_t* positions, const int32_t* n_positions,
                                int32_t n_sets, int32_t max_pos, int32_t broadcast, void* cost,
                                int32_t* worst_case, sp_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * f1 -- block-aware placement ("clip every checkpoint position to the block boundaries",
 * B = 128; P:397 B = 64).
 *
 * sp_place_checkpoints_grid: the exact DP with checkpoints restricted to multiples of B
 * (S:208 candidate_grid).  Outputs as sp_place_checkpoints (positions are multiples of B; at
 * most min(M, floor(N/B)) of them; cost = sum_t c_t (t - l(t;C)) exactly).  Computed as the
 * unrestricted DP on the block-aggregated histogram C_k = sum_{t in [kB,(k+1)B)} c_t plus the
 * placement-independent constant sum_t c_t (t - B floor(t/B)).  Canonical
 * output: the colex-minimal optimal grid set (reading R13).  Errors as sp_place_checkpoints,
 * plus BAD_ARGUMENT for B < 1.
 * sp_clip_to_blocks: post-hoc clipping, per entry: floor(c / B) B, zeros dropped, duplicates
 * merged; n_positions < 0 (a per-entry status) is passed through.
 * ---------------------------------------------------------------------------------------- */
size_t sp_place_checkpoints_grid_workspace_bytes(int32_t n_entries, int32_t N, int32_t M,
                                                 int32_t B);
sp_status sp_place_checkpoints_grid(const void* weights, sp_weight_type wtype, int32_t n_entries,
                                    int32_t N, int32_t M, int32_t B, int32_t* positions,
                                    int32_t* n_positions, void* cost, void* cost_by_budget,
                                    void* workspace, size_t workspace_bytes, sp_stream_t stream);
sp_status sp_clip_to_blocks(const int32_t* positions /*[E][max_pos]*/,
                            const int32_t* n_positions /*[E]*/, int32_t n_entries,
                            int32_t max_pos, int32_t B, int32_t* out_positions /*[E][max_pos]*/,
                            int32_t* out_n /*[E]*/, sp_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * f2 -- Thm 4's exponentially weighted empirical overlap histogram, batched over
 * entries; the estimator the paper re-solves the placement from (g = 0.99):
 *   p_t = (1 - g) / (1 - g^t) sum_{s=1..t} g^(t-s) e_{T_s}      (g = 1: the empirical law, Thm 3)
 * State per entry e (device, caller-owned, zero-initialised for a fresh estimator):
 *   W     double [E][N+1]  weights relative to the epoch tau: decayed weights w = W g^(t - tau)
 *   t     int64  [E]       observations so far;   tau  int64 [E]   reference epoch
 * sp_gamma_observe appends one batch of observations GROUPED BY ENTRY, in arrival order within
 * each entry: obs_off int64 [E+1] (CSR offsets), depth int32 [obs_off[E]] (e.g. sp_overlap_hist's
 * lcp_out).  Only hits are samples of T in {1..N}: a depth < 1 (a miss) is
 * skipped -- no weight, t unchanged; depths > N are clamped to N.  Hit number t+1 adds
 * g^-(t+1-tau) to W[e][depth]; the row is rescaled (tau = t) before exponents pass 2^64.  t counts
 * hits.  fp64 atomics: the
 * summation order (not the value) of equal-depth observations in one batch is unspecified.
 * W can be handed to sp_place_checkpoints (SP_W_PROB_F64) directly: it differs from p_t by a
 * positive per-entry factor, and the placement is scale-invariant.
 * sp_gamma_snapshot writes p_t (double [E][N+1], bins 1..N sum to 1, bin 0 = 0; all zero when
 * t = 0).
 * Errors: BAD_LENGTH (N < 1, N > SP_MAX_N, E < 0), BAD_ARGUMENT (g outside (0, 1], NULL), CUDA.
 * ---------------------------------------------------------------------------------------- */
sp_status sp_gamma_observe(double* W, int64_t* t, int64_t* tau, const int64_t* obs_off,
                           const int32_t* depth, int32_t n_entries, int32_t N, double gamma,
                           sp_stream_t stream);
sp_status sp_gamma_snapshot(const double* W, const int64_t* t, const int64_t* tau,
                            int32_t n_entries, int32_t N, double gamma, double* p_out,
                            sp_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * f4 -- longest-prefix search over ALL cached entries (the trie remark of P:189-190: a request
 * reuses the deepest cached prefix; SPEC match_longest_prefix S:375-383): for each request, the
 * entry e maximising LCP(entry_e, request); ties -> the most recent insertion (largest
 * insertion[e]; the entry index when insertion is NULL; equal values -> larger index);
 * maximum 0 -> no match.
 * sp_prefix_index_build sorts the entries by tokens (device merge sort) and builds a sparse
 * table for range "most recent" queries, into the caller's index buffer of
 * sp_prefix_index_workspace_bytes(E) bytes (device).  Rebuild whenever the cache changes.
 * sp_match_longest_prefix: one warp per request, O(log E) warp-cooperative comparisons:
 *   match_entry int32 [R] (-1 = no match), match_depth int32 [R] (the raw LCP; clamp to N
 *   before feeding a histogram, as sp_overlap_hist does).
 * Token layout as sp_overlap_hist (int32 CSR, int64 offsets).  Errors: BAD_LENGTH (E < 0,
 * R < 0), BAD_ARGUMENT (NULL), WORKSPACE, CUDA.
 * ---------------------------------------------------------------------------------------- */
size_t sp_prefix_index_workspace_bytes(int32_t n_entries);
sp_status sp_prefix_index_build(const int32_t* entry_tokens, const int64_t* entry_off,
                                int32_t n_entries, const int64_t* insertion, void* index,
                                size_t index_bytes, sp_stream_t stream);
sp_status sp_match_longest_prefix(const int32_t* entry_tokens, const int64_t* entry_off,
                                  int32_t n_entries, const void* index, const int32_t* req_tokens,
                                  const int64_t* req_off, int64_t n_requests,
                                  int32_t* match_entry, int32_t* match_depth, sp_stream_t stream);

/* Host-side helpers for the Table 1 baselines.  out_host must hold M (resp.
 * floor(N/B)) ints.  Return the number of positions written, or a negative sp_status. */
int32_t sp_balanced_positions(int32_t N, int32_t M, int32_t* out_host);
int32_t sp_block_positions(int32_t N, int32_t B, int32_t* out_host);
/* sqrt(L) schedule: multiples of floor(sqrt(N)).  out_host holds N ints. */
int32_t sp_sqrt_positions(int32_t N, int32_t* out_host);
/* logarithmic schedule (SPEC's reading S:198): round(N (2^i - 1) / (2^M - 1)), i = 1..M,
 * clamped to [1, N], duplicates dropped; 1 <= M <= min(N, 62).  out_host holds M ints. */
int32_t sp_log_positions(int32_t N, int32_t M, int32_t* out_host);

const char* sp_status_string(sp_status status);
/* Last CUDA error text seen by this thread (static storage, never NULL). */
const char* sp_last_error_string(void);
/* Library version string, e.g. "sparseprefix 0.1 sm_100a". */
const char* sp_version(void);

/* Comparison / test hooks -- not needed by callers.  Process-wide values that steer which
 * kernel path a call takes (the results are the same on every path; the parity tests run each):
 *   SP_DBG_NO_HULL       1: the DP uses the divide-and-conquer kernel only
 *   SP_DBG_HULL_LEAN     1: the int32 hull path uses dp_lean_kernel
 *   SP_DBG_HULL_SPLIT    -1 automatic (default), 0 never, 1 always two warps per entry
 *   SP_DBG_HULL_LOGCAP   > 0: argmin-log capacity override (forces the log-full fallback)
 *   SP_DBG_HULL_NO_ORDER 1: no largest-first entry order
 *   SP_DBG_EVAL_PATH     0 automatic, 1 chunked kernel, 2 4-byte-prefix kernel, 3 2-byte-prefix
 * Initial values come from the environment variables of the same names (SP_NO_HULL, ...), read
 * once per process; sp_debug_set returns the previous value (or -SP_ERR_BAD_ARGUMENT for an
 * unknown flag).  Read on the host at launch time: not stream-ordered. */
enum { SP_DBG_NO_HULL = 0, SP_DBG_HULL_LEAN = 1, SP_DBG_HULL_SPLIT = 2, SP_DBG_HULL_LOGCAP = 3,
       SP_DBG_HULL_NO_ORDER = 4, SP_DBG_EVAL_PATH = 5, SP_DBG_COUNT = 6 };
int sp_debug_set(int flag, int value);
int sp_debug_get(int flag);

#ifdef __cplusplus
}
#endif
#endif /* SPARSE_PREFIX_H */
