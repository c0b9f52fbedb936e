/*
 * oracle/sp_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the sparse-prefix-caching hot path of
 * arXiv 2605.05219 ("PAPER.md" below; "P:L" = PAPER.md line L, "S:L" = SPEC.md line L).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  It shares no code, header, table or helper with the CUDA product path
 * (paper_2605_05219_b200/csrc, include/), and the product path never loads it.
 *
 * Conventions
 *   - counts c[0..N] are int64; bin 0 is the "miss" bin and is ignored by the objective
 *     (T ranges over {1..N}; hits only).
 *   - all DP tables are row-major [(M+1)][(N+1)].
 *   - checkpoint sets are ascending int32 arrays.
 *   - every function that can fail returns 0 on success and a negative value on bad input.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py (see DESIGN.md
 * "Oracle pins").  None is "parity unpinned".
 */
#ifndef SP_ORACLE_H
#define SP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* a1+a2: literal LCP loop + histogram.
 * hist[E][N+1] is ACCUMULATED; lcp_out[R] may be NULL.  nthreads >= 1. */
int or_lcp_hist(const int32_t* entry_tokens, const int64_t* entry_off, int32_t n_entries,
                const int32_t* req_tokens, const int64_t* req_off, const int32_t* req_entry,
                int64_t n_requests, int32_t N, int32_t* hist, int32_t* lcp_out, int nthreads);

/* a3: P_j = sum_{t<=j} c_t, T_j = sum_{t<=j} t c_t, j = 0..N, P_0 = T_0 = 0 (Thm 2). */
int or_prefix(const int64_t* c, int32_t N, int64_t* P, int64_t* T);

/* a4 (definition): O(N^2 M) recurrence of Thm 2, w(s,j) in the form of P:758.
 * dp[0][j] = T_j, dp[m][0] = 0; opt[m][j] = leftmost argmin s (opt[0][*] = opt[*][0] = 0). */
int or_dp_naive(const int64_t* c, int32_t N, int32_t M, int64_t* dp, int32_t* opt);

/* a4 (paper's algorithm): monotone convex-hull trick, O(NM). */
int or_dp_cht(const int64_t* c, int32_t N, int32_t M, int64_t* dp, int32_t* opt);

/* a5: canonical backtrack ("rule B"): from (M, N) follow opt, stop when P_j == 0.
 * Writes at most M ascending positions; returns the count (>= 0). */
int or_backtrack(const int32_t* opt, const int64_t* P, int32_t N, int32_t M, int32_t* pos);

/* definitional objective: sum_{t=1}^N c_t (t - l(t;C)), l from P:133-137. */
int64_t or_expected_cost(const int64_t* c, int32_t N, const int32_t* pos, int32_t k);

/* definitional worst case max_{1<=t<=N} r(t;C) (distribution-free). */
int32_t or_worst_case(int32_t N, const int32_t* pos, int32_t k);

/* exhaustive search over all subsets of {1..N} of size <= M with the definitional cost;
 * returns the minimum cost in *cost and the colex-minimal optimal subset in pos. */
int or_brute_force(const int64_t* c, int32_t N, int32_t M, int32_t* pos, int32_t* k,
                   int64_t* cost);

/* Table 1 baselines. Return the number of positions written. */
int or_balanced(int32_t N, int32_t M, int32_t* pos);
int or_block(int32_t N, int32_t B, int32_t* pos);

/* fp64 variant reference: naive O(N^2 M) recurrence on real weights, computed in long double
 * (P:255-266).  dp as long double -> returned as double; opt leftmost argmin. */
int or_dp_naive_f64(const double* w, int32_t N, int32_t M, double* dp, int32_t* opt);
/* definitional fp64 objective, accumulated in long double. */
double or_expected_cost_f64(const double* w, int32_t N, const int32_t* pos, int32_t k);

/* f1 block-aware placement.
 * or_dp_grid_naive: the recurrence of Thm 2 with candidate positions restricted to multiples of
 *   B (the block-restricted DP of S:208): dp[m][j] = min over s in {B, 2B, ..} with s <= j.
 * or_clip_to_blocks: floor each position to a multiple of B, drop zeros, merge duplicates.
 * or_sqrt_positions: multiples of floor(sqrt(N)) up to N (Table 1).
 * or_log_positions: round(N (2^i - 1) / (2^M - 1)), i = 1..M, clamped to [1, N], deduplicated
 *   (SPEC's reading S:198 of P:358). Return the number of positions. */
int or_dp_grid_naive(const int64_t* c, int32_t N, int32_t M, int32_t B, int64_t* dp, int32_t* opt);
int or_clip_to_blocks(const int32_t* pos, int32_t k, int32_t B, int32_t* out);
int or_sqrt_positions(int32_t N, int32_t* out);
int or_log_positions(int32_t N, int32_t M, int32_t* out);

/* Batched drivers (threaded across entries, pthreads) used by tests and the CPU baseline.
 * hist: int32 [E][N+1].  algo: 0 = naive, 1 = CHT.  pos [E][M] zero-padded, npos [E],
 * cost [E] (= dp[M][N]), cost_by_budget [E][M+1] or NULL. */
int or_place_batch(const int32_t* hist, int32_t n_entries, int32_t N, int32_t M, int algo,
                   int32_t* pos, int32_t* npos, int64_t* cost, int64_t* cost_by_budget,
                   int nthreads);

/* Batched definitional evaluation.  If broadcast, positions is [S][max_pos] and n_positions
 * [S] shared by all entries, else [E][S][max_pos] and [E][S].  cost/worst are [E][S]. */
int or_eval_batch(const int32_t* hist, int32_t n_entries, int32_t N, const int32_t* positions,
                  const int32_t* n_positions, int32_t n_sets, int32_t max_pos, int broadcast,
                  int64_t* cost, int32_t* worst, int nthreads);

/* f2: Thm 4's exponentially weighted empirical histogram, definitional O(t N):
 * p[d] = (1-g)/(1-g^t) sum_{s<=t} g^(t-s) [T_s = d]  (g = 1: empirical frequencies).
 * depths[t] in arrival order; the samples T_s are the hits (depth >= 1, clamped to N): a miss
 * is not a sample of T in {1..N} (reading R15).  p[N+1] sums to 1 over bins
 * 1..N (bin 0 stays 0); all zero when the stream has no hit. */
int or_gamma_hist(const int32_t* depths, int64_t t, int32_t N, double gamma, double* p);
/* Thm 4's variance term sqrt(N (1-g)/(1+g) (1+g^t)/(1-g^t)). */
double or_gamma_variance_term(double gamma, int64_t t, int32_t N);

/* f4: longest-prefix match of each request against all cached entries,
 * brute force.  Ties -> most recent insertion (insertion[e], or the entry index when NULL; equal
 * values -> larger index); no match (max LCP 0) -> entry -1, depth 0.  Depth is the raw LCP. */
int or_match_longest_prefix(const int32_t* ent_tok, const int64_t* ent_off, int32_t E,
                            const int64_t* insertion, const int32_t* req_tok,
                            const int64_t* req_off, int64_t R, int32_t* match_entry,
                            int32_t* match_depth);

#ifdef __cplusplus
}
#endif
#endif
