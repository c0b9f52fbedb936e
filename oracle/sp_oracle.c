/*
 * oracle/sp_oracle.c -- TEST INFRASTRUCTURE ONLY (see sp_oracle.h).
 *
 * A plain, slow, obviously-correct CPU reference written from PAPER.md (arXiv 2605.05219).
 * Every function cites the passage it follows.  Nothing here is blocked, fused or reordered
 * beyond what the cited definition/algorithm states.  Integer arithmetic that could exceed
 * int64 is carried in __int128.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
 * may load the compiled liboracle.so; the CUDA product path shares no code with this file.
 */
#include "sp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

/* ------------------------------------------------------------------------------------------ */
/* a1 + a2: overlap depth of each request and the per-entry histogram.                         */
/* P:133-137 defines the overlap depth t as the number of leading tokens a request shares with */
/* the cached prefix; P:189-190 reduces the trie to independent single-prefix problems, so     */
/* each request is matched against its own entry; S:327 clamps depths beyond N to N.           */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  const int32_t *ent, *req, *req_entry;
  const int64_t *ent_off, *req_off;
  int32_t E, N;
  int64_t R;
  int32_t *hist, *lcp;
  int64_t next;
  int bad;
} lcp_job;

static void* lcp_worker(void* arg) {
  lcp_job* J = (lcp_job*)arg;
  for (;;) {
    int64_t r0 = __atomic_fetch_add(&J->next, 1024, __ATOMIC_RELAXED);
    if (r0 >= J->R) break;
    int64_t r1 = r0 + 1024 < J->R ? r0 + 1024 : J->R;
    for (int64_t r = r0; r < r1; ++r) {
      int32_t e = J->req_entry[r];
      if (e < 0 || e >= J->E) { __atomic_store_n(&J->bad, 1, __ATOMIC_RELAXED); continue; }
      int64_t eo = J->ent_off[e], el = J->ent_off[e + 1] - eo;
      int64_t ro = J->req_off[r], rl = J->req_off[r + 1] - ro;
      int64_t lim = el < rl ? el : rl;
      int64_t t = 0;
      while (t < lim && J->req[ro + t] == J->ent[eo + t]) ++t;   /* literal LCP loop */
      if (t > J->N) t = J->N;                                     /* clamp     */
      __atomic_fetch_add(&J->hist[(int64_t)e * (J->N + 1) + t], 1, __ATOMIC_RELAXED);
      if (J->lcp) J->lcp[r] = (int32_t)t;
    }
  }
  return NULL;
}

static int run_threads(void* (*fn)(void*), void* job, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads == 1) { fn(job); return 0; }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  if (!th) return -1;
  for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, fn, job);
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
  return 0;
}

int or_lcp_hist(const int32_t* entry_tokens, const int64_t* entry_off, int32_t n_entries,
                const int32_t* req_tokens, const int64_t* req_off, const int32_t* req_entry,
                int64_t n_requests, int32_t N, int32_t* hist, int32_t* lcp_out, int nthreads) {
  if (N < 1 || n_entries < 0 || n_requests < 0) return -1;
  lcp_job J = {entry_tokens, req_tokens, req_entry, entry_off, req_off, n_entries, N,
               n_requests, hist, lcp_out, 0, 0};
  if (run_threads(lcp_worker, &J, nthreads)) return -3;
  return J.bad ? -2 : 0;
}

/* ------------------------------------------------------------------------------------------ */
/* a3: prefix sums P_j = sum_{t=1}^j p_t, T_j = sum_{t=1}^j t p_t (Thm 2), with counts   */
/* c_t in place of p_t (p = c/n; the argmin is scale invariant).  P_0 = T_0 = 0 (used at s = 1 */
/* in w(s,j) = (T_j - T_{s-1}) - s (P_j - P_{s-1})).                                     */
/* ------------------------------------------------------------------------------------------ */
int or_prefix(const int64_t* c, int32_t N, int64_t* P, int64_t* T) {
  if (N < 1) return -1;
  P[0] = 0;
  T[0] = 0;
  for (int32_t j = 1; j <= N; ++j) {
    P[j] = P[j - 1] + c[j];
    T[j] = T[j - 1] + (int64_t)j * c[j];
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* a4, definition: Thm 2                                                          */
/*   dp[0,j] = sum_{t<=j} p_t t = T_j                                                          */
/*   dp[m,j] = min_{1<=s<=j} dp[m-1,s-1] + w(s,j),   w(s,j) = sum_{t=s}^j p_t (t-s)   */
/* evaluated directly in O(N^2 M) with w(s,j) = (T_j - T_{s-1}) - s(P_j - P_{s-1}).      */
/* The paper leaves dp[m>=1, 0] undefined (a min over an empty set); we take 0 (the */
/* "at most m checkpoints" reading; reading R1).  s is scanned upward with a strict  */
/* '<', so opt[m][j] is the lowest-index (leftmost) argmin (reading R3).              */
/* ------------------------------------------------------------------------------------------ */
int or_dp_naive(const int64_t* c, int32_t N, int32_t M, int64_t* dp, int32_t* opt) {
  if (N < 1) return -1;
  if (M < 0 || M > N) return -2;
  int64_t* P = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
  int64_t* T = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
  if (!P || !T) { free(P); free(T); return -3; }
  or_prefix(c, N, P, T);
  const int64_t W = (int64_t)N + 1;
  for (int32_t j = 0; j <= N; ++j) { dp[j] = T[j]; opt[j] = 0; }
  for (int32_t m = 1; m <= M; ++m) {
    dp[m * W + 0] = 0;
    opt[m * W + 0] = 0;
    for (int32_t j = 1; j <= N; ++j) {
      i128 best = 0;
      int32_t arg = -1;
      for (int32_t s = 1; s <= j; ++s) {
        i128 w = (i128)(T[j] - T[s - 1]) - (i128)s * (P[j] - P[s - 1]);
        i128 v = (i128)dp[(m - 1) * W + (s - 1)] + w;
        if (arg < 0 || v < best) { best = v; arg = s; }
      }
      dp[m * W + j] = (int64_t)best;
      opt[m * W + j] = arg;
    }
  }
  free(P);
  free(T);
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* a4, the paper's algorithm: monotone convex-hull trick (Thm 2; proof P:755-773).   */
/*   dp[m,j] = T_j + min_{1<=s<=j} (dp[m-1,s-1] - T_{s-1} + s P_{s-1} - s P_j)   */
/* Line s: slope -s, intercept B_s = dp[m-1,s-1] - T_{s-1} + s P_{s-1}, queried at x = P_j.    */
/* Slopes strictly decrease in s; queries are non-decreasing in j.  Lines are      */
/* added in order s = 1..N, line j before query j (the constraint s <= j).                      */
/* Tie handling ("the monotone-pointer technique handles ties") made precise as     */
/* the back pops a middle line b between a and the new line c iff                   */
/*   (B_c - B_a)(s_b - s_a) <= (B_b - B_a)(s_c - s_a)                                          */
/* (b is never the leftmost minimum), and the front advances only when the next line is        */
/* STRICTLY better at x = P_j, so the reported argmin is the leftmost one.                     */
/* ------------------------------------------------------------------------------------------ */
int or_dp_cht(const int64_t* c, int32_t N, int32_t M, int64_t* dp, int32_t* opt) {
  if (N < 1) return -1;
  if (M < 0 || M > N) return -2;
  int64_t* P = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
  int64_t* T = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
  int32_t* ls = (int32_t*)malloc(sizeof(int32_t) * (size_t)(N + 1));
  i128* lb = (i128*)malloc(sizeof(i128) * (size_t)(N + 1));
  if (!P || !T || !ls || !lb) { free(P); free(T); free(ls); free(lb); return -3; }
  or_prefix(c, N, P, T);
  const int64_t W = (int64_t)N + 1;
  for (int32_t j = 0; j <= N; ++j) { dp[j] = T[j]; opt[j] = 0; }
  for (int32_t m = 1; m <= M; ++m) {
    const int64_t* prev = dp + (m - 1) * W;
    dp[m * W + 0] = 0;
    opt[m * W + 0] = 0;
    int32_t head = 0, tail = 0;
    for (int32_t j = 1; j <= N; ++j) {
      /* add line s = j */
      i128 Bj = (i128)prev[j - 1] - T[j - 1] + (i128)j * P[j - 1];
      while (tail - head >= 2) {
        int32_t a = tail - 2, b = tail - 1;
        i128 lhs = (Bj - lb[a]) * (i128)(ls[b] - ls[a]);
        i128 rhs = (lb[b] - lb[a]) * (i128)(j - ls[a]);
        if (lhs <= rhs) --tail; else break;
      }
      ls[tail] = j;
      lb[tail] = Bj;
      ++tail;
      /* query x = P_j */
      i128 x = P[j];
      while (tail - head >= 2) {
        i128 v0 = lb[head] - (i128)ls[head] * x;
        i128 v1 = lb[head + 1] - (i128)ls[head + 1] * x;
        if (v1 < v0) ++head; else break;
      }
      i128 v = lb[head] - (i128)ls[head] * x;
      dp[m * W + j] = (int64_t)(T[j] + v);
      opt[m * W + j] = ls[head];
    }
  }
  free(P); free(T); free(ls); free(lb);
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* a5: argmin backtrack.  The paper fixes only the recurrence; SURVEY F3 fixes the  */
/* canonical output ("rule B", reading R3): start at (m, j) = (M, N); while m > 0 and */
/* P_j > 0: s = opt[m][j], emit s, j = s - 1, m = m - 1.  Emitted positions are reversed into  */
/* ascending order.                                                                             */
/* ------------------------------------------------------------------------------------------ */
int or_backtrack(const int32_t* opt, const int64_t* P, int32_t N, int32_t M, int32_t* pos) {
  const int64_t W = (int64_t)N + 1;
  int32_t j = N, m = M, k = 0;
  while (m > 0 && P[j] > 0) {
    int32_t s = opt[m * W + j];
    pos[k++] = s;
    j = s - 1;
    --m;
  }
  for (int32_t a = 0, b = k - 1; a < b; ++a, --b) { int32_t t = pos[a]; pos[a] = pos[b]; pos[b] = t; }
  return k;
}

/* ------------------------------------------------------------------------------------------ */
/* Definitional objective: E[r(T;C)] = sum_{t=1}^N p_t (t - l(t;C)), with          */
/* l(t;C) = max({0} U {c in C : c <= t}), here with counts (numerator n E[r]).     */
/* ------------------------------------------------------------------------------------------ */
static int32_t reusable_depth(const int32_t* pos, int32_t k, int32_t t) {
  int32_t l = 0;                                     /* max({0} U {c in C : c <= t}) */
  for (int32_t i = 0; i < k; ++i)
    if (pos[i] <= t && pos[i] > l) l = pos[i];
  return l;
}

int64_t or_expected_cost(const int64_t* c, int32_t N, const int32_t* pos, int32_t k) {
  i128 s = 0;
  for (int32_t t = 1; t <= N; ++t) s += (i128)c[t] * (t - reusable_depth(pos, k, t));
  return (int64_t)s;
}

/* worst case max_t r(t;C) over ALL t in 1..N (distribution-free; Thm 1.2). */
int32_t or_worst_case(int32_t N, const int32_t* pos, int32_t k) {
  int32_t w = 0;
  for (int32_t t = 1; t <= N; ++t) {
    int32_t r = t - reusable_depth(pos, k, t);
    if (r > w) w = r;
  }
  return w;
}

/* ------------------------------------------------------------------------------------------ */
/* Brute force: every C subset of {1..N} with |C| <= M (budget semantics),     */
/* definitional cost above.  Among optimal sets return the colex-minimal one: compare the      */
/* descending sequences lexicographically, a proper prefix first.                   */
/* ------------------------------------------------------------------------------------------ */
static int colex_less(const int32_t* a, int32_t ka, const int32_t* b, int32_t kb) {
  int32_t i = ka - 1, j = kb - 1;
  while (i >= 0 && j >= 0) {
    if (a[i] != b[j]) return a[i] < b[j];
    --i; --j;
  }
  return ka < kb;   /* a is a proper prefix (in descending order) of b */
}

int or_brute_force(const int64_t* c, int32_t N, int32_t M, int32_t* pos, int32_t* k,
                   int64_t* cost) {
  if (N < 1) return -1;
  if (M < 0 || M > N) return -2;
  int32_t cur[64] = {0}, best[64] = {0};
  if (M > 64) return -4;
  int64_t best_cost = or_expected_cost(c, N, cur, 0);   /* the empty set */
  int32_t best_k = 0;
  for (int32_t size = 1; size <= M; ++size) {
    for (int32_t i = 0; i < size; ++i) cur[i] = i + 1;   /* first combination */
    for (;;) {
      int64_t v = or_expected_cost(c, N, cur, size);
      if (v < best_cost || (v == best_cost && colex_less(cur, size, best, best_k))) {
        best_cost = v;
        best_k = size;
        memcpy(best, cur, sizeof(int32_t) * (size_t)size);
      }
      int32_t i = size - 1;                                /* next combination */
      while (i >= 0 && cur[i] == N - size + i + 1) --i;
      if (i < 0) break;
      ++cur[i];
      for (int32_t q = i + 1; q < size; ++q) cur[q] = cur[q - 1] + 1;
    }
  }
  memcpy(pos, best, sizeof(int32_t) * (size_t)best_k);
  *k = best_k;
  *cost = best_cost;
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Table 1 baselines.  Balanced: floor(i (L+1) / (M+1)), i = 1..M.  Block:  */
/* B, 2B, ..., floor(L/B) B.                                                            */
/* ------------------------------------------------------------------------------------------ */
int or_balanced(int32_t N, int32_t M, int32_t* pos) {
  if (N < 1) return -1;
  if (M < 0 || M > N) return -2;
  for (int32_t i = 1; i <= M; ++i) pos[i - 1] = (int32_t)(((int64_t)i * (N + 1)) / (M + 1));
  return M;
}

int or_block(int32_t N, int32_t B, int32_t* pos) {
  if (N < 1 || B < 1) return -1;
  int32_t k = 0;
  for (int64_t p = B; p <= N; p += B) pos[k++] = (int32_t)p;
  return k;
}

/* ------------------------------------------------------------------------------------------ */
/* fp64 variant: the same recurrence on real weights p_t, evaluated in long double */
/* (64-bit mantissa) so that its own rounding is far below the 1e-12 tolerance being tested.   */
/* ------------------------------------------------------------------------------------------ */
int or_dp_naive_f64(const double* w, int32_t N, int32_t M, double* dp, int32_t* opt) {
  if (N < 1) return -1;
  if (M < 0 || M > N) return -2;
  long double* P = (long double*)malloc(sizeof(long double) * (size_t)(N + 1));
  long double* T = (long double*)malloc(sizeof(long double) * (size_t)(N + 1));
  long double* D = (long double*)malloc(sizeof(long double) * (size_t)(M + 1) * (size_t)(N + 1));
  if (!P || !T || !D) { free(P); free(T); free(D); return -3; }
  P[0] = 0; T[0] = 0;
  for (int32_t j = 1; j <= N; ++j) { P[j] = P[j - 1] + w[j]; T[j] = T[j - 1] + (long double)j * w[j]; }
  const int64_t W = (int64_t)N + 1;
  for (int32_t j = 0; j <= N; ++j) { D[j] = T[j]; opt[j] = 0; }
  for (int32_t m = 1; m <= M; ++m) {
    D[m * W] = 0;
    opt[m * W] = 0;
    for (int32_t j = 1; j <= N; ++j) {
      long double best = 0;
      int32_t arg = -1;
      for (int32_t s = 1; s <= j; ++s) {
        long double v = D[(m - 1) * W + s - 1] + (T[j] - T[s - 1]) - (long double)s * (P[j] - P[s - 1]);
        if (arg < 0 || v < best) { best = v; arg = s; }
      }
      D[m * W + j] = best;
      opt[m * W + j] = arg;
    }
  }
  for (int64_t i = 0; i < (int64_t)(M + 1) * W; ++i) dp[i] = (double)D[i];
  free(P); free(T); free(D);
  return 0;
}

double or_expected_cost_f64(const double* w, int32_t N, const int32_t* pos, int32_t k) {
  long double s = 0;
  for (int32_t t = 1; t <= N; ++t) s += (long double)w[t] * (t - reusable_depth(pos, k, t));
  return (double)s;
}

/* ------------------------------------------------------------------------------------------ */
/* f1: block-aware placement.  The block-restricted DP (S:206-214 candidate_grid) is Thm 2's   */
/* recurrence with the last checkpoint s restricted to multiples of B; with the    */
/* at-most reading R1 dp[m][0..B-1] is the no-checkpoint cost T_j.  Leftmost argmin as before.  */
/* ------------------------------------------------------------------------------------------ */
int or_dp_grid_naive(const int64_t* c, int32_t N, int32_t M, int32_t B, int64_t* dp, int32_t* opt) {
  if (N < 1 || B < 1) return -1;
  if (M < 0 || M > N) return -2;
  int64_t* P = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
  int64_t* T = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
  if (!P || !T) { free(P); free(T); return -3; }
  or_prefix(c, N, P, T);
  const int64_t W = (int64_t)N + 1;
  for (int32_t j = 0; j <= N; ++j) { dp[j] = T[j]; opt[j] = 0; }
  for (int32_t m = 1; m <= M; ++m) {
    for (int32_t j = 0; j <= N; ++j) {
      if (j < B) {                  /* no grid position at or below j: no checkpoint usable */
        dp[m * W + j] = T[j];
        opt[m * W + j] = 0;
        continue;
      }
      i128 best = 0;
      int32_t arg = 0;
      for (int32_t s = B; s <= j; s += B) {   /* leftmost argmin over grid candidates */
        i128 w = (i128)(T[j] - T[s - 1]) - (i128)s * (P[j] - P[s - 1]);
        i128 v = (i128)dp[(m - 1) * W + (s - 1)] + w;
        if (arg == 0 || v < best) { best = v; arg = s; }
      }
      dp[m * W + j] = (int64_t)best;
      opt[m * W + j] = arg;
    }
  }
  free(P);
  free(T);
  return 0;
}

int or_clip_to_blocks(const int32_t* pos, int32_t k, int32_t B, int32_t* out) {
  if (B < 1 || k < 0) return -1;
  int32_t n = 0;
  for (int32_t i = 0; i < k; ++i) {
    int32_t f = (pos[i] / B) * B;            /* clip DOWN: a state above t cannot serve t */
    if (f <= 0) continue;                   /* zeros dropped */
    if (n > 0 && out[n - 1] == f) continue; /* duplicates merged (input ascending) */
    out[n++] = f;
  }
  return n;
}

int or_sqrt_positions(int32_t N, int32_t* out) {
  if (N < 1) return -1;
  int32_t q = 1;
  while ((int64_t)(q + 1) * (q + 1) <= N) ++q;   /* floor(sqrt(N)) */
  return or_block(N, q, out);
}

int or_log_positions(int32_t N, int32_t M, int32_t* out) {
  if (N < 1) return -1;
  if (M < 1 || M > N || M > 62) return -2;
  const i128 den = ((i128)1 << M) - 1;
  int32_t n = 0;
  for (int32_t i = 1; i <= M; ++i) {
    const i128 num = (i128)N * (((i128)1 << i) - 1);
    int64_t r = (int64_t)((2 * num + den) / (2 * den));   /* round half up */
    if (r < 1) r = 1;
    if (r > N) r = N;
    if (n > 0 && out[n - 1] >= r) continue;
    out[n++] = (int32_t)r;
  }
  return n;
}

/* ------------------------------------------------------------------------------------------ */
/* Batched drivers: one entry at a time per thread (entries are independent problems,          */
/* P:189-190).                                                                                  */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  const int32_t* hist;
  int32_t E, N, M, algo;
  int32_t *pos, *npos;
  int64_t *cost, *cbb;
  int32_t next;
  int err;
} place_job;

static void* place_worker(void* arg) {
  place_job* J = (place_job*)arg;
  const int64_t W = (int64_t)J->N + 1;
  int64_t* c = (int64_t*)malloc(sizeof(int64_t) * (size_t)W);
  int64_t* P = (int64_t*)malloc(sizeof(int64_t) * (size_t)W);
  int64_t* T = (int64_t*)malloc(sizeof(int64_t) * (size_t)W);
  int64_t* dp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(J->M + 1) * (size_t)W);
  int32_t* opt = (int32_t*)malloc(sizeof(int32_t) * (size_t)(J->M + 1) * (size_t)W);
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(J->M + 1));
  if (!c || !P || !T || !dp || !opt || !tmp) { J->err = -3; goto out; }
  for (;;) {
    int32_t e = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    if (e >= J->E) break;
    for (int64_t t = 0; t < W; ++t) c[t] = J->hist[(int64_t)e * W + t];
    int rc = J->algo == 0 ? or_dp_naive(c, J->N, J->M, dp, opt) : or_dp_cht(c, J->N, J->M, dp, opt);
    if (rc) { J->err = rc; continue; }
    or_prefix(c, J->N, P, T);
    int32_t k = or_backtrack(opt, P, J->N, J->M, tmp);
    for (int32_t i = 0; i < J->M; ++i) J->pos[(int64_t)e * J->M + i] = i < k ? tmp[i] : 0;
    J->npos[e] = k;
    J->cost[e] = dp[(int64_t)J->M * W + J->N];
    if (J->cbb)
      for (int32_t m = 0; m <= J->M; ++m) J->cbb[(int64_t)e * (J->M + 1) + m] = dp[(int64_t)m * W + J->N];
  }
out:
  free(c); free(P); free(T); free(dp); free(opt); free(tmp);
  return NULL;
}

int or_place_batch(const int32_t* hist, int32_t n_entries, int32_t N, int32_t M, int algo,
                   int32_t* pos, int32_t* npos, int64_t* cost, int64_t* cost_by_budget,
                   int nthreads) {
  if (N < 1 || n_entries < 0) return -1;
  if (M < 0 || M > N) return -2;
  place_job J = {hist, n_entries, N, M, algo, pos, npos, cost, cost_by_budget, 0, 0};
  if (run_threads(place_worker, &J, nthreads)) return -3;
  return J.err;
}

typedef struct {
  const int32_t *hist, *positions, *npos;
  int32_t E, N, S, max_pos;
  int broadcast;
  int64_t* cost;
  int32_t* worst;
  int32_t next;
  int err;
} eval_job;

static void* eval_worker(void* arg) {
  eval_job* J = (eval_job*)arg;
  const int64_t W = (int64_t)J->N + 1;
  int64_t* c = (int64_t*)malloc(sizeof(int64_t) * (size_t)W);
  if (!c) { J->err = -3; return NULL; }
  for (;;) {
    int32_t e = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    if (e >= J->E) break;
    for (int64_t t = 0; t < W; ++t) c[t] = J->hist[(int64_t)e * W + t];
    for (int32_t q = 0; q < J->S; ++q) {
      int64_t set = J->broadcast ? q : (int64_t)e * J->S + q;
      const int32_t* p = J->positions + set * J->max_pos;
      int32_t k = J->npos[set];
      int ok = k >= 0 && k <= J->max_pos;
      for (int32_t i = 0; ok && i < k; ++i)
        if (p[i] < 1 || p[i] > J->N || (i > 0 && p[i] <= p[i - 1])) ok = 0;
      if (!ok) { J->err = -5; continue; }
      J->cost[(int64_t)e * J->S + q] = or_expected_cost(c, J->N, p, k);
      if (J->worst) J->worst[(int64_t)e * J->S + q] = or_worst_case(J->N, p, k);
    }
  }
  free(c);
  return NULL;
}

int or_eval_batch(const int32_t* hist, int32_t n_entries, int32_t N, const int32_t* positions,
                  const int32_t* n_positions, int32_t n_sets, int32_t max_pos, int broadcast,
                  int64_t* cost, int32_t* worst, int nthreads) {
  if (N < 1 || n_entries < 0 || n_sets < 0 || max_pos < 0) return -1;
  eval_job J = {hist, positions, n_positions, n_entries, N, n_sets, max_pos, broadcast,
                cost, worst, 0, 0};
  if (run_threads(eval_worker, &J, nthreads)) return -3;
  return J.err;
}

/* ------------------------------------------------------------------------------------------ */
/* f2: the exponentially weighted empirical histogram of Thm 4, written out as its */
/* definition: p_t = (1 - g) / (1 - g^t) * sum_{s=1..t} g^(t-s) e_{T_s}, 0 < g < 1, and the   */
/* plain empirical distribution (1/t) sum_s e_{T_s} for g = 1 (Thm 3's estimator).  Depths are */
/* clamped to [0, N] (S:327 design decision; bin 0 = miss).  O(t) per call, long double.      */
/* ------------------------------------------------------------------------------------------ */
int or_gamma_hist(const int32_t* depths, int64_t t, int32_t N, double gamma, double* p) {
  if (N < 1 || t < 0 || !(gamma > 0.0 && gamma <= 1.0)) return -1;
  /* the samples T_s are the HITS of the stream, in order: T in {1..N}, conditioning on
     hits (DESIGN reading R15); a miss (depth < 1) is not a sample */
  int64_t h = 0;
  for (int64_t s = 0; s < t; ++s) h += depths[s] >= 1;
  for (int32_t d = 0; d <= N; ++d) p[d] = 0.0;
  if (h == 0) return 0;
  long double* acc = (long double*)calloc((size_t)N + 1, sizeof(long double));
  if (!acc) return -3;
  int64_t s = 0;   /* sample index 1..h */
  for (int64_t i = 0; i < t; ++i) {
    int32_t d = depths[i];
    if (d < 1) continue;
    ++s;
    if (d > N) d = N;                                              /* clamp */
    acc[d] += powl((long double)gamma, (long double)(h - s));     /* gamma^(t-s) e_{T_s} */
  }
  long double norm;
  if (gamma == 1.0) norm = 1.0L / (long double)h;
  else norm = (1.0L - (long double)gamma) / (1.0L - powl((long double)gamma, (long double)h));
  for (int32_t d = 0; d <= N; ++d) p[d] = (double)(acc[d] * norm);
  free(acc);
  return 0;
}

/* Thm 4's variance term sqrt(N (1-g)/(1+g) (1+g^t)/(1-g^t)), closed form. */
double or_gamma_variance_term(double gamma, int64_t t, int32_t N) {
  const long double g = gamma, gt = powl(g, (long double)t);
  return (double)sqrtl((long double)N * (1.0L - g) / (1.0L + g) * (1.0L + gt) / (1.0L - gt));
}

/* ------------------------------------------------------------------------------------------ */
/* f4: longest-prefix match of each request against ALL cached entries (the trie remark of     */
/* P:189-190; SPEC match_longest_prefix S:375-383), by brute force: the literal LCP loop against */
/* every entry, keeping the maximum; ties -> the most recent insertion (largest insertion[e],  */
/* entry index when insertion == NULL; equal insertion values -> larger entry index); a maximum */
/* of 0 -> no match (entry -1, depth 0).                                                      */
/* ------------------------------------------------------------------------------------------ */
int or_match_longest_prefix(const int32_t* ent_tok, const int64_t* ent_off, int32_t E,
                            const int64_t* insertion, const int32_t* req_tok,
                            const int64_t* req_off, int64_t R, int32_t* match_entry,
                            int32_t* match_depth) {
  if (E < 0 || R < 0) return -1;
  for (int64_t r = 0; r < R; ++r) {
    const int32_t* q = req_tok + req_off[r];
    const int64_t ql = req_off[r + 1] - req_off[r];
    int64_t best = 0;
    int32_t who = -1;
    for (int32_t e = 0; e < E; ++e) {
      const int32_t* x = ent_tok + ent_off[e];
      const int64_t xl = ent_off[e + 1] - ent_off[e];
      int64_t t = 0;
      while (t < ql && t < xl && q[t] == x[t]) ++t;
      if (t == 0) continue;
      if (t > best) { best = t; who = e; continue; }
      if (t == best) {
        const int64_t iw = insertion ? insertion[who] : who, ie = insertion ? insertion[e] : e;
        if (ie > iw || (ie == iw && e > who)) who = e;
      }
    }
    match_entry[r] = who;
    match_depth[r] = (int32_t)best;
  }
  return 0;
}
