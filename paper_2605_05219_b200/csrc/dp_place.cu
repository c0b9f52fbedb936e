// dp_place.cu -- a3 + a4 + a5 (+ a7): prefix sums, the exact checkpoint-placement DP and the
// argmin backtrack (Thm 2; proof P:755-774).  SURVEY 8(a) rows a3-a5, a7.
//
// Per layer m the DP is a row-minimum problem on the matrix
//     A_m[j][s] = b_s - s P_j      (1 <= s <= j),   b_s = e_{m-1}(s-1) + s P_{s-1}
// where e_m(j) = dp[m][j] - T_j (the rewrite of P:760-762; T_j cancels out of every comparison,
// so only T_N is ever needed).  A_m is totally monotone (w(s,j) is Monge), so the
// leftmost row argmin opt_m(j) is non-decreasing in j.  Instead of the paper's sequential
// convex-hull trick we solve each layer with a level-synchronous divide-and-conquer over rows:
// at level k every row j = h(2i+1) (h = 2^(L-1-k)) is solved with the bracket
//     [max(opt_m(j-h), opt_{m-1}(j)), min(opt_m(j+h), j)]
// (neighbours solved at earlier levels; opt_{m-1}(j) <= opt_m(j) is the layer bound, DESIGN.md
// reading R6).  Candidates of a row are split across a group of G threads (G chosen per level
// so each thread does ~8 evaluations) and reduced with a lexicographic (value, index) shuffle
// min, which makes every argmin the lowest index (reading R3).  No tensor cores: min-plus.
//
// Layout: one CTA per entry (persistent grid, entries strided over CTAs).  b_s lives in shared
// memory (int32 when the guard 2 n N < 2^31 makes 32-bit arithmetic exact -- bit-identical
// results; int64 / double otherwise, then in the slot's global/L2 scratch); opt_m(j) for the
// current layer lives in shared memory (uint16); P_j, b_next and the full argmin table
// opt[M][N+1] (uint16) live in the CTA's workspace slot.
#include <map>
#include <mutex>
#include <utility>
#include <climits>
#include <cstdlib>
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "dp_internal.cuh"

namespace sp {

#ifndef SP_DP_NT
#define SP_DP_NT 1024
#endif
constexpr int DP_NT = SP_DP_NT;
constexpr int DP_NW = DP_NT / 32;
constexpr int T_INLINE = 8;   // rows with at most this many candidates: one thread solves it
constexpr int PS = 64;        // candidates per piece of a queued (long) row (top levels)
constexpr int QMAX = 128;     // queued rows per top level
constexpr int PMAX = 1024;    // pieces per top level
constexpr int RB = 2;         // rows per thread per batch in the bracket pass
#ifndef SP_SEG_ROWS
#define SP_SEG_ROWS 512
#endif
constexpr int SEG_ROWS = SP_SEG_ROWS; // rows per warp-owned segment (the subtree below the top levels)
#ifndef SP_WCAP
#define SP_WCAP 32
#endif
constexpr int WCAP = SP_WCAP;      // long rows a warp can defer per segment level
#ifndef SP_TW
#define SP_TW 8
#endif
constexpr int TW = SP_TW;         // rows longer than this are solved warp-cooperatively

// ------------------------------------------------------------------------------------------
// value-type traits
// ------------------------------------------------------------------------------------------
template <typename VT>
struct Lim;
template <>
struct Lim<int32_t> {
  static __device__ __forceinline__ int32_t inf() { return INT_MAX; }
};
template <>
struct Lim<int64_t> {
  static __device__ __forceinline__ int64_t inf() { return LLONG_MAX; }
};
template <>
struct Lim<double> {
  static __device__ __forceinline__ double inf() { return INFINITY; }
};

// candidate value b_s - s P_j (exact for the integer types; one rounding for double)
__device__ __forceinline__ int32_t cand(int32_t b, int s, int32_t Pj) { return b - s * Pj; }
__device__ __forceinline__ int64_t cand(int64_t b, int s, int64_t Pj) { return b - (int64_t)s * Pj; }
__device__ __forceinline__ double cand(double b, int s, double Pj) { return fma(-(double)s, Pj, b); }
// next-layer intercept e + s P
__device__ __forceinline__ int32_t icpt(int32_t e, int s, int32_t P) { return e + s * P; }
__device__ __forceinline__ int64_t icpt(int64_t e, int s, int64_t P) { return e + (int64_t)s * P; }
__device__ __forceinline__ double icpt(double e, int s, double P) { return fma((double)s, P, e); }

// weight type -> prefix / cost type
template <typename WT>
struct WTraits {
  using PT = int64_t;   // P_j storage
  using CT = int64_t;   // cost type
};
template <>
struct WTraits<double> {
  using PT = double;
  using CT = double;
};

// ------------------------------------------------------------------------------------------
// double-double helpers (a7: compensated prefix sums and final cost)
// ------------------------------------------------------------------------------------------
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  double s = a.hi + b.hi;
  double bb = s - a.hi;
  double err = (a.hi - (s - bb)) + (b.hi - bb);
  err += a.lo + b.lo;
  double h = s + err;
  return dd{h, err - (h - s)};
}
__device__ __forceinline__ dd dd_from_prod(double a, double b) {
  double p = a * b;
  return dd{p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_shfl_up(dd v, int o) {
  return dd{__shfl_up_sync(FULL, v.hi, o), __shfl_up_sync(FULL, v.lo, o)};
}
__device__ __forceinline__ dd dd_shfl_xor(dd v, int o) {
  return dd{__shfl_xor_sync(FULL, v.hi, o), __shfl_xor_sync(FULL, v.lo, o)};
}

__host__ __device__ __forceinline__ size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// workspace slot layout (bytes):
//   P 8B[N+1] | bA 8B[N+1] | bB 8B[N+1] | opt uint16[M][N+1] | P32 int32[N+1]
__host__ __device__ __forceinline__ size_t slot_opt_off(int N) { return 3 * align256(8 * (size_t)(N + 1)); }
// argmin-table row stride: N+1 rounded up to 8 entries so every row is 16-byte aligned
__host__ __device__ __forceinline__ int opt_ld(int N) { return (N + 1 + 7) & ~7; }
__host__ __device__ __forceinline__ size_t slot_p32_off(int N, int M) {
  return slot_opt_off(N) + align256(2 * (size_t)(M > 0 ? M : 1) * opt_ld(N));
}
__host__ __device__ __forceinline__ size_t slot_bytes(int N, int M) {
  return slot_p32_off(N, M) + align256(4 * (size_t)(N + 1));
}

struct DpParams {
  const void* w;
  int E, N, M, L;
  int32_t* pos;
  int32_t* npos;
  void* cost;
  void* cbb;
  uint8_t* ws;
  size_t slot;
  int smem_b;   // 1: the int32 b array fits in shared memory next to opt_m
  int32_t* fpos;   // f3 frontier: [E][M][M] positions of every budget m = 1..M (row m-1), or NULL
  int32_t* fn;     // f3 frontier: [E][M] counts (or a negative status), or NULL
  uint8_t* slots;  // this kernel's per-CTA slots
  const int32_t* list;     // entries to solve (the hull kernel's fallbacks), or NULL = all E
  const unsigned* list_n;  // device count of `list`
};

constexpr int TOPP_CAP = 160;
constexpr int TQCAP = 2048;   // task-pool slots
#ifdef SP_TIMING
#define SP_T0() long long _t = clock64()
#define SP_TICK(sh, i)                                                  \
  do {                                                                  \
    const long long _n = clock64();                                     \
    if (threadIdx.x == 0) (sh).tclk[i] += (unsigned long long)(_n - _t); \
    _t = _n;                                                            \
  } while (0)
#else
#define SP_T0() (void)0
#define SP_TICK(sh, i) (void)0
#endif
struct Shared {
  uint64_t mbar;                  // TMA bulk-copy completion barrier
  int64_t topP[TOPP_CAP];         // P_j of the top-level rows (j multiple of h0), as VT
  unsigned long long tclk[10];    // SP_TIMING: per-phase cycles of this CTA
  unsigned long long ctr[3];      // per-level queue counters (triple-buffered)
  int segctr;                     // next segment to grab
  int tq[TQCAP];                  // task pool slots (-1 = not yet pushed)
  int tq_head, tq_tail, tq_total;
  int nmulti[3];                  // queued rows with more than one piece
  unsigned long long evals;
  int64_t wbuf[DP_NW + 1];
  double dbuf[2 * (DP_NW + 1)];
  int32_t red_s[DP_NW];
  unsigned phase;
  int err;
};

template <typename VT, typename PT, typename CT>
struct LayerCtx {
  VT* b;                    // b_s, s = 1..N (shared or global)
  VT* bnext;                // global
  uint16_t* sopt;           // shared opt_m
  uint16_t* optout;         // global opt table row m
  const uint16_t* optprev;  // global opt table row m-1 (NULL at m = 1)
  const PT* P;              // global P_j
  int N, m;
  CT TN;
  CT* cbb_e;                // cost_by_budget row of this entry or NULL
  CT* cost_e;               // cost of this entry, written at m == M
  bool last;                // m == M
  int* err;
};

// scratch for the long-row queue of one level, carved from dynamic shared memory
template <typename VT>
struct Scratch {
  int* qj;     // [QMAX] row j
  int* qlo;    // [QMAX] bracket low end
  int* qlen;   // [QMAX] bracket length (0 = dead entry)
  int* qpb;    // [QMAX] first piece
  VT* qP;      // [QMAX] P_j
  VT* pv;      // [PMAX] piece minima
  int* ps;     // [PMAX] piece argmins
};

template <typename VT>
__host__ __device__ __forceinline__ size_t wlist_bytes() {
  return (size_t)DP_NW * WCAP * (12 + sizeof(VT));
}

constexpr int TOPR = 64;   // rows a lean top level handles
template <typename VT>
__host__ __device__ __forceinline__ size_t top_scratch_bytes() {
  return (size_t)TOPR * DP_NW * (sizeof(VT) + 4) + 3 * TOPR * 4;
}

template <typename VT>
__host__ __device__ __forceinline__ size_t scratch_bytes() {
  const size_t q = align256((size_t)QMAX * (16 + sizeof(VT))) + align256((size_t)PMAX * (4 + sizeof(VT)));
  const size_t w = align256(wlist_bytes<VT>());
  const size_t t = align256(top_scratch_bytes<VT>());
  const size_t m = q > w ? q : w;   // the phases never overlap: one union
  return m > t ? m : t;
}

template <typename VT>
__device__ __forceinline__ Scratch<VT> carve(uint8_t* base) {
  Scratch<VT> S;
  S.qj = reinterpret_cast<int*>(base);
  S.qlo = S.qj + QMAX;
  S.qlen = S.qlo + QMAX;
  S.qpb = S.qlen + QMAX;
  S.qP = reinterpret_cast<VT*>(S.qpb + QMAX);
  uint8_t* b2 = base + align256((size_t)QMAX * (16 + sizeof(VT)));
  S.pv = reinterpret_cast<VT*>(b2);
  S.ps = reinterpret_cast<int*>(S.pv + PMAX);
  return S;
}

template <typename VT>
__device__ __forceinline__ void lex_min(VT& bv, int& bs, VT ov, int os) {
  if (ov < bv || (ov == bv && os < bs)) {
    bv = ov;
    bs = os;
  }
}

template <typename VT>
__device__ __forceinline__ VT vmin(VT a, VT b) { return a < b ? a : b; }

// Leftmost argmin of b_s - s P_j over s = s0, s0 + st, ... <= s1 (s increasing).  The main loop
// takes groups of four: the group minimum (2 min instructions for int32: VIMNMX + VIMNMX3)
// replaces the running minimum only when strictly smaller, so the first group holding the
// minimum wins; its lowest candidate equal to the minimum is recovered afterwards.
template <typename VT>
__device__ __forceinline__ void eval_range(const VT* __restrict__ b, VT Pj, int s0, int s1,
                                           int st, VT& bv, int& bs) {
  VT best = Lim<VT>::inf();
  int bg = -1;
  int s = s0;
  for (; s + 3 * st <= s1; s += 4 * st) {
    const VT v0 = cand(b[s], s, Pj);
    const VT v1 = cand(b[s + st], s + st, Pj);
    const VT v2 = cand(b[s + 2 * st], s + 2 * st, Pj);
    const VT v3 = cand(b[s + 3 * st], s + 3 * st, Pj);
    const VT m = vmin(vmin(v0, v1), vmin(v2, v3));
    if (m < best) {
      best = m;
      bg = s;
    }
  }
  int arg = INT_MAX;
  if (bg >= 0) {
#pragma unroll
    for (int k = 3; k >= 0; --k)
      if (cand(b[bg + k * st], bg + k * st, Pj) == best) arg = bg + k * st;
  }
  for (; s <= s1; s += st) {
    const VT v = cand(b[s], s, Pj);
    if (v < best) {
      best = v;
      arg = s;
    }
  }
  bv = best;
  bs = arg;
}

// plain leftmost argmin over s = s0..s1 (short rows)
template <typename VT>
__device__ __forceinline__ void eval_short(const VT* __restrict__ b, VT Pj, int s0, int s1,
                                           VT& bv, int& bs) {
  VT best = Lim<VT>::inf();
  int arg = INT_MAX;
  for (int s = s0; s <= s1; ++s) {
    const VT v = cand(b[s], s, Pj);
    if (v < best) {
      best = v;
      arg = s;
    }
  }
  bv = best;
  bs = arg;
}

// The argmin table row of a layer is copied from shared memory by one TMA bulk store at the end
// of the layer (cp.async.bulk shared -> global), not by a scattered 2-byte store per row.
#ifndef SP_OPT_PER_ROW
constexpr bool kOptBulk = true;
#else
constexpr bool kOptBulk = false;
#endif
template <typename Ctx>
__device__ __forceinline__ void put_opt(const Ctx& c, int j, int v) {
  if constexpr (!kOptBulk) c.optout[j] = (uint16_t)v;
}

template <typename VT, typename Ctx>
__device__ __forceinline__ void row_write(const Ctx& c, int j, int lo, int hi, VT Pj, VT bv,
                                          int bs) {
  if (lo > hi || bs == INT_MAX) {   // empty bracket: never expected (reading R6 self-check)
    atomicExch(c.err, SP_ERR_INTERNAL);
    bs = max(1, min(lo, j));
    bv = 0;
  }
  c.sopt[j] = (uint16_t)bs;
  put_opt(c, j, bs);
  if (j < c.N) c.bnext[j + 1] = icpt(bv, j + 1, Pj);
  if (j == c.N) {
    const auto V = c.TN + bv;   // dp[m][N] = T_N + e_m(N)
    if (c.cbb_e) c.cbb_e[c.m] = V;
    if (c.last) *c.cost_e = V;
  }
}

// SP_DEBUG builds check every bracket before it is scanned (1 <= lo <= hi <= j < N, the bound
// rows already solved) and flag the entry (n_positions = -SP_ERR_INTERNAL) instead of reading
// out of range; compute-sanitizer is not available on this pool.
#ifdef SP_DEBUG
#define SP_CHECK_BRACKET(c, j, lo, hi)                                                  \
  do {                                                                                 \
    if (!((lo) >= 1 && (lo) <= (hi) && (hi) <= (j) && (j) <= (c).N)) {                 \
      atomicExch((c).err, SP_ERR_INTERNAL);                                            \
      (lo) = 1;                                                                        \
      (hi) = 0;                                                                        \
    }                                                                                  \
  } while (0)
#else
#define SP_CHECK_BRACKET(c, j, lo, hi) (void)0
#endif

// fp64: rounding can make neighbouring brackets cross by a hair; clamp instead of flagging
__device__ __forceinline__ void fix_bracket(double*, int& lo, int hi) {
  if (lo > hi) lo = hi;
}
template <typename VT>
__device__ __forceinline__ void fix_bracket(VT*, int&, int) {}

// One D&C level: every row j = h(2i+1) <= N, i < R.
//  phase 1  each thread takes rows i = tid + u NT, loads their brackets and P_j in batches of
//           RB (independent loads in flight), solves rows with <= T_INLINE candidates itself and
//           queues the longer ones, reserving ceil(len / PS) pieces with one 64-bit atomic
//           (queue index and piece base in one word, so queue order == piece order);
//  phase 2  threads take pieces p = tid + k NT; piece k of a row scans s = lo + k + i np
//           (interleaved so that neighbouring lanes read neighbouring words of b);
//  phase 3  one warp per queued row reduces its pieces (lexicographic (value, index) min) and
//           writes the row.
// Returns after its last barrier; the caller adds none.
template <typename VT, typename Ctx>
__device__ void run_level(const Ctx& c, Shared& sh, const Scratch<VT>& S, int h, int R,
                          int lvl, unsigned long long& nev) {
  unsigned long long* ctr = &sh.ctr[lvl % 3];
  if (threadIdx.x == 0) {   // last used two levels ago
    sh.ctr[(lvl + 1) % 3] = 0;
    sh.nmulti[(lvl + 1) % 3] = 0;
  }
  const int N = c.N;
  for (int i0 = threadIdx.x; i0 < R; i0 += DP_NT * RB) {
    int jj[RB], lo[RB], hi[RB];
    VT Pj[RB];
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int i = i0 + u * DP_NT;
      jj[u] = 0;
      lo[u] = 1;
      hi[u] = 0;
      Pj[u] = 0;
      if (i < R && h * (2 * i + 1) < N) {   // row N is solved first
        const int j = h * (2 * i + 1);
        const int l = max((int)c.sopt[j - h], (int)c.sopt[j]);   // opt_m(j-h), opt_{m-1}(j)
        const int r = min((int)c.sopt[min(j + h, N)], j);
        jj[u] = j;
        lo[u] = l;
        hi[u] = r;
        Pj[u] = (VT)c.P[j];
      }
    }
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      if (jj[u] == 0) continue;
      const int j = jj[u];
      int l = lo[u];
      const int r = hi[u];
      fix_bracket((VT*)nullptr, l, r);
      const int len = r - l + 1;
      if (len > 0) nev += (unsigned)len;
      if (len > T_INLINE) {
        const int np = (len + PS - 1) / PS;
        const unsigned long long old = atomicAdd(ctr, (1ull << 32) | (unsigned long long)np);
        const int q = (int)(old >> 32), pb = (int)(old & 0xffffffffu);
        if (q < QMAX) {
          const bool fits = pb + np <= PMAX;
          S.qj[q] = j;
          S.qlo[q] = l;
          S.qlen[q] = fits ? len : 0;   // a dead entry keeps the piece order intact
          S.qpb[q] = pb;
          S.qP[q] = Pj[u];
          if (fits) {
            if (np > 1) atomicAdd(&sh.nmulti[lvl % 3], 1);
            continue;
          }
        }
        // no room: solve it here (correct, just slower)
      }
      VT bv;
      int bs;
      if (len <= T_INLINE) eval_short(c.b, Pj[u], l, r, bv, bs);
      else eval_range(c.b, Pj[u], l, r, 1, bv, bs);
      row_write(c, j, l, r, Pj[u], bv, bs);
    }
  }
  __syncthreads();   // B1: inline rows written, queue complete
  const unsigned long long tot = *ctr;
  const int Q = min((int)(tot >> 32), QMAX);
  const int NP = min((int)(tot & 0xffffffffu), PMAX);
  if (Q == 0) return;
  const int nmulti = sh.nmulti[lvl % 3];
  // phase 2: thread t takes the contiguous pieces [t per, (t+1) per): one binary search, then walk
  {
    const int per = (NP + DP_NT - 1) / DP_NT;
    const int p0 = threadIdx.x * per, p1 = min(p0 + per, NP);
    if (p0 < p1) {
      int a = 0, z = Q - 1;   // last queue entry with qpb <= p0
      while (a < z) {
        const int mid = (a + z + 1) >> 1;
        if (S.qpb[mid] <= p0) a = mid; else z = mid - 1;
      }
      for (int p = p0; p < p1; ++p) {
        while (a + 1 < Q && S.qpb[a + 1] <= p) ++a;
        const int len = S.qlen[a];
        const int np = (len + PS - 1) / PS;
        const int k = p - S.qpb[a];
        if (k >= np) continue;
        VT bv;
        int bs;
        const int lo = S.qlo[a];
        eval_range(c.b, S.qP[a], lo + k, lo + len - 1, np, bv, bs);
        if (np == 1) {
          row_write(c, S.qj[a], lo, lo + len - 1, S.qP[a], bv, bs);
        } else {
          S.pv[p] = bv;
          S.ps[p] = bs;
        }
      }
    }
  }
  __syncthreads();   // B2: single-piece rows written, piece minima of the others stored
  if (nmulti == 0) return;
  // phase 3: rows with several pieces; one thread per row (<= 64 pieces) or one warp
  for (int q = threadIdx.x; q < Q; q += DP_NT) {
    const int len = S.qlen[q];
    const int np = (len + PS - 1) / PS;
    if (np < 2 || np > 64) continue;
    const int pb = S.qpb[q];
    VT bv = S.pv[pb];
    int bs = S.ps[pb];
    for (int k = 1; k < np; ++k) lex_min(bv, bs, S.pv[pb + k], S.ps[pb + k]);
    row_write(c, S.qj[q], S.qlo[q], S.qlo[q] + len - 1, S.qP[q], bv, bs);
  }
  const int lane = lane_id();
  for (int q = warp_id(); q < Q; q += DP_NW) {
    const int len = S.qlen[q];
    const int np = (len + PS - 1) / PS;
    if (np <= 64) continue;
    const int pb = S.qpb[q];
    VT bv = Lim<VT>::inf();
    int bs = INT_MAX;
    for (int k = lane; k < np; k += 32) lex_min(bv, bs, S.pv[pb + k], S.ps[pb + k]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const VT ov = __shfl_xor_sync(FULL, bv, o);
      const int os = __shfl_xor_sync(FULL, bs, o);
      lex_min(bv, bs, ov, os);
    }
    if (lane == 0) row_write(c, S.qj[q], S.qlo[q], S.qlo[q] + len - 1, S.qP[q], bv, bs);
  }
  __syncthreads();   // B3: queued rows written
}

// ---- warp-cooperative leftmost argmin of b_s - s P over s in [lo, hi] ------------------------
// Generic version: lanes stride the candidates, lexicographic (value, index) shuffle reduction.
template <typename VT>
__device__ __forceinline__ void warp_row_min(const VT* __restrict__ b, VT Pj, int lo, int hi,
                                             VT& bv, int& bs) {
  const int lane = lane_id();
  bv = Lim<VT>::inf();
  bs = INT_MAX;
  for (int s = lo + lane; s <= hi; s += 32) {
    const VT v = cand(b[s], s, Pj);
    if (v < bv) {
      bv = v;
      bs = s;
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const VT ov = __shfl_xor_sync(FULL, bv, o);
    const int os = __shfl_xor_sync(FULL, bs, o);
    lex_min(bv, bs, ov, os);
  }
}

// Exact-int32 version: each lane scans 16-byte aligned groups of four candidates (one LDS.128,
// a VIMNMX3-based min of four, index kept per group), the unaligned head/tail candidates go to
// lanes 0-2, and the warp reduction is two REDUX instructions (min value, then min index among
// the lanes holding it) -- the leftmost argmin, exactly.
template <>
__device__ __forceinline__ void warp_row_min<int32_t>(const int32_t* __restrict__ b, int32_t Pj,
                                                      int lo, int hi, int32_t& bv, int& bs) {
#ifdef SP_WRM_STRIDED
  {   // lanes stride the candidates with a strict '<' (leftmost per lane), two REDUX
    const int lane = lane_id();
    int best = INT_MAX, arg = INT_MAX;
#pragma unroll 2
    for (int s = lo + lane; s <= hi; s += 32) {
      const int v = b[s] - s * Pj;
      if (v < best) {
        best = v;
        arg = s;
      }
    }
    const int vmin = __reduce_min_sync(FULL, best);
    bs = __reduce_min_sync(FULL, best == vmin ? arg : INT_MAX);
    bv = vmin;
    return;
  }
#endif
  const int lane = lane_id();
  int best = INT_MAX, arg = INT_MAX;
  const int a = min(hi + 1, (lo + 3) & ~3);        // first aligned candidate
  const int nfull = (hi + 1 - a) >> 2;              // aligned groups of 4
  const int t0 = a + 4 * nfull;                     // first tail candidate
  if (lane < a - lo) {                              // head: at most 3 candidates
    const int s = lo + lane;
    best = b[s] - s * Pj;
    arg = s;
  }
  int gb = INT_MAX, gi = -1;
  for (int g = lane; g < nfull; g += 32) {
    const int s = a + 4 * g;
    const int4 q = *reinterpret_cast<const int4*>(b + s);
    const int v0 = q.x - s * Pj, v1 = q.y - (s + 1) * Pj;
    const int v2 = q.z - (s + 2) * Pj, v3 = q.w - (s + 3) * Pj;
    const int m = min(min(v0, v1), min(v2, v3));
    if (m < gb) {
      gb = m;
      gi = s;
    }
  }
  if (gi >= 0 && gb < best) {   // head candidates (if any) have smaller indices: strict '<'
    int k = gi + 3;
#pragma unroll
    for (int d = 2; d >= 0; --d)
      if (b[gi + d] - (gi + d) * Pj == gb) k = gi + d;
    best = gb;
    arg = k;
  }
  if (lane < hi + 1 - t0) {                         // tail: at most 3 candidates
    const int s = t0 + lane;
    const int v = b[s] - s * Pj;
    if (v < best) {
      best = v;
      arg = s;
    }
  }
  const int vmin = __reduce_min_sync(FULL, best);
  bs = __reduce_min_sync(FULL, best == vmin ? arg : INT_MAX);
  bv = vmin;
}

// ---- warp-level argmin reduction of per-lane (value, index) pairs -----------------------------
template <typename VT>
__device__ __forceinline__ void warp_lexmin(VT& bv, int& bs) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const VT ov = __shfl_xor_sync(FULL, bv, o);
    const int os = __shfl_xor_sync(FULL, bs, o);
    lex_min(bv, bs, ov, os);
  }
}
template <>
__device__ __forceinline__ void warp_lexmin<int32_t>(int32_t& bv, int& bs) {
  const int vmin = __reduce_min_sync(FULL, bv);
  bs = __reduce_min_sync(FULL, bv == vmin ? bs : INT_MAX);
  bv = vmin;
}

// Lean top level (R <= TOPR rows, all long): every warp computes the R brackets itself (two rows
// per lane, shuffle scan of the lengths), the level's candidates are flattened over all threads
// (warp w owns [w*32C, (w+1)*32C), lane l takes every 32nd candidate so b reads are
// conflict-free), each warp reduces per row with warp_lexmin and stores a partial, and one
// thread per row finalises.  Two barriers, no global loads (P of top rows cached in smem).
template <typename VT, typename Ctx>
__device__ void top_level(const Ctx& c, Shared& sh, uint8_t* scratch, const VT* topP, int h0,
                          int h, int R, int lvl, unsigned long long& nev) {
  const int N = c.N, lane = lane_id(), w = warp_id();
  if (threadIdx.x == 0) {   // keep run_level's counter rotation valid
    sh.ctr[(lvl + 1) % 3] = 0;
    sh.nmulti[(lvl + 1) % 3] = 0;
  }
  VT* pv = reinterpret_cast<VT*>(scratch);                       // [TOPR][DP_NW]
  int* ps = reinterpret_cast<int*>(pv + TOPR * DP_NW);           // [TOPR][DP_NW]
  int* rlo = ps + TOPR * DP_NW;                                  // [TOPR]
  int* rlen = rlo + TOPR;                                        // [TOPR]
  int* rst = rlen + TOPR;                                        // [TOPR]
  int lo[2], len[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = lane + 32 * u;
    const int j = h * (2 * i + 1);
    lo[u] = 1;
    len[u] = 0;
    if (i < R && j < N) {
      const int l = max((int)c.sopt[j - h], (int)c.sopt[j]);   // opt_m(j-h), opt_{m-1}(j)
      const int r = min((int)c.sopt[min(j + h, N)], j);
      lo[u] = l;
      len[u] = max(r - l + 1, 0);
    }
  }
  int inc0 = len[0], inc1 = len[1];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y0 = __shfl_up_sync(FULL, inc0, o), y1 = __shfl_up_sync(FULL, inc1, o);
    if (lane >= o) {
      inc0 += y0;
      inc1 += y1;
    }
  }
  const int tot0 = __shfl_sync(FULL, inc0, 31);
  const int W = tot0 + __shfl_sync(FULL, inc1, 31);
  const int st0 = inc0 - len[0], st1 = tot0 + inc1 - len[1];
  if (w == 0) {   // every warp computed the same; warp 0 records it for the finalisers
    rlo[lane] = lo[0];
    rlen[lane] = len[0];
    rst[lane] = st0;
    rlo[lane + 32] = lo[1];
    rlen[lane + 32] = len[1];
    rst[lane + 32] = st1;
  }
  if (threadIdx.x == 0) nev += (unsigned)W;
  const int C = (W + DP_NT - 1) / DP_NT;   // candidates per thread
  const int wb = w * 32 * C, we = min(wb + 32 * C, W);
  if (wb < we) {
    // rows are contiguous in the flattened order: the first row of this warp is the number of
    // rows that end at or before wb
    const int rfirst = __popc(__ballot_sync(FULL, st0 + len[0] <= wb)) +
                       __popc(__ballot_sync(FULL, st1 + len[1] <= wb));
    for (int r = rfirst; r < 64; ++r) {
      const int sr = r < 32 ? __shfl_sync(FULL, st0, r & 31) : __shfl_sync(FULL, st1, r & 31);
      if (sr >= we) break;
      const int lr = r < 32 ? __shfl_sync(FULL, len[0], r & 31) : __shfl_sync(FULL, len[1], r & 31);
      const int lor = r < 32 ? __shfl_sync(FULL, lo[0], r & 31) : __shfl_sync(FULL, lo[1], r & 31);
      if (lr == 0) continue;
      const int j = h * (2 * r + 1);
      const VT Pj = topP[j / h0];
      const int fa = max(sr, wb), fz = min(sr + lr, we);
      int f = wb + lane;
      if (f < fa) f += ((fa - f + 31) >> 5) << 5;
      VT bv = Lim<VT>::inf();
      int bs = INT_MAX;
      for (; f < fz; f += 32) {
        const int s = lor + (f - sr);
        const VT v = cand(c.b[s], s, Pj);
        if (v < bv) {
          bv = v;
          bs = s;
        }
      }
      warp_lexmin(bv, bs);
      if (lane == 0) {
        pv[r * DP_NW + w] = bv;
        ps[r * DP_NW + w] = bs;
      }
    }
  }
  __syncthreads();   // partials of every (row, warp) stored, row info recorded
  // finalise: warp r reduces row r's partials (lane q holds warp q's, if warp q touched it)
  for (int r = w; r < R; r += DP_NW) {
    const int j = h * (2 * r + 1);
    if (j >= N) continue;
    const int lr = rlen[r];
    VT bv = Lim<VT>::inf();
    int bs = INT_MAX;
    if (lr > 0) {
      const int sr = rst[r];
      const int w0 = sr / (32 * C), w1 = (sr + lr - 1) / (32 * C);
      for (int q = w0 + lane; q <= w1; q += 32) lex_min(bv, bs, pv[r * DP_NW + q], ps[r * DP_NW + q]);
    }
    warp_lexmin(bv, bs);
    if (lane == 0) {
      if (bs == INT_MAX) {   // empty bracket: never expected (reading R6 self-check)
        atomicExch(c.err, SP_ERR_INTERNAL);
        bs = max(1, min(rlo[r], j));
        bv = 0;
      }
      c.sopt[j] = (uint16_t)bs;
      put_opt(c, j, bs);
      c.bnext[j + 1] = icpt(bv, j + 1, topP[j / h0]);
    }
  }
  __syncthreads();   // row results visible to the next level
}

// Row N first (every layer): the whole CTA splits [max(1, opt_{m-1}(N)), N] and reduces.  With
// opt_m(N) known, every other row j has the right bound sopt[min(j + h, N)] (monotonicity), so
// the per-row code below needs no boundary branches.
template <typename VT, typename Ctx>
__device__ void solve_row_N(const Ctx& c, Shared& sh, unsigned long long& nev) {
  const int N = c.N;
  const int lo = c.sopt[N], hi = N;   // sopt[N] = opt_{m-1}(N), or 1 before layer 1
  const VT Pj = (VT)c.P[N];
  VT bv = Lim<VT>::inf();
  int bs = INT_MAX;
  for (int s = lo + (int)threadIdx.x; s <= hi; s += DP_NT) {
    const VT v = cand(c.b[s], s, Pj);
    if (v < bv) {
      bv = v;
      bs = s;
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const VT ov = __shfl_xor_sync(FULL, bv, o);
    const int os = __shfl_xor_sync(FULL, bs, o);
    lex_min(bv, bs, ov, os);
  }
  __syncthreads();   // sopt[N] read by everyone before it is rewritten
  VT* red = reinterpret_cast<VT*>(sh.wbuf);   // DP_NW values of VT fit in wbuf
  if (lane_id() == 0) {
    red[warp_id()] = bv;
    sh.red_s[warp_id()] = bs;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < DP_NW; ++w) lex_min(bv, bs, red[w], sh.red_s[w]);
    nev += (unsigned)(hi - lo + 1);
    row_write(c, N, lo, hi, Pj, bv, bs);
  }
  __syncthreads();
}

// Levels below the top ones: the rows split into segments (s h0, (s+1) h0) whose subtrees are
// independent once the top levels are solved.  Each warp grabs whole segments (dynamic, one smem
// counter) and solves their levels with __syncwarp only: lanes take rows; rows longer than TW are
// deferred to a warp list and solved cooperatively (lanes stride the candidates, coalesced in b,
// then a lexicographic shuffle min).  Warps overlap each other's L2 latencies.
// Levels below the top ones: the rows split into segments (s h0, (s+1) h0) whose subtrees are
// independent once the top levels are solved.  Each warp grabs whole segments (dynamic, one smem
// counter) and solves their levels with __syncwarp only: lanes take rows; rows longer than TW are
// deferred to a warp list and solved cooperatively (warp_row_min).  Warps overlap each other's
// latencies.
// Solve the subtree of one warp-owned segment (base, base + h0): levels K0..L-1 with
// __syncwarp only (lanes take rows; rows longer than TW deferred to a warp list and solved
// cooperatively with warp_row_min).
template <typename VT, typename Ctx>
__device__ void segment_body(const Ctx& c, uint8_t* scratch, int L, int K0, int seg,
                             unsigned& nv
#ifdef SP_TIMING
                             , long long& t_pass, long long& t_long
#endif
                             ) {
  const int N = c.N;
  const int h0 = 1 << (L - K0);
  const int lane = lane_id(), w = warp_id();
  int* lj = reinterpret_cast<int*>(scratch) + w * 3 * WCAP;
  int* llo = lj + WCAP;
  int* llen = llo + WCAP;
  VT* lP = reinterpret_cast<VT*>(reinterpret_cast<int*>(scratch) + DP_NW * 3 * WCAP) + w * WCAP;
  const VT* __restrict__ b = c.b;
  const uint16_t* sopt = c.sopt;
    const int base = seg * h0;
  for (int k = K0; k < L; ++k) {
    const int h = 1 << (L - 1 - k);
    const int nr = 1 << (k - K0);
    int cnt = 0;
#ifdef SP_TIMING
    long long t1 = clock64();
#endif
    for (int i0 = 0; i0 < nr; i0 += 32) {
      const int i = i0 + lane;
      const int j = base + h * (2 * i + 1);
      const bool valid = i < nr && j < N;   // row N is solved first
      int lo = 1, hi = 0;
      VT Pj = 0;
      if (valid) {
        lo = max((int)sopt[j - h], (int)sopt[j]);   // opt_m(j-h), opt_{m-1}(j)
        hi = min((int)sopt[min(j + h, N)], j);
        Pj = (VT)c.P[j];
      }
      fix_bracket((VT*)nullptr, lo, hi);
      if (valid) SP_CHECK_BRACKET(c, j, lo, hi);
      const int len = hi - lo + 1;
      nv += valid ? (unsigned)len : 0u;
      const bool lng = valid && len > TW;
      const unsigned bal = __ballot_sync(FULL, lng);
      const int pos = cnt + __popc(bal & ((1u << lane) - 1));
      cnt += __popc(bal);
      if (lng && pos < WCAP) {
        lj[pos] = j;
        llo[pos] = lo;
        llen[pos] = len;
        lP[pos] = Pj;
      }
      if (valid && (!lng || pos >= WCAP)) {   // short row, or the list is full
        VT best = Lim<VT>::inf();
        int arg = INT_MAX;
#pragma unroll 1
        for (int s = lo; s <= hi; ++s) {
          const VT v = cand(b[s], s, Pj);
          if (v < best) {
            best = v;
            arg = s;
          }
        }
        if (arg == INT_MAX) {   // empty bracket: never expected (reading R6 self-check)
          atomicExch(c.err, SP_ERR_INTERNAL);
          arg = max(1, min(lo, j));
          best = 0;
        }
        c.sopt[j] = (uint16_t)arg;
        put_opt(c, j, arg);
        c.bnext[j + 1] = icpt(best, j + 1, Pj);
      }
    }
    cnt = min(cnt, WCAP);
    __syncwarp();
#ifdef SP_TIMING
    long long t2 = clock64();
    t_pass += t2 - t1;
#endif
    for (int q = 0; q < cnt; ++q) {
      const int j = lj[q], lo = llo[q], len = llen[q];
      const VT Pj = lP[q];
      VT bv;
      int bs;
      warp_row_min(b, Pj, lo, lo + len - 1, bv, bs);
      if (lane == 0) {
        c.sopt[j] = (uint16_t)bs;
        put_opt(c, j, bs);
        c.bnext[j + 1] = icpt(bv, j + 1, Pj);
      }
    }
    __syncwarp();
#ifdef SP_TIMING
    t_long += clock64() - t2;
#endif
  }
  }

template <typename VT, typename Ctx>
__device__ void run_segments(const Ctx& c, Shared& sh, uint8_t* scratch, int L, int K0,
                             unsigned long long& nev) {
  const int N = c.N;
  const int h0 = 1 << (L - K0);
  const int NS = N / h0 + 1;
  const int lane = lane_id(), w = warp_id();
  int* lj = reinterpret_cast<int*>(scratch) + w * 3 * WCAP;
  int* llo = lj + WCAP;
  int* llen = llo + WCAP;
  VT* lP = reinterpret_cast<VT*>(reinterpret_cast<int*>(scratch) + DP_NW * 3 * WCAP) + w * WCAP;
  const VT* __restrict__ b = c.b;
  const uint16_t* sopt = c.sopt;
  unsigned nv = 0;
#ifdef SP_TIMING
  long long t_long = 0, t_pass = 0;
#endif
  for (;;) {
    int seg = 0;
    if (lane == 0) seg = atomicAdd(&sh.segctr, 1);
    seg = __shfl_sync(FULL, seg, 0);
    if (seg >= NS) break;
    const int base = seg * h0;
    for (int k = K0; k < L; ++k) {
      const int h = 1 << (L - 1 - k);
      const int nr = 1 << (k - K0);
      int cnt = 0;
#ifdef SP_TIMING
      long long t1 = clock64();
#endif
      for (int i0 = 0; i0 < nr; i0 += 32) {
        const int i = i0 + lane;
        const int j = base + h * (2 * i + 1);
        const bool valid = i < nr && j < N;   // row N is solved first
        int lo = 1, hi = 0;
        VT Pj = 0;
        if (valid) {
          lo = max((int)sopt[j - h], (int)sopt[j]);   // opt_m(j-h), opt_{m-1}(j)
          hi = min((int)sopt[min(j + h, N)], j);
          Pj = (VT)c.P[j];
        }
        fix_bracket((VT*)nullptr, lo, hi);
        if (valid) SP_CHECK_BRACKET(c, j, lo, hi);
        const int len = hi - lo + 1;
        nv += valid ? (unsigned)len : 0u;
        const bool lng = valid && len > TW;
        const unsigned bal = __ballot_sync(FULL, lng);
        const int pos = cnt + __popc(bal & ((1u << lane) - 1));
        cnt += __popc(bal);
        if (lng && pos < WCAP) {
          lj[pos] = j;
          llo[pos] = lo;
          llen[pos] = len;
          lP[pos] = Pj;
        }
        if (valid && (!lng || pos >= WCAP)) {   // short row, or the list is full
          VT best = Lim<VT>::inf();
          int arg = INT_MAX;
#pragma unroll 1
          for (int s = lo; s <= hi; ++s) {
            const VT v = cand(b[s], s, Pj);
            if (v < best) {
              best = v;
              arg = s;
            }
          }
          if (arg == INT_MAX) {   // empty bracket: never expected (reading R6 self-check)
            atomicExch(c.err, SP_ERR_INTERNAL);
            arg = max(1, min(lo, j));
            best = 0;
          }
          c.sopt[j] = (uint16_t)arg;
          put_opt(c, j, arg);
          c.bnext[j + 1] = icpt(best, j + 1, Pj);
        }
      }
      cnt = min(cnt, WCAP);
      __syncwarp();
#ifdef SP_TIMING
      long long t2 = clock64();
      t_pass += t2 - t1;
#endif
      for (int q = 0; q < cnt; ++q) {
        const int j = lj[q], lo = llo[q], len = llen[q];
        const VT Pj = lP[q];
        VT bv;
        int bs;
        warp_row_min(b, Pj, lo, lo + len - 1, bv, bs);
        if (lane == 0) {
          c.sopt[j] = (uint16_t)bs;
          put_opt(c, j, bs);
          c.bnext[j + 1] = icpt(bv, j + 1, Pj);
        }
      }
      __syncwarp();
#ifdef SP_TIMING
      t_long += clock64() - t2;
#endif
    }
  }
  nev += nv;
#ifdef SP_TIMING
  if (lane == 0) {
    atomicAdd(&sh.tclk[7], (unsigned long long)t_long);
    atomicAdd(&sh.tclk[6], (unsigned long long)t_pass);   // tclk[6] is reused below as max
  }
#endif
}

// ---- the dynamic task pool (replaces barrier-synchronous top levels) -------------------------
// A task is an interval (a, a + 2^lg) whose endpoints a and a + 2^lg (or N) are solved.  Internal
// tasks (2^lg > h0) solve their mid row a + 2^(lg-1) with one warp (warp_row_min: REDUX argmin)
// and push both halves; segment tasks (2^lg == h0) solve their whole subtree (segment_body).
// Node (a, 2^lg) exists iff a + 1 < N, so the number of tasks per layer is known up front and a
// warp pops indices until they run out, spinning (nanosleep) on slots whose parent has not
// finished yet.  A popped task's parent is always being processed by a non-spinning warp, so the
// pool cannot deadlock.  Release/acquire through __threadfence_block + volatile slots.
__device__ __forceinline__ int task_count(int N, int L, int lg0) {
  int T = 0;
  for (int lg = lg0; lg <= L; ++lg) T += ((N - 2) >> lg) + 1;
  return T;
}

template <typename VT, typename Ctx>
__device__ void run_tasks(const Ctx& c, Shared& sh, uint8_t* scratch, int L, int K0,
                          unsigned long long& nev) {
  const int N = c.N, lane = lane_id();
  const int lg0 = L - K0;   // segment length h0 = 2^lg0
  volatile int* tq = sh.tq;
  const int total = sh.tq_total;
  unsigned nv = 0;
#ifdef SP_TIMING
  long long t_pass = 0, t_long = 0;
#endif
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(&sh.tq_head, 1);
    idx = __shfl_sync(FULL, idx, 0);
    if (idx >= total) break;
    int code = 0;
    if (lane == 0) {
      while ((code = tq[idx]) < 0) __nanosleep(20);
    }
    code = __shfl_sync(FULL, code, 0);
    __threadfence_block();   // acquire: the parent's rows are visible
    const int a = code >> 5, lg = code & 31;
    if (lg == lg0) {
      segment_body<VT>(c, scratch, L, K0, a >> lg0, nv
#ifdef SP_TIMING
                       , t_pass, t_long
#endif
      );
      continue;
    }
    const int h = 1 << (lg - 1);
    const int mid = a + h;
    if (mid < N) {   // (mid == N is solved first; mid > N does not exist)
      int lo = max((int)c.sopt[a], (int)c.sopt[mid]);   // opt_m(a), opt_{m-1}(mid)
      int hi = min((int)c.sopt[min(a + 2 * h, N)], mid);
      SP_CHECK_BRACKET(c, mid, lo, hi);
      const VT Pj = (VT)c.P[mid];
      VT bv;
      int bs;
      warp_row_min(c.b, Pj, lo, hi, bv, bs);
      if (lane == 0) {
        nv += (unsigned)max(hi - lo + 1, 0);
        if (bs == INT_MAX) {   // empty bracket: never expected (reading R6 self-check)
          atomicExch(c.err, SP_ERR_INTERNAL);
          bs = max(1, min(lo, mid));
          bv = 0;
        }
        c.sopt[mid] = (uint16_t)bs;
        put_opt(c, mid, bs);
        c.bnext[mid + 1] = icpt(bv, mid + 1, Pj);
      }
    }
    if (lane == 0) {
      __threadfence_block();   // release: the mid row before the children become ready
      const bool left = a + 1 < N, right = mid + 1 < N;
      int t = atomicAdd(&sh.tq_tail, (int)left + (int)right);
      if (left) tq[t++] = (a << 5) | (lg - 1);
      if (right) tq[t] = (mid << 5) | (lg - 1);
    }
    __syncwarp();
  }
  nev += nv;
#ifdef SP_TIMING
  if (lane == 0) {
    atomicAdd(&sh.tclk[7], (unsigned long long)t_long);
    atomicAdd(&sh.tclk[6], (unsigned long long)t_pass);
  }
#endif
}

// ---- TMA bulk copy global -> shared (cp.async.bulk, completion on an mbarrier) ---------------
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, unsigned bytes,
                                         uint64_t* mbar, unsigned& phase) {
  const unsigned mb = (unsigned)__cvta_generic_to_shared(mbar);
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
                 : "memory");
    const unsigned sd = (unsigned)__cvta_generic_to_shared(smem_dst);
    for (unsigned off = 0; off < bytes; off += 32768u) {
      const unsigned n = min(32768u, bytes - off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(sd + off),
          "l"((const char*)gmem_src + off), "r"(n), "r"(mb)
          : "memory");
    }
  }
  asm volatile(
      "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; "
      "@!p bra WAIT_%=; }" ::"r"(mb),
      "r"(phase)
      : "memory");
  phase ^= 1u;
}

// Solve one entry with value type VT; b in shared memory (BS) or in the slot's global arrays.
template <typename VT, bool BS, typename PT, typename CT>
__device__ void solve_entry(const DpParams& p, Shared& sh, VT* smem_b, uint16_t* sopt,
                            uint8_t* scratch, int e, CT TN, const PT* P, unsigned& phase) {
  const int N = p.N, M = p.M;
  uint8_t* slot = p.slots + (size_t)blockIdx.x * p.slot;
  VT* bA = reinterpret_cast<VT*>(slot + align256(8 * (size_t)(N + 1)));
  VT* bB = reinterpret_cast<VT*>(slot + 2 * align256(8 * (size_t)(N + 1)));
  uint16_t* opt = reinterpret_cast<uint16_t*>(slot + slot_opt_off(N));
  const Scratch<VT> S = carve<VT>(scratch);

  VT* b = BS ? smem_b : bA;
  VT* bnext = bB;
  // layer 1: e_0 == 0 => b_s = s P_{s-1}
  for (int s = threadIdx.x + 1; s <= N; s += DP_NT) b[s] = icpt((VT)0, s, (VT)P[s - 1]);
  if (threadIdx.x < 3) {
    sh.ctr[threadIdx.x] = 0;
    sh.nmulti[threadIdx.x] = 0;
  }
  // sopt[0] = 1 is the virtual row 0 (lower bound 1); sopt[j] = 1 makes the layer bound
  // max(., opt_{m-1}(j)) a no-op in layer 1
  for (int j = threadIdx.x; j <= N; j += DP_NT) sopt[j] = 1;
  __syncthreads();

  LayerCtx<VT, PT, CT> c;
  c.sopt = sopt;
  c.P = P;
  c.N = N;
  c.TN = TN;
  c.cbb_e = p.cbb ? reinterpret_cast<CT*>(p.cbb) + (int64_t)e * (M + 1) : nullptr;
  c.cost_e = reinterpret_cast<CT*>(p.cost) + e;
  c.err = &sh.err;
  unsigned long long nev = 0;
  int lvl = 0;
  // top levels: every level whose rows are multiples of h0 = SEG_ROWS (or all levels if N is small)
  int K0 = p.L;
  if (N >= 2 * SEG_ROWS) K0 = p.L - 31 + __clz(SEG_ROWS);   // 2^(L-K0) = SEG_ROWS
  const int h0 = 1 << (p.L - K0);
  VT* topP = reinterpret_cast<VT*>(sh.topP);
  const bool use_topP = K0 < p.L && N / h0 + 1 <= TOPP_CAP;
  const int tq_total = K0 < p.L ? task_count(N, p.L, p.L - K0) : 0;
#ifdef SP_NO_TASKS
  const bool use_tasks = false;
#else
  const bool use_tasks = tq_total <= TQCAP;
#endif
  if (use_topP)
    for (int k = threadIdx.x; k <= N / h0; k += DP_NT) topP[k] = (VT)P[k * h0];
  __syncthreads();
  for (int m = 1; m <= M; ++m) {
    c.b = b;
    c.bnext = bnext;
    c.m = m;
    c.last = (m == M);
    c.optout = opt + (size_t)(m - 1) * opt_ld(N);
    c.optprev = m >= 2 ? opt + (size_t)(m - 2) * opt_ld(N) : nullptr;
    SP_T0();
    solve_row_N<VT>(c, sh, nev);
    SP_TICK(sh, 0);
    if (K0 < p.L && use_tasks) {
      // dynamic task pool: top-level rows and warp-owned segments, no barriers in between
      for (int t = threadIdx.x; t < tq_total; t += DP_NT) sh.tq[t] = t == 0 ? (0 << 5) | p.L : -1;
      if (threadIdx.x == 0) {
        sh.tq_head = 0;
        sh.tq_tail = 1;
        sh.tq_total = tq_total;
      }
      __syncthreads();
#ifdef SP_TIMING
      const long long ts = clock64();
#endif
      run_tasks<VT>(c, sh, scratch, p.L, K0, nev);
#ifdef SP_TIMING
      if (lane_id() == 0) {
        const unsigned long long d = (unsigned long long)(clock64() - ts);
        atomicAdd(&sh.tclk[4], d);
        atomicMax(&sh.tclk[8], d);
      }
#endif
      __syncthreads();
#ifdef SP_TIMING
      if (threadIdx.x == 0) {
        sh.tclk[5] += sh.tclk[8];
        sh.tclk[8] = 0;
      }
#endif
      SP_TICK(sh, 2);
    } else {
    // top levels: CTA-cooperative (few rows, long brackets)
    for (int k = 0; k < K0; ++k, ++lvl) {
      const int h = 1 << (p.L - 1 - k);
      const int R = ((N / h) + 1) >> 1;
      if (R <= TOPR) {
        if (use_topP) top_level<VT>(c, sh, scratch, topP, h0, h, R, lvl, nev);
        else top_level<VT>(c, sh, scratch, P, 1, h, R, lvl, nev);   // P straight from L2
      } else {
        run_level<VT>(c, sh, S, h, R, lvl, nev);
      }
    }
    SP_TICK(sh, 1);
    // the rest: warp-owned segments
    if (K0 < p.L) {
      if (threadIdx.x == 0) sh.segctr = 0;
      __syncthreads();
#ifdef SP_TIMING
      const long long ts = clock64();
#endif
      run_segments<VT>(c, sh, scratch, p.L, K0, nev);
#ifdef SP_TIMING
      if (lane_id() == 0) {   // per-warp busy time in the segment phase (imbalance)
        const unsigned long long d = (unsigned long long)(clock64() - ts);
        atomicAdd(&sh.tclk[4], d);
        atomicMax(&sh.tclk[8], d);
      }
#endif
      __syncthreads();
#ifdef SP_TIMING
      if (threadIdx.x == 0) {
        sh.tclk[5] += sh.tclk[8];
        sh.tclk[8] = 0;
      }
#endif
    }
    SP_TICK(sh, 2);
    }
    if (kOptBulk && threadIdx.x == 0) {   // every row of the layer is in sopt (barrier above)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(c.optout),
                   "r"((unsigned)__cvta_generic_to_shared(sopt)), "r"((unsigned)(2 * opt_ld(N)))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (m == M) {   // the backtrack (thread 0) reads the table next
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
    }
    if (m < M) {
      if (threadIdx.x == 0) bnext[1] = 0;   // e_m(0) + 1 * P_0 = 0
      if constexpr (BS) {
        // all rows are written (last level ended on a barrier): reload b from b_next by TMA
        bulk_g2s(b, bnext, (unsigned)((4 * (N + 1) + 15) & ~15), &sh.mbar, phase);
      } else {
        VT* t = b;
        b = bnext;
        bnext = t;
      }
      // sopt is rewritten by the next layer only after the bulk store has read it
      if (kOptBulk && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncthreads();
    }
    SP_TICK(sh, 3);
  }
  atomicAdd(&sh.evals, nev);
}

// ---- a3 for counts: P_j (int64) and T_N, block-wide scan over bins 1..N --------------------
template <typename WT>
__device__ void prefix_counts(const WT* we, int N, int64_t* P, int32_t* P32, Shared& sh,
                              int64_t& TN, int64_t& n, int& neg) {
  int64_t carry = 0, tpart = 0;
  int bad = 0;
  for (int base = 0; base <= N; base += DP_NT) {
    const int t = base + threadIdx.x;
    int64_t cnt = 0;
    if (t >= 1 && t <= N) cnt = (int64_t)we[t];
    // 1: a negative count (BAD_ARGUMENT); 2: a count >= 2^47, which could wrap the int64 sums
    // (N <= 2^16 such counts stay below 2^63, so n and the 2 n N < 2^62 guard are then exact)
    bad |= (cnt < 0 ? 1 : 0) | (cnt >= (int64_t(1) << 47) ? 2 : 0);
    int64_t tot;
    const int64_t ex = block_exclusive_scan<DP_NT>(cnt, sh.wbuf, &tot);
    if (t <= N) {
      P[t] = carry + ex + cnt;
      P32[t] = (int32_t)(carry + ex + cnt);   // used only when the int32 path is exact
    }
    carry += tot;
    tpart += (int64_t)t * cnt;
  }
  TN = block_sum<DP_NT>(tpart, sh.wbuf);
  n = carry;
  neg = (__syncthreads_or(bad & 1) ? 1 : 0) | (__syncthreads_or(bad & 2) ? 2 : 0);
}

// ---- a3/a7 for fp64 weights: double-double block scan, P_j rounded once ---------------------
__device__ dd block_exclusive_scan_dd(dd x, Shared& sh, dd* total) {
  const int lane = lane_id(), w = warp_id();
  dd inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    dd y = dd_shfl_up(inc, o);
    if (lane >= o) inc = dd_add(inc, y);
  }
  __syncthreads();
  if (lane == 31) {
    sh.dbuf[2 * w] = inc.hi;
    sh.dbuf[2 * w + 1] = inc.lo;
  }
  __syncthreads();
  if (w == 0) {
    dd v = lane < DP_NW ? dd{sh.dbuf[2 * lane], sh.dbuf[2 * lane + 1]} : dd{0.0, 0.0};
    dd vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      dd y = dd_shfl_up(vi, o);
      if (lane >= o) vi = dd_add(vi, y);
    }
    dd ex = dd_add(vi, dd{-v.hi, -v.lo});
    __syncwarp();
    if (lane < DP_NW) {
      sh.dbuf[2 * lane] = ex.hi;
      sh.dbuf[2 * lane + 1] = ex.lo;
    }
    if (lane == DP_NW - 1) {
      sh.dbuf[2 * DP_NW] = vi.hi;
      sh.dbuf[2 * DP_NW + 1] = vi.lo;
    }
  }
  __syncthreads();
  dd r = dd_add(dd{sh.dbuf[2 * w], sh.dbuf[2 * w + 1]}, dd_add(inc, dd{-x.hi, -x.lo}));
  *total = dd{sh.dbuf[2 * DP_NW], sh.dbuf[2 * DP_NW + 1]};
  return r;
}

__device__ void prefix_f64(const double* we, int N, double* P, Shared& sh, double& TN,
                           double& n, int& neg) {
  dd carry{0.0, 0.0}, tpart{0.0, 0.0};
  int bad = 0;
  for (int base = 0; base <= N; base += DP_NT) {
    const int t = base + threadIdx.x;
    double x = 0.0;
    if (t >= 1 && t <= N) x = we[t];
    bad |= !(x >= 0.0) || isinf(x);
    dd tot;
    const dd ex = block_exclusive_scan_dd(dd{x, 0.0}, sh, &tot);
    if (t <= N) {
      const dd inc = dd_add(dd_add(carry, ex), dd{x, 0.0});
      P[t] = inc.hi + inc.lo;
    }
    carry = dd_add(carry, tot);
    tpart = dd_add(tpart, dd_from_prod((double)t, x));
  }
  // block sum of tpart
  dd tt;
  block_exclusive_scan_dd(tpart, sh, &tt);
  TN = tt.hi + tt.lo;
  n = carry.hi + carry.lo;
  neg = __syncthreads_or(bad);
}

// definitional cost sum_t w_t (t - l(t;C)) in double-double, block-parallel (fp64 variant)
__device__ double eval_cost_f64(const double* we, int N, const int32_t* pos, int k, Shared& sh) {
  dd acc{0.0, 0.0};
  for (int t = 1 + threadIdx.x; t <= N; t += DP_NT) {
    // l(t) = largest position <= t (binary search over the ascending positions)
    int a = 0, z = k;   // count of positions <= t
    while (a < z) {
      const int mid = (a + z) >> 1;
      if (pos[mid] <= t) a = mid + 1; else z = mid;
    }
    const int l = a > 0 ? pos[a - 1] : 0;
    acc = dd_add(acc, dd_from_prod(we[t], (double)(t - l)));
  }
  dd tot;
  block_exclusive_scan_dd(acc, sh, &tot);
  return tot.hi + tot.lo;
}

// dynamic shared memory: opt_m (uint16[N+1]) | int32 b (if it fits) + int32-path scratch,
// overlapped with the int64/fp64-path scratch (those paths keep b in global memory)
__host__ __device__ __forceinline__ size_t dyn_smem_bytes(int N, bool smem_b) {
  const size_t a = smem_b ? align256(4 * (size_t)(N + 1)) : 0;
  const size_t n32 = a + scratch_bytes<int32_t>();
  const size_t n64 = scratch_bytes<int64_t>();
  return align256(2 * (size_t)(N + 1)) + (n32 > n64 ? n32 : n64);
}

template <typename WT>
__global__ void __launch_bounds__(DP_NT, 1) dp_place_kernel(DpParams p) {
  using PT = typename WTraits<WT>::PT;
  using CT = typename WTraits<WT>::CT;
  constexpr bool F64 = sizeof(WT) == 8 && std::is_floating_point<WT>::value;
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ Shared sh;
  const int N = p.N, M = p.M;
  uint16_t* sopt = reinterpret_cast<uint16_t*>(dsm);
  uint8_t* after_sopt = dsm + align256(2 * (size_t)(N + 1));
  int32_t* smem_b32 = reinterpret_cast<int32_t*>(after_sopt);
  uint8_t* scratch32 = after_sopt + (p.smem_b ? align256(4 * (size_t)(N + 1)) : 0);
  uint8_t* scratch64 = after_sopt;
  const WT* w = reinterpret_cast<const WT*>(p.w);
  CT* cost = reinterpret_cast<CT*>(p.cost);
  CT* cbb = reinterpret_cast<CT*>(p.cbb);
  unsigned phase = 0;   // TMA mbarrier parity, identical in every thread
  if (threadIdx.x < 10) sh.tclk[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    const unsigned mb = (unsigned)__cvta_generic_to_shared(&sh.mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int n_items = p.list ? (int)*p.list_n : p.E;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int e = p.list ? p.list[it] : it;
    uint8_t* slot = p.slots + (size_t)blockIdx.x * p.slot;
    PT* P = reinterpret_cast<PT*>(slot);
    int32_t* P32 = reinterpret_cast<int32_t*>(slot + slot_p32_off(N, M));
    const WT* we = w + (int64_t)e * (N + 1);
    CT TN, n;
    int neg;
    if constexpr (F64) {
      prefix_f64(we, N, P, sh, TN, n, neg);
    } else {
      prefix_counts<WT>(we, N, P, P32, sh, TN, n, neg);
    }
    if (threadIdx.x == 0) {
      sh.err = 0;
      sh.evals = 0;
      if (cbb) cbb[(int64_t)e * (M + 1)] = TN;   // V_0 = T_N
      cost[e] = TN;
    }
    __syncthreads();

    // ---- a4: the DP ----------------------------------------------------------------------
    int status = 0, path = -1;
    if (neg & 1) {
      status = SP_ERR_BAD_ARGUMENT;
    } else if (neg & 2) {
      status = SP_ERR_OVERFLOW;
    } else if (M > 0) {
      if constexpr (F64) {
        solve_entry<double, false, PT, CT>(p, sh, nullptr, sopt, scratch64, e, TN, P, phase);
        path = 2;
      } else {
        // narrow (exact int32) when 2 n N < 2^31, else int64 (exact when 2 n N < 2^62)
        const bool narrow = n < (int64_t(1) << 30) / N;
        const bool wide_ok = n < (int64_t(1) << 61) / N;
        if (narrow) {
          if (p.smem_b)
            solve_entry<int32_t, true, int32_t, CT>(p, sh, smem_b32, sopt, scratch32, e, TN, P32,
                                                    phase);
          else
            solve_entry<int32_t, false, int32_t, CT>(p, sh, nullptr, sopt, scratch32, e, TN, P32,
                                                     phase);
          path = 0;
        } else if (wide_ok) {
          solve_entry<int64_t, false, PT, CT>(p, sh, nullptr, sopt, scratch64, e, TN, P, phase);
          path = 1;
        } else {
          status = SP_ERR_OVERFLOW;
        }
      }
    }
    __syncthreads();
    if (sh.err) status = sh.err;
    if (threadIdx.x == 0) {
      sp_dp_stats* st = reinterpret_cast<sp_dp_stats*>(p.ws);
      atomicAdd(&st->evaluations, sh.evals);
      if (path == 0) atomicAdd(&st->entries_i32, 1ull);
      if (path == 1) atomicAdd(&st->entries_i64, 1ull);
      if (path == 2) atomicAdd(&st->entries_f64, 1ull);
    }

    // ---- a5: rule-B backtrack (one thread; <= M dependent reads) ---------------------------
    int32_t* out = p.pos + (int64_t)e * M;
    if (threadIdx.x == 0) {
      int k = 0;
      if (status == 0 && M > 0) {
        const uint16_t* opt = reinterpret_cast<const uint16_t*>(slot + slot_opt_off(N));
        int j = N, m = M;
        while (m > 0 && P[j] > 0) {
          const int s = opt[(size_t)(m - 1) * opt_ld(N) + j];
          out[k++] = s;
          j = s - 1;
          --m;
        }
        for (int a = 0, z = k - 1; a < z; ++a, --z) {
          const int tmp = out[a];
          out[a] = out[z];
          out[z] = tmp;
        }
      }
      for (int q = k; q < M; ++q) out[q] = 0;
      p.npos[e] = status ? -status : k;
      sh.red_s[0] = status ? -1 : k;
    }
    if (p.fpos && M > 0) {
      // f3: the canonical placement of EVERY budget m <= M from the same argmin table (layers
      // 1..m of an M-layer run are exactly an m-layer run): thread m-1 backtracks budget m
      __syncthreads();
      const int st = sh.red_s[0];
      const uint16_t* opt = reinterpret_cast<const uint16_t*>(slot + slot_opt_off(N));
      for (int mb = threadIdx.x + 1; mb <= M; mb += DP_NT) {
        int32_t* fo = p.fpos + ((int64_t)e * M + (mb - 1)) * M;
        int k = 0;
        if (st >= 0) {
          int j = N, m = mb;
          while (m > 0 && P[j] > 0) {
            const int s = opt[(size_t)(m - 1) * opt_ld(N) + j];
            fo[k++] = s;
            j = s - 1;
            --m;
          }
          for (int a = 0, z = k - 1; a < z; ++a, --z) {
            const int tmp = fo[a];
            fo[a] = fo[z];
            fo[z] = tmp;
          }
        }
        for (int q = k; q < M; ++q) fo[q] = 0;
        p.fn[(int64_t)e * M + mb - 1] = st >= 0 ? k : st;
      }
    }
    if constexpr (F64) {
      // a7: report the definitional cost of the returned placement, compensated (the DP's own
      // V_M carries ~M N eps P_N absolute rounding)
      __syncthreads();
      const int k = sh.red_s[0];
      if (k >= 0 && M > 0 && cbb) {
        // V_1..V_M as the definitional costs of the canonical placement of every budget (the
        // same backtrack from the argmin table), so that cost_by_budget meets the 1e-12 bound
        // (SURVEY 8(c) a7); the loop ends with budget M, whose placement stays in `out`
        const uint16_t* opt = reinterpret_cast<const uint16_t*>(slot + slot_opt_off(N));
        for (int mb = 1; mb <= M; ++mb) {
          if (threadIdx.x == 0) {
            int kk = 0, j = N, m = mb;
            while (m > 0 && P[j] > 0) {
              const int s = opt[(size_t)(m - 1) * opt_ld(N) + j];
              out[kk++] = s;
              j = s - 1;
              --m;
            }
            for (int a = 0, z = kk - 1; a < z; ++a, --z) {
              const int tmp = out[a];
              out[a] = out[z];
              out[z] = tmp;
            }
            sh.red_s[1] = kk;
          }
          __syncthreads();
          const int kk = sh.red_s[1];
          const double v = eval_cost_f64(we, N, out, kk, sh);
          if (threadIdx.x == 0) cbb[(int64_t)e * (M + 1) + mb] = v;
          __syncthreads();
        }
        for (int q = k + threadIdx.x; q < M; q += DP_NT) out[q] = 0;
        if (threadIdx.x == 0) cost[e] = cbb[(int64_t)e * (M + 1) + M];
      } else if (k >= 0 && M > 0) {
        const double v = eval_cost_f64(we, N, out, k, sh);
        if (threadIdx.x == 0) cost[e] = v;
      }
    }
    __syncthreads();
  }
#ifdef SP_TIMING
  if (threadIdx.x < 8) atomicAdd(reinterpret_cast<unsigned long long*>(p.ws) + 8 + threadIdx.x, sh.tclk[threadIdx.x]);
#endif
}

}  // namespace sp

static bool dp_smem_b_fits(int N) {
  return sp::dyn_smem_bytes(N, true) + sizeof(sp::Shared) + 1024 <= 227 * 1024;
}

static size_t dp_dyn_smem(int N, bool smem_b) { return sp::dyn_smem_bytes(N, smem_b); }

// resident CTAs per SM of dp_place_kernel<WT> (cached per device and shared-memory size: no
// attribute or occupancy query on every call once warm)
template <typename WT>
static int dp_grid_t(int E, int N) {
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, std::pair<int, int>> cache;   // -> (sms, occ)
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t dyn = dp_dyn_smem(N, dp_smem_b_fits(N));
  int sms = 148, occ = 1;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, dyn});
    if (it != cache.end()) {
      sms = it->second.first;
      occ = it->second.second;
    } else {
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      // opt in to the most dynamic shared memory the kernel can have (static + dynamic <= the
      // per-block opt-in limit), once per device: every later size fits
      int optin = 227 * 1024;
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncAttributes fa;
      if (cudaFuncGetAttributes(&fa, sp::dp_place_kernel<WT>) == cudaSuccess)
        cudaFuncSetAttribute(sp::dp_place_kernel<WT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - (int)fa.sharedSizeBytes);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sp::dp_place_kernel<WT>, sp::DP_NT, dyn);
      if (occ < 1) occ = 1;
      cache[{dev, dyn}] = {sms, occ};
    }
  }
  long g = (long)sms * occ;
  if (g > E) g = E;
  return (int)(g < 1 ? 1 : g);
}

static int dp_grid(int E, int N) {
  // the workspace must fit whichever weight type is launched: take the largest grid
  int g = dp_grid_t<int32_t>(E, N);
  g = std::max(g, dp_grid_t<int64_t>(E, N));
  g = std::max(g, dp_grid_t<double>(E, N));
  return g;
}

extern "C" size_t sp_place_checkpoints_workspace_bytes(int32_t n_entries, int32_t N, int32_t M) {
  if (N < 1 || N > SP_MAX_N || n_entries < 0 || M < 0 || M > N) return 0;
  if (n_entries == 0) return 0;
  size_t hull = 0;
  if (M > 0) {
    const int gh = std::max(std::max(sp_hull_grid(n_entries, N, M, SP_W_COUNTS_I32),
                                     sp_hull_grid(n_entries, N, M, SP_W_COUNTS_I64)),
                            sp_hull_grid(n_entries, N, M, SP_W_PROB_F64));
    hull = 3 * sp::align256(4 * (size_t)n_entries) + sp::align256(sp_hull_wg_bytes(n_entries, N, M)) +
           sp::align256(sp_hull_order_bytes(n_entries)) + (size_t)gh * sp_hull_slot_bytes(N, M);
  }
  return SP_WS_STATS_BYTES + hull + (size_t)dp_grid(n_entries, N) * sp::slot_bytes(N, M);
}

static sp_status place_impl(const void* weights, sp_weight_type wtype, int32_t n_entries,
                            int32_t N, int32_t M, int32_t* positions, int32_t* n_positions,
                            void* cost, void* cost_by_budget, int32_t* fpos, int32_t* fn,
                            void* workspace, size_t workspace_bytes, sp_stream_t stream);

extern "C" sp_status sp_place_checkpoints(const void* weights, sp_weight_type wtype,
                                          int32_t n_entries, int32_t N, int32_t M,
                                          int32_t* positions, int32_t* n_positions, void* cost,
                                          void* cost_by_budget, void* workspace,
                                          size_t workspace_bytes, sp_stream_t stream) {
  return place_impl(weights, wtype, n_entries, N, M, positions, n_positions, cost,
                    cost_by_budget, nullptr, nullptr, workspace, workspace_bytes, stream);
}

extern "C" sp_status sp_place_checkpoints_frontier(const void* weights, sp_weight_type wtype,
                                                   int32_t n_entries, int32_t N, int32_t M,
                                                   int32_t* frontier_positions,
                                                   int32_t* frontier_n, void* cost_by_budget,
                                                   int32_t* positions, int32_t* n_positions,
                                                   void* cost, void* workspace,
                                                   size_t workspace_bytes, sp_stream_t stream) {
  if (M > 0 && (!frontier_positions || !frontier_n)) return SP_ERR_BAD_ARGUMENT;
  return place_impl(weights, wtype, n_entries, N, M, positions, n_positions, cost,
                    cost_by_budget, frontier_positions, frontier_n, workspace, workspace_bytes,
                    stream);
}

static sp_status place_impl(const void* weights, sp_weight_type wtype,
                            int32_t n_entries, int32_t N, int32_t M, int32_t* positions,
                            int32_t* n_positions, void* cost, void* cost_by_budget, int32_t* fpos,
                            int32_t* fn, void* workspace, size_t workspace_bytes,
                            sp_stream_t stream) {
  if (N < 1 || N > SP_MAX_N || n_entries < 0) return SP_ERR_BAD_LENGTH;
  if (M < 0 || M > N) return SP_ERR_BUDGET_TOO_LARGE;
  if (wtype != SP_W_COUNTS_I32 && wtype != SP_W_COUNTS_I64 && wtype != SP_W_PROB_F64)
    return SP_ERR_BAD_ARGUMENT;
  if (n_entries == 0) return SP_OK;
  if (!weights || !n_positions || !cost || (M > 0 && !positions)) return SP_ERR_BAD_ARGUMENT;
  int grid = 0;
  if (wtype == SP_W_COUNTS_I32) grid = dp_grid_t<int32_t>(n_entries, N);
  else if (wtype == SP_W_COUNTS_I64) grid = dp_grid_t<int64_t>(n_entries, N);
  else grid = dp_grid_t<double>(n_entries, N);
  // the hull kernels (dp_hull.cu: int32 / int64 for counts, double for fp64 weights) solve every
  // entry they can and list the rest (bad weights, nN >= 2^46, ring overflow) for the D&C kernel
  const bool use_hull = M > 0 && !sp_debug_get(SP_DBG_NO_HULL);
  const int hgrid = use_hull ? sp_hull_grid(n_entries, N, M, wtype) : 0;
  const size_t fb_off = SP_WS_STATS_BYTES;
  const size_t wide_off = fb_off + (use_hull ? sp::align256(4 * (size_t)n_entries) : 0);
  const size_t fwd_off = wide_off + (use_hull ? sp::align256(4 * (size_t)n_entries) : 0);
  const size_t pool_off = fwd_off + (use_hull ? sp::align256(4 * (size_t)n_entries) : 0);
  const size_t order_off = pool_off + (use_hull ? sp::align256(sp_hull_wg_bytes(n_entries, N, M)) : 0);
  const size_t hull_off = order_off + (use_hull ? sp::align256(sp_hull_order_bytes(n_entries)) : 0);
  const size_t dc_off = hull_off + (size_t)hgrid * (use_hull ? sp_hull_slot_bytes(N, M) : 0);
  const size_t need = dc_off + (size_t)grid * sp::slot_bytes(N, M);
  if (!workspace || workspace_bytes < need) return SP_ERR_WORKSPACE;
  sp::DpParams p;
  p.w = weights;
  p.E = n_entries;
  p.N = N;
  p.M = M;
  p.L = 32 - __builtin_clz((unsigned)N);   // 2^L > N >= 2^(L-1)
  p.pos = positions;
  p.npos = n_positions;
  p.cost = cost;
  p.cbb = cost_by_budget;
  p.ws = (uint8_t*)workspace;
  p.slot = sp::slot_bytes(N, M);
  p.smem_b = dp_smem_b_fits(N) ? 1 : 0;
  p.fpos = fpos;
  p.fn = fn;
  p.slots = (uint8_t*)workspace + dc_off;
  p.list = use_hull ? reinterpret_cast<const int32_t*>((uint8_t*)workspace + fb_off) : nullptr;
  p.list_n = reinterpret_cast<const unsigned*>((uint8_t*)workspace + SP_WS_FB_COUNT_OFF);
  const size_t dyn = dp_dyn_smem(N, p.smem_b);
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(workspace, 0, SP_WS_STATS_BYTES, st) != cudaSuccess) SP_CHECK_LAUNCH();
  if (use_hull) {
    const cudaError_t he = sp_hull_launch(
        weights, wtype, n_entries, N, M, positions, n_positions, cost, cost_by_budget, fpos, fn,
        (uint8_t*)workspace,
        reinterpret_cast<int32_t*>((uint8_t*)workspace + fb_off),
        reinterpret_cast<int32_t*>((uint8_t*)workspace + wide_off),
        reinterpret_cast<int32_t*>((uint8_t*)workspace + fwd_off), (uint8_t*)workspace + pool_off,
        (uint8_t*)workspace + order_off, (uint8_t*)workspace + hull_off, hgrid, st);
    if (he != cudaSuccess) {
      sp_set_cuda_error(he);
      return SP_ERR_CUDA;
    }
  }
  if (wtype == SP_W_COUNTS_I32) sp::dp_place_kernel<int32_t><<<grid, sp::DP_NT, dyn, st>>>(p);
  else if (wtype == SP_W_COUNTS_I64) sp::dp_place_kernel<int64_t><<<grid, sp::DP_NT, dyn, st>>>(p);
  else sp::dp_place_kernel<double><<<grid, sp::DP_NT, dyn, st>>>(p);
  SP_CHECK_LAUNCH();
  return SP_OK;
}
