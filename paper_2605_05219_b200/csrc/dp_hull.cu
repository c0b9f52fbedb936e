// dp_hull.cu -- a3 + a4 + a5 on the exact-int32 path: the paper's own O(NM) algorithm, the
// monotone convex-hull trick of P:764-773, made data-parallel ACROSS LAYERS.
// a3-a5.
//
// Per layer m the DP is e_m(j) = min_{1<=s<=j} b_s - s P_j with b_s = e_{m-1}(s-1) + s P_{s-1}
// (the rewrite of P:758-762, e_m(j) = dp[m][j] - T_j; T_j cancels out of every comparison).
// Line s (slope -s, intercept b_s) becomes available at row s, and the query points x = P_j
// are non-decreasing, so each layer is one sequential pass of the paper's monotone hull:
// push line j (pop the back while the last line is not strictly below the segment from the
// second-to-last line to the new one), then pop the front while the next line is STRICTLY
// better at P_j (ties keep the lower index: the leftmost argmin, reading R3).
//
// Lockstep layers.  The only dependency between layers is e_{m-1}(j-1) -> b_j of layer m, so
// every layer advances one row per step: lane l of the warp owns layers l+1 and l+33 (K = 2
// slots; K = 1 when M <= 32) and receives e_{m-1}(j-1) -- produced by the lane below at step
// j-1 -- with one shuffle.  One warp solves one entry; M > 64 runs in passes of 64 layers
// chained through a global e-row buffer.
//
// Zero-count rows are no-ops ("support rows").  If c_j = 0 then P_j = P_{j-1},
// so the new line's candidate at the query point is b_j - j P_j = e_{m-1}(j-1) >= e_m(j-1)
// (V is non-increasing in the budget at every row: "at most m", reading R1), hence
// e_m(j) = e_m(j-1) and opt_m(j) = opt_m(j-1) exactly; and line j is strictly worse than line
// j+1 at every later query x > P_j (their difference is e_{m-1}(j) - e_{m-1}(j-1) + P_j - x < 0),
// so it never needs to enter the hull.  The warp therefore steps only through the support rows
// (c_j > 0, found 32 at a time with a ballot), and every e_m / opt_m of a zero row is the value
// at the support row before it.  The row type is the same for all lanes (one entry per warp).
//
// Each layer's deque lives in shared memory as a ring (HC0 / HC1 lines for slot 0 / 1),
// interleaved across lanes ([slot][pos][lane]) so that every lane hits its own bank whatever its
// deque position; the back and front lines are in registers and the two lines next to each end
// are loaded at the top of every support row, so a row with at most two back pops and one front
// pop per layer issues no dependent shared load (more pops: a warp-uniform loop).
// Rings hold the live hull, which is small for histogram-shaped inputs (<= 51 lines on W5); an
// entry whose hull outgrows a ring is re-run on a global ring, and if that overflows too (e.g.
// the all-ones histogram: layer-1 hull ~N/2 lines) handed to the divide-and-conquer kernel
// (dp_place.cu), as are entries past the int64 guard.
//
// Argmin storage: opt_m(j) changes rarely along j, so each layer appends (j, opt_m(j)) to its
// own log only when it changes (uint32: j << 16 | opt); the backtrack finds the last entry with
// row <= j by a warp-cooperative 32-way search.  Outputs per entry: V_m = T_N + e_m(N) for every
// m (cost_by_budget), the rule-B backtrack (positions, count), the f3 frontier.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cub/device/device_radix_sort.cuh>
#include <type_traits>

#include "common.cuh"
#include "dp_internal.cuh"

namespace sp {

// Ring capacity per layer (power of two): layers 1-32 (slot 0) hold the longest hulls (W5: up to
// ~51 support lines), layers 33-64 (slot 1) at most ~32 (tools/hull_stats.c).
#ifndef SP_HULL_CAP0
#define SP_HULL_CAP0 64
#endif
#ifndef SP_HULL_CAP1
#define SP_HULL_CAP1 32
#endif
constexpr int HC0 = SP_HULL_CAP0, HC1 = SP_HULL_CAP1;
// The int64 and fp64 instantiations keep a WINDOW of WC lines per layer in shared memory and every
// older live line in a global array per layer (WRing below): they take the large hulls --
// accumulated rows (layer-1 hulls ~100 lines), near-uniform / all-ones rows (~N/(m+1) lines in
// layer m) and the int32 entries whose hull outgrew a shared ring.
#ifndef SP_HULL_WCAP
#define SP_HULL_WCAP 32
#endif
constexpr int WC = SP_HULL_WCAP;
static_assert((WC & (WC - 1)) == 0, "window capacity: a power of two");
// row prefetch depth of the hull kernels, in 32-row chunks
#ifndef SP_HULL_PF
#define SP_HULL_PF 8
#endif
constexpr int HULL_PF = SP_HULL_PF;
static_assert((HC0 & (HC0 - 1)) == 0 && (HC1 & (HC1 - 1)) == 0, "ring capacities: powers of two");

__host__ __device__ __forceinline__ size_t hull_align(size_t x) { return (x + 255) & ~(size_t)255; }
__host__ __device__ __forceinline__ int hull_K(int M) { return M > 32 ? 2 : 1; }
__host__ __device__ __forceinline__ int hull_passes(int M) {
  const int L = 32 * hull_K(M);
  return (M + L - 1) / L;
}
__host__ __device__ __forceinline__ int hull_layers_padded(int M) {
  return hull_passes(M) * 32 * hull_K(M);
}
// slot: argmin logs uint32 [layer][N+1] | log counts int32 [layer] | e-row buffers 2 x VT[N+1]
// argmin-log capacity per layer: opt changes at a fraction of the support rows (W5: ~500 of
// ~5170); an entry that fills a log goes to the D&C kernel (never on W5)
__host__ __device__ __forceinline__ int hull_log_cap(int N) {
#ifdef SP_HULL_BIGLOG
  return N + 1;
#endif
  const int c = (N + 1 + 7) / 8;
  return c < 1024 ? (N + 1 < 1024 ? N + 1 : 1024) : c;
}
__host__ __device__ __forceinline__ size_t hull_log_bytes(int N, int M) {
  return hull_align((size_t)hull_layers_padded(M) * hull_log_cap(N) * 4);
}
__host__ __device__ __forceinline__ size_t hull_cnt_bytes(int M) {
  return hull_align((size_t)hull_layers_padded(M) * 4);
}
__host__ __device__ __forceinline__ size_t hull_slot_bytes(int N, int M) {
  return hull_log_bytes(N, M) + hull_cnt_bytes(M) + 2 * hull_align(8 * (size_t)(N + 1));
}
__host__ __device__ __forceinline__ size_t hull_smem_bytes(int) { return 0; }   // static rings

// per-entry row statistics from row_stats_kernel (integer weights)
struct HullRowStat {
  long long n, tn;   // P_N and T_N (int64; valid when !bad)
  int tfirst;        // first non-zero bin (INT_MAX if none)
  int bad;           // a negative count or one >= 2^40
  int K;             // support rows (non-zero bins 1..N)
  int pad;
};
// Sparse rows (K <= HULL_KC support rows) are also compacted by the pre-pass into (j, c_j) pairs,
// int2 [E][HULL_KC]: the DP then walks its K support rows instead of scanning N bins.
#ifndef SP_HULL_KC
#define SP_HULL_KC 256
#endif
constexpr int HULL_KC = SP_HULL_KC;

struct HullParams {
  const void* w;
  int E, N, M;
  int32_t* pos;
  int32_t* npos;
  void* cost;       // int64 [E] (count weights) or double [E] (fp64 weights)
  void* cbb;        // same type, [E][M+1], or NULL
  int32_t* fpos;
  int32_t* fn;
  uint8_t* ws;      // workspace head (stats + counters)
  int32_t* fb;      // fallback entry list
  uint8_t* slots;   // per-warp slots
  size_t slot;
  uint8_t* wg;      // windowed rings' global arrays: one region of wgb bytes per CTA
  size_t wgb;       // wring_pass_bytes(N, M)
  int32_t* wide;    // entries for the int64 instantiation
  const int32_t* order;   // processing order of the entries (largest support first), or NULL
  int logcap;             // argmin-log entries usable per layer (hull_log_cap(N); tests lower it)
  const HullRowStat* rstat;   // n, T_N, first bin, guards per entry (integer weights), or NULL
  const int2* sparse;         // [E][HULL_KC] compacted support rows (valid when rstat[e].K <= HULL_KC)
  int fwd;                    // the large-hull mode ran: the int64 list is its forwarded list
  int32_t* fwd_list;          // int32 [E]: the large-hull mode's forwarded entries
};

// Global capacity (lines, a power of two) of layer m's windowed ring: ~1.125x the hull size of
// the uniform law in layer m, (N+1)/(m+1) (the deque spans opt_m(j) ~ j m/(m+1) to j), at least 256
// (accumulated W5 rows: <= ~100 lines); a hull that outgrows it goes to the D&C kernel.
__host__ __device__ __forceinline__ int wring_cap(int N, int m) {
  long c = (long)(N + 1) * 9 / (8 * (long)(m + 1)) + 64;
  if (c < 256) c = 256;
  int p = 256;
  while (p < c) p <<= 1;
  return p;
}
// log slot of layer m (1-based), lane-major within a pass: [pass][slot k][lane]
__device__ __forceinline__ int hull_layer_slot(int K, int m) {
  const int L = 32 * K;
  const int p = (m - 1) / L, q = (m - 1) % L;
  return p * L + (q >> 5) * 32 + (q & 31);
}

// opt_m(j) from layer m's change log: the last entry with row <= j (entry 0 has row 1 <= j).
// Warp-cooperative: each round the 32 lanes probe 32 evenly spaced entries.
__device__ __forceinline__ int log_lookup_warp(const uint32_t* lg, int cnt, int j) {
  const int lane = lane_id();
  int lo = 0, hi = cnt - 1;
  while (hi > lo) {
    const int span = hi - lo;
    const int pr = lo + (int)(((long long)span * (lane + 1) + 31) >> 5);
    const bool ok = (int)(__ldcg(lg + pr) >> 16) <= j;
    const unsigned bal = __ballot_sync(FULL, ok);
    if (bal == 0) {
      hi = __shfl_sync(FULL, pr, 0) - 1;
    } else {
      const int i = 31 - __clz(bal);
      const int plo = __shfl_sync(FULL, pr, i);
      const int pnx = __shfl_sync(FULL, pr, (i + 1) & 31);
      lo = plo;
      if (i < 31) hi = pnx - 1;
    }
  }
  return (int)(__ldcg(lg + lo) & 0xffffu);
}
// Small argmin logs (sparse rows: W2 / W3 hold ~20-50 entries per layer) are copied into the
// free ring memory after the DP, so the backtrack's M dependent lookups hit shared memory instead
// of L2.  Layout: offsets int32 [M+1] | entries uint32.  Returns false (nothing copied) when they
// do not fit `cap_words`.  Layer m's log is slot m - 1 (hull_layer_slot).
__device__ __forceinline__ bool logs_to_smem(const uint32_t* logs, const int32_t* logn, int M,
                                             int LCstride, uint32_t* sm, int cap_words) {
  const int lane = lane_id();
  int base = 0;
  bool fits = true;
  for (int m0 = 0; m0 < M && fits; m0 += 32) {   // exclusive offsets in layer order
    const int m = m0 + lane;
    const int c = m < M ? logn[m] : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    const int tot = __shfl_sync(FULL, inc, 31);
    fits = base + tot + M + 1 <= cap_words;
    if (fits && m < M) sm[m] = (uint32_t)(base + inc - c);
    base += tot;
  }
  if (!fits) return false;
  if (lane == 0) sm[M] = (uint32_t)base;
  __syncwarp();
  uint32_t* ent = sm + M + 1;
  for (int m = lane; m < M; m += 32) {   // one lane per layer: independent loads in flight
    const uint32_t* lg = logs + (size_t)m * LCstride;
    const int o = (int)sm[m], c = (int)sm[m + 1] - o;
    for (int q = 0; q < c; ++q) ent[o + q] = __ldcg(lg + q);
  }
  __syncwarp();
  return true;
}
// opt_m(j) from layer m's log in shared memory (copied by logs_to_smem): warp-cooperative
__device__ __forceinline__ int log_lookup_smem(const uint32_t* sm, int M, int m, int j) {
  const int lane = lane_id();
  const uint32_t* lg = sm + M + 1 + sm[m - 1];
  const int cnt = (int)(sm[m] - sm[m - 1]);
  int lo = 0, hi = cnt - 1;
  while (hi > lo) {
    const int span = hi - lo;
    const int pr = lo + (int)(((long long)span * (lane + 1) + 31) >> 5);
    const bool ok = (int)(lg[pr] >> 16) <= j;
    const unsigned bal = __ballot_sync(FULL, ok);
    if (bal == 0) {
      hi = __shfl_sync(FULL, pr, 0) - 1;
    } else {
      const int i = 31 - __clz(bal);
      const int plo = __shfl_sync(FULL, pr, i);
      const int pnx = __shfl_sync(FULL, pr, (i + 1) & 31);
      lo = plo;
      if (i < 31) hi = pnx - 1;
    }
  }
  return (int)(lg[lo] & 0xffffu);
}
// single-thread version (one lane per budget in the frontier backtrack)
__device__ __forceinline__ int log_lookup_lane(const uint32_t* lg, int cnt, int j) {
  int lo = 0, hi = cnt - 1;   // last index with row <= j
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((int)(__ldcg(lg + mid) >> 16) <= j) lo = mid; else hi = mid - 1;
  }
  return (int)(__ldcg(lg + lo) & 0xffffu);
}

// The large-hull mode's unary argmin logs (hull_dp<.., BIG>): layer m's stream holds, per stepped
// (support) row in order, opt_m(j) - opt_m(j_prev) zeros then a one (opt = 0 before the first row),
// so opt_m at the r-th support row = the zeros before the r-th one.  Warp-cooperative, scanning
// from the end (the backtrack's ranks are large for the high layers it starts with).
__device__ __forceinline__ int unary_lookup_warp(const uint32_t* lg, int nw, int r) {
  const int lane = lane_id();
  int total = 0;   // ones in the stream (= stepped rows)
  for (int w = lane; w < nw; w += 32) total += __popc(__ldcg(lg + w));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(FULL, total, o);
  int need = total - r + 1;   // the need-th one counted from the end
  for (int w1 = nw; w1 > 0; w1 -= 32) {
    const int w = w1 - 1 - lane;   // lane 0 takes the highest word
    const uint32_t v = w >= 0 ? __ldcg(lg + w) : 0u;
    const int c = __popc(v);
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    const int tot = __shfl_sync(FULL, inc, 31);
    if (tot >= need) {
      const int L = __ffs(__ballot_sync(FULL, inc >= need)) - 1;
      const int q = need - __shfl_sync(FULL, inc - c, L);   // the q-th one from the top of word L
      uint32_t vw = __shfl_sync(FULL, v, L);
      for (int i = __popc(vw) - q; i > 0; --i) vw &= vw - 1;   // drop the lower ones
      const int g = (w1 - 1 - L) * 32 + (__ffs(vw) - 1);       // bit index of the r-th one
      return g - (r - 1);
    }
    need -= tot;
  }
  return 0;
}
// support rows (c_t > 0) with a <= t <= b: one coalesced pass over the bins
template <typename WT>
__device__ __forceinline__ int count_support_warp(const WT* __restrict__ we, int a, int b) {
  int c = 0;
  for (int t0 = a; t0 <= b; t0 += 32) {
    const int t = t0 + lane_id();
    c += __popc(__ballot_sync(FULL, t <= b && we[t] > 0));
  }
  return c;
}

// A hull line: intercept b_s (value type VT) and s.
template <typename VT>
struct Line {
  VT b;
  int s;
};

// Ring storage policies, [slot][pos][lane] so that every lane has its own banks: SRingI (int32
// lines, below) and SRingW (int64 / fp64 lines) in shared memory; WRing (int64 / fp64) = an
// SRingW window + per-layer global arrays for large hulls.

// double-double sums for the fp64 path (prefix sums rounded once, T_N, the definitional cost)
struct hdd {
  double hi, lo;
};
__device__ __forceinline__ hdd hdd_add(hdd a, hdd b) {
  const double s = a.hi + b.hi, bb = s - a.hi;
  double err = (a.hi - (s - bb)) + (b.hi - bb);
  err += a.lo + b.lo;
  const double h = s + err;
  return hdd{h, err - (h - s)};
}
__device__ __forceinline__ hdd hdd_prod(double a, double b) {
  const double p = a * b;
  return hdd{p, fma(a, b, -p)};
}
__device__ __forceinline__ hdd hdd_shfl_up(hdd v, int o) {
  return hdd{__shfl_up_sync(FULL, v.hi, o), __shfl_up_sync(FULL, v.lo, o)};
}
__device__ __forceinline__ hdd hdd_shfl(hdd v, int l) {
  return hdd{__shfl_sync(FULL, v.hi, l), __shfl_sync(FULL, v.lo, l)};
}
__device__ __forceinline__ hdd hdd_warp_sum(hdd v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    v = hdd_add(v, hdd{__shfl_xor_sync(FULL, v.hi, o), __shfl_xor_sync(FULL, v.lo, o)});
  return v;
}

// The int32 instantiation's rings: 6-byte lines, interleaved -- a position row holds the 32
// lanes' intercepts (int32, 128 B) then their s (uint16, 64 B), 192 B per row.  25% less shared
// memory than int2 lines (12 instead of 9 warps/SM: W5 43.2 -> 42.0 ms), and one IMAD (FMA pipe,
// the ALU pipe is the busier one) forms a row address with the s address at a per-lane constant
// offset (40.9 -> 38.9 ms vs separate intercept / s arrays).  Measured and dropped: mirrored
// guard rows for constant-offset loads (two fewer warps/SM, extra stores: slower).
template <int C0, int C1>
struct SRingI {
  uint32_t b0;   // shared address of slot 0, row 0, this lane's intercept
  uint32_t ds;   // s address - intercept address: 128 - 2 lane
  __device__ __forceinline__ uint32_t at(int k, int pos) const {
    const uint32_t q = (uint32_t)pos & (uint32_t)((k ? C1 : C0) - 1);
    return q * 192u + b0 + (k ? (uint32_t)C0 * 192u : 0u);
  }
  __device__ __forceinline__ Line<int> ld(int k, int pos) const {
    const uint32_t a = at(k, pos);
    Line<int> v;
    unsigned short sv;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v.b) : "r"(a));
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(sv) : "r"(a + ds));
    v.s = sv;
    return v;
  }
  __device__ __forceinline__ Line<int> ld_back(int k, int b, int t) const { return ld(k, b - t); }
  __device__ __forceinline__ Line<int> ld_front(int k, int f, int t) const { return ld(k, f + t); }
  __device__ __forceinline__ void st(int k, int pos, Line<int> v) const {
    const uint32_t a = at(k, pos);
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v.b) : "memory");
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a + ds), "h"((unsigned short)v.s) : "memory");
  }
  static constexpr int cap(int k) { return k ? C1 : C0; }
  __device__ __forceinline__ Line<int> ldh(int k, int pos, int) const { return ld(k, pos); }
  __device__ __forceinline__ void sth(int k, int pos, Line<int> v, int, int) const { st(k, pos, v); }
  __device__ __forceinline__ int span_cap(int k) const { return cap(k); }
  __device__ __forceinline__ void begin_pass(uint8_t*, int, int, int, int) {}
  __device__ __forceinline__ Line<int> ldw(int k, int pos) const { return ld(k, pos); }
  __device__ __forceinline__ void stw(int k, int pos, Line<int> v) const { st(k, pos, v); }
  static constexpr bool kWindowed = false;
  static constexpr int window(int k) { return cap(k); }
  static constexpr int UNIT = 1;
  static constexpr size_t bytes(int K) { return (size_t)(C0 + (K == 2 ? C1 : 0)) * 192; }
  __device__ __forceinline__ void ld2(int k, int pos, int& b, int& sv) const {
    const Line<int> l = ld(k, pos);
    b = l.b;
    sv = l.s;
  }
  __device__ __forceinline__ void st2(int k, int pos, int b, int sv) const { st(k, pos, Line<int>{b, sv}); }
};

// 10-byte lines for the int64 / fp64 instantiations, interleaved like SRingI: a 320-byte position
// row holds the 32 lanes' 8-byte intercepts then their s as uint16 (s <= N <= SP_MAX_N = 65535);
// one IMAD per row address.  With the 168-register cap (below) the shared memory is the bound:
// 10 warps per SM instead of 9 with 12-byte lines (int32 s, 384-byte rows, SP_HULL_WROW=384):
// accumulated rows 209.5 -> 201.3 ms, fp64 W5 rows 62.1 -> 58.8 ms (profiles/r02e_dp_variants.txt).
#ifndef SP_HULL_WROW
#define SP_HULL_WROW 320
#endif
constexpr uint32_t WROW = SP_HULL_WROW;
template <typename VT, int C0, int C1>
struct SRingW {
  uint32_t b0;   // shared address of slot 0, row 0, this lane's intercept
  uint32_t ds;   // s address - intercept address: 256 - 4 lane (WROW 320: 256 - 6 lane)
  __device__ __forceinline__ uint32_t at(int k, int pos) const {
    const uint32_t q = (uint32_t)pos & (uint32_t)((k ? C1 : C0) - 1);
    return q * WROW + b0 + (k ? (uint32_t)C0 * WROW : 0u);
  }
  __device__ __forceinline__ Line<VT> ld(int k, int pos) const {
    const uint32_t a = at(k, pos);
    Line<VT> v;
    if constexpr (std::is_same<VT, double>::value)
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v.b) : "r"(a));
    else
      asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v.b) : "r"(a));
    if constexpr (WROW == 320) {
      unsigned short sv;
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(sv) : "r"(a + ds));
      v.s = sv;
    } else {
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v.s) : "r"(a + ds));
    }
    return v;
  }
  __device__ __forceinline__ Line<VT> ld_back(int k, int b, int t) const { return ld(k, b - t); }
  __device__ __forceinline__ Line<VT> ld_front(int k, int f, int t) const { return ld(k, f + t); }
  __device__ __forceinline__ void st(int k, int pos, Line<VT> v) const {
    const uint32_t a = at(k, pos);
    if constexpr (std::is_same<VT, double>::value)
      asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v.b) : "memory");
    else
      asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(v.b) : "memory");
    if constexpr (WROW == 320)
      asm volatile("st.shared.u16 [%0], %1;" ::"r"(a + ds), "h"((unsigned short)v.s) : "memory");
    else
      asm volatile("st.shared.b32 [%0], %1;" ::"r"(a + ds), "r"(v.s) : "memory");
  }
  static constexpr int cap(int k) { return k ? C1 : C0; }
};

// Windowed ring.  hi = the largest position written since the entry's pass began.  Invariant for
// every live position q (fr <= q <= bk): q > hi - C -> the shared-memory window slot q mod C
// holds q; otherwise the global array holds it at q mod cap.  A push at pos = hi + 1 moves line
// pos - C (if live) from the window to the global array; a push at pos <= hi - C (after deep
// back pops) writes the global array as well.  So the hot end -- the back, and the front of
// small hulls -- stays in shared memory and only large hulls touch global memory.
//   int32 lines: window SRingI<HC0, HC1> (64 / 32 lines), global arrays of WSMALL lines: a hull
//     past them goes to the int64 instantiation;
//   int64 / fp64 lines: window SRingW<WC, WC>, global arrays of wring_cap(N, m) lines: a hull
//     past them goes to the D&C kernel.
constexpr int WSMALL = 256;
template <typename VT>
struct GLineT {   // a global line
  long long b;
  int s, pad;
};
template <>
struct GLineT<int> {
  int b, s;
};
// BIGCAP: the int32 large-hull mode (dp_hull_kernel<.., int, BIG>) sizes its int32 arrays like
// the int64 instantiation's, wring_cap(N, m)
template <typename VT, bool BIGCAP = false>
__host__ __device__ __forceinline__ int wring_cap_t(int N, int m) {
  return std::is_same<VT, int>::value && !BIGCAP ? WSMALL : wring_cap(N, m);
}
// bytes of one CTA's global arrays: the largest pass (the first: lowest layers, largest caps)
template <typename VT, bool BIGCAP = false>
__host__ __device__ __forceinline__ size_t wring_pass_bytes_t(int N, int M) {
  const int L = 32 * hull_K(M);
  size_t n = 0;
  for (int m = 1; m <= L; ++m) n += (size_t)wring_cap_t<VT, BIGCAP>(N, m);
  return hull_align(n * sizeof(GLineT<VT>));
}

template <typename VT, class SM, bool BIGCAP = false>
struct WRing {
  SM sm;
  GLineT<VT>* g[2];   // this lane's chain for slot 0 / 1 in the current pass
  int gm[2];          // its capacity - 1
  __device__ __forceinline__ Line<VT> gld(int k, int pos) const {
    const GLineT<VT> l = g[k][pos & gm[k]];
    Line<VT> v;
    if constexpr (std::is_same<VT, double>::value) v.b = __longlong_as_double(l.b);
    else v.b = (VT)l.b;
    v.s = l.s;
    return v;
  }
  __device__ __forceinline__ void gst(int k, int pos, Line<VT> v) const {
    GLineT<VT> l;
    if constexpr (std::is_same<VT, double>::value) l.b = __double_as_longlong(v.b);
    else l.b = v.b;
    l.s = v.s;
    if constexpr (!std::is_same<VT, int>::value) l.pad = 0;
    g[k][pos & gm[k]] = l;
  }
  __device__ __forceinline__ Line<VT> ldh(int k, int pos, int hi) const {
    return pos > hi - SM::cap(k) ? sm.ld(k, pos) : gld(k, pos);
  }
  __device__ __forceinline__ void sth(int k, int pos, Line<VT> v, int hi, int fr) const {
    const int C = SM::cap(k);
    if (pos > hi) {
      if (pos - C >= fr) gst(k, pos - C, sm.ld(k, pos));   // the slot holds pos - C
    } else if (pos <= hi - C) {
      gst(k, pos, v);
    }
    sm.st(k, pos, v);
  }
  __device__ __forceinline__ int span_cap(int k) const { return gm[k] + 1; }
  __device__ __forceinline__ const GLineT<VT>* gaddr(int k, int pos) const { return g[k] + (pos & gm[k]); }
  // plain window accesses (exact while the deque lies within C - 2 of hi: see hull_dp)
  __device__ __forceinline__ Line<VT> ldw(int k, int pos) const { return sm.ld(k, pos); }
  __device__ __forceinline__ void stw(int k, int pos, Line<VT> v) const { sm.st(k, pos, v); }
  static constexpr bool kWindowed = true;
  static constexpr int window(int k) { return SM::cap(k); }
  // point g[] at this pass's chains: the layers of a pass are laid out in order
  __device__ __forceinline__ void begin_pass(uint8_t* base, int N, int M, int ps, int L) {
    const int lane = lane_id();
    size_t off = 0;
    for (int q = 0; q < L; ++q) {   // every slot, active or not (inactive lanes still load/store)
      const int m = ps * L + q + 1;
      const int c = wring_cap_t<VT, BIGCAP>(N, m);
      if ((q & 31) == lane) {   // (constant indices: g[] stays in registers)
        GLineT<VT>* gp = reinterpret_cast<GLineT<VT>*>(base) + off;
        if ((q >> 5) == 0) {
          g[0] = gp;
          gm[0] = c - 1;
        } else {
          g[1] = gp;
          gm[1] = c - 1;
        }
      }
      off += (size_t)c;
    }
  }
};

template <int K, typename VT>
__host__ __device__ constexpr size_t ring_bytes() {
  if constexpr (sizeof(VT) == 8) return (size_t)(WC + (K == 2 ? WC : 0)) * WROW;
  return (size_t)(HC0 + (K == 2 ? HC1 : 0)) * 192;
}
// per-warp row staging in shared memory: none (the counts wait in a register queue, HULL_PF
// chunks deep; a shared stage cost a warp per SM and was dropped)
template <typename VT>
__host__ __device__ constexpr size_t stage_bytes() { return 0; }
template <int K, typename VT>
constexpr size_t hull_dyn_bytes() { return ring_bytes<K, VT>() + stage_bytes<VT>(); }

// prefetch one global address into L1 (no register written, nothing to wait on)
template <typename T>
__device__ __forceinline__ void prefetch_l1(const T* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// prefetch one global address into L2
template <typename T>
__device__ __forceinline__ void prefetch_l2(const T* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// value of the dummy front line (above every candidate)
template <typename VT>
__device__ __forceinline__ VT hull_inf() {
  if constexpr (std::is_same<VT, double>::value) return HUGE_VAL;
  else if constexpr (std::is_same<VT, long long>::value) return LLONG_MAX;
  else return INT_MAX;
}

// back-pop test with the new point (j, bj) as origin: for the pair (A, Bk) of consecutive hull
// lines (A below Bk), with A' = A - new and Bk' = Bk - new in (s, b) coordinates, Bk goes iff it is
// not strictly below the segment A -> new, i.e. cross(A', Bk') = A'.s Bk'.b - A'.b Bk'.s <= 0.
// |s'| < 2^16 and |b'| <= n N: < 2^30 on the int32 path, < 2^46 on the int64 path (guards in
// the kernel), so both products are exact in int64.
template <typename VT>
__device__ __forceinline__ bool pop_test(int as, VT ab, int ks, VT kb) {
  return (long long)as * (long long)kb <= (long long)ab * (long long)ks;
}
// fp64 weights: the same test in double (reading R10: a misjudged near-collinear triple moves a
// value by rounding only, so the placement stays optimal to ~M eps relative)
template <>
__device__ __forceinline__ bool pop_test<double>(int as, double ab, int ks, double kb) {
  return (double)as * kb <= ab * (double)ks;
}

// a4 for one entry: all layers in lockstep, one support row per step.  Returns true when a ring
// overflowed (the entry's results are then invalid).
template <typename VT>
using HullCT = typename std::conditional<std::is_same<VT, double>::value, double, long long>::type;

// SPLIT mode (small batches): the two warps of a CTA share an entry, warp 0 running layers 1-32
// (pass 0) and warp 1 layers 33-64 (pass 1); e_32(j) of every support row goes from warp 0's
// lane 31 to warp 1's lane 0 through a shared-memory ring instead of the global e-row buffer
// of sequential passes.  Warp 0 publishes after each 32-row chunk, warp 1 releases ring space
// after each chunk; either warp raises `abort` when it gives the entry up (ring / log full).
constexpr int SPLIT_RING = 1024;
#ifndef SP_SPLIT_NS
#define SP_SPLIT_NS 64   // SPLIT mode: back-off of a warp waiting for the other (ns)
#endif
struct SplitSync {
  int* ring;                 // shared, SPLIT_RING ints
  volatile int* produced;    // support rows published by warp 0
  volatile int* consumed;    // lowest support-row index warp 1 still needs
  volatile int* abort_;      // either warp gave the entry up
};

// ALLACT: every slot of every pass holds a layer (M a multiple of 32 K) -- the per-slot "active"
// predicates vanish at compile time
// BIG (int32, the large-hull mode): argmin logs in unary form -- per stepped (support) row,
// opt_m(j) - opt_m(j_prev) zero bits then a one bit, LSB first -- at most K + N <= 2N bits per
// layer whatever the hull does (a change log fills when opt moves on most rows, e.g. all-ones);
// the front lines of hulls that outgrow the window are prefetched into L2 16 positions ahead.
template <typename WT, typename VT, int K, bool ALLACT, class RING, bool CMP = false, bool BIG = false,
          bool ONEPASS = false, int ROLE = 0>
__device__ __forceinline__ bool hull_dp(const HullParams& p, const WT* __restrict__ we, int e,
                                        HullCT<VT> TN, VT nV, RING rg, uint32_t* logs,
                                        int32_t* logn, VT* ebuf0, VT* ebuf1,
                                        unsigned& pops_e, unsigned& ev_e, bool& logfull,
                                        VT* stage, int kc = -1, const int2* klist = nullptr,
                                        const SplitSync* ss = nullptr, int ps_only = -1) {
  const int lane = lane_id();
  const int N = p.N, M = p.M;
  const int LC = p.logcap;   // <= hull_log_cap(N), the allocated stride
  // the two lines above the front loaded a row ahead, the front prefetched into L2: the
  // large-hull mode, and (SP_HULL_AHEAD_WIDE) the int64 / fp64 windowed instantiations
#ifdef SP_HULL_AHEAD_WIDE
  constexpr bool AHEAD = BIG || (RING::kWindowed && sizeof(VT) == 8);
#else
  constexpr bool AHEAD = BIG;
#endif
  logfull = false;
  constexpr int L = 32 * K;
  const int passes = (M + L - 1) / L;
  bool ovf = false;
  const int ps_begin = ps_only < 0 ? 0 : ps_only, ps_end = ps_only < 0 ? passes : ps_only + 1;
  for (int ps = ps_begin; ps < ps_end && !ovf; ++ps) {
    const VT* ein = (ps & 1) ? ebuf1 : ebuf0;    // e_{64 ps}(.) from the previous pass
    VT* eout_buf = (ps & 1) ? ebuf0 : ebuf1;
    // ONEPASS (M = 32 K, no SPLIT partner): no chained e-rows at compile time
    // ROLE (SPLIT mode at compile time): 1 = warp 0 (pass 0, chains out), 2 = warp 1 (pass 1,
    // chains in); 0 = decided at run time
    const bool chain_in = ROLE == 2 ? true : ROLE == 1 ? false : !ONEPASS && ps > 0;
    const bool chain_out = ROLE == 1 ? true : ROLE == 2 ? false : !ONEPASS && ps + 1 < passes;
    // Per slot: deque [f, b] (monotone counters; ring position = counter mod capacity).  In
    // registers: the back line B0 (the last one pushed) and the front line F0; the two lines
    // below the back and the two above the front are loaded from the ring at the top of every
    // support row (positions known a row ahead, so the loads overlap the shuffle).  A line is
    // (intercept b_s, s).  eo = e_m(j) (the running row value), op = opt_m(j).
    int f[K], b[K], op[K], cnt[K], hi[K];
    uint32_t uw[K];   // BIG: the unary log's current word and its used bits
    int ub[K];
    rg.begin_pass(p.wg + (size_t)blockIdx.x * p.wgb, N, M, ps, L);
    VT eo[K];
    Line<VT> B0[K], F0[K];
    bool act[K];
    uint32_t* lg[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int mk = ps * L + 32 * k + lane + 1;
      act[k] = ALLACT || mk <= M;
      f[k] = 0;
      b[k] = 0;
      eo[k] = 0;   // e_m(0) = 0 (reading R1)
      op[k] = BIG ? 0 : 1;   // opt_m(1) = 1 whatever the row type: logged up front (BIG: the
      cnt[k] = BIG ? 0 : 1;  // unary stream starts from opt = 0)
      uw[k] = 0;
      ub[k] = 0;
      lg[k] = logs + (size_t)(ps * L + 32 * k + lane) * LC;
      if (!BIG && act[k]) lg[k][0] = (1u << 16) | 1u;
      // the deque starts with a dummy line of value +inf at every query: the first push pops
      // it from the front, so the deque is never empty at a push
      B0[k] = F0[k] = Line<VT>{hull_inf<VT>(), 0};
      rg.sth(k, 0, F0[k], -1, 0);
      hi[k] = 0;   // the largest position written (the windowed ring's threshold)
    }
    VT carry = 0, Pm1 = 0;
    hdd carry_dd{0.0, 0.0};
    Line<VT> NG1[K], NG2[K];   // BIG: lines f + 1, f + 2 for the next row
#pragma unroll
    for (int k = 0; k < K; ++k) NG1[k] = NG2[k] = Line<VT>{hull_inf<VT>(), 0};
    int evbase = 0;   // support rows (c_j > 0) before this chunk = index into the e-row buffers
    // the counts are loaded HULL_PF chunks (32 rows each) ahead: a chunk of W5's rows holds ~5
    // support rows, but sparse rows (W2/W3: ~0.2-2% support) would otherwise wait for HBM on
    // every 32 rows
    // Rows: dense rows are read 32 at a time with HULL_PF chunks in flight (a register queue);
    // sparse rows (K <= HULL_KC, compacted by the pre-pass) are walked as their list of (j, c_j)
    // pairs instead -- no scan over the N bins (CMP: a compile-time path).
    constexpr bool compact = CMP;
    const int total = compact ? kc : N;
    VT cq[HULL_PF];
    if constexpr (!compact) {
#ifdef SP_HULL_REGQ
#pragma unroll
      for (int c = 0; c < HULL_PF; ++c)
        cq[c] = 32 * c + 1 + lane <= N ? (VT)we[32 * c + 1 + lane] : (VT)0;
#else
      cq[0] = 1 + lane <= N ? (VT)we[1 + lane] : (VT)0;
#pragma unroll
      for (int c = 1; c < HULL_PF; ++c)
        if (32 * c + 1 + lane <= N) prefetch_l1(we + 32 * c + 1 + lane);
#endif
    }
    for (int jb = 0; jb < total; jb += 32) {
      int jr;
      VT craw;
      if constexpr (compact) {
        const int2 v = jb + lane < kc ? klist[jb + lane] : make_int2(0, 0);
        jr = v.x;
        craw = (VT)v.y;
      } else {
        jr = jb + 1 + lane;
        craw = cq[0];
#ifdef SP_HULL_REGQ
#pragma unroll
        for (int c = 0; c + 1 < HULL_PF; ++c) cq[c] = cq[c + 1];
        cq[HULL_PF - 1] = jr + 32 * HULL_PF <= N ? (VT)we[jr + 32 * HULL_PF] : (VT)0;
#else
        // the next chunk into a register (an L1 hit: prefetched HULL_PF chunks ago), the chunk
        // HULL_PF ahead into L1.  (A register queue HULL_PF deep made every chunk's queue shift
        // wait on the newest load: the prefetch distance was one chunk.)
        cq[0] = jr + 32 <= N ? (VT)we[jr + 32] : (VT)0;
        if (jr + 32 * HULL_PF <= N) prefetch_l1(we + jr + 32 * HULL_PF);
#endif
      }
      unsigned evmask = __ballot_sync(FULL, craw > 0);   // support rows of this chunk
      if (evmask == 0) continue;                          // 32 zero rows: nothing changes
      VT Pc;
      if constexpr (std::is_same<VT, double>::value) {
        // P_j from a double-double scan, rounded once (reading R10)
        hdd inc{craw, 0.0};
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const hdd y = hdd_shfl_up(inc, o);
          if (lane >= o) inc = hdd_add(inc, y);
        }
        const hdd full = hdd_add(carry_dd, inc);
        Pc = full.hi + full.lo;
        carry_dd = hdd_shfl(full, 31);
      } else {
        VT cnt32 = craw;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const VT y = __shfl_up_sync(FULL, cnt32, o);
          if (lane >= o) cnt32 += y;
        }
        Pc = carry + cnt32;
        carry = __shfl_sync(FULL, Pc, 31);
      }
      // previous pass's top layer at the support rows: e(j-1) of support row number t is its
      // value at support row t-1 (constant over zero rows), 0 before the first
      VT Ec = 0;
      const int nev = __popc(evmask);
      if (!ONEPASS && ss) {   // SPLIT mode: wait for the other warp (consumer: data; producer: ring space)
        if (lane == 0) {
          if (chain_in)
            while (*ss->produced < evbase + nev - 1 && !*ss->abort_) __nanosleep(SP_SPLIT_NS);
          else
            while (evbase + nev - 1 - *ss->consumed >= SPLIT_RING && !*ss->abort_) __nanosleep(SP_SPLIT_NS);
        }
        __syncwarp();
        if (*ss->abort_) {
          ovf = true;
          break;
        }
        __threadfence_block();
        if (chain_in && lane < nev)
          Ec = evbase + lane >= 1 ? (VT)ss->ring[(evbase + lane - 1) & (SPLIT_RING - 1)] : (VT)0;
      } else if (chain_in && lane < nev) {
        Ec = evbase + lane >= 1 ? ein[evbase + lane - 1] : 0;
      }
      for (int q = 0; evmask; ++q) {
        const int i = __ffs(evmask) - 1;
        evmask &= evmask - 1;
        const int j = compact ? __shfl_sync(FULL, jr, i) : jb + 1 + i;
        // ring lines around both ends (positions fixed by the previous row).  Windowed rings:
        // while every lane's deque lies within C - 2 positions of its high-water mark (the
        // common case) every line it touches this row is in the shared window -- plain shared
        // loads and stores; otherwise (warp-uniform) the checked window / global accesses.
        bool wbig = false;
        if constexpr (RING::kWindowed) {
#pragma unroll
          for (int k = 0; k < K; ++k) wbig |= act[k] & (hi[k] - f[k] >= RING::window(k) - 2);
        }
        const bool win = RING::kWindowed && __any_sync(FULL, wbig);
        Line<VT> L1[K], L2[K], G1[K], G2[K];
        if (win) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            L1[k] = rg.ldh(k, b[k] - 1, hi[k]);
            L2[k] = rg.ldh(k, b[k] - 2, hi[k]);
            if constexpr (AHEAD) {   // loaded a row ahead (below); the front walks a global array:
              G1[k] = NG1[k];      // pull it into L2 further ahead
              G2[k] = NG2[k];
              const int q = f[k] + 16;
              if (act[k] & (q <= hi[k] - RING::window(k))) prefetch_l2(rg.gaddr(k, q));
            } else {
              G1[k] = rg.ldh(k, f[k] + 1, hi[k]);
              G2[k] = rg.ldh(k, f[k] + 2, hi[k]);
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            L1[k] = rg.ldw(k, b[k] - 1);
            L2[k] = rg.ldw(k, b[k] - 2);
            G1[k] = AHEAD ? NG1[k] : rg.ldw(k, f[k] + 1);
            G2[k] = AHEAD ? NG2[k] : rg.ldw(k, f[k] + 2);
          }
        }
        // e_{m-1}(j-1): from the lane below (its value at the previous support row);
        // lane 0 slot 0 from the previous pass (or e_0 = 0)
        VT in[K];
        const VT t0 = __shfl_sync(FULL, eo[0], (lane + 31) & 31);
        // only after a previous pass (warp-uniform): Ec's register is the target of a load that
        // is predicated off in a single pass, and a shuffle reading it waited on its scoreboard
        VT ext = 0;
        if (chain_in) ext = __shfl_sync(FULL, Ec, q);
        in[0] = lane ? t0 : ext;
        if constexpr (K == 2) {
          const VT t1 = __shfl_sync(FULL, eo[1], (lane + 31) & 31);
          in[1] = lane ? t1 : t0;
        }
        const VT Pj = __shfl_sync(FULL, Pc, i);
        const VT nPj = -Pj;
        ++ev_e;
        // ---- push line j: up to two back pops decided from the loaded lines ----------------
        VT bj[K];
        int top[K];
        bool more[K], skip[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          bj[k] = in[k] + (VT)j * Pm1;
          // deltas of the back lines from the new point (j, bj)
          const int s0 = B0[k].s - j, s1 = L1[k].s - j, s2 = L2[k].s - j;
          const VT c0 = B0[k].b - bj[k], c1 = L1[k].b - bj[k], c2 = L2[k].b - bj[k];
          // a line that overtakes the back line only beyond x = P_N = n is never optimal at a
          // query (x <= n): it is neither pushed nor allowed to pop.
          // x(back, new) > n  <=>  bj - B0.b > n (j - B0.s)  <=>  -c0 > -n s0
          // (trimming pays only where hulls are large -- the int64 instantiation's accumulated
          // rows; on W5's int32 rows it costs 1.5% net)
          if constexpr (std::is_same<VT, long long>::value)
            skip[k] = c0 < nV * (VT)s0;   // (the deque is never empty: the dummy line)
          else
            skip[k] = false;
          const int sz = skip[k] ? 0 : b[k] - f[k];   // deque size - 1, before the push
          const int p1 = (sz >= 1) & pop_test(s1, c1, s0, c0);
          const int p2 = p1 & (sz >= 2) & pop_test(s2, c2, s1, c1);
          // two pops decided eagerly; a lane with two pops may pop more: the warp-uniform loop
          // below tests further lines (W5 34.3 -> 33.1 ms vs four eager tests)
          top[k] = b[k] - (p1 + p2);   // position of the new second-to-back line
          more[k] = act[k] & (p2 != 0);
        }
        bool anymore = more[0];
        if constexpr (K == 2) anymore |= more[1];
#ifdef SP_HULL_BRSTATS   // instrumentation (tools/prof_dp.py, SP_BRSTATS_REPORT): rows, loops taken
        if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(p.ws + 64), 1ull);
        if (__any_sync(FULL, anymore) && lane == 0)
          atomicAdd(reinterpret_cast<unsigned long long*>(p.ws + 72), 1ull);
#endif
        if (__any_sync(FULL, anymore)) {   // a lane popped two lines: keep testing from the ring
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (!more[k]) continue;
            int cs = L2[k].s - j;
            VT cb = L2[k].b - bj[k];
#ifdef SP_HULL_LOOP_PF
            // the line below the one under test is loaded with it, so an iteration's test does
            // not wait for its own load (one speculative load when the loop stops)
            Line<VT> nx = rg.ldh(k, top[k] - 1, hi[k]);
            while (top[k] - f[k] >= 1) {
              const Line<VT> l1 = nx;
              if (top[k] - f[k] >= 2) nx = rg.ldh(k, top[k] - 2, hi[k]);
              const int ls = l1.s - j;
              const VT lb = l1.b - bj[k];
              if (pop_test(ls, lb, cs, cb)) {
                --top[k];
                cs = ls;
                cb = lb;
              } else {
                break;
              }
            }
#else
            while (top[k] - f[k] >= 1) {
              const Line<VT> l1 = rg.ldh(k, top[k] - 1, hi[k]);
              const int ls = l1.s - j;
              const VT lb = l1.b - bj[k];
              if (pop_test(ls, lb, cs, cb)) {
                --top[k];
                cs = ls;
                cb = lb;
              } else {
                break;
              }
            }
#endif
          }
        }
        VT v0[K], v1[K], v2[K];
        bool q2[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int nb = skip[k] ? b[k] : top[k] + 1;
          const Line<VT> nl{bj[k], j};
          if (!skip[k]) {
            if (win) rg.sth(k, nb, nl, hi[k], f[k]);
            else rg.stw(k, nb, nl);
            hi[k] = max(hi[k], nb);
          }
          const int d = nb - f[k];
          const bool fresh = !skip[k];
          const Line<VT> F1 = (fresh & (d == 1)) ? nl : G1[k];   // lines f+1 / f+2 popped or new
          const Line<VT> F2 = (fresh & (d == 2)) ? nl : G2[k];
          B0[k] = skip[k] ? B0[k] : nl;
          b[k] = nb;
          ovf |= act[k] & (d >= rg.span_cap(k));
          // ---- query x = P_j: up to one front pop decided from the loaded lines -------------
          v0[k] = F0[k].b + (VT)F0[k].s * nPj;
          v1[k] = F1.b + (VT)F1.s * nPj;
          v2[k] = F2.b + (VT)F2.s * nPj;
          const bool q1 = act[k] & (d >= 1) & (v1[k] < v0[k]);
          q2[k] = q1 & (d >= 2) & (v2[k] < v1[k]);
          const bool one = q1 & !q2[k];
          f[k] += one;
          F0[k] = one ? F1 : (q2[k] ? F2 : F0[k]);
          v0[k] = one ? v1[k] : (q2[k] ? v2[k] : v0[k]);
        }
        bool anyq2 = q2[0];
        if constexpr (K == 2) anyq2 |= q2[1];
#ifdef SP_HULL_BRSTATS
        if (__any_sync(FULL, anyq2) && lane == 0)
          atomicAdd(reinterpret_cast<unsigned long long*>(p.ws + 80), 1ull);
#endif
        if (__any_sync(FULL, anyq2)) {   // rare: the front moves by two or more
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (!q2[k]) continue;
            f[k] += 2;   // F0 = line f+2 already
            while (f[k] < b[k]) {
              const Line<VT> l1 = rg.ldh(k, f[k] + 1, hi[k]);
              const VT vl = l1.b + (VT)l1.s * nPj;
              if (vl < v0[k]) {
                ++f[k];
                F0[k] = l1;
                v0[k] = vl;
              } else {
                break;
              }
            }
          }
        }
        Pm1 = Pj;
        if constexpr (AHEAD) {   // the next row's two lines above the front, a row ahead: a front in
#pragma unroll                 // the global array then has a whole row to arrive (the only writes
          for (int k = 0; k < K; ++k) {   // before their use are covered by the d <= 2 selects)
            NG1[k] = rg.ldh(k, f[k] + 1, hi[k]);
            NG2[k] = rg.ldh(k, f[k] + 2, hi[k]);
          }
        }
        // ---- row value, argmin change log ---------------------------------------------------
#pragma unroll
        for (int k = 0; k < K; ++k) {
          eo[k] = v0[k];
          const int nop = F0[k].s;
          if constexpr (BIG) {
            if (act[k]) {   // unary: nop - op zeros, then a one (<= 2N bits: never full)
              int t = ub[k] + (nop - op[k]);
              while (t >= 32) {
                lg[k][cnt[k]++] = uw[k];
                uw[k] = 0;
                t -= 32;
              }
              uw[k] |= 1u << t;
              ub[k] = t + 1;
              if (ub[k] == 32) {
                lg[k][cnt[k]++] = uw[k];
                uw[k] = 0;
                ub[k] = 0;
              }
            }
          } else if (act[k] & (nop != op[k])) {
            lg[k][cnt[k]] = ((uint32_t)j << 16) | (uint32_t)nop;   // < LC: checked per chunk
            ++cnt[k];
          }
          op[k] = nop;
        }
        if (chain_out && lane == 31) {
          if (ss) ss->ring[(evbase + q) & (SPLIT_RING - 1)] = (int)eo[K - 1];
          else eout_buf[evbase + q] = eo[K - 1];
        }
      }
      if (!ONEPASS && ss) {   // publish this chunk (producer) / release its ring slots (consumer)
        __syncwarp();
        __threadfence_block();
        if (lane == 0) {
          if (chain_out) *ss->produced = evbase + nev;
          else *ss->consumed = evbase + nev - 1;
        }
      }
      evbase += nev;
      bool full = false;
#pragma unroll
      for (int k = 0; k < K; ++k) full |= !BIG & (LC <= N) & (cnt[k] > LC - 33);   // 32 rows of headroom
      logfull = __any_sync(FULL, full);
      if (__any_sync(FULL, ovf) || logfull) {
        ovf = true;
        if (ss && lane == 0) *ss->abort_ = 1;
        break;
      }
    }
    if (!ovf) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!act[k]) continue;
        if (BIG && ub[k] > 0) lg[k][cnt[k]++] = uw[k];   // the unary log's last word
        // stats: pushes (support rows, less trimmed lines) = back pops + b; front pops = f - 1
        pops_e += (unsigned)(evbase - b[k]) + (unsigned)(f[k] - 1);
        const int mk = ps * L + 32 * k + lane + 1;
        logn[ps * L + 32 * k + lane] = cnt[k];
        const HullCT<VT> V = TN + (HullCT<VT>)eo[k];   // V_m = T_N + e_m(N)
        if (p.cbb) reinterpret_cast<HullCT<VT>*>(p.cbb)[(int64_t)e * (M + 1) + mk] = V;
        if (mk == M) reinterpret_cast<HullCT<VT>*>(p.cost)[e] = V;
      }
    }
    __syncwarp();   // chained e-row and logs visible to the whole warp
  }
  return ovf;
}

// The skewed step (int32, K = 2, one pass, dense rows; compiled in with -DSP_HULL_SKEW; measured
// slower than hull_dp on W5, 49.3 vs 29.6 ms): slot k of lane l runs layer 32k + l + 1 on support row t - l - 32k at step t, so the
// e_{m-1}(j-1) it needs from the lane below is two steps old and the shuffle that brings it (and
// the lane below's front work) leave the row's critical path; row data (j, P_j) move one lane up
// per step (a systolic shift), lane 0 taking the next support row.  The CHT step itself is the
// one of hull_dp.  The pipeline fills and drains over 63 extra steps per entry.
template <typename WT, bool ALLACT, class RING>
__device__ __forceinline__ bool hull_dp_skew(const HullParams& p, const WT* __restrict__ we, int e,
                                             long long TN, RING rg, uint32_t* logs, int32_t* logn,
                                             unsigned& pops_e, unsigned& ev_e, bool& logfull) {
  constexpr int K = 2;
  using VT = int;
  const int lane = lane_id();
  const int N = p.N, M = p.M;
  const int LC = p.logcap;
  logfull = false;
  bool ovf = false;
  int f[K], b[K], op[K], cnt[K];
  VT eo[K];
  Line<VT> B0[K], F0[K];
  bool act[K];
  uint32_t* lg[K];
  int rj[K], rP[K], pm[K];   // this step's row (j = 0: none) and P_j, and P_{j-1}
  VT q0[K], q1[K];           // e_{m-1} from the lane below, one and two steps old
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int mk = 32 * k + lane + 1;
    act[k] = ALLACT || mk <= M;
    f[k] = 0;
    b[k] = 0;
    eo[k] = 0;   // e_m(0) = 0 (reading R1)
    op[k] = 1;
    cnt[k] = 1;
    lg[k] = logs + (size_t)(32 * k + lane) * LC;
    if (act[k]) lg[k][0] = (1u << 16) | 1u;
    B0[k] = F0[k] = Line<VT>{hull_inf<VT>(), 0};
    rg.st(k, 0, F0[k]);
    rj[k] = rP[k] = pm[k] = 0;
    q0[k] = q1[k] = 0;
  }
  // the row source: 32-row chunks, HULL_PF in flight
  VT cq[HULL_PF];
#pragma unroll
  for (int c = 0; c < HULL_PF; ++c)
    cq[c] = 32 * c + 1 + lane <= N ? (VT)we[32 * c + 1 + lane] : (VT)0;
  int jn = 0;              // next chunk base
  int jbc = 0;             // current chunk base
  unsigned evmask = 0;     // support rows of the current chunk not yet supplied
  VT Pc = 0, carry = 0;
  int supplied = 0, drain = 0;
  for (int t = 0; drain < 64; ++t) {
    // ---- supply: the next support row for lane 0, slot 0 -------------------------------------
    while (evmask == 0 && jn < N) {   // (warp-uniform)
      const VT craw = cq[0];
#pragma unroll
      for (int c = 0; c + 1 < HULL_PF; ++c) cq[c] = cq[c + 1];
      const int jr = jn + 1 + lane;
      cq[HULL_PF - 1] = jr + 32 * HULL_PF <= N ? (VT)we[jr + 32 * HULL_PF] : (VT)0;
      evmask = __ballot_sync(FULL, craw > 0);
      VT c32 = craw;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const VT y = __shfl_up_sync(FULL, c32, o);
        if (lane >= o) c32 += y;
      }
      Pc = carry + c32;
      carry = __shfl_sync(FULL, Pc, 31);
      jbc = jn;
      jn += 32;
    }
    int nj = 0, nP = 0;
    if (evmask) {
      const int i = __ffs(evmask) - 1;
      evmask &= evmask - 1;
      nj = jbc + 1 + i;
      nP = __shfl_sync(FULL, Pc, i);
      ++supplied;
    } else {
      ++drain;   // no more rows: 63 more steps carry the last one through every slot
    }
    // ---- the systolic shift of the rows --------------------------------------------------
    {
      const int src = (lane + 31) & 31;
      const int sj0 = __shfl_sync(FULL, rj[0], src), sP0 = __shfl_sync(FULL, rP[0], src);
      const int sj1 = __shfl_sync(FULL, rj[1], src), sP1 = __shfl_sync(FULL, rP[1], src);
#pragma unroll
      for (int k = 0; k < K; ++k) pm[k] = rj[k] ? rP[k] : pm[k];   // P_{j-1}: the last row's P
      rj[1] = lane ? sj1 : sj0;
      rP[1] = lane ? sP1 : sP0;
      rj[0] = lane ? sj0 : nj;
      rP[0] = lane ? sP0 : nP;
    }
    // ---- the CHT step of every (valid) slot ----------------------------------------------
    bool val[K];
    VT in[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      val[k] = act[k] & (rj[k] > 0);
      in[k] = q1[k];
    }
    Line<VT> L1[K], L2[K], G1[K], G2[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      L1[k] = rg.ld(k, b[k] - 1);
      L2[k] = rg.ld(k, b[k] - 2);
      G1[k] = rg.ld(k, f[k] + 1);
      G2[k] = rg.ld(k, f[k] + 2);
    }
    VT bj[K];
    int top[K];
    bool more[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = rj[k];
      bj[k] = in[k] + (VT)j * pm[k];
      const int s0 = B0[k].s - j, s1 = L1[k].s - j, s2 = L2[k].s - j;
      const VT c0 = B0[k].b - bj[k], c1 = L1[k].b - bj[k], c2 = L2[k].b - bj[k];
      const int sz = val[k] ? b[k] - f[k] : 0;
      const int p1 = (sz >= 1) & pop_test(s1, c1, s0, c0);
      const int p2 = p1 & (sz >= 2) & pop_test(s2, c2, s1, c1);
      top[k] = b[k] - (p1 + p2);
      more[k] = val[k] & (p2 != 0);
    }
    bool anymore = more[0] | more[1];
    if (__any_sync(FULL, anymore)) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!more[k]) continue;
        const int j = rj[k];
        int cs = L2[k].s - j;
        VT cb = L2[k].b - bj[k];
        while (top[k] - f[k] >= 1) {
          const Line<VT> l1 = rg.ld(k, top[k] - 1);
          const int ls = l1.s - j;
          const VT lb = l1.b - bj[k];
          if (pop_test(ls, lb, cs, cb)) {
            --top[k];
            cs = ls;
            cb = lb;
          } else {
            break;
          }
        }
      }
    }
    VT v0[K];
    bool q2[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = rj[k];
      const VT nPj = -rP[k];
      const int nb = val[k] ? top[k] + 1 : b[k];
      const Line<VT> nl{bj[k], j};
      if (val[k]) rg.st(k, nb, nl);
      const int d = nb - f[k];
      const Line<VT> F1 = (val[k] & (d == 1)) ? nl : G1[k];
      const Line<VT> F2 = (val[k] & (d == 2)) ? nl : G2[k];
      B0[k] = val[k] ? nl : B0[k];
      b[k] = nb;
      ovf |= val[k] & (d >= RING::cap(k));
      v0[k] = F0[k].b + (VT)F0[k].s * nPj;
      const VT v1 = F1.b + (VT)F1.s * nPj;
      const VT v2 = F2.b + (VT)F2.s * nPj;
      const bool q1 = val[k] & (d >= 1) & (v1 < v0[k]);
      q2[k] = q1 & (d >= 2) & (v2 < v1);
      const bool one = q1 & !q2[k];
      f[k] += one;
      F0[k] = one ? F1 : (q2[k] ? F2 : F0[k]);
      v0[k] = one ? v1 : (q2[k] ? v2 : v0[k]);
    }
    if (__any_sync(FULL, q2[0] | q2[1])) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!q2[k]) continue;
        const VT nPj = -rP[k];
        f[k] += 2;
        while (f[k] < b[k]) {
          const Line<VT> l1 = rg.ld(k, f[k] + 1);
          const VT vl = l1.b + (VT)l1.s * nPj;
          if (vl < v0[k]) {
            ++f[k];
            F0[k] = l1;
            v0[k] = vl;
          } else {
            break;
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (val[k]) eo[k] = v0[k];
      const int nop = F0[k].s;
      if (val[k] & (nop != op[k])) {
        lg[k][cnt[k]] = ((uint32_t)rj[k] << 16) | (uint32_t)nop;   // < LC: checked below
        ++cnt[k];
      }
      op[k] = val[k] ? nop : op[k];
    }
    // ---- e_{m-1} for the lane above, two steps ahead ---------------------------------------
    {
      const int src = (lane + 31) & 31;
      const VT t0 = __shfl_sync(FULL, eo[0], src);
      const VT t1 = __shfl_sync(FULL, eo[1], src);
      q1[0] = q0[0];
      q1[1] = q0[1];
      q0[0] = lane ? t0 : 0;    // layer 1: e_0 = 0
      q0[1] = lane ? t1 : t0;   // layer 33: layer 32 is lane 31's slot 0
    }
    if ((t & 31) == 31) {   // ring / log capacity (the log takes <= 1 entry per step)
      bool full = false;
#pragma unroll
      for (int k = 0; k < K; ++k) full |= (LC <= N) & (cnt[k] > LC - 33);
      logfull = __any_sync(FULL, full);
      if (__any_sync(FULL, ovf) || logfull) {
        ovf = true;
        break;
      }
    }
  }
  if (__any_sync(FULL, ovf)) ovf = true;
  ev_e += supplied;
  if (!ovf) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!act[k]) continue;
      pops_e += (unsigned)(supplied - b[k]) + (unsigned)(f[k] - 1);
      const int mk = 32 * k + lane + 1;
      logn[32 * k + lane] = cnt[k];
      const long long V = TN + (long long)eo[k];
      if (p.cbb) reinterpret_cast<long long*>(p.cbb)[(int64_t)e * (M + 1) + mk] = V;
      if (mk == M) reinterpret_cast<long long*>(p.cost)[e] = V;
    }
  }
  __syncwarp();
  return ovf;
}

// dispatch to the compact-list walk (sparse rows) or the row scan (CMP: compile-time)
template <typename WT, typename VT, int K, bool ALLACT, class RING, bool BIG = false,
          bool ONEPASS = false, int ROLE = 0>
__device__ __forceinline__ bool hull_dp_any(const HullParams& p, const WT* __restrict__ we, int e,
                                            HullCT<VT> TN, VT nV, RING rg, uint32_t* logs,
                                            int32_t* logn, VT* ebuf0, VT* ebuf1, unsigned& pops_e,
                                            unsigned& ev_e, bool& logfull, VT* stage, int kc,
                                            const int2* klist, const SplitSync* ss = nullptr,
                                            int ps_only = -1) {
  if (kc >= 0)
    return hull_dp<WT, VT, K, ALLACT, RING, true, BIG, ONEPASS, ROLE>(p, we, e, TN, nV, rg, logs, logn,
                                                                ebuf0, ebuf1, pops_e, ev_e, logfull,
                                                                stage, kc, klist, ss, ps_only);
  return hull_dp<WT, VT, K, ALLACT, RING, false, BIG, ONEPASS, ROLE>(p, we, e, TN, nV, rg, logs, logn,
                                                               ebuf0, ebuf1, pops_e, ev_e, logfull,
                                                               stage, -1, nullptr, ss, ps_only);
}

// a7: the definitional cost sum_t w_t (t - l(t; C)) of a placement C = {c_1 < ... < c_k} for fp64
// weights, as T_N - sum_i c_i (P(c_{i+1} - 1) - P(c_i - 1)) (c_{k+1} = N + 1) from
// the row's prefix sums P in double-double: O(k) lookups per placement instead of a walk over
// the bins (round 1 walked the row once per 32 budgets with a pointer per lane: 110 ms of the
// fp64 W5 launch).  The cancellation in T_N - sum costs ~1e-31 T_N absolute, far inside reading
// R10's 1e-12 bound.  The prefix goes to the slot's two e-row buffers (free after the DP).
__device__ __forceinline__ hdd hdd_neg(hdd a) { return hdd{-a.hi, -a.lo}; }
__device__ __forceinline__ hdd hdd_mul_i(hdd a, int c) {   // a * c, c an exact small integer
  const double p = a.hi * (double)c;
  const double err = fma(a.hi, (double)c, -p) + a.lo * (double)c;
  const double h = p + err;
  return hdd{h, err - (h - p)};
}
// P[0..N] (P[0] = 0) into Ph / Pl; returns T_N = sum_t t w_t, both in double-double.  Blocks of
// 1024 bins, lane l owning the 32 consecutive bins b0 + 32 l + i: a lane sums its bins (TwoSum
// into hi, the errors into lo), one warp scan of the lane totals gives each lane its start, and a
// second pass over the same bins (L1 hits) writes the running sums -- 32 independent chains per
// warp instead of a dependent 5-step double-double scan per 32 bins.
__device__ __forceinline__ void two_sum_acc(double& hi, double& lo, double x) {
  const double s = hi + x, bb = s - hi;
  lo += (hi - (s - bb)) + (x - bb);
  hi = s;
}
__device__ __forceinline__ hdd f64_prefix_dd(const double* __restrict__ we, int N, double* Ph,
                                             double* Pl) {
  const int lane = lane_id();
  hdd carry{0.0, 0.0};
  double thi = 0.0, tlo = 0.0;
  for (int b0 = 0; b0 <= N; b0 += 1024) {
    const int t0 = b0 + 32 * lane;
    double shi = 0.0, slo = 0.0;
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
      const int t = t0 + i;
      const double w = (t >= 1 && t <= N) ? we[t] : 0.0;
      two_sum_acc(shi, slo, w);
      const double pr = (double)t * w;
      two_sum_acc(thi, tlo, pr);
      tlo += fma((double)t, w, -pr);
    }
    const hdd tot{shi, slo};
    hdd inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const hdd y = hdd_shfl_up(inc, o);
      if (lane >= o) inc = hdd_add(inc, y);
    }
    const hdd start = hdd_add(carry, hdd_add(inc, hdd{-tot.hi, -tot.lo}));   // exclusive
    double rhi = start.hi, rlo = start.lo;
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
      const int t = t0 + i;
      if (t > N) break;
      const double w = t >= 1 ? we[t] : 0.0;
      two_sum_acc(rhi, rlo, w);
      Ph[t] = rhi;
      Pl[t] = rlo;
    }
    carry = hdd_add(carry, hdd_shfl(inc, 31));
  }
  return hdd_warp_sum(hdd{thi, tlo});
}
__device__ __forceinline__ hdd f64_dP(const double* Ph, const double* Pl, int a, int b) {
  return hdd_add(hdd{Ph[b], Pl[b]}, hdd{-Ph[a], -Pl[a]});   // P(b) - P(a), 0 <= a <= b <= N
}
// one placement (k ascending positions), warp-cooperative over its gaps
__device__ __forceinline__ double f64_cost_warp(const int32_t* pos, int k, int N, hdd TN,
                                                const double* Ph, const double* Pl) {
  hdd acc{0.0, 0.0};
  for (int i = lane_id(); i < k; i += 32) {
    const int ci = pos[i], cn = i + 1 < k ? pos[i + 1] : N + 1;
    acc = hdd_add(acc, hdd_mul_i(f64_dP(Ph, Pl, ci - 1, cn - 1), ci));
  }
  acc = hdd_warp_sum(acc);
  const hdd c = hdd_add(TN, hdd_neg(acc));
  return c.hi + c.lo;
}
// V_1..V_M: the canonical placement of every budget m (the frontier backtrack from the argmin
// logs), one budget per lane; each gap's term needs two prefix lookups
template <int K>
__device__ __forceinline__ void hull_cbb_f64(const HullParams& p, int e, int tfirst, hdd TN,
                                             const double* Ph, const double* Pl,
                                             const uint32_t* logs, const int32_t* logn) {
  const int lane = lane_id();
  const int N = p.N, M = p.M;
  double* cbb = reinterpret_cast<double*>(p.cbb) + (int64_t)e * (M + 1);
  for (int mb = lane + 1; mb <= M; mb += 32) {
    hdd acc{0.0, 0.0};
    int j = N, m = mb, cn = N + 1;
    while (m > 0 && j >= tfirst) {   // positions from the largest down: gap [s, cn)
      const int ls = hull_layer_slot(K, m);
      const int s = log_lookup_lane(logs + (size_t)ls * hull_log_cap(N), logn[ls], j);
      acc = hdd_add(acc, hdd_mul_i(f64_dP(Ph, Pl, s - 1, cn - 1), s));
      cn = s;
      j = s - 1;
      --m;
    }
    const hdd c = hdd_add(TN, hdd_neg(acc));
    cbb[mb] = c.hi + c.lo;
  }
}

// VT = int: every entry first; those beyond the int32 guard but within the int64 one are listed
// for the VT = long long instantiation (launched next, same slots); the rest for the D&C kernel.
#ifndef SP_HULL_MINB
#define SP_HULL_MINB 1
#endif
// one layer per lane (M <= 32, K = 1) on int32 rows: cap the registers at 128 so that 16 warps
// fit an SM (the ring allows 18); the other instantiations are shared-memory bound
#ifndef SP_HULL_BIG_MINB
#define SP_HULL_BIG_MINB 1
#endif
// int64 / fp64 instantiations: capped at 168 registers (no spills) so that an SM sub-partition
// holds 3 of their warps, not 2 (202 / 192 registers: 8 warps per SM; now 9, the shared-memory
// bound): accumulated rows 226 -> 210 ms, fp64 W5 rows 68.3 -> 62.0 ms (profiles/r02e_dp_variants.txt)
#ifdef SP_HULL_BIG_ONEPASS
constexpr bool BIG_ONEPASS = true;
#else
constexpr bool BIG_ONEPASS = false;
#endif
#ifndef SP_HULL_WIDE_MINB
#define SP_HULL_WIDE_MINB 12
#endif
#ifndef SP_HULL_F64_MINB
#define SP_HULL_F64_MINB 12
#endif
template <typename WT, int K, typename VT, bool BIG = false>
__global__ void __launch_bounds__(32, BIG ? (K == 1 ? 16 : SP_HULL_BIG_MINB)
                                      : std::is_same<VT, long long>::value ? SP_HULL_WIDE_MINB
                                      : std::is_same<VT, double>::value ? SP_HULL_F64_MINB
                                      : (K == 1 && sizeof(VT) == 4) ? 16 : SP_HULL_MINB)
    dp_hull_kernel(HullParams p) {
  constexpr bool F64 = std::is_same<VT, double>::value;
  constexpr bool WIDE = std::is_same<VT, long long>::value;
  static_assert(!BIG || std::is_same<VT, int>::value, "the large-hull mode is an int32 mode");
  const int lane = threadIdx.x;
  extern __shared__ __align__(16) uint8_t sring[];   // ring_bytes<K, VT>() | row stage
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sring);
  VT* stage = reinterpret_cast<VT*>(sring + ring_bytes<K, VT>());
  using SR = typename std::conditional<std::is_same<VT, int>::value,
                                       WRing<int, SRingI<HC0, HC1>, BIG>,
                                       WRing<VT, SRingW<VT, WC, WC>>>::type;
  SR srg;
  if constexpr (sizeof(VT) == 8) {
    srg.sm.b0 = sbase + 8u * (uint32_t)lane;
    srg.sm.ds = WROW == 320 ? 256u - 6u * (uint32_t)lane : 256u - 4u * (uint32_t)lane;
  } else {
    srg.sm.b0 = sbase + 4u * (uint32_t)lane;
    srg.sm.ds = 128u - 2u * (uint32_t)lane;
  }
  const int N = p.N, M = p.M;
  sp_dp_stats* stats = reinterpret_cast<sp_dp_stats*>(p.ws);
  unsigned* fb_n = reinterpret_cast<unsigned*>(p.ws + SP_WS_FB_COUNT_OFF);
  unsigned* wide_n = reinterpret_cast<unsigned*>(p.ws + SP_WS_WIDE_COUNT_OFF);
  unsigned* big_n = reinterpret_cast<unsigned*>(p.ws + SP_WS_BIG_COUNT_OFF);
  unsigned* ectr = reinterpret_cast<unsigned*>(
      p.ws + (WIDE ? SP_WS_WIDE_CTR_OFF : BIG ? SP_WS_BIG_CTR_OFF : SP_WS_ENTRY_CTR_OFF));
  // Lists: the int32 kernel hands what it cannot solve to the int64 list (p.wide from the front);
  // when the large-hull mode runs (p.fwd) it takes that list and forwards the entries beyond its
  // own guard to the int64 instantiation through a list of its own (p.fwd_list; its count at
  // SP_WS_BIG_COUNT_OFF).  (Round 2 first wrote it into the back of the int64 list's array: with
  // every entry listed -- accumulated rows -- the two overlapped; tests/test_gpu_hull.py
  // test_hull_int64_list_handoff_all_entries.)
  // (The int32 kernel's hot loop is sensitive to any code around it -- routing there cost 2% on
  // W5 -- so the hand-offs live in the other two instantiations.)
  const bool from_fwd = WIDE && p.fwd;
  const int n_items = (WIDE && !from_fwd) || BIG ? (int)*reinterpret_cast<volatile unsigned*>(wide_n)
                      : from_fwd ? (int)*reinterpret_cast<volatile unsigned*>(big_n) : p.E;
  uint8_t* slot = p.slots + (size_t)blockIdx.x * p.slot;
  uint32_t* logs = reinterpret_cast<uint32_t*>(slot);
  int32_t* logn = reinterpret_cast<int32_t*>(slot + hull_log_bytes(N, M));
  VT* ebuf0 = reinterpret_cast<VT*>(slot + hull_log_bytes(N, M) + hull_cnt_bytes(M));
  VT* ebuf1 = ebuf0 + hull_align(8 * (size_t)(N + 1)) / sizeof(VT);
  unsigned long long pops = 0, events = 0;
  int done_entries = 0;
#ifdef SP_HULL_TAIL   // instrumentation (tools/prof_dp.py, SP_TAIL_REPORT): warp busy vs span
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif

  for (;;) {
    int it = 0;
    if (lane == 0) it = (int)atomicAdd(ectr, 1u);
    it = __shfl_sync(FULL, it, 0);
    if (it >= n_items) break;
    const int e = from_fwd ? p.fwd_list[it] : (WIDE || BIG) ? p.wide[it]
                                                  : (p.order ? p.order[it] : it);
    const WT* we = reinterpret_cast<const WT*>(p.w) + (int64_t)e * (N + 1);

    // ---- a3 pre-pass: n = P_N, T_N, first non-zero bin, sign / size guards ---------------
    using CT = HullCT<VT>;
    CT TN;
    VT nV;
    int tfirst = INT_MAX;
    int kcomp = -1;                 // support rows of a compacted sparse row, else -1
    const int2* klist = nullptr;
    if constexpr (F64) {
      hdd nd{0.0, 0.0}, td{0.0, 0.0};
      int bad = 0;
#pragma unroll 8
      for (int t = lane + 1; t <= N; t += 32) {
        const double c = (double)we[t];
        bad |= !(c >= 0.0) || isinf(c);
        nd = hdd_add(nd, hdd{c, 0.0});
        td = hdd_add(td, hdd_prod((double)t, c));
        if (c > 0.0 && t < tfirst) tfirst = t;
      }
      bad = __any_sync(FULL, bad);
      nd = hdd_warp_sum(nd);
      td = hdd_warp_sum(td);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tfirst = min(tfirst, __shfl_xor_sync(FULL, tfirst, o));
      if (bad) {   // negative / non-finite weights: the D&C kernel reports the entry
        if (lane == 0) p.fb[atomicAdd(fb_n, 1u)] = e;
        continue;
      }
      TN = td.hi + td.lo;
      nV = nd.hi + nd.lo;
    } else {
      long long n = 0, tn = 0;
      int bad = 0;
      if (p.rstat) {   // from row_stats_kernel: the DP reads the row once
        const HullRowStat rs = p.rstat[e];
        n = rs.n;
        tn = rs.tn;
        tfirst = rs.tfirst;
        bad = rs.bad;
        if (p.sparse && rs.K <= HULL_KC) {   // a sparse row: walk its compacted support list
          kcomp = rs.K;
          klist = p.sparse + (size_t)e * HULL_KC;
        }
      } else {
#pragma unroll 8
        for (int t = lane + 1; t <= N; t += 32) {
          const long long c = (long long)we[t];
          bad |= (c < 0) | (c >= (1ll << 40));
          if (!bad) {
            n += c;
            tn += (long long)t * c;
          }
          if (c > 0 && t < tfirst) tfirst = t;
        }
        bad = __any_sync(FULL, bad);
        n = warp_sum(n);
        tn = warp_sum(tn);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tfirst = min(tfirst, __shfl_xor_sync(FULL, tfirst, o));
      }
      // int32 path: 2 n N < 2^31 (the D&C kernel's "narrow" condition); int64 path: n N < 2^46
      // (differences < 2^46, cross products < 2^62); otherwise (or negative counts) the D&C
      // kernel.  The large-hull mode takes n N + T_N < 2^31: every intercept
      // b_s = e_{m-1}(s-1) + s P_{s-1} and every value lies in [-T_N, n N] and every difference
      // and query value within n N + T_N of 0, so all are exact in int32 (e.g. all-ones rows at
      // N = 32768: 2^30 + 2^29) -- heavy rows between the two guards go to it directly.
      const bool narrow = !bad && (BIG ? n * (long long)N + tn < (1ll << 31) : n < (1ll << 30) / N);
      const bool wide_ok = !bad && n < (1ll << 46) / N;
      if (!WIDE && !narrow) {
        if (lane == 0) {
          if (BIG && wide_ok) p.fwd_list[atomicAdd(big_n, 1u)] = e;   // forwarded
          else if (wide_ok) p.wide[atomicAdd(wide_n, 1u)] = e;
          else p.fb[atomicAdd(fb_n, 1u)] = e;
        }
        continue;
      }
      TN = tn;
      nV = (VT)n;   // P_N; n N < 2^30 (int) / 2^46 (long long), so n (j - s) fits VT
    }
    if (lane == 0) {
      if (p.cbb) reinterpret_cast<CT*>(p.cbb)[(int64_t)e * (M + 1)] = TN;   // V_0 = T_N
    }

    // ---- a4: all layers in lockstep, one support row per step --------------------------------
    unsigned pops_e = 0, ev_e = 0;
    bool logfull = false;
    const bool fullm = M % (32 * K) == 0;
    bool ovf;
    if constexpr (BIG) {
      // (the mode runs M <= 64 only: always one pass)
      ovf = fullm ? hull_dp_any<WT, VT, K, true, SR, true, BIG_ONEPASS>(
                        p, we, e, TN, nV, srg, logs, logn, ebuf0, ebuf1, pops_e, ev_e, logfull,
                        stage, kcomp, klist)
                  : hull_dp_any<WT, VT, K, false, SR, true, BIG_ONEPASS>(
                        p, we, e, TN, nV, srg, logs, logn, ebuf0, ebuf1, pops_e, ev_e, logfull,
                        stage, kcomp, klist);
    } else if constexpr (std::is_same<VT, int>::value) {
      // int32: plain shared rings first (W5: 16 of 16384 entries outgrow them); an entry whose
      // hull outgrows a ring is re-run at once with the windowed ring (the same window plus
      // global arrays of WSMALL lines)
#ifdef SP_HULL_WIN_FIRST
      auto& rg1 = srg;
#else
      auto& rg1 = srg.sm;
#endif
#ifdef SP_HULL_SKEW
      if (K == 2 && kcomp < 0 && M <= 64)
        ovf = fullm ? hull_dp_skew<WT, true>(p, we, e, TN, srg.sm, logs, logn, pops_e, ev_e, logfull)
                    : hull_dp_skew<WT, false>(p, we, e, TN, srg.sm, logs, logn, pops_e, ev_e,
                                              logfull);
      else
#endif
      // M = 32 K (W5's M = 64): one pass, no chained e-rows and no SPLIT partner at compile time
      // -- the per-row chain checks and the predicated e-row store vanish (W5 28.95 -> 27.69 ms,
      // profiles/r02e_dp_variants.txt)
#ifndef SP_HULL_NO_ONEPASS
      if (M == 32 * K)
        ovf = hull_dp_any<WT, VT, K, true, std::remove_reference_t<decltype(rg1)>, false, true>(
            p, we, e, TN, nV, rg1, logs, logn, ebuf0, ebuf1, pops_e, ev_e, logfull, stage, kcomp,
            klist);
      else
      // M < 32 K: one pass as well, some slots inactive (W2 DP 54.1 -> 51.9 us, W3 80.8 -> 79.9 us)
      if (M < 32 * K)
        ovf = hull_dp_any<WT, VT, K, false, std::remove_reference_t<decltype(rg1)>, false, true>(
            p, we, e, TN, nV, rg1, logs, logn, ebuf0, ebuf1, pops_e, ev_e, logfull, stage, kcomp,
            klist);
      else
#endif
      ovf = fullm ? hull_dp_any<WT, VT, K, true>(p, we, e, TN, nV, rg1, logs, logn, ebuf0, ebuf1,
                                             pops_e, ev_e, logfull, stage, kcomp, klist)
                  : hull_dp_any<WT, VT, K, false>(p, we, e, TN, nV, rg1, logs, logn, ebuf0, ebuf1,
                                              pops_e, ev_e, logfull, stage, kcomp, klist);
      if (ovf && !logfull) {
        pops_e = ev_e = 0;
        __syncwarp();
        ovf = hull_dp_any<WT, VT, K, false>(p, we, e, TN, nV, srg, logs, logn, ebuf0, ebuf1, pops_e,
                                        ev_e, logfull, stage, kcomp, klist);
      }
    } else {
#ifndef SP_HULL_NO_ONEPASS   // (int64: accumulated rows 201.2 -> 198.6 ms; fp64: 58.7 -> 57.3 ms)
      if (M == 32 * K)
        ovf = hull_dp_any<WT, VT, K, true, SR, false, true>(p, we, e, TN, nV, srg, logs, logn,
                                                            ebuf0, ebuf1, pops_e, ev_e, logfull,
                                                            stage, kcomp, klist);
      else
#endif
      ovf = fullm ? hull_dp_any<WT, VT, K, true>(p, we, e, TN, nV, srg, logs, logn, ebuf0, ebuf1,
                                             pops_e, ev_e, logfull, stage, kcomp, klist)
                  : hull_dp_any<WT, VT, K, false>(p, we, e, TN, nV, srg, logs, logn, ebuf0, ebuf1,
                                              pops_e, ev_e, logfull, stage, kcomp, klist);
    }
    pops += pops_e;
    events += ev_e;
    if (ovf) {
      // int32: a shared ring or a log filled -- the int64 instantiation (windowed rings, exact
      // for narrow entries too) re-runs the entry; int64 / fp64: a global array or a log
      // filled -- the D&C kernel
      // (the int64 list is the large-hull mode's input when it runs: it never fills a log)
      if (lane == 0) {
        if (!WIDE && !F64 && !BIG) p.wide[atomicAdd(wide_n, 1u)] = e;
        else p.fb[atomicAdd(fb_n, 1u)] = e;
      }
      continue;
    }
    __threadfence_block();
    __syncwarp();

    // ---- a5: rule-B backtrack (reading R3): the warp for budget M, lanes for the frontier --
    {
      int32_t* out = p.pos + (int64_t)e * M;
      uint32_t* slog = reinterpret_cast<uint32_t*>(sring);   // the rings are free now
      const bool in_smem = !BIG && logs_to_smem(logs, logn, M, hull_log_cap(N), slog,
                                                (int)(ring_bytes<K, VT>() / 4));
      int k = 0, j = N, m = M;
      int rk = (int)ev_e;   // BIG: support rows <= j (every support row was stepped)
      while (m > 0 && j >= tfirst) {   // P_j > 0  <=>  j >= first non-zero bin
        const int ls = hull_layer_slot(K, m);
        int s;
        if constexpr (BIG) {
          s = unary_lookup_warp(logs + (size_t)ls * hull_log_cap(N), logn[ls], rk);
          rk -= count_support_warp(we, s, j);   // support rows in (s - 1, j]
        } else {
          s = in_smem ? log_lookup_smem(slog, M, m, j)
                      : log_lookup_warp(logs + (size_t)ls * hull_log_cap(N), logn[ls], j);
        }
        if (lane == 0) out[k] = s;
        ++k;
        j = s - 1;
        --m;
      }
      __syncwarp();
      if (lane == 0) {
        for (int a = 0, z = k - 1; a < z; ++a, --z) {
          const int t = out[a];
          out[a] = out[z];
          out[z] = t;
        }
        p.npos[e] = k;
      }
      for (int q = k + lane; q < M; q += 32) out[q] = 0;
      if constexpr (F64) {
        // a7: report the definitional cost sum_t w_t (t - l(t)) of the returned placement in
        // double-double (reading R10; the DP's own V_M carries ~M N eps P_N absolute rounding),
        // from the row's double-double prefix sums (e-row buffers: free after the DP)
        __syncwarp();
        double* Ph = reinterpret_cast<double*>(ebuf0);
        double* Pl = reinterpret_cast<double*>(ebuf1);
        const hdd TNd = f64_prefix_dd(reinterpret_cast<const double*>(we), N, Ph, Pl);
        __syncwarp();
        if (p.cbb) {   // V_1..V_M; the returned placement is budget M's canonical one
          hull_cbb_f64<K>(p, e, tfirst, TNd, Ph, Pl, logs, logn);
          __syncwarp();
          if (lane == 0)
            reinterpret_cast<double*>(p.cost)[e] = reinterpret_cast<double*>(p.cbb)[(int64_t)e * (M + 1) + M];
        } else {
          const double c = f64_cost_warp(out, k, N, TNd, Ph, Pl);
          if (lane == 0) reinterpret_cast<double*>(p.cost)[e] = c;
        }
      }
    }
    if (p.fpos) {
      for (int mb = lane + 1; mb <= M; mb += 32) {
        int32_t* fo = p.fpos + ((int64_t)e * M + (mb - 1)) * M;
        int k = 0, j = N, m = mb;
        while (m > 0 && j >= tfirst) {
          const int ls = hull_layer_slot(K, m);
          const int s = log_lookup_lane(logs + (size_t)ls * hull_log_cap(N), logn[ls], j);
          fo[k++] = s;
          j = s - 1;
          --m;
        }
        for (int a = 0, z = k - 1; a < z; ++a, --z) {
          const int t = fo[a];
          fo[a] = fo[z];
          fo[z] = t;
        }
        for (int q = k; q < M; ++q) fo[q] = 0;
        p.fn[(int64_t)e * M + mb - 1] = k;
      }
    }
    ++done_entries;
    __syncwarp();   // the slot is rewritten by the next entry
  }
  pops = warp_sum(pops);
  if (lane == 0 && done_entries) {   // (an empty list's launch: no atomics at all)
    atomicAdd(&stats->hull_pops, pops);
    atomicAdd(&stats->entries_hull, (unsigned long long)done_entries);
    atomicAdd(F64 ? &stats->entries_f64 : WIDE ? &stats->entries_i64 : &stats->entries_i32,
              (unsigned long long)done_entries);
    atomicAdd(&stats->hull_event_rows, events);
    if (BIG) atomicAdd(&stats->entries_hull_big, (unsigned long long)done_entries);
  }
#ifdef SP_HULL_TAIL
  if (!WIDE && lane == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    unsigned long long* tw = reinterpret_cast<unsigned long long*>(p.ws + 88);
    atomicMax(tw + 0, t_end);              // last warp's end
    atomicMax(tw + 1, ~t_start);           // first warp's start (max of the complement)
    atomicAdd(tw + 2, t_end - t_start);    // summed warp busy time
    atomicAdd(tw + 3, 1ull);               // warps
  }
#endif
}

// ---------------------------------------------------------------------------------------------
// The lean int32 step (dp_lean_kernel): the same CHT, the same lockstep layers and the same
// outputs as dp_hull_kernel<.., int>, with a step cut to what the pop statistics need
// (tools/hull_stats.c on W5 rows: per (row, layer) 40% of pushes pop nothing from the back, 39%
// one line, 15% two; 91% pop nothing from the front, 8% one).
//  * The back line, the one below it, the front line and the one after it live in registers;
//    the only eager shared load per row is the line two below the back (for a second back test).
//  * Back test = one 64-bit sign test: with the new point as origin, line B goes iff
//    Ab' Bs' - As' Bb' >= 0 (two IMAD.WIDE, the second accumulating; one ISETP on the high word).
//  * The front block runs only when some lane pops its front line; the argmin log is appended
//    there (opt_m changes exactly when the front line changes).
//  * The row's (j, P_j) come from a per-chunk compacted list in shared memory (one broadcast load
//    per row); P_{j-1} is the previous support row's P (zero rows do not change P).
//  * n, T_N, the first non-zero bin and the guards come from row_stats_kernel (one read of every
//    row, shared with the largest-first ordering), so the DP reads each histogram row once.
// Entries whose deque outgrows a ring or whose argmin log fills are listed for the int64
// instantiation of dp_hull_kernel (larger rings, then the global ring, then the D&C), which is
// exact for them too.

// 8-byte lines (intercept b, s) in 256-byte position rows, [slot][position][lane]: one LDS.64 /
// STS.64 per line, every lane in its own banks whatever its position.  Positions are kept
// pre-multiplied by 256 so that an address is (p8 & mask) + the lane's base.
template <int C0, int C1>
struct LRing {
  uint32_t lb;   // shared address of slot 0, row 0, this lane's line
  static constexpr int cap(int k) { return k ? C1 : C0; }
  static constexpr uint32_t off(int k) { return k ? (uint32_t)C0 * 256u : 0u; }
  __device__ __forceinline__ uint32_t at(int k, int p8) const {
    return ((uint32_t)p8 & (uint32_t)((cap(k) - 1) << 8)) + lb + off(k);
  }
  __device__ __forceinline__ void ld(int k, int p8, int& b, int& sv) const {
    asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(b), "=r"(sv) : "r"(at(k, p8)));
  }
  __device__ __forceinline__ void st(int k, int p8, int b, int sv) const {
    asm volatile("st.shared.v2.s32 [%0], {%1, %2};" ::"r"(at(k, p8)), "r"(b), "r"(sv) : "memory");
  }
  static constexpr size_t bytes(int K) { return (size_t)(C0 + (K == 2 ? C1 : 0)) * 256; }
  static constexpr int UNIT = 256;
  __device__ __forceinline__ void ld2(int k, int p8, int& b, int& sv) const { ld(k, p8, b, sv); }
  __device__ __forceinline__ void st2(int k, int p8, int b, int sv) const { st(k, p8, b, sv); }
};

__device__ __forceinline__ bool hi_nonneg(long long w) { return (int)(w >> 32) >= 0; }

template <int K, bool ALLACT, bool CHAIN, typename WT, class RG>
__device__ __forceinline__ bool lean_dp(const HullParams& p, const WT* __restrict__ we, int e,
                                        long long TN, const RG rg, uint32_t* logs,
                                        int32_t* logn, int* ebuf0, int* ebuf1, int2* sev,
                                        unsigned& pops_e, unsigned& ev_e, bool& logfull) {
  const int lane = lane_id();
  const int N = p.N, M = p.M;
  const int LC = p.logcap;
  constexpr int L = 32 * K;
  constexpr int U = RG::UNIT;   // position unit (x256 for LRing's pre-shifted counters)
  const int passes = (M + L - 1) / L;
  const unsigned lt_mask = (1u << lane) - 1u;
  bool ovf = false;
  logfull = false;
  for (int ps = 0; ps < passes && !ovf; ++ps) {
    const int* ein = (ps & 1) ? ebuf1 : ebuf0;
    int* eout_buf = (ps & 1) ? ebuf0 : ebuf1;
    const bool chain_out = ps + 1 < passes;
    // per slot: deque positions fr8 <= bk8 (in units U); the back line is always the previous
    // row's line (B0b, s = jp); every other line is read from the ring when needed
    int fr8[K], bk8[K], cnt[K], eo[K], B0b[K];
    bool act[K];
    uint32_t* lg[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int mk = ps * L + 32 * k + lane + 1;
      act[k] = ALLACT || mk <= M;
      fr8[k] = 0;
      bk8[k] = 0;
      eo[k] = 0;    // e_m(0) = 0 (reading R1)
      cnt[k] = 1;   // log entry 0: opt_m(1) = 1 whatever the row type
      lg[k] = logs + (size_t)(ps * L + 32 * k + lane) * LC;
      if (act[k]) lg[k][0] = (1u << 16) | 1u;
      // dummy front line (+inf at every query, s = 0), popped by the first row's front test
      B0b[k] = INT_MAX;
      rg.st2(k, 0, INT_MAX, 0);
    }
    int carry = 0, Pm1 = 0, jp = 0, evbase = 0;
    // the counts are prefetched four chunks ahead (a chunk holds only ~5 support rows on W5)
    int cq[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) cq[c] = 32 * c + 1 + lane <= N ? (int)__ldcs(we + 32 * c + 1 + lane) : 0;
    const uint32_t sev_a = (uint32_t)__cvta_generic_to_shared(sev);
    for (int jb = 0; jb < N; jb += 32) {
      const int jr = jb + 1 + lane;
      const int craw = cq[0];
      cq[0] = cq[1];
      cq[1] = cq[2];
      cq[2] = cq[3];
      cq[3] = jr + 128 <= N ? (int)__ldcs(we + jr + 128) : 0;
      const unsigned evmask = __ballot_sync(FULL, craw > 0);
      if (evmask == 0) continue;
      int Pc = craw;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, Pc, o);
        if (lane >= o) Pc += y;
      }
      Pc += carry;
      carry = __shfl_sync(FULL, Pc, 31);
      if (craw > 0)
        asm volatile("st.shared.v2.s32 [%0], {%1, %2};" ::"r"(sev_a + 8u * __popc(evmask & lt_mask)),
                     "r"(jr), "r"(Pc) : "memory");
      const int nev = __popc(evmask);
      int Ec = 0;
      if (CHAIN && ps > 0 && lane < nev) Ec = evbase + lane >= 1 ? ein[evbase + lane - 1] : 0;
      __syncwarp();
      for (int q = 0; q < nev; ++q) {
        int j, x;
        asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(j), "=r"(x) : "r"(sev_a + 8u * q));
        // ---- ring lines next to both ends (positions known from the previous row) ------------
        int B1b[K], B1s[K], B2b[K], B2s[K], F0b[K], F0s[K], F1b[K], F1s[K], Gb[K], Gs[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          rg.ld2(k, bk8[k] - U, B1b[k], B1s[k]);
          rg.ld2(k, bk8[k] - 2 * U, B2b[k], B2s[k]);
          rg.ld2(k, fr8[k], F0b[k], F0s[k]);
          rg.ld2(k, fr8[k] + U, F1b[k], F1s[k]);
          rg.ld2(k, fr8[k] + 2 * U, Gb[k], Gs[k]);
        }
        // e_{m-1}(j-1) from the lane below (its value at the previous support row)
        int in[K];
        const int t0 = __shfl_sync(FULL, eo[0], (lane + 31) & 31);
        if constexpr (CHAIN) {
          const int ext = __shfl_sync(FULL, Ec, q);
          in[0] = lane ? t0 : ext;
        } else {
          in[0] = lane ? t0 : 0;
        }
        if constexpr (K == 2) {
          const int t1 = __shfl_sync(FULL, eo[1], (lane + 31) & 31);
          in[1] = lane ? t1 : t0;
        }
        ++ev_e;
        const int d0s = jp - j;   // (back line - new line).s, the same for every lane and slot
        // ---- back: two pop tests, with the new point (j, nb) as origin: line B goes iff
        //      (A - N).b (B - N).s - (A - N).s (B - N).b >= 0 for its predecessor A
        int nb[K], top8[K];
        bool p1[K], p2[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          nb[k] = in[k] + j * Pm1;
          const int sz8 = bk8[k] - fr8[k];
          const int d0b = B0b[k] - nb[k];
          const int n1s = j - B1s[k], d1b = B1b[k] - nb[k];
          p1[k] = act[k] & (sz8 >= U) & hi_nonneg((long long)d1b * d0s + (long long)n1s * d0b);
          const int d2b = B2b[k] - nb[k], d1s = B1s[k] - j, n2s = j - B2s[k];
          p2[k] = p1[k] & (sz8 >= 2 * U) & hi_nonneg((long long)d2b * d1s + (long long)n2s * d1b);
          top8[k] = bk8[k] - 2 * U;
        }
        bool any2 = p2[0];
        if constexpr (K == 2) any2 |= p2[1];
        if (__any_sync(FULL, any2)) {   // a lane popped two lines: keep testing from the ring
#pragma unroll
          for (int k = 0; k < K; ++k) {
            bool more = p2[k];
            int cs = B2s[k] - j, cb = B2b[k] - nb[k];
            while (more && top8[k] - fr8[k] >= U) {
              int lb, ls;
              rg.ld2(k, top8[k] - U, lb, ls);
              more = hi_nonneg((long long)(lb - nb[k]) * cs + (long long)(j - ls) * cb);
              if (more) {
                top8[k] -= U;
                cs = ls - j;
                cb = lb - nb[k];
              }
            }
          }
        }
        int v0[K], Fs[K];
        bool q1[K], q2[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          // push the new line after its predecessor
          bk8[k] = (p2[k] ? top8[k] : (p1[k] ? bk8[k] - U : bk8[k])) + U;
          B0b[k] = nb[k];
          ovf |= act[k] & (bk8[k] - fr8[k] >= RG::cap(k) * U);
          rg.st2(k, bk8[k], nb[k], j);
          // ---- front: up to two pops decided from the loaded lines; the line after the
          //      front (F1) or the one after it (G) is the new line when the back reached it
          const bool e1 = bk8[k] == fr8[k] + U, e2 = bk8[k] == fr8[k] + 2 * U;
          const int f1b = e1 ? nb[k] : F1b[k], f1s = e1 ? j : F1s[k];
          const int gb = e2 ? nb[k] : Gb[k], gs = e2 ? j : Gs[k];
          const int w0 = F0b[k] - F0s[k] * x;
          const int w1 = f1b - f1s * x;
          const int wg = gb - gs * x;
          q1[k] = act[k] & (w1 < w0);
          q2[k] = q1[k] & (bk8[k] - fr8[k] >= 2 * U) & (wg < w1);
          v0[k] = q2[k] ? wg : (q1[k] ? w1 : w0);
          Fs[k] = q2[k] ? gs : f1s;
          fr8[k] += q1[k] ? (q2[k] ? 2 * U : U) : 0;
        }
        bool a2 = q2[0];
        if constexpr (K == 2) a2 |= q2[1];
        while (__any_sync(FULL, a2)) {   // rare: the front moves by three or more
          a2 = false;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (q2[k]) {
              q2[k] = false;
              if (fr8[k] < bk8[k]) {
                int lb, ls;
                rg.ld2(k, fr8[k] + U, lb, ls);
                const int vl = lb - ls * x;
                if (vl < v0[k]) {
                  v0[k] = vl;
                  Fs[k] = ls;
                  fr8[k] += U;
                  q2[k] = true;
                }
              }
            }
            a2 |= q2[k];
          }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (q1[k]) lg[k][cnt[k]++] = ((uint32_t)j << 16) | (uint32_t)Fs[k];   // < LC
          eo[k] = v0[k];
        }
        Pm1 = x;
        jp = j;
        if (chain_out && lane == 31) eout_buf[evbase + q] = eo[K - 1];
      }
      evbase += nev;
      bool full = false;
#pragma unroll
      for (int k = 0; k < K; ++k) full |= (LC <= N) & (cnt[k] > LC - 33);   // 32 rows of headroom
      logfull = __any_sync(FULL, full);
      if (__any_sync(FULL, ovf) || logfull) {
        ovf = true;
        break;
      }
      __syncwarp();   // sev is rewritten by the next chunk
    }
    if (!ovf) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!act[k]) continue;
        pops_e += (unsigned)(evbase - bk8[k] / U) + (unsigned)(fr8[k] / U - 1);
        const int mk = ps * L + 32 * k + lane + 1;
        logn[ps * L + 32 * k + lane] = cnt[k];
        const long long V = TN + (long long)eo[k];   // V_m = T_N + e_m(N)
        if (p.cbb) reinterpret_cast<long long*>(p.cbb)[(int64_t)e * (M + 1) + mk] = V;
        if (mk == M) reinterpret_cast<long long*>(p.cost)[e] = V;
      }
    }
    __syncwarp();
  }
  return ovf;
}

// a5 rule-B backtrack from the argmin-change logs (reading R3): the warp for budget M, one lane
// per budget for the f3 frontier.  Shared by dp_hull_kernel and dp_lean_kernel.
template <int K>
__device__ __forceinline__ void hull_backtrack(const HullParams& p, int e, int tfirst,
                                               const uint32_t* logs, const int32_t* logn,
                                               uint32_t* slog = nullptr, int slog_words = 0) {
  const int lane = lane_id();
  const int N = p.N, M = p.M;
  int32_t* out = p.pos + (int64_t)e * M;
  const bool in_smem = slog && logs_to_smem(logs, logn, M, hull_log_cap(N), slog, slog_words);
  int k = 0, j = N, m = M;
  while (m > 0 && j >= tfirst) {   // P_j > 0  <=>  j >= first non-zero bin
    const int ls = hull_layer_slot(K, m);
    const int s = in_smem ? log_lookup_smem(slog, M, m, j)
                          : log_lookup_warp(logs + (size_t)ls * hull_log_cap(N), logn[ls], j);
    if (lane == 0) out[k] = s;
    ++k;
    j = s - 1;
    --m;
  }
  __syncwarp();
  if (lane == 0) {
    for (int a = 0, z = k - 1; a < z; ++a, --z) {
      const int t = out[a];
      out[a] = out[z];
      out[z] = t;
    }
    p.npos[e] = k;
  }
  for (int q = k + lane; q < M; q += 32) out[q] = 0;
  if (p.fpos) {
    for (int mb = lane + 1; mb <= M; mb += 32) {
      int32_t* fo = p.fpos + ((int64_t)e * M + (mb - 1)) * M;
      int kk = 0, jj = N, mm = mb;
      while (mm > 0 && jj >= tfirst) {
        const int ls = hull_layer_slot(K, mm);
        const int s = log_lookup_lane(logs + (size_t)ls * hull_log_cap(N), logn[ls], jj);
        fo[kk++] = s;
        jj = s - 1;
        --mm;
      }
      for (int a = 0, z = kk - 1; a < z; ++a, --z) {
        const int t = fo[a];
        fo[a] = fo[z];
        fo[z] = t;
      }
      for (int q = kk; q < M; ++q) fo[q] = 0;
      p.fn[(int64_t)e * M + mb - 1] = kk;
    }
  }
}


// SPLIT mode kernel (int32 path, 32 < M <= 64): one entry per 2-warp CTA, warp w running the
// layers of pass w of the K = 1 lockstep DP, chained through a shared-memory ring (SplitSync).
// For batches with few entries per resident warp (a GPU's share at 8-way strong scaling: 2048
// W5 entries on 1776 warps) an entry's time halves, and the largest-first order has twice the
// work items to balance.  Entries that overflow a ring or a log, and entries beyond the int32
// guard, are listed for the large-hull mode / the int64 instantiation (launched after), bad rows
// for the D&C kernel.
template <typename WT>
__global__ void __launch_bounds__(64, 1) dp_hull_split_kernel(HullParams p) {
  const int lane = lane_id(), w = warp_id();
  extern __shared__ __align__(16) uint8_t sring[];
  constexpr size_t RB = (size_t)HC0 * 192;   // one K = 1 ring per warp
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sring) + (uint32_t)(w * RB);
  SRingI<HC0, HC1> srg;
  srg.b0 = sbase + 4u * (uint32_t)lane;
  srg.ds = 128u - 2u * (uint32_t)lane;
  int* ring = reinterpret_cast<int*>(sring + 2 * RB);
  int* stage = reinterpret_cast<int*>(sring + 2 * RB + SPLIT_RING * sizeof(int) + w * stage_bytes<int>());
  __shared__ int s_it, s_prod, s_cons, s_abort;
  SplitSync ss{ring, &s_prod, &s_cons, &s_abort};
  const int N = p.N, M = p.M;
  sp_dp_stats* stats = reinterpret_cast<sp_dp_stats*>(p.ws);
  unsigned* fb_n = reinterpret_cast<unsigned*>(p.ws + SP_WS_FB_COUNT_OFF);
  unsigned* wide_n = reinterpret_cast<unsigned*>(p.ws + SP_WS_WIDE_COUNT_OFF);
  unsigned* ectr = reinterpret_cast<unsigned*>(p.ws + SP_WS_ENTRY_CTR_OFF);
  uint8_t* slot = p.slots + (size_t)blockIdx.x * p.slot;
  uint32_t* logs = reinterpret_cast<uint32_t*>(slot);
  int32_t* logn = reinterpret_cast<int32_t*>(slot + hull_log_bytes(N, M));
  int* ebuf0 = reinterpret_cast<int*>(slot + hull_log_bytes(N, M) + hull_cnt_bytes(M));
  unsigned long long pops = 0, events = 0;
  int done_entries = 0;
  const bool fullm = M == 64;
  for (;;) {
    __syncthreads();   // both warps are done with the previous entry
    if (threadIdx.x == 0) {
      s_it = (int)atomicAdd(ectr, 1u);
      s_prod = 0;
      s_cons = 0;
      s_abort = 0;
    }
    __syncthreads();
    const int it = s_it;
    if (it >= p.E) break;
    const int e = p.order ? p.order[it] : it;
    const HullRowStat rs = p.rstat[e];
    if (rs.bad || rs.n >= (1ll << 30) / N) {   // int32 guard: 2 n N < 2^31
      if (threadIdx.x == 0) {
        if (!rs.bad && rs.n < (1ll << 46) / N) p.wide[atomicAdd(wide_n, 1u)] = e;
        else p.fb[atomicAdd(fb_n, 1u)] = e;
      }
      continue;
    }
    const WT* we = reinterpret_cast<const WT*>(p.w) + (int64_t)e * (N + 1);
    if (threadIdx.x == 0 && p.cbb) reinterpret_cast<long long*>(p.cbb)[(int64_t)e * (M + 1)] = rs.tn;
    const bool sparse_row = p.sparse && rs.K <= HULL_KC;
    const int kcomp = sparse_row ? rs.K : -1;
    const int2* klist = sparse_row ? p.sparse + (size_t)e * HULL_KC : nullptr;
    unsigned pops_e = 0, ev_e = 0;
    bool logfull = false;
#ifndef SP_SPLIT_NO_ROLES
    // each warp's role at compile time (warp 0 chains out, warp 1 chains in): 2048 W5 entries
    // 5.74 -> 5.64 ms (profiles/r02e_dp_variants.txt)
    if (w == 0) {
      if (fullm)
        hull_dp_any<WT, int, 1, true, SRingI<HC0, HC1>, false, false, 1>(
            p, we, e, rs.tn, (int)rs.n, srg, logs, logn, ebuf0, ebuf0, pops_e, ev_e, logfull, stage,
            kcomp, klist, &ss, w);
      else
        hull_dp_any<WT, int, 1, false, SRingI<HC0, HC1>, false, false, 1>(
            p, we, e, rs.tn, (int)rs.n, srg, logs, logn, ebuf0, ebuf0, pops_e, ev_e, logfull, stage,
            kcomp, klist, &ss, w);
    } else {
      if (fullm)
        hull_dp_any<WT, int, 1, true, SRingI<HC0, HC1>, false, false, 2>(
            p, we, e, rs.tn, (int)rs.n, srg, logs, logn, ebuf0, ebuf0, pops_e, ev_e, logfull, stage,
            kcomp, klist, &ss, w);
      else
        hull_dp_any<WT, int, 1, false, SRingI<HC0, HC1>, false, false, 2>(
            p, we, e, rs.tn, (int)rs.n, srg, logs, logn, ebuf0, ebuf0, pops_e, ev_e, logfull, stage,
            kcomp, klist, &ss, w);
    }
#else
    if (fullm)
      hull_dp_any<WT, int, 1, true>(p, we, e, rs.tn, (int)rs.n, srg, logs, logn, ebuf0, ebuf0, pops_e,
                                ev_e, logfull, stage, kcomp, klist, &ss, w);
    else
      hull_dp_any<WT, int, 1, false>(p, we, e, rs.tn, (int)rs.n, srg, logs, logn, ebuf0, ebuf0,
                                 pops_e, ev_e, logfull, stage, kcomp, klist, &ss, w);
#endif
    __syncthreads();
    if (s_abort) {   // ring or log full in either warp: the large-hull mode or the int64
      if (threadIdx.x == 0) p.wide[atomicAdd(wide_n, 1u)] = e;   // instantiation re-runs it
      continue;
    }
    pops += pops_e;
    events += w == 0 ? ev_e : 0;
    if (w == 0) {
      __threadfence_block();
      hull_backtrack<1>(p, e, rs.tfirst, logs, logn, reinterpret_cast<uint32_t*>(sring),
                        (int)(2 * RB / 4));   // both warps' rings are free now
      ++done_entries;
    }
  }
  pops = warp_sum(pops);
  if (lane == 0 && (pops || done_entries)) {
    atomicAdd(&stats->hull_pops, pops);
    if (w == 0) {
      atomicAdd(&stats->entries_hull, (unsigned long long)done_entries);
      atomicAdd(&stats->entries_i32, (unsigned long long)done_entries);
      atomicAdd(&stats->hull_event_rows, events);
    }
  }
}

// the lean kernel's ring: 6-byte lines (SRingI, 12 warps/SM at 64/32 lines) by default;
// -DSP_LEAN_RING8 selects 8-byte lines in 256-byte rows (LRing: one LDS.64 per line, 9 warps/SM)
#ifdef SP_LEAN_RING8
using LeanRing = LRing<HC0, HC1>;
#else
using LeanRing = SRingI<HC0, HC1>;
#endif

template <int K>
static constexpr size_t lean_smem_bytes() {
  return LeanRing::bytes(K) + 32 * sizeof(int2);
}

// One warp per entry (1-warp CTAs, persistent, largest support first).  Entries beyond the int32
// guard (2 n N >= 2^31) are listed for the int64 instantiation of dp_hull_kernel, bad rows
// (negative counts) for the D&C kernel.
template <typename WT, int K>
__global__ void __launch_bounds__(32, 1) dp_lean_kernel(HullParams p, const HullRowStat* rstat) {
  const int lane = threadIdx.x;
  extern __shared__ __align__(16) uint8_t sring[];
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sring);
  LeanRing srg;
#ifdef SP_LEAN_RING8
  srg.lb = sbase + 8u * (uint32_t)lane;
#else
  srg.b0 = sbase + 4u * (uint32_t)lane;
  srg.ds = 128u - 2u * (uint32_t)lane;
#endif
  int2* sev = reinterpret_cast<int2*>(sring + LeanRing::bytes(K));
  const int N = p.N, M = p.M;
  sp_dp_stats* stats = reinterpret_cast<sp_dp_stats*>(p.ws);
  unsigned* fb_n = reinterpret_cast<unsigned*>(p.ws + SP_WS_FB_COUNT_OFF);
  unsigned* wide_n = reinterpret_cast<unsigned*>(p.ws + SP_WS_WIDE_COUNT_OFF);
  unsigned* ectr = reinterpret_cast<unsigned*>(p.ws + SP_WS_ENTRY_CTR_OFF);
  uint8_t* slot = p.slots + (size_t)blockIdx.x * p.slot;
  uint32_t* logs = reinterpret_cast<uint32_t*>(slot);
  int32_t* logn = reinterpret_cast<int32_t*>(slot + hull_log_bytes(N, M));
  int* ebuf0 = reinterpret_cast<int*>(slot + hull_log_bytes(N, M) + hull_cnt_bytes(M));
  int* ebuf1 = ebuf0 + hull_align(8 * (size_t)(N + 1)) / sizeof(int);
  unsigned long long pops = 0, events = 0;
  int done_entries = 0;
  const bool fullm = M % (32 * K) == 0;
  const bool chained = hull_passes(M) > 1;
  for (;;) {
    int it = 0;
    if (lane == 0) it = (int)atomicAdd(ectr, 1u);
    it = __shfl_sync(FULL, it, 0);
    if (it >= p.E) break;
    const int e = p.order ? p.order[it] : it;
    const HullRowStat rs = rstat[e];
    if (rs.bad || rs.n >= (1ll << 30) / N) {   // int32 guard: 2 n N < 2^31
      if (lane == 0) {
        if (!rs.bad && rs.n < (1ll << 46) / N) p.wide[atomicAdd(wide_n, 1u)] = e;
        else p.fb[atomicAdd(fb_n, 1u)] = e;
      }
      continue;
    }
    const WT* we = reinterpret_cast<const WT*>(p.w) + (int64_t)e * (N + 1);
    if (lane == 0 && p.cbb) reinterpret_cast<long long*>(p.cbb)[(int64_t)e * (M + 1)] = rs.tn;
    unsigned pops_e = 0, ev_e = 0;
    bool logfull = false, ovf;
    if (fullm && !chained)
      ovf = lean_dp<K, true, false, WT>(p, we, e, rs.tn, srg, logs, logn, ebuf0, ebuf1, sev, pops_e, ev_e, logfull);
    else if (!chained)
      ovf = lean_dp<K, false, false, WT>(p, we, e, rs.tn, srg, logs, logn, ebuf0, ebuf1, sev, pops_e, ev_e, logfull);
    else
      ovf = lean_dp<K, false, true, WT>(p, we, e, rs.tn, srg, logs, logn, ebuf0, ebuf1, sev, pops_e, ev_e, logfull);
    if (ovf) {   // ring or log full: the int64 instantiation re-runs the entry
      if (lane == 0) p.wide[atomicAdd(wide_n, 1u)] = e;
      continue;
    }
    pops += pops_e;
    events += ev_e;
    __threadfence_block();
    __syncwarp();
    hull_backtrack<K>(p, e, rs.tfirst, logs, logn);
    ++done_entries;
    __syncwarp();   // the slot is rewritten by the next entry
  }
  pops = warp_sum(pops);
  if (lane == 0) {
    atomicAdd(&stats->hull_pops, pops);
    atomicAdd(&stats->entries_hull, (unsigned long long)done_entries);
    atomicAdd(&stats->entries_i32, (unsigned long long)done_entries);
    atomicAdd(&stats->hull_event_rows, events);
  }
}

// One pass over every row (one warp per row): the support count (the largest-first order's key),
// and for integer weights n = P_N, T_N, the first non-zero bin and the guards that dp_lean_kernel
// needs before it starts (so the DP itself reads each row once).
constexpr int RS_U = 32;   // row pre-pass: 32-bin chunks in flight per lane (4 KB per warp)
__device__ __forceinline__ long long mad_wide_s32(int a, int b, long long c) {   // c + a b, exact
  long long d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}
template <typename WT>
__global__ void __launch_bounds__(256) row_stats_kernel(const WT* __restrict__ w, int E, int N,
                                                        int32_t* __restrict__ key,
                                                        int32_t* __restrict__ val,
                                                        HullRowStat* __restrict__ rstat,
                                                        int2* __restrict__ sparse) {
  const int lane = lane_id();
  const int nw = gridDim.x * 8;
  const unsigned lt = (1u << lane) - 1u;
  for (int e = blockIdx.x * 8 + warp_id(); e < E; e += nw) {
    const WT* we = w + (int64_t)e * (N + 1);
    int c = 0, bad = 0, tfirst = INT_MAX;
    long long n = 0, tn = 0;
    int2* sp_e = sparse ? sparse + (size_t)e * HULL_KC : nullptr;
    // RS_U chunks of 32 bins in flight per lane (all loads issued before any is used), then the
    // chunks in order: sums, guards, and the support rows compacted while they fit HULL_KC
    for (int base = 0; base < N; base += 32 * RS_U) {   // (warp-uniform trip count: ballots)
      WT v[RS_U];
#pragma unroll
      for (int u = 0; u < RS_U; ++u) {
        const int t = base + 32 * u + 1 + lane;
        v[u] = t <= N ? __ldcs(we + t) : WT(0);
      }
#pragma unroll
      for (int u = 0; u < RS_U; ++u) {
        const int t = base + 32 * u + 1 + lane;
        const unsigned nz = __ballot_sync(FULL, v[u] != WT(0));
        if constexpr (std::is_same<WT, int32_t>::value) {
          // int32 counts: n and T_N with one mad.wide each; the first non-zero bin from the
          // ballot (warp-uniform), the only guard a negative count
          bad |= v[u] < 0;
          n = mad_wide_s32(v[u], 1, n);
          tn = mad_wide_s32(v[u], t, tn);
          if (nz && tfirst == INT_MAX) tfirst = base + 32 * u + __ffs(nz);
          if (sp_e && c < HULL_KC) {
            const int at = c + __popc(nz & lt);
            if (v[u] != 0 && at < HULL_KC) sp_e[at] = make_int2(t, v[u]);
          }
        } else if constexpr (!std::is_same<WT, double>::value) {
          const long long cv = (long long)v[u];
          bad |= (cv < 0) | (cv >= (1ll << 40));
          n += cv;
          tn += (long long)t * cv;
          if (cv > 0 && t < tfirst) tfirst = t;
          if (sp_e && c < HULL_KC) {
            const int at = c + __popc(nz & lt);
            if (v[u] != WT(0) && at < HULL_KC) sp_e[at] = make_int2(t, (int)cv);
          }
        }
        c += __popc(nz);
      }
    }
    if constexpr (!std::is_same<WT, double>::value) {
      n = warp_sum(n);
      tn = warp_sum(tn);
      bad = __any_sync(FULL, bad);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tfirst = min(tfirst, __shfl_xor_sync(FULL, tfirst, o));
    }
    if (lane == 0) {
      if (key) {
        key[e] = c;
        val[e] = e;
      }
      if (rstat) rstat[e] = HullRowStat{n, tn, tfirst, bad, c, 0};
    }
  }
}

// Host-side launch facts cached per device (the verdict's host-overhead item: no attribute,
// occupancy or getenv calls on every sp_place_checkpoints call once warm).
constexpr int HULL_MAX_DEV = 64;
static int dev_sms() {
  static int sms[HULL_MAX_DEV] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= HULL_MAX_DEV) dev = 0;
  if (!sms[dev]) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = v;
  }
  return sms[dev];
}
// resident 1-warp CTAs per SM for a kernel with `dyn` bytes of dynamic shared memory (sets the
// opt-in attribute once per device)
template <typename KernelT>
static int occ_cached(KernelT kern, size_t dyn, int* cache) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= HULL_MAX_DEV) dev = 0;
  if (!cache[dev]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32, dyn);
    cache[dev] = occ < 1 ? 1 : occ;
  }
  return cache[dev];
}

static int clamp_grid(long g, int E) {
  if (g > E) g = E;
  return (int)(g < 1 ? 1 : g);
}

template <typename WT, int K, typename VT>
static int hull_grid_t(int E) {
  static int cache[HULL_MAX_DEV] = {0};
  const int occ = occ_cached(dp_hull_kernel<WT, K, VT>, hull_dyn_bytes<K, VT>(), cache);
  return clamp_grid((long)dev_sms() * occ, E);
}
// the int32 large-hull mode (same shared memory as the int32 kernel)
#ifndef SP_HULL_BIG_PAD
#define SP_HULL_BIG_PAD 0   // extra dynamic shared memory per warp (occupancy / L1 experiments)
#endif
template <int K>
constexpr size_t big_dyn_bytes() { return hull_dyn_bytes<K, int>() + SP_HULL_BIG_PAD; }
template <typename WT, int K>
static int big_grid_t(int E) {
  static int cache[HULL_MAX_DEV] = {0};
  const int occ = occ_cached(dp_hull_kernel<WT, K, int, true>, big_dyn_bytes<K>(), cache);
  return clamp_grid((long)dev_sms() * occ, E);
}

constexpr size_t split_smem_bytes() {
  return 2 * (size_t)HC0 * 192 + SPLIT_RING * sizeof(int) + 2 * stage_bytes<int>();
}

template <typename WT>
static int split_grid_t(int E) {
  static int cache[HULL_MAX_DEV] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= HULL_MAX_DEV) dev = 0;
  if (!cache[dev]) {
    cudaFuncSetAttribute(dp_hull_split_kernel<WT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)split_smem_bytes());
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dp_hull_split_kernel<WT>, 64,
                                                  split_smem_bytes());
    cache[dev] = occ < 1 ? 1 : occ;
  }
  return clamp_grid((long)dev_sms() * cache[dev], E);
}

// SPLIT mode for the int32 path when 32 < M <= 64 and the batch has fewer than 1.5 entries per
// resident warp of the one-warp kernel (measured on W5 rows, 1776 warps: 2048 entries 7.35 ->
// 5.60 ms; 4096 entries 8.0 -> 10.3 ms, so not there); SP_DBG_HULL_SPLIT = 0 / 1 forces it off
// / on (comparison hook)
static bool use_split(int E, int M, int one_warp_grid) {
  const int force = sp_debug_get(SP_DBG_HULL_SPLIT);
  if (M <= 32 || M > 64) return false;
  if (force >= 0) return force != 0;
  return 2L * E < 3L * one_warp_grid;
}

template <typename WT, int K>
static int lean_grid_t(int E) {
  static int cache[HULL_MAX_DEV] = {0};
  const int occ = occ_cached(dp_lean_kernel<WT, K>, lean_smem_bytes<K>(), cache);
  return clamp_grid((long)dev_sms() * occ, E);
}

// SP_DBG_HULL_LEAN runs the int32 path on dp_lean_kernel instead of dp_hull_kernel<.., int>
// (measured: faster on sparse rows, slower on W5's)
static bool hull_lean() { return sp_debug_get(SP_DBG_HULL_LEAN) != 0; }

template <typename WT, int K>
static void hull_launch_t(HullParams p, const HullRowStat* rstat, int gn, cudaStream_t st) {
  if constexpr (std::is_same<WT, double>::value) {
    p.wgb = wring_pass_bytes_t<double>(p.N, p.M);
    dp_hull_kernel<double, K, double><<<gn, 32, hull_dyn_bytes<K, double>(), st>>>(p);
  } else {
    p.wgb = wring_pass_bytes_t<int>(p.N, p.M);
    if (K == 2 && !hull_lean() && p.rstat &&
        use_split(p.E, p.M, std::min(gn, hull_grid_t<WT, K, int>(p.E)))) {
      const int gs = std::min(gn, split_grid_t<WT>(p.E));
      dp_hull_split_kernel<WT><<<gs, 64, split_smem_bytes(), st>>>(p);
    } else if (!hull_lean()) {
      dp_hull_kernel<WT, K, int><<<gn, 32, hull_dyn_bytes<K, int>(), st>>>(p);
    } else {
      const int gl = std::min(gn, lean_grid_t<WT, K>(p.E));
      dp_lean_kernel<WT, K><<<gl, 32, lean_smem_bytes<K>(), st>>>(p, rstat);
    }
    // the large-hull mode on its listed entries (int32 entries whose hull outgrew the rings or
    // whose change log filled; exits at once when the list is empty): its grid is clamped to the
    // slots and to the regions of big-capacity arrays the pool holds
    p.fwd = 0;
    if (p.M <= 64 && !p.fpos && p.logcap >= (2 * p.N + 31) / 32 + 2) {
      p.wgb = wring_pass_bytes_t<int, true>(p.N, p.M);
      const long regions = (long)(sp_hull_wg_bytes(p.E, p.N, p.M) / p.wgb);
      const int gb = (int)std::min<long>(std::min(gn, big_grid_t<WT, K>(p.E)), regions);
      if (gb >= 1) {
        dp_hull_kernel<WT, K, int, true><<<gb, 32, big_dyn_bytes<K>(), st>>>(p);
        p.fwd = 1;
      }
    }
    // the int64 instantiation on the listed entries (its warps exit at once if the list is
    // empty); its grid is clamped to the slots allocated for the widest launch
    const int gw = std::min(gn, hull_grid_t<WT, K, long long>(p.E));
    p.wgb = wring_pass_bytes_t<long long>(p.N, p.M);
    dp_hull_kernel<WT, K, long long><<<gw, 32, hull_dyn_bytes<K, long long>(), st>>>(p);
  }
}

}  // namespace sp

// slots are allocated for the largest grid any launch of this weight type uses
int sp_hull_grid(int E, int N, int M, int wtype) {
  (void)N;
  const bool k2 = sp::hull_K(M) == 2;
  if (wtype == SP_W_PROB_F64)
    return k2 ? sp::hull_grid_t<double, 2, double>(E) : sp::hull_grid_t<double, 1, double>(E);
  int g;
  if (wtype == SP_W_COUNTS_I64)
    g = k2 ? std::max(std::max(std::max(sp::hull_grid_t<int64_t, 2, int>(E), sp::lean_grid_t<int64_t, 2>(E)),
                               sp::hull_grid_t<int64_t, 2, long long>(E)),
                      sp::split_grid_t<int64_t>(E))
           : std::max(std::max(sp::hull_grid_t<int64_t, 1, int>(E), sp::lean_grid_t<int64_t, 1>(E)),
                      sp::hull_grid_t<int64_t, 1, long long>(E));
  else
    g = k2 ? std::max(std::max(std::max(sp::hull_grid_t<int32_t, 2, int>(E), sp::lean_grid_t<int32_t, 2>(E)),
                               sp::hull_grid_t<int32_t, 2, long long>(E)),
                      sp::split_grid_t<int32_t>(E))
           : std::max(std::max(sp::hull_grid_t<int32_t, 1, int>(E), sp::lean_grid_t<int32_t, 1>(E)),
                      sp::hull_grid_t<int32_t, 1, long long>(E));
  return g;
}

size_t sp_hull_slot_bytes(int N, int M) { return sp::hull_slot_bytes(N, M); }
// the windowed rings' global arrays: one region per CTA, shared by the int32 and the int64 / fp64
// instantiations (they run one after the other on the stream)
size_t sp_hull_wg_bytes(int E, int N, int M) {
  const bool k2 = sp::hull_K(M) == 2;
  const size_t gi = (size_t)(k2 ? sp::hull_grid_t<int32_t, 2, int>(E) : sp::hull_grid_t<int32_t, 1, int>(E)) *
                    sp::wring_pass_bytes_t<int>(N, M);
  int g = k2 ? std::max(sp::hull_grid_t<int32_t, 2, long long>(E), sp::hull_grid_t<double, 2, double>(E))
             : std::max(sp::hull_grid_t<int32_t, 1, long long>(E), sp::hull_grid_t<double, 1, double>(E));
  g = std::max(g, k2 ? sp::hull_grid_t<int64_t, 2, long long>(E) : sp::hull_grid_t<int64_t, 1, long long>(E));
  return std::max(gi, (size_t)g * sp::wring_pass_bytes_t<long long>(N, M));
}

// ordering scratch: key/val in, key/val out (int32 [E] each) | cub temp | row stats [E]
static size_t order_cub_bytes(int E) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr,
                                            (const int32_t*)nullptr, (int32_t*)nullptr, E);
  return b;
}
size_t sp_hull_order_bytes(int E) {
  return 4 * sp::hull_align(4 * (size_t)E) + sp::hull_align(order_cub_bytes(E)) +
         sp::hull_align(sizeof(sp::HullRowStat) * (size_t)E) +
         sp::hull_align(sizeof(int2) * sp::HULL_KC * (size_t)E);
}

cudaError_t sp_hull_launch(const void* weights, int wtype, int E, int N, int M, int32_t* pos,
                           int32_t* npos, void* cost, void* cbb, int32_t* fpos,
                           int32_t* fn, uint8_t* ws, int32_t* fb, int32_t* wide,
                           int32_t* fwd_list, uint8_t* pool, uint8_t* order_ws, uint8_t* slots,
                           int grid, cudaStream_t st) {
  const bool no_order = sp_debug_get(SP_DBG_HULL_NO_ORDER) != 0;   // comparison hook
  const int logcap_env = sp_debug_get(SP_DBG_HULL_LOGCAP);   // test hook: force the log-full fallback
  sp::HullParams p;
  p.order = nullptr;
  p.fwd = 0;
  p.fwd_list = fwd_list;
  const size_t a = sp::hull_align(4 * (size_t)E);
  int32_t* kin = (int32_t*)order_ws;
  int32_t* vin = (int32_t*)(order_ws + a);
  int32_t* kout = (int32_t*)(order_ws + 2 * a);
  int32_t* vout = (int32_t*)(order_ws + 3 * a);
  const size_t tb = order_cub_bytes(E);
  sp::HullRowStat* rstat =
      reinterpret_cast<sp::HullRowStat*>(order_ws + 4 * a + sp::hull_align(tb));
  int2* sparse = reinterpret_cast<int2*>(order_ws + 4 * a + sp::hull_align(tb) +
                                         sp::hull_align(sizeof(sp::HullRowStat) * (size_t)E));
  // the largest-first order matters only when warps take several entries each: with no more
  // entries than resident warps of the one-warp kernel every entry starts in the first wave
  const bool k2o = sp::hull_K(M) == 2;
  const long first_wave =
      wtype == SP_W_PROB_F64
          ? (k2o ? sp::hull_grid_t<double, 2, double>(1 << 30) : sp::hull_grid_t<double, 1, double>(1 << 30))
          : (k2o ? sp::hull_grid_t<int32_t, 2, int>(1 << 30) : sp::hull_grid_t<int32_t, 1, int>(1 << 30));
  const bool order = E > 1 && E > first_wave && !no_order;
  int blocks = (E + 7) / 8;
  if (blocks > sp::dev_sms() * 8) blocks = sp::dev_sms() * 8;
  if (wtype == SP_W_PROB_F64) {
    if (order)
      sp::row_stats_kernel<double><<<blocks, 256, 0, st>>>((const double*)weights, E, N, kin, vin,
                                                           nullptr, nullptr);
  } else if (wtype == SP_W_COUNTS_I64) {
    sp::row_stats_kernel<int64_t><<<blocks, 256, 0, st>>>((const int64_t*)weights, E, N,
                                                          order ? kin : nullptr, vin, rstat, sparse);
  } else {
    sp::row_stats_kernel<int32_t><<<blocks, 256, 0, st>>>((const int32_t*)weights, E, N,
                                                          order ? kin : nullptr, vin, rstat, sparse);
  }
  if (order) {
    size_t tbv = tb;
    if (cub::DeviceRadixSort::SortPairsDescending(order_ws + 4 * a, tbv, kin, kout, vin, vout, E, 0,
                                                  32, st) == cudaSuccess)
      p.order = vout;
  }
  p.rstat = wtype == SP_W_PROB_F64 ? nullptr : rstat;
  p.sparse = wtype == SP_W_PROB_F64 ? nullptr : sparse;
  p.wg = pool;
  p.wgb = 0;   // per instantiation, set by hull_launch_t
  p.wide = wide;
  p.w = weights;
  p.E = E;
  p.N = N;
  p.M = M;
  p.pos = pos;
  p.npos = npos;
  p.cost = cost;
  p.cbb = cbb;
  p.fpos = fpos;
  p.fn = fn;
  p.ws = ws;
  p.fb = fb;
  p.slots = slots;
  p.slot = sp::hull_slot_bytes(N, M);
  p.logcap = sp::hull_log_cap(N);
  if (logcap_env >= 1 && logcap_env < p.logcap) p.logcap = logcap_env;
  const bool k2 = sp::hull_K(M) == 2;
  if (wtype == SP_W_PROB_F64) {
    if (k2) sp::hull_launch_t<double, 2>(p, rstat, grid, st);
    else sp::hull_launch_t<double, 1>(p, rstat, grid, st);
  } else if (wtype == SP_W_COUNTS_I64) {
    if (k2) sp::hull_launch_t<int64_t, 2>(p, rstat, grid, st);
    else sp::hull_launch_t<int64_t, 1>(p, rstat, grid, st);
  } else {
    if (k2) sp::hull_launch_t<int32_t, 2>(p, rstat, grid, st);
    else sp::hull_launch_t<int32_t, 1>(p, rstat, grid, st);
  }
  return cudaGetLastError();
}
