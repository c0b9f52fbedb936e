// expected_recompute.cu -- a6: expected recomputation and worst case of given placements
// (baseline evaluation: balanced / block schedules of Table 1; objective P:171-173).
//
// For C = {c_1 < ... < c_k}, c_0 = 0, c_{k+1} = N+1, segment i holds depths [c_i, c_{i+1}-1]
// whose reusable depth is c_i, so
//     cost = sum_i sum_{t in seg i} c_t (t - c_i) = T_N - sum_{i=1}^k c_i (P(c_{i+1}-1) - P(c_i-1))
// (the w(s,j) decomposition of P:758 summed over the segments), and
//     worst = max_i (c_{i+1} - c_i) - 1.
// Three kernels, all reading each histogram row once:
//   eval_bcast_kernel   int32 counts, <= 4 placement sets shared by every entry (the Table 1
//                       baselines; the bench's path): per-CTA tables l(t; C) in shared memory,
//                       then a balanced streaming pass over (entry, slice) items.
//   eval_p32_kernel     other int32 cases: the row's prefix sums in shared memory, one warp per
//                       placement.
//   eval_kernel         int64 / fp64 weights: 32-bin chunk prefix sums (double-double for fp64).
// Count types are exact in int64.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include <atomic>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"

namespace sp {

constexpr int EV_NT = 256;
constexpr int EV_NW = EV_NT / 32;
constexpr int EV_MAXCH = 2049;   // (SP_MAX_N + 1) / 32 + 1

struct ddv {
  double hi, lo;
};
__device__ __forceinline__ ddv add(ddv a, ddv b) {
  double s = a.hi + b.hi;
  double bb = s - a.hi;
  double err = (a.hi - (s - bb)) + (b.hi - bb) + a.lo + b.lo;
  double h = s + err;
  return ddv{h, err - (h - s)};
}
__device__ __forceinline__ ddv neg(ddv a) { return ddv{-a.hi, -a.lo}; }
__device__ __forceinline__ ddv mul_int(ddv a, int c) {
  double p = a.hi * c;
  double e = fma(a.hi, (double)c, -p) + a.lo * c;
  double h = p + e;
  return ddv{h, e - (h - p)};
}
__device__ __forceinline__ int64_t add(int64_t a, int64_t b) { return a + b; }
__device__ __forceinline__ int64_t neg(int64_t a) { return -a; }
__device__ __forceinline__ int64_t mul_int(int64_t a, int c) { return a * c; }

template <typename WT>
struct EvTraits {
  using A = int64_t;
  using CT = int64_t;
  static __device__ __forceinline__ A from(WT x) { return (int64_t)x; }
  static __device__ __forceinline__ A prod(int t, WT x) { return (int64_t)t * (int64_t)x; }
  static __device__ __forceinline__ CT out(A a) { return a; }
  static __device__ __forceinline__ CT bad() { return -1; }
  static __device__ __forceinline__ A shfl_xor(A a, int o) { return __shfl_xor_sync(FULL, a, o); }
  static __device__ __forceinline__ A shfl_up(A a, int o) { return __shfl_up_sync(FULL, a, o); }
  static __device__ __forceinline__ A shfl_idx(A a, int l) { return __shfl_sync(FULL, a, l); }
};
template <>
struct EvTraits<double> {
  using A = ddv;
  using CT = double;
  static __device__ __forceinline__ A from(double x) { return ddv{x, 0.0}; }
  static __device__ __forceinline__ A prod(int t, double x) {
    double p = t * x;
    return ddv{p, fma((double)t, x, -p)};
  }
  static __device__ __forceinline__ CT out(A a) { return a.hi + a.lo; }
  static __device__ __forceinline__ CT bad() { return NAN; }
  static __device__ __forceinline__ A shfl_xor(A a, int o) {
    return ddv{__shfl_xor_sync(FULL, a.hi, o), __shfl_xor_sync(FULL, a.lo, o)};
  }
  static __device__ __forceinline__ A shfl_up(A a, int o) {
    return ddv{__shfl_up_sync(FULL, a.hi, o), __shfl_up_sync(FULL, a.lo, o)};
  }
  static __device__ __forceinline__ A shfl_idx(A a, int l) {
    return ddv{__shfl_sync(FULL, a.hi, l), __shfl_sync(FULL, a.lo, l)};
  }
};

template <typename A, typename Tr>
__device__ __forceinline__ A warp_reduce(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = add(v, Tr::shfl_xor(v, o));
  return v;
}

template <typename WT>
__global__ void __launch_bounds__(EV_NT)
    eval_kernel(const WT* __restrict__ w, int E, int N, const int32_t* __restrict__ positions,
                const int32_t* __restrict__ npos, int S, int max_pos, int broadcast,
                typename EvTraits<WT>::CT* __restrict__ cost, int32_t* __restrict__ worst) {
  using Tr = EvTraits<WT>;
  using A = typename Tr::A;
  __shared__ A chp[EV_MAXCH + 1];   // chp[c] = sum of bins < 32 c (bin 0 excluded)
  __shared__ A wsum[EV_NW];
  __shared__ A sh_TN;
  const int lane = lane_id(), wid = warp_id();
  const int nch = (N + 1 + 31) / 32;

  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    const WT* we = w + (int64_t)e * (N + 1);
    // -- chunk sums (warp per chunk) and T_N ------------------------------------------------
    A tpart = A{};
    for (int c = wid; c < nch; c += EV_NW) {
      const int t = 32 * c + lane;
      const WT x = (t >= 1 && t <= N) ? we[t] : WT(0);
      A s = warp_reduce<A, Tr>(Tr::from(x));
      tpart = add(tpart, Tr::prod(t, x));
      if (lane == 0) chp[c + 1] = s;
    }
    tpart = warp_reduce<A, Tr>(tpart);
    if (lane == 0) wsum[wid] = tpart;
    __syncthreads();
    if (wid == 0) {   // warp scan of the chunk sums, 32 chunks per step
      A run = A{};
      if (lane == 0) chp[0] = run;
      for (int base = 1; base <= nch; base += 32) {
        const int c = base + lane;
        A inc = c <= nch ? chp[c] : A{};
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const A y = Tr::shfl_up(inc, o);
          if (lane >= o) inc = add(inc, y);
        }
        if (c <= nch) chp[c] = add(run, inc);
        run = add(run, Tr::shfl_idx(inc, 31));
      }
      if (lane == 0) {
        A tn = A{};
        for (int q = 0; q < EV_NW; ++q) tn = add(tn, wsum[q]);
        sh_TN = tn;
      }
    }
    __syncthreads();
    const A TN = sh_TN;

    // P(x) = sum_{t=1}^x w_t
    auto Pof = [&](int x) -> A {
      const int c = x >> 5;
      A s = chp[c];
      for (int t = max(32 * c, 1); t <= x; ++t) s = add(s, Tr::from(we[t]));
      return s;
    };

    // -- one warp per placement --------------------------------------------------------------
    for (int q = wid; q < S; q += EV_NW) {
      const int64_t set = broadcast ? q : (int64_t)e * S + q;
      const int32_t* pc = positions + set * max_pos;
      const int k = npos[set];
      bool ok = k >= 0 && k <= max_pos;
      A acc = A{};
      int gmax = 0;
      if (ok) {
        for (int i = lane; i <= k; i += 32) {   // gap i: (c_i, c_{i+1})
          const int ci = i == 0 ? 0 : pc[i - 1];
          const int cn = i == k ? N + 1 : pc[i];
          if (cn <= ci || cn > N + 1 || (i > 0 && ci < 1)) ok = false;
          gmax = max(gmax, cn - ci);
          if (i >= 1 && ok) {
            // c_i (P(c_{i+1} - 1) - P(c_i - 1))
            const A d = add(Pof(cn - 1), neg(Pof(ci - 1)));
            acc = add(acc, mul_int(d, ci));
          }
        }
      }
      ok = __all_sync(FULL, ok);
      acc = warp_reduce<A, Tr>(acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gmax = max(gmax, __shfl_xor_sync(FULL, gmax, o));
      if (lane == 0) {
        const int64_t oi = (int64_t)e * S + q;
        cost[oi] = ok ? Tr::out(add(TN, neg(acc))) : Tr::bad();
        if (worst) worst[oi] = ok ? gmax - 1 : -SP_ERR_BAD_POSITIONS;
      }
    }
    __syncthreads();
  }
}

// ---- int32 counts: the whole prefix row in shared memory ----------------------------------
// One 512-thread CTA per entry (persistent over entries).  The row is read in rounds of 16K
// bins: warp w owns 1024 consecutive bins, lane l holds bins 32u + l (u < 32) -- all 32 loads of
// a lane are issued before any is used, so a round keeps the whole 128 KB segment in flight.
// Each warp scans its segment in place (prefix relative to the segment start, int32) and the
// segment offsets (int64) go to woff[], so P(x) = seg[x] + woff[x >> 10]: one shared lookup per
// query instead of a 32-bin partial sum.  A segment whose own total reaches 2^31 (never on W5)
// makes the entry use exact int64 partial sums from global memory instead.
// ST = uint16_t: in-segment prefixes in 2 bytes (exact while a 1024-bin segment holds < 2^16
// counts -- W5's rows hold <= 16404 in all): 64 KB of shared memory per entry, 3 CTAs of 256
// threads per SM instead of 1 of 512.
template <typename ST, int EP_NT>
__global__ void __launch_bounds__(EP_NT)
    eval_p32_kernel(const int32_t* __restrict__ w, int E, int N,
                    const int32_t* __restrict__ positions, const int32_t* __restrict__ npos,
                    int S, int max_pos, int broadcast, int stage_sets,
                    int64_t* __restrict__ cost, int32_t* __restrict__ worst) {
  constexpr int EP_NW = EP_NT / 32;
  extern __shared__ __align__(16) unsigned char seg_raw[];
  ST* seg = reinterpret_cast<ST*>(seg_raw);   // [nseg * 1024] in-segment prefixes
  __shared__ long long woff[65];                     // exclusive segment offsets
  __shared__ long long wtot[EP_NW], tsum[EP_NW];
  __shared__ long long sh_carry, sh_TN;
  __shared__ int sh_big;
  const int lane = lane_id(), wid = warp_id();
  // segments cover bins 1..N (bin 0, the misses, is not in the objective): index x - 1 holds
  // P(x) relative to its segment -- N = 8192 is 8 segments, one round of 8 warps (round 1
  // scanned bins 0..N: a ninth segment of one bin and a second round)
  const int nseg = (N + 1023) / 1024;
  // broadcast sets staged once per CTA (stage_sets: the host checked they fit): positions as
  // uint16 (<= SP_MAX_N), and per set its worst case, or -1 for a malformed set
  uint16_t* spos = reinterpret_cast<uint16_t*>(seg_raw + (size_t)nseg * 1024 * sizeof(ST));
  int* sgap = reinterpret_cast<int*>(spos + (((size_t)S * max_pos + 1) & ~(size_t)1));
  if (stage_sets) {
    for (int q = wid; q < S; q += EP_NW) {
      const int32_t* pc = positions + (int64_t)q * max_pos;
      const int k = npos[q];
      bool ok = k >= 0 && k <= max_pos;
      int gmax = 0;
      if (ok) {
        for (int i = lane; i <= k; i += 32) {
          const int ci = i == 0 ? 0 : pc[i - 1];
          const int cn = i == k ? N + 1 : pc[i];
          if (cn <= ci || cn > N + 1 || (i > 0 && ci < 1)) ok = false;
          gmax = max(gmax, cn - ci);
          if (i < k) spos[(size_t)q * max_pos + i] = (uint16_t)cn;
        }
      }
      ok = __all_sync(FULL, ok);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gmax = max(gmax, __shfl_xor_sync(FULL, gmax, o));
      if (lane == 0) sgap[q] = ok ? gmax : -1;
    }
    __syncthreads();
  }
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    const int32_t* we = w + (int64_t)e * (N + 1);
    long long tpart = 0;
    int big = 0;
    if (threadIdx.x == 0) sh_carry = 0;
    for (int r0 = 0; r0 < nseg; r0 += EP_NW) {   // one round: segments r0 .. r0 + 31
      const int sg = r0 + wid;
      const int b0 = sg * 1024;
      int32_t v[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int t = b0 + 32 * u + lane + 1;
        v[u] = (sg < nseg && t <= N) ? __ldcs(we + t) : 0;
      }
      int run32 = 0;
      long long ls = 0;
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int t = b0 + 32 * u + lane + 1;
        tpart += (long long)t * v[u];
        ls += v[u];
        int inc = v[u];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL, inc, o);
          if (lane >= o) inc += y;
        }
        // exact while the segment total < 2^31 (checked below)
        if (sg < nseg) seg[b0 + 32 * u + lane] = (ST)(run32 + inc);
        run32 += __shfl_sync(FULL, inc, 31);
      }
      const long long run = warp_sum(ls);
      big |= run >= (sizeof(ST) == 2 ? (1ll << 16) : (1ll << 31));
      if (lane == 0) wtot[wid] = sg < nseg ? run : 0;
      __syncthreads();
      if (wid == 0) {   // exclusive scan of this round's segment totals
        const long long c0 = sh_carry;
        const long long x = lane < EP_NW ? wtot[lane] : 0;
        long long inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const long long y = __shfl_up_sync(FULL, inc, o);
          if (lane >= o) inc += y;
        }
        if (r0 + lane < nseg) woff[r0 + lane] = c0 + inc - x;
        if (lane == 31) sh_carry = c0 + inc;
      }
      __syncthreads();
    }
    tpart = warp_sum(tpart);
    big = __any_sync(FULL, big);
    if (lane == 0) tsum[wid] = tpart;
    if (threadIdx.x == 0) sh_big = 0;
    __syncthreads();
    if (lane == 0 && big) sh_big = 1;
    if (threadIdx.x == 0) {
      long long tn = 0;
      for (int q = 0; q < EP_NW; ++q) tn += tsum[q];
      sh_TN = tn;
    }
    __syncthreads();
    const long long TN = sh_TN;
    const bool exact32 = !sh_big;
    auto Pof = [&](int x) -> long long {
      if (x <= 0) return 0;
      const int i = x - 1;   // bin x sits at index x - 1
      if (exact32) return (long long)seg[i] + woff[i >> 10];
      long long s = woff[i >> 10];   // a huge segment: sum its bins from global memory
      for (int t = ((i >> 10) << 10) + 1; t <= x; ++t) s += we[t];
      return s;
    };
    if (stage_sets) {
      // (set, 32-gap group) items over all warps: gap i >= 1 of set q adds c_i (P(c_{i+1} - 1) -
      // P(c_i - 1)), both positions read from the staged copy
      for (int q = wid; q < S; q += EP_NW) {
        const int k = npos[q];
        const int g = sgap[q];
        long long acc = 0;
        if (g >= 0) {
          const uint16_t* sp = spos + (size_t)q * max_pos;
          for (int i = 1 + lane; i <= k; i += 32) {
            const int ci = sp[i - 1];
            const int cn = i == k ? N + 1 : sp[i];
            acc += (long long)ci * (Pof(cn - 1) - Pof(ci - 1));
          }
          acc = warp_sum(acc);
        }
        if (lane == 0) {
          const int64_t oi = (int64_t)e * S + q;
          cost[oi] = g >= 0 ? TN - acc : -1;
          if (worst) worst[oi] = g >= 0 ? g - 1 : -SP_ERR_BAD_POSITIONS;
        }
      }
      __syncthreads();
      continue;
    }
    for (int q = wid; q < S; q += EP_NW) {
      const int64_t set = broadcast ? q : (int64_t)e * S + q;
      const int32_t* pc = positions + set * max_pos;
      const int k = npos[set];
      bool ok = k >= 0 && k <= max_pos;
      long long acc = 0;
      int gmax = 0;
      if (ok) {
        for (int i = lane; i <= k; i += 32) {   // gap i: (c_i, c_{i+1})
          const int ci = i == 0 ? 0 : pc[i - 1];
          const int cn = i == k ? N + 1 : pc[i];
          if (cn <= ci || cn > N + 1 || (i > 0 && ci < 1)) ok = false;
          gmax = max(gmax, cn - ci);
          if (i >= 1 && ok) acc += (long long)ci * (Pof(cn - 1) - Pof(ci - 1));
        }
      }
      ok = __all_sync(FULL, ok);
      acc = warp_sum(acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gmax = max(gmax, __shfl_xor_sync(FULL, gmax, o));
      if (lane == 0) {
        const int64_t oi = (int64_t)e * S + q;
        cost[oi] = ok ? TN - acc : -1;
        if (worst) worst[oi] = ok ? gmax - 1 : -SP_ERR_BAD_POSITIONS;
      }
    }
    __syncthreads();
  }
}

// int32 counts, placements shared by every entry (broadcast: the Table 1 baselines): with the
// reusable depth l(t; C) of every bin tabulated, the cost is a single streaming pass,
//     cost = T_N - sum_t c_t l(t; C)      (l(t; C) = largest position <= t, 0 if none)
// i.e. a product of the count matrix with S fixed columns l(.; C_s).  Each CTA (one per SM)
// validates the sets, computes their worst cases and fills the uint16 tables l[s][t] in shared
// memory once; then its warps stream row slices (EB_U coalesced loads in flight per lane, no
// phases, no barriers), accumulate c_t t and c_t l[s][t] and add them into cost atomically.  HBM-bound: the row is
// read once.  Exact in int64 (|c_t| < 2^31, t, l <= SP_MAX_N).
#ifndef SP_EVAL_BCAST_NT
#define SP_EVAL_BCAST_NT 1024
#endif
#ifndef SP_EVAL_BCAST_U
#define SP_EVAL_BCAST_U 12
#endif
constexpr int EB_NT = SP_EVAL_BCAST_NT;
constexpr int EB_U = SP_EVAL_BCAST_U;
constexpr int EB_MAXS = 4;
static_assert(EB_U >= 1 && EB_U <= 16, "the 32-bit fast path needs EB_U <= 16");
constexpr int EB_FB = EB_U <= 1 ? 16 : EB_U <= 2 ? 15 : EB_U <= 4 ? 14 : EB_U <= 8 ? 13 : 12;
constexpr size_t EB_SMEM_MAX = 200 * 1024;   // tables: S (N+1+SL) 2 bytes

__device__ __forceinline__ long long mad_wide(int a, int b, long long c) {   // c + a b, exact
  long long d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

template <int SN>   // SN = S, the number of broadcast sets
__global__ void __launch_bounds__(EB_NT, 1)
    eval_bcast_kernel(const int32_t* __restrict__ w, int E, int N,
                      const int32_t* __restrict__ positions, const int32_t* __restrict__ npos,
                      int S, int max_pos, int64_t* __restrict__ cost, int32_t* __restrict__ worst) {
  extern __shared__ __align__(16) uint16_t ltab[];   // [S][N+1]
  __shared__ int sh_ok[SN], sh_gap[SN];
  constexpr int NW = EB_NT / 32;
  const int lane = lane_id(), wid = warp_id();
  const int rowlen = N + 1;
  constexpr int SL = 32 * EB_U;
  const int tstride = rowlen + SL;   // table stride: padded with l = 0 past the row
  // ---- sets: validity and worst case (warp q: set q) ---------------------------------------
  if (wid < S) {
    const int32_t* pc = positions + (int64_t)wid * max_pos;
    const int k = npos[wid];
    bool ok = k >= 0 && k <= max_pos;
    int g = 0;
    if (ok) {
      for (int i = lane; i <= k; i += 32) {   // gap i: (c_i, c_{i+1})
        const int ci = i == 0 ? 0 : pc[i - 1];
        const int cn = i == k ? N + 1 : pc[i];
        if (cn <= ci || cn > N + 1 || (i > 0 && ci < 1)) ok = false;
        g = max(g, cn - ci);
      }
    }
    ok = __all_sync(FULL, ok);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) g = max(g, __shfl_xor_sync(FULL, g, o));
    if (lane == 0) {
      sh_ok[wid] = ok;
      sh_gap[wid] = g;
    }
  }
  __syncthreads();
  // ---- tables: l[s][t] = c_i on segment i = [c_i, c_{i+1}) (one warp per segment) ------------
  for (int s = 0; s < S; ++s) {
    if (!sh_ok[s]) continue;
    const int32_t* pc = positions + (int64_t)s * max_pos;
    const int k = npos[s];
    uint16_t* lt = ltab + (size_t)s * tstride;
    for (int i = wid; i <= k; i += NW) {
      const int ci = i == 0 ? 0 : pc[i - 1];
      const int cn = i == k ? N + 1 : pc[i];
      for (int t = ci + lane; t < cn; t += 32) lt[t] = (uint16_t)ci;
    }
    for (int t = rowlen + (int)threadIdx.x; t < tstride; t += EB_NT) lt[t] = 0;
  }
  __syncthreads();
  // ---- work items: (entry, 32 EB_U-bin slice of its row).  Warp w takes the contiguous item
  // range [w I / W, (w+1) I / W) (perfect balance, whatever E), reading slice i+1 while it
  // computes slice i.  Lane l reads bins l, l + 32, ... (coalesced 128-byte loads,
  // conflict-free table lookups).  The cost is linear in the bins, so a warp adds its share of
  // an entry with one 64-bit atomic per set into cost (zeroed by the host call) when it leaves
  // the entry; the slice-0 item writes the worst case and the flag of a malformed set (which
  // receives no atomics).
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(ltab);
  const uint32_t sstride = 2u * (uint32_t)tstride;   // bytes between two sets' tables
  const int nsl = (N + SL) / SL;   // slices per row (N + 1 bins)
  const int64_t items = (int64_t)E * nsl;
  const int64_t gw = (int64_t)blockIdx.x * NW + wid, nwt = (int64_t)gridDim.x * NW;
  const int64_t i0 = items * gw / nwt, i1 = items * (gw + 1) / nwt;
  if (i0 >= i1) return;
  int e = (int)(i0 / nsl), sl = (int)(i0 - (int64_t)e * nsl);
  // one slice of a row into registers: unpredicated unless it is the row's ragged last slice
  auto load_slice = [&](int ee, int ss, int (&dst)[EB_U]) {
    const int32_t* we = w + (int64_t)ee * rowlen + ss * SL + lane;
    if (ss * SL + SL <= rowlen) {
#pragma unroll
      for (int u = 0; u < EB_U; ++u) dst[u] = __ldcs(we + 32 * u);
    } else {
      const int lim = rowlen - ss * SL - lane;   // bins of this lane still inside the row: > 32 u
#pragma unroll
      for (int u = 0; u < EB_U; ++u) dst[u] = 32 * u < lim ? __ldcs(we + 32 * u) : 0;
    }
  };
  int c[EB_U];
  load_slice(e, sl, c);
  long long tsum = 0, acc[SN];
#pragma unroll
  for (int q = 0; q < SN; ++q) acc[q] = 0;
  for (int rem = (int)(i1 - i0); rem > 0; --rem) {
    int en = e, sn = sl + 1;
    if (sn == nsl) {
      sn = 0;
      ++en;
    }
    const bool more = rem > 1;
    int cn[EB_U];
    if (more) load_slice(en, sn, cn);
    const int tb = sl * SL;
    // 32-bit fast path: when every count of the slice is in [0, 2^EB_FB), a lane's EB_U products
    // c_t t and c_t l sum to < EB_U 2^EB_FB 2^16 <= 2^32 (t, l <= SP_MAX_N < 2^16), so each lane
    // accumulates the slice in uint32 and widens once; the tables are padded by SL entries
    // (l = 0 past the row, c = 0 there) so the lookups need no clamp.  Otherwise int64 per bin.
    unsigned orc = 0;
#pragma unroll
    for (int u = 0; u < EB_U; ++u) orc |= (unsigned)c[u];
    if (__all_sync(FULL, (orc >> EB_FB) == 0)) {
      const uint32_t a0 = sbase + 2u * (uint32_t)(tb + lane);
      uint32_t aq[SN], s32[SN];
#pragma unroll
      for (int q = 0; q < SN; ++q) {
        aq[q] = a0 + (uint32_t)q * sstride;
        s32[q] = 0;
      }
      uint32_t t32 = 0;
#pragma unroll
      for (int u = 0; u < EB_U; ++u) {
        t32 += (uint32_t)c[u] * (uint32_t)(tb + 32 * u + lane);
#pragma unroll
        for (int q = 0; q < SN; ++q) {
          unsigned short l;
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(l) : "r"(aq[q] + 64u * u));
          s32[q] += (uint32_t)c[u] * (uint32_t)l;
        }
      }
      tsum += (long long)t32;
#pragma unroll
      for (int q = 0; q < SN; ++q) acc[q] += (long long)s32[q];
    } else {
#pragma unroll
      for (int u = 0; u < EB_U; ++u) {
        const int t = tb + 32 * u + lane;   // <= N + SL: c = 0 and l = 0 past the row
        tsum = mad_wide(c[u], t, tsum);
        const uint32_t a = sbase + 2u * (uint32_t)t;
#pragma unroll
        for (int q = 0; q < SN; ++q) {
          unsigned short l;
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(l) : "r"(a + q * sstride));
          acc[q] = mad_wide(c[u], (int)l, acc[q]);
        }
      }
    }
    if (sl == 0 && lane == 0) {
#pragma unroll
      for (int q = 0; q < SN; ++q) {
        const int64_t oi = (int64_t)e * S + q;
        if (!sh_ok[q]) cost[oi] = -1;
        if (worst) worst[oi] = sh_ok[q] ? sh_gap[q] - 1 : -SP_ERR_BAD_POSITIONS;
      }
    }
    if (sn == 0 || !more) {   // leaving entry e: add this warp's share
      tsum = warp_sum(tsum);
#pragma unroll
      for (int q = 0; q < SN; ++q) {
        const long long a = warp_sum(acc[q]);
        if (lane == 0 && sh_ok[q])
          atomicAdd(reinterpret_cast<unsigned long long*>(cost + (int64_t)e * S + q),
                    (unsigned long long)(tsum - a));
        acc[q] = 0;
      }
      tsum = 0;
    }
#pragma unroll
    for (int u = 0; u < EB_U; ++u) c[u] = cn[u];
    e = en;
    sl = sn;
  }
}

// fp64 weights, <= 4 broadcast sets (the bench's `--weights f64` evaluation, a7): the same
// tabulated l[s][t] in shared memory, but cost_s = sum_t w_t (t - l_s(t)) summed directly -- every
// term is >= 0, so nothing cancels -- with each product exact (fma) and a compensated running sum
// per lane (Neumaier), combined over the warp in double-double: relative error ~1e-16, inside
// reading R10's 1e-12.  One warp per entry (no atomics: deterministic), EB_U loads in flight per
// lane, the next slice prefetched.  Bin 0 (misses) contributes nothing.
constexpr int EF_U = 8;
template <int SN>
__global__ void __launch_bounds__(EB_NT, 1)
    eval_bcast_f64_kernel(const double* __restrict__ w, int E, int N,
                          const int32_t* __restrict__ positions, const int32_t* __restrict__ npos,
                          int S, int max_pos, double* __restrict__ cost,
                          int32_t* __restrict__ worst) {
  extern __shared__ __align__(16) uint16_t ltab[];   // [S][N+1+SL]
  __shared__ int sh_ok[SN], sh_gap[SN];
  constexpr int NW = EB_NT / 32;
  constexpr int SL = 32 * EF_U;
  const int lane = lane_id(), wid = warp_id();
  const int rowlen = N + 1;
  const int tstride = rowlen + SL;
  if (wid < S) {   // validity and worst case (warp q: set q)
    const int32_t* pc = positions + (int64_t)wid * max_pos;
    const int k = npos[wid];
    bool ok = k >= 0 && k <= max_pos;
    int g = 0;
    if (ok) {
      for (int i = lane; i <= k; i += 32) {
        const int ci = i == 0 ? 0 : pc[i - 1];
        const int cn = i == k ? N + 1 : pc[i];
        if (cn <= ci || cn > N + 1 || (i > 0 && ci < 1)) ok = false;
        g = max(g, cn - ci);
      }
    }
    ok = __all_sync(FULL, ok);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) g = max(g, __shfl_xor_sync(FULL, g, o));
    if (lane == 0) {
      sh_ok[wid] = ok;
      sh_gap[wid] = g;
    }
  }
  __syncthreads();
  for (int s = 0; s < S; ++s) {   // l[s][t] = c_i on [c_i, c_{i+1}); padded with 0
    if (!sh_ok[s]) continue;
    const int32_t* pc = positions + (int64_t)s * max_pos;
    const int k = npos[s];
    uint16_t* lt = ltab + (size_t)s * tstride;
    for (int i = wid; i <= k; i += NW) {
      const int ci = i == 0 ? 0 : pc[i - 1];
      const int cn = i == k ? N + 1 : pc[i];
      for (int t = ci + lane; t < cn; t += 32) lt[t] = (uint16_t)ci;
    }
    for (int t = rowlen + (int)threadIdx.x; t < tstride; t += EB_NT) lt[t] = 0;
  }
  __syncthreads();
  const int nsl = (N + SL) / SL;
  for (int e = blockIdx.x * NW + wid; e < E; e += gridDim.x * NW) {
    const double* we = w + (int64_t)e * rowlen + lane;
    double hi[SN], lo[SN];
#pragma unroll
    for (int q = 0; q < SN; ++q) hi[q] = lo[q] = 0.0;
    double x[EF_U], xn[EF_U];
    auto load = [&](int sl, double (&d)[EF_U]) {
      const int base = sl * SL;
#pragma unroll
      for (int u = 0; u < EF_U; ++u) {
        const int t = base + 32 * u + lane;
        d[u] = (t >= 1 && t <= N) ? __ldcs(we + base + 32 * u) : 0.0;
      }
    };
    load(0, x);
    for (int sl = 0; sl < nsl; ++sl) {
      if (sl + 1 < nsl) load(sl + 1, xn);
#pragma unroll
      for (int u = 0; u < EF_U; ++u) {
        const int t = sl * SL + 32 * u + lane;
#pragma unroll
        for (int q = 0; q < SN; ++q) {
          const int d = t - (int)ltab[(size_t)q * tstride + t];
          const double pr = x[u] * (double)d;
          const double pe = fma(x[u], (double)d, -pr);   // the product's exact remainder
          const double sm = hi[q] + pr;                   // Neumaier: sm + err = hi + pr
          const double err = fabs(hi[q]) >= fabs(pr) ? (hi[q] - sm) + pr : (pr - sm) + hi[q];
          hi[q] = sm;
          lo[q] += err + pe;
        }
      }
#pragma unroll
      for (int u = 0; u < EF_U; ++u) x[u] = xn[u];
    }
#pragma unroll
    for (int q = 0; q < SN; ++q) {
      ddv v = add(ddv{hi[q], 0.0}, ddv{lo[q], 0.0});
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        v = add(v, ddv{__shfl_xor_sync(FULL, v.hi, o), __shfl_xor_sync(FULL, v.lo, o)});
      if (lane == 0) {
        const int64_t oi = (int64_t)e * S + q;
        cost[oi] = sh_ok[q] ? v.hi + v.lo : NAN;
        if (worst) worst[oi] = sh_ok[q] ? sh_gap[q] - 1 : -SP_ERR_BAD_POSITIONS;
      }
    }
  }
}

}  // namespace sp

// Launch facts cached per device (no attribute / occupancy query on every call once warm).
constexpr int EV_MAX_DEV = 64;
static int eval_dev() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 || dev >= EV_MAX_DEV ? 0 : dev;
}
static int eval_sms() {
  static std::atomic<int> sms[EV_MAX_DEV];
  const int dev = eval_dev();
  int v = sms[dev].load(std::memory_order_relaxed);
  if (!v) {
    v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}
// opt in, once per (device, kernel slot), to the most dynamic shared memory the kernel can have
// (static + dynamic <= the per-block opt-in limit): every later size fits
template <typename K>
static void eval_smem_attr(K kern, int slot) {
  static std::atomic<bool> done[EV_MAX_DEV][8];
  const int dev = eval_dev();
  if (!done[dev][slot].load(std::memory_order_acquire)) {
    int optin = 227 * 1024;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           optin - (int)fa.sharedSizeBytes);
    done[dev][slot].store(true, std::memory_order_release);
  }
}
// resident CTAs per SM for `dyn` bytes (cached per device, kernel slot and size)
template <typename K>
static int eval_occ(K kern, int nt, size_t dyn, int slot) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, size_t>, int> cache;
  const int dev = eval_dev();
  eval_smem_attr(kern, slot);
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(dev, slot, dyn);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, dyn);
  cache[key] = occ;
  return occ;
}

extern "C" sp_status sp_expected_recompute(const void* weights, sp_weight_type wtype,
                                           int32_t n_entries, int32_t N,
                                           const int32_t* positions, const int32_t* n_positions,
                                           int32_t n_sets, int32_t max_pos, int32_t broadcast,
                                           void* cost, int32_t* worst_case, sp_stream_t stream) {
  if (N < 1 || N > SP_MAX_N || n_entries < 0 || n_sets < 0 || max_pos < 0)
    return SP_ERR_BAD_LENGTH;
  if (wtype != SP_W_COUNTS_I32 && wtype != SP_W_COUNTS_I64 && wtype != SP_W_PROB_F64)
    return SP_ERR_BAD_ARGUMENT;
  if (n_entries == 0 || n_sets == 0) return SP_OK;
  if (!weights || !n_positions || !cost || (max_pos > 0 && !positions))
    return SP_ERR_BAD_ARGUMENT;
  const int sms = eval_sms();
  const int grid = n_entries < sms * 8 ? n_entries : sms * 8;
  cudaStream_t st = (cudaStream_t)stream;
  const int path = sp_debug_get(SP_DBG_EVAL_PATH);   // 0 auto; 1 chunked, 2 p32, 3 prefix
  const size_t tab = (size_t)n_sets * (N + 1 + 32 * sp::EB_U) * sizeof(uint16_t);
  if (wtype == SP_W_COUNTS_I32 && path == 0 && broadcast && n_sets <= sp::EB_MAXS &&
      tab <= sp::EB_SMEM_MAX) {
    auto kern = n_sets == 1   ? sp::eval_bcast_kernel<1>
                : n_sets == 2 ? sp::eval_bcast_kernel<2>
                : n_sets == 3 ? sp::eval_bcast_kernel<3>
                              : sp::eval_bcast_kernel<4>;
    eval_smem_attr(kern, n_sets - 1);
    if (cudaMemsetAsync(cost, 0, (size_t)n_entries * n_sets * sizeof(int64_t), st) != cudaSuccess)
      return SP_ERR_CUDA;
    kern<<<sms, sp::EB_NT, tab, st>>>(
        (const int32_t*)weights, n_entries, N, positions, n_positions, n_sets, max_pos,
        (int64_t*)cost, worst_case);
  } else if (wtype == SP_W_PROB_F64 && path == 0 && broadcast && n_sets <= sp::EB_MAXS &&
             (size_t)n_sets * (N + 1 + 32 * sp::EF_U) * sizeof(uint16_t) <= sp::EB_SMEM_MAX) {
    auto kern = n_sets == 1   ? sp::eval_bcast_f64_kernel<1>
                : n_sets == 2 ? sp::eval_bcast_f64_kernel<2>
                : n_sets == 3 ? sp::eval_bcast_f64_kernel<3>
                              : sp::eval_bcast_f64_kernel<4>;
    eval_smem_attr(kern, n_sets - 1);   // (its own per-type slots, like the int32 kernels')
    const int nw = sp::EB_NT / 32;
    const int g = std::min((n_entries + nw - 1) / nw, sms);
    kern<<<g, sp::EB_NT, (size_t)n_sets * (N + 1 + 32 * sp::EF_U) * sizeof(uint16_t), st>>>(
        (const double*)weights, n_entries, N, positions, n_positions, n_sets, max_pos,
        (double*)cost, worst_case);
  } else if (wtype == SP_W_COUNTS_I32 && path != 1) {
    const int nseg = (N + 1023) / 1024;   // bins 1..N (eval_p32_kernel)
    const bool wide = path == 2;   // 4-byte prefixes (tests / comparison)
    size_t dyn = (size_t)nseg * 1024 * (wide ? 4 : 2);
    // broadcast sets staged in shared memory when they fit in 32 KB more
    const size_t sets_bytes = (((size_t)n_sets * max_pos + 1) & ~(size_t)1) * 2 + (size_t)n_sets * 4;
    const int stage = broadcast && sets_bytes <= 32 * 1024;
    if (stage) dyn += sets_bytes;
    const int occ = wide ? eval_occ(sp::eval_p32_kernel<int32_t, 512>, 512, dyn, 4)
                         : eval_occ(sp::eval_p32_kernel<uint16_t, 256>, 256, dyn, 5);
    const long gcap = (long)sms * (occ < 1 ? 1 : occ);
    const int g2 = n_entries < gcap ? n_entries : (int)gcap;
    if (wide)
      sp::eval_p32_kernel<int32_t, 512><<<g2, 512, dyn, st>>>(
          (const int32_t*)weights, n_entries, N, positions, n_positions, n_sets, max_pos,
          broadcast, stage, (int64_t*)cost, worst_case);
    else
      sp::eval_p32_kernel<uint16_t, 256><<<g2, 256, dyn, st>>>(
          (const int32_t*)weights, n_entries, N, positions, n_positions, n_sets, max_pos,
          broadcast, stage, (int64_t*)cost, worst_case);
  } else if (wtype == SP_W_COUNTS_I32)
    sp::eval_kernel<int32_t><<<grid, sp::EV_NT, 0, st>>>(
        (const int32_t*)weights, n_entries, N, positions, n_positions, n_sets, max_pos,
        broadcast, (int64_t*)cost, worst_case);
  else if (wtype == SP_W_COUNTS_I64)
    sp::eval_kernel<int64_t><<<grid, sp::EV_NT, 0, st>>>(
        (const int64_t*)weights, n_entries, N, positions, n_positions, n_sets, max_pos,
        broadcast, (int64_t*)cost, worst_case);
  else
    sp::eval_kernel<double><<<grid, sp::EV_NT, 0, st>>>(
        (const double*)weights, n_entries, N, positions, n_positions, n_sets, max_pos,
        broadcast, (double*)cost, worst_case);
  SP_CHECK_LAUNCH();
  return SP_OK;
}
