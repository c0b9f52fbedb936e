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
#include <climits>
#include <cmath>

#include "common.cuh"

namespace sp {

constexpr int DP_NT = 512;
constexpr int DP_NW = DP_NT / 32;
constexpr int DP_TPL = 8;   // target candidate evaluations per thread per row

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

// workspace slot layout (bytes): P 8B[N+1] | bA 8B[N+1] | bB 8B[N+1] | opt uint16[M][N+1]
__host__ __device__ __forceinline__ size_t slot_bytes(int N, int M) {
  return 3 * align256(8 * (size_t)(N + 1)) + align256(2 * (size_t)(M > 0 ? M : 1) * (N + 1));
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
};

struct Shared {
  int64_t wbuf[DP_NW + 1];
  double dbuf[2 * (DP_NW + 1)];
  int64_t red_v[DP_NW];
  int32_t red_s[DP_NW];
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

__device__ __forceinline__ unsigned group_mask(int G) {
  if (G >= 32) return FULL;
  const unsigned base = (threadIdx.x & 31) & ~(unsigned)(G - 1);
  return ((1u << G) - 1) << base;
}

template <typename VT>
__device__ __forceinline__ void lex_min(VT& bv, int& bs, VT ov, int os) {
  if (ov < bv || (ov == bv && os < bs)) {
    bv = ov;
    bs = os;
  }
}

// bracket of row j at the level with half-spacing h
template <typename Ctx>
__device__ __forceinline__ void row_bracket(const Ctx& c, int j, int h, int& lo, int& hi) {
  lo = 1;
  hi = j;
  const int jl = j - h, jr = j + h;
  if (jl >= 1) lo = c.sopt[jl];
  if (jr <= c.N) hi = min((int)c.sopt[jr], j);
  if (c.optprev) lo = max(lo, (int)c.optprev[j]);
}

// per-thread scan of candidates s = lo + t, lo + t + G, ... <= hi (s increasing: strict '<'
// keeps the lowest index within the thread)
template <typename VT>
__device__ __forceinline__ void scan_candidates(const VT* __restrict__ b, VT Pj, int lo, int hi,
                                                int t, int G, VT& bv, int& bs) {
  int s = lo + t;
#pragma unroll 4
  for (; s <= hi; s += G) {
    const VT v = cand(b[s], s, Pj);
    if (v < bv) {
      bv = v;
      bs = s;
    }
  }
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
  c.optout[j] = (uint16_t)bs;
  if (j < c.N) c.bnext[j + 1] = icpt(bv, j + 1, Pj);
  if (j == c.N) {
    const auto V = c.TN + bv;   // dp[m][N] = T_N + e_m(N)
    if (c.cbb_e) c.cbb_e[c.m] = V;
    if (c.last) *c.cost_e = V;
  }
}

// fp64: rounding can make neighbouring brackets cross by a hair; clamp instead of flagging
template <typename Ctx>
__device__ __forceinline__ void fix_bracket(const Ctx&, double*, int& lo, int hi) {
  if (lo > hi) lo = hi;
}
template <typename Ctx, typename VT>
__device__ __forceinline__ void fix_bracket(const Ctx&, VT*, int&, int) {}

// one level, groups of G <= 32 threads per row (rows strided over groups)
template <typename VT, int G, typename Ctx>
__device__ void level_small(const Ctx& c, int h, int R) {
  const int gid = threadIdx.x / G, t = threadIdx.x % G;
  constexpr int NG = DP_NT / G;
  const unsigned gmask = group_mask(G);
  for (int i = gid; i < R; i += NG) {
    const int j = h * (2 * i + 1);
    int lo, hi;
    row_bracket(c, j, h, lo, hi);
    fix_bracket(c, (VT*)nullptr, lo, hi);
    const VT Pj = (VT)c.P[j];
    VT bv = Lim<VT>::inf();
    int bs = INT_MAX;
    scan_candidates(c.b, Pj, lo, hi, t, G, bv, bs);
#pragma unroll
    for (int o = G / 2; o >= 1; o >>= 1) {
      const VT ov = __shfl_xor_sync(gmask, bv, o);
      const int os = __shfl_xor_sync(gmask, bs, o);
      lex_min(bv, bs, ov, os);
    }
    if (t == 0) row_write(c, j, lo, hi, Pj, bv, bs);
  }
}

// one level, groups of G > 32 threads (several warps) per row; uniform trip count so that
// __syncthreads can be used for the cross-warp reduction
template <typename VT, int G, typename Ctx>
__device__ void level_big(const Ctx& c, Shared& sh, int h, int R) {
  const int gid = threadIdx.x / G, t = threadIdx.x % G;
  constexpr int NG = DP_NT / G, WPG = G / 32;
  const int iters = (R + NG - 1) / NG;
  for (int it = 0; it < iters; ++it) {
    const int i = it * NG + gid;
    const bool valid = i < R;
    int lo = 1, hi = 0, j = 1;
    VT Pj = 0;
    VT bv = Lim<VT>::inf();
    int bs = INT_MAX;
    if (valid) {
      j = h * (2 * i + 1);
      row_bracket(c, j, h, lo, hi);
      fix_bracket(c, (VT*)nullptr, lo, hi);
      Pj = (VT)c.P[j];
      scan_candidates(c.b, Pj, lo, hi, t, G, bv, bs);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const VT ov = __shfl_xor_sync(FULL, bv, o);
      const int os = __shfl_xor_sync(FULL, bs, o);
      lex_min(bv, bs, ov, os);
    }
    if (lane_id() == 0) {
      // stored through the int64 buffer (doubles by bit pattern)
      if constexpr (sizeof(VT) == 8) {
        sh.red_v[warp_id()] = *reinterpret_cast<const int64_t*>(&bv);
      } else {
        sh.red_v[warp_id()] = (int64_t)bv;
      }
      sh.red_s[warp_id()] = bs;
    }
    __syncthreads();
    if (valid && t == 0) {
      for (int q = 1; q < WPG; ++q) {
        VT ov;
        if constexpr (sizeof(VT) == 8) {
          ov = *reinterpret_cast<const VT*>(&sh.red_v[warp_id() + q]);
        } else {
          ov = (VT)sh.red_v[warp_id() + q];
        }
        lex_min(bv, bs, ov, sh.red_s[warp_id() + q]);
      }
      row_write(c, j, lo, hi, Pj, bv, bs);
    }
    __syncthreads();
  }
}

template <typename VT, typename Ctx>
__device__ void run_level(const Ctx& c, Shared& sh, int h, int R) {
  // expected bracket width ~ 2h; aim at DP_TPL evaluations per thread, but use every thread
  int G = 1;
  const int want = (2 * h) / DP_TPL;
  while (G * 2 <= want && G < DP_NT) G *= 2;
  int rp = 1;
  while (rp < R) rp *= 2;
  const int need = DP_NT / rp;   // 0 when R > DP_NT
  if (G < need) G = need;
  switch (G) {
    case 1: level_small<VT, 1>(c, h, R); break;
    case 2: level_small<VT, 2>(c, h, R); break;
    case 4: level_small<VT, 4>(c, h, R); break;
    case 8: level_small<VT, 8>(c, h, R); break;
    case 16: level_small<VT, 16>(c, h, R); break;
    case 32: level_small<VT, 32>(c, h, R); break;
    case 64: level_big<VT, 64>(c, sh, h, R); break;
    case 128: level_big<VT, 128>(c, sh, h, R); break;
    case 256: level_big<VT, 256>(c, sh, h, R); break;
    default: level_big<VT, 512>(c, sh, h, R); break;
  }
}

template <typename PT>
__device__ __forceinline__ uint8_t* slot_of(const DpParams& p) {
  return p.ws + (size_t)blockIdx.x * p.slot;
}

// Solve one entry with value type VT; b in shared memory (BS) or in the slot's global arrays.
template <typename VT, bool BS, typename PT, typename CT>
__device__ void solve_entry(const DpParams& p, Shared& sh, VT* smem_b, uint16_t* sopt, int e,
                            CT TN) {
  const int N = p.N, M = p.M;
  uint8_t* slot = p.ws + (size_t)blockIdx.x * p.slot;
  const PT* P = reinterpret_cast<const PT*>(slot);
  VT* bA = reinterpret_cast<VT*>(slot + align256(8 * (size_t)(N + 1)));
  VT* bB = reinterpret_cast<VT*>(slot + 2 * align256(8 * (size_t)(N + 1)));
  uint16_t* opt = reinterpret_cast<uint16_t*>(slot + 3 * align256(8 * (size_t)(N + 1)));

  VT* b = BS ? smem_b : bA;
  VT* bnext = bB;
  // layer 1: e_0 == 0 => b_s = s P_{s-1}
  for (int s = threadIdx.x + 1; s <= N; s += DP_NT) b[s] = icpt((VT)0, s, (VT)P[s - 1]);
  __syncthreads();

  LayerCtx<VT, PT, CT> c;
  c.sopt = sopt;
  c.P = P;
  c.N = N;
  c.TN = TN;
  c.cbb_e = p.cbb ? reinterpret_cast<CT*>(p.cbb) + (int64_t)e * (M + 1) : nullptr;
  c.cost_e = reinterpret_cast<CT*>(p.cost) + e;
  c.err = &sh.err;
  for (int m = 1; m <= M; ++m) {
    c.b = b;
    c.bnext = bnext;
    c.m = m;
    c.last = (m == M);
    c.optout = opt + (size_t)(m - 1) * (N + 1);
    c.optprev = m >= 2 ? opt + (size_t)(m - 2) * (N + 1) : nullptr;
    for (int k = 0; k < p.L; ++k) {
      const int h = 1 << (p.L - 1 - k);
      const int R = ((N / h) + 1) >> 1;
      run_level<VT>(c, sh, h, R);
      __syncthreads();
    }
    if (m < M) {
      if (BS) {
        for (int s = threadIdx.x + 2; s <= N; s += DP_NT) b[s] = bnext[s];
        if (threadIdx.x == 0) b[1] = 0;   // e_m(0) + 1 * P_0 = 0
      } else {
        if (threadIdx.x == 0) bnext[1] = 0;
        VT* t = b;
        b = bnext;
        bnext = t;
      }
      __syncthreads();
    }
  }
}

// ---- a3 for counts: P_j (int64) and T_N, block-wide scan over bins 1..N --------------------
template <typename WT>
__device__ void prefix_counts(const WT* we, int N, int64_t* P, Shared& sh, int64_t& TN,
                              int64_t& n, int& neg) {
  int64_t carry = 0, tpart = 0;
  int bad = 0;
  for (int base = 0; base <= N; base += DP_NT) {
    const int t = base + threadIdx.x;
    int64_t cnt = 0;
    if (t >= 1 && t <= N) cnt = (int64_t)we[t];
    bad |= cnt < 0;
    int64_t tot;
    const int64_t ex = block_exclusive_scan<DP_NT>(cnt, sh.wbuf, &tot);
    if (t <= N) P[t] = carry + ex + cnt;
    carry += tot;
    tpart += (int64_t)t * cnt;
  }
  TN = block_sum<DP_NT>(tpart, sh.wbuf);
  n = carry;
  neg = __syncthreads_or(bad);
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

template <typename WT>
__global__ void __launch_bounds__(DP_NT) dp_place_kernel(DpParams p) {
  using PT = typename WTraits<WT>::PT;
  using CT = typename WTraits<WT>::CT;
  constexpr bool F64 = sizeof(WT) == 8 && std::is_floating_point<WT>::value;
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ Shared sh;
  const int N = p.N, M = p.M;
  uint16_t* sopt = reinterpret_cast<uint16_t*>(dsm);
  int32_t* smem_b32 = reinterpret_cast<int32_t*>(dsm + align256(2 * (size_t)(N + 1)));
  const WT* w = reinterpret_cast<const WT*>(p.w);
  CT* cost = reinterpret_cast<CT*>(p.cost);
  CT* cbb = reinterpret_cast<CT*>(p.cbb);

  for (int e = blockIdx.x; e < p.E; e += gridDim.x) {
    uint8_t* slot = p.ws + (size_t)blockIdx.x * p.slot;
    PT* P = reinterpret_cast<PT*>(slot);
    const WT* we = w + (int64_t)e * (N + 1);
    CT TN, n;
    int neg;
    if constexpr (F64) {
      prefix_f64(we, N, P, sh, TN, n, neg);
    } else {
      prefix_counts<WT>(we, N, P, sh, TN, n, neg);
    }
    if (threadIdx.x == 0) {
      sh.err = 0;
      if (cbb) cbb[(int64_t)e * (M + 1)] = TN;   // V_0 = T_N
      cost[e] = TN;
    }
    __syncthreads();

    // ---- a4: the DP ----------------------------------------------------------------------
    int status = 0;
    if (neg) {
      status = SP_ERR_BAD_ARGUMENT;
    } else if (M > 0) {
      if constexpr (F64) {
        solve_entry<double, false, PT, CT>(p, sh, nullptr, sopt, e, TN);
      } else {
        // narrow (exact int32) when 2 n N < 2^31, else int64 (exact when 2 n N < 2^62)
        const bool narrow = n < (int64_t(1) << 30) / N;
        const bool wide_ok = n < (int64_t(1) << 61) / N;
        if (narrow) {
          if (p.smem_b) solve_entry<int32_t, true, PT, CT>(p, sh, smem_b32, sopt, e, TN);
          else solve_entry<int32_t, false, PT, CT>(p, sh, nullptr, sopt, e, TN);
        } else if (wide_ok) {
          solve_entry<int64_t, false, PT, CT>(p, sh, nullptr, sopt, e, TN);
        } else {
          status = SP_ERR_OVERFLOW;
        }
      }
    }
    __syncthreads();
    if (sh.err) status = sh.err;

    // ---- a5: rule-B backtrack (one thread; <= M dependent reads) ---------------------------
    int32_t* out = p.pos + (int64_t)e * M;
    if (threadIdx.x == 0) {
      int k = 0;
      if (status == 0 && M > 0) {
        const uint16_t* opt =
            reinterpret_cast<const uint16_t*>(slot + 3 * align256(8 * (size_t)(N + 1)));
        int j = N, m = M;
        while (m > 0 && P[j] > 0) {
          const int s = opt[(size_t)(m - 1) * (N + 1) + j];
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
    if constexpr (F64) {
      // a7: report the definitional cost of the returned placement, compensated (the DP's own
      // V_M carries ~M N eps P_N absolute rounding)
      __syncthreads();
      const int k = sh.red_s[0];
      if (k >= 0 && M > 0) {
        const double v = eval_cost_f64(we, N, out, k, sh);
        if (threadIdx.x == 0) cost[e] = v;
      }
    }
    __syncthreads();
  }
}

}  // namespace sp

static size_t dp_dyn_smem(int N, bool smem_b) {
  size_t s = sp::align256(2 * (size_t)(N + 1));
  if (smem_b) s += sp::align256(4 * (size_t)(N + 1));
  return s;
}

static bool dp_smem_b_fits(int N) {
  return dp_dyn_smem(N, true) + sizeof(sp::Shared) + 1024 <= 227 * 1024;
}

template <typename WT>
static int dp_grid_t(int E, int N) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t dyn = dp_dyn_smem(N, dp_smem_b_fits(N));
  int occ = 1;
  cudaFuncSetAttribute(sp::dp_place_kernel<WT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)dyn);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sp::dp_place_kernel<WT>, sp::DP_NT, dyn);
  if (occ < 1) occ = 1;
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
  return (size_t)dp_grid(n_entries, N) * sp::slot_bytes(N, M);
}

extern "C" sp_status sp_place_checkpoints(const void* weights, sp_weight_type wtype,
                                          int32_t n_entries, int32_t N, int32_t M,
                                          int32_t* positions, int32_t* n_positions, void* cost,
                                          void* cost_by_budget, void* workspace,
                                          size_t workspace_bytes, sp_stream_t stream) {
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
  const size_t need = (size_t)grid * sp::slot_bytes(N, M);
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
  const size_t dyn = dp_dyn_smem(N, p.smem_b);
  cudaStream_t st = (cudaStream_t)stream;
  if (wtype == SP_W_COUNTS_I32) sp::dp_place_kernel<int32_t><<<grid, sp::DP_NT, dyn, st>>>(p);
  else if (wtype == SP_W_COUNTS_I64) sp::dp_place_kernel<int64_t><<<grid, sp::DP_NT, dyn, st>>>(p);
  else sp::dp_place_kernel<double><<<grid, sp::DP_NT, dyn, st>>>(p);
  SP_CHECK_LAUNCH();
  return SP_OK;
}
