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
// The only dependency between layers is e_{m-1}(j-1) -> b_j of layer m.  So every layer can
// advance one row per step in lockstep: lane l of the warp owns layers l+1 and l+33 (K = 2
// slots; K = 1 when M <= 32), and at step j it receives e_{m-1}(j-1) -- produced by the lane
// below at step j-1 -- with one shuffle.  One warp solves one entry; a step costs O(1)
// amortised per layer (the paper's bound), with no barriers, no brackets and no D&C levels.
// M > 64 runs in passes of 64 layers chained through a global e-row buffer.
//
// Each layer's deque lives in shared memory as a ring of HC lines, interleaved across lanes
// ([pos][slot][lane]) so that every lane hits its own bank whatever its deque position.  The
// rings hold the live hull, which is small for histogram-shaped inputs (tools/hull_stats:
// <= 51 lines on W5); an entry whose hull outgrows a ring (e.g. the all-ones histogram, whose
// layer-1 hull holds ~N/2 lines) is handed to the divide-and-conquer kernel (dp_place.cu) in
// the same launch sequence, as are entries needing int64 / fp64 arithmetic.
//
// Outputs per entry: the argmin table (uint16, [pass][j][lane][slot], 2 B per cell) in the
// warp's workspace slot; V_m = T_N + e_m(N) for every m (cost_by_budget); the rule-B backtrack
// (positions, count) by lane 0; the f3 frontier by all lanes.
#include <climits>

#include "common.cuh"
#include "dp_internal.cuh"

namespace sp {

#ifndef SP_HULL_CAP
#define SP_HULL_CAP 64
#endif
constexpr int HC = SP_HULL_CAP;   // ring capacity per layer (power of two)
static_assert((HC & (HC - 1)) == 0, "ring capacity must be a power of two");

__host__ __device__ __forceinline__ size_t hull_align(size_t x) { return (x + 255) & ~(size_t)255; }
__host__ __device__ __forceinline__ int hull_K(int M) { return M > 32 ? 2 : 1; }
__host__ __device__ __forceinline__ int hull_passes(int M) {
  const int L = 32 * hull_K(M);
  return (M + L - 1) / L;
}
// slot: opt table [passes][N+1][32K] uint16 | e-row buffers 2 x int32[N+1]
__host__ __device__ __forceinline__ size_t hull_opt_bytes(int N, int M) {
  return hull_align((size_t)hull_passes(M) * (N + 1) * 32 * hull_K(M) * 2);
}
__host__ __device__ __forceinline__ size_t hull_slot_bytes(int N, int M) {
  return hull_opt_bytes(N, M) + 2 * hull_align(4 * (size_t)(N + 1));
}
__host__ __device__ __forceinline__ size_t hull_smem_bytes(int M) {
  return (size_t)HC * 32 * hull_K(M) * 8;   // int2 (b, s) per line
}

struct HullParams {
  const void* w;
  int E, N, M;
  int32_t* pos;
  int32_t* npos;
  int64_t* cost;
  int64_t* cbb;
  int32_t* fpos;
  int32_t* fn;
  uint8_t* ws;      // workspace head (stats + counters)
  int32_t* fb;      // fallback entry list
  uint8_t* slots;   // per-warp slots
  size_t slot;
};

// back-pop test, all int32 inputs exact (|b| <= nN < 2^30, so differences fit int32):
// the back line (s2, b2) goes if it is not strictly below the segment (s1, b1) -> (j, bj),
// i.e. (bj - b1)(s2 - s1) <= (b2 - b1)(j - s1).  Products < 2^46 in int64.
__device__ __forceinline__ bool back_dominated(int db_new, int ds_old, int db_old, int ds_new) {
  return (long long)db_new * ds_old <= (long long)db_old * ds_new;
}

// opt table element of layer q (0-based within its pass) at row j
__device__ __forceinline__ int hull_opt_at(const uint16_t* T, int N, int K, int m, int j) {
  const int L = 32 * K;
  const int p = (m - 1) / L, q = (m - 1) % L;
  return T[((size_t)p * (N + 1) + j) * L + (q & 31) * K + (q >> 5)];
}

template <typename WT, int K>
__global__ void __launch_bounds__(32) dp_hull_kernel(HullParams p) {
  extern __shared__ __align__(16) int2 ring[];   // [HC][K][32] lines (b, s)
  const int lane = threadIdx.x;
  const int N = p.N, M = p.M;
  constexpr int L = 32 * K;
  const int passes = (M + L - 1) / L;
  sp_dp_stats* stats = reinterpret_cast<sp_dp_stats*>(p.ws);
  unsigned* fb_n = reinterpret_cast<unsigned*>(p.ws + SP_WS_FB_COUNT_OFF);
  unsigned* ectr = reinterpret_cast<unsigned*>(p.ws + SP_WS_ENTRY_CTR_OFF);
  uint8_t* slot = p.slots + (size_t)blockIdx.x * p.slot;
  uint16_t* optT = reinterpret_cast<uint16_t*>(slot);
  int32_t* ebuf0 = reinterpret_cast<int32_t*>(slot + hull_opt_bytes(N, M));
  int32_t* ebuf1 = reinterpret_cast<int32_t*>(slot + hull_opt_bytes(N, M) + hull_align(4 * (size_t)(N + 1)));
  unsigned long long tests = 0;
  int done_entries = 0;

  for (;;) {
    int e = 0;
    if (lane == 0) e = (int)atomicAdd(ectr, 1u);
    e = __shfl_sync(FULL, e, 0);
    if (e >= p.E) break;
    const WT* we = reinterpret_cast<const WT*>(p.w) + (int64_t)e * (N + 1);

    // ---- a3 pre-pass: n = P_N, T_N, first non-zero bin, sign / size guards ---------------
    long long n = 0, TN = 0;
    int bad = 0, tfirst = INT_MAX;
    for (int t = lane + 1; t <= N; t += 32) {
      const long long c = (long long)we[t];
      bad |= (c < 0) | (c >= (1ll << 30));
      if (!bad) {
        n += c;
        TN += (long long)t * c;
      }
      if (c > 0 && t < tfirst) tfirst = t;
    }
    bad = __any_sync(FULL, bad);
    n = warp_sum(n);
    TN = warp_sum(TN);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tfirst = min(tfirst, __shfl_xor_sync(FULL, tfirst, o));
    // exact-int32 guard 2 n N < 2^31 (the D&C kernel's "narrow" condition); else fall back
    if (bad || n >= (1ll << 30) / N) {
      if (lane == 0) p.fb[atomicAdd(fb_n, 1u)] = e;
      continue;
    }
    if (lane == 0) {
      if (p.cbb) p.cbb[(int64_t)e * (M + 1)] = TN;   // V_0 = T_N
    }

    // ---- a4: all layers in lockstep, one row per step ---------------------------------------
    bool ovf = false;
    unsigned tests_e = 0;
    for (int ps = 0; ps < passes && !ovf; ++ps) {
      const int32_t* ein = (ps & 1) ? ebuf1 : ebuf0;    // e_{64 ps}(.) from the previous pass
      int32_t* eout_buf = (ps & 1) ? ebuf0 : ebuf1;
      const bool chain_in = ps > 0, chain_out = ps + 1 < passes;
      // Per slot: deque [f, b] (monotone counters; ring index & (HC-1)).  Cached in registers:
      // B0 = line b (back), B1 = line b-1, X1 = line b-2, X2 = line b-3 (prefetched after the
      // push), F0 = line f (front), F1 = line f+1.  A line is int2 (x = intercept b_s, y = s).
      int f[K], b[K], eo[K], mlay[K];
      int2 B0[K], B1[K], X1[K], X2[K], F0[K], F1[K];
      bool act[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        mlay[k] = ps * L + 32 * k + lane + 1;
        act[k] = mlay[k] <= M;
        f[k] = 0;
        b[k] = -1;
        eo[k] = 0;   // e_m(0) = 0 (reading R1)
        B0[k] = B1[k] = X1[k] = X2[k] = F0[k] = F1[k] = make_int2(0, 1);
      }
      if (chain_out && lane == 0) eout_buf[0] = 0;
      int32_t carry = 0, Pm1 = 0;
      uint16_t* optP = optT + (size_t)ps * (N + 1) * L;
      for (int jb = 0; jb < N; jb += 32) {
        const int jr = jb + 1 + lane;
        int32_t cnt = jr <= N ? (int32_t)we[jr] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(FULL, cnt, o);
          if (lane >= o) cnt += y;
        }
        const int32_t Pc = carry + cnt;
        carry = __shfl_sync(FULL, Pc, 31);
        int32_t Ec = 0;
        if (chain_in && jr <= N) Ec = ein[jr - 1];
        const int nstep = min(32, N - jb);
        for (int i = 0; i < nstep; ++i) {
          const int j = jb + 1 + i;
          const int32_t Pj = __shfl_sync(FULL, Pc, i);
          // e_{m-1}(j-1): from the lane below (previous step); lane 0 slot 0 from outside
          int32_t in[K];
          const int32_t t0 = __shfl_sync(FULL, eo[0], (lane + 31) & 31);
          const int32_t ext = chain_in ? __shfl_sync(FULL, Ec, i) : 0;
          in[0] = lane ? t0 : ext;
          if constexpr (K == 2) {
            const int32_t t1 = __shfl_sync(FULL, eo[1], (lane + 31) & 31);
            in[1] = lane ? t1 : t0;
          }
          // (1) back tests for both slots, branch-free: up to three pops from registers
          int bj[K], npop[K];
          bool more[K];
#pragma unroll
          for (int k = 0; k < K; ++k) {
            bj[k] = in[k] + j * Pm1;
            const int sz = b[k] - f[k] + 1;   // deque size before the push
            const bool t1 = sz >= 2 && back_dominated(bj[k] - B1[k].x, B0[k].y - B1[k].y,
                                                      B0[k].x - B1[k].x, j - B1[k].y);
            const bool t2 = sz >= 3 && back_dominated(bj[k] - X1[k].x, B1[k].y - X1[k].y,
                                                      B1[k].x - X1[k].x, j - X1[k].y);
            const bool t3 = sz >= 4 && back_dominated(bj[k] - X2[k].x, X1[k].y - X2[k].y,
                                                      X1[k].x - X2[k].x, j - X2[k].y);
            npop[k] = t1 ? (t2 ? (t3 ? 3 : 2) : 1) : 0;
            more[k] = act[k] && t1 && t2 && t3;
          }
          // (2) push line j (rare: more than three pops -> keep popping from the ring)
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (!act[k]) continue;
            int2 nb1 = npop[k] == 0 ? B0[k] : npop[k] == 1 ? B1[k] : npop[k] == 2 ? X1[k] : X2[k];
            int top = b[k] - npop[k];   // index of the new second-to-back line
            if (more[k]) {
              int2* rk = ring + k * 32 + lane;
              while (top - f[k] >= 1) {
                const int2 l1 = rk[((top - 1) & (HC - 1)) * L];
                if (back_dominated(bj[k] - l1.x, nb1.y - l1.y, nb1.x - l1.x, j - l1.y)) {
                  --top;
                  nb1 = l1;
                  ++npop[k];
                } else {
                  break;
                }
              }
            }
            tests_e += (unsigned)npop[k];
            const int nb = top + 1;
            const int2 nl = make_int2(bj[k], j);
            int2* rk = ring + k * 32 + lane;
            rk[(nb & (HC - 1)) * L] = nl;
            if (nb == f[k]) F0[k] = nl;                // the deque was empty (first row)
            if (nb == f[k] + 1) F1[k] = nl;            // line f+1 was popped or is new
            B1[k] = nb1;
            B0[k] = nl;
            b[k] = nb;
            ovf |= (nb - f[k]) >= HC;
            X1[k] = rk[((nb - 2) & (HC - 1)) * L];     // prefetch for the next step's tests
            X2[k] = rk[((nb - 3) & (HC - 1)) * L];
          }
          // (3) query x = P_j: pop the front while the next line is strictly better
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (!act[k]) continue;
            int v0 = F0[k].x - F0[k].y * Pj;
            int v1 = F1[k].x - F1[k].y * Pj;
            if (f[k] < b[k] && v1 < v0) {   // rare
              int2* rk = ring + k * 32 + lane;
              do {
                ++f[k];
                ++tests_e;
                F0[k] = F1[k];
                v0 = v1;
                if (f[k] < b[k]) {
                  F1[k] = rk[((f[k] + 1) & (HC - 1)) * L];
                  v1 = F1[k].x - F1[k].y * Pj;
                }
              } while (f[k] < b[k] && v1 < v0);
            }
            eo[k] = v0;
          }
          // argmin row j of this pass: [j][lane][slot]
          if constexpr (K == 2) {
            reinterpret_cast<uint32_t*>(optP + (size_t)j * L)[lane] =
                (uint32_t)F0[0].y | ((uint32_t)F0[1].y << 16);
          } else {
            optP[(size_t)j * L + lane] = (uint16_t)F0[0].y;
          }
          if (chain_out && lane == 31) eout_buf[j] = eo[K - 1];
          Pm1 = Pj;
        }
        if (__any_sync(FULL, ovf)) {
          ovf = true;
          break;
        }
      }
      if (!ovf) {   // V_m = T_N + e_m(N)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (!act[k]) continue;
          const long long V = TN + (long long)eo[k];
          if (p.cbb) p.cbb[(int64_t)e * (M + 1) + mlay[k]] = V;
          if (mlay[k] == M) p.cost[e] = V;
        }
      }
      __syncwarp();   // chained e-row visible to the next pass
    }
    tests += tests_e;
    if (ovf) {
      if (lane == 0) p.fb[atomicAdd(fb_n, 1u)] = e;
      continue;
    }
    __syncwarp();   // the argmin table is complete and visible to every lane

    // ---- a5: rule-B backtrack (reading R3): lane 0 for budget M, all lanes for the frontier
    if (lane == 0) {
      int32_t* out = p.pos + (int64_t)e * M;
      int k = 0, j = N, m = M;
      while (m > 0 && j >= tfirst) {   // P_j > 0  <=>  j >= first non-zero bin
        const int s = hull_opt_at(optT, N, K, m, j);
        out[k++] = s;
        j = s - 1;
        --m;
      }
      for (int a = 0, z = k - 1; a < z; ++a, --z) {
        const int t = out[a];
        out[a] = out[z];
        out[z] = t;
      }
      for (int q = k; q < M; ++q) out[q] = 0;
      p.npos[e] = k;
    }
    if (p.fpos) {
      for (int mb = lane + 1; mb <= M; mb += 32) {
        int32_t* fo = p.fpos + ((int64_t)e * M + (mb - 1)) * M;
        int k = 0, j = N, m = mb;
        while (m > 0 && j >= tfirst) {
          const int s = hull_opt_at(optT, N, K, m, j);
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
  tests = warp_sum(tests);
  if (lane == 0) {
    atomicAdd(&stats->hull_tests, tests);
    atomicAdd(&stats->entries_hull, (unsigned long long)done_entries);
    atomicAdd(&stats->entries_i32, (unsigned long long)done_entries);
  }
}

template <typename WT, int K>
static int hull_grid_t(int E, int M) {
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t dyn = hull_smem_bytes(M);
  cudaFuncSetAttribute(dp_hull_kernel<WT, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dp_hull_kernel<WT, K>, 32, dyn);
  if (occ < 1) occ = 1;
  long g = (long)sms * occ;
  if (g > E) g = E;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace sp

int sp_hull_grid(int E, int N, int M, int wtype) {
  (void)N;
  const bool k2 = sp::hull_K(M) == 2;
  if (wtype == SP_W_COUNTS_I64)
    return k2 ? sp::hull_grid_t<int64_t, 2>(E, M) : sp::hull_grid_t<int64_t, 1>(E, M);
  return k2 ? sp::hull_grid_t<int32_t, 2>(E, M) : sp::hull_grid_t<int32_t, 1>(E, M);
}

size_t sp_hull_slot_bytes(int N, int M) { return sp::hull_slot_bytes(N, M); }

cudaError_t sp_hull_launch(const void* weights, int wtype, int E, int N, int M, int32_t* pos,
                           int32_t* npos, int64_t* cost, int64_t* cbb, int32_t* fpos,
                           int32_t* fn, uint8_t* ws, int32_t* fb, uint8_t* slots, int grid,
                           cudaStream_t st) {
  sp::HullParams p;
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
  const size_t dyn = sp::hull_smem_bytes(M);
  const bool k2 = sp::hull_K(M) == 2;
  if (wtype == SP_W_COUNTS_I64) {
    if (k2) sp::dp_hull_kernel<int64_t, 2><<<grid, 32, dyn, st>>>(p);
    else sp::dp_hull_kernel<int64_t, 1><<<grid, 32, dyn, st>>>(p);
  } else {
    if (k2) sp::dp_hull_kernel<int32_t, 2><<<grid, 32, dyn, st>>>(p);
    else sp::dp_hull_kernel<int32_t, 1><<<grid, 32, dyn, st>>>(p);
  }
  return cudaGetLastError();
}
