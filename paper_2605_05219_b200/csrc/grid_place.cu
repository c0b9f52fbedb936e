// grid_place.cu -- f1: block-aware placement ("clip every checkpoint position to the block
// boundaries", B = 128; P:397 B = 64) -- SURVEY 8(f) f1.
//
// (1) The exact block-restricted DP (S:206-214 candidate_grid).  With checkpoints restricted to
//     multiples of B, a depth t in [kB, (k+1)B) can reuse at most kB, so
//         sum_t c_t (t - l(t;C)) = sum_t c_t (t - B floor(t/B))  +  B sum_k C_k (k - l'(k;C'))
//     with C_k = sum_{t in [kB,(k+1)B)} c_t and C' = C / B: the grid problem IS the unrestricted
//     problem on the block-aggregated histogram C (N' = floor(N/B), M' = min(M, N')), plus a
//     constant.  The order-preserving map k -> kB keeps the canonical (colex-minimal) optimum.
//     So: aggregate (this file), run the DP kernel (dp_place.cu), scale back (this file).
// (2) Post-hoc clipping: floor every position to a multiple of B, drop zeros, merge
//     duplicates -- the paper's measured configuration.
// (3) Host generators for the sqrt(L) and logarithmic (SPEC's reading S:198)
//     baselines.
#include <climits>
#include <cmath>

#include "common.cuh"

namespace sp {

constexpr int GR_NT = 256;

template <typename WT, typename AT>
__global__ void __launch_bounds__(GR_NT)
    grid_aggregate_kernel(const WT* __restrict__ w, int E, int N, int B, AT* __restrict__ agg,
                          AT* __restrict__ cst) {
  __shared__ AT red[GR_NT / 32];
  const int Nb = N / B;
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    const WT* we = w + (int64_t)e * (N + 1);
    AT* ae = agg + (int64_t)e * (Nb + 1);
    AT part = 0;
    for (int k = threadIdx.x; k <= Nb; k += GR_NT) {
      AT sum = 0;
      const int t0 = max(k * B, 1), t1 = (k == Nb) ? N : (k + 1) * B - 1;
      for (int t = t0; t <= t1; ++t) {
        const AT x = (AT)we[t];
        sum += x;
        part += x * (AT)(t - k * B);   // the placement-independent part
      }
      ae[k] = (k == 0) ? (AT)0 : sum;   // depths below B can never reuse a grid checkpoint
    }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
    if (lane_id() == 0) red[warp_id()] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      AT s = 0;
      for (int q = 0; q < GR_NT / 32; ++q) s += red[q];
      cst[e] = s;
    }
    __syncthreads();
  }
}

template <typename CT>
__global__ void grid_finalize_kernel(int E, int M, int Mb, int has_dp, int B,
                                     const int32_t* __restrict__ pos_t,
                                     const int32_t* __restrict__ npos_t, const CT* __restrict__ cost_t,
                                     const CT* __restrict__ cbb_t, const CT* __restrict__ cst,
                                     int32_t* __restrict__ positions, int32_t* __restrict__ n_positions,
                                     CT* __restrict__ cost, CT* __restrict__ cbb) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int k = has_dp ? npos_t[e] : 0;   // negative = per-entry status from the DP
    for (int i = 0; i < M; ++i)
      positions[(int64_t)e * M + i] = (k > 0 && i < k) ? B * pos_t[(int64_t)e * Mb + i] : 0;
    n_positions[e] = k;
    const CT c0 = cst[e];
    cost[e] = (has_dp ? (CT)B * cost_t[e] : (CT)0) + c0;
    if (cbb)
      for (int m = 0; m <= M; ++m)
        cbb[(int64_t)e * (M + 1) + m] =
            (has_dp ? (CT)B * cbb_t[(int64_t)e * (Mb + 1) + min(m, Mb)] : (CT)0) + c0;
  }
}

__global__ void clip_kernel(const int32_t* __restrict__ pos, const int32_t* __restrict__ npos,
                            int E, int max_pos, int B, int32_t* __restrict__ out,
                            int32_t* __restrict__ nout) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int k = npos[e];
    int n = 0, last = 0;
    for (int i = 0; i < k && i < max_pos; ++i) {
      const int f = (pos[(int64_t)e * max_pos + i] / B) * B;   // clip DOWN
      if (f <= 0 || f == last) continue;                      // zeros dropped, duplicates merged
      out[(int64_t)e * max_pos + n++] = f;
      last = f;
    }
    for (int i = n; i < max_pos; ++i) out[(int64_t)e * max_pos + i] = 0;
    nout[e] = k < 0 ? k : n;
  }
}

}  // namespace sp

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" size_t sp_place_checkpoints_grid_workspace_bytes(int32_t n_entries, int32_t N,
                                                            int32_t M, int32_t B) {
  if (N < 1 || N > SP_MAX_N || n_entries < 0 || M < 0 || M > N || B < 1) return 0;
  const int Nb = N / B, Mb = M < Nb ? M : Nb;
  const size_t E = (size_t)n_entries;
  size_t s = al256(E * (Nb + 1) * 8) + al256(E * 8) * 2 + al256(E * (Mb + 1) * 8) +
             al256(E * (Mb > 0 ? Mb : 1) * 4) + al256(E * 4);
  if (Nb >= 1) s += sp_place_checkpoints_workspace_bytes(n_entries, Nb, Mb);
  return s;
}

extern "C" sp_status sp_place_checkpoints_grid(const void* weights, sp_weight_type wtype,
                                               int32_t n_entries, int32_t N, int32_t M, int32_t B,
                                               int32_t* positions, int32_t* n_positions, void* cost,
                                               void* cost_by_budget, void* workspace,
                                               size_t workspace_bytes, sp_stream_t stream) {
  if (N < 1 || N > SP_MAX_N || n_entries < 0) return SP_ERR_BAD_LENGTH;
  if (M < 0 || M > N) return SP_ERR_BUDGET_TOO_LARGE;
  if (B < 1) return SP_ERR_BAD_ARGUMENT;
  if (wtype != SP_W_COUNTS_I32 && wtype != SP_W_COUNTS_I64 && wtype != SP_W_PROB_F64)
    return SP_ERR_BAD_ARGUMENT;
  if (n_entries == 0) return SP_OK;
  if (!weights || !n_positions || !cost || (M > 0 && !positions)) return SP_ERR_BAD_ARGUMENT;
  if (!workspace || workspace_bytes < sp_place_checkpoints_grid_workspace_bytes(n_entries, N, M, B))
    return SP_ERR_WORKSPACE;
  const int Nb = N / B, Mb = M < Nb ? M : Nb;
  const size_t E = (size_t)n_entries;
  const bool f64 = wtype == SP_W_PROB_F64;
  uint8_t* p = (uint8_t*)workspace;
  void* agg = p;          p += al256(E * (Nb + 1) * 8);
  void* cst = p;          p += al256(E * 8);
  void* cost_t = p;       p += al256(E * 8);
  void* cbb_t = p;        p += al256(E * (Mb + 1) * 8);
  int32_t* pos_t = (int32_t*)p; p += al256(E * (Mb > 0 ? Mb : 1) * 4);
  int32_t* npos_t = (int32_t*)p; p += al256(E * 4);
  void* dpws = p;
  const size_t dpws_bytes = workspace_bytes - (size_t)(p - (uint8_t*)workspace);
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = n_entries < sms * 8 ? n_entries : sms * 8;
  if (wtype == SP_W_COUNTS_I32)
    sp::grid_aggregate_kernel<int32_t, int64_t><<<grid, sp::GR_NT, 0, st>>>(
        (const int32_t*)weights, n_entries, N, B, (int64_t*)agg, (int64_t*)cst);
  else if (wtype == SP_W_COUNTS_I64)
    sp::grid_aggregate_kernel<int64_t, int64_t><<<grid, sp::GR_NT, 0, st>>>(
        (const int64_t*)weights, n_entries, N, B, (int64_t*)agg, (int64_t*)cst);
  else
    sp::grid_aggregate_kernel<double, double><<<grid, sp::GR_NT, 0, st>>>(
        (const double*)weights, n_entries, N, B, (double*)agg, (double*)cst);
  SP_CHECK_LAUNCH();
  if (Nb >= 1) {
    const sp_status s = sp_place_checkpoints(agg, f64 ? SP_W_PROB_F64 : SP_W_COUNTS_I64,
                                             n_entries, Nb, Mb, Mb > 0 ? pos_t : nullptr, npos_t,
                                             cost_t, cbb_t, dpws, dpws_bytes, stream);
    if (s != SP_OK) return s;
  }
  const int fg = (n_entries + 255) / 256;
  if (f64)
    sp::grid_finalize_kernel<double><<<fg, 256, 0, st>>>(
        n_entries, M, Mb, Nb >= 1 ? 1 : 0, B, pos_t, npos_t, (const double*)cost_t,
        (const double*)cbb_t, (const double*)cst, positions, n_positions, (double*)cost,
        (double*)cost_by_budget);
  else
    sp::grid_finalize_kernel<int64_t><<<fg, 256, 0, st>>>(
        n_entries, M, Mb, Nb >= 1 ? 1 : 0, B, pos_t, npos_t, (const int64_t*)cost_t,
        (const int64_t*)cbb_t, (const int64_t*)cst, positions, n_positions, (int64_t*)cost,
        (int64_t*)cost_by_budget);
  SP_CHECK_LAUNCH();
  return SP_OK;
}

extern "C" sp_status sp_clip_to_blocks(const int32_t* positions, const int32_t* n_positions,
                                       int32_t n_entries, int32_t max_pos, int32_t B,
                                       int32_t* out_positions, int32_t* out_n, sp_stream_t stream) {
  if (n_entries < 0 || max_pos < 0) return SP_ERR_BAD_LENGTH;
  if (B < 1) return SP_ERR_BAD_ARGUMENT;
  if (n_entries == 0) return SP_OK;
  if (!n_positions || !out_n || (max_pos > 0 && (!positions || !out_positions)))
    return SP_ERR_BAD_ARGUMENT;
  sp::clip_kernel<<<(n_entries + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      positions, n_positions, n_entries, max_pos, B, out_positions, out_n);
  SP_CHECK_LAUNCH();
  return SP_OK;
}

// sqrt(L) schedule: multiples of floor(sqrt(N)) up to N (Table 1)
extern "C" int32_t sp_sqrt_positions(int32_t N, int32_t* out_host) {
  if (N < 1 || N > SP_MAX_N) return -SP_ERR_BAD_LENGTH;
  int32_t q = 1;
  while ((int64_t)(q + 1) * (q + 1) <= N) ++q;
  return sp_block_positions(N, q, out_host);
}

// logarithmic schedule (SPEC's reading S:198): round(N (2^i - 1) / (2^M - 1)), i = 1..M,
// clamped to [1, N], duplicates dropped -- dense near the start, gaps growing geometrically
extern "C" int32_t sp_log_positions(int32_t N, int32_t M, int32_t* out_host) {
  if (N < 1 || N > SP_MAX_N) return -SP_ERR_BAD_LENGTH;
  if (M < 1 || M > N || M > 62) return -SP_ERR_BUDGET_TOO_LARGE;
  if (!out_host) return -SP_ERR_BAD_ARGUMENT;
  const __int128 den = ((__int128)1 << M) - 1;
  int32_t n = 0;
  for (int32_t i = 1; i <= M; ++i) {
    const __int128 num = (__int128)N * (((__int128)1 << i) - 1);
    int64_t r = (int64_t)((2 * num + den) / (2 * den));
    if (r < 1) r = 1;
    if (r > N) r = N;
    if (n > 0 && out_host[n - 1] >= r) continue;
    out_host[n++] = (int32_t)r;
  }
  return n;
}
