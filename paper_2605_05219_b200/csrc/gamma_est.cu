// gamma_est.cu -- f2: the exponentially weighted empirical overlap histogram of Thm 4
// (P:323-352), batched over cache entries; it is the estimator the paper's method re-solves the
// placement from ("gamma = 0.99, re-solving and updating the histogram every 10 requests").
// SURVEY 8(f) f2.
//
//   p_t = (1 - g) / (1 - g^t) * sum_{s=1..t} g^(t-s) e_{T_s}          (g = 1: 1/t)
//
// Global-scale representation (one row per entry, never an O(N) sweep per observation): the row
// W[e][.] holds the weights relative to a reference epoch tau, w = W * g^(t - tau).  Observation
// number t+1 (depth d) makes w' = g w + e_d, i.e. W[d] += g^-(t + 1 - tau).  When the exponent's
// magnitude would pass 2^64 the row is rescaled by g^(t - tau) and tau = t.  The decayed weights
// differ from p_t by a per-entry positive factor, so the fp64 DP (argmin scale-invariant)
// can be run on W directly; sp_gamma_snapshot returns the normalised p_t.
//
// One warp per entry (grid-stride): lanes take the entry's observations of the batch in chunks
// whose exponents stay below 2^64, add their increments with fp64 atomics, and the warp rescales
// the row between chunks when needed.  Misses (depth < 1) are not samples of T (reading R15).
#include <cmath>

#include "common.cuh"

namespace sp {

constexpr int GE_NT = 256;

__global__ void __launch_bounds__(GE_NT)
    gamma_observe_kernel(double* __restrict__ W, int64_t* __restrict__ tcount,
                         int64_t* __restrict__ tau, const int64_t* __restrict__ obs_off,
                         const int32_t* __restrict__ depth, int E, int N, double g, double lg2inv,
                         int chunk) {
  const int lane = lane_id();
  const int nw = gridDim.x * (GE_NT / 32);
  for (int e = blockIdx.x * (GE_NT / 32) + warp_id(); e < E; e += nw) {
    const int64_t o0 = obs_off[e], n = obs_off[e + 1] - o0;
    if (n <= 0) continue;
    double* row = W + (int64_t)e * (N + 1);
    int64_t t = tcount[e], ta = tau[e];
    for (int64_t c0 = 0; c0 < n; c0 += chunk) {
      const int64_t c1 = min(n, c0 + (int64_t)chunk);
      // rescale first if this chunk's exponents would pass 2^64 (never for g = 1)
      if (g < 1.0 && (double)(t + (c1 - c0) - ta) * lg2inv > 64.0) {
        const double sc = pow(g, (double)(t - ta));
        __syncwarp();
        for (int d = lane; d <= N; d += 32) row[d] *= sc;
        __syncwarp();
        ta = t;
      }
      // only hits are samples (T in {1..N}; conditioning on hits; reading
      // R15): a miss (depth < 1) neither adds weight nor advances t, so each hit's exponent is
      // its rank among the hits (ballot + popc over each 32-observation group)
      const unsigned lt = (1u << lane) - 1u;
      for (int64_t i0 = c0; i0 < c1; i0 += 32) {
        const int64_t i = i0 + lane;
        int d = i < c1 ? depth[o0 + i] : 0;
        const bool hit = d >= 1;
        const unsigned bal = __ballot_sync(FULL, hit);
        if (hit) {
          d = d > N ? N : d;   // clamp
          const int64_t x = t + __popc(bal & lt) + 1 - ta;
          const double inc = g < 1.0 ? pow(g, -(double)x) : 1.0;
          atomicAdd(row + d, inc);
        }
        t += __popc(bal);
      }
      __syncwarp();
    }
    if (lane == 0) {
      tcount[e] = t;
      tau[e] = ta;
    }
  }
}

__global__ void __launch_bounds__(GE_NT)
    gamma_snapshot_kernel(const double* __restrict__ W, const int64_t* __restrict__ tcount,
                          const int64_t* __restrict__ tau, int E, int N, double g,
                          double* __restrict__ p) {
  const int64_t total = (int64_t)E * (N + 1);
  for (int64_t k = (int64_t)blockIdx.x * GE_NT + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * GE_NT) {
    const int e = (int)(k / (N + 1));
    const int64_t t = tcount[e];
    double s = 0.0;
    if (t > 0) s = g < 1.0 ? pow(g, (double)(t - tau[e])) * (1.0 - g) / (1.0 - pow(g, (double)t))
                           : 1.0 / (double)t;
    p[k] = W[k] * s;
  }
}

}  // namespace sp

static bool bad_gamma(double g) { return !(g > 0.0 && g <= 1.0); }

extern "C" sp_status sp_gamma_observe(double* W, int64_t* t, int64_t* tau, const int64_t* obs_off,
                                      const int32_t* depth, int32_t n_entries, int32_t N,
                                      double gamma, sp_stream_t stream) {
  if (N < 1 || N > SP_MAX_N || n_entries < 0) return SP_ERR_BAD_LENGTH;
  if (bad_gamma(gamma)) return SP_ERR_BAD_ARGUMENT;
  if (n_entries == 0) return SP_OK;
  if (!W || !t || !tau || !obs_off) return SP_ERR_BAD_ARGUMENT;   // depth: NULL iff batch empty
  const double lg2inv = gamma < 1.0 ? -log2(gamma) : 0.0;
  // observations per chunk so that a chunk spans at most 2^32 of exponent range
  int chunk = 1 << 20;
  if (gamma < 1.0) chunk = (int)std::fmax(1.0, std::fmin((double)(1 << 20), 32.0 / lg2inv));
  int blocks = (n_entries + sp::GE_NT / 32 - 1) / (sp::GE_NT / 32);
  if (blocks > 148 * 16) blocks = 148 * 16;
  sp::gamma_observe_kernel<<<blocks, sp::GE_NT, 0, (cudaStream_t)stream>>>(
      W, t, tau, obs_off, depth, n_entries, N, gamma, lg2inv, chunk);
  SP_CHECK_LAUNCH();
  return SP_OK;
}

extern "C" sp_status sp_gamma_snapshot(const double* W, const int64_t* t, const int64_t* tau,
                                       int32_t n_entries, int32_t N, double gamma, double* p_out,
                                       sp_stream_t stream) {
  if (N < 1 || N > SP_MAX_N || n_entries < 0) return SP_ERR_BAD_LENGTH;
  if (bad_gamma(gamma)) return SP_ERR_BAD_ARGUMENT;
  if (n_entries == 0) return SP_OK;
  if (!W || !t || !tau || !p_out) return SP_ERR_BAD_ARGUMENT;
  const int64_t total = (int64_t)n_entries * (N + 1);
  int64_t blocks = (total + sp::GE_NT - 1) / sp::GE_NT;
  if (blocks > 148 * 32) blocks = 148 * 32;
  sp::gamma_snapshot_kernel<<<(unsigned)blocks, sp::GE_NT, 0, (cudaStream_t)stream>>>(
      W, t, tau, n_entries, N, gamma, p_out);
  SP_CHECK_LAUNCH();
  return SP_OK;
}
