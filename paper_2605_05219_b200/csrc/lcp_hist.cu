// lcp_hist.cu -- a1 + a2: overlap depth (LCP) of each request with its cache entry and the
// per-entry overlap-depth histogram.
//
// HBM-bound streaming compare.  One warp per request: each lane loads 16 B (4 tokens) of the
// request and of the entry per step, two steps per iteration (256 tokens / warp / iteration,
// 2 KB in flight per warp); the first mismatch is found with __ballot_sync + __ffs and ends the
// request (early exit; the over-read past the mismatch is < 256 tokens).  Request tokens are
// read once (streaming loads, evict-first); entry tokens are re-read by every request of the
// same entry, which the generator/serving order keeps adjacent, so they stay L2-resident.
#include "common.cuh"

namespace sp {

constexpr int LCP_WARPS = 8;

// mismatch bits (bit k set if token q+k < lim differs) for one 4-token group at q (q % 4 == 0
// relative to 16-byte aligned bases a, b).
__device__ __forceinline__ unsigned group_mismatch(const int32_t* __restrict__ a,
                                                   const int32_t* __restrict__ b, int64_t q,
                                                   int64_t lim) {
  if (q + 3 < lim) {
    const int4 va = __ldcs(reinterpret_cast<const int4*>(a + q));
    const int4 vb = __ldg(reinterpret_cast<const int4*>(b + q));
    return (unsigned)(va.x != vb.x) | ((unsigned)(va.y != vb.y) << 1) |
           ((unsigned)(va.z != vb.z) << 2) | ((unsigned)(va.w != vb.w) << 3);
  }
  unsigned m = 0;
  for (int k = 0; k < 4; ++k)
    if (q + k < lim && __ldcs(a + q + k) != __ldg(b + q + k)) m |= 1u << k;
  return m;
}

__global__ void __launch_bounds__(LCP_WARPS * 32)
    lcp_hist_kernel(const int32_t* __restrict__ ent, const int64_t* __restrict__ eoff,
                    int32_t n_entries, const int32_t* __restrict__ req,
                    const int64_t* __restrict__ roff, const int32_t* __restrict__ rent,
                    int64_t n_req, int32_t N, int32_t* __restrict__ hist,
                    int32_t* __restrict__ lcp_out, int vec_ok) {
  const int64_t r = (int64_t)blockIdx.x * LCP_WARPS + warp_id();
  if (r >= n_req) return;
  const int lane = lane_id();
  const int32_t e = __ldg(rent + r);
  if (e < 0 || e >= n_entries) {
    if (lane == 0 && lcp_out) lcp_out[r] = -1;
    return;
  }
  const int64_t eo = __ldg(eoff + e), el = __ldg(eoff + e + 1) - eo;
  const int64_t ro = __ldg(roff + r), rl = __ldg(roff + r + 1) - ro;
  const int64_t lim = min(min(el, rl), (int64_t)N);   // depths clamp to N
  const int32_t* a = req + ro;
  const int32_t* b = ent + eo;
  int64_t t = lim;
  if (vec_ok && ((eo | ro) & 3) == 0) {
    for (int64_t p = 0; p < lim; p += 256) {
      const int64_t q0 = p + 4 * lane, q1 = q0 + 128;
      const unsigned m0 = group_mismatch(a, b, q0, lim);
      const unsigned m1 = group_mismatch(a, b, q1, lim);
      const unsigned b0 = __ballot_sync(FULL, m0 != 0);
      const unsigned b1 = __ballot_sync(FULL, m1 != 0);
      if (b0 | b1) {
        const int f = b0 ? __ffs(b0) - 1 : __ffs(b1) - 1;
        const unsigned mf = __shfl_sync(FULL, b0 ? m0 : m1, f);
        t = p + (b0 ? 0 : 128) + 4 * f + (__ffs(mf) - 1);
        break;
      }
    }
  } else {
    // unaligned rows: coalesced scalar loads, 128 tokens per iteration
    for (int64_t p = 0; p < lim; p += 128) {
      unsigned bits[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t q = p + 32 * k + lane;
        bits[k] = __ballot_sync(FULL, q < lim && __ldcs(a + q) != __ldg(b + q));
      }
      const unsigned any = bits[0] | bits[1] | bits[2] | bits[3];
      if (any) {
        int k = 0;
        while (!bits[k]) ++k;
        t = p + 32 * k + (__ffs(bits[k]) - 1);
        break;
      }
    }
  }
  if (lane == 0) {
    if (hist) atomicAdd(hist + (int64_t)e * (N + 1) + t, 1);
    if (lcp_out) lcp_out[r] = (int32_t)t;
  }
}

__global__ void accumulate_depths_kernel(const int32_t* __restrict__ entry,
                                         const int32_t* __restrict__ depth, int64_t n,
                                         int32_t e_begin, int32_t e_end, int32_t N,
                                         int32_t* __restrict__ hist) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = entry[i], d = depth[i];
    if (e >= e_begin && e < e_end && d >= 0 && d <= N)
      atomicAdd(hist + (int64_t)(e - e_begin) * (N + 1) + d, 1);
  }
}

}  // namespace sp

extern "C" sp_status sp_overlap_hist(const int32_t* entry_tokens, const int64_t* entry_off,
                                     int32_t n_entries, const int32_t* req_tokens,
                                     const int64_t* req_off, const int32_t* req_entry,
                                     int64_t n_requests, int32_t N, int32_t* hist,
                                     int32_t* lcp_out, sp_stream_t stream) {
  if (N < 1 || N > SP_MAX_N || n_entries < 0 || n_requests < 0) return SP_ERR_BAD_LENGTH;
  if (n_requests == 0) return SP_OK;
  if (!entry_tokens || !entry_off || !req_tokens || !req_off || !req_entry || (!hist && !lcp_out))
    return SP_ERR_BAD_ARGUMENT;
  // the 16-byte vector path needs 16-byte aligned token bases (offsets are checked per row)
  const int vec_ok = (((uintptr_t)entry_tokens | (uintptr_t)req_tokens) & 15) == 0;
  const int64_t blocks = (n_requests + sp::LCP_WARPS - 1) / sp::LCP_WARPS;
  if (blocks > 0x7fffffffLL) return SP_ERR_BAD_LENGTH;
  sp::lcp_hist_kernel<<<(unsigned)blocks, sp::LCP_WARPS * 32, 0, (cudaStream_t)stream>>>(
      entry_tokens, entry_off, n_entries, req_tokens, req_off, req_entry, n_requests, N, hist,
      lcp_out, vec_ok);
  SP_CHECK_LAUNCH();
  return SP_OK;
}

extern "C" sp_status sp_accumulate_depths(const int32_t* entry, const int32_t* depth, int64_t n,
                                          int32_t e_begin, int32_t e_end, int32_t N,
                                          int32_t* hist, sp_stream_t stream) {
  if (N < 1 || N > SP_MAX_N || n < 0 || e_end < e_begin) return SP_ERR_BAD_LENGTH;
  if (n == 0 || e_end == e_begin) return SP_OK;
  if (!entry || !depth || !hist) return SP_ERR_BAD_ARGUMENT;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  sp::accumulate_depths_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      entry, depth, n, e_begin, e_end, N, hist);
  SP_CHECK_LAUNCH();
  return SP_OK;
}
