// prefix_match.cu -- f4: longest-prefix search of each request over ALL cached entries (the
// trie remark of P:189-190: a request reuses the deepest cached prefix; SPEC match_longest_prefix
// S:375-383).  SURVEY 8(f) f4: the step before a1 in a serving system.
//
// Index (sp_prefix_index_build): the entries sorted lexicographically by their token sequences
// (cub::DeviceMergeSort with a token-comparing functor; ties by entry id, a total order) and a
// sparse table over the sorted order answering "most recent insertion in positions [a, b]" in
// O(1) (level k holds the winner of each 2^k-wide window).
//
// Query (sp_match_longest_prefix), one warp per request, every comparison warp-cooperative
// (32 tokens per step, __ballot_sync + __ffs for the first mismatch, as in a1):
//   1. binary search the request's insertion position p in the sorted order;
//   2. for sorted strings, LCP(S[i], q) is non-decreasing for i < p and non-increasing for
//      i >= p, so the maximum t* is at S[p-1] or S[p];
//   3. the entries reaching t* form the contiguous range [a, b] around p, found by two binary
//      searches that compare only the first t* tokens;
//   4. the most recent of them from the sparse table (ties: larger entry id).
// t* = 0 -> no match (-1, 0).  The depth is the raw LCP (the caller clamps to N, as a1 does).
#include <cub/device/device_merge_sort.cuh>

#include "common.cuh"

namespace sp {

struct TokLess {   // lexicographic order of entries by tokens; a proper prefix first; then by id
  const int32_t* tok;
  const int64_t* off;
  __device__ bool operator()(const int32_t& a, const int32_t& b) const {
    const int32_t* x = tok + off[a];
    const int32_t* y = tok + off[b];
    const int64_t xl = off[a + 1] - off[a], yl = off[b + 1] - off[b];
    const int64_t n = xl < yl ? xl : yl;
    for (int64_t i = 0; i < n; ++i)
      if (x[i] != y[i]) return x[i] < y[i];
    if (xl != yl) return xl < yl;
    return a < b;
  }
};

// the more recent of two entries (insertion value, then entry id)
__device__ __forceinline__ int32_t recent(const int64_t* ins, int32_t a, int32_t b) {
  const int64_t ia = ins ? ins[a] : a, ib = ins ? ins[b] : b;
  return (ib > ia || (ib == ia && b > a)) ? b : a;
}

__global__ void iota_kernel(int32_t* __restrict__ perm, int64_t* __restrict__ ins, int E) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) {
    perm[i] = i;
    if (ins) ins[i] = i;   // no insertion order given: the entry index is the insertion order
  }
}

__global__ void st_level_kernel(const int32_t* __restrict__ perm, const int64_t* ins,
                                int32_t* __restrict__ st, int E, int k) {
  const int w = 1 << k;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) {
    int32_t v;
    if (k == 0) {
      v = perm[i];
    } else {
      const int32_t* prev = st + (size_t)(k - 1) * E;
      v = prev[i];
      if (i + w / 2 < E) v = recent(ins, v, prev[i + w / 2]);
    }
    st[(size_t)k * E + i] = v;
  }
}

// warp-cooperative LCP of x[0..xl) and q[0..ql), capped at cap
__device__ __forceinline__ int64_t warp_lcp(const int32_t* __restrict__ x, int64_t xl,
                                            const int32_t* __restrict__ q, int64_t ql,
                                            int64_t cap) {
  const int lane = lane_id();
  int64_t n = xl < ql ? xl : ql;
  if (cap < n) n = cap;
  for (int64_t base = 0; base < n; base += 32) {
    const int64_t i = base + lane;
    const bool mis = i < n && x[i] != q[i];
    const unsigned bal = __ballot_sync(FULL, mis);
    if (bal) return base + __ffs(bal) - 1;
  }
  return n;
}

// is entry e lexicographically before the request q?  (lcp = their LCP)
__device__ __forceinline__ bool entry_less(const int32_t* x, int64_t xl, const int32_t* q,
                                           int64_t ql, int64_t l) {
  if (l == xl) return xl < ql;   // entry is a prefix of q (equal: not less)
  if (l == ql) return false;     // q is a proper prefix of the entry
  return x[l] < q[l];
}

__global__ void __launch_bounds__(256)
    match_kernel(const int32_t* __restrict__ etok, const int64_t* __restrict__ eoff, int E,
                 const int32_t* __restrict__ perm, const int32_t* __restrict__ st,
                 const int64_t* __restrict__ ins,
                 const int32_t* __restrict__ rtok, const int64_t* __restrict__ roff, int64_t R,
                 int32_t* __restrict__ out_e, int32_t* __restrict__ out_d) {
  const int lane = lane_id();
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + warp_id(); r < R; r += nw) {
    const int32_t* q = rtok + roff[r];
    const int64_t ql = roff[r + 1] - roff[r];
    auto ent = [&](int i, const int32_t*& x, int64_t& xl) {
      const int e = perm[i];
      x = etok + eoff[e];
      xl = eoff[e + 1] - eoff[e];
    };
    // 1. insertion position p = #entries lexicographically before q
    int lo = 0, hi = E;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const int32_t* x;
      int64_t xl;
      ent(mid, x, xl);
      const int64_t l = warp_lcp(x, xl, q, ql, INT64_MAX);
      if (entry_less(x, xl, q, ql, l)) lo = mid + 1; else hi = mid;
    }
    const int p = lo;
    // 2. the maximum LCP is at a neighbour of p
    int64_t tl = 0, tr = 0;
    const int32_t* x;
    int64_t xl;
    if (p > 0) {
      ent(p - 1, x, xl);
      tl = warp_lcp(x, xl, q, ql, INT64_MAX);
    }
    if (p < E) {
      ent(p, x, xl);
      tr = warp_lcp(x, xl, q, ql, INT64_MAX);
    }
    const int64_t ts = tl > tr ? tl : tr;
    int32_t who = -1;
    if (ts > 0) {
      // 3. [a, b]: the entries whose LCP with q reaches ts (contiguous around p)
      int a = p, b = p - 1;
      if (tl == ts) {   // first i in [0, p-1] with LCP >= ts (non-decreasing there)
        int l2 = 0, h2 = p - 1;
        while (l2 < h2) {
          const int mid = (l2 + h2) >> 1;
          ent(mid, x, xl);
          if (warp_lcp(x, xl, q, ql, ts) >= ts) h2 = mid; else l2 = mid + 1;
        }
        a = l2;
        b = p - 1;
      }
      if (tr == ts) {   // last i in [p, E-1] with LCP >= ts (non-increasing there)
        int l2 = p, h2 = E - 1;
        while (l2 < h2) {
          const int mid = (l2 + h2 + 1) >> 1;
          ent(mid, x, xl);
          if (warp_lcp(x, xl, q, ql, ts) >= ts) l2 = mid; else h2 = mid - 1;
        }
        if (tl != ts) a = p;
        b = l2;
      }
      // 4. most recent insertion in [a, b]: two overlapping power-of-two windows
      const int k = 31 - __clz(b - a + 1);
      who = recent(ins, st[(size_t)k * E + a], st[(size_t)k * E + b - (1 << k) + 1]);
    }
    if (lane == 0) {
      out_e[r] = who;
      out_d[r] = (int32_t)ts;
    }
  }
}

}  // namespace sp

// ---- host side -------------------------------------------------------------------------------
// index workspace: perm int32[E] | insertion int64[E] | sparse table int32[levels][E] | cub temp
static int st_levels(int E) { return E > 1 ? 32 - __builtin_clz((unsigned)(E - 1)) + 1 : 1; }
static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }
static size_t cub_sort_bytes(int E) {
  size_t b = 0;
  cub::DeviceMergeSort::SortKeys(nullptr, b, (int32_t*)nullptr, E, sp::TokLess{nullptr, nullptr});
  return b;
}

extern "C" size_t sp_prefix_index_workspace_bytes(int32_t n_entries) {
  if (n_entries < 0) return 0;
  const int E = n_entries;
  return al256(4 * (size_t)E) + al256(8 * (size_t)E) + al256(4 * (size_t)st_levels(E) * E) +
         al256(cub_sort_bytes(E)) + 256;
}

extern "C" sp_status sp_prefix_index_build(const int32_t* entry_tokens, const int64_t* entry_off,
                                           int32_t n_entries, const int64_t* insertion,
                                           void* index, size_t index_bytes, sp_stream_t stream) {
  if (n_entries < 0) return SP_ERR_BAD_LENGTH;
  if (n_entries == 0) return SP_OK;
  if (!entry_off || !index) return SP_ERR_BAD_ARGUMENT;
  const int E = n_entries;
  if (index_bytes < sp_prefix_index_workspace_bytes(E)) return SP_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* w = (uint8_t*)index;
  int32_t* perm = (int32_t*)w;
  int64_t* ins = (int64_t*)(w + al256(4 * (size_t)E));
  int32_t* tab = (int32_t*)(w + al256(4 * (size_t)E) + al256(8 * (size_t)E));
  void* tmp = w + al256(4 * (size_t)E) + al256(8 * (size_t)E) + al256(4 * (size_t)st_levels(E) * E);
  size_t tb = cub_sort_bytes(E);
  // perm = 0..E-1 (a one-level table write doubles as the identity), insertion copy
  if (insertion) {
    if (cudaMemcpyAsync(ins, insertion, 8 * (size_t)E, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      SP_CHECK_LAUNCH();
  }
  sp::iota_kernel<<<(E + 255) / 256, 256, 0, st>>>(perm, insertion ? nullptr : ins, E);
  SP_CHECK_LAUNCH();
  if (cub::DeviceMergeSort::SortKeys(tmp, tb, perm, E, sp::TokLess{entry_tokens, entry_off}, st) !=
      cudaSuccess)
    SP_CHECK_LAUNCH();
  const int L = st_levels(E);
  for (int k = 0; k < L; ++k) {
    int blocks = (E + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    sp::st_level_kernel<<<blocks, 256, 0, st>>>(perm, ins, tab, E, k);
  }
  SP_CHECK_LAUNCH();
  return SP_OK;
}

extern "C" sp_status sp_match_longest_prefix(const int32_t* entry_tokens, const int64_t* entry_off,
                                             int32_t n_entries, const void* index,
                                             const int32_t* req_tokens, const int64_t* req_off,
                                             int64_t n_requests, int32_t* match_entry,
                                             int32_t* match_depth, sp_stream_t stream) {
  if (n_entries < 0 || n_requests < 0) return SP_ERR_BAD_LENGTH;
  if (n_requests == 0) return SP_OK;
  if (!req_off || !match_entry || !match_depth) return SP_ERR_BAD_ARGUMENT;
  if (n_entries > 0 && (!entry_off || !index)) return SP_ERR_BAD_ARGUMENT;
  const int E = n_entries;
  const uint8_t* w = (const uint8_t*)index;
  const int32_t* perm = (const int32_t*)w;
  const int64_t* ins = (const int64_t*)(w + al256(4 * (size_t)E));
  const int32_t* tab = (const int32_t*)(w + al256(4 * (size_t)E) + al256(8 * (size_t)E));
  int64_t blocks = (n_requests + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  sp::match_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      entry_tokens, entry_off, E, perm, tab, E > 0 ? ins : nullptr, req_tokens, req_off,
      n_requests, match_entry, match_depth);
  SP_CHECK_LAUNCH();
  return SP_OK;
}
