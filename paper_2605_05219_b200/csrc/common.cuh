// common.cuh -- small device helpers shared by the libsparseprefix kernels (product path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sparse_prefix.h"

namespace sp {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Block-wide exclusive scan of one int64 per thread.  `warp_buf` needs NT/32 int64 slots.
// Returns the exclusive prefix; *total receives the block total.  Contains 3 __syncthreads.
template <int NT>
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t x, int64_t* warp_buf,
                                                        int64_t* total) {
  constexpr int NW = NT / 32;
  const int lane = lane_id(), w = warp_id();
  int64_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  __syncthreads();  // warp_buf may still be read by a previous call
  if (lane == 31) warp_buf[w] = inc;
  __syncthreads();
  if (w == 0) {
    int64_t v = lane < NW ? warp_buf[lane] : 0;
    int64_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(FULL, vi, o);
      if (lane >= o) vi += y;
    }
    if (lane < NW) warp_buf[lane] = vi - v;   // exclusive warp offsets
    if (lane == NW - 1) warp_buf[NW] = vi;    // block total
  }
  __syncthreads();
  int64_t r = warp_buf[w] + inc - x;
  *total = warp_buf[NW];
  return r;
}

template <int NT>
__device__ __forceinline__ int64_t block_sum(int64_t x, int64_t* warp_buf) {
  int64_t t;
  block_exclusive_scan<NT>(x, warp_buf, &t);
  return t;
}

}  // namespace sp

// host-side error plumbing (sp_api.cu)
extern "C" void sp_set_cuda_error(cudaError_t e);
#define SP_CHECK_LAUNCH()                          \
  do {                                             \
    cudaError_t _e = cudaGetLastError();           \
    if (_e != cudaSuccess) {                       \
      sp_set_cuda_error(_e);                       \
      return SP_ERR_CUDA;                          \
    }                                              \
  } while (0)
