// dp_internal.cuh -- internal plumbing between the two DP kernels (dp_hull.cu, dp_place.cu):
// workspace layout and the hull-kernel launch helpers.  Product path only.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

// Workspace head (SP_WS_STATS_BYTES): sp_dp_stats at 0, SP_TIMING counters at 64..127, and two
// internal counters, zeroed by the launch's header memset:
#define SP_WS_FB_COUNT_OFF 192    // unsigned: entries handed from the hull kernel to the D&C
#define SP_WS_ENTRY_CTR_OFF 200   // unsigned: next entry for the hull kernel's warps
#define SP_WS_WIDE_COUNT_OFF 216  // unsigned: entries listed for the int64 hull instantiation
#define SP_WS_WIDE_CTR_OFF 220    // unsigned: next listed entry for the int64 instantiation
#define SP_WS_BIG_COUNT_OFF 224   // unsigned: entries the large-hull mode forwarded to the int64 one
#define SP_WS_BIG_CTR_OFF 228     // unsigned: next listed entry for the large-hull mode

// Workspace after the head:  fallback list int32[E] | int64-path list int32[E] | the large-hull
// mode's forwarded list int32[E] | windowed rings' global arrays (int64 / fp64 instantiations)
// | ordering scratch (support counts, radix sort) | hull slots | D&C slots
// (each 256-B aligned)
int sp_hull_grid(int E, int N, int M, int wtype);
size_t sp_hull_slot_bytes(int N, int M);
size_t sp_hull_wg_bytes(int E, int N, int M);
size_t sp_hull_order_bytes(int E);
cudaError_t sp_hull_launch(const void* weights, int wtype, int E, int N, int M, int32_t* pos,
                           int32_t* npos, void* cost, void* cbb, int32_t* fpos,
                           int32_t* fn, uint8_t* ws, int32_t* fb, int32_t* wide,
                           int32_t* fwd_list, uint8_t* pool, uint8_t* order_ws, uint8_t* slots,
                           int grid, cudaStream_t st);
