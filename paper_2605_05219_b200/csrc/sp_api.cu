// sp_api.cu -- host-side pieces of the C ABI: status strings, error text, version, and the
// Table 1 baseline generators.
#include <cstdio>
#include <cstring>

#include "common.cuh"

static thread_local char g_last_error[256] = "no error";

extern "C" void sp_set_cuda_error(cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", cudaGetErrorName(e),
           cudaGetErrorString(e));
}

extern "C" const char* sp_last_error_string(void) { return g_last_error; }

extern "C" const char* sp_version(void) { return "sparseprefix 0.1 sm_100a"; }

extern "C" const char* sp_status_string(sp_status s) {
  switch (s) {
    case SP_OK: return "SP_OK";
    case SP_ERR_BAD_LENGTH: return "SP_ERR_BAD_LENGTH";
    case SP_ERR_BUDGET_TOO_LARGE: return "SP_ERR_BUDGET_TOO_LARGE";
    case SP_ERR_BAD_ARGUMENT: return "SP_ERR_BAD_ARGUMENT";
    case SP_ERR_OVERFLOW: return "SP_ERR_OVERFLOW";
    case SP_ERR_BAD_POSITIONS: return "SP_ERR_BAD_POSITIONS";
    case SP_ERR_WORKSPACE: return "SP_ERR_WORKSPACE";
    case SP_ERR_CUDA: return "SP_ERR_CUDA";
    case SP_ERR_INTERNAL: return "SP_ERR_INTERNAL";
  }
  return "SP_ERR_UNKNOWN";
}

// Balanced schedule c_i = floor(i (N+1) / (M+1)), i = 1..M (Table 1; proof P:519-521).
extern "C" int32_t sp_balanced_positions(int32_t N, int32_t M, int32_t* out_host) {
  if (N < 1 || N > SP_MAX_N) return -SP_ERR_BAD_LENGTH;
  if (M < 0 || M > N) return -SP_ERR_BUDGET_TOO_LARGE;
  if (M > 0 && !out_host) return -SP_ERR_BAD_ARGUMENT;
  for (int32_t i = 1; i <= M; ++i) out_host[i - 1] = (int32_t)(((int64_t)i * (N + 1)) / (M + 1));
  return M;
}

// Block schedule B, 2B, ..., floor(N/B) B (Table 1).
extern "C" int32_t sp_block_positions(int32_t N, int32_t B, int32_t* out_host) {
  if (N < 1 || N > SP_MAX_N) return -SP_ERR_BAD_LENGTH;
  if (B < 1) return -SP_ERR_BAD_ARGUMENT;
  const int32_t k = N / B;
  if (k > 0 && !out_host) return -SP_ERR_BAD_ARGUMENT;
  for (int32_t i = 1; i <= k; ++i) out_host[i - 1] = i * B;
  return k;
}
