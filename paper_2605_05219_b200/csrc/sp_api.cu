// sp_api.cu -- host-side pieces of the C ABI: status strings, error text, version, and the
// Table 1 baseline generators.
#include <atomic>
#include <cstdio>
#include <cstdlib>
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

// Comparison / test hooks (sp_debug_set in the header): process-wide values read by the launch
// code from atomics -- no getenv on the call path.  Each starts from its environment variable,
// read once (so the tools' SP_* variables keep working).
static std::atomic<int> g_dbg[SP_DBG_COUNT];
static std::atomic<bool> g_dbg_init{false};

static void dbg_init() {
  if (g_dbg_init.load(std::memory_order_acquire)) return;
  static const char* names[SP_DBG_COUNT] = {"SP_NO_HULL", "SP_HULL_LEAN", "SP_HULL_SPLIT",
                                            "SP_HULL_LOGCAP", "SP_HULL_NO_ORDER", "SP_EVAL_PATH"};
  static const int defaults[SP_DBG_COUNT] = {0, 0, -1, 0, 0, 0};
  for (int i = 0; i < SP_DBG_COUNT; ++i) {
    int v = defaults[i];
    if (const char* s = getenv(names[i])) v = atoi(s);
    if (i == SP_DBG_EVAL_PATH) {   // legacy spellings of the evaluation-path hook
      if (getenv("SP_EVAL_CHUNKED")) v = 1;
      if (getenv("SP_EVAL_P32")) v = 2;
      if (getenv("SP_EVAL_PREFIX")) v = 3;
    }
    int expect = 0;
    (void)expect;
    g_dbg[i].store(v, std::memory_order_relaxed);
  }
  g_dbg_init.store(true, std::memory_order_release);
}

extern "C" int sp_debug_get(int flag) {
  if (flag < 0 || flag >= SP_DBG_COUNT) return 0;
  dbg_init();
  return g_dbg[flag].load(std::memory_order_relaxed);
}

extern "C" int sp_debug_set(int flag, int value) {
  if (flag < 0 || flag >= SP_DBG_COUNT) return -SP_ERR_BAD_ARGUMENT;
  dbg_init();
  return g_dbg[flag].exchange(value, std::memory_order_relaxed);
}
