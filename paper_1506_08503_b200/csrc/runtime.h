// runtime.h -- internal host runtime of libgaes_b200.so shared by its
// translation units: per-thread error state, launch accounting, environment
// knobs and the reference's ShiftRows source tables.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>

#include "../../include/gaes_b200.h"

namespace gaes {
namespace rt {

constexpr int kVersion = 10000;  // 1.0.0
inline constexpr uint8_t kShiftRowsSrc[16] = {0, 5, 10, 15, 4, 9, 14, 3, 8, 13, 2, 7, 12, 1, 6, 11};  // aes_cbc.py:41
inline constexpr uint8_t kInvShiftRowsSrc[16] = {0, 13, 10, 7, 4, 1, 14, 11, 8, 5, 2, 15, 12, 9, 6, 3};  // :42

extern thread_local std::string t_err;   // gaes_last_error() of this thread
extern std::atomic<uint64_t> g_launches;  // gaes_launch_count()
extern std::mutex g_name_mu;
extern std::string g_last_kernel;         // gaes_last_kernel()
extern std::atomic<int> g_num_gpus;       // gaes_set_num_gpus()
extern std::atomic<int> g_variant;        // gaes_set_variant()
extern std::atomic<int64_t> g_keys_expanded;  // keys expanded by host many-key jobs (gaes_debug_counters)

// Records msg as this thread's last error and returns code.
int fail(int code, const std::string& msg);
// Counts one launch of `name` (bench.py's gpu_launches).
void note_kernel(const char* name);
int env_int(const char* name, int dflt);
// Measurement-only overrides of the settled tuning choices, all through one
// variable: GAES_TUNE="KEY=VALUE,KEY=VALUE" (keys: PDL, EARLY, ILP, TEXS,
// TEXIN, ROWS_TMA, ROWS_TMA_MIN_GROUPS, NT, MEMCPY_GRAIN_KB, ZEROCOPY_MB,
// SMALL_ZEROCOPY_KB, SMALL_BLOCKS_PER_SM, ROWS_QUAD, CHUNK_MB, PAGEABLE_CHUNK_MB,
// LANES).  Unset in normal
// use: the defaults are the measured choices.  Returns `dflt`
// for keys not given.
int tune_int(const char* key, int dflt);

}  // namespace rt
}  // namespace gaes

#define GAES_CK(expr)                                                                                      \
  do {                                                                                                     \
    cudaError_t e_ = (expr);                                                                               \
    if (e_ != cudaSuccess)                                                                                 \
      return ::gaes::rt::fail(GAES_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));             \
  } while (0)
