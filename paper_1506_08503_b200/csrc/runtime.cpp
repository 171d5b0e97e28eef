// runtime.cpp -- see runtime.h.
#include "runtime.h"

#include <cstdlib>

namespace gaes {
namespace rt {

thread_local std::string t_err;
std::atomic<uint64_t> g_launches{0};
std::mutex g_name_mu;
std::string g_last_kernel = "";
std::atomic<int> g_num_gpus{0};
std::atomic<int> g_variant{0};
std::atomic<int64_t> g_keys_expanded{0};

int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

void note_kernel(const char* name) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  std::lock_guard<std::mutex> lk(g_name_mu);
  g_last_kernel = name;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::atoi(v);
}

int tune_int(const char* key, int dflt) {
  const char* v = std::getenv("GAES_TUNE");
  if (!v || !*v) return dflt;
  const std::string all(v), k(key);
  size_t pos = 0;
  while (pos < all.size()) {
    size_t end = all.find(',', pos);
    if (end == std::string::npos) end = all.size();
    const std::string item = all.substr(pos, end - pos);
    const size_t eq = item.find('=');
    if (eq != std::string::npos && item.substr(0, eq) == k) return std::atoi(item.c_str() + eq + 1);
    pos = end + 1;
  }
  return dflt;
}

}  // namespace rt
}  // namespace gaes
