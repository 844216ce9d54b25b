// Per-kernel timing with CUDA events recorded on the launching stream, plus a launch counter.
// Used by bench.py to measure the dominant kernel's average launch duration inside the timed region.
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pscwin.h"
#include "prof.h"

namespace pscwin {

namespace {
struct Rec {
  const char* name;
  cudaEvent_t a, b;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
bool g_on = false;
long long g_launches = 0;

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

ProfScope::ProfScope(const char* name, cudaStream_t s) : name_(name), s_(s), a_(nullptr) {
  std::lock_guard<std::mutex> lk(g_mu);
  ++g_launches;
  if (g_on) {
    a_ = get_event();
    cudaEventRecord((cudaEvent_t)a_, s_);
  }
}

ProfScope::~ProfScope() {
  if (!a_) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t b = get_event();
  cudaEventRecord(b, s_);
  g_recs.push_back({name_, (cudaEvent_t)a_, b});
}

}  // namespace pscwin

using namespace pscwin;

extern "C" void pscwin_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = on != 0;
  for (auto& r : g_recs) {
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
}

extern "C" int64_t pscwin_launch_count(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_launches;
}

extern "C" int pscwin_profile_read(char* names, size_t names_len, double* total_ms, int32_t* counts,
                                   int32_t max_entries) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::vector<std::string> keys;
  std::vector<double> ms;
  std::vector<int> cnt;
  for (auto& r : g_recs) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    size_t i = 0;
    for (; i < keys.size(); ++i)
      if (keys[i] == r.name) break;
    if (i == keys.size()) {
      keys.push_back(r.name);
      ms.push_back(0.0);
      cnt.push_back(0);
    }
    ms[i] += t;
    cnt[i] += 1;
  }
  std::string joined;
  int n = (int)keys.size() < max_entries ? (int)keys.size() : max_entries;
  for (int i = 0; i < n; ++i) {
    if (total_ms) total_ms[i] = ms[i];
    if (counts) counts[i] = cnt[i];
    joined += keys[i];
    joined += '\n';
  }
  if (names && names_len) {
    size_t m = joined.size() < names_len - 1 ? joined.size() : names_len - 1;
    memcpy(names, joined.data(), m);
    names[m] = 0;
  }
  return n;
}
