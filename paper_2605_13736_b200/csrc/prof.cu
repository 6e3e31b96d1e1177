// prof.cu — launch counter and per-kernel-class CUDA-event timing (used by
// bench.py to measure the dominant kernel's average launch duration on the
// stream it is launched on; off by default, never active during graph capture).
#include <algorithm>
#include <atomic>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

bool g_mds_prof = false;
static std::atomic<unsigned long long> g_launches{0};
static std::mutex g_mu;
struct Rec { int cls; cudaEvent_t a, b; };
static std::vector<Rec> g_recs;
static std::vector<cudaEvent_t> g_pool;
static cudaEvent_t g_open_ev = nullptr;

static cudaEvent_t get_event() {
  if (!g_pool.empty()) { cudaEvent_t e = g_pool.back(); g_pool.pop_back(); return e; }
  cudaEvent_t e; cudaEventCreate(&e); return e;
}

void mds_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void mds_prof_start(int cls, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_open_ev = get_event();
  cudaEventRecord(g_open_ev, st);
}

void mds_prof_stop(int cls, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t b = get_event();
  cudaEventRecord(b, st);
  g_recs.push_back(Rec{cls, g_open_ev, b});
  g_open_ev = nullptr;
}

extern "C" unsigned long long mds_launch_count(void) { return g_launches.load(); }

bool mds_once_per_device(const void* key) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> seen;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return true;
  std::lock_guard<std::mutex> lk(mu);
  return seen.insert(std::make_pair(dev, key)).second;
}

// launch-structure variants (include/mds.h mds_set_variant); never read from the environment
MdsVariant g_mds_var;

extern "C" int mds_set_variant(const char* key, long long value) {
  if (!key) return MDS_ERR_ARG;
  std::string k(key);
  MdsVariant& v = g_mds_var;
  if (k == "default") { v = MdsVariant(); return MDS_OK; }
  if (k == "tail_rows") { v.tail_rows = value; return MDS_OK; }
  if (k == "exact_rows") { if (value < 32) return MDS_ERR_ARG; v.exact_rows = value; return MDS_OK; }
  if (k == "cond_group") { if (value < 1 || value > 65536) return MDS_ERR_ARG; v.cond_group = (int)value; return MDS_OK; }
  if (k == "cdense_ctas") { if (value < 0 || value > 8) return MDS_ERR_ARG; v.cdense_ctas = (int)value; return MDS_OK; }
  int* flag = k == "no_tma" ? &v.no_tma : k == "no_lookahead" ? &v.no_lookahead
            : k == "static_sched" ? &v.static_sched : k == "no_snake" ? &v.no_snake
            : k == "no_cprefetch" ? &v.no_cprefetch : k == "upd_inplace" ? &v.upd_inplace
            : k == "upd_main" ? &v.upd_main : k == "slow_1cta" ? &v.slow_1cta
            : k == "exact_no_ls" ? &v.exact_no_ls : k == "f2_trsm" ? &v.f2_trsm
            : k == "no_pdl" ? &v.no_pdl : k == "ozaki" ? &v.ozaki : k == "exact_cluster" ? &v.exact_cluster
            : k == "cdense_serial" ? &v.cdense_serial : k == "cdense_tma" ? &v.cdense_tma
            : k == "cond_prio" ? &v.cond_prio : k == "fac_prio" ? &v.fac_prio : nullptr;
  if (!flag) return MDS_ERR_ARG;
  *flag = value ? 1 : 0;
  return MDS_OK;
}

extern "C" int mds_profile_begin(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& r : g_recs) { g_pool.push_back(r.a); g_pool.push_back(r.b); }
  g_recs.clear();
  g_mds_prof = true;
  return MDS_OK;
}

// per-launch timeline of the last profiled region: (class, start_ms, end_ms) relative to the first event
static std::vector<double> g_timeline;
extern "C" int64_t mds_profile_timeline(double* out3, int64_t cap) {
  std::lock_guard<std::mutex> lk(g_mu);
  const int64_t n = (int64_t)g_timeline.size() / 3;
  for (int64_t i = 0; i < std::min(n, cap) * 3; i++) out3[i] = g_timeline[i];
  return n;
}

extern "C" int mds_profile_end(double* ms_by_class, int64_t* launches_by_class, int ncls) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_mds_prof = false;
  if (ncls < PC_COUNT || !ms_by_class || !launches_by_class) return MDS_ERR_ARG;
  for (int c = 0; c < ncls; c++) { ms_by_class[c] = 0.0; launches_by_class[c] = 0; }
  g_timeline.clear();
  for (auto& r : g_recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return MDS_ERR_CUDA;
    float ms = 0.f, t0 = 0.f, t1 = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    cudaEventElapsedTime(&t0, g_recs[0].a, r.a);
    cudaEventElapsedTime(&t1, g_recs[0].a, r.b);
    ms_by_class[r.cls] += ms;
    launches_by_class[r.cls] += 1;
    g_timeline.push_back((double)r.cls);
    g_timeline.push_back((double)t0);
    g_timeline.push_back((double)t1);
  }
  for (auto& r : g_recs) { g_pool.push_back(r.a); g_pool.push_back(r.b); }
  g_recs.clear();
  return MDS_OK;
}
