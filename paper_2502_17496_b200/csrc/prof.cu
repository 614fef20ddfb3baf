// prof.cu — opt-in launch timing with CUDA events: (1) the profiling pass (every launch bracketed by
// events; never inside a graph capture) and (2) the live watch of one kernel inside a benchmark's
// timed region (event pairs supplied by the caller, recorded as event nodes when captured).
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include "internal.h"

namespace spk {
namespace {
struct Rec {
  const char* name;
  int bound;
  double flops, bytes;
  cudaEvent_t e0, e1;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
bool g_on = false;
struct Watch {
  std::string name;   // "*": every launch
  std::vector<cudaEvent_t> b, e;
  std::vector<const char*> names;   // kernel name of each pair used
  int next = 0;
} g_watch;
bool g_watch_on = false;

cudaError_t record(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) cs = cudaStreamCaptureStatusNone;
  // inside a capture the record must become an event node of the graph (timed at every replay)
  return cudaEventRecordWithFlags(ev, s, cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal
                                                                               : cudaEventRecordDefault);
}
}  // namespace

bool prof_on() { return g_on || g_watch_on; }

ProfScope::ProfScope(const char* name, int bound, double flops, double bytes, cudaStream_t s) : st(s) {
  if (g_watch_on) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_watch.next < (int)g_watch.b.size() && (g_watch.name == "*" || g_watch.name == name)) {
      wslot = g_watch.next++;
      g_watch.names.push_back(name);
      record(g_watch.b[wslot], s);
    }
  }
  if (!g_on) return;
  cudaStreamCaptureStatus cs;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
  Rec r{name, bound, flops, bytes, nullptr, nullptr};
  cudaEventCreate(&r.e0);
  cudaEventCreate(&r.e1);
  cudaEventRecord(r.e0, s);
  std::lock_guard<std::mutex> lk(g_mu);
  slot = (int)g_recs.size();
  g_recs.push_back(r);
}

ProfScope::~ProfScope() {
  if (wslot >= 0) {
    std::lock_guard<std::mutex> lk(g_mu);
    record(g_watch.e[wslot], st);
  }
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventRecord(g_recs[slot].e1, st);
}

}  // namespace spk

extern "C" {

void spikerl_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(spk::g_mu);
  for (auto& r : spk::g_recs) { cudaEventDestroy(r.e0); cudaEventDestroy(r.e1); }
  spk::g_recs.clear();
  spk::g_on = on != 0;
}

int spikerl_prof_watch(const char* name, void* const* ev_begin, void* const* ev_end, int n) {
  std::lock_guard<std::mutex> lk(spk::g_mu);
  spk::g_watch = spk::Watch{};
  spk::g_watch_on = false;
  if (!name) return SPIKERL_OK;
  if (n < 1 || !ev_begin || !ev_end) { spk::set_error("spikerl_prof_watch: bad arguments"); return SPIKERL_E_ARG; }
  spk::g_watch.name = name;
  for (int i = 0; i < n; ++i) {
    if (!ev_begin[i] || !ev_end[i]) { spk::set_error("spikerl_prof_watch: null event"); return SPIKERL_E_ARG; }
    spk::g_watch.b.push_back((cudaEvent_t)ev_begin[i]);
    spk::g_watch.e.push_back((cudaEvent_t)ev_end[i]);
  }
  spk::g_watch_on = true;
  return SPIKERL_OK;
}

int spikerl_prof_watch_count(void) {
  std::lock_guard<std::mutex> lk(spk::g_mu);
  return spk::g_watch.next;
}

const char* spikerl_prof_watch_name(int i) {
  std::lock_guard<std::mutex> lk(spk::g_mu);
  return (i >= 0 && i < (int)spk::g_watch.names.size()) ? spk::g_watch.names[i] : "";
}

int spikerl_prof_timeline(spikerl_prof_span* out, int max_entries) {
  std::lock_guard<std::mutex> lk(spk::g_mu);
  if (spk::g_recs.empty()) return 0;
  cudaEvent_t t0 = spk::g_recs[0].e0;
  for (auto& r : spk::g_recs)
    if (cudaEventSynchronize(r.e1) != cudaSuccess) { spk::set_error("prof: event sync failed"); return -1; }
  int n = 0;
  for (auto& r : spk::g_recs) {
    if (out && n < max_entries) {
      spikerl_prof_span& e = out[n];
      memset(&e, 0, sizeof(e));
      strncpy(e.name, r.name, sizeof(e.name) - 1);
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, t0, r.e0);
      cudaEventElapsedTime(&b, t0, r.e1);
      e.start_ms = a;
      e.end_ms = b;
    }
    ++n;
  }
  return n;
}

int spikerl_prof_summary(spikerl_prof_entry* out, int max_entries) {
  std::lock_guard<std::mutex> lk(spk::g_mu);
  std::map<std::string, spikerl_prof_entry> agg;
  for (auto& r : spk::g_recs) {
    if (cudaEventSynchronize(r.e1) != cudaSuccess) { spk::set_error("prof: event sync failed"); return -1; }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.e0, r.e1);
    auto& e = agg[r.name];
    if (e.launches == 0) {
      memset(&e, 0, sizeof(e));
      strncpy(e.name, r.name, sizeof(e.name) - 1);
      e.bound = r.bound;
    }
    e.launches += 1;
    e.total_ms += ms;
    e.flops += r.flops;
    e.bytes += r.bytes;
  }
  int n = 0;
  for (auto& kv : agg) {
    if (n < max_entries && out) out[n] = kv.second;
    ++n;
  }
  return n;
}

}  // extern "C"

namespace spk {

int aux_pool(AuxPool** out) {
  static AuxPool pool[16];
  static bool made[16] = {};
  int dev = 0;
  SPK_CHECK_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 16) { set_error("device index %d out of range", dev); return SPIKERL_E_ARG; }
  if (!made[dev]) {
    for (auto& x : pool[dev].side) SPK_CHECK_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    for (auto& e : pool[dev].ev) SPK_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    made[dev] = true;
  }
  *out = &pool[dev];
  return SPIKERL_OK;
}

int stream_after(cudaStream_t dst, cudaStream_t src, cudaEvent_t ev) {
  SPK_CHECK_CUDA(cudaEventRecord(ev, src));
  SPK_CHECK_CUDA(cudaStreamWaitEvent(dst, ev, 0));
  return SPIKERL_OK;
}

}  // namespace spk
