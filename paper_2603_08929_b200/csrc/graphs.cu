// graphs.cu — CUDA-graph replay of small sorts (DESIGN.md §6 "Small n").
//
// Below 2^24 keys a sort is a handful of dependent launches whose host enqueue costs ~2.5-3.8 us
// per kernel launch on B200 with this driver (tools/exp/launch_cost.cu): 6 launches + 1 memset
// are ~19 us of host time before the last kernel is even queued.  The
// launch sequence of a sort depends only on (dtype, n, direction, buffers, workspace, device) --
// every data-dependent decision (trivial digits, presorted input, pass variants) is taken on the
// device from the plan in the workspace -- so the library captures it once into a CUDA graph
// and replays that graph (one host launch) on later calls with the same arguments.
//
// First call with a key: plain launches (this also runs the one-time set-up: function
// attributes, the lane-order self-test).  Second call: capture on a private stream, instantiate,
// launch.  Later calls: cudaGraphLaunch on the caller's stream.  Not used while the caller's
// stream is itself being captured (the caller's graph takes the kernels), while per-launch
// profiling is on, or with BSORT_GRAPH=0.  At most 64 graphs are kept (least recently used
// evicted).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace bsort {
namespace {

struct Entry {
  GraphKey key;
  int uses = 0;  // calls seen with this key; -1 = capture failed, never graph it
  cudaGraphExec_t exec = nullptr;
  uint64_t kernels = 0;  // kernel launches inside the graph (launch counter)
  uint64_t stamp = 0;
};

std::mutex g_mu;
std::vector<Entry> g_entries;
uint64_t g_clock = 0;
cudaStream_t g_cap_stream[64] = {};
constexpr size_t MAX_GRAPHS = 64;

bool same(const GraphKey& a, const GraphKey& b) { return std::memcmp(&a, &b, sizeof(GraphKey)) == 0; }

bool graphs_enabled() {
  static const bool on = [] {
    const char* e = getenv("BSORT_GRAPH");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

bsort_status_t run_graphed(const GraphKey& key, cudaStream_t s, const std::function<bsort_status_t(cudaStream_t)>& run) {
  if (!graphs_enabled() || profiling_on()) return run(s);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return run(s);
  }
  std::unique_lock<std::mutex> lk(g_mu);
  Entry* e = nullptr;
  for (auto& x : g_entries)
    if (same(x.key, key)) e = &x;
  if (!e) {
    if (g_entries.size() >= MAX_GRAPHS) {  // evict the least recently used
      size_t v = 0;
      for (size_t i = 1; i < g_entries.size(); ++i)
        if (g_entries[i].stamp < g_entries[v].stamp) v = i;
      if (g_entries[v].exec) cudaGraphExecDestroy(g_entries[v].exec);
      g_entries.erase(g_entries.begin() + v);
    }
    g_entries.push_back(Entry{key});
    e = &g_entries.back();
  }
  e->stamp = ++g_clock;
  if (e->exec) {
    cudaGraphExec_t ex = e->exec;
    const uint64_t k = e->kernels;
    lk.unlock();
    const cudaError_t r = cudaGraphLaunch(ex, s);
    if (r != cudaSuccess) {
      set_last_cuda_error(r);
      cudaGetLastError();
      return BSORT_ERROR_CUDA;
    }
    add_launches(k);
    return BSORT_SUCCESS;
  }
  if (e->uses < 0 || ++e->uses < 2) {
    lk.unlock();
    return run(s);
  }
  // second call with this key: capture the launch sequence on a private stream
  const int dev = key.device;
  if (!g_cap_stream[dev] && cudaStreamCreateWithFlags(&g_cap_stream[dev], cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    g_cap_stream[dev] = nullptr;
    e->uses = -1;
    lk.unlock();
    return run(s);
  }
  cudaStream_t cap = g_cap_stream[dev];
  cudaGraph_t g = nullptr;
  const uint64_t c0 = launch_count_now();
  bsort_status_t st = BSORT_ERROR_CUDA;
  if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
    st = run(cap);
    if (cudaStreamEndCapture(cap, &g) != cudaSuccess) g = nullptr;
  }
  const uint64_t k = launch_count_now() - c0;
  add_launches(-k);  // captured, not run
  cudaGraphExec_t ex = nullptr;
  if (st == BSORT_SUCCESS && g && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess) {
    e->exec = ex;
    e->kernels = k;
  } else {
    e->uses = -1;
    ex = nullptr;
  }
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();
  lk.unlock();
  if (!ex) return run(s);
  const cudaError_t r = cudaGraphLaunch(ex, s);
  if (r != cudaSuccess) {
    set_last_cuda_error(r);
    cudaGetLastError();
    return BSORT_ERROR_CUDA;
  }
  add_launches(k);
  return BSORT_SUCCESS;
}

}  // namespace bsort
