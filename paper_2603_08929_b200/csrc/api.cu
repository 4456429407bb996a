// api.cu — the extern "C" boundary (include/bsort.h): validation, path selection (§8 a2),
// workspace handling, the host-only splitter math of the MSD partition, diagnostics.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include "paths.cuh"

namespace bsort {

static std::atomic<uint64_t> g_launches{0};
static thread_local int t_last_err = 0;

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_count_now() { return g_launches.load(std::memory_order_relaxed); }
void add_launches(int64_t k) { g_launches.fetch_add((uint64_t)k, std::memory_order_relaxed); }
void set_last_cuda_error(cudaError_t e) { t_last_err = (int)e; }

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  return dev;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

bool dtype_info(bsort_dtype_t dt, DtypeInfo* o) {
  switch (dt) {
    case BSORT_U8: *o = {1, KIND_U}; return true;
    case BSORT_I8: *o = {1, KIND_I}; return true;
    case BSORT_U16: *o = {2, KIND_U}; return true;
    case BSORT_I16: *o = {2, KIND_I}; return true;
    case BSORT_U32: *o = {4, KIND_U}; return true;
    case BSORT_I32: *o = {4, KIND_I}; return true;
    case BSORT_F32: *o = {4, KIND_F}; return true;
    case BSORT_U64: *o = {8, KIND_U}; return true;
    case BSORT_I64: *o = {8, KIND_I}; return true;
    case BSORT_F64: *o = {8, KIND_F}; return true;
    case BSORT_F16: *o = {2, KIND_F}; return true;
    case BSORT_BF16: *o = {2, KIND_F}; return true;
    default: return false;
  }
}

// ------------------------------------------------------------------------- profiler
namespace {
struct ProfRec {
  int kind;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::atomic<bool> g_prof_any{false};  // lock-free fast path for prof_begin/prof_end when off
std::vector<ProfRec> g_prof_recs;
std::vector<cudaEvent_t> g_event_pool;
thread_local cudaEvent_t t_open_event = nullptr;

cudaEvent_t take_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

bool profiling_on() { return g_prof_any.load(std::memory_order_relaxed); }

void prof_begin(int, cudaStream_t s) {
  if (!g_prof_any.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_prof_on) return;
  t_open_event = take_event();
  cudaEventRecord(t_open_event, s);
}

void prof_end(int kind, cudaStream_t s) {
  if (!g_prof_any.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_prof_on || !t_open_event) return;
  cudaEvent_t b = take_event();
  cudaEventRecord(b, s);
  g_prof_recs.push_back({kind, t_open_event, b});
  t_open_event = nullptr;
}

}  // namespace bsort

using namespace bsort;

namespace {

bool aligned_to(const void* p, int bytes) { return ((uintptr_t)p % (uintptr_t)bytes) == 0; }

size_t workspace_bytes(const DtypeInfo& di, uint64_t n) {
  if (n <= 1) return 0;
  return di.bytes <= 2 ? counting_workspace_bytes(di.bytes, n) : lsd_workspace_bytes(di.bytes, n);
}

bsort_status_t validate(bsort_dtype_t dtype, const void* p, uint64_t n, bsort_direction_t dir, DtypeInfo* di) {
  if (!dtype_info(dtype, di)) return BSORT_ERROR_UNSUPPORTED_DTYPE;
  if (dir != BSORT_ASCENDING && dir != BSORT_DESCENDING) return BSORT_ERROR_INVALID_ARGUMENT;
  if (n > 0 && p == nullptr) return BSORT_ERROR_INVALID_ARGUMENT;
  if (n > 0 && !aligned_to(p, di->bytes)) return BSORT_ERROR_INVALID_ARGUMENT;
  return BSORT_SUCCESS;
}

bsort_status_t sort_ws_impl(const DtypeInfo& di, void* keys, uint64_t n, bsort_direction_t dir, void* ws,
                            size_t wsb, cudaStream_t s) {
  if (n <= 1) return BSORT_SUCCESS;
  if (ws == nullptr || !aligned_to(ws, 256)) return BSORT_ERROR_INVALID_ARGUMENT;
  const bool desc = dir == BSORT_DESCENDING;
  return di.bytes <= 2 ? counting_sort(di, keys, n, desc, ws, wsb, s)
                       : lsd_sort(di, keys, nullptr, n, desc, ws, wsb, s);
}

// Sorts of up to GRAPH_MAX_N keys replay a cached CUDA graph of their launch sequence (graphs.cu).
constexpr uint64_t GRAPH_MAX_N = 1ull << 24;

bsort_status_t sort_ws_graphed(bsort_dtype_t dtype, const DtypeInfo& di, void* keys, uint64_t n,
                               bsort_direction_t dir, void* ws, size_t wsb, cudaStream_t s) {
  if (n > GRAPH_MAX_N) return sort_ws_impl(di, keys, n, dir, ws, wsb, s);
  GraphKey k{};
  k.dtype = (uint64_t)dtype;
  k.desc = dir == BSORT_DESCENDING;
  k.device = (uint64_t)current_device();
  k.n = n;
  k.keys = (uint64_t)(uintptr_t)keys;
  k.ws = (uint64_t)(uintptr_t)ws;
  k.wsb = wsb;
  return run_graphed(k, s, [&](cudaStream_t st) { return sort_ws_impl(di, keys, n, dir, ws, wsb, st); });
}

}  // namespace

extern "C" {

size_t bsort_workspace_bytes(bsort_dtype_t dtype, uint64_t n) {
  DtypeInfo di;
  if (!dtype_info(dtype, &di)) return 0;
  return workspace_bytes(di, n);
}

bsort_status_t bsort_sort_ws(bsort_dtype_t dtype, void* dev_keys, uint64_t n, bsort_direction_t direction,
                             void* workspace, size_t workspace_bytes_, void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_keys, n, direction, &di);
  if (st != BSORT_SUCCESS) return st;
  if (n <= 1) return BSORT_SUCCESS;
  if (workspace_bytes_ < workspace_bytes(di, n)) return BSORT_ERROR_WORKSPACE_TOO_SMALL;
  return sort_ws_graphed(dtype, di, dev_keys, n, direction, workspace, workspace_bytes_, (cudaStream_t)stream);
}

size_t bsort_inplace_workspace_bytes(bsort_dtype_t dtype, uint64_t n, uint64_t chunk_keys) {
  DtypeInfo di;
  if (!dtype_info(dtype, &di)) return 0;
  return inplace_workspace_bytes(di.bytes, n, chunk_keys);
}

bsort_status_t bsort_sort_inplace_ws(bsort_dtype_t dtype, void* dev_keys, uint64_t n, bsort_direction_t direction,
                                     uint64_t chunk_keys, void* workspace, size_t workspace_bytes_, void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_keys, n, direction, &di);
  if (st != BSORT_SUCCESS) return st;
  if (n <= 1) return BSORT_SUCCESS;
  if (workspace_bytes_ < inplace_workspace_bytes(di.bytes, n, chunk_keys)) return BSORT_ERROR_WORKSPACE_TOO_SMALL;
  if (workspace == nullptr || !aligned_to(workspace, 256)) return BSORT_ERROR_INVALID_ARGUMENT;
  return inplace_sort(di, dev_keys, n, direction == BSORT_DESCENDING, chunk_keys, workspace, workspace_bytes_,
                      (cudaStream_t)stream);
}

bsort_status_t bsort_sort(bsort_dtype_t dtype, void* dev_keys, uint64_t n, bsort_direction_t direction,
                          void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_keys, n, direction, &di);
  if (st != BSORT_SUCCESS || n <= 1) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t wsb = workspace_bytes(di, n);
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, wsb, s);
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    cudaGetLastError();
    return BSORT_ERROR_OUT_OF_MEMORY;
  }
  st = sort_ws_graphed(dtype, di, dev_keys, n, direction, ws, wsb, s);
  e = cudaFreeAsync(ws, s);
  if (st == BSORT_SUCCESS && e != cudaSuccess) {
    set_last_cuda_error(e);
    return BSORT_ERROR_CUDA;
  }
  return st;
}

bsort_status_t bsort_sort_host(bsort_dtype_t dtype, void* host_keys, uint64_t n, bsort_direction_t direction,
                               void* dev_keys, void* workspace, size_t workspace_bytes_, void* stream) {
  return bsort_sort_host_to(dtype, host_keys, host_keys, n, direction, dev_keys, workspace, workspace_bytes_,
                            stream);
}

bsort_status_t bsort_sort_host_to(bsort_dtype_t dtype, const void* host_in, void* host_out, uint64_t n,
                                  bsort_direction_t direction, void* dev_keys, void* workspace,
                                  size_t workspace_bytes_, void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_keys, n, direction, &di);
  if (st != BSORT_SUCCESS) return st;
  if (n > 0 && (host_in == nullptr || host_out == nullptr)) return BSORT_ERROR_INVALID_ARGUMENT;
  if (n == 0) return BSORT_SUCCESS;
  if (n > 1 && workspace_bytes_ < workspace_bytes(di, n)) return BSORT_ERROR_WORKSPACE_TOO_SMALL;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = (size_t)n * di.bytes;
  prof_begin(PROF_H2D, s);
  BSORT_CUDA(cudaMemcpyAsync(dev_keys, host_in, bytes, cudaMemcpyHostToDevice, s));
  prof_end(PROF_H2D, s);
  st = sort_ws_graphed(dtype, di, dev_keys, n, direction, workspace, workspace_bytes_, s);
  if (st != BSORT_SUCCESS) return st;
  prof_begin(PROF_D2H, s);
  BSORT_CUDA(cudaMemcpyAsync(host_out, dev_keys, bytes, cudaMemcpyDeviceToHost, s));
  prof_end(PROF_D2H, s);
  return BSORT_SUCCESS;
}

// ----------------------------------------------------------------------- key-value (N3)

size_t bsort_pairs_workspace_bytes(bsort_dtype_t dtype, uint64_t n) {
  DtypeInfo di;
  if (!dtype_info(dtype, &di) || di.bytes < 4 || n <= 1) return 0;
  return lsd_workspace_bytes(di.bytes, n, true);
}

bsort_status_t bsort_sort_pairs_ws(bsort_dtype_t dtype, void* dev_keys, uint32_t* dev_values, uint64_t n,
                                   bsort_direction_t direction, void* workspace, size_t workspace_bytes_,
                                   void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_keys, n, direction, &di);
  if (st != BSORT_SUCCESS) return st;
  if (di.bytes < 4) return BSORT_ERROR_UNSUPPORTED_DTYPE;
  if (n > 0 && (dev_values == nullptr || !aligned_to(dev_values, 4))) return BSORT_ERROR_INVALID_ARGUMENT;
  if (n <= 1) return BSORT_SUCCESS;
  if (workspace == nullptr || !aligned_to(workspace, 256)) return BSORT_ERROR_INVALID_ARGUMENT;
  if (workspace_bytes_ < lsd_workspace_bytes(di.bytes, n, true)) return BSORT_ERROR_WORKSPACE_TOO_SMALL;
  return lsd_sort(di, dev_keys, dev_values, n, direction == BSORT_DESCENDING, workspace, workspace_bytes_,
                  (cudaStream_t)stream);
}

bsort_status_t bsort_sort_pairs(bsort_dtype_t dtype, void* dev_keys, uint32_t* dev_values, uint64_t n,
                                bsort_direction_t direction, void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_keys, n, direction, &di);
  if (st != BSORT_SUCCESS) return st;
  if (di.bytes < 4) return BSORT_ERROR_UNSUPPORTED_DTYPE;
  if (n > 0 && (dev_values == nullptr || !aligned_to(dev_values, 4))) return BSORT_ERROR_INVALID_ARGUMENT;
  if (n <= 1) return BSORT_SUCCESS;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t wsb = lsd_workspace_bytes(di.bytes, n, true);
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, wsb, s);
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    cudaGetLastError();
    return BSORT_ERROR_OUT_OF_MEMORY;
  }
  st = lsd_sort(di, dev_keys, dev_values, n, direction == BSORT_DESCENDING, ws, wsb, s);
  e = cudaFreeAsync(ws, s);
  if (st == BSORT_SUCCESS && e != cudaSuccess) {
    set_last_cuda_error(e);
    return BSORT_ERROR_CUDA;
  }
  return st;
}

// ------------------------------------------------------------------------ distributed

bsort_status_t bsort_dist_top_hist(bsort_dtype_t dtype, const void* dev_keys, uint64_t n,
                                   bsort_direction_t direction, uint64_t* dev_hist, void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_keys, n, direction, &di);
  if (st != BSORT_SUCCESS) return st;
  if (di.bytes < 4) return BSORT_ERROR_UNSUPPORTED_DTYPE;
  if (dev_hist == nullptr || !aligned_to(dev_hist, 8)) return BSORT_ERROR_INVALID_ARGUMENT;
  return dist_top_hist(di, dev_keys, n, direction == BSORT_DESCENDING, dev_hist, (cudaStream_t)stream);
}

bsort_status_t bsort_dist_splitters(const uint64_t* hist, int nranks, uint32_t* cuts) {
  if (!hist || !cuts || nranks < 1 || nranks > BSORT_DIST_MAX_RANKS) return BSORT_ERROR_INVALID_ARGUMENT;
  unsigned __int128 total = 0;
  for (int b = 0; b < BSORT_DIST_BINS; ++b) total += hist[b];
  cuts[0] = 0;
  cuts[nranks] = BSORT_DIST_BINS;
  uint64_t prefix = 0;  // sum(hist[0..b))
  int b = 0;
  for (int r = 1; r < nranks; ++r) {
    const uint64_t target = (uint64_t)((total * (unsigned __int128)r) / (unsigned __int128)nranks);
    while (b < BSORT_DIST_BINS && prefix < target) prefix += hist[b++];
    cuts[r] = (uint32_t)b;
  }
  return BSORT_SUCCESS;
}

bsort_status_t bsort_dist_send_counts(const uint64_t* local_hist, const uint32_t* cuts, int nranks,
                                      uint64_t* send_counts) {
  if (!local_hist || !cuts || !send_counts || nranks < 1 || nranks > BSORT_DIST_MAX_RANKS)
    return BSORT_ERROR_INVALID_ARGUMENT;
  if (cuts[0] != 0 || cuts[nranks] != BSORT_DIST_BINS) return BSORT_ERROR_INVALID_ARGUMENT;
  for (int q = 0; q < nranks; ++q) {
    if (cuts[q] > cuts[q + 1]) return BSORT_ERROR_INVALID_ARGUMENT;
    uint64_t c = 0;
    for (uint32_t b = cuts[q]; b < cuts[q + 1]; ++b) c += local_hist[b];
    send_counts[q] = c;
  }
  return BSORT_SUCCESS;
}

size_t bsort_dist_partition_workspace_bytes(bsort_dtype_t dtype, uint64_t n, int nranks) {
  DtypeInfo di;
  if (!dtype_info(dtype, &di) || di.bytes < 4) return 0;
  return dist_partition_workspace_bytes(di.bytes, n, nranks);
}

bsort_status_t bsort_dist_partition(bsort_dtype_t dtype, const void* dev_in, uint64_t n,
                                    bsort_direction_t direction, const uint32_t* cuts,
                                    const uint64_t* send_counts, int nranks, void* dev_out, void* workspace,
                                    size_t workspace_bytes_, void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_in, n, direction, &di);
  if (st != BSORT_SUCCESS) return st;
  if (di.bytes < 4) return BSORT_ERROR_UNSUPPORTED_DTYPE;
  if (!cuts || !send_counts || nranks < 1 || nranks > BSORT_DIST_MAX_RANKS) return BSORT_ERROR_INVALID_ARGUMENT;
  if (cuts[0] != 0 || cuts[nranks] != BSORT_DIST_BINS) return BSORT_ERROR_INVALID_ARGUMENT;
  for (int q = 0; q < nranks; ++q)
    if (cuts[q] > cuts[q + 1]) return BSORT_ERROR_INVALID_ARGUMENT;
  if (n == 0) return BSORT_SUCCESS;
  if (!dev_out || !aligned_to(dev_out, di.bytes) || dev_out == dev_in) return BSORT_ERROR_INVALID_ARGUMENT;
  if (!workspace || !aligned_to(workspace, 256)) return BSORT_ERROR_INVALID_ARGUMENT;
  return dist_partition(di, dev_in, n, direction == BSORT_DESCENDING, cuts, send_counts, nranks, dev_out,
                        nullptr, workspace, workspace_bytes_, (cudaStream_t)stream);
}

bsort_status_t bsort_dist_partition_remote(bsort_dtype_t dtype, const void* dev_in, uint64_t n,
                                           bsort_direction_t direction, const uint32_t* cuts,
                                           const uint64_t* send_counts, int nranks,
                                           const uint64_t* dst_addrs, void* workspace,
                                           size_t workspace_bytes_, void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_in, n, direction, &di);
  if (st != BSORT_SUCCESS) return st;
  if (di.bytes < 4) return BSORT_ERROR_UNSUPPORTED_DTYPE;
  if (!cuts || !send_counts || !dst_addrs || nranks < 1 || nranks > BSORT_DIST_MAX_RANKS)
    return BSORT_ERROR_INVALID_ARGUMENT;
  if (cuts[0] != 0 || cuts[nranks] != BSORT_DIST_BINS) return BSORT_ERROR_INVALID_ARGUMENT;
  for (int q = 0; q < nranks; ++q) {
    if (cuts[q] > cuts[q + 1]) return BSORT_ERROR_INVALID_ARGUMENT;
    if (send_counts[q] > 0 && (dst_addrs[q] == 0 || dst_addrs[q] % di.bytes != 0)) return BSORT_ERROR_INVALID_ARGUMENT;
  }
  if (n == 0) return BSORT_SUCCESS;
  if (!workspace || !aligned_to(workspace, 256)) return BSORT_ERROR_INVALID_ARGUMENT;
  return dist_partition(di, dev_in, n, direction == BSORT_DESCENDING, cuts, send_counts, nranks, nullptr,
                        dst_addrs, workspace, workspace_bytes_, (cudaStream_t)stream);
}

// ------------------------------------------------------------- exact splitting (N2)

namespace {
bool increasing(const uint64_t* v, int m) {
  for (int j = 1; j < m; ++j)
    if (v[j] <= v[j - 1]) return false;
  return true;
}
}  // namespace

// Host planning of exact splitting (pure host; the Python orchestration calls these through
// ctypes; tests pin them against brute force and against an independent numpy restatement in
// tests/_exact_ref.py).
bsort_status_t bsort_dist_exact_boundaries(const uint64_t* hg, int nranks, int key_bits, bsort_refine_fn refine,
                                           void* ctx, uint64_t* values, int* m_out, int* idx, uint64_t* quota,
                                           int* levels_out) {
  if (!hg || !refine || !values || !m_out || !idx || !quota || nranks < 1 || nranks > BSORT_DIST_MAX_RANKS)
    return BSORT_ERROR_INVALID_ARGUMENT;
  if (key_bits != 32 && key_bits != 64) return BSORT_ERROR_INVALID_ARGUMENT;
  const int R = nranks - 1;
  unsigned __int128 N = 0;
  for (int b = 0; b < BSORT_DIST_BINS; ++b) N += hg[b];
  std::vector<uint64_t> T(R), pv(R), below(R);
  std::vector<int> bits(R, 16);
  std::vector<uint64_t> cum(BSORT_DIST_BINS);
  uint64_t acc = 0;
  for (int b = 0; b < BSORT_DIST_BINS; ++b) cum[b] = (acc += hg[b]);
  for (int i = 0; i < R; ++i) {
    T[i] = (uint64_t)((N * (unsigned __int128)(i + 1)) / (unsigned __int128)nranks);
    const int b = (int)(std::upper_bound(cum.begin(), cum.end(), T[i]) - cum.begin());  // bin of rank T_i
    if (b >= BSORT_DIST_BINS) return BSORT_ERROR_INVALID_ARGUMENT;  // T_i >= N: empty input
    pv[i] = (uint64_t)b;
    below[i] = b > 0 ? cum[b - 1] : 0;
  }
  int levels = 0;
  std::vector<uint64_t> H;
  for (int level_bits = 16; level_bits < key_bits; level_bits += 16) {
    std::vector<uint64_t> prefixes;
    for (int i = 0; i < R; ++i)
      if (T[i] > below[i]) prefixes.push_back(pv[i]);
    if (prefixes.empty()) break;
    std::sort(prefixes.begin(), prefixes.end());
    prefixes.erase(std::unique(prefixes.begin(), prefixes.end()), prefixes.end());
    const int mm = (int)prefixes.size();
    H.assign((size_t)mm * BSORT_DIST_BINS, 0);
    if (refine(ctx, prefixes.data(), mm, level_bits, H.data()) != 0) return BSORT_ERROR_CUDA;
    ++levels;
    for (int i = 0; i < R; ++i) {
      if (T[i] <= below[i]) continue;
      const int row = (int)(std::lower_bound(prefixes.begin(), prefixes.end(), pv[i]) - prefixes.begin());
      const uint64_t* h = H.data() + (size_t)row * BSORT_DIST_BINS;
      const uint64_t res = T[i] - below[i];
      uint64_t c = 0;
      int sb = 0;
      for (; sb < BSORT_DIST_BINS; ++sb) {  // first sub-bin whose inclusive count exceeds res
        if (c + h[sb] > res) break;
        c += h[sb];
      }
      if (sb >= BSORT_DIST_BINS) return BSORT_ERROR_INVALID_ARGUMENT;  // inconsistent histograms
      below[i] += c;
      pv[i] = (pv[i] << 16) | (uint64_t)sb;
      bits[i] += 16;
    }
  }
  std::vector<uint64_t> K(R);
  for (int i = 0; i < R; ++i) K[i] = pv[i] << (key_bits - bits[i]);
  std::vector<uint64_t> v(K);
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  for (size_t j = 0; j < v.size(); ++j) values[j] = v[j];
  for (int i = 0; i < R; ++i) {
    idx[i] = (int)(std::lower_bound(v.begin(), v.end(), K[i]) - v.begin());
    quota[i] = T[i] - below[i];
  }
  *m_out = (int)v.size();
  if (levels_out) *levels_out = levels;
  return BSORT_SUCCESS;
}

bsort_status_t bsort_dist_exact_send_counts(const uint64_t* cc, int nranks, int m, int rank, const int* idx,
                                            const uint64_t* quota, uint64_t* send_counts) {
  if (!cc || !send_counts || nranks < 1 || nranks > BSORT_DIST_MAX_RANKS || rank < 0 || rank >= nranks || m < 0)
    return BSORT_ERROR_INVALID_ARGUMENT;
  if (nranks > 1 && (!idx || !quota || m < 1)) return BSORT_ERROR_INVALID_ARGUMENT;
  const int C = 2 * m + 1;
  const uint64_t* mine = cc + (size_t)rank * C;
  std::vector<uint64_t> start(C + 1, 0);
  for (int c = 0; c < C; ++c) start[c + 1] = start[c] + mine[c];
  uint64_t prev = 0;
  for (int r = 0; r + 1 < nranks; ++r) {
    const int j = idx[r];
    if (j < 0 || j >= m) return BSORT_ERROR_INVALID_ARGUMENT;
    uint64_t eq_before = 0;  // keys equal to values[j] on lower ranks
    for (int q = 0; q < rank; ++q) eq_before += cc[(size_t)q * C + 2 * j + 1];
    const uint64_t want = quota[r] > eq_before ? quota[r] - eq_before : 0;
    const uint64_t share = std::min(want, mine[2 * j + 1]);
    const uint64_t split = start[2 * j + 1] + share;
    if (split < prev) return BSORT_ERROR_INVALID_ARGUMENT;
    send_counts[r] = split - prev;
    prev = split;
  }
  send_counts[nranks - 1] = start[C] - prev;
  return BSORT_SUCCESS;
}

bsort_status_t bsort_dist_refine_hist(bsort_dtype_t dtype, const void* dev_keys, uint64_t n,
                                      bsort_direction_t direction, const uint64_t* prefixes, int m,
                                      int prefix_bits, uint64_t* dev_hist, void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_keys, n, direction, &di);
  if (st != BSORT_SUCCESS) return st;
  if (di.bytes < 4) return BSORT_ERROR_UNSUPPORTED_DTYPE;
  if (!prefixes || m < 1 || m > BSORT_DIST_MAX_RANKS || !increasing(prefixes, m)) return BSORT_ERROR_INVALID_ARGUMENT;
  if (prefix_bits < 16 || prefix_bits % 16 != 0 || prefix_bits + 16 > di.bytes * 8) return BSORT_ERROR_INVALID_ARGUMENT;
  if (!dev_hist || !aligned_to(dev_hist, 8)) return BSORT_ERROR_INVALID_ARGUMENT;
  return dist_refine_hist(di, dev_keys, n, direction == BSORT_DESCENDING, prefixes, m, prefix_bits, dev_hist,
                          (cudaStream_t)stream);
}

bsort_status_t bsort_dist_class_hist(bsort_dtype_t dtype, const void* dev_keys, uint64_t n,
                                     bsort_direction_t direction, const uint64_t* values, int m,
                                     uint64_t* dev_counts, void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_keys, n, direction, &di);
  if (st != BSORT_SUCCESS) return st;
  if (di.bytes < 4) return BSORT_ERROR_UNSUPPORTED_DTYPE;
  if (!values || m < 1 || m > BSORT_DIST_MAX_RANKS || !increasing(values, m)) return BSORT_ERROR_INVALID_ARGUMENT;
  if (!dev_counts || !aligned_to(dev_counts, 8)) return BSORT_ERROR_INVALID_ARGUMENT;
  return dist_class_hist(di, dev_keys, n, direction == BSORT_DESCENDING, values, m, dev_counts,
                         (cudaStream_t)stream);
}

size_t bsort_dist_class_partition_workspace_bytes(void) { return dist_class_partition_workspace_bytes(); }

bsort_status_t bsort_dist_partition_classes(bsort_dtype_t dtype, const void* dev_in, uint64_t n,
                                            bsort_direction_t direction, const uint64_t* values, int m,
                                            const uint64_t* class_counts, void* dev_out, void* workspace,
                                            size_t workspace_bytes_, void* stream) {
  DtypeInfo di;
  bsort_status_t st = validate(dtype, dev_in, n, direction, &di);
  if (st != BSORT_SUCCESS) return st;
  if (di.bytes < 4) return BSORT_ERROR_UNSUPPORTED_DTYPE;
  if (!values || !class_counts || m < 1 || m > BSORT_DIST_MAX_RANKS || !increasing(values, m))
    return BSORT_ERROR_INVALID_ARGUMENT;
  if (n == 0) return BSORT_SUCCESS;
  if (!dev_out || !aligned_to(dev_out, di.bytes) || dev_out == dev_in) return BSORT_ERROR_INVALID_ARGUMENT;
  if (!workspace || !aligned_to(workspace, 256)) return BSORT_ERROR_INVALID_ARGUMENT;
  if (workspace_bytes_ < dist_class_partition_workspace_bytes()) return BSORT_ERROR_WORKSPACE_TOO_SMALL;
  return dist_partition_classes(di, dev_in, n, direction == BSORT_DESCENDING, values, m, class_counts, dev_out,
                                workspace, (cudaStream_t)stream);
}

// ------------------------------------------------------------------------ diagnostics

const char* bsort_status_string(bsort_status_t s) {
  switch (s) {
    case BSORT_SUCCESS: return "success";
    case BSORT_ERROR_INVALID_ARGUMENT: return "invalid argument";
    case BSORT_ERROR_UNSUPPORTED_DTYPE: return "unsupported dtype";
    case BSORT_ERROR_OUT_OF_MEMORY: return "out of device memory";
    case BSORT_ERROR_WORKSPACE_TOO_SMALL: return "workspace too small";
    case BSORT_ERROR_CUDA: return "CUDA error";
    case BSORT_ERROR_NCCL: return "NCCL error";
    case BSORT_ERROR_CAPACITY: return "output capacity too small";
    default: return "unknown status";
  }
}

int bsort_last_cuda_error(void) { return t_last_err; }
const char* bsort_version(void) { return "bsort-b200 0.1 (sm_100a)"; }
uint64_t bsort_launch_count(void) { return g_launches.load(); }

void bsort_profile_enable(int on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& r : g_prof_recs) {
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_prof_recs.clear();
  g_prof_on = on != 0;
  g_prof_any.store(on != 0, std::memory_order_relaxed);
}

int bsort_profile_read(double* ms, uint64_t* launches) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (int k = 0; k < BSORT_PROF_KINDS; ++k) {
    if (ms) ms[k] = 0.0;
    if (launches) launches[k] = 0;
  }
  for (auto& r : g_prof_recs) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (ms) ms[r.kind] += t;
    if (launches) launches[r.kind] += 1;
  }
  return BSORT_PROF_KINDS;
}

const char* bsort_profile_kind_name(int k) {
  static const char* names[BSORT_PROF_KINDS] = {"memset", "onesweep_hist", "plan_scan", "onesweep_pass",
                                                "copy_back", "count_hist", "count_scan", "count_fill",
                                                "dist_tophist", "dist_partition", "h2d", "d2h", "dist_a2a"};
  return (k >= 0 && k < BSORT_PROF_KINDS) ? names[k] : "?";
}

}  // extern "C"
