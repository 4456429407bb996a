// comm.cu — native multi-GPU sort over NCCL (SURVEY §8 b: bsort_comm_* / bsort_sort_dist).
//
// The whole MSD path of §8 a7-a11 in one C call, built only from this library's own ABI
// (bsort_dist_top_hist, bsort_dist_splitters, bsort_dist_send_counts, bsort_dist_partition,
// bsort_sort_ws) plus NCCL collectives on the caller's stream:
//
//   a7  top-16-bit histogram            -> ncclAllReduce(sum) of 65,536 u64
//   a8  splitters + send counts (host)  -> ncclAllGather of every rank's (send counts, capacity)
//   a9  P-way partition by destination  (unstable one-sweep pass into a bucketed scratch copy)
//   a10 grouped ncclSend / ncclRecv     (keys to their owners, rank-ordered in dev_out)
//   a11 local one-sweep LSD sort of dev_out
//
// NCCL is bound at run time (dlopen "libnccl.so.2"): libbsort.so has no link-time NCCL
// dependency, and inside a PyTorch process the already-loaded libnccl (same soname) is reused.
// Host syncs: after the histogram all-reduce (splitters are host math), after the counts
// all-gather (receive sizes and the capacity check, which every rank evaluates for every rank so
// that a too-small dev_out makes ALL ranks return BSORT_ERROR_CAPACITY before any key moves) and
// after the exchange (failure detection).  BSORT_DIST_FUSED (§8 N1) replaces a9 + a10 by the
// partition kernel writing every key straight into its owner's receive buffer over CUDA IPC peer
// mappings, between two device-side barriers (k_peer_barrier).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "bsort.h"
#include "common.cuh"

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  // failure detection (optional symbols: without them waits are plain stream syncs)
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    bool all = true;
    auto get = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      all = all && fp != nullptr;
    };
    get(api.GetUniqueId, "ncclGetUniqueId");
    get(api.CommInitRank, "ncclCommInitRank");
    get(api.CommDestroy, "ncclCommDestroy");
    get(api.AllReduce, "ncclAllReduce");
    get(api.AllGather, "ncclAllGather");
    get(api.Send, "ncclSend");
    get(api.Recv, "ncclRecv");
    get(api.GroupStart, "ncclGroupStart");
    get(api.GroupEnd, "ncclGroupEnd");
    api.ok = all;
    api.CommGetAsyncError =
        reinterpret_cast<decltype(api.CommGetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
    api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(dlsym(h, "ncclCommAbort"));
  });
  return api;
}

thread_local int t_last_nccl = 0;

bsort_status_t nccl_status(ncclResult_t r) {
  if (r == ncclSuccess) return BSORT_SUCCESS;
  t_last_nccl = (int)r;
  return BSORT_ERROR_NCCL;
}

bsort_status_t cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return BSORT_SUCCESS;
  bsort::set_last_cuda_error(e);
  cudaGetLastError();
  return BSORT_ERROR_CUDA;
}

#define NCCL_TRY(x)                                   \
  do {                                                \
    bsort_status_t st_ = nccl_status(x);              \
    if (st_ != BSORT_SUCCESS) return st_;             \
  } while (0)
#define CUDA_TRY(x)                                   \
  do {                                                \
    bsort_status_t st_ = cuda_status(x);              \
    if (st_ != BSORT_SUCCESS) return st_;             \
  } while (0)
#define BS_TRY(x)                                     \
  do {                                                \
    bsort_status_t st_ = (x);                         \
    if (st_ != BSORT_SUCCESS) return st_;             \
  } while (0)

int key_bytes(bsort_dtype_t dt) {
  switch (dt) {
    case BSORT_U32: case BSORT_I32: case BSORT_F32: return 4;
    case BSORT_U64: case BSORT_I64: case BSORT_F64: return 8;
    default: return 0;
  }
}

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

struct bsort_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0;
  int rank = 0;
  int device = 0;
  bool aborted = false;  // ncclCommAbort was called (peer failure / timeout): unusable
  // Grow-only device workspace reused by every bsort_sort_dist call on this communicator (a
  // fresh multi-GiB cudaMallocAsync per call would remap pages whenever the pool trims).
  // ws_done is recorded after each call's last use; the next call's stream waits on it.
  void* ws = nullptr;
  size_t ws_bytes = 0;
  cudaEvent_t ws_done = nullptr;
  // Fused exchange (BSORT_DIST_FUSED): this rank's receive buffer and signal pad
  // (cudaMalloc, exported by CUDA IPC handle), every peer's mapped into this process, and the
  // barrier epoch (the same on every rank: each fused call runs the same two barriers).
  void* rbuf = nullptr;
  size_t rbytes = 0;
  unsigned* pad = nullptr;  // [BSORT_DIST_MAX_RANKS] arrival epochs of each peer, then [1] error
  void* peer_rbuf[BSORT_DIST_MAX_RANKS] = {};
  unsigned* peer_pad[BSORT_DIST_MAX_RANKS] = {};
  unsigned char* hbuf = nullptr;  // device staging of the all-gathered IPC handles
  unsigned epoch = 0;
};

namespace {

// Wait for the stream while watching the communicator (SURVEY §8 failure detection): a peer that
// dies mid-collective leaves the stream pending forever, so poll cudaStreamQuery and
// ncclCommGetAsyncError; on an asynchronous NCCL error, or after BSORT_NCCL_TIMEOUT_S seconds
// (default 300; 0 = no limit), abort the communicator (its pending collectives are cancelled and
// the stream drains) and return BSORT_ERROR_NCCL (bsort_last_nccl_error holds the NCCL code,
// ncclInternalError for a timeout).  Every later call on the communicator fails.
double nccl_timeout_s() {
  static const double v = [] {
    const char* e = getenv("BSORT_NCCL_TIMEOUT_S");
    return e ? atof(e) : 300.0;
  }();
  return v;
}

bsort_status_t abort_comm(bsort_comm* c, ncclResult_t why) {
  NcclApi& N = nccl();
  if (N.CommAbort && c->comm && !c->aborted) N.CommAbort(c->comm);
  c->aborted = true;
  return nccl_status(why == ncclSuccess ? ncclInternalError : why);
}

bsort_status_t wait_watching(cudaStream_t s, bsort_comm* c) {
  NcclApi& N = nccl();
  if (!N.CommGetAsyncError) return cuda_status(cudaStreamSynchronize(s));
  const double limit = nccl_timeout_s();
  const auto t0 = std::chrono::steady_clock::now();
  unsigned spins = 0;
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return BSORT_SUCCESS;
    if (q != cudaErrorNotReady) return cuda_status(q);
    ncclResult_t ae = ncclSuccess;
    if (N.CommGetAsyncError(c->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
      return abort_comm(c, ae);
    if (limit > 0 && std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit)
      return abort_comm(c, ncclInternalError);
    if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

}  // namespace

namespace {

// The communicator's cached workspace, at least `bytes`, ordered after its previous use on
// whatever stream that was.  Growing frees the old block stream-ordered (its contents are dead:
// callers grow only between phases).  nullptr on allocation failure.
void* comm_ws(bsort_comm* c, size_t bytes, cudaStream_t s) {
  if (c->ws_done) cudaStreamWaitEvent(s, c->ws_done, 0);
  if (bytes <= c->ws_bytes && c->ws) return c->ws;
  if (c->ws) cudaFreeAsync(c->ws, s);
  c->ws = nullptr;
  c->ws_bytes = 0;
  if (cudaMallocAsync(&c->ws, bytes, s) != cudaSuccess) {
    cudaGetLastError();
    c->ws = nullptr;
    return nullptr;
  }
  c->ws_bytes = bytes;
  return c->ws;
}

// Marks the end of a call's use of the cached workspace (on every exit path).
struct WsUse {
  bsort_comm* c;
  cudaStream_t s;
  ~WsUse() {
    if (!c->ws_done && cudaEventCreateWithFlags(&c->ws_done, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      c->ws_done = nullptr;
      cudaStreamSynchronize(s);  // no event: order the next call by draining this one
      return;
    }
    cudaEventRecord(c->ws_done, s);
  }
};

struct RefineCtx {
  NcclApi* N;
  bsort_comm* c;
  bsort_dtype_t dtype;
  const void* keys;
  uint64_t n;
  bsort_direction_t dir;
  uint64_t* dev_hist;  // BSORT_DIST_MAX_RANKS * 65536 u64
  cudaStream_t s;
};

// bsort_refine_fn for the native exact mode: local refinement histograms, NCCL all-reduce, D2H.
int refine_cb(void* p, const uint64_t* prefixes, int m, int prefix_bits, uint64_t* hist) {
  auto* r = static_cast<RefineCtx*>(p);
  if (bsort_dist_refine_hist(r->dtype, r->keys, r->n, r->dir, prefixes, m, prefix_bits, r->dev_hist, r->s) !=
      BSORT_SUCCESS)
    return 1;
  const size_t cnt = (size_t)m * BSORT_DIST_BINS;
  if (r->N->AllReduce(r->dev_hist, r->dev_hist, cnt, ncclUint64, ncclSum, r->c->comm, r->s) != ncclSuccess) return 2;
  if (cudaMemcpyAsync(hist, r->dev_hist, cnt * 8, cudaMemcpyDeviceToHost, r->s) != cudaSuccess) return 3;
  return wait_watching(r->s, r->c) == BSORT_SUCCESS ? 0 : 4;
}

// ---------------------------------------------------------------- fused exchange (§8 N1)

struct PeerPads {
  unsigned* p[BSORT_DIST_MAX_RANKS];
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Device-side barrier over the ranks' signal pads (no host round trip): thread q tells rank q
// that this rank reached barrier `epoch` (a system-scope release store into q's pad, over
// NVLink for a peer) and waits until rank q has told this rank the same.  The release orders
// every earlier write of this stream -- the partition kernel's remote stores -- before the
// signal.  A peer that never arrives (dead process) would hang the stream: after timeout_ns
// the thread gives up and sets the error word, which the host checks.
__global__ void k_peer_barrier(PeerPads pads, unsigned* mine, int me, int P, unsigned epoch,
                               unsigned long long timeout_ns) {
  const int q = threadIdx.x;
  if (q >= P) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pads.p[q] + me), "r"(epoch) : "memory");
  const unsigned long long t0 = globaltimer_ns();
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + q) : "memory");
    if ((int)(v - epoch) >= 0) break;
    if (timeout_ns && globaltimer_ns() - t0 > timeout_ns) {
      atomicExch(mine + BSORT_DIST_MAX_RANKS, 1u);
      break;
    }
    __nanosleep(256);
  }
}

bsort_status_t peer_barrier(bsort_comm* c, cudaStream_t s) {
  PeerPads pp{};
  for (int q = 0; q < c->nranks; ++q) pp.p[q] = c->peer_pad[q];
  const double lim = nccl_timeout_s();
  const unsigned long long tns = lim > 0 ? (unsigned long long)(lim * 1e9) : 0ull;
  BSORT_LAUNCH(bsort::PROF_DIST_PART, s,
               k_peer_barrier<<<1, 64, 0, s>>>(pp, c->pad, c->rank, c->nranks, ++c->epoch, tns));
  return BSORT_SUCCESS;
}

// All-gather of one 64-byte CUDA IPC handle per rank (through NCCL) and the mapping of every
// peer's allocation into this process; out[me] = mine.
bsort_status_t exchange_handles(bsort_comm* c, void* mine, void** out, cudaStream_t s) {
  NcclApi& N = nccl();
  const int P = c->nranks, me = c->rank;
  out[me] = mine;
  if (P == 1) return BSORT_SUCCESS;
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, mine));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  CUDA_TRY(cudaMemcpyAsync(c->hbuf + (size_t)me * 64, &h, 64, cudaMemcpyHostToDevice, s));
  NCCL_TRY(N.AllGather(c->hbuf + (size_t)me * 64, c->hbuf, 64, ncclUint8, c->comm, s));
  std::vector<cudaIpcMemHandle_t> all(P);
  CUDA_TRY(cudaMemcpyAsync(all.data(), c->hbuf, (size_t)P * 64, cudaMemcpyDeviceToHost, s));
  BS_TRY(wait_watching(s, c));
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    void* p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, all[q], cudaIpcMemLazyEnablePeerAccess));
    out[q] = p;
  }
  return BSORT_SUCCESS;
}

void close_peers(bsort_comm* c, void** arr) {
  for (int q = 0; q < c->nranks; ++q) {
    if (q != c->rank && arr[q]) cudaIpcCloseMemHandle(arr[q]);
    arr[q] = nullptr;
  }
}

// First fused call: signal pads (zeroed; epochs only grow) and the handle staging buffer.
bsort_status_t ensure_pads(bsort_comm* c, cudaStream_t s) {
  if (c->pad) return BSORT_SUCCESS;
  CUDA_TRY(cudaMalloc(&c->hbuf, (size_t)BSORT_DIST_MAX_RANKS * 64));
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&c->pad), (BSORT_DIST_MAX_RANKS + 32) * sizeof(unsigned)));
  CUDA_TRY(cudaMemsetAsync(c->pad, 0, (BSORT_DIST_MAX_RANKS + 32) * sizeof(unsigned), s));
  CUDA_TRY(cudaStreamSynchronize(s));  // zeroed before any peer can signal into it
  void* tmp[BSORT_DIST_MAX_RANKS] = {};
  BS_TRY(exchange_handles(c, c->pad, tmp, s));
  for (int q = 0; q < c->nranks; ++q) c->peer_pad[q] = static_cast<unsigned*>(tmp[q]);
  return BSORT_SUCCESS;
}

// Receive buffers of at least `bytes` on EVERY rank (collective: all ranks evaluate the same
// condition from the all-gathered counts, so they grow together).  Old mappings are closed and
// the old buffer freed only after every rank has mapped the new one (NCCL all-reduce as the
// barrier).
bsort_status_t ensure_rbuf(bsort_comm* c, size_t bytes, cudaStream_t s) {
  if (bytes <= c->rbytes && c->rbuf) return BSORT_SUCCESS;
  NcclApi& N = nccl();
  const size_t nb = round_up(std::max(bytes, c->rbytes + c->rbytes / 2), 1 << 21);
  void* fresh = nullptr;
  CUDA_TRY(cudaMalloc(&fresh, nb));
  void* old = c->rbuf;
  close_peers(c, c->peer_rbuf);
  c->rbuf = fresh;
  c->rbytes = nb;
  BS_TRY(exchange_handles(c, fresh, c->peer_rbuf, s));
  if (old) {
    NCCL_TRY(N.AllReduce(c->hbuf, c->hbuf, 1, ncclUint8, ncclMax, c->comm, s));
    BS_TRY(wait_watching(s, c));
    cudaFree(old);
  }
  return BSORT_SUCCESS;
}

bsort_status_t sort_dist_impl(bsort_dtype_t dtype, const void* dev_in, uint64_t n, void* dev_out, uint64_t cap,
                              uint64_t* n_out, bsort_direction_t dir, bool exact, bool fused, bsort_comm* c,
                              cudaStream_t s) {
  NcclApi& N = nccl();
  if (c->aborted) return nccl_status(ncclInvalidUsage);
  const int P = c->nranks, me = c->rank;
  const int es = key_bytes(dtype);
  exact = exact && P > 1;  // one rank: every key stays, both modes coincide

  // One device block: [global hist | local hist | counts | refinement hists | bucketed keys | ws]
  // The local sort's workspace reuses the bucketed keys + partition workspace after the exchange.
  // Counts: bin mode P x (P+1) (send counts + capacity), exact mode P x (2(P-1)+2) (class counts +
  // capacity).
  const size_t hist_b = (size_t)BSORT_DIST_BINS * 8;
  const int CW = exact ? 2 * (P - 1) + 2 : P + 1;  // u64 words per rank in the gathered counts
  const size_t cnt_b = round_up((size_t)P * CW * 8, 256);
  const size_t ref_b = exact ? (size_t)(P - 1) * BSORT_DIST_BINS * 8 : 0;
  const size_t bucket_b = fused ? 0 : round_up((size_t)n * es, 256);  // fused: no bucketed copy
  const size_t part_ws = exact ? bsort_dist_class_partition_workspace_bytes()
                               : bsort_dist_partition_workspace_bytes(dtype, n, P);
  const size_t head = 2 * hist_b + cnt_b + ref_b;
  // the communicator's cached workspace: [head | tail], the tail holding the partition phase;
  // the local sort's workspace (size known only after the counts all-gather) reuses the whole
  // block, grown if needed once the partition phase is dead
  const size_t tail = bucket_b + part_ws;
  WsUse use{c, s};
  char* base = static_cast<char*>(comm_ws(c, head + tail, s));
  if (!base) return BSORT_ERROR_OUT_OF_MEMORY;
  uint64_t* g_hist = reinterpret_cast<uint64_t*>(base);
  uint64_t* l_hist = reinterpret_cast<uint64_t*>(base + hist_b);
  uint64_t* d_cnt = reinterpret_cast<uint64_t*>(base + 2 * hist_b);
  char* bucket = base + head;
  char* ws = bucket + bucket_b;

  // a7: local histogram, global = all-reduce(sum)
  BS_TRY(bsort_dist_top_hist(dtype, dev_in, n, dir, l_hist, s));
  NCCL_TRY(N.AllReduce(l_hist, g_hist, BSORT_DIST_BINS, ncclUint64, ncclSum, c->comm, s));
  std::vector<uint64_t> hist(2 * (size_t)BSORT_DIST_BINS);
  CUDA_TRY(cudaMemcpyAsync(hist.data(), g_hist, 2 * hist_b, cudaMemcpyDeviceToHost, s));
  BS_TRY(wait_watching(s, c));

  // a8: per-destination counts of every rank, all-gathered with every rank's capacity.
  // sendm[src * P + dst] = keys src sends to dst; caps[q] = rank q's out_capacity.
  std::vector<uint64_t> sendm((size_t)P * P), caps(P);
  std::vector<uint32_t> cuts(P + 1);
  std::vector<uint64_t> values(P), quota(P), my_classes;
  std::vector<int> idx(P);
  int m = 0;
  if (!exact) {
    std::vector<uint64_t> mine(P + 1);
    BS_TRY(bsort_dist_splitters(hist.data(), P, cuts.data()));
    BS_TRY(bsort_dist_send_counts(hist.data() + BSORT_DIST_BINS, cuts.data(), P, mine.data()));
    mine[P] = cap;
    CUDA_TRY(cudaMemcpyAsync(d_cnt + (size_t)me * CW, mine.data(), CW * 8, cudaMemcpyHostToDevice, s));
    NCCL_TRY(N.AllGather(d_cnt + (size_t)me * CW, d_cnt, CW, ncclUint64, c->comm, s));
    std::vector<uint64_t> all((size_t)P * CW);
    CUDA_TRY(cudaMemcpyAsync(all.data(), d_cnt, all.size() * 8, cudaMemcpyDeviceToHost, s));
    BS_TRY(wait_watching(s, c));
    for (int q = 0; q < P; ++q) {
      for (int d = 0; d < P; ++d) sendm[(size_t)q * P + d] = all[(size_t)q * CW + d];
      caps[q] = all[(size_t)q * CW + P];
    }
  } else {
    // §8 N2: exact boundaries by refinement histograms, then class counts of every rank
    uint64_t N_total = 0;
    for (int b = 0; b < BSORT_DIST_BINS; ++b) N_total += hist[b];
    if (N_total > 0) {
      RefineCtx rc{&N, c, dtype, dev_in, n, dir, reinterpret_cast<uint64_t*>(base + 2 * hist_b + cnt_b), s};
      BS_TRY(bsort_dist_exact_boundaries(hist.data(), P, es * 8, refine_cb, &rc, values.data(), &m, idx.data(),
                                         quota.data(), nullptr));
      const int C = 2 * m + 1;
      BS_TRY(bsort_dist_class_hist(dtype, dev_in, n, dir, values.data(), m, d_cnt + (size_t)me * CW, s));
      CUDA_TRY(cudaMemcpyAsync(d_cnt + (size_t)me * CW + C, &cap, 8, cudaMemcpyHostToDevice, s));
      NCCL_TRY(N.AllGather(d_cnt + (size_t)me * CW, d_cnt, CW, ncclUint64, c->comm, s));
      std::vector<uint64_t> all((size_t)P * CW);
      CUDA_TRY(cudaMemcpyAsync(all.data(), d_cnt, all.size() * 8, cudaMemcpyDeviceToHost, s));
      BS_TRY(wait_watching(s, c));
      std::vector<uint64_t> cc((size_t)P * C);
      for (int q = 0; q < P; ++q) {
        for (int k = 0; k < C; ++k) cc[(size_t)q * C + k] = all[(size_t)q * CW + k];
        caps[q] = all[(size_t)q * CW + C];
      }
      for (int q = 0; q < P; ++q)  // every rank's send counts follow from the gathered classes
        BS_TRY(bsort_dist_exact_send_counts(cc.data(), P, m, q, idx.data(), quota.data(), &sendm[(size_t)q * P]));
      my_classes.assign(cc.begin() + (size_t)me * C, cc.begin() + (size_t)(me + 1) * C);
    } else {  // no keys anywhere: nothing moves (capacities irrelevant)
      for (int q = 0; q < P; ++q) caps[q] = ~0ull;
    }
  }
  auto sent = [&](int src, int dst) { return sendm[(size_t)src * P + dst]; };

  // capacity: every rank checks every rank, so all return the same status
  uint64_t recv_total = 0;
  bool overflow = false;
  for (int q = 0; q < P; ++q) {
    uint64_t tot = 0;
    for (int r = 0; r < P; ++r) tot += sent(r, q);
    if (q == me) recv_total = tot;
    if (tot > caps[q]) overflow = true;
  }
  if (n_out) *n_out = recv_total;
  if (overflow) return BSORT_ERROR_CAPACITY;

  if (fused) {
    // §8 N1: the partition's write-out IS the exchange -- keys for rank q are stored straight
    // into q's receive buffer (peer-mapped over NVLink) at the slots after the keys of the ranks
    // before this one; two device-side barriers replace the host syncs of the NCCL exchange.
    BS_TRY(ensure_pads(c, s));
    uint64_t need = 1;
    for (int q = 0; q < P; ++q) {
      uint64_t tot = 0;
      for (int r = 0; r < P; ++r) tot += sent(r, q);
      need = std::max(need, tot);
    }
    BS_TRY(ensure_rbuf(c, (size_t)need * es, s));
    std::vector<uint64_t> dst(P);
    for (int q = 0; q < P; ++q) {
      uint64_t off = 0;
      for (int r = 0; r < me; ++r) off += sent(r, q);
      dst[q] = reinterpret_cast<uint64_t>(c->peer_rbuf[q]) + off * es;
    }
    BS_TRY(peer_barrier(c, s));  // every owner is done with its buffer's previous contents
    if (n > 0)
      BS_TRY(bsort_dist_partition_remote(dtype, dev_in, n, dir, cuts.data(), &sendm[(size_t)me * P], P, dst.data(),
                                         ws, part_ws, s));
    BS_TRY(peer_barrier(c, s));  // every rank's keys for this rank have landed
    unsigned err = 0;
    CUDA_TRY(cudaMemcpyAsync(&err, c->pad + BSORT_DIST_MAX_RANKS, sizeof(err), cudaMemcpyDeviceToHost, s));
    BS_TRY(wait_watching(s, c));
    if (err) return abort_comm(c, ncclRemoteError);  // a peer never reached the barrier
    if (recv_total > 1) {
      const size_t wsb = bsort_workspace_bytes(dtype, recv_total);
      void* sws = comm_ws(c, wsb, s);
      if (!sws) return BSORT_ERROR_OUT_OF_MEMORY;
      BS_TRY(bsort_sort_ws(dtype, c->rbuf, recv_total, dir, sws, wsb, s));
    }
    if (recv_total)
      CUDA_TRY(cudaMemcpyAsync(dev_out, c->rbuf, (size_t)recv_total * es, cudaMemcpyDeviceToDevice, s));
    return BSORT_SUCCESS;
  }

  // a9: bucketed copy (bucket q = keys for rank q, contiguous)
  if (n > 0) {
    if (exact)
      BS_TRY(bsort_dist_partition_classes(dtype, dev_in, n, dir, values.data(), m, my_classes.data(), bucket, ws,
                                          part_ws, s));
    else
      BS_TRY(bsort_dist_partition(dtype, dev_in, n, dir, cuts.data(), &sendm[(size_t)me * P], P, bucket, ws,
                                  part_ws, s));
  }

  // a10: grouped send/recv; rank r's keys land at sum_{r'<r} sent(r', me) in dev_out
  bsort::prof_begin(bsort::PROF_DIST_A2A, s);
  NCCL_TRY(N.GroupStart());
  ncclResult_t first = ncclSuccess;
  uint64_t soff = 0, roff = 0;
  for (int q = 0; q < P; ++q) {
    const uint64_t sc = sent(me, q), rc = sent(q, me);
    ncclResult_t r = ncclSuccess;
    if (sc) r = N.Send(bucket + soff * es, sc * es, ncclUint8, q, c->comm, s);
    if (first == ncclSuccess) first = r;
    if (rc) r = N.Recv(static_cast<char*>(dev_out) + roff * es, rc * es, ncclUint8, q, c->comm, s);
    if (first == ncclSuccess) first = r;
    soff += sc;
    roff += rc;
  }
  const ncclResult_t ge = N.GroupEnd();
  bsort::prof_end(bsort::PROF_DIST_A2A, s);
  NCCL_TRY(first);
  NCCL_TRY(ge);
  // the exchange is where a dead peer would hang every rank: wait for it watching the comm
  BS_TRY(wait_watching(s, c));

  // a11: local sort of the received keys in the cached workspace (everything in it is dead
  // now), grown to the local sort's size for recv_total keys if that exceeds it
  if (recv_total > 1) {
    const size_t wsb = bsort_workspace_bytes(dtype, recv_total);
    void* sws = comm_ws(c, wsb, s);
    if (!sws) return BSORT_ERROR_OUT_OF_MEMORY;
    BS_TRY(bsort_sort_ws(dtype, dev_out, recv_total, dir, sws, wsb, s));
  }
  return BSORT_SUCCESS;
}

}  // namespace

extern "C" {

bsort_status_t bsort_get_unique_id(uint8_t id[128]) {
  if (!id) return BSORT_ERROR_INVALID_ARGUMENT;
  NcclApi& N = nccl();
  if (!N.ok) return BSORT_ERROR_NCCL;
  ncclUniqueId u;
  NCCL_TRY(N.GetUniqueId(&u));
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
  return BSORT_SUCCESS;
}

bsort_status_t bsort_comm_init(bsort_comm_t* out, const uint8_t id[128], int nranks, int rank) {
  if (!out || !id || nranks < 1 || nranks > BSORT_DIST_MAX_RANKS || rank < 0 || rank >= nranks)
    return BSORT_ERROR_INVALID_ARGUMENT;
  NcclApi& N = nccl();
  if (!N.ok) return BSORT_ERROR_NCCL;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  auto* c = new bsort_comm;
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->device);
  ncclResult_t r = N.CommInitRank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_status(r);
  }
  *out = c;
  return BSORT_SUCCESS;
}

bsort_status_t bsort_comm_destroy(bsort_comm_t c) {
  if (!c) return BSORT_ERROR_INVALID_ARGUMENT;
  NcclApi& N = nccl();
  // an aborted communicator was already released by ncclCommAbort
  ncclResult_t r = N.ok && c->comm && !c->aborted ? N.CommDestroy(c->comm) : ncclSuccess;
  if (c->ws_done) {
    cudaEventSynchronize(c->ws_done);
    cudaEventDestroy(c->ws_done);
  }
  if (c->ws) cudaFree(c->ws);
  close_peers(c, c->peer_rbuf);
  close_peers(c, reinterpret_cast<void**>(c->peer_pad));
  if (c->rbuf) cudaFree(c->rbuf);
  if (c->pad) cudaFree(c->pad);
  if (c->hbuf) cudaFree(c->hbuf);
  delete c;
  return nccl_status(r);
}

int bsort_comm_size(bsort_comm_t c) { return c ? c->nranks : 0; }
int bsort_comm_rank(bsort_comm_t c) { return c ? c->rank : -1; }

bsort_status_t bsort_sort_dist(bsort_dtype_t dtype, const void* dev_in, uint64_t n_local, void* dev_out,
                               uint64_t out_capacity, uint64_t* n_out, bsort_direction_t direction,
                               bsort_comm_t comm, void* stream) {
  if (!comm || !comm->comm) return BSORT_ERROR_INVALID_ARGUMENT;
  if (direction != BSORT_ASCENDING && direction != BSORT_DESCENDING) return BSORT_ERROR_INVALID_ARGUMENT;
  const int es = key_bytes(dtype);
  if (es == 0) return BSORT_ERROR_UNSUPPORTED_DTYPE;
  if (n_local > 0 && (!dev_in || (uintptr_t)dev_in % es)) return BSORT_ERROR_INVALID_ARGUMENT;
  if (out_capacity > 0 && (!dev_out || (uintptr_t)dev_out % es)) return BSORT_ERROR_INVALID_ARGUMENT;
  if (dev_out && dev_in && dev_out == dev_in && n_local > 0) return BSORT_ERROR_INVALID_ARGUMENT;
  return sort_dist_impl(dtype, dev_in, n_local, dev_out, out_capacity, n_out, direction, false, false, comm,
                        (cudaStream_t)stream);
}

bsort_status_t bsort_sort_dist_ex(bsort_dtype_t dtype, const void* dev_in, uint64_t n_local, void* dev_out,
                                  uint64_t out_capacity, uint64_t* n_out, bsort_direction_t direction,
                                  unsigned flags, bsort_comm_t comm, void* stream) {
  if ((flags & ~(BSORT_DIST_EXACT | BSORT_DIST_FUSED)) != 0) return BSORT_ERROR_INVALID_ARGUMENT;
  if ((flags & BSORT_DIST_EXACT) && (flags & BSORT_DIST_FUSED)) return BSORT_ERROR_INVALID_ARGUMENT;
  if (!comm || !comm->comm) return BSORT_ERROR_INVALID_ARGUMENT;
  if (direction != BSORT_ASCENDING && direction != BSORT_DESCENDING) return BSORT_ERROR_INVALID_ARGUMENT;
  const int es = key_bytes(dtype);
  if (es == 0) return BSORT_ERROR_UNSUPPORTED_DTYPE;
  if (n_local > 0 && (!dev_in || (uintptr_t)dev_in % es)) return BSORT_ERROR_INVALID_ARGUMENT;
  if (out_capacity > 0 && (!dev_out || (uintptr_t)dev_out % es)) return BSORT_ERROR_INVALID_ARGUMENT;
  if (dev_out && dev_in && dev_out == dev_in && n_local > 0) return BSORT_ERROR_INVALID_ARGUMENT;
  return sort_dist_impl(dtype, dev_in, n_local, dev_out, out_capacity, n_out, direction,
                        (flags & BSORT_DIST_EXACT) != 0, (flags & BSORT_DIST_FUSED) != 0, comm, (cudaStream_t)stream);
}

int bsort_last_nccl_error(void) { return t_last_nccl; }

}  // extern "C"
