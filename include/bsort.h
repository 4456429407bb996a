/*
 * bsort.h — C ABI of the B200-native bsort hot path (arxiv 2603.08929).
 *
 * What is computed.  bsort_sort() puts n keys of one of ten machine types into the order the
 * paper defines (problem statement PAPER P:27 "a monotonically non-decreasing or
 * non-increasing sequence"): numeric order for unsigned and two's-complement keys
 * (Algorithms 2-3) and, for IEEE-754 keys, sign -> exponent -> mantissa order with
 * negatives inverted (Algorithms 4-5 and Theorems 2-3), which places
 * -NaN(larger payload first) < -inf < ... < -0 < +0 < ... < +inf < +NaN(larger payload last)
 * (P:609-617).  Descending is exactly the reverse.  The order is a total order on bit
 * patterns, so the output is unique and compared bit-for-bit (no float arithmetic on keys).
 *
 * How (not part of the contract): an order-preserving key transform fused into every kernel;
 * 32/64-bit keys by a one-sweep LSD radix sort (8-bit digits); 8/16-bit keys by one counting
 * pass.  See DESIGN.md.
 *
 * Conventions for every entry point:
 *  - All sizes are 64-bit.  `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Work is enqueued on `stream`; calls return after enqueue (no host sync) unless
 *    stated otherwise.  Asynchronous kernel faults surface at the caller's next sync.
 *  - Device pointers must be device-accessible and aligned to the element size.  No other
 *    alignment is required.
 *  - Argument errors return before anything is enqueued and leave all buffers untouched.
 *  - The library keeps no hidden state besides a device-property cache, the launch counter and
 *    the optional profiler.  Concurrent calls on different streams with distinct workspaces
 *    are safe.
 *  - On BSORT_ERROR_CUDA, bsort_last_cuda_error() returns the raw cudaError_t (thread-local).
 */
#ifndef BSORT_H
#define BSORT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Key types: Table II word sizes plus the unsigned variants, and the half-width
 * floats f16/bf16 (the paper's method applies to any float layout sign | exponent | mantissa,
 * P:498).  Values are ABI. */
typedef enum {
  BSORT_U8 = 0,
  BSORT_I8 = 1,
  BSORT_U16 = 2,
  BSORT_I16 = 3,
  BSORT_U32 = 4,
  BSORT_I32 = 5,
  BSORT_F32 = 6,
  BSORT_U64 = 7,
  BSORT_I64 = 8,
  BSORT_F64 = 9,
  BSORT_F16 = 10,  /* IEEE binary16 (1 | 5 | 10), same order rules as f32/f64 */
  BSORT_BF16 = 11  /* bfloat16 (1 | 8 | 7) */
} bsort_dtype_t;

/* Sort direction: Algorithm 1's boolean `asc`. */
typedef enum { BSORT_ASCENDING = 0, BSORT_DESCENDING = 1 } bsort_direction_t;

typedef enum {
  BSORT_SUCCESS = 0,
  BSORT_ERROR_INVALID_ARGUMENT = 1,   /* NULL/misaligned pointer, bad enum, bad nranks/cuts  */
  BSORT_ERROR_UNSUPPORTED_DTYPE = 2,  /* dtype not valid for this entry point               */
  BSORT_ERROR_OUT_OF_MEMORY = 3,      /* cudaMallocAsync of the internal workspace failed    */
  BSORT_ERROR_WORKSPACE_TOO_SMALL = 4,/* workspace_bytes < the *_workspace_bytes() figure    */
  BSORT_ERROR_CUDA = 5,               /* a CUDA runtime call or launch failed                */
  BSORT_ERROR_NCCL = 6,               /* NCCL missing or an NCCL call failed (bsort_last_nccl_error) */
  BSORT_ERROR_CAPACITY = 7            /* bsort_sort_dist: some rank's dev_out is too small    */
} bsort_status_t;

/* ----------------------------------------------------------------------- single GPU */

/* Bytes of scratch device memory bsort_sort_ws() needs for (dtype, n) on the CURRENT device.
 * 0 for n <= 1.  32/64-bit keys: n*sizeof(key) ping-pong buffer + histograms + look-back
 * descriptors; 8/16-bit keys: histogram only (the counting path is in place). */
size_t bsort_workspace_bytes(bsort_dtype_t dtype, uint64_t n);

/* Sort `n` keys at `dev_keys` in place.  Scratch is allocated with cudaMallocAsync on
 * `stream` and released with cudaFreeAsync on the same stream. */
bsort_status_t bsort_sort(bsort_dtype_t dtype, void* dev_keys, uint64_t n,
                          bsort_direction_t direction, void* stream);

/* As bsort_sort(), with caller-owned scratch: `workspace` (device, 256-byte aligned) of at
 * least bsort_workspace_bytes(dtype, n) bytes.  The workspace must not be used by anything
 * else until the enqueued work completes. */
bsort_status_t bsort_sort_ws(bsort_dtype_t dtype, void* dev_keys, uint64_t n,
                             bsort_direction_t direction, void* workspace,
                             size_t workspace_bytes, void* stream);

/* End-to-end form with HOST keys: enqueues host->device copy of `host_keys` into `dev_keys`
 * (n keys, caller-owned), the sort, and the device->host copy back into `host_keys`.
 * `host_keys` should be pinned (cudaHostAlloc / torch pin_memory) for the copies to be
 * asynchronous; the caller synchronises `stream` before reading `host_keys`. */
bsort_status_t bsort_sort_host(bsort_dtype_t dtype, void* host_keys, uint64_t n,
                               bsort_direction_t direction, void* dev_keys, void* workspace,
                               size_t workspace_bytes, void* stream);

/* Out-of-place end-to-end form: H2D of `host_in` (n keys, read only) into `dev_keys`, the sort,
 * and D2H of the result into `host_out` (n keys; may equal host_in, then this is
 * bsort_sort_host).  Both host buffers should be pinned.  Because host_in is never written, a
 * caller can keep several sorts in flight on different streams (each with its own dev_keys,
 * workspace and host_out): one sort's D2H then overlaps the next one's H2D and sort, and PCIe
 * carries both directions at once.  Errors as bsort_sort_host(). */
bsort_status_t bsort_sort_host_to(bsort_dtype_t dtype, const void* host_in, void* host_out, uint64_t n,
                                  bsort_direction_t direction, void* dev_keys, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* ----------------------------------------------------------- key-value sort
 * Sort n keys of a 32/64-bit dtype (u32/i32/f32/u64/i64/f64; 8/16-bit keys return
 * BSORT_ERROR_UNSUPPORTED_DTYPE) and move the n uint32 values at dev_values (device,
 * 4-byte aligned) with them: afterwards value i is the one that was paired with key i.  Keys end
 * up exactly as bsort_sort() leaves them; the order of the values of EQUAL keys is unspecified
 * (the sort is not stable).  argsort: pass values 0..n-1.  The workspace holds an extra n
 * uint32 ping-pong buffer.  Errors as bsort_sort(). */
size_t bsort_pairs_workspace_bytes(bsort_dtype_t dtype, uint64_t n);
bsort_status_t bsort_sort_pairs_ws(bsort_dtype_t dtype, void* dev_keys, uint32_t* dev_values, uint64_t n,
                                   bsort_direction_t direction, void* workspace, size_t workspace_bytes,
                                   void* stream);
bsort_status_t bsort_sort_pairs(bsort_dtype_t dtype, void* dev_keys, uint32_t* dev_values, uint64_t n,
                                bsort_direction_t direction, void* stream);

/* ------------------------------------------------ in-place mode / hybrid
 * Sorts like bsort_sort() (same order, same result bit for bit) with O(n/128 + SMs*128 KiB)
 * scratch plus the LSD scratch of `chunk_keys` keys, instead of an n-key buffer: 256-way MSD
 * partitions IN PLACE (the paper's Algorithm 1 generalised from one bit to one 8-bit digit,
 * P:151-157, recursing MSD-first like Algorithm 2; Theorem 5's in-place property,
 * P:761-775), until every group of consecutive buckets holds at most chunk_keys keys; each group
 * is then sorted by the one-sweep LSD path (the paper's hybrid idea).
 * chunk_keys = 0 picks max(2^22, n/32) (capped at n).  8/16-bit keys use the counting path, which
 * is in place already.  Blocks the host once per partition (bucket sizes decide the recursion).
 * Workspace: bsort_inplace_workspace_bytes(dtype, n, chunk_keys) bytes, 256-byte aligned. */
size_t bsort_inplace_workspace_bytes(bsort_dtype_t dtype, uint64_t n, uint64_t chunk_keys);
bsort_status_t bsort_sort_inplace_ws(bsort_dtype_t dtype, void* dev_keys, uint64_t n,
                                     bsort_direction_t direction, uint64_t chunk_keys, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* ------------------------------------------------------ multi-GPU building blocks (MSD)
 * The distributed sort (BASELINE.json cfg5) is an MSD range partition on the top 16 bits of
 * the transformed key (the paper's sign -> exponent -> mantissa hierarchy, makes
 * the top bits of the key the most significant), one key exchange, and a local bsort_sort.
 * The collectives themselves (all-reduce of the histogram, all-to-all of counts and keys)
 * are issued by the caller over its process group (paper_2603_08929_b200.sort_dist does it
 * with torch.distributed / NCCL); these calls are the compute steps around them. */

#define BSORT_DIST_BINS 65536
#define BSORT_DIST_MAX_RANKS 64

/* dev_hist[b] (uint64, BSORT_DIST_BINS entries, overwritten) = number of the n keys at
 * dev_keys whose transformed key (direction folded in) has top-16-bit value b.
 * 32/64-bit dtypes only. */
bsort_status_t bsort_dist_top_hist(bsort_dtype_t dtype, const void* dev_keys, uint64_t n,
                                   bsort_direction_t direction, uint64_t* dev_hist,
                                   void* stream);

/* HOST function (no GPU).  From the global histogram (host, BSORT_DIST_BINS entries) pick
 * cuts[0..nranks] (host): cuts[0] = 0, cuts[nranks] = BSORT_DIST_BINS and, for 0 < r < nranks,
 * cuts[r] = the smallest bin b with sum(hist[0..b)) >= floor(r * total / nranks).  Rank r owns
 * bins [cuts[r], cuts[r+1]).  cuts is non-decreasing. */
bsort_status_t bsort_dist_splitters(const uint64_t* host_global_hist, int nranks,
                                    uint32_t* host_cuts);

/* HOST function.  send_counts[q] (host, nranks entries) = sum of local_hist over q's bins. */
bsort_status_t bsort_dist_send_counts(const uint64_t* host_local_hist, const uint32_t* host_cuts,
                                      int nranks, uint64_t* host_send_counts);

size_t bsort_dist_partition_workspace_bytes(bsort_dtype_t dtype, uint64_t n, int nranks);

/* Partition of the n keys at dev_in into dev_out (n keys, distinct from dev_in), grouped by
 * destination rank q = the rank owning the key's top-16-bit bin under host_cuts (nranks+1
 * entries).  host_send_counts (nranks entries, from bsort_dist_send_counts on this rank's
 * histogram, summing to n) fixes the bucket starts: bucket q begins at sum(send_counts[0..q)).
 * Keys keep their raw bits.  The order inside a bucket is unspecified (every rank sorts what it
 * receives, so the MSD step needs no stability).  Returns BSORT_ERROR_INVALID_ARGUMENT if the
 * send counts do not sum to n. */
bsort_status_t bsort_dist_partition(bsort_dtype_t dtype, const void* dev_in, uint64_t n,
                                    bsort_direction_t direction, const uint32_t* host_cuts,
                                    const uint64_t* host_send_counts, int nranks, void* dev_out,
                                    void* workspace, size_t workspace_bytes, void* stream);

/* Fused partition + exchange.  As bsort_dist_partition, but every key of
 * destination rank q is stored directly at a slot in the device byte range
 * [dst_addrs[q], dst_addrs[q] + host_send_counts[q] * sizeof(key)) -- normally rank q's
 * receive buffer mapped into this process (torch symmetric memory / CUDA IPC peer mapping over
 * NVLink), at the offset where this rank's keys for q begin (the exclusive prefix, over source
 * ranks, of what q receives).  No local bucketed copy and no separate keys all-to-all: the
 * partition's coalesced write-out is the exchange.  Exactly host_send_counts[q] keys land in
 * range q, in unspecified order.  dst_addrs (host, nranks entries) must be element-aligned and
 * non-null where host_send_counts[q] > 0.  The caller synchronises the ranks (e.g. a barrier
 * after this stream's work completes) before any rank reads its receive buffer.  Workspace as
 * bsort_dist_partition_workspace_bytes(). */
bsort_status_t bsort_dist_partition_remote(bsort_dtype_t dtype, const void* dev_in, uint64_t n,
                                           bsort_direction_t direction, const uint32_t* host_cuts,
                                           const uint64_t* host_send_counts, int nranks,
                                           const uint64_t* host_dst_addrs, void* workspace,
                                           size_t workspace_bytes, void* stream);

/* Exact splitting: the building blocks that make every rank's shard exactly
 * floor((r+1)N/P) - floor(rN/P) keys whatever the skew (paper_2603_08929_b200.sort_dist(...,
 * exact=True) drives them).  All keys below are TRANSFORMED keys (the order key with the
 * direction folded in), as unsigned integers of the dtype's width.
 *
 * bsort_dist_refine_hist: dev_hist (uint64, m * 65536, overwritten) counts, for each of the m
 * prefixes (host, strictly increasing), the keys whose top `prefix_bits` bits equal
 * prefixes[j], binned by their next 16 bits: dev_hist[j * 65536 + b].  prefix_bits is a
 * multiple of 16 with prefix_bits + 16 <= key bits. */
bsort_status_t bsort_dist_refine_hist(bsort_dtype_t dtype, const void* dev_keys, uint64_t n,
                                      bsort_direction_t direction, const uint64_t* host_prefixes, int m,
                                      int prefix_bits, uint64_t* dev_hist, void* stream);

/* Classes against m distinct split keys values[0..m) (host, strictly increasing, transformed):
 * class 2j holds the keys strictly between values[j-1] and values[j] (values[-1] = -inf,
 * values[m] = +inf), class 2j+1 the keys equal to values[j].  bsort_dist_class_hist writes the
 * 2m+1 class counts to dev_counts (uint64).  bsort_dist_partition_classes partitions the n keys
 * into dev_out grouped by class in increasing class order (class c starts at the sum of
 * host_class_counts[0..c)), order within a class unspecified; the counts must be this rank's
 * (summing to n).  Workspace: bsort_dist_class_partition_workspace_bytes(). */
bsort_status_t bsort_dist_class_hist(bsort_dtype_t dtype, const void* dev_keys, uint64_t n,
                                     bsort_direction_t direction, const uint64_t* host_values, int m,
                                     uint64_t* dev_counts, void* stream);
size_t bsort_dist_class_partition_workspace_bytes(void);
bsort_status_t bsort_dist_partition_classes(bsort_dtype_t dtype, const void* dev_in, uint64_t n,
                                            bsort_direction_t direction, const uint64_t* host_values, int m,
                                            const uint64_t* host_class_counts, void* dev_out,
                                            void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------ native multi-GPU sort (SURVEY §8 b)
 * The complete MSD path (a7-a11) in one call over an NCCL communicator owned by the library:
 * top-16-bit histogram + ncclAllReduce, host splitters (bsort_dist_splitters), ncclAllGather of
 * every rank's send counts and capacity, P-way partition, grouped ncclSend/ncclRecv of the keys,
 * local bsort_sort_ws.  NCCL is loaded at run time (libnccl.so.2); if it cannot be loaded these
 * calls return BSORT_ERROR_NCCL.  One process (or thread) per GPU; each rank calls collectively
 * with its own communicator.
 *
 * bsort_get_unique_id: a fresh ncclUniqueId (128 bytes) on one rank, to be broadcast by the
 * caller.  bsort_comm_init: collective over the nranks ranks, on the CURRENT device; *out owns
 * an ncclComm_t until bsort_comm_destroy.
 *
 * bsort_sort_dist: 32/64-bit dtypes (u32/i32/f32/u64/i64/f64; others UNSUPPORTED_DTYPE).
 * dev_in (n_local keys) is read and may NOT be modified (kept intact); dev_out (device,
 * out_capacity keys, distinct from dev_in) receives this rank's shard sorted in `direction`;
 * the concatenation of the shards over ranks 0..P-1 is the global order.  Shard boundaries are
 * bin-granular (reading Q16).  *n_out (host, nullable) = this rank's shard size.
 * If any rank's shard exceeds its out_capacity, EVERY rank returns BSORT_ERROR_CAPACITY after
 * the counts exchange with nothing written to dev_out (n_out still set).  Blocks the host three
 * times (after the histogram all-reduce, after the counts all-gather, after the keys exchange);
 * scratch is cudaMallocAsync'ed on `stream` (n_local keys + partition workspace; the local
 * sort's workspace is sized from the received count and reuses that block when it fits).
 * Failure detection: while it waits, the call polls ncclCommGetAsyncError; on an asynchronous
 * NCCL error, or when a wait exceeds BSORT_NCCL_TIMEOUT_S seconds (environment, default 300,
 * 0 = no limit: a dead peer), it calls ncclCommAbort and returns BSORT_ERROR_NCCL
 * (bsort_last_nccl_error: the NCCL code, ncclInternalError for a timeout); the communicator is
 * then unusable (later calls return BSORT_ERROR_NCCL; bsort_comm_destroy still frees it). */
typedef struct bsort_comm* bsort_comm_t;
bsort_status_t bsort_get_unique_id(uint8_t id[128]);
bsort_status_t bsort_comm_init(bsort_comm_t* out, const uint8_t id[128], int nranks, int rank);
bsort_status_t bsort_comm_destroy(bsort_comm_t comm);
int bsort_comm_size(bsort_comm_t comm);
int bsort_comm_rank(bsort_comm_t comm);
bsort_status_t bsort_sort_dist(bsort_dtype_t dtype, const void* dev_in, uint64_t n_local, void* dev_out,
                               uint64_t out_capacity, uint64_t* n_out, bsort_direction_t direction,
                               bsort_comm_t comm, void* stream);
/* bsort_sort_dist with options.  flags: 0 = as bsort_sort_dist; BSORT_DIST_EXACT = exact
 * splitting: rank r's shard is exactly floor((r+1)N/P) - floor(rN/P) keys whatever
 * the key distribution (equal keys are split across ranks in rank order).  Exact splitting adds
 * one key read + an all-reduce of m x 65536 u64 per refinement level (bsort_dist_exact_boundaries)
 * and a class histogram + all-gather; it blocks the host once more per level. */
#define BSORT_DIST_EXACT 1u
/* BSORT_DIST_FUSED: no bucketed copy and no NCCL keys exchange -- the partition
 * kernel stores every key directly into its owner's receive buffer, which the communicator owns
 * (cudaMalloc, mapped into every rank by CUDA IPC: all ranks must be processes of one node with
 * peer access), between two device-side barriers on signal pads in the same mapped memory
 * (a peer that never arrives fails the call after BSORT_NCCL_TIMEOUT_S).  The owner sorts its
 * buffer and copies the shard to dev_out.  The receive buffer grows collectively (all ranks
 * decide from the same all-gathered counts) and lives until bsort_comm_destroy.  Not combinable
 * with BSORT_DIST_EXACT (BSORT_ERROR_INVALID_ARGUMENT). */
#define BSORT_DIST_FUSED 2u
bsort_status_t bsort_sort_dist_ex(bsort_dtype_t dtype, const void* dev_in, uint64_t n_local, void* dev_out,
                                  uint64_t out_capacity, uint64_t* n_out, bsort_direction_t direction,
                                  unsigned flags, bsort_comm_t comm, void* stream);
int bsort_last_nccl_error(void);          /* raw ncclResult_t of the last NCCL failure (thread-local) */

/* Host planning of exact splitting (pure host code, no device work; used by
 * bsort_sort_dist_ex(BSORT_DIST_EXACT)).  bsort_dist_exact_boundaries: from the GLOBAL top-16-bit
 * histogram (BSORT_DIST_BINS entries) of N keys of `key_bits` (32 or 64) bits, finds for every
 * boundary r = 1..nranks-1 the transformed key K_r of global rank T_r = floor(r N / nranks) and
 * quota_r = T_r - #{keys < K_r}, descending the key 16 bits at a time (the MSD digit order of
 * P:427-433).  `refine(ctx, prefixes, m, prefix_bits, hist)` must fill hist (m * 65536 u64) with
 * the GLOBAL next-16-bit histograms below the m strictly increasing prefixes (for example
 * bsort_dist_refine_hist + an all-reduce) and return 0.  Outputs: values[0..*m) the distinct
 * K's (increasing), idx[r-1] the index of K_r in values, quota[r-1], *levels the number of
 * refine calls.  Arrays hold nranks-1 entries.  N == 0 with nranks > 1 is INVALID_ARGUMENT.
 * bsort_dist_exact_send_counts: this rank's per-destination counts over its keys grouped by the
 * 2m+1 classes (bsort_dist_partition_classes order), given every rank's class counts
 * (class_counts_all[q * (2m+1) + c]): the keys equal to values[j] go left of boundary r in rank
 * order, quota_r of them in total, so every shard ends exactly at global rank T_r. */
typedef int (*bsort_refine_fn)(void* ctx, const uint64_t* prefixes, int m, int prefix_bits, uint64_t* hist);
bsort_status_t bsort_dist_exact_boundaries(const uint64_t* host_global_hist, int nranks, int key_bits,
                                           bsort_refine_fn refine, void* ctx, uint64_t* values, int* m,
                                           int* idx, uint64_t* quota, int* levels);
bsort_status_t bsort_dist_exact_send_counts(const uint64_t* class_counts_all, int nranks, int m, int rank,
                                            const int* idx, const uint64_t* quota, uint64_t* send_counts);

/* ----------------------------------------------------------------------- diagnostics */

const char* bsort_status_string(bsort_status_t status);
int bsort_last_cuda_error(void);          /* raw cudaError_t of the last failure (thread-local) */
const char* bsort_version(void);

/* Device self-checks of hardware behaviour the fast paths rely on, run on the CURRENT device
 * (the library also runs them implicitly once per device on first use).  Check 1: lanes of
 * one warp instruction that atomically add to the same shared-memory word receive the old
 * values in ascending lane order (the stable rankings of the round-2 look-back pass and of the
 * small-n kernel use that value as the key's rank; where it fails those kernels are not used).
 * Returns 0 when every check holds, else a bitmask of failed checks (bit 0 = check 1), or -1
 * when no device is usable.  Synchronous; allocates 8 bytes; do not call during graph capture. */
int bsort_selftest(void);

/* Total number of kernels this library has launched since it was loaded (all threads). */
uint64_t bsort_launch_count(void);

/* Optional per-kernel timing with CUDA events recorded on the launching stream around every
 * kernel this library launches.  bsort_profile_enable(1) clears and starts recording,
 * bsort_profile_enable(0) stops.  bsort_profile_read() synchronises the recorded events and
 * fills, per kernel kind (BSORT_PROF_KINDS entries), the summed milliseconds and launch count;
 * returns the number of kinds.  Kind names: bsort_profile_kind_name().  Kind 12 ("dist_a2a") is
 * not a kernel: it brackets bsort_sort_dist's grouped NCCL send/recv (the key exchange). */
#define BSORT_PROF_KINDS 13
void bsort_profile_enable(int on);
int bsort_profile_read(double* ms_per_kind, uint64_t* launches_per_kind);
const char* bsort_profile_kind_name(int kind);

#ifdef __cplusplus
}
#endif
#endif /* BSORT_H */
