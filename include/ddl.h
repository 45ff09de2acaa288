/*
 * ddl.h -- C ABI of libddl: PowerAI DDL's topology-aware gradient all-reduce, rebuilt
 * B200-native (hand-written sm_100a kernels reading peer GPUs' memory over NVLink 5 /
 * NVSwitch, device-side flag barriers).
 *
 * The operation (§2.1): synchronous-SGD all-reduce "decompose[d] ...
 * into a series of reduce-scatter and all-gather patterns in a topology-aware fashion".
 * The ranks are factorised as dims = {g_0, ..., g_{k-1}}, INNERMOST FIRST (prod = nranks;
 * "2x4" = 2 outer x 4 inner = {4, 2}); coordinates c_d(r) = floor(r / G_d) mod g_d with
 * G_d = prod_{j<d} g_j.  Reduce-scatter phases run d = 0..k-1, then
 * all-gather phases d = k-1..0.  A dim with g_d = 1 has no phase.
 *
 * Results (identical on every rank): y[e] = F_dims(x_0[e], ..., x_{P-1}[e]) where F folds
 * each dim's group in ascending coordinate, innermost dim first:
 *   int32    two's-complement wrapping sum (exact; equals the plain sum in any order)
 *   float32  every add IEEE round-to-nearest-even, no FMA, no flush-to-zero
 *   bfloat16 fp32 adds within a phase, RNE to bf16 at every phase boundary
 *   DDL_AVG  one multiply by fl32(1/P) of the fully reduced fp32 value, fused into the
 *            last reduce-scatter phase (before the output cast); int32 + AVG unsupported.
 * The result never depends on the algorithm chosen (hierarchical or one-shot) -- see
 * DESIGN.md "Readings" for every reading of the paper behind these rules.
 *
 * Block layout: count elements are split into P blocks of q elements,
 * q = roundup(ceil(count/P), 16 B / sizeof(elem)); block b = [min(n,bq), min(n,(b+1)q)).
 * After the reduce-scatter phases rank r holds block r.
 *
 * Conventions for every call below:
 *   - Buffers are device pointers unless stated; counts are in ELEMENTS.
 *   - Collective calls are asynchronous on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream).  Argument errors return synchronously and enqueue
 *     nothing.  Device-side errors (a peer that never arrives: DDL_ERR_TIMEOUT) are
 *     sticky and read with ddl_async_error().
 *   - Every rank calls the same sequence of collectives with equal (count, dtype, op)
 *     (DDL_CHECK=1 verifies it on the device: DDL_ERR_MISMATCH).  Calls on one
 *     communicator must be ordered (one stream, or externally serialised): the device
 *     barriers of consecutive calls are told apart by a per-rank call counter.
 *   - Calls are CUDA-graph capturable: all per-call state (the call counter, the flags)
 *     lives in device memory.  One exception: ddl_group_reduce_scatter grows its loopback
 *     workspace on demand, which cannot happen inside a capture -- a captured call that
 *     would need a larger workspace returns DDL_ERR_TOO_LARGE (make one uncaptured call
 *     of the largest size first).
 *   - Calls whose per-CTA slice would reach 1 GiB (only with DDL_CTAS forced tiny and
 *     multi-GiB messages) are cut into waves, or return DDL_ERR_TOO_LARGE.
 *   - The caller owns buffers, streams and the comm handle; the library owns its
 *     workspace, flags and IPC mappings and releases them in ddl_finalize().  No C++
 *     exception crosses the ABI and the library never aborts the process.
 *   - Device buffers must be 16-byte aligned (DDL_ERR_INVALID_ARGUMENT otherwise).
 */
#ifndef DDL_H
#define DDL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DDL_MAX_RANKS 16   /* ranks per communicator (and virtual ranks in loopback) */
#define DDL_MAX_DIMS 8

typedef struct ddl_comm* ddl_comm_t;

typedef enum {
  DDL_SUCCESS = 0,
  DDL_ERR_INVALID_ARGUMENT = 1, /* null/unaligned pointer, bad enum, bad handle bytes     */
  DDL_ERR_BAD_DIMS = 2,         /* prod(dims) != nranks, g_d < 1, ndims > 8 (SPEC BadArity) */
  DDL_ERR_UNSUPPORTED = 3,      /* int32 + AVG, nranks > DDL_MAX_RANKS                     */
  DDL_ERR_CUDA = 4,             /* a CUDA runtime call failed (no GPU, OOM, launch error)  */
  DDL_ERR_NO_PEER_ACCESS = 5,   /* a peer GPU is not reachable by P2P                       */
  DDL_ERR_NOT_CONNECTED = 6,    /* collective called before ddl_connect                     */
  DDL_ERR_TOO_LARGE = 7,        /* message exceeds the workspace on a staged path           */
  DDL_ERR_TIMEOUT = 8,          /* (async) a device barrier waited longer than the timeout  */
  DDL_ERR_MISMATCH = 9          /* ranks disagree: handles (nranks/dims/sizes) at connect, or (async, DDL_CHECK=1) the call signature */
} ddl_result_t;

typedef enum { DDL_INT32 = 0, DDL_FLOAT32 = 1, DDL_BFLOAT16 = 2 } ddl_dtype_t;
typedef enum { DDL_SUM = 0, DDL_AVG = 1 } ddl_op_t;

/* Implementation choice per call ("mix-and-match", P:L54 (3)).  AUTO picks, by message
 * size: LL (multi-process comms only, <= the LL threshold, default 64 KiB: inputs pushed to
 * every peer with the call counter in every 64-bit word, no barrier), ONESHOT (<= the
 * one-shot threshold: every rank reads all inputs), HIER otherwise.  All three compute the
 * same F_dims.  LL forced on a message that does not fit its receive slots (sized from the
 * LL threshold at init) or on a loopback comm falls through to the AUTO rules. */
typedef enum { DDL_ALGO_AUTO = 0, DDL_ALGO_HIER = 1, DDL_ALGO_ONESHOT = 2, DDL_ALGO_LL = 3 } ddl_algo_t;

/* ------------------------------------------------------------------ host-only helpers */
/* These never touch the GPU; they expose the planner the kernels use, for tests.       */

int ddl_version(void);                                   /* 100 * major + minor           */
/* Build options: bit 0 = the experiment kernels PATH 3 (DDL_DYN) and PATH 4 (DDL_STEAL)
 * are compiled in (DDL_EXPERIMENTAL=1 bash build.sh); without them ddl_init /
 * ddl_loopback_init return DDL_ERR_UNSUPPORTED when DDL_DYN or DDL_STEAL is set. */
int ddl_build_flags(void);
const char* ddl_result_string(ddl_result_t r);           /* static string, never NULL     */
const char* ddl_last_error_string(void);                 /* last CUDA failure text (this thread) */

/* Validate a factorisation. */
ddl_result_t ddl_check_dims(int nranks, const int* dims, int ndims);

/* q, the block size in elements, for an all-reduce of `count` elements (layout above). */
size_t ddl_block_elems(size_t count, int nranks, ddl_dtype_t dtype);

/* Group of `rank` in dim d: members_out[v] = rank + (v - c_d(rank)) * G_d, v < g_d. */
ddl_result_t ddl_plan_group(int nranks, const int* dims, int ndims, int rank, int d, int* members_out);

/* A_d(rank) = { b : c_j(b) = c_j(rank) for all j < d }, ascending, d in [0, ndims]:
 * the blocks `rank` reduces in RS phase d-1 / receives in AG phase d-1.
 * blocks_out needs room for nranks entries; *nblocks_out = nranks / G_d. */
ddl_result_t ddl_plan_blocks(int nranks, const int* dims, int ndims, int rank, int d,
                             int* blocks_out, int* nblocks_out);

/* The device barrier schedule of one hierarchical call (2L+1 barriers, L = number of dims
 * with g_d > 1): for barrier j, peers_out[j*nranks + i] (i < counts_out[j]) are the ranks
 * `rank` signals and waits for.  *nbarriers_out = 2L+1 (0 when nranks == 1). */
ddl_result_t ddl_plan_barriers(int nranks, const int* dims, int ndims, int rank,
                               int* peers_out, int* counts_out, int* nbarriers_out);

/* Bytes `rank` reads from peers in each phase of an all-reduce of `count` elements:
 * rs_out[d], ag_out[d] for d < ndims (0 for dims with g_d = 1).  SPEC S:L371. */
ddl_result_t ddl_plan_traffic(size_t count, ddl_dtype_t dtype, int nranks, const int* dims, int ndims,
                              int rank, uint64_t* rs_out, uint64_t* ag_out);

/* ------------------------------------------------------------------ multi-process comm */
/* One process per GPU (the paper's MPI-like `rank`, §2.1; dims as SPEC S:L264-270:
 * innermost first, prod(dims) == nranks, g_d >= 1).  Bootstrap: ddl_init -> ddl_export_handle -> (caller all-gathers
 * the handles, e.g. torch.distributed.all_gather_object) -> ddl_connect(all, rank order).
 * The handle bytes carry a cudaIpc memory handle of this rank's flag+workspace block. */

ddl_result_t ddl_init(ddl_comm_t* comm, int rank, int nranks, const int* dims, int ndims,
                      int cuda_device, size_t max_bytes);
size_t ddl_handle_size(void);
ddl_result_t ddl_export_handle(ddl_comm_t comm, void* out /* ddl_handle_size() bytes */);
ddl_result_t ddl_connect(ddl_comm_t comm, const void* all_handles /* nranks * handle_size */);

/* The symmetric zero-copy buffer (max_bytes, 256-B aligned).  An all-reduce on a buffer
 * inside it, at the SAME offset on every rank, reads peers' data in place (no staging). */
ddl_result_t ddl_buffer(ddl_comm_t comm, void** dev_ptr, size_t* bytes);
/* NVLS phases (P:L54 (3) "mix and match" per decomposed piece): an
 * NVSwitch multicast object per live dim's group, so that phase d runs IN the switch --
 * multimem.ld_reduce for the reduce-scatter (the switch sums the g_d members' copies),
 * multimem.st for the all-gather (one store reaches every member).  Per GPU that moves
 * ~S(1+1/P) bytes per direction instead of 2S(P-1)/P.  Setup is collective, in four
 * rounds; after each of the first three the caller all-gathers every rank's blob
 * (ddl_nvls_blob_size() bytes, rank order) and passes the result to the next call:
 *   ddl_nvls_prepare(comm, bytes, mine)      -> all-gather -> all
 *   ddl_nvls_attach(comm, all, mine)         -> all-gather -> all
 *   ddl_nvls_bind(comm, all, mine)           -> all-gather -> all
 *   ddl_nvls_commit(comm, all)               -> DDL_SUCCESS: NVLS on; DDL_ERR_UNSUPPORTED: off
 * A rank that cannot take part (no multicast support or fabric, one GPU per process not
 * given, a failed import / bind) reports it in its blob, and commit then turns NVLS off on
 * every rank (resources released; all calls keep the direct P2P phases) -- never a hang.
 * Requires ddl_connect first.  `bytes` is the NVLS buffer size per rank (rounded up to the
 * multicast granularity).  All-reduces of buffers inside ddl_nvls_buffer() (same offset on
 * every rank, count * size a multiple of 16 B) run the dims in *dims_mask in the switch
 * (DDL_NVLS_DIMS=bitmask of dims restricts them; default every live dim) and the rest as
 * direct phases over the peers' unicast mappings.  Numerics: the switch's fold order is not
 * specified, so fp32 / bf16 results of NVLS phases are gated by the Higham bound instead of
 * bit-exactness (int32: exact); reading 15. */
size_t ddl_nvls_blob_size(void);
ddl_result_t ddl_nvls_prepare(ddl_comm_t comm, size_t bytes, void* blob_out);
ddl_result_t ddl_nvls_attach(ddl_comm_t comm, const void* all_blobs, void* blob_out);
ddl_result_t ddl_nvls_bind(ddl_comm_t comm, const void* all_blobs, void* blob_out);
ddl_result_t ddl_nvls_commit(ddl_comm_t comm, const void* all_blobs);
ddl_result_t ddl_nvls_buffer(ddl_comm_t comm, void** dev_ptr, size_t* bytes, int* dims_mask);
/* Self-test of the NVLS setup's descriptor exchange (abstract Unix sockets + SCM_RIGHTS)
 * inside this process; no GPU.  0 = success. */
int ddl_debug_nvls_fd_selftest(void);

/* Rank `peer`'s symmetric buffer as mapped into this process (cudaIpc over NVLink; this
 * rank's own buffer for peer == rank).  For measurement and diagnostics (bench.py's
 * peer-copy peak); writing into it races with the peer's collectives unless the caller
 * orders them.  DDL_ERR_NOT_CONNECTED before ddl_connect. */
ddl_result_t ddl_peer_buffer(ddl_comm_t comm, int peer, void** dev_ptr, size_t* bytes);
/* Enqueue one copy of `bytes` from this rank's symmetric buffer (+src_offset) into rank
 * `peer`'s (+dst_offset) over the cudaIpc mapping (cudaMemcpyAsync: the copy engines) --
 * the peer-copy reference bench.py measures beside the NVLink roofline.  Same caveat as
 * ddl_peer_buffer: the caller orders it against the peer's collectives. */
ddl_result_t ddl_peer_copy(ddl_comm_t comm, int peer, size_t src_offset, size_t dst_offset, size_t bytes,
                           void* stream);

/* Registered buffers (SURVEY 8(b) ddl_register): persistent user buffers -- e.g. DDP's
 * gradient buckets -- made zero-copy.  Collective: every rank calls
 * ddl_register_export(ptr, bytes) on ITS buffer (equal bytes on every rank), the caller
 * all-gathers the ddl_reg_handle_size() blobs in rank order, and every rank calls
 * ddl_register_connect(ptr, blobs) -> reg_id.  Afterwards an all-reduce on any sub-range
 * of the buffer, at the SAME offset on every rank, reads peers in place.  The buffer must
 * come from cudaMalloc (or torch's default caching allocator) and outlive the
 * registration; ddl_deregister (or ddl_finalize) unmaps it.  At most 64 registrations. */
size_t ddl_reg_handle_size(void);
ddl_result_t ddl_register_export(ddl_comm_t comm, void* ptr, size_t bytes, void* handle_out);
ddl_result_t ddl_register_connect(ddl_comm_t comm, void* ptr, const void* all_handles, int* reg_id);
ddl_result_t ddl_deregister(ddl_comm_t comm, int reg_id);

/* In-place all-reduce of buf[0, count) -- "one all-reduce operation decomposed into a series
 * of reduce-scatter and all-gather patterns in a topology-aware fashion" (§2.1):
 * RS phases innermost dim first, AG phases outermost first; avg multiplies
 * the fully reduced fp32 value by fl32(1/P) once (DESIGN reading 5).  buf inside ddl_buffer() or a registered buffer:
 * zero-copy; any other device buffer: staged through the workspace (count * size <=
 * max_bytes). */
ddl_result_t ddl_allreduce(ddl_comm_t comm, void* buf, size_t count, ddl_dtype_t dtype,
                           ddl_op_t op, void* stream);

/* Grouped all-reduce: nbufs independent in-place all-reduces (e.g. the gradient buckets of
 * one SGD step) in as few launches as possible.  bufs[i] holds counts[i]
 * elements (16-B aligned, not overlapping one another; counts[i] == 0 is skipped); every
 * rank passes the same nbufs and counts in the same order.  Buffers in the LL / one-shot size regime, staged (not
 * symmetric / registered) buffers, and every buffer under DDL_CHECK or a non-default
 * phase kernel (DDL_NO_TMA register-staged fallback, DDL_STEAL / DDL_DYN / DDL_STREAM
 * experiments) are all-reduced first by single ddl_allreduce calls, in order; the remaining zero-copy buffers share one launch
 * per 8 buffers, split over DDL_CHANNELS (default 2) channels of CTAs that each run their
 * buffers' hierarchical schedules one after another, so that one channel's barrier waits
 * and L2-bound phases overlap another's HBM / NVLink-bound phases.  Results are
 * bit-identical to nbufs single ddl_allreduce calls (same fold order per element).  Same
 * errors as ddl_allreduce; asynchronous on stream. */
ddl_result_t ddl_allreduce_many(ddl_comm_t comm, void* const* bufs, const size_t* counts, int nbufs,
                                ddl_dtype_t dtype, ddl_op_t op, void* stream);

/* The reduce-scatter half of the decomposition alone.
 * NCCL layout: sendbuf holds nranks * recvcount elements; rank r receives elements
 * [r*recvcount, (r+1)*recvcount) of the reduced vector.  sendbuf is not modified.
 * The partial sums live in the workspace: nranks * recvcount * size <= max_bytes.  A
 * sendbuf in the symmetric / a registered buffer is read in place (no copy-in). */
ddl_result_t ddl_reduce_scatter(ddl_comm_t comm, const void* sendbuf, void* recvbuf, size_t recvcount,
                                ddl_dtype_t dtype, ddl_op_t op, void* stream);

/* The all-gather half of the decomposition alone.
 * Rank r's sendcount elements land at [r*sendcount, (r+1)*sendcount) of every rank's
 * recvbuf (nranks * sendcount elements).  A recvbuf in the symmetric / a registered buffer
 * is gathered into in place; otherwise staged through the workspace (<= max_bytes). */
ddl_result_t ddl_allgather(ddl_comm_t comm, const void* sendbuf, void* recvbuf, size_t sendcount,
                           ddl_dtype_t dtype, void* stream);

/* Sticky device-side error of this comm (synchronises the device to read it). */
ddl_result_t ddl_async_error(ddl_comm_t comm);

/* Algorithm override: algo, and the one-shot threshold in bytes (AUTO only). */
ddl_result_t ddl_set_algo(ddl_comm_t comm, ddl_algo_t algo, size_t oneshot_max_bytes);

/* LL threshold in bytes for AUTO (default 65536, env DDL_LL_MAX_BYTES; 0 = never LL).  The
 * receive slots are sized at ddl_init from the threshold then in force (2 * nranks * 2 *
 * threshold bytes per rank), so raising it later only helps up to that size.  Every rank
 * must set the same value (the algorithm is chosen locally from it). */
ddl_result_t ddl_set_ll_max(ddl_comm_t comm, size_t ll_max_bytes);

/* Barrier-spin timeout in milliseconds (default 10000; env DDL_TIMEOUT_MS). */
ddl_result_t ddl_set_timeout(ddl_comm_t comm, uint64_t timeout_ms);

/* Algorithm AUTO would use for this message (for tests / bench labelling). */
ddl_algo_t ddl_algo_for(ddl_comm_t comm, size_t count, ddl_dtype_t dtype);

/* Number of CTAs per rank a call of this size launches. */
int ddl_ctas_for(ddl_comm_t comm, size_t count, ddl_dtype_t dtype);

/* Test hook: virtual/process rank `rank` skips its part of every following call (-1 = off),
 * so its peers' barriers time out (DDL_ERR_TIMEOUT via ddl_async_error).  Never use in
 * production: the skipped rank's data is not reduced. */
ddl_result_t ddl_debug_skip_rank(ddl_comm_t comm, int rank);

/* Debug: with DDL_TRACE=1 set at init, every CTA stamps %globaltimer (ns) at each phase
 * boundary of each call (overwriting the previous call's stamps).  Copies the
 * [nranks][cmax][40] uint64 timeline of the last call to host_out (synchronises).
 * cmax = 4 * SM count.  DDL_ERR_UNSUPPORTED when tracing is off. */
ddl_result_t ddl_debug_trace(ddl_comm_t comm, void* host_out, size_t bytes);

/* Test hook: connect nranks communicators that all live in THIS process on ONE GPU
 * (comms[r] = rank r's handle from ddl_init, same dims/max_bytes), without cudaIpc: peers'
 * workspaces are addressed directly.  Each rank's calls then run the multi-process kernel
 * path (per-rank launches on the caller's streams, .sys-scope flags, zero-copy and staged
 * buffers) with the ranks' kernels co-resident on one GPU (CTA budget divided by nranks). */
ddl_result_t ddl_debug_connect_local(ddl_comm_t* comms, int nranks);

/* Test hook: register ptrs[r] (bytes each) for the in-process communicators comms[r]
 * (see ddl_debug_connect_local) without cudaIpc; same reg_id on every rank. */
ddl_result_t ddl_debug_register_local(ddl_comm_t* comms, void* const* ptrs, size_t bytes, int nranks, int* reg_id);

/* Collective teardown: every rank must have finished all calls (host barrier first).
 * Unmaps peers, frees the workspace, destroys the handle.  NULL is a no-op. */
ddl_result_t ddl_finalize(ddl_comm_t comm);

/* ------------------------------------------------------------------ loopback (1 GPU) */
/* P virtual ranks in ONE GPU's memory (used by the parity tests and the 1-GPU benchmark).
 * All-reduces (ddl_group_allreduce, ddl_group_allreduce_many) run the column-chain kernels
 * (csrc/ddl_chain.cuh): the schedule's RS / AG phases per column
 * of every block in one thread, every load and store of the schedule, bit-identical results;
 * no barrier is needed because a column's phases run in program order in that thread.  With
 * DDL_LB_CHAIN=0 (or the debug hooks ddl_debug_skip_rank / DDL_TRACE) they run the
 * multi-process path's slice kernels instead -- same block layout and barrier protocol, all
 * P ranks in one cooperative launch (deadlock-free), "peer" pointers local -- as do the
 * loopback reduce-scatter / allgather. */

ddl_result_t ddl_loopback_init(ddl_comm_t* comm, int nranks, const int* dims, int ndims, int cuda_device);
/* The same under SURVEY 8(b)'s name and argument list (max_bytes is unused: loopback calls
 * work on the caller's buffers in place; reduce-scatter grows its workspace on demand). */
ddl_result_t ddl_init_loopback(ddl_comm_t* comm, int nranks, const int* dims, int ndims, int cuda_device,
                               size_t max_bytes);

/* bufs: host array of nranks device pointers (distinct, 16-B aligned, count elements
 * each); in place. */
ddl_result_t ddl_group_allreduce(ddl_comm_t comm, void* const* bufs, size_t count, ddl_dtype_t dtype,
                                 ddl_op_t op, void* stream);
/* Grouped all-reduce in loopback: bufs[i * nranks + r] is virtual rank r's copy of buffer i
 * (counts[i] elements); otherwise as ddl_allreduce_many (one launch per 8 buffers; with the
 * slice kernels, one-shot-sized buffers go through single ddl_group_allreduce calls first).
 * DDL_ERR_TOO_LARGE (nothing enqueued) if a buffer exceeds 2^31 16-byte columns. */
ddl_result_t ddl_group_allreduce_many(ddl_comm_t comm, void* const* bufs, const size_t* counts, int nbufs,
                                      ddl_dtype_t dtype, ddl_op_t op, void* stream);
/* sendbufs[r]: nranks*recvcount elements (not modified); recvbufs[r]: recvcount.
 * Uses a library workspace of nranks * nranks * recvcount elements (grown on demand;
 * DDL_ERR_TOO_LARGE if it must grow while the stream is being captured). */
ddl_result_t ddl_group_reduce_scatter(ddl_comm_t comm, const void* const* sendbufs, void* const* recvbufs,
                                      size_t recvcount, ddl_dtype_t dtype, ddl_op_t op, void* stream);
/* sendbufs[r]: sendcount elements; recvbufs[r]: nranks*sendcount elements. */
ddl_result_t ddl_group_allgather(ddl_comm_t comm, const void* const* sendbufs, void* const* recvbufs,
                                 size_t sendcount, ddl_dtype_t dtype, void* stream);

/* ------------------------------------------------------------------ local reduce (K5) */
/* out[e] = scale * sum_{j<g} ins[j][e], folded in ascending j in fp32 (int32: wrapping,
 * scale must be 1), one multiply by fl32(scale) (skipped when scale == 1), then the output
 * cast (bf16: RNE).  ins: host array of g device pointers (g in [1, 64]); out may alias
 * ins[0].  The 1-GPU HBM-roofline kernel of SURVEY.md 8(a) a8. */
ddl_result_t ddl_local_reduce(const void* const* ins, int g, void* out, size_t count, ddl_dtype_t dtype,
                              float scale, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DDL_H */
