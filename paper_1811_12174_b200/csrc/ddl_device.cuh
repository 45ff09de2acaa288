// ddl_device.cuh -- sm_100a kernels of libddl.
//
//   ddl_hier_kernel    one launch = one whole hierarchical collective: copy-in (staged),
//                      RS phases d = live[0..L-1] (K1) with the fused 1/P + cast epilogue
//                      in the last one (K3), AG phases d = live[L-1..0] (K2), copy-out,
//                      separated by 2L+1 per-CTA device barriers (K4).
//   ddl_oneshot_kernel small messages: every rank reads all P inputs, folds them in the
//                      nested order of the dims (same F_dims as the hierarchy), 2 barriers.
//   ddl_ll_kernel      smallest messages across processes: inputs pushed with the epoch in
//                      every 64-bit word (LL protocol), no barrier, same nested fold.
//   ddl_local_reduce_kernel  K5: out = s * sum_j in_j over local buffers (HBM roofline).
//
// Work split (a4 "per-CTA slices"): a block of q elements is cut into nctas slices; CTA c
// handles slice c of every block in every phase, so CTA c only ever depends on CTA c of its
// peers and the barriers are per CTA (no grid-wide sync).  In loopback mode the P virtual
// ranks are gridDim.y and all P * nctas CTAs are co-resident (cooperative launch).
//
// Memory ordering (cross-GPU): all threads' stores -> __syncthreads -> one lane per peer
// st.release.sys of the epoch into the peer's flag slot; waiters spin with ld.acquire.sys on
// their local slot, then __syncthreads.  Data loads that may target memory another agent
// wrote during this launch use ld.global.cg (L2 / remote, never a stale L1 line).
// Numerics: __fadd_rn / __fmul_rn (never contracted into FMA), RNE bf16 cast, int32 adds in
// uint32 (wrap); the fold order is ascending group coordinate.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "ddl_plan.h"

namespace ddl {

#ifndef DDL_MUTATE
#define DDL_MUTATE 0  // 1-3: deliberately wrong kernels for scripts/gpu_mutation_check.sh (never in a product build)
#endif
constexpr int kThreads = 512;
constexpr int kMaxLocalIn = 64;

enum Mode : int {
  kCinAll = 1,    // copy cin[me] -> work[me] (all blocks, this CTA's slices) before the start
  kCinOwn = 2,    // copy cin[me] (one block of q elems) -> work[me] block me
  kRS = 4,
  kAG = 8,
  kCoutAll = 16,  // copy work[me] -> cout[me] (all blocks) after the AG phases
  kScratch = 32,  // one-shot, multi-process: inputs published through double-buffered scratch
};

enum DType : int { kI32 = 0, kF32 = 1, kBF16 = 2 };
enum Op : int { kSum = 0, kAvg = 1 };
enum Err : int { kErrTimeout = 8, kErrMismatch = 9 };

struct KParams {
  Topo t;
  int rank;            // this process's rank (multi-process); loopback: me = blockIdx.y
  int loopback;
  int gpu_scope;       // every rank on this GPU (loopback, in-process groups): .gpu-scope flags suffice
  int op;
  int cmax;            // CTA stride of the flag slots
  float scale;         // fl32(1/P) for avg
  int skip_rank;       // test hook: this rank's CTAs return at once (-1: none)
  uint64_t n;          // elements of the full vector
  uint64_t q;          // block elements
  uint64_t slice;      // elements per CTA slice (hier: of a block; one-shot: of the vector)
  uint64_t timeout_ns;
  int* err;            // sticky device error word (local)
  uint32_t* flags[kMaxRanks];   // each rank's flag region (peer-mapped); [cmax epochs][slots][cmax][P]
  const void* in[kMaxRanks];    // where RS phase live[0] (and the one-shot) reads each rank's input
  void* work[kMaxRanks];        // each rank's working buffer (partials, gathered blocks)
  void* out[kMaxRanks];         // last RS phase / one-shot destination of each rank (block offsets apply)
  const void* cin[kMaxRanks];   // copy-in source of each rank
  void* cout[kMaxRanks];        // copy-out destination of each rank
  int mode;
  int transposed;      // loopback hierarchical / grouped kernels: grid (P, ctas) -- blockIdx.x is the
                       // rank, .y the CTA, so a slice chain's P CTAs are dispatched back to back
  int l2hint;          // L2 eviction priorities (default 47 = bits 0-3 + 5): bit 0: the first RS phase's inputs
                       // loaded evict_first (each is read once); bit 1: allgather stores
                       // evict_first (final, never re-read in the call); bit 2: later RS phases'
                       // loads evict_first (partials, consumed); bit 3: non-last RS phases' stores
                       // evict_last (partials the next phase reads); bit 4: also the last RS
                       // phase's stores (off: they would linger as evict_last after the call);
                       // bit 5: bit 1 only for the last AG phase (earlier AG phases' stores are
                       // the next AG phase's sources); bit 6: those earlier stores evict_last
  int nwaves;          // hier: slices per CTA, run one after another (wave w = slice w*gridDim.x + blockIdx.x)
  uint64_t* trace;     // debug (DDL_TRACE=1): [P][cmax][kTraceEvents] globaltimer stamps, else null
  int stream_every;    // PATH 5: publish progress every k chunks (and at the phase end)
  uint32_t sig;        // DDL_CHECK=1: signature of (count, dtype, op, algorithm); 0 = no check
  char* scratch[kMaxRanks];  // kScratch: each rank's one-shot scratch (two halves, by call parity)
  uint64_t scratch_half;     // bytes per half
  char* ll[kMaxRanks];       // LL one-shot: each rank's receive region (two halves of P slots)
  uint64_t ll_slot;          // bytes per source slot (half = P slots)
  // NVLS phases (PATH 7): mc[d] = this rank's dim-d group multicast
  // mapping at the buffer's offset; dims whose bit is set in nvls_mask reduce with
  // multimem.ld_reduce (RS) and broadcast with multimem.st (AG), the others run the
  // register-staged direct phases over the peers' unicast mappings
  char* mc[kMaxDims];
  int nvls_mask;
  int deep_copy;     // copy phases (AG, copy-in/out) through the kCopySub-deep sub-stage pipeline
  int nvls_emulate;  // test hook (DDL_NVLS_EMULATE=1): the NVLS phases' data flow done with unicast
                     // loads / stores (RS folds the members in DESCENDING coordinate -- an order
                     // other than the direct path's; AG stores each own vector into every member)
};
constexpr int kTraceEvents = 128;

// This CTA's index within its rank and the rank's CTA count (the grid is (ctas, P) in
// loopback, or transposed to (P, ctas) for the grouped kernel with DDL_TRANSPOSE=1).
__device__ __forceinline__ int cta_id(const KParams& p) { return p.transposed ? (int)blockIdx.y : (int)blockIdx.x; }
__device__ __forceinline__ int cta_count(const KParams& p) { return p.transposed ? (int)gridDim.y : (int)gridDim.x; }

// Debug timeline: thread 0 of each CTA stamps the global timer at event ev.
__device__ __forceinline__ void trace_ev(const KParams& p, int me, int ev) {
  if (p.trace && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[((size_t)me * p.cmax + cta_id(p)) * kTraceEvents + ev] = t;
    if (ev == 0) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      p.trace[((size_t)me * p.cmax + cta_id(p)) * kTraceEvents + kTraceEvents - 1] = smid;
    }
  }
}

struct LRParams {
  const void* in[kMaxLocalIn];
  void* out;
  uint64_t n;
  int g;
  float scale;
};

// Programmatic dependent launch: every kernel is launched with programmatic stream
// serialisation allowed, so its CTAs may be scheduled while the previous kernel on the
// stream drains.  griddepcontrol.wait blocks until that kernel has completed and its memory
// is visible -- before any global access here -- and launch_dependents lets the next
// kernel's CTAs be scheduled as soon as SMs free up (they wait the same way).
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------------------------ element traits
template <typename T> struct Tr;
template <> struct Tr<int32_t> {  // int32: wrapping adds in uint32
  using Acc = uint32_t;
  static constexpr int W = 4;
  __device__ static Acc to(uint32_t bits) { return bits; }
  __device__ static uint32_t from(Acc a) { return a; }
  __device__ static Acc add(Acc a, Acc b) { return a + b; }
  __device__ static Acc mul(Acc a, float) { return a; }
  __device__ static Acc round(Acc a) { return a; }
};
template <> struct Tr<float> {
  using Acc = float;
  static constexpr int W = 4;
  __device__ static Acc to(uint32_t bits) { return __uint_as_float(bits); }
  __device__ static uint32_t from(Acc a) { return __float_as_uint(a); }
  __device__ static Acc add(Acc a, Acc b) { return __fadd_rn(a, b); }
  __device__ static Acc mul(Acc a, float s) { return __fmul_rn(a, s); }
  __device__ static Acc round(Acc a) { return a; }
};
template <> struct Tr<__nv_bfloat16> {  // bf16 bits in memory, fp32 accumulation
  using Acc = float;
  static constexpr int W = 8;
  __device__ static Acc to(uint32_t bits16) { return __uint_as_float(bits16 << 16); }
  __device__ static uint32_t from(Acc a) {
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a));
  }
  __device__ static Acc add(Acc a, Acc b) { return __fadd_rn(a, b); }
  __device__ static Acc mul(Acc a, float s) { return __fmul_rn(a, s); }
  __device__ static Acc round(Acc a) { return to(from(a)); }  // bf16 phase-boundary rounding
};

// Unpack / pack one 16-byte vector (W elements).
template <typename T>
__device__ __forceinline__ void unpack(const uint4& r, typename Tr<T>::Acc* a) {
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
  if constexpr (Tr<T>::W == 8) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[2 * i] = Tr<T>::to(w[i] & 0xFFFFu);
      a[2 * i + 1] = Tr<T>::to(w[i] >> 16);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = Tr<T>::to(w[i]);
  }
}
template <typename T>
__device__ __forceinline__ uint4 pack(const typename Tr<T>::Acc* a) {
  uint32_t w[4];
  if constexpr (Tr<T>::W == 8) {
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = Tr<T>::from(a[2 * i]) | (Tr<T>::from(a[2 * i + 1]) << 16);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = Tr<T>::from(a[i]);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <typename T>
__device__ __forceinline__ uint32_t ld_elem(const char* p) {
  if constexpr (sizeof(T) == 2) return (uint32_t)__ldcg(reinterpret_cast<const unsigned short*>(p));
  else return __ldcg(reinterpret_cast<const unsigned int*>(p));
}
template <typename T>
__device__ __forceinline__ void st_elem(char* p, uint32_t v) {
  if constexpr (sizeof(T) == 2) *reinterpret_cast<unsigned short*>(p) = (unsigned short)v;
  else *reinterpret_cast<unsigned int*>(p) = v;
}
__device__ __forceinline__ uint4 ld_vec(const char* p) { return __ldcg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ void st_vec(char* p, const uint4& v) { *reinterpret_cast<uint4*>(p) = v; }
__device__ __forceinline__ void st_vec_hint(char* p, const uint4& v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(pol)
               : "memory");
}

// ------------------------------------------------------------------------ device barrier (K4)
// Flag signal / poll.  Across GPUs the scope must be .sys; in loopback mode every agent is
// on this GPU and .gpu scope suffices (a cheaper MEMBAR).
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v, bool gpu_scope) {
  if (gpu_scope) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p, bool gpu_scope) {
  uint32_t v;
  if (gpu_scope) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t* flag_slot(const KParams& p, uint32_t* base, int slot, int cta, int src) {
  return base + p.cmax + ((size_t)slot * p.cmax + cta) * p.t.P + src;
}

// Barrier `slot` of CTA blockIdx.x of rank `me` with `np` peers given by peer(l).
// Returns false (after recording DDL_ERR_TIMEOUT) if a peer did not arrive in time.
// DDL_CHECK: each rank's call signature, written into the peer's slot before the first
// barrier's release (so the acquire of the epoch makes it visible).
__device__ __forceinline__ uint32_t* sig_slot(const KParams& p, uint32_t* base, int cta, int src);

template <typename PeerFn>
__device__ __forceinline__ bool dbarrier(const KParams& p, int me, int slot, int np, uint32_t epoch, PeerFn peer,
                                         bool check_sig = false) {
  __syncthreads();  // every thread's stores of the previous phase precede the release below
  int fail = 0;
  if (threadIdx.x < np) {
    const int m = peer(threadIdx.x);
    const bool chk = check_sig && p.sig;
    if (chk) *(volatile uint32_t*)sig_slot(p, p.flags[m], cta_id(p), me) = p.sig;
    st_release(flag_slot(p, p.flags[m], slot, cta_id(p), me), epoch, p.gpu_scope);
    const uint32_t* f = flag_slot(p, p.flags[me], slot, cta_id(p), m);
    uint64_t t0 = 0;
    uint32_t spins = 0;
    while ((int32_t)(ld_acquire(f, p.gpu_scope) - epoch) < 0) {
      if ((++spins & 1023u) == 0) {
        const uint64_t now = globaltimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > p.timeout_ns) {
          atomicCAS(p.err, 0, kErrTimeout);
          fail = 1;
          break;
        }
      }
    }
    if (!fail && chk && *(volatile uint32_t*)sig_slot(p, p.flags[me], cta_id(p), m) != p.sig) {
      atomicCAS(p.err, 0, kErrMismatch);  // ranks disagree on (count, dtype, op, algorithm)
      fail = 1;
    }
  }
  return __syncthreads_or(fail) == 0;
}

constexpr int kNumSlots = 2 * kMaxDims + 1;
constexpr int kPrePhase = kNumSlots;      // copy-in / nothing, before barrier 0
constexpr int kPostPhase = kNumSlots + 1; // copy-out, after the end barrier
constexpr int kRankStateWords = 16 + 2 * (kNumSlots + 2) + kNumSlots * kMaxRanks;

__device__ __forceinline__ uint32_t* rank_state(const KParams& p, int r) {
  return p.flags[r] + p.cmax + (size_t)kNumSlots * p.cmax * p.t.P;
}
__device__ __forceinline__ uint32_t* rs_arrive(uint32_t* rs, int j) { return rs + 16 + j; }
__device__ __forceinline__ uint32_t* rs_work(uint32_t* rs, int j) { return rs + 16 + (kNumSlots + 2) + j; }
__device__ __forceinline__ uint32_t* rs_flag(uint32_t* rs, int slot, int src) {
  return rs + 16 + 2 * (kNumSlots + 2) + slot * kMaxRanks + src;
}

__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t* a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(a), "r"(v) : "memory");
  return old;
}

// Call epochs are per RANK (identical on every rank: all ranks make the same calls), so flags
// written by any CTA of a rank compare against the same number whatever the CTA count of
// each call.  Every CTA reads it at start; the last CTA to finish the call (end arrival)
// advances it -- by then every CTA of the rank has read it.  The steal counters (PATH 4) are
// reset there too.  Layout after the rank state:
//   steal[0] end arrival, steal[16 + j*cmax + s] tickets, steal[16 + (kNumSlots + j)*cmax + s] done.
__device__ __forceinline__ uint32_t* steal_base(const KParams& p, int r) { return rank_state(p, r) + kRankStateWords; }
__device__ __forceinline__ uint32_t* steal_tick(const KParams& p, int r, int j) {
  return steal_base(p, r) + 16 + (size_t)j * p.cmax;
}
__device__ __forceinline__ uint32_t* steal_done(const KParams& p, int r, int j) {
  return steal_base(p, r) + 16 + (size_t)(kNumSlots + j) * p.cmax;
}

// after the steal counters: the PATH 5 progress words (kNumSlots x cmax u64), then the
// DDL_CHECK signatures [cmax][kMaxRanks]
__device__ __forceinline__ uint32_t* sig_slot(const KParams& p, uint32_t* base, int cta, int src) {
  uint32_t* end = base + p.cmax + (size_t)kNumSlots * p.cmax * p.t.P + kRankStateWords + 16 +
                  2 * (size_t)kNumSlots * p.cmax;
  uint64_t* prog = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(end) + 7) & ~(uintptr_t)7);
  uint32_t* sig = reinterpret_cast<uint32_t*>(prog + (size_t)kNumSlots * p.cmax);
  return sig + (size_t)cta * kMaxRanks + src;
}

__device__ __forceinline__ uint32_t rank_epoch_begin(const KParams& p, int me) {
  __shared__ uint32_t s_epoch;
  if (threadIdx.x == 0) s_epoch = *rank_state(p, me) + 1;
  __syncthreads();
  return s_epoch;
}

__device__ __forceinline__ void rank_epoch_end(const KParams& p, int me, uint32_t e, int steal_phases) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t* sb = steal_base(p, me);
    const uint32_t old = atom_add_acq_rel_gpu(sb, 1);
    s_last = (old == (uint32_t)cta_count(p) - 1);
    if (s_last) *sb = 0;
  }
  __syncthreads();
  if (s_last) {
    for (int j = 0; j < steal_phases; ++j)
      for (uint32_t i = threadIdx.x; i < (uint32_t)cta_count(p); i += blockDim.x) {
        steal_tick(p, me, j)[i] = 0;
        steal_done(p, me, j)[i] = 0;
      }
    if (threadIdx.x == 0) *rank_state(p, me) = e;
  }
}

// ------------------------------------------------------------------------ block/slice helpers
// CTA c handles, for every block b of a phase's block set, the elements
// [b*q + c*slice, b*q + min((c+1)*slice, q)) clipped to n.  The part that is a whole number
// of W-wide vectors goes through the 16-byte path; a ragged remainder (only where the
// slice is cut by n) goes element by element.
struct Span {
  uint64_t e0;    // first element of this CTA's slice of the block
  uint32_t nvec;  // full W-wide vectors
  uint32_t rem;   // trailing elements after them (< W)
};

template <int W>
__device__ __forceinline__ Span slice_span(const KParams& p, int b, int sidx) {
  Span s{0, 0, 0};
  const uint64_t cbase = (uint64_t)sidx * p.slice;
  if (cbase >= p.q) return s;
  const uint64_t e0 = (uint64_t)b * p.q + cbase;
  if (e0 >= p.n) return s;
  uint64_t len = p.q - cbase < p.slice ? p.q - cbase : p.slice;
  if (len > p.n - e0) len = p.n - e0;
  s.e0 = e0;
  s.nvec = (uint32_t)(len / W);
  s.rem = (uint32_t)(len - (uint64_t)s.nvec * W);
  return s;
}

// ------------------------------------------------------------------------ phase units
// A phase is a list of "units": this CTA's slice of one block, read from g sources (RS: the
// group-d members, ascending coordinate) or one source (AG: the peer that owns the block;
// copy-in/out: the user buffer / the work buffer), written to one destination at the same
// element offsets.  Both data paths below (register-staged and TMA-staged) walk the same
// unit list, kept in a small shared-memory table per phase.
enum PhaseKind : int { kPhRS = 0, kPhAG = 1, kPhCin = 2, kPhCinOwn = 3, kPhCout = 4 };

struct PhaseCtx {
  int kind, d, g, nunits, nb, c;
  int s;  // slice index this CTA handles in this phase (blockIdx.x, or w*gridDim.x + blockIdx.x)
  bool first, last;
};

__device__ __forceinline__ PhaseCtx phase_ctx(const KParams& p, int me, int kind, int d, bool first, bool last) {
  const Topo& t = p.t;
  PhaseCtx x;
  x.kind = kind;
  x.d = d;
  x.first = first;
  x.last = last;
  x.c = 0;
  x.nb = 0;
  x.g = 1;
  x.s = cta_id(p);
  if (kind == kPhRS) {
    x.g = t.g[d];
    x.nb = nblocks(t, d + 1);
    x.nunits = x.nb;
  } else if (kind == kPhAG) {
    x.c = coord(t, me, d);
    x.nb = nblocks(t, d + 1);
    x.nunits = (t.g[d] - 1) * x.nb;
  } else if (kind == kPhCinOwn) {
    x.nunits = 1;
  } else {
    x.nunits = t.P;
  }
  return x;
}

// Block of unit u; for AG also the source rank.
__device__ __forceinline__ int unit_block(const KParams& p, int me, const PhaseCtx& x, int u, int* srank) {
  const Topo& t = p.t;
  *srank = me;
  switch (x.kind) {
    case kPhRS: return block_of(t, me, x.d + 1, u);
    case kPhAG: {
      const int l = u / x.nb;
      const int bi = u - l * x.nb;
      const int m = member(t, me, x.d, l < x.c ? l : l + 1);
      *srank = m;
      return block_of(t, m, x.d + 1, bi);
    }
    case kPhCinOwn: return me;
    default: return u;
  }
}

// Base of source v of a unit (element offsets apply on top).
template <typename T>
__device__ __forceinline__ const char* src_base(const KParams& p, int me, const PhaseCtx& x, int v, int srank) {
  switch (x.kind) {
    case kPhRS: {
      const int m = member(p.t, me, x.d, v);
      return static_cast<const char*>(x.first ? p.in[m] : p.work[m]);
    }
    case kPhAG: return static_cast<const char*>(p.work[srank]);
    case kPhCin: return static_cast<const char*>(p.cin[me]);
    case kPhCinOwn: return static_cast<const char*>(p.cin[me]) - (size_t)me * p.q * sizeof(T);
    default: return static_cast<const char*>(p.work[me]);
  }
}
__device__ __forceinline__ char* dst_base(const KParams& p, int me, const PhaseCtx& x) {
  switch (x.kind) {
    case kPhRS: return static_cast<char*>(x.last ? p.out[me] : p.work[me]);
    case kPhCout: return static_cast<char*>(p.cout[me]);
    default: return static_cast<char*>(p.work[me]);
  }
}

struct UnitDesc {
  uint64_t e0;      // first element of this CTA's slice of the unit's block
  uint32_t bytes;   // whole W-element items, in bytes
  uint32_t rem;     // ragged elements after them
  const char* src;  // copies (AG / copy-in / copy-out): the unit's source buffer base
};

// ------------------------------------------------------------------------ register-staged phases
// Every thread walks the flattened (unit, vector) item list of the phase with U items in
// flight: all loads of its U items (g each for RS) are issued before any fold/store, so a
// phase of many small units costs one memory round trip, not one per unit.  PATH 0 runs the
// same code element-wise (unaligned reduce-scatter / allgather layouts).
template <typename T, bool VEC, int G>
__device__ __forceinline__ void ldg_phase_g(const KParams& p, const PhaseCtx& x, char* dst, const UnitDesc* units,
                                            const uint32_t* pref, const char* const* srcs) {
  using A = typename Tr<T>::Acc;
  constexpr int W = VEC ? Tr<T>::W : 1;
  constexpr int GC = G > 0 ? G : 8;                                  // loads per item per round
  constexpr int GG = G > 0 ? G : 1;
  constexpr int U = G == 1 ? 8 : (G > 0 && 4 / GG > 0 ? 4 / GG : 1);  // items per thread per iteration
  const bool rs = G != 1;
  const int g = rs ? x.g : 1;
  const bool do_scale = rs && x.last && p.op == kAvg;
  const char* sreg[GC];
  if constexpr (G > 1) {
#pragma unroll
    for (int v = 0; v < G; ++v) sreg[v] = srcs[v];
  }
  const uint32_t total = pref[x.nunits];
  int k = 0;  // unit cursor (items only increase along a thread's walk)
  for (uint32_t base = threadIdx.x; base < total; base += U * blockDim.x) {
    size_t off[U];  // byte offset of the item (same in sources and destination)
    const char* us[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t it = base + u * blockDim.x;
      off[u] = ~(size_t)0;
      if (it < total) {
        while (it >= pref[k + 1]) ++k;
        off[u] = (units[k].e0 + (size_t)(it - pref[k]) * W) * sizeof(T);
        us[u] = units[k].src;
      }
    }
    A acc[U][W];
    for (int v0 = 0; v0 < g; v0 += GC) {
      if constexpr (G == 0) {
#pragma unroll
        for (int v = 0; v < GC; ++v) sreg[v] = v0 + v < g ? srcs[v0 + v] : nullptr;
      }
      uint4 raw[U][GC];
      uint32_t raw1[U][GC];
#pragma unroll
      for (int v = 0; v < GC; ++v) {
        if (v0 + v >= g) break;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (off[u] == ~(size_t)0) continue;
          const char* ps = (G == 1 ? us[u] : sreg[v]) + off[u];
          if constexpr (VEC) raw[u][v] = ld_vec(ps);
          else raw1[u][v] = ld_elem<T>(ps);
        }
      }
      if constexpr (G == 1) {  // copy: store the raw bits
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (off[u] == ~(size_t)0) continue;
          if constexpr (VEC) st_vec(dst + off[u], raw[u][0]);
          else st_elem<T>(dst + off[u], raw1[u][0]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int v = 0; v < GC; ++v) {
            if (v0 + v >= g) break;
            A y[W];
            if constexpr (VEC) unpack<T>(raw[u][v], y);
            else y[0] = Tr<T>::to(raw1[u][v]);
#pragma unroll
            for (int i = 0; i < W; ++i) acc[u][i] = (v0 + v == 0) ? y[i] : Tr<T>::add(acc[u][i], y[i]);
          }
          if (v0 + GC >= g && off[u] != ~(size_t)0) {  // fold complete: epilogue (K3) and store
            if (do_scale) {
#pragma unroll
              for (int i = 0; i < W; ++i) acc[u][i] = Tr<T>::mul(acc[u][i], p.scale);
            }
            if constexpr (VEC) st_vec(dst + off[u], pack<T>(acc[u]));
            else st_elem<T>(dst + off[u], Tr<T>::from(acc[u][0]));
          }
        }
      }
    }
  }
}

// Fill the phase's unit table (and RS source table); shared by both data paths.
template <typename T, int W>
__device__ __forceinline__ void fill_units(const KParams& p, int me, const PhaseCtx& x, UnitDesc* units,
                                           const char** srcs, uint32_t* pref) {
  __syncthreads();  // the previous phase's readers of the tables are done
  if ((int)threadIdx.x < x.nunits) {
    int sr;
    const Span sp = slice_span<W>(p, unit_block(p, me, x, threadIdx.x, &sr), x.s);
    units[threadIdx.x] = UnitDesc{sp.e0, sp.nvec * (uint32_t)(W * sizeof(T)), sp.rem,
                                  x.kind == kPhRS ? nullptr : src_base<T>(p, me, x, 0, sr)};
  }
  if (x.kind == kPhRS && (int)threadIdx.x < x.g) srcs[threadIdx.x] = src_base<T>(p, me, x, threadIdx.x, me);
  __syncthreads();
  if (threadIdx.x == 0 && pref) {
    uint32_t acc = 0;
    for (int u = 0; u < x.nunits; ++u) {
      pref[u] = acc;
      acc += units[u].bytes / (uint32_t)(W * sizeof(T));
    }
    pref[x.nunits] = acc;
  }
  __syncthreads();
}

// ragged remainders (< 16 B where a slice is cut by n), element by element
template <typename T>
__device__ __forceinline__ void ragged_tails(const KParams& p, const PhaseCtx& x, char* dst, const UnitDesc* units,
                                             const char* const* srcs) {
  using A = typename Tr<T>::Acc;
  const bool do_scale = x.kind == kPhRS && x.last && p.op == kAvg;
  for (int u = 0; u < x.nunits; ++u) {
    const UnitDesc ud = units[u];
    if (threadIdx.x < ud.rem) {
      const size_t o = (ud.e0 + (size_t)ud.bytes / sizeof(T) + threadIdx.x) * sizeof(T);
      if (x.kind == kPhRS) {
        A a = 0;
        for (int v = 0; v < x.g; ++v) {
          const A y = Tr<T>::to(ld_elem<T>(srcs[v] + o));
          a = v == 0 ? y : Tr<T>::add(a, y);
        }
        if (do_scale) a = Tr<T>::mul(a, p.scale);
        st_elem<T>(dst + o, Tr<T>::from(a));
      } else {
        st_elem<T>(dst + o, ld_elem<T>(ud.src + o));
      }
    }
  }
}

template <typename T, bool VEC>
__device__ void ldg_phase(const KParams& p, int me, const PhaseCtx& x) {
  constexpr int W = VEC ? Tr<T>::W : 1;
  __shared__ UnitDesc s_units[kMaxRanks];
  __shared__ const char* s_srcs[kMaxRanks];
  __shared__ uint32_t s_pref[kMaxRanks + 1];
  fill_units<T, W>(p, me, x, s_units, s_srcs, s_pref);
  char* dst = dst_base(p, me, x);
  if (x.kind != kPhRS) ldg_phase_g<T, VEC, 1>(p, x, dst, s_units, s_pref, s_srcs);
  else switch (x.g) {
      case 2: ldg_phase_g<T, VEC, 2>(p, x, dst, s_units, s_pref, s_srcs); break;
      case 4: ldg_phase_g<T, VEC, 4>(p, x, dst, s_units, s_pref, s_srcs); break;
      case 8: ldg_phase_g<T, VEC, 8>(p, x, dst, s_units, s_pref, s_srcs); break;
      default: ldg_phase_g<T, VEC, 0>(p, x, dst, s_units, s_pref, s_srcs); break;
    }
  ragged_tails<T>(p, x, dst, s_units, s_srcs);
}

// ------------------------------------------------------------------------ TMA-staged phases
// The 16-byte-vector path of every phase (RS, AG, copy-in/out) runs through a kStages-deep
// shared-memory ring filled by bulk asynchronous copies (cp.async.bulk, the TMA engine's
// linear mode) from local or peer-mapped global memory.  One elected thread issues the
// copies and arms an mbarrier per stage with the expected byte count; all 512 threads wait
// on it, fold the g staged segments in ascending member order from shared memory, and
// store the result with 16-byte st.global.  Bytes in flight per SM = CTAs/SM * kStages *
// kStageBytes (default 2 * 2 * 48 KB), independent of registers -- the latency-hiding budget
// HBM and NVLink need (round-1 ncu: the register-staged path sat at 16 warps/SM and 48% of
// DRAM peak).  Defaults picked by the stage/size sweep in profiles/r01_tma_sweep.txt.
#ifndef DDL_TMA_STAGES
#define DDL_TMA_STAGES 2
#endif
#ifndef DDL_TMA_STAGE_KB
#define DDL_TMA_STAGE_KB 48
#endif
#ifndef DDL_TMA_MINBLOCKS
#define DDL_TMA_MINBLOCKS 2
#endif
constexpr int kStages = DDL_TMA_STAGES;
constexpr uint32_t kStageBytes = DDL_TMA_STAGE_KB * 1024;
// Copy phases (allgather, copy-in/out) run the same ring as kCopySub smaller sub-stages with
// their own mbarriers (more loads in flight, each store issued as its load lands; -0.7 % on
// the bench step, profiles/r02_ab/r02_ab11.txt; DDL_DEEP_COPY=0: the 2-stage ring as for RS).
#ifndef DDL_COPY_SUB
#define DDL_COPY_SUB 8
#endif
#ifndef DDL_COPY_LAG
#define DDL_COPY_LAG 2
#endif
constexpr int kCopySub = DDL_COPY_SUB;
constexpr size_t kTmaSmem =
    (size_t)kStages * kStageBytes + kStages * sizeof(uint64_t) + 16 + kCopySub * sizeof(uint64_t);

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return (uint32_t)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "DDL_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra DDL_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// The same with an L2 eviction-priority policy (createpolicy).
__device__ __forceinline__ void tma_load_hint(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_store_hint(void* gdst, const void* ssrc, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes), "l"(pol)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Bulk store shared -> global (async proxy), grouped per thread.
__device__ __forceinline__ void tma_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {  // sources of all my bulk stores read
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {  // all my bulk stores performed
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// Make data that generic-proxy stores (this CTA's or a peer's, acquired through a device
// barrier) visible to this thread's subsequent async-proxy (bulk copy) reads.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

struct Pipe {
  char* smem;
  uint64_t* bar;
  uint32_t* stored;  // PATH 5: consumer warps that finished storing a chunk (monotone, smem)
  uint64_t* cbar;    // kCopySub sub-stage barriers of the deep copy pipeline
  uint32_t seq;      // chunks consumed so far by this CTA (identical in every thread)
  uint32_t sseq;     // chunks counted in *stored so far (stream phases only)
  uint32_t cseq;     // sub-stage chunks consumed by the deep copy pipeline (thread 0)
};

__device__ __forceinline__ void pipe_init(Pipe& pp) {
  extern __shared__ __align__(128) char dsmem[];
  pp.smem = dsmem;
  pp.bar = reinterpret_cast<uint64_t*>(dsmem + (size_t)kStages * kStageBytes);
  pp.stored = reinterpret_cast<uint32_t*>(pp.bar + kStages);
  pp.cbar = reinterpret_cast<uint64_t*>(dsmem + (size_t)kStages * kStageBytes + kStages * sizeof(uint64_t) + 16);
  pp.seq = 0;
  pp.sseq = 0;
  pp.cseq = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&pp.bar[s], 1);
    for (int s = 0; s < kCopySub; ++s) mbar_init(&pp.cbar[s], 1);
    *pp.stored = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

template <typename T>
__device__ void tma_phase(const KParams& p, int me, const PhaseCtx& x, Pipe& pp) {
  using A = typename Tr<T>::Acc;
  constexpr int W = Tr<T>::W;
  __shared__ UnitDesc s_units[kMaxRanks];
  __shared__ const char* s_srcs[kMaxRanks];
  const uint32_t CB = (kStageBytes / (uint32_t)x.g) & ~15u;  // bytes per source per stage
  const bool do_scale = x.kind == kPhRS && x.last && p.op == kAvg;
  char* dst = dst_base(p, me, x);
  fill_units<T, W>(p, me, x, s_units, s_srcs, nullptr);
  if (x.kind != kPhRS && p.deep_copy) {
    // Deep copy pipeline (default; DDL_DEEP_COPY=0 turns it off): thread 0 streams the phase through
    // kCopySub sub-stages of the ring -- kCopySub - kLag loads in flight, every bulk store
    // issued as soon as its load lands, a sub-stage reloaded once the store issued kLag
    // chunks earlier has read it -- while the other threads go straight to the ragged tails.
    constexpr uint32_t SB = (uint32_t)(kStages * kStageBytes / kCopySub) & ~15u;
    constexpr int kLag = DDL_COPY_LAG;
    if (threadIdx.x == 0) {
      uint32_t ctot = 0;
      for (int u = 0; u < x.nunits; ++u) ctot += (s_units[u].bytes + SB - 1) / SB;
      const bool evf = x.kind == kPhAG && (p.l2hint & 2) && (x.last || !(p.l2hint & 32));
      const uint64_t pol = evf ? policy_evict_first() : 0;
      int lu = 0, su = 0;
      uint32_t loff = 0, soff = 0;
      auto next_chunk = [&](int& u, uint32_t& off) -> uint32_t {  // bytes of the chunk at (u, off)
        while (off >= s_units[u].bytes) {
          ++u;
          off = 0;
        }
        return min(SB, s_units[u].bytes - off);
      };
      auto issue = [&](uint32_t j) {
        const uint32_t bytes = next_chunk(lu, loff);
        const int sub = (int)((pp.cseq + j) % kCopySub);
        mbar_arm(&pp.cbar[sub], bytes);
        tma_load(pp.smem + (size_t)sub * SB, s_units[lu].src + s_units[lu].e0 * sizeof(T) + loff, bytes,
                 &pp.cbar[sub]);
        loff += bytes;
      };
      if (ctot) fence_proxy_async_global();
#if DDL_MUTATE == 3  // mutation check: every copy phase drops its last chunk
      if (ctot > 1) --ctot;
#endif
      for (uint32_t j = 0; j < ctot && j < (uint32_t)kCopySub; ++j) issue(j);
      for (uint32_t j = 0; j < ctot; ++j) {
        const uint32_t cs = pp.cseq + j;
        const int sub = (int)(cs % kCopySub);
        const uint32_t bytes = next_chunk(su, soff);
        mbar_wait(&pp.cbar[sub], (cs / kCopySub) & 1u);
        char* pd = dst + s_units[su].e0 * sizeof(T) + soff;
        if (evf) tma_store_hint(pd, pp.smem + (size_t)sub * SB, bytes, pol);
        else tma_store(pd, pp.smem + (size_t)sub * SB, bytes);
        soff += bytes;
        if (j >= (uint32_t)kLag && j - kLag + kCopySub < ctot) {
          asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kLag) : "memory");
          issue(j - kLag + kCopySub);
        }
      }
      // the tail: stores whose sub-stages are not reloaded
      tma_store_wait_all();
      fence_proxy_async_global();
      pp.cseq += ctot;
    }
    ragged_tails<T>(p, x, dst, s_units, s_srcs);
    return;
  }
  uint32_t total = 0;
  for (int u = 0; u < x.nunits; ++u) total += (s_units[u].bytes + CB - 1) / CB;

  // producer state (thread 0 only): next unit / byte offset to issue
  int pu = 0;
  uint32_t poff = 0;
  auto issue = [&](uint32_t sq) {
    while (poff >= s_units[pu].bytes) {
      ++pu;
      poff = 0;
    }
    const UnitDesc ud = s_units[pu];
    const uint32_t bytes = min(CB, ud.bytes - poff);
    const int st = (int)(sq % kStages);
    char* sbase = pp.smem + (size_t)st * kStageBytes;
    const size_t go = ud.e0 * sizeof(T) + poff;
    mbar_arm(&pp.bar[st], bytes * (uint32_t)x.g);
    if (x.kind == kPhRS && ((x.first && (p.l2hint & 1)) || (!x.first && (p.l2hint & 4)))) {
      const uint64_t pol = policy_evict_first();
      for (int v = 0; v < x.g; ++v) tma_load_hint(sbase + (size_t)v * CB, s_srcs[v] + go, bytes, &pp.bar[st], pol);
    } else if (x.kind == kPhRS) {
      for (int v = 0; v < x.g; ++v) tma_load(sbase + (size_t)v * CB, s_srcs[v] + go, bytes, &pp.bar[st]);
    } else {
      tma_load(sbase, ud.src + go, bytes, &pp.bar[st]);
    }
    poff += bytes;
  };
  if (threadIdx.x == 0 && total) {
    fence_proxy_async_global();
    for (uint32_t j = 0; j < total && j < (uint32_t)kStages; ++j) issue(pp.seq + j);
  }

  int cu = 0;
  uint32_t coff = 0;
  for (uint32_t j = 0; j < total; ++j) {
    while (coff >= s_units[cu].bytes) {
      ++cu;
      coff = 0;
    }
    const uint32_t bytes = min(CB, s_units[cu].bytes - coff);
    const uint32_t sq = pp.seq + j;
    const int st = (int)(sq % kStages);
    const char* sbase = pp.smem + (size_t)st * kStageBytes;
    char* pd = dst + s_units[cu].e0 * sizeof(T) + coff;
    mbar_wait(&pp.bar[st], (sq / kStages) & 1u);
    const uint32_t nv = bytes / 16u;
    if (x.kind == kPhRS) {
      // partials of a non-last RS phase are read again by the next phase (and later
      // overwritten): keep them in L2 (evict_last, bit 3); the last phase's results keep the
      // normal priority unless bit 4 (they would otherwise linger as evict_last after the call)
      const bool keep = (p.l2hint & 8) && (!x.last || (p.l2hint & 16));
      const uint64_t pol_last = keep ? policy_evict_last() : 0;
      for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
        A acc[W];
#if DDL_MUTATE == 1  // mutation check (scripts/gpu_mutation_check.sh): fold the members in descending order
        unpack<T>(*reinterpret_cast<const uint4*>(sbase + (size_t)(x.g - 1) * CB + (size_t)i * 16), acc);
        for (int v = x.g - 2; v >= 0; --v) {
#else
        unpack<T>(*reinterpret_cast<const uint4*>(sbase + (size_t)i * 16), acc);
        for (int v = 1; v < x.g; ++v) {
#endif
          A y[W];
          unpack<T>(*reinterpret_cast<const uint4*>(sbase + (size_t)v * CB + (size_t)i * 16), y);
#pragma unroll
          for (int k = 0; k < W; ++k) acc[k] = Tr<T>::add(acc[k], y[k]);
        }
#if DDL_MUTATE == 2  // mutation check: the fused 1/P scale dropped
        if (false) {
#else
        if (do_scale) {
#endif
#pragma unroll
          for (int k = 0; k < W; ++k) acc[k] = Tr<T>::mul(acc[k], p.scale);
        }
        if (keep) st_vec_hint(pd + (size_t)i * 16, pack<T>(acc), pol_last);
        else st_vec(pd + (size_t)i * 16, pack<T>(acc));
      }
    } else if (threadIdx.x == 0) {
      // copy: one bulk store from the stage (async proxy); the stage is reusable once the
      // store has read it
      // AG stores: evict_first (bit 1) -- with bit 5 only in the LAST allgather phase, whose
      // stores nobody reads again in the call; an earlier AG phase's stores are the next AG
      // phase's sources (normal priority, or evict_last with bit 6)
      const bool ag_first = x.kind == kPhAG && (p.l2hint & 2) && (x.last || !(p.l2hint & 32));
      const bool ag_last = x.kind == kPhAG && !x.last && (p.l2hint & 64);
      if (ag_first) tma_store_hint(pd, sbase, bytes, policy_evict_first());
      else if (ag_last) tma_store_hint(pd, sbase, bytes, policy_evict_last());
      else tma_store(pd, sbase, bytes);
      tma_store_wait_read();
    }
    coff += bytes;
    __syncthreads();  // every thread is done with stage st
    if (threadIdx.x == 0 && j + kStages < total) issue(sq + kStages);
  }
  if (x.kind != kPhRS && threadIdx.x == 0) {
    tma_store_wait_all();        // the bulk stores are performed ...
    fence_proxy_async_global();  // ... and ordered before this thread's generic operations
  }
  pp.seq += total;
  ragged_tails<T>(p, x, dst, s_units, s_srcs);
}

// Experimental kernel variants (PATH 3 rank-level dynamic, PATH 4 work stealing, PATH 5
// streaming): parity-tested, measured slower than PATH 2 in loopback.
// ------------------------------------------------------------------------ NVLS phases (PATH 7)
// "mix and match ... reduce-scatter and all-gather implementations" per decomposed piece
// (P:L54 (3)): on an NVSwitch with multicast (NVLS), phase d of a group can run IN the switch.
// RS: rank r loads each 16-B vector of its blocks A_{d+1}(r) through the group's multicast
// address with multimem.ld_reduce -- the switch returns the sum over the g_d members' copies
// (fold order chosen by the switch: not the direct path's ascending order, so fp32 / bf16
// are tolerance-gated, int32 stays exact) -- applies the fused 1/P scale in the last RS
// phase and stores locally.  AG: rank r multicast-stores its blocks A_{d+1}(r) once
// (multimem.st): the switch writes them into every member.  Per GPU that moves ~S(1+1/P)
// bytes per direction instead of 2S(P-1)/P.  Buffers are 16-B multiples (host-checked), so
// spans have no ragged tail.  Accesses through the multicast alias and the unicast alias of
// the same memory are ordered with fence.proxy.alias around every phase (and the device
// barriers' release/acquire at .sys scope order them across GPUs).
__device__ __forceinline__ void fence_proxy_alias() { asm volatile("fence.proxy.alias;" ::: "memory"); }

template <typename T>
__device__ __forceinline__ uint4 mc_ld_reduce(const char* a);
template <>
__device__ __forceinline__ uint4 mc_ld_reduce<float>(const char* a) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a) : "memory");
  return v;
}
template <>
__device__ __forceinline__ uint4 mc_ld_reduce<__nv_bfloat16>(const char* a) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a) : "memory");
  return v;
}
template <>
__device__ __forceinline__ uint4 mc_ld_reduce<int32_t>(const char* a) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(w[k]) : "l"(a + 4 * k) : "memory");
  return make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ void mc_st(char* a, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(a), "f"(__uint_as_float(v.x)),
               "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)), "f"(__uint_as_float(v.w))
               : "memory");
}

template <typename T>
__device__ void nvls_phase(const KParams& p, int me, const PhaseCtx& x) {
  using A = typename Tr<T>::Acc;
  constexpr int W = Tr<T>::W;
  const Topo& t = p.t;
  const int nb = nblocks(t, x.d + 1);
  const bool rs = x.kind == kPhRS;
  const bool do_scale = rs && x.last && p.op == kAvg;
  char* mc = p.mc[x.d];
  char* dst = dst_base(p, me, x);
  const char* own = static_cast<const char*>(p.work[me]);
  fence_proxy_alias();
  for (int u = 0; u < nb; ++u) {
    const Span sp = slice_span<W>(p, block_of(t, me, x.d + 1, u), x.s);  // RS: reduce; AG: broadcast
    for (uint32_t i = threadIdx.x; i < sp.nvec; i += blockDim.x) {
      const size_t off = (sp.e0 + (uint64_t)i * W) * sizeof(T);
      if (p.nvls_emulate) {
        if (rs) {
          A a[W];
          for (int v = x.g - 1; v >= 0; --v) {
            const int m = member(t, me, x.d, v);
            A y[W];
            unpack<T>(ld_vec(static_cast<const char*>(x.first ? p.in[m] : p.work[m]) + off), y);
#pragma unroll
            for (int k = 0; k < W; ++k) a[k] = v == x.g - 1 ? y[k] : Tr<T>::add(a[k], y[k]);
          }
          if (do_scale) {
#pragma unroll
            for (int k = 0; k < W; ++k) a[k] = Tr<T>::mul(a[k], p.scale);
          }
          st_vec(dst + off, pack<T>(a));
        } else {
          const uint4 v = ld_vec(own + off);
          for (int l = 0; l < t.g[x.d]; ++l) st_vec(static_cast<char*>(p.work[member(t, me, x.d, l)]) + off, v);
        }
        continue;
      }
      if (rs) {
        uint4 v = mc_ld_reduce<T>(mc + off);
        if (do_scale) {
          A a[W];
          unpack<T>(v, a);
#pragma unroll
          for (int k = 0; k < W; ++k) a[k] = Tr<T>::mul(a[k], p.scale);
          v = pack<T>(a);
        }
        st_vec(dst + off, v);
      } else {
        mc_st(mc + off, ld_vec(own + off));
      }
    }
  }
  fence_proxy_alias();
}

#include "ddl_device_variants.cuh"

// ------------------------------------------------------------------------ the hierarchical kernel
// PATH: 0 = element-wise loads (unaligned RS/AG layouts), 1 = 16-byte register-staged
// loads, 2 = 16-byte TMA-staged (default), 4 = TMA-staged with work stealing, 5 = streaming,
// 6 = TMA-staged in waves (large messages), 7 = NVLS phases (multimem) where p.nvls_mask says,
// register-staged direct phases elsewhere.
template <typename T, int PATH>
__global__ void __launch_bounds__(kThreads, (PATH >= 2 && PATH != 7) ? DDL_TMA_MINBLOCKS : 1) ddl_hier_kernel(const __grid_constant__ KParams p) {
  pdl_begin();
  constexpr bool VEC = PATH >= 1;
  constexpr bool NVLS = PATH == 7;  // NVLS phases where nvls_mask says, register-staged elsewhere
  constexpr bool TMA = PATH >= 2 && !NVLS;
  constexpr bool STEAL = PATH == 4;
  constexpr bool STREAM = PATH == 5;
  constexpr bool WAVES = PATH == 6;
  const int me = p.loopback ? (p.transposed ? (int)blockIdx.x : (int)blockIdx.y) : p.rank;
  const uint32_t e = rank_epoch_begin(p, me);
  if (me == p.skip_rank) return;
  const Topo& t = p.t;
  const int L = t.nlive;
  const int me_ = me;
  auto group_peer = [&](int j) { return [&p, me_, j](int l) { return barrier_peer(p.t, me_, j, l); }; };
  Pipe pp;
  if constexpr (TMA) pipe_init(pp);

  auto run = [&](const PhaseCtx& x, int j) {
    if constexpr (STREAM) {
      // Streaming needs every source block's producing phase to publish progress; the
      // copy-in of an allgather-only call does not, so that mode keeps its barriers.
      if ((x.kind == kPhRS || x.kind == kPhAG) && (p.mode & kRS)) {
        stream_phase<T>(p, me, x, pp, j, j > 0, e);
        return;
      }
    }
    if constexpr (STEAL) {
      if (x.kind == kPhRS || x.kind == kPhAG) {
        steal_phase<T>(p, me, x, pp, j);
        return;
      }
    }
    if constexpr (NVLS) {
      if ((x.kind == kPhRS || x.kind == kPhAG) && ((p.nvls_mask >> x.d) & 1)) {
        nvls_phase<T>(p, me, x);
        return;
      }
      fence_proxy_alias();  // sources may have been written through a multicast alias
    }
    if constexpr (TMA) tma_phase<T>(p, me, x, pp);
    else ldg_phase<T, VEC>(p, me, x);
  };
  // STEAL: before signalling barrier j, wait until this CTA's slice of phase j-1 is done
  PhaseCtx prev{};
  bool have_prev = false;
  auto settle = [&](int j) -> bool {
    if constexpr (STEAL) {
      if (have_prev) return own_slice_done<T>(p, me, prev, j - 1);
    }
    return true;
  };
  // trace events: 0 start, 1 after copy-in, 2+2j after barrier j, 3+2j after the phase it gates,
  // 2+2*(2L) after the end barrier (waves > 1: the last wave's)
  trace_ev(p, me, 0);
  // Loopback: every virtual rank's inputs are ready when the launch starts and nothing can
  // touch any buffer before the whole launch ends (stream order), so the start barrier
  // (when there is no copy-in) and the end barrier are implied by the kernel boundary.
  const bool cin = (p.mode & (kCinAll | kCinOwn)) != 0;
  const bool implied_start = p.loopback && !cin;
  // Waves: the call is nwaves independent all-reduces of disjoint element sets (slice
  // w*gridDim.x + blockIdx.x of every block), run one after another by each CTA, so the
  // working set of a wave can stay in L2 and one CTA's barrier waits overlap other CTAs'
  // streaming.  Wave w's barriers release epoch e+w (the rank epoch advances by nwaves per
  // call; flags are monotone, so a peer already in a later wave also satisfies the wait).
  // Without copy-in the inputs of every wave are ready at the call start (barrier 0 of wave 0
  // covers them) and no wave writes what another wave reads, so barrier 0 of waves > 0 is
  // skipped; with copy-in it publishes that wave's copied slice.
  // (PATH 6 only: the TMA-staged kernel with the wave loop compiled in, so PATH 2's code and
  // registers stay those of a single wave -- the loop cost PATH 2 1-4 % at 8-64 MiB and made
  // the register-staged kernel spill at its 128-register cap)
  const int nw = (WAVES && p.nwaves > 1) ? p.nwaves : 1;
  uint32_t ew = e;
#pragma unroll 1
  for (int w = 0; w < nw; ++w) {
    ew = e + (uint32_t)w;
    const int sidx = w * cta_count(p) + cta_id(p);
    const bool tr = w == nw - 1;
    auto ctx = [&](int kind, int d, bool first, bool last) {
      PhaseCtx x = phase_ctx(p, me, kind, d, first, last);
      x.s = sidx;
      return x;
    };
    if (p.mode & kCinAll) run(ctx(kPhCin, 0, false, false), -1);
    if ((p.mode & kCinOwn) && p.cin[me] != static_cast<const char*>(p.work[me]) + (size_t)me * p.q * sizeof(T))
      run(ctx(kPhCinOwn, 0, false, false), -1);
    if (tr) trace_ev(p, me, 1);
    const bool skip_b0 = (w == 0 && implied_start) || (w > 0 && !cin);
    if (p.mode & kRS) {
      for (int j = 0; j < L; ++j) {
        if (!settle(j)) return;
        if (!(j == 0 && skip_b0) && !(STREAM && j > 0) &&
            !dbarrier(p, me, j, barrier_npeers(t, j), ew, group_peer(j), j == 0 && w == 0))
          return;
        if (tr) trace_ev(p, me, 2 + 2 * j);
        prev = ctx(kPhRS, t.live[j], j == 0, j == L - 1);
        run(prev, j);
        have_prev = true;
        if (tr) trace_ev(p, me, 3 + 2 * j);
      }
    }
    if (p.mode & kAG) {
      for (int jj = 0; jj < L; ++jj) {
        const int j = L + jj;
        if (!settle(j)) return;
        if (!(STREAM && (p.mode & kRS)) && !((p.mode & kRS) == 0 && jj == 0 && w > 0 && !cin) &&
            !dbarrier(p, me, j, barrier_npeers(t, j), ew, group_peer(j), jj == 0 && !(p.mode & kRS) && w == 0))
          return;
        if constexpr (NVLS) {
          // an NVLS allgather PUSHES (multimem.st) into the members of its group: before this
          // rank forwards what it received, the previous AG phase's group must have finished
          // pushing into it -- a barrier with that group too (its own slot, 2L+jj)
          const int pd = jj > 0 ? t.live[L - jj] : -1;
          if (pd >= 0 && ((p.nvls_mask >> pd) & 1)) {
            auto pushers = [&t, me_, pd](int l) {
              const int c = coord(t, me_, pd);
              return member(t, me_, pd, l < c ? l : l + 1);
            };
            if (!dbarrier(p, me, 2 * L + jj, t.g[pd] - 1, ew, pushers)) return;
          }
        }
        if (tr) trace_ev(p, me, 2 + 2 * j);
        prev = ctx(kPhAG, t.live[L - 1 - jj], false, jj == L - 1);
        run(prev, j);
        have_prev = true;
        if (tr) trace_ev(p, me, 3 + 2 * j);
      }
    }
    const int last_phase = (p.mode & kAG) ? 2 * L - 1 : L - 1;
    if (p.mode & kCoutAll) {
      if (!settle(last_phase + 1)) return;
      __syncthreads();
      run(ctx(kPhCout, 0, false, false), -1);
    }
    if (w == nw - 1 && L > 0 && !p.loopback) {
      if (!(p.mode & kCoutAll) && !settle(last_phase + 1)) return;
      if (!dbarrier(p, me, 2 * L, barrier_npeers(t, 2 * L), ew, group_peer(2 * L))) return;
    }
  }
  trace_ev(p, me, 2 + 2 * (2 * L));
  rank_epoch_end(p, me, ew, STEAL ? 2 * L : 0);
}

// ------------------------------------------------------------------------ grouped all-reduce
// Several independent buffers ("buckets", e.g. DDP gradient buckets) all-reduced by ONE
// launch.  The grid is split into channels (contiguous CTA ranges); channel ch runs its
// buckets one after another, each with the full hierarchical schedule of a4-a7 on its own
// CTAs (CTA c of a channel handles slice c of every block of the bucket), so one channel's
// L2-bound phases and barrier waits overlap another channel's DRAM-bound phases.  Per bucket
// the fold order is that of a single ddl_allreduce (only the slicing differs), so results
// are bit-identical to it.  Bucket k of a channel releases epoch e+k (the rank epoch advances
// by the longest channel's bucket count); zero-copy buffers only (no copy-in), so barrier 0
// runs only before a channel's first bucket (and not at all in loopback).
constexpr int kMaxBuckets = 8;
constexpr int kMaxChannels = 4;
struct MBucket {
  uint64_t n, q, slice;  // slice: per CTA per wave
  int nwaves;            // waves of this bucket (slice w * channel CTAs + c in wave w)
  void* buf[kMaxRanks];  // every rank's copy (loopback: the virtual ranks' buffers; else peer-mapped)
};
struct MParams {
  KParams p;
  MBucket b[kMaxBuckets];
  int nchan;
  int cta0[kMaxChannels + 1];  // channel ch owns CTAs [cta0[ch], cta0[ch+1])
  int bk0[kMaxChannels + 1];   // and runs buckets order[bk0[ch] .. bk0[ch+1]) in that order
  int order[kMaxBuckets];
  int maxk;                    // most bucket-waves in one channel
};

template <typename T>
__global__ void __launch_bounds__(kThreads, DDL_TMA_MINBLOCKS) ddl_multi_kernel(const __grid_constant__ MParams mp) {
  pdl_begin();
  __shared__ KParams sp;  // this CTA's working copy: per bucket n, q, slice and buffers change
  const KParams& p0 = mp.p;
  const int me = p0.loopback ? (p0.transposed ? (int)blockIdx.x : (int)blockIdx.y) : p0.rank;
  const uint32_t e = rank_epoch_begin(p0, me);
  if (me == p0.skip_rank) return;
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(&p0);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&sp);
    for (uint32_t i = threadIdx.x; i < sizeof(KParams) / 4; i += blockDim.x) dst[i] = src[i];
  }
  int ch = 0;
  const int cid = cta_id(p0);
  while (cid >= mp.cta0[ch + 1]) ++ch;
  const int lc = cid - mp.cta0[ch];
  const Topo& t = p0.t;
  const int L = t.nlive;
  const int me_ = me;
  auto group_peer = [&](int j) { return [&t, me_, j](int l) { return barrier_peer(t, me_, j, l); }; };
  Pipe pp;
  pipe_init(pp);  // (its __syncthreads also publishes sp)
  trace_ev(p0, me, 0);
  // trace (DDL_TRACE=1): event 1 + 2*(seq*2L + j) after barrier j of bucket-wave seq, +1 after its phase
  auto tev = [&](int seq_, int j, int after) {
    const int ev = 1 + 2 * (seq_ * 2 * t.nlive + j) + after;
    if (ev < kTraceEvents - 1) trace_ev(p0, me, ev);
  };
  const int cc = mp.cta0[ch + 1] - mp.cta0[ch];
  const int nk = mp.bk0[ch + 1] - mp.bk0[ch];
  uint32_t ew = e;
  int seq = 0;  // bucket-waves done by this channel
#pragma unroll 1
  for (int kw = 0; kw < nk; ++kw) {
    const MBucket& B = mp.b[mp.order[mp.bk0[ch] + kw]];
#pragma unroll 1
    for (int w = 0; w < (B.nwaves > 1 ? B.nwaves : 1); ++w, ++seq) {
    const int k = seq;
    ew = e + (uint32_t)k;
    __syncthreads();  // the previous bucket's readers of sp are done
    if (threadIdx.x == 0) {
      sp.n = B.n;
      sp.q = B.q;
      sp.slice = B.slice;
    }
    if ((int)threadIdx.x < t.P) {
      sp.in[threadIdx.x] = B.buf[threadIdx.x];
      sp.work[threadIdx.x] = B.buf[threadIdx.x];
      sp.out[threadIdx.x] = B.buf[threadIdx.x];
    }
    __syncthreads();
    const KParams& p = sp;
    for (int j = 0; j < L; ++j) {
      if (!(j == 0 && (k > 0 || p0.loopback)) && !dbarrier(p, me, j, barrier_npeers(t, j), ew, group_peer(j)))
        return;
      tev(k, j, 0);
      PhaseCtx x = phase_ctx(p, me, kPhRS, t.live[j], j == 0, j == L - 1);
      x.s = w * cc + lc;
      tma_phase<T>(p, me, x, pp);
      tev(k, j, 1);
    }
    for (int jj = 0; jj < L; ++jj) {
      const int j = L + jj;
      if (!dbarrier(p, me, j, barrier_npeers(t, j), ew, group_peer(j))) return;
      tev(k, j, 0);
      PhaseCtx x = phase_ctx(p, me, kPhAG, t.live[L - 1 - jj], false, jj == L - 1);
      x.s = w * cc + lc;
      tma_phase<T>(p, me, x, pp);
      tev(k, j, 1);
    }
    }
  }
  if (nk > 0 && L > 0 && !p0.loopback && !dbarrier(sp, me, 2 * L, barrier_npeers(t, 2 * L), ew, group_peer(2 * L)))
    return;
  rank_epoch_end(p0, me, e + (uint32_t)(mp.maxk > 0 ? mp.maxk - 1 : 0), 0);
}

// ------------------------------------------------------------------------ one-shot (a9)
// Every rank reads slice c of all P inputs, folds them in the nested order of the live dims
// (level j folds consecutive groups of g_{live[j]} values, rounding at each level like a
// phase boundary, the avg multiply fused into the last level), waits until every rank has
// finished reading, then writes its result.  K = number of live dims (templated so the
// level accumulators stay in registers).

// Feed value x (of rank r, ascending) into the level accumulators; when the last level
// completes, its (scaled, rounded) value is written to res.
template <typename T, int K, int NA>
__device__ __forceinline__ void nested_feed(const KParams& p, const int* gl, const int* Gl, int r,
                                            typename Tr<T>::Acc (*lvl)[NA], typename Tr<T>::Acc* x,
                                            typename Tr<T>::Acc* res) {
  using A = typename Tr<T>::Acc;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int pos = (r / Gl[j]) % gl[j];
#pragma unroll
    for (int k = 0; k < NA; ++k) lvl[j][k] = pos == 0 ? x[k] : Tr<T>::add(lvl[j][k], x[k]);
    if (pos != gl[j] - 1) break;  // group of level j not complete yet
    const bool top = (j == K - 1);
#pragma unroll
    for (int k = 0; k < NA; ++k) {
      A y = lvl[j][k];
      if (top && p.op == kAvg) y = Tr<T>::mul(y, p.scale);
      x[k] = Tr<T>::round(y);
      if (top) res[k] = x[k];
    }
  }
}

template <typename T, int K, int R>
__global__ void __launch_bounds__(kThreads, 1) ddl_oneshot_kernel(const __grid_constant__ KParams p) {
  pdl_begin();
  using A = typename Tr<T>::Acc;
  constexpr int W = Tr<T>::W;
  constexpr int CH = 8;
  const int me = p.loopback ? (int)blockIdx.y : p.rank;
  const uint32_t e = rank_epoch_begin(p, me);
  if (me == p.skip_rank) return;
  const Topo& t = p.t;
  const int P = t.P;
  int gl[K], Gl[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    gl[j] = t.g[t.live[j]];
    Gl[j] = t.G[t.live[j]];
  }
  // R vectors per thread, strided by the CTA width: item i covers elements eoff[i] .. +W
  const uint64_t lo = (uint64_t)blockIdx.x * p.slice;
  const uint64_t hi = lo + p.slice < p.n ? lo + p.slice : p.n;
  auto all = [me](int l) { return all_peer(me, l); };

  // kScratch (multi-process): my input goes to scratch half (e & 1); peers read only the
  // scratch, never my buffer, so the result can be written without a second barrier.  A
  // half is reused two calls later, when every peer has provably finished this call (it
  // signalled the call in between).
  const char* src_of[kMaxRanks];
  for (int r = 0; r < P; ++r)
    src_of[r] = (p.mode & kScratch) ? p.scratch[r] + (e & 1u) * p.scratch_half : static_cast<const char*>(p.in[r]);
  if (p.mode & (kCinAll | kScratch)) {  // publish this CTA's slice of my input
    const char* s = static_cast<const char*>(p.cin[me]);
    char* w = (p.mode & kScratch) ? const_cast<char*>(src_of[me]) : static_cast<char*>(p.work[me]);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint64_t eo = lo + ((uint64_t)i * blockDim.x + threadIdx.x) * W;
      if (eo + W <= hi) st_vec(w + eo * sizeof(T), ld_vec(s + eo * sizeof(T)));
      else
        for (uint64_t x = eo; x < hi; ++x) st_elem<T>(w + x * sizeof(T), ld_elem<T>(s + x * sizeof(T)));
    }
  }
  // loopback without copy-in: inputs are ready at launch (see ddl_hier_kernel)
  if (!(p.loopback && !(p.mode & kCinAll)) && !dbarrier(p, me, 0, P - 1, e, all, true)) return;

  A res[R][W];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const uint64_t eoff = lo + ((uint64_t)i * blockDim.x + threadIdx.x) * W;
    const bool full = eoff + W <= hi;
    const int ntail = (!full && eoff < hi) ? (int)(hi - eoff) : 0;
    if (full) {
      A lvl[K][W];
      for (int r0 = 0; r0 < P; r0 += CH) {
        uint4 raw[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          if (r0 + k >= P) break;
          raw[k] = ld_vec(src_of[r0 + k] + eoff * sizeof(T));
        }
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          if (r0 + k >= P) break;
          A x[W];
          unpack<T>(raw[k], x);
          nested_feed<T, K, W>(p, gl, Gl, r0 + k, lvl, x, res[i]);
        }
      }
    } else {
      for (int k = 0; k < ntail; ++k) {  // ragged end of the vector, one element at a time
        A lvl1[K][1];
        A r1[1];
        for (int r = 0; r < P; ++r) {
          A x[1] = {Tr<T>::to(ld_elem<T>(src_of[r] + (eoff + k) * sizeof(T)))};
          nested_feed<T, K, 1>(p, gl, Gl, r, lvl1, x, r1);
        }
        res[i][k] = r1[0];
      }
    }
  }
  if (!(p.mode & kScratch) && !dbarrier(p, me, 1, P - 1, e, all)) return;
  char* o = static_cast<char*>(p.out[me]);
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const uint64_t eoff = lo + ((uint64_t)i * blockDim.x + threadIdx.x) * W;
    if (eoff + W <= hi) st_vec(o + eoff * sizeof(T), pack<T>(res[i]));
    else
      for (uint64_t x = eoff; x < hi; ++x) st_elem<T>(o + x * sizeof(T), Tr<T>::from(res[i][x - eoff]));
  }
  rank_epoch_end(p, me, e, 0);
}

// ------------------------------------------------------------------------ LL one-shot (a9)
// Small messages across processes ("LL-style flags carried in the
// payload").  Every rank PUSHES its input to every peer as 16-byte lines of two 64-bit words
// {data32 | epoch << 32}: a 64-bit aligned store is single-copy atomic, so a word whose high
// half equals this call's epoch carries this call's data -- no flag barrier, no fence, one
// NVLink crossing per value (the pull one-shot needs a barrier round trip, then a remote-read
// round trip).  Each rank then polls its own receive slots and folds the P values of every
// line in the nested order of the dims (nested_feed, the same F_dims as every other path).
// Receive region: two halves by call parity, slot r of a half holds rank r's lines; a half
// is rewritten two calls later, when every peer has provably finished reading it (to push
// call e+2 a peer must have finished call e+1, which needed this rank's call-e+1 data, sent
// only after this rank finished call e).  The region holds nothing but LL words, so a stale
// word carries an older epoch (epochs start at 1; the region is zeroed at init).
__device__ __forceinline__ void st_ll(char* p, uint64_t a, uint64_t b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_ll(const char* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
// The 8 data bytes of a line as Acc values (2 x 32-bit, or 4 x bf16).
template <typename T>
__device__ __forceinline__ void unpack8(uint32_t lo, uint32_t hi, typename Tr<T>::Acc* a) {
  if constexpr (sizeof(T) == 2) {
    a[0] = Tr<T>::to(lo & 0xFFFFu);
    a[1] = Tr<T>::to(lo >> 16);
    a[2] = Tr<T>::to(hi & 0xFFFFu);
    a[3] = Tr<T>::to(hi >> 16);
  } else {
    a[0] = Tr<T>::to(lo);
    a[1] = Tr<T>::to(hi);
  }
}

// This thread's 8 data bytes of line i (a ragged last line element by element, zero padded
// on the wire only).
template <typename T>
__device__ __forceinline__ void ll_load(const char* src, int nvalid, uint32_t* d) {
  constexpr int NE = 8 / (int)sizeof(T);
  d[0] = d[1] = 0u;
  if (nvalid == NE) {
    const uint2 v = __ldcg(reinterpret_cast<const uint2*>(src));
    d[0] = v.x;
    d[1] = v.y;
  } else {
    for (int k = 0; k < nvalid; ++k) {
      const uint32_t b = ld_elem<T>(src + k * sizeof(T));
      if constexpr (sizeof(T) == 2) d[k >> 1] |= b << (16 * (k & 1));
      else d[k] = b;
    }
  }
}

template <typename T, int K>
__global__ void __launch_bounds__(kThreads, 1) ddl_ll_kernel(const __grid_constant__ KParams p) {
  pdl_begin();
  using A = typename Tr<T>::Acc;
  constexpr int NE = 8 / (int)sizeof(T);  // elements per 8 data bytes
  constexpr int CH = 8;
  const int me = p.loopback ? (int)blockIdx.y : p.rank;  // loopback: grid (ctas, P), co-resident
  const uint32_t e = rank_epoch_begin(p, me);
  if (me == p.skip_rank) return;
  const Topo& t = p.t;
  const int P = t.P;
  int gl[K], Gl[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    gl[j] = t.g[t.live[j]];
    Gl[j] = t.G[t.live[j]];
  }
  const uint64_t nbytes = p.n * sizeof(T);
  const uint64_t nlines = (nbytes + 7) / 8;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t half = (uint64_t)(e & 1u) * (uint64_t)P * p.ll_slot;
  const char* in = static_cast<const char*>(p.cin[me]);
  auto nvalid_of = [&](uint64_t i) {
    const uint64_t left = (nbytes - i * 8) / sizeof(T);
    return left < (uint64_t)NE ? (int)left : NE;
  };
  // 1. push: every line to every peer (fire and forget)
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nlines; i += stride) {
    uint32_t d[2];
    ll_load<T>(in + i * 8, nvalid_of(i), d);
    const uint64_t w0 = ((uint64_t)e << 32) | d[0], w1 = ((uint64_t)e << 32) | d[1];
    for (int m = 0; m < P; ++m)
      if (m != me) st_ll(p.ll[m] + half + (uint64_t)me * p.ll_slot + i * 16, w0, w1);
  }
  // 2. poll my receive slots, fold in the nested order, write (line i is written only by
  //    this thread, after its own input bytes were read again)
  int fail = 0;
  uint64_t t0 = 0;
  uint32_t spins = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nlines && !fail; i += stride) {
    const int nvalid = nvalid_of(i);
    uint32_t d[2];
    ll_load<T>(in + i * 8, nvalid, d);
    const char* mine = p.ll[me] + half + i * 16;
    A lvl[K][NE];
    A res[NE];
    for (int r0 = 0; r0 < P; r0 += CH) {
      uint64_t a[CH], b[CH];
#pragma unroll
      for (int k = 0; k < CH; ++k) {  // all loads of the chunk in flight at once
        const int r = r0 + k;
        if (r >= P) break;
        if (r == me) {
          a[k] = ((uint64_t)e << 32) | d[0];
          b[k] = ((uint64_t)e << 32) | d[1];
        } else {
          ld_ll(mine + (uint64_t)r * p.ll_slot, a[k], b[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int r = r0 + k;
        if (r >= P) break;
        while (!fail && ((uint32_t)(a[k] >> 32) != e || (uint32_t)(b[k] >> 32) != e)) {
          if ((++spins & 255u) == 0) {
            const uint64_t now = globaltimer();
            if (t0 == 0) t0 = now;
            else if (now - t0 > p.timeout_ns) {
              atomicCAS(p.err, 0, kErrTimeout);
              fail = 1;
            }
          }
          ld_ll(mine + (uint64_t)r * p.ll_slot, a[k], b[k]);
        }
        A x[NE];
        unpack8<T>((uint32_t)a[k], (uint32_t)b[k], x);
        nested_feed<T, K, NE>(p, gl, Gl, r, lvl, x, res);
      }
    }
    if (fail) break;
    char* o = static_cast<char*>(p.out[me]) + i * 8;
    if (nvalid == NE) {
      uint32_t w[2];
      if constexpr (sizeof(T) == 2) {
        w[0] = Tr<T>::from(res[0]) | (Tr<T>::from(res[1]) << 16);
        w[1] = Tr<T>::from(res[2]) | (Tr<T>::from(res[3]) << 16);
      } else {
        w[0] = Tr<T>::from(res[0]);
        w[1] = Tr<T>::from(res[1]);
      }
      *reinterpret_cast<uint2*>(o) = make_uint2(w[0], w[1]);
    } else {
      for (int k = 0; k < nvalid; ++k) st_elem<T>(o + k * sizeof(T), Tr<T>::from(res[k]));
    }
  }
  if (__syncthreads_or(fail)) return;  // the call counter stays (like a failed barrier)
  rank_epoch_end(p, me, e, 0);
}

// ------------------------------------------------------------------------ K5 local reduce
// out = s * sum_{j<g} in_j, ascending j.  Grid-stride over 16-byte vectors, up to 8 input
// loads in flight per thread, streaming cache hints (every byte is touched once).
template <typename T, bool VEC>
__global__ void __launch_bounds__(kThreads, 2) ddl_local_reduce_kernel(const __grid_constant__ LRParams p) {
  pdl_begin();
  using A = typename Tr<T>::Acc;
  constexpr int W = VEC ? Tr<T>::W : 1;
  constexpr int CH = 8;
  const uint64_t nitems = p.n / W;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const bool do_scale = p.scale != 1.0f;
  for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < nitems; it += stride) {
    A acc[W];
    for (int j0 = 0; j0 < p.g; j0 += CH) {
      uint4 raw[CH];
      uint32_t raw1[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        if (j0 + j >= p.g) break;
        const char* ps = static_cast<const char*>(p.in[j0 + j]) + it * W * sizeof(T);
        if constexpr (VEC) raw[j] = __ldcs(reinterpret_cast<const uint4*>(ps));
        else raw1[j] = ld_elem<T>(ps);
      }
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        if (j0 + j >= p.g) break;
        A x[W];
        if constexpr (VEC) unpack<T>(raw[j], x);
        else x[0] = Tr<T>::to(raw1[j]);
#pragma unroll
        for (int i = 0; i < W; ++i) acc[i] = (j0 + j == 0) ? x[i] : Tr<T>::add(acc[i], x[i]);
      }
    }
    if (do_scale) {
#pragma unroll
      for (int i = 0; i < W; ++i) acc[i] = Tr<T>::mul(acc[i], p.scale);
    }
    char* pd = static_cast<char*>(p.out) + it * W * sizeof(T);
    if constexpr (VEC) __stcs(reinterpret_cast<uint4*>(pd), pack<T>(acc));
    else st_elem<T>(pd, Tr<T>::from(acc[0]));
  }
  if constexpr (VEC) {  // the last n % W elements
    if (blockIdx.x == 0) {
      const uint64_t e = nitems * W + threadIdx.x;
      if (e < p.n) {
        A a = Tr<T>::to(ld_elem<T>(static_cast<const char*>(p.in[0]) + e * sizeof(T)));
        for (int j = 1; j < p.g; ++j)
          a = Tr<T>::add(a, Tr<T>::to(ld_elem<T>(static_cast<const char*>(p.in[j]) + e * sizeof(T))));
        if (do_scale) a = Tr<T>::mul(a, p.scale);
        st_elem<T>(static_cast<char*>(p.out) + e * sizeof(T), Tr<T>::from(a));
      }
    }
  }
}

// K5 through the TMA ring: every CTA streams chunks (g input segments of CB bytes each,
// bulk-copied into a 2 x 48 KiB shared-memory ring by one elected thread, mbarrier
// expect-tx), folds them in ascending j from shared memory and streams the result out.
// Chunk k of the vector goes to CTA k mod grid.  The ragged end (< 16 B) is element-wise.
template <typename T>
__global__ void __launch_bounds__(kThreads, DDL_TMA_MINBLOCKS) ddl_local_reduce_tma_kernel(
    const __grid_constant__ LRParams p) {
  pdl_begin();
  using A = typename Tr<T>::Acc;
  constexpr int W = Tr<T>::W;
  extern __shared__ __align__(128) char dsmem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsmem + (size_t)kStages * kStageBytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t CB = (kStageBytes / (uint32_t)p.g) & ~15u;
  const uint64_t vbytes = (p.n / W) * 16ull;              // whole vectors
  const uint64_t nchunks = (vbytes + CB - 1) / CB;
  const bool do_scale = p.scale != 1.0f;
  // this CTA's chunks: blockIdx.x, blockIdx.x + gridDim.x, ...
  const uint64_t mine = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto issue = [&](uint64_t k) {  // k-th chunk of this CTA -> stage k % kStages
    const uint64_t chunk = blockIdx.x + k * gridDim.x;
    const uint64_t off = chunk * CB;
    const uint32_t bytes = (uint32_t)(vbytes - off < CB ? vbytes - off : CB);
    const int st = (int)(k % kStages);
    char* sb = dsmem + (size_t)st * kStageBytes;
    mbar_arm(&bar[st], bytes * (uint32_t)p.g);
    for (int j = 0; j < p.g; ++j)
      tma_load(sb + (size_t)j * CB, static_cast<const char*>(p.in[j]) + off, bytes, &bar[st]);
  };
  if (threadIdx.x == 0)
    for (uint64_t k = 0; k < mine && k < (uint64_t)kStages; ++k) issue(k);
  for (uint64_t k = 0; k < mine; ++k) {
    const uint64_t chunk = blockIdx.x + k * gridDim.x;
    const uint64_t off = chunk * CB;
    const uint32_t bytes = (uint32_t)(vbytes - off < CB ? vbytes - off : CB);
    const int st = (int)(k % kStages);
    const char* sb = dsmem + (size_t)st * kStageBytes;
    mbar_wait(&bar[st], (uint32_t)((k / kStages) & 1u));
    char* pd = static_cast<char*>(p.out) + off;
    for (uint32_t i = threadIdx.x; i < bytes / 16u; i += blockDim.x) {
      A acc[W];
      unpack<T>(*reinterpret_cast<const uint4*>(sb + (size_t)i * 16), acc);
      for (int j = 1; j < p.g; ++j) {
        A y[W];
        unpack<T>(*reinterpret_cast<const uint4*>(sb + (size_t)j * CB + (size_t)i * 16), y);
#pragma unroll
        for (int q = 0; q < W; ++q) acc[q] = Tr<T>::add(acc[q], y[q]);
      }
      if (do_scale) {
#pragma unroll
        for (int q = 0; q < W; ++q) acc[q] = Tr<T>::mul(acc[q], p.scale);
      }
      __stcs(reinterpret_cast<uint4*>(pd + (size_t)i * 16), pack<T>(acc));
    }
    __syncthreads();  // stage st consumed
    if (threadIdx.x == 0 && k + kStages < mine) issue(k + kStages);
  }
  if (blockIdx.x == 0) {  // the last n % W elements
    const uint64_t e = (p.n / W) * W + threadIdx.x;
    if (e < p.n) {
      A a = Tr<T>::to(ld_elem<T>(static_cast<const char*>(p.in[0]) + e * sizeof(T)));
      for (int j = 1; j < p.g; ++j)
        a = Tr<T>::add(a, Tr<T>::to(ld_elem<T>(static_cast<const char*>(p.in[j]) + e * sizeof(T))));
      if (do_scale) a = Tr<T>::mul(a, p.scale);
      st_elem<T>(static_cast<char*>(p.out) + e * sizeof(T), Tr<T>::from(a));
    }
  }
}

}  // namespace ddl
