// ddl_device.cuh -- sm_100a kernels of libddl.
//
//   ddl_hier_kernel    one launch = one whole hierarchical collective: copy-in (staged),
//                      RS phases d = live[0..L-1] (K1) with the fused 1/P + cast epilogue
//                      in the last one (K3), AG phases d = live[L-1..0] (K2), copy-out,
//                      separated by 2L+1 per-CTA device barriers (K4).
//   ddl_oneshot_kernel small messages: every rank reads all P inputs, folds them in the
//                      nested order of the dims (same F_dims as the hierarchy), 2 barriers.
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

constexpr int kThreads = 512;
constexpr int kMaxLocalIn = 64;

enum Mode : int {
  kCinAll = 1,    // copy cin[me] -> work[me] (all blocks, this CTA's slices) before the start
  kCinOwn = 2,    // copy cin[me] (one block of q elems) -> work[me] block me
  kRS = 4,
  kAG = 8,
  kCoutAll = 16,  // copy work[me] -> cout[me] (all blocks) after the AG phases
};

enum DType : int { kI32 = 0, kF32 = 1, kBF16 = 2 };
enum Op : int { kSum = 0, kAvg = 1 };
enum Err : int { kErrTimeout = 8 };

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
  uint64_t* trace;     // debug (DDL_TRACE=1): [P][cmax][kTraceEvents] globaltimer stamps, else null
  int stream_every;    // PATH 5: publish progress every k chunks (and at the phase end)
};
constexpr int kTraceEvents = 40;

// Debug timeline: thread 0 of each CTA stamps the global timer at event ev.
__device__ __forceinline__ void trace_ev(const KParams& p, int me, int ev) {
  if (p.trace && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[((size_t)me * p.cmax + blockIdx.x) * kTraceEvents + ev] = t;
    if (ev == 0) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      p.trace[((size_t)me * p.cmax + blockIdx.x) * kTraceEvents + kTraceEvents - 1] = smid;
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
template <typename PeerFn>
__device__ __forceinline__ bool dbarrier(const KParams& p, int me, int slot, int np, uint32_t epoch, PeerFn peer) {
  __syncthreads();  // every thread's stores of the previous phase precede the release below
  int fail = 0;
  if (threadIdx.x < np) {
    const int m = peer(threadIdx.x);
    st_release(flag_slot(p, p.flags[m], slot, blockIdx.x, me), epoch, p.gpu_scope);
    const uint32_t* f = flag_slot(p, p.flags[me], slot, blockIdx.x, m);
    uint64_t t0 = 0;
    uint32_t spins = 0;
    while ((int32_t)(ld_acquire(f, p.gpu_scope) - epoch) < 0) {
      if ((++spins & 1023u) == 0) {
        const uint64_t now = globaltimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > p.timeout_ns) {
          atomicExch(p.err, kErrTimeout);
          fail = 1;
          break;
        }
      }
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
    s_last = (old == gridDim.x - 1);
    if (s_last) *sb = 0;
  }
  __syncthreads();
  if (s_last) {
    for (int j = 0; j < steal_phases; ++j)
      for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
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
__device__ __forceinline__ Span slice_span(const KParams& p, int b) {
  Span s{0, 0, 0};
  const uint64_t cbase = (uint64_t)blockIdx.x * p.slice;
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
    const Span sp = slice_span<W>(p, unit_block(p, me, x, threadIdx.x, &sr));
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
constexpr size_t kTmaSmem = (size_t)kStages * kStageBytes + kStages * sizeof(uint64_t) + 16;

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
  uint32_t seq;      // chunks consumed so far by this CTA (identical in every thread)
  uint32_t sseq;     // chunks counted in *stored so far (stream phases only)
};

__device__ __forceinline__ void pipe_init(Pipe& pp) {
  extern __shared__ __align__(128) char dsmem[];
  pp.smem = dsmem;
  pp.bar = reinterpret_cast<uint64_t*>(dsmem + (size_t)kStages * kStageBytes);
  pp.stored = reinterpret_cast<uint32_t*>(pp.bar + kStages);
  pp.seq = 0;
  pp.sseq = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&pp.bar[s], 1);
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
    if (x.kind == kPhRS) {
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
      for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
        A acc[W];
        unpack<T>(*reinterpret_cast<const uint4*>(sbase + (size_t)i * 16), acc);
        for (int v = 1; v < x.g; ++v) {
          A y[W];
          unpack<T>(*reinterpret_cast<const uint4*>(sbase + (size_t)v * CB + (size_t)i * 16), y);
#pragma unroll
          for (int k = 0; k < W; ++k) acc[k] = Tr<T>::add(acc[k], y[k]);
        }
        if (do_scale) {
#pragma unroll
          for (int k = 0; k < W; ++k) acc[k] = Tr<T>::mul(acc[k], p.scale);
        }
        st_vec(pd + (size_t)i * 16, pack<T>(acc));
      }
    } else if (threadIdx.x == 0) {
      // copy: one bulk store from the stage (async proxy); the stage is reusable once the
      // store has read it
      tma_store(pd, sbase, bytes);
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

// ------------------------------------------------------------------------ work stealing (PATH 4)
// PATH 2's per-CTA slices and per-slice barriers, plus stealing: a CTA that has finished its
// own slice of a phase takes chunks of other slices of the same rank (per-slice ticket
// counters); every processed chunk is counted in its slice's done counter (release), and
// the slice's owner, before signalling the next barrier for its slice, waits until all the
// slice's chunks are done (acquire) -- whoever processed them.  Round-1 traces showed the
// per-CTA phase time is SYSTEMATICALLY SM-dependent (same SMs 25% slower every call,
// scripts/trace_variance.py), so static equal slices leave fast SMs idle at every barrier.
// MEASURED (round 1): parity-green but 5-95% SLOWER than PATH 2 on 8-32 MB messages (the
// per-chunk ticket atomics and the end-of-phase steal scan cost more than the imbalance
// they remove).  Kept behind DDL_STEAL=1.

// vector bytes / remainder of unit (block b) in slice s
template <int W, typename T>
__device__ __forceinline__ void slice_unit_span(const KParams& p, int b, int s, uint64_t* e0, uint32_t* vb,
                                                uint32_t* rem) {
  *vb = 0;
  *rem = 0;
  *e0 = 0;
  const uint64_t cbase = (uint64_t)s * p.slice;
  if (cbase >= p.q) return;
  const uint64_t e = (uint64_t)b * p.q + cbase;
  if (e >= p.n) return;
  uint64_t len = p.q - cbase < p.slice ? p.q - cbase : p.slice;
  if (len > p.n - e) len = p.n - e;
  *e0 = e;
  *vb = (uint32_t)(len / W) * 16u;
  *rem = (uint32_t)(len % W);
}
__device__ __forceinline__ uint32_t unit_chunks(uint32_t vb, uint32_t rem, uint32_t CB) {
  return vb ? (vb + CB - 1) / CB : (rem ? 1u : 0u);
}
template <typename T>
__device__ uint32_t slice_chunks(const KParams& p, int me, const PhaseCtx& x, int s) {
  constexpr int W = Tr<T>::W;
  const uint32_t CB = (kStageBytes / (uint32_t)x.g) & ~15u;
  uint32_t k = 0;
  for (int u = 0; u < x.nunits; ++u) {
    int sr;
    uint64_t e0;
    uint32_t vb, rem;
    slice_unit_span<W, T>(p, unit_block(p, me, x, u, &sr), s, &e0, &vb, &rem);
    k += unit_chunks(vb, rem, CB);
  }
  return k;
}

__device__ __forceinline__ void red_release_add(uint32_t* a, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

// The owner of slice blockIdx.x waits until every chunk of its slice in phase j is done.
template <typename T>
__device__ __forceinline__ bool own_slice_done(const KParams& p, int me, const PhaseCtx& x, int j) {
  __shared__ int s_fail;
  if (threadIdx.x == 0) {
    s_fail = 0;
    const uint32_t K = slice_chunks<T>(p, me, x, blockIdx.x);
    const uint32_t* d = steal_done(p, me, j) + blockIdx.x;
    uint64_t t0 = 0;
    uint32_t spins = 0;
    while (ld_acquire(d, true) < K) {
      if ((++spins & 1023u) == 0) {
        const uint64_t now = globaltimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > p.timeout_ns) {
          atomicExch(p.err, kErrTimeout);
          s_fail = 1;
          break;
        }
      }
    }
  }
  __syncthreads();
  return s_fail == 0;
}

struct StealDesc {
  char* dst;       // destination of the chunk's first byte
  uint32_t bytes;  // vector bytes (0: remainder-only chunk)
  int slice;       // -1: terminator
};

template <typename T>
__device__ void steal_phase(const KParams& p, int me, const PhaseCtx& x, Pipe& pp, int j) {
  using A = typename Tr<T>::Acc;
  constexpr int W = Tr<T>::W;
  __shared__ const char* s_srcs[kMaxRanks];
  __shared__ const char* s_usrc[kMaxRanks];
  __shared__ int s_blk[kMaxRanks];
  __shared__ StealDesc s_desc[kStages];
  // producer's (thread 0) view of the slice it is currently taking chunks from
  __shared__ uint64_t s_e0[kMaxRanks];
  __shared__ uint32_t s_vb[kMaxRanks], s_rem[kMaxRanks], s_kp[kMaxRanks + 1];
  const uint32_t CB = (kStageBytes / (uint32_t)x.g) & ~15u;
  const bool rs = x.kind == kPhRS;
  const bool do_scale = rs && x.last && p.op == kAvg;
  char* dst = dst_base(p, me, x);
  uint32_t* tick = steal_tick(p, me, j);
  uint32_t* done = steal_done(p, me, j);
  const int C = gridDim.x;
  const int own = blockIdx.x;

  __syncthreads();  // previous phase's readers of the tables are done
  if ((int)threadIdx.x < x.nunits) {
    int sr;
    s_blk[threadIdx.x] = unit_block(p, me, x, threadIdx.x, &sr);
    s_usrc[threadIdx.x] = rs ? nullptr : src_base<T>(p, me, x, 0, sr);
  }
  if (rs && (int)threadIdx.x < x.g) s_srcs[threadIdx.x] = src_base<T>(p, me, x, threadIdx.x, me);
  __syncthreads();

  auto load_slice = [&](int sl) -> uint32_t {  // thread 0: span table of slice sl, returns its chunks
    uint32_t k = 0;
    for (int u = 0; u < x.nunits; ++u) {
      uint64_t e0;
      uint32_t vb, rem;
      slice_unit_span<W, T>(p, s_blk[u], sl, &e0, &vb, &rem);
      s_e0[u] = e0;
      s_vb[u] = vb;
      s_rem[u] = rem;
      s_kp[u] = k;
      k += unit_chunks(vb, rem, CB);
    }
    s_kp[x.nunits] = k;
    return k;
  };
  int cur = own;
  uint32_t kcur = 0, tkt = 0, kmax = 0;  // kmax: chunks of slice 0, the largest slice
  bool finished = false;
  auto next_chunk = [&](uint32_t* to) -> bool {
    for (;;) {
      if (cur < 0) return false;
      if (tkt < kcur) {
        *to = tkt;
        tkt = atomicAdd(&tick[cur], 1u);  // prefetch the next ticket of this slice
        return true;
      }
      // steal: probe the following slices 8 at a time (independent loads, one round trip)
      // for one whose ticket counter is below the largest slice's chunk count
      int found = -1;
      while (found < 0) {
        uint32_t tv[8];
        int sl[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          sl[i] = (cur + 1 + i) % C;
          tv[i] = *(volatile uint32_t*)&tick[sl[i]];
        }
        int adv = 8;
#pragma unroll
        for (int i = 7; i >= 0; --i)
          if (sl[i] == own) adv = i;  // wrapped back to our own slice: scan complete
        for (int i = 0; i < adv && found < 0; ++i)
          if (tv[i] < kmax) found = sl[i];
        if (found < 0) {
          if (adv < 8) {
            cur = -1;
            return false;
          }
          cur = (cur + 8) % C;
        }
      }
      cur = found;
      kcur = load_slice(cur);
      tkt = 0xffffffffu;  // no ticket of the new slice yet
      if (kcur == 0 || *(volatile uint32_t*)&tick[cur] >= kcur) continue;
      tkt = atomicAdd(&tick[cur], 1u);
    }
  };
  auto fill = [&](uint32_t sq) {
    if (finished) return;
    const int st = (int)(sq % kStages);
    uint32_t t;
    if (!next_chunk(&t)) {
      finished = true;
      s_desc[st] = StealDesc{nullptr, 0, -1};
      mbar_arm(&pp.bar[st], 0);
      return;
    }
    int u = 0;
    while (t >= s_kp[u + 1]) ++u;
    const uint32_t k = s_kp[u + 1] - s_kp[u];
    const uint32_t off = (t - s_kp[u]) * CB;
    const uint32_t vb = s_vb[u], rem = s_rem[u];
    const uint64_t e0 = s_e0[u];
    const uint32_t bytes = vb > off ? min(CB, vb - off) : 0;
    const size_t go = e0 * sizeof(T) + off;
    if (t - s_kp[u] == k - 1 && rem) {  // the unit's ragged remainder, element-wise, by the producer
      const size_t o0 = (e0 + vb / 16u * W) * sizeof(T);
      for (uint32_t i = 0; i < rem; ++i) {
        const size_t o = o0 + i * sizeof(T);
        if (rs) {
          A a = 0;
          for (int v = 0; v < x.g; ++v) {
            const A y = Tr<T>::to(ld_elem<T>(s_srcs[v] + o));
            a = v == 0 ? y : Tr<T>::add(a, y);
          }
          if (do_scale) a = Tr<T>::mul(a, p.scale);
          st_elem<T>(dst + o, Tr<T>::from(a));
        } else {
          st_elem<T>(dst + o, ld_elem<T>(s_usrc[u] + o));
        }
      }
    }
    s_desc[st] = StealDesc{dst + go, bytes, cur};
    mbar_arm(&pp.bar[st], bytes * (uint32_t)x.g);
    if (bytes) {
      char* sb = pp.smem + (size_t)st * kStageBytes;
      if (rs) {
        for (int v = 0; v < x.g; ++v) tma_load(sb + (size_t)v * CB, s_srcs[v] + go, bytes, &pp.bar[st]);
      } else {
        tma_load(sb, s_usrc[u] + go, bytes, &pp.bar[st]);
      }
    }
  };
  if (threadIdx.x == 0) {
    fence_proxy_async_global();
    kmax = load_slice(0);
    kcur = load_slice(own);
    tkt = atomicAdd(&tick[own], 1u);
    for (int st = 0; st < kStages; ++st) fill(pp.seq + st);
  }

  // consumers; thread 0 also counts the chunks it saw per slice and publishes each slice's
  // count (one release per slice switch) -- the slice owner waits for the total
  int cnt_slice = -1;
  uint32_t cnt = 0;
  for (uint32_t k = 0;; ++k) {
    const uint32_t sq = pp.seq + k;
    const int st = (int)(sq % kStages);
    mbar_wait(&pp.bar[st], (sq / kStages) & 1u);
    const StealDesc d = s_desc[st];
    if (d.slice < 0) {
      pp.seq += k + 1;
      break;
    }
    const char* sbase = pp.smem + (size_t)st * kStageBytes;
    const uint32_t nv = d.bytes / 16u;
    if (rs) {
      for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
        A a[W];
        unpack<T>(*reinterpret_cast<const uint4*>(sbase + (size_t)i * 16), a);
        for (int v = 1; v < x.g; ++v) {
          A y[W];
          unpack<T>(*reinterpret_cast<const uint4*>(sbase + (size_t)v * CB + (size_t)i * 16), y);
#pragma unroll
          for (int q = 0; q < W; ++q) a[q] = Tr<T>::add(a[q], y[q]);
        }
        if (do_scale) {
#pragma unroll
          for (int q = 0; q < W; ++q) a[q] = Tr<T>::mul(a[q], p.scale);
        }
        st_vec(d.dst + (size_t)i * 16, pack<T>(a));
      }
    } else {
      for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x)
        st_vec(d.dst + (size_t)i * 16, *reinterpret_cast<const uint4*>(sbase + (size_t)i * 16));
    }
    __syncthreads();  // stage st consumed; the chunk's stores precede any later release
    if (threadIdx.x == 0) {
      if (d.slice != cnt_slice) {
        if (cnt) red_release_add(&done[cnt_slice], cnt);
        cnt_slice = d.slice;
        cnt = 0;
      }
      ++cnt;
      fill(sq + kStages);
    }
  }
  if (threadIdx.x == 0 && cnt) red_release_add(&done[cnt_slice], cnt);
}

// ------------------------------------------------------------------------ streaming (PATH 5)
// PATH 2 without the inner phase barriers: every CTA publishes, per data phase, how many of
// its chunks are done (a 64-bit (epoch << 32 | count) word, st.release after each chunk), and
// the producer thread of a consumer CTA waits, per chunk it is about to load, only for the
// producer chunks that cover exactly the bytes it needs.  With static slices the producer of
// slice c of any block is always CTA c of the source rank, so the dependency is a count, not
// a barrier: phase d+1 of a slice starts as soon as its first source chunks exist, while
// slower CTAs are still finishing phase d.  (Start and end barriers stay.)
__device__ __forceinline__ uint64_t* prog_word(const KParams& p, int r, int jphase) {
  uint32_t* end = steal_base(p, r) + 16 + 2 * (size_t)kNumSlots * p.cmax;
  uint64_t* base = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(end) + 7) & ~(uintptr_t)7);
  return base + (size_t)jphase * p.cmax;
}
__device__ __forceinline__ void st_release64(uint64_t* a, uint64_t v, bool gpu_scope) {
  if (gpu_scope) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
  else asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire64(const uint64_t* a, bool gpu_scope) {
  uint64_t v;
  if (gpu_scope) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  else asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}

__device__ __forceinline__ PhaseCtx data_phase(const KParams& p, int m, int jj) {
  const int L = p.t.nlive;
  if (jj < L) return phase_ctx(p, m, kPhRS, p.t.live[jj], jj == 0, jj == L - 1);
  return phase_ctx(p, m, kPhAG, p.t.live[2 * L - 1 - jj], false, false);
}
__device__ __forceinline__ uint32_t phase_cb(const PhaseCtx& x) { return (kStageBytes / (uint32_t)x.g) & ~15u; }

// The data phase in which rank m last wrote block b (-1: before the first barrier).
__device__ __forceinline__ int final_phase(const KParams& p, int b, int m) {
  const Topo& t = p.t;
  const int L = t.nlive;
  if (b == m) return (p.mode & kRS) ? L - 1 : -1;
  int idx = -1;
  for (int i = 0; i < L; ++i)
    if (coord(t, b, t.live[i]) != coord(t, m, t.live[i])) idx = i;
  return 2 * L - 1 - idx;  // AG phase of the outermost dim where b and m differ
}

// Where block b (slice c) sits in rank m's phase jj: chunks before its unit, its own chunk
// count, the phase's total, and the phase's chunk bytes.
template <typename T>
__device__ void locate(const KParams& p, int m, int jj, int b, int c, uint32_t* before, uint32_t* own,
                       uint32_t* total, uint32_t* cb) {
  constexpr int W = Tr<T>::W;
  const PhaseCtx x = data_phase(p, m, jj);
  const uint32_t CB = phase_cb(x);
  uint32_t acc = 0, mine = 0, pre = 0;
  for (int u = 0; u < x.nunits; ++u) {
    int sr;
    const int bu = unit_block(p, m, x, u, &sr);
    uint64_t e0;
    uint32_t vb, rem;
    slice_unit_span<W, T>(p, bu, c, &e0, &vb, &rem);
    const uint32_t k = (vb + CB - 1) / CB;
    if (bu == b) {
      pre = acc;
      mine = k;
    }
    acc += k;
  }
  *before = pre;
  *own = mine;
  *total = acc;
  *cb = CB;
}

template <typename T>
__device__ void stream_phase(const KParams& p, int me, const PhaseCtx& x, Pipe& pp, int jphase, bool wait,
                             uint32_t epoch) {
  using A = typename Tr<T>::Acc;
  constexpr int W = Tr<T>::W;
  __shared__ UnitDesc s_units[kMaxRanks];
  __shared__ const char* s_srcs[kMaxRanks];
  // per (unit, source): source rank, its phase, chunks before the block there, chunk bytes,
  // the block's chunks, the phase total
  __shared__ int s_nr[kMaxRanks][kMaxRanks], s_np[kMaxRanks][kMaxRanks];
  __shared__ uint32_t s_nb[kMaxRanks][kMaxRanks], s_ncb[kMaxRanks][kMaxRanks], s_nown[kMaxRanks][kMaxRanks],
      s_ntot[kMaxRanks][kMaxRanks];
  const uint32_t CB = phase_cb(x);
  const bool rs = x.kind == kPhRS;
  const bool do_scale = rs && x.last && p.op == kAvg;
  const int c = blockIdx.x;
  const int nsrc = rs ? x.g : 1;
  char* dst = dst_base(p, me, x);
  fill_units<T, W>(p, me, x, s_units, s_srcs, nullptr);
  uint32_t total = 0;
  for (int u = 0; u < x.nunits; ++u) total += (s_units[u].bytes + CB - 1) / CB;
  const uint64_t ehi = (uint64_t)epoch << 32;
  uint64_t* myprog = prog_word(p, me, jphase) + c;

  if (wait && threadIdx.x == 0) {  // dependency tables
    for (int u = 0; u < x.nunits; ++u) {
      int sr;
      const int b = unit_block(p, me, x, u, &sr);
      for (int v = 0; v < nsrc; ++v) {
        const int m = rs ? member(p.t, me, x.d, v) : sr;
        const int ph = rs ? jphase - 1 : final_phase(p, b, m);
        s_nr[u][v] = m;
        s_np[u][v] = (m == me || ph < 0) ? -1 : ph;  // own data: written by this CTA already
        if (s_np[u][v] >= 0) locate<T>(p, m, ph, b, c, &s_nb[u][v], &s_nown[u][v], &s_ntot[u][v], &s_ncb[u][v]);
      }
    }
  }
  auto wait_for = [&](int u, uint32_t end_bytes, bool whole_phase) -> bool {
    for (int v = 0; v < nsrc; ++v) {
      const int ph = s_np[u][v];
      if (ph < 0) continue;
      uint32_t need = whole_phase ? s_ntot[u][v] + 1
                                  : s_nb[u][v] + min(s_nown[u][v], (end_bytes + s_ncb[u][v] - 1) / s_ncb[u][v]);
      const uint64_t* w = prog_word(p, s_nr[u][v], ph) + c;
      uint64_t t0 = 0;
      uint32_t spins = 0;
      while (ld_acquire64(w, p.gpu_scope) < (ehi | need)) {
        if ((++spins & 1023u) == 0) {
          const uint64_t now = globaltimer();
          if (t0 == 0) t0 = now;
          else if (now - t0 > p.timeout_ns) {
            atomicExch(p.err, kErrTimeout);
            return false;
          }
        }
      }
    }
    return true;
  };

  __shared__ int s_fail;
  if (threadIdx.x == 0) s_fail = 0;
  int pu = 0;
  uint32_t poff = 0;
  bool failed = false;
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
    if (wait && !failed) {
      if (!wait_for(pu, poff + bytes, false)) failed = true;
      fence_proxy_async_global();
    }
    mbar_arm(&pp.bar[st], failed ? 0 : bytes * (uint32_t)x.g);
    if (!failed) {
      if (rs) {
        for (int v = 0; v < x.g; ++v) tma_load(sbase + (size_t)v * CB, s_srcs[v] + go, bytes, &pp.bar[st]);
      } else {
        tma_load(sbase, ud.src + go, bytes, &pp.bar[st]);
      }
    }
    poff += bytes;
  };
  if (threadIdx.x == 0 && total) {
    fence_proxy_async_global();
    for (uint32_t j = 0; j < total && j < (uint32_t)kStages; ++j) issue(pp.seq + j);
  }

  // warps 0..14 consume; warp 15 only publishes progress (its release fences never stall
  // the consumers): each consumer warp counts itself in *pp.stored after storing a chunk
  // (release, CTA scope); the signal lane waits for all 15 and releases (epoch << 32 | chunks
  // done) at GPU/system scope -- cumulative over the warps' stores.
  constexpr uint32_t kCons = kThreads - 32;
  const bool signaller = threadIdx.x >= kCons;
  if (signaller) {
    if (threadIdx.x == kCons) {
      for (uint32_t j = 0; j < total; ++j) {
        const uint32_t want = (pp.sseq + j + 1) * (kCons / 32);  // every consumer warp stored chunk j
        uint32_t got;
        do {
          asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(got) : "r"(smem_u32(pp.stored)) : "memory");
        } while ((int32_t)(got - want) < 0);
        if ((j + 1) % p.stream_every == 0 || j + 1 == total) st_release64(myprog, ehi | (j + 1), p.gpu_scope);
      }
    }
  }
  int cu = 0;
  uint32_t coff = 0;
  for (uint32_t j = 0; j < total && !signaller; ++j) {
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
    if (rs) {
      for (uint32_t i = threadIdx.x; i < nv; i += kCons) {
        A acc[W];
        unpack<T>(*reinterpret_cast<const uint4*>(sbase + (size_t)i * 16), acc);
        for (int v = 1; v < x.g; ++v) {
          A y[W];
          unpack<T>(*reinterpret_cast<const uint4*>(sbase + (size_t)v * CB + (size_t)i * 16), y);
#pragma unroll
          for (int k = 0; k < W; ++k) acc[k] = Tr<T>::add(acc[k], y[k]);
        }
        if (do_scale) {
#pragma unroll
          for (int k = 0; k < W; ++k) acc[k] = Tr<T>::mul(acc[k], p.scale);
        }
        st_vec(pd + (size_t)i * 16, pack<T>(acc));
      }
    } else {
      for (uint32_t i = threadIdx.x; i < nv; i += kCons)
        st_vec(pd + (size_t)i * 16, *reinterpret_cast<const uint4*>(sbase + (size_t)i * 16));
    }
    coff += bytes;
    __syncwarp();  // this warp's stores of the chunk precede lane 0's release below
    if ((threadIdx.x & 31) == 0)
      asm volatile("red.release.cta.shared::cta.add.u32 [%0], 1;" ::"r"(smem_u32(pp.stored)) : "memory");
    asm volatile("bar.sync 1, %0;" ::"r"(kCons) : "memory");  // stage st consumed by all consumers
    if (threadIdx.x == 0 && j + kStages < total) issue(sq + kStages);
  }
  __syncthreads();  // the signal warp has published every chunk
  pp.seq += total;
  pp.sseq += total;
  if (threadIdx.x == 0 && failed) s_fail = 1;
  // ragged remainders: their sources must have finished the whole producing phase
  bool any_rem = false;
  for (int u = 0; u < x.nunits; ++u) any_rem |= s_units[u].rem != 0;
  if (any_rem) {
    if (wait && threadIdx.x == 0 && !failed) {
      for (int u = 0; u < x.nunits; ++u)
        if (s_units[u].rem && !wait_for(u, 0, true)) {
          s_fail = 1;
          break;
        }
    }
    __syncthreads();
    ragged_tails<T>(p, x, dst, s_units, s_srcs);
  }
  __syncthreads();
  if (threadIdx.x == 32) st_release64(myprog, ehi | (total + 1), p.gpu_scope);  // phase complete
}

// ------------------------------------------------------------------------ the hierarchical kernel
// PATH: 0 = element-wise loads (unaligned RS/AG layouts), 1 = 16-byte register-staged
// loads, 2 = 16-byte TMA-staged (default), 4 = TMA-staged with work stealing.
template <typename T, int PATH>
__global__ void __launch_bounds__(kThreads, PATH >= 2 ? DDL_TMA_MINBLOCKS : 1) ddl_hier_kernel(const __grid_constant__ KParams p) {
  constexpr bool VEC = PATH >= 1;
  constexpr bool TMA = PATH >= 2;
  constexpr bool STEAL = PATH == 4;
  constexpr bool STREAM = PATH == 5;
  const int me = p.loopback ? (int)blockIdx.y : p.rank;
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
      if (x.kind == kPhRS || x.kind == kPhAG) {
        const int first = (p.mode & kRS) ? 0 : L;
        stream_phase<T>(p, me, x, pp, j, j > first, e);
        return;
      }
    }
    if constexpr (STEAL) {
      if (x.kind == kPhRS || x.kind == kPhAG) {
        steal_phase<T>(p, me, x, pp, j);
        return;
      }
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
  // 2+2*(2L) after the end barrier
  trace_ev(p, me, 0);
  if (p.mode & kCinAll) run(phase_ctx(p, me, kPhCin, 0, false, false), -1);
  if ((p.mode & kCinOwn) && p.cin[me] != static_cast<const char*>(p.work[me]) + (size_t)me * p.q * sizeof(T))
    run(phase_ctx(p, me, kPhCinOwn, 0, false, false), -1);
  trace_ev(p, me, 1);
  // Loopback: every virtual rank's inputs are ready when the launch starts and nothing can
  // touch any buffer before the whole launch ends (stream order), so the start barrier
  // (when there is no copy-in) and the end barrier are implied by the kernel boundary.
  const bool implied_start = p.loopback && !(p.mode & (kCinAll | kCinOwn));
  if (p.mode & kRS) {
    for (int j = 0; j < L; ++j) {
      if (!settle(j)) return;
      if (!(j == 0 && implied_start) && !(STREAM && j > 0) &&
          !dbarrier(p, me, j, barrier_npeers(t, j), e, group_peer(j)))
        return;
      trace_ev(p, me, 2 + 2 * j);
      prev = phase_ctx(p, me, kPhRS, t.live[j], j == 0, j == L - 1);
      run(prev, j);
      have_prev = true;
      trace_ev(p, me, 3 + 2 * j);
    }
  }
  if (p.mode & kAG) {
    for (int jj = 0; jj < L; ++jj) {
      const int j = L + jj;
      if (!settle(j)) return;
      if (!(STREAM && (jj > 0 || (p.mode & kRS))) && !dbarrier(p, me, j, barrier_npeers(t, j), e, group_peer(j)))
        return;
      trace_ev(p, me, 2 + 2 * j);
      prev = phase_ctx(p, me, kPhAG, t.live[L - 1 - jj], false, false);
      run(prev, j);
      have_prev = true;
      trace_ev(p, me, 3 + 2 * j);
    }
  }
  const int last_phase = (p.mode & kAG) ? 2 * L - 1 : L - 1;
  if (p.mode & kCoutAll) {
    if (!settle(last_phase + 1)) return;
    __syncthreads();
    run(phase_ctx(p, me, kPhCout, 0, false, false), -1);
  }
  if (L > 0 && !p.loopback) {
    if (!(p.mode & kCoutAll) && !settle(last_phase + 1)) return;
    if (!dbarrier(p, me, 2 * L, barrier_npeers(t, 2 * L), e, group_peer(2 * L))) return;
  }
  trace_ev(p, me, 2 + 2 * (2 * L));
  rank_epoch_end(p, me, e, STEAL ? 2 * L : 0);
}

// ------------------------------------------------------------------------ rank-level, dynamic (PATH 3)
// The same schedule, with the work of a phase shared DYNAMICALLY by all CTAs of a rank
// (a ticket counter hands out chunks), and RANK-level barriers: when the last CTA of rank r
// finishes phase j it signals the ranks that gate on it (barrier j+1's group, and r itself);
// every CTA of those ranks waits for all of them before phase j+1.  Round-1 traces
// (scripts/trace_call.py) showed per-CTA static slices finishing a phase up to 10-26 us
// apart on one GPU, and every barrier waiting for the slowest CTA; dynamic chunks bound the
// spread by one chunk.  All CTAs of all ranks must be co-resident (as for PATH 0-2).
// MEASURED (round 1, loopback 8 ranks): 10-45% SLOWER than PATH 2 -- the spread is drain
// latency of the last chunks, not load imbalance, and a rank-level barrier waits for the
// slowest CTA of every member.  Kept behind DDL_DYN=1 (parity-tested), not the default.
//
// Rank state (in each rank's flag region, after the per-CTA area):
//   [0] call epoch of this rank, then arrive[j] / work[j] counters per phase j (pre-phase =
//   kPrePhase), then flags[slot][src]: src signalled slot with its epoch.
// Barrier-slot peer lists: barrier j's group (j < 2L) or every group (j = 2L), plus r itself
// (its own other CTAs wrote data this rank reads next).  Lane l < npeers+1.
__device__ __forceinline__ int rank_barrier_member(const Topo& t, int me, int slot, int l) {
  const int np = barrier_npeers(t, slot);
  return l < np ? barrier_peer(t, me, slot, l) : me;
}

// Phase j of rank me done by this CTA: arrive; the last CTA resets the phase counters and
// signals `slot` to its group + itself.
__device__ __forceinline__ void rank_arrive(const KParams& p, int me, int j, int slot, uint32_t epoch) {
  __syncthreads();  // this CTA's stores of phase j precede the release RMW below
  if (threadIdx.x == 0) {
    uint32_t* rs = rank_state(p, me);
    const uint32_t old = atom_add_acq_rel_gpu(rs_arrive(rs, j), 1);
    if (old == gridDim.x - 1) {  // last CTA of this rank: everything rank me wrote is visible to it
      *rs_arrive(rs, j) = 0;
      *rs_work(rs, j) = 0;
      if (slot >= 0) {
        const int np = barrier_npeers(p.t, slot);
        for (int l = 0; l <= np; ++l) {
          const int m = rank_barrier_member(p.t, me, slot, l);
          st_release(rs_flag(rank_state(p, m), slot, me), epoch, p.gpu_scope);
        }
      }
    }
  }
}

// Wait until every member of `slot` (group + me) has signalled it for this call.
__device__ __forceinline__ bool rank_wait(const KParams& p, int me, int slot, uint32_t epoch) {
  const int nw = barrier_npeers(p.t, slot) + 1;
  int fail = 0;
  if ((int)threadIdx.x < nw) {
    const int m = rank_barrier_member(p.t, me, slot, threadIdx.x);
    const uint32_t* f = rs_flag(rank_state(p, me), slot, m);
    uint64_t t0 = 0;
    uint32_t spins = 0;
    while ((int32_t)(ld_acquire(f, p.gpu_scope) - epoch) < 0) {
      if ((++spins & 1023u) == 0) {
        const uint64_t now = globaltimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > p.timeout_ns) {
          atomicExch(p.err, kErrTimeout);
          fail = 1;
          break;
        }
      }
    }
  }
  return __syncthreads_or(fail) == 0;
}

struct ChunkDesc {
  uint32_t unit;
  uint32_t off;    // byte offset in the unit
  uint32_t bytes;  // 0 = no more chunks for this CTA in this phase
  uint32_t last;   // this chunk ends its unit (the unit's ragged remainder goes with it)
};

// One phase with chunks handed out by the rank's ticket counter.  Units are whole blocks.
template <typename T>
__device__ void dyn_phase(const KParams& p, int me, const PhaseCtx& x, Pipe& pp, uint32_t* work) {
  using A = typename Tr<T>::Acc;
  constexpr int W = Tr<T>::W;
  __shared__ UnitDesc s_units[kMaxRanks];
  __shared__ const char* s_srcs[kMaxRanks];
  __shared__ uint32_t s_cpref[kMaxRanks + 1];
  __shared__ ChunkDesc s_desc[kStages];
  const uint32_t CB = (kStageBytes / (uint32_t)x.g) & ~15u;
  const bool do_scale = x.kind == kPhRS && x.last && p.op == kAvg;
  char* dst = dst_base(p, me, x);

  __syncthreads();  // previous phase's readers of the tables are done
  if ((int)threadIdx.x < x.nunits) {
    int sr;
    const int b = unit_block(p, me, x, threadIdx.x, &sr);
    const uint64_t e0 = (uint64_t)b * p.q;
    const uint64_t len = e0 >= p.n ? 0 : (p.q < p.n - e0 ? p.q : p.n - e0);
    const uint32_t nvec = (uint32_t)(len / W);
    s_units[threadIdx.x] = UnitDesc{e0, nvec * 16u, (uint32_t)(len - (uint64_t)nvec * W),
                                    x.kind == kPhRS ? nullptr : src_base<T>(p, me, x, 0, sr)};
  }
  if (x.kind == kPhRS && (int)threadIdx.x < x.g) s_srcs[threadIdx.x] = src_base<T>(p, me, x, threadIdx.x, me);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (int u = 0; u < x.nunits; ++u) {
      s_cpref[u] = acc;
      // a unit with only a ragged remainder still gets one (empty) chunk to carry it
      acc += s_units[u].bytes ? (s_units[u].bytes + CB - 1) / CB : (s_units[u].rem ? 1u : 0u);
    }
    s_cpref[x.nunits] = acc;
  }
  __syncthreads();
  const uint32_t total = s_cpref[x.nunits];

  // producer (thread 0): tickets -> stage descriptors + bulk loads
  uint32_t ticket = 0;
  bool done = false;
  auto fill = [&](uint32_t sq) {
    if (done) return;  // the terminator is already queued
    const int st = (int)(sq % kStages);
    ChunkDesc d{0, 0, 0, 0};
    if (ticket < total) {
      int u = 0;
      while (ticket >= s_cpref[u + 1]) ++u;
      const UnitDesc ud = s_units[u];
      d.unit = u;
      d.off = (ticket - s_cpref[u]) * CB;
      d.bytes = ud.bytes > d.off ? min(CB, ud.bytes - d.off) : 0;
      d.last = 0x80000000u | (ticket + 1 == s_cpref[u + 1] ? 1u : 0u);  // valid | ends its unit
      s_desc[st] = d;
      mbar_arm(&pp.bar[st], d.bytes * (uint32_t)x.g);
      const size_t go = ud.e0 * sizeof(T) + d.off;
      if (d.bytes) {
        char* sb = pp.smem + (size_t)st * kStageBytes;
        if (x.kind == kPhRS) {
          for (int v = 0; v < x.g; ++v) tma_load(sb + (size_t)v * CB, s_srcs[v] + go, d.bytes, &pp.bar[st]);
        } else {
          tma_load(sb, ud.src + go, d.bytes, &pp.bar[st]);
        }
      }
      ticket = atomicAdd(work, 1u);  // prefetch the next ticket
    } else {
      done = true;
      s_desc[st] = d;  // terminator (no valid bit)
      mbar_arm(&pp.bar[st], 0);
    }
  };
  if (threadIdx.x == 0) {
    fence_proxy_async_global();
    ticket = atomicAdd(work, 1u);
    for (int s = 0; s < kStages; ++s) {
      fill(pp.seq + s);
      if (done) break;
    }
  }

  for (uint32_t k = 0;; ++k) {
    const uint32_t sq = pp.seq + k;
    const int st = (int)(sq % kStages);
    mbar_wait(&pp.bar[st], (sq / kStages) & 1u);
    const ChunkDesc d = s_desc[st];
    if (!(d.last & 0x80000000u)) {  // terminator: this CTA is done with the phase
      pp.seq += k + 1;
      break;
    }
    const UnitDesc ud = s_units[d.unit];
    const char* sbase = pp.smem + (size_t)st * kStageBytes;
    char* pd = dst + ud.e0 * sizeof(T) + d.off;
    const uint32_t nv = d.bytes / 16u;
    if (x.kind == kPhRS) {
      for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
        A acc[W];
        unpack<T>(*reinterpret_cast<const uint4*>(sbase + (size_t)i * 16), acc);
        for (int v = 1; v < x.g; ++v) {
          A y[W];
          unpack<T>(*reinterpret_cast<const uint4*>(sbase + (size_t)v * CB + (size_t)i * 16), y);
#pragma unroll
          for (int q = 0; q < W; ++q) acc[q] = Tr<T>::add(acc[q], y[q]);
        }
        if (do_scale) {
#pragma unroll
          for (int q = 0; q < W; ++q) acc[q] = Tr<T>::mul(acc[q], p.scale);
        }
        st_vec(pd + (size_t)i * 16, pack<T>(acc));
      }
    } else {
      for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x)
        st_vec(pd + (size_t)i * 16, *reinterpret_cast<const uint4*>(sbase + (size_t)i * 16));
    }
    if ((d.last & 1u) && threadIdx.x < ud.rem) {  // the unit's ragged remainder, element-wise
      const size_t o = (ud.e0 + (size_t)ud.bytes / sizeof(T) + threadIdx.x) * sizeof(T);
      if (x.kind == kPhRS) {
        A a = 0;
        for (int v = 0; v < x.g; ++v) {
          const A y = Tr<T>::to(ld_elem<T>(s_srcs[v] + o));
          a = v == 0 ? y : Tr<T>::add(a, y);
        }
        if (do_scale) a = Tr<T>::mul(a, p.scale);
        st_elem<T>(dst + o, Tr<T>::from(a));
      } else {
        st_elem<T>(dst + o, ld_elem<T>(ud.src + o));
      }
    }
    __syncthreads();  // every thread is done with stage st
    if (threadIdx.x == 0) fill(sq + kStages);
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads, DDL_TMA_MINBLOCKS) ddl_dyn_kernel(const __grid_constant__ KParams p) {
  const int me = p.loopback ? (int)blockIdx.y : p.rank;
  uint32_t* rs = rank_state(p, me);
  const uint32_t e = rank_epoch_begin(p, me);
  if (me == p.skip_rank) return;
  const Topo& t = p.t;
  const int L = t.nlive;
  Pipe pp;
  pipe_init(pp);
  trace_ev(p, me, 0);
  // pre-phase: copy-in (staged paths), then "my inputs are ready" = barrier 0 (or L for AG-only)
  const int first_slot = (p.mode & kRS) ? 0 : L;
  if (p.mode & kCinAll) dyn_phase<T>(p, me, phase_ctx(p, me, kPhCin, 0, false, false), pp, rs_work(rs, kPrePhase));
  if ((p.mode & kCinOwn) && p.cin[me] != static_cast<const char*>(p.work[me]) + (size_t)me * p.q * sizeof(T))
    dyn_phase<T>(p, me, phase_ctx(p, me, kPhCinOwn, 0, false, false), pp, rs_work(rs, kPrePhase));
  rank_arrive(p, me, kPrePhase, first_slot, e);
  trace_ev(p, me, 1);
  // phases j = first_slot .. last; phase j follows barrier j, and its completion signals
  // barrier j+1 (or the end barrier 2L after the last phase)
  const int last_slot = (p.mode & kAG) ? 2 * L - 1 : L - 1;
  for (int j = first_slot; j <= last_slot; ++j) {
    if (!rank_wait(p, me, j, e)) return;
    trace_ev(p, me, 2 + 2 * j);
    const PhaseCtx x = j < L ? phase_ctx(p, me, kPhRS, t.live[j], j == 0, j == L - 1)
                             : phase_ctx(p, me, kPhAG, t.live[2 * L - 1 - j], false, false);
    dyn_phase<T>(p, me, x, pp, rs_work(rs, j));
    rank_arrive(p, me, j, j == last_slot ? 2 * L : j + 1, e);
    trace_ev(p, me, 3 + 2 * j);
  }
  if (!rank_wait(p, me, 2 * L, e)) return;
  if (p.mode & kCoutAll) {
    dyn_phase<T>(p, me, phase_ctx(p, me, kPhCout, 0, false, false), pp, rs_work(rs, kPostPhase));
    rank_arrive(p, me, kPostPhase, -1, e);
  }
  trace_ev(p, me, 2 + 2 * (2 * L));
  rank_epoch_end(p, me, e, 0);
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

  if (p.mode & kCinAll) {  // staged: publish this CTA's slice of my input
    const char* s = static_cast<const char*>(p.cin[me]);
    char* w = static_cast<char*>(p.work[me]);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint64_t eo = lo + ((uint64_t)i * blockDim.x + threadIdx.x) * W;
      if (eo + W <= hi) st_vec(w + eo * sizeof(T), ld_vec(s + eo * sizeof(T)));
      else
        for (uint64_t x = eo; x < hi; ++x) st_elem<T>(w + x * sizeof(T), ld_elem<T>(s + x * sizeof(T)));
    }
  }
  // loopback without copy-in: inputs are ready at launch (see ddl_hier_kernel)
  if (!(p.loopback && !(p.mode & kCinAll)) && !dbarrier(p, me, 0, P - 1, e, all)) return;

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
          raw[k] = ld_vec(static_cast<const char*>(p.in[r0 + k]) + eoff * sizeof(T));
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
          A x[1] = {Tr<T>::to(ld_elem<T>(static_cast<const char*>(p.in[r]) + (eoff + k) * sizeof(T)))};
          nested_feed<T, K, 1>(p, gl, Gl, r, lvl1, x, r1);
        }
        res[i][k] = r1[0];
      }
    }
  }
  if (!dbarrier(p, me, 1, P - 1, e, all)) return;
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

// ------------------------------------------------------------------------ K5 local reduce
// out = s * sum_{j<g} in_j, ascending j.  Grid-stride over 16-byte vectors, up to 8 input
// loads in flight per thread, streaming cache hints (every byte is touched once).
template <typename T, bool VEC>
__global__ void __launch_bounds__(kThreads, 2) ddl_local_reduce_kernel(const __grid_constant__ LRParams p) {
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

}  // namespace ddl
