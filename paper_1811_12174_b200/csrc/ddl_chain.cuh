// ddl_chain.cuh -- the loopback column-chain kernels (round 2).
//
// Loopback runs all P virtual ranks in ONE GPU's HBM.  Every phase of the hierarchical schedule
// (a4 RS, a5 epilogue, a6 AG) is elementwise across ranks at a fixed element offset: the values
// rank r holds at offset e after any phase depend only on the P ranks' values at offset e.  So
// the schedule factorises into independent COLUMNS -- one 16-byte vector offset of a block,
// across the P virtual ranks' buffers -- and one thread can run the whole schedule for its
// column, phase after phase, with every load and store the schedule makes:
//
//   RS phase d (live dims ascending): every writer r (b in A_{d+1}(r)) folds its g_d group
//     members' values in ascending coordinate (inputs in the first live phase, the previous
//     phase's partials after it) and stores the result into its own buffer; the last RS phase
//     fuses the fl32(1/P) multiply (avg) and the I/O cast (K3).
//   AG phase d (live dims descending): every rank r with b in A_d(r) \ A_{d+1}(r) loads the
//     block's copy held by its group-d member with coordinate beta_d(b) and stores it.
//
// The phase order of a column is the schedule's; a phase's sources are the previous phase's
// stores made by the SAME thread (program order on the same addresses), so the 2L+1 device
// barriers of the per-CTA slice kernels (a7) are not needed when the whole slice chain is one
// thread -- and neither is the drift between CTAs that the barriers expose.
// The fold order, rounding points and bytes touched are exactly those of the slice kernels, so
// results are bit-identical to them and to the oracle (tests/test_gpu_chain.py).
//
// Why: the slice kernels move a bucket's partials through HBM-sized phases, so
// the partials of a whole bucket are live at once (more than L2 keeps) and every phase ends in
// a barrier; here a column's partials live for a few microseconds, are re-read from L1 / L2 and
// overwritten there before they are ever written back: DRAM sees each virtual rank's input
// read once and its result written once (the compulsory 2*P*S).
//
// Three kernels:
//   ddl_chain_tma_kernel  (default for P = 4/8; compile-time topology, P = 2/4/8) a producer warp
//       bulk-copies (TMA, cp.async.bulk) the first RS phase's sources of a tile -- kTmaCons
//       consecutive columns of one block -- into a shared-memory ring; the consumer threads fold
//       from it and run the later phases with LDG / STG.  The HBM reads in flight cost no
//       registers and no L1 miss slots (profiles/r02_ab/r02_chain14-17.txt: 0.256 vs 0.296 ms).
//   ddl_chain_ct_kernel   (default for P = 2, DDL_CHAIN_TMA=0 everywhere) the same with the
//       first-phase loads as LDG.
//   ddl_chain_kernel      (any P <= 16, DDL_CHAIN_GENERIC=1 everywhere) runtime topology, one
//       column per thread.
// Columns of several buffers (the grouped all-reduce of DDP buckets) are concatenated and
// walked by a persistent grid; every column is the same work, so the load is balanced.
#pragma once
#include "ddl_device.cuh"

namespace ddl {

// Cache policy per access class (0 ld.global.cg, 1 .cs, 2 .ca), measured in
// profiles/r02_ab/r02_chain*.txt: the first RS phase's loads (HBM) .cg, the later phases'
// re-reads of the column's own partials / finals .ca (L1 hits: the thread stored them a few
// instructions earlier), final stores default (DDL_CHAIN_FINCS=1: .cs).
// Why .ca is safe although L1 is not coherent across SMs: a re-read only ever targets bytes
// the same thread stored earlier in this launch (every column belongs to exactly one thread),
// and a thread's own stores are visible to its later loads through its SM's L1 (write-
// through); bytes of other columns that share the 128-B line may be stale in this L1, but no
// thread of this SM ever reads them, and L1 is invalidated at every launch.
#ifndef DDL_CHAIN_FIRST
#define DDL_CHAIN_FIRST 0
#endif
#ifndef DDL_CHAIN_REREAD
#define DDL_CHAIN_REREAD 2
#endif
#ifndef DDL_CHAIN_FINCS
#define DDL_CHAIN_FINCS 0
#endif
#ifndef DDL_CHAIN_MINB  // resident 256-thread CTAs per SM: generic kernel
#define DDL_CHAIN_MINB 2
#endif
#ifndef DDL_CHAIN_CT_MINB  // ... and the LDG compile-time-topology kernel (64 registers)
#define DDL_CHAIN_CT_MINB 4
#endif
#ifndef DDL_CHAIN_TMA_DEFAULT  // loopback default: the TMA-fed kernel (1), the LDG one (0), or -1 = TMA from P = 4
#define DDL_CHAIN_TMA_DEFAULT -1
#endif
#ifndef DDL_CHAIN_TMA_CONS  // TMA-fed kernel: consumer threads = columns per tile
#define DDL_CHAIN_TMA_CONS 320
#endif
#ifndef DDL_CHAIN_TMA_STAGES  // ... and ring stages (2 x 8 ranks x 320 x 16 B = 80 KB)
#define DDL_CHAIN_TMA_STAGES 2
#endif
#ifndef DDL_CHAIN_TMA_MINB  // ... and resident CTAs per SM the register budget is sized for (2: slower, r02_chain18)
#define DDL_CHAIN_TMA_MINB 1
#endif
constexpr int kChainThreads = 256;
constexpr int kTmaCons = DDL_CHAIN_TMA_CONS;
constexpr int kTmaStages = DDL_CHAIN_TMA_STAGES;
static_assert(kTmaCons % 32 == 0 && kTmaCons + 32 <= 1024, "consumer warps + one producer warp");

struct CBucket {
  uint64_t n;            // elements
  uint64_t q;            // block elements (a multiple of the 16-byte vector width)
  uint32_t vq;           // vectors per block, q / W
  uint32_t vfull;        // CT kernels: rows (vector offset v of all P blocks) whose P columns are
                         // whole vectors -- all but at most ~P rows of a buffer
  uint32_t col0;         // first column of this buffer in the launch's column space (generic
                         // kernel: all P * vq columns; CT kernels: the P * (vq - vfull) tail columns)
  uint32_t row0;         // CT kernels: first of its vfull full rows in the row space
  char* buf[kMaxRanks];  // every virtual rank's copy
};
struct CParams {
  Topo t;
  int op;
  float scale;  // fl32(1/P) for avg
  int nb;
  uint32_t ncols;
  uint32_t nrows;
  CBucket b[kMaxBuckets];
};

// 16-byte vector or single element ("lane") of a column
template <typename T, bool VEC>
struct ColIO;
template <typename T>
struct ColIO<T, true> {
  using R = uint4;
  static constexpr int N = Tr<T>::W;
  __device__ static R ld(const char* a, int how) {  // how: 0 .cg, 1 .cs, 2 .ca
    R v;
    if (how == 1)
      asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a));
    else if (how == 2)
      asm volatile("ld.global.ca.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a));
    else
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a));
    return v;
  }
  __device__ static void st(char* a, const R& v, bool stream) {
    if (stream)
      asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    else
      asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  }
  __device__ static void unpack_(const R& r, typename Tr<T>::Acc* a) { unpack<T>(r, a); }
  __device__ static R pack_(const typename Tr<T>::Acc* a) { return pack<T>(a); }
};
template <typename T>
struct ColIO<T, false> {
  using R = uint32_t;
  static constexpr int N = 1;
  __device__ static R ld(const char* a, int how) {
    uint32_t v;
    if constexpr (sizeof(T) == 2) {
      unsigned short h;
      if (how == 2) asm volatile("ld.global.ca.u16 %0, [%1];" : "=h"(h) : "l"(a));
      else asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(h) : "l"(a));
      v = h;
    } else {
      if (how == 2) asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(a));
      else asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(a));
    }
    return v;
  }
  __device__ static void st(char* a, const R& v, bool) {
    if constexpr (sizeof(T) == 2) asm volatile("st.global.u16 [%0], %1;" ::"l"(a), "h"((unsigned short)v) : "memory");
    else asm volatile("st.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
  }
  __device__ static void unpack_(const R& r, typename Tr<T>::Acc* a) { a[0] = Tr<T>::to(r); }
  __device__ static R pack_(const typename Tr<T>::Acc* a) { return Tr<T>::from(a[0]); }
};

// ------------------------------------------------------------------------ generic kernel
// The whole schedule for one column: block b, byte offset off (the same in every rank's buffer).
// MP >= P: compile-time bound of the register arrays (all indices compile-time after unrolling).
// Loads are asm volatile: never merged with or forwarded from the thread's own earlier stores,
// so every re-read of the schedule is executed.
template <typename T, bool VEC, int MP>
__device__ __forceinline__ void chain_column(const CParams& p, char* const* buf, uint32_t b, size_t off) {
  using IO = ColIO<T, VEC>;
  using A = typename Tr<T>::Acc;
  constexpr int N = IO::N;
  const Topo& t = p.t;
  const int P = t.P;
  const int L = t.nlive;
  // ---- reduce-scatter phases (a4), live dims ascending; the last fuses the epilogue (a5)
  for (int li = 0; li < L; ++li) {
    const int d = t.live[li];
    const int g = t.g[d], Gd = t.G[d], Gd1 = t.G[d + 1];
    const int sb = (int)(b % (uint32_t)Gd);   // holders of column b before phase d: sb + i*Gd
    const int wb = (int)(b % (uint32_t)Gd1);  // writers after it: wb + j*Gd1 (coordinate beta_d(b))
    const int nsrc = P / Gd;
    const bool last = li == L - 1;
    typename IO::R raw[MP];
#pragma unroll
    for (int i = 0; i < MP; ++i)
      if (i < nsrc) raw[i] = IO::ld(buf[sb + i * Gd] + off, li == 0 ? DDL_CHAIN_FIRST : DDL_CHAIN_REREAD);
    // source i = v + j*g is member v (ascending coordinate) of writer j's group
    A acc[N];
    int v = 0, j = 0;
#pragma unroll
    for (int i = 0; i < MP; ++i) {
      if (i < nsrc) {
        A y[N];
        IO::unpack_(raw[i], y);
#pragma unroll
        for (int k = 0; k < N; ++k) acc[k] = v == 0 ? y[k] : Tr<T>::add(acc[k], y[k]);
        if (++v == g) {
          if (last && p.op == kAvg && DDL_MUTATE != 8) {  // mutation 8: generic kernel drops the 1/P scale
#pragma unroll
            for (int k = 0; k < N; ++k) acc[k] = Tr<T>::mul(acc[k], p.scale);
          }
          IO::st(buf[wb + j * Gd1] + off, IO::pack_(acc), last && DDL_CHAIN_FINCS);
          v = 0;
          ++j;
        }
      }
    }
  }
  // ---- allgather phases (a6), live dims descending: receivers of phase d load the copy of
  // the member of their group-d with coordinate beta_d(b) (it holds the block), then store it
  for (int li = L - 1; li >= 0; --li) {
    const int d = t.live[li];
    const int g = t.g[d], Gd = t.G[d];
    const int sb = (int)(b % (uint32_t)Gd);
    const int beta = (int)((b / (uint32_t)Gd) % (uint32_t)g);
    const int n = P / Gd;  // ranks with b in A_d: sb + (v + j*g)*Gd; holders are those with v == beta
    typename IO::R raw[MP];
#pragma unroll
    for (int i = 0; i < MP; ++i)
      if (i < n && i % g != beta) raw[i] = IO::ld(buf[sb + (i - i % g + beta) * Gd] + off, DDL_CHAIN_REREAD);
#pragma unroll
    for (int i = 0; i < MP; ++i)
      if (i < n && i % g != beta) IO::st(buf[sb + i * Gd] + off, raw[i], DDL_CHAIN_FINCS);
  }
}

// every rank pointer of every buffer of the launch, for dynamic indexing
struct ChainSmem {
  char* buf[kMaxBuckets][kMaxRanks];
};
__device__ __forceinline__ void load_ptrs(const CParams& p, ChainSmem& s) {
  for (int i = threadIdx.x; i < p.nb * kMaxRanks; i += blockDim.x)
    s.buf[i / kMaxRanks][i % kMaxRanks] = p.b[i / kMaxRanks].buf[i % kMaxRanks];
}

template <typename T, int MP>
__global__ void __launch_bounds__(kChainThreads, DDL_CHAIN_MINB) ddl_chain_kernel(const __grid_constant__ CParams p) {
  __shared__ ChainSmem s;
  load_ptrs(p, s);
  __syncthreads();
  pdl_begin();
  constexpr int W = Tr<T>::W;
  const uint32_t stride = gridDim.x * blockDim.x;
  int k = 0;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < p.ncols; c += stride) {
    while (k + 1 < p.nb && c >= p.b[k + 1].col0) ++k;  // a thread's columns only increase
    const CBucket& B = p.b[k];
    const uint32_t lc = c - B.col0;
    const uint32_t b = lc / B.vq;
    const uint64_t e0 = (uint64_t)b * B.q + (uint64_t)(lc - b * B.vq) * W;
    if (e0 >= B.n) continue;  // past the end of a ragged last block
    if (e0 + W <= B.n) {
      chain_column<T, true, MP>(p, s.buf[k], b, e0 * sizeof(T));
    } else {
      for (uint64_t e = e0; e < B.n; ++e) chain_column<T, false, MP>(p, s.buf[k], b, e * sizeof(T));
    }
  }
}

// ------------------------------------------------------------------------ compile-time topologies
// The same schedule with the live dims as template parameters and the block b of a column a
// compile-time constant: every rank index, group member and fold position is then a constant,
// and a thread's work per column is its loads, adds and stores (the generic kernel spends most
// of its instructions on the index arithmetic: 0.47 vs 0.30 ms per bench step).
template <int L_, int g0, int g1 = 1, int g2 = 1, int g3 = 1>
struct CT {
  static constexpr int L = L_;
  __host__ __device__ static constexpr int g(int l) { return l == 0 ? g0 : l == 1 ? g1 : l == 2 ? g2 : g3; }
  __host__ __device__ static constexpr int G(int l) { return l == 0 ? 1 : G(l - 1) * g(l - 1); }  // G of live dim l
  static constexpr int P = G(L_);
};
template <int V>
struct IC {
  static constexpr int value = V;
};
template <int I, int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(IC<I>{});
    static_for<I + 1, N>(f);
  }
}

// The column of block B at byte offset off in every rank's buffer (base[r] + off).
template <typename T, class TP, int B>
struct CTCol {
  using IO = ColIO<T, true>;
  using A = typename Tr<T>::Acc;
  using Raw = typename IO::R;
  static constexpr int N = IO::N;
  static constexpr int P = TP::P;

  // RS phase li: load the P / G_li holders of the column, then every writer folds its g members
  template <int li>
  __device__ __forceinline__ static void rs_load(char* const* base, size_t off, Raw* raw) {
    constexpr int Gd = TP::G(li);
    constexpr int sb = B % Gd;
#pragma unroll
    for (int i = 0; i < P / Gd; ++i)
      raw[i] = IO::ld(base[sb + i * Gd] + off, li == 0 ? DDL_CHAIN_FIRST : DDL_CHAIN_REREAD);
  }
  template <int li>
  __device__ __forceinline__ static void rs_fold(const CParams& p, char* const* base, size_t off, const Raw* raw) {
    constexpr int g = TP::g(li), Gd1 = TP::G(li + 1);
    constexpr int wb = B % Gd1;
    constexpr bool last = li == TP::L - 1;
#pragma unroll
    for (int j = 0; j < P / Gd1; ++j) {  // writer wb + j*Gd1 folds members v = 0..g-1 (source v + j*g)
      A acc[N];
#if DDL_MUTATE == 4  // mutation check (scripts/gpu_mutation_check.sh): members folded in descending order
      IO::unpack_(raw[j * g + g - 1], acc);
#pragma unroll
      for (int v = g - 2; v >= 0; --v) {
#else
      IO::unpack_(raw[j * g], acc);
#pragma unroll
      for (int v = 1; v < g; ++v) {
#endif
        A y[N];
        IO::unpack_(raw[j * g + v], y);
#pragma unroll
        for (int k = 0; k < N; ++k) acc[k] = Tr<T>::add(acc[k], y[k]);
      }
      if (last && p.op == kAvg && DDL_MUTATE != 5) {  // mutation 5: the fused 1/P scale dropped
#pragma unroll
        for (int k = 0; k < N; ++k) acc[k] = Tr<T>::mul(acc[k], p.scale);
      }
      IO::st(base[wb + j * Gd1] + off, IO::pack_(acc), last && DDL_CHAIN_FINCS);
    }
  }
  // AG phase li: every receiver loads the holder's copy, then all of them store
  template <int li>
  __device__ __forceinline__ static void ag(char* const* base, size_t off) {
    constexpr int g = TP::g(li), Gd = TP::G(li);
    constexpr int sb = B % Gd, beta = (B / Gd) % g, n = P / Gd;
    Raw raw[n];
#pragma unroll
    for (int i = 0; i < n; ++i)
      if (i % g != beta) raw[i] = IO::ld(base[sb + (i - i % g + beta) * Gd] + off, DDL_CHAIN_REREAD);
#pragma unroll
    for (int i = 0; i < n; ++i)
      if (i % g != beta && !(DDL_MUTATE == 6 && li == 0 && i == n - 1 - (beta == n - 1)))  // mutation 6: a receiver skipped
        IO::st(base[sb + i * Gd] + off, raw[i], DDL_CHAIN_FINCS);
  }
  // every phase after the first RS phase's fold
  __device__ __forceinline__ static void after_first(const CParams& p, char* const* base, size_t off) {
    static_for<1, TP::L>([&](auto lc) {
      constexpr int li = decltype(lc)::value;
      Raw raw[P / TP::G(li)];
      rs_load<li>(base, off, raw);
      rs_fold<li>(p, base, off, raw);
    });
    static_for<0, TP::L>([&](auto lc) { ag<TP::L - 1 - decltype(lc)::value>(base, off); });
  }
  __device__ __forceinline__ static void run(const CParams& p, char* const* base, size_t off) {
    Raw raw[P];
    rs_load<0>(base, off, raw);
    rs_fold<0>(p, base, off, raw);
    after_first(p, base, off);
  }
};

// one column of the CT kernels' tail rows (whole vector or ragged), out of line: rare, and it
// keeps the generic code's registers out of the hot loop
template <typename T, int MP>
__device__ __noinline__ void chain_cold(const CParams& p, char* const* base, uint32_t b, uint64_t e0, uint64_t n) {
  if (e0 + Tr<T>::W <= n) chain_column<T, true, MP>(p, base, b, e0 * sizeof(T));
  else for (uint64_t e = e0; e < n; ++e) chain_column<T, false, MP>(p, base, b, e * sizeof(T));
}

// The rows vfull .. vq-1 of every buffer (the ragged last block, blocks past n), one column
// (b, v) per step of nthreads threads numbered tid.
template <typename T, int P>
__device__ __forceinline__ void chain_tail_rows(const CParams& p, const ChainSmem& s, uint32_t tid, uint32_t nthreads) {
  constexpr int W = Tr<T>::W;
  int k = 0;
  for (uint32_t c = tid; c < p.ncols; c += nthreads) {
    while (k + 1 < p.nb && c >= p.b[k + 1].col0) ++k;
    const CBucket& Bk = p.b[k];
    const uint32_t tail_rows = Bk.vq - Bk.vfull;
    const uint32_t lc = c - Bk.col0;
    const uint32_t b = lc / tail_rows;
    const uint64_t e0 = (uint64_t)b * Bk.q + (uint64_t)(Bk.vfull + (lc - b * tail_rows)) * W;
    if (e0 < Bk.n) chain_cold<T, P>(p, s.buf[k], b, e0, Bk.n);
  }
}

// LDG kernel (DDL_CHAIN_TMA=0): the grid walks block 0's column of every full row, then block
// 1's, ... (block-major), then the tail rows.
template <typename T, class TP>
__global__ void __launch_bounds__(kChainThreads, DDL_CHAIN_CT_MINB) ddl_chain_ct_kernel(const __grid_constant__ CParams p) {
  __shared__ ChainSmem s;
  load_ptrs(p, s);
  __syncthreads();
  pdl_begin();
  constexpr int P = TP::P;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  static_for<0, P>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    int k = 0;
    for (uint32_t v = tid; v < p.nrows; v += stride) {
      while (k + 1 < p.nb && v >= p.b[k + 1].row0) ++k;
      const uint64_t qb = p.b[k].q * sizeof(T);
      CTCol<T, TP, b>::run(p, s.buf[k], (uint64_t)(v - p.b[k].row0) * 16u + b * qb);
    }
  });
  chain_tail_rows<T, P>(p, s, tid, stride);
}

// ------------------------------------------------------------------------ TMA-fed column chain
// Tile = kTmaCons consecutive full rows of one block b of one buffer (block-major order).  A
// producer warp bulk-copies the P ranks' segments of each tile (the first RS phase's sources)
// into a kTmaStages-deep shared-memory ring (mbarrier expect-tx per stage); consumer thread i
// takes column i of the tile from the ring, folds and stores it (RS phase 0), releases the
// stage (one arrival per warp on its empty barrier) and runs the later phases with LDG / STG.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// ring stages for P ranks: kTmaStages at P = 8, more for smaller P so that the ring (the bytes
// in flight per CTA) stays at kTmaStages x 8 x kTmaCons x 16 B
__host__ __device__ constexpr int chain_tma_stages(int P) { return P >= 8 ? kTmaStages : kTmaStages * (8 / P); }
inline size_t chain_tma_smem(int P) {
  return (size_t)chain_tma_stages(P) * P * kTmaCons * 16 + 2 * chain_tma_stages(P) * sizeof(uint64_t);
}

template <typename T, class TP>
__global__ void __launch_bounds__(kTmaCons + 32, DDL_CHAIN_TMA_MINB) ddl_chain_tma_kernel(const __grid_constant__ CParams p) {
  constexpr int P = TP::P;
  constexpr int S = chain_tma_stages(P);
  constexpr uint32_t SEG = kTmaCons * 16;  // bytes of one rank's segment of a tile
  using Raw = typename ColIO<T, true>::R;
  extern __shared__ __align__(128) char dsm[];
  char* ring = dsm;  // [stage][rank][SEG]
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + (size_t)S * P * SEG);
  uint64_t* empty = full + S;
  __shared__ ChainSmem s;
  __shared__ uint32_t s_ch0[kMaxBuckets + 1];  // first chunk (kTmaCons full rows) of each buffer
  load_ptrs(p, s);
  if (threadIdx.x == 0) {
    uint32_t c = 0;
    for (int k = 0; k < p.nb; ++k) {
      s_ch0[k] = c;
      c += (p.b[k].vfull + kTmaCons - 1) / kTmaCons;
    }
    s_ch0[p.nb] = c;
    for (int st = 0; st < S; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kTmaCons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_begin();
  const uint32_t C = s_ch0[p.nb];
  const uint32_t ntiles = (uint32_t)P * C;
  // tile t: block b = t / C, chunk t % C -> buffer k, rows [r0, r0 + rn)
  auto tile_of = [&](uint32_t t, int& b, int& k, uint32_t& r0, uint32_t& rn) {
    b = (int)(t / C);
    const uint32_t ci = t - (uint32_t)b * C;
    k = 0;
    while (k + 1 < p.nb && ci >= s_ch0[k + 1]) ++k;
    r0 = (ci - s_ch0[k]) * kTmaCons;
    rn = min((uint32_t)kTmaCons, p.b[k].vfull - r0);
  };
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == kTmaCons / 32) {  // producer warp
    if (lane == 0) {
      uint32_t i = 0;
      for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int st = (int)(i % S);
        if (i >= (uint32_t)S) mbar_wait(&empty[st], ((i / S) - 1) & 1u);
        int b, k;
        uint32_t r0, rn;
        tile_of(t, b, k, r0, rn);
        const uint64_t qb = p.b[k].q * sizeof(T);
        mbar_arm(&full[st], (uint32_t)P * rn * 16u);
#pragma unroll
        for (int r = 0; r < P; ++r)
          tma_load(ring + ((size_t)st * P + r) * SEG, s.buf[k][r] + (uint64_t)b * qb + (uint64_t)r0 * 16u, rn * 16u,
                   &full[st]);
      }
    }
    return;
  }
  uint32_t i = 0;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
    const int st = (int)(i % S);
    int b, k;
    uint32_t r0, rn;
    tile_of(t, b, k, r0, rn);
    const uint64_t qb = p.b[k].q * sizeof(T);
    const bool mine = (uint32_t)threadIdx.x < rn;
    const uint64_t off = (uint64_t)b * qb + (uint64_t)(r0 + threadIdx.x) * 16u;
    mbar_wait(&full[st], (i / S) & 1u);
    static_for<0, P>([&](auto bc) {  // b is uniform over the CTA: one branch taken
      constexpr int B = decltype(bc)::value;
      if (b != B) return;
      using Cl = CTCol<T, TP, B>;
      if (mine) {
        Raw raw[P];
#pragma unroll
        for (int r = 0; r < P; ++r)  // (mutation 7: two ranks' segments swapped)
          raw[r] = reinterpret_cast<const Raw*>(ring + ((size_t)st * P + (DDL_MUTATE == 7 && (r == 1 || r == 2) ? 3 - r : r)) * SEG)[threadIdx.x];
        Cl::template rs_fold<0>(p, s.buf[k], off, raw);  // consumes raw: the stage is free
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (mine) Cl::after_first(p, s.buf[k], off);
    });
  }
  chain_tail_rows<T, P>(p, s, blockIdx.x * kTmaCons + threadIdx.x, gridDim.x * kTmaCons);
}

}  // namespace ddl
