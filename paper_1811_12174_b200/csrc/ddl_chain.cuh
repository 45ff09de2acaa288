// ddl_chain.cuh -- the loopback column-chain kernel (round 2).
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
// Why: the slice kernels move a column's partials through HBM-sized phases,
// so the partials of a whole bucket are live at once (more than L2 keeps) and every phase ends
// in a barrier; here a column's partials live for a few microseconds, so they are re-read from
// L1/L2 and overwritten there before they are ever written back: DRAM sees each virtual rank's
// input read once and its result written once (the compulsory 2*P*S).
//
// Columns of several buffers (the grouped all-reduce of DDP buckets) are concatenated into one
// column space and walked grid-stride by a persistent grid; every column is the same work, so
// the load is balanced without any scheduling.
#pragma once
#include "ddl_device.cuh"

namespace ddl {

#ifndef DDL_CHAIN_MINB
#define DDL_CHAIN_MINB 2
#endif
// CT kernels' cache policy per access class (0 ld.global.cg, 1 .cs, 2 .ca): the first RS phase's
// loads (HBM), the later phases' re-reads of the column's own partials / finals; final stores .cs
#ifndef DDL_CHAIN_FIRST
#define DDL_CHAIN_FIRST 0
#endif
#ifndef DDL_CHAIN_REREAD
#define DDL_CHAIN_REREAD 2
#endif
#ifndef DDL_CHAIN_FINCS
#define DDL_CHAIN_FINCS 0
#endif
#ifndef DDL_CHAIN_NB  // columns per thread in lockstep (divides P)
#define DDL_CHAIN_NB 1
#endif
#ifndef DDL_CHAIN_CT_MINB
#define DDL_CHAIN_CT_MINB 4
#endif
#ifndef DDL_CHAIN_VPT  // adjacent vectors per thread (the CT kernels' full rows are cut into groups of VPT)
#define DDL_CHAIN_VPT 1
#endif
constexpr int kChainVPT = DDL_CHAIN_VPT;
#ifndef DDL_CHAIN_PF  // BMAJOR loop: L2 prefetch of the first-phase sources this many grid strides ahead (0 off)
#define DDL_CHAIN_PF 0
#endif
#ifndef DDL_CHAIN_PF_BULK
#define DDL_CHAIN_PF_BULK 0
#endif
#ifndef DDL_CHAIN_SPLIT
#define DDL_CHAIN_SPLIT 0
#endif
#ifndef DDL_CHAIN_FLAT
#define DDL_CHAIN_FLAT 0
#endif
#ifndef DDL_CHAIN_BMAJOR
#define DDL_CHAIN_BMAJOR 1
#endif
#ifndef DDL_CHAIN_ASYNC  // CT kernels: the next column's first-phase loads staged by cp.async
#define DDL_CHAIN_ASYNC 0
#endif
constexpr int kChainThreads = 256;

struct CBucket {
  uint64_t n;            // elements
  uint64_t q;            // block elements (a multiple of the 16-byte vector width)
  uint32_t vq;           // vectors per block, q / W
  uint32_t col0;         // first column of this buffer in the launch's column space (generic kernel;
                         // CT kernels: of its P * (vq - vfull) tail columns)
  uint32_t row0;         // CT kernels: first of its vfull full rows (vector offset v of all P blocks)
  uint32_t vfull;        // CT kernels: rows whose P columns are all whole vectors
  char* buf[kMaxRanks];  // every virtual rank's copy
};
struct CParams {
  Topo t;
  int op;
  float scale;  // fl32(1/P) for avg
  int nb;
  uint32_t ncols;
  uint32_t nrows;
  int hint;     // cache policy bits (DDL_CHAIN_HINTS): 1 first-phase loads streaming (.cs, else .cg),
                // 2 re-reads through L1 (.ca, else .cg), 4 final stores streaming (.cs)
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

// The whole schedule for one column: block b, byte offset off (the same in every rank's buffer).
// MP >= P: compile-time bound of the register arrays (all indices compile-time after unrolling).
template <typename T, bool VEC, int MP>
__device__ __forceinline__ void chain_column(const CParams& p, char* const* buf, uint32_t b, size_t off) {
  using IO = ColIO<T, VEC>;
  using A = typename Tr<T>::Acc;
  constexpr int N = IO::N;
  const Topo& t = p.t;
  const int P = t.P;
  const int L = t.nlive;
  const int reread = (p.hint & 2) ? 2 : 0;
  // ---- reduce-scatter phases (a4), live dims ascending; the last fuses the epilogue (a5)
  for (int li = 0; li < L; ++li) {
    const int d = t.live[li];
    const int g = t.g[d], Gd = t.G[d], Gd1 = t.G[d + 1];
    const int sb = (int)(b % (uint32_t)Gd);   // holders of column b before phase d: sb + i*Gd
    const int wb = (int)(b % (uint32_t)Gd1);  // writers after it: wb + j*Gd1 (coordinate beta_d(b))
    const int nsrc = P / Gd;
    const bool last = li == L - 1;
    const int how = li == 0 ? ((p.hint & 1) ? 1 : 0) : reread;
    typename IO::R raw[MP];
#pragma unroll
    for (int i = 0; i < MP; ++i)
      if (i < nsrc) raw[i] = IO::ld(buf[sb + i * Gd] + off, how);
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
          if (last && p.op == kAvg) {
#pragma unroll
            for (int k = 0; k < N; ++k) acc[k] = Tr<T>::mul(acc[k], p.scale);
          }
          IO::st(buf[wb + j * Gd1] + off, IO::pack_(acc), last && (p.hint & 4));
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
    const int g = t.g[d], Gd = t.G[d], Gd1 = t.G[d + 1];
    const int sb = (int)(b % (uint32_t)Gd);
    const int beta = (int)((b / (uint32_t)Gd) % (uint32_t)g);
    const int n = P / Gd;  // ranks with b in A_d: sb + (v + j*g)*Gd; holders are those with v == beta
    typename IO::R raw[MP];
#pragma unroll
    for (int i = 0; i < MP; ++i)
      if (i < n && i % g != beta) raw[i] = IO::ld(buf[sb + (i - i % g + beta) * Gd] + off, reread);
#pragma unroll
    for (int i = 0; i < MP; ++i)
      if (i < n && i % g != beta) IO::st(buf[sb + i * Gd] + off, raw[i], (p.hint & 4) != 0);
  }
}

template <typename T, int MP>
__global__ void __launch_bounds__(kChainThreads, DDL_CHAIN_MINB) ddl_chain_kernel(const __grid_constant__ CParams p) {
  __shared__ char* s_buf[kMaxBuckets][kMaxRanks];  // every buffer's rank pointers (dynamic index)
  for (int i = threadIdx.x; i < p.nb * kMaxRanks; i += blockDim.x) s_buf[i / kMaxRanks][i % kMaxRanks] = p.b[i / kMaxRanks].buf[i % kMaxRanks];
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
      chain_column<T, true, MP>(p, s_buf[k], b, e0 * sizeof(T));
    } else {
      for (uint64_t e = e0; e < B.n; ++e) chain_column<T, false, MP>(p, s_buf[k], b, e * sizeof(T));
    }
  }
}

// ------------------------------------------------------------------------ compile-time topologies
// The same schedule with the live dims as template parameters and the block b of a column a
// compile-time constant: every rank index, group member and fold position is then a constant,
// and a thread's work per column is its loads, adds and stores (the generic kernel above spends
// most of its instructions on the index arithmetic).  One thread handles row v: column v of
// every block b = 0..P-1 (its P columns are independent; each runs the whole schedule).
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

// Column of block B at byte offset off in every rank's buffer (base[r] + off), in two parts so
// that a thread can issue the next column's first-phase loads (its HBM reads) before this
// column's later phases (L2 round trips): ct_first loads the first RS phase's sources, ct_rest
// folds and stores them and runs every later phase.
// Columns of blocks B0 .. B0+NB-1 of one row (byte offsets off + j*qb, j < NB, in every rank's
// buffer base[r]), run in lockstep: each phase issues the loads of all NB columns before any of
// their folds / stores, so a thread has NB independent chains in flight (NB x the memory-level
// parallelism of one column, at NB x the registers).
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}

template <typename T, class TP, int B0, int NB, bool ADJ = false>
struct CTCols {
  using IO = ColIO<T, true>;
  using A = typename Tr<T>::Acc;
  using Raw = typename IO::R;
  static constexpr int N = IO::N;
  static constexpr int P = TP::P;
  // lockstep column c: block B0 + c at off + c*qb, or (ADJ) block B0 at the c-th adjacent vector
  __device__ __forceinline__ static constexpr int blk(int c) { return ADJ ? B0 : B0 + c; }
  __device__ __forceinline__ static uint64_t cst(int c, uint64_t qb) { return ADJ ? (uint64_t)c * 16u : c * qb; }

  template <int li>
  using RawPh = Raw[NB][P / TP::G(li)];  // sources of RS phase li: the P / G_li holders of the column

  template <int li>
  __device__ __forceinline__ static void rs_load(char* const* base, size_t off, uint64_t qb, RawPh<li>& raw) {
    constexpr int Gd = TP::G(li);
    constexpr int nsrc = P / Gd;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      const int sb = blk(c) % Gd;  // (constant after unrolling)
#pragma unroll
      for (int i = 0; i < nsrc; ++i)
        raw[c][i] = IO::ld(base[sb + i * Gd] + off + cst(c, qb), li == 0 ? DDL_CHAIN_FIRST : DDL_CHAIN_REREAD);
    }
  }

  template <int li>
  __device__ __forceinline__ static void rs_fold(const CParams& p, char* const* base, size_t off, uint64_t qb,
                                                 const RawPh<li>& raw) {
    constexpr int g = TP::g(li), Gd1 = TP::G(li + 1);
    constexpr bool last = li == TP::L - 1;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      const int wb = blk(c) % Gd1;
#pragma unroll
      for (int j = 0; j < P / Gd1; ++j) {  // writer wb + j*Gd1 folds members v = 0..g-1 (source v + j*g)
        A acc[N];
        IO::unpack_(raw[c][j * g], acc);
#pragma unroll
        for (int v = 1; v < g; ++v) {
          A y[N];
          IO::unpack_(raw[c][j * g + v], y);
#pragma unroll
          for (int k = 0; k < N; ++k) acc[k] = Tr<T>::add(acc[k], y[k]);
        }
        if (last && p.op == kAvg) {
#pragma unroll
          for (int k = 0; k < N; ++k) acc[k] = Tr<T>::mul(acc[k], p.scale);
        }
        IO::st(base[wb + j * Gd1] + off + cst(c, qb), IO::pack_(acc), last && DDL_CHAIN_FINCS);
      }
    }
  }

  template <int li>
  __device__ __forceinline__ static void rs(const CParams& p, char* const* base, size_t off, uint64_t qb) {
    RawPh<li> raw;
    rs_load<li>(base, off, qb, raw);
    rs_fold<li>(p, base, off, qb, raw);
  }

  template <int li>
  __device__ __forceinline__ static void ag(char* const* base, size_t off, uint64_t qb) {
    constexpr int g = TP::g(li), Gd = TP::G(li);
    constexpr int n = P / Gd;
    Raw raw[NB][n];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      const int sb = blk(c) % Gd, beta = (blk(c) / Gd) % g;
#pragma unroll
      for (int i = 0; i < n; ++i)
        if (i % g != beta) raw[c][i] = IO::ld(base[sb + (i - i % g + beta) * Gd] + off + cst(c, qb), DDL_CHAIN_REREAD);
    }
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      const int sb = blk(c) % Gd, beta = (blk(c) / Gd) % g;
#pragma unroll
      for (int i = 0; i < n; ++i)
        if (i % g != beta) IO::st(base[sb + i * Gd] + off + cst(c, qb), raw[c][i], DDL_CHAIN_FINCS);
    }
  }

  // Split form (DDL_CHAIN_SPLIT, NB = 1): an RS phase writer by writer (its g_d sources loaded,
  // folded, stored, then the next writer) and an AG phase holder by holder (each receiver's load
  // of the holder's copy, then their stores): at most max(g_d) values in registers instead of
  // P / G_d, so more threads fit an SM (the column chain is latency-bound).
  template <int li>
  __device__ __forceinline__ static void rs_split(const CParams& p, char* const* base, size_t off) {
    constexpr int g = TP::g(li), Gd = TP::G(li), Gd1 = TP::G(li + 1);
    constexpr int sb = B0 % Gd, wb = B0 % Gd1;
    constexpr bool last = li == TP::L - 1;
#pragma unroll
    for (int j = 0; j < P / Gd1; ++j) {
      Raw raw[g];
#pragma unroll
      for (int v = 0; v < g; ++v)
        raw[v] = IO::ld(base[sb + (v + j * g) * Gd] + off, li == 0 ? DDL_CHAIN_FIRST : DDL_CHAIN_REREAD);
      A acc[N];
      IO::unpack_(raw[0], acc);
#pragma unroll
      for (int v = 1; v < g; ++v) {
        A y[N];
        IO::unpack_(raw[v], y);
#pragma unroll
        for (int k = 0; k < N; ++k) acc[k] = Tr<T>::add(acc[k], y[k]);
      }
      if (last && p.op == kAvg) {
#pragma unroll
        for (int k = 0; k < N; ++k) acc[k] = Tr<T>::mul(acc[k], p.scale);
      }
      IO::st(base[wb + j * Gd1] + off, IO::pack_(acc), last && DDL_CHAIN_FINCS);
    }
  }
  template <int li>
  __device__ __forceinline__ static void ag_split(char* const* base, size_t off) {
    constexpr int g = TP::g(li), Gd = TP::G(li), Gd1 = TP::G(li + 1);
    constexpr int sb = B0 % Gd, beta = (B0 / Gd) % g;
#pragma unroll
    for (int j = 0; j < P / Gd1; ++j) {
      Raw raw[g];
#pragma unroll
      for (int v = 0; v < g; ++v)
        if (v != beta) raw[v] = IO::ld(base[sb + (beta + j * g) * Gd] + off, DDL_CHAIN_REREAD);
#pragma unroll
      for (int v = 0; v < g; ++v)
        if (v != beta) IO::st(base[sb + (v + j * g) * Gd] + off, raw[v], DDL_CHAIN_FINCS);
    }
  }
  __device__ __forceinline__ static void run_split(const CParams& p, char* const* base, size_t off) {
    static_for<0, TP::L>([&](auto lc) { rs_split<decltype(lc)::value>(p, base, off); });
    static_for<0, TP::L>([&](auto lc) { ag_split<TP::L - 1 - decltype(lc)::value>(base, off); });
  }

  // every phase after the first RS phase's fold
  __device__ __forceinline__ static void after_first(const CParams& p, char* const* base, size_t off, uint64_t qb) {
    static_for<1, TP::L>([&](auto lc) { rs<decltype(lc)::value>(p, base, off, qb); });
    // allgather phases (a6), live dims descending
    static_for<0, TP::L>([&](auto lc) { ag<TP::L - 1 - decltype(lc)::value>(base, off, qb); });
  }
  __device__ __forceinline__ static void run(const CParams& p, char* const* base, size_t off, uint64_t qb) {
#if DDL_CHAIN_FLAT  // MEASUREMENT ONLY (never a product build): the same fold in registers, P loads and P
                    // stores per column, no intermediate stores / re-reads -- the HBM floor of the access pattern
   if constexpr (TP::L == 2) {
    RawPh<0> raw;
    rs_load<0>(base, off, qb, raw);
    constexpr int g0 = TP::g(0), g1 = TP::g(1);
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      A fin[N];
#pragma unroll
      for (int j = 0; j < g1; ++j) {
        A acc[N];
        IO::unpack_(raw[c][j * g0], acc);
#pragma unroll
        for (int v = 1; v < g0; ++v) {
          A y[N];
          IO::unpack_(raw[c][j * g0 + v], y);
#pragma unroll
          for (int k = 0; k < N; ++k) acc[k] = Tr<T>::add(acc[k], y[k]);
        }
        Raw rr = IO::pack_(acc);
        IO::unpack_(rr, acc);
#pragma unroll
        for (int k = 0; k < N; ++k) fin[k] = j == 0 ? acc[k] : Tr<T>::add(fin[k], acc[k]);
      }
      if (p.op == kAvg) {
#pragma unroll
        for (int k = 0; k < N; ++k) fin[k] = Tr<T>::mul(fin[k], p.scale);
      }
      const Raw out = IO::pack_(fin);
#pragma unroll
      for (int i = 0; i < P; ++i) IO::st(base[i] + off + cst(c, qb), out, DDL_CHAIN_FINCS);
    }
   } else {
    rs<0>(p, base, off, qb);
    after_first(p, base, off, qb);
   }
#else
    if constexpr (DDL_CHAIN_SPLIT && NB == 1) {
      run_split(p, base, off);
    } else {
      // reduce-scatter phases (a4), live dims ascending; the last fuses the epilogue (a5)
      rs<0>(p, base, off, qb);
      after_first(p, base, off, qb);
    }
#endif
  }
};

// ragged tail of a column (elements of a last block that do not fill a vector): element-wise,
// out of line (rare; keeps the hot loop small)
template <typename T, int MP>
__device__ __noinline__ void chain_tail(const CParams& p, char* const* base, uint32_t b, uint64_t e0, uint64_t n) {
  for (uint64_t e = e0; e < n; ++e) chain_column<T, false, MP>(p, base, b, e * sizeof(T));
}
// one column of the CT kernels' tail rows (whole vector or ragged), out of line
template <typename T, int MP>
__device__ __noinline__ void chain_cold(const CParams& p, char* const* base, uint32_t b, uint64_t e0, uint64_t n) {
  if (e0 + Tr<T>::W <= n) chain_column<T, true, MP>(p, base, b, e0 * sizeof(T));
  else for (uint64_t e = e0; e < n; ++e) chain_column<T, false, MP>(p, base, b, e * sizeof(T));
}

// Rows are split per buffer into "full" rows (v < vfull: the column of every block is a whole
// vector -- all but at most ~P rows of a buffer) walked by the hot loop, and the few remaining
// rows (ragged last block, blocks past n) walked afterwards column by column with the generic
// code, so that the hot loop has no bounds checks and no calls.
template <typename T, class TP>
__global__ void __launch_bounds__(kChainThreads, DDL_CHAIN_CT_MINB) ddl_chain_ct_kernel(const __grid_constant__ CParams p) {
  __shared__ char* s_buf[kMaxBuckets][kMaxRanks];
  for (int i = threadIdx.x; i < p.nb * kMaxRanks; i += blockDim.x)
    s_buf[i / kMaxRanks][i % kMaxRanks] = p.b[i / kMaxRanks].buf[i % kMaxRanks];
  __syncthreads();
  pdl_begin();
  constexpr int W = Tr<T>::W;
  constexpr int P = TP::P;
  using Raw = typename ColIO<T, true>::R;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  int k = 0;
#if DDL_CHAIN_ASYNC
  // The first RS phase's P loads of the NEXT column (HBM reads) are issued as cp.async copies into
  // this thread's shared-memory slot while the current column runs its later phases (L2 round
  // trips): they hold no registers while in flight.  Columns in the order (row, block).
  __shared__ uint4 s_stage[P][kChainThreads];  // [rank][thread]: a warp's 16-B copies are contiguous
  auto stage = [&](char* const* bs, uint64_t o) {
#pragma unroll
    for (int i = 0; i < P; ++i) cp_async16(&s_stage[i][threadIdx.x], bs[i] + o);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto row_of = [&](uint32_t v, int& kk, uint64_t& qb, uint64_t& off) {
    while (kk + 1 < p.nb && v >= p.b[kk + 1].row0) ++kk;
    qb = p.b[kk].q * sizeof(T);
    off = (uint64_t)(v - p.b[kk].row0) * 16u;  // column (b, v) is at b*qb + v*16
  };
  if (tid < p.nrows) {
    uint64_t qb0, off0;
    row_of(tid, k, qb0, off0);
    stage(s_buf[k], off0);
  }
  for (uint32_t v = tid; v < p.nrows; v += stride) {
    uint64_t qb, off;
    row_of(v, k, qb, off);
    char* const* base = s_buf[k];
    static_for<0, P>([&](auto bc) {
      constexpr int b = decltype(bc)::value;
      using C = CTCols<T, TP, b, 1>;
      typename C::template RawPh<0> raw;
      asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
      for (int i = 0; i < P; ++i) raw[0][i] = s_stage[i][threadIdx.x];
      C::template rs_fold<0>(p, base, off + b * qb, qb, raw);  // consumes raw: the slot is free again
      if constexpr (b + 1 < P) {
        stage(base, off + (b + 1) * qb);
      } else if (v + stride < p.nrows) {
        int k2 = k;
        uint64_t qb2, off2;
        row_of(v + stride, k2, qb2, off2);
        stage(s_buf[k2], off2);
      }
      C::after_first(p, base, off + b * qb, qb);
    });
  }
  if (false)
#endif
#if DDL_CHAIN_BMAJOR  // A/B: block-major order (the grid walks block 0's columns of every row, then block 1's, ...)
  static_for<0, P>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    int kb = 0;
    for (uint32_t v = tid; v < p.nrows; v += stride) {
      while (kb + 1 < p.nb && v >= p.b[kb + 1].row0) ++kb;
      const uint64_t qb = p.b[kb].q * sizeof(T);
      const uint64_t off = (uint64_t)(v - p.b[kb].row0) * 16u + b * qb;
#if DDL_CHAIN_PF
      // L2 prefetch of the first RS phase's sources DDL_CHAIN_PF grid strides ahead (same
      // buffer only): no registers held, the later loads find them in L2
      {
        const uint32_t vn = v + DDL_CHAIN_PF * stride;
        if (vn < (kb + 1 < p.nb ? p.b[kb + 1].row0 : p.nrows)) {
          const uint64_t offn = off + (uint64_t)DDL_CHAIN_PF * stride * 16u;
#if DDL_CHAIN_PF_BULK  // one lane per warp: a bulk L2 prefetch of the warp's 512 B per rank
          if ((threadIdx.x & 31) == 0)
#pragma unroll
            for (int i = 0; i < P; ++i)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], 512;" ::"l"(s_buf[kb][i] + offn) : "memory");
#else
#pragma unroll
          for (int i = 0; i < P; ++i) asm volatile("prefetch.global.L2 [%0];" ::"l"(s_buf[kb][i] + offn));
#endif
        }
      }
#endif
      CTCols<T, TP, b, 1>::run(p, s_buf[kb], off, qb);
    }
  });
  if (false)
#endif
#if DDL_CHAIN_VPT > 1  // A/B: VPT adjacent vectors of each block per thread, in lockstep
  for (uint32_t v = tid * DDL_CHAIN_VPT; v < p.nrows; v += stride * DDL_CHAIN_VPT) {
    while (k + 1 < p.nb && v >= p.b[k + 1].row0) ++k;
    const uint64_t qb = p.b[k].q * sizeof(T);
    const uint64_t off = (uint64_t)(v - p.b[k].row0) * 16u;
    char* const* base = s_buf[k];
    static_for<0, P>([&](auto bc) {
      constexpr int b = decltype(bc)::value;
      CTCols<T, TP, b, DDL_CHAIN_VPT, true>::run(p, base, off + b * qb, qb);
    });
  }
  if (false)
#endif
  for (uint32_t v = tid; v < p.nrows; v += stride) {
    while (k + 1 < p.nb && v >= p.b[k + 1].row0) ++k;
    const uint64_t qb = p.b[k].q * sizeof(T);
    const uint64_t off = (uint64_t)(v - p.b[k].row0) * 16u;  // column (b, v) is at b*qb + v*16
    char* const* base = s_buf[k];
    static_for<0, P / DDL_CHAIN_NB>([&](auto gc) {
      constexpr int b0 = decltype(gc)::value * DDL_CHAIN_NB;
      CTCols<T, TP, b0, DDL_CHAIN_NB>::run(p, base, off + b0 * qb, qb);
    });
  }
  // the rest: rows vfull .. vq-1 of every buffer, one column (b, v) per step
  k = 0;
  for (uint32_t c = tid; c < p.ncols; c += stride) {
    while (k + 1 < p.nb && c >= p.b[k + 1].col0) ++k;
    const CBucket& B = p.b[k];
    const uint32_t tail_rows = B.vq - B.vfull;
    const uint32_t lc = c - B.col0;
    const uint32_t b = lc / tail_rows;
    const uint64_t e0 = (uint64_t)b * B.q + (uint64_t)(B.vfull + (lc - b * tail_rows)) * W;
    if (e0 < B.n) chain_cold<T, P>(p, s_buf[k], b, e0, B.n);
  }
}

// ------------------------------------------------------------------------ TMA-fed column chain
// DDL_CHAIN_TMA: the CT kernel with the first RS phase's loads (the HBM reads) moved off the
// threads: a producer warp bulk-copies (cp.async.bulk) the P ranks' segments of a tile --
// kTmaCons consecutive full rows of one block b -- into a kTmaStages-deep shared-memory ring;
// each of the kTmaCons consumer threads takes its column's P sources from the ring, folds and
// stores them (RS phase 0), releases the stage, and runs the later phases with LDG / STG as in
// ddl_chain_ct_kernel.  The reads in flight then cost no registers and no L1 miss slots.
#ifndef DDL_CHAIN_TMA_DEFAULT  // loopback default: the TMA-fed kernel (1) or the LDG one (0)
#define DDL_CHAIN_TMA_DEFAULT 1
#endif
#ifndef DDL_CHAIN_TMA_CONS
#define DDL_CHAIN_TMA_CONS 320
#endif
#ifndef DDL_CHAIN_TMA_STAGES
#define DDL_CHAIN_TMA_STAGES 2
#endif
constexpr int kTmaCons = DDL_CHAIN_TMA_CONS;
constexpr int kTmaStages = DDL_CHAIN_TMA_STAGES;
template <int P>
constexpr size_t chain_tma_smem() {
  return (size_t)kTmaStages * P * kTmaCons * 16 + 2 * kTmaStages * sizeof(uint64_t);
}

template <typename T, class TP>
__global__ void __launch_bounds__(kTmaCons + 32, 1) ddl_chain_tma_kernel(const __grid_constant__ CParams p) {
  constexpr int W = Tr<T>::W;
  constexpr int P = TP::P;
  constexpr uint32_t SEG = kTmaCons * 16;  // bytes of one rank's segment of a tile
  using Raw = typename ColIO<T, true>::R;
  extern __shared__ __align__(128) char dsm[];
  char* ring = dsm;  // [stage][rank][SEG]
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + (size_t)kTmaStages * P * SEG);
  uint64_t* empty = full + kTmaStages;
  __shared__ char* s_buf[kMaxBuckets][kMaxRanks];
  __shared__ uint32_t s_ch0[kMaxBuckets + 1];  // first chunk (kTmaCons full rows) of each buffer
  for (int i = threadIdx.x; i < p.nb * kMaxRanks; i += blockDim.x)
    s_buf[i / kMaxRanks][i % kMaxRanks] = p.b[i / kMaxRanks].buf[i % kMaxRanks];
  if (threadIdx.x == 0) {
    uint32_t c = 0;
    for (int k = 0; k < p.nb; ++k) {
      s_ch0[k] = c;
      c += (p.b[k].vfull + kTmaCons - 1) / kTmaCons;
    }
    s_ch0[p.nb] = c;
    for (int st = 0; st < kTmaStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kTmaCons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_begin();
  const uint32_t C = s_ch0[p.nb];
  const uint32_t ntiles = (uint32_t)P * C;
  // tile t: block b = t / C (block-major), chunk t % C -> buffer k, rows [r0, r0 + rn)
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
        const int st = (int)(i % kTmaStages);
        if (i >= (uint32_t)kTmaStages) mbar_wait(&empty[st], ((i / kTmaStages) - 1) & 1u);
        int b, k;
        uint32_t r0, rn;
        tile_of(t, b, k, r0, rn);
        const uint64_t qb = p.b[k].q * sizeof(T);
        mbar_arm(&full[st], (uint32_t)P * rn * 16u);
#pragma unroll
        for (int r = 0; r < P; ++r)
          tma_load(ring + ((size_t)st * P + r) * SEG, s_buf[k][r] + (uint64_t)b * qb + (uint64_t)r0 * 16u, rn * 16u,
                   &full[st]);
      }
    }
    return;
  }
  uint32_t i = 0;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
    const int st = (int)(i % kTmaStages);
    int b, k;
    uint32_t r0, rn;
    tile_of(t, b, k, r0, rn);
    const uint64_t qb = p.b[k].q * sizeof(T);
    const bool mine = (uint32_t)threadIdx.x < rn;
    const uint64_t off = (uint64_t)b * qb + (uint64_t)(r0 + threadIdx.x) * 16u;
    mbar_wait(&full[st], (i / kTmaStages) & 1u);
    static_for<0, P>([&](auto bc) {
      constexpr int B = decltype(bc)::value;
      if (b != B) return;
      using Cl = CTCols<T, TP, B, 1>;
      typename Cl::template RawPh<0> raw;
      if (mine) {
#pragma unroll
        for (int r = 0; r < P; ++r) raw[0][r] = reinterpret_cast<const Raw*>(ring + ((size_t)st * P + r) * SEG)[threadIdx.x];
        Cl::template rs_fold<0>(p, s_buf[k], off, qb, raw);  // consumes raw: the stage is free
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (mine) Cl::after_first(p, s_buf[k], off, qb);
    });
  }
  // the rest: rows vfull .. vq-1 of every buffer, one column (b, v) per consumer step
  const uint32_t cstride = gridDim.x * kTmaCons;
  int k = 0;
  for (uint32_t c = blockIdx.x * kTmaCons + threadIdx.x; c < p.ncols; c += cstride) {
    while (k + 1 < p.nb && c >= p.b[k + 1].col0) ++k;
    const CBucket& Bk = p.b[k];
    const uint32_t tail_rows = Bk.vq - Bk.vfull;
    const uint32_t lc = c - Bk.col0;
    const uint32_t b = lc / tail_rows;
    const uint64_t e0 = (uint64_t)b * Bk.q + (uint64_t)(Bk.vfull + (lc - b * tail_rows)) * W;
    if (e0 < Bk.n) chain_cold<T, P>(p, s_buf[k], b, e0, Bk.n);
  }
}

}  // namespace ddl
