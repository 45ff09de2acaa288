// ddl_plan.h -- the phase planner shared by libddl's host code and its kernels.
//
// Everything here is integer bookkeeping of SURVEY.md 8(a) rows a1/a3/a7 (§2.1,
// P:L52-54): mixed-radix coordinates, groups, the strided block
// sets A_d(r), and the 2L+1 device barriers of one call.  __host__ __device__ so that the
// host-side query functions exported for tests (ddl_plan_*) and the kernels execute the
// very same code.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define DDL_HD __host__ __device__ __forceinline__
#else
#define DDL_HD inline
#endif

namespace ddl {

constexpr int kMaxRanks = 16;
constexpr int kMaxDims = 8;

struct Topo {
  int P;                  // nranks
  int k;                  // ndims
  int g[kMaxDims];        // group size per dim, innermost first
  int G[kMaxDims + 1];    // G[d] = prod_{j<d} g[j]; G[k] = P
  int nlive;              // dims with g > 1
  int live[kMaxDims];     // their indices, ascending
};

// c_d(r) = floor(r / G_d) mod g_d
DDL_HD int coord(const Topo& t, int r, int d) { return (r / t.G[d]) % t.g[d]; }

// m_v: member of r's group in dim d whose coordinate d is v
DDL_HD int member(const Topo& t, int r, int d, int v) { return r + (v - coord(t, r, d)) * t.G[d]; }

// A_{d}(r) is { (r mod G_d) + i * G_d : i < P / G_d }: the blocks agreeing with r on all
// coordinates below d.  (Blocks are mixed-radix numbered like ranks.)
DDL_HD int nblocks(const Topo& t, int d) { return t.P / t.G[d]; }
DDL_HD int block_of(const Topo& t, int r, int d, int i) { return (r % t.G[d]) + i * t.G[d]; }

// Barrier schedule of one hierarchical call, L = nlive, 2L+1 barriers:
//   j = 0           : start, with group live[0]          (inputs of RS live[0] ready)
//   j = 1..L-1      : before RS live[j], group live[j]   (partials of RS live[j-1] ready)
//   j = L           : before AG live[L-1], group live[L-1]
//   j = L+1..2L-1   : before AG live[2L-1-j], that group (AG live[2L-j] done)
//   j = 2L          : end, with EVERY group of r         (every peer finished reading r)
// barrier_npeers / barrier_peer enumerate the peers (r itself excluded), one lane each.
DDL_HD int barrier_dim(const Topo& t, int j) {
  const int L = t.nlive;
  if (j < L) return t.live[j];
  if (j == L) return t.live[L - 1];
  if (j < 2 * L) return t.live[2 * L - 1 - j];
  return -1;  // end barrier: all live dims
}

DDL_HD int barrier_npeers(const Topo& t, int j) {
  const int d = barrier_dim(t, j);
  if (d >= 0) return t.g[d] - 1;
  int n = 0;
  for (int li = 0; li < t.nlive; ++li) n += t.g[t.live[li]] - 1;
  return n;
}

// The l-th peer (l < barrier_npeers) of rank r in barrier j.  One lane per peer on device.
DDL_HD int barrier_peer(const Topo& t, int r, int j, int l) {
  int d = barrier_dim(t, j);
  if (d < 0) {  // end barrier: walk the live dims
    for (int li = 0; li < t.nlive; ++li) {
      const int dd = t.live[li];
      if (l < t.g[dd] - 1) { d = dd; break; }
      l -= t.g[dd] - 1;
    }
  }
  const int c = coord(t, r, d);
  const int v = l < c ? l : l + 1;  // skip r itself
  return member(t, r, d, v);
}

// One-shot barriers (2 of them): every other rank.
DDL_HD int all_peer(int r, int l) { return l < r ? l : l + 1; }

// Returns 0 on success, else a nonzero code (bad dims).
DDL_HD int make_topo(Topo* t, int P, const int* dims, int ndims) {
  if (P < 1 || ndims < 1 || ndims > kMaxDims) return 1;
  long long prod = 1;
  for (int d = 0; d < ndims; ++d) {
    if (dims[d] < 1) return 1;
    prod *= dims[d];
    if (prod > (1 << 20)) return 1;
  }
  if (prod != P) return 1;
  t->P = P;
  t->k = ndims;
  t->G[0] = 1;
  t->nlive = 0;
  for (int d = 0; d < kMaxDims; ++d) t->g[d] = 1;
  for (int d = 0; d < ndims; ++d) {
    t->g[d] = dims[d];
    t->G[d + 1] = t->G[d] * dims[d];
    if (dims[d] > 1) t->live[t->nlive++] = d;
  }
  for (int d = ndims + 1; d <= kMaxDims; ++d) t->G[d] = P;
  return 0;
}

// q = roundup(ceil(n / P), V), V = 16 / elem_size
DDL_HD uint64_t block_elems(uint64_t n, int P, int elem_size) {
  const uint64_t V = 16 / elem_size;
  const uint64_t per = (n + P - 1) / P;
  return (per + V - 1) / V * V;
}

}  // namespace ddl
