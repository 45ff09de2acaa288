// ddl_device_variants.cuh -- experimental variants of the hierarchical kernel, selected by
// DDL_DYN / DDL_STEAL / DDL_STREAM (all parity-tested; all measured slower than the default
// per-CTA-slice TMA path in loopback -- DESIGN.md 9.3 has the numbers).  Included by
// ddl_device.cuh inside namespace ddl, after the helpers they share.
#pragma once

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
          atomicCAS(p.err, 0, kErrTimeout);
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
            atomicCAS(p.err, 0, kErrTimeout);
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
          atomicCAS(p.err, 0, kErrTimeout);
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
  pdl_begin();
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

