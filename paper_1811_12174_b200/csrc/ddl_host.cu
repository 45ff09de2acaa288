// ddl_host.cu -- libddl's C ABI (include/ddl.h): communicator lifecycle, cudaIpc peer
// mapping, the per-call planner (block size, CTA slices, algorithm choice) and the kernel
// launches.  See DESIGN.md for the design and the paper citations.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "ddl.h"
#include "ddl_device.cuh"
#include "ddl_chain.cuh"
#include "ddl_plan.h"
#include "ddl_nvls.h"

using namespace ddl;

#ifndef DDL_EXPERIMENTAL
#define DDL_EXPERIMENTAL 0  // 1: also compile the PATH 3 / PATH 4 experiment kernels
#endif
static_assert(DDL_MAX_RANKS == kMaxRanks, "header / planner rank limit");
static_assert(DDL_MAX_DIMS == kMaxDims, "header / planner dims limit");

namespace {

constexpr uint32_t kMagic = 0xDD1A11EDu;

thread_local std::string g_last_error;

ddl_result_t cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  if (std::getenv("DDL_DEBUG")) std::fprintf(stderr, "[ddl] %s\n", g_last_error.c_str());
  return DDL_ERR_CUDA;
}
#define DDL_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

// Switches to the communicator's device for the duration of an API call and restores the
// caller's current device afterwards (the ABI never leaves the caller's device changed).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};
#define DDL_ON_DEVICE(dev)                                              \
  DeviceGuard dg_(dev);                                                 \
  if (dg_.err != cudaSuccess) return cuda_fail(dg_.err, "cudaSetDevice")

size_t env_size(const char* name, size_t dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return (size_t)std::strtoull(v, nullptr, 10);
}

int elem_size(ddl_dtype_t dt) { return dt == DDL_BFLOAT16 ? 2 : 4; }
bool valid_dtype(int dt) { return dt == DDL_INT32 || dt == DDL_FLOAT32 || dt == DDL_BFLOAT16; }
bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

struct Handle {  // exported per rank, all-gathered by the caller
  uint32_t magic;
  int32_t rank, nranks, ndims;
  int32_t dims[kMaxDims];
  int32_t cmax;
  int32_t pad;
  uint64_t flags_bytes, max_bytes, alloc_bytes, scratch_half, ll_slot;
  char pci[32];
  cudaIpcMemHandle_t ipc;
};

struct RegHandle {  // exported per rank by ddl_register_export, all-gathered by the caller
  uint32_t magic;
  int32_t rank;
  uint64_t bytes;
  uint64_t offset;  // registered pointer - base of its cudaMalloc allocation
  cudaIpcMemHandle_t ipc;
};
constexpr uint32_t kRegMagic = 0xDD1A4E61u;

typedef int (*CuMemGetAddressRange)(unsigned long long*, size_t*, unsigned long long);

// Base of the cudaMalloc allocation containing ptr (driver entry point, no libcuda link).
cudaError_t alloc_base(const void* ptr, char** base) {
  static CuMemGetAddressRange fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
    if (e != cudaSuccess || !f) return e != cudaSuccess ? e : cudaErrorNotSupported;
    fn = reinterpret_cast<CuMemGetAddressRange>(f);
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (unsigned long long)(uintptr_t)ptr) != 0) return cudaErrorInvalidValue;
  *base = reinterpret_cast<char*>(b);
  return cudaSuccess;
}

}  // namespace

struct ddl_comm {
  bool loopback = false;
  int rank = 0;
  int P = 1;
  int ndims = 1;
  int dims[kMaxDims] = {1};
  Topo topo{};
  int device = 0;
  int num_sms = 148;
  int cmax = 0;
  size_t flags_bytes = 0;  // per rank
  size_t max_bytes = 0;
  // multi-process: [flags | symmetric buffer | staging], one allocation, one IPC handle
  char* alloc = nullptr;
  size_t alloc_bytes = 0;
  char* peer_base[kMaxRanks] = {};
  bool peer_mapped[kMaxRanks] = {};
  bool connected = false;
  // loopback: P flag regions + RS workspace
  char* lb_flags = nullptr;
  char* lb_ws = nullptr;
  size_t lb_ws_bytes = 0;  // per virtual rank
  char* lb_ll = nullptr;   // loopback LL receive regions: P x (two halves of P slots of ll_slot bytes)
  int* err = nullptr;      // sticky device error
  ddl_algo_t algo = DDL_ALGO_AUTO;
  size_t oneshot_max = 512 << 10;  // crossover measured in loopback (profiles/r01_oneshot_crossover.txt)
  size_t min_slice_bytes = 16 << 10;
  int ctas_limit = 0;  // 0 = occupancy bound
  uint64_t timeout_ns = 10ull * 1000 * 1000 * 1000;
  int skip_rank = -1;
  bool use_tma = true;
  bool use_steal = false;  // DDL_STEAL=1: per-CTA slices + work stealing (PATH 4)
  bool check = false;       // DDL_CHECK=1: ranks compare (count, dtype, op, algorithm) at the first barrier
  bool use_stream = false;  // DDL_STREAM=1: no inner phase barriers, per-chunk progress (PATH 5)
  bool use_dyn = false;     // DDL_DYN=1: rank-level barriers + dynamic chunks (measured slower)
  int gpu_share = 1;        // ranks sharing this GPU (loopback: P; in-process test groups: P)
  uint64_t* trace = nullptr;  // DDL_TRACE=1: per-CTA phase timeline (debug)
  size_t tma_min_slice_bytes = 16 << 10;  // TMA path only when per-CTA slices are at least this big
  int channels = 2;                        // DDL_CHANNELS: channels of a grouped all-reduce
  int transpose = 1;                       // DDL_TRANSPOSE: loopback grids (P, ctas) (profiles/r01_transpose_ab.txt)
  int l2hint = 47;                         // DDL_L2_HINTS: KParams::l2hint bits (profiles/r01_l2_hints.txt, r02_ab2)
  int group_waves = 1;                     // DDL_GROUP_WAVES: waves per bucket in a grouped all-reduce (0 = auto)
  size_t group_wave_bytes = 0;             // DDL_GROUP_WAVE_MB: per-wave partial footprint budget (0 = off)
  int group_order = 0;                     // DDL_GROUP_ORDER: 0 LPT (longest first), 1 ascending within a channel
  int deep_copy = 1;                       // DDL_DEEP_COPY: copy phases through the deep sub-stage pipeline
  int waves = 0;                           // DDL_WAVES: slices per CTA per hierarchical call (0 = auto)
  size_t wave_slice_bytes = 112 << 10;     // auto: target per-CTA slice of one wave
  size_t min_wave_slice_bytes = 16 << 10;  // no waves below this slice size
  bool use_pdl = true;  // programmatic dependent launch (DDL_PDL=0: plain stream order)
  bool force_sys = false;  // DDL_FORCE_SYS_SCOPE=1: .sys flags even when every rank shares this GPU
  bool debug = false;      // DDL_DEBUG: one stderr line per launch
  int stream_every = 1;    // DDL_STREAM_EVERY (PATH 5)
  int lb_chain = 1;        // DDL_LB_CHAIN: loopback all-reduces through the column-chain kernel (0: the
                           // per-CTA slice kernels with device barriers, as across processes)
  bool chain_generic = false;  // DDL_CHAIN_GENERIC=1: the generic chain kernel also where a CT kernel exists
  int chain_tma = DDL_CHAIN_TMA_DEFAULT;  // DDL_CHAIN_TMA: the TMA-fed CT kernel (ddl_chain.cuh): 1 on, 0 off,
                                          // -1 auto = from P = 4 (at P = 2 the LDG form is as fast or
                                          // faster: profiles/r02_ab/r02_p2_ab.txt)

  uint32_t* flags_of(int r) const {
    if (loopback) return reinterpret_cast<uint32_t*>(lb_flags + (size_t)r * flags_bytes);
    return reinterpret_cast<uint32_t*>(r == rank ? alloc : peer_base[r]);
  }
  char* sym_of(int r) const { return (r == rank ? alloc : peer_base[r]) + flags_bytes; }
  // registered user buffers (ddl_register_*): zero-copy at the same offset on every rank
  struct Reg {
    bool used = false;
    char* local = nullptr;
    size_t bytes = 0;
    char* peer[kMaxRanks] = {};      // every rank's registered pointer, as mapped here
    char* mapped[kMaxRanks] = {};    // IPC mapping bases this registration opened (to close)
  };
  static constexpr int kMaxRegs = 64;
  Reg regs[kMaxRegs];
  // IPC mappings of peer allocations, shared by registrations of the same allocation
  struct Mapping {
    int rank;
    cudaIpcMemHandle_t h;
    char* base;
    int refs;
  };
  std::vector<Mapping> maps;
  char* stage_of(int r) const { return (r == rank ? alloc : peer_base[r]) + flags_bytes + max_bytes; }
  size_t scratch_half = 0;  // one-shot scratch: two halves after the staging area
  char* scratch_of(int r) const { return stage_of(r) + max_bytes; }
  // LL receive region after the scratch: two halves of P slots of ll_slot bytes
  size_t ll_max = 64 << 10;  // AUTO uses LL up to this message size (DDL_LL_MAX_BYTES, 0 = off)
  size_t ll_slot = 0;
  nvls::State nvls;          // NVLS phases (ddl_nvls_*), multi-process only
  int nvls_dims_mask = -1;   // DDL_NVLS_DIMS: which live dims may run in the switch (bit d; -1 all)
  bool nvls_emulate = false; // DDL_NVLS_EMULATE=1 (test hook): hierarchical calls run PATH 7 with the
                             // NVLS phases' data flow emulated by unicast accesses (one GPU)
  char* ll_of(int r) const {
    if (loopback) return lb_ll + (size_t)r * 2 * (size_t)P * ll_slot;
    return scratch_of(r) + 2 * scratch_half;
  }
};

extern "C" {
static void preload_kernels();
}

namespace {

// Launch with the optional cooperative (loopback: all P x nctas CTAs co-resident) and
// programmatic-dependent-launch attributes (every kernel starts with pdl_begin()).
cudaError_t launch_ex(const void* fn, dim3 grid, size_t smem, cudaStream_t s, void** args, bool coop, bool pdl,
                      int threads = kThreads) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

bool pdl_default() {
  static const bool on = env_size("DDL_PDL", 1) != 0;
  return on;
}

// Resident CTAs (kThreads each) per SM for a kernel, cached.
int blocks_per_sm(const void* fn, size_t smem = 0, int threads = kThreads) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(fn);
  if (it != cache.end()) return it->second;
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem) != cudaSuccess) nb = 1;
  if (nb < 1) nb = 1;
  cache[fn] = nb;
  return nb;
}

void apply_env(ddl_comm* c) {
  c->timeout_ns = env_size("DDL_TIMEOUT_MS", 10000) * 1000000ull;
  c->oneshot_max = env_size("DDL_ONESHOT_MAX_BYTES", c->oneshot_max);
  c->min_slice_bytes = env_size("DDL_MIN_SLICE_BYTES", c->min_slice_bytes);
  c->ctas_limit = (int)env_size("DDL_CTAS", 0);
  c->use_tma = env_size("DDL_NO_TMA", 0) == 0;
  c->use_dyn = env_size("DDL_DYN", 0) != 0;
  c->use_steal = env_size("DDL_STEAL", 0) != 0;
  c->use_stream = env_size("DDL_STREAM", 0) != 0;
  c->check = env_size("DDL_CHECK", 0) != 0;
  c->tma_min_slice_bytes = env_size("DDL_TMA_MIN_SLICE_BYTES", c->tma_min_slice_bytes);
  c->ll_max = env_size("DDL_LL_MAX_BYTES", c->ll_max);
  c->use_pdl = env_size("DDL_PDL", 1) != 0;
  c->channels = (int)env_size("DDL_CHANNELS", c->channels);
  c->group_waves = (int)env_size("DDL_GROUP_WAVES", c->group_waves);
  c->group_wave_bytes = env_size("DDL_GROUP_WAVE_MB", c->group_wave_bytes >> 20) << 20;
  c->group_order = (int)env_size("DDL_GROUP_ORDER", c->group_order);
  c->deep_copy = (int)env_size("DDL_DEEP_COPY", c->deep_copy);
  c->nvls_dims_mask = std::getenv("DDL_NVLS_DIMS") ? (int)env_size("DDL_NVLS_DIMS", 0) : -1;
  c->nvls_emulate = env_size("DDL_NVLS_EMULATE", 0) != 0;
  c->l2hint = (int)env_size("DDL_L2_HINTS", c->l2hint);
  c->transpose = (int)env_size("DDL_TRANSPOSE", c->transpose);
  if (c->channels < 1) c->channels = 1;
  if (c->channels > kMaxChannels) c->channels = kMaxChannels;
  c->waves = (int)env_size("DDL_WAVES", c->waves);
  if (c->waves > 64) c->waves = 64;
  c->wave_slice_bytes = env_size("DDL_WAVE_SLICE_BYTES", c->wave_slice_bytes);
  if (c->wave_slice_bytes < 4096) c->wave_slice_bytes = 4096;
  c->min_wave_slice_bytes = env_size("DDL_MIN_WAVE_SLICE_BYTES", c->min_wave_slice_bytes);
  c->force_sys = env_size("DDL_FORCE_SYS_SCOPE", 0) != 0;
  c->debug = std::getenv("DDL_DEBUG") != nullptr;
  c->stream_every = (int)env_size("DDL_STREAM_EVERY", 1);
  c->lb_chain = (int)env_size("DDL_LB_CHAIN", c->lb_chain);
  c->chain_generic = env_size("DDL_CHAIN_GENERIC", 0) != 0;
  if (const char* v = std::getenv("DDL_CHAIN_TMA")) c->chain_tma = *v ? (int)std::strtol(v, nullptr, 10) : c->chain_tma;
  if (c->stream_every < 1) c->stream_every = 1;
  if (const char* a = std::getenv("DDL_ALGO")) {
    if (!std::strcmp(a, "hier")) c->algo = DDL_ALGO_HIER;
    else if (!std::strcmp(a, "oneshot")) c->algo = DDL_ALGO_ONESHOT;
    else if (!std::strcmp(a, "ll")) c->algo = DDL_ALGO_LL;
    else c->algo = DDL_ALGO_AUTO;
  }
}

ddl_result_t common_init(ddl_comm* c, int nranks, const int* dims, int ndims, int dev) {
  if (!dims) return DDL_ERR_INVALID_ARGUMENT;
  if (nranks > kMaxRanks) return DDL_ERR_UNSUPPORTED;
  if (make_topo(&c->topo, nranks, dims, ndims)) return DDL_ERR_BAD_DIMS;
  c->P = nranks;
  c->ndims = ndims;
  for (int d = 0; d < ndims; ++d) c->dims[d] = dims[d];
  c->device = dev;
  DDL_CUDA(cudaSetDevice(dev));
  DDL_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev));
  c->cmax = c->num_sms * 4;
  const size_t words = (size_t)c->cmax * (1 + (size_t)kNumSlots * nranks) + kRankStateWords +
                       16 + 2 * (size_t)kNumSlots * c->cmax +  // + steal counters
                       2 + 2 * (size_t)kNumSlots * c->cmax +   // + streaming progress words
                       (size_t)c->cmax * kMaxRanks;             // + DDL_CHECK signatures
  c->flags_bytes = (words * 4 + 65535) / 65536 * 65536;
  apply_env(c);
#if !DDL_EXPERIMENTAL
  // the rank-level dynamic (PATH 3) and work-stealing (PATH 4) kernels were measured slower
  // and are only compiled with DDL_EXPERIMENTAL=1 bash build.sh
  if (c->use_dyn || c->use_steal) return DDL_ERR_UNSUPPORTED;
#endif
  preload_kernels();
  if (env_size("DDL_TRACE", 0)) {
    const size_t tb = (size_t)nranks * c->cmax * kTraceEvents * sizeof(uint64_t);
    DDL_CUDA(cudaMalloc(&c->trace, tb));
    DDL_CUDA(cudaMemset(c->trace, 0, tb));
  }
  return DDL_SUCCESS;
}

// ---------------------------------------------------------------- per-call plan
// UnitDesc::bytes and the register-staged item prefixes are 32-bit: one CTA's slice of a
// block must stay below this many bytes (reached only with DDL_CTAS tiny and multi-GiB
// messages).  Larger slices are cut into waves where the kernel has them, else the call
// returns DDL_ERR_TOO_LARGE -- never a silent wrap.
constexpr uint64_t kMaxSliceBytes = 1ull << 30;

struct Plan {
  uint64_t q = 0;
  uint64_t slice = 0;
  int nctas = 0;
  bool vec = true;
  int path = 2;  // hierarchical kernel variant: 0 element-wise, 1 register-staged, 2 TMA-staged,
                 // 3 TMA-staged with rank-level barriers and dynamic chunks
  bool oneshot = false;
  bool ll = false;  // LL one-shot (multi-process small messages)
  int r = 1;        // one-shot: vectors per thread
  int nwaves = 1;   // hierarchical: slices per CTA, run as successive waves
};

template <typename T>
const void* hier_fn(int path) {
  if (path == 7) return (const void*)ddl_hier_kernel<T, 7>;
  if (path == 6) return (const void*)ddl_hier_kernel<T, 6>;
  if (path == 5) return (const void*)ddl_hier_kernel<T, 5>;
#if DDL_EXPERIMENTAL
  if (path == 4) return (const void*)ddl_hier_kernel<T, 4>;
  if (path == 3) return (const void*)ddl_dyn_kernel<T>;
#else
  if (path == 3 || path == 4) return nullptr;
#endif
  if (path == 2) return (const void*)ddl_hier_kernel<T, 2>;
  return path == 1 ? (const void*)ddl_hier_kernel<T, 1> : (const void*)ddl_hier_kernel<T, 0>;
}
template <typename T, int R>
const void* oneshot_fn_r(int K) {
  switch (K) {
    case 1: return (const void*)ddl_oneshot_kernel<T, 1, R>;
    case 2: return (const void*)ddl_oneshot_kernel<T, 2, R>;
    case 3: return (const void*)ddl_oneshot_kernel<T, 3, R>;
    case 4: return (const void*)ddl_oneshot_kernel<T, 4, R>;
    default: return nullptr;
  }
}
template <typename T>
const void* oneshot_fn(int K, int R) {
  return R == 4 ? oneshot_fn_r<T, 4>(K) : R == 2 ? oneshot_fn_r<T, 2>(K) : oneshot_fn_r<T, 1>(K);
}
template <typename T>
const void* ll_fn(int K) {
  switch (K) {
    case 1: return (const void*)ddl_ll_kernel<T, 1>;
    case 2: return (const void*)ddl_ll_kernel<T, 2>;
    case 3: return (const void*)ddl_ll_kernel<T, 3>;
    case 4: return (const void*)ddl_ll_kernel<T, 4>;
    default: return nullptr;
  }
}
const void* ll_fn_dt(ddl_dtype_t dt, int K) {
  if (dt == DDL_INT32) return ll_fn<int32_t>(K);
  if (dt == DDL_FLOAT32) return ll_fn<float>(K);
  return ll_fn<__nv_bfloat16>(K);
}
const void* hier_fn_dt(ddl_dtype_t dt, int path) {
  if (dt == DDL_INT32) return hier_fn<int32_t>(path);
  if (dt == DDL_FLOAT32) return hier_fn<float>(path);
  return hier_fn<__nv_bfloat16>(path);
}
size_t hier_smem(int path) { return (path >= 2 && path != 7) ? kTmaSmem : 0; }
const void* oneshot_fn_dt(ddl_dtype_t dt, int K, int R) {
  if (dt == DDL_INT32) return oneshot_fn<int32_t>(K, R);
  if (dt == DDL_FLOAT32) return oneshot_fn<float>(K, R);
  return oneshot_fn<__nv_bfloat16>(K, R);
}

// CTAs per rank that may be resident at once (loopback: all P ranks share the GPU).
int cap_per_rank(const ddl_comm* c, const void* fn, size_t smem = 0) {
  int cap = blocks_per_sm(fn, smem) * c->num_sms;
  cap /= c->gpu_share;
  if (c->ctas_limit > 0 && c->ctas_limit < cap) cap = c->ctas_limit;
  if (cap > c->cmax) cap = c->cmax;
  return cap < 1 ? 1 : cap;
}

Plan plan_hier(const ddl_comm* c, uint64_t n, uint64_t q, ddl_dtype_t dt, bool vec) {
  Plan pl;
  pl.q = q;
  pl.vec = vec;
  const int w = elem_size(dt);
  const uint64_t W = vec ? 16 / w : 1;
  pl.path = !vec ? 0 : (c->use_tma ? (c->use_dyn ? 3 : (c->use_steal ? 4 : (c->use_stream ? 5 : 2))) : 1);
  int cap = cap_per_rank(c, hier_fn_dt(dt, pl.path), hier_smem(pl.path));
  if (pl.path >= 2 && q * w < c->tma_min_slice_bytes * (uint64_t)cap) {
    // small per-CTA slices: the register-staged path has lower per-phase latency
    pl.path = 1;
    cap = cap_per_rank(c, hier_fn_dt(dt, 1), 0);
  }
  uint64_t want = (q * w + c->min_slice_bytes - 1) / c->min_slice_bytes;
  if (want < 1) want = 1;
  if (want > (uint64_t)cap) want = cap;
  uint64_t slice = (q + want - 1) / want;
  slice = (slice + W - 1) / W * W;
  if (slice == 0) slice = W;
  pl.slice = slice;
  pl.nctas = (int)((q + slice - 1) / slice);
  if (pl.nctas < 1) pl.nctas = 1;
  // Waves (TMA-staged PATH 2 only): the same CTAs walk nwaves slices each, one wave after another.
  // Auto (DDL_WAVES unset): about one wave per wave_slice_bytes of per-CTA slice, at most 32,
  // when every rank is on this GPU (loopback / in-process: measured 6-17 % faster from 64 MiB
  // up, slower below, profiles/r01_waves_sweep.txt); across GPUs one wave until the barrier
  // cost over NVLink is measured.  DDL_WAVES=k forces k.
  int waves = c->waves;
  if (waves == 0) {
    const uint64_t sb = pl.slice * (uint64_t)w;
    waves = (c->gpu_share == c->P) ? (int)std::min<uint64_t>(32, sb / c->wave_slice_bytes) : 1;
  }
  if (pl.path == 2 && pl.slice * (uint64_t)w > kMaxSliceBytes)  // 32-bit slice fields: cut into waves
    waves = std::max<int>(waves, (int)((pl.slice * (uint64_t)w + kMaxSliceBytes - 1) / kMaxSliceBytes));
  if (waves > 1 && pl.path == 2) {
    uint64_t s2 = (q + (uint64_t)pl.nctas * waves - 1) / ((uint64_t)pl.nctas * waves);
    s2 = (s2 + W - 1) / W * W;
    if (s2 * w >= c->min_wave_slice_bytes) {
      pl.slice = s2;
      pl.nwaves = (int)((q + (uint64_t)pl.nctas * s2 - 1) / ((uint64_t)pl.nctas * s2));
      if (pl.nwaves > 1) pl.path = 6;  // the TMA-staged kernel with the wave loop compiled in
      if (pl.path == 6 && cap_per_rank(c, hier_fn_dt(dt, 6), hier_smem(6)) < pl.nctas) {
        pl.path = 2;  // the wave kernel would not keep every CTA resident: one wave
        pl.nwaves = 1;
        pl.slice = slice;
      }
    }
  }
  (void)n;
  return pl;
}

bool plan_oneshot(const ddl_comm* c, uint64_t n, ddl_dtype_t dt, Plan* pl) {
  const int K = c->topo.nlive;
  for (int R : {1, 2, 4}) {  // fewest vectors per thread that fit the resident CTAs
    const void* fn = oneshot_fn_dt(dt, K, R);
    if (!fn) return false;
    const uint64_t per_cta = (uint64_t)kThreads * R * (16 / elem_size(dt));
    const uint64_t ctas = (n + per_cta - 1) / per_cta;
    if (ctas > (uint64_t)cap_per_rank(c, fn)) continue;
    pl->oneshot = true;
    pl->vec = true;
    pl->q = 0;
    pl->r = R;
    pl->slice = per_cta;
    pl->nctas = (int)ctas;
    return true;
  }
  return false;
}

// LL one-shot: multi-process only, 8 data bytes per thread and line, the message must fit a
// receive slot (16 bytes per 8 data bytes); not with DDL_CHECK (no barrier to carry the
// signature).  ALGO_LL forces it wherever it fits, AUTO up to ll_max bytes.
// Loopback runs it only when forced (ALGO_LL): all virtual ranks in one cooperative launch,
// so the kernel can be profiled under kernel serialisation; AUTO keeps LL for the cross-GPU
// latency regime it is built for.
bool use_chain(const ddl_comm* c);

bool use_ll(const ddl_comm* c, uint64_t n, ddl_dtype_t dt, Plan* pl) {
  if (c->P < 2 || c->check) return false;
  if (c->loopback && (c->algo != DDL_ALGO_LL || !c->lb_ll)) return false;
  if (c->algo != DDL_ALGO_LL && c->algo != DDL_ALGO_AUTO) return false;
  const uint64_t bytes = n * (uint64_t)elem_size(dt);
  if (c->algo == DDL_ALGO_AUTO && bytes > c->ll_max) return false;
  const uint64_t lines = (bytes + 7) / 8;
  if (lines * 16 > c->ll_slot) return false;
  const void* fn = ll_fn_dt(dt, c->topo.nlive);
  if (!fn) return false;
  uint64_t ctas = (lines + kThreads - 1) / kThreads;  // one line per thread, grid-stride past the cap
  const uint64_t cap = (uint64_t)cap_per_rank(c, fn);
  if (ctas > cap) ctas = cap;
  pl->ll = true;
  pl->oneshot = false;
  pl->q = 0;
  pl->slice = 0;
  pl->nctas = (int)ctas;
  return true;
}

bool use_oneshot(const ddl_comm* c, uint64_t n, ddl_dtype_t dt, Plan* pl) {
  if (c->P < 2 || c->algo == DDL_ALGO_HIER) return false;
  // loopback: the column-chain kernel beats the one-shot at every size (one launch, no
  // barrier; 3.6 vs 13 us at 0.5-1 MiB, profiles/r02c_loopback_sweep.csv): AUTO never picks it
  if (c->algo == DDL_ALGO_AUTO && use_chain(c)) return false;
  if (!c->loopback && n * (uint64_t)elem_size(dt) > c->scratch_half) return false;  // scratch-bound
  if (c->algo == DDL_ALGO_AUTO && n * (uint64_t)elem_size(dt) > c->oneshot_max) return false;
  return plan_oneshot(c, n, dt, pl);
}

KParams base_params(const ddl_comm* c, uint64_t n, ddl_op_t op) {
  KParams p;
  std::memset(&p, 0, sizeof(p));
  p.t = c->topo;
  p.rank = c->rank;
  p.loopback = c->loopback ? 1 : 0;
  p.gpu_scope = (c->gpu_share == c->P && !c->force_sys) ? 1 : 0;
  p.op = op;
  p.cmax = c->cmax;
  p.scale = 1.0f / (float)c->P;  // fl32(1/P)
  p.skip_rank = c->skip_rank;
  p.n = n;
  p.timeout_ns = c->timeout_ns;
  p.err = c->err;
  p.trace = c->trace;
  p.stream_every = c->stream_every;
  p.l2hint = c->l2hint;
  p.deep_copy = c->deep_copy;
  for (int r = 0; r < c->P; ++r) p.flags[r] = c->flags_of(r);
  return p;
}

ddl_result_t launch(const ddl_comm* c, const KParams& p0, const Plan& pl, ddl_dtype_t dt, void* stream) {
  KParams p = p0;
  if (c->check && !c->loopback) {  // FNV-1a over what every rank must agree on
    uint32_t h = 2166136261u;
    const uint64_t vals[] = {p.n, (uint64_t)dt, (uint64_t)p.op, (uint64_t)p.mode, (uint64_t)pl.oneshot,
                             (uint64_t)pl.path, (uint64_t)pl.nctas, p.q, (uint64_t)pl.ll, (uint64_t)pl.nwaves};
    for (uint64_t v : vals)
      for (int b = 0; b < 8; ++b) h = (h ^ (uint32_t)((v >> (8 * b)) & 0xFF)) * 16777619u;
    p.sig = h | 1u;
  }
  const void* fn = pl.ll        ? ll_fn_dt(dt, c->topo.nlive)
                   : pl.oneshot ? oneshot_fn_dt(dt, c->topo.nlive, pl.r)
                                : hier_fn_dt(dt, pl.path);
  if (!fn) return DDL_ERR_UNSUPPORTED;
  if (!pl.oneshot && !pl.ll && pl.slice * (uint64_t)elem_size(dt) > kMaxSliceBytes) return DDL_ERR_TOO_LARGE;
  if (c->nvls_emulate && !pl.oneshot && !pl.ll && pl.vec && pl.path != 7 && (p.mode & (kRS | kAG)) &&
      (p.n * (uint64_t)elem_size(dt)) % 16 == 0) {
    // test hook: the same call through PATH 7 with every live dim's phases "in the switch",
    // emulated by unicast accesses (so the NVLS data flow runs on one GPU)
    Plan pe = pl;
    pe.path = 7;
    pe.nwaves = 1;
    const int cap = cap_per_rank(c, hier_fn_dt(dt, 7), 0);
    if (pe.nctas > cap) {
      const uint64_t W = 16 / elem_size(dt);
      uint64_t slice = (pe.q + cap - 1) / cap;
      slice = (slice + W - 1) / W * W;
      pe.slice = slice;
      pe.nctas = (int)((pe.q + slice - 1) / slice);
      p.slice = slice;
    }
    p.nvls_emulate = 1;
    p.nvls_mask = c->nvls_dims_mask & ((1 << kMaxDims) - 1);
    return launch(c, p, pe, dt, stream);
  }
  p.nwaves = (pl.oneshot || pl.ll) ? 1 : pl.nwaves;
  const size_t smem = (pl.oneshot || pl.ll) ? 0 : hier_smem(pl.path);
  blocks_per_sm(fn, smem);  // sets the dynamic shared-memory attribute once
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  void* args[] = {const_cast<KParams*>(&p)};
  if (c->debug)
    std::fprintf(stderr, "[ddl] %s n=%llu q=%llu slice=%llu ctas=%d waves=%d path=%d mode=%d P=%d loopback=%d\n",
                 pl.ll ? "ll" : pl.oneshot ? "oneshot" : "hier", (unsigned long long)p.n, (unsigned long long)p.q,
                 (unsigned long long)p.slice, pl.nctas, p.nwaves, pl.path, p.mode, c->P, (int)c->loopback);
  if (c->loopback) {
    // hierarchical kernels without the experimental variants: transposed grid (DDL_TRANSPOSE)
    const bool tr = c->transpose && !pl.oneshot && !pl.ll && (pl.path <= 2 || pl.path == 6);
    p.transposed = tr ? 1 : 0;
    DDL_CUDA(launch_ex(fn, tr ? dim3(c->P, pl.nctas) : dim3(pl.nctas, c->P), smem, s, args, true, c->use_pdl));
  } else {
    DDL_CUDA(launch_ex(fn, dim3(pl.nctas), smem, s, args, false, c->use_pdl));
  }
  return DDL_SUCCESS;
}

// ---------------------------------------------------------------- NVLS (ddl_nvls.h)
bool nvls_owns(const ddl_comm* c, const void* buf, size_t bytes) {
  const char* b = static_cast<const char*>(buf);
  return c->nvls.stage == 4 && c->nvls.uc[c->rank] && b >= c->nvls.uc[c->rank] &&
         b + bytes <= c->nvls.uc[c->rank] + c->nvls.bytes;
}

// An all-reduce of a buffer inside the NVLS region: the hierarchical schedule with the
// switch running the phases of the dims in nvls.mask (PATH 7), zero-copy through every
// rank's unicast mapping of its NVLS memory; the one-shot / LL regimes and counts that are
// not whole 16-B vectors keep the direct kernels on the same mappings.
ddl_result_t nvls_allreduce(const ddl_comm* c, KParams& p, void* buf, size_t count, ddl_dtype_t dt, void* stream) {
  const size_t off = (size_t)(static_cast<char*>(buf) - c->nvls.uc[c->rank]);
  const int w = elem_size(dt);
  Plan pl;
  const bool one = use_oneshot(c, count, dt, &pl);
  const bool vec = (count * (size_t)w) % 16 == 0;
  if (!one) {
    pl = plan_hier(c, count, block_elems(count, c->P, w), dt, true);
    if (vec && c->nvls.mask) {  // PATH 7: register-staged kernel with the NVLS phases compiled in
      pl.path = 7;
      pl.nwaves = 1;
      const int cap = cap_per_rank(c, hier_fn_dt(dt, 7), 0);
      if (pl.nctas > cap) {
        uint64_t slice = (pl.q + cap - 1) / cap;
        slice = (slice + 16 / w - 1) / (16 / w) * (16 / w);
        pl.slice = slice;
        pl.nctas = (int)((pl.q + slice - 1) / slice);
      }
      for (int d = 0; d < c->topo.k; ++d) p.mc[d] = c->nvls.mcva[d] ? c->nvls.mcva[d] + off : nullptr;
      p.nvls_mask = c->nvls.mask;
    }
  }
  p.q = pl.q;
  p.slice = pl.slice;
  for (int m = 0; m < c->P; ++m) {
    char* base = c->nvls.uc[m] + off;
    p.in[m] = base;
    p.work[m] = base;
    p.out[m] = base;
  }
  if (one) {  // inputs published through the scratch halves, as for any one-shot call
    p.mode = kScratch;
    p.cin[c->rank] = buf;
    p.out[c->rank] = buf;
    for (int m = 0; m < c->P; ++m) p.scratch[m] = c->scratch_of(m);
    p.scratch_half = c->scratch_half;
  } else {
    p.mode = kRS | kAG;
  }
  return launch(c, p, pl, dt, stream);
}

// ---------------------------------------------------------------- loopback column-chain kernel
// (ddl_chain.cuh) The loopback all-reduce (single or grouped) as independent columns, each
// running the whole schedule in one thread.  Not used with the debug hooks that need the
// slice kernels' barriers (skip_rank, trace), the NVLS emulation or the experiment variants.
bool use_chain(const ddl_comm* c) {
  return c->loopback && c->lb_chain && c->skip_rank < 0 && !c->trace && !c->nvls_emulate && !c->use_dyn &&
         !c->use_steal && !c->use_stream;
}

// Column-chain kernels: a compile-time-topology kernel (rows of P columns) for the live-dim
// sequences of P = 2, 4, 8; the generic kernel (one column per thread) otherwise (at P = 16
// the compile-time kernel's P-wide register arrays spill).
template <typename T>
const void* chain_ct_t(const Topo& t) {
  int g[4] = {1, 1, 1, 1};
  const int L = t.nlive;
  if (L < 1 || L > 4) return nullptr;
  for (int l = 0; l < L; ++l) g[l] = t.g[t.live[l]];
#define DDL_CT(L_, a, b, c, d)                                               \
  if (L == L_ && g[0] == a && g[1] == b && g[2] == c && g[3] == d)          \
    return (const void*)ddl_chain_ct_kernel<T, CT<L_, a, b, c, d>>;
  DDL_CT(1, 2, 1, 1, 1)
  DDL_CT(1, 4, 1, 1, 1) DDL_CT(2, 2, 2, 1, 1)
  DDL_CT(1, 8, 1, 1, 1) DDL_CT(2, 4, 2, 1, 1) DDL_CT(2, 2, 4, 1, 1) DDL_CT(3, 2, 2, 2, 1)
#undef DDL_CT
  return nullptr;
}
template <typename T>
const void* chain_tma_t(const Topo& t) {
  int g[4] = {1, 1, 1, 1};
  const int L = t.nlive;
  if (L < 1 || L > 4) return nullptr;
  for (int l = 0; l < L; ++l) g[l] = t.g[t.live[l]];
#define DDL_CT(L_, a, b, c, d)                                               \
  if (L == L_ && g[0] == a && g[1] == b && g[2] == c && g[3] == d)          \
    return (const void*)ddl_chain_tma_kernel<T, CT<L_, a, b, c, d>>;
  DDL_CT(1, 2, 1, 1, 1)
  DDL_CT(1, 4, 1, 1, 1) DDL_CT(2, 2, 2, 1, 1)
  DDL_CT(1, 8, 1, 1, 1) DDL_CT(2, 4, 2, 1, 1) DDL_CT(2, 2, 4, 1, 1) DDL_CT(3, 2, 2, 2, 1)
#undef DDL_CT
  return nullptr;
}
const void* chain_tma_dt(ddl_dtype_t dt, const Topo& t) {
  if (dt == DDL_INT32) return chain_tma_t<int32_t>(t);
  if (dt == DDL_FLOAT32) return chain_tma_t<float>(t);
  return chain_tma_t<__nv_bfloat16>(t);
}

template <typename T>
const void* chain_fn_t(const Topo& t, bool generic, bool* ct) {
  if (!generic) {
    if (const void* f = chain_ct_t<T>(t)) {
      *ct = true;
      return f;
    }
  }
  *ct = false;
  if (t.P <= 4) return (const void*)ddl_chain_kernel<T, 4>;
  if (t.P <= 8) return (const void*)ddl_chain_kernel<T, 8>;
  return (const void*)ddl_chain_kernel<T, 16>;
}
const void* chain_fn_dt(ddl_dtype_t dt, const Topo& t, bool generic, bool* ct) {
  if (dt == DDL_INT32) return chain_fn_t<int32_t>(t, generic, ct);
  if (dt == DDL_FLOAT32) return chain_fn_t<float>(t, generic, ct);
  return chain_fn_t<__nv_bfloat16>(t, generic, ct);
}

// Buffers i < nb with counts ns[i] and every rank's pointer ptrs[i * P + m]: their columns
// (P blocks of q / W vectors each) concatenated, at most kMaxBuckets buffers and 2^31 columns
// per launch; one persistent grid (resident CTAs x SMs) walks them grid-stride.
ddl_result_t launch_chain(const ddl_comm* c, const uint64_t* ns, void* const* ptrs, int nb, ddl_dtype_t dt,
                                 ddl_op_t op, void* stream) {
  bool ct = false;
  const void* fn = chain_fn_dt(dt, c->topo, c->chain_generic, &ct);
  // TMA-fed variant of the compile-time-topology kernel (DDL_CHAIN_TMA)
  const bool tma = c->chain_tma > 0 || (c->chain_tma < 0 && c->P >= 4);
  const void* tfn = (ct && tma) ? chain_tma_dt(dt, c->topo) : nullptr;
  const size_t tsmem = chain_tma_smem(c->P);
  if (tfn) fn = tfn;
  const int w = elem_size(dt);
  const uint64_t W = 16 / w;
  const uint64_t kMaxCols = 1ull << 31;
  // every buffer must fit one launch's 31-bit column / row space: refuse before enqueuing any
  for (int j = 0; j < nb; ++j)
    if ((uint64_t)c->P * (block_elems(ns[j], c->P, w) / W) > kMaxCols) return DDL_ERR_TOO_LARGE;
  int i = 0;
  while (i < nb) {
    CParams cp;
    std::memset(&cp, 0, sizeof(cp));
    cp.t = c->topo;
    cp.op = op;
    cp.scale = 1.0f / (float)c->P;  // fl32(1/P)
    uint64_t cols = 0, rows = 0;
    while (i < nb && cp.nb < kMaxBuckets) {
      const uint64_t n = ns[i];
      const uint64_t q = block_elems(n, c->P, w);
      const uint64_t vq = q / W;
      // CT kernels: rows v < vfull have a whole vector in every block (the last block holds
      // n - (P-1) q elements); the other rows' columns go through the generic column code
      const uint64_t last = n > (uint64_t)(c->P - 1) * q ? n - (uint64_t)(c->P - 1) * q : 0;
      const uint64_t vfull = ct ? std::min<uint64_t>(vq, last / W) : 0;
      const uint64_t bc = (uint64_t)c->P * (vq - vfull);
      if (bc > kMaxCols || vfull > kMaxCols) return DDL_ERR_TOO_LARGE;
      if (cols + bc > kMaxCols || rows + vfull > kMaxCols) break;
      CBucket& B = cp.b[cp.nb++];
      B.n = n;
      B.q = q;
      B.vq = (uint32_t)vq;
      B.vfull = (uint32_t)vfull;
      B.col0 = (uint32_t)cols;
      B.row0 = (uint32_t)rows;
      for (int m = 0; m < c->P; ++m) B.buf[m] = static_cast<char*>(ptrs[(size_t)i * c->P + m]);
      cols += bc;
      rows += vfull;
      ++i;
    }
    cp.ncols = (uint32_t)cols;
    cp.nrows = (uint32_t)rows;
    if (!cols && !rows) continue;
    const int threads = tfn ? kTmaCons + 32 : kChainThreads;
    const size_t smem = tfn ? tsmem : 0;
    const uint64_t need = tfn ? (uint64_t)c->P * ((rows + kTmaCons - 1) / kTmaCons + cp.nb)
                              : (std::max(rows, ct ? 0 : cols) + kChainThreads - 1) / kChainThreads;
    const uint64_t cap = (uint64_t)blocks_per_sm(fn, smem, threads) * c->num_sms;
    const int grid = (int)std::max<uint64_t>(1, std::min(need, c->ctas_limit > 0 ? (uint64_t)c->ctas_limit : cap));
    if (c->debug)
      std::fprintf(stderr, "[ddl] chain (%s): %d buffers, %llu full rows, %llu tail columns, grid %d\n",
                   tfn ? "tma" : ct ? "ct" : "generic", cp.nb, (unsigned long long)rows, (unsigned long long)cols, grid);
    void* args[] = {&cp};
    DDL_CUDA(launch_ex(fn, dim3(grid), smem, static_cast<cudaStream_t>(stream), args, false, c->use_pdl, threads));
  }
  return DDL_SUCCESS;
}

ddl_result_t check_common(const ddl_comm* c, ddl_dtype_t dt, ddl_op_t op) {
  if (!c) return DDL_ERR_INVALID_ARGUMENT;
  if (!valid_dtype(dt) || (op != DDL_SUM && op != DDL_AVG)) return DDL_ERR_INVALID_ARGUMENT;
  if (dt == DDL_INT32 && op == DDL_AVG) return DDL_ERR_UNSUPPORTED;
  if (!c->loopback && !c->connected && c->P > 1) return DDL_ERR_NOT_CONNECTED;
  return DDL_SUCCESS;
}

// If [ptr, ptr+bytes) lies in the symmetric buffer or in a registered buffer, fill peer[m]
// with every rank's address of the same offset and return true (zero-copy).
bool zero_copy_peers(const ddl_comm* c, const void* ptr, size_t bytes, const char** peer) {
  const char* q = static_cast<const char*>(ptr);
  const char* sym = c->alloc + c->flags_bytes;
  if (q >= sym && q + bytes <= sym + c->max_bytes) {
    for (int m = 0; m < c->P; ++m) peer[m] = c->sym_of(m) + (q - sym);
    return true;
  }
  for (int k = 0; k < ddl_comm::kMaxRegs; ++k) {
    const ddl_comm::Reg& g = c->regs[k];
    if (g.used && q >= g.local && q + bytes <= g.local + g.bytes) {
      for (int m = 0; m < c->P; ++m) peer[m] = g.peer[m] + (q - g.local);
      return true;
    }
  }
  return false;
}

// Local copy (P = 1 reduce-scatter / allgather) through the local-reduce kernel.
ddl_result_t local_copy(const void* src, void* dst, size_t count, ddl_dtype_t dt, void* stream) {
  if (src == dst || count == 0) return DDL_SUCCESS;
  const void* ins[1] = {src};
  return ddl_local_reduce(ins, 1, dst, count, dt, 1.0f, stream);
}

}  // namespace

extern "C" {

int ddl_version(void) { return 103; }  // 1.03: loopback LL, ddl_peer_buffer, ddl_build_flags
int ddl_build_flags(void) { return DDL_EXPERIMENTAL ? 1 : 0; }

const char* ddl_result_string(ddl_result_t r) {
  switch (r) {
    case DDL_SUCCESS: return "success";
    case DDL_ERR_INVALID_ARGUMENT: return "invalid argument";
    case DDL_ERR_BAD_DIMS: return "bad dims (product != nranks, g < 1 or too many dims)";
    case DDL_ERR_UNSUPPORTED: return "unsupported";
    case DDL_ERR_CUDA: return "CUDA error";
    case DDL_ERR_NO_PEER_ACCESS: return "no peer access";
    case DDL_ERR_NOT_CONNECTED: return "not connected";
    case DDL_ERR_TOO_LARGE: return "message larger than the workspace";
    case DDL_ERR_TIMEOUT: return "device barrier timeout";
    case DDL_ERR_MISMATCH: return "ranks disagree (handles at connect, or the call signature with DDL_CHECK=1)";
  }
  return "unknown";
}

const char* ddl_last_error_string(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------------ planner queries
ddl_result_t ddl_check_dims(int nranks, const int* dims, int ndims) {
  if (!dims) return DDL_ERR_INVALID_ARGUMENT;
  Topo t;
  return make_topo(&t, nranks, dims, ndims) ? DDL_ERR_BAD_DIMS : DDL_SUCCESS;
}

size_t ddl_block_elems(size_t count, int nranks, ddl_dtype_t dtype) {
  if (nranks < 1 || !valid_dtype(dtype)) return 0;
  return (size_t)block_elems(count, nranks, elem_size(dtype));
}

ddl_result_t ddl_plan_group(int nranks, const int* dims, int ndims, int rank, int d, int* members_out) {
  Topo t;
  if (!dims || !members_out) return DDL_ERR_INVALID_ARGUMENT;
  if (make_topo(&t, nranks, dims, ndims)) return DDL_ERR_BAD_DIMS;
  if (rank < 0 || rank >= nranks || d < 0 || d >= ndims) return DDL_ERR_INVALID_ARGUMENT;
  for (int v = 0; v < t.g[d]; ++v) members_out[v] = member(t, rank, d, v);
  return DDL_SUCCESS;
}

ddl_result_t ddl_plan_blocks(int nranks, const int* dims, int ndims, int rank, int d, int* blocks_out,
                             int* nblocks_out) {
  Topo t;
  if (!dims || !blocks_out || !nblocks_out) return DDL_ERR_INVALID_ARGUMENT;
  if (make_topo(&t, nranks, dims, ndims)) return DDL_ERR_BAD_DIMS;
  if (rank < 0 || rank >= nranks || d < 0 || d > ndims) return DDL_ERR_INVALID_ARGUMENT;
  *nblocks_out = nblocks(t, d);
  for (int i = 0; i < *nblocks_out; ++i) blocks_out[i] = block_of(t, rank, d, i);
  return DDL_SUCCESS;
}

ddl_result_t ddl_plan_barriers(int nranks, const int* dims, int ndims, int rank, int* peers_out,
                               int* counts_out, int* nbarriers_out) {
  Topo t;
  if (!dims || !peers_out || !counts_out || !nbarriers_out) return DDL_ERR_INVALID_ARGUMENT;
  if (make_topo(&t, nranks, dims, ndims)) return DDL_ERR_BAD_DIMS;
  if (rank < 0 || rank >= nranks) return DDL_ERR_INVALID_ARGUMENT;
  const int nb = t.nlive ? 2 * t.nlive + 1 : 0;
  *nbarriers_out = nb;
  for (int j = 0; j < nb; ++j) {
    counts_out[j] = barrier_npeers(t, j);
    for (int l = 0; l < counts_out[j]; ++l) peers_out[j * nranks + l] = barrier_peer(t, rank, j, l);
  }
  return DDL_SUCCESS;
}

ddl_result_t ddl_plan_traffic(size_t count, ddl_dtype_t dtype, int nranks, const int* dims, int ndims, int rank,
                              uint64_t* rs_out, uint64_t* ag_out) {
  Topo t;
  if (!dims || !rs_out || !ag_out || !valid_dtype(dtype)) return DDL_ERR_INVALID_ARGUMENT;
  if (make_topo(&t, nranks, dims, ndims)) return DDL_ERR_BAD_DIMS;
  if (rank < 0 || rank >= nranks) return DDL_ERR_INVALID_ARGUMENT;
  const int w = elem_size(dtype);
  const uint64_t n = count, q = block_elems(count, nranks, w);
  auto len = [&](int b) -> uint64_t {
    const uint64_t lo = (uint64_t)b * q < n ? (uint64_t)b * q : n;
    const uint64_t hi = (uint64_t)(b + 1) * q < n ? (uint64_t)(b + 1) * q : n;
    return hi - lo;
  };
  for (int d = 0; d < ndims; ++d) {
    rs_out[d] = ag_out[d] = 0;
    if (t.g[d] == 1) continue;
    for (int i = 0; i < nblocks(t, d + 1); ++i)
      rs_out[d] += (uint64_t)(t.g[d] - 1) * len(block_of(t, rank, d + 1, i)) * w;
    for (int v = 0; v < t.g[d]; ++v) {
      const int m = member(t, rank, d, v);
      if (m == rank) continue;
      for (int i = 0; i < nblocks(t, d + 1); ++i) ag_out[d] += len(block_of(t, m, d + 1, i)) * w;
    }
  }
  return DDL_SUCCESS;
}

// ------------------------------------------------------------------ multi-process comm
ddl_result_t ddl_init(ddl_comm_t* comm, int rank, int nranks, const int* dims, int ndims, int cuda_device,
                      size_t max_bytes) {
  if (!comm || rank < 0 || rank >= nranks) return DDL_ERR_INVALID_ARGUMENT;
  *comm = nullptr;
  DeviceGuard guard(cuda_device < 0 ? 0 : cuda_device);
  ddl_comm* c = new (std::nothrow) ddl_comm();
  if (!c) return DDL_ERR_CUDA;
  ddl_result_t r = common_init(c, nranks, dims, ndims, cuda_device);
  if (r != DDL_SUCCESS) {
    delete c;
    return r;
  }
  c->rank = rank;
  c->max_bytes = (max_bytes + 4095) / 4096 * 4096;
  c->scratch_half = ((c->oneshot_max > (512u << 10) ? c->oneshot_max : (512u << 10)) + 4095) / 4096 * 4096;
  c->ll_slot = (2 * c->ll_max + 4095) / 4096 * 4096;  // 16 bytes per 8 data bytes
  c->alloc_bytes = c->flags_bytes + 2 * c->max_bytes + 2 * c->scratch_half + 2 * (size_t)nranks * c->ll_slot;
  cudaError_t e = cudaMalloc(&c->alloc, c->alloc_bytes);
  if (e == cudaSuccess) e = cudaMemset(c->alloc, 0, c->flags_bytes);
  // LL words carry the call epoch (>= 1): the region must start with none that could match
  if (e == cudaSuccess && c->ll_slot) e = cudaMemset(c->ll_of(rank), 0, 2 * (size_t)nranks * c->ll_slot);
  if (e == cudaSuccess) e = cudaMalloc(&c->err, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->err, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (c->alloc) cudaFree(c->alloc);
    if (c->err) cudaFree(c->err);
    delete c;
    return cuda_fail(e, "ddl_init allocation");
  }
  c->connected = (nranks == 1);
  *comm = c;
  return DDL_SUCCESS;
}

size_t ddl_handle_size(void) { return sizeof(Handle); }

ddl_result_t ddl_export_handle(ddl_comm_t c, void* out) {
  if (!c || !out || c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  Handle h;
  std::memset(&h, 0, sizeof(h));
  h.magic = kMagic;
  h.rank = c->rank;
  h.nranks = c->P;
  h.ndims = c->ndims;
  for (int d = 0; d < c->ndims; ++d) h.dims[d] = c->dims[d];
  h.cmax = c->cmax;
  h.flags_bytes = c->flags_bytes;
  h.max_bytes = c->max_bytes;
  h.scratch_half = c->scratch_half;
  h.ll_slot = c->ll_slot;
  h.alloc_bytes = c->alloc_bytes;
  DDL_ON_DEVICE(c->device);
  DDL_CUDA(cudaDeviceGetPCIBusId(h.pci, sizeof(h.pci), c->device));
  DDL_CUDA(cudaIpcGetMemHandle(&h.ipc, c->alloc));
  std::memcpy(out, &h, sizeof(h));
  return DDL_SUCCESS;
}

ddl_result_t ddl_connect(ddl_comm_t c, const void* all_handles) {
  if (!c || !all_handles || c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  if (c->connected) return DDL_SUCCESS;
  DDL_ON_DEVICE(c->device);
  const Handle* hs = static_cast<const Handle*>(all_handles);
  for (int m = 0; m < c->P; ++m) {
    const Handle& h = hs[m];
    if (h.magic != kMagic || h.rank != m) return DDL_ERR_INVALID_ARGUMENT;
    if (h.nranks != c->P || h.ndims != c->ndims || h.cmax != c->cmax || h.flags_bytes != c->flags_bytes ||
        h.max_bytes != c->max_bytes || h.scratch_half != c->scratch_half || h.ll_slot != c->ll_slot)
      return DDL_ERR_MISMATCH;
    for (int d = 0; d < c->ndims; ++d)
      if (h.dims[d] != c->dims[d]) return DDL_ERR_MISMATCH;
  }
  for (int m = 0; m < c->P; ++m) {
    if (m == c->rank) continue;
    const Handle& h = hs[m];
    int pdev = -1;
    if (cudaDeviceGetByPCIBusId(&pdev, h.pci) == cudaSuccess && pdev != c->device) {
      int ok = 0;
      DDL_CUDA(cudaDeviceCanAccessPeer(&ok, c->device, pdev));
      if (!ok) return DDL_ERR_NO_PEER_ACCESS;
    }
    cudaGetLastError();
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h.ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    c->peer_base[m] = static_cast<char*>(ptr);
    c->peer_mapped[m] = true;
  }
  c->connected = true;
  return DDL_SUCCESS;
}

// ------------------------------------------------------------------ NVLS setup rounds
size_t ddl_nvls_blob_size(void) { return sizeof(nvls::Blob); }

// Self-test of the NVLS descriptor exchange (no GPU): two "ranks" in this process, each with
// an fd server, send each other two descriptors (a pipe's ends) over the abstract Unix
// sockets; the received descriptors must refer to the same pipe.  Returns 0 on success.
int ddl_debug_nvls_fd_selftest(void) {
  char name[2][64];
  const int srv[2] = {nvls::fd_server_open(name[0], 0), nvls::fd_server_open(name[1], 1)};
  if (srv[0] < 0 || srv[1] < 0) return 1;
  int pfd[2];
  if (pipe(pfd) != 0) return 2;
  std::vector<std::vector<int>> got0(2, std::vector<int>(kMaxDims + 1, -1)), got1 = got0;
  bool ok0 = false, ok1 = false;
  std::thread t0([&] { ok0 = nvls::fd_recv_all(srv[0], 1, 5000, &got0); });
  std::thread t1([&] { ok1 = nvls::fd_recv_all(srv[1], 1, 5000, &got1); });
  const bool s0 = nvls::fd_send(name[1], 0, {0, 3}, {pfd[0], pfd[1]});  // rank 0 -> rank 1
  const bool s1 = nvls::fd_send(name[0], 1, {0}, {pfd[1]});             // rank 1 -> rank 0
  t0.join();
  t1.join();
  int rc = (ok0 && ok1 && s0 && s1) ? 0 : 3;
  if (!rc) {  // write through the received write end, read through the received read end
    const char msg = 'x';
    char back = 0;
    if (write(got1[0][3], &msg, 1) != 1 || read(got1[0][0], &back, 1) != 1 || back != 'x') rc = 4;
    if (!rc && (write(got0[1][0], &msg, 1) != 1 || read(pfd[0], &back, 1) != 1)) rc = 5;
  }
  for (auto* g : {&got0, &got1})
    for (auto& v : *g)
      for (int fd : v)
        if (fd >= 0) close(fd);
  close(pfd[0]);
  close(pfd[1]);
  close(srv[0]);
  close(srv[1]);
  return rc;
}

static nvls::Blob* blob_of(const void* all, int r) {
  return reinterpret_cast<nvls::Blob*>(const_cast<char*>(static_cast<const char*>(all)) + (size_t)r * sizeof(nvls::Blob));
}
static void blob_init(ddl_comm* c, nvls::Blob* b) {
  std::memset(b, 0, sizeof(*b));
  b->magic = nvls::kBlobMagic;
  b->rank = c->rank;
  b->pid = (int32_t)getpid();
  b->phys_fd = -1;
  for (int d = 0; d < kMaxDims; ++d) b->mc_fd[d] = -1;
}
// every rank's blob of this round is well-formed and OK
static bool all_ok(const ddl_comm* c, const void* all) {
  for (int r = 0; r < c->P; ++r) {
    const nvls::Blob* b = blob_of(all, r);
    if (b->magic != nvls::kBlobMagic || b->rank != r || b->status != nvls::kOk) return false;
  }
  return true;
}

ddl_result_t ddl_nvls_prepare(ddl_comm_t c, size_t bytes, void* out) {
  if (!c || !out || c->loopback || !c->connected || bytes == 0) return DDL_ERR_INVALID_ARGUMENT;
  DDL_ON_DEVICE(c->device);
  nvls::Blob* b = static_cast<nvls::Blob*>(out);
  blob_init(c, b);
  nvls::teardown(c->nvls, c->topo, c->rank);
  nvls::State& s = c->nvls;
  s.dev = c->device;
  nvls::Api& a = nvls::api();
  if (!a.ok || c->P < 2) { b->status = nvls::kNoApi; return DDL_SUCCESS; }
  int mcs = 0;
  if (a.deviceGet(&s.cudev, c->device) != CUDA_SUCCESS ||
      a.getAttr(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, s.cudev) != CUDA_SUCCESS || !mcs) {
    b->status = nvls::kNoMulticast;
    return DDL_SUCCESS;
  }
  // granularity: the multicast granularity for the largest group, and the allocation one
  size_t gran = 2u << 20;
  for (int li = 0; li < c->topo.nlive; ++li) {
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.numDevices = (unsigned)c->topo.g[c->topo.live[li]];
    mp.size = bytes;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t g = 0;
    // the minimum granularity (2 MiB here): the recommended one is 512 MiB per rank
    if (a.mcGranularity(&g, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) == CUDA_SUCCESS && g > gran) gran = g;
  }
  {  // and the physical allocation's granularity
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = c->device;
    size_t g = 0;
    if (a.memGranularity(&g, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM) == CUDA_SUCCESS && g > gran) gran = g;
  }
  s.gran = gran;
  s.bytes = (bytes + gran - 1) / gran * gran;
  b->bytes = s.bytes;
  // this rank's NVLS memory: exportable by fabric handle if creation AND export work (a
  // fabric export needs the fabric manager / IMEX service), else by file descriptor.  The
  // handle type must be the same on every rank: attach checks it.
  const bool no_fabric = env_size("DDL_NVLS_NO_FABRIC", 0) != 0;
  for (CUmemAllocationHandleType ht : {CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR}) {
    if (ht == CU_MEM_HANDLE_TYPE_FABRIC && no_fabric) continue;
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = c->device;
    ap.requestedHandleTypes = ht;
    if (a.memCreate(&s.phys, s.bytes, &ap, 0) != CUDA_SUCCESS) {
      s.phys = 0;
      continue;
    }
    bool ok;
    if (ht == CU_MEM_HANDLE_TYPE_FABRIC) {
      ok = a.memExport(&b->phys_fab, s.phys, ht, 0) == CUDA_SUCCESS;
    } else {
      int fd = -1;
      ok = a.memExport(&fd, s.phys, ht, 0) == CUDA_SUCCESS;
      s.phys_fd = fd;
      b->phys_fd = fd;
    }
    if (ok) {
      s.htype = ht;
      break;
    }
    a.memRelease(s.phys);
    s.phys = 0;
  }
  if (!s.phys) { b->status = nvls::kAllocFailed; return DDL_SUCCESS; }
  b->htype = (int32_t)s.htype;
  if (s.htype == CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) {  // descriptors travel over a socket
    s.server = nvls::fd_server_open(b->sock, c->rank);
    if (s.server < 0) { b->status = nvls::kAllocFailed; return DDL_SUCCESS; }
  }
  // the multicast object of every live dim whose group I lead (c_d = 0)
  for (int li = 0; li < c->topo.nlive; ++li) {
    const int d = c->topo.live[li];
    if (coord(c->topo, c->rank, d) != 0) continue;
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.numDevices = (unsigned)c->topo.g[d];
    mp.size = s.bytes;
    mp.handleTypes = s.htype;
    if (a.mcCreate(&s.mc[d], &mp) != CUDA_SUCCESS) { s.mc[d] = 0; b->status = nvls::kCreateFailed; return DDL_SUCCESS; }
    if (s.htype == CU_MEM_HANDLE_TYPE_FABRIC) {
      if (a.memExport(&b->mc_fab[d], s.mc[d], s.htype, 0) != CUDA_SUCCESS) { b->status = nvls::kCreateFailed; return DDL_SUCCESS; }
    } else {
      int fd = -1;
      if (a.memExport(&fd, s.mc[d], s.htype, 0) != CUDA_SUCCESS) { b->status = nvls::kCreateFailed; return DDL_SUCCESS; }
      s.mc_fd[d] = fd;
      b->mc_fd[d] = fd;
    }
  }
  s.stage = 1;
  b->status = nvls::kOk;
  return DDL_SUCCESS;
}

ddl_result_t ddl_nvls_attach(ddl_comm_t c, const void* all, void* out) {
  if (!c || !all || !out || c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  DDL_ON_DEVICE(c->device);
  nvls::Blob* b = static_cast<nvls::Blob*>(out);
  blob_init(c, b);
  nvls::State& s = c->nvls;
  nvls::Api& a = nvls::api();
  if (s.stage != 1 || !all_ok(c, all)) { b->status = nvls::kPeerFailed; return DDL_SUCCESS; }
  for (int r = 0; r < c->P; ++r)
    if (blob_of(all, r)->bytes != s.bytes || blob_of(all, r)->htype != (int32_t)s.htype) {
      b->status = nvls::kPeerFailed;
      return DDL_SUCCESS;
    }
  // POSIX fds: every rank sends its memory's descriptor (and those of the multicast objects it
  // leads) to every peer while a thread receives the peers' -- all inside this round
  if (s.htype == CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) {
    s.rx.assign(c->P, std::vector<int>(kMaxDims + 1, -1));
    bool rx_ok = false;
    std::thread rx([&] { rx_ok = nvls::fd_recv_all(s.server, c->P - 1, 30000, &s.rx); });
    std::vector<int> tags{0}, fds{s.phys_fd};
    for (int li = 0; li < c->topo.nlive; ++li) {
      const int d = c->topo.live[li];
      if (s.mc_fd[d] >= 0) {
        tags.push_back(1 + d);
        fds.push_back(s.mc_fd[d]);
      }
    }
    bool tx_ok = true;
    for (int m = 0; m < c->P; ++m)
      if (m != c->rank) tx_ok = nvls::fd_send(blob_of(all, m)->sock, c->rank, tags, fds) && tx_ok;
    rx.join();
    if (!rx_ok || !tx_ok) { b->status = nvls::kImportFailed; return DDL_SUCCESS; }
  }
  auto rx_fd = [&](int m, int tag) { return s.rx.empty() ? -1 : s.rx[m][tag]; };
  // unicast mappings: my memory and every peer's
  if (nvls::map_rw(s.phys, s.bytes, s.gran, c->device, &s.uc[c->rank]) != CUDA_SUCCESS) { b->status = nvls::kMapFailed; return DDL_SUCCESS; }
  for (int m = 0; m < c->P; ++m) {
    if (m == c->rank) continue;
    const nvls::Blob* pb = blob_of(all, m);
    if (nvls::import_handle(&s.peer_phys[m], s.htype, rx_fd(m, 0), &pb->phys_fab) != CUDA_SUCCESS) {
      s.peer_phys[m] = 0;
      b->status = nvls::kImportFailed;
      return DDL_SUCCESS;
    }
    if (nvls::map_rw(s.peer_phys[m], s.bytes, s.gran, c->device, &s.uc[m]) != CUDA_SUCCESS) { b->status = nvls::kMapFailed; return DDL_SUCCESS; }
  }
  // join every live dim's group multicast object
  for (int li = 0; li < c->topo.nlive; ++li) {
    const int d = c->topo.live[li];
    const int lead = member(c->topo, c->rank, d, 0);
    if (lead != c->rank) {
      const nvls::Blob* lb = blob_of(all, lead);
      if (nvls::import_handle(&s.mc[d], s.htype, rx_fd(lead, 1 + d), &lb->mc_fab[d]) != CUDA_SUCCESS) {
        s.mc[d] = 0;
        b->status = nvls::kImportFailed;
        return DDL_SUCCESS;
      }
    }
    if (a.mcAddDevice(s.mc[d], s.cudev) != CUDA_SUCCESS) { b->status = nvls::kAddFailed; return DDL_SUCCESS; }
    s.mc_added[d] = true;
  }
  s.stage = 2;
  b->status = nvls::kOk;
  return DDL_SUCCESS;
}

ddl_result_t ddl_nvls_bind(ddl_comm_t c, const void* all, void* out) {
  if (!c || !all || !out || c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  DDL_ON_DEVICE(c->device);
  nvls::Blob* b = static_cast<nvls::Blob*>(out);
  blob_init(c, b);
  nvls::State& s = c->nvls;
  nvls::Api& a = nvls::api();
  if (s.stage != 2 || !all_ok(c, all)) { b->status = nvls::kPeerFailed; return DDL_SUCCESS; }
  for (int li = 0; li < c->topo.nlive; ++li) {  // every member has added its device: bind and map
    const int d = c->topo.live[li];
    if (a.mcBindMem(s.mc[d], 0, s.phys, 0, s.bytes, 0) != CUDA_SUCCESS) { b->status = nvls::kBindFailed; return DDL_SUCCESS; }
    s.mc_bound[d] = true;
    if (nvls::map_rw(s.mc[d], s.bytes, s.gran, c->device, &s.mcva[d]) != CUDA_SUCCESS) { b->status = nvls::kMapFailed; return DDL_SUCCESS; }
  }
  s.stage = 3;
  b->status = nvls::kOk;
  return DDL_SUCCESS;
}

ddl_result_t ddl_nvls_commit(ddl_comm_t c, const void* all) {
  if (!c || !all || c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  DDL_ON_DEVICE(c->device);
  nvls::State& s = c->nvls;
  if (s.stage != 3 || !all_ok(c, all)) {
    nvls::teardown(s, c->topo, c->rank);
    return DDL_ERR_UNSUPPORTED;
  }
  DDL_CUDA(cudaMemset(s.uc[c->rank], 0, s.bytes));
  DDL_CUDA(cudaDeviceSynchronize());
  s.mask = 0;
  for (int li = 0; li < c->topo.nlive; ++li) {
    const int d = c->topo.live[li];
    if (c->nvls_dims_mask & (1 << d)) s.mask |= 1 << d;
  }
  s.stage = 4;
  return DDL_SUCCESS;
}

ddl_result_t ddl_nvls_buffer(ddl_comm_t c, void** dev_ptr, size_t* bytes, int* dims_mask) {
  if (!c || !dev_ptr || !bytes || c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  if (c->nvls.stage != 4) return DDL_ERR_UNSUPPORTED;
  *dev_ptr = c->nvls.uc[c->rank];
  *bytes = c->nvls.bytes;
  if (dims_mask) *dims_mask = c->nvls.mask;
  return DDL_SUCCESS;
}

ddl_result_t ddl_peer_buffer(ddl_comm_t c, int peer, void** dev_ptr, size_t* bytes) {
  if (!c || !dev_ptr || !bytes || c->loopback || peer < 0 || peer >= c->P) return DDL_ERR_INVALID_ARGUMENT;
  if (peer != c->rank && !c->peer_mapped[peer]) return DDL_ERR_NOT_CONNECTED;
  *dev_ptr = c->sym_of(peer);
  *bytes = c->max_bytes;
  return DDL_SUCCESS;
}

ddl_result_t ddl_peer_copy(ddl_comm_t c, int peer, size_t src_offset, size_t dst_offset, size_t bytes, void* stream) {
  if (!c || c->loopback || peer < 0 || peer >= c->P) return DDL_ERR_INVALID_ARGUMENT;
  if (src_offset + bytes > c->max_bytes || dst_offset + bytes > c->max_bytes) return DDL_ERR_TOO_LARGE;
  if (peer != c->rank && !c->peer_mapped[peer]) return DDL_ERR_NOT_CONNECTED;
  DDL_ON_DEVICE(c->device);
  DDL_CUDA(cudaMemcpyAsync(c->sym_of(peer) + dst_offset, c->sym_of(c->rank) + src_offset, bytes,
                           cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  return DDL_SUCCESS;
}

ddl_result_t ddl_buffer(ddl_comm_t c, void** dev_ptr, size_t* bytes) {
  if (!c || !dev_ptr || !bytes || c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  *dev_ptr = c->alloc + c->flags_bytes;
  *bytes = c->max_bytes;
  return DDL_SUCCESS;
}

ddl_result_t ddl_allreduce(ddl_comm_t c, void* buf, size_t count, ddl_dtype_t dt, ddl_op_t op, void* stream) {
  ddl_result_t r = check_common(c, dt, op);
  if (r != DDL_SUCCESS) return r;
  if (c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  if (count == 0 || c->P == 1) return DDL_SUCCESS;
  if (!buf || !aligned16(buf)) return DDL_ERR_INVALID_ARGUMENT;
  const size_t bytes = count * elem_size(dt);
  char* sym = c->alloc + c->flags_bytes;
  const bool in_sym = (char*)buf >= sym && (char*)buf + bytes <= sym + c->max_bytes;
  const ddl_comm::Reg* reg = nullptr;
  for (int k = 0; k < ddl_comm::kMaxRegs && !in_sym && !reg; ++k) {
    const ddl_comm::Reg& g = c->regs[k];
    if (g.used && (char*)buf >= g.local && (char*)buf + bytes <= g.local + g.bytes) reg = &g;
  }
  const bool zero_copy = in_sym || reg;
  DDL_ON_DEVICE(c->device);
  KParams p = base_params(c, count, op);
  Plan pl;
  const bool in_nvls = !zero_copy && nvls_owns(c, buf, bytes);
  if (!zero_copy && !in_nvls && bytes > c->max_bytes) return DDL_ERR_TOO_LARGE;
  if (use_ll(c, count, dt, &pl)) {
    p.cin[c->rank] = buf;
    p.out[c->rank] = buf;
    for (int m = 0; m < c->P; ++m) p.ll[m] = c->ll_of(m);
    p.ll_slot = c->ll_slot;
    return launch(c, p, pl, dt, stream);
  }
  if (in_nvls) return nvls_allreduce(c, p, buf, count, dt, stream);
  const bool one = use_oneshot(c, count, dt, &pl);
  if (!one) pl = plan_hier(c, count, block_elems(count, c->P, elem_size(dt)), dt, true);
  p.q = pl.q;
  p.slice = pl.slice;
  const size_t off = in_sym ? (size_t)((char*)buf - sym) : reg ? (size_t)((char*)buf - reg->local) : 0;
  for (int m = 0; m < c->P; ++m) {
    char* base = in_sym ? c->sym_of(m) + off : reg ? reg->peer[m] + off : c->stage_of(m);
    p.in[m] = base;
    p.work[m] = base;
    p.out[m] = base;
  }
  if (one) {
    // one barrier: inputs are published through the double-buffered scratch
    p.mode = kScratch;
    p.cin[c->rank] = buf;
    p.out[c->rank] = buf;
    for (int m = 0; m < c->P; ++m) p.scratch[m] = c->scratch_of(m);
    p.scratch_half = c->scratch_half;
  } else {
    p.mode = kRS | kAG | (zero_copy ? 0 : (kCinAll | kCoutAll));
    p.cin[c->rank] = buf;
    p.cout[c->rank] = buf;
  }
  return launch(c, p, pl, dt, stream);
}

ddl_result_t ddl_reduce_scatter(ddl_comm_t c, const void* sendbuf, void* recvbuf, size_t recvcount, ddl_dtype_t dt,
                                ddl_op_t op, void* stream) {
  ddl_result_t r = check_common(c, dt, op);
  if (r != DDL_SUCCESS) return r;
  if (c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  if (recvcount == 0) return DDL_SUCCESS;
  if (!sendbuf || !recvbuf || !aligned16(sendbuf) || !aligned16(recvbuf)) return DDL_ERR_INVALID_ARGUMENT;
  const int w = elem_size(dt);
  if (c->P == 1) return local_copy(sendbuf, recvbuf, recvcount, dt, stream);
  const size_t n = recvcount * (size_t)c->P;
  if (n * w > c->max_bytes) return DDL_ERR_TOO_LARGE;
  DDL_ON_DEVICE(c->device);
  const bool vec = (recvcount * w) % 16 == 0;
  Plan pl = plan_hier(c, n, recvcount, dt, vec);
  KParams p = base_params(c, n, op);
  p.q = pl.q;
  p.slice = pl.slice;
  for (int m = 0; m < c->P; ++m) {
    p.in[m] = c->stage_of(m);
    p.work[m] = c->stage_of(m);
  }
  p.cin[c->rank] = sendbuf;
  p.out[c->rank] = static_cast<char*>(recvbuf) - (ptrdiff_t)c->rank * (ptrdiff_t)(recvcount * w);
  p.mode = kCinAll | kRS;
  // zero-copy input: peers' phase-0 reads come straight from their (symmetric or
  // registered) send buffers; the partials still go to the staging workspace (send is const)
  const char* sp[kMaxRanks];
  if (zero_copy_peers(c, sendbuf, n * w, sp)) {
    for (int m = 0; m < c->P; ++m) p.in[m] = sp[m];
    p.mode = kRS;
  }
  return launch(c, p, pl, dt, stream);
}

ddl_result_t ddl_allgather(ddl_comm_t c, const void* sendbuf, void* recvbuf, size_t sendcount, ddl_dtype_t dt,
                           void* stream) {
  ddl_result_t r = check_common(c, dt, DDL_SUM);
  if (r != DDL_SUCCESS) return r;
  if (c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  if (sendcount == 0) return DDL_SUCCESS;
  if (!sendbuf || !recvbuf || !aligned16(sendbuf) || !aligned16(recvbuf)) return DDL_ERR_INVALID_ARGUMENT;
  const int w = elem_size(dt);
  if (c->P == 1) return local_copy(sendbuf, recvbuf, sendcount, dt, stream);
  const size_t n = sendcount * (size_t)c->P;
  const char* chk[kMaxRanks];
  if (n * w > c->max_bytes && !zero_copy_peers(c, recvbuf, n * w, chk)) return DDL_ERR_TOO_LARGE;
  DDL_ON_DEVICE(c->device);
  const bool vec = (sendcount * w) % 16 == 0;
  Plan pl = plan_hier(c, n, sendcount, dt, vec);
  KParams p = base_params(c, n, DDL_SUM);
  p.q = pl.q;
  p.slice = pl.slice;
  for (int m = 0; m < c->P; ++m) p.work[m] = c->stage_of(m);
  p.cin[c->rank] = sendbuf;
  p.cout[c->rank] = recvbuf;
  p.mode = kCinOwn | kAG | kCoutAll;
  // zero-copy output: gather straight into every rank's (symmetric or registered) recvbuf
  const char* rp[kMaxRanks];
  if (zero_copy_peers(c, recvbuf, n * w, rp)) {
    for (int m = 0; m < c->P; ++m) p.work[m] = const_cast<char*>(rp[m]);
    p.mode = kCinOwn | kAG;
  }
  return launch(c, p, pl, dt, stream);
}

ddl_result_t ddl_async_error(ddl_comm_t c) {
  if (!c) return DDL_ERR_INVALID_ARGUMENT;
  DDL_ON_DEVICE(c->device);
  DDL_CUDA(cudaDeviceSynchronize());
  int v = 0;
  DDL_CUDA(cudaMemcpy(&v, c->err, sizeof(int), cudaMemcpyDeviceToHost));
  return (ddl_result_t)v;
}

ddl_result_t ddl_set_algo(ddl_comm_t c, ddl_algo_t algo, size_t oneshot_max_bytes) {
  if (!c || algo < DDL_ALGO_AUTO || algo > DDL_ALGO_LL) return DDL_ERR_INVALID_ARGUMENT;
  c->algo = algo;
  c->oneshot_max = oneshot_max_bytes;
  return DDL_SUCCESS;
}

ddl_result_t ddl_set_ll_max(ddl_comm_t c, size_t ll_max_bytes) {
  if (!c) return DDL_ERR_INVALID_ARGUMENT;
  c->ll_max = ll_max_bytes;  // eligibility is also bounded by the receive slot size from init
  return DDL_SUCCESS;
}

ddl_result_t ddl_set_timeout(ddl_comm_t c, uint64_t timeout_ms) {
  if (!c) return DDL_ERR_INVALID_ARGUMENT;
  c->timeout_ns = timeout_ms * 1000000ull;
  return DDL_SUCCESS;
}

ddl_algo_t ddl_algo_for(ddl_comm_t c, size_t count, ddl_dtype_t dt) {
  if (!c || !valid_dtype(dt)) return DDL_ALGO_AUTO;
  Plan pl;
  if (use_ll(c, count, dt, &pl)) return DDL_ALGO_LL;
  return use_oneshot(c, count, dt, &pl) ? DDL_ALGO_ONESHOT : DDL_ALGO_HIER;
}

int ddl_ctas_for(ddl_comm_t c, size_t count, ddl_dtype_t dt) {
  if (!c || !valid_dtype(dt) || count == 0) return 0;
  Plan pl;
  if (use_ll(c, count, dt, &pl) || use_oneshot(c, count, dt, &pl)) return pl.nctas;
  return plan_hier(c, count, block_elems(count, c->P, elem_size(dt)), dt, true).nctas;
}

ddl_result_t ddl_debug_skip_rank(ddl_comm_t c, int rank) {
  if (!c) return DDL_ERR_INVALID_ARGUMENT;
  c->skip_rank = rank;
  return DDL_SUCCESS;
}

ddl_result_t ddl_debug_trace(ddl_comm_t c, void* host_out, size_t bytes) {
  if (!c || !host_out) return DDL_ERR_INVALID_ARGUMENT;
  if (!c->trace) return DDL_ERR_UNSUPPORTED;
  const size_t tb = (size_t)c->P * c->cmax * kTraceEvents * sizeof(uint64_t);
  if (bytes < tb) return DDL_ERR_INVALID_ARGUMENT;
  DDL_CUDA(cudaDeviceSynchronize());
  DDL_CUDA(cudaMemcpy(host_out, c->trace, tb, cudaMemcpyDeviceToHost));
  return DDL_SUCCESS;
}

ddl_result_t ddl_debug_connect_local(ddl_comm_t* comms, int nranks) {
  if (!comms || nranks < 1 || nranks > kMaxRanks) return DDL_ERR_INVALID_ARGUMENT;
  for (int r = 0; r < nranks; ++r) {
    const ddl_comm* c = comms[r];
    if (!c || c->loopback || c->rank != r || c->P != nranks) return DDL_ERR_INVALID_ARGUMENT;
    if (c->ndims != comms[0]->ndims || c->max_bytes != comms[0]->max_bytes || c->cmax != comms[0]->cmax ||
        c->device != comms[0]->device || c->scratch_half != comms[0]->scratch_half ||
        c->ll_slot != comms[0]->ll_slot)
      return DDL_ERR_MISMATCH;
    for (int d = 0; d < c->ndims; ++d)
      if (c->dims[d] != comms[0]->dims[d]) return DDL_ERR_MISMATCH;
  }
  for (int r = 0; r < nranks; ++r) {
    ddl_comm* c = comms[r];
    for (int m = 0; m < nranks; ++m) c->peer_base[m] = m == r ? nullptr : comms[m]->alloc;
    c->gpu_share = nranks;
    // The P ranks' kernels share this GPU's SMs from P streams.  Each kernel is sized to a
    // 1/P share (cap_per_rank), so one kernel per rank always fits -- but programmatic
    // dependent launch could let a rank's NEXT kernel take SM slots early (waiting in
    // griddepcontrol.wait) while another rank's current kernel still needs them.  Plain
    // stream order here (with one GPU per rank, as in production, this cannot starve: a
    // dependent grid only launches after every CTA of its predecessor is resident).
    c->use_pdl = false;
    c->connected = true;
  }
  return DDL_SUCCESS;
}

size_t ddl_reg_handle_size(void) { return sizeof(RegHandle); }

ddl_result_t ddl_register_export(ddl_comm_t c, void* ptr, size_t bytes, void* out) {
  if (!c || !ptr || !out || c->loopback || bytes == 0 || !aligned16(ptr)) return DDL_ERR_INVALID_ARGUMENT;
  DDL_ON_DEVICE(c->device);
  char* base = nullptr;
  DDL_CUDA(alloc_base(ptr, &base));
  RegHandle h;
  std::memset(&h, 0, sizeof(h));
  h.magic = kRegMagic;
  h.rank = c->rank;
  h.bytes = bytes;
  h.offset = (uint64_t)((char*)ptr - base);
  DDL_CUDA(cudaIpcGetMemHandle(&h.ipc, base));
  std::memcpy(out, &h, sizeof(h));
  return DDL_SUCCESS;
}

static int free_reg(ddl_comm* c) {
  for (int k = 0; k < ddl_comm::kMaxRegs; ++k)
    if (!c->regs[k].used) return k;
  return -1;
}

ddl_result_t ddl_register_connect(ddl_comm_t c, void* ptr, const void* all_handles, int* reg_id) {
  if (!c || !ptr || !all_handles || !reg_id || c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  const RegHandle* hs = static_cast<const RegHandle*>(all_handles);
  for (int m = 0; m < c->P; ++m)
    if (hs[m].magic != kRegMagic || hs[m].rank != m) return DDL_ERR_INVALID_ARGUMENT;
  for (int m = 0; m < c->P; ++m)
    if (hs[m].bytes != hs[c->rank].bytes) return DDL_ERR_MISMATCH;
  const int k = free_reg(c);
  if (k < 0) return DDL_ERR_UNSUPPORTED;
  DDL_ON_DEVICE(c->device);
  ddl_comm::Reg g;
  g.local = static_cast<char*>(ptr);
  g.bytes = hs[c->rank].bytes;
  for (int m = 0; m < c->P; ++m) {
    if (m == c->rank) {
      g.peer[m] = g.local;
      continue;
    }
    char* base = nullptr;
    for (auto& mp : c->maps)
      if (mp.rank == m && !std::memcmp(&mp.h, &hs[m].ipc, sizeof(cudaIpcMemHandle_t))) {
        base = mp.base;
        ++mp.refs;
      }
    if (!base) {
      void* v = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&v, hs[m].ipc, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle (register)");
      base = static_cast<char*>(v);
      c->maps.push_back(ddl_comm::Mapping{m, hs[m].ipc, base, 1});
    }
    g.mapped[m] = base;
    g.peer[m] = base + hs[m].offset;
  }
  g.used = true;
  c->regs[k] = g;
  *reg_id = k;
  return DDL_SUCCESS;
}

static void release_reg(ddl_comm* c, int k) {
  ddl_comm::Reg& g = c->regs[k];
  for (int m = 0; m < kMaxRanks; ++m) {
    if (!g.mapped[m]) continue;
    for (size_t i = 0; i < c->maps.size(); ++i)
      if (c->maps[i].base == g.mapped[m] && c->maps[i].rank == m && --c->maps[i].refs == 0) {
        cudaIpcCloseMemHandle(c->maps[i].base);
        c->maps.erase(c->maps.begin() + i);
        break;
      }
  }
  g = ddl_comm::Reg();
}

ddl_result_t ddl_deregister(ddl_comm_t c, int reg_id) {
  if (!c || reg_id < 0 || reg_id >= ddl_comm::kMaxRegs || !c->regs[reg_id].used) return DDL_ERR_INVALID_ARGUMENT;
  DeviceGuard dg_(c->device);
  cudaDeviceSynchronize();
  release_reg(c, reg_id);
  return DDL_SUCCESS;
}

ddl_result_t ddl_debug_register_local(ddl_comm_t* comms, void* const* ptrs, size_t bytes, int nranks, int* reg_id) {
  if (!comms || !ptrs || !reg_id || nranks < 1 || nranks > kMaxRanks || bytes == 0) return DDL_ERR_INVALID_ARGUMENT;
  int k = -1;
  for (int kk = 0; kk < ddl_comm::kMaxRegs && k < 0; ++kk) {
    bool ok = true;
    for (int r = 0; r < nranks; ++r) ok = ok && !comms[r]->regs[kk].used;
    if (ok) k = kk;
  }
  if (k < 0) return DDL_ERR_UNSUPPORTED;
  for (int r = 0; r < nranks; ++r) {
    if (!ptrs[r] || !aligned16(ptrs[r])) return DDL_ERR_INVALID_ARGUMENT;
    ddl_comm::Reg& g = comms[r]->regs[k];
    g = ddl_comm::Reg();
    g.used = true;
    g.local = static_cast<char*>(ptrs[r]);
    g.bytes = bytes;
    for (int m = 0; m < nranks; ++m) g.peer[m] = static_cast<char*>(ptrs[m]);
  }
  *reg_id = k;
  return DDL_SUCCESS;
}

ddl_result_t ddl_finalize(ddl_comm_t c) {
  if (!c) return DDL_SUCCESS;
  DeviceGuard dg_(c->device);
  cudaDeviceSynchronize();
  for (int k = 0; k < ddl_comm::kMaxRegs; ++k)
    if (c->regs[k].used) release_reg(c, k);
  if (!c->loopback) nvls::teardown(c->nvls, c->topo, c->rank);
  for (int m = 0; m < kMaxRanks; ++m)
    if (c->peer_mapped[m]) cudaIpcCloseMemHandle(c->peer_base[m]);
  if (c->alloc) cudaFree(c->alloc);
  if (c->lb_flags) cudaFree(c->lb_flags);
  if (c->lb_ws) cudaFree(c->lb_ws);
  if (c->lb_ll) cudaFree(c->lb_ll);
  if (c->err) cudaFree(c->err);
  if (c->trace) cudaFree(c->trace);
  delete c;
  return DDL_SUCCESS;
}

// ------------------------------------------------------------------ loopback
ddl_result_t ddl_init_loopback(ddl_comm_t* comm, int nranks, const int* dims, int ndims, int cuda_device,
                               size_t max_bytes) {
  (void)max_bytes;
  return ddl_loopback_init(comm, nranks, dims, ndims, cuda_device);
}

ddl_result_t ddl_loopback_init(ddl_comm_t* comm, int nranks, const int* dims, int ndims, int cuda_device) {
  if (!comm) return DDL_ERR_INVALID_ARGUMENT;
  *comm = nullptr;
  DeviceGuard guard(cuda_device < 0 ? 0 : cuda_device);
  ddl_comm* c = new (std::nothrow) ddl_comm();
  if (!c) return DDL_ERR_CUDA;
  c->loopback = true;
  c->gpu_share = nranks;
  ddl_result_t r = common_init(c, nranks, dims, ndims, cuda_device);
  if (r != DDL_SUCCESS) {
    delete c;
    return r;
  }
  cudaError_t e = cudaMalloc(&c->lb_flags, c->flags_bytes * nranks);
  if (e == cudaSuccess) e = cudaMemset(c->lb_flags, 0, c->flags_bytes * nranks);
  // LL receive regions (forced ALGO_LL only): zeroed, so a stale word never carries a live epoch
  c->ll_slot = (2 * c->ll_max + 4095) / 4096 * 4096;
  const size_t ll_bytes = (size_t)nranks * 2 * (size_t)nranks * c->ll_slot;
  if (e == cudaSuccess && ll_bytes) e = cudaMalloc(&c->lb_ll, ll_bytes);
  if (e == cudaSuccess && ll_bytes) e = cudaMemset(c->lb_ll, 0, ll_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->err, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->err, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (c->lb_flags) cudaFree(c->lb_flags);
    if (c->lb_ll) cudaFree(c->lb_ll);
      if (c->err) cudaFree(c->err);
    delete c;
    return cuda_fail(e, "ddl_loopback_init allocation");
  }
  c->connected = true;
  *comm = c;
  return DDL_SUCCESS;
}

static ddl_result_t check_ptrs(const ddl_comm* c, const void* const* ptrs) {
  if (!ptrs) return DDL_ERR_INVALID_ARGUMENT;
  for (int r = 0; r < c->P; ++r)
    if (!ptrs[r] || !aligned16(ptrs[r])) return DDL_ERR_INVALID_ARGUMENT;
  return DDL_SUCCESS;
}

// ---------------------------------------------------------------- grouped all-reduce (one launch)
static const void* multi_fn_dt(ddl_dtype_t dt) {
  if (dt == DDL_INT32) return (const void*)ddl_multi_kernel<int32_t>;
  if (dt == DDL_FLOAT32) return (const void*)ddl_multi_kernel<float>;
  return (const void*)ddl_multi_kernel<__nv_bfloat16>;
}

// Launch the grouped kernel for buckets i < nb with element counts ns[i] and every rank's
// buffer ptrs[i * P + m] (hierarchical-sized, 16-B aligned, zero-copy), at most kMaxBuckets
// per launch.  Buckets go to channels longest-first onto the least-loaded channel; each
// channel gets CTAs in proportion to its bytes and runs its buckets in their given order.
// The grouped kernel runs the TMA-staged phases only.  With DDL_NO_TMA (the register-staged
// fallback should bulk copies from peer memory fail) or an experimental variant selected,
// every bucket goes through a single call instead, so the variant choice holds everywhere.
static bool grouped_kernel_ok(const ddl_comm* c) {
  return c->use_tma && !c->use_dyn && !c->use_steal && !c->use_stream;
}

static ddl_result_t launch_multi(const ddl_comm* c, const uint64_t* ns, void* const* ptrs, int nb, ddl_dtype_t dt,
                                 ddl_op_t op, void* stream) {
  const void* fn = multi_fn_dt(dt);
  blocks_per_sm(fn, kTmaSmem);
  const int C = cap_per_rank(c, fn, kTmaSmem);
  const int w = elem_size(dt);
  const uint64_t W = 16 / w;
  for (int g0 = 0; g0 < nb; g0 += kMaxBuckets) {
    const int gn = std::min(kMaxBuckets, nb - g0);
    MParams mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.p = base_params(c, 0, op);
    mp.p.mode = kRS | kAG;
    int K = std::min(std::min(c->channels, gn), std::min(C, kMaxChannels));
    if (K < 1) K = 1;
    int idx[kMaxBuckets], chan_of[kMaxBuckets];
    uint64_t load[kMaxChannels] = {0};
    for (int i = 0; i < gn; ++i) idx[i] = i;
    std::stable_sort(idx, idx + gn, [&](int a, int b) { return ns[g0 + a] > ns[g0 + b]; });
    for (int j = 0; j < gn; ++j) {
      int best = 0;
      for (int ch = 1; ch < K; ++ch)
        if (load[ch] < load[best]) best = ch;
      chan_of[idx[j]] = best;
      load[best] += ns[g0 + idx[j]];
    }
    uint64_t total = 0;
    for (int ch = 0; ch < K; ++ch) total += load[ch];
    int cc[kMaxChannels], used = 0;
    for (int ch = 0; ch < K; ++ch) {
      cc[ch] = std::max(1, (int)((double)C * (double)load[ch] / (double)(total ? total : 1)));
      used += cc[ch];
    }
    while (used > C) {  // (rounding up to 1 CTA can overshoot)
      int big = 0;
      for (int ch = 1; ch < K; ++ch)
        if (cc[ch] > cc[big]) big = ch;
      --cc[big];
      --used;
    }
    while (used < C) {  // leftovers to the channel with the most bytes per CTA
      int best = 0;
      for (int ch = 1; ch < K; ++ch)
        if ((double)load[ch] / cc[ch] > (double)load[best] / cc[best]) best = ch;
      ++cc[best];
      ++used;
    }
    mp.nchan = K;
    int pos = 0, maxk = 0;
    for (int ch = 0; ch <= kMaxChannels; ++ch) {
      mp.cta0[ch] = ch == 0 ? 0 : mp.cta0[ch - 1] + (ch - 1 < K ? cc[ch - 1] : 0);
      if (ch < kMaxChannels) mp.bk0[ch] = pos;
      if (ch < K) {
        int k = 0;
        const int first = pos;
        for (int i = 0; i < gn; ++i)
          if (chan_of[i] == ch) {
            mp.order[pos++] = i;
            ++k;
          }
        if (c->group_order == 1)  // ascending size within the channel
          std::stable_sort(mp.order + first, mp.order + pos, [&](int a, int b) { return ns[g0 + a] < ns[g0 + b]; });
        maxk = std::max(maxk, k);
      }
    }
    mp.bk0[kMaxChannels] = pos;
    mp.maxk = maxk;
    int waves_of[kMaxBuckets];
    for (int i = 0; i < gn; ++i) {
      const uint64_t n = ns[g0 + i];
      const uint64_t q = block_elems(n, c->P, w);
      const int nc = cc[chan_of[i]];
      uint64_t slice = (q + nc - 1) / nc;
      slice = (slice + W - 1) / W * W;
      int nw = 1;
      // Waves per bucket (DDL_GROUP_WAVES; 0 = auto: about one per wave_slice_bytes of per-CTA
      // slice, rounded): a smaller working set per wave keeps more partials in L2 while the
      // other channels stream.
      int gw = c->group_waves;
      if (gw == 0) gw = (int)std::min<uint64_t>(32, (slice * w + c->wave_slice_bytes / 2) / c->wave_slice_bytes);
      // Footprint budget (every rank on this GPU): the first RS phase leaves P * n * w / g_0
      // bytes of partials in this GPU's memory for the next phase; cut the bucket into waves
      // so that one wave's partials fit the budget (they then stay in L2 until consumed).
      if (c->group_wave_bytes && c->gpu_share == c->P && c->topo.nlive > 1) {
        const uint64_t fp = (uint64_t)c->P * n * w / (uint64_t)c->topo.g[c->topo.live[0]];
        gw = std::max<int>(gw, (int)std::min<uint64_t>(32, (fp + c->group_wave_bytes - 1) / c->group_wave_bytes));
      }
      if (slice * w > kMaxSliceBytes)  // 32-bit slice fields: cut into waves
        gw = std::max<int>(gw, (int)((slice * w + kMaxSliceBytes - 1) / kMaxSliceBytes));
      if (gw > 1) {
        uint64_t s2 = (q + (uint64_t)nc * gw - 1) / ((uint64_t)nc * gw);
        s2 = (s2 + W - 1) / W * W;
        if (s2 * w >= c->min_wave_slice_bytes) {
          slice = s2;
          nw = (int)((q + (uint64_t)nc * s2 - 1) / ((uint64_t)nc * s2));
        }
      }
      if (slice * w > kMaxSliceBytes) return DDL_ERR_TOO_LARGE;
      waves_of[i] = nw;
      mp.b[i].n = n;
      mp.b[i].q = q;
      mp.b[i].nwaves = nw;
      mp.b[i].slice = slice ? slice : W;
      for (int m = 0; m < c->P; ++m) mp.b[i].buf[m] = ptrs[(size_t)(g0 + i) * c->P + m];
    }
    mp.maxk = 0;
    for (int ch = 0; ch < K; ++ch) {
      int kw = 0;
      for (int j = mp.bk0[ch]; j < mp.bk0[ch + 1]; ++j) kw += waves_of[mp.order[j]];
      mp.maxk = std::max(mp.maxk, kw);
    }
    maxk = mp.maxk;
    void* args[] = {&mp};
    if (c->debug)
      std::fprintf(stderr, "[ddl] multi: %d buckets, %d channels, ctas %d (%d/%d/%d/%d), maxk %d\n", gn, K, C,
                   cc[0], K > 1 ? cc[1] : 0, K > 2 ? cc[2] : 0, K > 3 ? cc[3] : 0, maxk);
    mp.p.transposed = (c->loopback && c->transpose) ? 1 : 0;
    const dim3 grid = !c->loopback ? dim3(C) : mp.p.transposed ? dim3(c->P, C) : dim3(C, c->P);
    DDL_CUDA(launch_ex(fn, grid, kTmaSmem, static_cast<cudaStream_t>(stream), args, c->loopback, c->use_pdl));
  }
  return DDL_SUCCESS;
}

// Load every kernel of the library once per process, at the first communicator.  With CUDA's
// lazy module loading a kernel's first launch (or occupancy query) loads it, which can wait
// for the device to go idle -- and a device-side barrier kernel already running waits for a
// peer's launch that the blocked host thread has not issued yet (seen with several ranks in
// one process: a timeout on the first call of a new kernel).  Loading up front also keeps
// the load off the first call's latency.
static void preload_kernels() {
  static std::once_flag once;
  std::call_once(once, [] {
    std::vector<const void*> fns;
    for (ddl_dtype_t dt : {DDL_INT32, DDL_FLOAT32, DDL_BFLOAT16}) {
      for (int path = 0; path <= 7; ++path) fns.push_back(hier_fn_dt(dt, path));
      for (int K = 1; K <= 4; ++K) {
        fns.push_back(ll_fn_dt(dt, K));
        for (int R : {1, 2, 4}) fns.push_back(oneshot_fn_dt(dt, K, R));
      }
      fns.push_back(multi_fn_dt(dt));
      for (int P : {2, 4, 6, 8, 16}) {  // the flat topology's kernel per P (CT for 2, 4, 8; generic else)
        Topo t;
        make_topo(&t, P, &P, 1);
        bool ct;
        fns.push_back(chain_fn_dt(dt, t, false, &ct));
        fns.push_back(chain_fn_dt(dt, t, true, &ct));
      }
    }
    fns.push_back((const void*)ddl_local_reduce_kernel<int32_t, true>);
    fns.push_back((const void*)ddl_local_reduce_kernel<int32_t, false>);
    fns.push_back((const void*)ddl_local_reduce_kernel<float, true>);
    fns.push_back((const void*)ddl_local_reduce_kernel<float, false>);
    fns.push_back((const void*)ddl_local_reduce_kernel<__nv_bfloat16, true>);
    fns.push_back((const void*)ddl_local_reduce_kernel<__nv_bfloat16, false>);
    fns.push_back((const void*)ddl_local_reduce_tma_kernel<int32_t>);
    fns.push_back((const void*)ddl_local_reduce_tma_kernel<float>);
    fns.push_back((const void*)ddl_local_reduce_tma_kernel<__nv_bfloat16>);
    for (const void* fn : fns) {
      cudaFuncAttributes a;
      if (fn) (void)cudaFuncGetAttributes(&a, fn);
    }
    (void)cudaGetLastError();
  });
}

ddl_result_t ddl_group_allreduce_many(ddl_comm_t c, void* const* bufs, const size_t* counts, int nbufs,
                                      ddl_dtype_t dt, ddl_op_t op, void* stream) {
  ddl_result_t r = check_common(c, dt, op);
  if (r != DDL_SUCCESS) return r;
  if (!c->loopback || nbufs < 0 || (nbufs > 0 && (!bufs || !counts))) return DDL_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < nbufs; ++i)
    if (counts[i] && (r = check_ptrs(c, bufs + (size_t)i * c->P)) != DDL_SUCCESS) return r;
  if (c->P == 1) return DDL_SUCCESS;
  DDL_ON_DEVICE(c->device);
  // small buckets (one-shot regime) and empty ones go through single calls first, in order
  std::vector<uint64_t> ns;
  std::vector<void*> ptrs;
  for (int i = 0; i < nbufs; ++i) {
    if (!counts[i]) continue;
    Plan pl;
    if ((!grouped_kernel_ok(c) && !use_chain(c)) || use_oneshot(c, counts[i], dt, &pl)) {
      if ((r = ddl_group_allreduce(c, bufs + (size_t)i * c->P, counts[i], dt, op, stream)) != DDL_SUCCESS) return r;
      continue;
    }
    ns.push_back(counts[i]);
    for (int m = 0; m < c->P; ++m) ptrs.push_back(bufs[(size_t)i * c->P + m]);
  }
  if (ns.empty()) return DDL_SUCCESS;
  if (use_chain(c)) return launch_chain(c, ns.data(), ptrs.data(), (int)ns.size(), dt, op, stream);
  return launch_multi(c, ns.data(), ptrs.data(), (int)ns.size(), dt, op, stream);
}

ddl_result_t ddl_allreduce_many(ddl_comm_t c, void* const* bufs, const size_t* counts, int nbufs, ddl_dtype_t dt,
                                ddl_op_t op, void* stream) {
  ddl_result_t r = check_common(c, dt, op);
  if (r != DDL_SUCCESS) return r;
  if (c->loopback || nbufs < 0 || (nbufs > 0 && (!bufs || !counts))) return DDL_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < nbufs; ++i)
    if (counts[i] && (!bufs[i] || !aligned16(bufs[i]))) return DDL_ERR_INVALID_ARGUMENT;
  if (c->P == 1) return DDL_SUCCESS;
  DDL_ON_DEVICE(c->device);
  // buckets that are not zero-copy (staged), in the LL / one-shot regime, or checked with
  // DDL_CHECK go through single calls first, in order; the rest share one launch
  std::vector<uint64_t> ns;
  std::vector<void*> ptrs;
  for (int i = 0; i < nbufs; ++i) {
    if (!counts[i]) continue;
    const char* peer[kMaxRanks];
    Plan pl;
    const bool single = c->check || !grouped_kernel_ok(c) || use_ll(c, counts[i], dt, &pl) ||
                        use_oneshot(c, counts[i], dt, &pl) ||
                        !zero_copy_peers(c, bufs[i], counts[i] * elem_size(dt), peer);
    if (single) {
      if ((r = ddl_allreduce(c, bufs[i], counts[i], dt, op, stream)) != DDL_SUCCESS) return r;
      continue;
    }
    ns.push_back(counts[i]);
    for (int m = 0; m < c->P; ++m) ptrs.push_back(const_cast<char*>(peer[m]));
  }
  if (ns.empty()) return DDL_SUCCESS;
  return launch_multi(c, ns.data(), ptrs.data(), (int)ns.size(), dt, op, stream);
}

ddl_result_t ddl_group_allreduce(ddl_comm_t c, void* const* bufs, size_t count, ddl_dtype_t dt, ddl_op_t op,
                                 void* stream) {
  ddl_result_t r = check_common(c, dt, op);
  if (r != DDL_SUCCESS) return r;
  if (!c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  if (count == 0 || c->P == 1) return DDL_SUCCESS;
  if ((r = check_ptrs(c, bufs)) != DDL_SUCCESS) return r;
  DDL_ON_DEVICE(c->device);
  KParams p = base_params(c, count, op);
  Plan pl;
  if (use_ll(c, count, dt, &pl)) {
    for (int m = 0; m < c->P; ++m) {
      p.cin[m] = bufs[m];
      p.out[m] = bufs[m];
      p.ll[m] = c->ll_of(m);
    }
    p.ll_slot = c->ll_slot;
    return launch(c, p, pl, dt, stream);
  }
  const bool one = use_oneshot(c, count, dt, &pl);
  if (!one && use_chain(c)) {
    const uint64_t n = count;
    return launch_chain(c, &n, bufs, 1, dt, op, stream);
  }
  if (!one) pl = plan_hier(c, count, block_elems(count, c->P, elem_size(dt)), dt, true);
  p.q = pl.q;
  p.slice = pl.slice;
  for (int m = 0; m < c->P; ++m) {
    p.in[m] = bufs[m];
    p.work[m] = bufs[m];
    p.out[m] = bufs[m];
  }
  p.mode = one ? 0 : (kRS | kAG);
  return launch(c, p, pl, dt, stream);
}

ddl_result_t ddl_group_reduce_scatter(ddl_comm_t c, const void* const* sendbufs, void* const* recvbufs,
                                      size_t recvcount, ddl_dtype_t dt, ddl_op_t op, void* stream) {
  ddl_result_t r = check_common(c, dt, op);
  if (r != DDL_SUCCESS) return r;
  if (!c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  if (recvcount == 0) return DDL_SUCCESS;
  if ((r = check_ptrs(c, sendbufs)) != DDL_SUCCESS) return r;
  if ((r = check_ptrs(c, recvbufs)) != DDL_SUCCESS) return r;
  if (c->P == 1) return local_copy(sendbufs[0], recvbufs[0], recvcount, dt, stream);
  const int w = elem_size(dt);
  const size_t n = recvcount * (size_t)c->P;
  DDL_ON_DEVICE(c->device);
  const size_t need = (n * w + 255) / 256 * 256;
  if (need > c->lb_ws_bytes) {
    // growing the workspace synchronises and reallocates: not allowed inside stream capture
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    DDL_CUDA(cudaStreamIsCapturing(static_cast<cudaStream_t>(stream), &cap));
    if (cap != cudaStreamCaptureStatusNone) return DDL_ERR_TOO_LARGE;
    DDL_CUDA(cudaDeviceSynchronize());
    if (c->lb_ws) cudaFree(c->lb_ws);
    c->lb_ws = nullptr;
    c->lb_ws_bytes = 0;
    DDL_CUDA(cudaMalloc(&c->lb_ws, need * c->P));
    c->lb_ws_bytes = need;
  }
  const bool vec = (recvcount * w) % 16 == 0;
  Plan pl = plan_hier(c, n, recvcount, dt, vec);
  KParams p = base_params(c, n, op);
  p.q = pl.q;
  p.slice = pl.slice;
  for (int m = 0; m < c->P; ++m) {
    p.in[m] = sendbufs[m];
    p.work[m] = c->lb_ws + (size_t)m * c->lb_ws_bytes;
    p.out[m] = static_cast<char*>(recvbufs[m]) - (ptrdiff_t)m * (ptrdiff_t)(recvcount * w);
  }
  p.mode = kRS;
  return launch(c, p, pl, dt, stream);
}

ddl_result_t ddl_group_allgather(ddl_comm_t c, const void* const* sendbufs, void* const* recvbufs,
                                 size_t sendcount, ddl_dtype_t dt, void* stream) {
  ddl_result_t r = check_common(c, dt, DDL_SUM);
  if (r != DDL_SUCCESS) return r;
  if (!c->loopback) return DDL_ERR_INVALID_ARGUMENT;
  if (sendcount == 0) return DDL_SUCCESS;
  if ((r = check_ptrs(c, sendbufs)) != DDL_SUCCESS) return r;
  if ((r = check_ptrs(c, recvbufs)) != DDL_SUCCESS) return r;
  if (c->P == 1) return local_copy(sendbufs[0], recvbufs[0], sendcount, dt, stream);
  const int w = elem_size(dt);
  const size_t n = sendcount * (size_t)c->P;
  DDL_ON_DEVICE(c->device);
  const bool vec = (sendcount * w) % 16 == 0;
  Plan pl = plan_hier(c, n, sendcount, dt, vec);
  KParams p = base_params(c, n, DDL_SUM);
  p.q = pl.q;
  p.slice = pl.slice;
  for (int m = 0; m < c->P; ++m) {
    p.work[m] = recvbufs[m];
    p.cin[m] = sendbufs[m];
  }
  p.mode = kCinOwn | kAG;
  return launch(c, p, pl, dt, stream);
}

// ------------------------------------------------------------------ K5 local reduce
ddl_result_t ddl_local_reduce(const void* const* ins, int g, void* out, size_t count, ddl_dtype_t dt, float scale,
                              void* stream) {
  if (!ins || !out || g < 1 || g > kMaxLocalIn || !valid_dtype(dt)) return DDL_ERR_INVALID_ARGUMENT;
  if (dt == DDL_INT32 && scale != 1.0f) return DDL_ERR_UNSUPPORTED;
  if (count == 0) return DDL_SUCCESS;
  LRParams p;
  std::memset(&p, 0, sizeof(p));
  bool vec = aligned16(out);
  for (int j = 0; j < g; ++j) {
    if (!ins[j]) return DDL_ERR_INVALID_ARGUMENT;
    p.in[j] = ins[j];
    vec = vec && aligned16(ins[j]);
  }
  p.out = out;
  p.n = count;
  p.g = g;
  p.scale = scale;
  const void* fn;
  if (dt == DDL_INT32) fn = vec ? (const void*)ddl_local_reduce_kernel<int32_t, true> : (const void*)ddl_local_reduce_kernel<int32_t, false>;
  else if (dt == DDL_FLOAT32) fn = vec ? (const void*)ddl_local_reduce_kernel<float, true> : (const void*)ddl_local_reduce_kernel<float, false>;
  else fn = vec ? (const void*)ddl_local_reduce_kernel<__nv_bfloat16, true> : (const void*)ddl_local_reduce_kernel<__nv_bfloat16, false>;
  int dev = 0, sms = 148;
  DDL_CUDA(cudaGetDevice(&dev));
  DDL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // large aligned reductions (>= 32 MiB out) stream through the TMA ring: +2-6% at 64-256 MiB,
  // slower below (scripts/k5_bench.py); DDL_LR_NO_TMA=1 forces the register path
  static const bool lr_tma = env_size("DDL_LR_NO_TMA", 0) == 0;
  if (vec && count * elem_size(dt) >= (32u << 20) && lr_tma) {
    const void* tfn = dt == DDL_INT32 ? (const void*)ddl_local_reduce_tma_kernel<int32_t>
                      : dt == DDL_FLOAT32 ? (const void*)ddl_local_reduce_tma_kernel<float>
                                          : (const void*)ddl_local_reduce_tma_kernel<__nv_bfloat16>;
    const int per_sm = blocks_per_sm(tfn, kTmaSmem);
    void* targs[] = {&p};
    DDL_CUDA(launch_ex(tfn, dim3((unsigned)(per_sm * sms)), kTmaSmem, static_cast<cudaStream_t>(stream), targs,
                       false, pdl_default()));
    return DDL_SUCCESS;
  }
  const int W = vec ? 16 / elem_size(dt) : 1;
  const uint64_t items = (count + W - 1) / W;
  uint64_t grid = (uint64_t)blocks_per_sm(fn) * sms;
  const uint64_t need = (items + kThreads - 1) / kThreads;
  if (need < grid) grid = need;
  if (grid < 1) grid = 1;
  void* args[] = {&p};
  DDL_CUDA(launch_ex(fn, dim3((unsigned)grid), 0, static_cast<cudaStream_t>(stream), args, false, pdl_default()));
  return DDL_SUCCESS;
}

}  // extern "C"
