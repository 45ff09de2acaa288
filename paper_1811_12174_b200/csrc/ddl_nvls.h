// ddl_nvls.h -- host side of the NVLS phases (§2.1
// feature (3): "mix and match" reduce-scatter / all-gather implementations per decomposed
// piece).  Included by ddl_host.cu only.
//
// An NVSwitch multicast object per (live dim d, group): the group's leader (c_d = 0) creates
// it for g_d devices and exports a shareable handle; every member imports it, adds its device,
// binds its own NVLS memory and maps the multicast range.  Every rank's NVLS memory is also
// exported and mapped by every peer (unicast), so phases NOT run in the switch read peers
// directly, as in the cudaIpc path.  Four collective rounds, each an all-gather of a fixed-size
// blob done by the caller (the Python binding uses the process group):
//   prepare -> attach -> bind -> commit.
// Any failure on any rank (no multicast support, no fabric manager, one GPU, ...) makes every
// rank fall back to the direct P2P phases: commit enables NVLS only when all ranks succeeded.
//
// Driver entry points are resolved at run time (cudaGetDriverEntryPoint), so libddl keeps
// linking only the static CUDA runtime.  Handle exchange: CU_MEM_HANDLE_TYPE_FABRIC when the
// allocation and its export support it (a 64-byte blob in the all-gathered round), else POSIX
// file descriptors, passed between the ranks' processes over abstract-namespace Unix domain
// sockets with SCM_RIGHTS during the attach round (works without ptrace rights over sibling
// processes, which pidfd_getfd would need).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <poll.h>
#include <sys/socket.h>
#include <sys/syscall.h>
#include <sys/un.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>


namespace ddl {
namespace nvls {

struct Api {
  bool ok = false;
  CUresult (*getAttr)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*deviceGet)(CUdevice*, int) = nullptr;
  CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long) = nullptr;
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*mcGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) =
      nullptr;
  CUresult (*memGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*memExport)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) =
      nullptr;
  CUresult (*memImport)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
};

template <typename F>
inline bool resolve(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p) {
    (void)cudaGetLastError();
    return false;
  }
  *fn = reinterpret_cast<F>(p);
  return true;
}

inline Api& api() {
  static Api a = [] {
    Api x;
    x.ok = resolve("cuDeviceGetAttribute", &x.getAttr) && resolve("cuDeviceGet", &x.deviceGet) &&
           resolve("cuMulticastCreate", &x.mcCreate) &&
           resolve("cuMulticastAddDevice", &x.mcAddDevice) && resolve("cuMulticastBindMem", &x.mcBindMem) &&
           resolve("cuMulticastUnbind", &x.mcUnbind) && resolve("cuMulticastGetGranularity", &x.mcGranularity) &&
           resolve("cuMemCreate", &x.memCreate) && resolve("cuMemGetAllocationGranularity", &x.memGranularity) &&
           resolve("cuMemExportToShareableHandle", &x.memExport) &&
           resolve("cuMemImportFromShareableHandle", &x.memImport) && resolve("cuMemAddressReserve", &x.addrReserve) &&
           resolve("cuMemAddressFree", &x.addrFree) && resolve("cuMemMap", &x.memMap) &&
           resolve("cuMemUnmap", &x.memUnmap) && resolve("cuMemSetAccess", &x.setAccess) &&
           resolve("cuMemRelease", &x.memRelease);
    return x;
  }();
  return a;
}

constexpr uint32_t kBlobMagic = 0xDD1A7715u;
enum Status : int32_t { kOk = 0, kNoApi = 1, kNoMulticast = 2, kAllocFailed = 3, kCreateFailed = 4,
                        kImportFailed = 5, kAddFailed = 6, kBindFailed = 7, kMapFailed = 8, kPeerFailed = 9 };

// One rank's contribution to a round (all-gathered by the caller, nranks * sizeof(Blob)).
struct Blob {
  uint32_t magic;
  int32_t rank;
  int32_t status;  // Status of this rank after the round
  int32_t htype;   // CUmemAllocationHandleType used (FABRIC or POSIX_FILE_DESCRIPTOR)
  int32_t pid;
  int32_t phys_fd;
  uint64_t bytes;  // rounded NVLS bytes per rank (all ranks equal)
  int32_t mc_fd[kMaxDims];
  CUmemFabricHandle phys_fab;
  CUmemFabricHandle mc_fab[kMaxDims];
  char sock[64];   // abstract Unix socket name of this rank's fd server (POSIX fd exchange)
};

// ---- file-descriptor exchange over abstract-namespace Unix domain sockets (SCM_RIGHTS)
// Message: int32 sender, int32 n, int32 tags[n] (tag 0 = the sender's NVLS memory, 1 + d =
// the multicast object of dim d it leads), with the n descriptors attached.
inline socklen_t sock_addr(const char* name, sockaddr_un* a) {
  std::memset(a, 0, sizeof(*a));
  a->sun_family = AF_UNIX;
  const size_t len = std::strlen(name);
  std::memcpy(a->sun_path + 1, name, len);  // leading NUL: abstract namespace
  return (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + len);
}

inline int fd_server_open(char* name_out, int rank) {
  static std::atomic<unsigned> seq{0};
  std::snprintf(name_out, 63, "ddl-nvls-%d-%d-%u", (int)getpid(), rank, seq.fetch_add(1));
  const int s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
  if (s < 0) return -1;
  sockaddr_un a;
  const socklen_t len = sock_addr(name_out, &a);
  if (bind(s, reinterpret_cast<sockaddr*>(&a), len) != 0 || listen(s, 64) != 0) {
    close(s);
    return -1;
  }
  return s;
}

inline bool fd_send(const char* peer_name, int sender, const std::vector<int>& tags, const std::vector<int>& fds) {
  const int s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
  if (s < 0) return false;
  sockaddr_un a;
  const socklen_t len = sock_addr(peer_name, &a);
  bool ok = false;
  for (int attempt = 0; attempt < 3000 && !ok; ++attempt) {  // the peer's server exists since prepare
    ok = connect(s, reinterpret_cast<sockaddr*>(&a), len) == 0;
    if (!ok) usleep(1000);
  }
  if (ok) {
    int32_t hdr[2 + kMaxDims + 1];
    const int n = (int)fds.size();
    hdr[0] = sender;
    hdr[1] = n;
    for (int i = 0; i < n; ++i) hdr[2 + i] = tags[i];
    iovec iov{hdr, (size_t)(2 + n) * sizeof(int32_t)};
    char ctrl[CMSG_SPACE(sizeof(int) * (kMaxDims + 1))];
    std::memset(ctrl, 0, sizeof(ctrl));
    msghdr m;
    std::memset(&m, 0, sizeof(m));
    m.msg_iov = &iov;
    m.msg_iovlen = 1;
    if (n > 0) {
      m.msg_control = ctrl;
      m.msg_controllen = CMSG_SPACE(sizeof(int) * n);
      cmsghdr* c = CMSG_FIRSTHDR(&m);
      c->cmsg_level = SOL_SOCKET;
      c->cmsg_type = SCM_RIGHTS;
      c->cmsg_len = CMSG_LEN(sizeof(int) * n);
      std::memcpy(CMSG_DATA(c), fds.data(), sizeof(int) * n);
    }
    ok = sendmsg(s, &m, 0) == (ssize_t)iov.iov_len;
  }
  close(s);
  return ok;
}

// Accept `expect` messages (timeout_ms overall); got[sender][tag] = received descriptor.
inline bool fd_recv_all(int server, int expect, int timeout_ms, std::vector<std::vector<int>>* got) {
  int done = 0;
  while (done < expect) {
    pollfd pf{server, POLLIN, 0};
    if (poll(&pf, 1, timeout_ms) <= 0) return false;
    const int c = accept4(server, nullptr, nullptr, SOCK_CLOEXEC);
    if (c < 0) return false;
    int32_t hdr[2 + kMaxDims + 1];
    iovec iov{hdr, sizeof(hdr)};
    char ctrl[CMSG_SPACE(sizeof(int) * (kMaxDims + 1))];
    msghdr m;
    std::memset(&m, 0, sizeof(m));
    m.msg_iov = &iov;
    m.msg_iovlen = 1;
    m.msg_control = ctrl;
    m.msg_controllen = sizeof(ctrl);
    const ssize_t r = recvmsg(c, &m, 0);
    close(c);
    if (r < (ssize_t)(2 * sizeof(int32_t))) return false;
    const int sender = hdr[0], n = hdr[1];
    if (sender < 0 || sender >= (int)got->size() || n < 0 || n > kMaxDims + 1) return false;
    int fds[kMaxDims + 1];
    cmsghdr* cm = CMSG_FIRSTHDR(&m);
    if (n > 0) {
      if (!cm || cm->cmsg_type != SCM_RIGHTS) return false;
      std::memcpy(fds, CMSG_DATA(cm), sizeof(int) * n);
    }
    for (int i = 0; i < n; ++i) {
      const int tag = hdr[2 + i];
      if (tag < 0 || tag > kMaxDims) return false;
      (*got)[sender][tag] = fds[i];
    }
    ++done;
  }
  return true;
}

// Per-communicator state.
struct State {
  int stage = 0;  // 0 none, 1 prepared, 2 attached, 3 bound, 4 ready
  int dev = 0;          // runtime ordinal (access descriptors take it)
  CUdevice cudev = 0;   // driver handle of that device (multicast calls)
  size_t gran = 0;      // multicast / allocation granularity: VA alignment
  CUmemAllocationHandleType htype = CU_MEM_HANDLE_TYPE_NONE;
  size_t bytes = 0;
  CUmemGenericAllocationHandle phys = 0;
  int phys_fd = -1;
  char* uc[kMaxRanks] = {};                        // unicast mappings: own (uc[rank]) and peers'
  CUmemGenericAllocationHandle peer_phys[kMaxRanks] = {};
  CUmemGenericAllocationHandle mc[kMaxDims] = {};  // multicast object of my dim-d group
  int mc_fd[kMaxDims];
  bool mc_added[kMaxDims] = {};
  bool mc_bound[kMaxDims] = {};
  char* mcva[kMaxDims] = {};
  int mask = 0;  // dims running in the switch (after commit)
  int server = -1;                                 // fd server socket (POSIX fd exchange)
  std::vector<std::vector<int>> rx;                // [sender][tag] descriptors received
  State() {
    for (int d = 0; d < kMaxDims; ++d) mc_fd[d] = -1;
  }
};

// Import a peer's shareable handle: its fabric blob, or the descriptor it sent us.
inline CUresult import_handle(CUmemGenericAllocationHandle* h, CUmemAllocationHandleType ht, int local_fd,
                              const CUmemFabricHandle* fab) {
  Api& a = api();
  if (ht == CU_MEM_HANDLE_TYPE_FABRIC) return a.memImport(h, const_cast<CUmemFabricHandle*>(fab), ht);
  if (local_fd < 0) return CUDA_ERROR_INVALID_HANDLE;
  return a.memImport(h, reinterpret_cast<void*>((uintptr_t)local_fd), ht);
}

inline CUresult map_rw(CUmemGenericAllocationHandle h, size_t bytes, size_t align, int dev, char** va) {
  Api& a = api();
  CUdeviceptr p = 0;
  CUresult r = a.addrReserve(&p, bytes, align, 0, 0);
  if (r != CUDA_SUCCESS) return r;
  r = a.memMap(p, bytes, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    a.addrFree(p, bytes);
    return r;
  }
  CUmemAccessDesc acc;
  std::memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = a.setAccess(p, bytes, &acc, 1);
  if (r != CUDA_SUCCESS) {
    a.memUnmap(p, bytes);
    a.addrFree(p, bytes);
    return r;
  }
  *va = reinterpret_cast<char*>(p);
  return CUDA_SUCCESS;
}

inline void unmap(char** va, size_t bytes) {
  if (*va) {
    api().memUnmap((CUdeviceptr)*va, bytes);
    api().addrFree((CUdeviceptr)*va, bytes);
    *va = nullptr;
  }
}

// Release everything (any stage); safe to call twice.
inline void teardown(State& s, const Topo& t, int rank) {
  if (!api().ok) return;
  for (int d = 0; d < kMaxDims; ++d) {
    unmap(&s.mcva[d], s.bytes);
    if (s.mc_bound[d]) api().mcUnbind(s.mc[d], s.cudev, 0, s.bytes);
    s.mc_bound[d] = false;
    if (s.mc[d]) api().memRelease(s.mc[d]);
    s.mc[d] = 0;
    if (s.mc_fd[d] >= 0) close(s.mc_fd[d]);
    s.mc_fd[d] = -1;
    s.mc_added[d] = false;
  }
  for (int m = 0; m < t.P; ++m) {
    unmap(&s.uc[m], s.bytes);
    if (m != rank && s.peer_phys[m]) api().memRelease(s.peer_phys[m]);
    s.peer_phys[m] = 0;
  }
  if (s.phys) api().memRelease(s.phys);
  s.phys = 0;
  if (s.phys_fd >= 0) close(s.phys_fd);
  s.phys_fd = -1;
  if (s.server >= 0) close(s.server);
  s.server = -1;
  for (auto& v : s.rx)
    for (int& fd : v)
      if (fd >= 0) {
        close(fd);
        fd = -1;
      }
  s.rx.clear();
  s.mask = 0;
  s.stage = 0;
}

}  // namespace nvls
}  // namespace ddl
