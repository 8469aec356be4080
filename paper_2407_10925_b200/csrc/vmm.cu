// vmm.cu -- one contiguous virtual address range over the shards of a table (host code).
//
// The sharded quarter table gives every shard a fixed stride of the table's
// virtual address range: shard k's stored blocks live at [k * stride, k * stride + bytes_k).
// The kernels then address the whole table through one base pointer with the (shard-major)
// global slot numbers of the block map -- the unsharded sweep and bound kernels, unchanged.
//
// Physical memory: one cuMemCreate allocation per shard on its GPU.  Virtual mode (one process)
// maps all P of them; process mode maps its own and the peers' allocations, whose POSIX file
// descriptors (cuMemExportToShareableHandle) travel between the processes over Unix domain
// sockets (SCM_RIGHTS) at creation -- the fd is only meaningful inside the process that got it.
#include <cuda.h>
#include <errno.h>
#include <poll.h>
#include <stdio.h>
#include <string.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include "lcsb_internal.cuh"

namespace lcsbk {

// Driver entry points resolved at run time through the runtime (cudaGetDriverEntryPoint): the
// library does not link libcuda, so it still loads on a machine without a driver (the CPU tests).
namespace {
struct DriverApi {
  bool ok = false;
  CUresult (*getErrorString)(CUresult, const char**) = nullptr;
  CUresult (*getGranularity)(size_t*, const CUmemAllocationProp*,
                             CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*addressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) =
      nullptr;
  CUresult (*addressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                     unsigned long long) = nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                  unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*exportHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                           unsigned long long) = nullptr;
  CUresult (*importHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) =
      nullptr;
};

template <typename F>
bool entry(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult st;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &st) != cudaSuccess ||
      st != cudaDriverEntryPointSuccess || !p) {
    cudaGetLastError();
    return false;
  }
  fn = reinterpret_cast<F>(p);
  return true;
}

const DriverApi& drv() {
  static DriverApi d = [] {
    DriverApi a;
    a.ok = entry("cuGetErrorString", a.getErrorString) &&
           entry("cuMemGetAllocationGranularity", a.getGranularity) &&
           entry("cuMemAddressReserve", a.addressReserve) &&
           entry("cuMemAddressFree", a.addressFree) && entry("cuMemCreate", a.create) &&
           entry("cuMemRelease", a.release) && entry("cuMemMap", a.map) &&
           entry("cuMemUnmap", a.unmap) && entry("cuMemSetAccess", a.setAccess) &&
           entry("cuMemExportToShareableHandle", a.exportHandle) &&
           entry("cuMemImportFromShareableHandle", a.importHandle);
    return a;
  }();
  return d;
}
}  // namespace

static bool cu_ok(CUresult r, char* why, size_t wl, const char* what) {
  if (r == CUDA_SUCCESS) return true;
  const char* s = nullptr;
  if (drv().getErrorString) drv().getErrorString(r, &s);
  snprintf(why, wl, "%s: %s", what, s ? s : "unknown error");
  return false;
}

size_t vmm_granularity(int device) {
  if (!drv().ok) return 2ull << 20;
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof prop);
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0;
  if (drv().getGranularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) !=
          CUDA_SUCCESS ||
      g == 0)
    g = 2ull << 20;
  return g;
}

bool vmm_reserve(VmmTable* t, int P, size_t stride, int device, char* why, size_t wl) {
  memset(t, 0, sizeof *t);
  if (!drv().ok) {
    snprintf(why, wl, "the CUDA driver's virtual memory management entry points are unavailable");
    return false;
  }
  t->P = P;
  t->stride = stride;
  t->device = device;
  CUdeviceptr va = 0;
  if (!cu_ok(drv().addressReserve(&va, stride * (size_t)P, 0, 0, 0), why, wl, "cuMemAddressReserve"))
    return false;
  t->base = (void*)va;
  return true;
}

static bool map_handle(VmmTable* t, int k, CUmemGenericAllocationHandle h, char* why, size_t wl) {
  const CUdeviceptr at = (CUdeviceptr)t->base + (CUdeviceptr)k * t->stride;
  if (!cu_ok(drv().map(at, t->stride, 0, h, 0), why, wl, "cuMemMap")) return false;
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof acc);
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = t->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (!cu_ok(drv().setAccess(at, t->stride, &acc, 1), why, wl, "cuMemSetAccess")) {
    drv().unmap(at, t->stride);
    return false;
  }
  t->handle[k] = (unsigned long long)h;
  t->mapped[k] = 1;
  return true;
}

bool vmm_create_shard(VmmTable* t, int k, bool exportable, char* why, size_t wl) {
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof prop);
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = t->device;
  if (exportable) prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle h;
  if (!cu_ok(drv().create(&h, t->stride, &prop, 0), why, wl, "cuMemCreate")) return false;
  if (!map_handle(t, k, h, why, wl)) {
    drv().release(h);
    return false;
  }
  return true;
}

bool vmm_export_fd(VmmTable* t, int k, int* fd, char* why, size_t wl) {
  return cu_ok(drv().exportHandle(fd, (CUmemGenericAllocationHandle)t->handle[k],
                                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
               why, wl, "cuMemExportToShareableHandle");
}

bool vmm_import_fd(VmmTable* t, int k, int fd, char* why, size_t wl) {
  CUmemGenericAllocationHandle h;
  if (!cu_ok(drv().importHandle(&h, (void*)(uintptr_t)fd,
                                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
             why, wl, "cuMemImportFromShareableHandle"))
    return false;
  if (!map_handle(t, k, h, why, wl)) {
    drv().release(h);
    return false;
  }
  return true;
}

void vmm_release(VmmTable* t) {
  if (!t->base) return;
  for (int k = 0; k < t->P; ++k)
    if (t->mapped[k]) {
      drv().unmap((CUdeviceptr)t->base + (CUdeviceptr)k * t->stride, t->stride);
      drv().release((CUmemGenericAllocationHandle)t->handle[k]);
      t->mapped[k] = 0;
    }
  drv().addressFree((CUdeviceptr)t->base, t->stride * (size_t)t->P);
  t->base = nullptr;
}

// ---------------------------------------------------------------- fd exchange (SCM_RIGHTS)
// Every rank listens on the abstract Unix socket "\0lcsb-<token>-<rank>"; after a barrier every
// rank connects to each peer and sends its n fds in one message; then it accepts the P - 1
// connections of its peers and receives theirs.  `token` is agreed by the caller (rank 0's).

static void sock_name(sockaddr_un* a, socklen_t* len, uint64_t token, int rank) {
  memset(a, 0, sizeof *a);
  a->sun_family = AF_UNIX;
  const int n = snprintf(a->sun_path + 1, sizeof a->sun_path - 1, "lcsb-%016llx-%d",
                         (unsigned long long)token, rank);
  *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
}

int fdx_listen(uint64_t token, int rank, char* why, size_t wl) {
  const int s = socket(AF_UNIX, SOCK_STREAM, 0);
  if (s < 0) {
    snprintf(why, wl, "socket: %s", strerror(errno));
    return -1;
  }
  sockaddr_un a;
  socklen_t len;
  sock_name(&a, &len, token, rank);
  if (bind(s, (sockaddr*)&a, len) != 0 || listen(s, 64) != 0) {
    snprintf(why, wl, "bind/listen on the fd-exchange socket: %s", strerror(errno));
    close(s);
    return -1;
  }
  return s;
}

bool fdx_send(uint64_t token, int from, int to, const int* fds, int n, char* why, size_t wl) {
  const int s = socket(AF_UNIX, SOCK_STREAM, 0);
  if (s < 0) {
    snprintf(why, wl, "socket: %s", strerror(errno));
    return false;
  }
  sockaddr_un a;
  socklen_t len;
  sock_name(&a, &len, token, to);
  bool ok = false;
  for (int attempt = 0; attempt < 200 && !ok; ++attempt) {  // the peer listens (barrier before)
    ok = connect(s, (sockaddr*)&a, len) == 0;
    if (!ok) usleep(10000);
  }
  if (!ok) {
    snprintf(why, wl, "connect to rank %d: %s", to, strerror(errno));
    close(s);
    return false;
  }
  int32_t hdr[2] = {from, n};
  iovec iov = {hdr, sizeof hdr};
  char cbuf[CMSG_SPACE(sizeof(int) * 8)];
  memset(cbuf, 0, sizeof cbuf);
  msghdr m;
  memset(&m, 0, sizeof m);
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = cbuf;
  m.msg_controllen = CMSG_SPACE(sizeof(int) * n);
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int) * n);
  memcpy(CMSG_DATA(c), fds, sizeof(int) * n);
  ok = sendmsg(s, &m, 0) == (ssize_t)sizeof hdr;
  if (!ok) snprintf(why, wl, "sendmsg to rank %d: %s", to, strerror(errno));
  close(s);
  return ok;
}

// accept one connection; returns the sender's rank and its n fds in fds[0..n)
bool fdx_recv(int lsock, int* from, int* fds, int n, char* why, size_t wl) {
  pollfd pf = {lsock, POLLIN, 0};
  if (poll(&pf, 1, 120000) != 1) {
    snprintf(why, wl, "no peer connected to the fd-exchange socket within 120 s");
    return false;
  }
  const int s = accept(lsock, nullptr, nullptr);
  if (s < 0) {
    snprintf(why, wl, "accept: %s", strerror(errno));
    return false;
  }
  int32_t hdr[2] = {-1, 0};
  iovec iov = {hdr, sizeof hdr};
  char cbuf[CMSG_SPACE(sizeof(int) * 8)];
  msghdr m;
  memset(&m, 0, sizeof m);
  m.msg_iov = &iov;
  m.msg_iovlen = 1;
  m.msg_control = cbuf;
  m.msg_controllen = sizeof cbuf;
  const ssize_t r = recvmsg(s, &m, 0);
  close(s);
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  if (r != (ssize_t)sizeof hdr || hdr[1] != n || !c || c->cmsg_type != SCM_RIGHTS ||
      c->cmsg_len != CMSG_LEN(sizeof(int) * n)) {
    snprintf(why, wl, "malformed fd-exchange message");
    return false;
  }
  memcpy(fds, CMSG_DATA(c), sizeof(int) * n);
  *from = hdr[0];
  return true;
}

}  // namespace lcsbk
