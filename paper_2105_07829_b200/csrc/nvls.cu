// nvls.cu — NVLink SHARP multicast buffers for the pull (A8, SURVEY §8 NEXT #2:
// "K5 multicasts p via NVLS multimem.st").  Host code only.
//
// The server kernel stores each owned unit's p once through the multicast
// address of P; the NVSwitch writes it into every rank's P, so the update
// kernel reads every p from local HBM (no per-peer reads, no copy kernel).
// Setup per group of n ranks on n distinct devices:
//   1. rank 0 creates the multicast object (cuMulticastCreate, POSIX-fd
//      handle) and hands the fd to the other processes over an abstract
//      unix socket (SCM_RIGHTS); in-process groups share the handle directly;
//   2. every rank adds its device (cuMulticastAddDevice) — all before any bind;
//   3. every rank allocates its P (cuMemCreate), binds it to the object
//      (cuMulticastBindMem) and maps both the unicast and the multicast range.
// Driver entry points come from cudaGetDriverEntryPointByVersion (no link-time
// libcuda dependency).
#include <cuda.h>
#include <cuda_runtime.h>
#include <errno.h>
#include <string.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <sys/time.h>
#include <time.h>
#include <unistd.h>

#include <string>

#include "nvls.h"

namespace bpc {

namespace {

struct Drv {
  bool ok = false;
  CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long) = nullptr;
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*mcGran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*memGran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*exportH)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
  CUresult (*importH)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*devGet)(CUdevice*, int) = nullptr;
  CUresult (*devAttr)(int*, CUdevice_attribute, CUdevice) = nullptr;
};

Drv load_drv() {
  Drv d;
  auto get = [&](const char* name, auto& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion(name, &p, 12010, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p) {
      (void)cudaGetLastError();
      return false;
    }
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
    return true;
  };
  d.ok = get("cuMulticastCreate", d.mcCreate) && get("cuMulticastAddDevice", d.mcAddDevice) &&
         get("cuMulticastBindMem", d.mcBindMem) && get("cuMulticastUnbind", d.mcUnbind) &&
         get("cuMulticastGetGranularity", d.mcGran) && get("cuMemCreate", d.memCreate) &&
         get("cuMemGetAllocationGranularity", d.memGran) && get("cuMemAddressReserve", d.addrReserve) &&
         get("cuMemAddressFree", d.addrFree) && get("cuMemMap", d.map) && get("cuMemUnmap", d.unmap) &&
         get("cuMemSetAccess", d.setAccess) && get("cuMemRelease", d.release) &&
         get("cuMemExportToShareableHandle", d.exportH) && get("cuMemImportFromShareableHandle", d.importH) &&
         get("cuDeviceGet", d.devGet) && get("cuDeviceGetAttribute", d.devAttr);
  return d;
}

Drv& drv() {
  static Drv d = load_drv();
  return d;
}

#define DRV(call, what)                            \
  do {                                             \
    CUresult _r = (call);                          \
    if (_r != CUDA_SUCCESS) {                      \
      if (err) *err = std::string(what) + " failed (CUresult " + std::to_string((int)_r) + ")"; \
      return false;                                \
    }                                              \
  } while (0)

}  // namespace

bool nvls_supported(int device) {
  Drv& d = drv();
  if (!d.ok) return false;
  CUdevice dev;
  int a = 0;
  if (d.devGet(&dev, device) != CUDA_SUCCESS) return false;
  if (d.devAttr(&a, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return false;
  return a != 0;
}

bool nvls_size(int ndev, int device, uint64_t bytes, uint64_t* size, std::string* err) {
  Drv& d = drv();
  CUmulticastObjectProp mp = {};
  mp.numDevices = (unsigned)ndev;
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g1 = 0, g2 = 0;
  DRV(d.mcGran(&g1, &mp, CU_MULTICAST_GRANULARITY_MINIMUM), "cuMulticastGetGranularity");
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  DRV(d.memGran(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "cuMemGetAllocationGranularity");
  const uint64_t g = g1 > g2 ? g1 : g2;
  *size = (bytes + g - 1) / g * g;
  if (*size == 0) *size = g;
  return true;
}

bool nvls_create(int ndev, uint64_t size, uint64_t* mc, std::string* err) {
  Drv& d = drv();
  CUmulticastObjectProp mp = {};
  mp.numDevices = (unsigned)ndev;
  mp.size = size;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle h;
  DRV(d.mcCreate(&h, &mp), "cuMulticastCreate");
  *mc = (uint64_t)h;
  return true;
}

bool nvls_export(uint64_t mc, int* fd, std::string* err) {
  Drv& d = drv();
  DRV(d.exportH(fd, (CUmemGenericAllocationHandle)mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
      "cuMemExportToShareableHandle");
  return true;
}

bool nvls_import(int fd, uint64_t* mc, std::string* err) {
  Drv& d = drv();
  CUmemGenericAllocationHandle h;
  DRV(d.importH(&h, (void*)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), "cuMemImportFromShareableHandle");
  *mc = (uint64_t)h;
  return true;
}

bool nvls_add_device(uint64_t mc, int device, std::string* err) {
  Drv& d = drv();
  CUdevice dev;
  DRV(d.devGet(&dev, device), "cuDeviceGet");
  DRV(d.mcAddDevice((CUmemGenericAllocationHandle)mc, dev), "cuMulticastAddDevice");
  return true;
}

bool nvls_bind_map(uint64_t mc, int device, uint64_t size, NvlsMap* m, std::string* err) {
  Drv& d = drv();
  *m = NvlsMap{};
  m->size = size;
  m->device = device;
  m->mc_handle = mc;
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;   // as the multicast object
  CUmemGenericAllocationHandle ph;
  DRV(d.memCreate(&ph, size, &ap, 0), "cuMemCreate");
  m->phys = (uint64_t)ph;
  m->have_phys = true;
  DRV(d.mcBindMem((CUmemGenericAllocationHandle)mc, 0, ph, 0, size, 0), "cuMulticastBindMem");
  m->bound = true;
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = device;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mv = 0;
  DRV(d.addrReserve(&uc, size, 0, 0, 0), "cuMemAddressReserve (unicast)");
  m->uc = (void*)uc;
  DRV(d.map(uc, size, 0, ph, 0), "cuMemMap (unicast)");
  m->uc_mapped = true;
  DRV(d.setAccess(uc, size, &ad, 1), "cuMemSetAccess (unicast)");
  DRV(d.addrReserve(&mv, size, 0, 0, 0), "cuMemAddressReserve (multicast)");
  m->mc = (void*)mv;
  DRV(d.map(mv, size, 0, (CUmemGenericAllocationHandle)mc, 0), "cuMemMap (multicast)");
  m->mc_mapped = true;
  DRV(d.setAccess(mv, size, &ad, 1), "cuMemSetAccess (multicast)");
  return true;
}

void nvls_release(NvlsMap* m) {
  Drv& d = drv();
  if (!d.ok) return;
  if (m->mc_mapped) d.unmap((CUdeviceptr)m->mc, m->size);
  if (m->mc) d.addrFree((CUdeviceptr)m->mc, m->size);
  if (m->uc_mapped) d.unmap((CUdeviceptr)m->uc, m->size);
  if (m->uc) d.addrFree((CUdeviceptr)m->uc, m->size);
  if (m->bound) {
    CUdevice dev;
    if (d.devGet(&dev, m->device) == CUDA_SUCCESS) d.mcUnbind((CUmemGenericAllocationHandle)m->mc_handle, dev, 0, m->size);
  }
  if (m->have_phys) d.release((CUmemGenericAllocationHandle)m->phys);
  *m = NvlsMap{};
}

void nvls_release_handle(uint64_t mc) {
  Drv& d = drv();
  if (d.ok && mc) d.release((CUmemGenericAllocationHandle)mc);
}

// ---------------------------------------------------------------- fd passing
namespace {
void sock_name(const std::string& tag, sockaddr_un* a, socklen_t* len) {
  memset(a, 0, sizeof(*a));
  a->sun_family = AF_UNIX;
  const std::string name = "bpc-nvls-" + tag;   // abstract namespace: leading NUL
  const size_t n = std::min(name.size(), sizeof(a->sun_path) - 2);
  memcpy(a->sun_path + 1, name.data(), n);
  *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
}
}  // namespace

int fd_listen(const std::string& tag, std::string* err) {
  const int s = socket(AF_UNIX, SOCK_STREAM, 0);
  if (s < 0) {
    *err = std::string("socket: ") + strerror(errno);
    return -1;
  }
  sockaddr_un a;
  socklen_t len;
  sock_name(tag, &a, &len);
  timeval tv = {30, 0};   // accept() gives up after 30 s (a peer that never connects)
  setsockopt(s, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof(tv));
  if (bind(s, (sockaddr*)&a, len) != 0 || listen(s, 64) != 0) {
    *err = std::string("bind/listen: ") + strerror(errno);
    close(s);
    return -1;
  }
  return s;
}

bool fd_serve(int lsock, int fd, int npeers, std::string* err) {
  for (int i = 0; i < npeers; i++) {
    const int c = accept(lsock, nullptr, nullptr);
    if (c < 0) {
      *err = std::string("accept: ") + strerror(errno);
      return false;
    }
    char byte = 0;
    iovec io = {&byte, 1};
    char cbuf[CMSG_SPACE(sizeof(int))];
    memset(cbuf, 0, sizeof(cbuf));
    msghdr msg = {};
    msg.msg_iov = &io;
    msg.msg_iovlen = 1;
    msg.msg_control = cbuf;
    msg.msg_controllen = sizeof(cbuf);
    cmsghdr* cm = CMSG_FIRSTHDR(&msg);
    cm->cmsg_level = SOL_SOCKET;
    cm->cmsg_type = SCM_RIGHTS;
    cm->cmsg_len = CMSG_LEN(sizeof(int));
    memcpy(CMSG_DATA(cm), &fd, sizeof(int));
    const bool ok = sendmsg(c, &msg, 0) == 1;
    close(c);
    if (!ok) {
      *err = std::string("sendmsg: ") + strerror(errno);
      return false;
    }
  }
  return true;
}

int fd_fetch(const std::string& tag, double timeout_s, std::string* err) {
  sockaddr_un a;
  socklen_t len;
  sock_name(tag, &a, &len);
  timespec t0;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (;;) {
    const int s = socket(AF_UNIX, SOCK_STREAM, 0);
    if (s < 0) {
      *err = std::string("socket: ") + strerror(errno);
      return -1;
    }
    if (connect(s, (sockaddr*)&a, len) == 0) {
      char byte;
      iovec io = {&byte, 1};
      char cbuf[CMSG_SPACE(sizeof(int))];
      msghdr msg = {};
      msg.msg_iov = &io;
      msg.msg_iovlen = 1;
      msg.msg_control = cbuf;
      msg.msg_controllen = sizeof(cbuf);
      const ssize_t r = recvmsg(s, &msg, 0);
      close(s);
      cmsghdr* cm = r == 1 ? CMSG_FIRSTHDR(&msg) : nullptr;
      if (!cm || cm->cmsg_type != SCM_RIGHTS) {
        *err = "recvmsg: no descriptor";
        return -1;
      }
      int fd;
      memcpy(&fd, CMSG_DATA(cm), sizeof(int));
      return fd;
    }
    close(s);
    timespec t1;
    clock_gettime(CLOCK_MONOTONIC, &t1);
    if ((t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec) > timeout_s) {
      *err = "connect to the multicast handle server timed out";
      return -1;
    }
    usleep(2000);
  }
}

}  // namespace bpc
