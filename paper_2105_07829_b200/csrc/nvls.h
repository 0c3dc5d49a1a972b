// nvls.h — NVLink SHARP multicast buffers (nvls.cu), internal to libbpc.
#pragma once
#include <stdint.h>

#include <string>

namespace bpc {

// one rank's P bound to a multicast object: unicast (local reads) and
// multicast (multimem.st to every rank) mappings of the same bytes
struct NvlsMap {
  void* uc = nullptr;
  void* mc = nullptr;
  uint64_t size = 0;
  uint64_t phys = 0, mc_handle = 0;
  int device = -1;
  bool have_phys = false, bound = false, uc_mapped = false, mc_mapped = false;
};

bool nvls_supported(int device);   // CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED and the driver entry points
bool nvls_size(int ndev, int device, uint64_t bytes, uint64_t* size, std::string* err);   // granularity-rounded
bool nvls_create(int ndev, uint64_t size, uint64_t* mc, std::string* err);
bool nvls_export(uint64_t mc, int* fd, std::string* err);
bool nvls_import(int fd, uint64_t* mc, std::string* err);
bool nvls_add_device(uint64_t mc, int device, std::string* err);
bool nvls_bind_map(uint64_t mc, int device, uint64_t size, NvlsMap* m, std::string* err);
void nvls_release(NvlsMap* m);          // unmap, unbind, free (idempotent)
void nvls_release_handle(uint64_t mc);  // this process's reference to the multicast object

// the multicast handle between processes: rank 0 listens on an abstract unix
// socket named by `tag` and hands the fd to npeers connections (SCM_RIGHTS)
int fd_listen(const std::string& tag, std::string* err);
bool fd_serve(int lsock, int fd, int npeers, std::string* err);
int fd_fetch(const std::string& tag, double timeout_s, std::string* err);

}  // namespace bpc
