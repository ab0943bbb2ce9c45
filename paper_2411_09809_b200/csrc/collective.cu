// Combining per-GPU partials through the C ABI: the one
// data-path collective of a multi-GPU evaluation is a sum of a few float64
// partials (count, dev_sum, occlusions), so a host that is not Python (no
// torch.distributed) can still shard the unit space and combine the shards
// through this library.
//
//   glr_allreduce_sum_f64      one process driving `ndev` GPUs: a cached
//                              ncclCommInitAll communicator per device list,
//                              one grouped ncclAllReduce, synchronised;
//   glr_nccl_unique_id /       one process per GPU: the host distributes the
//   glr_nccl_comm_init /       128-byte id by its own means (file, socket,
//   glr_allreduce_sum_f64_comm MPI), every rank creates its communicator and
//   glr_nccl_comm_destroy      the allreduce is asynchronous on its stream.
//
// NCCL is opened with dlopen on first use (soname libnccl.so.2): inside a
// torch process that resolves to the copy torch already loaded, and the
// library itself keeps no link-time dependency on NCCL, so it loads on hosts
// without it (the other entry points do not need it).
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <vector>

#include "common.cuh"

namespace glr {
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t *, int, const int *) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) {
      const char *e = dlerror();
      a.why = e ? e : "libnccl.so.2 not found";
      return a;
    }
    bool all = true;
    auto sym = [&](auto &fn, const char *name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      all = all && fn != nullptr;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommInitAll, "ncclCommInitAll");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = all;
    if (!all) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

int nccl_check(ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return GLR_OK;
  set_error("%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
  return GLR_ENCCL;
}

#define GLR_NCCL(call)                                       \
  do {                                                       \
    int _rc = ::glr::nccl_check((call), #call);              \
    if (_rc != GLR_OK) return _rc;                           \
  } while (0)

int need_nccl(const char *fn) {
  if (nccl().ok) return GLR_OK;
  set_error("%s: NCCL unavailable (%s)", fn, nccl().why.c_str());
  return GLR_ENCCL;
}

// ncclCommInitAll communicators (and one stream per device), cached per
// device list; guarded by a mutex (the only mutable global of the library).
struct CommSet {
  std::vector<int> devs;
  std::vector<ncclComm_t> comms;
  std::vector<cudaStream_t> streams;
};
std::mutex g_comm_mu;
std::vector<CommSet> g_comm_sets;

struct DeviceGuard {
  int dev = -1;
  DeviceGuard() { cudaGetDevice(&dev); }
  ~DeviceGuard() {
    if (dev >= 0) cudaSetDevice(dev);
  }
};

}  // namespace
}  // namespace glr

extern "C" {

int glr_allreduce_sum_f64(int ndev, const int *devices, double **d_bufs, int count) {
  using namespace glr;
  if (ndev < 1 || devices == nullptr || d_bufs == nullptr || count < 0) {
    set_error("glr_allreduce_sum_f64: invalid arguments");
    return GLR_EARG;
  }
  for (int i = 0; i < ndev; ++i)
    if (d_bufs[i] == nullptr && count > 0) {
      set_error("glr_allreduce_sum_f64: d_bufs[%d] is NULL", i);
      return GLR_EARG;
    }
  if (count == 0) return GLR_OK;
  if (int rc = need_nccl("glr_allreduce_sum_f64")) return rc;
  std::lock_guard<std::mutex> lock(g_comm_mu);
  DeviceGuard guard;
  CommSet *set = nullptr;
  for (auto &s : g_comm_sets)
    if ((int)s.devs.size() == ndev && std::equal(s.devs.begin(), s.devs.end(), devices))
      set = &s;
  if (set == nullptr) {
    CommSet s;
    s.devs.assign(devices, devices + ndev);
    s.comms.resize(ndev);
    s.streams.resize(ndev);
    GLR_NCCL(nccl().CommInitAll(s.comms.data(), ndev, devices));
    for (int i = 0; i < ndev; ++i) {
      GLR_CUDA(cudaSetDevice(devices[i]));
      GLR_CUDA(cudaStreamCreateWithFlags(&s.streams[i], cudaStreamNonBlocking));
    }
    g_comm_sets.push_back(std::move(s));
    set = &g_comm_sets.back();
  }
  // the callers' buffers were written on their devices' default streams (or
  // any stream the caller synchronised): order behind the legacy stream
  for (int i = 0; i < ndev; ++i) {
    GLR_CUDA(cudaSetDevice(devices[i]));
    GLR_CUDA(cudaDeviceSynchronize());
  }
  GLR_NCCL(nccl().GroupStart());
  for (int i = 0; i < ndev; ++i) {
    GLR_CUDA(cudaSetDevice(devices[i]));
    ncclResult_t r = nccl().AllReduce(d_bufs[i], d_bufs[i], (size_t)count, ncclFloat64,
                                      ncclSum, set->comms[i], set->streams[i]);
    if (r != ncclSuccess) {
      nccl().GroupEnd();
      return nccl_check(r, "ncclAllReduce");
    }
  }
  GLR_NCCL(nccl().GroupEnd());
  for (int i = 0; i < ndev; ++i) {
    GLR_CUDA(cudaSetDevice(devices[i]));
    GLR_CUDA(cudaStreamSynchronize(set->streams[i]));
  }
  return GLR_OK;
}

int glr_nccl_unique_id(void *id_out) {
  using namespace glr;
  if (id_out == nullptr) {
    set_error("glr_nccl_unique_id: invalid arguments");
    return GLR_EARG;
  }
  if (int rc = need_nccl("glr_nccl_unique_id")) return rc;
  ncclUniqueId id;
  GLR_NCCL(nccl().GetUniqueId(&id));
  memcpy(id_out, &id, sizeof(id));
  return GLR_OK;
}

int glr_nccl_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

int glr_nccl_comm_init(const void *id, int rank, int world, void **comm_out) {
  using namespace glr;
  if (id == nullptr || comm_out == nullptr || world < 1 || rank < 0 || rank >= world) {
    set_error("glr_nccl_comm_init: invalid arguments");
    return GLR_EARG;
  }
  if (int rc = need_nccl("glr_nccl_comm_init")) return rc;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  GLR_NCCL(nccl().CommInitRank(&c, world, uid, rank));
  *comm_out = c;
  return GLR_OK;
}

int glr_allreduce_sum_f64_comm(void *comm, double *d_buf, int count, void *stream) {
  using namespace glr;
  if (comm == nullptr || count < 0 || (count > 0 && d_buf == nullptr)) {
    set_error("glr_allreduce_sum_f64_comm: invalid arguments");
    return GLR_EARG;
  }
  if (count == 0) return GLR_OK;
  if (int rc = need_nccl("glr_allreduce_sum_f64_comm")) return rc;
  GLR_NCCL(nccl().AllReduce(d_buf, d_buf, (size_t)count, ncclFloat64, ncclSum,
                            static_cast<ncclComm_t>(comm), as_stream(stream)));
  return GLR_OK;
}

int glr_nccl_comm_destroy(void *comm) {
  using namespace glr;
  if (comm == nullptr) return GLR_OK;
  if (int rc = need_nccl("glr_nccl_comm_destroy")) return rc;
  GLR_NCCL(nccl().CommDestroy(static_cast<ncclComm_t>(comm)));
  return GLR_OK;
}

}  // extern "C"
