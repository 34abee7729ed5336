// Communicators for strip-sharded multi-GPU solves: NCCL (dlopen'ed, so the
// library loads on hosts without NCCL or GPUs) and host callbacks.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include "comm.cuh"
#include "common.cuh"

namespace msgpu {

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = dlerror() ? dlerror() : "libnccl not found";
      return;
    }
#define MS_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    MS_SYM(getUniqueId, "ncclGetUniqueId");
    MS_SYM(commInitRank, "ncclCommInitRank");
    MS_SYM(commDestroy, "ncclCommDestroy");
    MS_SYM(allReduce, "ncclAllReduce");
    MS_SYM(broadcast, "ncclBroadcast");
    MS_SYM(send, "ncclSend");
    MS_SYM(recv, "ncclRecv");
    MS_SYM(groupStart, "ncclGroupStart");
    MS_SYM(groupEnd, "ncclGroupEnd");
    MS_SYM(errorString, "ncclGetErrorString");
#undef MS_SYM
  });
  if (!api.allReduce) throw Error(MS_E_CUDA, "NCCL unavailable: " + err);
  return api;
}

#define MS_NCCL(call)                                                                      \
  do {                                                                                     \
    ncclResult_t r__ = (call);                                                             \
    if (r__ != ncclSuccess)                                                                \
      throw Error(MS_E_CUDA, std::string("NCCL: ") + nccl().errorString(r__) + " (" #call ")"); \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().commDestroy(comm);
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    MS_NCCL(nccl().allReduce(buf, buf, n, ncclFloat64, ncclSum, comm, st));
  }
  void broadcast(void* buf, size_t bytes, int root, cudaStream_t st) override {
    MS_NCCL(nccl().broadcast(buf, buf, bytes, ncclUint8, root, comm, st));
  }
  void sendrecv(const Xfer* x, int n, cudaStream_t st) override {
    MS_NCCL(nccl().groupStart());
    for (int i = 0; i < n; ++i) {
      if (x[i].dst >= 0 && x[i].sb) MS_NCCL(nccl().send(x[i].s, x[i].sb, ncclUint8, x[i].dst, comm, st));
      if (x[i].src >= 0 && x[i].rb) MS_NCCL(nccl().recv(x[i].r, x[i].rb, ncclUint8, x[i].src, comm, st));
    }
    MS_NCCL(nccl().groupEnd());
  }
  void allreduce_sendrecv(double* buf, size_t n, const Xfer* x, int nx, cudaStream_t st) override {
    MS_NCCL(nccl().groupStart());
    MS_NCCL(nccl().allReduce(buf, buf, n, ncclFloat64, ncclSum, comm, st));
    for (int i = 0; i < nx; ++i) {
      if (x[i].dst >= 0 && x[i].sb) MS_NCCL(nccl().send(x[i].s, x[i].sb, ncclUint8, x[i].dst, comm, st));
      if (x[i].src >= 0 && x[i].rb) MS_NCCL(nccl().recv(x[i].r, x[i].rb, ncclUint8, x[i].src, comm, st));
    }
    MS_NCCL(nccl().groupEnd());
  }
  bool capturable() const override { return true; }
};

struct CallbackComm : Comm {
  ms_comm_callbacks cb{};
  void check(int rc, const char* what) {
    if (rc != 0) throw Error(MS_E_CUDA, std::string("communicator callback failed: ") + what);
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    MS_CUDA(cudaStreamSynchronize(st));
    check(cb.allreduce_sum(cb.user, buf, (int64_t)n), "allreduce");
  }
  void broadcast(void* buf, size_t bytes, int root, cudaStream_t st) override {
    MS_CUDA(cudaStreamSynchronize(st));
    check(cb.broadcast(cb.user, buf, (int64_t)bytes, root), "broadcast");
  }
  void sendrecv(const Xfer* x, int n, cudaStream_t st) override {
    MS_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < n; ++i)
      check(cb.sendrecv(cb.user, x[i].s, (int64_t)x[i].sb, x[i].dst, x[i].r, (int64_t)x[i].rb, x[i].src),
            "sendrecv");
  }
  bool capturable() const override { return false; }
};

}  // namespace

int nccl_unique_id(void* out128) {
  ncclUniqueId id;
  MS_NCCL(nccl().getUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
  memcpy(out128, &id, sizeof(id));
  return MS_OK;
}

std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* unique_id, int device) {
  std::unique_ptr<NcclComm> c(new NcclComm());
  c->rank = rank;
  c->world = world;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  MS_CUDA(cudaSetDevice(device));
  MS_NCCL(nccl().commInitRank(&c->comm, world, id, rank));
  return c;
}

std::unique_ptr<Comm> make_callback_comm(int rank, int world, const ms_comm_callbacks* cb) {
  if (!cb || !cb->allreduce_sum || !cb->broadcast || !cb->sendrecv)
    throw Error(MS_E_INVALID, "incomplete communicator callbacks");
  std::unique_ptr<CallbackComm> c(new CallbackComm());
  c->rank = rank;
  c->world = world;
  c->cb = *cb;
  return c;
}

}  // namespace msgpu
