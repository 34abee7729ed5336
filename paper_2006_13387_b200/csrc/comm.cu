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
  void sendrecv2(const void* s0, size_t sb0, int dst0, void* r0, size_t rb0, int src0, const void* s1,
                 size_t sb1, int dst1, void* r1, size_t rb1, int src1, cudaStream_t st) override {
    MS_NCCL(nccl().groupStart());
    if (dst0 >= 0 && sb0) MS_NCCL(nccl().send(s0, sb0, ncclUint8, dst0, comm, st));
    if (src0 >= 0 && rb0) MS_NCCL(nccl().recv(r0, rb0, ncclUint8, src0, comm, st));
    if (dst1 >= 0 && sb1) MS_NCCL(nccl().send(s1, sb1, ncclUint8, dst1, comm, st));
    if (src1 >= 0 && rb1) MS_NCCL(nccl().recv(r1, rb1, ncclUint8, src1, comm, st));
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
  void sendrecv2(const void* s0, size_t sb0, int dst0, void* r0, size_t rb0, int src0, const void* s1,
                 size_t sb1, int dst1, void* r1, size_t rb1, int src1, cudaStream_t st) override {
    MS_CUDA(cudaStreamSynchronize(st));
    check(cb.sendrecv(cb.user, s0, (int64_t)sb0, dst0, r0, (int64_t)rb0, src0), "sendrecv");
    check(cb.sendrecv(cb.user, s1, (int64_t)sb1, dst1, r1, (int64_t)rb1, src1), "sendrecv");
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
