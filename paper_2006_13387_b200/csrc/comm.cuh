// Communicator abstraction for strip-sharded multi-GPU solves.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <memory>

#include "../../include/msgpu.h"

namespace msgpu {

// one point-to-point exchange: send `sb` bytes from s to rank `dst` and receive
// `rb` bytes into r from rank `src` (either side may be -1 / 0 bytes)
struct Xfer {
  const void* s;
  size_t sb;
  int dst;
  void* r;
  size_t rb;
  int src;
};

// All operations are stream-ordered on `st` and act on device buffers.
struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t st) = 0;
  virtual void broadcast(void* buf, size_t bytes, int root, cudaStream_t st) = 0;
  // all n exchanges as one group (NCCL: one ncclGroupStart/End); messages
  // between a pair of ranks match in list order
  virtual void sendrecv(const Xfer* x, int n, cudaStream_t st) = 0;
  void sendrecv2(const void* s0, size_t sb0, int dst0, void* r0, size_t rb0, int src0, const void* s1,
                 size_t sb1, int dst1, void* r1, size_t rb1, int src1, cudaStream_t st) {
    const Xfer x[2] = {{s0, sb0, dst0, r0, rb0, src0}, {s1, sb1, dst1, r1, rb1, src1}};
    sendrecv(x, 2, st);
  }
  // allreduce(buf[0..n)) and the n_x exchanges as ONE group (NCCL: one
  // ncclGroupStart/End, one launch); the default runs them one after the other
  virtual void allreduce_sendrecv(double* buf, size_t n, const Xfer* x, int nx, cudaStream_t st) {
    allreduce_sum(buf, n, st);
    sendrecv(x, nx, st);
  }
  // may the operations be captured into a CUDA graph
  virtual bool capturable() const = 0;
};

// NCCL (libnccl.so.2 is dlopen'ed on first use)
std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* unique_id, int device);
int nccl_unique_id(void* out128);

// host callbacks (test harnesses, e.g. torch.distributed gloo on one GPU)
std::unique_ptr<Comm> make_callback_comm(int rank, int world, const ms_comm_callbacks* cb);

// strip partition of `nrows` block rows over `world` ranks: rank r owns
// [lo, hi), sizes differing by at most one, lower ranks larger
inline void strip_rows(int nrows, int world, int rank, int& lo, int& hi) {
  const int base = nrows / world, extra = nrows % world;
  lo = rank * base + (rank < extra ? rank : extra);
  hi = lo + base + (rank < extra ? 1 : 0);
}

}  // namespace msgpu
