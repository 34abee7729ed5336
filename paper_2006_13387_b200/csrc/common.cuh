// Shared device helpers for the msgpu kernels (sm_100a, fp64 throughout).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace msgpu {

// Host-side count of this thread's kernel launches (every <<<>>> site of the
// library increments it right after the launch; ms_pcg_solve reports the
// difference, with graph replays adding their captured kernel count).
inline long long& ms_launch_counter() {
  static thread_local long long c = 0;
  return c;
}
inline void ms_count_launch() { ++ms_launch_counter(); }


// Host-side error type carrying an ABI status code.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define MS_CUDA(call)                                                                 \
  do {                                                                                \
    cudaError_t err__ = (call);                                                       \
    if (err__ != cudaSuccess)                                                         \
      throw ::msgpu::Error(-3, std::string(#call ": ") + cudaGetErrorString(err__) + \
                                   " @" __FILE__ ":" + std::to_string(__LINE__));     \
  } while (0)

constexpr int kWarp = 32;
constexpr int kReduceThreads = 256;

// Structured-grid description shared by every kernel.
struct Grid {
  int nx, ny;      // elements per axis
  int nnx;         // nodes per row = nx + 1
  int64_t n_nodes; // (nx+1)(ny+1); full vector = [x-plane | y-plane]
  double h;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree).  `sh` needs blockDim.x/32 doubles.
// Result valid in all threads.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// fixed-order sum of nb partials by one block: thread i sums partials i,
// i+T, ... (L2 loads, 8 in flight per thread), then the block tree
__device__ __forceinline__ double reduce_partials_fixed(const double* partials, unsigned int nb, double* sh) {
  double s = 0.0;
  unsigned int i = threadIdx.x;
  for (; i + 7 * blockDim.x < nb; i += 8 * blockDim.x) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(partials + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; i < nb; i += blockDim.x) s += __ldcg(partials + i);
  return block_sum(s, sh);
}

// "Last block finishes" deterministic grid reduction: every block writes its
// partial; the last one to arrive (atomic ticket) sums all partials in index
// order.  Returns true in the finishing block (all threads), with *out set.
__device__ __forceinline__ bool grid_reduce_last(double blockval, double* partials,
                                                 unsigned int* ticket, double* out,
                                                 double* sh) {
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x + gridDim.x * blockIdx.y] = blockval;
    __threadfence();
    unsigned int nb = gridDim.x * gridDim.y;
    unsigned int t = atomicAdd(ticket, 1u);
    am_last = (t == nb - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  const double s = reduce_partials_fixed(partials, gridDim.x * gridDim.y, sh);
  if (threadIdx.x == 0) {
    *out = s;
    *ticket = 0u;  // re-arm for the next launch
  }
  return true;
}

// Bitwise multi-rank mode (MS_DIST_BITWISE): every block writes its partial
// to its GLOBAL slot (the block's index in the one-rank grid); the ranks'
// partial arrays (zero where another rank owns the block) are summed
// exactly by an allreduce and reduced by k_reduce_partials with the same
// fixed order and block size as the one-rank finishing block.
__device__ __forceinline__ bool grid_reduce_dist(double blockval, double* partials, unsigned int gidx,
                                                 bool global_slots, unsigned int* ticket, double* out,
                                                 double* sh) {
  if (global_slots) {
    if (threadIdx.x == 0) partials[gidx] = blockval;
    return false;
  }
  return grid_reduce_last(blockval, partials, ticket, out, sh);
}

// ---- device-side bounds checks (compute-sanitizer is not available on the GPU pool) ----
// `make check` builds build/check/libmsgpu_check.so with -DMS_BOUNDS_CHECK: the
// index computations of the ring / halo / gather code assert their ranges and
// trap with a message; tests/test_gpu_bounds.py runs every level-1 layout and
// the multi-rank strips through that library.  Compiled out of the product build.
#ifdef MS_BOUNDS_CHECK
#include <cstdio>
#define MS_BCHECK(cond)                                                                        \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("msgpu bounds check failed: %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                               \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define MS_BCHECK(cond) \
  do {                  \
  } while (0)
#endif

// ---- bulk async copy (TMA engine, 1-D) + mbarrier helpers (sm_90+/sm_100a) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "MS_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra MS_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// shared-memory load of a double, 0.0 when !pred: zero and predicated load
// into the same register (the C ternary compiles to zero + load into a
// temporary + two predicated moves).  volatile: stays between the mbarrier
// wait and the refill of the stage it reads (both volatile asm).
__device__ __forceinline__ double lds_or_zero(const double* p, bool pred) {
  double v;
  asm volatile(
      "{\n"
      ".reg .pred q;\n"
      "setp.ne.u32 q, %2, 0;\n"
      "mov.b64 %0, 0;\n"
      "@q ld.shared.f64 %0, [%1];\n"
      "}\n"
      : "=d"(v)
      : "r"(smem_u32(p)), "r"((uint32_t)pred));
  return v;
}

// 8-byte asynchronous global -> shared copy (cp.async, LDGSTS); ok == false
// zero-fills the destination (src must still be a valid address)
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// global -> shared bulk copy; bytes and both addresses multiples of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace msgpu
