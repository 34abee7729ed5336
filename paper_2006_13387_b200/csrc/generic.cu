// Kernels of the generic PCG entry point (ms_pcg_solve_generic): the
// reference's pcg_solve takes ANY `A @ v` / callable operator and any
// `.apply` / callable preconditioner (krylov.py:73-78, 90).  The fused fast
// path (ms_pcg_solve) covers the Q1 elasticity operator with the two-level
// preconditioner; everything else runs the same recurrence on device-resident
// free-dof vectors with these unfused kernels and a CSR operator.
#include "generic.cuh"

namespace msgpu {

// p.q -> alpha = rz / (p.q) (krylov.py:115)
__global__ void __launch_bounds__(kReduceThreads)
    k_pq(int64_t n, const double* __restrict__ p, const double* __restrict__ q, PcgScalars* sc,
         double* partials, double* alpha_hist) {
  if (sc->done) return;
  __shared__ double sred[kReduceThreads / 32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) acc += p[i] * q[i];
  const double bs = block_sum(acc, sred);
  double tot;
  if (grid_reduce_last(bs, partials, &sc->tickets[0], &tot, sred)) {
    if (threadIdx.x == 0) fin_alpha(sc, tot, alpha_hist);
  }
}

void launch_pq(int64_t n, const double* p, const double* q, PcgScalars* sc, double* partials,
               double* alpha_hist, cudaStream_t st) {
  { k_pq<<<reduce_blocks(), kReduceThreads, 0, st>>>(n, p, q, sc, partials, alpha_hist); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// p = z + beta p (krylov.py:128; beta = 0 on the first call: p = z)
__global__ void __launch_bounds__(256)
    k_direction(int64_t n, const double* __restrict__ z, double* __restrict__ p, const PcgScalars* sc) {
  if (sc->done) return;
  const double beta = sc->beta;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));  // two roundings, like numpy's z + beta * p
}

void launch_direction(int64_t n, const double* z, double* p, const PcgScalars* sc, cudaStream_t st) {
  { k_direction<<<reduce_blocks(), 256, 0, st>>>(n, z, p, sc); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// y = A x for a CSR matrix: L lanes per row (L = 2, 8 or 32 by mean row
// length), products summed in column order per lane, lanes by xor shuffles.
template <int L>
__global__ void __launch_bounds__(256)
    k_csr_spmv(int64_t n, const int64_t* __restrict__ indptr, const int* __restrict__ indices,
               const double* __restrict__ data, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / L;
  const int sub = threadIdx.x % L;
  double acc = 0.0;
  if (row < n) {
    const int64_t e1 = indptr[row + 1];
    for (int64_t e = indptr[row] + sub; e < e1; e += L) acc = fma(data[e], __ldg(x + indices[e]), acc);
  }
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (row < n && sub == 0) y[row] = acc;
}

void launch_csr_spmv(int64_t n, int64_t nnz, const int64_t* indptr, const int* indices, const double* data,
                     const double* x, double* y, cudaStream_t st) {
  if (n == 0) return;
  const double mean = (double)nnz / (double)n;
  const int L = mean <= 4.0 ? 2 : (mean <= 48.0 ? 8 : 32);
  const int blocks = div_up(n * L, 256);
  if (L == 2) {
    k_csr_spmv<2><<<blocks, 256, 0, st>>>(n, indptr, indices, data, x, y);
  } else if (L == 8) {
    k_csr_spmv<8><<<blocks, 256, 0, st>>>(n, indptr, indices, data, x, y);
  } else {
    k_csr_spmv<32><<<blocks, 256, 0, st>>>(n, indptr, indices, data, x, y);
  }
  ms_count_launch();
  MS_CUDA(cudaGetLastError());
}

}  // namespace msgpu
