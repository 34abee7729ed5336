// Unfused PCG vector kernels and the CSR operator of ms_pcg_solve_generic.
#pragma once

#include "operator.cuh"

namespace msgpu {

// p.q -> alpha (uses tickets[0] like the fused matvec)
void launch_pq(int64_t n, const double* p, const double* q, PcgScalars* sc, double* partials,
               double* alpha_hist, cudaStream_t st);
// p = z + beta p
void launch_direction(int64_t n, const double* z, double* p, const PcgScalars* sc, cudaStream_t st);
// y = A x, A in CSR (int64 row pointers, int32 column indices)
void launch_csr_spmv(int64_t n, int64_t nnz, const int64_t* indptr, const int* indices, const double* data,
                     const double* x, double* y, cudaStream_t st);

}  // namespace msgpu
