// Batched dense SPD inverses in packed 64x64 lower tiles, and packed SYMVs.
#pragma once

#include "banded.cuh"
#include "common.cuh"

namespace msgpu {

constexpr int kTile = 64;
__host__ __device__ inline int64_t packed_tiles(int nt) { return (int64_t)nt * (nt + 1) / 2; }
__host__ __device__ inline int64_t tile_index(int i, int j) { return (int64_t)i * (i + 1) / 2 + j; }
__host__ __device__ inline int64_t packed_words(int nt) { return packed_tiles(nt) * kTile * kTile; }

// B symmetric positive definite matrices, each nt x nt packed lower tiles (a
// matrix of order N < nt*64 is padded with an identity block) stored at
// P + b * packed_words(nt).  On exit X + b * packed_words(nt) holds the
// inverse (full symmetric diagonal tiles, lower off-diagonal tiles); P is
// overwritten by the Cholesky factor and W (same size as P) is workspace.
// *fail receives 1 + (b * nt * 64 + row) of the first non-positive pivot.
void dense_spd_inverse_batched(int nt, int B, double* P, double* W, double* X, int* fail,
                               cudaStream_t st);

// single matrix from a row-major N x N array (lower triangle read): the
// coarse operator K0 (coarse.py:136-147)
void dense_spd_inverse(int N, const double* A, double* packed_inv, double* work, int* fail,
                       cudaStream_t st);
size_t dense_spd_inverse_work_bytes(int N);

// Cholesky factor only (the reference's cho_factor, coarse.py:143): packed_L
// (packed_words(nt)) <- L, diag_inv (nt * 64 * 64) <- the inverses of its
// diagonal tiles; work: packed_words(nt) doubles.
void dense_cholesky(int N, const double* A, double* packed_L, double* diag_inv, double* work, int* fail,
                    cudaStream_t st);
// y = L^-T L^-1 f (cho_solve, coarse.py:154): blocked forward/backward
// triangular solves; t, yscratch: nt*64 doubles; sync: trsv_sync_ints(N) ints.
size_t trsv_sync_ints(int N);
void launch_trsv_packed(int N, const double* L, const double* Dinv, const double* f, double* t,
                        double* yscratch, double* y, int* sync, const int* done, cudaStream_t st);

// y = X f for one packed symmetric matrix; `part` needs packed_tiles(nt)*2*64 doubles.
// [t_begin, t_end): only these packed tiles contribute (a rank's share of a
// sharded coarse solve; the caller sums y over ranks); default all.
void launch_symv_packed(int N, const double* X, const double* f, double* y, double* part,
                        const int* done, cudaStream_t st, int64_t t_begin = 0, int64_t t_end = -1);

// level-1 band (unfactored, column-band layout of BandSys) -> packed tiles,
// for systems [s0, s0 + B) into P (B matrices of nt tiles)
void launch_band_to_tiles(const BandSys* sys, int s0, int B, int nt, const double* band, double* P,
                          cudaStream_t st);

// level-1 apply with explicit packed inverses: per subdomain s, gather R_s r,
// y_s = X_s (R_s r) into ybuf[yoff_s ...]; one CTA per subdomain, y and the
// gathered residual in shared memory, tiles streamed with register prefetch.
void launch_l1_dense_apply(const Grid& g, const BandSys* sys, int nsys, int nt, const double* X,
                           const double* r, double* ybuf, const int* done, cudaStream_t st);

}  // namespace msgpu
