// Batched dense SPD inverses on packed 64x64 lower tiles, and their SYMVs.
//
// Used twice:
//  * the coarse operator K0 (batch 1): replaces LAPACK ?potrf/?potrs
//    (coarse.py:143,154) -- applying the explicit packed inverse is one
//    bandwidth-bound SYMV per PCG iteration instead of two latency-bound
//    triangular sweeps;
//  * the MS_LOCAL_DENSE_INV level-1 variant (batch = subdomains): the
//    "overlapping local subdomain inverses as batched dense fp64 GEMV" of the
//    design brief, replacing SuperLU (schwarz.py:97-109).
// Tiled right-looking Cholesky (potrf/trsm/syrk), triangular inverse (trtri)
// and L^-T L^-1 (lauum); every tile kernel takes the batch index from
// blockIdx.y and works on packed lower tiles.
#include <algorithm>
#include <cstdlib>

#include "dense.cuh"

namespace msgpu {

constexpr int T = kTile;
constexpr int TP = T + 4;  // shared-memory tile pitch: the DMMA fragment loads are bank-conflict free
constexpr int kTT = 256;   // threads per tile CTA (8 warps)

// 64x64 tile products on the FP64 tensor cores (DMMA, mma.sync m8n8k4):
// warp w owns rows 32 (w / 4) + 8 rb + g and columns 16 (w % 4) + 8 cb +
// 2 t + e of the tile (g = lane / 4, t = lane % 4), i.e. 4 x 2 m8n8 blocks.
struct TileAcc {
  double v[4][2][2];
};

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void frag_pos(int rb, int cb, int e, int& row, int& col) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  row = 32 * (w >> 2) + 8 * rb + (lane >> 2);
  col = 16 * (w & 3) + 8 * cb + 2 * (lane & 3) + e;
}

// acc += sA * sB where sA[r][q], sB[q][c] are 64x64 row-major in smem (pitch TP)
__device__ __forceinline__ void tile_mma(TileAcc& acc, const double* sA, const double* sB) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const double* pa = sA + (32 * (w >> 2) + g) * TP + t;
  const double* pb = sB + t * TP + 16 * (w & 3) + g;
#pragma unroll 4
  for (int k = 0; k < T; k += 4) {
    double a[4], b[2];
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) a[rb] = pa[8 * rb * TP + k];
#pragma unroll
    for (int cb = 0; cb < 2; ++cb) b[cb] = pb[k * TP + 8 * cb];
#pragma unroll
    for (int rb = 0; rb < 4; ++rb)
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) dmma_8x8x4(acc.v[rb][cb], a[rb], b[cb]);
  }
}

// load a 64x64 tile (row-major, contiguous) into smem (pitch TP), optionally transposed
__device__ __forceinline__ void tile_load(double* s, const double* g, bool trans) {
  for (int t = threadIdx.x; t < T * T; t += blockDim.x) {
    const int r = t / T, c = t % T;
    if (trans)
      s[c * TP + r] = g[t];
    else
      s[r * TP + c] = g[t];
  }
}

__device__ __forceinline__ void acc_zero(TileAcc& a) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) a.v[i][j][0] = a.v[i][j][1] = 0.0;
}

__device__ __forceinline__ void acc_store(const TileAcc& a, double* g, double scale, bool add) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int row, col;
        frag_pos(i, j, e, row, col);
        const int idx = row * T + col;
        g[idx] = add ? g[idx] + scale * a.v[i][j][e] : scale * a.v[i][j][e];
      }
}

// the accumulator into a shared-memory tile (pitch TP)
__device__ __forceinline__ void acc_to_smem(const TileAcc& a, double* s) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int row, col;
        frag_pos(i, j, e, row, col);
        s[row * TP + col] = a.v[i][j][e];
      }
}

__device__ __forceinline__ void tile_ij(int64_t t, int& i, int& j) {
  i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((int64_t)(i + 1) * (i + 2) / 2 <= t) ++i;
  while ((int64_t)i * (i + 1) / 2 > t) --i;
  j = (int)(t - (int64_t)i * (i + 1) / 2);
}

// ---------------------------------------------------------------------------
__global__ void k_pack_tiles(int N, int nt, const double* __restrict__ A, double* __restrict__ P) {
  const int64_t total = packed_words(nt);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int i, j;
    tile_ij(t / (T * T), i, j);
    const int within = (int)(t % (T * T));
    const int r = i * T + within / T, c = j * T + within % T;
    P[t] = (r < N && c < N) ? A[(int64_t)r * N + c] : (r == c ? 1.0 : 0.0);
  }
}

__global__ void k_band_to_tiles(const BandSys* __restrict__ sys, int s0, int nt,
                                const double* __restrict__ band, double* __restrict__ P) {
  const int b = blockIdx.y;
  const BandSys s = sys[s0 + b];
  const int S = s.bw + 1;
  const double* A = band + s.foff;
  double* Pb = P + (int64_t)b * packed_words(nt);
  const int64_t total = packed_words(nt);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int i, j;
    tile_ij(t / (T * T), i, j);
    const int within = (int)(t % (T * T));
    const int R = i * T + within / T, Cc = j * T + within % T;
    double v;
    if (R < s.n && Cc < s.n) {
      const int lo = min(R, Cc), d = abs(R - Cc);
      v = d <= s.bw ? A[(int64_t)lo * S + d] : 0.0;
    } else {
      v = (R == Cc) ? 1.0 : 0.0;
    }
    Pb[t] = v;
  }
}

void launch_band_to_tiles(const BandSys* sys, int s0, int B, int nt, const double* band, double* P,
                          cudaStream_t st) {
  { k_band_to_tiles<<<dim3(256, B), 256, 0, st>>>(sys, s0, nt, band, P); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// Cholesky of diagonal tile k in place (lower), plus its triangular inverse
// written to tile (k,k) of W.
__global__ void __launch_bounds__(kTT) k_potrf_tile(int k, int nt, double* __restrict__ P,
                                                    double* __restrict__ W, int* fail) {
  extern __shared__ double sm[];
  double* a = sm;
  double* inv = sm + T * TP;  // pitch T
  const int64_t mw = packed_words(nt);
  double* D = P + blockIdx.y * mw + tile_index(k, k) * T * T;
  tile_load(a, D, false);
  __syncthreads();
  for (int c = 0; c < T; ++c) {
    double d = a[c * TP + c];
    if (!(d > 0.0)) {
      if (threadIdx.x == 0) atomicCAS(fail, 0, (int)(blockIdx.y * nt * T + k * T + c + 1));
      d = 1.0;
    }
    const double s = sqrt(d);
    __syncthreads();
    if (threadIdx.x == 0) a[c * TP + c] = s;
    for (int r = c + 1 + threadIdx.x; r < T; r += blockDim.x) a[r * TP + c] /= s;
    __syncthreads();
    for (int t = threadIdx.x; t < (T - c - 1) * (T - c - 1); t += blockDim.x) {
      const int r = c + 1 + t / (T - c - 1), q = c + 1 + t % (T - c - 1);
      if (q <= r) a[r * TP + q] -= a[r * TP + c] * a[q * TP + c];
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < T * T; t += blockDim.x) {
    const int r = t / T, c = t % T;
    if (c > r) a[r * TP + c] = 0.0;
    D[t] = a[r * TP + c];
  }
  __syncthreads();
  // inverse of the lower-triangular tile, column j by thread j
  if (threadIdx.x < T) {
    const int j = threadIdx.x;
    for (int r = 0; r < T; ++r) {
      double s = (r == j) ? 1.0 : 0.0;
      for (int q = j; q < r; ++q) s -= a[r * TP + q] * inv[q * T + j];
      inv[r * T + j] = (r < j) ? 0.0 : s / a[r * TP + r];
    }
  }
  __syncthreads();
  double* Wk = W + blockIdx.y * mw + tile_index(k, k) * T * T;
  for (int t = threadIdx.x; t < T * T; t += blockDim.x) Wk[t] = inv[t];
}

// panel: L_ik = A_ik L_kk^-T = A_ik (Winv_kk)^T, i > k
__global__ void __launch_bounds__(kTT) k_trsm_tiles(int k, int nt, double* __restrict__ P,
                                                    const double* __restrict__ W) {
  extern __shared__ double sm[];
  double* sA = sm;
  double* sB = sm + T * TP;
  const int64_t mw = packed_words(nt);
  P += blockIdx.y * mw;
  W += blockIdx.y * mw;
  const int i = k + 1 + blockIdx.x;
  double* Aik = P + tile_index(i, k) * T * T;
  tile_load(sA, Aik, false);
  tile_load(sB, W + tile_index(k, k) * T * T, true);
  __syncthreads();
  TileAcc acc;
  acc_zero(acc);
  tile_mma(acc, sA, sB);
  __syncthreads();
  acc_store(acc, Aik, 1.0, false);
}

// trailing update A_ij -= L_ik L_jk^T for k < j <= i
__global__ void __launch_bounds__(kTT) k_syrk_tiles(int k, int nt, double* __restrict__ P) {
  extern __shared__ double sm[];
  double* sA = sm;
  double* sB = sm + T * TP;
  P += blockIdx.y * packed_words(nt);
  const int m = nt - k - 1;
  int ii, jj;
  tile_ij(blockIdx.x, ii, jj);
  if (ii >= m) return;
  const int i = k + 1 + ii, j = k + 1 + jj;
  tile_load(sA, P + tile_index(i, k) * T * T, false);
  tile_load(sB, P + tile_index(j, k) * T * T, true);
  __syncthreads();
  TileAcc acc;
  acc_zero(acc);
  tile_mma(acc, sA, sB);
  acc_store(acc, P + tile_index(i, j) * T * T, -1.0, true);
}

// W_ij = -W_ii * sum_{l=j}^{i-1} L_il W_lj for i = j + d
__global__ void __launch_bounds__(kTT) k_trtri_tiles(int d, int nt, const double* __restrict__ P,
                                                     double* __restrict__ W) {
  extern __shared__ double sm[];
  double* sA = sm;
  double* sB = sm + T * TP;
  const int64_t mw = packed_words(nt);
  P += blockIdx.y * mw;
  W += blockIdx.y * mw;
  const int j = blockIdx.x, i = j + d;
  TileAcc acc;
  acc_zero(acc);
  for (int l = j; l < i; ++l) {
    __syncthreads();
    tile_load(sA, P + tile_index(i, l) * T * T, false);
    tile_load(sB, W + tile_index(l, j) * T * T, false);
    __syncthreads();
    tile_mma(acc, sA, sB);
  }
  __syncthreads();
  acc_to_smem(acc, sB);
  tile_load(sA, W + tile_index(i, i) * T * T, false);
  __syncthreads();
  TileAcc out;
  acc_zero(out);
  tile_mma(out, sA, sB);
  acc_store(out, W + tile_index(i, j) * T * T, -1.0, false);
}

// X_ij = sum_{l >= i} W_li^T W_lj  (i >= j) = (L^-T L^-1)_ij
__global__ void __launch_bounds__(kTT) k_lauum_tiles(int nt, const double* __restrict__ W,
                                                     double* __restrict__ X) {
  extern __shared__ double sm[];
  double* sA = sm;
  double* sB = sm + T * TP;
  const int64_t mw = packed_words(nt);
  W += blockIdx.y * mw;
  X += blockIdx.y * mw;
  int i, j;
  tile_ij(blockIdx.x, i, j);
  TileAcc acc;
  acc_zero(acc);
  for (int l = i; l < nt; ++l) {
    __syncthreads();
    tile_load(sA, W + tile_index(l, i) * T * T, true);
    tile_load(sB, W + tile_index(l, j) * T * T, false);
    __syncthreads();
    tile_mma(acc, sA, sB);
  }
  acc_store(acc, X + tile_index(i, j) * T * T, 1.0, false);
}

static void tile_kernels_configure() {
  const size_t smem = 2 * T * TP * sizeof(double);
  static bool attr_done[64] = {};  // function attributes are per device
  int dev = 0;
  MS_CUDA(cudaGetDevice(&dev));
  bool& attr = attr_done[dev < 64 ? dev : 63];
  if (!attr || dev >= 64) {
    MS_CUDA(cudaFuncSetAttribute(k_potrf_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MS_CUDA(cudaFuncSetAttribute(k_trsm_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MS_CUDA(cudaFuncSetAttribute(k_syrk_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MS_CUDA(cudaFuncSetAttribute(k_trtri_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MS_CUDA(cudaFuncSetAttribute(k_lauum_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
}

// right-looking tiled Cholesky: P <- L, W(k,k) <- L_kk^-1 (other W tiles zero)
static void tiled_cholesky(int nt, int B, double* P, double* W, int* fail, cudaStream_t st) {
  const size_t smem = 2 * T * TP * sizeof(double);
  tile_kernels_configure();
  MS_CUDA(cudaMemsetAsync(W, 0, (size_t)B * packed_words(nt) * sizeof(double), st));
  for (int k = 0; k < nt; ++k) {
    { k_potrf_tile<<<dim3(1, B), kTT, smem, st>>>(k, nt, P, W, fail); ms_count_launch(); }
    const int m = nt - k - 1;
    if (m > 0) {
      { k_trsm_tiles<<<dim3(m, B), kTT, smem, st>>>(k, nt, P, W); ms_count_launch(); }
      { k_syrk_tiles<<<dim3((unsigned)((int64_t)m * (m + 1) / 2), B), kTT, smem, st>>>(k, nt, P); ms_count_launch(); }
    }
  }
  MS_CUDA(cudaGetLastError());
}

void dense_spd_inverse_batched(int nt, int B, double* P, double* W, double* X, int* fail,
                               cudaStream_t st) {
  if (nt == 0 || B == 0) return;
  const size_t smem = 2 * T * TP * sizeof(double);
  tiled_cholesky(nt, B, P, W, fail, st);
  for (int d = 1; d < nt; ++d) { k_trtri_tiles<<<dim3(nt - d, B), kTT, smem, st>>>(d, nt, P, W); ms_count_launch(); }
  { k_lauum_tiles<<<dim3((unsigned)packed_tiles(nt), B), kTT, smem, st>>>(nt, W, X); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

__global__ void k_copy_diag_tiles(int nt, const double* __restrict__ W, double* __restrict__ D) {
  const int k = blockIdx.x;
  const double* src = W + tile_index(k, k) * T * T;
  for (int t = threadIdx.x; t < T * T; t += blockDim.x) D[(int64_t)k * T * T + t] = src[t];
}

void dense_cholesky(int N, const double* A, double* packed_L, double* diag_inv, double* work, int* fail,
                    cudaStream_t st) {
  if (N == 0) return;
  const int nt = div_up(N, T);
  { k_pack_tiles<<<148 * 8, 256, 0, st>>>(N, nt, A, packed_L); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
  tiled_cholesky(nt, 1, packed_L, work, fail, st);
  { k_copy_diag_tiles<<<nt, 256, 0, st>>>(nt, work, diag_inv); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// cho_solve (coarse.py:154, LAPACK ?potrs): forward L t = f, then backward
// L^T y = t, blocked by 64-row tiles of the packed factor.  One CTA per tile
// row; rows are claimed through an atomic ticket in dependency order, so a
// CTA only ever waits (spinning on a flag) for rows already claimed by a
// running CTA.  Row I: the off-diagonal products are accumulated in
// registers over all finished rows J (ascending J), reduced once, subtracted
// from the right-hand side, and the diagonal block is solved with the
// inverse L_II^-1 of the factorisation's diagonal tile.  Fixed order ->
// deterministic.  sync: 2 tickets + 2 nt flags, zeroed before every solve.
__device__ __forceinline__ void spin_flag(const int* flag) {
  if (threadIdx.x == 0) {
    while (*(volatile const int*)flag == 0) {
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256)
    k_trsv_fwd(int N, int nt, const double* __restrict__ L, const double* __restrict__ Dinv,
               const double* __restrict__ f, double* t, int* sync, const int* done) {
  if (done && *(volatile const int*)done) return;
  __shared__ int sI;
  __shared__ double s[T];
  if (threadIdx.x == 0) sI = atomicAdd(&sync[0], 1);
  __syncthreads();
  const int I = sI;
  int* flag = sync + 2;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double u[4] = {0.0, 0.0, 0.0, 0.0};
  for (int J = 0; J < I; ++J) {
    const double* Lt = L + tile_index(I, J) * T * T;
    double2 a[4][2];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const double2* row = reinterpret_cast<const double2*>(Lt + (ty * 4 + rr) * T + tx * 4);
      a[rr][0] = __ldg(row);
      a[rr][1] = __ldg(row + 1);
    }
    spin_flag(flag + J);
    double y[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) y[q] = __ldcg(t + J * T + tx * 4 + q);
#pragma unroll
    for (int rr = 0; rr < 4; ++rr)
      u[rr] += a[rr][0].x * y[0] + a[rr][0].y * y[1] + a[rr][1].x * y[2] + a[rr][1].y * y[3];
  }
#pragma unroll
  for (int rr = 0; rr < 4; ++rr)
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) u[rr] += __shfl_xor_sync(0xffffffffu, u[rr], o);
  if (tx == 0) {
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int row = I * T + ty * 4 + rr;
      s[ty * 4 + rr] = (row < N ? f[row] : 0.0) - u[rr];
    }
  }
  __syncthreads();
  const double* D = Dinv + (int64_t)I * T * T;
  double w[4];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const double* dr = D + (ty * 4 + rr) * T + tx * 4;
    w[rr] = dr[0] * s[tx * 4] + dr[1] * s[tx * 4 + 1] + dr[2] * s[tx * 4 + 2] + dr[3] * s[tx * 4 + 3];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) w[rr] += __shfl_xor_sync(0xffffffffu, w[rr], o);
  }
  if (tx == 0) {
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) t[I * T + ty * 4 + rr] = w[rr];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicExch(flag + I, 1);
}

__global__ void __launch_bounds__(256)
    k_trsv_bwd(int N, int nt, const double* __restrict__ L, const double* __restrict__ Dinv,
               const double* t, double* y, double* yscratch, int* sync, const int* done) {
  if (done && *(volatile const int*)done) return;
  __shared__ int sI;
  __shared__ double sv[16][T + 1];
  __shared__ double s[T];
  if (threadIdx.x == 0) sI = nt - 1 - atomicAdd(&sync[1], 1);
  __syncthreads();
  const int I = sI;
  int* flag = sync + 2 + nt;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int J = nt - 1; J > I; --J) {
    const double* Lt = L + tile_index(J, I) * T * T;
    double2 a[4][2];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const double2* row = reinterpret_cast<const double2*>(Lt + (ty * 4 + rr) * T + tx * 4);
      a[rr][0] = __ldg(row);
      a[rr][1] = __ldg(row + 1);
    }
    spin_flag(flag + J);
    double xr[4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) xr[rr] = __ldcg(yscratch + J * T + ty * 4 + rr);
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      v[0] += a[rr][0].x * xr[rr];
      v[1] += a[rr][0].y * xr[rr];
      v[2] += a[rr][1].x * xr[rr];
      v[3] += a[rr][1].y * xr[rr];
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) sv[ty][tx * 4 + q] = v[q];
  __syncthreads();
  if (threadIdx.x < T) {
    double acc = 0.0;
#pragma unroll
    for (int g = 0; g < 16; ++g) acc += sv[g][threadIdx.x];
    s[threadIdx.x] = __ldcg(t + I * T + threadIdx.x) - acc;
  }
  __syncthreads();
  // x_I = L_II^-T s: x[c] = sum_r Dinv[r][c] s[r]
  const double* D = Dinv + (int64_t)I * T * T;
  double w[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const double sr = s[ty * 4 + rr];
    const double* dr = D + (ty * 4 + rr) * T + tx * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] += dr[q] * sr;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) sv[ty][tx * 4 + q] = w[q];
  __syncthreads();
  if (threadIdx.x < T) {
    double acc = 0.0;
#pragma unroll
    for (int g = 0; g < 16; ++g) acc += sv[g][threadIdx.x];
    const int row = I * T + threadIdx.x;
    yscratch[row] = acc;
    if (row < N) y[row] = acc;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicExch(flag + I, 1);
}

size_t trsv_sync_ints(int N) { return 2 + 2 * (size_t)div_up(N, T); }

void launch_trsv_packed(int N, const double* L, const double* Dinv, const double* f, double* t,
                        double* yscratch, double* y, int* sync, const int* done, cudaStream_t st) {
  if (N == 0) return;
  const int nt = div_up(N, T);
  MS_CUDA(cudaMemsetAsync(sync, 0, trsv_sync_ints(N) * sizeof(int), st));
  { k_trsv_fwd<<<nt, 256, 0, st>>>(N, nt, L, Dinv, f, t, sync, done); ms_count_launch(); }
  { k_trsv_bwd<<<nt, 256, 0, st>>>(N, nt, L, Dinv, t, y, yscratch, sync, done); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

size_t dense_spd_inverse_work_bytes(int N) {
  const int nt = div_up(N, T);
  return (size_t)packed_words(nt) * sizeof(double) * 2;
}

void dense_spd_inverse(int N, const double* A, double* packed_inv, double* work, int* fail,
                       cudaStream_t st) {
  if (N == 0) return;
  const int nt = div_up(N, T);
  double* P = work;
  double* W = work + packed_words(nt);
  { k_pack_tiles<<<148 * 8, 256, 0, st>>>(N, nt, A, P); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
  dense_spd_inverse_batched(nt, 1, P, W, packed_inv, fail, st);
}

// ---------------------------------------------------------------------------
// packed-tile SYMV (batch 1): per tile, u = X_IJ f_J (-> y_I) and, off the
// diagonal, v = X_IJ^T f_I (-> y_J); partials are reduced in a fixed order.
// Each CTA streams kSymvTilesPerCta consecutive tiles, the next tile's 32 KB
// loaded into registers while the current one is reduced (one short-lived CTA
// per tile left the loads of a tile exposed: 143 us for config 3's 584 MB).
constexpr int kSymvTilesPerCta = 8;

__global__ void __launch_bounds__(256)
    k_symv_tiles(int N, int nt, const double* __restrict__ X, const double* __restrict__ f,
                 double* __restrict__ part, const int* done, int64_t t_begin, int64_t t_end) {
  if (done && *(volatile const int*)done) return;
  __shared__ double sv[2][16][T + 1];
  const int64_t t0 = t_begin + (int64_t)blockIdx.x * kSymvTilesPerCta;
  const int64_t t1 = t0 + kSymvTilesPerCta < t_end ? t0 + kSymvTilesPerCta : t_end;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double2 cur[8], nxt[8];
  auto load = [&](int64_t t, double2(&dst)[8]) {
    const double* Xt = X + t * T * T;
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const double2* row = reinterpret_cast<const double2*>(Xt + (ty * 4 + rr) * T + tx * 4);
      dst[2 * rr] = __ldg(row);
      dst[2 * rr + 1] = __ldg(row + 1);
    }
  };
  load(t0, cur);
  int i, j;
  tile_ij(t0, i, j);
  for (int64_t t = t0; t < t1; ++t) {
    if (t + 1 < t1) load(t + 1, nxt);
    double fj[4], fi[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cj = j * T + tx * 4 + q, ri = i * T + ty * 4 + q;
      fj[q] = cj < N ? f[cj] : 0.0;
      fi[q] = ri < N ? f[ri] : 0.0;
    }
    double u[4], v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const double2 x01 = cur[2 * rr], x23 = cur[2 * rr + 1];
      u[rr] = x01.x * fj[0] + x01.y * fj[1] + x23.x * fj[2] + x23.y * fj[3];
      v[0] += x01.x * fi[rr];
      v[1] += x01.y * fi[rr];
      v[2] += x23.x * fi[rr];
      v[3] += x23.y * fi[rr];
    }
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) u[rr] += __shfl_xor_sync(0xffffffffu, u[rr], o);
    }
    double* pu = part + t * 2 * T;
    double* pv = pu + T;
    if (tx == 0) {
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) pu[ty * 4 + rr] = u[rr];
    }
    // the staging buffer alternates, so one barrier per tile (every tile, also
    // the diagonal ones that stage nothing) orders a buffer's readers before
    // its next writers
    double(*sb)[T + 1] = sv[(t - t0) & 1];
    if (i != j) {
#pragma unroll
      for (int q = 0; q < 4; ++q) sb[ty][tx * 4 + q] = v[q];
    }
    __syncthreads();
    if (i != j && threadIdx.x < T) {
      double s = 0.0;
#pragma unroll
      for (int g = 0; g < 16; ++g) s += sb[g][threadIdx.x];
      pv[threadIdx.x] = s;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
    if (++j > i) {  // next tile of the packed lower-triangular order
      ++i;
      j = 0;
    }
  }
}

// The same tile products with the tiles streamed by the bulk-copy (TMA)
// engine: a tile is 32 KB of contiguous packed storage, so one cp.async.bulk
// per tile fills a shared-memory stage; 2 CTAs per SM x kSymvStages tiles in
// flight, each CTA a contiguous range of tiles.  Per-thread arithmetic and
// the partial layout are those of k_symv_tiles (bitwise the same y).
constexpr int kSymvStages = 3;

__global__ void __launch_bounds__(256, 2)
    k_symv_bulk(int N, int nt, const double* __restrict__ X, const double* __restrict__ f,
                double* __restrict__ part, const int* done, int64_t t_begin, int64_t t_end, int per) {
  if (done && *(volatile const int*)done) return;
  extern __shared__ __align__(128) double stage[];  // kSymvStages tiles, then the mbarriers
  __shared__ double sv[2][16][T + 1];
  uint64_t* bar = reinterpret_cast<uint64_t*>(stage + kSymvStages * T * T);
  const int64_t t0 = t_begin + (int64_t)blockIdx.x * per;
  const int64_t t1 = t0 + per < t_end ? t0 + per : t_end;
  if (t0 >= t1) return;
  MS_BCHECK(t0 >= 0 && t1 <= (int64_t)nt * (nt + 1) / 2);  // the CTA's tile range lies in the packed matrix
  constexpr uint32_t kTileBytes = T * T * sizeof(double);
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < kSymvStages; ++s2) mbar_init(bar + s2, 1);
    mbar_fence_init();
    for (int s2 = 0; s2 < kSymvStages && t0 + s2 < t1; ++s2) {
      mbar_expect_tx(bar + s2, kTileBytes);
      bulk_g2s(stage + s2 * T * T, X + (t0 + s2) * T * T, kTileBytes, bar + s2);
    }
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  int i, j;
  tile_ij(t0, i, j);
  int st = 0;
  uint32_t phase = 0;
  for (int64_t t = t0; t < t1; ++t) {
    double fj[4], fi[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cj = j * T + tx * 4 + q, ri = i * T + ty * 4 + q;
      fj[q] = cj < N ? f[cj] : 0.0;
      fi[q] = ri < N ? f[ri] : 0.0;
    }
    mbar_wait(bar + st, (phase >> st) & 1u);
    phase ^= 1u << st;
    const double* Xt = stage + st * T * T;
    double u[4], v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const double2* row = reinterpret_cast<const double2*>(Xt + (ty * 4 + rr) * T + tx * 4);
      const double2 x01 = row[0], x23 = row[1];
      u[rr] = x01.x * fj[0] + x01.y * fj[1] + x23.x * fj[2] + x23.y * fj[3];
      v[0] += x01.x * fi[rr];
      v[1] += x01.y * fi[rr];
      v[2] += x23.x * fi[rr];
      v[3] += x23.y * fi[rr];
    }
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) u[rr] += __shfl_xor_sync(0xffffffffu, u[rr], o);
    }
    double* pu = part + t * 2 * T;
    double* pv = pu + T;
    if (tx == 0) {
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) pu[ty * 4 + rr] = u[rr];
    }
    double(*sb)[T + 1] = sv[(t - t0) & 1];
    if (i != j) {
#pragma unroll
      for (int q = 0; q < 4; ++q) sb[ty][tx * 4 + q] = v[q];
    }
    __syncthreads();  // every thread has read the stage; the v staging is complete
    if (threadIdx.x == 0 && t + kSymvStages < t1) {
      mbar_expect_tx(bar + st, kTileBytes);
      bulk_g2s(stage + st * T * T, X + (t + kSymvStages) * T * T, kTileBytes, bar + st);
    }
    if (i != j && threadIdx.x < T) {
      double s = 0.0;
#pragma unroll
      for (int g = 0; g < 16; ++g) s += sb[g][threadIdx.x];
      pv[threadIdx.x] = s;
    }
    st = (st + 1 == kSymvStages) ? 0 : st + 1;
    if (++j > i) {
      ++i;
      j = 0;
    }
  }
}

static int symv_variant() {
  // A/B knob, read per launch (tests toggle it): 0 = register-prefetch tiles, 1 = bulk-copy stages
  const char* e = getenv("MS_SYMV");
  return e ? atoi(e) : 1;
}

// y_I = sum_J u(I,J) + sum_{I'>I} v(I',I): 8 groups of 64 threads split the
// tile list, then a fixed-order combine -> deterministic.
constexpr int kRedGroups = 8;
__global__ void __launch_bounds__(T* kRedGroups)
    k_symv_reduce(int N, int nt, const double* __restrict__ part, double* __restrict__ y,
                  const int* done, int64_t t_begin, int64_t t_end) {
  if (done && *(volatile const int*)done) return;
  __shared__ double s[kRedGroups][T];
  const int I = blockIdx.x, r = threadIdx.x % T, grp = threadIdx.x / T;
  double acc = 0.0;
  for (int t = grp; t < nt; t += kRedGroups) {
    const int64_t ti = (t <= I) ? tile_index(I, t) : tile_index(t, I);
    if (ti < t_begin || ti >= t_end) continue;  // another rank's tiles (sharded coarse solve)
    acc += (t <= I) ? part[ti * 2 * T + r] : part[ti * 2 * T + T + r];
  }
  s[grp][r] = acc;
  __syncthreads();
  const int row = I * T + threadIdx.x;
  if (threadIdx.x < T && row < N) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kRedGroups; ++q) v += s[q][threadIdx.x];
    y[row] = v;
  }
}

void launch_symv_packed(int N, const double* X, const double* f, double* y, double* part,
                        const int* done, cudaStream_t st, int64_t t_begin, int64_t t_end) {
  if (N == 0) return;
  const int nt = div_up(N, T);
  if (t_end < 0) t_end = packed_tiles(nt);
  if (t_end > t_begin && symv_variant() == 1) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ntile = t_end - t_begin;
    const int ctas = (int)std::min<int64_t>(ntile, 2 * sms);
    const int per = div_up(ntile, ctas);
    const size_t smem = (size_t)kSymvStages * T * T * sizeof(double) + kSymvStages * sizeof(uint64_t);
    static bool configured[64] = {};
    if (dev >= 64 || !configured[dev]) {
      MS_CUDA(cudaFuncSetAttribute(k_symv_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if (dev < 64) configured[dev] = true;
    }
    { k_symv_bulk<<<div_up(ntile, per), 256, smem, st>>>(N, nt, X, f, part, done, t_begin, t_end, per); ms_count_launch(); }
  } else if (t_end > t_begin)
    { k_symv_tiles<<<(unsigned)div_up(t_end - t_begin, kSymvTilesPerCta), 256, 0, st>>>(N, nt, X, f, part, done,
                                                                                         t_begin, t_end); ms_count_launch(); }
  { k_symv_reduce<<<nt, T * kRedGroups, 0, st>>>(N, nt, part, y, done, t_begin, t_end); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Level-1 apply with explicit inverses: CTA per subdomain streams its
// packed_tiles(nt) tiles (4x4 doubles per thread, next tile prefetched into
// registers) and accumulates y in shared memory in tile order.
constexpr int kDenseApplyThreads = 256;

__global__ void __launch_bounds__(kDenseApplyThreads)
    k_l1_dense_apply(Grid g, const BandSys* __restrict__ sys, int nt, const double* __restrict__ X,
                     const double* __restrict__ r, double* __restrict__ ybuf, const int* done) {
  if (done && *(volatile const int*)done) return;
  extern __shared__ double sm[];
  const int NP = nt * T;
  double* f = sm;                 // NP
  double* y = f + NP;             // NP
  double* sv = y + NP;            // 16 x (T+1)
  double* su = sv + 16 * (T + 1); // T
  const BandSys s = sys[blockIdx.x];
  for (int i = threadIdx.x; i < NP; i += blockDim.x) {
    double v = 0.0;
    if (i < s.n) {
      const int ln = s.ncomp == 2 ? (i >> 1) : i, c = s.ncomp == 2 ? (i & 1) : 0;
      int a, b;
      band_node_of(s, ln, a, b);
      v = r[c * g.n_nodes + (int64_t)b * g.nnx + a];
    }
    f[i] = v;
    y[i] = 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const double* Xs = X + (int64_t)blockIdx.x * packed_words(nt);
  const int64_t ntiles = packed_tiles(nt);
  double2 cur[8], nxt[8];
  auto load = [&](int64_t t, double2(&dst)[8]) {
    const double* Xt = Xs + t * T * T;
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const double2* row = reinterpret_cast<const double2*>(Xt + (ty * 4 + rr) * T + tx * 4);
      dst[2 * rr] = __ldg(row);
      dst[2 * rr + 1] = __ldg(row + 1);
    }
  };
  load(0, cur);
  int i = 0, j = 0;
  for (int64_t t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles) load(t + 1, nxt);
    double fj[4], fi[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      fj[q] = f[j * T + tx * 4 + q];
      fi[q] = f[i * T + ty * 4 + q];
    }
    double u[4], v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const double2 x01 = cur[2 * rr], x23 = cur[2 * rr + 1];
      u[rr] = x01.x * fj[0] + x01.y * fj[1] + x23.x * fj[2] + x23.y * fj[3];
      v[0] += x01.x * fi[rr];
      v[1] += x01.y * fi[rr];
      v[2] += x23.x * fi[rr];
      v[3] += x23.y * fi[rr];
    }
#pragma unroll
    for (int rr = 0; rr < 4; ++rr)
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) u[rr] += __shfl_xor_sync(0xffffffffu, u[rr], o);
    if (tx == 0)
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) su[ty * 4 + rr] = u[rr];
#pragma unroll
    for (int q = 0; q < 4; ++q) sv[ty * (T + 1) + tx * 4 + q] = v[q];
    __syncthreads();
    if (threadIdx.x < T) {
      y[i * T + threadIdx.x] += su[threadIdx.x];
    } else if (threadIdx.x < 2 * T && i != j) {
      const int c = threadIdx.x - T;
      double sacc = 0.0;
#pragma unroll
      for (int gq = 0; gq < 16; ++gq) sacc += sv[gq * (T + 1) + c];
      y[j * T + c] += sacc;
    }
    __syncthreads();
    if (++j > i) {
      ++i;
      j = 0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
  }
  double* out = ybuf + s.yoff;
  for (int k = threadIdx.x; k < s.n; k += blockDim.x) out[k] = y[k];
}

void launch_l1_dense_apply(const Grid& g, const BandSys* sys, int nsys, int nt, const double* X,
                           const double* r, double* ybuf, const int* done, cudaStream_t st) {
  if (nsys == 0) return;
  const size_t smem = sizeof(double) * ((size_t)2 * nt * T + 16 * (T + 1) + T);
  if (smem > 220 * 1024) throw Error(-1, "subdomain too large for the dense level-1 apply");
  MS_CUDA(cudaFuncSetAttribute(k_l1_dense_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  { k_l1_dense_apply<<<nsys, kDenseApplyThreads, smem, st>>>(g, sys, nt, X, r, ybuf, done); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

}  // namespace msgpu
