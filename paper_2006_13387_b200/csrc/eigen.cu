// Batched local heat eigensolves: shift-invert block subspace iteration with
// Rayleigh-Ritz by one-sided-in-shared-memory Jacobi, one CTA per centre.
//
// Replaces the dense LAPACK ?sygvx call of the reference
// (`sla.eigh(K, M, subset_by_index=[0, k-1])`, spectral.py:93-100) on the
// neighbourhood heat pencil (spectral.py:63-90), followed by the gap rule
// (spectral.py:161-186).  The pencil is never formed densely: K_H and M_H are
// applied as 9-point stencils from the E tile in shared memory, and
// (K_H + sigma M_H)^{-1} comes from the batched banded Cholesky.  For a pure
// Neumann neighbourhood the constant (exact kernel, spectral.py:37-45) is
// locked and deflated from the block every pass.
#include <math_constants.h>

#include <algorithm>

#include "eigen.cuh"

namespace msgpu {

constexpr int P = kEigBlock;
constexpr int kEigThreads = 256;

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    k_heat_assemble(Grid g, const double* __restrict__ E, const uint8_t* __restrict__ hdir,
                    HeatParam hp, double sigma, const BandSys* __restrict__ sys,
                    double* __restrict__ Lc, const double* __restrict__ sigma_per_sys) {
  const BandSys s = sys[blockIdx.x];
  if (sigma_per_sys) sigma = sigma_per_sys[blockIdx.x];
  const int S = s.bw + 1;
  const int64_t total = (int64_t)s.n * S;
  const int ex_lo = s.a0, ex_hi = s.a0 + s.w - 2, ey_lo = s.b0, ey_hi = s.b0 + s.hgt - 2;
  for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
    const int k = (int)(t / S), j = (int)(t % S);
    const int row = k + j;
    double v = 0.0;
    if (row < s.n) {
      int ak, bk, ar, br;
      band_node_of(s, k, ak, bk);
      band_node_of(s, row, ar, br);
      const int64_t nk = (int64_t)bk * g.nnx + ak, nr = (int64_t)br * g.nnx + ar;
      if (hdir[nk] || hdir[nr]) {
        v = (row == k) ? 1.0 : 0.0;
      } else if (abs(ar - ak) <= 1 && abs(br - bk) <= 1) {
        const int ilo = max(max(ak, ar) - 1, ex_lo), ihi = min(min(ak, ar), ex_hi);
        const int jlo = max(max(bk, br) - 1, ey_lo), jhi = min(min(bk, br), ey_hi);
        double kv = 0.0, mv = 0.0;
        for (int ej = jlo; ej <= jhi; ++ej)
          for (int ei = ilo; ei <= ihi; ++ei) {
            const int dk = (ak - ei), ek = (bk - ej), dr = (ar - ei), er = (br - ej);
            const int ck = dk + 3 * ek - 2 * dk * ek, cr = dr + 3 * er - 2 * dr * er;
            const double Ee = E[(int64_t)ej * g.nx + ei];
            kv += Ee * hp.lap[cr * 4 + ck];
            mv += Ee * hp.mel[cr * 4 + ck];
          }
        v = kv + sigma * mv;
      }
    }
    Lc[s.foff + t] = v;
  }
}

void launch_heat_assemble(const Grid& g, const double* E, const uint8_t* hdir,
                          const HeatParam& hp, double sigma, const BandSys* sys, int nsys,
                          double* Lc, cudaStream_t st, const double* sigma_per_sys) {
  if (nsys == 0) return;
  { k_heat_assemble<<<nsys, 256, 0, st>>>(g, E, hdir, hp, sigma, sys, Lc, sigma_per_sys); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// subspace iteration

struct EigCtx {
  BandSys s;
  int n, nex, ney;
  const double* sE;
  const uint8_t* dir;
  const double* lap;
  const double* mel;
};

// (K v)_i or (M v)_i on the closed neighbourhood (Neumann outside), band order
__device__ __forceinline__ double stencil(const EigCtx& c, const double* __restrict__ v, int i,
                                          const double* coef) {
  int a, b;
  band_node_of(c.s, i, a, b);
  const int la = a - c.s.a0, lb = b - c.s.b0;
  double acc = 0.0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int ex = la - 1 + (e == 1 || e == 2), ey = lb - 1 + (e >= 2);
    if (ex < 0 || ey < 0 || ex >= c.nex || ey >= c.ney) continue;
    const int cn = (e == 0) ? 2 : (e == 1) ? 3 : (e == 2) ? 0 : 1;
    const int gx = c.s.a0 + ex, gy = c.s.b0 + ey;
    const double x0 = v[band_local_node(c.s, gx, gy)];
    const double x1 = v[band_local_node(c.s, gx + 1, gy)];
    const double x2 = v[band_local_node(c.s, gx + 1, gy + 1)];
    const double x3 = v[band_local_node(c.s, gx, gy + 1)];
    const double* cr = coef + cn * 4;
    acc += c.sE[ey * c.nex + ex] * (cr[0] * x0 + cr[1] * x1 + cr[2] * x2 + cr[3] * x3);
  }
  return acc;
}

// (M 1)_i
__device__ __forceinline__ double mass_ones(const EigCtx& c, int i) {
  int a, b;
  band_node_of(c.s, i, a, b);
  const int la = a - c.s.a0, lb = b - c.s.b0;
  double acc = 0.0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int ex = la - 1 + (e == 1 || e == 2), ey = lb - 1 + (e >= 2);
    if (ex < 0 || ey < 0 || ex >= c.nex || ey >= c.ney) continue;
    const int cn = (e == 0) ? 2 : (e == 1) ? 3 : (e == 2) ? 0 : 1;
    const double* cr = c.mel + cn * 4;
    acc += c.sE[ey * c.nex + ex] * (cr[0] + cr[1] + cr[2] + cr[3]);
  }
  return acc;
}

__device__ __forceinline__ double hash_unif(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return (double)(x >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

// deterministic reduction of `nv` (<= P+1) per-thread values; result in out[0..nv)
__device__ __forceinline__ void block_sum_multi(double (&v)[P + 1], int nv, double* red,
                                                double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < P + 1; ++t) {
    if (t < nv) {
      double x = warp_sum(v[t]);
      if (lane == 0) red[t * 8 + wid] = x;
    }
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kEigThreads / 32; ++w) s += red[threadIdx.x * 8 + w];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

template <int NV>
__device__ __forceinline__ void block_sum_nv(double (&v)[NV], int nv, double* red, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    if (t < nv) {
      double x = warp_sum(v[t]);
      if (lane == 0) red[t * 8 + wid] = x;
    }
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kEigThreads / 32; ++w) s += red[threadIdx.x * 8 + w];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// The P columns of W (column-major, length n) solved in place, one warp per
// column: forward sweep on Lc, backward on Lr, each warp with its own
// register window and no block barrier between steps (band_sweep,
// banded.cuh).  The warps move through the same factor in near lockstep, so
// its columns are served from L1/L2.  T register slots: bw <= 32 T.
template <int T>
__device__ void band_solve_cols(const BandSys& s, const double* __restrict__ Lc,
                                const double* __restrict__ Lr, double* W, int ncols) {
  __syncthreads();  // W complete
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = warp; c < ncols; c += nw) {
    double* y = W + (int64_t)c * s.n;
    band_sweep<T, 1, kPD, false>(Lc + s.foff, s.n, s.bw, y, lane);
    __syncwarp();
    band_sweep<T, 1, kPD, true>(Lr + s.foff, s.n, s.bw, y, lane);
    __syncwarp();
  }
  __syncthreads();
}

// As band_solve_cols for an even number of columns, two per warp sharing each
// band read: a column pair is interleaved into `scratch` (2 n doubles per
// pair, free while the solve runs), swept with NR = 2 and copied back.  The
// arithmetic of each column is that of the one-column sweep (bit-identical).
#ifndef MS_EIG_PD2
#define MS_EIG_PD2 8
#endif
constexpr int kPD2 = MS_EIG_PD2;  // band columns prefetched ahead in the two-column sweeps

template <int T>
__device__ void band_solve_cols2(const BandSys& s, const double* __restrict__ Lc,
                                 const double* __restrict__ Lr, double* W, double* scratch, int ncols) {
  __syncthreads();  // W complete, scratch free
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int n = s.n;
  for (int pr = warp; 2 * pr < ncols; pr += nw) {
    double* y0 = W + (int64_t)(2 * pr) * n;
    double* y1 = y0 + n;
    double* yi = scratch + (int64_t)pr * 2 * n;
    for (int i = lane; i < n; i += 32) {
      yi[2 * i] = y0[i];
      yi[2 * i + 1] = y1[i];
    }
    __syncwarp();
    band_sweep<T, 2, kPD2, false>(Lc + s.foff, n, s.bw, yi, lane);
    __syncwarp();
    band_sweep<T, 2, kPD2, true>(Lr + s.foff, n, s.bw, yi, lane);
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      y0[i] = yi[2 * i];
      y1[i] = yi[2 * i + 1];
    }
    __syncwarp();
  }
  __syncthreads();
}

// cyclic Jacobi on the B x B symmetric matrix A (row stride B+1), one warp;
// relative-threshold rotations keep small eigenvalues of graded matrices
// accurate.  On exit: ritz ascending, V columns in the same order.
template <int B = P>
__device__ void jacobi_warp(double* A, double* V, double* ritz, int* order) {
  const int lane = threadIdx.x & 31;
  constexpr int LD = B + 1;
  if (lane < B)
    for (int j = 0; j < B; ++j) V[lane * LD + j] = (lane == j) ? 1.0 : 0.0;
  __syncwarp();
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < B - 1; ++p)
      for (int q = p + 1; q < B; ++q) {
        const double app = A[p * LD + p], aqq = A[q * LD + q], apq = A[p * LD + q];
        if (apq == 0.0 || fabs(apq) <= 1e-17 * sqrt(fabs(app) * fabs(aqq))) continue;
        rotated = true;
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        __syncwarp();
        if (lane < B && lane != p && lane != q) {
          const double alp = A[lane * LD + p], alq = A[lane * LD + q];
          const double nlp = c * alp - s * alq, nlq = s * alp + c * alq;
          A[lane * LD + p] = nlp;
          A[p * LD + lane] = nlp;
          A[lane * LD + q] = nlq;
          A[q * LD + lane] = nlq;
        }
        if (lane < B) {
          const double vlp = V[lane * LD + p], vlq = V[lane * LD + q];
          V[lane * LD + p] = c * vlp - s * vlq;
          V[lane * LD + q] = s * vlp + c * vlq;
        }
        __syncwarp();
        if (lane == 0) {
          A[p * LD + p] = app - t * apq;
          A[q * LD + q] = aqq + t * apq;
          A[p * LD + q] = 0.0;
          A[q * LD + p] = 0.0;
        }
        __syncwarp();
      }
    if (!rotated) break;
  }
  if (lane == 0) {
    for (int i = 0; i < B; ++i) order[i] = i;
    for (int i = 0; i < B; ++i)  // selection sort (stable on ties by index)
      for (int j = i + 1; j < B; ++j)
        if (A[order[j] * LD + order[j]] < A[order[i] * LD + order[i]]) {
          const int t = order[i];
          order[i] = order[j];
          order[j] = t;
        }
    for (int i = 0; i < B; ++i) ritz[i] = A[order[i] * LD + order[i]];
  }
  __syncwarp();
}

template <int T>
__global__ void __launch_bounds__(kEigThreads)
    k_subspace(Grid g, const double* __restrict__ E, const uint8_t* __restrict__ hdir,
               HeatParam hp, EigBatch eb, int max_pass, double tol) {
  extern __shared__ double sm[];
  const int kb = blockIdx.x, k = eb.k0 + kb;
  const BandSys s = eb.sys[kb];
  const int n = s.n, S = s.bw + 1;
  const int nex = 2 * eb.mex, ney = 2 * eb.mey;
  constexpr int LD = P + 1;
  double* sE = sm;
  double* win = sE + nex * ney;
  double* red = win + S * P;
  double* dots = red + (P + 1) * 8;
  double* Am = dots + (P + 1);
  double* Vm = Am + P * LD;
  double* ritz = Vm + P * LD;
  double* ritz_old = ritz + P;
  double* misc = ritz_old + P;  // [0]: u1 scale^2, [1]: neumann, [2]: converged
  int* order = reinterpret_cast<int*>(misc + 4);
  uint8_t* dir = reinterpret_cast<uint8_t*>(order + P);
  __shared__ double hlap[16], hmel[16];
  if (threadIdx.x < 16) {
    hlap[threadIdx.x] = hp.lap[threadIdx.x];
    hmel[threadIdx.x] = hp.mel[threadIdx.x];
  }
  for (int t = threadIdx.x; t < nex * ney; t += blockDim.x)
    sE[t] = E[(int64_t)(s.b0 + t / nex) * g.nx + s.a0 + t % nex];
  int ndir = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int a, b;
    band_node_of(s, i, a, b);
    dir[i] = hdir[(int64_t)b * g.nnx + a];
    ndir += dir[i];
  }
  __syncthreads();
  const EigCtx ctx{s, n, nex, ney, sE, dir, hlap, hmel};
  double* X = eb.work + (int64_t)kb * 2 * P * n;
  double* W = X + (int64_t)P * n;
  double v[P + 1];
  {
    v[0] = (double)ndir;
    double m1 = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m1 += mass_ones(ctx, i);
    v[1] = m1;
    block_sum_multi(v, 2, red, dots);
  }
  const bool neumann = dots[0] == 0.0;
  const double u1s2 = 1.0 / dots[1];  // (1/sqrt(1^T M 1))^2
  // random start, zero on Dirichlet nodes
  for (int t = threadIdx.x; t < n * P; t += blockDim.x) {
    const int c = t / n, i = t % n;
    X[t] = dir[i] ? 0.0 : hash_unif(((uint64_t)k << 32) ^ ((uint64_t)c << 24) ^ (uint64_t)i);
  }
  if (threadIdx.x < P) ritz_old[threadIdx.x] = 0.0;
  if (threadIdx.x == 0) misc[3] = -1.0;
  __syncthreads();
  const int need = kNeig - (neumann ? 1 : 0);
  int pass = 0;
  for (pass = 1; pass <= max_pass; ++pass) {
    // (1) W = M X, zero rows at Dirichlet nodes
    for (int t = threadIdx.x; t < n * P; t += blockDim.x) {
      const int c = t / n, i = t % n;
      W[t] = dir[i] ? 0.0 : stencil(ctx, X + (int64_t)c * n, i, hmel);
    }
    __syncthreads();
    // (2) W <- (K + sigma M)^{-1} W (X is dead until (3) rewrites it: scratch)
    static_assert(P % 2 == 0, "column pairs");
    band_solve_cols2<T>(s, eb.Lc, eb.Lr, W, X, P);
    // (3) M-orthonormalise W into X (CGS2 against the constant and earlier columns)
    for (int c = 0; c < P; ++c) {
      double* w = W + (int64_t)c * n;
      for (int rep = 0; rep < 2; ++rep) {
#pragma unroll
        for (int l = 0; l < P + 1; ++l) v[l] = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          const double mw = stencil(ctx, w, i, hmel);
#pragma unroll
          for (int l = 0; l < P; ++l)
            if (l < c) v[l] += mw * X[(int64_t)l * n + i];
          if (neumann) v[P] += mass_ones(ctx, i) * w[i];
        }
        block_sum_multi(v, P + 1, red, dots);
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          double x = w[i];
          for (int l = 0; l < c; ++l) x -= dots[l] * X[(int64_t)l * n + i];
          if (neumann && !dir[i]) x -= dots[P] * u1s2;
          w[i] = x;
        }
        __syncthreads();
      }
      double nrm = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) nrm += w[i] * stencil(ctx, w, i, hmel);
      v[0] = nrm;
      block_sum_multi(v, 1, red, dots);
      const double inv = dots[0] > 0.0 ? 1.0 / sqrt(dots[0]) : 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) X[(int64_t)c * n + i] = w[i] * inv;
      __syncthreads();
    }
    // (4) Rayleigh-Ritz matrix Kr = X^T K X
    for (int c = 0; c < P; ++c) {
#pragma unroll
      for (int l = 0; l < P + 1; ++l) v[l] = 0.0;
      const double* xc = X + (int64_t)c * n;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double kx = dir[i] ? 0.0 : stencil(ctx, xc, i, hlap);
#pragma unroll
        for (int l = 0; l < P; ++l)
          if (l <= c) v[l] += kx * X[(int64_t)l * n + i];
      }
      block_sum_multi(v, c + 1, red, dots);
      if (threadIdx.x <= c) {
        Am[threadIdx.x * LD + c] = dots[threadIdx.x];
        Am[c * LD + threadIdx.x] = dots[threadIdx.x];
      }
      __syncthreads();
    }
    // (5) Jacobi
    if (threadIdx.x < 32) jacobi_warp(Am, Vm, ritz, order);
    __syncthreads();
    // (6) X <- X V (Ritz order), node rows in registers
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double xr[P];
#pragma unroll
      for (int l = 0; l < P; ++l) xr[l] = X[(int64_t)l * n + i];
#pragma unroll
      for (int c = 0; c < P; ++c) {
        const int oc = order[c];
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) acc += xr[l] * Vm[l * LD + oc];
        W[(int64_t)c * n + i] = acc;
      }
    }
    __syncthreads();
    {
      double* t = X;
      X = W;
      W = t;
    }
    // (7) stopping rule.  Only the selection needs the 7 eigenvalues, and only
    // the selected modes' vectors enter the coarse space: the selected Ritz
    // values must be converged to `tol` (their subspace sits below a gap of
    // >= threshold, so it converges fast), the remaining ones to 1e-8 relative
    // (enough to certify the gap tests), and the provisional selection must be
    // the same as in the previous pass.
    if (threadIdx.x == 0) {
      const double scale = fabs(ritz[P - 1]);
      const int off = neumann ? 1 : 0;
      double lam[kNeig];
      if (neumann) lam[0] = 0.0;
      for (int i = 0; i < kNeig - off; ++i) lam[i + off] = ritz[i];
      int sel = eb.fixed ? eb.n_max : 1;
      if (!eb.fixed) {
        const int wn = min(eb.n_max + 1, kNeig);
        const double last = lam[wn - 1];
        const double eps = last != 0.0 ? 1e-14 * fabs(last) : 1e-300;
        for (int i = 1; i < wn; ++i)
          if (lam[i] / fmax(lam[i - 1], eps) >= eb.gap) sel = i;
        sel = min(sel, eb.n_max);
      }
      bool conv = pass >= 3 && sel == (int)misc[3];
      for (int i = 0; i < need; ++i) {
        const double t = (i + off < sel) ? tol : 1e-8;
        // absolute floor: Ritz values of tiny (island) modes jitter at the
        // round-off level eps * lambda_max of the pencil
        if (fabs(ritz[i] - ritz_old[i]) > t * fabs(ritz[i]) + fmax(1e-15 * scale, eb.lam_floor))
          conv = false;
      }
      for (int i = 0; i < P; ++i) ritz_old[i] = ritz[i];
      misc[3] = (double)sel;
      misc[2] = conv ? 1.0 : 0.0;
    }
    __syncthreads();
    if (misc[2] != 0.0) break;
  }
  // outputs: kNeig lowest pairs, ascending
  double* ev = eb.evecs + (int64_t)kb * kNeig * n;
  if (neumann) {
    // locked constant: lambda = 1^T K 1 / 1^T M 1 (round-off level)
    double kk = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      int a, b;
      band_node_of(s, i, a, b);
      const int la = a - s.a0, lb = b - s.b0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ex = la - 1 + (e == 1 || e == 2), ey = lb - 1 + (e >= 2);
        if (ex < 0 || ey < 0 || ex >= nex || ey >= ney) continue;
        const int cn = (e == 0) ? 2 : (e == 1) ? 3 : (e == 2) ? 0 : 1;
        kk += sE[ey * nex + ex] * (hlap[cn * 4] + hlap[cn * 4 + 1] + hlap[cn * 4 + 2] + hlap[cn * 4 + 3]);
      }
    }
    v[0] = kk;
    block_sum_multi(v, 1, red, dots);
    const double u1 = sqrt(u1s2);
    for (int i = threadIdx.x; i < n; i += blockDim.x) ev[i] = u1;
    if (threadIdx.x == 0) eb.evals[(int64_t)k * kNeig] = dots[0] * u1s2;
  }
  const int off = neumann ? 1 : 0;
  for (int t = threadIdx.x; t < (kNeig - off) * n; t += blockDim.x) {
    const int m = t / n, i = t % n;
    ev[(int64_t)(m + off) * n + i] = X[(int64_t)m * n + i];
  }
  if (threadIdx.x < kNeig - off) eb.evals[(int64_t)k * kNeig + off + threadIdx.x] = ritz[threadIdx.x];
  if (threadIdx.x == 0) {
    eb.passes[k] = min(pass, max_pass);
    eb.neumann[k] = neumann ? 1 : 0;
  }
}

// register slots T of the eigensolver's band sweeps: bw <= 32 T
template <template <int> class Launch, typename... A>
static void band_dispatch(int max_bw, A... args) {
  switch (std::max(1, div_up(max_bw, 32))) {
    case 1: Launch<1>::run(args...); break;
    case 2: Launch<2>::run(args...); break;
    case 3: Launch<3>::run(args...); break;
    case 4: Launch<4>::run(args...); break;
    case 5: Launch<5>::run(args...); break;
    case 6: Launch<6>::run(args...); break;
    default: throw Error(-1, "neighbourhood band too wide for the eigensolver (coarse blocks <= 46 elements)");
  }
}

template <int T>
struct SubspaceLaunch {
  static void run(const Grid& g, const double* E, const uint8_t* hdir, const HeatParam& hp, const EigBatch& b,
                  int max_pass, double tol, size_t smem, cudaStream_t st) {
    MS_CUDA(cudaFuncSetAttribute(k_subspace<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    { k_subspace<T><<<b.nk, kEigThreads, smem, st>>>(g, E, hdir, hp, b, max_pass, tol); ms_count_launch(); }
    MS_CUDA(cudaGetLastError());
  }
};

void launch_subspace(const Grid& g, const double* E, const uint8_t* hdir, const HeatParam& hp,
                     const EigBatch& b, int max_pass, double tol, cudaStream_t st) {
  if (b.nk == 0) return;
  int max_bw = 0, max_n = 0;
  // host copy of the batch's systems is not available here; bounds from geometry
  const int NLx = 2 * b.mex + 1, NLy = 2 * b.mey + 1;
  max_bw = std::min(NLx, NLy) + 1;
  max_n = NLx * NLy;
  const size_t smem = sizeof(double) * ((size_t)(2 * b.mex) * (2 * b.mey) + (size_t)(max_bw + 1) * P +
                                        (P + 1) * 8 + (P + 1) + 2 * P * (P + 1) + 2 * P + 4) +
                      sizeof(int) * P + (size_t)max_n + 16;
  if (smem > 220 * 1024) throw Error(-1, "neighbourhood too large for the eigensolver tile");
  band_dispatch<SubspaceLaunch>(max_bw, g, E, hdir, hp, b, max_pass, tol, smem, st);
}

// ---------------------------------------------------------------------------
// Randomized snapshot eigensolver, EH+Rot;Rand (spectral.py:103-158), one CTA
// per centre.  Same algorithm as the reference on the same forcings (host
// PCG64, seeds [seed, centre]) and the same shift sigma = 1e-8 tr(K)/n:
// F -= MZ (Z^T F)/G; U = deflate(B^-1 F); 3 x { U = orth(U); U = deflate(B^-1 M U) };
// Q = orthonormal basis of [U, Z] (1e-10 rank cut); Rayleigh-Ritz on (Q^T K Q,
// Q^T M Q).  Z = 1 on free nodes, deflate(X) = X - Z (MZ^T X)/G.
template <int B = P>
__device__ void cgs2_euclid(double* cols, int ncols, int n, double* red, double* dots,
                            double* keep_flag) {
  // in place Euclidean CGS2 of `ncols` columns; zeroes columns that vanish
  double v[B + 1];
  for (int c = 0; c < ncols; ++c) {
    double* w = cols + (int64_t)c * n;
    double nrm0 = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) nrm0 += w[i] * w[i];
#pragma unroll
    for (int l = 0; l < B + 1; ++l) v[l] = 0.0;
    v[0] = nrm0;
    block_sum_nv<B + 1>(v, 1, red, dots);
    nrm0 = dots[0];
    for (int rep = 0; rep < 2; ++rep) {
#pragma unroll
      for (int l = 0; l < B + 1; ++l) v[l] = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
#pragma unroll
        for (int l = 0; l < B; ++l)
          if (l < c) v[l] += cols[(int64_t)l * n + i] * w[i];
      }
      block_sum_nv<B + 1>(v, B + 1, red, dots);
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double x = w[i];
        for (int l = 0; l < c; ++l) x -= dots[l] * cols[(int64_t)l * n + i];
        w[i] = x;
      }
      __syncthreads();
    }
    double nrm = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) nrm += w[i] * w[i];
#pragma unroll
    for (int l = 0; l < B + 1; ++l) v[l] = 0.0;
    v[0] = nrm;
    block_sum_nv<B + 1>(v, 1, red, dots);
    const bool ok = dots[0] > 1e-20 * nrm0 && dots[0] > 0.0;
    const double inv = ok ? 1.0 / sqrt(dots[0]) : 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) w[i] *= inv;
    if (threadIdx.x == 0 && keep_flag) keep_flag[c] = ok ? 1.0 : 0.0;
    __syncthreads();
  }
}

template <int T, int B>
__global__ void __launch_bounds__(kEigThreads)
    k_randomized(Grid g, const double* __restrict__ E, const uint8_t* __restrict__ hdir,
                 HeatParam hp, EigBatch eb, const double* __restrict__ F, int ns, int nlx) {
  extern __shared__ double sm[];
  const int kb = blockIdx.x, k = eb.k0 + kb;
  const BandSys s = eb.sys[kb];
  const int n = s.n, S = s.bw + 1;
  const int nex = 2 * eb.mex, ney = 2 * eb.mey;
  constexpr int LD = B + 1;
  double* sE = sm;
  double* win = sE + nex * ney;
  double* red = win + S * B;
  double* dots = red + (B + 1) * 8;
  double* Am = dots + (B + 1);
  double* Vm = Am + B * LD;
  double* ritz = Vm + B * LD;
  double* keep = ritz + B;  // B flags
  double* misc = keep + B;
  int* order = reinterpret_cast<int*>(misc + 4);
  uint8_t* dir = reinterpret_cast<uint8_t*>(order + B);
  __shared__ double hlap[16], hmel[16];
  __shared__ double Lm[B][B + 1], Cm[B][B + 1];
  if (threadIdx.x < 16) {
    hlap[threadIdx.x] = hp.lap[threadIdx.x];
    hmel[threadIdx.x] = hp.mel[threadIdx.x];
  }
  for (int t = threadIdx.x; t < nex * ney; t += blockDim.x)
    sE[t] = E[(int64_t)(s.b0 + t / nex) * g.nx + s.a0 + t % nex];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int a, b;
    band_node_of(s, i, a, b);
    dir[i] = hdir[(int64_t)b * g.nnx + a];
  }
  __syncthreads();
  const EigCtx ctx{s, n, nex, ney, sE, dir, hlap, hmel};
  double* X = eb.work + (int64_t)kb * 2 * B * n;  // cols 0..B-3: basis; B-2: MZ; B-1: Z
  double* W = X + (int64_t)B * n;                 // solve workspace
  double* Zc = X + (int64_t)(B - 1) * n;
  double* MZ = X + (int64_t)(B - 2) * n;
  double v[B + 1];
  for (int i = threadIdx.x; i < n; i += blockDim.x) Zc[i] = dir[i] ? 0.0 : 1.0;
  __syncthreads();
  double G;
  {
#pragma unroll
    for (int l = 0; l < B + 1; ++l) v[l] = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double mz = dir[i] ? 0.0 : stencil(ctx, Zc, i, hmel);
      MZ[i] = mz;
      v[0] += Zc[i] * mz;
    }
    block_sum_nv<B + 1>(v, 1, red, dots);
    G = dots[0];
  }
  // forcings (lexicographic node index in F -> band order)
  const double* Fk = F + (int64_t)kb * ns * (nlx * (n / nlx));
  for (int t = threadIdx.x; t < n * B; t += blockDim.x) {
    const int c = t / n, i = t % n;
    double val = 0.0;
    if (c < ns && !dir[i]) {
      int a, b;
      band_node_of(s, i, a, b);
      val = Fk[(int64_t)c * n + (a - s.a0) + (int64_t)(b - s.b0) * nlx];
    }
    W[t] = val;
  }
  __syncthreads();
  // F -= MZ (Z^T F) / G
  {
#pragma unroll
    for (int l = 0; l < B + 1; ++l) v[l] = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
      for (int c = 0; c < B; ++c)
        if (c < ns) v[c] += Zc[i] * W[(int64_t)c * n + i];
    block_sum_nv<B + 1>(v, B + 1, red, dots);
    for (int t = threadIdx.x; t < n * ns; t += blockDim.x) {
      const int c = t / n, i = t % n;
      W[t] -= MZ[i] * (dots[c] / G);
    }
    __syncthreads();
  }
  auto deflate = [&]() {
#pragma unroll
    for (int l = 0; l < B + 1; ++l) v[l] = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
      for (int c = 0; c < B; ++c)
        if (c < ns) v[c] += MZ[i] * W[(int64_t)c * n + i];
    block_sum_nv<B + 1>(v, B + 1, red, dots);
    for (int t = threadIdx.x; t < n * ns; t += blockDim.x) {
      const int c = t / n, i = t % n;
      W[t] -= Zc[i] * (dots[c] / G);
    }
    __syncthreads();
  };
  band_solve_cols<T>(s, eb.Lc, eb.Lr, W, ns);
  deflate();
  for (int pass = 1; pass < 4; ++pass) {
    cgs2_euclid<B>(W, ns, n, red, dots, nullptr);
    for (int t = threadIdx.x; t < n * ns; t += blockDim.x) {
      const int c = t / n, i = t % n;
      X[t] = dir[i] ? 0.0 : stencil(ctx, W + (int64_t)c * n, i, hmel);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n * ns; t += blockDim.x) W[t] = X[t];
    __syncthreads();
    band_solve_cols<T>(s, eb.Lc, eb.Lr, W, ns);
    deflate();
  }
  // Q = orthonormal basis of [U, Z] (columns normalised first, 1e-10 rank cut)
  const int m0 = ns + 1;
  for (int t = threadIdx.x; t < n * m0; t += blockDim.x) {
    const int c = t / n, i = t % n;
    X[t] = (c < ns) ? W[t] : Zc[i];
  }
  __syncthreads();
  cgs2_euclid<B>(X, m0, n, red, dots, keep);
  int m = 0;
  if (threadIdx.x == 0) {
    // compact kept columns to the front (order preserved)
    int q = 0;
    for (int c = 0; c < m0; ++c)
      if (keep[c] != 0.0) order[q++] = c;
    misc[0] = (double)q;
  }
  __syncthreads();
  m = (int)misc[0];
  for (int q = 0; q < m; ++q) {
    const int c = order[q];
    if (c != q)
      for (int i = threadIdx.x; i < n; i += blockDim.x) X[(int64_t)q * n + i] = X[(int64_t)c * n + i];
    __syncthreads();
  }
  // Kr (-> Am) and Mr (-> Cm), column by column
  for (int pass = 0; pass < 2; ++pass) {
    const double* coef = pass == 0 ? hlap : hmel;
    for (int c = 0; c < m; ++c) {
#pragma unroll
      for (int l = 0; l < B + 1; ++l) v[l] = 0.0;
      const double* xc = X + (int64_t)c * n;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double ax = dir[i] ? 0.0 : stencil(ctx, xc, i, coef);
#pragma unroll
        for (int l = 0; l < B; ++l)
          if (l <= c) v[l] += ax * X[(int64_t)l * n + i];
      }
      block_sum_nv<B + 1>(v, c + 1, red, dots);
      if (threadIdx.x <= c) {
        if (pass == 0)
          Am[threadIdx.x * LD + c] = Am[c * LD + threadIdx.x] = dots[threadIdx.x];
        else
          Cm[threadIdx.x][c] = Cm[c][threadIdx.x] = dots[threadIdx.x];
      }
      __syncthreads();
    }
  }
  // generalized m x m eigenproblem: Mr = L L^T, C = L^-1 Kr L^-T (thread 0),
  // Jacobi on C padded to B x B with a huge diagonal
  if (threadIdx.x == 0) {
    for (int i = 0; i < m; ++i)
      for (int j = 0; j <= i; ++j) {
        double a = Cm[i][j];
        for (int q = 0; q < j; ++q) a -= Lm[i][q] * Lm[j][q];
        Lm[i][j] = (i == j) ? sqrt(fmax(a, 1e-300)) : a / Lm[j][j];
      }
    // T = L^-1 Kr (rows), then C = T L^-T
    for (int c = 0; c < m; ++c)
      for (int i = 0; i < m; ++i) {
        double a = Am[i * LD + c];
        for (int q = 0; q < i; ++q) a -= Lm[i][q] * Cm[q][c];
        Cm[i][c] = a / Lm[i][i];
      }
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        double a = Cm[i][j];
        for (int q = 0; q < j; ++q) a -= Am[i * LD + q] * Lm[j][q];
        Am[i * LD + j] = a / Lm[j][j];  // reuse Am as C (row i done before being read)
      }
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < B; ++j)
        if (i >= m || j >= m) Am[i * LD + j] = (i == j) ? 1e300 : 0.0;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < i; ++j) Am[i * LD + j] = Am[j * LD + i] = 0.5 * (Am[i * LD + j] + Am[j * LD + i]);
  }
  __syncthreads();
  if (threadIdx.x < 32) jacobi_warp<B>(Am, Vm, ritz, order);
  __syncthreads();
  // Ritz vectors: x = Q (L^-T y), y = Vm[:, order[c]]
  if (threadIdx.x == 0) {
    for (int c = 0; c < kNeig && c < m; ++c) {
      const int oc = order[c];
      for (int i = m - 1; i >= 0; --i) {
        double a = Vm[i * LD + oc];
        for (int q = i + 1; q < m; ++q) a -= Lm[q][i] * Cm[q][c];
        Cm[i][c] = a / Lm[i][i];  // coefficients of Ritz vector c
      }
    }
  }
  __syncthreads();
  double* ev = eb.evecs + (int64_t)kb * kNeig * n;
  const int kk = min(kNeig, m);
  for (int t = threadIdx.x; t < kNeig * n; t += blockDim.x) {
    const int c = t / n, i = t % n;
    double a = 0.0;
    if (c < kk)
      for (int q = 0; q < m; ++q) a += X[(int64_t)q * n + i] * Cm[q][c];
    ev[t] = a;
  }
  if (threadIdx.x < kNeig)
    eb.evals[(int64_t)k * kNeig + threadIdx.x] = threadIdx.x < kk ? ritz[threadIdx.x] : CUDART_NAN;
  if (threadIdx.x == 0) {
    eb.passes[k] = 4;
    eb.neumann[k] = 0;
  }
}

// sigma_k = 1e-8 * tr(K_free) / n_free on the closed neighbourhood (spectral.py:133)
__global__ void k_rand_sigma(Grid g, const double* __restrict__ E, const uint8_t* __restrict__ hdir,
                             HeatParam hp, const BandSys* __restrict__ sys, double* __restrict__ sigma) {
  __shared__ double sred[8];
  const BandSys s = sys[blockIdx.x];
  double tr = 0.0, nf = 0.0;
  for (int i = threadIdx.x; i < s.n; i += blockDim.x) {
    int a, b;
    band_node_of(s, i, a, b);
    if (hdir[(int64_t)b * g.nnx + a]) continue;
    nf += 1.0;
    // K_ii = sum over the node's elements inside the neighbourhood of E_e * lap[c][c]
    for (int e = 0; e < 4; ++e) {
      const int ei = a - 1 + (e == 1 || e == 2), ej = b - 1 + (e >= 2);
      if (ei < s.a0 || ej < s.b0 || ei > s.a0 + s.w - 2 || ej > s.b0 + s.hgt - 2) continue;
      const int cn = (e == 0) ? 2 : (e == 1) ? 3 : (e == 2) ? 0 : 1;
      tr += E[(int64_t)ej * g.nx + ei] * hp.lap[cn * 4 + cn];
    }
  }
  const double t = block_sum(tr, sred), m = block_sum(nf, sred);
  if (threadIdx.x == 0) sigma[blockIdx.x] = 1e-8 * (t / m);
}

void launch_rand_sigma(const Grid& g, const double* E, const uint8_t* hdir, const HeatParam& hp,
                       const BandSys* sys, int nsys, double* sigma, cudaStream_t st) {
  if (nsys == 0) return;
  { k_rand_sigma<<<nsys, 256, 0, st>>>(g, E, hdir, hp, sys, sigma); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// block size of the randomized solvers: 16 while the snapshots fit next to
// the kernel candidates (the common n_max + 5 = 11), else 32
int randomized_block(int ns) { return ns + 3 <= kEigBlock ? kEigBlock : 32; }

template <int T>
struct RandomizedLaunch {
  template <int B>
  static void go(const Grid& g, const double* E, const uint8_t* hdir, const HeatParam& hp, const EigBatch& b,
                 const double* F, int ns, int nlx, int max_bw, cudaStream_t st) {
    const int NLy = 2 * b.mey + 1;
    const size_t smem = sizeof(double) * ((size_t)(2 * b.mex) * (2 * b.mey) + (size_t)(max_bw + 1) * B +
                                          (B + 1) * 8 + (B + 1) + 2 * B * (B + 1) + 2 * B + 4) +
                        sizeof(int) * B + (size_t)nlx * NLy + 16;
    MS_CUDA(cudaFuncSetAttribute(k_randomized<T, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    { k_randomized<T, B><<<b.nk, kEigThreads, smem, st>>>(g, E, hdir, hp, b, F, ns, nlx); ms_count_launch(); }
    MS_CUDA(cudaGetLastError());
  }
  static void run(const Grid& g, const double* E, const uint8_t* hdir, const HeatParam& hp, const EigBatch& b,
                  const double* F, int ns, int nlx, int max_bw, cudaStream_t st) {
    if (randomized_block(ns) == kEigBlock)
      go<kEigBlock>(g, E, hdir, hp, b, F, ns, nlx, max_bw, st);
    else
      go<32>(g, E, hdir, hp, b, F, ns, nlx, max_bw, st);
  }
};

void launch_randomized(const Grid& g, const double* E, const uint8_t* hdir, const HeatParam& hp,
                       const EigBatch& b, const double* F, int ns, cudaStream_t st) {
  if (b.nk == 0) return;
  if (ns + 3 > 32) throw Error(-1, "too many snapshots for the randomized eigensolver (<= 29)");
  const int NLx = 2 * b.mex + 1, NLy = 2 * b.mey + 1;
  const int max_bw = std::min(NLx, NLy) + 1;
  band_dispatch<RandomizedLaunch>(max_bw, g, E, hdir, hp, b, F, ns, NLx, max_bw, st);
}

// ---------------------------------------------------------------------------
__global__ void k_select(int n_centers, const double* __restrict__ evals, int n_max,
                         double threshold, int fixed, int* __restrict__ nsel) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_centers) return;
  const double* lam = evals + (int64_t)k * kNeig;
  const int wn = min(n_max + 1, kNeig);
  if (fixed) {
    nsel[k] = min(n_max, kNeig);
    return;
  }
  const double last = lam[wn - 1];
  const double eps = last != 0.0 ? 1e-14 * fabs(last) : 1e-300;
  int sel = 1;
  for (int i = 1; i < wn; ++i)
    if (lam[i] / fmax(lam[i - 1], eps) >= threshold) sel = i;
  nsel[k] = min(sel, n_max);
}

void launch_select(int n_centers, const double* evals, int n_max, double threshold, int fixed,
                   int* nsel, cudaStream_t st) {
  if (n_centers == 0) return;
  { k_select<<<div_up(n_centers, 128), 128, 0, st>>>(n_centers, evals, n_max, threshold, fixed, nsel); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

__global__ void __launch_bounds__(256)
    k_compact_psi(EigBatch eb, int NLx, const int* __restrict__ nsel,
                  const int64_t* __restrict__ psioff, double* __restrict__ psi) {
  __shared__ double sval[8];
  __shared__ int sidx[8];
  const int kb = blockIdx.x, k = eb.k0 + kb;
  const BandSys s = eb.sys[kb];
  const int n = s.n;
  const double* ev = eb.evecs + (int64_t)kb * kNeig * n;
  for (int m = 0; m < nsel[k]; ++m) {
    const double* vm = ev + (int64_t)m * n;
    // argmax |v| in lexicographic order (ties: smallest index)
    double best = -1.0;
    int bidx = 0x7fffffff;
    for (int ln = threadIdx.x; ln < n; ln += blockDim.x) {
      const int a = s.a0 + ln % NLx, b = s.b0 + ln / NLx;
      const double x = fabs(vm[band_local_node(s, a, b)]);
      if (x > best || (x == best && ln < bidx)) {
        best = x;
        bidx = ln;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ob > best || (ob == best && oi < bidx)) {
        best = ob;
        bidx = oi;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      sval[threadIdx.x >> 5] = best;
      sidx[threadIdx.x >> 5] = bidx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < 8; ++w)
        if (sval[w] > sval[0] || (sval[w] == sval[0] && sidx[w] < sidx[0])) {
          sval[0] = sval[w];
          sidx[0] = sidx[w];
        }
    }
    __syncthreads();
    const int ib = sidx[0];
    const double sign =
        vm[band_local_node(s, s.a0 + ib % NLx, s.b0 + ib / NLx)] < 0.0 ? -1.0 : 1.0;
    double* out = psi + psioff[k] + (int64_t)m * n;
    for (int ln = threadIdx.x; ln < n; ln += blockDim.x) {
      const int a = s.a0 + ln % NLx, b = s.b0 + ln / NLx;
      out[ln] = sign * vm[band_local_node(s, a, b)];
    }
    __syncthreads();
  }
}

void launch_compact_psi(const EigBatch& b, int NLx, const int* nsel, const int64_t* psioff,
                        double* psi, cudaStream_t st) {
  if (b.nk == 0) return;
  { k_compact_psi<<<b.nk, 256, 0, st>>>(b, NLx, nsel, psioff, psi); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ===========================================================================
// Elasticity eigenproblems (EE, EE;Rand).  Same machinery as the heat kind on
// the two-component pencil: K_E = sum E_e k0 over the neighbourhood's elements
// (Neumann outside, whole-node Dirichlet at clamped nodes), M_E = sum E_e
// blockdiag(m_e, m_e) (assembly.py:236-259), unknowns node-interleaved.  On
// a pure Neumann neighbourhood the three rigid-body modes -- the exact kernel
// (spectral.py:37-45, assembly.py:262-273) -- are M-orthonormalised, locked
// and deflated, so the iteration only resolves the remaining kNeig - 3 pairs.

struct EigCtxE {
  BandSys s;
  int n, nex, ney;
  const double* sE;
  const uint8_t* dirn;  // per band-order node
  const double* ke;
  const double* mel;
};

// (K v)_i (mass = false) or (M v)_i on the closed neighbourhood, i = 2 ln + c
__device__ __forceinline__ double el_stencil(const EigCtxE& c, const double* __restrict__ v, int i,
                                             bool mass) {
  const int ln = i >> 1, comp = i & 1;
  int a, b;
  band_node_of(c.s, ln, a, b);
  const int la = a - c.s.a0, lb = b - c.s.b0;
  double acc = 0.0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int ex = la - 1 + (e == 1 || e == 2), ey = lb - 1 + (e >= 2);
    if (ex < 0 || ey < 0 || ex >= c.nex || ey >= c.ney) continue;
    const int cn = (e == 0) ? 2 : (e == 1) ? 3 : (e == 2) ? 0 : 1;
    const int gx = c.s.a0 + ex, gy = c.s.b0 + ey;
    const int l[4] = {band_local_node(c.s, gx, gy), band_local_node(c.s, gx + 1, gy),
                      band_local_node(c.s, gx + 1, gy + 1), band_local_node(c.s, gx, gy + 1)};
    double sacc = 0.0;
    if (mass) {
      const double* mr = c.mel + cn * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) sacc += mr[q] * v[2 * l[q] + comp];
    } else {
      const double* kr = c.ke + (comp * 4 + cn) * 8;
#pragma unroll
      for (int q = 0; q < 4; ++q) sacc += kr[q] * v[2 * l[q]] + kr[4 + q] * v[2 * l[q] + 1];
    }
    acc += c.sE[ey * c.nex + ex] * sacc;
  }
  return acc;
}

__global__ void __launch_bounds__(256)
    k_el_assemble(Grid g, const double* __restrict__ E, const uint8_t* __restrict__ hdir,
                  ElastParam ep, double sigma, const BandSys* __restrict__ sys,
                  double* __restrict__ Lc, const double* __restrict__ sigma_per_sys) {
  const BandSys s = sys[blockIdx.x];
  if (sigma_per_sys) sigma = sigma_per_sys[blockIdx.x];
  const int S = s.bw + 1;
  const int64_t total = (int64_t)s.n * S;
  const int ex_lo = s.a0, ex_hi = s.a0 + s.w - 2, ey_lo = s.b0, ey_hi = s.b0 + s.hgt - 2;
  for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
    const int k = (int)(t / S), j = (int)(t % S);
    const int row = k + j;
    double v = 0.0;
    if (row < s.n) {
      int ak, bk, ar, br;
      band_node_of(s, k >> 1, ak, bk);
      band_node_of(s, row >> 1, ar, br);
      const int ck = k & 1, cr = row & 1;
      const int64_t nk = (int64_t)bk * g.nnx + ak, nr = (int64_t)br * g.nnx + ar;
      if (hdir[nk] || hdir[nr]) {
        v = (row == k) ? 1.0 : 0.0;
      } else if (abs(ar - ak) <= 1 && abs(br - bk) <= 1) {
        const int ilo = max(max(ak, ar) - 1, ex_lo), ihi = min(min(ak, ar), ex_hi);
        const int jlo = max(max(bk, br) - 1, ey_lo), jhi = min(min(bk, br), ey_hi);
        double kv = 0.0, mv = 0.0;
        for (int ej = jlo; ej <= jhi; ++ej)
          for (int ei = ilo; ei <= ihi; ++ei) {
            const int dk = ak - ei, ek = bk - ej, dr = ar - ei, er = br - ej;
            const int qk = dk + 3 * ek - 2 * dk * ek, qr = dr + 3 * er - 2 * dr * er;
            const double Ee = E[(int64_t)ej * g.nx + ei];
            kv += Ee * ep.ke[(cr * 4 + qr) * 8 + ck * 4 + qk];
            if (cr == ck) mv += Ee * ep.mel[qr * 4 + qk];
          }
        v = kv + sigma * mv;
      }
    }
    Lc[s.foff + t] = v;
  }
}

void launch_el_assemble(const Grid& g, const double* E, const uint8_t* hdir, const ElastParam& ep,
                        double sigma, const BandSys* sys, int nsys, double* Lc, cudaStream_t st,
                        const double* sigma_per_sys) {
  if (nsys == 0) return;
  { k_el_assemble<<<nsys, 256, 0, st>>>(g, E, hdir, ep, sigma, sys, Lc, sigma_per_sys); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// shared-memory carve-up common to the two elasticity kernels
struct ElSmem {
  double *sE, *win, *red, *dots, *Am, *Vm, *ritz, *ritz_old, *misc;
  int* order;
  uint8_t* dirn;
};
constexpr int kElNV = P + 3;  // reduction width: P block columns + 3 kernel modes

template <int B = P>
__device__ __forceinline__ ElSmem el_smem(double* sm, int nex, int ney, int S, int NL) {
  constexpr int NV = B + 3;
  ElSmem m;
  m.sE = sm;
  m.win = m.sE + nex * ney;
  m.red = m.win + S * B;
  m.dots = m.red + NV * 8;
  m.Am = m.dots + NV;
  m.Vm = m.Am + B * (B + 1);
  m.ritz = m.Vm + B * (B + 1);
  m.ritz_old = m.ritz + B;
  m.misc = m.ritz_old + B;
  m.order = reinterpret_cast<int*>(m.misc + 4);
  m.dirn = reinterpret_cast<uint8_t*>(m.order + B);
  (void)NL;
  return m;
}

template <int B = P>
static size_t el_smem_bytes(int mex, int mey, int max_bw) {
  constexpr int NV = B + 3;
  const int NL = (2 * mex + 1) * (2 * mey + 1);
  return sizeof(double) * ((size_t)(2 * mex) * (2 * mey) + (size_t)(max_bw + 1) * B + NV * 8 + NV +
                           2 * B * (B + 1) + 2 * B + 4) +
         sizeof(int) * B + (size_t)NL + 16;
}

// M-orthonormal rigid-body modes Zo (3 columns) and MZo = M Zo, CGS2 in the M
// inner product; translations and the rotation about the neighbourhood centre
__device__ void el_rigid_modes(const EigCtxE& c, double h, int mex, int mey, double* Zo, double* MZo,
                               double* red, double* dots) {
  const int n = c.n;
  double v[kElNV];
  for (int j = 0; j < 3; ++j) {
    double* w = Zo + (int64_t)j * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int ln = i >> 1, comp = i & 1;
      int a, b;
      band_node_of(c.s, ln, a, b);
      const double x = (double)(a - c.s.a0 - mex) * h, y = (double)(b - c.s.b0 - mey) * h;
      w[i] = (j == 0) ? (comp == 0 ? 1.0 : 0.0) : (j == 1) ? (comp == 1 ? 1.0 : 0.0) : (comp == 0 ? -y : x);
    }
    __syncthreads();
    for (int rep = 0; rep < 2; ++rep) {
#pragma unroll
      for (int l = 0; l < kElNV; ++l) v[l] = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        for (int l = 0; l < j; ++l) v[l] += MZo[(int64_t)l * n + i] * w[i];
      block_sum_nv(v, 3, red, dots);
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double x = w[i];
        for (int l = 0; l < j; ++l) x -= dots[l] * Zo[(int64_t)l * n + i];
        w[i] = x;
      }
      __syncthreads();
    }
    double nrm = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double mw = el_stencil(c, w, i, true);
      MZo[(int64_t)j * n + i] = mw;
      nrm += mw * w[i];
    }
#pragma unroll
    for (int l = 0; l < kElNV; ++l) v[l] = 0.0;
    v[0] = nrm;
    block_sum_nv(v, 1, red, dots);
    const double inv = 1.0 / sqrt(dots[0]);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      w[i] *= inv;
      MZo[(int64_t)j * n + i] *= inv;
    }
    __syncthreads();
  }
}

template <int KJ>
__global__ void __launch_bounds__(kEigThreads)
    k_subspace_el(Grid g, const double* __restrict__ E, const uint8_t* __restrict__ hdir,
                  ElastParam ep, EigBatch eb, int max_pass, double tol) {
  extern __shared__ double sm[];
  const int kb = blockIdx.x, k = eb.k0 + kb;
  const BandSys s = eb.sys[kb];
  const int n = s.n, S = s.bw + 1, NLn = n / 2;
  const int nex = 2 * eb.mex, ney = 2 * eb.mey;
  constexpr int LD = P + 1;
  const ElSmem m = el_smem(sm, nex, ney, S, NLn);
  __shared__ double ske[64], smel[16];
  if (threadIdx.x < 64) ske[threadIdx.x] = ep.ke[threadIdx.x];
  if (threadIdx.x < 16) smel[threadIdx.x] = ep.mel[threadIdx.x];
  for (int t = threadIdx.x; t < nex * ney; t += blockDim.x)
    m.sE[t] = E[(int64_t)(s.b0 + t / nex) * g.nx + s.a0 + t % nex];
  int ndir = 0;
  for (int ln = threadIdx.x; ln < NLn; ln += blockDim.x) {
    int a, b;
    band_node_of(s, ln, a, b);
    m.dirn[ln] = hdir[(int64_t)b * g.nnx + a];
    ndir += m.dirn[ln];
  }
  __syncthreads();
  const EigCtxE ctx{s, n, nex, ney, m.sE, m.dirn, ske, smel};
  double* X = eb.work + (int64_t)kb * (2 * P + 6) * n;
  double* W = X + (int64_t)P * n;
  double* Zo = W + (int64_t)P * n;
  double* MZo = Zo + 3 * (int64_t)n;
  double v[kElNV];
#pragma unroll
  for (int l = 0; l < kElNV; ++l) v[l] = 0.0;
  v[0] = (double)ndir;
  block_sum_nv(v, 1, m.red, m.dots);
  const bool neumann = m.dots[0] == 0.0;
  const int nz = neumann ? 3 : 0;
  if (neumann) el_rigid_modes(ctx, g.h, eb.mex, eb.mey, Zo, MZo, m.red, m.dots);
  for (int t = threadIdx.x; t < n * P; t += blockDim.x) {
    const int c = t / n, i = t % n;
    X[t] = m.dirn[i >> 1] ? 0.0 : hash_unif(((uint64_t)k << 32) ^ ((uint64_t)c << 24) ^ (uint64_t)i);
  }
  if (threadIdx.x < P) m.ritz_old[threadIdx.x] = 0.0;
  __syncthreads();
  const int need = kNeig - nz;
  int pass = 0;
  for (pass = 1; pass <= max_pass; ++pass) {
    // (1) W = M X (zero rows at Dirichlet nodes)
    for (int t = threadIdx.x; t < n * P; t += blockDim.x) {
      const int c = t / n, i = t % n;
      W[t] = m.dirn[i >> 1] ? 0.0 : el_stencil(ctx, X + (int64_t)c * n, i, true);
    }
    __syncthreads();
    // (2) W <- (K + sigma M)^{-1} W
    band_solve_cols<KJ>(s, eb.Lc, eb.Lr, W, P);
    // (3) M-orthonormalise W into X against the locked modes and earlier columns
    for (int c = 0; c < P; ++c) {
      double* w = W + (int64_t)c * n;
      for (int rep = 0; rep < 2; ++rep) {
#pragma unroll
        for (int l = 0; l < kElNV; ++l) v[l] = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          const double mw = el_stencil(ctx, w, i, true);
#pragma unroll
          for (int l = 0; l < P; ++l)
            if (l < c) v[l] += mw * X[(int64_t)l * n + i];
          for (int j = 0; j < nz; ++j) v[P + j] += MZo[(int64_t)j * n + i] * w[i];
        }
        block_sum_nv(v, kElNV, m.red, m.dots);
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          double x = w[i];
          for (int l = 0; l < c; ++l) x -= m.dots[l] * X[(int64_t)l * n + i];
          for (int j = 0; j < nz; ++j) x -= m.dots[P + j] * Zo[(int64_t)j * n + i];
          w[i] = m.dirn[i >> 1] ? 0.0 : x;
        }
        __syncthreads();
      }
      double nrm = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) nrm += w[i] * el_stencil(ctx, w, i, true);
#pragma unroll
      for (int l = 0; l < kElNV; ++l) v[l] = 0.0;
      v[0] = nrm;
      block_sum_nv(v, 1, m.red, m.dots);
      const double inv = m.dots[0] > 0.0 ? 1.0 / sqrt(m.dots[0]) : 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) X[(int64_t)c * n + i] = w[i] * inv;
      __syncthreads();
    }
    // (4) Kr = X^T K X
    for (int c = 0; c < P; ++c) {
#pragma unroll
      for (int l = 0; l < kElNV; ++l) v[l] = 0.0;
      const double* xc = X + (int64_t)c * n;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double kx = m.dirn[i >> 1] ? 0.0 : el_stencil(ctx, xc, i, false);
#pragma unroll
        for (int l = 0; l < P; ++l)
          if (l <= c) v[l] += kx * X[(int64_t)l * n + i];
      }
      block_sum_nv(v, c + 1, m.red, m.dots);
      if (threadIdx.x <= c) {
        m.Am[threadIdx.x * LD + c] = m.dots[threadIdx.x];
        m.Am[c * LD + threadIdx.x] = m.dots[threadIdx.x];
      }
      __syncthreads();
    }
    // (5) Jacobi, (6) X <- X V
    if (threadIdx.x < 32) jacobi_warp(m.Am, m.Vm, m.ritz, m.order);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double xr[P];
#pragma unroll
      for (int l = 0; l < P; ++l) xr[l] = X[(int64_t)l * n + i];
#pragma unroll
      for (int c = 0; c < P; ++c) {
        const int oc = m.order[c];
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) acc += xr[l] * m.Vm[l * LD + oc];
        W[(int64_t)c * n + i] = acc;
      }
    }
    __syncthreads();
    {
      double* t = X;
      X = W;
      W = t;
    }
    // (7) stopping rule ('fixed' selection: the first n_max pairs to tol, the rest to 1e-8)
    if (threadIdx.x == 0) {
      const double scale = fabs(m.ritz[P - 1]);
      const int sel = eb.n_max;
      bool conv = pass >= 3;
      for (int i = 0; i < need; ++i) {
        const double t = (i + nz < sel) ? tol : 1e-8;
        if (fabs(m.ritz[i] - m.ritz_old[i]) > t * fabs(m.ritz[i]) + fmax(1e-15 * scale, eb.lam_floor))
          conv = false;
      }
      for (int i = 0; i < P; ++i) m.ritz_old[i] = m.ritz[i];
      m.misc[2] = conv ? 1.0 : 0.0;
    }
    __syncthreads();
    if (m.misc[2] != 0.0) break;
  }
  // outputs: kNeig lowest pairs, ascending; locked modes first (lambda = z^T K z)
  double* ev = eb.evecs + (int64_t)kb * kNeig * n;
  for (int j = 0; j < nz; ++j) {
    const double* z = Zo + (int64_t)j * n;
    double kk = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      kk += z[i] * el_stencil(ctx, z, i, false);
      ev[(int64_t)j * n + i] = z[i];
    }
#pragma unroll
    for (int l = 0; l < kElNV; ++l) v[l] = 0.0;
    v[0] = kk;
    block_sum_nv(v, 1, m.red, m.dots);
    if (threadIdx.x == 0) eb.evals[(int64_t)k * kNeig + j] = m.dots[0];
  }
  for (int t = threadIdx.x; t < (kNeig - nz) * n; t += blockDim.x) {
    const int q = t / n, i = t % n;
    ev[(int64_t)(q + nz) * n + i] = X[(int64_t)q * n + i];
  }
  if (threadIdx.x < kNeig - nz) eb.evals[(int64_t)k * kNeig + nz + threadIdx.x] = m.ritz[threadIdx.x];
  if (threadIdx.x == 0) {
    eb.passes[k] = min(pass, max_pass);
    eb.neumann[k] = neumann ? 1 : 0;
  }
}

template <int KJ>
struct SubspaceElLaunch {
  static void run(const Grid& g, const double* E, const uint8_t* hdir, const ElastParam& ep, const EigBatch& b,
                  int max_pass, double tol, size_t smem, cudaStream_t st) {
    MS_CUDA(cudaFuncSetAttribute(k_subspace_el<KJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    { k_subspace_el<KJ><<<b.nk, kEigThreads, smem, st>>>(g, E, hdir, ep, b, max_pass, tol); ms_count_launch(); }
    MS_CUDA(cudaGetLastError());
  }
};

void launch_subspace_el(const Grid& g, const double* E, const uint8_t* hdir, const ElastParam& ep,
                        const EigBatch& b, int max_bw, int max_pass, double tol, cudaStream_t st) {
  if (b.nk == 0) return;
  const size_t smem = el_smem_bytes(b.mex, b.mey, max_bw);
  if (smem > 220 * 1024) throw Error(-1, "neighbourhood too large for the elasticity eigensolver tile");
  band_dispatch<SubspaceElLaunch>(max_bw, g, E, hdir, ep, b, max_pass, tol, smem, st);
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    k_compact_psi_el(EigBatch eb, int NLx, const int* __restrict__ nsel, const int64_t* __restrict__ psioff,
                     double* __restrict__ psi) {
  __shared__ double sval[8];
  __shared__ int sidx[8];
  const int kb = blockIdx.x, k = eb.k0 + kb;
  const BandSys s = eb.sys[kb];
  const int n = s.n, NL = n / 2;
  const double* ev = eb.evecs + (int64_t)kb * kNeig * n;
  for (int mo = 0; mo < nsel[k]; ++mo) {
    const double* vm = ev + (int64_t)mo * n;
    // argmax |v| over (component, lexicographic node) order, ties: smallest index
    double best = -1.0;
    int bidx = 0x7fffffff;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const int c = t / NL, ln = t % NL;
      const double x = fabs(vm[2 * band_local_node(s, s.a0 + ln % NLx, s.b0 + ln / NLx) + c]);
      if (x > best || (x == best && t < bidx)) {
        best = x;
        bidx = t;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ob > best || (ob == best && oi < bidx)) {
        best = ob;
        bidx = oi;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      sval[threadIdx.x >> 5] = best;
      sidx[threadIdx.x >> 5] = bidx;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 1; w < 8; ++w)
        if (sval[w] > sval[0] || (sval[w] == sval[0] && sidx[w] < sidx[0])) {
          sval[0] = sval[w];
          sidx[0] = sidx[w];
        }
    __syncthreads();
    const int ib = sidx[0], cb = ib / NL, lb = ib % NL;
    const double sign = vm[2 * band_local_node(s, s.a0 + lb % NLx, s.b0 + lb / NLx) + cb] < 0.0 ? -1.0 : 1.0;
    double* out = psi + psioff[k] + (int64_t)mo * n;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const int c = t / NL, ln = t % NL;
      out[t] = sign * vm[2 * band_local_node(s, s.a0 + ln % NLx, s.b0 + ln / NLx) + c];
    }
    __syncthreads();
  }
}

void launch_compact_psi_el(const EigBatch& b, int NLx, const int* nsel, const int64_t* psioff,
                           double* psi, cudaStream_t st) {
  if (b.nk == 0) return;
  { k_compact_psi_el<<<b.nk, 256, 0, st>>>(b, NLx, nsel, psioff, psi); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// EE;Rand: the randomized snapshot solver (spectral.py:103-158) on the
// elasticity pencil, kernel candidates Z = the three rigid-body modes on the
// free dofs (kernel_basis, spectral.py:37-44): G = Z^T M Z,
// F -= MZ G^-1 Z^T F, deflate(X) = X - Z G^-1 MZ^T X, 4 shift-invert passes,
// orthonormal basis of [U, Z] (CGS2, rank cut), Rayleigh-Ritz.

__global__ void k_rand_sigma_el(Grid g, const double* __restrict__ E, const uint8_t* __restrict__ hdir,
                                ElastParam ep, const BandSys* __restrict__ sys, double* __restrict__ sigma) {
  __shared__ double sred[8];
  const BandSys s = sys[blockIdx.x];
  const int NLn = s.n / 2;
  double tr = 0.0, nf = 0.0;
  for (int ln = threadIdx.x; ln < NLn; ln += blockDim.x) {
    int a, b;
    band_node_of(s, ln, a, b);
    if (hdir[(int64_t)b * g.nnx + a]) continue;
    nf += 2.0;
    for (int e = 0; e < 4; ++e) {
      const int ei = a - 1 + (e == 1 || e == 2), ej = b - 1 + (e >= 2);
      if (ei < s.a0 || ej < s.b0 || ei > s.a0 + s.w - 2 || ej > s.b0 + s.hgt - 2) continue;
      const int cn = (e == 0) ? 2 : (e == 1) ? 3 : (e == 2) ? 0 : 1;
      const double Ee = E[(int64_t)ej * g.nx + ei];
      tr += Ee * ep.ke[cn * 8 + cn] + Ee * ep.ke[(4 + cn) * 8 + 4 + cn];
    }
  }
  const double t = block_sum(tr, sred), m = block_sum(nf, sred);
  if (threadIdx.x == 0) sigma[blockIdx.x] = 1e-8 * (t / m);
}

void launch_rand_sigma_el(const Grid& g, const double* E, const uint8_t* hdir, const ElastParam& ep,
                          const BandSys* sys, int nsys, double* sigma, cudaStream_t st) {
  if (nsys == 0) return;
  { k_rand_sigma_el<<<nsys, 256, 0, st>>>(g, E, hdir, ep, sys, sigma); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

template <int KJ, int B>
__global__ void __launch_bounds__(kEigThreads)
    k_randomized_el(Grid g, const double* __restrict__ E, const uint8_t* __restrict__ hdir, ElastParam ep,
                    EigBatch eb, const double* __restrict__ F, int ns, int nlx) {
  extern __shared__ double sm[];
  const int kb = blockIdx.x, k = eb.k0 + kb;
  const BandSys s = eb.sys[kb];
  const int n = s.n, S = s.bw + 1, NLn = n / 2;
  const int nex = 2 * eb.mex, ney = 2 * eb.mey;
  constexpr int LD = B + 1;
  const ElSmem m = el_smem<B>(sm, nex, ney, S, NLn);
  __shared__ double ske[64], smel[16], Gi[9], keep[B];
  __shared__ double Lm[B][B + 1], Cm[B][B + 1];
  if (threadIdx.x < 64) ske[threadIdx.x] = ep.ke[threadIdx.x];
  if (threadIdx.x < 16) smel[threadIdx.x] = ep.mel[threadIdx.x];
  for (int t = threadIdx.x; t < nex * ney; t += blockDim.x)
    m.sE[t] = E[(int64_t)(s.b0 + t / nex) * g.nx + s.a0 + t % nex];
  for (int ln = threadIdx.x; ln < NLn; ln += blockDim.x) {
    int a, b;
    band_node_of(s, ln, a, b);
    m.dirn[ln] = hdir[(int64_t)b * g.nnx + a];
  }
  __syncthreads();
  const EigCtxE ctx{s, n, nex, ney, m.sE, m.dirn, ske, smel};
  double* X = eb.work + (int64_t)kb * (2 * B + 6) * n;
  double* W = X + (int64_t)B * n;
  double* Z = W + (int64_t)B * n;
  double* MZ = Z + 3 * (int64_t)n;
  double v[(B + 3)];
  auto zero_v = [&]() {
#pragma unroll
    for (int l = 0; l < (B + 3); ++l) v[l] = 0.0;
  };
  // Z on the free dofs (rotation about the neighbourhood centre), MZ, G^-1
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int ln = i >> 1, comp = i & 1;
    int a, b;
    band_node_of(s, ln, a, b);
    const bool d = m.dirn[ln];
    const double x = (double)(a - s.a0 - eb.mex) * g.h, y = (double)(b - s.b0 - eb.mey) * g.h;
    Z[i] = d ? 0.0 : (comp == 0 ? 1.0 : 0.0);
    Z[n + i] = d ? 0.0 : (comp == 1 ? 1.0 : 0.0);
    Z[2 * n + i] = d ? 0.0 : (comp == 0 ? -y : x);
  }
  __syncthreads();
  zero_v();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const bool d = m.dirn[i >> 1];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double mz = d ? 0.0 : el_stencil(ctx, Z + (int64_t)j * n, i, true);
      MZ[(int64_t)j * n + i] = mz;
#pragma unroll
      for (int l = 0; l <= j; ++l) v[j * 3 + l] += Z[(int64_t)l * n + i] * mz;
    }
  }
  block_sum_nv(v, 9, m.red, m.dots);
  if (threadIdx.x == 0) {
    double G[3][3];
    for (int j = 0; j < 3; ++j)
      for (int l = 0; l <= j; ++l) G[j][l] = G[l][j] = m.dots[j * 3 + l];
    const double det = G[0][0] * (G[1][1] * G[2][2] - G[1][2] * G[2][1]) -
                       G[0][1] * (G[1][0] * G[2][2] - G[1][2] * G[2][0]) +
                       G[0][2] * (G[1][0] * G[2][1] - G[1][1] * G[2][0]);
    const double id = 1.0 / det;
    Gi[0] = (G[1][1] * G[2][2] - G[1][2] * G[2][1]) * id;
    Gi[1] = (G[0][2] * G[2][1] - G[0][1] * G[2][2]) * id;
    Gi[2] = (G[0][1] * G[1][2] - G[0][2] * G[1][1]) * id;
    Gi[3] = (G[1][2] * G[2][0] - G[1][0] * G[2][2]) * id;
    Gi[4] = (G[0][0] * G[2][2] - G[0][2] * G[2][0]) * id;
    Gi[5] = (G[0][2] * G[1][0] - G[0][0] * G[1][2]) * id;
    Gi[6] = (G[1][0] * G[2][1] - G[1][1] * G[2][0]) * id;
    Gi[7] = (G[0][1] * G[2][0] - G[0][0] * G[2][1]) * id;
    Gi[8] = (G[0][0] * G[1][1] - G[0][1] * G[1][0]) * id;
  }
  __syncthreads();
  // X - A G^-1 (B^T X) for the first ns columns of W (A, B in {Z, MZ})
  auto project = [&](const double* A, const double* B) {
    for (int c = 0; c < ns; ++c) {
      double* w = W + (int64_t)c * n;
      zero_v();
      for (int i = threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
        for (int j = 0; j < 3; ++j) v[j] += B[(int64_t)j * n + i] * w[i];
      block_sum_nv(v, 3, m.red, m.dots);
      double u[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) u[j] = Gi[j * 3] * m.dots[0] + Gi[j * 3 + 1] * m.dots[1] + Gi[j * 3 + 2] * m.dots[2];
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        w[i] -= A[i] * u[0] + A[n + i] * u[1] + A[2 * (int64_t)n + i] * u[2];
      __syncthreads();
    }
  };
  // forcings: [ns][2 NL] x-plane then y-plane (lexicographic) -> band order
  const int NLd = 2 * NLn;
  const double* Fk = F + (int64_t)kb * ns * NLd;
  for (int t = threadIdx.x; t < n * B; t += blockDim.x) {
    const int c = t / n, i = t % n;
    double val = 0.0;
    if (c < ns && !m.dirn[i >> 1]) {
      int a, b;
      band_node_of(s, i >> 1, a, b);
      val = Fk[(int64_t)c * NLd + (int64_t)(i & 1) * NLn + (a - s.a0) + (int64_t)(b - s.b0) * nlx];
    }
    W[t] = val;
  }
  __syncthreads();
  project(MZ, Z);  // F -= MZ G^-1 Z^T F
  band_solve_cols<KJ>(s, eb.Lc, eb.Lr, W, ns);
  project(Z, MZ);  // deflate
  for (int pass = 1; pass < 4; ++pass) {
    cgs2_euclid<B>(W, ns, n, m.red, m.dots, nullptr);
    for (int t = threadIdx.x; t < n * ns; t += blockDim.x) {
      const int c = t / n, i = t % n;
      X[t] = m.dirn[i >> 1] ? 0.0 : el_stencil(ctx, W + (int64_t)c * n, i, true);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n * ns; t += blockDim.x) W[t] = X[t];
    __syncthreads();
    band_solve_cols<KJ>(s, eb.Lc, eb.Lr, W, ns);
    project(Z, MZ);
  }
  // Q = orthonormal basis of [U, Z]
  const int m0 = ns + 3;
  for (int t = threadIdx.x; t < n * m0; t += blockDim.x) {
    const int c = t / n, i = t % n;
    X[t] = (c < ns) ? W[t] : Z[(int64_t)(c - ns) * n + i];
  }
  __syncthreads();
  cgs2_euclid<B>(X, m0, n, m.red, m.dots, keep);
  if (threadIdx.x == 0) {
    int q = 0;
    for (int c = 0; c < m0; ++c)
      if (keep[c] != 0.0) m.order[q++] = c;
    m.misc[0] = (double)q;
  }
  __syncthreads();
  const int mq = (int)m.misc[0];
  for (int q = 0; q < mq; ++q) {
    const int c = m.order[q];
    if (c != q)
      for (int i = threadIdx.x; i < n; i += blockDim.x) X[(int64_t)q * n + i] = X[(int64_t)c * n + i];
    __syncthreads();
  }
  // Kr (-> Am) and Mr (-> Cm)
  for (int ps = 0; ps < 2; ++ps) {
    for (int c = 0; c < mq; ++c) {
      zero_v();
      const double* xc = X + (int64_t)c * n;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double ax = m.dirn[i >> 1] ? 0.0 : el_stencil(ctx, xc, i, ps == 1);
#pragma unroll
        for (int l = 0; l < B; ++l)
          if (l <= c) v[l] += ax * X[(int64_t)l * n + i];
      }
      block_sum_nv(v, c + 1, m.red, m.dots);
      if (threadIdx.x <= c) {
        if (ps == 0)
          m.Am[threadIdx.x * LD + c] = m.Am[c * LD + threadIdx.x] = m.dots[threadIdx.x];
        else
          Cm[threadIdx.x][c] = Cm[c][threadIdx.x] = m.dots[threadIdx.x];
      }
      __syncthreads();
    }
  }
  // generalized mq x mq problem: Mr = L L^T, C = L^-1 Kr L^-T, Jacobi
  if (threadIdx.x == 0) {
    for (int i = 0; i < mq; ++i)
      for (int j = 0; j <= i; ++j) {
        double a = Cm[i][j];
        for (int q = 0; q < j; ++q) a -= Lm[i][q] * Lm[j][q];
        Lm[i][j] = (i == j) ? sqrt(fmax(a, 1e-300)) : a / Lm[j][j];
      }
    for (int c = 0; c < mq; ++c)
      for (int i = 0; i < mq; ++i) {
        double a = m.Am[i * LD + c];
        for (int q = 0; q < i; ++q) a -= Lm[i][q] * Cm[q][c];
        Cm[i][c] = a / Lm[i][i];
      }
    for (int i = 0; i < mq; ++i)
      for (int j = 0; j < mq; ++j) {
        double a = Cm[i][j];
        for (int q = 0; q < j; ++q) a -= m.Am[i * LD + q] * Lm[j][q];
        m.Am[i * LD + j] = a / Lm[j][j];
      }
    for (int i = 0; i < B; ++i)
      for (int j = 0; j < B; ++j)
        if (i >= mq || j >= mq) m.Am[i * LD + j] = (i == j) ? 1e300 : 0.0;
    for (int i = 0; i < mq; ++i)
      for (int j = 0; j < i; ++j)
        m.Am[i * LD + j] = m.Am[j * LD + i] = 0.5 * (m.Am[i * LD + j] + m.Am[j * LD + i]);
  }
  __syncthreads();
  if (threadIdx.x < 32) jacobi_warp<B>(m.Am, m.Vm, m.ritz, m.order);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int c = 0; c < kNeig && c < mq; ++c) {
      const int oc = m.order[c];
      for (int i = mq - 1; i >= 0; --i) {
        double a = m.Vm[i * LD + oc];
        for (int q = i + 1; q < mq; ++q) a -= Lm[q][i] * Cm[q][c];
        Cm[i][c] = a / Lm[i][i];
      }
    }
  }
  __syncthreads();
  double* ev = eb.evecs + (int64_t)kb * kNeig * n;
  const int kk = min(kNeig, mq);
  for (int t = threadIdx.x; t < kNeig * n; t += blockDim.x) {
    const int c = t / n, i = t % n;
    double a = 0.0;
    if (c < kk)
      for (int q = 0; q < mq; ++q) a += X[(int64_t)q * n + i] * Cm[q][c];
    ev[t] = a;
  }
  if (threadIdx.x < kNeig)
    eb.evals[(int64_t)k * kNeig + threadIdx.x] = threadIdx.x < kk ? m.ritz[threadIdx.x] : CUDART_NAN;
  if (threadIdx.x == 0) {
    eb.passes[k] = 4;
    eb.neumann[k] = 0;
  }
}

template <int KJ>
struct RandElLaunch {
  template <int B>
  static void go(const Grid& g, const double* E, const uint8_t* hdir, const ElastParam& ep, const EigBatch& b,
                 const double* F, int ns, int nlx, int max_bw, cudaStream_t st) {
    const size_t smem = el_smem_bytes<B>(b.mex, b.mey, max_bw);
    if (smem > 200 * 1024) throw Error(-1, "neighbourhood too large for the elasticity eigensolver tile");
    MS_CUDA(cudaFuncSetAttribute(k_randomized_el<KJ, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    { k_randomized_el<KJ, B><<<b.nk, kEigThreads, smem, st>>>(g, E, hdir, ep, b, F, ns, nlx); ms_count_launch(); }
    MS_CUDA(cudaGetLastError());
  }
  static void run(const Grid& g, const double* E, const uint8_t* hdir, const ElastParam& ep, const EigBatch& b,
                  const double* F, int ns, int nlx, int max_bw, cudaStream_t st) {
    if (randomized_block(ns) == kEigBlock)
      go<kEigBlock>(g, E, hdir, ep, b, F, ns, nlx, max_bw, st);
    else
      go<32>(g, E, hdir, ep, b, F, ns, nlx, max_bw, st);
  }
};

void launch_randomized_el(const Grid& g, const double* E, const uint8_t* hdir, const ElastParam& ep,
                          const EigBatch& b, int max_bw, const double* F, int ns, cudaStream_t st) {
  if (b.nk == 0) return;
  if (ns + 3 > 32) throw Error(-1, "too many snapshots for the randomized elasticity eigensolver (<= 29)");
  band_dispatch<RandElLaunch>(max_bw, g, E, hdir, ep, b, F, ns, 2 * b.mex + 1, max_bw, st);
}

}  // namespace msgpu
