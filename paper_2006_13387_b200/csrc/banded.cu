// Batched banded SPD kernels: level-1 band assembly, Cholesky, sweeps.
//
// Replaces the per-subdomain SuperLU factor/solve of the reference
// (`spla.splu(K_i).solve`, schwarz.py:97-109 build, :80-81 apply).  Each
// subdomain's unknowns are numbered node-interleaved along its short axis,
// which makes K_i a band of width 2*(short side)+3 (73 for the configs'
// 35x35-node subdomains); its Cholesky factor is 1.4 MB instead of the 24 MB
// of a packed dense inverse, so one apply streams ~8x fewer bytes.
#include <algorithm>

#include "banded.cuh"

namespace msgpu {

void band_setup(BandSys& s, int a0, int a1, int b0, int b1, int ncomp) {
  s.a0 = a0;
  s.b0 = b0;
  s.w = a1 - a0 + 1;
  s.hgt = b1 - b0 + 1;
  s.fastx = s.w <= s.hgt ? 1 : 0;
  s.ncomp = ncomp;
  s.n = ncomp * s.w * s.hgt;
  const int fast = s.fastx ? s.w : s.hgt;
  int bw = ncomp == 2 ? 2 * fast + 3 : fast + 1;
  s.bw = std::max(0, std::min(bw, s.n - 1));
  s.foff = 0;
  s.yoff = 0;
}

// ---------------------------------------------------------------------------
// Level-1 band assembly: entry (row = k + j, col = k) of A[idx][:, idx].
// Element contributions are summed in ascending element order, the order in
// which the reference's COO->CSR conversion sums duplicates (assembly.py:185-196),
// so the band holds the same bits as the reference's restricted CSR.
__global__ void __launch_bounds__(256)
    k_l1_assemble(Grid g, KeParam ke, const double* __restrict__ E,
                  const uint8_t* __restrict__ mask, const BandSys* __restrict__ sys,
                  double* __restrict__ Lc) {
  const BandSys s = sys[blockIdx.x];
  const int S = s.bw + 1;
  const int64_t total = (int64_t)s.n * S;
  for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
    const int k = (int)(t / S), j = (int)(t % S);
    const int row = k + j;
    double v = 0.0;
    if (row < s.n) {
      int ak, bk, ar, br;
      band_node_of(s, k >> 1, ak, bk);
      band_node_of(s, row >> 1, ar, br);
      const int ck = k & 1, cr = row & 1;
      const int64_t gk = ck * g.n_nodes + (int64_t)bk * g.nnx + ak;
      const int64_t gr = cr * g.n_nodes + (int64_t)br * g.nnx + ar;
      if (!mask[gk] || !mask[gr]) {
        v = (row == k) ? 1.0 : 0.0;
      } else if (abs(ar - ak) <= 1 && abs(br - bk) <= 1) {
        const int ilo = max(max(ak, ar) - 1, 0), ihi = min(min(ak, ar), g.nx - 1);
        const int jlo = max(max(bk, br) - 1, 0), jhi = min(min(bk, br), g.ny - 1);
        for (int ej = jlo; ej <= jhi; ++ej)
          for (int ei = ilo; ei <= ihi; ++ei) {
            const int crn_k = (ak - ei) + (bk - ej) * 3 - 2 * (bk - ej) * (ak - ei);
            const int crn_r = (ar - ei) + (br - ej) * 3 - 2 * (br - ej) * (ar - ei);
            // corner numbering (0,0)->0 (1,0)->1 (1,1)->2 (0,1)->3
            v += E[(int64_t)ej * g.nx + ei] * ke.k[(cr * 4 + crn_r) * 8 + ck * 4 + crn_k];
          }
      }
    }
    Lc[s.foff + t] = v;
  }
}

void launch_l1_assemble(const Grid& g, const KeParam& ke, const double* E, const uint8_t* mask,
                        const BandSys* sys, int nsys, double* Lc, cudaStream_t st) {
  if (nsys == 0) return;
  k_l1_assemble<<<nsys, 256, 0, st>>>(g, ke, E, mask, sys, Lc);
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Banded Cholesky, one CTA per system.  A sliding window of the next bw+1
// columns lives in shared memory (column c in slot c % S); each step k folds
// column k into the window with a rank-1 update a_j1 a_j2 / d and retires it.
__global__ void __launch_bounds__(256)
    k_band_potrf(const BandSys* __restrict__ sys, double* __restrict__ Lc,
                 double* __restrict__ Lr, int* fail) {
  extern __shared__ double smem[];
  const BandSys s = sys[blockIdx.x];
  const int bw = s.bw, S = bw + 1, n = s.n;
  double* W = smem;                                           // S*S
  short2* pairs = reinterpret_cast<short2*>(smem + S * S);    // bw(bw+1)/2
  const int npairs = bw * (bw + 1) / 2;
  if (threadIdx.x == 0) {
    int p = 0;
    for (int j2 = 1; j2 <= bw; ++j2)
      for (int j1 = j2; j1 <= bw; ++j1) pairs[p++] = make_short2((short)j1, (short)j2);
  }
  double* colc = Lc + s.foff;
  double* colr = Lr + s.foff;
  for (int t = threadIdx.x; t < S * S; t += blockDim.x) {
    const int c = t / S, j = t % S;
    W[t] = (c < n) ? colc[(int64_t)c * S + j] : 0.0;
  }
  __syncthreads();
  bool bad = false;
  for (int k = 0; k < n; ++k) {
    const int sk = k % S;
    double d = W[sk * S];
    if (!(d > 0.0)) {
      bad = true;
      d = 1.0;
    }
    const double invd = 1.0 / d;
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
      const short2 jj = pairs[p];
      const int j1 = jj.x, j2 = jj.y;
      W[((k + j2) % S) * S + (j1 - j2)] -= W[sk * S + j1] * W[sk * S + j2] * invd;
    }
    __syncthreads();
    const double lkk = sqrt(d), inv = 1.0 / lkk;
    for (int j = threadIdx.x; j < S; j += blockDim.x) {
      const double v = (j == 0) ? inv : W[sk * S + j] * inv;
      colc[(int64_t)k * S + j] = v;
      if (k + j < n) colr[(int64_t)(k + j) * S + j] = v;
      const int cn = k + S;  // next column into the freed slot
      W[sk * S + j] = (cn < n) ? colc[(int64_t)cn * S + j] : 0.0;
    }
    __syncthreads();
  }
  if (bad && threadIdx.x == 0) atomicCAS(fail, 0, (int)blockIdx.x + 1);
}

void launch_band_potrf(const BandSys* sys, int nsys, int max_bw, double* Lc, double* Lr, int* fail,
                       cudaStream_t st) {
  if (nsys == 0) return;
  const int S = max_bw + 1;
  const size_t smem = (size_t)S * S * sizeof(double) + (size_t)(max_bw * (max_bw + 1) / 2 + 1) * 4;
  if (smem > 220 * 1024) throw Error(-1, "band too wide for the shared-memory Cholesky window");
  MS_CUDA(cudaFuncSetAttribute(k_band_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_band_potrf<<<nsys, 256, smem, st>>>(sys, Lc, Lr, fail);
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Level-1 sweeps, one warp per subdomain.  Column-oriented (axpy) forward
// sweep over Lc, and the same over Lr for the backward sweep, so neither
// needs a reduction: the only loop-carried chain is the window slot of the
// next row.  Band columns are software-pipelined PD steps ahead in
// registers; lane l owns band offsets j = l+1+32t.
constexpr int kSolveWarps = 4;
constexpr int kPD = 8;

template <int JPL>
__global__ void __launch_bounds__(kSolveWarps * 32)
    k_l1_solve(Grid g, const BandSys* __restrict__ sys, int nsys, const double* __restrict__ Lc,
               const double* __restrict__ Lr, const double* __restrict__ r,
               double* __restrict__ ybuf, const int* done) {
  if (done && *(volatile const int*)done) return;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sid = blockIdx.x * kSolveWarps + warp;
  if (sid >= nsys) return;
  const BandSys s = sys[sid];
  const int S = s.bw + 1, n = s.n, bw = s.bw;
  double* acc = smem + warp * (JPL * 32 + 1);
  double* y = ybuf + s.yoff;

  // gather R_s r (node-interleaved local order)
  for (int i = lane; i < n; i += 32) {
    const int ln = s.ncomp == 2 ? (i >> 1) : i, c = s.ncomp == 2 ? (i & 1) : 0;
    int a, b;
    band_node_of(s, ln, a, b);
    y[i] = r[c * g.n_nodes + (int64_t)b * g.nnx + a];
  }
  __syncwarp();

  double lv[kPD][JPL], dv[kPD], rv[kPD];
  // ---- forward: L w = rhs ----
  {
    const double* L = Lc + s.foff;
    for (int i = lane; i < S && i < n; i += 32) acc[i] = y[i];
    __syncwarp();
    auto load = [&](int k, double(&l)[JPL], double& d, double& rr) {
#pragma unroll
      for (int t = 0; t < JPL; ++t) {
        const int j = lane + 1 + 32 * t;
        l[t] = (k < n && j <= bw) ? __ldg(L + (int64_t)k * S + j) : 0.0;
      }
      d = (k < n) ? __ldg(L + (int64_t)k * S) : 0.0;
      rr = (k + S < n) ? y[k + S] : 0.0;
    };
#pragma unroll
    for (int u = 0; u < kPD; ++u) load(u, lv[u], dv[u], rv[u]);
    for (int k0 = 0; k0 < n; k0 += kPD) {
#pragma unroll
      for (int u = 0; u < kPD; ++u) {
        const int k = k0 + u;
        if (k < n) {
          const int sk = k % S;
          const double wk = acc[sk] * dv[u];
#pragma unroll
          for (int t = 0; t < JPL; ++t) {
            const int j = lane + 1 + 32 * t;
            if (j <= bw) {
              const int sl = (sk + j) >= S ? sk + j - S : sk + j;
              acc[sl] -= lv[u][t] * wk;
            }
          }
          if (lane == 0) {
            y[k] = wk;
            if (k + S < n) acc[sk] = rv[u];
          }
          __syncwarp();
          load(k + kPD, lv[u], dv[u], rv[u]);
        }
      }
    }
  }
  __syncwarp();
  // ---- backward: L^T y = w ----
  {
    const double* L = Lr + s.foff;
    for (int i = lane; i < S && i < n; i += 32) {
      const int row = n - 1 - i;
      acc[row % S] = y[row];
    }
    __syncwarp();
    auto load = [&](int k, double(&l)[JPL], double& d, double& rr) {
#pragma unroll
      for (int t = 0; t < JPL; ++t) {
        const int j = lane + 1 + 32 * t;
        l[t] = (k >= 0 && j <= bw) ? __ldg(L + (int64_t)k * S + j) : 0.0;
      }
      d = (k >= 0) ? __ldg(L + (int64_t)k * S) : 0.0;
      rr = (k - S >= 0) ? y[k - S] : 0.0;
    };
#pragma unroll
    for (int u = 0; u < kPD; ++u) load(n - 1 - u, lv[u], dv[u], rv[u]);
    for (int k0 = 0; k0 < n; k0 += kPD) {
#pragma unroll
      for (int u = 0; u < kPD; ++u) {
        const int k = n - 1 - (k0 + u);
        if (k >= 0) {
          const int sk = k % S;
          const double yk = acc[sk] * dv[u];
#pragma unroll
          for (int t = 0; t < JPL; ++t) {
            const int j = lane + 1 + 32 * t;
            if (j <= bw && k - j >= 0) {
              const int sl = (sk - j) < 0 ? sk - j + S : sk - j;
              acc[sl] -= lv[u][t] * yk;
            }
          }
          if (lane == 0) {
            y[k] = yk;
            if (k - S >= 0) acc[sk] = rv[u];
          }
          __syncwarp();
          load(k - kPD, lv[u], dv[u], rv[u]);
        }
      }
    }
  }
}

template <int JPL>
static void solve_jpl(const Grid& g, const BandSys* sys, int nsys, const double* Lc,
                      const double* Lr, const double* r, double* ybuf, const int* done,
                      cudaStream_t st) {
  const size_t smem = (size_t)kSolveWarps * (JPL * 32 + 1) * sizeof(double);
  k_l1_solve<JPL><<<div_up(nsys, kSolveWarps), kSolveWarps * 32, smem, st>>>(g, sys, nsys, Lc, Lr,
                                                                             r, ybuf, done);
}

void launch_l1_solve(const Grid& g, const BandSys* sys, int nsys, int max_bw, const double* Lc,
                     const double* Lr, const double* r, double* ybuf, const int* done,
                     cudaStream_t st) {
  if (nsys == 0) return;
  const int jpl = std::max(1, div_up(max_bw, 32));
  switch (jpl) {
    case 1: solve_jpl<1>(g, sys, nsys, Lc, Lr, r, ybuf, done, st); break;
    case 2: solve_jpl<2>(g, sys, nsys, Lc, Lr, r, ybuf, done, st); break;
    case 3: solve_jpl<3>(g, sys, nsys, Lc, Lr, r, ybuf, done, st); break;
    case 4: solve_jpl<4>(g, sys, nsys, Lc, Lr, r, ybuf, done, st); break;
    case 5: solve_jpl<5>(g, sys, nsys, Lc, Lr, r, ybuf, done, st); break;
    case 6: solve_jpl<6>(g, sys, nsys, Lc, Lr, r, ybuf, done, st); break;
    case 7: solve_jpl<7>(g, sys, nsys, Lc, Lr, r, ybuf, done, st); break;
    case 8: solve_jpl<8>(g, sys, nsys, Lc, Lr, r, ybuf, done, st); break;
    default: throw Error(-1, "level-1 band wider than 256 unsupported");
  }
  MS_CUDA(cudaGetLastError());
}

}  // namespace msgpu
