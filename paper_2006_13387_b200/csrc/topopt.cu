// Topology-optimisation caller: the per-design-step
// coefficient pipeline of the reference's SIMP loop (topopt.py:123-216) kept
// on the device: density filter and its adjoint (DensityFilter,
// assembly.py:290-336), SIMP modulus (assembly.py:280-287) written straight
// into the operator, compliance sensitivity (topopt.py:59-70) and the
// optimality-criteria multiplier bisection (topopt.py:73-107).  All of them
// are single streaming passes over per-element arrays (HBM-bound); the OC
// bisection runs as a device state machine, one launch per volume evaluation.
#include <algorithm>

#include "topopt.cuh"

namespace msgpu {

constexpr int kFiltThreads = 256;
constexpr int kMaxSmemOff = 1024;

// ---------------------------------------------------------------------------
// filter: y_e = sum_k W_ek x_k in the reference's stored order (descending k),
// W_ek = inv_rowsum[e] * w[o]; explicit _rn intrinsics keep the products and
// sums uncontracted, as in scipy's csr_matvec.
__global__ void __launch_bounds__(kFiltThreads)
    k_filter_apply(FilterDev f, const double* __restrict__ x, double* __restrict__ y) {
  __shared__ int2 so[kMaxSmemOff];
  __shared__ double sw[kMaxSmemOff];
  const bool staged = f.noff <= kMaxSmemOff;
  if (staged)
    for (int o = threadIdx.x; o < f.noff; o += blockDim.x) {
      so[o] = f.off[o];
      sw[o] = f.w[o];
    }
  __syncthreads();
  const int64_t n = (int64_t)f.nx * f.ny;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % f.nx), j = (int)(e / f.nx);
    const double inv = f.inv_rowsum[e];
    double s = 0.0;
    for (int o = 0; o < f.noff; ++o) {
      const int2 d = staged ? so[o] : f.off[o];
      const int ik = i + d.x, jk = j + d.y;
      if (ik < 0 || ik >= f.nx || jk < 0 || jk >= f.ny) continue;
      const double wek = __dmul_rn(inv, staged ? sw[o] : f.w[o]);
      s = __dadd_rn(s, __dmul_rn(wek, __ldg(x + (int64_t)jk * f.nx + ik)));
    }
    y[e] = s;
  }
}

// adjoint: y_k = sum_e W_ek v_e, rows e ascending (= offsets descending, e = k - d)
__global__ void __launch_bounds__(kFiltThreads)
    k_filter_adjoint(FilterDev f, const double* __restrict__ v, double* __restrict__ y) {
  __shared__ int2 so[kMaxSmemOff];
  __shared__ double sw[kMaxSmemOff];
  const bool staged = f.noff <= kMaxSmemOff;
  if (staged)
    for (int o = threadIdx.x; o < f.noff; o += blockDim.x) {
      so[o] = f.off[o];
      sw[o] = f.w[o];
    }
  __syncthreads();
  const int64_t n = (int64_t)f.nx * f.ny;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(k % f.nx), j = (int)(k / f.nx);
    double s = 0.0;
    for (int o = 0; o < f.noff; ++o) {
      const int2 d = staged ? so[o] : f.off[o];
      const int ie = i - d.x, je = j - d.y;
      if (ie < 0 || ie >= f.nx || je < 0 || je >= f.ny) continue;
      const int64_t e = (int64_t)je * f.nx + ie;
      const double wek = __dmul_rn(__ldg(f.inv_rowsum + e), staged ? sw[o] : f.w[o]);
      s = __dadd_rn(s, __dmul_rn(wek, __ldg(v + e)));
    }
    y[k] = s;
  }
}

static int stream_blocks(int64_t n) { return (int)std::min<int64_t>(div_up(n, kFiltThreads), 16 * 148); }

void launch_filter_apply(const FilterDev& f, const double* x, double* y, cudaStream_t st) {
  const int64_t n = (int64_t)f.nx * f.ny;
  { k_filter_apply<<<stream_blocks(n), kFiltThreads, 0, st>>>(f, x, y); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

void launch_filter_adjoint(const FilterDev& f, const double* v, double* y, cudaStream_t st) {
  const int64_t n = (int64_t)f.nx * f.ny;
  { k_filter_adjoint<<<stream_blocks(n), kFiltThreads, 0, st>>>(f, v, y); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// numpy's float power fast paths (exponent 1, 2, 0.5) then the general pow
__device__ __forceinline__ double np_pow(double x, double p) {
  if (p == 2.0) return __dmul_rn(x, x);
  if (p == 1.0) return x;
  if (p == 0.5) return sqrt(x);
  return pow(x, p);
}

__device__ __forceinline__ double clip01(double x) { return fmin(fmax(x, 0.0), 1.0); }

// ---------------------------------------------------------------------------
__global__ void k_simp(int64_t n, const double* __restrict__ rho_f, double p, double E_min,
                       double E_max, double* __restrict__ E, int* bad) {
  const double span = E_max - E_min;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double x = rho_f[e];
    if (!(x >= -1e-12 && x <= 1.0 + 1e-12)) *bad = 1;
    E[e] = __dadd_rn(E_min, __dmul_rn(np_pow(clip01(x), p), span));
  }
}

void launch_simp(int64_t n, const double* rho_f, double p, double E_min, double E_max, double* E,
                 int* bad, cudaStream_t st) {
  { k_simp<<<stream_blocks(n), kFiltThreads, 0, st>>>(n, rho_f, p, E_min, E_max, E, bad); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kFiltThreads)
    k_compliance_sens(Grid g, KeParam ke, const double* __restrict__ u, const double* __restrict__ rho_f,
                      double p, double E_min, double E_max, double* __restrict__ sens) {
  const int64_t n = (int64_t)g.nx * g.ny;
  const double coef = -p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % g.nx), j = (int)(e / g.nx);
    const int64_t n0 = (int64_t)j * g.nnx + i;
    const int64_t nd[4] = {n0, n0 + 1, n0 + g.nnx + 1, n0 + g.nnx};
    double ue[8];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      ue[a] = __ldg(u + nd[a]);
      ue[4 + a] = __ldg(u + g.n_nodes + nd[a]);
    }
    double en = 0.0;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      double ka = 0.0;
#pragma unroll
      for (int b = 0; b < 8; ++b) ka = fma(ke.k[a * 8 + b], ue[b], ka);
      en = fma(ue[a], ka, en);
    }
    const double c = np_pow(clip01(rho_f[e]), p - 1.0);
    sens[e] = __dmul_rn(__dmul_rn(__dmul_rn(coef, c), E_max - E_min), en);
  }
}

void launch_compliance_sens(const Grid& g, const KeParam& ke, const double* u_full,
                            const double* rho_f, double p, double E_min, double E_max, double* sens,
                            cudaStream_t st) {
  const int64_t n = (int64_t)g.nx * g.ny;
  { k_compliance_sens<<<stream_blocks(n), kFiltThreads, 0, st>>>(g, ke, u_full, rho_f, p, E_min,
                                                               E_max, sens); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kFiltThreads)
    k_dot(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double* out,
          double* partials, unsigned int* ticket) {
  __shared__ double sh[kFiltThreads / 32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s = fma(__ldg(a + i), __ldg(b + i), s);
  s = block_sum(s, sh);
  grid_reduce_last(s, partials, ticket, out, sh);
}

void launch_dot(int64_t n, const double* a, const double* b, double* out, double* partials,
                unsigned int* ticket, cudaStream_t st) {
  { k_dot<<<kDotBlocks, kFiltThreads, 0, st>>>(n, a, b, out, partials, ticket); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// OC: candidate(lam) = clip(clip(rho * (max(-dg,0)/(lam vol))^damping,
//                                rho - move, rho + move), 0, 1)
__device__ __forceinline__ double oc_candidate(double rho, double dg, double vol, double lam,
                                               double move, double damping) {
  const double B = __ddiv_rn(fmax(-dg, 0.0), __dmul_rn(lam, vol));
  double r = __dmul_rn(rho, np_pow(B, damping));
  r = fmin(fmax(r, __dsub_rn(rho, move)), __dadd_rn(rho, move));
  return clip01(r);
}

__global__ void k_oc_init(OcState* s, double v_star, double move, double damping) {
  OcState t{};
  t.lo = 1e-9;
  t.hi = 1e9;
  t.v_star = v_star;
  t.move = move;
  t.damping = damping;
  t.phase = 0;
  t.count = 0;
  t.evals = 0;
  *s = t;
}

void launch_oc_init(OcState* s, double v_star, double move, double damping, cudaStream_t st) {
  { k_oc_init<<<1, 1, 0, st>>>(s, v_star, move, damping); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

__global__ void __launch_bounds__(kFiltThreads)
    k_oc_eval(int64_t n, const double* __restrict__ rho, const double* __restrict__ dg,
              const double* __restrict__ vol, const double* __restrict__ wv, OcState* s,
              double* partials, unsigned int* ticket) {
  __shared__ double sh[kFiltThreads / 32];
  __shared__ bool am_last;
  const OcState st = *s;
  if (st.phase >= 2) return;  // uniform: the state only changes in the last block
  const bool two = st.phase == 0;
  const double l1 = two ? st.lo : sqrt(st.lo * st.hi);
  const double l2 = st.hi;
  double a1 = 0.0, a2 = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double r = __ldg(rho + e), d = __ldg(dg + e), v = __ldg(vol + e), w = __ldg(wv + e);
    a1 = fma(w, oc_candidate(r, d, v, l1, st.move, st.damping), a1);
    if (two) a2 = fma(w, oc_candidate(r, d, v, l2, st.move, st.damping), a2);
  }
  a1 = block_sum(a1, sh);
  a2 = block_sum(a2, sh);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = a1;
    partials[2 * blockIdx.x + 1] = a2;
    __threadfence();
    am_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double m1 = 0.0, m2 = 0.0;
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    m1 += ((volatile double*)partials)[2 * b];
    m2 += ((volatile double*)partials)[2 * b + 1];
  }
  m1 = block_sum(m1, sh);
  m2 = block_sum(m2, sh);
  if (threadIdx.x == 0) {
    *ticket = 0u;
    OcState t = st;
    if (two) {  // topopt.py:92-97
      t.evals += 2;
      if (m1 >= t.v_star && t.v_star >= m2) {
        t.phase = 1;
        t.count = 0;
      } else {
        t.lo *= 0.5;
        t.hi *= 2.0;
        if (++t.count >= 64) t.phase = 3;
      }
    } else {  // topopt.py:99-106
      t.evals += 1;
      if (m1 > t.v_star)
        t.lo = l1;
      else
        t.hi = l1;
      ++t.count;
      if (fabs(m1 - t.v_star) <= 1e-8 * t.v_star || t.count >= 200) t.phase = 2;
    }
    *s = t;
  }
}

void launch_oc_eval(int64_t n, const double* rho, const double* dg, const double* vol,
                    const double* wv, OcState* s, double* partials, unsigned int* ticket,
                    cudaStream_t st) {
  { k_oc_eval<<<kDotBlocks, kFiltThreads, 0, st>>>(n, rho, dg, vol, wv, s, partials, ticket); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

__global__ void k_oc_final(int64_t n, const double* __restrict__ rho, const double* __restrict__ dg,
                           const double* __restrict__ vol, const OcState* s,
                           double* __restrict__ rho_new) {
  const OcState st = *s;
  const double lam = sqrt(st.lo * st.hi);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    rho_new[e] = oc_candidate(rho[e], dg[e], vol[e], lam, st.move, st.damping);
}

void launch_oc_final(int64_t n, const double* rho, const double* dg, const double* vol,
                     const OcState* s, double* rho_new, cudaStream_t st) {
  { k_oc_final<<<stream_blocks(n), kFiltThreads, 0, st>>>(n, rho, dg, vol, s, rho_new); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

}  // namespace msgpu
