// Coarse level of the EH+Rot preconditioner and the additive combine.
//
// Reference: coarse.py:58-168 (basis rows, K0, Cholesky, apply_inverse),
// grid.py:172-207 (partition of unity), schwarz.py:76-84 (additive apply).
// The basis is never materialised as a sparse R0: rows are rebuilt on the fly
// from the stored eigenvectors psi, the partition-of-unity table chi and the
// rotation formula, so one restriction/prolongation streams only psi.
#include <algorithm>
#include <vector>

#include "coarse.cuh"

namespace msgpu {

// ---------------------------------------------------------------------------
// partition of unity (grid.py:172-207), bit-exact: same IEEE operations in
// the same order (no FMA contraction), hat sums accumulated in centre order.
__device__ __forceinline__ double pou_raw(const CoarseDev& cd, int I, int J, int a, int b) {
  const double x = __dmul_rn((double)a, cd.h), y = __dmul_rn((double)b, cd.h);
  const double cx = __dmul_rn((double)(I * cd.mex), cd.h);
  const double cy = __dmul_rn((double)(J * cd.mey), cd.h);
  const double Hx = __dmul_rn((double)cd.mex, cd.h), Hy = __dmul_rn((double)cd.mey, cd.h);
  const double tx = __dsub_rn(1.0, __ddiv_rn(fabs(__dsub_rn(x, cx)), Hx));
  const double ty = __dsub_rn(1.0, __ddiv_rn(fabs(__dsub_rn(y, cy)), Hy));
  return __dmul_rn(fmax(0.0, tx), fmax(0.0, ty));
}

__device__ __forceinline__ int center_index(const CoarseDev& cd, int I, int J) {
  return (J - 1) * (cd.Nx - 1) + (I - 1);
}

__device__ __forceinline__ int local_node(const CoarseDev& cd, int I, int J, int a, int b) {
  return (a - (I - 1) * cd.mex) + (b - (J - 1) * cd.mey) * cd.NLx;
}

// rotation field [-(y - y_j), x - x_j] at node (a, b) (coarse.py:120-133), no FMA contraction
__device__ __forceinline__ void rot_xy(const CoarseDev& cd, int I, int J, int a, int b, double& rx,
                                       double& ry) {
  const double x = __dmul_rn((double)a, cd.h), y = __dmul_rn((double)b, cd.h);
  const double cx = __dmul_rn((double)(I * cd.mex), cd.h), cy = __dmul_rn((double)(J * cd.mey), cd.h);
  rx = -__dsub_rn(y, cy);
  ry = __dsub_rn(x, cx);
}

__global__ void k_pou_table(Grid g, CoarseDev cd, double* __restrict__ chi) {
  const int k = blockIdx.x;
  const int I = k % (cd.Nx - 1) + 1, J = k / (cd.Nx - 1) + 1;
  const int NL = cd.NLx * cd.NLy;
  for (int ln = threadIdx.x; ln < NL; ln += blockDim.x) {
    const int a = (I - 1) * cd.mex + ln % cd.NLx, b = (J - 1) * cd.mey + ln / cd.NLx;
    // centres whose closed neighbourhood contains (a, b), J-major
    const int ilo = max(1, (a + cd.mex - 1) / cd.mex - 1), ihi = min(cd.Nx - 1, a / cd.mex + 1);
    const int jlo = max(1, (b + cd.mey - 1) / cd.mey - 1), jhi = min(cd.Ny - 1, b / cd.mey + 1);
    double total = 0.0;
    for (int jj = jlo; jj <= jhi; ++jj)
      for (int ii = ilo; ii <= ihi; ++ii) total = __dadd_rn(total, pou_raw(cd, ii, jj, a, b));
    const double safe = total > 0.0 ? total : 1.0;
    chi[(int64_t)k * NL + ln] = __ddiv_rn(pou_raw(cd, I, J, a, b), safe);
  }
}

void launch_pou_table(const Grid& g, const CoarseDev& cd, double* chi, cudaStream_t st) {
  if (cd.n_centers == 0) return;
  { k_pou_table<<<cd.n_centers, 256, 0, st>>>(g, cd, chi); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// value of basis row `bi` of centre k at global node (a, b), component c.
// heat: bi < 2*nsel: mode bi/2 in slot bi%2; bi == 2*nsel: rotation.
// vec (EE): mode bi, component c of chi * psi (coarse.py:76-91).
__device__ __forceinline__ double basis_value(const CoarseDev& cd, int k, int I, int J, int bi,
                                              int nsel, int a, int b, int c) {
  const int NL = cd.NLx * cd.NLy;
  const int ln = local_node(cd, I, J, a, b);
  const double chi = cd.chi[(int64_t)k * NL + ln];
  if (cd.vec) return __dmul_rn(chi, cd.psi[cd.psioff[k] + ((int64_t)bi * 2 + c) * NL + ln]);
  if (bi < 2 * nsel) {
    if ((bi & 1) != c) return 0.0;
    return __dmul_rn(chi, cd.psi[cd.psioff[k] + (int64_t)(bi >> 1) * NL + ln]);
  }
  double rx, ry;
  rot_xy(cd, I, J, a, b, rx, ry);
  return __dmul_rn(chi, c == 0 ? rx : ry);
}

__device__ __forceinline__ int basis_row(const CoarseDev& cd, int k, int bi, int nsel) {
  return (cd.vec || bi < 2 * nsel) ? cd.hoff[k] + bi : cd.roff + k;
}

__device__ __forceinline__ int basis_count(const CoarseDev& cd, int nsel) {
  return cd.vec ? nsel : 2 * nsel + cd.enrich;
}


// ---------------------------------------------------------------------------
// Node-major coarse tables: for each node, the chi (and chi * psi_0) of the
// 4 corner centres of its coarse cell, so the per-iteration restriction and
// prolongation read one contiguous 32-byte record per node instead of 4-8
// scattered per-centre streams.
__device__ __forceinline__ void node_cell(const Grid& g, const CoarseDev& cd, int a, int b, int& ci,
                                          int& cj) {
  ci = min(a / cd.mex, cd.Nx - 1);
  cj = min(b / cd.mey, cd.Ny - 1);
}

__global__ void k_node_tables(Grid g, CoarseDev cd, double* __restrict__ chi4,
                              double* __restrict__ psi4) {
  const int NL = cd.NLx * cd.NLy;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < g.n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(n % g.nnx), b = (int)(n / g.nnx);
    int ci, cj;
    node_cell(g, cd, a, b, ci, cj);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int I = ci + (c & 1), J = cj + (c >> 1);
      double ch = 0.0, ps = 0.0;
      if (I >= 1 && I <= cd.Nx - 1 && J >= 1 && J <= cd.Ny - 1) {
        const int k = center_index(cd, I, J), ln = local_node(cd, I, J, a, b);
        ch = cd.chi[(int64_t)k * NL + ln];
        ps = __dmul_rn(ch, cd.psi[cd.psioff[k] + ln]);
      }
      chi4[n * 4 + c] = ch;
      psi4[n * 4 + c] = ps;
    }
  }
}

void launch_node_tables(const Grid& g, const CoarseDev& cd, double* chi4, double* psi4,
                        cudaStream_t st) {
  if (cd.n_centers == 0) return;
  { k_node_tables<<<148 * 8, 256, 0, st>>>(g, cd, chi4, psi4); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

__global__ void __launch_bounds__(256) k_psi0_const(CoarseDev cd, double* __restrict__ psi0c) {
  const int k = blockIdx.x, NL = cd.NLx * cd.NLy;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  if (cd.nsel[k] < 1) {  // no mode stored for this centre (CTA-uniform)
    if (threadIdx.x == 0) psi0c[k] = nan;
    return;
  }
  const double* ps = cd.psi + cd.psioff[k];
  const double v0 = ps[0];
  int same = 1;
  for (int i = threadIdx.x; i < NL; i += blockDim.x) same &= (ps[i] == v0) ? 1 : 0;
  same = __syncthreads_and(same);
  if (threadIdx.x == 0) psi0c[k] = same ? v0 : nan;
}

void launch_psi0_const(const CoarseDev& cd, double* psi0c, cudaStream_t st) {
  if (cd.n_centers == 0 || cd.vec) return;
  { k_psi0_const<<<cd.n_centers, 256, 0, st>>>(cd, psi0c); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// cell (ci, cj): node range and size (the last cell row / column owns the far boundary nodes)
__device__ __forceinline__ void cell_box(const Grid& g, int Nx, int Ny, int ci, int cj, int& a_lo, int& b_lo, int& w,
                                         int& hgt) {
  const int mx = g.nx / Nx, my = g.ny / Ny;
  a_lo = ci * mx;
  b_lo = cj * my;
  w = ((ci == Nx - 1) ? g.nx : a_lo + mx - 1) - a_lo + 1;
  hgt = ((cj == Ny - 1) ? g.ny : b_lo + my - 1) - b_lo + 1;
}

__global__ void __launch_bounds__(256) k_chi_dedup(Grid g, CoarseDev cd, int* __restrict__ chi_src) {
  const int ci = blockIdx.x, cj = blockIdx.y, Nx = cd.Nx, Ny = cd.Ny;
  // class representative: same position class per axis (first / interior / last)
  const int ri = (ci == 0 || ci == Nx - 1) ? ci : 1, rj = (cj == 0 || cj == Ny - 1) ? cj : 1;
  int a_lo, b_lo, w, hgt, ra, rb, rw, rh;
  cell_box(g, Nx, Ny, ci, cj, a_lo, b_lo, w, hgt);
  cell_box(g, Nx, Ny, ri, rj, ra, rb, rw, rh);
  int same = (rw == w && rh == hgt) ? 1 : 0;
  if (same && (ri != ci || rj != cj)) {
    for (int t = threadIdx.x; t < w * hgt; t += blockDim.x) {
      const int lb = t / w, la = t - lb * w;
      const int64_t n = (int64_t)(b_lo + lb) * g.nnx + a_lo + la, m = (int64_t)(rb + lb) * g.nnx + ra + la;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        same &= (__double_as_longlong(cd.chi4[n * 4 + c]) == __double_as_longlong(cd.chi4[m * 4 + c])) ? 1 : 0;
    }
  }
  same = __syncthreads_and(same);
  if (threadIdx.x == 0) chi_src[cj * Nx + ci] = same ? rj * Nx + ri : cj * Nx + ci;
}

void launch_chi_dedup(const Grid& g, const CoarseDev& cd, int* chi_src, cudaStream_t st) {
  if (cd.n_centers == 0 || cd.vec) return;
  { k_chi_dedup<<<dim3(cd.Nx, cd.Ny), 256, 0, st>>>(g, cd, chi_src); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// origin of the cell whose chi4 records this cell reads (CTA-uniform)
__device__ __forceinline__ void chi_origin(const Grid& g, const CoarseDev& cd, int ci, int cj, int a_lo, int b_lo,
                                           int& ca, int& cb) {
  ca = a_lo;
  cb = b_lo;
  if (cd.chi_src) {
    const int src = __ldg(cd.chi_src + cj * cd.Nx + ci);
    int w, hgt;
    cell_box(g, cd.Nx, cd.Ny, src % cd.Nx, src / cd.Nx, ca, cb, w, hgt);
  }
}

// mode-0 values of a cell's 4 corner centres when all of them are constant
// (then psi4 = chi4 * value needs no table read); CTA-uniform
__device__ __forceinline__ bool cell_psi0_const(const CoarseDev& cd, const bool cok[4], int ci, int cj, double pv0[4]) {
  bool all = cd.psi0c != nullptr;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    pv0[c] = 0.0;
    if (all && cok[c]) {
      const int I = ci + (c & 1), J = cj + (c >> 1);
      pv0[c] = __ldg(cd.psi0c + (J - 1) * (cd.Nx - 1) + (I - 1));
      all = pv0[c] == pv0[c];  // NaN: mode 0 of this centre is not constant
    }
  }
  return all;
}

// ---------------------------------------------------------------------------
// Cell-tiled restriction, optionally fused with the PCG residual update.
// One CTA per coarse cell accumulates, for each of its <= 4 corner centres,
// the mode-0 x/y rows and the rotation row over the cell's nodes (extra modes
// in a second pass), and writes them to rpart[cell][corner][slot]; the
// partials of the 4 cells around a centre are summed in a fixed order by
// k_restrict_reduce.  With UPD, the same pass performs x += alpha p,
// r -= alpha q and the ||r||^2 grid reduction / convergence test.
constexpr int kCellThreads = 256;

#ifndef MS_CR_MINB
#define MS_CR_MINB 5
#endif
#ifndef MS_CB_MINB
#define MS_CB_MINB 6
#endif
#ifndef MS_CB2_MINB
#define MS_CB2_MINB 5
#endif
#ifndef MS_CR2_TPB
#define MS_CR2_TPB 128
#endif
#ifndef MS_CR2_MINB
#define MS_CR2_MINB 4
#endif
template <bool UPD, bool VEC, int NU, int MINB, int TPB = kCellThreads>
__global__ void __launch_bounds__(TPB, MINB)
    k_cell_restrict(Grid g, CoarseDev cd, int has_coarse, int J0, double* __restrict__ x,
                    const double* __restrict__ p, double* __restrict__ r,
                    const double* __restrict__ q, PcgScalars* sc, double* partials,
                    double* res_hist, const int* done) {
  if (UPD ? sc->done : (done && *(volatile const int*)done)) return;
  __shared__ double sred[13 * (TPB / 32)];
  const int64_t nn = g.n_nodes;
  const int ci = blockIdx.x, cj = J0 + blockIdx.y, Nx = cd.Nx, Ny = cd.Ny;
  const int mx = g.nx / Nx, my = g.ny / Ny;
  const int a_lo = ci * mx, a_hi = (ci == Nx - 1) ? g.nx : a_lo + mx - 1;
  const int b_lo = cj * my, b_hi = (cj == Ny - 1) ? g.ny : b_lo + my - 1;
  const int w = a_hi - a_lo + 1, hgt = b_hi - b_lo + 1;
  const double alpha = UPD ? sc->alpha : 0.0;
  bool cok[4];
  int cns[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int I = ci + (c & 1), J = cj + (c >> 1);
    cok[c] = has_coarse && I >= 1 && I <= Nx - 1 && J >= 1 && J <= Ny - 1;
    cns[c] = cok[c] ? __ldg(cd.nsel + (J - 1) * (Nx - 1) + (I - 1)) : 0;
  }
  double pv0[4];
  const bool pconst = !VEC && has_coarse && cell_psi0_const(cd, cok, ci, cj, pv0);
  int cha = a_lo, chb = b_lo;  // origin of the cell whose chi4 records are read (bitwise identical ones)
  if (!VEC && has_coarse) chi_origin(g, cd, ci, cj, a_lo, b_lo, cha, chb);
  double acc[13];
#pragma unroll
  for (int v = 0; v < 13; ++v) acc[v] = 0.0;  // [4 corners][x, y, rot] + ||r||^2
  // NU nodes per thread in flight: all their loads are issued before the first
  // is consumed; per-node arithmetic and accumulation order do not depend on NU.
  const int total = w * hgt;
  const unsigned wmagic = 0xFFFFFFFFu / (unsigned)w + 1u;
  for (int t0 = threadIdx.x; t0 < total; t0 += NU * TPB) {
    int a[NU], b[NU];
    int64_t n[NU];
    bool ok[NU];
    double rx[NU], ry[NU], px[NU], py[NU], qx[NU], qy[NU], xx[NU], xy[NU];
    double2 c4[NU][2], p4[NU][2];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int t = t0 + u * TPB;
      ok[u] = t < total;
      const int tt = ok[u] ? t : 0;
      const int lbu = (int)__umulhi((unsigned)tt, wmagic);  // tt / w (exact: tt * w < 2^32)
      b[u] = b_lo + lbu;
      a[u] = a_lo + tt - lbu * w;
      n[u] = (int64_t)b[u] * g.nnx + a[u];
      MS_BCHECK(a[u] >= 0 && a[u] <= g.nx && b[u] >= 0 && b[u] <= g.ny && n[u] < nn);
      rx[u] = ok[u] ? r[n[u]] : 0.0;
      ry[u] = ok[u] ? r[n[u] + nn] : 0.0;
      if (UPD) {
        xx[u] = ok[u] ? x[n[u]] : 0.0;
        xy[u] = ok[u] ? x[n[u] + nn] : 0.0;
        px[u] = ok[u] ? p[n[u]] : 0.0;
        py[u] = ok[u] ? p[n[u] + nn] : 0.0;
        qx[u] = ok[u] ? q[n[u]] : 0.0;
        qy[u] = ok[u] ? q[n[u] + nn] : 0.0;
      }
      c4[u][0] = c4[u][1] = p4[u][0] = p4[u][1] = make_double2(0.0, 0.0);
      if (!VEC && has_coarse && ok[u]) {
        const int64_t nc4 = (int64_t)(chb + (b[u] - b_lo)) * g.nnx + cha + (a[u] - a_lo);
        const double2* c2 = reinterpret_cast<const double2*>(cd.chi4) + 2 * nc4;
        const double2* p2 = reinterpret_cast<const double2*>(cd.psi4) + 2 * n[u];
        c4[u][0] = __ldg(c2);
        c4[u][1] = __ldg(c2 + 1);
        if (!pconst) {
          p4[u][0] = __ldg(p2);
          p4[u][1] = __ldg(p2 + 1);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      if (!ok[u]) continue;
      double rxu = rx[u], ryu = ry[u];
      if (UPD) {
        x[n[u]] = xx[u] + alpha * px[u];
        x[n[u] + nn] = xy[u] + alpha * py[u];
        rxu -= alpha * qx[u];
        ryu -= alpha * qy[u];
        r[n[u]] = rxu;
        r[n[u] + nn] = ryu;
        acc[12] += rxu * rxu + ryu * ryu;
      }
      if (!VEC && has_coarse) {
        const double ch4[4] = {c4[u][0].x, c4[u][0].y, c4[u][1].x, c4[u][1].y};
        double ps4[4] = {p4[u][0].x, p4[u][0].y, p4[u][1].x, p4[u][1].y};
        if (pconst) {  // the table's own product (k_node_tables)
#pragma unroll
          for (int c = 0; c < 4; ++c) ps4[c] = __dmul_rn(ch4[c], pv0[c]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int I = ci + (c & 1), J = cj + (c >> 1);
          double ex, ey;
          rot_xy(cd, I, J, a[u], b[u], ex, ey);
          acc[3 * c] += ps4[c] * rxu;
          acc[3 * c + 1] += ps4[c] * ryu;
          acc[3 * c + 2] += __dmul_rn(ch4[c], ex) * rxu + __dmul_rn(ch4[c], ey) * ryu;
        }
      }
    }
  }
  // one multi-value block reduction (13 values)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < 13; ++v) {
    const double s = warp_sum(acc[v]);
    if (lane == 0) sred[v * (TPB / 32) + warp] = s;
  }
  __syncthreads();
  double* rp = cd.rpart + ((int64_t)cj * Nx + ci) * 4 * kSlots;
  __shared__ double rrblk;
  if (threadIdx.x < 13) {
    double s = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < TPB / 32; ++w2) s += sred[threadIdx.x * (TPB / 32) + w2];
    if (threadIdx.x == 12) {
      rrblk = s;
    } else if (!VEC && has_coarse) {
      const int c = threadIdx.x / 3, v = threadIdx.x % 3;
      rp[c * kSlots + (v == 2 ? 2 * kMaxModes : v)] = s;
    }
  }
  // vec basis: all modes in one pass, <= 4 corners x kMaxModes rows
  if constexpr (VEC) {
    __syncthreads();  // r of this cell is final
    const int NL = cd.NLx * cd.NLy;
    double va[4 * kMaxModes];
#pragma unroll
    for (int v = 0; v < 4 * kMaxModes; ++v) va[v] = 0.0;
    const double* psk[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int I = ci + (c & 1), J = cj + (c >> 1);
      psk[c] = cok[c] ? cd.psi + __ldg(cd.psioff + (J - 1) * (Nx - 1) + (I - 1)) : cd.psi;
    }
    for (int t = threadIdx.x; t < w * hgt; t += TPB) {
      const int b = b_lo + t / w, a = a_lo + t - (t / w) * w;
      const int64_t n = (int64_t)b * g.nnx + a;
      const double rx = r[n], ry = r[n + nn];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (!cok[c]) continue;
        const int I = ci + (c & 1), J = cj + (c >> 1);
        const int ln = (a - (I - 1) * cd.mex) + (b - (J - 1) * cd.mey) * cd.NLx;
        const double ch = cd.chi4[n * 4 + c];
#pragma unroll
        for (int m = 0; m < kMaxModes; ++m)
          if (m < cns[c]) {
            const double* pm = psk[c] + (int64_t)m * 2 * NL + ln;
            va[c * kMaxModes + m] += __dmul_rn(ch, __ldg(pm)) * rx + __dmul_rn(ch, __ldg(pm + NL)) * ry;
          }
      }
    }
#pragma unroll
    for (int v = 0; v < 4 * kMaxModes; ++v) {
      const int c = v / kMaxModes, m = v % kMaxModes;
      if (m < cns[c]) {  // CTA-uniform
        const double tv = block_sum(va[v], sred);
        if (threadIdx.x == 0) rp[c * kSlots + m] = tv;
      }
    }
  }
  // extra modes (rare): second pass over the cell for corners with nsel > 1
  if (!VEC && has_coarse && (cns[0] > 1 || cns[1] > 1 || cns[2] > 1 || cns[3] > 1)) {
    __syncthreads();  // r of this cell is final
    const int NL = cd.NLx * cd.NLy;
    for (int c = 0; c < 4; ++c) {
      const int I = ci + (c & 1), J = cj + (c >> 1);
      if (cns[c] <= 1) continue;
      const int k = (J - 1) * (Nx - 1) + (I - 1);
      const double* psk = cd.psi + __ldg(cd.psioff + k);
      for (int m = 1; m < cns[c]; ++m) {
        double sx = 0.0, sy = 0.0;
        for (int t = threadIdx.x; t < w * hgt; t += TPB) {
          const int b = b_lo + t / w, a = a_lo + t - (t / w) * w;
          const int64_t n = (int64_t)b * g.nnx + a;
          const int ln = (a - (I - 1) * cd.mex) + (b - (J - 1) * cd.mey) * cd.NLx;
          const double v = cd.chi4[n * 4 + c] * __ldg(psk + (int64_t)m * NL + ln);
          sx += v * r[n];
          sy += v * r[n + nn];
        }
        const double tx = block_sum(sx, sred), ty = block_sum(sy, sred);
        if (threadIdx.x == 0) {
          rp[c * kSlots + 2 * m] = tx;
          rp[c * kSlots + 2 * m + 1] = ty;
        }
      }
    }
  }
  if (!UPD) return;
  __syncthreads();
  double tot;
  if (grid_reduce_dist(threadIdx.x == 0 ? rrblk : 0.0, partials, (J0 + blockIdx.y) * gridDim.x + blockIdx.x,
                       sc->dist && sc->bitwise, &sc->tickets[1], &tot, sred)) {
    if (threadIdx.x == 0) {
      if (sc->dist)
        sc->part[PART_RR] = tot;
      else
        fin_res(sc, tot, res_hist);
    }
  }
}

static int restrict_nu() {
  static int v = [] {
    const char* e = getenv("MS_RESTRICT_NU");  // A/B knob: 1 = one node per thread in flight
    return (e && atoi(e) == 1) ? 1 : 2;
  }();
  return v;
}

int update_restrict_threads(const CoarseDev& cd) {
  return (!cd.vec && restrict_nu() == 2) ? MS_CR2_TPB : kCellThreads;
}
void launch_update_restrict(const Grid& g, int J0, int J1, double* x, const double* p, double* r,
                            const double* q, const CoarseDev& cd, PcgScalars* sc,
                            double* partials, double* res_hist, cudaStream_t st) {
  const dim3 grid(cd.Nx, J1 - J0);
  if (cd.vec)
    { k_cell_restrict<true, true, 1, MS_CR_MINB><<<grid, kCellThreads, 0, st>>>(g, cd, 1, J0, x, p, r, q, sc, partials,
                                                                  res_hist, nullptr); ms_count_launch(); }
  else if (restrict_nu() == 2)
    { k_cell_restrict<true, false, 2, MS_CR2_MINB, MS_CR2_TPB><<<grid, MS_CR2_TPB, 0, st>>>(g, cd, 1, J0, x, p, r, q, sc, partials,
                                                                      res_hist, nullptr); ms_count_launch(); }
  else
    { k_cell_restrict<true, false, 1, MS_CR_MINB><<<grid, kCellThreads, 0, st>>>(g, cd, 1, J0, x, p, r, q, sc, partials,
                                                                   res_hist, nullptr); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

void launch_restrict_cells(const Grid& g, int J0, int J1, const CoarseDev& cd, const double* r,
                           const int* done, cudaStream_t st) {
  const dim3 grid(cd.Nx, J1 - J0);
  if (cd.vec)
    { k_cell_restrict<false, true, 1, MS_CR_MINB><<<grid, kCellThreads, 0, st>>>(
        g, cd, 1, J0, nullptr, nullptr, const_cast<double*>(r), nullptr, nullptr, nullptr, nullptr, done); ms_count_launch(); }
  else if (restrict_nu() == 2)
    { k_cell_restrict<false, false, 2, 2><<<grid, kCellThreads, 0, st>>>(
        g, cd, 1, J0, nullptr, nullptr, const_cast<double*>(r), nullptr, nullptr, nullptr, nullptr, done); ms_count_launch(); }
  else
    { k_cell_restrict<false, false, 1, MS_CR_MINB><<<grid, kCellThreads, 0, st>>>(
        g, cd, 1, J0, nullptr, nullptr, const_cast<double*>(r), nullptr, nullptr, nullptr, nullptr, done); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// f0 rows of centre k = sum of the partials of the 4 cells around it, in
// J-major cell order; centre (I, J) is corner (I-ci) + 2 (J-cj) of cell (ci, cj)
__global__ void k_restrict_reduce(CoarseDev cd, double* __restrict__ f0, const int* done, int k_begin,
                                  int k_end) {
  if (done && *(volatile const int*)done) return;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = k_begin + t / kSlots, slot = t % kSlots;
  if (k >= k_end) return;
  const int nsel = cd.nsel[k];
  const bool rot = !cd.vec && slot == 2 * kMaxModes;
  if (!(slot < (cd.vec ? nsel : 2 * nsel) || (rot && cd.enrich))) return;
  const int I = k % (cd.Nx - 1) + 1, J = k / (cd.Nx - 1) + 1;
  double s = 0.0;
#pragma unroll
  for (int dy = 0; dy < 2; ++dy)
#pragma unroll
    for (int dx = 0; dx < 2; ++dx) {
      const int ci = I - 1 + dx, cj = J - 1 + dy;
      const int c = (I - ci) + 2 * (J - cj);
      s += cd.rpart[((int64_t)cj * cd.Nx + ci) * 4 * kSlots + c * kSlots + slot];
    }
  f0[rot ? cd.roff + k : cd.hoff[k] + slot] = s;
}

void launch_restrict_reduce(const CoarseDev& cd, double* f0, const int* done, cudaStream_t st,
                            int k_begin, int k_end) {
  if (k_end < 0) k_end = cd.n_centers;
  if (k_end <= k_begin) return;
  const int total = (k_end - k_begin) * kSlots;
  { k_restrict_reduce<<<div_up(total, 256), 256, 0, st>>>(cd, f0, done, k_begin, k_end); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// One CTA per coarse cell [ci*mex, (ci+1)*mex) x [cj*mey, (cj+1)*mey) (the last
// cell row/column also owns the domain's far boundary nodes).  Every node of
// the cell sees the same <= 4 coarse centres (ci..ci+1, cj..cj+1), so their
// metadata and y0 entries are CTA-uniform registers; the per-node work is the
// chi / psi loads and FMAs.  Level-1 covers: <= 2 per axis, unrolled 2x2 with
// predicated loads.  Summation order: level-1 in J-major subdomain order,
// coarse part in J-major centre order, then their sum.
constexpr int kCombineThreads = 256;

template <bool VEC>
__global__ void __launch_bounds__(kCombineThreads, MS_CB_MINB)
    k_combine(Grid g, const uint8_t* __restrict__ mask, L1Dev l1, int has_l1, CoarseDev cd,
              int has_coarse, int Nx, int Ny, int J0, const double* __restrict__ y0,
              const double* __restrict__ r, double* __restrict__ z, PcgScalars* sc,
              double* partials, double* beta_hist) {
  if (sc && sc->done) return;
  __shared__ double sred[kCombineThreads / 32];
  const int64_t nn = g.n_nodes;
  const int ci = blockIdx.x, cj = J0 + blockIdx.y;
  const int mx = g.nx / Nx, my = g.ny / Ny;
  const int a_lo = ci * mx, a_hi = (ci == Nx - 1) ? g.nx : a_lo + mx - 1;
  const int b_lo = cj * my, b_hi = (cj == Ny - 1) ? g.ny : b_lo + my - 1;
  const int w = a_hi - a_lo + 1, hgt = b_hi - b_lo + 1;
  // the cell's coarse centres, J-major: (ci,cj) (ci+1,cj) (ci,cj+1) (ci+1,cj+1)
  bool cok[4];
  int ck[4], cns[4];
  int64_t cpo[4];
  __shared__ double cy[4][2 * kMaxModes + 1];
  const int NL = has_coarse ? cd.NLx * cd.NLy : 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int I = ci + (c & 1), J = cj + (c >> 1);
    cok[c] = has_coarse && I >= 1 && I <= Nx - 1 && J >= 1 && J <= Ny - 1;
    ck[c] = cok[c] ? (J - 1) * (Nx - 1) + (I - 1) : 0;
    cns[c] = cok[c] ? __ldg(cd.nsel + ck[c]) : 0;
    cpo[c] = cok[c] ? __ldg(cd.psioff + ck[c]) : 0;
  }
  if (threadIdx.x < 4 * (2 * kMaxModes + 1)) {
    const int c = threadIdx.x / (2 * kMaxModes + 1), m = threadIdx.x % (2 * kMaxModes + 1);
    double v = 0.0;
    if (cok[c]) {
      if (m < (cd.vec ? cns[c] : 2 * cns[c]))
        v = y0[__ldg(cd.hoff + ck[c]) + m];
      else if (m == 2 * kMaxModes && cd.enrich)
        v = y0[cd.roff + ck[c]];
    }
    cy[c][m] = v;
  }
  __syncthreads();
  double dot = 0.0;
  for (int t = threadIdx.x; t < w * hgt; t += kCombineThreads) {
    const int b = b_lo + t / w, a = a_lo + t - (t / w) * w;
    const int64_t n = (int64_t)b * g.nnx + a;
    double zx = 0.0, zy = 0.0;
    if (has_l1) {
      const int Js[2] = {l1.ycov[b * 4], l1.ycov[b * 4 + 1]};
      const int Is[2] = {l1.xcov[a * 4], l1.xcov[a * 4 + 1]};
      double2 v[2][2];
#pragma unroll
      for (int tj = 0; tj < 2; ++tj)
#pragma unroll
        for (int ti = 0; ti < 2; ++ti) {
          const int J = Js[tj], I = Is[ti];
          v[tj][ti] = make_double2(0.0, 0.0);
          if (J >= 0 && I >= 0) {
            const int y0_ = l1.ylo[J], hy = l1.ylen[J], x0_ = l1.xlo[I], wx = l1.xlen[I];
            const int ln = (wx <= hy) ? (b - y0_) * wx + (a - x0_) : (a - x0_) * hy + (b - y0_);
            v[tj][ti] = __ldg(reinterpret_cast<const double2*>(l1.ybuf + l1.yoff[J * l1.NbX + I] + 2 * ln));
          }
        }
#pragma unroll
      for (int tj = 0; tj < 2; ++tj)
#pragma unroll
        for (int ti = 0; ti < 2; ++ti) {
          zx += v[tj][ti].x;
          zy += v[tj][ti].y;
        }
    }
    if (VEC && has_coarse) {
      double cxs = 0.0, cys = 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (!cok[c]) continue;
        const int I = ci + (c & 1), J = cj + (c >> 1);
        const int ln = (a - (I - 1) * cd.mex) + (b - (J - 1) * cd.mey) * cd.NLx;
        const double ch = cd.chi4[n * 4 + c];
        const double* ps = cd.psi + cpo[c] + ln;
        for (int m = 0; m < cns[c]; ++m) {
          cxs += __dmul_rn(ch, __ldg(ps + (int64_t)m * 2 * NL)) * cy[c][m];
          cys += __dmul_rn(ch, __ldg(ps + (int64_t)m * 2 * NL + NL)) * cy[c][m];
        }
      }
      zx += cxs;
      zy += cys;
    } else if (!VEC && has_coarse) {
      double cxs = 0.0, cys = 0.0;
      const double2* c2 = reinterpret_cast<const double2*>(cd.chi4) + 2 * n;
      const double2* p2 = reinterpret_cast<const double2*>(cd.psi4) + 2 * n;
      const double2 c4a = __ldg(c2), c4b = __ldg(c2 + 1), p4a = __ldg(p2), p4b = __ldg(p2 + 1);
      const double ch4[4] = {c4a.x, c4a.y, c4b.x, c4b.y};
      const double ps4[4] = {p4a.x, p4a.y, p4b.x, p4b.y};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (!cok[c]) continue;
        const int I = ci + (c & 1), J = cj + (c >> 1);
        cxs += ps4[c] * cy[c][0];
        cys += ps4[c] * cy[c][1];
        if (cns[c] > 1) {  // rare: extra modes from the per-centre store
          const int ln = (a - (I - 1) * cd.mex) + (b - (J - 1) * cd.mey) * cd.NLx;
          const double* ps = cd.psi + cpo[c] + ln;
          for (int m = 1; m < cns[c]; ++m) {
            const double vv = ch4[c] * __ldg(ps + (int64_t)m * NL);
            cxs += vv * cy[c][2 * m];
            cys += vv * cy[c][2 * m + 1];
          }
        }
        if (cd.enrich) {
          double ex, ey;
          rot_xy(cd, I, J, a, b, ex, ey);
          cxs += __dmul_rn(ch4[c], ex) * cy[c][2 * kMaxModes];
          cys += __dmul_rn(ch4[c], ey) * cy[c][2 * kMaxModes];
        }
      }
      zx += cxs;
      zy += cys;
    }
    zx = mask[n] ? zx : 0.0;
    zy = mask[n + nn] ? zy : 0.0;
    z[n] = zx;
    z[n + nn] = zy;
    if (sc) dot += zx * r[n] + zy * r[n + nn];
  }
  if (!sc) return;
  const double bs = block_sum(dot, sred);
  double tot;
  if (grid_reduce_dist(bs, partials, (J0 + blockIdx.y) * gridDim.x + blockIdx.x, sc->dist && sc->bitwise,
                       &sc->tickets[2], &tot, sred)) {
    if (threadIdx.x == 0) {
      if (sc->dist)
        sc->part[PART_RZ] = tot;
      else
        fin_beta(sc, tot, beta_hist);
    }
  }
}

// Same combine for the implicit (non-vector) basis with the level-1 cover
// metadata of the cell staged once per CTA: the per-node chain cover table ->
// subdomain extents -> local-vector offset -> y (three dependent global loads
// per node above) becomes shared-memory lookups plus the y load itself, and NU
// nodes per thread are in flight.  Same values, same summation order per
// thread as k_combine<false> (bitwise identical z and r.z).
constexpr int kCellMax = 72;  // largest cell side (nodes) the staged tables hold
template <int NU>
__global__ void __launch_bounds__(kCombineThreads, NU == 1 ? MS_CB2_MINB : 3)
    k_combine2(Grid g, const uint8_t* __restrict__ mask, L1Dev l1, CoarseDev cd, int has_coarse, int Nx, int Ny,
               int J0, const double* __restrict__ y0, const double* __restrict__ r, double* __restrict__ z,
               PcgScalars* sc, double* partials, double* beta_hist) {
  if (sc && sc->done) return;
  __shared__ double sred[kCombineThreads / 32];
  __shared__ int4 sx[2 * kCellMax], sy[2 * kCellMax];  // per column / row and cover: (I, lo, len, -)
  __shared__ int64_t syoff[16];                        // yoff of (Jmin + dj, Imin + di)
  const int64_t nn = g.n_nodes;
  const int ci = blockIdx.x, cj = J0 + blockIdx.y;
  const int mx = g.nx / Nx, my = g.ny / Ny;
  const int a_lo = ci * mx, a_hi = (ci == Nx - 1) ? g.nx : a_lo + mx - 1;
  const int b_lo = cj * my, b_hi = (cj == Ny - 1) ? g.ny : b_lo + my - 1;
  const int w = a_hi - a_lo + 1, hgt = b_hi - b_lo + 1;
  bool cok[4];
  int ck[4], cns[4];
  int64_t cpo[4];
  __shared__ double cy[4][2 * kMaxModes + 1];
  const int NL = has_coarse ? cd.NLx * cd.NLy : 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int I = ci + (c & 1), J = cj + (c >> 1);
    cok[c] = has_coarse && I >= 1 && I <= Nx - 1 && J >= 1 && J <= Ny - 1;
    ck[c] = cok[c] ? (J - 1) * (Nx - 1) + (I - 1) : 0;
    cns[c] = cok[c] ? __ldg(cd.nsel + ck[c]) : 0;
    cpo[c] = cok[c] ? __ldg(cd.psioff + ck[c]) : 0;
  }
  if (threadIdx.x < 4 * (2 * kMaxModes + 1)) {
    const int c = threadIdx.x / (2 * kMaxModes + 1), m = threadIdx.x % (2 * kMaxModes + 1);
    double v = 0.0;
    if (cok[c]) {
      if (m < 2 * cns[c])
        v = y0[__ldg(cd.hoff + ck[c]) + m];
      else if (m == 2 * kMaxModes && cd.enrich)
        v = y0[cd.roff + ck[c]];
    }
    cy[c][m] = v;
  }
  double pv0[4];
  const bool pconst = has_coarse && cell_psi0_const(cd, cok, ci, cj, pv0);
  int cha = a_lo, chb = b_lo;
  if (has_coarse) chi_origin(g, cd, ci, cj, a_lo, b_lo, cha, chb);
  // cover tables of the cell's columns and rows; covers are listed in
  // ascending block order, so the first cover of the first column / row is
  // the smallest block index of the cell
  // (the first COVERED column / row: clamped boundary nodes may have no cover)
  int Imin = -1, Jmin = -1;
  for (int a = a_lo; a <= a_hi && Imin < 0; ++a) Imin = __ldg(l1.xcov + a * 4);
  for (int b = b_lo; b <= b_hi && Jmin < 0; ++b) Jmin = __ldg(l1.ycov + b * 4);
  for (int t = threadIdx.x; t < 2 * (w + hgt); t += kCombineThreads) {
    const bool isx = t < 2 * w;
    const int u = isx ? t : t - 2 * w;
    const int pos = (isx ? a_lo : b_lo) + (u >> 1);
    const int B = __ldg((isx ? l1.xcov : l1.ycov) + pos * 4 + (u & 1));
    int4 e = make_int4(B, 0, 1, 0);
    if (B >= 0) {
      e.y = __ldg((isx ? l1.xlo : l1.ylo) + B);
      e.z = __ldg((isx ? l1.xlen : l1.ylen) + B);
    }
    (isx ? sx : sy)[u] = e;
  }
  if (threadIdx.x >= 64 && threadIdx.x < 80) {
    const int dj = (threadIdx.x - 64) >> 2, di = (threadIdx.x - 64) & 3;
    const int J = Jmin + dj, I = Imin + di;
    syoff[threadIdx.x - 64] = (Imin >= 0 && Jmin >= 0 && J < l1.NbY && I < l1.NbX) ? __ldg(l1.yoff + J * l1.NbX + I) : 0;
  }
  __syncthreads();
  double dot = 0.0;
  const int total = w * hgt;
  const unsigned wmagic = 0xFFFFFFFFu / (unsigned)w + 1u;  // floor(t / w) = umulhi(t, wmagic) for t * w < 2^32
  for (int t0 = threadIdx.x; t0 < total; t0 += NU * kCombineThreads) {
    int a[NU], b[NU];
    int64_t n[NU];
    bool ok[NU];
    double2 v[NU][2][2], c4a[NU], c4b[NU], p4a[NU], p4b[NU];
    double rx[NU], ry[NU];
    uint8_t mk[NU][2];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int t = t0 + u * kCombineThreads;
      ok[u] = t < total;
      const int tt = ok[u] ? t : 0;
      const int lb = (int)__umulhi((unsigned)tt, wmagic), la = tt - lb * w;  // tt / w (exact: tt * w < 2^32)
      b[u] = b_lo + lb;
      a[u] = a_lo + la;
      n[u] = (int64_t)b[u] * g.nnx + a[u];
#pragma unroll
      for (int tj = 0; tj < 2; ++tj)
#pragma unroll
        for (int ti = 0; ti < 2; ++ti) {
          const int4 ex = sx[2 * la + ti], ey = sy[2 * lb + tj];
          v[u][tj][ti] = make_double2(0.0, 0.0);
          if (ok[u] && ey.x >= 0 && ex.x >= 0) {
            const int ln = (ex.z <= ey.z) ? (b[u] - ey.y) * ex.z + (a[u] - ex.y) : (a[u] - ex.y) * ey.z + (b[u] - ey.y);
            MS_BCHECK(ex.x < l1.NbX && ey.x < l1.NbY && a[u] >= ex.y && a[u] < ex.y + ex.z && b[u] >= ey.y &&
                      b[u] < ey.y + ey.z && ln >= 0 && ln < ex.z * ey.z);
            const int dj = ey.x - Jmin, di = ex.x - Imin;
            const int64_t off = (dj >= 0 && dj < 4 && di >= 0 && di < 4) ? syoff[dj * 4 + di]
                                                                         : __ldg(l1.yoff + ey.x * l1.NbX + ex.x);
            v[u][tj][ti] = __ldg(reinterpret_cast<const double2*>(l1.ybuf + off + 2 * ln));
          }
        }
      c4a[u] = c4b[u] = p4a[u] = p4b[u] = make_double2(0.0, 0.0);
      if (has_coarse && ok[u]) {
        const int64_t nc4 = (int64_t)(chb + lb) * g.nnx + cha + la;
        const double2* c2 = reinterpret_cast<const double2*>(cd.chi4) + 2 * nc4;
        const double2* p2 = reinterpret_cast<const double2*>(cd.psi4) + 2 * n[u];
        c4a[u] = __ldg(c2);
        c4b[u] = __ldg(c2 + 1);
        if (!pconst) {
          p4a[u] = __ldg(p2);
          p4b[u] = __ldg(p2 + 1);
        }
      }
      mk[u][0] = ok[u] ? mask[n[u]] : 0;
      mk[u][1] = ok[u] ? mask[n[u] + nn] : 0;
      rx[u] = (sc && ok[u]) ? r[n[u]] : 0.0;
      ry[u] = (sc && ok[u]) ? r[n[u] + nn] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      if (!ok[u]) continue;
      double zx = 0.0, zy = 0.0;
#pragma unroll
      for (int tj = 0; tj < 2; ++tj)
#pragma unroll
        for (int ti = 0; ti < 2; ++ti) {
          zx += v[u][tj][ti].x;
          zy += v[u][tj][ti].y;
        }
      if (has_coarse) {
        double cxs = 0.0, cys = 0.0;
        const double ch4[4] = {c4a[u].x, c4a[u].y, c4b[u].x, c4b[u].y};
        double ps4[4] = {p4a[u].x, p4a[u].y, p4b[u].x, p4b[u].y};
        if (pconst) {
#pragma unroll
          for (int c = 0; c < 4; ++c) ps4[c] = __dmul_rn(ch4[c], pv0[c]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (!cok[c]) continue;
          const int I = ci + (c & 1), J = cj + (c >> 1);
          cxs += ps4[c] * cy[c][0];
          cys += ps4[c] * cy[c][1];
          if (cns[c] > 1) {  // rare: extra modes from the per-centre store
            const int ln = (a[u] - (I - 1) * cd.mex) + (b[u] - (J - 1) * cd.mey) * cd.NLx;
            const double* ps = cd.psi + cpo[c] + ln;
            for (int m = 1; m < cns[c]; ++m) {
              const double vv = ch4[c] * __ldg(ps + (int64_t)m * NL);
              cxs += vv * cy[c][2 * m];
              cys += vv * cy[c][2 * m + 1];
            }
          }
          if (cd.enrich) {
            double ex, ey;
            rot_xy(cd, I, J, a[u], b[u], ex, ey);
            cxs += __dmul_rn(ch4[c], ex) * cy[c][2 * kMaxModes];
            cys += __dmul_rn(ch4[c], ey) * cy[c][2 * kMaxModes];
          }
        }
        zx += cxs;
        zy += cys;
      }
      zx = mk[u][0] ? zx : 0.0;
      zy = mk[u][1] ? zy : 0.0;
      z[n[u]] = zx;
      z[n[u] + nn] = zy;
      if (sc) dot += zx * rx[u] + zy * ry[u];
    }
  }
  if (!sc) return;
  const double bs = block_sum(dot, sred);
  double tot;
  if (grid_reduce_dist(bs, partials, (J0 + blockIdx.y) * gridDim.x + blockIdx.x, sc->dist && sc->bitwise,
                       &sc->tickets[2], &tot, sred)) {
    if (threadIdx.x == 0) {
      if (sc->dist)
        sc->part[PART_RZ] = tot;
      else
        fin_beta(sc, tot, beta_hist);
    }
  }
}

static int combine_variant() {
  // A/B knob, read per launch (tests toggle it): 0 = per-node cover lookups, 1 / 2 = staged tables with 1 / 2
  // nodes per thread in flight (config 3 in the PCG loop: 0.139 / 0.133 / 0.201 ms -- two nodes in flight
  // spill at 3 CTAs per SM)
  const char* e = getenv("MS_COMBINE");
  return e ? atoi(e) : 1;
}

int combine_threads() { return kCombineThreads; }

void launch_combine(const Grid& g, const uint8_t* mask, const L1Dev* l1, const CoarseDev* cd,
                    int Nx, int Ny, const double* y0, const double* r, double* z, PcgScalars* sc,
                    double* partials, double* beta_hist, cudaStream_t st, int J0, int J1) {
  L1Dev l1v{};
  CoarseDev cdv{};
  if (l1) l1v = *l1;
  if (cd) cdv = *cd;
  if (J1 < 0) J1 = Ny;
  const int cell_w = g.nx / Nx + 1, cell_h = g.ny / Ny + 1;
  if (l1 && !(cd && cd->vec) && combine_variant() > 0 && cell_w <= kCellMax && cell_h <= kCellMax) {
    if (combine_variant() == 1)
      { k_combine2<1><<<dim3(Nx, J1 - J0), kCombineThreads, 0, st>>>(g, mask, l1v, cdv, cd ? 1 : 0, Nx, Ny, J0, y0, r, z,
                                                                    sc, partials, beta_hist); ms_count_launch(); }
    else
      { k_combine2<2><<<dim3(Nx, J1 - J0), kCombineThreads, 0, st>>>(g, mask, l1v, cdv, cd ? 1 : 0, Nx, Ny, J0, y0, r, z,
                                                                    sc, partials, beta_hist); ms_count_launch(); }
  } else if (cd && cd->vec)
    { k_combine<true><<<dim3(Nx, J1 - J0), kCombineThreads, 0, st>>>(g, mask, l1v, l1 ? 1 : 0, cdv, 1, Nx, Ny, J0,
                                                                   y0, r, z, sc, partials, beta_hist); ms_count_launch(); }
  else
    { k_combine<false><<<dim3(Nx, J1 - J0), kCombineThreads, 0, st>>>(g, mask, l1v, l1 ? 1 : 0, cdv, cd ? 1 : 0,
                                                                    Nx, Ny, J0, y0, r, z, sc, partials, beta_hist); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// K0 = R0 A R0^T.  Persistent CTAs over centres; for each basis vector a of
// centre k: v = Psi_a on closed omega_k, u = A v (matrix-free, elements of
// omega_k only), then K0[b][a] = Psi_b . u for every basis b of the <= 9
// centres whose neighbourhood overlaps omega_k.
__global__ void __launch_bounds__(256)
    k_k0_assemble(Grid g, KeParam ke, const double* __restrict__ E,
                  const uint8_t* __restrict__ mask, CoarseDev cd, double* __restrict__ K0,
                  double* __restrict__ scratch, int k_begin, int k_end) {
  __shared__ double sred[8];
  const int NL = cd.NLx * cd.NLy;
  double* v = scratch + (int64_t)blockIdx.x * 4 * NL;  // [2][NL]
  double* u = v + 2 * NL;                              // [2][NL]
  const int nex = 2 * cd.mex, ney = 2 * cd.mey;
  for (int k = k_begin + blockIdx.x; k < k_end; k += gridDim.x) {
    const int I = k % (cd.Nx - 1) + 1, J = k / (cd.Nx - 1) + 1;
    const int nsel = cd.nsel[k], nb = basis_count(cd, nsel);
    const int ax0 = (I - 1) * cd.mex, by0 = (J - 1) * cd.mey;
    for (int ai = 0; ai < nb; ++ai) {
      for (int ln = threadIdx.x; ln < NL; ln += blockDim.x) {
        const int a = ax0 + ln % cd.NLx, b = by0 + ln / cd.NLx;
        const int64_t n = (int64_t)b * g.nnx + a;
        v[ln] = mask[n] ? basis_value(cd, k, I, J, ai, nsel, a, b, 0) : 0.0;
        v[NL + ln] = mask[n + g.n_nodes] ? basis_value(cd, k, I, J, ai, nsel, a, b, 1) : 0.0;
      }
      __syncthreads();
      for (int ln = threadIdx.x; ln < NL; ln += blockDim.x) {
        const int la = ln % cd.NLx, lb = ln / cd.NLx;
        double qx = 0.0, qy = 0.0;
        const int exs[4] = {la - 1, la, la, la - 1};
        const int eys[4] = {lb - 1, lb - 1, lb, lb};
        const int cn[4] = {2, 3, 0, 1};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int ex = exs[e], ey = eys[e];
          if (ex < 0 || ey < 0 || ex >= nex || ey >= ney) continue;
          const double Ee = E[(int64_t)(by0 + ey) * g.nx + ax0 + ex];
          const int c = cn[e];
          const int l0 = ey * cd.NLx + ex;
          const int lnm[4] = {l0, l0 + 1, l0 + cd.NLx + 1, l0 + cd.NLx};
          double sx = 0.0, sy = 0.0;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const double vx = v[lnm[m]], vy = v[NL + lnm[m]];
            sx += ke.k[c * 8 + m] * vx + ke.k[c * 8 + 4 + m] * vy;
            sy += ke.k[(4 + c) * 8 + m] * vx + ke.k[(4 + c) * 8 + 4 + m] * vy;
          }
          qx += Ee * sx;
          qy += Ee * sy;
        }
        const int64_t n = (int64_t)(by0 + lb) * g.nnx + ax0 + la;
        u[ln] = mask[n] ? qx : 0.0;
        u[NL + ln] = mask[n + g.n_nodes] ? qy : 0.0;
      }
      __syncthreads();
      const int col = basis_row(cd, k, ai, nsel);
      for (int J2 = max(1, J - 1); J2 <= min(cd.Ny - 1, J + 1); ++J2)
        for (int I2 = max(1, I - 1); I2 <= min(cd.Nx - 1, I + 1); ++I2) {
          const int k2 = center_index(cd, I2, J2);
          const int nsel2 = cd.nsel[k2], nb2 = basis_count(cd, nsel2);
          // overlap of the closed neighbourhoods, in omega_k local coordinates
          const int xa = max(ax0, (I2 - 1) * cd.mex), xb = min(ax0 + nex, (I2 + 1) * cd.mex);
          const int ya = max(by0, (J2 - 1) * cd.mey), yb = min(by0 + ney, (J2 + 1) * cd.mey);
          const int wx = xb - xa + 1, wy = yb - ya + 1;
          for (int bi = 0; bi < nb2; ++bi) {
            double acc = 0.0;
            for (int t = threadIdx.x; t < wx * wy; t += blockDim.x) {
              const int a = xa + t % wx, b = ya + t / wx;
              const int ln = (a - ax0) + (b - by0) * cd.NLx;
              acc += basis_value(cd, k2, I2, J2, bi, nsel2, a, b, 0) * u[ln] +
                     basis_value(cd, k2, I2, J2, bi, nsel2, a, b, 1) * u[NL + ln];
            }
            const double s = block_sum(acc, sred);
            if (threadIdx.x == 0) K0[(int64_t)basis_row(cd, k2, bi, nsel2) * cd.N_c + col] = s;
          }
        }
      __syncthreads();
    }
  }
}

void launch_k0_assemble(const Grid& g, const KeParam& ke, const double* E, const uint8_t* mask,
                        const CoarseDev& cd, double* K0, double* scratch, int n_cta,
                        cudaStream_t st, int k_begin, int k_end) {
  if (cd.n_centers == 0) return;
  if (k_end < 0) k_end = cd.n_centers;
  { k_k0_assemble<<<n_cta, 256, 0, st>>>(g, ke, E, mask, cd, K0, scratch, k_begin, k_end); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

__global__ void k_symmetrize(int N, double* A) {
  const int64_t total = (int64_t)N * N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / N), j = (int)(t % N);
    if (j >= i) continue;
    const double v = 0.5 * (A[(int64_t)i * N + j] + A[(int64_t)j * N + i]);
    A[(int64_t)i * N + j] = v;
    A[(int64_t)j * N + i] = v;
  }
}

void launch_symmetrize(int N, double* A, cudaStream_t st) {
  if (N == 0) return;
  { k_symmetrize<<<148 * 4, 256, 0, st>>>(N, A); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

}  // namespace msgpu
