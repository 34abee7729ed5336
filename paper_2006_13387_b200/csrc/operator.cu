// Matrix-free Q1 plane-stress operator and fused PCG vector kernels.
//
// Replaces the scipy CSR matvec `op.matrix @ p` (krylov.py:90,114) over the
// assembled free-dof matrix (assembly.py:185-220).  Vectors live in the FULL
// component-grouped layout [x-plane | y-plane] of (nx+1)(ny+1) nodes each;
// constrained dofs are held at exactly zero by a byte mask, which makes the
// full-layout Krylov recurrence identical to the reference's free-dof one.
#include "operator.cuh"

namespace msgpu {

int reduce_blocks() { return 148 * 8; }

// ---------------------------------------------------------------------------
// q = K p (masked), optionally p = z + beta p_old first, with the p.q
// reduction and alpha = rz / (p.q) fused into the last CTA.
//
// One CTA = 32x8 nodes, one node per thread.  p (both components) and E are
// staged in shared memory with a one-node / one-element halo; out-of-domain
// entries are zero so the 4-element gather needs no branches.
__global__ void __launch_bounds__(MV_TX* MV_TY)
    k_matvec(Grid g, KeParam ke, const double* __restrict__ E, const uint8_t* __restrict__ mask,
             const double* __restrict__ z, const double* __restrict__ p_old,
             double* __restrict__ p_new, double* __restrict__ q, int mode, PcgScalars* sc,
             double* partials, double* alpha_hist) {
  if (mode == MV_PCG && sc->done) return;
  __shared__ double sp[2][MV_TY + 2][MV_TX + 2];
  __shared__ double sE[MV_TY + 1][MV_TX + 1];
  __shared__ double sred[MV_TX * MV_TY / 32];

  const int a0 = blockIdx.x * MV_TX, b0 = blockIdx.y * MV_TY;
  const int tid = threadIdx.x;
  const double beta = (mode == MV_PCG) ? sc->beta : 0.0;
  const int64_t nn = g.n_nodes;

  // stage p (nodes a0-1 .. a0+MV_TX, b0-1 .. b0+MV_TY)
  for (int t = tid; t < (MV_TY + 2) * (MV_TX + 2); t += blockDim.x) {
    const int ly = t / (MV_TX + 2), lx = t % (MV_TX + 2);
    const int a = a0 + lx - 1, b = b0 + ly - 1;
    double px = 0.0, py = 0.0;
    if (a >= 0 && a <= g.nx && b >= 0 && b <= g.ny) {
      const int64_t n = (int64_t)b * g.nnx + a;
      if (mode == MV_PCG) {
        px = z[n] + beta * p_old[n];
        py = z[n + nn] + beta * p_old[n + nn];
      } else {
        px = p_old[n];
        py = p_old[n + nn];
      }
    }
    sp[0][ly][lx] = px;
    sp[1][ly][lx] = py;
  }
  // stage E (elements a0-1 .. a0+MV_TX-1, b0-1 .. b0+MV_TY-1)
  for (int t = tid; t < (MV_TY + 1) * (MV_TX + 1); t += blockDim.x) {
    const int ly = t / (MV_TX + 1), lx = t % (MV_TX + 1);
    const int i = a0 + lx - 1, j = b0 + ly - 1;
    sE[ly][lx] = (i >= 0 && i < g.nx && j >= 0 && j < g.ny) ? E[(int64_t)j * g.nx + i] : 0.0;
  }
  __syncthreads();

  const int tx = tid % MV_TX, ty = tid / MV_TX;
  const int a = a0 + tx, b = b0 + ty;
  double dot = 0.0;
  if (a <= g.nx && b <= g.ny) {
    // elements around the node by their lower-left p-tile corner, with the
    // node's corner number inside each (0:(i,j) 1:(i+1,j) 2:(i+1,j+1) 3:(i,j+1))
    const int ex[4] = {tx, tx + 1, tx + 1, tx};
    const int ey[4] = {ty, ty, ty + 1, ty + 1};
    const int cn[4] = {2, 3, 0, 1};
    double qx = 0.0, qy = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double Ee = sE[ey[e]][ex[e]];
      const int c = cn[e];
      const double ux[4] = {sp[0][ey[e]][ex[e]], sp[0][ey[e]][ex[e] + 1], sp[0][ey[e] + 1][ex[e] + 1],
                            sp[0][ey[e] + 1][ex[e]]};
      const double uy[4] = {sp[1][ey[e]][ex[e]], sp[1][ey[e]][ex[e] + 1], sp[1][ey[e] + 1][ex[e] + 1],
                            sp[1][ey[e] + 1][ex[e]]};
      double sx = 0.0, sy = 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        sx += ke.k[c * 8 + m] * ux[m] + ke.k[c * 8 + 4 + m] * uy[m];
        sy += ke.k[(4 + c) * 8 + m] * ux[m] + ke.k[(4 + c) * 8 + 4 + m] * uy[m];
      }
      qx += Ee * sx;
      qy += Ee * sy;
    }
    const int64_t n = (int64_t)b * g.nnx + a;
    qx = mask[n] ? qx : 0.0;
    qy = mask[n + nn] ? qy : 0.0;
    q[n] = qx;
    q[n + nn] = qy;
    if (mode == MV_PCG) {
      const double px = sp[0][ty + 1][tx + 1], py = sp[1][ty + 1][tx + 1];
      p_new[n] = px;
      p_new[n + nn] = py;
      dot = px * qx + py * qy;
    }
  }
  if (mode != MV_PCG) return;
  const double bs = block_sum(dot, sred);
  double tot;
  if (grid_reduce_last(bs, partials, &sc->tickets[0], &tot, sred)) {
    if (threadIdx.x == 0) {
      sc->pq = tot;
      sc->alpha = sc->rz / tot;
      if (alpha_hist) alpha_hist[sc->iter] = sc->alpha;
    }
  }
}

void launch_matvec(const Grid& g, const KeParam& ke, const double* E, const uint8_t* mask,
                   const double* z, const double* p_old, double* p_new, double* q, int mode,
                   PcgScalars* sc, double* partials, double* alpha_hist, cudaStream_t st) {
  dim3 grid(div_up(g.nx + 1, MV_TX), div_up(g.ny + 1, MV_TY));
  k_matvec<<<grid, MV_TX * MV_TY, 0, st>>>(g, ke, E, mask, z, p_old, p_new, q, mode, sc, partials,
                                           alpha_hist);
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// x += alpha p ; r -= alpha q ; ||r||^2 -> residual, convergence flag.
__global__ void __launch_bounds__(kReduceThreads)
    k_pcg_update(int64_t n, double* __restrict__ x, const double* __restrict__ p,
                 double* __restrict__ r, const double* __restrict__ q, PcgScalars* sc,
                 double* partials, double* res_hist) {
  if (sc->done) return;
  __shared__ double sred[kReduceThreads / 32];
  const double alpha = sc->alpha;
  double acc = 0.0;
  const int64_t n2 = n >> 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  const double2* p2 = reinterpret_cast<const double2*>(p);
  const double2* q2 = reinterpret_cast<const double2*>(q);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 xv = x2[i], pv = p2[i], rv = r2[i], qv = q2[i];
    xv.x += alpha * pv.x;
    xv.y += alpha * pv.y;
    rv.x -= alpha * qv.x;
    rv.y -= alpha * qv.y;
    x2[i] = xv;
    r2[i] = rv;
    acc += rv.x * rv.x + rv.y * rv.y;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    x[n - 1] += alpha * p[n - 1];
    r[n - 1] -= alpha * q[n - 1];
    acc += r[n - 1] * r[n - 1];
  }
  const double bs = block_sum(acc, sred);
  double tot;
  if (grid_reduce_last(bs, partials, &sc->tickets[1], &tot, sred)) {
    if (threadIdx.x == 0) {
      sc->rr = tot;
      const double res = sqrt(tot) / sc->bnorm;
      sc->res = res;
      sc->iter += 1;
      if (res_hist) res_hist[sc->iter] = res;
      if (res <= sc->tol) {
        sc->converged = 1;
        sc->done = 1;
      } else if (sc->iter >= sc->maxit) {
        sc->done = 1;
      }
    }
  }
}

void launch_pcg_update(int64_t n, double* x, const double* p, double* r, const double* q,
                       PcgScalars* sc, double* partials, double* res_hist, cudaStream_t st) {
  k_pcg_update<<<reduce_blocks(), kReduceThreads, 0, st>>>(n, x, p, r, q, sc, partials, res_hist);
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kReduceThreads)
    k_rz(int64_t n, const double* __restrict__ r, const double* __restrict__ z, PcgScalars* sc,
         double* partials, double* beta_hist) {
  if (sc->done) return;
  __shared__ double sred[kReduceThreads / 32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    acc += r[i] * z[i];
  const double bs = block_sum(acc, sred);
  double tot;
  if (grid_reduce_last(bs, partials, &sc->tickets[2], &tot, sred)) {
    if (threadIdx.x == 0) {
      if (sc->first) {
        sc->beta = 0.0;
        sc->first = 0;
      } else {
        sc->beta = tot / sc->rz;
        if (beta_hist) beta_hist[sc->iter - 1] = sc->beta;
      }
      sc->rz = tot;
    }
  }
}

void launch_rz(int64_t n, const double* r, const double* z, PcgScalars* sc, double* partials,
               double* beta_hist, cudaStream_t st) {
  k_rz<<<reduce_blocks(), kReduceThreads, 0, st>>>(n, r, z, sc, partials, beta_hist);
  MS_CUDA(cudaGetLastError());
}

__global__ void __launch_bounds__(kReduceThreads)
    k_init_norm(int64_t n, const double* __restrict__ b, PcgScalars* sc, double* partials,
                double* res_hist) {
  __shared__ double sred[kReduceThreads / 32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    acc += b[i] * b[i];
  const double bs = block_sum(acc, sred);
  double tot;
  if (grid_reduce_last(bs, partials, &sc->tickets[3], &tot, sred)) {
    if (threadIdx.x == 0) {
      sc->bnorm = sqrt(tot);
      sc->res = 1.0;
      if (res_hist) res_hist[0] = 1.0;
      if (tot == 0.0) {
        sc->converged = 1;
        sc->done = 1;
      }
    }
  }
}

void launch_init_norm(int64_t n, const double* b, PcgScalars* sc, double* partials,
                      double* res_hist, cudaStream_t st) {
  k_init_norm<<<reduce_blocks(), kReduceThreads, 0, st>>>(n, b, sc, partials, res_hist);
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
__global__ void k_scatter_free(int64_t n_free, const int64_t* __restrict__ free_dofs,
                               const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_free;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[free_dofs[i]] = src[i];
}
__global__ void k_gather_free(int64_t n_free, const int64_t* __restrict__ free_dofs,
                              const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_free;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[free_dofs[i]];
}

void launch_scatter_free(int64_t n_free, const int64_t* free_dofs, const double* src_free,
                         double* dst_full, cudaStream_t st) {
  k_scatter_free<<<reduce_blocks(), 256, 0, st>>>(n_free, free_dofs, src_free, dst_full);
  MS_CUDA(cudaGetLastError());
}
void launch_gather_free(int64_t n_free, const int64_t* free_dofs, const double* src_full,
                        double* dst_free, cudaStream_t st) {
  k_gather_free<<<reduce_blocks(), 256, 0, st>>>(n_free, free_dofs, src_full, dst_free);
  MS_CUDA(cudaGetLastError());
}

}  // namespace msgpu
