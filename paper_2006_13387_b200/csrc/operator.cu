// Matrix-free Q1 plane-stress operator and fused PCG vector kernels.
//
// Replaces the scipy CSR matvec `op.matrix @ p` (krylov.py:90,114) over the
// assembled free-dof matrix (assembly.py:185-220).  Vectors live in the FULL
// component-grouped layout [x-plane | y-plane] of (nx+1)(ny+1) nodes each;
// constrained dofs are held at exactly zero by a byte mask, which makes the
// full-layout Krylov recurrence identical to the reference's free-dof one.
#include <algorithm>
#include <cstdlib>

#include "operator.cuh"

namespace msgpu {

int reduce_blocks() { return 148 * 8; }

// ---------------------------------------------------------------------------
// q = K p (masked), optionally p = z + beta p_old first, with the p.q
// reduction and alpha = rz / (p.q) fused into the last CTA.
//
// One CTA = 32x32 nodes, 256 threads, 4 vertically stacked nodes per thread.
// p (both components) and E are staged in shared memory with a one-node /
// one-element halo (out-of-domain entries are zero, so no branches).  The
// gather loops over the 4 corner roles c of a node inside its elements: the
// two Ke0 rows of corner c are read once per thread and reused for the
// thread's 4 nodes.
#ifndef MS_MV_NY
#define MS_MV_NY 16
#endif
constexpr int MV_NY = MS_MV_NY;  // nodes per CTA in y
constexpr int MV_RPT = MV_NY / MV_TY;  // nodes per thread

#ifndef MS_MV_MINB
#define MS_MV_MINB 5
#endif
// cp.async (LDGSTS) tile loads instead of register-staged loads: measured
// slower (config 3 matvec 0.099 -> 0.106 ms; 0.118 ms at 6 CTAs/SM), off
#ifndef MS_MV_ASYNC
#define MS_MV_ASYNC 0
#endif
__global__ void __launch_bounds__(MV_TX* MV_TY, MS_MV_MINB)
    k_matvec(Grid g, KeParam ke, const double* __restrict__ E, const uint8_t* __restrict__ mask,
             const double* __restrict__ z, const double* __restrict__ p_old,
             double* __restrict__ p_new, double* __restrict__ q, int mode, PcgScalars* sc,
             double* partials, double* alpha_hist, int b_lo, int b_hi, int tile_y0) {
  if (mode == MV_PCG && sc->done) return;
  __shared__ double sp[2][MV_NY + 2][MV_TX + 2];
  __shared__ double sE[MV_NY + 1][MV_TX + 1];
  __shared__ double sred[MV_TX * MV_TY / 32];
#if MS_MV_ASYNC
  __shared__ double so[2][MV_NY + 2][MV_TX + 2];  // p_old (PCG mode; sp receives z first)
#endif

  const int a0 = blockIdx.x * MV_TX, b0 = (blockIdx.y + tile_y0) * MV_NY;
  const int tid = threadIdx.x;
  const double beta = (mode == MV_PCG) ? sc->beta : 0.0;
  const int64_t nn = g.n_nodes;

  constexpr int kPT = (MV_NY + 2) * (MV_TX + 2);
#if MS_MV_ASYNC
  // Tile loads as asynchronous global->shared copies (cp.async, zero-filled
  // outside the domain): no register staging, every element of the tile in
  // flight at once; then p = z + beta p_old in shared memory.
  {
    constexpr int kET2 = (MV_NY + 1) * (MV_TX + 1);
    for (int t = tid; t < kPT; t += MV_TX * MV_TY) {
      const int ly = t / (MV_TX + 2), lx = t - ly * (MV_TX + 2);
      const int a = a0 + lx - 1, b = b0 + ly - 1;
      const bool ok = a >= 0 && a <= g.nx && b >= 0 && b <= g.ny;
      const int64_t n = ok ? (int64_t)b * g.nnx + a : 0;
      double* dx = (mode == MV_PCG) ? &so[0][ly][lx] : &sp[0][ly][lx];
      double* dy = (mode == MV_PCG) ? &so[1][ly][lx] : &sp[1][ly][lx];
      cp_async8(dx, p_old + n, ok);
      cp_async8(dy, p_old + n + nn, ok);
      if (mode == MV_PCG) {
        cp_async8(&sp[0][ly][lx], z + n, ok);
        cp_async8(&sp[1][ly][lx], z + n + nn, ok);
      }
    }
    for (int t = tid; t < kET2; t += MV_TX * MV_TY) {
      const int ly = t / (MV_TX + 1), lx = t - ly * (MV_TX + 1);
      const int i = a0 + lx - 1, j = b0 + ly - 1;
      const bool ok = i >= 0 && i < g.nx && j >= 0 && j < g.ny;
      cp_async8(&sE[ly][lx], E + (ok ? (int64_t)j * g.nx + i : 0), ok);
    }
    cp_async_wait_all();
    if (mode == MV_PCG) {
      for (int t = tid; t < kPT; t += MV_TX * MV_TY) {  // own elements only: no barrier needed before
        const int ly = t / (MV_TX + 2), lx = t - ly * (MV_TX + 2);
        sp[0][ly][lx] = sp[0][ly][lx] + beta * so[0][ly][lx];
        sp[1][ly][lx] = sp[1][ly][lx] + beta * so[1][ly][lx];
      }
    }
  }
#else
  // Tile loads: every global load of the thread is issued before the first
  // shared-memory store (compile-time trip counts, predicated), so each
  // thread keeps ~25 loads in flight instead of one dependent chain.
  constexpr int kPIt = (kPT + MV_TX * MV_TY - 1) / (MV_TX * MV_TY);
  constexpr int kET = (MV_NY + 1) * (MV_TX + 1);
  constexpr int kEIt = (kET + MV_TX * MV_TY - 1) / (MV_TX * MV_TY);
  {
    double zx[kPIt], zy[kPIt], ox[kPIt], oy[kPIt], ev[kEIt];
#pragma unroll
    for (int it = 0; it < kPIt; ++it) {
      const int t = tid + it * MV_TX * MV_TY;
      const int ly = t / (MV_TX + 2), lx = t - ly * (MV_TX + 2);
      const int a = a0 + lx - 1, b = b0 + ly - 1;
      zx[it] = zy[it] = ox[it] = oy[it] = 0.0;
      if (t < kPT && a >= 0 && a <= g.nx && b >= 0 && b <= g.ny) {
        const int64_t n = (int64_t)b * g.nnx + a;
        ox[it] = __ldg(p_old + n);
        oy[it] = __ldg(p_old + n + nn);
        if (mode == MV_PCG) {
          zx[it] = __ldg(z + n);
          zy[it] = __ldg(z + n + nn);
        }
      }
    }
#pragma unroll
    for (int it = 0; it < kEIt; ++it) {
      const int t = tid + it * MV_TX * MV_TY;
      const int ly = t / (MV_TX + 1), lx = t - ly * (MV_TX + 1);
      const int i = a0 + lx - 1, j = b0 + ly - 1;
      ev[it] = (t < kET && i >= 0 && i < g.nx && j >= 0 && j < g.ny) ? __ldg(E + (int64_t)j * g.nx + i) : 0.0;
    }
#pragma unroll
    for (int it = 0; it < kPIt; ++it) {
      const int t = tid + it * MV_TX * MV_TY;
      if (t < kPT) {
        const int ly = t / (MV_TX + 2), lx = t - ly * (MV_TX + 2);
        sp[0][ly][lx] = (mode == MV_PCG) ? zx[it] + beta * ox[it] : ox[it];
        sp[1][ly][lx] = (mode == MV_PCG) ? zy[it] + beta * oy[it] : oy[it];
      }
    }
#pragma unroll
    for (int it = 0; it < kEIt; ++it) {
      const int t = tid + it * MV_TX * MV_TY;
      if (t < kET) {
        const int ly = t / (MV_TX + 1), lx = t - ly * (MV_TX + 1);
        sE[ly][lx] = ev[it];
      }
    }
  }
#endif
  __syncthreads();

  const int tx = tid % MV_TX, ty = tid / MV_TX;
  const int X = tx + 1;                 // node column in the p tile
  const int Y0 = ty * MV_RPT + 1;       // first node row in the p tile
  double qx[MV_RPT], qy[MV_RPT];
#pragma unroll
  for (int r = 0; r < MV_RPT; ++r) qx[r] = qy[r] = 0.0;
  // corner role c of the node in element E(X+dx, Y+dy)
  const int dxs[4] = {0, -1, -1, 0};
  const int dys[4] = {0, 0, -1, -1};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double kx[8], ky[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      kx[m] = ke.k[c * 8 + m];
      ky[m] = ke.k[(4 + c) * 8 + m];
    }
    const int ex = X + dxs[c];
#pragma unroll
    for (int r = 0; r < MV_RPT; ++r) {
      const int ey = Y0 + r + dys[c];
      const double Ee = sE[ey][ex];
      const double u0 = sp[0][ey][ex], u1 = sp[0][ey][ex + 1], u2 = sp[0][ey + 1][ex + 1],
                   u3 = sp[0][ey + 1][ex];
      const double v0 = sp[1][ey][ex], v1 = sp[1][ey][ex + 1], v2 = sp[1][ey + 1][ex + 1],
                   v3 = sp[1][ey + 1][ex];
      const double sx = kx[0] * u0 + kx[1] * u1 + kx[2] * u2 + kx[3] * u3 + kx[4] * v0 +
                        kx[5] * v1 + kx[6] * v2 + kx[7] * v3;
      const double sy = ky[0] * u0 + ky[1] * u1 + ky[2] * u2 + ky[3] * u3 + ky[4] * v0 +
                        ky[5] * v1 + ky[6] * v2 + ky[7] * v3;
      qx[r] += Ee * sx;
      qy[r] += Ee * sy;
    }
  }
  double dot = 0.0;
  const int a = a0 + tx;
#pragma unroll
  for (int r = 0; r < MV_RPT; ++r) {
    const int b = b0 + ty * MV_RPT + r;
    if (a <= g.nx && b >= b_lo - 1 && b <= b_hi + 1 && b <= g.ny) {
      const int64_t n = (int64_t)b * g.nnx + a;
      MS_BCHECK(a >= 0 && b >= 0 && n < nn);
      const bool own = b >= b_lo && b <= b_hi;
      const double ox = mask[n] ? qx[r] : 0.0;
      const double oy = mask[n + nn] ? qy[r] : 0.0;
      if (own) {
        q[n] = ox;
        q[n + nn] = oy;
      }
      if (mode == MV_PCG) {
        const double px = sp[0][Y0 + r][X], py = sp[1][Y0 + r][X];
        p_new[n] = px;  // owned rows and one halo row on each side
        p_new[n + nn] = py;
        if (own) dot += px * ox + py * oy;
      }
    }
  }
  if (mode != MV_PCG) return;
  const double bs = block_sum(dot, sred);
  double tot;
  if (grid_reduce_dist(bs, partials, (blockIdx.y + tile_y0) * gridDim.x + blockIdx.x, sc->dist && sc->bitwise,
                       &sc->tickets[0], &tot, sred)) {
    if (threadIdx.x == 0) {
      if (sc->dist)
        sc->part[PART_PQ] = tot;
      else
        fin_alpha(sc, tot, alpha_hist);
    }
  }
}

// ---------------------------------------------------------------------------
// PCG-mode matvec with the tile loads of the NEXT tile in flight while the
// current one is computed: each CTA handles kMv2Tiles vertically adjacent
// 32 x 16 tiles; all their z / p_old / E tiles are requested up front as
// asynchronous global -> shared copies (cp.async, zero-filled outside the
// domain) into separate buffers, so the second tile's loads overlap the
// first tile's stencil.  (k_matvec above shows 25% of its stall samples at
// the barrier behind its tile loads and 33% on the loads themselves.)  Node
// -> thread mapping, per-thread arithmetic, the per-tile block sums and their
// partial slots are those of k_matvec: q, p and p.q are bitwise the same.
// One rank only (the strips of a multi-rank run keep k_matvec).
constexpr int kMv2Tiles = 2;
constexpr int kMv2PT = (MV_NY + 2) * (MV_TX + 2);
constexpr int kMv2ET = (MV_NY + 1) * (MV_TX + 1);
constexpr int kMv2Buf = 4 * kMv2PT + kMv2ET + 1;  // z(2) + p_old(2) + E, doubles per tile buffer

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(MV_TX* MV_TY, 4)
    k_matvec2(Grid g, KeParam ke, const double* __restrict__ E, const uint8_t* __restrict__ mask,
              const double* __restrict__ z, const double* __restrict__ p_old, double* __restrict__ p_new,
              double* __restrict__ q, PcgScalars* sc, double* partials, double* alpha_hist, int tiles_y) {
  if (sc->done) return;
  extern __shared__ double mv2[];
  __shared__ double sred[MV_TX * MV_TY / 32];
  __shared__ bool am_last;
  const int tid = threadIdx.x;
  const int a0 = blockIdx.x * MV_TX;
  const double beta = sc->beta;
  const int64_t nn = g.n_nodes;
  typedef double (*PTile)[MV_NY + 2][MV_TX + 2];
  typedef double (*ETile)[MV_TX + 1];
#pragma unroll
  for (int k = 0; k < kMv2Tiles; ++k) {
    const int tyk = blockIdx.y * kMv2Tiles + k;
    if (tyk < tiles_y) {
      double* buf = mv2 + k * kMv2Buf;
      PTile sz = reinterpret_cast<PTile>(buf);
      PTile so = reinterpret_cast<PTile>(buf + 2 * kMv2PT);
      ETile sE = reinterpret_cast<ETile>(buf + 4 * kMv2PT);
      const int b0 = tyk * MV_NY;
      for (int t = tid; t < kMv2PT; t += MV_TX * MV_TY) {
        const int ly = t / (MV_TX + 2), lx = t - ly * (MV_TX + 2);
        const int a = a0 + lx - 1, b = b0 + ly - 1;
        const bool ok = a >= 0 && a <= g.nx && b >= 0 && b <= g.ny;
        const int64_t n = ok ? (int64_t)b * g.nnx + a : 0;
        cp_async8(&so[0][ly][lx], p_old + n, ok);
        cp_async8(&so[1][ly][lx], p_old + n + nn, ok);
        cp_async8(&sz[0][ly][lx], z + n, ok);
        cp_async8(&sz[1][ly][lx], z + n + nn, ok);
      }
      for (int t = tid; t < kMv2ET; t += MV_TX * MV_TY) {
        const int ly = t / (MV_TX + 1), lx = t - ly * (MV_TX + 1);
        const int i = a0 + lx - 1, j = b0 + ly - 1;
        const bool ok = i >= 0 && i < g.nx && j >= 0 && j < g.ny;
        cp_async8(&sE[ly][lx], E + (ok ? (int64_t)j * g.nx + i : 0), ok);
      }
    }
    cp_async_commit();
  }
  const int tx = tid % MV_TX, ty = tid / MV_TX;
  const int X = tx + 1;
  const int Y0 = ty * MV_RPT + 1;
  const int dxs[4] = {0, -1, -1, 0};
  const int dys[4] = {0, 0, -1, -1};
#pragma unroll
  for (int k = 0; k < kMv2Tiles; ++k) {
    const int tyk = blockIdx.y * kMv2Tiles + k;
    if (tyk >= tiles_y) break;  // CTA-uniform
    if (k == 0)
      cp_async_wait_group<kMv2Tiles - 1>();
    else
      cp_async_wait_group<0>();
    double* buf = mv2 + k * kMv2Buf;
    PTile sp = reinterpret_cast<PTile>(buf);  // z in place -> p
    PTile so = reinterpret_cast<PTile>(buf + 2 * kMv2PT);
    ETile sE = reinterpret_cast<ETile>(buf + 4 * kMv2PT);
    // p = z + beta p_old on the entries this thread copied itself (its own copies are complete)
    for (int t = tid; t < kMv2PT; t += MV_TX * MV_TY) {
      const int ly = t / (MV_TX + 2), lx = t - ly * (MV_TX + 2);
      sp[0][ly][lx] = sp[0][ly][lx] + beta * so[0][ly][lx];
      sp[1][ly][lx] = sp[1][ly][lx] + beta * so[1][ly][lx];
    }
    __syncthreads();
    const int b0 = tyk * MV_NY;
    double qx[MV_RPT], qy[MV_RPT];
#pragma unroll
    for (int r = 0; r < MV_RPT; ++r) qx[r] = qy[r] = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double kx[8], ky[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        kx[m] = ke.k[c * 8 + m];
        ky[m] = ke.k[(4 + c) * 8 + m];
      }
      const int ex = X + dxs[c];
#pragma unroll
      for (int r = 0; r < MV_RPT; ++r) {
        const int ey = Y0 + r + dys[c];
        const double Ee = sE[ey][ex];
        const double u0 = sp[0][ey][ex], u1 = sp[0][ey][ex + 1], u2 = sp[0][ey + 1][ex + 1],
                     u3 = sp[0][ey + 1][ex];
        const double v0 = sp[1][ey][ex], v1 = sp[1][ey][ex + 1], v2 = sp[1][ey + 1][ex + 1],
                     v3 = sp[1][ey + 1][ex];
        const double sx = kx[0] * u0 + kx[1] * u1 + kx[2] * u2 + kx[3] * u3 + kx[4] * v0 +
                          kx[5] * v1 + kx[6] * v2 + kx[7] * v3;
        const double sy = ky[0] * u0 + ky[1] * u1 + ky[2] * u2 + ky[3] * u3 + ky[4] * v0 +
                          ky[5] * v1 + ky[6] * v2 + ky[7] * v3;
        qx[r] += Ee * sx;
        qy[r] += Ee * sy;
      }
    }
    double dot = 0.0;
    const int a = a0 + tx;
#pragma unroll
    for (int r = 0; r < MV_RPT; ++r) {
      const int b = b0 + ty * MV_RPT + r;
      if (a <= g.nx && b <= g.ny) {
        const int64_t n = (int64_t)b * g.nnx + a;
        MS_BCHECK(n < nn);
        const double ox = mask[n] ? qx[r] : 0.0;
        const double oy = mask[n + nn] ? qy[r] : 0.0;
        q[n] = ox;
        q[n + nn] = oy;
        const double px = sp[0][Y0 + r][X], py = sp[1][Y0 + r][X];
        p_new[n] = px;
        p_new[n + nn] = py;
        dot += px * ox + py * oy;
      }
    }
    const double bs = block_sum(dot, sred);
    if (tid == 0) partials[blockIdx.x + gridDim.x * tyk] = bs;  // the tile's slot in k_matvec's grid
  }
  // last CTA sums the per-tile partials in k_matvec's order
  if (tid == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(&sc->tickets[0], 1u);
    am_last = (t == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  const double tot = reduce_partials_fixed(partials, gridDim.x * (unsigned)tiles_y, sred);
  if (tid == 0) {
    sc->tickets[0] = 0u;
    fin_alpha(sc, tot, alpha_hist);
  }
}

static int matvec_variant() {
  // A/B knob, read per launch: 0 = k_matvec (register-staged tile loads, default), 1 = k_matvec2 (two tiles
  // per CTA, asynchronous copies of the second tile in flight behind the first tile's stencil).  Measured at
  // config 3 in the PCG loop: 0.096 ms vs 0.103 ms -- the 8-byte cp.async copies (the 2,049-double rows are
  // not 16-byte multiples) cost more issue slots than the overlap returns, so the variant stays opt-in.
  const char* e = getenv("MS_MATVEC");
  return e ? atoi(e) : 0;
}

int matvec_partial_slots(const Grid& g) { return div_up(g.nx + 1, MV_TX) * (g.ny / MV_NY + 1); }
int matvec_threads() { return MV_TX * MV_TY; }

__global__ void k_reduce_partials(const double* __restrict__ partials, int nb, double* out) {
  __shared__ double sh[32];
  const double s = reduce_partials_fixed(partials, (unsigned)nb, sh);
  if (threadIdx.x == 0) *out = s;
}

void launch_reduce_partials(const double* partials, int nb, int threads, double* out, cudaStream_t st) {
  { k_reduce_partials<<<1, threads, 0, st>>>(partials, nb, out); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

void launch_matvec(const Grid& g, const KeParam& ke, const double* E, const uint8_t* mask,
                   const double* z, const double* p_old, double* p_new, double* q, int mode,
                   PcgScalars* sc, double* partials, double* alpha_hist, cudaStream_t st,
                   int b_lo, int b_hi) {
  if (b_hi < 0) b_hi = g.ny;
  if (mode == MV_PCG && b_lo == 0 && b_hi == g.ny && matvec_variant() == 1) {
    const int tiles_y = g.ny / MV_NY + 1;
    const size_t smem = (size_t)kMv2Tiles * kMv2Buf * sizeof(double);
    static bool configured[64] = {};
    int dev = 0;
    MS_CUDA(cudaGetDevice(&dev));
    if (dev >= 64 || !configured[dev]) {
      MS_CUDA(cudaFuncSetAttribute(k_matvec2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if (dev < 64) configured[dev] = true;
    }
    dim3 grid2(div_up(g.nx + 1, MV_TX), div_up(tiles_y, kMv2Tiles));
    { k_matvec2<<<grid2, MV_TX * MV_TY, smem, st>>>(g, ke, E, mask, z, p_old, p_new, q, sc, partials, alpha_hist,
                                                    tiles_y); ms_count_launch(); }
    MS_CUDA(cudaGetLastError());
    return;
  }
  const int ty0 = std::max(0, b_lo - 1) / MV_NY, ty1 = std::min(g.ny, b_hi + 1) / MV_NY;
  dim3 grid(div_up(g.nx + 1, MV_TX), ty1 - ty0 + 1);
  { k_matvec<<<grid, MV_TX * MV_TY, 0, st>>>(g, ke, E, mask, z, p_old, p_new, q, mode, sc, partials,
                                           alpha_hist, b_lo, b_hi, ty0); ms_count_launch(); }
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
    if (threadIdx.x == 0) fin_res(sc, tot, res_hist);
  }
}

void launch_pcg_update(int64_t n, double* x, const double* p, double* r, const double* q,
                       PcgScalars* sc, double* partials, double* res_hist, cudaStream_t st) {
  { k_pcg_update<<<reduce_blocks(), kReduceThreads, 0, st>>>(n, x, p, r, q, sc, partials, res_hist); ms_count_launch(); }
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
    if (threadIdx.x == 0) fin_beta(sc, tot, beta_hist);
  }
}

void launch_rz(int64_t n, const double* r, const double* z, PcgScalars* sc, double* partials,
               double* beta_hist, cudaStream_t st) {
  { k_rz<<<reduce_blocks(), kReduceThreads, 0, st>>>(n, r, z, sc, partials, beta_hist); ms_count_launch(); }
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
  { k_init_norm<<<reduce_blocks(), kReduceThreads, 0, st>>>(n, b, sc, partials, res_hist); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
__global__ void k_finalize(PcgScalars* sc, int kind, double* hist) {
  // the partial of an iteration already marked done was never produced
  if (kind != PART_RR && sc->done) return;
  if (kind == PART_RR && sc->done) return;
  const double v = sc->part[kind];
  if (kind == PART_PQ)
    fin_alpha(sc, v, hist);
  else if (kind == PART_RR)
    fin_res(sc, v, hist);
  else
    fin_beta(sc, v, hist);
}

void launch_finalize(PcgScalars* sc, int kind, double* hist, cudaStream_t st) {
  { k_finalize<<<1, 1, 0, st>>>(sc, kind, hist); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

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
  { k_scatter_free<<<reduce_blocks(), 256, 0, st>>>(n_free, free_dofs, src_free, dst_full); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}
void launch_gather_free(int64_t n_free, const int64_t* free_dofs, const double* src_full,
                        double* dst_free, cudaStream_t st) {
  { k_gather_free<<<reduce_blocks(), 256, 0, st>>>(n_free, free_dofs, src_full, dst_free); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

}  // namespace msgpu
