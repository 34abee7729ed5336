// Batched banded SPD machinery: band assembly, Cholesky, sweeps.
#pragma once

#include "common.cuh"
#include "operator.cuh"

namespace msgpu {

// One banded SPD system.  Unknowns are node-interleaved (2*ln + c for
// elasticity, ln for scalar problems) over a rectangle of nodes numbered
// fast-axis first; the lower band is stored twice:
//   Lc[foff + k*(bw+1) + j] = L[k+j][k]   (column band, forward sweep)
//   Lr[foff + k*(bw+1) + j] = L[k][k-j]   (row band,    backward sweep)
// with the diagonal slot j=0 holding 1/L[k][k].
struct BandSys {
  int a0, b0;      // lower-left kept node (global node coordinates)
  int w, hgt;      // kept nodes along x / y
  int fastx;       // 1: x is the fast (short) axis
  int ncomp;       // 2 elasticity, 1 heat
  int nrhs;        // right-hand sides per solve: 1, or 2 for the heat level-1 (x and y blocks)
  int n;           // unknowns
  int bw;          // lower bandwidth
  int64_t foff;    // offset into Lc / Lr
  int64_t yoff;    // offset of the local vector in the solution buffer
};

__host__ __device__ inline int band_fast_len(const BandSys& s) { return s.fastx ? s.w : s.hgt; }

// local node index of global node (a, b) inside system s (no bounds check)
__host__ __device__ inline int band_local_node(const BandSys& s, int a, int b) {
  return s.fastx ? (b - s.b0) * s.w + (a - s.a0) : (a - s.a0) * s.hgt + (b - s.b0);
}
__host__ __device__ inline void band_node_of(const BandSys& s, int ln, int& a, int& b) {
  if (s.fastx) {
    a = s.a0 + ln % s.w;
    b = s.b0 + ln / s.w;
  } else {
    a = s.a0 + ln / s.hgt;
    b = s.b0 + ln % s.hgt;
  }
}

void band_setup(BandSys& s, int a0, int a1, int b0, int b1, int ncomp);

// Level-1 elasticity band: K_i = A[idx][:, idx] of the global operator
// (schwarz.py:97-109) with constrained dofs turned into identity rows.
void launch_l1_assemble(const Grid& g, const KeParam& ke, const double* E, const uint8_t* mask,
                        const BandSys* sys, int nsys, double* Lc, cudaStream_t st);

// Heat level-1 band (HH variants, schwarz.py:112-140): the E-weighted
// diffusion matrix restricted to the subdomain's kept nodes, constrained nodes
// (x-dof mask 0) as identity rows.  Elements of the whole mesh contribute.
void launch_l1_heat_assemble(const Grid& g, const double* lap, const double* E, const uint8_t* mask,
                             const BandSys* sys, int nsys, double* Lc, cudaStream_t st);

// fail = 1 unless every node is either fully constrained or fully free
void launch_whole_node_check(const Grid& g, const uint8_t* mask, int* fail, cudaStream_t st);

// In-place banded Cholesky of every system: Lc holds A's lower band on
// entry, L on exit (diag slot = 1/L_kk); Lr receives the row band.
// *fail gets (system index + 1) of a non-positive pivot, else stays 0.
void launch_band_potrf(const BandSys* sys, int nsys, int max_bw, double* Lc, double* Lr,
                       int* fail, cudaStream_t st, int ldl = 0);

// y_s = K_s^{-1} (R_s r) for every system, warp per system.  r is a full
// layout vector; the local solutions land in ybuf[yoff ...], node-interleaved
// (2 ln + c).  nrhs = 2: scalar systems applied to the x and y components in
// one sweep (the factor is read once for both).
void launch_l1_solve(const Grid& g, const BandSys* sys, int nsys, int max_bw, int nrhs,
                     const double* Lc, const double* Lr, const double* r, double* ybuf,
                     const int* done, cudaStream_t st);

}  // namespace msgpu
