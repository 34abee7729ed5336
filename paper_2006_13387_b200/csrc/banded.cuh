// Batched banded SPD machinery: band assembly, Cholesky, sweeps.
#pragma once

#include <cuda.h>

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
  // Twisted (two-sided) factorisation, 0 = plain.  With split m > 0 the
  // unknowns are [T | S | B] = [0, m) [m, m+bw) [m+bw, n): the "top" system
  // (rows [0, m+bw), natural order) is factored at foff, the "bottom" system
  // (rows [m, n) in reversed order) at foffB, each eliminating only its own
  // part; the separator S (bw unknowns; T and B do not couple across it)
  // gets the explicit inverse of its Schur complement at soff.  Both halves'
  // sweeps run concurrently (one warp each), which halves the dependent
  // chain of a solve for the same factor bytes (+bw/n).
  int m;
  int nelim;       // Cholesky: eliminate only the first nelim columns (<= 0: all)
  int64_t foffB;
  int64_t soff;
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
// Systems with 0 < nelim < n are eliminated for their first nelim columns
// only: the remaining bw x bw Schur complement is written (full, row-major)
// to schur + yoff and the last n - nelim columns of Lc / Lr become identity.
void launch_band_potrf(const BandSys* sys, int nsys, int max_bw, double* Lc, double* Lr,
                       int* fail, cudaStream_t st, int ldl = 0, double* schur = nullptr);

// Twisted level-1 build helpers (BandSys.m > 0).  twist_split: from the
// natural column bands (at nat[s].foff) write the top system's band at
// sys[s].foff (the separator block kept) and the bottom system's reversed
// band at sys[s].foffB (its separator block zero).  schur_inverse: Sinv =
// (W_T + flip(W_B))^-1 from the two partial factorisations' Schur windows
// (schur + 2 s max_bw^2, the bottom one max_bw^2 further), written full at
// Sinv + sys[s].soff; one CTA per system.
void launch_twist_split(const BandSys* nat, const BandSys* sys, int nsys, int max_bw, const double* band_nat,
                        double* Lc, cudaStream_t st);
void launch_schur_inverse(const BandSys* sys, int nsys, int max_bw, const double* schur, double* Sinv, int* fail,
                          cudaStream_t st);

// y_s = K_s^{-1} (R_s r) for every system, warp per system.  r is a full
// layout vector; the local solutions land in ybuf[yoff ...], node-interleaved
// (2 ln + c).  nrhs = 2: scalar systems applied to the x and y components in
// one sweep (the factor is read once for both).
// 2-D TMA descriptors of the column / row bands viewed as [columns][S]
// (every system with the same S, starting at a whole column): the padded
// level-1 ring loads 8-column boxes of P = 32 (T+1) words per column, the
// words past S zero-filled by the TMA (out of bounds in the inner dimension).
struct L1Maps {
  CUtensorMap c, r;
  bool valid = false;
};
// encodes a [cols][S] fp64 band at `band` (16-byte aligned, S even); T = ceil(bw / 32)
void make_band_map(CUtensorMap* map, const double* band, int64_t cols, int S, int T);

// Lr == nullptr: one factor copy, the backward sweep by dot products over the
// column band (half the factor bytes).  maps (valid): the padded TMA ring
// (uniform bw, elasticity bands).
// Sinv != nullptr: twisted systems (BandSys.m > 0).  min_bw: narrowest band
// among the systems (the shared-memory ring sweep needs min_bw > 32 (T - 1),
// T = ceil(max_bw / 32); narrower mixes take the register-prefetch sweep).
void launch_l1_solve(const Grid& g, const BandSys* sys, int nsys, int max_bw, int nrhs,
                     const double* Lc, const double* Lr, const double* r, double* ybuf,
                     const int* done, cudaStream_t st, const double* Sinv = nullptr, int min_bw = -1,
                     const L1Maps* maps = nullptr, bool unit = false);
bool ring_sweep_ok(int T, int min_bw);
bool l1_ring_sweeps_enabled();  // false under MS_L1_SWEEP=reg
bool l1_padded_ring_enabled();  // false under MS_L1_PAD=0

// ---------------------------------------------------------------------------
// One warp's banded sweep over a factor read from global memory (L2/L1),
// window in registers.  Column-oriented (axpy) substitution: after w_k is
// known, rows k+1..k+bw receive acc[k+j] -= L[k+j][k] * w_k.  Row r's
// accumulator lives in lane r % 32, register slot (r/32 - current block) --
// slots rotate every 32 steps, so all register indices are compile-time
// constants inside the unrolled 32-step block.  Per step the only cross-lane
// traffic is one shuffle broadcasting w_k from its owner lane; there is no
// shared memory and no warp barrier, so the band columns, prefetched PD steps
// ahead, stay in flight.  The backward sweep is the same recurrence on the
// row band Lr in reversed numbering (row' = n-1-row).  NR right-hand sides
// share each band read (y interleaved: y[row * NR + c]).
constexpr int kPD = 4;

template <int T, int NR, int PD, bool REV>
__device__ __forceinline__ void band_sweep(const double* __restrict__ L, int n, int bw,
                                           double* __restrict__ y, int lane) {
  constexpr int R = T + 1;  // register slots (blocks of 32 rows) per lane
  const int S = bw + 1;
  auto lcol = [&](int k) -> const double* {
    return REV ? L + (int64_t)(n - 1 - k) * S : L + (int64_t)k * S;
  };
  auto yat = [&](int r, int c) -> double* { return y + (int64_t)(REV ? (n - 1 - r) : r) * NR + c; };

  double acc[NR][R], rnext[NR];
#pragma unroll
  for (int c = 0; c < NR; ++c) {
#pragma unroll
    for (int s = 0; s < R - 1; ++s) {
      const int r = 32 * s + lane;
      acc[c][s] = r < n ? *yat(r, c) : 0.0;
    }
    acc[c][R - 1] = 0.0;
    rnext[c] = (32 * (R - 1) + lane < n) ? *yat(32 * (R - 1) + lane, c) : 0.0;
  }

  // prefetch ring: band values of the next PD steps
  double lv[PD][T], dv[PD];
  auto load = [&](int k, int u, double(&l)[T], double& d) {
    const int base = ((lane - u - 1) & 31) + 1;
    const bool ok = k < n;
    const double* col = lcol(ok ? k : 0);
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int j = base + 32 * t;
      l[t] = (ok && j <= bw) ? __ldg(col + j) : 0.0;
    }
    d = ok ? __ldg(col) : 0.0;
  };
#pragma unroll
  for (int u = 0; u < PD; ++u) load(u, u, lv[u], dv[u]);

  for (int k0 = 0; k0 < n; k0 += 32) {
    // rows of block (k0/32 + R-1) enter the window
#pragma unroll
    for (int c = 0; c < NR; ++c) {
      acc[c][R - 1] = rnext[c];
      const int r = k0 + 32 * R + lane;
      rnext[c] = r < n ? *yat(r, c) : 0.0;
    }
    double wout[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) wout[c] = 0.0;
#pragma unroll 1
    for (int u0 = 0; u0 < 32; u0 += PD) {
#pragma unroll
     for (int q = 0; q < PD; ++q) {
      const int u = u0 + q;
      const int k = k0 + u;
      if (k < n) {
        const bool hi = lane <= u;  // row k+base lies in the next block
#pragma unroll
        for (int c = 0; c < NR; ++c) {
          const double wloc = acc[c][0] * dv[q];
          const double wk = __shfl_sync(0xffffffffu, wloc, u);
          if (lane == u) wout[c] = wk;
#pragma unroll
          for (int t = 0; t < T; ++t) {
            const double upd = lv[q][t] * wk;  // zero when k+j is outside the band
            if (hi) {
              if (t + 1 < R) acc[c][t + 1] -= upd;
            } else {
              acc[c][t] -= upd;
            }
          }
        }
        load(k + PD, (u + PD) & 31, lv[q], dv[q]);
      }
     }
    }
#pragma unroll
    for (int c = 0; c < NR; ++c) {
      if (k0 + lane < n) *yat(k0 + lane, c) = wout[c];
      // rotate the register window by one block
#pragma unroll
      for (int s = 0; s < R - 1; ++s) acc[c][s] = acc[c][s + 1];
      acc[c][R - 1] = 0.0;
    }
  }
}



}  // namespace msgpu
