// Matrix-free Q1 elasticity operator and fused PCG vector kernels.
#pragma once

#include "common.cuh"

namespace msgpu {

// Device-resident PCG scalars: the whole loop runs without host round trips;
// the host polls `done` every few iterations.
struct PcgScalars {
  double rz;       // r.z of the current iterate
  double pq;       // p.q
  double alpha, beta;
  double rr;       // ||r||^2
  double bnorm;    // ||b||
  double tol;
  double res;      // ||r||/||b||
  int iter;        // iterations completed
  int maxit;
  int done;
  int converged;
  int first;       // next z.r reduction starts the recurrence (beta = 0)
  int dist;        // multi-rank: reductions leave partials in part[], finalised after allreduce
  int stop_after_beta;  // maxit reached unconverged: finish this iteration's z and beta, then stop
  int bitwise;     // multi-rank: block partials in global slots (bit-identical to one rank)
  double part[4];  // per-rank partial sums: [PART_PQ], [PART_RR], [PART_RZ]
  unsigned int tickets[8];
};

enum { PART_PQ = 0, PART_RR = 1, PART_RZ = 2 };

// scalar recurrences, shared by the single-rank last-CTA path and the
// multi-rank finalize kernel (krylov.py:115-129)
__device__ __forceinline__ void fin_alpha(PcgScalars* sc, double pq, double* alpha_hist) {
  sc->pq = pq;
  sc->alpha = sc->rz / pq;
  if (alpha_hist) alpha_hist[sc->iter] = sc->alpha;
}
__device__ __forceinline__ void fin_res(PcgScalars* sc, double rr, double* res_hist) {
  sc->rr = rr;
  const double res = sqrt(rr) / sc->bnorm;
  sc->res = res;
  sc->iter += 1;
  if (res_hist) res_hist[sc->iter] = res;
  if (res <= sc->tol) {
    sc->converged = 1;
    sc->done = 1;
  } else if (sc->iter >= sc->maxit) {
    // the reference still forms z = M r and beta of the last iteration
    // before leaving the loop (krylov.py:123-127): stop after the beta
    sc->stop_after_beta = 1;
  }
}
__device__ __forceinline__ void fin_beta(PcgScalars* sc, double rz, double* beta_hist) {
  if (sc->first) {
    sc->beta = 0.0;
    sc->first = 0;
  } else {
    sc->beta = rz / sc->rz;
    if (beta_hist) beta_hist[sc->iter - 1] = sc->beta;
  }
  sc->rz = rz;
  if (sc->stop_after_beta) sc->done = 1;
}

// multi-rank: finalize one allreduced partial (kind = PART_*)
void launch_finalize(PcgScalars* sc, int kind, double* hist, cudaStream_t st);
// *out = fixed-order sum of nb partials with `threads` threads (bitwise multi-rank mode)
void launch_reduce_partials(const double* partials, int nb, int threads, double* out, cudaStream_t st);
// the one-rank grid of the fused matvec: global partial slots and block size
int matvec_partial_slots(const Grid& g);
int matvec_threads();

// Element stiffness of the unit modulus Q1 plane-stress element, passed by
// value (kernel parameter space is a broadcast constant bank).
struct KeParam {
  double k[64];
};
struct LapParam {
  double lap[16];  // unit Q1 Laplacian element (assembly.py:133-140)
};

#ifndef MS_MV_TY
#define MS_MV_TY 8
#endif
constexpr int MV_TX = 32;        // nodes per CTA in x
constexpr int MV_TY = MS_MV_TY;  // threads per CTA in y

enum { MV_PLAIN = 0, MV_PCG = 1 };

// b_lo..b_hi: owned node rows (q and p.q there; p refreshed on b_lo-1..b_hi+1)
void launch_matvec(const Grid& g, const KeParam& ke, const double* E, const uint8_t* mask,
                   const double* z, const double* p_old, double* p_new, double* q, int mode,
                   PcgScalars* sc, double* partials, double* alpha_hist, cudaStream_t st,
                   int b_lo = 0, int b_hi = -1);

void launch_pcg_update(int64_t n, double* x, const double* p, double* r, const double* q,
                       PcgScalars* sc, double* partials, double* res_hist, cudaStream_t st);

// rz reduction -> beta (first call of a solve sets rz and beta = 0)
void launch_rz(int64_t n, const double* r, const double* z, PcgScalars* sc, double* partials,
               double* beta_hist, cudaStream_t st);

// sc->bnorm = ||b||, sc->res = 1, history[0] = 1
void launch_init_norm(int64_t n, const double* b, PcgScalars* sc, double* partials,
                      double* res_hist, cudaStream_t st);

void launch_scatter_free(int64_t n_free, const int64_t* free_dofs, const double* src_free,
                         double* dst_full, cudaStream_t st);
void launch_gather_free(int64_t n_free, const int64_t* free_dofs, const double* src_full,
                        double* dst_free, cudaStream_t st);

int reduce_blocks();

}  // namespace msgpu
