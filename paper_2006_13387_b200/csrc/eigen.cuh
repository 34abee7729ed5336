// Batched local heat eigensolves for the spectral coarse space.
#pragma once

#include "banded.cuh"
#include "common.cuh"

namespace msgpu {

constexpr int kEigBlock = 16;  // subspace block size p
constexpr int kNeig = 7;       // eigenpairs kept per centre: min(n_max+1, dim), n_max = 6

struct HeatParam {
  double lap[16];  // unit Q1 Laplacian element (assembly.py:133-140)
  double mel[16];  // Q1 mass element for side h (assembly.py:143-147)
};

struct EigBatch {
  int Nx, mex, mey;    // centre (I, J) geometry
  int k0, nk;          // first centre and number of centres in this batch
  const BandSys* sys;  // heat band systems of the batch (index = centre - k0)
  const double* Lc;
  const double* Lr;
  double* work;        // per centre: 2 * p * NL doubles
  double* evals;       // global: centre * kNeig (ascending)
  double* evecs;       // batch: (centre - k0) * kNeig * NL, band order, M-orthonormal
  int* passes;         // global: per centre
  int* neumann;        // global: per centre (1 if no heat-Dirichlet node in omega)
  int n_max;           // selection parameters, used by the stopping rule
  double gap;
  int fixed;
  double lam_floor;  // absolute convergence floor for Ritz values
};

// B = K_H + sigma M_H in band form (Dirichlet nodes -> identity rows)
void launch_heat_assemble(const Grid& g, const double* E, const uint8_t* hdir,
                          const HeatParam& hp, double sigma, const BandSys* sys, int nsys,
                          double* Lc, cudaStream_t st, const double* sigma_per_sys = nullptr);

// shift-invert block subspace iteration with Jacobi Rayleigh-Ritz, one CTA per centre
void launch_subspace(const Grid& g, const double* E, const uint8_t* hdir, const HeatParam& hp,
                     const EigBatch& b, int max_pass, double tol, cudaStream_t st);

// randomized snapshot eigensolver (EH+Rot;Rand): F = forcings of the batch,
// [centre][ns][NL] lexicographic closed-neighbourhood nodes (zero rows at
// Dirichlet nodes); factors of K + sigma_k M with the reference's shift
void launch_randomized(const Grid& g, const double* E, const uint8_t* hdir, const HeatParam& hp,
                       const EigBatch& b, const double* F, int ns, cudaStream_t st);

// per-centre reference shift sigma_k = 1e-8 tr(K_free)/n_free (spectral.py:133)
void launch_rand_sigma(const Grid& g, const double* E, const uint8_t* hdir, const HeatParam& hp,
                       const BandSys* sys, int nsys, double* sigma, cudaStream_t st);

// ---- elasticity eigenproblems (EE, EE;Rand; spectral.py:63-100 kind 'elasticity') ----
// Unknowns node-interleaved (2 ln + c) in the band order of the closed
// neighbourhood; evecs/work of an EigBatch then hold 2*NL values per vector.
struct ElastParam {
  double ke[64];   // unit-modulus Q1 plane-stress element, [comp*4 + corner] ordering
  double mel[16];  // Q1 mass element for side h (block-diagonal per component)
};

// B = K_E + sigma M_E in band form (whole-node Dirichlet -> identity rows)
void launch_el_assemble(const Grid& g, const double* E, const uint8_t* hdir, const ElastParam& ep,
                        double sigma, const BandSys* sys, int nsys, double* Lc, cudaStream_t st,
                        const double* sigma_per_sys = nullptr);

// shift-invert block subspace iteration (rigid-body modes locked on Neumann
// neighbourhoods); work holds (2p + 6) * n doubles per centre
void launch_subspace_el(const Grid& g, const double* E, const uint8_t* hdir, const ElastParam& ep,
                        const EigBatch& b, int max_bw, int max_pass, double tol, cudaStream_t st);

// randomized snapshot solver with the rigid-body modes as kernel candidates;
// F = [centre][ns][2 NL] (x-plane then y-plane, lexicographic, zero at Dirichlet)
void launch_randomized_el(const Grid& g, const double* E, const uint8_t* hdir, const ElastParam& ep,
                          const EigBatch& b, int max_bw, const double* F, int ns, cudaStream_t st);

// sigma_k = 1e-8 tr(K_free) / n_free (spectral.py:133), elasticity pencil
void launch_rand_sigma_el(const Grid& g, const double* E, const uint8_t* hdir, const ElastParam& ep,
                          const BandSys* sys, int nsys, double* sigma, cudaStream_t st);

// selected vectors -> psi store: per mode the x-part then the y-part over the
// closed neighbourhood (lexicographic), sign-normalised
void launch_compact_psi_el(const EigBatch& b, int NLx, const int* nsel, const int64_t* psioff,
                           double* psi, cudaStream_t st);

// block size of the randomized solvers for `ns` snapshots (16, or 32 above 13);
// their work buffers hold (2 B [+ 6 for elasticity]) * n doubles per centre
int randomized_block(int ns);

// gap / fixed selection on device (spectral.py:161-186)
void launch_select(int n_centers, const double* evals, int n_max, double threshold, int fixed,
                   int* nsel, cudaStream_t st);

// copy the selected vectors of a batch into the compact psi store (lexicographic
// closed-omega node order), sign-normalised: largest-|.| entry positive.
void launch_compact_psi(const EigBatch& b, int NLx, const int* nsel, const int64_t* psioff,
                        double* psi, cudaStream_t st);

}  // namespace msgpu
