// Topology-optimisation caller kernels: density filter,
// SIMP modulus, compliance sensitivity, optimality-criteria update.
#pragma once

#include "common.cuh"
#include "operator.cuh"

namespace msgpu {

// Row-normalised cone filter W (DensityFilter, assembly.py:290-336).  W has the
// same stencil at every element, truncated at the mesh edges; entry (e, k) =
// inv_rowsum[e] * w[o] for k = e + (dj nx + di).  Offsets are stored in
// descending (dj, di) order, the order of the reference's CSR rows.
struct FilterDev {
  int nx, ny, noff;
  const int2* off;          // (di, dj), descending column order
  const double* w;          // cone weight per offset
  const double* inv_rowsum;  // per element: 1 / sum of its (truncated) row
};

// y = W x (bit-exact with the reference's CSR matvec: sequential products and
// sums over the row in stored order, no contraction)
void launch_filter_apply(const FilterDev& f, const double* x, double* y, cudaStream_t st);
// y = W^T v (the reference's CSC matvec order: rows e ascending)
void launch_filter_adjoint(const FilterDev& f, const double* v, double* y, cudaStream_t st);

// E = E_min + clip(rho_f, 0, 1)^p (E_max - E_min); *bad = 1 if rho_f leaves
// [-1e-12, 1 + 1e-12] (simp_modulus, assembly.py:280-287)
void launch_simp(int64_t n, const double* rho_f, double p, double E_min, double E_max, double* E,
                 int* bad, cudaStream_t st);

// sens_e = -p clip(rho_f)^(p-1) (E_max - E_min) u_e^T k0 u_e (topopt.py:59-70)
void launch_compliance_sens(const Grid& g, const KeParam& ke, const double* u_full,
                            const double* rho_f, double p, double E_min, double E_max, double* sens,
                            cudaStream_t st);

// deterministic dot over n entries into *out (device); partials >= kDotBlocks
constexpr int kDotBlocks = 4 * 148;
void launch_dot(int64_t n, const double* a, const double* b, double* out, double* partials,
                unsigned int* ticket, cudaStream_t st);

// optimality-criteria bisection (oc_update, topopt.py:73-107) as a device state
// machine: each k_oc_eval launch measures the candidate volume(s) for the
// current multiplier(s) and its last block advances the bracket / bisection.
struct OcState {
  double lo, hi;      // multiplier bracket
  double v_star, move, damping;
  int phase;          // 0 bracketing, 1 bisecting, 2 done, 3 bracket failed
  int count;          // evaluations in the current phase
  int evals;          // total candidate-volume evaluations
  int pad;
};
void launch_oc_init(OcState* s, double v_star, double move, double damping, cudaStream_t st);
// wv = W^T volumes (or volumes when unfiltered): measure(lam) = wv . candidate(lam)
void launch_oc_eval(int64_t n, const double* rho, const double* dg, const double* vol,
                    const double* wv, OcState* s, double* partials, unsigned int* ticket,
                    cudaStream_t st);
void launch_oc_final(int64_t n, const double* rho, const double* dg, const double* vol,
                     const OcState* s, double* rho_new, cudaStream_t st);

}  // namespace msgpu
