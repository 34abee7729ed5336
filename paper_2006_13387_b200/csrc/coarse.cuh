// Coarse level (spectral EH+Rot space) and the preconditioner combine step.
#pragma once

#include "banded.cuh"
#include "dense.cuh"
#include "common.cuh"
#include "operator.cuh"

namespace msgpu {

// Level-1 geometry for the node-centric combine: subdomain (I, J) has kept
// node range [xlo[I], xlo[I]+xlen[I]-1] x [ylo[J], ...]; the covering lists
// give, per node column a (row b), up to 4 block indices I (J), ascending,
// -1 padded.  Subdomain s = J*NbX + I.
struct L1Dev {
  int NbX, NbY;
  const int* xlo;       // per block column I: first kept node, kept count
  const int* xlen;
  const int* ylo;       // per block row J
  const int* ylen;
  const int64_t* yoff;  // per subdomain: offset of its local vector in ybuf
  const int* xcov;      // (nx+1) * 4
  const int* ycov;      // (ny+1) * 4
  const double* ybuf;
};

// Coarse space on device.  Centre k = (I, J), 1 <= I < Nx, 1 <= J < Ny,
// k = (J-1)*(Nx-1) + (I-1) (the reference's neighbourhood order, grid.py:132).
struct CoarseDev {
  int Nx, Ny, mex, mey;
  int NLx, NLy;           // closed-omega nodes per axis: 2*mex+1, 2*mey+1
  int n_centers;
  int enrich;
  int vec;                // 1: elasticity basis (EE): one row per mode, psi has x and y parts
  int N_c;
  int roff;               // first rotation row = 2 * sum(nsel)
  double h;
  const int* nsel;        // per centre
  const int* hoff;        // per centre: first row (prefix sum of 2*nsel, or nsel if vec)
  const int64_t* psioff;  // per centre: offset into psi (nsel * NL values, 2 * nsel * NL if vec)
  const double* psi;      // selected eigenvectors on closed omega, lexicographic
                          // (vec: per mode the x-part then the y-part)
  const double* chi;      // per centre: partition of unity on closed omega (NL values)
  // node-major tables over the coarse cell containing each node: the 4 corner
  // centres (ci + (c&1), cj + (c>>1)), c = 0..3, J-major; zero where invalid
  const double* chi4;     // [n_nodes][4] chi of the corner centres
  const double* psi4;     // [n_nodes][4] chi * psi (mode 0) of the corner centres
  // per centre: the value of mode 0 when it is the constant vector (pure
  // Neumann neighbourhoods: the locked exact kernel of the heat pencil), NaN
  // otherwise.  A cell whose corner centres all have one skips the psi4
  // records: psi4 = chi4 * value, the product the table holds (nullptr: off)
  const double* psi0c;
  // per coarse cell: the cell whose chi4 records are bitwise identical to
  // this one's (itself when none of its class is).  On a uniform coarse grid
  // with exactly representable h every interior cell shares one 32 KB block
  // of records (likewise each edge class), which then lives in L2: the cell
  // kernels read chi4 through this map and move no DRAM bytes for it
  // (nullptr: off)
  const int* chi_src;
  double* rpart;          // [Nx*Ny cells][4][2*kMaxModes+1] restriction partials
};

constexpr int kMaxModes = 6;
constexpr int kSlots = 2 * kMaxModes + 1;  // heat x/y per mode + rotation

// node-major chi4 / psi4 from the per-centre tables
void launch_node_tables(const Grid& g, const CoarseDev& cd, double* chi4, double* psi4,
                        cudaStream_t st);
// chi_src[cell] = the class representative (interior / edge / corner cell, 9 classes) when this
// cell's chi4 block equals it bit for bit, else the cell itself
void launch_chi_dedup(const Grid& g, const CoarseDev& cd, int* chi_src, cudaStream_t st);
// psi0c[k] = the constant value of centre k's mode 0, NaN when it is not constant
void launch_psi0_const(const CoarseDev& cd, double* psi0c, cudaStream_t st);

// fused x += alpha p, r -= alpha q, ||r||^2 -> convergence, and restriction
// partial sums per coarse cell; then f0 = sum of the 4 cell partials per centre
// cells of coarse block rows [J0, J1) (the caller's strip)
// block sizes of the fused update + restriction and of the combine (their
// one-rank finishing blocks reduce the dot-product partials with them)
int update_restrict_threads(const CoarseDev& cd);
int combine_threads();
void launch_update_restrict(const Grid& g, int J0, int J1, double* x, const double* p, double* r,
                            const double* q, const CoarseDev& cd, PcgScalars* sc,
                            double* partials, double* res_hist, cudaStream_t st);
void launch_restrict_cells(const Grid& g, int J0, int J1, const CoarseDev& cd, const double* r,
                           const int* done, cudaStream_t st);
void launch_restrict_reduce(const CoarseDev& cd, double* f0, const int* done, cudaStream_t st,
                            int k_begin = 0, int k_end = -1);

// chi table, bit-identical to the reference's PoU (grid.py:172-207)
void launch_pou_table(const Grid& g, const CoarseDev& cd, double* chi, cudaStream_t st);


// z = sum_s R_s^T y_s (level-1, J-major order) + R0^T y0 (if cd) ; masked;
// optionally r.z -> beta (PCG mode when sc != nullptr).
void launch_combine(const Grid& g, const uint8_t* mask, const L1Dev* l1, const CoarseDev* cd,
                    int Nx, int Ny, const double* y0, const double* r, double* z, PcgScalars* sc,
                    double* partials, double* beta_hist, cudaStream_t st, int J0 = 0, int J1 = -1);

// K0 = R0 A R0^T (dense row-major N_c x N_c), symmetrised (coarse.py:161-168)
void launch_k0_assemble(const Grid& g, const KeParam& ke, const double* E, const uint8_t* mask,
                        const CoarseDev& cd, double* K0, double* scratch, int n_cta,
                        cudaStream_t st, int k_begin = 0, int k_end = -1);
void launch_symmetrize(int N, double* A, cudaStream_t st);

}  // namespace msgpu
