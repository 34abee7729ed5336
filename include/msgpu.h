/*
 * msgpu.h — C ABI of the B200-native two-level spectral Schwarz PCG solve path.
 *
 * The reference (mselast, pure Python) has no FFI; its drop-in boundary is the
 * duck-typed Python API listed in SURVEY.md §8(b).  Each entry point below
 * replaces one of those reference interfaces (file:line into
 * /root/reference/pkg/src/mselast/); paper_2006_13387_b200/ binds them with
 * ctypes and re-exposes the reference's Python names on top.
 *
 * Conventions
 *  - status codes: MS_OK (0) or a negative MS_E_* value; the message of the
 *    last failure on a context is returned by ms_last_error().  The Python
 *    layer maps MS_E_INVALID/MS_E_NOT_SPD to ValueError exactly where the
 *    reference raises ValueError (krylov.py:88-98, schwarz.py:77-78,
 *    coarse.py:142-147).
 *  - vectors crossing the ABI are FREE-dof vectors (length n_free) in the
 *    reference ordering: sorted free ids of the component-grouped full dof
 *    vector (assembly.py:150-205).  Pointers may be host or device memory
 *    (detected with cudaPointerGetAttributes); every call is synchronous
 *    with respect to the caller.
 *  - one CUDA stream per context; handles are not thread-safe, use one per
 *    thread.  No torch types cross this boundary.
 */
#ifndef MSGPU_H
#define MSGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSGPU_ABI_VERSION 4

enum {
  MS_OK = 0,
  MS_E_INVALID = -1,   /* bad argument / dimension mismatch            -> ValueError   */
  MS_E_NOT_SPD = -2,   /* non-positive pivot in a Cholesky factor        -> ValueError   */
  MS_E_CUDA = -3,      /* CUDA runtime failure                           -> RuntimeError */
  MS_E_NOMEM = -4,     /* device allocation failed                       -> MemoryError  */
  MS_E_STATE = -5,     /* call out of order (e.g. apply before build)    -> RuntimeError */
  MS_E_CALLBACK = -6   /* a host callback operator returned non-zero     -> the callback's own exception */
};

typedef struct ms_ctx ms_ctx;
typedef struct ms_problem ms_problem;
typedef struct ms_precond ms_precond;

/* level-1 subdomain layouts */
enum {
  MS_LEVEL1_NEIGHBORHOODS = 0, /* reference: subdomains = omega_j, strictly interior nodes (schwarz.py:97-109) */
  MS_LEVEL1_BLOCKS = 1         /* BASELINE configs: delta-extended HxH blocks               */
};

/* level-1 operator (PreconditionerVariant.level1, schwarz.py:24-41) */
enum {
  MS_L1_ELASTICITY = 0, /* EH, EH+Rot: restrictions of K (schwarz.py:97-109)                     */
  MS_L1_HEAT = 1        /* HH, HH+Rot: one scalar diffusion factor for both blocks (:112-140)    */
};

/* coarse-space eigenproblem kind (PreconditionerVariant.eig_kind, schwarz.py:24-41) */
enum {
  MS_EIG_HEAT = 0,       /* EH*, HH*: scalar diffusion pencil, gap rule, 2 rows per mode (+ rotation) */
  MS_EIG_ELASTICITY = 1  /* EE, EE;Rand: elasticity pencil, rule 'fixed', 1 vector row per mode      */
};

/* level-1 local solver */
enum {
  MS_LOCAL_BANDED = 0,  /* banded Cholesky factor, forward/backward sweeps per apply */
  MS_LOCAL_DENSE_INV = 1 /* explicit packed dense inverse, batched SYMV per apply     */
};

/* coarse solve K0^-1 f0 (CoarseOperator.solve, coarse.py:150-154) */
enum {
  MS_COARSE_INVERSE = 0, /* explicit packed K0^-1, one bandwidth-bound SYMV per apply (default)      */
  MS_COARSE_CHOLESKY = 1 /* the reference's arithmetic: Cholesky factor (cho_factor, coarse.py:143)
                            and forward + backward triangular solves (cho_solve, coarse.py:154)     */
};

/* Options of build_preconditioner("EH+Rot" / "EH", ...) — schwarz.py:54-59, :176-211. */
typedef struct ms_precond_opts {
  int Nx, Ny;            /* coarse blocks per axis (CoarsePartition, grid.py:117)        */
  int level1_kind;       /* MS_LEVEL1_*                                                 */
  int delta;             /* overlap in elements for MS_LEVEL1_BLOCKS                    */
  int n_max;             /* EigOptions.n_max (default 6)                                */
  double gap_threshold;  /* select_modes gap threshold (default 50.0, spectral.py:161)  */
  int enrich;            /* 1: EH+Rot (enrich_rotations, coarse.py:120); 0: EH          */
  int fixed_rule;        /* 0: rule 'gap' (heat default); 1: rule 'fixed'               */
  int local_solver;      /* MS_LOCAL_*                                                  */
  int use_coarse;        /* 1 (default); 0 drops level 2 (diagnostics)                  */
  const int64_t* heat_dirichlet_nodes; /* whole nodes clamped in the heat eigenproblems */
  int64_t n_heat_dirichlet;
  /* EH+Rot;Rand / EE;Rand (solve_local_eig_randomized, spectral.py:103-158):
   * forcings [n_centers][n_snapshots][d (2H+1)^2] (closed-neighbourhood nodes,
   * row-major; d = 2 for MS_EIG_ELASTICITY: x-plane then y-plane; zero at
   * clamped nodes) drawn by the caller from default_rng([seed, centre]) */
  int randomized;
  int n_snapshots;
  const double* snapshots;
  int level1_operator;   /* MS_L1_* (needs whole-node constraints for MS_L1_HEAT)       */
  int eig_kind;          /* MS_EIG_*: neighbourhood eigenproblem kind                   */
  int coarse_solve;      /* MS_COARSE_* (ABI 3)                                         */
} ms_precond_opts;

/* Build metadata, the `info` dict of schwarz.py:202-210 plus eigensolver stats. */
typedef struct ms_precond_info {
  int coarse_dim;        /* N_c                                               */
  int n_centers;         /* interior coarse nodes (neighbourhoods)            */
  int n_subdomains;      /* level-1 subdomains                                */
  int max_eig_passes;    /* subspace-iteration passes of the slowest centre   */
  double mean_eig_passes; /* mean passes over centres                          */
  double t_level1;       /* s, level-1 assembly + factorisation               */
  double t_eig;          /* s, batched eigensolves + selection                */
  double t_coarse;       /* s, eigensolves + basis + K0 + factor/inverse      */
  double local_bytes;    /* bytes of level-1 operator data read per apply     */
  double coarse_bytes;   /* bytes of coarse data (psi + K0^-1) read per apply */
  int level1_twisted;    /* 1: two-sided (twisted) level-1 factors, 2 warps per subdomain */
  int level1_copies;     /* banded factor copies read per apply: 1 (column band, dot-form
                            backward sweep) or 2 (column + row band)                        */
  int n_subdomains_local; /* level-1 subdomains owned by this rank (all of them on one rank)    */
  int level1_unit;       /* 1: unit-diagonal L D L^T level-1 factors (no pivot multiply on the
                            sweeps' dependent chain), 0: Cholesky factors                      */
} ms_precond_info;

/* SolveReport (krylov.py:17-35); history arrays are caller-provided. */
typedef struct ms_report {
  int64_t kernel_launches; /* msgpu kernels launched by the solve (incl. init)  */
  int iterations;
  int converged;
  double final_residual;  /* ||r_k|| / ||b|| of the recursive residual        */
  double t_solve;         /* s, device time of the PCG loop (CUDA events)      */
  double t_total;         /* s, wall time of the call incl. host<->device copy */
} ms_report;

/* ---- context ---------------------------------------------------------- */
int ms_ctx_create(int device, ms_ctx** out);
int ms_ctx_destroy(ms_ctx* ctx);
/* copies the last error message of `ctx` (or the global one when ctx==NULL) */
int ms_last_error(const ms_ctx* ctx, char* buf, size_t len);
int ms_abi_version(void);

/* Per-kernel CUDA-event profiling of the PCG hot path (bench.py's roofline):
 * device milliseconds and launch counts accumulated per component, launches
 * issued after convergence excluded.  Components: */
enum {
  MS_PROF_MATVEC = 0,       /* matrix-free operator + p update + p.q         */
  MS_PROF_UPDATE = 1,       /* x, r update + ||r||                            */
  MS_PROF_LEVEL1 = 2,       /* batched level-1 banded forward/backward sweeps */
  MS_PROF_RESTRICT = 3,     /* R0 r                                           */
  MS_PROF_COARSE_SOLVE = 4, /* K0^-1 f0 packed SYMV (2 kernels)               */
  MS_PROF_COMBINE = 5,      /* level-1 overlap sum + prolongation + r.z       */
  MS_PROF_N = 8
};
int ms_ctx_set_profiling(ms_ctx* ctx, int on); /* also resets the counters */
/* record only the components in `mask` (bit 1 << MS_PROF_*); 0 = off */
int ms_ctx_set_profiling_mask(ms_ctx* ctx, unsigned mask);
int ms_ctx_profile_get(const ms_ctx* ctx, double* ms, long long* counts); /* MS_PROF_N each */
/* the context's cudaStream_t (for event timing by callers) */
void* ms_ctx_stream(const ms_ctx* ctx);

/* ---- multi-GPU strips ----------------------------------
 * One process per GPU.  Attach a communicator to the context before creating
 * the problem; ms_precond_build then shards subdomain rows (coarse block rows)
 * across ranks, every rank holding full-size vectors but updating only its
 * strip, with halo exchanges (p/z: 1 node row, r: overlap+1 rows, level-1
 * boundary subdomain rows, one row of coarse-restriction cell partials),
 * allreduces of the three PCG dot products and of the coarse residual f0,
 * and a replicated K0^-1 SYMV.
 * The reference is single-process; these entry points have no counterpart. */
typedef struct ms_comm_callbacks {
  void* user;
  /* device buffers; called after the context stream is synchronised; must
   * complete before returning; return 0 on success */
  int (*allreduce_sum)(void* user, double* dev, int64_t n);
  int (*broadcast)(void* user, void* dev, int64_t bytes, int root);
  int (*sendrecv)(void* user, const void* send_dev, int64_t send_bytes, int dst, void* recv_dev,
                  int64_t recv_bytes, int src); /* dst/src may be -1 */
} ms_comm_callbacks;
int ms_nccl_unique_id(void* out128);
int ms_ctx_attach_nccl(ms_ctx* ctx, int rank, int world, const void* unique_id128);
int ms_ctx_attach_callbacks(ms_ctx* ctx, int rank, int world, const ms_comm_callbacks* cb);
/* exercises the attached communicator: out4 = {allreduce of rank+1, allreduce
 * of 2 (twice through a captured graph when the communicator is capturable),
 * broadcast of 10*rank+7 from rank 0, the left neighbour's rank via send/recv} */
int ms_comm_selftest(ms_ctx* ctx, double* out4);
/* synchronous copy between host and/or device buffers (callback helpers) */
int ms_copy(void* dst, const void* src, size_t bytes);
/* device memory held by the library's block cache (released buffers kept for
 * reuse, at most MS_CACHE_BYTES, default 32 GiB): *bytes = cached bytes of the
 * current device; with release != 0 they are returned to the driver first
 * (e.g. before a large allocation outside the library).  No reference
 * counterpart: scipy has no device memory. */
int ms_cache_trim(int release, size_t* bytes);
/* node-row halo plan of rank `rank` owning rows [lo, hi] of 0..ny, depth k:
 * out12 = {send_lo, send_n, dst, recv_lo, recv_n, src} for slot 0 (towards the
 * previous rank) then slot 1 (towards the next); pure arithmetic, no CUDA */
int ms_halo_plan(int lo, int hi, int ny, int k, int rank, int world, int* out12);
/* strip partition used for `nrows` block rows: rank owns [*lo, *hi) */
int ms_strip_rows(int nrows, int world, int rank, int* lo, int* hi);

/* 8x8 unit plane-stress Q1 element stiffness (E = 1), component-grouped,
 * bit-for-bit the reference's _unit_elasticity_element (assembly.py:100-116);
 * host arithmetic, no device needed. */
int ms_unit_element(double nu, double* Ke64);

/* ---- operator: assemble_elasticity (assembly.py:208-220) ---------------
 * E: per-element modulus, n_el = nx*ny, row-major (e = j*nx + i).
 * free_dofs: sorted ascending full-dof ids (component-grouped), n_free of them.
 * Replaces `assemble_elasticity(mesh, coeff, dirichlet)` and the SymmetricSparseOperator it returns. */
int ms_problem_create(ms_ctx* ctx, int nx, int ny, double h, double nu, const double* E,
                      const int64_t* free_dofs, int64_t n_free, ms_problem** out);
int ms_problem_destroy(ms_problem* prob);
int64_t ms_problem_n_free(const ms_problem* prob);
/* replace E in place (topology-optimisation loop, topopt.py:150-160) */
int ms_problem_set_modulus(ms_problem* prob, const double* E);
/* q = A p over free dofs — replaces `op.matrix @ p` (krylov.py:90,114). */
int ms_operator_apply(ms_problem* prob, const double* p, double* q);

/* ---- preconditioner: build_preconditioner (schwarz.py:176-211) ---------- */
int ms_precond_build(ms_problem* prob, const ms_precond_opts* opts, ms_precond** out);
int ms_precond_destroy(ms_precond* pc);
/* z = M^-1 r — TwoLevelPreconditioner.apply (schwarz.py:76-84) */
int ms_precond_apply(ms_precond* pc, const double* r, double* z);
/* z = R0^T K0^-1 R0 r only — CoarseOperator.apply_inverse (coarse.py:156-158) */
int ms_precond_apply_coarse(ms_precond* pc, const double* r, double* z);
/* info; mode_counts (length >= n_centers) and eigenvalues (n_centers x 7,
 * row-major, the k = min(n_max+1, dim) lowest per centre, NaN-padded) may be NULL. */
int ms_precond_info_get(const ms_precond* pc, ms_precond_info* info, int* mode_counts,
                        double* eigenvalues);
/* dense K0 (N_c x N_c, row-major, host buffer), reference row ordering (coarse.py:94-133) */
int ms_precond_coarse_matrix(const ms_precond* pc, double* K0);
/* Component microbenchmark: each hot-path kernel alone, `reps` launches
 * timed with CUDA events on the context stream; ms[MS_BENCH_N] = mean ms. */
enum {
  MS_BENCH_MATVEC = 0,
  MS_BENCH_LEVEL1 = 1,
  MS_BENCH_RESTRICT = 2,
  MS_BENCH_COARSE_SOLVE = 3,
  MS_BENCH_COMBINE = 4,
  MS_BENCH_COMBINE_L1 = 5,     /* level-1 overlap sum only  */
  MS_BENCH_COMBINE_COARSE = 6, /* coarse prolongation only  */
  MS_BENCH_N = 8
};
int ms_precond_bench(ms_precond* pc, int reps, double* ms);

/* ---- PCG: pcg_solve (krylov.py:81-134) ------------------------------------
 * pc may be NULL (plain CG, the 'None' variant).  x0 = 0.  Stops when
 * ||r_k|| <= tol ||b|| for the recursively updated residual.
 * residuals (>= maxit+1), alphas (>= maxit), betas (>= maxit) may be NULL. */
int ms_pcg_solve(ms_problem* prob, ms_precond* pc, const double* b, double tol, int maxit,
                 double* x, ms_report* rep, double* residuals, double* alphas, double* betas);

/* ---- Generic PCG: the duck-typed seams of pcg_solve (ABI 4) -----------------
 * The reference's pcg_solve accepts any sparse / dense matrix or callable as
 * A and any object with .apply, callable or None as M (krylov.py:73-78, 90).
 * ms_linop names one such operand: the Q1 problem, the two-level
 * preconditioner, a CSR matrix held on the device (ms_csr: scipy.sparse and
 * ndarray operands), or a host callback (callables / foreign .apply objects;
 * `in` and `out` are host vectors of n doubles, return 0 or non-zero to abort
 * with MS_E_CALLBACK).  The recurrence, its vectors and its dot products stay
 * on the device; same stopping rule and histories as ms_pcg_solve. */
typedef struct ms_csr ms_csr;
typedef int (*ms_apply_fn)(void* user, const double* in, double* out, int64_t n);
enum {
  MS_LINOP_NONE = 0,     /* identity (M = None)                       */
  MS_LINOP_PROBLEM = 1,  /* handle = ms_problem*  (op.matrix @ v)     */
  MS_LINOP_PRECOND = 2,  /* handle = ms_precond*  (M.apply)           */
  MS_LINOP_CSR = 3,      /* handle = ms_csr*      (A @ v)             */
  MS_LINOP_CALLBACK = 4  /* fn(user, in, out, n) on host vectors      */
};
typedef struct ms_linop {
  int kind;
  void* handle;
  ms_apply_fn fn;
  void* user;
} ms_linop;

/* n x n CSR matrix (int64 row pointers, int32 column indices) copied to the device. */
int ms_csr_create(ms_ctx* ctx, int64_t n, const int64_t* indptr, const int* indices,
                  const double* data, ms_csr** out);
int ms_csr_apply(ms_csr* A, const double* v, double* out); /* host or device vectors */
int ms_csr_destroy(ms_csr* A);

/* pcg_solve (krylov.py:81-134) for any A / M pair above; b and x host or device. */
int ms_pcg_solve_generic(ms_ctx* ctx, int64_t n, const ms_linop* A, const ms_linop* M,
                         const double* b, double tol, int maxit, double* x, ms_report* rep,
                         double* residuals, double* alphas, double* betas);

/* ---- Topology-optimisation caller --------------------
 * The per-design-step coefficient pipeline of the SIMP loop (topopt.py:123-216)
 * on the device.  Vectors may be host or device pointers (device ones stay on
 * the device; host ones are staged).  Element vectors have nx*ny entries in
 * element order e = j*nx + i; full-dof vectors are [x-plane | y-plane]. */
typedef struct ms_filter ms_filter;

/* DensityFilter(mesh, radius) (assembly.py:290-325): cone weights
 * max(0, radius - h |d|), rows normalised by their (edge-clipped) sums. */
int ms_filter_create(ms_ctx* ctx, int nx, int ny, double h, double radius, ms_filter** out);
int ms_filter_destroy(ms_filter* f);
/* DensityFilter.apply (assembly.py:327-328): out = W rho, bit-identical */
int ms_filter_apply(ms_filter* f, const double* rho, double* out);
/* DensityFilter.adjoint (assembly.py:330-331): out = W^T v, bit-identical */
int ms_filter_adjoint(ms_filter* f, const double* v, double* out);

/* simp_modulus (assembly.py:280-287) written straight into the operator's
 * modulus (replaces re-assembly, topopt.py:161-164).  MS_E_INVALID when
 * rho_f leaves [-1e-12, 1 + 1e-12] or p < 1. */
int ms_problem_set_density(ms_problem* prob, const double* rho_f, double p, double E_min,
                           double E_max);

/* compliance_and_sensitivity (topopt.py:59-70): *g0 = f.u,
 * sens_e = -p clip(rho_f,0,1)^(p-1) (E_max - E_min) u_e^T k0 u_e. */
int ms_compliance_sensitivity(ms_ctx* ctx, int nx, int ny, double nu, const double* u_full,
                              const double* f_full, const double* rho_f, double p, double E_min,
                              double E_max, double* g0, double* sens);

/* oc_update (topopt.py:73-107): multiplier bracket (64 tries) + bisection
 * (200 steps, |vol - v*| <= 1e-8 v*) on the device; the volume measure is
 * volumes . W rho_new (filt != NULL) or volumes . rho_new.  MS_E_STATE when
 * the bracket search fails (the reference's RuntimeError).  *evaluations
 * (may be NULL) receives the number of candidate-volume evaluations. */
int ms_oc_update(ms_ctx* ctx, int64_t n, const ms_filter* filt, const double* rho, const double* dg,
                 const double* volumes, double v_star, double move, double damping, double* rho_new,
                 int* evaluations);

/* x = A^-1 b for one dense SPD matrix (row-major N x N, lower triangle read)
 * with the coarse-solve kernels: mode MS_COARSE_INVERSE (tiled inverse +
 * packed SYMV) or MS_COARSE_CHOLESKY (tiled Cholesky + blocked triangular
 * solves, LAPACK ?potrf/?potrs as in CoarseOperator, coarse.py:143,154).
 * MS_E_NOT_SPD on a non-positive pivot. */
int ms_dense_spd_solve(ms_ctx* ctx, int N, const double* A, const double* b, double* x, int mode);

/* deterministic device dot product of n doubles (volume / compliance logs) */
int ms_dot(ms_ctx* ctx, int64_t n, const double* a, const double* b, double* out);

#ifdef __cplusplus
}
#endif
#endif /* MSGPU_H */
