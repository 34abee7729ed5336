// C ABI of the B200-native EH+Rot Schwarz PCG path (include/msgpu.h).
//
// Host-side orchestration only: geometry, offsets, allocation and kernel
// sequencing.  All arithmetic on vectors, factors and eigenproblems runs in
// the kernels of operator.cu / banded.cu / eigen.cu / coarse.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/msgpu.h"
#include "banded.cuh"
#include "coarse.cuh"
#include "comm.cuh"
#include "common.cuh"
#include "eigen.cuh"
#include "generic.cuh"
#include "operator.cuh"
#include "topopt.cuh"

using namespace msgpu;

constexpr int kPcgChunk = 8;  // iterations per host convergence poll / graph replay

namespace {

std::mutex g_err_mu;
std::string g_err;

// Device block cache.  A released block is kept (after a device
// synchronisation, which cudaFree would also perform, so no stream can still
// be using it) and handed to a later allocation of between half its size and
// its size on the same device: repeated builds -- config 5 rebuilds the
// preconditioner every step -- stop paying cudaMalloc/cudaFree of gigabytes.
// At most MS_CACHE_BYTES (default 32 GiB) stay cached; a failed cudaMalloc
// returns the device's cached blocks to the driver and retries.
struct BlockCache {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> idle;         // (device, bytes) -> block
  std::unordered_map<void*, std::pair<int, size_t>> owned;  // every block we allocated
  size_t cached = 0, limit = 0;
  BlockCache() {
    const char* e = getenv("MS_CACHE_BYTES");
    limit = e ? (size_t)strtoull(e, nullptr, 10) : ((size_t)32 << 30);
  }
  void flush(int dev) {
    std::lock_guard<std::mutex> lk(mu);
    for (auto it = idle.begin(); it != idle.end();) {
      if (it->first.first == dev) {
        cudaFree(it->second);
        owned.erase(it->second);
        cached -= it->first.second;
        it = idle.erase(it);
      } else {
        ++it;
      }
    }
  }
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache();  // never destroyed: no ordering issue at exit
  return *c;
}

void* dev_alloc(size_t bytes, cudaError_t* err) {
  int dev = 0;
  cudaGetDevice(&dev);
  BlockCache& c = block_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.idle.lower_bound({dev, bytes});
    if (it != c.idle.end() && it->first.first == dev && it->first.second <= 2 * bytes) {
      void* p = it->second;
      c.cached -= it->first.second;
      c.idle.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c.flush(dev);
    e = cudaMalloc(&p, bytes);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    *err = e;
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(c.mu);
  c.owned[p] = {dev, bytes};
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  BlockCache& c = block_cache();
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.owned.find(p);
  if (it == c.owned.end() || c.cached + it->second.second > c.limit) {
    if (it != c.owned.end()) c.owned.erase(it);
    cudaFree(p);
    return;
  }
  c.idle.insert({it->second, p});
  c.cached += it->second.second;
}

// twisted level-1 sweeps when all subdomain pairs fit in one wave (3 CTAs of
// 2 pairs per SM): below that the plain sweeps' per-step chain is exposed;
// above it the twisted kernel needs a second wave (measured at config 5,
// 1,024 subdomains: twisted 2.52e9 vs plain 3.29e9 DOF-iter/s; config 2,
// 256 subdomains: twisted 1.96e9 vs plain 1.35e9)
constexpr bool kL1UnitDefault = true;  // 1-4% faster sweeps in every regime (config 2: 0.188 -> 0.180 ms, config 3: 1.94 -> 1.93 ms)
static int twist_max_subdomains(int device) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms * 3 * 2;
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    dev_free(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    release();
    if (count == 0) count = 1;
    cudaError_t e = cudaSuccess;
    p = static_cast<T*>(dev_alloc(count * sizeof(T), &e));
    if (!p)
      throw Error(MS_E_NOMEM, "cudaMalloc of " + std::to_string(count * sizeof(T)) +
                                  " bytes failed: " + cudaGetErrorString(e));
    n = count;
  }
  void zero(cudaStream_t st) { MS_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), st)); }
  void upload(const T* h, size_t count, cudaStream_t st) {
    if (count > n) alloc(count);
    if (count) MS_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, st));
  }
};

bool is_device_ptr(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// element matrices, same formulas as the reference (assembly.py:83-147)
// Bit-for-bit the reference's numpy evaluation (assembly.py:100-116): C is
// divided entrywise by (1 - nu^2), and each inner product of the two small
// matmuls accumulates with fused multiply-adds from zero in index order, as
// the BLAS kernel behind `B.T @ C @ B` does (all 64 doubles equal the
// reference's for nu = 0.3 and 0.25, tests/golden/ref_elements.npz).
void unit_elasticity(double nu, double K[64]) {
  const double g[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};
  const double den = 1.0 - nu * nu;
  const double C[3][3] = {{1.0 / den, nu / den, 0.0 / den},
                          {nu / den, 1.0 / den, 0.0 / den},
                          {0.0 / den, 0.0 / den, ((1.0 - nu) / 2.0) / den}};
  double A[8][8] = {};
  for (double xi : g)
    for (double eta : g) {
      const double dx[4] = {-(1 - eta), 1 - eta, eta, -eta};
      const double dy[4] = {-(1 - xi), -xi, xi, 1 - xi};
      double B[3][8] = {};
      for (int m = 0; m < 4; ++m) {
        B[0][m] = dx[m];
        B[1][4 + m] = dy[m];
        B[2][m] = dy[m];
        B[2][4 + m] = dx[m];
      }
      double BtC[8][3];
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 3; ++j) {
          double s = 0.0;
          for (int l = 0; l < 3; ++l) s = std::fma(B[l][i], C[l][j], s);
          BtC[i][j] = s;
        }
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
          double s = 0.0;
          for (int l = 0; l < 3; ++l) s = std::fma(BtC[i][l], B[l][j], s);
          A[i][j] += 0.25 * s;
        }
    }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) K[i * 8 + j] = 0.5 * (A[i][j] + A[j][i]);
}

// largest eigenvalue of a symmetric PSD 8x8 matrix (power iteration)
double max_eig_sym8(const double* A) {
  double x[8], y[8], lam = 0.0;
  for (int i = 0; i < 8; ++i) x[i] = 1.0 + 0.1 * i;
  for (int it = 0; it < 500; ++it) {
    double nrm = 0.0;
    for (int i = 0; i < 8; ++i) {
      y[i] = 0.0;
      for (int j = 0; j < 8; ++j) y[i] += A[i * 8 + j] * x[j];
      nrm += y[i] * y[i];
    }
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) return 0.0;
    lam = 0.0;
    for (int i = 0; i < 8; ++i) lam += x[i] * y[i];
    double xn = 0.0;
    for (int i = 0; i < 8; ++i) xn += x[i] * x[i];
    lam /= xn;
    for (int i = 0; i < 8; ++i) x[i] = y[i] / nrm;
  }
  return lam;
}

void heat_elements(double h, HeatParam& hp) {
  const double g[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};
  double A[4][4] = {};
  for (double xi : g)
    for (double eta : g) {
      const double dx[4] = {-(1 - eta), 1 - eta, eta, -eta};
      const double dy[4] = {-(1 - xi), -xi, xi, 1 - xi};
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) A[i][j] += 0.25 * (dx[i] * dx[j] + dy[i] * dy[j]);
    }
  const double pat[4][4] = {{4, 2, 1, 2}, {2, 4, 2, 1}, {1, 2, 4, 2}, {2, 1, 2, 4}};
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      hp.lap[i * 4 + j] = A[i][j];
      hp.mel[i * 4 + j] = (h * h / 36.0) * pat[i][j];
    }
}

}  // namespace

// Optional CUDA-event profiling of every hot-path kernel launch, tagged with
// the PCG iteration it belongs to (launches after convergence are dropped).
// Launches of PCG iteration i use the fixed event pair tab[i % chunk][comp],
// so the same recording works under CUDA-graph capture (event-record nodes):
// after each replay the captured pairs are re-queued with their iteration.
struct Prof {
  bool on = false;
  unsigned mask = ~0u;  // components (1 << MS_PROF_*) that record events
  double ms[MS_PROF_N] = {};
  long long cnt[MS_PROF_N] = {};
  std::vector<cudaEvent_t> pool;
  cudaEvent_t tab[kPcgChunk][MS_PROF_N][2] = {};
  bool capturing = false;
  struct Rec {
    int comp, it;
    cudaEvent_t a, b;
  };
  std::vector<Rec> pending;
  std::vector<std::pair<int, int>> captured;  // (comp, iteration within chunk)
  cudaEvent_t make() {
    cudaEvent_t e;
    MS_CUDA(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t get() {
    if (pool.empty()) return make();
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  // under capture an event must be recorded as an external node to be timed
  void record(cudaEvent_t e, cudaStream_t st) {
    if (capturing)
      MS_CUDA(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else
      MS_CUDA(cudaEventRecord(e, st));
  }
  cudaEvent_t slot(int comp, int it, int side) {
    cudaEvent_t& e = tab[it % kPcgChunk][comp][side];
    if (!e) e = make();
    return e;
  }
  bool timing(unsigned bits) const { return on && (mask & bits) != 0u; }
  cudaEvent_t begin(int comp, int it, cudaStream_t st) {
    if (!on || !((mask >> comp) & 1u)) return nullptr;
    cudaEvent_t a = it >= 0 ? slot(comp, it, 0) : get();
    record(a, st);
    return a;
  }
  void end(int comp, int it, cudaStream_t st, cudaEvent_t a) {
    if (!on || !((mask >> comp) & 1u)) return;
    cudaEvent_t b = it >= 0 ? slot(comp, it, 1) : get();
    record(b, st);
    if (capturing)
      captured.push_back({comp, it % kPcgChunk});
    else
      pending.push_back({comp, it, a, b});
  }
  // after a replay of the captured chunk starting at iteration it0
  void replayed(int it0) {
    for (const auto& c : captured)
      pending.push_back({c.first, it0 + c.second, tab[c.second][c.first][0], tab[c.second][c.first][1]});
  }
  // call after a stream sync; keep records of iterations < valid_iters
  void flush(int valid_iters) {
    for (const Rec& r : pending) {
      if (r.it < valid_iters) {
        float t = 0.f;
        MS_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
        ms[r.comp] += t;
        cnt[r.comp] += 1;
      }
      if (r.it < 0) {
        pool.push_back(r.a);
        pool.push_back(r.b);
      }
    }
    pending.clear();
  }
};

struct ms_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  // side branch of the preconditioner apply: the coarse restriction + solve
  // run here, concurrently with the level-1 sweeps on `st` (single rank)
  cudaStream_t st2 = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  std::string err;
  Prof prof;
  std::unique_ptr<Comm> comm;  // multi-GPU strips (world > 1)
  // scratch of the caller-pipeline entry points (dot / OC reductions)
  DBuf<double> red;
  DBuf<unsigned int> ticket;
  DBuf<double> dval;
  void ensure_scratch() {
    if (red.p) return;
    red.alloc(2 * kDotBlocks);
    ticket.alloc(1);
    ticket.zero(st);
    dval.alloc(8);
  }
  int world() const { return comm ? comm->world : 1; }
  int rank() const { return comm ? comm->rank : 0; }
};

struct ms_problem {
  ms_ctx* ctx = nullptr;
  Grid g{};
  // owned node rows (strip); whole mesh on one rank, set by ms_precond_build otherwise
  int b_lo = 0, b_hi = -1;
  std::vector<int> rank_lo, rank_hi;  // every rank's owned node rows
  double nu = 0.3;
  KeParam ke{};
  DBuf<double> E;
  DBuf<uint8_t> mask;
  DBuf<int64_t> free_dofs;
  int64_t n_free = 0;
  int64_t n_full = 0;
  // PCG workspace (full layout)
  DBuf<double> x, r, z, p0, p1, q, tmp, tmp2;
  DBuf<PcgScalars> sc;
  DBuf<double> partials;
  DBuf<double> hres, halpha, hbeta;
  int hcap = 0;
  int hist_gen = 0;  // bumped when the history buffers move (captured graphs hold their addresses)
  // captured PCG chunk (CUDA graph) of plain CG solves; preconditioned solves
  // keep theirs in the ms_precond (it captures both objects' buffers)
  cudaGraphExec_t gexec = nullptr, gexec_prof = nullptr;
  long long gexec_kernels = 0, gexec_prof_kernels = 0;  // kernel nodes per replay
  int graph_gen = 0;
  unsigned prof_mask = 0;  // Prof::mask the profiling graph was captured with
  std::vector<std::pair<int, int>> captured;
  ~ms_problem() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (gexec_prof) cudaGraphExecDestroy(gexec_prof);
  }
  void ensure_workspace() {
    if (x.p) return;
    const cudaStream_t st = ctx->st;
    for (DBuf<double>* b : {&x, &r, &z, &p0, &p1, &q, &tmp, &tmp2}) {
      b->alloc(n_full);
      b->zero(st);
    }
    sc.alloc(1);
    partials.alloc(std::max<int64_t>(reduce_blocks(), (int64_t)div_up(g.nx + 1, MV_TX) * div_up(g.ny + 1, MV_TY)));
  }
};

struct ms_precond {
  ms_problem* prob = nullptr;
  int device = 0;
  cudaStream_t st = nullptr;  // copies: destroy must not touch prob
  ms_precond_opts opts{};
  std::vector<int64_t> heat_dir;
  // level 1
  int NbX = 0, NbY = 0, nsys = 0, max_bw = 0, min_bw = 0;
  std::vector<BandSys> hsys;
  DBuf<BandSys> sys;
  DBuf<double> Lc, Lr, ybuf, Xinv;
  DBuf<double> Sinv;   // twisted level 1: separator Schur inverses (empty: plain sweeps)
  bool twisted = false;
  bool one_copy = false;  // plain banded level 1 with the column band only (dot-form backward sweep)
  bool bitwise = false;   // multi-rank results bit-identical to one rank (MS_DIST_BITWISE=1)
  bool pad = false;       // padded TMA ring (uniform bw), maps below
  bool unit = false;      // unit-diagonal L D L^T level-1 factors (sweep chain without the pivot multiply)
  L1Maps maps;
  bool dense = false;  // MS_LOCAL_DENSE_INV: packed explicit inverses in Xinv
  int nrhs = 1;        // 2: heat level-1 (scalar factor applied to both blocks)
  int dense_nt = 0;
  DBuf<int> xcov, ycov, xlo_d, xlen_d, ylo_d, ylen_d;
  DBuf<int64_t> yoff_d;
  L1Dev l1{};
  // coarse
  bool has_coarse = false;
  CoarseDev cd{};
  DBuf<int> nsel, hoff;
  DBuf<int64_t> psioff;
  DBuf<double> psi, chi, K0inv, f0, y0, part, evals, K0keep, chi4, psi4, rpart, psi0c;
  DBuf<int> chi_src;
  // MS_COARSE_CHOLESKY: packed factor L (in K0inv), inverses of its diagonal
  // tiles, the forward-sweep result and the blocked-TRSV tickets/flags
  bool coarse_factor = false;
  DBuf<double> K0dinv, trsv_t, trsv_y;
  DBuf<int> trsv_sync;
  std::vector<int> h_nsel;
  std::vector<double> h_evals;
  int N_c = 0;
  int max_pass = 0;
  ms_precond_info info{};
  // strip ownership: level-1 subdomain rows [J0, J1) -> subdomains [s0, s1);
  // coarse cell rows [C0, C1); centres [kc0, kc1).  One rank owns everything.
  int J0 = 0, J1 = 0, s0 = 0, s1 = 0, C0 = 0, C1 = 0, kc0 = 0, kc1 = 0, halo_rows = 1;
  // packed K0^-1 tiles [sym_t0, sym_t1) of the sharded coarse solve (all on one rank)
  int64_t sym_t0 = 0, sym_t1 = -1;
  cudaGraphExec_t gexec = nullptr, gexec_prof = nullptr;  // captured PCG chunks for (prob, this)
  long long gexec_kernels = 0, gexec_prof_kernels = 0;     // kernel nodes per replay
  int graph_gen = 0;  // prob->hist_gen the graphs were captured with
  unsigned prof_mask = 0;  // Prof::mask the profiling graph was captured with
  std::vector<std::pair<int, int>> captured;
  ~ms_precond() {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (gexec_prof) cudaGraphExecDestroy(gexec_prof);
  }
};

#define MS_API_BEGIN try {
#define MS_API_END(ctxptr)                                  \
  }                                                         \
  catch (const Error& e) {                                  \
    set_error(ctxptr, e.what());                            \
    return e.code;                                          \
  }                                                         \
  catch (const std::exception& e) {                         \
    set_error(ctxptr, e.what());                            \
    return MS_E_CUDA;                                       \
  }                                                         \
  return MS_OK;

static void set_error(ms_ctx* ctx, const std::string& m) {
  if (ctx) ctx->err = m;
  std::lock_guard<std::mutex> lk(g_err_mu);
  g_err = m;
}

// ---------------------------------------------------------------------------
// helpers

static void check_fail(DBuf<int>& flag, cudaStream_t st, const char* what) {
  int h = 0;
  MS_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  MS_CUDA(cudaStreamSynchronize(st));
  if (h != 0)
    throw Error(MS_E_NOT_SPD, std::string(what) + " not positive definite (pivot/system " +
                                  std::to_string(h - 1) + ")");
}

// copy an ABI vector (host or device, free layout) into a full-layout device vector
static void load_free(ms_problem* P, const double* src, double* dst_full) {
  const cudaStream_t st = P->ctx->st;
  MS_CUDA(cudaMemsetAsync(dst_full, 0, P->n_full * sizeof(double), st));
  const double* dsrc = src;
  if (!is_device_ptr(src)) {
    MS_CUDA(cudaMemcpyAsync(P->tmp2.p, src, P->n_free * sizeof(double), cudaMemcpyHostToDevice, st));
    dsrc = P->tmp2.p;
  }
  launch_scatter_free(P->n_free, P->free_dofs.p, dsrc, dst_full, st);
}

static void store_free(ms_problem* P, const double* src_full, double* dst) {
  const cudaStream_t st = P->ctx->st;
  if (is_device_ptr(dst)) {
    launch_gather_free(P->n_free, P->free_dofs.p, src_full, dst, st);
  } else {
    launch_gather_free(P->n_free, P->free_dofs.p, src_full, P->tmp2.p, st);
    MS_CUDA(cudaMemcpyAsync(dst, P->tmp2.p, P->n_free * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  MS_CUDA(cudaStreamSynchronize(st));
}

static void level1_axis(int n_el, int nblocks, int kind, int delta, std::vector<int>& lo,
                        std::vector<int>& hi) {
  const int H = n_el / nblocks;
  lo.clear();
  hi.clear();
  if (kind == MS_LEVEL1_NEIGHBORHOODS) {
    for (int I = 1; I < nblocks; ++I) {
      lo.push_back((I - 1) * H + 1);
      hi.push_back((I + 1) * H - 1);
    }
  } else {
    for (int I = 0; I < nblocks; ++I) {
      const int e0 = std::max(0, I * H - delta), e1 = std::min(n_el, (I + 1) * H + delta);
      lo.push_back(e0 == 0 ? 0 : e0 + 1);
      hi.push_back(e1 == n_el ? n_el : e1 - 1);
    }
  }
}

// ---------------------------------------------------------------------------
// multi-rank helpers.  Every rank holds full-length vectors; rank r updates
// node rows [rank_lo[r], rank_hi[r]] ("owned") and receives halo rows.

static int row_hi(const ms_problem* P) { return P->b_hi < 0 ? P->g.ny : P->b_hi; }

// Halo plan for k node rows: rows [lo, hi] owned, neighbours prev/next.
// slot 0: send my lowest rows to prev, receive next's lowest rows above me;
// slot 1: send my highest rows to next, receive prev's highest rows below me.
struct HaloPlan {
  int send_lo[2], send_n[2], dst[2];
  int recv_lo[2], recv_n[2], src[2];
};

static HaloPlan halo_plan(int lo, int hi, int ny, int k, int rank, int world) {
  HaloPlan h{};
  const int prev = rank > 0 ? rank - 1 : -1, next = rank < world - 1 ? rank + 1 : -1;
  const int kd = std::min(k, hi - lo + 1);
  const int kb = std::min(k, lo), ka = std::min(k, ny - hi);
  h.dst[0] = prev;
  h.send_lo[0] = lo;
  h.send_n[0] = prev >= 0 ? kd : 0;
  h.src[0] = next;
  h.recv_lo[0] = hi + 1;
  h.recv_n[0] = next >= 0 ? ka : 0;
  h.dst[1] = next;
  h.send_lo[1] = hi - kd + 1;
  h.send_n[1] = next >= 0 ? kd : 0;
  h.src[1] = prev;
  h.recv_lo[1] = lo - kb;
  h.recv_n[1] = prev >= 0 ? kb : 0;
  return h;
}

// every non-empty send / receive segment of a transfer list must lie inside
// the buffer it addresses (host-side, always on: a wrong strip or halo plan
// fails here instead of corrupting a neighbour's rows)
static void check_xfers(const Xfer* x, int n, const void* base, size_t bytes, const char* what) {
  const char* lo = static_cast<const char*>(base);
  const char* hi = lo + bytes;
  for (int i = 0; i < n; ++i) {
    const char* s = static_cast<const char*>(x[i].s);
    const char* r = static_cast<const char*>(x[i].r);
    if ((x[i].sb && (s < lo || s + x[i].sb > hi)) || (x[i].rb && (r < lo || r + x[i].rb > hi)))
      throw Error(MS_E_STATE, std::string(what) + ": transfer " + std::to_string(i) + " leaves its buffer");
  }
}

// the 4 transfers of a k-row halo of both planes with the neighbouring strips
static void row_halo_xfers(ms_problem* P, Comm* c, double* v, int k, Xfer x[4]) {
  const HaloPlan h = halo_plan(P->b_lo, row_hi(P), P->g.ny, k, c->rank, c->world);
  const int64_t rowb = (int64_t)P->g.nnx * sizeof(double);
  for (int plane = 0; plane < 2; ++plane) {
    char* base = reinterpret_cast<char*>(v + plane * P->g.n_nodes);
    for (int q = 0; q < 2; ++q)
      x[plane * 2 + q] = {base + h.send_lo[q] * rowb, (size_t)(h.send_n[q] * rowb), h.dst[q],
                          base + h.recv_lo[q] * rowb, (size_t)(h.recv_n[q] * rowb), h.src[q]};
  }
  check_xfers(x, 4, v, (size_t)2 * P->g.n_nodes * sizeof(double), "row halo");
}

// exchange k node rows of both planes with the neighbouring strips
static void exchange_rows(ms_problem* P, double* v, int k) {
  Comm* c = P->ctx->comm.get();
  if (!c || c->world == 1 || k <= 0) return;
  // both planes and both neighbours in one group (one NCCL launch per halo)
  Xfer x[4];
  row_halo_xfers(P, c, v, k, x);
  c->sendrecv(x, 4, P->ctx->st);
}

// every rank ends with every rank's owned rows (solution / operator output)
static void allgather_rows(ms_problem* P, double* v) {
  Comm* c = P->ctx->comm.get();
  if (!c || c->world == 1) return;
  // no strip ownership before a preconditioner is built: every rank then
  // computes all rows (b_hi = -1), nothing to gather
  if ((int)P->rank_lo.size() < c->world || (int)P->rank_hi.size() < c->world) return;
  const int64_t rowb = (int64_t)P->g.nnx * sizeof(double);
  for (int r = 0; r < c->world; ++r)
    for (int plane = 0; plane < 2; ++plane) {
      char* base = reinterpret_cast<char*>(v + plane * P->g.n_nodes);
      c->broadcast(base + P->rank_lo[r] * rowb, (P->rank_hi[r] - P->rank_lo[r] + 1) * rowb, r, P->ctx->st);
    }
}

// level-1 solutions of the neighbours' boundary subdomain rows (their overlap
// reaches into my strip)
static void ybuf_xfers(ms_precond* pc, Comm* c, Xfer x[2]);
static void exchange_ybuf(ms_precond* pc) {
  ms_problem* P = pc->prob;
  Comm* c = P->ctx->comm.get();
  if (!c || c->world == 1) return;
  Xfer x[2];
  ybuf_xfers(pc, c, x);
  c->sendrecv(x, 2, P->ctx->st);
}
// the level-1 boundary subdomain-row solutions to and from the neighbours
static void ybuf_xfers(ms_precond* pc, Comm* c, Xfer x[2]) {
  const int r = c->rank, W = c->world;
  const int prev = r > 0 ? r - 1 : -1, next = r < W - 1 ? r + 1 : -1;
  auto seg = [&](int J, int64_t& off, int64_t& bytes) {
    const BandSys& a = pc->hsys[(size_t)J * pc->NbX];
    const BandSys& b = pc->hsys[(size_t)J * pc->NbX + pc->NbX - 1];
    off = a.yoff;
    bytes = (b.yoff + (int64_t)b.n * b.nrhs - a.yoff) * (int64_t)sizeof(double);
  };
  int64_t o_first, b_first, o_last, b_last, o_pl, b_pl, o_nf, b_nf;
  seg(pc->J0, o_first, b_first);
  seg(pc->J1 - 1, o_last, b_last);
  if (prev >= 0) seg(pc->J0 - 1, o_pl, b_pl); else o_pl = b_pl = 0;
  if (next >= 0) seg(pc->J1, o_nf, b_nf); else o_nf = b_nf = 0;
  double* y = pc->ybuf.p;
  x[0] = {y + o_first, (size_t)(prev >= 0 ? b_first : 0), prev, y + o_nf, (size_t)b_nf, next};
  x[1] = {y + o_last, (size_t)(next >= 0 ? b_last : 0), next, y + o_pl, (size_t)b_pl, prev};
  check_xfers(x, 2, y, pc->ybuf.n * sizeof(double), "level-1 boundary solutions");
}

// restriction partials of the cell row below my lowest centre row (prev's last)
// the restriction partials of the coarse-cell row below each strip (its
// centres' f0 rows need the 4 cells around them)
static void rpart_xfers(ms_precond* pc, Comm* c, Xfer x[2]) {
  const int r = c->rank, W = c->world;
  const int prev = r > 0 ? r - 1 : -1, next = r < W - 1 ? r + 1 : -1;
  const int64_t rowd = (int64_t)pc->cd.Nx * 4 * kSlots;
  double* rp = pc->rpart.p;
  x[0] = {nullptr, 0, -1, nullptr, 0, -1};
  x[1] = {rp + (pc->C1 - 1) * rowd, (size_t)(next >= 0 ? rowd * sizeof(double) : 0), next, rp + (pc->C0 - 1) * rowd,
          (size_t)(prev >= 0 ? rowd * sizeof(double) : 0), prev};
  check_xfers(x, 2, rp, pc->rpart.n * sizeof(double), "restriction partials");
}
static void exchange_rpart(ms_precond* pc) {
  ms_problem* P = pc->prob;
  Comm* c = P->ctx->comm.get();
  if (!c || c->world == 1) return;
  Xfer x[2];
  rpart_xfers(pc, c, x);
  c->sendrecv(x, 2, P->ctx->st);
}

// bitwise mode: the block partials of one dot product sit in their global
// slots on every rank (zero where another rank owns the block); summing the
// arrays over ranks is exact, and the fixed-order reduction with the
// producing kernel's block size gives the one-rank value bit for bit
static void dist_zero_partials(ms_problem* P, int nb) {
  MS_CUDA(cudaMemsetAsync(P->partials.p, 0, (size_t)nb * sizeof(double), P->ctx->st));
}
static void dist_reduce_bitwise(ms_problem* P, int kind, int nb, int threads, double* hist,
                                const Xfer* x = nullptr, int nx = 0) {
  Comm* c = P->ctx->comm.get();
  if (nx)
    c->allreduce_sendrecv(P->partials.p, nb, x, nx, P->ctx->st);
  else
    c->allreduce_sum(P->partials.p, nb, P->ctx->st);
  launch_reduce_partials(P->partials.p, nb, threads, &P->sc.p->part[kind], P->ctx->st);
  launch_finalize(P->sc.p, kind, hist, P->ctx->st);
}

static void dist_finalize(ms_problem* P, int kind, double* hist) {
  Comm* c = P->ctx->comm.get();
  if (!c || c->world == 1) return;
  c->allreduce_sum(&P->sc.p->part[kind], 1, P->ctx->st);
  launch_finalize(P->sc.p, kind, hist, P->ctx->st);
}

// y0 = K0^-1 f0: each rank streams its share of the packed inverse's tiles,
// the partial y0 are summed over ranks (N_c doubles)
// MS_COARSE_CHOLESKY: y0 = L^-T L^-1 f0 (cho_solve, coarse.py:154) with the
// full factor on every rank, no collective
static void coarse_solve(ms_precond* pc, const int* done, cudaStream_t st) {
  if (pc->coarse_factor) {
    launch_trsv_packed(pc->N_c, pc->K0inv.p, pc->K0dinv.p, pc->f0.p, pc->trsv_t.p, pc->trsv_y.p, pc->y0.p,
                       pc->trsv_sync.p, done, st);
    return;
  }
  launch_symv_packed(pc->N_c, pc->K0inv.p, pc->f0.p, pc->y0.p, pc->part.p, done, st, pc->sym_t0, pc->sym_t1);
  Comm* c = pc->prob->ctx->comm.get();
  if (c && c->world > 1 && !pc->bitwise) c->allreduce_sum(pc->y0.p, pc->N_c, st);  // bitwise: replicated
}

// precond apply on full-layout r -> z (device); sc/partials/beta_hist for PCG mode
// `restricted`: the cell restriction partials of r were already produced
// (fused into the residual update); only their reduction remains.
static int overlap_coarse() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MS_OVERLAP");
    v = (e && std::string(e) == "1") ? 1 : 0;  // opt-in: MS_OVERLAP=1
  }
  return v;
}

// coarse branch: f0 = R0 r (cell partials unless already fused), y0 = K0^-1 f0
// `rr_hist` != nullptr (multi-rank PCG iteration): the rank's ||r||^2 partial
// rides in slot N_c of the f0 allreduce instead of its own collective, and is
// finalised (residual, convergence flag) right after it.
static void coarse_restrict(ms_precond* pc, const double* r, const int* done, int it, bool restricted, bool dist,
                            cudaStream_t st, double* rr_hist = nullptr) {
  ms_problem* P = pc->prob;
  Prof& pf = P->ctx->prof;
  cudaEvent_t a = pf.begin(MS_PROF_RESTRICT, it, st);
  if (!restricted) launch_restrict_cells(P->g, pc->C0, pc->C1, pc->cd, r, done, st);
  if (dist) {
    exchange_rpart(pc);
    MS_CUDA(cudaMemsetAsync(pc->f0.p, 0, pc->N_c * sizeof(double), st));
  }
  launch_restrict_reduce(pc->cd, pc->f0.p, done, st, pc->kc0, pc->kc1);
  if (dist) {
    PcgScalars* sc = P->sc.p;
    if (rr_hist)
      MS_CUDA(cudaMemcpyAsync(pc->f0.p + pc->N_c, &sc->part[PART_RR], sizeof(double), cudaMemcpyDeviceToDevice, st));
    P->ctx->comm->allreduce_sum(pc->f0.p, pc->N_c + (rr_hist ? 1 : 0), st);
    if (rr_hist) {
      MS_CUDA(cudaMemcpyAsync(&sc->part[PART_RR], pc->f0.p + pc->N_c, sizeof(double), cudaMemcpyDeviceToDevice, st));
      launch_finalize(sc, PART_RR, rr_hist, st);
    }
  }
  pf.end(MS_PROF_RESTRICT, it, st, a);
}

static void coarse_branch(ms_precond* pc, const double* r, const int* done, int it, bool restricted, bool dist,
                          cudaStream_t st, double* rr_hist = nullptr) {
  coarse_restrict(pc, r, done, it, restricted, dist, st, rr_hist);
  Prof& pf = pc->prob->ctx->prof;
  cudaEvent_t a = pf.begin(MS_PROF_COARSE_SOLVE, it, st);
  coarse_solve(pc, done, st);
  pf.end(MS_PROF_COARSE_SOLVE, it, st, a);
}

// Multi-rank PCG apply with the collectives regrouped (5 communicator
// calls per iteration instead of 7): the restriction partials were fused
// into the residual update and exchanged together with the r halo, so the
// restriction reduce runs before the level-1 sweeps, and the sweeps'
// boundary solutions travel in the same group as the f0 (+ ||r||^2)
// allreduce.
static void precond_apply_dist_grouped(ms_precond* pc, const double* r, double* z, PcgScalars* sc,
                                       double* beta_hist, int it, double* rr_hist) {
  ms_problem* P = pc->prob;
  ms_ctx* ctx = P->ctx;
  const cudaStream_t st = ctx->st;
  Prof& pf = ctx->prof;
  Comm* c = ctx->comm.get();
  const int* done = &sc->done;
  const int ns = pc->s1 - pc->s0;
  cudaEvent_t a = pf.begin(MS_PROF_RESTRICT, it, st);
  MS_CUDA(cudaMemsetAsync(pc->f0.p, 0, pc->N_c * sizeof(double), st));
  launch_restrict_reduce(pc->cd, pc->f0.p, done, st, pc->kc0, pc->kc1);
  if (rr_hist)
    MS_CUDA(cudaMemcpyAsync(pc->f0.p + pc->N_c, &P->sc.p->part[PART_RR], sizeof(double), cudaMemcpyDeviceToDevice,
                            st));
  pf.end(MS_PROF_RESTRICT, it, st, a);
  if (ns > 0) {
    a = pf.begin(MS_PROF_LEVEL1, it, st);
    if (pc->dense)
      launch_l1_dense_apply(P->g, pc->sys.p + pc->s0, ns, pc->dense_nt, pc->Xinv.p, r, pc->ybuf.p, done, st);
    else
      launch_l1_solve(P->g, pc->sys.p + pc->s0, ns, pc->max_bw, pc->nrhs, pc->Lc.p, pc->Lr.p, r, pc->ybuf.p, done, st,
                      pc->twisted ? pc->Sinv.p : nullptr, pc->min_bw, &pc->maps, pc->unit);
    pf.end(MS_PROF_LEVEL1, it, st, a);
  }
  Xfer yx[2];
  ybuf_xfers(pc, c, yx);
  c->allreduce_sendrecv(pc->f0.p, pc->N_c + (rr_hist ? 1 : 0), yx, ns > 0 ? 2 : 0, st);
  if (rr_hist) {
    MS_CUDA(cudaMemcpyAsync(&P->sc.p->part[PART_RR], pc->f0.p + pc->N_c, sizeof(double), cudaMemcpyDeviceToDevice,
                            st));
    launch_finalize(P->sc.p, PART_RR, rr_hist, st);
  }
  a = pf.begin(MS_PROF_COARSE_SOLVE, it, st);
  coarse_solve(pc, done, st);
  pf.end(MS_PROF_COARSE_SOLVE, it, st, a);
  a = pf.begin(MS_PROF_COMBINE, it, st);
  const bool bitwise = pc->bitwise;
  if (bitwise) dist_zero_partials(P, pc->opts.Nx * pc->opts.Ny);
  launch_combine(P->g, P->mask.p, pc->nsys > 0 ? &pc->l1 : nullptr, &pc->cd, pc->opts.Nx, pc->opts.Ny, pc->y0.p, r,
                 z, sc, P->partials.p, beta_hist, st, pc->C0, pc->C1);
  pf.end(MS_PROF_COMBINE, it, st, a);
  Xfer x[4];
  row_halo_xfers(P, c, z, 1, x);
  if (bitwise) {
    dist_reduce_bitwise(P, PART_RZ, pc->opts.Nx * pc->opts.Ny, combine_threads(), beta_hist, x, 4);
  } else {
    c->allreduce_sendrecv(&P->sc.p->part[PART_RZ], 1, x, 4, st);
    launch_finalize(P->sc.p, PART_RZ, beta_hist, st);
  }
}

// precond apply on full-layout r -> z (device); sc/partials/beta_hist for PCG mode
// `restricted`: the cell restriction partials of r were already produced
// (fused into the residual update); only their reduction remains.
// With MS_OVERLAP=1, on one rank, the coarse branch forks onto ctx->st2 and
// runs concurrently with the level-1 sweeps.  Both are HBM streams and the
// sweeps already run at ~93% of peak, so the fork only pays when the SYMV's
// slack outweighs the sweeps' slowdown: measured -1.1% per iteration on one
// B200 and +1.0% on another (config 3), hence opt-in.  With a communicator the
// apply stays on one stream: collectives of one communicator must not run
// concurrently.
static void precond_apply_full(ms_precond* pc, const double* r, double* z, PcgScalars* sc,
                               double* beta_hist, int it = -1, bool restricted = false,
                               double* rr_hist = nullptr) {
  ms_problem* P = pc->prob;
  ms_ctx* ctx = P->ctx;
  const cudaStream_t st = ctx->st;
  Prof& pf = ctx->prof;
  const int* done = sc ? &sc->done : nullptr;
  cudaEvent_t a;
  const bool dist = ctx->world() > 1;
  const int ns = pc->s1 - pc->s0;
  // a per-component profile times the branch serialized (its events would
  // otherwise measure the branch stretched across the concurrent sweeps)
  const bool fork = pc->has_coarse && ns > 0 && !dist && overlap_coarse() != 0 &&
                    !pf.timing((1u << MS_PROF_RESTRICT) | (1u << MS_PROF_COARSE_SOLVE));
  if (fork) {
    MS_CUDA(cudaEventRecord(ctx->fork, st));
    MS_CUDA(cudaStreamWaitEvent(ctx->st2, ctx->fork, 0));
    coarse_branch(pc, r, done, it, restricted, dist, ctx->st2);
    MS_CUDA(cudaEventRecord(ctx->join, ctx->st2));
  }
  if (ns > 0) {
    a = pf.begin(MS_PROF_LEVEL1, it, st);
    if (pc->dense)
      launch_l1_dense_apply(P->g, pc->sys.p + pc->s0, ns, pc->dense_nt, pc->Xinv.p, r, pc->ybuf.p, done, st);
    else
      launch_l1_solve(P->g, pc->sys.p + pc->s0, ns, pc->max_bw, pc->nrhs, pc->Lc.p, pc->Lr.p, r, pc->ybuf.p, done, st,
                      pc->twisted ? pc->Sinv.p : nullptr, pc->min_bw, &pc->maps, pc->unit);
    pf.end(MS_PROF_LEVEL1, it, st, a);
    if (dist) exchange_ybuf(pc);
  }
  if (fork)
    MS_CUDA(cudaStreamWaitEvent(st, ctx->join, 0));
  else if (pc->has_coarse)
    coarse_branch(pc, r, done, it, restricted, dist, st, rr_hist);
  a = pf.begin(MS_PROF_COMBINE, it, st);
  const bool bitwise = dist && sc && pc->bitwise;
  if (bitwise) dist_zero_partials(P, pc->opts.Nx * pc->opts.Ny);
  launch_combine(P->g, P->mask.p, pc->nsys > 0 ? &pc->l1 : nullptr, pc->has_coarse ? &pc->cd : nullptr,
                 pc->opts.Nx, pc->opts.Ny, pc->y0.p, r, z, sc, P->partials.p, beta_hist, st, pc->C0, pc->C1);
  pf.end(MS_PROF_COMBINE, it, st, a);
  if (bitwise) {
    Xfer x[4];
    row_halo_xfers(P, ctx->comm.get(), z, 1, x);
    dist_reduce_bitwise(P, PART_RZ, pc->opts.Nx * pc->opts.Ny, combine_threads(), beta_hist, x, 4);
  } else if (dist) {
    if (sc) {
      // r.z allreduce and the z halo (the next matvec refreshes p on one halo
      // row) in one communicator group, then the beta / convergence finalise
      Comm* c = ctx->comm.get();
      Xfer x[4];
      row_halo_xfers(P, c, z, 1, x);
      c->allreduce_sendrecv(&P->sc.p->part[PART_RZ], 1, x, 4, st);
      launch_finalize(P->sc.p, PART_RZ, beta_hist, st);
    } else {
      exchange_rows(P, z, 1);
    }
  }
}


// ---------------------------------------------------------------------------
extern "C" {

int ms_abi_version(void) { return MSGPU_ABI_VERSION; }

int ms_unit_element(double nu, double* Ke64) {
  MS_API_BEGIN
  if (!Ke64) throw Error(MS_E_INVALID, "null argument");
  if (!(nu >= 0.0 && nu < 0.5)) throw Error(MS_E_INVALID, "Poisson ratio outside [0, 0.5)");
  unit_elasticity(nu, Ke64);
  MS_API_END(nullptr)
}

int ms_last_error(const ms_ctx* ctx, char* buf, size_t len) {
  if (!buf || len == 0) return MS_E_INVALID;
  std::string m;
  if (ctx)
    m = ctx->err;
  else {
    std::lock_guard<std::mutex> lk(g_err_mu);
    m = g_err;
  }
  std::strncpy(buf, m.c_str(), len - 1);
  buf[len - 1] = '\0';
  return MS_OK;
}

int ms_ctx_create(int device, ms_ctx** out) {
  ms_ctx* c = nullptr;
  MS_API_BEGIN
  if (!out) throw Error(MS_E_INVALID, "null output handle");
  int ndev = 0;
  MS_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) throw Error(MS_E_INVALID, "invalid CUDA device " + std::to_string(device));
  MS_CUDA(cudaSetDevice(device));
  c = new ms_ctx();
  c->device = device;
  MS_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  {
    int lo = 0, hi = 0;  // the short coarse branch gets SM slots first as level-1 CTAs retire
    MS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    MS_CUDA(cudaStreamCreateWithPriority(&c->st2, cudaStreamNonBlocking, hi));
  }
  MS_CUDA(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
  MS_CUDA(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
  *out = c;
  MS_API_END(c)
}

int ms_ctx_set_profiling(ms_ctx* ctx, int on) { return ms_ctx_set_profiling_mask(ctx, on ? ~0u : 0u); }

int ms_ctx_set_profiling_mask(ms_ctx* ctx, unsigned mask) {
  MS_API_BEGIN
  if (!ctx) throw Error(MS_E_INVALID, "null context");
  ctx->prof.on = mask != 0u;
  ctx->prof.mask = mask;
  for (int i = 0; i < MS_PROF_N; ++i) {
    ctx->prof.ms[i] = 0.0;
    ctx->prof.cnt[i] = 0;
  }
  MS_API_END(ctx)
}

int ms_ctx_profile_get(const ms_ctx* ctx, double* ms, long long* counts) {
  if (!ctx || !ms || !counts) return MS_E_INVALID;
  for (int i = 0; i < MS_PROF_N; ++i) {
    ms[i] = ctx->prof.ms[i];
    counts[i] = ctx->prof.cnt[i];
  }
  return MS_OK;
}

void* ms_ctx_stream(const ms_ctx* ctx) { return ctx ? (void*)ctx->st : nullptr; }

int ms_nccl_unique_id(void* out128) {
  MS_API_BEGIN
  if (!out128) throw Error(MS_E_INVALID, "null argument");
  nccl_unique_id(out128);
  MS_API_END(nullptr)
}

int ms_ctx_attach_nccl(ms_ctx* ctx, int rank, int world, const void* unique_id128) {
  MS_API_BEGIN
  if (!ctx || !unique_id128 || world < 1 || rank < 0 || rank >= world) throw Error(MS_E_INVALID, "bad argument");
  ctx->comm = make_nccl_comm(rank, world, unique_id128, ctx->device);
  MS_API_END(ctx)
}

int ms_comm_selftest(ms_ctx* ctx, double* out4) {
  MS_API_BEGIN
  if (!ctx || !out4) throw Error(MS_E_INVALID, "null argument");
  Comm* c = ctx->comm.get();
  if (!c) throw Error(MS_E_STATE, "no communicator attached");
  MS_CUDA(cudaSetDevice(ctx->device));
  const cudaStream_t st = ctx->st;
  const int R = c->rank, W = c->world;
  DBuf<double> buf;
  buf.alloc(5);
  const double h[5] = {(double)(R + 1), 2.0, (double)(10 * R + 7), (double)R, -1.0};
  buf.upload(h, 5, st);
  c->allreduce_sum(buf.p, 2, st);                        // -> W(W+1)/2, 2W
  c->broadcast(buf.p + 2, sizeof(double), 0, st);        // -> 7 (root 0)
  c->sendrecv2(buf.p + 3, sizeof(double), (R + 1) % W, buf.p + 4, sizeof(double), (R + W - 1) % W,
               nullptr, 0, -1, nullptr, 0, -1, st);      // ring: receive the left neighbour's rank
  if (c->capturable()) {                                 // the PCG chunks capture collectives in graphs
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    MS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    c->allreduce_sum(buf.p + 1, 1, st);
    MS_CUDA(cudaStreamEndCapture(st, &graph));
    MS_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    MS_CUDA(cudaGraphLaunch(exec, st));                  // -> 2W * W
    MS_CUDA(cudaGraphExecDestroy(exec));
    MS_CUDA(cudaGraphDestroy(graph));
  }
  double r[5];
  MS_CUDA(cudaMemcpyAsync(r, buf.p, sizeof(r), cudaMemcpyDeviceToHost, st));
  MS_CUDA(cudaStreamSynchronize(st));
  for (int i = 0; i < 4; ++i) out4[i] = r[i == 3 ? 4 : i];
  MS_API_END(ctx)
}

int ms_ctx_attach_callbacks(ms_ctx* ctx, int rank, int world, const ms_comm_callbacks* cb) {
  MS_API_BEGIN
  if (!ctx || world < 1 || rank < 0 || rank >= world) throw Error(MS_E_INVALID, "bad argument");
  ctx->comm = make_callback_comm(rank, world, cb);
  MS_API_END(ctx)
}

int ms_cache_trim(int release, size_t* bytes) {
  MS_API_BEGIN
  int dev = 0;
  MS_CUDA(cudaGetDevice(&dev));
  BlockCache& c = block_cache();
  if (release) c.flush(dev);
  if (bytes) {
    std::lock_guard<std::mutex> lk(c.mu);
    size_t b = 0;
    for (const auto& kv : c.idle)
      if (kv.first.first == dev) b += kv.first.second;
    *bytes = b;
  }
  MS_API_END(nullptr)
}

int ms_copy(void* dst, const void* src, size_t bytes) {
  MS_API_BEGIN
  if (bytes && (!dst || !src)) throw Error(MS_E_INVALID, "null argument");
  if (bytes) {
    MS_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
    // a pageable host->device cudaMemcpy may return before the DMA lands, and
    // the solver's streams do not order against the legacy stream: complete it
    MS_CUDA(cudaDeviceSynchronize());
  }
  MS_API_END(nullptr)
}

int ms_halo_plan(int lo, int hi, int ny, int k, int rank, int world, int* out12) {
  if (!out12 || world < 1 || rank < 0 || rank >= world) return MS_E_INVALID;
  const HaloPlan h = halo_plan(lo, hi, ny, k, rank, world);
  const int v[12] = {h.send_lo[0], h.send_n[0], h.dst[0], h.recv_lo[0], h.recv_n[0], h.src[0],
                     h.send_lo[1], h.send_n[1], h.dst[1], h.recv_lo[1], h.recv_n[1], h.src[1]};
  std::memcpy(out12, v, sizeof(v));
  return MS_OK;
}

int ms_strip_rows(int nrows, int world, int rank, int* lo, int* hi) {
  if (!lo || !hi || world < 1 || rank < 0 || rank >= world || nrows < world) return MS_E_INVALID;
  strip_rows(nrows, world, rank, *lo, *hi);
  return MS_OK;
}

int ms_ctx_destroy(ms_ctx* ctx) {
  if (!ctx) return MS_OK;
  cudaSetDevice(ctx->device);
  if (ctx->st) cudaStreamDestroy(ctx->st);
  if (ctx->st2) cudaStreamDestroy(ctx->st2);
  if (ctx->fork) cudaEventDestroy(ctx->fork);
  if (ctx->join) cudaEventDestroy(ctx->join);
  delete ctx;
  return MS_OK;
}

int ms_problem_create(ms_ctx* ctx, int nx, int ny, double h, double nu, const double* E,
                      const int64_t* free_dofs, int64_t n_free, ms_problem** out) {
  MS_API_BEGIN
  if (!ctx || !out || !E || (!free_dofs && n_free > 0)) throw Error(MS_E_INVALID, "null argument");
  if (nx < 1 || ny < 1) throw Error(MS_E_INVALID, "element counts must be positive");
  if (!(nu >= 0.0 && nu < 0.5)) throw Error(MS_E_INVALID, "Poisson ratio outside [0, 0.5)");
  if (n_free <= 0) throw Error(MS_E_INVALID, "empty free-dof set");
  MS_CUDA(cudaSetDevice(ctx->device));
  std::unique_ptr<ms_problem> P(new ms_problem());
  P->ctx = ctx;
  P->g.nx = nx;
  P->g.ny = ny;
  P->g.nnx = nx + 1;
  P->g.n_nodes = (int64_t)(nx + 1) * (ny + 1);
  P->g.h = h;
  P->nu = nu;
  P->n_full = 2 * P->g.n_nodes;
  P->n_free = n_free;
  if (n_free > P->n_full) throw Error(MS_E_INVALID, "more free dofs than dofs");
  unit_elasticity(nu, P->ke.k);
  const cudaStream_t st = ctx->st;
  const int64_t n_el = (int64_t)nx * ny;
  P->E.alloc(n_el);
  if (is_device_ptr(E))
    MS_CUDA(cudaMemcpyAsync(P->E.p, E, n_el * sizeof(double), cudaMemcpyDeviceToDevice, st));
  else
    P->E.upload(E, n_el, st);
  std::vector<int64_t> fd(n_free);
  if (is_device_ptr(free_dofs))
    MS_CUDA(cudaMemcpy(fd.data(), free_dofs, n_free * sizeof(int64_t), cudaMemcpyDeviceToHost));
  else
    std::memcpy(fd.data(), free_dofs, n_free * sizeof(int64_t));
  std::vector<uint8_t> mask(P->n_full, 0);
  for (int64_t i = 0; i < n_free; ++i) {
    if (fd[i] < 0 || fd[i] >= P->n_full || (i > 0 && fd[i] <= fd[i - 1]))
      throw Error(MS_E_INVALID, "free dofs must be sorted, unique and in range");
    mask[fd[i]] = 1;
  }
  P->free_dofs.upload(fd.data(), n_free, st);
  P->mask.upload(mask.data(), mask.size(), st);
  P->ensure_workspace();
  MS_CUDA(cudaStreamSynchronize(st));
  *out = P.release();
  MS_API_END(ctx)
}

int ms_problem_destroy(ms_problem* prob) {
  if (!prob) return MS_OK;
  cudaSetDevice(prob->ctx->device);
  cudaStreamSynchronize(prob->ctx->st);
  delete prob;
  return MS_OK;
}

int64_t ms_problem_n_free(const ms_problem* prob) { return prob ? prob->n_free : -1; }

int ms_problem_set_modulus(ms_problem* prob, const double* E) {
  MS_API_BEGIN
  if (!prob || !E) throw Error(MS_E_INVALID, "null argument");
  MS_CUDA(cudaSetDevice(prob->ctx->device));
  const int64_t n_el = (int64_t)prob->g.nx * prob->g.ny;
  MS_CUDA(cudaMemcpyAsync(prob->E.p, E, n_el * sizeof(double), cudaMemcpyDefault, prob->ctx->st));
  MS_CUDA(cudaStreamSynchronize(prob->ctx->st));
  MS_API_END(prob ? prob->ctx : nullptr)
}

int ms_operator_apply(ms_problem* P, const double* p, double* q) {
  MS_API_BEGIN
  if (!P || !p || !q) throw Error(MS_E_INVALID, "null argument");
  MS_CUDA(cudaSetDevice(P->ctx->device));
  load_free(P, p, P->tmp.p);
  launch_matvec(P->g, P->ke, P->E.p, P->mask.p, nullptr, P->tmp.p, nullptr, P->q.p, MV_PLAIN,
                nullptr, nullptr, nullptr, P->ctx->st, P->b_lo, row_hi(P));
  allgather_rows(P, P->q.p);
  store_free(P, P->q.p, q);
  MS_API_END(P ? P->ctx : nullptr)
}

int ms_precond_build(ms_problem* P, const ms_precond_opts* o, ms_precond** out) {
  MS_API_BEGIN
  if (!P || !o || !out) throw Error(MS_E_INVALID, "null argument");
  MS_CUDA(cudaSetDevice(P->ctx->device));
  const cudaStream_t st = P->ctx->st;
  const Grid& g = P->g;
  if (o->Nx < 1 || o->Ny < 1 || g.nx % o->Nx || g.ny % o->Ny)
    throw Error(MS_E_INVALID, "coarse mesh " + std::to_string(o->Nx) + "x" + std::to_string(o->Ny) +
                                  " not nested in fine mesh");
  if (o->n_max < 1) throw Error(MS_E_INVALID, "mode cap must be >= 1");
  if (o->n_max > kNeig - 1) throw Error(MS_E_INVALID, "n_max > 6 is not supported by the GPU eigensolver");
  if (o->level1_kind == MS_LEVEL1_BLOCKS && o->delta < 1)
    throw Error(MS_E_INVALID, "block level-1 needs overlap delta >= 1");
  if (o->local_solver != MS_LOCAL_BANDED && o->local_solver != MS_LOCAL_DENSE_INV)
    throw Error(MS_E_INVALID, "unknown local solver");
  if (o->coarse_solve != MS_COARSE_INVERSE && o->coarse_solve != MS_COARSE_CHOLESKY)
    throw Error(MS_E_INVALID, "unknown coarse solve");
  if (o->level1_operator != MS_L1_ELASTICITY && o->level1_operator != MS_L1_HEAT)
    throw Error(MS_E_INVALID, "unknown level-1 operator");
  const bool heat_l1 = o->level1_operator == MS_L1_HEAT;
  if (o->eig_kind != MS_EIG_HEAT && o->eig_kind != MS_EIG_ELASTICITY)
    throw Error(MS_E_INVALID, "unknown eigenproblem kind");
  const bool el = o->eig_kind == MS_EIG_ELASTICITY;
  if (el && o->enrich)
    throw Error(MS_E_INVALID, "rotation enrichment applies to heat bases, not the elasticity basis 'E'");
  const int nd = el ? 2 : 1;  // unknowns per node of the neighbourhood eigenproblems
  if (heat_l1 && o->local_solver != MS_LOCAL_BANDED)
    throw Error(MS_E_INVALID, "the heat level-1 uses the banded local solver");
  const int W = P->ctx->world(), R = P->ctx->rank();
  if (W > 1 && (o->level1_kind != MS_LEVEL1_BLOCKS || !o->use_coarse || o->Ny < W))
    throw Error(MS_E_INVALID, "multi-GPU strips need the block level-1 layout, a coarse level and Ny >= ranks");
  std::unique_ptr<ms_precond> pc(new ms_precond());
  pc->prob = P;
  pc->device = P->ctx->device;
  pc->st = P->ctx->st;
  pc->opts = *o;
  if (W > 1) {
    const char* e = getenv("MS_DIST_BITWISE");
    pc->bitwise = e && std::string(e) == "1";
  }
  if (o->heat_dirichlet_nodes && o->n_heat_dirichlet > 0)
    pc->heat_dir.assign(o->heat_dirichlet_nodes, o->heat_dirichlet_nodes + o->n_heat_dirichlet);
  pc->opts.heat_dirichlet_nodes = nullptr;
  pc->opts.snapshots = nullptr;
  if (o->randomized && (!o->snapshots || o->n_snapshots < 1 || o->n_snapshots + 3 > 32))
    throw Error(MS_E_INVALID, "randomized eigensolver needs 1..29 snapshots and the forcings array");
  DBuf<int> fail;
  fail.alloc(1);

  // ---------------- level 1 ----------------
  cudaEvent_t e0, e1, e2, e3;
  MS_CUDA(cudaEventCreate(&e0));
  MS_CUDA(cudaEventCreate(&e1));
  MS_CUDA(cudaEventCreate(&e2));
  MS_CUDA(cudaEventCreate(&e3));
  MS_CUDA(cudaEventRecord(e0, st));
  {
    std::vector<int> xlo, xhi, ylo, yhi;
    level1_axis(g.nx, o->Nx, o->level1_kind, o->delta, xlo, xhi);
    level1_axis(g.ny, o->Ny, o->level1_kind, o->delta, ylo, yhi);
    pc->NbX = (int)xlo.size();
    pc->NbY = (int)ylo.size();
    pc->nsys = pc->NbX * pc->NbY;
    // strip of subdomain rows owned by this rank (all of them on one rank)
    if (W > 1) {
      strip_rows(o->Ny, W, R, pc->J0, pc->J1);
    } else {
      pc->J0 = 0;
      pc->J1 = pc->NbY;
    }
    pc->s0 = pc->J0 * pc->NbX;
    pc->s1 = pc->J1 * pc->NbX;
    // coarse cells = coarse blocks (Ny rows whatever the level-1 layout)
    pc->C0 = W > 1 ? pc->J0 : 0;
    pc->C1 = W > 1 ? pc->J1 : o->Ny;
    if (W > 1) {
      const int mey = g.ny / o->Ny;
      P->rank_lo.assign(W, 0);
      P->rank_hi.assign(W, 0);
      for (int q = 0; q < W; ++q) {
        int a, b;
        strip_rows(o->Ny, W, q, a, b);
        P->rank_lo[q] = a * mey;
        P->rank_hi[q] = (b == o->Ny) ? g.ny : b * mey - 1;
      }
      P->b_lo = P->rank_lo[R];
      P->b_hi = P->rank_hi[R];
      pc->halo_rows = std::max(1, o->delta);
    }
    for (int J = 0; J < pc->NbY; ++J)
      for (int I = 0; I < pc->NbX; ++I) {
        BandSys s{};
        if (xhi[I] < xlo[I] || yhi[J] < ylo[J]) throw Error(MS_E_INVALID, "empty level-1 subdomain");
        band_setup(s, xlo[I], xhi[I], ylo[J], yhi[J], heat_l1 ? 1 : 2);
        if (heat_l1) s.nrhs = 2;
        pc->max_bw = std::max(pc->max_bw, s.bw);
        pc->hsys.push_back(s);
      }
    // Padded TMA ring for the elasticity bands (banded local solver, ring
    // sweeps): every system stored with the widest bandwidth so that all
    // columns share one stride S and the bands form one [columns][S] tensor
    // (boundary blocks are at most 2 band words narrower: zeros)
    pc->pad = !heat_l1 && o->local_solver == MS_LOCAL_BANDED && l1_ring_sweeps_enabled() &&
              l1_padded_ring_enabled() && pc->max_bw <= 8 * 32 - 1;
    if (pc->pad)
      for (BandSys& s : pc->hsys) s.bw = pc->max_bw;
    int64_t foff = 0, yoff = 0;
    for (int sid = 0; sid < (int)pc->hsys.size(); ++sid) {
      BandSys& s = pc->hsys[sid];
      s.foff = foff;  // factors stored for owned subdomains only
      s.yoff = yoff;
      // even offsets: the ring sweeps bulk-copy 16-byte aligned chunks
      if (sid >= pc->s0 && sid < pc->s1) foff += ((int64_t)s.n * (s.bw + 1) + 1) & ~(int64_t)1;
      yoff += (int64_t)s.n * s.nrhs;
    }
    std::vector<int> xcov((g.nx + 1) * 4, -1), ycov((g.ny + 1) * 4, -1);
    auto cover = [](const std::vector<int>& lo, const std::vector<int>& hi, int nn, std::vector<int>& cov) {
      for (int a = 0; a < nn; ++a) {
        int c = 0;
        for (int I = 0; I < (int)lo.size(); ++I)
          if (a >= lo[I] && a <= hi[I]) {
            if (c == 2) throw Error(MS_E_INVALID, "a node is covered by more than 2 subdomains per axis (overlap too large)");
            cov[a * 4 + c++] = I;
          }
      }
    };
    cover(xlo, xhi, g.nx + 1, xcov);
    cover(ylo, yhi, g.ny + 1, ycov);
    // Twisted (two-sided) level-1 factors when the per-GPU subdomain count is
    // too small to hide the sweeps' dependent chain (config 2,
    // config 3 at 8 GPUs); MS_L1_TWIST=0/1 forces it off/on.
    const int ns_own = pc->s1 - pc->s0;
    std::vector<BandSys> nat;  // natural band layout (assembly input)
    if (o->local_solver == MS_LOCAL_BANDED) {
      int tw_env = -1;
      if (const char* e = getenv("MS_L1_TWIST")) tw_env = std::atoi(e);
      bool ok = pc->max_bw <= 128;
      for (int q = pc->s0; q < pc->s1 && ok; ++q) ok = pc->hsys[q].n >= 4 * pc->hsys[q].bw;
      pc->min_bw = pc->max_bw;
      for (int q = pc->s0; q < pc->s1; ++q) pc->min_bw = std::min(pc->min_bw, pc->hsys[q].bw);
      ok = ok && ring_sweep_ok(std::max(1, div_up(pc->max_bw, 32)), pc->min_bw);
      pc->twisted = ok && (tw_env == 1 || (tw_env != 0 && ns_own <= twist_max_subdomains(pc->device)));
    }
    if (pc->twisted) {
      int64_t tw = 0, so = 0;
      for (int q = pc->s0; q < pc->s1; ++q) {
        BandSys& b = pc->hsys[q];
        nat.push_back(b);
        const int S = b.bw + 1;
        b.m = (b.n - b.bw) / 2;
        const int nT = b.m + b.bw, nB = b.n - b.m;
        b.foff = tw;
        b.foffB = tw + (((int64_t)nT * S + 1) & ~(int64_t)1);
        tw = b.foffB + (((int64_t)nB * S + 1) & ~(int64_t)1);
        b.soff = so;
        so += ((int64_t)b.bw * b.bw + 1) & ~(int64_t)1;
      }
      foff = tw;
      pc->Sinv.alloc(so + 2);
    }
    pc->sys.upload(pc->hsys.data(), pc->hsys.size(), st);
    pc->xcov.upload(xcov.data(), xcov.size(), st);
    pc->ycov.upload(ycov.data(), ycov.size(), st);
    pc->Lc.alloc(foff + 2);  // + slack: an aligned chunk may read one word past the last column
    pc->ybuf.alloc(yoff);
    fail.zero(st);
    const int ns = pc->s1 - pc->s0;
    if (heat_l1) {
      launch_whole_node_check(g, P->mask.p, fail.p, st);
      int bad = 0;
      MS_CUDA(cudaMemcpyAsync(&bad, fail.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      MS_CUDA(cudaStreamSynchronize(st));
      if (bad) throw Error(MS_E_INVALID, "heat level-1 (HH variants) needs whole-node constraints");
    }
    pc->dense = o->local_solver == MS_LOCAL_DENSE_INV;
    pc->nrhs = heat_l1 ? 2 : 1;
    // one factor copy (column band, dot-form backward sweeps) on request
    // (MS_L1_COPIES=1): half the factor bytes, but the backward sweep is
    // issue-bound (config 3: level 1 2.12 ms vs 1.94 ms with both bands)
    {
      int copies_env = 2;
      if (const char* e = getenv("MS_L1_COPIES")) copies_env = std::atoi(e);
      pc->one_copy = !pc->dense && copies_env == 1 && l1_ring_sweeps_enabled() &&
                     ring_sweep_ok(std::max(1, div_up(pc->max_bw, 32)), pc->min_bw);
    }
    // Unit-diagonal L D L^T factors (MS_L1_UNIT=0/1): the pivot multiply leaves
    // the sweeps' dependent chain (shuffle + FMA per step instead of multiply +
    // shuffle + FMA); two-band ring sweeps in the plain (non-padded) layout.
    {
      int unit_env = -1;
      if (const char* e = getenv("MS_L1_UNIT")) unit_env = std::atoi(e);
      const bool can = !pc->dense && !pc->one_copy && !pc->pad && l1_ring_sweeps_enabled() &&
                       ring_sweep_ok(std::max(1, div_up(pc->max_bw, 32)), pc->min_bw);
      pc->unit = can && (unit_env == 1 || (unit_env != 0 && kL1UnitDefault));
    }
    if (pc->twisted) {
      // natural bands (assembly) -> top / bottom bands -> partial Cholesky of
      // both halves -> explicit inverse of the separator's Schur complement
      int64_t fn = 0;
      for (BandSys& b : nat) {
        b.foff = fn;
        fn += ((int64_t)b.n * (b.bw + 1) + 1) & ~(int64_t)1;
      }
      DBuf<BandSys> nat_d, half_d;
      nat_d.upload(nat.data(), nat.size(), st);
      DBuf<double> natband;  // natural bands (fn <= foff words)
      natband.alloc(fn + 2);
      if (heat_l1) {
        HeatParam hp{};
        heat_elements(g.h, hp);
        launch_l1_heat_assemble(g, hp.lap, P->E.p, P->mask.p, nat_d.p, ns, natband.p, st);
      } else {
        launch_l1_assemble(g, P->ke, P->E.p, P->mask.p, nat_d.p, ns, natband.p, st);
      }
      launch_twist_split(nat_d.p, pc->sys.p + pc->s0, ns, pc->max_bw, natband.p, pc->Lc.p, st);
      natband.release();
      if (!pc->one_copy) {
        pc->Lr.alloc(foff + 2);
        pc->Lr.zero(st);
      }
      std::vector<BandSys> halves(2 * (size_t)ns);
      const int64_t mb2 = (int64_t)pc->max_bw * pc->max_bw;
      for (int i = 0; i < ns; ++i) {
        const BandSys& b = pc->hsys[pc->s0 + i];
        BandSys t = b, u = b;
        t.n = b.m + b.bw;
        t.nelim = b.m;
        t.yoff = 2 * i * mb2;
        u.foff = b.foffB;
        u.n = b.n - b.m;
        u.nelim = u.n - b.bw;
        u.yoff = (2 * i + 1) * mb2;
        t.m = u.m = 0;
        halves[2 * i] = t;
        halves[2 * i + 1] = u;
      }
      half_d.upload(halves.data(), halves.size(), st);
      DBuf<double> schur;
      schur.alloc((size_t)2 * ns * mb2);
      launch_band_potrf(half_d.p, 2 * ns, pc->max_bw, pc->Lc.p, pc->Lr.p, fail.p, st, pc->unit ? 2 : 0, schur.p);
      check_fail(fail, st, "level-1 subdomain matrix");
      launch_schur_inverse(pc->sys.p + pc->s0, ns, pc->max_bw, schur.p, pc->Sinv.p, fail.p, st);
      check_fail(fail, st, "level-1 subdomain separator");
    } else if (!pc->dense) {
      if (heat_l1) {
        HeatParam hp{};
        heat_elements(g.h, hp);
        launch_l1_heat_assemble(g, hp.lap, P->E.p, P->mask.p, pc->sys.p + pc->s0, ns, pc->Lc.p, st);
      } else {
        launch_l1_assemble(g, P->ke, P->E.p, P->mask.p, pc->sys.p + pc->s0, ns, pc->Lc.p, st);
      }
      if (!pc->one_copy) {
        pc->Lr.alloc(foff + 2);
        pc->Lr.zero(st);
      }
      launch_band_potrf(pc->sys.p + pc->s0, ns, pc->max_bw, pc->Lc.p, pc->Lr.p, fail.p, st, pc->unit ? 2 : 0);
      check_fail(fail, st, "level-1 subdomain matrix");
    } else {
      launch_l1_assemble(g, P->ke, P->E.p, P->mask.p, pc->sys.p + pc->s0, ns, pc->Lc.p, st);
      // explicit inverses: band -> packed tiles, batched tiled Cholesky inverse
      int max_n = 0;
      for (const BandSys& b : pc->hsys) max_n = std::max(max_n, b.n);
      pc->dense_nt = div_up(max_n, kTile);
      const int64_t mw = packed_words(pc->dense_nt);
      pc->Xinv.alloc((size_t)ns * mw);
      const int B = std::min(ns, 256);
      DBuf<double> Pw, Ww;
      Pw.alloc((size_t)B * mw);
      Ww.alloc((size_t)B * mw);
      for (int b0 = 0; b0 < ns; b0 += B) {
        const int nb = std::min(B, ns - b0);
        launch_band_to_tiles(pc->sys.p, pc->s0 + b0, nb, pc->dense_nt, pc->Lc.p, Pw.p, st);
        dense_spd_inverse_batched(pc->dense_nt, nb, Pw.p, Ww.p, pc->Xinv.p + (size_t)b0 * mw, fail.p, st);
      }
      check_fail(fail, st, "level-1 subdomain matrix");
      pc->Lc.release();
    }
    {
      std::vector<int> xl(pc->NbX), yl(pc->NbY);
      for (int I = 0; I < pc->NbX; ++I) xl[I] = xhi[I] - xlo[I] + 1;
      for (int J = 0; J < pc->NbY; ++J) yl[J] = yhi[J] - ylo[J] + 1;
      std::vector<int64_t> yo(pc->nsys);
      for (int s2 = 0; s2 < pc->nsys; ++s2) yo[s2] = pc->hsys[s2].yoff;
      pc->xlo_d.upload(xlo.data(), xlo.size(), st);
      pc->ylo_d.upload(ylo.data(), ylo.size(), st);
      pc->xlen_d.upload(xl.data(), xl.size(), st);
      pc->ylen_d.upload(yl.data(), yl.size(), st);
      pc->yoff_d.upload(yo.data(), yo.size(), st);
    }
    pc->l1 = L1Dev{pc->NbX, pc->NbY, pc->xlo_d.p, pc->xlen_d.p, pc->ylo_d.p, pc->ylen_d.p,
                   pc->yoff_d.p, pc->xcov.p, pc->ycov.p, pc->ybuf.p};
    if (pc->pad && !pc->dense) {
      const int S = pc->max_bw + 1, T = std::max(1, div_up(pc->max_bw, 32));
      const int64_t cols = foff / S;
      make_band_map(&pc->maps.c, pc->Lc.p, cols, S, T);
      if (pc->Lr.p) make_band_map(&pc->maps.r, pc->Lr.p, cols, S, T);
      pc->maps.valid = true;
    }
    pc->info.n_subdomains = pc->nsys;
    pc->info.level1_twisted = pc->twisted ? 1 : 0;
    pc->info.n_subdomains_local = pc->s1 - pc->s0;
    pc->info.level1_unit = pc->unit ? 1 : 0;
    pc->info.level1_copies = pc->dense ? 0 : (pc->one_copy ? 1 : 2);
    pc->info.local_bytes = pc->dense ? (double)ns * packed_words(pc->dense_nt) * sizeof(double)
                                     : (double)(foff * (pc->one_copy ? 1 : 2) + (pc->twisted ? pc->Sinv.n : 0)) *
                                           sizeof(double);
  }
  MS_CUDA(cudaEventRecord(e1, st));

  // ---------------- coarse space ----------------
  pc->has_coarse = o->use_coarse != 0 && o->Nx >= 2 && o->Ny >= 2;
  if (pc->has_coarse) {
    CoarseDev& cd = pc->cd;
    cd.Nx = o->Nx;
    cd.Ny = o->Ny;
    cd.mex = g.nx / o->Nx;
    cd.mey = g.ny / o->Ny;
    cd.NLx = 2 * cd.mex + 1;
    cd.NLy = 2 * cd.mey + 1;
    cd.n_centers = (o->Nx - 1) * (o->Ny - 1);
    cd.enrich = o->enrich ? 1 : 0;
    cd.vec = el ? 1 : 0;
    cd.h = g.h;
    const int nc = cd.n_centers;
    const int NL = cd.NLx * cd.NLy;
    if (NL < 4 * kEigBlock || cd.mex < 4 || cd.mey < 4)
      throw Error(MS_E_INVALID, "coarse blocks must be >= 4 elements per side (block eigensolver)");
    // heat Dirichlet node mask
    std::vector<uint8_t> hd(g.n_nodes, 0);
    for (int64_t nid : pc->heat_dir) {
      if (nid < 0 || nid >= g.n_nodes) throw Error(MS_E_INVALID, "heat Dirichlet node out of range");
      hd[nid] = 1;
    }
    DBuf<uint8_t> hdir;
    hdir.upload(hd.data(), hd.size(), st);
    HeatParam hp{};
    heat_elements(g.h, hp);
    ElastParam ep{};
    for (int i = 0; i < 64; ++i) ep.ke[i] = P->ke.k[i];
    for (int i = 0; i < 16; ++i) ep.mel[i] = hp.mel[i];
    // shift: relative 1e-12 of the pencil's spectral bound:
    // heat 24/h^2; elasticity lambda_max(k0) / lambda_min(m_e) = lambda_max(k0) 36/h^2
    const double bound = el ? max_eig_sym8(P->ke.k) * 36.0 / (g.h * g.h) : 24.0 / (g.h * g.h);
    const double sigma = 1e-12 * bound;
    const int NLd = nd * NL;  // values per eigenvector
    pc->evals.alloc((size_t)nc * kNeig);
    DBuf<int> passes, neumann;
    passes.alloc(nc);
    neumann.alloc(nc);
    pc->nsel.alloc(nc);
    pc->psioff.alloc(nc);
    pc->psi.alloc((size_t)nc * o->n_max * NLd);
    std::vector<int64_t> h_psioff(nc, 0);
    pc->h_nsel.assign(nc, 0);
    // owned centre rows: [max(J0,1), min(J1, Ny)) (centre row J sits on block row J)
    {
      const int cj0 = std::max(pc->C0, 1), cj1 = std::min(pc->C1, o->Ny);
      pc->kc0 = (cj0 - 1) * (o->Nx - 1);
      pc->kc1 = std::max(pc->kc0, (cj1 - 1) * (o->Nx - 1));
    }
    const int batch = std::min(std::max(pc->kc1 - pc->kc0, 1), 1024);
    DBuf<BandSys> hsysd;
    DBuf<double> hLc, hLr, work, evecs, rsig, rF;
    // own centres' vectors are compacted with local offsets, then placed at
    // their global offsets once every rank's mode counts are known
    DBuf<double> psi_local_buf;
    double* psi_local = pc->psi.p;
    if (W > 1) {
      psi_local_buf.alloc((size_t)std::max(pc->kc1 - pc->kc0, 1) * o->n_max * NLd);
      psi_local = psi_local_buf.p;
    }
    DBuf<int64_t> psioff_local;
    psioff_local.alloc(nc);
    std::vector<int64_t> h_psioff_local(nc, 0);
    int64_t psi_cursor = 0;
    for (int k0 = pc->kc0; k0 < pc->kc1; k0 += batch) {
      const int nk = std::min(batch, pc->kc1 - k0);
      std::vector<BandSys> hs(nk);
      int64_t foff = 0;
      int mbw = 0;
      for (int kb = 0; kb < nk; ++kb) {
        const int k = k0 + kb;
        const int I = k % (o->Nx - 1) + 1, J = k / (o->Nx - 1) + 1;
        BandSys s{};
        band_setup(s, (I - 1) * cd.mex, (I + 1) * cd.mex, (J - 1) * cd.mey, (J + 1) * cd.mey, nd);
        s.foff = foff;
        foff += (int64_t)s.n * (s.bw + 1);
        mbw = std::max(mbw, s.bw);
        hs[kb] = s;
      }
      if (!hLc.p || hLc.n < (size_t)foff) {
        hLc.alloc(foff);
        hLr.alloc(foff);
        const int wb = o->randomized ? randomized_block(o->n_snapshots) : kEigBlock;
        work.alloc((size_t)nk * (2 * wb + (el ? 6 : 0)) * NLd);
        evecs.alloc((size_t)nk * kNeig * NLd);
      }
      hsysd.upload(hs.data(), nk, st);
      MS_CUDA(cudaMemsetAsync(hLr.p, 0, foff * sizeof(double), st));
      fail.zero(st);
      if (o->randomized) {
        // the reference's shift (spectral.py:133) and this batch's forcings
        if (rsig.n < (size_t)nk) rsig.alloc(nk);
        if (el)
          launch_rand_sigma_el(g, P->E.p, hdir.p, ep, hsysd.p, nk, rsig.p, st);
        else
          launch_rand_sigma(g, P->E.p, hdir.p, hp, hsysd.p, nk, rsig.p, st);
        const size_t fcount = (size_t)nk * o->n_snapshots * NLd;
        if (rF.n < fcount) rF.alloc(fcount);
        MS_CUDA(cudaMemcpyAsync(rF.p, o->snapshots + (size_t)k0 * o->n_snapshots * NLd, fcount * sizeof(double),
                                cudaMemcpyDefault, st));
      }
      if (el)
        launch_el_assemble(g, P->E.p, hdir.p, ep, sigma, hsysd.p, nk, hLc.p, st, o->randomized ? rsig.p : nullptr);
      else
        launch_heat_assemble(g, P->E.p, hdir.p, hp, sigma, hsysd.p, nk, hLc.p, st,
                             o->randomized ? rsig.p : nullptr);
      // elasticity pencils: LDL^T (the shifted rigid-body kernel leaves round-off level pivots)
      launch_band_potrf(hsysd.p, nk, mbw, hLc.p, hLr.p, fail.p, st, el ? 1 : 0);
      check_fail(fail, st, el ? "neighbourhood elasticity pencil (K + sigma M)" : "neighbourhood heat pencil (K + sigma M)");
      const int fixed = el ? 1 : o->fixed_rule;
      EigBatch eb{o->Nx, cd.mex, cd.mey, k0, nk, hsysd.p, hLc.p, hLr.p, work.p, pc->evals.p,
                  evecs.p, passes.p, neumann.p, o->n_max, o->gap_threshold, fixed, 1e-15 * bound};
      if (el && o->randomized)
        launch_randomized_el(g, P->E.p, hdir.p, ep, eb, mbw, rF.p, o->n_snapshots, st);
      else if (el)
        launch_subspace_el(g, P->E.p, hdir.p, ep, eb, mbw, 300, 1e-12, st);
      else if (o->randomized)
        launch_randomized(g, P->E.p, hdir.p, hp, eb, rF.p, o->n_snapshots, st);
      else
        launch_subspace(g, P->E.p, hdir.p, hp, eb, 300, 1e-12, st);
      launch_select(nc, pc->evals.p, o->n_max, o->gap_threshold, fixed, pc->nsel.p, st);
      std::vector<int> bsel(nk);
      MS_CUDA(cudaMemcpyAsync(bsel.data(), pc->nsel.p + k0, nk * sizeof(int), cudaMemcpyDeviceToHost, st));
      MS_CUDA(cudaStreamSynchronize(st));
      for (int kb = 0; kb < nk; ++kb) {
        h_psioff_local[k0 + kb] = psi_cursor;
        psi_cursor += (int64_t)bsel[kb] * NLd;
        pc->h_nsel[k0 + kb] = bsel[kb];
      }
      psioff_local.upload(h_psioff_local.data(), nc, st);
      if (el)
        launch_compact_psi_el(eb, cd.NLx, pc->nsel.p, psioff_local.p, psi_local, st);
      else
        launch_compact_psi(eb, cd.NLx, pc->nsel.p, psioff_local.p, psi_local, st);
    }
    if (W > 1) {
      // every owner's eigenvalues, mode counts and passes to every rank
      Comm* cm = P->ctx->comm.get();
      for (int q = 0; q < W; ++q) {
        int a, b;
        strip_rows(o->Ny, W, q, a, b);
        const int qk0 = (std::max(a, 1) - 1) * (o->Nx - 1);
        const int qk1 = std::max(qk0, (std::min(b, o->Ny) - 1) * (o->Nx - 1));
        if (qk1 <= qk0) continue;
        cm->broadcast(pc->evals.p + (size_t)qk0 * kNeig, (size_t)(qk1 - qk0) * kNeig * sizeof(double), q, st);
        cm->broadcast(pc->nsel.p + qk0, (size_t)(qk1 - qk0) * sizeof(int), q, st);
        cm->broadcast(passes.p + qk0, (size_t)(qk1 - qk0) * sizeof(int), q, st);
      }
      MS_CUDA(cudaMemcpyAsync(pc->h_nsel.data(), pc->nsel.p, nc * sizeof(int), cudaMemcpyDeviceToHost, st));
      MS_CUDA(cudaStreamSynchronize(st));
    }
    // global psi offsets (prefix over all centres)
    psi_cursor = 0;
    for (int k = 0; k < nc; ++k) {
      h_psioff[k] = psi_cursor;
      psi_cursor += (int64_t)pc->h_nsel[k] * NLd;
    }
    pc->psioff.upload(h_psioff.data(), nc, st);
    if (W > 1) {
      Comm* cm = P->ctx->comm.get();
      if (pc->kc1 > pc->kc0) {
        const int64_t n_own = h_psioff[pc->kc1 - 1] + (int64_t)pc->h_nsel[pc->kc1 - 1] * NLd - h_psioff[pc->kc0];
        MS_CUDA(cudaMemcpyAsync(pc->psi.p + h_psioff[pc->kc0], psi_local, n_own * sizeof(double),
                                cudaMemcpyDeviceToDevice, st));
      }
      for (int q = 0; q < W; ++q) {
        int a, b;
        strip_rows(o->Ny, W, q, a, b);
        const int qk0 = (std::max(a, 1) - 1) * (o->Nx - 1);
        const int qk1 = std::max(qk0, (std::min(b, o->Ny) - 1) * (o->Nx - 1));
        if (qk1 <= qk0) continue;
        const int64_t o0 = h_psioff[qk0], o1 = h_psioff[qk1 - 1] + (int64_t)pc->h_nsel[qk1 - 1] * NLd;
        cm->broadcast(pc->psi.p + o0, (size_t)(o1 - o0) * sizeof(double), q, st);
      }
    }
    {
      std::vector<int> hp_(nc);
      MS_CUDA(cudaMemcpyAsync(hp_.data(), passes.p, nc * sizeof(int), cudaMemcpyDeviceToHost, st));
      MS_CUDA(cudaStreamSynchronize(st));
      pc->max_pass = *std::max_element(hp_.begin(), hp_.end());
      double sum = 0;
      for (int v : hp_) sum += v;
      pc->info.mean_eig_passes = sum / std::max(1, nc);
    }
    MS_CUDA(cudaEventRecord(e2, st));
    // offsets
    std::vector<int> h_hoff(nc);
    int acc = 0;
    for (int k = 0; k < nc; ++k) {
      h_hoff[k] = acc;
      acc += (el ? 1 : 2) * pc->h_nsel[k];
    }
    cd.roff = acc;
    pc->N_c = acc + (cd.enrich ? nc : 0);
    cd.N_c = pc->N_c;
    pc->hoff.upload(h_hoff.data(), nc, st);
    pc->chi.alloc((size_t)nc * NL);
    cd.nsel = pc->nsel.p;
    cd.hoff = pc->hoff.p;
    cd.psioff = pc->psioff.p;
    cd.psi = pc->psi.p;
    cd.chi = pc->chi.p;
    launch_pou_table(g, cd, pc->chi.p, st);
    pc->chi4.alloc((size_t)g.n_nodes * 4);
    pc->psi4.alloc((size_t)g.n_nodes * 4);
    pc->rpart.alloc((size_t)o->Nx * o->Ny * 4 * kSlots);
    pc->rpart.zero(st);
    launch_node_tables(g, cd, pc->chi4.p, pc->psi4.p, st);
    cd.chi4 = pc->chi4.p;
    cd.psi4 = pc->psi4.p;
    cd.rpart = pc->rpart.p;
    // constant mode 0 per centre (pure Neumann neighbourhoods): their cells
    // rebuild psi4 = chi4 * value instead of reading it (MS_PSI0_CONST=0: off)
    cd.psi0c = nullptr;
    cd.chi_src = nullptr;
    {
      // cells with bitwise identical chi4 records read one shared copy (MS_CHI_DEDUP=0: off)
      const char* e = getenv("MS_CHI_DEDUP");
      if (!cd.vec && !(e && std::atoi(e) == 0)) {
        pc->chi_src.alloc((size_t)o->Nx * o->Ny);
        launch_chi_dedup(g, cd, pc->chi_src.p, st);
        cd.chi_src = pc->chi_src.p;
      }
    }
    {
      const char* e = getenv("MS_PSI0_CONST");
      if (!cd.vec && !(e && std::atoi(e) == 0)) {
        pc->psi0c.alloc(nc);
        launch_psi0_const(cd, pc->psi0c.p, st);
        cd.psi0c = pc->psi0c.p;
      }
    }
    // K0 = R0 A R0^T, symmetrised, inverted
    const int N = pc->N_c;
    DBuf<double> K0;
    K0.alloc((size_t)N * N);
    K0.zero(st);
    const int ncta = std::max(1, std::min(pc->kc1 - pc->kc0, 148 * 4));
    DBuf<double> scratch;
    scratch.alloc((size_t)ncta * 4 * NL);
    // columns of the owned centres' basis functions; the sum over ranks is K0
    launch_k0_assemble(g, P->ke, P->E.p, P->mask.p, cd, K0.p, scratch.p, ncta, st, pc->kc0, pc->kc1);
    if (W > 1) P->ctx->comm->allreduce_sum(K0.p, (size_t)N * N, st);
    launch_symmetrize(N, K0.p, st);
    const int nt = div_up(N, kTile);
    pc->coarse_factor = o->coarse_solve == MS_COARSE_CHOLESKY;
    if (W > 1 && !pc->coarse_factor && !pc->bitwise) {  // balanced contiguous share of the packed tiles
      const int64_t ntl = packed_tiles(nt);
      pc->sym_t0 = ntl * R / W;
      pc->sym_t1 = ntl * (R + 1) / W;
    }
    pc->K0inv.alloc((size_t)packed_tiles(nt) * kTile * kTile);
    DBuf<double> inv_work;
    inv_work.alloc(dense_spd_inverse_work_bytes(N) / sizeof(double));
    fail.zero(st);
    if (pc->coarse_factor) {
      pc->K0dinv.alloc((size_t)nt * kTile * kTile);
      pc->trsv_t.alloc((size_t)nt * kTile);
      pc->trsv_y.alloc((size_t)nt * kTile);
      pc->trsv_sync.alloc(trsv_sync_ints(N));
      dense_cholesky(N, K0.p, pc->K0inv.p, pc->K0dinv.p, inv_work.p, fail.p, st);
    } else {
      dense_spd_inverse(N, K0.p, pc->K0inv.p, inv_work.p, fail.p, st);
    }
    check_fail(fail, st, "coarse operator: basis is rank deficient, K0");
    pc->f0.alloc(N + 1);  // + the ||r||^2 slot of the multi-rank PCG allreduce
    pc->y0.alloc(N);
    pc->part.alloc((size_t)packed_tiles(nt) * 2 * kTile);
    if ((size_t)N * N <= (size_t)4096 * 4096) {
      pc->K0keep.alloc((size_t)N * N);
      MS_CUDA(cudaMemcpyAsync(pc->K0keep.p, K0.p, (size_t)N * N * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    pc->h_evals.resize((size_t)nc * kNeig);
    MS_CUDA(cudaMemcpyAsync(pc->h_evals.data(), pc->evals.p, pc->h_evals.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, st));
    pc->info.coarse_bytes = (double)(psi_cursor + (int64_t)packed_tiles(nt) * kTile * kTile *
                                                      (pc->coarse_factor ? 2 : 1)) * sizeof(double);
  } else {
    MS_CUDA(cudaEventRecord(e2, st));
  }
  MS_CUDA(cudaEventRecord(e3, st));
  MS_CUDA(cudaStreamSynchronize(st));
  float t1 = 0, t2 = 0, t3 = 0;
  MS_CUDA(cudaEventElapsedTime(&t1, e0, e1));
  MS_CUDA(cudaEventElapsedTime(&t2, e1, e2));
  MS_CUDA(cudaEventElapsedTime(&t3, e1, e3));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  cudaEventDestroy(e3);
  pc->info.coarse_dim = pc->N_c;
  pc->info.n_centers = pc->has_coarse ? pc->cd.n_centers : 0;
  pc->info.max_eig_passes = pc->max_pass;
  pc->info.t_level1 = t1 * 1e-3;
  pc->info.t_eig = t2 * 1e-3;
  pc->info.t_coarse = t3 * 1e-3;
  *out = pc.release();
  MS_API_END(P ? P->ctx : nullptr)
}

int ms_precond_destroy(ms_precond* pc) {
  if (!pc) return MS_OK;
  cudaSetDevice(pc->device);
  cudaStreamSynchronize(pc->st);
  delete pc;
  return MS_OK;
}

int ms_precond_apply(ms_precond* pc, const double* r, double* z) {
  MS_API_BEGIN
  if (!pc || !r || !z) throw Error(MS_E_INVALID, "null argument");
  ms_problem* P = pc->prob;
  MS_CUDA(cudaSetDevice(P->ctx->device));
  load_free(P, r, P->r.p);
  precond_apply_full(pc, P->r.p, P->z.p, nullptr, nullptr);
  allgather_rows(P, P->z.p);
  store_free(P, P->z.p, z);
  MS_API_END(pc ? pc->prob->ctx : nullptr)
}

int ms_precond_apply_coarse(ms_precond* pc, const double* r, double* z) {
  MS_API_BEGIN
  if (!pc || !r || !z) throw Error(MS_E_INVALID, "null argument");
  if (!pc->has_coarse) throw Error(MS_E_STATE, "preconditioner has no coarse level");
  ms_problem* P = pc->prob;
  const cudaStream_t st = P->ctx->st;
  MS_CUDA(cudaSetDevice(P->ctx->device));
  load_free(P, r, P->r.p);
  const bool dist = P->ctx->world() > 1;
  launch_restrict_cells(P->g, pc->C0, pc->C1, pc->cd, P->r.p, nullptr, st);
  if (dist) {
    exchange_rpart(pc);
    MS_CUDA(cudaMemsetAsync(pc->f0.p, 0, pc->N_c * sizeof(double), st));
  }
  launch_restrict_reduce(pc->cd, pc->f0.p, nullptr, st, pc->kc0, pc->kc1);
  if (dist) P->ctx->comm->allreduce_sum(pc->f0.p, pc->N_c, st);
  coarse_solve(pc, nullptr, st);
  launch_combine(P->g, P->mask.p, nullptr, &pc->cd, pc->opts.Nx, pc->opts.Ny, pc->y0.p, P->r.p, P->z.p,
                 nullptr, nullptr, nullptr, st, pc->C0, pc->C1);
  allgather_rows(P, P->z.p);
  store_free(P, P->z.p, z);
  MS_API_END(pc ? pc->prob->ctx : nullptr)
}

int ms_precond_info_get(const ms_precond* pc, ms_precond_info* info, int* mode_counts,
                        double* eigenvalues) {
  MS_API_BEGIN
  if (!pc) throw Error(MS_E_INVALID, "null argument");
  if (info) *info = pc->info;
  if (mode_counts && pc->has_coarse)
    std::memcpy(mode_counts, pc->h_nsel.data(), pc->h_nsel.size() * sizeof(int));
  if (eigenvalues && pc->has_coarse)
    std::memcpy(eigenvalues, pc->h_evals.data(), pc->h_evals.size() * sizeof(double));
  MS_API_END(nullptr)
}

int ms_precond_bench(ms_precond* pc, int reps, double* ms) {
  MS_API_BEGIN
  if (!pc || !ms || reps < 1) throw Error(MS_E_INVALID, "bad argument");
  ms_problem* P = pc->prob;
  MS_CUDA(cudaSetDevice(P->ctx->device));
  const cudaStream_t st = P->ctx->st;
  cudaEvent_t e0, e1;
  MS_CUDA(cudaEventCreate(&e0));
  MS_CUDA(cudaEventCreate(&e1));
  auto timeit = [&](auto&& fn) {
    fn();  // warm
    MS_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < reps; ++i) fn();
    MS_CUDA(cudaEventRecord(e1, st));
    MS_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    MS_CUDA(cudaEventElapsedTime(&t, e0, e1));
    return (double)t / reps;
  };
  const Grid& g = P->g;
  double* r = P->r.p;
  for (int i = 0; i < MS_BENCH_N; ++i) ms[i] = 0.0;
  ms[MS_BENCH_MATVEC] = timeit([&] {
    launch_matvec(g, P->ke, P->E.p, P->mask.p, nullptr, r, nullptr, P->q.p, MV_PLAIN, nullptr, nullptr,
                  nullptr, st);
  });
  if (pc->nsys > 0)
    ms[MS_BENCH_LEVEL1] = timeit([&] {
      if (pc->dense)
        launch_l1_dense_apply(g, pc->sys.p + pc->s0, pc->s1 - pc->s0, pc->dense_nt, pc->Xinv.p, r, pc->ybuf.p,
                              nullptr, st);
      else
        launch_l1_solve(g, pc->sys.p + pc->s0, pc->s1 - pc->s0, pc->max_bw, pc->nrhs, pc->Lc.p, pc->Lr.p, r,
                        pc->ybuf.p, nullptr, st, pc->twisted ? pc->Sinv.p : nullptr, pc->min_bw, &pc->maps, pc->unit);
    });
  if (pc->has_coarse) {
    ms[MS_BENCH_RESTRICT] = timeit([&] {
      launch_restrict_cells(g, pc->C0, pc->C1, pc->cd, r, nullptr, st);
      launch_restrict_reduce(pc->cd, pc->f0.p, nullptr, st, pc->kc0, pc->kc1);
    });
    ms[MS_BENCH_COARSE_SOLVE] = timeit([&] {
      if (pc->coarse_factor)
        launch_trsv_packed(pc->N_c, pc->K0inv.p, pc->K0dinv.p, pc->f0.p, pc->trsv_t.p, pc->trsv_y.p, pc->y0.p,
                           pc->trsv_sync.p, nullptr, st);
      else
        launch_symv_packed(pc->N_c, pc->K0inv.p, pc->f0.p, pc->y0.p, pc->part.p, nullptr, st);
    });
    ms[MS_BENCH_COMBINE_COARSE] = timeit([&] {
      launch_combine(g, P->mask.p, nullptr, &pc->cd, pc->opts.Nx, pc->opts.Ny, pc->y0.p, r, P->z.p,
                     nullptr, nullptr, nullptr, st);
    });
  }
  if (pc->nsys > 0)
    ms[MS_BENCH_COMBINE_L1] = timeit([&] {
      launch_combine(g, P->mask.p, &pc->l1, nullptr, pc->opts.Nx, pc->opts.Ny, pc->y0.p, r, P->z.p,
                     nullptr, nullptr, nullptr, st);
    });
  ms[MS_BENCH_COMBINE] = timeit([&] {
    launch_combine(g, P->mask.p, pc->nsys > 0 ? &pc->l1 : nullptr, pc->has_coarse ? &pc->cd : nullptr,
                   pc->opts.Nx, pc->opts.Ny, pc->y0.p, r, P->z.p, nullptr, nullptr, nullptr, st);
  });
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  MS_API_END(pc ? pc->prob->ctx : nullptr)
}

int ms_precond_coarse_matrix(const ms_precond* pc, double* K0) {
  MS_API_BEGIN
  if (!pc || !K0) throw Error(MS_E_INVALID, "null argument");
  if (!pc->K0keep.p) throw Error(MS_E_STATE, "K0 is only retained for N_c <= 4096");
  MS_CUDA(cudaSetDevice(pc->prob->ctx->device));
  MS_CUDA(cudaMemcpy(K0, pc->K0keep.p, (size_t)pc->N_c * pc->N_c * sizeof(double), cudaMemcpyDeviceToHost));
  MS_API_END(nullptr)
}

int ms_pcg_solve(ms_problem* P, ms_precond* pc, const double* b, double tol, int maxit, double* x,
                 ms_report* rep, double* residuals, double* alphas, double* betas) {
  MS_API_BEGIN
  if (!P || !b || !x) throw Error(MS_E_INVALID, "null argument");
  if (!(tol > 0.0 && tol < 1.0)) throw Error(MS_E_INVALID, "tolerance must be in (0, 1)");
  if (maxit < 0) throw Error(MS_E_INVALID, "maxit must be >= 0");
  if (pc && pc->prob != P) throw Error(MS_E_INVALID, "preconditioner built for another problem");
  MS_CUDA(cudaSetDevice(P->ctx->device));
  const auto wall0 = std::chrono::steady_clock::now();
  const long long launches0 = ms_launch_counter();
  const cudaStream_t st = P->ctx->st;
  if (P->hcap < maxit + 1) {
    P->hres.alloc(maxit + 1);
    P->halpha.alloc(std::max(maxit, 1));
    P->hbeta.alloc(std::max(maxit, 1));
    P->hcap = maxit + 1;
    ++P->hist_gen;
  }
  // graphs captured against the previous history buffers must not be replayed
  auto drop = [](cudaGraphExec_t& g) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  };
  if (P->graph_gen != P->hist_gen) {
    drop(P->gexec);
    drop(P->gexec_prof);
    P->graph_gen = P->hist_gen;
  }
  if (pc && pc->graph_gen != P->hist_gen) {
    drop(pc->gexec);
    drop(pc->gexec_prof);
    pc->graph_gen = P->hist_gen;
  }
  // a profiling graph records the events of the mask it was captured with
  unsigned& pmask = pc ? pc->prof_mask : P->prof_mask;
  if (P->ctx->prof.on && pmask != P->ctx->prof.mask) {
    drop(pc ? pc->gexec_prof : P->gexec_prof);
    pmask = P->ctx->prof.mask;
  }
  load_free(P, b, P->r.p);  // r = b
  P->x.zero(st);
  P->p0.zero(st);
  P->p1.zero(st);
  const bool dist = P->ctx->world() > 1;
  if (dist && (!pc || !pc->has_coarse))
    throw Error(MS_E_INVALID, "multi-GPU solves need the two-level preconditioner");
  PcgScalars hs{};
  hs.tol = tol;
  hs.maxit = maxit;
  hs.first = 1;
  hs.dist = dist ? 1 : 0;
  hs.bitwise = (dist && pc && pc->bitwise) ? 1 : 0;
  hs.done = maxit == 0 ? 1 : 0;
  MS_CUDA(cudaMemcpyAsync(P->sc.p, &hs, sizeof(hs), cudaMemcpyHostToDevice, st));
  cudaEvent_t t0, t1;
  MS_CUDA(cudaEventCreate(&t0));
  MS_CUDA(cudaEventCreate(&t1));
  MS_CUDA(cudaEventRecord(t0, st));
  const int64_t n = P->n_full;
  launch_init_norm(n, P->r.p, P->sc.p, P->partials.p, P->hres.p, st);
  double* zp = pc ? P->z.p : P->r.p;
  if (pc)
    precond_apply_full(pc, P->r.p, P->z.p, P->sc.p, P->hbeta.p);
  else
    launch_rz(n, P->r.p, P->r.p, P->sc.p, P->partials.p, P->hbeta.p, st);
  int it = 0;
  int done = 0;
  const int chunk = kPcgChunk;
  auto launch_iter = [&](int i) {
    double* pold = (i & 1) ? P->p1.p : P->p0.p;
    double* pnew = (i & 1) ? P->p0.p : P->p1.p;
    Prof& pf = P->ctx->prof;
    const bool bitwise = dist && pc && pc->bitwise;
    cudaEvent_t a = pf.begin(MS_PROF_MATVEC, i, st);
    if (bitwise) dist_zero_partials(P, matvec_partial_slots(P->g));
    launch_matvec(P->g, P->ke, P->E.p, P->mask.p, zp, pold, pnew, P->q.p, MV_PCG, P->sc.p,
                  P->partials.p, P->halpha.p, st, P->b_lo, row_hi(P));
    pf.end(MS_PROF_MATVEC, i, st, a);
    if (bitwise)
      dist_reduce_bitwise(P, PART_PQ, matvec_partial_slots(P->g), matvec_threads(), P->halpha.p);
    else if (dist)
      dist_finalize(P, PART_PQ, P->halpha.p);
    a = pf.begin(MS_PROF_UPDATE, i, st);
    const bool fused = pc && pc->has_coarse;
    if (bitwise) dist_zero_partials(P, pc->opts.Nx * pc->opts.Ny);
    if (fused)  // residual update + coarse restriction partials in one pass
      launch_update_restrict(P->g, pc->C0, pc->C1, P->x.p, pnew, P->r.p, P->q.p, pc->cd, P->sc.p,
                             P->partials.p, P->hres.p, st);
    else
      launch_pcg_update(n, P->x.p, pnew, P->r.p, P->q.p, P->sc.p, P->partials.p, P->hres.p, st);
    pf.end(MS_PROF_UPDATE, i, st, a);
    // multi-rank with a coarse space: ||r||^2 is summed inside the f0 allreduce
    // (one collective fewer per iteration); the level-1 sweeps of the converged
    // iteration then still run, their output unused
    const bool rr_in_f0 = dist && fused && !bitwise;
    if (dist) {
      if (bitwise)
        dist_reduce_bitwise(P, PART_RR, pc->opts.Nx * pc->opts.Ny, update_restrict_threads(pc->cd), P->hres.p);
      else if (!rr_in_f0)
        dist_finalize(P, PART_RR, P->hres.p);
      // level-1 subdomains reach delta rows out (without a preconditioner the
      // next matvec needs r (= z) on one halo row); the restriction partials
      // of the boundary cell row travel in the same group
      Comm* c = P->ctx->comm.get();
      Xfer x[6];
      row_halo_xfers(P, c, P->r.p, pc ? pc->halo_rows : 1, x);
      int nx = 4;
      if (fused) {
        rpart_xfers(pc, c, x + 4);
        nx = 6;
      }
      c->sendrecv(x, nx, st);
    }
    if (dist && fused) {
      precond_apply_dist_grouped(pc, P->r.p, P->z.p, P->sc.p, P->hbeta.p, i, rr_in_f0 ? P->hres.p : nullptr);
    } else if (pc) {
      precond_apply_full(pc, P->r.p, P->z.p, P->sc.p, P->hbeta.p, i, fused, rr_in_f0 ? P->hres.p : nullptr);
    } else {
      a = pf.begin(MS_PROF_COMBINE, i, st);
      launch_rz(n, P->r.p, P->r.p, P->sc.p, P->partials.p, P->hbeta.p, st);
      pf.end(MS_PROF_COMBINE, i, st, a);
    }
  };
  // A chunk of iterations (even length, so the p double-buffer parity is the
  // same at every chunk start) is captured once per (problem, preconditioner)
  // into a CUDA graph and replayed; the device `done` flag turns iterations
  // past convergence into no-ops.  Profiling mode launches directly.
  Prof& prof = P->ctx->prof;
  const bool use_graph = maxit >= chunk && (!dist || P->ctx->comm->capturable());
  cudaGraphExec_t& gexec = prof.on ? (pc ? pc->gexec_prof : P->gexec_prof) : (pc ? pc->gexec : P->gexec);
  long long& gkernels = prof.on ? (pc ? pc->gexec_prof_kernels : P->gexec_prof_kernels)
                                : (pc ? pc->gexec_kernels : P->gexec_kernels);
  if (use_graph && !gexec) {
    cudaGraph_t graph;
    prof.capturing = true;
    prof.captured.clear();
    const long long c0 = ms_launch_counter();
    MS_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < chunk; ++i) launch_iter(i);
    MS_CUDA(cudaStreamEndCapture(st, &graph));
    gkernels = ms_launch_counter() - c0;  // captured, not launched: counted per replay
    ms_launch_counter() = c0;
    prof.capturing = false;
    MS_CUDA(cudaGraphInstantiate(&gexec, graph, 0));
    MS_CUDA(cudaGraphDestroy(graph));
    if (prof.on) (pc ? pc->captured : P->captured) = prof.captured;
  }
  if (prof.on && use_graph) prof.captured = pc ? pc->captured : P->captured;
  while (!done && it < maxit) {
    if (use_graph && it + chunk <= maxit) {
      MS_CUDA(cudaGraphLaunch(gexec, st));
      ms_launch_counter() += gkernels;
      if (prof.on) prof.replayed(it);
      it += chunk;
    } else {
      const int upto = std::min(maxit, it + chunk);
      for (; it < upto; ++it) launch_iter(it);
    }
    MS_CUDA(cudaMemcpyAsync(&hs, P->sc.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    MS_CUDA(cudaStreamSynchronize(st));
    done = hs.done;
    // the iteration that converged keeps its launches; later ones were no-ops
    P->ctx->prof.flush(done ? hs.iter : it);
  }
  MS_CUDA(cudaEventRecord(t1, st));
  MS_CUDA(cudaMemcpyAsync(&hs, P->sc.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
  allgather_rows(P, P->x.p);
  store_free(P, P->x.p, x);
  float ms = 0.f;
  MS_CUDA(cudaEventElapsedTime(&ms, t0, t1));
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  const int iters = hs.iter;
  if (residuals) MS_CUDA(cudaMemcpy(residuals, P->hres.p, (iters + 1) * sizeof(double), cudaMemcpyDefault));
  if (alphas && iters > 0) MS_CUDA(cudaMemcpy(alphas, P->halpha.p, iters * sizeof(double), cudaMemcpyDefault));
  // the reference records beta after every non-final iteration: k - 1 on
  // convergence, k when maxit stops an unconverged solve (krylov.py:123-127)
  const int nbeta = hs.converged ? iters - 1 : iters;
  if (betas && nbeta > 0) MS_CUDA(cudaMemcpy(betas, P->hbeta.p, nbeta * sizeof(double), cudaMemcpyDefault));
  if (rep) {
    // counted at every launch site (graph replays add their kernel nodes);
    // includes the no-op kernels of a chunk's iterations past convergence
    rep->kernel_launches = ms_launch_counter() - launches0;
    rep->iterations = iters;
    rep->converged = hs.converged;
    rep->final_residual = hs.res;
    rep->t_solve = ms * 1e-3;
    rep->t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  }
  MS_API_END(P ? P->ctx : nullptr)
}

// ---------------------------------------------------------------------------
// Generic PCG (the reference's duck-typed seams, krylov.py:73-78, 90):
// any operator (the Q1 problem, a CSR matrix on the device, a host callback)
// with any preconditioner (none, the two-level one, a host callback).  The
// Krylov vectors, dot products and scalar recurrences stay on the device; a
// callback sees host copies of its input / output.

struct ms_csr {
  ms_ctx* ctx = nullptr;
  int64_t n = 0, nnz = 0;
  DBuf<int64_t> indptr;
  DBuf<int> indices;
  DBuf<double> data, vin, vout;
};

int ms_csr_create(ms_ctx* ctx, int64_t n, const int64_t* indptr, const int* indices, const double* data,
                  ms_csr** out) {
  MS_API_BEGIN
  if (!ctx || !indptr || !out || n < 1) throw Error(MS_E_INVALID, "null argument or empty matrix");
  MS_CUDA(cudaSetDevice(ctx->device));
  const int64_t nnz = indptr[n];
  if (indptr[0] != 0 || nnz < 0 || (nnz > 0 && (!indices || !data)))
    throw Error(MS_E_INVALID, "malformed CSR row pointers");
  for (int64_t i = 0; i < n; ++i)
    if (indptr[i + 1] < indptr[i]) throw Error(MS_E_INVALID, "CSR row pointers must be non-decreasing");
  for (int64_t e = 0; e < nnz; ++e)
    if (indices[e] < 0 || indices[e] >= n) throw Error(MS_E_INVALID, "CSR column index out of range");
  auto A = std::make_unique<ms_csr>();
  A->ctx = ctx;
  A->n = n;
  A->nnz = nnz;
  A->indptr.upload(indptr, n + 1, ctx->st);
  A->indices.upload(indices, nnz, ctx->st);
  A->data.upload(data, nnz, ctx->st);
  MS_CUDA(cudaStreamSynchronize(ctx->st));
  *out = A.release();
  MS_API_END(ctx)
}

int ms_csr_destroy(ms_csr* A) {
  if (!A) return MS_OK;
  cudaSetDevice(A->ctx->device);
  cudaStreamSynchronize(A->ctx->st);
  delete A;
  return MS_OK;
}

int ms_csr_apply(ms_csr* A, const double* v, double* out) {
  MS_API_BEGIN
  if (!A || !v || !out) throw Error(MS_E_INVALID, "null argument");
  MS_CUDA(cudaSetDevice(A->ctx->device));
  const cudaStream_t st = A->ctx->st;
  const double* dv = v;
  if (!is_device_ptr(v)) {
    if (A->vin.n < (size_t)A->n) A->vin.alloc(A->n);
    MS_CUDA(cudaMemcpyAsync(A->vin.p, v, A->n * sizeof(double), cudaMemcpyHostToDevice, st));
    dv = A->vin.p;
  }
  double* dout = out;
  const bool host_out = !is_device_ptr(out);
  if (host_out) {
    if (A->vout.n < (size_t)A->n) A->vout.alloc(A->n);
    dout = A->vout.p;
  }
  launch_csr_spmv(A->n, A->nnz, A->indptr.p, A->indices.p, A->data.p, dv, dout, st);
  if (host_out) MS_CUDA(cudaMemcpyAsync(out, dout, A->n * sizeof(double), cudaMemcpyDeviceToHost, st));
  MS_CUDA(cudaStreamSynchronize(st));
  MS_API_END(A ? A->ctx : nullptr)
}

namespace {
struct PinnedBuf {
  double* p = nullptr;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void alloc(int64_t n) { MS_CUDA(cudaMallocHost(&p, n * sizeof(double))); }
};

// out = Op(in), both device vectors of length n
void linop_apply(ms_ctx* ctx, const ms_linop* op, int64_t n, const double* in, double* out, PinnedBuf& hin,
                 PinnedBuf& hout) {
  const cudaStream_t st = ctx->st;
  switch (op ? op->kind : MS_LINOP_NONE) {
    case MS_LINOP_NONE:
      MS_CUDA(cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      break;
    case MS_LINOP_PROBLEM: {
      const int rc = ms_operator_apply(static_cast<ms_problem*>(op->handle), in, out);
      if (rc != MS_OK) throw Error(rc, ctx->err.empty() ? "operator apply failed" : ctx->err);
      break;
    }
    case MS_LINOP_PRECOND: {
      const int rc = ms_precond_apply(static_cast<ms_precond*>(op->handle), in, out);
      if (rc != MS_OK) throw Error(rc, ctx->err.empty() ? "preconditioner apply failed" : ctx->err);
      break;
    }
    case MS_LINOP_CSR: {
      ms_csr* A = static_cast<ms_csr*>(op->handle);
      launch_csr_spmv(A->n, A->nnz, A->indptr.p, A->indices.p, A->data.p, in, out, st);
      break;
    }
    case MS_LINOP_CALLBACK: {
      if (!hin.p) hin.alloc(n);
      if (!hout.p) hout.alloc(n);
      MS_CUDA(cudaMemcpyAsync(hin.p, in, n * sizeof(double), cudaMemcpyDeviceToHost, st));
      MS_CUDA(cudaStreamSynchronize(st));
      const int rc = op->fn(op->user, hin.p, hout.p, n);
      if (rc != 0) throw Error(MS_E_CALLBACK, "operator / preconditioner callback failed");
      MS_CUDA(cudaMemcpyAsync(out, hout.p, n * sizeof(double), cudaMemcpyHostToDevice, st));
      break;
    }
    default:
      throw Error(MS_E_INVALID, "unknown ms_linop kind");
  }
}

int64_t linop_dim(const ms_linop* op) {
  if (!op) return -1;
  switch (op->kind) {
    case MS_LINOP_PROBLEM: return op->handle ? static_cast<ms_problem*>(op->handle)->n_free : -1;
    case MS_LINOP_PRECOND: return op->handle ? static_cast<ms_precond*>(op->handle)->prob->n_free : -1;
    case MS_LINOP_CSR: return op->handle ? static_cast<ms_csr*>(op->handle)->n : -1;
    default: return -1;
  }
}
}  // namespace

int ms_pcg_solve_generic(ms_ctx* ctx, int64_t n, const ms_linop* A, const ms_linop* M, const double* b,
                         double tol, int maxit, double* x, ms_report* rep, double* residuals, double* alphas,
                         double* betas) {
  MS_API_BEGIN
  if (!ctx || !A || !b || !x || n < 1) throw Error(MS_E_INVALID, "null argument");
  if (!(tol > 0.0 && tol < 1.0)) throw Error(MS_E_INVALID, "tolerance must be in (0, 1)");
  if (maxit < 0) throw Error(MS_E_INVALID, "maxit must be >= 0");
  if (A->kind == MS_LINOP_NONE || A->kind == MS_LINOP_PRECOND) throw Error(MS_E_INVALID, "A must be an operator");
  if (M && M->kind != MS_LINOP_NONE && M->kind != MS_LINOP_PRECOND && M->kind != MS_LINOP_CALLBACK)
    throw Error(MS_E_INVALID, "M must be none, a two-level preconditioner or a callback");
  if ((A->kind == MS_LINOP_CALLBACK && !A->fn) || (M && M->kind == MS_LINOP_CALLBACK && !M->fn))
    throw Error(MS_E_INVALID, "callback operator without a function");
  for (const ms_linop* op : {A, M}) {
    const int64_t d = linop_dim(op);
    if (d >= 0 && d != n) throw Error(MS_E_INVALID, "operator dimension does not match the right-hand side");
    // native operands run on their own context's stream: it must be the solve's
    const ms_ctx* oc = !op || !op->handle ? ctx
                       : op->kind == MS_LINOP_PROBLEM ? static_cast<ms_problem*>(op->handle)->ctx
                       : op->kind == MS_LINOP_PRECOND ? static_cast<ms_precond*>(op->handle)->prob->ctx
                       : op->kind == MS_LINOP_CSR ? static_cast<ms_csr*>(op->handle)->ctx
                                                  : ctx;
    if (oc != ctx) throw Error(MS_E_INVALID, "operand created on another context");
  }
  if (ctx->world() > 1) throw Error(MS_E_INVALID, "the generic PCG runs on one rank");
  MS_CUDA(cudaSetDevice(ctx->device));
  const auto wall0 = std::chrono::steady_clock::now();
  const long long launches0 = ms_launch_counter();
  const cudaStream_t st = ctx->st;
  const bool precond = M && M->kind != MS_LINOP_NONE;
  DBuf<double> xd, r, p, z, q, partials, hres, halpha, hbeta;
  DBuf<PcgScalars> sc;
  xd.alloc(n);
  r.alloc(n);
  p.alloc(n);
  q.alloc(n);
  if (precond) z.alloc(n);
  partials.alloc(reduce_blocks() + 8);
  hres.alloc(maxit + 1);
  halpha.alloc(std::max(maxit, 1));
  hbeta.alloc(std::max(maxit, 1));
  sc.alloc(1);
  PinnedBuf hin, hout;
  MS_CUDA(cudaMemcpyAsync(r.p, b, n * sizeof(double), cudaMemcpyDefault, st));  // r = b
  xd.zero(st);
  p.zero(st);
  PcgScalars hs{};
  hs.tol = tol;
  hs.maxit = maxit;
  hs.first = 1;
  hs.done = maxit == 0 ? 1 : 0;
  MS_CUDA(cudaMemcpyAsync(sc.p, &hs, sizeof(hs), cudaMemcpyHostToDevice, st));
  cudaEvent_t t0, t1;
  MS_CUDA(cudaEventCreate(&t0));
  MS_CUDA(cudaEventCreate(&t1));
  MS_CUDA(cudaEventRecord(t0, st));
  launch_init_norm(n, r.p, sc.p, partials.p, hres.p, st);
  auto poll = [&]() {
    MS_CUDA(cudaMemcpyAsync(&hs, sc.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    MS_CUDA(cudaStreamSynchronize(st));
  };
  // callbacks synchronise every iteration anyway; device-only operators are polled every 8
  const bool host_side = A->kind == MS_LINOP_CALLBACK || (precond && M->kind == MS_LINOP_CALLBACK);
  const int every = host_side ? 1 : 8;
  poll();  // zero right-hand side: converged before the first apply
  double* zp = precond ? z.p : r.p;
  if (!hs.done) {
    if (precond) linop_apply(ctx, M, n, r.p, z.p, hin, hout);
    launch_rz(n, r.p, zp, sc.p, partials.p, hbeta.p, st);
  }
  int it = 0;
  while (!hs.done && it < maxit) {
    launch_direction(n, zp, p.p, sc.p, st);                       // p = z + beta p
    linop_apply(ctx, A, n, p.p, q.p, hin, hout);                  // q = A p
    launch_pq(n, p.p, q.p, sc.p, partials.p, halpha.p, st);       // alpha
    launch_pcg_update(n, xd.p, p.p, r.p, q.p, sc.p, partials.p, hres.p, st);  // x, r, ||r||
    ++it;
    if (host_side) {
      poll();
      if (hs.converged) break;  // the reference leaves before the next M apply (krylov.py:121-123)
    }
    if (precond) linop_apply(ctx, M, n, r.p, z.p, hin, hout);
    launch_rz(n, r.p, zp, sc.p, partials.p, hbeta.p, st);         // beta
    if (!host_side && (it % every == 0 || it == maxit)) poll();
  }
  MS_CUDA(cudaEventRecord(t1, st));
  poll();
  MS_CUDA(cudaMemcpyAsync(x, xd.p, n * sizeof(double), cudaMemcpyDefault, st));
  MS_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  MS_CUDA(cudaEventElapsedTime(&ms, t0, t1));
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  const int iters = hs.iter;
  if (residuals) MS_CUDA(cudaMemcpy(residuals, hres.p, (iters + 1) * sizeof(double), cudaMemcpyDefault));
  if (alphas && iters > 0) MS_CUDA(cudaMemcpy(alphas, halpha.p, iters * sizeof(double), cudaMemcpyDefault));
  const int nbeta = hs.converged ? iters - 1 : iters;
  if (betas && nbeta > 0) MS_CUDA(cudaMemcpy(betas, hbeta.p, nbeta * sizeof(double), cudaMemcpyDefault));
  if (rep) {
    rep->kernel_launches = ms_launch_counter() - launches0;
    rep->iterations = iters;
    rep->converged = hs.converged;
    rep->final_residual = hs.res;
    rep->t_solve = ms * 1e-3;
    rep->t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  }
  MS_API_END(ctx)
}

// ---------------------------------------------------------------------------
// Topology-optimisation caller

struct ms_filter {
  ms_ctx* ctx = nullptr;
  int nx = 0, ny = 0;
  DBuf<int2> off;
  DBuf<double> w, inv;
  FilterDev dev{};
};

// numpy's pairwise float64 summation (the reduction behind scipy's
// W.sum(axis=1) through np.add.reduceat): n < 8 sequential, n <= 128 eight
// accumulators, larger blocks split in two
static double np_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

// an ABI vector of n doubles on the device (host inputs are staged)
struct DevIn {
  const double* d = nullptr;
  DBuf<double> buf;
  DevIn(const double* p, int64_t n, cudaStream_t st) {
    if (is_device_ptr(p)) {
      d = p;
    } else {
      buf.upload(p, n, st);
      d = buf.p;
    }
  }
};
struct DevOut {
  double* user;
  double* d = nullptr;
  int64_t n;
  DBuf<double> buf;
  DevOut(double* p, int64_t n_, cudaStream_t) : user(p), n(n_) {
    if (is_device_ptr(p)) {
      d = p;
    } else {
      buf.alloc(n);
      d = buf.p;
    }
  }
  void finish(cudaStream_t st) {
    if (d != user) MS_CUDA(cudaMemcpyAsync(user, d, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    MS_CUDA(cudaStreamSynchronize(st));
  }
};

int ms_filter_create(ms_ctx* ctx, int nx, int ny, double h, double radius, ms_filter** out) {
  MS_API_BEGIN
  if (!ctx || !out) throw Error(MS_E_INVALID, "null argument");
  if (nx < 1 || ny < 1 || !(h > 0)) throw Error(MS_E_INVALID, "bad mesh");
  if (radius < 0) throw Error(MS_E_INVALID, "filter radius must be nonnegative");
  MS_CUDA(cudaSetDevice(ctx->device));
  const cudaStream_t st = ctx->st;
  // stencil (assembly.py:303-314): offsets with radius - h |d| > 0, weight max(0, .)
  int reach = radius > 0 ? (int)std::ceil(radius / h) - 1 : 0;
  reach = std::max(reach, 0);
  std::vector<int2> offs;
  std::vector<double> wts;
  for (int di = -reach; di <= reach; ++di)
    for (int dj = -reach; dj <= reach; ++dj) {
      const double dist = h * std::hypot((double)di, (double)dj);
      if (radius - dist > 0) {
        offs.push_back(make_int2(di, dj));
        wts.push_back(radius > 0 ? std::max(radius - dist, 0.0) : 1.0);
      }
    }
  if (offs.empty()) {
    offs.push_back(make_int2(0, 0));
    wts.push_back(radius > 0 ? std::max(radius - h * std::hypot(0.0, 0.0), 0.0) : 1.0);
  }
  // descending column order (dj, di): the stored order of the reference's rows
  std::vector<int> ord(offs.size());
  for (size_t o = 0; o < ord.size(); ++o) ord[o] = (int)o;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) {
    return offs[a].y != offs[b].y ? offs[a].y > offs[b].y : offs[a].x > offs[b].x;
  });
  std::vector<int2> soff(ord.size());
  std::vector<double> sw(ord.size());
  for (size_t o = 0; o < ord.size(); ++o) {
    soff[o] = offs[ord[o]];
    sw[o] = wts[ord[o]];
  }
  // row sums a[0] + pairwise(a[1:]) over ascending columns; rows only differ
  // by how the stencil is clipped at the edges, so memoise per clip class
  const int64_t n = (int64_t)nx * ny;
  std::vector<double> inv(n);
  std::vector<double> cache;
  const int R1 = reach + 1;
  cache.assign((size_t)R1 * R1 * R1 * R1, 0.0);
  std::vector<char> have(cache.size(), 0);
  std::vector<double> row;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int li = std::min(i, reach), ri = std::min(nx - 1 - i, reach);
      const int lj = std::min(j, reach), rj = std::min(ny - 1 - j, reach);
      const size_t key = (((size_t)li * R1 + ri) * R1 + lj) * R1 + rj;
      if (!have[key]) {
        row.clear();
        for (int o = (int)soff.size() - 1; o >= 0; --o) {  // ascending columns
          const int ik = i + soff[o].x, jk = j + soff[o].y;
          if (ik >= 0 && ik < nx && jk >= 0 && jk < ny) row.push_back(sw[o]);
        }
        cache[key] = row[0] + np_pairwise(row.data() + 1, (int64_t)row.size() - 1);
        have[key] = 1;
      }
      inv[(int64_t)j * nx + i] = 1.0 / cache[key];
    }
  std::unique_ptr<ms_filter> f(new ms_filter());
  f->ctx = ctx;
  f->nx = nx;
  f->ny = ny;
  f->off.upload(soff.data(), soff.size(), st);
  f->w.upload(sw.data(), sw.size(), st);
  f->inv.upload(inv.data(), inv.size(), st);
  MS_CUDA(cudaStreamSynchronize(st));
  f->dev = FilterDev{nx, ny, (int)soff.size(), f->off.p, f->w.p, f->inv.p};
  *out = f.release();
  MS_API_END(ctx)
}

int ms_filter_destroy(ms_filter* f) {
  MS_API_BEGIN
  if (f) {
    cudaSetDevice(f->ctx->device);
    delete f;
  }
  MS_API_END(nullptr)
}

static int filter_run(ms_filter* f, const double* x, double* y, bool adjoint) {
  MS_API_BEGIN
  if (!f || !x || !y) throw Error(MS_E_INVALID, "null argument");
  MS_CUDA(cudaSetDevice(f->ctx->device));
  const cudaStream_t st = f->ctx->st;
  const int64_t n = (int64_t)f->nx * f->ny;
  DevIn in(x, n, st);
  DevOut o(y, n, st);
  if (in.d == o.d) throw Error(MS_E_INVALID, "filter output must not alias its input");
  if (adjoint)
    launch_filter_adjoint(f->dev, in.d, o.d, st);
  else
    launch_filter_apply(f->dev, in.d, o.d, st);
  o.finish(st);
  MS_API_END(f ? f->ctx : nullptr)
}

int ms_filter_apply(ms_filter* f, const double* rho, double* out) { return filter_run(f, rho, out, false); }
int ms_filter_adjoint(ms_filter* f, const double* v, double* out) { return filter_run(f, v, out, true); }

int ms_problem_set_density(ms_problem* P, const double* rho_f, double p, double E_min, double E_max) {
  MS_API_BEGIN
  if (!P || !rho_f) throw Error(MS_E_INVALID, "null argument");
  if (p < 1) throw Error(MS_E_INVALID, "penalization exponent must be >= 1");
  MS_CUDA(cudaSetDevice(P->ctx->device));
  const cudaStream_t st = P->ctx->st;
  const int64_t n = (int64_t)P->g.nx * P->g.ny;
  DevIn in(rho_f, n, st);
  DBuf<int> bad;
  bad.alloc(1);
  bad.zero(st);
  launch_simp(n, in.d, p, E_min, E_max, P->E.p, bad.p, st);
  int hb = 0;
  MS_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  MS_CUDA(cudaStreamSynchronize(st));
  if (hb) throw Error(MS_E_INVALID, "density out of [0, 1]");
  MS_API_END(P ? P->ctx : nullptr)
}

int ms_compliance_sensitivity(ms_ctx* ctx, int nx, int ny, double nu, const double* u_full,
                              const double* f_full, const double* rho_f, double p, double E_min,
                              double E_max, double* g0, double* sens) {
  MS_API_BEGIN
  if (!ctx || !u_full || !f_full || !rho_f || !g0 || !sens) throw Error(MS_E_INVALID, "null argument");
  if (nx < 1 || ny < 1) throw Error(MS_E_INVALID, "bad mesh");
  MS_CUDA(cudaSetDevice(ctx->device));
  const cudaStream_t st = ctx->st;
  ctx->ensure_scratch();
  Grid g{nx, ny, nx + 1, (int64_t)(nx + 1) * (ny + 1), 1.0 / nx};
  const int64_t n_el = (int64_t)nx * ny, n_dofs = 2 * g.n_nodes;
  DevIn u(u_full, n_dofs, st), f(f_full, n_dofs, st), r(rho_f, n_el, st);
  DevOut o(sens, n_el, st);
  KeParam ke{};
  unit_elasticity(nu, ke.k);
  launch_dot(n_dofs, f.d, u.d, ctx->dval.p, ctx->red.p, ctx->ticket.p, st);
  launch_compliance_sens(g, ke, u.d, r.d, p, E_min, E_max, o.d, st);
  MS_CUDA(cudaMemcpyAsync(g0, ctx->dval.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  o.finish(st);
  MS_API_END(ctx)
}

int ms_dense_spd_solve(ms_ctx* ctx, int N, const double* A, const double* b, double* x, int mode) {
  MS_API_BEGIN
  if (!ctx || !A || !b || !x || N < 1) throw Error(MS_E_INVALID, "bad argument");
  if (mode != MS_COARSE_INVERSE && mode != MS_COARSE_CHOLESKY) throw Error(MS_E_INVALID, "unknown solve mode");
  MS_CUDA(cudaSetDevice(ctx->device));
  const cudaStream_t st = ctx->st;
  DevIn dA(A, (int64_t)N * N, st), db(b, N, st);
  DevOut dx(x, N, st);
  const int nt = div_up(N, kTile);
  DBuf<double> M, work;
  DBuf<int> fail;
  fail.alloc(1);
  fail.zero(st);
  M.alloc((size_t)packed_words(nt));
  work.alloc(dense_spd_inverse_work_bytes(N) / sizeof(double));
  if (mode == MS_COARSE_CHOLESKY) {
    DBuf<double> dinv, t, ys;
    DBuf<int> sync;
    dinv.alloc((size_t)nt * kTile * kTile);
    t.alloc((size_t)nt * kTile);
    ys.alloc((size_t)nt * kTile);
    sync.alloc(trsv_sync_ints(N));
    dense_cholesky(N, dA.d, M.p, dinv.p, work.p, fail.p, st);
    check_fail(fail, st, "dense matrix");
    launch_trsv_packed(N, M.p, dinv.p, db.d, t.p, ys.p, dx.d, sync.p, nullptr, st);
    dx.finish(st);
  } else {
    DBuf<double> part;
    part.alloc((size_t)packed_tiles(nt) * 2 * kTile);
    dense_spd_inverse(N, dA.d, M.p, work.p, fail.p, st);
    check_fail(fail, st, "dense matrix");
    launch_symv_packed(N, M.p, db.d, dx.d, part.p, nullptr, st);
    dx.finish(st);
  }
  MS_API_END(ctx)
}

int ms_dot(ms_ctx* ctx, int64_t n, const double* a, const double* b, double* out) {
  MS_API_BEGIN
  if (!ctx || !a || !b || !out || n < 0) throw Error(MS_E_INVALID, "bad argument");
  MS_CUDA(cudaSetDevice(ctx->device));
  const cudaStream_t st = ctx->st;
  ctx->ensure_scratch();
  DevIn da(a, n, st), db(b, n, st);
  launch_dot(n, da.d, db.d, ctx->dval.p, ctx->red.p, ctx->ticket.p, st);
  MS_CUDA(cudaMemcpyAsync(out, ctx->dval.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  MS_CUDA(cudaStreamSynchronize(st));
  MS_API_END(ctx)
}

int ms_oc_update(ms_ctx* ctx, int64_t n, const ms_filter* filt, const double* rho, const double* dg,
                 const double* volumes, double v_star, double move, double damping, double* rho_new,
                 int* evaluations) {
  MS_API_BEGIN
  if (!ctx || !rho || !dg || !volumes || !rho_new || n < 1) throw Error(MS_E_INVALID, "bad argument");
  if (filt && (int64_t)filt->nx * filt->ny != n) throw Error(MS_E_INVALID, "filter does not match the design");
  MS_CUDA(cudaSetDevice(ctx->device));
  const cudaStream_t st = ctx->st;
  ctx->ensure_scratch();
  DevIn r(rho, n, st), d(dg, n, st), v(volumes, n, st);
  DevOut o(rho_new, n, st);
  // measure(lam) = volumes . W candidate(lam) = (W^T volumes) . candidate(lam)
  DBuf<double> wv;
  const double* wvp = v.d;
  if (filt) {
    wv.alloc(n);
    launch_filter_adjoint(filt->dev, v.d, wv.p, st);
    wvp = wv.p;
  }
  DBuf<OcState> state;
  state.alloc(1);
  launch_oc_init(state.p, v_star, move, damping, st);
  OcState hs{};
  for (int launched = 0; launched < 64 + 200;) {
    for (int b = 0; b < 8 && launched < 64 + 200; ++b, ++launched)
      launch_oc_eval(n, r.d, d.d, v.d, wvp, state.p, ctx->red.p, ctx->ticket.p, st);
    MS_CUDA(cudaMemcpyAsync(&hs, state.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    MS_CUDA(cudaStreamSynchronize(st));
    if (hs.phase >= 2) break;
  }
  if (evaluations) *evaluations = hs.evals;
  if (hs.phase == 3) throw Error(MS_E_STATE, "OC bisection failed to bracket the volume constraint");
  launch_oc_final(n, r.d, d.d, v.d, state.p, o.d, st);
  o.finish(st);
  MS_API_END(ctx)
}

}  // extern "C"
