// Batched banded SPD kernels: level-1 band assembly, Cholesky, sweeps.
//
// Replaces the per-subdomain SuperLU factor/solve of the reference
// (`spla.splu(K_i).solve`, schwarz.py:97-109 build, :80-81 apply).  Each
// subdomain's unknowns are numbered node-interleaved along its short axis,
// which makes K_i a band of width 2*(short side)+3 (73 for the configs'
// 35x35-node subdomains); its Cholesky factor is 1.4 MB instead of the 24 MB
// of a packed dense inverse, so one apply streams ~8x fewer bytes.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "banded.cuh"

namespace msgpu {

void band_setup(BandSys& s, int a0, int a1, int b0, int b1, int ncomp) {
  s.a0 = a0;
  s.b0 = b0;
  s.w = a1 - a0 + 1;
  s.hgt = b1 - b0 + 1;
  s.fastx = s.w <= s.hgt ? 1 : 0;
  s.ncomp = ncomp;
  s.nrhs = 1;
  s.n = ncomp * s.w * s.hgt;
  const int fast = s.fastx ? s.w : s.hgt;
  int bw = ncomp == 2 ? 2 * fast + 3 : fast + 1;
  s.bw = std::max(0, std::min(bw, s.n - 1));
  s.foff = 0;
  s.yoff = 0;
}

// ---------------------------------------------------------------------------
// Level-1 band assembly: entry (row = k + j, col = k) of A[idx][:, idx].
// Element contributions are summed in ascending element order, the order in
// which the reference's COO->CSR conversion sums duplicates (assembly.py:185-196),
// so the band holds the same bits as the reference's restricted CSR.
__global__ void __launch_bounds__(256)
    k_l1_assemble(Grid g, KeParam ke, const double* __restrict__ E,
                  const uint8_t* __restrict__ mask, const BandSys* __restrict__ sys,
                  double* __restrict__ Lc) {
  const BandSys s = sys[blockIdx.x];
  const int S = s.bw + 1;
  const int64_t total = (int64_t)s.n * S;
  for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
    const int k = (int)(t / S), j = (int)(t % S);
    const int row = k + j;
    double v = 0.0;
    if (row < s.n) {
      int ak, bk, ar, br;
      band_node_of(s, k >> 1, ak, bk);
      band_node_of(s, row >> 1, ar, br);
      const int ck = k & 1, cr = row & 1;
      const int64_t gk = ck * g.n_nodes + (int64_t)bk * g.nnx + ak;
      const int64_t gr = cr * g.n_nodes + (int64_t)br * g.nnx + ar;
      if (!mask[gk] || !mask[gr]) {
        v = (row == k) ? 1.0 : 0.0;
      } else if (abs(ar - ak) <= 1 && abs(br - bk) <= 1) {
        const int ilo = max(max(ak, ar) - 1, 0), ihi = min(min(ak, ar), g.nx - 1);
        const int jlo = max(max(bk, br) - 1, 0), jhi = min(min(bk, br), g.ny - 1);
        for (int ej = jlo; ej <= jhi; ++ej)
          for (int ei = ilo; ei <= ihi; ++ei) {
            const int crn_k = (ak - ei) + (bk - ej) * 3 - 2 * (bk - ej) * (ak - ei);
            const int crn_r = (ar - ei) + (br - ej) * 3 - 2 * (br - ej) * (ar - ei);
            // corner numbering (0,0)->0 (1,0)->1 (1,1)->2 (0,1)->3
            v += E[(int64_t)ej * g.nx + ei] * ke.k[(cr * 4 + crn_r) * 8 + ck * 4 + crn_k];
          }
      }
    }
    Lc[s.foff + t] = v;
  }
}

void launch_l1_assemble(const Grid& g, const KeParam& ke, const double* E, const uint8_t* mask,
                        const BandSys* sys, int nsys, double* Lc, cudaStream_t st) {
  if (nsys == 0) return;
  { k_l1_assemble<<<nsys, 256, 0, st>>>(g, ke, E, mask, sys, Lc); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// Heat level-1 band: entry (k + j, k) of D[sidx][:, sidx] (schwarz.py:124-128),
// D the E-weighted Q1 Laplacian (assembly.py:223-233); same element order as
// the reference's duplicate summation.
__global__ void __launch_bounds__(256)
    k_l1_heat_assemble(Grid g, LapParam lp, const double* __restrict__ E,
                       const uint8_t* __restrict__ mask, const BandSys* __restrict__ sys,
                       double* __restrict__ Lc) {
  const BandSys s = sys[blockIdx.x];
  const int S = s.bw + 1;
  const int64_t total = (int64_t)s.n * S;
  for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
    const int k = (int)(t / S), j = (int)(t % S);
    const int row = k + j;
    double v = 0.0;
    if (row < s.n) {
      int ak, bk, ar, br;
      band_node_of(s, k, ak, bk);
      band_node_of(s, row, ar, br);
      const int64_t gk = (int64_t)bk * g.nnx + ak, gr = (int64_t)br * g.nnx + ar;
      if (!mask[gk] || !mask[gr]) {
        v = (row == k) ? 1.0 : 0.0;
      } else if (abs(ar - ak) <= 1 && abs(br - bk) <= 1) {
        const int ilo = max(max(ak, ar) - 1, 0), ihi = min(min(ak, ar), g.nx - 1);
        const int jlo = max(max(bk, br) - 1, 0), jhi = min(min(bk, br), g.ny - 1);
        for (int ej = jlo; ej <= jhi; ++ej)
          for (int ei = ilo; ei <= ihi; ++ei) {
            const int dk = ak - ei, ek = bk - ej, dr = ar - ei, er = br - ej;
            const int ck = dk + 3 * ek - 2 * dk * ek, cr = dr + 3 * er - 2 * dr * er;
            v += E[(int64_t)ej * g.nx + ei] * lp.lap[cr * 4 + ck];
          }
      }
    }
    Lc[s.foff + t] = v;
  }
}

void launch_l1_heat_assemble(const Grid& g, const double* lap, const double* E, const uint8_t* mask,
                             const BandSys* sys, int nsys, double* Lc, cudaStream_t st) {
  if (nsys == 0) return;
  LapParam lp;
  for (int i = 0; i < 16; ++i) lp.lap[i] = lap[i];
  { k_l1_heat_assemble<<<nsys, 256, 0, st>>>(g, lp, E, mask, sys, Lc); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

__global__ void k_whole_node_check(int64_t n_nodes, const uint8_t* __restrict__ mask, int* fail) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_nodes;
       i += (int64_t)gridDim.x * blockDim.x)
    if (mask[i] != mask[i + n_nodes]) *fail = 1;
}

void launch_whole_node_check(const Grid& g, const uint8_t* mask, int* fail, cudaStream_t st) {
  { k_whole_node_check<<<4 * 148, 256, 0, st>>>(g.n_nodes, mask, fail); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Banded Cholesky, one CTA per system.  A sliding window of the next bw+1
// columns lives in shared memory (column c in slot c % S); each step k folds
// column k into the window with a rank-1 update a_j1 a_j2 / d and retires it.
// ldl = 1: square-root-free L D L^T (pivots may be negative, e.g. round-off
// level pivots of shifted singular pencils); stored so that the same sweeps
// apply it: Lc holds the Schur column a_{k+j,k} with 1/d_k on the diagonal
// (forward sweep -> D^-1 L^-1 b), Lr the unit factor l_{k+j,k} with 1.
// ldl = 2: the same L D L^T of an SPD band (pivots must be positive) stored
// for the UNIT sweeps: both bands hold the unit factor, Lc with 1/d_k on the
// diagonal (applied once per row after the forward sweep), Lr with 1 -- the
// sweeps' dependent chain is then shuffle + FMA per step, no multiply.
__global__ void __launch_bounds__(256)
    k_band_potrf(const BandSys* __restrict__ sys, double* __restrict__ Lc,
                 double* __restrict__ Lr, int* fail, int ldl, double* __restrict__ schur) {
  extern __shared__ double smem[];
  const BandSys s = sys[blockIdx.x];
  const int bw = s.bw, S = bw + 1, n = s.n;
  const int ne = (s.nelim > 0 && s.nelim < n) ? s.nelim : n;  // columns eliminated
  double* W = smem;                                           // S*S
  short2* pairs = reinterpret_cast<short2*>(smem + S * S);    // bw(bw+1)/2
  const int npairs = bw * (bw + 1) / 2;
  if (threadIdx.x == 0) {
    int p = 0;
    for (int j2 = 1; j2 <= bw; ++j2)
      for (int j1 = j2; j1 <= bw; ++j1) pairs[p++] = make_short2((short)j1, (short)j2);
  }
  double* colc = Lc + s.foff;
  double* colr = Lr ? Lr + s.foff : nullptr;  // row band: only for the two-copy sweeps
  for (int t = threadIdx.x; t < S * S; t += blockDim.x) {
    const int c = t / S, j = t % S;
    W[t] = (c < n) ? colc[(int64_t)c * S + j] : 0.0;
  }
  __syncthreads();
  bool bad = false;
  for (int k = 0; k < ne; ++k) {
    const int sk = k % S;
    double d = W[sk * S];
    if (ldl == 1 ? !(d != 0.0 && isfinite(d)) : !(d > 0.0)) {
      bad = true;
      d = 1.0;
    }
    const double invd = 1.0 / d;
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
      const short2 jj = pairs[p];
      const int j1 = jj.x, j2 = jj.y;
      W[((k + j2) % S) * S + (j1 - j2)] -= W[sk * S + j1] * W[sk * S + j2] * invd;
    }
    __syncthreads();
    const double lkk = ldl ? 1.0 : sqrt(d), inv = 1.0 / lkk;
    for (int j = threadIdx.x; j < S; j += blockDim.x) {
      double vc, vr;
      if (ldl == 2) {
        vr = (j == 0) ? 1.0 : W[sk * S + j] * invd;
        vc = (j == 0) ? invd : vr;
      } else if (ldl) {
        vc = (j == 0) ? invd : W[sk * S + j];
        vr = (j == 0) ? 1.0 : W[sk * S + j] * invd;
      } else {
        vc = vr = (j == 0) ? inv : W[sk * S + j] * inv;
      }
      colc[(int64_t)k * S + j] = vc;
      if (Lr && k + j < n) colr[(int64_t)(k + j) * S + j] = vr;
      const int cn = k + S;  // next column into the freed slot
      W[sk * S + j] = (cn < n) ? colc[(int64_t)cn * S + j] : 0.0;
    }
    __syncthreads();
  }
  if (ne < n) {
    // partial factorisation (twisted level 1): the window holds the Schur
    // complement of the last cnt = n - ne unknowns; dump it, make the
    // remaining columns identity
    const int cnt = n - ne;
    double* out = schur + s.yoff;
    for (int t = threadIdx.x; t < cnt * cnt; t += blockDim.x) {
      const int i = t / cnt, i2 = t % cnt;
      const int lo = min(i, i2), d = abs(i - i2);
      out[t] = W[((ne + lo) % S) * S + d];
    }
    for (int t = threadIdx.x; t < cnt * S; t += blockDim.x) {
      const int k = ne + t / S, j = t % S;
      const double v = j == 0 ? 1.0 : 0.0;
      colc[(int64_t)k * S + j] = v;
      if (Lr && k + j < n) colr[(int64_t)(k + j) * S + j] = v;
    }
  }
  if (bad && threadIdx.x == 0) atomicCAS(fail, 0, (int)blockIdx.x + 1);
}

// top / bottom column bands of the twisted systems from the natural band
__global__ void __launch_bounds__(256)
    k_twist_split(const BandSys* __restrict__ nat, const BandSys* __restrict__ sys,
                  const double* __restrict__ band, double* __restrict__ Lc) {
  const BandSys s = sys[blockIdx.x];
  const int64_t fn = nat[blockIdx.x].foff;
  const int S = s.bw + 1, n = s.n, m = s.m, nT = m + s.bw, nB = n - m;
  for (int64_t t = threadIdx.x; t < (int64_t)nT * S; t += blockDim.x) {
    const int k = (int)(t / S), j = (int)(t % S);
    Lc[s.foff + t] = (k + j < nT) ? band[fn + t] : 0.0;  // separator block kept
  }
  for (int64_t t = threadIdx.x; t < (int64_t)nB * S; t += blockDim.x) {
    const int q = (int)(t / S), j = (int)(t % S);
    // bottom-local column q = natural column n-1-q; row q+j = natural n-1-q-j
    const int cn = n - 1 - q;
    const bool ok = q + j < nB && q < nB - s.bw;  // separator block of B is zero
    Lc[s.foffB + t] = ok ? band[fn + (int64_t)(cn - j) * S + j] : 0.0;
  }
}

void launch_twist_split(const BandSys* nat, const BandSys* sys, int nsys, int max_bw, const double* band_nat,
                        double* Lc, cudaStream_t st) {
  (void)max_bw;
  if (nsys == 0) return;
  { k_twist_split<<<nsys, 256, 0, st>>>(nat, sys, band_nat, Lc); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// Sinv = (W_T + flip(W_B))^-1 by in-place Gauss-Jordan with diagonal pivots
// (SPD: no pivoting needed); W_T at schur + 2 s max_bw^2, W_B max_bw^2
// after it, in the bottom system's reversed order.
__global__ void __launch_bounds__(256)
    k_schur_inverse(const BandSys* __restrict__ sys, const double* __restrict__ schur,
                    double* __restrict__ Sinv, int* fail, int stride) {
  extern __shared__ double A[];
  const BandSys s = sys[blockIdx.x];
  const int bw = s.bw;
  const double* WT = schur + (int64_t)blockIdx.x * 2 * stride;
  const double* WB = WT + stride;
  for (int t = threadIdx.x; t < bw * bw; t += blockDim.x) {
    const int i = t / bw, j = t % bw;
    A[t] = WT[t] + WB[(bw - 1 - i) * bw + (bw - 1 - j)];
  }
  bool bad = false;
  for (int k = 0; k < bw; ++k) {
    __syncthreads();
    double d = A[k * bw + k];
    if (!(d > 0.0)) {
      bad = true;
      d = 1.0;
    }
    const double inv = 1.0 / d;
    for (int t = threadIdx.x; t < bw * bw; t += blockDim.x) {
      const int i = t / bw, j = t % bw;
      if (i != k && j != k) A[t] -= A[i * bw + k] * A[k * bw + j] * inv;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < bw; t += blockDim.x) {
      if (t != k) {
        A[k * bw + t] *= inv;
        A[t * bw + k] = -A[t * bw + k] * inv;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) A[k * bw + k] = inv;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < bw * bw; t += blockDim.x) {
    const int i = t / bw, j = t % bw;
    Sinv[s.soff + t] = 0.5 * (A[t] + A[j * bw + i]);  // symmetric to round-off; keep it exact
  }
  if (bad && threadIdx.x == 0) atomicCAS(fail, 0, (int)blockIdx.x + 1);
}

void launch_schur_inverse(const BandSys* sys, int nsys, int max_bw, const double* schur, double* Sinv, int* fail,
                          cudaStream_t st) {
  if (nsys == 0) return;
  const size_t smem = (size_t)max_bw * max_bw * sizeof(double);
  if (smem > 220 * 1024) throw Error(-1, "separator too wide for the twisted level-1");
  MS_CUDA(cudaFuncSetAttribute(k_schur_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  { k_schur_inverse<<<nsys, 256, smem, st>>>(sys, schur, Sinv, fail, max_bw * max_bw); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

void launch_band_potrf(const BandSys* sys, int nsys, int max_bw, double* Lc, double* Lr, int* fail,
                       cudaStream_t st, int ldl, double* schur) {
  if (nsys == 0) return;
  const int S = max_bw + 1;
  const size_t smem = (size_t)S * S * sizeof(double) + (size_t)(max_bw * (max_bw + 1) / 2 + 1) * 4;
  if (smem > 220 * 1024) throw Error(-1, "band too wide for the shared-memory Cholesky window");
  MS_CUDA(cudaFuncSetAttribute(k_band_potrf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  { k_band_potrf<<<nsys, 256, smem, st>>>(sys, Lc, Lr, fail, ldl, schur); ms_count_launch(); }
  MS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Level-1 sweeps, one warp per subdomain, window held in registers
// (band_sweep, banded.cuh); the default kernel streams the band through
// shared-memory rings instead (k_l1_solve_ring below).
constexpr int kSolveWarps = 4;
#ifndef MS_PD_HEAT
#define MS_PD_HEAT 8
#endif
constexpr int kPDHeat = MS_PD_HEAT;

template <int T, int NR>
__global__ void __launch_bounds__(kSolveWarps * 32)
    k_l1_solve(Grid g, const BandSys* __restrict__ sys, int nsys, const double* __restrict__ Lc,
               const double* __restrict__ Lr, const double* __restrict__ r,
               double* __restrict__ ybuf, const int* done) {
  if (done && *(volatile const int*)done) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sid = blockIdx.x * kSolveWarps + warp;
  if (sid >= nsys) return;
  const BandSys s = sys[sid];
  double* y = ybuf + s.yoff;
  // gather R_s r (node-interleaved local order; NR = 2: scalar rows, 2 rhs)
  for (int i = lane; i < s.n * NR; i += 32) {
    const int ln = i >> 1, c = i & 1;
    int a, b;
    band_node_of(s, ln, a, b);
    y[i] = r[c * g.n_nodes + (int64_t)b * g.nnx + a];
  }
  __syncwarp();
  // narrow scalar bands: deeper prefetch keeps enough bytes in flight per warp
  constexpr int PD = NR == 2 ? kPDHeat : kPD;
  band_sweep<T, NR, PD, false>(Lc + s.foff, s.n, s.bw, y, lane);
  __syncwarp();
  band_sweep<T, NR, PD, true>(Lr + s.foff, s.n, s.bw, y, lane);
}

// ---------------------------------------------------------------------------
// Same sweeps with the band streamed through shared memory by the bulk-copy
// (TMA) engine: each warp owns a ring of kNst stages of kCh band columns; lane
// 0 re-arms a stage's mbarrier and issues one cp.async.bulk per chunk as soon
// as the chunk kNst back has been consumed.  The bytes in flight no longer
// cost registers (the prefetch ring of band_sweep does), so narrow bands (the
// heat level-1, 37 words per column) keep HBM busy too.
#ifndef MS_TMA_CH
#define MS_TMA_CH 8
#endif
#ifndef MS_TMA_NST
#define MS_TMA_NST 2  // 2 stages: 4 CTAs (16 warps) per SM; config 3 level 1 1.99 -> 1.94 ms vs 3 stages
#endif
#ifndef MS_TMA_WARPS
#define MS_TMA_WARPS 4
#endif
#ifndef MS_L1_MINB
#define MS_L1_MINB 3  // register budget sized for >= 3 resident CTAs per SM (~128 registers)
#endif
constexpr int kCh = MS_TMA_CH;  // band columns per stage (divides 32)
constexpr int kChWide = 16;    // per stage for launches of at most one CTA per SM (wide_chunks)
constexpr int kNst = MS_TMA_NST;  // default stages per warp (bandwidth-bound launches)
constexpr int kMaxNst = 8;        // deepest ring a launch may ask for (latency-bound launches, pick_nst)
constexpr int kTmaWarps = MS_TMA_WARPS;
static_assert(32 % kCh == 0, "stage width must divide 32");

struct Ring {
  double* buf;     // kNst stages of `stage` words
  uint64_t* bar;   // kNst mbarriers
  int stage;       // words per stage (even)
  int nst;         // stages of this launch (2..kMaxNst)
  uint32_t phase;  // parity bit per stage
};

// Padded ring (elasticity bands, S = bw + 1 even): every band column gets its
// own P = 32 (T + 1) word slot in the stage, words [S, P) of every slot and a
// 32-word guard before the first stage stay zero.  A sweep step then reads
// its R = T + 1 coefficients (band offsets 32 s + lane - u) and the pivot
// with unconditional loads at compile-time offsets: rows outside the band
// read zeros.  The copies are one bulk copy per column (S * 8 bytes, 16-byte
// aligned because S is even), issued by lanes 0..cnt-1.
template <int T>
__host__ __device__ constexpr int pad_slot_words() {
  return 32 * (T + 1);
}
constexpr int kPadGuard = 32;

// ring shared-memory header: kTmaWarps * kNst mbarriers, rounded to 16 words
// (the stages stay 128-byte aligned)
constexpr int kRingHeaderWords = (kTmaWarps * kMaxNst + 15) & ~15;  // 128-byte aligned stages (TMA boxes)

// per-warp ring words: kNst stages (+ the zero guard of the padded layout)
__host__ __device__ inline int ring_warp_words(int stage_words, bool pad, int nst) {
  return nst * stage_words + (pad ? kPadGuard : 0);
}

__device__ __forceinline__ void ring_init(Ring& rg, double* smem, int warp, int lane, int stage_words, int nst,
                                          bool pad = false) {
  rg.nst = nst;
  rg.bar = reinterpret_cast<uint64_t*>(smem) + warp * nst;
  double* base = smem + kRingHeaderWords + (size_t)warp * ring_warp_words(stage_words, pad, nst);
  rg.buf = base + (pad ? kPadGuard : 0);
  rg.stage = stage_words;
  rg.phase = 0;
  if (pad) {  // guard and slot tails must read zero; the copies never touch them
    for (int i = lane; i < ring_warp_words(stage_words, pad, nst); i += 32) base[i] = 0.0;
    __syncwarp();
  }
  if (lane == 0) {
    for (int st = 0; st < nst; ++st) mbar_init(rg.bar + st, 1);
    mbar_fence_init();
  }
}



// first physical column and count of chunk c (steps [c kCh, c kCh + cnt))
__device__ __forceinline__ void chunk_cols(bool rev, int n, int c, int& start, int& cnt, int ch = kCh) {
  const int k0 = c * ch;
  cnt = min(ch, n - k0);
  start = rev ? n - k0 - cnt : k0;
}

// padded stage fill: one 2-D TMA box of kCh columns x P words (the words
// past S zero-filled); all lanes call, lane 0 issues
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

template <bool REV, int P>
__device__ __forceinline__ void ring_issue_pad(Ring& rg, const CUtensorMap* map, int col0, int n, int c, int lane,
                                               int st) {
  if (lane != 0) return;
  int start, cnt;
  chunk_cols(REV, n, c, start, cnt);
  mbar_expect_tx(rg.bar + st, (uint32_t)(kCh * P * 8));
  tma_load_2d(rg.buf + (size_t)st * rg.stage, map, 0, col0 + start, rg.bar + st);
}

template <bool REV, int CH = kCh>
__device__ __forceinline__ void ring_issue(Ring& rg, const double* L, int n, int S, int c, int st) {
  int start, cnt;
  chunk_cols(REV, n, c, start, cnt, CH);
  const int64_t w0 = (int64_t)start * S;
  const int64_t a = w0 & ~(int64_t)1;  // 16-byte aligned source (L itself is)
  const uint32_t words = (uint32_t)((cnt * S + (int)(w0 - a) + 1) & ~1);
  MS_BCHECK(st >= 0 && st < rg.nst && cnt >= 1 && start >= 0 && start + cnt <= n);
  MS_BCHECK((int)words <= rg.stage);                          // the chunk fits its shared-memory stage
  MS_BCHECK(a >= 0 && a + (int64_t)words <= (int64_t)n * S + 2);  // and stays inside the system's band (+ slack)
  mbar_expect_tx(rg.bar + st, words * 8u);
  bulk_g2s(rg.buf + (size_t)st * rg.stage, L + a, words * 8u, rg.bar + st);
}

// ym(r): address of the NR values of the sweep's r-th row (r counts the
// sweep's own steps, i.e. already reversed for REV)
// CH: band columns per ring stage.  8 for bandwidth-bound launches (more
// resident CTAs); 16 when the launch fits one wave: the per-chunk work --
// mbarrier wait, warp sync, lane 0 re-arming the stage and issuing the next
// bulk copy -- sits on the warp's dependent stream, and halving the chunk
// count took config 2's twisted level 1 from 0.180 to 0.156 ms (32 columns
// per stage spill: 0.32 ms).  (Software-pipelining the steps -- step q + 1's
// loads issued inside step q's shuffle shadow -- measured the same, 0.159 ms.)
struct NoInput {};  // the sweep reads its right-hand side where it writes its result

// rd(r, c): value of the sweep's input row r, right-hand side c, when it is not
// stored at ym(r) yet -- the forward sweeps gather R_s r from the global vector
// as they go (one value per lane and 32 steps) instead of a separate gather
// pass that writes y and reads it back.
template <int T, int NR, bool REV, bool PAD, bool UNIT = false, int CH = kCh, class YMap, class RMap = NoInput>
__device__ __forceinline__ void band_sweep_ring(const double* __restrict__ L, int n, int bw, YMap ym,
                                                int lane, Ring& rg, const CUtensorMap* map = nullptr,
                                                int col0 = 0, RMap rd = RMap{}) {
  constexpr int R = T + 1;
  constexpr int P = pad_slot_words<T>();
  const int S = bw + 1;
  static_assert(32 % CH == 0 && (!PAD || CH == kCh), "stage width must divide 32; padded TMA boxes are kCh wide");
  const int nch = (n + CH - 1) / CH;
  if (PAD) {
    for (int c = 0; c < min(rg.nst, nch); ++c) ring_issue_pad<REV, P>(rg, map, col0, n, c, lane, c);
  } else if (lane == 0) {
    for (int c = 0; c < min(rg.nst, nch); ++c) ring_issue<REV, CH>(rg, L, n, S, c, c);
  }
  auto yat = [&](int r, int c) -> double* { return ym(r) + c; };
  auto input = [&](int r, int c) -> double {
    if constexpr (std::is_same<RMap, NoInput>::value)
      return *yat(r, c);
    else
      return rd(r, c);
  };

  double acc[NR][R], rnext[NR];
#pragma unroll
  for (int c = 0; c < NR; ++c) {
#pragma unroll
    for (int s = 0; s < R - 1; ++s) {
      const int r = 32 * s + lane;
      acc[c][s] = r < n ? input(r, c) : 0.0;
    }
    acc[c][R - 1] = 0.0;
    rnext[c] = (32 * (R - 1) + lane < n) ? input(32 * (R - 1) + lane, c) : 0.0;
  }

  int stc = 0;
  for (int k0 = 0; k0 < n; k0 += 32) {
#pragma unroll
    for (int c = 0; c < NR; ++c) {
      acc[c][R - 1] = rnext[c];
      const int r = k0 + 32 * R + lane;
      rnext[c] = r < n ? input(r, c) : 0.0;
    }
    double dsave = 0.0;  // 1/L_kk of this lane's row of the block
    double yfin[NR];     // PAD: the row's final value, captured at its pivot step
#pragma unroll
    for (int c = 0; c < NR; ++c) yfin[c] = 0.0;
#pragma unroll 1
    for (int h = 0; h < 32 && k0 + h < n; h += CH) {
      const int ch = (k0 + h) / CH;
      const int st = stc;  // ch % nst as a running counter (nst is a per-launch value)
      stc = (stc + 1 == rg.nst) ? 0 : stc + 1;
      mbar_wait(rg.bar + st, (rg.phase >> st) & 1u);
      rg.phase ^= 1u << st;
      int start, cnt;
      chunk_cols(REV, n, ch, start, cnt, CH);
      if (PAD) {
        // slot q of the stage = column start + q; this lane's coefficient of
        // step q (u = h + q) sits at slot(q) + lane - u
        const double* sb = rg.buf + (size_t)st * rg.stage;
        const double* sl = sb + (lane - h);
        auto stepP = [&](int q, int slot) {
          const int u = h + q;
          const double* colq = sb + slot * P;
          const double* a = sl + (slot * P - q);
          double m[R];
#pragma unroll
          for (int s2 = 0; s2 < R; ++s2) m[s2] = a[32 * s2];
          const double d = colq[0];
#pragma unroll
          for (int c = 0; c < NR; ++c) {
            const double wk = __shfl_sync(0xffffffffu, acc[c][0] * d, u);
            yfin[c] = (lane == u) ? wk : yfin[c];
#pragma unroll
            for (int s2 = 0; s2 < R; ++s2) acc[c][s2] = fma(-m[s2], wk, acc[c][s2]);
          }
        };
        if (cnt == CH) {
#pragma unroll
          for (int q = 0; q < CH; ++q) stepP(q, REV ? CH - 1 - q : q);
        } else {
#pragma unroll
          for (int q = 0; q < CH; ++q)
            if (q < cnt) stepP(q, REV ? cnt - 1 - q : q);
        }
        __syncwarp();  // every lane is done with this stage before it is refilled
        if (ch + rg.nst < nch) ring_issue_pad<REV, P>(rg, map, col0, n, ch + rg.nst, lane, st);
        continue;
      }
      const double* sb = rg.buf + (size_t)st * rg.stage + (int)(((int64_t)start * S) & 1);
      // Step u of the block: lane owns row k0 + 32 s + lane in slot s, i.e.
      // band offset j = 32 s + lane - u from the pivot row; rows outside
      // 1..bw get a zero coefficient (no selects on the update path).
      // (An address-select form -- masked-out slots read a zero slot, slots
      // 1..T-2 unpredicated, validity masks per chunk -- issues ~30% fewer
      // instructions per step but measured 4-15% slower: 0.39 -> 0.47 ms at
      // config 2, 1.92 -> 2.00 ms at config 3.)
      auto step = [&](int q) {
        const int u = h + q;
        const double* col = sb + (REV ? (cnt - 1 - q) : q) * S;
        const int jl = lane - u;
        double m[R];
        m[0] = lds_or_zero(col + jl, jl >= 1 && jl <= bw);
#pragma unroll
        for (int s = 1; s < R; ++s) m[s] = lds_or_zero(col + jl + 32 * s, jl + 32 * s <= bw);
        const double d = lds_or_zero(col, true);
        if (lane == u) dsave = d;
#pragma unroll
        for (int c = 0; c < NR; ++c) {
          // UNIT: unit-diagonal factor, the pivot row's accumulator is final as it stands
          const double wk = __shfl_sync(0xffffffffu, UNIT ? acc[c][0] : acc[c][0] * d, u);
#pragma unroll
          for (int s = 0; s < R; ++s) acc[c][s] = fma(-m[s], wk, acc[c][s]);
        }
      };
      if (cnt == CH) {
#pragma unroll
        for (int q = 0; q < CH; ++q) step(q);
      } else {
#pragma unroll
        for (int q = 0; q < CH; ++q)
          if (q < cnt) step(q);
      }
      __syncwarp();  // every lane is done with this stage before it is refilled
      if (lane == 0 && ch + rg.nst < nch) ring_issue<REV, CH>(rg, L, n, S, ch + rg.nst, st);
    }
    // slot 0 of lane L stopped changing at step L: it holds row k0+L's final
    // accumulator, and w = acc * (1/L_kk) exactly as the pivot step formed it
    // (PAD: the pivot lane's slot 0 takes one more, meaningless update; its
    // value was captured at the pivot step instead, the same product)
#pragma unroll
    for (int c = 0; c < NR; ++c) {
      if (k0 + lane < n) *yat(k0 + lane, c) = PAD ? yfin[c] : acc[c][0] * dsave;
#pragma unroll
      for (int s = 0; s < R - 1; ++s) acc[c][s] = acc[c][s + 1];
      acc[c][R - 1] = 0.0;
    }
  }
}

// Backward sweep L^T x = w from the COLUMN band (the same bytes the forward
// sweep reads: one factor copy instead of a column and a row band).  Each
// chunk of kCh columns = kCh rows, processed top row first:
//  A) every row's dot product with the already final x of the rows above the
//     chunk (x_{k+j}, j beyond the chunk, from a 128-row circular window in
//     shared memory): 4 lanes per row, each a quarter of the j's, reduced by
//     two xor shuffles -- all rows of the chunk in parallel;
//  B) the chunk's own kCh x kCh triangle in order: row q's x is broadcast
//     and the later rows of the chunk accumulate L[k_p + (p - q)][k_p] x_q.
// Dependent chain per row: one shuffle + fma + mul (B); the window products
// (A) are off the chain.  rows k = natural numbering of the system; ym(k)
// addresses row k's NR values (w on entry, x on exit).
template <int T, int NR, bool PAD, class YMap>
__device__ __forceinline__ void band_sweep_dot(const double* __restrict__ L, int n, int bw, YMap ym, int lane,
                                               Ring& rg, double* __restrict__ xw,
                                               const CUtensorMap* map = nullptr, int col0 = 0) {
  constexpr int kWin = 128;       // window rows (>= bw + kCh); stored twice so reads never wrap
  constexpr int kA = 8 * T;       // phase-A terms per lane: j = pc + 1 + g + 4 i <= 32 T
  constexpr int P = pad_slot_words<T>();
  const int S = bw + 1;
  const int nch = (n + kCh - 1) / kCh;
  if (PAD) {
    for (int c = 0; c < min(rg.nst, nch); ++c) ring_issue_pad<true, P>(rg, map, col0, n, c, lane, c);
  } else if (lane == 0) {
    for (int c = 0; c < min(rg.nst, nch); ++c) ring_issue<true>(rg, L, n, S, c, c);
  }
  for (int i = lane; i < 2 * kWin * NR; i += 32) xw[i] = 0.0;
  __syncwarp();
  const int p = lane >> 2, gq = lane & 3;
  // the group's row of chunk ch (position pc from the chunk top)
  auto row_of = [&](int ch, int& start, int& cnt, int& pc) {
    chunk_cols(true, n, ch, start, cnt);
    pc = p < cnt ? p : 0;
    return start + cnt - 1 - pc;
  };
  // w (the forward sweep's output) of the next chunk's rows is loaded one
  // chunk ahead: the L2 latency stays off the chunk's dependent chain
  double wnext[NR];
  {
    int s0, c0, p0;
    const int k0 = row_of(0, s0, c0, p0);
#pragma unroll
    for (int c = 0; c < NR; ++c) wnext[c] = ym(k0)[c];
  }
  int stc = 0;
  for (int ch = 0; ch < nch; ++ch) {
    const int st = stc;
    stc = (stc + 1 == rg.nst) ? 0 : stc + 1;
    int start, cnt, pc;
    const int k = row_of(ch, start, cnt, pc);
    double wp[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) wp[c] = wnext[c];
    if (ch + 1 < nch) {
      int s1, c1, p1;
      const int k1 = row_of(ch + 1, s1, c1, p1);
#pragma unroll
      for (int c = 0; c < NR; ++c) wnext[c] = ym(k1)[c];
    }
    mbar_wait(rg.bar + st, (rg.phase >> st) & 1u);
    rg.phase ^= 1u << st;
    const double* sb = rg.buf + (size_t)st * rg.stage + (PAD ? 0 : (int)(((int64_t)start * S) & 1));
    const double* col = sb + (cnt - 1 - pc) * (PAD ? P : S);  // its column: L[k + j][k], j = 0..bw
    // (A) rows above the chunk: j = pc + 1 + gq + 4 i, row k + j = start + cnt + gq + 4 i
    // (independent of the group: the window reads are broadcasts)
    {
      const double* cj = col + pc + 1 + gq;
      const double* xj = xw + (((start + cnt + gq) & (kWin - 1)) * NR);
      const int jmax = bw - pc - 1 - gq;  // valid i: 4 i <= jmax
      double acc[4][NR];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < NR; ++c) acc[u][c] = 0.0;
#pragma unroll
      for (int i = 0; i < kA; ++i) {
        if (PAD || 4 * i <= jmax) {  // padded slots read zero beyond the band
          const double lv = cj[4 * i];
#pragma unroll
          for (int c = 0; c < NR; ++c) acc[i & 3][c] = fma(lv, xj[4 * i * NR + c], acc[i & 3][c]);
        }
      }
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        double sum = (acc[0][c] + acc[1][c]) + (acc[2][c] + acc[3][c]);
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        wp[c] -= sum;
      }
    }
    // (B) the chunk's triangle: row q's x broadcast from its group, the later
    // rows p > q accumulate L[k_p + (p - q)][k_p] x_q
    const double d = col[0];
    double lq[kCh];
#pragma unroll
    for (int q = 0; q < kCh; ++q) lq[q] = col[max(p - q, 0)];
    double t[NR], xm[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) t[c] = xm[c] = 0.0;
#pragma unroll
    for (int q = 0; q < kCh; ++q) {
      if (q < cnt) {
#pragma unroll
        for (int c = 0; c < NR; ++c) {
          const double x = __shfl_sync(0xffffffffu, (wp[c] - t[c]) * d, 4 * q);
          xm[c] = (p == q) ? x : xm[c];
          t[c] = fma(lq[q], x, t[c]);
        }
      }
    }
    if (gq == 0 && p < cnt) {
      const int slot = (k & (kWin - 1)) * NR;
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        xw[slot + c] = xm[c];
        xw[slot + kWin * NR + c] = xm[c];
        ym(k)[c] = xm[c];
      }
    }
    __syncwarp();  // window writes visible; every lane done with the stage before it is refilled
    if (PAD) {
      if (ch + rg.nst < nch) ring_issue_pad<true, P>(rg, map, col0, n, ch + rg.nst, lane, st);
    } else if (lane == 0 && ch + rg.nst < nch) {
      ring_issue<true>(rg, L, n, S, ch + rg.nst, st);
    }
  }
}

static int ring_stage_words(int max_bw, int ch = kCh) { return (ch * (max_bw + 1) + 3) & ~1; }

template <int T, int NR, bool PAD, bool UNIT, int CH>
__global__ void __launch_bounds__(kTmaWarps * 32, MS_L1_MINB)
    k_l1_solve_ring(Grid g, const BandSys* __restrict__ sys, int nsys, const double* __restrict__ Lc,
                    const double* __restrict__ Lr, const double* __restrict__ r,
                    double* __restrict__ ybuf, const int* done, int stage_words,
                    const __grid_constant__ CUtensorMap mapc, const __grid_constant__ CUtensorMap mapr,
                    int fwd_only, int nst) {
  if (done && *(volatile const int*)done) return;
  extern __shared__ __align__(128) double smem_ring[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sid = blockIdx.x * kTmaWarps + warp;
  if (sid >= nsys) return;
  Ring rg;
  ring_init(rg, smem_ring, warp, lane, stage_words, nst, PAD);
  const BandSys s = sys[sid];
  double* y = ybuf + s.yoff;
  const int n = s.n;
  const int64_t nn = g.n_nodes;
  // R_s r, gathered by the forward sweep itself: entry i = row * NR + c of the
  // subdomain's node-interleaved vector is component i & 1 of local node i >> 1
  auto gather = [&](int row, int c) -> double {
    const int i = row * NR + c;
    int a, b;
    band_node_of(s, i >> 1, a, b);
    MS_BCHECK(a >= 0 && a <= g.nx && b >= 0 && b <= g.ny);
    return __ldg(r + (i & 1) * nn + (int64_t)b * g.nnx + a);
  };
  const int col0 = PAD ? (int)(s.foff / (s.bw + 1)) : 0;  // the system's first column in the TMA view
  band_sweep_ring<T, NR, false, PAD, UNIT, CH>(Lc + s.foff, n, s.bw, [&](int q) { return y + (int64_t)q * NR; }, lane,
                                               rg, &mapc, col0, gather);
  if (fwd_only) return;  // the backward sweep follows in k_l1_bwd_window
  __syncwarp();
  if (Lr) {
    band_sweep_ring<T, NR, true, PAD, UNIT, CH>(Lr + s.foff, n, s.bw, [&](int r) { return y + (int64_t)(n - 1 - r) * NR; },
                                      lane, rg, &mapr, col0);
  } else {  // one factor copy: backward sweep by dot products over the column band
    double* xw = smem_ring + kRingHeaderWords + (size_t)kTmaWarps * ring_warp_words(stage_words, PAD, nst) +
                 (size_t)warp * 256 * NR;
    if constexpr (kCh == 8 && CH == kCh)
      band_sweep_dot<T, NR, PAD>(Lc + s.foff, n, s.bw, [&](int k) { return y + (int64_t)k * NR; }, lane, rg, xw,
                                 &mapc, col0);
    else
      __trap();  // the dot-form sweep is laid out for 8-column stages
  }
}

// Twisted sweeps: warp pair per subdomain (even warp: top system, odd warp:
// bottom system), both forward sweeps concurrently, the separator solved by
// the pair with the explicit Schur inverse, both backward sweeps
// concurrently.  y stays in natural order (what the combine reads); the
// bottom system's separator partials live in shared memory.
__device__ __forceinline__ void pair_sync(int pair) {
  asm volatile("bar.sync %0, 64;" ::"r"(pair + 1) : "memory");
}

template <int T, int NR, bool PAD, bool UNIT, int CH>
__global__ void __launch_bounds__(kTmaWarps * 32, MS_L1_MINB)
    k_l1_solve_twist(Grid g, const BandSys* __restrict__ sys, int nsys, const double* __restrict__ Lc,
                     const double* __restrict__ Lr, const double* __restrict__ Sinv,
                     const double* __restrict__ r, double* __restrict__ ybuf, const int* done, int stage_words,
                     int max_bw, const __grid_constant__ CUtensorMap mapc,
                     const __grid_constant__ CUtensorMap mapr, int nst) {
  static_assert(kTmaWarps % 2 == 0, "warp pairs");
  if (done && *(volatile const int*)done) return;
  extern __shared__ __align__(128) double smem_ring[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, role = warp & 1;  // role 0: top, 1: bottom
  const int sid = blockIdx.x * (kTmaWarps / 2) + pair;
  if (sid >= nsys) return;  // both warps of a pair leave together
  Ring rg;
  ring_init(rg, smem_ring, warp, lane, stage_words, nst, PAD);
  const size_t ring_words = kRingHeaderWords + (size_t)kTmaWarps * ring_warp_words(stage_words, PAD, nst);
  double* sB = smem_ring + ring_words + (size_t)pair * 2 * NR * max_bw;  // bottom separator partials
  double* tS = sB + NR * max_bw;                                       // separator right-hand side
  const BandSys s = sys[sid];
  const int n = s.n, bw = s.bw, m = s.m, nT = m + bw, nB = n - m;
  MS_BCHECK(bw >= 1 && bw <= max_bw && m >= 1 && nT <= n && nB >= bw && nst >= 2 && nst <= kMaxNst);
  double* y = ybuf + s.yoff;
  // R_s r is gathered by the forward sweeps themselves (top warp: rows [0, nT)
  // incl. the separator's; bottom warp: its own rows [nT, n) in reverse, its
  // separator rows start from zero and end as the partials -L_SB y_B in sB)
  const int64_t nn = g.n_nodes;
  auto gather = [&](int row, int c) -> double {
    const int i = row * NR + c;
    int a, b;
    band_node_of(s, i >> 1, a, b);
    MS_BCHECK(a >= 0 && a <= g.nx && b >= 0 && b <= g.ny);
    return __ldg(r + (i & 1) * nn + (int64_t)b * g.nnx + a);
  };
  const int nb_own = nB - bw;
  auto ymB = [&](int q) { return q < nb_own ? y + (int64_t)(n - 1 - q) * NR : sB + (q - nb_own) * NR; };
  if constexpr (CH == kChWide) {
    // latency-bound launches (one warp per scheduler): a separate gather pass
    // keeps the index arithmetic off the sweeps' in-order stream (config 2:
    // 0.157 ms vs 0.162 ms with the gather inside the sweeps)
    const int i0 = role ? nT * NR : 0, i1 = role ? n * NR : nT * NR;
    for (int i = i0 + lane; i < i1; i += 32) y[i] = gather(i / NR, i % NR);
    if (role)
      for (int i = lane; i < NR * bw; i += 32) sB[i] = 0.0;
    __syncwarp();
    if (role == 0)
      band_sweep_ring<T, NR, false, PAD, UNIT, CH>(Lc + s.foff, nT, bw, [&](int q) { return y + (int64_t)q * NR; },
                                                   lane, rg, &mapc, PAD ? (int)(s.foff / (bw + 1)) : 0);
    else
      band_sweep_ring<T, NR, false, PAD, UNIT, CH>(Lc + s.foffB, nB, bw, ymB, lane, rg, &mapc,
                                                   PAD ? (int)(s.foffB / (bw + 1)) : 0);
  } else if (role == 0) {
    band_sweep_ring<T, NR, false, PAD, UNIT, CH>(Lc + s.foff, nT, bw, [&](int q) { return y + (int64_t)q * NR; }, lane,
                                                 rg, &mapc, PAD ? (int)(s.foff / (bw + 1)) : 0, gather);
  } else {
    band_sweep_ring<T, NR, false, PAD, UNIT, CH>(
        Lc + s.foffB, nB, bw, ymB, lane, rg, &mapc, PAD ? (int)(s.foffB / (bw + 1)) : 0,
        [&](int q, int c) -> double { return q < nb_own ? gather(n - 1 - q, c) : 0.0; });
  }
  pair_sync(pair);
  // separator: t = (r_S - L_ST y_T) + (- L_SB y_B); x_S = Sinv t
  const int tid = role * 32 + lane;
  for (int i = tid; i < NR * bw; i += 64) {
    const int row = i / NR, c = i % NR;
    tS[i] = y[(int64_t)(m + row) * NR + c] + sB[(bw - 1 - row) * NR + c];
  }
  pair_sync(pair);
  const double* Si = Sinv + s.soff;
  for (int j = tid; j < bw; j += 64) {
    double acc[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) acc[c] = 0.0;
    for (int i = 0; i < bw; ++i) {
      const double v = __ldg(Si + (int64_t)i * bw + j);  // symmetric: column j = row j, coalesced over j
#pragma unroll
      for (int c = 0; c < NR; ++c) acc[c] = fma(v, tS[i * NR + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NR; ++c) y[(int64_t)(m + j) * NR + c] = acc[c];
  }
  pair_sync(pair);
  if (!Lr) {  // one factor copy: both backward sweeps by dot products over the column bands
    double* xw = smem_ring + ring_words + (size_t)(kTmaWarps / 2) * 2 * NR * max_bw + (size_t)warp * 256 * NR;
    if constexpr (kCh != 8 || CH != kCh) {
      __trap();  // the dot-form sweep is laid out for 8-column stages
    } else if (role == 0)
      band_sweep_dot<T, NR, PAD>(Lc + s.foff, nT, bw, [&](int k) { return y + (int64_t)k * NR; }, lane, rg, xw,
                                 &mapc, PAD ? (int)(s.foff / (bw + 1)) : 0);
    else  // bottom-local row k = natural n - 1 - k (its separator rows now hold x_S)
      band_sweep_dot<T, NR, PAD>(Lc + s.foffB, nB, bw, [&](int k) { return y + (int64_t)(n - 1 - k) * NR; }, lane,
                                 rg, xw, &mapc, PAD ? (int)(s.foffB / (bw + 1)) : 0);
    return;
  }
  if (role == 0) {
    band_sweep_ring<T, NR, true, PAD, UNIT, CH>(Lr + s.foff, nT, bw, [&](int q) { return y + (int64_t)(nT - 1 - q) * NR; },
                                      lane, rg, &mapr, PAD ? (int)(s.foff / (bw + 1)) : 0);
  } else {
    band_sweep_ring<T, NR, true, PAD, UNIT, CH>(Lr + s.foffB, nB, bw, [&](int q) { return y + (int64_t)(m + q) * NR; }, lane,
                                      rg, &mapr, PAD ? (int)(s.foffB / (bw + 1)) : 0);
  }
}

// ---------------------------------------------------------------------------
// One-copy backward sweep in axpy form from the COLUMN band: x = L^-T w.
// Pivot k (descending) updates the rows k - j with L[k][k-j] = col_{k-j}[j],
// so every lane reads its own row's column at band offset j = 32 s + lane - u
// (consecutive lanes: stride S - 1 words, no bank conflicts), and the columns
// of the last bw + 1 pivots must stay in shared memory: one warp per CTA
// streams its band through a deep ring of kWCh-column chunks; a chunk is
// refilled right after its own pivots (its columns' last use), the chunks a
// pivot reaches down to are waited for before its chunk starts.  The forward
// sweep ran before in k_l1_solve_ring (fwd_only).  Half the factor bytes of
// the two-band sweeps; the deep ring caps residency at 4 warps per SM.
constexpr int kWCh = 4;
static bool use_window_bwd();

__host__ __device__ inline int win_stages(int bw) { return (bw + 3 + 12 + kWCh - 1) / kWCh + 1; }  // + ~12 rows of prefetch
__host__ __device__ inline int win_stage_words(int bw) { return (kWCh * (bw + 1) + 3) & ~1; }
__host__ __device__ inline int win_header_words(int nst) { return (nst + 15) & ~15; }

template <int T>
__global__ void __launch_bounds__(32, 4)
    k_l1_bwd_window(const BandSys* __restrict__ sys, int nsys, const double* __restrict__ Lc,
                    double* __restrict__ ybuf, const int* done, int nst, int stage_words) {
  if (done && *(volatile const int*)done) return;
  extern __shared__ __align__(128) double smw[];
  const int lane = threadIdx.x;
  const int sid = blockIdx.x;
  if (sid >= nsys) return;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smw);
  double* buf = smw + win_header_words(nst);
  const BandSys s = sys[sid];
  const int n = s.n, bw = s.bw, S = bw + 1;
  const double* L = Lc + s.foff;
  double* y = ybuf + s.yoff;
  const int nch = (n + kWCh - 1) / kWCh;
  // REV chunk c: columns [start, start + cnt), the highest first
  auto chunk = [&](int c, int& start, int& cnt) {
    const int k0 = c * kWCh;
    cnt = min(kWCh, n - k0);
    start = n - k0 - cnt;
  };
  auto issue = [&](int c) {
    int start, cnt;
    chunk(c, start, cnt);
    const int64_t w0 = (int64_t)start * S;
    const int64_t a = w0 & ~(int64_t)1;
    const uint32_t words = (uint32_t)((cnt * S + (int)(w0 - a) + 1) & ~1);
    MS_BCHECK((int)words <= stage_words && a >= 0 && a + (int64_t)words <= (int64_t)n * S + 2);
    const int st = c % nst;
    mbar_expect_tx(bar + st, words * 8u);
    bulk_g2s(buf + (size_t)st * stage_words, L + a, words * 8u, bar + st);
  };
  // shared address of column `col` (its chunk is resident)
  auto colp = [&](int col) -> const double* {
    const int c = (n - 1 - col) / kWCh;
    int start, cnt;
    chunk(c, start, cnt);
    return buf + (size_t)(c % nst) * stage_words + (int)(((int64_t)start * S) & 1) + (col - start) * S;
  };
  if (lane == 0) {
    for (int st = 0; st < nst; ++st) mbar_init(bar + st, 1);
    mbar_fence_init();
    for (int c = 0; c < min(nst, nch); ++c) issue(c);
  }
  __syncwarp();
  uint64_t phase = 0;
  int waited = 0;
  const int ahead = (bw + kWCh - 1) / kWCh + 1;  // chunks below a pivot chunk its updates reach
  constexpr int R = T + 1;
  // REV numbering: sweep row r = natural row n - 1 - r
  auto yat = [&](int r) -> double* { return y + (n - 1 - r); };
  double acc[R], rnext;
#pragma unroll
  for (int sl = 0; sl < R - 1; ++sl) {
    const int r = 32 * sl + lane;
    acc[sl] = r < n ? *yat(r) : 0.0;
  }
  acc[R - 1] = 0.0;
  rnext = (32 * (R - 1) + lane < n) ? *yat(32 * (R - 1) + lane) : 0.0;
  for (int r0 = 0; r0 < n; r0 += 32) {
    acc[R - 1] = rnext;
    {
      const int r = r0 + 32 * R + lane;
      rnext = r < n ? *yat(r) : 0.0;
    }
    // this lane's rows in the block's slots and their columns' bases:
    // coefficient of pivot u for slot sl = col_{row}[32 sl + lane - u]
    const double* base[R];
    bool rowok[R];
    double dsave = 0.0;
#pragma unroll 1
    for (int h = 0; h < 32 && r0 + h < n; h += kWCh) {
      const int ch = (r0 + h) / kWCh;
      const int need = min(ch + ahead, nch - 1);
      while (waited <= need) {
        const int st = waited % nst;
        mbar_wait(bar + st, (uint32_t)((phase >> st) & 1u));
        phase ^= 1ull << st;
        ++waited;
      }
      if (h == 0) {  // slot bases once per block (their chunks are resident now)
#pragma unroll
        for (int sl = 0; sl < R; ++sl) {
          const int col = n - 1 - (r0 + 32 * sl + lane);
          rowok[sl] = col >= 0 && col < n;
          base[sl] = (rowok[sl] ? colp(col) : buf) + 32 * sl + lane;
        }
      }
      int start, cnt;
      chunk(ch, start, cnt);
      const double* pcol = colp(start + cnt - 1);  // pivot columns: pcol - q S
      auto step = [&](int q) {
        const int u = h + q;
        double m[R];
#pragma unroll
        for (int sl = 0; sl < R; ++sl) {
          const int j = 32 * sl + lane - u;
          m[sl] = lds_or_zero(base[sl] - u, rowok[sl] && j >= 1 && j <= bw);
        }
        const double d = lds_or_zero(pcol - q * S, true);
        if (lane == u) dsave = d;
        const double wk = __shfl_sync(0xffffffffu, acc[0] * d, u);
#pragma unroll
        for (int sl = 0; sl < R; ++sl) acc[sl] = fma(-m[sl], wk, acc[sl]);
      };
      if (cnt == kWCh) {
#pragma unroll
        for (int q = 0; q < kWCh; ++q) step(q);
      } else {
#pragma unroll
        for (int q = 0; q < kWCh; ++q)
          if (q < cnt) step(q);
      }
      __syncwarp();  // chunk ch's pivots are done: its columns are dead
      if (lane == 0 && ch + nst < nch) issue(ch + nst);
    }
    if (r0 + lane < n) *yat(r0 + lane) = acc[0] * dsave;
#pragma unroll
    for (int sl = 0; sl < R - 1; ++sl) acc[sl] = acc[sl + 1];
    acc[R - 1] = 0.0;
  }
}

// ring shared memory of a launch: header + per-warp rings (+ extras)
template <int T>
static int ring_stage_words_t(int max_bw, bool pad, int ch = kCh) {
  return pad ? kCh * pad_slot_words<T>() : ring_stage_words(max_bw, ch);
}

// 16-column ring stages for launches of at most one CTA per SM, 8 otherwise
// (MS_L1_CH=8 / 16 forces one): see band_sweep_ring.  At two CTAs per SM the
// two widths measure the same (config 3's 8-GPU strip twisted: 0.277 ms with
// 3 x 8 or 2 x 16 columns; its 4-GPU strip plain: within run-to-run noise).
static bool wide_chunks(int ctas) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("MS_L1_CH");
    env = e ? std::atoi(e) : -1;
  }
  if (env == kCh) return false;
  if (env == kChWide) return true;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return ctas <= sms;
}
static size_t ring_bytes(int stage_words, bool pad, int nst) {
  return ((size_t)kRingHeaderWords + (size_t)kTmaWarps * ring_warp_words(stage_words, pad, nst)) * sizeof(double);
}

// Ring depth of a launch.  Launches of several waves are bandwidth-bound:
// 2 stages keep 4 CTAs per SM resident (config 3: 1.94 ms vs 1.99 ms with
// 3).  A launch that fits one wave is bound by its bytes in flight per warp
// instead, so the shared memory its few CTAs leave free goes into deeper
// rings (MS_L1_NST overrides; measured with the twisted kernel: config 2,
// one CTA per SM, 0.207 / 0.197 / 0.181 / 0.180 ms at 2 / 3 / 4 / 6 stages;
// config 3's 8-GPU strip, two CTAs per SM, 0.283 / 0.277 / 0.289 ms at
// 2 / 3 / 4).
static int pick_nst(int ctas, size_t stage_bytes_cta, size_t extra_bytes) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("MS_L1_NST");
    env = e ? std::atoi(e) : -1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int per_sm = div_up(ctas, sms);
  int nst = env >= 2 ? env : (per_sm == 1 ? 4 : (per_sm == 2 ? 3 : kNst));
  nst = std::min(nst, kMaxNst);
  // the wave's CTAs must stay co-resident (227 KB per SM, 1 KB reserved per CTA)
  const size_t budget = (size_t)227 * 1024 / std::max(1, std::min(per_sm, 4)) - 1024;
  while (nst > 2 && kRingHeaderWords * sizeof(double) + extra_bytes + nst * stage_bytes_cta > budget) --nst;
  return nst;
}

template <class K>
static void set_smem(K kernel, size_t smem, size_t* configured) {
  int dev = 0;
  MS_CUDA(cudaGetDevice(&dev));
  if (dev >= 64 || smem > configured[dev]) {
    MS_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (dev < 64) configured[dev] = smem;
  }
}

static const L1Maps& no_maps() {
  static L1Maps m{};
  return m;
}

template <int T, int NR, bool PAD, bool UNIT, int CH = kCh>
static void solve_twist_t(const Grid& g, const BandSys* sys, int nsys, int max_bw, const double* Lc,
                          const double* Lr, const double* Sinv, const double* r, double* ybuf, const int* done,
                          cudaStream_t st, const L1Maps& maps) {
  const int sw = ring_stage_words_t<T>(max_bw, PAD, CH);
  const size_t extra = (size_t)(kTmaWarps / 2) * 2 * NR * max_bw * sizeof(double) +
                       (Lr ? 0 : (size_t)kTmaWarps * 256 * NR * sizeof(double));  // separator + dot-sweep windows
  const int nst = pick_nst(div_up(nsys, kTmaWarps / 2), (size_t)kTmaWarps * sw * sizeof(double),
                           extra + (PAD ? kTmaWarps * kPadGuard * sizeof(double) : 0));
  const size_t smem = ring_bytes(sw, PAD, nst) + extra;
  static size_t configured[64] = {};
  set_smem(k_l1_solve_twist<T, NR, PAD, UNIT, CH>, smem, configured);
  { k_l1_solve_twist<T, NR, PAD, UNIT, CH><<<div_up(nsys, kTmaWarps / 2), kTmaWarps * 32, smem, st>>>(
      g, sys, nsys, Lc, Lr, Sinv, r, ybuf, done, sw, max_bw, maps.c, maps.r, nst); ms_count_launch(); }
}

template <int T, int NR, bool PAD, bool UNIT, int CH = kCh>
static void solve_ring_t(const Grid& g, const BandSys* sys, int nsys, int max_bw, const double* Lc,
                         const double* Lr, const double* r, double* ybuf, const int* done,
                         cudaStream_t st, const L1Maps& maps) {
  const int sw = ring_stage_words_t<T>(max_bw, PAD, CH);
  // + the dot sweep's x windows (one factor copy)
  const size_t extra = Lr ? 0 : (size_t)kTmaWarps * 256 * NR * sizeof(double);
  const int nst = pick_nst(div_up(nsys, kTmaWarps), (size_t)kTmaWarps * sw * sizeof(double),
                           extra + (PAD ? kTmaWarps * kPadGuard * sizeof(double) : 0));
  const size_t smem = ring_bytes(sw, PAD, nst) + extra;
  static size_t configured[64] = {};  // per instantiation and device
  set_smem(k_l1_solve_ring<T, NR, PAD, UNIT, CH>, smem, configured);
  const bool window = !Lr && NR == 1 && use_window_bwd();
  { k_l1_solve_ring<T, NR, PAD, UNIT, CH><<<div_up(nsys, kTmaWarps), kTmaWarps * 32, smem, st>>>(
      g, sys, nsys, Lc, Lr, r, ybuf, done, sw, maps.c, maps.r, window ? 1 : 0, nst); ms_count_launch(); }
  if (window) {
    const int nst = win_stages(max_bw), wsw = win_stage_words(max_bw);
    const size_t wsmem = ((size_t)win_header_words(nst) + (size_t)nst * wsw) * sizeof(double);
    static size_t wconf[64] = {};
    set_smem(k_l1_bwd_window<T>, wsmem, wconf);
    { k_l1_bwd_window<T><<<nsys, 32, wsmem, st>>>(sys, nsys, Lc, ybuf, done, nst, wsw); ms_count_launch(); }
  }
}

// Padded TMA-tensor ring for the elasticity bands on request (MS_L1_PAD=1):
// leaner steps (unconditional loads at immediate offsets) pay off only in the
// latency-bound regime (config 2: level 1 0.327 -> 0.306 ms plain, 0.206 ->
// 0.197 ms twisted, 3 stages); bandwidth-bound it is slower (config 3: 1.99
// -> 2.33 ms: 73% more shared-memory traffic per band column)
bool l1_padded_ring_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MS_L1_PAD");
    v = (e && std::string(e) == "1") ? 1 : 0;
  }
  return v == 1;
}

// one factor copy, plain level 1: backward sweep in axpy form from a deep
// shared-memory window of the column band (default), or the dot-product form
// (MS_L1_BWD=dot)
static bool use_window_bwd() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MS_L1_BWD");
    v = (e && std::string(e) == "dot") ? 0 : 1;
  }
  return v == 1;
}

static bool use_ring_sweeps() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MS_L1_SWEEP");
    v = (e && std::string(e) == "reg") ? 0 : 1;
  }
  return v == 1;
}

bool ring_sweep_ok(int T, int min_bw) { return T <= 1 || min_bw > 32 * (T - 1); }

void make_band_map(CUtensorMap* map, const double* band, int64_t cols, int S, int T) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    MS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) throw Error(-1, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)S, (cuuint64_t)cols};
  const cuuint64_t strides[1] = {(cuuint64_t)S * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)(32 * (T + 1)), (cuuint32_t)kCh};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(band), dims, strides, box,
                            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(-1, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}
bool l1_ring_sweeps_enabled() { return use_ring_sweeps(); }

template <int T, int NR>
static void solve_t(const Grid& g, const BandSys* sys, int nsys, int max_bw, const double* Lc,
                    const double* Lr, const double* r, double* ybuf, const int* done, cudaStream_t st,
                    const double* Sinv, bool ring_ok, const L1Maps* maps, bool unit) {
  // padded TMA ring: elasticity bands with their tensor maps (uniform bw)
  const bool pad = NR == 1 && maps && maps->valid;
  const L1Maps& mp = pad ? *maps : no_maps();
  // unit-diagonal factors: two-band ring sweeps without the padded layout only
  if (unit && (pad || !Lr || !(Sinv || (use_ring_sweeps() && ring_ok))))
    throw Error(-1, "unit-diagonal level-1 factors need the two-band ring sweeps");
  if (Sinv) {
    if (pad)
      solve_twist_t<T, NR, NR == 1, false>(g, sys, nsys, max_bw, Lc, Lr, Sinv, r, ybuf, done, st, mp);
    else if (unit && T <= 4 && wide_chunks(div_up(nsys, kTmaWarps / 2)))
      solve_twist_t<T, NR, false, true, (T <= 4 ? kChWide : kCh)>(g, sys, nsys, max_bw, Lc, Lr, Sinv, r, ybuf, done, st,
                                                                  mp);
    else if (unit)
      solve_twist_t<T, NR, false, true>(g, sys, nsys, max_bw, Lc, Lr, Sinv, r, ybuf, done, st, mp);
    else
      solve_twist_t<T, NR, false, false>(g, sys, nsys, max_bw, Lc, Lr, Sinv, r, ybuf, done, st, mp);
    return;
  }
  if (use_ring_sweeps() && ring_ok) {
    if (pad)
      solve_ring_t<T, NR, NR == 1, false>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, mp);
    else if (unit && T <= 4 && wide_chunks(div_up(nsys, kTmaWarps)))
      solve_ring_t<T, NR, false, true, (T <= 4 ? kChWide : kCh)>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, mp);
    else if (unit)
      solve_ring_t<T, NR, false, true>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, mp);
    else
      solve_ring_t<T, NR, false, false>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, mp);
    return;
  }
  if (!Lr) throw Error(-1, "the register-prefetch level-1 sweeps need the row band (two factor copies)");
  { k_l1_solve<T, NR><<<div_up(nsys, kSolveWarps), kSolveWarps * 32, 0, st>>>(g, sys, nsys, Lc, Lr, r,
                                                                            ybuf, done); ms_count_launch(); }
}

void launch_l1_solve(const Grid& g, const BandSys* sys, int nsys, int max_bw, int nrhs,
                     const double* Lc, const double* Lr, const double* r, double* ybuf,
                     const int* done, cudaStream_t st, const double* Sinv, int min_bw, const L1Maps* maps,
                     bool unit) {
  if (nsys == 0) return;
  const int T = std::max(1, div_up(max_bw, 32));
  if (min_bw < 0) min_bw = max_bw;
  // the ring step assumes slots 1..T-2 inside every band
  const bool ring_ok = ring_sweep_ok(T, min_bw);
  if (Sinv && !ring_ok) throw Error(-1, "twisted level-1 needs every band wider than 32 (T - 1)");
  if (nrhs == 1) {
    switch (T) {
      case 1: solve_t<1, 1>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      case 2: solve_t<2, 1>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      case 3: solve_t<3, 1>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      case 4: solve_t<4, 1>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      case 5: solve_t<5, 1>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      case 6: solve_t<6, 1>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      case 7: solve_t<7, 1>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      case 8: solve_t<8, 1>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      default: throw Error(-1, "level-1 band wider than 256 unsupported");
    }
  } else if (nrhs == 2) {
    switch (T) {
      case 1: solve_t<1, 2>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      case 2: solve_t<2, 2>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      case 3: solve_t<3, 2>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      case 4: solve_t<4, 2>(g, sys, nsys, max_bw, Lc, Lr, r, ybuf, done, st, Sinv, ring_ok, maps, unit); break;
      default: throw Error(-1, "heat level-1 band wider than 128 unsupported");
    }
  } else {
    throw Error(-1, "nrhs must be 1 or 2");
  }
  MS_CUDA(cudaGetLastError());
}

}  // namespace msgpu
