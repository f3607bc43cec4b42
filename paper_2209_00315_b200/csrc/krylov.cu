// krylov.cu -- device-resident FGMRES(restart) with CGS2 and per-slice PCG
// (see krylov.cuh).  Every scalar decision is taken on the device by the last
// block of a fused reduction; the host only emits kernels and loops.
#include "krylov.cuh"
#include <cmath>
#include <cstdlib>

namespace bbot {

constexpr int BS = 256;
constexpr double TINY = 1e-300;

// ------------------------------------------------------------ BLAS-1 kernels
__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}
__global__ void k_scale(const double* __restrict__ a, double s, double* __restrict__ b, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = s * a[i];
}
__global__ void k_axpby(double alpha, const double* __restrict__ a, double beta, double* __restrict__ b, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = alpha * a[i] + beta * b[i];
}
void dev_copy(Dev& d, const double* a, double* b, long long n) {
  launch(d, k_copy, dim3(nblocks(n, BS)), dim3(BS), 0, a, b, n);
}
void dev_scale(Dev& d, const double* a, double s, double* b, long long n) {
  launch(d, k_scale, dim3(nblocks(n, BS)), dim3(BS), 0, a, s, b, n);
}
void dev_axpby(Dev& d, double alpha, const double* a, double beta, double* b, long long n) {
  launch(d, k_axpby, dim3(nblocks(n, BS)), dim3(BS), 0, alpha, a, beta, b, n);
}

// ------------------------------------------------------------ FGMRES kernels
// Grid (parts, owned slices): block (p, y) handles chunk p of the y-th owned slice.  All
// vectors are in global layout (length n); only owned slices are touched.

// chunk [beg, end) of this block in global indices; loff: global -> slab-local basis index
__device__ __forceinline__ void seg_chunk(const SegArgs& A, int& s, long long& beg, long long& end,
                                          long long* loff = nullptr) {
  long long base, l;
  A.set.slice(blockIdx.y, s, base, l);
  long long chunk = (l + A.parts - 1) / A.parts;
  beg = base + (long long)blockIdx.x * chunk;
  end = base + min(l, (long long)(blockIdx.x + 1) * chunk);
  if (beg > end) beg = end;
  if (loff) *loff = A.set.local_base(blockIdx.y) - base;
}

// out[k] = sum over slices s = 0..S-1 (in order) of tot[s][k], k < cnt; all threads of one
// block; identical code in the fused last block and in the finishing kernel
__device__ __forceinline__ void seg_total(const SegArgs& A, int cnt, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int S = A.set.S();
  for (int k = w; k < cnt; k += nw) {
    double v = 0.0;
    for (int s = lane; s < S; s += 32) v += __ldcg(A.tot + (size_t)s * GM_NRP + k);
    v = warp_sum(v);
    if (lane == 0) out[k] = v;
  }
  __syncthreads();
}

// block partials of cnt values; the last block of each slice turns that slice's partials into
// its slice totals (fixed order over the parts), and the last slice to finish (fused) the
// slice totals into out[0..cnt).  Returns true in every thread of the block that must run
// the epilogue.
template <int NR>
__device__ __forceinline__ bool seg_commit(const double (&acc)[NR], int cnt, const SegArgs& A, int s, double* out) {
  __shared__ double shn[NR][33];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NR; k++)
    if (k < cnt) {
      double v = warp_sum(acc[k]);
      if (lane == 0) shn[k][w] = v;
    }
  __syncthreads();
  for (int k = w; k < cnt; k += nw) {
    double v = lane < nw ? shn[k][lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) {
      A.partial[((size_t)s * A.parts + blockIdx.x) * GM_NRP + k] = v;
      __threadfence();
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {       // last block of this slice?
    __threadfence();
    unsigned t = atomicAdd(A.counter + 1 + s, 1u);
    s_last = (t == (unsigned)A.parts - 1) ? 1 : 0;
    if (s_last) A.counter[1 + s] = 0u;
  }
  __syncthreads();
  if (!s_last) return false;
  for (int k = w; k < cnt; k += nw) {
    double v = 0.0;
    for (int p = lane; p < A.parts; p += 32) v += __ldcg(A.partial + ((size_t)s * A.parts + p) * GM_NRP + k);
    v = warp_sum(v);
    if (lane == 0) A.tot[(size_t)s * GM_NRP + k] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {       // last slice of the launch?
    unsigned t = atomicAdd(A.counter, 1u);
    s_last = (t == (unsigned)A.set.owned() - 1) ? 1 : 0;
    if (s_last) {
      __threadfence();
      A.counter[0] = 0u;
    }
  }
  __syncthreads();
  if (!s_last || !A.fused) return false;
  seg_total(A, cnt, out);
  return true;
}

// ---- epilogues (run by one block: the fused last block or the finishing kernel)
struct EpiResid {      // beta = ||b - op(x)||: start a cycle or stop
  GmresScal* G;
  __device__ void operator()(const double* out) const {
    if (threadIdx.x != 0) return;
    double beta = sqrt(out[0]);
    G->beta = beta;
    G->res = beta;
    G->j = 0;
    G->jj = 0;
    if (!(beta > G->target)) {
      G->conv = 1;
      G->flag_inner = 0;
    } else {
      G->flag_inner = 1;
      for (int i = 0; i <= GM_MAXR; i++) G->g[i] = 0.0;
      G->g[0] = beta;
    }
  }
};
struct EpiStore {      // h1 / h2 <- the j+1 dots
  double* dst;
  int cnt;
  __device__ void operator()(const double* out) const {
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) dst[k] = out[k];
  }
};
struct EpiNorm {       // *norm = sqrt(sum)
  double* norm;
  __device__ void operator()(const double* out) const {
    if (threadIdx.x == 0) *norm = sqrt(out[0]);
  }
};
struct EpiGivens {     // Hessenberg column, Givens rotations, residual estimate, inner decision (Saad)
  GmresScal* G;
  LoopCtl inner;
  __device__ void operator()(const double* out) const {
    if (threadIdx.x != 0) return;
    const int j = G->j;
    const int r = G->restart;
    double hn = sqrt(out[0]);
    double* H = G->H;
    for (int i = 0; i <= j; i++) H[i * GM_MAXR + j] = G->h1[i] + G->h2[i];
    H[(j + 1) * GM_MAXR + j] = hn;
    for (int i = 0; i < j; i++) {
      double t = G->cs[i] * H[i * GM_MAXR + j] + G->sn[i] * H[(i + 1) * GM_MAXR + j];
      H[(i + 1) * GM_MAXR + j] = -G->sn[i] * H[i * GM_MAXR + j] + G->cs[i] * H[(i + 1) * GM_MAXR + j];
      H[i * GM_MAXR + j] = t;
    }
    double den = hypot(H[j * GM_MAXR + j], H[(j + 1) * GM_MAXR + j]);
    G->cs[j] = H[j * GM_MAXR + j] / den;
    G->sn[j] = H[(j + 1) * GM_MAXR + j] / den;
    H[j * GM_MAXR + j] = den;
    H[(j + 1) * GM_MAXR + j] = 0.0;
    G->g[j + 1] = -G->sn[j] * G->g[j];
    G->g[j] = G->cs[j] * G->g[j];
    double res = fabs(G->g[j + 1]);
    G->res = res;
    G->jj = j + 1;
    G->its += 1;
    G->total_its += 1;
    G->hn = hn;
    if (hn <= TINY) G->brk = 1;
    int cont = !(res <= G->target || G->its >= G->maxit || G->brk) && (j + 1 < r);
    G->j = j + 1;
    G->flag_inner = cont;
    inner.set(cont);
  }
};

template <class Epi>
__global__ void k_seg_finish(SegArgs A, int cnt, Epi epi) {
  __shared__ double out[GM_NRP];
  seg_total(A, cnt, out);
  epi(out);
}
// the multi-dot variant: the count j + 1 lives on the device
__global__ void k_seg_finish_dots(SegArgs A, GmresScal* G, int which) {
  __shared__ double out[GM_NRP];
  const int cnt = G->j + 1;
  seg_total(A, cnt, out);
  EpiStore{which == 0 ? G->h1 : G->h2, cnt}(out);
}

__global__ void k_gm_init(GmresScal* G, const double* scale, double tol, int maxit, int restart) {
  G->its = 0;
  G->conv = 0;
  G->brk = 0;
  G->maxit = maxit;
  G->restart = restart;
  G->scale = *scale;
  G->target = tol * G->scale;
  G->res = 0.0;
  G->jj = 0;
  G->flag_outer = 1;
  G->flag_inner = 0;
}

// w = b - w (w = op(x) on entry);  beta = ||w||
__global__ void k_gm_residual(const double* __restrict__ b, double* __restrict__ w, SegArgs A, EpiResid epi) {
  int s;
  long long beg, end;
  seg_chunk(A, s, beg, end);
  double acc[1] = {0.0};
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double v = b[i] - w[i];
    w[i] = v;
    acc[0] += v * v;
  }
  __shared__ double out[1];
  if (seg_commit<1>(acc, 1, A, s, out)) epi(out);
}

// b = -a, ||a||  (inner GMRES right-hand side)
__global__ void k_gm_neg_norm(const double* __restrict__ a, double* __restrict__ b, SegArgs A, EpiNorm epi) {
  int s;
  long long beg, end;
  seg_chunk(A, s, beg, end);
  double acc[1] = {0.0};
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double v = a[i];
    b[i] = -v;
    acc[0] += v * v;
  }
  __shared__ double out[1];
  if (seg_commit<1>(acc, 1, A, s, out)) epi(out);
}

// ||a||  (no write)
__global__ void k_gm_norm(const double* __restrict__ a, SegArgs A, EpiNorm epi) {
  int s;
  long long beg, end;
  seg_chunk(A, s, beg, end);
  double acc[1] = {0.0};
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double v = a[i];
    acc[0] += v * v;
  }
  __shared__ double out[1];
  if (seg_commit<1>(acc, 1, A, s, out)) epi(out);
}

// V[j] = w / s and vin = V[j], s = beta (start) or hn (Arnoldi), only if the inner loop continues
__global__ void k_gm_scale(long long nl, const double* __restrict__ w, double* __restrict__ V,
                           double* __restrict__ vin, const GmresScal* G, int start, SegArgs A) {
  if (!G->flag_inner) return;
  int s;
  long long beg, end, lo;
  seg_chunk(A, s, beg, end, &lo);
  double sc = start ? G->beta : G->hn;
  int j = start ? 0 : G->j;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double v = w[i] / sc;
    V[(size_t)j * nl + i + lo] = v;
    vin[i] = v;
  }
}

// basis vectors loaded together per row in the two-pass CGS2 middle step
constexpr int GM_GRP = 8;

// h[k] = V[k] . w for k <= j (one pass over w, one register accumulator per k);
// optionally copy zout -> Z[j] in the same pass
template <bool COPYZ, int NR>
__global__ void __launch_bounds__(256) k_gm_dots(long long nl, const double* __restrict__ V,
                                                 const double* __restrict__ w, const double* __restrict__ zout,
                                                 double* __restrict__ Z, GmresScal* G, SegArgs A) {
  const int j = G->j;
  int s;
  long long beg, end, lo;
  seg_chunk(A, s, beg, end, &lo);
  double acc[NR];
#pragma unroll
  for (int k = 0; k < NR; k++) acc[k] = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double wi = w[i];
    if (COPYZ) Z[(size_t)j * nl + i + lo] = zout[i];
#pragma unroll
    for (int k = 0; k < NR; k++)
      if (k <= j) acc[k] += V[(size_t)k * nl + i + lo] * wi;
  }
  __shared__ double out[NR];
  if (seg_commit<NR>(acc, j + 1, A, s, out)) EpiStore{G->h1, j + 1}(out);
}

// CGS2 middle step in one pass: w -= sum_{k<=j} h1[k] V[k] (first projection),
// then h2[k] = V[k] . w for the second, reusing the V entries just loaded
template <int NR>
__global__ void __launch_bounds__(256) k_gm_orth_dots(long long nl, const double* __restrict__ V,
                                                      double* __restrict__ w, GmresScal* G, SegArgs A) {
  const int j = G->j;
  __shared__ double hs[GM_MAXR + 1];
  if (threadIdx.x <= (unsigned)j) hs[threadIdx.x] = G->h1[threadIdx.x];
  __syncthreads();
  int s;
  long long beg, end, lo;
  seg_chunk(A, s, beg, end, &lo);
  double acc[NR];
#pragma unroll
  for (int k = 0; k < NR; k++) acc[k] = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    if constexpr (NR <= 16) {
      // T-GMRES (NR = 12): pass 1 the projection sum (k ascending), pass 2 re-reads V[k]
      // (L1/L2) for the dots -- fewer registers than holding the row's NR values across both
      // (8 loads in flight per group: 153 -> 115 ms per C4 step; groups of 4: 157 ms); at
      // NR = 32 the re-read costs more than it saves (109 -> 330 ms), so the values stay live
      double sm = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < NR; k0 += GM_GRP) {
        if (k0 > j) break;
        double vk[GM_GRP];
#pragma unroll
        for (int t = 0; t < GM_GRP; t++) vk[t] = k0 + t <= j ? V[(size_t)(k0 + t) * nl + i + lo] : 0.0;
#pragma unroll
        for (int t = 0; t < GM_GRP; t++)
          if (k0 + t <= j) sm += hs[k0 + t] * vk[t];
      }
      double v = w[i] - sm;
      w[i] = v;
#pragma unroll
      for (int k0 = 0; k0 < NR; k0 += GM_GRP) {
        if (k0 > j) break;
        double vk[GM_GRP];
#pragma unroll
        for (int t = 0; t < GM_GRP; t++) vk[t] = k0 + t <= j ? V[(size_t)(k0 + t) * nl + i + lo] : 0.0;
#pragma unroll
        for (int t = 0; t < GM_GRP; t++)
          if (k0 + t <= j) acc[k0 + t] += vk[t] * v;
      }
    } else {
      double vk[NR];
      double sm = 0.0;
#pragma unroll
      for (int k = 0; k < NR; k++) {
        vk[k] = 0.0;
        if (k <= j) {
          vk[k] = V[(size_t)k * nl + i + lo];
          sm += hs[k] * vk[k];
        }
      }
      double v = w[i] - sm;
      w[i] = v;
#pragma unroll
      for (int k = 0; k < NR; k++)
        if (k <= j) acc[k] += vk[k] * v;
    }
  }
  __shared__ double out[NR];
  if (seg_commit<NR>(acc, j + 1, A, s, out)) EpiStore{G->h2, j + 1}(out);
}

// w -= sum_{k<=j} h2[k] V[k];  ||w|| -> Givens epilogue
__global__ void __launch_bounds__(256) k_gm_orth(long long nl, const double* __restrict__ V, double* __restrict__ w,
                                                 GmresScal* G, SegArgs A, EpiGivens epi) {
  const int j = G->j;
  __shared__ double hs[GM_MAXR + 1];
  if (threadIdx.x <= (unsigned)j) hs[threadIdx.x] = G->h2[threadIdx.x];
  __syncthreads();
  int s;
  long long beg, end, lo;
  seg_chunk(A, s, beg, end, &lo);
  double acc[1] = {0.0};
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double sm = 0.0;
    for (int k = 0; k <= j; k++) sm += hs[k] * V[(size_t)k * nl + i + lo];
    double v = w[i] - sm;
    w[i] = v;
    acc[0] += v * v;
  }
  __shared__ double out[1];
  if (seg_commit<1>(acc, 1, A, s, out)) epi(out);
}

// x += Z y with y = H^{-1} g (back substitution, redundantly per block); block (0,0) also
// takes the restart decision for the outer loop
__global__ void __launch_bounds__(256) k_gm_update(long long nl, const double* __restrict__ Z, double* __restrict__ x,
                                                   GmresScal* G, LoopCtl outer, SegArgs A) {
  __shared__ double y[GM_MAXR];
  const int jj = G->jj;
  if (threadIdx.x == 0) {
    for (int i = jj - 1; i >= 0; i--) {
      double acc = G->g[i];
      for (int k = i + 1; k < jj; k++) acc -= G->H[i * GM_MAXR + k] * y[k];
      y[i] = acc / G->H[i * GM_MAXR + i];
    }
  }
  __syncthreads();
  int s;
  long long beg, end, lo;
  seg_chunk(A, s, beg, end, &lo);
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double sm = 0.0;
    for (int k = 0; k < jj; k++) sm += y[k] * Z[(size_t)k * nl + i + lo];
    if (jj > 0) x[i] += sm;
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    if (G->res <= G->target || G->brk) G->conv = 1;
    int cont = !G->conv && G->its < G->maxit;
    G->flag_outer = cont;
    outer.set(cont);
  }
}

__global__ void k_gm_reset_total(GmresScal* G) { G->total_its = 0; }

// parts per slice: a function of the global slice structure only (P-invariant): ~4096 blocks
// over all slices (several waves to stream HBM), at most one block per 1024 values
static int seg_parts(const SliceSet& st) {
  long long L = st.S_phi > 0 ? st.N : st.nbar;
  long long by_len = (L + 1023) / 1024;
  long long by_grid = std::max(1LL, 4096LL / std::max(1, st.S()));
  return (int)std::max(1LL, std::min(by_len, by_grid));
}

void DevGmres::ensure(Dev& d, const SliceSet& set_, int restart_, Comm* comm_) {
  if (restart_ > GM_MAXR) throw Error(BBOT_E_INPUT, "restart > 32 not supported");
  set = set_;
  comm = comm_;
  parts = seg_parts(set);
  const long long n_ = set.len(), nl_ = set.len_owned();
  if (n == n_ && nl == nl_ && restart == restart_ && V.p) return;
  n = n_;
  nl = nl_;
  restart = restart_;
  V.alloc((size_t)(restart + 1) * nl, d.stream);     // time slabs: the basis is slab-local (memory / P)
  Z.alloc((size_t)restart * nl, d.stream);
  w.alloc(n, d.stream);
  vin.alloc(n, d.stream);
  zout.alloc(n, d.stream);
  partial.alloc((size_t)set.S() * parts * GM_NRP, d.stream);
  tot.alloc((size_t)set.S() * GM_NRP, d.stream);
  tot.zero();
  if (counter.n != (size_t)set.S() + 1) {
    counter.alloc((size_t)set.S() + 1, d.stream);
    counter.zero();
  }
  if (!sc.p) {
    sc.alloc(1, d.stream);
    BB_CUDA(cudaMemsetAsync(sc.p, 0, sizeof(GmresScal), d.stream));
  }
}

// the slice totals of every rank to every rank: the potential and the density slices are
// two slab-partitioned ranges of the [S][GM_NRP] array
void DevGmres::allgather_tot(Dev& d) {
  if (set.S_phi > 0) comm->allgather(d, Layout::uniform(set.S_phi, GM_NRP), tot.p);
  if (set.S_rho > 0) comm->allgather(d, Layout::uniform(set.S_rho, GM_NRP), tot.p + (size_t)set.S_phi * GM_NRP);
}

void DevGmres::reset_total(Dev& d) { launch(d, k_gm_reset_total, dim3(1), dim3(1), 0, sc.p); }

void DevGmres::neg_norm(Dev& d, const double* a, double* b, double* norm) {
  const bool fused = comm == nullptr;
  launch(d, k_gm_neg_norm, dim3(parts, set.owned()), dim3(BS), 0, a, b, seg(fused ? 1 : 0), EpiNorm{norm});
  if (!fused) {
    allgather_tot(d);
    launch(d, k_seg_finish<EpiNorm>, dim3(1), dim3(BS), 0, seg(0), 1, EpiNorm{norm});
  }
}

void DevGmres::norm(Dev& d, const double* a, double* norm) {
  const bool fused = comm == nullptr;
  launch(d, k_gm_norm, dim3(parts, set.owned()), dim3(BS), 0, a, seg(fused ? 1 : 0), EpiNorm{norm});
  if (!fused) {
    allgather_tot(d);
    launch(d, k_seg_finish<EpiNorm>, dim3(1), dim3(BS), 0, seg(0), 1, EpiNorm{norm});
  }
}

void DevGmres::emit(Dev& d, Reducer& red, const DevOp& op, const DevOp& pre, const double* b, double* x,
                    const double* scale, double tol, int maxit) {
  (void)red;
  const bool fused = comm == nullptr;
  const dim3 grid(parts, set.owned());
  GmresScal* G = sc.p;
  launch(d, k_gm_init, dim3(1), dim3(1), 0, G, scale, tol, maxit, restart);
  BB_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), d.stream));
  auto finish = [&](int cnt, auto epi) {
    if (fused) return;
    allgather_tot(d);
    launch(d, k_seg_finish<decltype(epi)>, dim3(1), dim3(BS), 0, seg(0), cnt, epi);
  };
  dev_while(d, dev_field(G, &GmresScal::flag_outer), [&](const LoopCtl& outer) {
    op(x, w.p);                                               // x = 0 in the first cycle: w = 0 exactly
    launch(d, k_gm_residual, grid, dim3(BS), 0, b, w.p, seg(fused), EpiResid{G});
    finish(1, EpiResid{G});
    launch(d, k_gm_scale, grid, dim3(BS), 0, nl, (const double*)w.p, V.p, vin.p, (const GmresScal*)G, 1, seg(fused));
    dev_while(d, dev_field(G, &GmresScal::flag_inner), [&](const LoopCtl& inner) {
      pre(vin.p, zout.p);
      op(zout.p, w.p);
      // CGS2: two classical Gram-Schmidt passes; the dot counts (j + 1) live on the device,
      // the finishing kernel of the split path reads them from G as well
      if (restart <= 12)
        launch(d, k_gm_dots<true, 12>, grid, dim3(BS), 0, nl, (const double*)V.p, (const double*)w.p,
               (const double*)zout.p, Z.p, G, seg(fused));
      else
        launch(d, k_gm_dots<true, GM_MAXR>, grid, dim3(BS), 0, nl, (const double*)V.p, (const double*)w.p,
               (const double*)zout.p, Z.p, G, seg(fused));
      if (!fused) {
        allgather_tot(d);
        launch(d, k_seg_finish_dots, dim3(1), dim3(BS), 0, seg(0), G, 0);
      }
      if (restart <= 12)
        launch(d, k_gm_orth_dots<12>, grid, dim3(BS), 0, nl, (const double*)V.p, w.p, G, seg(fused));
      else
        launch(d, k_gm_orth_dots<GM_MAXR>, grid, dim3(BS), 0, nl, (const double*)V.p, w.p, G, seg(fused));
      if (!fused) {
        allgather_tot(d);
        launch(d, k_seg_finish_dots, dim3(1), dim3(BS), 0, seg(0), G, 1);
      }
      launch(d, k_gm_orth, grid, dim3(BS), 0, nl, (const double*)V.p, w.p, G, seg(fused), EpiGivens{G, inner});
      finish(1, EpiGivens{G, inner});
      launch(d, k_gm_scale, grid, dim3(BS), 0, nl, (const double*)w.p, V.p, vin.p, (const GmresScal*)G, 0,
             seg(fused));
    });
    launch(d, k_gm_update, grid, dim3(BS), 0, nl, (const double*)Z.p, x, G, outer, seg(fused));
  });
}

// ------------------------------------------------------------ per-slice PCG
__global__ void k_pcg_start(long long L, const double* __restrict__ b, double* __restrict__ r, double* s, int* its,
                            PcgScal* P, int maxit, RedArgs R, int own_begin, int own_end) {
  int k = blockIdx.y;
  const int ns = gridDim.y;
  long long beg, end;
  red_chunk(L, R.parts, beg, end);
  double acc = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double v = b[(size_t)k * L + i];
    r[(size_t)k * L + i] = v;
    acc += v * v;
  }
  if (!red_commit(acc, R)) return;
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int q = threadIdx.x; q < ns; q += blockDim.x) {
    double bn = sqrt(R.out[q]);
    s[PS_BN * ns + q] = bn;
    s[PS_RN * ns + q] = bn;
    const bool act = bn > 0.0 && q >= own_begin && q < own_end;   // other ranks' slices never iterate
    s[PS_ACTIVE * ns + q] = act ? 1.0 : 0.0;
    s[PS_BETA * ns + q] = 0.0;
    its[q] = 0;
    if (act) atomicOr(&any, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    P->it = 0;
    P->maxit = maxit;
    P->flag = (any && maxit > 0) ? 1 : 0;
  }
}

__global__ void k_pcg_rz(long long L, const double* __restrict__ r, const double* __restrict__ z, RedArgs R,
                         PcgRzFin fin) {
  int k = blockIdx.y;
  long long beg, end;
  red_chunk(L, R.parts, beg, end);
  double acc = 0.0;
  if (fin.s[PS_ACTIVE * gridDim.y + k] == 0.0) end = beg;   // converged slice
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) acc += r[(size_t)k * L + i] * z[(size_t)k * L + i];
  if (red_commit(acc, R)) fin(R.out);
}

__global__ void __launch_bounds__(256, 8) k_pcg_xr(long long L, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                         const double* __restrict__ q, double* s, const int* its, PcgScal* P, double tol, RedArgs R,
                         LoopCtl ctl) {
  int k = blockIdx.y;
  const int ns = gridDim.y;
  const double a = s[PS_ALPHA * ns + k];
  long long beg, end;
  red_chunk(L, R.parts, beg, end);
  if (s[PS_ACTIVE * ns + k] == 0.0) end = beg;   // converged slice: frozen
  double acc = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    size_t t = (size_t)k * L + i;
    x[t] += a * p[t];
    double rv = r[t] - a * q[t];
    r[t] = rv;
    acc += rv * rv;
  }
  if (!red_commit(acc, R)) return;
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int w = threadIdx.x; w < ns; w += blockDim.x) {
    double rn = sqrt(R.out[w]);
    s[PS_RN * ns + w] = rn;
    double act = s[PS_ACTIVE * ns + w];
    if (act != 0.0 && !(rn > tol * s[PS_BN * ns + w])) act = 0.0;
    s[PS_ACTIVE * ns + w] = act;
    if (act != 0.0) atomicOr(&any, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int it = P->it + 1;
    P->it = it;
    int cont = any && it < P->maxit;
    if (!cont) {
      int mx = 0;
      long long tot = 0;
      for (int w = 0; w < ns; w++) {
        mx = max(mx, its[w]);
        tot += its[w];
      }
      P->A_max = max(P->A_max, mx);
      P->A_total += tot;
    }
    ctl.set(cont);
  }
}

__global__ void k_pcg_reset(PcgScal* P) {
  P->A_max = 0;
  P->A_total = 0;
}

void DevPcg::ensure(Dev& d, long long n_, int ns_) {
  if (n == n_ && nslices == ns_ && r.p) return;
  n = n_;
  nslices = ns_;
  r.alloc(n, d.stream);
  z.alloc(n, d.stream);
  p.alloc(n, d.stream);
  q.alloc(n, d.stream);
  s.alloc((size_t)PS_COUNT * ns_, d.stream);
  its.alloc(ns_, d.stream);
  if (!sc.p) {
    sc.alloc(1, d.stream);
    BB_CUDA(cudaMemsetAsync(sc.p, 0, sizeof(PcgScal), d.stream));
  }
}

void DevPcg::reset_stats(Dev& d) { launch(d, k_pcg_reset, dim3(1), dim3(1), 0, sc.p); }

}  // namespace bbot
