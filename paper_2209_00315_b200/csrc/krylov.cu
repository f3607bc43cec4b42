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
__global__ void k_neg_norm(long long n, const double* __restrict__ a, double* __restrict__ b, RedArgs R,
                           double* norm) {
  long long beg, end;
  red_chunk(n, R.parts, beg, end);
  double acc = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double v = a[i];
    b[i] = -v;
    acc += v * v;
  }
  if (red_commit(acc, R) && threadIdx.x == 0) *norm = sqrt(R.out[0]);
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
void dev_neg_norm(Dev& d, Reducer& red, const double* a, double* b, long long n, double* norm) {
  int parts = red.parts_for(n, 1);
  launch(d, k_neg_norm, dim3(parts), dim3(BS), 0, n, a, b, red.args(parts, 1, norm), norm);
}

// ------------------------------------------------------------ FGMRES kernels
// All take the device scalar block G.  Vectors have length n; V is [(r+1)][n].

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

// w = b - w (w = op(x) on entry);  beta = ||w||; start a cycle or stop
__global__ void k_gm_residual(long long n, const double* __restrict__ b, double* __restrict__ w, GmresScal* G,
                              RedArgs R) {
  long long beg, end;
  red_chunk(n, R.parts, beg, end);
  double acc = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double v = b[i] - w[i];
    w[i] = v;
    acc += v * v;
  }
  if (red_commit(acc, R) && threadIdx.x == 0) {
    double beta = sqrt(R.out[0]);
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
}

// V[j] = w / s and vin = V[j], s = beta (start) or hn (Arnoldi), only if the inner loop continues
__global__ void k_gm_scale(long long n, const double* __restrict__ w, double* __restrict__ V,
                           double* __restrict__ vin, const GmresScal* G, int start) {
  if (!G->flag_inner) return;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = start ? G->beta : G->hn;
  int j = start ? 0 : G->j;
  double v = w[i] / s;
  V[(size_t)j * n + i] = v;
  vin[i] = v;
}

// h[k] = V[k] . w for k <= j (one pass over w, one register accumulator per k);
// optionally copy zout -> Z[j] in the same pass
template <bool COPYZ, int NR>
__global__ void __launch_bounds__(256) k_gm_dots(long long n, const double* __restrict__ V,
                                                 const double* __restrict__ w, const double* __restrict__ zout,
                                                 double* __restrict__ Z, GmresScal* G, int which, RedArgs R) {
  const int j = G->j;
  long long beg, end;
  red_chunk(n, R.parts, beg, end);
  double acc[NR];
#pragma unroll
  for (int k = 0; k < NR; k++) acc[k] = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double wi = w[i];
    if (COPYZ) Z[(size_t)j * n + i] = zout[i];
#pragma unroll
    for (int k = 0; k < NR; k++)
      if (k <= j) acc[k] += V[(size_t)k * n + i] * wi;
  }
  block_sum_many<NR>(acc, j + 1, R.partial, R.parts);
  if (!red_last_block(R.counter)) return;
  double* out = which == 0 ? G->h1 : G->h2;
  red_finish(R.partial, R.parts, j + 1, out);
}

// CGS2 middle step in one pass: w -= sum_{k<=j} h1[k] V[k] (first projection),
// then h2[k] = V[k] . w for the second, reusing the V entries just loaded
template <int NR>
__global__ void __launch_bounds__(256) k_gm_orth_dots(long long n, const double* __restrict__ V,
                                                      double* __restrict__ w, GmresScal* G, RedArgs R) {
  const int j = G->j;
  __shared__ double hs[GM_MAXR + 1];
  if (threadIdx.x <= (unsigned)j) hs[threadIdx.x] = G->h1[threadIdx.x];
  __syncthreads();
  long long beg, end;
  red_chunk(n, R.parts, beg, end);
  double acc[NR];
#pragma unroll
  for (int k = 0; k < NR; k++) acc[k] = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double vk[NR];
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < NR; k++) {
      vk[k] = 0.0;
      if (k <= j) {
        vk[k] = V[(size_t)k * n + i];
        s += hs[k] * vk[k];
      }
    }
    double v = w[i] - s;
    w[i] = v;
#pragma unroll
    for (int k = 0; k < NR; k++)
      if (k <= j) acc[k] += vk[k] * v;
  }
  block_sum_many<NR>(acc, j + 1, R.partial, R.parts);
  if (!red_last_block(R.counter)) return;
  red_finish(R.partial, R.parts, j + 1, G->h2);
}

// w -= sum_{k<=j} h[k] V[k]  (h = h1 or h2); with GIVENS: partial ||w||^2 and,
// in the last block, the Hessenberg column, Givens rotations, residual estimate
// and the inner-loop decision (Saad's FGMRES).
template <bool GIVENS>
__global__ void __launch_bounds__(256) k_gm_orth(long long n, const double* __restrict__ V, double* __restrict__ w,
                                                 GmresScal* G, int which, RedArgs R, LoopCtl inner) {
  const int j = G->j;
  const double* h = which == 0 ? G->h1 : G->h2;
  __shared__ double hs[GM_MAXR + 1];
  if (threadIdx.x <= (unsigned)j) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  long long beg, end;
  red_chunk(n, R.parts, beg, end);
  double acc = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k <= j; k++) s += hs[k] * V[(size_t)k * n + i];
    double v = w[i] - s;
    w[i] = v;
    acc += v * v;
  }
  if (!GIVENS) return;
  if (!red_commit(acc, R) || threadIdx.x != 0) return;
  const int r = G->restart;
  double hn = sqrt(R.out[0]);
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

// x += Z y with y = H^{-1} g (back substitution, redundantly per block); block 0
// also takes the restart decision for the outer loop.
__global__ void __launch_bounds__(256) k_gm_update(long long n, const double* __restrict__ Z, double* __restrict__ x,
                                                   GmresScal* G, LoopCtl outer) {
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
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < jj; k++) s += y[k] * Z[(size_t)k * n + i];
    if (jj > 0) x[i] += s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (G->res <= G->target || G->brk) G->conv = 1;
    int cont = !G->conv && G->its < G->maxit;
    G->flag_outer = cont;
    outer.set(cont);
  }
}

__global__ void k_gm_reset_total(GmresScal* G) { G->total_its = 0; }

void DevGmres::ensure(Dev& d, long long n_, int restart_) {
  if (restart_ > GM_MAXR) throw Error(BBOT_E_INPUT, "restart > 32 not supported");
  if (n == n_ && restart == restart_ && V.p) return;
  n = n_;
  restart = restart_;
  V.alloc((size_t)(restart + 1) * n, d.stream);
  Z.alloc((size_t)restart * n, d.stream);
  w.alloc(n, d.stream);
  vin.alloc(n, d.stream);
  zout.alloc(n, d.stream);
  if (!sc.p) {
    sc.alloc(1, d.stream);
    BB_CUDA(cudaMemsetAsync(sc.p, 0, sizeof(GmresScal), d.stream));
  }
}

void DevGmres::reset_total(Dev& d) { launch(d, k_gm_reset_total, dim3(1), dim3(1), 0, sc.p); }

static int dot_parts_cap() {   // GPU-only tuning knob (env A/B): blocks of the CGS2 multi-dot kernels
  static const int v = [] { const char* e = getenv("BBOT_DOT_PARTS"); return e ? atoi(e) : 0; }();
  return v;
}

void DevGmres::emit(Dev& d, Reducer& red, const DevOp& op, const DevOp& pre, const double* b, double* x,
                    const double* scale, double tol, int maxit) {
  const int parts = dot_parts_cap() > 0 ? std::min(red.parts_for(n, 1), dot_parts_cap()) : red.parts_for(n, 1);
  const unsigned nb = nblocks(n, BS);
  const unsigned nb_upd = std::min<unsigned>(nb, 8u * d.num_sms);
  GmresScal* G = sc.p;
  double* rout = reinterpret_cast<double*>(dev_field(G, &GmresScal::red_out));
  launch(d, k_gm_init, dim3(1), dim3(1), 0, G, scale, tol, maxit, restart);
  BB_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), d.stream));
  dev_while(d, dev_field(G, &GmresScal::flag_outer), [&](const LoopCtl& outer) {
    op(x, w.p);                                               // x = 0 in the first cycle: w = 0 exactly
    launch(d, k_gm_residual, dim3(parts), dim3(BS), 0, n, b, w.p, G, red.args(parts, 1, rout));
    launch(d, k_gm_scale, dim3(nb), dim3(BS), 0, n, (const double*)w.p, V.p, vin.p, (const GmresScal*)G, 1);
    dev_while(d, dev_field(G, &GmresScal::flag_inner), [&](const LoopCtl& inner) {
      pre(vin.p, zout.p);
      op(zout.p, w.p);
      // CGS2: two classical Gram-Schmidt passes
      if (restart <= 12)
        launch(d, k_gm_dots<true, 12>, dim3(parts), dim3(BS), 0, n, (const double*)V.p, (const double*)w.p,
               (const double*)zout.p, Z.p, G, 0, red.args(parts, restart + 1, nullptr));
      else
        launch(d, k_gm_dots<true, GM_MAXR>, dim3(parts), dim3(BS), 0, n, (const double*)V.p, (const double*)w.p,
               (const double*)zout.p, Z.p, G, 0, red.args(parts, restart + 1, nullptr));
      if (restart <= 12)
        launch(d, k_gm_orth_dots<12>, dim3(parts), dim3(BS), 0, n, (const double*)V.p, w.p, G,
               red.args(parts, restart + 1, nullptr));
      else
        launch(d, k_gm_orth_dots<GM_MAXR>, dim3(parts), dim3(BS), 0, n, (const double*)V.p, w.p, G,
               red.args(parts, restart + 1, nullptr));
      launch(d, k_gm_orth<true>, dim3(parts), dim3(BS), 0, n, (const double*)V.p, w.p, G, 1,
             red.args(parts, 1, rout), inner);
      launch(d, k_gm_scale, dim3(nb), dim3(BS), 0, n, (const double*)w.p, V.p, vin.p, (const GmresScal*)G, 0);
    });
    launch(d, k_gm_update, dim3(nb_upd), dim3(BS), 0, n, (const double*)Z.p, x, G, outer);
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

__global__ void k_pcg_xr(long long L, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
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
