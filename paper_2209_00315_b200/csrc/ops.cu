// ops.cu -- a2 (J_P matvec), pieces of the BB apply (a4), recovery (a6),
// Newton update (a7) and the kinetic energy (D12).
//
// Slice conventions (0-based): phi slice kk = 0..K holds phi^{kk+1}; state rho
// slice k0 = 0..K-1 holds rho^{k0+1}; rho_ext slice j holds rho^j (j = 0..K+1).
#include "ops.cuh"

namespace bbot {

constexpr int BS = 256;

// ---------------------------------------------------------------- generic reductions
struct WSlice {          // sum_i w_i x[k][i]   (w = nullptr -> 1)
  const double* w;
  const double* x;
  long long L;
  __device__ double operator()(int k, long long i) const {
    double v = x[(size_t)k * L + i];
    return w ? w[i] * v : v;
  }
};

__global__ void k_sub_slice(long long L, int ns, double* __restrict__ x, const double* __restrict__ S,
                            double scale) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L * ns) return;
  x[t] -= S[t / L] * scale;
}
__global__ void k_sub_slice_w_rng(long long L, long long t0, long long t1, double* __restrict__ x,
                                  const double* __restrict__ w, const double* __restrict__ S, double scale) {
  long long t = t0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= t1) return;
  long long k = t / L;
  x[t] -= w[t - k * L] * S[k] * scale;
}
// x -= w_i S[k] * scale
__global__ void k_sub_slice_w(long long L, int ns, double* __restrict__ x, const double* __restrict__ w,
                              const double* __restrict__ S, double scale) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L * ns) return;
  long long k = t / L;
  x[t] -= w[t - k * L] * S[k] * scale;
}

__global__ void k_sub_slice_rng(long long L, long long t0, long long t1, double* __restrict__ x,
                                const double* __restrict__ S, double scale) {
  long long t = t0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= t1) return;
  x[t] -= S[t / L] * scale;
}

// x -= S[k] * scale on the slices [k0, k1) of a vector of L-value slices (the full-vector
// launch when they are all of them -- identical values)
static void sub_slice(bbot_ctx* c, double* x, long long L, int k0, int k1, int ns, const double* S, double scale) {
  if (k0 == 0 && k1 == ns)
    launch(c->dev, k_sub_slice, dim3(nblocks(L * ns, BS)), dim3(BS), 0, L, ns, x, S, scale);
  else if (k1 > k0)
    launch(c->dev, k_sub_slice_rng, dim3(nblocks(L * (k1 - k0), BS)), dim3(BS), 0, L, k0 * L, k1 * L, x, S, scale);
}

// slices [k0, k1) of an ns-slice vector: arithmetic mean removed per slice
static void remove_slice_mean_rng(bbot_ctx* c, double* x, int ns, long long L, int k0, int k1) {
  double* S = c->scal.p;
  c->red.slice_sum_range(WSlice{nullptr, x, L}, L, k0, k1, ns, S);
  sub_slice(c, x, L, k0, k1, ns, S, 1.0 / (double)L);
}

void remove_slice_mean(bbot_ctx* c, double* x, int ns, long long L) {
  if (ns == c->g.K + 1 && L == c->g.N) remove_slice_mean_rng(c, x, ns, L, c->pa(), c->pb());
  else remove_slice_mean_rng(c, x, ns, L, 0, ns);
}

// ---------------------------------------------------------------- B row (coarse)
// (B x)^k_i, k = k0+1 (1-based):  Pi^T M (x^{k+1} - x^k)/dt
//   + 1/2 sum_{sigma in E(i)} R_E[sigma,i] |e| [g^k (x^k_L - x^k_R) + g^{k+1} (x^{k+1}_L - x^{k+1}_R)]  (D5, A5)
//   harmonic R_H (f4): R_E[sigma,i] -> J_H(rho-bar^k)[sigma,i] per slice (Lagrangian Hessian)
struct BRow {
  int N, NE, nbar;
  double dt;
  const double *cf, *gphi, *ce_coef, *e_len;
  const int *ce_edge, *eL, *eR;
  int harm;
  const double *lam, *rho_ext;
  __device__ double operator()(const double* x, int k0, long long i) const {
    const double* x0 = x + (size_t)k0 * N;
    const double* x1 = x + (size_t)(k0 + 1) * N;
    double tt = 0.0;
    for (int q = 0; q < 3; q++) {
      long long f = 3 * i + q;
      tt += cf[f] * (x1[f] - x0[f]);
    }
    tt /= dt;
    const double* g0 = gphi + (size_t)k0 * NE;
    const double* g1 = gphi + (size_t)(k0 + 1) * NE;
    double sp = 0.0;
    if (!harm) {
      for (int q = 0; q < CE_MAX; q++) {
        int e = ce_edge[(size_t)q * nbar + i];
        if (e < 0) break;
        int L = eL[e], R = eR[e];
        sp += ce_coef[(size_t)q * nbar + i] * e_len[e] * (g0[e] * (x0[L] - x0[R]) + g1[e] * (x1[L] - x1[R]));
      }
      return tt + 0.5 * sp;
    }
    const double* r0 = rho_ext + (size_t)k0 * nbar;
    const double* r1 = rho_ext + (size_t)(k0 + 1) * nbar;
    const double* r2 = rho_ext + (size_t)(k0 + 2) * nbar;
    for (int q = 0; q < CE_MAX; q++) {
      int e = ce_edge[(size_t)q * nbar + i];
      if (e < 0) break;
      int L = eL[e], R = eR[e];
      int pL = L / 3, pR = R / 3;
      Recon a = Recon::eval(1, lam[e], 0.5 * (r1[pL] + r0[pL]), 0.5 * (r1[pR] + r0[pR]));   // phi slice k0
      Recon b = Recon::eval(1, lam[e], 0.5 * (r2[pL] + r1[pL]), 0.5 * (r2[pR] + r1[pR]));   // phi slice k0+1
      double ja = (pL == i ? a.ja : 0.0) + (pR == i ? a.jb : 0.0);
      double jb = (pL == i ? b.ja : 0.0) + (pR == i ? b.jb : 0.0);
      sp += e_len[e] * (ja * g0[e] * (x0[L] - x0[R]) + jb * g1[e] * (x1[L] - x1[R]));
    }
    return tt + 0.5 * sp;
  }
};

// harmonic R_H (f4): (W u)_{k0,i}, W = dF_rho/drho = sum_k 1/8 (u_k u_k^T) (x) H_k (oracle ops.W):
//   1/8 [H_{k0} (u^{k0} + u^{k0-1}) + H_{k0+1} (u^{k0} + u^{k0+1})]_i   (0-based rho slices,
//   H_kk from phi slice kk), (H v)_i = sum_{sigma in E(i), two parents} D g^2 [h_ii v_i + h_ij v_j]
struct WRow {
  int nbar, NE, K;
  const int *ce_edge, *eL, *eR;
  const double *lam, *e_len, *w_len, *gphi, *rho_ext;
  __device__ double operator()(const double* y, const double* shift, double sc, int k0, long long i) const {
    auto u = [&](int k, int j) -> double {
      if (k < 0 || k >= K) return 0.0;
      double v = y[(size_t)k * nbar + j];
      return shift ? v - shift[k] * sc : v;
    };
    double acc = 0.0;
    for (int side = 0; side < 2; side++) {
      int kk = k0 + side;
      int ko = side ? k0 + 1 : k0 - 1;          // the other rho slice coupled through phi slice kk
      const double* ra = rho_ext + (size_t)(kk + 1) * nbar;
      const double* rb = rho_ext + (size_t)kk * nbar;
      const double* gk = gphi + (size_t)kk * NE;
      for (int q = 0; q < CE_MAX; q++) {
        int e = ce_edge[(size_t)q * nbar + i];
        if (e < 0) break;
        int pL = eL[e] / 3, pR = eR[e] / 3;
        if (pL == pR) continue;
        double haa, hab, hbb;
        Recon::hess(lam[e], 0.5 * (ra[pL] + rb[pL]), 0.5 * (ra[pR] + rb[pR]), haa, hab, hbb);
        double vL = u(k0, pL) + u(ko, pL), vR = u(k0, pR) + u(ko, pR);
        double hv = pL == i ? haa * vL + hab * vR : hab * vL + hbb * vR;
        acc += w_len[e] * e_len[e] * gk[e] * gk[e] * hv;
      }
    }
    return 0.125 * acc;
  }
};

// (B^T u)^k_f, k = kk+1:  M Pi (u^{k-1} - u^k)/dt + 1/2 sum_{sigma ni f} E[f,sigma] |e| g^k (R_E (u^{k-1}+u^k))_sigma
// u given as y (state layout) minus a per-slice constant shift[k0]*sc (P^T), shift may be null.  (D6)
struct BtRow {
  int N, NE, nbar, K;
  double dt;
  const double *cf, *gphi, *e_len, *lam;
  const int *fe, *eL, *eR;
  int harm;
  const double* rho_ext;
  __device__ double operator()(const double* y, const double* shift, double sc, int kk, long long f) const {
    auto u = [&](int k0, int j) -> double {
      if (k0 < 0 || k0 >= K) return 0.0;
      double v = y[(size_t)k0 * nbar + j];
      return shift ? v - shift[k0] * sc : v;
    };
    int pf = (int)(f / 3);
    double tt = cf[f] * (u(kk - 1, pf) - u(kk, pf)) / dt;
    const double* gk = gphi + (size_t)kk * NE;
    double sp = 0.0;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      int e = fe[t * N + f];
      if (e < 0) continue;
      int L = eL[e], R = eR[e];
      int pL = L / 3, pR = R / 3;
      double l = lam[e];
      double ru;
      if (!harm) {
        ru = l * (u(kk - 1, pL) + u(kk, pL)) + (1.0 - l) * (u(kk - 1, pR) + u(kk, pR));
      } else {     // J_H(rho-bar^k) (f4)
        const double* ra = rho_ext + (size_t)(kk + 1) * nbar;
        const double* rb = rho_ext + (size_t)kk * nbar;
        Recon r = Recon::eval(1, l, 0.5 * (ra[pL] + rb[pL]), 0.5 * (ra[pR] + rb[pR]));
        ru = r.ja * (u(kk - 1, pL) + u(kk, pL)) + r.jb * (u(kk - 1, pR) + u(kk, pR));
      }
      double sgn = (L == f) ? 1.0 : -1.0;
      sp += sgn * e_len[e] * gk[e] * ru;
    }
    return tt + 0.5 * sp;
  }
};

static BRow make_brow(bbot_ctx* c) {
  DevGeom& g = c->g;
  return BRow{g.N, g.NE, g.nbar, g.dt, g.c.p, c->as.gphi.p, g.ce_coef.p, g.e_len.p, g.ce_edge.p, g.eL.p, g.eR.p,
              c->opts.recon, g.lam.p, c->rho_ext.p};
}
static BtRow make_btrow(bbot_ctx* c) {
  DevGeom& g = c->g;
  return BtRow{g.N, g.NE, g.nbar, g.K, g.dt, g.c.p, c->as.gphi.p, g.e_len.p, g.lam.p, g.fadj_e.p, g.eL.p, g.eR.p,
               c->opts.recon, c->rho_ext.p};
}
static WRow make_wrow(bbot_ctx* c) {
  DevGeom& g = c->g;
  return WRow{g.nbar, g.NE, g.K, g.ce_edge.p, g.eL.p, g.eR.p, g.lam.p, g.e_len.p, g.w_len.p, c->as.gphi.p,
              c->rho_ext.p};
}

// ---------------------------------------------------------------- a2: J_P
__global__ void k_jp_y1(long long n, int N, const double* __restrict__ Aoff, const int* __restrict__ fnb, BtRow bt,
                        const double* __restrict__ x1, const double* __restrict__ x2, const double* __restrict__ S,
                        double inv_area, double* __restrict__ y1, long long t0) {
  long long t = t0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int kk = (int)(t / N);
  long long f = t - (long long)kk * N;
  const double* xs = x1 + (size_t)kk * N;
  const double* o = Aoff + (size_t)kk * 4 * N + f;
  double xf = xs[f], acc = 0.0;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    int c = fnb[q * N + f];
    if (c >= 0) acc -= o[(size_t)q * N] * (xf - xs[c]);     // omega_e (x_f - x_c), A_k x
  }
  y1[t] = acc + bt(x2, S, inv_area, kk, f);     // A x1 + B^T P^T x2
}

struct JpT {   // t = B x1 - C_H P^T x2 (C_H = C - W; W = 0 for R_E), stored; returns t (for P)
  BRow br;
  const double *x1, *x2, *S, *Cd;
  double inv_area;
  double* out;
  int nbar;
  int harm;
  WRow wr;
  __device__ double operator()(int k0, long long i) const {
    size_t t = (size_t)k0 * nbar + i;
    double u = x2[t] - S[k0] * inv_area;
    double v = br(x1, k0, i) - Cd[t] * u;
    if (harm) v += wr(x2, S, inv_area, k0, i);
    out[t] = v;
    return v;
  }
};

void jp_matvec(bbot_ctx* c, const double* x, double* y) {
  DevGeom& g = c->g;
  long long n = c->n(), m = c->m();
  int K = g.K;
  const double* x1 = x;
  const double* x2 = x + n;
  double* S1 = c->scal.p;            // c-bar weighted slice sums of x2 (P^T)
  double* S2 = c->scal.p + (K + 2);  // plain slice sums of t (P)
  if (c->slab()) {   // time slabs: one-slice halos of x1 (B, right) and x2 (B^T P^T, left), own rows only
    Layout Lp = Layout::uniform(K + 1, g.N), Lr = Layout::uniform(K, g.nbar);
    c->comm->halo(c->dev, Lp, const_cast<double*>(x1));
    c->comm->halo(c->dev, Lr, const_cast<double*>(x2));
    const int pa = c->pa(), pb = c->pb(), ra = c->ra(), rb = c->rb();
    // c-bar sums of the left halo slice (B^T P^T) -- and of the right one for W (harmonic)
    c->red.slice_sum_range(WSlice{g.cbar.p, x2, g.nbar}, g.nbar, std::max(0, ra - 1),
                           c->opts.recon ? std::min(K, rb + 1) : rb, K, S1);
    launch(c->dev, k_jp_y1, dim3(nblocks((long long)(pb - pa) * g.N, BS)), dim3(BS), 0, (long long)pb * g.N, g.N,
           (const double*)c->as.Aoff.p, (const int*)g.fadj_nb.p, make_btrow(c), x1, x2, (const double*)S1,
           1.0 / g.area, y, (long long)pa * g.N);
    c->red.slice_sum_range(JpT{make_brow(c), x1, x2, S1, c->as.Cd.p, 1.0 / g.area, y + n, g.nbar, c->opts.recon,
                               make_wrow(c)},
                           g.nbar, ra, rb, K, S2);
    if (rb > ra)
      launch(c->dev, k_sub_slice_w_rng, dim3(nblocks((long long)(rb - ra) * g.nbar, BS)), dim3(BS), 0,
             (long long)g.nbar, (long long)ra * g.nbar, (long long)rb * g.nbar, y + n, (const double*)g.cbar.p,
             (const double*)S2, 1.0 / g.area);
    return;
  }
  c->red.slice_sum(WSlice{g.cbar.p, x2, g.nbar}, g.nbar, K, S1, false);
  launch(c->dev, k_jp_y1, dim3(nblocks(n, BS)), dim3(BS), 0, n, g.N, (const double*)c->as.Aoff.p,
         (const int*)g.fadj_nb.p, make_btrow(c), x1, x2, (const double*)S1,
         1.0 / g.area, y, 0LL);
  c->red.slice_sum(JpT{make_brow(c), x1, x2, S1, c->as.Cd.p, 1.0 / g.area, y + n, g.nbar, c->opts.recon,
                       make_wrow(c)},
                   g.nbar, K, S2, false);
  launch(c->dev, k_sub_slice_w, dim3(nblocks(m, BS)), dim3(BS), 0, (long long)g.nbar, K, y + n,
         (const double*)g.cbar.p, (const double*)S2, 1.0 / g.area);
}

// ---------------------------------------------------------------- NEXT f1: SIMPLE
// J on the saddle-point system (eq:saddle-point): y1 = A x1 + B^T x2, y2 = B x1 - C x2
__global__ void k_j_y2(long long m, int nbar, BRow br, const double* __restrict__ x1, const double* __restrict__ x2,
                       const double* __restrict__ Cd, double* __restrict__ y2) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  int k0 = (int)(t / nbar);
  y2[t] = br(x1, k0, t - (long long)k0 * nbar) - Cd[t] * x2[t];
}

void j_matvec(bbot_ctx* c, const double* x, double* y) {
  DevGeom& g = c->g;
  long long n = c->n(), m = c->m();
  launch(c->dev, k_jp_y1, dim3(nblocks(n, BS)), dim3(BS), 0, n, g.N, (const double*)c->as.Aoff.p,
         (const int*)g.fadj_nb.p, make_btrow(c), x, x + n, (const double*)nullptr, 0.0, y, 0LL);
  launch(c->dev, k_j_y2, dim3(nblocks(m, BS)), dim3(BS), 0, m, g.nbar, make_brow(c), x, x + n,
         (const double*)c->as.Cd.p, y + n);
}

// SIMPLE apply (eq:sca-precs), step 1: z1 = diag(A)^-1 r1 (into w), c = r2 - B z1 (into cvec)
__global__ void k_simple_z1(long long n, const double* __restrict__ r1, const double* __restrict__ dAinv,
                            double* __restrict__ z1) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) z1[t] = r1[t] * dAinv[t];
}
__global__ void k_simple_c(long long m, int nbar, BRow br, const double* __restrict__ r2,
                           const double* __restrict__ z1, double* __restrict__ cvec) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  int k0 = (int)(t / nbar);
  cvec[t] = r2[t] - br(z1, k0, t - (long long)k0 * nbar);
}
// step 3: out1 = diag(A)^-1 (r1 - B^T z2), out2 = z2
__global__ void k_simple_out(long long n, long long m, int N, BtRow bt, const double* __restrict__ r1,
                             const double* __restrict__ dAinv, const double* __restrict__ z2,
                             double* __restrict__ out) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    int kk = (int)(t / N);
    out[t] = (r1[t] - bt(z2, nullptr, 0.0, kk, t - (long long)kk * N)) * dAinv[t];
  } else if (t < n + m) {
    out[t] = z2[t - n];
  }
}

void simple_c(bbot_ctx* c, const double* r, double* z1, double* cvec) {
  DevGeom& g = c->g;
  long long n = c->n(), m = c->m();
  launch(c->dev, k_simple_z1, dim3(nblocks(n, BS)), dim3(BS), 0, n, r, (const double*)c->as.dAinv.p, z1);
  launch(c->dev, k_simple_c, dim3(nblocks(m, BS)), dim3(BS), 0, m, g.nbar, make_brow(c), r + n, (const double*)z1,
         cvec);
}
void simple_out(bbot_ctx* c, const double* r, const double* z2, double* out) {
  long long n = c->n(), m = c->m();
  launch(c->dev, k_simple_out, dim3(nblocks(n + m, BS)), dim3(BS), 0, n, m, c->g.N, make_btrow(c), r,
         (const double*)c->as.dAinv.p, z2, out);
}

// ---------------------------------------------------------------- NEXT f2: HSS
// (oracle/hss.py; eq:prec-hss, eq:solve-K, eq:solve-laplacians)
// -c = -(b + B^ a/alpha) with a = sA r1, b = -sC r2:  -c = sC (r2 - B(dAinv r1)/alpha)
__global__ void k_hss_c(long long m, int nbar, double inv_alpha, BRow br, const double* __restrict__ r2,
                        const double* __restrict__ w, const double* __restrict__ sC, double* __restrict__ negc) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  int k0 = (int)(t / nbar);
  negc[t] = sC[t] * (r2[t] - br(w, k0, t - (long long)k0 * nbar) * inv_alpha);
}
__global__ void k_mul(long long n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ c) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) c[t] = a[t] * b[t];
}
// u = (a - B^T v)/alpha = sA (r1 - B^T(sC v))/alpha  (w = sC v)
__global__ void k_hss_u(long long n, int N, double inv_alpha, BtRow bt, const double* __restrict__ r1,
                        const double* __restrict__ w, const double* __restrict__ sA, double* __restrict__ u) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int kk = (int)(t / N);
  u[t] = sA[t] * (r1[t] - bt(w, nullptr, 0.0, kk, t - (long long)kk * N)) * inv_alpha;
}
// z1 = sA x (in place), z2 = sC v / (1 + alpha)
__global__ void k_hss_out(long long n, long long m, double inv_1pa, const double* __restrict__ sA,
                          const double* __restrict__ sC, const double* __restrict__ v, double* __restrict__ z) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) z[t] *= sA[t];
  else if (t < n + m) z[t] = sC[t - n] * v[t - n] * inv_1pa;
}

void hss_c(bbot_ctx* c, const double* r, double* negc) {
  DevGeom& g = c->g;
  long long n = c->n(), m = c->m();
  launch(c->dev, k_mul, dim3(nblocks(n, BS)), dim3(BS), 0, n, r, (const double*)c->as.dAinv.p, c->tmp_n.p);
  launch(c->dev, k_hss_c, dim3(nblocks(m, BS)), dim3(BS), 0, m, g.nbar, 1.0 / c->opts.alpha_hss, make_brow(c),
         r + n, (const double*)c->tmp_n.p, (const double*)c->as.sC.p, negc);
}
void hss_u(bbot_ctx* c, const double* r, const double* v, double* w, double* u) {
  long long n = c->n(), m = c->m();
  launch(c->dev, k_mul, dim3(nblocks(m, BS)), dim3(BS), 0, m, v, (const double*)c->as.sC.p, w);
  launch(c->dev, k_hss_u, dim3(nblocks(n, BS)), dim3(BS), 0, n, c->g.N, 1.0 / c->opts.alpha_hss, make_btrow(c), r,
         (const double*)w, (const double*)c->as.sA.p, u);
}
void hss_out(bbot_ctx* c, const double* v, double* z) {
  long long n = c->n(), m = c->m();
  launch(c->dev, k_hss_out, dim3(nblocks(n + m, BS)), dim3(BS), 0, n, m, 1.0 / (1.0 + c->opts.alpha_hss),
         (const double*)c->as.sA.p, (const double*)c->as.sC.p, v, z);
}

// ---------------------------------------------------------------- y = T x, y = A x
template <class V>
__global__ void k_spmv(V v, const double* __restrict__ x, double* __restrict__ y, long long r0, long long r1) {
  long long r = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  double acc = 0.0;
  v.row(r, [&](long long col, double a) { acc += a * x[col]; });
  y[r] = acc;
}

void apply_T(bbot_ctx* c, const double* x, double* y) {
  SliceEllView v = view_T(c);
  if (c->slab()) {   // time slabs: z halos from both neighbours (T is block tridiagonal in time), own rows
    c->comm->halo(c->dev, Layout::uniform(c->g.K, c->g.nbar), const_cast<double*>(x));
    long long r0 = (long long)c->ra() * c->g.nbar, r1 = (long long)c->rb() * c->g.nbar;
    launch(c->dev, k_spmv<SliceEllView>, dim3(nblocks(std::max(1LL, r1 - r0), BS)), dim3(BS), 0, v, x, y, r0, r1);
    return;
  }
  launch(c->dev, k_spmv<SliceEllView>, dim3(nblocks(v.nrows, BS)), dim3(BS), 0, v, x, y, 0LL, v.nrows);
}
void apply_A(bbot_ctx* c, const double* x, double* y) {
  LapView v = view_A(c);
  launch(c->dev, k_spmv<LapView>, dim3(nblocks(v.nrows, BS)), dim3(BS), 0, v, x, y, 0LL, v.nrows);
}

// ---------------------------------------------------------------- a4 pieces
struct AtZ {   // v = (Atilde_k z)_i / cbar_i, stored; returns cbar_i v (for P^T)
  int nbar, NEbar;
  const double *z, *omegabar, *cbar;
  const int *cadj_e, *cadj_nb;
  double* out;
  __device__ double operator()(int k0, long long i) const {
    const double* zs = z + (size_t)k0 * nbar;
    const double* ob = omegabar + (size_t)k0 * NEbar;
    double zi = zs[i], acc = 0.0;
    for (int t = 0; t < 3; t++) {
      int e = cadj_e[t * nbar + i];
      if (e >= 0) acc += ob[e] * (zi - zs[cadj_nb[t * nbar + i]]);
    }
    double v = acc / cbar[i];
    out[(size_t)k0 * nbar + i] = v;
    return cbar[i] * v;
  }
};

void bb_y_from_z(bbot_ctx* c, const double* z, double* y) {   // per density slice: the slab's own slices
  DevGeom& g = c->g;
  double* S = c->scal.p;
  c->red.slice_sum_range(AtZ{g.nbar, g.NEbar, z, c->as.omegabar.p, g.cbar.p, g.cadj_e.p, g.cadj_nb.p, y}, g.nbar,
                         c->ra(), c->rb(), g.K, S);
  sub_slice(c, y, g.nbar, c->ra(), c->rb(), g.K, S, 1.0 / g.area);
}

struct RhsA {  // b = r1 - B^T y, stored; returns b
  BtRow bt;
  const double *r1, *y;
  double* out;
  int N;
  __device__ double operator()(int kk, long long f) const {
    size_t t = (size_t)kk * N + f;
    double v = r1[t] - bt(y, nullptr, 0.0, kk, f);
    out[t] = v;
    return v;
  }
};

void bb_rhs_A(bbot_ctx* c, const double* r1, const double* y, double* b) {
  DevGeom& g = c->g;
  double* S = c->scal.p;
  if (c->slab()) c->comm->halo(c->dev, Layout::uniform(g.K, g.nbar), const_cast<double*>(y));   // B^T: y^{k-1}
  c->red.slice_sum_range(RhsA{make_btrow(c), r1, y, b, g.N}, g.N, c->pa(), c->pb(), g.K + 1, S);
  sub_slice(c, b, g.N, c->pa(), c->pb(), g.K + 1, S, 1.0 / (double)g.N);
}

// ---------------------------------------------------------------- solve(rhs)
// A caller-given (f; g; h) of (3.1) replaces the Newton residual
// (oracle/bb.py BBSolver.solve_rhs).  (4.17) needs 1^T f^k = 0 per slice (A30), so the
// slice masses of drho are fixed first from the phi rows' slice sums,
//   c-bar^T (drho^{k-1} - drho^k)/dt = 1^T f^k  ->  m_k = m_{k-1} - dt 1^T f^k, m_0 = 0,
// drho0^k = (m_k/|Omega|) 1, and (f - B^T drho0; g; h - s drho0) is solved; afterwards
// drho += drho0.  g~ = g - Mbar h / rho, rhs (f; P g~) (BB) or (f; g~)
// (SIMPLE), stop at eps ||(f;g;h)||_2.
__global__ void k_user_gt(long long m, int nbar, const double* __restrict__ cbar, const double* __restrict__ g,
                          const double* __restrict__ h, const double* __restrict__ rho, double* __restrict__ gt) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  int i = (int)(t % nbar);
  gt[t] = g[t] - cbar[i] * h[t] / rho[t];
}
struct SqSum {
  const double* a;
  long long L;
  __device__ double operator()(int k, long long i) const {
    double v = a[(size_t)k * L + i];
    return v * v;
  }
};
// drho0[k0][i] = m_{k0+1} / |Omega|,  m_k = -dt sum_{j<=k} Sf[j-1]  (1-based k)
__global__ void k_mass_drho0(long long m, int nbar, double dt, double inv_area, const double* __restrict__ Sf,
                             double* __restrict__ drho0) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  int k0 = (int)(t / nbar);
  double acc = 0.0;
  for (int j = 0; j <= k0; j++) acc += Sf[j];
  drho0[t] = -dt * acc * inv_area;
}
__global__ void k_user_shift(long long n, long long m, int N, BtRow bt, const double* __restrict__ drho0,
                             const double* __restrict__ s, double* __restrict__ f, double* __restrict__ h) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    int kk = (int)(t / N);
    f[t] -= bt(drho0, nullptr, 0.0, kk, t - (long long)kk * N);     // f - B^T drho0
  } else if (t < n + m) {
    h[t - n] -= s[t - n] * drho0[t - n];                                // h - s drho0
  }
}
// harmonic R_H (f4): g -= W drho0 (the (2,2) block acts on the slice-mass part too)
__global__ void k_user_gshift(long long m, int nbar, WRow wr, const double* __restrict__ drho0,
                              const double* __restrict__ gin, double* __restrict__ gout) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  int k0 = (int)(t / nbar);
  gout[t] = gin[t] - wr(drho0, nullptr, 0.0, k0, t - (long long)k0 * nbar);
}
__global__ void k_add(long long n, const double* __restrict__ a, double* __restrict__ b) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) b[t] += a[t];
}
__global__ void k_rhs2(long long m, int nbar, double area, const double* __restrict__ cbar,
                       const double* __restrict__ gt, const double* __restrict__ S, double* __restrict__ out);  // assemble.cu

void set_user_rhs(bbot_ctx* c) {   // as.f, as.g, as.h hold the caller's (f; g; h)
  DevGeom& g = c->g;
  Assembled& A = c->as;
  cudaStream_t s = c->dev.stream;
  long long n = c->n(), m = c->m();
  int K = g.K;
  double* sc = c->scal.p;
  // ||(f;g;h)|| of the caller's right-hand side
  c->red.slice_sum(SqSum{A.f.p, g.N}, g.N, K + 1, sc, false);
  c->red.slice_sum(SqSum{A.g.p, g.nbar}, g.nbar, K, sc + K + 1, false);
  c->red.slice_sum(SqSum{A.h.p, g.nbar}, g.nbar, K, sc + 2 * K + 1, false);
  std::vector<double> hs(3 * K + 1);
  BB_CUDA(cudaMemcpyAsync(hs.data(), sc, (3 * K + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
  sync(c->dev);
  // slice-mass step
  if (c->drho0.n != (size_t)m) c->drho0.alloc(m, s);
  c->red.slice_sum(WSlice{nullptr, A.f.p, g.N}, g.N, K + 1, sc, false);
  launch(c->dev, k_mass_drho0, dim3(nblocks(m, BS)), dim3(BS), 0, m, g.nbar, g.dt, 1.0 / g.area, (const double*)sc,
         c->drho0.p);
  launch(c->dev, k_user_shift, dim3(nblocks(n + m, BS)), dim3(BS), 0, n, m, g.N, make_btrow(c),
         (const double*)c->drho0.p, (const double*)c->s.p, A.f.p, A.h.p);
  if (c->opts.recon) {
    BB_CUDA(cudaMemcpyAsync(A.gt.p, A.g.p, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
    launch(c->dev, k_user_gshift, dim3(nblocks(m, BS)), dim3(BS), 0, m, g.nbar, make_wrow(c),
           (const double*)c->drho0.p, (const double*)A.gt.p, A.g.p);
  }
  // g~ and the right-hand side of (4.17) / the saddle-point system
  launch(c->dev, k_user_gt, dim3(nblocks(m, BS)), dim3(BS), 0, m, g.nbar, (const double*)g.cbar.p,
         (const double*)A.g.p, (const double*)A.h.p, (const double*)(c->rho_ext.p + g.nbar), A.gt.p);
  BB_CUDA(cudaMemcpyAsync(A.rhs.p, A.f.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (A.precond != 0) {
    BB_CUDA(cudaMemcpyAsync(A.rhs.p + n, A.gt.p, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
  } else {
    c->red.slice_sum(WSlice{nullptr, A.gt.p, g.nbar}, g.nbar, K, sc + 3 * K + 1, false);
    launch(c->dev, k_rhs2, dim3(nblocks(m, BS)), dim3(BS), 0, m, g.nbar, g.area, (const double*)g.cbar.p,
           (const double*)A.gt.p, (const double*)(sc + 3 * K + 1), A.rhs.p + n);
  }
  double tot = 0.0;
  for (double v : hs) tot += v;
  A.scale = std::sqrt(tot);
  BB_CUDA(cudaMemcpyAsync(A.dscale.p, &A.scale, sizeof(double), cudaMemcpyHostToDevice, s));
  sync(c->dev);
  A.rhs_user = true;
}

void finish_user_solve(bbot_ctx* c) {   // drho += drho0
  launch(c->dev, k_add, dim3(nblocks(c->m(), BS)), dim3(BS), 0, c->m(), (const double*)c->drho0.p, c->drho.p);
}

// ---------------------------------------------------------------- a6 recovery
struct QSum {  // q = g~ - B dphit + C_H drho ; returns q  (C_H = C - W, W = 0 for R_E)
  BRow br;
  const double *dphit, *drho, *gt, *Cd;
  int nbar;
  int harm;
  WRow wr;
  __device__ double operator()(int k0, long long i) const {
    size_t t = (size_t)k0 * nbar + i;
    double q = gt[t] - br(dphit, k0, i) + Cd[t] * drho[t];
    if (harm) q -= wr(drho, nullptr, 0.0, k0, i);
    return q;
  }
};

__global__ void k_prefix_shift(int K, double dt, double inv_area, const double* __restrict__ qs, double* shift) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double acc = 0.0;
  shift[0] = 0.0;
  for (int j = 0; j < K; j++) {
    acc += dt * (qs[j] * inv_area);      // sum_{i<k} dt dlambda^i  (4.15, A10)
    shift[j + 1] = acc;
  }
}

__global__ void k_add_shift(long long n, int N, const double* __restrict__ src, const double* __restrict__ shift,
                            double* __restrict__ dst, long long t0) {
  long long t = t0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  dst[t] = src[t] + shift[t / N];
}

__global__ void k_ds(long long m, const double* __restrict__ h, const double* __restrict__ s,
                     const double* __restrict__ drho, const double* __restrict__ rho, double* __restrict__ ds,
                     long long t0) {
  long long t = t0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  ds[t] = (h[t] - s[t] * drho[t]) / rho[t];
}

// a6 on a time slab: the same steps on the rank's own slices; B dphit needs the right
// dphit halo, the time prefix of dlambda all K slice sums (allgathered, then summed in
// order on every rank); the direction is then allgathered for the replicated update (a7)
static void recover_slab(bbot_ctx* c) {
  DevGeom& g = c->g;
  long long n = c->n(), m = c->m();
  int K = g.K;
  cudaStream_t s = c->dev.stream;
  const int pa = c->pa(), pb = c->pb(), ra = c->ra(), rb = c->rb();
  double* S = c->scal.p;
  double* shift = c->scal.p + 2 * (K + 2);
  BB_CUDA(cudaMemcpyAsync(c->drho.p, c->sol.p + n, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
  c->red.slice_sum_range(WSlice{g.cbar.p, c->drho.p, g.nbar}, g.nbar, ra, rb, K, S);
  sub_slice(c, c->drho.p, g.nbar, ra, rb, K, S, 1.0 / g.area);
  double* dphit = c->tmp_n.p;
  BB_CUDA(cudaMemcpyAsync(dphit, c->sol.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  c->red.slice_sum_range(WSlice{g.c.p, dphit, g.N}, g.N, pa, pb, K + 1, S);
  sub_slice(c, dphit, g.N, pa, pb, K + 1, S, 1.0 / g.area);
  c->comm->halo(c->dev, Layout::uniform(K + 1, g.N), dphit);
  if (c->opts.recon) c->comm->halo(c->dev, Layout::uniform(K, g.nbar), c->drho.p);   // W couples k-1, k+1
  c->red.slice_sum_range(QSum{make_brow(c), dphit, c->drho.p, c->as.gt.p, c->as.Cd.p, g.nbar, c->opts.recon, make_wrow(c)}, g.nbar, ra, rb, K, S);
  c->comm->allgather(c->dev, Layout::uniform(K, 1), S);
  launch(c->dev, k_prefix_shift, dim3(1), dim3(32), 0, K, g.dt, 1.0 / g.area, (const double*)S, shift);
  launch(c->dev, k_add_shift, dim3(nblocks((long long)(pb - pa) * g.N, BS)), dim3(BS), 0, (long long)pb * g.N, g.N,
         (const double*)dphit, (const double*)shift, c->dphi.p, (long long)pa * g.N);
  if (rb > ra)
    launch(c->dev, k_ds, dim3(nblocks((long long)(rb - ra) * g.nbar, BS)), dim3(BS), 0, (long long)rb * g.nbar,
           (const double*)c->as.h.p, (const double*)c->s.p, (const double*)c->drho.p,
           (const double*)(c->rho_ext.p + g.nbar), c->ds.p, (long long)ra * g.nbar);
  c->comm->allgather(c->dev, Layout::uniform(K + 1, g.N), c->dphi.p);
  c->comm->allgather(c->dev, Layout::uniform(K, g.nbar), c->drho.p);
  c->comm->allgather(c->dev, Layout::uniform(K, g.nbar), c->ds.p);
}

void recover(bbot_ctx* c) {
  DevGeom& g = c->g;
  long long n = c->n(), m = c->m();
  int K = g.K;
  cudaStream_t s = c->dev.stream;
  if (c->as.precond != 0) {    // SIMPLE / HSS on (eq:saddle-point): dphi = x1, drho = x2, ds
    BB_CUDA(cudaMemcpyAsync(c->dphi.p, c->sol.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    BB_CUDA(cudaMemcpyAsync(c->drho.p, c->sol.p + n, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
    launch(c->dev, k_ds, dim3(nblocks(m, BS)), dim3(BS), 0, m, (const double*)c->as.h.p, (const double*)c->s.p,
           (const double*)c->drho.p, (const double*)(c->rho_ext.p + g.nbar), c->ds.p, 0LL);
    return;
  }
  if (c->slab()) {
    recover_slab(c);
    return;
  }
  double* S = c->scal.p;
  double* shift = c->scal.p + 2 * (K + 2);
  // drho = P^T y  (A30)
  BB_CUDA(cudaMemcpyAsync(c->drho.p, c->sol.p + n, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
  c->red.slice_sum(WSlice{g.cbar.p, c->drho.p, g.nbar}, g.nbar, K, S, false);
  launch(c->dev, k_sub_slice, dim3(nblocks(m, BS)), dim3(BS), 0, (long long)g.nbar, K, c->drho.p, (const double*)S,
         1.0 / g.area);
  // dphit -= c^T dphit^k / |Omega|  (A11), kept in tmp_n
  double* dphit = c->tmp_n.p;
  BB_CUDA(cudaMemcpyAsync(dphit, c->sol.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  c->red.slice_sum(WSlice{g.c.p, dphit, g.N}, g.N, K + 1, S, false);
  launch(c->dev, k_sub_slice, dim3(nblocks(n, BS)), dim3(BS), 0, (long long)g.N, K + 1, dphit, (const double*)S,
         1.0 / g.area);
  // dlambda = E-bar(g~ - B dphit + C drho)/|Omega|
  c->red.slice_sum(QSum{make_brow(c), dphit, c->drho.p, c->as.gt.p, c->as.Cd.p, g.nbar, c->opts.recon, make_wrow(c)}, g.nbar, K, S, false);
  launch(c->dev, k_prefix_shift, dim3(1), dim3(32), 0, K, g.dt, 1.0 / g.area, (const double*)S, shift);
  launch(c->dev, k_add_shift, dim3(nblocks(n, BS)), dim3(BS), 0, n, g.N, (const double*)dphit, (const double*)shift,
         c->dphi.p, 0LL);
  launch(c->dev, k_ds, dim3(nblocks(m, BS)), dim3(BS), 0, m, (const double*)c->as.h.p, (const double*)c->s.p,
         (const double*)c->drho.p, (const double*)(c->rho_ext.p + g.nbar), c->ds.p, 0LL);
}

// ---------------------------------------------------------------- a7 update
struct RatioMin {
  long long m;
  const double *rho, *drho, *s, *ds;
  __device__ double operator()(int, long long i) const {
    double x, d;
    if (i < m) { x = rho[i]; d = drho[i]; }
    else { x = s[i - m]; d = ds[i - m]; }
    return d < 0.0 ? -x / d : 1e300;
  }
};

__global__ void k_update(long long n, long long m, double tau, const double* __restrict__ minv,
                         double* __restrict__ phi, double* __restrict__ rho, double* __restrict__ s,
                         const double* __restrict__ dphi, const double* __restrict__ drho,
                         const double* __restrict__ ds, double* __restrict__ alpha_out) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double mv = *minv;
  double a = 1.0;
  if (mv < 1e299) a = fmin(1.0, tau * mv);       // A20
  if (t == 0) *alpha_out = a;
  if (t < n) phi[t] += a * dphi[t];
  else if (t < n + m) rho[t - n] += a * drho[t - n];
  else if (t < n + 2 * m) s[t - n - m] += a * ds[t - n - m];
}

__global__ void k_renorm(long long m, int nbar, double target, const double* __restrict__ mass,
                         double* __restrict__ rho) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  rho[t] = rho[t] * (target / mass[t / nbar]);   // Remark 3.2
}

double newton_update(bbot_ctx* c, double tau) {
  DevGeom& g = c->g;
  long long n = c->n(), m = c->m();
  double* S = c->scal.p;
  double* rho = c->rho_ext.p + g.nbar;
  c->red.slice_min(RatioMin{m, rho, c->drho.p, c->s.p, c->ds.p}, 2 * m, 1, S + 3 * (g.K + 2));
  launch(c->dev, k_update, dim3(nblocks(n + 2 * m, BS)), dim3(BS), 0, n, m, tau, (const double*)(S + 3 * (g.K + 2)),
         c->phi.p, rho, c->s.p, (const double*)c->dphi.p, (const double*)c->drho.p, (const double*)c->ds.p,
         S + 3 * (g.K + 2) + 1);
  // target mass c-bar^T rho^0
  c->red.slice_sum(WSlice{g.cbar.p, c->rho_ext.p, g.nbar}, g.nbar, 1, S + 3 * (g.K + 2) + 2, false);
  c->red.slice_sum(WSlice{g.cbar.p, rho, g.nbar}, g.nbar, g.K, S, false);
  double target = read_scalar(c->dev, S + 3 * (g.K + 2) + 2);
  launch(c->dev, k_renorm, dim3(nblocks(m, BS)), dim3(BS), 0, m, g.nbar, target, (const double*)S, rho);
  c->as.valid = false;
  return read_scalar(c->dev, S + 3 * (g.K + 2) + 1);
}

// ---------------------------------------------------------------- D12
struct KeF {
  int N, NE, nbar;
  const int *eL, *eR;
  const double *lam, *e_len, *w_len, *phi, *rho_ext;
  int harm;
  __device__ double operator()(int kk, long long e) const {
    int L = eL[e], R = eR[e];
    int pL = L / 3, pR = R / 3;
    const double* ra = rho_ext + (size_t)(kk + 1) * nbar;
    const double* rb = rho_ext + (size_t)kk * nbar;
    double l = lam[e];
    double rt = Recon::eval(harm, l, 0.5 * (ra[pL] + rb[pL]), 0.5 * (ra[pR] + rb[pR])).f;   // R_E or R_H
    double dphi = phi[(size_t)kk * N + L] - phi[(size_t)kk * N + R];
    return e_len[e] * rt / w_len[e] * dphi * dphi;       // phi^T A_k phi edge by edge
  }
};

double kinetic_energy(bbot_ctx* c) {
  DevGeom& g = c->g;
  double* S = c->scal.p;
  c->red.slice_sum(KeF{g.N, g.NE, g.nbar, g.eL.p, g.eR.p, g.lam.p, g.e_len.p, g.w_len.p, c->phi.p, c->rho_ext.p, c->opts.recon},
                   g.NE, g.K + 1, S, false);
  std::vector<double> h(g.K + 1);
  BB_CUDA(cudaMemcpyAsync(h.data(), S, (g.K + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->dev.stream));
  sync(c->dev);
  double ke = 0.0;
  for (double v : h) ke += g.dt * 0.5 * v;
  return ke;
}

// ---------------------------------------------------------------- state helpers
__global__ void k_init_state(long long n, long long m, double rho0, double mu0, double* phi, double* rho, double* s) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) phi[t] = 0.0;
  if (t < m) { rho[t] = rho0; s[t] = mu0 / rho0; }
}

void init_state(bbot_ctx* c, double mu0) {
  DevGeom& g = c->g;
  double* S = c->scal.p;
  c->red.slice_sum(WSlice{g.cbar.p, c->rho_ext.p, g.nbar}, g.nbar, 1, S, false);
  double mass = read_scalar(c->dev, S);
  long long n = c->n(), m = c->m();
  launch(c->dev, k_init_state, dim3(nblocks(std::max(n, m), BS)), dim3(BS), 0, n, m, mass / g.area, mu0, c->phi.p,
         c->rho_ext.p + g.nbar, c->s.p);
  c->mu = mu0;
  c->as.valid = false;
  c->have_dir = false;
}

struct PosMin {
  long long m;
  const double *rho, *s;
  __device__ double operator()(int, long long i) const { return i < m ? rho[i] : s[i - m]; }
};

void check_state(bbot_ctx* c) {
  long long m = c->m();
  double* S = c->scal.p;
  c->red.slice_min(PosMin{m, c->rho_ext.p + c->g.nbar, c->s.p}, 2 * m, 1, S);
  double mn = read_scalar(c->dev, S);
  BB_REQUIRE(mn > 0.0, BBOT_E_STATE, "state has rho <= 0 or s <= 0");
}

}  // namespace bbot
