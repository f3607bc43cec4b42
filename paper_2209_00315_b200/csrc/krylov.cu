// krylov.cu -- FGMRES(restart) with CGS2 and per-slice PCG (see krylov.cuh).
#include "krylov.cuh"
#include <cmath>

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
__global__ void k_scale_inv_dev(const double* __restrict__ a, const double* __restrict__ s, double* __restrict__ b,
                                long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double v = *s;
  if (i < n) b[i] = v > TINY ? a[i] / v : 0.0;
}
__global__ void k_axpby(double alpha, const double* __restrict__ a, double beta, double* __restrict__ b, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = alpha * a[i] + beta * b[i];
}
__global__ void k_sub(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ c, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) c[i] = a[i] - b[i];
}
// w[i] += sign * sum_k h[k] V[k][i]
__global__ void k_multi_axpy(double* __restrict__ w, const double* __restrict__ V, const double* __restrict__ h,
                             int cnt, long long n, double sign) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int k = 0; k < cnt; k++) acc += h[k] * V[(size_t)k * n + i];
  w[i] += sign * acc;
}

struct DotVW {
  const double* V;
  const double* w;
  long long n;
  __device__ double operator()(int k, long long i) const { return V[(size_t)k * n + i] * w[i]; }
};
struct Sq {
  const double* a;
  __device__ double operator()(int, long long i) const { return a[i] * a[i]; }
};
struct SliceDot {
  const double* a;
  const double* b;
  long long L;
  __device__ double operator()(int k, long long i) const { return a[(size_t)k * L + i] * b[(size_t)k * L + i]; }
};

void dev_copy(Dev& d, const double* a, double* b, long long n) {
  launch(d, k_copy, dim3(nblocks(n, BS)), dim3(BS), 0, a, b, n);
}
void dev_scale(Dev& d, const double* a, double s, double* b, long long n) {
  launch(d, k_scale, dim3(nblocks(n, BS)), dim3(BS), 0, a, s, b, n);
}
void dev_axpby(Dev& d, double alpha, const double* a, double beta, double* b, long long n) {
  launch(d, k_axpby, dim3(nblocks(n, BS)), dim3(BS), 0, alpha, a, beta, b, n);
}
double dev_norm(Dev& d, Reducer& red, const double* a, long long n, double* dscratch) {
  red.slice_sum(Sq{a}, n, 1, dscratch, true);
  return read_scalar(d, dscratch);
}

// ------------------------------------------------------------ FGMRES
void Fgmres::ensure(Dev& d, long long n_, int restart_) {
  if (n == n_ && restart == restart_ && V.p) return;
  n = n_;
  restart = restart_;
  V.alloc((size_t)(restart + 1) * n, d.stream);
  Z.alloc((size_t)restart * n, d.stream);
  w.alloc(n, d.stream);
  hdev.alloc(2 * (restart + 2) + 2, d.stream);
  ydev.alloc(restart + 1, d.stream);
  if (hhost) cudaFreeHost(hhost);
  hhost = nullptr;
  BB_CUDA(cudaMallocHost((void**)&hhost, sizeof(double) * (2 * (restart_ + 2) + 8)));
}
Fgmres::~Fgmres() {
  if (hhost) cudaFreeHost(hhost);
}

KrylovResult Fgmres::solve(Dev& d, Reducer& red, const DevOp& op, const DevOp& pre, const double* b, double* x,
                           double scale, double tol, int maxit) {
  KrylovResult R;
  const double target = tol * scale;
  unsigned nb = nblocks(n, BS);
  BB_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), d.stream));
  double* hd = hdev.p;                      // [0..r]: h, [r+1..2r+1]: h2, [2r+2]: norm
  const int r = restart;
  // r0 = b
  red.slice_sum(Sq{b}, n, 1, hd + 2 * r + 2, true);
  double beta = read_scalar(d, hd + 2 * r + 2);
  if (!(beta > target)) { R.converged = true; R.res = beta; return R; }
  launch(d, k_scale, dim3(nb), dim3(BS), 0, b, 1.0 / beta, V.p, n);
  std::vector<double> H((size_t)(r + 1) * r), cs(r), sn(r), g(r + 1), y(r);
  double res = beta;
  int its = 0;
  bool conv = false;
  while (true) {
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int jj = 0;
    bool breakdown = false;
    for (int j = 0; j < r; j++) {
      double* Vj = V.p + (size_t)j * n;
      double* Zj = Z.p + (size_t)j * n;
      pre(Vj, Zj);
      op(Zj, w.p);
      its++;
      // CGS2
      red.slice_sum(DotVW{V.p, w.p, n}, n, j + 1, hd, false);
      launch(d, k_multi_axpy, dim3(nb), dim3(BS), 0, w.p, (const double*)V.p, (const double*)hd, j + 1, n, -1.0);
      red.slice_sum(DotVW{V.p, w.p, n}, n, j + 1, hd + r + 1, false);
      launch(d, k_multi_axpy, dim3(nb), dim3(BS), 0, w.p, (const double*)V.p, (const double*)(hd + r + 1), j + 1,
             n, -1.0);
      red.slice_sum(Sq{w.p}, n, 1, hd + 2 * r + 2, true);
      launch(d, k_scale_inv_dev, dim3(nb), dim3(BS), 0, (const double*)w.p, (const double*)(hd + 2 * r + 2),
             V.p + (size_t)(j + 1) * n, n);
      BB_CUDA(cudaMemcpyAsync(hhost, hd, sizeof(double) * (2 * r + 3), cudaMemcpyDeviceToHost, d.stream));
      sync(d);
      double hn = hhost[2 * r + 2];
      for (int i = 0; i <= j; i++) H[(size_t)i * r + j] = hhost[i] + hhost[r + 1 + i];
      H[(size_t)(j + 1) * r + j] = hn;
      for (int i = 0; i < j; i++) {
        double t = cs[i] * H[(size_t)i * r + j] + sn[i] * H[(size_t)(i + 1) * r + j];
        H[(size_t)(i + 1) * r + j] = -sn[i] * H[(size_t)i * r + j] + cs[i] * H[(size_t)(i + 1) * r + j];
        H[(size_t)i * r + j] = t;
      }
      double den = std::hypot(H[(size_t)j * r + j], H[(size_t)(j + 1) * r + j]);
      cs[j] = H[(size_t)j * r + j] / den;
      sn[j] = H[(size_t)(j + 1) * r + j] / den;
      H[(size_t)j * r + j] = den;
      H[(size_t)(j + 1) * r + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      res = std::fabs(g[j + 1]);
      jj = j + 1;
      if (hn <= TINY) breakdown = true;
      if (res <= target || its >= maxit || breakdown) break;
    }
    for (int i = jj - 1; i >= 0; i--) {
      double acc = g[i];
      for (int k = i + 1; k < jj; k++) acc -= H[(size_t)i * r + k] * y[k];
      y[i] = acc / H[(size_t)i * r + i];
    }
    BB_CUDA(cudaMemcpyAsync(ydev.p, y.data(), jj * sizeof(double), cudaMemcpyHostToDevice, d.stream));
    launch(d, k_multi_axpy, dim3(nb), dim3(BS), 0, x, (const double*)Z.p, (const double*)ydev.p, jj, n, 1.0);
    sync(d);  // y lives on the host stack
    if (res <= target || breakdown) { conv = true; break; }
    if (its >= maxit) break;
    // restart with the true residual
    op(x, w.p);
    launch(d, k_sub, dim3(nb), dim3(BS), 0, b, (const double*)w.p, w.p, n);
    red.slice_sum(Sq{w.p}, n, 1, hd + 2 * r + 2, true);
    beta = read_scalar(d, hd + 2 * r + 2);
    res = beta;
    if (beta <= target) { conv = true; break; }
    launch(d, k_scale, dim3(nb), dim3(BS), 0, (const double*)w.p, 1.0 / beta, V.p, n);
  }
  R.its = its;
  R.converged = conv;
  R.res = res;
  return R;
}

// ------------------------------------------------------------ per-slice PCG
// sc layout: [0] bn [1] rn [2] rz [3] rzn [4] pq [5] alpha [6] beta [7] active, each nslices
__global__ void k_pcg_init(int ns, double* sc, int* its) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ns) return;
  sc[7 * ns + k] = sc[0 * ns + k] > 0.0 ? 1.0 : 0.0;
  sc[1 * ns + k] = sc[0 * ns + k];
  its[k] = 0;
}
__global__ void k_pcg_alpha(int ns, double* sc, int* its) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ns) return;
  double act = sc[7 * ns + k];
  double pq = sc[4 * ns + k];
  if (act != 0.0 && !(pq > 0.0)) act = 0.0;
  sc[7 * ns + k] = act;
  sc[5 * ns + k] = act != 0.0 ? sc[2 * ns + k] / pq : 0.0;
  its[k] += act != 0.0 ? 1 : 0;
}
__global__ void k_pcg_xr(long long L, int ns, const double* __restrict__ sc, double* __restrict__ x,
                         double* __restrict__ r, const double* __restrict__ p, const double* __restrict__ q) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L * ns) return;
  double a = sc[5 * ns + i / L];
  x[i] += a * p[i];
  r[i] -= a * q[i];
}
__global__ void k_pcg_check(int ns, double* sc, double tol, int* any) {
  // single block
  int cnt = 0;
  for (int k = threadIdx.x; k < ns; k += blockDim.x) {
    double act = sc[7 * ns + k];
    if (act != 0.0 && !(sc[1 * ns + k] > tol * sc[0 * ns + k])) act = 0.0;
    sc[7 * ns + k] = act;
    cnt += act != 0.0;
  }
  cnt = __syncthreads_count(cnt > 0);
  if (threadIdx.x == 0) *any = cnt;
}
__global__ void k_pcg_beta(int ns, double* sc) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ns) return;
  double act = sc[7 * ns + k];
  double rz = sc[2 * ns + k], rzn = sc[3 * ns + k];
  sc[6 * ns + k] = act != 0.0 ? rzn / (rz != 0.0 ? rz : 1.0) : 0.0;
  if (act != 0.0) sc[2 * ns + k] = rzn;
}
__global__ void k_pcg_p(long long L, int ns, const double* __restrict__ sc, const double* __restrict__ z,
                        double* __restrict__ p) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L * ns) return;
  p[i] = z[i] + sc[6 * ns + i / L] * p[i];
}

std::vector<int> PcgSlices::solve(Dev& d, Reducer& red, const DevOp& op, const DevOp& pre, const double* b,
                                  double* x, int ns, long long L, double tol, int maxit) {
  long long N = L * ns;
  cudaStream_t s = d.stream;
  if (n != N) {
    n = N;
    r.alloc(N, s); z.alloc(N, s); p.alloc(N, s); q.alloc(N, s);
  }
  if (nslices != ns || !sc.p) {
    nslices = ns;
    sc.alloc(8 * (size_t)ns, s);
    its.alloc(ns, s);
    any.alloc(1, s);
  }
  unsigned nb = nblocks(N, BS), nbs = nblocks(ns, 128);
  double* S = sc.p;
  BB_CUDA(cudaMemsetAsync(x, 0, N * sizeof(double), s));
  dev_copy(d, b, r.p, N);
  red.slice_sum(SliceDot{b, b, L}, L, ns, S + 0 * ns, true);
  launch(d, k_pcg_init, dim3(nbs), dim3(128), 0, ns, S, its.p);
  launch(d, k_pcg_check, dim3(1), dim3(1024), 0, ns, S, -1.0, any.p);  // any active?
  std::vector<int> out(ns, 0);
  if (read_scalar(d, any.p) == 0) return out;
  pre(r.p, z.p);
  dev_copy(d, z.p, p.p, N);
  red.slice_sum(SliceDot{r.p, z.p, L}, L, ns, S + 2 * ns, false);
  for (int it = 0; it < maxit; it++) {
    op(p.p, q.p);
    red.slice_sum(SliceDot{p.p, q.p, L}, L, ns, S + 4 * ns, false);
    launch(d, k_pcg_alpha, dim3(nbs), dim3(128), 0, ns, S, its.p);
    launch(d, k_pcg_xr, dim3(nb), dim3(BS), 0, L, ns, (const double*)S, x, r.p, (const double*)p.p,
           (const double*)q.p);
    red.slice_sum(SliceDot{r.p, r.p, L}, L, ns, S + 1 * ns, true);
    launch(d, k_pcg_check, dim3(1), dim3(1024), 0, ns, S, tol, any.p);
    if (read_scalar(d, any.p) == 0) break;
    pre(r.p, z.p);
    red.slice_sum(SliceDot{r.p, z.p, L}, L, ns, S + 3 * ns, false);
    launch(d, k_pcg_beta, dim3(nbs), dim3(128), 0, ns, S);
    launch(d, k_pcg_p, dim3(nb), dim3(BS), 0, L, ns, (const double*)S, (const double*)z.p, p.p);
  }
  BB_CUDA(cudaMemcpyAsync(out.data(), its.p, ns * sizeof(int), cudaMemcpyDeviceToHost, s));
  sync(d);
  return out;
}

}  // namespace bbot
