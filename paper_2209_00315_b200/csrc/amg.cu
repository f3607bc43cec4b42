// amg.cu -- I3 device aggregation AMG: setup (strength graph, matching,
// Galerkin, coarsest inverse) and the V(1,1) cycle.  Definition: amg.cuh and
// DESIGN.md §2 (I3); the oracle (oracle/amg.py) implements the same algorithm
// independently.
#include "amg.cuh"
#include <climits>

namespace bbot {

constexpr double AMG_TAU = 1e-8;        // near-tie tolerance (relative)
constexpr double AMG_DECOUPLED = 1e-10; // rows with max strength <= this*|a_ii| do not propose
constexpr int MATCH_ROUNDS = 16;
constexpr int GAL_CAP = 128;            // max distinct columns of a coarse row
constexpr int MAX_LEVELS = 25;
constexpr int BS = 256;

// ------------------------------------------------------------ strength graph
template <class V>
__global__ void k_sg_count(V v, const int* __restrict__ sl, int* cnt, double* adiag) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= v.nrows) return;
  int s = sl[r];
  int c_ = 0;
  double dg = 0.0;
  v.row(r, [&](long long c, double a) {
    if (c == r) dg += a;
    else if (sl[c] == s) c_++;
  });
  cnt[r] = c_;
  adiag[r] = fabs(dg);
}

template <class V>
__global__ void k_sg_fill(V v, const int* __restrict__ sl, const long long* __restrict__ sp, int* sj,
                          double* sw) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= v.nrows) return;
  int s = sl[r];
  long long p0 = sp[r], p = p0;
  v.row(r, [&](long long c, double a) {
    if (c != r && sl[c] == s) {
      sj[p] = (int)c;
      sw[p] = fabs(a);
      p++;
    }
  });
  // insertion sort by column
  for (long long i = p0 + 1; i < p; i++) {
    int cj = sj[i];
    double cw = sw[i];
    long long j = i - 1;
    while (j >= p0 && sj[j] > cj) {
      sj[j + 1] = sj[j];
      sw[j + 1] = sw[j];
      j--;
    }
    sj[j + 1] = cj;
    sw[j + 1] = cw;
  }
}

__global__ void k_sg_sym(long long n, const long long* __restrict__ sp, const int* __restrict__ sj,
                         const double* __restrict__ sw, double* sws) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (long long p = sp[r]; p < sp[r + 1]; p++) {
    int c = sj[p];
    long long lo = sp[c], hi = sp[c + 1];
    while (lo < hi) {
      long long mid = (lo + hi) >> 1;
      if (sj[mid] < r) lo = mid + 1;
      else hi = mid;
    }
    double t = (lo < sp[c + 1] && sj[lo] == r) ? sw[lo] : 0.0;
    sws[p] = (sw[p] + t) * 0.5;
  }
}

// ------------------------------------------------------------ matching
__global__ void k_fill_i32(long long n, int* a, int v) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

__global__ void k_propose(long long n, const long long* __restrict__ sp, const int* __restrict__ sj,
                          const double* __restrict__ sw, const double* __restrict__ adiag,
                          const int* __restrict__ free_, int* prop) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  if (!free_[r]) { prop[r] = -1; return; }
  double M = -1.0;
  for (long long p = sp[r]; p < sp[r + 1]; p++)
    if (free_[sj[p]]) M = fmax(M, sw[p]);
  if (!(M > AMG_DECOUPLED * adiag[r])) { prop[r] = -1; return; }
  double thr = (1.0 - AMG_TAU) * M;
  int best = INT_MAX;
  for (long long p = sp[r]; p < sp[r + 1]; p++) {
    int c = sj[p];
    if (free_[c] && sw[p] >= thr && c < best) best = c;
  }
  prop[r] = best;
}

__global__ void k_accept(long long n, const int* __restrict__ prop, int* partner, int* free_) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int p = prop[r];
  if (free_[r] && p >= 0 && prop[p] == (int)r) {
    partner[r] = p;
    free_[r] = 0;
  }
}

__global__ void k_leader_flag(long long n, const int* __restrict__ partner, int* flag) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int p = partner[r];
  flag[r] = (p < 0 || r < p) ? 1 : 0;
}

__global__ void k_make_agg(long long n, const int* __restrict__ partner, const long long* __restrict__ cidx,
                           const int* __restrict__ sl, int* agg, int* slc) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int p = partner[r];
  long long leader = (p < 0) ? r : (r < p ? r : (long long)p);
  agg[r] = (int)cidx[leader];
  if (leader == r) slc[cidx[r]] = sl[r];
}

__global__ void k_compose(long long n, const int* __restrict__ a1, const int* __restrict__ a2, int* a) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) a[r] = a2[a1[r]];
}

// ------------------------------------------------------------ members
__global__ void k_count_members(long long n, const int* __restrict__ agg, int* cnt) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) atomicAdd(&cnt[agg[r]], 1);
}
__global__ void k_fill_members(long long n, const int* __restrict__ agg, const long long* __restrict__ mptr,
                               int* cur, int* midx) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int a = agg[r];
  int pos = atomicAdd(&cur[a], 1);
  midx[mptr[a] + pos] = (int)r;
}
__global__ void k_sort_members(long long nc, const long long* __restrict__ mptr, int* midx) {
  long long I = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nc) return;
  long long b = mptr[I], e = mptr[I + 1];
  for (long long i = b + 1; i < e; i++) {
    int v = midx[i];
    long long j = i - 1;
    while (j >= b && midx[j] > v) { midx[j + 1] = midx[j]; j--; }
    midx[j + 1] = v;
  }
}

// ------------------------------------------------------------ Galerkin
template <class V, bool FILL>
__global__ void k_galerkin(V v, long long nc, const long long* __restrict__ mptr, const int* __restrict__ midx,
                           const int* __restrict__ agg, int* cnt, const long long* __restrict__ rp, int* ci,
                           double* cv, int* err) {
  long long I = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nc) return;
  int cols[GAL_CAP];
  double vals[GAL_CAP];
  int len = 0;
  bool over = false;
  for (long long p = mptr[I]; p < mptr[I + 1]; p++) {
    long long m = midx[p];
    v.row(m, [&](long long c, double a) {
      int J = agg[c];
      int lo = 0, hi = len;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (cols[mid] < J) lo = mid + 1;
        else hi = mid;
      }
      if (lo < len && cols[lo] == J) {
        vals[lo] += a;
      } else if (len < GAL_CAP) {
        for (int q = len; q > lo; q--) { cols[q] = cols[q - 1]; vals[q] = vals[q - 1]; }
        cols[lo] = J;
        vals[lo] = a;
        len++;
      } else {
        over = true;
      }
    });
  }
  if (over) atomicExch(err, 1);
  if (!FILL) {
    cnt[I] = len;
  } else {
    long long o = rp[I];
    for (int q = 0; q < len; q++) { ci[o + q] = cols[q]; cv[o + q] = vals[q]; }
  }
}

template <class V>
__global__ void k_dinv(V v, double* dinv) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= v.nrows) return;
  double dg = 0.0;
  v.row(r, [&](long long c, double a) { if (c == r) dg += a; });
  dinv[r] = 1.0 / dg;
}

__global__ void k_slice_ptr(long long n, const int* __restrict__ sl, int nslices, long long* sptr) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int s = sl[r];
  int prev = r == 0 ? -1 : sl[r - 1];
  for (int k = prev + 1; k <= s; k++) sptr[k] = r;
  if (r == n - 1)
    for (int k = s + 1; k <= nslices; k++) sptr[k] = n;
}

// ------------------------------------------------------------ V-cycle kernels
template <class V>
__global__ void k_down(V v, const double* __restrict__ dinv, const double* __restrict__ b, double om,
                       double* __restrict__ x, double* __restrict__ res) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= v.nrows) return;
  double acc = b[r];
  v.row(r, [&](long long c, double a) { acc -= a * (om * dinv[c] * b[c]); });
  x[r] = om * dinv[r] * b[r];
  res[r] = acc;
}

__global__ void k_restrict(long long nc, const long long* __restrict__ mptr, const int* __restrict__ midx,
                           const double* __restrict__ r, double* bc) {
  long long I = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nc) return;
  double acc = 0.0;
  for (long long p = mptr[I]; p < mptr[I + 1]; p++) acc += r[midx[p]];
  bc[I] = acc;
}

template <class V>
__global__ void k_up(V v, const double* __restrict__ dinv, const double* __restrict__ b, double om,
                     const double* __restrict__ x, const int* __restrict__ agg, const double* __restrict__ xc,
                     double* __restrict__ xo) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= v.nrows) return;
  double acc = b[r];
  v.row(r, [&](long long c, double a) { acc -= a * (x[c] + xc[agg[c]]); });
  xo[r] = (x[r] + xc[agg[r]]) + om * dinv[r] * acc;
}

// ------------------------------------------------------------ coarsest
// mode A: per slice, grounded at the slice's first row; Gauss-Jordan with partial
// pivoting on [B | I] in shared memory, B = block without row/col 0.
__global__ void k_coarseA_setup(const long long* __restrict__ sptr, CsrView A, int cm, double* cinv) {
  extern __shared__ double sm[];
  int k = blockIdx.x;
  long long s0 = sptr[k];
  int nl = (int)(sptr[k + 1] - s0) - 1;   // grounded size
  if (nl <= 0) return;
  int w = 2 * nl;
  double* M = sm;                          // nl x 2nl
  __shared__ int piv;
  for (int t = threadIdx.x; t < nl * w; t += blockDim.x) M[t] = 0.0;
  __syncthreads();
  for (int i = threadIdx.x; i < nl; i += blockDim.x) {
    long long row = s0 + 1 + i;
    for (long long p = A.rp[row]; p < A.rp[row + 1]; p++) {
      long long c = A.ci[p] - (s0 + 1);
      if (c >= 0 && c < nl) M[i * w + c] += A.v[p];
    }
    M[i * w + nl + i] = 1.0;
  }
  __syncthreads();
  for (int p = 0; p < nl; p++) {
    if (threadIdx.x == 0) {
      int best = p;
      double bv = fabs(M[p * w + p]);
      for (int i = p + 1; i < nl; i++)
        if (fabs(M[i * w + p]) > bv) { bv = fabs(M[i * w + p]); best = i; }
      piv = best;
    }
    __syncthreads();
    if (piv != p)
      for (int j = threadIdx.x; j < w; j += blockDim.x) {
        double t = M[p * w + j];
        M[p * w + j] = M[piv * w + j];
        M[piv * w + j] = t;
      }
    __syncthreads();
    double pv = M[p * w + p];
    __syncthreads();
    for (int j = threadIdx.x; j < w; j += blockDim.x) M[p * w + j] /= pv;
    __syncthreads();
    for (int t = threadIdx.x; t < nl * w; t += blockDim.x) {
      int i = t / w, j = t - i * w;
      if (i != p && j != p) M[i * w + j] -= M[i * w + p] * M[p * w + j];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nl; i += blockDim.x)
      if (i != p) M[i * w + p] = 0.0;
    __syncthreads();
  }
  double* out = cinv + (size_t)k * cm * cm;
  for (int t = threadIdx.x; t < nl * nl; t += blockDim.x) {
    int i = t / nl, j = t - i * nl;
    out[i * cm + j] = M[i * w + nl + j];
  }
}

__global__ void k_coarseA_apply(const long long* __restrict__ sptr, int cm, const double* __restrict__ cinv,
                                const double* __restrict__ b, double* x) {
  __shared__ double xs[256];
  int k = blockIdx.x;
  long long s0 = sptr[k];
  int nloc = (int)(sptr[k + 1] - s0);
  if (nloc <= 0) return;
  const double* inv = cinv + (size_t)k * cm * cm;
  for (int j = threadIdx.x; j < nloc; j += blockDim.x) {
    double acc = 0.0;
    if (j > 0)
      for (int l = 1; l < nloc; l++) acc += inv[(j - 1) * cm + (l - 1)] * b[s0 + l];
    xs[j] = acc;
  }
  __syncthreads();
  double sum = 0.0;
  for (int j = threadIdx.x; j < nloc; j += blockDim.x) sum += xs[j];
  sum = block_sum(sum);
  __shared__ double mean;
  if (threadIdx.x == 0) mean = sum / nloc;
  __syncthreads();
  for (int j = threadIdx.x; j < nloc; j += blockDim.x) x[s0 + j] = xs[j] - mean;
}

// mode T: dense Gauss-Jordan in global memory, two launches per pivot
__global__ void k_csr_to_dense(CsrView A, int n, double* D, double* I) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (long long p = A.rp[r]; p < A.rp[r + 1]; p++) D[r * n + A.ci[p]] += A.v[p];
  I[r * n + r] = 1.0;
}

__global__ void k_gj_pivot(int n, int p, double* D, double* I, double* fcol) {
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  double best = -1.0;
  int besti = p;
  for (int i = p + threadIdx.x; i < n; i += blockDim.x) {
    double v = fabs(D[(size_t)i * n + p]);
    if (v > best) { best = v; besti = i; }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = besti;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      double v2 = bv[threadIdx.x + o];
      int i2 = bi[threadIdx.x + o];
      if (v2 > bv[threadIdx.x] || (v2 == bv[threadIdx.x] && i2 < bi[threadIdx.x])) {
        bv[threadIdx.x] = v2;
        bi[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  int piv = bi[0];
  if (piv != p)
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double t = D[(size_t)p * n + j]; D[(size_t)p * n + j] = D[(size_t)piv * n + j]; D[(size_t)piv * n + j] = t;
      t = I[(size_t)p * n + j]; I[(size_t)p * n + j] = I[(size_t)piv * n + j]; I[(size_t)piv * n + j] = t;
    }
  __syncthreads();
  double pv = D[(size_t)p * n + p];
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    D[(size_t)p * n + j] /= pv;
    I[(size_t)p * n + j] /= pv;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) fcol[i] = (i == p) ? 0.0 : D[(size_t)i * n + p];
}

__global__ void k_gj_elim(int n, int p, double* D, double* I, const double* __restrict__ fcol) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long tot = (long long)n * n;
  if (t >= tot) return;
  int i = (int)(t / n), j = (int)(t - (long long)i * n);
  if (i == p) return;
  double f = fcol[i];
  if (f == 0.0) return;
  if (j > p) D[(size_t)i * n + j] -= f * D[(size_t)p * n + j];
  else if (j == p) D[(size_t)i * n + j] = 0.0;
  I[(size_t)i * n + j] -= f * I[(size_t)p * n + j];
}

__global__ void k_dense_mv(int n, const double* __restrict__ A, const double* __restrict__ b, double* x) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= n) return;
  double acc = 0.0;
  for (int j = lane; j < n; j += 32) acc += A[(size_t)warp * n + j] * b[j];
  acc = warp_sum(acc);
  if (lane == 0) x[warp] = acc;
}

// view -> CSR (used when level 0 is itself the coarsest level)
template <class V>
__global__ void k_view_count(V v, int* cnt) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= v.nrows) return;
  int c_ = 0;
  v.row(r, [&](long long, double) { c_++; });
  cnt[r] = c_;
}
template <class V>
__global__ void k_view_fill(V v, const long long* __restrict__ rp, int* ci, double* cv) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= v.nrows) return;
  long long p = rp[r];
  v.row(r, [&](long long c, double a) { ci[p] = (int)c; cv[p] = a; p++; });
}

// ------------------------------------------------------------ host drivers
namespace {

struct Sg {  // strength graph work buffers
  DBuf<long long> sp;
  DBuf<int> sj;
  DBuf<double> sw, sws, adiag;
};

template <class T>
void grow(DBuf<T>& b, size_t n, cudaStream_t s) {
  if (b.n < n) b.alloc(n, s);
}

template <class V>
void match_pass(Dev& d, const V& v, const int* sl, AmgWork& w, Sg& sg, DBuf<int>& agg, long long& nc,
                DBuf<int>& slc) {
  long long n = v.nrows;
  cudaStream_t s = d.stream;
  unsigned nb = nblocks(n, BS);
  grow(w.cnt, n, s);
  grow(sg.adiag, n, s);
  launch(d, k_sg_count<V>, dim3(nb), dim3(BS), 0, v, sl, w.cnt.p, sg.adiag.p);
  grow(sg.sp, n + 1, s);
  exclusive_scan_i32(d, w.cnt.p, sg.sp.p, n, w.ws);
  long long nnz = read_scalar(d, sg.sp.p + n);
  grow(sg.sj, std::max(1LL, nnz), s);
  grow(sg.sw, std::max(1LL, nnz), s);
  grow(sg.sws, std::max(1LL, nnz), s);
  launch(d, k_sg_fill<V>, dim3(nb), dim3(BS), 0, v, sl, (const long long*)sg.sp.p, sg.sj.p, sg.sw.p);
  launch(d, k_sg_sym, dim3(nb), dim3(BS), 0, n, (const long long*)sg.sp.p, (const int*)sg.sj.p,
         (const double*)sg.sw.p, sg.sws.p);
  grow(w.free_, n, s);
  grow(w.prop, n, s);
  grow(w.partner, n, s);
  grow(w.flag, n, s);
  launch(d, k_fill_i32, dim3(nb), dim3(BS), 0, n, w.free_.p, 1);
  launch(d, k_fill_i32, dim3(nb), dim3(BS), 0, n, w.partner.p, -1);
  for (int it = 0; it < MATCH_ROUNDS; it++) {
    launch(d, k_propose, dim3(nb), dim3(BS), 0, n, (const long long*)sg.sp.p, (const int*)sg.sj.p,
           (const double*)sg.sws.p, (const double*)sg.adiag.p, (const int*)w.free_.p, w.prop.p);
    launch(d, k_accept, dim3(nb), dim3(BS), 0, n, (const int*)w.prop.p, w.partner.p, w.free_.p);
  }
  launch(d, k_leader_flag, dim3(nb), dim3(BS), 0, n, (const int*)w.partner.p, w.flag.p);
  grow(w.cidx, n + 1, s);
  exclusive_scan_i32(d, w.flag.p, w.cidx.p, n, w.ws);
  nc = read_scalar(d, w.cidx.p + n);
  agg.alloc(n, s);
  slc.alloc(std::max(1LL, nc), s);
  launch(d, k_make_agg, dim3(nb), dim3(BS), 0, n, (const int*)w.partner.p, (const long long*)w.cidx.p, sl,
         agg.p, slc.p);
}

void build_members(Dev& d, const int* agg, long long n, long long nc, DBuf<long long>& mptr, DBuf<int>& midx,
                   AmgWork& w) {
  cudaStream_t s = d.stream;
  grow(w.cnt, nc, s);
  BB_CUDA(cudaMemsetAsync(w.cnt.p, 0, nc * sizeof(int), s));
  launch(d, k_count_members, dim3(nblocks(n, BS)), dim3(BS), 0, n, agg, w.cnt.p);
  mptr.alloc(nc + 1, s);
  exclusive_scan_i32(d, w.cnt.p, mptr.p, nc, w.ws);
  midx.alloc(n, s);
  BB_CUDA(cudaMemsetAsync(w.cnt.p, 0, nc * sizeof(int), s));
  launch(d, k_fill_members, dim3(nblocks(n, BS)), dim3(BS), 0, n, agg, (const long long*)mptr.p, w.cnt.p,
         midx.p);
  launch(d, k_sort_members, dim3(nblocks(nc, BS)), dim3(BS), 0, nc, (const long long*)mptr.p, midx.p);
}

template <class V>
void galerkin(Dev& d, const V& v, long long nc, const long long* mptr, const int* midx, const int* agg,
              AmgLevel& out, AmgWork& w) {
  cudaStream_t s = d.stream;
  grow(w.cnt, nc, s);
  grow(w.err, 1, s);
  BB_CUDA(cudaMemsetAsync(w.err.p, 0, sizeof(int), s));
  unsigned nb = nblocks(nc, 128);
  launch(d, k_galerkin<V, false>, dim3(nb), dim3(128), 0, v, nc, mptr, midx, agg, w.cnt.p,
         (const long long*)nullptr, (int*)nullptr, (double*)nullptr, w.err.p);
  out.rp.alloc(nc + 1, s);
  exclusive_scan_i32(d, w.cnt.p, out.rp.p, nc, w.ws);
  long long nnz = read_scalar(d, out.rp.p + nc);
  BB_REQUIRE(read_scalar(d, w.err.p) == 0, BBOT_E_INTERNAL, "AMG Galerkin: coarse row wider than GAL_CAP");
  out.ci.alloc(std::max(1LL, nnz), s);
  out.v.alloc(std::max(1LL, nnz), s);
  launch(d, k_galerkin<V, true>, dim3(nb), dim3(128), 0, v, nc, mptr, midx, agg, (int*)nullptr,
         (const long long*)out.rp.p, out.ci.p, out.v.p, w.err.p);
  out.n = nc;
}

std::vector<long long> slice_ptrs(Dev& d, const int* sl, long long n, int nslices, AmgWork& w) {
  grow(w.lptr, nslices + 1, d.stream);
  launch(d, k_slice_ptr, dim3(nblocks(n, BS)), dim3(BS), 0, n, sl, nslices, w.lptr.p);
  std::vector<long long> h(nslices + 1);
  BB_CUDA(cudaMemcpyAsync(h.data(), w.lptr.p, (nslices + 1) * sizeof(long long), cudaMemcpyDeviceToHost,
                          d.stream));
  sync(d);
  return h;
}

}  // namespace

template <class V0>
void amg_setup(Dev& d, AmgHierarchy& H, const V0& v0, const int* slice0, int nslices, int mode, double omega,
               int coarse_max, AmgWork& w) {
  cudaStream_t s = d.stream;
  H.clear();
  H.mode = mode;
  H.omega = omega;
  H.nslices = nslices;
  H.lv.emplace_back();
  {
    AmgLevel& L0 = H.lv[0];
    L0.n = v0.nrows;
    L0.slice_of.alloc(L0.n, s);
    BB_CUDA(cudaMemcpyAsync(L0.slice_of.p, slice0, L0.n * sizeof(int), cudaMemcpyDeviceToDevice, s));
  }
  Sg sg;
  for (int l = 0;; l++) {
    long long n = H.lv[l].n;
    {
      AmgLevel& L = H.lv[l];
      L.dinv.alloc(n, s);
      L.b.alloc(n, s);
      L.x.alloc(n, s);
      L.r.alloc(n, s);
      L.xt.alloc(n, s);
      if (l == 0) launch(d, k_dinv<V0>, dim3(nblocks(n, BS)), dim3(BS), 0, v0, L.dinv.p);
      else launch(d, k_dinv<CsrView>, dim3(nblocks(n, BS)), dim3(BS), 0, L.view(), L.dinv.p);
      L.sptr = slice_ptrs(d, L.slice_of.p, n, nslices, w);
    }
    std::vector<long long>& sp = H.lv[l].sptr;
    long long maxs = 0;
    for (int k = 0; k < nslices; k++) maxs = std::max(maxs, sp[k + 1] - sp[k]);
    bool small = (mode == 0) ? (maxs <= coarse_max) : (n <= coarse_max);
    if (small || l + 1 >= MAX_LEVELS) break;
    // pass 1 on level l
    DBuf<int> agg1, sl1, agg2, sl2;
    long long nc1 = 0, nc2 = 0;
    AmgLevel A1;
    DBuf<long long> m1p;
    DBuf<int> m1i;
    if (l == 0) match_pass(d, v0, H.lv[0].slice_of.p, w, sg, agg1, nc1, sl1);
    else match_pass(d, H.lv[l].view(), H.lv[l].slice_of.p, w, sg, agg1, nc1, sl1);
    build_members(d, agg1.p, n, nc1, m1p, m1i, w);
    if (l == 0) galerkin(d, v0, nc1, m1p.p, m1i.p, agg1.p, A1, w);
    else galerkin(d, H.lv[l].view(), nc1, m1p.p, m1i.p, agg1.p, A1, w);
    // pass 2 on the Galerkin matrix of pass 1
    match_pass(d, A1.view(), sl1.p, w, sg, agg2, nc2, sl2);
    if ((double)nc2 > 0.9 * (double)n) break;
    DBuf<long long> m2p;
    DBuf<int> m2i;
    build_members(d, agg2.p, nc1, nc2, m2p, m2i, w);
    AmgLevel next;
    galerkin(d, A1.view(), nc2, m2p.p, m2i.p, agg2.p, next, w);
    next.slice_of = std::move(sl2);
    {
      AmgLevel& L = H.lv[l];
      L.nc = nc2;
      L.agg.alloc(n, s);
      launch(d, k_compose, dim3(nblocks(n, BS)), dim3(BS), 0, n, (const int*)agg1.p, (const int*)agg2.p, L.agg.p);
      build_members(d, L.agg.p, n, nc2, L.mptr, L.midx, w);
    }
    H.lv.push_back(std::move(next));
    sync(d);  // temporaries (A1, agg1, ...) are freed stream-ordered; keep host state simple
  }
  // coarsest
  AmgLevel& C = H.lv.back();
  if (H.lv.size() == 1) {   // level 0 is the coarsest: materialise it as CSR
    long long n = C.n;
    grow(w.cnt, n, s);
    launch(d, k_view_count<V0>, dim3(nblocks(n, BS)), dim3(BS), 0, v0, w.cnt.p);
    C.rp.alloc(n + 1, s);
    exclusive_scan_i32(d, w.cnt.p, C.rp.p, n, w.ws);
    long long nnz = read_scalar(d, C.rp.p + n);
    C.ci.alloc(std::max(1LL, nnz), s);
    C.v.alloc(std::max(1LL, nnz), s);
    launch(d, k_view_fill<V0>, dim3(nblocks(n, BS)), dim3(BS), 0, v0, (const long long*)C.rp.p, C.ci.p, C.v.p);
  }
  if (mode == 0) {
    long long maxs = 0;
    for (int k = 0; k < nslices; k++) maxs = std::max(maxs, C.sptr[k + 1] - C.sptr[k]);
    BB_REQUIRE(maxs <= 121, BBOT_E_INTERNAL, "AMG(A): coarsest slice block too large");
    H.cm = (int)std::max(1LL, maxs - 1);
    H.cinv.alloc((size_t)nslices * H.cm * H.cm, s);
    H.cinv.zero();
    H.csptr.alloc(nslices + 1, s);
    BB_CUDA(cudaMemcpyAsync(H.csptr.p, C.sptr.data(), (nslices + 1) * sizeof(long long), cudaMemcpyHostToDevice, s));
    size_t smem = (size_t)H.cm * 2 * H.cm * sizeof(double);
    BB_CUDA(cudaFuncSetAttribute(k_coarseA_setup, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch(d, k_coarseA_setup, dim3(nslices), dim3(256), smem, (const long long*)H.csptr.p, C.view(), H.cm, H.cinv.p);
  } else {
    long long n = C.n;
    BB_REQUIRE(n <= 8192, BBOT_E_INTERNAL, "AMG(T): coarsest level too large");
    H.cm = (int)n;
    DBuf<double> D, fcol;
    D.alloc((size_t)n * n, s);
    D.zero();
    H.cinv.alloc((size_t)n * n, s);
    H.cinv.zero();
    fcol.alloc(n, s);
    launch(d, k_csr_to_dense, dim3(nblocks(n, BS)), dim3(BS), 0, C.view(), (int)n, D.p, H.cinv.p);
    for (int p = 0; p < n; p++) {
      launch(d, k_gj_pivot, dim3(1), dim3(1024), 0, (int)n, p, D.p, H.cinv.p, fcol.p);
      launch(d, k_gj_elim, dim3(nblocks(n * n, BS)), dim3(BS), 0, (int)n, p, D.p, H.cinv.p, (const double*)fcol.p);
    }
    sync(d);
  }
  H.ready = true;
}

static void coarse_solve(Dev& d, AmgHierarchy& H, const double* b, double* x) {
  AmgLevel& C = H.lv.back();
  if (H.mode == 0)
    launch(d, k_coarseA_apply, dim3(H.nslices), dim3(128), 0, (const long long*)H.csptr.p, H.cm,
           (const double*)H.cinv.p, b, x);
  else
    launch(d, k_dense_mv, dim3(nblocks((long long)C.n * 32, 256)), dim3(256), 0, (int)C.n,
           (const double*)H.cinv.p, b, x);
}

template <class V0>
void amg_vcycle(Dev& d, AmgHierarchy& H, const V0& v0, const double* b, double* x) {
  int L = (int)H.lv.size();
  if (L == 1) { coarse_solve(d, H, b, x); return; }
  double om = H.omega;
  for (int l = 0; l < L - 1; l++) {
    AmgLevel& lv = H.lv[l];
    unsigned nb = nblocks(lv.n, BS);
    if (l == 0)
      launch(d, k_down<V0>, dim3(nb), dim3(BS), 0, v0, (const double*)lv.dinv.p, b, om, lv.x.p, lv.r.p);
    else
      launch(d, k_down<CsrView>, dim3(nb), dim3(BS), 0, lv.view(), (const double*)lv.dinv.p,
             (const double*)lv.b.p, om, lv.x.p, lv.r.p);
    launch(d, k_restrict, dim3(nblocks(lv.nc, BS)), dim3(BS), 0, lv.nc, (const long long*)lv.mptr.p,
           (const int*)lv.midx.p, (const double*)lv.r.p, H.lv[l + 1].b.p);
  }
  coarse_solve(d, H, H.lv[L - 1].b.p, H.lv[L - 1].x.p);
  for (int l = L - 2; l >= 0; l--) {
    AmgLevel& lv = H.lv[l];
    unsigned nb = nblocks(lv.n, BS);
    if (l == 0) {
      launch(d, k_up<V0>, dim3(nb), dim3(BS), 0, v0, (const double*)lv.dinv.p, b, om, (const double*)lv.x.p,
             (const int*)lv.agg.p, (const double*)H.lv[1].x.p, x);
    } else {
      launch(d, k_up<CsrView>, dim3(nb), dim3(BS), 0, lv.view(), (const double*)lv.dinv.p,
             (const double*)lv.b.p, om, (const double*)lv.x.p, (const int*)lv.agg.p,
             (const double*)H.lv[l + 1].x.p, lv.xt.p);
      std::swap(lv.x, lv.xt);
    }
  }
}

template void amg_setup<EdgeLapView>(Dev&, AmgHierarchy&, const EdgeLapView&, const int*, int, int, double, int,
                                     AmgWork&);
template void amg_setup<SliceEllView>(Dev&, AmgHierarchy&, const SliceEllView&, const int*, int, int, double, int,
                                      AmgWork&);
template void amg_vcycle<EdgeLapView>(Dev&, AmgHierarchy&, const EdgeLapView&, const double*, double*);
template void amg_vcycle<SliceEllView>(Dev&, AmgHierarchy&, const SliceEllView&, const double*, double*);

}  // namespace bbot
