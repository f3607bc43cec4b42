// krylov.cuh -- I1/I5: right-preconditioned flexible GMRES(restart) with CGS2
// ("applied as right preconditioners within a FGMRES cycle",
// [Saad 1993]; cap P:1770) and I4: per-time-slice PCG.
//
// Device-resident: the Hessenberg matrix, Givens rotations, residual estimate,
// per-slice PCG scalars, iteration counters and loop conditions all live in
// device memory and are updated by the last block of the fused reduction that
// produces them (common.cuh).  The host only *issues* work: each solver is a
// capture function that emits kernels and device loops (dev_while), so a whole
// nested solve can be recorded once into a CUDA graph with conditional WHILE
// nodes and replayed with no host round trip, or run eagerly (host reads the
// loop flags) for per-launch profiling.  Both modes run the same kernels on the
// same data and give bitwise-identical results.
#pragma once
#include "common.cuh"
#include "pcg_fin.cuh"
#include "comm.cuh"
#include <functional>

namespace bbot {

using DevOp = std::function<void(const double*, double*)>;

constexpr int GM_MAXR = 32;   // max restart length (CGS2 dot kernel keeps one accumulator per basis vector)

// device scalar block of one GMRES instance
struct GmresScal {
  double H[(GM_MAXR + 1) * GM_MAXR];   // row-major (GM_MAXR+1) x GM_MAXR
  double cs[GM_MAXR], sn[GM_MAXR], g[GM_MAXR + 1];
  double h1[GM_MAXR + 1], h2[GM_MAXR + 1];
  double beta, res, target, hn, scale;
  double red_out[4];                    // reduction results consumed by the epilogues
  int j, its, jj, conv, brk, maxit, restart;
  int flag_outer, flag_inner;
  long long total_its;                  // accumulated over a whole Newton solve (inner T statistic)
};

// Slice structure of a Krylov vector in global layout: S_phi potential slices of N values,
// then S_rho density slices of nbar values (FGMRES on (4.17): both; T-GMRES: density only).
// A rank computes its owned slices: phi [pa, pb), rho [ra, rb) (time slabs, comm.cuh).
struct SliceSet {
  long long N = 0, nbar = 0, n_phi = 0;   // n_phi = S_phi * N (offset of the density part)
  int S_phi = 0, S_rho = 0;
  int pa = 0, pb = 0, ra = 0, rb = 0;
  __host__ __device__ int owned() const { return (pb - pa) + (rb - ra); }
  __host__ __device__ int S() const { return S_phi + S_rho; }
  __host__ __device__ long long len() const { return n_phi + (long long)S_rho * nbar; }
  // values of the owned slices (the slab-local length of the Krylov basis)
  __host__ __device__ long long len_owned() const { return (long long)(pb - pa) * N + (long long)(rb - ra) * nbar; }
  // offset of the y-th owned slice in the slab-local basis
  __host__ __device__ long long local_base(int y) const {
    return y < pb - pa ? (long long)y * N : (long long)(pb - pa) * N + (long long)(y - (pb - pa)) * nbar;
  }
  // y-th owned slice -> global slice id s, first element, length
  __device__ __forceinline__ void slice(int y, int& s, long long& base, long long& l) const {
    if (y < pb - pa) {
      s = pa + y;
      base = (long long)s * N;
      l = N;
    } else {
      int q = ra + (y - (pb - pa));
      s = S_phi + q;
      base = n_phi + (long long)q * nbar;
      l = nbar;
    }
  }
};

// Reductions of a Krylov instance (I6): every dot/norm is the sum over slices,
// in slice order, of per-slice totals, each the fixed-order sum of `parts` block partials of
// that slice -- a function of the slice lengths only, so the time-slab decomposition (any P)
// reproduces the single-GPU bits.  P = 1: the last block finishes the reduction and runs the
// epilogue in the same launch; P > 1: the slice totals are allgathered and a one-block
// kernel finishes with the same code.
constexpr int GM_NRP = GM_MAXR + 1;     // values per slice total (multi-dots)
struct SegArgs {
  SliceSet set;
  int parts;
  double* partial;      // [S][parts][GM_NRP]
  double* tot;          // [S][GM_NRP]
  unsigned* counter;    // [1 + S]: slices finished; per slice: blocks finished
  int fused;            // 1: the last block finishes (single rank)
};

struct DevGmres {
  long long n = 0;          // global vector length (w, vin, zout, x, b: global layout)
  long long nl = 0;         // slab-local length of the basis V, Z (= n on one rank)
  int restart = 0;
  SliceSet set;
  int parts = 1;
  Comm* comm = nullptr;
  DBuf<double> V, Z, w, vin, zout;     // V [(r+1)][nl], Z [r][nl] (slab-local); vin/zout: fixed pre in/out
  DBuf<double> partial, tot;
  DBuf<unsigned> counter;
  DBuf<GmresScal> sc;
  void ensure(Dev& d, const SliceSet& set_, int restart_, Comm* comm_);
  SegArgs seg(int fused) const { return SegArgs{set, parts, partial.p, tot.p, counter.p, fused}; }
  // Emit: x = FGMRES(op, pre) solution of op x = b from x0 = 0, stopping when the
  // Arnoldi residual <= tol * (*scale) (scale: device scalar).  op / pre are
  // capture functions (op(in, out), pre(in, out)) computing the owned slices of `out`
  // (they exchange the halos they need themselves); pre is always called with (vin, zout).
  // Nothing is read back.
  void emit(Dev& d, Reducer& red, const DevOp& op, const DevOp& pre, const double* b, double* x,
            const double* scale, double tol, int maxit);
  // b = -a and *norm = ||a||_2 on this instance's slice set (the inner GMRES right-hand side)
  void neg_norm(Dev& d, const double* a, double* b, double* norm);
  // *norm = ||a||_2 on this instance's slice set
  void norm(Dev& d, const double* a, double* norm);
  void reset_total(Dev& d);
  void allgather_tot(Dev& d);
};

struct DevPcg {
  long long n = 0;
  int nslices = 0;
  DBuf<double> r, z, p, q;
  DBuf<double> s;             // [8][nslices]: bn rn rz pq alpha beta active tmp
  DBuf<int> its;              // [nslices]
  DBuf<PcgScal> sc;
  void ensure(Dev& d, long long n_, int nslices_);
  // Emit: per-slice PCG on the block-diagonal operator whose rows the view V
  // yields (V::row), preconditioned by pre(r, z); x0 = 0; stop a slice at
  // ||r^k|| <= tol ||b^k||; cap maxit.  Defined below.
  // pre(r, z, fuse): z = M r; if fuse != nullptr the preconditioner must also
  // emit the per-slice reduction r.z with fuse's epilogue (fused into its last
  // kernel), else the PCG launches it separately.
  // Only slices in [own_begin, own_end) iterate (multi-GPU time slabs: the others
  // are some other rank's; they are skipped by every kernel and x is left as 0).
  template <class V, class Pre>
  void emit(Dev& d, Reducer& red, const V& view, const Pre& pre, const double* b, double* x,
            long long slice_len, double tol, int maxit, int own_begin = 0, int own_end = 1 << 30);
  void reset_stats(Dev& d);
};

// BLAS-1 helpers
void dev_copy(Dev& d, const double* a, double* b, long long n);
void dev_scale(Dev& d, const double* a, double s, double* b, long long n);
void dev_axpby(Dev& d, double alpha, const double* a, double beta, double* b, long long n);  // b = alpha a + beta b

// r = b, bn = ||b^k||, active = bn > 0, its = 0, it = 0; loop flag = any active
__global__ void k_pcg_start(long long L, const double* __restrict__ b, double* __restrict__ r, double* s, int* its,
                            PcgScal* P, int maxit, RedArgs R, int own_begin, int own_end);
// rz_new = r.z; beta (it > 0) and rz update
__global__ void k_pcg_rz(long long L, const double* __restrict__ r, const double* __restrict__ z, RedArgs R,
                         PcgRzFin fin);
// x += alpha p, r -= alpha q; rn; active &= rn > tol bn; it++; loop condition; stats at exit
__global__ void __launch_bounds__(256, 8) k_pcg_xr(long long L, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                         const double* __restrict__ q, double* s, const int* its, PcgScal* P, double tol, RedArgs R,
                         LoopCtl L_);

// p = z + beta p;  q = A z + beta q  (= A p, since q held A p_old);  partial p.q
template <class V>
__global__ void __launch_bounds__(256, BBOT_LAP_MINB) k_pcg_pq(V v, long long L, const double* __restrict__ z, double* __restrict__ p,
                         double* __restrict__ q, const double* __restrict__ s, RedArgs R, PcgAlphaFin fin) {
  int k = blockIdx.y;
  int ns = gridDim.y;
  double beta = s[PS_BETA * ns + k];
  long long beg, end;
  red_chunk(L, R.parts, beg, end);
  if (s[PS_ACTIVE * ns + k] == 0.0) end = beg;   // converged slice: frozen, nothing to do
  double acc = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    long long row = (long long)k * L + i;
    double az = 0.0;
    v.row(row, [&](long long c, double a) { az += a * z[c]; });
    double pv = z[row] + beta * p[row];
    double qv = az + beta * q[row];
    p[row] = pv;
    q[row] = qv;
    acc += pv * qv;
  }
  if (red_commit(acc, R)) fin(R.out);
}

template <class V, class Pre>
void DevPcg::emit(Dev& d, Reducer& red, const V& view, const Pre& pre, const double* b, double* x,
                  long long L, double tol, int maxit, int own_begin, int own_end) {
  const int ns = nslices;
  const int BS = Reducer::BS;
  int parts = red.parts_for(L, ns);
  double* S = s.p;
  double* out = S + PS_TMP * ns;
  BB_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), d.stream));
  BB_CUDA(cudaMemsetAsync(p.p, 0, n * sizeof(double), d.stream));
  BB_CUDA(cudaMemsetAsync(q.p, 0, n * sizeof(double), d.stream));
  launch(d, k_pcg_start, dim3(parts, ns), dim3(BS), 0, L, b, r.p, S, its.p, sc.p, maxit,
         red.args(parts, ns, out), own_begin, own_end);
  dev_while(d, dev_field(sc.p, &PcgScal::flag), [&](const LoopCtl& ctl) {
    SliceDotFuse fz{red.args(parts, ns, out), parts, ns, L, PcgRzFin{S, sc.p, ns}, S + PS_ACTIVE * ns};
    if (!pre(r.p, z.p, &fz))
      launch(d, k_pcg_rz, dim3(parts, ns), dim3(BS), 0, L, (const double*)r.p, (const double*)z.p, fz.R, fz.fin);
    launch(d, k_pcg_pq<V>, dim3(parts, ns), dim3(BS), 0, view, L, (const double*)z.p, p.p, q.p, (const double*)S,
           red.args(parts, ns, out), PcgAlphaFin{S, its.p, ns});
    launch(d, k_pcg_xr, dim3(parts, ns), dim3(BS), 0, L, x, r.p, (const double*)p.p, (const double*)q.p, S,
           (const int*)its.p, sc.p, tol, red.args(parts, ns, out), ctl);
  });
}

}  // namespace bbot
