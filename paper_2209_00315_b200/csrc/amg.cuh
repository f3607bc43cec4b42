// amg.cuh -- I3: device pairwise-aggregation AMG (the role of AGMG).
//
// The algorithm is the build's own, deterministic definition (DESIGN.md §2 I3,
// identical to oracle/amg.py): strength |a_ij| within a time slice; 16
// synchronous rounds of mutual-strongest-neighbour matching with near-ties
// (relative 1e-8) broken towards the lower index; two passes per level
// (aggregates <= 4 rows); piecewise-constant prolongation; Galerkin coarse
// operators; damped-Jacobi V(1,1); coarsest: per-slice grounded dense inverse
// (mode A, singular Laplacians) or one dense inverse (mode T).
//
// Level 0 is never materialised as CSR: it is read through a "view" -- the
// edge-weight form of the blocks A_k (EdgeLapView) or the slice-shared ELL of T
// (SliceEllView).  Coarse levels are CSR (int64 row pointers).
#pragma once
#include "common.cuh"
#include "pcg_fin.cuh"

namespace bbot {

// rows r = kk*N + f;  A_k = E diag(omega_k) E^T
struct EdgeLapView {
  int N, NE;
  long long nrows;
  const int* fe;        // [4][N] fine edge ids (-1 pad)
  const int* fnb;       // [4][N] neighbours
  const double* om;     // [K+1][NE]
  template <class F>
  __device__ __forceinline__ void row(long long r, F&& f) const {
    int kk = (int)(r / N);
    int fc = (int)(r - (long long)kk * N);
    const double* w = om + (size_t)kk * NE;
    long long base = (long long)kk * N;
    double d = 0.0;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      int e = fe[t * N + fc];
      if (e >= 0) {
        double o = w[e];
        d += o;
        f(base + fnb[t * N + fc], -o);
      }
    }
    f(r, d);
  }
};

// rows r = k0*nbar + i; T values tv[((k0*3 + d)*W + s)*nbar + i], column
// (k0+d-1)*nbar + tcol[s*nbar + i]
struct SliceEllView {
  int nbar, K, W;
  long long nrows;
  const int* tcol;
  const double* tv;
  template <class F>
  __device__ __forceinline__ void row(long long r, F&& f) const {
    int k0 = (int)(r / nbar);
    int i = (int)(r - (long long)k0 * nbar);
    for (int d = 0; d < 3; d++) {
      int kk = k0 + d - 1;
      if (kk < 0 || kk >= K) continue;
      const double* vv = tv + ((size_t)(k0 * 3 + d) * W) * nbar + i;
      for (int s = 0; s < W; s++) {
        int c = tcol[(size_t)s * nbar + i];
        if (c < 0) break;
        f((long long)kk * nbar + c, vv[(size_t)s * nbar]);
      }
    }
  }
};

struct CsrView {
  long long nrows;
  const long long* rp;
  const int* ci;
  const double* v;
  template <class F>
  __device__ __forceinline__ void row(long long r, F&& f) const {
    for (long long p = rp[r]; p < rp[r + 1]; p++) f((long long)ci[p], v[p]);
  }
};

struct AmgLevel {
  long long n = 0, nc = 0;
  // CSR (levels >= 1)
  DBuf<long long> rp;
  DBuf<int> ci;
  DBuf<double> v;
  DBuf<double> dinv;
  DBuf<int> slice_of;     // row -> slice
  DBuf<int> agg;          // row -> coarse row (not at the coarsest)
  DBuf<long long> mptr;   // coarse row -> members (ascending)
  DBuf<int> midx;
  DBuf<double> b, x, r, xt;      // x: pre-smoothed iterate; xt: this level's V-cycle output
  std::vector<long long> sptr;   // host slice pointers
  DBuf<long long> dsptr;         // the same on the device (per-slice coarse tail)
  CsrView view() const { return CsrView{n, rp.p, ci.p, v.p}; }
};

struct AmgHierarchy {
  int mode = 0;            // 0 = A (per-slice grounded coarsest), 1 = T (dense coarsest)
  double omega = 0.7;
  int nslices = 0;
  std::vector<AmgLevel> lv;
  // coarsest
  DBuf<double> cinv;       // mode A: [nslices][cm][cm] (grounded), mode T: [nc][nc]
  int cm = 0;              // mode A: max rows per slice - 1; mode T: nc
  DBuf<long long> csptr;   // mode A: coarsest slice pointers (device)
  int tail = 0;            // mode A: first level handled by the per-slice tail kernel
  bool ready = false;
  void clear() { lv.clear(); ready = false; }
};

struct AmgWork {
  DBuf<int> free_, prop, partner, flag, cnt;
  DBuf<long long> cidx, ws, lptr;
  DBuf<int> err;
};

template <class V0>
void amg_setup(Dev& d, AmgHierarchy& H, const V0& v0, const int* slice0, int nslices, int mode,
               double omega, int coarse_max, AmgWork& w);
// x = one V(1,1) cycle applied to b.  If fuse != nullptr (level-0 rows are
// slice-major, fuse->L per slice) the last kernel also reduces b.x per slice and
// runs fuse->fin (the PCG r.z step); returns true iff it did.
template <class V0>
bool amg_vcycle(Dev& d, AmgHierarchy& H, const V0& v0, const double* b, double* x,
                const SliceDotFuse* fuse = nullptr);

}  // namespace bbot
