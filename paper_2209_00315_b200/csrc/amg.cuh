// amg.cuh -- I3: device aggregation AMG (the role of AGMG).
//
// The algorithm is the build's own, deterministic definition (DESIGN.md §2 I3,
// identical to oracle/amg.py): strength (|a_ij| + |a_ji|)/2 within a time slice;
// 16 synchronous rounds of mutual-strongest-neighbour matching, near-ties
// (relative 1e-8) broken by a fixed hash priority; leftover rows attached to the
// pair of their strongest matched neighbour; two passes per level;
// piecewise-constant prolongation; Galerkin coarse operators; damped-Jacobi
// V(1,1); K-cycle coarse corrections on deep AMG(A) hierarchies; coarsest:
// per-slice grounded dense inverse (mode A, singular Laplacians) or one dense
// inverse (mode T).
//
// Level 0 is never materialised as CSR: it is read through a "view" -- the
// cell-ELL form of the blocks A_k (LapView) or the slice-shared ELL of T
// (SliceEllView).  Coarse levels: CSR for setup, SELL-32 for the sweeps.
#pragma once
#include "common.cuh"
#include "pcg_fin.cuh"

namespace bbot {

// rows r = kk*N + f;  A_k = E diag(omega_k) E^T, stored per cell
// ("cell-ELL"): off[(kk*4 + t)*N + f] = -omega of the t-th edge of kite f (0 pad),
// neighbour nb[t*N + f] (-1 pad, shared by all slices).  Slot-major, so a warp
// reads 32 consecutive doubles per slot; the diagonal is recomputed as the sum
// of the edge weights in slot order (no separate array).
struct LapView {
  int N;
  long long nrows;
  const int* nb;        // [4][N]
  const double* off;    // [K+1][4][N]
  template <class F>
  __device__ __forceinline__ void row(long long r, F&& f) const {
    int kk = (int)(r / N);
    int fc = (int)(r - (long long)kk * N);
    const double* o = off + (size_t)kk * 4 * N + fc;
    long long base = (long long)kk * N;
    double d = 0.0;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      int c = nb[t * N + fc];
      if (c >= 0) {
        double a = o[(size_t)t * N];
        d -= a;
        f(base + c, a);
      }
    }
    f(r, d);
  }
  // slice-batched kernels: the neighbour slots of kite fc, loaded once and shared by
  // the rows kk*N + fc of several slices (nb is common to all slices)
  __device__ __forceinline__ void nbrs(int fc, int (&c)[4]) const {
#pragma unroll
    for (int t = 0; t < 4; t++) c[t] = nb[t * N + fc];
  }
  // row kk*N + fc with preloaded slots: row()'s entries, values and order exactly
  template <class F>
  __device__ __forceinline__ void row_nb(int kk, int fc, const int (&c)[4], F&& f) const {
    const double* o = off + (size_t)kk * 4 * N + fc;
    long long base = (long long)kk * N;
    double d = 0.0;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      if (c[t] >= 0) {
        double a = o[(size_t)t * N];
        d -= a;
        f(base + c[t], a);
      }
    }
    f(base + fc, d);
  }
};

// HSS (NEXT f2): the diagonally scaled, shifted blocks
//   Â_k + alpha I = D_A^{-1/2} A_k D_A^{-1/2} + alpha I,  sA = D_A^{-1/2} (per row),
// read from the same cell-ELL storage as LapView (nothing extra is stored).
struct ScaledLapView {
  int N;
  long long nrows;
  const int* nb;        // [4][N]
  const double* off;    // [K+1][4][N]
  const double* sA;     // [n]
  double alpha;
  template <class F>
  __device__ __forceinline__ void row(long long r, F&& f) const {
    int kk = (int)(r / N);
    int fc = (int)(r - (long long)kk * N);
    const double* o = off + (size_t)kk * 4 * N + fc;
    long long base = (long long)kk * N;
    const double sr = sA[r];
    double d = 0.0;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      int c = nb[t * N + fc];
      if (c >= 0) {
        double a = o[(size_t)t * N];
        d -= a;
        f(base + c, a * sr * sA[base + c]);
      }
    }
    f(r, d * sr * sr + alpha);
  }
};

// rows r = k0*nbar + i; T values tv[((k0*3 + d)*W + s)*nbar + i], column
// (k0+d-1)*nbar + tcol[s*nbar + i]; unused slots (tcol = -1) hold exactly 0 and
// are read as column i (adds an exact 0; no data-dependent loop exit)
struct SliceEllView {
  int nbar, K, W;
  long long nrows;
  const int* tcol;
  const double* tv;
  // common width of the refined meshes, fully unrolled: the W column indices
  // (shared by the three time offsets) and each block's W values are loaded before
  // any gather is issued -- more independent loads in flight per warp.  Same
  // callback order as the generic loop (bitwise identical results).
  template <int WC, class F>
  __device__ __forceinline__ void row_fixed(int k0, int i, F&& f) const {
    int cols[WC];
#pragma unroll
    for (int s = 0; s < WC; s++) {
      int c = tcol[(size_t)s * nbar + i];
      cols[s] = c < 0 ? i : c;
    }
#pragma unroll
    for (int d = 0; d < 3; d++) {
      int kk = k0 + d - 1;
      if (kk < 0 || kk >= K) continue;
      const double* vv = tv + ((size_t)(k0 * 3 + d) * WC) * nbar + i;
      double vals[WC];
#pragma unroll
      for (int s = 0; s < WC; s++) vals[s] = vv[(size_t)s * nbar];
      const long long base = (long long)kk * nbar;
#pragma unroll
      for (int s = 0; s < WC; s++) f(base + cols[s], vals[s]);
    }
  }
  template <class F>
  __device__ __forceinline__ void row(long long r, F&& f) const {
    int k0 = (int)(r / nbar);
    int i = (int)(r - (long long)k0 * nbar);
    if (W == 10) {
      row_fixed<10>(k0, i, f);
      return;
    }
    for (int d = 0; d < 3; d++) {
      int kk = k0 + d - 1;
      if (kk < 0 || kk >= K) continue;
      const double* vv = tv + ((size_t)(k0 * 3 + d) * W) * nbar + i;
#pragma unroll 4
      for (int s = 0; s < W; s++) {
        int c = tcol[(size_t)s * nbar + i];
        f((long long)kk * nbar + (c < 0 ? i : c), vv[(size_t)s * nbar]);
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

// SELL-32: rows in chunks of 32; chunk c holds w[c] slots of 32 entries
// (slot-major: entry s of row r at off[c] + s*32 + (r & 31)), columns in CSR
// order, padded with (column r, value 0) so the slot loop has no data-dependent
// exit and its loads issue back to back (a padded term adds an exact 0).  A
// warp reads one 256-byte segment per slot.  Used by the V-cycle sweeps of the
// coarse levels; setup keeps the CSR.
struct SellView {
  long long nrows;
  const long long* off;
  const int* w;
  const int* ci;
  const double* v;
  template <class F>
  __device__ __forceinline__ void row(long long r, F&& f) const {
    long long ch = r >> 5;
    long long base = off[ch] + (r & 31);
    int wc = w[ch];
#pragma unroll 4
    for (int s = 0; s < wc; s++) f((long long)ci[base + (long long)s * 32], v[base + (long long)s * 32]);
  }
};

// Skip rows of converged time slices (PCG on the block-diagonal A, mode A only):
// AMG(A) never couples slices, so leaving a frozen slice's rows untouched changes
// nothing on the active ones.  active == nullptr: no skipping.
struct SliceSkip {
  const double* active;   // [nslices] 1.0 / 0.0
  const int* slice_of;    // row -> slice (coarse levels), or nullptr: slice = row / L
  long long L;
  __device__ __forceinline__ bool skip(long long r) const {
    if (!active) return false;
    long long k = slice_of ? (long long)slice_of[r] : r / L;
    return active[k] == 0.0;
  }
};

// rows [r0, r1) of a level a launch covers (time slabs: the rank's own slices)
struct RowRange {
  long long r0, r1;
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
  DBuf<double> kc1, kv, krc;     // K-cycle work vectors (mode A tail levels)
  std::vector<long long> sptr;   // host slice pointers
  DBuf<long long> dsptr;         // the same on the device (per-slice coarse tail)
  DBuf<long long> sl_off;        // SELL-32 copy of the CSR (V-cycle sweeps)
  DBuf<int> sl_w, sl_ci;
  DBuf<double> sl_v;
  SellView sell() const { return SellView{n, sl_off.p, sl_w.p, sl_ci.p, sl_v.p}; }
  CsrView view() const { return CsrView{n, rp.p, ci.p, v.p}; }
};

struct AmgHierarchy {
  int mode = 0;            // 0 = A (per-slice grounded coarsest), 1 = T (dense coarsest),
                           // 2 = As (HSS shifted blocks: per slice, nonsingular coarsest)
  double omega = 0.7;
  int nslices = 0;
  std::vector<AmgLevel> lv;
  // coarsest
  DBuf<double> cinv;       // mode A: [nslices][cm][cm] (grounded), mode T: [nc][nc]
  int cm = 0;              // mode A: max rows per slice - 1; mode T: nc
  DBuf<long long> csptr;   // mode A: coarsest slice pointers (device)
  int tail = 0;            // mode A: first level handled by the per-slice tail kernel
  DBuf<char> tail_args;    // the tail kernel's level table (device; TailArgs / TailTArgs)
  int tail_cl = 1;         // cluster size of the tail launch
  bool cjac = false;       // mode T: coarsening stalled above coarse_max -> the coarsest "solve"
                           // is one l1-Jacobi sweep from zero (exact on a diagonal matrix)
  bool ready = false;
  void clear() { lv.clear(); ready = false; tail = 0; tail_cl = 1; cjac = false; }
};

struct AmgWork {
  DBuf<int> free_, prop, partner, flag, cnt;
  DBuf<long long> cidx, ws, lptr;
  DBuf<long long> ub, goff;      // Galerkin: per coarse row entry bound, scratch offsets
  DBuf<int> gcols;
  DBuf<double> gvals;
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
                const SliceDotFuse* fuse = nullptr, const double* active = nullptr);
// The V-cycle of a mode-T hierarchy (AMG(T)) on the time slab of a multi-rank context: every
// grid-wide level sweeps its own slices' rows [ra, rb) (slice-grouped coarse rows) after a
// one-slice halo exchange of the vector the sweep gathers from; the coarse tail (or the
// coarsest solve) runs redundantly on every rank on the allgathered input.  Same sums in the
// same order as amg_vcycle (bitwise equal to the single-GPU cycle).
class Comm;
// Slice batching of the level-0 AMG(A) / PCG kernels on LapView (GPU-only launch shape,
// bitwise-neutral): slices per block, 1 = unbatched.  Env BBOT_LAP_SB (A/B runs).
int lap_sb();
bool lap_expl();             // explicit load-phase variants (env BBOT_LAP_SB_EXPL)   // resident CTAs per SM requested (env BBOT_LAP_SB_MINB)
template <class V0>
void amg_vcycle_slab(Dev& d, AmgHierarchy& H, const V0& v0, const double* b, double* x, Comm& comm, int ra, int rb);

}  // namespace bbot
