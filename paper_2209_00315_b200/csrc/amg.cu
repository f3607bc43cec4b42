// amg.cu -- I3 device aggregation AMG: setup (strength graph, matching,
// Galerkin, coarsest inverse) and the V(1,1) cycle.  Definition: amg.cuh and
// DESIGN.md §2 (I3); the oracle (oracle/amg.py) implements the same algorithm
// independently.
#include "amg.cuh"
#include "comm.cuh"
#include <climits>
#include <type_traits>
#include <cooperative_groups.h>
#include <chrono>
#include <memory>
#include <mutex>
namespace cg = cooperative_groups;

namespace bbot {

constexpr double AMG_TAU = 1e-8;        // near-tie tolerance (relative)
constexpr double AMG_DECOUPLED = 1e-10; // rows with max strength <= this*|a_ii| do not propose
constexpr int MATCH_ROUNDS = 16;
constexpr int GAL_LOCAL = 48;           // coarse rows up to this many entries merge in local arrays
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

// tie-break priority among near-equal strengths: (lowbias32(j), j), lowest wins
__device__ __forceinline__ unsigned long long amg_prio(int j) {
  unsigned x = (unsigned)j;
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return ((unsigned long long)x << 32) | (unsigned)j;
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
  unsigned long long best = ~0ULL;
  for (long long p = sp[r]; p < sp[r + 1]; p++) {
    int c = sj[p];
    if (free_[c] && sw[p] >= thr) {
      unsigned long long pc = amg_prio(c);
      if (pc < best) best = pc;
    }
  }
  prop[r] = (int)(best & 0xffffffffULL);
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

// Aggregate leader of every row (I3): a pair's smaller row; a row left free
// joins the pair of its strongest matched neighbour t(i) = min{ j matched :
// s_ij >= (1 - tau) M'_i }, M'_i = max over matched j, if M'_i > 1e-10 |a_ii|;
// otherwise it is a singleton.  flag = 1 on leaders.
__global__ void k_attach(long long n, const long long* __restrict__ sp, const int* __restrict__ sj,
                         const double* __restrict__ sw, const double* __restrict__ adiag,
                         const int* __restrict__ partner, int* lead, int* flag) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int p = partner[r];
  long long L = r;
  if (p >= 0) {
    L = r < p ? r : p;
  } else {
    double M = -1.0;
    for (long long q = sp[r]; q < sp[r + 1]; q++)
      if (partner[sj[q]] >= 0) M = fmax(M, sw[q]);
    if (M > AMG_DECOUPLED * adiag[r]) {
      double thr = (1.0 - AMG_TAU) * M;
      unsigned long long bp = ~0ULL;
      for (long long q = sp[r]; q < sp[r + 1]; q++) {
        int c = sj[q];
        if (partner[c] >= 0 && sw[q] >= thr) {
          unsigned long long pc = amg_prio(c);
          if (pc < bp) bp = pc;
        }
      }
      int best = (int)(bp & 0xffffffffULL);
      int pc = partner[best];
      L = best < pc ? best : pc;
    }
  }
  lead[r] = (int)L;
  flag[r] = L == r ? 1 : 0;
}

__global__ void k_make_agg(long long n, const int* __restrict__ lead, const long long* __restrict__ cidx,
                           const int* __restrict__ sl, int* agg, int* slc) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  long long leader = lead[r];
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
// Coarse row I of A_c = P^T A P: the union of the member rows' columns mapped through agg,
// values summed in (member, entry) order, columns ascending.  Rows whose upper bound
// ub[I] = sum of the member row lengths fits GAL_LOCAL are merged in registers/local
// memory; wider rows (dense coarse graphs, e.g. AMG(S-hat) across time) are merged in a
// global scratch segment of ub[I] entries at goff[I] -- no width cap.
template <class V>
__global__ void k_gal_ub(V v, long long nc, const long long* __restrict__ mptr, const int* __restrict__ midx,
                         long long* ub) {
  long long I = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nc) return;
  long long u = 0;
  for (long long p = mptr[I]; p < mptr[I + 1]; p++) v.row(midx[p], [&](long long, double) { u++; });
  ub[I] = u;
}
__global__ void k_gal_big(long long nc, const long long* __restrict__ ub, long long* big) {
  long long I = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (I < nc) big[I] = ub[I] > GAL_LOCAL ? ub[I] : 0;
}

template <class V>
__device__ __forceinline__ int gal_merge(const V& v, long long I, const long long* __restrict__ mptr,
                                         const int* __restrict__ midx, const int* __restrict__ agg, int* cols,
                                         double* vals) {
  int len = 0;
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
      } else {
        for (int q = len; q > lo; q--) { cols[q] = cols[q - 1]; vals[q] = vals[q - 1]; }
        cols[lo] = J;
        vals[lo] = a;
        len++;
      }
    });
  }
  return len;
}

// BIG = false: rows with ub <= GAL_LOCAL (local arrays); BIG = true: the others (scratch)
template <class V, bool FILL, bool BIG>
__global__ void k_galerkin(V v, long long nc, const long long* __restrict__ mptr, const int* __restrict__ midx,
                           const int* __restrict__ agg, const long long* __restrict__ ub,
                           const long long* __restrict__ goff, int* gcols, double* gvals, int* cnt,
                           const long long* __restrict__ rp, int* ci, double* cv) {
  long long I = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nc) return;
  if ((ub[I] > GAL_LOCAL) != BIG) return;
  int lcols[BIG ? 1 : GAL_LOCAL];
  double lvals[BIG ? 1 : GAL_LOCAL];
  int* cols = BIG ? gcols + goff[I] : lcols;
  double* vals = BIG ? gvals + goff[I] : lvals;
  int len = gal_merge(v, I, mptr, midx, agg, cols, vals);
  if (!FILL) {
    cnt[I] = len;
  } else {
    long long o = rp[I];
    for (int q = 0; q < len; q++) { ci[o + q] = cols[q]; cv[o + q] = vals[q]; }
  }
}

// smoother diagonal: mode A the diagonal of the (Laplacian) row; mode T the l1 row
// sum sum_j |a_ij| (l1-Jacobi, I3: T's diagonal can be negative on real IPM iterates,
// C2 at mu = 0.25) -- summed in the row's entry order (the oracle sums CSR columns in
// ascending order; rounding-level differences only)
template <class V>
__global__ void k_dinv(V v, double* dinv, int l1) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= v.nrows) return;
  double dg = 0.0;
  if (l1) v.row(r, [&](long long c, double a) { dg += fabs(a); });
  else v.row(r, [&](long long c, double a) { if (c == r) dg += a; });
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
                       double* __restrict__ x, double* __restrict__ res, SliceSkip sk, RowRange rr) {
  long long r = rr.r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rr.r1 || sk.skip(r)) return;
  double acc = b[r];
  v.row(r, [&](long long c, double a) { acc -= a * (om * dinv[c] * b[c]); });
  x[r] = om * dinv[r] * b[r];
  res[r] = acc;
}

// mode-A coarse levels, BBOT_SELL_RES (the level-0 trick of k_up_dot_res on the SELL levels):
// the pre-sweep keeps only its residual (x = om D^-1 b is recomputed where needed) and the
// post-sweep starts from it, b - A (x + P xc) = res - A (P xc): one gather per entry
// (xc[agg[c]]) instead of two (x[c] too), no x in memory.  Rounding differs from k_up's order.
template <class V>
__global__ void k_down_nx(V v, const double* __restrict__ dinv, const double* __restrict__ b, double om,
                          double* __restrict__ res, SliceSkip sk, RowRange rr) {
  long long r = rr.r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rr.r1 || sk.skip(r)) return;
  double acc = b[r];
  v.row(r, [&](long long c, double a) { acc -= a * (om * dinv[c] * b[c]); });
  res[r] = acc;
}
template <class V>
__global__ void k_up_res(V v, const double* __restrict__ dinv, const double* __restrict__ b, double om,
                         const double* __restrict__ res, const int* __restrict__ agg, const double* __restrict__ xc,
                         double* __restrict__ xo, SliceSkip sk) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= v.nrows || sk.skip(r)) return;
  double acc = res[r];
  v.row(r, [&](long long c, double a) { acc -= a * xc[agg[c]]; });
  const double w = om * dinv[r];
  xo[r] = (w * b[r] + xc[agg[r]]) + w * acc;
}

__global__ void k_restrict(long long nc, const long long* __restrict__ mptr, const int* __restrict__ midx,
                           const double* __restrict__ r, double* bc, SliceSkip sk, RowRange rr) {
  long long I = rr.r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= rr.r1 || sk.skip(I)) return;
  double acc = 0.0;
  for (long long p = mptr[I]; p < mptr[I + 1]; p++) acc += r[midx[p]];   // P^T r, members ascending
  bc[I] = acc;
}



// pre-smoothing x = om D^-1 b first, then the residual sweep reads x (same
// expression order as k_down: bitwise identical), one gather per entry
__global__ void k_jacobi0(long long n, const double* __restrict__ dinv, const double* __restrict__ b, double om,
                          double* __restrict__ x, RowRange rr) {
  long long r = rr.r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rr.r1) x[r] = om * dinv[r] * b[r];
}
template <class V>
__global__ void k_resid(V v, const double* __restrict__ b, const double* __restrict__ x, double* __restrict__ res,
                        RowRange rr) {
  long long r = rr.r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rr.r1) return;
  double acc = b[r];
  v.row(r, [&](long long c, double a) { acc -= a * x[c]; });
  res[r] = acc;
}

// coarse levels, split pre-smoothing (BBOT_DOWN_SPLIT): x = om D^-1 b, then r = b - A x with one
// gather per entry instead of k_down's two (dinv[c], b[c]); the same values (bitwise)
__global__ void k_jacobi_sk(long long n, const double* __restrict__ dinv, const double* __restrict__ b, double om,
                            double* __restrict__ x, SliceSkip sk) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n && !sk.skip(r)) x[r] = om * dinv[r] * b[r];
}
template <class V>
__global__ void k_resid_sk(V v, const double* __restrict__ b, const double* __restrict__ x, double* __restrict__ res,
                           SliceSkip sk) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= v.nrows || sk.skip(r)) return;
  double acc = b[r];
  v.row(r, [&](long long c, double a) { acc -= a * x[c]; });
  res[r] = acc;
}

// xp = x + P xc (prolongated coarse correction), then the post-smoothing sweep on xp:
// two launches instead of k_up's chained gathers (neighbour -> agg -> xc) on each of
// T's ~27 entries per row; the same sums in the same order (bitwise identical)
__global__ void k_prolong(long long n, const double* __restrict__ x, const int* __restrict__ agg,
                          const double* __restrict__ xc, double* __restrict__ xp, SliceSkip sk, RowRange rr) {
  long long r = rr.r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rr.r1 && !sk.skip(r)) xp[r] = x[r] + xc[agg[r]];
}

// AMG(A) level 0 after k_prolong: post-smoothing on xp fused with the per-slice dot
// b.z (the PCG r.z step) -- k_up_dot's values exactly, one gather level per entry
template <class V>
__global__ void k_post_dot(V v, const double* __restrict__ dinv, const double* __restrict__ b, double om,
                           const double* __restrict__ xp, double* __restrict__ xo, long long L, RedArgs R,
                           PcgRzFin fin, const double* active) {
  int k = blockIdx.y;
  long long beg, end;
  red_chunk(L, R.parts, beg, end);
  if (active && active[k] == 0.0) end = beg;     // converged slice: nothing to do (partial 0)
  double dot = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    long long r = (long long)k * L + i;
    double acc = b[r];
    v.row(r, [&](long long c, double a) { acc -= a * xp[c]; });
    double z = xp[r] + om * dinv[r] * acc;
    xo[r] = z;
    dot += b[r] * z;
  }
  if (red_commit(dot, R)) fin(R.out);
}
template <class V>
__global__ void k_post(V v, const double* __restrict__ dinv, const double* __restrict__ b, double om,
                       const double* __restrict__ xp, double* __restrict__ xo, RowRange rr) {
  long long r = rr.r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rr.r1) return;
  double acc = b[r];
  v.row(r, [&](long long c, double a) { acc -= a * xp[c]; });
  xo[r] = xp[r] + om * dinv[r] * acc;
}

template <class V>
__global__ void k_up(V v, const double* __restrict__ dinv, const double* __restrict__ b, double om,
                     const double* __restrict__ x, const int* __restrict__ agg, const double* __restrict__ xc,
                     double* __restrict__ xo, SliceSkip sk) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= v.nrows || sk.skip(r)) return;
  double acc = b[r];
  v.row(r, [&](long long c, double a) { acc -= a * (x[c] + xc[agg[c]]); });
  xo[r] = (x[r] + xc[agg[r]]) + om * dinv[r] * acc;
}

// level-0 prolongation + post-smoothing fused with the per-slice dot b.xo
// (grid (parts, ns) over slice-major rows; PCG: r.z with its beta epilogue)
template <class V>
__global__ void __launch_bounds__(256, BBOT_LAP_MINB) k_up_dot(V v, const double* __restrict__ dinv, const double* __restrict__ b, double om,
                         const double* __restrict__ x, const int* __restrict__ agg, const double* __restrict__ xc,
                         double* __restrict__ xo, long long L, RedArgs R, PcgRzFin fin, const double* active) {
  int k = blockIdx.y;
  long long beg, end;
  red_chunk(L, R.parts, beg, end);
  if (active && active[k] == 0.0) end = beg;     // converged slice: nothing to do (partial 0)
  double dot = 0.0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) {
    long long r = (long long)k * L + i;
    double acc = b[r];
    v.row(r, [&](long long c, double a) { acc -= a * (x[c] + xc[agg[c]]); });
    double z = (x[r] + xc[agg[r]]) + om * dinv[r] * acc;
    xo[r] = z;
    dot += b[r] * z;
  }
  if (red_commit(dot, R)) fin(R.out);
}

// ---- slice-batched level-0 pre-smoothing (LapView).  The level-0 sweeps of AMG(A) are
// latency-bound (ncu: ~85 % of warp samples in long-scoreboard stalls at full occupancy,
// DRAM at ~51-55 % of peak).  k_down_sb's block (x, j) runs kites x*256.. of the NS = 2
// slices 2j, 2j+1: each thread loads kite i's neighbour slots once (nb is shared by all
// slices) and sweeps the rows kk*N + i of both slices -- the same rows and the same
// expression order as k_down (bitwise identical).  Measured on C4: k_down<LapView> 721 ->
// 624 ms per solve.  The same batching of k_up_dot / k_pcg_pq (2 or 4 slices, 4-8 CTAs per
// SM) and an explicit all-loads-first variant of all three measured slower on C4 (k_up_dot
// 929 -> 1107-3058 ms, k_pcg_pq 716 -> 770-1351 ms; profiles/r2z_ab_lap_sb_C4.log) and were
// removed.
int lap_sb() {
  const char* e = getenv("BBOT_LAP_SB");
  int v = e ? atoi(e) : 2;
  return v == 2 ? 2 : 1;
}

template <int NS, bool WX>
__global__ void __launch_bounds__(256, 6) k_down_sb(LapView v, const double* __restrict__ dinv,
                                                    const double* __restrict__ b, double om, double* __restrict__ x,
                                                    double* __restrict__ res, const double* __restrict__ active,
                                                    int ns) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int k0 = blockIdx.y * NS;
  if (i >= v.N) return;
  int c[4];
  v.nbrs(i, c);
#pragma unroll
  for (int s = 0; s < NS; s++) {
    const int kk = k0 + s;
    if (kk >= ns || (active && active[kk] == 0.0)) continue;
    const long long r = (long long)kk * v.N + i;
    double acc = b[r];
    v.row_nb(kk, i, c, [&](long long cc, double a) { acc -= a * (om * dinv[cc] * b[cc]); });
    if (WX) x[r] = om * dinv[r] * b[r];
    res[r] = acc;
  }
}

// ---- residual-based post sweeps (BBOT_LAP_RES, BBOT_SELL_RES; both on by default)
int lap_res() {
  const char* e = getenv("BBOT_LAP_RES");
  return e ? atoi(e) != 0 : BBOT_LAP_RES_DEFAULT;
}
int lap_rdinv() {
  const char* e = getenv("BBOT_LAP_RDINV");
  return e ? atoi(e) != 0 : BBOT_LAP_RDINV_DEFAULT;
}
int sell_res() {
  const char* e = getenv("BBOT_SELL_RES");
  return e ? atoi(e) != 0 : BBOT_SELL_RES_DEFAULT;
}

// Level 0 of AMG(A) (LapView): the post sweep from the pre-sweep's residual.  With x = om D^-1 b and
// res = b - A x (k_down), b - A (x + P xc) = res - A (P xc): the sweep gathers only the
// coarse correction xc[agg[c]] of the neighbours (4 gathers per kite less, no x in HBM at
// all: x_r is recomputed from b_r and dinv_r).  Mathematically the same z; rounding differs
// from k_up_dot's order at the 1e-16 level.
template <bool RDINV>
__global__ void __launch_bounds__(256, BBOT_LAP_MINB) k_up_dot_res(LapView v, const double* __restrict__ dinv,
                         const double* __restrict__ b, double om, const double* __restrict__ res,
                         const int* __restrict__ agg, const double* __restrict__ xc, double* __restrict__ xo,
                         RedArgs R, PcgRzFin fin, const double* active) {
  const int k = blockIdx.y;
  long long beg, end;
  red_chunk(v.N, R.parts, beg, end);
  if (active && active[k] == 0.0) end = beg;     // converged slice: nothing to do (partial 0)
  const long long base = (long long)k * v.N;
  const double* o = v.off + (size_t)k * 4 * v.N;
  const int* ag = agg + base;
  double dot = 0.0;
  for (int fc = (int)beg + threadIdx.x; fc < (int)end; fc += blockDim.x) {
    const long long r = base + fc;
    double acc = res[r], dg = 0.0;
    const double cr = xc[ag[fc]];
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const int c = v.nb[t * v.N + fc];
      if (c >= 0) {
        const double a = o[(size_t)t * v.N + fc];
        dg -= a;
        acc -= a * xc[ag[c]];
      }
    }
    acc -= dg * cr;
    // RDINV: dinv[r] = 1 / (sum of the slots, in slot order) is k_dinv's value exactly
    const double br = b[r], w = om * (RDINV ? 1.0 / dg : dinv[r]);
    const double z = (w * br + cr) + w * acc;
    xo[r] = z;
    dot += br * z;
  }
  if (red_commit(dot, R)) fin(R.out);
}

// level 0 of an AMG(A) hierarchy on the plain cell-ELL view, slice-major rows of N
template <class V0>
static bool lap_batched(const V0& v0, const AmgHierarchy& H) {
  if constexpr (std::is_same<V0, LapView>::value)
    return lap_sb() > 1 && H.mode != 1 && H.nslices > 0 && (long long)v0.N * H.nslices == H.lv[0].n;
  else
    return false;
}

// ------------------------------------------------------------ coarsest
// mode A: per slice, grounded at the slice's first row; Gauss-Jordan with partial
// pivoting on [B | I] in shared memory, B = block without row/col 0.
// grounded = 0 (mode As): the whole block is inverted (nonsingular shifted Laplacian).
__global__ void k_coarseA_setup(const long long* __restrict__ sptr, CsrView A, int cm, double* cinv, int grounded) {
  extern __shared__ double sm[];
  int k = blockIdx.x;
  long long s0 = sptr[k] + (grounded ? 1 : 0) - 1;   // first row of the block is s0 + 1
  int nl = (int)(sptr[k + 1] - sptr[k]) - (grounded ? 1 : 0);
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
                                const double* __restrict__ b, double* x, int grounded) {
  __shared__ double xs[256];
  int k = blockIdx.x;
  long long s0 = sptr[k];
  int nloc = (int)(sptr[k + 1] - s0);
  if (nloc <= 0) return;
  const double* inv = cinv + (size_t)k * cm * cm;
  if (!grounded) {                 // mode As: x = inv b on the slice block
    for (int j = threadIdx.x; j < nloc; j += blockDim.x) {
      double acc = 0.0;
      for (int l = 0; l < nloc; l++) acc += inv[j * cm + l] * b[s0 + l];
      x[s0 + j] = acc;
    }
    return;
  }
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

// ------------------------------------------------------------ per-slice coarse tail (mode A)
// AMG(A) never aggregates across time slices (I3), so below the first level with
// <= TAIL_ROWS rows per slice the rest of the cycle is independent per slice:
// one thread-block CLUSTER per slice (CL CTAs, CL = 148 / slices, <= 8) runs the
// restriction from level tail-1 and the whole coarse cycle -- damped-Jacobi
// V(1,1) steps, the K-cycle coarse corrections (two flexible-CG steps, per-slice
// dots reduced across the cluster through distributed shared memory in a fixed
// order; I3 / oracle amg.kstep) and the grounded coarsest solve -- with cluster
// barriers (barrier.cluster, release/acquire) instead of kernel launches.  The
// level table lives in device memory (TailArgs), read through a pointer.
// GPU-only tuning knobs (not part of the algorithm; env overrides for A/B runs)
static long long tune_env(const char* name, long long dflt) {
  const char* e = getenv(name);
  return e ? atoll(e) : dflt;
}
static const long long TAIL_ROWS = tune_env("BBOT_TAIL_ROWS", 0);       // A-tail for shallow hierarchies (0: none)
static const long long TAILT_ROWS = tune_env("BBOT_TAILT_ROWS", 16384); // first T-tail level: <= rows in total
static const int TAIL_CL = (int)tune_env("BBOT_TAIL_CL", 1);            // A-tail cluster size (0: 148/slices)
static const bool UP_SPLIT = tune_env("BBOT_UP_SPLIT", 0) != 0;        // A level 0: prolong + post_dot
static const bool SELL_SPLIT = tune_env("BBOT_SELL_SPLIT", 1) != 0;    // T coarse levels: prolong + post
static const bool DOWN_SPLIT = tune_env("BBOT_DOWN_SPLIT", 0) != 0;    // coarse levels: jacobi + resid
static const int TAILA_THREADS = (int)tune_env("BBOT_TAILA_BS", 512);    // k_tailA block size (<= TAIL_BS); 512: C4 krylov 6.71 -> 6.62 s vs 1024 (profiles/r4k_ab_tail_bs_C4.log)
constexpr int KC_ROWS = 4096;        // == oracle KC_ROWS
constexpr int KC_MIN_LEVELS = 7;     // == oracle KC_MIN_LEVELS: K-cycle only in deep hierarchies
constexpr int TAIL_MAXL = 24;
constexpr int TAIL_BS = 1024;
constexpr int TAIL_MAXCL = 8;

struct TailLevel {
  SellView A;
  const double* dinv;
  double *b, *x, *r, *xo;      // xo: level output (xt, or x at the coarsest)
  double *kc1, *kv, *krc;      // K-cycle work vectors
  const long long* mptr;       // members of the next level's rows (restriction)
  const int* midx;
  const int* agg;
  const long long* sptr;       // device slice pointers
  int kc;                      // 1: the coarse correction into this level is a K-cycle step
};
struct TailArgs {
  int first, last;             // levels first..last (last = coarsest)
  double om;
  int cm;
  int grounded;                // 1: mode A (grounded + mean removed), 0: mode As (plain)
  const double* cinv;
  // restriction into level `first` from level first-1
  const long long* mptr0;
  const int* midx0;
  const double* r0;
  TailLevel lv[TAIL_MAXL];
};

struct TailPos {               // this CTA: slice k, rank c of cs CTAs in the slice's cluster
  int k, c, cs;
  __device__ long long first_row(long long s0) const { return s0 + (long long)c * blockDim.x + threadIdx.x; }
  __device__ long long stride() const { return (long long)cs * blockDim.x; }
};

// a one-CTA cluster (the default) synchronises with a block barrier: bar.sync instead of the
// cluster-scope release/acquire barrier, ~a hundred of which separate the levels of one tail
__device__ __forceinline__ void tail_sync(const TailPos& P) {
  if (P.cs == 1) __syncthreads();
  else cg::this_cluster().sync();
}

// per-slice dot over rows [s0, s1): block sums, then every CTA adds the cluster's
// partials in rank order (identical result everywhere)
__device__ __forceinline__ double tail_dot(const double* u, const double* v, long long s0, long long s1,
                                           const TailPos& P) {
  __shared__ double part;
  double acc = 0.0;
  for (long long r = P.first_row(s0); r < s1; r += P.stride()) acc += u[r] * v[r];
  acc = block_sum(acc);
  if (threadIdx.x == 0) part = acc;
  if (P.cs == 1) {                 // the same sum as the loop below with one term
    __syncthreads();
    double tot = 0.0;
    tot += part;
    __syncthreads();
    return tot;
  }
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  double tot = 0.0;
  for (int q = 0; q < P.cs; q++) tot += *cl.map_shared_rank(&part, q);
  cl.sync();
  return tot;
}
__device__ __forceinline__ double tail_div(double a, double b) { return b != 0.0 ? a / b : 0.0; }

// NV per-slice dots at once (the K-cycle's dots fused into the passes that produce their
// operands): per value a warp butterfly, one shared-memory exchange, every thread summing the
// warps' partials in warp order (then the cluster's CTAs in rank order) -- one barrier pair
// for all NV values instead of one tail_dot (two block barriers + two more) per value
template <int NV>
__device__ __forceinline__ void tail_reduce(const double (&acc)[NV], double (&tot)[NV], const TailPos& P) {
  __shared__ double shr[NV][32];
  __shared__ double part[NV];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; k++) {
    double v = warp_sum(acc[k]);
    if (lane == 0) shr[k][w] = v;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; k++) {
    double t = 0.0;
    for (int q = 0; q < nw; q++) t += shr[k][q];
    tot[k] = t;
  }
  if (P.cs == 1) {
    __syncthreads();                   // shr reused by the next call
    return;
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < NV; k++) part[k] = tot[k];
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
#pragma unroll
  for (int k = 0; k < NV; k++) {
    double t = 0.0;
    for (int q = 0; q < P.cs; q++) t += cl.map_shared_rank(part, q)[k];
    tot[k] = t;
  }
  cl.sync();
}

__device__ void tail_cycle(const TailArgs* __restrict__ T, int q, const TailPos& P);

// K-cycle step at tail level q: input lv[q].b (= rc), output lv[q].xo (oracle amg.kstep).
// Each dot is accumulated in the pass that produces its operands (row-local products), and
// the dots of one pass are reduced together: rho1 = c1.v1 and a1 = c1.rc with v1 = A c1;
// g = c2.v1, a2 = c2.r2 and beta = c2.v2 with v2 = A c2 -- five barrier-separated dot phases
// of the latency-bound tail become two
__device__ void tail_kstep(const TailArgs* __restrict__ T, int q, const TailPos& P) {
  const TailLevel& L = T->lv[q];
  const long long s0 = L.sptr[P.k], s1 = L.sptr[P.k + 1];
  for (long long r = P.first_row(s0); r < s1; r += P.stride()) L.krc[r] = L.b[r];
  tail_sync(P);
  tail_cycle(T, q, P);                                   // c1 -> xo
  double a2v[2] = {0.0, 0.0}, t2[2];
  for (long long r = P.first_row(s0); r < s1; r += P.stride()) {
    const double c1 = L.xo[r];
    L.kc1[r] = c1;
    double av = 0.0;
    L.A.row(r, [&](long long col, double a) { av += a * L.xo[col]; });
    L.kv[r] = av;                                        // v1 = A c1
    a2v[0] += c1 * av;
    a2v[1] += c1 * L.krc[r];
  }
  tail_reduce<2>(a2v, t2, P);
  const double rho1 = t2[0], a1 = t2[1];
  const double f1 = tail_div(a1, rho1);
  for (long long r = P.first_row(s0); r < s1; r += P.stride()) L.b[r] = L.krc[r] - f1 * L.kv[r];   // r2
  tail_sync(P);
  tail_cycle(T, q, P);                                   // c2 -> xo
  double a3v[3] = {0.0, 0.0, 0.0}, t3[3];
  for (long long r = P.first_row(s0); r < s1; r += P.stride()) {
    const double c2 = L.xo[r];
    double av = 0.0;
    L.A.row(r, [&](long long col, double a) { av += a * L.xo[col]; });
    a3v[0] += c2 * L.kv[r];                              // g = c2.v1
    a3v[1] += c2 * L.b[r];                               // a2 = c2.r2
    a3v[2] += c2 * av;                                   // beta = c2.v2
    L.kv[r] = av;                                        // v2 = A c2
  }
  tail_reduce<3>(a3v, t3, P);
  const double g = t3[0], a2 = t3[1], beta = t3[2];
  const double rho2 = beta - g * tail_div(g, rho1);
  const double g2 = tail_div(a2, rho2);
  const double e1 = f1 - g * tail_div(g2, rho1);
  for (long long r = P.first_row(s0); r < s1; r += P.stride()) L.xo[r] = e1 * L.kc1[r] + g2 * L.xo[r];
  tail_sync(P);
}

// cycle of tail level q: input lv[q].b, output lv[q].xo
__device__ void tail_cycle(const TailArgs* __restrict__ T, int q, const TailPos& P) {
  const int tid = threadIdx.x, bs = blockDim.x;
  const int nl = T->last - T->first;
  const double om = T->om;
  if (q == nl) {   // coarsest: grounded at the slice's first row, then the slice mean removed
    __shared__ double xs[128];
    __shared__ double mean;
    const TailLevel& C = T->lv[nl];
    long long s0 = C.sptr[P.k];
    int nloc = (int)(C.sptr[P.k + 1] - s0);
    const double* inv = T->cinv + (size_t)P.k * T->cm * T->cm;
    if (!T->grounded) {                         // mode As: nonsingular block, plain solve
      if (P.c == 0)
        for (int j = tid; j < nloc; j += bs) {
          double acc = 0.0;
          for (int l = 0; l < nloc; l++) acc += inv[j * T->cm + l] * C.b[s0 + l];
          C.xo[s0 + j] = acc;
        }
      tail_sync(P);
      return;
    }
    for (int j = tid; j < nloc; j += bs) {      // every CTA of the cluster computes it (tiny)
      double acc = 0.0;
      if (j > 0)
        for (int l = 1; l < nloc; l++) acc += inv[(j - 1) * T->cm + (l - 1)] * C.b[s0 + l];
      xs[j] = acc;
    }
    __syncthreads();
    if (tid < 32) {
      double sum = 0.0;
      for (int j = tid; j < nloc; j += 32) sum += xs[j];
      sum = warp_sum(sum);
      if (tid == 0) mean = nloc > 0 ? sum / nloc : 0.0;
    }
    __syncthreads();
    if (P.c == 0)
      for (int j = tid; j < nloc; j += bs) C.xo[s0 + j] = xs[j] - mean;
    tail_sync(P);
    return;
  }
  const TailLevel& L = T->lv[q];
  const long long s0 = L.sptr[P.k], s1 = L.sptr[P.k + 1];
  for (long long r = P.first_row(s0); r < s1; r += P.stride()) {
    double acc = L.b[r];
    L.A.row(r, [&](long long c, double a) { acc -= a * (om * L.dinv[c] * L.b[c]); });
    L.x[r] = om * L.dinv[r] * L.b[r];
    L.r[r] = acc;
  }
  tail_sync(P);
  const TailLevel& C = T->lv[q + 1];
  const long long c0 = C.sptr[P.k], c1 = C.sptr[P.k + 1];
  for (long long I = P.first_row(c0); I < c1; I += P.stride()) {
    double acc = 0.0;
    for (long long p = L.mptr[I]; p < L.mptr[I + 1]; p++) acc += L.r[L.midx[p]];
    C.b[I] = acc;
  }
  tail_sync(P);
  if (C.kc) tail_kstep(T, q + 1, P);
  else tail_cycle(T, q + 1, P);
  const double* xc = C.xo;
  for (long long r = P.first_row(s0); r < s1; r += P.stride()) {
    double acc = L.b[r];
    L.A.row(r, [&](long long c, double a) { acc -= a * (L.x[c] + xc[L.agg[c]]); });
    L.xo[r] = (L.x[r] + xc[L.agg[r]]) + om * L.dinv[r] * acc;
  }
  tail_sync(P);
}

__global__ void __launch_bounds__(TAIL_BS) k_tailA(const TailArgs* __restrict__ T, const double* active) {
  cg::cluster_group cl = cg::this_cluster();
  TailPos P{(int)(blockIdx.x / cl.num_blocks()), (int)cl.block_rank(), (int)cl.num_blocks()};
  if (active && active[P.k] == 0.0) return;        // converged slice (the whole cluster leaves)
  {   // restriction from level first-1 (rows of slice k at level `first` are contiguous)
    const TailLevel& F = T->lv[0];
    long long s0 = F.sptr[P.k], s1 = F.sptr[P.k + 1];
    for (long long I = P.first_row(s0); I < s1; I += P.stride()) {
      double acc = 0.0;
      for (long long p = T->mptr0[I]; p < T->mptr0[I + 1]; p++) acc += T->r0[T->midx0[p]];
      F.b[I] = acc;
    }
  }
  tail_sync(P);
  if (T->lv[0].kc) tail_kstep(T, 0, P);
  else tail_cycle(T, 0, P);
}

// ------------------------------------------------------------ coarse tail of AMG(T)
// T couples neighbouring time slices, so its coarse levels are not independent per
// slice; instead ONE cluster of up to 16 CTAs (16 K threads, one row each at the
// first tail level) runs every level with <= TAILT_ROWS rows -- pre-smoothing +
// residual + restriction, the dense coarsest solve (warp per row), prolongation +
// post-smoothing -- separated by cluster barriers: a dozen latency-bound launches
// per V-cycle become one.  Arithmetic per row is that of k_down/k_restrict/
// k_dense_mv/k_up (same order).

struct TailTLevel {
  SellView A;
  long long n;
  const double* dinv;
  double *b, *x, *r, *xo;
  const long long* mptr;
  const int* midx;
  const int* agg;
};
struct TailTArgs {
  int first, last;
  double om;
  int nc;                       // coarsest size (dense inverse nc x nc)
  const double* cinv;
  const long long* mptr0;
  const int* midx0;
  const double* r0;
  TailTLevel lv[TAIL_MAXL];
};

// restrict_first = 0: level `first`'s right-hand side is already in place (time slabs:
// restricted slab by slab, then allgathered)
__global__ void __launch_bounds__(TAIL_BS) k_tailT(const TailTArgs* __restrict__ T, int restrict_first) {
  cg::cluster_group cl = cg::this_cluster();
  const long long g0 = (long long)cl.block_rank() * blockDim.x + threadIdx.x;
  const long long gs = (long long)cl.num_blocks() * blockDim.x;
  const double om = T->om;
  const int nl = T->last - T->first;
  if (restrict_first) {
    const TailTLevel& F = T->lv[0];
    for (long long I = g0; I < F.n; I += gs) {
      double acc = 0.0;
      for (long long p = T->mptr0[I]; p < T->mptr0[I + 1]; p++) acc += T->r0[T->midx0[p]];
      F.b[I] = acc;
    }
  }
  cl.sync();
  for (int q = 0; q < nl; q++) {
    const TailTLevel& L = T->lv[q];
    for (long long r = g0; r < L.n; r += gs) {
      double acc = L.b[r];
      L.A.row(r, [&](long long c, double a) { acc -= a * (om * L.dinv[c] * L.b[c]); });
      L.x[r] = om * L.dinv[r] * L.b[r];
      L.r[r] = acc;
    }
    cl.sync();
    const TailTLevel& C = T->lv[q + 1];
    for (long long I = g0; I < C.n; I += gs) {
      double acc = 0.0;
      for (long long p = L.mptr[I]; p < L.mptr[I + 1]; p++) acc += L.r[L.midx[p]];
      C.b[I] = acc;
    }
    cl.sync();
  }
  {   // coarsest: x = inv(T_c) b, one warp per row (as k_dense_mv)
    const TailTLevel& C = T->lv[nl];
    const int n = T->nc;
    const int lane = threadIdx.x & 31;
    const long long w0 = g0 >> 5, ws = gs >> 5;
    for (long long row = w0; row < n; row += ws) {
      double acc = 0.0;
#pragma unroll 8
      for (int j = lane; j < n; j += 32) acc += T->cinv[(size_t)row * n + j] * C.b[j];
      acc = warp_sum(acc);
      if (lane == 0) C.xo[row] = acc;
    }
  }
  cl.sync();
  for (int q = nl - 1; q >= 0; q--) {
    const TailTLevel& L = T->lv[q];
    const double* xc = T->lv[q + 1].xo;
    for (long long r = g0; r < L.n; r += gs) {
      double acc = L.b[r];
      L.A.row(r, [&](long long c, double a) { acc -= a * (L.x[c] + xc[L.agg[c]]); });
      L.xo[r] = (L.x[r] + xc[L.agg[r]]) + om * L.dinv[r] * acc;
    }
    cl.sync();
  }
}

// mode T: dense Gauss-Jordan in global memory, two launches per pivot
__global__ void k_csr_to_dense(CsrView A, int n, double* D, double* I) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (long long p = A.rp[r]; p < A.rp[r + 1]; p++) D[r * n + A.ci[p]] += A.v[p];
  I[r * n + r] = 1.0;
}

// Gauss-Jordan inverse with partial pivoting as ONE cooperative launch (one grid
// barrier per pivot instead of two launches).  Rows are not swapped: the pivot
// of column p is the unused row of largest |D[i][p]| (ties -> lower index); every
// other row is eliminated against it; each block, having updated its own rows,
// already proposes its candidate for column p+1, so a step needs one barrier.
// At the end pivot row piv[p] holds D[piv[p]][p] e_p^T | (that multiple of row p
// of the inverse): inv[p][:] = I[piv[p]][:] / D[piv[p]][p].
constexpr int GJ_BS = 256;
constexpr int GJ_MAXOWN = 1024;         // rows per block (n <= 8192, >= 8 blocks)
__global__ void __launch_bounds__(GJ_BS) k_gj_coop(int n, double* D, double* I, double* cand_v, int* cand_i,
                                                    int* used, int* piv, double* out) {
  cg::grid_group grid = cg::this_grid();
  const int nb = gridDim.x, tid = threadIdx.x;
  __shared__ double sv[GJ_BS];
  __shared__ int si[GJ_BS];
  __shared__ int s_piv;
  __shared__ double fs[GJ_MAXOWN];      // multipliers of the rows this block owns
  // rows owned by this block: i = blockIdx.x + q*nb
  auto propose = [&](int col) {
    double best = -1.0;
    int bi = INT_MAX;
    for (int i = blockIdx.x + tid * nb; i < n; i += nb * GJ_BS) {
      if (used[i]) continue;
      double v = fabs(D[(size_t)i * n + col]);
      if (v > best || (v == best && i < bi)) { best = v; bi = i; }
    }
    sv[tid] = best;
    si[tid] = bi;
    __syncthreads();
    for (int o = GJ_BS / 2; o > 0; o >>= 1) {
      if (tid < o) {
        double v2 = sv[tid + o];
        int i2 = si[tid + o];
        if (v2 > sv[tid] || (v2 == sv[tid] && i2 < si[tid])) { sv[tid] = v2; si[tid] = i2; }
      }
      __syncthreads();
    }
    if (tid == 0) {
      cand_v[(col & 1) * nb + blockIdx.x] = sv[0];
      cand_i[(col & 1) * nb + blockIdx.x] = si[0];
    }
    __syncthreads();
  };
  propose(0);
  grid.sync();
  for (int p = 0; p < n; p++) {
    if (tid < 32) {   // every block reduces the candidates identically (warp, fixed order)
      double best = -1.0;
      int bi = INT_MAX;
      for (int b = tid; b < nb; b += 32) {
        double v = cand_v[(p & 1) * nb + b];
        int i = cand_i[(p & 1) * nb + b];
        if (v > best || (v == best && i < bi)) { best = v; bi = i; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        double v2 = __shfl_down_sync(0xffffffffu, best, o);
        int i2 = __shfl_down_sync(0xffffffffu, bi, o);
        if (v2 > best || (v2 == best && i2 < bi)) { best = v2; bi = i2; }
      }
      if (tid == 0) s_piv = bi;
    }
    __syncthreads();
    const int pr = s_piv;
    const double pv = D[(size_t)pr * n + p];
    // eliminate column p from every other row owned by this block: all multipliers
    // first (one barrier), then the (row, column) updates as one flat loop
    const int nown = (n - 1 - (int)blockIdx.x) / nb + 1;     // rows i = blockIdx.x + q*nb
    for (int q = tid; q < nown; q += GJ_BS) {
      int i = blockIdx.x + q * nb;
      fs[q] = (i == pr) ? 0.0 : D[(size_t)i * n + p] / pv;
    }
    __syncthreads();
    {   // warp per owned row, lanes over columns (coalesced, independent iterations)
      const int lane = tid & 31, wp = tid >> 5, nw = GJ_BS / 32;
      const double* Dp = D + (size_t)pr * n;
      const double* Ip = I + (size_t)pr * n;
      for (int q = wp; q < nown; q += nw) {
        const double f = fs[q];
        if (f == 0.0) continue;                       // warp-uniform
        double* Di = D + (size_t)(blockIdx.x + q * nb) * n;
        double* Ii = I + (size_t)(blockIdx.x + q * nb) * n;
#pragma unroll 4
        for (int j = lane; j < n; j += 32) {
          double dv = j > p ? Di[j] - f * Dp[j] : (j == p ? 0.0 : Di[j]);
          Di[j] = dv;
          Ii[j] -= f * Ip[j];
        }
      }
    }
    if (tid == 0 && blockIdx.x == 0) piv[p] = pr;
    if (blockIdx.x == pr % nb && tid == 0) used[pr] = 1;
    __syncthreads();
    if (p + 1 < n) propose(p + 1);
    grid.sync();
  }
  for (long long t = (long long)blockIdx.x * GJ_BS + tid; t < (long long)n * n; t += (long long)nb * GJ_BS) {
    int r = (int)(t / n), j = (int)(t - (long long)r * n);
    int pr = piv[r];
    out[t] = I[(size_t)pr * n + j] / D[(size_t)pr * n + r];
  }
}

__global__ void k_dense_mv(int n, const double* __restrict__ A, const double* __restrict__ b, double* x) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= n) return;
  double acc = 0.0;
#pragma unroll 8   // loads issued ahead; the single accumulator keeps the summation order
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

// ------------------------------------------------------------ CSR -> SELL-32
__global__ void k_sell_width(long long n, const long long* __restrict__ rp, int* w, long long* w32) {
  long long ch = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long nch = (n + 31) >> 5;
  if (ch >= nch) return;
  int mx = 0;
  for (long long r = ch * 32; r < n && r < ch * 32 + 32; r++) mx = max(mx, (int)(rp[r + 1] - rp[r]));
  w[ch] = mx;
  w32[ch] = 32LL * mx;
}
__global__ void k_sell_fill(long long n, const long long* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, const long long* __restrict__ off,
                            const int* __restrict__ w, int* sci, double* sv) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  long long ch = r >> 5;
  long long base = off[ch] + (r & 31);
  int len = (int)(rp[r + 1] - rp[r]);
  for (int s = 0; s < w[ch]; s++) {
    if (s < len) {
      sci[base + (long long)s * 32] = ci[rp[r] + s];
      sv[base + (long long)s * 32] = v[rp[r] + s];
    } else {
      sci[base + (long long)s * 32] = (int)r;     // padding: own row, value 0
      sv[base + (long long)s * 32] = 0.0;
    }
  }
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
  launch(d, k_attach, dim3(nb), dim3(BS), 0, n, (const long long*)sg.sp.p, (const int*)sg.sj.p,
         (const double*)sg.sws.p, (const double*)sg.adiag.p, (const int*)w.partner.p, w.prop.p, w.flag.p);
  grow(w.cidx, n + 1, s);
  exclusive_scan_i32(d, w.flag.p, w.cidx.p, n, w.ws);
  nc = read_scalar(d, w.cidx.p + n);
  agg.alloc(n, s);
  slc.alloc(std::max(1LL, nc), s);
  launch(d, k_make_agg, dim3(nb), dim3(BS), 0, n, (const int*)w.prop.p, (const long long*)w.cidx.p, sl,
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
  grow(w.ub, nc, s);
  grow(w.goff, nc + 1, s);
  unsigned nb = nblocks(nc, 128);
  launch(d, k_gal_ub<V>, dim3(nb), dim3(128), 0, v, nc, mptr, midx, w.ub.p);
  launch(d, k_gal_big, dim3(nb), dim3(128), 0, nc, (const long long*)w.ub.p, w.goff.p);
  exclusive_scan(d, w.goff.p, w.goff.p, nc, w.ws);
  long long gtot = read_scalar(d, w.goff.p + nc);
  if (gtot > 0) {
    grow(w.gcols, gtot, s);
    grow(w.gvals, gtot, s);
  }
  auto pass = [&](auto fill, int* cnt, const long long* rp, int* ci, double* cv) {
    constexpr bool F = decltype(fill)::value;
    launch(d, k_galerkin<V, F, false>, dim3(nb), dim3(128), 0, v, nc, mptr, midx, agg, (const long long*)w.ub.p,
           (const long long*)w.goff.p, w.gcols.p, w.gvals.p, cnt, rp, ci, cv);
    if (gtot > 0)
      launch(d, k_galerkin<V, F, true>, dim3(nb), dim3(128), 0, v, nc, mptr, midx, agg, (const long long*)w.ub.p,
             (const long long*)w.goff.p, w.gcols.p, w.gvals.p, cnt, rp, ci, cv);
  };
  pass(std::false_type{}, w.cnt.p, (const long long*)nullptr, (int*)nullptr, (double*)nullptr);
  out.rp.alloc(nc + 1, s);
  exclusive_scan_i32(d, w.cnt.p, out.rp.p, nc, w.ws);
  long long nnz = read_scalar(d, out.rp.p + nc);
  out.ci.alloc(std::max(1LL, nnz), s);
  out.v.alloc(std::max(1LL, nnz), s);
  pass(std::true_type{}, (int*)nullptr, (const long long*)out.rp.p, out.ci.p, out.v.p);
  out.n = nc;
}

void build_sell(Dev& d, AmgLevel& L, AmgWork& w) {
  cudaStream_t s = d.stream;
  long long n = L.n, nch = (n + 31) >> 5;
  L.sl_w.alloc(std::max(1LL, nch), s);
  DBuf<long long> w32;
  w32.alloc(std::max(1LL, nch), s);
  L.sl_off.alloc(nch + 1, s);
  launch(d, k_sell_width, dim3(nblocks(nch, BS)), dim3(BS), 0, n, (const long long*)L.rp.p, L.sl_w.p, w32.p);
  exclusive_scan(d, w32.p, L.sl_off.p, nch, w.ws);
  long long tot = read_scalar(d, L.sl_off.p + nch);
  L.sl_ci.alloc(std::max(1LL, tot), s);
  L.sl_v.alloc(std::max(1LL, tot), s);
  launch(d, k_sell_fill, dim3(nblocks(n, BS)), dim3(BS), 0, n, (const long long*)L.rp.p, (const int*)L.ci.p,
         (const double*)L.v.p, (const long long*)L.sl_off.p, (const int*)L.sl_w.p, L.sl_ci.p, L.sl_v.p);
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

static void tail_args(AmgHierarchy& H, TailArgs& T);
static double* level_out(AmgHierarchy& H, int l);

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
  const bool timing = getenv("BBOT_TIMING") != nullptr;
  auto t_lv = std::chrono::steady_clock::now();
  for (int l = 0;; l++) {
    long long n = H.lv[l].n;
    {
      AmgLevel& L = H.lv[l];
      L.dinv.alloc(n, s);
      L.b.alloc(n, s);
      L.x.alloc(n, s);
      L.r.alloc(n, s);
      L.xt.alloc(n, s);
      if (l == 0) launch(d, k_dinv<V0>, dim3(nblocks(n, BS)), dim3(BS), 0, v0, L.dinv.p, (int)(mode == 1));
      else launch(d, k_dinv<CsrView>, dim3(nblocks(n, BS)), dim3(BS), 0, L.view(), L.dinv.p, (int)(mode == 1));
      L.sptr = slice_ptrs(d, L.slice_of.p, n, nslices, w);
    }
    std::vector<long long>& sp = H.lv[l].sptr;
    long long maxs = 0;
    for (int k = 0; k < nslices; k++) maxs = std::max(maxs, sp[k + 1] - sp[k]);
    bool small = (mode != 1) ? (maxs <= coarse_max) : (n <= coarse_max);
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
    if (timing)
      fprintf(stderr, "[bbot]   amg mode %d level %d (%lld rows): %.2f ms\n", mode, l, n,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_lv).count());
    t_lv = std::chrono::steady_clock::now();
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
  if (mode != 1) {
    const int grounded = mode == 0 ? 1 : 0;
    long long maxs = 0;
    for (int k = 0; k < nslices; k++) maxs = std::max(maxs, C.sptr[k + 1] - C.sptr[k]);
    BB_REQUIRE(maxs - grounded <= 120, BBOT_E_INTERNAL, "AMG(A): coarsest slice block too large");
    H.cm = (int)std::max(1LL, maxs - grounded);
    H.cinv.alloc((size_t)nslices * H.cm * H.cm, s);
    H.cinv.zero();
    H.csptr.alloc(nslices + 1, s);
    BB_CUDA(cudaMemcpyAsync(H.csptr.p, C.sptr.data(), (nslices + 1) * sizeof(long long), cudaMemcpyHostToDevice, s));
    size_t smem = (size_t)H.cm * 2 * H.cm * sizeof(double);
    BB_CUDA(cudaFuncSetAttribute(k_coarseA_setup, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch(d, k_coarseA_setup, dim3(nslices), dim3(256), smem, (const long long*)H.csptr.p, C.view(), H.cm, H.cinv.p,
           grounded);
  } else if (C.n > coarse_max) {   // stalled coarsening: Jacobi coarsest (oracle/amg.py)
    H.cjac = true;
    H.cm = (int)C.n;
  } else {
    long long n = C.n;
    H.cm = (int)n;
    DBuf<double> D;
    D.alloc((size_t)n * n, s);
    D.zero();
    H.cinv.alloc((size_t)n * n, s);
    DBuf<double> Iw, cv;
    DBuf<int> ci, used, piv;
    Iw.alloc((size_t)n * n, s);
    Iw.zero();
    launch(d, k_csr_to_dense, dim3(nblocks(n, BS)), dim3(BS), 0, C.view(), (int)n, D.p, Iw.p);
    int per_sm = 0;
    BB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gj_coop, GJ_BS, 0));
    // few blocks: each pivot step is latency-bound (candidate reduction + one grid
    // barrier), and the elimination of an n <= 1024 system needs little parallelism
    int nbk = std::max(1, std::min(per_sm * d.num_sms, (int)std::min<long long>((n + 7) / 8, 128)));
    nbk = std::max(nbk, (int)((n + GJ_MAXOWN - 1) / GJ_MAXOWN));
    cv.alloc(2 * (size_t)nbk, s);
    ci.alloc(2 * (size_t)nbk, s);
    used.alloc(n, s);
    used.zero();
    piv.alloc(n, s);
    int ni = (int)n;
    double* Dp = D.p;
    double* Ip = Iw.p;
    double* cvp = cv.p;
    int* cip = ci.p;
    int* up = used.p;
    int* pp = piv.p;
    double* op = H.cinv.p;
    void* args[] = {&ni, &Dp, &Ip, &cvp, &cip, &up, &pp, &op};
    BB_CUDA(cudaLaunchCooperativeKernel((const void*)k_gj_coop, dim3(nbk), dim3(GJ_BS), args, 0, d.stream));
    d.launches++;
    sync(d);
  }
  for (size_t l = 1; l < H.lv.size(); l++) build_sell(d, H.lv[l], w);
  // mode T: the coarse tail starts at the first coarse level with <= TAILT_ROWS rows
  if (mode == 1 && H.lv.size() >= 3 && !H.cjac) {
    int L = (int)H.lv.size();
    H.tail = 0;
    for (int l = 1; l < L - 1; l++)
      if (H.lv[l].n <= TAILT_ROWS && L - l <= TAIL_MAXL) { H.tail = l; break; }
    if (H.tail > 0) {
      std::unique_ptr<TailTArgs> stage(new TailTArgs());   // per call (no shared static state)
      TailTArgs& hostTT = *stage;
      AmgLevel& P = H.lv[H.tail - 1];
      hostTT.first = H.tail;
      hostTT.last = L - 1;
      hostTT.om = H.omega;
      hostTT.nc = (int)H.lv[L - 1].n;
      hostTT.cinv = H.cinv.p;
      hostTT.mptr0 = P.mptr.p;
      hostTT.midx0 = P.midx.p;
      hostTT.r0 = P.r.p;
      for (int l = H.tail; l < L; l++) {
        AmgLevel& A = H.lv[l];
        TailTLevel& t = hostTT.lv[l - H.tail];
        t.A = A.sell();
        t.n = A.n;
        t.dinv = A.dinv.p;
        t.b = A.b.p;
        t.x = A.x.p;
        t.r = A.r.p;
        t.xo = level_out(H, l);
        t.mptr = A.mptr.p;
        t.midx = A.midx.p;
        t.agg = A.agg.p;
      }
      H.tail_args.alloc(sizeof(TailTArgs), s);
      BB_CUDA(cudaMemcpyAsync(H.tail_args.p, &hostTT, sizeof(TailTArgs), cudaMemcpyHostToDevice, s));
      H.tail_cl = 16;
      static std::once_flag attr_once;
      std::call_once(attr_once, [] { cudaFuncSetAttribute(k_tailT, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); });
      sync(d);
    }
  }
  // mode A: the per-slice tail kernel (where the K-cycle lives) starts at the first K-cycle
  // level (hierarchies of >= KC_MIN_LEVELS levels, <= KC_ROWS rows per slice); shallower
  // hierarchies run every level as graph-replayed grid kernels, which measured faster on
  // C2 than any in-kernel fusion of the coarse levels (172.8 vs 185-299 ms per step),
  // unless BBOT_TAIL_ROWS asks for a tail.
  if (timing) {
    sync(d);
    fprintf(stderr, "[bbot]   amg mode %d coarsest (%lld rows) + SELL: %.2f ms\n", mode, H.lv.back().n,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_lv).count());
  }
  if (mode != 1) H.tail = 0;
  if (mode != 1 && H.lv.size() >= 2) {
    int L = (int)H.lv.size();
    long long lim = L >= KC_MIN_LEVELS ? (long long)KC_ROWS : TAIL_ROWS;
    for (int l = 1; l < L && lim > 0; l++) {
      long long mx = 0;
      for (int k = 0; k < nslices; k++) mx = std::max(mx, H.lv[l].sptr[k + 1] - H.lv[l].sptr[k]);
      if (mx <= lim && L - l <= TAIL_MAXL) {
        H.tail = l;
        break;
      }
    }
    std::unique_ptr<TailArgs> stage(new TailArgs());   // staging; the copy completes before the sync below
    TailArgs& hostT = *stage;
    for (int l = std::max(1, H.tail); H.tail > 0 && l < L; l++) {
      AmgLevel& A = H.lv[l];
      A.dsptr.alloc(nslices + 1, s);
      BB_CUDA(cudaMemcpyAsync(A.dsptr.p, A.sptr.data(), (nslices + 1) * sizeof(long long), cudaMemcpyHostToDevice,
                              s));
      A.kc1.alloc(A.n, s);
      A.kv.alloc(A.n, s);
      A.krc.alloc(A.n, s);
    }
    if (H.tail > 0) {
      tail_args(H, hostT);
      H.tail_args.alloc(sizeof(TailArgs), s);
      BB_CUDA(cudaMemcpyAsync(H.tail_args.p, &hostT, sizeof(TailArgs), cudaMemcpyHostToDevice, s));
    }
    sync(d);   // the host slice-pointer vectors / staging are sources of the async copies above
  }
  H.ready = true;
}

static void coarse_solve(Dev& d, AmgHierarchy& H, const double* b, double* x) {
  AmgLevel& C = H.lv.back();
  if (H.mode != 1)
    launch(d, k_coarseA_apply, dim3(H.nslices), dim3(128), 0, (const long long*)H.csptr.p, H.cm,
           (const double*)H.cinv.p, b, x, H.mode == 0 ? 1 : 0);
  else if (H.cjac)
    launch(d, k_jacobi0, dim3(nblocks(C.n, 256)), dim3(256), 0, C.n, (const double*)C.dinv.p, b, H.omega, x,
           RowRange{0, C.n});
  else
    launch(d, k_dense_mv, dim3(nblocks((long long)C.n * 32, 256)), dim3(256), 0, (int)C.n,
           (const double*)H.cinv.p, b, x);
}

// output buffer of level l in the V-cycle (no buffer swapping: capture-safe)
static double* level_out(AmgHierarchy& H, int l) {
  return l == (int)H.lv.size() - 1 ? H.lv[l].x.p : H.lv[l].xt.p;
}

static void tail_args(AmgHierarchy& H, TailArgs& T) {
  int L = (int)H.lv.size();
  T.first = H.tail;
  T.last = L - 1;
  T.om = H.omega;
  T.cm = H.cm;
  T.grounded = H.mode == 0 ? 1 : 0;
  T.cinv = H.cinv.p;
  AmgLevel& P = H.lv[H.tail - 1];
  T.mptr0 = P.mptr.p;
  T.midx0 = P.midx.p;
  T.r0 = P.r.p;
  for (int l = H.tail; l < L; l++) {
    AmgLevel& A = H.lv[l];
    TailLevel& t = T.lv[l - H.tail];
    t.A = A.sell();
    t.dinv = A.dinv.p;
    t.b = A.b.p;
    t.x = A.x.p;
    t.r = A.r.p;
    t.xo = level_out(H, l);
    t.kc1 = A.kc1.p;
    t.kv = A.kv.p;
    t.krc = A.krc.p;
    t.mptr = A.mptr.p;
    t.midx = A.midx.p;
    t.agg = A.agg.p;
    t.sptr = A.dsptr.p;
    long long mx = 0;
    for (int k = 0; k < H.nslices; k++) mx = std::max(mx, A.sptr[k + 1] - A.sptr[k]);
    t.kc = (L >= KC_MIN_LEVELS && l < L - 1 && mx <= KC_ROWS) ? 1 : 0;   // K-cycle levels (oracle amg.setup)
  }
}

template <class V0>
bool amg_vcycle(Dev& d, AmgHierarchy& H, const V0& v0, const double* b, double* x, const SliceDotFuse* fuse,
                const double* active) {
  int L = (int)H.lv.size();
  if (L == 1) { coarse_solve(d, H, b, x); return false; }
  double om = H.omega;
  if (H.mode == 1) active = nullptr;                // T couples slices: never skip
  const long long L0 = H.lv[0].n / std::max(1, H.nslices);
  auto skip_at = [&](int l) { return SliceSkip{active, l == 0 ? nullptr : (const int*)H.lv[l].slice_of.p, L0}; };
  // grid-wide levels: 0 .. stop-1; below: the per-slice tail (mode A) or more grid levels
  int stop = H.tail > 0 ? H.tail : L - 1;
  for (int l = 0; l < stop; l++) {
    AmgLevel& lv = H.lv[l];
    unsigned nb = nblocks(lv.n, BS);
    if (l == 0 && H.mode == 1) {   // T level 0: Jacobi step first, then a plain residual sweep
      launch(d, k_jacobi0, dim3(nb), dim3(BS), 0, lv.n, (const double*)lv.dinv.p, b, om, lv.x.p, RowRange{0, lv.n});
      launch(d, k_resid<V0>, dim3(nb), dim3(BS), 0, v0, b, (const double*)lv.x.p, lv.r.p, RowRange{0, lv.n});
    } else if (l == 0 && lap_batched<V0>(v0, H)) {
      if constexpr (std::is_same<V0, LapView>::value) {
        // the residual-based post sweep recomputes x = om D^-1 b: no x in HBM
        const bool wx = !(fuse && !UP_SPLIT && lap_res() && fuse->L == v0.N);
        if (wx)
          launch(d, k_down_sb<2, true>, dim3(nblocks(v0.N, BS), (H.nslices + 1) / 2), dim3(BS), 0, v0,
                 (const double*)lv.dinv.p, b, om, lv.x.p, lv.r.p, active, H.nslices);
        else
          launch(d, k_down_sb<2, false>, dim3(nblocks(v0.N, BS), (H.nslices + 1) / 2), dim3(BS), 0, v0,
                 (const double*)lv.dinv.p, b, om, lv.x.p, lv.r.p, active, H.nslices);
      }
    } else if (l == 0)
      launch(d, k_down<V0>, dim3(nb), dim3(BS), 0, v0, (const double*)lv.dinv.p, b, om, lv.x.p, lv.r.p, skip_at(0),
             RowRange{0, lv.n});
    else if (H.mode != 1 && sell_res())
      launch(d, k_down_nx<SellView>, dim3(nb), dim3(BS), 0, lv.sell(), (const double*)lv.dinv.p,
             (const double*)lv.b.p, om, lv.r.p, skip_at(l), RowRange{0, lv.n});
    else if (DOWN_SPLIT) {
      launch(d, k_jacobi_sk, dim3(nb), dim3(BS), 0, lv.n, (const double*)lv.dinv.p, (const double*)lv.b.p, om,
             lv.x.p, skip_at(l));
      launch(d, k_resid_sk<SellView>, dim3(nb), dim3(BS), 0, lv.sell(), (const double*)lv.b.p, (const double*)lv.x.p,
             lv.r.p, skip_at(l));
    } else
      launch(d, k_down<SellView>, dim3(nb), dim3(BS), 0, lv.sell(), (const double*)lv.dinv.p,
             (const double*)lv.b.p, om, lv.x.p, lv.r.p, skip_at(l), RowRange{0, lv.n});
    if (!(H.tail > 0 && l == stop - 1))
      launch(d, k_restrict, dim3(nblocks(lv.nc, BS)), dim3(BS), 0, lv.nc, (const long long*)lv.mptr.p,
             (const int*)lv.midx.p, (const double*)lv.r.p, H.lv[l + 1].b.p, skip_at(l + 1), RowRange{0, lv.nc});
  }
  if (H.mode != 1 && H.tail > 0) {
    int cl = TAIL_CL > 0 ? std::min(TAIL_CL, TAIL_MAXCL)
                         : std::max(1, std::min(TAIL_MAXCL, d.num_sms / std::max(1, H.nslices)));
    launch_cluster(d, k_tailA, dim3(H.nslices * cl), dim3(std::min(TAIL_BS, TAILA_THREADS)), 0, cl,
                   (const TailArgs*)H.tail_args.p, active);
  } else if (H.tail > 0) {
    launch_cluster(d, k_tailT, dim3(H.tail_cl), dim3(TAIL_BS), 0, H.tail_cl, (const TailTArgs*)H.tail_args.p, 1);
  } else {
    coarse_solve(d, H, H.lv[L - 1].b.p, H.lv[L - 1].x.p);
  }
  for (int l = stop - 1; l >= 0; l--) {
    AmgLevel& lv = H.lv[l];
    unsigned nb = nblocks(lv.n, BS);
    double* out = l == 0 ? x : level_out(H, l);
    const double* xc = level_out(H, l + 1);
    if (l == 0 && fuse && UP_SPLIT) {     // prolongate first, then the sweep fused with r.z
      launch(d, k_prolong, dim3(nb), dim3(BS), 0, lv.n, (const double*)lv.x.p, (const int*)lv.agg.p, xc, lv.xt.p,
             skip_at(0), RowRange{0, lv.n});
      launch(d, k_post_dot<V0>, dim3(fuse->parts, fuse->ns), dim3(BS), 0, v0, (const double*)lv.dinv.p, b, om,
             (const double*)lv.xt.p, out, fuse->L, fuse->R, fuse->fin, active);
    } else if (l == 0 && fuse && lap_batched<V0>(v0, H) && lap_res() && fuse->L == lv.n / H.nslices) {
      if constexpr (std::is_same<V0, LapView>::value) {
        if (lap_rdinv())
          launch(d, k_up_dot_res<true>, dim3(fuse->parts, fuse->ns), dim3(BS), 0, v0, (const double*)lv.dinv.p, b,
                 om, (const double*)lv.r.p, (const int*)lv.agg.p, xc, out, fuse->R, fuse->fin, active);
        else
          launch(d, k_up_dot_res<false>, dim3(fuse->parts, fuse->ns), dim3(BS), 0, v0, (const double*)lv.dinv.p, b,
                 om, (const double*)lv.r.p, (const int*)lv.agg.p, xc, out, fuse->R, fuse->fin, active);
      }
    } else if (l == 0 && fuse) {
      launch(d, k_up_dot<V0>, dim3(fuse->parts, fuse->ns), dim3(BS), 0, v0, (const double*)lv.dinv.p, b, om,
             (const double*)lv.x.p, (const int*)lv.agg.p, xc, out, fuse->L, fuse->R, fuse->fin, active);
    } else if (l == 0 && H.mode == 1) {   // T level 0: prolongate first, then a plain sweep
      launch(d, k_prolong, dim3(nb), dim3(BS), 0, lv.n, (const double*)lv.x.p, (const int*)lv.agg.p, xc, lv.xt.p,
             SliceSkip{nullptr, nullptr, 1}, RowRange{0, lv.n});
      launch(d, k_post<V0>, dim3(nb), dim3(BS), 0, v0, (const double*)lv.dinv.p, b, om, (const double*)lv.xt.p, out,
             RowRange{0, lv.n});
    } else if (l == 0) {
      launch(d, k_up<V0>, dim3(nb), dim3(BS), 0, v0, (const double*)lv.dinv.p, b, om, (const double*)lv.x.p,
             (const int*)lv.agg.p, xc, out, skip_at(0));
    } else if (H.mode != 1 && sell_res()) {
      launch(d, k_up_res<SellView>, dim3(nb), dim3(BS), 0, lv.sell(), (const double*)lv.dinv.p,
             (const double*)lv.b.p, om, (const double*)lv.r.p, (const int*)lv.agg.p, xc, out, skip_at(l));
    } else if (H.mode == 1 && SELL_SPLIT) {   // T coarse level: prolongate into r (free here), then sweep
      launch(d, k_prolong, dim3(nb), dim3(BS), 0, lv.n, (const double*)lv.x.p, (const int*)lv.agg.p, xc, lv.r.p,
             SliceSkip{nullptr, nullptr, 1}, RowRange{0, lv.n});
      launch(d, k_post<SellView>, dim3(nb), dim3(BS), 0, lv.sell(), (const double*)lv.dinv.p, (const double*)lv.b.p,
             om, (const double*)lv.r.p, out, RowRange{0, lv.n});
    } else {
      launch(d, k_up<SellView>, dim3(nb), dim3(BS), 0, lv.sell(), (const double*)lv.dinv.p,
             (const double*)lv.b.p, om, (const double*)lv.x.p, (const int*)lv.agg.p, xc, out, skip_at(l));
    }
  }
  return fuse != nullptr;
}

template <class V0>
void amg_vcycle_slab(Dev& d, AmgHierarchy& H, const V0& v0, const double* b, double* x, Comm& comm, int ra, int rb) {
  BB_REQUIRE(H.mode == 1, BBOT_E_INTERNAL, "amg_vcycle_slab: mode-T hierarchies only");
  const int L = (int)H.lv.size();
  const double om = H.omega;
  // level 0 is slice-structured (T couples slice k with k +- 1: one-slice halos); the coarse
  // levels are grouped by time block (A42: aggregates span the slices of a block), so their
  // halos are whole neighbouring blocks and the rank's rows are its blocks [ra/B, rb/B)
  const int K = v0.K;
  const long long tnbar = v0.nbar;
  const int TB = time_block_size(K);
  auto lay = [&](int l) {
    if (l == 0) return Layout::uniform(K, tnbar);
    Layout Ly;
    Ly.off = H.lv[l].sptr;
    Ly.unit = TB;
    return Ly;
  };
  auto rng = [&](int l) {
    if (l == 0) return RowRange{(long long)ra * tnbar, (long long)rb * tnbar};
    return RowRange{H.lv[l].sptr[ra / TB], H.lv[l].sptr[std::min(rb / TB, H.nslices)]};
  };
  auto grid = [&](const RowRange& r) { return dim3(nblocks(std::max(1LL, r.r1 - r.r0), BS)); };
  const SliceSkip none{nullptr, nullptr, 1};
  if (L == 1) {                        // level 0 is the coarsest: solve it redundantly
    AmgLevel& C = H.lv[0];
    RowRange r = rng(0);
    if (r.r1 > r.r0)
      BB_CUDA(cudaMemcpyAsync(C.b.p + r.r0, b + r.r0, (r.r1 - r.r0) * sizeof(double), cudaMemcpyDeviceToDevice,
                              d.stream));
    comm.allgather(d, lay(0), C.b.p);
    coarse_solve(d, H, C.b.p, x);
    return;
  }
  const int stop = H.tail > 0 ? H.tail : L - 1;
  for (int l = 0; l < stop; l++) {
    AmgLevel& lv = H.lv[l];
    RowRange r = rng(l);
    if (l == 0) {
      launch(d, k_jacobi0, grid(r), dim3(BS), 0, lv.n, (const double*)lv.dinv.p, b, om, lv.x.p, r);
      comm.halo(d, lay(0), lv.x.p);
      launch(d, k_resid<V0>, grid(r), dim3(BS), 0, v0, b, (const double*)lv.x.p, lv.r.p, r);
    } else {
      comm.halo(d, lay(l), lv.b.p);
      launch(d, k_down<SellView>, grid(r), dim3(BS), 0, lv.sell(), (const double*)lv.dinv.p, (const double*)lv.b.p,
             om, lv.x.p, lv.r.p, none, r);
    }
    RowRange rc = rng(l + 1);
    launch(d, k_restrict, grid(rc), dim3(BS), 0, lv.nc, (const long long*)lv.mptr.p, (const int*)lv.midx.p,
           (const double*)lv.r.p, H.lv[l + 1].b.p, none, rc);
  }
  if (H.tail > 0) {
    comm.allgather(d, lay(H.tail), H.lv[H.tail].b.p);
    launch_cluster(d, k_tailT, dim3(H.tail_cl), dim3(TAIL_BS), 0, H.tail_cl, (const TailTArgs*)H.tail_args.p, 0);
  } else {
    comm.allgather(d, lay(L - 1), H.lv[L - 1].b.p);
    coarse_solve(d, H, H.lv[L - 1].b.p, H.lv[L - 1].x.p);
  }
  for (int l = stop - 1; l >= 0; l--) {
    AmgLevel& lv = H.lv[l];
    RowRange r = rng(l);
    double* out = l == 0 ? x : level_out(H, l);
    const double* xc = level_out(H, l + 1);
    double* tmp = l == 0 ? lv.xt.p : lv.r.p;      // the prolongated iterate x + P xc
    launch(d, k_prolong, grid(r), dim3(BS), 0, lv.n, (const double*)lv.x.p, (const int*)lv.agg.p, xc, tmp, none, r);
    comm.halo(d, lay(l), tmp);
    if (l == 0)
      launch(d, k_post<V0>, grid(r), dim3(BS), 0, v0, (const double*)lv.dinv.p, b, om, (const double*)tmp, out, r);
    else
      launch(d, k_post<SellView>, grid(r), dim3(BS), 0, lv.sell(), (const double*)lv.dinv.p, (const double*)lv.b.p,
             om, (const double*)tmp, out, r);
  }
}

template void amg_setup<LapView>(Dev&, AmgHierarchy&, const LapView&, const int*, int, int, double, int,
                                     AmgWork&);
template void amg_setup<SliceEllView>(Dev&, AmgHierarchy&, const SliceEllView&, const int*, int, int, double, int,
                                      AmgWork&);
template bool amg_vcycle<LapView>(Dev&, AmgHierarchy&, const LapView&, const double*, double*,
                                  const SliceDotFuse*, const double*);
template void amg_setup<ScaledLapView>(Dev&, AmgHierarchy&, const ScaledLapView&, const int*, int, int, double, int,
                                       AmgWork&);
template bool amg_vcycle<ScaledLapView>(Dev&, AmgHierarchy&, const ScaledLapView&, const double*, double*,
                                        const SliceDotFuse*, const double*);
template bool amg_vcycle<SliceEllView>(Dev&, AmgHierarchy&, const SliceEllView&, const double*, double*,
                                       const SliceDotFuse*, const double*);
template void amg_vcycle_slab<SliceEllView>(Dev&, AmgHierarchy&, const SliceEllView&, const double*, double*, Comm&,
                                            int, int);

}  // namespace bbot
