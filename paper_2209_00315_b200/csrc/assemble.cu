// assemble.cu -- a1 + a3: geometry upload with the fixed index tables, and the
// per-Newton-step assembly kernels.
//
// a1:
//   rho~^k = R_E((rho^k + rho^{k-1})/2), omega^k = |e| rho~^k / |w|, g^k = grad phi^k
//   F_phi^k = -M Pi (rho^k - rho^{k-1})/dt + A_k phi^k                     (2.5)
//   F_rho^k = Pi^T M (phi^{k+1} - phi^k)/dt + 1/4 DR((g^k)^2 + (g^{k+1})^2) + Mbar s^k  (2.6, A5)
//   F_s^k   = rho^k s^k - mu                                                (2.7)
//   f, g, h = -F;  g~ = g - Mbar h / rho;  rhs = (f; P g~)                  ((3.2), (4.17))
// a3 (A8): omegabar^k = |e-bar| R-bar rho^k / |w-bar|,
//   T = diag(s/rho) Atilde - B M^-1 Btilde assembled row by row in the
//   slice-shared ELL layout (ctx.cuh).
#include "ops.cuh"
#include <map>
#include <set>
#include <algorithm>

namespace bbot {

constexpr int BS = 256;

// ---------------------------------------------------------------- tables
void upload_geometry(bbot_ctx* c, const Geometry& hg, int K) {
  DevGeom& g = c->g;
  cudaStream_t s = c->dev.stream;
  g.nbar = hg.nbar;
  g.N = hg.N;
  g.NE = hg.NE;
  g.NEbar = hg.NEbar;
  g.K = K;
  g.dt = 1.0 / (K + 1);   // P:158, A4
  g.area = hg.area;
  const int nbar = hg.nbar, N = hg.N;
  g.cbar.upload(hg.cbar, s);
  g.c.upload(hg.c, s);
  g.ebL.upload(hg.ebL, s);
  g.ebR.upload(hg.ebR, s);
  std::vector<double> ebc(hg.NEbar);
  for (int e = 0; e < hg.NEbar; e++) ebc[e] = hg.ebar_len[e] / hg.wbar_len[e];
  g.ebar_coef.upload(ebc, s);
  g.lam_bar.upload(hg.lam_bar, s);
  g.cadj_e.upload(hg.cadj_e, s);
  g.cadj_nb.upload(hg.cadj_nb, s);
  g.eL.upload(hg.eL, s);
  g.eR.upload(hg.eR, s);
  g.e_len.upload(hg.e_len, s);
  g.w_len.upload(hg.w_len, s);
  g.lam.upload(hg.lam, s);
  g.fadj_e.upload(hg.fadj_e, s);
  g.fadj_nb.upload(hg.fadj_nb, s);

  // E(i): fine edges with R_E[sigma,i] != 0, coefficient R_E[sigma,i]
  std::vector<std::vector<std::pair<int, double>>> Ei(nbar);
  for (int e = 0; e < hg.NE; e++) {
    int pL = hg.eL[e] / 3, pR = hg.eR[e] / 3;
    double l = hg.lam[e];
    if (pL == pR) {
      Ei[pL].push_back({e, l + (1.0 - l)});
    } else {
      Ei[pL].push_back({e, l});
      Ei[pR].push_back({e, 1.0 - l});
    }
  }
  std::vector<int> ce_edge((size_t)CE_MAX * nbar, -1);
  std::vector<double> ce_coef((size_t)CE_MAX * nbar, 0.0);
  for (int i = 0; i < nbar; i++) {
    BB_REQUIRE((int)Ei[i].size() <= CE_MAX, BBOT_E_GEOMETRY, "coarse cell with too many fine edges");
    for (size_t q = 0; q < Ei[i].size(); q++) {
      ce_edge[q * nbar + i] = Ei[i][q].first;
      ce_coef[q * nbar + i] = Ei[i][q].second;
    }
  }
  g.ce_edge.upload(ce_edge, s);
  g.ce_coef.upload(ce_coef, s);

  // type-b edges of each fine cell
  std::vector<std::vector<int>> tb(N);
  for (int e = 0; e < hg.NE; e++)
    if (hg.etype[e] == 1) {
      tb[hg.eL[e]].push_back(e);
      tb[hg.eR[e]].push_back(e);
    }
  // F(i), S(i) and positions
  std::vector<int> fi_cell((size_t)FI_MAX * nbar, -1), fi_child((size_t)FI_MAX * nbar, 0),
      fi_ppos((size_t)FI_MAX * nbar, 0), fi_edge((size_t)FI_MAX * FI_EMAX * nbar, -1),
      fi_tbe((size_t)FI_MAX * TB_MAX * nbar, -1), fi_tbpL((size_t)FI_MAX * TB_MAX * nbar, 0),
      fi_tbpR((size_t)FI_MAX * TB_MAX * nbar, 0), ca_pos(3 * (size_t)nbar, 0);
  std::vector<double> fi_alpha((size_t)FI_MAX * FI_EMAX * nbar, 0.0), fi_tbbeta((size_t)FI_MAX * TB_MAX * nbar, 0.0);
  std::vector<std::vector<int>> S(nbar), Fl(nbar);
  int W = 0;
  for (int i = 0; i < nbar; i++) {
    std::vector<int> F = {3 * i, 3 * i + 1, 3 * i + 2};
    std::set<int> foreign;
    for (auto& pe : Ei[i]) {
      int L = hg.eL[pe.first], R = hg.eR[pe.first];
      if (L / 3 != i) foreign.insert(L);
      if (R / 3 != i) foreign.insert(R);
    }
    for (int f : foreign) F.push_back(f);
    BB_REQUIRE((int)F.size() <= FI_MAX, BBOT_E_GEOMETRY, "B row too wide");
    Fl[i] = F;
    std::set<int> cols;
    for (int f : F) {
      cols.insert(f / 3);
      for (int e : tb[f]) {
        cols.insert(hg.eL[e] / 3);
        cols.insert(hg.eR[e] / 3);
      }
    }
    for (int t = 0; t < 3; t++)
      if (hg.cadj_nb[(size_t)t * nbar + i] >= 0) cols.insert(hg.cadj_nb[(size_t)t * nbar + i]);
    cols.erase(i);
    S[i].push_back(i);
    for (int cc : cols) S[i].push_back(cc);
    W = std::max(W, (int)S[i].size());
    auto pos = [&](int j) {
      auto it = std::find(S[i].begin(), S[i].end(), j);
      return (int)(it - S[i].begin());
    };
    for (size_t q = 0; q < F.size(); q++) {
      int f = F[q];
      fi_cell[q * nbar + i] = f;
      fi_child[q * nbar + i] = (f / 3 == i) ? 1 : 0;
      fi_ppos[q * nbar + i] = pos(f / 3);
      int ne = 0;
      for (auto& pe : Ei[i]) {
        int e = pe.first;
        if (hg.eL[e] != f && hg.eR[e] != f) continue;
        BB_REQUIRE(ne < FI_EMAX, BBOT_E_GEOMETRY, "too many B edges per fine cell");
        fi_edge[(q * FI_EMAX + ne) * nbar + i] = e;
        fi_alpha[(q * FI_EMAX + ne) * nbar + i] = 0.5 * pe.second * hg.e_len[e] * (hg.eL[e] == f ? 1.0 : -1.0);
        ne++;
      }
      BB_REQUIRE((int)tb[f].size() <= TB_MAX, BBOT_E_GEOMETRY, "fine cell with > 2 half coarse edges");
      for (size_t t = 0; t < tb[f].size(); t++) {
        int e = tb[f][t];
        double Rf = (hg.eL[e] == f) ? hg.lam[e] : 1.0 - hg.lam[e];
        fi_tbe[(q * TB_MAX + t) * nbar + i] = e;
        fi_tbbeta[(q * TB_MAX + t) * nbar + i] = 0.5 * Rf * hg.e_len[e];
        fi_tbpL[(q * TB_MAX + t) * nbar + i] = pos(hg.eL[e] / 3);
        fi_tbpR[(q * TB_MAX + t) * nbar + i] = pos(hg.eR[e] / 3);
      }
    }
    for (int t = 0; t < 3; t++) {
      int nb = hg.cadj_nb[(size_t)t * nbar + i];
      ca_pos[(size_t)t * nbar + i] = nb >= 0 ? pos(nb) : 0;
    }
  }
  BB_REQUIRE(W <= W_MAX, BBOT_E_GEOMETRY, "T stencil wider than W_MAX");
  // SIMPLE (NEXT f1): S-hat = C + B diag(A)^-1 B^T couples rows i, j whose B rows share a
  // fine cell; every such j lies in S(i) (a fine cell adjacent to a child of j across a
  // coarse boundary is reached through a type-b edge), so S-hat uses T's pattern.
  {
    std::vector<std::vector<std::pair<int, int>>> holders(N);   // f -> (j, index of f in F(j))
    for (int j = 0; j < nbar; j++)
      for (size_t q = 0; q < Fl[j].size(); q++) holders[Fl[j][q]].push_back({j, (int)q});
    std::vector<int> fv_j((size_t)FI_MAX * FV_MAX * nbar, -1), fv_q((size_t)FI_MAX * FV_MAX * nbar, 0),
        fv_pos((size_t)FI_MAX * FV_MAX * nbar, 0);
    for (int i = 0; i < nbar; i++)
      for (size_t q = 0; q < Fl[i].size(); q++) {
        const auto& hl = holders[Fl[i][q]];
        BB_REQUIRE((int)hl.size() <= FV_MAX, BBOT_E_GEOMETRY, "fine cell in too many B rows");
        for (size_t t = 0; t < hl.size(); t++) {
          auto it = std::find(S[i].begin(), S[i].end(), hl[t].first);
          BB_REQUIRE(it != S[i].end(), BBOT_E_INTERNAL, "S-hat column outside the T pattern");
          size_t at = (q * FV_MAX + t) * nbar + i;
          fv_j[at] = hl[t].first;
          fv_q[at] = hl[t].second;
          fv_pos[at] = (int)(it - S[i].begin());
        }
      }
    g.fv_j.upload(fv_j, s);
    g.fv_q.upload(fv_q, s);
    g.fv_pos.upload(fv_pos, s);
  }
  g.W = W;
  long long ssum = 0;
  for (int i = 0; i < nbar; i++) ssum += (long long)S[i].size();
  g.Tnnz = ssum * (3LL * K - 2);            // slices k0-1 and k0+1 missing at the two ends
  std::vector<int> tcol((size_t)W * nbar, -1);
  for (int i = 0; i < nbar; i++)
    for (size_t q = 0; q < S[i].size(); q++) tcol[q * nbar + i] = S[i][q];
  g.tcol.upload(tcol, s);
  g.fi_cell.upload(fi_cell, s);
  g.fi_child.upload(fi_child, s);
  g.fi_ppos.upload(fi_ppos, s);
  g.fi_edge.upload(fi_edge, s);
  g.fi_alpha.upload(fi_alpha, s);
  g.fi_tbe.upload(fi_tbe, s);
  g.fi_tbbeta.upload(fi_tbbeta, s);
  g.fi_tbpL.upload(fi_tbpL, s);
  g.fi_tbpR.upload(fi_tbpR, s);
  g.ca_pos.upload(ca_pos, s);
  // AMG level-0 slice maps (AMG(T): row -> time block)
  std::vector<int> slA((size_t)N * (K + 1)), slT((size_t)nbar * K);
  for (int k = 0; k <= K; k++) std::fill(slA.begin() + (size_t)k * N, slA.begin() + (size_t)(k + 1) * N, k);
  for (int k = 0; k < K; k++)   // AMG(T): time blocks (A42)
    std::fill(slT.begin() + (size_t)k * nbar, slT.begin() + (size_t)(k + 1) * nbar, time_block_of(K, k));
  g.slice_A.upload(slA, s);
  g.slice_T.upload(slT, s);
  std::vector<int> slS((size_t)nbar * K, 0);
  g.slice_S.upload(slS, s);
  BB_CUDA(cudaStreamSynchronize(s));
}

LapView view_A(bbot_ctx* c) { return LapView{c->g.N, c->n(), c->g.fadj_nb.p, c->as.Aoff.p}; }
ScaledLapView view_As(bbot_ctx* c) {
  return ScaledLapView{c->g.N, c->n(), c->g.fadj_nb.p, c->as.Aoff.p, c->as.sA.p, c->opts.alpha_hss};
}
SliceEllView view_T(bbot_ctx* c) {
  return SliceEllView{c->g.nbar, c->g.K, c->g.W, c->m(), c->g.tcol.p, c->as.Tv.p};
}

// ---------------------------------------------------------------- edge assembly
__global__ void k_edges(int K, int N, int NE, int nbar, const int* __restrict__ eL, const int* __restrict__ eR,
                        const double* __restrict__ lam, const double* __restrict__ e_len,
                        const double* __restrict__ w_len, const double* __restrict__ phi,
                        const double* __restrict__ rho_ext, double* __restrict__ omega, double* __restrict__ gphi,
                        int harm) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)(K + 1) * NE) return;
  int kk = (int)(t / NE);
  int e = (int)(t - (long long)kk * NE);
  int L = eL[e], R = eR[e];
  int pL = L / 3, pR = R / 3;
  const double* ra = rho_ext + (size_t)(kk + 1) * nbar;   // rho^k   (k = kk+1, 1-based)
  const double* rb = rho_ext + (size_t)kk * nbar;         // rho^{k-1}
  double l = lam[e];
  double rt = Recon::eval(harm, l, 0.5 * (ra[pL] + rb[pL]), 0.5 * (ra[pR] + rb[pR])).f;   // R_E or R_H
  double wl = w_len[e];
  omega[t] = e_len[e] * rt / wl;
  gphi[t] = (phi[(size_t)kk * N + L] - phi[(size_t)kk * N + R]) / wl;
}

// A_k in cell-ELL: Aoff[kk][t][f] = -omega^k of the t-th edge of kite f (0 pad)
__global__ void k_cell_lap(long long n, int N, int NE, const int* __restrict__ fe, const double* __restrict__ omega,
                           double* __restrict__ Aoff) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int kk = (int)(r / N);
  int f = (int)(r - (long long)kk * N);
  const double* om = omega + (size_t)kk * NE;
  double* o = Aoff + (size_t)kk * 4 * N + f;
#pragma unroll
  for (int t = 0; t < 4; t++) {
    int e = fe[t * N + f];
    o[(size_t)t * N] = e >= 0 ? -om[e] : 0.0;
  }
}

__global__ void k_coarse_edges(int K, int NEbar, int nbar, const int* __restrict__ ebL, const int* __restrict__ ebR,
                               const double* __restrict__ lam_bar, const double* __restrict__ ebar_coef,
                               const double* __restrict__ rho_ext, double* __restrict__ omegabar, int harm) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)K * NEbar) return;
  int k0 = (int)(t / NEbar);
  int e = (int)(t - (long long)k0 * NEbar);
  const double* r = rho_ext + (size_t)(k0 + 1) * nbar;
  double l = lam_bar[e];
  omegabar[t] = ebar_coef[e] * Recon::eval(harm, l, r[ebL[e]], r[ebR[e]]).f;   // R-bar (A35) or R-bar_H (A40)
}

// harmonic reconstruction (NEXT f4): sr = diag(C_H) / cbar = (C - diag W) / cbar, the diagonal
// the BB preconditioner uses in T (Remark 3.3); diag W at row (k0, i) =
// 1/8 sum over phi slices kk = k0, k0+1 of sum_{sigma in E(i), two parents} D (g^kk)^2 h_ii
__global__ void k_harm_sr(long long m, int nbar, int NE, const int* __restrict__ ce_edge,
                          const int* __restrict__ eL, const int* __restrict__ eR, const double* __restrict__ lam,
                          const double* __restrict__ e_len, const double* __restrict__ w_len,
                          const double* __restrict__ gphi, const double* __restrict__ rho_ext,
                          const double* __restrict__ cbar, const double* __restrict__ Cd, double* __restrict__ sr) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  int k0 = (int)(t / nbar);
  int i = (int)(t - (long long)k0 * nbar);
  double wd = 0.0;
  for (int side = 0; side < 2; side++) {
    int kk = k0 + side;
    const double* ra = rho_ext + (size_t)(kk + 1) * nbar;
    const double* rb = rho_ext + (size_t)kk * nbar;
    const double* gk = gphi + (size_t)kk * NE;
    for (int q = 0; q < CE_MAX; q++) {
      int e = ce_edge[(size_t)q * nbar + i];
      if (e < 0) break;
      int pL = eL[e] / 3, pR = eR[e] / 3;
      if (pL == pR) continue;             // one parent: R_H is linear there
      double haa, hab, hbb;
      Recon::hess(lam[e], 0.5 * (ra[pL] + rb[pL]), 0.5 * (ra[pR] + rb[pR]), haa, hab, hbb);
      wd += w_len[e] * e_len[e] * gk[e] * gk[e] * (pL == i ? haa : hbb);
    }
  }
  sr[t] = (Cd[t] - 0.125 * wd) / cbar[i];
}

__global__ void k_cdiag(long long m, int nbar, const double* __restrict__ cbar, const double* __restrict__ s,
                        const double* __restrict__ rho_ext, double* __restrict__ Cd, double* __restrict__ sr) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  int i = (int)(t % nbar);
  double q = s[t] / rho_ext[nbar + t];
  sr[t] = q;
  Cd[t] = cbar[i] * q;       // C = Mbar diag(s/rho)  (A7)
}

void assemble_edges(bbot_ctx* c) {
  DevGeom& g = c->g;
  Assembled& A = c->as;
  cudaStream_t s = c->dev.stream;
  long long ne = (long long)(g.K + 1) * g.NE;
  if (A.omega.n != (size_t)ne) {
    A.omega.alloc(ne, s);
    A.gphi.alloc(ne, s);
    A.Aoff.alloc((size_t)4 * c->n(), s);
    A.omegabar.alloc((size_t)g.K * g.NEbar, s);
    A.Cd.alloc(c->m(), s);
    A.sr.alloc(c->m(), s);
  }
  const int harm = c->opts.recon;
  launch(c->dev, k_edges, dim3(nblocks(ne, BS)), dim3(BS), 0, g.K, g.N, g.NE, g.nbar, (const int*)g.eL.p,
         (const int*)g.eR.p, (const double*)g.lam.p, (const double*)g.e_len.p, (const double*)g.w_len.p,
         (const double*)c->phi.p, (const double*)c->rho_ext.p, A.omega.p, A.gphi.p, harm);
  launch(c->dev, k_cell_lap, dim3(nblocks(c->n(), BS)), dim3(BS), 0, c->n(), g.N, g.NE, (const int*)g.fadj_e.p,
         (const double*)A.omega.p, A.Aoff.p);
  long long nce = (long long)g.K * g.NEbar;
  launch(c->dev, k_coarse_edges, dim3(nblocks(nce, BS)), dim3(BS), 0, g.K, g.NEbar, g.nbar, (const int*)g.ebL.p,
         (const int*)g.ebR.p, (const double*)g.lam_bar.p, (const double*)g.ebar_coef.p,
         (const double*)c->rho_ext.p, A.omegabar.p, harm);
  launch(c->dev, k_cdiag, dim3(nblocks(c->m(), BS)), dim3(BS), 0, c->m(), g.nbar, (const double*)g.cbar.p,
         (const double*)c->s.p, (const double*)c->rho_ext.p, A.Cd.p, A.sr.p);
  if (harm)
    launch(c->dev, k_harm_sr, dim3(nblocks(c->m(), BS)), dim3(BS), 0, c->m(), g.nbar, g.NE, (const int*)g.ce_edge.p,
           (const int*)g.eL.p, (const int*)g.eR.p, (const double*)g.lam.p, (const double*)g.e_len.p,
           (const double*)g.w_len.p, (const double*)A.gphi.p, (const double*)c->rho_ext.p,
           (const double*)g.cbar.p, (const double*)A.Cd.p, A.sr.p);
}

// ---------------------------------------------------------------- residuals
struct FPhiF {
  int N, NE, nbar;
  double dt;
  const double *cf, *phi, *rho_ext, *omega;
  const int *fe, *fnb;
  double* fout;
  __device__ double operator()(int kk, long long f) const {
    int pf = (int)(f / 3);
    double ra = rho_ext[(size_t)(kk + 1) * nbar + pf], rb = rho_ext[(size_t)kk * nbar + pf];
    const double* ph = phi + (size_t)kk * N;
    const double* om = omega + (size_t)kk * NE;
    double pfv = ph[f];
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      int e = fe[t * N + f];
      if (e >= 0) acc += om[e] * (pfv - ph[fnb[t * N + f]]);
    }
    double F = -cf[f] * (ra - rb) / dt + acc;
    fout[(size_t)kk * N + f] = -F;
    return F * F;
  }
};

struct FRhoF {
  int N, NE, nbar;
  double dt, mu;
  const double *cf, *cbar, *phi, *gphi, *s, *rho_ext, *ce_coef, *e_len, *w_len;
  const int* ce_edge;
  double *g, *h, *gt;
  int harm;
  const int *eL, *eR;
  const double* lam;
  __device__ double operator()(int k0, long long i) const {
    const double* p0 = phi + (size_t)k0 * N;
    const double* p1 = phi + (size_t)(k0 + 1) * N;
    double tt = 0.0;
    for (int q = 0; q < 3; q++) {
      long long f = 3 * i + q;
      tt += cf[f] * ((p1[f] - p0[f]) / dt);
    }
    const double* g0 = gphi + (size_t)k0 * NE;
    const double* g1 = gphi + (size_t)(k0 + 1) * NE;
    double dr = 0.0;
    if (!harm) {
      for (int q = 0; q < CE_MAX; q++) {
        int e = ce_edge[(size_t)q * nbar + i];
        if (e < 0) break;
        dr += ce_coef[(size_t)q * nbar + i] * w_len[e] * e_len[e] * (g0[e] * g0[e] + g1[e] * g1[e]);
      }
    } else {    // 1/4 [J(rho-bar^k)^T D (g^k)^2 + J(rho-bar^{k+1})^T D (g^{k+1})^2]  (f4)
      const double* r0 = rho_ext + (size_t)k0 * nbar;
      const double* r1 = rho_ext + (size_t)(k0 + 1) * nbar;
      const double* r2 = rho_ext + (size_t)(k0 + 2) * nbar;
      for (int q = 0; q < CE_MAX; q++) {
        int e = ce_edge[(size_t)q * nbar + i];
        if (e < 0) break;
        int pL = eL[e] / 3, pR = eR[e] / 3;
        Recon a = Recon::eval(1, lam[e], 0.5 * (r1[pL] + r0[pL]), 0.5 * (r1[pR] + r0[pR]));
        Recon b = Recon::eval(1, lam[e], 0.5 * (r2[pL] + r1[pL]), 0.5 * (r2[pR] + r1[pR]));
        double ja = (pL == i ? a.ja : 0.0) + (pR == i ? a.jb : 0.0);
        double jb = (pL == i ? b.ja : 0.0) + (pR == i ? b.jb : 0.0);
        dr += w_len[e] * e_len[e] * (ja * g0[e] * g0[e] + jb * g1[e] * g1[e]);
      }
    }
    size_t t = (size_t)k0 * nbar + i;
    double si = s[t], ri = rho_ext[nbar + t];
    double Frho = tt + 0.25 * dr + cbar[i] * si;
    double Fs = ri * si - mu;
    double gg = -Frho, hh = -Fs;
    g[t] = gg;
    h[t] = hh;
    gt[t] = gg - cbar[i] * hh / ri;
    return Frho * Frho + Fs * Fs;
  }
};

struct GtSum {
  int nbar;
  const double* gt;
  __device__ double operator()(int k0, long long i) const { return gt[(size_t)k0 * nbar + i]; }
};

__global__ void k_rhs2(long long m, int nbar, double area, const double* __restrict__ cbar,
                       const double* __restrict__ gt, const double* __restrict__ S, double* __restrict__ out) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  int k0 = (int)(t / nbar);
  int i = (int)(t - (long long)k0 * nbar);
  out[t] = gt[t] - cbar[i] * S[k0] / area;     // P g~
}

void compute_residual(bbot_ctx* c, bool write_rhs) {
  DevGeom& g = c->g;
  Assembled& A = c->as;
  cudaStream_t s = c->dev.stream;
  long long n = c->n(), m = c->m();
  if (A.f.n != (size_t)n) {
    A.f.alloc(n, s);
    A.g.alloc(m, s);
    A.h.alloc(m, s);
    A.gt.alloc(m, s);
    A.rhs.alloc(n + m, s);
  }
  assemble_edges(c);
  int K = g.K;
  double* sc = c->scal.p;   // [0, K+1): F_phi^2 per slice; [K+1, 2K+1): F_rho^2+F_s^2; [2K+1, 3K+1): sum g~
  c->red.slice_sum(FPhiF{g.N, g.NE, g.nbar, g.dt, g.c.p, c->phi.p, c->rho_ext.p, A.omega.p, g.fadj_e.p, g.fadj_nb.p,
                         A.f.p},
                   g.N, K + 1, sc, false);
  c->red.slice_sum(FRhoF{g.N, g.NE, g.nbar, g.dt, c->mu, g.c.p, g.cbar.p, c->phi.p, A.gphi.p, c->s.p, c->rho_ext.p,
                         g.ce_coef.p, g.e_len.p, g.w_len.p, g.ce_edge.p, A.g.p, A.h.p, A.gt.p, c->opts.recon, g.eL.p,
                         g.eR.p, g.lam.p},
                   g.nbar, K, sc + K + 1, false);
  std::vector<double> hs(2 * K + 1);
  if (write_rhs) {
    c->red.slice_sum(GtSum{g.nbar, A.gt.p}, g.nbar, K, sc + 2 * K + 1, false);
    BB_CUDA(cudaMemcpyAsync(A.rhs.p, A.f.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (c->opts.precond != 0)    // SIMPLE / HSS: the unprojected saddle-point system
      BB_CUDA(cudaMemcpyAsync(A.rhs.p + n, A.gt.p, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
    else
      launch(c->dev, k_rhs2, dim3(nblocks(m, BS)), dim3(BS), 0, m, g.nbar, g.area, (const double*)g.cbar.p,
             (const double*)A.gt.p, (const double*)(sc + 2 * K + 1), A.rhs.p + n);
  }
  BB_CUDA(cudaMemcpyAsync(hs.data(), sc, (2 * K + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
  sync(c->dev);
  double tot = 0.0;
  for (double v : hs) tot += v;
  A.res_norm = std::sqrt(tot);
  A.scale = A.res_norm;      // ||(f;g;h)|| = ||F||
  if (write_rhs) BB_CUDA(cudaMemcpyAsync(A.dscale.p, &A.scale, sizeof(double), cudaMemcpyHostToDevice, s));
}

// ---------------------------------------------------------------- T assembly
constexpr int T_KCH = 4;   // slices per thread (table reuse through L1)

__global__ void __launch_bounds__(128) k_assemble_T(
    int nbar, int K, int NE, int NEbar, int W, double dt, const double* __restrict__ cf,
    const double* __restrict__ gphi, const double* __restrict__ omegabar, const double* __restrict__ sr,
    const int* __restrict__ cadj_e, const int* __restrict__ ca_pos, const int* __restrict__ fi_cell,
    const int* __restrict__ fi_child, const int* __restrict__ fi_ppos, const int* __restrict__ fi_edge,
    const double* __restrict__ fi_alpha, const int* __restrict__ fi_tbe, const double* __restrict__ fi_tbbeta,
    const int* __restrict__ fi_tbpL, const int* __restrict__ fi_tbpR, double* __restrict__ Tv, int harm,
    const int* __restrict__ eL, const int* __restrict__ eR, const double* __restrict__ lam,
    const double* __restrict__ rho_ext) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nbar) return;
  int kb = blockIdx.y * T_KCH, ke = min(K, kb + T_KCH);
  for (int k0 = kb; k0 < ke; k0++) {
    double acc[3 * W_MAX];
    for (int t = 0; t < 3 * W; t++) acc[t] = 0.0;
    for (int side = 0; side < 2; side++) {
      int kp = k0 + side;                 // 0-based phi slice of the B column / B~ row
      bool lo_ok = kp - 1 >= 0, hi_ok = kp <= K - 1;
      const double* gk = gphi + (size_t)kp * NE;
      // harmonic R_H (f4): the tables hold the arithmetic weights (R_E[sigma,i], R_f[sigma,f]);
      // scale them to the Jacobian J_H(rho-bar^kp) / J_f at this slice
      auto rec = [&](int ed) {
        const double* ra = rho_ext + (size_t)(kp + 1) * nbar;
        const double* rb = rho_ext + (size_t)kp * nbar;
        int pL = eL[ed] / 3, pR = eR[ed] / 3;
        return Recon::eval(1, lam[ed], 0.5 * (ra[pL] + rb[pL]), 0.5 * (ra[pR] + rb[pR]));
      };
      for (int q = 0; q < FI_MAX; q++) {
        int f = fi_cell[q * nbar + i];
        if (f < 0) break;
        double cfv = cf[f];
        // B[(k0,i),(kp,f)]
        double b = fi_child[q * nbar + i] ? (side ? cfv : -cfv) / dt : 0.0;
        for (int e = 0; e < FI_EMAX; e++) {
          int ed = fi_edge[(q * FI_EMAX + e) * nbar + i];
          if (ed < 0) break;
          double al = fi_alpha[(q * FI_EMAX + e) * nbar + i];
          if (harm) {
            Recon r = rec(ed);
            double l = lam[ed];
            int pL = eL[ed] / 3, pR = eR[ed] / 3;
            al *= ((pL == i ? r.ja : 0.0) + (pR == i ? r.jb : 0.0)) / ((pL == i ? l : 0.0) + (pR == i ? 1.0 - l : 0.0));
          }
          b += al * gk[ed];
        }
        b = b / cfv;                      // M^-1
        // row (kp, f) of B~: time part c_f (z^{hi} - z^{lo})/dt at par(f)
        double tc = cfv / dt;
        int pp = fi_ppos[q * nbar + i];
        if (hi_ok) acc[(side + 1) * W + pp] -= b * tc;
        if (lo_ok) acc[side * W + pp] += b * tc;
        // space part 1/2 R_f |e| g (zbar_parL - zbar_parR) on half coarse edges
        for (int t = 0; t < TB_MAX; t++) {
          int ed = fi_tbe[(q * TB_MAX + t) * nbar + i];
          if (ed < 0) break;
          double be = fi_tbbeta[(q * TB_MAX + t) * nbar + i];
          if (harm) {
            Recon r = rec(ed);
            be *= eL[ed] == f ? r.ja / lam[ed] : r.jb / (1.0 - lam[ed]);
          }
          double v = b * (be * gk[ed]);
          int pL = fi_tbpL[(q * TB_MAX + t) * nbar + i], pR = fi_tbpR[(q * TB_MAX + t) * nbar + i];
          if (hi_ok) { acc[(side + 1) * W + pL] -= v; acc[(side + 1) * W + pR] += v; }
          if (lo_ok) { acc[side * W + pL] -= v; acc[side * W + pR] += v; }
        }
      }
    }
    // diag(s/rho) Atilde_k
    double q = sr[(size_t)k0 * nbar + i];
    const double* ob = omegabar + (size_t)k0 * NEbar;
    for (int t = 0; t < 3; t++) {
      int e = cadj_e[t * nbar + i];
      if (e < 0) continue;
      double o = q * ob[e];
      acc[W] += o;
      acc[W + ca_pos[t * nbar + i]] -= o;
    }
    for (int d = 0; d < 3; d++)
      for (int sl = 0; sl < W; sl++) Tv[((size_t)(k0 * 3 + d) * W + sl) * nbar + i] = acc[d * W + sl];
  }
}

// ---------------------------------------------------------------- S-hat assembly (NEXT f1)
// SIMPLE (A31): S-hat = -S~ = C + B diag(A)^-1 B^T, block tridiagonal,
// in T's slice-shared ELL layout.  Row (k0, i):
//   sum over phi slices kp in {k0, k0+1}, fine cells f in F(i), rows (k1, j) of B holding f:
//   B[(k0,i),(kp,f)] / A_kp[f,f] * B[(k1,j),(kp,f)],   k1 in {kp (side 0), kp-1 (side 1)}
// plus C[(k0,i)] on the diagonal.  B entries as in k_assemble_T / BRow (D5, A5).
__global__ void k_dainv(long long n, int N, const double* __restrict__ Aoff, double* __restrict__ dAinv) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int kk = (int)(r / N);
  int f = (int)(r - (long long)kk * N);
  const double* o = Aoff + (size_t)kk * 4 * N + f;
  double d = 0.0;
#pragma unroll
  for (int t = 0; t < 4; t++) d -= o[(size_t)t * N];     // pad slots hold 0
  dAinv[r] = 1.0 / d;
}

__global__ void __launch_bounds__(128) k_assemble_S(
    int nbar, int K, int N, int NE, int W, double dt, const double* __restrict__ cf,
    const double* __restrict__ gphi, const double* __restrict__ dAinv, const double* __restrict__ Cd,
    const int* __restrict__ fi_cell, const int* __restrict__ fi_child, const int* __restrict__ fi_edge,
    const double* __restrict__ fi_alpha, const int* __restrict__ fv_j, const int* __restrict__ fv_q,
    const int* __restrict__ fv_pos, double* __restrict__ Sv) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nbar) return;
  int kb = blockIdx.y * T_KCH, ke = min(K, kb + T_KCH);
  for (int k0 = kb; k0 < ke; k0++) {
    double acc[3 * W_MAX];
    for (int t = 0; t < 3 * W; t++) acc[t] = 0.0;
    for (int side = 0; side < 2; side++) {
      int kp = k0 + side;
      const double* gk = gphi + (size_t)kp * NE;
      const double* dinv = dAinv + (size_t)kp * N;
      for (int q = 0; q < FI_MAX; q++) {
        int f = fi_cell[q * nbar + i];
        if (f < 0) break;
        double tp = fi_child[q * nbar + i] ? cf[f] / dt : 0.0;
        double sp = 0.0;
        for (int e = 0; e < FI_EMAX; e++) {
          int ed = fi_edge[(q * FI_EMAX + e) * nbar + i];
          if (ed < 0) break;
          sp += fi_alpha[(q * FI_EMAX + e) * nbar + i] * gk[ed];
        }
        double w = ((side ? tp : -tp) + sp) * dinv[f];
        for (int t = 0; t < FV_MAX; t++) {
          size_t at = (size_t)(q * FV_MAX + t) * nbar + i;
          int j = fv_j[at];
          if (j < 0) break;
          int qj = fv_q[at], pj = fv_pos[at];
          double tpj = fi_child[qj * nbar + j] ? cf[f] / dt : 0.0;
          double spj = 0.0;
          for (int e = 0; e < FI_EMAX; e++) {
            int ed = fi_edge[(qj * FI_EMAX + e) * nbar + j];
            if (ed < 0) break;
            spj += fi_alpha[(qj * FI_EMAX + e) * nbar + j] * gk[ed];
          }
          if (kp <= K - 1) acc[(kp - k0 + 1) * W + pj] += w * (spj - tpj);   // row (kp, j), side 0
          if (kp >= 1) acc[(kp - k0) * W + pj] += w * (spj + tpj);           // row (kp-1, j), side 1
        }
      }
    }
    acc[W] += Cd[(size_t)k0 * nbar + i];
    for (int d = 0; d < 3; d++)
      for (int sl = 0; sl < W; sl++) Sv[((size_t)(k0 * 3 + d) * W + sl) * nbar + i] = acc[d * W + sl];
  }
}

// HSS (NEXT f2): sA = diag(A)^-1/2, sC = C^-1/2, c2 = alpha^2 C
__global__ void k_hss_scal(long long n, long long m, double al, const double* __restrict__ dAinv,
                           const double* __restrict__ Cd, double* __restrict__ sA, double* __restrict__ sC,
                           double* __restrict__ c2) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) sA[t] = sqrt(dAinv[t]);
  if (t < m) {
    sC[t] = 1.0 / sqrt(Cd[t]);
    c2[t] = al * al * Cd[t];
  }
}
// T-slot values *= inv_alpha sC_row sC_col  (rows k0*nbar+i, column (k0+d-1)*nbar + tcol[s][i])
__global__ void k_hss_scale_S(int nbar, int K, int W, double inv_alpha, const int* __restrict__ tcol,
                              const double* __restrict__ sC, double* __restrict__ Tv) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)K * nbar) return;
  int k0 = (int)(t / nbar), i = (int)(t - (long long)k0 * nbar);
  const double sr = inv_alpha * sC[t];
  for (int d = 0; d < 3; d++) {
    int kk = k0 + d - 1;
    if (kk < 0 || kk >= K) continue;
    for (int s = 0; s < W; s++) {
      int col = tcol[(size_t)s * nbar + i];
      size_t at = ((size_t)(k0 * 3 + d) * W + s) * nbar + i;
      Tv[at] = col < 0 ? 0.0 : Tv[at] * sr * sC[(size_t)kk * nbar + col];
    }
  }
}

void assemble_T(bbot_ctx* c) {
  DevGeom& g = c->g;
  Assembled& A = c->as;
  size_t nv = (size_t)g.K * 3 * g.W * g.nbar;
  if (A.Tv.n != nv) A.Tv.alloc(nv, c->dev.stream);
  A.precond = c->opts.precond;
  if (c->opts.precond != 0) {
    const bool hss = c->opts.precond == 2;
    const long long n = c->n(), m = c->m();
    if (A.dAinv.n != (size_t)n) A.dAinv.alloc(n, c->dev.stream);
    launch(c->dev, k_dainv, dim3(nblocks(n, 256)), dim3(256), 0, n, g.N, (const double*)A.Aoff.p, A.dAinv.p);
    const double* cd = A.Cd.p;
    const double al = c->opts.alpha_hss;
    if (hss) {     // scalings D^-1/2 and the diagonal alpha^2 C of alpha^2 C + B D_A^-1 B^T
      if (A.sA.n != (size_t)n) A.sA.alloc(n, c->dev.stream);
      if (A.sC.n != (size_t)m) { A.sC.alloc(m, c->dev.stream); A.c2.alloc(m, c->dev.stream); }
      launch(c->dev, k_hss_scal, dim3(nblocks(std::max(n, m), 256)), dim3(256), 0, n, m, al,
             (const double*)A.dAinv.p, (const double*)A.Cd.p, A.sA.p, A.sC.p, A.c2.p);
      cd = A.c2.p;
    }
    dim3 grid(nblocks(g.nbar, 128), (g.K + T_KCH - 1) / T_KCH);
    launch(c->dev, k_assemble_S, grid, dim3(128), 0, g.nbar, g.K, g.N, g.NE, g.W, g.dt, (const double*)g.c.p,
           (const double*)A.gphi.p, (const double*)A.dAinv.p, cd, (const int*)g.fi_cell.p,
           (const int*)g.fi_child.p, (const int*)g.fi_edge.p, (const double*)g.fi_alpha.p, (const int*)g.fv_j.p,
           (const int*)g.fv_q.p, (const int*)g.fv_pos.p, A.Tv.p);
    if (hss)       // S_K = alpha I + B^ B^T / alpha = (1/alpha) D_C^-1/2 (alpha^2 C + B D_A^-1 B^T) D_C^-1/2
      launch(c->dev, k_hss_scale_S, dim3(nblocks((long long)g.K * g.nbar, 256)), dim3(256), 0, g.nbar, g.K, g.W,
             1.0 / al, (const int*)g.tcol.p, (const double*)A.sC.p, A.Tv.p);
    return;
  }
  dim3 grid(nblocks(g.nbar, 128), (g.K + T_KCH - 1) / T_KCH);
  launch(c->dev, k_assemble_T, grid, dim3(128), 0, g.nbar, g.K, g.NE, g.NEbar, g.W, g.dt, (const double*)g.c.p,
         (const double*)A.gphi.p, (const double*)A.omegabar.p, (const double*)A.sr.p, (const int*)g.cadj_e.p,
         (const int*)g.ca_pos.p, (const int*)g.fi_cell.p, (const int*)g.fi_child.p, (const int*)g.fi_ppos.p,
         (const int*)g.fi_edge.p, (const double*)g.fi_alpha.p, (const int*)g.fi_tbe.p, (const double*)g.fi_tbbeta.p,
         (const int*)g.fi_tbpL.p, (const int*)g.fi_tbpR.p, A.Tv.p, c->opts.recon, (const int*)g.eL.p,
         (const int*)g.eR.p, (const double*)g.lam.p, (const double*)c->rho_ext.p);
}

}  // namespace bbot
