// capi.cu -- the C-ABI (include/bbot.h).  Argument checking, host<->device
// marshalling, exception -> status translation, and the IPM loop (a7).
#include "ops.cuh"
#include <chrono>
#include <cmath>
#include <cstring>
#include <cxxabi.h>
#include <map>
#include <cstdlib>

using namespace bbot;

namespace {

bbot_status fail(bbot_ctx* c, const Error& e) {
  if (c) c->err = e.what();
  return e.status;
}

#define API_BEGIN(ctx) \
  try {
#define API_END(ctx)                                              \
  }                                                               \
  catch (const Error& e) { return fail(ctx, e); }                 \
  catch (const std::exception& e) {                               \
    if (ctx) (ctx)->err = e.what();                               \
    return BBOT_E_INTERNAL;                                       \
  }                                                               \
  return BBOT_OK;

void copy_in(bbot_ctx* c, double* dst, const double* src, long long n, bbot_mem mem) {
  BB_REQUIRE(src != nullptr || n == 0, BBOT_E_INPUT, "null input pointer");
  if (n == 0) return;
  BB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double),
                          mem == BBOT_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->dev.stream));
  if (mem == BBOT_MEM_HOST) sync(c->dev);
}
void copy_out(bbot_ctx* c, double* dst, const double* src, long long n, bbot_mem mem) {
  if (!dst || n == 0) return;
  BB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double),
                          mem == BBOT_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c->dev.stream));
  if (mem == BBOT_MEM_HOST) sync(c->dev);
}
// time slabs: the owned slices of an (n+m) vector to every rank (whole-vector API outputs)
void allgather_nm(bbot_ctx* c, double* v) {
  if (!c->slab()) return;
  c->comm->allgather(c->dev, Layout::uniform(c->g.K + 1, c->g.N), v);
  c->comm->allgather(c->dev, Layout::uniform(c->g.K, c->g.nbar), v + c->n());
}

void check_opts(const bbot_solver_opts& o) {
  BB_REQUIRE(o.eps_out > 0 && o.eps_T > 0 && o.eps_A > 0, BBOT_E_INPUT, "tolerances must be > 0");
  BB_REQUIRE(o.restart >= 1 && o.restart <= GM_MAXR && o.maxit >= 1, BBOT_E_INPUT, "bad FGMRES restart/maxit");
  BB_REQUIRE(o.restart_T >= 1 && o.restart_T <= GM_MAXR && o.maxit_inner >= 1, BBOT_E_INPUT, "bad inner caps");
  BB_REQUIRE(o.omega_A > 0 && o.omega_A < 2 && o.omega_T > 0 && o.omega_T < 2, BBOT_E_INPUT, "bad Jacobi weight");
  BB_REQUIRE(o.coarse_max_A >= 2 && o.coarse_max_A <= 120 && o.coarse_max_T >= 1 && o.coarse_max_T <= 8192,
             BBOT_E_INPUT, "bad coarse sizes");
  BB_REQUIRE(o.precond >= 0 && o.precond <= 2, BBOT_E_INPUT, "precond must be 0 (BB), 1 (SIMPLE) or 2 (HSS)");
  BB_REQUIRE(o.alpha_hss > 0 && o.eps_in_hss > 0, BBOT_E_INPUT, "bad HSS alpha / eps_in");
  BB_REQUIRE(o.recon == 0 || o.recon == 1, BBOT_E_INPUT, "recon must be 0 (arithmetic) or 1 (harmonic)");
  BB_REQUIRE(o.recon == 0 || o.precond == 0, BBOT_E_INPUT, "the harmonic reconstruction is built for BB (precond 0)");
  BB_REQUIRE(o.coarse_max_S >= 1 && o.coarse_max_S <= 8192, BBOT_E_INPUT, "bad coarse_max_S");
}

}  // namespace

extern "C" {

void bbot_default_solver_opts(bbot_solver_opts* o) {
  if (!o) return;
  o->eps_out = 1e-10;
  o->eps_T = 1e-1;
  o->eps_A = 1e-3;
  o->restart = 30;
  o->maxit = 400;
  o->restart_T = 10;
  o->maxit_inner = 50;
  o->omega_A = 2.0 / 3.0;
  o->omega_T = 1.0;
  o->coarse_max_A = 64;
  o->coarse_max_T = 1024;
  o->precond = 0;
  o->coarse_max_S = 256;
  o->alpha_hss = 0.5;
  o->eps_in_hss = 1e-1;
  o->recon = 0;
}

void bbot_default_ipm_opts(bbot_ipm_opts* o) {
  if (!o) return;
  o->mu0 = 1.0;
  o->mu_factor = 0.5;
  o->mu_min = 1e-8;
  o->newton_rel_tol = 1e-2;
  o->newton_abs_floor = 1e-11;
  o->frac_to_boundary = 0.95;
  o->newton_max = 30;
  o->max_mu_steps = 0;
  o->mu_tight = 0.3;
  o->eps_A_tight = 1e-5;
  o->simple_below_mu = 0.0;
}

bbot_status bbot_create(const double* vertices, int nv, const int* tris, int nt, int K, const double* rho_in,
                        const double* rho_f, const bbot_solver_opts* opts, void* stream, bbot_ctx** out) {
  if (!out) return BBOT_E_INPUT;
  *out = nullptr;
  bbot_ctx* c = new bbot_ctx();
  try {
    BB_REQUIRE(K >= 1, BBOT_E_INPUT, "K must be >= 1");
    BB_REQUIRE(rho_in && rho_f, BBOT_E_INPUT, "null densities");
    if (opts) c->opts = *opts;
    else bbot_default_solver_opts(&c->opts);
    check_opts(c->opts);
    c->dev.stream = (cudaStream_t)stream;
    int devid = 0;
    BB_CUDA(cudaGetDevice(&devid));
    c->devid = devid;
    device_pool();   // the library's private pool on this device (common.cu)
    {   // the AMG(A) tail kernel recurses through the K-cycle levels (depth <= 2 x levels);
        // the previous limit is restored by bbot_destroy
      size_t stk = 0;
      BB_CUDA(cudaDeviceGetLimit(&stk, cudaLimitStackSize));
      c->stack_prev = stk;
      if (stk < 4096) BB_CUDA(cudaDeviceSetLimit(cudaLimitStackSize, 4096));
    }
    BB_CUDA(cudaDeviceGetAttribute(&c->dev.num_sms, cudaDevAttrMultiProcessorCount, devid));
    c->red.init(&c->dev, std::max(K + 2, 64));
    BB_CUDA(cudaStreamCreateWithFlags(&c->dev2.stream, cudaStreamNonBlocking));
    c->dev2.num_sms = c->dev.num_sms;
    if (const char* e = getenv("BBOT_EAGER")) c->use_graph = (atoi(e) == 0);
    if (const char* e = getenv("BBOT_SYNC_CHECK")) c->dev.sync_check = (atoi(e) != 0);
    for (int i = 0; i < nt; i++)
      BB_REQUIRE(rho_in[i] >= 0 && rho_f[i] >= 0 && std::isfinite(rho_in[i]) && std::isfinite(rho_f[i]),
                 BBOT_E_INPUT, "densities must be finite and >= 0");
    c->hg = build_geometry(vertices, nv, tris, nt);
    upload_geometry(c, c->hg, K);
    cudaStream_t s = c->dev.stream;
    long long n = c->n(), m = c->m();
    c->phi.alloc(n, s);
    c->rho_ext.alloc((size_t)(K + 2) * nt, s);
    c->s.alloc(m, s);
    BB_CUDA(cudaMemcpyAsync(c->rho_ext.p, rho_in, nt * sizeof(double), cudaMemcpyHostToDevice, s));
    BB_CUDA(cudaMemcpyAsync(c->rho_ext.p + (size_t)(K + 1) * nt, rho_f, nt * sizeof(double), cudaMemcpyHostToDevice,
                            s));
    c->sol.alloc(n + m, s);
    c->dphi.alloc(n, s);
    c->drho.alloc(m, s);
    c->ds.alloc(m, s);
    c->tmp_n.alloc(n, s);
    c->tmp_n2.alloc(n, s);
    c->tmp_m.alloc(m, s);
    c->tmp_m2.alloc(m, s);
    c->scal.alloc(8 * (size_t)(K + 2) + 64, s);
    c->as.dscale.alloc(1, s);
    init_state(c, 1.0);
    sync(c->dev);
  } catch (const Error& e) {
    bbot_status st = e.status;
    fprintf(stderr, "bbot_create: %s\n", e.what());
    delete c;
    return st;
  }
  *out = c;
  return BBOT_OK;
}

void bbot_destroy(bbot_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->dev.stream);
  drop_solve_graph(c);
  drop_dist(c);
  cudaStream_t s2 = c->dev2.stream;
  if (s2) cudaStreamSynchronize(s2);
  size_t stk = c->stack_prev;
  delete c;
  if (s2) cudaStreamDestroy(s2);
  if (stk > 0 && stk < 4096) cudaDeviceSetLimit(cudaLimitStackSize, stk);
}

const char* bbot_last_error(const bbot_ctx* c) { return c ? c->err.c_str() : "null context"; }

bbot_status bbot_sizes(const bbot_ctx* c, long long* nbar, long long* N, long long* NE, int* K, long long* n,
                       long long* m) {
  if (!c) return BBOT_E_INPUT;
  if (nbar) *nbar = c->g.nbar;
  if (N) *N = c->g.N;
  if (NE) *NE = c->g.NE;
  if (K) *K = c->g.K;
  if (n) *n = c->n();
  if (m) *m = c->m();
  return BBOT_OK;
}

bbot_status bbot_T_info(const bbot_ctx* c, int* W, long long* nnz) {
  if (!c) return BBOT_E_INPUT;
  if (W) *W = c->g.W;
  if (nnz) *nnz = c->g.Tnnz;
  return BBOT_OK;
}

bbot_status bbot_set_opts(bbot_ctx* c, const bbot_solver_opts* o) {
  if (!c || !o) return BBOT_E_INPUT;
  API_BEGIN(c)
  check_opts(*o);
  c->opts = *o;
  c->as.valid = false;
  drop_solve_graph(c);
  API_END(c)
}

bbot_status bbot_set_state(bbot_ctx* c, const double* phi, const double* rho, const double* s, double mu,
                           bbot_mem mem) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  BB_REQUIRE(mu >= 0 && std::isfinite(mu), BBOT_E_INPUT, "mu must be >= 0");
  copy_in(c, c->phi.p, phi, c->n(), mem);
  copy_in(c, c->rho_ext.p + c->g.nbar, rho, c->m(), mem);
  copy_in(c, c->s.p, s, c->m(), mem);
  c->mu = mu;
  c->as.valid = false;
  c->have_dir = false;
  check_state(c);
  API_END(c)
}

bbot_status bbot_get_state(bbot_ctx* c, double* phi, double* rho, double* s, double* mu, bbot_mem mem) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  copy_out(c, phi, c->phi.p, c->n(), mem);
  copy_out(c, rho, c->rho_ext.p + c->g.nbar, c->m(), mem);
  copy_out(c, s, c->s.p, c->m(), mem);
  if (mu) *mu = c->mu;
  API_END(c)
}

bbot_status bbot_init_state(bbot_ctx* c, double mu0) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  BB_REQUIRE(mu0 > 0, BBOT_E_INPUT, "mu0 must be > 0");
  init_state(c, mu0);
  sync(c->dev);
  API_END(c)
}

bbot_status bbot_residual(bbot_ctx* c, double* F_phi, double* F_rho, double* F_s, double* norm, bbot_mem mem) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  compute_residual(c, true);
  c->as.valid = false;   // T / AMG not rebuilt here
  long long n = c->n(), m = c->m();
  // the kernels store f = -F etc.; return F
  if (F_phi) {
    dev_scale(c->dev, c->as.f.p, -1.0, c->tmp_n.p, n);
    copy_out(c, F_phi, c->tmp_n.p, n, mem);
  }
  if (F_rho) {
    dev_scale(c->dev, c->as.g.p, -1.0, c->tmp_m.p, m);
    copy_out(c, F_rho, c->tmp_m.p, m, mem);
  }
  if (F_s) {
    dev_scale(c->dev, c->as.h.p, -1.0, c->tmp_m2.p, m);
    copy_out(c, F_s, c->tmp_m2.p, m, mem);
  }
  sync(c->dev);
  if (norm) *norm = c->as.res_norm;
  API_END(c)
}

bbot_status bbot_assemble(bbot_ctx* c) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  assemble_all(c, nullptr);
  API_END(c)
}

bbot_status bbot_jp_matvec(bbot_ctx* c, const double* x, double* y, bbot_mem mem) {
  if (!c || !x || !y) return BBOT_E_INPUT;
  API_BEGIN(c)
  BB_REQUIRE(c->as.valid, BBOT_E_ORDER, "bbot_jp_matvec before bbot_assemble");
  long long nm = c->n() + c->m();
  if (c->tmp_nm.n != (size_t)nm) { c->tmp_nm.alloc(nm, c->dev.stream); c->tmp_nm2.alloc(nm, c->dev.stream); }
  copy_in(c, c->tmp_nm.p, x, nm, mem);
  if (c->as.precond != 0) j_matvec(c, c->tmp_nm.p, c->tmp_nm2.p);   // SIMPLE / HSS: (eq:saddle-point)
  else jp_matvec(c, c->tmp_nm.p, c->tmp_nm2.p);
  allgather_nm(c, c->tmp_nm2.p);    // time slabs: every rank returns the whole product
  copy_out(c, y, c->tmp_nm2.p, nm, mem);
  sync(c->dev);
  API_END(c)
}

bbot_status bbot_bb_apply(bbot_ctx* c, const double* r, double* z, bbot_mem mem, int* inner_T_its,
                          int* inner_A_its_max) {
  if (!c || !r || !z) return BBOT_E_INPUT;
  API_BEGIN(c)
  BB_REQUIRE(c->as.valid, BBOT_E_ORDER, "bbot_bb_apply before bbot_assemble");
  long long nm = c->n() + c->m();
  if (c->tmp_nm.n != (size_t)nm) { c->tmp_nm.alloc(nm, c->dev.stream); c->tmp_nm2.alloc(nm, c->dev.stream); }
  copy_in(c, c->tmp_nm.p, r, nm, mem);
  bb_apply(c, c->tmp_nm.p, c->tmp_nm2.p, inner_T_its, inner_A_its_max);
  allgather_nm(c, c->tmp_nm2.p);
  copy_out(c, z, c->tmp_nm2.p, nm, mem);
  sync(c->dev);
  API_END(c)
}

bbot_status bbot_solve(bbot_ctx* c, double* dphi, double* drho, double* ds, bbot_solve_stats* st, bbot_mem mem) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  bbot_solve_stats loc;
  memset(&loc, 0, sizeof(loc));
  if (c->as.valid && c->as.rhs_user) {   // a bbot_solve_rhs replaced the Newton right-hand side
    compute_residual(c, true);
    c->as.rhs_user = false;
  }
  solve(c, &loc);
  copy_out(c, dphi, c->dphi.p, c->n(), mem);
  copy_out(c, drho, c->drho.p, c->m(), mem);
  copy_out(c, ds, c->ds.p, c->m(), mem);
  if (st) *st = loc;
  API_END(c)
}

bbot_status bbot_solve_rhs(bbot_ctx* c, const double* f, const double* g, const double* h, double* dphi,
                           double* drho, double* ds, bbot_solve_stats* st, bbot_mem mem) {
  if (!c || !f || !g || !h) return BBOT_E_INPUT;
  API_BEGIN(c)
  BB_REQUIRE(c->as.valid, BBOT_E_ORDER, "bbot_solve_rhs before bbot_assemble");
  long long n = c->n(), m = c->m();
  copy_in(c, c->as.f.p, f, n, mem);
  copy_in(c, c->as.g.p, g, m, mem);
  copy_in(c, c->as.h.p, h, m, mem);
  set_user_rhs(c);
  bbot_solve_stats loc;
  memset(&loc, 0, sizeof(loc));
  solve(c, &loc);
  finish_user_solve(c);
  c->have_dir = false;     // not a Newton direction of the state: bbot_newton_update refuses it
  copy_out(c, dphi, c->dphi.p, n, mem);
  copy_out(c, drho, c->drho.p, m, mem);
  copy_out(c, ds, c->ds.p, m, mem);
  if (st) *st = loc;
  API_END(c)
}

bbot_status bbot_newton_update(bbot_ctx* c, double tau, double* alpha) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  BB_REQUIRE(c->have_dir, BBOT_E_ORDER, "bbot_newton_update without a direction");
  BB_REQUIRE(tau > 0 && tau <= 1, BBOT_E_INPUT, "frac_to_boundary in (0,1]");
  double a = newton_update(c, tau);
  c->have_dir = false;
  if (alpha) *alpha = a;
  API_END(c)
}

bbot_status bbot_ipm_run(bbot_ctx* c, const bbot_ipm_opts* po, bbot_ipm_stats* st, bbot_ipm_cb cb, void* user) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  bbot_ipm_opts o;
  if (po) o = *po;
  else bbot_default_ipm_opts(&o);
  BB_REQUIRE(o.mu0 > 0 && o.mu_factor > 0 && o.mu_factor < 1 && o.mu_min > 0 && o.newton_max >= 1, BBOT_E_INPUT,
             "bad IPM options");
  auto t0 = std::chrono::steady_clock::now();
  bbot_ipm_stats S;
  memset(&S, 0, sizeof(S));
  // A17 schedule
  std::vector<double> mus;
  for (int j = 0;; j++) {
    double mu = o.mu0 * std::pow(o.mu_factor, j);
    if (!(mu >= o.mu_min * (1 - 1e-12))) break;
    mus.push_back(mu);
  }
  if (o.max_mu_steps > 0 && (int)mus.size() > o.max_mu_steps) mus.resize(o.max_mu_steps);
  BB_REQUIRE(o.eps_A_tight > 0, BBOT_E_INPUT, "bad eps_A_tight");
  const double eps_A0 = c->opts.eps_A;
  const int precond0 = c->opts.precond;
  struct Restore {           // the caller's eps_A and preconditioner come back even if a solve throws
    double& ref;
    double val;
    int& pref;
    int pval;
    ~Restore() {
      ref = val;
      pref = pval;
    }
  } restore{c->opts.eps_A, eps_A0, c->opts.precond, precond0};
  c->mu = o.mu0;
  compute_residual(c, false);
  double F0 = c->as.res_norm;
  for (double mu : mus) {
    c->mu = mu;
    // A14': tighter A_k solves once mu < mu_tight (the solve graph is re-captured per assembly)
    c->opts.eps_A = mu >= o.mu_tight ? eps_A0 : std::min(eps_A0, o.eps_A_tight);
    double tol = std::max(o.newton_rel_tol * mu, o.newton_abs_floor) * F0;   // A18
    for (int it = 0; it < o.newton_max; it++) {
      bbot_ipm_record rec;
      memset(&rec, 0, sizeof(rec));
      // A34: the mu-switched BB -> SIMPLE hybrid
      c->opts.precond = mu < o.simple_below_mu && c->opts.recon == 0 ? 1 : precond0;
      assemble_all(c, nullptr);
      solve(c, &rec.solve);
      rec.alpha = newton_update(c, o.frac_to_boundary);
      c->have_dir = false;
      compute_residual(c, false);
      rec.mu = mu;
      rec.newton = it;
      rec.res_norm = c->as.res_norm;
      S.n_systems++;
      S.total_outer += rec.solve.outer_its;
      S.total_inner_T += rec.solve.inner_T_its;
      if (!rec.solve.converged) S.n_unconverged++;
      if (cb) cb(&rec, user);
      if (rec.res_norm <= tol) break;
    }
  }
  c->opts.eps_A = eps_A0;
  c->opts.precond = precond0;
  S.final_mu = c->mu;
  S.kinetic_energy = kinetic_energy(c);
  S.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  c->as.valid = false;
  if (st) *st = S;
  API_END(c)
}

bbot_status bbot_kinetic_energy(bbot_ctx* c, double* ke) {
  if (!c || !ke) return BBOT_E_INPUT;
  API_BEGIN(c)
  *ke = kinetic_energy(c);
  API_END(c)
}

bbot_status bbot_get_T(bbot_ctx* c, long long* nnz, long long* rowptr, int* cols, double* vals) {
  if (!c || !nnz) return BBOT_E_INPUT;
  API_BEGIN(c)
  BB_REQUIRE(c->as.valid, BBOT_E_ORDER, "bbot_get_T before bbot_assemble");
  DevGeom& g = c->g;
  std::vector<int> tcol = c->g.tcol.download();
  std::vector<double> tv = c->as.Tv.download();
  int nbar = g.nbar, K = g.K, W = g.W;
  long long cnt = 0;
  std::vector<std::pair<int, double>> row;
  for (int k0 = 0; k0 < K; k0++)
    for (int i = 0; i < nbar; i++) {
      row.clear();
      for (int d = 0; d < 3; d++) {
        int kk = k0 + d - 1;
        if (kk < 0 || kk >= K) continue;
        for (int s = 0; s < W; s++) {
          int col = tcol[(size_t)s * nbar + i];
          if (col < 0) break;
          row.push_back({kk * nbar + col, tv[((size_t)(k0 * 3 + d) * W + s) * nbar + i]});
        }
      }
      std::sort(row.begin(), row.end());
      if (rowptr) {
        rowptr[(size_t)k0 * nbar + i] = cnt;
        for (size_t q = 0; q < row.size(); q++) {
          cols[cnt + q] = row[q].first;
          vals[cnt + q] = row[q].second;
        }
      }
      cnt += (long long)row.size();
    }
  if (rowptr) rowptr[(size_t)K * nbar] = cnt;
  *nnz = cnt;
  API_END(c)
}

bbot_status bbot_amg_info(bbot_ctx* c, int which, int* nlevels, long long* sizes) {
  if (!c || !nlevels) return BBOT_E_INPUT;
  AmgHierarchy& H = which == 0 ? c->amgA : c->amgT;
  *nlevels = (int)H.lv.size();
  if (sizes)
    for (size_t l = 0; l < H.lv.size() && l < 32; l++) sizes[l] = H.lv[l].n;
  return BBOT_OK;
}

bbot_status bbot_amg_level_info(bbot_ctx* c, int which, int level, long long* n, long long* nnz, long long* nc,
                                int* tail) {
  if (!c) return BBOT_E_INPUT;
  AmgHierarchy& H = which == 0 ? c->amgA : c->amgT;
  if (level < 0 || level >= (int)H.lv.size()) return BBOT_E_INPUT;
  AmgLevel& L = H.lv[level];
  if (n) *n = L.n;
  if (nnz) *nnz = L.rp.p ? (long long)L.ci.n : -1;   // level 0 is read through a view (no CSR): -1
  if (nc) *nc = L.nc;
  if (tail) *tail = H.tail;
  return BBOT_OK;
}

bbot_status bbot_amg_agg(bbot_ctx* c, int which, int level, int* agg) {
  if (!c || !agg) return BBOT_E_INPUT;
  API_BEGIN(c)
  AmgHierarchy& H = which == 0 ? c->amgA : c->amgT;
  BB_REQUIRE(level >= 0 && level + 1 < (int)H.lv.size(), BBOT_E_INPUT, "no aggregation at this level");
  std::vector<int> a = H.lv[level].agg.download();
  memcpy(agg, a.data(), a.size() * sizeof(int));
  API_END(c)
}

bbot_status bbot_amg_vcycle(bbot_ctx* c, int which, const double* b, double* x, bbot_mem mem) {
  if (!c || !b || !x) return BBOT_E_INPUT;
  API_BEGIN(c)
  BB_REQUIRE(c->as.valid, BBOT_E_ORDER, "bbot_amg_vcycle before bbot_assemble");
  BB_REQUIRE(which == 0 || which == 1, BBOT_E_INPUT, "which must be 0 (AMG(A)) or 1 (AMG(T))");
  BB_REQUIRE(!(which == 0 ? c->amgA : c->amgT).lv.empty(), BBOT_E_ORDER,
             "bbot_amg_vcycle: that hierarchy was not built by the last assembly (SIMPLE builds AMG(S-hat) only)");
  long long len = which == 0 ? c->n() : c->m();
  double* tb = which == 0 ? c->tmp_n.p : c->tmp_m.p;
  double* tx = which == 0 ? c->tmp_n2.p : c->tmp_m2.p;
  copy_in(c, tb, b, len, mem);
  if (which == 0 && c->as.precond == 2) amg_vcycle(c->dev, c->amgA, view_As(c), tb, tx);
  else if (which == 0) amg_vcycle(c->dev, c->amgA, view_A(c), tb, tx);
  else amg_vcycle(c->dev, c->amgT, view_T(c), tb, tx);
  copy_out(c, x, tx, len, mem);
  sync(c->dev);
  API_END(c)
}

long long bbot_launch_count(const bbot_ctx* c) { return c ? c->dev.launches : 0; }

bbot_status bbot_mem_usage(const bbot_ctx* c, long long* used_bytes, long long* peak_bytes) {
  if (!c || !used_bytes || !peak_bytes) return BBOT_E_INPUT;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->devid);
  cudaMemPool_t pool = bbot::device_pool();
  unsigned long long used = 0, high = 0;   // cuuint64_t
  cudaError_t e1 = cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
  cudaError_t e2 = cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &high);
  cudaSetDevice(prev);
  if (e1 != cudaSuccess || e2 != cudaSuccess) return BBOT_E_CUDA;
  *used_bytes = (long long)used;
  *peak_bytes = (long long)high;
  return BBOT_OK;
}

bbot_status bbot_nccl_unique_id(unsigned char out[128]) {
  if (!out) return BBOT_E_INPUT;
  try {
    nccl_unique_id(out);
  } catch (const Error& e) {
    fprintf(stderr, "bbot_nccl_unique_id: %s\n", e.what());
    return e.status;
  }
  return BBOT_OK;
}

bbot_status bbot_set_dist(bbot_ctx* c, int rank, int nranks, const unsigned char* uid) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  BB_REQUIRE(uid != nullptr || nranks == 1, BBOT_E_INPUT, "bbot_set_dist: NCCL unique id required (nranks > 1)");
  set_dist(c, rank, nranks, uid, 0);
  API_END(c)
}

bbot_status bbot_set_dist_virtual(bbot_ctx* c, int rank, int nranks, long long group) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  set_dist(c, rank, nranks, nullptr, group);
  API_END(c)
}

bbot_status bbot_slab_plan(int Kp1, int nranks, int rank, int S, int* lo, int* hi) {
  if (nranks < 1 || rank < 0 || rank >= nranks || S < 0 || !lo || !hi) return BBOT_E_INPUT;
  slab_owned(Kp1, nranks, rank, S, *lo, *hi);
  return BBOT_OK;
}

bbot_status bbot_time_blocks(int K, int* block_size, int* nblocks) {
  if (K < 1 || !block_size || !nblocks) return BBOT_E_INPUT;
  *block_size = time_block_size(K);
  *nblocks = time_blocks(K);
  return BBOT_OK;
}

bbot_status bbot_get_slab(const bbot_ctx* c, int* k_begin, int* k_end) {
  if (!c) return BBOT_E_INPUT;
  if (k_begin) *k_begin = c->nranks > 1 ? c->own_begin : 0;
  if (k_end) *k_end = c->nranks > 1 ? c->own_end : c->g.K + 1;
  return BBOT_OK;
}

bbot_status bbot_set_exec_mode(bbot_ctx* c, int use_graph) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  c->use_graph = use_graph != 0;
  drop_solve_graph(c);
  API_END(c)
}

bbot_status bbot_prof_start(bbot_ctx* c) {
  if (!c) return BBOT_E_INPUT;
  c->dev.prof = true;
  return BBOT_OK;
}

bbot_status bbot_prof_stop(bbot_ctx* c, char* buf, long long buflen, long long* needed) {
  if (!c) return BBOT_E_INPUT;
  API_BEGIN(c)
  Dev& d = c->dev;
  d.prof = false;
  sync(d);
  std::map<std::pair<const void*, long long>, std::pair<long long, double>> agg;
  for (auto& r : d.recs) {
    float ms = 0;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& a = agg[{r.fn, r.grid}];
    a.first++;
    a.second += ms;
    d.pool.push_back(r.a);
    d.pool.push_back(r.b);
  }
  d.recs.clear();
  std::string out;
  for (auto& kv : agg) {
    const char* nm = nullptr;
    std::string name = "?";
    if (cudaFuncGetName(&nm, kv.first.first) == cudaSuccess && nm) {
      int stt = 0;
      char* dm = abi::__cxa_demangle(nm, nullptr, nullptr, &stt);
      name = (stt == 0 && dm) ? dm : nm;
      free(dm);
    }
    char line[96];
    snprintf(line, sizeof(line), "\t%lld\t%.6f\t%lld\n", kv.second.first, kv.second.second, kv.first.second);
    out += name + line;
  }
  if (needed) *needed = (long long)out.size() + 1;
  if (buf && buflen > 0) {
    size_t n = std::min((size_t)buflen - 1, out.size());
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  API_END(c)
}

}  // extern "C"
