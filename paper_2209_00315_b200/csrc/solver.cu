// solver.cu -- orchestration of one Newton system: assembly + BB setup (a1, a3),
// the BB preconditioner apply (a4), FGMRES on (4.17) (a5), recovery (a6).
#include "ops.cuh"

namespace bbot {

void apply_A(bbot_ctx* c, const double* x, double* y);   // ops.cu

namespace {
struct EvTimer {
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit EvTimer(cudaStream_t st) : s(st) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  double ms() {
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float t = 0;
    cudaEventElapsedTime(&t, a, b);
    return t;
  }
  ~EvTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};
}  // namespace

void assemble_all(bbot_ctx* c, bbot_solve_stats* st) {
  const bbot_solver_opts& o = c->opts;
  EvTimer t0(c->dev.stream);
  compute_residual(c, true);
  assemble_T(c);
  double ta = t0.ms();
  EvTimer t1(c->dev.stream);
  AmgWork& w = c->amgw;
  amg_setup(c->dev, c->amgA, view_A(c), c->g.slice_A.p, c->g.K + 1, 0, o.omega_A, o.coarse_max_A, w);
  amg_setup(c->dev, c->amgT, view_T(c), c->g.slice_T.p, c->g.K, 1, o.omega_T, o.coarse_max_T, w);
  double ts = t1.ms();
  c->as.valid = true;
  if (st) {
    st->t_assemble_ms = ta;
    st->t_setup_ms = ts;
    st->amg_levels_A = (int)c->amgA.lv.size();
    st->amg_levels_T = (int)c->amgT.lv.size();
    st->scale = c->as.scale;
  }
}

void bb_apply(bbot_ctx* c, const double* r, double* z) {
  const bbot_solver_opts& o = c->opts;
  long long n = c->n(), m = c->m();
  const double* r1 = r;
  const double* r2 = r + n;
  double* z1 = z;
  double* z2 = z + n;
  // (i) T z = -r2, GMRES(restart_T) right-preconditioned by one AMG(T) V-cycle (4.26, A9)
  dev_scale(c->dev, r2, -1.0, c->tmp_m.p, m);
  double nr2 = dev_norm(c->dev, c->red, r2, m, c->scal.p);
  SliceEllView vT = view_T(c);
  c->innerT.ensure(c->dev, m, o.restart_T);
  KrylovResult kt = c->innerT.solve(
      c->dev, c->red, [&](const double* x, double* y) { apply_T(c, x, y); },
      [&](const double* x, double* y) { amg_vcycle(c->dev, c->amgT, vT, x, y); }, c->tmp_m.p, c->tmp_m2.p, nr2,
      o.eps_T, o.maxit_inner);
  c->bb_T_its += kt.its;
  // (ii) y = P^T Mbar^-1 Atilde z   (A12)
  bb_y_from_z(c, c->tmp_m2.p, z2);
  // (iii) b = r1 - B^T P^T y, slice means removed (compatibility)
  bb_rhs_A(c, r1, z2, c->tmp_n2.p);
  // (iv) A_k x^k = b^k, per-slice PCG + AMG(A) V-cycle (4.20), then slice means removed
  EdgeLapView vA = view_A(c);
  std::vector<int> its = c->pcg.solve(
      c->dev, c->red, [&](const double* x, double* y) { apply_A(c, x, y); },
      [&](const double* x, double* y) { amg_vcycle(c->dev, c->amgA, vA, x, y); }, c->tmp_n2.p, z1, c->g.K + 1,
      c->g.N, o.eps_A, o.maxit_inner);
  for (int v : its) {
    c->bb_A_max = std::max(c->bb_A_max, v);
    c->bb_A_total += v;
  }
  remove_slice_mean(c, z1, c->g.K + 1, c->g.N);
}

void solve(bbot_ctx* c, bbot_solve_stats* st) {
  const bbot_solver_opts& o = c->opts;
  BB_REQUIRE(c->as.valid, BBOT_E_ORDER, "bbot_solve before bbot_assemble");
  long long n = c->n(), m = c->m();
  c->bb_T_its = 0;
  c->bb_A_max = 0;
  c->bb_A_total = 0;
  c->outer.ensure(c->dev, n + m, o.restart);
  EvTimer t0(c->dev.stream);
  KrylovResult kr = c->outer.solve(
      c->dev, c->red, [&](const double* x, double* y) { jp_matvec(c, x, y); },
      [&](const double* x, double* y) { bb_apply(c, x, y); }, c->as.rhs.p, c->sol.p, c->as.scale, o.eps_out,
      o.maxit);
  double tk = t0.ms();
  EvTimer t1(c->dev.stream);
  recover(c);
  double tr = t1.ms();
  c->have_dir = true;
  if (st) {
    st->outer_its = kr.its;
    st->inner_T_its = c->bb_T_its;
    st->inner_A_its_max = c->bb_A_max;
    st->inner_A_its_total = c->bb_A_total;
    st->converged = kr.converged ? 1 : 0;
    st->scale = c->as.scale;
    st->rel_res = c->as.scale > 0 ? kr.res / c->as.scale : 0.0;
    st->t_krylov_ms = tk;
    st->t_recover_ms = tr;
  }
}

}  // namespace bbot
