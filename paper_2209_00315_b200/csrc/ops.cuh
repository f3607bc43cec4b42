// ops.cuh -- declarations of the per-Newton-step kernels (assemble.cu, ops.cu)
// and of the solver orchestration (solver.cu).
#pragma once
#include "ctx.cuh"

namespace bbot {

// assemble.cu
void upload_geometry(bbot_ctx* c, const Geometry& g, int K);
void assemble_edges(bbot_ctx* c);                    // omega, gphi, omegabar, C, s/rho
void compute_residual(bbot_ctx* c, bool write_rhs);  // F (as f,g,h = -F), g~, rhs, norms
void assemble_T(bbot_ctx* c);                        // T values
LapView view_A(bbot_ctx* c);
ScaledLapView view_As(bbot_ctx* c);                  // HSS: A^ + alpha I
SliceEllView view_T(bbot_ctx* c);

// ops.cu
void jp_matvec(bbot_ctx* c, const double* x, double* y);                    // (4.17)
void apply_T(bbot_ctx* c, const double* x, double* y);                      // y = T x
void bb_y_from_z(bbot_ctx* c, const double* z, double* y);                  // y = P^T Mbar^-1 Atilde z
void bb_rhs_A(bbot_ctx* c, const double* r1, const double* y, double* b);   // b = r1 - B^T y, slice means removed
void remove_slice_mean(bbot_ctx* c, double* x, int ns, long long L);         // arithmetic mean per slice
void j_matvec(bbot_ctx* c, const double* x, double* y);                     // (eq:saddle-point)
void simple_c(bbot_ctx* c, const double* r, double* z1, double* cvec);      // z1 = diag(A)^-1 r1, c = r2 - B z1
void simple_out(bbot_ctx* c, const double* r, const double* z2, double* out);  // (diag(A)^-1(r1 - B^T z2); z2)
void hss_c(bbot_ctx* c, const double* r, double* negc);                     // -c = sC (r2 - B(dAinv r1)/alpha)
void hss_u(bbot_ctx* c, const double* r, const double* v, double* w, double* u);   // u = sA (r1 - B^T(sC v))/alpha
void hss_out(bbot_ctx* c, const double* v, double* z);                      // z1 *= sA, z2 = sC v/(1+alpha)
void set_user_rhs(bbot_ctx* c);                                            // solve(rhs): (f;g;h) in as.f/g/h
void finish_user_solve(bbot_ctx* c);                                       // drho += drho0
void recover(bbot_ctx* c);                                                   // a6
double newton_update(bbot_ctx* c, double tau);                              // a7 step + renormalise
double kinetic_energy(bbot_ctx* c);
void init_state(bbot_ctx* c, double mu0);
void check_state(bbot_ctx* c);

// solver.cu
void assemble_all(bbot_ctx* c, bbot_solve_stats* st);
void bb_apply(bbot_ctx* c, const double* r, double* z, int* its_T, int* its_A_max);   // eager
void solve(bbot_ctx* c, bbot_solve_stats* st);                                          // graph (or eager)
void drop_solve_graph(bbot_ctx* c);

// dist.cu
void nccl_unique_id(unsigned char out[128]);
void set_dist(bbot_ctx* c, int rank, int nranks, const unsigned char* uid, long long group);
void drop_dist(bbot_ctx* c);

}  // namespace bbot
