// ctx.cuh -- the opaque bbot_ctx: device-resident geometry, state, per-Newton-
// step assembly, AMG hierarchies and Krylov workspaces.
//
// HBM layout: everything slice-major fp64.
//   phi      [K+1][N]          rho_ext [K+2][Nbar] (slices 0 and K+1 = rho_in, rho_f)
//   s        [K][Nbar]         omega, gphi [K+1][N_E]   (edge weights, grad phi)
//   omegabar [K][Nbar_E]       T values [K][3][W][Nbar] (slot-major ELL, pattern shared
//                                                        by all slices: tcol [W][Nbar])
#pragma once
#include "common.cuh"
#include "geometry.h"
#include "amg.cuh"
#include "krylov.cuh"
#include "comm.cuh"
#include <string>
#include <memory>

namespace bbot {

// Per-coarse-cell tables for B rows and T assembly (built on the host, tassemble.cu).
constexpr int CE_MAX = 9;    // fine edges sigma with R_E[sigma,i] != 0 (3 type a + <= 6 type b)
constexpr int FI_MAX = 9;    // fine cells in a B row (3 children + <= 6 across i's boundary)
constexpr int FI_EMAX = 4;   // edges of E(i) incident to such a fine cell
constexpr int TB_MAX = 2;    // type-b edges of a fine cell
constexpr int W_MAX = 16;    // T spatial stencil width cap
constexpr int FV_MAX = 6;    // coarse cells j whose B row holds a given fine cell (SIMPLE)

struct DevGeom {
  int nbar = 0, N = 0, NE = 0, NEbar = 0, K = 0, W = 0;
  long long Tnnz = 0;                         // structural nnz of T
  double dt = 0, area = 0;
  DBuf<double> cbar, c;                       // areas
  DBuf<int> ebL, ebR;                         // coarse internal edges
  DBuf<double> ebar_coef, lam_bar;            // |e-bar|/|w-bar|, lambda-bar
  DBuf<int> cadj_e, cadj_nb;                  // [3][nbar]
  DBuf<int> eL, eR;                           // fine internal edges
  DBuf<double> e_len, w_len, lam;
  DBuf<int> fadj_e, fadj_nb;                  // [4][N]
  // B-row edge list per coarse cell: (edge, R_E[sigma,i])
  DBuf<int> ce_edge;                          // [CE_MAX][nbar], -1 pad
  DBuf<double> ce_coef;                       // [CE_MAX][nbar]
  // T assembly tables
  DBuf<int> tcol;                             // [W][nbar] spatial columns, -1 pad; tcol[0][i] = i
  DBuf<int> fi_cell;                          // [FI_MAX][nbar] fine cell, -1 pad
  DBuf<int> fi_child;                         // [FI_MAX][nbar] 1 if child of i
  DBuf<int> fi_ppos;                          // [FI_MAX][nbar] pos of par(f) in S(i)
  DBuf<int> fi_edge;                          // [FI_MAX][FI_EMAX][nbar]
  DBuf<double> fi_alpha;                      // [FI_MAX][FI_EMAX][nbar] 1/2 R_E|e| E[f,sigma]
  DBuf<int> fi_tbe;                           // [FI_MAX][TB_MAX][nbar] type-b edges of f
  DBuf<double> fi_tbbeta;                     // [FI_MAX][TB_MAX][nbar] 1/2 R_f[sigma,f]|e|
  DBuf<int> fi_tbpL, fi_tbpR;                 // [FI_MAX][TB_MAX][nbar] pos of par L/R in S(i)
  DBuf<int> ca_pos;                           // [3][nbar] pos of coarse neighbour in S(i)
  // SIMPLE S-hat assembly (NEXT f1): for the q-th fine cell f of B row i, the rows j whose
  // B row also holds f: j, the index of f in F(j), and the position of j in S(i)
  DBuf<int> fv_j, fv_q, fv_pos;               // [FI_MAX][FV_MAX][nbar], fv_j = -1 pad
  DBuf<int> slice_A, slice_T;                 // row -> slice for AMG level 0
  DBuf<int> slice_S;                          // all 0: AMG(S-hat) aggregates across time (A32)
};

struct Assembled {
  bool valid = false;
  DBuf<double> omega, gphi;       // [K+1][NE]
  DBuf<double> Aoff;              // [K+1][4][N] A_k off-diagonals per kite slot (cell-ELL, -omega)
  DBuf<double> omegabar;          // [K][NEbar]
  DBuf<double> Cd, sr;            // C = cbar s/rho, s/rho  (m)
  DBuf<double> f, g, h, gt;       // RHS pieces
  DBuf<double> rhs;               // (f; P gt) (BB) or (f; gt) (SIMPLE)  (n+m)
  DBuf<double> Tv;                // [K][3][W][nbar]: T (BB) or S-hat = C + B diag(A)^-1 B^T (SIMPLE)
  DBuf<double> dAinv;             // 1 / diag(A)  (n; SIMPLE, HSS)
  DBuf<double> sA, sC, c2;        // HSS: diag(A)^-1/2 (n), C^-1/2 (m), alpha^2 C (m)
  int precond = 0;                // preconditioner the assembly was built for
  double scale = 0;               // ||(f;g;h)||
  DBuf<double> dscale;            // the same on the device (read by the captured solve)
  double res_norm = 0;            // ||F||
  bool rhs_user = false;          // f, g, h, rhs hold a caller's right-hand side (bbot_solve_rhs)
};

struct bbot_ctx_impl;

}  // namespace bbot

struct bbot_ctx {
  int devid = 0;                 // CUDA device of the context (every host thread of a call sets it)
  size_t stack_prev = 0;         // device stack limit before bbot_create
  bbot::Dev dev;
  bbot::Reducer red;
  bbot_solver_opts opts;
  std::string err;
  bbot::Geometry hg;           // host geometry (kept for inspection)
  bbot::DevGeom g;
  // state
  bbot::DBuf<double> phi, rho_ext, s;
  double mu = 1.0;
  bbot::Assembled as;
  bbot::AmgHierarchy amgA, amgT;
  bbot::AmgWork amgw;
  // AMG(T) is set up concurrently with AMG(A): its own stream + host thread (solver.cu)
  bbot::Dev dev2;
  bbot::AmgWork amgw2;
  // direction
  bool have_dir = false;
  bbot::DBuf<double> sol, dphi, drho, ds;
  bbot::DBuf<double> drho0;      // solve(rhs): slice-mass part of drho
  // workspaces
  bbot::DevGmres outer, innerT;
  bbot::DevPcg pcg;
  // CUDA graph of one whole solve (FGMRES + BB applies + recovery), captured
  // after each assembly (the AMG hierarchies it reads are rebuilt per step)
  bool use_graph = true;
  cudaGraphExec_t solve_exec = nullptr;
  double t_capture_ms = 0;      // last capture + instantiate (0 when the graph was replayed)
  double t_assemble_ms = 0, t_setup_ms = 0;   // last bbot_assemble
  bbot::DBuf<double> tmp_n, tmp_n2, tmp_m, tmp_m2, tmp_nm, tmp_nm2;
  bbot::DBuf<double> scal;      // device scalars / per-slice scratch (>= 8*(K+2))
  bbot::DBuf<long long> scan_ws;
  bbot::DBuf<double> nrm_T;      // ||r2|| of the current BB apply (device scalar)
  // multi-GPU time slabs (dist.cu, comm.cuh): owned potential slices [own_begin, own_end)
  int rank = 0, nranks = 1, own_begin = 0, own_end = 1 << 30;
  std::unique_ptr<bbot::Comm> comm;   // NCCL or virtual exchange layer (nranks > 1)
  bool slab() const { return nranks > 1; }
  // owned slices: potential [pa, pb), density [ra, rb)  (all of them on one rank)
  int pa() const { return slab() ? own_begin : 0; }
  int pb() const { return slab() ? own_end : g.K + 1; }
  int ra() const { return std::min(pa(), g.K); }
  int rb() const { return std::min(pb(), g.K); }
  long long n() const { return (long long)g.N * (g.K + 1); }
  long long m() const { return (long long)g.nbar * g.K; }
};
