/* bbot.h -- C-ABI of libbbot.so, the B200-native (sm_100a, fp64) hot path of
 * arXiv 2209.00315: the BB-preconditioned Krylov solve of the interior-point
 * Newton saddle-point system of the two-level TPFA finite-volume discretisation
 * of the Benamou-Brenier optimal-transport problem, plus the per-Newton-step
 * assembly, recovery and the IPM loop that feed it.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n (LaTeX source of the
 * paper).  Equation numbers follow the LaTeX labels; readings A1-A30 of the
 * paper's ambiguities are listed in DESIGN.md §2.
 *
 * Conventions (all calls):
 *  - Sizes: Nbar coarse triangles, N = 3 Nbar fine kites, K interior density
 *    levels, Delta t = 1/(K+1), n = N (K+1) potential unknowns,
 *    m = Nbar K density unknowns.
 *  - Vectors are slice-major fp64: phi = (phi^1;...;phi^{K+1}), slice k holds
 *    N values, fine kite 3t+s = kite at local vertex s of triangle t;
 *    rho = (rho^1;...;rho^K), s likewise, Nbar values per slice.
 *  - bbot_mem tells whether a vector pointer is HOST memory or DEVICE memory on
 *    the context's device.  Host pointers are copied synchronously inside the
 *    call; device pointers must stay valid until the call returns and are used
 *    on the context's stream.  The caller owns every buffer it passes; the
 *    library owns its device workspace (cudaMallocAsync on the ctx stream).
 *  - Every call returns a bbot_status; bbot_last_error() holds a message.
 *    Non-convergence (FGMRES cap, "the 400 limit") is recorded in the
 *    stats (converged = 0) and returns BBOT_OK: the best iterate is kept.
 *  - Calls on one context are serialised; a context is not thread-safe.
 *  - There is no CPU fallback: every arithmetic step runs in CUDA kernels.
 */
#ifndef BBOT_H
#define BBOT_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bbot_ctx bbot_ctx;

typedef enum {
  BBOT_OK = 0,
  BBOT_E_INPUT = 1,     /* bad argument (NULL, size, K < 1, option out of range)        */
  BBOT_E_GEOMETRY = 2,  /* mesh not acute / not CCW / not TPFA-admissible      */
  BBOT_E_STATE = 3,     /* rho <= 0 or s <= 0 in a state (IPM interior)           */
  BBOT_E_NOCONV = 4,    /* reserved (non-convergence is reported in stats, not here)     */
  BBOT_E_CUDA = 5,      /* CUDA runtime error (message has the CUDA string)              */
  BBOT_E_NCCL = 6,      /* NCCL error or libnccl.so.2 not loadable                       */
  BBOT_E_NOMEM = 7,     /* device allocation failed                                     */
  BBOT_E_INTERNAL = 8,  /* internal capacity exceeded (AMG row too wide) / bug           */
  BBOT_E_ORDER = 9      /* call order (e.g. solve before assemble)                      */
} bbot_status;

typedef enum { BBOT_MEM_HOST = 0, BBOT_MEM_DEVICE = 1 } bbot_mem;

/* Solver options (A14-A16, I3).  Defaults in brackets. */
typedef struct {
  double eps_out;      /* outer FGMRES tol on ||res(4.17)|| / ||(f;g;h)|| [1e-10] (A16) */
  double eps_T;        /* inner GMRES tol for T z = -r2, relative [1e-1]           */
  double eps_A;        /* inner PCG tol for A_k x = b, relative [1e-3] (A14; paper 5e-2)    */
  int restart;         /* FGMRES restart [30] (A15), 1..32                                  */
  int maxit;           /* FGMRES cap [400]                                         */
  int restart_T;       /* inner GMRES restart [10], 1..32                                   */
  int maxit_inner;     /* inner caps (T GMRES total its, per-slice PCG its) [50]            */
  double omega_A;      /* damped-Jacobi weight, AMG(A) [2/3]                                */
  double omega_T;      /* l1-Jacobi weight, AMG(T) [1.0] (D = sum_j |T_ij|, I3)             */
  int coarse_max_A;    /* AMG(A) coarsest: max rows per time slice [64]                     */
  int coarse_max_T;    /* AMG(T) coarsest: max rows in total [1024]                         */
  int precond;         /* 0 = BB on (4.17) [0]; 2 = HSS (below); 1 = SIMPLE on the saddle-point system
                        * (eq:saddle-point) with eq:sca-precs: FGMRES
                        * on J = [[A, B^T],[B, -C]], rhs (f; g~); the inner solve is
                        * S-hat = C + B diag(A)^-1 B^T (stored in T's slot, A31/A32) by
                        * GMRES(restart_T) + AMG, eps_T; recovery dphi = x1, drho = x2.   */
  int coarse_max_S;    /* AMG(S-hat) coarsest: max rows in total [256] (A32)                 */
  /* precond = 2: HSS (NEXT f2, eq:prec-hss) on the same saddle-point system as
   * SIMPLE, diagonally scaled: M^-1 = D^-1/2 H_a^-1 K_a^-1 D^-1/2 diag(I,-I),
   * D = diag(diag(A), C); K_a^-1 by the dual Schur complement a I + B^ B^T/a (eq:solve-K,
   * stored in T's slot, GMRES(restart_T) + AMG), H_a^-1 by per-slice PCG + AMG on the scaled
   * shifted Laplacians A^_k + a I (eq:solve-laplacians); both inner solves to eps_in_hss. */
  double alpha_hss;    /* HSS relaxation parameter [0.5]                              */
  double eps_in_hss;   /* HSS inner tolerance [1e-1]                                  */
  int recon;           /* density reconstruction on the fine edges [0]: 0 = weighted
                        * arithmetic mean (A3); 1 = weighted HARMONIC mean (NEXT f4, Remark 3.3,
                        * DESIGN.md A39-A41): A_k, F_phi, F_rho, B, B^T, the kinetic energy and
                        * the Newton (2,2) block W = dF_rho/drho follow R_H; (4.17) carries
                        * C_H = C - W, the BB preconditioner diag(C_H) in T, the coarse harmonic
                        * mean in Atilde and the fine Jacobian in Btilde.  BB only.          */
} bbot_solver_opts;

typedef struct {
  int outer_its;            /* FGMRES iterations (P:601 Outer/Lin.sys)                     */
  int inner_T_its;          /* total T-GMRES iterations (P:607 Inner/Outer numerator)      */
  int inner_A_its_max;      /* max per-slice PCG iterations in any apply                   */
  long long inner_A_its_total;
  int converged;            /* 1 if ||res|| <= eps_out ||(f;g;h)||                          */
  double rel_res;           /* final Arnoldi residual / ||(f;g;h)||                         */
  double scale;             /* ||(f;g;h)||                                                  */
  double t_assemble_ms;     /* a1 + T assembly                                              */
  double t_setup_ms;        /* AMG(A) + AMG(T) setup (the paper's "% preprocess")   */
  double t_krylov_ms;       /* FGMRES incl. BB applies                                      */
  double t_recover_ms;      /* a6 (inside the solve graph: 0 when the solve ran as a graph)   */
  int amg_levels_A, amg_levels_T;
  double t_graph_ms;        /* host time to capture + instantiate the solve graph (0 on replay) */
} bbot_solve_stats;

typedef struct {
  double mu0;               /* [1]     (A17)                                                */
  double mu_factor;         /* [0.5]   (A17)                                                */
  double mu_min;            /* [1e-8]  (A17: last mu = 2^-26)                                */
  double newton_rel_tol;    /* [1e-2]  stop ||F|| <= max(tol*mu, floor)*||F(x0;mu0)|| (A18)  */
  double newton_abs_floor;  /* [1e-11]                                                      */
  double frac_to_boundary;  /* [0.95]  (A20)                                                */
  int newton_max;           /* [30]    Newton steps per mu (A18)                             */
  int max_mu_steps;         /* [0 = all] truncate the mu schedule                           */
  double mu_tight;          /* [0.3]   below this mu the A_k solves tighten ... (A14')       */
  double eps_A_tight;       /* [1e-5]  ... to this relative tolerance                        */
  double simple_below_mu;   /* [0]     A34: SIMPLE (precond 1) for every mu below this       */
} bbot_ipm_opts;

typedef struct {
  double mu; int newton; double alpha; double res_norm;
  bbot_solve_stats solve;
} bbot_ipm_record;

typedef void (*bbot_ipm_cb)(const bbot_ipm_record* rec, void* user);

typedef struct {
  int n_systems;            /* Newton systems solved                                        */
  long long total_outer;    /* sum of outer iterations                                      */
  long long total_inner_T;
  int n_unconverged;        /* systems that hit the FGMRES cap (the paper's dagger)         */
  double final_mu;
  double kinetic_energy;    /* D12 at the final state                                       */
  double wall_ms;
  int n_simple_fallback;    /* always 0 (kept for ABI stability): AMG(S-hat) coarse rows have no
                             * width cap any more, so every SIMPLE system is solved with SIMPLE */
} bbot_ipm_stats;

void bbot_default_solver_opts(bbot_solver_opts* o);
void bbot_default_ipm_opts(bbot_ipm_opts* o);

/* Create a context on the current CUDA device.
 * vertices: host, nv x 2 (x,y); tris: host, nt x 3 vertex indices, CCW.
 * rho_in / rho_f: host, nt coarse cell averages, >= 0, equal mass.
 * Builds the coarse + fine TPFA geometry on the host (readings A2, A3),
 * validates it (acute, CCW, orthogonal, |w| > 0) -> BBOT_E_GEOMETRY, and
 * uploads it.  opts may be NULL (defaults).  stream: a cudaStream_t or NULL
 * (the legacy default stream).  The state is set to the A19 initial point
 * at mu = 1. */
bbot_status bbot_create(const double* vertices, int nv, const int* tris, int nt, int K,
                        const double* rho_in, const double* rho_f,
                        const bbot_solver_opts* opts, void* stream, bbot_ctx** out);
void bbot_destroy(bbot_ctx* ctx);
const char* bbot_last_error(const bbot_ctx* ctx);

bbot_status bbot_sizes(const bbot_ctx* ctx, long long* nbar, long long* N, long long* NE,
                       int* K, long long* n, long long* m);
bbot_status bbot_set_opts(bbot_ctx* ctx, const bbot_solver_opts* opts);
/* T storage: spatial stencil width W (slots per slice offset) and structural nnz. */
bbot_status bbot_T_info(const bbot_ctx* ctx, int* W, long long* nnz);

/* State (phi n, rho m, s m) and the barrier parameter mu.  set_state checks
 * rho > 0 and s > 0 (BBOT_E_STATE) and invalidates the assembly. */
bbot_status bbot_set_state(bbot_ctx* ctx, const double* phi, const double* rho,
                           const double* s, double mu, bbot_mem mem);
bbot_status bbot_get_state(bbot_ctx* ctx, double* phi, double* rho, double* s,
                           double* mu, bbot_mem mem);
/* A19 initial point: rho^k uniform with the boundary mass, s = mu0/rho, phi = 0. */
bbot_status bbot_init_state(bbot_ctx* ctx, double mu0);

/* Residuals (2.5)-(2.7) (A5, A6) at the current state; any output may be
 * NULL.  norm = ||(F_phi;F_rho;F_s)||_2. */
bbot_status bbot_residual(bbot_ctx* ctx, double* F_phi, double* F_rho, double* F_s,
                          double* norm, bbot_mem mem);

/* a1 + a3: per-Newton-step assembly at the current state: edge weights, grad phi,
 * C = Mbar diag(s/rho) (A7), RHS (f; P g~) ((4.17)), Atilde,
 * T = C Mbar^-1 Atilde - B M^-1 Btilde ((4.26), A8) and both AMG hierarchies.
 * With precond = 1 (SIMPLE): RHS (f; g~), S-hat in place of T, AMG(S-hat) only. */
bbot_status bbot_assemble(bbot_ctx* ctx);

/* a2: y = J_P x with J_P = [[A, B^T P^T],[P B, -P C P^T]] ((4.17));
 * after a SIMPLE assembly, y = J x with J = [[A, B^T],[B, -C]].
 * x, y: n+m vectors. Requires bbot_assemble. */
bbot_status bbot_jp_matvec(bbot_ctx* ctx, const double* x, double* y, bbot_mem mem);

/* a4: z = BB-preconditioner applied to r (n+m) -- or, after a SIMPLE assembly, the
 * SIMPLE preconditioner (eq:sca-precs; inner_T_its = S-hat GMRES its, A its 0):
 * T z2 = -r2 (GMRES+AMG(T)),
 * y = P^T Mbar^-1 Atilde z2, b = r1 - B^T P^T y (slice means removed),
 * A_k x^k = b^k (PCG+AMG(A)), out (x; y)  ((4.18)-(4.20), (4.26), A9, A12, A14). */
bbot_status bbot_bb_apply(bbot_ctx* ctx, const double* r, double* z, bbot_mem mem,
                          int* inner_T_its, int* inner_A_its_max);

/* a5 + a6: FGMRES on (4.17) with the BB preconditioner (or, after a SIMPLE assembly, on
 * the saddle-point system with SIMPLE; recovery dphi = x1, drho = x2), then recovery of
 * (dphi, drho, ds); st also reports the timings of the last bbot_assemble.
 * (dphi, drho, ds) ((4.15) with A10, A30).  Outputs may be
 * NULL (the direction is always kept in the context for bbot_newton_update). */
bbot_status bbot_solve(bbot_ctx* ctx, double* dphi, double* drho, double* ds,
                       bbot_solve_stats* st, bbot_mem mem);

/* solve(rhs) -> direction (north star): the Newton system (3.1)
 * of the last bbot_assemble with a CALLER-GIVEN right-hand side:
 *   [[A, B^T, 0], [B, 0, Mbar], [0, diag(s), diag(rho)]] (dphi; drho; ds) = (f; g; h).
 * f: n, g: m, h: m (slice-major, as the state; `mem` says host or device).  ds is
 * eliminated: g~ = g - Mbar h / rho; FGMRES (BB: on (4.17) with rhs (f; P g~),
 * P:1424-1448; SIMPLE: on the saddle-point system with rhs (f; g~)) stops at
 * eps_out ||(f;g;h)||_2; recovery as bbot_solve.  Solvability: (3.1) is
 * singular along (1;0;0) (Remark 3.1), so sum_k 1^T f^k must vanish.  (4.17)
 * needs 1^T f^k = 0 slice by slice (A30); the slice masses m_k = c-bar^T drho^k are fixed
 * first from the phi rows' slice sums (m_k = m_{k-1} - dt 1^T f^k) and the rest is solved
 * through (4.17).  For an f outside the range the solve runs to the cap (converged = 0).
 * The operator is NOT rebuilt: it stays the one of the last assembly; the next bbot_solve
 * re-derives the Newton right-hand side
 * itself.  The direction is not kept for bbot_newton_update. */
bbot_status bbot_solve_rhs(bbot_ctx* ctx, const double* f, const double* g, const double* h, double* dphi,
                           double* drho, double* ds, bbot_solve_stats* st, bbot_mem mem);

/* a7: step length (fraction to boundary, A20), update of (phi, rho, s) with the
 * last direction, per-slice renormalisation of rho (Remark 3.2). */
bbot_status bbot_newton_update(bbot_ctx* ctx, double frac_to_boundary, double* alpha);

/* a7: full IPM run from the current state (mu schedule A17, Newton stop A18); with
 * o->simple_below_mu > 0 every Newton system at mu below it uses SIMPLE (A34). */
bbot_status bbot_ipm_run(bbot_ctx* ctx, const bbot_ipm_opts* o, bbot_ipm_stats* st,
                         bbot_ipm_cb cb, void* user);

/* D12: KE = sum_k Delta t 1/2 phi^k^T A_k phi^k at the current state. */
bbot_status bbot_kinetic_energy(bbot_ctx* ctx, double* ke);

/* ---- inspection (parity tests, profiling) ---- */
/* T (or S-hat after a SIMPLE assembly) as host CSR (rows m; columns sorted).  Call with rowptr == NULL to get nnz. */
bbot_status bbot_get_T(bbot_ctx* ctx, long long* nnz, long long* rowptr, int* cols, double* vals);
/* which: 0 = AMG(A), 1 = AMG(T).  sizes: >= 32 entries. */
bbot_status bbot_amg_info(bbot_ctx* ctx, int which, int* nlevels, long long* sizes);
/* level `level` of hierarchy `which`: rows n, stored nnz (-1 on level 0, which is read
 * through the operator's own view, not stored), coarse rows nc (0 at the coarsest), and
 * the first level handled by the per-slice tail kernel (0: none).  For byte models. */
bbot_status bbot_amg_level_info(bbot_ctx* ctx, int which, int level, long long* n, long long* nnz, long long* nc,
                                int* tail);
/* fine-row -> coarse-row map of level `level` (host, length sizes[level]). */
bbot_status bbot_amg_agg(bbot_ctx* ctx, int which, int level, int* agg);
/* one V-cycle x = M^-1 b on level 0 of hierarchy `which` (length n or m). */
bbot_status bbot_amg_vcycle(bbot_ctx* ctx, int which, const double* b, double* x, bbot_mem mem);
/* count of CUDA kernel launches issued EAGERLY by this context since creation
 * (kernels replayed from the solve's CUDA graph are not counted; run the same
 * solve with bbot_set_exec_mode(ctx, 0) or under the profiler to count them). */
long long bbot_launch_count(const bbot_ctx* ctx);
/* Device memory of the library's private stream-ordered pool on the context's device (every
 * bbot buffer -- state, assembly, AMG hierarchies, Krylov workspaces -- is allocated from it;
 * contexts of one process on one device share the pool): *used_bytes = currently allocated,
 * *peak_bytes = high-water mark since the pool was created.  BBOT_E_INPUT on NULL. */
bbot_status bbot_mem_usage(const bbot_ctx* ctx, long long* used_bytes, long long* peak_bytes);
/* Multi-GPU time slabs ("well suited for
 * parallelization"), one rank per GPU.  Rank r owns whole AMG(T) time blocks (bbot_time_blocks:
 * B slices, nb = floor(K/B) blocks): the potential slices [k_begin, k_end),
 * k_begin = B floor(r nb / P) (k_end of the last rank = K+1), and the density slices
 * [k_begin, min(k_end, K)); P <= nb.  The Newton SOLVE is decomposed: the FGMRES and T-GMRES Krylov vectors, J_P
 * (4.17), the T-solve (T SpMV and every grid-wide level of the AMG(T) V-cycle), the BB glue
 * (4.18)-(4.20), the per-slice A_k PCG solves and the recovery (a6) run on the owned slices,
 * with one-slice halo exchanges (x1 from the right and x2, y from the left for J_P, B, B^T;
 * z from both sides for T and for each AMG(T) level; dphit from the right for the delta-lambda
 * sums) and allgathers of per-slice reduction totals: every dot / norm is the in-order sum of
 * per-slice totals whose block partition depends only on the slice length, so the result is
 * bitwise equal to the single-GPU solve for every P.  The coarse AMG(T) tail (<= 16384 rows)
 * runs redundantly on the allgathered level.  Replicated (every rank, bitwise equal): the
 * state, assembly, AMG setups, the Newton update (the direction is allgathered after the
 * recovery).  Memory is not divided in this scope (global-layout vectors on every rank).
 * Multi-rank solves are issued eagerly (host-driven loops; BB preconditioner only).
 * bbot_nccl_unique_id: on rank 0; the caller broadcasts the 128 bytes.
 * bbot_set_dist: after bbot_create, before bbot_assemble (NCCL, uid required for P > 1).
 * bbot_set_dist_virtual: P contexts of ONE process (one host thread per rank, each calling
 * the same sequence of API calls concurrently) exchanging by device-to-device copies through
 * a process-wide group `group` -- the decomposition on a single GPU, for testing. */
bbot_status bbot_nccl_unique_id(unsigned char out[128]);
bbot_status bbot_set_dist(bbot_ctx* ctx, int rank, int nranks, const unsigned char* uid);
bbot_status bbot_set_dist_virtual(bbot_ctx* ctx, int rank, int nranks, long long group);
bbot_status bbot_get_slab(const bbot_ctx* ctx, int* k_begin, int* k_end);
/* The ownership rule of the exchange layer (host only, no GPU): rank `rank` of `nranks` owns
 * the slices [*lo, *hi) of a slice-structured vector with S slices when the slabs are cut
 * over Kp1 = K+1 potential slices; its halos are slices *lo-1 (from rank-1) and *hi (from
 * rank+1).  Slabs are unions of whole AMG(T) time blocks (bbot_time_blocks): the first
 * slice of rank r is B * floor(r * nb / P) (the last rank also owns slice K).  For the
 * exchange-plan tests.  BBOT_E_INPUT on a bad rank / count. */
bbot_status bbot_slab_plan(int Kp1, int nranks, int rank, int S, int* lo, int* hi);
/* The time blocks of AMG(T) (A42; the aggregation unit of T, whose rows couple
 * consecutive time slices through the time Laplacian in -B M^-1 B~, eq. (4.26)):
 * *block_size = B consecutive density slices (B = 1 in this build: multi-slice blocks were
 * measured and not adopted), *nblocks = floor(K/B), the last block taking the remainder.
 * Host only.  BBOT_E_INPUT if K < 1. */
bbot_status bbot_time_blocks(int K, int* block_size, int* nblocks);

/* Execution mode of bbot_solve.  1 (default): the whole solve -- FGMRES, the BB
 * applies with their inner GMRES / per-slice PCG loops, recovery -- is captured
 * once per bbot_assemble into one CUDA graph whose loops are conditional WHILE
 * nodes driven by device-side convergence tests, and replayed with a single
 * launch (no host round trip inside the solve).  0: the same kernels are issued
 * eagerly and the host reads each loop condition.  Results are bitwise
 * identical.  Between bbot_prof_start and bbot_prof_stop solves run eagerly. */
bbot_status bbot_set_exec_mode(bbot_ctx* ctx, int use_graph);
/* Per-launch profiler: between start and stop every kernel launch is bracketed
 * by CUDA events on the context stream (adds ~2 event records per launch; use
 * for kernel shares, not for the headline timing).  stop writes a text table
 * "demangled-name<TAB>launches<TAB>total_ms<TAB>grid-CTAs" (one line per kernel and
 * grid size) into buf (NUL-terminated,
 * truncated to buflen) and the required size into *needed. */
bbot_status bbot_prof_start(bbot_ctx* ctx);
bbot_status bbot_prof_stop(bbot_ctx* ctx, char* buf, long long buflen, long long* needed);

#ifdef __cplusplus
}
#endif
#endif /* BBOT_H */
