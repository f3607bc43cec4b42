// krylov.cuh -- I1/I5: right-preconditioned flexible GMRES(restart) with CGS2
// ([Saad 1993]; cap P:1770) and I4: per-time-slice PCG
// (P:1469).  Host control, device work: all vector arithmetic in kernels with
// deterministic reductions; the (restart+1) x restart Hessenberg and its Givens
// rotations live on the host (a few hundred flops per iteration).
#pragma once
#include "common.cuh"
#include <functional>

namespace bbot {

using DevOp = std::function<void(const double*, double*)>;

struct KrylovResult {
  int its = 0;
  bool converged = false;
  double res = 0;
};

struct Fgmres {
  long long n = 0;
  int restart = 0;
  DBuf<double> V, Z, w, hdev, ydev;
  DBuf<double> hpin_dummy;
  double* hhost = nullptr;   // pinned
  void ensure(Dev& d, long long n_, int restart_);
  ~Fgmres();
  // x = 0 initial guess; stops when the Arnoldi residual <= tol*scale.
  KrylovResult solve(Dev& d, Reducer& red, const DevOp& op, const DevOp& pre, const double* b, double* x,
                     double scale, double tol, int maxit);
};

struct PcgSlices {
  long long n = 0;
  int nslices = 0;
  DBuf<double> r, z, p, q;
  DBuf<double> sc;        // per-slice scalars: bn rn rz rzn pq alpha beta active
  DBuf<int> its, any;
  // returns per-slice iteration counts (host)
  std::vector<int> solve(Dev& d, Reducer& red, const DevOp& op, const DevOp& pre, const double* b, double* x,
                         int nslices, long long slice_len, double tol, int maxit);
};

// BLAS-1 helpers (deterministic)
void dev_copy(Dev& d, const double* a, double* b, long long n);
void dev_scale(Dev& d, const double* a, double s, double* b, long long n);
void dev_axpby(Dev& d, double alpha, const double* a, double beta, double* b, long long n);  // b = alpha a + beta b
double dev_norm(Dev& d, Reducer& red, const double* a, long long n, double* dscratch);

}  // namespace bbot
