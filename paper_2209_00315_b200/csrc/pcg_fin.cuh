// pcg_fin.cuh -- per-slice PCG (I4) device scalars and the epilogues of
// the fused reductions that update them.  Shared by krylov.cuh (the PCG driver)
// and amg.cu (the AMG(A) V-cycle fuses r.z into its last level-0 kernel).
#pragma once
#include "common.cuh"

namespace bbot {

// per-slice PCG device scalars: [slice] arrays + loop state
struct PcgScal {
  int it, maxit, flag;
  int A_max;                  // max per-slice iteration count over the applies of one solve
  long long A_total;          // sum of per-slice iteration counts over the applies of one solve
};

// ---- PCG kernel pieces shared with the operator emitter (solver.cu)
// Layout of DevPcg::s (doubles, each [nslices]).
enum { PS_BN = 0, PS_RN, PS_RZ, PS_PQ, PS_ALPHA, PS_BETA, PS_ACTIVE, PS_TMP, PS_COUNT };

// Epilogue of the fused "p = z + beta p, q = A z + beta q, partial p.q" kernel:
// alpha = rz / pq on active slices (a slice with pq <= 0 stops), its += active.
struct PcgAlphaFin {
  double* s;
  int* its;
  int ns;
  __device__ void operator()(const double* out) const {
    for (int k = threadIdx.x; k < ns; k += blockDim.x) {
      double act = s[PS_ACTIVE * ns + k];
      double pq = out[k];
      if (act != 0.0 && !(pq > 0.0)) act = 0.0;
      s[PS_ACTIVE * ns + k] = act;
      s[PS_ALPHA * ns + k] = act != 0.0 ? s[PS_RZ * ns + k] / pq : 0.0;
      its[k] += act != 0.0 ? 1 : 0;
    }
  }
};

// Epilogue of the per-slice r.z reduction: beta (it > 0) and rz update.
struct PcgRzFin {
  double* s;
  const PcgScal* P;
  int ns;
  __device__ void operator()(const double* out) const {
    const int it = P->it;
    for (int q = threadIdx.x; q < ns; q += blockDim.x) {
      double rzn = out[q];
      if (it == 0) {
        s[PS_RZ * ns + q] = rzn;
        s[PS_BETA * ns + q] = 0.0;
      } else {
        double act = s[PS_ACTIVE * ns + q];
        double rz = s[PS_RZ * ns + q];
        s[PS_BETA * ns + q] = act != 0.0 ? rzn / (rz != 0.0 ? rz : 1.0) : 0.0;
        if (act != 0.0) s[PS_RZ * ns + q] = rzn;
      }
    }
  }
};

// A per-slice dot fused into a producer kernel: grid (parts, ns) over [ns][L].
struct SliceDotFuse {
  RedArgs R;
  int parts, ns;
  long long L;
  PcgRzFin fin;
  const double* active;   // [ns] slices still iterating (others are skipped by the producer)
};

}  // namespace bbot
