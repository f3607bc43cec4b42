// comm.cuh -- the exchange layer of the time-slab decomposition.
//
// Every slice-structured vector lives in GLOBAL layout on every rank (slice k at the same
// offset everywhere); a rank computes only the slices of its slab.  Rank q of P owns the
// potential slices [a_q, a_{q+1}), a_q = floor(q (K+1) / P), and -- for every vector whose
// slices are density (time-level) slices, S = K of them, and for every level of AMG(T),
// whose coarse rows stay slice-grouped -- the slices [min(a_q, S), min(a_{q+1}, S)).
// A Layout is the slice offsets of one such vector (S + 1 entries, host).
//
// Two operations, both in place on the global-layout buffer:
//   halo(L, base)       slice lo-1 from the left neighbour and slice hi from the right one
//                       (the one-slice halos of J_P, B, B^T, the T SpMV and its V-cycle levels)
//   allgather(L, base)  every rank's owned slices to every rank (slice-partial reduction
//                       totals, the coarse tail input, the Newton direction)
// Backends: NCCL (one process per GPU, grouped send/recv and broadcasts over NVLink /
// NVSwitch) and VIRTUAL (P contexts of one process, one host thread each, exchanging by
// device-to-device copies through a shared table of buffer pointers, host barriers between
// the phases) -- the second runs the whole decomposed solve on one GPU for the P-invariance
// tests.  Calls are eager (the multi-rank solve is issued eagerly: its loops are host-driven).
#pragma once
#include "common.cuh"
#include <memory>

namespace bbot {

struct Layout {
  std::vector<long long> off;     // S + 1 element offsets
  int S() const { return (int)off.size() - 1; }
  static Layout uniform(int S, long long len, long long base = 0) {
    Layout L;
    L.off.resize(S + 1);
    for (int s = 0; s <= S; s++) L.off[s] = base + (long long)s * len;
    return L;
  }
};

int slab_begin(int nslices, int rank, int nranks);
// owned slices [lo, hi) of rank q for a layout of S slices (slab basis: Kp1 potential slices)
inline void slab_owned(int Kp1, int nranks, int q, int S, int& lo, int& hi) {
  lo = std::min(slab_begin(Kp1, q, nranks), S);
  hi = std::min(slab_begin(Kp1, q + 1, nranks), S);
}

class Comm {
 public:
  int rank = 0, nranks = 1, Kp1 = 1;      // Kp1: number of potential slices (slab basis)
  virtual ~Comm() {}
  // owned slices [lo, hi) of a layout with S slices
  void owned(int S, int q, int& lo, int& hi) const { slab_owned(Kp1, nranks, q, S, lo, hi); }
  virtual void halo(Dev& d, const Layout& L, double* base) = 0;
  virtual void allgather(Dev& d, const Layout& L, double* base) = 0;
  virtual void barrier(Dev& d) = 0;
};

std::unique_ptr<Comm> make_nccl_comm(int rank, int nranks, int Kp1, const unsigned char* uid);
std::unique_ptr<Comm> make_virtual_comm(int rank, int nranks, int Kp1, long long group);

}  // namespace bbot
