// comm.cuh -- the exchange layer of the time-slab decomposition.
//
// Every slice-structured vector lives in GLOBAL layout on every rank (slice k at the same
// offset everywhere); a rank computes only the slices of its slab.  Rank q of P owns the
// potential slices [a_q, a_{q+1}), a_q = B floor(q nb / P) (whole time blocks of B slices,
// A42; a_P = K+1), and -- for every vector whose slices are density (time-level) slices,
// S = K of them -- the slices [min(a_q, S), min(a_{q+1}, S)); on the coarse levels of
// AMG(T), whose rows are grouped by time block (Layout::unit = B), the blocks
// [a_q / B, min(a_{q+1} / B, nb)).
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
  int unit = 1;                   // density slices per layout entry (AMG(T) coarse levels: a time block)
  int S() const { return (int)off.size() - 1; }
  static Layout uniform(int S, long long len, long long base = 0) {
    Layout L;
    L.off.resize(S + 1);
    for (int s = 0; s <= S; s++) L.off[s] = base + (long long)s * len;
    return L;
  }
};

// A42: AMG(T) aggregates within time blocks of B consecutive density slices (nb = floor(K/B)
// blocks, the last one taking the remainder) -- the same rule as oracle/amg.py::time_blocks.
// The slabs are unions of whole blocks, so the decomposition stays exact (P <= nb).  B = 1
// (I3's within-slice aggregation): blocks of max(1, floor(K/8)) slices cut the T iterations
// 2-3x on some systems and doubled them on others (A42), so they are not used.
inline int time_block_size(int K) { (void)K; return 1; }   // A42 measured: blocks of max(1, K/8) not adopted
inline int time_blocks(int K) { return std::max(1, K / time_block_size(K)); }
inline int time_block_of(int K, int k) { return std::min(k / time_block_size(K), time_blocks(K) - 1); }

// first potential slice of rank `rank` (rank == nranks: Kp1): a_r = B floor(r nb / P)
int slab_begin(int Kp1, int rank, int nranks);
// owned entries [lo, hi) of rank q for a layout of S entries of `unit` slices each
// (slab basis: Kp1 potential slices; unit > 1 only on block-aligned slab boundaries)
inline void slab_owned(int Kp1, int nranks, int q, int S, int& lo, int& hi, int unit = 1) {
  lo = std::min(slab_begin(Kp1, q, nranks) / unit, S);
  hi = std::min(slab_begin(Kp1, q + 1, nranks) / unit, S);
}

class Comm {
 public:
  int rank = 0, nranks = 1, Kp1 = 1;      // Kp1: number of potential slices (slab basis)
  virtual ~Comm() {}
  // owned entries [lo, hi) of a layout
  void owned(const Layout& L, int q, int& lo, int& hi) const { slab_owned(Kp1, nranks, q, L.S(), lo, hi, L.unit); }
  virtual void halo(Dev& d, const Layout& L, double* base) = 0;
  virtual void allgather(Dev& d, const Layout& L, double* base) = 0;
  virtual void barrier(Dev& d) = 0;
};

std::unique_ptr<Comm> make_nccl_comm(int rank, int nranks, int Kp1, const unsigned char* uid);
std::unique_ptr<Comm> make_virtual_comm(int rank, int nranks, int Kp1, long long group);

}  // namespace bbot
