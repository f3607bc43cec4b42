// geometry.h -- L0: host construction of the two-level TPFA geometry
// (§2.1) and of the fixed index tables the device kernels
// use.  Built once per context; uploaded to HBM; shared by every time slice.
#pragma once
#include <vector>
#include <cstdint>

namespace bbot {

struct Geometry {
  int nbar = 0, N = 0, NE = 0, NEbar = 0;
  double area = 0;                       // |Omega| = sum cbar
  // coarse cells (T-bar)
  std::vector<double> cbar;              // |c-bar|
  std::vector<double> ccx, ccy;          // circumcentres
  // coarse internal edges: L < R
  std::vector<int> ebL, ebR;
  std::vector<double> ebar_len, wbar_len, lam_bar;
  std::vector<int> cadj_e, cadj_nb;      // [3][nbar] coarse edge id / neighbour, -1 pad
  // fine kites: cell 3t+s at vertex s of triangle t
  std::vector<double> c;                 // |c|
  std::vector<double> xx, xy;            // cell points (v+cc)/2 (A2)
  // fine internal edges
  std::vector<int> eL, eR;               // L < R
  std::vector<double> e_len, w_len, lam; // |e|, |w|, lambda (A3)
  std::vector<int8_t> etype;             // 0: midpoint-circumcentre, 1: half coarse edge
  std::vector<int> fadj_e, fadj_nb;      // [4][N] fine edge id / neighbour, -1 pad
};

// Throws Error(BBOT_E_GEOMETRY) if a triangle is not CCW, not acute, or the
// meshes are not TPFA-admissible (|w| > 0, cell-point segment orthogonal to
// the edge).
Geometry build_geometry(const double* verts, int nv, const int* tris, int nt);

}  // namespace bbot
