// geometry.cpp -- L0 host geometry (§2.1).
//
// Coarse mesh: acute CCW triangles; internal edges only.
// Fine mesh: 3 kites per triangle "joining the edges midpoints to the
// triangle's circumcenter"; kite 3t+s sits at local vertex s.
// Cell points: circumcentres (coarse) and (v + cc)/2 (fine, reading A2).
// lambda_sigma = d(x_L, sigma) / (d(x_L, sigma) + d(x_R, sigma)) (reading A3).
// Edge orientation: L = lower cell index.
#include "geometry.h"
#include "common.cuh"
#include <cmath>
#include <algorithm>
#include <numeric>

namespace bbot {

namespace {
struct P2 { double x, y; };
inline P2 sub(P2 a, P2 b) { return {a.x - b.x, a.y - b.y}; }
inline double dot(P2 a, P2 b) { return a.x * b.x + a.y * b.y; }
inline double cross(P2 a, P2 b) { return a.x * b.y - a.y * b.x; }
inline double norm(P2 a) { return std::hypot(a.x, a.y); }
inline P2 mid(P2 a, P2 b) { return {0.5 * (a.x + b.x), 0.5 * (a.y + b.y)}; }

// distance from p to the line through a, b
inline double line_dist(P2 p, P2 a, P2 b) {
  P2 d = sub(b, a);
  return std::fabs(cross(d, sub(p, a))) / norm(d);
}
// circumcentre via the perpendicular-bisector system relative to a
inline P2 circumcentre(P2 a, P2 b, P2 c) {
  P2 u = sub(b, a), v = sub(c, a);
  double den = 2.0 * cross(u, v);
  double uu = dot(u, u), vv = dot(v, v);
  return {a.x + (v.y * uu - u.y * vv) / den, a.y + (u.x * vv - v.x * uu) / den};
}
}  // namespace

Geometry build_geometry(const double* verts, int nv, const int* tris, int nt) {
  BB_REQUIRE(nv >= 3 && nt >= 1 && verts && tris, BBOT_E_INPUT, "empty mesh");
  Geometry g;
  g.nbar = nt;
  g.N = 3 * nt;
  auto V = [&](int i) { return P2{verts[2 * i], verts[2 * i + 1]}; };
  g.cbar.resize(nt);
  g.ccx.resize(nt);
  g.ccy.resize(nt);
  for (int t = 0; t < nt; t++) {
    int a = tris[3 * t], b = tris[3 * t + 1], c = tris[3 * t + 2];
    BB_REQUIRE(a >= 0 && a < nv && b >= 0 && b < nv && c >= 0 && c < nv, BBOT_E_INPUT,
               "triangle vertex index out of range");
    P2 pa = V(a), pb = V(b), pc = V(c);
    double ar = 0.5 * cross(sub(pb, pa), sub(pc, pa));
    BB_REQUIRE(ar > 0, BBOT_E_GEOMETRY, "triangle " + std::to_string(t) + " is not CCW / degenerate");
    // strictly acute: every corner has a positive dot product
    P2 P[3] = {pa, pb, pc};
    for (int s = 0; s < 3; s++) {
      double d = dot(sub(P[(s + 1) % 3], P[s]), sub(P[(s + 2) % 3], P[s]));
      BB_REQUIRE(d > 0, BBOT_E_GEOMETRY, "triangle " + std::to_string(t) + " is not acute (P:99)");
    }
    g.cbar[t] = ar;
    P2 cc = circumcentre(pa, pb, pc);
    g.ccx[t] = cc.x;
    g.ccy[t] = cc.y;
  }
  g.area = 0;
  for (double v : g.cbar) g.area += v;

  // ---- coarse internal edges: sort half-edges by (vmin, vmax, tri)
  struct HE { int v0, v1, t, s; };
  std::vector<HE> he(3 * (size_t)nt);
  for (int t = 0; t < nt; t++)
    for (int s = 0; s < 3; s++) {
      int a = tris[3 * t + s], b = tris[3 * t + (s + 1) % 3];
      he[3 * (size_t)t + s] = {std::min(a, b), std::max(a, b), t, s};
    }
  std::sort(he.begin(), he.end(), [](const HE& x, const HE& y) {
    if (x.v0 != y.v0) return x.v0 < y.v0;
    if (x.v1 != y.v1) return x.v1 < y.v1;
    return x.t < y.t;
  });
  g.cadj_e.assign(3 * (size_t)nt, -1);
  g.cadj_nb.assign(3 * (size_t)nt, -1);
  std::vector<int> eva, evb;
  for (size_t i = 0; i + 1 < he.size(); i++) {
    if (he[i].v0 == he[i + 1].v0 && he[i].v1 == he[i + 1].v1) {
      BB_REQUIRE(i + 2 >= he.size() || !(he[i + 2].v0 == he[i].v0 && he[i + 2].v1 == he[i].v1),
                 BBOT_E_GEOMETRY, "non-manifold edge");
      int tL = he[i].t, tR = he[i + 1].t;  // sorted by t within equal keys
      int e = (int)g.ebL.size();
      g.ebL.push_back(tL);
      g.ebR.push_back(tR);
      eva.push_back(he[i].v0);
      evb.push_back(he[i].v1);
      // slot-major [3][nbar]: slot = local edge index s of the triangle
      g.cadj_e[(size_t)he[i].s * nt + tL] = e;
      g.cadj_nb[(size_t)he[i].s * nt + tL] = tR;
      g.cadj_e[(size_t)he[i + 1].s * nt + tR] = e;
      g.cadj_nb[(size_t)he[i + 1].s * nt + tR] = tL;
      i++;
    }
  }
  g.NEbar = (int)g.ebL.size();
  g.ebar_len.resize(g.NEbar);
  g.wbar_len.resize(g.NEbar);
  g.lam_bar.resize(g.NEbar);
  for (int e = 0; e < g.NEbar; e++) {
    P2 a = V(eva[e]), b = V(evb[e]);
    P2 cL{g.ccx[g.ebL[e]], g.ccy[g.ebL[e]]}, cR{g.ccx[g.ebR[e]], g.ccy[g.ebR[e]]};
    g.ebar_len[e] = norm(sub(a, b));
    g.wbar_len[e] = norm(sub(cL, cR));
    double dL = line_dist(cL, a, b), dR = line_dist(cR, a, b);
    g.lam_bar[e] = dL / (dL + dR);
    double orth = std::fabs(dot(sub(cL, cR), sub(b, a))) / (g.wbar_len[e] * g.ebar_len[e]);
    BB_REQUIRE(g.wbar_len[e] > 1e-12 && orth <= 1e-10, BBOT_E_GEOMETRY,
               "coarse mesh not TPFA-admissible at edge " + std::to_string(e));
  }

  // ---- fine kites
  int N = g.N;
  g.c.resize(N);
  g.xx.resize(N);
  g.xy.resize(N);
  for (int t = 0; t < nt; t++) {
    P2 P[3] = {V(tris[3 * t]), V(tris[3 * t + 1]), V(tris[3 * t + 2])};
    P2 cc{g.ccx[t], g.ccy[t]};
    for (int s = 0; s < 3; s++) {
      P2 v = P[s], m1 = mid(P[s], P[(s + 1) % 3]), m0 = mid(P[(s + 2) % 3], P[s]);
      // kite (v, m1, cc, m0): two triangles sharing the diagonal v-cc
      double ar = 0.5 * (cross(sub(m1, v), sub(cc, v)) + cross(sub(cc, v), sub(m0, v)));
      int f = 3 * t + s;
      g.c[f] = ar;
      g.xx[f] = 0.5 * (v.x + cc.x);
      g.xy[f] = 0.5 * (v.y + cc.y);
    }
  }

  // ---- fine internal edges: type a (3 per triangle), then type b (2 per coarse edge)
  auto add_edge = [&](int f1, int f2, P2 s0, P2 s1, int8_t type) {
    int L = std::min(f1, f2), R = std::max(f1, f2);
    P2 xL{g.xx[L], g.xy[L]}, xR{g.xx[R], g.xy[R]};
    double el = norm(sub(s0, s1)), wl = norm(sub(xL, xR));
    double dL = line_dist(xL, s0, s1), dR = line_dist(xR, s0, s1);
    double orth = std::fabs(dot(sub(xL, xR), sub(s1, s0))) / (wl * el);
    BB_REQUIRE(wl > 1e-12 && el > 0 && orth <= 1e-10, BBOT_E_GEOMETRY,
               "fine mesh not TPFA-admissible");
    g.eL.push_back(L);
    g.eR.push_back(R);
    g.e_len.push_back(el);
    g.w_len.push_back(wl);
    g.lam.push_back(dL / (dL + dR));
    g.etype.push_back(type);
  };
  for (int t = 0; t < nt; t++) {
    P2 P[3] = {V(tris[3 * t]), V(tris[3 * t + 1]), V(tris[3 * t + 2])};
    P2 cc{g.ccx[t], g.ccy[t]};
    for (int s = 0; s < 3; s++)
      add_edge(3 * t + s, 3 * t + (s + 1) % 3, mid(P[s], P[(s + 1) % 3]), cc, 0);
  }
  auto slot_of = [&](int t, int v) {
    for (int s = 0; s < 3; s++)
      if (tris[3 * t + s] == v) return s;
    return -1;
  };
  // at va for every edge, then at vb (same order as a plain enumeration)
  for (int pass = 0; pass < 2; pass++)
    for (int e = 0; e < g.NEbar; e++) {
      int v = pass == 0 ? eva[e] : evb[e];
      int tL = g.ebL[e], tR = g.ebR[e];
      P2 m = mid(V(eva[e]), V(evb[e]));
      add_edge(3 * tL + slot_of(tL, v), 3 * tR + slot_of(tR, v), V(v), m, 1);
    }
  g.NE = (int)g.eL.size();
  BB_REQUIRE(g.NE == 2 * g.NEbar + 3 * g.nbar, BBOT_E_GEOMETRY, "fine edge count (P:110)");

  // ---- fine adjacency [4][N]
  g.fadj_e.assign(4 * (size_t)N, -1);
  g.fadj_nb.assign(4 * (size_t)N, -1);
  std::vector<int> deg(N, 0);
  for (int e = 0; e < g.NE; e++) {
    int L = g.eL[e], R = g.eR[e];
    BB_REQUIRE(deg[L] < 4 && deg[R] < 4, BBOT_E_GEOMETRY, "fine cell with > 4 edges");
    g.fadj_e[(size_t)deg[L] * N + L] = e;
    g.fadj_nb[(size_t)deg[L] * N + L] = R;
    deg[L]++;
    g.fadj_e[(size_t)deg[R] * N + R] = e;
    g.fadj_nb[(size_t)deg[R] * N + R] = L;
    deg[R]++;
  }
  return g;
}

}  // namespace bbot
