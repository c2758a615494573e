// rr_oracle.cpp -- plain, slow, single-threaded fp64 CPU oracle of the residual path integral estimator.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library.  The product path (paper_2406_16302_b200) never
// links, imports or calls it, and the two share no code, headers, tables or constants.
//
// What it computes (paper = /root/reference/PAPER.md, cited as P:Lnnn; SPEC = SPEC.md as S:Lnnn):
//   * the primal path integral I^D(F) of Eq.1-2 with a unidirectional NEE/BSDF-MIS path
//     tracer (an estimator independent of the residual code path), and
//   * the residual estimator of I^D(N) - I^D(O) (Eq.3-5): the seven sampling techniques of
//     Sec.4, balance-heuristic MIS over N_D+N_G+1 candidates evaluated from
//     explicit per-path pdf products (the "two tables" of P:L356 written out directly), the path mapping
//     of Sec.5 (random-seed replay P:L414-416, object transform P:L381-385, dynamic<->ghost pair
//     P:L418-420, keep-vertex reconnection with the Jacobian of P:L397-401 and criteria P:L403-411),
//     rejection and two-way mapping;
//   * optionally (flags bit 32) GGX directions from the visible-normal distribution (Heitz 2018), one of
//     the variance-only variants of SURVEY 8(f) row 4.
// Where the paper is silent the reading of SURVEY.md 8(c) (C1-C12) is followed; DESIGN.md lists them.
//
// Every quantity is computed in double precision from the fp32 scene arrays.  The only fp32 data are
// the triangle-selection CDF tables (rounded to fp32 by the recipe of SURVEY 8(c) C3 so that both
// implementations take the same discrete decision) and the u01 variates, which are exact in fp32.
//
// Parity pins live in tests/test_oracle_*.py (closed forms, brute force, furnace, identity edit,
// albedo scale, convergence against the independent primal renderer, {l,7}-mask agreement).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

// ------------------------------------------------------------------------------------------------
// fp64 vector helpers
// ------------------------------------------------------------------------------------------------
struct V3 {
  double x, y, z;
};
inline V3 v3(double x, double y, double z) { return V3{x, y, z}; }
inline V3 operator+(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
inline V3 operator-(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
inline V3 operator*(V3 a, double s) { return v3(a.x * s, a.y * s, a.z * s); }
inline V3 operator*(double s, V3 a) { return v3(a.x * s, a.y * s, a.z * s); }
inline V3 mul(V3 a, V3 b) { return v3(a.x * b.x, a.y * b.y, a.z * b.z); }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x); }
inline double len(V3 a) { return std::sqrt(dot(a, a)); }
inline V3 normalize(V3 a) { return a * (1.0 / len(a)); }
inline bool same(V3 a, V3 b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
inline bool nonzero(V3 a) { return a.x != 0.0 || a.y != 0.0 || a.z != 0.0; }
const double PI = 3.14159265358979323846;

// ------------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon, Moraes, Dror, Shaw 2011, "Parallel random numbers: as easy as 1, 2, 3")
// Counter layout: ctr = (i lo, i hi, l | side<<8, 2*slot + call), key = seed.
// ------------------------------------------------------------------------------------------------
void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// u01(x) = (x >> 8) * 2^-24: exact in fp32 and fp64, in [0, 1).
inline double u01(uint32_t x) { return (double)(x >> 8) * (1.0 / 16777216.0); }

struct Stream {  // one residual sample's random numbers: technique l, side s, sample index i
  uint64_t seed, i;
  uint32_t l, side;
  // 8 dims of slot `slot`
  void dims(uint32_t slot, double d[8]) const {
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    for (uint32_t call = 0; call < 2; ++call) {
      uint32_t ctr[4] = {(uint32_t)(i & 0xffffffffu), (uint32_t)(i >> 32), l | (side << 8), 2u * slot + call};
      uint32_t o[4];
      philox4x32_10(ctr, key, o);
      for (int k = 0; k < 4; ++k) d[4 * call + k] = u01(o[k]);
    }
  }
};

// ------------------------------------------------------------------------------------------------
// Scene, states, placements
// ------------------------------------------------------------------------------------------------
enum { MAT_LAMBERT = 0, MAT_GGX = 1 };
struct Mat {
  int type;
  V3 albedo;
  double alpha;
  bool vndf = false;  // GGX directions sampled from the visible normals of wi (RR_VNDF)
};
struct Tri {
  V3 v0, v1, v2;
  V3 n;  // wound geometric normal (world)
  int id;
  int obj;
};

struct AABB {
  V3 lo, hi;
  void reset() {
    lo = v3(1e300, 1e300, 1e300);
    hi = v3(-1e300, -1e300, -1e300);
  }
  void grow(V3 p) {
    lo = v3(std::min(lo.x, p.x), std::min(lo.y, p.y), std::min(lo.z, p.z));
    hi = v3(std::max(hi.x, p.x), std::max(hi.y, p.y), std::max(hi.z, p.z));
  }
};

// Plain median-split BVH over triangles in world space (fp64).
struct BVH {
  struct Node {
    AABB box;
    int left = -1, right = -1, first = 0, count = 0;
  };
  std::vector<Tri> tris;
  std::vector<int> order;
  std::vector<Node> nodes;

  void build(std::vector<Tri> t) {
    tris = std::move(t);
    order.resize(tris.size());
    for (size_t k = 0; k < order.size(); ++k) order[k] = (int)k;
    nodes.clear();
    if (!tris.empty()) build_rec(0, (int)tris.size());
  }
  V3 centroid(int k) const { return (tris[k].v0 + tris[k].v1 + tris[k].v2) * (1.0 / 3.0); }
  int build_rec(int lo, int hi) {
    int id = (int)nodes.size();
    nodes.push_back(Node());
    AABB b, cb;
    b.reset();
    cb.reset();
    for (int k = lo; k < hi; ++k) {
      const Tri& t = tris[order[k]];
      b.grow(t.v0); b.grow(t.v1); b.grow(t.v2);
      cb.grow(centroid(order[k]));
    }
    nodes[id].box = b;
    if (hi - lo <= 4) {
      nodes[id].first = lo;
      nodes[id].count = hi - lo;
      return id;
    }
    V3 ext = cb.hi - cb.lo;
    int axis = (ext.x >= ext.y && ext.x >= ext.z) ? 0 : (ext.y >= ext.z ? 1 : 2);
    int mid = (lo + hi) / 2;
    std::nth_element(order.begin() + lo, order.begin() + mid, order.begin() + hi, [&](int a, int c) {
      V3 ca = centroid(a), cc = centroid(c);
      double va = axis == 0 ? ca.x : (axis == 1 ? ca.y : ca.z);
      double vc = axis == 0 ? cc.x : (axis == 1 ? cc.y : cc.z);
      return va < vc;
    });
    int l = build_rec(lo, mid);
    int r = build_rec(mid, hi);
    nodes[id].left = l;
    nodes[id].right = r;
    return id;
  }
  static bool box_hit(const AABB& b, V3 o, V3 inv, double tmin, double tmax) {
    double t0 = (b.lo.x - o.x) * inv.x, t1 = (b.hi.x - o.x) * inv.x;
    if (t0 > t1) std::swap(t0, t1);
    tmin = std::max(tmin, t0); tmax = std::min(tmax, t1);
    t0 = (b.lo.y - o.y) * inv.y; t1 = (b.hi.y - o.y) * inv.y;
    if (t0 > t1) std::swap(t0, t1);
    tmin = std::max(tmin, t0); tmax = std::min(tmax, t1);
    t0 = (b.lo.z - o.z) * inv.z; t1 = (b.hi.z - o.z) * inv.z;
    if (t0 > t1) std::swap(t0, t1);
    tmin = std::max(tmin, t0); tmax = std::min(tmax, t1);
    return tmin <= tmax * (1.0 + 1e-12) + 1e-300;
  }
  // Moeller-Trumbore ray/triangle; returns t or -1.
  static double tri_hit(const Tri& t, V3 o, V3 d) {
    V3 e1 = t.v1 - t.v0, e2 = t.v2 - t.v0;
    V3 p = cross(d, e2);
    double det = dot(e1, p);
    if (det == 0.0) return -1.0;
    double inv = 1.0 / det;
    V3 s = o - t.v0;
    double u = dot(s, p) * inv;
    if (u < 0.0 || u > 1.0) return -1.0;
    V3 q = cross(s, e1);
    double v = dot(d, q) * inv;
    if (v < 0.0 || u + v > 1.0) return -1.0;
    return dot(e2, q) * inv;
  }
  // visit every triangle whose t is in (tmin, tmax); f(tri index, t) returns the new tmax
  template <class F>
  void traverse(V3 o, V3 d, double tmin, double tmax, F f) const {
    if (nodes.empty()) return;
    V3 inv = v3(1.0 / d.x, 1.0 / d.y, 1.0 / d.z);
    int stack[256];
    int sp = 0;
    stack[sp++] = 0;
    while (sp) {
      const Node& n = nodes[stack[--sp]];
      if (!box_hit(n.box, o, inv, tmin, tmax)) continue;
      if (n.count) {
        for (int k = n.first; k < n.first + n.count; ++k) {
          double t = tri_hit(tris[order[k]], o, d);
          if (t > tmin && t < tmax) tmax = f(order[k], t, tmax);
        }
      } else {
        stack[sp++] = n.left;
        stack[sp++] = n.right;
      }
    }
  }
};

struct Hit {
  bool ok = false;
  double t = 0;
  const Tri* tri = nullptr;
};

struct Crossing {
  V3 p, n;
  double t;
};

struct Scene {
  // inputs
  std::vector<V3> pos;
  std::vector<int> idx;
  std::vector<int> tri_obj;
  std::vector<int> obj_mat;
  std::vector<V3> obj_emit;
  std::vector<uint32_t> obj_flags;
  std::vector<Mat> mats;
  V3 cam_pos, cam_look, cam_up;
  double vfov;
  int W, H;
  double eps_rel;
  // edits
  std::vector<int> edited;          // object id -> 1 if in the edited (dynamic) set
  std::vector<int> moved;           // object id -> 1 if old/new transforms differ bitwise
  std::vector<double> xf[2];        // per object 12 doubles per state (F=0: new, F=1: old)
  std::vector<int> has_mat;
  std::vector<Mat> emat[2];
  bool vndf = false;                // render option RR_VNDF (flags bit 32) of the current residual call
  bool t6_light = false;            // render option RR_T6_TOWARD_LIGHT (flags bit 512)
  std::vector<V3> emit_centroid;    // area-weighted centroid of each emitter object (world)
  // derived
  double diag, eps;
  V3 cf, cr, cu;  // camera basis
  double tanX, tanY, Aplane;
  BVH bvh_static;
  BVH bvh_dyn[2];  // edited objects placed at M_F
  std::vector<Tri> tri_world[2];  // per state, every triangle placed (static ones identical)
  // sampling tables: fp32 CDFs as data
  struct TriSet {
    std::vector<int> tris;
    std::vector<float> cdf;
    double area = 0;
  };
  TriSet edited_set, moved_set;
  std::vector<TriSet> emitters;
  std::vector<int> emitter_index;  // object -> emitter index or -1
};

inline V3 xform_point(const double* m, V3 p) {
  return v3(m[0] * p.x + m[1] * p.y + m[2] * p.z + m[3], m[4] * p.x + m[5] * p.y + m[6] * p.z + m[7],
            m[8] * p.x + m[9] * p.y + m[10] * p.z + m[11]);
}

// world-space triangle of tri k placed in state F
Tri make_tri(const Scene& S, int k, int F) {
  int o = S.tri_obj[k];
  V3 a = S.pos[S.idx[3 * k]], b = S.pos[S.idx[3 * k + 1]], c = S.pos[S.idx[3 * k + 2]];
  if (S.edited[o]) {
    const double* m = &S.xf[F][12 * o];
    a = xform_point(m, a); b = xform_point(m, b); c = xform_point(m, c);
  }
  Tri t;
  t.v0 = a; t.v1 = b; t.v2 = c;
  t.n = normalize(cross(b - a, c - a));
  t.id = k;
  t.obj = o;
  return t;
}

double tri_area_object_space(const Scene& S, int k) {
  V3 a = S.pos[S.idx[3 * k]], b = S.pos[S.idx[3 * k + 1]], c = S.pos[S.idx[3 * k + 2]];
  return 0.5 * len(cross(b - a, c - a));
}

void build_set(const Scene& S, Scene::TriSet& ts) {
  // fp64 prefix sum in triangle order, divided by the total, rounded to fp32
  double total = 0;
  std::vector<double> pre(ts.tris.size());
  for (size_t k = 0; k < ts.tris.size(); ++k) {
    total += tri_area_object_space(S, ts.tris[k]);
    pre[k] = total;
  }
  ts.area = total;
  ts.cdf.resize(ts.tris.size());
  for (size_t k = 0; k < ts.tris.size(); ++k) ts.cdf[k] = (float)(pre[k] / total);
  if (!ts.cdf.empty()) ts.cdf.back() = 1.0f;
}

Mat mat_of(const Scene& S, int obj, int F) {
  Mat m = (S.edited[obj] && S.has_mat[obj]) ? S.emat[F][obj] : S.mats[S.obj_mat[obj]];
  m.vndf = S.vndf && m.type == MAT_GGX;
  return m;
}

// ------------------------------------------------------------------------------------------------
// ray queries in View_F = static BLAS + edited objects at M_F (ghosts transparent)
// ------------------------------------------------------------------------------------------------
struct Counters {
  uint64_t closest = 0, shadow = 0;
};

Hit closest(const Scene& S, int F, V3 o, V3 d, int excl, Counters* C) {
  if (C) C->closest++;
  Hit h;
  double best = 1e300;
  auto visit = [&](const BVH& b) {
    b.traverse(o, d, S.eps, best, [&](int k, double t, double tmax) {
      if (b.tris[k].id == excl) return tmax;
      if (t < best) {
        best = t;
        h.ok = true;
        h.t = t;
        h.tri = &b.tris[k];
      }
      return best;
    });
  };
  visit(S.bvh_static);
  visit(S.bvh_dyn[F]);
  return h;
}

// segment (a,b): visible iff no triangle of View_F in (eps, len - eps), endpoint prims excluded
bool visible(const Scene& S, int F, V3 a, V3 b, int excl_a, int excl_b, Counters* C) {
  if (C) C->shadow++;
  V3 dv = b - a;
  double L = len(dv);
  if (!(L > 2.0 * S.eps)) return false;
  V3 d = dv * (1.0 / L);
  bool blocked = false;
  auto visit = [&](const BVH& bv) {
    if (blocked) return;
    bv.traverse(a, d, S.eps, L - S.eps, [&](int k, double, double tmax) {
      int id = bv.tris[k].id;
      if (id == excl_a || id == excl_b) return tmax;
      blocked = true;
      return -1.0;  // terminate
    });
  };
  visit(S.bvh_static);
  visit(S.bvh_dyn[F]);
  return !blocked;
}

// The ghost point x_G a T4 / T5 / T6 sample passed its edge through (reading 12): the edge crosses
// the ghost there by construction, so that crossing is a candidate whether or not a ray query finds it.
struct SeedCrossing {
  int edge = -1;  // path edge (i, i+1) through x_G; -1: none
  V3 p, n;        // x_G and the ghost's normal there
  int tri = -1;   // the ghost triangle x_G was sampled on
};

// ghost crossings of segment (a,b) in state F: hits of moved objects placed at M_Fbar in
// (eps, len - eps), sorted by t, hits within 1e-6 diag merged.  seed: a crossing known to
// lie on the segment (x_G of the sample that produced it); a hit within the merge distance of it is the
// same crossing, and so is a hit of the seed's own triangle (a segment crosses a plane once).
std::vector<Crossing> crossings(const Scene& S, int F, V3 a, V3 b, const SeedCrossing* seed = nullptr) {
  std::vector<Crossing> out;
  V3 dv = b - a;
  double L = len(dv);
  if (!(L > 2.0 * S.eps)) return out;
  V3 d = dv * (1.0 / L);
  const BVH& g = S.bvh_dyn[1 - F];
  std::vector<std::pair<double, const Tri*>> hits;
  g.traverse(a, d, S.eps, L - S.eps, [&](int k, double t, double tmax) {
    if (S.moved[g.tris[k].obj]) hits.push_back({t, &g.tris[k]});
    return tmax;
  });
  std::sort(hits.begin(), hits.end(), [](const std::pair<double, const Tri*>& x,
                                         const std::pair<double, const Tri*>& y) { return x.first < y.first; });
  double tol = 1e-6 * S.diag;
  double ts = seed ? dot(seed->p - a, d) : 0.0;
  bool seeded = false;
  auto put_seed = [&]() {
    Crossing c;
    c.t = ts;
    c.p = seed->p;
    c.n = seed->n;
    out.push_back(c);
    seeded = true;
  };
  for (auto& h : hits) {
    if (seed && (std::fabs(h.first - ts) < tol || h.second->id == seed->tri)) continue;  // the known crossing itself
    if (seed && !seeded && h.first > ts) put_seed();
    if (!out.empty() && h.first - out.back().t < tol) continue;
    Crossing c;
    c.t = h.first;
    c.p = a + d * h.first;
    c.n = h.second->n;
    out.push_back(c);
  }
  if (seed && !seeded) put_seed();
  return out;
}

// ------------------------------------------------------------------------------------------------
// camera: pinhole, A_plane = 4 tanX tanY, W_e = 1/(A cos^4), p(x_E) := 1
// ------------------------------------------------------------------------------------------------
V3 camera_dir(const Scene& S, double sx, double sy) {
  return normalize(S.cf + S.cr * ((2.0 * sx / S.W - 1.0) * S.tanX) + S.cu * ((1.0 - 2.0 * sy / S.H) * S.tanY));
}
// returns pixel index or -1
int project(const Scene& S, V3 x) {
  V3 q = x - S.cam_pos;
  double c = dot(q, S.cf);
  if (!(c > 0)) return -1;
  double sx = (dot(q, S.cr) / (c * S.tanX) + 1.0) * S.W * 0.5;
  double sy = (1.0 - dot(q, S.cu) / (c * S.tanY)) * S.H * 0.5;
  double fx = std::floor(sx), fy = std::floor(sy);
  if (fx < 0 || fy < 0 || fx >= S.W || fy >= S.H) return -1;
  return (int)fy * S.W + (int)fx;
}

// ------------------------------------------------------------------------------------------------
// BSDFs: two-sided, reflection-only; wi points toward the previous vertex
// ------------------------------------------------------------------------------------------------
void onb(V3 n, V3& b1, V3& b2) {  // Duff et al. 2017
  double sign = std::copysign(1.0, n.z);
  double a = -1.0 / (sign + n.z);
  double b = n.x * n.y * a;
  b1 = v3(1.0 + sign * n.x * n.x * a, sign * b, -sign * n.x);
  b2 = v3(b, sign + n.y * n.y * a, -n.y);
}
V3 local_to_world(V3 n, double x, double y, double z) {
  V3 b1, b2;
  onb(n, b1, b2);
  return b1 * x + b2 * y + n * z;
}
double ggx_D(double a, double nh) {
  double a2 = a * a;
  double t = nh * nh * (a2 - 1.0) + 1.0;
  return a2 / (PI * t * t);
}
double ggx_G1(double a, double nv) {
  nv = std::fabs(nv);
  return 2.0 * nv / (nv + std::sqrt(a * a + (1.0 - a * a) * nv * nv));
}
V3 bsdf_eval(const Mat& m, V3 n, V3 wi, V3 wo) {
  V3 ns = dot(n, wi) > 0 ? n : n * -1.0;
  double ci = dot(ns, wi), co = dot(ns, wo);
  if (!(ci > 0) || !(co > 0)) return v3(0, 0, 0);
  if (m.type == MAT_LAMBERT) return m.albedo * (1.0 / PI);
  V3 h = normalize(wi + wo);
  double nh = dot(ns, h);
  double D = ggx_D(m.alpha, nh);
  double G = ggx_G1(m.alpha, ci) * ggx_G1(m.alpha, co);
  double fw = std::pow(1.0 - std::fabs(dot(wi, h)), 5.0);
  V3 F = m.albedo + (v3(1, 1, 1) - m.albedo) * fw;
  return F * (D * G / (4.0 * ci * co));
}
double bsdf_pdf(const Mat& m, V3 n, V3 wi, V3 wo) {
  V3 ns = dot(n, wi) > 0 ? n : n * -1.0;
  double ci = dot(ns, wi), co = dot(ns, wo);
  if (!(ci > 0) || !(co > 0)) return 0.0;
  if (m.type == MAT_LAMBERT) return co / PI;
  V3 h = normalize(wi + wo);
  double nh = dot(ns, h);
  // VNDF (Heitz 2018): h has density D_wi(h) = G1(wi) max(0, wi.h) D(h) / (n.wi); with the reflection
  // Jacobian 1 / (4 wo.h) and wo.h = wi.h this is G1(wi) D(h) / (4 n.wi)
  if (m.vndf) return ggx_G1(m.alpha, ci) * ggx_D(m.alpha, nh) / (4.0 * ci);
  return ggx_D(m.alpha, nh) * std::fabs(nh) / (4.0 * std::fabs(dot(wo, h)));
}
// Visible-normal sample of the GGX distribution (Heitz 2018, "Sampling the GGX distribution of visible
// normals", Listing 1), isotropic alpha, in the frame (b1, b2, ns) of local_to_world:
//   1. stretch wi: Vh = normalize(a wi_x, a wi_y, wi_z);
//   2. basis T1 = normalize(-Vh_y, Vh_x, 0) (e_x if Vh = e_z), T2 = Vh x T1;
//   3. disk point (r cos phi, r sin phi), r = sqrt(u1), phi = 2 pi u2, its second coordinate warped to the
//      projected hemisphere: t2 = (1 - s) sqrt(1 - t1^2) + s t2 with s = (1 + Vh_z) / 2;
//   4. Nh = t1 T1 + t2 T2 + sqrt(max(0, 1 - t1^2 - t2^2)) Vh;
//   5. unstretch: h = normalize(a Nh_x, a Nh_y, max(0, Nh_z)).
V3 ggx_vndf_half(double a, V3 ns, V3 wi, double u1, double u2) {
  V3 b1, b2;
  onb(ns, b1, b2);
  V3 vh = normalize(v3(a * dot(wi, b1), a * dot(wi, b2), dot(wi, ns)));
  double lensq = vh.x * vh.x + vh.y * vh.y;
  V3 t1v = lensq > 0 ? v3(-vh.y, vh.x, 0.0) * (1.0 / std::sqrt(lensq)) : v3(1.0, 0.0, 0.0);
  V3 t2v = cross(vh, t1v);
  double r = std::sqrt(u1), phi = 2.0 * PI * u2;
  double t1 = r * std::cos(phi), t2 = r * std::sin(phi);
  double sw = 0.5 * (1.0 + vh.z);
  t2 = (1.0 - sw) * std::sqrt(1.0 - t1 * t1) + sw * t2;
  V3 nh = t1v * t1 + t2v * t2 + vh * std::sqrt(std::max(0.0, 1.0 - t1 * t1 - t2 * t2));
  V3 hl = normalize(v3(a * nh.x, a * nh.y, std::max(0.0, nh.z)));
  return local_to_world(ns, hl.x, hl.y, hl.z);
}
bool bsdf_sample(const Mat& m, V3 n, V3 wi, double u1, double u2, V3& wo) {
  V3 ns = dot(n, wi) > 0 ? n : n * -1.0;
  if (m.type == MAT_LAMBERT) {
    double r = std::sqrt(u1), phi = 2.0 * PI * u2;
    wo = normalize(local_to_world(ns, r * std::cos(phi), r * std::sin(phi), std::sqrt(std::max(0.0, 1.0 - u1))));
    return true;
  }
  double a = m.alpha;
  if (m.vndf) {
    V3 h = normalize(ggx_vndf_half(a, ns, wi, u1, u2));
    wo = h * (2.0 * dot(wi, h)) - wi;
    if (!(dot(wo, ns) > 0)) return false;
    wo = normalize(wo);
    return true;
  }
  double tan2 = a * a * u1 / (1.0 - u1);
  double ct = 1.0 / std::sqrt(1.0 + tan2);
  double st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
  double phi = 2.0 * PI * u2;
  V3 h = normalize(local_to_world(ns, st * std::cos(phi), st * std::sin(phi), ct));
  wo = h * (2.0 * dot(wi, h)) - wi;
  if (!(dot(wo, ns) > 0)) return false;
  wo = normalize(wo);
  return true;
}
double roughness(const Mat& m) { return m.type == MAT_LAMBERT ? 1e300 : m.alpha; }

// ------------------------------------------------------------------------------------------------
// path vertices and explicit paths
// ------------------------------------------------------------------------------------------------
enum { K_CAM = 0, K_SURF = 1, K_LIGHT = 2 };
struct Vtx {
  V3 p, n;
  int tri = -1, obj = -1;
  int kind = K_SURF;
};
// Two vertices of the base and mapped paths coincide iff they are the same primitive of the same hit
// instance at the same point.  A vertex on a MOVED object lies on a different instance in each state
// (dyn at M_F vs dyn at M_Fbar), so it never coincides (SURVEY 8(c) C7 "hit divergence").
bool same_vtx_moved(const std::vector<int>& moved, const Vtx& a, const Vtx& b) {
  if (a.obj >= 0 && moved[a.obj]) return false;
  return a.tri == b.tri && a.kind == b.kind && same(a.p, b.p) && same(a.n, b.n);
}
Vtx vtx_of_hit(V3 o, V3 d, const Hit& h) {
  Vtx v;
  v.p = o + d * h.t;
  v.n = h.tri->n;
  v.tri = h.tri->id;
  v.obj = h.tri->obj;
  v.kind = K_SURF;
  return v;
}
Vtx cam_vtx(const Scene& S) {
  Vtx v;
  v.p = S.cam_pos;
  v.n = S.cf;
  v.kind = K_CAM;
  return v;
}

// sample a point on a triangle set: first k with cdf[k] > u; su = sqrt(u1)
Vtx sample_set(const Scene& S, const Scene::TriSet& ts, int F, double u0, double u1, double u2) {
  int n = (int)ts.cdf.size();
  int k = (int)(std::upper_bound(ts.cdf.begin(), ts.cdf.end(), (float)u0) - ts.cdf.begin());
  if (k >= n) k = n - 1;
  int tri = ts.tris[k];
  Tri t = make_tri(S, tri, F);
  double su = std::sqrt(u1);
  double b0 = 1.0 - su, b1 = u2 * su;
  Vtx v;
  int o = S.tri_obj[tri];
  V3 a = S.pos[S.idx[3 * tri]], b = S.pos[S.idx[3 * tri + 1]], c = S.pos[S.idx[3 * tri + 2]];
  V3 x = a * b0 + b * b1 + c * (1.0 - b0 - b1);  // object (or world for static) space
  if (S.edited[o]) x = xform_point(&S.xf[F][12 * o], x);
  v.p = x;
  v.n = t.n;
  v.tri = tri;
  v.obj = o;
  v.kind = K_SURF;
  return v;
}
// NEE emitter sample: object o = min(floor(d3 n_obj), n_obj-1), area-uniform within it (C3).
// *pdf (optional): the density the sampler drew x_L with, 1/n_obj * 1/A_o, from its own choice of o.
Vtx sample_emitter(const Scene& S, const double d[8], double* pdf = nullptr) {
  int ne = (int)S.emitters.size();
  int e = std::min((int)std::floor(d[3] * ne), ne - 1);
  Vtx v = sample_set(S, S.emitters[e], 0, d[4], d[5], d[6]);  // emitters never move
  v.kind = K_LIGHT;
  if (pdf) *pdf = (1.0 / ne) * (1.0 / S.emitters[e].area);
  return v;
}
double p_light(const Scene& S, const Vtx& L) {
  int e = S.emitter_index[L.obj];
  return 1.0 / ((double)S.emitters.size() * S.emitters[e].area);
}
V3 emission(const Scene& S, const Vtx& L, V3 toward) {  // front face only
  if (dot(L.n, toward - L.p) > 0) return S.obj_emit[L.obj];
  return v3(0, 0, 0);
}

// ------------------------------------------------------------------------------------------------
// path contribution f_F (Eq.2) and MIS denominator Pi_F
// x_0 = E (camera), x_{k-1} = L (emitter)
// ------------------------------------------------------------------------------------------------
struct Path {
  std::vector<Vtx> x;
  int pixel = -1;
};

struct Cand {
  int tech;
  int elem;  // vertex index or edge index
  int sub;   // crossing index on the edge
};

struct Eval {
  V3 f = v3(0, 0, 0);
  double Pi = 0;
  int n_cand = 0;
  bool walk_edge_blocked = false;
  std::vector<int> edge_vis;
  std::vector<std::vector<Crossing>> cross;
  bool dynamic = false;         // some vertex on an edited object or some edge crossing a ghost
  std::vector<Cand> cands;      // the candidates of Pi, in order, and each one's technique pdf (C5 table)
  std::vector<double> cand_p;
};

double geo(const Vtx& a, const Vtx& b) {  // G = |cos_a||cos_b| / d^2 (n_{x_E} := camera forward)
  V3 d = b.p - a.p;
  double d2 = dot(d, d);
  V3 w = d * (1.0 / std::sqrt(d2));
  return std::fabs(dot(a.n, w)) * std::fabs(dot(b.n, w)) / d2;
}

// area pdf of generating x_to from x_from, given incoming direction toward x_prev (walk order)
double area_pdf(const Scene& S, int F, const Vtx& prev, const Vtx& from, const Vtx& to) {
  Mat m = mat_of(S, from.obj, F);
  V3 wi = normalize(prev.p - from.p);
  V3 d = to.p - from.p;
  double d2 = dot(d, d);
  V3 wo = d * (1.0 / std::sqrt(d2));
  return bsdf_pdf(m, from.n, wi, wo) * std::fabs(dot(to.n, wo)) / d2;
}

double p_cam(const Scene& S, const Vtx& x1) {
  V3 d = x1.p - S.cam_pos;
  double d2 = dot(d, d);
  V3 w = d * (1.0 / std::sqrt(d2));
  double c = dot(w, S.cf);
  if (!(c > 0)) return 0.0;
  return std::fabs(dot(x1.n, w)) / (S.Aplane * c * c * c * d2);
}

// Candidate techniques of a path with k vertices:
// T7 always; one per dynamic vertex x_i (i = k-2 -> T1, i = 1 -> T2, else T3); one per ghost
// crossing on edge (i, i+1) (i = 0 -> T5, i+1 = k-1 -> T4, else T6); k = 2 has none besides T7.
std::vector<Cand> enumerate_candidates(int k, const std::vector<int>& dyn, const std::vector<int>& ncross, int mask) {
  std::vector<Cand> c;
  auto on = [&](int l) { return (mask >> (l - 1)) & 1; };
  if (k >= 3) {
    for (int i = 1; i <= k - 2; ++i) {
      if (!dyn[i]) continue;
      int l = (i == k - 2) ? 1 : (i == 1 ? 2 : 3);
      if (on(l)) c.push_back({l, i, 0});
    }
    for (int i = 0; i <= k - 2; ++i) {
      for (int g = 0; g < ncross[i]; ++g) {
        int l = (i == 0) ? 5 : (i + 1 == k - 1 ? 4 : 6);
        if (on(l)) c.push_back({l, i, g});
      }
    }
    // deterministic order: by element index, then technique
    std::stable_sort(c.begin(), c.end(), [](const Cand& a, const Cand& b) {
      return a.elem != b.elem ? a.elem < b.elem : a.tech < b.tech;
    });
  }
  if (on(7)) c.push_back({7, 0, 0});
  return c;
}

struct Ctx {
  const Scene* S;
  int mask;     // effective technique mask
  Counters C;
  std::vector<double>* recon_out = nullptr;  // test export: geometry of accepted reconnections (orc_reconnections)
};

// T6's direction density p_dir(d | x_G) (technique (6) "a direction uniformly toward the light").
// Default (C12 #9): uniform on the sphere, 1/(4 pi).  RR_T6_TOWARD_LIGHT: an emitter object e is chosen
// uniformly and d is uniform on the hemisphere facing its centroid c_e, so the density of d is the mixture
// (1/n_e) sum_e [d . (c_e - x_G) > 0] / (2 pi); +d is the emitter side.
double t6_pdir(const Scene& S, V3 xg, V3 d) {
  if (!S.t6_light) return 1.0 / (4.0 * PI);
  int n = 0;
  for (const V3& c : S.emit_centroid) n += dot(d, c - xg) > 0 ? 1 : 0;
  return (double)n / ((double)S.emit_centroid.size() * 2.0 * PI);
}

Eval eval_path(Ctx& cx, int F, const Path& P, bool check_walk_vis = true, const SeedCrossing* seed = nullptr) {
  const Scene& S = *cx.S;
  Eval ev;
  const std::vector<Vtx>& x = P.x;
  int k = (int)x.size();
  if (k < 2) return ev;
  // ---- visibility of every edge (Eq.2 V) and crossings of every edge
  ev.edge_vis.assign(k - 1, 1);
  ev.cross.resize(k - 1);
  for (int e = 0; e < k - 1; ++e) {
    if (check_walk_vis) ev.edge_vis[e] = visible(S, F, x[e].p, x[e + 1].p, x[e].tri, x[e + 1].tri, &cx.C) ? 1 : 0;
    ev.cross[e] = crossings(S, F, x[e].p, x[e + 1].p, (seed && seed->edge == e) ? seed : nullptr);
  }
  // ---- f (Eq.2)
  V3 f = v3(1, 1, 1);
  {
    V3 d = x[1].p - x[0].p;
    double c = dot(normalize(d), S.cf);
    if (!(c > 0)) return ev;
    double We = 1.0 / (S.Aplane * c * c * c * c);
    f = f * (We * geo(x[0], x[1]));
  }
  for (int i = 1; i <= k - 2; ++i) {
    Mat m = mat_of(S, x[i].obj, F);
    V3 wi = normalize(x[i - 1].p - x[i].p), wo = normalize(x[i + 1].p - x[i].p);
    f = mul(f, bsdf_eval(m, x[i].n, wi, wo)) * geo(x[i], x[i + 1]);
  }
  f = mul(f, emission(S, x[k - 1], x[k - 2].p));
  for (int e = 0; e < k - 1; ++e)
    if (!ev.edge_vis[e]) f = v3(0, 0, 0);
  ev.f = f;
  // ---- per-vertex forward / reverse area pdfs; fwd[1] = camera, rev up to k-3
  std::vector<double> fwd(k, 0.0), rev(k, 0.0);
  fwd[1] = p_cam(S, x[1]);
  for (int m = 2; m <= k - 2; ++m) fwd[m] = area_pdf(S, F, x[m - 2], x[m - 1], x[m]);
  for (int m = 1; m <= k - 3; ++m) rev[m] = area_pdf(S, F, x[m + 2], x[m + 1], x[m]);
  double pL = (k >= 3) ? p_light(S, x[k - 1]) : 0.0;
  // ---- candidates
  std::vector<int> dyn(k, 0), nc(k - 1, 0);
  for (int i = 1; i <= k - 2; ++i) dyn[i] = (x[i].kind == K_SURF && S.edited[x[i].obj]) ? 1 : 0;
  for (int e = 0; e < k - 1; ++e) nc[e] = (int)ev.cross[e].size();
  for (int i = 0; i < k; ++i) ev.dynamic = ev.dynamic || dyn[i] || (i < k - 1 && nc[i] > 0);
  std::vector<Cand> cands = enumerate_candidates(k, dyn, nc, cx.mask);
  ev.n_cand = (int)cands.size();
  double pA_D = S.edited_set.area > 0 ? 1.0 / S.edited_set.area : 0.0;
  double pA_G = S.moved_set.area > 0 ? 1.0 / S.moved_set.area : 0.0;
  double Pi = 0;
  for (const Cand& c : cands) {
    double p = 1.0;
    switch (c.tech) {
      case 7:  // p_cam(x_1) prod_{m=2}^{k-2} fwd_m p_L  (k = 2: p_cam)
        p = fwd[1];
        for (int m = 2; m <= k - 2; ++m) p *= fwd[m];
        if (k >= 3) p *= pL;
        break;
      case 1:  // p_L p_A(x_{k-2}) prod_{m=1}^{k-3} rev_m
        p = pL * pA_D;
        for (int m = 1; m <= k - 3; ++m) p *= rev[m];
        break;
      case 2:  // p_A(x_1) prod_{m=2}^{k-2} fwd_m p_L   (p(x_E) = 1)
        p = pA_D;
        for (int m = 2; m <= k - 2; ++m) p *= fwd[m];
        p *= pL;
        break;
      case 3: {  // prod_{m<i} rev_m p_A(x_i) p_cos(x_{i+1}|x_i) prod_{m>=i+2} fwd_m p_L
        int i = c.elem;
        for (int m = 1; m <= i - 1; ++m) p *= rev[m];
        p *= pA_D;
        V3 d = x[i + 1].p - x[i].p;
        double d2 = dot(d, d);
        V3 w = d * (1.0 / std::sqrt(d2));
        p *= std::max(0.0, dot(x[i].n, w)) / PI * std::fabs(dot(x[i + 1].n, w)) / d2;
        for (int m = i + 2; m <= k - 2; ++m) p *= fwd[m];
        p *= pL;
        break;
      }
      case 4: {  // p_L p_{G->x_{k-2}}(x_L) prod_{m=1}^{k-3} rev_m   (Eq. vertex1pdf)
        const Crossing& g = ev.cross[c.elem][c.sub];
        const Vtx& xl = x[k - 1];
        const Vtx& x1 = x[k - 2];
        V3 w = normalize(x1.p - xl.p);
        V3 dg = g.p - xl.p, d1 = x1.p - xl.p;
        p = pL * pA_G * dot(dg, dg) / std::fabs(dot(g.n, w)) * std::fabs(dot(x1.n, w)) / dot(d1, d1);
        for (int m = 1; m <= k - 3; ++m) p *= rev[m];
        break;
      }
      case 5: {  // p_{G->x_1}(x_E) prod_{m=2}^{k-2} fwd_m p_L
        const Crossing& g = ev.cross[0][c.sub];
        V3 w = normalize(x[1].p - x[0].p);
        V3 dg = g.p - x[0].p, d1 = x[1].p - x[0].p;
        p = pA_G * dot(dg, dg) / std::fabs(dot(g.n, w)) * std::fabs(dot(x[1].n, w)) / dot(d1, d1);
        for (int m = 2; m <= k - 2; ++m) p *= fwd[m];
        p *= pL;
        break;
      }
      case 6: {  // prod_{m<i} rev_m p(x_G) g_{G,x_i,x_{i+1}} prod_{m>=i+2} fwd_m p_L
        int i = c.elem;
        const Crossing& g = ev.cross[i][c.sub];
        for (int m = 1; m <= i - 1; ++m) p *= rev[m];
        V3 d = x[i + 1].p - x[i].p;
        double d2 = dot(d, d);
        V3 w = d * (1.0 / std::sqrt(d2));
        double gg = std::fabs(dot(x[i].n, w)) * std::fabs(dot(x[i + 1].n, w)) / std::fabs(dot(g.n, w)) *
                    t6_pdir(S, g.p, w) / d2;
        p *= pA_G * gg;
        for (int m = i + 2; m <= k - 2; ++m) p *= fwd[m];
        p *= pL;
        break;
      }
    }
    Pi += p;
    ev.cand_p.push_back(p);
  }
  ev.cands = cands;
  ev.Pi = Pi;
  return ev;
}

// ------------------------------------------------------------------------------------------------
// techniques: generate walks; connections are formed afterwards
// ------------------------------------------------------------------------------------------------
struct Walk {
  std::vector<Vtx> v;   // v[0] = predecessor of the first walk vertex (E, x_L, x_D, ...); v[1..] walk
  std::vector<V3> wo;   // wo[m]: direction sampled at v[m] (valid if wo_ok[m])
  std::vector<int> wo_ok;
  // pA[m] (m >= 1): the area density with which the generator produced v[m], recorded at generation time
  // from the sampled direction and hit distance (pdf_w |n.w| / t^2, or the technique's start density).
  // Only the technique-pdf self-consistency pin reads it.
  std::vector<double> pA;
  int n() const { return (int)v.size() - 1; }
};

struct Gen {
  bool ok = false;
  int tech = 0;
  int F = 0;
  int pixel = -1;       // T7 / T2 / T5 fixed pixel
  Vtx start;            // x_D / x_G (x_G is not a vertex)
  Vtx xL;               // T1 / T4 emitter vertex
  Walk A;               // single walk; sensor-side walk for T3/T6
  Walk B;               // emitter-side walk for T3/T6
  bool emit_direct = false;  // T7: x_1 reached (k = 2 candidate)
  double pdf0 = 1.0;    // recorded density of the start event not held in A.pA / B.pA (x_L; T3 x_D; T6 (x_G, d))
};

// continue a walk from v[n] using slots slot0 + m for walk vertex m, until `nmax` walk vertices
void extend_walk(Ctx& cx, int F, const Stream& st, Walk& w, int slot0, int nmax) {
  const Scene& S = *cx.S;
  while (w.n() < nmax) {
    int m = w.n();
    const Vtx& cur = w.v[m];
    double d[8];
    st.dims((uint32_t)(slot0 + m), d);
    Mat mt = mat_of(S, cur.obj, F);
    V3 wi = normalize(w.v[m - 1].p - cur.p);
    V3 wo;
    bool ok = bsdf_sample(mt, cur.n, wi, d[1], d[2], wo);
    w.wo.resize(m + 1);
    w.wo_ok.resize(m + 1, 0);
    w.wo[m] = ok ? wo : v3(0, 0, 0);
    w.wo_ok[m] = ok ? 1 : 0;
    if (!ok) break;
    Hit h = closest(S, F, cur.p, wo, cur.tri, &cx.C);
    if (!h.ok) break;
    w.v.push_back(vtx_of_hit(cur.p, wo, h));
    w.pA.resize(w.v.size(), 0.0);
    w.pA[m + 1] = bsdf_pdf(mt, cur.n, wi, wo) * std::fabs(dot(h.tri->n, wo)) / (h.t * h.t);
  }
}

// T3's emitter-side direction at x_D: cosine-weighted about +n as wound (C12 #8); *pdf = the
// density of the sampled local z = sqrt(1 - u3), i.e. cos(theta) / pi
V3 t3_light_dir(V3 n, double u3, double u4, double* pdf) {
  double r = std::sqrt(u3), phi = 2.0 * PI * u4, z = std::sqrt(std::max(0.0, 1.0 - u3));
  *pdf = z / PI;
  return normalize(local_to_world(n, r * std::cos(phi), r * std::sin(phi), z));
}

Gen generate(Ctx& cx, int tech, int F, const Stream& st, int D) {
  const Scene& S = *cx.S;
  Gen g;
  g.tech = tech;
  g.F = F;
  double d0[8];
  st.dims(0, d0);
  Vtx E = cam_vtx(S);
  switch (tech) {
    case 7: {  // PT with static paths rejected: pixel i mod N_pix, jitter d0,d1
      int npix = S.W * S.H;
      int pix = (int)(st.i % (uint64_t)npix);
      g.pixel = pix;
      double sx = (pix % S.W) + d0[0], sy = (pix / S.W) + d0[1];
      V3 dir = camera_dir(S, sx, sy);
      Hit h = closest(S, F, S.cam_pos, dir, -1, &cx.C);
      if (!h.ok) return g;
      g.ok = true;
      g.A.v.push_back(E);
      g.A.v.push_back(vtx_of_hit(S.cam_pos, dir, h));
      {  // film point uniform over the film plane (density 1/A_plane) -> solid angle (/cos^3) -> area
        double c = dot(dir, S.cf);
        g.A.pA = {0.0, (1.0 / S.Aplane) / (c * c * c) * std::fabs(dot(h.tri->n, dir)) / (h.t * h.t)};
      }
      g.emit_direct = true;
      extend_walk(cx, F, st, g.A, 0, D - 1);
      return g;
    }
    case 1: {  // dynamic from emitter
      if (S.edited_set.tris.empty()) return g;
      Vtx xd = sample_set(S, S.edited_set, F, d0[0], d0[1], d0[2]);
      Vtx xl = sample_emitter(S, d0, &g.pdf0);
      if (!(dot(xl.n, xd.p - xl.p) > 0)) return g;          // back-facing emitter
      if (!visible(S, F, xd.p, xl.p, xd.tri, xl.tri, &cx.C)) return g;  // "fails if blocked" P:L286
      g.ok = true;
      g.start = xd;
      g.xL = xl;
      g.A.v.push_back(xl);
      g.A.v.push_back(xd);
      g.A.pA = {0.0, 1.0 / S.edited_set.area};
      extend_walk(cx, F, st, g.A, 0, D - 1);
      return g;
    }
    case 2: {  // dynamic from sensor
      if (S.edited_set.tris.empty()) return g;
      Vtx xd = sample_set(S, S.edited_set, F, d0[0], d0[1], d0[2]);
      int pix = project(S, xd.p);
      if (pix < 0) return g;
      if (!visible(S, F, xd.p, S.cam_pos, xd.tri, -1, &cx.C)) return g;
      g.ok = true;
      g.pixel = pix;
      g.start = xd;
      g.A.v.push_back(E);
      g.A.v.push_back(xd);
      g.A.pA = {0.0, 1.0 / S.edited_set.area};
      extend_walk(cx, F, st, g.A, 0, D - 1);
      return g;
    }
    case 3: {  // dynamic two ends
      if (S.edited_set.tris.empty()) return g;
      Vtx xd = sample_set(S, S.edited_set, F, d0[0], d0[1], d0[2]);
      double pdf_wl;
      V3 wl = t3_light_dir(xd.n, d0[3], d0[4], &pdf_wl);
      Mat mt = mat_of(S, xd.obj, F);
      V3 we;
      if (!bsdf_sample(mt, xd.n, wl, d0[6], d0[7], we)) return g;
      if (D < 4) return g;
      Hit hy = closest(S, F, xd.p, wl, xd.tri, &cx.C);
      if (!hy.ok) return g;
      Hit hz = closest(S, F, xd.p, we, xd.tri, &cx.C);
      if (!hz.ok) return g;
      g.ok = true;
      g.start = xd;
      g.pdf0 = 1.0 / S.edited_set.area;
      g.B.v.push_back(xd);
      g.B.v.push_back(vtx_of_hit(xd.p, wl, hy));
      // cosine density of omega_L, and the BSDF density of omega_E
      g.B.pA = {0.0, pdf_wl * std::fabs(dot(hy.tri->n, wl)) / (hy.t * hy.t)};
      g.A.v.push_back(xd);
      g.A.v.push_back(vtx_of_hit(xd.p, we, hz));
      g.A.pA = {0.0, bsdf_pdf(mt, xd.n, wl, we) * std::fabs(dot(hz.tri->n, we)) / (hz.t * hz.t)};
      extend_walk(cx, F, st, g.B, 16, D - 3);
      extend_walk(cx, F, st, g.A, 0, D - 3);
      return g;
    }
    case 4: {  // ghost from emitter
      if (S.moved_set.tris.empty()) return g;
      Vtx xg = sample_set(S, S.moved_set, 1 - F, d0[0], d0[1], d0[2]);  // ghost_F = moved at M_Fbar
      Vtx xl = sample_emitter(S, d0, &g.pdf0);
      V3 dv = xg.p - xl.p;
      double dl = len(dv);
      if (!(dl > S.eps)) return g;
      V3 dir = dv * (1.0 / dl);
      if (!(dot(xl.n, dir) > 0)) return g;
      Hit h = closest(S, F, xl.p, dir, xl.tri, &cx.C);
      if (!h.ok || !(h.t > dl + S.eps)) return g;
      g.ok = true;
      g.start = xg;
      g.xL = xl;
      g.A.v.push_back(xl);
      g.A.v.push_back(vtx_of_hit(xl.p, dir, h));
      // x_G area-uniform, converted to the solid angle at x_L and then to the area at x_1
      g.A.pA = {0.0, (1.0 / S.moved_set.area) * dl * dl / std::fabs(dot(xg.n, dir)) * std::fabs(dot(h.tri->n, dir)) /
                         (h.t * h.t)};
      extend_walk(cx, F, st, g.A, 0, D - 1);
      return g;
    }
    case 5: {  // ghost from sensor
      if (S.moved_set.tris.empty()) return g;
      Vtx xg = sample_set(S, S.moved_set, 1 - F, d0[0], d0[1], d0[2]);
      int pix = project(S, xg.p);
      if (pix < 0) return g;
      V3 dv = xg.p - S.cam_pos;
      double dg = len(dv);
      V3 dir = dv * (1.0 / dg);
      Hit h = closest(S, F, S.cam_pos, dir, -1, &cx.C);
      if (!h.ok || !(h.t > dg + S.eps)) return g;
      g.ok = true;
      g.pixel = pix;
      g.start = xg;
      g.A.v.push_back(E);
      g.A.v.push_back(vtx_of_hit(S.cam_pos, dir, h));
      g.A.pA = {0.0, (1.0 / S.moved_set.area) * dg * dg / std::fabs(dot(xg.n, dir)) * std::fabs(dot(h.tri->n, dir)) /
                         (h.t * h.t)};
      extend_walk(cx, F, st, g.A, 0, D - 1);
      return g;
    }
    case 6: {  // ghost two ends: full-sphere direction, p_dir = 1/(4 pi)
      if (S.moved_set.tris.empty()) return g;
      Vtx xg = sample_set(S, S.moved_set, 1 - F, d0[0], d0[1], d0[2]);
      V3 dir;
      if (!S.t6_light) {  // uniform sphere: z = 1 - 2 u
        double z = 1.0 - 2.0 * d0[3];
        double rr = std::sqrt(std::max(0.0, 1.0 - z * z)), phi = 2.0 * PI * d0[4];
        dir = v3(rr * std::cos(phi), rr * std::sin(phi), z);
      } else {  // toward the light: emitter e from d5, d uniform on the hemisphere about c_e - x_G (z = u)
        int ne = (int)S.emit_centroid.size();
        int e = std::min((int)std::floor(d0[5] * ne), ne - 1);
        V3 ax = normalize(S.emit_centroid[e] - xg.p);
        double z = d0[3], rr = std::sqrt(std::max(0.0, 1.0 - z * z)), phi = 2.0 * PI * d0[4];
        dir = normalize(local_to_world(ax, rr * std::cos(phi), rr * std::sin(phi), z));
      }
      if (D < 3) return g;
      Hit hy = closest(S, F, xg.p, dir, -1, &cx.C);
      if (!hy.ok) return g;
      Hit hz = closest(S, F, xg.p, dir * -1.0, -1, &cx.C);
      if (!hz.ok) return g;
      g.ok = true;
      g.start = xg;
      // (x_G, d) -> (z_1, y_1): p_A(x_G) p_dir |n_y.d| |n_z.d| / (|n_G.d| |y_1 - z_1|^2), |y_1 - z_1| = t_y + t_z
      g.pdf0 = (1.0 / S.moved_set.area) * t6_pdir(S, xg.p, dir) * std::fabs(dot(hy.tri->n, dir)) *
               std::fabs(dot(hz.tri->n, dir)) / (std::fabs(dot(xg.n, dir)) * (hy.t + hz.t) * (hy.t + hz.t));
      g.A.pA = g.B.pA = {0.0, 1.0};
      Vtx y1 = vtx_of_hit(xg.p, dir, hy), z1 = vtx_of_hit(xg.p, dir * -1.0, hz);
      g.B.v.push_back(z1);
      g.B.v.push_back(y1);
      g.A.v.push_back(y1);
      g.A.v.push_back(z1);
      extend_walk(cx, F, st, g.B, 16, D - 2);
      extend_walk(cx, F, st, g.A, 0, D - 2);
      return g;
    }
  }
  return g;
}

// connection keys: kind 0 = direct emission (T7, k=2), 1 = NEE at walk vertex a, 2 = sensor at a,
// 3 = bidirectional (t = a, s = b) for T3/T6
struct Key {
  int kind, a, b;
  bool operator==(const Key& o) const { return kind == o.kind && a == o.a && b == o.b; }
};

struct Conn {
  Key key;
  Path path;
  int walk_index;   // single-walk techniques: the walk vertex the connection is made from
  double pdf_rec = 0;         // product of the densities the generator recorded for this path (C5 pin)
  int prod_tech = 0, prod_elem = 0;  // the producing candidate: technique and vertex / edge index
};

// The producing ghost crossing of a connection path of a T4 / T5 / T6 sample (none for the other techniques)
SeedCrossing seed_of(const Gen& g, const Conn& c) {
  SeedCrossing sd;
  if (g.tech < 4 || g.tech > 6) return sd;
  int k = (int)c.path.x.size();
  sd.edge = g.tech == 5 ? 0 : (g.tech == 4 ? k - 2 : c.prod_elem);
  sd.p = g.start.p;
  sd.n = g.start.n;
  sd.tri = g.start.tri;
  return sd;
}

// Build every connection path of a generated sample (in its own state)
std::vector<Conn> connections(Ctx& cx, const Gen& g, const Stream& st, int D) {
  const Scene& S = *cx.S;
  std::vector<Conn> out;
  if (!g.ok) return out;
  Vtx E = cam_vtx(S);
  double pL_nee = 0;
  auto nee = [&](int slot) {
    double d[8];
    st.dims((uint32_t)slot, d);
    return sample_emitter(S, d, &pL_nee);
  };
  auto prod = [](const Walk& w, int n) {  // product of the recorded densities of walk vertices 1..n
    double p = 1.0;
    for (int m = 1; m <= n; ++m) p *= w.pA[m];
    return p;
  };
  auto E_rooted = [&](int jmin) {  // T7 / T2 / T5: (E, v_1..v_j, L_j) with NEE slot j
    for (int j = std::max(1, jmin); j <= g.A.n() && j + 1 <= D; ++j) {
      Conn c;
      c.key = {1, j, 0};
      c.walk_index = j;
      c.path.x.push_back(E);
      for (int m = 1; m <= j; ++m) c.path.x.push_back(g.A.v[m]);
      c.path.x.push_back(nee(j));
      c.path.pixel = g.pixel;
      c.pdf_rec = g.pdf0 * prod(g.A, j) * pL_nee;
      c.prod_tech = g.tech;
      c.prod_elem = g.tech == 2 ? 1 : 0;  // T2: x_D = x_1; T5: the crossing on edge (0, 1); T7: -
      out.push_back(c);
    }
  };
  auto L_rooted = [&]() {  // T1 / T4: (E, v_j..v_1, x_L), pixel = projection of v_j
    for (int j = 1; j <= g.A.n() && j + 1 <= D; ++j) {
      Conn c;
      c.key = {2, j, 0};
      c.walk_index = j;
      c.path.x.push_back(E);
      for (int m = j; m >= 1; --m) c.path.x.push_back(g.A.v[m]);
      c.path.x.push_back(g.xL);
      c.path.pixel = project(S, g.A.v[j].p);
      c.pdf_rec = g.pdf0 * prod(g.A, j);
      c.prod_tech = g.tech;
      c.prod_elem = j;  // T1: x_D = x_{k-2}; T4: the crossing on edge (k-2, k-1)
      out.push_back(c);
    }
  };
  switch (g.tech) {
    case 7:
      if (g.emit_direct && D >= 1) {
        Conn c;
        c.key = {0, 1, 0};
        c.walk_index = 1;
        Vtx L = g.A.v[1];
        L.kind = K_LIGHT;
        c.path.x = {E, L};
        c.path.pixel = g.pixel;
        c.pdf_rec = g.pdf0 * g.A.pA[1];
        c.prod_tech = 7;
        // only an emitter reached directly contributes (C12 #4)
        if (S.emitter_index[L.obj] >= 0) out.push_back(c);
      }
      E_rooted(1);
      break;
    case 2:
      E_rooted(2);  // no NEE at x_D: 3-vertex paths belong to T1
      break;
    case 5:
      E_rooted(1);
      break;
    case 1:
    case 4:
      L_rooted();
      break;
    case 3:
    case 6: {
      // T3: (E, z_t..z_1, x_D, y_1..y_s, L_s), t+s+2 <= D; T6: (E, z_t..z_1, y_1..y_s, L_s), t+s+1 <= D
      int extra = g.tech == 3 ? 2 : 1;
      for (int t = 1; t <= g.A.n(); ++t) {
        for (int s = 1; s <= g.B.n(); ++s) {
          if (t + s + extra > D) continue;
          Conn c;
          c.key = {3, t, s};
          c.walk_index = 0;
          c.path.x.push_back(E);
          for (int m = t; m >= 1; --m) c.path.x.push_back(g.A.v[m]);
          if (g.tech == 3) c.path.x.push_back(g.start);
          for (int m = 1; m <= s; ++m) c.path.x.push_back(g.B.v[m]);
          c.path.x.push_back(nee(16 + s));
          c.path.pixel = project(S, g.A.v[t].p);
          c.pdf_rec = g.pdf0 * prod(g.A, t) * prod(g.B, s) * pL_nee;
          c.prod_tech = g.tech;
          c.prod_elem = g.tech == 3 ? t + 1 : t;  // T3: x_D = x_{t+1}; T6: the crossing on edge (t, t+1)
          out.push_back(c);
        }
      }
      break;
    }
  }
  return out;
}

// ------------------------------------------------------------------------------------------------
// residual records and the estimator for one sample
// ------------------------------------------------------------------------------------------------
enum { ST_ACCEPTED = 0, ST_REJECTED = 1, ST_UNPAIRED = 2, ST_MAPPED_ONLY = 3 };
enum { RJ_NONE = 0, RJ_OCCLUDED = 1, RJ_JACOBIAN = 2, RJ_MULTI = 3, RJ_TARGET = 4, RJ_SUFFIX_DYN = 5 };

}  // namespace

extern "C" {

typedef struct {
  int32_t tech, side;
  uint64_t i;
  int32_t key_kind, key_a, key_b;
  int32_t status, reason;
  int32_t pix_p;
  double term_p[3];
  int32_t pix_q;
  double term_q[3];
  double R;
  double v_p[3], v_q[3];
  int32_t n_cand_p, n_cand_q;
} orc_record;

typedef struct {
  uint64_t samples, connections, accepted, rejected, unpaired, mapped_only, reconnected;
  uint64_t closest_rays, shadow_rays, splats, offscreen;
  uint64_t rejected_by[8];
} orc_stats;

typedef struct {
  int32_t n_vertices;
  const float* positions;
  int32_t n_triangles;
  const uint32_t* indices;
  const uint32_t* tri_object;
  int32_t n_objects;
  const uint32_t* obj_material;
  const float* obj_emission;
  const uint32_t* obj_flags;
  int32_t n_materials;
  const uint32_t* mat_type;
  const float* mat_albedo;
  const float* mat_roughness;
  float cam_pos[3], cam_look[3], cam_up[3];
  float vfov_deg;
  int32_t width, height;
  float eps_rel;
  int32_t n_edits;
  const uint32_t* edit_object;
  const float* edit_old_xform;
  const float* edit_new_xform;
  const uint32_t* edit_has_material;
  const uint32_t* edit_mat_type;    // 2 per edit (old, new)
  const float* edit_mat_albedo;     // 6 per edit
  const float* edit_mat_roughness;  // 2 per edit
} orc_input;

typedef struct {
  uint32_t spp;
  uint64_t seed;
  uint32_t max_depth;
  uint32_t technique_mask;
  uint32_t flags;  // 1 TWO_WAY, 2 RECONNECT, 4 REJECT_MULTI, 32 VNDF (GGX visible-normal sampling),
                   // 64 DIAG_ONE_WAY_ABLATION (one-way with the two-way pairing rules; deliberately biased),
                   // 256 NO_PATH_MAPPING (two-way sampling, no mapped paths, static paths rejected),
                   // 512 T6_TOWARD_LIGHT (T6 directions on the hemisphere toward an emitter),
                   // 1024 TOBJ_MIDPATH (object transform of the first mid-path hit on a moved object),
                   // 2048 RECONNECT_BIDIR (reconnection inside the T3 / T6 emitter-side sub-walk)
  double jacobian_max, alpha_min, dmin_rel;
} orc_args;

}  // extern "C"

namespace {

struct Oracle {
  Scene S;
  std::string err;
};

int effective_mask(const Scene& S, uint32_t mask) {
  if (S.moved_set.tris.empty()) mask &= ~(uint32_t)((1 << 3) | (1 << 4) | (1 << 5));  // T4-T6 off
  if (S.edited_set.tris.empty()) mask &= ~(uint32_t)((1 << 0) | (1 << 1) | (1 << 2));
  return (int)mask;
}
bool edited_equals_moved(const Scene& S) {
  for (size_t o = 0; o < S.edited.size(); ++o)
    if (S.edited[o] != S.moved[o]) return false;
  return true;
}
// paired technique l': T2<->T5 only when both are enabled and every edit is a move
int paired_tech(const Scene& S, int mask, int l) {
  bool pair25 = ((mask >> 1) & 1) && ((mask >> 4) & 1) && !S.moved_set.tris.empty() && edited_equals_moved(S);
  if (pair25 && l == 2) return 5;
  if (pair25 && l == 5) return 2;
  return l;
}

// R of a reconnected pair (SURVEY 8(c) C7 "R"): the walk-order area pdfs of the mapped suffix in Fbar over
// those of the base suffix in F, from the reconnection edge v_w -> v_{w+1} to the connection's walk vertex j.
// The mapped walk is q = (v'_0..v'_w, v_{w+1}..v_j): its prefix from `mapped`, its suffix from `base`.
double reconnect_R(const Scene& S, int F, const Walk& base, const Walk& mapped, int w, int j) {
  auto qv = [&](int m) -> const Vtx& { return m <= w ? mapped.v[m] : base.v[m]; };
  auto pv = [&](int m) -> const Vtx& { return base.v[m]; };
  double num = 1.0, den = 1.0;
  for (int m = w + 1; m <= j; ++m) {
    num *= area_pdf(S, 1 - F, qv(m - 2), qv(m - 1), qv(m));
    den *= area_pdf(S, F, pv(m - 2), pv(m - 1), pv(m));
  }
  return num / den;
}

struct SampleOut {
  std::vector<orc_record> recs;
};

// One residual sample (technique l, side s, index i): base in F, mapped in Fbar.
void residual_sample(Ctx& cx, const orc_args& A, int l, int side, uint64_t i, double* img, orc_stats* stats,
                     std::vector<orc_record>* recs) {
  const Scene& S = *cx.S;
  const int D = (int)A.max_depth;
  const int F = side, Fb = 1 - side;  // F = 0: new (N); F = 1: old (O)
  const double sigma = side == 0 ? 1.0 : -1.0;
  // Diagnostic one-way ablation (SURVEY 8(c) C8 last bullet): side N only, N_pix spp samples
  // per technique, reconnection / rejection as in two-way mode, but a rejected or unpaired base path keeps
  // weight 1 and paths of O that no N sample maps to are never counted.  It is the estimator P:L425 warns
  // about ("two-way path mapping to ensure the coverage"): biased by construction, a test mode only.
  const bool diag = (A.flags & 64) != 0 && !(A.flags & 1);
  // "Incremental w/o PM" (Table num_of_dynamics): both frames rendered separately with
  // the dynamic sampling techniques, no path mapping.  Every base connection is unpaired (weight 2 per side) and
  // a path with no dynamic vertex and no ghost crossing in its own state (a static path, equal f and Pi in both
  // states) is rejected outright: those cancel between the two states in expectation.
  const bool nopm = (A.flags & 256) != 0 && (A.flags & 1);
  const bool two_way = A.flags & 1, paired = two_way || diag;
  const bool reconnect = (A.flags & 2) && paired, reject_multi = (A.flags & 4) && paired;
  const double spp = (double)A.spp;
  Stream st{A.seed, i, (uint32_t)l, (uint32_t)side};
  int lq = paired_tech(S, cx.mask, l);

  Gen gp = generate(cx, l, F, st, D);
  Gen gq = nopm ? Gen() : generate(cx, lq, Fb, st, D);  // random-seed replay: same counters
  // ---- "transform with object movement" on a mid-path hit (RR_TOBJ_MIDPATH; reading 18):
  // while the pair has not diverged, the first walk vertex x_m (m >= 2) that the base path finds on a MOVED
  // object is mapped to the same object-space point in the other state, t(x_m) = M_Fbar M_F^-1 x_m (|t'| = 1),
  // instead of replaying the ray; the mapped walk continues by replay from there.  The edge x_{m-1} -> t(x_m)
  // must be unoccluded in View_Fbar, else every connection at walk index >= m is rejected; the connections that
  // use it carry R_T = p_Fbar(t(x_m) | x_{m-1}) / p_F(x_m | x_{m-1}) (walk-order area pdfs).  For the mapping to
  // stay a bijection, a base vertex x_m on static geometry whose REPLAYED partner lies on a moved object rejects
  // the pair from m on (that partner maps by t to another path; replaying would map two paths onto x_m's path).
  const bool single_walk = (l != 3 && l != 6);
  int mT = -1;
  bool tobj_fail = false, tobj_reject = false;
  double RT = 1.0;
  if ((A.flags & 1024) && paired && single_walk && gp.ok && gq.ok) {
    const int na = gp.A.n(), nb = gq.A.n();
    for (int m = 2; m <= na && m - 1 <= nb; ++m) {
      const int a = m - 1;  // the pair must coincide up to x_{m-1} and leave it in the same direction
      if (!same_vtx_moved(S.moved, gp.A.v[a], gq.A.v[a])) break;
      bool pa = a < (int)gp.A.wo_ok.size() && gp.A.wo_ok[a], qa = a < (int)gq.A.wo_ok.size() && gq.A.wo_ok[a];
      if (!pa || !qa || !same(gp.A.wo[a], gq.A.wo[a])) break;
      if (S.moved[gp.A.v[m].obj]) {
        mT = m;
        break;
      }
      if (m <= nb && S.moved[gq.A.v[m].obj]) {  // static base vertex, replayed partner on a moved object
        mT = m;
        tobj_reject = true;
        break;
      }
    }
    if (mT > 0 && !tobj_reject) {
      const Vtx& x = gp.A.v[mT];
      const double* MF = &S.xf[F][12 * x.obj];
      const double* MB = &S.xf[Fb][12 * x.obj];
      // object space: R_F^T (x - t_F); then placed at M_Fbar (rigid transforms, C7)
      V3 d = x.p - v3(MF[3], MF[7], MF[11]);
      V3 po = v3(MF[0] * d.x + MF[4] * d.y + MF[8] * d.z, MF[1] * d.x + MF[5] * d.y + MF[9] * d.z,
                 MF[2] * d.x + MF[6] * d.y + MF[10] * d.z);
      V3 no = v3(MF[0] * x.n.x + MF[4] * x.n.y + MF[8] * x.n.z, MF[1] * x.n.x + MF[5] * x.n.y + MF[9] * x.n.z,
                 MF[2] * x.n.x + MF[6] * x.n.y + MF[10] * x.n.z);
      Vtx t = x;
      t.p = xform_point(MB, po);
      t.n = normalize(v3(MB[0] * no.x + MB[1] * no.y + MB[2] * no.z, MB[4] * no.x + MB[5] * no.y + MB[6] * no.z,
                         MB[8] * no.x + MB[9] * no.y + MB[10] * no.z));
      gq.A.v.resize(mT);
      gq.A.v.push_back(t);
      if ((int)gq.A.wo.size() > mT) { gq.A.wo.resize(mT); gq.A.wo_ok.resize(mT); }
      gq.A.pA.resize(mT + 1, 0.0);
      RT = area_pdf(S, Fb, gq.A.v[mT - 2], gq.A.v[mT - 1], t) / area_pdf(S, F, gp.A.v[mT - 2], gp.A.v[mT - 1], x);
      tobj_fail = !(RT > 0) || !std::isfinite(RT) ||
                  !visible(S, Fb, gq.A.v[mT - 1].p, t.p, gq.A.v[mT - 1].tri, t.tri, &cx.C);
      extend_walk(cx, Fb, st, gq.A, 0, D - 1);  // random-seed replay from t(x_m) on
    }
  }
  std::vector<Conn> cp = connections(cx, gp, st, D);
  std::vector<Conn> cq = connections(cx, gq, st, D);
  if (stats) stats->samples++;

  // ---- divergence and the reconnection index w (single-walk techniques)
  bool single = (l != 3 && l != 6);
  int w = -1;
  bool recon_fail = false;
  int recon_reason = RJ_NONE;
  int nA = gp.ok ? gp.A.n() : 0, nB = gq.ok ? gq.A.n() : 0;
  if (reconnect && single && gp.ok && gq.ok) {
    bool div = false;
    for (int m = 1; m <= std::min(nA, nB); ++m) {
      const Vtx& a = gp.A.v[m];
      const Vtx& b = gq.A.v[m];
      if (!same_vtx_moved(S.moved, a, b)) div = true;
      bool a_ok = m < (int)gp.A.wo_ok.size() && gp.A.wo_ok[m];
      bool b_ok = m < (int)gq.A.wo_ok.size() && gq.A.wo_ok[m];
      bool dir_div = (a_ok != b_ok) || (a_ok && b_ok && !same(gp.A.wo[m], gq.A.wo[m]));
      // diverged at m: a hit divergence at some index <= m or a direction divergence at <= m
      bool d_here = div || dir_div;
      if (d_here && roughness(mat_of(S, a.obj, F)) >= A.alpha_min && roughness(mat_of(S, b.obj, Fb)) >= A.alpha_min) {
        w = m;
        break;
      }
      if (dir_div) div = true;
    }
    if (w > 0 && w + 1 <= nA) {
      const Vtx& vw = gp.A.v[w];
      const Vtx& vq = gq.A.v[w];
      const Vtx& t1 = gp.A.v[w + 1];
      double dmin = A.dmin_rel * S.diag;
      if (S.edited[t1.obj]) { recon_fail = true; recon_reason = RJ_TARGET; }                          // (1) P:L406
      else if (roughness(mat_of(S, t1.obj, F)) < A.alpha_min) { recon_fail = true; recon_reason = RJ_TARGET; }  // (2)
      else if (std::min(len(vw.p - t1.p), len(vq.p - t1.p)) < dmin) { recon_fail = true; recon_reason = RJ_TARGET; }  // (3)
      else if (!visible(S, Fb, vq.p, t1.p, vq.tri, t1.tri, &cx.C)) { recon_fail = true; recon_reason = RJ_OCCLUDED; }
      else {
        // paper Jacobian (Eq. P:L397-401) at the reconnection; symmetric band [1/Jmax, Jmax]
        V3 a = normalize(vq.p - t1.p), b = normalize(vw.p - t1.p);
        double Jg = std::fabs(dot(t1.n, a)) / std::fabs(dot(t1.n, b)) * dot(vw.p - t1.p, vw.p - t1.p) /
                    dot(vq.p - t1.p, vq.p - t1.p);
        if (!(Jg <= A.jacobian_max && Jg >= 1.0 / A.jacobian_max)) { recon_fail = true; recon_reason = RJ_JACOBIAN; }
      }
    }
  }

  // ---- reconnection inside the two-ended techniques' emitter-side sub-walk (RR_RECONNECT_BIDIR, P:L387-411;
  // DESIGN.md reading 19): the single-walk rule applied to walk B (v[0] = x_D for T3, z_1 for T6; v[1..] = y):
  // the first index where the pair is diverged and both vertices are rough reconnects the mapped y'_w to the
  // base's y_{w+1}, with the same target conditions, rejections and R; at most one reconnection per path (the
  // sensor-side walk stays replayed).
  int wB = -1;
  bool reconB_fail = false;
  int reconB_reason = RJ_NONE;
  if (reconnect && !single && (A.flags & 2048) && gp.ok && gq.ok) {
    bool div = false;
    const int na = gp.B.n(), nb = gq.B.n();
    for (int m = 1; m <= std::min(na, nb); ++m) {
      const Vtx& a = gp.B.v[m];
      const Vtx& b = gq.B.v[m];
      if (!same_vtx_moved(S.moved, a, b) || !same_vtx_moved(S.moved, gp.B.v[m - 1], gq.B.v[m - 1])) div = true;
      bool a_ok = m < (int)gp.B.wo_ok.size() && gp.B.wo_ok[m];
      bool b_ok = m < (int)gq.B.wo_ok.size() && gq.B.wo_ok[m];
      bool dir_div = (a_ok != b_ok) || (a_ok && b_ok && !same(gp.B.wo[m], gq.B.wo[m]));
      if ((div || dir_div) && roughness(mat_of(S, a.obj, F)) >= A.alpha_min &&
          roughness(mat_of(S, b.obj, Fb)) >= A.alpha_min) {
        wB = m;
        break;
      }
      if (dir_div) div = true;
    }
    if (wB > 0 && wB + 1 <= na) {
      const Vtx& vw = gp.B.v[wB];
      const Vtx& vq = gq.B.v[wB];
      const Vtx& t1 = gp.B.v[wB + 1];
      double dmin = A.dmin_rel * S.diag;
      if (S.edited[t1.obj]) { reconB_fail = true; reconB_reason = RJ_TARGET; }
      else if (roughness(mat_of(S, t1.obj, F)) < A.alpha_min) { reconB_fail = true; reconB_reason = RJ_TARGET; }
      else if (std::min(len(vw.p - t1.p), len(vq.p - t1.p)) < dmin) { reconB_fail = true; reconB_reason = RJ_TARGET; }
      else if (!visible(S, Fb, vq.p, t1.p, vq.tri, t1.tri, &cx.C)) { reconB_fail = true; reconB_reason = RJ_OCCLUDED; }
      else {
        V3 a = normalize(vq.p - t1.p), b = normalize(vw.p - t1.p);
        double Jg = std::fabs(dot(t1.n, a)) / std::fabs(dot(t1.n, b)) * dot(vw.p - t1.p, vw.p - t1.p) /
                    dot(vq.p - t1.p, vq.p - t1.p);
        if (!(Jg <= A.jacobian_max && Jg >= 1.0 / A.jacobian_max)) { reconB_fail = true; reconB_reason = RJ_JACOBIAN; }
      }
    }
  }

  auto find_q = [&](const Key& k) -> const Conn* {
    for (const Conn& c : cq)
      if (c.key == k) return &c;
    return nullptr;
  };
  auto splat = [&](int pix, const double t[3]) {
    if (t[0] == 0.0 && t[1] == 0.0 && t[2] == 0.0) return;
    if (pix < 0) {
      if (stats) stats->offscreen++;
      return;
    }
    if (stats) stats->splats++;
    for (int c = 0; c < 3; ++c) img[3 * pix + c] += t[c];
  };
  auto value = [&](const Eval& e, double out[3]) {
    bool zero = !(e.Pi > 0);
    out[0] = zero ? 0.0 : e.f.x / e.Pi;
    out[1] = zero ? 0.0 : e.f.y / e.Pi;
    out[2] = zero ? 0.0 : e.f.z / e.Pi;
  };
  auto count_dyn = [&](const Path& P) {
    int n = 0;
    for (size_t m = 1; m + 1 < P.x.size(); ++m)
      if (S.edited[P.x[m].obj]) n++;
    return n;
  };
  auto same_path = [&](const Path& a, const Path& b) {
    if (a.x.size() != b.x.size()) return false;
    for (size_t m = 0; m < a.x.size(); ++m)
      if (!same_vtx_moved(S.moved, a.x[m], b.x[m])) return false;
    return true;
  };

  std::vector<const Conn*> used_q;
  for (const Conn& c : cp) {
    if (stats) stats->connections++;
    orc_record r;
    std::memset(&r, 0, sizeof(r));
    r.tech = l; r.side = side; r.i = i;
    r.key_kind = c.key.kind; r.key_a = c.key.a; r.key_b = c.key.b;
    r.pix_p = c.path.pixel;
    r.pix_q = -1;
    r.R = 1.0;
    const SeedCrossing sp = seed_of(gp, c);
    Eval ep = eval_path(cx, F, c.path, true, &sp);
    double vp[3];
    value(ep, vp);
    if (nopm && !ep.dynamic) vp[0] = vp[1] = vp[2] = 0.0;
    r.n_cand_p = ep.n_cand;
    for (int ch = 0; ch < 3; ++ch) r.v_p[ch] = vp[ch];

    // ---- the mapped path q (replay, or reconnected suffix) in Fbar
    bool have_q = false;
    Path q;
    double R = 1.0;
    int status = ST_ACCEPTED, reason = RJ_NONE;
    Eval eq;
    const Conn* cq_match = find_q(c.key);
    if (cq_match) used_q.push_back(cq_match);
    int j = c.walk_index;
    bool recon_here = (w > 0 && single && j >= w + 1 && c.key.kind != 0);
    const bool tobj_here = mT > 0 && j >= mT && c.key.kind != 0;
    if (tobj_here && (tobj_fail || tobj_reject)) {  // t(x_m) hidden from x_{m-1} in View_Fbar, or the replayed
      status = ST_REJECTED;                         // partner lies on a moved object: no mapping from x_m on
      reason = tobj_fail ? RJ_OCCLUDED : RJ_TARGET;
    } else if (recon_here) {
      if (recon_fail) {
        status = ST_REJECTED;
        reason = recon_reason;
      } else {
        // q: mapped prefix v'_1..v'_w + base suffix v_{w+1}..v_j + the base connection endpoint
        std::vector<Vtx> walk_q;
        for (int m = 1; m <= w; ++m) walk_q.push_back(gq.A.v[m]);
        for (int m = w + 1; m <= j; ++m) walk_q.push_back(gp.A.v[m]);
        // later base vertices on dyn_F reject the rest
        for (int m = w + 2; m <= j; ++m)
          if (S.edited[gp.A.v[m].obj]) { status = ST_REJECTED; reason = RJ_SUFFIX_DYN; }
        if (status == ST_ACCEPTED) {
          q.pixel = c.path.pixel;
          if (c.key.kind == 1) {  // E-rooted: (E, walk_q, L)
            q.x.push_back(c.path.x.front());
            for (auto& v : walk_q) q.x.push_back(v);
            q.x.push_back(c.path.x.back());
          } else {  // L-rooted: (E, reversed walk_q, x_L)
            q.x.push_back(c.path.x.front());
            for (int m = (int)walk_q.size() - 1; m >= 0; --m) q.x.push_back(walk_q[m]);
            q.x.push_back(c.path.x.back());
          }
          SeedCrossing sq;  // the mapped T4 / T5's x_G' on q's first / last edge (reconnection: single walks only)
          if (gq.tech == 4 || gq.tech == 5) {
            sq.edge = gq.tech == 5 ? 0 : (int)q.x.size() - 2;
            sq.p = gq.start.p;
            sq.n = gq.start.n;
            sq.tri = gq.start.tri;
          }
          eq = eval_path(cx, Fb, q, true, &sq);
          // walk edges of q from the reconnection on must be unoccluded in View_Fbar
          int k = (int)q.x.size();
          for (int e = 0; e < k - 1; ++e) {
            bool conn_edge = (c.key.kind == 1) ? (e == k - 2) : (e == 0);
            if (conn_edge) continue;
            if (!eq.edge_vis[e]) { status = ST_REJECTED; reason = RJ_OCCLUDED; }
          }
          if (status == ST_ACCEPTED) {
            // connection edge: V = 0 zeroes the term, it does not reject
            // R = p_Fbar(suffix | q prefix) / p_F(suffix | p prefix)   (SURVEY 8(c) C7 "R")
            // walk-order vertex m of q: mapped prefix for m <= w, base suffix after
            R = reconnect_R(S, F, gp.A, gq.A, w, j) * (tobj_here ? RT : 1.0);
            if (!(R > 0) || !std::isfinite(R)) { status = ST_REJECTED; reason = RJ_TARGET; }
            have_q = status == ST_ACCEPTED;
            if (stats && have_q) stats->reconnected++;
            if (have_q && cx.recon_out) {  // geometry of the reconnection for the R pins (test export)
              Walk qw;  // q's walk: mapped prefix, base suffix; R of the inverse map q -> p swaps the roles
              for (int m = 0; m <= j; ++m) qw.v.push_back(m <= w ? gq.A.v[m] : gp.A.v[m]);
              double Rinv = reconnect_R(S, Fb, qw, gp.A, w, j);
              std::vector<double>& o = *cx.recon_out;
              o.push_back(j - w); o.push_back(R); o.push_back(Rinv);
              const Vtx* vs[6] = {&gp.A.v[w - 1], &gp.A.v[w], &gq.A.v[w - 1], &gq.A.v[w], &gp.A.v[w + 1],
                                  j >= w + 2 ? &gp.A.v[w + 2] : &gp.A.v[w + 1]};
              for (const Vtx* v : vs) {
                o.push_back(v->p.x); o.push_back(v->p.y); o.push_back(v->p.z);
                o.push_back(v->n.x); o.push_back(v->n.y); o.push_back(v->n.z);
              }
            }
          }
        }
      }
    } else if (wB > 0 && c.key.kind == 3 && c.key.b >= wB + 1) {  // reconnected emitter side (reading 19)
      const int t = c.key.a, sb = c.key.b;
      if (reconB_fail) {
        status = ST_REJECTED;
        reason = reconB_reason;
      } else if (t > gq.A.n()) {
        status = ST_UNPAIRED;  // the mapped sensor side lacks z'_t
      } else {
        for (int m = wB + 2; m <= sb; ++m)
          if (S.edited[gp.B.v[m].obj]) { status = ST_REJECTED; reason = RJ_SUFFIX_DYN; }
        if (status == ST_ACCEPTED) {
          q.x.push_back(c.path.x.front());
          for (int m = t; m >= 1; --m) q.x.push_back(gq.A.v[m]);
          if (l == 3) q.x.push_back(gq.start);
          for (int m = 1; m <= wB; ++m) q.x.push_back(gq.B.v[m]);
          for (int m = wB + 1; m <= sb; ++m) q.x.push_back(gp.B.v[m]);
          q.x.push_back(c.path.x.back());  // the same NEE vertex (slot 16 + s)
          q.pixel = project(S, gq.A.v[t].p);
          SeedCrossing sq;
          if (gq.tech == 6) {
            sq.edge = t;
            sq.p = gq.start.p;
            sq.n = gq.start.n;
            sq.tri = gq.start.tri;
          }
          eq = eval_path(cx, Fb, q, true, &sq);
          // the reconnection edge (y'_w, y_{w+1}) and every later walk edge of q must be unoccluded in View_Fbar
          // (C7); other edges only zero V (f = 0), the connection edges included
          const int k = (int)q.x.size(), er = t + (l == 3 ? 1 : 0) + wB;
          for (int e = er; e < k - 2; ++e)
            if (!eq.edge_vis[e]) { status = ST_REJECTED; reason = RJ_OCCLUDED; }
          if (status == ST_ACCEPTED) {
            R = reconnect_R(S, F, gp.B, gq.B, wB, sb);
            if (!(R > 0) || !std::isfinite(R)) { status = ST_REJECTED; reason = RJ_TARGET; }
            have_q = status == ST_ACCEPTED;
            if (stats && have_q) stats->reconnected++;
          }
        }
      }
    } else if (cq_match) {
      q = cq_match->path;
      const SeedCrossing sq = seed_of(gq, *cq_match);
      eq = eval_path(cx, Fb, q, true, &sq);
      have_q = true;
      if (tobj_here) R = RT;
    } else {
      status = ST_UNPAIRED;
    }
    if (have_q && reject_multi) {  // base hits dynamic objects more than once (diverged pairs only)
      if (!same_path(c.path, q) && (count_dyn(c.path) >= 2 || count_dyn(q) >= 2)) {
        status = ST_REJECTED;
        reason = RJ_MULTI;
        have_q = false;
      }
    }
    if (status == ST_REJECTED) have_q = false;

    double vq[3] = {0, 0, 0};
    if (have_q) {
      value(eq, vq);
      r.n_cand_q = eq.n_cand;
      r.pix_q = q.pixel;
    }
    for (int ch = 0; ch < 3; ++ch) r.v_q[ch] = vq[ch];
    r.status = status;
    r.reason = reason;
    r.R = R;
    if (diag) {  // one-way weights with the two-way pairing: accepted +v_N - R v_O, else +v_N (no coverage of O)
      for (int ch = 0; ch < 3; ++ch) {
        r.term_p[ch] = vp[ch] / spp;
        r.term_q[ch] = (status == ST_ACCEPTED) ? -R * vq[ch] / spp : 0.0;
      }
    } else if (two_way) {
      double wgt = (status == ST_ACCEPTED) ? 1.0 : 2.0;
      for (int ch = 0; ch < 3; ++ch) {
        r.term_p[ch] = wgt * sigma / spp * vp[ch];
        r.term_q[ch] = (status == ST_ACCEPTED) ? -sigma / spp * R * vq[ch] : 0.0;
      }
    } else {
      for (int ch = 0; ch < 3; ++ch) {
        r.term_p[ch] = vp[ch] / spp;
        r.term_q[ch] = have_q ? -vq[ch] / spp : 0.0;
      }
    }
    if (stats) {
      if (status == ST_ACCEPTED) stats->accepted++;
      else if (status == ST_REJECTED) { stats->rejected++; stats->rejected_by[reason & 7]++; }
      else stats->unpaired++;
    }
    // pre-sum same-pixel pairs before splatting
    if (r.pix_q == r.pix_p) {
      double t[3] = {r.term_p[0] + r.term_q[0], r.term_p[1] + r.term_q[1], r.term_p[2] + r.term_q[2]};
      splat(r.pix_p, t);
    } else {
      splat(r.pix_p, r.term_p);
      splat(r.pix_q, r.term_q);
    }
    if (recs) recs->push_back(r);
  }
  // one-way mode: every replayed connection of the paired technique contributes -v_O(q)/spp (C8)
  if (!paired) {
    for (const Conn& c : cq) {
      bool used = false;
      for (const Conn* u : used_q)
        if (u == &c) used = true;
      if (used) continue;
      const SeedCrossing sq = seed_of(gq, c);
      Eval eq = eval_path(cx, Fb, c.path, true, &sq);
      double vq[3];
      value(eq, vq);
      orc_record r;
      std::memset(&r, 0, sizeof(r));
      r.tech = l; r.side = side; r.i = i;
      r.key_kind = c.key.kind; r.key_a = c.key.a; r.key_b = c.key.b;
      r.status = ST_MAPPED_ONLY;
      r.pix_p = -1;
      r.pix_q = c.path.pixel;
      r.R = 1.0;
      r.n_cand_q = eq.n_cand;
      for (int ch = 0; ch < 3; ++ch) {
        r.term_q[ch] = -vq[ch] / spp;
        r.v_q[ch] = vq[ch];
      }
      if (stats) stats->mapped_only++;
      splat(r.pix_q, r.term_q);
      if (recs) recs->push_back(r);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// primal renderer: unidirectional PT with NEE + BSDF sampling combined by the balance heuristic
// (an estimator independent of the residual code path).  Paths with <= D edges.
// Streams: counter (pixel-sample index lo/hi, 0x80 | stream_state << 8, 2*vertex + call), key = seed; the
// stream state is F by default (independent streams per state).  With the same stream state for both
// states the two images use the same random numbers, so their difference is a correlated (low-variance)
// but still unbiased estimate of I^D(N) - I^D(O): the reference of the convergence pins.
// ------------------------------------------------------------------------------------------------
void primal_pixel_sample(Ctx& cx, int F, uint64_t seed, uint64_t idx, int D, double* img, int stream_state) {
  const Scene& S = *cx.S;
  Stream st{seed, idx, 0x80u, (uint32_t)stream_state};  // technique id 0x80 is never used by the residual streams
  int npix = S.W * S.H;
  int pix = (int)(idx % (uint64_t)npix);
  double d0[8];
  st.dims(0, d0);
  double sx = (pix % S.W) + d0[0], sy = (pix / S.W) + d0[1];
  V3 dir = camera_dir(S, sx, sy);
  V3 thr = v3(1, 1, 1);  // W_e G / p_cam = 1
  V3 L = v3(0, 0, 0);
  Hit h = closest(S, F, S.cam_pos, dir, -1, &cx.C);
  if (!h.ok) return;
  Vtx prev = cam_vtx(S);
  Vtx cur = vtx_of_hit(S.cam_pos, dir, h);
  double prev_pdf_w = -1.0;  // solid-angle pdf of the BSDF direction that produced `cur` (-1: camera)
  for (int edges = 1; edges <= D; ++edges) {
    // emission reached at `cur` (path with `edges` edges)
    if (S.emitter_index[cur.obj] >= 0) {
      V3 Le = emission(S, cur, prev.p);
      if (nonzero(Le)) {
        double w = 1.0;
        if (prev_pdf_w >= 0) {  // balance heuristic vs NEE, both in solid angle at prev
          V3 d = cur.p - prev.p;
          double d2 = dot(d, d);
          double pl = p_light(S, cur) * d2 / std::fabs(dot(cur.n, normalize(d)));
          w = prev_pdf_w / (prev_pdf_w + pl);
        }
        L = L + mul(thr, Le) * w;
      }
    }
    if (edges == D) break;
    double d[8];
    st.dims((uint32_t)edges, d);
    Mat mt = mat_of(S, cur.obj, F);
    V3 wi = normalize(prev.p - cur.p);
    // NEE (path with edges+1 edges)
    {
      Vtx xl = sample_emitter(S, d);
      V3 dl = xl.p - cur.p;
      double d2 = dot(dl, dl);
      V3 wl = dl * (1.0 / std::sqrt(d2));
      V3 Le = emission(S, xl, cur.p);
      if (nonzero(Le) && visible(S, F, cur.p, xl.p, cur.tri, xl.tri, &cx.C)) {
        V3 fr = bsdf_eval(mt, cur.n, wi, wl);
        double cosl = std::fabs(dot(xl.n, wl));
        double pl_w = p_light(S, xl) * d2 / cosl;
        double pb_w = bsdf_pdf(mt, cur.n, wi, wl);
        double w = pl_w / (pl_w + pb_w);
        double g = std::fabs(dot(cur.n, wl)) * cosl / d2;
        L = L + mul(mul(thr, fr), Le) * (g / p_light(S, xl) * w);
      }
    }
    V3 wo;
    if (!bsdf_sample(mt, cur.n, wi, d[1], d[2], wo)) break;
    double pw = bsdf_pdf(mt, cur.n, wi, wo);
    if (!(pw > 0)) break;
    V3 fr = bsdf_eval(mt, cur.n, wi, wo);
    thr = mul(thr, fr) * (std::fabs(dot(cur.n, wo)) / pw);
    Hit hn = closest(S, F, cur.p, wo, cur.tri, &cx.C);
    if (!hn.ok) break;
    prev = cur;
    cur = vtx_of_hit(cur.p, wo, hn);
    prev_pdf_w = pw;
  }
  for (int c = 0; c < 3; ++c) img[3 * pix + c] += (c == 0 ? L.x : (c == 1 ? L.y : L.z));
}

bool load_scene(Oracle& O, const orc_input* in) {
  Scene& S = O.S;
  S.pos.resize(in->n_vertices);
  for (int k = 0; k < in->n_vertices; ++k)
    S.pos[k] = v3(in->positions[3 * k], in->positions[3 * k + 1], in->positions[3 * k + 2]);
  S.idx.assign(in->indices, in->indices + 3 * in->n_triangles);
  S.tri_obj.assign(in->tri_object, in->tri_object + in->n_triangles);
  int no = in->n_objects;
  S.obj_mat.assign(in->obj_material, in->obj_material + no);
  S.obj_emit.resize(no);
  for (int o = 0; o < no; ++o)
    S.obj_emit[o] = v3(in->obj_emission[3 * o], in->obj_emission[3 * o + 1], in->obj_emission[3 * o + 2]);
  S.obj_flags.assign(in->obj_flags, in->obj_flags + no);
  S.mats.resize(in->n_materials);
  for (int m = 0; m < in->n_materials; ++m) {
    S.mats[m].type = (int)in->mat_type[m];
    S.mats[m].albedo = v3(in->mat_albedo[3 * m], in->mat_albedo[3 * m + 1], in->mat_albedo[3 * m + 2]);
    S.mats[m].alpha = in->mat_roughness[m];
  }
  for (int k = 0; k < 3 * in->n_triangles; ++k)
    if (S.idx[k] < 0 || S.idx[k] >= in->n_vertices) { O.err = "index out of range"; return false; }
  for (int k = 0; k < in->n_triangles; ++k)
    if (S.tri_obj[k] < 0 || S.tri_obj[k] >= no) { O.err = "tri_object out of range"; return false; }
  for (int o = 0; o < no; ++o)
    if (S.obj_mat[o] < 0 || S.obj_mat[o] >= in->n_materials) { O.err = "material out of range"; return false; }
  S.cam_pos = v3(in->cam_pos[0], in->cam_pos[1], in->cam_pos[2]);
  S.cam_look = v3(in->cam_look[0], in->cam_look[1], in->cam_look[2]);
  S.cam_up = v3(in->cam_up[0], in->cam_up[1], in->cam_up[2]);
  S.vfov = in->vfov_deg;
  S.W = in->width;
  S.H = in->height;
  S.eps_rel = in->eps_rel;
  // edits
  S.edited.assign(no, 0);
  S.moved.assign(no, 0);
  S.has_mat.assign(no, 0);
  for (int F = 0; F < 2; ++F) {
    S.xf[F].assign(12 * no, 0.0);
    S.emat[F].resize(no);
    for (int o = 0; o < no; ++o) {
      S.xf[F][12 * o + 0] = S.xf[F][12 * o + 5] = S.xf[F][12 * o + 10] = 1.0;
    }
  }
  for (int o = 0; o < no; ++o)
    if (S.obj_flags[o] & 1u) S.edited[o] = 1;
  for (int e = 0; e < in->n_edits; ++e) {
    int o = (int)in->edit_object[e];
    if (o < 0 || o >= no || !(S.obj_flags[o] & 1u)) { O.err = "edit on a non-dynamic object"; return false; }
    const float* xo = in->edit_old_xform + 12 * e;
    const float* xn = in->edit_new_xform + 12 * e;
    for (int k = 0; k < 12; ++k) {
      S.xf[0][12 * o + k] = xn[k];
      S.xf[1][12 * o + k] = xo[k];
    }
    S.moved[o] = std::memcmp(xo, xn, 12 * sizeof(float)) != 0 ? 1 : 0;
    S.has_mat[o] = in->edit_has_material[e] ? 1 : 0;
    if (S.has_mat[o]) {
      for (int F = 0; F < 2; ++F) {
        int which = F == 0 ? 1 : 0;  // state N uses the new material, O the old one
        Mat m;
        m.type = (int)in->edit_mat_type[2 * e + which];
        const float* al = in->edit_mat_albedo + 6 * e + 3 * which;
        m.albedo = v3(al[0], al[1], al[2]);
        m.alpha = in->edit_mat_roughness[2 * e + which];
        S.emat[F][o] = m;
      }
    }
  }
  for (int o = 0; o < no; ++o)
    if (S.moved[o] && nonzero(S.obj_emit[o])) { O.err = "moved objects must not emit"; return false; }
  // diagonal over static, non-environment geometry (C12 #13)
  AABB box;
  box.reset();
  bool any = false;
  for (int k = 0; k < in->n_triangles; ++k) {
    int o = S.tri_obj[k];
    if (S.edited[o] || (S.obj_flags[o] & 2u)) continue;
    for (int c = 0; c < 3; ++c) box.grow(S.pos[S.idx[3 * k + c]]);
    any = true;
  }
  if (!any) {
    for (int k = 0; k < in->n_triangles; ++k)
      for (int c = 0; c < 3; ++c) {
        int o = S.tri_obj[k];
        V3 p = S.pos[S.idx[3 * k + c]];
        if (S.edited[o]) p = xform_point(&S.xf[0][12 * o], p);
        box.grow(p);
      }
  }
  S.diag = len(box.hi - box.lo);
  S.eps = S.eps_rel * S.diag;
  // camera basis
  S.cf = normalize(S.cam_look - S.cam_pos);
  S.cr = normalize(cross(S.cf, S.cam_up));
  S.cu = cross(S.cr, S.cf);
  S.tanY = std::tan(S.vfov * PI / 360.0);
  S.tanX = S.tanY * (double)S.W / (double)S.H;
  S.Aplane = 4.0 * S.tanX * S.tanY;
  // placed triangles and BVHs
  std::vector<Tri> st, dn, dold;
  for (int k = 0; k < in->n_triangles; ++k) {
    int o = S.tri_obj[k];
    if (S.edited[o]) {
      dn.push_back(make_tri(S, k, 0));
      dold.push_back(make_tri(S, k, 1));
    } else {
      st.push_back(make_tri(S, k, 0));
    }
  }
  S.bvh_static.build(st);
  S.bvh_dyn[0].build(dn);
  S.bvh_dyn[1].build(dold);
  // sampling sets
  S.emitter_index.assign(no, -1);
  for (int o = 0; o < no; ++o) {
    if (!nonzero(S.obj_emit[o])) continue;
    Scene::TriSet ts;
    for (int k = 0; k < in->n_triangles; ++k)
      if (S.tri_obj[k] == o) ts.tris.push_back(k);
    if (ts.tris.empty()) continue;
    build_set(S, ts);
    S.emitter_index[o] = (int)S.emitters.size();
    S.emitters.push_back(ts);
  }
  for (int k = 0; k < in->n_triangles; ++k) {
    int o = S.tri_obj[k];
    if (S.edited[o]) S.edited_set.tris.push_back(k);
    if (S.moved[o]) S.moved_set.tris.push_back(k);
  }
  if (!S.edited_set.tris.empty()) build_set(S, S.edited_set);
  if (!S.moved_set.tris.empty()) build_set(S, S.moved_set);
  if (S.emitters.empty()) { O.err = "scene has no emitter"; return false; }
  for (const Scene::TriSet& ts : S.emitters) {  // axes of T6's "toward the light" hemispheres
    V3 c = v3(0, 0, 0);
    double a = 0;
    for (int k : ts.tris) {
      Tri t = make_tri(S, k, 0);
      double ak = 0.5 * len(cross(t.v1 - t.v0, t.v2 - t.v0));
      c = c + (t.v0 + t.v1 + t.v2) * (ak / 3.0);
      a += ak;
    }
    S.emit_centroid.push_back(c * (1.0 / a));
  }
  return true;
}

}  // namespace

extern "C" {

void* orc_create(const orc_input* in, char* err, int err_len) {
  Oracle* O = new Oracle();
  if (!load_scene(*O, in)) {
    if (err && err_len > 0) std::snprintf(err, (size_t)err_len, "%s", O->err.c_str());
    delete O;
    return nullptr;
  }
  return O;
}

void orc_destroy(void* h) { delete (Oracle*)h; }

int orc_effective_mask(void* h, uint32_t mask) { return effective_mask(((Oracle*)h)->S, mask); }
int orc_paired_tech(void* h, uint32_t mask, int l) {
  Oracle* O = (Oracle*)h;
  return paired_tech(O->S, effective_mask(O->S, mask), l);
}
double orc_scene_eps(void* h) { return ((Oracle*)h)->S.eps; }
double orc_scene_diag(void* h) { return ((Oracle*)h)->S.diag; }

// Residual samples [i0, i1) of technique `tech` (1..7) on side `side` (0 = base in N, 1 = base in O).
// img: H*W*3 doubles, accumulated.  recs (may be null): up to cap records.
int orc_residual(void* h, const orc_args* A, int tech, int side, uint64_t i0, uint64_t i1, double* img,
                 orc_record* recs, int64_t cap, int64_t* n_recs, orc_stats* stats) {
  Oracle* O = (Oracle*)h;
  O->S.vndf = (A->flags & 32u) != 0;
  O->S.t6_light = (A->flags & 512u) != 0;
  Ctx cx;
  cx.S = &O->S;
  cx.mask = effective_mask(O->S, A->technique_mask);
  if (!((cx.mask >> 6) & 1)) return -1;  // T7 required
  if (!((cx.mask >> (tech - 1)) & 1)) return 0;
  std::vector<orc_record> rv;
  std::vector<orc_record>* rp = recs ? &rv : nullptr;
  int64_t n = 0;
  for (uint64_t i = i0; i < i1; ++i) {
    rv.clear();
    residual_sample(cx, *A, tech, side, i, img, stats, rp);
    if (recs)
      for (auto& r : rv)
        if (n < cap) recs[n++] = r;
  }
  if (n_recs) *n_recs = n;
  if (stats) {
    stats->closest_rays += cx.C.closest;
    stats->shadow_rays += cx.C.shadow;
  }
  return 0;
}

// Primal render of state F (0 = N, 1 = O): samples idx in [i0, i1) (pixel = idx mod N_pix).
int orc_primal_streams(void* h, int F, int stream_state, uint64_t seed, int D, uint64_t i0, uint64_t i1, double* img,
                       orc_stats* stats) {
  Oracle* O = (Oracle*)h;
  O->S.vndf = false;  // the primal renderer samples GGX from D(h) |n.h|
  O->S.t6_light = false;
  Ctx cx;
  cx.S = &O->S;
  cx.mask = 0x7F;
  for (uint64_t i = i0; i < i1; ++i) primal_pixel_sample(cx, F, seed, i, D, img, stream_state);
  if (stats) {
    stats->closest_rays += cx.C.closest;
    stats->shadow_rays += cx.C.shadow;
  }
  return 0;
}
int orc_primal(void* h, int F, uint64_t seed, int D, uint64_t i0, uint64_t i1, double* img, orc_stats* stats) {
  return orc_primal_streams(h, F, F, seed, D, i0, i1, img, stats);
}

// Technique-pdf self-consistency: for every connection of the base samples [i0, i1)
// of (tech, side), the product of the densities the generator recorded while sampling the path, and the
// technique pdf eval_path assigns to the producing candidate (C5 table; for T4-T6 the crossing at x_G).
// out: 3 doubles per connection {recorded, eval_path candidate pdf (-1: producer not among the
// candidates), #candidates}.  Returns the number of connections (up to cap written).
int64_t orc_pdf_check(void* h, const orc_args* A, int tech, int side, uint64_t i0, uint64_t i1, double* out,
                      int64_t cap) {
  Oracle* O = (Oracle*)h;
  O->S.vndf = (A->flags & 32u) != 0;
  O->S.t6_light = (A->flags & 512u) != 0;
  const Scene& S = O->S;
  Ctx cx;
  cx.S = &S;
  cx.mask = effective_mask(S, A->technique_mask);
  int64_t n = 0;
  for (uint64_t i = i0; i < i1; ++i) {
    Stream st{A->seed, i, (uint32_t)tech, (uint32_t)side};
    Gen g = generate(cx, tech, side, st, (int)A->max_depth);
    for (const Conn& c : connections(cx, g, st, (int)A->max_depth)) {
      Eval ev = eval_path(cx, side, c.path, false);
      double pc = -1.0;
      int k = (int)c.path.x.size();
      for (size_t a = 0; a < ev.cands.size(); ++a) {
        const Cand& cd = ev.cands[a];
        if (cd.tech != c.prod_tech) continue;
        if (c.prod_tech == 7) { pc = ev.cand_p[a]; break; }
        int elem = c.prod_tech == 1 ? k - 2 : (c.prod_tech == 4 ? k - 2 : c.prod_elem);
        if (cd.elem != elem) continue;
        if (c.prod_tech >= 4 && c.prod_tech <= 6) {  // the crossing through x_G
          if (len(ev.cross[cd.elem][cd.sub].p - g.start.p) > 1e-6 * S.diag) continue;
        }
        pc = ev.cand_p[a];
        break;
      }
      if (n < cap) {
        out[3 * n] = c.pdf_rec;
        out[3 * n + 1] = pc;
        out[3 * n + 2] = (double)ev.cands.size();
      }
      n++;
    }
  }
  return n;
}

// Accepted reconnections of the samples [i0, i1) of (tech, side) (test export for the R pins, SURVEY 8(c)
// C11): 39 doubles each = {j - w, R, R of the inverse map q -> p, then (position, normal) of v_{w-1}, v_w,
// v'_{w-1}, v'_w, v_{w+1}, v_{w+2} (= v_{w+1} when j = w + 1)}.  Returns the number of reconnections.
int64_t orc_reconnections(void* h, const orc_args* A, int tech, int side, uint64_t i0, uint64_t i1, double* out,
                          int64_t cap) {
  Oracle* O = (Oracle*)h;
  O->S.vndf = (A->flags & 32u) != 0;
  O->S.t6_light = (A->flags & 512u) != 0;
  Ctx cx;
  cx.S = &O->S;
  cx.mask = effective_mask(O->S, A->technique_mask);
  if (!((cx.mask >> 6) & 1)) return -1;
  std::vector<double> rec;
  cx.recon_out = &rec;
  std::vector<double> img(3 * (size_t)O->S.W * O->S.H, 0.0);
  for (uint64_t i = i0; i < i1; ++i) residual_sample(cx, *A, tech, side, i, img.data(), nullptr, nullptr);
  int64_t n = (int64_t)(rec.size() / 39);
  std::memcpy(out, rec.data(), sizeof(double) * 39 * (size_t)std::min(n, cap));
  return n;
}

// T3's emitter-side start direction for normal n and slot-0 dims (u3, u4): out = {w, recorded pdf}
void orc_t3_light_dir(const double n[3], double u3, double u4, double out[4]) {
  double pdf;
  V3 w = t3_light_dir(v3(n[0], n[1], n[2]), u3, u4, &pdf);
  out[0] = w.x; out[1] = w.y; out[2] = w.z; out[3] = pdf;
}

// debug: print the base / mapped connection paths of one sample
void orc_debug_sample(void* h, const orc_args* A, int tech, int side, uint64_t i) {
  Oracle* O = (Oracle*)h;
  O->S.vndf = (A->flags & 32u) != 0;
  O->S.t6_light = (A->flags & 512u) != 0;
  Ctx cx;
  cx.S = &O->S;
  cx.mask = effective_mask(O->S, A->technique_mask);
  Stream st{A->seed, i, (uint32_t)tech, (uint32_t)side};
  int lq = paired_tech(O->S, cx.mask, tech);
  for (int which = 0; which < 2; ++which) {
    int F = which == 0 ? side : 1 - side;
    Gen g = generate(cx, which == 0 ? tech : lq, F, st, (int)A->max_depth);
    std::printf("%s tech %d state %d ok %d start (%g %g %g) tri %d\n", which == 0 ? "BASE" : "MAPPED",
                which == 0 ? tech : lq, F, (int)g.ok, g.start.p.x, g.start.p.y, g.start.p.z, g.start.tri);
    std::vector<Conn> cs = connections(cx, g, st, (int)A->max_depth);
    for (const Conn& c : cs) {
      std::printf("  key %d %d %d :", c.key.kind, c.key.a, c.key.b);
      for (const Vtx& v : c.path.x) std::printf(" [%d o%d e%d (%.17g %.17g %.17g) (%.17g %.17g %.17g)]", v.tri, v.obj, v.obj >= 0 ? O->S.edited[v.obj] : -1, v.p.x, v.p.y, v.p.z, v.n.x, v.n.y, v.n.z);
      std::printf("\n");
    }
  }
  std::fflush(stdout);
}

// ---------------------------------------- unit-test exports ----------------------------------------
void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) { philox4x32_10(ctr, key, out); }
double orc_u01(uint32_t x) { return u01(x); }
void orc_stream_dims(uint64_t seed, uint64_t i, uint32_t l, uint32_t side, uint32_t slot, double out[8]) {
  Stream st{seed, i, l, side};
  st.dims(slot, out);
}

// closest hit in View_F: out = {t, tri, obj, px, py, pz, nx, ny, nz} (t = -1 on miss)
void orc_closest(void* h, int F, const double o[3], const double d[3], int excl, double out[9]) {
  Oracle* O = (Oracle*)h;
  Hit hh = closest(O->S, F, v3(o[0], o[1], o[2]), normalize(v3(d[0], d[1], d[2])), excl, nullptr);
  if (!hh.ok) { out[0] = -1; return; }
  Vtx v = vtx_of_hit(v3(o[0], o[1], o[2]), normalize(v3(d[0], d[1], d[2])), hh);
  double r[9] = {hh.t, (double)v.tri, (double)v.obj, v.p.x, v.p.y, v.p.z, v.n.x, v.n.y, v.n.z};
  std::memcpy(out, r, sizeof(r));
}
// brute-force closest hit over every placed triangle (for the BVH pin)
void orc_closest_brute(void* h, int F, const double o[3], const double d[3], int excl, double out[2]) {
  Oracle* O = (Oracle*)h;
  const Scene& S = O->S;
  V3 oo = v3(o[0], o[1], o[2]), dd = normalize(v3(d[0], d[1], d[2]));
  double best = 1e300;
  int bt = -1;
  for (int k = 0; k < (int)S.tri_obj.size(); ++k) {
    if (k == excl) continue;
    Tri t = make_tri(S, k, F);
    double tt = BVH::tri_hit(t, oo, dd);
    if (tt > S.eps && tt < best) { best = tt; bt = k; }
  }
  out[0] = bt < 0 ? -1 : best;
  out[1] = bt;
}
int orc_visible(void* h, int F, const double a[3], const double b[3], int ea, int eb) {
  Oracle* O = (Oracle*)h;
  return visible(O->S, F, v3(a[0], a[1], a[2]), v3(b[0], b[1], b[2]), ea, eb, nullptr) ? 1 : 0;
}
// crossings of segment (a,b) in state F: writes up to cap {t, px,py,pz, nx,ny,nz}; returns count
int orc_crossings(void* h, int F, const double a[3], const double b[3], double* out, int cap) {
  Oracle* O = (Oracle*)h;
  std::vector<Crossing> c = crossings(O->S, F, v3(a[0], a[1], a[2]), v3(b[0], b[1], b[2]));
  for (int k = 0; k < (int)c.size() && k < cap; ++k) {
    double r[7] = {c[k].t, c[k].p.x, c[k].p.y, c[k].p.z, c[k].n.x, c[k].n.y, c[k].n.z};
    std::memcpy(out + 7 * k, r, sizeof(r));
  }
  return (int)c.size();
}
// brute-force crossing count (every moved triangle at M_Fbar, no BVH, no dedup)
int orc_crossings_brute(void* h, int F, const double a[3], const double b[3]) {
  Oracle* O = (Oracle*)h;
  const Scene& S = O->S;
  V3 aa = v3(a[0], a[1], a[2]), bb = v3(b[0], b[1], b[2]);
  double L = len(bb - aa);
  V3 d = (bb - aa) * (1.0 / L);
  int n = 0;
  for (int k = 0; k < (int)S.tri_obj.size(); ++k) {
    if (!S.moved[S.tri_obj[k]]) continue;
    Tri t = make_tri(S, k, 1 - F);
    double tt = BVH::tri_hit(t, aa, d);
    if (tt > S.eps && tt < L - S.eps) n++;
  }
  return n;
}

// BSDF: mat = {type, albedo r,g,b, alpha}; out_eval[3], returns pdf
double orc_bsdf(const double mat[5], const double n[3], const double wi[3], const double wo[3], double out_eval[3]) {
  Mat m;
  m.type = (int)mat[0] == 2 ? MAT_GGX : (int)mat[0];  // 2: GGX with visible-normal sampling
  m.vndf = (int)mat[0] == 2;
  m.albedo = v3(mat[1], mat[2], mat[3]);
  m.alpha = mat[4];
  V3 e = bsdf_eval(m, v3(n[0], n[1], n[2]), v3(wi[0], wi[1], wi[2]), v3(wo[0], wo[1], wo[2]));
  out_eval[0] = e.x; out_eval[1] = e.y; out_eval[2] = e.z;
  return bsdf_pdf(m, v3(n[0], n[1], n[2]), v3(wi[0], wi[1], wi[2]), v3(wo[0], wo[1], wo[2]));
}
int orc_bsdf_sample(const double mat[5], const double n[3], const double wi[3], double u1, double u2, double wo[3]) {
  Mat m;
  m.type = (int)mat[0] == 2 ? MAT_GGX : (int)mat[0];  // 2: GGX with visible-normal sampling
  m.vndf = (int)mat[0] == 2;
  m.albedo = v3(mat[1], mat[2], mat[3]);
  m.alpha = mat[4];
  V3 w;
  bool ok = bsdf_sample(m, v3(n[0], n[1], n[2]), v3(wi[0], wi[1], wi[2]), u1, u2, w);
  wo[0] = w.x; wo[1] = w.y; wo[2] = w.z;
  return ok ? 1 : 0;
}

// G(x,y) with normals
double orc_geometric_term(const double x[3], const double nx[3], const double y[3], const double ny[3]) {
  Vtx a, b;
  a.p = v3(x[0], x[1], x[2]); a.n = v3(nx[0], nx[1], nx[2]);
  b.p = v3(y[0], y[1], y[2]); b.n = v3(ny[0], ny[1], ny[2]);
  return geo(a, b);
}
// Eq. vertex1pdf: p(x_G) |x_G - a|^2 / |n_G.w| * |n_1.w| / |x_1 - a|^2
double orc_vertex1pdf(double pG, const double a[3], const double xg[3], const double ng[3], const double x1[3],
                      const double n1[3]) {
  V3 A = v3(a[0], a[1], a[2]), G = v3(xg[0], xg[1], xg[2]), X = v3(x1[0], x1[1], x1[2]);
  V3 w = normalize(X - A);
  return pG * dot(G - A, G - A) / std::fabs(dot(v3(ng[0], ng[1], ng[2]), w)) *
         std::fabs(dot(v3(n1[0], n1[1], n1[2]), w)) / dot(X - A, X - A);
}
// g_{G,x1,x2}
double orc_g_term(double pdir, const double ng[3], const double x1[3], const double n1[3], const double x2[3],
                  const double n2[3]) {
  V3 X1 = v3(x1[0], x1[1], x1[2]), X2 = v3(x2[0], x2[1], x2[2]);
  V3 w = normalize(X2 - X1);
  return std::fabs(dot(v3(n1[0], n1[1], n1[2]), w)) * std::fabs(dot(v3(n2[0], n2[1], n2[2]), w)) /
         std::fabs(dot(v3(ng[0], ng[1], ng[2]), w)) * pdir / dot(X2 - X1, X2 - X1);
}
// reconnection Jacobian (Eq. P:L397-401): cos(t(x_{i-1}) <- x_i)/cos(x_{i-1} <- x_i) |x_{i-1}-x_i|^2/|t(x_{i-1})-x_i|^2
double orc_reconnect_jacobian(const double xprev[3], const double tprev[3], const double xi[3], const double ni[3]) {
  V3 P = v3(xprev[0], xprev[1], xprev[2]), T = v3(tprev[0], tprev[1], tprev[2]), X = v3(xi[0], xi[1], xi[2]);
  V3 n = v3(ni[0], ni[1], ni[2]);
  return std::fabs(dot(n, normalize(T - X))) / std::fabs(dot(n, normalize(P - X))) * dot(P - X, P - X) / dot(T - X, T - X);
}
// candidates of a structural path: k vertices, dyn[k] flags, ncross[k-1]; writes (tech, elem) pairs
int orc_candidates(int k, const int32_t* dyn, const int32_t* ncross, int mask, int32_t* out, int cap) {
  std::vector<int> d(dyn, dyn + k), n(ncross, ncross + (k - 1));
  std::vector<Cand> c = enumerate_candidates(k, d, n, mask);
  for (int a = 0; a < (int)c.size() && a < cap; ++a) {
    out[2 * a] = c[a].tech;
    out[2 * a + 1] = c[a].elem;
  }
  return (int)c.size();
}
// sample a point on the edited (which=0) / moved (1) set or emitter object e (which=2+e) in state F
int orc_sample_set(void* h, int which, int F, double u0, double u1, double u2, double out[7]) {
  Oracle* O = (Oracle*)h;
  const Scene& S = O->S;
  const Scene::TriSet* ts = which == 0 ? &S.edited_set : (which == 1 ? &S.moved_set : &S.emitters[which - 2]);
  if (ts->tris.empty()) return -1;
  Vtx v = sample_set(S, *ts, F, u0, u1, u2);
  double r[7] = {v.p.x, v.p.y, v.p.z, v.n.x, v.n.y, v.n.z, (double)v.tri};
  std::memcpy(out, r, sizeof(r));
  return 0;
}
double orc_set_area(void* h, int which) {
  Oracle* O = (Oracle*)h;
  const Scene& S = O->S;
  const Scene::TriSet* ts = which == 0 ? &S.edited_set : (which == 1 ? &S.moved_set : &S.emitters[which - 2]);
  return ts->area;
}
int orc_project(void* h, const double x[3]) { return project(((Oracle*)h)->S, v3(x[0], x[1], x[2])); }

}  // extern "C"
