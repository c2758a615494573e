// rr_residual.cu -- the residual path integral estimator on the GPU (sm_100a).
//
// One thread = one residual sample (technique l, side s, index i).  The base path is
// generated in state F = side, the mapped path in Fbar with the same Philox counters (random-seed replay,
// P:L414-416) by the paired technique (dynamic<->ghost pair T2<->T5).  The two walks run in
// lockstep so that the static-BLAS traversal is shared while the walks have not diverged (A3), the
// reconnection ("keep vertex the same") is decided at the first diverged rough vertex, and
// connections are evaluated and splatted as soon as they are formed.
//
// MIS is evaluated per connection path as ratios to the PT (T7) pdf: every candidate pdf
// p_c / p_T7 reduces to products of per-edge reverse/forward pdf ratios (the 1/d^2 factors cancel), and
// ghost crossings enter only through three per-edge sums (count, sum 1/|cos_G|, sum d^2/|cos_G| toward
// either endpoint), so no per-crossing records are stored (P:L354 realised as running sums).
#include <cuda_runtime.h>

#include "rr_device.cuh"
#include "rr_kernels.h"

namespace rr {

enum { ST_ACCEPTED = 0, ST_REJECTED = 1, ST_UNPAIRED = 2, ST_MAPPED_ONLY = 3 };
enum { RJ_NONE = 0, RJ_OCCLUDED = 1, RJ_JACOBIAN = 2, RJ_MULTI = 3, RJ_TARGET = 4, RJ_SUFFIX_DYN = 5 };

struct PV {  // path vertex in one state
  float3 p, n;
  int tri, obj;  // tri = -1: camera; obj = -1: camera
};

// forward declaration of the object flags lookup used below
__device__ __forceinline__ uint32_t oflags(const DevScene& S, int obj);
// base and mapped vertices coincide iff same primitive, same point, and not on a MOVED object (a vertex
// on a moved object lies on a different hit instance in each state)
__device__ __forceinline__ bool same_pv(const DevScene& S, const PV& a, const PV& b) {
  if (oflags(S, a.obj) & OBJ_MOVED) return false;
  return a.tri == b.tri && eq3(a.p, b.p) && eq3(a.n, b.n);
}
__device__ __forceinline__ PV cam_pv(const DevScene& S) {
  PV v;
  v.p = S.cam_pos;
  v.n = S.cf;
  v.tri = -1;
  v.obj = -1;
  return v;
}
__device__ __forceinline__ uint32_t oflags(const DevScene& S, int obj) { return obj < 0 ? 0u : __ldg(&S.obj_flags[obj]); }
__device__ __forceinline__ bool edited(const DevScene& S, int obj) { return (oflags(S, obj) & OBJ_EDITED) != 0u; }

// hit -> vertex in state F
__device__ __forceinline__ PV hit_pv(const DevScene& S, const Hit& h, float3 o, float3 d, int F) {
  PV v;
  v.p = o + d * h.t;
  const float4* tp = S.ltris + 3 * h.leaf;
  float4 a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
  float3 n = cross3(f3(b.x - a.x, b.y - a.y, b.z - a.z), f3(c.x - a.x, c.y - a.y, c.z - a.z));
  if (h.inst >= 0) n = xf_vec(S.inst[h.inst].M[F], n);
  v.n = norm3_exact(n);
  v.tri = __float_as_int(a.w);
  v.obj = (int)__ldg(&S.tri_obj[v.tri]);
  return v;
}

// area-uniform point on a triangle set (C3): first k with cdf[k] > u0; su = sqrt(u1); b0 = 1-su; b1 = u2 su
__device__ PV sample_set(const DevScene& S, const uint32_t* tris, const float* cdf, int n, int F, float u0, float u1,
                         float u2) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldg(&cdf[mid]) > u0) hi = mid; else lo = mid + 1;
  }
  int tri = (int)__ldg(&tris[lo]);
  float4 a = __ldg(&S.tverts[3 * tri]), b = __ldg(&S.tverts[3 * tri + 1]), c = __ldg(&S.tverts[3 * tri + 2]);
  float su = sqrtf(u1);
  float b0 = 1.0f - su, b1 = u2 * su, b2 = 1.0f - b0 - b1;
  float3 x = f3(a.x, a.y, a.z) * b0 + f3(b.x, b.y, b.z) * b1 + f3(c.x, c.y, c.z) * b2;
  float3 nrm = cross3(f3(b.x - a.x, b.y - a.y, b.z - a.z), f3(c.x - a.x, c.y - a.y, c.z - a.z));
  int obj = (int)__ldg(&S.tri_obj[tri]);
  int k = __ldg(&S.obj_inst[obj]);
  if (k >= 0) {
    x = xf_point(S.inst[k].M[F], x);
    nrm = xf_vec(S.inst[k].M[F], nrm);
  }
  PV v;
  v.p = x;
  v.n = norm3_exact(nrm);
  v.tri = tri;
  v.obj = obj;
  return v;
}
// NEE emitter sample (C3): object min(floor(d3 n_obj), n_obj-1), then area-uniform within it
__device__ __forceinline__ PV sample_emitter(const DevScene& S, float d3, float d4, float d5, float d6) {
  int e = min((int)floorf(d3 * (float)S.n_emit), S.n_emit - 1);
  int off = __ldg(&S.emit_off[e]), cnt = __ldg(&S.emit_cnt[e]);
  return sample_set(S, S.emit_tris + off, S.emit_cdf + off, cnt, 0, d4, d5, d6);
}

// ------------------------------------------------------------------------------------------------
// query helpers (both states at once where the geometry is shared; A3/A3b/A4)
// ------------------------------------------------------------------------------------------------
struct Trace2 {
  bool ok[2];
  PV v[2];
  Cross c[2];
};
// closest hit from o along d in View_F for each requested state, with the ghost crossings of the
// resulting edge (eps, t_F - eps).  The static BLAS is traversed once.
__device__ Trace2 trace2(const DevScene& S, float3 o, float3 d, int excl, bool want0, bool want1, QCount& qc) {
  Trace2 r;
  r.ok[0] = r.ok[1] = false;
  WRay wr = make_wray(o, d);
  Hit hs = closest_static(S, wr, S.eps, excl);
  qc.closest++;
  for (int F = 0; F < 2; ++F) {
    if (!(F == 0 ? want0 : want1)) continue;
    Hit h = hs;
    closest_dyn(S, F, o, d, S.eps, excl, h);
    if (h.leaf < 0) continue;
    r.ok[F] = true;
    r.v[F] = hit_pv(S, h, o, d, F);
    r.c[F] = S.n_moved > 0 ? crossings(S, F, o, d, S.eps, h.t - S.eps, h.t) : cross_zero();
    if (S.n_moved > 0) qc.inst++;
  }
  return r;
}
struct Seg2 {
  bool vis[2];
  Cross c[2];
};
// segment a -> b: visibility in View_F (both endpoint triangles excluded) and ghost crossings per state
__device__ Seg2 seg2(const DevScene& S, float3 a, float3 b, int ea, int eb, bool want0, bool want1, QCount& qc) {
  Seg2 r;
  r.vis[0] = r.vis[1] = false;
  r.c[0] = r.c[1] = cross_zero();
  float3 dv = b - a;
  float L = sqrtf(dot3(dv, dv));
  if (!(L > 2.0f * S.eps)) return r;
  float3 d = dv * (1.0f / L);
  WRay wr = make_wray(a, d);
  bool sblock = occluded_static(S, wr, S.eps, L - S.eps, ea, eb);
  qc.shadow++;
  for (int F = 0; F < 2; ++F) {
    if (!(F == 0 ? want0 : want1)) continue;
    r.vis[F] = !sblock && !occluded_dyn(S, F, a, d, S.eps, L - S.eps, ea, eb);
    if (S.n_moved > 0) {
      r.c[F] = crossings(S, F, a, d, S.eps, L - S.eps, L);
      qc.inst++;
    }
  }
  return r;
}
__device__ __forceinline__ Cross swapc(Cross c) {
  float t = c.sa;
  c.sa = c.sb;
  c.sb = t;
  return c;
}

// area pdf of generating `to` from `from` with the walk arriving from `prev` (state F)
__device__ __forceinline__ float area_pdf(const DevScene& S, int F, const PV& prev, const PV& from, const PV& to) {
  Mat m = load_mat(S, (uint32_t)from.obj, F);
  float3 wi = norm3_exact(prev.p - from.p);
  float3 dv = to.p - from.p;
  float d2 = dot3(dv, dv);
  float3 wo = dv * (1.0f / sqrtf(d2));
  return bsdf_pdf(m, from.n, wi, wo) * fabsf(dot3(to.n, wo)) / d2;
}

// ------------------------------------------------------------------------------------------------
// value of a connection path v = f / Pi (Eq.2; balance heuristic P:L351-353), in state F.
// x[0] = E, x[k-1] = L; e[i] = crossings of edge (x_i, x_{i+1}) with sa measured from x_i, sb from x_{i+1}.
// Computed as (f / p_T7) / (1 + sum_c p_c / p_T7).
// ------------------------------------------------------------------------------------------------
__device__ float3 path_value(const DevScene& S, const PV* x, const Cross* e, int k, int F, uint32_t mask) {
  const float3 zero = f3(0.f, 0.f, 0.f);
  float3 d01 = x[1].p - x[0].p;
  float dd01 = dot3(d01, d01);
  float3 w01 = d01 * (1.0f / sqrtf(dd01));
  float cth = dot3(w01, S.cf);
  if (!(cth > 0.0f)) return zero;
  const PV& L = x[k - 1];
  float4 le4 = __ldg(&S.obj_emit[L.obj]);
  float3 Le = f3(le4.x, le4.y, le4.z);
  if (!(dot3(L.n, x[k - 2].p - L.p) > 0.0f)) return zero;  // front face only
  if (k == 2) return Le;                                     // direct view: W_e G / p_cam = 1, Pi = p_T7
  float cos1 = fabsf(dot3(x[1].n, w01));
  float invpcam = S.Aplane * cth * cth * cth * dd01 / cos1;  // 1 / p_cam(x_1)
  float pL = __ldg(&S.emit_pL[__ldg(&S.obj_emitter[L.obj])]);
  const bool t1 = mask & 1u, t2 = mask & 2u, t3 = mask & 4u, t4 = mask & 8u, t5 = mask & 16u, t6 = mask & 32u;
  float3 T = f3(1.f, 1.f, 1.f);
  float sum = 1.0f;  // T7
  if (t5 && e[0].n > 0.0f) sum += S.pA_G * S.Aplane * cth * cth * cth * e[0].sa;
  float Q = 1.0f;  // prod_{m < i} rev_m / fwd_{m+1}
  for (int i = 1; i <= k - 2; ++i) {
    Mat m = load_mat(S, (uint32_t)x[i].obj, F);
    float3 wi = norm3_exact(x[i - 1].p - x[i].p);
    float3 dv = x[i + 1].p - x[i].p;
    float d2 = dot3(dv, dv);
    float3 wo = dv * (1.0f / sqrtf(d2));
    float3 rho = bsdf_eval(m, x[i].n, wi, wo);
    float pf = bsdf_pdf(m, x[i].n, wi, wo);
    float cout = fabsf(dot3(x[i].n, wo));
    float cin_next = fabsf(dot3(x[i + 1].n, wo));
    bool dyn = edited(S, x[i].obj);
    if (!(pf > 0.0f)) return zero;  // f = 0 (rho = 0 exactly where pf = 0 for these BSDFs)
    if (i < k - 2) {
      T = mul3(T, rho * (cout / pf));
    } else {
      T = mul3(mul3(T, rho), Le) * (cout * cin_next / d2 / pL);
    }
    float base = S.pA_D * invpcam * Q;
    if (dyn) {
      if (i == k - 2) { if (t1) sum += base; }                          // T1: adjacent to the emitter
      else if (i == 1) { if (t2) sum += S.pA_D * invpcam; }             // T2: adjacent to the sensor
      else if (t3) sum += base * (fmaxf(0.0f, dot3(x[i].n, wo)) * RR_INV_PI_F) / pf;  // T3
    }
    if (e[i].n > 0.0f) {
      if (i + 1 == k - 1) { if (t4) sum += S.pA_G * e[i].sb * cout / d2 * invpcam * Q; }  // T4 (Eq. vertex1pdf)
      else if (t6) sum += S.pA_G * (0.25f * RR_INV_PI_F) * e[i].s0 * cout / pf * invpcam * Q;  // T6
    }
    if (i <= k - 3) {  // q_i = rev_i / fwd_{i+1} on edge (i, i+1)
      Mat mn = load_mat(S, (uint32_t)x[i + 1].obj, F);
      float pr = bsdf_pdf(mn, x[i + 1].n, norm3_exact(x[i + 2].p - x[i + 1].p), wo * -1.0f);
      Q *= pr * cout / (pf * cin_next);
    }
  }
  return T * (1.0f / sum);
}

// ------------------------------------------------------------------------------------------------
// splat + records + statistics
// ------------------------------------------------------------------------------------------------
struct Out {
  const KArgs* A;
  QCount qc;
  uint32_t conns, acc, rej, unp, monly, recon, splats, offscreen, zero;
  uint32_t rejby[6];
};
__device__ __forceinline__ void splat(Out& o, int pix, float3 t) {
  if (t.x == 0.0f && t.y == 0.0f && t.z == 0.0f) return;
  if (pix < 0) {
    o.offscreen++;
    return;
  }
  o.splats++;
  atomicAdd(reinterpret_cast<float4*>(o.A->image) + pix, make_float4(t.x, t.y, t.z, 0.0f));
}
__device__ void emit_record(Out& o, uint64_t i, int kind, int a, int b, int status, int reason, int pix_p, float3 tp,
                            int pix_q, float3 tq, float R) {
  const KArgs& A = *o.A;
  if (status == ST_ACCEPTED) o.acc++;
  else if (status == ST_REJECTED) { o.rej++; o.rejby[reason < 6 ? reason : 0]++; }
  else if (status == ST_UNPAIRED) o.unp++;
  else o.monly++;
  if (status != ST_MAPPED_ONLY) o.conns++;
  if (pix_p == pix_q) {
    float3 s = tp + tq;
    if (s.x == 0.0f && s.y == 0.0f && s.z == 0.0f && (tp.x != 0.0f || tp.y != 0.0f || tp.z != 0.0f)) o.zero++;
    if (!A.dump) splat(o, pix_p, s);
  } else if (!A.dump) {
    splat(o, pix_p, tp);
    splat(o, pix_q, tq);
  }
  if (A.dump) {
    unsigned long long slot = atomicAdd(A.rec_count, 1ull);
    if (slot < A.rec_cap) {
      rr_path_record r;
      r.tech = A.tech;
      r.side = A.side;
      r.i = i;
      r.key_kind = kind;
      r.key_a = a;
      r.key_b = b;
      r.status = status;
      r.reason = reason;
      r.pix_p = pix_p;
      r.term_p[0] = tp.x; r.term_p[1] = tp.y; r.term_p[2] = tp.z;
      r.pix_q = pix_q;
      r.term_q[0] = tq.x; r.term_q[1] = tq.y; r.term_q[2] = tq.z;
      r.R = R;
      A.recs[slot] = r;
    }
  }
}
// terms of one connection pair and splat
__device__ void finish(Out& o, uint64_t i, int kind, int a, int b, int status, int reason, int pix_p, float3 vp,
                       int pix_q, float3 vq, float R) {
  const KArgs& A = *o.A;
  float3 tp, tq;
  if (A.two_way) {
    float wgt = (status == ST_ACCEPTED) ? 1.0f : 2.0f;
    tp = vp * (wgt * A.sigma * A.inv_spp);
    tq = (status == ST_ACCEPTED) ? vq * (-A.sigma * A.inv_spp * R) : f3(0.f, 0.f, 0.f);
    if (status != ST_ACCEPTED) pix_q = -1;
  } else {
    tp = vp * A.inv_spp;
    tq = vq * (-A.inv_spp);
  }
  emit_record(o, i, kind, a, b, status, reason, pix_p, tp, pix_q, tq, R);
}

// ------------------------------------------------------------------------------------------------
// single-walk techniques: T7, T1, T2, T4, T5  (E-rooted: T7, T2, T5; L-rooted: T1, T4)
// ------------------------------------------------------------------------------------------------
struct Walk {
  PV v[RR_MAXV];
  Cross ex[RR_MAXV];  // ex[m]: crossings of the walk edge v[m-1] -> v[m], sa measured from v[m-1]
  int n;              // number of walk vertices (0: the technique failed)
  int pixel;          // fixed pixel (T7, T2, T5)
};

// start of a single-walk technique in state F (C4).  For T7 the caller traces both states.
__device__ void start_single(const DevScene& S, int tech, int F, const float d0[8], const KArgs& A, uint64_t i,
                             Walk& W, QCount& qc) {
  W.n = 0;
  W.pixel = -1;
  PV E = cam_pv(S);
  switch (tech) {
    case 1: {  // dynamic from emitter
      if (S.n_edited == 0) return;
      PV xd = sample_set(S, S.edited_tris, S.edited_cdf, S.n_edited, F, d0[0], d0[1], d0[2]);
      PV xl = sample_emitter(S, d0[3], d0[4], d0[5], d0[6]);
      if (!(dot3(xl.n, xd.p - xl.p) > 0.0f)) return;
      Seg2 s = seg2(S, xl.p, xd.p, xl.tri, xd.tri, F == 0, F == 1, qc);  // "fails if blocked"
      if (!s.vis[F]) return;
      W.v[0] = xl; W.v[1] = xd; W.ex[1] = s.c[F]; W.n = 1;
      return;
    }
    case 2: {  // dynamic from sensor
      if (S.n_edited == 0) return;
      PV xd = sample_set(S, S.edited_tris, S.edited_cdf, S.n_edited, F, d0[0], d0[1], d0[2]);
      int pix = project(S, xd.p);
      if (pix < 0) return;
      Seg2 s = seg2(S, E.p, xd.p, -1, xd.tri, F == 0, F == 1, qc);
      if (!s.vis[F]) return;
      W.v[0] = E; W.v[1] = xd; W.ex[1] = s.c[F]; W.n = 1; W.pixel = pix;
      return;
    }
    case 4: {  // ghost from emitter: x_G on ghost_F = moved objects at M_Fbar
      if (S.n_moved == 0) return;
      PV xg = sample_set(S, S.moved_tris, S.moved_cdf, S.n_moved, 1 - F, d0[0], d0[1], d0[2]);
      PV xl = sample_emitter(S, d0[3], d0[4], d0[5], d0[6]);
      float3 dv = xg.p - xl.p;
      float dl = sqrtf(dot3(dv, dv));
      if (!(dl > S.eps)) return;
      float3 dir = dv * (1.0f / dl);
      if (!(dot3(xl.n, dir) > 0.0f)) return;
      Trace2 t = trace2(S, xl.p, dir, xl.tri, F == 0, F == 1, qc);
      if (!t.ok[F]) return;
      float3 q = t.v[F].p - xl.p;
      if (!(sqrtf(dot3(q, q)) > dl + S.eps)) return;
      W.v[0] = xl; W.v[1] = t.v[F]; W.ex[1] = t.c[F]; W.n = 1;
      return;
    }
    case 5: {  // ghost from sensor
      if (S.n_moved == 0) return;
      PV xg = sample_set(S, S.moved_tris, S.moved_cdf, S.n_moved, 1 - F, d0[0], d0[1], d0[2]);
      int pix = project(S, xg.p);
      if (pix < 0) return;
      float3 dv = xg.p - E.p;
      float dg = sqrtf(dot3(dv, dv));
      float3 dir = dv * (1.0f / dg);
      Trace2 t = trace2(S, E.p, dir, -1, F == 0, F == 1, qc);
      if (!t.ok[F]) return;
      float3 q = t.v[F].p - E.p;
      if (!(sqrtf(dot3(q, q)) > dg + S.eps)) return;
      W.v[0] = E; W.v[1] = t.v[F]; W.ex[1] = t.c[F]; W.n = 1; W.pixel = pix;
      return;
    }
  }
}

__device__ __forceinline__ bool nee_ok(int tech, int m) { return tech == 2 ? m >= 2 : true; }

__device__ void sample_single(const DevScene& S, const KArgs& A, uint64_t i, const Rng& rng, Out& o) {
  const int F = A.side, Fb = 1 - A.side;
  const int l = A.tech, lq = A.tech_q;
  const int D = A.max_depth;
  const bool Lroot = (l == 1 || l == 4);
  float d0[8];
  rng.dims(0, d0);
  Walk P, Q;
  PV E = cam_pv(S);
  if (l == 7) {  // same pixel and jitter in both states: one trace serves both (A3)
    int npix = S.W * S.H;
    int pix = (int)(i % (uint64_t)npix);
    float3 dir = camera_dir(S, (float)(pix % S.W) + d0[0], (float)(pix / S.W) + d0[1]);
    Trace2 t = trace2(S, E.p, dir, -1, true, true, o.qc);
    P.n = Q.n = 0;
    P.pixel = Q.pixel = pix;
    if (t.ok[F]) { P.v[0] = E; P.v[1] = t.v[F]; P.ex[1] = t.c[F]; P.n = 1; }
    if (t.ok[Fb]) { Q.v[0] = E; Q.v[1] = t.v[Fb]; Q.ex[1] = t.c[Fb]; Q.n = 1; }
  } else {
    start_single(S, l, F, d0, A, i, P, o.qc);
    start_single(S, lq, Fb, d0, A, i, Q, o.qc);
  }
  if (P.n == 0 && (A.two_way || Q.n == 0)) return;

  const int maxW = D - 1 > 1 ? D - 1 : 1;  // walk vertices needed (connections at j <= D-1; T7 emission at 1)
  int recon = 0;                            // 0 none, 1 reconnected at w, 2 failed at w
  int w = 0;
  int reject_from = 1 << 30, reject_reason = RJ_NONE;
  float R1 = 1.0f, R2 = 1.0f;
  bool rdiv = false, hdiv = false;
  int dynP = 0, dynQ = 0;
  bool Pend = P.n == 0, Qend = Q.n == 0;

  for (int m = 1;; ++m) {
    bool hasP = m <= P.n, hasQ = m <= Q.n;
    if (!hasP && (A.two_way || !hasQ)) break;
    bool vdiff = hasP && hasQ && !same_pv(S, P.v[m], Q.v[m]);
    hdiv = hdiv || vdiff || (hasP != hasQ);
    if (hasP && edited(S, P.v[m].obj)) dynP++;
    if (hasQ && edited(S, Q.v[m].obj)) dynQ++;

    // ---------------- connections at walk vertex m
    if (!Lroot) {
      // direct view of an emitter (T7 only, k = 2)
      if (l == 7 && m == 1) {
        bool pe = hasP && __ldg(&S.obj_emitter[P.v[1].obj]) >= 0;
        bool qe = hasQ && __ldg(&S.obj_emitter[Q.v[1].obj]) >= 0;
        PV x[2];
        Cross ce[1];
        float3 vp = f3(0.f, 0.f, 0.f), vq = vp;
        if (pe) { x[0] = E; x[1] = P.v[1]; ce[0] = P.ex[1]; vp = path_value(S, x, ce, 2, F, A.mask); }
        if (qe) { x[0] = E; x[1] = Q.v[1]; ce[0] = Q.ex[1]; vq = path_value(S, x, ce, 2, Fb, A.mask); }
        if (pe) {
          int st = qe ? ST_ACCEPTED : ST_UNPAIRED;
          if (st == ST_ACCEPTED && A.reject_multi && hdiv && (dynP >= 2 || dynQ >= 2)) st = ST_REJECTED;
          finish(o, i, 0, 1, 0, st, st == ST_REJECTED ? RJ_MULTI : RJ_NONE, P.pixel, vp, Q.pixel, vq, 1.0f);
        } else if (qe && !A.two_way) {
          finish(o, i, 0, 1, 0, ST_MAPPED_ONLY, RJ_NONE, -1, f3(0.f, 0.f, 0.f), Q.pixel, vq, 1.0f);
        }
      }
      // NEE at v_m: path (E, v_1..v_m, L), slot m
      if (m + 1 <= D) {
        bool pc = hasP && nee_ok(l, m);
        bool reconnected_here = (recon == 1 && m >= w + 1);
        bool qc_ = hasQ && nee_ok(lq, m) && !(recon == 2 && m >= w + 1);
        if (reconnected_here && m >= reject_from) qc_ = false;
        if (pc || (qc_ && !A.two_way)) {
          float d[8];
          rng.dims((uint32_t)m, d);
          PV L = sample_emitter(S, d[3], d[4], d[5], d[6]);
          Seg2 sp, sq;
          bool shared = pc && qc_ && same_pv(S, P.v[m], Q.v[m]);
          if (shared) {
            sp = seg2(S, P.v[m].p, L.p, P.v[m].tri, L.tri, true, true, o.qc);
            sq = sp;
          } else {
            if (pc) sp = seg2(S, P.v[m].p, L.p, P.v[m].tri, L.tri, F == 0, F == 1, o.qc);
            if (qc_) sq = seg2(S, Q.v[m].p, L.p, Q.v[m].tri, L.tri, Fb == 0, Fb == 1, o.qc);
          }
          PV x[RR_MAXV + 1];
          Cross ce[RR_MAXV + 1];
          float3 vp = f3(0.f, 0.f, 0.f), vq = vp;
          if (pc && sp.vis[F]) {
            x[0] = E;
            for (int j = 1; j <= m; ++j) { x[j] = P.v[j]; ce[j - 1] = P.ex[j]; }
            x[m + 1] = L;
            ce[m] = sp.c[F];
            vp = path_value(S, x, ce, m + 2, F, A.mask);
          }
          if (qc_ && sq.vis[Fb]) {
            x[0] = E;
            for (int j = 1; j <= m; ++j) { x[j] = Q.v[j]; ce[j - 1] = Q.ex[j]; }
            x[m + 1] = L;
            ce[m] = sq.c[Fb];
            vq = path_value(S, x, ce, m + 2, Fb, A.mask);
          }
          if (pc) {
            int st = ST_ACCEPTED, rs = RJ_NONE;
            float R = 1.0f;
            if (recon == 2 && m >= w + 1) { st = ST_REJECTED; rs = reject_reason; }
            else if (reconnected_here && m >= reject_from) { st = ST_REJECTED; rs = reject_reason; }
            else if (!qc_) st = ST_UNPAIRED;
            else if (reconnected_here) {
              R = R1 * (m >= w + 2 ? R2 : 1.0f);
              if (!(R > 0.0f) || !isfinite(R)) { st = ST_REJECTED; rs = RJ_TARGET; }
            }
            if (st == ST_ACCEPTED && A.reject_multi && hdiv && (dynP >= 2 || dynQ >= 2)) { st = ST_REJECTED; rs = RJ_MULTI; }
            finish(o, i, 1, m, 0, st, rs, P.pixel, vp, Q.pixel, vq, R);
          } else if (qc_ && !A.two_way) {
            finish(o, i, 1, m, 0, ST_MAPPED_ONLY, RJ_NONE, -1, f3(0.f, 0.f, 0.f), Q.pixel, vq, 1.0f);
          }
        }
      }
    } else if (m + 1 <= D) {
      // sensor connection at v_m: path (E, v_m..v_1, x_L)
      bool pc = hasP;
      bool reconnected_here = (recon == 1 && m >= w + 1);
      bool qc_ = hasQ && !(recon == 2 && m >= w + 1);
      if (reconnected_here && m >= reject_from) qc_ = false;
      if (pc || (qc_ && !A.two_way)) {
        Seg2 sp, sq;
        int pixp = -1, pixq = -1;
        bool shared = pc && qc_ && same_pv(S, P.v[m], Q.v[m]);
        if (pc) pixp = project(S, P.v[m].p);
        if (qc_) pixq = project(S, Q.v[m].p);
        if (shared) {
          sp = seg2(S, P.v[m].p, E.p, P.v[m].tri, -1, true, true, o.qc);
          sq = sp;
        } else {
          if (pc) sp = seg2(S, P.v[m].p, E.p, P.v[m].tri, -1, F == 0, F == 1, o.qc);
          if (qc_) sq = seg2(S, Q.v[m].p, E.p, Q.v[m].tri, -1, Fb == 0, Fb == 1, o.qc);
        }
        PV x[RR_MAXV + 1];
        Cross ce[RR_MAXV + 1];
        float3 vp = f3(0.f, 0.f, 0.f), vq = vp;
        if (pc && sp.vis[F]) {
          x[0] = E;
          ce[0] = swapc(sp.c[F]);
          for (int j = 1; j <= m; ++j) { x[j] = P.v[m + 1 - j]; ce[j] = swapc(P.ex[m + 1 - j]); }
          x[m + 1] = P.v[0];
          vp = path_value(S, x, ce, m + 2, F, A.mask);
        }
        if (qc_ && sq.vis[Fb]) {
          x[0] = E;
          ce[0] = swapc(sq.c[Fb]);
          for (int j = 1; j <= m; ++j) { x[j] = Q.v[m + 1 - j]; ce[j] = swapc(Q.ex[m + 1 - j]); }
          x[m + 1] = Q.v[0];
          vq = path_value(S, x, ce, m + 2, Fb, A.mask);
        }
        if (pc) {
          int st = ST_ACCEPTED, rs = RJ_NONE;
          float R = 1.0f;
          if (recon == 2 && m >= w + 1) { st = ST_REJECTED; rs = reject_reason; }
          else if (reconnected_here && m >= reject_from) { st = ST_REJECTED; rs = reject_reason; }
          else if (!qc_) st = ST_UNPAIRED;
          else if (reconnected_here) {
            R = R1 * (m >= w + 2 ? R2 : 1.0f);
            if (!(R > 0.0f) || !isfinite(R)) { st = ST_REJECTED; rs = RJ_TARGET; }
          }
          if (st == ST_ACCEPTED && A.reject_multi && hdiv && (dynP >= 2 || dynQ >= 2)) { st = ST_REJECTED; rs = RJ_MULTI; }
          finish(o, i, 2, m, 0, st, rs, pixp, vp, pixq, vq, R);
        } else if (qc_ && !A.two_way) {
          finish(o, i, 2, m, 0, ST_MAPPED_ONLY, RJ_NONE, -1, f3(0.f, 0.f, 0.f), pixq, vq, 1.0f);
        }
      }
    }
    if (m >= maxW) break;

    // ---------------- advance the walks from v_m (slot m)
    float d[8];
    rng.dims((uint32_t)m, d);
    bool qActive = (recon == 0) && hasQ && !Qend;
    bool okP = false, okQ = false;
    float3 woP, woQ;
    Mat mp, mq;
    if (hasP && !Pend) {
      mp = load_mat(S, (uint32_t)P.v[m].obj, F);
      okP = bsdf_sample(mp, P.v[m].n, norm3_exact(P.v[m - 1].p - P.v[m].p), d[1], d[2], woP);
    }
    if (qActive) {
      mq = load_mat(S, (uint32_t)Q.v[m].obj, Fb);
      okQ = bsdf_sample(mq, Q.v[m].n, norm3_exact(Q.v[m - 1].p - Q.v[m].p), d[1], d[2], woQ);
    }
    bool dirdiv = qActive && hasP && !Pend && ((okP != okQ) || (okP && okQ && !eq3(woP, woQ)));
    bool div_m = rdiv || vdiff || dirdiv;
    bool shared = qActive && okP && okQ && !vdiff && !dirdiv;
    bool gotP = false;
    if (okP) {
      Trace2 t = trace2(S, P.v[m].p, woP, P.v[m].tri, F == 0 || shared, F == 1 || shared, o.qc);
      if (t.ok[F]) { P.v[m + 1] = t.v[F]; P.ex[m + 1] = t.c[F]; P.n = m + 1; gotP = true; }
      if (shared) {
        if (t.ok[Fb]) { Q.v[m + 1] = t.v[Fb]; Q.ex[m + 1] = t.c[Fb]; Q.n = m + 1; }
        else Qend = true;
      }
    }
    if (hasP && !gotP) Pend = true;
    if (A.reconnect && recon == 0 && qActive && hasP && div_m && rough_enough(mp, A.alpha_min) &&
        rough_enough(mq, A.alpha_min)) {
      // reconnection at w = m to the base vertex v_{m+1}
      w = m;
      if (!gotP) {
        recon = 2;
        reject_from = m + 1;
        reject_reason = RJ_TARGET;
      } else {
        const PV& vw = P.v[m];
        const PV& vq = Q.v[m];
        const PV& tg = P.v[m + 1];
        float3 a = vq.p - tg.p, b = vw.p - tg.p;
        float la2 = dot3(a, a), lb2 = dot3(b, b);
        int rs = RJ_NONE;
        Seg2 s;
        if (edited(S, tg.obj)) rs = RJ_TARGET;                                              // (1) P:L406
        else if (!rough_enough(load_mat(S, (uint32_t)tg.obj, F), A.alpha_min)) rs = RJ_TARGET;  // (2) P:L408
        else if (fminf(sqrtf(lb2), sqrtf(la2)) < A.dmin) rs = RJ_TARGET;                   // (3) P:L410
        else {
          s = seg2(S, vq.p, tg.p, vq.tri, tg.tri, Fb == 0, Fb == 1, o.qc);
          if (!s.vis[Fb]) rs = RJ_OCCLUDED;
          else {
            float Jg = fabsf(dot3(tg.n, a * (1.0f / sqrtf(la2)))) / fabsf(dot3(tg.n, b * (1.0f / sqrtf(lb2)))) * lb2 / la2;
            if (!(Jg <= A.jacobian_max && Jg >= 1.0f / A.jacobian_max)) rs = RJ_JACOBIAN;
          }
        }
        if (rs == RJ_NONE) {
          R1 = area_pdf(S, Fb, Q.v[m - 1], vq, tg) / area_pdf(S, F, P.v[m - 1], vw, tg);
          recon = 1;
          Q.v[m + 1] = tg;
          Q.ex[m + 1] = s.c[Fb];
          Q.n = m + 1;
        } else {
          recon = 2;
          reject_from = m + 1;
          reject_reason = rs;
        }
      }
    } else if (qActive && !shared) {
      if (okQ) {
        Trace2 t = trace2(S, Q.v[m].p, woQ, Q.v[m].tri, Fb == 0, Fb == 1, o.qc);
        if (t.ok[Fb]) { Q.v[m + 1] = t.v[Fb]; Q.ex[m + 1] = t.c[Fb]; Q.n = m + 1; }
        else Qend = true;
      } else {
        Qend = true;
      }
    } else if (recon == 1 && m >= w + 1 && gotP) {
      // shared suffix edge v_m -> v_{m+1}, re-checked against dyn_Fbar only (instance query), with the
      // Fbar ghost crossings for the mapped path's MIS
      const PV& a = P.v[m];
      const PV& b = P.v[m + 1];
      float3 dv = b.p - a.p;
      float L = sqrtf(dot3(dv, dv));
      float3 dir = dv * (1.0f / L);
      bool occ = occluded_dyn(S, Fb, a.p, dir, S.eps, L - S.eps, a.tri, b.tri);
      Cross c = S.n_moved > 0 ? crossings(S, Fb, a.p, dir, S.eps, L - S.eps, L) : cross_zero();
      o.qc.inst++;
      if (occ && m + 1 < reject_from) { reject_from = m + 1; reject_reason = RJ_OCCLUDED; }
      if (edited(S, b.obj) && m + 1 < reject_from) { reject_from = m + 1; reject_reason = RJ_SUFFIX_DYN; }
      Q.v[m + 1] = b;
      Q.ex[m + 1] = c;
      Q.n = m + 1;
      if (m == w + 1) {
        R2 = area_pdf(S, Fb, Q.v[w], a, b) / area_pdf(S, F, P.v[w], a, b);
      }
    }
    rdiv = div_m;
    if (recon == 1 && m >= w + 1 && !gotP) break;
    if (Pend && (A.two_way || Qend || recon != 0)) break;
  }
}

// ------------------------------------------------------------------------------------------------
// two-ended techniques T3 / T6: pure replay
// ------------------------------------------------------------------------------------------------
struct Side {  // one sub-walk with its per-vertex connection
  PV v[RR_MAXV - 2];
  Cross ex[RR_MAXV - 2];
  Cross cc[RR_MAXV - 2];  // connection-edge crossings (sensor: from v toward E; NEE: from v toward L)
  PV L[RR_MAXV - 2];      // NEE vertex (emitter side)
  int pix[RR_MAXV - 2];   // sensor pixel (sensor side), -1 if none
  uint8_t vis[RR_MAXV - 2];
  int n;
};
struct Bidir {
  bool ok;
  PV start;
  Side A, B;  // A: sensor side (slots t), B: emitter side (slots 16 + s)
};

__device__ void extend_side(const DevScene& S, int F, const Rng& rng, Side& W, int slot0, int nmax, QCount& qc) {
  while (W.n < nmax) {
    int m = W.n;
    float d[8];
    rng.dims((uint32_t)(slot0 + m), d);
    Mat mt = load_mat(S, (uint32_t)W.v[m].obj, F);
    float3 wo;
    if (!bsdf_sample(mt, W.v[m].n, norm3_exact(W.v[m - 1].p - W.v[m].p), d[1], d[2], wo)) break;
    Trace2 t = trace2(S, W.v[m].p, wo, W.v[m].tri, F == 0, F == 1, qc);
    if (!t.ok[F]) break;
    W.v[m + 1] = t.v[F];
    W.ex[m + 1] = t.c[F];
    W.n = m + 1;
  }
}

__device__ void gen_bidir(const DevScene& S, const KArgs& A, int tech, int F, const Rng& rng, Bidir& G, QCount& qc) {
  G.ok = false;
  G.A.n = G.B.n = 0;
  const int D = A.max_depth;
  float d0[8];
  rng.dims(0, d0);
  int nmax;
  if (tech == 3) {
    if (S.n_edited == 0 || D < 4) return;
    PV xd = sample_set(S, S.edited_tris, S.edited_cdf, S.n_edited, F, d0[0], d0[1], d0[2]);
    float r = sqrtf(d0[3]), s, c;
    sincosf(2.0f * RR_PI_F * d0[4], &s, &c);
    float3 wl = norm3_exact(to_world(xd.n, r * c, r * s, sqrtf(fmaxf(0.0f, 1.0f - d0[3]))));
    Mat mt = load_mat(S, (uint32_t)xd.obj, F);
    float3 we;
    if (!bsdf_sample(mt, xd.n, wl, d0[6], d0[7], we)) return;
    Trace2 ty = trace2(S, xd.p, wl, xd.tri, F == 0, F == 1, qc);
    if (!ty.ok[F]) return;
    Trace2 tz = trace2(S, xd.p, we, xd.tri, F == 0, F == 1, qc);
    if (!tz.ok[F]) return;
    G.start = xd;
    G.B.v[0] = xd; G.B.v[1] = ty.v[F]; G.B.ex[1] = ty.c[F]; G.B.n = 1;
    G.A.v[0] = xd; G.A.v[1] = tz.v[F]; G.A.ex[1] = tz.c[F]; G.A.n = 1;
    nmax = D - 3;
  } else {
    if (S.n_moved == 0 || D < 3) return;
    PV xg = sample_set(S, S.moved_tris, S.moved_cdf, S.n_moved, 1 - F, d0[0], d0[1], d0[2]);
    float z = 1.0f - 2.0f * d0[3];
    float rr = 2.0f * sqrtf(d0[3] * (1.0f - d0[3])), s, c;  // sqrt(1 - z^2) = 2 sqrt(u (1-u)), no cancellation
    sincosf(2.0f * RR_PI_F * d0[4], &s, &c);
    float3 dir = f3(rr * c, rr * s, z);
    Trace2 ty = trace2(S, xg.p, dir, -1, F == 0, F == 1, qc);
    if (!ty.ok[F]) return;
    Trace2 tz = trace2(S, xg.p, dir * -1.0f, -1, F == 0, F == 1, qc);
    if (!tz.ok[F]) return;
    PV y1 = ty.v[F], z1 = tz.v[F];
    // crossings of the whole edge (z_1, y_1), which passes through x_G
    float3 dv = z1.p - y1.p;
    float L = sqrtf(dot3(dv, dv));
    Cross cyz = (S.n_moved > 0 && L > 2.0f * S.eps) ? crossings(S, F, y1.p, dv * (1.0f / L), S.eps, L - S.eps, L) : cross_zero();
    qc.inst++;
    G.start = xg;
    G.A.v[0] = y1; G.A.v[1] = z1; G.A.ex[1] = cyz; G.A.n = 1;
    G.B.v[0] = z1; G.B.v[1] = y1; G.B.ex[1] = swapc(cyz); G.B.n = 1;
    nmax = D - 2;
  }
  G.ok = true;
  extend_side(S, F, rng, G.A, 0, nmax, qc);
  extend_side(S, F, rng, G.B, 16, nmax, qc);
  PV E = cam_pv(S);
  for (int t = 1; t <= G.A.n; ++t) {  // sensor connections
    const PV& z = G.A.v[t];
    G.A.pix[t] = project(S, z.p);
    Seg2 s = seg2(S, z.p, E.p, z.tri, -1, F == 0, F == 1, qc);
    G.A.vis[t] = s.vis[F];
    G.A.cc[t] = s.c[F];
  }
  for (int sdx = 1; sdx <= G.B.n; ++sdx) {  // NEE, slot 16 + s
    const PV& y = G.B.v[sdx];
    float d[8];
    rng.dims((uint32_t)(16 + sdx), d);
    PV L = sample_emitter(S, d[3], d[4], d[5], d[6]);
    G.B.L[sdx] = L;
    Seg2 s = seg2(S, y.p, L.p, y.tri, L.tri, F == 0, F == 1, qc);
    G.B.vis[sdx] = s.vis[F];
    G.B.cc[sdx] = s.c[F];
  }
}

// path (E, z_t..z_1, [x_D], y_1..y_s, L) of a two-ended sample
__device__ int bidir_path(const Bidir& G, int tech, int t, int s, const DevScene& S, PV* x, Cross* ce) {
  int k = 0;
  x[k] = cam_pv(S);
  ce[k] = swapc(G.A.cc[t]);
  ++k;
  for (int j = t; j >= 1; --j) {
    x[k] = G.A.v[j];
    if (j >= 2) ce[k] = swapc(G.A.ex[j]);
    ++k;
  }
  if (tech == 3) {
    ce[k - 1] = swapc(G.A.ex[1]);  // (z_1, x_D)
    x[k] = G.start;
    ce[k] = G.B.ex[1];             // (x_D, y_1)
    ++k;
  } else {
    ce[k - 1] = G.B.ex[1];         // (z_1, y_1) through x_G
  }
  for (int j = 1; j <= s; ++j) {
    x[k] = G.B.v[j];
    ce[k] = (j < s) ? G.B.ex[j + 1] : G.B.cc[s];
    ++k;
  }
  x[k] = G.B.L[s];
  ++k;
  return k;
}

__device__ void sample_bidir(const DevScene& S, const KArgs& A, uint64_t i, const Rng& rng, Out& o) {
  const int F = A.side, Fb = 1 - A.side;
  const int l = A.tech;
  Bidir P, Q;
  gen_bidir(S, A, l, F, rng, P, o.qc);
  gen_bidir(S, A, l, Fb, rng, Q, o.qc);
  if (!P.ok && (A.two_way || !Q.ok)) return;
  const int extra = (l == 3) ? 2 : 1;
  const int D = A.max_depth;
  PV x[RR_MAXV + 2];
  Cross ce[RR_MAXV + 2];
  // divergence / dynamic-vertex prefix data per side
  bool sdiff = P.ok && Q.ok && (l == 3) && !same_pv(S, P.start, Q.start);
  int nA = P.ok ? P.A.n : 0, nB = P.ok ? P.B.n : 0;
  int mA = Q.ok ? Q.A.n : 0, mB = Q.ok ? Q.B.n : 0;
  int NA = max(nA, mA), NB = max(nB, mB);
  for (int t = 1; t <= NA; ++t) {
    for (int s = 1; s <= NB; ++s) {
      if (t + s + extra > D) continue;
      bool pc = t <= nA && s <= nB;
      bool qc_ = t <= mA && s <= mB;
      if (!pc && (A.two_way || !qc_)) continue;
      float3 vp = f3(0.f, 0.f, 0.f), vq = vp;
      int pixp = -1, pixq = -1;
      if (pc) {
        pixp = P.A.pix[t];
        if (P.A.vis[t] && P.B.vis[s]) {
          int k = bidir_path(P, l, t, s, S, x, ce);
          vp = path_value(S, x, ce, k, F, A.mask);
        }
      }
      if (qc_) {
        pixq = Q.A.pix[t];
        if (Q.A.vis[t] && Q.B.vis[s]) {
          int k = bidir_path(Q, l, t, s, S, x, ce);
          vq = path_value(S, x, ce, k, Fb, A.mask);
        }
      }
      if (pc) {
        int st = qc_ ? ST_ACCEPTED : ST_UNPAIRED, rs = RJ_NONE;
        if (st == ST_ACCEPTED && A.reject_multi) {
          bool dv = sdiff;
          int dp = (l == 3) ? 1 : 0, dq = dp;
          for (int j = (l == 3 ? 1 : 0); j <= t; ++j) {
            if (!same_pv(S, P.A.v[j], Q.A.v[j])) dv = true;
            if (j >= 1) { dp += edited(S, P.A.v[j].obj); dq += edited(S, Q.A.v[j].obj); }
          }
          for (int j = 1; j <= s; ++j) {
            if (!same_pv(S, P.B.v[j], Q.B.v[j])) dv = true;
            dp += edited(S, P.B.v[j].obj);
            dq += edited(S, Q.B.v[j].obj);
          }
          if (dv && (dp >= 2 || dq >= 2)) { st = ST_REJECTED; rs = RJ_MULTI; }
        }
        finish(o, i, 3, t, s, st, rs, pixp, vp, pixq, vq, 1.0f);
      } else {
        finish(o, i, 3, t, s, ST_MAPPED_ONLY, RJ_NONE, -1, f3(0.f, 0.f, 0.f), pixq, vq, 1.0f);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// kernel: grid-stride over this shard's samples of one (technique, side)
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void warp_add(unsigned long long* p, uint32_t v) {
  uint32_t s = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(p, (unsigned long long)s);
}

__global__ void __launch_bounds__(128) k_residual(const __grid_constant__ DevScene S, const __grid_constant__ KArgs A) {
  Out o;
  o.A = &A;
  o.qc.closest = o.qc.shadow = o.qc.inst = 0;
  o.conns = o.acc = o.rej = o.unp = o.monly = o.recon = o.splats = o.offscreen = o.zero = 0;
  for (int r = 0; r < 6; ++r) o.rejby[r] = 0;
  uint32_t nsamp = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t base = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // all lanes iterate the same number of times (warp-synchronous reductions at the end)
  for (uint64_t li = base; li - threadIdx.x % 32 < A.n_local; li += stride) {
    if (li >= A.n_local) continue;
    uint64_t i;
    if (A.dump) {
      i = A.i_begin + li;
    } else {
      uint64_t blk = li >> 16, off = li & 0xFFFFull;
      i = ((blk * A.shard_count + A.shard_index) << 16) | off;
      if (i >= A.n_total) continue;
    }
    Rng rng;
    rng.i_lo = (uint32_t)i;
    rng.i_hi = (uint32_t)(i >> 32);
    rng.ls = (uint32_t)A.tech | ((uint32_t)A.side << 8);
    rng.k0 = (uint32_t)A.seed;
    rng.k1 = (uint32_t)(A.seed >> 32);
    nsamp++;
    if (A.tech == 3 || A.tech == 6) sample_bidir(S, A, i, rng, o);
    else sample_single(S, A, i, rng, o);
  }
  unsigned long long* st = A.stats;
  warp_add(st + STAT_SAMPLES, nsamp);
  warp_add(st + STAT_CONNECTIONS, o.conns);
  warp_add(st + STAT_ACCEPTED, o.acc);
  warp_add(st + STAT_REJECTED, o.rej);
  warp_add(st + STAT_UNPAIRED, o.unp);
  warp_add(st + STAT_MAPPED_ONLY, o.monly);
  warp_add(st + STAT_CLOSEST, o.qc.closest);
  warp_add(st + STAT_SHADOW, o.qc.shadow);
  warp_add(st + STAT_INST, o.qc.inst);
  warp_add(st + STAT_SPLATS, o.splats);
  warp_add(st + STAT_OFFSCREEN, o.offscreen);
  warp_add(st + STAT_ZERO, o.zero);
  for (int r = 0; r < 6; ++r) warp_add(st + STAT_REJBY + r, o.rejby[r]);
}

__global__ void k_philox(uint32_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint4 c = make_uint4(ctr[4 * t], ctr[4 * t + 1], ctr[4 * t + 2], ctr[4 * t + 3]);
  uint4 r = philox4x32_10(c, make_uint2(k0, k1));
  out[4 * t] = r.x; out[4 * t + 1] = r.y; out[4 * t + 2] = r.z; out[4 * t + 3] = r.w;
}

__global__ void k_trace(const __grid_constant__ DevScene S, int F, uint32_t n, const float* rays, float* hits) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const float* r = rays + 8 * t;
  float3 o = f3(r[0], r[1], r[2]);
  float3 d = norm3_exact(f3(r[3], r[4], r[5]));
  int excl = __float_as_int(r[6]);
  QCount qc;
  Trace2 tr = trace2(S, o, d, excl, F == 0, F == 1, qc);
  float* h = hits + 8 * t;
  if (!tr.ok[F]) {
    h[0] = -1.0f;
    return;
  }
  const PV& v = tr.v[F];
  float3 q = v.p - o;
  h[0] = sqrtf(dot3(q, q));
  h[1] = __int_as_float(v.tri);
  h[2] = v.p.x; h[3] = v.p.y; h[4] = v.p.z;
  h[5] = v.n.x; h[6] = v.n.y; h[7] = v.n.z;
}

__global__ void k_segment(const __grid_constant__ DevScene S, uint32_t n, const float* segs, float* out) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const float* s = segs + 6 * t;
  QCount qc;
  Seg2 r = seg2(S, f3(s[0], s[1], s[2]), f3(s[3], s[4], s[5]), -1, -1, true, true, qc);
  float* o = out + 10 * t;
  for (int F = 0; F < 2; ++F) {
    o[5 * F] = r.vis[F] ? 1.0f : 0.0f;
    o[5 * F + 1] = r.c[F].n;
    o[5 * F + 2] = r.c[F].s0;
    o[5 * F + 3] = r.c[F].sa;
    o[5 * F + 4] = r.c[F].sb;
  }
}

// ---- host launchers
void launch_residual(const DevScene& S, const KArgs& A, int grid, cudaStream_t st) {
  k_residual<<<grid, 128, 0, st>>>(S, A);
}
void launch_philox(uint32_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out, cudaStream_t st) {
  k_philox<<<(n + 255) / 256, 256, 0, st>>>(n, ctr, k0, k1, out);
}
void launch_trace(const DevScene& S, int F, uint32_t n, const float* rays, float* hits, cudaStream_t st) {
  k_trace<<<(n + 127) / 128, 128, 0, st>>>(S, F, n, rays, hits);
}
void launch_segment(const DevScene& S, uint32_t n, const float* segs, float* out, cudaStream_t st) {
  k_segment<<<(n + 127) / 128, 128, 0, st>>>(S, n, segs, out);
}

}  // namespace rr
