// rr_shade.cuh -- path vertices, area sampling, BSDF-driven pdfs, the MIS-weighted value of a connection
// path (ratio form) and the splat / record sink.  Shared by the residual kernels (rr_residual.cu).
#pragma once
#include "rr_device.cuh"
#include "rr_kernels.h"

namespace rr {

enum { ST_ACCEPTED = 0, ST_REJECTED = 1, ST_UNPAIRED = 2, ST_MAPPED_ONLY = 3 };
enum { RJ_NONE = 0, RJ_OCCLUDED = 1, RJ_JACOBIAN = 2, RJ_MULTI = 3, RJ_TARGET = 4, RJ_SUFFIX_DYN = 5 };

struct PV {  // path vertex in one state
  P3 p;          // position (fp64, see rr_device.cuh)
  float3 n;
  int tri, obj;  // tri = -1: camera; obj = -1: camera
};

// forward declaration of the object flags lookup used below
__device__ __forceinline__ uint32_t oflags(const DevScene& S, int obj);
// base and mapped vertices coincide iff same primitive, same point, and not on a MOVED object (a vertex
// on a moved object lies on a different hit instance in each state)
__device__ __forceinline__ bool same_pv(const DevScene& S, const PV& a, const PV& b) {
  if (oflags(S, a.obj) & OBJ_MOVED) return false;
  return a.tri == b.tri && eqp(a.p, b.p) && eq3(a.n, b.n);
}
__device__ __forceinline__ PV cam_pv(const DevScene& S) {
  PV v;
  v.p = p3(S.cam_pos);
  v.n = S.cf;
  v.tri = -1;
  v.obj = -1;
  return v;
}
__device__ __forceinline__ uint32_t oflags(const DevScene& S, int obj) { return obj < 0 ? 0u : __ldg(&S.obj_flags[obj]); }
__device__ __forceinline__ bool edited(const DevScene& S, int obj) { return (oflags(S, obj) & OBJ_EDITED) != 0u; }

// hit -> vertex in state F: the fp64 intersection of the ray (o, d) with the hit triangle's plane
__device__ __forceinline__ PV hit_pv(const DevScene& S, const Hit& h, P3 o, float3 d, int F) {
  PV v;
  const float4* tp = S.ltris + 3 * h.leaf;
  float4 a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
  float3 n = cross3(f3(b.x - a.x, b.y - a.y, b.z - a.z), f3(c.x - a.x, c.y - a.y, c.z - a.z));
  {
    P3 A = make_double3(a.x, a.y, a.z), B = make_double3(b.x, b.y, b.z), C = make_double3(c.x, c.y, c.z);
    if (h.inst >= 0) {
      const float* M = S.inst[h.inst].M[F];
      A = xf_point_d(M, A);
      B = xf_point_d(M, B);
      C = xf_point_d(M, C);
    }
    double e1x = B.x - A.x, e1y = B.y - A.y, e1z = B.z - A.z, e2x = C.x - A.x, e2y = C.y - A.y, e2z = C.z - A.z;
    double nx = e1y * e2z - e1z * e2y, ny = e1z * e2x - e1x * e2z, nz = e1x * e2y - e1y * e2x;
    double den = nx * d.x + ny * d.y + nz * d.z;
    double t = (den != 0.0) ? (nx * (A.x - o.x) + ny * (A.y - o.y) + nz * (A.z - o.z)) / den : (double)h.t;
    v.p = make_double3(o.x + t * d.x, o.y + t * d.y, o.z + t * d.z);
  }
  if (h.inst >= 0) n = xf_vec(S.inst[h.inst].M[F], n);
  v.n = norm3_exact(n);
  v.tri = __float_as_int(a.w);
  v.obj = (int)__ldg(&S.tri_obj[v.tri]);
  return v;
}

// area-uniform point on a triangle set (C3): first k with cdf[k] > u0; su = sqrt(u1); b0 = 1-su; b1 = u2 su
__device__ inline PV sample_set(const DevScene& S, const uint32_t* tris, const float* cdf, int n, int F, float u0, float u1,
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
  P3 x = make_double3((double)a.x * b0 + (double)b.x * b1 + (double)c.x * b2, (double)a.y * b0 + (double)b.y * b1 + (double)c.y * b2,
                      (double)a.z * b0 + (double)b.z * b1 + (double)c.z * b2);
  float3 nrm = cross3(f3(b.x - a.x, b.y - a.y, b.z - a.z), f3(c.x - a.x, c.y - a.y, c.z - a.z));
  int obj = (int)__ldg(&S.tri_obj[tri]);
  int k = __ldg(&S.obj_inst[obj]);
  if (k >= 0) {
    x = xf_point_d(S.inst[k].M[F], x);
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

__device__ __forceinline__ Cross swapc(Cross c) {
  float t = c.sa;
  c.sa = c.sb;
  c.sb = t;
  return c;
}

// area pdf of generating `to` from `from` with the walk arriving from `prev` (state F)
__device__ __forceinline__ float area_pdf(const DevScene& S, int F, const PV& prev, const PV& from, const PV& to) {
  Mat m = load_mat(S, (uint32_t)from.obj, F);
  float3 wi = norm3_exact(sub3(prev.p, from.p));
  float3 dv = sub3(to.p, from.p);
  float d2 = dot3(dv, dv);
  float3 wo = dv * (1.0f / sqrtf(d2));
  return bsdf_pdf(m, from.n, wi, wo) * fabsf(dot3(to.n, wo)) / d2;
}

// ------------------------------------------------------------------------------------------------
// value of a connection path v = f / Pi (Eq.2; balance heuristic P:L351-353), in state F.
// x[0] = E, x[k-1] = L; e[i] = crossings of edge (x_i, x_{i+1}) with sa measured from x_i, sb from x_{i+1}.
// Computed as (f / p_T7) / (1 + sum_c p_c / p_T7).  mask bit 8 (RR_NO_PATH_MAPPING): a static path (no vertex
// on an edited object, no ghost crossing on any edge) has value 0.
// ------------------------------------------------------------------------------------------------
template <class Path>
__device__ inline float3 path_value_t(const DevScene& S, const Path& px, int k, int F, uint32_t mask) {
  const float3 zero = f3(0.f, 0.f, 0.f);
  float3 d01 = sub3(px.v(1).p, px.v(0).p);
  float dd01 = dot3(d01, d01);
  float3 w01 = d01 * (1.0f / sqrtf(dd01));
  float cth = dot3(w01, S.cf);
  if (!(cth > 0.0f)) return zero;
  const PV& L = px.v(k - 1);
  float4 le4 = __ldg(&S.obj_emit[L.obj]);
  float3 Le = f3(le4.x, le4.y, le4.z);
  if (!(dot3(L.n, sub3(px.v(k - 2).p, L.p)) > 0.0f)) return zero;  // front face only
  const bool reject_static = (mask & 0x100u) != 0;
  bool dyn_any = px.c(0).n > 0.0f;
  if (k == 2) return (reject_static && !dyn_any) ? zero : Le;  // direct view: W_e G / p_cam = 1, Pi = p_T7
  float cos1 = fabsf(dot3(px.v(1).n, w01));
  float invpcam = S.Aplane * cth * cth * cth * dd01 / cos1;  // 1 / p_cam(x_1)
  float pL = __ldg(&S.emit_pL[__ldg(&S.obj_emitter[L.obj])]);
  const bool t1 = mask & 1u, t2 = mask & 2u, t3 = mask & 4u, t4 = mask & 8u, t5 = mask & 16u, t6 = mask & 32u;
  float3 T = f3(1.f, 1.f, 1.f);
  float sum = 1.0f;  // T7
  if (t5 && px.c(0).n > 0.0f) sum += S.pA_G * S.Aplane * cth * cth * cth * px.c(0).sa;
  float Q = 1.0f;  // prod_{m < i} rev_m / fwd_{m+1}
  for (int i = 1; i <= k - 2; ++i) {
    Mat m = load_mat(S, (uint32_t)px.v(i).obj, F);
    float3 wi = norm3_exact(sub3(px.v(i - 1).p, px.v(i).p));
    float3 dv = sub3(px.v(i + 1).p, px.v(i).p);
    float d2 = dot3(dv, dv);
    float3 wo = dv * (1.0f / sqrtf(d2));
    float3 rho = bsdf_eval(m, px.v(i).n, wi, wo);
    float pf = bsdf_pdf(m, px.v(i).n, wi, wo);
    float cout = fabsf(dot3(px.v(i).n, wo));
    float cin_next = fabsf(dot3(px.v(i + 1).n, wo));
    bool dyn = edited(S, px.v(i).obj);
    dyn_any = dyn_any || dyn || px.c(i).n > 0.0f;
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
      else if (t3) sum += base * (fmaxf(0.0f, dot3(px.v(i).n, wo)) * RR_INV_PI_F) / pf;  // T3
    }
    if (px.c(i).n > 0.0f) {
      if (i + 1 == k - 1) { if (t4) sum += S.pA_G * px.c(i).sb * cout / d2 * invpcam * Q; }  // T4 (Eq. vertex1pdf)
      else if (t6) sum += S.pA_G * (0.25f * RR_INV_PI_F) * px.c(i).s0 * cout / pf * invpcam * Q;  // T6
    }
    if (i <= k - 3) {  // q_i = rev_i / fwd_{i+1} on edge (i, i+1)
      Mat mn = load_mat(S, (uint32_t)px.v(i + 1).obj, F);
      float pr = bsdf_pdf(mn, px.v(i + 1).n, norm3_exact(sub3(px.v(i + 2).p, px.v(i + 1).p)), wo * -1.0f);
      Q *= pr * cout / (pf * cin_next);
    }
  }
  if (reject_static && !dyn_any) return zero;
  return T * (1.0f / sum);
}

// the connection path as two contiguous arrays x[0..k-1], e[0..k-2]
struct PathArrays {
  const PV* x;
  const Cross* e;
  __device__ __forceinline__ const PV& v(int i) const { return x[i]; }
  __device__ __forceinline__ Cross c(int i) const { return e[i]; }
};
__device__ inline float3 path_value(const DevScene& S, const PV* x, const Cross* e, int k, int F, uint32_t mask) {
  return path_value_t(S, PathArrays{x, e}, k, F, mask);
}

// ------------------------------------------------------------------------------------------------
// splat + records + statistics
// ------------------------------------------------------------------------------------------------
#ifndef RR_SPLAT_MATCH
#define RR_SPLAT_MATCH 0  // 1: warp-aggregated splat (tools/variants.py knob; measured)
#endif
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
#if RR_SPLAT_MATCH
  // warp-aggregated splat (measured and rejected): the lanes splatting in this
  // instruction are grouped by pixel (__match_any_sync), each group's terms are summed by a rank-ordered
  // shuffle tree and the group's lowest lane issues one atomicAdd
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, pix);
  if (__any_sync(act, peers & (peers - 1))) {  // some group has more than one lane
    const unsigned lane = threadIdx.x & 31u;
    const unsigned rank = __popc(peers & ((1u << lane) - 1u));
    const unsigned cnt = __popc(peers);
    for (unsigned step = 1; step < 32; step <<= 1) {
      if (!__any_sync(act, step < cnt)) break;
      // the lane of rank (rank + step) in my group, if any
      unsigned above = peers >> lane >> 1;  // peers above me, bit 0 = lane + 1
      int src = -1;
      if ((rank & (2 * step - 1)) == 0 && rank + step < cnt) {
        unsigned m = above;
        for (unsigned k = 1; k < step; ++k) m &= m - 1;  // drop the (step - 1) nearest peers above
        src = (int)lane + __ffs(m);
      }
      float x = __shfl_sync(act, t.x, src < 0 ? (int)lane : src);
      float y = __shfl_sync(act, t.y, src < 0 ? (int)lane : src);
      float z = __shfl_sync(act, t.z, src < 0 ? (int)lane : src);
      if (src >= 0) { t.x += x; t.y += y; t.z += z; }
    }
    if (rank != 0) return;
  }
#endif
  atomicAdd(reinterpret_cast<float4*>(o.A->image) + pix, make_float4(t.x, t.y, t.z, 0.0f));
}
__device__ inline void emit_record(Out& o, uint64_t i, int kind, int a, int b, int status, int reason, int pix_p, float3 tp,
                            int pix_q, float3 tq, float R) {
  const KArgs& A = *o.A;
  if (status == ST_ACCEPTED) {
    o.acc++;
    if (R != 1.0f) atomicAdd(A.stats + STAT_RHIST + min(max(ilogbf(R) + 8, 0), 15), 1ull);  // R histogram (rare)
  }
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
__device__ inline void finish(Out& o, uint64_t i, int kind, int a, int b, int status, int reason, int pix_p, float3 vp,
                       int pix_q, float3 vq, float R) {
  const KArgs& A = *o.A;
  float3 tp, tq;
  if (A.diag) {  // diagnostic one-way ablation: weight 1 for every base term, the partner only when accepted
    tp = vp * A.inv_spp;
    tq = (status == ST_ACCEPTED) ? vq * (-A.inv_spp * R) : f3(0.f, 0.f, 0.f);
    if (status != ST_ACCEPTED) pix_q = -1;
  } else if (A.two_way) {
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


}  // namespace rr
