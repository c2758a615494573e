// rr_residual.cu -- the residual path integral estimator on the GPU (sm_100a).
//
// One residual sample = one technique invocation (technique l, side s, index i).  The
// base path is generated in state F = side, the mapped path in Fbar with the same Philox counters
// (random-seed replay) by the paired technique (dynamic<->ghost pair T2<->T5).
//
// Execution model (B200): persistent lanes, each running a sample as a state machine.  Every step a lane
// consumes the results of the ray queries it issued in the previous step, advances its sample (shading,
// MIS, mapping, splat) and issues the next batch of queries (<= NQ).  The queries of all lanes then run
// through run_query(), the kernel's single traversal site (rr_query.cuh), so divergent samples still
// traverse in SIMT lockstep.  A lane whose sample finishes refills from a global sample counter
// (warp-aggregated atomics): finished paths never occupy a lane ("compaction + refill", A9).
//
// The two walks of a single-walk sample run in lockstep so that the static-BLAS traversal is shared while
// they have not diverged (A3), the reconnection ("keep vertex the same") is decided at the first
// diverged rough vertex, and connections are evaluated and splatted as soon as they are formed.
#ifndef RR_VNDF_KERNELS
#define RR_VNDF_KERNELS 0  // 1: this TU is the RR_VNDF instantiation (rr_residual_vndf.cu)
#endif
#ifndef RR_VAR_KERNELS
#define RR_VAR_KERNELS 0  // 1: this TU is the mapping-variants instantiation (rr_residual_var.cu)
#endif
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#if !RR_VNDF_KERNELS && !RR_VAR_KERNELS
#include <cub/device/device_radix_sort.cuh>  // sample_order (T3 / T6 processing order)
#endif

#include "rr_device.cuh"
#include "rr_kernels.h"
#include "rr_query.cuh"
#include "rr_shade.cuh"

namespace rr {
// the state machines and kernels live in a namespace per instantiation: kplain (default) and kvndf (GGX
// visible-normal sampling compiled in), so that the default kernels carry no code of the variant
#if RR_VNDF_KERNELS
namespace kvndf {
#elif RR_VAR_KERNELS
namespace kvar {
#else
namespace kplain {
#endif
// RR_T6_TOWARD_LIGHT (kvar only): the path runs this query's edge against its direction (crossing p_dir)
#if RR_VAR_KERNELS
__device__ __forceinline__ Query orient(Query q, bool rev) {
  q.rev = rev ? 1 : 0;
  return q;
}
#define RR_ORIENT(q, rev) orient(q, rev)
#else
#define RR_ORIENT(q, rev) (q)
#endif

#define NQ 10
#define FULLMASK 0xffffffffu

struct Batch {  // the query batch of one lane (thread-local)
  Query q[NQ];
  QRes r[NQ];
  int n;
  __device__ __forceinline__ int push(const Query& x) {
    q[n] = x;
    return n++;
  }
};
__device__ __forceinline__ int bit(int F) { return 1 << F; }

// ------------------------------------------------------------------------------------------------
// single-walk techniques: T7, T1, T2, T4, T5  (E-rooted: T7, T2, T5; L-rooted: T1, T4)
// ------------------------------------------------------------------------------------------------
struct SWalk {
  PV v[RR_MAXV];
  Cross ex[RR_MAXV];  // ex[m]: crossings of the walk edge v[m-1] -> v[m], sa measured from v[m-1]
  int n;              // number of walk vertices (0: the technique failed)
  int pixel;          // fixed pixel (T7, T2, T5)
};
// the connection path of a single walk read in place (no copy into path arrays): E-rooted (T7 / T2 / T5)
// (E, v_1..v_m, L) or L-rooted (T1 / T4) (E, v_m..v_1, x_L); cn = the connection edge's crossings as queried
// (from v_m toward L, or from v_m toward E)
struct SPathView {
  const SWalk* W;
  const PV* E;
  const PV* L;
  Cross cn;
  int m;
  bool lroot;
  __device__ __forceinline__ const PV& v(int i) const {
    if (i == 0) return *E;
    if (i <= m) return lroot ? W->v[m + 1 - i] : W->v[i];
    return lroot ? W->v[0] : *L;
  }
  __device__ __forceinline__ Cross c(int i) const {
    if (!lroot) return i < m ? W->ex[i + 1] : cn;
    return i == 0 ? swapc(cn) : swapc(W->ex[m + 1 - i]);
  }
};
struct SStart {  // start element of one side, kept between issue and consume
  PV a, b;
  float dl;
  float3 dir;
  int pix, qi;
};
struct SState {
  uint64_t i;
  Rng rng;
  int pc, m;
  SWalk P, Q;
  SStart sp, sq;
  int recon, w, reject_from, reject_reason;  // recon: 0 none, 1 reconnected, 2 failed, 3 pending visibility
  float R1, R2;
  bool rdiv, hdiv, Pend, Qend, suffix_pending;
  int dynP, dynQ;
  // temporaries of the current step
  int q_recon, q_suffix, q_cp, q_cq, q_wp, q_wq;
  bool pc_, qc_, okP, okQ, walk_shared, attempt, qActive, div_m, has_conn;
  PV L;
  int pixp, pixq;
  float3 woP, woQ;
#if RR_VAR_KERNELS
  // RR_TOBJ_MIDPATH: walk index of the mapped vertex t(x_m) (0 none), its state (1 visibility pending, 2 mapped,
  // 3 occluded, 4 static base vertex with a replayed partner on a moved object) and R_T
  int tobj_m, tobj_st, q_tobj;
  float RT;
#endif
};

__device__ __forceinline__ bool nee_ok(int tech, int m) { return tech == 2 ? m >= 2 : true; }
// the sample's own ghost crossing on the queried edge (Query::seed_t; reading 12)
__device__ __forceinline__ Query seeded(Query q, float t, const PV& xg) {
  q.seed_t = t;
  q.seed_tri = xg.tri;
  return q;
}

// issue the start query of one side
__device__ void start_issue(const DevScene& S, int tech, int F, const float d0[8], SStart& s, Batch& B) {
  s.qi = -1;
  PV E = cam_pv(S);
  switch (tech) {
    case 1: {  // dynamic from emitter: x_D, x_L, "fails if blocked"
      if (S.n_edited == 0) return;
      s.b = sample_set(S, S.edited_tris, S.edited_cdf, S.n_edited, F, d0[0], d0[1], d0[2]);
      s.a = sample_emitter(S, d0[3], d0[4], d0[5], d0[6]);
      if (!(dot3(s.a.n, sub3(s.b.p, s.a.p)) > 0.0f)) return;
      s.qi = B.push(mk_seg(s.a.p, s.b.p, s.a.tri, s.b.tri, bit(F)));
      return;
    }
    case 2: {  // dynamic from sensor
      if (S.n_edited == 0) return;
      s.b = sample_set(S, S.edited_tris, S.edited_cdf, S.n_edited, F, d0[0], d0[1], d0[2]);
      s.pix = project(S, s.b.p);
      if (s.pix < 0) return;
      s.qi = B.push(mk_seg(E.p, s.b.p, -1, s.b.tri, bit(F)));
      return;
    }
    case 4: {  // ghost from emitter: x_G on ghost_F = moved objects at M_Fbar
      if (S.n_moved == 0) return;
      PV xg = sample_set(S, S.moved_tris, S.moved_cdf, S.n_moved, 1 - F, d0[0], d0[1], d0[2]);
      s.a = sample_emitter(S, d0[3], d0[4], d0[5], d0[6]);
      float3 dv = sub3(xg.p, s.a.p);
      s.dl = sqrtf(dot3(dv, dv));
      if (!(s.dl > S.eps)) return;
      s.dir = dv * (1.0f / s.dl);
      if (!(dot3(s.a.n, s.dir) > 0.0f)) return;
      s.b = xg;  // for its crossing (start_consume)
      s.qi = B.push(seeded(mk_ray(s.a.p, s.dir, s.a.tri, bit(F)), s.dl, xg));
      return;
    }
    case 5: {  // ghost from sensor
      if (S.n_moved == 0) return;
      PV xg = sample_set(S, S.moved_tris, S.moved_cdf, S.n_moved, 1 - F, d0[0], d0[1], d0[2]);
      s.pix = project(S, xg.p);
      if (s.pix < 0) return;
      float3 dv = sub3(xg.p, E.p);
      s.dl = sqrtf(dot3(dv, dv));
      s.dir = dv * (1.0f / s.dl);
      s.b = xg;
      s.qi = B.push(seeded(mk_ray(E.p, s.dir, -1, bit(F)), s.dl, xg));
      return;
    }
  }
}
__device__ void start_consume(const DevScene& S, int tech, int F, const SStart& s, const Batch& B, SWalk& W) {
  W.n = 0;
  W.pixel = -1;
  if (s.qi < 0) return;
  const QRes& r = B.r[s.qi];
  PV E = cam_pv(S);
  if (tech == 1 || tech == 2) {
    if (!r.ok[F]) return;
    W.v[0] = tech == 1 ? s.a : E;
    W.v[1] = s.b;
    W.ex[1] = r.c[F];
    W.n = 1;
    W.pixel = tech == 2 ? s.pix : -1;
  } else {
    if (!r.ok[F]) return;
    P3 o = tech == 4 ? s.a.p : E.p;
    PV h = hit_pv(S, r.h[F], o, s.dir, F);
    float3 q = sub3(h.p, o);
    if (!(sqrtf(dot3(q, q)) > s.dl + S.eps)) return;  // the first hit lies beyond x_G
    W.v[0] = tech == 4 ? s.a : E;
    W.v[1] = h;
    W.ex[1] = add_seed(r.c[F], s.dl, r.h[F].t, 1.0f / fabsf(dot3(s.b.n, s.dir)));  // + the crossing at x_G
    W.n = 1;
    W.pixel = tech == 5 ? s.pix : -1;
  }
}

// issue the queries of walk vertex m (connection at m, walk step from m, pending reconnection/suffix checks)
__device__ __forceinline__ void single_issue(const DevScene& S, const KArgs& A, SState& st, Batch& B) {
  const int F = A.side, Fb = 1 - F, l = A.tech, lq = A.tech_q, D = A.max_depth, m = st.m;
  const bool Lroot = (l == 1 || l == 4);
  const int maxW = D - 1 > 1 ? D - 1 : 1;
  SWalk& P = st.P;
  SWalk& Q = st.Q;
  PV E = cam_pv(S);
  st.q_recon = st.q_suffix = st.q_cp = st.q_cq = st.q_wp = st.q_wq = -1;
  bool hasP = m <= P.n, hasQ = m <= Q.n;
  bool vdiff = hasP && hasQ && !same_pv(S, P.v[m], Q.v[m]);
  st.hdiv = st.hdiv || vdiff || (hasP != hasQ);
  if (hasP && edited(S, P.v[m].obj)) st.dynP++;
  if (hasQ && edited(S, Q.v[m].obj)) st.dynQ++;
  if (st.recon == 3)
    st.q_recon = B.push(RR_ORIENT(mk_seg(Q.v[st.w].p, P.v[st.w + 1].p, Q.v[st.w].tri, P.v[st.w + 1].tri, bit(Fb)), Lroot));
#if RR_VAR_KERNELS
  st.q_tobj = -1;
  if (st.tobj_st == 1)  // x_{m-1} -> t(x_m) in View_Fbar, and the edge's ghost crossings for Q's MIS
    st.q_tobj = B.push(RR_ORIENT(mk_seg(Q.v[m - 1].p, Q.v[m].p, Q.v[m - 1].tri, Q.v[m].tri, bit(Fb)), Lroot));
#endif
  if (st.suffix_pending)
    st.q_suffix = B.push(RR_ORIENT(mk_seg(P.v[m - 1].p, P.v[m].p, P.v[m - 1].tri, P.v[m].tri, bit(Fb), true), Lroot));
  float d[8];
  st.rng.dims((uint32_t)m, d);
  // ---- connection at m
  st.has_conn = false;
  st.pc_ = st.qc_ = false;
  if (m + 1 <= D) {
    bool failed_q = (st.recon == 2 && m >= st.w + 1);
    if (!Lroot) {
      st.pc_ = hasP && nee_ok(l, m);
      st.qc_ = hasQ && nee_ok(lq, m) && !failed_q;
      if (st.pc_ || (st.qc_ && !A.two_way)) {
        st.has_conn = true;
        st.L = sample_emitter(S, d[3], d[4], d[5], d[6]);
        bool shared = st.pc_ && st.qc_ && same_pv(S, P.v[m], Q.v[m]);
        if (shared) {
          st.q_cp = st.q_cq = B.push(mk_seg(P.v[m].p, st.L.p, P.v[m].tri, st.L.tri, 3));
        } else {
          if (st.pc_) st.q_cp = B.push(mk_seg(P.v[m].p, st.L.p, P.v[m].tri, st.L.tri, bit(F)));
          if (st.qc_) st.q_cq = B.push(mk_seg(Q.v[m].p, st.L.p, Q.v[m].tri, st.L.tri, bit(Fb)));
        }
      }
    } else {
      st.pc_ = hasP;
      st.qc_ = hasQ && !failed_q;
      if (st.pc_ || (st.qc_ && !A.two_way)) {
        st.has_conn = true;
        st.pixp = st.pc_ ? project(S, P.v[m].p) : -1;
        st.pixq = st.qc_ ? project(S, Q.v[m].p) : -1;
        // a vertex that projects outside the image has a zero-valued sensor connection (reading 4): no query
        const bool tp = st.pc_ && st.pixp >= 0, tq = st.qc_ && st.pixq >= 0;
        bool shared = tp && tq && same_pv(S, P.v[m], Q.v[m]);
        if (shared) {
          st.q_cp = st.q_cq = B.push(mk_seg(P.v[m].p, E.p, P.v[m].tri, -1, 3));
        } else {
          if (tp) st.q_cp = B.push(mk_seg(P.v[m].p, E.p, P.v[m].tri, -1, bit(F)));
          if (tq) st.q_cq = B.push(mk_seg(Q.v[m].p, E.p, Q.v[m].tri, -1, bit(Fb)));
        }
      }
    }
  }
  // ---- walk step from v_m (slot m)
  st.okP = st.okQ = st.walk_shared = st.attempt = false;
  st.qActive = (st.recon == 0) && hasQ && !st.Qend;
  st.div_m = st.rdiv || vdiff;
  if (m < maxW) {
    Mat mp, mq;
    if (hasP && !st.Pend) {
      mp = load_mat(S, (uint32_t)P.v[m].obj, F);
      st.okP = bsdf_sample(mp, P.v[m].n, norm3_exact(sub3(P.v[m - 1].p, P.v[m].p)), d[1], d[2], st.woP);
    }
    if (st.qActive) {
      mq = load_mat(S, (uint32_t)Q.v[m].obj, Fb);
      st.okQ = bsdf_sample(mq, Q.v[m].n, norm3_exact(sub3(Q.v[m - 1].p, Q.v[m].p)), d[1], d[2], st.woQ);
    }
    bool dirdiv = st.qActive && hasP && !st.Pend && ((st.okP != st.okQ) || (st.okP && st.okQ && !eq3(st.woP, st.woQ)));
    st.div_m = st.rdiv || vdiff || dirdiv;
    st.walk_shared = st.qActive && st.okP && st.okQ && !vdiff && !dirdiv;
    st.attempt = A.reconnect && st.recon == 0 && st.qActive && hasP && st.div_m && rough_enough(mp, A.alpha_min) &&
                 rough_enough(mq, A.alpha_min);
    if (st.okP) st.q_wp = B.push(RR_ORIENT(mk_ray(P.v[m].p, st.woP, P.v[m].tri, bit(F) | (st.walk_shared ? bit(Fb) : 0)), Lroot));
    if (st.qActive && st.okQ && !st.walk_shared && !st.attempt)
      st.q_wq = B.push(RR_ORIENT(mk_ray(Q.v[m].p, st.woQ, Q.v[m].tri, bit(Fb)), Lroot));
  }
}

// consume the results of walk vertex m; returns false when the sample is finished
__device__ __forceinline__ bool single_consume(const DevScene& S, const KArgs& A, SState& st, const Batch& B, Out& o) {
  const int F = A.side, Fb = 1 - F, l = A.tech, D = A.max_depth, m = st.m;
  const bool Lroot = (l == 1 || l == 4);
  const int maxW = D - 1 > 1 ? D - 1 : 1;
  SWalk& P = st.P;
  SWalk& Q = st.Q;
  PV E = cam_pv(S);
  const uint64_t i = st.i;
  bool hasP = m <= P.n, hasQ = m <= Q.n;
#if RR_VAR_KERNELS
  if (st.q_tobj >= 0) {
    const QRes& r = B.r[st.q_tobj];
    st.tobj_st = r.ok[Fb] ? 2 : 3;
    Q.ex[m] = r.c[Fb];
    if (st.tobj_st == 3) st.Qend = true;  // no mapped path from x_m on
  }
#endif
  // ---- pending reconnection edge (checked in View_Fbar)
  if (st.q_recon >= 0) {
    const QRes& r = B.r[st.q_recon];
    if (!r.ok[Fb]) {
      st.recon = 2;
      if (st.w + 1 < st.reject_from) { st.reject_from = st.w + 1; st.reject_reason = RJ_OCCLUDED; }
    } else {
      st.recon = 1;
      Q.ex[st.w + 1] = r.c[Fb];
      o.recon++;
    }
  }
  // ---- shared suffix edge v_{m-1} -> v_m re-checked against dyn_Fbar only
  if (st.q_suffix >= 0) {
    const QRes& r = B.r[st.q_suffix];
    if (!r.ok[Fb] && m < st.reject_from) { st.reject_from = m; st.reject_reason = RJ_OCCLUDED; }
    Q.ex[m] = r.c[Fb];
    st.suffix_pending = false;
  }
  // ---- direct view of an emitter (T7 only, k = 2)
  if (l == 7 && m == 1) {
    bool pe = hasP && __ldg(&S.obj_emitter[P.v[1].obj]) >= 0;
    bool qe = hasQ && __ldg(&S.obj_emitter[Q.v[1].obj]) >= 0;
    float3 vp = f3(0.f, 0.f, 0.f), vq = vp;
    if (pe) vp = path_value_t(S, SPathView{&P, &E, nullptr, cross_zero(), 1, false}, 2, F, A.mask);
    if (qe) vq = path_value_t(S, SPathView{&Q, &E, nullptr, cross_zero(), 1, false}, 2, Fb, A.mask);
    if (pe) {
      int stt = qe ? ST_ACCEPTED : ST_UNPAIRED;
      if (stt == ST_ACCEPTED && A.reject_multi && st.hdiv && (st.dynP >= 2 || st.dynQ >= 2)) stt = ST_REJECTED;
      finish(o, i, 0, 1, 0, stt, stt == ST_REJECTED ? RJ_MULTI : RJ_NONE, P.pixel, vp, Q.pixel, vq, 1.0f);
    } else if (qe && !A.two_way) {
      finish(o, i, 0, 1, 0, ST_MAPPED_ONLY, RJ_NONE, -1, f3(0.f, 0.f, 0.f), Q.pixel, vq, 1.0f);
    }
  }
  // ---- connection at m
  if (st.has_conn) {
    const bool reconnected_here = (st.recon == 1 && m >= st.w + 1);
    bool qc_ = st.qc_ && !(st.recon == 2 && m >= st.w + 1) && !(reconnected_here && m >= st.reject_from);
    float3 vp = f3(0.f, 0.f, 0.f), vq = vp;
    int pixp, pixq;
    if (!Lroot) {
      pixp = P.pixel;
      pixq = Q.pixel;
      if (st.pc_ && B.r[st.q_cp].ok[F])
        vp = path_value_t(S, SPathView{&P, &E, &st.L, B.r[st.q_cp].c[F], m, false}, m + 2, F, A.mask);
      if (qc_ && B.r[st.q_cq].ok[Fb])
        vq = path_value_t(S, SPathView{&Q, &E, &st.L, B.r[st.q_cq].c[Fb], m, false}, m + 2, Fb, A.mask);
    } else {
      pixp = st.pixp;
      pixq = st.pixq;
      if (st.pc_ && st.q_cp >= 0 && B.r[st.q_cp].ok[F])
        vp = path_value_t(S, SPathView{&P, &E, nullptr, B.r[st.q_cp].c[F], m, true}, m + 2, F, A.mask);
      if (qc_ && st.q_cq >= 0 && B.r[st.q_cq].ok[Fb])
        vq = path_value_t(S, SPathView{&Q, &E, nullptr, B.r[st.q_cq].c[Fb], m, true}, m + 2, Fb, A.mask);
    }
    const int kind = Lroot ? 2 : 1;
    if (st.pc_) {
      int stt = ST_ACCEPTED, rs = RJ_NONE;
      float R = 1.0f;
#if RR_VAR_KERNELS
      const bool tobj_here = st.tobj_m > 0 && m >= st.tobj_m;
      if (tobj_here && st.tobj_st >= 3) { stt = ST_REJECTED; rs = st.tobj_st == 3 ? RJ_OCCLUDED : RJ_TARGET; }
      else
#endif
      if (st.recon == 2 && m >= st.w + 1) { stt = ST_REJECTED; rs = st.reject_reason; }
      else if (reconnected_here && m >= st.reject_from) { stt = ST_REJECTED; rs = st.reject_reason; }
      else if (!qc_) stt = ST_UNPAIRED;
      else if (reconnected_here) {
        R = st.R1 * (m >= st.w + 2 ? st.R2 : 1.0f);
        if (!(R > 0.0f) || !isfinite(R)) { stt = ST_REJECTED; rs = RJ_TARGET; }
      }
#if RR_VAR_KERNELS
      if (tobj_here && stt == ST_ACCEPTED) R *= st.RT;  // the object-transformed vertex (R_T; reading 18)
#endif
      if (stt == ST_ACCEPTED && A.reject_multi && st.hdiv && (st.dynP >= 2 || st.dynQ >= 2)) { stt = ST_REJECTED; rs = RJ_MULTI; }
      finish(o, i, kind, m, 0, stt, rs, pixp, vp, pixq, vq, R);
    } else if (qc_ && !A.two_way) {
      finish(o, i, kind, m, 0, ST_MAPPED_ONLY, RJ_NONE, -1, f3(0.f, 0.f, 0.f), pixq, vq, 1.0f);
    }
  }
  if (m >= maxW) return false;
  // ---- walk results
  bool gotP = false;
  if (st.okP) {
    const QRes& r = B.r[st.q_wp];
    if (r.ok[F]) {
      P.v[m + 1] = hit_pv(S, r.h[F], P.v[m].p, st.woP, F);
      P.ex[m + 1] = r.c[F];
      P.n = m + 1;
      gotP = true;
    }
    if (st.walk_shared) {
      if (r.ok[Fb]) {
        Q.v[m + 1] = hit_pv(S, r.h[Fb], Q.v[m].p, st.woQ, Fb);
        Q.ex[m + 1] = r.c[Fb];
        Q.n = m + 1;
      } else {
        st.Qend = true;
      }
#if RR_VAR_KERNELS
      // RR_TOBJ_MIDPATH: on the undiverged pair's first mid-path hit of a MOVED object the mapped
      // vertex is the same object-space point in Fbar, t(x) = M_Fbar M_F^-1 x (|t'| = 1), instead of the replayed
      // hit; a static base vertex whose replayed partner lies on a moved object rejects the pair from there on
      if (A.tobj && st.tobj_st == 0) {
        const bool pm = gotP && (oflags(S, P.v[m + 1].obj) & OBJ_MOVED);
        const bool qm = r.ok[Fb] && (oflags(S, Q.v[m + 1].obj) & OBJ_MOVED);
        if (pm) {
          const PV& x = P.v[m + 1];
          const DevInstance& I = S.inst[__ldg(&S.obj_inst[x.obj])];
          PV t = x;
          t.p = xf_point_d(I.M[Fb], xf_point_d(I.Mi[F], x.p));
          t.n = norm3_exact(xf_vec(I.M[Fb], xf_vec(I.Mi[F], x.n)));
          Q.v[m + 1] = t;
          Q.n = m + 1;
          st.Qend = false;
          st.tobj_m = m + 1;
          st.tobj_st = 1;  // visibility of Q.v[m] -> t with the next batch
          st.RT = area_pdf(S, Fb, Q.v[m - 1], Q.v[m], t) / area_pdf(S, F, P.v[m - 1], P.v[m], x);
          if (!(st.RT > 0.0f) || !isfinite(st.RT)) { st.tobj_st = 3; st.Qend = true; }
        } else if (qm) {
          st.tobj_m = m + 1;
          st.tobj_st = 4;
          st.Qend = true;
        }
      }
#endif
    }
  }
  if (hasP && !gotP) st.Pend = true;
  if (st.attempt) {
    // reconnection at w = m to the base vertex v_{m+1}
    st.w = m;
    if (!gotP) {
      st.recon = 2;
      st.reject_from = m + 1;
      st.reject_reason = RJ_TARGET;
    } else {
      const PV& vw = P.v[m];
      const PV& vq = Q.v[m];
      const PV& tg = P.v[m + 1];
      float3 a = sub3(vq.p, tg.p), b = sub3(vw.p, tg.p);
      float la2 = dot3(a, a), lb2 = dot3(b, b);
      int rs = RJ_NONE;
      if (edited(S, tg.obj)) rs = RJ_TARGET;                                                // (1) P:L406
      else if (!rough_enough(load_mat(S, (uint32_t)tg.obj, F), A.alpha_min)) rs = RJ_TARGET;  // (2) P:L408
      else if (fminf(sqrtf(lb2), sqrtf(la2)) < A.dmin) rs = RJ_TARGET;                     // (3) P:L410
      else {
        float Jg = fabsf(dot3(tg.n, a * (1.0f / sqrtf(la2)))) / fabsf(dot3(tg.n, b * (1.0f / sqrtf(lb2)))) * lb2 / la2;
        if (!(Jg <= A.jacobian_max && Jg >= 1.0f / A.jacobian_max)) rs = RJ_JACOBIAN;
      }
      if (rs == RJ_NONE) {
        st.R1 = area_pdf(S, Fb, Q.v[m - 1], vq, tg) / area_pdf(S, F, P.v[m - 1], vw, tg);
        st.recon = 3;  // visibility of v'_w -> v_{w+1} in View_Fbar is checked with the next batch
        Q.v[m + 1] = tg;
        Q.n = m + 1;
      } else {
        st.recon = 2;
        st.reject_from = m + 1;
        st.reject_reason = rs;
      }
    }
  } else if (st.qActive && !st.walk_shared) {
    if (st.okQ) {
      const QRes& r = B.r[st.q_wq];
      if (r.ok[Fb]) {
        Q.v[m + 1] = hit_pv(S, r.h[Fb], Q.v[m].p, st.woQ, Fb);
        Q.ex[m + 1] = r.c[Fb];
        Q.n = m + 1;
      } else {
        st.Qend = true;
      }
    } else {
      st.Qend = true;
    }
  } else if (st.recon == 1 && m >= st.w + 1 && gotP) {
    const PV& a = P.v[m];
    const PV& b = P.v[m + 1];
    st.suffix_pending = true;
    if (edited(S, b.obj) && m + 1 < st.reject_from) { st.reject_from = m + 1; st.reject_reason = RJ_SUFFIX_DYN; }
    Q.v[m + 1] = b;
    Q.n = m + 1;
    if (m == st.w + 1) st.R2 = area_pdf(S, Fb, Q.v[st.w], a, b) / area_pdf(S, F, P.v[st.w], a, b);
  }
  st.rdiv = st.div_m;
  if (st.recon == 1 && m >= st.w + 1 && !gotP) return false;
  if (st.Pend && (A.two_way || st.Qend || st.recon != 0)) return false;
  int mn = m + 1;
  bool hasP2 = mn <= P.n, hasQ2 = mn <= Q.n;
  if (!hasP2 && (A.two_way || !hasQ2)) return false;
  return true;
}

// advance one single-walk sample: consume the last batch (if any), issue the next; false when done
__device__ __forceinline__ bool single_step(const DevScene& S, const KArgs& A, SState& st, Batch& B, Out& o) {
  const int F = A.side, Fb = 1 - F;
  while (true) {
    if (st.pc == 0) {
      float d0[8];
      st.rng.dims(0, d0);
      B.n = 0;
      if (A.tech == 7) {  // same pixel and jitter in both states: one trace serves both (A3)
        int npix = S.W * S.H;
        int pix = (int)(st.i % (uint64_t)npix);
        st.sp.dir = camera_dir(S, (float)(pix % S.W) + d0[0], (float)(pix / S.W) + d0[1]);
        st.sp.pix = st.sq.pix = pix;
        st.sp.qi = st.sq.qi = B.push(mk_ray(p3(S.cam_pos), st.sp.dir, -1, A.nopm ? bit(F) : 3));
      } else {
        start_issue(S, A.tech, F, d0, st.sp, B);
        st.sq.qi = -1;
        if (!A.nopm) start_issue(S, A.tech_q, Fb, d0, st.sq, B);  // no mapped path without path mapping
      }
      st.pc = 1;
      if (B.n > 0) return true;
      continue;
    }
    if (st.pc == 1) {
      if (A.tech == 7) {
        PV E = cam_pv(S);
        st.P.n = st.Q.n = 0;
        st.P.pixel = st.Q.pixel = st.sp.pix;
        const QRes& r = B.r[st.sp.qi];
        if (r.ok[F]) { st.P.v[0] = E; st.P.v[1] = hit_pv(S, r.h[F], E.p, st.sp.dir, F); st.P.ex[1] = r.c[F]; st.P.n = 1; }
        if (r.ok[Fb] && !A.nopm) { st.Q.v[0] = E; st.Q.v[1] = hit_pv(S, r.h[Fb], E.p, st.sp.dir, Fb); st.Q.ex[1] = r.c[Fb]; st.Q.n = 1; }
      } else {
        start_consume(S, A.tech, F, st.sp, B, st.P);
        start_consume(S, A.tech_q, Fb, st.sq, B, st.Q);
      }
      if (st.P.n == 0 && (A.two_way || st.Q.n == 0)) return false;
      st.m = 1;
      st.recon = 0;
      st.w = 0;
      st.reject_from = 1 << 30;
      st.reject_reason = RJ_NONE;
      st.R1 = st.R2 = 1.0f;
      st.rdiv = st.hdiv = st.suffix_pending = false;
#if RR_VAR_KERNELS
      st.tobj_m = st.tobj_st = 0;
      st.RT = 1.0f;
#endif
      st.dynP = st.dynQ = 0;
      st.Pend = st.P.n == 0;
      st.Qend = st.Q.n == 0;
      st.pc = 2;
      B.n = 0;
      single_issue(S, A, st, B);
      if (B.n > 0) return true;
      continue;
    }
    if (!single_consume(S, A, st, B, o)) return false;
    st.m++;
    B.n = 0;
    single_issue(S, A, st, B);
    if (B.n > 0) return true;
  }
}

// ------------------------------------------------------------------------------------------------
// two-ended techniques T3 / T6: pure replay
// ------------------------------------------------------------------------------------------------
#define BMAX (RR_MAXD - 2)
struct BSide {  // one sub-walk with its per-vertex connection
  PV v[BMAX + 1];
  Cross ex[BMAX + 1];
  Cross cc[BMAX + 1];  // connection-edge crossings (sensor: from v toward E; NEE: from v toward L)
  uint8_t vis[BMAX + 1];
  int n, nconn;        // walk vertices; vertices whose connection is done
  bool ended;
  int qw;              // query index of the pending walk step (-1 none)
  int qc;              // query index of the pending connection (-1 none)
  float3 wd;
};
struct BPath {
  bool ok;
  PV start;
  float3 dir0, dir1;
  int q0, q1, qyz;
  bool jvis;   // T6: the edge (z_1, y_1) through x_G is unoccluded in View_F (else every path has f = 0)
  BSide A, B;  // A: sensor side (slots t), B: emitter side (slots 16 + s)
#if RR_VAR_KERNELS
  bool follow;  // RR_RECONNECT_BIDIR: this (mapped) path's emitter side is the base's from the reconnection on
#endif
};
struct BState {
  uint64_t i;
  Rng rng;
  int pc, nmax;
  BPath P, Q;
#if RR_VAR_KERNELS
  // RR_RECONNECT_BIDIR (reading 19): rb 0 searching, 1 reconnected (edge visibility pending), 2
  // reconnected, 3 failed (rb_reason), 4 no reconnection possible; wb the walk-B index; suffix rejection from
  // rb_from; pending queries q_rb (reconnection edge), q_sfx (suffix edge against dyn_Fbar)
  int rb, wb, rb_reason, rb_from, sfx_reason, q_rb, q_sfx, sfx_j;
  bool divb, okPb, okQb;
  float R1, R2;
#endif
};

__device__ void bidir_start_issue(const DevScene& S, const KArgs& A, int tech, int F, const Rng& rng, BPath& G, Batch& B,
                                  bool skip = false) {
  G.ok = false;
  G.jvis = true;
  G.q0 = G.q1 = G.qyz = -1;
  G.A.n = G.B.n = G.A.nconn = G.B.nconn = 0;
  G.A.ended = G.B.ended = false;
  G.A.qw = G.B.qw = G.A.qc = G.B.qc = -1;
#if RR_VAR_KERNELS
  G.follow = false;
#endif
  if (skip) return;  // the mapped path of RR_NO_PATH_MAPPING: none
  const int D = A.max_depth;
  float d0[8];
  rng.dims(0, d0);
  if (tech == 3) {
    if (S.n_edited == 0 || D < 4) return;
    PV xd = sample_set(S, S.edited_tris, S.edited_cdf, S.n_edited, F, d0[0], d0[1], d0[2]);
    float r = sqrtf(d0[3]), s, c;
    sincosf(2.0f * RR_PI_F * d0[4], &s, &c);
    float3 wl = norm3_exact(to_world(xd.n, r * c, r * s, sqrtf(fmaxf(0.0f, 1.0f - d0[3]))));
    Mat mt = load_mat(S, (uint32_t)xd.obj, F);
    float3 we;
    if (!bsdf_sample(mt, xd.n, wl, d0[6], d0[7], we)) return;
    G.start = xd;
    G.dir0 = wl;
    G.dir1 = we;
    G.q0 = B.push(mk_ray(xd.p, wl, xd.tri, bit(F)));
    G.q1 = B.push(RR_ORIENT(mk_ray(xd.p, we, xd.tri, bit(F)), true));  // the sensor side runs against the path
  } else {
    if (S.n_moved == 0 || D < 3) return;
    PV xg = sample_set(S, S.moved_tris, S.moved_cdf, S.n_moved, 1 - F, d0[0], d0[1], d0[2]);
#if RR_VAR_KERNELS
    float3 dir;
    if (A.t6_centroid) {
      // "uniformly toward the light": emitter e from d5, d uniform on the hemisphere about c_e - x_G
      const int e = min((int)floorf(d0[5] * (float)A.n_centroid), A.n_centroid - 1);
      const float4 ce = __ldg(A.t6_centroid + e);
      const float3 ax = norm3_exact(sub3(make_double3(ce.x, ce.y, ce.z), xg.p));
      float z = d0[3];
      float rr = sqrtf(fmaxf(0.0f, 1.0f - z * z)), s, c;
      sincosf(2.0f * RR_PI_F * d0[4], &s, &c);
      dir = norm3_exact(to_world(ax, rr * c, rr * s, z));
    } else {  // uniform sphere
      float z = 1.0f - 2.0f * d0[3];
      float rr = 2.0f * sqrtf(d0[3] * (1.0f - d0[3])), s, c;
      sincosf(2.0f * RR_PI_F * d0[4], &s, &c);
      dir = f3(rr * c, rr * s, z);
    }
#else
    float z = 1.0f - 2.0f * d0[3];
    float rr = 2.0f * sqrtf(d0[3] * (1.0f - d0[3])), s, c;  // sqrt(1 - z^2), no cancellation
    sincosf(2.0f * RR_PI_F * d0[4], &s, &c);
    float3 dir = f3(rr * c, rr * s, z);
#endif
    G.start = xg;
    G.dir0 = dir;
    G.dir1 = dir * -1.0f;
    // the start rays' own ghost crossings are not used (the edge (z_1, y_1) is queried as a whole next step)
    G.q0 = B.push(mk_ray(xg.p, dir, -1, bit(F) | QW_NO_CROSS));
    G.q1 = B.push(mk_ray(xg.p, G.dir1, -1, bit(F) | QW_NO_CROSS));
  }
}
__device__ void bidir_start_consume(const DevScene& S, int tech, int F, BPath& G, const Batch& B) {
  if (G.q0 < 0) return;
  const QRes& ry = B.r[G.q0];
  const QRes& rz = B.r[G.q1];
  if (!ry.ok[F] || !rz.ok[F]) return;
  PV y1 = hit_pv(S, ry.h[F], G.start.p, G.dir0, F);
  PV z1 = hit_pv(S, rz.h[F], G.start.p, G.dir1, F);
  G.ok = true;
  if (tech == 3) {
    G.B.v[0] = G.start; G.B.v[1] = y1; G.B.ex[1] = ry.c[F]; G.B.n = 1;
    G.A.v[0] = G.start; G.A.v[1] = z1; G.A.ex[1] = rz.c[F]; G.A.n = 1;
  } else {
    G.A.v[0] = y1; G.A.v[1] = z1; G.A.n = 1;  // edge (z_1, y_1): crossings by a segment query next step
    G.B.v[0] = z1; G.B.v[1] = y1; G.B.n = 1;
    G.A.ex[1] = G.B.ex[1] = cross_zero();
  }
}
// issue the next queries of one path: T6 edge crossings, pending connections, walk steps
__device__ void bidir_issue(const DevScene& S, const KArgs& A, int tech, int F, const Rng& rng, int nmax, BPath& G,
                            Batch& B, bool first) {
  G.qyz = -1;
  G.A.qw = G.B.qw = G.A.qc = G.B.qc = -1;
  if (!G.ok) return;
  if (first && tech == 6 && S.n_moved > 0) {  // crossings of the whole edge y_1 -> z_1, x_G among them
    // its visibility too: the edge must be unoccluded in View_F like every edge of a path (Eq.2 V) -- it is not,
    // e.g., when x_G also lies on the real object's surface (coplanar faces of a horizontal move)
    Query q = mk_seg(G.A.v[0].p, G.A.v[1].p, G.A.v[0].tri, G.A.v[1].tri, bit(F));
    G.qyz = B.push(RR_ORIENT(seeded(q, norm3f(sub3(G.start.p, G.A.v[0].p)), G.start), true));
  }
  PV E = cam_pv(S);
  for (int side = 0; side < 2; ++side) {
    BSide& W = side == 0 ? G.A : G.B;
    if (W.nconn < W.n) {  // connection of the newest vertex
      int t = W.nconn + 1;
      const PV& v = W.v[t];
      if (side == 0) {
        if (project(S, v.p) < 0) {  // the sensor connection cannot reach the image: value 0 (reading 4)
          W.vis[t] = 0;
          W.cc[t] = cross_zero();
          W.nconn = t;
        } else {
          W.qc = B.push(mk_seg(v.p, E.p, v.tri, -1, bit(F)));
        }
      } else {
        float d[8];
        rng.dims((uint32_t)(16 + t), d);
        PV Lt = sample_emitter(S, d[3], d[4], d[5], d[6]);  // regenerated from the same slot in bidir_path
        W.qc = B.push(mk_seg(v.p, Lt.p, v.tri, Lt.tri, bit(F)));
      }
    }
#if RR_VAR_KERNELS
    if (side == 1 && G.follow) continue;  // the emitter side follows the base walk (no rays of its own)
#endif
    if (!W.ended && W.n < nmax) {
      int m = W.n;
      float d[8];
      rng.dims((uint32_t)((side == 0 ? 0 : 16) + m), d);
      Mat mt = load_mat(S, (uint32_t)W.v[m].obj, F);
      if (bsdf_sample(mt, W.v[m].n, norm3_exact(sub3(W.v[m - 1].p, W.v[m].p)), d[1], d[2], W.wd))
        W.qw = B.push(RR_ORIENT(mk_ray(W.v[m].p, W.wd, W.v[m].tri, bit(F)), side == 0));  // side A: against the path
      else
        W.ended = true;
    } else {
      W.ended = true;
    }
  }
}
__device__ void bidir_consume(const DevScene& S, const KArgs& A, int F, BPath& G, const Batch& B) {
  if (!G.ok) return;
  if (G.qyz >= 0) {  // crossings of the edge y_1 -> z_1, plus the crossing at x_G
    const float3 dv = sub3(G.A.v[1].p, G.A.v[0].p);
    const float L = norm3f(dv);
#if RR_VAR_KERNELS
    const float pd = A.t6_centroid ? t6_pdir4pi(A.t6_centroid, A.n_centroid, f3of(G.start.p), G.dir0) : 1.0f;  // +d: z_1 -> y_1
#else
    const float pd = 1.0f;
#endif
    G.A.ex[1] = add_seed(B.r[G.qyz].c[F], norm3f(sub3(G.start.p, G.A.v[0].p)), L,
                         L / fabsf(dot3(G.start.n, dv)) * pd);
    G.jvis = B.r[G.qyz].ok[F] != 0;
    G.B.ex[1] = swapc(G.A.ex[1]);
  }
  for (int side = 0; side < 2; ++side) {
    BSide& W = side == 0 ? G.A : G.B;
    if (W.qc >= 0) {
      int t = W.nconn + 1;
      W.vis[t] = B.r[W.qc].ok[F];
      W.cc[t] = B.r[W.qc].c[F];
      W.nconn = t;
    }
    if (W.qw >= 0) {
      const QRes& r = B.r[W.qw];
      if (r.ok[F]) {
        int m = W.n;
        W.v[m + 1] = hit_pv(S, r.h[F], W.v[m].p, W.wd, F);
        W.ex[m + 1] = r.c[F];
        W.n = m + 1;
      } else {
        W.ended = true;
      }
    }
  }
}

// path (E, z_t..z_1, [x_D], y_1..y_s, L) of a two-ended sample; L is re-drawn from slot 16 + s
__device__ int bidir_path(const BPath& G, int tech, int t, int s, const DevScene& S, const Rng& rng, PV* x, Cross* ce) {
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
  float d[8];
  rng.dims((uint32_t)(16 + s), d);
  x[k] = sample_emitter(S, d[3], d[4], d[5], d[6]);
  ++k;
  return k;
}

__device__ __noinline__ void bidir_finish(const DevScene& S, const KArgs& A, BState& st, Out& o) {
  const int F = A.side, Fb = 1 - A.side, l = A.tech, D = A.max_depth;
  BPath& P = st.P;
  BPath& Q = st.Q;
  const int extra = (l == 3) ? 2 : 1;
  PV x[RR_MAXV + 2];
  Cross ce[RR_MAXV + 2];
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
        pixp = project(S, P.A.v[t].p);
        if (P.A.vis[t] && P.B.vis[s] && P.jvis) {
          int k = bidir_path(P, l, t, s, S, st.rng, x, ce);
          vp = path_value(S, x, ce, k, F, A.mask);
        }
      }
      if (qc_) {
        pixq = project(S, Q.A.v[t].p);
        if (Q.A.vis[t] && Q.B.vis[s] && Q.jvis) {
          int k = bidir_path(Q, l, t, s, S, st.rng, x, ce);
          vq = path_value(S, x, ce, k, Fb, A.mask);
        }
      }
      if (pc) {
        int stt = qc_ ? ST_ACCEPTED : ST_UNPAIRED, rs = RJ_NONE;
        float R = 1.0f;
#if RR_VAR_KERNELS
        if (A.recon_bidir && st.rb >= 1 && st.rb <= 3 && s >= st.wb + 1) {  // reconnected emitter side
          if (st.rb == 3) { stt = ST_REJECTED; rs = st.rb_reason; }
          else if (s >= st.rb_from) { stt = ST_REJECTED; rs = st.sfx_reason; }
          else if (stt == ST_ACCEPTED) {
            R = st.R1 * (s >= st.wb + 2 ? st.R2 : 1.0f);
            if (!(R > 0.0f) || !isfinite(R)) { stt = ST_REJECTED; rs = RJ_TARGET; }
          }
        }
#endif
        if (stt == ST_ACCEPTED && A.reject_multi) {
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
          if (dv && (dp >= 2 || dq >= 2)) { stt = ST_REJECTED; rs = RJ_MULTI; }
        }
        finish(o, st.i, 3, t, s, stt, rs, pixp, vp, pixq, vq, R);
      } else {
        finish(o, st.i, 3, t, s, ST_MAPPED_ONLY, RJ_NONE, -1, f3(0.f, 0.f, 0.f), pixq, vq, 1.0f);
      }
    }
  }
}

#if RR_VAR_KERNELS
// RR_RECONNECT_BIDIR (P:L387-411 inside the two-ended techniques; reading 19): after the round that
// extended both emitter sides from index m (lockstep), decide the reconnection at m exactly as the single walks do
// -- the first index where the pair is diverged (a different vertex, or different directions sampled at a shared
// one) and both vertices are rough reconnects Q's y'_m to the base's y_{m+1} -- then let Q's emitter side follow
// the base's: copied vertices, its own NEE connections, each later edge re-checked against dyn_Fbar only.
__device__ void bidir_recon_step(const DevScene& S, const KArgs& A, BState& st, const Batch& B, int m_before_p,
                                 int m_before_q) {
  const int F = A.side, Fb = 1 - F;
  BPath& P = st.P;
  BPath& Q = st.Q;
  if (st.q_rb >= 0) {  // the reconnection edge y'_w -> y_{w+1} in View_Fbar
    const QRes& r = B.r[st.q_rb];
    if (r.ok[Fb]) { st.rb = 2; Q.B.ex[st.wb + 1] = r.c[Fb]; }
    else { st.rb = 3; st.rb_reason = RJ_OCCLUDED; }
  }
  if (st.q_sfx >= 0) {  // a shared suffix edge against dyn_Fbar only
    const QRes& r = B.r[st.q_sfx];
    if (!r.ok[Fb] && st.sfx_j < st.rb_from) { st.rb_from = st.sfx_j; st.sfx_reason = RJ_OCCLUDED; }
    Q.B.ex[st.sfx_j] = r.c[Fb];
  }
  st.q_rb = st.q_sfx = -1;
  if (st.rb == 1 || st.rb == 2) {  // follow: copy the base's newest emitter-side vertex
    if (P.B.n > Q.B.n) {
      const int j = P.B.n;
      Q.B.v[j] = P.B.v[j];
      Q.B.n = j;
      st.sfx_j = j;  // edge (y_{j-1}, y_j) to re-check with the next batch
      if (edited(S, P.B.v[j].obj) && j < st.rb_from) { st.rb_from = j; st.sfx_reason = RJ_SUFFIX_DYN; }
      if (j == st.wb + 2) st.R2 = area_pdf(S, Fb, Q.B.v[st.wb], P.B.v[j - 1], P.B.v[j]) /
                                  area_pdf(S, F, P.B.v[st.wb], P.B.v[j - 1], P.B.v[j]);
    } else {
      st.sfx_j = 0;
    }
    Q.B.ended = P.B.ended;
    return;
  }
  if (st.rb != 0) return;
  // search at index m = the vertex both emitter sides stood on before this round's walk step
  const int m = m_before_p;
  if (m < 1 || m != m_before_q) { if (m >= 1) st.rb = 4; return; }
  st.divb = st.divb || !same_pv(S, P.B.v[m], Q.B.v[m]);
  const bool dirdiv = (st.okPb != st.okQb) || (st.okPb && st.okQb && !eq3(P.B.wd, Q.B.wd));
  const Mat mp = load_mat(S, (uint32_t)P.B.v[m].obj, F), mq = load_mat(S, (uint32_t)Q.B.v[m].obj, Fb);
  if ((st.divb || dirdiv) && rough_enough(mp, A.alpha_min) && rough_enough(mq, A.alpha_min)) {
    st.wb = m;
    if (P.B.n < m + 1) { st.rb = 4; return; }  // no target: the base has no connection beyond m
    const PV& vw = P.B.v[m];
    const PV& vq = Q.B.v[m];
    const PV& tg = P.B.v[m + 1];
    float3 a = sub3(vq.p, tg.p), b = sub3(vw.p, tg.p);
    float la2 = dot3(a, a), lb2 = dot3(b, b);
    int rs = RJ_NONE;
    if (edited(S, tg.obj)) rs = RJ_TARGET;
    else if (!rough_enough(load_mat(S, (uint32_t)tg.obj, F), A.alpha_min)) rs = RJ_TARGET;
    else if (fminf(sqrtf(lb2), sqrtf(la2)) < A.dmin) rs = RJ_TARGET;
    else {
      float Jg = fabsf(dot3(tg.n, a * (1.0f / sqrtf(la2)))) / fabsf(dot3(tg.n, b * (1.0f / sqrtf(lb2)))) * lb2 / la2;
      if (!(Jg <= A.jacobian_max && Jg >= 1.0f / A.jacobian_max)) rs = RJ_JACOBIAN;
    }
    if (rs != RJ_NONE) { st.rb = 3; st.rb_reason = rs; return; }
    st.R1 = area_pdf(S, Fb, Q.B.v[m - 1], vq, tg) / area_pdf(S, F, P.B.v[m - 1], vw, tg);
    st.rb = 1;
    Q.B.v[m + 1] = tg;  // Q's own hit at m + 1 (if any) is dropped; its emitter side follows the base's
    Q.B.n = m + 1;
    Q.B.ended = P.B.ended;
    Q.follow = true;
    st.sfx_j = 0;
    return;
  }
  if (dirdiv) st.divb = true;
}
#endif

__device__ bool bidir_step(const DevScene& S, const KArgs& A, BState& st, Batch& B, Out& o) {
  const int F = A.side, Fb = 1 - F, l = A.tech;
  while (true) {
    if (st.pc == 0) {
      B.n = 0;
      st.nmax = l == 3 ? A.max_depth - 3 : A.max_depth - 2;
      bidir_start_issue(S, A, l, F, st.rng, st.P, B);
      bidir_start_issue(S, A, l, Fb, st.rng, st.Q, B, A.nopm != 0);
      st.pc = 1;
      if (B.n > 0) return true;
      continue;
    }
    if (st.pc == 1) {
      bidir_start_consume(S, l, F, st.P, B);
      bidir_start_consume(S, l, Fb, st.Q, B);
      if (!st.P.ok && (A.two_way || !st.Q.ok)) return false;
      B.n = 0;
      bidir_issue(S, A, l, F, st.rng, st.nmax, st.P, B, true);
      bidir_issue(S, A, l, Fb, st.rng, st.nmax, st.Q, B, true);
#if RR_VAR_KERNELS
      st.rb = 0;
      st.wb = 0;
      st.rb_reason = st.sfx_reason = RJ_NONE;
      st.rb_from = 1 << 30;
      st.q_rb = st.q_sfx = -1;
      st.sfx_j = 0;
      st.R1 = st.R2 = 1.0f;
      st.divb = st.P.ok && st.Q.ok && !same_pv(S, st.P.B.v[0], st.Q.B.v[0]);
      st.okPb = st.P.B.qw >= 0;
      st.okQb = st.Q.B.qw >= 0;
#endif
      st.pc = 2;
      if (B.n > 0) return true;
      continue;
    }
#if RR_VAR_KERNELS
    const int mbp = st.P.B.n, mbq = st.Q.B.n;  // emitter-side index before this round's walk step
#endif
    bidir_consume(S, A, F, st.P, B);
    bidir_consume(S, A, Fb, st.Q, B);
#if RR_VAR_KERNELS
    if (A.recon_bidir && st.P.ok && st.Q.ok) bidir_recon_step(S, A, st, B, mbp, mbq);
#endif
    B.n = 0;
    bidir_issue(S, A, l, F, st.rng, st.nmax, st.P, B, false);
    bidir_issue(S, A, l, Fb, st.rng, st.nmax, st.Q, B, false);
#if RR_VAR_KERNELS
    if (A.recon_bidir && st.P.ok && st.Q.ok) {
      st.okPb = st.P.B.qw >= 0;  // a direction was sampled at the emitter side's newest vertex
      st.okQb = st.Q.B.qw >= 0;
      if (st.rb == 1)
        st.q_rb = B.push(mk_seg(st.Q.B.v[st.wb].p, st.Q.B.v[st.wb + 1].p, st.Q.B.v[st.wb].tri,
                                st.Q.B.v[st.wb + 1].tri, bit(Fb)));
      if ((st.rb == 1 || st.rb == 2) && st.sfx_j > st.wb + 1)
        st.q_sfx = B.push(mk_seg(st.Q.B.v[st.sfx_j - 1].p, st.Q.B.v[st.sfx_j].p, st.Q.B.v[st.sfx_j - 1].tri,
                                 st.Q.B.v[st.sfx_j].tri, bit(Fb), true));
    }
#endif
    if (B.n > 0) return true;
    bidir_finish(S, A, st, o);
    return false;
  }
}

// ------------------------------------------------------------------------------------------------
// kernel: persistent lanes over this shard's samples of one (technique, side)
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void warp_add(unsigned long long* p, uint32_t v) {
  uint32_t s = __reduce_add_sync(FULLMASK, v);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(p, (unsigned long long)s);
}

// warp-aggregated fetch of the next local sample slot for every lane in `need`
__device__ __forceinline__ uint64_t fetch_work(unsigned long long* counter, bool need) {
  unsigned m = __ballot_sync(FULLMASK, need);
  unsigned long long base = 0;
  int lane = threadIdx.x & 31;
  if (m) {
    int leader = __ffs(m) - 1;
    if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
    base = __shfl_sync(FULLMASK, base, leader);
  }
  return base + __popc(m & ((1u << lane) - 1u));
}

// ------------------------------------------------------------------------------------------------
// kernel: persistent lanes over this shard's samples of one (technique, side).  The 32 lanes of a warp
// advance their samples in lockstep, then trace the queries the step issued through the single traversal
// site (rr_query.cuh).
// ------------------------------------------------------------------------------------------------
#ifndef RR_BLOCK
#define RR_BLOCK 128  // threads per block of the residual kernels
#endif
#ifndef RR_MIN_BLOCKS
#define RR_MIN_BLOCKS 16  // resident blocks per SM requested from the register allocator (32 registers:
                          // latency hiding beats the spills)
#endif

#ifndef RR_MEGA_SYNC
#define RR_MEGA_SYNC false  // traversal with a ballot per iteration in the megakernels (rr_query.cuh traverse)
#endif
template <class State, bool BIDIR, bool COUNT>
__device__ __forceinline__ void residual_loop(const DevScene& S, const KArgs& A) {
  Out o;
  o.A = &A;
  o.qc.closest = o.qc.shadow = o.qc.inst = 0;
  o.qc.tc.nodes = o.qc.tc.tris = 0;
#if RR_COUNT_JOBS
  if (COUNT) o.qc.tc.inst_nodes = o.qc.tc.ghost_nodes = 0;
#endif
  o.conns = o.acc = o.rej = o.unp = o.monly = o.recon = o.splats = o.offscreen = o.zero = 0;
  for (int r = 0; r < 6; ++r) o.rejby[r] = 0;
  uint32_t nsamp = 0;
  State st;
  const int lane = threadIdx.x & 31;
  Batch B;
  B.n = 0;
  unsigned long long sc[5] = {0, 0, 0, 0, 0};  // scheduler occupancy (rr_stats.sched)
  bool active = false, more = true;
  while (true) {
    // refill: lanes without a sample take the next local slot (warp-aggregated atomics)
    if (!active) B.n = 0;
    while (true) {
      bool need = !active && more;
      const unsigned nm = __ballot_sync(FULLMASK, need);
      if (!nm) break;
      // batch refill: free lanes wait until A.refill_min lanes are free (or none is busy), then take consecutive
      // (ordered, hence neighbouring) samples together, so the warp's lanes start and advance in step
      if (__popc(nm) < A.refill_min && __any_sync(FULLMASK, active)) break;
      uint64_t li = fetch_work(A.work, need);
      if (need) {
        if (li >= A.n_local) {
          more = false;
        } else {
          uint64_t i;
          bool valid = true;
          if (A.dump) {
            i = A.i_begin + li;
          } else {
            if (A.perm) li = __ldg(A.perm + li);  // T3 / T6: start-ray order (sample_order)
            uint64_t blk = li >> 16, off = li & 0xFFFFull;
            i = ((blk * A.shard_count + A.shard_index) << 16) | off;
            valid = i < A.n_total;
          }
          if (valid) {
            nsamp++;
            st.i = i;
            st.rng.i_lo = (uint32_t)i;
            st.rng.i_hi = (uint32_t)(i >> 32);
            st.rng.ls = (uint32_t)A.tech | ((uint32_t)A.side << 8);
            st.rng.k0 = (uint32_t)A.seed;
            st.rng.k1 = (uint32_t)(A.seed >> 32);
            st.pc = 0;
            bool go;
            if constexpr (BIDIR) go = bidir_step(S, A, st, B, o);
            else go = single_step(S, A, st, B, o);
            active = go;
            if (!go) B.n = 0;
          }
        }
      }
    }
    // every lane's queries through the single traversal site, in lockstep over the batch index
    int nmax = (int)__reduce_max_sync(FULLMASK, (unsigned)B.n);
    if (nmax == 0 && !__any_sync(FULLMASK, active || more)) break;
    const unsigned total = __reduce_add_sync(FULLMASK, (unsigned)B.n);
    if (lane == 0) {
      sc[0]++;
      sc[3] += total;
    }
    sc[4] += active;
    for (int k = 0; k < nmax; ++k)
#if RR_VAR_KERNELS
      if (k < B.n) run_query<COUNT, RR_MEGA_SYNC>(S, B.q[k], B.r[k], o.qc, A.t6_centroid, A.n_centroid);
#else
      if (k < B.n) run_query<COUNT, RR_MEGA_SYNC>(S, B.q[k], B.r[k], o.qc);
#endif
    if (active) {
      sc[2]++;
      bool go;
      if constexpr (BIDIR) go = bidir_step(S, A, st, B, o);
      else go = single_step(S, A, st, B, o);
      active = go;
      if (!active) B.n = 0;
    }
  }
  unsigned long long* stt = A.stats;
  warp_add(stt + STAT_SAMPLES, nsamp);
  warp_add(stt + STAT_CONNECTIONS, o.conns);
  warp_add(stt + STAT_ACCEPTED, o.acc);
  warp_add(stt + STAT_REJECTED, o.rej);
  warp_add(stt + STAT_UNPAIRED, o.unp);
  warp_add(stt + STAT_MAPPED_ONLY, o.monly);
  warp_add(stt + STAT_RECONNECTED, o.recon);
  warp_add(stt + STAT_CLOSEST, o.qc.closest);
  warp_add(stt + STAT_SHADOW, o.qc.shadow);
  warp_add(stt + STAT_INST, o.qc.inst);
  warp_add(stt + STAT_NODES, o.qc.tc.nodes);
  warp_add(stt + STAT_TRIS, o.qc.tc.tris);
  warp_add(stt + STAT_SPLATS, o.splats);
  warp_add(stt + STAT_OFFSCREEN, o.offscreen);
  warp_add(stt + STAT_ZERO, o.zero);
  for (int r = 0; r < 6; ++r) warp_add(stt + STAT_REJBY + r, o.rejby[r]);
  for (int r = 0; r < 5; ++r)
    if (sc[r]) atomicAdd(stt + STAT_SCHED + r, sc[r]);
#if RR_COUNT_JOBS
  if (COUNT) {  // sched[6] / [7]: nodes fetched in dynamic-instance jobs / in ghost-crossing jobs
    warp_add(stt + STAT_SCHED + 6, o.qc.tc.inst_nodes);
    warp_add(stt + STAT_SCHED + 7, o.qc.tc.ghost_nodes);
  }
#endif
}

template <bool COUNT>
__global__ void __launch_bounds__(RR_BLOCK, RR_MIN_BLOCKS) k_residual_single(const __grid_constant__ DevScene S, const __grid_constant__ KArgs A) {
  residual_loop<SState, false, COUNT>(S, A);
}
template <bool COUNT>
#ifndef RR_MIN_BLOCKS_BIDIR
#define RR_MIN_BLOCKS_BIDIR RR_MIN_BLOCKS
#endif
__global__ void __launch_bounds__(RR_BLOCK, RR_MIN_BLOCKS_BIDIR) k_residual_bidir(const __grid_constant__ DevScene S, const __grid_constant__ KArgs A) {
  residual_loop<BState, true, COUNT>(S, A);
}

inline void launch_kernels(const DevScene& S, const KArgs& A, int grid, cudaStream_t st) {
  const bool bidir = A.tech == 3 || A.tech == 6;
  if (A.count) {
    if (bidir) k_residual_bidir<true><<<grid, RR_BLOCK, 0, st>>>(S, A);
    else k_residual_single<true><<<grid, RR_BLOCK, 0, st>>>(S, A);
  } else {
    if (bidir) k_residual_bidir<false><<<grid, RR_BLOCK, 0, st>>>(S, A);
    else k_residual_single<false><<<grid, RR_BLOCK, 0, st>>>(S, A);
  }
}
}  // namespace kplain / kvndf

#if RR_VAR_KERNELS
void launch_residual_var(const DevScene& S, const KArgs& A, int grid, cudaStream_t st) {
  kvar::launch_kernels(S, A, grid, st);
}
#elif RR_VNDF_KERNELS
void launch_residual_vndf(const DevScene& S0, const KArgs& A, int grid, cudaStream_t st) {
  DevScene S = S0;
  S.mat_type = A.mat_type_vndf;  // GGX = 2: visible-normal sampling
  kvndf::launch_kernels(S, A, grid, st);
}
#else
using namespace kplain;  // helpers of the state machines (bit(), ...) used by the test kernels below

__global__ void k_philox(uint32_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint4 c = make_uint4(ctr[4 * t], ctr[4 * t + 1], ctr[4 * t + 2], ctr[4 * t + 3]);
  uint4 r = philox4x32_10(c, make_uint2(k0, k1));
  out[4 * t] = r.x; out[4 * t + 1] = r.y; out[4 * t + 2] = r.z; out[4 * t + 3] = r.w;
}

__device__ __forceinline__ void trace_store(const DevScene& S, int F, const float* r, const QRes& res, float* h) {
  float3 o = f3(r[0], r[1], r[2]);
  float3 d = norm3_exact(f3(r[3], r[4], r[5]));
  if (!res.ok[F]) {
    h[0] = -1.0f;
    return;
  }
  PV v = hit_pv(S, res.h[F], p3(o), d, F);
  float3 q = sub3(v.p, p3(o));
  h[0] = sqrtf(dot3(q, q));
  h[1] = __int_as_float(v.tri);
  h[2] = (float)v.p.x; h[3] = (float)v.p.y; h[4] = (float)v.p.z;
  h[5] = v.n.x; h[6] = v.n.y; h[7] = v.n.z;
}
__device__ __forceinline__ Query trace_query(const float* r, int F) {
  float3 o = f3(r[0], r[1], r[2]);
  float3 d = norm3_exact(f3(r[3], r[4], r[5]));
  return mk_ray(p3(o), d, __float_as_int(r[6]), bit(F));
}

__global__ void k_trace(const __grid_constant__ DevScene S, int F, uint32_t n, const float* rays, float* hits) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  QCount qc = {};
  QRes res;
  run_query<true, true>(S, trace_query(rays + 8 * t, F), res, qc);
  trace_store(S, F, rays + 8 * t, res, hits + 8 * t);
}

__global__ void k_segment(const __grid_constant__ DevScene S, uint32_t n, const float* segs, float* out) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const float* s = segs + 6 * t;
  QCount qc = {};
  QRes r;
  run_query<true, true>(S, mk_seg(p3(f3(s[0], s[1], s[2])), p3(f3(s[3], s[4], s[5])), -1, -1, 3), r, qc);
  float* o = out + 10 * t;
  for (int F = 0; F < 2; ++F) {
    o[5 * F] = r.ok[F] ? 1.0f : 0.0f;
    o[5 * F + 1] = r.c[F].n;
    o[5 * F + 2] = r.c[F].s0;
    o[5 * F + 3] = r.c[F].sa;
    o[5 * F + 4] = r.c[F].sb;
  }
}

// ---- processing order (sample_order): sort key of the base path's start ray
#ifndef RR_SORT_KEY
#define RR_SORT_KEY 2  // 0: direction major, 1: position major (7 bits per axis), 2: finer directions, 3: position major (8 bits)
#endif
#if RR_SORT_KEY == 3
#define RR_SORT_BITS 31
#else
#define RR_SORT_BITS 28
#endif
__device__ __forceinline__ uint32_t spread7(uint32_t v) {  // 7 bits -> every third bit
  v &= 0x7Fu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
__device__ __forceinline__ uint32_t spread2(uint32_t v) {  // 14 bits -> every second bit
  v &= 0x3FFFu;
  v = (v | (v << 8)) & 0x00FF00FFu;
  v = (v | (v << 4)) & 0x0F0F0F0Fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}
__global__ void k_sample_keys(const __grid_constant__ DevScene S, const __grid_constant__ KArgs A, float3 blo,
                              float3 bsc, uint32_t* keys, uint32_t* vals) {
  for (uint64_t li = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; li < A.n_local;
       li += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t blk = li >> 16, off = li & 0xFFFFull;
    const uint64_t i = ((blk * A.shard_count + A.shard_index) << 16) | off;
    uint32_t key = (1u << RR_SORT_BITS) - 1u;
    if (i < A.n_total) {
      Rng rng;
      rng.i_lo = (uint32_t)i;
      rng.i_hi = (uint32_t)(i >> 32);
      rng.ls = (uint32_t)A.tech | ((uint32_t)A.side << 8);
      rng.k0 = (uint32_t)A.seed;
      rng.k1 = (uint32_t)(A.seed >> 32);
      float d0[8];
      rng.dims(0, d0);
      if (A.tech == 7) {  // camera rays: pixels in 2D Morton order (the samples of a pixel stay in index order)
        const uint32_t npix = (uint32_t)(S.W * S.H), pix = (uint32_t)(i % npix);
        key = spread2(pix % (uint32_t)S.W) | (spread2(pix / (uint32_t)S.W) << 1);
        keys[li] = key;
        vals[li] = (uint32_t)li;
        continue;
      }
      P3 x;
      float3 dir = f3(0.0f, 0.0f, 1.0f);
      if (A.tech == 6) {  // x_G and the uniform-sphere direction (bidir_start_issue)
        x = sample_set(S, S.moved_tris, S.moved_cdf, S.n_moved, 1 - A.side, d0[0], d0[1], d0[2]).p;
        const float z = 1.0f - 2.0f * d0[3], rr = 2.0f * sqrtf(d0[3] * (1.0f - d0[3]));
        float sn, cs;
        sincosf(2.0f * RR_PI_F * d0[4], &sn, &cs);
        dir = f3(rr * cs, rr * sn, z);
      } else if (A.tech == 3) {  // x_D and its cosine-distributed emitter-side direction
        const PV xd = sample_set(S, S.edited_tris, S.edited_cdf, S.n_edited, A.side, d0[0], d0[1], d0[2]);
        x = xd.p;
        const float r = sqrtf(d0[3]);
        float sn, cs;
        sincosf(2.0f * RR_PI_F * d0[4], &sn, &cs);
        dir = to_world(xd.n, r * cs, r * sn, sqrtf(fmaxf(0.0f, 1.0f - d0[3])));
      } else if (A.tech == 4 || A.tech == 5) {  // x_G (start_issue): the start ray's far end
        x = sample_set(S, S.moved_tris, S.moved_cdf, S.n_moved, 1 - A.side, d0[0], d0[1], d0[2]).p;
      } else {  // T1 / T2: x_D
        x = sample_set(S, S.edited_tris, S.edited_cdf, S.n_edited, A.side, d0[0], d0[1], d0[2]).p;
      }
      // the start point in the box of its sample set (blo, 1 / extent = bsc), [0, 1) per axis
      const float3 q = f3((float)(x.x - blo.x) * bsc.x, (float)(x.y - blo.y) * bsc.y, (float)(x.z - blo.z) * bsc.z);
#if RR_SORT_KEY == 2
      // finer direction bins (5 bits of z, 5 of the azimuth), 6 bits per axis of the start point
      const uint32_t zb = min(31u, (uint32_t)((1.0f - dir.z) * 16.0f));
      const uint32_t pb = min(31u, (uint32_t)((atan2f(dir.y, dir.x) + RR_PI_F) * (32.0f / (2.0f * RR_PI_F))));
      const uint32_t mx = (uint32_t)fminf(fmaxf(q.x * 64.0f, 0.0f), 63.0f);
      const uint32_t my = (uint32_t)fminf(fmaxf(q.y * 64.0f, 0.0f), 63.0f);
      const uint32_t mz = (uint32_t)fminf(fmaxf(q.z * 64.0f, 0.0f), 63.0f);
      key = ((zb << 5 | pb) << 18) | (spread7(mx) << 2) | (spread7(my) << 1) | spread7(mz);
#else
      // direction bin (3 bits of z, 4 bits of the azimuth) and the start point's Morton code in a cube of 2 diag
      // about the camera (7 bits per axis); RR_SORT_KEY 0: direction major, 1: position major
      const uint32_t zb = min(7u, (uint32_t)((1.0f - dir.z) * 4.0f));
      const uint32_t pb = min(15u, (uint32_t)((atan2f(dir.y, dir.x) + RR_PI_F) * (16.0f / (2.0f * RR_PI_F))));
      const uint32_t mx = (uint32_t)fminf(fmaxf(q.x * 128.0f, 0.0f), 127.0f);
      const uint32_t my = (uint32_t)fminf(fmaxf(q.y * 128.0f, 0.0f), 127.0f);
      const uint32_t mz = (uint32_t)fminf(fmaxf(q.z * 128.0f, 0.0f), 127.0f);
      const uint32_t mort = (spread7(mx) << 2) | (spread7(my) << 1) | spread7(mz);
#if RR_SORT_KEY == 1
      key = (mort << 7) | (zb << 4 | pb);
#elif RR_SORT_KEY == 3
      {  // position major with 8 bits per axis
        const uint32_t ax = (uint32_t)fminf(fmaxf(q.x * 256.0f, 0.0f), 255.0f);
        const uint32_t ay = (uint32_t)fminf(fmaxf(q.y * 256.0f, 0.0f), 255.0f);
        const uint32_t az = (uint32_t)fminf(fmaxf(q.z * 256.0f, 0.0f), 255.0f);
        const uint32_t m8 = (spread7(ax >> 1) << 5) | (spread7(ay >> 1) << 4) | (spread7(az >> 1) << 3) |
                            ((ax & 1u) << 2) | ((ay & 1u) << 1) | (az & 1u);
        key = (m8 << 7) | (zb << 4 | pb);
      }
#else
      key = ((zb << 4 | pb) << 21) | mort;
#endif
#endif
    }
    keys[li] = key;
    vals[li] = (uint32_t)li;
  }
}
size_t sample_order(const DevScene& S, const KArgs& A, const float lo[3], const float hi[3], uint32_t* keys,
                    uint32_t* vals, uint32_t* keys2, uint32_t* perm, void* tmp, size_t tmp_bytes, cudaStream_t st) {
  const int n = (int)A.n_local;
  if (!keys) {
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, n, 0, RR_SORT_BITS, st);
    return need;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float3 blo = f3(lo[0], lo[1], lo[2]), bsc;
  bsc.x = 1.0f / fmaxf(hi[0] - lo[0], 1e-20f);
  bsc.y = 1.0f / fmaxf(hi[1] - lo[1], 1e-20f);
  bsc.z = 1.0f / fmaxf(hi[2] - lo[2], 1e-20f);
  k_sample_keys<<<sms * 8, 256, 0, st>>>(S, A, blo, bsc, keys, vals);
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, perm, n, 0, RR_SORT_BITS, st);
  return 0;
}

// ---- host launchers
// persistent lanes: one wave of resident blocks on every SM (fewer for tiny launches)
int residual_grid(bool bidir, uint64_t n) {
  // SM count and occupancy per device (a process may drive several GPUs, one context each)
  struct Dev { int sms = 0, occ[2] = {0, 0}; };
  static Dev cache[64];
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  Dev d;
  {
    std::lock_guard<std::mutex> lk(mu);
    Dev& c = cache[dev & 63];
    if (!c.sms) {
      cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ[0], kplain::k_residual_single<false>, RR_BLOCK, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ[1], kplain::k_residual_bidir<false>, RR_BLOCK, 0);
    }
    d = c;
  }
  uint64_t g = (n + RR_BLOCK - 1) / RR_BLOCK;
  uint64_t cap = (uint64_t)d.sms * (uint64_t)std::max(1, d.occ[bidir ? 1 : 0]);
  return (int)std::max<uint64_t>(1, std::min(g, cap));
}
int residual_block() { return RR_BLOCK; }
void launch_residual(const DevScene& S, const KArgs& A, int grid, cudaStream_t st) {
  if (A.t6_centroid || A.tobj || A.recon_bidir) launch_residual_var(S, A, grid, st);  // SURVEY 8(f) row 4 variants
  else if (A.mat_type_vndf) launch_residual_vndf(S, A, grid, st);  // RR_VNDF: the other instantiation
  else kplain::launch_kernels(S, A, grid, st);
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

#endif  // RR_VNDF_KERNELS / RR_VAR_KERNELS
}  // namespace rr
