// rr_query.cuh -- the one generic ray query of the residual kernels.
//
// Every traversal of the estimator goes through a Tracer, which contains the library's ONLY traversal loop:
// a query is decomposed into BLAS jobs (the static BLAS once, then each dynamic instance under the
// transform of each requested state, then each MOVED instance under the other state's transform for the
// ghost crossings).  Jobs of all kinds run through the same budgeted traversal loop, so lanes that trace
// queries of different kinds still execute one instruction stream.
//
// The residual kernels trace through a block-wide query queue (rr_residual.cu): any lane of the block traces
// any lane's query, so a lane never waits for the slowest query of its warp.
//
//  QT_CLOSEST: closest hit of the ray (o, d) in View_F = static + dyn at M_F (ghosts transparent),
//              t in (eps, inf), origin triangle excluded, for each requested state F; plus the ghost
//              crossings of the resulting edge in (eps, t_F - eps).  The static BLAS is traversed
//              once for both states.
//  QT_SEG:     visibility of the segment (o, o + L d) in View_F, t in (eps, L - eps), both endpoint
//              triangles excluded; plus its ghost crossings per state.  dyn_only skips the static BLAS
//              (re-check of a shared suffix edge against dyn_Fbar, P:L429 / P:L500).
#pragma once
#include "rr_device.cuh"

namespace rr {

enum { QT_CLOSEST = 0, QT_SEG = 1 };
#define RR_EMPTY (-2147483647 - 1)  // no node (stack exhausted) / no postponed leaf
#ifndef RR_LEAF_BATCH
#define RR_LEAF_BATCH 8              // run the postponed leaf tests once this many lanes of the warp hold one
#endif

struct __align__(16) Query {
  float3 o, d;
  float tmax;            // QT_SEG: segment length L; QT_CLOSEST: unused
  int ea, eb;            // excluded triangles (origin, end)
  uint8_t type, want;    // want: bit F set -> evaluate state F
  uint8_t dyn_only, pad;
};

struct __align__(16) QRes {
  Hit h[2];        // QT_CLOSEST: hit per state (leaf < 0: miss)
  Cross c[2];      // ghost crossings per state
  uint8_t ok[2];   // QT_CLOSEST: hit found; QT_SEG: visible
};

__device__ __forceinline__ float sel(int F, float a0, float a1) { return F ? a1 : a0; }

struct Tracer {
  // query
  float3 qo, qd;
  float L, thi;
  int ea, eb, want;
  bool seg, dyn_only, done, degen;  // degen: segment too short to test (reported as not visible)
  // per-state results (kept as scalar pairs so that they stay in registers)
  float bt0, bt1;     // closest t so far
  int bl0, bl1;       // leaf of the closest hit (-1 none)
  int bi0, bi1;       // instance of the closest hit (-1 static)
  bool blk0, blk1, sblock;
  Cross c0, c1;
  float seen[8];
  int ns, seen_state;
  // current job
  int j, kind, F, k;
  bool in_job;
  float tmin, tmax, Lc;
  WRay wr;
  int node, leaf, sp;
  int stack[RR_STACK];

  __device__ __forceinline__ void begin(const DevScene& S, const Query& q) {
    qo = q.o;
    qd = q.d;
    L = q.tmax;
    ea = q.ea;
    eb = q.eb;
    want = q.want;
    seg = q.type == QT_SEG;
    dyn_only = q.dyn_only != 0;
    thi = seg ? L - S.eps : RR_TMAX;
    bt0 = bt1 = thi;
    bl0 = bl1 = -1;
    bi0 = bi1 = -1;
    blk0 = blk1 = sblock = false;
    c0 = c1 = cross_zero();
    ns = 0;
    seen_state = -1;
    j = -1;
    in_job = false;
    degen = done = seg && !(L > 2.0f * S.eps);
  }

  // set up the next job of the query; false when the query is complete
  __device__ __forceinline__ bool next_job(const DevScene& S, QCount& qc) {
    if (done) return false;
    const int NI = S.n_inst;
    const int njobs = 1 + 4 * NI;
    while (++j < njobs) {
      int root;
      float3 o = qo, d = qd;
      tmin = S.eps;
      if (j == 0) {
        kind = 0;
        F = 0;
        if (dyn_only || S.static_root < 0) continue;
        root = S.static_root;
        tmax = thi;
        if (seg) qc.shadow++; else qc.closest++;
      } else {
        int jj = j - 1, grp = jj / NI;
        k = jj - grp * NI;
        kind = grp < 2 ? 1 : 2;
        F = grp & 1;
        if (!((want >> F) & 1)) continue;
        if (seg && (sblock || (F ? blk1 : blk0))) continue;
        const DevInstance& I = S.inst[k];
        if (kind == 2 && !I.moved) continue;
        float bt = sel(F, bt0, bt1);
        if (kind == 2 && !seg && (F ? bl1 : bl0) < 0) continue;  // escaped ray: no edge, no crossings
        int place = kind == 1 ? F : 1 - F;
        tmax = kind == 1 ? bt : (seg ? L - S.eps : bt - S.eps);
        float3 inv = f3(1.0f / d.x, 1.0f / d.y, 1.0f / d.z);
        if (!inst_box(I, place, o, inv, tmin, tmax)) continue;
        o = xf_point(I.Mi[place], qo);
        d = xf_vec(I.Mi[place], qd);
        root = I.root;
        if (kind == 2) {
          qc.inst++;
          if (seen_state != F) {
            ns = 0;
            seen_state = F;
          }
        }
      }
      Lc = seg ? L : sel(F, bt0, bt1);  // segment length for the (L - t) crossing sums
      wr = make_wray(o, d);
      node = root;
      leaf = RR_EMPTY;
      sp = 0;
      in_job = true;
      return true;
    }
    done = true;
    return false;
  }

  // triangle li hit at t in (tmin, tmax); returns false when the job terminates (any hit)
  __device__ __forceinline__ bool accept(const DevScene& S, int li, float t, int id) {
    if (kind == 2) {  // ghost crossing (all hits, dedup within dedup_tol)
      for (int a = 0; a < ns; ++a)
        if (fabsf(seen[a] - t) < S.dedup_tol) return true;
      if (ns < 8) seen[ns++] = t;
      const float4* tp = S.ltris + 3 * li;
      float4 a4 = __ldg(tp), b4 = __ldg(tp + 1), c4 = __ldg(tp + 2);
      float3 nrm = norm3_exact(cross3(f3(b4.x - a4.x, b4.y - a4.y, b4.z - a4.z), f3(c4.x - a4.x, c4.y - a4.y, c4.z - a4.z)));
      float inv_c = 1.0f / fabsf(dot3(nrm, wr.d));
      float ta = t * t * inv_c, tb = (Lc - t) * (Lc - t) * inv_c;
      if (F) {
        c1.n += 1.0f; c1.s0 += inv_c; c1.sa += ta; c1.sb += tb;
      } else {
        c0.n += 1.0f; c0.s0 += inv_c; c0.sa += ta; c0.sb += tb;
      }
      return true;
    }
    if (id == ea || (seg && id == eb)) return true;
    if (seg) {  // any hit
      if (kind == 0) sblock = true;
      else if (F) blk1 = true;
      else blk0 = true;
      return false;
    }
    if (kind == 0) {
      bt0 = bt1 = t;
      bl0 = bl1 = li;
      bi0 = bi1 = -1;
    } else if (F) {
      bt1 = t;
      bl1 = li;
      bi1 = k;
    } else {
      bt0 = t;
      bl0 = li;
      bi0 = k;
    }
    tmax = t;
    return true;
  }

  // advance the current job by at most `budget` traversal steps (one inner node or one triangle each).
  // The hot fields are copied to locals so that they stay in registers for the whole turn.
  __device__ __forceinline__ void run(const DevScene& S, TCount& tc, int budget) {
    const WRay r = wr;
    const float tlo = tmin;
    float thi_ = tmax;
    int nd = node, s = sp;
    uint32_t nn = 0, nt = 0;
    for (int it = 0; it < budget; ++it) {
      if (nd >= 0) {
        nn++;
        const float4* p = S.nodes + 4 * nd;
        float4 n0 = __ldg(p), n1 = __ldg(p + 1), n2 = __ldg(p + 2), n3 = __ldg(p + 3);
        bool h0, h1;
        float t0, t1;
        box2(r, n0, n1, n2, tlo, thi_, h0, h1, t0, t1);
        int ch0 = __float_as_int(n3.x), ch1 = __float_as_int(n3.y);
        if (h0 && h1) {
          if (t1 < t0) {
            int t = ch0;
            ch0 = ch1;
            ch1 = t;
          }
          if (s < RR_STACK) stack[s++] = ch1;
          nd = ch0;
        } else if (h0) {
          nd = ch0;
        } else if (h1) {
          nd = ch1;
        } else {
          nd = s > 0 ? stack[--s] : RR_EMPTY;
        }
      } else {  // leaf: a single triangle
        int li = ~nd;
        nd = s > 0 ? stack[--s] : RR_EMPTY;
        nt++;
        const float4* tp = S.ltris + 3 * li;
        float4 a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
        float t = tri_hit(r, a, b, c);
        if (t > tlo && t < thi_) {
          tmax = thi_;
          if (!accept(S, li, t, __float_as_int(a.w))) nd = RR_EMPTY;
          thi_ = tmax;
        }
      }
      if (nd == RR_EMPTY) {
        in_job = false;
        break;
      }
    }
    node = nd;
    sp = s;
    tmax = thi_;
    tc.nodes += nn;
    tc.tris += nt;
  }

  // Warp-synchronous traversal: called by ALL 32 lanes of the warp (lanes without a job idle) for a uniform
  // number of steps, with a warp barrier per step so that the lanes stay converged.  A lane that reaches a
  // leaf postpones it (one slot, `leaf`) and keeps descending; the leaf tests run only once enough lanes of
  // the warp hold one (or lanes are stuck behind theirs), so the long triangle test runs on many lanes at
  // once (after Aila & Laine 2009, "while-while" with leaf postponing).
  __device__ __forceinline__ void run_sync(const DevScene& S, TCount& tc, int steps) {
    const WRay r = wr;
    const float tlo = tmin;
    float thi_ = tmax;
    int nd = in_job ? node : RR_EMPTY, s = sp, pend = in_job ? leaf : RR_EMPTY;
    uint32_t nn = 0, nt = 0;
    for (int it = 0; it < steps; ++it) {
      if (nd >= 0) {
        nn++;
        const float4* p = S.nodes + 4 * nd;
        float4 n0 = __ldg(p), n1 = __ldg(p + 1), n2 = __ldg(p + 2), n3 = __ldg(p + 3);
        bool h0, h1;
        float t0, t1;
        box2(r, n0, n1, n2, tlo, thi_, h0, h1, t0, t1);
        int ch0 = __float_as_int(n3.x), ch1 = __float_as_int(n3.y);
        if (h0 && h1) {
          if (t1 < t0) {
            int t = ch0;
            ch0 = ch1;
            ch1 = t;
          }
          if (s < RR_STACK) stack[s++] = ch1;
          nd = ch0;
        } else if (h0) {
          nd = ch0;
        } else if (h1) {
          nd = ch1;
        } else {
          nd = s > 0 ? stack[--s] : RR_EMPTY;
        }
      }
      if (nd < 0 && nd != RR_EMPTY && pend == RR_EMPTY) {  // postpone the reached leaf
        pend = nd;
        nd = s > 0 ? stack[--s] : RR_EMPTY;
      }
      const unsigned want = __ballot_sync(0xffffffffu, pend != RR_EMPTY);
      const unsigned stuck = __ballot_sync(0xffffffffu, pend != RR_EMPTY && nd < 0);
      if (__popc(want) >= RR_LEAF_BATCH || stuck) {
        if (pend != RR_EMPTY) {  // leaf: a single triangle
          int li = ~pend;
          pend = RR_EMPTY;
          nt++;
          const float4* tp = S.ltris + 3 * li;
          float4 a = __ldg(tp), b = __ldg(tp + 1), c = __ldg(tp + 2);
          float t = tri_hit(r, a, b, c);
          if (t > tlo && t < thi_) {
            tmax = thi_;
            if (!accept(S, li, t, __float_as_int(a.w))) nd = RR_EMPTY;
            thi_ = tmax;
          }
        }
      }
      __syncwarp();
    }
    if (in_job) {
      if (nd == RR_EMPTY && pend == RR_EMPTY) in_job = false;
      node = nd;
      leaf = pend;
      sp = s;
      tmax = thi_;
    }
    tc.nodes += nn;
    tc.tris += nt;
  }

  __device__ __forceinline__ void result(QRes& r) const {
    r.c[0] = c0;
    r.c[1] = c1;
    r.ok[0] = r.ok[1] = 0;
    r.h[0].leaf = r.h[1].leaf = -1;
    r.h[0].inst = r.h[1].inst = -1;
    r.h[0].t = r.h[1].t = 0.0f;
    if (degen) return;
    if (want & 1) {
      if (seg) r.ok[0] = (!sblock && !blk0) ? 1 : 0;
      else { r.ok[0] = bl0 >= 0 ? 1 : 0; r.h[0].t = bt0; r.h[0].leaf = bl0; r.h[0].inst = bi0; }
    }
    if (want & 2) {
      if (seg) r.ok[1] = (!sblock && !blk1) ? 1 : 0;
      else { r.ok[1] = bl1 >= 0 ? 1 : 0; r.h[1].t = bt1; r.h[1].leaf = bl1; r.h[1].inst = bi1; }
    }
  }
};

// one query traced by one thread (test kernels)
__device__ __noinline__ void run_query(const DevScene& S, const Query& q, QRes& r, QCount& qc) {
  Tracer T;
  T.begin(S, q);
  while (T.next_job(S, qc))
    while (T.in_job) T.run(S, qc.tc, 1 << 30);
  T.result(r);
}

__device__ __forceinline__ Query mk_ray(P3 o, float3 d, int excl, int want) {
  Query q;
  q.o = f3of(o);
  q.d = d;
  q.tmax = RR_TMAX;
  q.ea = excl;
  q.eb = -1;
  q.type = QT_CLOSEST;
  q.want = (uint8_t)want;
  q.dyn_only = 0;
  return q;
}
__device__ __forceinline__ Query mk_seg(P3 a, P3 b, int ea, int eb, int want, bool dyn_only = false) {
  Query q;
  double dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
  double L = sqrt(dx * dx + dy * dy + dz * dz);
  q.o = f3of(a);
  q.d = f3((float)(dx / L), (float)(dy / L), (float)(dz / L));
  q.tmax = (float)L;
  q.ea = ea;
  q.eb = eb;
  q.type = QT_SEG;
  q.want = (uint8_t)want;
  q.dyn_only = dyn_only ? 1 : 0;
  return q;
}

}  // namespace rr
