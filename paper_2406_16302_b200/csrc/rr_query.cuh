// rr_query.cuh -- the one generic ray query of the residual kernels.
//
// Every traversal of the residual kernels goes through run_batch() (a lane's whole query batch in one
// warp-synchronous loop); run_query() (one query, one traverse() per BLAS job) serves the stand-alone trace /
// segment kernels and the primal renderer.  A query is decomposed into BLAS jobs (the static BLAS once, then
// each dynamic instance under the transform of each requested state, then each MOVED instance under the other
// state's transform for the ghost crossings); both loops share the node and triangle steps (node_step,
// tri_hit), so lanes that trace queries of different kinds execute one instruction stream.
//
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
// Query::want: bit F = evaluate state F; QW_NO_CROSS = the caller does not use this query's ghost crossings (their
// jobs are skipped; QRes::c stays zero)
enum { QW_NO_CROSS = 4 };
// cache policy of the BVH node / leaf-row loads (tuning knob; __ldg = read-only path through L1)
#ifndef RR_NODE_LD
#define RR_NODE_LD __ldg
#endif
#ifndef RR_TRI_LD
#define RR_TRI_LD __ldg
#endif







struct __align__(16) Query {
  float3 o, d;
  float tmax;            // QT_SEG: segment length L; QT_CLOSEST: unused
  int ea, eb;            // excluded triangles (origin, end)
  uint8_t type, want;    // want: bit F set -> evaluate state F
  uint8_t dyn_only;
  uint8_t rev;           // RR_T6_TOWARD_LIGHT kernels: the path runs this edge against the query's direction
  // x_G of a T4 / T5 / T6 sample on this ray / segment (reading 12): seed_t > 0 its distance,
  // seed_tri its ghost triangle.  The ghost-crossing jobs skip that crossing (a hit of triangle seed_tri, or within
  // dedup_tol of seed_t); the consumer adds it exactly (add_seed), so it counts once whether or not the
  // non-watertight triangle test finds it.  seed_t = 0: none.
  float seed_t;
  int seed_tri;
};

struct __align__(16) QRes {
  Hit h[2];        // QT_CLOSEST: hit per state (leaf < 0: miss)
  Cross c[2];      // ghost crossings per state
  uint8_t ok[2];   // QT_CLOSEST: hit found; QT_SEG: visible
};

// ------------------------------------------------------------------------------------------------
// BVH2 traversal (64-byte nodes, single-triangle leaves; rr_lbvh.cu): nearer hit child first, the other
// pushed.
//
// Convergence (B200 / independent thread scheduling).  Lanes of a warp that take different branches of a
// traversal iteration (descend / push / pop / leaf) are merged again only at a convergence barrier; with the
// barrier after the loop (where the compiler puts it for a plain while loop) every lane runs its whole traversal
// alone: ncu measured 1.6 active threads per warp instruction on random camera rays in a stand-alone trace kernel
// (profiles/r2_trace_convergence.md).  The SYNC loop therefore ends each iteration with a __ballot_sync over the
// lanes still traversing, and a lane that has finished leaves after that ballot (its bit is cleared from the next
// iteration's mask): the group stays converged, one node (or leaf) per lane per iteration -- same nodes, same
// results, 372 -> 1193 Mrays/s on config 4 (rr_trace), 8.3 active threads per instruction.  The residual
// megakernels keep the plain loop (SYNC = false; see traverse()).
// ------------------------------------------------------------------------------------------------

// one internal node: both child boxes against (tmin, tmax); descend into the nearer hit child and push the other.
// Returns true when neither child is hit (the caller pops).
__device__ __forceinline__ bool node_step(const DevScene& S, const WRay& r, float tmin, float tmax, int& node,
                                          int* stack, int& sp) {
  const float4* nd = S.nodes + 4 * node;
  float4 n0 = RR_NODE_LD(nd), n1 = RR_NODE_LD(nd + 1), n2 = RR_NODE_LD(nd + 2), n3 = RR_NODE_LD(nd + 3);
  bool h0, h1;
  float t0, t1;
  box2(r, n0, n1, n2, tmin, tmax, h0, h1, t0, t1);
  int c0 = __float_as_int(n3.x), c1 = __float_as_int(n3.y);
  if (h0 && h1) {
    if (t1 < t0) {
      int t = c0;
      c0 = c1;
      c1 = t;
    }
    if (sp < RR_STACK) stack[sp++] = c1;
    node = c0;
    return false;
  }
  if (h0) {
    node = c0;
    return false;
  }
  if (h1) {
    node = c1;
    return false;
  }
  return true;
}

// leaf triangle li: the unit-triangle test (Woop 2004): plane distance, then barycentrics u, v of the plane point.
// True for a hit with t in (tmin, tmax).
__device__ __forceinline__ bool tri_hit(const DevScene& S, const WRay& r, int li, float tmin, float tmax, float& t) {
  const float4* xp = S.lxf + 3 * li;
  const float4 m2 = RR_TRI_LD(xp + 2);
  // explicit FMAs (the library builds with -fmad=false; rounding here is the same for both states)
  const float oz = fmaf(m2.x, r.o.x, fmaf(m2.y, r.o.y, fmaf(m2.z, r.o.z, m2.w)));
  const float dz = fmaf(m2.x, r.d.x, fmaf(m2.y, r.d.y, m2.z * r.d.z));
  t = __fdividef(-oz, dz);  // 2 ulp; the hit point itself is recomputed in fp64 (hit_pv)
  if (!(t > tmin && t < tmax)) return false;
  const float4 m0 = RR_TRI_LD(xp);
  const float u = fmaf(t, fmaf(m0.x, r.d.x, fmaf(m0.y, r.d.y, m0.z * r.d.z)),
                       fmaf(m0.x, r.o.x, fmaf(m0.y, r.o.y, fmaf(m0.z, r.o.z, m0.w))));
  if (!(u >= 0.0f && u <= 1.0f)) return false;
  const float4 m1 = RR_TRI_LD(xp + 1);
  const float v = fmaf(t, fmaf(m1.x, r.d.x, fmaf(m1.y, r.d.y, m1.z * r.d.z)),
                       fmaf(m1.x, r.o.x, fmaf(m1.y, r.o.y, fmaf(m1.z, r.o.z, m1.w))));
  return v >= 0.0f && u + v <= 1.0f;
}

// One traversal of one BLAS.  leaf(li, t, tmax, id) is called for every triangle hit with t in (tmin, tmax) and
// returns the new tmax (negative: terminate).  id = the triangle's global id (stored in the first vertex's w).
// SYNC: the ballot-per-iteration loop (stand-alone kernels, whose lanes enter converged).  The residual
// megakernels use SYNC = false: there the lanes reach a traversal in small groups (per query slot and BLAS job),
// and the ballot, the uniform job loop and the extra live registers cost more than the reconvergence returns
// (config 4: 9.63 s vs 8.42 s, round-2 rejected designs).
template <bool COUNT, bool SYNC, class Leaf>
__device__ __forceinline__ void traverse(const DevScene& S, int root, const WRay& r, float tmin, float tmax, Leaf leaf,
                                         TCount& tc) {
  int stack[RR_STACK];
  int sp = 0;
  int node = root;
  uint32_t nn = 0, nt = 0;
  if constexpr (!SYNC) {
    // the residual megakernels' loop, as tuned there (descend with continue, pop at the bottom)
    while (true) {
      if (node >= 0) {
        if (COUNT) nn++;
        const float4* nd = S.nodes + 4 * node;
        float4 n0 = RR_NODE_LD(nd), n1 = RR_NODE_LD(nd + 1), n2 = RR_NODE_LD(nd + 2), n3 = RR_NODE_LD(nd + 3);
        bool h0, h1;
        float t0, t1;
        box2(r, n0, n1, n2, tmin, tmax, h0, h1, t0, t1);
        int c0 = __float_as_int(n3.x), c1 = __float_as_int(n3.y);
        if (h0 && h1) {
          if (t1 < t0) {
            int t = c0;
            c0 = c1;
            c1 = t;
          }
          if (sp < RR_STACK) stack[sp++] = c1;
          node = c0;
          continue;
        } else if (h0) {
          node = c0;
          continue;
        } else if (h1) {
          node = c1;
          continue;
        }
      } else {
        int li = ~node;
        if (COUNT) nt++;
        float t;
        if (tri_hit(S, r, li, tmin, tmax, t)) {
          tmax = leaf(li, t, tmax, __float_as_int(__ldg(S.ltris + 3 * li).w));
          if (tmax < 0.0f) break;
        }
      }
      if (sp == 0) break;
      node = stack[--sp];
    }
    tc.nodes += nn;
    tc.tris += nt;
    return;
  }
  unsigned live = __activemask();
  bool done = false;
  while (true) {
    bool pop;
    if (node >= 0) {
      if (COUNT) nn++;
      pop = node_step(S, r, tmin, tmax, node, stack, sp);
    } else {
      const int li = ~node;
      if (COUNT) nt++;
      pop = true;
      float t;
      if (tri_hit(S, r, li, tmin, tmax, t)) {
        tmax = leaf(li, t, tmax, __float_as_int(__ldg(S.ltris + 3 * li).w));
        if (tmax < 0.0f) done = true;
      }
    }
    if (pop && !done) {
      if (sp == 0) done = true;
      else node = stack[--sp];
    }
    live = __ballot_sync(live, !done);  // the lanes still traversing: the next iteration's group
    if (done) break;
  }
  tc.nodes += nn;
  tc.tris += nt;
}

#if defined(RR_VAR_KERNELS) && RR_VAR_KERNELS
// RR_T6_TOWARD_LIGHT: 4 pi p_dir(d | x) of T6's direction d at a ghost point x (the oracle's t6_pdir):
// (2 / n_e) #{e : d . (c_e - x) > 0}; 1 for the uniform sphere
__device__ __forceinline__ float t6_pdir4pi(const float4* c, int n, float3 x, float3 d) {
  int k = 0;
  for (int e = 0; e < n; ++e) {
    const float4 ce = __ldg(c + e);
    k += dot3(d, f3(ce.x - x.x, ce.y - x.y, ce.z - x.z)) > 0.0f ? 1 : 0;
  }
  return 2.0f * (float)k / (float)n;
}
#endif

template <bool COUNT, bool SYNC>
__device__ __forceinline__ void run_query(const DevScene& S, const Query& q, QRes& r, QCount& qc
#if defined(RR_VAR_KERNELS) && RR_VAR_KERNELS
                                          , const float4* t6c, int t6n
#endif
) {
  const bool seg = q.type == QT_SEG;
  const float L = q.tmax;
  r.ok[0] = r.ok[1] = 0;
  r.c[0] = r.c[1] = cross_zero();
  r.h[0].t = r.h[1].t = 0.0f;
  r.h[0].leaf = r.h[1].leaf = -1;
  r.h[0].inst = r.h[1].inst = -1;
  if (seg && !(L > 2.0f * S.eps)) return;  // too short to test: reported as not visible
  float best_t[2], thi = seg ? L - S.eps : RR_TMAX;
  int best_leaf[2] = {-1, -1}, best_inst[2] = {-1, -1};
  best_t[0] = best_t[1] = thi;
  bool blocked[2] = {false, false};
  bool sblock = false;
  float seen[8];
  int ns = 0, seen_state = -1;
  const int NI = S.n_inst;
  const int njobs = 1 + 4 * NI;
  // SYNC: the job loop is uniform over the calling group (every lane runs every j; a lane that skips job j waits
  // at the __syncwarp below), so the lanes that do need job j enter traverse() together and stay converged.
  // Otherwise a skipped job is a plain `continue` (mine stays true).
  const unsigned grp_mask = SYNC ? __activemask() : 0u;
#define RR_SKIP_JOB          \
  {                          \
    if (SYNC) mine = false;  \
    else continue;           \
  }
  for (int j = 0; j < njobs; ++j) {
    int kind, F = 0, k = -1;
    bool mine = true;
    if (j == 0) {
      kind = 0;
      if (q.dyn_only || S.static_root < 0) RR_SKIP_JOB
    } else {
      int jj = j - 1, grp = jj / NI;
      k = jj - grp * NI;
      kind = grp < 2 ? 1 : 2;
      F = grp & 1;
      if (!((q.want >> F) & 1)) RR_SKIP_JOB
      else if (seg && (sblock || blocked[F])) RR_SKIP_JOB
      else if (kind == 2 && (!S.inst[k].moved || (q.want & QW_NO_CROSS))) RR_SKIP_JOB
      else if (kind == 2 && !seg && best_leaf[F] < 0) RR_SKIP_JOB  // escaped ray: no edge, no crossings
    }
    if (mine) {
    int root, place = 0;
    float tmin = S.eps, tmax;
    float3 o = q.o, d = q.d;
    if (kind == 0) {
      root = S.static_root;
      tmax = thi;
      if (seg) qc.shadow++; else qc.closest++;
    } else {
      const DevInstance& I = S.inst[k];
      place = kind == 1 ? F : 1 - F;
      tmax = kind == 1 ? best_t[F] : (seg ? L - S.eps : best_t[F] - S.eps);
      float3 inv = rcp3(d);
      if (!inst_box(I, place, o, inv, tmin, tmax)) RR_SKIP_JOB
      o = xf_point(I.Mi[place], q.o);
      d = xf_vec(I.Mi[place], q.d);
      root = I.root;
      if (mine && kind == 2) {
        qc.inst++;
        if (seen_state != F) {
          ns = 0;
          seen_state = F;
        }
      }
    }
    if (mine) {
    const float Lc = seg ? L : best_t[F];  // segment length for the (L - t) crossing sums
    WRay wr = make_wray(o, d);
#if RR_COUNT_JOBS
    const uint32_t nodes0 = COUNT ? qc.tc.nodes : 0;
#endif
    traverse<COUNT, SYNC>(S, root, wr, tmin, tmax, [&](int li, float t, float tm, int id) -> float {
      if (kind == 2) {  // ghost crossing (all hits, dedup within dedup_tol)
        if (fabsf(t - q.seed_t) < S.dedup_tol || (id == q.seed_tri && q.seed_t > 0.0f)) return tm;  // x_G: added exactly
        for (int a = 0; a < ns; ++a)
          if (fabsf(seen[a] - t) < S.dedup_tol) return tm;
        seen[ns < 8 ? ns++ : 7] = t;  // beyond 8 crossings: dedup against the first 7 and the latest one
        const float4* tp = S.ltris + 3 * li;
        float4 a4 = __ldg(tp), b4 = __ldg(tp + 1), c4 = __ldg(tp + 2);
        float3 nrm = norm3_exact(cross3(f3(b4.x - a4.x, b4.y - a4.y, b4.z - a4.z), f3(c4.x - a4.x, c4.y - a4.y, c4.z - a4.z)));
        float inv_c = 1.0f / fabsf(dot3(nrm, d));
#if defined(RR_VAR_KERNELS) && RR_VAR_KERNELS
        // s0 carries 4 pi p_dir of the path's direction through this crossing (T6's candidate pdf)
        const float3 xw = q.o + q.d * t;
        const float pd = t6c ? t6_pdir4pi(t6c, t6n, xw, q.rev ? q.d * -1.0f : q.d) : 1.0f;
#else
        const float pd = 1.0f;
#endif
        Cross& cc = r.c[F];
        cc.n += 1.0f;
        cc.s0 += inv_c * pd;
        cc.sa += t * t * inv_c;
        cc.sb += (Lc - t) * (Lc - t) * inv_c;
        return tm;
      }
      if (id == q.ea || (seg && id == q.eb)) return tm;
      if (seg) {  // any hit
        if (kind == 0) sblock = true; else blocked[F] = true;
        return -1.0f;
      }
      if (kind == 0) {
        best_t[0] = best_t[1] = t;
        best_leaf[0] = best_leaf[1] = li;
        best_inst[0] = best_inst[1] = -1;
      } else {
        best_t[F] = t;
        best_leaf[F] = li;
        best_inst[F] = k;
      }
      return t;
    }, qc.tc);
#if RR_COUNT_JOBS
    if (COUNT && kind != 0) {
      qc.tc.inst_nodes += qc.tc.nodes - nodes0;
      if (kind == 2) qc.tc.ghost_nodes += qc.tc.nodes - nodes0;
    }
#endif
    }  // mine (after the instance-box test)
    }  // mine
    if (SYNC) __syncwarp(grp_mask);
  }
#undef RR_SKIP_JOB
  for (int F = 0; F < 2; ++F) {
    if (!((q.want >> F) & 1)) continue;
    if (seg) {
      r.ok[F] = (!sblock && !blocked[F]) ? 1 : 0;
    } else {
      r.ok[F] = best_leaf[F] >= 0 ? 1 : 0;
      r.h[F].t = best_t[F];
      r.h[F].leaf = best_leaf[F];
      r.h[F].inst = best_inst[F];
    }
  }
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
#if defined(RR_VAR_KERNELS) && RR_VAR_KERNELS
  q.rev = 0;
#endif
  q.seed_t = 0.0f;
  q.seed_tri = -1;
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
#if defined(RR_VAR_KERNELS) && RR_VAR_KERNELS
  q.rev = 0;
#endif
  q.seed_t = 0.0f;
  q.seed_tri = -1;
  return q;
}
// the crossing at x_G (distance t along an edge of length L, 1/|cos_G| = ic) added to an edge's crossing sums
__device__ __forceinline__ Cross add_seed(Cross c, float t, float L, float ic) {
  c.n += 1.0f;
  c.s0 += ic;
  c.sa += t * t * ic;
  c.sb += (L - t) * (L - t) * ic;
  return c;
}

}  // namespace rr
