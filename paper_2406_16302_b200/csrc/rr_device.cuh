// rr_device.cuh -- device-side scene layout, Philox, BSDFs, camera and LBVH traversal (sm_100a).
//
// Paper: /root/reference/PAPER.md (P:Lnnn).  Readings of unstated details: SURVEY.md 8(c) C1-C12, listed
// in DESIGN.md.  fp32 throughout; the only shared "data" with any other implementation are the input
// arrays and the fp32 triangle-selection CDFs built by the host code of this library (rr_capi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define RR_MAX_INST 8
#define RR_MAXD 10          // RR_MAX_DEPTH: max path edges
#define RR_MAXV (RR_MAXD + 1)
#define RR_PI_F 3.14159265358979323846f
#define RR_INV_PI_F 0.318309886183790671538f
#define RR_STACK 64
#define RR_TMAX 1.0e30f  // every query's tmax is below the 'empty child' sentinel box at 3e38

namespace rr {

// ------------------------------------------------------------------------------------------------
// float3 helpers
// ------------------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ float3 f3(float x, float y, float z) { return make_float3(x, y, z); }
__host__ __device__ __forceinline__ float3 operator+(float3 a, float3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
__host__ __device__ __forceinline__ float3 operator-(float3 a, float3 b) { return f3(a.x - b.x, a.y - b.y, a.z - b.z); }
__host__ __device__ __forceinline__ float3 operator*(float3 a, float s) { return f3(a.x * s, a.y * s, a.z * s); }
__host__ __device__ __forceinline__ float3 operator*(float s, float3 a) { return f3(a.x * s, a.y * s, a.z * s); }
__host__ __device__ __forceinline__ float3 mul3(float3 a, float3 b) { return f3(a.x * b.x, a.y * b.y, a.z * b.z); }
__host__ __device__ __forceinline__ float dot3(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__host__ __device__ __forceinline__ float3 cross3(float3 a, float3 b) {
  return f3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ float3 norm3_exact(float3 a) { return a * (1.0f / sqrtf(dot3(a, a))); }
__device__ __forceinline__ float norm3f(float3 a) { return sqrtf(dot3(a, a)); }
__device__ __forceinline__ bool eq3(float3 a, float3 b) {
  return __float_as_uint(a.x) == __float_as_uint(b.x) && __float_as_uint(a.y) == __float_as_uint(b.y) &&
         __float_as_uint(a.z) == __float_as_uint(b.z);
}
// Path-vertex positions are kept in fp64 (P3): a hit point is the exact intersection of the fp32 ray with
// the triangle's plane, and the vector between two vertices is formed in fp64 before it is rounded, so a
// short path edge keeps full fp32 relative precision in its direction and length.
typedef double3 P3;
__device__ __forceinline__ P3 p3(float3 a) { return make_double3(a.x, a.y, a.z); }
__device__ __forceinline__ float3 f3of(P3 a) { return f3((float)a.x, (float)a.y, (float)a.z); }
__device__ __forceinline__ float3 sub3(P3 a, P3 b) { return f3((float)(a.x - b.x), (float)(a.y - b.y), (float)(a.z - b.z)); }
__device__ __forceinline__ bool eqp(P3 a, P3 b) {
  return __double_as_longlong(a.x) == __double_as_longlong(b.x) && __double_as_longlong(a.y) == __double_as_longlong(b.y) &&
         __double_as_longlong(a.z) == __double_as_longlong(b.z);
}
__device__ __forceinline__ P3 xf_point_d(const float* m, P3 p) {
  return make_double3(fma((double)m[0], p.x, fma((double)m[1], p.y, fma((double)m[2], p.z, (double)m[3]))),
                      fma((double)m[4], p.x, fma((double)m[5], p.y, fma((double)m[6], p.z, (double)m[7]))),
                      fma((double)m[8], p.x, fma((double)m[9], p.y, fma((double)m[10], p.z, (double)m[11]))));
}
__device__ __forceinline__ float3 xf_point(const float* m, float3 p) {
  return f3(fmaf(m[0], p.x, fmaf(m[1], p.y, fmaf(m[2], p.z, m[3]))),
            fmaf(m[4], p.x, fmaf(m[5], p.y, fmaf(m[6], p.z, m[7]))),
            fmaf(m[8], p.x, fmaf(m[9], p.y, fmaf(m[10], p.z, m[11]))));
}
__device__ __forceinline__ float3 xf_vec(const float* m, float3 v) {
  return f3(fmaf(m[0], v.x, fmaf(m[1], v.y, m[2] * v.z)), fmaf(m[4], v.x, fmaf(m[5], v.y, m[6] * v.z)),
            fmaf(m[8], v.x, fmaf(m[9], v.y, m[10] * v.z)));
}

// ------------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. 2011).  Counter: (i lo, i hi, l | side << 8,
// 2*slot + call), key = seed.  u01(x) = (x >> 8) * 2^-24 (exact in fp32).
// ------------------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
#else
    uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
__device__ __forceinline__ float u01f(uint32_t x) { return (float)(x >> 8) * (1.0f / 16777216.0f); }

struct Rng {  // the random numbers of one residual sample (technique l, side, index i)
  uint32_t i_lo, i_hi, ls, k0, k1;
  __device__ void dims(uint32_t slot, float d[8]) const {
    uint2 key = make_uint2(k0, k1);
    uint4 a = philox4x32_10(make_uint4(i_lo, i_hi, ls, 2u * slot), key);
    uint4 b = philox4x32_10(make_uint4(i_lo, i_hi, ls, 2u * slot + 1u), key);
    d[0] = u01f(a.x); d[1] = u01f(a.y); d[2] = u01f(a.z); d[3] = u01f(a.w);
    d[4] = u01f(b.x); d[5] = u01f(b.y); d[6] = u01f(b.z); d[7] = u01f(b.w);
  }
  __device__ void dims_lo(uint32_t slot, float d[4]) const {  // d0..d3 only
    uint4 a = philox4x32_10(make_uint4(i_lo, i_hi, ls, 2u * slot), make_uint2(k0, k1));
    d[0] = u01f(a.x); d[1] = u01f(a.y); d[2] = u01f(a.z); d[3] = u01f(a.w);
  }
  __device__ void dims_hi(uint32_t slot, float d[4]) const {  // d4..d7 only
    uint4 b = philox4x32_10(make_uint4(i_lo, i_hi, ls, 2u * slot + 1u), make_uint2(k0, k1));
    d[0] = u01f(b.x); d[1] = u01f(b.y); d[2] = u01f(b.z); d[3] = u01f(b.w);
  }
};

// ------------------------------------------------------------------------------------------------
// Device scene.  Object flags: bit0 edited (dynamic set), bit1 moved (ghost set), bit2 emitter.
// BVH2 node = 4 float4 (64 B): (c0.lo.x, c0.hi.x, c0.lo.y, c0.hi.y), (c1 ... same), (c0.lo.z, c0.hi.z,
// c1.lo.z, c1.hi.z), (child0, child1 as int bits, -, -).  child >= 0: internal node, < 0: leaf ~idx.
// Leaf triangle = 3 float4 (v0.xyz + global tri id bits, v1, v2) in BLAS space.
// ------------------------------------------------------------------------------------------------
enum { OBJ_EDITED = 1u, OBJ_MOVED = 2u, OBJ_EMITTER = 4u };

struct DevInstance {
  int obj, root, moved, pad;
  float M[2][12];   // object -> world, state 0 = new (N), 1 = old (O)
  float Mi[2][12];  // world -> object
  float lo[2][3], hi[2][3];
};

struct DevScene {
  const float4* nodes;
  const float4* ltris;
  const float4* lxf;          // [3 per leaf] world->unit-triangle rows (rr_lbvh.cu unit_triangle)
  int static_root;  // -1: no static geometry
  int n_inst;
  DevInstance inst[RR_MAX_INST];
  const float4* tverts;      // [3T] by global triangle id (object space for dynamic objects)
  const uint32_t* tri_obj;
  const uint32_t* obj_flags;
  const int* obj_inst;
  const uint32_t* obj_mat[2];
  const float4* mat;         // albedo rgb, alpha
  const uint32_t* mat_type;   // 0 Lambert, 1 GGX; RR_VNDF renders get a copy with GGX as 2 (visible normals)
  const float4* obj_emit;
  const int* obj_emitter;
  int n_emit;
  const int* emit_off;
  const int* emit_cnt;
  const float* emit_pL;
  const uint32_t* emit_tris;
  const float* emit_cdf;
  int n_edited;
  const uint32_t* edited_tris;
  const float* edited_cdf;
  float pA_D;
  int n_moved;
  const uint32_t* moved_tris;
  const float* moved_cdf;
  float pA_G;
  float3 cam_pos, cf, cr, cu;
  float tanX, tanY, Aplane;
  int W, H;
  float eps, diag, dedup_tol;
};

// ------------------------------------------------------------------------------------------------
// BSDFs: two-sided, reflection only; wi points toward the previous vertex.
// ------------------------------------------------------------------------------------------------
struct Mat {
  uint32_t type;
  float3 albedo;
  float alpha;
};
__device__ __forceinline__ Mat load_mat(const DevScene& S, uint32_t obj, int F) {
  uint32_t m = __ldg(&S.obj_mat[F][obj]);
  float4 a = __ldg(&S.mat[m]);
  Mat r;
  r.type = __ldg(&S.mat_type[m]);
  r.albedo = f3(a.x, a.y, a.z);
  r.alpha = a.w;
  return r;
}
__device__ __forceinline__ void onb(float3 n, float3& b1, float3& b2) {  // Duff et al. 2017
  float sign = copysignf(1.0f, n.z);
  float a = -1.0f / (sign + n.z);
  float b = n.x * n.y * a;
  b1 = f3(1.0f + sign * n.x * n.x * a, sign * b, -sign * n.x);
  b2 = f3(b, sign + n.y * n.y * a, -n.y);
}
__device__ __forceinline__ float3 to_world(float3 n, float x, float y, float z) {
  float3 b1, b2;
  onb(n, b1, b2);
  return b1 * x + b2 * y + n * z;
}
// D(h) = a^2 / (pi ((n.h)^2 (a^2 - 1) + 1)^2), with the denominator written as sin^2 + a^2 cos^2 and
// sin^2 = |n x h|^2 so that sharp lobes (a = 0.1) do not lose fp32 precision to cancellation
__device__ __forceinline__ float ggx_D(float a, float3 n, float3 h) {
  float a2 = a * a;
  float nh = dot3(n, h);
  float3 c = cross3(n, h);
  float t = dot3(c, c) + a2 * nh * nh;
  return a2 / (RR_PI_F * t * t);
}
__device__ __forceinline__ float ggx_G1(float a, float nv) {
  nv = fabsf(nv);
  return 2.0f * nv / (nv + sqrtf(a * a + (1.0f - a * a) * nv * nv));
}
__device__ __forceinline__ float3 bsdf_eval(const Mat& m, float3 n, float3 wi, float3 wo) {
  float3 ns = dot3(n, wi) > 0.0f ? n : n * -1.0f;
  float ci = dot3(ns, wi), co = dot3(ns, wo);
  if (!(ci > 0.0f) || !(co > 0.0f)) return f3(0.f, 0.f, 0.f);
  if (m.type == 0) return m.albedo * RR_INV_PI_F;
  float3 h = norm3_exact(wi + wo);
  float D = ggx_D(m.alpha, ns, h);
  float G = ggx_G1(m.alpha, ci) * ggx_G1(m.alpha, co);
  float x = 1.0f - fabsf(dot3(wi, h));
  float x2 = x * x;
  float fw = x2 * x2 * x;
  float3 F = m.albedo + (f3(1.f, 1.f, 1.f) - m.albedo) * fw;
  return F * (D * G / (4.0f * ci * co));
}
// GGX visible-normal sampling (RR_VNDF) is compiled only into the kernels of rr_residual_vndf.cu
// (RR_VNDF_KERNELS = 1): its branches in the default kernels cost 2.5% of a config-4 render
#if defined(RR_VNDF_KERNELS) && RR_VNDF_KERNELS
__device__ __forceinline__ float ggx_vndf_pdf(float a, float ci, float3 ns, float3 h) {
  return ggx_G1(a, ci) * ggx_D(a, ns, h) / (4.0f * ci);
}
#endif
__device__ __forceinline__ float bsdf_pdf(const Mat& m, float3 n, float3 wi, float3 wo) {
  float3 ns = dot3(n, wi) > 0.0f ? n : n * -1.0f;
  float ci = dot3(ns, wi), co = dot3(ns, wo);
  if (!(ci > 0.0f) || !(co > 0.0f)) return 0.0f;
  if (m.type == 0) return co * RR_INV_PI_F;
  float3 h = norm3_exact(wi + wo);
  // VNDF: D_wi(h) / (4 wo.h) with D_wi(h) = G1(wi) (wi.h) D(h) / (n.wi) and wo.h = wi.h
#if defined(RR_VNDF_KERNELS) && RR_VNDF_KERNELS
  if (m.type == 2) return ggx_vndf_pdf(m.alpha, ci, ns, h);
#endif
  return ggx_D(m.alpha, ns, h) * fabsf(dot3(ns, h)) / (4.0f * fabsf(dot3(wo, h)));
}
// half vector from the GGX visible normals of wi (Heitz 2018, isotropic): stretch wi, sample the projected
// hemisphere of the stretched view (disk point warped by s = (1 + Vh_z) / 2), unstretch; frame of to_world
#if defined(RR_VNDF_KERNELS) && RR_VNDF_KERNELS
__device__ __forceinline__ float3 ggx_vndf_half(float a, float3 ns, float3 wi, float u1, float u2) {
  float3 b1, b2;
  onb(ns, b1, b2);
  float3 vh = norm3_exact(f3(a * dot3(wi, b1), a * dot3(wi, b2), dot3(wi, ns)));
  float lensq = vh.x * vh.x + vh.y * vh.y;
  float3 T1 = lensq > 0.0f ? f3(-vh.y, vh.x, 0.0f) * (1.0f / sqrtf(lensq)) : f3(1.0f, 0.0f, 0.0f);
  float3 T2 = cross3(vh, T1);
  float r = sqrtf(u1), sp, cp;
  sincosf(2.0f * RR_PI_F * u2, &sp, &cp);
  float t1 = r * cp, t2 = r * sp;
  float sw = 0.5f * (1.0f + vh.z);
  t2 = (1.0f - sw) * sqrtf(1.0f - t1 * t1) + sw * t2;
  float3 nh = T1 * t1 + T2 * t2 + vh * sqrtf(fmaxf(0.0f, 1.0f - t1 * t1 - t2 * t2));
  float3 hl = norm3_exact(f3(a * nh.x, a * nh.y, fmaxf(0.0f, nh.z)));
  return to_world(ns, hl.x, hl.y, hl.z);
}
#endif
__device__ __forceinline__ bool bsdf_sample(const Mat& m, float3 n, float3 wi, float u1, float u2, float3& wo) {
  float3 ns = dot3(n, wi) > 0.0f ? n : n * -1.0f;
  if (m.type == 0) {
    float r = sqrtf(u1), phi = 2.0f * RR_PI_F * u2;
    float s, c;
    sincosf(phi, &s, &c);
    wo = norm3_exact(to_world(ns, r * c, r * s, sqrtf(fmaxf(0.0f, 1.0f - u1))));
    return true;
  }
  float a = m.alpha;
#if defined(RR_VNDF_KERNELS) && RR_VNDF_KERNELS
  if (m.type == 2) {
    float3 h = norm3_exact(ggx_vndf_half(a, ns, wi, u1, u2));
    float3 w = h * (2.0f * dot3(wi, h)) - wi;
    if (!(dot3(w, ns) > 0.0f)) return false;
    wo = norm3_exact(w);
    return true;
  }
#endif
  float tan2 = a * a * u1 / (1.0f - u1);
  float ct = 1.0f / sqrtf(1.0f + tan2);
  float st = sqrtf(tan2) * ct;  // sin = tan cos: no cancellation for the small angles of sharp lobes
  float s, c;
  sincosf(2.0f * RR_PI_F * u2, &s, &c);
  float3 h = norm3_exact(to_world(ns, st * c, st * s, ct));
  float3 w = h * (2.0f * dot3(wi, h)) - wi;
  if (!(dot3(w, ns) > 0.0f)) return false;
  wo = norm3_exact(w);
  return true;
}
__device__ __forceinline__ bool rough_enough(const Mat& m, float alpha_min) { return m.type == 0 || m.alpha >= alpha_min; }

// ------------------------------------------------------------------------------------------------
// camera (C1): pinhole, A_plane = 4 tanX tanY, W_e = 1/(A cos^4), p(x_E) := 1
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ float3 camera_dir(const DevScene& S, float sx, float sy) {
  return norm3_exact(S.cf + S.cr * ((2.0f * sx / (float)S.W - 1.0f) * S.tanX) +
                     S.cu * ((1.0f - 2.0f * sy / (float)S.H) * S.tanY));
}
__device__ __forceinline__ int project(const DevScene& S, P3 x) {
  float3 q = sub3(x, p3(S.cam_pos));
  float c = dot3(q, S.cf);
  if (!(c > 0.0f)) return -1;
  float sx = (dot3(q, S.cr) / (c * S.tanX) + 1.0f) * (float)S.W * 0.5f;
  float sy = (1.0f - dot3(q, S.cu) / (c * S.tanY)) * (float)S.H * 0.5f;
  float fx = floorf(sx), fy = floorf(sy);
  if (!(fx >= 0.0f) || !(fy >= 0.0f) || fx >= (float)S.W || fy >= (float)S.H) return -1;
  return (int)fy * S.W + (int)fx;
}

// ------------------------------------------------------------------------------------------------
// ray / box.  The ray / triangle test is the unit-triangle test of rr_query.cuh (rows built by rr_lbvh.cu).
// ------------------------------------------------------------------------------------------------
struct WRay {
  float3 o, d, inv;
};
// reciprocal direction for the slab tests: the fast (2-ulp, no slow path) reciprocal is inside the tests'
// conservative margin (box2: 1.0000004)
__device__ __forceinline__ float3 rcp3(float3 d) {
  return f3(__fdividef(1.0f, d.x), __fdividef(1.0f, d.y), __fdividef(1.0f, d.z));
}
__device__ __forceinline__ WRay make_wray(float3 o, float3 d) {
  WRay r;
  r.o = o;
  r.d = d;
  r.inv = rcp3(d);
  return r;
}
__device__ __forceinline__ void box2(const WRay& r, float4 n0, float4 n1, float4 n2, float tmin, float tmax,
                                     bool& h0, bool& h1, float& t0, float& t1) {
  float lx0 = (n0.x - r.o.x) * r.inv.x, hx0 = (n0.y - r.o.x) * r.inv.x;
  float ly0 = (n0.z - r.o.y) * r.inv.y, hy0 = (n0.w - r.o.y) * r.inv.y;
  float lz0 = (n2.x - r.o.z) * r.inv.z, hz0 = (n2.y - r.o.z) * r.inv.z;
  float lx1 = (n1.x - r.o.x) * r.inv.x, hx1 = (n1.y - r.o.x) * r.inv.x;
  float ly1 = (n1.z - r.o.y) * r.inv.y, hy1 = (n1.w - r.o.y) * r.inv.y;
  float lz1 = (n2.z - r.o.z) * r.inv.z, hz1 = (n2.w - r.o.z) * r.inv.z;
  float a0 = fmaxf(fmaxf(fminf(lx0, hx0), fminf(ly0, hy0)), fmaxf(fminf(lz0, hz0), tmin));
  float b0 = fminf(fminf(fmaxf(lx0, hx0), fmaxf(ly0, hy0)), fminf(fmaxf(lz0, hz0), tmax));
  float a1 = fmaxf(fmaxf(fminf(lx1, hx1), fminf(ly1, hy1)), fmaxf(fminf(lz1, hz1), tmin));
  float b1 = fminf(fminf(fmaxf(lx1, hx1), fmaxf(ly1, hy1)), fminf(fmaxf(lz1, hz1), tmax));
  const float g = 1.0000004f;  // conservative slab test
  h0 = a0 <= b0 * g;
  h1 = a1 <= b1 * g;
  t0 = a0;
  t1 = a1;
}

#ifndef RR_COUNT_JOBS
#define RR_COUNT_JOBS 0  // 1: diagnostic build (tools/variants.py) that also splits node fetches by BLAS job kind
#endif
struct TCount {  // traversal work of one thread: internal nodes fetched, triangles tested (64 B / 48 B each)
  uint32_t nodes, tris;
#if RR_COUNT_JOBS
  uint32_t inst_nodes, ghost_nodes;  // of which in dynamic-instance BLAS jobs / ghost-crossing jobs (diagnostic build)
#endif
};


// world AABB of instance k in state F vs ray segment
__device__ __forceinline__ bool inst_box(const DevInstance& I, int F, float3 o, float3 inv, float tmin, float tmax) {
  float lx = (I.lo[F][0] - o.x) * inv.x, hx = (I.hi[F][0] - o.x) * inv.x;
  float ly = (I.lo[F][1] - o.y) * inv.y, hy = (I.hi[F][1] - o.y) * inv.y;
  float lz = (I.lo[F][2] - o.z) * inv.z, hz = (I.hi[F][2] - o.z) * inv.z;
  float a = fmaxf(fmaxf(fminf(lx, hx), fminf(ly, hy)), fmaxf(fminf(lz, hz), tmin));
  float b = fminf(fminf(fmaxf(lx, hx), fmaxf(ly, hy)), fminf(fmaxf(lz, hz), tmax));
  return a <= b * 1.0000004f;
}

// ------------------------------------------------------------------------------------------------
// Queries in View_F = static BLAS + edited objects at M_F (ghosts transparent)
// ------------------------------------------------------------------------------------------------
struct Hit {
  float t;
  int leaf;   // leaf triangle index (-1: miss)
  int inst;   // -1 static, else instance index
};
struct Cross {  // ghost crossings of one segment: count, sum 1/|cos_G|, sum t^2/|cos_G|, sum (L-t)^2/|cos_G|
  float n, s0, sa, sb;
};
__device__ __forceinline__ Cross cross_zero() { Cross c; c.n = c.s0 = c.sa = c.sb = 0.0f; return c; }

struct QCount {  // per-thread query counters
  uint32_t closest, shadow, inst;
  TCount tc;
};

}  // namespace rr
