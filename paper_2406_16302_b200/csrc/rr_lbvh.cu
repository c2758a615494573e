// rr_lbvh.cu -- GPU LBVH build (Karras 2012 "Maximizing parallelism in the construction of BVHs,
// octrees, and k-d trees"): 63-bit Morton codes of triangle centroids, CUB radix sort, binary radix tree
// from longest common prefixes (duplicate keys broken by index), bottom-up AABB refit with atomic
// arrival counters, and packing into 64-byte BVH2 nodes.  The build is SAH-free (north star); RR_ROTATE passes of
// local tree rotations (k_rotate) then shrink child boxes without deepening the tree.
// Replaces the paper's Embree BVH.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rr_device.cuh"
#include "rr_internal.h"

namespace rr {

#ifndef RR_CUBIC_KEYS
#define RR_CUBIC_KEYS 1  // Morton codes over the centroid bounds' enclosing cube (cubic cells)
#endif
#ifndef RR_MORTON_BITS
#define RR_MORTON_BITS 63  // 21 bits per axis (30: 10 bits per axis)
#endif
#if RR_MORTON_BITS == 63
typedef unsigned long long MortonKey;
#define RR_MORTON_CELLS 2097152
#else
typedef uint32_t MortonKey;
#define RR_MORTON_CELLS 1024
#endif

struct Box {
  float lo[3], hi[3];
};
// boxes written by other threads of the same launch: read through L2 (L1 is not coherent)
__device__ __forceinline__ Box load_box_cg(const Box* b) {
  const float* f = (const float*)b;
  Box r;
  for (int q = 0; q < 3; ++q) {
    r.lo[q] = __ldcg(f + q);
    r.hi[q] = __ldcg(f + 3 + q);
  }
  return r;
}

__global__ void k_centroid_bounds(const float4* __restrict__ tris, int n, float* __restrict__ partial) {
  __shared__ float s[6][256];
  float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    float4 a = tris[3 * k], b = tris[3 * k + 1], c = tris[3 * k + 2];
    float cx = (a.x + b.x + c.x) * (1.0f / 3.0f), cy = (a.y + b.y + c.y) * (1.0f / 3.0f), cz = (a.z + b.z + c.z) * (1.0f / 3.0f);
    lo[0] = fminf(lo[0], cx); lo[1] = fminf(lo[1], cy); lo[2] = fminf(lo[2], cz);
    hi[0] = fmaxf(hi[0], cx); hi[1] = fmaxf(hi[1], cy); hi[2] = fmaxf(hi[2], cz);
  }
  for (int a = 0; a < 3; ++a) {
    s[a][threadIdx.x] = lo[a];
    s[3 + a][threadIdx.x] = hi[a];
  }
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      for (int a = 0; a < 3; ++a) {
        s[a][threadIdx.x] = fminf(s[a][threadIdx.x], s[a][threadIdx.x + st]);
        s[3 + a][threadIdx.x] = fmaxf(s[3 + a][threadIdx.x], s[3 + a][threadIdx.x + st]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int a = 0; a < 6; ++a) partial[6 * blockIdx.x + a] = s[a][0];
}

__device__ __forceinline__ uint32_t expand_bits(uint32_t v) {
  v = (v * 0x00010001u) & 0xFF0000FFu;
  v = (v * 0x00000101u) & 0x0F00F00Fu;
  v = (v * 0x00000011u) & 0xC30C30C3u;
  v = (v * 0x00000005u) & 0x49249249u;
  return v;
}

// 21 bits per axis -> 63-bit key
__device__ __forceinline__ uint64_t expand_bits21(uint64_t v) {
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

__global__ void k_morton(const float4* __restrict__ tris, int n, const float* __restrict__ partial, int nblocks,
                         MortonKey* __restrict__ keys, uint32_t* __restrict__ vals) {
  float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
  for (int b = 0; b < nblocks; ++b)
    for (int a = 0; a < 3; ++a) {
      lo[a] = fminf(lo[a], partial[6 * b + a]);
      hi[a] = fmaxf(hi[a], partial[6 * b + 3 + a]);
    }
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  float4 A = tris[3 * k], B = tris[3 * k + 1], C = tris[3 * k + 2];
  float c[3] = {(A.x + B.x + C.x) * (1.0f / 3.0f), (A.y + B.y + C.y) * (1.0f / 3.0f), (A.z + B.z + C.z) * (1.0f / 3.0f)};
  uint32_t q[3];
  const float cube = fmaxf(fmaxf(hi[0] - lo[0], hi[1] - lo[1]), hi[2] - lo[2]);
  for (int a = 0; a < 3; ++a) {
    float ext = RR_CUBIC_KEYS ? cube : hi[a] - lo[a];
    float u = ext > 0.0f ? (c[a] - lo[a]) / ext : 0.5f;
    q[a] = (uint32_t)fminf(fmaxf(u * (float)RR_MORTON_CELLS, 0.0f), (float)(RR_MORTON_CELLS - 1));
  }
#if RR_MORTON_BITS == 63
  keys[k] = (expand_bits21(q[0]) << 2) | (expand_bits21(q[1]) << 1) | expand_bits21(q[2]);
#else
  keys[k] = (expand_bits(q[0]) << 2) | (expand_bits(q[1]) << 1) | expand_bits(q[2]);
#endif
  vals[k] = (uint32_t)k;
}

__device__ __forceinline__ int delta(const MortonKey* keys, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  MortonKey a = keys[i], b = keys[j];
  if (a == b) return 8 * (int)sizeof(MortonKey) + __clz((uint32_t)i ^ (uint32_t)j);
#if RR_MORTON_BITS == 63
  return __clzll((long long)(a ^ b));
#else
  return __clz(a ^ b);
#endif
}

// internal node i of the radix tree: children (encoded: >= 0 internal, < 0 leaf ~k) and parents
__global__ void k_karras(const MortonKey* __restrict__ keys, int n, int* __restrict__ child, int* __restrict__ parent_int,
                         int* __restrict__ parent_leaf) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  int d = (delta(keys, n, i, i + 1) - delta(keys, n, i, i - 1)) >= 0 ? 1 : -1;
  int dmin = delta(keys, n, i, i - d);
  int lmax = 2;
  while (delta(keys, n, i, i + lmax * d) > dmin) lmax *= 2;
  int l = 0;
  for (int t = lmax / 2; t >= 1; t /= 2)
    if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
  int j = i + l * d;
  int dnode = delta(keys, n, i, j);
  int s = 0;
  for (int div = 2;; div *= 2) {
    int t = (l + div - 1) / div;
    if (delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
    if (t <= 1) break;
  }
  int gamma = i + s * d + min(d, 0);
  int lo = min(i, j), hi = max(i, j);
  int left = (lo == gamma) ? ~gamma : gamma;
  int right = (hi == gamma + 1) ? ~(gamma + 1) : gamma + 1;
  child[2 * i] = left;
  child[2 * i + 1] = right;
  if (left < 0) parent_leaf[~left] = i; else parent_int[left] = i;
  if (right < 0) parent_leaf[~right] = i; else parent_int[right] = i;
}

__global__ void k_refit(const float4* __restrict__ tris, const uint32_t* __restrict__ order, int n,
                        const int* __restrict__ child, const int* __restrict__ parent_int,
                        const int* __restrict__ parent_leaf, Box* __restrict__ ibox, Box* __restrict__ lbox,
                        int* __restrict__ counter) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  uint32_t t = order[k];
  float4 a = tris[3 * t], b = tris[3 * t + 1], c = tris[3 * t + 2];
  Box bx;
  bx.lo[0] = fminf(a.x, fminf(b.x, c.x)); bx.hi[0] = fmaxf(a.x, fmaxf(b.x, c.x));
  bx.lo[1] = fminf(a.y, fminf(b.y, c.y)); bx.hi[1] = fmaxf(a.y, fmaxf(b.y, c.y));
  bx.lo[2] = fminf(a.z, fminf(b.z, c.z)); bx.hi[2] = fmaxf(a.z, fmaxf(b.z, c.z));
  lbox[k] = bx;
  if (n == 1) return;
  __threadfence();
  int p = parent_leaf[k];
  while (p >= 0) {
    if (atomicAdd(&counter[p], 1) == 0) return;  // first arrival stops; the second one merges
    __threadfence();
    int c0 = child[2 * p], c1 = child[2 * p + 1];
    Box b0 = c0 < 0 ? load_box_cg(lbox + ~c0) : load_box_cg(ibox + c0);
    Box b1 = c1 < 0 ? load_box_cg(lbox + ~c1) : load_box_cg(ibox + c1);
    Box m;
    for (int q = 0; q < 3; ++q) {
      m.lo[q] = fminf(b0.lo[q], b1.lo[q]);
      m.hi[q] = fmaxf(b0.hi[q], b1.hi[q]);
    }
    ibox[p] = m;
    __threadfence();
    p = p == 0 ? -1 : parent_int[p];
  }
}

// world -> unit-triangle affine map of a triangle (Woop 2004): rows r_k with translation, computed in fp64;
// a point x on the triangle's plane has barycentrics (r0 . x + w0, r1 . x + w1), and r2 . x + w2 is its
// signed distance to the plane in units of |e1 x e2|^-1.  Degenerate triangles get NaN rows (never hit).
__device__ void unit_triangle(float4 a, float4 b, float4 c, float4* out) {
  double ax = a.x, ay = a.y, az = a.z;
  double e1x = b.x - ax, e1y = b.y - ay, e1z = b.z - az, e2x = c.x - ax, e2y = c.y - ay, e2z = c.z - az;
  double nx = e1y * e2z - e1z * e2y, ny = e1z * e2x - e1x * e2z, nz = e1x * e2y - e1y * e2x;
  double det = nx * nx + ny * ny + nz * nz;
  if (!(det > 0.0)) {
    for (int r = 0; r < 3; ++r) out[r] = make_float4(0.0f, 0.0f, 0.0f, __int_as_float(0x7fc00000));
    return;
  }
  double inv = 1.0 / det;
  double r0x = (e2y * nz - e2z * ny) * inv, r0y = (e2z * nx - e2x * nz) * inv, r0z = (e2x * ny - e2y * nx) * inv;
  double r1x = (ny * e1z - nz * e1y) * inv, r1y = (nz * e1x - nx * e1z) * inv, r1z = (nx * e1y - ny * e1x) * inv;
  double r2x = nx * inv, r2y = ny * inv, r2z = nz * inv;
  out[0] = make_float4((float)r0x, (float)r0y, (float)r0z, (float)(-(r0x * ax + r0y * ay + r0z * az)));
  out[1] = make_float4((float)r1x, (float)r1y, (float)r1z, (float)(-(r1x * ax + r1y * ay + r1z * az)));
  out[2] = make_float4((float)r2x, (float)r2y, (float)r2z, (float)(-(r2x * ax + r2y * ay + r2z * az)));
}

__global__ void k_pack(const float4* __restrict__ tris, const uint32_t* __restrict__ order, int n,
                       const int* __restrict__ child, const Box* __restrict__ ibox, const Box* __restrict__ lbox,
                       float4* __restrict__ nodes, float4* __restrict__ ltris, float4* __restrict__ lxf, int node_base,
                       int leaf_base) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) {
    uint32_t t = order[k];
    ltris[3 * (leaf_base + k)] = tris[3 * t];
    ltris[3 * (leaf_base + k) + 1] = tris[3 * t + 1];
    ltris[3 * (leaf_base + k) + 2] = tris[3 * t + 2];
    unit_triangle(tris[3 * t], tris[3 * t + 1], tris[3 * t + 2], lxf + 3 * (leaf_base + k));
  }
  int ninternal = n > 1 ? n - 1 : 1;
  if (k >= ninternal) return;
  int c0, c1;
  Box b0, b1;
  if (n == 1) {
    c0 = -1;  // ~0 -> leaf 0
    b0 = lbox[0];
    c1 = -1;
    for (int q = 0; q < 3; ++q) { b1.lo[q] = 3e38f; b1.hi[q] = 3e38f; }  // a point beyond every tmax (<= 1e30): never entered
  } else {
    c0 = child[2 * k];
    c1 = child[2 * k + 1];
    b0 = c0 < 0 ? lbox[~c0] : ibox[c0];
    b1 = c1 < 0 ? lbox[~c1] : ibox[c1];
  }
  int e0 = c0 < 0 ? ~(leaf_base + ~c0) : node_base + c0;
  int e1 = c1 < 0 ? ~(leaf_base + ~c1) : node_base + c1;
  float4* nd = nodes + 4 * (node_base + k);
  nd[0] = make_float4(b0.lo[0], b0.hi[0], b0.lo[1], b0.hi[1]);
  nd[1] = make_float4(b1.lo[0], b1.hi[0], b1.lo[1], b1.hi[1]);
  nd[2] = make_float4(b0.lo[2], b0.hi[2], b1.lo[2], b1.hi[2]);
  nd[3] = make_float4(__int_as_float(e0), __int_as_float(e1), 0.0f, 0.0f);
}

#ifndef RR_ROTATE
#define RR_ROTATE 4  // bottom-up tree-rotation passes over the packed nodes after the LBVH build (k_rotate; 0: the plain radix tree)
#endif
#ifndef RR_ROTATE_SLACK
#define RR_ROTATE_SLACK 0  // levels by which a rotation may raise its subtree's height (0: never deeper than the radix tree)
#endif
// ------------------------------------------------------------------------------------------------
// Tree rotations (Kensler 2008 "Tree rotations for improving bounding volume hierarchies"), bottom-up over the
// packed BVH2 nodes with the refit's arrival counters: the second thread to reach a node N = (A, B) finds both
// subtrees final, and may swap a child with a grandchild on the other side (B <-> A0 / A1, A <-> B0 / B1) or two
// grandchildren (A0 <-> B0 / B1) when that shrinks the surface area of the re-formed child box(es).  Only N and
// its children are rewritten; N's own box (held by its parent) is the union of the same leaves and does not
// change.  A rotation is taken only if the height of N's subtree does not grow, so the tree never gets deeper
// than the LBVH it started from (the traversal-stack bound checked at upload still holds).  Not an SAH build:
// the topology stays the radix tree's up to these local swaps.
struct PNode {
  Box b[2];
  int e[2];
};
__device__ __forceinline__ PNode load_pnode_cg(const float4* nodes, int idx) {
  const float4 a = __ldcg(nodes + 4 * idx), b = __ldcg(nodes + 4 * idx + 1), c = __ldcg(nodes + 4 * idx + 2),
               d = __ldcg(nodes + 4 * idx + 3);
  PNode n;
  n.b[0].lo[0] = a.x; n.b[0].hi[0] = a.y; n.b[0].lo[1] = a.z; n.b[0].hi[1] = a.w; n.b[0].lo[2] = c.x; n.b[0].hi[2] = c.y;
  n.b[1].lo[0] = b.x; n.b[1].hi[0] = b.y; n.b[1].lo[1] = b.z; n.b[1].hi[1] = b.w; n.b[1].lo[2] = c.z; n.b[1].hi[2] = c.w;
  n.e[0] = __float_as_int(d.x);
  n.e[1] = __float_as_int(d.y);
  return n;
}
__device__ __forceinline__ void store_pnode(float4* nodes, int idx, const PNode& n) {
  float4* nd = nodes + 4 * idx;
  nd[0] = make_float4(n.b[0].lo[0], n.b[0].hi[0], n.b[0].lo[1], n.b[0].hi[1]);
  nd[1] = make_float4(n.b[1].lo[0], n.b[1].hi[0], n.b[1].lo[1], n.b[1].hi[1]);
  nd[2] = make_float4(n.b[0].lo[2], n.b[0].hi[2], n.b[1].lo[2], n.b[1].hi[2]);
  nd[3] = make_float4(__int_as_float(n.e[0]), __int_as_float(n.e[1]), 0.0f, 0.0f);
}
__device__ __forceinline__ Box box_union(const Box& a, const Box& b) {
  Box m;
  for (int q = 0; q < 3; ++q) {
    m.lo[q] = fminf(a.lo[q], b.lo[q]);
    m.hi[q] = fmaxf(a.hi[q], b.hi[q]);
  }
  return m;
}
__device__ __forceinline__ float half_area(const Box& b) {
  const float dx = b.hi[0] - b.lo[0], dy = b.hi[1] - b.lo[1], dz = b.hi[2] - b.lo[2];
  return dx * dy + dy * dz + dz * dx;
}
__global__ void k_rotate(float4* __restrict__ nodes, int n, int node_base, int leaf_base, int* __restrict__ parent_int,
                         int* __restrict__ parent_leaf, int* __restrict__ counter, int* __restrict__ hgt,
                         unsigned int* __restrict__ n_rot, int slack) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int p = parent_leaf[k];
  while (p >= 0) {
    __threadfence();
    if (atomicAdd(&counter[p], 1) == 0) return;  // first arrival stops; the second one owns the node
    __threadfence();
    PNode N = load_pnode_cg(nodes, node_base + p);
    PNode C[2];
    int h[2], hc[2][2];
    bool inner[2];
    for (int s = 0; s < 2; ++s) {
      inner[s] = N.e[s] >= 0;
      h[s] = 0;
      hc[s][0] = hc[s][1] = 0;
      if (inner[s]) {
        C[s] = load_pnode_cg(nodes, N.e[s]);
        for (int g = 0; g < 2; ++g) hc[s][g] = C[s].e[g] < 0 ? 0 : __ldcg(hgt + (C[s].e[g] - node_base));
        h[s] = 1 + max(hc[s][0], hc[s][1]);
      }
    }
    const int h_old = 1 + max(h[0], h[1]);
    const int h_lim = h_old + slack;  // slack 0: the subtree's height never grows
    // candidates: kind 0: child (1 - s) <-> grandchild g of inner child s;  kind 1: grandchild (0, 0) <-> (1, g)
    float best = 0.0f;
    int bk = -1, bs = 0, bg = 0;
    for (int s = 0; s < 2; ++s) {
      if (!inner[s]) continue;
      const float base = half_area(N.b[s]);
      for (int g = 0; g < 2; ++g) {
        // child s re-formed from (other child, grandchild 1 - g); grandchild g moves up
        const float d = half_area(box_union(N.b[1 - s], C[s].b[1 - g])) - base;
        const int hs = 1 + max(h[1 - s], hc[s][1 - g]);
        const int hn = 1 + max(hs, hc[s][g]);
        if (d < best - 1e-4f * base && hn <= h_lim) {
          best = d;
          bk = 0; bs = s; bg = g;
        }
      }
    }
    if (inner[0] && inner[1]) {
      const float base = half_area(N.b[0]) + half_area(N.b[1]);
      for (int g = 0; g < 2; ++g) {
        // A' = (B_g, A_1), B' = (A_0, B_{1-g})
        const float d = half_area(box_union(C[1].b[g], C[0].b[1])) + half_area(box_union(C[0].b[0], C[1].b[1 - g])) - base;
        const int ha = 1 + max(hc[1][g], hc[0][1]), hb = 1 + max(hc[0][0], hc[1][1 - g]);
        if (d < best - 1e-4f * base && 1 + max(ha, hb) <= h_lim) {
          best = d;
          bk = 1; bs = 0; bg = g;
        }
      }
    }
    int h_new = h_old;
    if (bk == 0) {
      const int s = bs, g = bg, up = C[s].e[g], down = N.e[1 - s];
      const int cs = N.e[s] - node_base;  // local index of the re-formed child
      const Box upb = C[s].b[g];
      C[s].b[g] = N.b[1 - s];
      C[s].e[g] = down;
      N.b[1 - s] = upb;
      N.e[1 - s] = up;
      N.b[s] = box_union(C[s].b[0], C[s].b[1]);
      const int hs = 1 + max(h[1 - s], hc[s][1 - g]);
      store_pnode(nodes, N.e[s], C[s]);
      store_pnode(nodes, node_base + p, N);
      hgt[cs] = hs;
      h_new = 1 + max(hs, hc[s][g]);
      if (down < 0) parent_leaf[~down - leaf_base] = cs; else parent_int[down - node_base] = cs;
      if (up < 0) parent_leaf[~up - leaf_base] = p; else parent_int[up - node_base] = p;
      atomicAdd(n_rot, 1u);
    } else if (bk == 1) {
      const int g = bg, x = C[0].e[0], y = C[1].e[g];
      const int ca = N.e[0] - node_base, cb = N.e[1] - node_base;
      const Box bx = C[0].b[0], by = C[1].b[g];
      C[0].b[0] = by; C[0].e[0] = y;
      C[1].b[g] = bx; C[1].e[g] = x;
      N.b[0] = box_union(C[0].b[0], C[0].b[1]);
      N.b[1] = box_union(C[1].b[0], C[1].b[1]);
      store_pnode(nodes, N.e[0], C[0]);
      store_pnode(nodes, N.e[1], C[1]);
      store_pnode(nodes, node_base + p, N);
      const int ha = 1 + max(hc[1][g], hc[0][1]), hb = 1 + max(hc[0][0], hc[1][1 - g]);
      hgt[ca] = ha;
      hgt[cb] = hb;
      h_new = 1 + max(ha, hb);
      if (y < 0) parent_leaf[~y - leaf_base] = ca; else parent_int[y - node_base] = ca;
      if (x < 0) parent_leaf[~x - leaf_base] = cb; else parent_int[x - node_base] = cb;
      atomicAdd(n_rot, 1u);
    }
    hgt[p] = h_new;
    p = p == 0 ? -1 : parent_int[p];
  }
}

// Build one BLAS over n >= 1 triangles (3 float4 each, device).  Writes max(n-1,1) nodes at node_base and n
// leaf triangles at leaf_base.  Returns the root node index (node_base).  h_keys (optional, host, n): sort
// keys to use instead of the triangles' own Morton codes (object-grouped keys, rr_capi.cu).
int build_lbvh(const float4* d_tris, int n, float4* d_nodes, float4* d_ltris, float4* d_lxf, int node_base,
               int leaf_base, cudaStream_t st, const unsigned long long* h_keys) {
  const int TB = 256;
  int nb = (n + TB - 1) / TB;
  int nred = nb < 1024 ? nb : 1024;
  DevBuf<float> partial(6 * nred);
  DevBuf<MortonKey> keys(n), keys2(n);
  DevBuf<uint32_t> vals(n), vals2(n);
  DevBuf<int> child(2 * (n > 1 ? n - 1 : 1)), pint(n > 1 ? n - 1 : 1), pleaf(n), counter(n > 1 ? n - 1 : 1);
  DevBuf<Box> ibox(n > 1 ? n - 1 : 1), lbox(n);
  if (h_keys && sizeof(MortonKey) == sizeof(unsigned long long)) {
    std::vector<uint32_t> iota(n);
    for (int k = 0; k < n; ++k) iota[k] = (uint32_t)k;
    cudaMemcpyAsync(keys.p, h_keys, n * sizeof(MortonKey), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(vals.p, iota.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
  } else {
    k_centroid_bounds<<<nred, TB, 0, st>>>(d_tris, n, partial.p);
    k_morton<<<nb, TB, 0, st>>>(d_tris, n, partial.p, nred, keys.p, vals.p);
  }
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys2.p, vals.p, vals2.p, n, 0, RR_MORTON_BITS, st);
  DevBuf<char> tmp(tmp_bytes);
  cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, keys2.p, vals.p, vals2.p, n, 0, RR_MORTON_BITS, st);
  cudaMemsetAsync(counter.p, 0, sizeof(int) * (n > 1 ? n - 1 : 1), st);
  cudaMemsetAsync(pint.p, 0xff, sizeof(int) * (n > 1 ? n - 1 : 1), st);
  if (n > 1) k_karras<<<(n - 1 + TB - 1) / TB, TB, 0, st>>>(keys2.p, n, child.p, pint.p, pleaf.p);
  k_refit<<<nb, TB, 0, st>>>(d_tris, vals2.p, n, child.p, pint.p, pleaf.p, ibox.p, lbox.p, counter.p);
  k_pack<<<nb, TB, 0, st>>>(d_tris, vals2.p, n, child.p, ibox.p, lbox.p, d_nodes, d_ltris, d_lxf, node_base, leaf_base);
  if (RR_ROTATE > 0 && n >= 3) {
    DevBuf<int> hgt(n - 1);
    DevBuf<unsigned int> nrot(1);
    auto rotate = [&](int slack) {
      for (int pass = 0; pass < RR_ROTATE; ++pass) {
        cudaMemsetAsync(counter.p, 0, sizeof(int) * (n - 1), st);
        cudaMemsetAsync(nrot.p, 0, sizeof(unsigned int), st);
        k_rotate<<<nb, TB, 0, st>>>(d_nodes, n, node_base, leaf_base, pint.p, pleaf.p, counter.p, hgt.p, nrot.p, slack);
        if (getenv("RR_ROTATE_LOG")) {  // diagnostics: rotations taken per pass
          unsigned int r = 0;
          cudaMemcpyAsync(&r, nrot.p, sizeof(r), cudaMemcpyDeviceToHost, st);
          cudaStreamSynchronize(st);
          fprintf(stderr, "lbvh n=%d rotate pass %d (slack %d): %u rotations\n", n, pass, slack, r);
        }
      }
      int h0 = 0;  // height of the rotated tree (hgt of the root)
      cudaMemcpyAsync(&h0, hgt.p, sizeof(int), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      return h0;
    };
    int h0 = rotate(RR_ROTATE_SLACK);
    // rotations with slack may deepen the tree: if it no longer fits the traversal stack with room for an extra
    // root above it, restore the radix tree (child / box arrays are untouched) and rotate without slack, which
    // never deepens it
    if (RR_ROTATE_SLACK > 0 && h0 > RR_STACK - 2) {
      cudaMemsetAsync(pint.p, 0xff, sizeof(int) * (n - 1), st);
      k_karras<<<(n - 1 + TB - 1) / TB, TB, 0, st>>>(keys2.p, n, child.p, pint.p, pleaf.p);
      k_pack<<<nb, TB, 0, st>>>(d_tris, vals2.p, n, child.p, ibox.p, lbox.p, d_nodes, d_ltris, d_lxf, node_base, leaf_base);
      h0 = rotate(0);
    }
    if (getenv("RR_ROTATE_LOG")) fprintf(stderr, "lbvh n=%d height after rotations %d\n", n, h0);
  }
  cudaStreamSynchronize(st);
  return node_base;
}

}  // namespace rr
