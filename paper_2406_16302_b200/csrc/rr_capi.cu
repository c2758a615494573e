// rr_capi.cu -- C ABI (include/rr.h): scene upload + LBVH build, set_edit, render_residual, stats,
// test-only exports.  Host-side derivations are done in fp64 and rounded once to fp32:
// triangle-selection CDFs (prefix sums in triangle order / total), emitter and area pdfs, camera basis,
// rigid-transform inverses.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <unordered_map>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges of the host API calls in Nsight timelines

#include "../../include/rr.h"
#include "rr_device.cuh"
#include "rr_internal.h"
#include "rr_kernels.h"
#ifndef RR_SAMPLE_SORT
#define RR_SAMPLE_SORT 1  // T3 / T6 samples processed in start-ray order (sample_order); 0: index order
#endif
#ifndef RR_REFILL
#define RR_REFILL 32  // lanes of a warp refilled together (1: immediate per-lane refill)
#endif
#ifndef RR_SORT_MASK
#define RR_SORT_MASK 0x7Fu  // techniques sorted (bit l-1): all (T7 by 2D Morton order of its pixel)
#endif

using namespace rr;

namespace {
struct NvtxRange {  // RAII range around one ABI call
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

struct rr_ctx {
  int device = 0;
  std::string err;
  bool have_scene = false;
  // host copies of the scene
  std::vector<float> pos;
  std::vector<uint32_t> idx, tri_obj;
  std::vector<rr_object> objects;
  std::vector<rr_material> materials;
  rr_camera cam;
  double diag = 1.0;
  std::vector<int> dyn_objects;  // dynamic object ids in order (instance k -> object)
  std::vector<int> obj_inst;
  std::vector<int> inst_root;
  int bvh_depth = 0;               // deepest root-to-leaf path over all BLAS roots, in inner nodes
  std::vector<float> inst_bbox;   // 6 per instance, object space
  // device buffers
  DevBuf<float4> nodes, ltris, lxf, tverts, mat, obj_emit;
  DevBuf<uint32_t> d_tri_obj, obj_flags, mat_type, mat_type_vndf, obj_mat0, obj_mat1, emit_tris, edited_tris, moved_tris;
  DevBuf<int> d_obj_inst, obj_emitter, emit_off, emit_cnt;
  DevBuf<float> emit_pL, emit_cdf, edited_cdf, moved_cdf;
  DevBuf<float4> emit_centroid;      // RR_T6_TOWARD_LIGHT: area-weighted centroid of each emitter (world, set_edit)
  std::vector<std::vector<uint32_t>> emit_tris_host;
  DevBuf<unsigned long long> stats, work;
  // T3 / T6 processing order (sample_order): sort keys / slots, sorted keys, permutation, CUB scratch (grow-only)
  DevBuf<uint32_t> ord_keys, ord_vals, ord_keys2, ord_perm;
  DevBuf<unsigned char> ord_tmp;
  DevScene S;
  uint32_t last_mask = 0;
  int edited_equals_moved = 0;
  std::vector<uint32_t> flags_host;
  // timings
  cudaEvent_t ev[32];  // render start, then (start, end) of each residual launch
  int n_sorted = 0;     // residual launches of the last render that had the sample-ordering pre-pass
  int n_ev = 0;
  bool ev_init = false;
};

#ifndef RR_GROUPED_KEYS
#define RR_GROUPED_KEYS 1  // static BLAS sorted by object-grouped keys (object Morton, then triangle Morton)
#endif
#ifndef RR_CUBIC_KEYS
#define RR_CUBIC_KEYS 1  // Morton keys over cubic cells (largest extent on every axis)
#endif
#ifndef RR_LARGE_FRAC
#define RR_LARGE_FRAC 0.05  // "large" static triangle: box diagonal > this fraction of the static scene's
#endif

namespace {

rr_status fail(rr_ctx* c, rr_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}
rr_status cuda_check(rr_ctx* c, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, RR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return RR_OK;
}

// fp64 prefix sum of triangle areas in triangle order, divided by the total, rounded to fp32
double build_cdf(const rr_ctx* c, const std::vector<uint32_t>& tris, std::vector<float>& cdf) {
  double total = 0;
  std::vector<double> pre(tris.size());
  for (size_t k = 0; k < tris.size(); ++k) {
    uint32_t t = tris[k];
    const float* a = &c->pos[3 * c->idx[3 * t]];
    const float* b = &c->pos[3 * c->idx[3 * t + 1]];
    const float* d = &c->pos[3 * c->idx[3 * t + 2]];
    double e1[3] = {(double)b[0] - a[0], (double)b[1] - a[1], (double)b[2] - a[2]};
    double e2[3] = {(double)d[0] - a[0], (double)d[1] - a[1], (double)d[2] - a[2]};
    double cx = e1[1] * e2[2] - e1[2] * e2[1], cy = e1[2] * e2[0] - e1[0] * e2[2], cz = e1[0] * e2[1] - e1[1] * e2[0];
    total += 0.5 * std::sqrt(cx * cx + cy * cy + cz * cz);
    pre[k] = total;
  }
  cdf.resize(tris.size());
  for (size_t k = 0; k < tris.size(); ++k) cdf[k] = (float)(pre[k] / total);
  if (!cdf.empty()) cdf.back() = 1.0f;
  return total;
}

float int_bits(int k) {
  float f;
  std::memcpy(&f, &k, sizeof(f));
  return f;
}

void set_identity(float* m) {
  std::memset(m, 0, 12 * sizeof(float));
  m[0] = m[5] = m[10] = 1.0f;
}

}  // namespace

extern "C" {

rr_status rr_create(int cuda_device, rr_ctx** out) {
  if (!out) return RR_E_INVALID;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || cuda_device < 0 || cuda_device >= n) {
    cudaGetLastError();
    return RR_E_CUDA;
  }
  if (cudaSetDevice(cuda_device) != cudaSuccess) return RR_E_CUDA;
  rr_ctx* c = new rr_ctx();
  c->device = cuda_device;
  std::memset(&c->S, 0, sizeof(c->S));
  try {
    c->stats.alloc(STAT_COUNT);
    c->work.alloc(16);
  } catch (...) {
    delete c;
    return RR_E_OOM;
  }
  *out = c;
  return RR_OK;
}

void rr_destroy(rr_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->ev_init)
    for (int k = 0; k < 32; ++k) cudaEventDestroy(c->ev[k]);
  delete c;
}

const char* rr_last_error(const rr_ctx* c) { return c ? c->err.c_str() : "null context"; }

rr_status rr_scene_upload(rr_ctx* c, const rr_scene_desc* d) {
  NvtxRange nvtx_("rr_scene_upload");
  if (!c || !d) return fail(c, RR_E_INVALID, "null argument");
  if (!d->positions || !d->indices || !d->tri_object || !d->objects || !d->materials)
    return fail(c, RR_E_INVALID, "null array in scene description");
  if (d->n_triangles == 0 || d->n_objects == 0 || d->n_materials == 0)
    return fail(c, RR_E_INVALID, "empty scene");
  if (d->camera.width == 0 || d->camera.height == 0) return fail(c, RR_E_INVALID, "empty image");
  cudaSetDevice(c->device);
  const uint32_t T = d->n_triangles, O = d->n_objects, M = d->n_materials;
  for (uint64_t k = 0; k < 3ull * T; ++k)
    if (d->indices[k] >= d->n_vertices) return fail(c, RR_E_INVALID, "triangle index out of range");
  for (uint32_t k = 0; k < T; ++k)
    if (d->tri_object[k] >= O) return fail(c, RR_E_INVALID, "tri_object out of range");
  int n_emit_obj = 0, n_dyn = 0;
  for (uint32_t o = 0; o < O; ++o) {
    const rr_object& ob = d->objects[o];
    if (ob.material >= M) return fail(c, RR_E_INVALID, "object material out of range");
    for (int q = 0; q < 3; ++q)
      if (!(ob.emission[q] >= 0.0f)) return fail(c, RR_E_INVALID, "negative emission");
    if (ob.emission[0] > 0 || ob.emission[1] > 0 || ob.emission[2] > 0) n_emit_obj++;
    if (ob.flags & RR_OBJ_DYNAMIC) n_dyn++;
  }
  if (n_emit_obj == 0) return fail(c, RR_E_INVALID, "scene has no emitter");
  {  // an emitter or dynamic object without triangles would give p_L = 1/0 or an empty BLAS: refuse it
    std::vector<uint32_t> cnt(O, 0);
    for (uint32_t k = 0; k < T; ++k) cnt[d->tri_object[k]]++;
    for (uint32_t o = 0; o < O; ++o) {
      const rr_object& ob = d->objects[o];
      bool emits = ob.emission[0] > 0 || ob.emission[1] > 0 || ob.emission[2] > 0;
      if (cnt[o] == 0 && (emits || (ob.flags & RR_OBJ_DYNAMIC)))
        return fail(c, RR_E_INVALID, "emitting or dynamic object " + std::to_string(o) + " has no triangles");
    }
  }
  if (n_dyn > RR_MAX_INST) return fail(c, RR_E_INVALID, "too many dynamic objects (max 8)");
  for (uint32_t m = 0; m < M; ++m) {
    const rr_material& mt = d->materials[m];
    if (mt.type > 1) return fail(c, RR_E_INVALID, "unknown material type");
    if (mt.type == RR_GGX && !(mt.roughness > 0.0f && mt.roughness <= 1.0f)) return fail(c, RR_E_INVALID, "GGX roughness out of (0,1]");
  }
  c->have_scene = false;
  c->pos.assign(d->positions, d->positions + 3ull * d->n_vertices);
  c->idx.assign(d->indices, d->indices + 3ull * T);
  c->tri_obj.assign(d->tri_object, d->tri_object + T);
  c->objects.assign(d->objects, d->objects + O);
  c->materials.assign(d->materials, d->materials + M);
  c->cam = d->camera;
  for (uint32_t k = 0; k < T; ++k) {
    const float* a = &c->pos[3 * c->idx[3 * k]];
    const float* b = &c->pos[3 * c->idx[3 * k + 1]];
    const float* e = &c->pos[3 * c->idx[3 * k + 2]];
    double e1[3] = {(double)b[0] - a[0], (double)b[1] - a[1], (double)b[2] - a[2]};
    double e2[3] = {(double)e[0] - a[0], (double)e[1] - a[1], (double)e[2] - a[2]};
    double cx = e1[1] * e2[2] - e1[2] * e2[1], cy = e1[2] * e2[0] - e1[0] * e2[2], cz = e1[0] * e2[1] - e1[1] * e2[0];
    if (!(cx * cx + cy * cy + cz * cz > 0.0)) return fail(c, RR_E_INVALID, "degenerate triangle (area 0)");
  }
  try {
    // ---- scene diagonal over static, non-environment geometry (C12 #13)
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    bool any = false;
    for (uint32_t k = 0; k < T; ++k) {
      const rr_object& ob = c->objects[c->tri_obj[k]];
      if ((ob.flags & RR_OBJ_DYNAMIC) || (ob.flags & RR_OBJ_ENV)) continue;
      any = true;
      for (int v = 0; v < 3; ++v)
        for (int q = 0; q < 3; ++q) {
          double x = c->pos[3 * c->idx[3 * k + v] + q];
          lo[q] = std::min(lo[q], x);
          hi[q] = std::max(hi[q], x);
        }
    }
    if (!any)
      for (uint32_t k = 0; k < 3 * T; ++k)
        for (int q = 0; q < 3; ++q) {
          double x = c->pos[3 * c->idx[k] + q];
          lo[q] = std::min(lo[q], x);
          hi[q] = std::max(hi[q], x);
        }
    c->diag = std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) + (hi[2] - lo[2]) * (hi[2] - lo[2]));
    // ---- per-triangle vertices (BLAS space) and object ids
    std::vector<float4> tv(3ull * T);
    for (uint32_t k = 0; k < T; ++k)
      for (int v = 0; v < 3; ++v) {
        const float* p = &c->pos[3 * c->idx[3 * k + v]];
        tv[3ull * k + v] = make_float4(p[0], p[1], p[2], v == 0 ? int_bits((int)k) : 0.0f);
      }
    c->tverts.upload(tv.data(), tv.size());
    c->d_tri_obj.upload(c->tri_obj.data(), T);
    // ---- objects
    c->dyn_objects.clear();
    c->obj_inst.assign(O, -1);
    std::vector<int> emitter(O, -1);
    std::vector<uint32_t> flags(O, 0);
    std::vector<float4> emit(O);
    int ne = 0;
    for (uint32_t o = 0; o < O; ++o) {
      const rr_object& ob = c->objects[o];
      if (ob.flags & RR_OBJ_DYNAMIC) {
        c->obj_inst[o] = (int)c->dyn_objects.size();
        c->dyn_objects.push_back((int)o);
        flags[o] |= OBJ_EDITED;
      }
      emit[o] = make_float4(ob.emission[0], ob.emission[1], ob.emission[2], 0.0f);
      if (ob.emission[0] > 0 || ob.emission[1] > 0 || ob.emission[2] > 0) {
        emitter[o] = ne++;
        flags[o] |= OBJ_EMITTER;
      }
    }
    c->flags_host = flags;
    c->obj_emit.upload(emit.data(), O);
    c->obj_emitter.upload(emitter.data(), O);
    c->d_obj_inst.upload(c->obj_inst.data(), O);
    // ---- emitters: per emitter object its triangles (in triangle order), CDF, p_L = 1/(n_emit A_o)
    std::vector<std::vector<uint32_t>> etris(ne);
    std::vector<std::vector<uint32_t>> dtris(c->dyn_objects.size());
    std::vector<uint32_t> stris, edited;
    for (uint32_t k = 0; k < T; ++k) {
      int o = (int)c->tri_obj[k];
      if (emitter[o] >= 0) etris[emitter[o]].push_back(k);
      if (c->obj_inst[o] >= 0) {
        dtris[c->obj_inst[o]].push_back(k);
        edited.push_back(k);
      } else {
        stris.push_back(k);
      }
    }
    std::vector<int> eoff(ne), ecnt(ne);
    std::vector<float> epl(ne), ecdf;
    std::vector<uint32_t> eall;
    for (int e = 0; e < ne; ++e) {
      std::vector<float> cd;
      double area = build_cdf(c, etris[e], cd);
      eoff[e] = (int)eall.size();
      ecnt[e] = (int)etris[e].size();
      epl[e] = (float)(1.0 / ((double)ne * area));
      eall.insert(eall.end(), etris[e].begin(), etris[e].end());
      ecdf.insert(ecdf.end(), cd.begin(), cd.end());
    }
    c->emit_tris_host = etris;
    c->emit_off.upload(eoff.data(), ne);
    c->emit_cnt.upload(ecnt.data(), ne);
    c->emit_pL.upload(epl.data(), ne);
    c->emit_tris.upload(eall.data(), eall.size());
    c->emit_cdf.upload(ecdf.data(), ecdf.size());
    // ---- edited set (all dynamic objects)
    float pA_D = 0.0f;
    if (!edited.empty()) {
      std::vector<float> cd;
      double area = build_cdf(c, edited, cd);
      pA_D = (float)(1.0 / area);
      c->edited_tris.upload(edited.data(), edited.size());
      c->edited_cdf.upload(cd.data(), cd.size());
    }
    // ---- BLASes: static (world space) + one per dynamic object (object space)
    size_t total_nodes = stris.empty() ? 0 : std::max<size_t>(stris.size() - 1, 1) + 2;  // + split root, 2nd BLAS
    size_t total_leaves = stris.size();
    for (auto& v : dtris) {
      total_nodes += std::max<size_t>(v.size() > 0 ? v.size() - 1 : 0, 1);
      total_leaves += v.size();
    }
    c->nodes.alloc(4 * total_nodes);
    c->ltris.alloc(3 * total_leaves);
    c->lxf.alloc(3 * total_leaves);
    cudaStream_t st = 0;
    int node_base = 0, leaf_base = 0;
    // Object-grouped sort keys for a static BLAS: (30-bit Morton code of the object's centroid, 4-bit tie
    // break among objects in the same cell, 27-bit Morton code of the triangle within its object's box), so
    // the Karras tree splits between objects first and every object's triangles form their own subtrees
    // (SAH-free).
    auto grouped_keys = [&](const std::vector<uint32_t>& tl, std::vector<unsigned long long>& keys) {
      std::unordered_map<uint32_t, int> slot;
      std::vector<std::array<float, 6>> ob;  // per object: box lo, hi
      std::vector<int> tob(tl.size());
      for (size_t k = 0; k < tl.size(); ++k) {
        uint32_t o = c->tri_obj[tl[k]];
        auto it = slot.find(o);
        int j;
        if (it == slot.end()) {
          j = (int)ob.size();
          slot[o] = j;
          ob.push_back({3e38f, 3e38f, 3e38f, -3e38f, -3e38f, -3e38f});
        } else {
          j = it->second;
        }
        tob[k] = j;
        for (int v = 0; v < 3; ++v) {
          const float4& p = tv[3ull * tl[k] + v];
          const float q[3] = {p.x, p.y, p.z};
          for (int a = 0; a < 3; ++a) {
            ob[j][a] = std::min(ob[j][a], q[a]);
            ob[j][3 + a] = std::max(ob[j][3 + a], q[a]);
          }
        }
      }
      float clo[3] = {3e38f, 3e38f, 3e38f}, chi[3] = {-3e38f, -3e38f, -3e38f};
      for (auto& b : ob)
        for (int a = 0; a < 3; ++a) {
          float m = 0.5f * (b[a] + b[3 + a]);
          clo[a] = std::min(clo[a], m);
          chi[a] = std::max(chi[a], m);
        }
      auto spread = [](uint64_t v, int bits) {  // bit i -> bit 3i
        uint64_t r = 0;
        for (int i = 0; i < bits; ++i) r |= ((v >> i) & 1ull) << (3 * i);
        return r;
      };
      auto quant = [](float x, float lo, float hi, int bits) {
        float e = hi - lo;
        double u = e > 0 ? ((double)x - lo) / e : 0.5;
        double m = (double)((1u << bits) - 1);
        return (uint64_t)std::min(m, std::max(0.0, u * (1u << bits)));
      };
      float cext[3], cmax = 0.0f;  // cubic cells (RR_CUBIC_KEYS): split where the extent is largest
      for (int a = 0; a < 3; ++a) cmax = std::max(cmax, chi[a] - clo[a]);
      for (int a = 0; a < 3; ++a) cext[a] = RR_CUBIC_KEYS ? cmax : chi[a] - clo[a];
      std::vector<std::pair<uint64_t, int>> om(ob.size());
      for (size_t j = 0; j < ob.size(); ++j) {
        uint64_t code = 0;
        for (int a = 0; a < 3; ++a)
          code |= spread(quant(0.5f * (ob[j][a] + ob[j][3 + a]), clo[a], clo[a] + cext[a], 10), 10) << (2 - a);
        om[j] = {code, (int)j};
      }
      std::sort(om.begin(), om.end());
      std::vector<uint64_t> hi_key(ob.size());
      for (size_t r = 0; r < om.size(); ++r) {
        int tie = 0;
        if (r > 0 && om[r].first == om[r - 1].first) tie = std::min<int>(15, (int)(hi_key[om[r - 1].second] & 15) + 1);
        hi_key[om[r].second] = (om[r].first << 4) | (uint64_t)tie;
      }
      keys.resize(tl.size());
      for (size_t k = 0; k < tl.size(); ++k) {
        const auto& b = ob[tob[k]];
        const float4 &p0 = tv[3ull * tl[k]], &p1 = tv[3ull * tl[k] + 1], &p2 = tv[3ull * tl[k] + 2];
        const float cen[3] = {(p0.x + p1.x + p2.x) / 3.0f, (p0.y + p1.y + p2.y) / 3.0f, (p0.z + p1.z + p2.z) / 3.0f};
        uint64_t local = 0;
        float lext = 0.0f;
        for (int a = 0; a < 3; ++a) lext = RR_CUBIC_KEYS ? std::max(lext, b[3 + a] - b[a]) : 0.0f;
        for (int a = 0; a < 3; ++a)
          local |= spread(quant(cen[a], b[a], b[a] + (RR_CUBIC_KEYS ? lext : b[3 + a] - b[a]), 9), 9) << (2 - a);
        keys[k] = (hi_key[tob[k]] << 27) | local;
      }
    };
    auto build = [&](const std::vector<uint32_t>& tl, bool grouped = false) {
      std::vector<float4> tb(3 * tl.size());
      for (size_t k = 0; k < tl.size(); ++k)
        for (int v = 0; v < 3; ++v) tb[3 * k + v] = tv[3ull * tl[k] + v];
      DevBuf<float4> dt;
      dt.upload(tb.data(), tb.size());
      std::vector<unsigned long long> keys;
      if (grouped && RR_GROUPED_KEYS) grouped_keys(tl, keys);
      int root = build_lbvh(dt.p, (int)tl.size(), c->nodes.p, c->ltris.p, c->lxf.p, node_base, leaf_base, st,
                            keys.empty() ? nullptr : keys.data());
      node_base += (int)std::max<size_t>(tl.size() - 1, 1);
      leaf_base += (int)tl.size();
      return root;
    };
    // Static BLAS: triangles whose box diagonal exceeds RR_LARGE_FRAC of the static scene's get their own
    // LBVH under an extra root, so that a few huge triangles (a ground plane, light quads) do not inflate
    // the boxes of every Morton-ordered subtree they land in (SAH-free).
    int static_root = -1;
    if (!stris.empty()) {
      auto box_of = [&](const std::vector<uint32_t>& tl, float lo[3], float hi[3]) {
        for (int a = 0; a < 3; ++a) { lo[a] = 3e38f; hi[a] = -3e38f; }
        for (uint32_t t : tl)
          for (int v = 0; v < 3; ++v) {
            const float4& p = tv[3ull * t + v];
            lo[0] = std::min(lo[0], p.x); hi[0] = std::max(hi[0], p.x);
            lo[1] = std::min(lo[1], p.y); hi[1] = std::max(hi[1], p.y);
            lo[2] = std::min(lo[2], p.z); hi[2] = std::max(hi[2], p.z);
          }
      };
      float slo[3], shi[3];
      box_of(stris, slo, shi);
      double sd = std::sqrt((double)(shi[0] - slo[0]) * (shi[0] - slo[0]) + (double)(shi[1] - slo[1]) * (shi[1] - slo[1]) +
                            (double)(shi[2] - slo[2]) * (shi[2] - slo[2]));
      std::vector<uint32_t> small, large;
      for (uint32_t t : stris) {
        float lo[3], hi[3];
        box_of(std::vector<uint32_t>{t}, lo, hi);
        double d = std::sqrt((double)(hi[0] - lo[0]) * (hi[0] - lo[0]) + (double)(hi[1] - lo[1]) * (hi[1] - lo[1]) +
                             (double)(hi[2] - lo[2]) * (hi[2] - lo[2]));
        (d > RR_LARGE_FRAC * sd ? large : small).push_back(t);
      }
      if (large.empty() || small.empty()) {
        static_root = build(stris, true);
      } else {
        const int top = node_base++;  // the extra root, reserved in total_nodes
        int rs = build(small, true), rl = build(large);
        float a0[3], b0[3], a1[3], b1[3];
        box_of(small, a0, b0);
        box_of(large, a1, b1);
        float4 nd[4] = {make_float4(a0[0], b0[0], a0[1], b0[1]), make_float4(a1[0], b1[0], a1[1], b1[1]),
                        make_float4(a0[2], b0[2], a1[2], b1[2]), make_float4(0.f, 0.f, 0.f, 0.f)};
        std::memcpy(&nd[3].x, &rs, 4);
        std::memcpy(&nd[3].y, &rl, 4);
        cudaMemcpy(c->nodes.p + 4 * top, nd, sizeof(nd), cudaMemcpyHostToDevice);
        static_root = top;
      }
    }
    c->inst_root.clear();
    c->inst_bbox.clear();
    for (auto& v : dtris) {
      c->inst_root.push_back(build(v));
      float bl[3] = {3e38f, 3e38f, 3e38f}, bh[3] = {-3e38f, -3e38f, -3e38f};
      for (uint32_t t : v)
        for (int q = 0; q < 3; ++q)
          for (int a = 0; a < 3; ++a) {
            float x = c->pos[3 * c->idx[3 * t + q] + a];
            bl[a] = std::min(bl[a], x);
            bh[a] = std::max(bh[a], x);
          }
      for (int a = 0; a < 3; ++a) c->inst_bbox.push_back(bl[a]);
      for (int a = 0; a < 3; ++a) c->inst_bbox.push_back(bh[a]);
    }
    if (cuda_check(c, "lbvh build") != RR_OK) return RR_E_CUDA;
    // ---- traversal-stack bound: traverse() pushes at most one child per inner node on the path, so a tree
    // deeper than RR_STACK inner nodes could drop subtrees; refuse it instead (Morton ties of 61-bit keys
    // keep real scenes far below: config 4 measures 36, config 3 28).
    if (node_base > 0) {
      std::vector<int2> kids((size_t)node_base);
      if (cudaMemcpy2D(kids.data(), sizeof(int2), reinterpret_cast<const char*>(c->nodes.p) + 3 * sizeof(float4),
                       4 * sizeof(float4), sizeof(int2), (size_t)node_base, cudaMemcpyDeviceToHost) != cudaSuccess)
        return cuda_check(c, "bvh depth check");
      std::vector<int> roots(c->inst_root);
      roots.push_back(static_root);
      int depth = 0;
      std::vector<std::pair<int, int>> todo;
      for (int r : roots) {
        todo.assign(1, {r, 0});
        while (!todo.empty()) {
          auto [n, d] = todo.back();
          todo.pop_back();
          if (n < 0) continue;
          depth = std::max(depth, d + 1);
          if (d + 1 > RR_STACK || n >= node_base) break;
          todo.push_back({kids[n].x, d + 1});
          todo.push_back({kids[n].y, d + 1});
        }
      }
      c->bvh_depth = depth;
      if (depth > RR_STACK)
        return fail(c, RR_E_INVALID, "scene BVH deeper than the traversal stack (" + std::to_string(RR_STACK) + ")");
    }
    // ---- materials: scene materials + 2 slots (old, new) per dynamic object for edits
    c->obj_flags.upload(flags.data(), O);
    // ---- device scene
    DevScene& S = c->S;
    std::memset(&S, 0, sizeof(S));
    S.nodes = c->nodes.p;
    S.ltris = c->ltris.p;
    S.lxf = c->lxf.p;
    S.static_root = static_root;
    S.n_inst = (int)c->dyn_objects.size();
    S.tverts = c->tverts.p;
    S.tri_obj = c->d_tri_obj.p;
    S.obj_flags = c->obj_flags.p;
    S.obj_inst = c->d_obj_inst.p;
    S.obj_emit = c->obj_emit.p;
    S.obj_emitter = c->obj_emitter.p;
    S.n_emit = ne;
    S.emit_off = c->emit_off.p;
    S.emit_cnt = c->emit_cnt.p;
    S.emit_pL = c->emit_pL.p;
    S.emit_tris = c->emit_tris.p;
    S.emit_cdf = c->emit_cdf.p;
    S.n_edited = (int)edited.size();
    S.edited_tris = c->edited_tris.p;
    S.edited_cdf = c->edited_cdf.p;
    S.pA_D = pA_D;
    // camera basis (fp64 -> fp32)
    double e[3] = {d->camera.pos[0], d->camera.pos[1], d->camera.pos[2]};
    double fw[3] = {d->camera.look_at[0] - e[0], d->camera.look_at[1] - e[1], d->camera.look_at[2] - e[2]};
    double fl = std::sqrt(fw[0] * fw[0] + fw[1] * fw[1] + fw[2] * fw[2]);
    for (double& x : fw) x /= fl;
    double up[3] = {d->camera.up[0], d->camera.up[1], d->camera.up[2]};
    double r[3] = {fw[1] * up[2] - fw[2] * up[1], fw[2] * up[0] - fw[0] * up[2], fw[0] * up[1] - fw[1] * up[0]};
    double rl = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    for (double& x : r) x /= rl;
    double u[3] = {r[1] * fw[2] - r[2] * fw[1], r[2] * fw[0] - r[0] * fw[2], r[0] * fw[1] - r[1] * fw[0]};
    double tanY = std::tan((double)d->camera.vfov_deg * 3.14159265358979323846 / 360.0);
    double tanX = tanY * (double)d->camera.width / (double)d->camera.height;
    S.cam_pos = f3((float)e[0], (float)e[1], (float)e[2]);
    S.cf = f3((float)fw[0], (float)fw[1], (float)fw[2]);
    S.cr = f3((float)r[0], (float)r[1], (float)r[2]);
    S.cu = f3((float)u[0], (float)u[1], (float)u[2]);
    S.tanX = (float)tanX;
    S.tanY = (float)tanY;
    S.Aplane = (float)(4.0 * tanX * tanY);
    S.W = (int)d->camera.width;
    S.H = (int)d->camera.height;
    S.diag = (float)c->diag;
    S.eps = (float)(d->eps_rel * c->diag);
    S.dedup_tol = (float)(1e-6 * c->diag);
  } catch (std::bad_alloc&) {
    return fail(c, RR_E_OOM, "device allocation failed during scene upload");
  }
  c->have_scene = true;
  return rr_set_edit(c, 0, nullptr);
}

rr_status rr_set_edit(rr_ctx* c, uint32_t n, const rr_edit* edits) {
  NvtxRange nvtx_("rr_set_edit");
  if (!c) return RR_E_INVALID;
  if (!c->have_scene) return fail(c, RR_E_STATE, "set_edit before scene upload");
  if (n && !edits) return fail(c, RR_E_INVALID, "null edit list");
  cudaSetDevice(c->device);
  const uint32_t O = (uint32_t)c->objects.size();
  const int ND = (int)c->dyn_objects.size();
  std::vector<int> seen(O, 0);
  for (uint32_t k = 0; k < n; ++k) {
    uint32_t o = edits[k].object;
    if (o >= O || c->obj_inst[o] < 0) return fail(c, RR_E_INVALID, "edit on a non-dynamic object");
    if (seen[o]++) return fail(c, RR_E_INVALID, "object edited twice");
    for (const float* m : {edits[k].old_xform, edits[k].new_xform}) {  // rigidity (C7)
      double R[9] = {m[0], m[1], m[2], m[4], m[5], m[6], m[8], m[9], m[10]};
      double worst = 0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          double s = 0;
          for (int q = 0; q < 3; ++q) s += R[3 * q + a] * R[3 * q + b];
          worst = std::max(worst, std::fabs(s - (a == b ? 1.0 : 0.0)));
        }
      double det = R[0] * (R[4] * R[8] - R[5] * R[7]) - R[1] * (R[3] * R[8] - R[5] * R[6]) + R[2] * (R[3] * R[7] - R[4] * R[6]);
      if (!(worst <= 1e-5) || !(det > 0)) return fail(c, RR_E_INVALID, "non-rigid transform");
    }
    if (edits[k].has_material)
      for (const rr_material* mt : {&edits[k].old_material, &edits[k].new_material}) {
        if (mt->type > 1) return fail(c, RR_E_INVALID, "unknown material type in edit");
        if (mt->type == RR_GGX && !(mt->roughness > 0.0f && mt->roughness <= 1.0f))
          return fail(c, RR_E_INVALID, "GGX roughness out of (0,1]");
      }
    bool moved = std::memcmp(edits[k].old_xform, edits[k].new_xform, 12 * sizeof(float)) != 0;
    const rr_object& ob = c->objects[o];
    if (moved && (ob.emission[0] > 0 || ob.emission[1] > 0 || ob.emission[2] > 0))
      return fail(c, RR_E_INVALID, "moved objects must not emit");
  }
  // the previous render may still read the per-state tables on its stream: wait for its last event only
  if (c->ev_init && c->n_ev > 0) cudaEventSynchronize(c->ev[c->n_ev - 1]);
  try {
    DevScene& S = c->S;
    std::vector<rr_material> mats = c->materials;
    std::vector<uint32_t> om0(O), om1(O);
    for (uint32_t o = 0; o < O; ++o) om0[o] = om1[o] = c->objects[o].material;
    std::vector<uint32_t> flags = c->flags_host;
    for (int k = 0; k < ND; ++k) {
      DevInstance& I = S.inst[k];
      I.obj = c->dyn_objects[k];
      I.root = c->inst_root[k];
      I.moved = 0;
      set_identity(I.M[0]);
      set_identity(I.M[1]);
    }
    for (uint32_t k = 0; k < n; ++k) {
      const rr_edit& e = edits[k];
      int ik = c->obj_inst[e.object];
      DevInstance& I = S.inst[ik];
      std::memcpy(I.M[0], e.new_xform, 12 * sizeof(float));  // state 0 = new (N)
      std::memcpy(I.M[1], e.old_xform, 12 * sizeof(float));  // state 1 = old (O)
      I.moved = std::memcmp(e.old_xform, e.new_xform, 12 * sizeof(float)) != 0;
      if (I.moved) flags[e.object] |= OBJ_MOVED;
      if (e.has_material) {
        om1[e.object] = (uint32_t)mats.size();
        mats.push_back(e.old_material);
        om0[e.object] = (uint32_t)mats.size();
        mats.push_back(e.new_material);
      }
    }
    {  // emitter centroids in world space (emitters never move; a material-edited emitter sits at its M_N)
      const size_t ne = c->emit_tris_host.size();
      std::vector<float4> cen(ne);
      for (size_t e = 0; e < ne; ++e) {
        double cx = 0, cy = 0, cz = 0, at = 0;
        for (uint32_t t : c->emit_tris_host[e]) {
          double v[3][3];
          const int ik = c->obj_inst[c->tri_obj[t]];
          for (int a = 0; a < 3; ++a) {
            const float* p = &c->pos[3 * c->idx[3 * t + a]];
            for (int q = 0; q < 3; ++q) v[a][q] = p[q];
            if (ik >= 0) {
              const float* m = S.inst[ik].M[0];
              double w[3];
              for (int q = 0; q < 3; ++q) w[q] = m[4 * q] * v[a][0] + m[4 * q + 1] * v[a][1] + m[4 * q + 2] * v[a][2] + m[4 * q + 3];
              for (int q = 0; q < 3; ++q) v[a][q] = w[q];
            }
          }
          double e1[3], e2[3];
          for (int q = 0; q < 3; ++q) { e1[q] = v[1][q] - v[0][q]; e2[q] = v[2][q] - v[0][q]; }
          double nx = e1[1] * e2[2] - e1[2] * e2[1], ny = e1[2] * e2[0] - e1[0] * e2[2], nz = e1[0] * e2[1] - e1[1] * e2[0];
          double ak = 0.5 * std::sqrt(nx * nx + ny * ny + nz * nz);
          cx += ak * (v[0][0] + v[1][0] + v[2][0]) / 3.0;
          cy += ak * (v[0][1] + v[1][1] + v[2][1]) / 3.0;
          cz += ak * (v[0][2] + v[1][2] + v[2][2]) / 3.0;
          at += ak;
        }
        cen[e] = make_float4((float)(cx / at), (float)(cy / at), (float)(cz / at), 0.0f);
      }
      c->emit_centroid.upload_reuse(cen.data(), ne);
    }
    int n_moved = 0;
    std::vector<uint32_t> moved_tris;
    for (int k = 0; k < ND; ++k) {
      DevInstance& I = S.inst[k];
      for (int F = 0; F < 2; ++F) {
        const float* m = I.M[F];
        // inverse of [R|t] in fp64: [R^T | -R^T t]
        double inv[12];
        for (int a = 0; a < 3; ++a) {
          for (int b = 0; b < 3; ++b) inv[4 * a + b] = m[4 * b + a];
          inv[4 * a + 3] = -((double)m[a] * m[3] + (double)m[4 + a] * m[7] + (double)m[8 + a] * m[11]);
        }
        for (int q = 0; q < 12; ++q) I.Mi[F][q] = (float)inv[q];
        // world AABB of the placed object (8 corners, fp64), padded
        const float* bb = &c->inst_bbox[6 * k];
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        for (int cnr = 0; cnr < 8; ++cnr) {
          double p[3] = {bb[(cnr & 1) ? 3 : 0], bb[(cnr & 2) ? 4 : 1], bb[(cnr & 4) ? 5 : 2]};
          for (int a = 0; a < 3; ++a) {
            double x = m[4 * a] * p[0] + m[4 * a + 1] * p[1] + m[4 * a + 2] * p[2] + m[4 * a + 3];
            lo[a] = std::min(lo[a], x);
            hi[a] = std::max(hi[a], x);
          }
        }
        double pad = 1e-5 * c->diag + 1e-6;
        for (int a = 0; a < 3; ++a) {
          I.lo[F][a] = (float)(lo[a] - pad);
          I.hi[F][a] = (float)(hi[a] + pad);
        }
      }
      if (I.moved) n_moved++;
    }
    for (uint32_t t = 0; t < (uint32_t)c->tri_obj.size(); ++t) {
      int o = (int)c->tri_obj[t];
      int ik = c->obj_inst[o];
      if (ik >= 0 && S.inst[ik].moved) moved_tris.push_back(t);
    }
    int eq = 1;
    for (int k = 0; k < ND; ++k)
      if (!S.inst[k].moved) eq = 0;
    c->edited_equals_moved = eq;
    std::vector<float4> m4(mats.size());
    std::vector<uint32_t> mt(mats.size());
    for (size_t k = 0; k < mats.size(); ++k) {
      m4[k] = make_float4(mats[k].albedo[0], mats[k].albedo[1], mats[k].albedo[2], mats[k].roughness);
      mt[k] = mats[k].type;
    }
    c->mat.upload_reuse(m4.data(), m4.size());
    c->mat_type.upload_reuse(mt.data(), mt.size());
    for (auto& t : mt) t = t == RR_GGX ? 2u : t;  // RR_VNDF renders: GGX sampled from the visible normals
    c->mat_type_vndf.upload_reuse(mt.data(), mt.size());
    c->obj_mat0.upload_reuse(om0.data(), O);
    c->obj_mat1.upload_reuse(om1.data(), O);
    c->obj_flags.upload_reuse(flags.data(), O);
    S.mat = c->mat.p;
    S.mat_type = c->mat_type.p;
    S.obj_mat[0] = c->obj_mat0.p;
    S.obj_mat[1] = c->obj_mat1.p;
    S.obj_flags = c->obj_flags.p;
    S.n_moved = 0;
    S.pA_G = 0.0f;
    if (!moved_tris.empty()) {
      std::vector<float> cd;
      double area = build_cdf(c, moved_tris, cd);
      c->moved_tris.upload_reuse(moved_tris.data(), moved_tris.size());
      c->moved_cdf.upload_reuse(cd.data(), cd.size());
      S.n_moved = (int)moved_tris.size();
      S.moved_tris = c->moved_tris.p;
      S.moved_cdf = c->moved_cdf.p;
      S.pA_G = (float)(1.0 / area);
    }
  } catch (std::bad_alloc&) {
    return fail(c, RR_E_OOM, "device allocation failed in set_edit");
  }
  return cuda_check(c, "set_edit");
}

static rr_status check_args(rr_ctx* c, const rr_render_args* a) {
  if (!a) return fail(c, RR_E_INVALID, "null args");
  if (a->spp == 0) return fail(c, RR_E_INVALID, "spp must be >= 1");
  if ((a->flags & RR_TWO_WAY) && (a->spp & 1)) return fail(c, RR_E_INVALID, "spp must be even with RR_TWO_WAY");
  if (a->max_depth < 1 || a->max_depth > RR_MAX_DEPTH) return fail(c, RR_E_INVALID, "max_depth out of [1, 10]");
  if (!(a->technique_mask & 0x40u)) return fail(c, RR_E_INVALID, "technique mask must contain T7");
  if (a->technique_mask & ~0x7Fu) return fail(c, RR_E_INVALID, "unknown technique bits");
  if (a->layer_mask & ~0x7Fu) return fail(c, RR_E_INVALID, "unknown layer bits");
  if (!(a->flags & (RR_TWO_WAY | RR_DIAG_ONE_WAY_ABLATION)) && (a->flags & (RR_RECONNECT | RR_REJECT_MULTI)))
    return fail(c, RR_E_INVALID, "RR_RECONNECT / RR_REJECT_MULTI require RR_TWO_WAY (or RR_DIAG_ONE_WAY_ABLATION)");
  if ((a->flags & RR_TWO_WAY) && (a->flags & RR_DIAG_ONE_WAY_ABLATION))
    return fail(c, RR_E_INVALID, "RR_DIAG_ONE_WAY_ABLATION is one-way: RR_TWO_WAY must be off");
  if ((a->flags & RR_NO_PATH_MAPPING) &&
      (!(a->flags & RR_TWO_WAY) || (a->flags & (RR_RECONNECT | RR_REJECT_MULTI | RR_DIAG_ONE_WAY_ABLATION))))
    return fail(c, RR_E_INVALID, "RR_NO_PATH_MAPPING needs RR_TWO_WAY without RR_RECONNECT / RR_REJECT_MULTI");
  if ((a->flags & RR_VNDF) && (a->flags & RR_T6_TOWARD_LIGHT))
    return fail(c, RR_E_INVALID, "RR_VNDF and RR_T6_TOWARD_LIGHT are separate kernel variants; choose one");
  if ((a->flags & RR_TOBJ_MIDPATH) && (!(a->flags & (RR_TWO_WAY | RR_DIAG_ONE_WAY_ABLATION)) || (a->flags & RR_VNDF) ||
                                      (a->flags & RR_NO_PATH_MAPPING)))
    return fail(c, RR_E_INVALID, "RR_TOBJ_MIDPATH maps paired paths: needs RR_TWO_WAY (not with RR_VNDF / RR_NO_PATH_MAPPING)");
  if ((a->flags & RR_RECONNECT_BIDIR) && (!(a->flags & RR_RECONNECT) || (a->flags & RR_VNDF)))
    return fail(c, RR_E_INVALID, "RR_RECONNECT_BIDIR extends RR_RECONNECT (not with RR_VNDF)");
  if (a->flags & ~(RR_TWO_WAY | RR_RECONNECT | RR_REJECT_MULTI | RR_ACCUMULATE | RR_COUNT_TRAVERSAL | RR_VNDF |
                   RR_DIAG_ONE_WAY_ABLATION | RR_NO_PATH_MAPPING | RR_T6_TOWARD_LIGHT | RR_TOBJ_MIDPATH |
                   RR_RECONNECT_BIDIR))
    return fail(c, RR_E_INVALID, "unknown flag bits");
  if (a->shard_count == 0 || a->shard_index >= a->shard_count) return fail(c, RR_E_INVALID, "bad shard");
  return RR_OK;
}

static uint32_t eff_mask(const rr_ctx* c, uint32_t mask) {
  if (c->S.n_moved == 0) mask &= ~0x38u;   // T4-T6 need a ghost set
  if (c->S.n_edited == 0) mask &= ~0x07u;
  return mask;
}
static int paired(const rr_ctx* c, uint32_t mask, int l) {
  bool pair25 = (mask & 2u) && (mask & 16u) && c->S.n_moved > 0 && c->edited_equals_moved;
  if (pair25 && l == 2) return 5;
  if (pair25 && l == 5) return 2;
  return l;
}
static KArgs make_kargs(rr_ctx* c, const rr_render_args* a, uint32_t mask, int l, int side) {
  KArgs K;
  std::memset(&K, 0, sizeof(K));
  K.tech = l;
  K.tech_q = paired(c, mask, l);
  K.side = side;
  K.max_depth = (int)a->max_depth;
  K.mask = mask;
  // paired control flow (no mapped-only partner terms; reconnection / rejection allowed) in two-way mode and in
  // the diagnostic one-way ablation; the ablation changes the weights only (rr_shade.cuh finish)
  K.two_way = (a->flags & (RR_TWO_WAY | RR_DIAG_ONE_WAY_ABLATION)) ? 1 : 0;
  K.diag = (a->flags & RR_DIAG_ONE_WAY_ABLATION) ? 1 : 0;
  K.nopm = (a->flags & RR_NO_PATH_MAPPING) ? 1 : 0;
  if (K.nopm) K.mask |= 0x100u;  // path_value: static paths rejected
  K.count = (a->flags & RR_COUNT_TRAVERSAL) ? 1 : 0;
  K.mat_type_vndf = (a->flags & RR_VNDF) ? c->mat_type_vndf.p : nullptr;
  K.t6_centroid = (a->flags & RR_T6_TOWARD_LIGHT) ? c->emit_centroid.p : nullptr;
  K.n_centroid = (int)c->emit_centroid.n;
  K.tobj = (a->flags & RR_TOBJ_MIDPATH) ? 1 : 0;
  K.recon_bidir = (a->flags & RR_RECONNECT_BIDIR) ? 1 : 0;
  K.reconnect = (a->flags & RR_RECONNECT) ? 1 : 0;
  K.reject_multi = (a->flags & RR_REJECT_MULTI) ? 1 : 0;
  K.seed = a->seed;
  K.sigma = side == 0 ? 1.0f : -1.0f;
  K.inv_spp = 1.0f / (float)a->spp;
  K.jacobian_max = a->jacobian_max > 0 ? a->jacobian_max : 10.0f;
  K.alpha_min = a->alpha_min;
  K.dmin = (float)(a->dmin_rel * c->diag);
  uint64_t npix = (uint64_t)c->cam.width * c->cam.height;
  K.n_total = (a->flags & RR_TWO_WAY) ? npix * a->spp / 2 : npix * a->spp;
  K.shard_index = a->shard_index;
  K.shard_count = a->shard_count;
  uint64_t nb = (K.n_total + 0xFFFF) >> 16;
  uint64_t local_blocks = nb > a->shard_index ? (nb - a->shard_index + a->shard_count - 1) / a->shard_count : 0;
  K.n_local = local_blocks << 16;
  K.stats = c->stats.p;
  K.perm = nullptr;
  // batch refill (rr_residual.cu residual_loop): a warp's free lanes take new samples together once RR_REFILL lanes
  // are free, so the lanes of a batch start from neighbouring (ordered) samples and advance in step; T1 / T4 (short,
  // emitter-rooted samples of very different lengths) with half warps (config 4: 4.93 s at 32 for every technique
  // vs 7.01 s with immediate refill; T1 / T4 alone were faster at 8-16)
  K.refill_min = (l == 1 || l == 4) ? RR_REFILL / 2 : RR_REFILL;
  return K;
}
// grid of one residual launch (persistent lanes, rr_residual.cu)
static int prepare_launch(rr_ctx*, KArgs& K) { return residual_grid(K.tech == 3 || K.tech == 6, K.n_local); }

rr_status rr_render_residual(rr_ctx* c, const rr_render_args* a, float* d_image, uint64_t stream) {
  NvtxRange nvtx_("rr_render_residual");
  if (!c) return RR_E_INVALID;
  if (!c->have_scene) return fail(c, RR_E_STATE, "render before scene upload");
  if (!d_image) return fail(c, RR_E_INVALID, "null image");
  rr_status s = check_args(c, a);
  if (s != RR_OK) return s;
  cudaSetDevice(c->device);
  if (cuda_check(c, "before render") != RR_OK) return RR_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  if (!c->ev_init) {
    for (int k = 0; k < 32; ++k) cudaEventCreate(&c->ev[k]);
    c->ev_init = true;
  }
  uint32_t mask = eff_mask(c, a->technique_mask);
  c->last_mask = mask;
  size_t img_bytes = (size_t)c->cam.width * c->cam.height * 4 * sizeof(float);
  if (!(a->flags & RR_ACCUMULATE)) cudaMemsetAsync(d_image, 0, img_bytes, st);
  cudaMemsetAsync(c->stats.p, 0, STAT_COUNT * sizeof(unsigned long long), st);
  cudaMemsetAsync(c->work.p, 0, 16 * sizeof(unsigned long long), st);
  int ne = 0, nl = 0;
  c->n_sorted = 0;
  cudaEventRecord(c->ev[ne++], st);
  int sides = (a->flags & RR_TWO_WAY) ? 2 : 1;
  for (int l = 1; l <= 7; ++l) {
    if (!((mask >> (l - 1)) & 1u)) continue;
    if (a->layer_mask && !((a->layer_mask >> (l - 1)) & 1u)) continue;  // per-technique layer
    for (int side = 0; side < sides; ++side) {
      KArgs K = make_kargs(c, a, mask, l, side);
      K.image = d_image;
      K.work = c->work.p + (nl++);
      if (K.n_local == 0) continue;
#if RR_SAMPLE_SORT
      const bool sortable = (l <= 3 && c->S.n_edited > 0) || (l >= 4 && l <= 6 && c->S.n_moved > 0) ||
                            (l == 7 && c->cam.width <= 16384 && c->cam.height <= 8192);
      // start-ray order (sample_order); small launches keep index order (the sort's two extra launches cost more)
      if (((RR_SORT_MASK >> (l - 1)) & 1u) && sortable && K.n_local >= (1ull << 18)) {
        try {
          const size_t n = (size_t)K.n_local;
          // box of the start points: the dynamic (edited) objects in state `side` for T1-T3, the moved objects at
          // the other state's placement (the base path's ghosts) for T4-T6
          float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
          const int place = l <= 3 ? side : 1 - side;
          for (int k = 0; k < c->S.n_inst; ++k) {
            const DevInstance& I = c->S.inst[k];
            if (l >= 4 && !I.moved) continue;
            for (int q = 0; q < 3; ++q) {
              lo[q] = std::min(lo[q], I.lo[place][q]);
              hi[q] = std::max(hi[q], I.hi[place][q]);
            }
          }
          const size_t need = sample_order(c->S, K, lo, hi, nullptr, nullptr, nullptr, nullptr, nullptr, 0, st);
          if (c->ord_perm.cap < n) {
            for (DevBuf<uint32_t>* b : {&c->ord_keys, &c->ord_vals, &c->ord_keys2, &c->ord_perm}) {
              b->alloc(n);
              b->cap = n;
            }
          }
          if (c->ord_tmp.cap < need) {
            c->ord_tmp.alloc(need);
            c->ord_tmp.cap = need;
          }
          sample_order(c->S, K, lo, hi, c->ord_keys.p, c->ord_vals.p, c->ord_keys2.p, c->ord_perm.p, c->ord_tmp.p,
                       c->ord_tmp.cap, st);
          K.perm = c->ord_perm.p;
          c->n_sorted++;
        } catch (std::bad_alloc&) {
          K.perm = nullptr;  // no scratch: index order (same image)
        }
      }
#endif
      if (ne < 31) cudaEventRecord(c->ev[ne++], st);
      launch_residual(c->S, K, prepare_launch(c, K), st);
      if (ne < 32) cudaEventRecord(c->ev[ne++], st);
    }
  }
  c->n_ev = ne;
  return cuda_check(c, "render launch");
}

rr_status rr_render_primal(rr_ctx* c, uint32_t state, uint32_t spp, uint64_t seed, uint32_t max_depth, uint32_t flags,
                           float* d_image, uint64_t stream) {
  NvtxRange nvtx_("rr_render_primal");
  if (!c) return RR_E_INVALID;
  if (!c->have_scene) return fail(c, RR_E_STATE, "render before scene upload");
  if (!d_image || spp == 0 || state > 1 || max_depth < 1 || max_depth > RR_MAX_DEPTH)
    return fail(c, RR_E_INVALID, "bad primal render arguments");
  cudaSetDevice(c->device);
  if (cuda_check(c, "before primal") != RR_OK) return RR_E_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(d_image, 0, (size_t)c->cam.width * c->cam.height * 4 * sizeof(float), st);
  cudaMemsetAsync(c->stats.p, 0, STAT_COUNT * sizeof(unsigned long long), st);
  if (flags & ~(uint32_t)(RR_COUNT_TRAVERSAL | RR_PRIMAL_SHARED_STREAMS)) return fail(c, RR_E_INVALID, "unknown primal flag bits");
  launch_primal(c->S, (int)state, seed, (int)max_depth, spp, d_image, c->stats.p, (flags & RR_COUNT_TRAVERSAL) != 0,
                (flags & RR_PRIMAL_SHARED_STREAMS) != 0, st);
  return cuda_check(c, "primal launch");
}

rr_status rr_render_residual_host(rr_ctx* c, const rr_render_args* a, float* h_image) {
  if (!c || !h_image) return fail(c, RR_E_INVALID, "null argument");
  if (!c->have_scene) return fail(c, RR_E_STATE, "render before scene upload");
  cudaSetDevice(c->device);
  size_t n = (size_t)c->cam.width * c->cam.height * 4;
  try {
    DevBuf<float> img(n);
    if (a && (a->flags & RR_ACCUMULATE)) cudaMemcpy(img.p, h_image, n * sizeof(float), cudaMemcpyHostToDevice);
    rr_status s = rr_render_residual(c, a, img.p, 0);
    if (s != RR_OK) return s;
    if (cudaMemcpy(h_image, img.p, n * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess)
      return cuda_check(c, "copy back");
  } catch (std::bad_alloc&) {
    return fail(c, RR_E_OOM, "image allocation failed");
  }
  return cuda_check(c, "render_host");
}

rr_status rr_get_stats(rr_ctx* c, rr_stats* out) {
  if (!c || !out) return RR_E_INVALID;
  cudaSetDevice(c->device);
  unsigned long long h[STAT_COUNT];
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_check(c, "stats sync");
  cudaMemcpy(h, c->stats.p, sizeof(h), cudaMemcpyDeviceToHost);
  std::memset(out, 0, sizeof(*out));
  out->samples = h[STAT_SAMPLES];
  out->connections = h[STAT_CONNECTIONS];
  out->accepted = h[STAT_ACCEPTED];
  out->rejected = h[STAT_REJECTED];
  out->unpaired = h[STAT_UNPAIRED];
  out->mapped_only = h[STAT_MAPPED_ONLY];
  out->reconnected = h[STAT_RECONNECTED];
  out->closest_rays = h[STAT_CLOSEST];
  out->shadow_rays = h[STAT_SHADOW];
  out->instance_queries = h[STAT_INST];
  out->splats = h[STAT_SPLATS];
  out->offscreen = h[STAT_OFFSCREEN];
  out->zero_pairs = h[STAT_ZERO];
  out->nodes_visited = h[STAT_NODES];
  out->tris_tested = h[STAT_TRIS];
  for (int r = 0; r < 6; ++r) out->rejected_by[r] = h[STAT_REJBY + r];
  for (int r = 0; r < 8; ++r) out->sched[r] = h[STAT_SCHED + r];
  for (int r = 0; r < 16; ++r) out->r_hist[r] = h[STAT_RHIST + r];
  out->sched[5] = (uint64_t)c->bvh_depth;
  out->sched[1] = (uint64_t)c->n_sorted;
  out->effective_mask = c->last_mask;
  out->n_moved = 0;
  for (int k = 0; k < c->S.n_inst; ++k) out->n_moved += c->S.inst[k].moved ? 1 : 0;
  return cuda_check(c, "get_stats");
}

rr_status rr_last_timings(rr_ctx* c, float* out, uint32_t n) {
  if (!c || !out) return RR_E_INVALID;
  cudaSetDevice(c->device);
  for (uint32_t k = 0; k < n; ++k) out[k] = 0.0f;
  if (c->n_ev < 3) return RR_OK;
  cudaEventSynchronize(c->ev[c->n_ev - 1]);
  if (n > 0) cudaEventElapsedTime(&out[0], c->ev[0], c->ev[c->n_ev - 1]);
  float kern = 0.0f;
  for (int k = 1; 2 * k < c->n_ev; ++k) {  // launch k: events 2k-1 (start) and 2k (end)
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, c->ev[2 * k - 1], c->ev[2 * k]);
    kern += ms;
    if ((uint32_t)k < n && k < 15) out[k] = ms;
  }
  if (n > 15) out[15] = out[0] - kern;  // outside the residual kernels: clears and the ordering pre-passes
  return cuda_check(c, "timings");
}

rr_status rr_dump_paths(rr_ctx* c, const rr_render_args* a, uint32_t technique, uint32_t side, uint64_t i_begin,
                        uint64_t i_end, rr_path_record* host_out, uint64_t capacity, uint64_t* n_out) {
  if (!c || !host_out || !n_out) return fail(c, RR_E_INVALID, "null argument");
  if (!c->have_scene) return fail(c, RR_E_STATE, "dump before scene upload");
  rr_status s = check_args(c, a);
  if (s != RR_OK) return s;
  if (technique < 1 || technique > 7 || side > 1 || i_end < i_begin) return fail(c, RR_E_INVALID, "bad range");
  cudaSetDevice(c->device);
  *n_out = 0;
  uint32_t mask = eff_mask(c, a->technique_mask);
  if (!((mask >> (technique - 1)) & 1u) || i_end == i_begin) return RR_OK;
  try {
    DevBuf<rr_path_record> recs(capacity ? capacity : 1);
    DevBuf<unsigned long long> cnt(1);
    DevBuf<float> img(4);
    cudaMemset(cnt.p, 0, sizeof(unsigned long long));
    cudaMemset(c->stats.p, 0, STAT_COUNT * sizeof(unsigned long long));
    cudaMemset(c->work.p, 0, 16 * sizeof(unsigned long long));
    KArgs K = make_kargs(c, a, mask, (int)technique, (int)side);
    K.work = c->work.p;
    K.image = img.p;
    K.dump = 1;
    K.i_begin = i_begin;
    K.n_local = i_end - i_begin;
    K.recs = recs.p;
    K.rec_count = cnt.p;
    K.rec_cap = capacity;
    launch_residual(c->S, K, prepare_launch(c, K), 0);
    if (cudaDeviceSynchronize() != cudaSuccess) return cuda_check(c, "dump");
    unsigned long long n = 0;
    cudaMemcpy(&n, cnt.p, sizeof(n), cudaMemcpyDeviceToHost);
    uint64_t m = std::min<uint64_t>(n, capacity);
    if (m) cudaMemcpy(host_out, recs.p, m * sizeof(rr_path_record), cudaMemcpyDeviceToHost);
    *n_out = m;
  } catch (std::bad_alloc&) {
    return fail(c, RR_E_OOM, "record buffer allocation failed");
  }
  return cuda_check(c, "dump");
}

rr_status rr_trace(rr_ctx* c, uint32_t state, uint32_t n, const float* d_rays, float* d_hits, uint64_t stream) {
  if (!c || (n && (!d_rays || !d_hits)) || state > 1) return fail(c, RR_E_INVALID, "bad argument");
  if (!c->have_scene) return fail(c, RR_E_STATE, "trace before scene upload");
  cudaSetDevice(c->device);
  if (n) launch_trace(c->S, (int)state, n, d_rays, d_hits, (cudaStream_t)stream);
  return cuda_check(c, "trace");
}

rr_status rr_segment(rr_ctx* c, uint32_t n, const float* d_segs, float* d_out, uint64_t stream) {
  if (!c || (n && (!d_segs || !d_out))) return fail(c, RR_E_INVALID, "bad argument");
  if (!c->have_scene) return fail(c, RR_E_STATE, "segment before scene upload");
  cudaSetDevice(c->device);
  if (n) launch_segment(c->S, n, d_segs, d_out, (cudaStream_t)stream);
  return cuda_check(c, "segment");
}

rr_status rr_philox(rr_ctx* c, uint32_t n, const uint32_t* d_ctr, uint32_t key_lo, uint32_t key_hi, uint32_t* d_out,
                    uint64_t stream) {
  if (!c || (n && (!d_ctr || !d_out))) return fail(c, RR_E_INVALID, "bad argument");
  cudaSetDevice(c->device);
  if (n) launch_philox(n, d_ctr, key_lo, key_hi, d_out, (cudaStream_t)stream);
  return cuda_check(c, "philox");
}

}  // extern "C"
