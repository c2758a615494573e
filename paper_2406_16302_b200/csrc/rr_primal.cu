// rr_primal.cu -- GPU primal renderer I^D(F) (the image a residual is added to).
//
// Unidirectional path tracing of the primal path integral (Eq.1-2) in state F, paths
// of at most D edges, with next-event estimation and BSDF sampling combined by the balance heuristic in
// solid angle.  Random numbers: Philox counter (sample index lo/hi, 0x80 | stream_state << 8, 2 slot + call),
// key = seed -- technique id 0x80 is never used by the residual streams; stream_state = F, or 0 for both states
// (RR_PRIMAL_SHARED_STREAMS: the two images then use the same random numbers and their difference is a
// correlated, unbiased estimate of I(N) - I(O), the quality harness's reference).  Composite: I_new = I_old +
// residual.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "rr_device.cuh"
#include "rr_kernels.h"
#include "rr_query.cuh"
#include "rr_shade.cuh"

namespace rr {

#define RR_PRIMAL_BLOCK 128

__device__ __forceinline__ float3 emitted(const DevScene& S, const PV& x, P3 toward) {  // front face only
  if (!(dot3(x.n, sub3(toward, x.p)) > 0.0f)) return f3(0.f, 0.f, 0.f);
  float4 e = __ldg(&S.obj_emit[x.obj]);
  return f3(e.x, e.y, e.z);
}
__device__ __forceinline__ bool nonzero3(float3 v) { return v.x != 0.0f || v.y != 0.0f || v.z != 0.0f; }

template <bool COUNT>
__global__ void __launch_bounds__(RR_PRIMAL_BLOCK, 8) k_primal(const __grid_constant__ DevScene S, int F, uint64_t seed,
                                                              int D, uint64_t n, float inv_spp, float* image,
                                                              unsigned long long* stats, int stream_state) {
  QCount qc = {};
  const int npix = S.W * S.H;
  const PV E = cam_pv(S);
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < n; idx += (uint64_t)gridDim.x * blockDim.x) {
    Rng rng;
    rng.i_lo = (uint32_t)idx;
    rng.i_hi = (uint32_t)(idx >> 32);
    rng.ls = 0x80u | ((uint32_t)stream_state << 8);
    rng.k0 = (uint32_t)seed;
    rng.k1 = (uint32_t)(seed >> 32);
    const int pix = (int)(idx % (uint64_t)npix);
    float d[8];
    rng.dims(0, d);
    float3 dir = camera_dir(S, (float)(pix % S.W) + d[0], (float)(pix / S.W) + d[1]);
    QRes r;
    run_query<COUNT, true>(S, mk_ray(E.p, dir, -1, (1 << F) | QW_NO_CROSS), r, qc);
    if (!r.ok[F]) continue;
    PV prev = E, cur = hit_pv(S, r.h[F], E.p, dir, F);
    float3 thr = f3(1.f, 1.f, 1.f), L = f3(0.f, 0.f, 0.f);  // W_e G / p_cam = 1
    float prev_pdf_w = -1.0f;  // solid-angle pdf of the BSDF direction that produced `cur` (-1: camera)
    for (int edges = 1; edges <= D; ++edges) {
      // emission reached at `cur` (path with `edges` edges)
      const int em = __ldg(&S.obj_emitter[cur.obj]);
      if (em >= 0) {
        float3 Le = emitted(S, cur, prev.p);
        if (nonzero3(Le)) {
          float w = 1.0f;
          if (prev_pdf_w >= 0.0f) {  // balance heuristic vs NEE, both in solid angle at prev
            float3 dv = sub3(cur.p, prev.p);
            float d2 = dot3(dv, dv);
            float pl = __ldg(&S.emit_pL[em]) * d2 / fabsf(dot3(cur.n, norm3_exact(dv)));
            w = prev_pdf_w / (prev_pdf_w + pl);
          }
          L = L + mul3(thr, Le) * w;
        }
      }
      if (edges == D) break;
      rng.dims((uint32_t)edges, d);
      const Mat mt = load_mat(S, (uint32_t)cur.obj, F);
      const float3 wi = norm3_exact(sub3(prev.p, cur.p));
      {  // next-event estimation (path with edges + 1 edges)
        PV xl = sample_emitter(S, d[3], d[4], d[5], d[6]);
        float3 dl = sub3(xl.p, cur.p);
        float d2 = dot3(dl, dl);
        float3 wl = dl * (1.0f / sqrtf(d2));
        float3 Le = emitted(S, xl, cur.p);
        if (nonzero3(Le)) {
          run_query<COUNT, true>(S, mk_seg(cur.p, xl.p, cur.tri, xl.tri, (1 << F) | QW_NO_CROSS), r, qc);
          if (r.ok[F]) {
            float3 fr = bsdf_eval(mt, cur.n, wi, wl);
            float cosl = fabsf(dot3(xl.n, wl));
            float pL = __ldg(&S.emit_pL[__ldg(&S.obj_emitter[xl.obj])]);
            float pl_w = pL * d2 / cosl;
            float pb_w = bsdf_pdf(mt, cur.n, wi, wl);
            float w = pl_w / (pl_w + pb_w);
            float g = fabsf(dot3(cur.n, wl)) * cosl / d2;
            L = L + mul3(mul3(thr, fr), Le) * (g / pL * w);
          }
        }
      }
      float3 wo;
      if (!bsdf_sample(mt, cur.n, wi, d[1], d[2], wo)) break;
      float pw = bsdf_pdf(mt, cur.n, wi, wo);
      if (!(pw > 0.0f)) break;
      float3 fr = bsdf_eval(mt, cur.n, wi, wo);
      thr = mul3(thr, fr) * (fabsf(dot3(cur.n, wo)) / pw);
      run_query<COUNT, true>(S, mk_ray(cur.p, wo, cur.tri, (1 << F) | QW_NO_CROSS), r, qc);
      if (!r.ok[F]) break;
      prev = cur;
      cur = hit_pv(S, r.h[F], prev.p, wo, F);
      prev_pdf_w = pw;
    }
    if (nonzero3(L)) atomicAdd(reinterpret_cast<float4*>(image) + pix, make_float4(L.x * inv_spp, L.y * inv_spp, L.z * inv_spp, 0.0f));
  }
  if (stats) {
    atomicAdd(stats + STAT_CLOSEST, (unsigned long long)qc.closest);
    atomicAdd(stats + STAT_SHADOW, (unsigned long long)qc.shadow);
    if (COUNT) {
      atomicAdd(stats + STAT_NODES, (unsigned long long)qc.tc.nodes);
      atomicAdd(stats + STAT_TRIS, (unsigned long long)qc.tc.tris);
    }
  }
}

void launch_primal(const DevScene& S, int F, uint64_t seed, int D, uint32_t spp, float* image,
                   unsigned long long* stats, bool count, bool shared_streams, cudaStream_t st) {
  static int grids[64] = {0};  // per device
  static std::mutex mu;
  int dev = 0, grid = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!grids[dev & 63]) {
      int sms = 148, occ = 1;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_primal<false>, RR_PRIMAL_BLOCK, 0);
      grids[dev & 63] = sms * std::max(1, occ);
    }
    grid = grids[dev & 63];
  }
  uint64_t n = (uint64_t)S.W * S.H * spp;
  int g = (int)std::min<uint64_t>((uint64_t)grid, (n + RR_PRIMAL_BLOCK - 1) / RR_PRIMAL_BLOCK);
  const int ss = shared_streams ? 0 : F;
  if (count) k_primal<true><<<g, RR_PRIMAL_BLOCK, 0, st>>>(S, F, seed, D, n, 1.0f / (float)spp, image, stats, ss);
  else k_primal<false><<<g, RR_PRIMAL_BLOCK, 0, st>>>(S, F, seed, D, n, 1.0f / (float)spp, image, stats, ss);
}

}  // namespace rr
