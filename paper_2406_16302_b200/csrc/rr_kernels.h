// rr_kernels.h -- kernel argument block and launchers (internal; not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rr.h"
#include "rr_device.cuh"

namespace rr {

enum {
  STAT_SAMPLES = 0, STAT_CONNECTIONS, STAT_ACCEPTED, STAT_REJECTED, STAT_UNPAIRED, STAT_MAPPED_ONLY,
  STAT_RECONNECTED, STAT_CLOSEST, STAT_SHADOW, STAT_INST, STAT_SPLATS, STAT_OFFSCREEN, STAT_ZERO,
  STAT_NODES, STAT_TRIS, STAT_REJBY, STAT_SCHED = STAT_REJBY + 6, STAT_RHIST = STAT_SCHED + 8,
  STAT_COUNT = STAT_RHIST + 16
};

struct KArgs {
  int tech, tech_q, side, max_depth;
  uint32_t mask;
  int two_way, reconnect, reject_multi;  // two_way: paired control flow (RR_TWO_WAY or the diagnostic ablation)
  int diag;                              // RR_DIAG_ONE_WAY_ABLATION weights
  int nopm;                              // RR_NO_PATH_MAPPING: no mapped path (mask bit 8: static paths rejected)
  uint64_t seed;
  float sigma, inv_spp, jacobian_max, alpha_min, dmin;
  uint64_t n_total;                  // samples of this (technique, side) over all shards
  uint64_t n_local;                  // local sample slots (shard blocks * 2^16, or the dump range)
  uint64_t shard_index, shard_count;
  float* image;                      // H*W*4
  unsigned long long* stats;         // STAT_COUNT counters
  unsigned long long* work;          // sample-slot counter of this launch (zeroed before the launch)
  int dump;
  int count;                         // count node fetches / triangle tests (RR_COUNT_TRAVERSAL)
  const uint32_t* mat_type_vndf;     // RR_VNDF: material types with GGX = 2 (visible-normal sampling), else null
  const float4* t6_centroid;         // RR_T6_TOWARD_LIGHT: emitter centroids (world), else null
  int n_centroid;
  int tobj;                          // RR_TOBJ_MIDPATH (variants instantiation)
  int recon_bidir;                   // RR_RECONNECT_BIDIR (variants instantiation)
  uint64_t i_begin;
  const uint32_t* perm;              // processing order of the local slots (sample_order), else null
  int refill_min;                    // free lanes of a warp that take new samples together (1: each at once)
  rr_path_record* recs;
  unsigned long long* rec_count;
  uint64_t rec_cap;
};

void launch_residual(const DevScene& S, const KArgs& A, int grid, cudaStream_t st);
void launch_residual_vndf(const DevScene& S, const KArgs& A, int grid, cudaStream_t st);  // rr_residual_vndf.cu
void launch_residual_var(const DevScene& S, const KArgs& A, int grid, cudaStream_t st);   // rr_residual_var.cu
int residual_grid(bool bidir, uint64_t n);  // blocks of residual_block() threads for n sample slots
int residual_block();
void launch_primal(const DevScene& S, int F, uint64_t seed, int D, uint32_t spp, float* image,
                   unsigned long long* stats, bool count, bool shared_streams, cudaStream_t st);
// Processing order of T1-T6: the local sample slots sorted by the start ray of their base path (Morton code of the
// start point, then direction bin), so that a warp's lanes trace neighbouring rays.  Returns the bytes of
// scratch needed when keys == nullptr.  Order only: every sample is still rendered once (rr_residual.cu).
// lo / hi: world box of the start points (the technique's sample set in the base path's state).
size_t sample_order(const DevScene& S, const KArgs& A, const float lo[3], const float hi[3], uint32_t* keys,
                    uint32_t* vals, uint32_t* keys2, uint32_t* perm, void* tmp, size_t tmp_bytes, cudaStream_t st);
void launch_philox(uint32_t n, const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out, cudaStream_t st);
void launch_trace(const DevScene& S, int F, uint32_t n, const float* rays, float* hits, cudaStream_t st);
void launch_segment(const DevScene& S, uint32_t n, const float* segs, float* out, cudaStream_t st);

}  // namespace rr
