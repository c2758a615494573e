/* rr.h -- C ABI of the B200-native residual path integral renderer (arXiv 2406.16302).
 *
 * Paper: /root/reference/PAPER.md (cited P:Lnnn); blueprint: SURVEY.md section 8 (cited C1..C12).
 * The library estimates the residual image I_new - I_old (Eq.3-5) between two states of a
 * scene that differ by rigid moves and/or material edits of "dynamic" objects, with the seven sampling
 * techniques of Sec.4, balance-heuristic MIS, the path mapping of Sec.5
 * and two-way mapping.  All arithmetic runs in the library's sm_100a kernels.
 *
 * Conventions shared by every entry point
 *  - Every function returns rr_status (0 = RR_OK).  On failure rr_last_error(ctx) describes the cause.
 *  - Host arrays passed in are COPIED during the call; the caller keeps ownership.
 *  - Device pointers (d_*) are caller-owned device memory on the context's device; the library only
 *    reads/writes them on the caller's stream (cuda_stream, a cudaStream_t passed as uint64_t; 0 = the
 *    legacy default stream).
 *  - A context is bound to one CUDA device and is NOT thread-safe; separate contexts are independent.
 *  - Asynchronous kernel faults surface as RR_E_CUDA at the next call.
 *  - No PyTorch (or any other framework) type crosses this boundary.
 */
#ifndef RR_H_
#define RR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rr_ctx rr_ctx; /* opaque, one per CUDA device */

typedef enum {
  RR_OK = 0,
  RR_E_INVALID = -1, /* bad argument: null pointer, id out of range, non-rigid transform, odd spp with
                        RR_TWO_WAY, edit on a non-dynamic object, technique mask without T7, ... */
  RR_E_STATE = -2,   /* call order: render/set_edit before scene upload */
  RR_E_CUDA = -3,    /* CUDA runtime failure (including an earlier asynchronous fault) */
  RR_E_OOM = -4      /* device allocation failed */
} rr_status;

/* ---------------------------------------------------------------------------------------------
 * Scene description.  Geometry is triangles only, with geometric normals
 * n = normalize((v1-v0) x (v2-v0)) ("as wound").  BSDFs are two-sided and reflection-only.
 * ------------------------------------------------------------------------------------------- */
enum { RR_LAMBERT = 0, RR_GGX = 1 };
typedef struct {
  uint32_t type;     /* RR_LAMBERT: rho = albedo/pi;  RR_GGX: Walter D, separable Smith G,
                        Schlick F with F0 = albedo (C3) */
  float albedo[3];   /* in [0,1] */
  float roughness;   /* GGX alpha in (0,1] (alpha = stated roughness, not squared); ignored for Lambert */
} rr_material;

enum { RR_OBJ_DYNAMIC = 1u, /* may be edited: its triangles are given in OBJECT space */
       RR_OBJ_ENV = 2u };   /* environment stand-in: excluded from the scene diagonal (C12 #24) */
typedef struct {
  uint32_t material; /* index into rr_scene_desc.materials */
  float emission[3]; /* front-face radiance; > 0 makes the object an emitter. Moved objects
                        must not emit (C1). */
  uint32_t flags;    /* RR_OBJ_* */
} rr_object;

typedef struct {
  float pos[3], look_at[3], up[3]; /* pinhole at pos, looking at look_at */
  float vfov_deg;                  /* vertical field of view */
  uint32_t width, height;          /* image size; pixel (0,0) is the top-left */
} rr_camera;

typedef struct {
  uint32_t n_vertices;
  const float* positions;      /* [n_vertices*3] xyz; static objects in world space, dynamic ones in object space */
  uint32_t n_triangles;
  const uint32_t* indices;     /* [n_triangles*3] */
  const uint32_t* tri_object;  /* [n_triangles] object id of each triangle */
  uint32_t n_objects;
  const rr_object* objects;    /* [n_objects] */
  uint32_t n_materials;
  const rr_material* materials;/* [n_materials] */
  rr_camera camera;
  float eps_rel;               /* ray epsilon = eps_rel * diagonal of static non-environment geometry */
} rr_scene_desc;

/* ---------------------------------------------------------------------------------------------
 * Edit: the state change old -> new of one dynamic object.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  uint32_t object;
  float old_xform[12], new_xform[12]; /* 3x4 row-major [R|t], x' = R x + t; R must be a rotation
                                         (|R^T R - I|_inf <= 1e-5, det > 0).  The object is "moved" iff
                                         the two transforms differ bitwise (C7). */
  uint32_t has_material;              /* 0: the object's scene material in both states */
  rr_material old_material, new_material;
} rr_edit;

/* ---------------------------------------------------------------------------------------------
 * Render arguments
 * ------------------------------------------------------------------------------------------- */
enum {
  RR_TWO_WAY = 1u,     /* sample both states, half the budget each (C8) */
  RR_RECONNECT = 2u,   /* "keep vertex the same" reconnection; requires RR_TWO_WAY */
  RR_REJECT_MULTI = 4u,/* reject diverged pairs with >= 2 dynamic vertices; requires RR_TWO_WAY */
  RR_ACCUMULATE = 8u,  /* add into d_image instead of overwriting it */
  RR_COUNT_TRAVERSAL = 16u,/* count BVH node fetches / triangle tests into rr_stats (diagnostic, ~3% slower) */
  RR_VNDF = 32u,           /* sample GGX directions from the visible normals of the incoming direction (Heitz
                              2018) instead of D(h)|n.h|; pdfs and MIS follow.  A variance-only variant
                              (SURVEY 8(f) row 4); residual renders only (the primal renderer ignores it) */
  RR_PRIMAL_SHARED_STREAMS = 128u, /* rr_render_primal only: the same random numbers for both states (Philox stream
                              state 0), so that primal(new) - primal(old) is a correlated, unbiased estimate of the
                              residual (the quality harness's reference, independent of the residual estimator) */
  RR_NO_PATH_MAPPING = 256u, /* "incremental w/o PM" (Table num_of_dynamics): both states
                              sampled by every technique (RR_TWO_WAY required, RR_RECONNECT / RR_REJECT_MULTI off),
                              no mapped path -- each base connection splats 2 sigma_F v_F(p) / spp, and a path with
                              no vertex on an edited object and no ghost crossing in its own state (a static path,
                              equal in both states) is rejected.  Unbiased; the ablation of path mapping */
  RR_T6_TOWARD_LIGHT = 512u, /* T6 samples its direction "uniformly toward the light": an emitter
                              object e is chosen uniformly (slot-0 d5) and d is uniform on the hemisphere facing e's
                              area-weighted centroid, +d the emitter side; every T6 candidate pdf uses the mixture
                              density (1/n_e) sum_e [d.(c_e - x_G) > 0] / (2 pi).  A variance-only variant (SURVEY
                              8(f) row 4), compiled into the variants kernel instantiation; exclusive with RR_VNDF */
  RR_TOBJ_MIDPATH = 1024u,  /* "transform with object movement" on a mid-path hit: while a pair is
                              undiverged, the first walk vertex x_m (m >= 2) the base path finds on a MOVED object maps
                              to the same object-space point in the other state, t(x_m) = M_Fbar M_F^-1 x_m
                              (|t'| = 1), with R_T = ratio of the walk-order area pdfs of x_m and t(x_m); the edge to
                              t(x_m) must be unoccluded in the other state, and a static base vertex whose replayed
                              partner lies on a moved object is rejected from there (the mapping stays a bijection).
                              Single-walk techniques; needs RR_TWO_WAY (or the diagnostic ablation); SURVEY 8(f) row 4,
                              variants instantiation, exclusive with RR_VNDF */
  RR_RECONNECT_BIDIR = 2048u, /* reconnection inside the two-ended techniques (T3 / T6): the single-
                              walk rule applied to the emitter-side sub-walk -- at its first index where the pair is
                              diverged and both vertices are rough the mapped y'_w reconnects to the base's y_{w+1}
                              (same target conditions, Jacobian band, rejections and R); the sensor side stays
                              replayed, so a path reconnects at most once.  Needs RR_RECONNECT; SURVEY 8(f) row 4,
                              variants instantiation, exclusive with RR_VNDF */
  RR_DIAG_ONE_WAY_ABLATION = 64u /* DIAGNOSTIC, deliberately biased: one-way
                              (side N only, N_pix*spp samples per technique, RR_TWO_WAY must be off) but with the
                              two-way pairing rules (RR_RECONNECT / RR_REJECT_MULTI allowed); accepted pairs splat
                              +v_N(p) - R v_O(q), rejected / unpaired base paths +v_N(p) with weight 1, and O paths
                              that no N sample maps to are never counted.  The estimator P:L425 warns against
                              ("two-way path mapping to ensure the coverage"); the two-way-necessity test mode. */
};
#define RR_PAPER_FLAGS (RR_TWO_WAY | RR_RECONNECT | RR_REJECT_MULTI)
#define RR_MAX_DEPTH 10

typedef struct {
  uint32_t spp;            /* samples per pixel per technique (P:L624 footnote); even with RR_TWO_WAY */
  uint64_t seed;           /* Philox4x32-10 key (C2) */
  uint32_t max_depth;      /* D = max number of path edges, 1..RR_MAX_DEPTH (C12 #1) */
  uint32_t technique_mask; /* bit l-1 enables technique l (T1..T7); must contain T7 (bit 6) */
  uint32_t flags;          /* RR_* flags above; RR_PAPER_FLAGS = the paper's method; mask 0x40 + flags 0 =
                              correlated PT.  RR_RECONNECT / RR_REJECT_MULTI need RR_TWO_WAY or
                              RR_DIAG_ONE_WAY_ABLATION; the latter excludes RR_TWO_WAY; RR_NO_PATH_MAPPING needs
                              RR_TWO_WAY alone (RR_E_INVALID otherwise) */
  float jacobian_max;      /* 10 */
  float alpha_min;         /* roughness threshold, 0.1 */
  float dmin_rel;          /* distance threshold / scene diagonal, 0.01 */
  uint32_t shard_index, shard_count; /* sample-index sharding: blocks of 2^16 indices, block-cyclic */
  uint32_t layer_mask;     /* techniques whose samples are rendered (bit l-1; 0 = all of technique_mask).  MIS
                              weights still use technique_mask, so the per-technique layers of one mask add up
                              to its full estimate (Fig. importance_sample rows B/C) */
} rr_render_args;

typedef struct {
  uint64_t samples;        /* residual samples (technique invocations on one side), incl. failed ones */
  uint64_t connections;    /* emitted base connections */
  uint64_t accepted, rejected, unpaired, mapped_only, reconnected;
  uint64_t closest_rays;   /* closest-hit queries traversing the static BLAS */
  uint64_t shadow_rays;    /* any-hit (connection) queries traversing the static BLAS */
  uint64_t instance_queries; /* dynamic-instance-only queries (crossings / re-checks), not in Mrays */
  uint64_t splats, offscreen, zero_pairs;
  uint64_t nodes_visited;  /* BVH2 internal nodes fetched (64 B each), all traversals (RR_COUNT_TRAVERSAL, else 0) */
  uint64_t tris_tested;    /* leaf triangles tested (48 B each), all traversals (RR_COUNT_TRAVERSAL, else 0) */
  uint64_t rejected_by[8]; /* by reason: 1 occluded, 2 jacobian, 3 multi, 4 target, 5 suffix-dynamic */
  uint32_t effective_mask; /* technique mask after auto-disable (T4-T6 off without moved objects) */
  uint32_t n_moved;        /* moved objects in the current edit */
  uint64_t sched[8];       /* warp-scheduler occupancy of the residual kernels (diagnostics): [0] warp
                              rounds, [2] sample steps, [3] queries per round summed, [4] lanes holding
                              a sample summed over rounds, [5] deepest BVH root-to-leaf path in inner
                              nodes (scene property; upload fails above RR_STACK = 64), [6] / [7] internal nodes fetched
                              in dynamic-instance / ghost-crossing BLAS jobs (RR_COUNT_TRAVERSAL in a library built with
                              -DRR_COUNT_JOBS=1, tools/variants.py; else 0), [1] residual launches that
                              had the sample-ordering pre-pass (one key kernel + one CUB radix sort each) */
  uint64_t r_hist[16];     /* accepted connections of reconnected pairs (R != 1, C7) by floor(log2 R) + 8, clamped to
                              [0, 15]: bin b holds R in [2^(b-8), 2^(b-7)) (SURVEY 8(f) row 3, R statistics) */
} rr_stats;

/* one record per emitted base connection (C10), for parity tests */
typedef struct {
  int32_t tech, side;
  uint64_t i;
  int32_t key_kind, key_a, key_b; /* kind 0 direct emission, 1 NEE at walk vertex a, 2 sensor at a,
                                     3 bidirectional (t = a, s = b) */
  int32_t status, reason;         /* 0 accepted, 1 rejected, 2 unpaired, 3 mapped-only (one-way) */
  int32_t pix_p;
  float term_p[3];
  int32_t pix_q;
  float term_q[3];
  float R;
} rr_path_record;

/* ---------------------------------------------------------------------------------------------
 * Entry points
 * ------------------------------------------------------------------------------------------- */
/* Create a context on CUDA device `cuda_device`.  Errors: RR_E_INVALID (null out), RR_E_CUDA. */
rr_status rr_create(int cuda_device, rr_ctx** out);
/* Free every device allocation of the context.  Null is ignored. */
void rr_destroy(rr_ctx* ctx);
/* Text of the last error on this context (never null; "" if none). */
const char* rr_last_error(const rr_ctx* ctx);

/* Upload a scene: validates it (indices in range, areas > 0, material ids exist, emission >= 0,
 * at least one emitter), copies it, builds the GPU LBVHs (one static BLAS, one BLAS per dynamic object
 * in object space; "two extra acceleration structures" realised as per-state instance
 * transforms) and the area-sampling tables.  Resets the edit to identity.  Synchronous. */
rr_status rr_scene_upload(rr_ctx* ctx, const rr_scene_desc* desc);

/* Set the state change.  Objects flagged RR_OBJ_DYNAMIC but not listed keep an
 * identity edit.  Checks rigidity; derives the moved (ghost) set; with no moved object T4-T6 are dropped
 * from every render.  No BVH rebuild.  Errors: RR_E_INVALID, RR_E_STATE. */
rr_status rr_set_edit(rr_ctx* ctx, uint32_t n, const rr_edit* edits);

/* Render this shard's residual estimate into d_image_rgba (H*W*4 fp32, device, channel 3 = 0), the
 * final normalised estimate: the sum over all shards is the full estimate of I_new - I_old.
 * Asynchronous on cuda_stream: the call only enqueues work there (memsets, the sample-ordering pre-pass, one
 * kernel per (technique, side)) and never synchronises, so after one warm-up render with the same arguments
 * (which grows the context's scratch buffers) it may run under CUDA stream capture and be replayed as a graph;
 * rr_last_timings is then meaningless until the next direct render.
 * Errors: RR_E_INVALID, RR_E_STATE, RR_E_CUDA, RR_E_OOM. */
rr_status rr_render_residual(rr_ctx* ctx, const rr_render_args* args, float* d_image_rgba, uint64_t cuda_stream);

/* Same as rr_render_residual but with HOST image memory (h_image_rgba, H*W*4 fp32): the library copies
 * the result back (blocking).  Used for end-to-end timing through the public API. */
rr_status rr_render_residual_host(rr_ctx* ctx, const rr_render_args* args, float* h_image_rgba);

/* Primal image I^D(state) (Eq.1-2; state 0 = new, 1 = old) by unidirectional path
 * tracing with next-event estimation and BSDF sampling combined by the balance heuristic, spp samples per
 * pixel, paths of <= max_depth edges, Philox key `seed` (streams disjoint from the residual ones).  Writes
 * (overwrites) d_image_rgba (H*W*4 fp32, device, channel 3 = 0); `flags`: RR_COUNT_TRAVERSAL counts node
 * fetches into rr_stats, RR_PRIMAL_SHARED_STREAMS uses one stream for both states (other bits: RR_E_INVALID).  The image a residual is added to: I_new = I_old + residual.
 * Asynchronous on cuda_stream.  Errors: RR_E_INVALID (null image, spp = 0, max_depth out of 1..RR_MAX_DEPTH,
 * state > 1), RR_E_STATE (before upload), RR_E_CUDA. */
rr_status rr_render_primal(rr_ctx* ctx, uint32_t state, uint32_t spp, uint64_t seed, uint32_t max_depth,
                           uint32_t flags, float* d_image_rgba, uint64_t cuda_stream);

/* Counters of the last render (blocking: synchronises the context's device). */
rr_status rr_get_stats(rr_ctx* ctx, rr_stats* out);

/* ---- test-only exports --------------------------------------------------------------------- */
/* Closest hit in View_state (state 0 = new, 1 = old) for n rays.  d_rays: [n*8] floats
 * (ox,oy,oz,dx,dy,dz, excluded triangle id as float bits, unused); d_hits: [n*8] floats
 * (t or -1, triangle id as float bits, px,py,pz, nx,ny,nz). */
rr_status rr_trace(rr_ctx* ctx, uint32_t state, uint32_t n, const float* d_rays, float* d_hits, uint64_t cuda_stream);
/* Segment queries for n segments d_segs [n*6] (a, b): d_out [n*10] floats = per state F in {0,1}:
 * visible(F), crossing count, sum 1/|cos|, sum t^2/|cos|, sum (len-t)^2/|cos| (C1 ghost crossings). */
rr_status rr_segment(rr_ctx* ctx, uint32_t n, const float* d_segs, float* d_out, uint64_t cuda_stream);
/* Philox4x32-10 on the device: d_ctr [n*4], key = (key_lo, key_hi), d_out [n*4]. */
rr_status rr_philox(rr_ctx* ctx, uint32_t n, const uint32_t* d_ctr, uint32_t key_lo, uint32_t key_hi,
                    uint32_t* d_out, uint64_t cuda_stream);
/* Per-connection records of samples [i_begin, i_end) of one (technique, side) into host memory
 * (blocking).  *n_out = number of records (up to capacity). */
rr_status rr_dump_paths(rr_ctx* ctx, const rr_render_args* args, uint32_t technique, uint32_t side,
                        uint64_t i_begin, uint64_t i_end, rr_path_record* host_out, uint64_t capacity,
                        uint64_t* n_out);
/* Timing of the last render's kernels, in ms (events on the render stream): out[0] = total,
 * out[1..14] = per (technique, side) residual kernel (its own launch only), out[15] = the rest of the render
 * (image / counter clears and the sample-ordering pre-passes).  Blocking. */
rr_status rr_last_timings(rr_ctx* ctx, float* out, uint32_t n);

#ifdef __cplusplus
}
#endif
#endif /* RR_H_ */
