/*
 * mcx.h — C ABI of the B200 mesh-intersection backend (libmcx.so).
 *
 * This is the drop-in boundary for the reference's mesh-search backend seam:
 * the `backend` argument of isect.pair_candidates / isect.find_intersections
 * (reference SPEC.md:469, 478; CLI `intersect --backend`).
 * The reference is a Python package with no FFI of its own, so
 * each entry point below names the reference operation it replaces; the ctypes
 * binding a maintainer would add is in INTEGRATION.md.
 *
 * Two layers:
 *  1. Device-pointer calls (mcx_pack … mcx_records): plain pointers and sizes;
 *     "dev" pointers are CUDA device pointers owned by the caller (the Python
 *     host allocates them as torch tensors); scratch comes from a caller
 *     workspace (size from mcx_*_workspace_bytes).
 *  2. The host-to-host runtime (mcx_context_* … mcx_find_intersections): the
 *     reference's find_intersections / layer-pair task loop as ONE call per
 *     job on host grids — upload, pack, search, records, sort, dedup and the
 *     records text all on the device; results are returned in host memory
 *     owned by the context (valid until its next call).  A context owns one
 *     device's streams, stream-ordered allocations and pinned staging buffers;
 *     use one context per host thread (contexts are independent).
 *
 * Conventions
 *  - Every call returns a status: MCX_OK, or an error whose text is available
 *    from mcx_last_error() (thread-local).  MCX_E_CAPACITY (device-pointer
 *    calls only) means the output buffer was too small; stats->n_hits then
 *    holds the exact required count, so the caller grows the buffer and reruns
 *    (results are deterministic as a set).
 *  - The calling thread's current CUDA device is preserved by every call.
 *  - Arithmetic contract: SURVEY.md §7.3 (canonical FMA-free FP64 op sequence),
 *    bit-identical to the CPU oracle on identically packed triangles.
 */
#ifndef MCX_H_
#define MCX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCX_ABI_VERSION 3

#define MCX_OK 0
#define MCX_E_CAPACITY 1
#define MCX_E_CUDA 2
#define MCX_E_ARG 3

/* Per-triangle AABB records in HBM:
 *  box: [n_tri][8] doubles = lo[4], hi[4] (exact AABB over the 3 vertices), 64 B.
 * The solve geometry (origin, edges, bivector, norm) is rebuilt from the grid for
 * the rare box survivors with the packing's own op sequence, so it is not stored. */
#define MCX_BOX_STRIDE 8

/* Search modes (identical results; they differ in how pairs are rejected). */
#define MCX_MODE_BRUTE 0     /* every (iA, iB) pair gets the 8-compare FP64 AABB test   */
#define MCX_MODE_CULL 1      /* exact union-box culling first                          */
#define MCX_MODE_PREFILTER 2 /* every pair tested, first by a conservative packed-
                                integer test on 3-bit quantised boxes (fma + alu
                                pipes), its rare passes by the exact FP64 test; calls
                                below 2^28 pairs use the FP64 sweep (faster there)   */

/* Pipelines (what is searched). */
#define MCX_PIPE_TRIANGLE 0 /* triangle pairs: triangle AABB test, then the precise test */
#define MCX_PIPE_SPEC 1     /* the SPEC's literal quad pipeline: quad
                               AABB + Moller survivors, then the 4 triangle-pair precise
                               tests of each survivor; hits are triangle pairs as above.
                               MCX_MODE_CULL only (brute force would test the same quads). */

/* Storage orders of the packed triangle records (mcx_pack). */
#define MCX_ORDER_NATURAL 0 /* record t at position t = 2·(i + N·k) + τ               */
#define MCX_ORDER_TILED 1   /* 16×16-quad tiles of 4×4-quad sub-tiles (spatially
                               compact 32/512/1024-record blocks for culling)        */

/* Hierarchy granularity (records per level box). */
#define MCX_GROUP 32   /* gbox: one box per 32 records                               */
#define MCX_TILE 512   /* tbox: one box per 512 records (B side)                     */
#define MCX_BLOCK 1024 /* bbox: one box per 1024 records (A side; = mcx_a_block())   */

typedef struct mcx_mesh_dev {
  uint64_t n_tri;         /* number of triangles = 2·N·(M−1)                         */
  const double* coords;   /* device, (4, M, N) grid: four column-major N×M planes
                             x, y, px, py                 */
  uint32_t N, M;          /* θ points, s columns                                     */
  const double* box;      /* device, [n_tri][8] in storage order, 16-byte aligned     */
  const uint32_t* perm;   /* device, [n_tri] storage position → original triangle
                             index 2·(i + N·k) + τ; NULL = natural order              */
  const double* gbox;     /* device, [⌈n/32⌉][8] group boxes; MODE_CULL / PIPE_SPEC */
  const double* tbox;     /* device, [⌈n/512⌉][8]                                    */
  const double* bbox;     /* device, [⌈n/1024⌉][8]                                   */
  const uint32_t* status; /* device flag written by mcx_pack (nonzero: non-finite
                             coordinates); checked by the searches; may be NULL      */
  uint32_t plane_rows;    /* rows between the x, y, px, py planes: 0 → M (a contiguous
                             grid); the parent's M when coords is a column range of a
                             larger resident grid (a half-layer view, mcx_mesh_view_columns) */
  uint32_t reserved;
} mcx_mesh_dev;

/* One intersecting triangle pair: A triangle ia, B triangle ib (original indices
 * 2·(i + N·k) + τ), and the solution of p + s·e1 + t·e2 = q + a·f1 + b·f2
 * (Eq. 26; the SPEC's (a, b, c, d) = (s, t, a, b)).  40 bytes. */
typedef struct mcx_hit {
  uint32_t ia, ib;
  double s, t, a, b;
} mcx_hit;

typedef struct mcx_stats {
  uint64_t n_pairs;     /* logical pairs covered (triangle pairs; PIPE_SPEC: quad pairs) */
  uint64_t n_tested;    /* box tests executed (== n_pairs in MCX_MODE_BRUTE)             */
  uint64_t n_aabb_pass; /* pairs that passed the AABB test (PIPE_SPEC: quad pairs)        */
  uint64_t n_singular;  /* precise tests rejected by the singular gate     */
  uint64_t n_hits;      /* accepted triangle pairs (may exceed the hit capacity)          */
  double kernel_ms;     /* device time of the search kernels (CUDA events, opts->timing)  */
  uint64_t n_exact_tests; /* exact FP64 box tests run (MCX_MODE_PREFILTER: pairs the
                             quantised test passed; otherwise == n_tested)                */
  uint64_t n_candidates;  /* PIPE_SPEC: quad pairs surviving AABB and Moller (the SPEC's
                             pair_candidates count); otherwise n_aabb_pass */
} mcx_stats;

typedef struct mcx_opts {
  int device;            /* CUDA device ordinal                                      */
  void* stream;          /* cudaStream_t (NULL = legacy default stream)              */
  uint64_t a_begin;      /* A storage range [a_begin, a_end); a_end = 0 → n_tri      */
  uint64_t a_end;
  uint32_t shard_index;  /* cyclic sharding of the absolute A blocks [1024 b, 1024 b +  */
  uint32_t shard_count;  /*   1024): this call takes b % count == index; 0 → 1        */
  int mode;              /* MCX_MODE_BRUTE, MCX_MODE_CULL or MCX_MODE_PREFILTER       */
  int timing;            /* nonzero: record CUDA events and fill stats->kernel_ms    */
  void* workspace;       /* device scratch, >= mcx_workspace_bytes() bytes           */
  uint64_t workspace_bytes;
  int pipeline;          /* MCX_PIPE_TRIANGLE (0) or MCX_PIPE_SPEC                   */
  uint64_t cand_cap;     /* capacity of the compacted box-test survivor list in the
                            workspace (16 B each); 0 → MCX_DEFAULT_CAND_CAP.  On
                            overflow the call fails with MCX_E_CAPACITY and the
                            stats' n_aabb_pass sum is the exact size to regrow to  */
  int orient;            /* MCX_ORIENT_AS_GIVEN (0) or MCX_ORIENT_LARGER_A: a task whose
                            B has more triangles than A (and no A range) is searched
                            with the roles exchanged, so the larger mesh is the one
                            that is blocked and sharded and the
                            smaller one is replicated; the precise test still runs as
                            (A, B) and hits keep A/B indices, so results are
                            bit-identical to MCX_ORIENT_AS_GIVEN                    */
} mcx_opts;

#define MCX_ORIENT_AS_GIVEN 0
#define MCX_ORIENT_LARGER_A 1

#define MCX_DEFAULT_CAND_CAP (1u << 20)

/* One search task of a batch (e.g. one layer-pair of the reference's plan,
 * SPEC.md:382-405): A's storage range [a_begin, a_end) (a_end = 0 → all)
 * against all of B.  Both meshes must live on opts->device. */
typedef struct mcx_task {
  const mcx_mesh_dev* A;
  const mcx_mesh_dev* B;
  uint64_t a_begin;
  uint64_t a_end;
} mcx_task;

/* A-block granularity of the kernel and of cyclic sharding. */
uint32_t mcx_a_block(void);

/* Device scratch the search needs for these meshes and options (16-byte aligned).
 * The search runs in three stages (PAPER.md kernel steps 1-9, Fig. 1): box tests
 * over all pairs (brute / prefilter / culled), compaction of the survivors into a
 * candidate list in the workspace, and the precise test (or Moller) over that list. */
uint64_t mcx_workspace_bytes(const mcx_mesh_dev* A, const mcx_mesh_dev* B, const mcx_opts* opts);
uint64_t mcx_batch_workspace_bytes(const mcx_task* tasks, uint32_t n_tasks, const mcx_opts* opts);

/* Canonical triangle packing on the device (replaces the host-side triangle
 * construction of PAPER.md kernel steps 3-4 / SPEC Quad4 split).
 * coords: device, (4, M, N) float64 = four column-major N×M planes (x, y, px, py)
 * of one half-layer.  Writes the exact AABB of each of
 * the 2·N·(M−1) triangles in the given storage order (perm: storage position →
 * original index; required for MCX_ORDER_TILED, may be NULL for NATURAL) and, when
 * gbox/tbox/bbox are non-NULL, the culling hierarchy of those records (exact union
 * boxes per 32 / 512 / 1024 consecutive records) in the same pass.  *status (device,
 * may be NULL) becomes nonzero if any coordinate is NaN/Inf; searches given that
 * mesh then fail with MCX_E_ARG (the AABB contract assumes finite inputs). */
int mcx_pack(const double* coords, uint32_t N, uint32_t M, int order, double* box, uint32_t* perm,
             double* gbox, double* tbox, double* bbox, uint32_t* status, int device, void* stream);

/* Exact union boxes over consecutive records of any box array: gbox per 32, tbox per
 * 512, bbox per 1024 (mcx_pack already writes them for its own records). */
int mcx_levels(const double* box, uint64_t n_tri, double* gbox, double* tbox, double* bbox,
               int device, void* stream);

/* Triangle-level intersection search of A against B (replaces the reference's
 * rejection kernel + findall compaction + host precise test: PAPER.md kernel
 * steps 1-9 and Fig. 1, SPEC isect.pair_candidates + find_intersections,
 * SPEC.md:469-486).  Writes up to `cap` hits (unordered) to hits (device) and
 * fills *stats (host).  Synchronises opts->stream before returning. */
int mcx_search(const mcx_mesh_dev* A, const mcx_mesh_dev* B, const mcx_opts* opts,
               mcx_hit* hits, uint64_t cap, mcx_stats* stats);

/* Many searches in ONE launch per kernel (the reference's layer-pair task loop,
 * SPEC.md:402, 504, run as one device job).  Hits of all tasks share `hits` (up to
 * cap); hit_task[k] (device, may be NULL) is the task index of hits[k]; stats[t]
 * (host, n_tasks entries) gets task t's counters.  opts->a_begin/a_end are ignored
 * (per-task ranges are in the tasks).  Synchronises opts->stream once, at the end. */
int mcx_search_batch(const mcx_task* tasks, uint32_t n_tasks, const mcx_opts* opts,
                     mcx_hit* hits, uint32_t* hit_task, uint64_t cap, mcx_stats* stats);

/* Quad-pair candidate list of the SPEC-literal predicate: not aabb_reject (quad
 * boxes) and not moller_reject (PAPER.md kernel steps
 * 5-7), brute force over all quad pairs.  A, B given as half-layer grids (device,
 * (4, M, N)).  Writes up to cap quad-pair gids (u64, unordered; gid = i + N1·j +
 * N1·N2·k1 + N1·N2·(M1−1)·l1); stats: n_pairs = n_tested = quad pairs,
 * n_aabb_pass = quad-AABB survivors, n_singular = Moller rejections, n_hits =
 * n_candidates = the exact survivor count (the compaction counter).
 * Workspace: 1024 + 64·(N_A(M_A−1) + N_B(M_B−1)) bytes + 16 per quad-AABB survivor it
 * can hold (MCX_E_CAPACITY with stats->n_aabb_pass set if that is too small),
 * 16-byte aligned.  Synchronises the stream. */
int mcx_pair_candidates(const double* coords_a, uint32_t NA, uint32_t MA,
                        const double* coords_b, uint32_t NB, uint32_t MB,
                        int device, void* stream, void* workspace, uint64_t workspace_bytes,
                        uint64_t* gids, uint64_t cap, mcx_stats* stats);

/* The same SPEC-literal candidate list from packed meshes (any storage order) with
 * exact union-box culling: quads are record pairs, the quad box is the union of its
 * two triangle boxes (= the SPEC quad AABB), the Moller stage reads the grids.
 * Identical gid set and counters to mcx_pair_candidates; stats: n_pairs = quad pairs,
 * n_tested = quad-box tests run, n_aabb_pass = quad-AABB survivors, n_singular =
 * Moller rejections, n_hits = n_candidates = candidates.  opts->mode is ignored
 * (always culls); sharding applies. */
int mcx_pair_candidates_mesh(const mcx_mesh_dev* A, const mcx_mesh_dev* B, const mcx_opts* opts,
                             uint64_t* gids, uint64_t cap, mcx_stats* stats);
uint64_t mcx_pair_candidates_mesh_workspace_bytes(const mcx_mesh_dev* A, const mcx_mesh_dev* B,
                                                  const mcx_opts* opts);

/* Device-side record fields for hits:
 * gid[k] (u64), point[k][4] = p + s·e1 + t·e2 from A's grid, params[k][4]
 * = (θ_u, s_u, θ_s, s_s) per Eqs. (28)-(29) (T² by its vertex map).  coords_a: A's
 * (4, MA, NA) grid; s_a/s_b: the half-layers' s-values (device).  Hit indices are
 * validated against the grids (MCX_E_ARG if any is out of range).  Enqueued on
 * `stream`; synchronises it only to report an invalid index. */
int mcx_records(const mcx_hit* hits, uint64_t n, const double* coords_a, uint32_t NA, uint32_t MA,
                const double* s_a, uint32_t NB, uint32_t MB, const double* s_b, uint64_t* gid,
                double* point, double* params, int device, void* stream);

/* ------------------------------------------------------------------ host-to-host runtime */

/* One IntersectionRecord, 128 bytes. */
typedef struct mcx_record {
  uint64_t gid;        /* quad-pair gid                                  */
  uint32_t ia, ib;     /* original triangle indices (τ_A = ia & 1, τ_B = ib & 1)        */
  double point[4];     /* x, y, px, py = p + s·e1 + t·e2                                */
  double bary[4];      /* (a, b, c, d) of Eq. (26)                                       */
  double params[4];    /* θ_u, s_u, θ_s, s_s (Eqs. 28-29)                                */
  uint32_t task;       /* job index within the call                                     */
  uint32_t pad[3];
} mcx_record;

/* Layer-pair tag of a job: the records text's "n1 sign1 n2 sign2" (sign: +1 / -1). */
typedef struct mcx_layer {
  int32_t n1, sign1, n2, sign2;
} mcx_layer;

typedef struct mcx_context mcx_context;
typedef struct mcx_mesh mcx_mesh;  /* a half-layer resident on a context's device */

int mcx_context_create(int device, mcx_context** ctx);
int mcx_context_destroy(mcx_context* ctx);

/* Upload a half-layer (host (4, M, N) grid + its M s-values; pinned memory gives an
 * asynchronous copy) and pack it on the context's device.  The mesh stays resident
 * until mcx_mesh_free.  mcx_mesh_view exposes it to the device-pointer calls. */
int mcx_mesh_load(mcx_context* ctx, const double* coords, uint32_t N, uint32_t M, const double* s_values,
                  mcx_mesh** mesh);
int mcx_mesh_free(mcx_mesh* mesh);
const mcx_mesh_dev* mcx_mesh_view(const mcx_mesh* mesh);

/* A whole globalized mesh uploaded once, NOT packed: the source of zero-copy half-layer
 * views (a half-layer is a contiguous column range of its mesh). */
int mcx_grid_load(mcx_context* ctx, const double* coords, uint32_t N, uint32_t M, const double* s_values,
                  mcx_mesh** grid);
/* The half-layer of columns [c0, c1] (c1 > c0) of a resident grid or mesh, packed on the
 * device from the parent's memory (no upload; plane_rows = the parent's M).  The parent
 * must outlive the view. */
int mcx_mesh_view_columns(mcx_context* ctx, const mcx_mesh* parent, uint32_t c0, uint32_t c1, mcx_mesh** view);

typedef struct mcx_job {
  const mcx_mesh* A;   /* unstable half-layer U_n1^sign1                                */
  const mcx_mesh* B;   /* stable half-layer S_n2^sign2                                  */
  mcx_layer layer;
} mcx_job;

typedef struct mcx_find_opts {
  int mode;            /* MCX_MODE_*                                                    */
  int pipeline;        /* MCX_PIPE_*                                                    */
  int dedup;           /* nonzero: drop records within 1e-9 (max-norm) of a kept earlier
                          record of the same job                          */
  int text;            /* nonzero: also produce the records text          */
  uint32_t shard_index, shard_count; /* cyclic A-block shard of every job (0, 0 → all) */
  int orient;          /* MCX_ORIENT_*, as mcx_opts.orient                               */
} mcx_find_opts;

/* Run every job on the context's device as one batched search, then on the device:
 * record fields, sort by (job, gid, τ_A, τ_B), 1e-9 dedup, and (opts->text) the
 * "%.17g" records text, one line per record in that order (byte-identical to
 * Python's f"{v:.17g}").  *records / *text point into context-owned pinned memory
 * valid until the context's next call.  stats: n_jobs entries (host). */
int mcx_intersect(mcx_context* ctx, const mcx_job* jobs, uint32_t n_jobs, const mcx_find_opts* opts,
                  const mcx_record** records, uint64_t* n_records, const char** text, uint64_t* text_bytes,
                  mcx_stats* stats);

/* find_intersections on host grids in one call: both half-layers
 * are uploaded (B's copy overlapping A's packing), packed, searched and turned into
 * records as mcx_intersect does; the meshes are released afterwards (their device
 * memory is recycled by the context's stream-ordered pool). */
int mcx_find_intersections(mcx_context* ctx, const double* coords_a, uint32_t NA, uint32_t MA,
                           const double* s_a, const double* coords_b, uint32_t NB, uint32_t MB,
                           const double* s_b, mcx_layer layer, const mcx_find_opts* opts,
                           const mcx_record** records, uint64_t* n_records, const char** text,
                           uint64_t* text_bytes, mcx_stats* stats);

/* mcx_find_intersections on half-layers read in place from larger host meshes: plane_a /
 * plane_b = the host grid's plane stride in doubles (0: N·M).  A half-layer is a column
 * range of its mesh, contiguous within each plane, so the reference's
 * HalfLayer views need no host copy. */
int mcx_find_intersections_strided(mcx_context* ctx, const double* coords_a, uint32_t NA, uint32_t MA,
                                   uint64_t plane_a, const double* s_a, const double* coords_b, uint32_t NB,
                                   uint32_t MB, uint64_t plane_b, const double* s_b, mcx_layer layer,
                                   const mcx_find_opts* opts, const mcx_record** records, uint64_t* n_records,
                                   const char** text, uint64_t* text_bytes, mcx_stats* stats);

/* Post-process a hit list that is already on the host (e.g. gathered from several
 * GPUs' shards of one job): records, sort, dedup and text exactly as mcx_intersect. */
int mcx_finish_hits(mcx_context* ctx, const mcx_hit* hits, uint64_t n_hits, const mcx_mesh* A,
                    const mcx_mesh* B, mcx_layer layer, const mcx_find_opts* opts, const mcx_record** records,
                    uint64_t* n_records, const char** text, uint64_t* text_bytes);

/* "%.17g" of one double exactly as the device formatter writes it (host build of the
 * same code; for tests).  Writes a NUL-terminated string of at most 32 bytes. */
int mcx_format_g17(double v, char* out);

const char* mcx_last_error(void);
int mcx_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MCX_H_ */
