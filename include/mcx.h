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
 * Conventions
 *  - Plain pointers and sizes only.  "dev" pointers are CUDA device pointers
 *    owned by the caller (the Python host allocates them as torch tensors);
 *    the library never allocates device or host memory, scratch comes from the
 *    caller's workspace (size from mcx_workspace_bytes).
 *  - Every call returns a status: MCX_OK, or an error whose text is available
 *    from mcx_last_error() (thread-local).  MCX_E_CAPACITY means the hit buffer
 *    was too small; stats->n_hits then holds the exact required count, so the
 *    caller grows the buffer and reruns (results are deterministic as a set).
 *  - Reentrant across devices: one host thread per GPU; no global mutable
 *    state.  Work is enqueued on opts->stream.
 *  - Arithmetic contract: SURVEY.md §7.3 (canonical FMA-free FP64 op sequence),
 *    bit-identical to the CPU oracle on identically packed triangles.
 */
#ifndef MCX_H_
#define MCX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCX_ABI_VERSION 2

#define MCX_OK 0
#define MCX_E_CAPACITY 1
#define MCX_E_CUDA 2
#define MCX_E_ARG 3

/* Per-triangle records in HBM.
 *  box: [n_tri][8] doubles = lo[4], hi[4] (exact AABB over the 3 vertices), 64 B.
 *  geo: [n_tri][MCX_GEO_STRIDE] doubles = p[4], e1[4], e2[4],
 *       P[6] (= e1∧e2 in order 01,02,03,12,13,23), nrm (= ‖e1‖·‖e2‖), pad. */
#define MCX_BOX_STRIDE 8
#define MCX_GEO_STRIDE 20

/* Search modes. */
#define MCX_MODE_BRUTE 0 /* every (iA, iB) pair gets the 8-compare AABB test       */
#define MCX_MODE_CULL 1  /* exact block-AABB culling first; identical hit set      */
#define MCX_MODE_PREFILTER 2 /* every pair tested, first by a conservative packed-
                                integer test on 3-bit quantised boxes (fma + alu
                                pipes), its rare passes by the exact FP64 test;
                                identical hit set                                   */

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
  const double* box;      /* device, [n_tri][8] in storage order, 16-byte aligned     */
  const double* geo;      /* device, [n_tri][20] in storage order, 16-byte aligned    */
  const uint32_t* perm;   /* device, [n_tri] storage position → original triangle
                             index 2·(i + N·k) + τ; NULL = natural order              */
  const double* gbox;     /* device, [⌈n/32⌉][8] group boxes (mcx_levels); MODE_CULL */
  const double* tbox;     /* device, [⌈n/512⌉][8]                                    */
  const double* bbox;     /* device, [⌈n/1024⌉][8]                                   */
  const uint32_t* status; /* device flag written by mcx_pack (nonzero: non-finite
                             coordinates); checked by the searches; may be NULL      */
} mcx_mesh_dev;

/* One intersecting triangle pair: A triangle ia, B triangle ib, and the
 * solution of p + s·e1 + t·e2 = q + a·f1 + b·f2 (Eq. 26; the SPEC's
 * (a, b, c, d) = (s, t, a, b)).  40 bytes. */
typedef struct mcx_hit {
  uint32_t ia, ib;
  double s, t, a, b;
} mcx_hit;

typedef struct mcx_stats {
  uint64_t n_pairs;     /* logical triangle pairs covered by the call               */
  uint64_t n_tested;    /* pair AABB tests executed (== n_pairs in MCX_MODE_BRUTE)   */
  uint64_t n_aabb_pass; /* pairs that passed the triangle AABB test (solved)        */
  uint64_t n_singular;  /* solved pairs rejected by the singular gate */
  uint64_t n_hits;      /* accepted pairs (may exceed the hit capacity)            */
  double kernel_ms;     /* device time of the search kernels (CUDA events)         */
  uint64_t n_exact_tests; /* exact FP64 box tests run (MCX_MODE_PREFILTER: pairs the
                             quantised test passed; otherwise == n_tested)           */
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
} mcx_opts;

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

/* Device scratch the search needs for these meshes and options (16-byte aligned). */
uint64_t mcx_workspace_bytes(const mcx_mesh_dev* A, const mcx_mesh_dev* B, const mcx_opts* opts);
uint64_t mcx_batch_workspace_bytes(const mcx_task* tasks, uint32_t n_tasks, const mcx_opts* opts);

/* Canonical triangle packing on the device (replaces the host-side triangle
 * construction of PAPER.md kernel steps 3-4 / SPEC Quad4 split).
 * coords: device, (4, M, N) float64 = four column-major N×M planes (x, y, px, py)
 * of one half-layer.  Writes box/geo (and perm, if
 * non-NULL) for the 2·N·(M−1) triangles in the given storage order; every record
 * is bit-identical to the CPU oracle's packing of that triangle.  *status (device,
 * may be NULL) becomes nonzero if any coordinate is NaN/Inf; searches given that
 * mesh then fail with MCX_E_ARG (the AABB contract assumes finite inputs). */
int mcx_pack(const double* coords, uint32_t N, uint32_t M, int order, double* box, double* geo,
             uint32_t* perm, uint32_t* status, int device, void* stream);

/* Exact union boxes over consecutive records: gbox per 32, tbox per 512, bbox per
 * 1024 (needed by MCX_MODE_CULL).  Enqueued on `stream`. */
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
 * SPEC.md:402, 504, run as one device job): every task's work units go into a
 * single grid (brute) or a single flattened culling pass (cull).  Hits of all
 * tasks share `hits` (up to cap); hit_task[k] (device, may be NULL) is the task
 * index of hits[k]; stats[t] (host, n_tasks entries) gets task t's counters.
 * opts->a_begin/a_end are ignored (per-task ranges are in the tasks).
 * Synchronises opts->stream once, at the end. */
int mcx_search_batch(const mcx_task* tasks, uint32_t n_tasks, const mcx_opts* opts,
                     mcx_hit* hits, uint32_t* hit_task, uint64_t cap, mcx_stats* stats);

/* Quad-pair candidate list of the SPEC-literal predicate: not aabb_reject (quad
 * boxes) and not moller_reject (PAPER.md kernel steps
 * 5-7).  A, B given as half-layer grids (device, (4, M, N)).  Writes up to cap
 * quad-pair gids (u64, unordered; gid = i + N1·j + N1·N2·k1 + N1·N2·(M1−1)·l1,
 * SPEC.md:433) and *n_out = exact survivor count (the compaction counter,
 * SPEC.md:491).  Synchronises the stream. */
int mcx_pair_candidates(const double* coords_a, uint32_t NA, uint32_t MA,
                        const double* coords_b, uint32_t NB, uint32_t MB,
                        int device, void* stream, void* workspace, uint64_t workspace_bytes,
                        uint64_t* gids, uint64_t cap, uint64_t* n_out);
/* workspace for mcx_pair_candidates: 1024 + 64·(N_A(M_A−1) + N_B(M_B−1)) bytes, 16-byte aligned. */

/* The same SPEC-literal candidate list from packed meshes (mcx_pack + mcx_levels of the
 * two grids, any storage order) with exact union-box culling: quads are record pairs,
 * the quad box is the union of its two triangle boxes (= the SPEC quad AABB), the
 * Moller stage reads the grids.  Identical gid set and counters to
 * mcx_pair_candidates; stats: n_pairs = quad pairs, n_tested = quad-box tests run,
 * n_aabb_pass = quad-AABB survivors, n_singular = Moller rejections, n_hits =
 * candidates.  opts->mode is ignored (always culls); sharding applies. */
int mcx_pair_candidates_mesh(const mcx_mesh_dev* A, const double* coords_a, uint32_t NA, uint32_t MA,
                             const mcx_mesh_dev* B, const double* coords_b, uint32_t NB, uint32_t MB,
                             const mcx_opts* opts, uint64_t* gids, uint64_t cap, mcx_stats* stats);
uint64_t mcx_pair_candidates_mesh_workspace_bytes(const mcx_mesh_dev* A, const mcx_mesh_dev* B,
                                                  const mcx_opts* opts);

/* Device-side record fields for hits:
 * gid[k] (u64), point[k][4] = p + s·e1 + t·e2 from A's grid, params[k][4]
 * = (θ_u, s_u, θ_s, s_s) per Eqs. (28)-(29) (T² by its vertex map), bit-identical to
 * isect.hits_to_records.  coords_a: A's (4, MA, NA) grid; s_a/s_b: the half-layers'
 * s-values (device).  Enqueued on `stream`. */
int mcx_records(const mcx_hit* hits, uint64_t n, const double* coords_a, uint32_t NA, uint32_t MA,
                const double* s_a, uint32_t NB, uint32_t MB, const double* s_b, uint64_t* gid,
                double* point, double* params, int device, void* stream);

const char* mcx_last_error(void);
int mcx_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MCX_H_ */
