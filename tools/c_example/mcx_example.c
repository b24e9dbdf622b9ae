/*
 * Minimal C host for the C ABI (include/mcx.h): no Python, no torch.
 *
 * Builds a synthetic pair of half-layer grids on the host, uploads them with
 * cudaMalloc/cudaMemcpy, packs them on the device (mcx_pack), runs the search in
 * every mode (mcx_search) and prints one line per mode:
 *   mode n_pairs n_tested n_aabb_pass n_singular n_hits checksum kernel_ms
 * The checksum is an order-independent sum over hits of (ia * 1000003 + ib), so the
 * modes must print the same hit count and checksum.  Then the host-to-host runtime
 * (mcx_context_create + mcx_find_intersections from the host grids) prints
 *   runtime n_hits n_records text_bytes checksum
 * with the same checksum over the (deduplicated) records' triangle pairs.
 *
 * Build (tools/c_example/Makefile): gcc + libcudart + libmcx.so.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "mcx.h"

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d CUDA error %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)
#define MK(x)                                                                        \
  do {                                                                               \
    int r_ = (x);                                                                    \
    if (r_ != MCX_OK) {                                                              \
      fprintf(stderr, "%s:%d mcx error %d: %s\n", __FILE__, __LINE__, r_, mcx_last_error()); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

/* a wavy annulus in 4D: (cos θ, sin θ, 0, 0) + smooth perturbations depending on a phase */
static void grid(double* c, uint32_t N, uint32_t M, double phase) {
  for (uint32_t k = 0; k < M; ++k) {
    const double s = -1.0 + 2.0 * k / (M - 1);
    for (uint32_t i = 0; i < N; ++i) {
      const double th = 2.0 * M_PI * i / N;
      const double v[4] = {cos(th) + 0.2 * s * cos(2 * th + phase), sin(th) + 0.2 * s * sin(3 * th - phase),
                           0.3 * s + 0.1 * sin(th + phase), 0.3 * s * cos(th - 2 * phase)};
      for (int d = 0; d < 4; ++d) c[(uint64_t)d * M * N + (uint64_t)k * N + i] = v[d];
    }
  }
}

typedef struct {
  double *coords, *box, *gbox, *tbox, *bbox;
  uint32_t *perm, *status;
  mcx_mesh_dev dev;
} mesh_t;

static void upload(mesh_t* m, const double* host, uint32_t N, uint32_t M) {
  const uint64_t n = 2ull * N * (M - 1);
  CK(cudaMalloc((void**)&m->coords, sizeof(double) * 4 * N * M));
  CK(cudaMemcpy(m->coords, host, sizeof(double) * 4 * N * M, cudaMemcpyHostToDevice));
  CK(cudaMalloc((void**)&m->box, sizeof(double) * MCX_BOX_STRIDE * n));
  CK(cudaMalloc((void**)&m->perm, sizeof(uint32_t) * n));
  CK(cudaMalloc((void**)&m->status, sizeof(uint32_t)));
  CK(cudaMalloc((void**)&m->gbox, sizeof(double) * 8 * ((n + MCX_GROUP - 1) / MCX_GROUP)));
  CK(cudaMalloc((void**)&m->tbox, sizeof(double) * 8 * ((n + MCX_TILE - 1) / MCX_TILE)));
  CK(cudaMalloc((void**)&m->bbox, sizeof(double) * 8 * ((n + MCX_BLOCK - 1) / MCX_BLOCK)));
  MK(mcx_pack(m->coords, N, M, MCX_ORDER_TILED, m->box, m->perm, m->gbox, m->tbox, m->bbox, m->status, 0, NULL));
  memset(&m->dev, 0, sizeof(m->dev));  /* plane_rows = 0: a contiguous grid */
  m->dev.n_tri = n;
  m->dev.coords = m->coords;
  m->dev.N = N;
  m->dev.M = M;
  m->dev.box = m->box;
  m->dev.perm = m->perm;
  m->dev.gbox = m->gbox;
  m->dev.tbox = m->tbox;
  m->dev.bbox = m->bbox;
  m->dev.status = m->status;
}

int main(int argc, char** argv) {
  const uint32_t N = argc > 1 ? (uint32_t)atoi(argv[1]) : 256, M = argc > 2 ? (uint32_t)atoi(argv[2]) : 129;
  if (mcx_version() != MCX_ABI_VERSION) {
    fprintf(stderr, "ABI mismatch\n");
    return 1;
  }
  double* ha = (double*)malloc(sizeof(double) * 4 * N * M);
  double* hb = (double*)malloc(sizeof(double) * 4 * N * M);
  grid(ha, N, M, 0.0);
  grid(hb, N, M, 0.7);
  mesh_t A, B;
  upload(&A, ha, N, M);
  upload(&B, hb, N, M);
  const uint64_t cap = 1 << 20;
  mcx_hit* dhits;
  CK(cudaMalloc((void**)&dhits, sizeof(mcx_hit) * cap));
  mcx_hit* hh = (mcx_hit*)malloc(sizeof(mcx_hit) * cap);
  const int modes[3] = {MCX_MODE_BRUTE, MCX_MODE_CULL, MCX_MODE_PREFILTER};
  const char* names[3] = {"brute", "cull", "prefilter"};
  for (int mi = 0; mi < 3; ++mi) {
    mcx_opts o = {0};
    o.device = 0;
    o.mode = modes[mi];
    o.timing = 1;
    o.workspace_bytes = mcx_workspace_bytes(&A.dev, &B.dev, &o);
    CK(cudaMalloc(&o.workspace, o.workspace_bytes));
    mcx_stats st;
    MK(mcx_search(&A.dev, &B.dev, &o, dhits, cap, &st));
    CK(cudaMemcpy(hh, dhits, sizeof(mcx_hit) * st.n_hits, cudaMemcpyDeviceToHost));
    unsigned long long sum = 0;
    for (uint64_t h = 0; h < st.n_hits; ++h) sum += (unsigned long long)hh[h].ia * 1000003ull + hh[h].ib;
    printf("%s %llu %llu %llu %llu %llu %llu %.3f\n", names[mi], (unsigned long long)st.n_pairs,
           (unsigned long long)st.n_tested, (unsigned long long)st.n_aabb_pass, (unsigned long long)st.n_singular,
           (unsigned long long)st.n_hits, sum, st.kernel_ms);
    CK(cudaFree(o.workspace));
  }
  /* the host-to-host runtime: host grids in, records + records text out */
  double* sv = (double*)malloc(sizeof(double) * M);
  for (uint32_t k = 0; k < M; ++k) sv[k] = -1.0 + 2.0 * k / (M - 1);
  mcx_context* ctx = NULL;
  MK(mcx_context_create(0, &ctx));
  mcx_find_opts fo = {MCX_MODE_CULL, MCX_PIPE_TRIANGLE, 0, 1, 0, 0, MCX_ORIENT_LARGER_A}; /* no dedup */
  mcx_layer layer = {1, 1, 1, -1};
  const mcx_record* recs = NULL;
  const char* text = NULL;
  uint64_t n_recs = 0, n_text = 0;
  mcx_stats st;
  MK(mcx_find_intersections(ctx, ha, N, M, sv, hb, N, M, sv, layer, &fo, &recs, &n_recs, &text, &n_text, &st));
  unsigned long long sum = 0;
  for (uint64_t r = 0; r < n_recs; ++r) sum += (unsigned long long)recs[r].ia * 1000003ull + recs[r].ib;
  printf("runtime %llu %llu %llu %llu\n", (unsigned long long)st.n_hits, (unsigned long long)n_recs,
         (unsigned long long)n_text, sum);
  MK(mcx_context_destroy(ctx));
  return 0;
}
