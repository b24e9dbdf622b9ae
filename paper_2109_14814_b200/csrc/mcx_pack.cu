// mcx_pack.cu — canonical triangle packing and the culling hierarchy (libmcx.so).
//
// pack_kernel: quad (i, k) of a (4, M, N) half-layer grid → triangles T¹ = {v00,
// v10, v01}, T² = {v10, v01, v11} with θ wrapping mod N (PAPER.md
// T^{u1}/T^{u2} vertex sets), packed as origin + two edges + bivector + norm and an
// exact AABB, with the op sequence of oracle/canonical.py:pack (bit-identical).
// Original triangle index t = 2·(i + N·k) + τ (PAPER.md kernel step 3).  In the
// tiled order the record of t is stored at 2·storage_quad(i, k) + τ and perm[]
// maps storage position → t, so the search can emit original indices.
//
// levels: exact unions of AABBs over consecutive storage ranges — groups of 32
// (gbox), B tiles of 512 (tbox) and A blocks of 1024 (bbox) — the hierarchy that
// MCX_MODE_CULL rejects whole blocks with.  A union box is disjoint from another
// box only if every member is, so culling never changes the hit set.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mcx.h"
#include "mcx_common.cuh"

namespace mcx {

__global__ void pack_kernel(const double* __restrict__ coords, uint32_t N, uint32_t M, int tiled,
                            double* __restrict__ box, double* __restrict__ geo, uint32_t* __restrict__ perm,
                            uint32_t* __restrict__ status) {
  const uint64_t n_tri = 2ull * N * (M - 1);
  bool bad = false;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n_tri;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t q = t >> 1;
    const int tau = (int)(t & 1);
    const uint32_t i = (uint32_t)(q % N), k = (uint32_t)(q / N);
    const uint32_t ip = (i + 1 == N) ? 0 : i + 1;
    const uint64_t dst = tiled ? 2 * storage_quad(i, k, N, M - 1) + tau : t;
    double v0[4], v1[4], v2[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double* pl = coords + (uint64_t)c * M * N;
      const double w00 = __ldg(pl + (uint64_t)k * N + i), w10 = __ldg(pl + (uint64_t)k * N + ip);
      const double w01 = __ldg(pl + (uint64_t)(k + 1) * N + i), w11 = __ldg(pl + (uint64_t)(k + 1) * N + ip);
      v0[c] = __dadd_rn(tau ? w01 : w00, 0.0);  // canonicalise -0.0
      v1[c] = __dadd_rn(w10, 0.0);
      v2[c] = __dadd_rn(tau ? w11 : w01, 0.0);
      bad |= !(isfinite(v0[c]) && isfinite(v1[c]) && isfinite(v2[c]));
    }
    double b[8], g[20];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      b[c] = fmin(fmin(v0[c], v1[c]), v2[c]);
      b[4 + c] = fmax(fmax(v0[c], v1[c]), v2[c]);
      g[c] = v0[c];
      g[4 + c] = __dsub_rn(v1[c], v0[c]);
      g[8 + c] = __dsub_rn(v2[c], v0[c]);
    }
    const double* e1 = g + 4;
    const double* e2 = g + 8;
    const int bi[6] = {0, 0, 0, 1, 1, 2}, bj[6] = {1, 2, 3, 2, 3, 3};
#pragma unroll
    for (int p = 0; p < 6; ++p)
      g[12 + p] = __dsub_rn(__dmul_rn(e1[bi[p]], e2[bj[p]]), __dmul_rn(e1[bj[p]], e2[bi[p]]));
    double n1 = __dmul_rn(e1[0], e1[0]);
    n1 = __dadd_rn(n1, __dmul_rn(e1[1], e1[1]));
    n1 = __dadd_rn(n1, __dmul_rn(e1[2], e1[2]));
    n1 = __dadd_rn(n1, __dmul_rn(e1[3], e1[3]));
    double n2 = __dmul_rn(e2[0], e2[0]);
    n2 = __dadd_rn(n2, __dmul_rn(e2[1], e2[1]));
    n2 = __dadd_rn(n2, __dmul_rn(e2[2], e2[2]));
    n2 = __dadd_rn(n2, __dmul_rn(e2[3], e2[3]));
    g[18] = __dmul_rn(__dsqrt_rn(n1), __dsqrt_rn(n2));
    g[19] = 0.0;
    // 16-byte vector stores (records are 64 / 160 B, 16-byte aligned)
    double2* bo = reinterpret_cast<double2*>(box + dst * MCX_BOX_STRIDE);
    double2* go = reinterpret_cast<double2*>(geo + dst * MCX_GEO_STRIDE);
#pragma unroll
    for (int v = 0; v < 4; ++v) bo[v] = make_double2(b[2 * v], b[2 * v + 1]);
#pragma unroll
    for (int v = 0; v < 10; ++v) go[v] = make_double2(g[2 * v], g[2 * v + 1]);
    if (perm) perm[dst] = (uint32_t)t;
  }
  if (status && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(status, 1u);
}

// Culling hierarchy in one pass: one CTA per A block of 1024 records (= 2 B tiles
// = 32 groups).  Each thread unions 4 consecutive records, 8 lanes form a group
// (shuffle), the CTA's 32 group boxes give its 2 tile boxes and its block box.
__global__ void __launch_bounds__(256) levels_kernel(const Box* __restrict__ box, uint64_t n, Box* __restrict__ gbox,
                                                     Box* __restrict__ tbox, Box* __restrict__ bbox) {
  __shared__ Box gsm[A_BLOCK / GROUP];
  const uint64_t blk = blockIdx.x;
  const int tid = threadIdx.x;
  double lo[4], hi[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) { lo[c] = __longlong_as_double(0x7ff0000000000000ll); hi[c] = -lo[c]; }
  const uint64_t r0 = blk * A_BLOCK + 4ull * tid;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (r0 + u < n) {
      const double2* s = reinterpret_cast<const double2*>(box + r0 + u);
      const double2 a = __ldg(s), b = __ldg(s + 1), c = __ldg(s + 2), d = __ldg(s + 3);
      lo[0] = fmin(lo[0], a.x); lo[1] = fmin(lo[1], a.y); lo[2] = fmin(lo[2], b.x); lo[3] = fmin(lo[3], b.y);
      hi[0] = fmax(hi[0], c.x); hi[1] = fmax(hi[1], c.y); hi[2] = fmax(hi[2], d.x); hi[3] = fmax(hi[3], d.y);
    }
  }
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  }
  const uint64_t ng = (n + GROUP - 1) / GROUP;
  if ((tid & 7) == 0) {
    Box r;
#pragma unroll
    for (int c = 0; c < 4; ++c) { r.lo[c] = lo[c]; r.hi[c] = hi[c]; }
    gsm[tid >> 3] = r;
    const uint64_t g = blk * (A_BLOCK / GROUP) + (tid >> 3);
    if (g < ng) gbox[g] = r;
  }
  __syncthreads();
  if (tid < 3) {
    const int g0 = tid == 2 ? 0 : tid * (TILE / GROUP);
    const int g1 = tid == 2 ? A_BLOCK / GROUP : g0 + TILE / GROUP;
    Box r = gsm[g0];
    for (int g = g0 + 1; g < g1; ++g)
#pragma unroll
      for (int c = 0; c < 4; ++c) { r.lo[c] = fmin(r.lo[c], gsm[g].lo[c]); r.hi[c] = fmax(r.hi[c], gsm[g].hi[c]); }
    if (tid == 2) {
      bbox[blk] = r;
    } else {
      const uint64_t tt = blk * (A_BLOCK / TILE) + tid;
      if (tt < (n + TILE - 1) / TILE) tbox[tt] = r;
    }
  }
}

static unsigned grid_for(uint64_t work, int threads) {
  uint64_t b = (work + threads - 1) / threads;
  if (b > 148ull * 64) b = 148ull * 64;
  return (unsigned)(b ? b : 1);
}

}  // namespace mcx

extern "C" {

int mcx_pack(const double* coords, uint32_t N, uint32_t M, int order, double* box, double* geo, uint32_t* perm,
             uint32_t* status, int device, void* stream) {
  using namespace mcx;
  if (N < 1 || M < 2) return set_error(MCX_E_ARG, "pack needs N >= 1 and M >= 2 (got N=%u, M=%u)", N, M);
  if (2ull * N * (M - 1) >= (1ull << 31)) return set_error(MCX_E_ARG, "triangle count must be < 2^31");
  if (order != MCX_ORDER_NATURAL && order != MCX_ORDER_TILED) return set_error(MCX_E_ARG, "unknown order %d", order);
  if (!coords || !box || !geo) return set_error(MCX_E_ARG, "null buffer");
  if (((uintptr_t)box | (uintptr_t)geo) & 15) return set_error(MCX_E_ARG, "box/geo must be 16-byte aligned");
  CUDA_TRY(cudaSetDevice(device));
  const uint64_t n = 2ull * N * (M - 1);
  if (status) CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(uint32_t), (cudaStream_t)stream));
  pack_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(coords, N, M, order == MCX_ORDER_TILED, box, geo,
                                                                  perm, status);
  CUDA_TRY(cudaGetLastError());
  return MCX_OK;
}

int mcx_levels(const double* box, uint64_t n_tri, double* gbox, double* tbox, double* bbox, int device,
               void* stream) {
  using namespace mcx;
  if (!box || !gbox || !tbox || !bbox) return set_error(MCX_E_ARG, "null buffer");
  if (((uintptr_t)box | (uintptr_t)gbox | (uintptr_t)tbox | (uintptr_t)bbox) & 15)
    return set_error(MCX_E_ARG, "level boxes must be 16-byte aligned");
  if (n_tri == 0) return MCX_OK;
  CUDA_TRY(cudaSetDevice(device));
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t nb = (n_tri + A_BLOCK - 1) / A_BLOCK;
  if (nb > 0x7fffffffull) return set_error(MCX_E_ARG, "too many records");
  levels_kernel<<<(unsigned)nb, 256, 0, s>>>(reinterpret_cast<const Box*>(box), n_tri, reinterpret_cast<Box*>(gbox),
                                             reinterpret_cast<Box*>(tbox), reinterpret_cast<Box*>(bbox));
  CUDA_TRY(cudaGetLastError());
  return MCX_OK;
}

}  // extern "C"
