// mcx_records.cu — device-side post-processing of hits into record fields
// (Eqs. 28-29).
//
// For every hit (original triangle indices iA, iB and the solution s, t, a, b):
//   gid    = i + N1·j + N1·N2·k1 + N1·N2·(M1−1)·l1
//   point  = (p + s·e1) + t·e2 from A's grid, FMA-free
//   params = (θ_u, s_u, θ_s, s_s) estimates: T¹ by Eqs. (28)-(29),
//            T² by the affine map of its vertex parameters
// with exactly the op sequence of isect.hits_to_records (NumPy), so device and
// host records are bit-identical; the host keeps only sorting, dedup and text.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mcx.h"
#include "mcx_common.cuh"

namespace mcx {

#define MCX_TWO_PI 6.283185307179586  // fl(2π) = 2.0 * numpy.pi

// θ_i = fl(fl(2π·i) / N) as reference fourier.grid_points computes it; θ_N = fl(2π).
__device__ __forceinline__ double theta(uint32_t i, uint32_t N) {
  return i == N ? MCX_TWO_PI : __ddiv_rn(__dmul_rn(MCX_TWO_PI, (double)i), (double)N);
}

__device__ __forceinline__ void estimate(uint32_t i, uint32_t k, uint32_t N, const double* sv, int tau, double x,
                                         double y, double& th, double& ss) {
  const double th0 = theta(i, N), th1 = theta(i + 1, N);
  const double s0 = __ldg(sv + k), s1 = __ldg(sv + k + 1);
  if (tau == 0) {
    th = dadd(dmul(dsub(1.0, x), th0), dmul(x, th1));
    ss = dadd(dmul(dsub(1.0, y), s0), dmul(y, s1));
  } else {
    const double xy = dadd(x, y);
    th = dadd(dmul(dsub(1.0, xy), th0), dmul(xy, th1));
    ss = dadd(dmul(dsub(1.0, x), s1), dmul(x, s0));
  }
}

__global__ void records_kernel(const mcx_hit* __restrict__ hits, uint64_t n, const double* __restrict__ cA,
                               uint32_t NA, uint32_t MA, const double* __restrict__ sA, uint32_t NB, uint32_t MB,
                               const double* __restrict__ sB, uint64_t* __restrict__ gid, double* __restrict__ point,
                               double* __restrict__ params) {
  for (uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; h < n; h += (uint64_t)gridDim.x * blockDim.x) {
    const mcx_hit H = hits[h];
    const int tauA = H.ia & 1, tauB = H.ib & 1;
    const uint32_t qa = H.ia >> 1, qb = H.ib >> 1;
    const uint32_t i = qa % NA, k1 = qa / NA, j = qb % NB, l1 = qb / NB;
    const uint64_t n12 = (uint64_t)NA * NB;
    gid[h] = i + (uint64_t)NA * j + n12 * k1 + n12 * (uint64_t)(MA - 1) * l1;
    const uint32_t ip = (i + 1 == NA) ? 0 : i + 1;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double* pl = cA + (uint64_t)c * MA * NA;
      const double v00 = pl[(uint64_t)k1 * NA + i], v10 = pl[(uint64_t)k1 * NA + ip];
      const double v01 = pl[(uint64_t)(k1 + 1) * NA + i], v11 = pl[(uint64_t)(k1 + 1) * NA + ip];
      const double p = tauA ? v01 : v00;
      const double e1 = dsub(v10, p);
      const double e2 = dsub(tauA ? v11 : v01, p);
      point[4 * h + c] = dadd(dadd(p, dmul(H.s, e1)), dmul(H.t, e2));
    }
    double th, ss;
    estimate(i, k1, NA, sA, tauA, H.s, H.t, th, ss);
    params[4 * h + 0] = th;
    params[4 * h + 1] = ss;
    estimate(j, l1, NB, sB, tauB, H.a, H.b, th, ss);
    params[4 * h + 2] = th;
    params[4 * h + 3] = ss;
  }
}

}  // namespace mcx

extern "C" int mcx_records(const mcx_hit* hits, uint64_t n, const double* coords_a, uint32_t NA, uint32_t MA,
                           const double* s_a, uint32_t NB, uint32_t MB, const double* s_b, uint64_t* gid,
                           double* point, double* params, int device, void* stream) {
  using namespace mcx;
  if (n == 0) return MCX_OK;
  if (!hits || !coords_a || !s_a || !s_b || !gid || !point || !params) return set_error(MCX_E_ARG, "null buffer");
  if (NA < 1 || NB < 1 || MA < 2 || MB < 2) return set_error(MCX_E_ARG, "half-layers need >= 2 columns");
  CUDA_TRY(cudaSetDevice(device));
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  records_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(hits, n, coords_a, NA, MA, s_a, NB, MB, s_b, gid,
                                                                     point, params);
  CUDA_TRY(cudaGetLastError());
  return MCX_OK;
}
