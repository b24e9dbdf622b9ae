// mcx_records.cuh — record fields of one hit (SPEC.md:427-430,
// 433, 499; Eqs. 28-29), shared by mcx_records and the device-side records
// pipeline of the host runtime (mcx_runtime.cu).
//
// For a hit (original triangle indices iA, iB and the solution s, t, a, b):
//   gid    = i + N1·j + N1·N2·k1 + N1·N2·(M1−1)·l1
//   point  = (p + s·e1) + t·e2 from A's grid, FMA-free
//   params = (θ_u, s_u, θ_s, s_s) estimates: T¹ by Eqs. (28)-(29),
//            T² by the affine map of its vertex parameters
// with exactly the op sequence of isect.record_fields (NumPy), so device and host
// records are bit-identical.
#pragma once
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

// true iff the hit's triangle indices lie inside the two grids
__device__ __forceinline__ bool hit_in_range(const mcx_hit& H, uint32_t NA, uint32_t MA, uint32_t NB, uint32_t MB) {
  return (uint64_t)H.ia < 2ull * NA * (MA - 1) && (uint64_t)H.ib < 2ull * NB * (MB - 1);
}

// MpA: plane stride of A's grid in rows (MA for a contiguous grid).
__device__ __forceinline__ void record_fields(const mcx_hit& H, const double* __restrict__ cA, uint32_t NA,
                                              uint32_t MA, uint32_t MpA, const double* __restrict__ sA, uint32_t NB,
                                              uint32_t MB, const double* __restrict__ sB, uint64_t& gid,
                                              double point[4], double params[4]) {
  const int tauA = H.ia & 1, tauB = H.ib & 1;
  const uint32_t qa = H.ia >> 1, qb = H.ib >> 1;
  const uint32_t i = qa % NA, k1 = qa / NA, j = qb % NB, l1 = qb / NB;
  const uint64_t n12 = (uint64_t)NA * NB;
  gid = i + (uint64_t)NA * j + n12 * k1 + n12 * (uint64_t)(MA - 1) * l1;
  const uint32_t ip = (i + 1 == NA) ? 0 : i + 1;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double* pl = cA + (uint64_t)c * MpA * NA;
    const double v00 = pl[(uint64_t)k1 * NA + i], v10 = pl[(uint64_t)k1 * NA + ip];
    const double v01 = pl[(uint64_t)(k1 + 1) * NA + i], v11 = pl[(uint64_t)(k1 + 1) * NA + ip];
    const double p = tauA ? v01 : v00;
    const double e1 = dsub(v10, p);
    const double e2 = dsub(tauA ? v11 : v01, p);
    point[c] = dadd(dadd(p, dmul(H.s, e1)), dmul(H.t, e2));
  }
  estimate(i, k1, NA, sA, tauA, H.s, H.t, params[0], params[1]);
  estimate(j, l1, NB, sB, tauB, H.a, H.b, params[2], params[3]);
}

}  // namespace mcx
