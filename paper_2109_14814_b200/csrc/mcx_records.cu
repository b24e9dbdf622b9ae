// mcx_records.cu — device-side record fields of a hit list (mcx_records; the
// per-field code is mcx_records.cuh, shared with the host runtime's records pipeline).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mcx.h"
#include "mcx_common.cuh"
#include "mcx_records.cuh"

namespace mcx {

__global__ void records_kernel(const mcx_hit* __restrict__ hits, uint64_t n, const double* __restrict__ cA,
                               uint32_t NA, uint32_t MA, const double* __restrict__ sA, uint32_t NB, uint32_t MB,
                               const double* __restrict__ sB, uint64_t* __restrict__ gid, double* __restrict__ point,
                               double* __restrict__ params, unsigned* __restrict__ bad) {
  for (uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; h < n; h += (uint64_t)gridDim.x * blockDim.x) {
    const mcx_hit H = hits[h];
    if (!hit_in_range(H, NA, MA, NB, MB)) {  // never read outside the grids
      atomicOr(bad, 1u);
      gid[h] = ~0ull;
      continue;
    }
    uint64_t g;
    double pt[4], pr[4];
    record_fields(H, cA, NA, MA, MA, sA, NB, MB, sB, g, pt, pr);
    gid[h] = g;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      point[4 * h + c] = pt[c];
      params[4 * h + c] = pr[c];
    }
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
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(device));
  cudaStream_t s = (cudaStream_t)stream;
  unsigned* bad = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&bad, sizeof(unsigned), s));
  CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(unsigned), s));
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  records_kernel<<<(unsigned)blocks, 256, 0, s>>>(hits, n, coords_a, NA, MA, s_a, NB, MB, s_b, gid, point, params,
                                                  bad);
  CUDA_TRY(cudaGetLastError());
  unsigned h_bad = 0;
  CUDA_TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaFreeAsync(bad, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (h_bad) return set_error(MCX_E_ARG, "hit triangle index outside the %ux%u / %ux%u grids", NA, MA, NB, MB);
  return MCX_OK;
}
