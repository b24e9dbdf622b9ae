// Device %.17g formatter throughput (csrc/mcx_format.cuh): one double per thread over
// many CTAs, and the latency of one thread formatting a run of values back to back.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2109_14814_b200/csrc \
//        -o tools/microbench/fmt_bench tools/microbench/fmt_bench.cu && tools/microbench/fmt_bench
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <random>
#include <vector>

#include "mcx_format.cuh"

__global__ void fmt_many(const double* v, int n, char* out, int* len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  char buf[32];
  const int k = mcx::fmt::fmt_g17(v[i], buf);
  for (int j = 0; j < k; ++j) out[(size_t)i * 32 + j] = buf[j];
  len[i] = k;
}

__global__ void fmt_chain(const double* v, int n, long long* cycles, int* sink) {
  char buf[32];
  int acc = 0;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc += mcx::fmt::fmt_g17(v[i], buf) + buf[acc & 15];
  const long long t1 = clock64();
  *cycles = t1 - t0;
  *sink = acc;
}

// one warp formatting records lines: lane f < 17 formats field f (the small path's layout)
__global__ void fmt_lines(const double* v, int nlines, long long* cycles, int* sink) {
  const int lane = threadIdx.x & 31;
  char buf[32];
  int acc = 0;
  const long long t0 = clock64();
  for (int p = 0; p < nlines; ++p) {
    const double* x = v + 12 * p;
    if (lane < 17)
      acc += mcx::fmt::fmt_field(buf, lane, 3, 1, 2, -1, 1234567ull + p, x, x + 4, x + 8) + buf[acc & 15];
  }
  const long long t1 = clock64();
  if (lane == 0) *cycles = t1 - t0;
  sink[lane] = acc;
}

int main() {
  const int n = 1 << 20;
  std::vector<double> h(n);
  std::mt19937_64 rng(7);
  std::normal_distribution<double> g;
  for (int i = 0; i < n; ++i) h[i] = (i % 100 == 0) ? g(rng) * 1e-30 : g(rng);  // 1% tiny (bigint path)
  double* dv;
  char* out;
  int *len, *sink;
  long long* cyc;
  cudaMalloc(&dv, n * 8);
  cudaMalloc(&out, (size_t)n * 32);
  cudaMalloc(&len, n * 4);
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 4);
  cudaMemcpy(dv, h.data(), n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fmt_many<<<n / 256, 256>>>(dv, n, out, len);
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) fmt_many<<<n / 256, 256>>>(dv, n, out, len);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("fmt_many: %.1f ns per value over the GPU (%.3f ms per 1M)\n", ms / 10 * 1e6 / n, ms / 10);
  for (int tiny = 0; tiny < 2; ++tiny) {
    std::vector<double> c(1000);
    for (int i = 0; i < 1000; ++i) c[i] = tiny ? g(rng) * 1e-30 : g(rng);
    cudaMemcpy(dv, c.data(), 1000 * 8, cudaMemcpyHostToDevice);
    fmt_chain<<<1, 1>>>(dv, 1000, cyc, sink);
    long long hc;
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    printf("fmt_chain (%s values): %lld cycles per value, one thread\n", tiny ? "1e-30-sized" : "O(1)", hc / 1000);
  }
  {
    std::vector<double> c(12 * 100);
    for (auto& x : c) x = g(rng);
    cudaMemcpy(dv, c.data(), c.size() * 8, cudaMemcpyHostToDevice);
    int* sk;
    cudaMalloc(&sk, 32 * 4);
    fmt_lines<<<1, 32>>>(dv, 100, cyc, sk);
    long long hc;
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    printf("fmt_lines: %lld cycles per 17-field line, one warp\n", hc / 100);
  }
  return 0;
}
