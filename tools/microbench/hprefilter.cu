// Inner-loop microbenchmark: FP64 DSETP pair test vs a conservative fp16x2
// prefilter (HSET2 + LOP3), both with B boxes from shared memory and one warp
// vote per B box, as in search_brute_kernel.  Prints pair tests / clk / SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int NB = 512, PASSES = 64;

template <int R>
__global__ void __launch_bounds__(256) k_d(const double* in, unsigned* out) {
  __shared__ double2 sb[NB][4];
  for (int i = threadIdx.x; i < NB * 4; i += blockDim.x)
    sb[i / 4][i % 4] = make_double2(in[i % 8] + 3.0 * i, in[(i + 1) % 8] - 3.0 * i);
  double alo[R][4], ahi[R][4];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) { alo[r][c] = in[c] + threadIdx.x + r; ahi[r][c] = in[8 + c] + threadIdx.x * 2 + r; }
  unsigned acc = 0;
  __syncthreads();
  for (int it = 0; it < PASSES; ++it) {
#pragma unroll 4
    for (int j = 0; j < NB; ++j) {
      const double2 l01 = sb[j][0], l23 = sb[j][1], h01 = sb[j][2], h23 = sb[j][3];
      bool any = false;
#pragma unroll
      for (int r = 0; r < R; ++r)
        any |= (l01.x <= ahi[r][0]) & (alo[r][0] <= h01.x) & (l01.y <= ahi[r][1]) & (alo[r][1] <= h01.y) &
               (l23.x <= ahi[r][2]) & (alo[r][2] <= h23.x) & (l23.y <= ahi[r][3]) & (alo[r][3] <= h23.y);
      if (__any_sync(0xffffffffu, any)) acc += j;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__device__ __forceinline__ unsigned hle(unsigned a, unsigned b) {  // 0xffff per half where a <= b
  unsigned r;
  asm("set.le.u32.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// B: L = (lo01, lo23, -hi01, -hi23) ; A: H = (hi01, hi23, -lo01, -lo23): overlap iff L_B <= H_A (8 halves)
template <int R>
__global__ void __launch_bounds__(256) k_h(const double* in, unsigned* out) {
  __shared__ uint4 sb[NB];
  for (int i = threadIdx.x; i < NB; i += blockDim.x) {
    __half2 a = __floats2half2_rn((float)(in[i % 8] + 0.01 * i), (float)(in[(i + 3) % 8] - 0.01 * i));
    uint4 v; v.x = *(unsigned*)&a; v.y = v.x ^ 0x00010001u; v.z = v.x ^ 0x80008000u; v.w = v.y ^ 0x80008000u;
    sb[i] = v;
  }
  uint4 ah[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    __half2 a = __floats2half2_rn((float)(in[r] + 0.001 * threadIdx.x), (float)(in[8 + r] - 0.002 * threadIdx.x));
    ah[r].x = *(unsigned*)&a; ah[r].y = ah[r].x ^ 0x00020002u; ah[r].z = ah[r].x ^ 0x80008000u; ah[r].w = ah[r].y ^ 0x80008000u;
  }
  unsigned acc = 0;
  __syncthreads();
  for (int it = 0; it < PASSES; ++it) {
#pragma unroll 4
    for (int j = 0; j < NB; ++j) {
      const uint4 b = sb[j];
      unsigned m = 0xffffffffu;
      bool any = false;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const unsigned x = hle(b.x, ah[r].x) & hle(b.y, ah[r].y) & hle(b.z, ah[r].z) & hle(b.w, ah[r].w);
        any |= (x == 0xffffffffu);
      }
      (void)m;
      if (__any_sync(0xffffffffu, any)) acc += j;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// Same, combining R results in one mask before a single compare (fewer ISETP).
template <int R>
__global__ void __launch_bounds__(256) k_h2(const double* in, unsigned* out) {
  __shared__ uint4 sb[NB];
  for (int i = threadIdx.x; i < NB; i += blockDim.x) {
    __half2 a = __floats2half2_rn((float)(in[i % 8] + 0.01 * i), (float)(in[(i + 3) % 8] - 0.01 * i));
    uint4 v; v.x = *(unsigned*)&a; v.y = v.x ^ 0x00010001u; v.z = v.x ^ 0x80008000u; v.w = v.y ^ 0x80008000u;
    sb[i] = v;
  }
  uint4 ah[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    __half2 a = __floats2half2_rn((float)(in[r] + 0.001 * threadIdx.x), (float)(in[8 + r] - 0.002 * threadIdx.x));
    ah[r].x = *(unsigned*)&a; ah[r].y = ah[r].x ^ 0x00020002u; ah[r].z = ah[r].x ^ 0x80008000u; ah[r].w = ah[r].y ^ 0x80008000u;
  }
  unsigned acc = 0;
  __syncthreads();
  for (int it = 0; it < PASSES; ++it) {
#pragma unroll 4
    for (int j = 0; j < NB; ++j) {
      const uint4 b = sb[j];
      unsigned orr = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        // a pair survives iff all four masks are all-ones: ~(x&y&z&w) == 0
        const unsigned x = hle(b.x, ah[r].x) & hle(b.y, ah[r].y) & hle(b.z, ah[r].z) & hle(b.w, ah[r].w);
        orr |= (~x == 0u) ? 1u : 0u;
      }
      if (__any_sync(0xffffffffu, orr != 0)) acc += j;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// Mixed: RD A boxes tested exactly in FP64 (DSETP, fp64 pipe) and RH A boxes by the
// fp16x2 conservative prefilter (HSET2 on the fma pipe + LOP3 on the alu pipe), one vote.
template <int RD, int RH, int MINB>
__global__ void __launch_bounds__(256, MINB) k_mix(const double* in, unsigned* out) {
  __shared__ double2 sb[NB][4];
  __shared__ uint4 sh[NB];
  for (int i = threadIdx.x; i < NB * 4; i += blockDim.x)
    sb[i / 4][i % 4] = make_double2(in[i % 8] + 3.0 * i, in[(i + 1) % 8] - 3.0 * i);
  for (int i = threadIdx.x; i < NB; i += blockDim.x) {
    __half2 a = __floats2half2_rn((float)(in[i % 8] + 0.01 * i), (float)(in[(i + 3) % 8] - 0.01 * i));
    uint4 v; v.x = *(unsigned*)&a; v.y = v.x ^ 0x00010001u; v.z = v.x ^ 0x80008000u; v.w = v.y ^ 0x80008000u;
    sh[i] = v;
  }
  double alo[RD][4], ahi[RD][4];
#pragma unroll
  for (int r = 0; r < RD; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) { alo[r][c] = in[c] + threadIdx.x + r; ahi[r][c] = in[8 + c] + threadIdx.x * 2 + r; }
  uint4 ah[RH];
#pragma unroll
  for (int r = 0; r < RH; ++r) {
    __half2 a = __floats2half2_rn((float)(in[r] + 0.001 * threadIdx.x), (float)(in[8 + r] - 0.002 * threadIdx.x));
    ah[r].x = *(unsigned*)&a; ah[r].y = ah[r].x ^ 0x00020002u; ah[r].z = ah[r].x ^ 0x80008000u; ah[r].w = ah[r].y ^ 0x80008000u;
  }
  unsigned acc = 0;
  __syncthreads();
  for (int it = 0; it < PASSES; ++it) {
#pragma unroll 4
    for (int j = 0; j < NB; ++j) {
      const double2 l01 = sb[j][0], l23 = sb[j][1], h01 = sb[j][2], h23 = sb[j][3];
      const uint4 b = sh[j];
      bool any = false;
#pragma unroll
      for (int r = 0; r < RD; ++r)
        any |= (l01.x <= ahi[r][0]) & (alo[r][0] <= h01.x) & (l01.y <= ahi[r][1]) & (alo[r][1] <= h01.y) &
               (l23.x <= ahi[r][2]) & (alo[r][2] <= h23.x) & (l23.y <= ahi[r][3]) & (alo[r][3] <= h23.y);
#pragma unroll
      for (int r = 0; r < RH; ++r) {
        const unsigned x = hle(b.x, ah[r].x) & hle(b.y, ah[r].y) & hle(b.z, ah[r].z) & hle(b.w, ah[r].w);
        any |= (x == 0xffffffffu);
      }
      if (__any_sync(0xffffffffu, any)) acc += j;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class K>
int run(const char* name, K k, int R, const double* d_in, unsigned* d_out, int nsm, int minb) {
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0));
  const int grid = nsm * occ * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<grid, 256>>>(d_in, d_out);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k<<<grid, 256>>>(d_in, d_out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double pairs = (double)grid * 256 * R * NB * PASSES;
  const double per_s = pairs / (best * 1e-3);
  printf("{\"kernel\": \"%s\", \"R\": %d, \"occ\": %d, \"ms\": %.3f, \"pairs_per_s\": %.4e, \"pairs_per_clk_per_sm\": %.3f}\n",
         name, R, occ, best, per_s, per_s / (nsm * clk_khz * 1e3));
  (void)minb;
  return 0;
}

__device__ __forceinline__ unsigned imad_sub(unsigned a, unsigned m1, unsigned b) {  // a - b on the fma pipe
  unsigned r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(m1), "r"(a));
  return r;
}

// Guard-bit SWAR on quantised boxes: W words per box side (W=4: two 15-bit fields per word,
// W=2: four 7-bit fields per word).  x = (H_A | G) - L_B on the fma pipe (IMAD), all guards set = pass.
template <int W, int R, int MINB>
__global__ void __launch_bounds__(256, MINB) k_swar(const double* in, unsigned* out, unsigned m1) {
  constexpr unsigned G = (W == 4) ? 0x80008000u : 0x80808080u;
  __shared__ uint4 sb[NB];
  for (int i = threadIdx.x; i < NB; i += blockDim.x) {
    unsigned v = (unsigned)(in[i % 8] * 1000.0) * 2654435761u + i * 40503u;
    sb[i] = make_uint4(v & ~G, (v * 3u) & ~G, (v * 5u) & ~G, (v * 7u) & ~G);
  }
  unsigned ah[R][W];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int w = 0; w < W; ++w) ah[r][w] = ((unsigned)(in[(r + w) % 16] * 977.0) * 2246822519u + threadIdx.x * 7919u) | G;
  unsigned acc = 0;
  __syncthreads();
  for (int it = 0; it < PASSES; ++it) {
#pragma unroll 4
    for (int j = 0; j < NB; ++j) {
      unsigned b[4];
      if (W == 4) { const uint4 t = sb[j]; b[0] = t.x; b[1] = t.y; b[2] = t.z; b[3] = t.w; }
      else { const uint2 t = reinterpret_cast<const uint2*>(sb)[j]; b[0] = t.x; b[1] = t.y; b[2] = b[3] = 0; }
      bool any = false;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (W == 4) {
          const unsigned x0 = imad_sub(ah[r][0], m1, b[0]), x1 = imad_sub(ah[r][1], m1, b[1]);
          const unsigned x2 = imad_sub(ah[r][2], m1, b[2]), x3 = imad_sub(ah[r][3], m1, b[3]);
          any |= ((x0 & x1 & x2 & x3 & G) == G);
        } else {
          const unsigned x0 = imad_sub(ah[r][0], m1, b[0]), x1 = imad_sub(ah[r][1], m1, b[1]);
          any |= ((x0 & x1 & G) == G);
        }
      }
      if (__any_sync(0xffffffffu, any)) acc += j;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class K>
int run2(const char* name, K k, int R, const double* d_in, unsigned* d_out, int nsm) {
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0));
  const int grid = nsm * occ * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<grid, 256>>>(d_in, d_out, 0xffffffffu);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k<<<grid, 256>>>(d_in, d_out, 0xffffffffu);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double pairs = (double)grid * 256 * R * NB * PASSES;
  const double per_s = pairs / (best * 1e-3);
  printf("{\"kernel\": \"%s\", \"R\": %d, \"occ\": %d, \"ms\": %.3f, \"pairs_per_s\": %.4e, \"pairs_per_clk_per_sm\": %.3f}\n",
         name, R, occ, best, per_s, per_s / (nsm * clk_khz * 1e3));
  return 0;
}

__device__ __forceinline__ unsigned alu_sub(unsigned a, unsigned b) {
  unsigned r;
  asm("sub.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// 3 instructions per pair: 2 subtractions + LOP3 with predicate output chained by AND
// (PTX lop3.and.b32 d|p).  MIX: every MIX-th pair does its second subtraction on the alu pipe.
template <int R, int MIX>
__global__ void __launch_bounds__(256, 1) k_swar3(const double* in, unsigned* out, unsigned m1) {
  constexpr unsigned G = 0x80808080u;
  __shared__ uint2 sb[NB];
  for (int i = threadIdx.x; i < NB; i += blockDim.x) {
    unsigned v = (unsigned)(in[i % 8] * 1000.0) * 2654435761u + i * 40503u;
    sb[i] = make_uint2(v & ~G, (v * 3u) & ~G);
  }
  unsigned ah[R][2];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int w = 0; w < 2; ++w) ah[r][w] = ((unsigned)(in[(r * 2 + w) % 16] * 977.0 + r) * 2246822519u + threadIdx.x * 7919u) | G;
  unsigned acc = 0;
  __syncthreads();
  for (int it = 0; it < PASSES; ++it) {
#pragma unroll 4
    for (int j = 0; j < NB; ++j) {
      const uint2 b = sb[j];
      unsigned x[2 * R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        x[2 * r] = imad_sub(ah[r][0], m1, b.x);
        x[2 * r + 1] = (MIX > 0 && r % MIX == MIX - 1) ? alu_sub(ah[r][1], b.y) : imad_sub(ah[r][1], m1, b.y);
      }
      unsigned allfail = 1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        unsigned d;
        asm("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n lop3.and.b32 %0|p, %2, %3, %4, 0x2a, p;\n selp.u32 %1, 1, 0, p;\n}"
            : "=r"(d), "+r"(allfail) : "r"(x[2 * r]), "r"(x[2 * r + 1]), "r"(G));
      }
      if (__any_sync(0xffffffffu, allfail == 0)) acc += j;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double h[16]; for (int i = 0; i < 16; ++i) h[i] = 0.1 * i - 0.7;
  double* d_in; unsigned* d_out;
  CK(cudaMalloc(&d_in, sizeof(h)));
  CK(cudaMemcpy(d_in, h, sizeof(h), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&d_out, 148 * 64 * 256 * 8 * sizeof(unsigned)));
  run("dsetp", k_d<4>, 4, d_in, d_out, nsm, 2);
  run("hset2", k_h<4>, 4, d_in, d_out, nsm, 2);
  run("hset2", k_h<8>, 8, d_in, d_out, nsm, 2);
  run("hset2_or", k_h2<4>, 4, d_in, d_out, nsm, 2);
  run("hset2_or", k_h2<8>, 8, d_in, d_out, nsm, 2);
  run("hset2_or", k_h2<16>, 16, d_in, d_out, nsm, 2);
  run("mix_d4_h4_m1", k_mix<4, 4, 1>, 8, d_in, d_out, nsm, 1);
  run("mix_d4_h4_m2", k_mix<4, 4, 2>, 8, d_in, d_out, nsm, 2);
  run("mix_d4_h2_m2", k_mix<4, 2, 2>, 6, d_in, d_out, nsm, 2);
  run("mix_d2_h4_m2", k_mix<2, 4, 2>, 6, d_in, d_out, nsm, 2);
  run("mix_d4_h8_m1", k_mix<4, 8, 1>, 12, d_in, d_out, nsm, 1);
  run("mix_d2_h2_m3", k_mix<2, 2, 3>, 4, d_in, d_out, nsm, 3);
  run("mix_d3_h3_m2", k_mix<3, 3, 2>, 6, d_in, d_out, nsm, 2);
  run("mix_d4_h6_m1", k_mix<4, 6, 1>, 10, d_in, d_out, nsm, 1);
  run("mix_d2_h6_m2", k_mix<2, 6, 2>, 8, d_in, d_out, nsm, 2);
  run("mix_d3_h4_m2", k_mix<3, 4, 2>, 7, d_in, d_out, nsm, 2);
  run2("swar15", k_swar<4, 8, 1>, 8, d_in, d_out, nsm);
  run2("swar15", k_swar<4, 4, 1>, 4, d_in, d_out, nsm);
  run2("swar7", k_swar<2, 8, 1>, 8, d_in, d_out, nsm);
  run2("swar7", k_swar<2, 16, 1>, 16, d_in, d_out, nsm);
  run2("swar7", k_swar<2, 32, 1>, 32, d_in, d_out, nsm);
  run2("swar3_mix0", k_swar3<16, 0>, 16, d_in, d_out, nsm);
  run2("swar3_mix2", k_swar3<16, 2>, 16, d_in, d_out, nsm);
  run2("swar3_mix3", k_swar3<16, 3>, 16, d_in, d_out, nsm);
  run2("swar3_mix1", k_swar3<16, 1>, 16, d_in, d_out, nsm);
  run2("swar3_r32_mix2", k_swar3<32, 2>, 32, d_in, d_out, nsm);
  return 0;
}
