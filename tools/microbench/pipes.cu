// Pipe-throughput microbenchmark for the compare-bound pair-test kernel.
//
// Measures, in lane-ops per SM-cycle (clock64 inside the kernel, all CTAs
// co-resident), the issue rate of the instructions a triangle-AABB test can be
// built from on sm_100a:
//   dfma   : DFMA            (the FP64 FLOP peak denominator)
//   dsetp  : DSETP.*.AND     (8 per triangle pair in the FP64 AABB test)
//   fsetp  : FSETP.*.AND     (FP32 conservative prefilter candidate)
//   hsetp2 : HSETP2.*.AND    (2 fp16 compares per lane-op)
//   iswar  : IADD3 + LOP3    (guard-bit SWAR compare on packed 15-bit fields)
// Output: one JSON line per op.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_dfma(const double* in, void* outv, long long* cyc) {
  double* out = (double*)outv;
  double a0 = in[threadIdx.x & 7], a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = in[8], c = in[9];
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// 4 independent chains of 8 predicate-ANDed FP64 compares per asm block.
__global__ void k_dsetp(const double* in, void* outv, long long* cyc) {
  unsigned* out = (unsigned*)outv;
  double x[8], y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { x[k] = in[k]; y[k] = in[8 + k] + threadIdx.x; }
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    unsigned r0, r1, r2, r3;
    asm volatile(
        "{\n .reg .pred p0, p1, p2, p3;\n"
        " setp.le.f64 p0, %4, %12;\n setp.le.f64 p1, %5, %13;\n setp.le.f64 p2, %6, %14;\n setp.le.f64 p3, %7, %15;\n"
        " setp.le.and.f64 p0, %5, %13, p0;\n setp.le.and.f64 p1, %6, %14, p1;\n setp.le.and.f64 p2, %7, %15, p2;\n setp.le.and.f64 p3, %8, %16, p3;\n"
        " setp.le.and.f64 p0, %6, %14, p0;\n setp.le.and.f64 p1, %7, %15, p1;\n setp.le.and.f64 p2, %8, %16, p2;\n setp.le.and.f64 p3, %9, %17, p3;\n"
        " setp.le.and.f64 p0, %7, %15, p0;\n setp.le.and.f64 p1, %8, %16, p1;\n setp.le.and.f64 p2, %9, %17, p2;\n setp.le.and.f64 p3, %10, %18, p3;\n"
        " setp.le.and.f64 p0, %8, %16, p0;\n setp.le.and.f64 p1, %9, %17, p1;\n setp.le.and.f64 p2, %10, %18, p2;\n setp.le.and.f64 p3, %11, %19, p3;\n"
        " setp.le.and.f64 p0, %9, %17, p0;\n setp.le.and.f64 p1, %10, %18, p1;\n setp.le.and.f64 p2, %11, %19, p2;\n setp.le.and.f64 p3, %4, %12, p3;\n"
        " setp.le.and.f64 p0, %10, %18, p0;\n setp.le.and.f64 p1, %11, %19, p1;\n setp.le.and.f64 p2, %4, %12, p2;\n setp.le.and.f64 p3, %5, %13, p3;\n"
        " setp.le.and.f64 p0, %11, %19, p0;\n setp.le.and.f64 p1, %4, %12, p1;\n setp.le.and.f64 p2, %5, %13, p2;\n setp.le.and.f64 p3, %6, %14, p3;\n"
        " selp.u32 %0, 1, 0, p0;\n selp.u32 %1, 1, 0, p1;\n selp.u32 %2, 1, 0, p2;\n selp.u32 %3, 1, 0, p3;\n}\n"
        : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
        : "d"(x[0]), "d"(x[1]), "d"(x[2]), "d"(x[3]), "d"(x[4]), "d"(x[5]), "d"(x[6]), "d"(x[7]),
          "d"(y[0]), "d"(y[1]), "d"(y[2]), "d"(y[3]), "d"(y[4]), "d"(y[5]), "d"(y[6]), "d"(y[7]));
    acc += r0 + r1 + r2 + r3;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_fsetp(const float* in, void* outv, long long* cyc) {
  unsigned* out = (unsigned*)outv;
  float x[8], y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { x[k] = in[k]; y[k] = in[8 + k] + threadIdx.x; }
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    unsigned r0, r1, r2, r3;
    asm volatile(
        "{\n .reg .pred p0, p1, p2, p3;\n"
        " setp.le.f32 p0, %4, %12;\n setp.le.f32 p1, %5, %13;\n setp.le.f32 p2, %6, %14;\n setp.le.f32 p3, %7, %15;\n"
        " setp.le.and.f32 p0, %5, %13, p0;\n setp.le.and.f32 p1, %6, %14, p1;\n setp.le.and.f32 p2, %7, %15, p2;\n setp.le.and.f32 p3, %8, %16, p3;\n"
        " setp.le.and.f32 p0, %6, %14, p0;\n setp.le.and.f32 p1, %7, %15, p1;\n setp.le.and.f32 p2, %8, %16, p2;\n setp.le.and.f32 p3, %9, %17, p3;\n"
        " setp.le.and.f32 p0, %7, %15, p0;\n setp.le.and.f32 p1, %8, %16, p1;\n setp.le.and.f32 p2, %9, %17, p2;\n setp.le.and.f32 p3, %10, %18, p3;\n"
        " setp.le.and.f32 p0, %8, %16, p0;\n setp.le.and.f32 p1, %9, %17, p1;\n setp.le.and.f32 p2, %10, %18, p2;\n setp.le.and.f32 p3, %11, %19, p3;\n"
        " setp.le.and.f32 p0, %9, %17, p0;\n setp.le.and.f32 p1, %10, %18, p1;\n setp.le.and.f32 p2, %11, %19, p2;\n setp.le.and.f32 p3, %4, %12, p3;\n"
        " setp.le.and.f32 p0, %10, %18, p0;\n setp.le.and.f32 p1, %11, %19, p1;\n setp.le.and.f32 p2, %4, %12, p2;\n setp.le.and.f32 p3, %5, %13, p3;\n"
        " setp.le.and.f32 p0, %11, %19, p0;\n setp.le.and.f32 p1, %4, %12, p1;\n setp.le.and.f32 p2, %5, %13, p2;\n setp.le.and.f32 p3, %6, %14, p3;\n"
        " selp.u32 %0, 1, 0, p0;\n selp.u32 %1, 1, 0, p1;\n selp.u32 %2, 1, 0, p2;\n selp.u32 %3, 1, 0, p3;\n}\n"
        : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
        : "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]), "f"(x[7]),
          "f"(y[0]), "f"(y[1]), "f"(y[2]), "f"(y[3]), "f"(y[4]), "f"(y[5]), "f"(y[6]), "f"(y[7]));
    acc += r0 + r1 + r2 + r3;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// f16x2: setp.le.and.f16x2 gives two predicates (one per half); 4 chains x 4 ops.
__global__ void k_hsetp2(const unsigned* in, void* outv, long long* cyc) {
  unsigned* out = (unsigned*)outv;
  unsigned x[4], y[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { x[k] = in[k]; y[k] = in[4 + k] ^ (threadIdx.x & 1); }
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    unsigned r0, r1, r2, r3;
    asm volatile(
        "{\n .reg .pred p0, q0, p1, q1, p2, q2, p3, q3;\n"
        " setp.le.f16x2 p0|q0, %4, %8;\n setp.le.f16x2 p1|q1, %5, %9;\n setp.le.f16x2 p2|q2, %6, %10;\n setp.le.f16x2 p3|q3, %7, %11;\n"
        " setp.le.and.f16x2 p0|q0, %5, %9, p0;\n setp.le.and.f16x2 p1|q1, %6, %10, p1;\n setp.le.and.f16x2 p2|q2, %7, %11, p2;\n setp.le.and.f16x2 p3|q3, %4, %8, p3;\n"
        " setp.le.and.f16x2 p0|q0, %6, %10, q0;\n setp.le.and.f16x2 p1|q1, %7, %11, q1;\n setp.le.and.f16x2 p2|q2, %4, %8, q2;\n setp.le.and.f16x2 p3|q3, %5, %9, q3;\n"
        " setp.le.and.f16x2 p0|q0, %7, %11, p0;\n setp.le.and.f16x2 p1|q1, %4, %8, p1;\n setp.le.and.f16x2 p2|q2, %5, %9, p2;\n setp.le.and.f16x2 p3|q3, %6, %10, p3;\n"
        " and.pred p0, p0, q0;\n and.pred p1, p1, q1;\n and.pred p2, p2, q2;\n and.pred p3, p3, q3;\n"
        " selp.u32 %0, 1, 0, p0;\n selp.u32 %1, 1, 0, p1;\n selp.u32 %2, 1, 0, p2;\n selp.u32 %3, 1, 0, p3;\n}\n"
        : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
        : "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]));
    acc += r0 + r1 + r2 + r3;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// Guard-bit SWAR: per pair, 4 words of two 15-bit fields: x = (A|G) - B, and = x0&x1&x2, and2 = t&x3&G.
__global__ void k_iswar(const unsigned* in, void* outv, long long* cyc) {
  unsigned* out = (unsigned*)outv;
  unsigned a[4][4], b[4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int k = 0; k < 4; ++k) a[r][k] = in[r * 4 + k] | 0x80008000u;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = in[16 + k] + threadIdx.x;
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      unsigned x0, x1, x2, x3, t;
      asm volatile("sub.u32 %0, %1, %2;" : "=r"(x0) : "r"(a[r][0]), "r"(b[0]));
      asm volatile("sub.u32 %0, %1, %2;" : "=r"(x1) : "r"(a[r][1]), "r"(b[1]));
      asm volatile("sub.u32 %0, %1, %2;" : "=r"(x2) : "r"(a[r][2]), "r"(b[2]));
      asm volatile("sub.u32 %0, %1, %2;" : "=r"(x3) : "r"(a[r][3]), "r"(b[3]));
      asm volatile("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(t) : "r"(x0), "r"(x1), "r"(x2));
      asm volatile("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(t) : "r"(t), "r"(x3), "r"(0x80008000u));
      acc += t;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) b[k] += 1;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}


// DSETP with B operands loaded from shared memory every iteration (like the search
// inner loop): 4 LDS.128 + 4 chains x 8 DSETP per iteration.  Measures the DSETP
// issue rate when ptxas cannot hoist the compares.
__global__ void k_dsetp_smem(const double* in, void* outv, long long* cyc) {
  unsigned* out = (unsigned*)outv;
  __shared__ double2 sb[512][4];
  for (int i = threadIdx.x; i < 512 * 4; i += blockDim.x) sb[i / 4][i % 4] = make_double2(in[i % 8] + i, in[(i + 1) % 8] - i);
  double alo[4][4], ahi[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) { alo[r][c] = in[c] + threadIdx.x + r; ahi[r][c] = in[8 + c] + threadIdx.x * 2 + r; }
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 512 * 8; ++it) {
#pragma unroll 2
    for (int j = 0; j < 512; ++j) {
      const double2 l01 = sb[j][0], l23 = sb[j][1], h01 = sb[j][2], h23 = sb[j][3];
      bool p[4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        p[r] = (l01.x <= ahi[r][0]) & (alo[r][0] <= h01.x) & (l01.y <= ahi[r][1]) & (alo[r][1] <= h01.y) &
               (l23.x <= ahi[r][2]) & (alo[r][2] <= h23.x) & (l23.y <= ahi[r][3]) & (alo[r][3] <= h23.y);
      acc += (p[0] | p[1] | p[2] | p[3]) ? 1u : 0u;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}


// FSETP with B operands from shared memory each iteration: 2 LDS.128 (8 floats) +
// R chains x 8 FSETP — the FP32 conservative-prefilter variant of the inner loop.
template <int R>
__global__ void k_fsetp_smem(const double* in, void* outv, long long* cyc) {
  unsigned* out = (unsigned*)outv;
  __shared__ float4 sb[512][2];
  for (int i = threadIdx.x; i < 512 * 2; i += blockDim.x)
    sb[i / 2][i % 2] = make_float4(in[i % 8] + i, in[(i + 1) % 8] - i, in[(i + 2) % 8] + 0.5f * i, in[(i + 3) % 8]);
  float alo[R][4], ahi[R][4];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) { alo[r][c] = in[c] + threadIdx.x + r; ahi[r][c] = in[8 + c] + threadIdx.x * 2 + r; }
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 512 * 8; ++it) {
#pragma unroll 4
    for (int j = 0; j < 512; ++j) {
      const float4 l = sb[j][0], h = sb[j][1];
      bool any = false;
#pragma unroll
      for (int r = 0; r < R; ++r)
        any |= (l.x <= ahi[r][0]) & (alo[r][0] <= h.x) & (l.y <= ahi[r][1]) & (alo[r][1] <= h.y) &
               (l.z <= ahi[r][2]) & (alo[r][2] <= h.z) & (l.w <= ahi[r][3]) & (alo[r][3] <= h.w);
      acc += __any_sync(0xffffffffu, any) ? 1u : 0u;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}


// Mixed-pipe pair test: 4 DSETP (B.lo <= A.hi, FP64 pipe) + 4 FSETP (A.lo_rd <= B.hi_ru,
// ALU pipe) per pair; B record = lo[4] double + hi[4] float (48 B = 3 LDS.128).
template <int R>
__global__ void k_mixed_smem(const double* in, void* outv, long long* cyc) {
  unsigned* out = (unsigned*)outv;
  struct __align__(16) MB { double lo[4]; float hi[4]; };
  __shared__ MB sb[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) {
    for (int c = 0; c < 4; ++c) { sb[i].lo[c] = in[c] + i * 1e-3; sb[i].hi[c] = (float)(in[4 + c] - i * 1e-3); }
  }
  double ahi[R][4];
  float alo[R][4];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) { alo[r][c] = in[c] + threadIdx.x + r; ahi[r][c] = in[8 + c] + threadIdx.x * 2 + r; }
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 512 * 8; ++it) {
#pragma unroll 4
    for (int j = 0; j < 512; ++j) {
      const double2 l01 = *reinterpret_cast<const double2*>(&sb[j].lo[0]);
      const double2 l23 = *reinterpret_cast<const double2*>(&sb[j].lo[2]);
      const float4 h = *reinterpret_cast<const float4*>(&sb[j].hi[0]);
      bool any = false;
#pragma unroll
      for (int r = 0; r < R; ++r)
        any |= (l01.x <= ahi[r][0]) & (alo[r][0] <= h.x) & (l01.y <= ahi[r][1]) & (alo[r][1] <= h.y) &
               (l23.x <= ahi[r][2]) & (alo[r][2] <= h.z) & (l23.y <= ahi[r][3]) & (alo[r][3] <= h.w);
      acc += __any_sync(0xffffffffu, any) ? 1u : 0u;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}


// Mixed-pipe with ND FP64 compares (DSETP) + (8-ND) FP32 conservative compares (FSETP)
// per pair.  B record: 4 doubles (lo) + 4 floats (hi) as before; the first ND compares
// use doubles (4 lo-vs-hi + (ND-4) hi-vs-lo on doubles held in A registers).
template <int R, int ND>
__global__ void k_mixed2_smem(const double* in, void* outv, long long* cyc) {
  unsigned* out = (unsigned*)outv;
  struct __align__(16) MB { double lo[4]; double hi[2]; float hif[2]; float pad[2]; };
  __shared__ MB sb[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) {
    for (int c = 0; c < 4; ++c) sb[i].lo[c] = in[c] + i * 1e-3;
    for (int c = 0; c < 2; ++c) { sb[i].hi[c] = in[4 + c] - i * 1e-3; sb[i].hif[c] = (float)(in[6 + c] - i * 1e-3); }
  }
  double ahi[R][4], alod[R][2];
  float alof[R][2];
#pragma unroll
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int c = 0; c < 4; ++c) ahi[r][c] = in[8 + c] + threadIdx.x * 2 + r;
#pragma unroll
    for (int c = 0; c < 2; ++c) { alod[r][c] = in[c] + threadIdx.x + r; alof[r][c] = (float)(in[2 + c] + threadIdx.x + r); }
  }
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 512 * 8; ++it) {
#pragma unroll 4
    for (int j = 0; j < 512; ++j) {
      const double2 l01 = *reinterpret_cast<const double2*>(&sb[j].lo[0]);
      const double2 l23 = *reinterpret_cast<const double2*>(&sb[j].lo[2]);
      const double2 h01 = *reinterpret_cast<const double2*>(&sb[j].hi[0]);
      const float2 h23 = *reinterpret_cast<const float2*>(&sb[j].hif[0]);
      bool any = false;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        bool p = (l01.x <= ahi[r][0]) & (l01.y <= ahi[r][1]) & (l23.x <= ahi[r][2]) & (l23.y <= ahi[r][3]);
        if (ND >= 6) p = p & (alod[r][0] <= h01.x) & (alod[r][1] <= h01.y);
        else { p = p & ((float)alod[r][0] <= (float)h01.x) & ((float)alod[r][1] <= (float)h01.y); }
        p = p & (alof[r][0] <= h23.x) & (alof[r][1] <= h23.y);
        any |= p;
      }
      acc += __any_sync(0xffffffffu, any) ? 1u : 0u;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// DFMA with loop-carried dependence through 8 accumulators AND an smem operand.
__global__ void k_dadd_chain(const double* in, void* outv, long long* cyc) {
  double* out = (double*)outv;
  double a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = in[k % 8] + threadIdx.x + k;
  const double b = in[8];
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = a[k] + b;
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = a[k] - b;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0; for (int k = 0; k < 16; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K, typename T>
static int run(const char* name, K kern, const T* din, void* dout, long long* dcyc, int nsm, int threads,
               double lane_ops_per_thread, int repeats) {
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0));
  int grid = nsm * occ;
  long long* hcyc = new long long[grid];
  double best = 0, best_ms = 0;
  for (int rep = 0; rep < repeats; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<grid, threads>>>(din, dout, dcyc);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(hcyc, dcyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost));
    double mean = 0;
    for (int i = 0; i < grid; ++i) mean += hcyc[i];
    mean /= grid;
    double per_sm_clk = occ * threads * lane_ops_per_thread / mean;
    if (per_sm_clk > best) { best = per_sm_clk; best_ms = ms; }
  }
  double clk_ghz = 0;
  {
    // implied clock = cycles / elapsed
    double mean = 0; for (int i = 0; i < grid; ++i) mean += hcyc[i]; mean /= grid;
    clk_ghz = mean / (best_ms * 1e6);
  }
  double total = (double)grid * threads * lane_ops_per_thread;
  printf("{\"op\": \"%s\", \"lane_ops_per_clk_per_sm_clock64\": %.3f, \"lane_ops_per_s\": %.4e, \"per_sm_per_clk_at_1965\": %.2f, \"occ\": %d, \"threads\": %d, \"ms\": %.3f, \"implied_ghz\": %.3f}\n",
         name, best, total / (best_ms * 1e-3), total / (best_ms * 1e-3) / nsm / 1.965e9, occ, threads, best_ms, clk_ghz);
  delete[] hcyc;
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0, l2 = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"clock_khz\": %d, \"l2_bytes\": %d, \"smem_per_block_optin\": %zu, \"regs_per_sm\": %d}\n",
         p.name, p.multiProcessorCount, p.major, p.minor, clk_khz, l2, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  int nsm = p.multiProcessorCount;
  double* dd; float* df; unsigned* du; void* dout; long long* dcyc;
  double hd[16]; float hf[16]; unsigned hu[32];
  for (int i = 0; i < 16; ++i) { hd[i] = 0.5 + i; hf[i] = 0.5f + i; }
  for (int i = 0; i < 32; ++i) hu[i] = 0x3c003c00u + i;
  CK(cudaMalloc(&dd, sizeof(hd))); CK(cudaMalloc(&df, sizeof(hf))); CK(cudaMalloc(&du, sizeof(hu)));
  CK(cudaMalloc(&dout, 64 << 20)); CK(cudaMalloc(&dcyc, 1 << 20));
  CK(cudaMemcpy(dd, hd, sizeof(hd), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(df, hf, sizeof(hf), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(du, hu, sizeof(hu), cudaMemcpyHostToDevice));
  for (int threads : {256, 512}) {
    run("dsetp_smem", k_dsetp_smem, dd, dout, dcyc, nsm, threads, 32.0 * (ITERS / 512 * 8) * 512, 3);
    run("dadd", k_dadd_chain, dd, dout, dcyc, nsm, threads, 32.0 * ITERS, 3);
    run("fsetp_smem_r4", k_fsetp_smem<4>, dd, dout, dcyc, nsm, threads, 32.0 * (ITERS / 512 * 8) * 512, 3);
    run("mixed_smem_r4", k_mixed_smem<4>, dd, dout, dcyc, nsm, threads, 32.0 * (ITERS / 512 * 8) * 512, 3);
    run("mixed2_r4_6d2f", k_mixed2_smem<4, 6>, dd, dout, dcyc, nsm, threads, 32.0 * (ITERS / 512 * 8) * 512, 3);
    run("mixed2_r5_6d2f", k_mixed2_smem<5, 6>, dd, dout, dcyc, nsm, threads, 40.0 * (ITERS / 512 * 8) * 512, 3);
    run("mixed_smem_r6", k_mixed_smem<6>, dd, dout, dcyc, nsm, threads, 48.0 * (ITERS / 512 * 8) * 512, 3);
    run("mixed_smem_r8", k_mixed_smem<8>, dd, dout, dcyc, nsm, threads, 64.0 * (ITERS / 512 * 8) * 512, 3);
    run("fsetp_smem_r8", k_fsetp_smem<8>, dd, dout, dcyc, nsm, threads, 64.0 * (ITERS / 512 * 8) * 512, 3);
    run("dfma", k_dfma, dd, dout, dcyc, nsm, threads, 32.0 * ITERS, 3);
    run("dsetp", k_dsetp, dd, dout, dcyc, nsm, threads, 32.0 * ITERS, 3);
    run("fsetp", k_fsetp, df, dout, dcyc, nsm, threads, 32.0 * ITERS, 3);
    run("hsetp2", k_hsetp2, du, dout, dcyc, nsm, threads, 16.0 * ITERS, 3);
    run("iswar_alu", k_iswar, du, dout, dcyc, nsm, threads, 24.0 * ITERS, 3);
  }
  return 0;
}
