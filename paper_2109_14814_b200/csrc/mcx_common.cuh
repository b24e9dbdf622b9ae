// mcx_common.cuh — shared device helpers: error state, mbarrier / bulk-copy PTX,
// and the canonical FP64 triangle-pair solve.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/mcx.h"

namespace mcx {

// ------------------------------------------------------------ geometry constants
constexpr int A_BLOCK = 1024;  // A triangles per CTA / shard block (absolute: block b = [1024 b, 1024 b + 1024))
constexpr int TILE = 512;      // B triangles per shared-memory tile (cull level-1 B unit)
constexpr int GROUP = 32;      // triangles per warp group (cull level-2 unit, both meshes)
constexpr int ORDER_TILE_Q = 16;  // tiled storage order: 16x16-quad tiles ...
constexpr int ORDER_SUB_Q = 4;    // ... of 4x4-quad sub-tiles (= one 32-triangle group)

struct __align__(16) Box {
  double lo[4];
  double hi[4];
};

// Storage position of quad (i, k) (i = θ index < N, k = column < MQ = M-1) in the
// tiled order: row-major 16x16-quad tiles, inside them row-major 4x4 sub-tiles,
// inside those row-major quads; ragged edge tiles/sub-tiles keep their true size,
// so the map is a bijection onto [0, N·MQ).  A full sub-tile is one 32-triangle
// group, a full tile one 512-triangle B tile, two adjacent tiles one A block.
__host__ __device__ __forceinline__ uint64_t storage_quad(uint32_t i, uint32_t k, uint32_t N, uint32_t MQ) {
  const uint32_t T = ORDER_TILE_Q, S = ORDER_SUB_Q;
  const uint32_t tk = k / T, ti = i / T;
  const uint32_t hq = min(T, MQ - tk * T), wq = min(T, N - ti * T);
  const uint64_t off_tile = (uint64_t)tk * T * N + (uint64_t)ti * T * hq;
  const uint32_t kk = k - tk * T, ii = i - ti * T;
  const uint32_t sk = kk / S, si = ii / S;
  const uint32_t hs = min(S, hq - sk * S), ws = min(S, wq - si * S);
  const uint32_t off_sub = sk * S * wq + si * S * hs;
  return off_tile + off_sub + (kk - sk * S) * ws + (ii - si * S);
}

// Inverse of storage_quad: storage quad index sq → (i, k).  Every tile row but the
// last holds T·N quads, every tile of a row but the last T·hq, and so on down to the
// 4×4 sub-tiles, so each level's index is a plain division by the full-size stride.
__host__ __device__ __forceinline__ void quad_of_storage(uint64_t sq, uint32_t N, uint32_t MQ, uint32_t& i,
                                                         uint32_t& k) {
  const uint32_t T = ORDER_TILE_Q, S = ORDER_SUB_Q;
  const uint32_t tk = (uint32_t)(sq / ((uint64_t)T * N));
  uint32_t r = (uint32_t)(sq - (uint64_t)tk * T * N);
  const uint32_t hq = min(T, MQ - tk * T);
  const uint32_t ti = r / (T * hq);
  r -= ti * T * hq;
  const uint32_t wq = min(T, N - ti * T);
  const uint32_t sk = r / (S * wq);
  r -= sk * S * wq;
  const uint32_t hs = min(S, hq - sk * S);
  const uint32_t si = r / (S * hs);
  r -= si * S * hs;
  const uint32_t ws = min(S, wq - si * S);
  i = ti * T + si * S + r % ws;
  k = tk * T + sk * S + r / ws;
}

// The same map in 32-bit arithmetic (every storage index is < 2^30: the triangle count
// is < 2^31) — no 64-bit division subroutine in the device code that calls it.
__device__ __forceinline__ void quad_of_storage32(uint32_t sq, uint32_t N, uint32_t MQ, uint32_t& i, uint32_t& k) {
  const uint32_t T = ORDER_TILE_Q, S = ORDER_SUB_Q;
  const uint32_t TN = N <= (0xffffffffu / T) ? T * N : 0xffffffffu;  // sq < TN whenever T·N overflows
  const uint32_t tk = sq / TN;
  uint32_t r = sq - tk * TN;
  const uint32_t hq = min(T, MQ - tk * T);
  const uint32_t ti = r / (T * hq);
  r -= ti * T * hq;
  const uint32_t wq = min(T, N - ti * T);
  const uint32_t sk = r / (S * wq);
  r -= sk * S * wq;
  const uint32_t hs = min(S, hq - sk * S);
  const uint32_t si = r / (S * hs);
  r -= si * S * hs;
  const uint32_t ws = min(S, wq - si * S);
  i = ti * T + si * S + r % ws;
  k = tk * T + sk * S + r / ws;
}

// ------------------------------------------------------------ error state
// Thread-local, so concurrent host threads (one per GPU) never clobber each other.
extern thread_local char g_err[512];

inline int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

// Saves the calling thread's current device and restores it on scope exit, so no
// entry point leaves the caller's device switched (include/mcx.h conventions).
struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  DeviceGuard() { ok = cudaGetDevice(&prev) == cudaSuccess; }
  ~DeviceGuard() {
    int cur = -1;
    if (ok && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return ::mcx::set_error(MCX_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,          \
                              cudaGetErrorString(_e));                                        \
  } while (0)

// Pinned host staging for the small table uploads of a search.  A pageable source
// makes cudaMemcpyAsync stage the copy and wait for the stream's earlier work, which
// serialises the host with the GPU on a latency-critical path; the host runtime
// (mcx_runtime.cu) installs a context-owned pinned buffer for the duration of a call.
struct HostStage {
  char* p = nullptr;
  size_t cap = 0, used = 0;
};
extern thread_local HostStage* g_stage;

struct StageScope {
  HostStage* prev;
  explicit StageScope(HostStage* s) : prev(g_stage) {
    if (s) s->used = 0;
    g_stage = s;
  }
  ~StageScope() { g_stage = prev; }
};

inline cudaError_t h2d_async(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  HostStage* st = g_stage;
  if (st && st->p && st->used + bytes <= st->cap) {
    char* q = st->p + st->used;
    memcpy(q, src, bytes);
    st->used += (bytes + 15) & ~(size_t)15;
    return cudaMemcpyAsync(dst, q, bytes, cudaMemcpyHostToDevice, s);
  }
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
}

// ------------------------------------------------------- mbarrier + bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred done;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      " @!done bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk async copy global → shared (SASS: UBLKCP), completion on `bar`.
// bytes must be a multiple of 16 and both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Non-coherent 16-byte load that the compiler cannot CSE (used to rematerialise
// register-resident data instead of keeping it live across a rare slow path).
__device__ __forceinline__ void ld_nc_v2(const double* p, double& x, double& y) {
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "l"(p));
}

// ------------------------------------------------------- canonical FP64 solve
// FMA-free, fixed association order; see oracle/canonical.py:pack / solve_pairs.
#define MCX_SING_RTOL 1e-12

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// Vertex addressing of original triangle t for the solve.  The solve reads vertices
// through non-CSE-able loads and re-derives an edge each time it needs one: the
// values (and bits) are those of the packing, v + 0.0 then v1 − v0, while the live
// register set stays small enough for the hot loops around it.
struct TriRef {
  const double* c;
  uint32_t plane, o[3];  // plane stride; offsets of v0, v1, v2 within a plane (N·M < 2^32)
};

// Mp = rows between the x, y, px, py planes (M, or the parent grid's M for a column view).
__device__ __forceinline__ TriRef tri_ref(const double* c, uint32_t N, uint32_t Mp, uint32_t t) {
  const uint32_t q = t >> 1, tau = t & 1;
  const uint32_t i = q % N, k = q / N;
  const uint32_t ip = (i + 1 == N) ? 0 : i + 1;
  const uint32_t r0 = k * N, r1 = r0 + N;
  TriRef T;
  T.c = c;
  T.plane = Mp * N;
  T.o[0] = (tau ? r1 : r0) + i;
  T.o[1] = r0 + ip;
  T.o[2] = r1 + (tau ? ip : i);
  return T;
}

__device__ __forceinline__ double ld_vol(const double* p) {
  double x;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(x) : "l"(p));
  return x;
}

__device__ __forceinline__ double vert(const TriRef& T, int v, int d) {
  return dadd(ld_vol(T.c + ((uint64_t)d * T.plane + T.o[v])), 0.0);
}

// e = v_which − v0 (which = 1: e1, 2: e2), the packing's edge.
__device__ __forceinline__ void edge(const TriRef& T, int which, double e[4]) {
#pragma unroll
  for (int d = 0; d < 4; ++d) e[d] = dsub(vert(T, which, d), vert(T, 0, d));
}

// P = e1∧e2 (order 01, 02, 03, 12, 13, 23) and nrm = ‖e1‖·‖e2‖, left-to-right sums.
__device__ __forceinline__ void biv_norm(const TriRef& T, double P[6], double& nrm) {
  double e1[4], e2[4];
  edge(T, 1, e1);
  edge(T, 2, e2);
  const int bi[6] = {0, 0, 0, 1, 1, 2}, bj[6] = {1, 2, 3, 2, 3, 3};
#pragma unroll
  for (int p = 0; p < 6; ++p) P[p] = dsub(dmul(e1[bi[p]], e2[bj[p]]), dmul(e1[bj[p]], e2[bi[p]]));
  double n1 = dmul(e1[0], e1[0]), n2 = dmul(e2[0], e2[0]);
#pragma unroll
  for (int d = 1; d < 4; ++d) {
    n1 = dadd(n1, dmul(e1[d], e1[d]));
    n2 = dadd(n2, dmul(e2[d], e2[d]));
  }
  nrm = dmul(__dsqrt_rn(n1), __dsqrt_rn(n2));
}

// g_j = Σ_i r_i K_ij for the antisymmetric K of bivector B (order 01,02,03,12,13,23)
__device__ __forceinline__ void contract(const double r[4], const double B[6], double c[4]) {
  c[0] = dsub(dsub(dmul(r[2], B[4]), dmul(r[1], B[5])), dmul(r[3], B[3]));
  c[1] = dadd(dsub(dmul(r[0], B[5]), dmul(r[2], B[2])), dmul(r[3], B[1]));
  c[2] = dsub(dsub(dmul(r[1], B[2]), dmul(r[0], B[4])), dmul(r[3], B[0]));
  c[3] = dadd(dsub(dmul(r[0], B[3]), dmul(r[1], B[1])), dmul(r[2], B[0]));
}

__device__ __forceinline__ double dot4(const double c[4], const double x[4]) {
  double d = dmul(c[0], x[0]);
  d = dadd(d, dmul(c[1], x[1]));
  d = dadd(d, dmul(c[2], x[2]));
  d = dadd(d, dmul(c[3], x[3]));
  return d;
}

// The precise test of original triangles ta of grid A and tb of
// grid B (MpA / MpB: their plane strides in rows, see tri_ref).  Returns 0 = miss, 1 = hit (sol = s, t, a, b), 2 = singular (gate,
// SPEC.md:464).  Only AABB survivors get here (1e-7..1e-3 of the pairs), so the
// triangle geometry is rebuilt from the grids (L1/L2) instead of being stored.
__device__ __forceinline__ int solve_tri(const double* __restrict__ cA, uint32_t NA, uint32_t MpA, uint32_t ta,
                                         const double* __restrict__ cB, uint32_t NB, uint32_t MpB, uint32_t tb,
                                         double sol[4]) {
  const TriRef A = tri_ref(cA, NA, MpA, ta), B = tri_ref(cB, NB, MpB, tb);
  double Pa[6], Qb[6], nA, nB;
  biv_norm(A, Pa, nA);
  biv_norm(B, Qb, nB);
  double r[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) r[c] = dsub(vert(B, 0, c), vert(A, 0, c));
  double D = dsub(dmul(Pa[0], Qb[5]), dmul(Pa[1], Qb[4]));
  D = dadd(D, dmul(Pa[2], Qb[3]));
  D = dadd(D, dmul(Pa[3], Qb[2]));
  D = dsub(D, dmul(Pa[4], Qb[1]));
  D = dadd(D, dmul(Pa[5], Qb[0]));
  const double thr = dmul(dmul(nA, nB), MCX_SING_RTOL);
  if (fabs(D) <= thr) return 2;
  double g[4], h[4], x[4];
  contract(r, Qb, g);
  contract(r, Pa, h);
  edge(A, 2, x);
  const double s = __ddiv_rn(dot4(g, x), D);
  edge(A, 1, x);
  const double t = __ddiv_rn(-dot4(g, x), D);
  edge(B, 2, x);
  const double a = __ddiv_rn(-dot4(h, x), D);
  edge(B, 1, x);
  const double b = __ddiv_rn(dot4(h, x), D);
  if (s >= 0.0 && t >= 0.0 && a >= 0.0 && b >= 0.0 && dadd(s, t) <= 1.0 && dadd(a, b) <= 1.0) {
    sol[0] = s;
    sol[1] = t;
    sol[2] = a;
    sol[3] = b;
    return 1;
  }
  return 0;
}

// ------------------------------------------- SPEC-literal Moller quick test
// Mirrors oracle/serial.py (_plane/_side_reject) op for op.  Quad q = i + N·k1 of a
// (4, M, N) grid; vertices v00 v10 v01 v11; projection (x, y, px).
#define MCX_DEGEN_RTOL2 1e-28

__device__ __forceinline__ void quad_verts(const double* __restrict__ c, uint32_t N, uint32_t Mp, uint32_t q,
                                           double V[4][3]) {
  const uint32_t i = q % N, k = q / N;
  const uint32_t ip = (i + 1 == N) ? 0 : i + 1;
  const uint64_t idx[4] = {(uint64_t)k * N + i, (uint64_t)k * N + ip, (uint64_t)(k + 1) * N + i,
                           (uint64_t)(k + 1) * N + ip};
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int d = 0; d < 3; ++d) V[v][d] = __ldg(c + (uint64_t)d * Mp * N + idx[v]);
}

// All four Vo vertices strictly on one side of the plane of T¹(Vq) and of T²(Vq).
__device__ __forceinline__ bool side_reject(const double Vq[4][3], const double Vo[4][3]) {
  const int tri[2][3] = {{0, 1, 2}, {2, 1, 3}};
  bool out = true;
#pragma unroll
  for (int T = 0; T < 2; ++T) {
    const double* O = Vq[tri[T][0]];
    double U[3], W[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      U[d] = dsub(Vq[tri[T][1]][d], O[d]);
      W[d] = dsub(Vq[tri[T][2]][d], O[d]);
    }
    const double N0 = dsub(dmul(U[1], W[2]), dmul(U[2], W[1]));
    const double N1 = dsub(dmul(U[2], W[0]), dmul(U[0], W[2]));
    const double N2 = dsub(dmul(U[0], W[1]), dmul(U[1], W[0]));
    const double nn = dadd(dadd(dmul(N0, N0), dmul(N1, N1)), dmul(N2, N2));
    const double uu = dadd(dadd(dmul(U[0], U[0]), dmul(U[1], U[1])), dmul(U[2], U[2]));
    const double ww = dadd(dadd(dmul(W[0], W[0]), dmul(W[1], W[1])), dmul(W[2], W[2]));
    const bool degen = nn < dmul(dmul(uu, ww), MCX_DEGEN_RTOL2);
    bool pos = true, neg = true;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double f = dadd(dadd(dmul(N0, dsub(Vo[m][0], O[0])), dmul(N1, dsub(Vo[m][1], O[1]))),
                            dmul(N2, dsub(Vo[m][2], O[2])));
      pos = pos && (f > 0.0);
      neg = neg && (f < 0.0);
    }
    out = out && !degen && (pos || neg);
  }
  return out;
}

__device__ __forceinline__ bool moller_reject(const double* cA, uint32_t NA, uint32_t MpA, uint32_t qa,
                                              const double* cB, uint32_t NB, uint32_t MpB, uint32_t qb) {
  double VA[4][3], VB[4][3];
  quad_verts(cA, NA, MpA, qa, VA);
  quad_verts(cB, NB, MpB, qb, VB);
  return side_reject(VA, VB) || side_reject(VB, VA);
}

}  // namespace mcx
