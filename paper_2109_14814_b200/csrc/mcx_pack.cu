// mcx_pack.cu — canonical triangle boxes and the culling hierarchy in one pass (libmcx.so).
//
// pack_kernel: persistent CTAs, each walking 1024-record blocks of the storage order
// (blk0 + blockIdx.x, step gridDim.x), one thread per storage quad of a block.  The
// thread inverts the storage map to its quad (i, k) of the (4, M, N) half-layer grid,
// builds T¹ = {v00, v10, v01} and T² = {v10, v01, v11} with θ wrapping mod N
// (PAPER.md T^{u1}/T^{u2} vertex sets) and writes their exact AABBs.
// Original triangle index t = 2·(i + N·k) + τ (PAPER.md kernel step 3); perm[] maps
// storage position → t so searches can emit original indices.
//
// Input: a block of two full 16×16-quad tiles reads a 17 × 33-vertex window of each of
// the 4 planes.  The window of the NEXT block is copied into shared memory (cp.async,
// no registers) while the current one is computed and written, so the grid reads
// overlap the stores and each vertex is read from HBM/L2 once instead of by 4 quads.
// Ragged edge blocks (partial tiles) load their vertices directly.
//
// Output is destination-ordered: the block's 1024 boxes (64 KB) are staged in shared
// memory and leave as fully coalesced 16-byte stores (consecutive threads, consecutive
// 16 B), perm with coalesced 8-byte stores, and the level boxes of the block come from
// the same registers: 16 quads (a half warp) = one 32-record group (shuffles), 8 warps
// = one 512-record tile, the CTA = one 1024-record block.  (A single cp.async.bulk
// shared → global copy measured the same and is invisible to compute-sanitizer's
// initcheck, which then flags every later read of the boxes.)  A union box is disjoint from
// another box only if every member is, so culling never changes the hit set.
//
// Per record: 16 B of grid read, 64 B box + 4 B perm + 2.2 B of level boxes written —
// HBM-bound.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/mcx.h"
#include "mcx_common.cuh"
#include "mcx_internal.cuh"

namespace mcx {

constexpr int PACK_THREADS = A_BLOCK / 2;  // one thread per storage quad of a block

// The grid window of a block of two full tiles: 17 vertex rows × 33 vertex columns per
// plane, rows padded to 36 doubles (≡ 4 mod 16, so the 4×4-quad sub-tile a half-warp
// reads covers 16 distinct bank pairs).
constexpr int WIN_ROWS = ORDER_TILE_Q + 1;
constexpr int WIN_COLS = 2 * ORDER_TILE_Q + 1;
constexpr int WIN_STRIDE = 36;
constexpr int WIN_PLANE = WIN_ROWS * WIN_STRIDE;
constexpr int WIN_LOADS = 4 * WIN_ROWS * WIN_COLS;

// 16-byte slot q of the staged boxes lives at q with its column (q mod 8) XORed by its
// 128-byte row (q / 8) mod 8
__device__ __forceinline__ uint32_t swz(uint32_t q) { return q ^ ((q >> 3) & 7); }
__device__ __forceinline__ unsigned dlo(double x) { return (unsigned)__double2loint(x); }
__device__ __forceinline__ unsigned dhi(double x) { return (unsigned)__double2hiint(x); }

struct PackSmem {
  Box box[A_BLOCK];              // staging: warp w owns records [64 w, 64 w + 64)
  Box gsm[2][A_BLOCK / GROUP];   // group boxes of this block and of the previous one
  double win[2][4 * WIN_PLANE];
  unsigned long long wbar[2];    // bulk-copy completion of win[0], win[1]
};

#ifndef PACK_MIN_BLOCKS
#define PACK_MIN_BLOCKS 2
#endif

// min / max of canonical values (finite or ±Inf, no −0.0 mixed with +0.0 — see the
// callers) as compare + select: 3 instructions where fmin/fmax spend 4 on NaN quieting.
// A NaN input makes the mesh unusable (status flag), so its boxes are never searched.
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double dmax(double a, double b) { return b > a ? b : a; }

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Storage-map geometry of block blk: tile row tk, offset rt inside it; `regular` = the
// block lies in full tiles of one tile row (bit-field decode), `windowed` = and starts
// on a tile boundary (exactly two tiles: the shared-memory window path).  One 32-bit
// division (storage indices are < 2^30: the triangle count is < 2^31).
struct BlockGeom {
  uint32_t tk, rt;
  bool regular, windowed;
};
__device__ __forceinline__ BlockGeom block_geom(uint64_t blk, uint32_t N, uint32_t MQ, uint32_t TN, int tiled) {
  BlockGeom g;
  const uint32_t sq0 = (uint32_t)(blk * PACK_THREADS);
  g.tk = sq0 / TN;
  g.rt = sq0 - g.tk * TN;
  g.regular = tiled && g.tk * ORDER_TILE_Q + ORDER_TILE_Q <= MQ && g.rt + PACK_THREADS <= ((N / ORDER_TILE_Q) << 8);
  g.windowed = g.regular && (g.rt & 255) == 0;
  return g;
}

// All threads: cp.async the window of a windowed block into `win` (one commit group).
__device__ __forceinline__ void fetch_window(double* win, const double* __restrict__ coords, uint32_t N,
                                             uint64_t plane, const BlockGeom& g, int tid) {
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(win);
  const uint32_t row0 = g.tk * ORDER_TILE_Q, i0 = (g.rt >> 8) * ORDER_TILE_Q;
#pragma unroll
  for (int u = 0; u < (WIN_LOADS + PACK_THREADS - 1) / PACK_THREADS; ++u) {
    const int e = tid + u * PACK_THREADS;
    if (e < WIN_LOADS) {
      const int p = e / (WIN_ROWS * WIN_COLS), rem = e - p * (WIN_ROWS * WIN_COLS);
      const int r = rem / WIN_COLS, cc = rem - r * WIN_COLS;
      uint32_t col = i0 + cc;
      if (col >= N) col -= N;  // the last window column of the last tiles wraps to θ index 0
      cp_async8(sbase + 8u * (p * WIN_PLANE + r * WIN_STRIDE + cc), coords + p * plane + (uint64_t)(row0 + r) * N + col);
    }
  }
}

__global__ void __launch_bounds__(PACK_THREADS, PACK_MIN_BLOCKS)
    pack_kernel(const double* __restrict__ coords, uint32_t N, uint32_t M, uint32_t Mp, int tiled,
                Box* __restrict__ box, uint32_t* __restrict__ perm, Box* __restrict__ gbox, Box* __restrict__ tbox,
                Box* __restrict__ bbox, uint32_t* __restrict__ status, uint32_t blk0, uint32_t blk1) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PackSmem& S = *reinterpret_cast<PackSmem*>(smem_raw);
  const uint32_t MQ = M - 1;
  const uint64_t nq = (uint64_t)N * MQ;
  const uint64_t n = 2 * nq;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t TN = N <= (0xffffffffu / ORDER_TILE_Q) ? (uint32_t)ORDER_TILE_Q * N : 0xffffffffu;
  const uint64_t plane = (uint64_t)Mp * N;  // Mp: plane stride in rows
  // the thread's quad inside a windowed block: tile tid >> 8, 4×4 sub-tile, quad
  const uint32_t rr = tid & 255;
  const uint32_t li = (tid >> 8) * ORDER_TILE_Q + ((rr >> 4) & 3) * ORDER_SUB_Q + (rr & 3);
  const uint32_t lk = (rr >> 6) * ORDER_SUB_Q + ((rr >> 2) & 3);
  bool bad = false;
  const int warp = tid >> 5;
  // window rows by bulk copies (one 272-byte row per thread of warps 0-2: plane wp, row wr;
  // measured faster than one lane per plane issuing 17 rows) when every row start is
  // 16-byte aligned; else 8-byte cp.async per element
  const bool bulk = !(N & 1u) && !(reinterpret_cast<uintptr_t>(coords) & 15);
  const uint32_t wp = tid / WIN_ROWS, wr = tid - wp * WIN_ROWS;
  if (tid == 0) {
    mbar_init(&S.wbar[0], 1);
    mbar_init(&S.wbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // windowed blocks only.  Columns [i0, i0 + 34) of rows row0 .. row0 + 16 (column i0 + 33
  // is padding: N even and i0 + 32 < N give i0 + 34 <= N); at the right edge (i0 + 32 = N)
  // window column 32 is θ index 0, copied as the 16 bytes of columns 0-1.  Thread 0's
  // arrive.expect_tx may land before or after the copies' complete_tx (tx-count is signed).
  auto issue_window = [&](int buf, const BlockGeom& gw) {
    if (bulk) {
      const uint32_t row0 = gw.tk * ORDER_TILE_Q, i0 = (gw.rt >> 8) * ORDER_TILE_Q;
      const bool wrap = i0 + 2 * ORDER_TILE_Q == N;
      if (tid == 0) mbar_arrive_expect_tx(&S.wbar[buf], 4 * WIN_ROWS * (wrap ? 256 + 16 : 272));
      if (tid < 4 * WIN_ROWS) {
        double* dst = S.win[buf] + wp * WIN_PLANE + wr * WIN_STRIDE;
        const double* src = coords + wp * plane + (uint64_t)(row0 + wr) * N;
        bulk_g2s(dst, src + i0, wrap ? 256 : 272, &S.wbar[buf]);
        if (wrap) bulk_g2s(dst + 2 * ORDER_TILE_Q, src, 16, &S.wbar[buf]);
      }
    } else {
      fetch_window(S.win[buf], coords, N, plane, gw, tid);
    }
  };
  // tile and block boxes of block pb from its 32 group boxes gs (warp 0): lane l reduces
  // component c = l & 7 over groups 8·(l >> 3) .. +7 (hi components negated), xor 8 gives
  // the lane's 512-record tile, xor 16 the block
  auto level_boxes = [&](const Box* gsb, uint64_t pb) {
    const double* gs = reinterpret_cast<const double*>(gsb);
    const int c = lane & 7;
    const unsigned long long neg = c >= 4 ? 0x8000000000000000ull : 0ull;
    const double* src = gs + 64 * (lane >> 3) + c;
    double m = __longlong_as_double(__double_as_longlong(src[0]) ^ neg);
#pragma unroll
    for (int q = 1; q < 8; ++q) m = dmin(m, __longlong_as_double(__double_as_longlong(src[8 * q]) ^ neg));
    m = dmin(m, __shfl_xor_sync(0xffffffffu, m, 8));
    const uint64_t tt = pb * (A_BLOCK / TILE) + (lane >> 4);
    if (!(lane & 8) && tt < (n + TILE - 1) / TILE)
      reinterpret_cast<double*>(tbox)[tt * 8 + c] = __longlong_as_double(__double_as_longlong(m) ^ neg);
    m = dmin(m, __shfl_xor_sync(0xffffffffu, m, 16));
    if (lane < 8) reinterpret_cast<double*>(bbox)[pb * 8 + c] = __longlong_as_double(__double_as_longlong(m) ^ neg);
  };
  const bool levels = gbox && tbox && bbox;
  uint64_t blk = blk0 + blockIdx.x, prev = ~0ull;
  uint32_t wph = 0;  // bit b: parity of the next wait on wbar[b]
  if (blk < blk1) {
    const BlockGeom g = block_geom(blk, N, MQ, TN, tiled);
    if (g.windowed) issue_window(0, g);
  }
  cp_async_commit();
  int it = 0;
  for (; blk < blk1; ++it, blk += gridDim.x) {
    const BlockGeom g = block_geom(blk, N, MQ, TN, tiled);
    const int buf = it & 1;
    const double* win = S.win[buf];
    if (g.windowed && bulk) {
      mbar_wait(&S.wbar[buf], (wph >> buf) & 1u);
      wph ^= 1u << buf;
    }
    cp_async_wait_all();
    // the window is visible; every thread is done with the previous block (its window
    // buffer is free, its group boxes are in gsm[buf ^ 1])
    __syncthreads();
    if (levels && warp == 0 && prev != ~0ull) level_boxes(S.gsm[buf ^ 1], prev);
    {
      const uint64_t nb = blk + gridDim.x;
      if (nb < blk1) {
        const BlockGeom gn = block_geom(nb, N, MQ, TN, tiled);
        if (gn.windowed) issue_window(buf ^ 1, gn);
      }
      cp_async_commit();
    }
    const uint64_t sq = blk * PACK_THREADS + tid;  // storage quad of this thread
    double qlo[4], qhi[4];  // union of the quad's two triangle boxes
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      qlo[c] = __longlong_as_double(0x7ff0000000000000ll);
      qhi[c] = -qlo[c];
    }
    if (sq < nq) {
      uint32_t i, k;
      double w00[4], w10[4], w01[4], w11[4];
      if (g.windowed) {
        i = (g.rt >> 8) * ORDER_TILE_Q + li;
        k = g.tk * ORDER_TILE_Q + lk;
        const double* w = win + lk * WIN_STRIDE + li;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          w00[c] = w[c * WIN_PLANE];
          w10[c] = w[c * WIN_PLANE + 1];
          w01[c] = w[c * WIN_PLANE + WIN_STRIDE];
          w11[c] = w[c * WIN_PLANE + WIN_STRIDE + 1];
        }
      } else {
        if (g.regular) {
          const uint32_t r = g.rt + tid, q = r & 255;  // tile r >> 8, 4×4 sub-tile q >> 4, quad q & 15
          i = (r >> 8) * ORDER_TILE_Q + ((q >> 4) & 3) * ORDER_SUB_Q + (q & 3);
          k = g.tk * ORDER_TILE_Q + (q >> 6) * ORDER_SUB_Q + ((q >> 2) & 3);
        } else if (tiled) {
          quad_of_storage32((uint32_t)sq, N, MQ, i, k);
        } else {
          i = (uint32_t)sq % N;
          k = (uint32_t)sq / N;
        }
        const uint32_t ip = (i + 1 == N) ? 0 : i + 1;
        const uint64_t r0 = (uint64_t)k * N, r1 = r0 + N;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double* pl = coords + c * plane;
          w00[c] = __ldg(pl + r0 + i);
          w10[c] = __ldg(pl + r0 + ip);
          w01[c] = __ldg(pl + r1 + i);
          w11[c] = __ldg(pl + r1 + ip);
        }
      }
      const uint32_t t0 = 2 * (i + N * k);
      // T¹ = (v00, v10, v01), T² = (v01, v10, v11) — the vertex sets of tri_verts, −0.0
      // canonicalised.  B200 has no FP64 min/max instruction (each is a DSETP + 2
      // selects), so the two triangles share min/max(v10, v01); min/max of finite
      // non-NaN values is exact and order-free, so the boxes are the bits of the
      // three-way min/max (NaN/Inf inputs flag the mesh as unusable anyway).
      Box b1, b2;
      // non-finite check: x − x is 0 for finite x and NaN for ±Inf / NaN, so the sum of the
      // 16 differences is NaN iff some vertex coordinate is not finite (no overflow possible)
      double nf = 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double a = dadd(w00[c], 0.0), b = dadd(w10[c], 0.0), d = dadd(w01[c], 0.0), e = dadd(w11[c], 0.0);
        nf = dadd(nf, dadd(dadd(dsub(a, a), dsub(b, b)), dadd(dsub(d, d), dsub(e, e))));
        const double mn = dmin(b, d), mx = dmax(b, d);
        b1.lo[c] = dmin(a, mn);
        b1.hi[c] = dmax(a, mx);
        b2.lo[c] = dmin(e, mn);
        b2.hi[c] = dmax(e, mx);
        qlo[c] = dmin(b1.lo[c], b2.lo[c]);
        qhi[c] = dmax(b1.hi[c], b2.hi[c]);
      }
      bad |= !(nf == 0.0);
      // staging stores: chunk j (16 B) of record r = 2·tid + τ sits at 16-byte slot
      // swz(4r + j); lanes are 128 B apart, so the XOR swizzle spreads each 8-lane phase
      // over all 8 bank columns (unswizzled: 8-way conflicts)
      uint4* st = reinterpret_cast<uint4*>(S.box);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        st[swz(8 * tid + j)] =
            make_uint4(dlo(b1.lo[2 * j]), dhi(b1.lo[2 * j]), dlo(b1.lo[2 * j + 1]), dhi(b1.lo[2 * j + 1]));
        st[swz(8 * tid + 2 + j)] =
            make_uint4(dlo(b1.hi[2 * j]), dhi(b1.hi[2 * j]), dlo(b1.hi[2 * j + 1]), dhi(b1.hi[2 * j + 1]));
        st[swz(8 * tid + 4 + j)] =
            make_uint4(dlo(b2.lo[2 * j]), dhi(b2.lo[2 * j]), dlo(b2.lo[2 * j + 1]), dhi(b2.lo[2 * j + 1]));
        st[swz(8 * tid + 6 + j)] =
            make_uint4(dlo(b2.hi[2 * j]), dhi(b2.hi[2 * j]), dlo(b2.hi[2 * j + 1]), dhi(b2.hi[2 * j + 1]));
      }
      if (perm) reinterpret_cast<uint2*>(perm)[sq] = make_uint2(t0, t0 + 1);
    }
    // the warp's staged records leave as coalesced 16-byte stores (no CTA barrier: each
    // warp stages and copies only its own 64 records)
    __syncwarp();
    {
      const uint64_t r0 = blk * A_BLOCK;
      const uint32_t n16 = (uint32_t)(min((uint64_t)A_BLOCK, n - r0) * (sizeof(Box) / 16));
      const uint32_t q1 = min(n16, (uint32_t)(warp + 1) * 256u);
      const uint4* src = reinterpret_cast<const uint4*>(S.box);
      uint4* dst = reinterpret_cast<uint4*>(box + r0);
      const uint32_t q0 = warp * 256u + lane;
      if (q1 == (uint32_t)(warp + 1) * 256u) {
        // full warp range: swz(q0 + 32 k) = (q0 ^ s0 ^ 4·(k & 1)) + 32 k with s0 = (q0 >> 3) & 7
        // (adding 32 k leaves bits 0-2 alone and adds 4 k to bits 3-5), so two base addresses
        // and immediate offsets
        const uint4* se = src + (q0 ^ ((q0 >> 3) & 7u));
        const uint4* so = src + (q0 ^ ((q0 >> 3) & 7u) ^ 4u);
#pragma unroll
        for (int k = 0; k < 8; ++k) dst[q0 + 32 * k] = (k & 1) ? so[32 * k] : se[32 * k];
      } else {
        for (uint32_t q = q0; q < q1; q += 32) dst[q] = src[swz(q)];
      }
    }
    if (levels) {
      // group = 16 consecutive storage quads = half a warp.  Reduce-scatter instead of an
      // all-reduce: v = the quad box with its hi half negated (every step is then a min;
      // the canonicalised inputs hold no −0, so the negated zeros are all −0 and the
      // result bits equal the unnegated max); at xor 8 / 4 / 2 each lane keeps half of
      // what it holds, xor 1 completes, and lane pair p of the half-warp holds component
      // p of the group box — 8 shuffled values per lane instead of 32.
      const int hl = lane & 15;
      const bool x3 = hl & 8, x2 = hl & 4, x1 = hl & 2;
      double v4[4], v2[2];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double lo = qlo[j], nhi = -qhi[j];
        v4[j] = dmin(x3 ? nhi : lo, __shfl_xor_sync(0xffffffffu, x3 ? lo : nhi, 8));
      }
#pragma unroll
      for (int j = 0; j < 2; ++j)
        v2[j] = dmin(x2 ? v4[2 + j] : v4[j], __shfl_xor_sync(0xffffffffu, x2 ? v4[j] : v4[2 + j], 4));
      double v1 = dmin(x1 ? v2[1] : v2[0], __shfl_xor_sync(0xffffffffu, x1 ? v2[0] : v2[1], 2));
      v1 = dmin(v1, __shfl_xor_sync(0xffffffffu, v1, 1));
      const int comp = (hl >> 1);  // = 4·x3 + 2·x2 + x1: lo[0..3], hi[0..3]
      const uint64_t ng = (n + GROUP - 1) / GROUP;
      double* gs = reinterpret_cast<double*>(S.gsm[buf]);
      if (!(lane & 1)) {
        const uint64_t gi = blk * (A_BLOCK / GROUP) + (tid >> 4);
        const double val = x3 ? -v1 : v1;
        gs[(tid >> 4) * 8 + comp] = val;
        if (gi < ng) reinterpret_cast<double*>(gbox)[gi * 8 + comp] = val;
      }
    }
    prev = blk;
  }
  __syncthreads();  // the last block's group boxes
  if (levels && warp == 0 && prev != ~0ull) level_boxes(S.gsm[(it - 1) & 1], prev);
  cp_async_wait_all();
  if (status && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, 1u);
}

// Culling hierarchy of an arbitrary box array: one CTA per 1024-record block.  Each
// thread unions 4 consecutive records, 8 lanes form a group (shuffle), the CTA's 32
// group boxes give its 2 tile boxes and its block box.
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

uint64_t pack_blocks(uint32_t N, uint32_t M) { return (2ull * N * (M - 1) + A_BLOCK - 1) / A_BLOCK; }

// Enqueue the fused pack of blocks [b0, b1) (b1 = 0: all) on `stream` (device already
// current).  The status flag is cleared by the launch that starts at block 0.
int pack_enqueue(const double* coords, uint32_t N, uint32_t M, int order, double* box, uint32_t* perm, double* gbox,
                 double* tbox, double* bbox, uint32_t* status, cudaStream_t stream, uint64_t b0, uint64_t b1,
                 uint32_t Mp) {
  if (Mp == 0) Mp = M;
  if (Mp < M) return set_error(MCX_E_ARG, "plane stride of %u rows < M = %u", Mp, M);
  if (N < 1 || M < 2) return set_error(MCX_E_ARG, "pack needs N >= 1 and M >= 2 (got N=%u, M=%u)", N, M);
  if (2ull * N * (M - 1) >= (1ull << 31)) return set_error(MCX_E_ARG, "triangle count must be < 2^31");
  if (order != MCX_ORDER_NATURAL && order != MCX_ORDER_TILED) return set_error(MCX_E_ARG, "unknown order %d", order);
  if (!coords || !box) return set_error(MCX_E_ARG, "null buffer");
  if (order == MCX_ORDER_TILED && !perm)
    return set_error(MCX_E_ARG, "MCX_ORDER_TILED needs a perm buffer (searches emit original indices through it)");
  if (((uintptr_t)box | (uintptr_t)gbox | (uintptr_t)tbox | (uintptr_t)bbox) & 15)
    return set_error(MCX_E_ARG, "box and level buffers must be 16-byte aligned");
  if (perm && ((uintptr_t)perm & 7)) return set_error(MCX_E_ARG, "perm must be 8-byte aligned");
  if ((gbox != nullptr) != (tbox != nullptr) || (gbox != nullptr) != (bbox != nullptr))
    return set_error(MCX_E_ARG, "gbox, tbox and bbox must be given together");
  const uint64_t nblk = pack_blocks(N, M);
  if (b1 == 0 || b1 > nblk) b1 = nblk;
  if (b0 >= b1) return MCX_OK;
  static_assert(sizeof(PackSmem) <= 227 * 1024, "pack smem");
  int dev = 0;
  uint64_t slots;
  CUDA_TRY(cudaGetDevice(&dev));
  if (int rc = kernel_prepare(reinterpret_cast<const void*>(pack_kernel), PACK_THREADS, sizeof(PackSmem), 100, dev,
                              &slots))
    return rc;
  if (status && b0 == 0) CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(uint32_t), stream));
  const unsigned grid = (unsigned)std::min<uint64_t>(b1 - b0, slots);  // persistent CTAs
  pack_kernel<<<grid, PACK_THREADS, sizeof(PackSmem), stream>>>(
      coords, N, M, Mp, order == MCX_ORDER_TILED, reinterpret_cast<Box*>(box), perm, reinterpret_cast<Box*>(gbox),
      reinterpret_cast<Box*>(tbox), reinterpret_cast<Box*>(bbox), status, (uint32_t)b0, (uint32_t)b1);
  CUDA_TRY(cudaGetLastError());
  return MCX_OK;
}

}  // namespace mcx

extern "C" {

int mcx_pack(const double* coords, uint32_t N, uint32_t M, int order, double* box, uint32_t* perm, double* gbox,
             double* tbox, double* bbox, uint32_t* status, int device, void* stream) {
  using namespace mcx;
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(device));
  return pack_enqueue(coords, N, M, order, box, perm, gbox, tbox, bbox, status, (cudaStream_t)stream, 0, 0, M);
}

int mcx_levels(const double* box, uint64_t n_tri, double* gbox, double* tbox, double* bbox, int device,
               void* stream) {
  using namespace mcx;
  if (!box || !gbox || !tbox || !bbox) return set_error(MCX_E_ARG, "null buffer");
  if (((uintptr_t)box | (uintptr_t)gbox | (uintptr_t)tbox | (uintptr_t)bbox) & 15)
    return set_error(MCX_E_ARG, "level boxes must be 16-byte aligned");
  if (n_tri == 0) return MCX_OK;
  DeviceGuard guard;
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
