// mcx_search.cu — sm_100a triangle-pair intersection search (libmcx.so).
//
// Replaces the reference's rejection kernel, findall compaction and host-side
// precise test (PAPER.md "Computational Implementation", kernel steps 1-9 and
// Fig. 1; SPEC isect.pair_candidates / find_intersections).
//
// MCX_MODE_BRUTE — search_brute_kernel: every pair gets the AABB test.
//   * A triangles live in registers: each thread owns R = 4 triangle AABBs
//     (8 doubles each), a CTA of 256 threads one absolute A block of 1024
//     storage positions.
//   * B triangle AABBs stream through shared memory in tiles of 512 (32 KB)
//     with a 2-stage ring of 1-D bulk async copies (cp.async.bulk → UBLKCP)
//     completed on mbarriers.  Every B box is a warp-uniform broadcast
//     (4 × LDS.128) that serves 32·R = 128 pair tests.
//   * Pair test = 8 FP64 compares (DSETP), strict-separation semantics of
//     SPEC.md:442-450 (touching boxes are not rejected).
//   * Rare survivors are pushed by warp ballot into a per-warp shared-memory
//     queue; when 32 are queued the warp solves them lane-parallel with the
//     canonical FMA-free FP64 bivector-Cramer sequence, rebuilding
//     the two triangles' geometry from the grids (L1/L2) with the packing's ops.  Hits are compacted with one atomic
//     per warp into the global (iA, iB, s, t, a, b) list (no flag buffer).
//
// MCX_MODE_PREFILTER — mcx_prefilter.cuh: every pair tested by a conservative packed-
//   integer test on quantised boxes, its passes by the exact FP64 test.
//
// MCX_MODE_CULL — the same predicate and the same survivor path behind two levels
//   of exact box culling over the tiled storage order (mcx_pack.cu):
//   cull_blocks_kernel tests every (A block of 1024, B tile of 512) union-box pair
//   and compacts the overlapping ones; cull_pairs_kernel takes them, tests the
//   32×16 (A group, B group) union boxes of 32 triangles each, and runs the pair
//   test only inside overlapping groups.  A union box is disjoint from another box
//   only if all its members are, so the AABB-pass set, singular count and hit set
//   are identical to MCX_MODE_BRUTE; only n_tested shrinks.
//
// MCX_PIPE_SPEC — the SPEC's literal pipeline on the culling
//   kernels: quads are record pairs, quad-box survivors go through the SPEC-literal
//   Moller test and its candidates through the 4 triangle-pair precise tests.
//
// The solve uses only __dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn (never contracted
// into DFMA) and the file is compiled with --fmad=false, so the op sequence is
// bit-identical to oracle/canonical.py.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "../../include/mcx.h"
#include "mcx_common.cuh"
#include "mcx_search.cuh"
#include "mcx_prefilter.cuh"
#include "mcx_internal.cuh"

namespace mcx {

int kernel_prepare(const void* fn, int threads, size_t smem, int carveout, int device, uint64_t* slots) {
  struct Key {
    const void* fn;
    int device, threads, carveout;
    size_t smem;
    bool operator==(const Key& o) const {
      return fn == o.fn && device == o.device && threads == o.threads && carveout == o.carveout && smem == o.smem;
    }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      return std::hash<const void*>()(k.fn) ^ (size_t)k.device * 0x9e3779b97f4a7c15ull ^ (k.smem << 20) ^
             ((size_t)k.threads << 8) ^ (size_t)(k.carveout + 1);
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, uint64_t, Hash> cache;
  const Key key{fn, device, threads, carveout, smem};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *slots = it->second;
      return MCX_OK;
    }
  }
  int sms = 148, occ = 1;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (carveout >= 0) CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carveout));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem));
  *slots = (uint64_t)sms * (occ > 0 ? occ : 1);
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = *slots;
  return MCX_OK;
}

// ------------------------------------------------------------ brute kernel
template <int KIND, class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB) search_brute_kernel(const Batch Bt) {
  constexpr int R = C::R, THREADS = C::THREADS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SearchSmem<C>& S = *reinterpret_cast<SearchSmem<C>*>(smem_raw);
  __shared__ SearchParams Ps;
  __shared__ uint64_t s_unit;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- task of this CTA (1-D grid over all tasks' (A block, B chunk) units)
  if (tid == 0) {
    const uint32_t t = find_task(Bt, blockIdx.x);
    Ps = Bt.tasks[t];
    s_unit = blockIdx.x - Bt.prefix[t];
  }
  __syncthreads();
  const SearchParams& P = Ps;
  const uint64_t unit = s_unit;

  // ---- absolute A block (cyclic shard) and B chunk of this CTA
  const uint64_t gblk = P.blk_first + (unit / P.nchunk) * P.shard_count;
  const uint64_t a0 = gblk * A_BLOCK;
  const uint64_t b0 = (unit % P.nchunk) * P.b_chunk;
  const uint64_t b1 = min(b0 + P.b_chunk, P.nB);
  const int ntiles = (int)((b1 - b0 + TILE - 1) / TILE);

  // ---- mbarrier ring setup + prologue copies (one elected thread)
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&S.full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < STAGES && s < ntiles; ++s) {
      const uint64_t tb = b0 + (uint64_t)s * TILE;
      const uint32_t bytes = (uint32_t)(min((uint64_t)TILE, b1 - tb) * sizeof(Box));
      mbar_arrive_expect_tx(&S.full[s], bytes);
      bulk_g2s(&S.tile[s][0], P.boxB + tb, bytes, &S.full[s]);
    }
  }

  // ---- A triangles into registers (out-of-range slots get empty boxes).  A survivor
  // flush only appends to the candidate list (the precise test is solve_kernel's),
  // so the boxes stay live across it and the hot loop fits 2 CTAs/SM.
  double alo[R][4], ahi[R][4];
  uint32_t aidx[R];
#pragma unroll
  for (int r = 0; r < R; ++r) aidx[r] = (uint32_t)(a0 + (uint64_t)r * THREADS + tid);
  auto load_a = [&]() {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (aidx[r] >= P.a_begin && aidx[r] < P.a_end) {
        const double* src = reinterpret_cast<const double*>(P.boxA + aidx[r]);
        ld_nc_v2(src + 0, alo[r][0], alo[r][1]);
        ld_nc_v2(src + 2, alo[r][2], alo[r][3]);
        ld_nc_v2(src + 4, ahi[r][0], ahi[r][1]);
        ld_nc_v2(src + 6, ahi[r][2], ahi[r][3]);
      } else {
        empty_box(alo[r], ahi[r]);
      }
    }
  };
  load_a();

  uint2* q = S.queue[warp];
  int qn = 0;
  const unsigned lt_mask = (1u << lane) - 1u;

  for (int t = 0; t < ntiles; ++t) {
    const int s = t % STAGES;
    mbar_wait(&S.full[s], (uint32_t)((t / STAGES) & 1));
    const uint64_t tb = b0 + (uint64_t)t * TILE;
    const int nvalid = (int)min((uint64_t)TILE, b1 - tb);
    const Box* tile = S.tile[s];
    // JB B triangles per warp vote: JB·R independent predicate chains in flight.
    auto step = [&](int j, auto jb_c) {
      constexpr int NJ = decltype(jb_c)::value;
      bool p[NJ][R];
      bool any = false;
#pragma unroll
      for (int u = 0; u < NJ; ++u) {
        const double2* bp = reinterpret_cast<const double2*>(tile + j + u);
        const double2 l01 = bp[0], l23 = bp[1], h01 = bp[2], h23 = bp[3];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          p[u][r] = (l01.x <= ahi[r][0]) & (alo[r][0] <= h01.x) & (l01.y <= ahi[r][1]) & (alo[r][1] <= h01.y) &
                    (l23.x <= ahi[r][2]) & (alo[r][2] <= h23.x) & (l23.y <= ahi[r][3]) & (alo[r][3] <= h23.y);
          any |= p[u][r];
        }
      }
      if (__any_sync(0xffffffffu, any)) {
#pragma unroll
        for (int u = 0; u < NJ; ++u) {
          const uint32_t ib = (uint32_t)(tb + j + u);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const unsigned m = __ballot_sync(0xffffffffu, p[u][r]);
            if (p[u][r]) q[qn + __popc(m & lt_mask)] = make_uint2(aidx[r], ib);
            qn += __popc(m);
          }
        }
        __syncwarp();
        if (qn >= 32) {
          do {
            qn -= 32;
            flush_queue(P, Bt, q + qn, 32, lane);
          } while (qn >= 32);
        }
      }
    };
    if constexpr (C::PF == 1) {
      // software-pipelined: the LDS of box j+1 is issued before the compares of box j
      const double2* bp0 = reinterpret_cast<const double2*>(tile);
      double2 n01 = bp0[0], n23 = bp0[1], m01 = bp0[2], m23 = bp0[3];
#pragma unroll(C::UNROLL)
      for (int j = 0; j < nvalid; ++j) {
        const double2 l01 = n01, l23 = n23, h01 = m01, h23 = m23;
        const double2* bp = reinterpret_cast<const double2*>(tile + min(j + 1, nvalid - 1));
        n01 = bp[0]; n23 = bp[1]; m01 = bp[2]; m23 = bp[3];
        bool p[R];
        bool any = false;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          p[r] = (l01.x <= ahi[r][0]) & (alo[r][0] <= h01.x) & (l01.y <= ahi[r][1]) & (alo[r][1] <= h01.y) &
                 (l23.x <= ahi[r][2]) & (alo[r][2] <= h23.x) & (l23.y <= ahi[r][3]) & (alo[r][3] <= h23.y);
          any |= p[r];
        }
        if (__any_sync(0xffffffffu, any)) {
          const uint32_t ib = (uint32_t)(tb + j);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const unsigned m = __ballot_sync(0xffffffffu, p[r]);
            if (p[r]) q[qn + __popc(m & lt_mask)] = make_uint2(aidx[r], ib);
            qn += __popc(m);
          }
          __syncwarp();
          if (qn >= 32) {
            do {
              qn -= 32;
              flush_queue(P, Bt, q + qn, 32, lane);
            } while (qn >= 32);
          }
        }
      }
    } else {
      const int nmain = nvalid - nvalid % C::JB;
#pragma unroll(C::UNROLL)
      for (int j = 0; j < nmain; j += C::JB) step(j, std::integral_constant<int, C::JB>());
      for (int j = nmain; j < nvalid; ++j) step(j, std::integral_constant<int, 1>());
    }
    __syncthreads();  // every warp is done reading stage s
    if (tid == 0 && t + STAGES < ntiles) {
      const uint64_t nb = b0 + (uint64_t)(t + STAGES) * TILE;
      const uint32_t bytes = (uint32_t)(min((uint64_t)TILE, b1 - nb) * sizeof(Box));
      mbar_arrive_expect_tx(&S.full[s], bytes);
      bulk_g2s(&S.tile[s][0], P.boxB + nb, bytes, &S.full[s]);
    }
  }
  __syncwarp();
  if (qn > 0) flush_queue(P, Bt, q, qn, lane);
}

// OR of every task's input-mesh status flags (non-finite coordinates) into *flag.
__global__ void status_kernel(const SearchParams* __restrict__ tasks, uint32_t n, unsigned long long* flag) {
  unsigned v = 0;
  for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
    if (tasks[t].statusA) v |= *tasks[t].statusA;
    if (tasks[t].statusB) v |= *tasks[t].statusB;
  }
  v = __any_sync(0xffffffffu, v != 0);
  if (threadIdx.x == 0 && v) atomicOr(flag, 1ull);
}

// ------------------------------------------------------------ cull kernels
// Level 1: work item = (unit of CULL_UNIT consecutive local A blocks of one task, chunk of
// B tiles), grid-stride: every thread holds the unit's block boxes in registers and sweeps
// the chunk's B tile boxes with coalesced 64-byte loads, the next one loaded while the
// current one is tested (each tile box serves CULL_UNIT tests); overlapping (task, x, y)
// are compacted with one atomic per warp.  Bt.prefix here is the per-task prefix of units.
// The B tiles are chunked only when the units alone would not fill the resident CTA slots.
constexpr int CULL_UNIT = 4;
constexpr int CULL_YCHUNK = 512;  // fewest B tiles per chunk when the tiles are split

__device__ __forceinline__ Box ldg_box(const Box* p) {
  const double2* s = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(s), b = __ldg(s + 1), c = __ldg(s + 2), d = __ldg(s + 3);
  Box r;
  r.lo[0] = a.x; r.lo[1] = a.y; r.lo[2] = b.x; r.lo[3] = b.y;
  r.hi[0] = c.x; r.hi[1] = c.y; r.hi[2] = d.x; r.hi[3] = d.y;
  return r;
}

__global__ void __launch_bounds__(256, 2) cull_blocks_kernel(const Batch Bt) {
  const uint64_t nyc = Bt.cull_ychunks;
  const uint64_t items = Bt.cull_items;  // a kernel parameter: no load before the first item
  const int tid = threadIdx.x, lane = tid & 31;
  for (uint64_t w = blockIdx.x; w < items; w += gridDim.x) {
    // every thread reads the item's task and A block boxes itself (same addresses: L1
    // broadcasts) and keeps the boxes in registers — no single-thread prologue behind a CTA
    // barrier (it was a third of the kernel's stall samples)
    const uint64_t u = w / nyc, yc = (w - u * nyc) * Bt.cull_ychunk;
    const uint32_t t = find_task(Bt, u);
    const SearchParams& P = Bt.tasks[t];
    const uint64_t x0 = (u - __ldg(Bt.prefix + t)) * CULL_UNIT;
    const uint32_t nx = (uint32_t)min((uint64_t)CULL_UNIT, P.my_blocks - x0);
    const Box* tb = P.tboxB;
    const uint64_t yend = min(P.nB ? P.ntilesB : 0, yc + Bt.cull_ychunk);  // yc >= ntiles: nothing
    Box abox[CULL_UNIT];
#pragma unroll
    for (uint32_t k = 0; k < CULL_UNIT; ++k) {
      if (k < nx) {
        abox[k] = ldg_box(P.bboxA + P.blk_first + (x0 + k) * P.shard_count);
      } else {
        empty_box(abox[k].lo, abox[k].hi);
      }
    }
    // software-pipelined sweep: the next round's tile box is loaded before this round's is
    // tested, so a CTA's dependent chain is ~3 round trips plus compute, not one per round
    auto tile = [&](uint64_t y) {
      Box r;
      if (y < yend) {
        r = ldg_box(tb + y);
      } else {
        empty_box(r.lo, r.hi);
      }
      return r;
    };
    Box bc = tile(yc + tid);
    for (uint64_t y0 = yc; y0 < yend; y0 += blockDim.x) {
      const Box bn = tile(y0 + blockDim.x + tid);
      const uint64_t y = y0 + tid;
#pragma unroll
      for (uint32_t k = 0; k < CULL_UNIT; ++k) {
        const bool ov = k < nx && y < yend && box_overlap(abox[k], bc);
        const unsigned m = __ballot_sync(0xffffffffu, ov);
        if (m) {
          const int leader = __ffs(m) - 1;
          unsigned long long pos = 0;
          if (lane == leader) pos = atomicAdd(Bt.list_count, (unsigned long long)__popc(m));
          pos = __shfl_sync(0xffffffffu, pos, leader) + __popc(m & ((1u << lane) - 1u));
          if (ov && pos < Bt.blk_cap) Bt.blk_list[pos] = make_uint4(t, (uint32_t)x0 + k, (uint32_t)y, 0);
        }
      }
      bc = bn;
    }
  }
}

constexpr int CULL_THREADS = 256;
constexpr int CULL_WARPS = CULL_THREADS / 32;
constexpr int GPAIRS = (A_BLOCK / GROUP) * (TILE / GROUP);  // 32 × 16 group pairs per block pair

struct CullSmem {
  Box bst[CULL_WARPS][GROUP];  // the B group of the warp's current group pair (one load per lane)
  uint2 queue[CULL_WARPS][64];
  uint16_t gpair[GPAIRS];
  unsigned int n_gpair[2];  // by entry parity: the next entry's counter is reset before this one's barrier
};

// Level 2 + pair tests: one CTA per overlapping (task, A block, B tile), persistent.
// KIND_TRI: one A triangle per lane against the 32 B triangles of a group.
// KIND_QUAD: quads are record pairs (2s, 2s+1 = T¹, T² of one quad), quad box = union
// of the two triangle boxes (= the SPEC's quad AABB); lane = (A quad l & 15, half of
// the B group's 16 quads); survivors go through the SPEC-literal Moller stage.
template <int KIND>
__global__ void __launch_bounds__(CULL_THREADS) cull_pairs_kernel(const Batch Bt) {
  __shared__ CullSmem S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  unsigned long long n_tested = 0;
  uint2* q = S.queue[warp];
  int qn = 0;
  uint32_t cur_task = 0xffffffffu;
  if (tid < 2) S.n_gpair[tid] = 0;
  __syncthreads();
  const uint64_t nlist = min((uint64_t)*(volatile unsigned long long*)Bt.list_count, Bt.blk_cap);
  const uint64_t e0 = Bt.list_done ? min((uint64_t)*Bt.list_done, nlist) : 0;
  uint32_t par = 0;
  // the task's parameters are read from the task table by every thread (L1 broadcasts), not
  // copied to shared memory by one thread behind a barrier
  for (uint64_t e = e0 + blockIdx.x; e < nlist; e += gridDim.x, par ^= 1u) {
    const uint4 txy = Bt.blk_list[e];
    if (txy.x != cur_task) {
      // task switch: drain this warp's queue and counters against the old task first
      if (cur_task != 0xffffffffu) {
        __syncwarp();
        if (qn > 0) flush_queue(Bt.tasks[cur_task], Bt, q, qn, lane);
        qn = 0;
        flush_tested(Bt.tasks[cur_task], lane, n_tested);
        n_tested = 0;
      }
      cur_task = txy.x;
    }
    const SearchParams P = Bt.tasks[cur_task];  // by value: the fields stay in registers across the stores below
    const uint64_t gblk = P.blk_first + (uint64_t)txy.y * P.shard_count;
    // the previous entry's counter: every thread read it before that entry's closing barrier,
    // and the next entry's atomics come after this entry's barrier
    if (tid == 0) S.n_gpair[par ^ 1u] = 0;
    const uint64_t ngA = (P.nA + GROUP - 1) / GROUP, ngB = (P.nB + GROUP - 1) / GROUP;
    // every thread's group-box loads are issued before any compaction atomic
    static_assert(GPAIRS % CULL_THREADS == 0, "group pairs per thread");
    bool gov[GPAIRS / CULL_THREADS];
#pragma unroll
    for (int i = 0; i < GPAIRS / CULL_THREADS; ++i) {
      const int k = tid + i * CULL_THREADS;
      const uint64_t ga = gblk * (A_BLOCK / GROUP) + k / (TILE / GROUP);
      const uint64_t gb = (uint64_t)txy.z * (TILE / GROUP) + k % (TILE / GROUP);
      gov[i] = ga < ngA && gb < ngB && box_overlap(ldg_box(P.gboxA + ga), ldg_box(P.gboxB + gb));
    }
#pragma unroll
    for (int i = 0; i < GPAIRS / CULL_THREADS; ++i)
      if (gov[i]) S.gpair[atomicAdd(&S.n_gpair[par], 1u)] = (uint16_t)(tid + i * CULL_THREADS);
    __syncthreads();
    const int ng = (int)S.n_gpair[par];
    for (int w = warp; w < ng; w += CULL_WARPS) {
      const int k = S.gpair[w];
      const uint64_t ga0 = gblk * A_BLOCK + (uint64_t)(k / (TILE / GROUP)) * GROUP;
      const uint64_t jb0 = (uint64_t)txy.z * TILE + (uint64_t)(k % (TILE / GROUP)) * GROUP;
      // stage the B group in shared memory, one record per lane, so the loop below reads
      // it at shared-memory latency instead of one dependent L2 round trip per record
      // (the load is issued here, the shared-memory store after the lane's A loads, so both
      // round trips overlap)
      Box* sb = S.bst[warp];
      const bool vbl = jb0 + lane < P.nB;
      Box bl;
      if (vbl) bl = ldg_box(P.boxB + jb0 + lane);
      auto stage = [&]() {
        __syncwarp();  // the previous group pair's reads of sb are done
        if (vbl) sb[lane] = bl;
        __syncwarp();
      };
      if constexpr (KIND == KIND_TRI) {
        const uint64_t ia = ga0 + lane;
        const bool va = ia >= P.a_begin && ia < P.a_end;
        double alo[4], ahi[4];
        if (va) {
          const double2* s = reinterpret_cast<const double2*>(P.boxA + ia);
          const double2 a = __ldg(s), b = __ldg(s + 1), c = __ldg(s + 2), d = __ldg(s + 3);
          alo[0] = a.x; alo[1] = a.y; alo[2] = b.x; alo[3] = b.y;
          ahi[0] = c.x; ahi[1] = c.y; ahi[2] = d.x; ahi[3] = d.y;
        } else {
          empty_box(alo, ahi);
        }
        stage();
        const int nb = (int)min((uint64_t)GROUP, P.nB - jb0);
        const unsigned vmask = __ballot_sync(0xffffffffu, va);
        if (lane == 0) n_tested += (unsigned long long)__popc(vmask) * nb;
        // all 32 tests first (independent shared loads and compares, a bit per B record),
        // then one ballot per B record that some lane keeps
        unsigned pm = 0;
#pragma unroll
        for (int j = 0; j < GROUP; ++j) {
          if (j < nb) {
            const double2* bp = reinterpret_cast<const double2*>(sb + j);
            const double2 l01 = bp[0], l23 = bp[1], h01 = bp[2], h23 = bp[3];
            const bool p = (l01.x <= ahi[0]) & (alo[0] <= h01.x) & (l01.y <= ahi[1]) & (alo[1] <= h01.y) &
                           (l23.x <= ahi[2]) & (alo[2] <= h23.x) & (l23.y <= ahi[3]) & (alo[3] <= h23.y);
            pm |= (unsigned)p << j;
          }
        }
        unsigned anyj = __reduce_or_sync(0xffffffffu, pm);
        while (anyj) {
          const int j = __ffs(anyj) - 1;
          anyj &= anyj - 1;
          const bool p = (pm >> j) & 1u;
          const unsigned m = __ballot_sync(0xffffffffu, p);
          if (p) q[qn + __popc(m & lt_mask)] = make_uint2((uint32_t)ia, (uint32_t)(jb0 + j));
          qn += __popc(m);
          __syncwarp();
          if (qn >= 32) {
            qn -= 32;
            flush_queue(P, Bt, q + qn, 32, lane);
          }
        }
      } else {
        const uint64_t ra = ga0 + 2 * (uint64_t)(lane & 15);  // T¹ record of this lane's A quad
        const bool va = ra >= P.a_begin && ra + 2 <= P.a_end;
        double alo[4], ahi[4];
        empty_box(alo, ahi);
        if (va) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const Box bx = P.boxA[ra + u];
#pragma unroll
            for (int c = 0; c < 4; ++c) { alo[c] = fmin(alo[c], bx.lo[c]); ahi[c] = fmax(ahi[c], bx.hi[c]); }
          }
        }
        const uint32_t qa = va ? (P.permA ? __ldg(P.permA + ra) >> 1 : (uint32_t)(ra >> 1)) : 0u;
        stage();
        // all 8 quad-box tests first (a bit per B quad), then one ballot per B quad that some
        // lane keeps
        constexpr int NQ = (GROUP / 2) / 2;
        const uint64_t rb0 = jb0 + 2 * (uint64_t)((lane >> 4) * NQ);  // T¹ record of the lane's first B quad
        unsigned pm = 0;
#pragma unroll
        for (int jj = 0; jj < NQ; ++jj) {
          const uint64_t rb = rb0 + 2 * (uint64_t)jj;
          if (rb + 1 < P.nB && va) {
            double blo[4], bhi[4];
            empty_box(blo, bhi);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const Box bx = sb[rb - jb0 + u];
#pragma unroll
              for (int c = 0; c < 4; ++c) { blo[c] = fmin(blo[c], bx.lo[c]); bhi[c] = fmax(bhi[c], bx.hi[c]); }
            }
            ++n_tested;
            const bool p = (blo[0] <= ahi[0]) & (alo[0] <= bhi[0]) & (blo[1] <= ahi[1]) & (alo[1] <= bhi[1]) &
                           (blo[2] <= ahi[2]) & (alo[2] <= bhi[2]) & (blo[3] <= ahi[3]) & (alo[3] <= bhi[3]);
            pm |= (unsigned)p << jj;
          }
        }
        unsigned anyj = __reduce_or_sync(0xffffffffu, pm);
        while (anyj) {
          const int jj = __ffs(anyj) - 1;
          anyj &= anyj - 1;
          const bool p = (pm >> jj) & 1u;
          const unsigned m = __ballot_sync(0xffffffffu, p);
          if (p) {
            const uint64_t rb = rb0 + 2 * (uint64_t)jj;
            const uint32_t qb = P.permB ? __ldg(P.permB + rb) >> 1 : (uint32_t)(rb >> 1);
            q[qn + __popc(m & lt_mask)] = make_uint2(qa, qb);
          }
          qn += __popc(m);
          __syncwarp();
          if (qn >= 32) {
            qn -= 32;
            flush_queue(P, Bt, q + qn, 32, lane);
          }
        }
      }
    }
    __syncthreads();  // gpair list reused by the next entry
  }
  if (cur_task != 0xffffffffu) {
    __syncwarp();
    if (qn > 0) flush_queue(Bt.tasks[cur_task], Bt, q, qn, lane);
    flush_tested(Bt.tasks[cur_task], lane, n_tested);
  }
}

// --------------------------------------------------------------- host side
template <int KIND, class C>
static int launch_brute_cfg(std::vector<SearchParams>& T, Batch& Bt, std::vector<uint64_t>& prefix, void* dev_tab,
                            int device, cudaStream_t stream) {
  const size_t smem = sizeof(SearchSmem<C>);
  uint64_t slots = 0, total = 0;
  int rc = resident_slots(search_brute_kernel<KIND, C>, C::THREADS, smem, device, &slots);
  if (rc == MCX_OK) rc = upload_plan(T, Bt, prefix, dev_tab, slots, 16, stream, &total);
  if (rc != MCX_OK || total == 0) return rc;
  search_brute_kernel<KIND, C><<<(unsigned)total, C::THREADS, smem, stream>>>(Bt);
  CUDA_TRY(cudaGetLastError());
  return MCX_OK;
}

template <int KIND>
static int launch_brute(std::vector<SearchParams>& T, Batch& Bt, std::vector<uint64_t>& prefix, void* dev_tab,
                        int device, cudaStream_t stream) {
  switch (variant_from_env()) {
    case 1: return launch_brute_cfg<KIND, Cfg<4, 2, 1, 2, 0>>(T, Bt, prefix, dev_tab, device, stream);
    case 2: return launch_brute_cfg<KIND, Cfg<4, 2, 1, 8, 1>>(T, Bt, prefix, dev_tab, device, stream);
    case 3: return launch_brute_cfg<KIND, Cfg<4, 2, 1, 2, 1>>(T, Bt, prefix, dev_tab, device, stream);
    default: return launch_brute_cfg<KIND, Cfg<4, 2, 1, 4, 1>>(T, Bt, prefix, dev_tab, device, stream);
  }
}

template <int KIND>
static int launch_cull(std::vector<SearchParams>& T, Batch& Bt, std::vector<uint64_t>& prefix, void* dev_tab,
                       int device, cudaStream_t stream) {
  prefix.assign(T.size() + 1, 0);  // per-task prefix of level-1 units (CULL_UNIT A blocks each)
  for (size_t t = 0; t < T.size(); ++t)
    prefix[t + 1] = prefix[t] + (T[t].nB ? (T[t].my_blocks + CULL_UNIT - 1) / CULL_UNIT : 0);
  const uint64_t total = prefix.back();
  const size_t tab = sizeof(SearchParams) * T.size();
  CUDA_TRY(h2d_async(dev_tab, T.data(), tab, stream));
  CUDA_TRY(h2d_async((char*)dev_tab + tab, prefix.data(), sizeof(uint64_t) * prefix.size(), stream));
  dstamp(stream, "    cull: task table uploaded");
  if (total == 0) return MCX_OK;
  Bt.tasks = reinterpret_cast<const SearchParams*>(dev_tab);
  Bt.prefix = reinterpret_cast<const uint64_t*>((char*)dev_tab + tab);
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device);
  uint64_t maxt = 1;
  for (const SearchParams& P : T) maxt = std::max<uint64_t>(maxt, P.nB ? P.ntilesB : 0);
  // split the B tiles only as far as needed to fill the resident CTA slots (C3: 256 units
  // -> 1 chunk, one wave), never below CULL_YCHUNK tiles
  const uint64_t want = std::max<uint64_t>(1, (uint64_t)dev_sms * 2 / total);  // 2 resident CTAs per SM
  const uint64_t nyc = std::min<uint64_t>(want, (maxt + CULL_YCHUNK - 1) / CULL_YCHUNK);
  Bt.cull_ychunk = (maxt + nyc - 1) / nyc;
  Bt.cull_ychunks = (uint32_t)((maxt + Bt.cull_ychunk - 1) / Bt.cull_ychunk);
  Bt.cull_items = total * Bt.cull_ychunks;
  uint64_t g1 = Bt.cull_items;
  if (g1 > (uint64_t)dev_sms * 8) g1 = (uint64_t)dev_sms * 8;
  cull_blocks_kernel<<<(unsigned)g1, 256, 0, stream>>>(Bt);
  CUDA_TRY(cudaGetLastError());
  dstamp(stream, "    cull: level 1 done");
  cull_pairs_kernel<KIND><<<(unsigned)(dev_sms * 8), CULL_THREADS, 0, stream>>>(Bt);
  CUDA_TRY(cudaGetLastError());
  dstamp(stream, "    cull: level 2 + pair tests done");
  return MCX_OK;
}

// Stage 3 over the candidate list the sweep kernels compacted (count read on the device).
template <int KIND>
static int launch_solve(const Batch& Bt, int device, cudaStream_t stream) {
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device);
  solve_kernel<KIND><<<(unsigned)(dev_sms * 4), 256, 0, stream>>>(Bt);
  CUDA_TRY(cudaGetLastError());
  return MCX_OK;
}

struct Timing {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ~Timing() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
};

// Absolute-block shard geometry: blocks b in [⌊a_begin/1024⌋, ⌈a_end/1024⌉) with b % count == index.
struct ShardGeom {
  uint64_t first, my_blocks, na;
};

static ShardGeom shard_geom(uint64_t a_begin, uint64_t a_end, uint32_t sidx, uint32_t scount) {
  ShardGeom g = {0, 0, 0};
  if (a_end <= a_begin) return g;
  const uint64_t b_lo = a_begin / A_BLOCK, b_hi = (a_end + A_BLOCK - 1) / A_BLOCK;
  g.first = b_lo + ((uint64_t)sidx + scount - b_lo % scount) % scount;
  if (g.first >= b_hi) return g;
  g.my_blocks = (b_hi - g.first + scount - 1) / scount;
  for (uint64_t x = 0; x < g.my_blocks; ++x) {
    const uint64_t b = g.first + x * scount;
    const uint64_t lo = b * A_BLOCK > a_begin ? b * A_BLOCK : a_begin;
    const uint64_t hi = (b + 1) * A_BLOCK < a_end ? (b + 1) * A_BLOCK : a_end;
    g.na += hi - lo;
  }
  return g;
}

// The roles a task is searched with (MCX_ORIENT_LARGER_A exchanges A and B when B is the
// larger mesh and A has no range): *A is blocked / sharded, [*a0, *a1) its range.
struct Oriented {
  const mcx_mesh_dev *A, *B;
  uint64_t a0, a1;
  bool swap;
};

static Oriented orient_task(const mcx_task& tk, const mcx_opts* o) {
  Oriented r{tk.A, tk.B, tk.a_begin, 0, false};
  if (!tk.A || !tk.B) return r;
  const bool whole = tk.a_begin == 0 && (tk.a_end == 0 || tk.a_end == tk.A->n_tri);
  r.swap = o && o->orient == MCX_ORIENT_LARGER_A && whole && tk.B->n_tri > tk.A->n_tri;
  if (r.swap) {
    r.A = tk.B;
    r.B = tk.A;
    r.a0 = 0;
  }
  r.a1 = r.swap ? r.A->n_tri : (tk.a_end ? tk.a_end : tk.A->n_tri);
  return r;
}

// Workspace layout: [0, 64) shared counters (emit, list count); then 64 B of
// counters per task; then the task table + prefix; then the cull block list.
static uint64_t align16(uint64_t v) { return (v + 15) & ~15ull; }

struct WsLayout {
  uint64_t counters, table, list, total, list_cap, cand, cand_cap;
  uint64_t jobs, quant;  // MCX_MODE_PREFILTER: fp32-box job table, then the boxes of each distinct mesh
};

// MCX_MODE_PREFILTER: the distinct meshes of a batch (by box pointer, in order of
// first appearance), each converted to conservative fp32 boxes once per call.
static void distinct_meshes(const mcx_task* tasks, uint32_t n, std::vector<const mcx_mesh_dev*>& out,
                            std::unordered_map<const double*, size_t>* index = nullptr) {
  std::unordered_map<const double*, size_t> local;
  std::unordered_map<const double*, size_t>& idx = index ? *index : local;
  out.clear();
  idx.clear();
  for (uint32_t t = 0; t < n; ++t)
    for (const mcx_mesh_dev* m : {tasks[t].A, tasks[t].B})
      if (m && idx.emplace(m->box, out.size()).second) out.push_back(m);
}

// Stepped batches: header words 5 / 6 ← the block-list / candidate counts (1 and 3).
__global__ void mark_done_kernel(unsigned long long* h) {
  h[5] = h[1];
  h[6] = h[3];
}

static WsLayout ws_layout(const mcx_task* tasks, uint32_t n, const mcx_opts* o) {
  WsLayout L;
  L.counters = 64;
  L.table = align16(64 + 64ull * n);
  L.list = align16(L.table + sizeof(SearchParams) * n + 8ull * (n + 1));
  L.list_cap = 0;
  if (o && (o->mode == MCX_MODE_CULL || o->pipeline == MCX_PIPE_SPEC)) {
    const uint32_t scount = o->shard_count ? o->shard_count : 1;
    for (uint32_t t = 0; t < n; ++t) {
      const Oriented ot = orient_task(tasks[t], o);
      const mcx_mesh_dev* A = ot.A;
      const mcx_mesh_dev* B = ot.B;
      if (!A || !B) continue;
      const ShardGeom g = shard_geom(ot.a0, ot.a1, o->shard_index % scount, scount);
      L.list_cap += g.my_blocks * ((B->n_tri + TILE - 1) / TILE);
    }
  }
  L.cand = align16(L.list + 16 * L.list_cap);
  L.cand_cap = (o && o->cand_cap) ? o->cand_cap : MCX_DEFAULT_CAND_CAP;
  L.jobs = align16(L.cand + 16 * L.cand_cap);
  L.quant = L.jobs;
  L.total = L.jobs;
  if (o && o->mode == MCX_MODE_PREFILTER) {
    std::vector<const mcx_mesh_dev*> ms;
    distinct_meshes(tasks, n, ms);
    L.quant = align16(L.jobs + sizeof(FboxJob) * ms.size());
    L.total = L.quant;
    for (const mcx_mesh_dev* m : ms) L.total += 32 * m->n_tri;
  }
  return L;
}

// MCX_MODE_PREFILTER below this many pairs per call runs the FP64 sweep instead: the
// quantised sweep's per-warp setup (frames, A words, B quantisation) and its slow path
// dominate small or dense batches (measured crossover between 6.7e7 and 1.1e9 pairs,
// DESIGN.md §5); results are identical either way.
// MCX_PREFILTER_MIN_PAIRS overrides it (tests use 0 to exercise the quantised kernel on
// small inputs).
static uint64_t prefilter_min_pairs() {
  const char* v = getenv("MCX_PREFILTER_MIN_PAIRS");
  return v ? strtoull(v, nullptr, 10) : (1ull << 28);
}

// Per-task stats and status from the workspace header (h: 8 shared + 8 per task u64s;
// h[4] = 1 if MCX_MODE_PREFILTER ran as the FP64 sweep).
int batch_stats(const unsigned long long* h, uint32_t n, const mcx_opts* o, uint64_t cap, mcx_stats* st, float ms) {
  const bool spec = o->pipeline == MCX_PIPE_SPEC;
  const int mode = (o->mode == MCX_MODE_PREFILTER && (h[4] & 0xff)) ? MCX_MODE_BRUTE : o->mode;
  const uint64_t cand_cap = o->cand_cap ? o->cand_cap : MCX_DEFAULT_CAND_CAP;
  for (uint32_t t = 0; t < n; ++t) {
    const unsigned long long* c = h + 8 + 8ull * t;
    st[t].n_hits = c[0];
    st[t].n_aabb_pass = c[1];
    st[t].n_singular = c[2];
    st[t].n_tested = mode == MCX_MODE_CULL ? c[3] : st[t].n_pairs;
    st[t].n_exact_tests = mode == MCX_MODE_BRUTE ? st[t].n_pairs : c[3];
    st[t].n_candidates = spec ? c[4] : c[1];
    st[t].kernel_ms = ms;
  }
  if (h[2]) return set_error(MCX_E_ARG, "non-finite (NaN/Inf) coordinates in an input mesh (mcx_pack status)");
  if (h[3] > cand_cap)
    return set_error(MCX_E_CAPACITY, "candidate capacity %llu < %llu box-test survivors (opts->cand_cap)",
                     (unsigned long long)cand_cap, h[3]);
  if (h[0] > cap)
    return set_error(MCX_E_CAPACITY, "hit capacity %llu < %llu hits", (unsigned long long)cap, h[0]);
  return MCX_OK;
}

int launch_batch(const mcx_task* tasks, uint32_t n, const mcx_opts* o, mcx_hit* hits, uint32_t* hit_task,
                 uint64_t cap, mcx_stats* st, unsigned long long* h_counters, const BatchStep* step,
                 bool header_later) {
  if (!tasks || n == 0 || !o || !st) return set_error(MCX_E_ARG, "null argument or empty batch");
  cudaStream_t stream = (cudaStream_t)o->stream;
  const uint32_t scount = o->shard_count ? o->shard_count : 1;
  const uint32_t sidx = o->shard_index;
  if (sidx >= scount) return set_error(MCX_E_ARG, "shard_index %u >= shard_count %u", sidx, scount);
  if (o->mode != MCX_MODE_BRUTE && o->mode != MCX_MODE_CULL && o->mode != MCX_MODE_PREFILTER)
    return set_error(MCX_E_ARG, "unknown mode %d", o->mode);
  if (o->pipeline != MCX_PIPE_TRIANGLE && o->pipeline != MCX_PIPE_SPEC)
    return set_error(MCX_E_ARG, "unknown pipeline %d", o->pipeline);
  if (o->pipeline == MCX_PIPE_SPEC && o->mode != MCX_MODE_CULL)
    return set_error(MCX_E_ARG, "MCX_PIPE_SPEC runs on the culling kernels only (mode MCX_MODE_CULL)");
  const bool spec = o->pipeline == MCX_PIPE_SPEC;
  if (spec)
    for (uint32_t t = 0; t < n; ++t)
      if ((tasks[t].a_begin | tasks[t].a_end) & 1)
        return set_error(MCX_E_ARG, "task %u: MCX_PIPE_SPEC needs an A range of whole quads (even bounds)", t);
  if (cap > 0 && !hits) return set_error(MCX_E_ARG, "null hit buffer with nonzero capacity");
  if (step && (o->mode != MCX_MODE_CULL || o->orient != MCX_ORIENT_AS_GIVEN || !step->whole))
    return set_error(MCX_E_ARG, "stepped batches run MCX_MODE_CULL on pre-oriented tasks");
  const WsLayout L = ws_layout(step ? step->whole : tasks, n, o);
  if (!o->workspace || o->workspace_bytes < L.total || ((uintptr_t)o->workspace & 15))
    return set_error(MCX_E_ARG, "workspace too small or misaligned (need %llu bytes, 16-byte aligned)",
                     (unsigned long long)L.total);
  char* ws = (char*)o->workspace;
  std::vector<const mcx_mesh_dev*> meshes;
  std::unordered_map<const double*, size_t> mesh_index;
  std::vector<FboxJob> jobs;
  if (o->mode == MCX_MODE_PREFILTER) {
    distinct_meshes(tasks, n, meshes, &mesh_index);
    uint64_t off = L.quant;
    for (const mcx_mesh_dev* m : meshes) {
      jobs.push_back(FboxJob{reinterpret_cast<const Box*>(m->box), reinterpret_cast<float4*>(ws + off), m->n_tri});
      off += 32 * m->n_tri;
    }
  }
  auto fbox_of = [&](const mcx_mesh_dev* m) -> float4* { return jobs[mesh_index.at(m->box)].dst; };
  if (o->orient != MCX_ORIENT_AS_GIVEN && o->orient != MCX_ORIENT_LARGER_A)
    return set_error(MCX_E_ARG, "unknown orient %d", o->orient);
  std::vector<SearchParams> T(n);
  for (uint32_t t = 0; t < n; ++t) {
    if (!tasks[t].A || !tasks[t].B) return set_error(MCX_E_ARG, "task %u: null mesh", t);
    if (tasks[t].a_end > tasks[t].A->n_tri || tasks[t].a_begin > (tasks[t].a_end ? tasks[t].a_end : tasks[t].A->n_tri))
      return set_error(MCX_E_ARG, "task %u: A range [%llu, %llu) outside [0, %llu)", t,
                       (unsigned long long)tasks[t].a_begin, (unsigned long long)tasks[t].a_end,
                       (unsigned long long)tasks[t].A->n_tri);
    const Oriented ot = orient_task(tasks[t], o);  // the sweep blocks / shards the larger mesh; the solve un-swaps
    const bool swap = ot.swap;
    const mcx_mesh_dev* A = ot.A;
    const mcx_mesh_dev* B = ot.B;
    const uint64_t a_begin = ot.a0;
    const uint64_t a_end = ot.a1;
    if (a_end > A->n_tri || a_begin > a_end)
      return set_error(MCX_E_ARG, "task %u: A range [%llu, %llu) outside [0, %llu)", t, (unsigned long long)a_begin,
                       (unsigned long long)a_end, (unsigned long long)A->n_tri);
    if (A->n_tri >= (1ull << 31) || B->n_tri >= (1ull << 31))
      return set_error(MCX_E_ARG, "task %u: triangle counts must be < 2^31", t);
    if (!A->box || !B->box || !A->coords || !B->coords) return set_error(MCX_E_ARG, "task %u: null box/coords", t);
    if (((uintptr_t)A->box | (uintptr_t)B->box) & 15)
      return set_error(MCX_E_ARG, "task %u: box pointers must be 16-byte aligned", t);
    if (A->M < 2 || B->M < 2 || A->n_tri != 2ull * A->N * (A->M - 1) || B->n_tri != 2ull * B->N * (B->M - 1))
      return set_error(MCX_E_ARG, "task %u: n_tri does not match the N x M grid", t);
    if (o->mode == MCX_MODE_CULL && (!A->gbox || !A->bbox || !B->gbox || !B->tbox))
      return set_error(MCX_E_ARG, "task %u: MCX_MODE_CULL needs level boxes (mcx_pack) on both meshes", t);
    const ShardGeom g = shard_geom(a_begin, a_end, sidx, scount);
    SearchParams& P = T[t];
    P = SearchParams{};
    P.boxA = reinterpret_cast<const Box*>(A->box);
    P.permA = A->perm;
    P.boxB = reinterpret_cast<const Box*>(B->box);
    P.permB = B->perm;
    P.coordsA = A->coords;
    P.coordsB = B->coords;
    P.NA = A->N; P.MA = A->M; P.NB = B->N; P.MB = B->M;
    P.MpA = A->plane_rows ? A->plane_rows : A->M;
    P.MpB = B->plane_rows ? B->plane_rows : B->M;
    P.nA = A->n_tri;
    P.a_begin = a_begin;
    P.a_end = a_end;
    P.blk_first = g.first;
    P.my_blocks = g.my_blocks;
    P.nB = B->n_tri;
    P.ntilesB = (B->n_tri + TILE - 1) / TILE;
    P.shard_count = scount;
    P.task = t;
    P.swapped = (swap || (step && step->swap)) ? 1u : 0u;
    P.counters = reinterpret_cast<unsigned long long*>(ws + L.counters + 64ull * t);
    P.gboxA = reinterpret_cast<const Box*>(A->gbox);
    P.bboxA = reinterpret_cast<const Box*>(A->bbox);
    P.gboxB = reinterpret_cast<const Box*>(B->gbox);
    P.tboxB = reinterpret_cast<const Box*>(B->tbox);
    P.statusA = A->status;
    P.statusB = B->status;
    if (o->mode == MCX_MODE_PREFILTER) {
      P.fA = fbox_of(A);
      P.fB = fbox_of(B);
    }
    st[t] = mcx_stats{};
    st[t].n_pairs = spec ? (g.na / 2) * (B->n_tri / 2) : g.na * B->n_tri;
  }
  if (!step || step->first) CUDA_TRY(cudaMemsetAsync(ws, 0, L.counters + 64ull * n, stream));
  uint64_t batch_pairs = 0;
  for (uint32_t t = 0; t < n; ++t) batch_pairs += st[t].n_pairs;
  const bool pf_as_brute = o->mode == MCX_MODE_PREFILTER && batch_pairs < prefilter_min_pairs();
  if (pf_as_brute) CUDA_TRY(cudaMemsetAsync(ws + 32, 1, 1, stream));  // header word 4: "ran as the FP64 sweep"
  Batch Bt = {};
  Bt.n_tasks = n;
  Bt.hits = hits;
  Bt.hit_task = hit_task;
  Bt.cap = cap;
  Bt.emit = reinterpret_cast<unsigned long long*>(ws);
  Bt.list_count = reinterpret_cast<unsigned long long*>(ws) + 1;
  Bt.blk_list = reinterpret_cast<uint4*>(ws + L.list);
  Bt.blk_cap = L.list_cap;
  Bt.cand = reinterpret_cast<uint4*>(ws + L.cand);
  Bt.cand_cap = L.cand_cap;
  Bt.cand_count = reinterpret_cast<unsigned long long*>(ws) + 3;
  Bt.list_done = reinterpret_cast<unsigned long long*>(ws) + 5;
  Bt.cand_done = reinterpret_cast<unsigned long long*>(ws) + 6;
  Timing tm;
  if (o->timing) {
    CUDA_TRY(cudaEventCreate(&tm.e0));
    CUDA_TRY(cudaEventCreate(&tm.e1));
    CUDA_TRY(cudaEventRecord(tm.e0, stream));
  }
  std::vector<uint64_t> prefix;
  int rc = spec ? launch_cull<KIND_SPEC>(T, Bt, prefix, ws + L.table, o->device, stream)
                 : (o->mode == MCX_MODE_BRUTE || pf_as_brute)
                     ? launch_brute<KIND_TRI>(T, Bt, prefix, ws + L.table, o->device, stream)
                 : o->mode == MCX_MODE_CULL ? launch_cull<KIND_TRI>(T, Bt, prefix, ws + L.table, o->device, stream)
                                            : launch_prefilter(T, Bt, prefix, ws + L.table, jobs, ws + L.jobs,
                                                               o->device, stream);
  if (rc != MCX_OK) return rc;
  if (Bt.tasks) {  // the solve stage also ORs the tasks' non-finite flags into the header
    Bt.status_flag = reinterpret_cast<unsigned long long*>(ws) + 2;
    rc = spec ? launch_solve<KIND_SPEC>(Bt, o->device, stream) : launch_solve<KIND_TRI>(Bt, o->device, stream);
    if (rc != MCX_OK) return rc;
    dstamp(stream, "    solve done");
  } else {  // no work units → no table upload by a launcher: check the flags directly
    CUDA_TRY(h2d_async(ws + L.table, T.data(), sizeof(SearchParams) * n, stream));
    status_kernel<<<1, 32, 0, stream>>>(reinterpret_cast<const SearchParams*>(ws + L.table), n,
                                        reinterpret_cast<unsigned long long*>(ws) + 2);
    CUDA_TRY(cudaGetLastError());
  }
  if (step) {  // the next step starts where this one's lists end
    mark_done_kernel<<<1, 1, 0, stream>>>(reinterpret_cast<unsigned long long*>(ws));
    CUDA_TRY(cudaGetLastError());
  }
  if (o->timing) CUDA_TRY(cudaEventRecord(tm.e1, stream));
  if (h_counters) {  // asynchronous: the caller synchronises and calls batch_stats
    if (!header_later)
      CUDA_TRY(cudaMemcpyAsync(h_counters, ws, sizeof(unsigned long long) * (8 + 8ull * n), cudaMemcpyDeviceToHost,
                               stream));
    return MCX_OK;
  }
  std::vector<unsigned long long> h(8 + 8ull * n);
  CUDA_TRY(cudaMemcpyAsync(h.data(), ws, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  float ms = 0.f;
  if (o->timing) CUDA_TRY(cudaEventElapsedTime(&ms, tm.e0, tm.e1));
  return batch_stats(h.data(), n, o, cap, st, ms);
}

// Quad AABBs of a half-layer grid: quad q = i + N·k1 over vertices v00 v10 v01 v11.
__global__ void quad_box_kernel(const double* __restrict__ coords, uint32_t N, uint32_t M, Box* __restrict__ box) {
  const uint64_t nq = (uint64_t)N * (M - 1);
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(q % N), k = (uint32_t)(q / N);
    const uint32_t ip = (i + 1 == N) ? 0 : i + 1;
    Box b;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double* pl = coords + (uint64_t)c * M * N;
      const double w00 = pl[(uint64_t)k * N + i], w10 = pl[(uint64_t)k * N + ip];
      const double w01 = pl[(uint64_t)(k + 1) * N + i], w11 = pl[(uint64_t)(k + 1) * N + ip];
      b.lo[c] = fmin(fmin(fmin(w00, w10), w01), w11);
      b.hi[c] = fmax(fmax(fmax(w00, w10), w01), w11);
    }
    box[q] = b;
  }
}

// pair_candidates workspace header: counters (128 B) + one task table entry + prefix.
constexpr uint64_t PC_HEADER = 1024;
static_assert(256 + sizeof(SearchParams) + 16 <= PC_HEADER, "pair_candidates header too small");

static int launch_pair_candidates(const double* cA, uint32_t NA, uint32_t MA, const double* cB, uint32_t NB,
                                  uint32_t MB, int device, cudaStream_t stream, void* ws, uint64_t ws_bytes,
                                  uint64_t* gids, uint64_t cap, mcx_stats* st) {
  if (NA < 1 || NB < 1 || MA < 2 || MB < 2) return set_error(MCX_E_ARG, "half-layers need >= 2 columns");
  const uint64_t nqA = (uint64_t)NA * (MA - 1), nqB = (uint64_t)NB * (MB - 1);
  if (nqA >= (1ull << 31) || nqB >= (1ull << 31)) return set_error(MCX_E_ARG, "quad counts must be < 2^31");
  const uint64_t need = PC_HEADER + (nqA + nqB) * sizeof(Box);
  if (!ws || ws_bytes < need + 16 || ((uintptr_t)ws & 15))
    return set_error(MCX_E_ARG, "workspace too small or misaligned (need %llu bytes + 16 per candidate)",
                     (unsigned long long)need);
  if (cap > 0 && !gids) return set_error(MCX_E_ARG, "null gid buffer with nonzero capacity");
  unsigned long long* counters = (unsigned long long*)ws;
  Box* boxA = reinterpret_cast<Box*>((char*)ws + PC_HEADER);
  Box* boxB = boxA + nqA;
  CUDA_TRY(cudaMemsetAsync(counters, 0, 16 * sizeof(unsigned long long), stream));
  quad_box_kernel<<<(unsigned)min((nqA + 255) / 256, (uint64_t)148 * 64), 256, 0, stream>>>(cA, NA, MA, boxA);
  quad_box_kernel<<<(unsigned)min((nqB + 255) / 256, (uint64_t)148 * 64), 256, 0, stream>>>(cB, NB, MB, boxB);
  CUDA_TRY(cudaGetLastError());
  SearchParams P = {};
  P.boxA = boxA;
  P.boxB = boxB;
  P.nA = nqA;
  P.a_begin = 0;
  P.a_end = nqA;
  P.blk_first = 0;
  P.my_blocks = (nqA + A_BLOCK - 1) / A_BLOCK;
  P.nB = nqB;
  P.ntilesB = (nqB + TILE - 1) / TILE;
  P.shard_count = 1;
  P.counters = counters + 8;
  P.coordsA = cA;
  P.coordsB = cB;
  P.NA = NA; P.MA = MA; P.NB = NB; P.MB = MB;
  P.MpA = MA; P.MpB = MB;
  Batch Bt = {};
  Bt.n_tasks = 1;
  Bt.gids = gids;
  Bt.cap = cap;
  Bt.emit = counters;
  Bt.cand_count = counters + 3;
  Bt.cand = reinterpret_cast<uint4*>((char*)ws + need);
  Bt.cand_cap = (ws_bytes - need) / 16;
  std::vector<SearchParams> T(1, P);
  std::vector<uint64_t> prefix;
  int rc = launch_brute<KIND_QUAD>(T, Bt, prefix, (char*)ws + 256, device, stream);
  if (rc == MCX_OK && Bt.tasks) rc = launch_solve<KIND_QUAD>(Bt, device, stream);
  if (rc != MCX_OK) return rc;
  unsigned long long h[16];
  CUDA_TRY(cudaMemcpyAsync(h, counters, sizeof(h), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  *st = mcx_stats{};
  st->n_pairs = nqA * nqB;
  st->n_tested = st->n_exact_tests = nqA * nqB;
  st->n_aabb_pass = h[8 + 1];
  st->n_singular = h[8 + 2];  // Moller-rejected quad pairs
  st->n_hits = st->n_candidates = h[8 + 0];
  if (h[3] > Bt.cand_cap)
    return set_error(MCX_E_CAPACITY, "workspace holds %llu quad-box survivors, %llu needed (16 B each)",
                     (unsigned long long)Bt.cand_cap, h[3]);
  if (h[0] > cap) return set_error(MCX_E_CAPACITY, "candidate capacity %llu < %llu", (unsigned long long)cap, h[0]);
  return MCX_OK;
}

// SPEC-literal pair_candidates over packed meshes with exact culling (quads = record
// pairs); same survivor set and counters as launch_pair_candidates.
static int launch_pair_candidates_mesh(const mcx_mesh_dev* A, const mcx_mesh_dev* B, const mcx_opts* o, uint64_t* gids,
                                       uint64_t cap, mcx_stats* st) {
  if (!A || !B || !o || !st) return set_error(MCX_E_ARG, "null argument");
  if (!A->coords || !B->coords || !A->box || !B->box) return set_error(MCX_E_ARG, "null mesh buffer");
  if (A->M < 2 || B->M < 2 || A->n_tri != 2ull * A->N * (A->M - 1) || B->n_tri != 2ull * B->N * (B->M - 1))
    return set_error(MCX_E_ARG, "mesh record counts do not match the grids");
  const double *cA = A->coords, *cB = B->coords;
  const uint32_t NA = A->N, MA = A->M, NB = B->N, MB = B->M;
  if (!A->gbox || !A->bbox || !B->gbox || !B->tbox) return set_error(MCX_E_ARG, "meshes need level boxes");
  if (cap > 0 && !gids) return set_error(MCX_E_ARG, "null gid buffer with nonzero capacity");
  const uint32_t scount = o->shard_count ? o->shard_count : 1;
  if (o->shard_index >= scount) return set_error(MCX_E_ARG, "shard_index >= shard_count");
  mcx_opts oc = *o;
  oc.mode = MCX_MODE_CULL;
  mcx_task t = {A, B, 0, 0};
  const WsLayout L = ws_layout(&t, 1, &oc);
  if (!o->workspace || o->workspace_bytes < L.total || ((uintptr_t)o->workspace & 15))
    return set_error(MCX_E_ARG, "workspace too small or misaligned (need %llu bytes)", (unsigned long long)L.total);
  cudaStream_t stream = (cudaStream_t)o->stream;
  char* ws = (char*)o->workspace;
  const ShardGeom g = shard_geom(0, A->n_tri, o->shard_index, scount);
  std::vector<SearchParams> T(1);
  SearchParams& P = T[0];
  P = SearchParams{};
  P.boxA = reinterpret_cast<const Box*>(A->box);
  P.permA = A->perm;
  P.boxB = reinterpret_cast<const Box*>(B->box);
  P.permB = B->perm;
  P.nA = A->n_tri;
  P.a_begin = 0;
  P.a_end = A->n_tri;
  P.blk_first = g.first;
  P.my_blocks = g.my_blocks;
  P.nB = B->n_tri;
  P.ntilesB = (B->n_tri + TILE - 1) / TILE;
  P.shard_count = scount;
  P.counters = reinterpret_cast<unsigned long long*>(ws + L.counters);
  P.gboxA = reinterpret_cast<const Box*>(A->gbox);
  P.bboxA = reinterpret_cast<const Box*>(A->bbox);
  P.gboxB = reinterpret_cast<const Box*>(B->gbox);
  P.tboxB = reinterpret_cast<const Box*>(B->tbox);
  P.statusA = A->status;
  P.statusB = B->status;
  P.coordsA = cA;
  P.coordsB = cB;
  P.NA = NA; P.MA = MA; P.NB = NB; P.MB = MB;
  P.MpA = A->plane_rows ? A->plane_rows : MA;
  P.MpB = B->plane_rows ? B->plane_rows : MB;
  *st = mcx_stats{};
  st->n_pairs = (g.na / 2) * (B->n_tri / 2);  // quad pairs
  CUDA_TRY(cudaMemsetAsync(ws, 0, L.counters + 64, stream));
  Batch Bt = {};
  Bt.n_tasks = 1;
  Bt.gids = gids;
  Bt.cap = cap;
  Bt.emit = reinterpret_cast<unsigned long long*>(ws);
  Bt.list_count = reinterpret_cast<unsigned long long*>(ws) + 1;
  Bt.blk_list = reinterpret_cast<uint4*>(ws + L.list);
  Bt.blk_cap = L.list_cap;
  Bt.cand = reinterpret_cast<uint4*>(ws + L.cand);
  Bt.cand_cap = L.cand_cap;
  Bt.cand_count = reinterpret_cast<unsigned long long*>(ws) + 3;
  Bt.list_done = reinterpret_cast<unsigned long long*>(ws) + 5;
  Bt.cand_done = reinterpret_cast<unsigned long long*>(ws) + 6;
  Timing tm;
  if (o->timing) {
    CUDA_TRY(cudaEventCreate(&tm.e0));
    CUDA_TRY(cudaEventCreate(&tm.e1));
    CUDA_TRY(cudaEventRecord(tm.e0, stream));
  }
  std::vector<uint64_t> prefix;
  int rc = launch_cull<KIND_QUAD>(T, Bt, prefix, ws + L.table, o->device, stream);
  if (rc == MCX_OK && Bt.tasks) rc = launch_solve<KIND_QUAD>(Bt, o->device, stream);
  if (rc != MCX_OK) return rc;
  if (o->timing) CUDA_TRY(cudaEventRecord(tm.e1, stream));
  status_kernel<<<1, 32, 0, stream>>>(reinterpret_cast<const SearchParams*>(ws + L.table), 1,
                                      reinterpret_cast<unsigned long long*>(ws) + 2);
  CUDA_TRY(cudaGetLastError());
  unsigned long long h[16];
  CUDA_TRY(cudaMemcpyAsync(h, ws, sizeof(h), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  const unsigned long long* c = h + 8;
  st->n_hits = c[0];
  st->n_aabb_pass = c[1];
  st->n_singular = c[2];  // Moller-rejected quad pairs
  st->n_tested = c[3];
  st->n_exact_tests = c[3];
  st->n_candidates = c[0];
  if (o->timing) {
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, tm.e0, tm.e1));
    st->kernel_ms = ms;
  }
  if (h[2]) return set_error(MCX_E_ARG, "non-finite (NaN/Inf) coordinates in an input mesh (mcx_pack status)");
  if (h[3] > L.cand_cap)
    return set_error(MCX_E_CAPACITY, "candidate-list capacity %llu < %llu quad-box survivors (opts->cand_cap)",
                     (unsigned long long)L.cand_cap, h[3]);
  if (c[0] > cap) return set_error(MCX_E_CAPACITY, "candidate capacity %llu < %llu", (unsigned long long)cap, c[0]);
  return MCX_OK;
}

thread_local char g_err[512] = "";
thread_local HostStage* g_stage = nullptr;

}  // namespace mcx

extern "C" {

uint32_t mcx_a_block(void) { return mcx::A_BLOCK; }

uint64_t mcx_workspace_bytes(const mcx_mesh_dev* A, const mcx_mesh_dev* B, const mcx_opts* o) {
  mcx_task t = {A, B, o ? o->a_begin : 0, o ? o->a_end : 0};
  return mcx::ws_layout(&t, 1, o).total;
}

uint64_t mcx_batch_workspace_bytes(const mcx_task* tasks, uint32_t n_tasks, const mcx_opts* o) {
  if (!tasks) return 0;
  return mcx::ws_layout(tasks, n_tasks, o).total;
}

int mcx_search(const mcx_mesh_dev* A, const mcx_mesh_dev* B, const mcx_opts* o, mcx_hit* hits, uint64_t cap,
               mcx_stats* st) {
  using namespace mcx;
  if (!A || !B || !o || !st) return set_error(MCX_E_ARG, "null argument");
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(o->device));
  mcx_task t = {A, B, o->a_begin, o->a_end};
  return launch_batch(&t, 1, o, hits, nullptr, cap, st, nullptr);
}

int mcx_search_batch(const mcx_task* tasks, uint32_t n_tasks, const mcx_opts* o, mcx_hit* hits, uint32_t* hit_task,
                     uint64_t cap, mcx_stats* stats) {
  using namespace mcx;
  if (!o) return set_error(MCX_E_ARG, "null options");
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(o->device));
  return launch_batch(tasks, n_tasks, o, hits, hit_task, cap, stats, nullptr);
}

int mcx_pair_candidates(const double* coords_a, uint32_t NA, uint32_t MA, const double* coords_b, uint32_t NB,
                        uint32_t MB, int device, void* stream, void* workspace, uint64_t workspace_bytes,
                        uint64_t* gids, uint64_t cap, mcx_stats* stats) {
  using namespace mcx;
  if (!coords_a || !coords_b || !stats) return set_error(MCX_E_ARG, "null argument");
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(device));
  return launch_pair_candidates(coords_a, NA, MA, coords_b, NB, MB, device, (cudaStream_t)stream, workspace,
                                workspace_bytes, gids, cap, stats);
}

int mcx_pair_candidates_mesh(const mcx_mesh_dev* A, const mcx_mesh_dev* B, const mcx_opts* opts, uint64_t* gids,
                             uint64_t cap, mcx_stats* stats) {
  using namespace mcx;
  if (!opts) return set_error(MCX_E_ARG, "null options");
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(opts->device));
  return launch_pair_candidates_mesh(A, B, opts, gids, cap, stats);
}

uint64_t mcx_pair_candidates_mesh_workspace_bytes(const mcx_mesh_dev* A, const mcx_mesh_dev* B, const mcx_opts* o) {
  if (!A || !B || !o) return 0;
  mcx_opts oc = *o;
  oc.mode = MCX_MODE_CULL;
  mcx_task t = {A, B, 0, 0};
  return mcx::ws_layout(&t, 1, &oc).total;
}

const char* mcx_last_error(void) { return mcx::g_err; }

int mcx_version(void) { return MCX_ABI_VERSION; }

}  // extern "C"
