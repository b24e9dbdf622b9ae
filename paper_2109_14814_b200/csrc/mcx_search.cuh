// mcx_search.cuh — types and device/host helpers shared by the search kernels
// (mcx_search.cu: FP64 brute force + culling; mcx_prefilter.cuh: prefilter mode).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "../../include/mcx.h"
#include "mcx_common.cuh"
#include "mcx_internal.cuh"

namespace mcx {

constexpr int STAGES = 2;

// Kernel variant: R A triangles per thread, MINB resident CTAs per SM (register cap).
template <int R_, int MINB_, int JB_ = 1, int UNROLL_ = 2, int PF_ = 0>
struct Cfg {
  static constexpr int PF = PF_;             // prefetch the next B box before testing the current
  static constexpr int R = R_;
  static constexpr int MINB = MINB_;
  static constexpr int JB = JB_;             // B triangles per warp vote
  static constexpr int UNROLL = UNROLL_;     // inner-loop unroll
  static constexpr int THREADS = A_BLOCK / R_;
  static constexpr int WARPS = THREADS / 32;
  static constexpr int QCAP = 32 * R_ * JB_ + 32;  // per-warp survivor queue capacity
};

// What a box-test survivor (candidate) is and what the solve stage does with it:
//  KIND_TRI  — (storage A record, storage B record): precise test → triangle hit;
//  KIND_QUAD — (A quad, B quad), original quad indices: Moller → quad-pair gid
//              (SPEC pair_candidates);
//  KIND_SPEC — (A quad, B quad): Moller, then the 4 triangle-pair precise tests of
//              each candidate → triangle hits (SPEC find_intersections).
enum Kind { KIND_TRI = 0, KIND_QUAD = 1, KIND_SPEC = 2 };

// Per-task parameters (one entry of the device task table; a single search is a
// batch of one).  Pointers are device pointers.
struct __align__(16) SearchParams {
  const Box* boxA;
  const uint32_t* permA;    // storage → original index (NULL = identity)
  const Box* boxB;
  const uint32_t* permB;
  uint64_t nA;
  uint64_t a_begin, a_end;  // A storage range
  uint64_t blk_first;       // first absolute A block of this shard
  uint64_t my_blocks;       // A blocks of this shard
  uint64_t nB;
  uint64_t b_chunk, nchunk; // brute: B triangles per CTA (multiple of TILE), chunks
  uint64_t ntilesB;
  uint32_t shard_count, task;
  uint32_t swapped;  // MCX_ORIENT_LARGER_A exchanged the roles: "A" here is the caller's B
  // per task: [0] emitted, [1] aabb pass, [2] singular (KIND_QUAD: Moller-rejected), [3] tested,
  // [4] KIND_SPEC: Moller survivors (candidates)
  unsigned long long* counters;
  // MCX_MODE_CULL
  const Box* gboxA;
  const Box* bboxA;
  const Box* gboxB;
  const Box* tboxB;
  const uint32_t* statusA;  // mcx_pack non-finite flags (may be NULL)
  const uint32_t* statusB;
  // half-layer grids (4, M, N): the solve rebuilds triangle geometry from them; Moller
  const double* coordsA;
  const double* coordsB;
  uint32_t NA, MA, NB, MB;
  uint32_t MpA, MpB;  // plane strides in rows (the parent grid's M for a column view)
  // MCX_MODE_PREFILTER only: conservative fp32 boxes {lo_rd[4]}, {hi_ru[4]} per record
  float4* fA;
  float4* fB;
};

// MCX_MODE_PREFILTER: conservative fp32 boxes of one distinct mesh of the batch.
struct FboxJob {
  const Box* src;
  float4* dst;  // [n][2]: lo rounded toward −∞, hi toward +∞
  uint64_t n;
};

// Whole-launch parameters: the task table and the shared outputs.
struct Batch {
  const SearchParams* tasks;
  uint32_t n_tasks;
  const uint64_t* prefix;        // [n_tasks + 1] exclusive prefix of per-task work units
  mcx_hit* hits;                 // KIND_TRI output (original indices)
  uint32_t* hit_task;            // task id of each hit (NULL: single task)
  uint64_t* gids;                // KIND_QUAD output
  uint64_t cap;
  unsigned long long* emit;      // shared output position counter
  unsigned long long* status_flag;  // header word: any task's mesh has non-finite coordinates
  uint4* cand;                   // box-test survivors {A index, B index, task, 0} (compacted)
  uint64_t cand_cap;
  unsigned long long* cand_count;
  uint4* blk_list;               // cull: overlapping (task, local A block, B tile)
  uint64_t blk_cap;
  unsigned long long* list_count;
  // entries [*list_done, *list_count) / [*cand_done, *cand_count) are this launch's work
  // (header words 5 / 6: nonzero only in the later steps of a stepped batch)
  const unsigned long long* list_done;
  const unsigned long long* cand_done;
  uint32_t neg1;                 // 0xffffffff, a runtime operand so the packed subtract stays an IMAD
  const struct FboxJob* fjobs;   // MCX_MODE_PREFILTER: one fp32-box conversion per distinct mesh
  uint32_t n_fjobs;
  uint32_t cull_ychunks;         // cull level 1: B tile chunks per unit ...
  uint64_t cull_ychunk;          // ... of this many tiles
  uint64_t cull_items;           // level-1 work items (units × chunks; known on the host)
};

// Task owning work unit u: the last t with prefix[t] <= u (n_tasks is small).
__device__ __forceinline__ uint32_t find_task(const Batch& Bt, uint64_t u) {
  uint32_t lo = 0, hi = Bt.n_tasks - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (__ldg(Bt.prefix + mid) <= u) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <class C>
struct __align__(16) SearchSmem {
  Box tile[STAGES][TILE];
  uint2 queue[C::WARPS][C::QCAP];
  unsigned long long full[STAGES];
};

__device__ __forceinline__ bool box_overlap(const Box& a, const Box& b) {
  return (b.lo[0] <= a.hi[0]) & (a.lo[0] <= b.hi[0]) & (b.lo[1] <= a.hi[1]) & (a.lo[1] <= b.hi[1]) &
         (b.lo[2] <= a.hi[2]) & (a.lo[2] <= b.hi[2]) & (b.lo[3] <= a.hi[3]) & (a.lo[3] <= b.hi[3]);
}

__device__ __forceinline__ void empty_box(double lo[4], double hi[4]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    lo[c] = __longlong_as_double(0x7ff0000000000000ll);  // +inf: never overlaps
    hi[c] = -lo[c];
  }
}

// Stage 2 (compaction, Fig. 1): append this warp's queued box-test
// survivors [0, n) to the global candidate list — one atomic per 32 survivors,
// one coalesced 16-byte store per lane.  The count keeps running past cand_cap so
// the host learns the exact size to regrow to.
__device__ __forceinline__ void flush_queue(const SearchParams& P, const Batch& Bt, const uint2* q, int n,
                                            int lane) {
  unsigned long long base = 0;
  if (lane == 0) {
    base = atomicAdd(Bt.cand_count, (unsigned long long)n);
    atomicAdd(P.counters + 1, (unsigned long long)n);
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  if (lane < n && base + lane < Bt.cand_cap) {
    const uint2 e = q[lane];
    Bt.cand[base + lane] = make_uint4(e.x, e.y, P.task, 0u);
  }
  __syncwarp();
}

// Append this warp's accepted triangle hits (ballot + one atomic per warp for the
// output position; per-lane task counters, hits are rare).
__device__ __forceinline__ void emit_hits(const Batch& Bt, bool hit, uint32_t ia, uint32_t ib, const double sol[4],
                                          uint32_t task, unsigned long long* task_counters, int lane) {
  const unsigned hm = __ballot_sync(0xffffffffu, hit);
  if (!hm) return;
  const int leader = __ffs(hm) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(Bt.emit, (unsigned long long)__popc(hm));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (hit) {
    atomicAdd(task_counters + 0, 1ull);
    const unsigned long long pos = base + __popc(hm & ((1u << lane) - 1u));
    if (pos < Bt.cap) {
      mcx_hit h;
      h.ia = ia;
      h.ib = ib;
      h.s = sol[0]; h.t = sol[1]; h.a = sol[2]; h.b = sol[3];
      Bt.hits[pos] = h;
      if (Bt.hit_task) Bt.hit_task[pos] = task;
    }
  }
}

// Stage 3 (the precise test, PAPER.md "Precise Test"): one
// thread per candidate at full occupancy, apart from the compare-bound sweep kernels
// so their register budget holds only the box tests.
template <int KIND>
__global__ void __launch_bounds__(256) solve_kernel(const Batch Bt) {
  const uint64_t n = min((uint64_t)*(volatile unsigned long long*)Bt.cand_count, Bt.cand_cap);
  const uint64_t k0 = Bt.cand_done ? min((uint64_t)*Bt.cand_done, n) : 0;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x < 32 && Bt.status_flag) {
    // OR of every task's mcx_pack non-finite flags into the header (no separate launch)
    unsigned v = 0;
    for (uint32_t t = threadIdx.x; t < Bt.n_tasks; t += 32) {
      if (Bt.tasks[t].statusA) v |= *Bt.tasks[t].statusA;
      if (Bt.tasks[t].statusB) v |= *Bt.tasks[t].statusB;
    }
    if (__any_sync(0xffffffffu, v != 0) && threadIdx.x == 0) atomicOr(Bt.status_flag, 1ull);
  }
  if constexpr (KIND == KIND_SPEC) {
    // "for each surviving gid, runs all 4 triangle-pair precise tests": one
    // thread per (candidate, test) — the 4 solves of a quad pair run side by side instead of
    // as one thread's dependent chain (the stage is latency-bound: C3 has ~200 candidates);
    // each of the 4 threads runs the (identical) Moller test, the first counts it
    const uint64_t items = 4 * (n - k0);
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < items; base += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t it = base + threadIdx.x;
      const bool valid = it < items;
      const int v = (int)(it & 3);
      const uint4 c = valid ? Bt.cand[k0 + (it >> 2)] : make_uint4(0u, 0u, 0u, 0u);
      const SearchParams& P = Bt.tasks[c.z];
      const double* cA = P.swapped ? P.coordsB : P.coordsA;
      const double* cB = P.swapped ? P.coordsA : P.coordsB;
      const uint32_t NA = P.swapped ? P.NB : P.NA, MA = P.swapped ? P.MpB : P.MpA;
      const uint32_t NB = P.swapped ? P.NA : P.NB, MB = P.swapped ? P.MpA : P.MpB;
      const uint32_t qa = P.swapped ? c.y : c.x, qb = P.swapped ? c.x : c.y;
      const bool cand = valid && !moller_reject(cA, NA, MA, qa, cB, NB, MB, qb);
      if (cand && v == 0) atomicAdd(P.counters + 4, 1ull);
      const uint32_t ia = 2 * qa + (v >> 1), ib = 2 * qb + (v & 1);
      double sol[4];
      int rc = 0;
      if (cand) {
        rc = solve_tri(cA, NA, MA, ia, cB, NB, MB, ib, sol);
        if (rc == 2) atomicAdd(P.counters + 2, 1ull);
      }
      emit_hits(Bt, rc == 1, ia, ib, sol, c.z, P.counters, lane);
    }
  } else {
  for (uint64_t base = k0 + blockIdx.x * (uint64_t)blockDim.x; base < n; base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = base + threadIdx.x;
    const bool valid = k < n;
    const uint4 c = valid ? Bt.cand[k] : make_uint4(0u, 0u, 0u, 0u);
    const SearchParams& P = Bt.tasks[c.z];
    // the caller's (A, B) roles: the sweep may have run them exchanged (P.swapped)
    const double* cA = P.swapped ? P.coordsB : P.coordsA;
    const double* cB = P.swapped ? P.coordsA : P.coordsB;
    const uint32_t NA = P.swapped ? P.NB : P.NA, MA = P.swapped ? P.MpB : P.MpA;  // MA/MB: plane rows
    const uint32_t NB = P.swapped ? P.NA : P.NB, MB = P.swapped ? P.MpA : P.MpB;
    if (KIND == KIND_TRI) {
      double sol[4];
      int rc = 0;
      uint32_t ia = 0, ib = 0;
      if (valid) {
        const uint32_t i1 = P.permA ? __ldg(P.permA + c.x) : c.x;
        const uint32_t i2 = P.permB ? __ldg(P.permB + c.y) : c.y;
        ia = P.swapped ? i2 : i1;
        ib = P.swapped ? i1 : i2;
        rc = solve_tri(cA, NA, MA, ia, cB, NB, MB, ib, sol);
        if (rc == 2) atomicAdd(P.counters + 2, 1ull);
      }
      emit_hits(Bt, rc == 1, ia, ib, sol, c.z, P.counters, lane);
    } else if (KIND == KIND_QUAD) {
      const bool cand = valid && !moller_reject(P.coordsA, P.NA, P.MpA, c.x, P.coordsB, P.NB, P.MpB, c.y);
      if (valid && !cand) atomicAdd(P.counters + 2, 1ull);
      const unsigned hm = __ballot_sync(0xffffffffu, cand);
      if (hm) {
        const int leader = __ffs(hm) - 1;
        unsigned long long pos0 = 0;
        if (lane == leader) pos0 = atomicAdd(Bt.emit, (unsigned long long)__popc(hm));
        pos0 = __shfl_sync(0xffffffffu, pos0, leader);
        const unsigned long long pos = pos0 + __popc(hm & ((1u << lane) - 1u));
        if (cand) {
          atomicAdd(P.counters + 0, 1ull);
          atomicAdd(P.counters + 4, 1ull);
          if (pos < Bt.cap) {
            // quad indices qa = i + N1·k1, qb = j + N2·l1 → gid (PAPER.md kernel step 2)
            const uint64_t i = c.x % P.NA, k1 = c.x / P.NA, j = c.y % P.NB, l1 = c.y / P.NB;
            const uint64_t n12 = (uint64_t)P.NA * P.NB;
            Bt.gids[pos] = i + (uint64_t)P.NA * j + n12 * k1 + n12 * (uint64_t)(P.MA - 1) * l1;
          }
        }
      }
    }
  }
  }
}

// Per-task count of executed box tests (cull: pair tests; prefilter: exact FP64 box tests).
__device__ __forceinline__ void flush_tested(const SearchParams& P, int lane, unsigned long long n_tested) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n_tested += __shfl_xor_sync(0xffffffffu, n_tested, o);
  if (lane == 0 && n_tested) atomicAdd(P.counters + 3, n_tested);
}

// --------------------------------------------------------------- host side
// B chunk count for one task: every CTA of a task does the same work, so pick the
// count whose CTA total best fills whole waves of resident CTAs (the last partial
// wave idles the rest of the GPU), among counts giving >= 8 waves with chunks of
// >= min_tiles tiles (1 tile for small problems).
static void choose_chunks(SearchParams& P, uint64_t slots, uint64_t min_tiles = 16, uint64_t tile = TILE) {
  const uint64_t max_chunks = (P.nB + tile - 1) / tile;
  uint64_t nchunk = 1, chunk = max_chunks * tile;
  const uint64_t min_ch = (P.my_blocks * max_chunks < 8 * slots) ? tile : min_tiles * tile;
  double best = -1.0;
  for (uint64_t c = 1; c <= max_chunks && c <= 4096; ++c) {
    const uint64_t ch = ((P.nB + c - 1) / c + tile - 1) / tile * tile;
    const uint64_t nc = (P.nB + ch - 1) / ch;
    if (nc != c) continue;
    const uint64_t total = P.my_blocks * nc;
    const bool enough = total >= 8 * slots || nc == max_chunks;
    if (!enough && c < max_chunks && ch > min_ch) continue;
    const double eff = (double)total / (double)(((total + slots - 1) / slots) * slots);
    if (eff > best + 1e-3) {
      best = eff;
      nchunk = nc;
      chunk = ch;
    }
    if (best > 0.995 || ch <= min_ch) break;
  }
  P.nchunk = nchunk;
  P.b_chunk = chunk;
}

// Chunk every task for `slots` resident CTAs, build the per-task prefix of work units
// and upload the task table + prefix to dev_tab (stream-ordered).  *total = CTAs to
// launch; Bt's table pointers are set.  Shared by the brute and prefilter launchers.
static int upload_plan(std::vector<SearchParams>& T, Batch& Bt, std::vector<uint64_t>& prefix, void* dev_tab,
                       uint64_t slots, uint64_t min_tiles, cudaStream_t stream, uint64_t* total,
                       uint64_t tile = TILE) {
  prefix.assign(T.size() + 1, 0);
  for (size_t t = 0; t < T.size(); ++t) {
    if (T[t].my_blocks && T[t].nB) choose_chunks(T[t], slots, min_tiles, tile); else T[t].nchunk = 0;
    prefix[t + 1] = prefix[t] + T[t].my_blocks * T[t].nchunk;
  }
  *total = prefix.back();
  const size_t tab = sizeof(SearchParams) * T.size();
  CUDA_TRY(h2d_async(dev_tab, T.data(), tab, stream));
  CUDA_TRY(h2d_async((char*)dev_tab + tab, prefix.data(), sizeof(uint64_t) * prefix.size(), stream));
  if (*total > 0x7fffffffull) return set_error(MCX_E_ARG, "grid too large");
  Bt.tasks = reinterpret_cast<const SearchParams*>(dev_tab);
  Bt.prefix = reinterpret_cast<const uint64_t*>((char*)dev_tab + tab);
  return MCX_OK;
}

// Resident CTAs of `kernel` on the whole device (at least one per SM).
template <class K>
static int resident_slots(K kernel, int threads, size_t smem, int device, uint64_t* slots) {
  return kernel_prepare(reinterpret_cast<const void*>(kernel), threads, smem, -1, device, slots);
}

// Variant selection (MCX_VARIANT=0..3, for experiments; 0 = the tuned default:
// R = 4, 256 threads, 2 CTAs/SM, next B box prefetched from shared memory before
// the current one's compares, unroll 4 — no spills).
static int variant_from_env() {
  const char* v = getenv("MCX_VARIANT");
  return v ? atoi(v) : 0;
}

}  // namespace mcx
