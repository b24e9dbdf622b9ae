// mcx_runtime.cu — the host-to-host runtime of libmcx.so: the reference's
// find_intersections and layer-pair task loop as one
// call per job, everything after the H2D copy on the device.
//
//   mcx_mesh_load      H2D of a half-layer grid + s-values, fused pack (mcx_pack.cu)
//   mcx_intersect      1. batched search of all jobs (mcx_search.cu: box tests →
//                         candidate compaction → precise test), hits stay in HBM
//                      2. record keys: gid, τ_A, τ_B per hit
//                      3. sort by (job, gid, τ_A, τ_B)  (CUB radix sort: stable,
//                         LSD — (gid, τ) first, then job)
//                      4. record fields in that order (mcx_records.cuh: point,
//                         Eqs. 28-29 estimates), 128-byte mcx_record each
//                      5. 1e-9 dedup: close pairs from an x-sorted
//                         window scan, then the greedy rule resolved in rounds
//                      6. compaction of the kept records and the "%.17g" records
//                         text (mcx_format.cuh), both in record order
//                      7. D2H of the records and the text into pinned host memory
//   mcx_find_intersections   load A (stream 0) and B (stream 1, overlapping A's
//                      packing), mcx_intersect, release.
//
// Dedup contract (identical to isect._dedup_mask on the host): in record order, a
// record is dropped iff some KEPT earlier record of the same job has a point within
// 1e-9 in every coordinate (|fl(p − q)| ≤ 1e-9).  The greedy rule is resolved in
// rounds: a record with a kept close predecessor is dropped; a record whose close
// predecessors are all dropped is kept; the smallest undecided record is decided in
// every round, so the rounds terminate and give the sequential answer.
//
// Device memory comes from a per-context CUDA memory pool (stream-ordered
// cudaMallocFromPoolAsync, release threshold "never"), so repeated calls reuse it.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <vector>

#include <cooperative_groups.h>
#include <immintrin.h>

#include "../../include/mcx.h"
#include "mcx_common.cuh"
#include "mcx_format.cuh"
#include "mcx_internal.cuh"
#include "mcx_records.cuh"

#define MCX_DEDUP_TOL 1e-9

namespace cg = cooperative_groups;

namespace mcx {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

// Per-job parameters of the records stage (device table).
struct JobDev {
  const double* cA;
  const double* sA;
  const double* sB;
  uint32_t NA, MA, NB, MB;
  int32_t n1, sign1, n2, sign2;
  uint32_t MpA, pad;  // plane stride of A's grid in rows
};

// Pageable uploads (NumPy arrays): the driver stages a pageable cudaMemcpy through its
// own pinned buffer with one thread, ~12 GB/s on these hosts (97 MB in 8.1 ms, pinned
// 1.8 ms).  StagePool copies pageable bytes into a ring of pinned slots with several host
// threads while the previous slot's DMA runs.
// Copy into pinned staging memory with non-temporal stores: no read-for-ownership of the
// destination lines (host DRAM traffic 2 streams instead of 3) and the staged data does not
// evict the caches.  Falls back to memcpy without AVX2.
__attribute__((target("avx2"))) static void nt_copy_avx2(char* dst, const char* src, size_t n) {
  const size_t head = std::min(n, (size_t)((32 - ((uintptr_t)dst & 31)) & 31));
  memcpy(dst, src, head);
  dst += head; src += head; n -= head;
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256((const __m256i*)(src + i));
    const __m256i b = _mm256_loadu_si256((const __m256i*)(src + i + 32));
    const __m256i c = _mm256_loadu_si256((const __m256i*)(src + i + 64));
    const __m256i d = _mm256_loadu_si256((const __m256i*)(src + i + 96));
    _mm256_stream_si256((__m256i*)(dst + i), a);
    _mm256_stream_si256((__m256i*)(dst + i + 32), b);
    _mm256_stream_si256((__m256i*)(dst + i + 64), c);
    _mm256_stream_si256((__m256i*)(dst + i + 96), d);
  }
  memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}
static void stage_copy(char* dst, const char* src, size_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2") && !getenv("MCX_STAGE_MEMCPY");
  if (avx2 && n >= 4096) nt_copy_avx2(dst, src, n);
  else memcpy(dst, src, n);
}

struct StagePool {
  static constexpr int SLOTS = 3;
  static constexpr size_t SLOT_BYTES = 8u << 20;
  char* slot[SLOTS] = {};
  cudaEvent_t ev[SLOTS] = {};
  bool used[SLOTS] = {};
  int next = 0;
  // memcpy workers: job = up to 4 (src, len) segments gathered into dst, split in equal byte ranges
  std::vector<std::thread> th;
  std::mutex mu;
  std::condition_variable cv, done_cv;
  uint64_t gen = 0;
  int pending = 0;
  bool stop = false;
  const char* seg_src[4] = {};
  size_t seg_len[4] = {};
  int nseg = 0;
  char* dst = nullptr;
  size_t total = 0;
  int parts = 1;

  // copy bytes [lo, hi) of the gathered job
  void copy_range(size_t lo, size_t hi) {
    size_t off = 0;
    for (int k = 0; k < nseg && lo < hi; ++k) {
      const size_t a = std::max(lo, off), b = std::min(hi, off + seg_len[k]);
      if (a < b) stage_copy(dst + a, seg_src[k] + (a - off), b - a);
      off += seg_len[k];
    }
  }
  void worker(int id) {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return stop || gen != seen; });
      if (stop) return;
      seen = gen;
      const size_t lo = total * (size_t)id / parts, hi = total * (size_t)(id + 1) / parts;
      lk.unlock();
      copy_range(lo, hi);
      lk.lock();
      if (--pending == 0) done_cv.notify_one();
    }
  }
  void gather(char* d, const char* const* src, const size_t* len, int n) {
    size_t t = 0;
    for (int k = 0; k < n; ++k) t += len[k];
    if (th.empty()) {
      const unsigned hw = std::thread::hardware_concurrency();
      int nt = (int)std::min<unsigned>(8, hw > 2 ? hw / 2 : 1);
      if (const char* v = getenv("MCX_STAGE_THREADS")) nt = std::max(1, atoi(v));  // experiments
      for (int i = 1; i < nt; ++i) th.emplace_back(&StagePool::worker, this, i);
    }
    {
      std::lock_guard<std::mutex> lk(mu);
      for (int k = 0; k < n; ++k) { seg_src[k] = src[k]; seg_len[k] = len[k]; }
      nseg = n;
      dst = d;
      total = t;
      parts = (int)th.size() + 1;
      pending = (int)th.size();
      ++gen;
    }
    cv.notify_all();
    copy_range(0, t / parts);  // this thread's share
    std::unique_lock<std::mutex> lk(mu);
    done_cv.wait(lk, [&] { return pending == 0; });
  }
  ~StagePool() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    for (std::thread& t : th) t.join();
    for (int k = 0; k < SLOTS; ++k) {
      if (ev[k]) cudaEventDestroy(ev[k]);
      if (slot[k]) cudaFreeHost(slot[k]);
    }
  }
};

}  // namespace mcx

struct mcx_context {
  int device = 0;
  cudaStream_t s0 = nullptr, s1 = nullptr;
  cudaStream_t sc = nullptr;  // H2D copies of a chunked upload whose packs and searches run on s0
  cudaEvent_t ev = nullptr;
  cudaEvent_t cev[9] = {};  // chunk j copied (cev[8]: the allocations are made)
  cudaMemPool_t pool = nullptr;
  mcx::DevBuf ws, hits, hit_task, jobs, k0, k1, v0, v1, recs, recs_out, state, blocked, pairs, lens, offs, cub,
      text, small, flen, lines;
  mcx::HostBuf h_recs, h_text, h_small, h_counters;
  mcx::HostBuf h_map;    // mapped pinned memory the small-path kernel writes its results to
  mcx::HostStage stage;  // pinned staging of the per-call tables
  mcx::StagePool* up = nullptr;  // pinned staging ring for pageable grid uploads (lazy)
  uint64_t cand_cap = MCX_DEFAULT_CAND_CAP, hit_cap = 1 << 16, pair_cap = 1 << 12;
};

struct mcx_mesh {
  mcx_context* ctx = nullptr;
  bool owns_grid = true;  // false for a column view: coords / s_values belong to the parent
  double *coords = nullptr, *s_values = nullptr, *box = nullptr, *gbox = nullptr, *tbox = nullptr, *bbox = nullptr;
  uint32_t *perm = nullptr, *status = nullptr;
  mcx_mesh_dev view{};
};

namespace mcx {

static int ensure(mcx_context* c, DevBuf& b, size_t bytes, cudaStream_t s) {
  if (b.bytes >= bytes && b.p) return MCX_OK;
  if (b.p) CUDA_TRY(cudaFreeAsync(b.p, s));
  b.p = nullptr;
  b.bytes = 0;
  const size_t nb = std::max<size_t>(bytes + bytes / 2, 256);
  CUDA_TRY(cudaMallocFromPoolAsync(&b.p, nb, c->pool, s));
  b.bytes = nb;
  return MCX_OK;
}

static int ensure_host(HostBuf& b, size_t bytes) {
  if (b.bytes >= bytes && b.p) return MCX_OK;
  if (b.p) CUDA_TRY(cudaFreeHost(b.p));
  b.p = nullptr;
  b.bytes = 0;
  const size_t nb = std::max<size_t>(bytes + bytes / 2, 4096);
  CUDA_TRY(cudaMallocHost(&b.p, nb));
  b.bytes = nb;
  return MCX_OK;
}

static void release(mcx_context* c, DevBuf& b, cudaStream_t s) {
  if (b.p) cudaFreeAsync(b.p, s);
  b.p = nullptr;
  b.bytes = 0;
}

// Sources of at least this many bytes that are not page-locked go through the StagePool.
constexpr size_t STAGE_MIN_BYTES = 2u << 20;
static bool pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// H2D of `height` rows of `width` bytes (host pitch spitch, device pitch dpitch) on cs.
// Pageable sources: pieces of the rows gathered into pinned slots by the pool's threads,
// each slot's 2-D copy issued as soon as it is filled, a slot reused once its copy is done.
static cudaError_t h2d_rows(mcx_context* c, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                            size_t height, cudaStream_t cs, bool stage) {
  if (!stage || width * height < STAGE_MIN_BYTES || height > 4)
    return height == 1 ? cudaMemcpyAsync(dst, src, width, cudaMemcpyHostToDevice, cs)
                       : cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice, cs);
  if (!c->up) c->up = new StagePool();
  StagePool& P = *c->up;
  const size_t wp = (StagePool::SLOT_BYTES / height) & ~(size_t)15;  // piece width
  for (size_t w0 = 0; w0 < width; w0 += wp) {
    const size_t w = std::min(wp, width - w0);
    const int k = P.next;
    P.next = (k + 1) % StagePool::SLOTS;
    cudaError_t e = cudaSuccess;
    if (!P.slot[k]) {
      if ((e = cudaMallocHost((void**)&P.slot[k], StagePool::SLOT_BYTES)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&P.ev[k], cudaEventDisableTiming)) != cudaSuccess) return e;
    } else if (P.used[k] && (e = cudaEventSynchronize(P.ev[k])) != cudaSuccess) {
      return e;
    }
    const char* seg[4];
    size_t len[4];
    for (size_t r = 0; r < height; ++r) {
      seg[r] = (const char*)src + r * spitch + w0;
      len[r] = w;
    }
    P.gather(P.slot[k], seg, len, (int)height);
    e = height == 1 ? cudaMemcpyAsync((char*)dst + w0, P.slot[k], w, cudaMemcpyHostToDevice, cs)
                    : cudaMemcpy2DAsync((char*)dst + w0, dpitch, P.slot[k], w, w, height, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaEventRecord(P.ev[k], cs);
    if (e != cudaSuccess) return e;
    P.used[k] = true;
  }
  return cudaSuccess;
}

// MCX_TRACE=1: host timestamps of the runtime's stages on stderr (latency breakdown).
static bool trace_on() {
  static const bool on = getenv("MCX_TRACE") && atoi(getenv("MCX_TRACE")) > 0;
  return on;
}
static void trace(const char* what) {
  if (!trace_on()) return;
  static thread_local std::chrono::steady_clock::time_point t0;
  const auto now = std::chrono::steady_clock::now();
  if (!strcmp(what, "begin")) t0 = now;
  fprintf(stderr, "[mcx] %8.1f us  %s\n", std::chrono::duration<double, std::micro>(now - t0).count(), what);
}

// MCX_TRACE=2 adds device-side stamps: CUDA events recorded on the streams at the stages
// of a call, printed (µs after the first stamp) when the call ends.
struct DevStamps {
  cudaEvent_t ev[24] = {};
  const char* name[24] = {};
  int n = 0;
};
static thread_local DevStamps g_stamps;
static bool dtrace_on() {
  static const bool on = getenv("MCX_TRACE") && atoi(getenv("MCX_TRACE")) > 1;
  return on;
}
void dstamp(cudaStream_t s, const char* what) {
  if (!dtrace_on()) return;
  if (!strcmp(what, "begin")) g_stamps.n = 0;
  if (g_stamps.n >= 24) return;
  cudaEvent_t& e = g_stamps.ev[g_stamps.n];
  if (!e) cudaEventCreate(&e);
  cudaEventRecord(e, s);
  g_stamps.name[g_stamps.n++] = what;
}
static void dstamp_print() {
  if (!dtrace_on() || g_stamps.n == 0) return;
  for (int i = 0; i < g_stamps.n; ++i) {
    float ms = 0.f;
    cudaEventSynchronize(g_stamps.ev[i]);
    cudaEventElapsedTime(&ms, g_stamps.ev[0], g_stamps.ev[i]);
    fprintf(stderr, "[mcx-dev] %8.1f us  %s\n", 1e3 * ms, g_stamps.name[i]);
  }
  g_stamps.n = 0;
}

static int bits_for(uint64_t v) {  // bits to represent every value in [0, v]
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

// ------------------------------------------------------------------ kernels
// Order-preserving 64-bit key of a double (−0.0 just below +0.0).
__device__ __forceinline__ uint64_t ordered_key(double x) {
  const uint64_t u = __double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// 2. sort key of hit k: gid << 2 | τ_A << 1 | τ_B (job sorted in a second, stable pass)
__global__ void key_kernel(const mcx_hit* __restrict__ hits, const uint32_t* __restrict__ hit_task, uint64_t n,
                           const JobDev* __restrict__ jobs, uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
    const mcx_hit H = hits[k];
    const JobDev& J = jobs[hit_task ? hit_task[k] : 0];
    const uint32_t qa = H.ia >> 1, qb = H.ib >> 1;
    const uint64_t i = qa % J.NA, k1 = qa / J.NA, j = qb % J.NB, l1 = qb / J.NB;
    const uint64_t n12 = (uint64_t)J.NA * J.NB;
    const uint64_t gid = i + (uint64_t)J.NA * j + n12 * k1 + n12 * (uint64_t)(J.MA - 1) * l1;
    keys[k] = gid << 2 | (uint64_t)(H.ia & 1) << 1 | (H.ib & 1);
    vals[k] = (uint32_t)k;
  }
}

// job of the hit at each sorted position (second sort pass key)
__global__ void task_key_kernel(const uint32_t* __restrict__ order, const uint32_t* __restrict__ hit_task, uint64_t n,
                                uint64_t* __restrict__ keys) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x)
    keys[r] = hit_task[order[r]];
}

// 4. record r = fields of hit order[r]; xkey for the dedup sweep (order-preserving bits of x)
__global__ void record_kernel(const mcx_hit* __restrict__ hits, const uint32_t* __restrict__ hit_task,
                              const uint32_t* __restrict__ order, uint64_t n, const JobDev* __restrict__ jobs,
                              mcx_record* __restrict__ recs, uint64_t* __restrict__ xkeys, uint32_t* __restrict__ xvals) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = order[r];
    const mcx_hit H = hits[k];
    const uint32_t task = hit_task ? hit_task[k] : 0;
    const JobDev& J = jobs[task];
    mcx_record R;
    record_fields(H, J.cA, J.NA, J.MA, J.MpA, J.sA, J.NB, J.MB, J.sB, R.gid, R.point, R.params);
    R.ia = H.ia;
    R.ib = H.ib;
    R.bary[0] = H.s; R.bary[1] = H.t; R.bary[2] = H.a; R.bary[3] = H.b;
    R.task = task;
    R.pad[0] = R.pad[1] = R.pad[2] = 0;
    recs[r] = R;
    if (xkeys) {
      xkeys[r] = ordered_key(R.point[0]);
      xvals[r] = (uint32_t)r;
    }
  }
}

__global__ void xtask_key_kernel(const uint32_t* __restrict__ xorder, const mcx_record* __restrict__ recs, uint64_t n,
                                 uint64_t* __restrict__ keys) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x)
    keys[p] = recs[xorder[p]].task;
}

// 5a. close pairs.  The records are in (job, x-bucket) order, the bucket being the top 32
// bits of ordered_key(x) (relative width 2^-20; a 4-pass sort instead of 8).  From each
// position scan forward while the job matches and the bucket does not exceed that of
// fl(x + 2·tol) ≥ x + tol: every record within tol of x, before or after it in x, lies
// in that range, so each close pair is found from its earlier position.  The exact test
// is |fl(p − q)| ≤ tol in all 4 coordinates.  The count keeps running past cap.
__global__ void close_pairs_kernel(const uint32_t* __restrict__ xorder, const uint64_t* __restrict__ xkeys,
                                   const mcx_record* __restrict__ recs, uint64_t n, uint2* __restrict__ pairs,
                                   uint64_t cap, unsigned long long* __restrict__ count, uint8_t* __restrict__ state) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = xorder[p];
    const mcx_record& R = recs[r];
    const uint64_t hi = ordered_key(dadd(R.point[0], 2.0 * MCX_DEDUP_TOL)) >> 32;
    for (uint64_t q = p + 1; q < n; ++q) {
      if ((xkeys[q] >> 32) > hi) break;
      const uint32_t r2 = xorder[q];
      const mcx_record& S = recs[r2];
      if (S.task != R.task) break;
      if (fabs(dsub(S.point[0], R.point[0])) <= MCX_DEDUP_TOL && fabs(dsub(S.point[1], R.point[1])) <= MCX_DEDUP_TOL &&
          fabs(dsub(S.point[2], R.point[2])) <= MCX_DEDUP_TOL && fabs(dsub(S.point[3], R.point[3])) <= MCX_DEDUP_TOL) {
        const uint32_t e = min(r, r2), l = max(r, r2);
        const unsigned long long pos = atomicAdd(count, 1ull);
        if (pos < cap) pairs[pos] = make_uint2(e, l);
        state[l] = 0;  // has a close predecessor: undecided
      }
    }
  }
}

// 5b. greedy resolution in rounds, grid-wide (a cooperative launch: one grid sync per
// pass).  state: 1 kept, 2 dropped, 0 undecided.  Per round, one pass over the pairs
// marks "a kept predecessor" (bit 0: drop) and "an undecided predecessor" (bit 1: wait)
// per record — word-level atomicOr, so concurrent marks of one record never lose a bit —
// and one more decides: drop, keep (all predecessors dropped) or wait.
__global__ void __launch_bounds__(256) resolve_kernel(const uint2* __restrict__ pairs,
                                                      const unsigned long long* __restrict__ np_dev, uint64_t cap,
                                                      uint8_t* __restrict__ state, uint32_t* __restrict__ mark,
                                                      unsigned* __restrict__ left_flag) {
  cg::grid_group grid = cg::this_grid();
  // an overflowed pair list leaves undecided records without stored pairs: the host
  // sees the count, grows the list and reruns, so do nothing here
  if ((uint64_t)*np_dev > cap) return;
  const uint64_t np = *np_dev;
  const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
  for (int round = 0;; ++round) {
    for (uint64_t k = t0; k < np; k += stride) {
      const uint2 e = pairs[k];
      if (state[e.y] == 0) {
        const uint8_t se = state[e.x];
        const uint32_t bit = se == 1 ? 1u : (se == 0 ? 2u : 0u);
        if (bit) atomicOr(mark + (e.y >> 2), bit << (8 * (e.y & 3)));
      }
    }
    if (t0 == 0) left_flag[round & 1] = 0;  // the flag the next decision pass writes
    grid.sync();
    for (uint64_t k = t0; k < np; k += stride) {
      const uint32_t l = pairs[k].y;
      const uint32_t m = (mark[l >> 2] >> (8 * (l & 3))) & 3u;
      if (state[l] == 0) {
        if (m & 1u) state[l] = 2;
        else if (!(m & 2u)) state[l] = 1;
        else left_flag[round & 1] = 1;
      }
    }
    grid.sync();
    for (uint64_t k = t0; k < np; k += stride) {  // clear the marks of this round
      const uint32_t l = pairs[k].y;
      mark[l >> 2] = 0;
    }
    const bool more = *(volatile unsigned*)(left_flag + (round & 1)) != 0;
    grid.sync();
    if (!more) break;
  }
}

// 6. text, one thread per (record, field): field lengths; line lengths (0 for dropped
// records) and keep flags; then every field written at its offset after the scan.
__global__ void field_len_kernel(const mcx_record* __restrict__ recs, const uint8_t* __restrict__ state, uint64_t n,
                                 const JobDev* __restrict__ jobs, uint8_t* __restrict__ flen) {
  constexpr int F = fmt::LINE_FIELDS;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n * F; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = q / F;
    if (state && state[r] != 1) continue;
    const mcx_record& R = recs[r];
    const JobDev& J = jobs[R.task];
    char f[32];
    flen[q] = (uint8_t)fmt::fmt_field(f, (int)(q % F), J.n1, J.sign1, J.n2, J.sign2, R.gid, R.point, R.bary, R.params);
  }
}

__global__ void line_len_kernel(const uint8_t* __restrict__ state, uint64_t n, const uint8_t* __restrict__ flen,
                                uint32_t* __restrict__ lens, uint8_t* __restrict__ flags) {
  constexpr int F = fmt::LINE_FIELDS;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
    const bool keep = !state || state[r] == 1;
    flags[r] = keep;
    if (!lens) continue;
    uint32_t len = 0;
    if (keep)
      for (int f = 0; f < F; ++f) len += flen[r * F + f] + 1u;
    lens[r] = len;
  }
}

__global__ void field_write_kernel(const mcx_record* __restrict__ recs, const uint8_t* __restrict__ flags, uint64_t n,
                                   const JobDev* __restrict__ jobs, const uint64_t* __restrict__ incl,
                                   const uint32_t* __restrict__ lens, const uint8_t* __restrict__ flen,
                                   char* __restrict__ text) {
  constexpr int F = fmt::LINE_FIELDS;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n * F; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = q / F;
    const int f = (int)(q % F);
    if (!flags[r]) continue;
    uint64_t o = incl[r] - lens[r];
    for (int g = 0; g < f; ++g) o += flen[r * F + g] + 1u;
    const mcx_record& R = recs[r];
    const JobDev& J = jobs[R.task];
    char buf[32];
    int k = fmt::fmt_field(buf, f, J.n1, J.sign1, J.n2, J.sign2, R.gid, R.point, R.bary, R.params);
    buf[k++] = f == F - 1 ? '\n' : ' ';
    for (int i = 0; i < k; ++i) text[o + i] = buf[i];
  }
}

// find_intersections searches the larger mesh chunk by chunk during its upload
// (find_stepped) from this many triangles on (load_mesh splits it into >= 4 chunks)
// and is at least STEP_RATIO times the other mesh (which must be uploaded before the
// first step: two similar meshes share the link until the end, and the per-step fixed
// costs then follow the copy instead of hiding under it — measured on C3)
constexpr uint64_t STEP_MIN_TRI = 1ull << 18;
static uint64_t step_ratio() {  // MCX_STEP_RATIO overrides (experiments)
  const char* v = getenv("MCX_STEP_RATIO");
  return v ? strtoull(v, nullptr, 10) : 4;
}

// ------------------------------------------------------------------ small hit counts
// Steps 2-6 in ONE single-CTA kernel for n ≤ SMALL_N hits (the common case: a handful
// to a few hundred intersections per layer pair): bitonic sort of the (job, gid, τ_A,
// τ_B) keys in shared memory, records, the 1e-9 dedup (all earlier records of the job
// scanned; ≤ SMALL_K close predecessors each, else the general path reruns it), the
// greedy rule resolved in rounds, and block-scan compaction of records and text.
// The dedup scan reads the points and job ids from shared memory (structure of arrays:
// consecutive threads, consecutive words).  Keys are unique ((gid, τ) ↔ (iA, iB) within a job), so sort stability is moot.
constexpr int SMALL_N = 1024;
constexpr int SMALL_K = 8;
constexpr int REC_LINE_MAX = 352;  // ≥ the longest records line (349 bytes)
constexpr unsigned SMALL_NONE = 0xffffffffu;  // "no small-path text" (small_text_kernel)
constexpr int SMALL_TEXT_INLINE = 60;         // kept lines whose text post_small_kernel writes itself (≤ 1 field per thread)

struct SmallOut {
  unsigned long long kept, text_bytes, overflow;
};

// exclusive block prefix sum of v over 1024 threads (returns the total in *tot)
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_sums, uint32_t* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = warp_sums[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_sums[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  const uint32_t base = warp ? warp_sums[warp - 1] : 0u;
  *tot = warp_sums[31];
  __syncthreads();
  return base + x - v;
}

struct SmallSmem {
  unsigned long long key[SMALL_N];
  uint16_t idx[SMALL_N];
  uint16_t nb[SMALL_N][SMALL_K];
  uint8_t nnb[SMALL_N], state[SMALL_N];
  double px[4][SMALL_N];                             // record points (dedup scan)
  uint32_t ptask[SMALL_N];                           // record jobs
  uint32_t warp_sums[32];
  int overflow;
};

__device__ void format_line(uint32_t p, const mcx_record* __restrict__ recs, const JobDev* __restrict__ jobs,
                            char* __restrict__ slots, uint16_t* __restrict__ line_len, int lane);
__device__ uint32_t pack_text(uint32_t total, const char* __restrict__ slots, const uint16_t* __restrict__ line_len,
                              uint32_t* line_off, uint32_t* warp_sums, char* __restrict__ h_text);

// n = min(*n_dev, n_cap) is read on the device (the search's hit counter), so the
// kernel can follow the search without a host round trip; more than SMALL_N hits sets
// res->overflow = 2 and the host runs the general path.  Results (SmallOut, records,
// text) go straight to mapped host memory with coalesced 16-byte stores.
__global__ void __launch_bounds__(1024) post_small_kernel(const mcx_hit* __restrict__ hits,
                                                          const uint32_t* __restrict__ hit_task,
                                                          const unsigned long long* __restrict__ n_dev,
                                                          uint64_t n_cap, const JobDev* __restrict__ jobs,
                                                          int gid_shift, int dedup, int want_text,
                                                          mcx_record* __restrict__ recs, mcx_record* __restrict__ out,
                                                          unsigned* __restrict__ total_dev, char* __restrict__ slots,
                                                          uint16_t* __restrict__ line_len, SmallOut* __restrict__ res,
                                                          mcx_record* __restrict__ h_out, char* __restrict__ h_text) {
  extern __shared__ __align__(16) unsigned char small_raw[];
  SmallSmem& S = *reinterpret_cast<SmallSmem*>(small_raw);
  unsigned long long* key = S.key;
  uint16_t* idx = S.idx;
  auto& nb = S.nb;
  uint8_t* nnb = S.nnb;
  uint8_t* state = S.state;
  uint32_t* warp_sums = S.warp_sums;
  int& overflow = S.overflow;
  const int tid = threadIdx.x;
  if (tid == 0) {
    total_dev[0] = SMALL_NONE;  // until the records are complete (early exits)
    total_dev[1] = 0;           // small_text_kernel's CTA counter
  }
#if MCX_SMALL_PROF  // phase clocks (tools/microbench/build_variant.py -DMCX_SMALL_PROF=1)
  __shared__ long long tprof[11];
  if (tid == 0) tprof[10] = clock64();
#define SMALL_PHASE(id)              \
  do {                               \
    __syncthreads();                 \
    if (tid == 0) tprof[id] = clock64(); \
  } while (0)
#else
#define SMALL_PHASE(id) \
  do {                  \
  } while (0)
#endif
  const uint64_t n64 = min((uint64_t)*n_dev, n_cap);
  if (n64 > (uint64_t)SMALL_N) {
    if (tid == 0) {
      res->kept = res->text_bytes = 0;
      res->overflow = 2;
    }
    return;
  }
  const uint32_t n = (uint32_t)n64;
  uint32_t P = 1;
  while (P < n) P <<= 1;
  if (tid == 0) overflow = 0;
  for (uint32_t k = tid; k < P; k += blockDim.x) {
    unsigned long long kk = ~0ull;
    if (k < n) {
      const mcx_hit H = hits[k];
      const uint32_t t = hit_task ? hit_task[k] : 0u;
      const JobDev& J = jobs[t];
      const uint32_t qa = H.ia >> 1, qb = H.ib >> 1;
      const uint64_t i = qa % J.NA, k1 = qa / J.NA, j = qb % J.NB, l1 = qb / J.NB;
      const uint64_t n12 = (uint64_t)J.NA * J.NB;
      const uint64_t gid = i + (uint64_t)J.NA * j + n12 * k1 + n12 * (uint64_t)(J.MA - 1) * l1;
      kk = ((unsigned long long)t << gid_shift) | gid << 2 | (uint64_t)(H.ia & 1) << 1 | (H.ib & 1);
    }
    key[k] = kk;
    idx[k] = (uint16_t)k;
  }
  SMALL_PHASE(0);
  __syncthreads();
  for (uint32_t k = 2; k <= P; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = tid; i < P; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          if ((key[i] > key[l]) == up) {
            const unsigned long long tk = key[i];
            key[i] = key[l];
            key[l] = tk;
            const uint16_t ti = idx[i];
            idx[i] = idx[l];
            idx[l] = ti;
          }
        }
      }
      __syncthreads();
    }
  SMALL_PHASE(1);
  const uint32_t r = tid;  // one record per thread (n ≤ 1024 = blockDim)
  const bool valid = r < n;
  if (valid) {
    const uint32_t k = idx[r];
    const mcx_hit H = hits[k];
    const uint32_t t = hit_task ? hit_task[k] : 0u;
    const JobDev& J = jobs[t];
    mcx_record R;
    record_fields(H, J.cA, J.NA, J.MA, J.MpA, J.sA, J.NB, J.MB, J.sB, R.gid, R.point, R.params);
    R.ia = H.ia;
    R.ib = H.ib;
    R.bary[0] = H.s; R.bary[1] = H.t; R.bary[2] = H.a; R.bary[3] = H.b;
    R.task = t;
    R.pad[0] = R.pad[1] = R.pad[2] = 0;
    recs[r] = R;
#pragma unroll
    for (int c = 0; c < 4; ++c) S.px[c][r] = R.point[c];
    S.ptask[r] = t;
  }
  __syncthreads();  // records visible (global, L1 of this SM; points and jobs in shared memory)
  SMALL_PHASE(2);
  // dedup: close predecessors of r within its job (records of a job are contiguous)
  uint8_t cnt = 0;
  if (valid && dedup) {
    const double x0 = S.px[0][r], x1 = S.px[1][r], x2 = S.px[2][r], x3 = S.px[3][r];
    const uint32_t tr = S.ptask[r];
    // predecessors in descending order, 4 per iteration (independent shared loads);
    // the scan stops at the first record of another job
    auto close = [&](int e) {
      return fabs(dsub(x0, S.px[0][e])) <= MCX_DEDUP_TOL && fabs(dsub(x1, S.px[1][e])) <= MCX_DEDUP_TOL &&
             fabs(dsub(x2, S.px[2][e])) <= MCX_DEDUP_TOL && fabs(dsub(x3, S.px[3][e])) <= MCX_DEDUP_TOL;
    };
    bool stop = false;
    int e = (int)r - 1;
    for (; e >= 3 && !stop; e -= 4) {
      double xs[4];
      uint32_t ts[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        xs[u] = S.px[0][e - u];
        ts[u] = S.ptask[e - u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (stop) break;
        if (ts[u] != tr) {
          stop = true;
        } else if (fabs(dsub(x0, xs[u])) <= MCX_DEDUP_TOL && close(e - u)) {
          if (cnt < SMALL_K) nb[r][cnt] = (uint16_t)(e - u);
          ++cnt;
        }
      }
    }
    for (; e >= 0 && !stop; --e) {
      if (S.ptask[e] != tr) break;
      if (close(e)) {
        if (cnt < SMALL_K) nb[r][cnt] = (uint16_t)e;
        ++cnt;
      }
    }
    if (cnt > SMALL_K) overflow = 1;
  }
  if (valid) {
    nnb[r] = cnt;
    state[r] = cnt ? 0 : 1;
  }
  __syncthreads();
  SMALL_PHASE(3);
  if (overflow) {
    if (tid == 0) {
      res->kept = res->text_bytes = 0;
      res->overflow = 1;
    }
    return;
  }
  if (dedup) {
    for (;;) {  // decisions are monotone, so racing reads only delay them
      bool left = false;
      if (valid && state[r] == 0) {
        bool kept_pred = false, all_dropped = true;
        for (int q = 0; q < nnb[r]; ++q) {
          const uint8_t st = state[nb[r][q]];
          kept_pred |= st == 1;
          all_dropped &= st == 2;
        }
        if (kept_pred) state[r] = 2;
        else if (all_dropped) state[r] = 1;
        else left = true;
      }
      if (!__syncthreads_or(left)) break;
    }
  }
  SMALL_PHASE(4);
  const bool keep = valid && state[r] == 1;
  uint32_t total;
  const uint32_t pos = block_excl_scan(keep ? 1u : 0u, warp_sums, &total);
  if (keep) {
    out[pos] = recs[r];
  }
  __syncthreads();
  SMALL_PHASE(5);
  // text: up to SMALL_TEXT_INLINE kept lines here (one warp per line), more by
  // small_text_kernel over many SMs
  const bool text_here = want_text && total <= (uint32_t)SMALL_TEXT_INLINE;
  uint32_t tbytes = 0;
  if (text_here) {
    // one thread per (line, field) — all of a few lines' conversions side by side — each
    // field kept in its thread across the scans: lengths, line offsets, then the bytes
    // into the contiguous text (slots buffer) and 16-byte copies to the mapped host buffer
    constexpr int F = fmt::LINE_FIELDS;
    uint16_t* flen = S.idx;                                    // dead after the records
    uint32_t* line_off = reinterpret_cast<uint32_t*>(S.key);  // dead after the sort
    const uint32_t nf = total * F, p = tid / F, fi = tid % F;
    char f[32];
    int k = 0;
    if (tid < nf) {
      const mcx_record& R = out[p];
      const JobDev& J = jobs[R.task];
      k = fmt::fmt_field(f, (int)fi, J.n1, J.sign1, J.n2, J.sign2, R.gid, R.point, R.bary, R.params);
      f[k++] = fi == F - 1 ? '\n' : ' ';
    }
    flen[tid] = (uint16_t)k;
    __syncthreads();
    uint32_t len = 0;
    if (tid < total)
      for (int g = 0; g < F; ++g) len += flen[tid * F + g];
    const uint32_t off = block_excl_scan(len, warp_sums, &tbytes);
    if (tid < total) line_off[tid] = off;
    __syncthreads();
    if (tid < nf) {
      uint32_t o = line_off[p];
      for (uint32_t g = 0; g < fi; ++g) o += flen[p * F + g];
      for (int q = 0; q < k; ++q) slots[o + q] = f[q];
    }
    __syncthreads();
    const uint32_t t16 = tbytes / 16;
    const uint4* ts = reinterpret_cast<const uint4*>(slots);
    uint4* td = reinterpret_cast<uint4*>(h_text);
    for (uint32_t q = tid; q < t16; q += blockDim.x) td[q] = ts[q];
    for (uint32_t q = 16 * t16 + tid; q <= tbytes; q += blockDim.x) h_text[q] = q < tbytes ? slots[q] : '\0';
  }
  SMALL_PHASE(6);
  // coalesced copy-out to the mapped host buffers
  {
    const uint4* src = reinterpret_cast<const uint4*>(out);
    uint4* dst = reinterpret_cast<uint4*>(h_out);
    for (uint32_t q = tid; q < total * (sizeof(mcx_record) / 16); q += blockDim.x) dst[q] = src[q];
  }
  SMALL_PHASE(7);
  if (tid == 0) {
#if MCX_SMALL_PROF
    const char* nm[8] = {"keys", "sort", "records", "dedup", "resolve", "compact", "text", "copyout"};
    for (int q = 0; q < 8; ++q)
      printf("small %-10s %7lld cycles\n", nm[q], tprof[q] - (q ? tprof[q - 1] : tprof[10]));
#endif
    res->kept = total;
    res->text_bytes = tbytes;  // (small_text_kernel's otherwise)
    res->overflow = 0;
    *total_dev = want_text && !text_here ? total : SMALL_NONE;
  }
}

// Records text of the small path.  format_line: one warp formats kept line p into its
// fixed-stride slot — lane f formats field f (a line's 17 exact conversions side by side),
// a warp scan places them — and records the line length.
__device__ void format_line(uint32_t p, const mcx_record* __restrict__ recs, const JobDev* __restrict__ jobs,
                            char* __restrict__ slots, uint16_t* __restrict__ line_len, int lane) {
  constexpr int F = fmt::LINE_FIELDS;
  const mcx_record& R = recs[p];
  const JobDev& J = jobs[R.task];
  char f[32];
  int k = 0;
  if (lane < F) k = fmt::fmt_field(f, lane, J.n1, J.sign1, J.n2, J.sign2, R.gid, R.point, R.bary, R.params);
  const uint32_t lenf = lane < F ? k + 1u : 0u;  // + separator
  uint32_t incl = lenf;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane < F) {
    f[k] = lane == F - 1 ? '\n' : ' ';
    char* d = slots + (uint64_t)p * REC_LINE_MAX + (incl - lenf);
    for (int q = 0; q <= k; ++q) d[q] = f[q];
  }
  if (lane == F - 1) line_len[p] = (uint16_t)incl;
}

// pack_text (one CTA of 1024 threads): line offsets by a block scan, then the text written
// to the mapped host buffer in 16-byte stores, each gathered from the line slots (binary
// search for the line of its first byte; the 16 source offsets first, then 16 independent
// loads past L1 — other CTAs may have written the slots).  Returns the text length.
__device__ uint32_t pack_text(uint32_t total, const char* __restrict__ slots, const uint16_t* __restrict__ line_len,
                              uint32_t* line_off, uint32_t* warp_sums, char* __restrict__ h_text) {
  const int tid = threadIdx.x;
  uint32_t tbytes = 0;
  const uint32_t len_t = tid < total ? (uint32_t)*(const volatile uint16_t*)(line_len + tid) : 0u;
  const uint32_t off = block_excl_scan(len_t, warp_sums, &tbytes);
  if (tid < total) line_off[tid] = off;
  if (tid == 0) line_off[total] = tbytes;
  __syncthreads();
  const uint32_t nchunk = (tbytes + 1 + 15) / 16;  // + the terminator
  for (uint32_t q = tid; q < nchunk; q += blockDim.x) {
    uint32_t lo = 0, hi = total;  // the last line with line_off <= 16q
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (line_off[mid] <= 16 * q) lo = mid;
      else hi = mid;
    }
    union {
      char c[16];
      uint4 v;
    } w;
    uint32_t line = lo, src[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t b = 16 * q + i;
      while (line < total && b >= line_off[line + 1]) ++line;
      src[i] = b < tbytes ? line * REC_LINE_MAX + (b - line_off[line]) : 0xffffffffu;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) w.c[i] = src[i] != 0xffffffffu ? __ldcg(slots + src[i]) : '\0';
    reinterpret_cast<uint4*>(h_text)[q] = w.v;
  }
  return tbytes;
}

// The text of more than SMALL_TEXT_INLINE kept records (after post_small_kernel, same
// stream): 32 CTAs of 32 warps, lines dealt over the CTAs (SMs) first, one warp per line;
// the last CTA to finish (a device-scope counter) packs the text.  *total_dev = the kept
// count, SMALL_NONE when there is nothing to do here (overflow, general path, no text
// wanted, or post_small_kernel wrote the text itself).
__global__ void __launch_bounds__(1024) small_text_kernel(const mcx_record* __restrict__ recs,
                                                          const JobDev* __restrict__ jobs,
                                                          const unsigned* __restrict__ total_dev,
                                                          unsigned* __restrict__ done, char* __restrict__ slots,
                                                          uint16_t* __restrict__ line_len, char* __restrict__ h_text,
                                                          SmallOut* __restrict__ res) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t line_off[SMALL_N + 1];
  __shared__ bool last;
  const uint32_t total = *total_dev;
  if (total > (uint32_t)SMALL_N) return;  // uniform over the grid
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t p = warp * gridDim.x + blockIdx.x;
  if (p < total) format_line(p, recs, jobs, slots, line_len, lane);
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const uint32_t tbytes = pack_text(total, slots, line_len, line_off, warp_sums, h_text);
  if (tid == 0) {
    res->text_bytes = tbytes;
    *done = 0;  // for the next call
  }
}

static size_t n_jobs_of(const std::vector<JobDev>& jobs) { return jobs.size(); }

// Mapped host buffer of the small path: [SmallOut | SMALL_N records | SMALL_N lines].
static int small_map(mcx_context* c, SmallOut** so, mcx_record** recs, char** text) {
  const size_t bytes = 64 + sizeof(mcx_record) * SMALL_N + (size_t)REC_LINE_MAX * SMALL_N + 64;
  if (!c->h_map.p) {
    CUDA_TRY(cudaHostAlloc(&c->h_map.p, bytes, cudaHostAllocMapped));
    c->h_map.bytes = bytes;
  }
  char* base = (char*)c->h_map.p;
  *so = (SmallOut*)base;
  *recs = (mcx_record*)(base + 64);
  *text = base + 64 + sizeof(mcx_record) * SMALL_N;
  return MCX_OK;
}

// Enqueue the single-kernel post-processing on c->s0: n hits (n_dev == nullptr) or
// min(*n_dev, hit capacity) hits read on the device.  *queued = false if the sort key
// does not fit 64 bits (the general path handles that).
static int enqueue_small(mcx_context* c, const unsigned long long* n_dev, uint64_t n, const uint32_t* hit_task,
                         const std::vector<JobDev>& jobs, const mcx_find_opts* fo, bool text_ok, bool* queued) {
  cudaStream_t s = c->s0;
  *queued = false;
  uint64_t mg = 0;
  for (const JobDev& j : jobs) mg = std::max<uint64_t>(mg, (uint64_t)j.NA * (j.MA - 1) * j.NB * (j.MB - 1));
  const int shift = bits_for(mg) + 2, tb = std::max(1, bits_for(jobs.size() - 1));
  if (shift + tb > 64) return MCX_OK;
  const bool want_text = fo->text && text_ok;
  int rc;
  if ((rc = ensure(c, c->jobs, sizeof(JobDev) * jobs.size(), s)) ||
      (rc = ensure(c, c->recs, sizeof(mcx_record) * SMALL_N, s)) ||
      (rc = ensure(c, c->recs_out, sizeof(mcx_record) * SMALL_N, s)) || (rc = ensure(c, c->small, 64, s)) ||
      (rc = ensure(c, c->text, (size_t)REC_LINE_MAX * SMALL_N, s)) ||
      (rc = ensure(c, c->lines, (size_t)(REC_LINE_MAX + 2) * SMALL_N, s)))
    return rc;
  CUDA_TRY(h2d_async(c->jobs.p, jobs.data(), sizeof(JobDev) * jobs.size(), s));
  dstamp(s, "  small: job table uploaded");
  SmallOut* so;
  mcx_record* hr;
  char* ht;
  if ((rc = small_map(c, &so, &hr, &ht))) return rc;
  so->overflow = 3;  // "not run" until the kernel writes it
  unsigned long long* nd = (unsigned long long*)c->small.p + 4;
  if (!n_dev) {
    CUDA_TRY(cudaMemcpyAsync(nd, &n, 8, cudaMemcpyHostToDevice, s));  // 8 bytes, staged by the driver
    n_dev = nd;
  }
  uint64_t resident;
  if ((rc = kernel_prepare(reinterpret_cast<const void*>(post_small_kernel), 1024, sizeof(SmallSmem), -1,
                           c->device, &resident)))
    return rc;
  SmallOut* d_so;
  mcx_record* d_hr;
  char* d_ht;
  CUDA_TRY(cudaHostGetDevicePointer((void**)&d_so, so, 0));
  CUDA_TRY(cudaHostGetDevicePointer((void**)&d_hr, hr, 0));
  CUDA_TRY(cudaHostGetDevicePointer((void**)&d_ht, ht, 0));
  unsigned* total_dev = (unsigned*)c->small.p + 12;  // bytes 48-55 of the 64-byte scratch (+ the CTA counter)
  char* slots = (char*)c->lines.p;
  uint16_t* line_len = (uint16_t*)(slots + (size_t)REC_LINE_MAX * SMALL_N);
  post_small_kernel<<<1, 1024, sizeof(SmallSmem), s>>>(
      (const mcx_hit*)c->hits.p, hit_task, n_dev, n_dev == nd ? n : c->hit_cap, (const JobDev*)c->jobs.p, shift,
      fo->dedup ? 1 : 0, want_text ? 1 : 0, (mcx_record*)c->recs.p, (mcx_record*)c->recs_out.p, total_dev, slots,
      line_len, d_so, d_hr, d_ht);
  CUDA_TRY(cudaGetLastError());
  dstamp(s, "  small: post_small_kernel done");
  if (want_text) {  // exits at once unless post_small_kernel left more than SMALL_TEXT_INLINE lines to it
    small_text_kernel<<<SMALL_N / 32, 1024, 0, s>>>((const mcx_record*)c->recs_out.p, (const JobDev*)c->jobs.p,
                                                    total_dev, total_dev + 1, slots, line_len, d_ht, d_so);
    CUDA_TRY(cudaGetLastError());
  }
  *queued = true;
  return MCX_OK;
}

// After the stream synchronised: the small path's results, if it completed.
static bool take_small(mcx_context* c, const mcx_record** records, uint64_t* n_records, const char** text,
                       uint64_t* text_bytes) {
  SmallOut* so;
  mcx_record* hr;
  char* ht;
  if (small_map(c, &so, &hr, &ht) || so->overflow) return false;
  *records = hr;
  *n_records = so->kept;
  if (text && text_bytes) {
    *text = ht;
    *text_bytes = so->text_bytes;
  }
  return true;
}

static unsigned grid_of(uint64_t n) {
  uint64_t b = (n + 255) / 256;
  return (unsigned)std::min<uint64_t>(std::max<uint64_t>(b, 1), 148ull * 16);
}

// Steps 2-7 for n hits already in c->hits (hit_task: c->hit_task or null for one job).
static int postprocess(mcx_context* c, uint64_t n, const uint32_t* hit_task, const std::vector<JobDev>& jobs,
                       const mcx_find_opts* fo, const mcx_record** records, uint64_t* n_records, const char** text,
                       uint64_t* text_bytes, bool try_small = true) {
  cudaStream_t s = c->s0;
  *records = nullptr;
  *n_records = 0;
  if (text) *text = nullptr;
  if (text_bytes) *text_bytes = 0;
  if (n == 0) return MCX_OK;
  if (n > 0xffffffffull) return set_error(MCX_E_ARG, "more than 2^32 hits in one call");
  int rc = ensure(c, c->jobs, sizeof(JobDev) * jobs.size(), s);
  if (rc) return rc;
  CUDA_TRY(h2d_async(c->jobs.p, jobs.data(), sizeof(JobDev) * jobs.size(), s));
  const JobDev* J = (const JobDev*)c->jobs.p;
  const mcx_hit* H = (const mcx_hit*)c->hits.p;
  if (try_small && n <= (uint64_t)SMALL_N) {
    bool queued = false;
    if ((rc = enqueue_small(c, nullptr, n, n_jobs_of(jobs) > 1 ? hit_task : nullptr, jobs, fo, text && text_bytes,
                            &queued)))
      return rc;
    if (queued) {
      CUDA_TRY(cudaStreamSynchronize(s));
      if (take_small(c, records, n_records, text, text_bytes)) return MCX_OK;
    }
    // more than SMALL_K close predecessors somewhere: the general path below
  }
  if ((rc = ensure(c, c->k0, 8 * n, s)) || (rc = ensure(c, c->k1, 8 * n, s)) || (rc = ensure(c, c->v0, 4 * n, s)) ||
      (rc = ensure(c, c->v1, 4 * n, s)) || (rc = ensure(c, c->recs, sizeof(mcx_record) * n, s)) ||
      (rc = ensure(c, c->recs_out, sizeof(mcx_record) * n, s)) || (rc = ensure(c, c->state, n, s)) ||
      (rc = ensure(c, c->blocked, n + 4, s)) || (rc = ensure(c, c->lens, 4 * n, s)) ||
      (rc = ensure(c, c->offs, 8 * n, s)) || (rc = ensure(c, c->small, 64, s)))
    return rc;
  uint64_t max_gid = 0;
  for (const JobDev& j : jobs) max_gid = std::max<uint64_t>(max_gid, (uint64_t)j.NA * (j.MA - 1) * j.NB * (j.MB - 1));
  const int key_bits = bits_for(max_gid) + 2;
  if (key_bits > 64) return set_error(MCX_E_ARG, "gid range too large for a 64-bit sort key");
  const int task_bits = std::max(1, bits_for(jobs.size() - 1));
  const int ni = (int)n;
  // 2-3: sort hits by (gid, τ_A, τ_B), then stably by job
  key_kernel<<<grid_of(n), 256, 0, s>>>(H, hit_task, n, J, (uint64_t*)c->k0.p, (uint32_t*)c->v0.p);
  CUDA_TRY(cudaGetLastError());
  cub::DoubleBuffer<uint64_t> keys((uint64_t*)c->k0.p, (uint64_t*)c->k1.p);
  cub::DoubleBuffer<uint32_t> vals((uint32_t*)c->v0.p, (uint32_t*)c->v1.p);
  auto sort_pairs = [&](int bits) -> int {
    size_t tmp = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, vals, ni, 0, bits, s));
    int r = ensure(c, c->cub, tmp, s);
    if (r) return r;
    tmp = c->cub.bytes;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(c->cub.p, tmp, keys, vals, ni, 0, bits, s));
    return MCX_OK;
  };
  trace("big post: start");
  if ((rc = sort_pairs(key_bits))) return rc;
  if (hit_task && jobs.size() > 1) {
    task_key_kernel<<<grid_of(n), 256, 0, s>>>(vals.Current(), hit_task, n, keys.Current());
    CUDA_TRY(cudaGetLastError());
    if ((rc = sort_pairs(task_bits))) return rc;
  }
  // 4: records in sorted order (+ x keys for the dedup sweep)
  mcx_record* R = (mcx_record*)c->recs.p;
  const uint32_t* order = vals.Current();
  const bool dedup = fo->dedup && n > 1;
  uint64_t* xk = (keys.Current() == (uint64_t*)c->k0.p) ? (uint64_t*)c->k1.p : (uint64_t*)c->k0.p;
  uint32_t* xv = (order == (const uint32_t*)c->v0.p) ? (uint32_t*)c->v1.p : (uint32_t*)c->v0.p;
  record_kernel<<<grid_of(n), 256, 0, s>>>(H, hit_task, order, n, J, R, dedup ? xk : nullptr, xv);
  CUDA_TRY(cudaGetLastError());
  uint8_t* state = (uint8_t*)c->state.p;
  unsigned long long* pair_count = (unsigned long long*)c->small.p;
  if (dedup) {
    // 5: (job, x) order of the records, close pairs, greedy resolution
    cub::DoubleBuffer<uint64_t> xkeys(xk, xk == (uint64_t*)c->k0.p ? (uint64_t*)c->k1.p : (uint64_t*)c->k0.p);
    cub::DoubleBuffer<uint32_t> xvals(xv, xv == (uint32_t*)c->v0.p ? (uint32_t*)c->v1.p : (uint32_t*)c->v0.p);
    keys = xkeys;
    vals = xvals;
    {  // by the x bucket only: bits [32, 64) of the ordered key
      size_t tmp = 0;
      CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, vals, ni, 32, 64, s));
      if ((rc = ensure(c, c->cub, tmp, s))) return rc;
      tmp = c->cub.bytes;
      CUDA_TRY(cub::DeviceRadixSort::SortPairs(c->cub.p, tmp, keys, vals, ni, 32, 64, s));
    }
    if (jobs.size() > 1) {
      xtask_key_kernel<<<grid_of(n), 256, 0, s>>>(vals.Current(), R, n, keys.Current());
      CUDA_TRY(cudaGetLastError());
      if ((rc = sort_pairs(task_bits))) return rc;
    }
    // the pair count is checked at the next synchronisation (a rare overflow reruns this)
    c->pair_cap = std::max<uint64_t>(c->pair_cap, 4 * n);
    if ((rc = ensure(c, c->pairs, 8 * c->pair_cap, s))) return rc;
    CUDA_TRY(cudaMemsetAsync(state, 1, n, s));
    CUDA_TRY(cudaMemsetAsync(c->blocked.p, 0, n + 4, s));
    CUDA_TRY(cudaMemsetAsync(pair_count, 0, 8, s));
    close_pairs_kernel<<<grid_of(n), 256, 0, s>>>(vals.Current(), keys.Current(), R, n, (uint2*)c->pairs.p,
                                                   c->pair_cap, pair_count, state);
    CUDA_TRY(cudaGetLastError());
    {  // cooperative launch: every CTA co-resident (grid syncs between the passes)
      int sms = 148;
      uint64_t slots;
      if ((rc = kernel_prepare(reinterpret_cast<const void*>(resolve_kernel), 256, 0, -1, c->device, &slots))) return rc;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
      const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(slots, (uint64_t)sms * 2));
      const uint2* pr = (const uint2*)c->pairs.p;
      uint64_t pcap = c->pair_cap;
      uint32_t* mark = (uint32_t*)c->blocked.p;
      unsigned* left = (unsigned*)(pair_count + 2);
      void* args[] = {(void*)&pr, (void*)&pair_count, (void*)&pcap, (void*)&state, (void*)&mark, (void*)&left};
      CUDA_TRY(cudaLaunchCooperativeKernel((void*)resolve_kernel, dim3(g), dim3(256), args, 0, s));
    }
  }
  // 6: flags (+ text lengths), inclusive scan of the lengths, compaction, text
  uint8_t* flags = (uint8_t*)c->blocked.p;  // reused: resolution is done
  const bool want_text = fo->text && text && text_bytes;
  uint8_t* flen = nullptr;
  if (want_text) {
    if ((rc = ensure(c, c->flen, (size_t)fmt::LINE_FIELDS * n, s))) return rc;
    flen = (uint8_t*)c->flen.p;
    field_len_kernel<<<grid_of(fmt::LINE_FIELDS * n), 256, 0, s>>>(R, dedup ? state : nullptr, n, J, flen);
  }
  line_len_kernel<<<grid_of(n), 256, 0, s>>>(dedup ? state : nullptr, n, flen, want_text ? (uint32_t*)c->lens.p : nullptr,
                                             flags);
  CUDA_TRY(cudaGetLastError());
  unsigned long long* n_sel = pair_count + 1;
  {
    size_t tmp = 0;
    CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, tmp, R, flags, (mcx_record*)c->recs_out.p, n_sel, ni, s));
    if ((rc = ensure(c, c->cub, tmp, s))) return rc;
    tmp = c->cub.bytes;
    CUDA_TRY(cub::DeviceSelect::Flagged(c->cub.p, tmp, R, flags, (mcx_record*)c->recs_out.p, n_sel, ni, s));
  }
  uint64_t* incl = (uint64_t*)c->offs.p;
  if (want_text) {
    size_t tmp = 0;
    const uint32_t* lens = (const uint32_t*)c->lens.p;
    CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tmp, lens, incl, ni, s));
    if ((rc = ensure(c, c->cub, tmp, s))) return rc;
    tmp = c->cub.bytes;
    CUDA_TRY(cub::DeviceScan::InclusiveSum(c->cub.p, tmp, lens, incl, ni, s));
  }
  ensure_host(c->h_small, 64);
  uint64_t* hs = (uint64_t*)c->h_small.p;
  CUDA_TRY(cudaMemcpyAsync(hs, n_sel, 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(hs + 2, pair_count, 8, cudaMemcpyDeviceToHost, s));
  if (want_text) CUDA_TRY(cudaMemcpyAsync(hs + 1, incl + n - 1, 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  trace("big post: dedup + select + scan (synced)");
  if (dedup && hs[2] > c->pair_cap) {  // close-pair list overflowed: grow it and redo the stage
    c->pair_cap = hs[2] + 1024;
    return postprocess(c, n, hit_task, jobs, fo, records, n_records, text, text_bytes, false);
  }
  const uint64_t kept = hs[0], tbytes = want_text ? hs[1] : 0;
  if (want_text) {
    if ((rc = ensure(c, c->text, tbytes + 1, s))) return rc;
    field_write_kernel<<<grid_of(fmt::LINE_FIELDS * n), 256, 0, s>>>(R, flags, n, J, incl,
                                                                      (const uint32_t*)c->lens.p, flen,
                                                                      (char*)c->text.p);
    CUDA_TRY(cudaGetLastError());
  }
  // 7: D2H into pinned context memory
  if ((rc = ensure_host(c->h_recs, sizeof(mcx_record) * kept))) return rc;
  CUDA_TRY(cudaMemcpyAsync(c->h_recs.p, c->recs_out.p, sizeof(mcx_record) * kept, cudaMemcpyDeviceToHost, s));
  if (want_text) {
    if ((rc = ensure_host(c->h_text, tbytes + 1))) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->h_text.p, c->text.p, tbytes, cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  trace("big post: text + D2H (synced)");
  *records = (const mcx_record*)c->h_recs.p;
  *n_records = kept;
  if (want_text) {
    ((char*)c->h_text.p)[tbytes] = 0;
    *text = (const char*)c->h_text.p;
    *text_bytes = tbytes;
  }
  return MCX_OK;
}

static JobDev job_of(const mcx_mesh* A, const mcx_mesh* B, mcx_layer L) {
  JobDev j;
  j.cA = A->coords;
  j.sA = A->s_values;
  j.sB = B->s_values;
  j.NA = A->view.N;
  j.MA = A->view.M;
  j.NB = B->view.N;
  j.MB = B->view.M;
  j.MpA = A->view.plane_rows ? A->view.plane_rows : A->view.M;
  j.pad = 0;
  j.n1 = L.n1;
  j.sign1 = L.sign1;
  j.n2 = L.n2;
  j.sign2 = L.sign2;
  return j;
}

static int check_find_opts(const mcx_find_opts* fo) {
  if (!fo) return set_error(MCX_E_ARG, "null find options");
  if (fo->mode != MCX_MODE_BRUTE && fo->mode != MCX_MODE_CULL && fo->mode != MCX_MODE_PREFILTER)
    return set_error(MCX_E_ARG, "unknown mode %d", fo->mode);
  if (fo->pipeline != MCX_PIPE_TRIANGLE && fo->pipeline != MCX_PIPE_SPEC)
    return set_error(MCX_E_ARG, "unknown pipeline %d", fo->pipeline);
  return MCX_OK;
}

// After a search is enqueued on c->s0 (header copied to c->h_counters): queue the
// single-kernel post-processing, synchronise once, read the stats.  *retry: a capacity
// was exceeded (regrown here) — search again; *small_done: the records are ready.
static int after_search(mcx_context* c, const mcx_job* jobs, uint32_t n_jobs, const mcx_find_opts* fo,
                        const mcx_opts* o, const std::vector<JobDev>& jd, const mcx_record** records,
                        uint64_t* n_records, const char** text, uint64_t* text_bytes, mcx_stats* stats, bool* retry,
                        bool* small_done, uint64_t* total_hits) {
  *retry = false;
  *small_done = false;
  const unsigned long long* hc = (const unsigned long long*)c->h_counters.p;
  bool queued = false;
  int rc = enqueue_small(c, (const unsigned long long*)c->ws.p, 0,
                         n_jobs > 1 ? (const uint32_t*)c->hit_task.p : nullptr, jd, fo, text && text_bytes, &queued);
  if (rc) return rc;
  dstamp(c->s0, "small post (+ text) done");
  // the search header (hit / candidate counts, flags) after the post kernels, which read it
  // on the device: the copy is not on their critical path
  CUDA_TRY(cudaMemcpyAsync(c->h_counters.p, c->ws.p, sizeof(unsigned long long) * (8 + 8ull * n_jobs),
                           cudaMemcpyDeviceToHost, c->s0));
  CUDA_TRY(cudaStreamSynchronize(c->s0));
  trace("search + small post done (synced)");
  rc = batch_stats(hc, n_jobs, o, c->hit_cap, stats, 0.f);
  uint64_t total = 0, cands = 0;
  for (uint32_t t = 0; t < n_jobs; ++t) {
    total += stats[t].n_hits;
    cands += stats[t].n_aabb_pass;
  }
  *total_hits = total;
  if (rc == MCX_E_CAPACITY) {
    if (cands > c->cand_cap) c->cand_cap = cands + 1024;
    if (total > c->hit_cap) c->hit_cap = total + 1024;
    *retry = true;
    return MCX_OK;
  }
  if (rc == MCX_E_ARG && hc[2]) {  // non-finite coordinates: name the failing task
    for (uint32_t t = 0; t < n_jobs; ++t)
      for (const mcx_mesh* m : {jobs[t].A, jobs[t].B}) {
        uint32_t flag = 0;
        if (m->status) CUDA_TRY(cudaMemcpy(&flag, m->status, sizeof(flag), cudaMemcpyDeviceToHost));
        if (flag) {
          const mcx_layer& L = jobs[t].layer;
          return set_error(MCX_E_ARG, "job %u (layer pair %d %c %d %c): non-finite (NaN/Inf) coordinates in its %s "
                           "half-layer", t, L.n1, L.sign1 >= 0 ? '+' : '-', L.n2, L.sign2 >= 0 ? '+' : '-',
                           m == jobs[t].A ? "unstable (A)" : "stable (B)");
        }
      }
  }
  if (rc) return rc;
  *small_done = queued && take_small(c, records, n_records, text, text_bytes);
  return MCX_OK;
}

// Steps 1-7 for jobs whose meshes are resident (device current, all work on c->s0).
static int intersect(mcx_context* c, const mcx_job* jobs, uint32_t n_jobs, const mcx_find_opts* fo,
                     const mcx_record** records, uint64_t* n_records, const char** text, uint64_t* text_bytes,
                     mcx_stats* stats) {
  int rc = check_find_opts(fo);
  if (rc) return rc;
  if (!jobs || n_jobs == 0 || !records || !n_records || !stats) return set_error(MCX_E_ARG, "null argument");
  if (!c->stage.p) {
    CUDA_TRY(cudaMallocHost((void**)&c->stage.p, 1 << 20));
    c->stage.cap = 1 << 20;
  }
  StageScope scope(&c->stage);
  std::vector<mcx_task> tasks(n_jobs);
  std::vector<JobDev> jd(n_jobs);
  for (uint32_t t = 0; t < n_jobs; ++t) {
    if (!jobs[t].A || !jobs[t].B) return set_error(MCX_E_ARG, "job %u: null mesh", t);
    if (jobs[t].A->ctx != c || jobs[t].B->ctx != c) return set_error(MCX_E_ARG, "job %u: mesh of another context", t);
    if (!jobs[t].A->box || !jobs[t].B->box)
      return set_error(MCX_E_ARG, "job %u: an unpacked grid (mcx_grid_load) — search its column views", t);
    tasks[t] = mcx_task{&jobs[t].A->view, &jobs[t].B->view, 0, 0};
    jd[t] = job_of(jobs[t].A, jobs[t].B, jobs[t].layer);
  }
  mcx_opts o{};
  o.device = c->device;
  o.stream = c->s0;
  o.shard_index = fo->shard_index;
  o.shard_count = fo->shard_count;
  o.mode = fo->mode;
  o.pipeline = fo->pipeline;
  o.orient = fo->orient;
  uint64_t total = 0;
  bool small_done = false;
  for (int attempt = 0; attempt < 4; ++attempt) {
    o.cand_cap = c->cand_cap;
    const uint64_t wsb = mcx_batch_workspace_bytes(tasks.data(), n_jobs, &o);
    if ((rc = ensure(c, c->ws, wsb, c->s0)) || (rc = ensure(c, c->hits, sizeof(mcx_hit) * c->hit_cap, c->s0)) ||
        (rc = ensure(c, c->hit_task, 4 * c->hit_cap, c->s0)) ||
        (rc = ensure_host(c->h_counters, 8 * (8 + 8ull * n_jobs))))
      return rc;
    o.workspace = c->ws.p;
    o.workspace_bytes = c->ws.bytes;
    // search, then (optimistically) the single-kernel post-processing straight after it
    // on the device, one synchronisation for both
    unsigned long long* hc = (unsigned long long*)c->h_counters.p;
    dstamp(c->s0, "search start (s0)");
    rc = launch_batch(tasks.data(), n_jobs, &o, (mcx_hit*)c->hits.p, (uint32_t*)c->hit_task.p, c->hit_cap, stats, hc,
                      nullptr, /*header_later=*/true);
    if (rc) return rc;
    dstamp(c->s0, "search done");
    bool retry = false;
    rc = after_search(c, jobs, n_jobs, fo, &o, jd, records, n_records, text, text_bytes, stats, &retry, &small_done,
                      &total);
    if (retry) continue;
    break;
  }
  if (rc) return rc;
  if (small_done) return MCX_OK;
  return postprocess(c, total, n_jobs > 1 ? (const uint32_t*)c->hit_task.p : nullptr, jd, fo, records, n_records,
                     text, text_bytes, /*try_small=*/false);
}

// on_chunk(m, b0, b1): called after the pack of blocks [b0, b1) is enqueued (m->view
// is complete; the blocks are ready in stream order), e.g. to search them at once.
using ChunkFn = std::function<int(mcx_mesh*, uint64_t, uint64_t)>;

// cs (optional): the stream of the chunk copies — chunk j is copied on cs, then packed
// (and searched) on s after event cev[j], so the copies run back to back however long
// the per-chunk work on s takes.
// hplane: the host grid's plane stride in doubles (0: N·M, planes back to back) — a
// half-layer that is a column range of a larger host mesh is read in place.
static int load_mesh(mcx_context* c, const double* coords, uint32_t N, uint32_t M, const double* s_values,
                     cudaStream_t s, mcx_mesh** out, bool pack = true, const ChunkFn& on_chunk = ChunkFn(),
                     cudaStream_t cs = nullptr, uint64_t hplane = 0) {
  if (!coords || !s_values || !out) return set_error(MCX_E_ARG, "null argument");
  if (N < 1 || M < 2) return set_error(MCX_E_ARG, "a half-layer needs N >= 1 and M >= 2 (SPEC.md:473)");
  if (hplane == 0) hplane = (uint64_t)N * M;
  if (hplane < (uint64_t)N * M)
    return set_error(MCX_E_ARG, "host plane stride %llu < N*M = %llu", (unsigned long long)hplane,
                     (unsigned long long)N * M);
  const size_t hpitch = 8 * hplane;
  const uint64_t n = 2ull * N * (M - 1);
  if (n >= (1ull << 31)) return set_error(MCX_E_ARG, "triangle count must be < 2^31");
  mcx_mesh* m = new mcx_mesh();
  m->ctx = c;
  auto alloc = [&](void** p, size_t bytes) -> int {
    CUDA_TRY(cudaMallocFromPoolAsync(p, std::max<size_t>(bytes, 16), c->pool, s));
    return MCX_OK;
  };
  int rc = MCX_OK;
  const bool stage = 32ull * N * M >= STAGE_MIN_BYTES && !getenv("MCX_NO_STAGE") && pageable(coords);
  if ((rc = alloc((void**)&m->coords, 32ull * N * M)) || (rc = alloc((void**)&m->s_values, 8ull * M)) ||
      (!pack && (cudaMemcpyAsync(m->s_values, s_values, 8ull * M, cudaMemcpyHostToDevice, s) != cudaSuccess ||
                 (hplane == (uint64_t)N * M
                      ? h2d_rows(c, m->coords, 0, coords, 0, 32ull * N * M, 1, s, stage)
                      : h2d_rows(c, m->coords, 8ull * N * M, coords, hpitch, 8ull * N * M, 4, s, stage)) !=
                     cudaSuccess))) {
    mcx_mesh_free(m);
    return rc ? rc : set_error(MCX_E_CUDA, "grid upload failed");
  }
  if (!pack) {  // a grid: the source of column views only
    m->view = mcx_mesh_dev{n, m->coords, N, M, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, M, 0};
    *out = m;
    return MCX_OK;
  }
  if ((rc = alloc((void**)&m->box, 64 * n)) || (rc = alloc((void**)&m->perm, 4 * n)) ||
      (rc = alloc((void**)&m->gbox, 64 * ((n + GROUP - 1) / GROUP))) ||
      (rc = alloc((void**)&m->tbox, 64 * ((n + TILE - 1) / TILE))) ||
      (rc = alloc((void**)&m->bbox, 64 * ((n + A_BLOCK - 1) / A_BLOCK))) || (rc = alloc((void**)&m->status, 16))) {
    mcx_mesh_free(m);
    return rc;
  }
  m->view = mcx_mesh_dev{n, m->coords, N, M, m->box, m->perm, m->gbox, m->tbox, m->bbox, m->status, M, 0};
  cudaError_t e = cudaSuccess;
  if (cs) {  // the copy stream waits for the (stream-ordered) allocations on s
    e = cudaEventRecord(c->cev[8], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, c->cev[8], 0);
  } else {
    cs = s;
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(m->s_values, s_values, 8ull * M, cudaMemcpyHostToDevice, cs);
  // Upload and pack pipelined over chunks of whole 16-column tile rows: the blocks of
  // the tile rows a chunk completes are packed while the next chunk is copied, so only
  // the last chunk's packing follows the last byte of the H2D copy.
  const uint32_t MQ = M - 1, ntr = (MQ + ORDER_TILE_Q - 1) / ORDER_TILE_Q;
  const uint64_t nblk = pack_blocks(N, M), plane = (uint64_t)N * M * 8;
  const uint32_t nch = std::min<uint32_t>(n >= (1u << 20) ? 8 : (n >= (1u << 18) ? 4 : 1), ntr);
  uint64_t b_done = 0;
  uint32_t col_done = 0;
  for (uint32_t j = 0; j < nch && e == cudaSuccess && rc == MCX_OK; ++j) {
    const bool last = j + 1 == nch;
    const uint32_t tr1 = (uint32_t)((uint64_t)ntr * (j + 1) / nch);
    const uint32_t col1 = last ? M : std::min<uint32_t>(M, ORDER_TILE_Q * tr1 + 1);
    if (col1 > col_done)
      e = h2d_rows(c, m->coords + (uint64_t)col_done * N, plane, coords + (uint64_t)col_done * N, hpitch,
                   (uint64_t)(col1 - col_done) * N * 8, 4, cs, stage);
    if (e == cudaSuccess && cs != s) {
      e = cudaEventRecord(c->cev[j], cs);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s, c->cev[j], 0);
    }
    const uint64_t b1 = last ? nblk : 2ull * N * std::min<uint32_t>(MQ, ORDER_TILE_Q * tr1) / A_BLOCK;
    if (e == cudaSuccess && b1 > b_done) {  // (b1 = 0 would mean "all blocks" to pack_enqueue)
      rc = pack_enqueue(m->coords, N, M, MCX_ORDER_TILED, m->box, m->perm, m->gbox, m->tbox, m->bbox, m->status, s,
                        b_done, b1, M);
      if (rc == MCX_OK && on_chunk) rc = on_chunk(m, b_done, b1);
    }
    b_done = std::max(b_done, b1);
    col_done = col1;
  }
  dstamp(cs, "  last copy of a mesh done");
  dstamp(s, "  its last pack (+ step) done");
  if (e != cudaSuccess) rc = set_error(MCX_E_CUDA, "mesh upload: %s", cudaGetErrorString(e));
  if (rc) {
    if (cs != s) cudaStreamSynchronize(cs);  // no copy may still target the buffers freed below
    mcx_mesh_free(m);
    return rc;
  }
  *out = m;
  return MCX_OK;
}

// mcx_find_intersections, MCX_MODE_CULL on one device: the smaller mesh S is uploaded
// and packed on s1; the larger mesh L (the sweep side, SURVEY.md:379) is uploaded in
// chunks on s0 and the blocks of each chunk are searched against S as soon as they are
// packed (a stepped batch), so the search runs under the rest of the PCIe copy.
static int find_stepped(mcx_context* c, const double* coords_a, uint32_t NA, uint32_t MA, uint64_t pa,
                        const double* s_a, const double* coords_b, uint32_t NB, uint32_t MB, uint64_t pb,
                        const double* s_b, mcx_layer layer, const mcx_find_opts* fo, bool swap, mcx_mesh** A,
                        mcx_mesh** B, const mcx_record** records, uint64_t* n_records, const char** text,
                        uint64_t* text_bytes, mcx_stats* stats) {
  if (!c->stage.p) {
    CUDA_TRY(cudaMallocHost((void**)&c->stage.p, 1 << 20));
    c->stage.cap = 1 << 20;
  }
  StageScope scope(&c->stage);
  mcx_mesh** S = swap ? A : B;
  mcx_mesh** Lm = swap ? B : A;
  // every H2D copy on the one copy stream c->sc: S's chunks first at the full link rate,
  // then L's (packs of S on s1, packs and searches of L on s0, gated by chunk events)
  int rc = swap ? load_mesh(c, coords_a, NA, MA, s_a, c->s1, S, true, ChunkFn(), c->sc, pa)
                : load_mesh(c, coords_b, NB, MB, s_b, c->s1, S, true, ChunkFn(), c->sc, pb);
  trace("small mesh enqueued");
  if (rc) return rc;
  cudaError_t e = cudaEventRecord(c->ev, c->s1);
  if (e != cudaSuccess) return set_error(MCX_E_CUDA, "event: %s", cudaGetErrorString(e));
  mcx_opts o{};
  o.device = c->device;
  o.stream = c->s0;
  o.mode = MCX_MODE_CULL;
  o.pipeline = fo->pipeline;
  o.orient = MCX_ORIENT_AS_GIVEN;  // oriented here: L is the sweep side
  mcx_task whole{};
  uint64_t steps = 0;
  auto on_chunk = [&](mcx_mesh* m, uint64_t b0, uint64_t b1) -> int {
    int r = MCX_OK;
    if (steps == 0) {
      cudaError_t w = cudaStreamWaitEvent(c->s0, c->ev, 0);  // S is uploaded and packed
      if (w != cudaSuccess) return set_error(MCX_E_CUDA, "stream join: %s", cudaGetErrorString(w));
      whole = mcx_task{&m->view, &(*S)->view, 0, 0};
      o.cand_cap = c->cand_cap;
      const uint64_t wsb = mcx_batch_workspace_bytes(&whole, 1, &o);
      if ((r = ensure(c, c->ws, wsb, c->s0)) || (r = ensure(c, c->hits, sizeof(mcx_hit) * c->hit_cap, c->s0)) ||
          (r = ensure(c, c->hit_task, 4 * c->hit_cap, c->s0)) || (r = ensure_host(c->h_counters, 8 * 16)))
        return r;
      o.workspace = c->ws.p;
      o.workspace_bytes = c->ws.bytes;
    }
    const mcx_task t{&m->view, &(*S)->view, b0 * A_BLOCK, std::min<uint64_t>(b1 * A_BLOCK, m->view.n_tri)};
    const BatchStep step{&whole, steps == 0, swap};
    mcx_stats st{};
    r = launch_batch(&t, 1, &o, (mcx_hit*)c->hits.p, nullptr, c->hit_cap, &st,
                     (unsigned long long*)c->h_counters.p, &step, /*header_later=*/true);
    ++steps;
    return r;
  };
  rc = swap ? load_mesh(c, coords_b, NB, MB, s_b, c->s0, Lm, true, on_chunk, c->sc, pb)
            : load_mesh(c, coords_a, NA, MA, s_a, c->s0, Lm, true, on_chunk, c->sc, pa);
  trace("large mesh enqueued (stepped search)");
  if (rc) return rc;
  const mcx_job job{*A, *B, layer};
  const std::vector<JobDev> jd{job_of(*A, *B, layer)};
  bool retry = false, small_done = false;
  uint64_t total = 0;
  rc = after_search(c, &job, 1, fo, &o, jd, records, n_records, text, text_bytes, stats, &retry, &small_done, &total);
  if (rc) return rc;
  const bool spec = fo->pipeline == MCX_PIPE_SPEC;
  const uint64_t nA = (*A)->view.n_tri, nB = (*B)->view.n_tri;
  stats->n_pairs = spec ? (nA / 2) * (nB / 2) : nA * nB;
  if (retry) return intersect(c, &job, 1, fo, records, n_records, text, text_bytes, stats);  // regrown: from scratch
  if (small_done) return MCX_OK;
  return postprocess(c, total, nullptr, jd, fo, records, n_records, text, text_bytes, /*try_small=*/false);
}

}  // namespace mcx

extern "C" {

int mcx_context_create(int device, mcx_context** out) {
  using namespace mcx;
  if (!out) return set_error(MCX_E_ARG, "null argument");
  *out = nullptr;
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(device));
  mcx_context* c = new mcx_context();
  c->device = device;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  cudaError_t e = cudaMemPoolCreate(&c->pool, &props);
  if (e == cudaSuccess) {
    uint64_t keep = ~0ull;  // never hand memory back between calls
    e = cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->s0, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->s1, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->sc, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming);
  for (cudaEvent_t& ce : c->cev)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ce, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    mcx_context_destroy(c);
    return set_error(MCX_E_CUDA, "context creation: %s", cudaGetErrorString(e));
  }
  *out = c;
  return MCX_OK;
}

int mcx_context_destroy(mcx_context* c) {
  using namespace mcx;
  if (!c) return MCX_OK;
  DeviceGuard guard;
  cudaSetDevice(c->device);
  if (c->s0) {
    for (DevBuf* b : {&c->ws, &c->hits, &c->hit_task, &c->jobs, &c->k0, &c->k1, &c->v0, &c->v1, &c->recs, &c->recs_out,
                      &c->state, &c->blocked, &c->pairs, &c->lens, &c->offs, &c->cub, &c->text, &c->small, &c->flen,
                      &c->lines})
      release(c, *b, c->s0);
    cudaStreamSynchronize(c->s0);
  }
  for (HostBuf* b : {&c->h_recs, &c->h_text, &c->h_small, &c->h_counters, &c->h_map})
    if (b->p) cudaFreeHost(b->p);
  if (c->stage.p) cudaFreeHost(c->stage.p);
  if (c->sc) cudaStreamSynchronize(c->sc);
  delete c->up;  // joins the copy threads, frees the pinned slots
  if (c->ev) cudaEventDestroy(c->ev);
  for (cudaEvent_t ce : c->cev)
    if (ce) cudaEventDestroy(ce);
  if (c->s0) cudaStreamDestroy(c->s0);
  if (c->s1) cudaStreamDestroy(c->s1);
  if (c->sc) cudaStreamDestroy(c->sc);
  if (c->pool) cudaMemPoolDestroy(c->pool);
  delete c;
  return MCX_OK;
}

int mcx_mesh_load(mcx_context* c, const double* coords, uint32_t N, uint32_t M, const double* s_values,
                  mcx_mesh** mesh) {
  using namespace mcx;
  if (!c) return set_error(MCX_E_ARG, "null context");
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(c->device));
  int rc = load_mesh(c, coords, N, M, s_values, c->s0, mesh);
  if (rc == MCX_OK) CUDA_TRY(cudaStreamSynchronize(c->s0));
  return rc;
}

int mcx_mesh_free(mcx_mesh* m) {
  using namespace mcx;
  if (!m) return MCX_OK;
  mcx_context* c = m->ctx;
  DeviceGuard guard;
  cudaSetDevice(c->device);
  for (void* p : {m->owns_grid ? (void*)m->coords : nullptr, m->owns_grid ? (void*)m->s_values : nullptr, (void*)m->box,
                  (void*)m->perm, (void*)m->gbox, (void*)m->tbox, (void*)m->bbox, (void*)m->status})
    if (p) cudaFreeAsync(p, c->s0);
  delete m;
  return MCX_OK;
}

const mcx_mesh_dev* mcx_mesh_view(const mcx_mesh* m) { return m ? &m->view : nullptr; }

int mcx_grid_load(mcx_context* c, const double* coords, uint32_t N, uint32_t M, const double* s_values,
                  mcx_mesh** grid) {
  using namespace mcx;
  if (!c) return set_error(MCX_E_ARG, "null context");
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(c->device));
  int rc = load_mesh(c, coords, N, M, s_values, c->s0, grid, /*pack=*/false);
  if (rc == MCX_OK) CUDA_TRY(cudaStreamSynchronize(c->s0));
  return rc;
}

int mcx_mesh_view_columns(mcx_context* c, const mcx_mesh* parent, uint32_t c0, uint32_t c1, mcx_mesh** out) {
  using namespace mcx;
  if (!c || !parent || !out) return set_error(MCX_E_ARG, "null argument");
  if (parent->ctx != c) return set_error(MCX_E_ARG, "parent grid of another context");
  const uint32_t N = parent->view.N, Mp = parent->view.M;
  if (!(c0 < c1 && c1 < Mp))
    return set_error(MCX_E_ARG, "column range [%u, %u] must satisfy c0 < c1 < M = %u (SPEC.md:473)", c0, c1, Mp);
  const uint32_t M = c1 - c0 + 1;
  const uint64_t n = 2ull * N * (M - 1);
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->s0;
  mcx_mesh* m = new mcx_mesh();
  m->ctx = c;
  m->owns_grid = false;
  m->coords = parent->coords + (uint64_t)c0 * N;
  m->s_values = parent->s_values + c0;
  auto alloc = [&](void** p, size_t bytes) -> int {
    CUDA_TRY(cudaMallocFromPoolAsync(p, std::max<size_t>(bytes, 16), c->pool, s));
    return MCX_OK;
  };
  int rc = MCX_OK;
  if ((rc = alloc((void**)&m->box, 64 * n)) || (rc = alloc((void**)&m->perm, 4 * n)) ||
      (rc = alloc((void**)&m->gbox, 64 * ((n + GROUP - 1) / GROUP))) ||
      (rc = alloc((void**)&m->tbox, 64 * ((n + TILE - 1) / TILE))) ||
      (rc = alloc((void**)&m->bbox, 64 * ((n + A_BLOCK - 1) / A_BLOCK))) || (rc = alloc((void**)&m->status, 16)) ||
      (rc = pack_enqueue(m->coords, N, M, MCX_ORDER_TILED, m->box, m->perm, m->gbox, m->tbox, m->bbox, m->status, s,
                         0, 0, Mp))) {
    mcx_mesh_free(m);
    return rc;
  }
  m->view = mcx_mesh_dev{n, m->coords, N, M, m->box, m->perm, m->gbox, m->tbox, m->bbox, m->status, Mp, 0};
  *out = m;
  return MCX_OK;
}

int mcx_intersect(mcx_context* c, const mcx_job* jobs, uint32_t n_jobs, const mcx_find_opts* fo,
                  const mcx_record** records, uint64_t* n_records, const char** text, uint64_t* text_bytes,
                  mcx_stats* stats) {
  using namespace mcx;
  if (!c) return set_error(MCX_E_ARG, "null context");
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(c->device));
  return intersect(c, jobs, n_jobs, fo, records, n_records, text, text_bytes, stats);
}

int mcx_find_intersections(mcx_context* c, const double* coords_a, uint32_t NA, uint32_t MA, const double* s_a,
                           const double* coords_b, uint32_t NB, uint32_t MB, const double* s_b, mcx_layer layer,
                           const mcx_find_opts* fo, const mcx_record** records, uint64_t* n_records,
                           const char** text, uint64_t* text_bytes, mcx_stats* stats) {
  return mcx_find_intersections_strided(c, coords_a, NA, MA, 0, s_a, coords_b, NB, MB, 0, s_b, layer, fo, records,
                                        n_records, text, text_bytes, stats);
}

int mcx_find_intersections_strided(mcx_context* c, const double* coords_a, uint32_t NA, uint32_t MA,
                                   uint64_t plane_a, const double* s_a, const double* coords_b, uint32_t NB,
                                   uint32_t MB, uint64_t plane_b, const double* s_b, mcx_layer layer,
                                   const mcx_find_opts* fo, const mcx_record** records, uint64_t* n_records,
                                   const char** text, uint64_t* text_bytes, mcx_stats* stats) {
  using namespace mcx;
  if (!c) return set_error(MCX_E_ARG, "null context");
  int rc = check_find_opts(fo);
  if (rc) return rc;
  trace("begin");
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(c->device));
  dstamp(c->s0, "begin");
  mcx_mesh *A = nullptr, *B = nullptr;
  const uint64_t nA = (NA && MA >= 2) ? 2ull * NA * (MA - 1) : 0, nB = (NB && MB >= 2) ? 2ull * NB * (MB - 1) : 0;
  const bool swap = fo->orient == MCX_ORIENT_LARGER_A && nB > nA;
  const uint64_t nL = swap ? nB : nA, nS = swap ? nA : nB;  // L: the sweep side
  if (fo->mode == MCX_MODE_CULL && fo->shard_count <= 1 && nL >= STEP_MIN_TRI && nS && nS * step_ratio() <= nL &&
      !getenv("MCX_NO_STEPS")) {
    rc = find_stepped(c, coords_a, NA, MA, plane_a, s_a, coords_b, NB, MB, plane_b, s_b, layer, fo, swap, &A, &B,
                      records, n_records, text, text_bytes, stats);
    mcx_mesh_free(A);  // stream-ordered on s0, after everything above
    mcx_mesh_free(B);
    trace("end");
    dstamp_print();
    return rc;
  }
  // A packed on stream 0, B on stream 1; stream 0 waits for B.
  // every H2D copy on the copy stream c->sc, back to back at the link rate (A's chunks,
  // then B's); A's packs on s0 and B's on s1 follow their chunks through events, so no
  // copy waits for a pack
  rc = load_mesh(c, coords_a, NA, MA, s_a, c->s0, &A, true, ChunkFn(), c->sc, plane_a);
  trace("A enqueued");
  if (rc == MCX_OK) rc = load_mesh(c, coords_b, NB, MB, s_b, c->s1, &B, true, ChunkFn(), c->sc, plane_b);
  trace("B enqueued");
  if (rc == MCX_OK) {
    cudaError_t e = cudaEventRecord(c->ev, c->s1);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->s0, c->ev, 0);
    if (e != cudaSuccess) rc = set_error(MCX_E_CUDA, "stream join: %s", cudaGetErrorString(e));
  }
  if (rc == MCX_OK) {
    mcx_job j{A, B, layer};
    rc = intersect(c, &j, 1, fo, records, n_records, text, text_bytes, stats);
  }
  mcx_mesh_free(A);  // stream-ordered on s0, after everything above
  mcx_mesh_free(B);
  trace("end");
  dstamp_print();
  return rc;
}

int mcx_finish_hits(mcx_context* c, const mcx_hit* hits, uint64_t n_hits, const mcx_mesh* A, const mcx_mesh* B,
                    mcx_layer layer, const mcx_find_opts* fo, const mcx_record** records, uint64_t* n_records,
                    const char** text, uint64_t* text_bytes) {
  using namespace mcx;
  if (!c || !A || !B || !records || !n_records || (n_hits && !hits)) return set_error(MCX_E_ARG, "null argument");
  if (A->ctx != c || B->ctx != c) return set_error(MCX_E_ARG, "mesh of another context");
  int rc = check_find_opts(fo);
  if (rc) return rc;
  DeviceGuard guard;
  CUDA_TRY(cudaSetDevice(c->device));
  if ((rc = ensure(c, c->hits, sizeof(mcx_hit) * std::max<uint64_t>(n_hits, 1), c->s0))) return rc;
  if (n_hits) CUDA_TRY(cudaMemcpyAsync(c->hits.p, hits, sizeof(mcx_hit) * n_hits, cudaMemcpyHostToDevice, c->s0));
  // validate the indices on the device before any record reads the grids
  const uint64_t nA = A->view.n_tri, nB = B->view.n_tri;
  for (uint64_t k = 0; k < n_hits; ++k)
    if (hits[k].ia >= nA || hits[k].ib >= nB)
      return set_error(MCX_E_ARG, "hit %llu: triangle index outside the meshes", (unsigned long long)k);
  std::vector<JobDev> jd(1, job_of(A, B, layer));
  return postprocess(c, n_hits, nullptr, jd, fo, records, n_records, text, text_bytes);
}

int mcx_format_g17(double v, char* out) {
  if (!out) return mcx::set_error(MCX_E_ARG, "null buffer");
  const int n = mcx::fmt::fmt_g17(v, out);
  out[n] = 0;
  return n;
}

}  // extern "C"
