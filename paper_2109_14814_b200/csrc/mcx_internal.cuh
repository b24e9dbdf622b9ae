// mcx_internal.cuh — entry points shared between the translation units of libmcx.so
// (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mcx.h"

namespace mcx {

// mcx_pack.cu: the fused pack + levels kernel over 1024-record blocks [b0, b1) (b1 = 0:
// all), enqueued on `stream` (device current); pack_blocks = the block count.
uint64_t pack_blocks(uint32_t N, uint32_t M);
// Mp = plane stride in rows (0 → M; the parent's M for a column view of a larger grid).
int pack_enqueue(const double* coords, uint32_t N, uint32_t M, int order, double* box, uint32_t* perm, double* gbox,
                 double* tbox, double* bbox, uint32_t* status, cudaStream_t stream, uint64_t b0, uint64_t b1,
                 uint32_t Mp);

// mcx_search.cu: a batch of searches (device current).  h_counters == nullptr:
// synchronises o->stream and fills the stats.  Otherwise the workspace header (8 + 8·n
// u64s) is copied to h_counters (pinned) asynchronously, only stats[t].n_pairs is set,
// and the caller synchronises and calls batch_stats (requires o->timing == 0).
//
// step != nullptr: this call is one step of a sequence over A-ranges of the same tasks
// sharing one workspace (MCX_MODE_CULL only): the workspace layout is that of
// step->whole (the tasks with their full ranges), only the first step zeroes the
// counters, each step's cull / solve kernels take the block-list and candidate entries
// the previous steps left unprocessed (header words 5 and 6), and the tasks are used as
// given with the solve un-swapping every hit when step->swap (the caller oriented them).
struct BatchStep {
  const mcx_task* whole;
  bool first;
  bool swap;
};
// header_later: with h_counters, skip the header copy — the caller enqueues it (e.g.
// after kernels that only need the header on the device).
int launch_batch(const mcx_task* tasks, uint32_t n, const mcx_opts* o, mcx_hit* hits, uint32_t* hit_task,
                 uint64_t cap, mcx_stats* st, unsigned long long* h_counters, const BatchStep* step = nullptr,
                 bool header_later = false);
int batch_stats(const unsigned long long* h, uint32_t n, const mcx_opts* o, uint64_t cap, mcx_stats* st, float ms);

// mcx_search.cu: one-time per (kernel, device, threads, smem) launch setup — the
// dynamic shared memory opt-in (+ the shared-memory carveout when carveout >= 0) and
// the resident CTAs per SM × SM count — cached, since each of these host calls costs
// microseconds on every small search otherwise.  `device` is the current device.
int kernel_prepare(const void* fn, int threads, size_t smem, int carveout, int device, uint64_t* slots);

// mcx_runtime.cu: MCX_TRACE=2 device-side stamp (a CUDA event recorded on s, printed
// when the runtime call ends); no-op otherwise.
void dstamp(cudaStream_t s, const char* what);

}  // namespace mcx
