// mcx_prefilter.cuh — MCX_MODE_PREFILTER: every pair tested by a conservative
// packed-integer test on quantised boxes (fma + alu pipes), its passes by the exact
// FP64 test.  Included by mcx_search.cu (one translation unit).
#pragma once
#include "mcx_search.cuh"

namespace mcx {

// ------------------------------------------------------------ prefilter mode
// MCX_MODE_PREFILTER: every pair is tested, but first by a conservative integer
// test on quantised boxes that runs on the fma + alu pipes instead of the FP64 pipe
// (64 lanes/clk/SM on B200, 8 DSETP per pair); only pairs it cannot reject get the
// exact FP64 box test and then the canonical solve, so the AABB-pass / singular /
// hit sets are exactly those of MCX_MODE_BRUTE.
//   * fp32 boxes rounded outwards (lo toward −∞, hi toward +∞) are computed once per
//     call (fbox_kernel).  Every later step is a monotone fp32 function of them, so
//     A.lo ≤ B.hi ⇒ qlo_A ≤ qhi_B: the quantised test only ever keeps extra pairs.
//   * Frame = union box of the warp's own 512 A records (a 16×16-quad tile of the
//     tiled storage order; LCfg::WFRAME, else the CTA's 1024): o_c = min lo_c,
//     κ_c = 6 / (max hi_c − o_c) (0 if the extent is 0 or not finite);
//     q(x) = clamp(⌊(x − o)·κ⌋ or ⌈·⌉, 0, 6).  3 bits per bound suffice in a frame
//     that small, so all 8 compares of a pair fit ONE 32-bit word of eight 4-bit
//     fields (value 0..6 + guard bit 3).
//   * B words: nibble c = qlo_c, nibble 4+c = 6 − qhi_c.  A B record whose fp32 box
//     misses the frame cannot overlap any record of the block: it gets nibble 0 = 7,
//     which fails against every A word because qhi_A ≤ 6.
//   * A words: nibble c = 8 + qhi_c, nibble 4+c = 14 − qlo_c.  H − L then has, per
//     nibble, 8 + qhi_A − qlo_B ∈ [1, 15] (no borrow between nibbles) — guard bit
//     set iff qlo_B ≤ qhi_A — and 8 + qhi_B − qlo_A.  Invalid A slots: 0x77777777.
//   * Pair test (full words) = IMAD (L·(−1) + H, fma pipe) + half a LOP3.LUT.PAND (alu
//     pipe): one LOP3 with LUT ~x_a & ~x_b & G per two A words, predicate output ANDed
//     into one of 4 "all fail" chains — "both fail at a common guard position", a
//     conservative "both fail".  1.5 instructions per pair.  One warp vote per JB B
//     records.  The default kernel tests 4 of the 8 compares on 16-bit half words, two
//     pairs per subtraction, folded four per LOP3 into per-group accumulators (0.75
//     instructions per pair: "Half words" and "Accumulated folds" below), and runs the
//     full word test only on voting groups.
//   * B records reach shared memory as fp32 boxes (bulk copies, 8 KB stages); each
//     warp quantises each tile into its own frame (~1/20 of the test work) before
//     testing it.
//   * On a vote the warp re-tests that B record against its A words (kept in shared
//     memory) and runs the exact FP64 box test on the quantised passes from L1/L2;
//     survivors are queued and solved exactly like the FP64 kernel.
constexpr int Q_QCAP = 64;

// a − b computed as b·(−1) + a on the fma pipe (m1 = 0xffffffff at run time).
__device__ __forceinline__ unsigned imad_sub(unsigned a, unsigned m1, unsigned b) {
  unsigned r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(m1), "r"(a));
  return r;
}

// xa = ha − l with borrow-out, xb = hb − l − borrow.  H > L always holds (every H
// nibble ≥ 7 ≥ every L nibble, H ≠ L), so the borrow is 0 and xb = hb − l; the chain
// only makes ptxas put the first subtraction on the alu pipe (IADD3 with carry-out).
__device__ __forceinline__ void sub2_cc(unsigned& xa, unsigned& xb, unsigned ha, unsigned hb, unsigned l) {
  asm("sub.cc.u32 %0, %2, %4;\n subc.u32 %1, %3, %4;" : "=r"(xa), "=r"(xb) : "r"(ha), "r"(hb), "r"(l));
}

// Half words (LCfg::HALF): the fast sweep tests 4 of the 8 compares (both bounds of dims 0
// and 1) on 16-bit halves of the same words — nibbles 0, 1, 4, 5 — so one 32-bit subtraction
// tests two pairs: H = half(A_r) | half(A_r') << 16, L = half(B) · 0x10001.  Fields never
// borrow (H nibble ≥ 7 ≥ L nibble), and the frame-miss code (B nibble 0 = 7) is in the half.
// "All fail" must hold for every pair a LOP3 covers, and a 32-bit LOP3 ORs its bits, so one
// LOP3 per half: ~x_a & ~x_b & G_LO (pairs (r, u), (r″, u) fail at a common compare) and the
// same with G_HI — 1 instruction per pair instead of 1.5 (1 subtraction per 2 pairs on the
// fma pipe, 1 LOP3 per 2 pairs on the alu pipe).  A 4-compare pass is conservative for the
// 8-compare test, which the vote path then runs on the full words, so the exact-test, pass
// and hit sets are unchanged.
constexpr unsigned G_LO = 0x00008888u, G_HI = 0x88880000u;
__device__ __forceinline__ unsigned half16(unsigned w) { return (w & 0xffu) | ((w >> 8) & 0xff00u); }

// Accumulated folds (LCfg::ACC): y_k = ~x_a & ~x_b & y_k over the whole vote group of JB B
// records (y_k starts at G4; one LOP3 per two subtraction results = per 4 pair tests, no
// mask operand), then per accumulator "(y_k & G_LO) != 0 and (y_k & G_HI) != 0": every low
// (high) pair the accumulator saw fails at one common compare — a conservative "all fail".
// Weaker than the per-LOP3 test (the common compare must be shared by the whole group), but
// the B records that miss the warp's frame — nearly all of them — all fail at nibble 0, so
// a group votes only when it holds a record inside the frame; a vote re-runs the per-LOP3
// half test per record (exact "all four fail"), and its passes go to the full word test.
// Per 16 pairs: 8 subtractions (6 IMAD + 2 IADD3 via borrow chains) + 4 LOP3 = 12
// instructions, 6 per pipe: 0.75 per pair.
__device__ __forceinline__ unsigned fold2(unsigned xa, unsigned xb, unsigned y) {
  unsigned r;
  asm("lop3.b32 %0, %1, %2, %3, 0x02;" : "=r"(r) : "r"(xa), "r"(xb), "r"(y));
  return r;
}

constexpr int FTILE = 256;  // B records per stage (256 × 32 B = 8 KB)
constexpr unsigned G4 = 0x88888888u;

template <int QR_, int JB_, int UNROLL_, int MINB_ = 1, bool PAIR2_ = false, bool WFRAME_ = false, int CHAINS_ = 0,
          bool HALF_ = false, int FT_ = FTILE, bool SHQ_ = false, bool ACC_ = false, int CHMASK_ = 0,
          int ACCSETS_ = 1, bool ACCAND_ = false>
struct LCfg {
  // ACC: test the AND of the accumulators (one common failing compare over the whole group
  // — still conservative, cheaper than testing each accumulator)
  static constexpr bool ACCAND = ACCAND_;
  // ACC: accumulator sets, alternated by B record (more independent fold chains, and each
  // accumulator covers fewer pairs, so fewer spurious votes)
  static constexpr int ACCSETS = ACCSETS_;
  // ACC: bit st set = slot pair st (of 4 per B record) uses a borrow chain (overrides CHAINS)
  static constexpr int CHMASK = CHMASK_;
  // HALF only: fold every subtraction result of a vote group into 4 accumulators (one LOP3
  // per two results, no mask operand) and test the accumulators once per group — see
  // "Accumulated folds" above
  static constexpr bool ACC = ACC_ && HALF_;
  // per-warp frames, quantised by the whole CTA: a B record outside the union of the
  // CTA's frames is coded "miss" for every warp after ONE in-frame test instead of one per warp
  static constexpr bool SHQ = SHQ_ && WFRAME_;
  static constexpr int FT = FT_;  // B records per shared-memory stage
  // two pair tests per subtraction: 16-bit words holding the 4 compares of dims 0 and 1
  // (the full 8-compare word is re-tested on a vote) — see "Half words" above
  static constexpr bool HALF = HALF_;
  // pairs of A slots (of every 8) whose two subtractions form a borrow chain, so that ptxas
  // must put the first on the alu pipe (IADD3 with carry-out) instead of the fma pipe
  static constexpr int CHAINS = CHAINS_;
  static constexpr bool PAIR2 = PAIR2_;    // one LOP3 for two pair tests (conservative "both fail")
  static constexpr bool WFRAME = WFRAME_;  // one frame per warp (its 32·QR A records) instead of per CTA
  static constexpr int QR = QR_;
  static constexpr int JB = JB_;
  static constexpr int UNROLL = UNROLL_;
  static constexpr int MINB = MINB_;
  static constexpr int THREADS = A_BLOCK / QR_;
  static constexpr int WARPS = THREADS / 32;
  static_assert(WARPS >= 1 && THREADS % 32 == 0, "QR must leave whole warps in a 1024-record block");
  static constexpr int NF = WFRAME ? WARPS : 1;  // frames (and quantised B tiles) per CTA
};

template <class C>
struct __align__(16) LSmem {
  float4 tile[STAGES][C::FT][2];
  unsigned qt[C::NF][C::FT];
  uint2 queue[C::WARPS][Q_QCAP];
  float frame[C::WARPS][8];
  float fr[C::NF][16];
  float cfr[8];  // SHQ: union of the CTA's frames (lo_c, hi_c)
  unsigned aw[C::WARPS][C::QR][32];  // the A words, reloaded from here after a slow path
  unsigned long long full[STAGES];
};

// allfail &= "x_a and x_b have a guard bit clear at a common position" (LOP3 LUT 0x02 =
// ~x_a & ~x_b & G4): true only if both pairs fail, so it is a conservative "both fail"
// (a pass of either clears it; two fails at different positions give a spurious vote,
// which the slow path resolves).  One alu instruction per two pair tests.
__device__ __forceinline__ void fail_and2(unsigned& allfail, unsigned xa, unsigned xb) {
  // the LOP3 result register d is unused: only its != 0 predicate matters
  asm("{\n .reg .pred p;\n .reg .b32 d;\n setp.ne.u32 p, %0, 0;\n lop3.and.b32 d|p, %1, %2, %3, 0x02, p;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "+r"(allfail)
      : "r"(xa), "r"(xb), "r"(G4));
}

// allfail &= "x_a and x_b have a guard bit of mask g clear at a common position".
__device__ __forceinline__ void fail_and2m(unsigned& allfail, unsigned xa, unsigned xb, unsigned g) {
  asm("{\n .reg .pred p;\n .reg .b32 d;\n setp.ne.u32 p, %0, 0;\n lop3.and.b32 d|p, %1, %2, %3, 0x02, p;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "+r"(allfail)
      : "r"(xa), "r"(xb), "r"(g));
}

// allfail &= "x has a guard bit clear" (LOP3 LUT 0x0a = ~x & G4).
__device__ __forceinline__ void fail_and1(unsigned& allfail, unsigned x) {
  asm("{\n .reg .pred p;\n .reg .b32 d;\n setp.ne.u32 p, %0, 0;\n lop3.and.b32 d|p, %1, %1, %2, 0x0a, p;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "+r"(allfail)
      : "r"(x), "r"(G4));
}

// Conservative fp32 boxes of every distinct mesh of the batch (blockIdx.y = job).
__global__ void __launch_bounds__(256) fbox_kernel(const Batch Bt) {
  const FboxJob J = Bt.fjobs[blockIdx.y];
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < J.n; k += (uint64_t)gridDim.x * blockDim.x) {
    const double2* b = reinterpret_cast<const double2*>(J.src + k);
    const double2 l01 = __ldg(b), l23 = __ldg(b + 1), h01 = __ldg(b + 2), h23 = __ldg(b + 3);
    J.dst[2 * k] = make_float4(__double2float_rd(l01.x), __double2float_rd(l01.y), __double2float_rd(l23.x),
                               __double2float_rd(l23.y));
    J.dst[2 * k + 1] = make_float4(__double2float_ru(h01.x), __double2float_ru(h01.y), __double2float_ru(h23.x),
                                   __double2float_ru(h23.y));
  }
}

__device__ __forceinline__ unsigned qfloor(float x, float o, float k) {
  return (unsigned)__float2int_rd(fminf(fmaxf(__fmul_rn(__fsub_rn(x, o), k), 0.f), 6.f));
}
__device__ __forceinline__ unsigned qceil(float x, float o, float k) {
  return (unsigned)__float2int_ru(fminf(fmaxf(__fmul_rn(__fsub_rn(x, o), k), 0.f), 6.f));
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB) search_local_kernel(const Batch Bt) {
  constexpr int QR = C::QR;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  LSmem<C>& S = *reinterpret_cast<LSmem<C>*>(smem_raw);
  __shared__ SearchParams Ps;
  __shared__ uint64_t s_unit;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    const uint32_t t = find_task(Bt, blockIdx.x);
    Ps = Bt.tasks[t];
    s_unit = blockIdx.x - Bt.prefix[t];
  }
  __syncthreads();
  const SearchParams& P = Ps;
  const uint64_t unit = s_unit;
  const uint64_t gblk = P.blk_first + (unit / P.nchunk) * P.shard_count;
  const uint64_t a0 = gblk * A_BLOCK;
  const uint64_t b0 = (unit % P.nchunk) * P.b_chunk;
  const uint64_t b1 = min(b0 + P.b_chunk, P.nB);
  const int ntiles = (int)((b1 - b0 + C::FT - 1) / C::FT);
  const unsigned m1 = Bt.neg1;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&S.full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < STAGES && s < ntiles; ++s) {
      const uint64_t tb = b0 + (uint64_t)s * C::FT;
      const uint32_t bytes = (uint32_t)(min((uint64_t)C::FT, b1 - tb) * 32);
      mbar_arrive_expect_tx(&S.full[s], bytes);
      bulk_g2s(&S.tile[s][0][0], P.fB + 2 * tb, bytes, &S.full[s]);
    }
  }

  // ---- frame of the block: union of the CTA's valid A records (all warps)
  const uint32_t abase = (uint32_t)(a0 + (uint64_t)warp * (QR * 32) + lane);
  float lo[4], hi[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) { lo[c] = __int_as_float(0x7f800000); hi[c] = -lo[c]; }
#pragma unroll 4
  for (int r = 0; r < QR; ++r) {
    const uint32_t ia = abase + r * 32;
    if (ia >= P.a_begin && ia < P.a_end) {
      const float4 l = __ldg(P.fA + 2 * (uint64_t)ia), h = __ldg(P.fA + 2 * (uint64_t)ia + 1);
      lo[0] = fminf(lo[0], l.x); lo[1] = fminf(lo[1], l.y); lo[2] = fminf(lo[2], l.z); lo[3] = fminf(lo[3], l.w);
      hi[0] = fmaxf(hi[0], h.x); hi[1] = fmaxf(hi[1], h.y); hi[2] = fmaxf(hi[2], h.z); hi[3] = fmaxf(hi[3], h.w);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      lo[c] = fminf(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmaxf(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < 4; ++c) { S.frame[warp][c] = lo[c]; S.frame[warp][4 + c] = hi[c]; }
  }
  __syncthreads();
  // frame parameters in shared memory: fr[0..3] = o_c, fr[4..7] = κ_c, fr[8..11] = lo_c, fr[12..15] = hi_c
  const int fi = C::WFRAME ? warp : 0;  // this warp's frame / quantised B tile
  if ((C::WFRAME ? lane : tid) < 4) {
    const int c = C::WFRAME ? lane : tid;
    float l = S.frame[fi][c], h = S.frame[fi][4 + c];
    if (!C::WFRAME)
      for (int w = 1; w < C::WARPS; ++w) { l = fminf(l, S.frame[w][c]); h = fmaxf(h, S.frame[w][4 + c]); }
    const float e = __fsub_rn(h, l);
    float k = (e > 0.f && e < 3.0e38f) ? __fdiv_rn(6.f, e) : 0.f;  // also 0 for an empty frame (l > h)
    if (!(k < 3.0e38f)) k = 0.f;
    S.fr[fi][c] = (k > 0.f) ? l : 0.f;
    S.fr[fi][4 + c] = k;
    S.fr[fi][8 + c] = l;
    S.fr[fi][12 + c] = h;
  }
  if (C::SHQ && tid < 8) {
    float v = S.frame[0][tid];
    for (int w = 1; w < C::WARPS; ++w) v = tid < 4 ? fminf(v, S.frame[w][tid]) : fmaxf(v, S.frame[w][tid]);
    S.cfr[tid] = v;
  }
  __syncthreads();

  float cfr[8];  // SHQ: the CTA frame in registers (read once per B record)
#pragma unroll
  for (int c = 0; c < 8; ++c) cfr[c] = C::SHQ ? S.cfr[c] : 0.f;

  // ---- A words in registers
  auto a_word = [&](uint32_t ia) -> unsigned {
    const float* fr = S.fr[fi];
    const float4 l = __ldg(P.fA + 2 * (uint64_t)ia), h = __ldg(P.fA + 2 * (uint64_t)ia + 1);
    return ((8u + qceil(h.x, fr[0], fr[4])) << 0) | ((8u + qceil(h.y, fr[1], fr[5])) << 4) |
           ((8u + qceil(h.z, fr[2], fr[6])) << 8) | ((8u + qceil(h.w, fr[3], fr[7])) << 12) |
           ((14u - qfloor(l.x, fr[0], fr[4])) << 16) | ((14u - qfloor(l.y, fr[1], fr[5])) << 20) |
           ((14u - qfloor(l.z, fr[2], fr[6])) << 24) | ((14u - qfloor(l.w, fr[3], fr[7])) << 28);
  };
  for (int r = 0; r < QR; ++r) {
    const uint32_t ia = abase + r * 32;
    S.aw[warp][r][lane] = (ia >= P.a_begin && ia < P.a_end) ? a_word(ia) : 0x77777777u;  // all guards clear
  }
  __syncwarp();
  constexpr int NH = C::HALF ? QR / 2 : QR;
  unsigned hw[NH];
  auto load_a = [&]() {
    if constexpr (C::HALF) {
#pragma unroll
      for (int k = 0; k < NH; ++k)
        hw[k] = half16(*(volatile unsigned*)&S.aw[warp][2 * k][lane]) |
                (half16(*(volatile unsigned*)&S.aw[warp][2 * k + 1][lane]) << 16);
    } else {
#pragma unroll
      for (int r = 0; r < QR; ++r) hw[r] = *(volatile unsigned*)&S.aw[warp][r][lane];
    }
  };
  load_a();

  uint2* q = S.queue[warp];
  int qn = 0;
  unsigned long long n_exact = 0;
  const unsigned lt_mask = (1u << lane) - 1u;

  // Rare path for B record ib (word bw): the lane's quantised passes as a bit mask over
  // its A slots, then the exact FP64 box test for them only, one pass per lane per round.
  auto slow = [&](uint32_t ib, unsigned bw) {
    unsigned msk = 0;
#pragma unroll
    for (int r = 0; r < QR; ++r)  // invalid A slots never pass
      msk |= (((S.aw[warp][r][lane] - bw) & G4) == G4) ? (1u << r) : 0u;
    if (!__any_sync(0xffffffffu, msk != 0)) return;  // a spurious vote of the paired LOP3 test
    const double2* bp = reinterpret_cast<const double2*>(P.boxB + ib);
    const double2 l01 = __ldg(bp), l23 = __ldg(bp + 1), g01 = __ldg(bp + 2), g23 = __ldg(bp + 3);
    while (__any_sync(0xffffffffu, msk != 0)) {
      bool p = false;
      uint32_t ia = 0;
      if (msk) {
        const int r = __ffs(msk) - 1;
        msk &= msk - 1;
        ++n_exact;
        ia = abase + r * 32;
        const double2* ap = reinterpret_cast<const double2*>(P.boxA + ia);
        const double2 a01 = __ldg(ap), a23 = __ldg(ap + 1), c01 = __ldg(ap + 2), c23 = __ldg(ap + 3);
        p = (l01.x <= c01.x) & (a01.x <= g01.x) & (l01.y <= c01.y) & (a01.y <= g01.y) &
            (l23.x <= c23.x) & (a23.x <= g23.x) & (l23.y <= c23.y) & (a23.y <= g23.y);
      }
      const unsigned m = __ballot_sync(0xffffffffu, p);
      if (m) {
        if (p) q[qn + __popc(m & lt_mask)] = make_uint2(ia, ib);
        qn += __popc(m);
        __syncwarp();
        if (qn >= 32) {
          qn -= 32;
          flush_queue(P, Bt, q + qn, 32, lane);
        }
      }
    }
  };

  for (int t = 0; t < ntiles; ++t) {
    const int s = t % STAGES;
    mbar_wait(&S.full[s], (uint32_t)((t / STAGES) & 1));
    const uint64_t tb = b0 + (uint64_t)t * C::FT;
    const int nvalid = (int)min((uint64_t)C::FT, b1 - tb);
    // quantise this tile's B records into the frame (per CTA: all threads; per warp: its lanes)
    auto b_word_f = [&](const float4& l, const float4& h, const float* fr) -> unsigned {
      const bool in = (l.x <= fr[12]) & (fr[8] <= h.x) & (l.y <= fr[13]) & (fr[9] <= h.y) & (l.z <= fr[14]) &
                      (fr[10] <= h.z) & (l.w <= fr[15]) & (fr[11] <= h.w);
      unsigned w = 7u;  // misses the frame: nibble 0 = 7 fails against every A word
      if (in)
        w = qfloor(l.x, fr[0], fr[4]) | (qfloor(l.y, fr[1], fr[5]) << 4) | (qfloor(l.z, fr[2], fr[6]) << 8) |
            (qfloor(l.w, fr[3], fr[7]) << 12) | ((6u - qceil(h.x, fr[0], fr[4])) << 16) |
            ((6u - qceil(h.y, fr[1], fr[5])) << 20) | ((6u - qceil(h.z, fr[2], fr[6])) << 24) |
            ((6u - qceil(h.w, fr[3], fr[7])) << 28);
      return w;
    };
    auto b_word = [&](int j) -> unsigned { return b_word_f(S.tile[s][j][0], S.tile[s][j][1], S.fr[fi]); };
    auto enc = [](unsigned w) -> unsigned { return C::HALF ? half16(w) * 0x10001u : w; };  // HALF: the B half twice
    if constexpr (C::SHQ) {
      // a B record inside the CTA frame (rare) is quantised into each warp frame, every other
      // one gets the miss code; the frame test of a full tile's PER records per thread is
      // issued as independent loads and compare chains (it was latency-bound)
      auto in_cta = [&](const float4& l, const float4& h) -> bool {
        const bool i0 = (l.x <= cfr[4]) & (cfr[0] <= h.x) & (l.y <= cfr[5]) & (cfr[1] <= h.y);
        const bool i1 = (l.z <= cfr[6]) & (cfr[2] <= h.z) & (l.w <= cfr[7]) & (cfr[3] <= h.w);
        return i0 & i1;
      };
      auto put = [&](int j, bool in) {
        if (in) {
          const float4 l = S.tile[s][j][0], h = S.tile[s][j][1];
#pragma unroll
          for (int f = 0; f < C::NF; ++f) S.qt[f][j] = enc(b_word_f(l, h, S.fr[f]));
        } else {
#pragma unroll
          for (int f = 0; f < C::NF; ++f) S.qt[f][j] = enc(7u);
        }
      };
      constexpr int PER = C::FT / C::THREADS;
      if (PER >= 1 && C::FT % C::THREADS == 0 && nvalid == C::FT) {
        bool in[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) in[q] = in_cta(S.tile[s][tid + q * C::THREADS][0], S.tile[s][tid + q * C::THREADS][1]);
#pragma unroll
        for (int q = 0; q < PER; ++q) put(tid + q * C::THREADS, in[q]);
      } else {
        for (int j = tid; j < nvalid; j += C::THREADS) put(j, in_cta(S.tile[s][j][0], S.tile[s][j][1]));
      }
      __syncthreads();
    } else {
      for (int j = C::WFRAME ? lane : tid; j < nvalid; j += C::WFRAME ? 32 : C::THREADS) S.qt[fi][j] = enc(b_word(j));
      if constexpr (C::WFRAME) __syncwarp();  // each warp reads only the words it wrote
      else __syncthreads();
    }
    auto step = [&](int j, auto jb_c) {
      constexpr int NJ = decltype(jb_c)::value;
      unsigned bw[NJ];
      unsigned allfail[4] = {1, 1, 1, 1};
#pragma unroll
      for (int u = 0; u < NJ; ++u) {
        bw[u] = S.qt[fi][j + u];
        if constexpr (C::HALF) {
#pragma unroll
          for (int k = 0; k < NH; k += 2) {
            const unsigned xa = imad_sub(hw[k], m1, bw[u]), xb = imad_sub(hw[k + 1], m1, bw[u]);
            fail_and2m(allfail[k & 3], xa, xb, G_LO);
            fail_and2m(allfail[(k + 1) & 3], xa, xb, G_HI);
          }
        } else if constexpr (C::PAIR2) {
#pragma unroll
          for (int r = 0; r < QR; r += 2) {
            const int st = (r >> 1) & 7;  // chains spread evenly over the 8 slot pairs
            if (((st + 1) * C::CHAINS) / 8 != (st * C::CHAINS) / 8) {
              unsigned xa, xb;  // borrow chain: the first subtraction must be an alu IADD3
              sub2_cc(xa, xb, hw[r], hw[r + 1], bw[u]);
              fail_and2(allfail[(r >> 1) & 3], xa, xb);
            } else {
              fail_and2(allfail[(r >> 1) & 3], imad_sub(hw[r], m1, bw[u]), imad_sub(hw[r + 1], m1, bw[u]));
            }
          }
        } else {
#pragma unroll
          for (int r = 0; r < QR; ++r) fail_and1(allfail[r & 3], imad_sub(hw[r], m1, bw[u]));
        }
      }
      if (__any_sync(0xffffffffu, (allfail[0] & allfail[1] & allfail[2] & allfail[3]) == 0)) {
#pragma unroll 1
        for (int u = 0; u < NJ; ++u) slow((uint32_t)(tb + j + u), C::HALF ? b_word(j + u) : S.qt[fi][j + u]);
        load_a();
      }
    };
    // the per-record half test (HALF): true if some lane has a pair of B record j + u that
    // passes the 4 compares
    auto half_any = [&](unsigned b) -> bool {
      unsigned af[4] = {1, 1, 1, 1};
#pragma unroll
      for (int k = 0; k < NH; k += 2) {
        const unsigned xa = imad_sub(hw[k], m1, b), xb = imad_sub(hw[k + 1], m1, b);
        fail_and2m(af[k & 3], xa, xb, G_LO);
        fail_and2m(af[(k + 1) & 3], xa, xb, G_HI);
      }
      return __any_sync(0xffffffffu, (af[0] & af[1] & af[2] & af[3]) == 0);
    };
    auto step_acc = [&](int j, auto jb_c) {
      constexpr int NJ = decltype(jb_c)::value;
      constexpr int NY = NH / 2 * C::ACCSETS;
      unsigned y[NY];
#pragma unroll
      for (int k = 0; k < NY; ++k) y[k] = G4;
#pragma unroll
      for (int u = 0; u < NJ; ++u) {
        const unsigned b = S.qt[fi][j + u];
#pragma unroll
        for (int k = 0; k < NH; k += 2) {
          const int st = (k >> 1) & 3;
          unsigned xa, xb;
          constexpr int CH = C::CHAINS < 0 ? -C::CHAINS : C::CHAINS;
          const bool chain = C::CHMASK ? ((C::CHMASK >> st) & 1) : (((st + 1) * CH) / 4 != (st * CH) / 4);
          if (chain) {
            if constexpr (C::CHAINS < 0) {  // IADD3 with a (dead) carry-out: alu pipe, no chain
              asm("sub.cc.u32 %0, %1, %2;" : "=r"(xa) : "r"(hw[k]), "r"(b));
              xb = imad_sub(hw[k + 1], m1, b);
            } else {
              sub2_cc(xa, xb, hw[k], hw[k + 1], b);  // the first subtraction on the alu pipe
            }
          } else {
            xa = imad_sub(hw[k], m1, b);
            xb = imad_sub(hw[k + 1], m1, b);
          }
          const int ya = (u % C::ACCSETS) * (NH / 2) + (k >> 1);
          y[ya] = fold2(xa, xb, y[ya]);
        }
      }
      bool fail = true;
      if constexpr (C::ACCAND) {
        unsigned t = y[0];
#pragma unroll
        for (int k = 1; k < NY; ++k) t &= y[k];
        fail = ((t & G_LO) != 0u) & ((t & G_HI) != 0u);
      } else {
#pragma unroll
        for (int k = 0; k < NY; ++k) fail &= ((y[k] & G_LO) != 0u) & ((y[k] & G_HI) != 0u);
      }
      if (__any_sync(0xffffffffu, !fail)) {
        // B records of the group with a 4-compare pass somewhere in the warp, 64 per word
        constexpr int NW = (NJ + 63) / 64;
        uint64_t need[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) need[w] = 0;
#pragma unroll 1
        for (int u = 0; u < NJ; ++u)
          if (half_any(S.qt[fi][j + u])) need[u >> 6] |= 1ull << (u & 63);
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          while (need[w]) {
            const int u = w * 64 + __ffsll((long long)need[w]) - 1;
            need[w] &= need[w] - 1;
            slow((uint32_t)(tb + j + u), b_word(j + u));
          }
        }
        load_a();
      }
    };
    const int nmain = nvalid - nvalid % C::JB;
#pragma unroll(C::UNROLL)
    for (int j = 0; j < nmain; j += C::JB) {
      if constexpr (C::ACC) step_acc(j, std::integral_constant<int, C::JB>());
      else step(j, std::integral_constant<int, C::JB>());
    }
    for (int j = nmain; j < nvalid; ++j) step(j, std::integral_constant<int, 1>());
    __syncthreads();  // every warp is done reading stage s and qt
    if (tid == 0 && t + STAGES < ntiles) {
      const uint64_t nb = b0 + (uint64_t)(t + STAGES) * C::FT;
      const uint32_t bytes = (uint32_t)(min((uint64_t)C::FT, b1 - nb) * 32);
      mbar_arrive_expect_tx(&S.full[s], bytes);
      bulk_g2s(&S.tile[s][0][0], P.fB + 2 * nb, bytes, &S.full[s]);
    }
  }
  __syncwarp();
  if (qn > 0) flush_queue(P, Bt, q, qn, lane);
  flush_tested(P, lane, n_exact);
}

// MCX_MODE_PREFILTER: conservative fp32 boxes → prefilter search.
template <class C>
static int launch_local_cfg(std::vector<SearchParams>& T, Batch& Bt, std::vector<uint64_t>& prefix, void* dev_tab,
                            const std::vector<FboxJob>& jobs, void* dev_jobs, int device, cudaStream_t stream) {
  const size_t smem = sizeof(LSmem<C>);
  uint64_t slots = 0, total = 0;
  int rc = resident_slots(search_local_kernel<C>, C::THREADS, smem, device, &slots);
  if (rc == MCX_OK) rc = upload_plan(T, Bt, prefix, dev_tab, slots, 8, stream, &total, C::FT);
  if (rc != MCX_OK || total == 0) return rc;
  if (jobs.size() > 65535) return set_error(MCX_E_ARG, "MCX_MODE_PREFILTER supports at most 65535 meshes per batch");
  Bt.neg1 = 0xffffffffu;
  Bt.fjobs = reinterpret_cast<const FboxJob*>(dev_jobs);
  Bt.n_fjobs = (uint32_t)jobs.size();
  CUDA_TRY(h2d_async(dev_jobs, jobs.data(), sizeof(FboxJob) * jobs.size(), stream));
  uint64_t max_records = 0;
  for (const FboxJob& j : jobs) max_records = std::max<uint64_t>(max_records, j.n);
  const unsigned n = (unsigned)jobs.size();
  uint64_t gx = (max_records + 1023) / 1024;  // ~4 records per thread, ~2 blocks per search slot overall
  const uint64_t gcap = std::max<uint64_t>(1, 2 * slots / n);
  if (gx > gcap) gx = gcap;
  fbox_kernel<<<dim3((unsigned)gx, n), 256, 0, stream>>>(Bt);
  search_local_kernel<C><<<(unsigned)total, C::THREADS, smem, stream>>>(Bt);
  CUDA_TRY(cudaGetLastError());
  return MCX_OK;
}

// Variant selection (MCX_VARIANT, experiments; 0 = the tuned default: 16 A records per
// thread, 2-warp CTAs, 9 CTAs/SM (75 registers: the survivor flush only appends to the
// candidate list), one frame per warp, B tiles quantised by the whole CTA, one vote per 64 B
// records, half words — two pair tests per subtraction — folded into 4 accumulators (one
// LOP3 per four pair tests), 2 of every 8 subtractions on the alu pipe — DESIGN.md §5).
static int launch_prefilter(std::vector<SearchParams>& T, Batch& Bt, std::vector<uint64_t>& prefix,
                            void* dev_tab, const std::vector<FboxJob>& jobs, void* dev_jobs, int device,
                            cudaStream_t stream) {
#define MCX_LOCAL(...) launch_local_cfg<LCfg<__VA_ARGS__>>(T, Bt, prefix, dev_tab, jobs, dev_jobs, device, stream)
  switch (variant_from_env()) {
    case 1: return MCX_LOCAL(16, 16, 1, 8, true, true, 2);
    case 2: return MCX_LOCAL(16, 16, 1, 8, true, true, 3);
    case 3: return MCX_LOCAL(16, 16, 1, 8, true, true, 5);
    case 4: return MCX_LOCAL(16, 16, 1, 8, true, true, 6);
    case 5: return MCX_LOCAL(16, 16, 1, 1, true, true, 2);  // 6 CTAs/SM (150 registers)
    case 6: return MCX_LOCAL(16, 8, 1, 8, true, true, 4);
    case 7: return MCX_LOCAL(32, 16, 1, 4, true, true, 4);
    case 8: return MCX_LOCAL(16, 8, 1, 1, true);            // one frame per CTA
    case 9: return MCX_LOCAL(16, 8, 1);                     // one LOP3 per pair test
    case 10: return MCX_LOCAL(8, 8, 1, 1, true, true);
    case 11: return MCX_LOCAL(16, 32, 1, 8, true, true, 4);
    case 12: return MCX_LOCAL(16, 16, 1, 8, true, true, 4);
    case 13: return MCX_LOCAL(16, 64, 1, 9, true, true, 4);   // 9 CTAs/SM (112 registers)
    case 14: return MCX_LOCAL(16, 64, 1, 10, true, true, 4);  // 10 CTAs/SM
    case 15: return MCX_LOCAL(16, 32, 1, 10, true, true, 4);  // one vote per 32 B records, 10 CTAs/SM
    case 16: return MCX_LOCAL(16, 32, 1, 9, true, true, 4);
    case 17: return MCX_LOCAL(16, 64, 1, 8, true, true, 4);  // round 1 default (8 CTAs/SM, 116 registers)
    case 18: return MCX_LOCAL(16, 64, 1, 9, true, true, 4);         // round 2a: full words, 9 CTAs/SM
    case 19: return MCX_LOCAL(32, 64, 1, 9, true, true, 0, true);   // half words, 32 A records per lane
    case 20: return MCX_LOCAL(16, 32, 1, 9, true, true, 0, true);   // half words, one vote per 32 B records
    case 21: return MCX_LOCAL(32, 32, 1, 8, true, true, 0, true);
    case 22: return MCX_LOCAL(16, 64, 1, 9, true, false, 0, true);        // half words, one frame per CTA
    case 23: return MCX_LOCAL(16, 64, 1, 12, true, true, 0, true, 128);   // 128-record stages, 12 CTAs/SM
    case 24: return MCX_LOCAL(16, 32, 1, 12, true, true, 0, true, 128);
    case 25: return MCX_LOCAL(16, 128, 1, 9, true, true, 0, true);        // one vote per 128 B records
    case 26: return MCX_LOCAL(16, 64, 1, 6, true, true, 0, true, 512);    // 512-record stages
    case 27: return MCX_LOCAL(16, 64, 1, 9, true, true, 0, true, FTILE, true);  // CTA-shared quantisation
    case 28: return MCX_LOCAL(16, 32, 1, 9, true, true, 0, true, FTILE, true);
    case 29: return MCX_LOCAL(8, 64, 1, 8, true, true, 0, true, FTILE, true);   // 4 warps of 256-record frames
    case 30: return MCX_LOCAL(8, 128, 1, 8, true, true, 0, true, FTILE, true);
    case 31: return MCX_LOCAL(8, 64, 1, 6, true, true, 0, true, 512, true);
    case 32: return MCX_LOCAL(16, 64, 1, 9, true, true, 0, true);   // half words, per-warp quantisation
    case 33: return MCX_LOCAL(16, 64, 1, 9, true, true, 2, true, FTILE, true, true);  // accumulated folds
    case 34: return MCX_LOCAL(16, 32, 1, 9, true, true, 2, true, FTILE, true, true);
    case 35: return MCX_LOCAL(16, 64, 1, 9, true, true, 0, true, FTILE, true, true);  // no borrow chains
    case 36: return MCX_LOCAL(16, 64, 1, 9, true, true, 1, true, FTILE, true, true);
    case 37: return MCX_LOCAL(16, 64, 1, 9, true, true, -2, true, FTILE, true, true);  // plain IADD3 subtractions
    case 38: return MCX_LOCAL(16, 64, 1, 10, true, true, 2, true, FTILE, true, true);
    case 39: return MCX_LOCAL(16, 32, 1, 10, true, true, 2, true, FTILE, true, true);
    case 40: return MCX_LOCAL(16, 64, 2, 9, true, true, 2, true, FTILE, true, true);
    case 41: return MCX_LOCAL(16, 64, 1, 9, true, true, 0, true, FTILE, true);  // half words, CTA-shared quantisation
    case 42: return MCX_LOCAL(16, 64, 1, 12, true, true, 2, true, 128, true, true);  // 128-record stages, 12 CTAs/SM
    case 43: return MCX_LOCAL(16, 64, 1, 11, true, true, 2, true, 128, true, true);
    case 44: return MCX_LOCAL(16, 64, 1, 6, true, true, 2, true, 512, true, true);   // 512-record stages
    case 45: return MCX_LOCAL(16, 64, 1, 9, true, true, 2, true, FTILE, true, true, 0x5);  // chains on slot pairs 0, 2
    case 46: return MCX_LOCAL(16, 64, 1, 9, true, true, 2, true, FTILE, true, true, 0x3);  // 0, 1
    case 47: return MCX_LOCAL(16, 64, 1, 9, true, true, 2, true, FTILE, true, true, 0x9);  // 0, 3
    case 48: return MCX_LOCAL(16, 64, 1, 9, true, true, 2, true, FTILE, true, true, 0, 2);  // 2 accumulator sets
    case 49: return MCX_LOCAL(16, 64, 1, 8, true, true, 2, true, FTILE, true, true, 0, 4);  // 4 sets
    case 50: return MCX_LOCAL(16, 64, 1, 9, true, true, 2, true, FTILE, true, true, 0, 1, true);  // AND of the accumulators
    case 51: return MCX_LOCAL(16, 128, 1, 9, true, true, 2, true, FTILE, true, true, 0, 1, true);
    case 52: return MCX_LOCAL(16, 64, 1, 9, true, true, 2, true, FTILE, true, true);  // accumulators tested one by one
    default: return MCX_LOCAL(16, 64, 1, 9, true, true, 2, true, FTILE, true, true, 0, 1, true);  // + accumulated folds
  }
#undef MCX_LOCAL
}

}  // namespace mcx
