// mcx_format.cuh — the records text formatted on the device.
//
// fmt_g17(v) writes exactly what Python's f"{v:.17g}" writes (the reference's
// records writer, isect.IntersectionRecord.to_line): 17 significant digits,
// correctly rounded (round-half-even on the exact binary value), 'f' notation for
// decimal exponents −4 ≤ E < 17 and 'e' notation otherwise, insignificant trailing
// zeros and a bare decimal point removed, exponent with a sign and ≥ 2 digits,
// "inf" / "-inf" / "nan" / "-0".  The conversion is exact: v = m·2^e2 is scaled by
// 10^(16−E) in big-integer arithmetic (≤ 1184 bits for subnormals, 40 × 32-bit
// limbs), so every double — not only the O(1) coordinates of a mesh — prints like
// the host.  __host__ __device__: the same code is exported as mcx_format_g17 for
// the CPU tests that compare it with Python on millions of values.
#pragma once
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define MCX_HD __host__ __device__ __forceinline__
#else
#define MCX_HD inline
#endif

namespace mcx {
namespace fmt {

struct Big {
  uint32_t w[40];  // little-endian limbs
  int n;           // used limbs (no leading zero limb)
};

MCX_HD void big_set(Big& b, uint64_t v) {
  b.w[0] = (uint32_t)v;
  b.w[1] = (uint32_t)(v >> 32);
  b.n = b.w[1] ? 2 : (b.w[0] ? 1 : 0);
}

MCX_HD void big_mul(Big& b, uint32_t m) {
  uint64_t carry = 0;
  for (int i = 0; i < b.n; ++i) {
    const uint64_t t = (uint64_t)b.w[i] * m + carry;
    b.w[i] = (uint32_t)t;
    carry = t >> 32;
  }
  if (carry) b.w[b.n++] = (uint32_t)carry;
}

MCX_HD void big_shl(Big& b, int s) {
  const int ws = s >> 5, bs = s & 31;
  if (b.n == 0) return;
  if (bs) {
    uint32_t carry = 0;
    for (int i = 0; i < b.n; ++i) {
      const uint32_t x = b.w[i];
      b.w[i] = (x << bs) | carry;
      carry = x >> (32 - bs);
    }
    if (carry) b.w[b.n++] = carry;
  }
  if (ws) {
    for (int i = b.n - 1; i >= 0; --i) b.w[i + ws] = b.w[i];
    for (int i = 0; i < ws; ++i) b.w[i] = 0;
    b.n += ws;
  }
}

// b >>= s; returns true iff a 1 bit was shifted out
MCX_HD bool big_shr(Big& b, int s) {
  const int ws = s >> 5, bs = s & 31;
  bool sticky = false;
  if (ws >= b.n) {
    for (int i = 0; i < b.n; ++i) sticky |= b.w[i] != 0;
    b.n = 0;
    return sticky;
  }
  for (int i = 0; i < ws; ++i) sticky |= b.w[i] != 0;
  for (int i = 0; i + ws < b.n; ++i) b.w[i] = b.w[i + ws];
  b.n -= ws;
  if (bs) {
    sticky |= (b.w[0] & ((1u << bs) - 1u)) != 0;
    for (int i = 0; i < b.n; ++i) b.w[i] = (b.w[i] >> bs) | (i + 1 < b.n ? b.w[i + 1] << (32 - bs) : 0u);
  }
  while (b.n && !b.w[b.n - 1]) --b.n;
  return sticky;
}

// b /= d; returns the remainder
MCX_HD uint32_t big_div(Big& b, uint32_t d) {
  uint64_t r = 0;
  for (int i = b.n - 1; i >= 0; --i) {
    const uint64_t cur = (r << 32) | b.w[i];
    b.w[i] = (uint32_t)(cur / d);
    r = cur % d;
  }
  while (b.n && !b.w[b.n - 1]) --b.n;
  return (uint32_t)r;
}

MCX_HD uint64_t big_u64(const Big& b) {
  return b.n == 0 ? 0 : (b.n == 1 ? b.w[0] : ((uint64_t)b.w[1] << 32 | b.w[0]));
}

MCX_HD uint32_t pow10u(int k) {  // k in [0, 9]
  uint32_t p = 1;
  for (int i = 0; i < k; ++i) p *= 10;
  return p;
}

// 10^k for k in [0, 19] (< 2^64): five predicated multiplies instead of a k-long chain
MCX_HD uint64_t pow10_u64(int k) {
  uint64_t p = 1;
  if (k & 1) p *= 10u;
  if (k & 2) p *= 100u;
  if (k & 4) p *= 10000u;
  if (k & 8) p *= 100000000u;
  if (k & 16) p *= 10000000000000000ull;
  return p;
}

// round-half-even(|v| · 10^k) for finite v = m·2^e2 (m > 0)
MCX_HD uint64_t scaled_round(uint64_t m, int e2, int k) {
  // Fast path in 128-bit registers for the usual magnitudes (2m·10^k and its shift fit):
  // no local-memory big integer.  Same exact arithmetic, so the same digits.
  if (k >= 0 && k <= 22 && e2 > -127 && e2 <= 0) {
    // 2m·10^k < 2^54 · 10^22 < 2^128
    unsigned __int128 q = (unsigned __int128)(2 * m) * pow10_u64(k <= 19 ? k : 19);
    if (k > 19) q *= pow10_u64(k - 19);
    const int sh = -e2;
    const bool sticky = sh && (q & (((unsigned __int128)1 << sh) - 1)) != 0;
    q >>= sh;
    uint64_t d = (uint64_t)(q >> 1);
    if (((uint64_t)q & 1) && (sticky || (d & 1))) ++d;
    return d;
  }
  Big N;
  big_set(N, m);
  big_shl(N, 1);  // one extra bit: the half
  if (e2 > 0) big_shl(N, e2);
  for (int r = k; r > 0; r -= 9) big_mul(N, pow10u(r > 9 ? 9 : r));
  bool sticky = false;
  if (e2 < 0) sticky |= big_shr(N, -e2);
  for (int r = -k; r > 0; r -= 9) sticky |= big_div(N, pow10u(r > 9 ? 9 : r)) != 0;
  const uint64_t q = big_u64(N);  // floor(2·|v|·10^k) < 2^58
  uint64_t d = q >> 1;
  if ((q & 1) && (sticky || (d & 1))) ++d;
  return d;
}

// floor(log10(m·2^e2)) estimate, exact to ±1 (corrected by the caller)
MCX_HD int bit_length(uint64_t x) {  // x > 0
#ifdef __CUDA_ARCH__
  return 64 - __clzll((long long)x);
#else
  return 64 - __builtin_clzll(x);
#endif
}

MCX_HD int log10_estimate(uint64_t m, int e2) {
  const int bits = bit_length(m);
  const int e = e2 + bits - 1;  // 2^e <= v < 2^(e+1)
  // floor(e · log10 2) with log10 2 ≈ 78913 / 2^18 (exact floor for |e| < 1650)
  return (int)(((int64_t)e * 78913) >> 18);  // arithmetic shift: floor for e < 0 too
}

MCX_HD int put_u64(char* o, uint64_t v) {
  // 9-digit chunks in 32-bit arithmetic (one 64-bit division by a constant per chunk)
  char t[24];
  int n = 0;
  while (v >= 1000000000ull) {
    uint32_t c = (uint32_t)(v % 1000000000ull);
    v /= 1000000000ull;
    for (int i = 0; i < 9; ++i) {
      t[n++] = (char)('0' + c % 10u);
      c /= 10u;
    }
  }
  uint32_t c = (uint32_t)v;
  do {
    t[n++] = (char)('0' + c % 10u);
    c /= 10u;
  } while (c);
  for (int i = 0; i < n; ++i) o[i] = t[n - 1 - i];
  return n;
}

// Python f"{v:.17g}"; returns the length (≤ 24), no terminator.
MCX_HD int fmt_g17(double v, char* o) {
  uint64_t bits;
  memcpy(&bits, &v, 8);
  const bool neg = bits >> 63;
  const int be = (int)((bits >> 52) & 0x7ff);
  uint64_t m = bits & ((1ull << 52) - 1);
  int n = 0;
  if (be == 0x7ff) {
    if (m) {
      o[0] = 'n'; o[1] = 'a'; o[2] = 'n';
      return 3;
    }
    if (neg) o[n++] = '-';
    o[n++] = 'i'; o[n++] = 'n'; o[n++] = 'f';
    return n;
  }
  if (neg) o[n++] = '-';
  if (be == 0 && m == 0) {
    o[n++] = '0';
    return n;
  }
  int e2;
  if (be == 0) {
    e2 = -1074;
  } else {
    m |= 1ull << 52;
    e2 = be - 1075;
  }
  const uint64_t LO = 10000000000000000ull, HI = 100000000000000000ull;  // 1e16, 1e17
  int E = log10_estimate(m, e2);
  uint64_t D = 0;
  for (int it = 0; it < 4; ++it) {
    D = scaled_round(m, e2, 16 - E);
    if (D >= HI) { ++E; continue; }
    if (D < LO) { --E; continue; }
    break;
  }
  // the 17 digits as two independent 32-bit chains: D = hi·10^8 + lo (hi < 10^9)
  char d[17];
  uint32_t hi = (uint32_t)(D / 100000000ull), lo = (uint32_t)(D - (uint64_t)hi * 100000000ull);
  for (int i = 16; i >= 9; --i) {
    d[i] = (char)('0' + lo % 10u);
    lo /= 10u;
  }
  for (int i = 8; i >= 0; --i) {
    d[i] = (char)('0' + hi % 10u);
    hi /= 10u;
  }
  int last = 16;  // last significant digit
  while (last > 0 && d[last] == '0') --last;
  if (E >= -4 && E < 17) {
    if (E >= 0) {
      for (int i = 0; i <= E; ++i) o[n++] = d[i];
      if (last > E) {
        o[n++] = '.';
        for (int i = E + 1; i <= last; ++i) o[n++] = d[i];
      }
    } else {
      o[n++] = '0';
      o[n++] = '.';
      for (int i = 0; i < -E - 1; ++i) o[n++] = '0';
      for (int i = 0; i <= last; ++i) o[n++] = d[i];
    }
  } else {
    o[n++] = d[0];
    if (last > 0) {
      o[n++] = '.';
      for (int i = 1; i <= last; ++i) o[n++] = d[i];
    }
    o[n++] = 'e';
    o[n++] = E < 0 ? '-' : '+';
    const int a = E < 0 ? -E : E;
    if (a < 10) o[n++] = '0';
    n += put_u64(o + n, (uint64_t)a);
  }
  return n;
}

// Field f (0..16) of a records-file line: n1 sign1 n2 sign2 gid x y px
// py a b c d theta_u s_u theta_s s_s, written to o (≤ 24 bytes, no separator).
MCX_HD int fmt_field(char* o, int f, int n1, int sign1, int n2, int sign2, uint64_t gid, const double* point,
                     const double* bary, const double* params) {
  if (f == 0 || f == 2) {
    const int x = f == 0 ? n1 : n2;
    int k = 0;
    if (x < 0) o[k++] = '-';
    return k + put_u64(o + k, (uint64_t)(x < 0 ? -(int64_t)x : x));
  }
  if (f == 1 || f == 3) {
    o[0] = (f == 1 ? sign1 : sign2) >= 0 ? '+' : '-';
    return 1;
  }
  if (f == 4) return put_u64(o, gid);
  const int c = f - 5;
  return fmt_g17(c < 4 ? point[c] : (c < 8 ? bary[c - 4] : params[c - 8]), o);
}

constexpr int LINE_FIELDS = 17;

// One records-file line: the 17 fields separated by ' ' and ended by '\n'.  Each field
// is formatted into a local buffer and then copied to o (o == nullptr: length only);
// writing the fields straight through a pointer that may be local or global lost the
// stores in device code, so the two address spaces never mix here.
MCX_HD int fmt_record_line(char* o, int n1, int sign1, int n2, int sign2, uint64_t gid, const double* point,
                           const double* bary, const double* params) {
  char f[32];
  int n = 0;
  for (int field = 0; field < LINE_FIELDS; ++field) {
    int k = fmt_field(f, field, n1, sign1, n2, sign2, gid, point, bary, params);
    f[k++] = field == LINE_FIELDS - 1 ? '\n' : ' ';
    if (o)
      for (int i = 0; i < k; ++i) o[n + i] = f[i];
    n += k;
  }
  return n;
}

}  // namespace fmt
}  // namespace mcx
