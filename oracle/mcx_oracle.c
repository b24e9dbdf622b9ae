/*
 * O2 — canonical CPU oracle in C (OpenMP), TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs load
 * this library (oracle/liboracle_mcx.so), as the checker or the timed CPU
 * baseline.  The product (paper_2109_14814_b200/) never links or calls it.
 *
 * Same algorithm and the same IEEE-754 operation sequence as oracle/canonical.py
 * (O1), which restates the reference's specified search: triangle split
 * SPEC.md:423-426, bounding-box rejection SPEC.md:442-450 / PAPER.md "Bounding
 * Box Test", precise test SPEC.md:460-468 / PAPER.md Eq. (26), singular gate
 * SPEC.md:464.  Build with -ffp-contract=off (no FMA contraction) and without
 * -ffast-math so that every expression is a chain of single rounded ops.
 *
 * Two enumeration modes over the same predicate:
 *   sweep = 0 : brute force, every (iA, iB) pair  (the SPEC "parallel" backend,
 *               used as the timed CPU baseline)
 *   sweep = 1 : sweep-and-prune on x — only skips pairs whose x-intervals are
 *               disjoint, which the AABB test rejects anyway, so the hit set and
 *               the AABB-pass count are identical (used for full-size parity).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SING_RTOL 1e-12

typedef struct {
  uint64_t n;
  double *lo, *hi;   /* [4][n] SoA */
  double *geo;       /* [n][19]: p4 e1_4 e2_4 P6 nrm */
} packed_t;

static void pack(const double* coords, uint32_t N, uint32_t M, packed_t* out) {
  uint64_t nq = (uint64_t)N * (M - 1), n = 2 * nq;
  out->n = n;
  out->lo = (double*)malloc(sizeof(double) * 4 * n);
  out->hi = (double*)malloc(sizeof(double) * 4 * n);
  out->geo = (double*)malloc(sizeof(double) * 19 * n);
  for (uint32_t k = 0; k + 1 < M; ++k) {
    for (uint32_t i = 0; i < N; ++i) {
      uint32_t ip = (i + 1) % N;
      for (int tau = 0; tau < 2; ++tau) {
        uint64_t t = 2 * ((uint64_t)i + (uint64_t)N * k) + tau;
        double v0[4], v1[4], v2[4];
        for (int c = 0; c < 4; ++c) {
          const double* pl = coords + (uint64_t)c * M * N;
          double w00 = pl[(uint64_t)k * N + i], w10 = pl[(uint64_t)k * N + ip];
          double w01 = pl[(uint64_t)(k + 1) * N + i], w11 = pl[(uint64_t)(k + 1) * N + ip];
          if (tau == 0) { v0[c] = w00; v1[c] = w10; v2[c] = w01; }
          else          { v0[c] = w01; v1[c] = w10; v2[c] = w11; }
          v0[c] += 0.0; v1[c] += 0.0; v2[c] += 0.0;
        }
        double* g = out->geo + 19 * t;
        double e1[4], e2[4];
        for (int c = 0; c < 4; ++c) {
          double lo = fmin(fmin(v0[c], v1[c]), v2[c]);
          double hi = fmax(fmax(v0[c], v1[c]), v2[c]);
          out->lo[(uint64_t)c * n + t] = lo;
          out->hi[(uint64_t)c * n + t] = hi;
          e1[c] = v1[c] - v0[c];
          e2[c] = v2[c] - v0[c];
          g[c] = v0[c]; g[4 + c] = e1[c]; g[8 + c] = e2[c];
        }
        static const int bi[6] = {0, 0, 0, 1, 1, 2}, bj[6] = {1, 2, 3, 2, 3, 3};
        for (int q = 0; q < 6; ++q) {
          double x = e1[bi[q]] * e2[bj[q]];
          double y = e1[bj[q]] * e2[bi[q]];
          g[12 + q] = x - y;
        }
        double n1 = e1[0] * e1[0]; n1 = n1 + e1[1] * e1[1]; n1 = n1 + e1[2] * e1[2]; n1 = n1 + e1[3] * e1[3];
        double n2 = e2[0] * e2[0]; n2 = n2 + e2[1] * e2[1]; n2 = n2 + e2[2] * e2[2]; n2 = n2 + e2[3] * e2[3];
        g[18] = sqrt(n1) * sqrt(n2);
      }
    }
  }
}

static void unpack_free(packed_t* p) { free(p->lo); free(p->hi); free(p->geo); }

static inline void contract(const double* r, const double* B, double* c) {
  /* B: 0:01 1:02 2:03 3:12 4:13 5:23 */
  c[0] = (r[2] * B[4] - r[1] * B[5]) - r[3] * B[3];
  c[1] = (r[0] * B[5] - r[2] * B[2]) + r[3] * B[1];
  c[2] = (r[1] * B[2] - r[0] * B[4]) - r[3] * B[0];
  c[3] = (r[0] * B[3] - r[1] * B[1]) + r[2] * B[0];
}

static inline double dot4(const double* c, const double* x) {
  double d = c[0] * x[0];
  d = d + c[1] * x[1];
  d = d + c[2] * x[2];
  d = d + c[3] * x[3];
  return d;
}

/* returns 0 = miss, 1 = hit, 2 = singular */
static inline int solve(const double* A, const double* B, double* out) {
  const double *p = A, *e1 = A + 4, *e2 = A + 8, *P = A + 12;
  const double *q = B, *f1 = B + 4, *f2 = B + 8, *Q = B + 12;
  double r[4];
  for (int c = 0; c < 4; ++c) r[c] = q[c] - p[c];
  double D = P[0] * Q[5] - P[1] * Q[4];
  D = D + P[2] * Q[3];
  D = D + P[3] * Q[2];
  D = D - P[4] * Q[1];
  D = D + P[5] * Q[0];
  double thr = (A[18] * B[18]) * SING_RTOL;
  if (fabs(D) <= thr) return 2;
  double g[4], h[4];
  contract(r, Q, g);
  contract(r, P, h);
  double s = dot4(g, e2) / D;
  double t = -dot4(g, e1) / D;
  double a = -dot4(h, f2) / D;
  double b = dot4(h, f1) / D;
  if (s >= 0 && t >= 0 && a >= 0 && b >= 0 && (s + t) <= 1 && (a + b) <= 1) {
    out[0] = s; out[1] = t; out[2] = a; out[3] = b;
    return 1;
  }
  return 0;
}

typedef struct { uint32_t ia, ib; double v[4]; } hit_t;

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

typedef struct { double key; uint64_t idx; } kv_t;
static int cmp_kv(const void* a, const void* b) {
  const kv_t *x = (const kv_t*)a, *y = (const kv_t*)b;
  if (x->key < y->key) return -1;
  if (x->key > y->key) return 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

int mcxo_version(void) { return 1; }

int mcxo_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/*
 * Search triangles A[a0, a1) against all of B.  Hits (unsorted) go to
 * ia/ib/stab (stab: [cap][4] = s,t,a,b) up to cap; *n_hits = total count.
 * stats[0] = pairs enumerated (logical), stats[1] = AABB pass, stats[2] = singular.
 * Returns 0, or 1 if cap was exceeded.
 */
/* emit_all: record every AABB-pass pair (not only the accepted ones), stab = the solve's
 * (s, t, a, b) or NaNs if singular — the survivor list for arithmetic comparisons. */
static int search_packed(const packed_t* pA, const packed_t* pB, uint64_t a0, uint64_t a1, int sweep,
                         int nthreads, uint32_t* ia, uint32_t* ib, double* stab, uint64_t cap, uint64_t* n_hits,
                         uint64_t* stats, int emit_all) {
  const packed_t A = *pA, B = *pB;
  if (a1 > A.n) a1 = A.n;
  if (a0 > a1) a0 = a1;
  uint64_t nB = B.n;
  /* optional x-sort of B for sweep-and-prune (brute force reads B's packed arrays as they are) */
  uint64_t* perm = (uint64_t*)malloc(sizeof(uint64_t) * (nB ? nB : 1));
  double* slo = sweep ? (double*)malloc(sizeof(double) * 4 * (nB ? nB : 1)) : B.lo;
  double* shi = sweep ? (double*)malloc(sizeof(double) * 4 * (nB ? nB : 1)) : B.hi;
  double maxw = 0.0;
  if (sweep) {
    kv_t* kv = (kv_t*)malloc(sizeof(kv_t) * (nB ? nB : 1));
    for (uint64_t j = 0; j < nB; ++j) { kv[j].key = B.lo[j]; kv[j].idx = j; }
    qsort(kv, nB, sizeof(kv_t), cmp_kv);
    for (uint64_t j = 0; j < nB; ++j) perm[j] = kv[j].idx;
    free(kv);
  } else {
    for (uint64_t j = 0; j < nB; ++j) perm[j] = j;
  }
  if (sweep)
    for (uint64_t j = 0; j < nB; ++j) {
      for (int c = 0; c < 4; ++c) {
        slo[(uint64_t)c * nB + j] = B.lo[(uint64_t)c * nB + perm[j]];
        shi[(uint64_t)c * nB + j] = B.hi[(uint64_t)c * nB + perm[j]];
      }
      double w = shi[j] - slo[j];
      if (w > maxw) maxw = w;
    }
  maxw = maxw * (1.0 + 1e-9);
  (void)cmp_double;
  uint64_t tot_hits = 0, tot_pass = 0, tot_sing = 0, tot_pairs = 0;
  int overflow = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel reduction(+ : tot_pass, tot_sing, tot_pairs)
  {
    enum { BLK = 2048 };
    unsigned char m[BLK];
    hit_t* local = NULL;
    uint64_t nloc = 0, capl = 0;
#pragma omp for schedule(dynamic, 64)
    for (int64_t ta = (int64_t)a0; ta < (int64_t)a1; ++ta) {
      double la[4], ha[4];
      for (int c = 0; c < 4; ++c) { la[c] = A.lo[(uint64_t)c * A.n + ta]; ha[c] = A.hi[(uint64_t)c * A.n + ta]; }
      uint64_t j0 = 0, j1 = nB;
      if (sweep) {
        /* candidates: slo_x in [la_x - maxw, ha_x]  (superset of x-overlap) */
        double lo_key = (la[0] - maxw) - 1e-9 * (fabs(la[0]) + maxw);
        uint64_t L = 0, R = nB;
        while (L < R) { uint64_t mid = (L + R) / 2; if (slo[mid] < lo_key) L = mid + 1; else R = mid; }
        j0 = L > 0 ? L - 1 : 0;  /* one slack for rounding of la - maxw */
        L = j0; R = nB;
        while (L < R) { uint64_t mid = (L + R) / 2; if (slo[mid] <= ha[0]) L = mid + 1; else R = mid; }
        j1 = L;
      }
      tot_pairs += nB;
      for (uint64_t b0 = j0; b0 < j1; b0 += BLK) {
        uint64_t bn = j1 - b0 < BLK ? j1 - b0 : BLK;
        const double *l0 = slo + b0, *l1 = slo + nB + b0, *l2 = slo + 2 * nB + b0, *l3 = slo + 3 * nB + b0;
        const double *h0 = shi + b0, *h1 = shi + nB + b0, *h2 = shi + 2 * nB + b0, *h3 = shi + 3 * nB + b0;
        for (uint64_t j = 0; j < bn; ++j) {
          m[j] = (unsigned char)((l0[j] <= ha[0]) & (la[0] <= h0[j]) & (l1[j] <= ha[1]) & (la[1] <= h1[j]) &
                                 (l2[j] <= ha[2]) & (la[2] <= h2[j]) & (l3[j] <= ha[3]) & (la[3] <= h3[j]));
        }
        for (uint64_t j = 0; j < bn; j += 8) {
          uint64_t w = 0;
          uint64_t lim = bn - j < 8 ? bn - j : 8;
          memcpy(&w, m + j, lim);
          if (!w) continue;
          for (uint64_t u = 0; u < lim; ++u) {
            if (!m[j + u]) continue;
            uint64_t tb = perm[b0 + j + u];
            ++tot_pass;
            double sol[4] = {NAN, NAN, NAN, NAN};
            int rc = solve(A.geo + 19 * ta, B.geo + 19 * tb, sol);
            if (rc == 2) ++tot_sing;
            if (rc == 1 || emit_all) {
              if (nloc == capl) { capl = capl ? 2 * capl : 256; local = (hit_t*)realloc(local, sizeof(hit_t) * capl); }
              local[nloc].ia = (uint32_t)ta; local[nloc].ib = (uint32_t)tb;
              memcpy(local[nloc].v, sol, sizeof(sol));
              ++nloc;
            }
          }
        }
      }
    }
    uint64_t base;
#pragma omp atomic capture
    { base = tot_hits; tot_hits += nloc; }
    for (uint64_t u = 0; u < nloc; ++u) {
      if (base + u < cap) {
        ia[base + u] = local[u].ia; ib[base + u] = local[u].ib;
        memcpy(stab + 4 * (base + u), local[u].v, sizeof(double) * 4);
      }
    }
    free(local);
  }
  if (tot_hits > cap) overflow = 1;
  *n_hits = tot_hits;
  stats[0] = tot_pairs; stats[1] = tot_pass; stats[2] = tot_sing;
  free(perm);
  if (sweep) { free(slo); free(shi); }
  return overflow;
}

int mcxo_search(const double* coords_a, uint32_t NA, uint32_t MA,
                const double* coords_b, uint32_t NB, uint32_t MB,
                uint64_t a0, uint64_t a1, int sweep, int nthreads,
                uint32_t* ia, uint32_t* ib, double* stab, uint64_t cap,
                uint64_t* n_hits, uint64_t* stats) {
  packed_t A, B;
  pack(coords_a, NA, MA, &A);
  pack(coords_b, NB, MB, &B);
  int rc = search_packed(&A, &B, a0, a1, sweep, nthreads, ia, ib, stab, cap, n_hits, stats, 0);
  unpack_free(&A); unpack_free(&B);
  return rc;
}

/* Packed meshes kept across searches (the timed CPU baseline packs once, untimed). */
void* mcxo_pack_new(const double* coords, uint32_t N, uint32_t M) {
  packed_t* p = (packed_t*)malloc(sizeof(packed_t));
  pack(coords, N, M, p);
  return p;
}

void mcxo_pack_free(void* p) {
  if (!p) return;
  unpack_free((packed_t*)p);
  free(p);
}

int mcxo_search_packed(const void* A, const void* B, uint64_t a0, uint64_t a1, int sweep, int nthreads,
                       uint32_t* ia, uint32_t* ib, double* stab, uint64_t cap, uint64_t* n_hits, uint64_t* stats) {
  return search_packed((const packed_t*)A, (const packed_t*)B, a0, a1, sweep, nthreads, ia, ib, stab, cap, n_hits,
                       stats, 0);
}

/* Every AABB-pass pair of A x B (exact sweep), with the canonical solve's (s, t, a, b)
 * (NaNs when the singular gate fired or the solve produced none). */
int mcxo_survivors(const void* A, const void* B, int nthreads, uint32_t* ia, uint32_t* ib, double* stab,
                   uint64_t cap, uint64_t* n_out, uint64_t* stats) {
  return search_packed((const packed_t*)A, (const packed_t*)B, 0, ((const packed_t*)A)->n, 1, nthreads, ia, ib, stab,
                       cap, n_out, stats, 1);
}

/* Export the canonical packing (for checking the device packer): box [n][8] (lo4 hi4), geo [n][19]. */
int mcxo_pack(const double* coords, uint32_t N, uint32_t M, double* box, double* geo) {
  packed_t P;
  pack(coords, N, M, &P);
  for (uint64_t t = 0; t < P.n; ++t)
    for (int c = 0; c < 4; ++c) { box[8 * t + c] = P.lo[(uint64_t)c * P.n + t]; box[8 * t + 4 + c] = P.hi[(uint64_t)c * P.n + t]; }
  memcpy(geo, P.geo, sizeof(double) * 19 * P.n);
  unpack_free(&P);
  return 0;
}

/* ------------------------------------------------------------------------------------
 * O3 in C — the SPEC-literal serial backend (oracle/serial.py) at full scale: quad AABB
 * (exact x-sweep over quad boxes), the Moller quick test with serial.py's op sequence,
 * then the 4 canonical triangle-pair precise tests of every candidate.
 * stats: [0] quad pairs, [1] quad-AABB passes, [2] candidates, [3] singular solves.
 */
#define DEGEN_RTOL2 1e-28

static void quad_verts(const double* c, uint32_t N, uint32_t M, uint64_t q, double V[4][3]) {
  const uint32_t i = (uint32_t)(q % N), k = (uint32_t)(q / N), ip = (i + 1) % N;
  const uint64_t idx[4] = {(uint64_t)k * N + i, (uint64_t)k * N + ip, (uint64_t)(k + 1) * N + i,
                           (uint64_t)(k + 1) * N + ip};
  for (int v = 0; v < 4; ++v)
    for (int d = 0; d < 3; ++d) V[v][d] = c[(uint64_t)d * M * N + idx[v]];
}

static int side_reject(const double Vq[4][3], const double Vo[4][3]) {
  static const int tri[2][3] = {{0, 1, 2}, {2, 1, 3}};
  int out = 1;
  for (int T = 0; T < 2; ++T) {
    const double* O = Vq[tri[T][0]];
    double U[3], W[3];
    for (int d = 0; d < 3; ++d) {
      U[d] = Vq[tri[T][1]][d] - O[d];
      W[d] = Vq[tri[T][2]][d] - O[d];
    }
    const double N0 = U[1] * W[2] - U[2] * W[1];
    const double N1 = U[2] * W[0] - U[0] * W[2];
    const double N2 = U[0] * W[1] - U[1] * W[0];
    const double nn = (N0 * N0 + N1 * N1) + N2 * N2;
    const double uu = (U[0] * U[0] + U[1] * U[1]) + U[2] * U[2];
    const double ww = (W[0] * W[0] + W[1] * W[1]) + W[2] * W[2];
    const int degen = nn < (uu * ww) * DEGEN_RTOL2;
    int pos = 1, neg = 1;
    for (int m = 0; m < 4; ++m) {
      const double f = (N0 * (Vo[m][0] - O[0]) + N1 * (Vo[m][1] - O[1])) + N2 * (Vo[m][2] - O[2]);
      pos = pos && (f > 0.0);
      neg = neg && (f < 0.0);
    }
    out = out && !degen && (pos || neg);
  }
  return out;
}

typedef struct {
  uint64_t n;
  double *lo, *hi; /* [4][n] */
} qbox_t;

static void quad_boxes(const double* c, uint32_t N, uint32_t M, qbox_t* out) {
  const uint64_t n = (uint64_t)N * (M - 1);
  out->n = n;
  out->lo = (double*)malloc(sizeof(double) * 4 * (n ? n : 1));
  out->hi = (double*)malloc(sizeof(double) * 4 * (n ? n : 1));
  for (uint64_t q = 0; q < n; ++q) {
    double V[4][4];
    const uint32_t i = (uint32_t)(q % N), k = (uint32_t)(q / N), ip = (i + 1) % N;
    const uint64_t idx[4] = {(uint64_t)k * N + i, (uint64_t)k * N + ip, (uint64_t)(k + 1) * N + i,
                             (uint64_t)(k + 1) * N + ip};
    for (int v = 0; v < 4; ++v)
      for (int d = 0; d < 4; ++d) V[v][d] = c[(uint64_t)d * M * N + idx[v]];
    for (int d = 0; d < 4; ++d) {
      out->lo[(uint64_t)d * n + q] = fmin(fmin(fmin(V[0][d], V[1][d]), V[2][d]), V[3][d]);
      out->hi[(uint64_t)d * n + q] = fmax(fmax(fmax(V[0][d], V[1][d]), V[2][d]), V[3][d]);
    }
  }
}

int mcxo_spec_search(const double* coords_a, uint32_t NA, uint32_t MA, const double* coords_b, uint32_t NB,
                     uint32_t MB, int nthreads, uint32_t* ia, uint32_t* ib, double* stab, uint64_t cap,
                     uint64_t* n_hits, uint64_t* stats) {
  packed_t A, B;
  pack(coords_a, NA, MA, &A);
  pack(coords_b, NB, MB, &B);
  qbox_t QA, QB;
  quad_boxes(coords_a, NA, MA, &QA);
  quad_boxes(coords_b, NB, MB, &QB);
  const uint64_t nB = QB.n;
  kv_t* kv = (kv_t*)malloc(sizeof(kv_t) * (nB ? nB : 1));
  for (uint64_t j = 0; j < nB; ++j) { kv[j].key = QB.lo[j]; kv[j].idx = j; }
  qsort(kv, nB, sizeof(kv_t), cmp_kv);
  double maxw = 0.0;
  for (uint64_t j = 0; j < nB; ++j) {
    double w = QB.hi[j] - QB.lo[j];
    if (w > maxw) maxw = w;
  }
  maxw = maxw * (1.0 + 1e-9);
  uint64_t tot_hits = 0, tot_pass = 0, tot_cand = 0, tot_sing = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel reduction(+ : tot_pass, tot_cand, tot_sing)
  {
    hit_t* local = NULL;
    uint64_t nloc = 0, capl = 0;
#pragma omp for schedule(dynamic, 64)
    for (int64_t qa = 0; qa < (int64_t)QA.n; ++qa) {
      double la[4], ha[4];
      for (int c = 0; c < 4; ++c) { la[c] = QA.lo[(uint64_t)c * QA.n + qa]; ha[c] = QA.hi[(uint64_t)c * QA.n + qa]; }
      const double lo_key = (la[0] - maxw) - 1e-9 * (fabs(la[0]) + maxw);
      uint64_t L = 0, R = nB;
      while (L < R) { uint64_t mid = (L + R) / 2; if (kv[mid].key < lo_key) L = mid + 1; else R = mid; }
      uint64_t j = L > 0 ? L - 1 : 0;
      double VA[4][3];
      int have_va = 0;
      for (; j < nB && kv[j].key <= ha[0]; ++j) {
        const uint64_t qb = kv[j].idx;
        int ov = 1;
        for (int c = 0; c < 4 && ov; ++c)
          ov = !(ha[c] < QB.lo[(uint64_t)c * nB + qb] || QB.hi[(uint64_t)c * nB + qb] < la[c]);
        if (!ov) continue;
        ++tot_pass;
        if (!have_va) { quad_verts(coords_a, NA, MA, (uint64_t)qa, VA); have_va = 1; }
        double VB[4][3];
        quad_verts(coords_b, NB, MB, qb, VB);
        if (side_reject(VA, VB) || side_reject(VB, VA)) continue;
        ++tot_cand;
        for (int v = 0; v < 4; ++v) {
          const uint64_t ta = 2 * (uint64_t)qa + (v >> 1), tb = 2 * qb + (v & 1);
          double sol[4];
          const int rc = solve(A.geo + 19 * ta, B.geo + 19 * tb, sol);
          if (rc == 2) { ++tot_sing; continue; }
          if (rc == 1) {
            if (nloc == capl) { capl = capl ? 2 * capl : 256; local = (hit_t*)realloc(local, sizeof(hit_t) * capl); }
            local[nloc].ia = (uint32_t)ta; local[nloc].ib = (uint32_t)tb;
            memcpy(local[nloc].v, sol, sizeof(sol));
            ++nloc;
          }
        }
      }
    }
    uint64_t base;
#pragma omp atomic capture
    { base = tot_hits; tot_hits += nloc; }
    for (uint64_t u = 0; u < nloc; ++u)
      if (base + u < cap) {
        ia[base + u] = local[u].ia; ib[base + u] = local[u].ib;
        memcpy(stab + 4 * (base + u), local[u].v, sizeof(double) * 4);
      }
    free(local);
  }
  *n_hits = tot_hits;
  stats[0] = QA.n * QB.n; stats[1] = tot_pass; stats[2] = tot_cand; stats[3] = tot_sing;
  free(kv);
  free(QA.lo); free(QA.hi); free(QB.lo); free(QB.hi);
  unpack_free(&A); unpack_free(&B);
  return tot_hits > cap;
}
