/*
 * graphgen.c -- TEST / BASELINE INFRASTRUCTURE ONLY (linked into
 * liblegend_oracle.so next to legend_oracle.c).
 *
 * Host restatement of the benchmark's synthetic power-law graph generator
 * (paper_2505_09258_b200/csrc/graph.cu: powerlaw_kernel, detmath.cuh), so the
 * reference CPU arm of bench.py and the parity tests can build the SAME input
 * graph without loading the product library.  The reference itself has no
 * power-law generator (its legend_synth plants clusters,
 * proj/tools/synth_graph.cpp:47-66; SURVEY.md 0 finding 5); the output uses the
 * reference's edge record and kNoRelation convention (graph.hpp:17-25).
 *
 * Determinism: every floating-point step is an IEEE-exact operation (+, -, *,
 * /, floor) in the order the device uses; this file must be compiled without
 * FMA contraction (oracle/Makefile: -ffp-contract=off) so products and sums
 * round exactly like the device's -fmad=false code.  tests/test_gpu_graph.py
 * checks the device generator against this file edge for edge.
 *
 * lo_powerlaw_bucket scans all edges with POSIX threads (ranges in ingest
 * order, concatenated in order), because the reference arm needs one bucket
 * of a 1.3-1.8 billion edge graph.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

uint64_t lo_splitmix64(uint64_t* state); /* legend_oracle.c (rng.hpp:7-12) */

static uint64_t gg_bits(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  return b;
}
static double gg_from_bits(uint64_t b) {
  double x;
  memcpy(&x, &b, 8);
  return x;
}

/* detmath.cuh det_log: x = m 2^e, m in [sqrt(1/2), sqrt(2)), 2 atanh series */
double lo_det_log(double x) {
  const uint64_t b = gg_bits(x);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  double m = gg_from_bits((b & 0xfffffffffffffull) | (1023ull << 52));
  if (m > 0x1.6a09e667f3bcdp+0) {
    m = m * 0.5;
    e += 1;
  }
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
  static const double c[12] = {0x1.47ae147ae147bp-4, 0x1.642c8590b2164p-4, 0x1.8618618618618p-4,
                               0x1.af286bca1af28p-4, 0x1.e1e1e1e1e1e1ep-4, 0x1.1111111111111p-3,
                               0x1.3b13b13b13b14p-3, 0x1.745d1745d1746p-3, 0x1.c71c71c71c71cp-3,
                               0x1.2492492492492p-2, 0x1.999999999999ap-2, 0x1.5555555555555p-1};
  double q = c[0];
  for (int i = 1; i < 12; ++i) q = q * s2 + c[i];
  const double r = s * 2.0 + s * (s2 * q);
  const double de = (double)e;
  return de * 0x1.62e42fee00000p-1 + (r + de * 0x1.a39ef35793c76p-33);
}

/* detmath.cuh det_exp: y = k ln2 + r, Taylor to r^17, scaled by 2^k */
double lo_det_exp(double y) {
  const double k = floor(y * 0x1.71547652b82fep+0 + 0.5);
  const double r = (y - k * 0x1.62e42fee00000p-1) - k * 0x1.a39ef35793c76p-33;
  static const double c[18] = {
      0x1.952c77030ad4ap-49, 0x1.ae7f3e733b81fp-45, 0x1.ae7f3e733b81fp-41, 0x1.93974a8c07c9dp-37,
      0x1.6124613a86d09p-33, 0x1.1eed8eff8d898p-29, 0x1.ae64567f544e4p-26, 0x1.27e4fb7789f5cp-22,
      0x1.71de3a556c734p-19, 0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-13, 0x1.6c16c16c16c17p-10,
      0x1.1111111111111p-7,  0x1.5555555555555p-5,  0x1.5555555555555p-3,  0.5,
      1.0,                   1.0};
  double p = c[0];
  for (int i = 1; i < 18; ++i) p = p * r + c[i];
  const int ki = (int)k;
  return p * gg_from_bits((uint64_t)(ki + 1023) << 52);
}

double lo_det_pow(double x, double y) { return lo_det_exp(y * lo_det_log(x)); }

typedef struct {
  uint64_t V, R, mult, seed;
  double inv, span;
} gg_params;

static uint64_t gg_gcd(uint64_t x, uint64_t y) {
  while (y) {
    const uint64_t t = x % y;
    x = y;
    y = t;
  }
  return x;
}

/* graph.cu launch_generate_powerlaw: beta = 1/(alpha-1); multiplier coprime
 * with V walked up from 2654435761 mod V */
static int gg_setup(uint64_t V, uint64_t R, double alpha, uint64_t seed, gg_params* p) {
  if (!(alpha > 2.0) || V == 0) return 1;
  const double beta = 1.0 / (alpha - 1.0);
  uint64_t mult = 2654435761ull % V;
  if (mult == 0) mult = 1;
  while (gg_gcd(mult, V) != 1) mult = (mult + 1) % V ? (mult + 1) % V : 1;
  p->V = V;
  p->R = R;
  p->mult = mult;
  p->seed = seed;
  p->inv = 1.0 / (1.0 - beta);
  p->span = lo_det_pow((double)V, 1.0 / p->inv) - 1.0;
  return 0;
}

/* graph.cu powerlaw_kernel endpoint(): Zipf rank by inverse CDF, scattered
 * by (rank * mult) mod V (128-bit product reduced in 2^32 steps) */
static uint32_t gg_endpoint(const gg_params* p, uint64_t r) {
  const double u = (double)(r >> 11) * 0x1.0p-53;
  uint64_t rank = (uint64_t)lo_det_pow(1.0 + u * p->span, p->inv) - 1;
  if (rank >= p->V) rank = p->V - 1;
  const unsigned __int128 prod = (unsigned __int128)rank * p->mult;
  const uint64_t lo = (uint64_t)prod, hi = (uint64_t)(prod >> 64);
  uint64_t rem = hi % p->V;
  rem = ((rem << 32) | (lo >> 32)) % p->V;
  rem = ((rem << 32) | (lo & 0xffffffffull)) % p->V;
  return (uint32_t)rem;
}

static void gg_edge(const gg_params* p, uint64_t e, uint32_t* out, int need_dst) {
  uint64_t s = p->seed ^ (e * 0xd1342543de82ef95ull);
  const uint64_t a = lo_splitmix64(&s), b = lo_splitmix64(&s), c = lo_splitmix64(&s);
  out[0] = gg_endpoint(p, a);
  out[1] = p->R ? (uint32_t)(b % p->R) : 0xffffffffu;
  out[2] = need_dst ? gg_endpoint(p, c) : 0;
}

/* Edges [begin, end) of the graph (E only bounds the ids; edge e depends on
 * (seed, e, V, R, alpha) alone). */
int lo_powerlaw_edges(uint64_t V, uint64_t R, double alpha, uint64_t seed, uint64_t begin,
                      uint64_t end, uint32_t* out) {
  gg_params p;
  if (gg_setup(V, R, alpha, seed, &p)) return 1;
  for (uint64_t e = begin; e < end; ++e) gg_edge(&p, e, out + 3 * (e - begin), 1);
  return 0;
}

typedef struct {
  const gg_params* p;
  uint64_t begin, end, stride;
  uint32_t n, bi, bj;
  uint32_t* buf;
  uint64_t count, cap;
  int oom;
} gg_job;

static void* gg_scan(void* arg) {
  gg_job* j = (gg_job*)arg;
  uint32_t rec[3];
  for (uint64_t e = j->begin; e < j->end; ++e) {
    gg_edge(j->p, e, rec, 0);
    if (rec[0] / j->stride != j->bi) continue;
    uint64_t s = j->p->seed ^ (e * 0xd1342543de82ef95ull);
    lo_splitmix64(&s);
    lo_splitmix64(&s);
    rec[2] = gg_endpoint(j->p, lo_splitmix64(&s));
    if (rec[2] / j->stride != j->bj) continue;
    if (j->count == j->cap) {
      const uint64_t cap = j->cap ? 2 * j->cap : 4096;
      uint32_t* nb = (uint32_t*)realloc(j->buf, cap * 12);
      if (!nb) {
        j->oom = 1;
        return NULL;
      }
      j->buf = nb;
      j->cap = cap;
    }
    memcpy(j->buf + 3 * j->count, rec, 12);
    ++j->count;
  }
  return NULL;
}

/* Bucket (bi, bj) of make_partition_plan(graph, n) (graph.cpp:120-150: stride
 * = ceil(V / n), edges in ingest order) of the E-edge graph, scanned with
 * `threads` threads.  Writes up to `cap` records into out; *count = the
 * bucket's size (call with cap 0 to size the buffer). */
int lo_powerlaw_bucket(uint64_t V, uint64_t R, uint64_t E, double alpha, uint64_t seed,
                       uint32_t n, uint32_t bi, uint32_t bj, int threads, uint32_t* out,
                       uint64_t cap, uint64_t* count) {
  gg_params p;
  if (gg_setup(V, R, alpha, seed, &p) || n == 0) return 1;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  const uint64_t stride = (V + n - 1) / n;
  gg_job jobs[256];
  pthread_t tid[256];
  for (int t = 0; t < threads; ++t) {
    gg_job* j = &jobs[t];
    memset(j, 0, sizeof *j);
    j->p = &p;
    j->begin = E * (uint64_t)t / (uint64_t)threads;
    j->end = E * (uint64_t)(t + 1) / (uint64_t)threads;
    j->stride = stride;
    j->n = n;
    j->bi = bi;
    j->bj = bj;
    if (pthread_create(&tid[t], NULL, gg_scan, j)) {
      gg_scan(j);
      tid[t] = 0;
    }
  }
  int rc = 0;
  uint64_t total = 0;
  for (int t = 0; t < threads; ++t) {
    if (tid[t]) pthread_join(tid[t], NULL);
    if (jobs[t].oom) rc = 4;
  }
  for (int t = 0; t < threads; ++t) {
    if (!rc && out) {
      const uint64_t room = total < cap ? cap - total : 0;
      const uint64_t c = jobs[t].count < room ? jobs[t].count : room;
      memcpy(out + 3 * total, jobs[t].buf, c * 12);
    }
    total += jobs[t].count;
    free(jobs[t].buf);
  }
  *count = total;
  return rc;
}
