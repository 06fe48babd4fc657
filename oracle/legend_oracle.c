/*
 * legend_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded CPU restatement of the reference trainer's hot
 * path (arXiv 2505.09258 "Legend" reference, /root/reference/proj).  It is the
 * checker the CUDA path is compared against: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it.  The product path never links or
 * calls anything in this directory.
 *
 * Parity pinning: tests/test_oracle_pin.py compares every function here with
 * the reference library itself (oracle/_ref/liblegend_ref.so, built from the
 * unmodified reference sources by oracle/Makefile) and with the committed
 * golden vectors in tests/golden/ (generated from that library by
 * tests/golden/gen_golden.py).  The arithmetic below reproduces the
 * reference's FP64 operation order, so results are bit-identical to it.
 *
 * Every function cites the reference file:line it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define LO_OK 0
#define LO_INVALID 1   /* std::invalid_argument */
#define LO_LOGIC 2     /* std::logic_error */
#define LO_RANGE 3     /* std::out_of_range */
#define LO_NOMEM 4

#define LO_NO_REL 0xffffffffu      /* graph.hpp:17 kNoRelation */
#define LO_KIND_DOT 0              /* train.hpp:13 ScoreKind */
#define LO_KIND_DISTMULT 1
#define LO_KIND_COMPLEX 2
#define LO_KIND_TRANSE 3           /* not in the reference (train.hpp:13): defined below */

/* ------------------------------------------------------------------ RNG --- */

/* rng.hpp:7-12 */
uint64_t lo_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

typedef struct {
  uint64_t s[4];
} lo_rng;

/* rng.hpp:18-21: four splitmix64 outputs fill the xoshiro state */
void lo_rng_init(lo_rng* r, uint64_t seed) {
  uint64_t s = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = lo_splitmix64(&s);
}

static inline uint64_t lo_rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:23-33 xoshiro256** */
uint64_t lo_rng_next(lo_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = lo_rotl(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = lo_rotl(s[3], 45);
  return result;
}

/* rng.hpp:36 */
double lo_rng_double(lo_rng* r) { return (double)(lo_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:42-48: unbiased rejection sampling; rejected draws consume the stream */
uint64_t lo_rng_below(lo_rng* r, uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t x = lo_rng_next(r);
    if (x >= threshold) return x % bound;
  }
}

/* rng.hpp:57-67 */
uint64_t lo_derive_seed(uint64_t base, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t s = base;
  lo_splitmix64(&s);
  s ^= 0x516cc24f80775842ull + a;
  lo_splitmix64(&s);
  s ^= 0x2545f4914f6cdd1dull * (b + 1);
  lo_splitmix64(&s);
  s ^= 0x9e6c63d0876a9a47ull * (c + 1);
  return lo_splitmix64(&s);
}

/* ctypes helpers: raw stream, and next_below over a list of bounds */
void lo_rng_state(uint64_t seed, uint64_t out[4]) {
  lo_rng r;
  lo_rng_init(&r, seed);
  memcpy(out, r.s, sizeof r.s);
}

void lo_rng_u64(uint64_t seed, uint64_t skip, uint64_t n, uint64_t* out) {
  lo_rng r;
  lo_rng_init(&r, seed);
  for (uint64_t i = 0; i < skip; ++i) lo_rng_next(&r);
  for (uint64_t i = 0; i < n; ++i) out[i] = lo_rng_next(&r);
}

/* consumed = number of raw u64 draws used (n + rejections) */
void lo_rng_below_seq(uint64_t seed, uint64_t skip, const uint64_t* bounds, uint64_t n,
                      uint64_t* out, uint64_t* consumed) {
  lo_rng r;
  lo_rng_init(&r, seed);
  for (uint64_t i = 0; i < skip; ++i) lo_rng_next(&r);
  uint64_t used = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t bound = bounds[i];
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
      const uint64_t x = lo_rng_next(&r);
      ++used;
      if (x >= threshold) {
        out[i] = x % bound;
        break;
      }
    }
  }
  if (consumed) *consumed = used;
}

/* ------------------------------------------------------- partitions --- */

/* graph.cpp:120-150: stride = ceil(V/n); stable counting sort of edge indices
 * by bucket (src_part * n + dst_part). */
int lo_partition_plan(const uint32_t* edges, uint64_t num_edges, uint64_t num_nodes, uint32_t n,
                      uint64_t* stride_out, uint64_t* offsets, uint64_t* edge_order) {
  if (n < 1) return LO_INVALID;
  if (n > num_nodes) return LO_INVALID;
  if (num_edges == 0) return LO_INVALID;
  const uint64_t stride = (num_nodes + n - 1) / n;
  const uint64_t buckets = (uint64_t)n * n;
  memset(offsets, 0, (buckets + 1) * sizeof(uint64_t));
  for (uint64_t e = 0; e < num_edges; ++e) {
    const uint64_t b = (edges[3 * e] / stride) * n + edges[3 * e + 2] / stride;
    offsets[b + 1]++;
  }
  for (uint64_t b = 0; b < buckets; ++b) offsets[b + 1] += offsets[b];
  uint64_t* cursor = (uint64_t*)malloc(buckets * sizeof(uint64_t));
  if (!cursor) return LO_NOMEM;
  memcpy(cursor, offsets, buckets * sizeof(uint64_t));
  for (uint64_t e = 0; e < num_edges; ++e) {
    const uint64_t b = (edges[3 * e] / stride) * n + edges[3 * e + 2] / stride;
    edge_order[cursor[b]++] = e;
  }
  free(cursor);
  *stride_out = stride;
  return LO_OK;
}

/* --------------------------------------------------------- store init --- */

/* store.cpp:19-25 fill_uniform_rows: f32(U[-b, b)) with b = 0.5/sqrt(dim),
 * drawn in row-major order from Rng(stream_seed) (rng.hpp:36-39). */
void lo_init_rows(uint64_t stream_seed, uint64_t rows, uint32_t dim, float* out) {
  const double bound = 0.5 / sqrt((double)dim);
  lo_rng r;
  lo_rng_init(&r, stream_seed);
  const uint64_t total = rows * dim;
  const double lo = -bound, hi = bound;
  for (uint64_t i = 0; i < total; ++i) out[i] = (float)(lo + (hi - lo) * lo_rng_double(&r));
}

/* store.cpp:59-86 EmbeddingStore::create: partition p seeded with
 * derive_seed(seed, p), relations with derive_seed(seed, 0x52454c53);
 * optimizer state zero.  E and S are whole-graph row-major arrays whose
 * partition p occupies rows [stride*p, min(stride*(p+1), V)). */
void lo_store_init(uint32_t n, uint64_t num_nodes, uint32_t dim, uint64_t num_relations,
                   uint64_t seed, float* E, float* S, float* relE, float* relS) {
  const uint64_t stride = (num_nodes + n - 1) / n;
  for (uint32_t p = 0; p < n; ++p) {
    const uint64_t begin = stride * p;
    uint64_t end = stride * (p + 1);
    if (end > num_nodes) end = num_nodes;
    if (end <= begin) continue;
    lo_init_rows(lo_derive_seed(seed, p, 0, 0), end - begin, dim, E + begin * dim);
  }
  if (S) memset(S, 0, num_nodes * dim * sizeof(float));
  if (num_relations > 0) {
    lo_init_rows(lo_derive_seed(seed, 0x52454c53ull, 0, 0), num_relations, dim, relE);
    if (relS) memset(relS, 0, num_relations * dim * sizeof(float));
  }
}

/* ---------------------------------------------------------- sampling --- */

/* train.cpp:190-202 resident_node_count / resident_node_at over resident
 * ranges sorted by first node; train.cpp:365-373 sample_negatives. */
int lo_sample_negatives_rng(const uint64_t* first, const uint64_t* count, int nparts, uint32_t k,
                            uint64_t num_positives, lo_rng* rng, uint32_t* out) {
  if (k == 0) return LO_INVALID;
  uint64_t total = 0;
  for (int i = 0; i < nparts; ++i) total += count[i];
  if (total == 0) return LO_INVALID;
  const uint64_t draws = num_positives * k;
  for (uint64_t q = 0; q < draws; ++q) {
    uint64_t idx = lo_rng_below(rng, total);
    int i = 0;
    while (idx >= count[i]) {
      idx -= count[i];
      ++i;
    }
    out[q] = (uint32_t)(first[i] + idx);
  }
  return LO_OK;
}

int lo_sample_negatives(const uint64_t* first, const uint64_t* count, int nparts, uint32_t k,
                        uint64_t num_positives, uint64_t seed, uint64_t skip, uint32_t* out) {
  lo_rng r;
  lo_rng_init(&r, seed);
  for (uint64_t i = 0; i < skip; ++i) lo_rng_next(&r);
  return lo_sample_negatives_rng(first, count, nparts, k, num_positives, &r, out);
}

/* --------------------------------------------------- score / grad math --- */

/* train.cpp:39-60 combine_src_rel (IR1 = s (x) r) */
static void combine(int kind, uint32_t d, const float* src, const float* rel, double* out) {
  switch (kind) {
    case LO_KIND_DOT:
      for (uint32_t i = 0; i < d; ++i) out[i] = src[i];
      break;
    case LO_KIND_DISTMULT:
      for (uint32_t i = 0; i < d; ++i) out[i] = (double)src[i] * rel[i];
      break;
    case LO_KIND_TRANSE:
      for (uint32_t i = 0; i < d; ++i) out[i] = (double)src[i] + (double)rel[i];
      break;
    default: {
      const uint32_t h = d / 2;
      for (uint32_t i = 0; i < h; ++i) {
        const double sr = src[i], si = src[i + h];
        const double rr = rel[i], ri = rel[i + h];
        out[i] = sr * rr - si * ri;
        out[i + h] = sr * ri + si * rr;
      }
    }
  }
}

/* train.cpp:65-85 adjoint_combine: out += adj_other(mix) */
static void adjoint(int kind, uint32_t d, const float* other, const double* mix, double* out) {
  switch (kind) {
    case LO_KIND_DOT:
    case LO_KIND_TRANSE:
      for (uint32_t i = 0; i < d; ++i) out[i] += mix[i];
      break;
    case LO_KIND_DISTMULT:
      for (uint32_t i = 0; i < d; ++i) out[i] += (double)other[i] * mix[i];
      break;
    default: {
      const uint32_t h = d / 2;
      for (uint32_t i = 0; i < h; ++i) {
        const double orr = other[i], ori = other[i + h];
        out[i] += orr * mix[i] + ori * mix[i + h];
        out[i + h] += orr * mix[i + h] - ori * mix[i];
      }
    }
  }
}

/*
 * TransE -- NOT in the reference (ScoreKind, train.hpp:13; SPEC.md lists
 * translational models as a non-goal), so this restatement is its
 * definition ("parity unpinned" against the reference; the CUDA path is
 * checked against this).  Written in the reference's structure:
 *   u = s + r (IR1),  q_t = u - t,  D_t = sqrt(sum_i q_t[i]^2) (sequential),
 *   score f_t = -D_t, the same contrastive loss -(f_pos - LSE_j f_j),
 *   w_j = softmax weight, coef_pos = -1/D_pos, coef_j = w_j/D_j (0 when D = 0),
 *   node gradient contributions coef * (u - row) for dst and negatives,
 *   src and relation gradient mix = -coef_pos q_pos - sum_j coef_j q_j.
 */
static double transe_dist(uint32_t d, const double* u, const float* t) {
  double acc = 0.0;
  for (uint32_t i = 0; i < d; ++i) {
    const double q = u[i] - (double)t[i];
    acc += q * q;
  }
  return sqrt(acc);
}

/* train.cpp:342-354 adagrad_update (FP64 math, FP32 storage; the update uses
 * the unrounded accumulator a) */
static void adagrad_row(float* theta, float* acc, const double* g, uint32_t d, double lr,
                        double eps) {
  for (uint32_t i = 0; i < d; ++i) {
    const double gi = g[i];
    const double a = (double)acc[i] + gi * gi;
    acc[i] = (float)a;
    theta[i] = (float)((double)theta[i] - lr * gi / (sqrt(a) + eps));
  }
}

typedef struct {
  uint32_t id;
  uint32_t pad;
  uint64_t seq; /* enumeration order (p, slot) -- the std::map visit order */
} lo_contrib;

static int contrib_cmp(const void* a, const void* b) {
  const lo_contrib* x = (const lo_contrib*)a;
  const lo_contrib* y = (const lo_contrib*)b;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq ? 1 : 0);
}

static int check_model(int kind, uint32_t dim) {
  /* train.cpp:11-16 ScoreModel::validate */
  if (dim == 0) return LO_INVALID;
  if (kind == LO_KIND_COMPLEX && dim % 2 != 0) return LO_INVALID;
  if (kind < 0 || kind > 3) return LO_INVALID;
  return LO_OK;
}

/*
 * One training step: batch_loss (train.cpp:217-278), batch_gradients
 * (train.cpp:280-340) and, if apply, adagrad_step (train.cpp:356-363) on a
 * single all-resident table of num_nodes rows.  Gradients are accumulated per
 * node in the reference's std::map visit order: positives ascending, and per
 * positive dst, negatives j ascending, then src.  Optional outputs: the sorted
 * unique node / relation ids and their FP64 gradients.
 */
static int lo_batch_ex(int kind, uint32_t d, float* E, float* S, uint64_t num_nodes,
                       float* relE, float* relS, uint64_t num_rels, const uint32_t* edges,
                       uint64_t P, const uint32_t* negs, uint32_t k, double lr, double eps,
                       int apply_nodes, int apply_rels, double* loss_out, uint64_t* n_nodes_out,
                       uint32_t* node_ids, double* node_grads, uint64_t* n_rels_out,
                       uint32_t* rel_ids, double* rel_grads);

int lo_batch(int kind, uint32_t d, float* E, float* S, uint64_t num_nodes, float* relE,
             float* relS, uint64_t num_rels, const uint32_t* edges, uint64_t P,
             const uint32_t* negs, uint32_t k, double lr, double eps, int apply, double* loss_out,
             uint64_t* n_nodes_out, uint32_t* node_ids, double* node_grads, uint64_t* n_rels_out,
             uint32_t* rel_ids, double* rel_grads) {
  return lo_batch_ex(kind, d, E, S, num_nodes, relE, relS, num_rels, edges, P, negs, k, lr, eps,
                     apply, apply, loss_out, n_nodes_out, node_ids, node_grads, n_rels_out,
                     rel_ids, rel_grads);
}

static int lo_batch_ex(int kind, uint32_t d, float* E, float* S, uint64_t num_nodes,
                       float* relE, float* relS, uint64_t num_rels, const uint32_t* edges,
                       uint64_t P, const uint32_t* negs, uint32_t k, double lr, double eps,
                       int apply_nodes, int apply_rels, double* loss_out, uint64_t* n_nodes_out,
                       uint32_t* node_ids, double* node_grads, uint64_t* n_rels_out,
                       uint32_t* rel_ids, double* rel_grads) {
  int rc = check_model(kind, d);
  if (rc) return rc;
  if (k == 0) return LO_INVALID; /* train.cpp:219-221 */
  const int typed = kind != LO_KIND_DOT;
  for (uint64_t p = 0; p < P; ++p) {
    const uint32_t s = edges[3 * p], r = edges[3 * p + 1], t = edges[3 * p + 2];
    if (s >= num_nodes || t >= num_nodes) return LO_RANGE; /* train.cpp:157 */
    if (typed) {
      if (r == LO_NO_REL) return LO_INVALID; /* train.cpp:209-211 */
      if (r >= num_rels) return LO_RANGE;    /* train.cpp:176 */
    }
    for (uint32_t j = 0; j < k; ++j)
      if (negs[p * k + j] >= num_nodes) return LO_RANGE;
  }

  const uint64_t slots = (uint64_t)k + 2;
  double* ir1 = (double*)malloc((P ? P : 1) * d * sizeof(double));
  double* w = (double*)malloc((P ? P : 1) * k * sizeof(double));
  double* f = (double*)malloc(k * sizeof(double));
  lo_contrib* con = (lo_contrib*)malloc((P ? P : 1) * slots * sizeof(lo_contrib));
  double* mixes = (double*)malloc((P ? P : 1) * d * sizeof(double));
  double* rowsum = (double*)malloc((P ? P : 1) * sizeof(double));
  if (!ir1 || !w || !f || !con || !mixes || !rowsum) {
    free(ir1), free(w), free(f), free(con), free(mixes), free(rowsum);
    return LO_NOMEM;
  }

  /* batch_loss: train.cpp:236-275 */
  const int transe = kind == LO_KIND_TRANSE;
  double* dpos = (double*)malloc((P ? P : 1) * sizeof(double));
  double* dneg = (double*)malloc((P ? P : 1) * k * sizeof(double));
  double loss = 0.0;
  for (uint64_t p = 0; p < P; ++p) {
    const uint32_t s = edges[3 * p], r = edges[3 * p + 1], t = edges[3 * p + 2];
    double* x = ir1 + p * d;
    combine(kind, d, E + (uint64_t)s * d, typed ? relE + (uint64_t)r * d : NULL, x);
    const float* dst = E + (uint64_t)t * d;
    double pos = 0.0;
    if (transe) {
      dpos[p] = transe_dist(d, x, dst);
      pos = -dpos[p];
    } else {
      for (uint32_t i = 0; i < d; ++i) {
        const double term = x[i] * dst[i];
        pos += term;
      }
    }
    double row_max = -INFINITY;
    for (uint32_t j = 0; j < k; ++j) {
      const float* neg = E + (uint64_t)negs[p * k + j] * d;
      double fj = 0.0;
      if (transe) {
        dneg[p * k + j] = transe_dist(d, x, neg);
        fj = -dneg[p * k + j];
      } else {
        for (uint32_t i = 0; i < d; ++i) fj += x[i] * neg[i];
      }
      f[j] = fj;
      row_max = (row_max < fj) ? fj : row_max; /* std::max(row_max, f) */
    }
    double sum = 0.0;
    for (uint32_t j = 0; j < k; ++j) {
      const double ex = exp(f[j] - row_max);
      w[p * k + j] = ex;
      sum += ex;
    }
    rowsum[p] = sum; /* IR3 row sum; w holds IR3 until the gradient pass */
    loss += -(pos - (row_max + log(sum)));
  }

  /* batch_gradients: per-positive mix, then per-node accumulation in the
   * std::map visit order (train.cpp:298-333). */
  for (uint64_t p = 0; p < P; ++p) {
    const double inv_sum = 1.0 / rowsum[p];
    for (uint32_t j = 0; j < k; ++j) w[p * k + j] = w[p * k + j] * inv_sum;
    const float* dst = E + (uint64_t)edges[3 * p + 2] * d;
    double* mix = mixes + p * d;
    if (transe) {  /* coefficients replace w; mix = dL/du */
      const double* x = ir1 + p * d;
      const double cpos = dpos[p] > 0.0 ? -1.0 / dpos[p] : 0.0;
      dpos[p] = cpos;
      for (uint32_t i = 0; i < d; ++i) mix[i] = -(cpos * (x[i] - (double)dst[i]));
      for (uint32_t j = 0; j < k; ++j) {
        const double dj = dneg[p * k + j];
        const double cj = dj > 0.0 ? w[p * k + j] / dj : 0.0;
        w[p * k + j] = cj;
        const float* neg = E + (uint64_t)negs[p * k + j] * d;
        for (uint32_t i = 0; i < d; ++i) mix[i] -= cj * (x[i] - (double)neg[i]);
      }
    } else {
      for (uint32_t i = 0; i < d; ++i) mix[i] = -(double)dst[i];
      for (uint32_t j = 0; j < k; ++j) {
        const float* neg = E + (uint64_t)negs[p * k + j] * d;
        const double wj = w[p * k + j];
        for (uint32_t i = 0; i < d; ++i) mix[i] += wj * neg[i];
      }
    }
    con[p * slots].id = edges[3 * p + 2];
    con[p * slots].seq = p * slots;
    for (uint32_t j = 0; j < k; ++j) {
      con[p * slots + 1 + j].id = negs[p * k + j];
      con[p * slots + 1 + j].seq = p * slots + 1 + j;
    }
    con[p * slots + k + 1].id = edges[3 * p];
    con[p * slots + k + 1].seq = p * slots + k + 1;
  }
  qsort(con, P * slots, sizeof(lo_contrib), contrib_cmp);

  double* g = (double*)malloc(d * sizeof(double));
  uint64_t n_nodes = 0;
  /* First pass computes every gradient against the pre-update table; updates
   * are applied after all gradients exist (adagrad_step runs after
   * batch_gradients returns). */
  uint64_t uniq = 0;
  for (uint64_t c = 0; c < P * slots; ++c)
    if (c == 0 || con[c].id != con[c - 1].id) ++uniq;
  double* gall = (double*)malloc((uniq ? uniq : 1) * d * sizeof(double));
  uint32_t* gid = (uint32_t*)malloc((uniq ? uniq : 1) * sizeof(uint32_t));
  if (!g || !gall || !gid) {
    free(ir1), free(w), free(f), free(con), free(mixes), free(rowsum), free(g), free(gall),
        free(gid);
    return LO_NOMEM;
  }
  for (uint64_t c = 0; c < P * slots;) {
    const uint32_t id = con[c].id;
    double* acc = gall + n_nodes * d;
    for (uint32_t i = 0; i < d; ++i) acc[i] = 0.0;
    for (; c < P * slots && con[c].id == id; ++c) {
      const uint64_t p = con[c].seq / slots;
      const uint64_t slot = con[c].seq % slots;
      const double* x = ir1 + p * d;
      if (transe && slot <= k) { /* coef * (u - own row), own row pre-update */
        const double cf = slot == 0 ? dpos[p] : w[p * k + (slot - 1)];
        const float* own = E + (uint64_t)id * d;
        for (uint32_t i = 0; i < d; ++i) acc[i] += cf * (x[i] - (double)own[i]);
      } else if (slot == 0) {
        for (uint32_t i = 0; i < d; ++i) acc[i] -= x[i]; /* train.cpp:310 */
      } else if (slot <= k) {
        const double wj = w[p * k + (slot - 1)];
        for (uint32_t i = 0; i < d; ++i) acc[i] += wj * x[i]; /* train.cpp:320 */
      } else {
        const uint32_t r = edges[3 * p + 1];
        adjoint(kind, d, typed ? relE + (uint64_t)r * d : NULL, mixes + p * d,
                acc); /* train.cpp:327 */
      }
    }
    gid[n_nodes] = id;
    ++n_nodes;
  }

  /* relation gradients: train.cpp:328-332, positives ascending per relation */
  uint64_t n_rels = 0;
  double* rall = NULL;
  uint32_t* rid = NULL;
  if (typed && P > 0) {
    lo_contrib* rc2 = (lo_contrib*)malloc(P * sizeof(lo_contrib));
    rall = (double*)malloc(P * d * sizeof(double));
    rid = (uint32_t*)malloc(P * sizeof(uint32_t));
    for (uint64_t p = 0; p < P; ++p) {
      rc2[p].id = edges[3 * p + 1];
      rc2[p].seq = p;
    }
    qsort(rc2, P, sizeof(lo_contrib), contrib_cmp);
    for (uint64_t c = 0; c < P;) {
      const uint32_t id = rc2[c].id;
      double* acc = rall + n_rels * d;
      for (uint32_t i = 0; i < d; ++i) acc[i] = 0.0;
      for (; c < P && rc2[c].id == id; ++c) {
        const uint64_t p = rc2[c].seq;
        adjoint(kind, d, E + (uint64_t)edges[3 * p] * d, mixes + p * d, acc);
      }
      rid[n_rels++] = id;
    }
    free(rc2);
  }

  if (n_nodes_out) *n_nodes_out = n_nodes;
  if (n_rels_out) *n_rels_out = n_rels;
  if (node_ids) memcpy(node_ids, gid, n_nodes * sizeof(uint32_t));
  if (node_grads) memcpy(node_grads, gall, n_nodes * d * sizeof(double));
  if (rel_ids && n_rels) memcpy(rel_ids, rid, n_rels * sizeof(uint32_t));
  if (rel_grads && n_rels) memcpy(rel_grads, rall, n_rels * d * sizeof(double));

  /* train.cpp:356-363: nodes ascending, then relations */
  if (apply_nodes)
    for (uint64_t u = 0; u < n_nodes; ++u)
      adagrad_row(E + (uint64_t)gid[u] * d, S + (uint64_t)gid[u] * d, gall + u * d, d, lr, eps);
  if (apply_rels)
    for (uint64_t u = 0; u < n_rels; ++u)
      adagrad_row(relE + (uint64_t)rid[u] * d, relS + (uint64_t)rid[u] * d, rall + u * d, d, lr,
                  eps);
  if (loss_out) *loss_out = loss;
  free(ir1), free(w), free(f), free(con), free(mixes), free(rowsum), free(g), free(gall),
      free(gid);
  free(rall), free(rid), free(dpos), free(dneg);
  return LO_OK;
}

/* ------------------------------------------------------------- epoch --- */

/*
 * Real-train epoch (pipeline.cpp:273-322) restated over one all-resident
 * table, exactly as the reference's own test does (test_pipeline.cpp:227-269):
 * the negative-sampling pool of bucket g is the set of partitions resident in
 * the plan state that contains g.  states is num_states x 3 partition ids
 * (0xffffffff = unused slot, which lets n <= 3 run as one state holding every
 * partition); bucket_order is n*n (src_part, dst_part) pairs; state_offsets
 * has num_states + 1 entries.
 *
 * Optional dumps (NULL to skip): per-batch loss and unique node / relation
 * counts (max_batches entries), the shuffled in-bucket positions of every
 * trained edge (num_edges entries, in bucket_order), and every negative id
 * (num_edges * k entries).
 */
/* Shared-negative chunks (not a reference mode): with
 * chunk > 0 every run of `chunk` consecutive positives of a batch shares k
 * negatives.  A batch of cnt positives draws ceil(cnt / chunk) * k values
 * from the bucket stream (chunk-major, then j), right where the reference
 * draws its cnt * k, and the reference batch math runs on the expansion
 * negs[p * k + j] = shared[(p / chunk) * k + j].  neg_dump receives the
 * shared draws. */
static void expand_shared(const uint32_t* shared, uint64_t cnt, uint32_t k, uint32_t chunk,
                          uint32_t* out) {
  for (uint64_t p = 0; p < cnt; ++p)
    memcpy(out + p * k, shared + (p / chunk) * k, k * sizeof(uint32_t));
}

int lo_expand_shared(const uint32_t* shared, uint64_t cnt, uint32_t k, uint32_t chunk,
                     uint32_t* out) {
  if (chunk == 0 || k == 0) return LO_INVALID;
  expand_shared(shared, cnt, k, chunk, out);
  return LO_OK;
}

int lo_run_epoch_ex(const uint32_t* edges, uint64_t num_edges, uint64_t num_nodes,
                    uint64_t num_rels, uint32_t n, uint64_t stride, const uint64_t* bucket_offsets,
                    const uint64_t* edge_order, uint64_t num_states, const uint32_t* states,
                    const uint32_t* bucket_order, const uint64_t* state_offsets, int kind,
                    uint32_t d, double lr, double eps, uint32_t batch_size, uint32_t k,
                    uint32_t chunk, int shuffle, uint64_t seed, uint32_t epoch, float* E,
                    float* S, float* relE, float* relS, double* loss_sum_out,
                    uint64_t* edges_trained_out, uint64_t* buckets_trained_out,
                    uint64_t* num_batches_out, uint64_t max_batches, double* batch_loss,
                    uint64_t* batch_nodes, uint64_t* batch_rels, uint32_t* perm_dump,
                    uint32_t* neg_dump);

int lo_run_epoch(const uint32_t* edges, uint64_t num_edges, uint64_t num_nodes,
                 uint64_t num_rels, uint32_t n, uint64_t stride, const uint64_t* bucket_offsets,
                 const uint64_t* edge_order, uint64_t num_states, const uint32_t* states,
                 const uint32_t* bucket_order, const uint64_t* state_offsets, int kind, uint32_t d,
                 double lr, double eps, uint32_t batch_size, uint32_t k, int shuffle,
                 uint64_t seed, uint32_t epoch, float* E, float* S, float* relE, float* relS,
                 double* loss_sum_out, uint64_t* edges_trained_out, uint64_t* buckets_trained_out,
                 uint64_t* num_batches_out, uint64_t max_batches, double* batch_loss,
                 uint64_t* batch_nodes, uint64_t* batch_rels, uint32_t* perm_dump,
                 uint32_t* neg_dump) {
  return lo_run_epoch_ex(edges, num_edges, num_nodes, num_rels, n, stride, bucket_offsets,
                         edge_order, num_states, states, bucket_order, state_offsets, kind, d, lr,
                         eps, batch_size, k, 0, shuffle, seed, epoch, E, S, relE, relS,
                         loss_sum_out, edges_trained_out, buckets_trained_out, num_batches_out,
                         max_batches, batch_loss, batch_nodes, batch_rels, perm_dump, neg_dump);
}

int lo_run_epoch_ex(const uint32_t* edges, uint64_t num_edges, uint64_t num_nodes,
                    uint64_t num_rels, uint32_t n, uint64_t stride, const uint64_t* bucket_offsets,
                    const uint64_t* edge_order, uint64_t num_states, const uint32_t* states,
                    const uint32_t* bucket_order, const uint64_t* state_offsets, int kind,
                    uint32_t d, double lr, double eps, uint32_t batch_size, uint32_t k,
                    uint32_t chunk, int shuffle, uint64_t seed, uint32_t epoch, float* E,
                    float* S, float* relE, float* relS, double* loss_sum_out,
                    uint64_t* edges_trained_out, uint64_t* buckets_trained_out,
                    uint64_t* num_batches_out, uint64_t max_batches, double* batch_loss,
                    uint64_t* batch_nodes, uint64_t* batch_rels, uint32_t* perm_dump,
                    uint32_t* neg_dump) {
  int rc = check_model(kind, d);
  if (rc) return rc;
  if (kind != LO_KIND_DOT && num_rels == 0) return LO_INVALID; /* pipeline.cpp:228-230 */
  if (batch_size == 0 || k == 0) return LO_INVALID;
  const uint64_t G = (uint64_t)n * n;
  double loss_sum = 0.0;
  uint64_t edges_trained = 0, buckets_trained = 0, nb = 0, perm_pos = 0, neg_pos = 0;
  uint64_t state = 0;
  uint32_t* bucket = NULL;
  uint32_t* pos = NULL;
  uint32_t* negs = NULL;
  uint32_t* shared = NULL;
  uint32_t* batch_edges = NULL;
  uint64_t cap = 0;
  rc = LO_OK;
  for (uint64_t g = 0; g < G; ++g) {
    while (state + 1 < num_states && g >= state_offsets[state + 1]) ++state;
    const uint32_t bi = bucket_order[2 * g], bj = bucket_order[2 * g + 1];
    const uint64_t b = (uint64_t)bi * n + bj;
    const uint64_t m = bucket_offsets[b + 1] - bucket_offsets[b];
    if (m == 0) continue; /* pipeline.cpp:291: before the RNG is created */
    if (m > cap) {
      free(bucket), free(pos), free(negs), free(shared), free(batch_edges);
      cap = m;
      bucket = (uint32_t*)malloc(cap * 3 * sizeof(uint32_t));
      pos = (uint32_t*)malloc(cap * sizeof(uint32_t));
      uint64_t bcap = cap < batch_size ? cap : batch_size;
      negs = (uint32_t*)malloc(bcap * k * sizeof(uint32_t));
      shared = (uint32_t*)malloc(bcap * k * sizeof(uint32_t));
      batch_edges = (uint32_t*)malloc(bcap * 3 * sizeof(uint32_t));
      if (!bucket || !pos || !negs || !shared || !batch_edges) {
        rc = LO_NOMEM;
        goto done;
      }
    }
    for (uint64_t i = 0; i < m; ++i) { /* pipeline.cpp:293-295 */
      const uint64_t e = edge_order[bucket_offsets[b] + i];
      memcpy(bucket + 3 * i, edges + 3 * e, 3 * sizeof(uint32_t));
      pos[i] = (uint32_t)i;
    }
    lo_rng rng; /* pipeline.cpp:296 "bukt" stream */
    lo_rng_init(&rng, lo_derive_seed(seed, 0x62756b74ull, epoch, g));
    if (shuffle) { /* pipeline.cpp:297-301 Fisher-Yates */
      for (uint64_t i = m; i > 1; --i) {
        const uint64_t j = lo_rng_below(&rng, i);
        uint32_t tmp[3];
        memcpy(tmp, bucket + 3 * (i - 1), sizeof tmp);
        memcpy(bucket + 3 * (i - 1), bucket + 3 * j, sizeof tmp);
        memcpy(bucket + 3 * j, tmp, sizeof tmp);
        const uint32_t tp = pos[i - 1];
        pos[i - 1] = pos[j];
        pos[j] = tp;
      }
    }
    if (perm_dump) memcpy(perm_dump + perm_pos, pos, m * sizeof(uint32_t));
    perm_pos += m;
    /* resident pool of this state, ascending node ranges (train.cpp:112-119) */
    uint64_t first[3], count[3];
    int np = 0;
    uint32_t ids[3];
    for (int s2 = 0; s2 < 3; ++s2) {
      const uint32_t p = states[3 * state + s2];
      if (p == 0xffffffffu) continue;
      ids[np++] = p;
    }
    for (int a = 0; a < np; ++a)
      for (int c = a + 1; c < np; ++c)
        if (ids[c] < ids[a]) {
          uint32_t t = ids[a];
          ids[a] = ids[c];
          ids[c] = t;
        }
    for (int a = 0; a < np; ++a) {
      first[a] = stride * ids[a];
      uint64_t end = stride * (ids[a] + 1);
      if (end > num_nodes) end = num_nodes;
      count[a] = end - first[a];
    }
    for (uint64_t off = 0; off < m; off += batch_size) { /* pipeline.cpp:303-312 */
      const uint64_t cnt = (m - off) < batch_size ? (m - off) : batch_size;
      if (chunk) {
        const uint64_t nch = (cnt + chunk - 1) / chunk;
        rc = lo_sample_negatives_rng(first, count, np, k, nch, &rng, shared);
        if (rc) goto done;
        if (neg_dump) memcpy(neg_dump + neg_pos, shared, nch * k * sizeof(uint32_t));
        neg_pos += nch * k;
        expand_shared(shared, cnt, k, chunk, negs);
      } else {
        rc = lo_sample_negatives_rng(first, count, np, k, cnt, &rng, negs);
        if (rc) goto done;
        if (neg_dump) memcpy(neg_dump + neg_pos, negs, cnt * k * sizeof(uint32_t));
        neg_pos += cnt * k;
      }
      double l = 0.0;
      uint64_t un = 0, ur = 0;
      rc = lo_batch(kind, d, E, S, num_nodes, relE, relS, num_rels, bucket + 3 * off, cnt, negs,
                    k, lr, eps, 1, &l, &un, NULL, NULL, &ur, NULL, NULL);
      if (rc) goto done;
      if (nb < max_batches) {
        if (batch_loss) batch_loss[nb] = l;
        if (batch_nodes) batch_nodes[nb] = un;
        if (batch_rels) batch_rels[nb] = ur;
      }
      ++nb;
      loss_sum += l;
    }
    edges_trained += m;
    ++buckets_trained;
  }
done:
  free(bucket), free(pos), free(negs), free(shared), free(batch_edges);
  if (loss_sum_out) *loss_sum_out = loss_sum;
  if (edges_trained_out) *edges_trained_out = edges_trained;
  if (buckets_trained_out) *buckets_trained_out = buckets_trained;
  if (num_batches_out) *num_batches_out = nb;
  (void)num_edges;
  return rc;
}

/* ---------------------------------------------------------- evaluate --- */

/* train.cpp:375-412 evaluate over an all-resident table (train.cpp:414-421
 * loads every partition in order, so resident_node_at(i) == i). */
int lo_evaluate(int kind, uint32_t d, const float* E, uint64_t num_nodes, const float* relE,
                uint64_t num_rels, const uint32_t* test_edges, uint64_t T,
                uint32_t num_candidates, uint32_t hits_k, uint64_t seed, double* mrr_out,
                double* hits_out) {
  int rc = check_model(kind, d);
  if (rc) return rc;
  if (T == 0) return LO_INVALID;
  if (num_candidates == 0) return LO_INVALID;
  const int typed = kind != LO_KIND_DOT;
  double* ir1 = (double*)malloc(d * sizeof(double));
  double mrr = 0.0, hits = 0.0;
  for (uint64_t t = 0; t < T; ++t) {
    const uint32_t s = test_edges[3 * t], r = test_edges[3 * t + 1], dd = test_edges[3 * t + 2];
    if (typed && r == LO_NO_REL) {
      free(ir1);
      return LO_INVALID;
    }
    if (typed && r >= num_rels) {
      free(ir1);
      return LO_RANGE;
    }
    if (s >= num_nodes || dd >= num_nodes) {
      free(ir1);
      return LO_RANGE;
    }
    combine(kind, d, E + (uint64_t)s * d, typed ? relE + (uint64_t)r * d : NULL, ir1);
    double truth = 0.0;
    if (kind == LO_KIND_TRANSE) {
      truth = -transe_dist(d, ir1, E + (uint64_t)dd * d);
    } else {
      for (uint32_t i = 0; i < d; ++i) truth += ir1[i] * E[(uint64_t)dd * d + i];
    }
    lo_rng rng;
    lo_rng_init(&rng, lo_derive_seed(seed, 0x65766179ull, t, 0));
    uint64_t beaten = 0;
    for (uint32_t c = 0; c < num_candidates; ++c) {
      const uint64_t cand = lo_rng_below(&rng, num_nodes);
      double f = 0.0;
      if (kind == LO_KIND_TRANSE) {
        f = -transe_dist(d, ir1, E + cand * d);
      } else {
        for (uint32_t i = 0; i < d; ++i) f += ir1[i] * E[cand * d + i];
      }
      if (f >= truth) ++beaten;
    }
    const uint64_t rank = 1 + beaten;
    mrr += 1.0 / (double)rank;
    hits += rank <= hits_k ? 1.0 : 0.0;
  }
  free(ir1);
  *mrr_out = mrr / (double)T;
  *hits_out = hits / (double)T;
  return LO_OK;
}

/* The bucket shuffle of pipeline.cpp:297-301 applied to positions: perm[i] is
 * the original in-bucket index that ends at position i; consumed = raw draws. */
void lo_shuffle_perm(uint64_t seed, uint64_t m, uint32_t* perm, uint64_t* consumed) {
  lo_rng r;
  lo_rng_init(&r, seed);
  for (uint64_t i = 0; i < m; ++i) perm[i] = (uint32_t)i;
  uint64_t used = 0;
  for (uint64_t i = m; i > 1; --i) {
    const uint64_t bound = i;
    const uint64_t threshold = (0 - bound) % bound;
    uint64_t x;
    do {
      x = lo_rng_next(&r);
      ++used;
    } while (x < threshold);
    const uint64_t j = x % bound;
    const uint32_t t = perm[i - 1];
    perm[i - 1] = perm[j];
    perm[j] = t;
  }
  if (consumed) *consumed = used;
}

/* Bounded CPU-baseline sample of the real-train loop (pipeline.cpp:289-312)
 * for ONE bucket: copy, seeded Fisher-Yates shuffle, then up to max_batches
 * batches of sample_negatives + batch_loss + batch_gradients + adagrad_step.
 * The table holds rows [0, num_nodes); the pool lists the resident ranges. */
int lo_bucket_sample_ex(const uint32_t* bucket_edges, uint64_t m, const uint64_t* first,
                        const uint64_t* count, int nparts, uint64_t stream_seed, int shuffle,
                        uint32_t batch_size, uint32_t k, uint64_t max_batches, int kind,
                        uint32_t d, float* E, float* S, uint64_t num_nodes, float* relE,
                        float* relS, uint64_t num_rels, double lr, double eps, double* loss_sum,
                        uint64_t* edges_trained, double* batch_losses, uint64_t* batch_nodes);

int lo_bucket_sample(const uint32_t* bucket_edges, uint64_t m, const uint64_t* first,
                     const uint64_t* count, int nparts, uint64_t stream_seed, int shuffle,
                     uint32_t batch_size, uint32_t k, uint64_t max_batches, int kind, uint32_t d,
                     float* E, float* S, uint64_t num_nodes, float* relE, float* relS,
                     uint64_t num_rels, double lr, double eps, double* loss_sum,
                     uint64_t* edges_trained) {
  return lo_bucket_sample_ex(bucket_edges, m, first, count, nparts, stream_seed, shuffle,
                             batch_size, k, max_batches, kind, d, E, S, num_nodes, relE, relS,
                             num_rels, lr, eps, loss_sum, edges_trained, NULL, NULL);
}

/* The same with optional per-batch outputs (max_batches entries each): the
 * loss of every batch and |GradientSet.nodes|. */
int lo_bucket_sample_ex(const uint32_t* bucket_edges, uint64_t m, const uint64_t* first,
                        const uint64_t* count, int nparts, uint64_t stream_seed, int shuffle,
                        uint32_t batch_size, uint32_t k, uint64_t max_batches, int kind,
                        uint32_t d, float* E, float* S, uint64_t num_nodes, float* relE,
                        float* relS, uint64_t num_rels, double lr, double eps, double* loss_sum,
                        uint64_t* edges_trained, double* batch_losses, uint64_t* batch_nodes) {
  uint32_t* edges = (uint32_t*)malloc((m ? m : 1) * 3 * sizeof(uint32_t));
  uint32_t* negs = (uint32_t*)malloc((uint64_t)batch_size * k * sizeof(uint32_t));
  if (!edges || !negs) {
    free(edges), free(negs);
    return LO_NOMEM;
  }
  memcpy(edges, bucket_edges, m * 3 * sizeof(uint32_t));
  lo_rng rng;
  lo_rng_init(&rng, stream_seed);
  if (shuffle) {
    for (uint64_t i = m; i > 1; --i) {
      const uint64_t j = lo_rng_below(&rng, i);
      uint32_t t[3];
      memcpy(t, edges + 3 * (i - 1), sizeof t);
      memcpy(edges + 3 * (i - 1), edges + 3 * j, sizeof t);
      memcpy(edges + 3 * j, t, sizeof t);
    }
  }
  double total = 0.0;
  uint64_t done = 0, nb = 0;
  int rc = LO_OK;
  for (uint64_t off = 0; off < m && nb < max_batches; off += batch_size, ++nb) {
    const uint64_t cnt = (m - off) < batch_size ? (m - off) : batch_size;
    rc = lo_sample_negatives_rng(first, count, nparts, k, cnt, &rng, negs);
    if (rc) break;
    double l = 0.0;
    uint64_t nodes = 0;
    rc = lo_batch(kind, d, E, S, num_nodes, relE, relS, num_rels, edges + 3 * off, cnt, negs, k,
                  lr, eps, 1, &l, &nodes, NULL, NULL, NULL, NULL, NULL);
    if (rc) break;
    if (batch_losses) batch_losses[nb] = l;
    if (batch_nodes) batch_nodes[nb] = nodes;
    total += l;
    done += cnt;
  }
  free(edges), free(negs);
  *loss_sum = total;
  *edges_trained = done;
  return rc;
}

/*
 * Serialized restatement of the multi-GPU partition-round schedule
 * (SURVEY.md 8(e)).  items: count buckets in global order with
 * (src_part, dst_part, g, pool[3], round, pair) flattened as 8 u64 each;
 * bucket g uses the stream Rng(derive_seed(seed, "bukt", epoch, g)) and
 * samples negatives from its pool.  Pair j of a round runs on rank
 * j % num_ranks; a rank's batches (its buckets in order, shuffled, sliced)
 * run in lock step with the other ranks': at step k every rank's batch k
 * applies its node gradients (ranks own disjoint partitions) and the ranks'
 * relation gradients are summed in rank order, then one Adagrad step updates
 * every relation row any rank touched.
 */
typedef struct {
  uint64_t m, off;          /* bucket size and offset in edge_order */
  uint32_t* edges;          /* shuffled copy */
  uint32_t* negs;           /* m * k negative ids */
} lo_prepared;

int lo_run_rounds(const uint32_t* edges, uint64_t num_edges, uint64_t num_nodes,
                  uint64_t num_rels, uint32_t n, const uint64_t* items, uint64_t count,
                  uint32_t num_ranks, int kind, uint32_t d, double lr, double eps,
                  uint32_t batch_size, uint32_t k, int shuffle, uint64_t seed, uint32_t epoch,
                  float* E, float* S, float* relE, float* relS, double* loss_sum_out,
                  uint64_t* edges_trained_out) {
  int rc = check_model(kind, d);
  if (rc) return rc;
  if (kind != LO_KIND_DOT && num_rels == 0) return LO_INVALID;
  uint64_t stride = 0;
  uint64_t* offsets = (uint64_t*)malloc(((uint64_t)n * n + 1) * sizeof(uint64_t));
  uint64_t* order = (uint64_t*)malloc((num_edges ? num_edges : 1) * sizeof(uint64_t));
  rc = lo_partition_plan(edges, num_edges, num_nodes, n, &stride, offsets, order);
  if (rc) {
    free(offsets), free(order);
    return rc;
  }
  const int typed = kind != LO_KIND_DOT;
  double* rsum = typed ? (double*)malloc(num_rels * d * sizeof(double)) : NULL;
  uint8_t* rtouch = typed ? (uint8_t*)malloc(num_rels) : NULL;
  uint32_t* rid = typed ? (uint32_t*)malloc(((uint64_t)batch_size + 1) * sizeof(uint32_t)) : NULL;
  double* rg = typed ? (double*)malloc(((uint64_t)batch_size + 1) * d * sizeof(double)) : NULL;
  double loss_sum = 0.0;
  uint64_t edges_trained = 0;
  uint64_t i0 = 0;
  while (i0 < count && rc == 0) {
    const uint64_t round = items[8 * i0 + 6];
    uint64_t i1 = i0;
    while (i1 < count && items[8 * i1 + 6] == round) ++i1;
    /* per rank: prepare its buckets (shuffle + all negatives, stream order) */
    lo_prepared* prep = (lo_prepared*)calloc(i1 - i0, sizeof(lo_prepared));
    uint64_t* nbat = (uint64_t*)calloc(num_ranks, sizeof(uint64_t));
    for (uint64_t it = i0; it < i1; ++it) {
      const uint64_t* I = items + 8 * it;
      const uint64_t b = I[0] * n + I[1];
      lo_prepared* P = prep + (it - i0);
      P->off = offsets[b];
      P->m = offsets[b + 1] - offsets[b];
      nbat[I[7] % num_ranks] += (P->m + batch_size - 1) / batch_size;
      if (!P->m) continue;
      P->edges = (uint32_t*)malloc(P->m * 3 * sizeof(uint32_t));
      P->negs = (uint32_t*)malloc(P->m * k * sizeof(uint32_t));
      for (uint64_t e = 0; e < P->m; ++e)
        memcpy(P->edges + 3 * e, edges + 3 * order[P->off + e], 3 * sizeof(uint32_t));
      lo_rng rng;
      lo_rng_init(&rng, lo_derive_seed(seed, 0x62756b74ull, epoch, I[2]));
      if (shuffle)
        for (uint64_t i = P->m; i > 1; --i) {
          const uint64_t j = lo_rng_below(&rng, i);
          uint32_t t[3];
          memcpy(t, P->edges + 3 * (i - 1), sizeof t);
          memcpy(P->edges + 3 * (i - 1), P->edges + 3 * j, sizeof t);
          memcpy(P->edges + 3 * j, t, sizeof t);
        }
      uint64_t first[3], cnt[3];
      int np = 0;
      uint32_t ids[3];
      for (int q = 0; q < 3; ++q)
        if ((uint32_t)I[3 + q] != 0xffffffffu) ids[np++] = (uint32_t)I[3 + q];
      for (int a = 0; a < np; ++a)
        for (int c = a + 1; c < np; ++c)
          if (ids[c] < ids[a]) {
            uint32_t t = ids[a];
            ids[a] = ids[c];
            ids[c] = t;
          }
      for (int a = 0; a < np; ++a) {
        first[a] = stride * ids[a];
        uint64_t end = stride * (ids[a] + 1);
        if (end > num_nodes) end = num_nodes;
        cnt[a] = end - first[a];
      }
      rc = lo_sample_negatives_rng(first, cnt, np, k, P->m, &rng, P->negs);
      if (rc) break;
    }
    uint64_t steps = 0;
    for (uint32_t r = 0; r < num_ranks; ++r) steps = nbat[r] > steps ? nbat[r] : steps;
    for (uint64_t st = 0; st < steps && rc == 0; ++st) {
      if (typed) {
        memset(rsum, 0, num_rels * d * sizeof(double));
        memset(rtouch, 0, num_rels);
      }
      for (uint32_t r = 0; r < num_ranks && rc == 0; ++r) {
        /* this rank's batch st: walk its buckets in global order */
        uint64_t seen = 0;
        for (uint64_t it = i0; it < i1; ++it) {
          if (items[8 * it + 7] % num_ranks != r) continue;
          lo_prepared* P = prep + (it - i0);
          const uint64_t nb = (P->m + batch_size - 1) / batch_size;
          if (st < seen + nb) {
            const uint64_t off = (st - seen) * batch_size;
            const uint64_t cntp = (P->m - off) < batch_size ? (P->m - off) : batch_size;
            double l = 0.0;
            uint64_t nr = 0;
            rc = lo_batch_ex(kind, d, E, S, num_nodes, relE, relS, num_rels, P->edges + 3 * off,
                             cntp, P->negs + off * k, k, lr, eps, 1, 0, &l, NULL, NULL, NULL,
                             &nr, rid, rg);
            loss_sum += l;
            edges_trained += cntp;
            for (uint64_t u = 0; typed && u < nr; ++u) {
              rtouch[rid[u]] = 1;
              for (uint32_t e = 0; e < d; ++e) rsum[(uint64_t)rid[u] * d + e] += rg[u * d + e];
            }
            break;
          }
          seen += nb;
        }
      }
      for (uint64_t q = 0; typed && q < num_rels; ++q)
        if (rtouch[q])
          adagrad_row(relE + q * d, relS + q * d, rsum + q * d, d, lr, eps);
    }
    for (uint64_t it = i0; it < i1; ++it) free(prep[it - i0].edges), free(prep[it - i0].negs);
    free(prep), free(nbat);
    i0 = i1;
  }
  free(offsets), free(order), free(rsum), free(rtouch), free(rid), free(rg);
  *loss_sum_out = loss_sum;
  *edges_trained_out = edges_trained;
  return rc;
}

/* Exported pieces of the round restatement, for the CPU multi-rank tests:
 * one batch with node and relation updates applied separately, and the
 * relation Adagrad step over rows flagged as touched. */
int lo_batch_split(int kind, uint32_t d, float* E, float* S, uint64_t num_nodes, float* relE,
                   float* relS, uint64_t num_rels, const uint32_t* edges, uint64_t P,
                   const uint32_t* negs, uint32_t k, double lr, double eps, int apply_nodes,
                   int apply_rels, double* loss_out, uint64_t* n_rels_out, uint32_t* rel_ids,
                   double* rel_grads) {
  return lo_batch_ex(kind, d, E, S, num_nodes, relE, relS, num_rels, edges, P, negs, k, lr, eps,
                     apply_nodes, apply_rels, loss_out, NULL, NULL, NULL, n_rels_out, rel_ids,
                     rel_grads);
}

void lo_adagrad_touched(float* relE, float* relS, const double* summed, uint64_t R, uint32_t d,
                        double lr, double eps) {
  /* summed: R x (d+1), last column = touched flag (summed across ranks) */
  for (uint64_t r = 0; r < R; ++r)
    if (summed[r * (d + 1) + d] > 0.0) {
      double g[4096];
      for (uint32_t i = 0; i < d; ++i) g[i] = summed[r * (d + 1) + i];
      adagrad_row(relE + r * d, relS + r * d, g, d, lr, eps);
    }
}
