/*
 * oracle.c — CPU restatement of the reference batch-preparation path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline leg may load this library, and only as the checker
 * or the timed CPU baseline — never as part of the product path.
 *
 * Reference: /root/reference/pkg/src/mfgprep (numba, `mfgprep` 0.1.0).
 * Each function cites the reference lines it restates.  The restatement is
 * pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py -> tests/golden/ fixtures, checked by
 * tests/test_oracle.py).
 *
 * Build: see oracle/Makefile (gcc -O3 -fopenmp-free, pthreads).
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define GOLDEN 0x9E3779B97F4A7C15ull

/* rng.py:16-21 mix64 (splitmix64 finalizer) */
uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* sampler.py:241-247 HopStream.key_prefix */
uint64_t orc_hop_prefix(uint64_t seed, uint64_t batch, uint64_t hop) {
  uint64_t k = orc_mix64(seed ^ GOLDEN);
  k = orc_mix64(k ^ batch);
  return orc_mix64(k ^ (hop + 0x51EDull));
}

/* rng.py:33-35 stream_u64 */
static inline uint64_t stream_u64(uint64_t key, uint64_t ctr) {
  return orc_mix64(key + (ctr + 1) * GOLDEN);
}

/* _kernels.py:102-147 _sample_positions (vector_set variant) and the
 * take-all rule of hop_kernel (_kernels.py:168-170). Returns the count. */
int64_t orc_sample_positions(uint64_t key, int64_t deg, int64_t d, int64_t* out) {
  if (deg <= d) {
    for (int64_t p = 0; p < deg; ++p) out[p] = p;
    return deg;
  }
  int64_t acc = 0;
  uint64_t ctr = 0;
  while (acc < d) {
    const int64_t pos = (int64_t)(stream_u64(key, ctr) % (uint64_t)deg);
    ++ctr;
    int hit = 0;
    for (int64_t j = 0; j < acc; ++j)
      if (out[j] == pos) { hit = 1; break; }
    if (hit) continue;
    out[acc++] = pos;
  }
  return acc;
}

/* ---- insertion-ordered id map (sampler.py:106-171, flat_probing) -------- */
typedef struct {
  int64_t* table; /* slot -> local, -1 empty */
  int64_t cap;    /* power of two */
  int64_t* globals;
  int64_t gcap;
  int64_t size;
} IdMap;

static void map_init(IdMap* m, int64_t hint) {
  m->cap = 16;
  while (m->cap < 2 * hint) m->cap <<= 1;
  m->table = (int64_t*)malloc(sizeof(int64_t) * m->cap);
  memset(m->table, 0xFF, sizeof(int64_t) * m->cap);
  m->gcap = hint > 64 ? hint : 64;
  m->globals = (int64_t*)malloc(sizeof(int64_t) * m->gcap);
  m->size = 0;
}

static void map_free(IdMap* m) {
  free(m->table);
  free(m->globals);
}

static void map_reset(IdMap* m) {
  memset(m->table, 0xFF, sizeof(int64_t) * m->cap);
  m->size = 0;
}

/* sampler.py:131-145 ensure_capacity + _kernels.py:64-73 rehash_flat */
static void map_reserve(IdMap* m, int64_t extra) {
  const int64_t need = m->size + extra;
  if (need > m->gcap) {
    int64_t c = 2 * m->gcap > need ? 2 * m->gcap : need;
    m->globals = (int64_t*)realloc(m->globals, sizeof(int64_t) * c);
    m->gcap = c;
  }
  if (2 * need > m->cap) {
    int64_t c = m->cap;
    while (c < 2 * need) c <<= 1;
    free(m->table);
    m->table = (int64_t*)malloc(sizeof(int64_t) * c);
    memset(m->table, 0xFF, sizeof(int64_t) * c);
    m->cap = c;
    const uint64_t mask = (uint64_t)c - 1;
    for (int64_t e = 0; e < m->size; ++e) {
      uint64_t s = orc_mix64((uint64_t)m->globals[e]) & mask;
      while (m->table[s] != -1) s = (s + 1) & mask;
      m->table[s] = e;
    }
  }
}

/* _kernels.py:76-99 _map_get_or_insert (flat branch) */
static inline int64_t map_get_or_insert(IdMap* m, int64_t key) {
  const uint64_t mask = (uint64_t)m->cap - 1;
  uint64_t s = orc_mix64((uint64_t)key) & mask;
  while (m->table[s] != -1) {
    const int64_t l = m->table[s];
    if (m->globals[l] == key) return l;
    s = (s + 1) & mask;
  }
  m->globals[m->size] = key;
  m->table[s] = m->size;
  return m->size++;
}

typedef struct {
  const int64_t* indptr;
  const int32_t* indices;
  int64_t num_nodes;
} Graph;

/* One multi-hop sample (sampler.py:328-346 + hop_kernel fused path,
 * _kernels.py:150-185).  Layer arrays are written in EXPANSION order (hop 0
 * first); the caller reverses them into consumption order.  Scratch growth
 * mirrors _run_hop (sampler.py:284-300).  Returns 0, or -1 on overflow of
 * the caller's buffers (sizes given by *_cap). */
typedef struct {
  int64_t* src; /* concatenated src_local of all hops */
  int64_t src_cap;
  int64_t* dptr; /* concatenated dst_indptr (n_dst+1 each) */
  int64_t dptr_cap;
  int64_t meta[16][3]; /* per hop: num_dst, num_src, num_edges */
} HopOut;

static int multihop(const Graph* g, IdMap* m, const int64_t* seeds, int64_t nseeds,
                    const int32_t* per_hop, int L, uint64_t seed, int64_t batch, HopOut* o,
                    int64_t* pos_scratch) {
  map_reset(m);
  map_reserve(m, nseeds);
  for (int64_t i = 0; i < nseeds; ++i) map_get_or_insert(m, seeds[i]);
  int64_t soff = 0, doff = 0;
  for (int h = 0; h < L; ++h) {
    const int64_t fan = per_hop[L - 1 - h];
    const int64_t n_dst = m->size;
    /* hop_budget (_kernels.py:42-50) */
    int64_t budget = 0;
    for (int64_t i = 0; i < n_dst; ++i) {
      const int64_t v = m->globals[i];
      const int64_t deg = g->indptr[v + 1] - g->indptr[v];
      budget += deg < fan ? deg : fan;
    }
    map_reserve(m, budget);
    if (soff + budget > o->src_cap || doff + n_dst + 1 > o->dptr_cap) return -1;
    const uint64_t prefix = orc_hop_prefix(seed, (uint64_t)batch, (uint64_t)h);
    int64_t* dptr = o->dptr + doff;
    int64_t* src = o->src + soff;
    int64_t e = 0;
    for (int64_t i = 0; i < n_dst; ++i) {
      dptr[i] = e;
      const int64_t v = m->globals[i];
      const int64_t lo = g->indptr[v];
      const int64_t deg = g->indptr[v + 1] - lo;
      const uint64_t key = orc_mix64(prefix ^ (uint64_t)i);
      const int64_t cnt = orc_sample_positions(key, deg, fan, pos_scratch);
      for (int64_t j = 0; j < cnt; ++j)
        src[e++] = map_get_or_insert(m, (int64_t)g->indices[lo + pos_scratch[j]]);
    }
    dptr[n_dst] = e;
    o->meta[h][0] = n_dst;
    o->meta[h][1] = m->size;
    o->meta[h][2] = e;
    soff += e;
    doff += n_dst + 1;
  }
  return 0;
}

/* Public single-batch entry point.  globals_out must hold the final map
 * size; returns the number of nodes or -1. */
int64_t orc_multihop(const int64_t* indptr, const int32_t* indices, int64_t num_nodes,
                     const int64_t* seeds, int64_t nseeds, const int32_t* per_hop, int L,
                     uint64_t global_seed, int64_t batch_id, int64_t* globals_out,
                     int64_t globals_cap, int64_t* src_out, int64_t src_cap, int64_t* dptr_out,
                     int64_t dptr_cap, int64_t* meta_out /* L x 3 */) {
  Graph g = {indptr, indices, num_nodes};
  IdMap m;
  map_init(&m, nseeds);
  int64_t maxdeg = 1;
  int64_t* pos = NULL;
  int maxf = 1;
  for (int h = 0; h < L; ++h)
    if (per_hop[h] > maxf) maxf = per_hop[h];
  (void)maxdeg;
  pos = (int64_t*)malloc(sizeof(int64_t) * (maxf + 1));
  HopOut o;
  o.src = src_out;
  o.src_cap = src_cap;
  o.dptr = dptr_out;
  o.dptr_cap = dptr_cap;
  int rc = multihop(&g, &m, seeds, nseeds, per_hop, L, global_seed, batch_id, &o, pos);
  int64_t n = -1;
  if (rc == 0 && m.size <= globals_cap) {
    memcpy(globals_out, m.globals, sizeof(int64_t) * m.size);
    for (int h = 0; h < L; ++h)
      for (int k = 0; k < 3; ++k) meta_out[3 * h + k] = o.meta[h][k];
    n = m.size;
  }
  free(pos);
  map_free(&m);
  return n;
}

/* _kernels.py:233-244 _half_to_f32 (NaN -> canonical quiet NaN) */
static inline float half_to_f32(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000) << 16;
  const uint32_t e = (h >> 10) & 0x1F;
  const uint32_t mant = h & 0x3FF;
  union { uint32_t u; float f; } r;
  if (e == 0) {
    const float v = (float)mant * 5.960464477539063e-08f;
    return sign ? -v : v;
  }
  if (e == 31) {
    if (mant) { r.u = 0x7FC00000u; return r.f; }
    r.u = sign | 0x7F800000u;
    return r.f;
  }
  r.u = sign | ((e + 112) << 23) | (mant << 13);
  return r.f;
}

/* _kernels.py:247-252 gather_f16 */
void orc_gather_f16(const uint16_t* data, int64_t cols, const int64_t* ids, int64_t n,
                    float* out) {
  for (int64_t i = 0; i < n; ++i) {
    const uint16_t* row = data + ids[i] * cols;
    float* o = out + i * cols;
    for (int64_t j = 0; j < cols; ++j) o[j] = half_to_f32(row[j]);
  }
}

/* _kernels.py:225-230 gather_f32 */
void orc_gather_f32(const float* data, int64_t cols, const int64_t* ids, int64_t n, float* out) {
  for (int64_t i = 0; i < n; ++i) memcpy(out + i * cols, data + ids[i] * cols, 4 * cols);
}

/* _kernels.py:255-258 gather_labels */
void orc_gather_labels(const int64_t* y, const int64_t* ids, int64_t n, int64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = y[ids[i]];
}

/* ---- epoch prep: prep.py:226-334 EpochPrepRun with P workers ------------ */
/* Workers pull batch indices from a shared counter (dynamic load balance,
 * prep.py:255-262), sample then slice into a per-worker reusable slot
 * (prep.py:75-85, 264-270).  Per batch: nodes, edges, sampling and slicing
 * seconds are reported; a checksum of the prepared buffers guards against
 * dead-code elimination. */
typedef struct {
  const Graph* g;
  const void* feat;
  int feat_is_f16;
  int64_t cols;
  const int64_t* labels;
  const int64_t* seeds;    /* concatenated plan */
  const int64_t* offsets;  /* nbatch+1 */
  const int64_t* batch_ids;
  int64_t nbatch;
  const int32_t* per_hop;
  int L;
  uint64_t global_seed;
  atomic_long next;
  int64_t* stats; /* nbatch x 4: nodes, edges, sampling_ns, slicing_ns */
  uint64_t* checksums;
} EpochCtx;

static double now_s(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + 1e-9 * t.tv_nsec;
}

static void* epoch_worker(void* arg) {
  EpochCtx* c = (EpochCtx*)arg;
  IdMap m;
  map_init(&m, 1024);
  int maxf = 1;
  for (int h = 0; h < c->L; ++h)
    if (c->per_hop[h] > maxf) maxf = c->per_hop[h];
  int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (maxf + 1));
  HopOut o;
  o.src_cap = 1 << 16;
  o.dptr_cap = 1 << 16;
  o.src = (int64_t*)malloc(sizeof(int64_t) * o.src_cap);
  o.dptr = (int64_t*)malloc(sizeof(int64_t) * o.dptr_cap);
  float* fbuf = NULL;
  int64_t fcap = 0;
  int64_t* lbuf = NULL;
  int64_t lcap = 0;
  for (;;) {
    const int64_t b = atomic_fetch_add(&c->next, 1);
    if (b >= c->nbatch) break;
    const int64_t* seeds = c->seeds + c->offsets[b];
    const int64_t ns = c->offsets[b + 1] - c->offsets[b];
    const double t0 = now_s();
    while (multihop(c->g, &m, seeds, ns, c->per_hop, c->L, c->global_seed, c->batch_ids[b], &o,
                    pos) != 0) {
      o.src_cap *= 2;
      o.dptr_cap *= 2;
      o.src = (int64_t*)realloc(o.src, sizeof(int64_t) * o.src_cap);
      o.dptr = (int64_t*)realloc(o.dptr, sizeof(int64_t) * o.dptr_cap);
    }
    const double t1 = now_s();
    const int64_t need = m.size * c->cols;
    if (need > fcap) {
      free(fbuf);
      fcap = need;
      fbuf = (float*)malloc(sizeof(float) * fcap);
    }
    if (ns > lcap) {
      free(lbuf);
      lcap = ns;
      lbuf = (int64_t*)malloc(sizeof(int64_t) * lcap);
    }
    if (c->feat_is_f16)
      orc_gather_f16((const uint16_t*)c->feat, c->cols, m.globals, m.size, fbuf);
    else
      orc_gather_f32((const float*)c->feat, c->cols, m.globals, m.size, fbuf);
    if (c->labels) orc_gather_labels(c->labels, seeds, ns, lbuf);
    const double t2 = now_s();
    int64_t edges = 0;
    for (int h = 0; h < c->L; ++h) edges += o.meta[h][2];
    uint64_t ck = (uint64_t)m.size * 1315423911ull;
    if (m.size) {
      uint32_t u;
      memcpy(&u, fbuf + (m.size - 1) * c->cols, 4);
      ck ^= u;
    }
    c->stats[4 * b + 0] = m.size;
    c->stats[4 * b + 1] = edges;
    c->stats[4 * b + 2] = (int64_t)((t1 - t0) * 1e9);
    c->stats[4 * b + 3] = (int64_t)((t2 - t1) * 1e9);
    c->checksums[b] = ck;
  }
  free(pos);
  free(o.src);
  free(o.dptr);
  free(fbuf);
  free(lbuf);
  map_free(&m);
  return NULL;
}

/* Returns wall seconds of the epoch (prep.py:316-334 report.both_s). */
double orc_epoch_prep(const int64_t* indptr, const int32_t* indices, int64_t num_nodes,
                      const void* feat, int feat_is_f16, int64_t cols, const int64_t* labels,
                      const int64_t* seeds, const int64_t* offsets, const int64_t* batch_ids,
                      int64_t nbatch, const int32_t* per_hop, int L, uint64_t global_seed,
                      int nthreads, int64_t* stats, uint64_t* checksums) {
  Graph g = {indptr, indices, num_nodes};
  EpochCtx c;
  c.g = &g;
  c.feat = feat;
  c.feat_is_f16 = feat_is_f16;
  c.cols = cols;
  c.labels = labels;
  c.seeds = seeds;
  c.offsets = offsets;
  c.batch_ids = batch_ids;
  c.nbatch = nbatch;
  c.per_hop = per_hop;
  c.L = L;
  c.global_seed = global_seed;
  atomic_init(&c.next, 0);
  c.stats = stats;
  c.checksums = checksums;
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  const double t0 = now_s();
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, epoch_worker, &c);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  const double t1 = now_s();
  free(th);
  return t1 - t0;
}

/* ---- synthetic inputs: host restatement of the device generator --------- *
 * paper_2110_08450_b200/csrc/generate.cu (the on-device law of the reference's
 * synth_graph, graph.py:252-298) rebuilt bit for bit on the host: the checker
 * of the device generator (tests/test_gpu_generate.py) and the way bench.py's
 * reference arm builds the same inputs without loading the product library.
 * Every function takes a thread count and splits its index range. */
typedef struct {
  void (*fn)(void* ctx, int64_t b, int64_t e);
  void* ctx;
  int64_t n;
  int t, nt;
} ParJob;

static void* par_worker(void* arg) {
  ParJob* j = (ParJob*)arg;
  const int64_t b = j->n * j->t / j->nt, e = j->n * (j->t + 1) / j->nt;
  if (e > b) j->fn(j->ctx, b, e);
  return NULL;
}

static void par_for(int64_t n, int nthreads, void (*fn)(void*, int64_t, int64_t), void* ctx) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  ParJob jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].fn = fn;
    jobs[t].ctx = ctx;
    jobs[t].n = n;
    jobs[t].t = t;
    jobs[t].nt = nthreads;
    pthread_create(&th[t], NULL, par_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* common.cuh philox4x32_10 */
static inline void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

typedef struct { int64_t n; uint64_t seed; double scale, a; int64_t* degs; } DegCtx;

static void deg_range(void* p, int64_t b, int64_t e) {
  const DegCtx* c = (const DegCtx*)p;
  const uint32_t k0 = (uint32_t)c->seed ^ 0xDE6u, k1 = (uint32_t)(c->seed >> 32);
  for (int64_t v = b; v < e; ++v) {
    uint32_t r[4] = {(uint32_t)v, (uint32_t)((uint64_t)v >> 32), 0u, 5u};
    philox4x32_10(r, k0, k1);
    const uint64_t bits53 = (((uint64_t)r[0] << 21) ^ ((uint64_t)r[1] >> 11)) & ((1ull << 53) - 1);
    const double w = 1.0 - (double)bits53 * 0x1.0p-53;
    const double y = c->a == 2.0 ? 1.0 / sqrt(w) : pow(w, -1.0 / c->a);
    double d = rint(c->scale * y);
    if (d > (double)(c->n - 1)) d = (double)(c->n - 1);
    if (d < 0.0) d = 0.0;
    c->degs[v] = (int64_t)d;
  }
}

/* generate.cu degrees_kernel */
void orc_synth_degrees(int64_t n, uint64_t seed, double scale, double a, int64_t* degs,
                       int nthreads) {
  DegCtx c = {n, seed, scale, a, degs};
  par_for(n, nthreads, deg_range, &c);
}

typedef struct { int half_bits; uint32_t half_mask; uint32_t keys[6]; } Feistel;

static inline uint32_t feistel_f(uint32_t x, uint32_t k) {
  uint32_t h = x ^ k;
  h ^= h >> 16;
  h *= 0x7feb352du;
  h ^= h >> 15;
  h *= 0x846ca68bu;
  h ^= h >> 16;
  return h;
}

static inline uint64_t feistel_fwd(const Feistel* F, uint64_t x) {
  uint32_t L = (uint32_t)(x >> F->half_bits), R = (uint32_t)x & F->half_mask;
  for (int r = 0; r < 6; ++r) {
    const uint32_t nl = R;
    R = (L ^ feistel_f(R, F->keys[r])) & F->half_mask;
    L = nl;
  }
  return ((uint64_t)L << F->half_bits) | R;
}

static inline uint64_t feistel_inv(const Feistel* F, uint64_t y) {
  uint32_t L = (uint32_t)(y >> F->half_bits), R = (uint32_t)y & F->half_mask;
  for (int r = 5; r >= 0; --r) {
    const uint32_t nr = L;
    L = (R ^ feistel_f(L, F->keys[r])) & F->half_mask;
    R = nr;
  }
  return ((uint64_t)L << F->half_bits) | R;
}

typedef struct {
  const int64_t* indptr;
  int64_t n;
  int32_t* owner;
  Feistel F;
  int64_t n_stubs;
  int32_t* indices;
} PairCtx;

static void owner_range(void* p, int64_t b, int64_t e) {
  const PairCtx* c = (const PairCtx*)p;
  for (int64_t v = b; v < e; ++v)
    for (int64_t s = c->indptr[v]; s < c->indptr[v + 1]; ++s) c->owner[s] = (int32_t)v;
}

static void pair_range(void* p, int64_t b, int64_t e) {
  const PairCtx* c = (const PairCtx*)p;
  const uint64_t n = (uint64_t)c->n_stubs;
  for (int64_t s = b; s < e; ++s) {
    uint64_t q = (uint64_t)s;
    do { q = feistel_inv(&c->F, q); } while (q >= n);
    uint64_t x = q ^ 1ull;
    do { x = feistel_fwd(&c->F, x); } while (x >= n);
    c->indices[s] = c->owner[x];
  }
}

/* generate.cu owner_kernel + pairing_kernel + sal_gen_pairing's key schedule:
 * indices[s] = owner(P(P^-1(s) ^ 1)).  Returns 0, or -1 for an odd stub count. */
int orc_synth_pairing(const int64_t* indptr, int64_t n, uint64_t seed, int32_t* indices,
                      int nthreads) {
  const int64_t n_stubs = indptr[n];
  if (n_stubs % 2) return -1;
  PairCtx c;
  c.indptr = indptr;
  c.n = n;
  c.n_stubs = n_stubs;
  c.indices = indices;
  c.owner = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_stubs > 0 ? n_stubs : 1));
  if (!c.owner) return -2;
  int bits = 2;
  while ((1ull << bits) < (uint64_t)n_stubs) ++bits;
  if (bits & 1) ++bits;
  c.F.half_bits = bits / 2;
  c.F.half_mask = (uint32_t)((1ull << c.F.half_bits) - 1);
  uint64_t k = seed;
  for (int r = 0; r < 6; ++r) {
    k = orc_mix64(k + GOLDEN);
    c.F.keys[r] = (uint32_t)k;
  }
  par_for(n, nthreads, owner_range, &c);
  par_for(n_stubs, nthreads, pair_range, &c);
  free(c.owner);
  return 0;
}

/* IEEE binary32 -> binary16, round to nearest even (what __float2half_rn does) */
static inline uint16_t f32_to_f16_rne(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t ax = x & 0x7FFFFFFFu;
  if (ax >= 0x7F800000u) return (uint16_t)(sign | (ax > 0x7F800000u ? 0x7E00u : 0x7C00u));
  if (ax >= 0x477FF000u) return (uint16_t)(sign | 0x7C00u); /* >= 65520: inf */
  const uint32_t e = ax >> 23, m = (ax & 0x7FFFFFu) | 0x800000u;
  if (e < 113) { /* below 2^-14: subnormal half, unit 2^-24 */
    if (e < 102) return (uint16_t)sign;
    const int shift = 126 - (int)e; /* 14..24 */
    uint32_t q = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (q & 1u))) ++q;
    return (uint16_t)(sign | q);
  }
  uint32_t h = ((e - 112) << 10) | ((ax & 0x7FFFFFu) >> 13);
  const uint32_t rem = ax & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
  return (uint16_t)(sign | h);
}

uint16_t orc_f32_to_f16(float f) { return f32_to_f16_rne(f); }

typedef struct { int64_t row0; int32_t f; int64_t stride; uint64_t seed; uint16_t* out; } FeatCtx;

static void feat_range(void* p, int64_t b, int64_t e) {
  const FeatCtx* c = (const FeatCtx*)p;
  const uint32_t k0 = (uint32_t)c->seed, k1 = (uint32_t)(c->seed >> 32) ^ 0xF3A7u;
  for (int64_t i = b; i < e; ++i) {
    const int64_t row = c->row0 + i;
    uint16_t* dst = c->out + i * c->stride;
    for (int col = 0; col < c->f; col += 4) {
      uint32_t r[4] = {(uint32_t)row, (uint32_t)((uint64_t)row >> 32), (uint32_t)col, 7u};
      philox4x32_10(r, k0, k1);
      for (int j = 0; j < 4 && col + j < c->f; ++j) {
        const float u = (float)(r[j] >> 8) * (1.0f / 16777216.0f);
        dst[col + j] = f32_to_f16_rne(-1.0f + 2.0f * u);
      }
    }
  }
}

/* generate.cu features_kernel for rows [row0, row0 + nrows) into out (row
 * stride `stride` fp16 elements; padding columns untouched) */
void orc_synth_features(int64_t row0, int64_t nrows, int32_t f, int64_t stride, uint64_t seed,
                        uint16_t* out, int nthreads) {
  FeatCtx c = {row0, f, stride, seed, out};
  par_for(nrows, nthreads, feat_range, &c);
}

typedef struct { int32_t C; uint64_t seed; int64_t* out; } LabCtx;

static void lab_range(void* p, int64_t b, int64_t e) {
  const LabCtx* c = (const LabCtx*)p;
  const uint32_t k0 = (uint32_t)c->seed ^ 0x1ABE1u, k1 = (uint32_t)(c->seed >> 32);
  for (int64_t v = b; v < e; ++v) {
    uint32_t r[4] = {(uint32_t)v, (uint32_t)((uint64_t)v >> 32), 0u, 11u};
    philox4x32_10(r, k0, k1);
    c->out[v] = (int64_t)(((uint64_t)r[0] * (uint32_t)c->C) >> 32);
  }
}

/* generate.cu labels_kernel */
void orc_synth_labels(int64_t n, int32_t num_classes, uint64_t seed, int64_t* out, int nthreads) {
  LabCtx c = {num_classes, seed, out};
  par_for(n, nthreads, lab_range, &c);
}
