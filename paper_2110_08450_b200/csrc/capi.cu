// extern "C" boundary of libsalient_b200.so (declared in include/salient_b200.h).
//
// Argument validation happens here, before any launch, and reports through a
// thread-local message (the reference raises ValueError in Python before its
// kernels run: sampler.py:99-100, 311-317; prep.py:160-164).
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "common.cuh"
#include "salient_internal.h"

namespace {

thread_local char g_err[512] = "";
}  // namespace
namespace sal {
std::atomic<long long> g_launches{0};  // kernels enqueued by this library
void count_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
}  // namespace sal
namespace {
using sal::g_launches;

int counted(int rc, int kernels) {
  if (rc == SAL_OK) g_launches.fetch_add(kernels, std::memory_order_relaxed);
  return rc;
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

}  // namespace
namespace sal {
int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
}  // namespace sal
namespace {

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SAL_OK;
  return fail(SAL_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

sal::GraphDev to_dev(const sal_graph* g) {
  sal::GraphDev d;
  d.num_nodes = g->num_nodes;
  d.num_edges = g->num_edges;
  d.indptr = g->indptr;
  d.indices = g->indices;
  return d;
}

int idmap_dev(const sal_idmap* m, sal::IdMapDev* out) {
  if (m == nullptr || m->table == nullptr || m->globals == nullptr)
    return fail(SAL_EINVAL, "idmap: null table or globals");
  const int l2 = sal::log2_exact(m->table_cap);
  if (l2 < 4 || l2 > 31) return fail(SAL_EINVAL, "idmap: table_cap must be a power of two in [16, 2^31]");
  out->table = m->table;
  out->log2cap = l2;
  out->globals = m->globals;
  out->size_out = nullptr;
  return SAL_OK;
}

int64_t pow2_at_least(int64_t n) {
  int64_t p = 16;
  while (p < n) p <<= 1;
  return p;
}

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

}  // namespace

extern "C" {

int sal_version(void) { return 100; }

const char* sal_last_error(void) { return g_err; }

long long sal_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

uint64_t sal_hop_key_prefix(uint64_t global_seed, int64_t batch_id, int64_t hop) {
  return sal::hop_key_prefix(global_seed, (uint64_t)batch_id, (uint64_t)hop);
}

size_t sal_scan_ws_bytes(int64_t max_items) { return sal::scan_ws_bytes(max_items); }

// ---------------------------------------------------------------------------
// plan / layout (sampler.py:321-325 size_hint_for gives the same bound)
// ---------------------------------------------------------------------------
int sal_mfg_plan_init(sal_mfg_plan* plan, int32_t num_hops, const int32_t* per_hop,
                      int64_t max_seeds, int64_t num_nodes) {
  return sal_mfg_plan_init_ex(plan, num_hops, per_hop, max_seeds, num_nodes, 0);
}

int sal_mfg_plan_init_ex(sal_mfg_plan* plan, int32_t num_hops, const int32_t* per_hop,
                         int64_t max_seeds, int64_t num_nodes, int32_t flags) {
  if (plan == nullptr || per_hop == nullptr) return fail(SAL_EINVAL, "plan: null argument");
  if (flags & ~(SAL_MFG_LAST_HOP_EDGES | SAL_MFG_LAST_HOP_FUSED))
    return fail(SAL_EINVAL, "plan: unknown flags 0x%x", flags);
  if (flags & SAL_MFG_LAST_HOP_FUSED) flags |= SAL_MFG_LAST_HOP_EDGES;
  if (num_hops < 1 || num_hops > SAL_MAX_HOPS)
    return fail(SAL_EINVAL, "plan: need 1..%d hops, got %d", SAL_MAX_HOPS, num_hops);
  if (max_seeds < 0 || num_nodes < 0) return fail(SAL_EINVAL, "plan: negative size");
  if (num_nodes >= (1ll << 31)) return fail(SAL_EINVAL, "plan: graphs are limited to 2^31-1 nodes");
  memset(plan, 0, sizeof(*plan));
  plan->num_hops = num_hops;
  plan->max_seeds = max_seeds;
  int64_t nodes = max_seeds < num_nodes ? max_seeds : num_nodes;
  plan->node_cap[0] = nodes;
  for (int h = 0; h < num_hops; ++h) {
    const int32_t f = per_hop[num_hops - 1 - h];  // expansion hop h uses per_hop[L-1-h]
    if (f < 0) return fail(SAL_EINVAL, "plan: fanouts must be >= 0");
    plan->fanout[h] = f;
    plan->edge_cap[h] = nodes * (int64_t)f;
    int64_t next = nodes + nodes * (int64_t)f;
    if (next > num_nodes) next = num_nodes;
    if (next < nodes) next = nodes;
    nodes = next;
    plan->node_cap[h + 1] = nodes;
  }
  if (nodes >= (1ll << 31) - 1) return fail(SAL_EINVAL, "plan: node capacity exceeds int32");
  for (int h = 0; h < num_hops; ++h)
    if (plan->edge_cap[h] >= (1ll << 31) - 1)
      return fail(SAL_EINVAL, "plan: hop %d edge capacity exceeds int32", h);
  plan->flags = flags;
  // the id map holds every node, or (last hop edges-only) the nodes of hops 0..L-2
  const int64_t mapped = (flags & SAL_MFG_LAST_HOP_EDGES) ? plan->node_cap[num_hops - 1] : nodes;
  plan->table_cap = pow2_at_least(2 * (mapped > 8 ? mapped : 8));
  return SAL_OK;
}

// The look-back scan workspaces of one MFG build: hop h's count scan and its
// flag scan each get their own region inside layout.scan, so a single memset at
// hop 0 zeroes all of them and no scan waits on a reset.
static int64_t scan_region(const sal_mfg_plan* plan, int h, int flag, int64_t* bytes) {
  int64_t off = 0;
  for (int k = 0; k < plan->num_hops; ++k)
    for (int q = 0; q < 2; ++q) {
      const int64_t items = q ? plan->edge_cap[k] : plan->node_cap[k];
      const int64_t b = ((int64_t)sal::scan_ws_bytes(items > 0 ? items : 1) + 255) / 256 * 256;
      if (k == h && q == flag) {
        if (bytes) *bytes = b;
        return off;
      }
      off += b;
    }
  if (bytes) *bytes = 0;
  return off;  // total
}

int sal_mfg_layout_init(const sal_mfg_plan* plan, sal_mfg_layout* L) {
  if (plan == nullptr || L == nullptr) return fail(SAL_EINVAL, "layout: null argument");
  memset(L, 0, sizeof(*L));
  const int nh = plan->num_hops;
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    const int64_t o = off;
    off = align_up(off + (bytes > 0 ? bytes : 0), 256);
    return o;
  };
  int64_t max_e = 1, max_d = 1;
  for (int h = 0; h < nh; ++h) {
    if (plan->edge_cap[h] > max_e) max_e = plan->edge_cap[h];
    if (plan->node_cap[h] > max_d) max_d = plan->node_cap[h];
  }
  L->table = take(plan->table_cap * 8);
  L->globals = take(plan->node_cap[nh] * 4 + 4);
  L->sizes = take((nh + 1) * 8);
  L->etot = take(nh * 8);
  for (int h = 0; h < nh; ++h) {
    L->dst_indptr[h] = take((plan->node_cap[h] + 1) * 4);
    L->src_local[h] = take(plan->edge_cap[h] * 4 + 4);
  }
  L->src_glob = take(max_e * 4 + 4);
  L->slot = take(max_e * 4 + 4);
  L->rank = take(max_e * 4 + 4);
  (void)max_d;
  L->scan_bytes = scan_region(plan, plan->num_hops, 0, nullptr);
  L->scan = take(L->scan_bytes);
  L->total = off;
  return SAL_OK;
}

// hops [hop_begin, hop_end) of one batch's MFG (hop_begin == 0 also resets the map
// and inserts the seeds); sal_sample_mfg runs them all
static int sample_mfg_hops(const sal_graph* g, const sal_mfg_plan* plan, const sal_mfg_layout* L,
                           void* ws, const int64_t* seeds_base, const sal_batch_desc* desc,
                           uint64_t global_seed, int32_t rng_policy, int32_t hop_begin,
                           int32_t hop_end, void* stream,
                           const sal::PlanCursor* next = nullptr) {
  if (g == nullptr || plan == nullptr || L == nullptr || ws == nullptr || seeds_base == nullptr ||
      desc == nullptr)
    return fail(SAL_EINVAL, "sample_mfg: null argument");
  if (rng_policy != SAL_RNG_SPLITMIX && rng_policy != SAL_RNG_PHILOX)
    return fail(SAL_EINVAL, "sample_mfg: unknown rng policy %d", rng_policy);
  cudaStream_t st = (cudaStream_t)stream;
  char* base = (char*)ws;
  sal::IdMapDev m;
  m.table = (unsigned long long*)(base + L->table);
  m.log2cap = sal::log2_exact(plan->table_cap);
  m.globals = (int32_t*)(base + L->globals);
  int64_t* sizes = (int64_t*)(base + L->sizes);
  int64_t* etot = (int64_t*)(base + L->etot);
  m.size_out = sizes;
  const sal::GraphDev gd = to_dev(g);
  int32_t* src_glob = (int32_t*)(base + L->src_glob);
  int32_t* slot = (int32_t*)(base + L->slot);
  int32_t* rank = (int32_t*)(base + L->rank);
  void* scan = base + L->scan;

  if (hop_begin < 0 || hop_end > plan->num_hops || hop_begin > hop_end)
    return fail(SAL_EINVAL, "sample_mfg: hop range [%d, %d) outside [0, %d]", hop_begin, hop_end,
                plan->num_hops);
  cudaError_t e = cudaSuccess;
  int kernels = 0;
  // every scan has its own zeroed region (scan_region); hop 0's count runs on its
  // own, each later count rides in the previous hop's resolve launch
  auto scan_ws = [&](int h, int flag) {
    return (void*)((char*)scan + scan_region(plan, h, flag, nullptr));
  };
  if (hop_begin == 0) {
    // table + all scan workspaces as memset nodes: measured faster in the
    // overlapped step than a reset kernel, which takes SM slots from training
    if (!(plan->reset_in_aggregate && (plan->flags & SAL_MFG_LAST_HOP_FUSED))) {
      e = cudaMemsetAsync(m.table, 0xFF, plan->table_cap * 8, st);
      if (e == cudaSuccess) e = cudaMemsetAsync(scan, 0, L->scan_bytes, st);
      if (e != cudaSuccess) return cuda_status(e, "sample_mfg: table reset");
    }
    if (next != nullptr)   // *desc = the plan's next step, then its seeds
      e = sal::launch_seed_insert_next(seeds_base, *next, (sal::BatchDesc*)desc, m, st);
    else
      e = sal::launch_seed_insert(seeds_base, desc, m, plan->max_seeds, st);
    if (e != cudaSuccess) return cuda_status(e, "sample_mfg: seed insert");
    e = sal::launch_hop_count(gd, m.globals, sizes, plan->node_cap[0], plan->fanout[0],
                              (int32_t*)(base + L->dst_indptr[0]), etot, scan_ws(0, 0), st,
                              /*ws_zeroed=*/true);
    if (e != cudaSuccess) return cuda_status(e, "sample_mfg: hop count");
    kernels = 2;
  }
  // a fused last hop is sampled by sal_sample_aggregate
  const int32_t last = (plan->flags & SAL_MFG_LAST_HOP_FUSED) ? plan->num_hops - 1 : plan->num_hops;
  if (hop_end > last) hop_end = last;
  for (int h = hop_begin; h < hop_end; ++h) {
    int32_t* dst_indptr = (int32_t*)(base + L->dst_indptr[h]);
    int32_t* src_local = (int32_t*)(base + L->src_local[h]);
    sal::HopKey hk;
    hk.prefix = 0;
    hk.global_seed = global_seed;
    hk.hop = (uint32_t)h;
    hk.batch = 0;
    hk.derive = 1;
    const bool edges_only = (plan->flags & SAL_MFG_LAST_HOP_EDGES) && h == plan->num_hops - 1;
    if (edges_only) {  // global ids only; sizes[L] = -1 (written by the kernel)
      sal::IdMapDev none = m;
      none.table = nullptr;
      none.size_out = sizes + h + 1;
      e = sal::launch_hop_sample(gd, none, sizes + h, plan->node_cap[h], plan->fanout[h], hk,
                                 desc, rng_policy, nullptr, dst_indptr, src_glob, nullptr,
                                 nullptr, st, plan->sample_lanes, plan->sample_blocks_per_sm);
      if (e != cudaSuccess) return cuda_status(e, "sample_mfg: hop sample");
      return counted(SAL_OK, kernels + 1);
    }
    e = sal::launch_hop_sample(gd, m, sizes + h, plan->node_cap[h], plan->fanout[h], hk, desc,
                               rng_policy, nullptr, dst_indptr, src_glob, slot, nullptr, st,
                               plan->sample_lanes, plan->sample_blocks_per_sm);
    if (e != cudaSuccess) return cuda_status(e, "sample_mfg: hop sample");
    sal::NextCount nc;
    const bool has_next = h + 1 < last;
    if (has_next) {
      nc.g = gd;
      nc.fanout = plan->fanout[h + 1];
      nc.max_dst = plan->node_cap[h + 1];
      nc.dst_indptr = (int32_t*)(base + L->dst_indptr[h + 1]);
      nc.e_total = etot + h + 1;
      nc.scan_ws = scan_ws(h + 1, 0);
    }
    // resolve_in_aggregate: a fused plan's last sampled hop resolves inside
    // sal_sample_aggregate's kernel (off the chain that kernel waits for)
    const bool defer = plan->resolve_in_aggregate && last < plan->num_hops && h == last - 1;
    e = sal::launch_hop_relabel(m, etot + h, plan->edge_cap[h], sizes + h, sizes + h + 1,
                                src_glob, slot, rank, src_local, scan_ws(h, 1), st,
                                /*ws_zeroed=*/true, has_next ? &nc : nullptr, defer);
    if (e != cudaSuccess) return cuda_status(e, "sample_mfg: hop relabel");
    kernels += (defer || !has_next) ? 2 : 3;   // the last relabel resolves in its scan launch
  }
  return counted(SAL_OK, kernels);
}

int sal_sample_mfg(const sal_graph* g, const sal_mfg_plan* plan, const sal_mfg_layout* L,
                   void* ws, const int64_t* seeds_base, const sal_batch_desc* desc,
                   uint64_t global_seed, int32_t rng_policy, void* stream) {
  if (plan == nullptr) return fail(SAL_EINVAL, "sample_mfg: null argument");
  return sample_mfg_hops(g, plan, L, ws, seeds_base, desc, global_seed, rng_policy, 0,
                         plan->num_hops, stream);
}

int sal_sample_mfg_next(const sal_graph* g, const sal_mfg_plan* plan, const sal_mfg_layout* L,
                        void* ws, const int64_t* seeds_base, const int64_t* desc_all,
                        int64_t n_steps, int64_t* cursor, sal_batch_desc* desc_out,
                        uint64_t global_seed, int32_t rng_policy, void* stream) {
  if (plan == nullptr || desc_all == nullptr || cursor == nullptr || desc_out == nullptr)
    return fail(SAL_EINVAL, "sample_mfg_next: null argument");
  if (n_steps < 0) return fail(SAL_EINVAL, "sample_mfg_next: n_steps %lld < 0", (long long)n_steps);
  const sal::PlanCursor pc{desc_all, n_steps, cursor};
  return sample_mfg_hops(g, plan, L, ws, seeds_base, desc_out, global_seed, rng_policy, 0,
                         plan->num_hops, stream, &pc);
}

int sal_sample_aggregate(const sal_graph* g, const sal_mfg_plan* plan, const sal_mfg_layout* L,
                         void* ws, const sal_batch_desc* desc, uint64_t global_seed,
                         int32_t rng_policy, const void* table, int32_t table_dtype,
                         int64_t table_stride, int32_t cols, void* out, int32_t out_dtype,
                         int64_t out_stride, int64_t self_offset, void* stream) {
  if (g == nullptr || plan == nullptr || L == nullptr || ws == nullptr || desc == nullptr ||
      table == nullptr || out == nullptr)
    return fail(SAL_EINVAL, "sample_aggregate: null argument");
  if (!(plan->flags & SAL_MFG_LAST_HOP_FUSED))
    return fail(SAL_EINVAL, "sample_aggregate: the plan has no fused last hop "
                            "(SAL_MFG_LAST_HOP_FUSED)");
  if (rng_policy != SAL_RNG_SPLITMIX && rng_policy != SAL_RNG_PHILOX)
    return fail(SAL_EINVAL, "sample_aggregate: unknown rng policy %d", rng_policy);
  if (table_dtype != SAL_F16) return fail(SAL_EINVAL, "sample_aggregate: the table must be fp16");
  if (out_dtype != SAL_BF16 && out_dtype != SAL_F16)
    return fail(SAL_EINVAL, "sample_aggregate: out dtype must be bf16 or fp16");
  if (cols <= 0 || (cols * 2) % 16 != 0 || cols * 2 > 256)
    return fail(SAL_EINVAL, "sample_aggregate: cols * 2 must be a multiple of 16 in [16, 256], "
                            "got %d columns", cols);
  if ((table_stride * 2) % 16 != 0 || (out_stride * 2) % 16 != 0 ||
      ((uintptr_t)table % 16) != 0 || ((uintptr_t)out % 16) != 0 ||
      (self_offset >= 0 && (self_offset * 2) % 16 != 0))
    return fail(SAL_EINVAL, "sample_aggregate: table/out rows must be 16-byte aligned");
  const int h = plan->num_hops - 1;
  if (plan->fanout[h] > 32)
    return fail(SAL_EINVAL, "sample_aggregate: last-hop fanout %d > 32", plan->fanout[h]);
  char* base = (char*)ws;
  int64_t* sizes = (int64_t*)(base + L->sizes);
  sal::HopKey hk;
  hk.prefix = 0;
  hk.global_seed = global_seed;
  hk.hop = (uint32_t)h;
  hk.batch = 0;
  hk.derive = 1;
  sal::ResolveJob rj{};
  if (h >= 1 && plan->resolve_in_aggregate) {   // hop L-2's deferred resolve (sample_mfg_hops)
    rj.words = (const int32_t*)(base + L->slot);
    rj.e_total = (const int64_t*)(base + L->etot) + (h - 1);
    rj.size_old = sizes + (h - 1);
    rj.rank_of = (const int32_t*)(base + L->rank);
    rj.src_local = (int32_t*)(base + L->src_local[h - 1]);
  }
  return counted(
      cuda_status(sal::launch_sample_mean(to_dev(g), (const int32_t*)(base + L->globals),
                                          sizes + h, plan->node_cap[h], plan->fanout[h], hk, desc,
                                          rng_policy, table, table_stride, cols, out, out_dtype,
                                          out_stride, self_offset, sizes + h + 1,
                                          plan->aggregate_blocks_per_sm,
                                          plan->reset_in_aggregate
                                              ? (unsigned long long*)(base + L->table) : nullptr,
                                          plan->table_cap, base + L->scan, L->scan_bytes, rj,
                                          (cudaStream_t)stream),
                  "sample_aggregate"),
      1);
}

// ---------------------------------------------------------------------------
// hop-level operators
// ---------------------------------------------------------------------------
int sal_idmap_reset(const sal_idmap* m, void* stream) {
  sal::IdMapDev d;
  const int rc = idmap_dev(m, &d);
  if (rc) return rc;
  return cuda_status(cudaMemsetAsync(m->table, 0xFF, m->table_cap * 8, (cudaStream_t)stream),
                     "idmap_reset");
}

int sal_idmap_rehash(const sal_idmap* m, int64_t n, void* stream) {
  sal::IdMapDev d;
  const int rc = idmap_dev(m, &d);
  if (rc) return rc;
  if (n < 0 || n > m->globals_cap) return fail(SAL_EINVAL, "idmap_rehash: bad size %lld", (long long)n);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(m->table, 0xFF, m->table_cap * 8, st);
  if (e != cudaSuccess) return cuda_status(e, "idmap_rehash: reset");
  return counted(cuda_status(sal::launch_rehash(d, n, st), "idmap_rehash"), 1);
}

int sal_idmap_insert(const sal_idmap* m, const int64_t* keys, int64_t n,
                     const int64_t* size_old, int64_t* size_new, int64_t* n_dev_scratch,
                     int32_t* scratch_glob, int32_t* scratch_slot, int32_t* scratch_rank,
                     int32_t* local_out, void* scan_ws, void* stream) {
  sal::IdMapDev d;
  int rc = idmap_dev(m, &d);
  if (rc) return rc;
  if (n < 0) return fail(SAL_EINVAL, "idmap_insert: negative key count");
  if (n > 0 && keys == nullptr) return fail(SAL_EINVAL, "idmap_insert: null keys");
  if (size_old == nullptr || size_new == nullptr || n_dev_scratch == nullptr ||
      scratch_glob == nullptr || scratch_slot == nullptr || scratch_rank == nullptr ||
      scan_ws == nullptr)
    return fail(SAL_EINVAL, "idmap_insert: null scratch argument");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = sal::launch_keys_insert(keys, n, d, scratch_glob, scratch_slot, n_dev_scratch, st);
  if (e != cudaSuccess) return cuda_status(e, "idmap_insert");
  e = sal::launch_hop_relabel(d, n_dev_scratch, n, size_old, size_new, scratch_glob, scratch_slot,
                              scratch_rank, local_out, scan_ws, st);
  return counted(cuda_status(e, "idmap_insert: relabel"), 2);
}

int sal_hop_count(const sal_graph* g, const int32_t* globals, const int64_t* n_dst_dev,
                  int64_t max_dst, int32_t fanout, int32_t* dst_indptr, int64_t* e_total,
                  void* scan_ws, void* stream) {
  if (g == nullptr || globals == nullptr || n_dst_dev == nullptr || dst_indptr == nullptr ||
      e_total == nullptr || scan_ws == nullptr)
    return fail(SAL_EINVAL, "hop_count: null argument");
  if (fanout < 0) return fail(SAL_EINVAL, "hop_count: fanout must be >= 0");
  return counted(cuda_status(sal::launch_hop_count(to_dev(g), globals, n_dst_dev, max_dst, fanout,
                                           dst_indptr, e_total, scan_ws, (cudaStream_t)stream),
                     "hop_count"), 1);
}

int sal_hop_sample(const sal_graph* g, const sal_idmap* m, const int64_t* n_dst_dev,
                   int64_t max_dst, int32_t fanout, uint64_t key_prefix, int32_t rng_policy,
                   uint64_t global_seed, int64_t batch_id, int32_t hop,
                   const int64_t* inject_pos, const int32_t* dst_indptr, int32_t* src_glob,
                   int32_t* slot, int32_t* draws_out, void* stream) {
  return sal_hop_sample_tuned(g, m, n_dst_dev, max_dst, fanout, key_prefix, rng_policy,
                              global_seed, batch_id, hop, inject_pos, dst_indptr, src_glob, slot,
                              draws_out, 0, 0, stream);
}

int sal_hop_sample_tuned(const sal_graph* g, const sal_idmap* m, const int64_t* n_dst_dev,
                         int64_t max_dst, int32_t fanout, uint64_t key_prefix,
                         int32_t rng_policy, uint64_t global_seed, int64_t batch_id, int32_t hop,
                         const int64_t* inject_pos, const int32_t* dst_indptr,
                         int32_t* src_glob, int32_t* slot, int32_t* draws_out, int32_t lanes,
                         int32_t blocks_per_sm, void* stream) {
  if (lanes != 0 && lanes != 8 && lanes != 16 && lanes != 32)
    return fail(SAL_EINVAL, "hop_sample: lanes must be 0 (auto), 8, 16 or 32, got %d", lanes);
  if (blocks_per_sm < 0 || blocks_per_sm > 32)
    return fail(SAL_EINVAL, "hop_sample: blocks_per_sm must be in [0, 32], got %d", blocks_per_sm);
  sal::IdMapDev d;
  int rc = idmap_dev(m, &d);
  if (rc) return rc;
  if (g == nullptr || n_dst_dev == nullptr || dst_indptr == nullptr || src_glob == nullptr ||
      slot == nullptr)
    return fail(SAL_EINVAL, "hop_sample: null argument");
  if (rng_policy != SAL_RNG_SPLITMIX && rng_policy != SAL_RNG_PHILOX)
    return fail(SAL_EINVAL, "hop_sample: unknown rng policy %d", rng_policy);
  sal::HopKey hk;
  hk.prefix = key_prefix;
  hk.global_seed = global_seed;
  hk.hop = (uint32_t)hop;
  hk.batch = (uint32_t)batch_id;
  hk.derive = 0;
  return counted(cuda_status(sal::launch_hop_sample(to_dev(g), d, n_dst_dev, max_dst, fanout, hk, nullptr,
                                            rng_policy, inject_pos, dst_indptr, src_glob, slot,
                                            draws_out, (cudaStream_t)stream, lanes,
                                            blocks_per_sm),
                     "hop_sample"), 1);
}

int sal_hop_relabel(const sal_idmap* m, const int64_t* e_total, int64_t max_edges,
                    const int64_t* size_old, int64_t* size_new, const int32_t* src_glob,
                    const int32_t* slot, int32_t* rank, int32_t* src_local, void* scan_ws,
                    void* stream) {
  sal::IdMapDev d;
  int rc = idmap_dev(m, &d);
  if (rc) return rc;
  if (e_total == nullptr || size_old == nullptr || size_new == nullptr || src_glob == nullptr ||
      slot == nullptr || rank == nullptr || scan_ws == nullptr)
    return fail(SAL_EINVAL, "hop_relabel: null argument");
  return counted(cuda_status(sal::launch_hop_relabel(d, e_total, max_edges, size_old, size_new, src_glob,
                                             slot, rank, src_local, scan_ws,
                                             (cudaStream_t)stream),
                     "hop_relabel"), 1);
}

// ---------------------------------------------------------------------------
// slicing
// ---------------------------------------------------------------------------
static bool valid_dtype(int32_t t) { return t == SAL_F16 || t == SAL_F32 || t == SAL_BF16; }

int sal_gather_rows(const void* x, int64_t x_rows, int32_t cols, int64_t x_stride,
                    int32_t in_dtype, const void* ids, int32_t id_bytes, const int64_t* n_dev,
                    int64_t n, void* out, int64_t out_stride, int32_t out_dtype, void* stream) {
  if (!valid_dtype(in_dtype) || !valid_dtype(out_dtype))
    return fail(SAL_EINVAL, "gather_rows: unsupported dtype (%d -> %d)", in_dtype, out_dtype);
  if (id_bytes != 4 && id_bytes != 8) return fail(SAL_EINVAL, "gather_rows: id_bytes must be 4 or 8");
  if (cols < 0 || n < 0 || x_stride < cols || out_stride < cols)
    return fail(SAL_EINVAL, "gather_rows: bad shape");
  if (n == 0 && n_dev == nullptr) return SAL_OK;
  if (cols == 0) return SAL_OK;
  if (x == nullptr || ids == nullptr || out == nullptr)
    return fail(SAL_EINVAL, "gather_rows: null argument");
  return counted(cuda_status(sal::launch_gather_rows(x, x_rows, cols, x_stride, in_dtype, ids, id_bytes,
                                             n_dev, n, out, out_stride, out_dtype,
                                             (cudaStream_t)stream),
                     "gather_rows"), 1);
}

int sal_gather_labels(const int64_t* y, const int64_t* seeds_base, const sal_batch_desc* desc,
                      int64_t max_n, int64_t* out, void* stream) {
  if (y == nullptr || seeds_base == nullptr || desc == nullptr || out == nullptr)
    return fail(SAL_EINVAL, "gather_labels: null argument");
  return counted(cuda_status(
      sal::launch_gather_labels(y, seeds_base, desc, max_n, out, (cudaStream_t)stream),
      "gather_labels"), 1);
}

// ---------------------------------------------------------------------------
// aggregation
// ---------------------------------------------------------------------------
int sal_segment_mean_fwd(const int32_t* indptr, const int32_t* src, const int64_t* n_dst_dev,
                         int64_t n_pad, const void* h, int32_t h_dtype, int64_t h_stride,
                         int32_t f, void* out, int32_t out_dtype, int64_t out_stride,
                         void* stream) {
  return sal_segment_mean_fwd_ex(indptr, src, n_dst_dev, n_pad, h, h_dtype, h_stride, f, out,
                                 out_dtype, out_stride, 0, stream);
}

int sal_segment_mean_fwd_ex(const int32_t* indptr, const int32_t* src, const int64_t* n_dst_dev,
                            int64_t n_pad, const void* h, int32_t h_dtype, int64_t h_stride,
                            int32_t f, void* out, int32_t out_dtype, int64_t out_stride,
                            int32_t flags, void* stream) {
  if (flags & ~SAL_SEG_NO_PAD_FILL) return fail(SAL_EINVAL, "segment_mean_fwd: bad flags");
  if (!valid_dtype(h_dtype) || !valid_dtype(out_dtype))
    return fail(SAL_EINVAL, "segment_mean_fwd: unsupported dtype");
  if (f < 0 || n_pad < 0) return fail(SAL_EINVAL, "segment_mean_fwd: bad shape");
  if (n_pad == 0 || f == 0) return SAL_OK;
  if (indptr == nullptr || src == nullptr || h == nullptr || out == nullptr)
    return fail(SAL_EINVAL, "segment_mean_fwd: null argument");
  return counted(cuda_status(sal::launch_segment_mean_fwd(indptr, src, nullptr, n_dst_dev, n_pad, h,
                                                  h_dtype, h_stride, f, out, out_dtype,
                                                  out_stride, (cudaStream_t)stream,
                                                  !(flags & SAL_SEG_NO_PAD_FILL)),
                     "segment_mean_fwd"), 1);
}

int sal_segment_mean_fwd_global(const int32_t* indptr, const int32_t* src,
                                const int32_t* globals, const int64_t* n_dst_dev, int64_t n_pad,
                                const void* x, int32_t x_dtype, int64_t x_stride, int32_t f,
                                void* out, int32_t out_dtype, int64_t out_stride, void* stream) {
  if (!valid_dtype(x_dtype) || !valid_dtype(out_dtype))
    return fail(SAL_EINVAL, "segment_mean_fwd_global: unsupported dtype");
  if (f < 0 || n_pad < 0) return fail(SAL_EINVAL, "segment_mean_fwd_global: bad shape");
  if (n_pad == 0 || f == 0) return SAL_OK;
  if (indptr == nullptr || src == nullptr || globals == nullptr || x == nullptr || out == nullptr)
    return fail(SAL_EINVAL, "segment_mean_fwd_global: null argument");
  return counted(cuda_status(sal::launch_segment_mean_fwd(indptr, src, globals, n_dst_dev, n_pad, x,
                                                  x_dtype, x_stride, f, out, out_dtype,
                                                  out_stride, (cudaStream_t)stream),
                     "segment_mean_fwd_global"), 1);
}

int sal_segment_mean_bwd(const int32_t* indptr, const int32_t* src, const int64_t* n_dst_dev,
                         int64_t n_pad, const void* g_out, int32_t g_dtype, int64_t g_stride,
                         int32_t f, float* g_h, int64_t gh_stride, void* stream) {
  if (!valid_dtype(g_dtype)) return fail(SAL_EINVAL, "segment_mean_bwd: unsupported dtype");
  if (f < 0 || n_pad < 0) return fail(SAL_EINVAL, "segment_mean_bwd: bad shape");
  if (n_pad == 0 || f == 0) return SAL_OK;
  if (indptr == nullptr || src == nullptr || g_out == nullptr || g_h == nullptr)
    return fail(SAL_EINVAL, "segment_mean_bwd: null argument");
  return counted(cuda_status(sal::launch_segment_mean_bwd(indptr, src, n_dst_dev, n_pad, g_out, g_dtype,
                                                  g_stride, f, g_h, gh_stride,
                                                  (cudaStream_t)stream),
                     "segment_mean_bwd"), 1);
}

}  // extern "C"
