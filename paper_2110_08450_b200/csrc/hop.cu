// Per-hop MFG construction on device: count -> sample(+insert) -> relabel.
//
// Reference loops replaced (pkg/src/mfgprep):
//   hop_budget          _kernels.py:42-50    -> count_scan_kernel
//   _sample_positions   _kernels.py:102-147  -> sample_insert_kernel (warp per dst)
//   hop_kernel (fused)  _kernels.py:150-185  -> sample_insert + flag_scan + resolve
//   _map_get_or_insert  _kernels.py:76-99    -> open-addressing table, atomicMin
//   insert_keys         _kernels.py:216-222  -> keys_insert_kernel + flag_scan + resolve
//
// Relabel semantics (bit-exact with the reference's sequential map): a global
// id already in the map keeps its local; a new id receives
//     local = size_before_hop + #(distinct new ids whose first occurrence in
//             the edge sequence precedes this id's first occurrence).
// The edge sequence is (dst ascending, acceptance order), so "first
// occurrence" = minimum edge index, obtained with a 64-bit atomicMin on the
// packed slot word {key:32 | NEWF | first_edge:31}.
#include "common.cuh"
#include "salient_internal.h"
#include "sampling.cuh"

namespace sal {

constexpr uint64_t kEmpty = ~0ull;

SAL_DEVINL uint32_t table_hash(uint32_t key, int log2cap) {
  return (uint32_t)(((uint64_t)key * kGolden) >> (64 - log2cap));
}

// Get-or-insert a candidate (key, edge e).  Returns the slot index.
SAL_DEVINL uint32_t table_insert_min(unsigned long long* table, int log2cap, uint32_t key,
                                     uint32_t e) {
  const uint32_t mask = (1u << log2cap) - 1u;
  const unsigned long long mine = ((unsigned long long)key << 32) | (kNewFlag | e);
  uint32_t s = table_hash(key, log2cap);
  while (true) {
    unsigned long long w = *((volatile unsigned long long*)&table[s]);
    if (w == kEmpty) {
      const unsigned long long old = atomicCAS(&table[s], kEmpty, mine);
      if (old == kEmpty) return s;
      w = old;
    }
    if ((uint32_t)(w >> 32) == key) {
      if ((w & kNewFlag) && mine < w) atomicMin(&table[s], mine);
      return s;
    }
    s = (s + 1) & mask;
  }
}

// Insert an already-assigned (key, local) pair (seed destinations).
SAL_DEVINL void table_insert_assigned(unsigned long long* table, int log2cap, uint32_t key,
                                      uint32_t local) {
  const uint32_t mask = (1u << log2cap) - 1u;
  const unsigned long long mine = ((unsigned long long)key << 32) | local;
  uint32_t s = table_hash(key, log2cap);
  while (true) {
    const unsigned long long old = atomicCAS(&table[s], kEmpty, mine);
    if (old == kEmpty || (uint32_t)(old >> 32) == key) return;
    s = (s + 1) & mask;
  }
}

// ---------------------------------------------------------------------------
// seeds -> locals 0..n-1 (sampler.py:336-340: id_map.insert(seeds.dst_ids))
// ---------------------------------------------------------------------------

__global__ void seed_insert_kernel(const int64_t* __restrict__ seeds_base,
                                   const BatchDesc* __restrict__ desc,
                                   unsigned long long* table, int log2cap,
                                   int32_t* __restrict__ globals, int64_t* __restrict__ size0) {
  const int64_t n = desc->n_seeds;
  const int64_t* seeds = seeds_base + desc->seed_offset;
  if (blockIdx.x == 0 && threadIdx.x == 0) *size0 = n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = (uint32_t)seeds[i];
    globals[i] = (int32_t)key;
    table_insert_assigned(table, log2cap, key, (uint32_t)i);
  }
}

// seed insertion that first takes the next batch off a device epoch plan (what
// sal_plan_next does, folded in: one launch fewer at the head of the chain).  One
// block, so thread 0 alone reads and advances the cursor.
__global__ void __launch_bounds__(1024)
seed_insert_next_kernel(const int64_t* __restrict__ seeds_base,
                        const int64_t* __restrict__ desc_all, int64_t n_steps,
                        int64_t* __restrict__ cursor, BatchDesc* __restrict__ desc_out,
                        unsigned long long* table, int log2cap, int32_t* __restrict__ globals,
                        int64_t* __restrict__ size0) {
  __shared__ int64_t sh[3];
  if (threadIdx.x == 0) {
    const int64_t c = *cursor;
    const bool live = c < n_steps;
    sh[0] = live ? desc_all[3 * c + 0] : -1;
    sh[1] = live ? desc_all[3 * c + 1] : 0;
    sh[2] = live ? desc_all[3 * c + 2] : 0;
    desc_out->batch_id = sh[0];
    desc_out->seed_offset = sh[1];
    desc_out->n_seeds = sh[2];
    *cursor = c + 1;
    *size0 = sh[2];
  }
  __syncthreads();
  const int64_t n = sh[2];
  const int64_t* seeds = seeds_base + sh[1];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t key = (uint32_t)seeds[i];
    globals[i] = (int32_t)key;
    table_insert_assigned(table, log2cap, key, (uint32_t)i);
  }
}

// re-insert locals 0..n-1 into a fresh table (sampler.py:131-145 ensure_capacity)
__global__ void rehash_kernel(const int32_t* __restrict__ globals, int64_t n,
                              unsigned long long* table, int log2cap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    table_insert_assigned(table, log2cap, (uint32_t)globals[i], (uint32_t)i);
}

// ---------------------------------------------------------------------------
// count + exclusive scan: dst_indptr[i] = sum_{j<i} min(deg(globals[j]), f)
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

SAL_DEVINL void count_scan_tile(const int64_t* __restrict__ indptr,
                                const int32_t* __restrict__ globals,
                                const int64_t* __restrict__ n_dst_ptr, int32_t fanout,
                                int32_t* __restrict__ dst_indptr, int64_t* __restrict__ e_total,
                                ScanWs ws) {
  __shared__ uint64_t sh_scan[kScanThreads / kWarp + 1];
  __shared__ uint64_t sh_prefix;
  __shared__ int sh_tile;
  const int64_t n = *n_dst_ptr;
  const int64_t ntiles = n > 0 ? (n + kScanTile - 1) / kScanTile : 1;
  const int tile = grab_tile(ws, &sh_tile);
  if (tile >= ntiles) return;
  const int64_t base = (int64_t)tile * kScanTile + threadIdx.x * kScanItems;
  uint32_t c[kScanItems];
  uint64_t local = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    c[k] = 0;
    if (i < n) {
      const int32_t v = globals[i];
      const int64_t deg = ld_i64(indptr + v + 1) - ld_i64(indptr + v);
      c[k] = (uint32_t)(deg < fanout ? deg : fanout);
    }
    local += c[k];
  }
  uint64_t tile_total;
  uint64_t excl = block_exclusive_scan<uint64_t, kScanThreads>(local, sh_scan, &tile_total);
  const uint64_t prefix = lookback_prefix(ws, tile, tile_total, &sh_prefix);
  uint64_t run = prefix + excl;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    if (i < n) dst_indptr[i] = (int32_t)run;
    run += c[k];
  }
  if (tile == ntiles - 1 && threadIdx.x == kScanThreads - 1) {
    dst_indptr[n] = (int32_t)(prefix + tile_total);
    *e_total = (int64_t)(prefix + tile_total);
  }
}

__global__ void __launch_bounds__(kScanThreads)
count_scan_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ globals,
                  const int64_t* __restrict__ n_dst_ptr, int32_t fanout,
                  int32_t* __restrict__ dst_indptr, int64_t* __restrict__ e_total, ScanWs ws) {
  count_scan_tile(indptr, globals, n_dst_ptr, fanout, dst_indptr, e_total, ws);
}

// ---------------------------------------------------------------------------
// sampling (+ fused table insertion), one warp per destination
// ---------------------------------------------------------------------------
SAL_DEVINL void emit_edge(const int32_t* __restrict__ indices, int64_t slot_pos, int64_t e,
                          unsigned long long* table, int log2cap, int32_t* src_glob,
                          int32_t* __restrict__ slot) {
  const uint32_t key = (uint32_t)__ldg(indices + slot_pos);
  src_glob[e] = (int32_t)key;
  if (table != nullptr)  // null: edges-only hop (SAL_MFG_LAST_HOP_EDGES)
    slot[e] = (int32_t)table_insert_min(table, log2cap, key, (uint32_t)e);
}

// G lanes per destination (G = 32, 16 or 8; 32/G destinations per warp in
// flight).  Rejection sampling runs G draws per round: lane l of the group
// takes draw ctr + l; a draw is fresh if its position is not yet accepted and
// no lower lane of the group drew the same position this round; fresh draws
// are accepted in lane order until the fanout is reached — exactly the
// sequential loop of _sample_positions (_kernels.py:119-146).
// kMinBlocks = 8 holds the kernel to 32 registers (a few bytes of spill) so 64
// warps are resident instead of 48: the large hops (tens of thousands of
// destinations, several per group) are bound by how many insert chains are in
// flight — full 3-hop MFG 120.7 -> 107-112 us one batch at a time, 62.2 -> 59.0 us
// per batch at 8 streams (profiles/r2_ab_sample_regs.txt).  The small hops of the
// training chain measured 0.3 us per step slower that way and keep 6.
template <int kPolicy, int G, int kMinBlocks>
__global__ void __launch_bounds__(256, kMinBlocks)
sample_insert_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                     const int32_t* __restrict__ globals, const int64_t* __restrict__ n_dst_ptr,
                     int32_t fanout, HopKey hk, const BatchDesc* __restrict__ desc,
                     const int64_t* __restrict__ inject_pos, const int32_t* __restrict__ dst_indptr,
                     unsigned long long* table, int log2cap, int32_t* src_glob,
                     int32_t* __restrict__ slot, int32_t* __restrict__ draws_out,
                     int64_t* __restrict__ size_unknown) {
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  const unsigned lt_mask = ((1u << lane) - 1u) & gmask;
  const int64_t n = *n_dst_ptr;
  const int64_t group_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  // key prefix: by value (hop API) or derived on device from the batch id
  uint64_t prefix = hk.prefix;
  uint32_t batch = hk.batch;
  if (desc != nullptr) {
    batch = (uint32_t)desc->batch_id;
    if (hk.derive) prefix = hop_key_prefix(hk.global_seed, (uint64_t)desc->batch_id, hk.hop);
  }
  const uint2 pkey = make_uint2((uint32_t)hk.global_seed, (uint32_t)(hk.global_seed >> 32));
  __shared__ int32_t sh_acc[8][32];
  if (size_unknown != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *size_unknown = -1;

  for (int64_t i = group_id; i < n; i += ngroups) {
    const int32_t v = globals[i];
    const int64_t lo = ld_i64(indptr + v);
    const int64_t deg = ld_i64(indptr + v + 1) - lo;
    const int64_t out = dst_indptr[i];
    if (deg <= fanout) {  // take-all, CSR order, no draws (_kernels.py:168-174)
      if (draws_out != nullptr && gl == 0) draws_out[i] = 0;
      for (int64_t p = gl; p < deg; p += G)
        emit_edge(indices, lo + p, out + p, table, log2cap, src_glob, slot);
      continue;
    }
    if (inject_pos != nullptr) {  // positions injected from the reference
      for (int j = gl; j < fanout; j += G)
        emit_edge(indices, lo + inject_pos[out + j], out + j, table, log2cap, src_glob, slot);
      continue;
    }
    const uint64_t key = mix64(prefix ^ (uint64_t)i);  // _kernels.py:167
    const uint32_t udeg = (uint32_t)deg;
    const uint64_t recip = kPolicy == kRngSplitmix ? recip_u32(udeg) : 0ull;
    // accepted positions: this group's slice of shared memory when the fanout
    // fits, else staged in this destination's own output range
    int32_t* accepted = fanout <= G ? &sh_acc[threadIdx.x >> 5][grp * G] : src_glob + out;
    int acc = 0;
    uint32_t ctr = 0;
    while (acc < fanout) {
      const uint32_t pos = draw_position<kPolicy>(key, pkey, ctr + gl, (uint32_t)i, hk.hop,
                                                  batch, udeg, recip);
      bool hit = false;
      for (int j = 0; j < acc; ++j) hit |= ((uint32_t)accepted[j] == pos);
      const unsigned peers = __match_any_sync(gmask, pos) & gmask;
      const bool fresh = !hit && (peers & lt_mask) == 0;
      const unsigned fresh_mask = __ballot_sync(gmask, fresh) & gmask;
      const int rank = __popc(fresh_mask & lt_mask);
      if (fresh && acc + rank < fanout) accepted[acc + rank] = (int32_t)pos;
      const int nfresh = __popc(fresh_mask);
      if (draws_out != nullptr && acc + nfresh >= fanout && gl == 0) {
        // CounterRng.counter after the loop: index of the completing draw + 1
        unsigned m = fresh_mask >> (grp * G);
        for (int t = 1; t < fanout - acc; ++t) m &= m - 1;
        draws_out[i] = (int32_t)(ctr + __ffs(m));
      }
      acc += min(nfresh, fanout - acc);
      ctr += G;
      __syncwarp(gmask);
    }
    for (int j = gl; j < fanout; j += G) {
      const int64_t p = accepted[j];
      emit_edge(indices, lo + p, out + j, table, log2cap, src_glob, slot);
    }
    __syncwarp(gmask);
  }
}

// Generic get-or-insert of an arbitrary key sequence (IdMap.insert).
__global__ void keys_insert_kernel(const int64_t* __restrict__ keys, int64_t n,
                                   unsigned long long* table, int log2cap,
                                   int32_t* __restrict__ src_glob, int32_t* __restrict__ slot,
                                   int64_t* __restrict__ e_total) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *e_total = n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = (uint32_t)keys[e];
    src_glob[e] = (int32_t)key;
    slot[e] = (int32_t)table_insert_min(table, log2cap, key, (uint32_t)e);
  }
}

// ---------------------------------------------------------------------------
// relabel pass 1: first-occurrence flags -> scan -> new locals appended
// ---------------------------------------------------------------------------
// kResolve: the chain's last relabel (no next-hop count rides with its resolve)
// also runs pass 2 in the same launch.  Every edge already holds its table word;
// a first occurrence at edge `first` <= e lives in this tile or an earlier one,
// and tiles are taken in order (grab_tile), so an edge waits only for a tile that
// is already running: that tile sets kFlagRanks in its scan status once its
// rank_of entries are written.  A word read after the first's tile finalized its
// slot carries the local itself, so either reading resolves to the same local.
template <bool kResolve>
__global__ void __launch_bounds__(kScanThreads)
flag_scan_kernel(unsigned long long* table, const int32_t* __restrict__ slot,
                 const int32_t* __restrict__ src_glob, const int64_t* __restrict__ e_total,
                 const int64_t* __restrict__ size_old_ptr, int64_t* __restrict__ size_new_ptr,
                 int32_t* rank_of, int32_t* __restrict__ globals, ScanWs ws,
                 int32_t* __restrict__ word_out, int32_t* __restrict__ src_local) {
  __shared__ uint64_t sh_scan[kScanThreads / kWarp + 1];
  __shared__ uint64_t sh_prefix;
  __shared__ int sh_tile;
  const int64_t n = *e_total;
  const int64_t ntiles = n > 0 ? (n + kScanTile - 1) / kScanTile : 1;
  const int tile = grab_tile(ws, &sh_tile);
  if (tile >= ntiles) return;
  const int64_t size_old = *size_old_ptr;
  const int64_t base = (int64_t)tile * kScanTile + threadIdx.x * kScanItems;
  uint32_t flags = 0;
  uint64_t local = 0;
  unsigned long long words[kScanItems];
  int32_t slots[kScanItems];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t e = base + k;
    words[k] = 0;
    slots[k] = 0;
    if (e < n) {
      slots[k] = slot[e];
      const unsigned long long w = kResolve ? *((volatile unsigned long long*)&table[slots[k]])
                                            : table[slots[k]];
      words[k] = w;
      const uint32_t lo = (uint32_t)w;
      // deferred resolve: keep the edge's final table word (resolve_words, run later
      // without the table)
      if (word_out != nullptr) word_out[e] = (int32_t)lo;
      if ((lo & kNewFlag) && (lo & ~kNewFlag) == (uint32_t)e) {
        flags |= 1u << k;
        ++local;
      }
    }
  }
  uint64_t tile_total;
  uint64_t excl = block_exclusive_scan<uint64_t, kScanThreads>(local, sh_scan, &tile_total);
  const uint64_t prefix = lookback_prefix(ws, tile, tile_total, &sh_prefix);
  uint64_t run = prefix + excl;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (flags & (1u << k)) {
      const int64_t e = base + k;
      rank_of[e] = (int32_t)run;
      globals[size_old + run] = src_glob[e];
      ++run;
    }
  }
  if (tile == ntiles - 1 && threadIdx.x == kScanThreads - 1)
    *size_new_ptr = size_old + (int64_t)(prefix + tile_total);
  if (!kResolve) return;
  __syncthreads();  // this tile's ranks, for the block
  if (threadIdx.x == 0) {
    __threadfence();
    atomicOr(&ws.status[tile], (unsigned long long)kFlagRanks);
  }
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t e = base + k;
    if (e >= n) continue;
    const unsigned long long w = words[k];
    const uint32_t lo = (uint32_t)w;
    uint32_t loc = lo;
    if (lo & kNewFlag) {
      const uint32_t first = lo & ~kNewFlag;
      const int ft = (int)(first / kScanTile);
      if (ft != tile) {
        while ((*((volatile unsigned long long*)&ws.status[ft]) & kFlagRanks) == 0) {
        }
        __threadfence();
      }
      loc = (uint32_t)(size_old + *((volatile int32_t*)&rank_of[first]));
      if (first == (uint32_t)e) table[slots[k]] = (w & 0xFFFFFFFF00000000ull) | loc;
    }
    if (src_local != nullptr) src_local[e] = (int32_t)loc;
  }
}

// relabel pass 2: every edge resolves its local id; first occurrences
// finalize their slot so the next hop sees an assigned entry.
SAL_DEVINL void resolve_range(unsigned long long* table, const int32_t* __restrict__ slot,
                              const int64_t* __restrict__ e_total,
                              const int64_t* __restrict__ size_old_ptr,
                              const int32_t* __restrict__ rank_of,
                              int32_t* __restrict__ src_local, int64_t first, int64_t stride) {
  const int64_t n = *e_total;
  const int64_t size_old = *size_old_ptr;
  for (int64_t e = first; e < n; e += stride) {
    const int32_t s = slot[e];
    const unsigned long long w = *((volatile unsigned long long*)&table[s]);
    const uint32_t lo = (uint32_t)w;
    uint32_t local;
    if (lo & kNewFlag) {
      const uint32_t first = lo & ~kNewFlag;
      local = (uint32_t)(size_old + rank_of[first]);
      if (first == (uint32_t)e) table[s] = (w & 0xFFFFFFFF00000000ull) | local;
    } else {
      local = lo;
    }
    if (src_local != nullptr) src_local[e] = (int32_t)local;
  }
}

// resolve of hop h and the count + scan of hop h+1 in one launch: both read only
// what flag_scan(h) wrote (the new locals' global ids, the new map size), so the
// first `resolve_blocks` blocks resolve edges while the rest scan destinations
struct CountJob {
  const int64_t* indptr;
  const int32_t* globals;
  const int64_t* n_dst;
  int32_t fanout;
  int32_t* dst_indptr;
  int64_t* e_total;
  ScanWs ws;
};
__global__ void __launch_bounds__(kScanThreads)
resolve_count_kernel(unsigned long long* table, const int32_t* __restrict__ slot,
                     const int64_t* __restrict__ e_total, const int64_t* __restrict__ size_old_ptr,
                     const int32_t* __restrict__ rank_of, int32_t* __restrict__ src_local,
                     int resolve_blocks, CountJob cj) {
  if ((int)blockIdx.x < resolve_blocks)
    resolve_range(table, slot, e_total, size_old_ptr, rank_of, src_local,
                  blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                  (int64_t)resolve_blocks * blockDim.x);
  else
    count_scan_tile(cj.indptr, cj.globals, cj.n_dst, cj.fanout, cj.dst_indptr, cj.e_total, cj.ws);
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static int g_num_sms = 0;
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

int log2_exact(int64_t cap) {
  int l = 0;
  while ((1ll << l) < cap) ++l;
  return ((1ll << l) == cap) ? l : -1;
}

size_t scan_ws_bytes(int64_t max_items) {
  const int64_t tiles = (max_items + kScanTile - 1) / kScanTile + 1;
  return (size_t)(tiles * 8 + 16);
}

static ScanWs carve_scan_ws(void* p, int64_t max_items) {
  const int64_t tiles = (max_items + kScanTile - 1) / kScanTile + 1;
  ScanWs ws;
  ws.status = (unsigned long long*)p;
  ws.tile_counter = (unsigned int*)((char*)p + tiles * 8);
  return ws;
}

static int scan_grid(int64_t max_items) {
  const int64_t tiles = (max_items + kScanTile - 1) / kScanTile;
  return (int)(tiles > 0 ? tiles : 1);
}

cudaError_t launch_seed_insert(const int64_t* seeds_base, const BatchDesc* desc,
                               const IdMapDev& m, int64_t max_seeds, cudaStream_t st) {
  int grid = (int)((max_seeds + 255) / 256);
  if (grid < 1) grid = 1;
  seed_insert_kernel<<<grid, 256, 0, st>>>(seeds_base, desc, m.table, m.log2cap, m.globals,
                                           m.size_out);
  return cudaGetLastError();
}

cudaError_t launch_seed_insert_next(const int64_t* seeds_base, const PlanCursor& pc,
                                    BatchDesc* desc_out, const IdMapDev& m, cudaStream_t st) {
  seed_insert_next_kernel<<<1, 1024, 0, st>>>(seeds_base, pc.desc_all, pc.n_steps, pc.cursor,
                                              desc_out, m.table, m.log2cap, m.globals,
                                              m.size_out);
  return cudaGetLastError();
}

cudaError_t launch_rehash(const IdMapDev& m, int64_t n, cudaStream_t st) {
  int64_t grid = (n + 255) / 256;
  if (grid < 1) grid = 1;
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  rehash_kernel<<<(int)grid, 256, 0, st>>>(m.globals, n, m.table, m.log2cap);
  return cudaGetLastError();
}

cudaError_t launch_hop_count(const GraphDev& g, const int32_t* globals, const int64_t* n_dst,
                             int64_t max_dst, int32_t fanout, int32_t* dst_indptr,
                             int64_t* e_total, void* scan_ws, cudaStream_t st, bool ws_zeroed) {
  ScanWs ws = carve_scan_ws(scan_ws, max_dst);
  if (!ws_zeroed) {
    cudaError_t err = cudaMemsetAsync(scan_ws, 0, scan_ws_bytes(max_dst), st);
    if (err != cudaSuccess) return err;
  }
  count_scan_kernel<<<scan_grid(max_dst), kScanThreads, 0, st>>>(g.indptr, globals, n_dst, fanout,
                                                                dst_indptr, e_total, ws);
  return cudaGetLastError();
}

cudaError_t launch_hop_sample(const GraphDev& g, const IdMapDev& m, const int64_t* n_dst,
                              int64_t max_dst, int32_t fanout, HopKey hk, const BatchDesc* desc,
                              int32_t policy, const int64_t* inject_pos,
                              const int32_t* dst_indptr, int32_t* src_glob, int32_t* slot,
                              int32_t* draws_out, cudaStream_t st, int lanes,
                              int blocks_per_sm) {
  const int64_t warps_needed = max_dst > 0 ? max_dst : 1;
  int64_t grid = (warps_needed + 7) / 8;
  // default 8 blocks x 8 warps per SM, grid-stride
  const int64_t cap = (int64_t)num_sms() * (blocks_per_sm > 0 ? blocks_per_sm : 8);
  if (grid > cap) grid = cap;
  // lanes per destination: by default the smallest group that holds the fanout
  const int G = lanes == 8 || lanes == 16 || lanes == 32
                    ? lanes
                    : (fanout <= 8 ? 8 : (fanout <= 16 ? 16 : 32));
  grid = (warps_needed * G / 32 + 7) / 8;
  if (grid < 1) grid = 1;
  if (grid > cap) grid = cap;
  const bool wide = max_dst >= 16384;   // a large hop: the 64-warp variant
#define SAL_SAMPLE(P, GG)                                                                    \
  do {                                                                                       \
    if (wide)                                                                                \
      sample_insert_kernel<P, GG, 8><<<(int)grid, 256, 0, st>>>(                             \
          g.indptr, g.indices, m.globals, n_dst, fanout, hk, desc, inject_pos, dst_indptr,   \
          m.table, m.log2cap, src_glob, slot, draws_out,                                     \
          m.table == nullptr ? m.size_out : nullptr);                                        \
    else                                                                                     \
      sample_insert_kernel<P, GG, 6><<<(int)grid, 256, 0, st>>>(                             \
          g.indptr, g.indices, m.globals, n_dst, fanout, hk, desc, inject_pos, dst_indptr,   \
          m.table, m.log2cap, src_glob, slot, draws_out,                                     \
          m.table == nullptr ? m.size_out : nullptr);                                        \
  } while (0)
  if (policy == kRngSplitmix) {
    if (G == 8) SAL_SAMPLE(kRngSplitmix, 8);
    else if (G == 16) SAL_SAMPLE(kRngSplitmix, 16);
    else SAL_SAMPLE(kRngSplitmix, 32);
  } else {
    if (G == 8) SAL_SAMPLE(kRngPhilox, 8);
    else if (G == 16) SAL_SAMPLE(kRngPhilox, 16);
    else SAL_SAMPLE(kRngPhilox, 32);
  }
#undef SAL_SAMPLE
  return cudaGetLastError();
}

cudaError_t launch_keys_insert(const int64_t* keys, int64_t n, const IdMapDev& m,
                               int32_t* src_glob, int32_t* slot, int64_t* e_total,
                               cudaStream_t st) {
  int64_t grid = (n + 255) / 256;
  if (grid < 1) grid = 1;
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  keys_insert_kernel<<<(int)grid, 256, 0, st>>>(keys, n, m.table, m.log2cap, src_glob, slot,
                                                e_total);
  return cudaGetLastError();
}

cudaError_t launch_hop_relabel(const IdMapDev& m, const int64_t* e_total, int64_t max_edges,
                               const int64_t* size_old, int64_t* size_new,
                               const int32_t* src_glob, const int32_t* slot, int32_t* rank_of,
                               int32_t* src_local, void* scan_ws, cudaStream_t st,
                               bool ws_zeroed, const NextCount* next, bool defer_resolve) {
  ScanWs ws = carve_scan_ws(scan_ws, max_edges);
  cudaError_t err;
  if (!ws_zeroed) {
    err = cudaMemsetAsync(scan_ws, 0, scan_ws_bytes(max_edges), st);
    if (err != cudaSuccess) return err;
  }
  if (next == nullptr && !defer_resolve) {  // both passes in one launch
    flag_scan_kernel<true><<<scan_grid(max_edges), kScanThreads, 0, st>>>(
        m.table, slot, src_glob, e_total, size_old, size_new, rank_of, m.globals, ws, nullptr,
        src_local);
    return cudaGetLastError();
  }
  flag_scan_kernel<false><<<scan_grid(max_edges), kScanThreads, 0, st>>>(
      m.table, slot, src_glob, e_total, size_old, size_new, rank_of, m.globals, ws,
      defer_resolve ? const_cast<int32_t*>(slot) : nullptr, nullptr);
  err = cudaGetLastError();
  if (err != cudaSuccess || defer_resolve) return err;
  int64_t grid = (max_edges + 255) / 256;
  if (grid < 1) grid = 1;
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  // the next hop's count + scan rides in the same launch (its workspace is zeroed)
  CountJob cj;
  cj.indptr = next->g.indptr;
  cj.globals = m.globals;
  cj.n_dst = size_new;
  cj.fanout = next->fanout;
  cj.dst_indptr = next->dst_indptr;
  cj.e_total = next->e_total;
  cj.ws = carve_scan_ws(next->scan_ws, next->max_dst);
  const int cgrid = scan_grid(next->max_dst);
  resolve_count_kernel<<<(int)grid + cgrid, 256, 0, st>>>(m.table, slot, e_total, size_old,
                                                          rank_of, src_local, (int)grid, cj);
  return cudaGetLastError();
}

}  // namespace sal
