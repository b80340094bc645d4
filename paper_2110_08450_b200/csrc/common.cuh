// Shared device helpers for the SALIENT batch-preparation kernels (sm_100a).
//
// Conventions used by every kernel in this library:
//   * node ids on device are int32 (graphs up to 2^31-1 nodes); the CSR row
//     pointer is int64 (papers100M-shape graphs hold 1.6e9 slots);
//   * per-batch sizes live in device memory (int64) so consecutive hops chain
//     without a host sync and a whole batch can be captured in a CUDA graph;
//   * persistent grids are sized in multiples of the SM count (148 on B200)
//     and walk their work with grid-stride loops over the device-side count.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define SAL_DEVINL __device__ __forceinline__

namespace sal {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// splitmix64 (reference: pkg/src/mfgprep/rng.py:16-35, _kernels.py:30-39)
// ---------------------------------------------------------------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

SAL_DEVINL uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Row range [*b, *e) of part k of nparts over `rows` rows whose first *m_dev
// are live (static shapes pad to `rows`): the live rows are cut at multiples
// of 64, the last part runs to `rows`.  mean_bwd_t and the tcgen05 weight
// gradient agree on it, so part k of one can start as part k of the other ends
// (inner cuts never pass the 64-row chunk holding the last live row, so a
// weight-gradient chunk never reads rows a later mean_bwd_t part writes).
SAL_DEVINL void part_rows(const int64_t* m_dev, int64_t rows, int k, int nparts, int* b, int* e) {
  const int64_t mt = m_dev ? (*m_dev < rows ? *m_dev : rows) : rows;
  const int64_t cap = (mt + 63) / 64 * 64 < rows ? (mt + 63) / 64 * 64 : rows;
  auto bound = [&](int j) -> int {
    if (j <= 0) return 0;
    if (j >= nparts) return (int)rows;
    int64_t x = (mt * j + nparts - 1) / nparts;
    x = (x + 63) / 64 * 64;
    return (int)(x < cap ? x : cap);
  };
  *b = bound(k);
  *e = bound(k + 1);
}

// Dropout stream of the training step (relu_dropout_fwd_kernel and the fused
// tcgen05 epilogue must agree).  General p: 16 bits of uniform per element,
// two splitmix64 draws per group of 8 elements.  p == 0.5 exactly (the
// paper's setting): one keep bit per element, 64 elements per draw —
// keep(e) = bit (e % 64) of dropout_word64(key, e / 64), e = row * cols + col.
SAL_DEVINL uint64_t dropout_word64(uint64_t key_base, uint64_t e64) {
  return mix64(key_base ^ 0x6A09E667F3BCC909ull ^ (e64 * 0xD1B54A32D192ED03ull));
}

__host__ __device__ inline uint64_t mix64_hd(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// HopStream.key_prefix (sampler.py:241-247).
__host__ __device__ inline uint64_t hop_key_prefix(uint64_t seed, uint64_t batch,
                                                   uint64_t hop) {
  uint64_t k = mix64_hd(seed ^ kGolden);
  k = mix64_hd(k ^ batch);
  return mix64_hd(k ^ (hop + 0x51EDull));
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (north-star RNG policy; keyed on (seed, epoch|batch, hop, node))
// ---------------------------------------------------------------------------
SAL_DEVINL uint4 philox4x32_10(uint4 ctr, uint2 key) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, ctr.x);
    const uint32_t lo0 = 0xD2511F53u * ctr.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, ctr.z);
    const uint32_t lo1 = 0xCD9E8D57u * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += 0x9E3779B9u;
    key.y += 0xBB67AE85u;
  }
  return ctr;
}

// ---------------------------------------------------------------------------
// warp / block scans
// ---------------------------------------------------------------------------
template <typename T>
SAL_DEVINL T warp_inclusive_scan(T v, int lane) {
#pragma unroll
  for (int o = 1; o < kWarp; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

template <typename T>
SAL_DEVINL T warp_reduce_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exclusive block scan of one value per thread. `smem` needs >= nwarps+1 slots.
// Returns the exclusive prefix; *total receives the block sum.
template <typename T, int kThreads>
SAL_DEVINL T block_exclusive_scan(T v, T* smem, T* total) {
  constexpr int kWarps = kThreads / kWarp;
  const int lane = threadIdx.x & (kWarp - 1);
  const int warp = threadIdx.x >> 5;
  T inc = warp_inclusive_scan(v, lane);
  if (lane == kWarp - 1) smem[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < kWarps ? smem[lane] : T(0);
    T wi = warp_inclusive_scan(w, lane);
    if (lane < kWarps) smem[lane] = wi - w;
    if (lane == kWarps - 1) smem[kWarps] = wi;
  }
  __syncthreads();
  T out = smem[warp] + inc - v;
  *total = smem[kWarps];
  __syncthreads();
  return out;
}

// ---------------------------------------------------------------------------
// Decoupled look-back (single-pass device-wide scan).  Tile status words pack
// a 2-bit flag in the top bits and a 62-bit value.  The status array and the
// dynamic tile counter are zeroed by the host before each launch (one
// cudaMemsetAsync of the scan workspace).
// ---------------------------------------------------------------------------
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kFlagRanks = 1ull << 61;  // flag_scan_kernel<true>: the tile's ranks are written
constexpr uint64_t kValMask = (1ull << 61) - 1;

struct ScanWs {
  unsigned long long* status;  // [max_tiles]
  unsigned int* tile_counter;  // [1]
};

// Called by all threads of the block after the block aggregate is known.
// Returns the exclusive prefix of this tile (same value in all threads).
SAL_DEVINL uint64_t lookback_prefix(ScanWs ws, int tile, uint64_t agg, uint64_t* sh) {
  if (threadIdx.x < kWarp) {
    const int lane = threadIdx.x;
    if (tile == 0) {
      if (lane == 0) {
        atomicExch(&ws.status[0], (unsigned long long)(kFlagInc | agg));
        *sh = 0;
      }
    } else {
      if (lane == 0) atomicExch(&ws.status[tile], (unsigned long long)(kFlagAgg | agg));
      uint64_t prefix = 0;
      int base = tile - 1;
      while (true) {
        // each lane inspects one predecessor, lane 0 the nearest
        const int t = base - lane;
        uint64_t s;
        if (t >= 0) {
          do {
            s = *((volatile unsigned long long*)&ws.status[t]);
          } while ((s >> 62) == 0);
        } else {
          s = kFlagInc;  // virtual inclusive zero before tile 0
        }
        const unsigned inc_mask = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        const int first_inc = inc_mask ? __ffs(inc_mask) - 1 : kWarp;
        uint64_t v = (lane <= first_inc) ? (s & kValMask) : 0;
        v = warp_reduce_sum(v);
        prefix += v;
        if (inc_mask) break;
        base -= kWarp;
      }
      if (lane == 0) {
        __threadfence();
        atomicExch(&ws.status[tile], (unsigned long long)(kFlagInc | (prefix + agg)));
        *sh = prefix;
      }
    }
  }
  __syncthreads();
  return *sh;
}

SAL_DEVINL int grab_tile(ScanWs ws, int* sh) {
  if (threadIdx.x == 0) *sh = (int)atomicAdd(ws.tile_counter, 1u);
  __syncthreads();
  return *sh;
}

// ---------------------------------------------------------------------------
// cache-hinted memory helpers
// ---------------------------------------------------------------------------
SAL_DEVINL int4 ld_stream_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

SAL_DEVINL void st_stream_v4(int4* p, int4 v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w));
}

SAL_DEVINL int64_t ld_i64(const int64_t* p) { return __ldg((const long long*)p); }

// Predicated loads into registers the caller already holds ("+" operands): a
// load guarded by an `if` otherwise lands in a temporary and is copied into the
// live register right away, and that copy waits for the load — which serialises
// a software pipeline that means to consume the value an iteration later.
SAL_DEVINL void ldp_v4_stream(uint4& r, const void* p, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
      : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
      : "l"(p), "r"((int)pred));
}
SAL_DEVINL void ldp_s32(int32_t& r, const void* p, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.s32 %0, [%1];\n\t}"
      : "+r"(r)
      : "l"(p), "r"((int)pred));
}
SAL_DEVINL void ldp_s64(int64_t& r, const void* p, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.s64 %0, [%1];\n\t}"
      : "+l"(r)
      : "l"(p), "r"((int)pred));
}

}  // namespace sal
