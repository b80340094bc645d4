// Fused last hop: sample + layer-0 mean + self row, one warp per destination.
//
// In training and sampled inference the last hop of the MFG is consumed only
// by the layer-0 mean (mpnn.py:57-65), and its relabel is never needed (the
// rows are read straight from the feature table by global id).  So instead of
// materialising the hop (sample_insert_kernel -> src_glob, hop.cu) and reading
// it back in the mean (segment_mean_rows_pipe_kernel, segment.cu), one kernel
//   * draws the destination's fanout positions (the same sequential rejection
//     semantics as _kernels.py:102-147, 32 draws per round, accepted in draw
//     order, so the sample is bit-identical to sample_insert_kernel's),
//   * reads the sampled global ids from `indices`,
//   * sums their feature rows (fp32, the pipe kernel's exact summation order),
//   * writes the bf16 mean and the destination's own row (the layer-0 "cat"
//     buffer [mean | self]; the self row replaces gather_rows_warp_kernel).
// Per destination the chain is globals -> indptr -> draws -> indices -> rows;
// the loop is software-pipelined four deep (the globals of d+3W, the indptr of
// d+2W and the draws + index loads of d+W are issued while d's rows are in
// flight), so the steady state waits on the row loads alone.
//
// Reference: _kernels.py:150-185 (hop_kernel), :102-147 (_sample_positions),
// mpnn.py:57-65 (_mean_neighbors), prep.py:153-171 (slice_features).
#include <cuda_bf16.h>

#include <cstdlib>
#include <type_traits>


#include "common.cuh"
#include "salient_internal.h"
#include "sampling.cuh"

namespace sal {

template <typename T> struct CvtS;
template <> struct CvtS<__half> {
  static SAL_DEVINL float in(__half v) { return __half2float(v); }
  static SAL_DEVINL __half out(float v) { return __float2half_rn(v); }
};
template <> struct CvtS<__nv_bfloat16> {
  static SAL_DEVINL float in(__nv_bfloat16 v) { return __bfloat162float(v); }
  static SAL_DEVINL __nv_bfloat16 out(float v) { return __float2bfloat16_rn(v); }
};

// acc[0..7] += the 8 halves packed in v.  fp16 takes the sm_100 mixed-precision
// add (add.rn.f32.f16 -> FHADD, upper halves selected in the operand): one
// instruction per element, and bit-identical to convert-then-add (the fp16 ->
// fp32 conversion is exact).
SAL_DEVINL void fhadd2(float& a0, float& a1, unsigned w) {
  asm("{\n\t.reg .f16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
      "add.rn.f32.f16 %0, lo, %0;\n\tadd.rn.f32.f16 %1, hi, %1;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "r"(w));
}

template <typename TIn>
SAL_DEVINL void acc8(float* acc, const uint4& v) {
  if constexpr (sizeof(TIn) == 2 && std::is_same<TIn, __half>::value) {
    fhadd2(acc[0], acc[1], v.x);
    fhadd2(acc[2], acc[3], v.y);
    fhadd2(acc[4], acc[5], v.z);
    fhadd2(acc[6], acc[7], v.w);
  } else {
    const TIn* t = reinterpret_cast<const TIn*>(&v);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += CvtS<TIn>::in(t[j]);
  }
}

template <typename TOut>
SAL_DEVINL uint4 pack8(const float* f) {
  alignas(16) TOut t[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) t[j] = CvtS<TOut>::out(f[j]);
  return *reinterpret_cast<const uint4*>(t);
}

constexpr int kSmThreads = 128;   // 4 warps: finer shared-memory granularity per SM

// 1/c for c = 0..32, the correctly rounded fp32 values 1.f / (float)c gives
// (generated with numpy float32 division; hex literals are exact)
__constant__ float c_inv[33] = {
    0.0f, 0x1.0000000000000p+0f, 0x1.0000000000000p-1f, 0x1.5555560000000p-2f, 0x1.0000000000000p-2f, 0x1.99999a0000000p-3f, 0x1.5555560000000p-3f, 0x1.24924a0000000p-3f, 0x1.0000000000000p-3f, 0x1.c71c720000000p-4f, 0x1.99999a0000000p-4f, 0x1.745d180000000p-4f, 0x1.5555560000000p-4f, 0x1.3b13b20000000p-4f, 0x1.24924a0000000p-4f, 0x1.1111120000000p-4f, 0x1.0000000000000p-4f, 0x1.e1e1e20000000p-5f, 0x1.c71c720000000p-5f, 0x1.af286c0000000p-5f, 0x1.99999a0000000p-5f, 0x1.8618620000000p-5f, 0x1.745d180000000p-5f, 0x1.642c860000000p-5f, 0x1.5555560000000p-5f, 0x1.47ae140000000p-5f, 0x1.3b13b20000000p-5f, 0x1.2f684c0000000p-5f, 0x1.24924a0000000p-5f, 0x1.1a7b960000000p-5f, 0x1.1111120000000p-5f, 0x1.0842100000000p-5f, 0x1.0000000000000p-5f};

// One destination's sample: lane j < cnt receives the global id of accepted
// edge j in `sid` (a predicated load: the value is consumed an iteration later).
// deg <= fanout takes the whole row in CSR order (_kernels.py:168-174).
// recip = floor((2^64-1)/deg) (splitmix policy, deg > fanout, recip_u32).
template <int kPolicy>
SAL_DEVINL int sample_dst(const int32_t* __restrict__ indices, int d, int64_t lo, int64_t deg,
                          int32_t fanout, uint64_t prefix, uint2 pkey, uint32_t hop,
                          uint32_t batch, uint64_t recip, int32_t* accepted, int lane,
                          int32_t& sid) {
  if (deg <= fanout) {
    ldp_s32(sid, indices + lo + lane, lane < deg);
    return (int)deg;
  }
  const unsigned lt = (1u << lane) - 1u;
  const uint64_t key = mix64(prefix ^ (uint64_t)d);  // _kernels.py:167
  const uint32_t udeg = (uint32_t)deg;
  int acc = 0;
  uint32_t ctr = 0;
  while (acc < fanout) {
    const uint32_t pos =
        draw_position<kPolicy>(key, pkey, ctr + lane, (uint32_t)d, hop, batch, udeg, recip);
    bool hit = false;
    for (int j = 0; j < acc; ++j) hit |= ((uint32_t)accepted[j] == pos);
    const unsigned peers = __match_any_sync(0xffffffffu, pos);
    const bool fresh = !hit && (peers & lt) == 0;
    const unsigned fm = __ballot_sync(0xffffffffu, fresh);
    const int rank = __popc(fm & lt);
    if (fresh && acc + rank < fanout) accepted[acc + rank] = (int32_t)pos;
    acc += min(__popc(fm), fanout - acc);
    ctr += 32;
    __syncwarp();
  }
  const int p = lane < fanout ? accepted[lane] : 0;
  ldp_s32(sid, indices + lo + p, lane < fanout);
  __syncwarp();  // `accepted` is reused by the next destination
  return fanout;
}

// 16 bytes global -> shared, L2 policy evict_first: every feature row is read once per
// batch, so it should not push the step's reused tensors (the layer-0 input this
// kernel writes, the backward's gradients) out of L2
// pred false: the 16 bytes are zero-filled (src-size 0, nothing is read), so the
// consumer adds +0 for rows past the count without selecting
SAL_DEVINL void cp_async16(uint32_t smem, const void* gmem, bool pred, uint64_t policy) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(smem),
               "l"(gmem), "r"(pred ? 16 : 0), "l"(policy)
               : "memory");
}
// pred false: no copy at all (the self row's slot is shared by both lane groups)
SAL_DEVINL void cp_async16_if(uint32_t smem, const void* gmem, bool pred, uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %3;\n\t}" ::"r"(smem),
      "l"(gmem), "r"((int)pred), "l"(policy)
      : "memory");
}
SAL_DEVINL void st_v4_policy(void* p, uint4 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(policy)
               : "memory");
}
SAL_DEVINL uint64_t l2_evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SAL_DEVINL uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SAL_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
SAL_DEVINL void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Shared-memory stage of one destination: kRows sampled rows + its own row,
// 256 B each (16 lanes x 16 B; narrower tables leave the tail lanes idle).
template <int kRows>
__host__ __device__ constexpr int stage_bytes() { return (kRows + 1) * 256; }

// Warp per destination, five destinations in flight per warp:
//   d4: global id load            d3: row-pointer loads
//   d2: draws + sampled-id load   d1: rows -> shared memory (cp.async, 2 stages)
//   d : rows consumed from shared memory, mean + self row written
// No register holds a row, so the warp carries one destination's rows in flight
// while it accumulates the previous one, and every load result is consumed an
// iteration after it was issued.
template <int kPolicy, typename TIn, typename TOut, int kRows, bool kFull>
__global__ void __launch_bounds__(kSmThreads)
sample_mean_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                   const int32_t* __restrict__ globals, const int64_t* __restrict__ n_dst_ptr,
                   int32_t fanout, HopKey hk, const BatchDesc* __restrict__ desc,
                   const TIn* __restrict__ table, int64_t t_stride, int vpr,
                   TOut* __restrict__ out, int64_t out_stride, int64_t self_off,
                   int64_t* __restrict__ size_unknown, ulonglong2* __restrict__ reset_table,
                   int64_t table_pairs, uint4* __restrict__ reset_scan, int64_t scan_vecs,
                   ResolveJob resolve) {
  extern __shared__ __align__(16) unsigned char sm_stage[];
  if (resolve.src_local != nullptr)   // hop L-2's local ids (sal_sample_aggregate)
    resolve_words(resolve, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                  (int64_t)gridDim.x * blockDim.x);
  if (reset_table != nullptr) {
    // the id table and scan workspace of hops 0..L-2 are no longer read: leave them
    // reset for this workspace's next batch (sal_mfg_plan.reset_in_aggregate)
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t; i < table_pairs; i += nt) reset_table[i] = make_ulonglong2(~0ull, ~0ull);
    for (int64_t i = t; i < scan_vecs; i += nt) reset_scan[i] = make_uint4(0, 0, 0, 0);
  }
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int grp = lane >> 4, sub = lane & 15;
  const int n = (int)*n_dst_ptr;
  const int W = (int)((gridDim.x * blockDim.x) >> 5);
  uint64_t prefix = hk.prefix;
  uint32_t batch = hk.batch;
  if (desc != nullptr) {
    batch = (uint32_t)desc->batch_id;
    if (hk.derive) prefix = hop_key_prefix(hk.global_seed, (uint64_t)desc->batch_id, hk.hop);
  }
  const uint2 pkey = make_uint2((uint32_t)hk.global_seed, (uint32_t)(hk.global_seed >> 32));
  __shared__ int32_t sh_acc[kSmThreads / 32][32];
  int32_t* accepted = sh_acc[warp];
  if (size_unknown != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *size_unknown = -1;
  const bool vlane = kFull || sub < vpr;   // kFull: 256-byte rows, every lane busy
  const bool do_self = grp == 1 && vlane && self_off >= 0;
  const char* tbase = reinterpret_cast<const char*>(table) + sub * 16;
  const int64_t tbytes = t_stride * (int64_t)sizeof(TIn);
  // this warp's two stages; lane (grp, sub) owns bytes [sub*16, +16) of the rows
  // e = 2u + grp (and of the self row): it copies and reads only its own slots
  const uint32_t st0 = (uint32_t)__cvta_generic_to_shared(sm_stage) +
                       (uint32_t)(warp * 2 * stage_bytes<kRows>()) + sub * 16;
  const unsigned char* lst0 = sm_stage + warp * 2 * stage_bytes<kRows>() + sub * 16;

  int d = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (d >= n) return;

  const uint64_t pol = l2_evict_first_policy();
  // the [mean | self] rows are read again by the next step's layer-0 GEMM
  const uint64_t pol_out = l2_evict_last_policy();
  auto issue_rows = [&](int stage, int32_t sid, int cnt, int32_t v) {
    const uint32_t sb = st0 + stage * stage_bytes<kRows>();
#pragma unroll
    for (int u = 0; u < kRows / 2; ++u) {
      const int e = u * 2 + grp;
      const int id = __shfl_sync(0xffffffffu, sid, e);
      cp_async16(sb + e * 256, tbase + (int64_t)id * tbytes, e < cnt && vlane, pol);
    }
    cp_async16_if(sb + kRows * 256, tbase + (int64_t)v * tbytes, do_self, pol);
    cp_async_commit();
  };
  auto recip_of = [&](int64_t lo, int64_t hi) -> uint64_t {
    return (kPolicy == kRngSplitmix && hi - lo > fanout) ? recip_u32((uint32_t)(hi - lo)) : 0ull;
  };

  // prologue: d sampled + its rows issued, d1 sampled, d2's row pointers, d3's id
  int32_t vd = __ldg(globals + d);
  int32_t sid = 0;
  int cnt;
  {
    const int64_t lo = ld_i64(indptr + vd), hi = ld_i64(indptr + vd + 1);
    cnt = sample_dst<kPolicy>(indices, d, lo, hi - lo, fanout, prefix, pkey, hk.hop, batch,
                              recip_of(lo, hi), accepted, lane, sid);
  }
  issue_rows(0, sid, cnt, vd);
  int d1 = d + W;
  int32_t v1 = 0, sid1 = 0;
  int cnt1 = 0;
  if (d1 < n) {
    v1 = __ldg(globals + d1);
    const int64_t lo = ld_i64(indptr + v1), hi = ld_i64(indptr + v1 + 1);
    cnt1 = sample_dst<kPolicy>(indices, d1, lo, hi - lo, fanout, prefix, pkey, hk.hop, batch,
                               recip_of(lo, hi), accepted, lane, sid1);
  }
  int d2 = d1 + W;
  int32_t v2 = 0;
  int64_t lo2 = 0, hi2 = 0;
  if (d2 < n) {
    v2 = __ldg(globals + d2);
    lo2 = ld_i64(indptr + v2);
    hi2 = ld_i64(indptr + v2 + 1);
  }
  int d3 = d2 + W;
  int32_t v3 = 0;
  ldp_s32(v3, globals + d3, d3 < n);

  for (int it = 0;; ++it) {
    const int cur = it & 1;
    // d1's rows into the other stage (its sample was loaded last iteration)
    if (d1 < n) issue_rows(cur ^ 1, sid1, cnt1, v1);
    else cp_async_commit();   // keep one group per iteration
    // d4's id, d3's row pointers, d2's sample
    const int d4 = d3 + W;
    int32_t v4 = 0;
    ldp_s32(v4, globals + d4, d4 < n);
    int64_t lo3 = 0, hi3 = 0;
    ldp_s64(lo3, indptr + v3, d3 < n);
    ldp_s64(hi3, indptr + v3 + 1, d3 < n);
    int cnt2 = 0;
    int32_t sid2 = 0;
    if (d2 < n)
      cnt2 = sample_dst<kPolicy>(indices, d2, lo2, hi2 - lo2, fanout, prefix, pkey, hk.hop,
                                 batch, recip_of(lo2, hi2), accepted, lane, sid2);
    // consume d (stage cur): the pipe kernel's summation order (group partial sums
    // in edge order, one xor-shuffle), acc * (1/cnt)
    cp_async_wait1();
    const unsigned char* ls = lst0 + cur * stage_bytes<kRows>();
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    // branch-free: rows past the count were zero-filled and add +0 (acc starts at +0
    // and so is never -0, which makes the add an exact no-op)
#pragma unroll
    for (int u = 0; u < kRows / 2; ++u)
      acc8<TIn>(acc, *reinterpret_cast<const uint4*>(ls + (u * 2 + grp) * 256));
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], 16);
    if (cnt > 0) {
      const float inv = c_inv[cnt];   // == 1.f / (float)cnt
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] *= inv;
    }
    TOut* orow = out + (int64_t)d * out_stride;
    if (vlane) {
      if (grp == 0) {
        st_v4_policy(orow + sub * 8, pack8<TOut>(acc), pol_out);
      } else if (self_off >= 0) {
        // converted, not added to 0 (that would turn -0 into +0)
        const uint4 raw = *reinterpret_cast<const uint4*>(ls + kRows * 256);
        const TIn* t = reinterpret_cast<const TIn*>(&raw);
        float sv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) sv[j] = CvtS<TIn>::in(t[j]);
        st_v4_policy(orow + self_off + sub * 8, pack8<TOut>(sv), pol_out);
      }
    }
    if (d1 >= n) break;
    d = d1;
    cnt = cnt1;
    d1 = d2;
    v1 = v2;
    sid1 = sid2;
    cnt1 = cnt2;
    d2 = d3;
    v2 = v3;
    lo2 = lo3;
    hi2 = hi3;
    d3 = d4;
    v3 = v4;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int kRows>
static int sample_mean_bps() {
  // resident blocks per SM: the shared-memory stages (8 warps x 2 stages) bound it
  const int per_block = (kSmThreads / 32) * 2 * stage_bytes<kRows>();
  const int b = (227 * 1024) / (per_block + 1024);
  return b < 1 ? 1 : (b > 8 ? 8 : b);
}

template <int kPolicy, typename TO, int kRows>
static cudaError_t launch_sm(const GraphDev& g, const int32_t* globals, const int64_t* n_dst,
                             int64_t max_dst, int32_t fanout, HopKey hk, const BatchDesc* desc,
                             const void* table, int64_t t_stride, int vpr, void* out,
                             int64_t out_stride, int64_t self_off, int64_t* size_unknown,
                             int bps_cap, unsigned long long* reset_table, int64_t table_words,
                             void* reset_scan, int64_t scan_bytes, const ResolveJob& resolve,
                             cudaStream_t st) {
  const int smem = (kSmThreads / 32) * 2 * stage_bytes<kRows>();
  auto k = vpr == 16 ? sample_mean_kernel<kPolicy, __half, TO, kRows, true>
                     : sample_mean_kernel<kPolicy, __half, TO, kRows, false>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int64_t grid = (max_dst + kSmThreads / 32 - 1) / (kSmThreads / 32);
  int bps = sample_mean_bps<kRows>();
  if (bps_cap > 0 && bps_cap < bps) bps = bps_cap;
  if (const char* e = getenv("SAL_SAMPLE_MEAN_BPS")) {   // A/B knob (tools/)
    const int b = atoi(e);
    if (b >= 1 && b < bps) bps = b;
  }
  int64_t cap = (int64_t)num_sms() * bps;
  // A/B knob (tools/): SAL_SAMPLE_MEAN_DPW = destinations per warp (a non-persistent
  // grid of short-lived blocks the scheduler can interleave with other kernels)
  if (const char* e = getenv("SAL_SAMPLE_MEAN_DPW")) {
    const int dpw = atoi(e);
    if (dpw > 0) cap = (max_dst + (int64_t)dpw * (kSmThreads / 32) - 1) / ((int64_t)dpw * (kSmThreads / 32));
  }
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  k<<<(int)grid, kSmThreads, smem, st>>>(g.indptr, g.indices, globals, n_dst, fanout, hk, desc,
                                         (const __half*)table, t_stride, vpr, (TO*)out,
                                         out_stride, self_off, size_unknown,
                                         (ulonglong2*)reset_table, table_words / 2,
                                         (uint4*)reset_scan, reset_table ? scan_bytes / 16 : 0,
                                         resolve);
  return cudaGetLastError();
}

cudaError_t launch_sample_mean(const GraphDev& g, const int32_t* globals, const int64_t* n_dst,
                               int64_t max_dst, int32_t fanout, HopKey hk, const BatchDesc* desc,
                               int32_t policy, const void* table, int64_t t_stride, int32_t cols,
                               void* out, int32_t out_dtype, int64_t out_stride, int64_t self_off,
                               int64_t* size_unknown, int bps_cap, unsigned long long* reset_table,
                               int64_t table_words, void* reset_scan, int64_t scan_bytes,
                               const ResolveJob& resolve, cudaStream_t st) {
  const int vpr = cols * 2 / 16;
#define SAL_SM(P, TO, R)                                                                   \
  return launch_sm<P, TO, R>(g, globals, n_dst, max_dst, fanout, hk, desc, table, t_stride, \
                             vpr, out, out_stride, self_off, size_unknown, bps_cap, reset_table, \
                             table_words, reset_scan, scan_bytes, resolve, st)
// stage rows: the smallest of 8 / 16 / 20 / 32 that holds the fanout (shared memory per
// warp bounds the resident warps, and with them the rows in flight per SM)
#define SAL_SM_R(P, TO)                 \
  if (fanout <= 8) {                    \
    SAL_SM(P, TO, 8);                   \
  } else if (fanout <= 16) {            \
    SAL_SM(P, TO, 16);                  \
  } else if (fanout <= 20) {            \
    SAL_SM(P, TO, 20);                  \
  } else {                              \
    SAL_SM(P, TO, 32);                  \
  }
  if (out_dtype == SAL_BF16) {
    if (policy == kRngSplitmix) { SAL_SM_R(kRngSplitmix, __nv_bfloat16); }
    else { SAL_SM_R(kRngPhilox, __nv_bfloat16); }
  } else {
    if (policy == kRngSplitmix) { SAL_SM_R(kRngSplitmix, __half); }
    else { SAL_SM_R(kRngPhilox, __half); }
  }
#undef SAL_SM_R
#undef SAL_SM
}

}  // namespace sal
