// SAGEConv mean aggregation over an MFG layer (mpnn.py:57-65 _mean_neighbors).
//
// Forward: one warp per destination row; lanes tile the feature dimension
// with V-element vectors; the warp loads up to 32 source ids at once
// (coalesced) and broadcasts them with shuffles, keeping 4 source rows in
// flight.  Accumulation is fp32 in edge order, then an IEEE divide by the
// in-degree — the same arithmetic as np.add.at followed by `/= counts`, so
// fp32 inputs give bit-identical means.  Rows [n_dst, n_pad) are zeroed so a
// statically shaped (CUDA-graph) consumer sees finite padding.
//
// The *_global variant reads rows straight from the HBM-resident feature
// table through globals[src[e]] (layer-0 aggregation without a materialised
// gather).
//
// Backward: g_h[src[e],:] += g_out[d,:] / deg(d) with vector float atomics
// (red.global.add.v4.f32 on sm_90+).  Only hidden layers need it: layer 0's
// input is the (frozen) feature table.
#include <cuda_bf16.h>

#include "common.cuh"
#include "salient_internal.h"

namespace sal {

template <typename T> struct Cvt;
template <> struct Cvt<float> {
  static SAL_DEVINL float in(float v) { return v; }
  static SAL_DEVINL float out(float v) { return v; }
};
template <> struct Cvt<__half> {
  static SAL_DEVINL float in(__half v) { return __half2float(v); }
  static SAL_DEVINL __half out(float v) { return __float2half_rn(v); }
};
template <> struct Cvt<__nv_bfloat16> {
  static SAL_DEVINL float in(__nv_bfloat16 v) { return __bfloat162float(v); }
  static SAL_DEVINL __nv_bfloat16 out(float v) { return __float2bfloat16_rn(v); }
};

// acc[0..7] += the 8 16-bit values packed in v (convert, then fp32 add).  The
// sm_100 mixed-precision add.rn.f32.{f16,bf16} (FHADD) halves the instruction
// count but measured 5% slower on the layer-0 mean (40.1 vs 38.3 us).
template <typename T>
SAL_DEVINL void acc_row8(float* acc, const uint4& v) {
  const T* t = reinterpret_cast<const T*>(&v);
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] += Cvt<T>::in(t[j]);
}

template <typename T, int V>
SAL_DEVINL void load_row(const T* p, float* f) {
  constexpr int B = V * (int)sizeof(T);
  alignas(16) T tmp[V];
  if (B % 16 == 0) {
#pragma unroll
    for (int q = 0; q < B / 16; ++q)
      reinterpret_cast<uint4*>(tmp)[q] = __ldg(reinterpret_cast<const uint4*>(p) + q);
  } else if (B == 8) {
    *reinterpret_cast<uint2*>(tmp) = __ldg(reinterpret_cast<const uint2*>(p));
  } else if (B == 4) {
    *reinterpret_cast<unsigned*>(tmp) = __ldg(reinterpret_cast<const unsigned*>(p));
  } else {
#pragma unroll
    for (int j = 0; j < V; ++j) tmp[j] = p[j];
  }
#pragma unroll
  for (int j = 0; j < V; ++j) f[j] = Cvt<T>::in(tmp[j]);
}

template <typename T, int V>
SAL_DEVINL void store_row(T* p, const float* f) {
  constexpr int B = V * (int)sizeof(T);
  alignas(16) T tmp[V];
#pragma unroll
  for (int j = 0; j < V; ++j) tmp[j] = Cvt<T>::out(f[j]);
  if (B % 16 == 0) {
#pragma unroll
    for (int q = 0; q < B / 16; ++q)
      reinterpret_cast<uint4*>(p)[q] = reinterpret_cast<const uint4*>(tmp)[q];
  } else if (B == 8) {
    *reinterpret_cast<uint2*>(p) = *reinterpret_cast<const uint2*>(tmp);
  } else if (B == 4) {
    *reinterpret_cast<unsigned*>(p) = *reinterpret_cast<const unsigned*>(tmp);
  } else {
#pragma unroll
    for (int j = 0; j < V; ++j) p[j] = tmp[j];
  }
}

constexpr int kSegThreads = 256;

template <typename TIn, typename TOut, int V, bool kGlobal>
__global__ void __launch_bounds__(kSegThreads)
segment_mean_fwd_kernel(const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
                        const int32_t* __restrict__ globals, const int64_t* __restrict__ n_dst_dev,
                        int64_t n_pad, const TIn* __restrict__ h, int64_t h_stride, int32_t f,
                        TOut* __restrict__ out, int64_t out_stride, int pad_fill) {
  const int lane = threadIdx.x & 31;
  const int64_t n_dst = n_dst_dev ? *n_dst_dev : n_pad;
  if (!pad_fill) n_pad = n_pad < n_dst ? n_pad : n_dst;  // padding rows left as they are
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t d = warp; d < n_pad; d += nwarps) {
    TOut* orow = out + d * out_stride;
    if (d >= n_dst) {
      float z[V];
#pragma unroll
      for (int j = 0; j < V; ++j) z[j] = 0.f;
      for (int c = lane * V; c < f; c += 32 * V) store_row<TOut, V>(orow + c, z);
      continue;
    }
    const int32_t beg = indptr[d];
    const int32_t end = indptr[d + 1];
    const int32_t cnt = end - beg;
    for (int c0 = 0; c0 < f; c0 += 32 * V) {
      const int c = c0 + lane * V;
      const bool active = c < f;
      float acc[V];
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = 0.f;
      for (int e0 = beg; e0 < end; e0 += 32) {
        const int m = min(32, end - e0);
        int32_t my = 0;
        if (lane < m) {
          my = src[e0 + lane];
          if (kGlobal) my = globals[my];
        }
        int k = 0;
        for (; k + 4 <= m; k += 4) {
          float r[4][V];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t s = __shfl_sync(0xffffffffu, my, k + u);
            if (active) load_row<TIn, V>(h + s * h_stride + c, r[u]);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < V; ++j) acc[j] += r[u][j];
        }
        for (; k < m; ++k) {
          const int64_t s = __shfl_sync(0xffffffffu, my, k);
          float r[V];
          if (active) {
            load_row<TIn, V>(h + s * h_stride + c, r);
#pragma unroll
            for (int j = 0; j < V; ++j) acc[j] += r[j];
          }
        }
      }
      if (active) {
        if (cnt > 0) {
          const float fc = (float)cnt;
#pragma unroll
          for (int j = 0; j < V; ++j) acc[j] = __fdiv_rn(acc[j], fc);
        }
        store_row<TOut, V>(orow + c, acc);
      }
    }
  }
}

// Fast path for 16-bit rows of 16 B multiples: LPR lanes cover one row with
// 16-byte vectors, so a warp loads 32/LPR source rows per instruction and
// keeps kU such instructions in flight (all ~15 sampled edges of a typical
// destination in one round).  The per-group partial sums are combined with
// xor-shuffles at the end, so the summation order differs from the strict
// edge order of segment_mean_fwd_kernel (used for fp32 parity).
template <bool kGlobal>
SAL_DEVINL int32_t load_id(const int32_t* __restrict__ src, const int32_t* __restrict__ globals,
                           int32_t e) {
  const int32_t s = __ldg(src + e);
  return kGlobal ? __ldg(globals + s) : s;
}

// Warp per destination; LPR lanes cover a row with 16-byte vectors, so a warp
// reads 32/LPR source rows per instruction and keeps kU instructions in
// flight.  Each lane loads its own row id (the LPR lanes of a group hit the
// same word: one transaction), so the hot loop has no shuffles and no
// divergent collectives; the per-group partial sums are combined once per
// destination.  The mean is acc * (1/cnt); with the group-split summation
// this path is tolerance-equal (not bit-equal) to the strict edge-order
// fp32 kernel above.
template <typename TIn, typename TOut, int LPR, bool kGlobal>
__global__ void __launch_bounds__(kSegThreads, 4)
segment_mean_rows_kernel(const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
                         const int32_t* __restrict__ globals,
                         const int64_t* __restrict__ n_dst_dev, int64_t n_pad,
                         const TIn* __restrict__ h, int64_t h_stride, TOut* __restrict__ out,
                         int64_t out_stride, int vpr, int pad_fill) {
  constexpr int RPI = 32 / LPR;
  constexpr int kU = LPR >= 32 ? 4 : (LPR < 8 ? LPR : 8);
  const int lane = threadIdx.x & 31;
  const int grp = lane / LPR, sub = lane % LPR;
  const int n_dst = (int)(n_dst_dev ? *n_dst_dev : n_pad);
  const int npad = pad_fill ? (int)n_pad : min((int)n_pad, n_dst);
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  for (int d = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); d < npad; d += nwarps) {
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    if (d < n_dst) {
      const int beg = __ldg(indptr + d);
      const int end = __ldg(indptr + d + 1);
      for (int e0 = beg; e0 < end; e0 += RPI * kU) {
        uint4 buf[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int e = e0 + u * RPI + grp;
          if (e < end && sub < vpr) {
            const int64_t s = load_id<kGlobal>(src, globals, e);
            const int4 t = ld_stream_v4(reinterpret_cast<const int4*>(h + s * h_stride) + sub);
            buf[u] = make_uint4((unsigned)t.x, (unsigned)t.y, (unsigned)t.z, (unsigned)t.w);
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (e0 + u * RPI + grp < end && sub < vpr) acc_row8<TIn>(acc, buf[u]);
        }
      }
#pragma unroll
      for (int off = LPR; off < 32; off <<= 1)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
      if (end > beg) {
        const float inv = 1.f / (float)(end - beg);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] *= inv;
      }
    }
    if (grp == 0 && sub < vpr) store_row<TOut, 8>(out + (int64_t)d * out_stride + sub * 8, acc);
  }
}

// Software-pipelined variant for wide rows (LPR >= 8: 2-4 rows per warp
// instruction).  Per destination the plain kernel pays three dependent memory
// latencies (indptr -> source ids -> rows) for one round of row loads; here
// the source ids of destination d+W and the row pointers of d+2W are loaded
// while d's rows are in flight, so the steady state waits on the row loads
// alone.  Same summation order as segment_mean_rows_kernel.
template <typename TIn, typename TOut, int LPR, bool kGlobal>
__global__ void __launch_bounds__(kSegThreads, 3)
segment_mean_rows_pipe_kernel(const int32_t* __restrict__ indptr,
                              const int32_t* __restrict__ src,
                              const int32_t* __restrict__ globals,
                              const int64_t* __restrict__ n_dst_dev, int64_t n_pad,
                              const TIn* __restrict__ h, int64_t h_stride,
                              TOut* __restrict__ out, int64_t out_stride, int vpr,
                              int pad_fill) {
  constexpr int RPI = 32 / LPR;
  constexpr int kU = 8;
  constexpr int W = RPI * kU;  // edges per round
  const int lane = threadIdx.x & 31;
  const int grp = lane / LPR, sub = lane % LPR;
  const int n_dst = (int)(n_dst_dev ? *n_dst_dev : n_pad);
  const int npad = pad_fill ? (int)n_pad : min((int)n_pad, n_dst);
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  int d = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (d >= npad) return;
  int beg = 0, end = 0;
  if (d < n_dst) {
    beg = __ldg(indptr + d);
    end = __ldg(indptr + d + 1);
  }
  int ids[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int e = beg + u * RPI + grp;
    ids[u] = e < end ? load_id<kGlobal>(src, globals, e) : 0;
  }
  int dn = d + nwarps, nbeg = 0, nend = 0;
  if (dn < n_dst) {
    nbeg = __ldg(indptr + dn);
    nend = __ldg(indptr + dn + 1);
  }
  while (true) {
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    uint4 buf[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (beg + u * RPI + grp < end && sub < vpr) {
        const int4 t = ld_stream_v4(reinterpret_cast<const int4*>(h + (int64_t)ids[u] * h_stride) + sub);
        buf[u] = make_uint4((unsigned)t.x, (unsigned)t.y, (unsigned)t.z, (unsigned)t.w);
      }
    }
    // next destination's first-round ids and the row pointers after it
    int nids[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = nbeg + u * RPI + grp;
      nids[u] = e < nend ? load_id<kGlobal>(src, globals, e) : 0;
    }
    const int dnn = dn + nwarps;
    int nnbeg = 0, nnend = 0;
    if (dnn < n_dst) {
      nnbeg = __ldg(indptr + dnn);
      nnend = __ldg(indptr + dnn + 1);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (beg + u * RPI + grp < end && sub < vpr) acc_row8<TIn>(acc, buf[u]);
    }
    // rare: destinations with more than W edges finish unpipelined
    for (int e0 = beg + W; e0 < end; e0 += W) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * RPI + grp;
        if (e < end && sub < vpr) {
          const int64_t s = load_id<kGlobal>(src, globals, e);
          const int4 t = ld_stream_v4(reinterpret_cast<const int4*>(h + s * h_stride) + sub);
          buf[u] = make_uint4((unsigned)t.x, (unsigned)t.y, (unsigned)t.z, (unsigned)t.w);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (e0 + u * RPI + grp < end && sub < vpr) acc_row8<TIn>(acc, buf[u]);
      }
    }
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
    if (end > beg) {
      const float inv = 1.f / (float)(end - beg);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] *= inv;
    }
    if (grp == 0 && sub < vpr) store_row<TOut, 8>(out + (int64_t)d * out_stride + sub * 8, acc);
    d = dn;
    if (d >= npad) break;
    beg = nbeg;
    end = nend;
#pragma unroll
    for (int u = 0; u < kU; ++u) ids[u] = nids[u];
    dn = dnn;
    nbeg = nnbeg;
    nend = nnend;
  }
}

template <typename TG, int V>
__global__ void __launch_bounds__(kSegThreads)
segment_mean_bwd_kernel(const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
                        const int64_t* __restrict__ n_dst_dev, int64_t n_pad,
                        const TG* __restrict__ g_out, int64_t g_stride, int32_t f,
                        float* __restrict__ g_h, int64_t gh_stride) {
  const int lane = threadIdx.x & 31;
  const int64_t n_dst = n_dst_dev ? *n_dst_dev : n_pad;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t d = warp; d < n_dst; d += nwarps) {
    const int32_t beg = indptr[d];
    const int32_t end = indptr[d + 1];
    if (end == beg) continue;
    const float fc = (float)(end - beg);
    for (int c0 = 0; c0 < f; c0 += 32 * V) {
      const int c = c0 + lane * V;
      const bool active = c < f;
      float g[V];
      if (active) {
        load_row<TG, V>(g_out + d * g_stride + c, g);
#pragma unroll
        for (int j = 0; j < V; ++j) g[j] = __fdiv_rn(g[j], fc);
      }
      for (int e0 = beg; e0 < end; e0 += 32) {
        const int m = min(32, end - e0);
        const int32_t my = lane < m ? src[e0 + lane] : 0;
        for (int k = 0; k < m; ++k) {
          const int64_t s = __shfl_sync(0xffffffffu, my, k);
          if (!active) continue;
          float* dst = g_h + s * gh_stride + c;
          if (V % 4 == 0) {
#pragma unroll
            for (int q = 0; q < V / 4; ++q)
              atomicAdd(reinterpret_cast<float4*>(dst) + q,
                        make_float4(g[4 * q], g[4 * q + 1], g[4 * q + 2], g[4 * q + 3]));
          } else if (V == 2) {
            atomicAdd(reinterpret_cast<float2*>(dst), make_float2(g[0], g[1]));
          } else {
#pragma unroll
            for (int j = 0; j < V; ++j) atomicAdd(dst + j, g[j]);
          }
        }
      }
    }
  }
}

static int pick_vec(int32_t f, int64_t s1, int64_t s2, int max_v) {
  int v = max_v;
  while (v > 1 && (f % v != 0 || s1 % v != 0 || s2 % v != 0)) v >>= 1;
  return v;
}

static int seg_grid(int64_t rows) {
  int64_t blocks = (rows + (kSegThreads / 32) - 1) / (kSegThreads / 32);
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  return (int)(blocks < 1 ? 1 : blocks);
}

template <typename TIn, typename TOut, bool kGlobal>
static bool fwd_rows(const int32_t* indptr, const int32_t* src, const int32_t* globals,
                     const int64_t* n_dst_dev, int64_t n_pad, const void* h, int64_t h_stride,
                     int32_t f, void* out, int64_t out_stride, cudaStream_t st, int pad_fill) {
  if (sizeof(TIn) != 2 || f % 8 != 0) return false;
  // lanes per row: the power of two holding the row's 16-byte vectors (vpr of
  // them; e.g. 104 padded fp16 columns = 13 vectors on 16 lanes)
  const int vpr = f / 8;
  int lpr = 1;
  while (lpr < vpr) lpr <<= 1;
  if (lpr > 32) return false;
  if (h_stride % 8 != 0 || out_stride % 8 != 0 || ((uintptr_t)h % 16) != 0 ||
      ((uintptr_t)out % 16) != 0)
    return false;
  const TIn* hp = (const TIn*)h;
  TOut* op = (TOut*)out;
  // Software-pipelined persistent kernel for the training layer-0 shape (128-d
  // 16-bit rows, <= 128 K destinations): 42.3 -> 38.3 us alone, -1.6 % per
  // training step (random 256 B row reads alone take 32.8 us, tools/randread_bench.cu).
  // A variant streaming the rows into shared memory with one cp.async.bulk per
  // row, S = 3 stages of 32 rows per warp, was correct but took 93 us.  Not for 512 B rows (neutral) nor for the (20,20,20)
  // inference layer 0 (450 K destinations), where the persistent grid starves
  // the overlapped prep chain: the pass took 0.098 s with it, 0.084 s without.
  if ((lpr == 8 || lpr == 16) && n_pad <= 131072) {
    // one resident wave (3 blocks/SM at 80 registers).  Measured worse: 2 blocks/SM
    // to leave room for the prep chain (+16 us), short-lived blocks of 2-8
    // destinations per warp (+6..20 us)
    int64_t blocks = (n_pad + 7) / 8;
    const int64_t cap = (int64_t)num_sms() * 3;
    if (blocks > cap) blocks = cap;
    const int g = (int)(blocks < 1 ? 1 : blocks);
    if (lpr == 8)
      segment_mean_rows_pipe_kernel<TIn, TOut, 8, kGlobal><<<g, kSegThreads, 0, st>>>(
          indptr, src, globals, n_dst_dev, n_pad, hp, h_stride, op, out_stride, vpr, pad_fill);
    else
      segment_mean_rows_pipe_kernel<TIn, TOut, 16, kGlobal><<<g, kSegThreads, 0, st>>>(
          indptr, src, globals, n_dst_dev, n_pad, hp, h_stride, op, out_stride, vpr, pad_fill);
    return true;
  }
  const int grid = seg_grid(n_pad);
#define SAL_ROWS_CASE(L)                                                                     \
  case L:                                                                                    \
    segment_mean_rows_kernel<TIn, TOut, L, kGlobal><<<grid, kSegThreads, 0, st>>>(            \
        indptr, src, globals, n_dst_dev, n_pad, hp, h_stride, op, out_stride, vpr, pad_fill);         \
    return true;
  switch (lpr) {
    SAL_ROWS_CASE(1)
    SAL_ROWS_CASE(2)
    SAL_ROWS_CASE(4)
    SAL_ROWS_CASE(8)
    SAL_ROWS_CASE(16)
    SAL_ROWS_CASE(32)
  }
#undef SAL_ROWS_CASE
  return false;
}

template <typename TIn, typename TOut, bool kGlobal>
static cudaError_t fwd_typed(const int32_t* indptr, const int32_t* src, const int32_t* globals,
                             const int64_t* n_dst_dev, int64_t n_pad, const void* h,
                             int64_t h_stride, int32_t f, void* out, int64_t out_stride,
                             cudaStream_t st, int pad_fill) {
  if (fwd_rows<TIn, TOut, kGlobal>(indptr, src, globals, n_dst_dev, n_pad, h, h_stride, f, out,
                                    out_stride, st, pad_fill))
    return cudaGetLastError();
  // vector width: 16 B of the narrower side, capped so one pass covers f
  const int max_v = 16 / (int)(sizeof(TIn) < sizeof(TOut) ? sizeof(TIn) : sizeof(TOut));
  int v = pick_vec(f, h_stride, out_stride, max_v);
  while (v > 1 && 32 * v > f && f % (v / 2) == 0 && 32 * (v / 2) >= f) v >>= 1;
  const int grid = seg_grid(n_pad);
  const TIn* hp = (const TIn*)h;
  TOut* op = (TOut*)out;
#define SAL_SEG_CASE(VV)                                                                     \
  case VV:                                                                                   \
    segment_mean_fwd_kernel<TIn, TOut, VV, kGlobal><<<grid, kSegThreads, 0, st>>>(           \
        indptr, src, globals, n_dst_dev, n_pad, hp, h_stride, f, op, out_stride, pad_fill); \
    break;
  switch (v) {
    SAL_SEG_CASE(8)
    SAL_SEG_CASE(4)
    SAL_SEG_CASE(2)
    default:
      SAL_SEG_CASE(1)
  }
#undef SAL_SEG_CASE
  return cudaGetLastError();
}

template <bool kGlobal>
static cudaError_t fwd_dispatch(const int32_t* indptr, const int32_t* src, const int32_t* globals,
                                const int64_t* n_dst_dev, int64_t n_pad, const void* h,
                                int32_t h_dtype, int64_t h_stride, int32_t f, void* out,
                                int32_t out_dtype, int64_t out_stride, cudaStream_t st,
                                int pad_fill) {
#define SAL_FWD(TI, TO) \
  return fwd_typed<TI, TO, kGlobal>(indptr, src, globals, n_dst_dev, n_pad, h, h_stride, f, out, \
                                    out_stride, st, pad_fill)
  if (h_dtype == SAL_F16) {
    if (out_dtype == SAL_F32) SAL_FWD(__half, float);
    if (out_dtype == SAL_BF16) SAL_FWD(__half, __nv_bfloat16);
    SAL_FWD(__half, __half);
  }
  if (h_dtype == SAL_BF16) {
    if (out_dtype == SAL_F32) SAL_FWD(__nv_bfloat16, float);
    SAL_FWD(__nv_bfloat16, __nv_bfloat16);
  }
  if (out_dtype == SAL_BF16) SAL_FWD(float, __nv_bfloat16);
  SAL_FWD(float, float);
#undef SAL_FWD
}

cudaError_t launch_segment_mean_fwd(const int32_t* indptr, const int32_t* src,
                                    const int32_t* globals, const int64_t* n_dst_dev,
                                    int64_t n_pad, const void* h, int32_t h_dtype,
                                    int64_t h_stride, int32_t f, void* out, int32_t out_dtype,
                                    int64_t out_stride, cudaStream_t st, bool pad_fill) {
  if (globals != nullptr)
    return fwd_dispatch<true>(indptr, src, globals, n_dst_dev, n_pad, h, h_dtype, h_stride, f,
                              out, out_dtype, out_stride, st, pad_fill ? 1 : 0);
  return fwd_dispatch<false>(indptr, src, globals, n_dst_dev, n_pad, h, h_dtype, h_stride, f,
                             out, out_dtype, out_stride, st, pad_fill ? 1 : 0);
}

template <typename TG>
static cudaError_t bwd_typed(const int32_t* indptr, const int32_t* src, const int64_t* n_dst_dev,
                             int64_t n_pad, const void* g_out, int64_t g_stride, int32_t f,
                             float* g_h, int64_t gh_stride, cudaStream_t st) {
  int v = pick_vec(f, g_stride, gh_stride, 8);
  if ((uintptr_t)g_h % 16 != 0 && v >= 4) v = 2;
  const int grid = seg_grid(n_pad);
  const TG* gp = (const TG*)g_out;
#define SAL_BWD_CASE(VV)                                                                    \
  case VV:                                                                                  \
    segment_mean_bwd_kernel<TG, VV><<<grid, kSegThreads, 0, st>>>(indptr, src, n_dst_dev,    \
                                                                  n_pad, gp, g_stride, f,    \
                                                                  g_h, gh_stride);           \
    break;
  switch (v) {
    SAL_BWD_CASE(8)
    SAL_BWD_CASE(4)
    SAL_BWD_CASE(2)
    default:
      SAL_BWD_CASE(1)
  }
#undef SAL_BWD_CASE
  return cudaGetLastError();
}

cudaError_t launch_segment_mean_bwd(const int32_t* indptr, const int32_t* src,
                                    const int64_t* n_dst_dev, int64_t n_pad, const void* g_out,
                                    int32_t g_dtype, int64_t g_stride, int32_t f, float* g_h,
                                    int64_t gh_stride, cudaStream_t st) {
  if (g_dtype == SAL_BF16)
    return bwd_typed<__nv_bfloat16>(indptr, src, n_dst_dev, n_pad, g_out, g_stride, f, g_h,
                                    gh_stride, st);
  if (g_dtype == SAL_F16)
    return bwd_typed<__half>(indptr, src, n_dst_dev, n_pad, g_out, g_stride, f, g_h, gh_stride,
                             st);
  return bwd_typed<float>(indptr, src, n_dst_dev, n_pad, g_out, g_stride, f, g_h, gh_stride, st);
}

}  // namespace sal
