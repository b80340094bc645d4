// Fused kernels of the GraphSAGE training step.
//
// Activation layout ("cat"): the input of layer i is a [rows, 2f] buffer whose
// right half holds h_i and whose left half, for the first n_pad destination
// rows, receives mean_i — so each SAGEConv is ONE GEMM  [mean | h_dst] @
// [W_neigh | W_self]^T, and its backward is one weight-gradient GEMM plus
// one input-gradient GEMM.
//
//   plan_next       device epoch cursor -> sal_batch_desc (one captured CUDA
//                   graph prepares a new batch on every replay)
//   relu_dropout    y = relu(x) * keep / (1-p) into the next cat buffer; one
//                   bit per element records (x > 0 && keep)
//   lsm_nll         log_softmax + NLL (labels < 0 ignored) fused with its
//                   gradient (softmax - onehot) / count
//   transpose_*     per-batch reverse adjacency of an MFG layer (src -> dsts),
//                   built on the prep stream
//   mean_bwd_t      input gradient of a layer, gathered per source row:
//                   dz_prev[s] = mask(s) * scale * (dh_dst[s] + sum_{d: s in N(d)}
//                   dmean[d] / deg(d)) — no atomics on the feature rows, no
//                   zero-fill, relu/dropout backward fused
//   adam            fused Adam over the flat fp32 parameters + bf16 shadow refresh
//   step_tail       per-step bookkeeping (loss log, counters) in one launch
#include <cuda_bf16.h>

#include "common.cuh"
#include "salient_internal.h"

namespace sal {

// ---------------------------------------------------------------------------
__global__ void plan_next_kernel(const int64_t* __restrict__ desc_all, int64_t n_steps,
                                 int64_t* __restrict__ cursor, BatchDesc* __restrict__ out) {
  const int64_t c = *cursor;
  if (c < n_steps) {
    out->batch_id = desc_all[3 * c + 0];
    out->seed_offset = desc_all[3 * c + 1];
    out->n_seeds = desc_all[3 * c + 2];
  } else {
    out->batch_id = -1;
    out->seed_offset = 0;
    out->n_seeds = 0;
  }
  *cursor = c + 1;
}

// ---------------------------------------------------------------------------
template <typename T> struct F;
template <> struct F<float> {
  static SAL_DEVINL float in(float v) { return v; }
  static SAL_DEVINL float out(float v) { return v; }
};
template <> struct F<__nv_bfloat16> {
  static SAL_DEVINL float in(__nv_bfloat16 v) { return __bfloat162float(v); }
  static SAL_DEVINL __nv_bfloat16 out(float v) { return __float2bfloat16_rn(v); }
};
template <> struct F<__half> {
  static SAL_DEVINL float in(__half v) { return __half2float(v); }
  static SAL_DEVINL __half out(float v) { return __float2half_rn(v); }
};

template <typename T>
SAL_DEVINL void ld8(const T* p, float* v) {
  alignas(16) T t[8];
#pragma unroll
  for (int q = 0; q < (int)(8 * sizeof(T)) / 16; ++q)
    reinterpret_cast<uint4*>(t)[q] = __ldg(reinterpret_cast<const uint4*>(p) + q);
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = F<T>::in(t[j]);
}

template <typename T>
SAL_DEVINL void st8(T* p, const float* v) {
  alignas(16) T t[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) t[j] = F<T>::out(v[j]);
#pragma unroll
  for (int q = 0; q < (int)(8 * sizeof(T)) / 16; ++q)
    reinterpret_cast<uint4*>(p)[q] = reinterpret_cast<const uint4*>(t)[q];
}

// 8 consecutive columns of one row per thread (cols % 8 == 0); mask is dense
// row-major over [rows, cols] bits.
template <typename T>
__global__ void relu_dropout_fwd_kernel(const T* __restrict__ x, int64_t sx, T* __restrict__ y,
                                        int64_t sy, int64_t rows, int32_t cols,
                                        uint8_t* __restrict__ mask, float p, uint64_t seed,
                                        const int64_t* __restrict__ salt) {
  const uint32_t thresh = (uint32_t)(p * 65536.0f);
  const float scale = p > 0.f ? (p < 1.f ? 1.f / (1.f - p) : 0.f) : 1.f;
  const uint64_t key_base = mix64(seed ^ mix64((salt ? (uint64_t)*salt : 0ull) + 0x5EEDull));
  const uint32_t c8 = (uint32_t)cols / 8;
  const uint32_t n8 = (uint32_t)(rows * c8);  // < 2^32 groups per activation
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += gridDim.x * blockDim.x) {
    const uint32_t r = i / c8;
    const int c = (int)(i - r * c8) * 8;
    float v[8];
    ld8<T>(x + (int64_t)r * sx + c, v);
    if (p == 0.5f) {  // one keep bit per element (common.cuh dropout_word64)
      const uint32_t keep =
          (uint32_t)(dropout_word64(key_base, (uint64_t)(i >> 3)) >> (8 * (i & 7))) & 0xFFu;
      uint8_t bits = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool on = ((keep >> j) & 1u) && v[j] > 0.f;
        bits |= (uint8_t)on << j;
        v[j] = on ? v[j] * 2.f : 0.f;
      }
      st8<T>(y + (int64_t)r * sy + c, v);
      mask[i] = bits;
      continue;
    }
    // dropout stream: two splitmix64 draws per 8 elements, keyed on
    // (seed, step salt, element group) — 16 bits of uniform per element
    uint64_t r0 = ~0ull, r1 = ~0ull;
    if (p > 0.f) {
      const uint64_t k = key_base ^ ((uint64_t)i * 0xD1B54A32D192ED03ull);  // element group
      r0 = mix64(k);
      r1 = mix64(k + kGolden);
    }
    const uint32_t rr[4] = {(uint32_t)r0, (uint32_t)(r0 >> 32), (uint32_t)r1, (uint32_t)(r1 >> 32)};
    uint8_t bits = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t u16 = (rr[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
      const bool on = (u16 >= thresh) && v[j] > 0.f;
      bits |= (uint8_t)on << j;
      v[j] = on ? v[j] * scale : 0.f;
    }
    st8<T>(y + (int64_t)r * sy + c, v);
    mask[i] = bits;
  }
}

template <typename TDY, typename TDX>
__global__ void relu_dropout_bwd_kernel(const TDY* __restrict__ dy, int64_t sdy,
                                        const uint8_t* __restrict__ mask, TDX* __restrict__ dx,
                                        int64_t sdx, int64_t rows, int32_t cols, float p) {
  const float scale = p > 0.f ? (p < 1.f ? 1.f / (1.f - p) : 0.f) : 1.f;
  const uint32_t c8 = (uint32_t)cols / 8;
  const uint32_t n8 = (uint32_t)(rows * c8);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += gridDim.x * blockDim.x) {
    const uint32_t r = i / c8;
    const int c = (int)(i - r * c8) * 8;
    const uint8_t bits = mask[i];
    float v[8];
    ld8<TDY>(dy + (int64_t)r * sdy + c, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = ((bits >> j) & 1) ? v[j] * scale : 0.f;
    st8<TDX>(dx + (int64_t)r * sdx + c, v);
  }
}

// ---------------------------------------------------------------------------
// one warp per row; every block recounts the valid labels (B <= a few K)
template <typename T>
__global__ void lsm_nll_kernel(const T* __restrict__ logits, int64_t ld, int64_t rows, int32_t C,
                               const int64_t* __restrict__ labels, float* __restrict__ loss,
                               T* __restrict__ grad, int64_t ldg) {
  // one warp per row; a row of C <= 32 * kV logits is read once into registers
  // (wider rows re-read it per pass); one loss atomic per block
  constexpr int kV = 8;
  __shared__ float sh_cnt;
  __shared__ int warp_cnt[32];
  __shared__ float warp_loss[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c = 0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) c += labels[i] >= 0;
  c = warp_reduce_sum(c);
  if (lane == 0) warp_cnt[warp] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += warp_cnt[w];
    sh_cnt = (float)(t > 0 ? t : 1);
  }
  __syncthreads();
  const float inv = 1.f / sh_cnt;
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp;
  float my_loss = 0.f;
  if (row < rows) {
    const T* x = logits + row * ld;
    T* g = grad + row * ldg;
    const int64_t lab = labels[row];
    if (C <= 32 * kV) {
      float v[kV];
#pragma unroll
      for (int k = 0; k < kV; ++k) {
        const int j = lane + 32 * k;
        v[k] = j < C ? F<T>::in(x[j]) : -INFINITY;
      }
      float m = v[0];
#pragma unroll
      for (int k = 1; k < kV; ++k) m = fmaxf(m, v[k]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float sum = 0.f;
#pragma unroll
      for (int k = 0; k < kV; ++k)
        if (lane + 32 * k < C) sum += __expf(v[k] - m);
      sum = warp_reduce_sum(sum);
      const float lse = m + __logf(sum);
#pragma unroll
      for (int k = 0; k < kV; ++k) {
        const int j = lane + 32 * k;
        if (j < C)
          g[j] = F<T>::out(lab < 0 ? 0.f : (__expf(v[k] - lse) - (j == lab ? 1.f : 0.f)) * inv);
        if (j == lab) my_loss = (lse - v[k]) * inv;
      }
    } else {
      float m = -INFINITY;
      for (int j = lane; j < C; j += 32) m = fmaxf(m, F<T>::in(x[j]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float sum = 0.f;
      for (int j = lane; j < C; j += 32) sum += __expf(F<T>::in(x[j]) - m);
      sum = warp_reduce_sum(sum);
      const float lse = m + __logf(sum);
      for (int j = lane; j < C; j += 32) {
        const float xj = F<T>::in(x[j]);
        g[j] = F<T>::out(lab < 0 ? 0.f : (__expf(xj - lse) - (j == lab ? 1.f : 0.f)) * inv);
        if (j == lab) my_loss = (lse - xj) * inv;
      }
    }
  }
  my_loss = warp_reduce_sum(my_loss);   // the label's lane holds the row's loss
  if (lane == 0) warp_loss[warp] = my_loss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += warp_loss[w];
    atomicAdd(loss, t);
  }
}

// ---------------------------------------------------------------------------
// sampled-inference scoring: pred = argmax (first maximum, torch.argmax rule)
// of each logits row; counts[0] += #(pred == label), counts[1] += #(label >= 0).
// One warp per row, one pair of atomics per block.
template <typename T>
__global__ void argmax_correct_kernel(const T* __restrict__ logits, int64_t ld, int64_t rows,
                                      int32_t C, const int64_t* __restrict__ labels,
                                      unsigned long long* __restrict__ counts,
                                      int64_t* __restrict__ pred) {
  __shared__ int sh_ok, sh_tot;
  if (threadIdx.x == 0) sh_ok = sh_tot = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp;
  if (row < rows) {
    const T* x = logits + row * ld;
    float m = -INFINITY;
    int arg = C;
    for (int j = lane; j < C; j += 32) {
      const float v = F<T>::in(x[j]);
      if (v > m || (v != v && m == m)) { m = v; arg = j; }  // NaN counts as the maximum
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      const bool onan = om != om, mnan = m != m;
      if ((onan && !mnan) || (onan == mnan && (om > m || (om == m && oa < arg))) ||
          (onan && mnan && oa < arg)) {
        m = om;
        arg = oa;
      }
    }
    if (lane == 0) {
      if (pred) pred[row] = arg;
      const int64_t lab = labels[row];
      if (lab >= 0) {
        atomicAdd(&sh_tot, 1);
        if (lab == arg) atomicAdd(&sh_ok, 1);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && sh_tot) {
    atomicAdd(&counts[0], (unsigned long long)sh_ok);
    atomicAdd(&counts[1], (unsigned long long)sh_tot);
  }
}

// ---------------------------------------------------------------------------
// reverse adjacency of one MFG layer: for each source row s, the destinations
// d with s in N(d).  count -> exclusive scan -> fill (warp per destination).
__global__ void transpose_count_kernel(const int32_t* __restrict__ indptr,
                                       const int32_t* __restrict__ src,
                                       const int64_t* __restrict__ n_dst_dev, int64_t n_pad,
                                       int32_t* __restrict__ tcount) {
  const int64_t n = n_dst_dev ? *n_dst_dev : n_pad;
  const int64_t total = n > 0 ? indptr[n] : 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&tcount[src[e]], 1);
}

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

// exclusive scan of int32 counts over n items (n static), out[n] = total
__global__ void __launch_bounds__(kScanThreads)
scan_i32_kernel(const int32_t* __restrict__ in, int64_t n, int32_t* __restrict__ out, ScanWs ws) {
  __shared__ uint64_t sh_scan[kScanThreads / kWarp + 1];
  __shared__ uint64_t sh_prefix;
  __shared__ int sh_tile;
  const int64_t ntiles = n > 0 ? (n + kScanTile - 1) / kScanTile : 1;
  const int tile = grab_tile(ws, &sh_tile);
  if (tile >= ntiles) return;
  const int64_t base = (int64_t)tile * kScanTile + threadIdx.x * kScanItems;
  uint32_t c[kScanItems];
  uint64_t local = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    c[k] = (base + k < n) ? (uint32_t)in[base + k] : 0u;
    local += c[k];
  }
  uint64_t tile_total;
  const uint64_t excl = block_exclusive_scan<uint64_t, kScanThreads>(local, sh_scan, &tile_total);
  const uint64_t prefix = lookback_prefix(ws, tile, tile_total, &sh_prefix);
  uint64_t run = prefix + excl;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = (int32_t)run;
    run += c[k];
  }
  if (tile == ntiles - 1 && threadIdx.x == kScanThreads - 1) out[n] = (int32_t)(prefix + tile_total);
}

__global__ void transpose_fill_kernel(const int32_t* __restrict__ indptr,
                                      const int32_t* __restrict__ src,
                                      const int64_t* __restrict__ n_dst_dev, int64_t n_pad,
                                      const int32_t* __restrict__ tindptr,
                                      int32_t* __restrict__ tfill, int32_t* __restrict__ tdst,
                                      float* __restrict__ tw) {
  const int lane = threadIdx.x & 31;
  const int64_t n = n_dst_dev ? *n_dst_dev : n_pad;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t d = warp; d < n; d += nwarps) {
    const int32_t beg = indptr[d], end = indptr[d + 1];
    const float w = 1.f / (float)(end - beg);
    for (int32_t e = beg + lane; e < end; e += 32) {
      const int32_t s = src[e];
      const int32_t pos = tindptr[s] + atomicAdd(&tfill[s], 1);
      tdst[pos] = (int32_t)d;
      if (tw) tw[pos] = w;
    }
  }
}

// rows s < n whose input gradient is not a single scaled dA row: a self term
// (s < n_pad) or a number of in-edges other than one; appended in any order
__global__ void complex_rows_kernel(const int32_t* __restrict__ tindptr, int64_t n, int64_t n_pad,
                                    int32_t* __restrict__ list, int32_t* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  for (int64_t s0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; s0 < n;
       s0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = s0 + lane;
    bool c = false;
    if (s < n) c = s < n_pad || tindptr[s + 1] - tindptr[s] != 1;
    const unsigned m = __ballot_sync(0xffffffffu, c);
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(count, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (c) list[base + __popc(m & ((1u << lane) - 1u))] = (int32_t)s;
  }
}

// ---------------------------------------------------------------------------
// dz_prev[s, :] = mask_prev(s) * scale * (dA[s, f:2f] (s < n_pad) +
//                 sum_{d in T(s)} dA[d, 0:f] / deg(d));  warp per source row,
// 8 columns per lane (f <= 256 per pass, looped for wider rows)
// A warp takes 32 consecutive source rows: lane j fetches row j's reverse-
// adjacency bounds and its first in-edge (dst, 1/deg) in one coalesced pass;
// then the rows are finished kRows at a time with their self-term and
// first-edge rows loaded back to back (2 x kRows independent 16-byte loads
// per lane in flight).  Rows with more in-edges take a short extra loop.
template <typename TG, typename TO>
__global__ void __launch_bounds__(256, 3)
mean_bwd_t_kernel(const TG* __restrict__ dA, int64_t lda, int32_t f, int64_t n_pad,
                  const int32_t* __restrict__ indptr, const int32_t* __restrict__ tindptr,
                  const int32_t* __restrict__ tdst, const float* __restrict__ tw, int64_t rows,
                  const int64_t* __restrict__ m_dev, int part, int nparts,
                  const uint8_t* __restrict__ mask, float p, TO* __restrict__ dz, int64_t ldz,
                  int live) {
  constexpr int kRows = 4;
  constexpr int kChunk = 8;  // source rows per warp task (lanes 0..7 fetch metadata)
  const int lane = threadIdx.x & 31;
  const float scale = p > 0.f ? (p < 1.f ? 1.f / (1.f - p) : 0.f) : 1.f;
  // rows [rb, nrows) of this part (part_rows; the whole range when nparts == 1)
  int rb = 0, nrows = (int)rows;
  if (nparts > 1) part_rows(m_dev, rows, part, nparts, &rb, &nrows);
  if (live && m_dev) {   // only the 64-row chunks holding live rows (sal_mean_bwd_t_live)
    const int64_t cap = (*m_dev + 63) / 64 * 64;
    if (cap < nrows) nrows = (int)cap;
  }
  const int npad = (int)n_pad;
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  for (int base = rb + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kChunk; base < nrows;
       base += nwarps * kChunk) {
    // lane-parallel row metadata
    const int s_l = base + lane;
    int tb = 0, te = 0, d0 = -1;
    float w0 = 0.f;
    if (lane < kChunk && s_l < nrows) {
      tb = __ldg(tindptr + s_l);
      te = __ldg(tindptr + s_l + 1);
      if (te > tb) {
        d0 = __ldg(tdst + tb);
        w0 = tw ? __ldg(tw + tb) : 1.f / (float)(__ldg(indptr + d0 + 1) - __ldg(indptr + d0));
      }
    }
    const int nb = min(kChunk, nrows - base);
    for (int c0 = 0; c0 < f; c0 += 256) {
      const int c = c0 + lane * 8;
      const bool active = c < f;
      for (int r0 = 0; r0 < nb; r0 += kRows) {
        // raw 16-byte vectors in flight (converted after all loads are issued)
        uint4 self_raw[kRows][sizeof(TG) / 2], nb_raw[kRows][sizeof(TG) / 2];
        int dd[kRows];
        float ww[kRows];
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
          const int r = r0 + k;
          dd[k] = __shfl_sync(0xffffffffu, d0, r & 31);
          ww[k] = __shfl_sync(0xffffffffu, w0, r & 31);
          const int s = base + r;
#pragma unroll
          for (int q = 0; q < (int)sizeof(TG) / 2; ++q) {
            self_raw[k][q] = make_uint4(0, 0, 0, 0);
            nb_raw[k][q] = make_uint4(0, 0, 0, 0);
          }
          if (active && r < nb && s < npad) {
            const uint4* ps = reinterpret_cast<const uint4*>(dA + (int64_t)s * lda + f + c);
#pragma unroll
            for (int q = 0; q < (int)sizeof(TG) / 2; ++q) self_raw[k][q] = __ldg(ps + q);
          }
          if (active && r < nb && dd[k] >= 0) {
            const uint4* pn = reinterpret_cast<const uint4*>(dA + (int64_t)dd[k] * lda + c);
#pragma unroll
            for (int q = 0; q < (int)sizeof(TG) / 2; ++q) nb_raw[k][q] = __ldg(pn + q);
          }
        }
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
          const int r = r0 + k;
          if (r >= nb) break;
          const int s = base + r;
          const TG* sv = reinterpret_cast<const TG*>(self_raw[k]);
          const TG* nv = reinterpret_cast<const TG*>(nb_raw[k]);
          float acc[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = F<TG>::in(sv[j]) + F<TG>::in(nv[j]) * ww[k];
          const int rtb = __shfl_sync(0xffffffffu, tb, r & 31);
          const int rte = __shfl_sync(0xffffffffu, te, r & 31);
          for (int q = rtb + 1; q < rte; ++q) {  // further in-edges (rare)
            const int d = __ldg(tdst + q);
            const float w = tw ? __ldg(tw + q)
                               : 1.f / (float)(__ldg(indptr + d + 1) - __ldg(indptr + d));
            if (active) {
              float v[8];
              ld8<TG>(dA + (int64_t)d * lda + c, v);
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[j] += v[j] * w;
            }
          }
          if (active) {
            const uint8_t bits = mask[((int64_t)s * f + c) >> 3];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = ((bits >> j) & 1) ? acc[j] * scale : 0.f;
            st8<TO>(dz + (int64_t)s * ldz + c, acc);
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// The same input gradient in two disjoint passes (sal_mean_bwd):
//   * destination-major, warp per destination d: the source rows s of d with one
//     in-edge and no self term (s >= n_pad) — most rows of a sampled MFG — get
//     dz[s] = mask(s) * scale * (0 + dA[d, 0:f] * (1/deg d)): dA[d] is read once
//     for its ~fanout sources, and no reverse-adjacency chain is walked;
//   * source-major, warp per 32 source rows: every other row (self term, several
//     or no in-edges) as mean_bwd_t_kernel does it.
// Same arithmetic as mean_bwd_t_kernel row for row, so the output is bit-identical.
#ifndef SAL_MBS_MINB
#define SAL_MBS_MINB 3
#endif
template <typename TG, typename TO>
__global__ void __launch_bounds__(256, SAL_MBS_MINB)
mean_bwd_split_kernel(const TG* __restrict__ dA, int64_t lda, int32_t f, int64_t n_pad,
                      const int64_t* __restrict__ n_dst_dev, const int32_t* __restrict__ indptr,
                      const int32_t* __restrict__ src, const int32_t* __restrict__ tindptr,
                      const int32_t* __restrict__ tdst, const float* __restrict__ tw,
                      int64_t rows, const int64_t* __restrict__ m_dev, int live,
                      const uint8_t* __restrict__ mask, float p, TO* __restrict__ dz,
                      int64_t ldz, int dst_blocks, const int32_t* __restrict__ cplx,
                      const int32_t* __restrict__ n_cplx) {
  const int lane = threadIdx.x & 31;
  const float scale = p > 0.f ? (p < 1.f ? 1.f / (1.f - p) : 0.f) : 1.f;
  int nrows = (int)rows;
  if (live && m_dev) {
    const int64_t cap = (*m_dev + 63) / 64 * 64;
    if (cap < nrows) nrows = (int)cap;
  }
  const int npad = (int)n_pad;
  // the two passes' blocks interleaved in launch order, so both progress from the start
  const int src_blocks = (int)gridDim.x - dst_blocks;
  const int mpair = min(dst_blocks, src_blocks);
  int role, bidx;
  if ((int)blockIdx.x < 2 * mpair) {
    role = blockIdx.x & 1;
    bidx = blockIdx.x >> 1;
  } else {
    role = dst_blocks > src_blocks ? 0 : 1;
    bidx = mpair + ((int)blockIdx.x - 2 * mpair);
  }
  if (role == 0) {
    // ---- destination-major: single-in-edge rows without a self term
    const int n_dst = (int)(n_dst_dev ? *n_dst_dev : n_pad);
    const int nw = dst_blocks * (int)(blockDim.x >> 5);
    for (int d = (int)((bidx * blockDim.x + threadIdx.x) >> 5); d < n_dst; d += nw) {
      const int beg = __ldg(indptr + d), end = __ldg(indptr + d + 1);
      const float w = 1.f / (float)(end - beg);
      for (int e0 = beg; e0 < end; e0 += 32) {
        const int e = e0 + lane;
        int sj = -1;
        bool simple = false;
        if (e < end) {
          sj = __ldg(src + e);
          simple = sj >= npad && sj < nrows && __ldg(tindptr + sj + 1) - __ldg(tindptr + sj) == 1;
        }
        unsigned m = __ballot_sync(0xffffffffu, simple);
        if (!m) continue;
        for (int c0 = 0; c0 < f; c0 += 256) {
          const int c = c0 + lane * 8;
          const bool active = c < f;
          float v[8];
          if (active) {
            ld8<TG>(dA + (int64_t)d * lda + c, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = 0.f + v[j] * w;
          }
          // the mask bytes of up to 8 sources in flight, then their rows written
          unsigned mm = m;
          while (mm) {
            int sk[8];
            uint8_t bk[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int j = mm ? __ffs(mm) - 1 : -1;
              if (mm) mm &= mm - 1;
              sk[k] = __shfl_sync(0xffffffffu, sj, j < 0 ? 0 : j);
              if (j < 0) sk[k] = -1;
              bk[k] = (active && sk[k] >= 0) ? mask[((int64_t)sk[k] * f + c) >> 3] : (uint8_t)0;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              if (active && sk[k] >= 0) {
                float acc[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) acc[q] = ((bk[k] >> q) & 1) ? v[q] * scale : 0.f;
                st8<TO>(dz + (int64_t)sk[k] * ldz + c, acc);
              }
            }
          }
        }
      }
    }
    return;
  }
  // ---- source-major: the remaining rows (self term, several or no in-edges), 8
  // rows per warp task (rows below n_pad are all of this kind)
  constexpr int kChunk = 8;
  const int nw = src_blocks * (int)(blockDim.x >> 5);
  // with a prebuilt list of those rows (cplx, built beside the forward pass) the
  // tasks walk the list; else they scan every row
  const int nitems = cplx ? *n_cplx : nrows;
  for (int base = (int)((bidx * blockDim.x + threadIdx.x) >> 5) * kChunk;
       base < nitems; base += nw * kChunk) {
    int s_l = -1;
    int tb = 0, te = 0, d0 = -1;
    float w0 = 0.f;
    bool complex_row = false;
    if (lane < kChunk && base + lane < nitems) s_l = cplx ? __ldg(cplx + base + lane) : base + lane;
    if (s_l >= 0 && s_l < nrows) {
      tb = __ldg(tindptr + s_l);
      te = __ldg(tindptr + s_l + 1);
      complex_row = !(te - tb == 1 && s_l >= npad);
      if (complex_row && te > tb) {
        d0 = __ldg(tdst + tb);
        w0 = tw ? __ldg(tw + tb) : 1.f / (float)(__ldg(indptr + d0 + 1) - __ldg(indptr + d0));
      }
    }
    unsigned m = __ballot_sync(0xffffffffu, complex_row);
    // complex rows four at a time: self and first-edge rows loaded back to back
    while (m) {
      int rk[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        rk[k] = m ? __ffs(m) - 1 : -1;
        if (m) m &= m - 1;
      }
      for (int c0 = 0; c0 < f; c0 += 256) {
        const int c = c0 + lane * 8;
        const bool active = c < f;
        constexpr int V = (int)sizeof(TG) / 2;   // 16-byte vectors per 8 columns
        uint4 sraw[4][V], nraw[4][V];              // raw rows: converted after all loads
        float wk[4];
        uint8_t mk[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = rk[k] < 0 ? 0 : rk[k];
          const int dd = __shfl_sync(0xffffffffu, d0, r);
          wk[k] = __shfl_sync(0xffffffffu, w0, r);
          const int s = __shfl_sync(0xffffffffu, s_l, r);
#pragma unroll
          for (int q = 0; q < V; ++q) sraw[k][q] = nraw[k][q] = make_uint4(0, 0, 0, 0);
          mk[k] = 0;
          if (active && rk[k] >= 0) {
            if (s < npad) {
              const uint4* ps = reinterpret_cast<const uint4*>(dA + (int64_t)s * lda + f + c);
#pragma unroll
              for (int q = 0; q < V; ++q) sraw[k][q] = __ldg(ps + q);
            }
            if (dd >= 0) {
              const uint4* pn = reinterpret_cast<const uint4*>(dA + (int64_t)dd * lda + c);
#pragma unroll
              for (int q = 0; q < V; ++q) nraw[k][q] = __ldg(pn + q);
            }
            mk[k] = mask[((int64_t)s * f + c) >> 3];
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (rk[k] < 0) break;
          const int r = rk[k];
          const int s = __shfl_sync(0xffffffffu, s_l, r);
          const int rtb = __shfl_sync(0xffffffffu, tb, r);
          const int rte = __shfl_sync(0xffffffffu, te, r);
          if (!active) continue;
          const TG* sv = reinterpret_cast<const TG*>(sraw[k]);
          const TG* nv = reinterpret_cast<const TG*>(nraw[k]);
          float acc[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = F<TG>::in(sv[j]) + F<TG>::in(nv[j]) * wk[k];
          for (int q = rtb + 1; q < rte; ++q) {
            const int d = __ldg(tdst + q);
            const float w = tw ? __ldg(tw + q)
                               : 1.f / (float)(__ldg(indptr + d + 1) - __ldg(indptr + d));
            float v[8];
            ld8<TG>(dA + (int64_t)d * lda + c, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += v[j] * w;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = ((mk[k] >> j) & 1) ? acc[j] * scale : 0.f;
          st8<TO>(dz + (int64_t)s * ldz + c, acc);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Adam (torch.optim.Adam semantics, no weight decay) over flat fp32 params,
// bias correction from the device step counter; refreshes the bf16 shadow.
__global__ void adam_kernel(float* __restrict__ p, float* __restrict__ g,
                            float* __restrict__ m, float* __restrict__ v,
                            __nv_bfloat16* __restrict__ shadow, int64_t n, float lr, float b1,
                            float b2, float eps, const int64_t* __restrict__ t_dev,
                            int zero_grad) {
  const float t = (float)(*t_dev + 1);
  const float bc1 = 1.f - __powf(b1, t);
  const float bc2 = 1.f - __powf(b2, t);
  const float step = lr / bc1;
  const float rbc2 = rsqrtf(bc2);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    if (zero_grad) g[i] = 0.f;
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float pi = p[i] - step * mi / (sqrtf(vi) * rbc2 + eps);
    p[i] = pi;
    if (shadow) shadow[i] = __float2bfloat16_rn(pi);
  }
}

// the same update, 4 elements per thread (n % 4 == 0, 16-byte aligned buffers):
// a quarter of the threads, four independent element chains each
SAL_DEVINL void adam_elem(float& p, float& g, float& m, float& v, float b1, float b2,
                          float step, float rbc2, float eps, int zero_grad) {
  const float gi = g;
  if (zero_grad) g = 0.f;
  const float mi = b1 * m + (1.f - b1) * gi;
  const float vi = b2 * v + (1.f - b2) * gi * gi;
  m = mi;
  v = vi;
  p = p - step * mi / (sqrtf(vi) * rbc2 + eps);
}

__global__ void adam4_kernel(float4* __restrict__ p, float4* __restrict__ g,
                             float4* __restrict__ m, float4* __restrict__ v,
                             uint2* __restrict__ shadow, int64_t n4, float lr, float b1,
                             float b2, float eps, const int64_t* __restrict__ t_dev,
                             int zero_grad) {
  const float t = (float)(*t_dev + 1);
  const float step = lr / (1.f - __powf(b1, t));
  const float rbc2 = rsqrtf(1.f - __powf(b2, t));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 pi = p[i], gi = g[i], mi = m[i], vi = v[i];
    adam_elem(pi.x, gi.x, mi.x, vi.x, b1, b2, step, rbc2, eps, zero_grad);
    adam_elem(pi.y, gi.y, mi.y, vi.y, b1, b2, step, rbc2, eps, zero_grad);
    adam_elem(pi.z, gi.z, mi.z, vi.z, b1, b2, step, rbc2, eps, zero_grad);
    adam_elem(pi.w, gi.w, mi.w, vi.w, b1, b2, step, rbc2, eps, zero_grad);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
    if (zero_grad) g[i] = gi;
    if (shadow) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(pi.x, pi.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(pi.z, pi.w);
      shadow[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
  }
}

// adam4_kernel + step_tail_kernel in one launch: the block that finishes last (a
// ticket counter, reset by that block) does the per-step bookkeeping, after every
// block has read the step count it increments
__global__ void adam4_tail_kernel(float4* __restrict__ p, float4* __restrict__ g,
                                  float4* __restrict__ m, float4* __restrict__ v,
                                  uint2* __restrict__ shadow, int64_t n4, float lr, float b1,
                                  float b2, float eps, int64_t* __restrict__ t_dev, int zero_grad,
                                  float* __restrict__ loss, float* __restrict__ last,
                                  float* __restrict__ log, int64_t log_len,
                                  int64_t* __restrict__ step, unsigned int* __restrict__ ticket) {
  const float t = (float)(*t_dev + 1);
  const float stp = lr / (1.f - __powf(b1, t));
  const float rbc2 = rsqrtf(1.f - __powf(b2, t));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 pi = p[i], gi = g[i], mi = m[i], vi = v[i];
    adam_elem(pi.x, gi.x, mi.x, vi.x, b1, b2, stp, rbc2, eps, zero_grad);
    adam_elem(pi.y, gi.y, mi.y, vi.y, b1, b2, stp, rbc2, eps, zero_grad);
    adam_elem(pi.z, gi.z, mi.z, vi.z, b1, b2, stp, rbc2, eps, zero_grad);
    adam_elem(pi.w, gi.w, mi.w, vi.w, b1, b2, stp, rbc2, eps, zero_grad);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
    if (zero_grad) g[i] = gi;
    if (shadow) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(pi.x, pi.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(pi.z, pi.w);
      shadow[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ticket, 1u) == gridDim.x - 1) {   // every block has read *t_dev
      *ticket = 0;
      const int64_t s = *step;
      const float l = *loss;
      *loss = 0.f;
      *last = l;
      if (s >= 0 && s < log_len) log[s] = l;
      *step = s + 1;
      *t_dev += 1;
    }
  }
}

__global__ void step_tail_kernel(float* __restrict__ loss, float* __restrict__ last,
                                 float* __restrict__ log, int64_t log_len,
                                 int64_t* __restrict__ step, int64_t* __restrict__ adam_t) {
  const int64_t s = *step;
  const float l = *loss;
  *loss = 0.f;
  *last = l;
  if (s >= 0 && s < log_len) log[s] = l;
  *step = s + 1;
  if (adam_t) *adam_t += 1;
}

static int ew_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

static int warp_grid(int64_t rows) {
  int64_t g = (rows + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

static int done(int kernels) {
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  count_launch(kernels);
  return SAL_OK;
}

}  // namespace sal

extern "C" {

int sal_plan_next(const int64_t* desc_all, int64_t n_steps, int64_t* cursor, sal_batch_desc* out,
                  void* stream) {
  sal::plan_next_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(desc_all, n_steps, cursor, out);
  return sal::done(1);
}

int sal_relu_dropout_fwd(const void* x, int64_t sx, void* y, int64_t sy, int64_t rows,
                         int32_t cols, int32_t dtype, uint8_t* mask, float p, uint64_t seed,
                         const int64_t* salt_dev, void* stream) {
  if (cols % 8 != 0 || sx % 8 != 0 || sy % 8 != 0)
    return sal::set_error(SAL_EINVAL, "relu_dropout_fwd: invalid argument (cols % 8 != 0 || sx % 8 != 0 || sy % 8 != 0)");
  cudaStream_t st = (cudaStream_t)stream;
  const int g = sal::ew_grid(rows * (cols / 8));
  if (dtype == SAL_BF16)
    sal::relu_dropout_fwd_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(
        (const __nv_bfloat16*)x, sx, (__nv_bfloat16*)y, sy, rows, cols, mask, p, seed, salt_dev);
  else if (dtype == SAL_F32)
    sal::relu_dropout_fwd_kernel<float><<<g, 256, 0, st>>>((const float*)x, sx, (float*)y, sy,
                                                          rows, cols, mask, p, seed, salt_dev);
  else
    return sal::set_error(SAL_EINVAL, "relu_dropout_fwd: unsupported dtype or shape");
  return sal::done(1);
}

int sal_relu_dropout_bwd(const void* dy, int64_t sdy, int32_t dy_dtype, const uint8_t* mask,
                         void* dx, int64_t sdx, int32_t dx_dtype, int64_t rows, int32_t cols,
                         float p, void* stream) {
  if (cols % 8 != 0)
    return sal::set_error(SAL_EINVAL, "relu_dropout_bwd: invalid argument (cols % 8 != 0)");
  cudaStream_t st = (cudaStream_t)stream;
  const int g = sal::ew_grid(rows * (cols / 8));
  if (dy_dtype == SAL_F32 && dx_dtype == SAL_BF16)
    sal::relu_dropout_bwd_kernel<float, __nv_bfloat16><<<g, 256, 0, st>>>(
        (const float*)dy, sdy, mask, (__nv_bfloat16*)dx, sdx, rows, cols, p);
  else if (dy_dtype == SAL_BF16 && dx_dtype == SAL_BF16)
    sal::relu_dropout_bwd_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, st>>>(
        (const __nv_bfloat16*)dy, sdy, mask, (__nv_bfloat16*)dx, sdx, rows, cols, p);
  else if (dy_dtype == SAL_F32 && dx_dtype == SAL_F32)
    sal::relu_dropout_bwd_kernel<float, float><<<g, 256, 0, st>>>((const float*)dy, sdy, mask,
                                                                 (float*)dx, sdx, rows, cols, p);
  else
    return sal::set_error(SAL_EINVAL, "relu_dropout_bwd: unsupported dtype or shape");
  return sal::done(1);
}

int sal_lsm_nll(const void* logits, int64_t ld, int64_t rows, int32_t C, int32_t dtype,
                const int64_t* labels, float* loss, void* grad, int64_t ldg, void* stream) {
  if (rows <= 0) return SAL_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int warps = 8;
  const int grid = (int)((rows + warps - 1) / warps);
  if (dtype == SAL_BF16)
    sal::lsm_nll_kernel<__nv_bfloat16><<<grid, 32 * warps, 0, st>>>(
        (const __nv_bfloat16*)logits, ld, rows, C, labels, loss, (__nv_bfloat16*)grad, ldg);
  else if (dtype == SAL_F32)
    sal::lsm_nll_kernel<float><<<grid, 32 * warps, 0, st>>>((const float*)logits, ld, rows, C,
                                                           labels, loss, (float*)grad, ldg);
  else
    return sal::set_error(SAL_EINVAL, "lsm_nll: unsupported dtype or shape");
  return sal::done(1);
}

int sal_argmax_correct(const void* logits, int64_t ld, int64_t rows, int32_t C, int32_t dtype,
                       const int64_t* labels, int64_t* counts, int64_t* pred, void* stream) {
  if (rows < 0 || C <= 0 || !counts || !labels)
    return sal::set_error(SAL_EINVAL, "argmax_correct: invalid argument (rows < 0 || C <= 0 || !counts || !labels)");
  if (rows == 0) return SAL_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int warps = 8;
  const int grid = (int)((rows + warps - 1) / warps);
  unsigned long long* c = (unsigned long long*)counts;
  if (dtype == SAL_BF16)
    sal::argmax_correct_kernel<__nv_bfloat16><<<grid, 32 * warps, 0, st>>>(
        (const __nv_bfloat16*)logits, ld, rows, C, labels, c, pred);
  else if (dtype == SAL_F32)
    sal::argmax_correct_kernel<float><<<grid, 32 * warps, 0, st>>>((const float*)logits, ld,
                                                                  rows, C, labels, c, pred);
  else
    return sal::set_error(SAL_EINVAL, "argmax_correct: unsupported dtype or shape");
  return sal::done(1);
}

// transpose workspace: tcount, tfill (int32 [n+1] each), the complex-row count (int32,
// 16 B slot) and list (int32 [n]), then the scan workspace (16-byte aligned)
static int64_t tws_list_count_off(int64_t n) { return 8 * (n + 1); }
static int64_t tws_list_off(int64_t n) { return 8 * (n + 1) + 16; }
static int64_t tws_scan_off(int64_t n) { return (tws_list_off(n) + 4 * n + 15) / 16 * 16; }

size_t sal_transpose_ws_bytes(int64_t n_src_rows) {
  return (size_t)tws_scan_off(n_src_rows) + sal::scan_ws_bytes(n_src_rows) + 64;
}

int sal_transpose_complex_list(int64_t n_src_rows, int64_t* list_offset, int64_t* count_offset) {
  if (n_src_rows < 0 || list_offset == nullptr || count_offset == nullptr)
    return sal::set_error(SAL_EINVAL, "transpose_complex_list: bad arguments");
  *list_offset = tws_list_off(n_src_rows);
  *count_offset = tws_list_count_off(n_src_rows);
  return SAL_OK;
}

int sal_transpose_build(const int32_t* indptr, const int32_t* src, const int64_t* n_dst_dev,
                        int64_t n_pad, int64_t n_src_rows, int64_t max_edges, int32_t* tindptr,
                        int32_t* tdst, float* tw, void* ws, int32_t ws_zeroed, void* stream) {
  (void)max_edges;
  if (indptr == nullptr || src == nullptr || tindptr == nullptr || tdst == nullptr || ws == nullptr)
    return sal::set_error(SAL_EINVAL, "transpose_build: unsupported dtype or shape");
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* tcount = (int32_t*)ws;
  int32_t* tfill = tcount + (n_src_rows + 1);
  int32_t* ncplx = (int32_t*)((char*)ws + tws_list_count_off(n_src_rows));
  int32_t* cplx = (int32_t*)((char*)ws + tws_list_off(n_src_rows));
  char* scan = (char*)ws + tws_scan_off(n_src_rows);
  if (!ws_zeroed) {  // else the caller zeroed the whole ws (sal_zero_spans)
    if (cudaMemsetAsync(ws, 0, (size_t)tws_list_off(n_src_rows), st) != cudaSuccess)
      return SAL_ECUDA;
    const size_t sb = sal::scan_ws_bytes(n_src_rows);
    if (cudaMemsetAsync(scan, 0, sb, st) != cudaSuccess) return SAL_ECUDA;
  }
  sal::transpose_count_kernel<<<sal::ew_grid(n_pad * 16), 256, 0, st>>>(indptr, src, n_dst_dev,
                                                                         n_pad, tcount);
  sal::ScanWs sw;
  const int64_t tiles = (n_src_rows + sal::kScanTile - 1) / sal::kScanTile + 1;
  sw.status = (unsigned long long*)scan;
  sw.tile_counter = (unsigned int*)(scan + tiles * 8);
  const int sgrid = (int)((n_src_rows + sal::kScanTile - 1) / sal::kScanTile);
  sal::scan_i32_kernel<<<sgrid > 0 ? sgrid : 1, sal::kScanThreads, 0, st>>>(tcount, n_src_rows,
                                                                           tindptr, sw);
  sal::transpose_fill_kernel<<<sal::warp_grid(n_pad), 256, 0, st>>>(indptr, src, n_dst_dev, n_pad,
                                                                    tindptr, tfill, tdst, tw);
  // the rows sal_mean_bwd's source-major pass handles (self term, 0 or >= 2 in-edges)
  sal::complex_rows_kernel<<<sal::ew_grid(n_src_rows), 256, 0, st>>>(tindptr, n_src_rows, n_pad,
                                                                     cplx, ncplx);
  return sal::done(4);
}

static int mean_bwd_t_launch(const void* dA, int64_t lda, int32_t dA_dtype, int32_t f,
                             int64_t n_pad, const int32_t* indptr, const int32_t* tindptr,
                             const int32_t* tdst, const float* tw, int64_t rows,
                             const int64_t* m_dev, int32_t part, int32_t nparts,
                             const uint8_t* mask, float p, void* dz, int64_t ldz,
                             int32_t dz_dtype, void* stream, int live) {
  if (f % 8 != 0 || lda % 8 != 0 || ldz % 8 != 0)
    return sal::set_error(SAL_EINVAL, "mean_bwd_t_launch: invalid argument (f % 8 != 0 || lda % 8 != 0 || ldz % 8 != 0)");
  if (nparts < 1 || part < 0 || part >= nparts)
    return sal::set_error(SAL_EINVAL, "mean_bwd_t_launch: invalid argument (nparts < 1 || part < 0 || part >= nparts)");
  cudaStream_t st = (cudaStream_t)stream;
  const int g = sal::warp_grid((rows / nparts + 7) / 8);
  if (dA_dtype == SAL_BF16 && dz_dtype == SAL_BF16)
    sal::mean_bwd_t_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, st>>>(
        (const __nv_bfloat16*)dA, lda, f, n_pad, indptr, tindptr, tdst, tw, rows, m_dev, part,
        nparts, mask, p, (__nv_bfloat16*)dz, ldz, live);
  else if (dA_dtype == SAL_F32 && dz_dtype == SAL_F32)
    sal::mean_bwd_t_kernel<float, float><<<g, 256, 0, st>>>(
        (const float*)dA, lda, f, n_pad, indptr, tindptr, tdst, tw, rows, m_dev, part, nparts,
        mask, p, (float*)dz, ldz, live);
  else
    return sal::set_error(SAL_EINVAL, "mean_bwd_t_launch: unsupported dtype or shape");
  return sal::done(1);
}

int sal_mean_bwd_t(const void* dA, int64_t lda, int32_t dA_dtype, int32_t f, int64_t n_pad,
                   const int32_t* indptr, const int32_t* tindptr, const int32_t* tdst,
                   const float* tw, int64_t rows, const uint8_t* mask, float p, void* dz,
                   int64_t ldz, int32_t dz_dtype, void* stream) {
  return mean_bwd_t_launch(dA, lda, dA_dtype, f, n_pad, indptr, tindptr, tdst, tw, rows, nullptr,
                           0, 1, mask, p, dz, ldz, dz_dtype, stream, 0);
}

int sal_mean_bwd_t_live(const void* dA, int64_t lda, int32_t dA_dtype, int32_t f, int64_t n_pad,
                        const int32_t* indptr, const int32_t* tindptr, const int32_t* tdst,
                        const float* tw, int64_t rows, const int64_t* m_dev, const uint8_t* mask,
                        float p, void* dz, int64_t ldz, int32_t dz_dtype, void* stream) {
  if (m_dev == nullptr)
    return sal::set_error(SAL_EINVAL, "mean_bwd_t_live: invalid argument (m_dev == nullptr)");
  return mean_bwd_t_launch(dA, lda, dA_dtype, f, n_pad, indptr, tindptr, tdst, tw, rows, m_dev,
                           0, 1, mask, p, dz, ldz, dz_dtype, stream, 1);
}

int sal_mean_bwd(const void* dA, int64_t lda, int32_t dA_dtype, int32_t f, int64_t n_pad,
                 const int64_t* n_dst_dev, const int32_t* indptr, const int32_t* src,
                 const int32_t* tindptr, const int32_t* tdst, const float* tw,
                 const int32_t* cplx, const int32_t* n_cplx, int64_t rows,
                 const int64_t* m_dev, const uint8_t* mask, float p, void* dz, int64_t ldz,
                 int32_t dz_dtype, void* stream) {
  if ((cplx == nullptr) != (n_cplx == nullptr))
    return sal::set_error(SAL_EINVAL, "mean_bwd: cplx and n_cplx go together");
  if (dA == nullptr || indptr == nullptr || src == nullptr || tindptr == nullptr ||
      tdst == nullptr || mask == nullptr || dz == nullptr)
    return sal::set_error(SAL_EINVAL, "mean_bwd: null argument");
  if (f % 8 != 0 || lda % 8 != 0 || ldz % 8 != 0 || f <= 0)
    return sal::set_error(SAL_EINVAL, "mean_bwd: f, lda and ldz must be multiples of 8");
  if (rows < 0 || n_pad < 0 || n_pad > rows)
    return sal::set_error(SAL_EINVAL, "mean_bwd: bad row counts");
  if (rows == 0) return SAL_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int dst_blocks = (int)((n_pad + 7) / 8);
  const int cap = sal::num_sms() * 8;
  if (dst_blocks > cap) dst_blocks = cap;
  if (dst_blocks < 1) dst_blocks = 1;
  int src_blocks = (int)((rows + 63) / 64);   // 8 warps x 8-row tasks per block
  if (src_blocks > cap) src_blocks = cap;
  // walking a prebuilt list: a grid-stride pass over a fraction of the rows
  if (cplx != nullptr && src_blocks > sal::num_sms() * 2) src_blocks = sal::num_sms() * 2;
  if (src_blocks < 1) src_blocks = 1;
  const int g = dst_blocks + src_blocks;
  const int live = m_dev != nullptr;
  if (dA_dtype == SAL_BF16 && dz_dtype == SAL_BF16)
    sal::mean_bwd_split_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, st>>>(
        (const __nv_bfloat16*)dA, lda, f, n_pad, n_dst_dev, indptr, src, tindptr, tdst, tw,
        rows, m_dev, live, mask, p, (__nv_bfloat16*)dz, ldz, dst_blocks, cplx, n_cplx);
  else if (dA_dtype == SAL_F32 && dz_dtype == SAL_F32)
    sal::mean_bwd_split_kernel<float, float><<<g, 256, 0, st>>>(
        (const float*)dA, lda, f, n_pad, n_dst_dev, indptr, src, tindptr, tdst, tw, rows, m_dev,
        live, mask, p, (float*)dz, ldz, dst_blocks, cplx, n_cplx);
  else
    return sal::set_error(SAL_EINVAL, "mean_bwd: dtypes must be bf16/bf16 or f32/f32");
  return sal::done(1);
}

int sal_adam_step(float* param, float* grad, float* m, float* v, void* shadow_bf16,
                  int64_t n, float lr, float beta1, float beta2, float eps,
                  const int64_t* t_dev, int32_t zero_grad, void* stream) {
  if (param == nullptr || grad == nullptr || m == nullptr || v == nullptr || t_dev == nullptr)
    return sal::set_error(SAL_EINVAL, "adam_step: unsupported dtype or shape");
  const bool vec = n % 4 == 0 &&
                   ((uintptr_t)param | (uintptr_t)grad | (uintptr_t)m | (uintptr_t)v) % 16 == 0 &&
                   (uintptr_t)shadow_bf16 % 8 == 0;
  if (vec)
    sal::adam4_kernel<<<sal::ew_grid(n / 4), 256, 0, (cudaStream_t)stream>>>(
        (float4*)param, (float4*)grad, (float4*)m, (float4*)v, (uint2*)shadow_bf16, n / 4, lr,
        beta1, beta2, eps, t_dev, zero_grad);
  else
    sal::adam_kernel<<<sal::ew_grid(n), 256, 0, (cudaStream_t)stream>>>(
        param, grad, m, v, (__nv_bfloat16*)shadow_bf16, n, lr, beta1, beta2, eps, t_dev,
        zero_grad);
  return sal::done(1);
}

struct ZeroSpans {
  uint4* p[8];
  int64_t n16[8];
  int32_t n;
};
__global__ void zero_spans_kernel(ZeroSpans z) {
  for (int k = 0; k < z.n; ++k)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < z.n16[k];
         i += (int64_t)gridDim.x * blockDim.x)
      z.p[k][i] = make_uint4(0u, 0u, 0u, 0u);
}

int sal_zero_spans(void* const* ptrs, const int64_t* bytes, int32_t n, void* stream) {
  if (n < 0 || n > 8 || (n && (!ptrs || !bytes)))
    return sal::set_error(SAL_EINVAL, "zero_spans: invalid argument (n < 0 || n > 8 || (n && (!ptrs || !bytes)))");
  ZeroSpans z;
  z.n = n;
  int64_t most = 0;
  for (int k = 0; k < n; ++k) {
    if (((uintptr_t)ptrs[k] & 15) || (bytes[k] & 15))
      return sal::set_error(SAL_EINVAL, "zero_spans: invalid argument (((uintptr_t)ptrs[k] & 15) || (bytes[k] & 15))");
    z.p[k] = (uint4*)ptrs[k];
    z.n16[k] = bytes[k] / 16;
    if (z.n16[k] > most) most = z.n16[k];
  }
  if (n == 0 || most == 0) return SAL_OK;
  zero_spans_kernel<<<sal::ew_grid(most), 256, 0, (cudaStream_t)stream>>>(z);
  return sal::done(1);
}

int sal_adam_step_tail(float* param, float* grad, float* m, float* v, void* shadow_bf16,
                       int64_t n, float lr, float beta1, float beta2, float eps, int64_t* t_dev,
                       int32_t zero_grad, float* loss, float* last, float* log, int64_t log_len,
                       int64_t* step, unsigned int* ticket_dev, void* stream) {
  if (param == nullptr || grad == nullptr || m == nullptr || v == nullptr || t_dev == nullptr ||
      loss == nullptr || last == nullptr || step == nullptr || ticket_dev == nullptr)
    return sal::set_error(SAL_EINVAL, "adam_step_tail: null argument");
  if (n % 4 != 0 ||
      ((uintptr_t)param | (uintptr_t)grad | (uintptr_t)m | (uintptr_t)v) % 16 != 0 ||
      (uintptr_t)shadow_bf16 % 8 != 0)
    return sal::set_error(SAL_EINVAL, "adam_step_tail: n %% 4 and 16-byte aligned buffers needed");
  sal::adam4_tail_kernel<<<sal::ew_grid(n / 4), 256, 0, (cudaStream_t)stream>>>(
      (float4*)param, (float4*)grad, (float4*)m, (float4*)v, (uint2*)shadow_bf16, n / 4, lr,
      beta1, beta2, eps, t_dev, zero_grad, loss, last, log, log_len, step, ticket_dev);
  return sal::done(1);
}

int sal_step_tail(float* loss, float* last, float* log, int64_t log_len, int64_t* step,
                  int64_t* adam_t, void* stream) {
  sal::step_tail_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(loss, last, log, log_len, step,
                                                           adam_t);
  return sal::done(1);
}

}  // extern "C"
