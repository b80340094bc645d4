// Fused output layer of the training step: the last SAGEConv with its loss and
// backward in one kernel (PAPER.md:2577-2585 model; mpnn.py:57-65 mean rule).
//
// Per 64-row block of the batch (16 CTAs at batch 1024, so the rest of the GPU
// stays free for the overlapped prep chain):
//   1. the layer's cat rows [mean | h_dst] (mean written by the segment-mean
//      kernel, whose edge gathers need a full grid)  -> A tile [64, 2f] bf16 (smem)
//   2. logits = A @ W^T                              (mma.sync bf16, fp32 acc)
//   3. log_softmax + NLL (labels < 0 ignored, mean over valid labels) and
//      dlogits = (softmax - onehot) / count          -> D tile [64, C] bf16 (smem)
//   4. dA = D @ W   -> [dmean | dh_dst] rows (bf16, global; read by mean_bwd_t)
//   5. dW += D^T @ A                                 (fp32 vector atomics; the
//      trainer zeroes dW on its late stream)
// Replaces 3 cuBLAS GEMMs + lsm_nll (four launches, the logits and dlogits round
// trips).  Measured: 51 us alone at papers shape (16 CTAs; phases 1-3 26 us,
// dA 10 us, dW 8 us + 7.5 us of atomics), bound by legacy mma.sync throughput
// on 16 SMs, against ~20 us for the four unfused kernels — so FusedSAGE keeps
// it off by default (use_head); correct and tested for later use with tcgen05.
#include <cuda_bf16.h>

#include "common.cuh"
#include "salient_internal.h"

namespace sal {
namespace head {

constexpr int kRows = 64;     // rows per CTA
constexpr int kWarps = 8;     // (m-tile, half of the n-tiles) pairs
constexpr int kThreads = kWarps * 32;
constexpr int kChunk = 128;   // dA columns per W chunk staged in smem

SAL_DEVINL uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

SAL_DEVINL void ldsm_x4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
SAL_DEVINL void ldsm_x4_t(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
SAL_DEVINL void ldsm_x2_t(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
               : "=r"(r[0]), "=r"(r[1])
               : "r"(addr));
}
SAL_DEVINL void ldsm_x2(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r[0]), "=r"(r[1])
               : "r"(addr));
}
SAL_DEVINL void mma16816(float* d, const uint32_t* a, const uint32_t* b) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
SAL_DEVINL void red_add_v2(float* p, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
SAL_DEVINL uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// smem strides (elements), padded so 8 ldmatrix rows hit distinct bank groups
SAL_DEVINL int a_stride(int K) { return K + 8; }
SAL_DEVINL int d_stride(int CP) { return CP + 8; }
SAL_DEVINL int l_stride(int CP) { return CP + 4; }
constexpr int kWStride = kChunk + 8;

__host__ __device__ inline size_t smem_bytes(int K, int CP) {
  const size_t a = (size_t)kRows * (K + 8) * 2;
  const size_t l = (size_t)kRows * (CP + 4) * 4;
  const size_t w = (size_t)CP * (kChunk + 8) * 2;
  const size_t d = (size_t)kRows * (CP + 8) * 2;
  return a + (l > w ? l : w) + d;
}

// 16-byte async copy global -> shared (zero-filled when !valid): every load of a
// staging pass is in flight at once instead of one dependent load/store pair per
// thread-iteration (which cost ~50 us of exposed latency per launch, ncu)
SAL_DEVINL void cp16(void* sdst, const void* gsrc, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sdst)),
               "l"(gsrc), "r"(valid ? 16 : 0)
               : "memory");
}
SAL_DEVINL void cp_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
}

// W[0:c_pad, c0:c0+cw] -> Wc [CP][kWStride] (rows >= c_pad and columns >= cw zero);
// the caller waits (cp_wait_all) and synchronises
SAL_DEVINL void stage_w(const __nv_bfloat16* __restrict__ W, int K, int c_pad, int CP, int c0,
                        int cw, __nv_bfloat16* Wc) {
  for (int q = threadIdx.x; q < CP * (kChunk / 8); q += kThreads) {
    const int k = q / (kChunk / 8), c = (q % (kChunk / 8)) * 8;
    const bool ok = k < c_pad && c < cw;
    cp16(Wc + k * kWStride + c, ok ? (const void*)(W + (int64_t)k * K + c0 + c) : (const void*)W,
         ok);
  }
}

__global__ void __launch_bounds__(kThreads)
sage_head_kernel(const __nv_bfloat16* __restrict__ act, int64_t lda, int f, int n_rows,
                 const __nv_bfloat16* __restrict__ W,
                 int C, int c_pad, int CP, const int64_t* __restrict__ labels, int n_labels,
                 float* __restrict__ loss, float* __restrict__ dW, int64_t lddw,
                 __nv_bfloat16* __restrict__ dA, int64_t ldda) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int K = 2 * f;
  const int as = a_stride(K), ds = d_stride(CP), ls = l_stride(CP);
  __nv_bfloat16* As = reinterpret_cast<__nv_bfloat16*>(smem);
  uint8_t* mid = smem + (size_t)kRows * as * 2;
  float* Ls = reinterpret_cast<float*>(mid);
  __nv_bfloat16* Wc = reinterpret_cast<__nv_bfloat16*>(mid);
  const size_t lbytes = (size_t)kRows * ls * 4, wbytes = (size_t)CP * kWStride * 2;
  __nv_bfloat16* Ds = reinterpret_cast<__nv_bfloat16*>(mid + (lbytes > wbytes ? lbytes : wbytes));
  __shared__ int sh_cnt[kWarps];
  __shared__ float sh_loss[kWarps];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = blockIdx.x * kRows;

  // valid labels over the whole batch (lsm_nll: mean over rows with label >= 0)
  int cnt = 0;
  for (int i = threadIdx.x; i < n_labels; i += kThreads) cnt += labels[i] >= 0;
  cnt = warp_reduce_sum(cnt);
  if (lane == 0) sh_cnt[warp] = cnt;

  // 1. A tile = the layer's cat rows [mean | h_dst] (the mean was written by the
  //    segment-mean kernel before this one): 64 rows, 16-byte coalesced loads
  for (int q = threadIdx.x; q < kRows * (K / 8); q += kThreads) {
    const int r = q / (K / 8), c = (q % (K / 8)) * 8;
    const int R = r0 + r;
    cp16(As + (size_t)r * as + c, R < n_rows ? (const void*)(act + (int64_t)R * lda + c)
                                             : (const void*)act, R < n_rows);
  }
  cp_wait_all();
  __syncthreads();
  int total = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) total += sh_cnt[w];
  const float inv_cnt = 1.f / (float)(total > 0 ? total : 1);

  // warp w: m-tile (w & 3) = rows 16*(w&3).., half (w >> 2) of the n-tiles
  const int m0 = (warp & 3) * 16;
  const int half = warp >> 2;

  // 2. logits: W staged in smem 128 K-columns at a time (the Ls / Wc region);
  //    each warp keeps the accumulators of its half of the n-tiles
  const uint32_t a_base = smem_u32(As + (size_t)(m0 + (lane & 15)) * as + (lane >> 4) * 8);
  constexpr int kMaxNT = 16;   // CP <= 256 -> <= 32 n-tiles, half each
  const int ntc = CP / 8, nt_lo = half * ((ntc + 1) / 2), nt_hi = min(ntc, nt_lo + (ntc + 1) / 2);
  float acc2[kMaxNT][4];
#pragma unroll
  for (int j = 0; j < kMaxNT; ++j) acc2[j][0] = acc2[j][1] = acc2[j][2] = acc2[j][3] = 0.f;
  for (int c0 = 0; c0 < K; c0 += kChunk) {
    const int cw = min(kChunk, K - c0);
    stage_w(W, K, c_pad, CP, c0, cw, Wc);
    cp_wait_all();
    __syncthreads();
    for (int k0 = 0; k0 < cw; k0 += 16) {
      uint32_t a[4];
      ldsm_x4(a_base + (c0 + k0) * 2, a);
      uint32_t b[kMaxNT][2];
#pragma unroll
      for (int j = 0; j < kMaxNT; ++j)  // all B fragments first, then the MMAs
        if (nt_lo + j < nt_hi)
          ldsm_x2(smem_u32(Wc + ((nt_lo + j) * 8 + (lane & 7)) * kWStride + k0 +
                           8 * ((lane >> 3) & 1)), b[j]);
#pragma unroll
      for (int j = 0; j < kMaxNT; ++j)
        if (nt_lo + j < nt_hi) mma16816(acc2[j], a, b[j]);
    }
    __syncthreads();  // chunk consumed before the next one (or Ls) overwrites it
  }
#pragma unroll
  for (int j = 0; j < kMaxNT; ++j) {
    if (nt_lo + j < nt_hi) {
      const int col = (nt_lo + j) * 8 + 2 * t;
      Ls[(m0 + g) * ls + col] = acc2[j][0];
      Ls[(m0 + g) * ls + col + 1] = acc2[j][1];
      Ls[(m0 + g + 8) * ls + col] = acc2[j][2];
      Ls[(m0 + g + 8) * ls + col + 1] = acc2[j][3];
    }
  }
  __syncthreads();

  // 3. log_softmax + NLL and dlogits: warp w takes rows 8w .. 8w+7
  float wloss = 0.f;
  for (int rr = 0; rr < kRows / kWarps; ++rr) {
    const int r = warp * (kRows / kWarps) + rr, R = r0 + r;
    const float* x = Ls + r * ls;
    const int64_t lab = R < n_labels ? labels[R] : -1;
    float mx = -INFINITY;
    for (int j = lane; j < C; j += 32) mx = fmaxf(mx, x[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.f;
    for (int j = lane; j < C; j += 32) se += __expf(x[j] - mx);
    se = warp_reduce_sum(se);
    const float lse = mx + __logf(se);
    __nv_bfloat16* drow = Ds + (size_t)r * ds;
    for (int j = lane; j < CP; j += 32) {
      float d = 0.f;
      if (lab >= 0 && j < C) d = (__expf(x[j] - lse) - (j == lab ? 1.f : 0.f)) * inv_cnt;
      drow[j] = __float2bfloat16_rn(d);
    }
    if (lane == 0 && lab >= 0) wloss += (lse - x[lab]) * inv_cnt;
  }
  if (lane == 0) sh_loss[warp] = wloss;
  __syncthreads();  // Ds complete; Ls dead (the region becomes the W chunk buffer)
  if (threadIdx.x == 0) {
    float l = 0.f;
    for (int w = 0; w < kWarps; ++w) l += sh_loss[w];
    if (l != 0.f) atomicAdd(loss, l);
  }

  // 4. dA = D @ W: per 128-column chunk, warp w computes rows m0.. x 8 n-tiles
  const uint32_t d_base = smem_u32(Ds + (size_t)(m0 + (lane & 15)) * ds + (lane >> 4) * 8);
  for (int c0 = 0; c0 < K; c0 += kChunk) {
    const int cw = min(kChunk, K - c0);
    stage_w(W, K, c_pad, CP, c0, cw, Wc);
    cp_wait_all();
    __syncthreads();
    constexpr int kNT4 = kChunk / 16;   // 8 n-tiles per warp
    float acc[kNT4][4];
#pragma unroll
    for (int j = 0; j < kNT4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    for (int k0 = 0; k0 < CP; k0 += 16) {
      uint32_t a[4];
      ldsm_x4(d_base + k0 * 2, a);
      uint32_t b[kNT4][2];
#pragma unroll
      for (int j = 0; j < kNT4; ++j)
        ldsm_x2_t(smem_u32(Wc + (k0 + (lane & 15)) * kWStride + (half * kNT4 + j) * 8), b[j]);
#pragma unroll
      for (int j = 0; j < kNT4; ++j) mma16816(acc[j], a, b[j]);
    }
#pragma unroll
    for (int j = 0; j < kNT4; ++j) {
      const int cc = (half * kNT4 + j) * 8;
      if (cc >= cw) break;
      const int col = c0 + cc + 2 * t;
      const int Ra = r0 + m0 + g, Rb = Ra + 8;
      if (Ra < n_rows)
        *reinterpret_cast<uint32_t*>(dA + (int64_t)Ra * ldda + col) = pack_bf16(acc[j][0], acc[j][1]);
      if (Rb < n_rows)
        *reinterpret_cast<uint32_t*>(dA + (int64_t)Rb * ldda + col) = pack_bf16(acc[j][2], acc[j][3]);
    }
    __syncthreads();  // all warps done with this W chunk
  }

  // 5. dW += D^T @ A over the block's 64 rows: warp w takes n-tiles w, w+8, ...
  //    (4 at a time), all m-tiles of the classes
  for (int mt = 0; mt < CP / 16; ++mt) {
    const int cm = mt * 16;
    // A operand = D^T: 8x8 blocks of Ds transposed (rows of Ds are the K dim)
    const uint32_t dt_base =
        smem_u32(Ds + (size_t)((lane & 7) + 8 * (lane >> 4)) * ds + cm + 8 * ((lane >> 3) & 1));
    uint32_t at[kRows / 16][4];
#pragma unroll
    for (int kk = 0; kk < kRows / 16; ++kk) ldsm_x4_t(dt_base + (uint32_t)(kk * 16 * ds * 2), at[kk]);
    for (int nt = warp; nt < K / 8; nt += kWarps * 4) {
      float acc[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < kRows / 16; ++kk) {
        uint32_t b[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ntj = nt + j * kWarps;
          if (ntj < K / 8)
            ldsm_x2_t(smem_u32(As + (size_t)(kk * 16 + (lane & 15)) * as + ntj * 8), b[j]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (nt + j * kWarps < K / 8) mma16816(acc[j], at[kk], b[j]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ntj = nt + j * kWarps;
        if (ntj >= K / 8) break;
        const int col = ntj * 8 + 2 * t;
        const int ra = cm + g, rb = ra + 8;
        if (ra < c_pad) red_add_v2(dW + (int64_t)ra * lddw + col, acc[j][0], acc[j][1]);
        if (rb < c_pad) red_add_v2(dW + (int64_t)rb * lddw + col, acc[j][2], acc[j][3]);
      }
    }
  }
}

}  // namespace head
}  // namespace sal

extern "C" {

int sal_sage_head(const void* act, int64_t lda, int32_t f, int64_t n_rows, const void* W,
                  int32_t num_classes, int32_t c_pad, const int64_t* labels, int64_t n_labels,
                  float* loss, float* dW, int64_t lddw, void* dA, int64_t ldda, void* stream) {
  if (!act || !W || !labels || !loss || !dW || !dA) return SAL_EINVAL;
  const int K = 2 * f;
  const int CP = (c_pad + 15) / 16 * 16;
  if (f <= 0 || f % 8 || K > 512 || num_classes <= 0 || num_classes > c_pad || c_pad % 8 ||
      CP > 256 || lda % 8 || ldda % 8 || lddw % 2 || ((uintptr_t)act & 15) ||
      ((uintptr_t)W & 15) || ((uintptr_t)dA & 3))
    return SAL_EINVAL;
  if (n_rows <= 0) return SAL_OK;
  const size_t smem = sal::head::smem_bytes(K, CP);
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(sal::head::sage_head_kernel,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SAL_ECUDA;
    attr = smem;
  }
  const int grid = (int)((n_rows + sal::head::kRows - 1) / sal::head::kRows);
  sal::head::sage_head_kernel<<<grid, sal::head::kThreads, smem, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)act, lda, f, (int)n_rows, (const __nv_bfloat16*)W, num_classes, c_pad, CP, labels, (int)n_labels, loss, dW, lddw,
      (__nv_bfloat16*)dA, ldda);
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
}

}  // extern "C"
