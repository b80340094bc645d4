// Small fused kernels of the GraphSAGE training step:
//   * plan_next      — device-side epoch cursor -> sal_batch_desc (lets one
//                      captured CUDA graph prepare a different batch per replay)
//   * relu_dropout   — y = relu(x) * keep / (1-p); one bit per element records
//                      (x > 0 && keep) for the backward pass
//   * lsm_nll        — log_softmax + NLL (ignore_index -1, mean over valid rows)
//                      fused with its gradient (softmax - onehot) / count
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
template <typename T>
SAL_DEVINL float to_f(T v);
template <> SAL_DEVINL float to_f<float>(float v) { return v; }
template <> SAL_DEVINL float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
SAL_DEVINL T from_f(float v);
template <> SAL_DEVINL float from_f<float>(float v) { return v; }
template <> SAL_DEVINL __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// 8 elements per thread: one byte of the bit mask.
template <typename T>
__global__ void relu_dropout_fwd_kernel(const T* __restrict__ x, T* __restrict__ y,
                                        uint8_t* __restrict__ mask, int64_t n8, float p,
                                        uint64_t seed, const int64_t* __restrict__ salt) {
  const uint32_t thresh = (uint32_t)(p * 65536.0f);
  const float scale = p < 1.f ? 1.f / (1.f - p) : 0.f;
  const uint32_t s = salt ? (uint32_t)*salt : 0u;
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 r = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), s, 0x5EEDu), key);
    const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
    uint8_t bits = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float v = to_f<T>(x[8 * i + j]);
      const uint32_t u16 = (rr[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
      const bool keep = (p <= 0.f) || (u16 >= thresh);
      const bool on = keep && v > 0.f;
      bits |= (uint8_t)on << j;
      y[8 * i + j] = from_f<T>(on ? v * (p > 0.f ? scale : 1.f) : 0.f);
    }
    mask[i] = bits;
  }
}

template <typename TDY, typename TDX>
__global__ void relu_dropout_bwd_kernel(const TDY* __restrict__ dy,
                                        const uint8_t* __restrict__ mask, TDX* __restrict__ dx,
                                        int64_t n8, float p) {
  const float scale = p > 0.f ? (p < 1.f ? 1.f / (1.f - p) : 0.f) : 1.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t bits = mask[i];
    alignas(16) TDY in[8];
    alignas(16) TDX out[8];
#pragma unroll
    for (int q = 0; q < (int)(8 * sizeof(TDY)) / 16; ++q)
      reinterpret_cast<uint4*>(in)[q] = reinterpret_cast<const uint4*>(dy + 8 * i)[q];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      out[j] = from_f<TDX>(((bits >> j) & 1) ? to_f<TDY>(in[j]) * scale : 0.f);
#pragma unroll
    for (int q = 0; q < (int)(8 * sizeof(TDX)) / 16; ++q)
      reinterpret_cast<uint4*>(dx + 8 * i)[q] = reinterpret_cast<const uint4*>(out)[q];
  }
}

// ---------------------------------------------------------------------------
// one warp per row; every block recounts the valid labels (B <= a few K)
template <typename T>
__global__ void lsm_nll_kernel(const T* __restrict__ logits, int64_t ld, int64_t rows, int32_t C,
                               const int64_t* __restrict__ labels, float* __restrict__ loss,
                               T* __restrict__ grad, int64_t ldg) {
  __shared__ float sh_cnt;
  __shared__ int warp_cnt[32];
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
  if (row >= rows) return;
  const T* x = logits + row * ld;
  T* g = grad + row * ldg;
  const int64_t lab = labels[row];
  float m = -INFINITY;
  for (int j = lane; j < C; j += 32) m = fmaxf(m, to_f<T>(x[j]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f;
  for (int j = lane; j < C; j += 32) s += __expf(to_f<T>(x[j]) - m);
  s = warp_reduce_sum(s);
  const float lse = m + __logf(s);
  if (lab < 0) {
    for (int j = lane; j < C; j += 32) g[j] = from_f<T>(0.f);
    return;
  }
  for (int j = lane; j < C; j += 32) {
    const float pj = __expf(to_f<T>(x[j]) - lse);
    g[j] = from_f<T>((pj - (j == lab ? 1.f : 0.f)) * inv);
  }
  if (lane == 0) atomicAdd(loss, (lse - to_f<T>(x[lab])) * inv);
}

static int ew_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace sal

extern "C" {

int sal_plan_next(const int64_t* desc_all, int64_t n_steps, int64_t* cursor, sal_batch_desc* out,
                  void* stream) {
  sal::plan_next_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(desc_all, n_steps, cursor, out);
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
}

int sal_relu_dropout_fwd(const void* x, void* y, uint8_t* mask, int64_t n, int32_t dtype, float p,
                         uint64_t seed, const int64_t* salt_dev, void* stream) {
  if (n % 8 != 0) return SAL_EINVAL;
  const int64_t n8 = n / 8;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SAL_BF16)
    sal::relu_dropout_fwd_kernel<__nv_bfloat16><<<sal::ew_grid(n8), 256, 0, st>>>(
        (const __nv_bfloat16*)x, (__nv_bfloat16*)y, mask, n8, p, seed, salt_dev);
  else if (dtype == SAL_F32)
    sal::relu_dropout_fwd_kernel<float><<<sal::ew_grid(n8), 256, 0, st>>>(
        (const float*)x, (float*)y, mask, n8, p, seed, salt_dev);
  else
    return SAL_EINVAL;
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
}

int sal_relu_dropout_bwd(const void* dy, int32_t dy_dtype, const uint8_t* mask, void* dx,
                         int32_t dx_dtype, int64_t n, float p, void* stream) {
  if (n % 8 != 0) return SAL_EINVAL;
  const int64_t n8 = n / 8;
  cudaStream_t st = (cudaStream_t)stream;
  const int g = sal::ew_grid(n8);
  if (dy_dtype == SAL_F32 && dx_dtype == SAL_BF16)
    sal::relu_dropout_bwd_kernel<float, __nv_bfloat16><<<g, 256, 0, st>>>(
        (const float*)dy, mask, (__nv_bfloat16*)dx, n8, p);
  else if (dy_dtype == SAL_BF16 && dx_dtype == SAL_BF16)
    sal::relu_dropout_bwd_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, st>>>(
        (const __nv_bfloat16*)dy, mask, (__nv_bfloat16*)dx, n8, p);
  else if (dy_dtype == SAL_F32 && dx_dtype == SAL_F32)
    sal::relu_dropout_bwd_kernel<float, float><<<g, 256, 0, st>>>((const float*)dy, mask,
                                                                 (float*)dx, n8, p);
  else
    return SAL_EINVAL;
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
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
    return SAL_EINVAL;
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
}

}  // extern "C"
