// Feature / label slicing (prep.py:153-182; _kernels.py:225-258).
//
// out[i, :] = convert(X[ids[i], :]) — an HBM-bound row gather.  Each thread
// moves whole vectors (16 B when the row stride allows it, else 8/4/2 B),
// keeps kUnroll independent vectors in flight (ids first, then rows, then
// stores) and streams through L1 (ld.global.nc.L1::no_allocate).  Rows are
// flattened into (row, chunk) items so a warp covers two 256 B rows per
// instruction at f = 128 fp16.
//
// fp16 -> fp32 is exact; NaNs are canonicalised to 0x7FC00000 exactly as the
// reference's scalar _half_to_f32 does (_kernels.py:240-242: np.float32(nan)).
#include <cstdlib>
#include <cuda_bf16.h>

#include "common.cuh"
#include "salient_internal.h"

namespace sal {

template <int N> struct VecT;
template <> struct VecT<2> { typedef unsigned short T; };
template <> struct VecT<4> { typedef unsigned int T; };
template <> struct VecT<8> { typedef uint2 T; };
template <> struct VecT<16> { typedef uint4 T; };

template <int N>
SAL_DEVINL void load_vec(const void* p, void* dst) {
  typedef typename VecT<N>::T T;
  if (N == 16) {
    *reinterpret_cast<int4*>(dst) = ld_stream_v4(reinterpret_cast<const int4*>(p));
  } else {
    *reinterpret_cast<T*>(dst) = __ldg(reinterpret_cast<const T*>(p));
  }
}

template <int N>
SAL_DEVINL void store_vec(void* p, const void* src) {
  typedef typename VecT<N>::T T;
  *reinterpret_cast<T*>(p) = *reinterpret_cast<const T*>(src);
}

template <typename T> struct Elem;
template <> struct Elem<__half> {
  static SAL_DEVINL float to_f(__half v) { return __half2float(v); }
};
template <> struct Elem<__nv_bfloat16> {
  static SAL_DEVINL float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
};
template <> struct Elem<float> {
  static SAL_DEVINL float to_f(float v) { return v; }
};

template <typename TIn, typename TOut>
SAL_DEVINL TOut convert(TIn v);
template <> SAL_DEVINL __half convert<__half, __half>(__half v) { return v; }
template <> SAL_DEVINL float convert<float, float>(float v) { return v; }
template <> SAL_DEVINL __nv_bfloat16 convert<__nv_bfloat16, __nv_bfloat16>(__nv_bfloat16 v) {
  return v;
}
template <> SAL_DEVINL float convert<__half, float>(__half v) {
  const float f = __half2float(v);
  return (f != f) ? __int_as_float(0x7FC00000) : f;
}
template <> SAL_DEVINL float convert<__nv_bfloat16, float>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <> SAL_DEVINL __nv_bfloat16 convert<__half, __nv_bfloat16>(__half v) {
  return __float2bfloat16_rn(__half2float(v));
}
template <> SAL_DEVINL __nv_bfloat16 convert<float, __nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <> SAL_DEVINL __half convert<float, __half>(float v) { return __float2half_rn(v); }

constexpr int kGatherThreads = 256;
constexpr int kUnroll = 4;

template <typename TIn, typename TOut, int VIN, typename TId>
__global__ void __launch_bounds__(kGatherThreads)
gather_rows_kernel(const TIn* __restrict__ x, int64_t x_stride, const TId* __restrict__ ids,
                   const int64_t* __restrict__ n_dev, int64_t n_host, int32_t cpr,
                   TOut* __restrict__ out, int64_t out_stride) {
  constexpr int EPV = VIN / (int)sizeof(TIn);          // elements per vector
  constexpr int VOUT = EPV * (int)sizeof(TOut);        // output bytes per vector
  const int64_t n = n_dev ? *n_dev : n_host;
  const int64_t items = n * cpr;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; it < items; it += stride * kUnroll) {
    TIn buf[kUnroll][EPV];
    int64_t orow[kUnroll];
    int ochunk[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t k = it + u * stride;
      orow[u] = -1;
      if (k < items) {
        const int64_t r = k / cpr;
        const int c = (int)(k - r * cpr);
        const int64_t src = (int64_t)ids[r];
        orow[u] = r;
        ochunk[u] = c;
        load_vec<VIN>(x + src * x_stride + (int64_t)c * EPV, buf[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (orow[u] >= 0) {
        TOut o[EPV];
#pragma unroll
        for (int j = 0; j < EPV; ++j) o[j] = convert<TIn, TOut>(buf[u][j]);
        TOut* dst = out + orow[u] * out_stride + (int64_t)ochunk[u] * EPV;
        if (VOUT <= 16) {
          store_vec<(VOUT <= 16 ? VOUT : 16)>(dst, o);
        } else {
#pragma unroll
          for (int q = 0; q < VOUT / 16; ++q) store_vec<16>((char*)dst + 16 * q, (char*)o + 16 * q);
        }
      }
    }
  }
}

// Warp-row variant for rows of LPR x 16 B (LPR divides 32): a warp moves
// 32/LPR rows per instruction and keeps kRowUnroll such instructions in flight
// (each lane group loads its own row id — the group's lanes hit the same word,
// one L1 transaction).  This is the access pattern that reaches ~5.7 TB/s
// (88% of the measured copy peak) for random 256 B rows on B200 in
// tools/randread_bench.cu, the same as a sequential copy of equal size.
constexpr int kRowUnroll = 8;

template <typename TIn, typename TOut, int LPR, typename TId>
__global__ void __launch_bounds__(kGatherThreads, 4)
gather_rows_warp_kernel(const TIn* __restrict__ x, int64_t x_stride, const TId* __restrict__ ids,
                        const int64_t* __restrict__ n_dev, int64_t n_host, TOut* __restrict__ out,
                        int64_t out_stride) {
  constexpr int EPV = 16 / (int)sizeof(TIn);
  constexpr int VOUT = EPV * (int)sizeof(TOut);
  constexpr int RPI = 32 / LPR;
  constexpr int kStep = RPI * kRowUnroll;  // rows per warp iteration
  const int lane = threadIdx.x & 31;
  const int grp = lane / LPR, sub = lane % LPR;
  // row indices fit in int32 (a batch holds < 2^31 rows); only the table
  // offset needs 64 bits
  const int n = (int)(n_dev ? *n_dev : n_host);
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  for (int r0 = warp * kStep; r0 < n; r0 += nwarps * kStep) {
    uint4 buf[kRowUnroll];
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) {
      const int r = r0 + u * RPI + grp;
      if (r < n) {
        const TIn* row = x + (int64_t)ids[r] * x_stride;
        const int4 t = ld_stream_v4(reinterpret_cast<const int4*>(row) + sub);
        buf[u] = make_uint4((unsigned)t.x, (unsigned)t.y, (unsigned)t.z, (unsigned)t.w);
      }
    }
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) {
      const int r = r0 + u * RPI + grp;
      if (r < n) {
        const TIn* v = reinterpret_cast<const TIn*>(&buf[u]);
        TOut o[EPV];
#pragma unroll
        for (int j = 0; j < EPV; ++j) o[j] = convert<TIn, TOut>(v[j]);
        TOut* dst = out + (int64_t)r * out_stride + sub * EPV;
#pragma unroll
        for (int q = 0; q < (VOUT + 15) / 16; ++q) {
          if (VOUT >= 16)
            store_vec<16>((char*)dst + 16 * q, (char*)o + 16 * q);
          else
            store_vec<(VOUT < 16 ? VOUT : 16)>(dst, o);
        }
      }
    }
  }
}

template <typename TIn, typename TOut, typename TId>
static cudaError_t gather_dispatch(const void* x, int32_t cols, int64_t x_stride, const void* ids,
                                   const int64_t* n_dev, int64_t n, void* out,
                                   int64_t out_stride, cudaStream_t st) {
  // widest input vector that divides the row length, both strides and the
  // base pointers' alignment
  const int64_t in_row_bytes = (int64_t)cols * sizeof(TIn);
  int vin = 16;
  while (vin > (int)sizeof(TIn)) {
    const int vout = vin / (int)sizeof(TIn) * (int)sizeof(TOut);
    const bool ok = in_row_bytes % vin == 0 && (x_stride * (int64_t)sizeof(TIn)) % vin == 0 &&
                    ((uintptr_t)x % vin) == 0 &&
                    (out_stride * (int64_t)sizeof(TOut)) % (vout < 16 ? vout : 16) == 0 &&
                    ((uintptr_t)out % (vout < 16 ? vout : 16)) == 0;
    if (ok) break;
    vin >>= 1;
  }
  const int32_t cpr = (int32_t)(in_row_bytes / vin);
  if (vin == 16 && cpr <= 32 && (32 % cpr) == 0 && (int)sizeof(TIn) <= 16) {
    // whole rows per warp: the fast path for 16 B-aligned rows (f = 128 fp16 -> 16 lanes)
    const int64_t warps = (n + (32 / cpr) * kRowUnroll - 1) / ((32 / cpr) * kRowUnroll);
    int64_t wgrid = (warps + 7) / 8;
    const int64_t wcap = (int64_t)num_sms() * 8;
    if (wgrid > wcap) wgrid = wcap;
    if (wgrid < 1) wgrid = 1;
#define SAL_GW_CASE(L)                                                                       \
  case L:                                                                                    \
    gather_rows_warp_kernel<TIn, TOut, L, TId><<<(int)wgrid, kGatherThreads, 0, st>>>(        \
        (const TIn*)x, x_stride, (const TId*)ids, n_dev, n, (TOut*)out, out_stride);         \
    return cudaGetLastError();
    switch (cpr) {
      SAL_GW_CASE(1)
      SAL_GW_CASE(2)
      SAL_GW_CASE(4)
      SAL_GW_CASE(8)
      SAL_GW_CASE(16)
      SAL_GW_CASE(32)
    }
#undef SAL_GW_CASE
  }
  const int64_t max_items = n * (int64_t)cpr;
  int64_t grid = (max_items + kGatherThreads * kUnroll - 1) / (kGatherThreads * kUnroll);
  const int64_t cap = (int64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  const TIn* xp = (const TIn*)x;
  TOut* op = (TOut*)out;
  const TId* ip = (const TId*)ids;
#define SAL_GATHER_CASE(V)                                                              \
  case V:                                                                               \
    gather_rows_kernel<TIn, TOut, (V >= (int)sizeof(TIn) ? V : (int)sizeof(TIn)), TId> \
        <<<(int)grid, kGatherThreads, 0, st>>>(xp, x_stride, ip, n_dev, n, cpr, op,     \
                                               out_stride);                            \
    break;
  switch (vin) {
    SAL_GATHER_CASE(16)
    SAL_GATHER_CASE(8)
    SAL_GATHER_CASE(4)
    default:
      SAL_GATHER_CASE(2)
  }
#undef SAL_GATHER_CASE
  return cudaGetLastError();
}

template <typename TIn, typename TOut>
static cudaError_t gather_ids(const void* x, int32_t cols, int64_t x_stride, const void* ids,
                              int32_t id_bytes, const int64_t* n_dev, int64_t n, void* out,
                              int64_t out_stride, cudaStream_t st) {
  if (id_bytes == 4)
    return gather_dispatch<TIn, TOut, int32_t>(x, cols, x_stride, ids, n_dev, n, out, out_stride,
                                               st);
  return gather_dispatch<TIn, TOut, int64_t>(x, cols, x_stride, ids, n_dev, n, out, out_stride,
                                             st);
}

cudaError_t launch_gather_rows(const void* x, int64_t x_rows, int32_t cols, int64_t x_stride,
                               int32_t in_dtype, const void* ids, int32_t id_bytes,
                               const int64_t* n_dev, int64_t n, void* out, int64_t out_stride,
                               int32_t out_dtype, cudaStream_t st) {
  (void)x_rows;
  if (in_dtype == SAL_F16) {
    if (out_dtype == SAL_F32)
      return gather_ids<__half, float>(x, cols, x_stride, ids, id_bytes, n_dev, n, out,
                                       out_stride, st);
    if (out_dtype == SAL_F16)
      return gather_ids<__half, __half>(x, cols, x_stride, ids, id_bytes, n_dev, n, out,
                                        out_stride, st);
    return gather_ids<__half, __nv_bfloat16>(x, cols, x_stride, ids, id_bytes, n_dev, n, out,
                                             out_stride, st);
  }
  if (in_dtype == SAL_F32) {
    if (out_dtype == SAL_F32)
      return gather_ids<float, float>(x, cols, x_stride, ids, id_bytes, n_dev, n, out, out_stride,
                                      st);
    if (out_dtype == SAL_F16)
      return gather_ids<float, __half>(x, cols, x_stride, ids, id_bytes, n_dev, n, out,
                                       out_stride, st);
    return gather_ids<float, __nv_bfloat16>(x, cols, x_stride, ids, id_bytes, n_dev, n, out,
                                            out_stride, st);
  }
  if (out_dtype == SAL_F32)
    return gather_ids<__nv_bfloat16, float>(x, cols, x_stride, ids, id_bytes, n_dev, n, out,
                                            out_stride, st);
  return gather_ids<__nv_bfloat16, __nv_bfloat16>(x, cols, x_stride, ids, id_bytes, n_dev, n,
                                                  out, out_stride, st);
}

// rows [n_seeds, max_n) receive -1 (an ignore_index for a padded loss)
__global__ void gather_labels_kernel(const int64_t* __restrict__ y,
                                     const int64_t* __restrict__ seeds_base,
                                     const BatchDesc* __restrict__ desc, int64_t max_n,
                                     int64_t* __restrict__ out) {
  const int64_t n = desc->n_seeds;
  const int64_t* seeds = seeds_base + desc->seed_offset;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < max_n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < n ? y[seeds[i]] : -1;
}

cudaError_t launch_gather_labels(const int64_t* y, const int64_t* seeds_base,
                                 const BatchDesc* desc, int64_t max_n, int64_t* out,
                                 cudaStream_t st) {
  int64_t grid = (max_n + 255) / 256;
  if (grid < 1) grid = 1;
  if (grid > 1024) grid = 1024;
  gather_labels_kernel<<<(int)grid, 256, 0, st>>>(y, seeds_base, desc, max_n, out);
  return cudaGetLastError();
}

}  // namespace sal
