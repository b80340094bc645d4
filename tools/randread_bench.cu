// Random-row read microbenchmark for the roofline of the row gather and the
// layer-0 segment mean: how fast can B200 HBM3e serve random 256-byte rows?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o randread tools/randread_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <random>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// LPR lanes per 256 B row, U row-instructions in flight; reduce to one word per row
template <int LPR, int U, bool kWrite>
__global__ void __launch_bounds__(256) rows_kernel(const uint4* __restrict__ x, const int* __restrict__ ids,
                                                   int64_t n, uint4* __restrict__ out, unsigned* sink) {
  constexpr int VPL = 16 / LPR;  // 16-byte vectors per lane per row (row = 16 vectors)
  constexpr int RPI = 32 / LPR;
  const int lane = threadIdx.x & 31, grp = lane / LPR, sub = lane % LPR;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned acc = 0;
  for (int64_t r0 = warp * (RPI * U); r0 < n; r0 += nw * RPI * U) {
    uint4 b[U][VPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * RPI + grp;
      if (r < n) {
        const int64_t s = ids[r];
#pragma unroll
        for (int v = 0; v < VPL; ++v) b[u][v] = ldnc(x + s * 16 + sub * VPL + v);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * RPI + grp;
      if (r < n) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          if (kWrite) out[r * 16 + sub * VPL + v] = b[u][v];
          else acc ^= b[u][v].x ^ b[u][v].y ^ b[u][v].z ^ b[u][v].w;
        }
      }
    }
  }
  if (!kWrite && acc == 0x12345678u) *sink = acc;
}

__global__ void seq_copy(const uint4* __restrict__ x, uint4* __restrict__ y, int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = ldnc(x + i);
}

// TMA 1-D bulk copy of each row global -> shared, then bulk store shared -> global
__global__ void __launch_bounds__(128) bulk_kernel(const char* __restrict__ x, const int* __restrict__ ids,
                                                   int64_t n, char* __restrict__ out) {
  constexpr int RB = 256, DEPTH = 32;  // rows per CTA batch
  __shared__ __align__(128) char buf[DEPTH * RB];
  __shared__ __align__(8) unsigned long long bar;
  const int t = threadIdx.x;
  if (t == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"((unsigned)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  unsigned phase = 0;
  for (int64_t r0 = (int64_t)blockIdx.x * DEPTH; r0 < n; r0 += (int64_t)gridDim.x * DEPTH) {
    const int cnt = (int)((n - r0) < DEPTH ? (n - r0) : DEPTH);
    if (t == 0) {
      const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(b), "r"(cnt * RB));
      for (int k = 0; k < cnt; ++k) {
        const char* src = x + (int64_t)ids[r0 + k] * RB;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(buf + k * RB);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(dst), "l"(src), "r"(RB), "r"(b) : "memory");
      }
      asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }"
                   :: "r"(b), "r"(phase));
      for (int k = 0; k < cnt; ++k) {
        const unsigned s = (unsigned)__cvta_generic_to_shared(buf + k * RB);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(out + (r0 + k) * RB), "r"(s), "r"(RB) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      phase ^= 1;
    }
    __syncthreads();
  }
}

int main() {
  const int64_t rows = 111059956, n = 700000;
  const size_t bytes = (size_t)rows * 256;
  char* x; char* out; int* ids; unsigned* sink;
  CK(cudaMalloc(&x, bytes));
  CK(cudaMemset(x, 1, bytes));
  CK(cudaMalloc(&out, (size_t)n * 256 * 4));
  CK(cudaMalloc(&ids, n * 4 * 4));
  CK(cudaMalloc(&sink, 4));
  std::vector<int> h(n * 4);
  std::mt19937_64 g(1);
  for (auto& v : h) v = (int)(g() % rows);
  CK(cudaMemcpy(ids, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  int sms = 148;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* name, double bytes_moved, auto fn) {
    for (int w = 0; w < 3; ++w) fn(w);
    cudaEventRecord(a);
    const int it = 20;
    for (int i = 0; i < it; ++i) fn(i % 4);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / it;
    printf("%-44s %8.1f us  %7.0f GB/s\n", name, us, bytes_moved / (us * 1e-6) / 1e9);
  };
  const double rb = (double)n * 256;
  timeit("seq copy 180MB (r+w)", 2 * rb, [&](int k) { seq_copy<<<sms * 8, 256>>>((const uint4*)x + k * (n * 16), (uint4*)out, n * 16); });
  timeit("gather LPR16 U4 (r+w)", 2 * rb, [&](int k) { rows_kernel<16, 4, true><<<sms * 8, 256>>>((const uint4*)x, ids + k * n, n, (uint4*)out, sink); });
  timeit("gather LPR16 U8 (r+w)", 2 * rb, [&](int k) { rows_kernel<16, 8, true><<<sms * 8, 256>>>((const uint4*)x, ids + k * n, n, (uint4*)out, sink); });
  timeit("gather LPR8 U4 (r+w)", 2 * rb, [&](int k) { rows_kernel<8, 4, true><<<sms * 8, 256>>>((const uint4*)x, ids + k * n, n, (uint4*)out, sink); });
  timeit("gather LPR4 U2 (r+w)", 2 * rb, [&](int k) { rows_kernel<4, 2, true><<<sms * 8, 256>>>((const uint4*)x, ids + k * n, n, (uint4*)out, sink); });
  timeit("read LPR16 U4", rb, [&](int k) { rows_kernel<16, 4, false><<<sms * 8, 256>>>((const uint4*)x, ids + k * n, n, (uint4*)out, sink); });
  timeit("read LPR16 U8", rb, [&](int k) { rows_kernel<16, 8, false><<<sms * 8, 256>>>((const uint4*)x, ids + k * n, n, (uint4*)out, sink); });
  timeit("read LPR8 U4", rb, [&](int k) { rows_kernel<8, 4, false><<<sms * 8, 256>>>((const uint4*)x, ids + k * n, n, (uint4*)out, sink); });
  timeit("read LPR8 U8", rb, [&](int k) { rows_kernel<8, 8, false><<<sms * 8, 256>>>((const uint4*)x, ids + k * n, n, (uint4*)out, sink); });
  timeit("read LPR4 U4", rb, [&](int k) { rows_kernel<4, 4, false><<<sms * 8, 256>>>((const uint4*)x, ids + k * n, n, (uint4*)out, sink); });
  timeit("read LPR16 U8 grid x2", rb, [&](int k) { rows_kernel<16, 8, false><<<sms * 16, 256>>>((const uint4*)x, ids + k * n, n, (uint4*)out, sink); });
  timeit("bulk (TMA 1D) gather 32 rows/CTA", 2 * rb, [&](int k) { bulk_kernel<<<sms * 12, 128>>>(x, ids + k * n, n, out); });
  CK(cudaDeviceSynchronize());
  CK(cudaGetLastError());
  // sorted ids: locality bound
  std::sort(h.begin(), h.begin() + n);
  CK(cudaMemcpy(ids, h.data(), n * 4, cudaMemcpyHostToDevice));
  timeit("read LPR16 U8 sorted ids", rb, [&](int k) { rows_kernel<16, 8, false><<<sms * 8, 256>>>((const uint4*)x, ids, n, (uint4*)out, sink); });
  return 0;
}
