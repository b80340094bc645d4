// On-device synthetic graph generator.
//
// Same law as the reference's synth_graph (graph.py:252-280): Pareto degree
// sequence, stubs paired uniformly at random (configuration model, self
// loops and multi-edges kept), every pair stored in both directions.  The
// host generator needs ~15 min and ~100 GB of RAM at papers100M shape; here
// the pairing is a pseudo-random bijection of the stub index space (a
// cycle-walking Feistel network), so stub s is paired with
//     partner(s) = P(P^-1(s) xor 1)
// and indices[s] = owner(partner(s)) — one gather, no sort.  With slot s of
// node v stored at row position s - indptr[v], indptr is simply the exclusive
// scan of the degrees.
//
// Every draw is counter-based (Philox4x32-10 on the node / row index, Feistel
// keys from splitmix64 of the seed) and every float step is exactly rounded
// (sqrt and division at exponent 3, exact fp16 rounding of 24-bit uniforms),
// so oracle/oracle.c regenerates the identical graph on the host
// (orc_synth_*): the reference arm of bench.py builds its inputs without this
// library, and tests/test_gpu_generate.py checks the two bit for bit.
#include "common.cuh"
#include "salient_internal.h"

namespace sal {

struct Feistel {
  int half_bits;
  uint32_t half_mask;
  uint32_t keys[6];
};

SAL_DEVINL uint32_t feistel_f(uint32_t x, uint32_t k) {
  uint32_t h = x ^ k;
  h ^= h >> 16;
  h *= 0x7feb352du;
  h ^= h >> 15;
  h *= 0x846ca68bu;
  h ^= h >> 16;
  return h;
}

SAL_DEVINL uint64_t feistel_fwd(const Feistel& F, uint64_t x) {
  uint32_t L = (uint32_t)(x >> F.half_bits), R = (uint32_t)x & F.half_mask;
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    const uint32_t nl = R;
    R = (L ^ feistel_f(R, F.keys[r])) & F.half_mask;
    L = nl;
  }
  return ((uint64_t)L << F.half_bits) | R;
}

SAL_DEVINL uint64_t feistel_inv(const Feistel& F, uint64_t y) {
  uint32_t L = (uint32_t)(y >> F.half_bits), R = (uint32_t)y & F.half_mask;
#pragma unroll
  for (int r = 5; r >= 0; --r) {
    const uint32_t nr = L;
    L = (R ^ feistel_f(L, F.keys[r])) & F.half_mask;
    R = nr;
  }
  return ((uint64_t)L << F.half_bits) | R;
}

SAL_DEVINL uint64_t perm_fwd(const Feistel& F, uint64_t x, uint64_t n) {
  do { x = feistel_fwd(F, x); } while (x >= n);
  return x;
}

SAL_DEVINL uint64_t perm_inv(const Feistel& F, uint64_t y, uint64_t n) {
  do { y = feistel_inv(F, y); } while (y >= n);
  return y;
}

// Pareto degrees: deg(v) = rint(scale * (1 - u)^(-1/a)) clipped to [0, n-1]
// with u = 53-bit uniform of Philox((v, v>>32, 0, 5), key(seed)); numpy's
// 1 + pareto(a) is (1 - u)^(-1/a) (graph.py:270).  a == 2 (exponent 3, every
// configuration here) uses 1 / sqrt: both correctly rounded, so the host
// restatement is bit-exact; other exponents go through pow.
__global__ void degrees_kernel(int64_t n, uint64_t seed, double scale, double a,
                               int64_t* __restrict__ degs) {
  const uint2 key = make_uint2((uint32_t)seed ^ 0xDE6u, (uint32_t)(seed >> 32));
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint4 r = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(v >> 32), 0u, 5u), key);
    const uint64_t bits53 = (((uint64_t)r.x << 21) ^ ((uint64_t)r.y >> 11)) & ((1ull << 53) - 1);
    const double w = 1.0 - (double)bits53 * 0x1.0p-53;   // (0, 1], exact
    const double y = a == 2.0 ? 1.0 / sqrt(w) : pow(w, -1.0 / a);
    double d = rint(scale * y);
    if (d > (double)(n - 1)) d = (double)(n - 1);
    if (d < 0.0) d = 0.0;
    degs[v] = (int64_t)d;
  }
}

__global__ void owner_kernel(const int64_t* __restrict__ indptr, int64_t n,
                             int32_t* __restrict__ owner) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = indptr[v], hi = indptr[v + 1];
    for (int64_t s = lo; s < hi; ++s) owner[s] = (int32_t)v;
  }
}

__global__ void pairing_kernel(const int32_t* __restrict__ owner, int64_t n_stubs, Feistel F,
                               int32_t* __restrict__ indices) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_stubs;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t q = perm_inv(F, (uint64_t)s, (uint64_t)n_stubs);
    const uint64_t p = perm_fwd(F, q ^ 1ull, (uint64_t)n_stubs);
    indices[s] = owner[p];
  }
}

// uniform [-1, 1) features rounded to fp16 (graph.py:283-292 law)
__global__ void features_kernel(int64_t n, int32_t f, int64_t stride, uint64_t seed,
                                __half* __restrict__ out) {
  const int64_t quads_per_row = (f + 3) / 4;
  const int64_t total = n * quads_per_row;
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32) ^ 0xF3A7u);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = q / quads_per_row;
    const int c = (int)(q - row * quads_per_row) * 4;
    const uint4 r = philox4x32_10(make_uint4((uint32_t)row, (uint32_t)(row >> 32), (uint32_t)c, 7u), key);
    const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
    __half h[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __float2half_rn(-1.0f + 2.0f * ((rr[j] >> 8) * (1.0f / 16777216.0f)));
    __half* dst = out + row * stride + c;
    if (c + 4 <= f && ((uintptr_t)dst & 7) == 0) {
      *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(h);
    } else {
      for (int j = 0; j < 4 && c + j < f; ++j) dst[j] = h[j];
    }
  }
}

__global__ void labels_kernel(int64_t n, int32_t num_classes, uint64_t seed,
                              int64_t* __restrict__ out) {
  const uint2 key = make_uint2((uint32_t)seed ^ 0x1ABE1u, (uint32_t)(seed >> 32));
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint4 r = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(v >> 32), 0u, 11u), key);
    out[v] = (int64_t)(((uint64_t)r.x * (uint32_t)num_classes) >> 32);
  }
}

static int gen_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace sal

extern "C" {

int sal_gen_degrees(int64_t n, uint64_t seed, double scale, double a, int64_t* degs,
                    void* stream) {
  if (n < 0 || !(a > 1.0) || !(scale >= 0.0))
    return sal::set_error(SAL_EINVAL, "gen_degrees: invalid argument (n < 0 || !(a > 1.0) || !(scale >= 0.0))");
  if (n == 0) return SAL_OK;
  sal::degrees_kernel<<<sal::gen_grid(n), 256, 0, (cudaStream_t)stream>>>(n, seed, scale, a,
                                                                           degs);
  return cudaGetLastError() == cudaSuccess ? SAL_OK : SAL_ECUDA;
}

int sal_gen_owner(const int64_t* indptr, int64_t n, int32_t* owner, void* stream) {
  sal::owner_kernel<<<sal::gen_grid(n), 256, 0, (cudaStream_t)stream>>>(indptr, n, owner);
  return cudaGetLastError() == cudaSuccess ? SAL_OK : SAL_ECUDA;
}

int sal_gen_pairing(const int32_t* owner, int64_t n_stubs, uint64_t seed, int32_t* indices,
                    void* stream) {
  if (n_stubs % 2 != 0)
    return sal::set_error(SAL_EINVAL, "gen_pairing: invalid argument (n_stubs % 2 != 0)");
  sal::Feistel F;
  int bits = 2;
  while ((1ull << bits) < (uint64_t)n_stubs) ++bits;
  if (bits & 1) ++bits;
  F.half_bits = bits / 2;
  F.half_mask = (uint32_t)((1ull << F.half_bits) - 1);
  uint64_t k = seed;
  for (int r = 0; r < 6; ++r) {
    k = sal::mix64_hd(k + sal::kGolden);
    F.keys[r] = (uint32_t)k;
  }
  sal::pairing_kernel<<<sal::gen_grid(n_stubs), 256, 0, (cudaStream_t)stream>>>(owner, n_stubs, F,
                                                                             indices);
  return cudaGetLastError() == cudaSuccess ? SAL_OK : SAL_ECUDA;
}

int sal_gen_features_uniform(int64_t n, int32_t f, int64_t stride, uint64_t seed, void* out,
                             void* stream) {
  const int64_t quads = n * ((f + 3) / 4);
  sal::features_kernel<<<sal::gen_grid(quads), 256, 0, (cudaStream_t)stream>>>(
      n, f, stride, seed, (__half*)out);
  return cudaGetLastError() == cudaSuccess ? SAL_OK : SAL_ECUDA;
}

int sal_gen_labels_uniform(int64_t n, int32_t num_classes, uint64_t seed, int64_t* out,
                           void* stream) {
  sal::labels_kernel<<<sal::gen_grid(n), 256, 0, (cudaStream_t)stream>>>(n, num_classes, seed,
                                                                          out);
  return cudaGetLastError() == cudaSuccess ? SAL_OK : SAL_ECUDA;
}

}  // extern "C"
