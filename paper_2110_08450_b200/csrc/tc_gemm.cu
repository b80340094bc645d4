// Hand-written tcgen05 GEMMs for the SAGEConv layers (sm_100a).
//
// Forward:  y = relu_dropout( A[M, K] @ W[N, K]^T )  with A a "cat" buffer
//           [mean | h_dst] (bf16, K = 2f = 256 at layer 0, 512 at the hidden
//           layer) and W = [W_neigh | W_self] (N = 256).  Production kernel
//           (sage_fwd_tma_st_kernel<BN, K>): one CTA per SM and 128-column
//           block (grid.y), persistent over 128-row tiles; warp 0 streams A
//           K-blocks with TMA into a SWIZZLE_128B ring (8 stages at K = 256, 4
//           at K = 512) while the CTA's W block stays resident (loaded once);
//           warp 1 issues tcgen05.mma (M=128, N=BN, K=16) into one of two TMEM
//           accumulators; 16 epilogue warps
//           drain TMEM (tcgen05.ld 32x32b), apply ReLU + dropout, stage bf16
//           32x32 chunks in shared memory and write them with TMA bulk tensor
//           stores, plus the keep/relu bit mask — the GEMM output never
//           round-trips through HBM.  sage_fwd_kernel is the single-warpgroup
//           cp.async version kept as a reference point (tools/tc_bench.py).
//
// Weight gradient: dW[N, K] += dz[M, N]^T @ A[M, K] with both operands read
//           MN-major (row-major in HBM): each CTA reduces a contiguous range of
//           M rows into two TMEM accumulators (N = 2 x 128 rows of dW, 256
//           columns each) and adds its partial into the fp32 gradient with
//           vector atomics.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "salient_internal.h"

namespace sal {
namespace tc {

SAL_DEVINL uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor (cute/arch/mma_sm100_desc.hpp SmemDescriptor)
SAL_DEVINL uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                              uint32_t layout /*2 = SWIZZLE_128B*/) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, M x N, majors
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_mn_major, int b_mn_major) {
  return (1u << 4)                         // c_format = F32
         | (1u << 7)                       // a_format = BF16
         | (1u << 10)                      // b_format = BF16
         | ((uint32_t)a_mn_major << 15)    // a_major
         | ((uint32_t)b_mn_major << 16)    // b_major
         | ((uint32_t)(N >> 3) << 17)      // n_dim
         | ((uint32_t)(M >> 4) << 24);     // m_dim
}

SAL_DEVINL void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

SAL_DEVINL void mma_commit(void* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(mbar))
               : "memory");
}

SAL_DEVINL void mbar_init(void* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count));
}

SAL_DEVINL void mbar_wait(void* mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW%=:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W%=;\n\t}\n" ::"r"(
          smem_u32(mbar)),
      "r"(phase)
      : "memory");
}

SAL_DEVINL void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
SAL_DEVINL void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
SAL_DEVINL void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

SAL_DEVINL void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
SAL_DEVINL void cp_async_zero16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;" ::"r"(saddr), "l"(g) : "memory");
}
SAL_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
SAL_DEVINL void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 32 lanes x 32 columns of fp32 from TMEM (warp-collective)
SAL_DEVINL void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// K-major SWIZZLE_128B tile: row r, 16-byte chunk c of a 128-byte row slice
SAL_DEVINL uint32_t swz_k(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

// ---------------------------------------------------------------------------
// forward: M-tile 128, N = 256, K = 256 (4 K-blocks of 64)
// ---------------------------------------------------------------------------
constexpr int kFM = 128, kFN = 256, kFK = 256, kFKB = 64;
constexpr int kFThreads = 256;
constexpr uint32_t kBBytes = kFN * kFK * 2;     // 128 KB
constexpr uint32_t kABytes = kFM * kFK * 2;     // 64 KB
constexpr uint32_t kFSmem = kBBytes + kABytes + 1024 + 64;

// sal_tc_sage_fwd flags (the relu_dropout argument): bit 0 = ReLU + dropout
// epilogue, bit 1 = leave the padding tiles past *m_dev unwritten
constexpr int kReluDropout = 1, kNoPadFill = 2;

// Epilogue element math shared by the forward kernels: 32 consecutive fp32
// accumulator columns [c, c+32) of one row -> relu + dropout (scaled) in bf16
// plus the 32 keep bits; the dropout stream is relu_dropout_fwd_kernel's
// (common.cuh dropout_word64 for p == 0.5, 16-bit uniforms otherwise).
SAL_DEVINL uint32_t relu_dropout32(const uint32_t* r, int64_t row, int c, int relu_dropout,
                                   float p, float scale, uint32_t thresh, uint64_t key_base,
                                   __nv_bfloat16* o) {
  uint32_t bits = 0;
  if (!(relu_dropout & kReluDropout)) {
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = __float2bfloat16_rn(__uint_as_float(r[j]));
    return 0;
  }
  if (p == 0.5f || p == 0.f) {  // p = 0.5: one draw covers the 32 columns; p = 0: ReLU only
    const uint64_t e0 = (uint64_t)row * kFN + (uint64_t)c;
    const uint32_t keep =
        p > 0.f ? (uint32_t)(dropout_word64(key_base, e0 >> 6) >> (e0 & 63)) : 0xFFFFFFFFu;
    const float mult = p > 0.f ? 2.f : 1.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) bits |= (__uint_as_float(r[j]) > 0.f ? 1u : 0u) << j;
    bits &= keep;
    // word arithmetic instead of per-element selects: bf16x2(2 v) of every pair,
    // ANDed with 0xFFFF halves where the keep/ReLU bit is set.  The 4 bits of a
    // quad spread to the byte MSBs (one multiply; the 4 shifted copies do not
    // overlap), prmt's sign replication widens a byte MSB to a 16-bit half.
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(o);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t spread = (((bits >> (4 * q)) & 0xFu) * 0x10204080u) & 0x80808080u;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 4 * q + 2 * h;
        const __nv_bfloat162 b =
            __floats2bfloat162_rn(__uint_as_float(r[j]) * mult, __uint_as_float(r[j + 1]) * mult);
        uint32_t km;
        asm("prmt.b32 %0, %1, 0, %2;" : "=r"(km) : "r"(spread), "r"(h ? 0xBBAAu : 0x9988u));
        const uint32_t w = *reinterpret_cast<const uint32_t*>(&b) & km;
        o2[j >> 1] = *reinterpret_cast<const __nv_bfloat162*>(&w);
      }
    }
    return bits;
  }
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint64_t r0 = ~0ull, r1 = ~0ull;
    if (p > 0.f) {  // group i = row * 32 + col / 8
      const uint64_t i = (uint64_t)row * (kFN / 8) + (uint64_t)((c >> 3) + g);
      const uint64_t kk = key_base ^ (i * 0xD1B54A32D192ED03ull);
      r0 = mix64(kk);
      r1 = mix64(kk + kGolden);
    }
    const uint32_t rr[4] = {(uint32_t)r0, (uint32_t)(r0 >> 32), (uint32_t)r1,
                            (uint32_t)(r1 >> 32)};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float v = __uint_as_float(r[g * 8 + j]);
      const uint32_t u16 = (rr[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
      const bool on = (u16 >= thresh) && v > 0.f;
      bits |= (uint32_t)on << (g * 8 + j);
      o[g * 8 + j] = __float2bfloat16_rn(on ? v * scale : 0.f);
    }
  }
  return bits;
}

// load a [rows x 256] bf16 row-major block into 4 K-major SW128 K-block tiles
SAL_DEVINL void load_kmajor(uint32_t sbase, const __nv_bfloat16* g, int64_t ldg, int rows,
                            int valid_rows, int tid, int nthreads) {
  // 16-byte chunks: rows x 32 per row (256 bf16 = 512 B)
  const int chunks = rows * 32;
  for (int q = tid; q < chunks; q += nthreads) {
    const int r = q >> 5, cc = q & 31;          // cc: chunk within the 512-byte row
    const int kb = cc >> 3, c = cc & 7;         // K-block and chunk within its 128-byte slice
    const uint32_t dst = sbase + (uint32_t)kb * (uint32_t)(rows * 128) + swz_k(r, c);
    const __nv_bfloat16* src = g + (int64_t)r * ldg + cc * 8;
    if (r < valid_rows) cp_async16(dst, src);
    else cp_async_zero16(dst, g);
  }
}

__global__ void __launch_bounds__(kFThreads, 1)
sage_fwd_kernel(const __nv_bfloat16* __restrict__ A, int64_t lda, int M,
                const __nv_bfloat16* __restrict__ W, __nv_bfloat16* __restrict__ Y, int64_t ldy,
                uint8_t* __restrict__ mask, float p, uint64_t seed,
                const int64_t* __restrict__ salt, int relu_dropout) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sB = smem;
  uint8_t* sA = smem + kBBytes;
  uint64_t* mbar = (uint64_t*)(sA + kABytes);
  uint32_t* tmem_slot = (uint32_t*)(mbar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntiles = (M + kFM - 1) / kFM;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // resident weights + the first A tile
  load_kmajor(smem_u32(sB), W, kFK, kFN, kFN, tid, kFThreads);
  int tile = blockIdx.x;
  if (tile < ntiles)
    load_kmajor(smem_u32(sA), A + (int64_t)tile * kFM * lda, lda, kFM, min(kFM, M - tile * kFM),
                tid, kFThreads);
  cp_async_commit();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = make_idesc(kFM, kFN, 0, 0);
  const float scale = p > 0.f ? (p < 1.f ? 1.f / (1.f - p) : 0.f) : 1.f;
  const uint32_t thresh = (uint32_t)(p * 65536.0f);
  const uint64_t key_base = mix64(seed ^ mix64((salt ? (uint64_t)*salt : 0ull) + 0x5EEDull));
  uint32_t phase = 0;

  for (; tile < ntiles; tile += gridDim.x) {
    cp_async_wait_all();
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kb = 0; kb < kFK / kFKB; ++kb) {
#pragma unroll
        for (int k = 0; k < kFKB / 16; ++k) {
          const uint64_t a = make_desc(smem_u32(sA) + kb * (kFM * 128) + k * 32, 16, 1024, 2);
          const uint64_t b = make_desc(smem_u32(sB) + kb * (kFN * 128) + k * 32, 16, 1024, 2);
          mma_f16(tmem, a, b, idesc, (kb | k) != 0);
        }
      }
      mma_commit(mbar);
    }
    mbar_wait(mbar, phase);
    phase ^= 1;
    tc_fence_after();
    // A is free again: prefetch the next tile while the epilogue drains TMEM
    const int next = tile + gridDim.x;
    if (next < ntiles)
      load_kmajor(smem_u32(sA), A + (int64_t)next * kFM * lda, lda, kFM,
                  min(kFM, M - next * kFM), tid, kFThreads);
    cp_async_commit();
    // epilogue: warp w reads TMEM lanes 32*(w%4).., columns [128*(w/4), +128)
    const int row = tile * kFM + (warp & 3) * 32 + lane;
    const int col0 = (warp >> 2) * 128;
#pragma unroll 1
    for (int cc = 0; cc < 128; cc += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(col0 + cc), r);
      if (row < M) {
        const int c = col0 + cc;
        alignas(16) __nv_bfloat16 o[32];
        const uint32_t bits =
            relu_dropout32(r, row, c, relu_dropout, p, scale, thresh, key_base, o);
        uint4* dst = reinterpret_cast<uint4*>(Y + (int64_t)row * ldy + c);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = reinterpret_cast<const uint4*>(o)[q];
        if (relu_dropout)
          *reinterpret_cast<uint32_t*>(mask + (int64_t)row * (kFN / 8) + (c >> 3)) = bits;
      }
    }
    tc_fence_before();
    __syncthreads();  // TMEM drained before the next tile's MMA overwrites it
  }
  cp_async_wait_all();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// ---------------------------------------------------------------------------
// weight gradient: dW[256 x 256] += dz[M x 256]^T @ A[M x 256], MN-major operands
// ---------------------------------------------------------------------------
constexpr int kGN = 256;     // dW rows (f_out) = 2 UMMA M-halves of 128
constexpr int kGK = 256;     // dW cols (2 f_in) = UMMA N
constexpr int kGC = 64;      // M rows (GEMM K) per chunk
constexpr int kGThreads = 256;
// per chunk: dz^T operand 64 x 256 bf16 (32 KB) + A operand 64 x 256 (32 KB); 2 stages
constexpr uint32_t kGStage = 2u * kGC * 256u * 2u;
constexpr uint32_t kGSmem = 2 * kGStage + 1024 + 64;

// MN-major SW128 layout of a [kGC (k) x 256 (mn)] row-major block: atoms of
// 8 k-rows x 64 mn (1024 B), mn-groups at LBO = 1024 B, k-groups at SBO =
// 4 * 1024 B (the 4 mn-groups of a k-group are adjacent).
SAL_DEVINL uint32_t swz_mn(int k, int mnchunk) {
  const int g = mnchunk >> 3, c = mnchunk & 7;  // 64-element mn-group, 16-byte chunk in it
  return (uint32_t)((k >> 3) * 4096 + g * 1024 + (k & 7) * 128 + ((c ^ (k & 7)) << 4));
}

SAL_DEVINL void load_mnmajor(uint32_t sbase, const __nv_bfloat16* g, int64_t ldg, int valid,
                             int tid) {
  for (int q = tid; q < kGC * 32; q += kGThreads) {  // 64 rows x 32 chunks of 16 B
    const int k = q >> 5, cc = q & 31;
    const uint32_t dst = sbase + swz_mn(k, cc);
    if (k < valid) cp_async16(dst, g + (int64_t)k * ldg + cc * 8);
    else cp_async_zero16(dst, g);
  }
}

__global__ void __launch_bounds__(kGThreads, 1)
sage_wgrad_kernel(const __nv_bfloat16* __restrict__ dz, int64_t ldz,
                  const __nv_bfloat16* __restrict__ A, int64_t lda, int M, int rows_per_cta,
                  float* __restrict__ dW, int64_t lddw) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* mbar = (uint64_t*)(smem + 2 * kGStage);
  uint32_t* tmem_slot = (uint32_t*)(mbar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * rows_per_cta;
  const int m1 = min(M, m0 + rows_per_cta);
  const int nchunks = m1 > m0 ? (m1 - m0 + kGC - 1) / kGC : 0;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  auto stage_load = [&](int ch, int s) {
    const int mr = m0 + ch * kGC;
    const int valid = min(kGC, m1 - mr);
    const uint32_t base = smem_u32(smem + s * kGStage);
    load_mnmajor(base, dz + (int64_t)mr * ldz, ldz, valid, tid);            // dz^T operand
    load_mnmajor(base + kGStage / 2, A + (int64_t)mr * lda, lda, valid, tid);  // A operand
    cp_async_commit();
  };
  if (nchunks > 0) stage_load(0, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = make_idesc(128, kGK, 1, 1);
  uint32_t ph[2] = {0, 0};
  for (int ch = 0; ch < nchunks; ++ch) {
    const int s = ch & 1;
    if (ch + 1 < nchunks) {
      if (ch >= 1) {  // stage s^1 was last read by chunk ch-1's MMAs
        mbar_wait(&mbar[s ^ 1], ph[s ^ 1]);
        ph[s ^ 1] ^= 1;
      }
      stage_load(ch + 1, s ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      cp_async_wait_all();
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t base = smem_u32(smem + s * kGStage);
#pragma unroll
      for (int kk = 0; kk < kGC / 16; ++kk) {  // K step of 16 rows = 2 k-groups
#pragma unroll
        for (int h = 0; h < 2; ++h) {          // dW rows [128h, 128h+128): mn-groups 2h, 2h+1
          const uint64_t a = make_desc(base + kk * 8192 + h * 2048, 1024, 4096, 2);
          const uint64_t b = make_desc(base + kGStage / 2 + kk * 8192, 1024, 4096, 2);
          mma_f16(tmem + h * 256, a, b, idesc, (ch | kk) != 0);
        }
      }
      mma_commit(&mbar[s]);
    }
  }
  if (nchunks > 0) {
    const int s = (nchunks - 1) & 1;
    mbar_wait(&mbar[s], ph[s]);
    if (nchunks >= 2) {  // the other stage's last commit may still be pending
      mbar_wait(&mbar[s ^ 1], ph[s ^ 1]);
    }
    tc_fence_after();
    // epilogue: warp w -> TMEM lanes 32*(w%4) (dW rows within the half), half w/4
    const int h = warp >> 2;
    const int rrow = h * 128 + (warp & 3) * 32 + lane;
#pragma unroll 1
    for (int cc = 0; cc < kGK; cc += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(h * 256 + cc), r);
      float* dst = dW + (int64_t)rrow * lddw + cc;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        atomicAdd(reinterpret_cast<float4*>(dst) + q,
                  make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                              __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ===========================================================================
// TMA + warp-specialised versions (the production path)
// ===========================================================================
SAL_DEVINL void mbar_expect_tx(void* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)),
               "r"(bytes)
               : "memory");
}
SAL_DEVINL void mbar_arrive(void* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mbar)) : "memory");
}
SAL_DEVINL void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, void* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(mbar))
      : "memory");
}
SAL_DEVINL bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

// A K-block of the TMA forward: 128 rows x 64 K (16 KB, SWIZZLE_128B)
constexpr uint32_t kPABlk = kFM * kFKB * 2;

// forward v2: the epilogue stores through shared memory with TMA.  In v1 each
// epilogue lane writes its own TMEM row straight to HBM (st.global.v4 of 32
// different rows per instruction), so every store request costs 32 L1 tag
// cycles: 2.7 M of them per launch, ~9.6 us per SM at papers shape (ncu).
// Here each warp converts a 32-row x 32-column chunk, writes it into a 2 KB
// SWIZZLE_64B staging tile (conflict-free 16-byte shared stores) and one lane
// issues a bulk tensor store.  16 epilogue warps (4 per SM sub-partition,
// v1 had 2) hide the tcgen05.ld and RNG latency.
constexpr int kSEpiWarps = 16;
constexpr int kSThreads = (2 + kSEpiWarps) * 32;
constexpr uint32_t kSStage = 32 * 32 * 2;         // 2 KB staging per epilogue warp
// shared memory of an instantiation: W block [BN x FK] + the A ring, filling what
// the W block leaves (4 stages at 128 KB of W, 8 at 64 KB)
template <int BN, int FK>
struct FwdCfg {
  static constexpr uint32_t kW = (uint32_t)BN * FK * 2;
  static constexpr int kStages = kW >= 131072u ? 4 : 8;
  static constexpr uint32_t kSmem = kW + kStages * kPABlk + kSEpiWarps * kSStage + 1024 + 256;
  static_assert(kSmem <= 232448u, "shared memory");
};

SAL_DEVINL void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
      "r"(src), "r"(c0), "r"(c1)
      : "memory");
}
SAL_DEVINL void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
SAL_DEVINL void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
SAL_DEVINL void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// BN output columns per CTA (the W block [BN x FK] stays resident: 128 KB for
// (256, 256) and (128, 512)); blockIdx.y picks the column block n0 = BN * y of
// the N = kFN = 256 output columns (dropout indices and the mask use the full row)
template <int BN, int FK>
__global__ void __launch_bounds__(kSThreads, 1)
sage_fwd_tma_st_kernel(const __grid_constant__ CUtensorMap mapA,
                       const __grid_constant__ CUtensorMap mapW,
                       const __grid_constant__ CUtensorMap mapY, int M,
                       const int64_t* __restrict__ m_dev, uint8_t* __restrict__ mask, float p,
                       uint64_t seed, const int64_t* __restrict__ salt, int relu_dropout) {
  constexpr uint32_t kWB = FwdCfg<BN, FK>::kW;
  constexpr int kSt = FwdCfg<BN, FK>::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int n0 = (int)blockIdx.y * BN;
  uint8_t* sB = smem;
  uint8_t* sA = smem + kWB;
  uint8_t* sY = sA + kSt * kPABlk;
  uint64_t* bars = (uint64_t*)(sY + kSEpiWarps * kSStage);
  uint64_t* full = bars;                    // [kSt]
  uint64_t* empty = bars + kSt;        // [kSt]
  uint64_t* bfull = bars + 2 * kSt;    // W resident
  uint64_t* tfull = bars + 2 * kSt + 1;   // [2] accumulator ready
  uint64_t* tempty = bars + 2 * kSt + 3;  // [2] accumulator drained
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * kSt + 5);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (M + kFM - 1) / kFM;
  // tiles past the true row count (*m_dev, static shapes pad to M) are only
  // zero-filled: no TMA loads, no MMA
  const int m_true = m_dev ? (int)min((int64_t)M, *m_dev) : M;
  const int nfull = (m_true + kFM - 1) / kFM;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kSt; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(bfull, 1);
    mbar_init(&tfull[0], 1);
    mbar_init(&tfull[1], 1);
    mbar_init(&tempty[0], kSEpiWarps);
    mbar_init(&tempty[1], kSEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapY) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      mbar_expect_tx(bfull, kWB);
#pragma unroll
      for (int kb = 0; kb < FK / kFKB; ++kb)
        tma_load_2d(smem_u32(sB) + kb * (BN * 128), &mapW, kb * kFKB, n0, bfull);
      int stage = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < nfull; t += gridDim.x) {
        for (int kb = 0; kb < FK / kFKB; ++kb) {
          mbar_wait(&empty[stage], ph ^ 1);
          mbar_expect_tx(&full[stage], kPABlk);
          tma_load_2d(smem_u32(sA) + stage * kPABlk, &mapA, kb * kFKB, t * kFM, &full[stage]);
          if (++stage == kSt) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc(kFM, BN, 0, 0);
    mbar_wait(bfull, 0);
    int stage = 0;
    uint32_t ph = 0;
    int it = 0;
    for (int t = blockIdx.x; t < nfull; t += gridDim.x, ++it) {
      const int buf = it & 1;
      const uint32_t tph = (uint32_t)((it >> 1) & 1);
      mbar_wait(&tempty[buf], tph ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < FK / kFKB; ++kb) {
        mbar_wait(&full[stage], ph);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kFKB / 16; ++k) {
            const uint64_t a = make_desc(smem_u32(sA) + stage * kPABlk + k * 32, 16, 1024, 2);
            const uint64_t b = make_desc(smem_u32(sB) + kb * (BN * 128) + k * 32, 16, 1024, 2);
            mma_f16(tmem + buf * 256, a, b, idesc, (kb | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (kb == FK / kFKB - 1) mma_commit(&tfull[buf]);
        }
        __syncwarp();
        if (++stage == kSt) { stage = 0; ph ^= 1; }
      }
    }
  } else {
    // epilogue warp e = 0..15: TMEM lane group (warp % 4), column quarter e / 4
    const int e = warp - 2;
    const int lg = warp & 3;
    const int cq = e >> 2;
    uint8_t* stg = sY + e * kSStage;
    const uint32_t stg_s = smem_u32(stg);
    const float scale = p > 0.f ? (p < 1.f ? 1.f / (1.f - p) : 0.f) : 1.f;
    const uint32_t thresh = (uint32_t)(p * 65536.0f);
    const uint64_t key_base = mix64(seed ^ mix64((salt ? (uint64_t)*salt : 0ull) + 0x5EEDull));
    int it = 0;
    for (int t = blockIdx.x; t < nfull; t += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(&tfull[buf], (uint32_t)((it >> 1) & 1));
      tc_fence_after();
      const int row0 = t * kFM + lg * 32;
      const int row = row0 + lane;
#pragma unroll 1
      for (int cl = cq * (BN / 4); cl < (cq + 1) * (BN / 4); cl += 32) {
        const int c = n0 + cl;   // output column
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(buf * 256 + cl), r);
        alignas(16) __nv_bfloat16 o[32];
        const uint32_t bits =
            relu_dropout32(r, row, c, relu_dropout, p, scale, thresh, key_base, o);
        // staging tile free again (the previous bulk store has read it)
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
        // SWIZZLE_64B: 16-byte chunk q of row `lane` at lane*64 + ((q ^ ((lane>>1)&3)) << 4)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4*>(stg + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) =
              reinterpret_cast<const uint4*>(o)[q];
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&mapY, stg_s, c, row0);
          bulk_commit();
        }
        if ((relu_dropout & kReluDropout) && row < M)
          *reinterpret_cast<uint32_t*>(mask + (int64_t)row * (kFN / 8) + (c >> 3)) = bits;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
    // padding tiles: zero rows (finite, zero-gradient) without touching A or TMEM;
    // skipped entirely when the caller does not consume padding rows (kNoPadFill)
    const int first_pad = blockIdx.x + ((nfull - (int)blockIdx.x + (int)gridDim.x - 1) /
                                        (int)gridDim.x) * (int)gridDim.x;
    if (first_pad < ntiles && !(relu_dropout & kNoPadFill)) {
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<uint4*>(stg + lane * 64 + (q << 4)) = make_uint4(0, 0, 0, 0);
      fence_async_smem();
      __syncwarp();
      for (int t = first_pad > (int)blockIdx.x ? first_pad : (int)blockIdx.x; t < ntiles;
           t += gridDim.x) {
        if (t < nfull) continue;
        const int row0 = t * kFM + lg * 32;
        for (int c = n0 + cq * (BN / 4); c < n0 + (cq + 1) * (BN / 4); c += 32) {
          if (lane == 0) {
            tma_store_2d(&mapY, stg_s, c, row0);
            bulk_commit();
          }
          if ((relu_dropout & kReluDropout) && row0 + lane < M)
            *reinterpret_cast<uint32_t*>(mask + (int64_t)(row0 + lane) * (kFN / 8) + (c >> 3)) = 0u;
        }
      }
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// weight gradient with TMA, tiled split-K: CTA (tile, split) accumulates one
// 128 x 128 tile of dW (rows n0.., cols k0..) over a contiguous range of GEMM-K
// rows (= M rows of dz / A).  Splitting the output into tiles cuts the fp32
// partials the epilogue adds atomically (S x N x K instead of 148 x N x K);
// the CTAs of one split read the same dz/A rows at the same time, so the
// second read of each chunk hits L2.  Stage = dz chunk [64 rows x 128] + A
// chunk [64 x 128], each two TMA boxes of {64 mn, 64 k}.
// stage count (-DSAL_WGRAD_STAGES=N builds the A/B variants of
// profiles/r1_ab_wgrad_epilogue.txt; 3, 4 and 6 time alike alone, 6 is best in the step)
#ifndef SAL_WGRAD_STAGES
#define SAL_WGRAD_STAGES 6
#endif
constexpr int kQStages = SAL_WGRAD_STAGES;
constexpr int kQThreads = 192;
constexpr uint32_t kQHalf = kGC * 128 * 2;   // 16 KB per operand per stage
constexpr uint32_t kQStage = 2 * kQHalf;
constexpr uint32_t kQSmem = kQStages * kQStage + 1024 + 256;

__global__ void __launch_bounds__(kQThreads, 1)
sage_wgrad_tma_kernel(const __grid_constant__ CUtensorMap mapDz,
                      const __grid_constant__ CUtensorMap mapA, int M,
                      const int64_t* __restrict__ m_dev, int part, int nparts, int tiles_k,
                      float* __restrict__ dW, int64_t lddw) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + kQStages * kQStage);
  uint64_t* full = bars;
  uint64_t* empty = bars + kQStages;
  uint64_t* done = bars + 2 * kQStages;
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * kQStages + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, split = blockIdx.y;
  const int n0 = (tile / tiles_k) * 128, k0 = (tile % tiles_k) * 128;
  // GEMM-K rows: the true row count when given (rows past it are zero / padding),
  // split evenly over the grid's splits in whole 64-row chunks
  // (of part `part` of nparts: rows [pb, pe), part_rows)
  int pb = 0, pe = M;
  if (nparts > 1) part_rows(m_dev, M, part, nparts, &pb, &pe);
  const int Me = min(pe, m_dev ? (int)min((int64_t)M, *m_dev) : M);
  const int splits = (int)gridDim.y;
  const int span = max(Me - pb, 0);
  const int rows_per_split = ((span + splits - 1) / splits + kGC - 1) / kGC * kGC;
  const int m0 = pb + split * rows_per_split;
  const int m1 = min(Me, m0 + rows_per_split);
  const int nchunks = m1 > m0 ? (m1 - m0 + kGC - 1) / kGC : 0;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kQStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t ph = 0;
      for (int ch = 0; ch < nchunks; ++ch) {
        const int mr = m0 + ch * kGC;
        mbar_wait(&empty[stage], ph ^ 1);
        mbar_expect_tx(&full[stage], kQStage);
        const uint32_t base = smem_u32(smem + stage * kQStage);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          tma_load_2d(base + g * 8192, &mapDz, n0 + g * 64, mr, &full[stage]);
          tma_load_2d(base + kQHalf + g * 8192, &mapA, k0 + g * 64, mr, &full[stage]);
        }
        if (++stage == kQStages) { stage = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc(128, 128, 1, 1);
    int stage = 0;
    uint32_t ph = 0;
    for (int ch = 0; ch < nchunks; ++ch) {
      mbar_wait(&full[stage], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t base = smem_u32(smem + stage * kQStage);
#pragma unroll
        for (int kk = 0; kk < kGC / 16; ++kk) {
          // mn-groups of 64 at LBO 8 KB, 8-row k-groups at SBO 1 KB
          const uint64_t a = make_desc(base + kk * 2048, 8192, 1024, 2);
          const uint64_t b = make_desc(base + kQHalf + kk * 2048, 8192, 1024, 2);
          mma_f16(tmem, a, b, idesc, (ch | kk) != 0);
        }
        mma_commit(&empty[stage]);
        if (ch == nchunks - 1) mma_commit(done);
      }
      __syncwarp();
      if (++stage == kQStages) { stage = 0; ph ^= 1; }
    }
  } else if (nchunks > 0) {
    // epilogue warps 2..5: TMEM lane group warp % 4 -> dW rows n0 + 32 (warp % 4) + lane
    const int lg = warp & 3;
    mbar_wait(done, 0);
    tc_fence_after();
    const int rrow = n0 + lg * 32 + lane;
#pragma unroll 1
    for (int c4 = 0; c4 < 4; ++c4) {
      // splits start at different column blocks so their atomics spread over L2 slices
      const int cc = ((c4 + split) & 3) * 32;
      uint32_t r[32];
      tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)cc, r);
      float* dst = dW + (int64_t)rrow * lddw + k0 + cc;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        atomicAdd(reinterpret_cast<float4*>(dst) + q,
                  make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                              __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

// host: 2-D bf16 tensor map [rows x cols] (row stride in elements), SWIZZLE_128B
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static bool make_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                     uint64_t row_stride_elems, uint32_t box_cols, uint32_t box_rows,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  if (g_encode == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        fn == nullptr)
      return false;
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {row_stride_elems * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace tc
}  // namespace sal

extern "C" {

int sal_tc_sage_fwd(const void* A, int64_t lda, int64_t M, const int64_t* m_dev, const void* W,
                    int32_t N, int32_t K, void* Y, int64_t ldy, uint8_t* mask, float p,
                    uint64_t seed, const int64_t* salt_dev, int32_t relu_dropout, void* stream) {
  // two column blocks of 128 (grid.y); each CTA holds its [128 x K] W block
  // (K = 256: layer 0; K = 512: the hidden layer)
  if (N != sal::tc::kFN || (K != 256 && K != 512)) return SAL_EINVAL;
  if (lda % 8 || ldy % 8 || ((uintptr_t)A & 15) || ((uintptr_t)W & 15) || ((uintptr_t)Y & 15))
    return SAL_EINVAL;
  if (M <= 0) return SAL_OK;
  const int bn = 128;
  const int nblk = N / bn;
  CUtensorMap mA, mW, mY;
  if (!sal::tc::make_map(&mA, A, (uint64_t)M, (uint64_t)K, (uint64_t)lda, 64, 128) ||
      !sal::tc::make_map(&mW, W, (uint64_t)N, (uint64_t)K, (uint64_t)K, 64, (uint32_t)bn))
    return SAL_ECUDA;
  const int ntiles = (int)((M + 127) / 128);
  int grid = sal::num_sms() / nblk;
  if (grid > ntiles) grid = ntiles;
  if (!sal::tc::make_map(&mY, Y, (uint64_t)M, 256, (uint64_t)ldy, 32, 32,
                         CU_TENSOR_MAP_SWIZZLE_64B))
    return SAL_ECUDA;
  // 128-column blocks for both K: the W block is 64 KB at K = 256, leaving room
  // for an 8-stage A ring (179.0 against 179.5 us per step with 256-column tiles
  // and 4 stages; the kernel alone times the same)
  auto kern = K == 256 ? sal::tc::sage_fwd_tma_st_kernel<128, 256>
                       : sal::tc::sage_fwd_tma_st_kernel<128, 512>;
  const uint32_t smem =
      K == 256 ? sal::tc::FwdCfg<128, 256>::kSmem : sal::tc::FwdCfg<128, 512>::kSmem;
  static bool attr[2] = {false, false};
  if (!attr[K == 512]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr[K == 512] = true;
  }
  kern<<<dim3(grid, nblk), sal::tc::kSThreads, smem, (cudaStream_t)stream>>>(
      mA, mW, mY, (int)M, m_dev, mask, p, seed, salt_dev, relu_dropout);
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
}

int sal_tc_sage_fwd_simple(const void* A, int64_t lda, int64_t M, const void* W, int32_t N,
                           int32_t K, void* Y, int64_t ldy, uint8_t* mask, float p, uint64_t seed,
                           const int64_t* salt_dev, int32_t relu_dropout, void* stream) {
  if (N != sal::tc::kFN || K != sal::tc::kFK) return SAL_EINVAL;
  if (lda % 8 || ldy % 8 || ((uintptr_t)A & 15) || ((uintptr_t)W & 15) || ((uintptr_t)Y & 15))
    return SAL_EINVAL;
  if (M <= 0) return SAL_OK;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sal::tc::sage_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         sal::tc::kFSmem);
    attr = true;
  }
  const int ntiles = (int)((M + 127) / 128);
  int grid = sal::num_sms();
  if (grid > ntiles) grid = ntiles;
  sal::tc::sage_fwd_kernel<<<grid, sal::tc::kFThreads, sal::tc::kFSmem, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)A, lda, (int)M, (const __nv_bfloat16*)W, (__nv_bfloat16*)Y, ldy, mask,
      p, seed, salt_dev, relu_dropout);
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
}

int sal_tc_sage_wgrad_part(const void* dz, int64_t ldz, const void* A, int64_t lda, int64_t M,
                           const int64_t* m_dev, int32_t part, int32_t nparts, int32_t N,
                           int32_t K, float* dW, int64_t lddw, int32_t accumulate,
                           void* stream) {
  if (N <= 0 || K <= 0 || N % 128 || K % 128) return SAL_EINVAL;
  if (nparts < 1 || part < 0 || part >= nparts) return SAL_EINVAL;
  if (ldz % 8 || lda % 8 || ((uintptr_t)dz & 15) || ((uintptr_t)A & 15) || ((uintptr_t)dW & 15) ||
      lddw % 4 || lddw < K)
    return SAL_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (!accumulate &&
      cudaMemsetAsync(dW, 0, sizeof(float) * (size_t)N * (size_t)lddw, st) != cudaSuccess)
    return SAL_ECUDA;
  if (M <= 0) return SAL_OK;
  CUtensorMap mD, mA;
  if (!sal::tc::make_map(&mD, dz, (uint64_t)M, (uint64_t)N, (uint64_t)ldz, 64, 64) ||
      !sal::tc::make_map(&mA, A, (uint64_t)M, (uint64_t)K, (uint64_t)lda, 64, 64))
    return SAL_ECUDA;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sal::tc::sage_wgrad_tma_kernel,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, sal::tc::kQSmem);
    attr = true;
  }
  // one CTA per SM: tiles x splits ~ #SMs, splits of whole 64-row chunks
  const int tiles_k = K / 128;
  const int tiles = (N / 128) * tiles_k;
  int splits = sal::num_sms() / tiles;
  if (splits < 1) splits = 1;
  const int64_t Mp = (M + nparts - 1) / nparts;
  int rows = (int)((Mp + splits - 1) / splits);
  rows = (rows + 63) / 64 * 64;
  splits = (int)((Mp + rows - 1) / rows);
  sal::tc::sage_wgrad_tma_kernel<<<dim3(tiles, splits), sal::tc::kQThreads, sal::tc::kQSmem, st>>>(
      mD, mA, (int)M, m_dev, part, nparts, tiles_k, dW, lddw);
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
}

int sal_tc_sage_wgrad(const void* dz, int64_t ldz, const void* A, int64_t lda, int64_t M,
                      const int64_t* m_dev, int32_t N, int32_t K, float* dW, int64_t lddw,
                      int32_t accumulate, void* stream) {
  return sal_tc_sage_wgrad_part(dz, ldz, A, lda, M, m_dev, 0, 1, N, K, dW, lddw, accumulate,
                                stream);
}

int sal_tc_sage_wgrad_simple(const void* dz, int64_t ldz, const void* A, int64_t lda, int64_t M,
                             int32_t N, int32_t K, float* dW, int64_t lddw, void* stream) {
  if (N != sal::tc::kGN || K != sal::tc::kGK) return SAL_EINVAL;
  if (ldz % 8 || lda % 8 || ((uintptr_t)dz & 15) || ((uintptr_t)A & 15) || ((uintptr_t)dW & 15) ||
      lddw % 4)
    return SAL_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(dW, 0, sizeof(float) * (size_t)N * (size_t)lddw, st) != cudaSuccess)
    return SAL_ECUDA;
  if (M <= 0) return SAL_OK;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sal::tc::sage_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         sal::tc::kGSmem);
    attr = true;
  }
  int grid = sal::num_sms();
  int rows = (int)((M + grid - 1) / grid);
  rows = (rows + 63) / 64 * 64;
  grid = (int)((M + rows - 1) / rows);
  sal::tc::sage_wgrad_kernel<<<grid, sal::tc::kGThreads, sal::tc::kGSmem, st>>>(
      (const __nv_bfloat16*)dz, ldz, (const __nv_bfloat16*)A, lda, (int)M, rows, dW, lddw);
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
}

}  // extern "C"
