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
//           round-trips through HBM.
//
// Weight gradient: dW[N, K] += dz[M, N]^T @ A[M, K] with both operands read
//           MN-major (row-major in HBM): CTA (tile, split) reduces a contiguous
//           range of M rows into one 128 x 128 TMEM accumulator of dW and adds
//           its partial into the fp32 gradient with vector atomics.
//
// Rest of the step (sage_gemm_kernel<BN, B major, epilogue>): the input
//           gradients dA = dz @ W_cat (B MN-major, bf16 store epilogue) and the
//           output layer logits = A @ W^T whose epilogue is the loss
//           (log_softmax + NLL + dlogits) in training or argmax + correct count
//           in inference: no GEMM of the step goes through cuBLAS.
//
// Reference contraction: mpnn.py:82 (h_dst W_self^T + mean W_neigh^T) and its
// backward; the model around it is PAPER.md:2562-2586.
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


// ---------------------------------------------------------------------------
// forward: M-tile 128, N = 256, K = 256 (4 K-blocks of 64)
// ---------------------------------------------------------------------------
constexpr int kFM = 128, kFN = 256, kFKB = 64;

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
    // the staging tiles must stay valid until the bulk stores have read them; the
    // writes themselves complete with the grid (no need to wait for them here)
    if (lane == 0) bulk_wait_read0();
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
// stage count (-DSAL_WGRAD_STAGES=N builds the A/B variants).  3, 4 and 6 time alike
// alone (profiles/r1_ab_wgrad_epilogue.txt); with the fused last hop beside it, 3 stages
// (99 KB) let a weight-gradient CTA share an SM with three fused-kernel blocks:
// 164 -> 161 us per step (profiles/r2_ab_wgrad_stages.txt)
#ifndef SAL_WGRAD_STAGES
#define SAL_WGRAD_STAGES 3
#endif
constexpr int kGC = 64;      // GEMM-K rows (M rows of dz / A) per chunk
constexpr int kQStages = SAL_WGRAD_STAGES;
constexpr int kQThreads = 192;
constexpr uint32_t kQHalf = kGC * 128 * 2;   // 16 KB per operand per stage
constexpr uint32_t kQStage = 2 * kQHalf;
constexpr uint32_t kQSmem = kQStages * kQStage + 1024 + 256;

__global__ void __launch_bounds__(kQThreads, 1)
sage_wgrad_tma_kernel(const __grid_constant__ CUtensorMap mapDz,
                      const __grid_constant__ CUtensorMap mapA, int M,
                      const int64_t* __restrict__ m_dev, int tiles_k, int N,
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
  const int Me = m_dev ? (int)min((int64_t)M, *m_dev) : M;
  const int splits = (int)gridDim.y;
  const int rows_per_split = ((Me + splits - 1) / splits + kGC - 1) / kGC * kGC;
  const int m0 = split * rows_per_split;
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
    // (rows past N: the zero columns TMA filled in past dz's last column)
    const int lg = warp & 3;
    mbar_wait(done, 0);
    tc_fence_after();
    const int rrow = n0 + lg * 32 + lane;
    const bool live = rrow < N;
#pragma unroll 1
    for (int c4 = 0; c4 < 4; ++c4) {
      // splits start at different column blocks so their atomics spread over L2 slices
      const int cc = ((c4 + split) & 3) * 32;
      uint32_t r[32];
      tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)cc, r);
      float* dst = dW + (int64_t)rrow * lddw + k0 + cc;
      if (!live) continue;
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

// ===========================================================================
// The rest of the step's GEMMs.  These are small (a few hundred KB of operands),
// so they are latency-bound: a CTA's cost is the bytes it pulls from L2, not the
// MMAs.  Both kernels therefore cut the work into many small CTAs.
//
// sage_gemm_kernel<BN, B major>: C[M, N] = A[M, K] @ B, bf16 out, 128 x BN
//   tiles (BN = 64 for the input gradients dA = dz @ W_cat, B = W_cat [K, N]
//   row-major = MN-major operand), 4 epilogue warps, several CTAs per SM.
// sage_logits_kernel<BN, epilogue>: the output layer logits = A @ W^T (W K-major)
//   split over K across a cluster of 4 CTAs; the fp32 partial tiles are summed
//   through distributed shared memory and each CTA finishes a quarter of the
//   rows: log_softmax + NLL + dlogits (training, replaces lsm_nll) or argmax +
//   correct count (inference, replaces argmax_correct).
// ===========================================================================
constexpr int kEpiNll = 1, kEpiArgmax = 2;

struct GemmTail {
  int32_t C;                        // valid classes
  int32_t c_pad;                    // nll: dlogits row width written (<= BN)
  const int64_t* labels;            // labels[0:n_labels], < 0 ignored
  int64_t n_labels;
  float* loss;                      // nll: += mean NLL over labels >= 0
  __nv_bfloat16* dlog;              // nll: dlogits rows [M, ldd] (cols >= C zero)
  int64_t ldd;
  unsigned long long* counts;       // argmax: [0] += correct, [1] += labelled
};

// 16 lanes x 32 columns of fp32 from TMEM (warp-collective)
SAL_DEVINL void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int BN, int EW>
struct GemmCfg {
  static constexpr uint32_t kB = (uint32_t)BN * kFKB * 2;  // B K-block
  static constexpr uint32_t kStage = kPABlk + kB;
  static constexpr int kStages = 4;
  static constexpr uint32_t kSmem = kStages * kStage + EW * kSStage + 1024 + 256;
  static constexpr int kThreads = (2 + EW) * 32;
  static_assert(kSmem <= 232448u, "shared memory");
  static_assert(BN % 16 == 0 && BN <= 256, "UMMA N");
};

constexpr int kNEW = 4;   // epilogue warps of the store GEMM (one per TMEM lane quarter)

template <int BN, bool kBMN>
__global__ void __launch_bounds__(GemmCfg<BN, kNEW>::kThreads)
sage_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                 const __grid_constant__ CUtensorMap mapC, int M, int K,
                 const int64_t* __restrict__ m_dev, int pad_fill) {
  using Cfg = GemmCfg<BN, kNEW>;
  constexpr int kSt = Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int n0 = (int)blockIdx.y * BN;
  uint8_t* sRing = smem;                       // [kSt] x {A block, B block}
  uint8_t* sY = smem + kSt * Cfg::kStage;
  uint64_t* bars = (uint64_t*)(sY + kNEW * kSStage);
  uint64_t* full = bars;
  uint64_t* empty = bars + kSt;
  uint64_t* tfull = bars + 2 * kSt;        // [2]
  uint64_t* tempty = bars + 2 * kSt + 2;   // [2]
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * kSt + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (M + kFM - 1) / kFM;
  const int m_true = m_dev ? (int)min((int64_t)M, *m_dev) : M;
  const int nfull = (m_true + kFM - 1) / kFM;
  const int nkb = (K + kFKB - 1) / kFKB;
  constexpr uint32_t kTCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128
                            : 2 * BN <= 256 ? 256 : 512;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kSt; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kNEW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapC) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTCols));
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
      for (int t = blockIdx.x; t < nfull; t += gridDim.x) {
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], ph ^ 1);
          mbar_expect_tx(&full[stage], Cfg::kStage);
          const uint32_t sa = smem_u32(sRing) + stage * Cfg::kStage;
          tma_load_2d(sa, &mapA, kb * kFKB, t * kFM, &full[stage]);
          if (kBMN) {  // B rows = K, 64-column mn-groups of 8 KB
#pragma unroll
            for (int g = 0; g < BN / 64; ++g)
              tma_load_2d(sa + kPABlk + g * 8192, &mapB, n0 + g * 64, kb * kFKB, &full[stage]);
          } else {     // B rows = N (one box of BN rows x 64 K)
            tma_load_2d(sa + kPABlk, &mapB, kb * kFKB, n0, &full[stage]);
          }
          if (++stage == kSt) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc(kFM, BN, 0, kBMN ? 1 : 0);
    int stage = 0;
    uint32_t ph = 0;
    int it = 0;
    for (int t = blockIdx.x; t < nfull; t += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(&tempty[buf], (uint32_t)(((it >> 1) & 1) ^ 1));
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(sRing) + stage * Cfg::kStage;
#pragma unroll
          for (int k = 0; k < kFKB / 16; ++k) {
            const uint64_t a = make_desc(sa + k * 32, 16, 1024, 2);
            const uint64_t b = kBMN ? make_desc(sa + kPABlk + k * 2048, 8192, 1024, 2)
                                    : make_desc(sa + kPABlk + k * 32, 16, 1024, 2);
            mma_f16(tmem + buf * BN, a, b, idesc, (kb | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (kb == nkb - 1) mma_commit(&tfull[buf]);
        }
        __syncwarp();
        if (++stage == kSt) { stage = 0; ph ^= 1; }
      }
    }
  } else {
    // epilogue warp e: TMEM lane quarter e (= warp % 4), all BN columns
    const int e = warp - 2;
    const int lg = warp & 3;
    uint8_t* stg = sY + e * kSStage;
    const uint32_t stg_s = smem_u32(stg);
    int it = 0;
    for (int t = blockIdx.x; t < nfull; t += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait(&tfull[buf], (uint32_t)((it >> 1) & 1));
      tc_fence_after();
      const int row0 = t * kFM + lg * 32;
      const uint32_t tb = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(buf * BN);
#pragma unroll 1
      for (int cl = 0; cl < BN; cl += 32) {
        uint32_t r[32];
        tmem_ld32(tb + (uint32_t)cl, r);
        alignas(16) __nv_bfloat16 o[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) o[j] = __float2bfloat16_rn(__uint_as_float(r[j]));
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4*>(stg + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) =
              reinterpret_cast<const uint4*>(o)[q];
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {   // rows past M: clipped by the tensor map
          tma_store_2d(&mapC, stg_s, n0 + cl, row0);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
    if (pad_fill) {   // tiles past the true row count: zero rows, no loads, no MMA
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<uint4*>(stg + lane * 64 + (q << 4)) = make_uint4(0, 0, 0, 0);
      fence_async_smem();
      __syncwarp();
      for (int t = nfull + (int)blockIdx.x; t < ntiles; t += gridDim.x)
        for (int cl = 0; cl < BN; cl += 32)
          if (lane == 0) {
            tma_store_2d(&mapC, stg_s, n0 + cl, t * kFM + lg * 32);
            bulk_commit();
          }
    }
    // the staging tiles must stay valid until the bulk stores have read them; the
    // writes themselves complete with the grid (no need to wait for them here)
    if (lane == 0) bulk_wait_read0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTCols));
}

// ---------------------------------------------------------------------------
// The output layer in one kernel (training: logits, loss, dlogits, dA, dW; or
// inference: logits, argmax + correct count).  One cluster of CL = K/64 CTAs per
// 128-row tile; CTA r owns K-block r (features [64 r, 64 r + 64)):
//   1. logits partial [128 x BN] = A[:, Kr] @ W[:, Kr]^T in TMEM, stored fp32 to
//      an L2-resident scratch (distributed shared memory moves ~20 B/clk per SM,
//      far too little for CL fp32 partial tiles; L2 is several times faster);
//   2. cluster barrier; CTA r finishes rows [128 r / CL, ...): sums the CL
//      partials, log_softmax + NLL + dlogits (bf16 rows to the dlogits buffer);
//   3. cluster barrier; the tile's dlogits rows come back by TMA (K-major, SW128)
//      and dA[:, Kr] = dlogits @ W[:, Kr]    (B = the resident W block, MN-major view)
//          dW[:, Kr] += dlogits^T @ A[:, Kr] (A = the dlogits tile, MN-major view;
//                                             B = the resident A block, MN-major view)
// so A and W are read from HBM once and every GEMM of the layer is a tcgen05 MMA.
// ---------------------------------------------------------------------------
constexpr int kHEW = 8;                       // epilogue warps
constexpr int kHThreads = (2 + kHEW) * 32;

template <int BN>
struct HeadCfg {
  static constexpr uint32_t kA = (uint32_t)kFM * kFKB * 2;        // 16 KB A block
  static constexpr uint32_t kW = (uint32_t)BN * kFKB * 2;         // W block
  static constexpr uint32_t kD = 4u * kFM * kFKB * 2;             // dlogits tile, 256 classes
  static constexpr uint32_t kOffW = kA, kOffD = kA + kW;
  static constexpr uint32_t kSmem = kOffD + kD + 1024 + 256;
  static_assert(BN % 64 == 0 && BN <= 192, "classes per tile");
  static_assert(kSmem <= 232448u, "shared memory");
};

// SAL_HEAD_TRACE builds record %globaltimer at the head kernel's phase boundaries
// (CTA 0, thread 64: an epilogue warp) into sal_head_trace[] for tools/ timelines
#ifdef SAL_HEAD_TRACE
__device__ unsigned long long sal_head_trace[16];
#define HEAD_MARK(i)                                                                        \
  do {                                                                                      \
    if (blockIdx.x == 0 && threadIdx.x == 64) {                                             \
      unsigned long long g_;                                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                               \
      sal_head_trace[i] = g_;                                                               \
    }                                                                                       \
  } while (0)
#else
#define HEAD_MARK(i) \
  do {               \
  } while (0)
#endif

SAL_DEVINL void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
SAL_DEVINL uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int BN, int CL, int kEpi>
__global__ void __launch_bounds__(kHThreads, 1)
sage_head_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapW,
                 const __grid_constant__ CUtensorMap mapD, int M,
                 const int64_t* __restrict__ m_dev, GemmTail tl, float* __restrict__ part,
                 __nv_bfloat16* __restrict__ dA, int64_t ldda, float* __restrict__ dW,
                 int64_t lddw) {
  using Cfg = HeadCfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sW = smem + Cfg::kOffW;
  uint8_t* sD = smem + Cfg::kOffD;
  uint64_t* bars = (uint64_t*)(smem + Cfg::kOffD + Cfg::kD);
  uint64_t* ld_full = bars;
  uint64_t* lg_done = bars + 1;
  uint64_t* d_full = bars + 2;
  uint64_t* bw_done = bars + 3;
  uint32_t* tmem_slot = (uint32_t*)(bars + 4);
  __shared__ float sh_red[kHEW];
  __shared__ int sh_cnt[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int t = (int)blockIdx.x / CL;          // the cluster's 128-row tile
  const int k0 = (int)rank * kFKB;             // this CTA's K block = features [k0, k0+64)
  const int m_true = m_dev ? (int)min((int64_t)M, *m_dev) : M;
  const bool live = t * kFM < m_true;          // uniform over the cluster
  constexpr int rows_per = kFM / CL;           // rows each CTA finishes
  constexpr bool kTrain = kEpi == kEpiNll;
  // this tile's partials: [CL][128][BN] fp32
  float* tpart = part + (size_t)t * CL * kFM * BN;
  // TMEM columns: logits [0, BN), dA [256, 320), dW halves [320, 384) and [384, 448)
  constexpr uint32_t kTA = 256, kTW = 320;

  if (!live) {   // padding tile: zero dA and dlogits rows (read downstream), nothing else
    if (kTrain) {
      const int rows = min(kFM, M - t * kFM);
      for (int q = threadIdx.x; q < rows * 8; q += kHThreads)
        *reinterpret_cast<uint4*>(dA + (int64_t)(t * kFM + q / 8) * ldda + k0 + (q % 8) * 8) =
            make_uint4(0, 0, 0, 0);
      const int pc = tl.c_pad / 8;
      for (int q = threadIdx.x; q < rows_per * pc; q += kHThreads) {
        const int row = t * kFM + (int)rank * rows_per + q / pc;
        if (row < M)
          *reinterpret_cast<uint4*>(tl.dlog + (int64_t)row * tl.ldd + (q % pc) * 8) =
              make_uint4(0, 0, 0, 0);
      }
    }
    return;
  }

  HEAD_MARK(0);
  if (warp == 0 && lane == 0) {
    mbar_init(ld_full, 1);
    mbar_init(lg_done, 1);
    mbar_init(d_full, 1);
    mbar_init(bw_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapW) : "memory");
    if (kTrain) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapD) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 2 && lane < 2) sh_cnt[lane] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // ---- 1. logits partial over this CTA's K block
  float inv = 1.f;
  int64_t my_lab[rows_per / kHEW > 0 ? rows_per / kHEW : 1];
  if (warp == 0) {
    if (elect_one()) {
      mbar_expect_tx(ld_full, Cfg::kA + Cfg::kW);
      tma_load_2d(smem_u32(sA), &mapA, k0, t * kFM, ld_full);
      tma_load_2d(smem_u32(sW), &mapW, k0, 0, ld_full);
    }
  } else if (warp == 1) {
    mbar_wait(ld_full, 0);
    tc_fence_after();
    if (elect_one()) {
      const uint32_t idesc = make_idesc(kFM, BN, 0, 0);
#pragma unroll
      for (int k = 0; k < kFKB / 16; ++k)
        mma_f16(tmem, make_desc(smem_u32(sA) + k * 32, 16, 1024, 2),
                make_desc(smem_u32(sW) + k * 32, 16, 1024, 2), idesc, k ? 1u : 0u);
      mma_commit(lg_done);
    }
    __syncwarp();
  } else {
    const int e = warp - 2, lg = warp & 3, ch = e >> 2;
    // while the loads and the MMA run: the loss normaliser (labelled rows of the
    // whole batch) and the labels of the rows this warp finishes
    if (kTrain) {
      const int64_t nl = min((int64_t)M, tl.n_labels);
      int c = 0;
#pragma unroll 4
      for (int64_t i = e * 32 + lane; i < nl; i += kHEW * 32) c += tl.labels[i] >= 0;
      c = warp_reduce_sum(c);
      if (lane == 0) sh_red[e] = (float)c;
    }
#pragma unroll
    for (int i = 0; i < rows_per / kHEW; ++i) {
      const int row = t * kFM + (int)rank * rows_per + e + i * kHEW;
      my_lab[i] = row < M && row < tl.n_labels ? tl.labels[row] : -1;
    }
    HEAD_MARK(1);
    mbar_wait(lg_done, 0);
    HEAD_MARK(2);
    tc_fence_after();
    // drain: warp e reads TMEM lane quarter warp % 4, column half e / 4 (thread =
    // row), transposes each 32 x 32 chunk through shared memory (the idle dlogits
    // tile; row stride 36 floats: conflict-free v4 both ways) and writes it to the
    // scratch as 4 rows x 128 B per instruction
    float* stg = reinterpret_cast<float*>(sD) + e * (32 * 36);
    float* dst = tpart + ((size_t)rank * kFM + lg * 32) * BN;
    for (int c = ch * (BN / 2); c < (ch + 1) * (BN / 2); c += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)c, r);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(stg + lane * 36 + 4 * q) =
            make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                        __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int rr = 4 * q + (lane >> 3), cc = 4 * (lane & 7);
        __stcg(reinterpret_cast<float4*>(dst + (size_t)rr * BN + c + cc),
               *reinterpret_cast<const float4*>(stg + rr * 36 + cc));
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  HEAD_MARK(3);
  cluster_sync();   // every partial of the tile is in L2 (release / acquire, cluster scope)
  HEAD_MARK(4);

  // ---- 2. finish rows [rank * rows_per, +rows_per): lane j owns classes [8j, 8j + 8)
  if (warp >= 2) {
    const int e = warp - 2;
    if (kTrain) {
      float tot = 0.f;
      for (int w = 0; w < kHEW; ++w) tot += sh_red[w];
      inv = 1.f / (tot > 0.f ? tot : 1.f);
    }
    HEAD_MARK(5);
    float loss_acc = 0.f;
    const int c8 = lane * 8;
    // the partial sums of every row this warp finishes, all loads in flight at once
    // (the scratch lines are spread over both dies' L2: one round trip, not one per row)
    constexpr int kRW = rows_per / kHEW;
    float vv[kRW][8];
#pragma unroll
    for (int i = 0; i < kRW; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) vv[i][j] = 0.f;
    if (c8 < BN) {
      float4 x[kRW][CL], y[kRW][CL];
#pragma unroll
      for (int i = 0; i < kRW; ++i) {
        const int prow = (int)rank * rows_per + e + i * kHEW;
#pragma unroll
        for (int q = 0; q < CL; ++q) {
          const float4* src = reinterpret_cast<const float4*>(
              tpart + ((size_t)q * kFM + prow) * BN + c8);
          x[i][q] = __ldcg(src);
          y[i][q] = __ldcg(src + 1);
        }
      }
#pragma unroll
      for (int i = 0; i < kRW; ++i)
#pragma unroll
        for (int q = 0; q < CL; ++q) {
          vv[i][0] += x[i][q].x; vv[i][1] += x[i][q].y; vv[i][2] += x[i][q].z;
          vv[i][3] += x[i][q].w; vv[i][4] += y[i][q].x; vv[i][5] += y[i][q].y;
          vv[i][6] += y[i][q].z; vv[i][7] += y[i][q].w;
        }
    }
#pragma unroll
    for (int i = 0; i < kRW; ++i) {
      const int prow = (int)rank * rows_per + e + i * kHEW;
      const int row = t * kFM + prow;
      float* v = vv[i];
      const int64_t lab = my_lab[i];
      if (kTrain) {
        float g[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = 0.f;
        if (lab >= 0) {   // warp-uniform
          float m = -INFINITY;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (c8 + j < tl.C) m = fmaxf(m, v[j]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
          float s = 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (c8 + j < tl.C) s += __expf(v[j] - m);
          s = warp_reduce_sum(s);
          const float lse = m + __logf(s);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (c8 + j < tl.C) g[j] = (__expf(v[j] - lse) - (c8 + j == lab ? 1.f : 0.f)) * inv;
            if (c8 + j == lab) loss_acc += (lse - v[j]) * inv;
          }
        }
        if (row < M && c8 < tl.c_pad) {
          uint4 w;
          __nv_bfloat162 b0 = __floats2bfloat162_rn(g[0], g[1]);
          __nv_bfloat162 b1 = __floats2bfloat162_rn(g[2], g[3]);
          __nv_bfloat162 b2 = __floats2bfloat162_rn(g[4], g[5]);
          __nv_bfloat162 b3 = __floats2bfloat162_rn(g[6], g[7]);
          w.x = *reinterpret_cast<uint32_t*>(&b0);
          w.y = *reinterpret_cast<uint32_t*>(&b1);
          w.z = *reinterpret_cast<uint32_t*>(&b2);
          w.w = *reinterpret_cast<uint32_t*>(&b3);
          *reinterpret_cast<uint4*>(tl.dlog + (int64_t)row * tl.ldd + c8) = w;
        }
      } else if (row < M) {
        // first maximum over [0, C), NaN counting as the maximum (torch.argmax)
        float m = -INFINITY;
        int arg = tl.C;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (c8 + j < tl.C && (v[j] > m || (v[j] != v[j] && m == m))) { m = v[j]; arg = c8 + j; }
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
        if (lane == 0 && lab >= 0) {
          atomicAdd(&sh_cnt[1], 1);
          if (lab == arg) atomicAdd(&sh_cnt[0], 1);
        }
      }
    }
    HEAD_MARK(13);
    if (kTrain) {
      loss_acc = warp_reduce_sum(loss_acc);
      if (lane == 0 && loss_acc != 0.f) atomicAdd(tl.loss, loss_acc);
      // the dlogits rows come back through TMA (async proxy) after the barrier
      asm volatile("fence.proxy.async.global;" ::: "memory");
    } else {
      asm volatile("bar.sync 1, %0;" ::"n"(kHEW * 32) : "memory");
      if (e == 0 && lane == 0 && sh_cnt[1]) {
        atomicAdd(&tl.counts[0], (unsigned long long)sh_cnt[0]);
        atomicAdd(&tl.counts[1], (unsigned long long)sh_cnt[1]);
      }
    }
  }
  if (kTrain) {
    HEAD_MARK(6);
    cluster_sync();   // the tile's dlogits rows are all written
    HEAD_MARK(7);
    // ---- 3. dA[:, Kr] and dW[:, Kr]
    if (warp == 0) {
      if (elect_one()) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mbar_expect_tx(d_full, Cfg::kD);
#pragma unroll
        for (int b = 0; b < 4; ++b)   // classes past c_pad read as zero (tensor-map bounds)
          tma_load_2d(smem_u32(sD) + b * (kFM * 128), &mapD, b * 64, t * kFM, d_full);
      }
    } else if (warp == 1) {
      mbar_wait(d_full, 0);
      tc_fence_after();
      if (elect_one()) {
        // dA: M = 128 rows, N = 64 features, K = BN classes.  A = dlogits (K-major),
        // B = the W block as an MN-major operand (features contiguous, classes rows)
        const uint32_t ia = make_idesc(kFM, 64, 0, 1);
#pragma unroll
        for (int k = 0; k < BN / 16; ++k)
          mma_f16(tmem + kTA,
                  make_desc(smem_u32(sD) + (k >> 2) * (kFM * 128) + (k & 3) * 32, 16, 1024, 2),
                  make_desc(smem_u32(sW) + k * 2048, 8192, 1024, 2), ia, k ? 1u : 0u);
        // dW: M = 128 classes (two halves), N = 64 features, K = 128 rows.  A = the
        // dlogits tile as MN-major (classes contiguous), B = the A block as MN-major
        const uint32_t iw = make_idesc(kFM, 64, 1, 1);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h * kFM >= BN) break;
#pragma unroll
          for (int k = 0; k < kFM / 16; ++k)
            mma_f16(tmem + kTW + h * 64,
                    make_desc(smem_u32(sD) + 2 * h * (kFM * 128) + k * 2048, kFM * 128, 1024, 2),
                    make_desc(smem_u32(sA) + k * 2048, 8192, 1024, 2), iw, k ? 1u : 0u);
        }
        mma_commit(bw_done);
      }
      __syncwarp();
    } else {
      const int e = warp - 2, lg = warp & 3, ch = e >> 2;
      mbar_wait(bw_done, 0);
      HEAD_MARK(8);
      tc_fence_after();
      {   // dA rows lg*32 + lane, features k0 + 32 ch .. +32 (bf16)
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + kTA + (uint32_t)(32 * ch), r);
        const int row = t * kFM + lg * 32 + lane;
        if (row < M) {
          alignas(16) __nv_bfloat16 o[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __float2bfloat16_rn(__uint_as_float(r[j]));
          uint4* d = reinterpret_cast<uint4*>(dA + (int64_t)row * ldda + k0 + 32 * ch);
#pragma unroll
          for (int q = 0; q < 4; ++q) d[q] = reinterpret_cast<const uint4*>(o)[q];
        }
      }
      // dW rows = classes 128 h + lg*32 + lane, features k0 + 32 ch .. +32 (fp32 atomics)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h * kFM >= BN) break;
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + kTW + h * 64 + (uint32_t)(32 * ch), r);
        const int cls = h * kFM + lg * 32 + lane;
        if (cls < tl.c_pad) {
          float* d = dW + (int64_t)cls * lddw + k0 + 32 * ch;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            atomicAdd(reinterpret_cast<float4*>(d) + q,
                      make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                  __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])));
        }
      }
    }
  }
  HEAD_MARK(9);
  tc_fence_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
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

template <int BN, bool kBMN>
static int launch_gemm(const CUtensorMap& mA, const CUtensorMap& mB, const CUtensorMap& mC, int M,
                       int K, const int64_t* m_dev, int pad_fill, int nblk, cudaStream_t st) {
  using Cfg = GemmCfg<BN, kNEW>;
  auto kern = sage_gemm_kernel<BN, kBMN>;
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::kThreads, Cfg::kSmem) !=
            cudaSuccess || per_sm < 1)
      per_sm = 1;
  }
  const int ntiles = (M + kFM - 1) / kFM;
  int grid = num_sms() * per_sm / nblk;
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) grid = 1;
  kern<<<dim3(grid, nblk), Cfg::kThreads, Cfg::kSmem, st>>>(mA, mB, mC, M, K, m_dev, pad_fill);
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  count_launch(1);
  return SAL_OK;
}

template <int BN, int CL, int kEpi>
static int launch_head_cl(const CUtensorMap& mA, const CUtensorMap& mW, const CUtensorMap& mD,
                          int M, const int64_t* m_dev, const GemmTail& tl, float* part,
                          __nv_bfloat16* dA, int64_t ldda, float* dW, int64_t lddw,
                          cudaStream_t st) {
  auto kern = sage_head_kernel<BN, CL, kEpi>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, HeadCfg<BN>::kSmem);
    attr = true;
  }
  const int ntiles = (M + kFM - 1) / kFM;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ntiles * CL);
  cfg.blockDim = dim3(kHThreads);
  cfg.dynamicSmemBytes = HeadCfg<BN>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, mA, mW, mD, M, m_dev, tl, part, dA, ldda, dW, lddw) !=
      cudaSuccess)
    return set_error(SAL_ECUDA, "tc head: launch failed (%s)",
                     cudaGetErrorString(cudaGetLastError()));
  count_launch(1);
  return SAL_OK;
}

template <int BN, int kEpi>
static int launch_head_bn(const CUtensorMap& mA, const CUtensorMap& mW, const CUtensorMap& mD,
                          int M, int K, const int64_t* m_dev, const GemmTail& tl, float* part,
                          __nv_bfloat16* dA, int64_t ldda, float* dW, int64_t lddw,
                          cudaStream_t st) {
  switch (K / kFKB) {   // one CTA per 64-wide K block, the cluster covers K
    case 2:
      return launch_head_cl<BN, 2, kEpi>(mA, mW, mD, M, m_dev, tl, part, dA, ldda, dW, lddw, st);
    case 4:
      return launch_head_cl<BN, 4, kEpi>(mA, mW, mD, M, m_dev, tl, part, dA, ldda, dW, lddw, st);
    default:
      return launch_head_cl<BN, 8, kEpi>(mA, mW, mD, M, m_dev, tl, part, dA, ldda, dW, lddw, st);
  }
}

static int head_bn(int c_pad) { return c_pad <= 64 ? 64 : c_pad <= 128 ? 128 : 192; }

// the output layer (logits = A[M, K] @ W[c_pad, K]^T + loss / score epilogue and, in
// training, dA and dW); the UMMA N is the smallest instantiated width >= c_pad (W rows
// past c_pad read as zero)
template <int kEpi>
static int launch_head(const void* A, int64_t lda, int64_t M, const int64_t* m_dev, int32_t K,
                       const void* W, int64_t ldw, int32_t c_pad, const GemmTail& tl,
                       float* part, __nv_bfloat16* dA, int64_t ldda, float* dW, int64_t lddw,
                       cudaStream_t st) {
  const int bn = head_bn(c_pad);
  CUtensorMap mA, mW, mD;
  if (!make_map(&mA, A, (uint64_t)M, (uint64_t)K, (uint64_t)lda, 64, 128) ||
      !make_map(&mW, W, (uint64_t)c_pad, (uint64_t)K, (uint64_t)ldw, 64, (uint32_t)bn))
    return set_error(SAL_ECUDA, "tc head: cuTensorMapEncodeTiled failed");
  if (kEpi == kEpiNll &&
      !make_map(&mD, tl.dlog, (uint64_t)M, (uint64_t)c_pad, (uint64_t)tl.ldd, 64, 128))
    return set_error(SAL_ECUDA, "tc head: cuTensorMapEncodeTiled failed");
  if (kEpi != kEpiNll) mD = mA;
  switch (bn) {
    case 64:
      return launch_head_bn<64, kEpi>(mA, mW, mD, (int)M, K, m_dev, tl, part, dA, ldda, dW, lddw,
                                      st);
    case 128:
      return launch_head_bn<128, kEpi>(mA, mW, mD, (int)M, K, m_dev, tl, part, dA, ldda, dW, lddw,
                                       st);
    default:
      return launch_head_bn<192, kEpi>(mA, mW, mD, (int)M, K, m_dev, tl, part, dA, ldda, dW, lddw,
                                       st);
  }
}

static int check_logits_args(const void* A, int64_t lda, int32_t K, const void* W, int64_t ldw,
                             int32_t c_pad, int32_t C) {
  if ((K != 128 && K != 256 && K != 512) || c_pad <= 0 || c_pad % 16 || c_pad > 192 || C <= 0 ||
      C > c_pad)
    return set_error(SAL_EINVAL, "tc head: K=%d (128, 256 or 512), c_pad=%d (multiple of 16, "
                     "<= 192), classes=%d (<= c_pad)", K, c_pad, C);
  if (lda % 8 || ldw % 8 || ldw < K || ((uintptr_t)A & 15) || ((uintptr_t)W & 15))
    return set_error(SAL_EINVAL, "tc logits: operands must be 16-byte aligned rows");
  return SAL_OK;
}

}  // namespace tc
}  // namespace sal

extern "C" {

int sal_tc_sage_fwd(const void* A, int64_t lda, int64_t M, const int64_t* m_dev, const void* W,
                    int32_t N, int32_t K, void* Y, int64_t ldy, uint8_t* mask, float p,
                    uint64_t seed, const int64_t* salt_dev, int32_t relu_dropout, void* stream) {
  // two column blocks of 128 (grid.y); each CTA holds its [128 x K] W block
  // (K = 256: layer 0; K = 512: the hidden layer)
  if (N != sal::tc::kFN || (K != 256 && K != 512))
    return sal::set_error(SAL_EINVAL, "tc_sage_fwd: invalid argument (N != sal::tc::kFN || (K != 256 && K != 512))");
  if (lda % 8 || ldy % 8 || ((uintptr_t)A & 15) || ((uintptr_t)W & 15) || ((uintptr_t)Y & 15))
    return sal::set_error(SAL_EINVAL, "tc_sage_fwd: unsupported dtype or shape");
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

int sal_tc_sage_wgrad(const void* dz, int64_t ldz, const void* A, int64_t lda, int64_t M,
                      const int64_t* m_dev, int32_t N, int32_t K, float* dW, int64_t lddw,
                      int32_t accumulate, void* stream) {
  if (N <= 0 || K <= 0 || N % 16 || K % 128)
    return sal::set_error(SAL_EINVAL, "tc_sage_wgrad: N=%d must be a multiple of 16, K=%d of 128",
                          N, K);
  if (ldz % 8 || lda % 8 || ((uintptr_t)dz & 15) || ((uintptr_t)A & 15) || ((uintptr_t)dW & 15) ||
      lddw % 4 || lddw < K)
    return sal::set_error(SAL_EINVAL, "tc_sage_wgrad: operands must be 16-byte aligned");
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
  const int tiles = ((N + 127) / 128) * tiles_k;
  int splits = sal::num_sms() / tiles;
  if (splits < 1) splits = 1;
  int rows = (int)((M + splits - 1) / splits);
  rows = (rows + 63) / 64 * 64;
  // at least 256 rows per split: every split adds a full fp32 tile of atomics, which
  // costs more than its rows at small M (the output layer's 1024 rows)
  if (rows < 256) rows = 256;
  splits = (int)((M + rows - 1) / rows);
  sal::tc::sage_wgrad_tma_kernel<<<dim3(tiles, splits), sal::tc::kQThreads, sal::tc::kQSmem, st>>>(
      mD, mA, (int)M, m_dev, tiles_k, N, dW, lddw);
  if (cudaGetLastError() != cudaSuccess) return SAL_ECUDA;
  sal::count_launch(1);
  return SAL_OK;
}

int sal_tc_gemm_nn(const void* A, int64_t lda, int64_t M, const int64_t* m_dev, int32_t K,
                   const void* B, int64_t ldb, int32_t N, void* C, int64_t ldc, int32_t pad_fill,
                   void* stream) {
  if (K <= 0 || K % 16 || N <= 0 || N % 64)
    return sal::set_error(SAL_EINVAL, "tc_gemm_nn: K=%d must be a multiple of 16, N=%d of 64", K,
                          N);
  if (lda % 8 || ldb % 8 || ldc % 8 || ldb < N || ldc < N || ((uintptr_t)A & 15) ||
      ((uintptr_t)B & 15) || ((uintptr_t)C & 15))
    return sal::set_error(SAL_EINVAL, "tc_gemm_nn: operands must be 16-byte aligned rows");
  if (M <= 0) return SAL_OK;
  CUtensorMap mA, mB, mC;
  if (!sal::tc::make_map(&mA, A, (uint64_t)M, (uint64_t)K, (uint64_t)lda, 64, 128) ||
      !sal::tc::make_map(&mB, B, (uint64_t)K, (uint64_t)N, (uint64_t)ldb, 64, 64) ||
      !sal::tc::make_map(&mC, C, (uint64_t)M, (uint64_t)N, (uint64_t)ldc, 32, 32,
                         CU_TENSOR_MAP_SWIZZLE_64B))
    return sal::set_error(SAL_ECUDA, "tc_gemm_nn: cuTensorMapEncodeTiled failed");
  // 128 x 64 tiles: these GEMMs are small, so many CTAs each pulling little from L2
  // (SAL_GEMM_BN=128/256 selects wider tiles for A/B measurements)
  static int bn = 0;
  if (bn == 0) {
    const char* e = getenv("SAL_GEMM_BN");
    bn = e ? atoi(e) : 64;
    if (bn != 128 && bn != 256) bn = 64;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (bn == 256 && N % 256 == 0)
    return sal::tc::launch_gemm<256, true>(mA, mB, mC, (int)M, K, m_dev, pad_fill, N / 256, st);
  if (bn == 128 && N % 128 == 0)
    return sal::tc::launch_gemm<128, true>(mA, mB, mC, (int)M, K, m_dev, pad_fill, N / 128, st);
  return sal::tc::launch_gemm<64, true>(mA, mB, mC, (int)M, K, m_dev, pad_fill, N / 64, st);
}

#ifdef SAL_HEAD_TRACE
int sal_head_trace_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, sal::tc::sal_head_trace, sizeof(unsigned long long) * 16) ==
                 cudaSuccess
             ? SAL_OK
             : SAL_ECUDA;
}
#endif

size_t sal_tc_sage_head_ws_bytes(int64_t M, int32_t K, int32_t c_pad) {
  if (M <= 0 || K <= 0 || c_pad <= 0) return 0;
  const int64_t ntiles = (M + 127) / 128;
  return (size_t)ntiles * (size_t)(K / 64) * 128u * (size_t)sal::tc::head_bn(c_pad) * 4u;
}

int sal_tc_sage_head(const void* A, int64_t lda, int64_t M, const int64_t* m_dev, int32_t K,
                     const void* W, int64_t ldw, int32_t c_pad, int32_t num_classes,
                     const int64_t* labels, int64_t n_labels, float* loss, void* dlogits,
                     int64_t ldd, void* dA, int64_t ldda, float* dW, int64_t lddw, void* ws,
                     size_t ws_bytes, void* stream) {
  int rc = sal::tc::check_logits_args(A, lda, K, W, ldw, c_pad, num_classes);
  if (rc != SAL_OK) return rc;
  if (labels == nullptr || loss == nullptr || dlogits == nullptr || dA == nullptr ||
      dW == nullptr || ws == nullptr)
    return sal::set_error(SAL_EINVAL, "tc_sage_head: labels, loss, dlogits, dA, dW and the "
                          "workspace are required");
  if (ldd % 8 || ldd < c_pad || ((uintptr_t)dlogits & 15) || ldda % 8 || ldda < K ||
      ((uintptr_t)dA & 15) || lddw % 4 || lddw < K || ((uintptr_t)dW & 15) || ((uintptr_t)ws & 15))
    return sal::set_error(SAL_EINVAL, "tc_sage_head: dlogits / dA / dW rows must be 16-byte "
                          "aligned and wide enough");
  if (ws_bytes < sal_tc_sage_head_ws_bytes(M, K, c_pad))
    return sal::set_error(SAL_EINVAL, "tc_sage_head: workspace of %zu bytes < %zu", ws_bytes,
                          sal_tc_sage_head_ws_bytes(M, K, c_pad));
  if (M <= 0) return SAL_OK;
  sal::tc::GemmTail tl{};
  tl.C = num_classes;
  tl.c_pad = c_pad;
  tl.labels = labels;
  tl.n_labels = n_labels;
  tl.loss = loss;
  tl.dlog = (__nv_bfloat16*)dlogits;
  tl.ldd = ldd;
  return sal::tc::launch_head<sal::tc::kEpiNll>(A, lda, M, m_dev, K, W, ldw, c_pad, tl,
                                                (float*)ws, (__nv_bfloat16*)dA, ldda, dW, lddw,
                                                (cudaStream_t)stream);
}

int sal_tc_sage_logits_argmax(const void* A, int64_t lda, int64_t M, const int64_t* m_dev,
                              int32_t K, const void* W, int64_t ldw, int32_t c_pad,
                              int32_t num_classes, const int64_t* labels, int64_t n_labels,
                              int64_t* counts, void* ws, size_t ws_bytes, void* stream) {
  int rc = sal::tc::check_logits_args(A, lda, K, W, ldw, c_pad, num_classes);
  if (rc != SAL_OK) return rc;
  if (labels == nullptr || counts == nullptr || ws == nullptr || ((uintptr_t)ws & 15))
    return sal::set_error(SAL_EINVAL, "tc_sage_logits_argmax: labels, counts and an aligned "
                          "workspace are required");
  if (ws_bytes < sal_tc_sage_head_ws_bytes(M, K, c_pad))
    return sal::set_error(SAL_EINVAL, "tc_sage_logits_argmax: workspace of %zu bytes < %zu",
                          ws_bytes, sal_tc_sage_head_ws_bytes(M, K, c_pad));
  if (M <= 0) return SAL_OK;
  sal::tc::GemmTail tl{};
  tl.C = num_classes;
  tl.c_pad = c_pad;
  tl.labels = labels;
  tl.n_labels = n_labels;
  tl.counts = (unsigned long long*)counts;
  return sal::tc::launch_head<sal::tc::kEpiArgmax>(A, lda, M, m_dev, K, W, ldw, c_pad, tl,
                                                   (float*)ws, nullptr, 0, nullptr, 0,
                                                   (cudaStream_t)stream);
}

}  // extern "C"
