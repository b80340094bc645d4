// Draw -> position of the per-destination rejection sampler, shared by the
// hop kernels (hop.cu) and the fused last-hop aggregation (sample_mean.cu).
// Reference: _kernels.py:30-39 (splitmix64 stream), :119-146 (_sample_positions).
#pragma once

#include "common.cuh"
#include "salient_internal.h"

namespace sal {

// Exact z % d for d in [1, 2^32) without the u64 division routine: with the
// per-destination reciprocal m = floor((2^64-1)/d), q = umulhi(z, m) is at most
// 2 below floor(z/d), so r = z - q*d needs at most two corrections.
SAL_DEVINL uint32_t mod_by_recip(uint64_t z, uint32_t d, uint64_t m) {
  const uint64_t q = __umul64hi(z, m);
  uint64_t r = z - q * (uint64_t)d;
  if (r >= d) r -= d;
  if (r >= d) r -= d;
  return (uint32_t)r;
}

// floor((2^64-1)/d) for d in [1, 2^32) without the u64 division routine (a call,
// ~70 instructions and register pressure around it): q from the correctly
// rounded fp64 reciprocal is within ~2^10 of the answer, the remainder
// rem = (2^64-1) - q*d is exact in wrapping u64 arithmetic read as int64 (its true
// magnitude is < 2^43), one fp64 step brings it within one d, and the loops
// restore 0 <= rem < d — so the result is exact whatever the approximation error.
SAL_DEVINL uint64_t recip_u32(uint32_t d) {
  if (d <= 1) return ~0ull;
  const double r = __drcp_rn((double)d);
  uint64_t q = (uint64_t)(r * 18446744073709551616.0);  // r * 2^64 < 2^63
  int64_t rem = (int64_t)(~0ull - q * (uint64_t)d);
  const int64_t k = (int64_t)floor((double)rem * r);
  q += (uint64_t)k;
  rem -= k * (int64_t)d;
  while (rem < 0) {
    --q;
    rem += d;
  }
  while (rem >= (int64_t)d) {
    ++q;
    rem -= d;
  }
  return q;
}

// Draw -> position for the two RNG policies.  recip = floor((2^64-1)/deg).
template <int kPolicy>
SAL_DEVINL uint32_t draw_position(uint64_t key, uint2 pkey, uint32_t ctr, uint32_t dst,
                                  uint32_t hop, uint32_t batch, uint32_t deg, uint64_t recip) {
  if (kPolicy == kRngSplitmix) {
    // _kernels.py:37-39 + 120: mix64(key + (c+1)G) % deg  (u64 modulo)
    const uint64_t z = mix64(key + (uint64_t)(ctr + 1) * kGolden);
    return mod_by_recip(z, deg, recip);
  } else {
    const uint4 r = philox4x32_10(make_uint4(ctr, dst, hop, batch), pkey);
    return (uint32_t)(((uint64_t)r.x * deg) >> 32);
  }
}

// id-table word of a new key: {key:32 | kNewFlag | first_edge:31} (hop.cu)
constexpr uint32_t kNewFlag = 0x80000000u;

// Deferred relabel pass 2 of the last sampled hop of a fused plan, run by the fused
// last hop's kernel: every edge resolves its local id from the table word flag_scan
// kept for it (no table access; first occurrences need no finalising, the table is
// not read again for this batch)
SAL_DEVINL void resolve_words(const ResolveJob& j, int64_t first, int64_t stride) {
  const int64_t n = *j.e_total;
  const int64_t size_old = *j.size_old;
  for (int64_t e = first; e < n; e += stride) {
    const uint32_t lo = (uint32_t)j.words[e];
    j.src_local[e] = (lo & kNewFlag) ? (int32_t)(size_old + j.rank_of[lo & ~kNewFlag])
                                     : (int32_t)lo;
  }
}

}  // namespace sal
