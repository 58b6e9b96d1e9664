// numpy-compatible PCG64 (XSL-RR 128/64) on the device.
//
// The reference draws every random number through numpy's PCG64 Generator
// (solver.py:180,183,191,246,250,278-282).  To reproduce its runs bit for bit
// the device restates numpy's algorithms exactly (see oracle/np_random.py,
// which is pinned against the installed numpy):
//   next64      : state = state * M + inc (mod 2^128); rotr(hi ^ lo, state>>122)
//   next32      : low half of next64, high half buffered (has_uint32/uinteger)
//   next_double : (next64 >> 11) * 2^-53
//   lemire32    : buffered_bounded_lemire_uint32 (rejection on leftover)
//   interval    : random_interval (mask rejection), used by permutation()
// A jump-ahead (advance) lets many threads read disjoint stretches of one
// stream, which is how the mutation and init streams are parallelised.
#pragma once
#include <stdint.h>

namespace dpso {

struct u128 {
  uint64_t hi, lo;
};

__host__ __device__ __forceinline__ u128 mul128(u128 a, u128 b) {
#ifdef __CUDA_ARCH__
  uint64_t lo = a.lo * b.lo;
  uint64_t hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
#else
  unsigned __int128 p = (unsigned __int128)a.lo * b.lo;
  uint64_t lo = (uint64_t)p;
  uint64_t hi = (uint64_t)(p >> 64) + a.hi * b.lo + a.lo * b.hi;
#endif
  return {hi, lo};
}

__host__ __device__ __forceinline__ u128 add128(u128 a, u128 b) {
  uint64_t lo = a.lo + b.lo;
  uint64_t hi = a.hi + b.hi + (lo < a.lo ? 1ull : 0ull);
  return {hi, lo};
}

// PCG_DEFAULT_MULTIPLIER_128
__host__ __device__ __forceinline__ u128 pcg_mult() {
  return {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};
}

__host__ __device__ __forceinline__ uint64_t pcg_output(u128 s) {
  uint64_t x = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// Persistent stream state as stored in device memory (6 x u64 = 48 B).
struct PcgState {
  uint64_t state_hi, state_lo, inc_hi, inc_lo;
  uint64_t has_uint32;  // 0/1
  uint64_t uinteger;    // buffered high half
};

// LCG jump: returns (A, C) with state_{t+d} = A * state_t + C.
__host__ __device__ inline void pcg_jump_coeffs(uint64_t delta, u128 inc,
                                                u128* A_out, u128* C_out) {
  u128 cur_mult = pcg_mult();
  u128 cur_plus = inc;
  u128 acc_mult = {0, 1};
  u128 acc_plus = {0, 0};
  while (delta > 0) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, {0, 1}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  *A_out = acc_mult;
  *C_out = acc_plus;
}

__host__ __device__ inline u128 pcg_advance(u128 state, u128 inc,
                                            uint64_t delta) {
  u128 A, C;
  pcg_jump_coeffs(delta, inc, &A, &C);
  return add128(mul128(A, state), C);
}

// A sequential reader of one stream, held in registers.
struct Pcg {
  u128 s, inc;
  uint32_t has32;
  uint32_t u32buf;

  __device__ __forceinline__ void load(const PcgState& g) {
    s = {g.state_hi, g.state_lo};
    inc = {g.inc_hi, g.inc_lo};
    has32 = (uint32_t)g.has_uint32;
    u32buf = (uint32_t)g.uinteger;
  }
  __device__ __forceinline__ void store(PcgState& g) const {
    g.state_hi = s.hi;
    g.state_lo = s.lo;
    g.inc_hi = inc.hi;
    g.inc_lo = inc.lo;
    g.has_uint32 = has32;
    g.uinteger = u32buf;
  }
  __device__ __forceinline__ uint64_t next64() {
    s = add128(mul128(s, pcg_mult()), inc);
    return pcg_output(s);
  }
  __device__ __forceinline__ uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32buf;
    }
    uint64_t v = next64();
    has32 = 1;
    u32buf = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  __device__ __forceinline__ double next_double() {
    return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
  }
  // buffered_bounded_lemire_uint32 with rng in [1, 2^32-2]
  __device__ __forceinline__ uint32_t lemire32(uint32_t rng) {
    const uint32_t rng_excl = rng + 1u;
    uint64_t m = (uint64_t)next32() * rng_excl;
    uint32_t leftover = (uint32_t)m;
    if (leftover < rng_excl) {
      const uint32_t threshold = (0xFFFFFFFFu - rng) % rng_excl;
      while (leftover < threshold) {
        m = (uint64_t)next32() * rng_excl;
        leftover = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
  // random_bounded_uint64(state, 0, rng, 0, false) for rng < 2^32
  __device__ __forceinline__ uint32_t bounded(uint32_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return next32();
    return lemire32(rng);
  }
  // random_interval(max) for max < 2^32
  __device__ __forceinline__ uint32_t interval(uint32_t mx) {
    if (mx == 0) return 0;
    uint32_t mask = mx;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    uint32_t v;
    while ((v = (next32() & mask)) > mx) {
    }
    return v;
  }
  // Position this reader at u32 index q of the stream that starts at `g`
  // (q counts next32() calls; used to hand a stretch of a shared stream to
  // an independent thread).
  __device__ inline void seek_u32(const PcgState& g, uint64_t q) {
    load(g);
    if (q == 0) return;
    uint64_t fresh = q - has32;  // has32 == 1: first u32 came from buffer
    uint64_t outs = fresh / 2;
    s = pcg_advance(s, inc, outs);
    if (fresh & 1) {
      uint64_t v = next64();
      has32 = 1;
      u32buf = (uint32_t)(v >> 32);
    } else {
      has32 = 0;
    }
  }
};

// Lemire rejection predicate for a raw u32 draw (true = draw is rejected).
__device__ __forceinline__ bool lemire_rejects(uint32_t u, uint32_t rng) {
  const uint32_t rng_excl = rng + 1u;
  uint32_t leftover = (uint32_t)((uint64_t)u * rng_excl);
  if (leftover >= rng_excl) return false;
  const uint32_t threshold = (0xFFFFFFFFu - rng) % rng_excl;
  return leftover < threshold;
}

}  // namespace dpso
