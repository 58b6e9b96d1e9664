// Counter-based Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers:
// as easy as 1, 2, 3") for the production RNG mode (DPSO_RNG_PHILOX).
//
// Every draw is a pure function of (seed, purpose, owner, generation,
// counter), so the init, update and mutation draws of all particles are
// independent and generated in parallel — no sequential stream walk.  The
// algorithm consuming the draws is the reference's; only the random numbers
// differ from numpy's, so runs agree with the reference statistically, not
// bit for bit.
#pragma once
#include <stdint.h>

namespace dpso {

enum PhiloxTag : uint32_t {
  kTagInit = 0x494E4954u,    // "INIT"
  kTagUpdate = 0x55504454u,  // "UPDT"
  kTagMutate = 0x4D555441u,  // "MUTA"
};

__host__ __device__ __forceinline__ void philox_round(uint32_t (&c)[4],
                                                      uint32_t k0,
                                                      uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
#ifdef __CUDA_ARCH__
  const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
  const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
#else
  const uint64_t p0 = (uint64_t)M0 * c[0], p1 = (uint64_t)M1 * c[2];
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
  const uint32_t n0 = hi1 ^ c[1] ^ k0;
  const uint32_t n2 = hi0 ^ c[3] ^ k1;
  c[0] = n0;
  c[1] = lo1;
  c[2] = n2;
  c[3] = lo0;
}

__host__ __device__ __forceinline__ void philox4x32_10(uint32_t (&c)[4],
                                                       uint64_t key) {
  uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// A sequential u32 source over counters (owner, gen, tag, i) i = 0, 1, ...
struct PhiloxStream {
  uint64_t key;
  uint32_t owner, gen, tag, ctr;
  uint32_t buf[4];
  int left;

  __host__ __device__ void init(uint64_t k, uint32_t o, uint32_t g,
                                uint32_t t) {
    key = k;
    owner = o;
    gen = g;
    tag = t;
    ctr = 0;
    left = 0;
  }
  __host__ __device__ uint32_t next32() {
    if (left == 0) {
      uint32_t c[4] = {owner, gen, tag, ctr++};
      philox4x32_10(c, key);
      buf[0] = c[0];
      buf[1] = c[1];
      buf[2] = c[2];
      buf[3] = c[3];
      left = 4;
    }
    return buf[4 - left--];
  }
  // uniform double in [0, 1) with 53 random bits
  __host__ __device__ double next_double() {
    const uint32_t a = next32() >> 5, b = next32() >> 6;
    return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
  }
  // uniform integer in [0, rng] (Lemire, exact rejection)
  __host__ __device__ uint32_t bounded(uint32_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return next32();
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
};

// A keyed pseudorandom permutation of [0, n): a balanced 6-round Feistel
// network on 2h bits (2^(2h) >= n, so at most 4n) with cycle walking.  Round
// keys come from a Philox stream; the round function is a 32-bit avalanche
// mixer.  Every image is computed independently, so a CTA or warp fills a
// random permutation (or the first m images: an ordered m-subset) in
// parallel - the bijective-shuffle construction - where numpy's Fisher-Yates
// and Floyd samplers are serial.  Production (Philox) mode only.
struct FeistelPerm {
  static constexpr int kRounds = 6;
  uint32_t n, h, mask;
  uint32_t key[kRounds];

  __host__ __device__ void init(PhiloxStream& r, uint32_t n_) {
    n = n_;
    uint32_t bits = 1;
    while ((1u << bits) < n) ++bits;
    h = (bits + 1) / 2;
    mask = (1u << h) - 1u;
    for (int i = 0; i < kRounds; ++i) key[i] = r.next32();
  }
  __host__ __device__ static uint32_t mix(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
  }
  __host__ __device__ uint32_t round_trip(uint32_t x) const {
    uint32_t L = x >> h, R = x & mask;
#pragma unroll
    for (int i = 0; i < kRounds; ++i) {
      const uint32_t t = L ^ (mix(R ^ key[i]) & mask);
      L = R;
      R = t;
    }
    return (L << h) | R;
  }
  // image of x in [0, n)
  __host__ __device__ uint32_t operator()(uint32_t x) const {
    do {
      x = round_trip(x);
    } while (x >= n);
    return x;
  }
};

}  // namespace dpso
