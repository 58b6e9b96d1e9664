// numpy's SeedSequence(entropy).spawn(count) followed by PCG64(child): the
// per-particle stream states the reference creates at solver.py:278-282,
// computed natively (host code) instead of one Python big-int loop per
// child.  Same arithmetic as paper_1706_04399_b200/solver.py
// (_spawned_pcg64_states), which tests/test_lib_abi.py pins against numpy.
#include <stdint.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "dpso_internal.cuh"

namespace {

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

void spawn_range(const uint32_t* run, int nrun, int64_t lo, int64_t hi,
                 uint64_t* out) {
  const unsigned __int128 mult =
      ((unsigned __int128)2549297995355413924ull << 64) |
      4865540595714422341ull;
  std::vector<uint32_t> ent(nrun + 1);
  for (int64_t c = lo; c < hi; ++c) {
    for (int k = 0; k < nrun; ++k) ent[k] = run[k];
    ent[nrun] = (uint32_t)c;  // spawn key (c,)
    uint32_t hc = kInitA;
    auto hashmix = [&](uint32_t v) {
      v ^= hc;
      hc *= kMultA;
      v *= hc;
      return v ^ (v >> 16);
    };
    auto mix = [](uint32_t x, uint32_t y) {
      uint32_t r = kMixL * x - kMixR * y;
      return r ^ (r >> 16);
    };
    uint32_t pool[4];
    for (int k = 0; k < 4; ++k) pool[k] = hashmix(ent[k]);
    for (int s = 0; s < 4; ++s)
      for (int t = 0; t < 4; ++t)
        if (s != t) pool[t] = mix(pool[t], hashmix(pool[s]));
    for (int s = 4; s < nrun + 1; ++s)
      for (int t = 0; t < 4; ++t) pool[t] = mix(pool[t], hashmix(ent[s]));
    uint32_t hb = kInitB, w32[8];
    for (int k = 0; k < 8; ++k) {
      uint32_t v = pool[k % 4] ^ hb;
      hb *= kMultB;
      v *= hb;
      w32[k] = v ^ (v >> 16);
    }
    uint64_t w64[4];
    for (int j = 0; j < 4; ++j)
      w64[j] = (uint64_t)w32[2 * j] | ((uint64_t)w32[2 * j + 1] << 32);
    // pcg64_set_seed -> pcg_setseq_128_srandom_r
    const unsigned __int128 seed = ((unsigned __int128)w64[0] << 64) | w64[1];
    const unsigned __int128 inc =
        ((((unsigned __int128)w64[2] << 64) | w64[3]) << 1) | 1u;
    unsigned __int128 st = inc + seed;
    st = st * mult + inc;
    uint64_t* o = out + 6 * c;
    o[0] = (uint64_t)(st >> 64);
    o[1] = (uint64_t)st;
    o[2] = (uint64_t)(inc >> 64);
    o[3] = (uint64_t)inc;
    o[4] = 0;
    o[5] = 0;
  }
}

}  // namespace

extern "C" int dpso_spawn_pcg64_states(const uint32_t* entropy_words,
                                       int32_t n_words, int64_t count,
                                       uint64_t* out) {
  if (!entropy_words || n_words < 1 || count < 0 || (count && !out) ||
      count > 0xFFFFFFFFll)
    return dpso::api_fail(DPSO_EINVAL, "bad arguments");
  // a spawn key pads the run entropy to 4 words
  std::vector<uint32_t> run(entropy_words, entropy_words + n_words);
  while (run.size() < 4) run.push_back(0);
  const int64_t per = 4096;
  const int nt = (int)std::min<int64_t>(16, (count + per - 1) / per);
  if (nt <= 1) {
    spawn_range(run.data(), (int)run.size(), 0, count, out);
    return DPSO_OK;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) {
    const int64_t lo = count * t / nt, hi = count * (t + 1) / nt;
    th.emplace_back(spawn_range, run.data(), (int)run.size(), lo, hi, out);
  }
  for (auto& x : th) x.join();
  return DPSO_OK;
}
