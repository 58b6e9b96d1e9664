// Random mutation with elitism and canonical-form dedupe (solver.py:222-258).
//
// Pipeline (all kernels no-op unless ctl->mutating):
//   k_mut_hash    per particle: canonical rotation/direction (graph.py:106-115)
//                 and a 64-bit order-dependent hash of the canonical sequence
//   k_mut_rank    rank in (fitness, slot) order by counting (solver.py:223-224)
//   k_mut_dedupe  earliest-ranked particle with the same hash (candidate
//                 duplicate source)
//   k_mut_verify  one warp per candidate: exact canonical-form comparison
//                 (a hash collision falls back to an exact search)
//   k_mut_lists   survivors / dropped in rank order, keep = first ceil(S/3)
//                 survivors, events = non-kept slots in slot order
//   k_mut_copy    dropped #r copies body+fitness of survivors[r % S]
//   k_mut_walk    chains k = integers(1, k_hi+1) through the single mutation
//                 stream to find where every event's draws start.  The chain
//                 depends only on the stream, not on the swarm, so it is
//                 computed for all P potential events on a forked stream,
//                 concurrently with update/hash/rank/dedupe/lists/copy
//   k_mut_sample  one warp per event: regenerate its draws in parallel (PCG64
//                 jump-ahead), check Lemire rejections in parallel, numpy's
//                 Floyd sampler + shuffle (sequential, on precomputed values)
//   k_mut_fix     exact sequential re-walk from the first event whose draws
//                 needed a Lemire redraw (rare); persistent stream update
//   k_mut_swap    k disjoint swaps, fitness in reference order, pbest
//                 (solver.py:241-258)
#include <algorithm>

#include "dpso_internal.cuh"

namespace dpso {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// canonical element m (1 <= m < n) of tour t with 0 at position k
__device__ __forceinline__ int canon_at(const uint16_t* t, int n, int k,
                                        int rev, int m) {
  int idx = rev ? (k - m + n) % n : (k + m) % n;
  return t[idx];
}

__global__ void __launch_bounds__(128) k_mut_hash(SwarmView v,
                                                  int32_t* canon) {
  if (!v.ctl->mutating || v.ctl->done) return;
  const int p = blockIdx.x, n = v.n, tid = threadIdx.x;
  const uint16_t* t = v.x + (size_t)p * v.np;
  __shared__ int s_k;
  __shared__ unsigned long long s_h;
  if (tid == 0) s_h = 0ull;
  for (int i = tid; i < n; i += blockDim.x)
    if (t[i] == 0) s_k = i;
  __syncthreads();
  const int k = s_k;
  const int rev = (n > 2) && (t[(k - 1 + n) % n] < t[(k + 1) % n]);
  uint64_t h = 0;
  for (int m = 1 + tid; m < n; m += blockDim.x)
    h += mix64(((uint64_t)m << 32) | (uint64_t)canon_at(t, n, k, rev, m));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((tid & 31) == 0) atomicAdd(&s_h, (unsigned long long)h);
  __syncthreads();
  if (tid == 0) {
    v.hash[p] = s_h;
    canon[p] = k | (rev << 31);
  }
}

constexpr int kTile = 2048;

__global__ void __launch_bounds__(256) k_mut_rank(SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  __shared__ double s_f[kTile];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double fi = i < v.P ? v.fit[i] : 0.0;
  int cnt = 0;
  for (int base = 0; base < v.P; base += kTile) {
    const int m = min(kTile, v.P - base);
    __syncthreads();
    for (int u = threadIdx.x; u < m; u += blockDim.x) s_f[u] = v.fit[base + u];
    __syncthreads();
    if (i < v.P) {
      for (int u = 0; u < m; ++u) {
        const double f = s_f[u];
        const int j = base + u;
        cnt += (f < fi) || (f == fi && j < i);
      }
    }
  }
  if (i < v.P) {
    v.rank[i] = cnt;
    v.order[cnt] = i;
  }
}

// Earliest-ranked particle with the same canonical hash and a lower rank
// (-1: none) -> flag[i] holds that candidate + 1 until k_mut_verify.
__global__ void __launch_bounds__(256) k_mut_dedupe(SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  __shared__ unsigned long long s_h[kTile];
  __shared__ int s_r[kTile];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t hi = i < v.P ? v.hash[i] : 0;
  const int ri = i < v.P ? v.rank[i] : 0;
  int cand = -1, crank = 0x7fffffff;
  for (int base = 0; base < v.P; base += kTile) {
    const int m = min(kTile, v.P - base);
    __syncthreads();
    for (int u = threadIdx.x; u < m; u += blockDim.x) {
      s_h[u] = v.hash[base + u];
      s_r[u] = v.rank[base + u];
    }
    __syncthreads();
    if (i < v.P) {
      for (int u = 0; u < m; ++u) {
        const int r = s_r[u];
        if (s_h[u] == hi && r < ri && r < crank) {
          crank = r;
          cand = base + u;
        }
      }
    }
  }
  if (i < v.P) v.flag[i] = cand + 1;
}

__device__ bool warp_canon_equal(const SwarmView& v, const int32_t* canon,
                                 int a, int b) {
  const int n = v.n, lane = threadIdx.x & 31;
  const uint16_t* ta = v.x + (size_t)a * v.np;
  const uint16_t* tb = v.x + (size_t)b * v.np;
  const int ka = canon[a] & 0x7fffffff, ra = (int)((uint32_t)canon[a] >> 31);
  const int kb = canon[b] & 0x7fffffff, rb = (int)((uint32_t)canon[b] >> 31);
  int diff = 0;
  for (int m = 1 + lane; m < n; m += 32)
    diff |= canon_at(ta, n, ka, ra, m) != canon_at(tb, n, kb, rb, m);
  return !__any_sync(0xffffffffu, diff);
}

// One warp per particle: exact check of the hash candidate.  A particle is a
// dropped duplicate iff an earlier-ranked particle has the same canonical
// form (solver.py:227-233).  flag: 1 = dropped, 0 = survivor.
__global__ void __launch_bounds__(128) k_mut_verify(SwarmView v,
                                                    const int32_t* canon) {
  if (!v.ctl->mutating || v.ctl->done) return;
  const int i = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (i >= v.P) return;
  const int cand = v.flag[i] - 1;
  if (cand < 0) return;  // flag already 0
  int dropped = warp_canon_equal(v, canon, i, cand);
  if (!dropped) {
    // 64-bit hash collision with a different tour: exact search over every
    // earlier-ranked particle with the same hash (never seen in practice)
    if ((threadIdx.x & 31) == 0) v.ctl->collision = 1;
    const uint64_t hi = v.hash[i];
    const int ri = v.rank[i];
    for (int j = 0; j < v.P && !dropped; ++j)
      if (j != cand && v.hash[j] == hi && v.rank[j] < ri)
        dropped = warp_canon_equal(v, canon, i, j);
  }
  if ((threadIdx.x & 31) == 0) v.flag[i] = dropped;
}

template <int T>
__device__ int block_scan_excl(int val, int* s_w, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = val;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < T / 32 ? s_w[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < T / 32) s_w[lane] = w;
  }
  __syncthreads();
  int base = warp ? s_w[warp - 1] : 0;
  *total = s_w[T / 32 - 1];
  __syncthreads();
  return base + x - val;
}

__global__ void __launch_bounds__(1024) k_mut_lists(SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  __shared__ int s_w[32];
  const int P = v.P, tid = threadIdx.x;
  int surv_run = 0;
  for (int base = 0; base < P; base += 1024) {
    const int r = base + tid;
    const int i = r < P ? v.order[r] : 0;
    const int s = (r < P) ? !v.flag[i] : 0;
    int tot;
    const int ex = block_scan_excl<1024>(s, s_w, &tot);
    if (r < P) {
      if (s) {
        v.sidx[i] = surv_run + ex;
        v.surv_list[surv_run + ex] = i;
      } else {
        v.sidx[i] = r - (surv_run + ex);  // dropped index in rank order
      }
    }
    surv_run += tot;
  }
  const int S = surv_run;
  const int nkeep = (S + 2) / 3;  // ceil(S / 3)
  __syncthreads();
  int ev_run = 0;
  for (int base = 0; base < P; base += 1024) {
    const int i = base + tid;
    int kp = 0;
    if (i < P) {
      kp = !v.flag[i] && v.sidx[i] < nkeep;
      v.keep[i] = kp;
    }
    const int e = (i < P) && !kp;
    int tot;
    const int ex = block_scan_excl<1024>(e, s_w, &tot);
    if (e) v.ev_slot[ev_run + ex] = i;
    ev_run += tot;
  }
  if (tid == 0) {
    v.ctl->n_surv = S;
    v.ctl->n_drop = P - S;
    v.ctl->n_events = ev_run;
  }
}

__global__ void __launch_bounds__(128) k_mut_copy(SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  const int p = blockIdx.x;
  if (!v.flag[p]) return;
  const int S = v.ctl->n_surv;
  const int src = v.surv_list[v.sidx[p] % S];
  const uint16_t* a = v.x + (size_t)src * v.np;
  uint16_t* b = v.x + (size_t)p * v.np;
  for (int i = threadIdx.x; i < v.n; i += blockDim.x) b[i] = a[i];
  if (threadIdx.x == 0) v.fit[p] = v.fit[src];
}

// ---- the sequential stream walk ------------------------------------------
//
// The mutation stream is ONE numpy PCG64 stream consumed in slot order, so
// where event e's draws start depends on every earlier event's k.  The walk
// is split: (1) k_mut_walk chains only the k-draws (one thread, reading a
// shared-memory ring of the stream that the whole CTA refills: every thread
// holds the jump coefficients for its own offset, so a refill is one 128-bit
// multiply-add per generated output), assuming the Floyd/shuffle draws of
// each event need no Lemire redraw; (2) k_mut_sample verifies that
// assumption per event; (3) k_mut_fix redoes the walk exactly and
// sequentially from the first event that needed a redraw (rare path).

constexpr int kWalk = 1024;          // threads
constexpr int kRingSmem = 32768;     // u32 ring in shared memory (128 KiB)

// number of Floyd + shuffle draws of choice(n, 2k, replace=False) when no
// Lemire redraw happens (numpy _generator.pyx: Floyd skips j == 0; n > 10000
// with 2k > n // 50 uses the tail shuffle instead)
__device__ __forceinline__ int sample_draws(int n, int k) {
  const int size = 2 * k;
  const int jstart = max(n - size, 1);
  const int F = n - jstart;
  if (n > 10000 && size > n / 50) return F;
  return F + size - 1;
}

__device__ __forceinline__ uint32_t sample_bound(int n, int k, int d) {
  const int size = 2 * k;
  const int jstart = max(n - size, 1);
  const int F = n - jstart;
  if (n > 10000 && size > n / 50) return (uint32_t)(n - 1 - d);  // tail
  return d < F ? (uint32_t)(jstart + d) : (uint32_t)(size - 1 - (d - F));
}

constexpr int kWinEvents = 256;  // events chained per ring window (max)

// Ring size in u32 for n nodes: >= 4x the worst-case span of one event.
__host__ __device__ inline int64_t walk_ring_size(int n) {
  int64_t need = 4 * (64 + 2 * (int64_t)n);
  int64_t r = kRingSmem;
  while (r < need) r *= 2;
  return r;
}

__global__ void __launch_bounds__(kWalk) k_mut_walk(SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  extern __shared__ __align__(16) uint32_t ring_smem[];
  const int64_t kRing = walk_ring_size(v.n);
  // large n: the ring lives in global memory (L2)
  uint32_t* ring = kRing == kRingSmem ? ring_smem : v.walk_ring;
  const int out_per_thread = (int)(kRing / 2 / kWalk);
  __shared__ int64_t s_q, s_wbase;
  __shared__ int s_e, s_e0;
  __shared__ uint64_t s_base[2];
  __shared__ unsigned long long s_bad;  // (position << 16 | event offset)
  __shared__ int s_ek[kWinEvents];
  __shared__ int64_t s_ec[kWinEvents];
  const int tid = threadIdx.x;
  const PcgState g = v.streams[1];
  if (tid == 0) {
    *v.mut_start = g;
    s_q = 0;
    s_e = 0;
    s_wbase = -(int64_t)kRing;  // force a fill
    v.ctl->mut_bad = 0x7fffffff;
  }
  const int64_t h = (int64_t)g.has_uint32;
  const uint32_t ub = (uint32_t)g.uinteger;
  const u128 S0 = {g.state_hi, g.state_lo}, inc = {g.inc_hi, g.inc_lo};
  u128 A, C, At, Ct;
  pcg_jump_coeffs(kWalk, inc, &A, &C);
  pcg_jump_coeffs((uint64_t)tid, inc, &At, &Ct);
  const int n = v.n;
  const int k_hi = max(2, n / 4);
  const uint32_t rng_k = (uint32_t)(k_hi - 1);
  const int E = v.P;  // every potential event; k_mut_lists picks the first E
  const int margin = 64 + sample_draws(n, n / 2);  // worst-case event span
  __syncthreads();
  auto at = [&](int64_t q) -> uint32_t {
    return q < h ? ub : ring[q - h - s_wbase];
  };
  for (;;) {
    // refill so the ring starts at the chain position
    const int64_t f = s_q - h;
    if (f < 0 || f + margin > s_wbase + kRing) {
      const int64_t wb = f < 0 ? 0 : (f & ~(int64_t)1);
      if (tid == 0) {
        const u128 b = pcg_advance(S0, inc, (uint64_t)(wb / 2 + 1));
        s_base[0] = b.hi;
        s_base[1] = b.lo;
      }
      __syncthreads();
      u128 st = add128(mul128(At, {s_base[0], s_base[1]}), Ct);
      for (int r = 0; r < out_per_thread; ++r) {
        const uint64_t o = pcg_output(st);
        const int idx = 2 * (tid + kWalk * r);
        ring[idx] = (uint32_t)o;
        ring[idx + 1] = (uint32_t)(o >> 32);
        st = add128(mul128(A, st), C);
      }
      __syncthreads();
      if (tid == 0) s_wbase = wb;
      __syncthreads();
    }
    // (1) chain k-draws of the events whose whole draw span is in the ring
    if (tid == 0) {
      int64_t q = s_q;
      int e = s_e;
      s_e0 = e;
      while (e < E && e - s_e0 < kWinEvents) {
        if (q - h + margin > s_wbase + kRing) break;
        uint32_t u;
        do {
          u = at(q);
          ++q;
        } while (lemire_rejects(u, rng_k));
        const int kraw = (int)(((uint64_t)u * (rng_k + 1u)) >> 32) + 1;
        const int k = min(kraw, n / 2);
        s_ek[e - s_e0] = k;
        s_ec[e - s_e0] = q;
        if (k >= 1) q += sample_draws(n, k);
        ++e;
      }
      s_q = q;
      s_e = e;
      s_bad = ~0ull;
    }
    __syncthreads();
    // (2) every draw of those events checked for a Lemire redraw: warp w
    //     checks events w, w + 32, ... with its 32 lanes
    const int e0 = s_e0, ne = s_e - s_e0;
    const int lane = tid & 31, warp = tid >> 5;
    for (int w = warp; w < ne; w += kWalk / 32) {
      const int k = s_ek[w];
      if (k < 1) continue;
      const int D = sample_draws(n, k);
      const int64_t c0 = s_ec[w];
      int bad = 0x7fffffff;
      for (int d = lane; d < D; d += 32)
        if (bad == 0x7fffffff &&
            lemire_rejects(at(c0 + d), sample_bound(n, k, d)))
          bad = d;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
      if (lane == 0 && bad != 0x7fffffff)
        atomicMin(&s_bad, ((unsigned long long)(c0 + bad) << 16) | w);
    }
    __syncthreads();
    // (3) commit every event before the first one with a redraw (all warps),
    //     then thread 0 consumes that event exactly (redraws stay inside the
    //     ring margin) and the chain resumes after it
    const int upto = s_bad == ~0ull ? ne : (int)(s_bad & 0xFFFF);
    for (int w = tid; w < upto; w += kWalk) {
      const int k = s_ek[w];
      v.ev_k[e0 + w] = k;
      v.ev_cursor[e0 + w] = (uint64_t)s_ec[w];
      v.ev_end[e0 + w] =
          (uint64_t)(s_ec[w] + (k >= 1 ? sample_draws(n, k) : 0));
    }
    if (tid == 0) {
      if (upto < ne) {
        const int w = upto, k = s_ek[w];
        int64_t q = s_ec[w];
        const int D = sample_draws(n, k);
        bool ok = true;
        for (int d = 0; d < D && ok; ++d) {
          const uint32_t rng = sample_bound(n, k, d);
          if (rng == 0) continue;
          for (;;) {
            if (q - h - s_wbase >= kRing) {
              ok = false;  // redraw run beyond the ring: exact re-walk
              break;
            }
            if (!lemire_rejects(at(q), rng)) break;
            ++q;
          }
          ++q;
        }
        if (ok) {
          v.ev_k[e0 + w] = k;
          v.ev_cursor[e0 + w] = (uint64_t)s_ec[w];
          v.ev_end[e0 + w] = (uint64_t)q;
          s_q = q;
          s_e = e0 + w + 1;
        } else {
          v.ctl->mut_bad = e0 + w;  // k_mut_fix redoes events >= w exactly
          s_e = E;
        }
      }
    }
    __syncthreads();
    if (s_e >= E) break;
  }
}

// Numpy's choice(n, 2k, replace=False) from stream position `cur`, one
// thread: writes the 2k sampled positions to idx; returns the u32 consumed.
__device__ int64_t sample_event_seq(const PcgState& start, uint64_t cur,
                                    int n, int k, uint16_t* idx,
                                    uint32_t* bits, uint16_t* arr) {
  struct Counting {
    Pcg r;
    int64_t q = 0;
    __device__ uint32_t bounded(uint32_t rng) {
      if (rng == 0) return 0;
      const uint32_t rng_excl = rng + 1u;
      ++q;
      uint64_t m = (uint64_t)r.next32() * rng_excl;
      uint32_t leftover = (uint32_t)m;
      if (leftover < rng_excl) {
        const uint32_t threshold = (0xFFFFFFFFu - rng) % rng_excl;
        while (leftover < threshold) {
          ++q;
          m = (uint64_t)r.next32() * rng_excl;
          leftover = (uint32_t)m;
        }
      }
      return (uint32_t)(m >> 32);
    }
  } c;
  c.r.seek_u32(start, cur);
  const int size = 2 * k;
  if (n > 10000 && size > n / 50) {
    const int first = max(n - size, 1);
    for (int i = n - 1; i >= first; --i) {
      uint32_t j = c.bounded((uint32_t)i);
      uint16_t t = arr[i];
      arr[i] = arr[j];
      arr[j] = t;
    }
    for (int t = 0; t < size; ++t) idx[t] = arr[n - size + t];
  } else {
    for (int t = 0; t < size; ++t) {
      const uint32_t j = (uint32_t)(n - size + t);
      uint32_t val = c.bounded(j);
      if (bits[val >> 5] & (1u << (val & 31))) val = j;
      bits[val >> 5] |= 1u << (val & 31);
      idx[t] = (uint16_t)val;
    }
    for (int i = size - 1; i >= 1; --i) {
      uint32_t j = c.bounded((uint32_t)i);
      uint16_t t = idx[i];
      idx[i] = idx[j];
      idx[j] = t;
    }
  }
  return c.q;
}

// One warp per event.  Shared memory per warp: draw values (u32, D+1) and
// the n-bit Floyd bitmap (or arange(n) for the tail shuffle).
constexpr int kSampleWarps = 4;

__global__ void __launch_bounds__(kSampleWarps * 32) k_mut_sample(
    SwarmView v, int vals_cap, int scratch_words) {
  if (!v.ctl->mutating || v.ctl->done) return;
  extern __shared__ __align__(16) uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * (blockDim.x >> 5) + warp;
  if (e >= v.ctl->n_events) return;
  const int n = v.n, k = v.ev_k[e];
  if (k < 1) return;
  uint32_t* vals = sm + (size_t)warp * (vals_cap + scratch_words);
  uint32_t* bits = vals + vals_cap;
  uint16_t* arr = (uint16_t*)bits;
  uint16_t* idx = v.ev_idx + (size_t)e * v.np;
  const int size = 2 * k;
  const bool tail = (n > 10000) && size > n / 50;
  const uint64_t cur = v.ev_cursor[e];
  const int D = sample_draws(n, k);
  if (tail || vals_cap == 0) {
    // sequential sampler (tail shuffle, or n too large for a draw buffer)
    if (tail) {
      for (int i = lane; i < n; i += 32) arr[i] = (uint16_t)i;
    } else {
      for (int i = lane; i < (n + 31) / 32; i += 32) bits[i] = 0;
    }
    __syncwarp();
    if (lane == 0) sample_event_seq(*v.mut_start, cur, n, k, idx, bits, arr);
    return;
  }
  for (int i = lane; i < (n + 31) / 32; i += 32) bits[i] = 0;
  // --- generate the event's D draws in parallel
  const PcgState& g = *v.mut_start;
  const int64_t h = (int64_t)g.has_uint32;
  const u128 inc = {g.inc_hi, g.inc_lo};
  // fresh index of the first draw; outputs counted from 1
  const int64_t f0 = (int64_t)cur - h;  // >= 0: the k draw precedes cur
  const int64_t m0 = f0 / 2 + 1;
  const int skip = (int)(f0 & 1);  // first draw is the high half of m0
  const int nout = (skip + D + 1) / 2;
  u128 Al, Cl, A32, C32;
  pcg_jump_coeffs((uint64_t)lane, inc, &Al, &Cl);
  pcg_jump_coeffs(32, inc, &A32, &C32);
  u128 base = {0, 0};
  if (lane == 0)
    base = pcg_advance({g.state_hi, g.state_lo}, inc, (uint64_t)m0);
  base.hi = __shfl_sync(0xffffffffu, base.hi, 0);
  base.lo = __shfl_sync(0xffffffffu, base.lo, 0);
  u128 st = add128(mul128(Al, base), Cl);
  for (int o = lane; o < nout; o += 32) {
    const uint64_t out = pcg_output(st);
    const int d0 = 2 * o - skip;  // draw index of the low half
    if (d0 >= 0 && d0 < D) vals[d0] = (uint32_t)out;
    if (d0 + 1 >= 0 && d0 + 1 < D) vals[d0 + 1] = (uint32_t)(out >> 32);
    st = add128(mul128(A32, st), C32);
  }
  __syncwarp();
  // --- rejection check and bounded values, in parallel
  const int jstart = max(n - size, 1);
  const int F = n - jstart;
  int rej = 0;
  for (int d = lane; d < D; d += 32) {
    const uint32_t rng = d < F ? (uint32_t)(jstart + d)
                               : (uint32_t)(size - 1 - (d - F));
    const uint32_t u = vals[d];
    rej |= lemire_rejects(u, rng);
    vals[d] = (uint32_t)(((uint64_t)u * (rng + 1u)) >> 32);
  }
  if (__any_sync(0xffffffffu, rej)) {
    // this event holds a Lemire redraw (the walk accounted for it): sample
    // it exactly, sequentially
    __syncwarp();
    if (lane == 0) {
      for (int i = 0; i < (n + 31) / 32; ++i) bits[i] = 0;
      sample_event_seq(*v.mut_start, cur, n, k, idx, bits, arr);
    }
    return;
  }
  __syncwarp();
  if (lane == 0) {
    // Floyd: j = n - 2k .. n-1 (j == 0 takes no draw and yields 0)
    int d = 0;
    for (int t = 0; t < size; ++t) {
      const uint32_t j = (uint32_t)(n - size + t);
      uint32_t val = j == 0 ? 0u : vals[d++];
      if (bits[val >> 5] & (1u << (val & 31))) val = j;
      bits[val >> 5] |= 1u << (val & 31);
      idx[t] = (uint16_t)val;
    }
    // shuffle (numpy _shuffle_int): i = size-1 .. 1
    for (int i = size - 1; i >= 1; --i) {
      const uint32_t j = vals[d++];
      const uint16_t t = idx[i];
      idx[i] = idx[j];
      idx[j] = t;
    }
  }
}

// Rare path + stream bookkeeping: exact sequential re-walk from the first
// event the walk could not resolve (a redraw run beyond the ring margin,
// never seen), then advance the persistent stream past the last event used.
__global__ void __launch_bounds__(32) k_mut_fix(SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  if (threadIdx.x != 0) return;
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* bits = (uint32_t*)smem;
  uint16_t* arr = (uint16_t*)smem;
  const int n = v.n;
  const int E = v.ctl->n_events;
  const int bad = v.ctl->mut_bad;
  uint64_t q = 0;
  if (bad < E) {
    const int k_hi = max(2, n / 4);
    const uint32_t rng_k = (uint32_t)(k_hi - 1);
    if (bad > 0) q = v.ev_end[bad - 1];
    for (int e = bad; e < E; ++e) {
      Pcg r;
      r.seek_u32(*v.mut_start, q);
      uint32_t u;
      do {
        u = r.next32();
        ++q;
      } while (lemire_rejects(u, rng_k));
      const int kraw = (int)(((uint64_t)u * (rng_k + 1u)) >> 32) + 1;
      const int k = min(kraw, n / 2);
      v.ev_k[e] = k;
      v.ev_cursor[e] = q;
      if (k < 1) continue;
      const bool tail = (n > 10000) && 2 * k > n / 50;
      if (tail) {
        for (int i = 0; i < n; ++i) arr[i] = (uint16_t)i;
      } else {
        for (int i = 0; i < (n + 31) / 32; ++i) bits[i] = 0;
      }
      q += sample_event_seq(*v.mut_start, q, n, k,
                            v.ev_idx + (size_t)e * v.np, bits, arr);
    }
  } else if (E > 0) {
    q = v.ev_end[E - 1];
  }
  Pcg r;
  r.seek_u32(*v.mut_start, q);
  r.store(v.streams[1]);
  v.ctl->mut_q = q;
}

__global__ void __launch_bounds__(128) k_mut_swap(SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  const int e = blockIdx.x;
  if (e >= v.ctl->n_events) return;
  extern __shared__ __align__(16) unsigned char smem[];
  double* sd = (double*)smem;
  const int n = v.n, np = v.np, tid = threadIdx.x;
  const int p = v.ev_slot[e];
  const int k = v.ev_k[e];
  if (k < 1) return;
  const uint16_t* idx = v.ev_idx + (size_t)e * np;
  uint16_t* body = v.x + (size_t)p * np;
  // the k position pairs are disjoint (sampled without replacement)
  for (int t = tid; t < k; t += blockDim.x) {
    const int a = idx[2 * t], b = idx[2 * t + 1];
    const uint16_t x = body[a];
    body[a] = body[b];
    body[b] = x;
  }
  __syncthreads();
  double* dg = v.dcache + (size_t)p * np;
  for (int i = tid; i < n; i += blockDim.x) {
    const int a = body[i], b = body[i + 1 == n ? 0 : i + 1];
    const double d = v.cost[(size_t)a * v.ld + b];
    sd[i] = d;
    dg[i] = d;
  }
  __syncthreads();
  __shared__ int s_better;
  if (tid == 0) {
    const double f = seq_tour_sum(sd, n);
    v.fit[p] = f;
    s_better = f < v.pfit[p];
    if (s_better) v.pfit[p] = f;
  }
  __syncthreads();
  if (s_better) {
    uint16_t* pb = v.pbest + (size_t)p * np;
    for (int i = tid; i < n; i += blockDim.x) pb[i] = body[i];
  }
}

}  // namespace

int64_t walk_ring_bytes(int n) {
  const int64_t r = walk_ring_size(n);
  return r == kRingSmem ? 0 : 4 * r;  // global ring only when smem is short
}

cudaError_t launch_mutation_walk(const SwarmView& v, cudaStream_t s) {
  const size_t ring = (size_t)kRingSmem * 4;
  set_dyn_smem((const void*)k_mut_walk, ring);
  k_mut_walk<<<1, kWalk, ring, s>>>(v);
  return cudaGetLastError();
}

cudaError_t launch_mutation_pre(const SwarmView& v, cudaStream_t s) {
  const int P = v.P;
  // canon info (k | rev << 31) lives in the rank-order scratch `keep` until
  // k_mut_lists rewrites it
  int32_t* canon = v.keep;
  k_mut_hash<<<P, 128, 0, s>>>(v, canon);
  k_mut_rank<<<(P + 255) / 256, 256, 0, s>>>(v);
  k_mut_dedupe<<<(P + 255) / 256, 256, 0, s>>>(v);
  k_mut_verify<<<(P + 3) / 4, 128, 0, s>>>(v, canon);
  k_mut_lists<<<1, 1024, 0, s>>>(v);
  k_mut_copy<<<P, 128, 0, s>>>(v);
  return cudaGetLastError();
}

cudaError_t launch_mutation_post(const SwarmView& v, cudaStream_t s) {
  const int P = v.P;
  const int n = v.n;
  // per warp: draw values (<= 2n + 1 u32) + Floyd bitmap / tail arange;
  // without room for the draw buffer the warp samples sequentially
  const int scratch_words =
      (int)round_up(std::max<int64_t>((n + 31) / 32, (n + 1) / 2), 4);
  int vals_cap = (int)round_up(2 * (int64_t)n + 2, 4);
  constexpr size_t kBudget = 200 * 1024;
  if ((size_t)(vals_cap + scratch_words) * 4 > kBudget) vals_cap = 0;
  const size_t per_warp = (size_t)(vals_cap + scratch_words) * 4;
  const int warps =
      (int)std::max<size_t>(1, std::min<size_t>(kSampleWarps,
                                                kBudget / per_warp));
  const size_t smem = (size_t)warps * per_warp;
  set_dyn_smem((const void*)k_mut_sample, smem);
  k_mut_sample<<<(P + warps - 1) / warps, warps * 32, smem, s>>>(
      v, vals_cap, scratch_words);
  const size_t scratch =
      std::max<size_t>(round_up((n + 31) / 32 * 4, 16), 2 * (size_t)v.np);
  set_dyn_smem((const void*)k_mut_fix, scratch);
  k_mut_fix<<<1, 32, scratch, s>>>(v);
  const size_t sd = (size_t)8 * v.np;
  set_dyn_smem((const void*)k_mut_swap, sd);
  k_mut_swap<<<P, 128, sd, s>>>(v);
  return cudaGetLastError();
}

cudaError_t launch_mutation(const SwarmView& v, cudaStream_t s) {
  cudaError_t e = launch_mutation_walk(v, s);
  if (!e) e = launch_mutation_pre(v, s);
  if (!e) e = launch_mutation_post(v, s);
  return e;
}

}  // namespace dpso
