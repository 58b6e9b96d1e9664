// Random mutation with elitism and canonical-form dedupe (solver.py:222-258).
//
// Pipeline (all kernels no-op unless ctl->mutating):
//   k_mut_hash    per particle: canonical rotation/direction (graph.py:106-115)
//                 and a 64-bit order-dependent hash of the canonical sequence
//   k_mut_rank    rank in (fitness, slot) order by counting over a 2-D grid
//                 (solver.py:223-224)
//   k_mut_dedupe  earliest-ranked particle with the same hash (candidate
//                 duplicate source)
//   k_mut_verify  one warp per candidate: exact canonical-form comparison
//                 (a hash collision falls back to an exact search)
//   k_mut_lists   survivors / dropped in rank order, keep = first ceil(S/3)
//                 survivors, events = non-kept slots in slot order
//   k_mut_copy    dropped #r copies body+fitness (and edge costs) of
//                 survivors[r % S]
//   k_mut_gen/k_mut_walk/k_mut_sample/k_mut_fix: the mutation stream (see
//                 the section comment below)
//   k_mut_swap    k disjoint swaps, fitness in reference order, pbest
//                 (solver.py:241-258)
#include <cstdio>
#include <algorithm>

#include "dpso_internal.cuh"
#include "tma.cuh"
#include "philox.cuh"

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
    v.rank[p] = 0;             // k_mut_rank accumulates per column chunk
    v.flag[p] = 0x7fffffff;    // k_mut_dedupe: lowest candidate rank
  }
}

constexpr int kChunk = 1024;  // j values per CTA of the O(P^2) passes

// fitness as an order-preserving u64 (fp64 bits, sign folded; -0.0 reads as
// +0.0, since sorted() compares them equal): (key, slot) order is the
// reference's (fitness, slot) order (solver.py:223-224)
__device__ __forceinline__ uint64_t fit_key(double f) {
  if (f == 0.0) f = 0.0;
  const uint64_t b = (uint64_t)__double_as_longlong(f);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// rank in (fitness, slot) order by counting, P x P comparisons spread over
// a 2-D grid (x: 256 particles i per CTA, y: a chunk of kChunk particles j);
// each CTA adds its chunk's count (rank was zeroed by k_mut_hash)
__global__ void __launch_bounds__(256) k_mut_rank(SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  __shared__ uint64_t s_k[kChunk];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int base = blockIdx.y * kChunk;
  const int m = min(kChunk, v.P - base);
  for (int u = threadIdx.x; u < m; u += blockDim.x)
    s_k[u] = fit_key(v.fit[base + u]);
  __syncthreads();
  if (i >= v.P) return;
  const uint64_t ki = fit_key(v.fit[i]);
  int cnt = 0;
  for (int u = 0; u < m; ++u) {
    const uint64_t kj = s_k[u];
    cnt += (kj < ki) || (kj == ki && base + u < i);
  }
  if (cnt) atomicAdd(&v.rank[i], cnt);
}

// The lowest rank among earlier-ranked particles with the same canonical
// hash, over a 2-D grid as k_mut_rank (atomicMin into flag, which
// k_mut_hash set to "none"); the first chunk also records order[rank].
__global__ void __launch_bounds__(256) k_mut_dedupe(SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  __shared__ unsigned long long s_h[kChunk];
  __shared__ int s_r[kChunk];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int base = blockIdx.y * kChunk;
  const int m = min(kChunk, v.P - base);
  for (int u = threadIdx.x; u < m; u += blockDim.x) {
    s_h[u] = v.hash[base + u];
    s_r[u] = v.rank[base + u];
  }
  __syncthreads();
  if (i >= v.P) return;
  const uint64_t hi = v.hash[i];
  const int ri = v.rank[i];
  if (blockIdx.y == 0) v.order[ri] = i;
  int crank = 0x7fffffff;
  for (int u = 0; u < m; ++u) {
    const int r = s_r[u];
    if (s_h[u] == hi && r < ri && r < crank) crank = r;
  }
  if (crank != 0x7fffffff) atomicMin(&v.flag[i], crank);
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
  const int crank = v.flag[i];
  if (crank == 0x7fffffff) {  // no earlier particle with the same hash
    if ((threadIdx.x & 31) == 0) v.flag[i] = 0;
    return;
  }
  const int cand = v.order[crank];
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

// Swarms of P <= 1024: rank, dedupe, verify and lists in one CTA (one
// launch instead of four).  Rank: a bitonic sort of (fitness key, slot);
// dedupe: a bitonic sort of (hash, rank), each particle's candidate the
// first (lowest-ranked) member of its hash group - the values k_mut_rank /
// k_mut_dedupe compute by counting; then k_mut_verify's exact check by
// warps and k_mut_lists' scans.
template <typename K>
__device__ __forceinline__ void block_bitonic_1024(K* key, int* val) {
  const int tid = threadIdx.x;
  for (int k = 2; k <= 1024; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int ixj = tid ^ j;
      if (ixj > tid) {
        const K a = key[tid], b = key[ixj];
        const int va = val[tid], vb = val[ixj];
        const bool gt = a > b || (a == b && va > vb);
        if (gt == ((tid & k) == 0)) {
          key[tid] = b;
          key[ixj] = a;
          val[tid] = vb;
          val[ixj] = va;
        }
      }
      __syncthreads();
    }
}

__global__ void __launch_bounds__(1024) k_mut_small(SwarmView v,
                                                   const int32_t* canon) {
  if (!v.ctl->mutating || v.ctl->done) return;
  __shared__ unsigned long long s_k[1024];
  __shared__ int s_v[1024];
  __shared__ int s_w[32];
  const int P = v.P, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- rank: (fitness, slot) order (solver.py:223-224)
  s_k[tid] = tid < P ? fit_key(v.fit[tid]) : ~0ull;
  s_v[tid] = tid < P ? tid : 0x7fffffff;
  __syncthreads();
  block_bitonic_1024(s_k, s_v);
  if (tid < P) {
    v.rank[s_v[tid]] = tid;
    v.order[tid] = s_v[tid];
  }
  __syncthreads();
  // ---- dedupe candidates: the lowest-ranked particle of each hash group
  s_k[tid] = tid < P ? v.hash[tid] : ~0ull;
  s_v[tid] = tid < P ? v.rank[tid] : 0x7fffffff;
  __syncthreads();
  block_bitonic_1024(s_k, s_v);
  if (tid < P) {
    int q0 = tid;
    while (q0 > 0 && s_k[q0 - 1] == s_k[tid]) --q0;
    const int r = s_v[tid], r0 = s_v[q0];
    v.flag[v.order[r]] = r0 < r ? r0 : 0x7fffffff;
  }
  __syncthreads();
  // ---- verify (k_mut_verify): one warp per particle
  for (int i = warp; i < P; i += 32) {
    const int crank = v.flag[i];
    if (crank == 0x7fffffff) {
      if (lane == 0) v.flag[i] = 0;
      continue;
    }
    const int cand = v.order[crank];
    int dropped = warp_canon_equal(v, canon, i, cand);
    if (!dropped) {
      if (lane == 0) v.ctl->collision = 1;
      const uint64_t hi = v.hash[i];
      const int ri = v.rank[i];
      for (int j = 0; j < P && !dropped; ++j)
        if (j != cand && v.hash[j] == hi && v.rank[j] < ri)
          dropped = warp_canon_equal(v, canon, i, j);
    }
    if (lane == 0) v.flag[i] = dropped;
  }
  __syncthreads();
  // ---- lists (k_mut_lists, one 1024-block: P <= 1024)
  {
    const int r = tid;
    const int i = r < P ? v.order[r] : 0;
    const int sv = (r < P) ? !v.flag[i] : 0;
    int tot;
    const int ex = block_scan_excl<1024>(sv, s_w, &tot);
    if (r < P) {
      if (sv) {
        v.sidx[i] = ex;
        v.surv_list[ex] = i;
      } else {
        v.sidx[i] = r - ex;  // dropped index in rank order
      }
    }
    const int S = tot;
    const int nkeep = (S + 2) / 3;  // ceil(S / 3)
    __syncthreads();
    int kp = 0;
    if (tid < P) {
      kp = !v.flag[tid] && v.sidx[tid] < nkeep;
      v.keep[tid] = kp;
    }
    const int e = (tid < P) && !kp;
    int tot2;
    const int ex2 = block_scan_excl<1024>(e, s_w, &tot2);
    if (e) v.ev_slot[ex2] = tid;
    if (tid == 0) {
      v.ctl->n_surv = S;
      v.ctl->n_drop = P - S;
      v.ctl->n_events = tot2;
    }
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
  // and its edge costs: k_mut_swap re-gathers only the edges it touches
  const double* da = v.dcache + (size_t)src * v.np;
  double* db = v.dcache + (size_t)p * v.np;
  for (int i = threadIdx.x; i < v.n; i += blockDim.x) db[i] = da[i];
  if (threadIdx.x == 0) v.fit[p] = v.fit[src];
}

// ---- the mutation stream ----------------------------------------------------
//
// The mutation stream is ONE numpy PCG64 stream consumed in slot order, so
// where event e's draws start depends on every earlier event's k.  Steps:
//   k_mut_gen     (grid-wide) writes the span of the stream this call can
//                 use into an L2-resident buffer (fresh u32 index f ->
//                 mstream[f]); every thread jumps to its own chunk.
//   k_mut_walk    one CTA chains all P potential events exactly: warp 0
//                 chains the k-draws of a block of events speculatively
//                 through a shared-memory ring of stream segments fed by
//                 cp.async.bulk, all warps then test the block's draws for
//                 Lemire redraws, and only an event that holds one is
//                 consumed draw by draw.  It only needs the stream, so the
//                 walk for the NEXT call runs on a forked stream and
//                 overlaps the following generations (double-buffered by
//                 call parity).
//   k_mut_sample  one warp per event reads its draws from the buffer and
//                 runs numpy's Floyd sampler + shuffle; it re-checks its
//                 consumption against the walk's record (safety net).
//   k_mut_fix     the persistent stream update; the exact sequential
//                 sampler for the whole call only if the walk overflowed.

// Buffers of one mutation call (parity 0/1).
struct MutBufs {
  int32_t* ev_k;
  uint64_t* ev_cursor;
  uint64_t* ev_end;
  uint32_t* mstream;
  uint16_t* skip;  // per stream word: the skip of an event whose k-draw it is
  PcgState* start;
};

__device__ __forceinline__ MutBufs mut_bufs(const SwarmView& v, int par) {
  uint16_t* skips = reinterpret_cast<uint16_t*>(v.mstream + 2 * v.mstream_cap);
  return {v.ev_k + (size_t)par * v.P, v.ev_cursor + (size_t)par * v.P,
          v.ev_end + (size_t)par * v.P,
          v.mstream + (size_t)par * v.mstream_cap,
          skips + (size_t)par * v.mstream_cap, v.mut_start + par};
}

constexpr int kSeg = 4096;   // u32 per ring segment (16 KiB)
constexpr int kNSeg = 8;     // ring slots (128 KiB)

// number of Floyd + shuffle draws of choice(n, 2k, replace=False) when no
// Lemire redraw happens (numpy _generator.pyx: Floyd skips j == 0; n > 10000
// with 2k > n // 50 uses the tail shuffle instead)
__host__ __device__ __forceinline__ int sample_draws(int n, int k) {
  const int size = 2 * k;
  const int jstart = n - size > 1 ? n - size : 1;
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

constexpr int kGenPer = 64;  // outputs per k_mut_gen thread

// The event an accepted k-draw u opens: k = integers(1, k_hi + 1) clipped
// to n // 2 (solver.py:232-236), then its D Floyd/shuffle draws when none is
// redrawn.  skip = 1 + D, or 0 when the k-draw itself is rejected (Lemire).
struct KDraw {
  int n, n2;
  uint32_t mk, thr;  // k_hi and Lemire's rejection threshold for it
  __host__ __device__ static KDraw make(int n) {
    KDraw r;
    r.n = n;
    r.n2 = n / 2;
    r.mk = (uint32_t)(n / 4 > 2 ? n / 4 : 2);
    r.thr = (0u - r.mk) % r.mk;
    return r;
  }
  __device__ __forceinline__ int k(uint32_t u) const {
    return min((int)__umulhi(u, mk) + 1, n2);
  }
  __device__ __forceinline__ uint32_t skip(uint32_t u) const {
    if (u * mk < thr) return 0u;
    const int kk = k(u);
    return 1u + (uint32_t)(kk >= 1 ? sample_draws(n, kk) : 0);
  }
  // skips fit u16 (else the walker computes them itself)
  __host__ __device__ static bool fits16(int n) {
    const int kmax = (n / 4 > 2 ? n / 4 : 2) < n / 2 ? (n / 4 > 2 ? n / 4 : 2)
                                                      : n / 2;
    return 1 + sample_draws(n, kmax) <= 0xFFFF;
  }
};

// Prepares the NEXT mutation call: writes its stream span into the buffer
// of parity mut_cur ^ 1.
__global__ void __launch_bounds__(256) k_mut_gen(SwarmView v) {
  if (!v.ctl->mut_pending || v.ctl->done) return;
  const MutBufs b = mut_bufs(v, v.ctl->mut_cur ^ 1);
  const PcgState g = v.streams[1];
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c == 0) *b.start = g;
  const int64_t outs = v.mstream_cap / 2;
  const int64_t o0 = c * kGenPer;
  if (o0 >= outs) return;
  const u128 inc = {g.inc_hi, g.inc_lo};
  u128 st = pcg_advance({g.state_hi, g.state_lo}, inc, (uint64_t)o0 + 1);
  const u128 M = pcg_mult();
  uint2* out = reinterpret_cast<uint2*>(b.mstream);
  ushort2* sk = reinterpret_cast<ushort2*>(b.skip);
  const KDraw kd = KDraw::make(v.n);
  const bool skips = KDraw::fits16(v.n);
  for (int r = 0; r < kGenPer && o0 + r < outs; ++r) {
    const uint64_t o = pcg_output(st);
    const uint32_t lo = (uint32_t)o, hi = (uint32_t)(o >> 32);
    out[o0 + r] = make_uint2(lo, hi);
    if (skips)
      sk[o0 + r] = make_ushort2((uint16_t)kd.skip(lo), (uint16_t)kd.skip(hi));
    st = add128(mul128(st, M), inc);
  }
}

// The stream as seen from a thread: u32 at position q (counting next32()
// calls from the call's start, so q = 0 may be numpy's buffered half).
struct StreamView {
  const uint32_t* buf;
  int64_t h, cap;
  uint32_t ub;
  __device__ __forceinline__ uint32_t at(int64_t q) const {
    return q < h ? ub : buf[q - h];
  }
};

// Exact chain of all P potential events of the NEXT call (parity
// mut_cur ^ 1) from its start; one CTA of kWalkWarps warps.
//
// The stream is staged in a kNSeg-slot shared-memory ring of kSeg-word
// segments by cp.async.bulk (warp 0 issues, mbarrier completion, segments
// issued and waited on strictly in order, free slots refilled ahead of the
// walk).  The walk proceeds in speculative blocks over a window of W stream
// positions starting at the block start qs:
//   1. one thread chains the events starting in the window: a k-draw
//      (Lemire; its redraws are exact since they are serial), then a skip
//      of the D(k) Floyd/shuffle draws assuming none of them is redrawn;
//   2. all warps test every Floyd/shuffle draw of the block against its
//      Lemire bound (one warp per event);
//   3. the events before the first one holding a redraw (about 1e-7 per
//      draw at n = 1000) are committed; that event is consumed draw by draw
//      by warp 0 and the next block starts after it.
// So the recorded (k, cursor, end) of every event is exact; k_mut_sample
// re-checks its event against the record as a safety net.
constexpr int kWalkWarps = 16;
constexpr int kWalkThreads = kWalkWarps * 32;
constexpr int kBlockEv = 512;
constexpr int kWalkWin = 4 * kSeg;  // window cap (stream positions)

struct WalkSmem {
  uint64_t bars[kNSeg];
  int64_t cur[kBlockEv];      // first Floyd draw of event j (after its k)
  int32_t k[kBlockEv];        // its k
  int32_t off[kBlockEv + 1];  // prefix sums of the draw counts
  int64_t q;                  // next block start
  int32_t e;                  // next event
  int32_t nb, first_bad, stop;
};

__device__ __forceinline__ StreamView stream_view(const SwarmView& v,
                                                  const MutBufs& b) {
  const PcgState& g = *b.start;
  return {b.mstream, (int64_t)g.has_uint32, v.mstream_cap,
          (uint32_t)g.uinteger};
}

// walk window for n.  A block touches the window plus its longest event
// (+1 segment when unaligned); when 2W + Dmax fits in kNSeg - 2 segments,
// the next block's segments were already issued one block earlier, so the
// copies overlap the walk.  0 = an event alone does not fit the ring.
__host__ __device__ __forceinline__ int walk_window(int n) {
  const int k_hi = n / 4 > 2 ? n / 4 : 2;
  const int kmax = k_hi < n / 2 ? k_hi : n / 2;
  const int room = (kNSeg - 2) * kSeg - (1 + sample_draws(n, kmax));
  int w = room / 2 >= 1024 ? room / 2 : room;
  w = w < kWalkWin ? w : kWalkWin;
  return w >= 256 ? w : 0;
}

__global__ void __launch_bounds__(kWalkThreads) k_mut_walk(SwarmView v) {
  if (v.ctl->done || !v.ctl->mut_pending) return;
  extern __shared__ __align__(128) uint32_t ring[];
  uint16_t* sring = reinterpret_cast<uint16_t*>(ring + kNSeg * kSeg);
  __shared__ WalkSmem s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = v.ctl->mut_cur ^ 1;
  const MutBufs b = mut_bufs(v, par);
  const StreamView sv = stream_view(v, b);
  const int n = v.n, P = v.P;
  const int k_hi = max(2, n / 4);
  const int64_t nseg_total = (sv.cap + kSeg - 1) / kSeg;
  const int W = walk_window(n);
  const KDraw kd = KDraw::make(n);
  const bool skips = KDraw::fits16(n);
  const int Dmax = sample_draws(n, min(k_hi, n / 2));
  // segment sg sits in slot sg % kNSeg, so stream word f is ring[f & kMask]
  constexpr uint32_t kMask = kNSeg * kSeg - 1;
  static_assert((kNSeg & (kNSeg - 1)) == 0, "ring slots: a power of two");
  auto at = [&](int64_t q) -> uint32_t {
    return q < sv.h ? sv.ub : ring[(uint32_t)(q - sv.h) & kMask];
  };
  auto seg_of = [&](int64_t q) -> int64_t {
    return q - sv.h < 0 ? 0 : (q - sv.h) / kSeg;
  };
  // ring state, meaningful in warp 0 only (warp-uniform there)
  int64_t next_issue = 0, ready = -1;
  auto wait_upto = [&](int64_t sg_hi) {
    for (int64_t sg = ready + 1; sg <= sg_hi && sg < nseg_total; ++sg)
      mbar_wait(&s.bars[sg % kNSeg], (uint32_t)((sg / kNSeg) & 1));
    if (sg_hi > ready) ready = sg_hi;
  };
  // refill every slot below segment slo (no thread reads those any more)
  auto prefetch = [&](int64_t slo) {
    bool fenced = false;
    while (next_issue < slo + kNSeg && next_issue < nseg_total) {
      if (next_issue - kNSeg > ready) wait_upto(next_issue - kNSeg);
      if (lane == 0) {
        const int slot = (int)(next_issue % kNSeg);
        if (!fenced) fence_proxy_async();  // generic reads before the refill
        fenced = true;
        mbar_expect_tx(&s.bars[slot], kSeg * (skips ? 6 : 4));
        bulk_g2s(ring + (size_t)slot * kSeg, sv.buf + next_issue * kSeg,
                 kSeg * 4, &s.bars[slot]);
        if (skips)
          bulk_g2s(sring + (size_t)slot * kSeg, b.skip + next_issue * kSeg,
                   kSeg * 2, &s.bars[slot]);
      }
      ++next_issue;
    }
  };
  // positions [qlo, qhi] resident (qlo = the oldest position still needed)
  auto ensure = [&](int64_t qlo, int64_t qhi) -> bool {
    const int64_t slo = seg_of(qlo), shi = seg_of(qhi);
    if (shi >= nseg_total || shi - slo >= kNSeg) return false;
    if (shi >= next_issue) prefetch(slo);
    if (shi > ready) wait_upto(shi);
    return true;
  };

#ifdef DPSO_WALK_PROF
  long long t_ens = 0, t_chain = 0, t_check = 0, t_commit = 0, t0 = 0;
  int nblocks = 0;
#define WPROF(acc)                   \
  if (tid == 0) {                    \
    const long long t1 = clock64();  \
    acc += t1 - t0;                  \
    t0 = t1;                         \
  }
#else
#define WPROF(acc)
#endif
  if (tid == 0) {
    for (int i = 0; i < kNSeg; ++i) mbar_init(&s.bars[i], 1);
    fence_barrier_init();
    s.e = 0;
    s.q = 0;
    s.stop = W == 0;
  }
  __syncthreads();
  if (warp == 0) prefetch(0);

#ifdef DPSO_WALK_PROF
  if (tid == 0) t0 = clock64();
#endif
  while (!s.stop) {
#ifdef DPSO_WALK_PROF
    if (tid == 0) ++nblocks;
#endif
    const int64_t qs = s.q;
    const int e0 = s.e;
    // window [qs, qs + wlen) and every draw of an event starting in it
    const int64_t lim = sv.h + sv.cap;  // first position past the buffer
    const int wlen = (int)(lim - qs < W ? lim - qs : W);
    if (warp == 0) {
      prefetch(seg_of(qs));  // every slot below the block refills ahead
      if (!ensure(qs, qs + wlen + Dmax < lim ? qs + wlen + Dmax : lim - 1))
        if (lane == 0) s.stop = 1;
    }
    __syncthreads();
    WPROF(t_ens)
    if (s.stop) break;
    // ---- 1. the chain through the window (one thread) ----
    // per event: one shared load of the precomputed skip and an add
    if (tid == 0) {
      int nb = 0, tot = 0;
      const int nev = min(kBlockEv, P - e0);
      int64_t p = qs;
      const int64_t wend = qs + wlen;
      if (p < sv.h && p < wend && nb < nev) {  // numpy's buffered half
        const uint32_t sk = kd.skip(sv.ub);
        if (sk != 0) {
          s.cur[0] = p + 1;
          s.off[0] = 0;
          tot = (int)sk - 1;
          nb = 1;
        }
        p += sk != 0 ? sk : 1;
      }
      if (p >= sv.h) {
        // stream word index f = p - h (< cap < 2^31); branch-free body so
        // the loop-carried path is load -> select -> add
        uint32_t f = (uint32_t)(p - sv.h);
        const uint32_t fend = (uint32_t)(wend - sv.h);
        if (skips) {
          // the stores are unconditional (a rejected k-draw's slot is
          // overwritten by the next event): no branch on the chain
          int64_t* cur = s.cur;
          int32_t* off = s.off;
          const int64_t h1 = sv.h + 1;
          while (f < fend && nb < nev) {
            const uint32_t sk = sring[f & kMask];
            const int acc = sk != 0u;
            cur[nb] = h1 + f;
            off[nb] = tot;
            tot += acc ? (int)sk - 1 : 0;
            nb += acc;
            f += acc ? sk : 1u;
          }
        } else {
          while (f < fend && nb < nev) {
            const uint32_t sk = kd.skip(ring[f & kMask]);
            if (sk != 0) {
              s.cur[nb] = sv.h + f + 1;
              s.off[nb] = tot;
            }
            tot += sk != 0 ? (int)sk - 1 : 0;
            nb += sk != 0;
            f += sk != 0 ? sk : 1u;
          }
        }
        p = sv.h + f;
      }
      // only the last event can run past the buffer: drop it and stop
      int stop = 0;
      if (nb > 0 && p > lim) {
        --nb;
        tot = s.off[nb];
        stop = 1;
      }
      s.off[nb] = tot;
      s.nb = nb;
      s.first_bad = 0x7fffffff;
      s.q = p;  // provisional: the block end
      s.stop = stop || (nb == 0 && p >= lim);
    }
    __syncthreads();
    WPROF(t_chain)
    const int nb = s.nb;
    // ---- 2. every draw of the block against its Lemire bound ----
    // one warp per event; the bounds are affine in the draw index
    // (sample_bound): Floyd m = jstart + 1 + d, shuffle m = size - t,
    // tail shuffle m = n - d.  The scan tests only Lemire's necessary
    // condition leftover < m (two instructions per draw); an event where
    // it fires (~m / 2^32 per draw) is re-tested exactly.
    for (int j = warp; j < nb; j += kWalkWarps) {
      const int64_t cur = s.cur[j];
      const int k = kd.k(at(cur - 1));
      if (lane == 0) s.k[j] = k;
      if (k < 1) continue;
      const uint32_t fc = (uint32_t)(cur - sv.h);
      const int size = 2 * k;
      const int jstart = max(n - size, 1);
      const int F = n - jstart;
      const bool tail = n > 10000 && size > n / 50;
      uint32_t cand = 0;
      if (tail) {
        for (int t = lane; t < F; t += 32) {
          const uint32_t m = (uint32_t)(n - t);
          cand |= (ring[(fc + t) & kMask] * m) < m;
        }
      } else {
#pragma unroll 4
        for (int t = lane; t < F; t += 32) {
          const uint32_t m = (uint32_t)(jstart + 1 + t);
          cand |= (ring[(fc + t) & kMask] * m) < m;
        }
        const uint32_t fs = fc + (uint32_t)F;
#pragma unroll 4
        for (int t = lane; t < size - 1; t += 32) {
          const uint32_t m = (uint32_t)(size - t);
          cand |= (ring[(fs + t) & kMask] * m) < m;
        }
      }
      if (__any_sync(0xffffffffu, cand)) {  // rare: the exact test
        bool bad = false;
        const int D = s.off[j + 1] - s.off[j];
        for (int d = lane; d < D; d += 32)
          bad |= lemire_rejects(ring[(fc + d) & kMask], sample_bound(n, k, d));
        if (__any_sync(0xffffffffu, bad) && lane == 0)
          atomicMin(&s.first_bad, j);
      }
    }
    __syncthreads();
    WPROF(t_check)
    // ---- 3. commit; an event holding a redraw is consumed exactly ----
    const int fb = s.first_bad;
    const int ncommit = min(fb, nb);
    for (int t = tid; t < ncommit; t += kWalkThreads) {
      const int64_t cur = s.cur[t];
      b.ev_k[e0 + t] = s.k[t];
      b.ev_cursor[e0 + t] = (uint64_t)cur;
      b.ev_end[e0 + t] = (uint64_t)(cur + (s.off[t + 1] - s.off[t]));
    }
    if (fb < nb && warp == 0) {
      const int64_t cur = s.cur[fb];
      const int k = s.k[fb];
      const int D = s.off[fb + 1] - s.off[fb];
      int64_t p = cur;
      bool over = false;
      for (int d = 0; d < D && !over; ++d) {
        const uint32_t rng = sample_bound(n, k, d);
        if (rng == 0) continue;
        for (;;) {
          if (!ensure(cur, p)) {
            over = true;
            break;
          }
          if (!lemire_rejects(at(p), rng)) break;
          ++p;
        }
        ++p;
      }
      if (lane == 0) {
        b.ev_k[e0 + fb] = k;
        b.ev_cursor[e0 + fb] = (uint64_t)cur;
        b.ev_end[e0 + fb] = (uint64_t)p;
        s.q = p;
        s.e = e0 + fb + 1;
        s.stop = over;
      }
    } else if (fb >= nb && tid == 0) {
      s.e = e0 + nb;
    }
    __syncthreads();
    WPROF(t_commit)
    if (s.e >= P) break;
  }
#ifdef DPSO_WALK_PROF
  if (tid == 0)
    printf("walk: blocks %d events %d ensure %lld chain %lld check %lld "
           "commit %lld cycles\n", nblocks, s.e, t_ens, t_chain, t_check,
           t_commit);
#endif
  if (warp == 0) {
    // drain outstanding copies before the CTA exits
    wait_upto(next_issue - 1);
    if (lane == 0) {
      if (s.stop) v.ctl->mut_overflow |= 1 << par;
      v.ctl->mut_pending = 0;
    }
  }
}

// Numpy's choice(n, 2k, replace=False) read from a stream, one thread:
// writes the 2k sampled positions to idx; returns the u32 consumed (or -1
// if the buffer ran out).
template <typename Src>
__device__ int64_t sample_event_seq(Src& c, int n, int k, uint16_t* idx,
                                    uint32_t* bits, uint16_t* arr) {
  const int size = 2 * k;
  if (n > 10000 && size > n / 50) {
    for (int i = 0; i < n; ++i) arr[i] = (uint16_t)i;
    const int first = max(n - size, 1);
    for (int i = n - 1; i >= first; --i) {
      uint32_t j = c.bounded((uint32_t)i);
      uint16_t t = arr[i];
      arr[i] = arr[j];
      arr[j] = t;
    }
    for (int t = 0; t < size; ++t) idx[t] = arr[n - size + t];
  } else {
    for (int i = 0; i < (n + 31) / 32; ++i) bits[i] = 0;
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

// Lemire bounded draws with a u32 counter over a source of u32.
template <typename Next>
struct CountingBounded {
  Next next;
  int64_t q = 0;
  __device__ uint32_t bounded(uint32_t rng) {
    if (rng == 0) return 0;
    const uint32_t rng_excl = rng + 1u;
    ++q;
    uint64_t m = (uint64_t)next() * rng_excl;
    uint32_t leftover = (uint32_t)m;
    if (leftover < rng_excl) {
      const uint32_t threshold = (0xFFFFFFFFu - rng) % rng_excl;
      while (leftover < threshold) {
        ++q;
        m = (uint64_t)next() * rng_excl;
        leftover = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

struct BufNext {  // next32() over the generated stream buffer
  StreamView sv;
  int64_t pos;
  __device__ uint32_t operator()() {
    const int64_t p = pos++;
    // past the buffer: an always-accepted word, so the sampler terminates
    // (the caller flags the overflow and the exact fallback redoes the call)
    return p - sv.h < sv.cap ? sv.at(p) : 0xFFFFFFFFu;
  }
};

struct PcgNext {  // next32() regenerated from the stream state
  Pcg r;
  __device__ uint32_t operator()() { return r.next32(); }
};

// One warp per event.  Shared memory per warp: draw values (u32, D) and the
// n-bit Floyd bitmap (or arange(n) for the tail shuffle).
constexpr int kSampleWarps = 4;

// numpy's choice(n, 2k, replace=False) - Floyd's sampler then the
// _shuffle_int of the 2k values - from the event's bounded draws vals,
// data-parallel over one warp (the reference's loops are sequential):
//  Floyd: step t (value j_t = n - 2k + t) draws v_t; it adds j_t instead
//    iff v_t is already in the set: iff an earlier step drew v_t (the first
//    step to draw each value: an atomicMin per value) or v_t = j_s of an
//    earlier step s that itself collided (s = v_t - (n - 2k) < t):
//    col(t) = dup(t) or col(s), iterated to the fixpoint (links strictly
//    decrease).
//  Shuffle: step i = 2k-1 .. 1 swaps positions i and w_i <= i, and
//    position i is final after it.  Its value is whatever position w_i held
//    just before step i: the value written there by the most recent earlier
//    step (the smallest i' > i with w_i' = w_i), which is what position i'
//    held just before step i' (the smallest writer of i' above i'), and so
//    on back to an original value.  Each position's writers form a short
//    list (atomicExch heads), searched per query.
// first: max(n, 2k) words; nxt, sidx: 2k u16; col: 2k bytes.
__device__ void floyd_shuffle_warp(const uint32_t* vals, int n, int size,
                                   uint32_t* first, uint16_t* nxt,
                                   uint8_t* col, uint16_t* sidx,
                                   uint16_t* out, int lane) {
  const int nmz = n - size;  // j_t = nmz + t
  const int zero = nmz == 0 ? 1 : 0;  // j_0 == 0 takes no draw
  const int F = size - zero;         // Floyd draws
  auto vt = [&](int t) -> uint32_t {
    return (zero && t == 0) ? 0u : vals[t - zero];
  };
  for (int v = lane; v < n; v += 32) first[v] = 0xFFFFFFFFu;
  __syncwarp();
  for (int t = lane; t < size; t += 32) atomicMin(&first[vt(t)], (uint32_t)t);
  __syncwarp();
  for (int t = lane; t < size; t += 32) col[t] = first[vt(t)] < (uint32_t)t;
  __syncwarp();
  for (;;) {
    int changed = 0;
    for (int t = lane; t < size; t += 32) {
      if (col[t]) continue;
      const int v = (int)vt(t);
      if (v >= nmz && v - nmz < t && col[v - nmz]) {
        col[t] = 1;
        changed = 1;
      }
    }
    __syncwarp();
    if (!__any_sync(0xffffffffu, changed)) break;
  }
  for (int t = lane; t < size; t += 32)
    sidx[t] = (uint16_t)(col[t] ? (uint32_t)(nmz + t) : vt(t));
  // the shuffle: step i draws w_i = vals[F + size - 1 - i]; writer lists of
  // each position (heads in first[], links in nxt[])
  __syncwarp();
  for (int x = lane; x < size; x += 32) first[x] = 0xFFFFu;
  __syncwarp();
  for (int i = 1 + lane; i < size; i += 32)
    nxt[i] = (uint16_t)atomicExch(&first[vals[F + size - 1 - i]], (uint32_t)i);
  __syncwarp();
  // the smallest writer of position x above y (0xFFFF: none)
  auto above = [&](uint32_t x, uint32_t y) -> uint32_t {
    uint32_t best = 0xFFFFu;
    for (uint32_t w = first[x]; w != 0xFFFFu; w = nxt[w])
      if (w > y && w < best) best = w;
    return best;
  };
  for (int i = lane; i < size; i += 32) {
    uint32_t x = i == 0 ? 0u : vals[F + size - 1 - i];
    uint32_t w = above(x, (uint32_t)i);
    while (w != 0xFFFFu) {
      x = w;
      w = above(x, x);
    }
    out[i] = sidx[x];
  }
}

__global__ void __launch_bounds__(kSampleWarps * 32) k_mut_sample(
    SwarmView v, int vals_cap, int scratch_words, int par_m) {
  if (!v.ctl->mutating || v.ctl->done) return;
  const MutBufs b = mut_bufs(v, v.ctl->mut_cur);
  extern __shared__ __align__(16) uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * (blockDim.x >> 5) + warp;
  if (e >= v.ctl->n_events) return;
  const int n = v.n, k = b.ev_k[e];
  if (k < 1) return;
  // per warp: vals[vals_cap] | bits/arr[scratch_words] | sidx[idx_words]
  const int idx_words = (n + 1) / 2;
  const int par_words = par_m ? n + (3 * n + 3) / 4 + 1 : 0;
  uint32_t* vals =
      sm + (size_t)warp * (vals_cap + scratch_words + idx_words + par_words);
  uint32_t* bits = vals + vals_cap;
  uint16_t* arr = (uint16_t*)bits;
  uint16_t* idx = v.ev_idx + (size_t)e * v.np;
  const int size = 2 * k;
  const bool tail = (n > 10000) && size > n / 50;
  const StreamView sv = stream_view(v, b);
  const int64_t cur = (int64_t)b.ev_cursor[e];
  const int D = sample_draws(n, k);
  int rej = 0;
  if (!tail && D <= vals_cap && cur - sv.h + D <= sv.cap) {
    for (int d = lane; d < D; d += 32) {
      const uint32_t rng = sample_bound(n, k, d);
      const uint32_t u = sv.buf[cur - sv.h + d];
      rej |= lemire_rejects(u, rng);
      vals[d] = (uint32_t)(((uint64_t)u * (rng + 1u)) >> 32);
    }
    rej = __any_sync(0xffffffffu, rej);
    if (!rej && par_m) {
      // data-parallel Floyd + shuffle (floyd_shuffle_warp)
      __syncwarp();
      uint16_t* sidx = (uint16_t*)(bits + scratch_words);
      uint32_t* first = bits + scratch_words + idx_words;  // n words
      uint16_t* nxt = reinterpret_cast<uint16_t*>(first + n);
      uint8_t* col = reinterpret_cast<uint8_t*>(nxt + n);
      floyd_shuffle_warp(vals, n, size, first, nxt, col, sidx, idx, lane);
      return;
    }
    if (!rej) {
      __syncwarp();
      for (int i = lane; i < (n + 31) / 32; i += 32) bits[i] = 0;
      __syncwarp();
      // Floyd + shuffle on a shared-memory copy of idx (the serial steps are
      // dependent loads; global memory would put an L2 round trip in each)
      uint16_t* sidx = (uint16_t*)(bits + scratch_words);
      if (lane == 0) {
        // Floyd: j = n - 2k .. n-1 (j == 0 takes no draw and yields 0)
        int d = 0;
        for (int t = 0; t < size; ++t) {
          const uint32_t j = (uint32_t)(n - size + t);
          uint32_t val = j == 0 ? 0u : vals[d++];
          if (bits[val >> 5] & (1u << (val & 31))) val = j;
          bits[val >> 5] |= 1u << (val & 31);
          sidx[t] = (uint16_t)val;
        }
        // shuffle (numpy _shuffle_int): i = size-1 .. 1
        for (int i = size - 1; i >= 1; --i) {
          const uint32_t j = vals[d++];
          const uint16_t t = sidx[i];
          sidx[i] = sidx[j];
          sidx[j] = t;
        }
      }
      __syncwarp();
      for (int t = lane; t < size; t += 32) idx[t] = sidx[t];
      return;
    }
  }
  // sequential exact sampler: the event holds a redraw, uses the tail
  // shuffle, or is too large for the draw buffer
  if (lane == 0) {
    CountingBounded<BufNext> c{BufNext{sv, cur}};
    const int64_t used = sample_event_seq(c, n, k, idx, bits, arr);
    if (cur - sv.h + used > sv.cap)
      atomicOr(&v.ctl->mut_overflow, 1 << v.ctl->mut_cur);
    // the walk resolved redraws exactly; a mismatch would be a walk bug:
    // fall back to the exact sequential path
    if (cur + used != (int64_t)b.ev_end[e])
      atomicOr(&v.ctl->mut_overflow, 1 << v.ctl->mut_cur);
  }
}

// Exact sequential fallback (a third flagged round, or a buffer overflow -
// never seen) and the persistent stream update.
__global__ void __launch_bounds__(32) k_mut_fix(SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  if (threadIdx.x != 0) return;
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* bits = (uint32_t*)smem;
  uint16_t* arr = (uint16_t*)smem;
  const int par = v.ctl->mut_cur;
  const MutBufs b = mut_bufs(v, par);
  const int n = v.n;
  const int E = v.ctl->n_events;
  const bool overflow = (v.ctl->mut_overflow >> par) & 1;
  const int bad = overflow ? 0 : 0x7fffffff;  // redo the whole call exactly
  uint64_t q = 0;
  if (bad < E) {
    const int k_hi = max(2, n / 4);
    const uint32_t rng_k = (uint32_t)(k_hi - 1);
    int from = 0;
    if (!overflow) {
      q = b.ev_end[bad];  // the flagged event itself was sampled exactly
      from = bad + 1;
    }
    for (int e = from; e < E; ++e) {
      PcgNext pn;
      pn.r.seek_u32(*b.start, q);
      uint32_t u;
      do {
        u = pn.r.next32();
        ++q;
      } while (lemire_rejects(u, rng_k));
      const int kraw = (int)(((uint64_t)u * (rng_k + 1u)) >> 32) + 1;
      const int k = min(kraw, n / 2);
      b.ev_k[e] = k;
      b.ev_cursor[e] = q;
      if (k < 1) continue;
      CountingBounded<PcgNext> c{pn};
      q += sample_event_seq(c, n, k, v.ev_idx + (size_t)e * v.np, bits, arr);
    }
  } else if (E > 0) {
    q = b.ev_end[E - 1];
  }
  Pcg r;
  r.seek_u32(*b.start, q);
  r.store(v.streams[1]);
  v.ctl->mut_q = q;
  v.ctl->mut_overflow &= ~(1 << par);
  v.ctl->mut_pending = 1;  // the next call's walk may start
}

// Production RNG mode: every event's draws are Philox keyed by (slot,
// generation), so events are sampled independently with no stream walk:
// k = integers(1, k_hi + 1) semantics, then 2k distinct positions in random
// order (choice(n, 2k, replace=False)) as the first 2k images of a keyed
// Feistel permutation of [0, n), all lanes in parallel.  One warp per event.
__global__ void __launch_bounds__(kSampleWarps * 32) k_mut_sample_philox(
    SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * (blockDim.x >> 5) + warp;
  if (e >= v.ctl->n_events) return;
  const int n = v.n, P = v.P;
  const int slot = v.ev_slot[e];
  PhiloxStream r;
  r.init(v.philox_seed, (uint32_t)slot, (uint32_t)v.ctl->gen, kTagMutate);
  const int k_hi = max(2, n / 4);
  const int k = min((int)r.bounded((uint32_t)(k_hi - 1)) + 1, n / 2);
  if (lane == 0) v.ev_k[(size_t)v.ctl->mut_cur * P + e] = k;
  FeistelPerm perm;
  perm.init(r, (uint32_t)n);
  uint16_t* idx = v.ev_idx + (size_t)e * v.np;
  for (int t = lane; t < 2 * k; t += 32) idx[t] = (uint16_t)perm((uint32_t)t);
}

__global__ void __launch_bounds__(128) k_mut_swap(SwarmView v) {
  if (!v.ctl->mutating || v.ctl->done) return;
  const int e = blockIdx.x;
  if (e >= v.ctl->n_events) return;
  const int n = v.n, np = v.np, tid = threadIdx.x;
  const int p = v.ev_slot[e];
  const int k = v.ev_k[(size_t)v.ctl->mut_cur * v.P + e];
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
  // edge costs of the edges the swaps touched (i-1 and i for each swapped
  // position i; dcache holds the rest already - the copy from a survivor
  // brings its edges along); the fitness and pbest follow in k_fitness
  // (event list).  An edge two swaps share is written twice with the same
  // value.  Four gathers in flight per thread.
  double* dg = v.dcache + (size_t)p * np;
  const int ne = 4 * k;
  for (int e0 = tid; e0 < ne; e0 += 4 * blockDim.x) {
    double d[4];
    int at[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x;
      at[u] = -1;
      if (e < ne) {
        const int pos = idx[e >> 1];  // swapped position
        int i = (e & 1) ? pos : pos - 1;  // edge (i, i+1)
        if (i < 0) i += n;
        const int a = body[i], b = body[i + 1 == n ? 0 : i + 1];
        d[u] = ld_cost(v.cost + (size_t)a * v.ld + b);
        at[u] = i;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (at[u] >= 0) dg[at[u]] = d[u];
  }
}

}  // namespace

int64_t mstream_words(int n, int P) {
  const int k_hi = std::max(2, n / 4);
  const int kmax = std::min(k_hi, n / 2);
  const int64_t need = (int64_t)P * (1 + sample_draws(n, kmax)) + 4096;
  return round_up(need, kSeg) + kSeg;  // whole segments for the ring copies
}

cudaError_t launch_mutation_walk(const SwarmView& v, cudaStream_t s) {
  if (v.rng_mode == DPSO_RNG_PHILOX) return cudaSuccess;  // no stream walk
  const int64_t outs = v.mstream_cap / 2;
  const int64_t threads = (outs + kGenPer - 1) / kGenPer;
  k_mut_gen<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(v);
  const size_t smem = (size_t)kNSeg * kSeg * 6;  // words + skips
  set_dyn_smem((const void*)k_mut_walk, smem);
  k_mut_walk<<<1, kWalkThreads, smem, s>>>(v);
  return cudaGetLastError();
}

cudaError_t launch_mutation_pre(const SwarmView& v, cudaStream_t s) {
  const int P = v.P;
  // canon info (k | rev << 31) lives in the rank-order scratch `keep` until
  // k_mut_lists rewrites it
  int32_t* canon = v.keep;
  k_mut_hash<<<P, 128, 0, s>>>(v, canon);
  if (P <= 1024 && !getenv("DPSO_MUT_GRID")) {
    k_mut_small<<<1, 1024, 0, s>>>(v, canon);
  } else {
    const dim3 g2((P + 255) / 256, (P + kChunk - 1) / kChunk);
    k_mut_rank<<<g2, 256, 0, s>>>(v);
    k_mut_dedupe<<<g2, 256, 0, s>>>(v);
    k_mut_verify<<<(P + 3) / 4, 128, 0, s>>>(v, canon);
    k_mut_lists<<<1, 1024, 0, s>>>(v);
  }
  k_mut_copy<<<P, 128, 0, s>>>(v);
  return cudaGetLastError();
}

cudaError_t launch_mutation_post(const SwarmView& v, cudaStream_t s) {
  const int P = v.P;
  const int n = v.n;
  if (v.rng_mode == DPSO_RNG_PHILOX) {
    k_mut_sample_philox<<<(P + kSampleWarps - 1) / kSampleWarps,
                          kSampleWarps * 32, 0, s>>>(v);
    return cudaGetLastError();
  }
  // per warp: draw values + Floyd bitmap (n bits) / tail arange (n u16,
  // n > 10000 only); without room for the draw buffer the warp samples
  // sequentially.  An event draws D = F + 2k - 1 <= 4k <= n + 4 values
  // (k <= max(2, n / 4): solver.py:235-236): sizing the buffers by that
  // instead of 2n, and the bitmap by n bits, doubles the warps per SM at
  // C3 / C4
  const int scratch_words = (int)round_up(
      n > 10000 ? (n + 1) / 2 : (n + 31) / 32, 4);
  int vals_cap = (int)round_up((int64_t)n + 8, 4);
  const int idx_words = (n + 1) / 2;
  // the data-parallel sampler's arrays (n u32 + n u16 + n bytes per warp;
  // par_m = 1: on, 0: the serial lane-0 sampler)
  int par_m = getenv("DPSO_MUT_SERIAL") ? 0 : 1;
  const int par_words = par_m ? n + (3 * n + 3) / 4 + 1 : 0;
  constexpr size_t kBudget = 200 * 1024;
  if ((size_t)(vals_cap + scratch_words + idx_words + par_words) * 4 >
      kBudget) {
    vals_cap = 0;
    par_m = 0;
  }
  const size_t per_warp =
      (size_t)(vals_cap + scratch_words + idx_words + (par_m ? par_words : 0)) * 4;
  const int warps =
      (int)std::max<size_t>(1, std::min<size_t>(kSampleWarps,
                                                kBudget / per_warp));
  const size_t smem = (size_t)warps * per_warp;
  set_dyn_smem((const void*)k_mut_sample, smem);
  const unsigned grid = (unsigned)((P + warps - 1) / warps);
  k_mut_sample<<<grid, warps * 32, smem, s>>>(v, vals_cap, scratch_words,
                                              par_m);
  const size_t scratch =
      std::max<size_t>(round_up((n + 31) / 32 * 4, 16), 2 * (size_t)v.np);
  set_dyn_smem((const void*)k_mut_fix, scratch);
  k_mut_fix<<<1, 32, scratch, s>>>(v);
  return cudaGetLastError();
}

cudaError_t launch_mutation_swap(const SwarmView& v, cudaStream_t s) {
  k_mut_swap<<<v.P, 128, 0, s>>>(v);
  cudaError_t e = cudaGetLastError();
  return e ? e : launch_fitness(v, 1, s);
}

cudaError_t launch_mutation(const SwarmView& v, cudaStream_t s) {
  cudaError_t e = launch_mutation_pre(v, s);
  if (!e) e = launch_mutation_post(v, s);
  if (!e) e = launch_mutation_walk(v, s);
  if (!e) e = launch_mutation_swap(v, s);
  return e;
}

}  // namespace dpso
