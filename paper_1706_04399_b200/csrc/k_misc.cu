// Generation control, gbest/stall bookkeeping, swarm init, batch fitness and
// the nearest-neighbour construction.
//
//   k_gen_begin     gen += 1; mutation flag (solver.py:292-294, 304)
//   k_select        first-index argmin of fitness, improved flag
//                   (solver.py:307-308); optionally finalizes
//   k_finalize      argmin again after 2-opt (solver.py:318-319), gbest copy
//                   from the current position, stall, convergence, stall
//                   break (solver.py:320-328)
//   k_init_gen/scan generated init-stream windows + one-thread acceptance
//                   scan recording where each particle's draws start
//                   (solver.py:176-183)
//   k_init_build    per particle: seed / one-swap seed / permutation(n),
//                   fitness, pbest = self, vmap = identity (solver.py:37-45)
//   k_init_best     initial gbest = first minimum (solver.py:284-287)
//   k_tour_cost     _tour_cost (solver.py:48-54) for a batch of tours
//   k_nn            nearest-neighbour construction (baselines.py:110-116)
#include <float.h>
#include <math.h>
#include <stdlib.h>

#include <type_traits>

#include "dpso_internal.cuh"
#include "philox.cuh"
#include "tma.cuh"

namespace dpso {

namespace {

constexpr int kRed = 1024;

// First-index argmin over fit[0..P) with strict < (Python min / solver.py:284,
// 307): lexicographic (value, index) reduction.
__device__ void block_argmin(const double* fit, int P, double* s_v, int* s_i,
                             double* out_v, int* out_i) {
  const int tid = threadIdx.x;
  double bv = __longlong_as_double(0x7ff0000000000000ll);
  int bi = 0x7fffffff;
  for (int i = tid; i < P; i += blockDim.x) {
    double f = fit[i];
    if (bi == 0x7fffffff || f < bv) {
      bv = f;
      bi = i;
    }
  }
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
    int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    if (v2 < bv || (!(bv < v2) && i2 < bi)) {
      bv = v2;
      bi = i2;
    }
  }
  if (lane == 0) {
    s_v[warp] = bv;
    s_i[warp] = bi;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    bv = lane < nw ? s_v[lane] : __longlong_as_double(0x7ff0000000000000ll);
    bi = lane < nw ? s_i[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (v2 < bv || (!(bv < v2) && i2 < bi)) {
        bv = v2;
        bi = i2;
      }
    }
    if (lane == 0) {
      *out_v = bv;
      *out_i = bi;
    }
  }
  __syncthreads();
}

__global__ void k_gen_begin(SwarmView v) {
  if (threadIdx.x != 0) return;
  DevCtl* c = v.ctl;
  if (c->done) return;
  c->gen += 1;
  c->mutating = v.use_mutation && (c->gen % v.mutation_period == 0);
  if (c->mutating) {
    c->mut_cur ^= 1;  // use the buffers the walk prepared
    c->mut_bad = 0x7fffffff;
    c->mut_round = 0;
    c->mut_from = 0;
  }
  c->two_opt_ran = 0;
  c->improved = 0;
  c->vel_max = 0;
}

__global__ void __launch_bounds__(kRed) k_select(SwarmView v, int finalize) {
  DevCtl* c = v.ctl;
  if (c->done) return;
  __shared__ double s_v[32];
  __shared__ int s_i[32];
  __shared__ double bv;
  __shared__ int bi;
  block_argmin(v.fit, v.P, s_v, s_i, &bv, &bi);
  const int improved = bv < c->gbest_fit;
  __syncthreads();
  if (!finalize) {
    if (threadIdx.x == 0) {
      c->cand = bi;
      c->improved = improved;
    }
    return;
  }
  if (improved) {
    const uint16_t* src = v.x + (size_t)bi * v.np;
    for (int i = threadIdx.x; i < v.n; i += blockDim.x) v.gbest[i] = src[i];
  }
  if (threadIdx.x == 0) {
    c->cand = bi;
    c->improved = improved;
    if (improved) {
      c->gbest_fit = bv;
      c->stall = 0;
    } else {
      c->stall += 1;
    }
    v.conv[c->gen] = c->gbest_fit;
    c->gens_run = c->gen;
    if (c->stall >= v.stall_generations || c->gen >= v.max_generations)
      c->done = 1;
  }
}

__global__ void __launch_bounds__(kRed) k_finalize(SwarmView v) {
  DevCtl* c = v.ctl;
  if (c->done) return;
  __shared__ double s_v[32];
  __shared__ int s_i[32];
  __shared__ double bv;
  __shared__ int bi;
  __shared__ int s_improved;
  if (!c->improved) {
    // 2-opt ran for every particle: recompute cand (solver.py:318-319)
    block_argmin(v.fit, v.P, s_v, s_i, &bv, &bi);
    if (threadIdx.x == 0) {
      s_improved = bv < c->gbest_fit;
      c->two_opt_ran = 1;
      c->two_opt_count += 1;
    }
  } else {
    if (threadIdx.x == 0) {
      bi = c->cand;
      bv = v.fit[bi];
      s_improved = 1;
    }
  }
  __syncthreads();
  const int improved = s_improved;
  if (improved) {
    const uint16_t* src = v.x + (size_t)bi * v.np;
    for (int i = threadIdx.x; i < v.n; i += blockDim.x) v.gbest[i] = src[i];
  }
  if (threadIdx.x == 0) {
    c->cand = bi;
    if (improved) {
      c->gbest_fit = bv;
      c->stall = 0;
    } else {
      c->stall += 1;
    }
    v.conv[c->gen] = c->gbest_fit;
    c->gens_run = c->gen;
    if (c->stall >= v.stall_generations || c->gen >= v.max_generations)
      c->done = 1;
  }
}

// ---- island exchange on the device ---------------------------
// Record of one island: gbest fitness (fp64), rank (i64), gbest tour (np
// u16).  Every rank packs its record, an all_gather (NCCL, stream-ordered)
// concatenates them, and k_island_adopt picks the winner - smallest
// fitness, lowest rank on ties - and adopts its tour iff strictly better
// than the island's own gbest.  No host synchronisation anywhere.
struct IslandRec {
  double fit;
  int64_t rank;
};

__global__ void k_island_pack(SwarmView v, unsigned char* rec, int rank) {
  IslandRec* h = reinterpret_cast<IslandRec*>(rec);
  uint16_t* t = reinterpret_cast<uint16_t*>(rec + sizeof(IslandRec));
  if (threadIdx.x == 0) {
    h->fit = v.ctl->gbest_fit;
    h->rank = rank;
  }
  for (int i = threadIdx.x; i < v.np; i += blockDim.x)
    t[i] = i < v.n ? v.gbest[i] : (uint16_t)0;
}

__global__ void k_island_adopt(SwarmView v, const unsigned char* recs,
                               int64_t rec_bytes, int world, int rank) {
  __shared__ int s_win;
  __shared__ double s_fit;
  if (threadIdx.x == 0) {
    int win = -1;
    double wf = 0.0;
    int64_t wr = 0;
    for (int r = 0; r < world; ++r) {
      const IslandRec* h =
          reinterpret_cast<const IslandRec*>(recs + (size_t)r * rec_bytes);
      if (win < 0 || h->fit < wf || (h->fit == wf && h->rank < wr)) {
        win = r;
        wf = h->fit;
        wr = h->rank;
      }
    }
    const bool adopt = wr != rank && wf < v.ctl->gbest_fit;
    s_win = adopt ? win : -1;
    s_fit = wf;
  }
  __syncthreads();
  if (s_win < 0) return;
  const uint16_t* t = reinterpret_cast<const uint16_t*>(
      recs + (size_t)s_win * rec_bytes + sizeof(IslandRec));
  for (int i = threadIdx.x; i < v.n; i += blockDim.x) v.gbest[i] = t[i];
  if (threadIdx.x == 0) v.ctl->gbest_fit = s_fit;
}

// ---- init (numpy streams) --------------------------------------------------

// ---- init stream walk over a generated window buffer -----------------------
// The init stream (solver.py:176-183) is one numpy stream consumed by all
// particles in order, so where particle p's draws start depends on every
// earlier particle.  k_init_gen writes a window of the stream grid-wide;
// k_init_scan (one warp, speculative) runs numpy's acceptance tests over it
// from a shared-memory ring, records each particle's first draw and keeps
// its state on the device so it resumes in the next window.  The
// builder (k_init_build) then regenerates each particle's draws from its
// cursor by jump-ahead, in parallel.
struct InitScanState {
  int64_t q;      // u32 draws consumed
  int32_t p;      // particle in progress
  int32_t step;   // permutation: current max index i; seed: draw t (0..2)
  int32_t fresh;  // particle p not started yet
  int32_t done;
  int32_t fail;   // parallel walk ran off its buffer: sequential fallback
};

constexpr int kInitGenPer = 64;

__global__ void __launch_bounds__(256) k_init_gen(SwarmView v, int64_t win0) {
  const PcgState g = *v.init_start;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t outs = v.init_buf_cap / 2;
  const int64_t o0 = c * kInitGenPer;
  if (o0 >= outs) return;
  const u128 inc = {g.inc_hi, g.inc_lo};
  // window starts at fresh u32 index win0 (even): output win0/2 (0-based)
  u128 st = pcg_advance({g.state_hi, g.state_lo}, inc,
                        (uint64_t)(win0 / 2 + o0 + 1));
  const u128 M = pcg_mult();
  uint2* out = reinterpret_cast<uint2*>(v.init_buf);
  for (int r = 0; r < kInitGenPer && o0 + r < outs; ++r) {
    const uint64_t o = pcg_output(st);
    out[o0 + r] = make_uint2((uint32_t)o, (uint32_t)(o >> 32));
    st = add128(mul128(st, M), inc);
  }
}

// One thread.  The window (fresh u32 indices [win0, win0 + cap)) streams
// through a kINSeg-slot shared-memory ring of kISeg-word segments fed by
// cp.async.bulk, prefetched ahead.  The acceptance chain of numpy's masked
// rejection (random_interval) is inherently serial, but its loop-carried
// part is tiny: within a mask band a draw is accepted iff (u & mask) <= i,
// and i drops by the acceptance - a compare and a subtract per draw.  Groups
// of 8 draws (two 16-byte shared loads) run that chain back to back while
// the band cannot change inside the group; band changes, permutation ends,
// segment edges, seeded particles (a 3-draw Lemire pattern) and numpy's
// buffered half take the one-draw path.
constexpr int kISeg = 4096;  // u32 per ring segment (16 KiB)
constexpr int kINSeg = 8;    // ring slots (128 KiB), a power of two

__global__ void __launch_bounds__(32) k_init_scan(SwarmView v, int n_seed,
                                                  int64_t win0,
                                                  InitScanState* stp,
                                                  int stop_perm) {
  if (blockIdx.x != 0) return;
  extern __shared__ __align__(128) uint32_t ring[];
  __shared__ __align__(8) uint64_t bars[kINSeg];
  // All 32 lanes run the same scan (lane 0 issues copies and writes
  // results).  The loop-carried state gets a lane-dependent zero read from
  // shared memory, which keeps the chain on the vector datapath: with
  // provably uniform values the compiler moves it to the uniform datapath,
  // several times slower per dependent step.
  const int lane = threadIdx.x;
  __shared__ int s_zero[32];
  s_zero[lane] = 0;
  InitScanState st = *stp;
  if (st.done) return;
  const int n = v.n, P = v.P;
  const PcgState& g = *v.init_start;
  const int64_t h = (int64_t)g.has_uint32;
  const uint32_t ub = (uint32_t)g.uinteger;
  const int64_t cap = v.init_buf_cap;
  const int64_t wend = win0 + cap;  // fresh index past the window
  const uint32_t* buf = v.init_buf;
  const int64_t nseg = (cap + kISeg - 1) / kISeg;
  // ring: segment sg (of the window) in slot (sg - sg0) % kINSeg
  const int64_t f_start = st.q - h > win0 ? st.q - h : win0;
  const int64_t sg0 = (f_start - win0) / kISeg;
  int64_t next_issue = sg0, ready = sg0 - 1;
  if (lane == 0) {
    for (int i = 0; i < kINSeg; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  __syncwarp();
  auto wait_upto = [&](int64_t sg_hi) {
    for (int64_t sg = ready + 1; sg <= sg_hi && sg < nseg; ++sg)
      mbar_wait(&bars[(sg - sg0) % kINSeg],
                (uint32_t)(((sg - sg0) / kINSeg) & 1));
    if (sg_hi > ready) ready = sg_hi;
  };
  auto prefetch = [&](int64_t slo) {  // slots below segment slo are free
    while (next_issue < slo + kINSeg && next_issue < nseg) {
      if (next_issue - kINSeg > ready) wait_upto(next_issue - kINSeg);
      if (lane == 0) {
        const int slot = (int)((next_issue - sg0) % kINSeg);
        mbar_expect_tx(&bars[slot], kISeg * 4);
        bulk_g2s(ring + (size_t)slot * kISeg, buf + next_issue * kISeg,
                 kISeg * 4, &bars[slot]);
      }
      ++next_issue;
    }
  };
  constexpr uint32_t kMask = kINSeg * kISeg - 1;
  const uint32_t fbase = (uint32_t)(sg0 * kISeg);  // window offset of slot 0
  auto ridx = [&](int64_t f) -> uint32_t {  // ring index of fresh index f
    return ((uint32_t)(f - win0) - fbase) & kMask;
  };
  // make f's segment resident; returns the fresh index past it
  auto ensure_seg = [&](int64_t f) -> int64_t {
    const int64_t sg = (f - win0) / kISeg;
    prefetch(sg);
    wait_upto(sg);
    const int64_t e = win0 + (sg + 1) * kISeg;
    return e < wend ? e : wend;
  };
  auto mask_of = [](uint32_t x) {
    x |= x >> 1;
    x |= x >> 2;
    x |= x >> 4;
    x |= x >> 8;
    x |= x >> 16;
    return x;
  };
  int64_t resident_end = -1;  // fresh indices [.., resident_end) resident
  bool exhausted = false;
  while (st.p < P && !exhausted) {
    if (st.fresh) {
      // prefix mode: hand the permutation particles to the parallel walk
      if (stop_perm && st.p >= n_seed && st.q >= h) break;
      if (lane == 0) v.init_cursor[st.p] = (uint64_t)st.q;
      st.fresh = 0;
      if (st.p < n_seed)
        st.step = (st.p > 0 && n > 1) ? 0 : 3;  // 3 = no draws
      else
        st.step = n - 1;
    }
    if (st.p < n_seed ? st.step >= 3 : st.step <= 0) {
      ++st.p;
      st.fresh = 1;
      continue;
    }
    if (st.p >= n_seed && st.q >= h) {
      // a permutation in progress: the serial chain
      int64_t f = st.q - h;
      int S = st.step + s_zero[lane ^ 1];
      uint32_t mask = mask_of((uint32_t)S), half = mask >> 1;
      bool done = false;
      while (!done) {
        if (f >= wend) {
          exhausted = true;
          break;
        }
        if (f >= resident_end) resident_end = ensure_seg(f);
        // accepted iff (u & mask) <= S; S -= accepted, branch-free:
        // S += (int)((u & mask) - S - 1) >> 31.  Groups run while the band
        // (mask) cannot change inside them: at most `room` accepts
        // (room = S - half - 1 >= group size; no permutation end either).
        while (S - (int)half - 1 >= 32 && f + 32 <= resident_end) {
          uint32_t w[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) w[k] = ring[ridx(f + k)] & mask;
#pragma unroll
          for (int k = 0; k < 32; ++k)
            S += (int)(w[k] - (uint32_t)S - 1u) >> 31;
          f += 32;
        }
        // groups that may cross one band edge: each draw masked with this
        // band's mask and the next band's (half); the chain selects by
        // S > half.  With half >= G the group cannot cross a second edge
        // (S stays > half - G >= half / 2) nor end the permutation.
        auto group2 = [&](auto G) {
          constexpr int kG = decltype(G)::value;
          uint32_t v1[kG], v2[kG];
#pragma unroll
          for (int k = 0; k < kG; ++k) {
            const uint32_t w = ring[ridx(f + k)];
            v1[k] = w & mask;
            v2[k] = w & half;
          }
#pragma unroll
          for (int k = 0; k < kG; ++k) {
            const uint32_t vv = S > (int)half ? v1[k] : v2[k];
            S += (int)(vv - (uint32_t)S - 1u) >> 31;
          }
          f += kG;
          if (S <= (int)half) {
            mask = half;
            half >>= 1;
          }
        };
        if (half >= 32 && f + 16 <= resident_end) {
          group2(std::integral_constant<int, 16>());
          continue;
        }
        if (half >= 16 && f + 8 <= resident_end) {
          group2(std::integral_constant<int, 8>());
          continue;
        }
        const uint32_t u = ring[ridx(f)];
        ++f;
        if ((u & mask) <= (uint32_t)S) {
          --S;
          if (S == 0) {
            done = true;
          } else if (S <= (int)half) {
            mask = half;
            half >>= 1;
          }
        }
      }
      st.q = f + h;
      st.step = S;
      if (done) {
        ++st.p;
        st.fresh = 1;
      }
      continue;
    }
    // one-draw path: seeded particles and numpy's buffered half
    if (st.p < n_seed && st.step == 0 && n - 2 == 0) {
      st.step = 1;  // bounded(0) takes no draw
      continue;
    }
    uint32_t u;
    if (st.q < h) {
      u = ub;
    } else {
      const int64_t f = st.q - h;
      if (f >= wend) break;  // window exhausted: resume after the next gen
      if (f >= resident_end) resident_end = ensure_seg(f);
      u = ring[ridx(f)];
    }
    ++st.q;
    if (st.p < n_seed) {
      const uint32_t rng = st.step == 0 ? (uint32_t)(n - 2)
                           : st.step == 1 ? (uint32_t)(n - 1)
                                          : 1u;
      if (!lemire_rejects(u, rng)) ++st.step;
    } else {
      if ((u & mask_of((uint32_t)st.step)) <= (uint32_t)st.step) --st.step;
    }
  }
  wait_upto(next_issue - 1);  // drain outstanding copies
  if (lane == 0) {
    if (st.p >= P) {
      st.done = 1;
      Pcg r;
      r.seek_u32(g, (uint64_t)st.q);
      r.store(v.streams[0]);
    }
    *stp = st;
  }
}

__global__ void k_init_scan_begin(SwarmView v, InitScanState* stp) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  *v.init_start = v.streams[0];  // keep the start of the init stream
  InitScanState st;
  st.q = 0;
  st.p = 0;
  st.step = 0;
  st.fresh = 1;
  st.done = 0;
  st.fail = 0;
  *stp = st;
}

// Sequential fallback after a failed parallel walk: restart the scan state
// without re-reading streams[0] (the walk may already have advanced it).
__global__ void k_init_scan_reset(SwarmView v, InitScanState* stp) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  InitScanState st;
  st.q = 0;
  st.p = 0;
  st.step = 0;
  st.fresh = 1;
  st.done = 0;
  st.fail = 0;
  *stp = st;
}


// ---- parallel init walk ----------------------------------------------------
// The permutation particles' draws are a chain: particle p+1 starts where
// particle p's permutation(n) stopped consuming the stream.  Where a walk
// stops depends only on where it starts, so k_init_ends computes, for EVERY
// fresh index f of the generated span, the number of u32 words E[f] a
// permutation started at f consumes (numpy's masked rejection,
// random_interval: draw u accepted iff (u & mask(i)) <= i, i = n-1 .. 1).
// That is O(span x 1.4n) independent work instead of an O(span) serial
// chain.  The chain itself is then followed with pointer doubling:
// E^K by log2(K) squarings, one thread hops the P/K anchors, and P/K threads
// fill K particles each.  A walk that runs off the span marks -1 and the
// host falls back to the serial scan (k_init_scan), which stays exact.
constexpr int kEB = 256;   // starts per CTA (one per thread)
constexpr int kECH = 512;  // steps per staged chunk
constexpr int kEG = 8;     // draws per branch-free group

__device__ __forceinline__ uint32_t mask_cover(uint32_t x) {
  x |= x >> 1;
  x |= x >> 2;
  x |= x >> 4;
  x |= x >> 8;
  x |= x >> 16;
  return x;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                   smem_u32(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

__global__ void __launch_bounds__(kEB) k_init_ends(SwarmView v,
                                                   const InitScanState* stp) {
  __shared__ __align__(16) uint32_t sw[2][kEB + kECH];
  const int64_t L = v.init_buf_cap;
  const int64_t f0 = (int64_t)blockIdx.x * kEB;
  const int l = threadIdx.x;
  const int64_t f = f0 + l;
  int32_t* E = v.init_aux;
  if (stp->done) return;
  const int64_t lo = stp->q - (int64_t)v.init_start->has_uint32;
  if (f0 + kEB <= lo) {  // before the first permutation: never read
    if (f < L) E[f] = -1;
    return;
  }
  const uint32_t* buf = v.init_buf;
  auto stage = [&](int c, int b) {
    const int64_t w0 = f0 + (int64_t)c * kECH;
    for (int u = l; u < (kEB + kECH) / 4; u += kEB) {
      const int64_t w = w0 + 4 * u;
      if (w + 4 <= L) cp_async16(&sw[b][4 * u], buf + w);
    }
    cp_async_commit();
  };
  int S = v.n - 1;
  uint32_t mask = mask_cover((uint32_t)S), half = mask >> 1;
  bool active = f >= lo && f < L && S > 0;
  int32_t res = (S > 0) ? -1 : 0;
  stage(0, 0);
  for (int c = 0;; ++c) {
    cp_async_wait_all();
    if (!__syncthreads_or(active)) break;
    stage(c + 1, (c + 1) & 1);
    if (active) {
      const int64_t t0 = (int64_t)c * kECH;
      int lim = kECH;
      if (f + t0 + lim > L) lim = (int)(L - f - t0);
      const uint32_t* w = &sw[c & 1][l];
      int t = 0;
      while (t < lim) {
        if (S - (int)half - 1 >= kEG && t + kEG <= lim) {
          // no band edge and no end inside the group
          uint32_t u[kEG];
#pragma unroll
          for (int k = 0; k < kEG; ++k) u[k] = w[t + k] & mask;
#pragma unroll
          for (int k = 0; k < kEG; ++k)
            S += (int)(u[k] - (uint32_t)S - 1u) >> 31;
          t += kEG;
        } else if (half >= (uint32_t)kEG && t + kEG <= lim) {
          // at most one band edge inside the group (half >= 2G - 1)
          uint32_t v1[kEG], v2[kEG];
#pragma unroll
          for (int k = 0; k < kEG; ++k) {
            const uint32_t x = w[t + k];
            v1[k] = x & mask;
            v2[k] = x & half;
          }
#pragma unroll
          for (int k = 0; k < kEG; ++k) {
            const uint32_t vv = S > (int)half ? v1[k] : v2[k];
            S += (int)(vv - (uint32_t)S - 1u) >> 31;
          }
          t += kEG;
          if (S <= (int)half) {
            mask = half;
            half >>= 1;
          }
        } else {
          const uint32_t x = w[t];
          ++t;
          if ((x & mask) <= (uint32_t)S) {
            --S;
            if (S == 0) {
              res = (int32_t)(t0 + t);
              active = false;
              break;
            }
            if (S <= (int)half) {
              mask = half;
              half >>= 1;
            }
          }
        }
      }
      if (active && f + t0 + lim >= L) active = false;  // ran off: res = -1
    }
  }
  if (f < L) E[f] = f >= lo ? res : -1;
}

// F2[f] = F[f] + F[f + F[f]]: K-step walk lengths from K/2-step ones
__global__ void __launch_bounds__(256) k_init_square(const int32_t* F,
                                                     int32_t* F2, int64_t L) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < L;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = F[f];
    int32_t r = -1;
    if (a >= 0 && f + a < L) {
      const int32_t b = F[f + a];
      if (b >= 0) r = a + b;
    }
    F2[f] = r;
  }
}

// one thread: the start of every K-th permutation particle.
// anchor[0] = first permutation particle, anchor[1] = anchors (or -1),
// anchor[2 + j] = fresh index where particle anchor[0] + jK starts
__global__ void k_init_chain(SwarmView v, const InitScanState* stp,
                             const int32_t* FK, int K) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const InitScanState st = *stp;
  int64_t* anc = v.init_anchor;
  if (st.done) return;
  const int64_t L = v.init_buf_cap;
  int64_t f = st.q - (int64_t)v.init_start->has_uint32;
  anc[0] = st.p;
  int64_t j = 0;
  for (int64_t p = st.p; p < v.P; p += K) {
    anc[2 + j++] = f;
    if (p + K >= v.P) break;
    const int32_t a = (f >= 0 && f < L) ? FK[f] : -1;
    if (a < 0) {
      anc[1] = -1;
      return;
    }
    f += a;
  }
  anc[1] = j;
}

// thread j: particles anchor[0] + jK .. + K-1 from anchor j; the thread
// holding particle P-1 writes the final scan state and the stream position
__global__ void __launch_bounds__(128) k_init_fill(SwarmView v,
                                                   InitScanState* stp, int K) {
  const int64_t* anc = v.init_anchor;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (stp->done) return;
  const int64_t na = anc[1];
  if (na < 0) {
    if (j == 0) stp->fail = 1;
    return;
  }
  if (j >= na) return;
  const int64_t L = v.init_buf_cap;
  const int64_t h = (int64_t)v.init_start->has_uint32;
  const int32_t* E = v.init_aux;
  int64_t f = anc[2 + j];
  const int64_t p0 = anc[0] + j * K;
  for (int i = 0; i < K; ++i) {
    const int64_t p = p0 + i;
    if (p >= v.P) break;
    v.init_cursor[p] = (uint64_t)(f + h);
    const int32_t a = (f >= 0 && f < L) ? E[f] : -1;
    if (a < 0) {
      stp->fail = 1;
      return;
    }
    f += a;
    if (p == v.P - 1) {
      const int64_t q = f + h;
      stp->q = q;
      stp->p = v.P;
      stp->step = 0;
      stp->fresh = 1;
      stp->done = 1;
      Pcg r;
      r.seek_u32(*v.init_start, (uint64_t)q);
      r.store(v.streams[0]);
    }
  }
}

__global__ void __launch_bounds__(128) k_init_build(SwarmView v,
                                                    const uint16_t* seed,
                                                    int n_seed) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = v.n, np = v.np, tid = threadIdx.x;
  uint16_t* body = (uint16_t*)smem;
  for (int p = blockIdx.x; p < v.P; p += gridDim.x) {
    if (p < n_seed) {
      for (int i = tid; i < n; i += blockDim.x) body[i] = seed[i];
    } else {
      for (int i = tid; i < n; i += blockDim.x) body[i] = (uint16_t)i;
    }
    __syncthreads();
    if (v.rng_mode == DPSO_RNG_PHILOX) {
      // production mode: independent Philox draws per particle; one random
      // swap of the seed (two distinct positions), or a random permutation
      // as a keyed Feistel bijection filled by the whole CTA
      PhiloxStream r;
      r.init(v.philox_seed, (uint32_t)p, 0u, kTagInit);
      if (p < n_seed) {
        if (tid == 0 && p > 0 && n > 1) {
          const uint32_t a = r.bounded((uint32_t)(n - 1));
          uint32_t b = r.bounded((uint32_t)(n - 2));
          if (b >= a) ++b;
          const uint16_t x = body[a];
          body[a] = body[b];
          body[b] = x;
        }
      } else {
        FeistelPerm perm;
        perm.init(r, (uint32_t)n);
        for (int i = tid; i < n; i += blockDim.x)
          body[i] = (uint16_t)perm((uint32_t)i);
      }
    } else if (tid == 0) {
      Pcg r;
      r.seek_u32(*v.init_start, v.init_cursor[p]);
      if (p < n_seed) {
        if (p > 0 && n > 1) {
          uint32_t v0 = r.bounded((uint32_t)(n - 2));
          uint32_t v1 = r.bounded((uint32_t)(n - 1));
          if (v1 == v0) v1 = (uint32_t)(n - 1);
          uint32_t out[2] = {v0, v1};
          uint32_t jj = r.bounded(1u);
          uint32_t t = out[1];
          out[1] = out[jj];
          out[jj] = t;
          uint16_t x = body[out[0]];
          body[out[0]] = body[out[1]];
          body[out[1]] = x;
        }
      } else {
        for (int j = n - 1; j >= 1; --j) {
          uint32_t jj = r.interval((uint32_t)j);
          uint16_t x = body[j];
          body[j] = body[jj];
          body[jj] = x;
        }
      }
    }
    __syncthreads();
    uint16_t* xg = v.x + (size_t)p * np;
    uint16_t* pb = v.pbest + (size_t)p * np;
    double* dg = v.dcache + (size_t)p * np;
    for (int i = tid; i < n; i += blockDim.x) {
      int a = body[i], b = body[i + 1 == n ? 0 : i + 1];
      dg[i] = ld_cost(v.cost + (size_t)a * v.ld + b);
      xg[i] = (uint16_t)a;
      pb[i] = (uint16_t)a;
      if (v.vmap) v.vmap[(size_t)p * np + i] = (uint16_t)i;
      if (v.vinv) v.vinv[(size_t)p * np + i] = (uint16_t)i;
    }
    if (tid == 0 && v.vel_len) v.vel_len[p] = 0;
    __syncthreads();  // the fitness (fit = pfit) follows in k_fitness
  }
}

__global__ void __launch_bounds__(kRed) k_init_best(SwarmView v) {
  __shared__ double s_v[32];
  __shared__ int s_i[32];
  __shared__ double bv;
  __shared__ int bi;
  block_argmin(v.fit, v.P, s_v, s_i, &bv, &bi);
  const uint16_t* src = v.x + (size_t)bi * v.np;
  for (int i = threadIdx.x; i < v.n; i += blockDim.x) v.gbest[i] = src[i];
  if (threadIdx.x == 0) {
    DevCtl* c = v.ctl;
    c->gbest_fit = bv;
    c->cand = bi;
    c->gen = 0;
    c->stall = 0;
    c->done = 0;
    c->gens_run = 0;
    c->improved = 0;
    c->mutating = 0;
    c->two_opt_ran = 0;
    c->collision = 0;
    c->vel_overflow = 0;
    c->two_opt_count = 0;
    c->mut_cur = 0;
    c->mut_pending = v.use_mutation;  // first call's walk (parity 1)
    c->mut_overflow = 0;
    v.conv[0] = bv;
  }
}

// One warp per tour.
__global__ void __launch_bounds__(128) k_tour_cost(const double* cost,
                                                   int64_t ld, int n,
                                                   const uint16_t* tours,
                                                   int64_t stride, int count,
                                                   double* out,
                                                   double* dcache) {
  // one warp per tour, no shared memory (any n): lanes gather 32 edge costs
  // at a time, lane 0 sums them in the reference order (closing edge first,
  // _tour_cost solver.py:48-54) from warp shuffles
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 4 + warp;
  if (t >= count) return;
  const uint16_t* tour = tours + (size_t)t * stride;
  double total = 0.0;
  if (lane == 0)
    total = __dadd_rn(0.0, cost[(size_t)tour[n - 1] * ld + tour[0]]);
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    double dv = 0.0;
    if (i < n) {
      const int a = tour[i], b = tour[i + 1 == n ? 0 : i + 1];
      dv = cost[(size_t)a * ld + b];
      if (dcache) dcache[(size_t)t * stride + i] = dv;
    }
    const int m = min(32, n - 1 - i0);  // d_0 .. d_{n-2}
    for (int j = 0; j < 32; ++j) {
      const double x = __shfl_sync(0xffffffffu, dv, j);
      if (lane == 0 && j < m) total = __dadd_rn(total, x);
    }
  }
  if (lane == 0) out[t] = total;
}

// Greedy nearest neighbour from `start` (baselines.py:110-116): n-1 steps,
// each a CTA-wide argmin over unvisited nodes of row `cur` on (cost, index).
__global__ void __launch_bounds__(1024) k_nn(const double* cost, int64_t ld,
                                             int n, int start, int32_t* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* visited = smem;
  __shared__ double s_v[32];
  __shared__ int s_i[32];
  __shared__ int s_cur;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < n; i += blockDim.x) visited[i] = 0;
  __syncthreads();
  if (tid == 0) {
    visited[start] = 1;
    out[0] = start;
    s_cur = start;
  }
  __syncthreads();
  for (int step = 1; step < n; ++step) {
    const double* row = cost + (size_t)s_cur * ld;
    double bv = __longlong_as_double(0x7ff0000000000000ll);
    int bi = 0x7fffffff;
    for (int j = tid; j < n; j += blockDim.x) {
      if (!visited[j]) {
        double c = row[j];
        if (bi == 0x7fffffff || c < bv) {
          bv = c;
          bi = j;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      bool take = (i2 != 0x7fffffff) &&
                  (bi == 0x7fffffff || v2 < bv || (!(bv < v2) && i2 < bi));
      if (take) {
        bv = v2;
        bi = i2;
      }
    }
    if (lane == 0) {
      s_v[warp] = bv;
      s_i[warp] = bi;
    }
    __syncthreads();
    if (warp == 0) {
      const int nw = blockDim.x >> 5;
      bv = lane < nw ? s_v[lane] : __longlong_as_double(0x7ff0000000000000ll);
      bi = lane < nw ? s_i[lane] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        bool take = (i2 != 0x7fffffff) &&
                    (bi == 0x7fffffff || v2 < bv || (!(bv < v2) && i2 < bi));
        if (take) {
          bv = v2;
          bi = i2;
        }
      }
      if (lane == 0) {
        visited[bi] = 1;
        out[step] = bi;
        s_cur = bi;
      }
    }
    __syncthreads();
  }
}

// Python's builtin sum() over the closed tour's edges, as CPython 3.12+
// evaluates it for floats (bltinmodule.c builtin_sum_impl: the int start 0 is
// added to the first item, then Neumaier-compensated accumulation, and the
// compensation is added at the end when it is non-zero and finite).  This is
// what baselines.py:117 computes.
__global__ void k_pysum_tour(const double* cost, int64_t ld, int n,
                             const int32_t* body, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double f = 0.0, c = 0.0;
  for (int k = 0; k < n; ++k) {
    const double x = cost[(size_t)body[k] * ld + body[k + 1 == n ? 0 : k + 1]];
    if (k == 0) {
      f = x;  // int 0 + float x
      continue;
    }
    const double t = __dadd_rn(f, x);
    if (fabs(f) >= fabs(x))
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
    else
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f = __dadd_rn(f, c);
  *out = f;
}

}  // namespace

cudaError_t launch_pysum_tour(const double* cost, int64_t ld, int32_t n,
                              const int32_t* body, double* out,
                              cudaStream_t s) {
  k_pysum_tour<<<1, 32, 0, s>>>(cost, ld, n, body, out);
  return cudaGetLastError();
}

int64_t island_rec_bytes(int np) {
  return (int64_t)sizeof(IslandRec) + round_up(2 * (int64_t)np, 16);
}

cudaError_t launch_island_pack(const SwarmView& v, void* rec, int rank,
                               cudaStream_t s) {
  k_island_pack<<<1, 256, 0, s>>>(v, (unsigned char*)rec, rank);
  return cudaGetLastError();
}

cudaError_t launch_island_adopt(const SwarmView& v, const void* recs,
                                int world, int rank, cudaStream_t s) {
  k_island_adopt<<<1, 256, 0, s>>>(v, (const unsigned char*)recs,
                                   island_rec_bytes(v.np), world, rank);
  return cudaGetLastError();
}

cudaError_t launch_gen_begin(const SwarmView& v, cudaStream_t s) {
  k_gen_begin<<<1, 32, 0, s>>>(v);
  return cudaGetLastError();
}

cudaError_t launch_select(const SwarmView& v, bool finalize, cudaStream_t s) {
  k_select<<<1, kRed, 0, s>>>(v, finalize ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const SwarmView& v, cudaStream_t s) {
  k_finalize<<<1, kRed, 0, s>>>(v);
  return cudaGetLastError();
}

// Init of the numpy streams: the parallel walk when the expected span fits
// the buffer (init_parallel), else (or if a walk ran off the span) the
// serial scan, window by window (one sync per window; init runs once).
static cudaError_t init_serial(const SwarmView& v, int32_t n_seed,
                               InitScanState* stp, cudaStream_t s) {
  InitScanState h;
  const size_t ring = (size_t)kINSeg * kISeg * 4;
  cudaError_t e = set_dyn_smem((const void*)k_init_scan, ring);
  if (e) return e;
  for (int64_t win0 = 0;; win0 += v.init_buf_cap) {
    const int64_t outs = v.init_buf_cap / 2;
    const int64_t thr = (outs + kInitGenPer - 1) / kInitGenPer;
    k_init_gen<<<(unsigned)((thr + 255) / 256), 256, 0, s>>>(v, win0);
    k_init_scan<<<1, 32, ring, s>>>(v, n_seed, win0, stp, 0);
    e = cudaMemcpyAsync(&h, stp, sizeof h, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) return e;
    if (h.done) return cudaSuccess;
  }
}

static cudaError_t init_parallel(const SwarmView& v, int32_t n_seed,
                                 InitScanState* stp, cudaStream_t s,
                                 bool* ok) {
  const int64_t L = v.init_buf_cap;
  const int64_t outs = L / 2;
  const int64_t thr = (outs + kInitGenPer - 1) / kInitGenPer;
  k_init_gen<<<(unsigned)((thr + 255) / 256), 256, 0, s>>>(v, 0);
  // seeded particles (and a permutation whose first draw is numpy's
  // buffered half) stay on the serial scan: a few draws each
  const size_t ring = (size_t)kINSeg * kISeg * 4;
  cudaError_t e = set_dyn_smem((const void*)k_init_scan, ring);
  if (e) return e;
  k_init_scan<<<1, 32, ring, s>>>(v, n_seed, 0, stp, 1);
  k_init_ends<<<(unsigned)((L + kEB - 1) / kEB), kEB, 0, s>>>(v, stp);
  const int64_t perms = (int64_t)v.P - n_seed;
  int K = 1;
  while ((int64_t)K * K < perms) K <<= 1;
  const int32_t* FK = v.init_aux;
  int32_t* T[2] = {v.init_aux + L, v.init_aux + 2 * L};
  int lev = 0;
  for (int k = 1; k < K; k <<= 1, ++lev) {
    k_init_square<<<148 * 8, 256, 0, s>>>(FK, T[lev & 1], L);
    FK = T[lev & 1];
  }
  k_init_chain<<<1, 32, 0, s>>>(v, stp, FK, K);
  const int64_t na = (perms + K - 1) / K + 2;
  k_init_fill<<<(unsigned)((na + 127) / 128), 128, 0, s>>>(v, stp, K);
  InitScanState h;
  e = cudaMemcpyAsync(&h, stp, sizeof h, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) return e;
  *ok = h.done && !h.fail;
  return cudaSuccess;
}

cudaError_t launch_init(const SwarmView& v, const uint16_t* dev_seed,
                        int32_t n_seed, cudaStream_t s, int* path) {
  if (v.rng_mode == DPSO_RNG_NUMPY) {
    InitScanState* stp = reinterpret_cast<InitScanState*>(v.init_state);
    k_init_scan_begin<<<1, 32, 0, s>>>(v, stp);
    bool ok = false;
    cudaError_t e = cudaSuccess;
    if (v.init_parallel && !getenv("DPSO_INIT_SERIAL"))
      e = init_parallel(v, n_seed, stp, s, &ok);
    if (e) return e;
    if (!ok) {
      k_init_scan_reset<<<1, 32, 0, s>>>(v, stp);
      e = init_serial(v, n_seed, stp, s);
      if (e) return e;
    }
    if (path) *path = ok ? 1 : 0;
  }
  const size_t smem = round_up((int64_t)2 * v.np, 16);
  set_dyn_smem((const void*)k_init_build, smem);
  k_init_build<<<v.P, 128, smem, s>>>(v, dev_seed, n_seed);
  cudaError_t e = cudaGetLastError();
  return e ? e : launch_fitness(v, 2, s);
}

// numpy's permutation(n): mean and variance of the u32 draws one
// permutation consumes (masked rejection, accept probability (i+1)/(mask+1))
static void perm_draw_moments(int n, double* mean, double* var) {
  double m = 0.0, q = 0.0;
  for (int i = 1; i < n; ++i) {
    uint32_t mk = (uint32_t)i;
    mk |= mk >> 1;
    mk |= mk >> 2;
    mk |= mk >> 4;
    mk |= mk >> 8;
    mk |= mk >> 16;
    const double p = (i + 1.0) / ((double)mk + 1.0);
    m += 1.0 / p;
    q += (1.0 - p) / (p * p);
  }
  *mean = m;
  *var = q;
}

static int64_t init_span_words(int n, int P) {
  double mu, var;
  perm_draw_moments(n, &mu, &var);
  const double span = (double)P * (mu + 4.0) + 12.0 * sqrt((double)P * var) +
                      4.0 * mu + 8192.0;
  return round_up((int64_t)span, kISeg);
}

constexpr int64_t kInitParCap = 1ll << 28;  // u32 words (1 GiB + 3 GiB aux)

bool init_parallel_ok(int n, int P) {
  return init_span_words(n, P) <= kInitParCap;
}

int64_t init_buf_words(int n, int P) {
  if (init_parallel_ok(n, P)) return init_span_words(n, P);
  // serial scan: a window it resumes across
  int64_t want = (int64_t)P * (2 * (int64_t)n + 64) + 4096;
  const int64_t cap = 32ll << 20;  // 128 MiB window
  want = want < cap ? want : cap;
  return round_up(want, kISeg);  // whole ring segments
}

cudaError_t launch_init_best(const SwarmView& v, cudaStream_t s) {
  k_init_best<<<1, kRed, 0, s>>>(v);
  return cudaGetLastError();
}

cudaError_t launch_tour_cost_rows(const double* cost, int64_t ld, int32_t n,
                                  const uint16_t* tours, int64_t stride,
                                  int32_t count, double* out, double* dcache,
                                  cudaStream_t s) {
  k_tour_cost<<<(count + 3) / 4, 128, 0, s>>>(cost, ld, n, tours, stride,
                                              count, out, dcache);
  return cudaGetLastError();
}

cudaError_t launch_nn(const double* cost, int64_t ld, int32_t n, int32_t start,
                      int32_t* out, cudaStream_t s) {
  k_nn<<<1, 1024, round_up(n, 16), s>>>(cost, ld, n, start, out);
  return cudaGetLastError();
}

}  // namespace dpso
