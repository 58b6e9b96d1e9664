// Velocity / position update, fitness and pbest (solver.py:190-220).
//
// One CTA per particle.  For w == 1 (the paper default) the reference keeps
// a composed velocity permutation vmap and moves x <- vmap o x after folding
// the first k1 transpositions of the left-to-right repair x -> pbest and the
// first k2 of x -> gbest into it (solver.py:196-212).  The repair is a
// sequential scan in the reference; here it is computed data-parallel in
// shared memory:
//   pi(i)  = pos_x(T[i]);  emitting positions = non-maximal members of the
//            non-trivial pi-cycles (cycle maxima by pointer jumping);
//   t      = k-th emitting position (block scan);
//   cur_t[q] = T[q] (q <= t) or T[r], r = first position > t on the backward
//            pi-orbit of q (pointer jumping with threshold t);
//   sigma(x[q]) = cur_t[q];  vmap' = sigma2 o sigma1 o vmap;  x' = vmap' o x.
// Work is O(n log n) per particle with every thread busy; no transposition
// list is ever materialised.  Fitness is then summed in the reference's
// sequential order (closing edge first) so downstream decisions are exact.
//
// For w < 1 the reference keeps an explicit transposition list and replays
// it (solver.py:213-216); that path runs the repair sequentially in one
// thread per particle (k_update_seq) on a bounded per-particle ring.
#include <stdlib.h>

#include <algorithm>

#include "dpso_internal.cuh"
#include "philox.cuh"
#include "tma.cuh"

namespace dpso {

namespace {

// r1, r2 = p.rng.random(2) (solver.py:191): the particle's numpy stream, or
// Philox keyed by (particle, generation) in the production mode
__device__ __forceinline__ void draw_r1r2(const SwarmView& v, int p,
                                          double* r1, double* r2) {
  if (v.rng_mode == DPSO_RNG_PHILOX) {
    PhiloxStream ps;
    ps.init(v.philox_seed, (uint32_t)p, (uint32_t)v.ctl->gen, kTagUpdate);
    *r1 = ps.next_double();
    *r2 = ps.next_double();
    return;
  }
  Pcg r;
  r.load(v.streams[2 + p]);
  *r1 = r.next_double();
  *r2 = r.next_double();
  r.store(v.streams[2 + p]);
}

template <int T>
__device__ __forceinline__ int block_excl_scan(int val, int* s_warp,
                                               int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = val;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (T / 32) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (T / 32)) s_warp[lane] = w;  // inclusive per-warp totals
  }
  __syncthreads();
  int base = warp > 0 ? s_warp[warp - 1] : 0;
  *total = s_warp[T / 32 - 1];
  __syncthreads();
  return base + x - val;
}

// n u16 (16-B aligned rows) in 16-byte pieces plus a scalar tail; the
// padding past n is left alone
template <int T>
__device__ __forceinline__ void copy_row16(uint16_t* dst, const uint16_t* src,
                                           int n) {
  const int nv = n >> 3;
  for (int k = threadIdx.x; k < nv; k += T)
    reinterpret_cast<uint4*>(dst)[k] = reinterpret_cast<const uint4*>(src)[k];
  const int i = 8 * nv + (int)threadIdx.x;
  if (i < n) dst[i] = src[i];
}

// sigma (value permutation of the first prefix_len(c, L) repair
// transpositions of x -> target) into sout[value].  GT: the target is read
// from global memory (tgt_g) instead of a shared copy sT (large n: the
// low-shared-memory update); sout may then alias sW (written only after the
// last read of sW).
// emit (w < 1): also write the first k repair transpositions, in the
// reference's order, to emit[0 .. k) as (have | want << 16) and return k
// (the e-th emitting position p_e: want = T[p_e]; have = the value at p_e
// after the positions < p_e are repaired = T[r], r the first position >= p_e
// on p_e's backward pi-orbit - the sum of these walks is O(n log n))
template <int T, bool GT = false>
__device__ int sigma_pass(const uint16_t* __restrict__ tgt_g, double c,
                          int n, int R, const uint16_t* sx,
                          const uint16_t* sposx, uint16_t* sT, uint16_t* sB,
                          uint32_t* sW, uint16_t* sout, int* s_warp,
                          int* s_misc, uint32_t* emit = nullptr) {
  const int tid = threadIdx.x;
  if (GT) {
    sT = const_cast<uint16_t*>(tgt_g);  // reads only (via the cache)
  } else {
    copy_row16<T>(sT, tgt_g, n);
    __syncthreads();
  }
  // pi, its inverse (backward orbit), and (J, M) = (pi(p), p) for jumping
  // J is kept as a byte offset into sW when it fits 16 bits (n <= 16384):
  // a jump step is then LDS, LDS [sW + J], one SIMD max and one byte permute
  const bool jb = n <= 16384;
  for (int i = tid; i < n; i += T) {
    int pi = sposx[GT ? __ldg(tgt_g + i) : sT[i]];
    sB[pi] = (uint16_t)i;
    sW[i] = (uint32_t)(jb ? 4 * pi : pi) | ((uint32_t)i << 16);
  }
  __syncthreads();
  // cycle maxima: M(p) = max over 2^r orbit elements, J(p) = pi^(2^r)(p).
  // (J, M) is one 32-bit word, so in-place jumping reads consistent pairs.
  // Four elements per step with their loads in flight together (in place:
  // a word read after its owner's update has jumped further, which only
  // speeds convergence - M stays the max of a contiguous orbit segment)
  // A round in which no M changes ends the jumping: then every segment
  // already covers its cycle's maximum (the non-covering element nearest
  // the maximum would have picked it up from its jump target), so M is the
  // cycle maximum everywhere.  Converged swarms (x near its target: short
  // cycles) stop after a few rounds.
  if (jb) {
    const unsigned char* base = reinterpret_cast<const unsigned char*>(sW);
    for (int r = 0; r < R; ++r) {
      int changed = 0;
      for (int p0 = tid; p0 < n; p0 += 4 * T) {
        uint32_t w[4], w2[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int p = p0 + k * T;
          w[k] = p < n ? sW[p] : 0u;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          w2[k] = *reinterpret_cast<const uint32_t*>(base + (w[k] & 0xFFFFu));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int p = p0 + k * T;
          // low half: J of the target; high half: max of the two M
          const uint32_t m2 = __vmaxu2(w[k], w2[k]);
          if (p < n) {
            changed |= (m2 ^ w[k]) >> 16;
            sW[p] = __byte_perm(w2[k], m2, 0x7610);
          }
        }
      }
      if (!__syncthreads_or(changed)) break;
    }
  } else
  for (int r = 0; r < R; ++r) {
    for (int p0 = tid; p0 < n; p0 += 4 * T) {
      uint32_t w[4], w2[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int p = p0 + k * T;
        w[k] = p < n ? sW[p] : 0u;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) w2[k] = sW[w[k] & 0xFFFFu];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int p = p0 + k * T;
        if (p < n)
          sW[p] = (w2[k] & 0xFFFFu) | (max(w[k] >> 16, w2[k] >> 16) << 16);
      }
    }
    __syncthreads();
  }
  // emitting = not the maximum of its cycle; contiguous chunk per thread
  const int per = (n + T - 1) / T;
  const int c0 = min(n, tid * per), c1 = min(n, c0 + per);
  int cnt = 0;
  for (int p = c0; p < c1; ++p) cnt += ((int)(sW[p] >> 16) != p);
  int L;
  int excl = block_excl_scan<T>(cnt, s_warp, &L);
  const int k = prefix_len(c, L);
  if (k == 0) {
    for (int v = tid; v < n; v += T) sout[v] = (uint16_t)v;
    __syncthreads();
    return 0;
  }
  if (emit && excl < k) {
    int e = excl;
    for (int p = c0; p < c1 && e < k; ++p) {
      if ((int)(sW[p] >> 16) != p) {
        int b = sB[p];
        while (b < p) b = sB[b];
        const uint32_t want = GT ? __ldg(tgt_g + p) : sT[p];
        const uint32_t have = GT ? __ldg(tgt_g + b) : sT[b];
        emit[e++] = have | (want << 16);
      }
    }
  }
  if (excl <= k - 1 && k - 1 < excl + cnt) {
    int need = k - 1 - excl;
    for (int p = c0; p < c1; ++p) {
      if ((int)(sW[p] >> 16) != p) {
        if (need == 0) {
          s_misc[0] = p;
          break;
        }
        --need;
      }
    }
  }
  __syncthreads();
  const int t = s_misc[0];
  // cur_t[q] = T[q] for q <= t; for q > t, T[r] with r the first position
  // > t on q's backward orbit pi^-1(q), pi^-2(q), ... (q itself at the
  // latest).  A direct walk: the positions <= t skipped on the way are each
  // on exactly one walk, so the total work is O(n), and runs are short
  // (the prefix fraction is c = phi * r < 1).
  for (int q = tid; q < n; q += T) {
    uint16_t cur;
    if (q <= t) {
      cur = GT ? __ldg(tgt_g + q) : sT[q];
    } else {
      int b = sB[q];
      while (b <= t) b = sB[b];
      cur = GT ? __ldg(tgt_g + b) : sT[b];
    }
    sout[sx[q]] = cur;
  }
  __syncthreads();
  return k;
}

// x' is in sx: write x and the edge costs d_i (dcache).  The fitness and
// pbest (solver.py:217-220) follow in k_fitness, one warp per particle, so
// the sequential fp64 sums of all particles run concurrently instead of on
// one thread of each CTA.
// sold (nullable): the tour before the move; an edge whose two endpoints
// are unchanged keeps its cached cost (no gather, no store)
template <int T>
__device__ void finish_particle(const SwarmView& v, int p, const uint16_t* sx,
                                const uint16_t* sold = nullptr) {
  const int n = v.n, np = v.np, tid = threadIdx.x;
  uint16_t* xg = v.x + (size_t)p * np;
  double* dg = v.dcache + (size_t)p * np;
  // edge-cost gathers four at a time (L2 or, for a matrix beyond L2, HBM
  // latency: keep them in flight together)
  for (int i0 = tid; i0 < n; i0 += 4 * T) {
    double d[4];
    bool moved[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + k * T;
      moved[k] = false;
      if (i < n) {
        const int i1 = i + 1 == n ? 0 : i + 1;
        const int a = sx[i], b = sx[i1];
        moved[k] = !sold || a != sold[i] || b != sold[i1];
        if (moved[k]) d[k] = ld_cost(v.cost + (size_t)a * v.ld + b);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + k * T;
      if (moved[k]) dg[i] = d[k];
    }
  }
  copy_row16<T>(xg, sx, n);
  __syncthreads();
}

template <int T>
__global__ void __launch_bounds__(T) k_update_w1(SwarmView v, int R) {
  if (v.ctl->done) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = v.n, np = v.np, tid = threadIdx.x;
  uint16_t* sx = (uint16_t*)smem;
  uint16_t* sposx = sx + np;
  uint16_t* ssig1 = sposx + np;
  uint16_t* ssig2 = ssig1 + np;
  uint16_t* sT = ssig2 + np;
  uint16_t* sB = sT + np;
  uint32_t* sW = (uint32_t*)(sB + np);
  __shared__ int s_warp[32];
  __shared__ int s_misc[4];
  __shared__ double s_c[2];

  for (int p = blockIdx.x; p < v.P; p += gridDim.x) {
    const uint16_t* xg = v.x + (size_t)p * np;
    copy_row16<T>(sx, xg, n);
    __syncthreads();
    for (int i = tid; i < n; i += T) sposx[sx[i]] = (uint16_t)i;
    if (tid == 0) {
      double r1, r2;
      draw_r1r2(v, p, &r1, &r2);
      s_c[0] = __dmul_rn(v.cognitive, r1);
      s_c[1] = __dmul_rn(v.social, r2);
    }
    __syncthreads();
    sigma_pass<T>(v.pbest + (size_t)p * np, s_c[0], n, R, sx, sposx, sT, sB,
                  sW, ssig1, s_warp, s_misc);
    sigma_pass<T>(v.gbest, s_c[1], n, R, sx, sposx, sT, sB, sW, ssig2, s_warp,
                  s_misc);
    // vmap' = sigma2 o sigma1 o vmap (solver.py:201-209), x' = vmap' o x
    uint16_t* vm = v.vmap + (size_t)p * np;
    copy_row16<T>(sT, vm, n);
    __syncthreads();
    for (int u = tid; u < n; u += T) sB[u] = ssig2[ssig1[sT[u]]];
    __syncthreads();
    copy_row16<T>(vm, sB, n);
    // x' = vmap' o x into sposx (free now); sx keeps x for the edge reuse
    for (int i = tid; i < n; i += T) sposx[i] = sB[sx[i]];
    __syncthreads();
    finish_particle<T>(v, p, sposx, sx);
  }
}

// Large n (beyond what 16 B/node of shared memory allows, n > 14000): 10
// B/node - x, pos_x, the backward orbit and the jump words, which also hold
// sigma once the jumping is done; the targets are read through the cache and
// sigma1 is folded into vmap in global memory right away.
template <int T>
__global__ void __launch_bounds__(T) k_update_w1_lowmem(SwarmView v, int R) {
  if (v.ctl->done) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = v.n, np = v.np, tid = threadIdx.x;
  uint16_t* sx = (uint16_t*)smem;
  uint16_t* sposx = sx + np;
  uint16_t* sB = sposx + np;
  uint32_t* sW = (uint32_t*)(sB + np);
  uint16_t* ssig = (uint16_t*)sW;  // sigma after the jumping
  __shared__ int s_warp[32];
  __shared__ int s_misc[4];
  __shared__ double s_c[2];
  for (int p = blockIdx.x; p < v.P; p += gridDim.x) {
    copy_row16<T>(sx, v.x + (size_t)p * np, n);
    __syncthreads();
    for (int i = tid; i < n; i += T) sposx[sx[i]] = (uint16_t)i;
    if (tid == 0) {
      double r1, r2;
      draw_r1r2(v, p, &r1, &r2);
      s_c[0] = __dmul_rn(v.cognitive, r1);
      s_c[1] = __dmul_rn(v.social, r2);
    }
    __syncthreads();
    uint16_t* vm = v.vmap + (size_t)p * np;
    sigma_pass<T, true>(v.pbest + (size_t)p * np, s_c[0], n, R, sx, sposx,
                        nullptr, sB, sW, ssig, s_warp, s_misc);
    // vmap1 = sigma1 o vmap (solver.py:201-205), in place in global memory
    for (int u = tid; u < n; u += T) vm[u] = ssig[vm[u]];
    __syncthreads();
    sigma_pass<T, true>(v.gbest, s_c[1], n, R, sx, sposx, nullptr, sB, sW,
                        ssig, s_warp, s_misc);
    // vmap' = sigma2 o vmap1 into sB (free now) and global; x' = vmap' o x
    for (int u = tid; u < n; u += T) {
      const uint16_t w = ssig[vm[u]];
      sB[u] = w;
      vm[u] = w;
    }
    __syncthreads();
    for (int i = tid; i < n; i += T) sposx[i] = sB[sx[i]];
    __syncthreads();
    finish_particle<T>(v, p, sposx, sx);
  }
}

// ---- w < 1: explicit transposition lists (solver.py:213-216) -------------

__device__ int repair_seq(const uint16_t* sx, const uint16_t* tgt, int n,
                          uint16_t* cur, uint16_t* pos, uint32_t* out) {
  for (int i = 0; i < n; ++i) {
    cur[i] = sx[i];
    pos[sx[i]] = (uint16_t)i;
  }
  int cnt = 0;
  for (int i = 0; i < n; ++i) {
    uint16_t want = tgt[i], have = cur[i];
    if (have != want) {
      int j = pos[want];
      cur[j] = have;
      pos[have] = (uint16_t)j;
      out[cnt++] = (uint32_t)have | ((uint32_t)want << 16);
    }
  }
  return cnt;
}

// w < 1, CTA-parallel (solver.py:213-216): the velocity list v is kept,
// and with it V = the value map of the whole list (apply_open(body, v) ==
// V o body) and V^-1, so a generation never replays the list:
//   1. truncation to the kept prefix v[0:k0], k0 = _prefix_len(w, len):
//      V <- tau_{k0+1} o ... o tau_len o V (the dropped suffix undone, last
//      first, by left multiplication on V / V^-1: O(len - k0), one thread);
//   2. t1, t2 = the first k1 / k2 repair transpositions x -> pbest /
//      x -> gbest, data-parallel (sigma_pass, which also emits them in the
//      reference's order straight into v[k0 ..]);
//   3. V <- sigma2 o sigma1 o V, x' = V o x (as for w == 1).
// The lists grow on the host (ensure_velocity); overflow fails loudly.
template <int T>
__global__ void __launch_bounds__(T) k_update_wl(SwarmView v, int R) {
  if (v.ctl->done) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = v.n, np = v.np, tid = threadIdx.x;
  uint16_t* sx = (uint16_t*)smem;
  uint16_t* sposx = sx + np;
  uint16_t* ssig1 = sposx + np;
  uint16_t* ssig2 = ssig1 + np;
  uint16_t* sT = ssig2 + np;
  uint16_t* sB = sT + np;
  uint32_t* sW = (uint32_t*)(sB + np);
  uint16_t* sV = (uint16_t*)(sW + np);
  uint16_t* sVi = sV + np;
  __shared__ int s_warp[32];
  __shared__ int s_misc[4];
  __shared__ int s_k[4];
  __shared__ double s_c[2];
  const int64_t stride = v.vel_cap + 2 * (int64_t)n;
  for (int p = blockIdx.x; p < v.P; p += gridDim.x) {
    const uint16_t* xg = v.x + (size_t)p * np;
    uint16_t* vg = v.vmap + (size_t)p * np;
    uint16_t* vig = v.vinv + (size_t)p * np;
    uint32_t* lst = v.vel + (size_t)p * stride;
    copy_row16<T>(sx, xg, n);
    copy_row16<T>(sV, vg, n);
    copy_row16<T>(sVi, vig, n);
    __syncthreads();
    for (int i = tid; i < n; i += T) sposx[sx[i]] = (uint16_t)i;
    if (tid == 0) {
      double r1, r2;
      draw_r1r2(v, p, &r1, &r2);
      s_c[0] = __dmul_rn(v.cognitive, r1);
      s_c[1] = __dmul_rn(v.social, r2);
      const int len = v.vel_len[p];
      const int k0 = prefix_len(v.inertia, len);
      // undo the dropped suffix v[k0:len], last first
      for (int e = len - 1; e >= k0; --e) {
        const uint32_t ab = lst[e];
        const uint16_t a = ab & 0xFFFFu, b = ab >> 16;
        const uint16_t ia = sVi[a], ib = sVi[b];
        sV[ia] = b;
        sV[ib] = a;
        sVi[a] = ib;
        sVi[b] = ia;
      }
      s_k[0] = k0;
    }
    __syncthreads();
    const int k0 = s_k[0];
    // the lists have room for both prefixes (the host grows them); the
    // emission writes the entries it keeps only
    int k1 = sigma_pass<T>(v.pbest + (size_t)p * np, s_c[0], n, R, sx, sposx,
                           sT, sB, sW, ssig1, s_warp, s_misc, lst + k0);
    if (tid == 0) s_k[1] = k1;
    __syncthreads();
    k1 = s_k[1];
    int k2 = sigma_pass<T>(v.gbest, s_c[1], n, R, sx, sposx, sT, sB, sW,
                           ssig2, s_warp, s_misc, lst + k0 + k1);
    if (tid == 0) s_k[2] = k2;
    __syncthreads();
    k2 = s_k[2];
    if (tid == 0) {
      if ((int64_t)k0 + k1 + k2 > v.vel_cap) v.ctl->vel_overflow = 1;
      v.vel_len[p] = k0 + k1 + k2;
      atomicMax(&v.ctl->vel_max, k0 + k1 + k2);
    }
    // V' = sigma2 o sigma1 o V, V'^-1, x' = V' o x
    for (int u = tid; u < n; u += T) {
      const uint16_t w = ssig2[ssig1[sV[u]]];
      sT[u] = w;
      sB[w] = (uint16_t)u;
    }
    __syncthreads();
    copy_row16<T>(vg, sT, n);
    copy_row16<T>(vig, sB, n);
    for (int i = tid; i < n; i += T) sposx[i] = sT[sx[i]];
    __syncthreads();
    finish_particle<T>(v, p, sposx, sx);
  }
}

__global__ void __launch_bounds__(32) k_update_seq(SwarmView v) {
  if (v.ctl->done) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = v.n, np = v.np, tid = threadIdx.x;
  uint16_t* sx = (uint16_t*)smem;
  uint16_t* scur = sx + np;
  uint16_t* spos = scur + np;
  uint16_t* sgt = spos + np;
  for (int p = blockIdx.x; p < v.P; p += gridDim.x) {
    const uint16_t* xg = v.x + (size_t)p * np;
    for (int i = tid; i < n; i += 32) sx[i] = xg[i];
    __syncwarp();
    if (tid == 0) {
      double r1, r2;
      draw_r1r2(v, p, &r1, &r2);
      double c1 = __dmul_rn(v.cognitive, r1), c2 = __dmul_rn(v.social, r2);
      const int64_t stride = v.vel_cap + 2 * (int64_t)n;
      uint32_t* lst = v.vel + (size_t)p * stride;
      uint32_t* t1 = lst + v.vel_cap;
      uint32_t* t2 = t1 + n;
      const uint16_t* pb = v.pbest + (size_t)p * np;
      for (int i = 0; i < n; ++i) sgt[i] = pb[i];
      int L1 = repair_seq(sx, sgt, n, scur, spos, t1);
      int k1 = prefix_len(c1, L1);
      for (int i = 0; i < n; ++i) sgt[i] = v.gbest[i];
      int L2 = repair_seq(sx, sgt, n, scur, spos, t2);
      int k2 = prefix_len(c2, L2);
      int len = v.vel_len[p];
      int k0 = prefix_len(v.inertia, len);
      // the host grows the lists before every batch of generations
      // (dpso_api.cu ensure_velocity) so this cannot trigger; if it ever
      // does, the run fails loudly instead of diverging from the reference
      if ((int64_t)k0 + k1 + k2 > v.vel_cap) {
        v.ctl->vel_overflow = 1;
        k0 = k1 = k2 = 0;
      }
      for (int e = 0; e < k1; ++e) lst[k0 + e] = t1[e];
      for (int e = 0; e < k2; ++e) lst[k0 + k1 + e] = t2[e];
      len = k0 + k1 + k2;
      v.vel_len[p] = len;
      atomicMax(&v.ctl->vel_max, len);
      // _apply_open (solver.py:72-79) on the whole new velocity
      for (int i = 0; i < n; ++i) {
        scur[i] = sx[i];
        spos[sx[i]] = (uint16_t)i;
      }
      for (int e = 0; e < len; ++e) {
        uint32_t ab = lst[e];
        uint16_t a = ab & 0xFFFFu, b = ab >> 16;
        uint16_t ia = spos[a], ib = spos[b];
        scur[ia] = b;
        scur[ib] = a;
        spos[a] = ib;
        spos[b] = ia;
      }
      for (int i = 0; i < n; ++i) sx[i] = scur[i];
    }
    __syncwarp();
    finish_particle<32>(v, p, sx);
  }
}

// Fitness of a particle from its dcache row in the reference's order
// (_tour_cost, solver.py:48-54: the closing edge first, then left to
// right), then pbest (solver.py:217-220).  One warp per particle (all
// particles, or the mutated ones of this call: the mutation's event list,
// events with k < 1 leave their particle untouched).  The sum is one
// dependent fp64 chain; lane 0 feeds it from a 2-slot shared-memory ring of
// kFitChunk-double chunks that cp.async.bulk copies one chunk ahead, so the
// chain never waits on L2.
constexpr int kFitChunk = 256;  // doubles per chunk (2 KiB)
constexpr int kFitWarps = 4;    // particles per CTA

__device__ __noinline__ int fitness_lane0(const SwarmView& v, int p, int warp,
                                          bool init,
                                          double (*s_buf)[2][kFitChunk],
                                          uint64_t (*s_bar)[2]);

// use_list: 0 = every particle, 1 = the mutation's event list, 2 = init
// (every particle, fit = pfit, no control-block checks: the block is only
// written by k_init_best afterwards)
__global__ void __launch_bounds__(kFitWarps * 32) k_fitness(SwarmView v,
                                                            int use_list) {
  const bool init = use_list == 2;
  if (init) use_list = 0;
  if (!init && v.ctl->done) return;
  if (use_list && !v.ctl->mutating) return;
  __shared__ __align__(16) double s_buf[kFitWarps][2][kFitChunk];
  __shared__ __align__(8) uint64_t s_bar[kFitWarps][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * kFitWarps + warp;
  const int cnt = use_list ? v.ctl->n_events : v.P;
  if (t >= cnt) return;
  int p = t;
  if (use_list) {
    if (v.ev_k[(size_t)v.ctl->mut_cur * v.P + t] < 1) return;
    p = v.ev_slot[t];
  }
  // lane 0 sums; the warp then copies the tour into pbest if it improved
  // (solver.py:217-220), in 16-byte pieces
  int better = 0;
  if (lane == 0) better = fitness_lane0(v, p, warp, init, s_buf, s_bar);
  better = __shfl_sync(0xffffffffu, better, 0);
  if (better) {
    const uint4* src = reinterpret_cast<const uint4*>(v.x + (size_t)p * v.np);
    uint4* dst = reinterpret_cast<uint4*>(v.pbest + (size_t)p * v.np);
    for (int w = lane; w < v.np / 8; w += 32) dst[w] = src[w];
  }
}

__device__ __noinline__ int fitness_lane0(const SwarmView& v, int p, int warp,
                                          bool init,
                                          double (*s_buf)[2][kFitChunk],
                                          uint64_t (*s_bar)[2]) {
  const int n = v.n;
  const double* dg = v.dcache + (size_t)p * v.np;
  uint64_t* bar = s_bar[warp];
  mbar_init(&bar[0], 1);
  mbar_init(&bar[1], 1);
  fence_barrier_init();
  const int nch = (n + kFitChunk - 1) / kFitChunk;  // chunks of d_0..d_{n-1}
  auto issue = [&](int c) {
    const int lo = c * kFitChunk;
    const int len = min(kFitChunk, v.np - lo);  // np: whole 16-B units
    mbar_expect_tx(&bar[c & 1], (uint32_t)len * 8u);
    bulk_g2s(s_buf[warp][c & 1], dg + lo, (uint32_t)len * 8u, &bar[c & 1]);
  };
  issue(0);
  if (nch > 1) issue(1);
  double total = __dadd_rn(0.0, __ldg(dg + n - 1));
  const int m = n - 1;  // d_0 .. d_{n-2}
  for (int c = 0; c < nch; ++c) {
    mbar_wait(&bar[c & 1], (uint32_t)((c >> 1) & 1));
    const double* b = s_buf[warp][c & 1];
    const int lo = c * kFitChunk;
    const int hi = min(m, lo + kFitChunk);
    int i = lo;
    for (; i + 4 <= hi; i += 4) {
      const double2 x0 = *reinterpret_cast<const double2*>(b + (i - lo));
      const double2 x1 = *reinterpret_cast<const double2*>(b + (i - lo) + 2);
      total = __dadd_rn(total, x0.x);
      total = __dadd_rn(total, x0.y);
      total = __dadd_rn(total, x1.x);
      total = __dadd_rn(total, x1.y);
    }
    for (; i < hi; ++i) total = __dadd_rn(total, b[i - lo]);
    if (c + 2 < nch) issue(c + 2);  // the slot just read (generic reads
                                    // completed: their values are summed)
  }
  v.fit[p] = total;
  if (init) {
    v.pfit[p] = total;
    return 0;
  }
  const int better = total < v.pfit[p];
  if (better) v.pfit[p] = total;
  v.pbflag[p] = better;
  return better;
}

}  // namespace

static int ceil_log2(int n) {
  int r = 0;
  while ((1 << r) < n) ++r;
  return r;
}

cudaError_t launch_update(const SwarmView& v, cudaStream_t s) {
  const int grid = v.P;
  if (v.inertia == 1.0) {
    size_t smem = (size_t)16 * v.np;
    const int R = ceil_log2(v.n);
    // ~8 nodes per thread up to 512 threads: small CTAs keep many
    // particles per SM in flight (the work is barrier- and latency-bound)
    int T = 64;
    while (T < 512 && T * 8 < v.n) T <<= 1;
    if (const char* e = getenv("DPSO_UPD_T")) T = atoi(e);
    auto go = [&](auto k, int t) {
      set_dyn_smem((const void*)k, smem);
      k<<<grid, t, smem, s>>>(v, R);
    };
    // 10 B/node only where 16 no longer fits (n > 14000): at C5 (n =
    // 10000) two 10 B/node CTAs per SM measured slower (35 vs 27 ms) than
    // one 16 B/node CTA - the cached target reads and the global vmap fold
    // cost more than the extra occupancy gains.  DPSO_UPD_LOWMEM=1 forces it.
    const bool low = v.n > 14000 || getenv("DPSO_UPD_LOWMEM");
    if (low) {
      smem = (size_t)10 * v.np;
      auto go2 = [&](auto k, int t) {
        set_dyn_smem((const void*)k, smem);
        k<<<grid, t, smem, s>>>(v, R);
      };
      switch (T) {
        case 1024: go2(k_update_w1_lowmem<1024>, 1024); break;
        case 256: go2(k_update_w1_lowmem<256>, 256); break;
        default: go2(k_update_w1_lowmem<512>, 512); break;
      }
      return launch_fitness(v, 0, s);
    }
    switch (T) {
      case 64: go(k_update_w1<64>, 64); break;
      case 128: go(k_update_w1<128>, 128); break;
      case 512: go(k_update_w1<512>, 512); break;
      case 1024: go(k_update_w1<1024>, 1024); break;
      default: go(k_update_w1<256>, 256); break;
    }
  } else if (v.vinv && 20 * (size_t)v.np <= 200 * 1024 &&
             !getenv("DPSO_UPD_SEQ")) {
    const size_t smem = (size_t)20 * v.np;
    const int R = ceil_log2(v.n);
    int T = 64;
    while (T < 512 && T * 8 < v.n) T <<= 1;
    auto go = [&](auto k, int t) {
      set_dyn_smem((const void*)k, smem);
      k<<<grid, t, smem, s>>>(v, R);
    };
    switch (T) {
      case 64: go(k_update_wl<64>, 64); break;
      case 128: go(k_update_wl<128>, 128); break;
      case 512: go(k_update_wl<512>, 512); break;
      default: go(k_update_wl<256>, 256); break;
    }
  } else {
    // the sequential replay (n > ~5000 with w < 1, or DPSO_UPD_SEQ=1)
    size_t smem = (size_t)8 * v.np + (size_t)8 * v.np;
    set_dyn_smem((const void*)k_update_seq, smem);
    k_update_seq<<<grid, 32, smem, s>>>(v);
  }
  return launch_fitness(v, 0, s);
}

cudaError_t launch_fitness(const SwarmView& v, int use_list, cudaStream_t s) {
  // (the pbest copy of an improved particle is fused into k_fitness)
  k_fitness<<<(v.P + kFitWarps - 1) / kFitWarps, kFitWarps * 32, 0, s>>>(
      v, use_list);
  return cudaGetLastError();
}

}  // namespace dpso
