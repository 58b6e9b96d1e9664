// Bounded best-improvement 2-opt scan: the reference's argmin
// (solver.py:88-106) without visiting every pair.
//
// delta(i, j) = ((C[a_i,a_j] + C[s_i,s_j]) - d_i) - d_j over i < j, first
// row-major argmin, applied when < -1e-12.
//
// Bound.  With r(c) = min_{b != c} C[c][b] and q(c) = min_{b != c} C[b][c]
// (off-diagonal row / column minima, once per matrix), every pair has
//     C[a_i,a_j] + C[s_i,s_j] >= (r(a_i) + q(a_j) + r(s_i) + q(s_j)) / 2
//                              >= m_i + m_j,
//     m_k = min((r(a_k) + r(s_k)) / 2, (q(a_k) + q(s_k)) / 2),
// so delta(i, j) >= -(h_i + h_j) with h_k = d_k - m_k (the excess of edge k
// over its end points' cheapest edges).  A pair with h_i + h_j < -T can
// only have delta > T.
//
// Exactness.  Let T be the computed delta of some pair and Tq = min(T,
// -1e-12).  If the reference's minimum m is < -1e-12 then m <= Tq, so every
// pair achieving m has h_i + h_j >= -Tq and is evaluated here with the
// reference expression in fp64: the lexicographic (delta, i, j) minimum
// over the evaluated pairs is the reference's argmin, bit for bit.  If
// m >= -1e-12 the reference makes no move, and neither does the apply (the
// evaluated minimum is >= m).  The h values are rounded up to fp32 and the
// threshold -Tq - slack down (slack = 2^-40 max|C|, far above the fp64
// rounding of h and delta), so every skip is conservative.
//
// Per particle (one CTA of 256 threads, 128 for large swarms): the tour, d
// (dcache) and the cities' minima in shared memory, h over the tour, the
// row of largest h of each 8 threads (32 or 16 seed rows among the longest
// edges) and their pairs give T; then R = {i : h_i + max h >= -Tq} (every
// surviving pair has both rows in R) and its pairs with h_i + h_j >= -Tq
// (none between two rows below -Tq / 2).  The tours the swarm scans are
// far from 2-opt optimal: at C2 |R| is ~50 of 1000 rows and ~200 of the
// 499,500 pairs survive.  A particle with |R| above the list capacity (a
// near-2-opt-optimal tour: the bound is weak) goes to the row-per-lane
// band scan (k_two_opt_band.cu) through a particle list.
#include <float.h>
#include <limits.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "dpso_internal.cuh"

namespace dpso {

namespace {

constexpr int kBoundThreads = 256;  // one CTA per particle (at most)
constexpr int kAppliedTag = -3;     // as k_two_opt.cu: move already applied
constexpr int kSeedRows = 32;       // seed rows (one per 8 threads, at most)
constexpr int kPairCap = 256;       // pair-list entries per warp
constexpr int kMaxPeel = 64;        // rows peeled before the band fallback
constexpr size_t kBoundSmem = 200 * 1024;

struct BoundArgs {
  const double* cost;
  int64_t ld;
  const float2* cmn;  // per city {r(c), q(c)}, rounded down
  int n, np, count, chunks;
  const uint16_t* tours;
  const double* dcache;
  TwoOptRes* res;
  const DevCtl* ctl;
  int32_t* fb;  // [0] count, [1..] particles for the band scan
  unsigned long long* pairs;  // pairs evaluated (cumulative, diagnostic)
  double slack;
  int rmax;     // row-list capacity
  int maxpeel;  // rows peeled before the band fallback
  // the band scan's column records of a fallback particle, written here
  // (k_band_cols' layout: O = es a_c at k = c + 3, D = round(d_c s))
  int32_t* cols;
  int cw, es;
  double scale, vfrom, vto;
  int32_t* runs;  // passes with a fallback (DevCtl::band_runs), nullable
  // the move applied here (the 2-opt apply's work for the particles this
  // kernel resolves; k_two_opt_apply then skips them): tours and dcache
  // are written, fit / pfit / pbest (nullable) and delta_out (nullable)
  int apply, sym;
  uint16_t* tours_rw;
  double* dcache_rw;
  double* fit;
  double* pfit;
  uint16_t* pbest;
  double* delta_out;
  uint32_t off_d, off_h, off_c, off_pos, off_lh, off_pairs;  // shared
};

__device__ __forceinline__ bool lex_less(double d1, int i1, int j1, double d2,
                                         int i2, int j2) {
  if (d1 < d2) return true;
  if (d2 < d1) return false;
  return (i1 < i2) || (i1 == i2 && j1 < j2);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Evaluate a warp's pair list: tour-position pairs x | y << 16, with the
// reference expression in fp64, folded into the lane's (delta, i, j)
// minimum; U pairs per lane in flight (2 U independent gathers).
template <int U>
__device__ __forceinline__ void eval_list(const BoundArgs& a, int np,
                                          const uint32_t* pr,
                                          const uint16_t* tr,
                                          const double* dd, int lane,
                                          double& bd, int& bi, int& bj,
                                          int& evals) {
  evals += np;  // warp-uniform: counted once per warp (lane 0)
  for (int q0 = 0; q0 < np; q0 += 32 * U) {
    double A[U], B[U], di[U], dj[U];
    int I[U], J[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int q = q0 + 32 * k + lane;
      I[k] = -1;
      if (q < np) {
        const uint32_t uv = pr[q];
        const int pu = (int)(uv & 0xffffu), pv = (int)(uv >> 16);
        const int i = min(pu, pv), j = max(pu, pv);
        I[k] = i;
        J[k] = j;
        di[k] = dd[i];
        dj[k] = dd[j];
        A[k] = ld_cost(a.cost + (size_t)tr[i] * a.ld + tr[j]);
        B[k] = ld_cost(a.cost + (size_t)tr[i + 1] * a.ld + tr[j + 1]);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (I[k] < 0) continue;
      double t = __dadd_rn(A[k], B[k]);
      t = __dsub_rn(t, di[k]);
      t = __dsub_rn(t, dj[k]);
      if (lex_less(t, I[k], J[k], bd, bi, bj)) {
        bd = t;
        bi = I[k];
        bj = J[k];
      }
    }
  }
}

// Warp-wide minimum of d (every lane gets it).
__device__ __forceinline__ double warp_dmin(double d) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    d = fmin(d, __shfl_xor_sync(0xffffffffu, d, o));
  return d;
}

// CTA-wide minimum of d (every thread gets it): the seed threshold needs
// the value only.
__device__ __forceinline__ double cta_dmin(double d, double* rd, int lane,
                                           int warp, int nw) {
  d = warp_dmin(d);
  if (lane == 0) rd[warp] = d;
  __syncthreads();
  d = rd[0];
  for (int w = 1; w < nw; ++w) d = fmin(d, rd[w]);
  __syncthreads();
  return d;
}

// Warp-wide lexicographic (delta, i, j) minimum: the minimum delta, then
// the smallest (i, j) among the lanes holding it (i, j < 2^16), in lane 0.
__device__ __forceinline__ void warp_lexmin_fast(double& d, int& i, int& j) {
  const double m = warp_dmin(d);
  const unsigned key =
      d == m ? ((unsigned)i << 16) | (unsigned)j : 0xFFFFFFFFu;
  const unsigned k = __reduce_min_sync(0xffffffffu, key);
  d = m;
  i = k == 0xFFFFFFFFu ? INT_MAX : (int)(k >> 16);
  j = k == 0xFFFFFFFFu ? INT_MAX : (int)(k & 0xFFFFu);
}

// CTA-wide lexicographic minimum, in thread 0.
__device__ __forceinline__ void cta_lexmin(double& d, int& i, int& j,
                                           double* rd, int* ri, int* rj,
                                           int lane, int warp, int nw) {
  warp_lexmin_fast(d, i, j);
  if (lane == 0) {
    rd[warp] = d;
    ri[warp] = i;
    rj[warp] = j;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int w = 1; w < nw; ++w)
      if (lex_less(rd[w], ri[w], rj[w], d, i, j)) {
        d = rd[w];
        i = ri[w];
        j = rj[w];
      }
}

template <int NT, int SPW>
__global__ void __launch_bounds__(NT, 1024 / NT) k_two_opt_bound(BoundArgs a) {
  if (a.ctl && (a.ctl->done || a.ctl->improved)) return;  // no scan
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double s_rd[NT / 32];
  __shared__ int s_ri[NT / 32], s_rj[NT / 32];
  __shared__ float s_hmax[NT / 32];
  __shared__ int s_cnt[2];
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p = blockIdx.x;
  if (p >= a.count) return;
  const int n = a.n;
  const unsigned below = lanemask_lt();
  uint16_t* tr = reinterpret_cast<uint16_t*>(smem);  // tour, tr[n] = tr[0]
  const double* dd = a.dcache + (size_t)p * a.np;  // d in fp64 (cached)
  float* hv = reinterpret_cast<float*>(smem + a.off_h);
  float2* cm = reinterpret_cast<float2*>(smem + a.off_c);  // minima of a_i
  int* lpos = reinterpret_cast<int*>(smem + a.off_pos);
  float* lh = reinterpret_cast<float*>(smem + a.off_lh);
  uint32_t* pr = reinterpret_cast<uint32_t*>(smem + a.off_pairs) +
                 warp * kPairCap;
  const uint16_t* tour = a.tours + (size_t)p * a.np;
  const double* dg = dd;

  // ---- the tour, its edge costs (rounded up) and its cities' minima in
  // shared memory
  for (int i0 = 0; i0 < n; i0 += 4 * NT) {
    int t[4];
    double d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + k * NT + tid;
      if (i < n) {
        t[k] = tour[i];
        d[k] = dg[i];
      }
    }
    float2 c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i0 + k * NT + tid < n) c[k] = a.cmn[t[k]];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + k * NT + tid;
      if (i < n) {
        tr[i] = (uint16_t)t[k];
        hv[i] = __double2float_ru(d[k]);  // d rounded up; h below
        cm[i] = c[k];
      }
    }
  }
  if (tid == 0) {
    tr[n] = tr[0] = tour[0];
    s_cnt[0] = s_cnt[1] = 0;
  }
  __syncthreads();
  if (tid == 0) cm[n] = cm[0];
  __syncthreads();

  // ---- h_i >= d_i - m_i, in fp32 with every rounding upward (the minima
  // are rounded down); the thread's largest
  float lmax = -FLT_MAX;
  int larg = -1;
  for (int i = tid; i < n; i += NT) {
    const float2 ca = cm[i], cs = cm[i + 1];
    const float f = __fmul_rd(0.5f, __fadd_rd(ca.x, cs.x));
    const float g = __fmul_rd(0.5f, __fadd_rd(ca.y, cs.y));
    const float h = __fsub_ru(hv[i], fminf(f, g));
    hv[i] = h;
    if (larg < 0 || h > lmax) {
      lmax = h;
      larg = i;
    }
  }
  // seed rows: the largest h of each group of 32 / SPW threads (NT / 8 seeds among
  // the longest edges; any rows give a valid threshold, long edges a tight
  // one), and the maximum over the tour
  constexpr int GL = 32 / SPW;  // lanes per seed group
#pragma unroll
  for (int o = 1; o < GL; o <<= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, lmax, o);
    const int a2 = __shfl_xor_sync(0xffffffffu, larg, o);
    if (a2 >= 0 && (larg < 0 || m2 > lmax)) {
      lmax = m2;
      larg = a2;
    }
  }
  float hm = lmax;
#pragma unroll
  for (int o = GL; o < 32; o <<= 1)
    hm = fmaxf(hm, __shfl_xor_sync(0xffffffffu, hm, o));
  if (lane == 0) s_hmax[warp] = hm;
  __syncthreads();  // the minima (aliased by the row list) are dead now
  if (lane % GL == 0) lpos[warp * SPW + lane / GL] = larg;
  __syncthreads();
  float hmax = s_hmax[0];
  for (int w = 1; w < NW; ++w) hmax = fmaxf(hmax, s_hmax[w]);

  // ---- the seed rows' pairs (496 for 32 seeds)
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  double bd = kInf;
  int bi = INT_MAX, bj = INT_MAX;
  int sv = 0;  // seed pairs this thread evaluated
  {
    constexpr int S = SPW * NW;
    constexpr int NP = S * (S - 1) / 2;
    constexpr int KQ = (NP + NT - 1) / NT;
    double A[KQ], B[KQ], di[KQ], dj[KQ];
    int I[KQ], J[KQ];
#pragma unroll
    for (int k = 0; k < KQ; ++k) {
      const int q = tid + k * NT;
      I[k] = -1;
      if (q < NP) {
        // q -> (u, v), u < v: v (v - 1) / 2 <= q < v (v + 1) / 2
        int v = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)q)) * 0.5f);
        while (v * (v - 1) / 2 > q) --v;
        while ((v + 1) * v / 2 <= q) ++v;
        const int u = q - v * (v - 1) / 2;
        const int pu = lpos[u], pv = lpos[v];
        if (pu >= 0 && pv >= 0) {
          const int i = min(pu, pv), j = max(pu, pv);
          I[k] = i;
          J[k] = j;
          di[k] = dd[i];
          dj[k] = dd[j];
          A[k] = ld_cost(a.cost + (size_t)tr[i] * a.ld + tr[j]);
          B[k] = ld_cost(a.cost + (size_t)tr[i + 1] * a.ld + tr[j + 1]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < KQ; ++k) {
      if (I[k] < 0) continue;
      ++sv;
      double t = __dadd_rn(A[k], B[k]);
      t = __dsub_rn(t, di[k]);
      t = __dsub_rn(t, dj[k]);
      if (lex_less(t, I[k], J[k], bd, bi, bj)) {
        bd = t;
        bi = I[k];
        bj = J[k];
      }
    }
  }
  const double t0 = cta_dmin(bd, s_rd, lane, warp, NW);
  const double tq = fmin(t0, -1e-12);
  // skip a pair iff h_i + h_j < thr <= -tq - slack (exactly: the fp32
  // tests round up)
  const float thr = __double2float_rd(__dsub_rd(-tq, a.slack));
  // two rows below half the threshold cannot make a pair
  const float half = __fmul_rd(0.5f, thr);

  int np = 0, evals = (int)__reduce_add_sync(0xffffffffu, (unsigned)sv);
  // append position pairs to the warp's list (flushed when full)
  auto push = [&](bool take, int x, int y) {
    const unsigned bt = __ballot_sync(0xffffffffu, take);
    if (np + __popc(bt) > kPairCap) {
      __syncwarp();
      eval_list<2>(a, np, pr, tr, dd, lane, bd, bi, bj, evals);
      __syncwarp();
      np = 0;
    }
    if (take) pr[np + __popc(bt & below)] = (uint32_t)x | ((uint32_t)y << 16);
    np += __popc(bt);
  };
  // R(hc) = {i : h_i + hc >= thr}, hc the largest h left: both rows of
  // every remaining surviving pair.  Compacted as H (h >= half, from the
  // front of the list) and L (h < half, from the back); returns |R|.
  auto compact = [&](float hc) -> int {
    for (int i0 = 0; i0 < n; i0 += NT) {
      const int i = i0 + tid;
      const float h = i < n ? hv[i] : -FLT_MAX;
      const bool take = i < n && __fadd_ru(h, hc) >= thr;
      const bool hi = take && h >= half;
      const unsigned bh = __ballot_sync(0xffffffffu, hi);
      const unsigned bl = __ballot_sync(0xffffffffu, take && !hi);
      int baseh = 0, basel = 0;
      if (lane == 0) {
        if (bh) baseh = atomicAdd(&s_cnt[0], __popc(bh));
        if (bl) basel = atomicAdd(&s_cnt[1], __popc(bl));
      }
      baseh = __shfl_sync(0xffffffffu, baseh, 0);
      basel = __shfl_sync(0xffffffffu, basel, 0);
      if (hi) {
        const int slot = baseh + __popc(bh & below);
        if (slot < a.rmax) {
          lpos[slot] = i;
          lh[slot] = h;
        }
      } else if (take) {
        const int slot = a.rmax - 1 - (basel + __popc(bl & below));
        if (slot >= 0) {
          lpos[slot] = i;
          lh[slot] = h;
        }
      }
    }
    __syncthreads();
    const int r = s_cnt[0] + s_cnt[1];
    return r;
  };
  float hc = hmax;
  int cnt = compact(hc);
  // ---- peeling: while R is too large for the list, the row of largest h
  // is paired with every row it reaches and taken out (h = -FLT_MAX): hc
  // drops and R shrinks
  for (int peel = 0; cnt > a.rmax; ++peel) {
    // the first row of largest h
    int am = INT_MAX;
    float mv = -FLT_MAX;
    for (int i = tid; i < n; i += NT) {
      const float h = hv[i];
      if (h > mv) {  // ascending i per thread: the first of equal maxima
        mv = h;
        am = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, mv, o);
      const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
      if (m2 > mv || (m2 == mv && a2 < am)) {
        mv = m2;
        am = a2;
      }
    }
    if (lane == 0) {
      s_rj[warp] = am;
      s_hmax[warp] = mv;
    }
    __syncthreads();
    int m = INT_MAX;
    float hmv = -FLT_MAX;
    for (int w = 0; w < NW; ++w)
      if (s_hmax[w] > hmv || (s_hmax[w] == hmv && s_rj[w] < m)) {
        hmv = s_hmax[w];
        m = s_rj[w];
      }
    __syncthreads();
    if (peel >= a.maxpeel || m == INT_MAX || !(hmv > -FLT_MAX)) {
      // weak bound everywhere (a nearly 2-opt-optimal tour): the band
      // scan takes the particle; its column records from here
      int32_t* O = a.cols + (size_t)p * 2 * a.cw;
      int32_t* D = O + a.cw;
      for (int k = tid; k < a.cw; k += NT) {
        const int kk = k - 3;
        O[k] = (kk >= 0 && kk <= n) ? a.es * (int)tr[kk] : 0;  // tr[n] = a_0
        if (k < n) {
          double d = dd[k];
          if (a.vfrom > 0.0 && d == a.vfrom) d = a.vto;
          D[k] = __double2int_rn(d * a.scale);
        } else {
          D[k] = -0x40000000;
        }
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        const int at = atomicAdd(&a.fb[0], 1);
        a.fb[1 + at] = p;
        if (at == 0 && a.runs) atomicAdd(a.runs, 1);
      }
      return;
    }
    // row m against every row it reaches
    for (int i0 = 0; i0 < n; i0 += NT) {
      const int i = i0 + tid;
      const bool take = i < n && i != m && __fadd_ru(hmv, hv[i]) >= thr;
      push(take, m, i);
    }
    __syncthreads();
    if (tid == 0) {
      hv[m] = -FLT_MAX;
      s_cnt[0] = s_cnt[1] = 0;
    }
    __syncthreads();
    // the largest h left
    hc = -FLT_MAX;
    for (int i = tid; i < n; i += NT) hc = fmaxf(hc, hv[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      hc = fmaxf(hc, __shfl_xor_sync(0xffffffffu, hc, o));
    if (lane == 0) s_hmax[warp] = hc;
    __syncthreads();
    for (int w = 0; w < NW; ++w) hc = fmaxf(hc, s_hmax[w]);
    cnt = compact(hc);
  }
  // ---- R's pairs: H x H and H x L with h_u + h_v >= thr (two rows of L
  // sum below thr), warp-compacted, evaluated
  const int nh = s_cnt[0], nl = s_cnt[1];
  const int l0 = a.rmax - nl;  // L occupies [l0, rmax)
  for (int u = warp; u < nh; u += NW) {
    const float hu = lh[u];
    const int pu = lpos[u];
    for (int v0 = u + 1; v0 < nh; v0 += 32) {
      const int v = v0 + lane;
      const bool take = v < nh && __fadd_ru(hu, lh[v]) >= thr;
      push(take, pu, take ? lpos[v] : 0);
    }
    for (int v0 = l0; v0 < a.rmax; v0 += 32) {
      const int v = v0 + lane;
      const bool take = v < a.rmax && __fadd_ru(hu, lh[v]) >= thr;
      push(take, pu, take ? lpos[v] : 0);
    }
  }
  __syncwarp();
  eval_list<2>(a, np, pr, tr, dd, lane, bd, bi, bj, evals);
  if (lane == 0 && evals) atomicAdd(a.pairs, (unsigned long long)evals);
  cta_lexmin(bd, bi, bj, s_rd, s_ri, s_rj, lane, warp, NW);
  TwoOptRes* out = a.res + (size_t)p * a.chunks;
  if (!a.apply) {
    for (int c = tid; c < a.chunks; c += NT)
      out[c] = c == 0 ? TwoOptRes{bd, bi, bj}
                      : TwoOptRes{kInf, INT_MAX, INT_MAX};
    return;
  }
  // ---- the apply (k_two_opt_apply's steps, solver.py:101-104, 309-316):
  // reverse a[i+1 .. j] when delta < -1e-12, refresh the edge costs,
  // fitness += delta, pbest; the apply kernel skips this particle
  __shared__ int s_mv[3];
  __shared__ double s_dl;
  __shared__ int s_bt;
  if (tid == 0) {
    const int move = bd < -1e-12;  // n >= 4 here
    s_mv[0] = move;
    s_mv[1] = bi;
    s_mv[2] = bj;
    s_dl = move ? bd : 0.0;
    if (a.delta_out) a.delta_out[p] = s_dl;
    out[0] = TwoOptRes{kInf, kAppliedTag, kAppliedTag};
  }
  __syncthreads();
  if (!s_mv[0]) return;
  const int i = s_mv[1], j = s_mv[2], len = j - i;
  uint16_t* t = a.tours_rw + (size_t)p * a.np;
  double* dgw = a.dcache_rw + (size_t)p * a.np;
  // the new tour from the shared copy: positions i+1 .. j reversed
  for (int u = i + 1 + tid; u <= j; u += NT) t[u] = tr[i + j + 1 - u];
  if (a.sym) {
    // symmetric matrix: edge k in (i, j) of the new tour is old edge
    // i + j - k reversed (same cost bits); edges i and j are new
    const int m = len - 1;
    for (int u = tid; u < m / 2; u += NT) {
      const double y = dgw[i + 1 + u];
      dgw[i + 1 + u] = dgw[j - 1 - u];
      dgw[j - 1 - u] = y;
    }
    if (tid < 2) {
      const int k = tid == 0 ? i : j;
      const int x = tid == 0 ? tr[i] : tr[i + 1];
      const int y = tid == 0 ? tr[j] : tr[j + 1];  // tr[n] = a_0
      dgw[k] = ld_cost(a.cost + (size_t)x * a.ld + y);
    }
  } else {
    for (int k = i + tid; k <= j; k += NT) {
      // new edge k: (new a_k, new a_{k+1}) from the shared old tour
      const int x = k == i ? tr[i] : tr[i + j + 1 - k];
      const int y = k == j ? tr[j + 1] : tr[i + j - k];
      dgw[k] = ld_cost(a.cost + (size_t)x * a.ld + y);
    }
  }
  if (a.fit) {
    if (tid == 0) {
      const double f = __dadd_rn(a.fit[p], s_dl);
      a.fit[p] = f;
      s_bt = f < a.pfit[p];
      if (s_bt) a.pfit[p] = f;
    }
    __syncthreads();
    if (s_bt) {
      uint16_t* pb = a.pbest + (size_t)p * a.np;
      for (int u = tid; u < n; u += NT)
        pb[u] = (u > i && u <= j) ? tr[i + j + 1 - u] : tr[u];
    }
  }
}

// Off-diagonal row and column minima {r(c), q(c)}, rounded down to fp32
// (lower bounds stay lower bounds), one warp per city.
__global__ void k_bound_minima(const double* cost, int64_t ld, int n,
                               float2* out) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= n) return;
  double r = __longlong_as_double(0x7ff0000000000000ll), q = r;
  for (int b = lane; b < n; b += 32) {
    if (b == c) continue;
    r = fmin(r, cost[(size_t)c * ld + b]);
    q = fmin(q, cost[(size_t)b * ld + c]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r = fmin(r, __shfl_xor_sync(0xffffffffu, r, o));
    q = fmin(q, __shfl_xor_sync(0xffffffffu, q, o));
  }
  if (lane == 0)
    out[c] = make_float2(__double2float_rd(r), __double2float_rd(q));
}

struct BoundLayout {
  uint32_t off_d, off_h, off_c, off_pos, off_lh, off_pairs, bytes;
};

// dynamic shared memory of one CTA: tour (u16, n + 1), h (f32, n), then
// the cities' minima (f32 x 2, n + 1; the h pass only) aliased with the row
// list (positions, h; rmax each) and the warps' pair lists
BoundLayout bound_layout(int n, int rmax, int nt) {
  BoundLayout L;
  int64_t o = round_up(2 * (int64_t)(n + 1), 16);
  L.off_h = (uint32_t)o;
  o = round_up(o + 4 * (int64_t)n, 16);
  const int64_t u0 = o;
  L.off_c = (uint32_t)o;
  const int64_t cend = o + 8 * (int64_t)(n + 1);
  L.off_pos = (uint32_t)o;
  o = round_up(o + 4 * (int64_t)std::max(rmax, kSeedRows), 16);
  L.off_lh = (uint32_t)o;
  o = round_up(o + 4 * (int64_t)rmax, 16);
  L.off_pairs = (uint32_t)o;
  o += 4 * (int64_t)kPairCap * (nt / 32);
  (void)u0;
  L.off_d = 0;
  L.bytes = (uint32_t)round_up(std::max(o, cend), 128);
  return L;
}

int bound_rmax() {
  if (const char* e = getenv("DPSO_BOUND_RMAX")) {
    const int v = atoi(e);
    return v < kSeedRows ? kSeedRows : v;
  }
  return 256;
}

}  // namespace

int64_t bound_bytes(int n, int64_t count) {
  if (n < 4 || n > kBoundMaxN) return 0;
  return round_up(16 * (int64_t)n, 256) + 16 + 4 * (count + 2);
}

cudaError_t bound_prepare(const double* cost, int64_t ld, int32_t n,
                          void* buf, double maxabs, cudaStream_t s,
                          TwoOptPlan* pl) {
  pl->bound = 0;
  if (!buf || n < 4 || n > kBoundMaxN || !pl->band_mode) return cudaSuccess;
  if (const char* e = getenv("DPSO_BOUND"))
    if (atoi(e) == 0) return cudaSuccess;
  // finite matrices of moderate magnitude only (h and the threshold stay
  // finite); others keep the full scan
  if (!(maxabs < 1e300)) return cudaSuccess;
  const BoundLayout L = bound_layout(n, bound_rmax(), kBoundThreads);
  if (L.bytes > kBoundSmem) return cudaSuccess;
  float2* cmn = reinterpret_cast<float2*>(buf);
  k_bound_minima<<<(n + 7) / 8, 256, 0, s>>>(cost, ld, n, cmn);
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  pl->bound = 1;
  pl->bound_cmn = cmn;
  unsigned char* st =
      reinterpret_cast<unsigned char*>(buf) + round_up(16 * (int64_t)n, 256);
  pl->bound_pairs = reinterpret_cast<unsigned long long*>(st);
  pl->bound_fb = reinterpret_cast<int32_t*>(st + 16);
  e = cudaMemsetAsync(st, 0, 16, s);
  if (e) return e;
  pl->bound_slack = ldexp(maxabs, -40);
  return cudaSuccess;
}

cudaError_t launch_two_opt_bound(const TwoOptPlan& pl, int32_t n, int32_t np,
                                 const uint16_t* tours, const double* dcache,
                                 int32_t count, TwoOptRes* res, int32_t chunks,
                                 const DevCtl* ctl, cudaStream_t s,
                                 int32_t* runs, const BoundApply* ap) {
  BoundArgs a;
  memset(&a, 0, sizeof a);
  a.cost = pl.cost;
  a.ld = pl.ld;
  a.cmn = pl.bound_cmn;
  a.n = n;
  a.np = np;
  a.count = count;
  a.chunks = chunks;
  a.tours = tours;
  a.dcache = dcache;
  a.res = res;
  a.ctl = ctl;
  a.fb = pl.bound_fb;
  a.pairs = pl.bound_pairs;
  a.slack = pl.bound_slack;
  a.rmax = bound_rmax();
  a.maxpeel = kMaxPeel;
  a.cols = pl.band_cols;
  a.cw = band_cw(n);
  a.es = pl.band_es;
  a.scale = pl.band_scale;
  a.vfrom = pl.band_vfrom;
  a.vto = pl.band_vto;
  a.runs = runs;
  if (ap) {
    a.apply = 1;
    a.sym = pl.symmetric;
    a.tours_rw = ap->tours;
    a.dcache_rw = ap->dcache;
    a.fit = ap->fit;
    a.pfit = ap->pfit;
    a.pbest = ap->pbest;
    a.delta_out = ap->delta_out;
  }
  if (const char* e = getenv("DPSO_BOUND_PEEL")) a.maxpeel = atoi(e);
  // small swarms: 256 threads per particle (shorter per-particle latency
  // chains; 128 and 512 measured slower at C2: 0.066 / 0.055 vs 0.050 ms);
  // large swarms: 128 (more particles per SM, fewer seed pairs)
  bool wide = count < 148 * 16;
  constexpr int SPW_W = 4;  // seed rows per warp (2 measured slower at C2)
  if (const char* e = getenv("DPSO_BOUND_NT")) wide = atoi(e) == 256;
  const BoundLayout L = bound_layout(n, a.rmax, wide ? 256 : 128);
  a.off_d = L.off_d;
  a.off_h = L.off_h;
  a.off_c = L.off_c;
  a.off_pos = L.off_pos;
  a.off_lh = L.off_lh;
  a.off_pairs = L.off_pairs;
  const size_t smem = L.bytes;
  cudaError_t e = cudaMemsetAsync(a.fb, 0, 4, s);
  if (e) return e;
  const void* kern = wide ? (const void*)k_two_opt_bound<256, SPW_W>
                          : (const void*)k_two_opt_bound<128, 4>;
  e = set_dyn_smem(kern, smem);
  if (e) return e;
  if (count > 0) {
    if (wide)
      k_two_opt_bound<256, SPW_W><<<count, 256, smem, s>>>(a);
    else
      k_two_opt_bound<128, 4><<<count, 128, smem, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace dpso
