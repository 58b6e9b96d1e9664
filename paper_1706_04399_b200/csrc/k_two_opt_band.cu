// Best-improvement 2-opt scan, row-per-lane band formulation
// (solver.py:88-106: delta(i,j) = ((C[a_i,a_j] + C[s_i,s_j]) - d_i) - d_j
// over i < j, first row-major argmin, applied when < -1e-12).
//
// Write M[x][y] = C[a_x][a_y] (the tour-permuted matrix).  Then
// delta(i, j) = M[i][j] + M[i+1][j+1] - d_i - d_j: a pair needs two entries
// on one diagonal of M.
//
// One CTA owns a particle at a time and walks its pair rows in bands of 31.
// The 32 cost rows a_i0 .. a_i0+31 of a band are staged in shared memory
// (slot l = row a_{i0+l}) by 32 bulk copies.  Lane l of every warp owns pair
// row i = i0 + l.  The warps of the CTA split the band's columns; a warp
// sweeps its columns c in order, and at step c every lane gathers from its
// own slot at the SAME offset a_c:
//     G_l(c) = M[i0+l][c]        (one LDS per lane per step)
// The pair (i0+l, c-1) is G_l(c-1) + G_{l+1}(c) - d_i - d_{c-1}: its first
// term is the lane's previous gather, its second the same gather from slot
// l+1 - a second LDS at the lane's address plus the slot stride, which
// ptxas folds into [R + UR] addressing.  So each pair costs two
// conflict-free shared-memory loads, one IADD for the address, one IADD3
// and one min (DPSO_BAND_NBLDS=0: a shuffle from lane l+1 instead).
//
// Bank-conflict freedom: slot l's element a sits at byte l*(S+4) + 2a of the
// stage (S a multiple of 128), i.e. in bank (l + a/2) mod 32 - a different
// bank for every lane, whatever a is.  Bulk copies need 16-byte aligned
// destinations, so the 4-byte rotation comes from the source: the int16 row
// copy is kept in four versions in HBM/L2, version q shifted by 4q bytes,
// and slot l copies version l mod 4 to l*S + 16*(l div 4).
//
// Arithmetic is integer: rows are int16 round(C * s) (s a power of two),
// d values round(d * s).
//   EXACT   integer matrix, max|C| <= 32767, s = 1: every delta is exact;
//           each lane keeps its first minimum in (t, i, j) order, the
//           warp-wide threshold is lexicographic, so the result is the
//           reference's argmin bit for bit.
//   FILTER  otherwise: |t - delta*s| <= 2 (four roundings of <= 1/2), so the
//           reference's fp64 argmin and all its fp64 ties lie within 4 of
//           the integer minimum (the fp64 rounding of delta is < 2^-30 in
//           these units).  Each lane keeps the pairs within t_min + 4 as
//           candidates (<= 4 per lane); at the end of a particle the
//           candidates are re-evaluated with the reference expression in
//           fp64, the structural pairs (i, i+1) exactly from d.  A lane whose
//           list overflows sends the particle to the fp64 re-scan.
// The structural pairs (i, i+1) are arithmetic no-ops (exactly 0 in EXACT)
// and are not scanned; (0, n-1) is scanned (it is not a no-op for
// asymmetric matrices).
//
// Two rows per lane (RPL = 2, wherever two 64-slot stages fit: n up to
// ~600): 64-slot bands of 63 pair rows, lane l owning rows i0 + l and
// i0 + 32 + l; one address and one set of column records per column serve
// both rows (the second row's loads at uniform offsets 32 (S + 4) and
// 33 (S + 4)), each row set with its own lane state.
//
// Pipeline: persistent CTAs (one per SM), particles blockIdx.x + k*grid;
// a ring of 2-4 band stages filled by producer warps (bulk copies, full /
// empty mbarriers), consumed by consumer warps at their own pace (no CTA
// barrier per band; with 4 stages two warp groups take alternate bands); a
// CTA-wide running minimum caps every warp's hit threshold; the particle's
// column records (offsets 2*a_c and d values, k_band_cols) arrive on their
// own barrier; the last warp done with a particle reduces its result.
#include <float.h>
#include <limits.h>
#include <stdlib.h>
#include <string.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "dpso_internal.cuh"
#include "tma.cuh"

#ifndef DPSO_BAND_NBLDS
#define DPSO_BAND_NBLDS 1
#endif

namespace dpso {

namespace {

constexpr int kBandRows = 31;      // pair rows per band (lanes 0..30)
constexpr int kBandCand = 4;       // FILTER candidates per lane
constexpr int kBig = 0x40000000;   // dead column (D) / no candidate
constexpr int kNone = 0x20000000;  // no pair seen yet
constexpr int kBandWarps = 16;   // consumer warps
constexpr int kMaxStages = 4;
constexpr int kOvfTag = -2;        // as k_two_opt.cu's kOverflowTag
constexpr int kLaneState = 3 + 2 * kBandCand;  // ints per lane

struct BandArgs {
  const double* cost;   // fp64 matrix (FILTER re-evaluation)
  int64_t ld;
  const unsigned char* rows;  // 4 rotated int16 versions (band_rows_bytes)
  int line;             // bytes per row line
  uint32_t slot;        // S: bytes between slots of a stage
  int n, np, count, chunks;
  const uint16_t* tours;
  const double* dcache;
  TwoOptRes* res;
  const DevCtl* ctl;
  int32_t* ovf;         // [0] count, [1..] tasks for the fp64 re-scan
  double scale, vfrom, vto;
  int win;              // FILTER window (integer units)
  int cw;               // ints per column array
  const int32_t* cols;  // count x [O | D] (k_band_cols)
  int nst;              // stages in the row ring
  int ncb;              // column buffers / result slots (particles)
  int groups;           // warp groups scanning alternate bands (1 or 2)
  int probe;            // debug: 1 = stream the bands, skip the pairs;
                        // 2 = scan, but copy rows only into the first nst
                        // bands (later bands reuse them: consumer floor)
  int g4;               // rows staged by TMA gather4 (4 rows per copy)
  // particle list (the bounded scan's fallbacks): particles plist[0 ..
  // *pcnt - 1] instead of 0 .. count - 1; null = all
  const int32_t* plist;
  const int32_t* pcnt;
};

__device__ __forceinline__ int lds_s16(uint32_t addr) {
  int v;
  asm volatile("ld.shared.s16 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// a row element: int16 (ES = 2) or int8 (ES = 1, the rows of n > ~1400)
template <int ES>
__device__ __forceinline__ int lds_el(uint32_t addr) {
  if (ES == 2) return lds_s16(addr);
  int v;
  asm volatile("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ bool lex_lt(double d1, int i1, int j1, double d2,
                                       int i2, int j2) {
  if (d1 < d2) return true;
  if (d2 < d1) return false;
  return (i1 < i2) || (i1 == i2 && j1 < j2);
}

__device__ __forceinline__ void warp_lexmin(double& d, int& i, int& j) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double d2 = __shfl_xor_sync(0xffffffffu, d, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    const int j2 = __shfl_xor_sync(0xffffffffu, j, o);
    if (lex_lt(d2, i2, j2, d, i, j)) {
      d = d2;
      i = i2;
      j = j2;
    }
  }
}

// Threshold of a lane for its row i: a later pair (t, i, j) hits when
// t - D_i <= L - D_i.
//   EXACT: beats the warp best (wb, wi) lexicographically: t < wb, or
//          t == wb for a row above the best's (i < wi).
//   FILTER: within the window lim = t_min + win.
template <int MODE>
__device__ __forceinline__ int lane_limit(bool live, int Di, int i, int w0,
                                          int w1) {
  if (!live) return INT_MIN;
  if (MODE == 1) return w0 + Di - (i >= w1 ? 1 : 0);
  return w0 + Di;
}

// Entered by the whole warp (the pre-test is warp-uniform); updates the
// lane state (st: stride 32) and the warp state ws[0..1], returns the lane's
// new limit.
template <int MODE>
__device__ __noinline__ int band_hit(int u0, int u1, int u2, int u3, int u4,
                                     int u5, int u6, int u7, int c0, int i,
                                     int Di, int L, int live, int win,
                                     int* st, int* ws, int* cmin) {
  const int uv[8] = {u0, u1, u2, u3, u4, u5, u6, u7};
  const int lane = threadIdx.x & 31;
  if (MODE == 1) {
    int bt = st[0], bi = st[32], bj = st[64];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      // the lane's own pairs arrive in (i, j) order: its first minimum
      const int t = uv[g] - Di;
      if (live && t < bt) {
        bt = t;
        bi = i;
        bj = c0 + g;
      }
    }
    st[0] = bt;
    st[32] = bi;
    st[64] = bj;
    int wt = bt, wi = bi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int t2 = __shfl_xor_sync(0xffffffffu, wt, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, wi, o);
      if (t2 < wt || (t2 == wt && i2 < wi)) {
        wt = t2;
        wi = i2;
      }
    }
    {  // with the warp's best so far (two rows per lane: the other set's)
      const int ow = ws[0], oi = ws[1];
      if (ow < wt || (ow == wt && oi < wi)) {
        wt = ow;
        wi = oi;
      }
      __syncwarp();
    }
    // the CTA-wide minimum t over all warps of this particle: a pair above
    // it cannot be the argmin, so it caps every lane's limit (ties at it
    // still hit; the final reduction breaks them)
    int ct = wt;
    if (lane == 0) {
      ws[0] = wt;
      ws[1] = wi;
      ct = min(atomicMin(cmin, wt), wt);
    }
    ct = __shfl_sync(0xffffffffu, ct, 0);
    return min(lane_limit<1>(live, Di, i, wt, wi),
               live ? ct + Di : INT_MIN);
  }
  int lb = st[0], nc = st[32], of = st[64];
  int* cd = st + 96;
  int* cij = cd + 32 * kBandCand;
  int tv[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    tv[g] = (live && uv[g] <= L) ? uv[g] - Di : kBig;
    lb = min(lb, tv[g]);
  }
  int wm = lb;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    wm = min(wm, __shfl_xor_sync(0xffffffffu, wm, o));
  // the window around the CTA-wide minimum over all warps of the particle
  int cm = wm;
  if (lane == 0) cm = min(atomicMin(cmin, wm), wm);
  cm = __shfl_sync(0xffffffffu, cm, 0);
  const int lim = cm + win;
  int w = 0;
  for (int k = 0; k < nc; ++k) {
    const int dv = cd[32 * k];
    if (dv <= lim) {
      cd[32 * w] = dv;
      cij[32 * w] = cij[32 * k];
      ++w;
    }
  }
  nc = w;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    if (tv[g] <= lim) {
      if (nc < kBandCand) {
        cd[32 * nc] = tv[g];
        cij[32 * nc] = (i << 16) | (c0 + g);
        ++nc;
      } else {
        of = 1;
      }
    }
  }
  st[0] = lb;
  st[32] = nc;
  st[64] = of;
  if (lane == 0) ws[0] = lim;
  return lane_limit<2>(live, Di, i, lim, 0);
}

// Column arrays of every particle, precomputed for the scan (one CTA per
// particle): O[3 + k] = 2 a_k for k in [0, n] (a_n = a_0, byte offsets of
// the gathers), zero elsewhere; D[c] = round(d_c s) for c < n, -kBig past
// the end (dead columns).  The scan moves them to shared memory with one
// bulk copy per particle.
__global__ void k_band_cols(const uint16_t* tours, int np,
                            const double* dcache, int n, int cw, int count,
                            double scale, double vfrom, double vto,
                            int32_t* out, const DevCtl* ctl, int es,
                            const int32_t* plist, const int32_t* pcnt,
                            int32_t* runs) {
  if (ctl && (ctl->done || ctl->improved)) return;  // no scan this time
  const int q = blockIdx.x;
  const int cnt = pcnt ? *pcnt : count;
  if (runs && q == 0 && threadIdx.x == 0 && cnt > 0) atomicAdd(runs, 1);
  if (q >= cnt) return;
  const int p = plist ? plist[q] : q;
  const uint16_t* t = tours + (size_t)p * np;
  const double* dg = dcache + (size_t)p * np;
  int32_t* O = out + (size_t)p * 2 * cw;
  int32_t* D = O + cw;
  for (int k = threadIdx.x; k < cw; k += blockDim.x) {
    const int kk = k - 3;
    O[k] = (kk >= 0 && kk <= n) ? es * (int)t[kk == n ? 0 : kk] : 0;
    if (k < n) {
      double d = dg[k];
      if (vfrom > 0.0 && d == vfrom) d = vto;
      D[k] = __double2int_rn(d * scale);
    } else {
      D[k] = -kBig;
    }
  }
}

// Scan of one 8-column group [c0, c0 + 8) of a band by one warp: the lane's
// gathers G(c0 + 1 .. c0 + 8) at the group's offsets, the pairs (i, c0 + k)
// = G_l(c0 + k) + G_{l+1}(c0 + k + 1) - D[c0 + k], the warp-uniform
// pre-test against the lane limits.  MASK: columns c < i + 2 are dead
// (the band's triangle).
template <int MODE, bool MASK, int ES>
__device__ __forceinline__ void band_group(const int* O, const int* D,
                                           int c0, uint32_t R, int& prev,
                                           int& L, int i, int Di, bool live,
                                           int win, int* st, int* ws,
                                           int* cmin, uint32_t slot_next) {
  const int4 oa = *reinterpret_cast<const int4*>(O + 4 + c0);
  const int4 ob = *reinterpret_cast<const int4*>(O + 8 + c0);
  const int4 da = *reinterpret_cast<const int4*>(D + c0);
  const int4 db = *reinterpret_cast<const int4*>(D + c0 + 4);
  const int off[8] = {oa.x, oa.y, oa.z, oa.w, ob.x, ob.y, ob.z, ob.w};
  const int dv[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
  int g[8], u[8];
#if DPSO_BAND_NBLDS
  // the B term straight from slot l+1 (the next lane's row, S + 4 bytes
  // on): a second LDS with an immediate offset instead of a shuffle
  int nb[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t ad = R + (uint32_t)off[k];
    g[k] = lds_el<ES>(ad);
    nb[k] = lds_el<ES>(ad + slot_next);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) u[k] = (k ? g[k - 1] : prev) + nb[k] - dv[k];
#else
#pragma unroll
  for (int k = 0; k < 8; ++k) g[k] = lds_el<ES>(R + (uint32_t)off[k]);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int nb = __shfl_down_sync(0xffffffffu, g[k], 1);
    u[k] = (k ? g[k - 1] : prev) + nb - dv[k];
  }
#endif
  prev = g[7];
  if (MASK) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (c0 + k < i + 2) u[k] = kBig;
  }
  const int mn = min(min(min(u[0], u[1]), min(u[2], u[3])),
                     min(min(u[4], u[5]), min(u[6], u[7])));
  if (__any_sync(0xffffffffu, mn <= L))
    L = band_hit<MODE>(u[0], u[1], u[2], u[3], u[4], u[5], u[6], u[7], c0, i,
                       Di, L, live, win, st, ws, cmin);
}

// Two rows per lane (64-slot bands): lane l owns pair rows i0 + l (slots l,
// l + 1) and i0 + 32 + l (slots 32 + l, 33 + l).  One set of column records
// and one address per column serve both rows; the second row's loads sit
// at uniform offsets 32 (S + 4) and 33 (S + 4) from the first's.
// M1 / M2: the columns c < i + 2 of row set 1 / 2 are dead (the triangle).
template <int MODE, bool M1, bool M2>
__device__ __forceinline__ void band_group2(
    const int* O, const int* D, int c0, uint32_t R, int& prev, int& prev2,
    int& L, int& L2, int i, int i2, int Di, int Di2, bool live, bool live2,
    int win, int* st, int* st2, int* ws, int* cmin, uint32_t sn,
    uint32_t s32, uint32_t s33) {
  const int4 oa = *reinterpret_cast<const int4*>(O + 4 + c0);
  const int4 ob = *reinterpret_cast<const int4*>(O + 8 + c0);
  const int4 da = *reinterpret_cast<const int4*>(D + c0);
  const int4 db = *reinterpret_cast<const int4*>(D + c0 + 4);
  const int off[8] = {oa.x, oa.y, oa.z, oa.w, ob.x, ob.y, ob.z, ob.w};
  const int dv[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
  int g[8], nb[8], g2[8], nb2[8], u[8], u2[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t ad = R + (uint32_t)off[k];
    g[k] = lds_s16(ad);
    nb[k] = lds_s16(ad + sn);
    g2[k] = lds_s16(ad + s32);
    nb2[k] = lds_s16(ad + s33);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    u[k] = (k ? g[k - 1] : prev) + nb[k] - dv[k];
    u2[k] = (k ? g2[k - 1] : prev2) + nb2[k] - dv[k];
  }
  prev = g[7];
  prev2 = g2[7];
  if (M1) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (c0 + k < i + 2) u[k] = kBig;
  }
  if (M2) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (c0 + k < i2 + 2) u2[k] = kBig;
  }
  const int mn = min(min(min(u[0], u[1]), min(u[2], u[3])),
                     min(min(u[4], u[5]), min(u[6], u[7])));
  const int mn2 = min(min(min(u2[0], u2[1]), min(u2[2], u2[3])),
                      min(min(u2[4], u2[5]), min(u2[6], u2[7])));
  const bool h1 = mn <= L, h2 = mn2 <= L2;
  if (__any_sync(0xffffffffu, h1 || h2)) {
    if (__any_sync(0xffffffffu, h1))
      L = band_hit<MODE>(u[0], u[1], u[2], u[3], u[4], u[5], u[6], u[7], c0,
                         i, Di, L, live, win, st, ws, cmin);
    if (__any_sync(0xffffffffu, h2))
      L2 = band_hit<MODE>(u2[0], u2[1], u2[2], u2[3], u2[4], u2[5], u2[6],
                          u2[7], c0, i2, Di2, L2, live2, win, st2, ws, cmin);
  }
}

// Persistent CTAs: kBandWarps consumer warps + kProdWarps producer warps.
// CTA b scans particles b, b + grid, ...; a particle's bands run in order
// and band t sits in stage t % nst of a ring; a particle's column arrays
// have their own barrier (every warp group waits for them at its first band
// of the particle).  Producer warp w issues its
// 32 / kProdWarps rows of every band (bulk copies; a warp's copies
// serialize on the issue path, so several producers divide the issue time
// of a band) once the
// consumers have released the stage (empty barrier, one arrival per
// consumer warp), and producer 0 adds the particle's column arrays to its
// band 0 (full barrier: one expect-tx arrival per producer).  Consumer
// warps walk the bands at their own pace; a particle's result is reduced by
// the last consumer to finish it.  Column buffers and per-particle result
// slots rotate over ncb >= 2 particles, enough that the producers' lead of
// nst bands never reaches a buffer still in use.
constexpr int kProdWarps = 4;
constexpr int kMaxNcb = 8;

template <int MODE, int RPL, int ES>
__global__ void __launch_bounds__((kBandWarps + kProdWarps) * 32, 1)
    k_two_opt_band(BandArgs a, const __grid_constant__ CUtensorMap tm) {
  // RPL rows per lane: 32 RPL slots and 32 RPL - 1 pair rows per band
  constexpr int kSlots = 32 * RPL, kRows = kSlots - 1;
  if (a.ctl && (a.ctl->done || a.ctl->improved)) return;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ __align__(8) uint64_t colfull[kMaxNcb];
  __shared__ int s_fin[kMaxNcb], s_of[kMaxNcb];
  __shared__ int s_cmin[kMaxNcb];  // CTA-wide running minimum t, per slot
  __shared__ double s_rd[kMaxNcb][kBandWarps];
  __shared__ int s_ri[kMaxNcb][kBandWarps], s_rj[kMaxNcb][kBandWarps];
  __shared__ int s_ws[kBandWarps][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kBandWarps;
  const int n = a.n, nst = a.nst, ncb = a.ncb;
  const int nb = (n + kRows - 2) / kRows;  // bands: rows 0 .. n-2
  const int count = a.pcnt ? *a.pcnt : a.count;
  const int nmine =
      (int)blockIdx.x < count ? (count - 1 - (int)blockIdx.x) / gridDim.x + 1
                              : 0;
  if (nmine == 0) return;
  const int total = nmine * nb;
  const uint32_t S = a.slot;
  unsigned char* rowbuf = smem;
  const uint32_t stage_bytes = kSlots * S + 128 * RPL;
  int* cols = (int*)(smem + (size_t)nst * stage_bytes);  // [ncb][O | D]
  int* lstate = cols + ncb * 2 * a.cw;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const uint32_t colbytes = (uint32_t)(2 * a.cw * 4);

  if (threadIdx.x == 0) {
    for (int k = 0; k < nst; ++k) {
      mbar_init(&full[k], kProdWarps);
      mbar_init(&empty[k], NW / a.groups);
    }
    fence_barrier_init();
    for (int k = 0; k < ncb; ++k) mbar_init(&colfull[k], 1);
    for (int k = 0; k < kMaxNcb; ++k) {
      s_fin[k] = s_of[k] = 0;
      s_cmin[k] = kNone;
    }
  }
  __syncthreads();

  if (warp >= NW) {
    // ---- producer warp pw: rows rpp pw .. rpp pw + rpp - 1 of every band
    const int pw = warp - NW;
    constexpr int rpp = kSlots / kProdWarps;  // rows per producer warp
    int band = 0, pl = 0, cb = 0, s = 0, use = 0, cuse = 0;
    for (int t = 0; t < total; ++t) {
      if (use > 0) mbar_wait_backoff(&empty[s], (uint32_t)((use - 1) & 1));
      // from the particle's second band on, its cities come from the column
      // records in shared memory (O[3 + k] = 2 a_k) instead of a dependent
      // global load ahead of every copy
      if (band == 1) mbar_wait_backoff(&colfull[cb], (uint32_t)(cuse & 1));
      const int* Oc = cols + cb * 2 * a.cw + 3;
      const int pq = (int)blockIdx.x + pl * (int)gridDim.x;
      const int pp = a.plist ? a.plist[pq] : pq;
      const int i0 = band * kRows;  // kRows pair rows per band
      const int r0 = rpp * pw;
      const int nr = max(0, min(rpp, n - i0 - r0));
      const bool withcols = band == 0 && pw == 0;
      if (a.probe == 2 && t >= nst) {  // consumer floor: no row copies
        if (lane == 0) {
          mbar_expect_tx(&full[s], 0);
          if (withcols) mbar_expect_tx(&colfull[cb], colbytes);
        }
        __syncwarp();
        if (withcols && lane == 0)
          bulk_g2s(cols + cb * 2 * a.cw, a.cols + (size_t)pp * 2 * a.cw,
                   colbytes, &colfull[cb]);
        if (++s == nst) {
          s = 0;
          ++use;
        }
        if (++band == nb) {
          band = 0;
          ++pl;
          if (++cb == ncb) {
            cb = 0;
            ++cuse;
          }
        }
        continue;
      }
      unsigned char* stg = rowbuf + (size_t)s * stage_bytes;
      if (a.g4) {
        // groups of 4 slots: group g = pw + kProdWarps k (k < 8 / kProdWarps)
        // to stg + 4 g S (128-byte aligned), slot 4g + q from version q with
        // the box starting 16 g bytes before the line: slot l's element c
        // lands at l (S + 4) + 2c, the bulk-copy layout
        constexpr int gpp = kSlots / 4 / kProdWarps;
        const int rows_left = n - i0;
        int mine = 0;
#pragma unroll
        for (int k = 0; k < gpp; ++k) mine += 4 * (pw + kProdWarps * k) < rows_left;
        if (lane == 0) {
          mbar_expect_tx(&full[s], (uint32_t)mine * 4u * S);
          if (withcols) mbar_expect_tx(&colfull[cb], colbytes);
        }
        __syncwarp();
        const int g = pw + kProdWarps * lane;
        if (lane < gpp && 4 * g < rows_left) {
          fence_proxy_async();  // the consumers' reads of the stage first
          const uint16_t* tr = a.tours + (size_t)pp * a.np + i0 + 4 * g;
          int rw[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            rw[q] = q * n + (4 * g + q < rows_left
                                 ? (band ? Oc[i0 + 4 * g + q] >> (ES - 1)
                                         : (int)tr[q])
                                 : 0);
          // groups past the eighth: whole 128-byte steps of the shift go to
          // the destination (it must stay 128-byte aligned)
          tma_gather4(stg + (size_t)4 * g * S + 128 * (g >> 3), &tm,
                      -2 * (g & 7), rw[0], rw[1], rw[2], rw[3], &full[s]);
        }
      } else {
        if (lane == 0) {
          mbar_expect_tx(&full[s], (uint32_t)nr * (uint32_t)a.line);
          if (withcols) mbar_expect_tx(&colfull[cb], colbytes);
        }
        __syncwarp();
        if (lane < nr) {
          fence_proxy_async();  // the consumers' reads of the stage first
          const int l = r0 + lane;
          const int city = band ? Oc[i0 + l] >> (ES - 1)
                                : (int)a.tours[(size_t)pp * a.np + i0 + l];
          const unsigned char* src =
              a.rows + ((size_t)(l & 3) * n + city) * (size_t)a.line;
          bulk_g2s(stg + (size_t)l * S + 16 * (l >> 2), src,
                   (uint32_t)a.line, &full[s]);
        }
      }
      if (withcols && lane == 0)
        bulk_g2s(cols + cb * 2 * a.cw, a.cols + (size_t)pp * 2 * a.cw,
                 colbytes, &colfull[cb]);
      if (++s == nst) {
        s = 0;
        ++use;
      }
      if (++band == nb) {
        band = 0;
        ++pl;
        if (++cb == ncb) {
            cb = 0;
            ++cuse;
          }
      }
    }
    return;
  }

  // ---- consumer warp
  int* st = lstate + warp * kLaneState * 32 * RPL + lane;
  int* st2 = st + kLaneState * 32;  // RPL == 2: the lane's second row
  int* ws = s_ws[warp];
  auto reset_state = [&]() {
    st[0] = MODE == 1 ? kNone : kBig;
    st[32] = MODE == 1 ? INT_MAX : 0;
    st[64] = MODE == 1 ? INT_MAX : 0;
    if (RPL == 2) {
      st2[0] = MODE == 1 ? kNone : kBig;
      st2[32] = MODE == 1 ? INT_MAX : 0;
      st2[64] = MODE == 1 ? INT_MAX : 0;
    }
    if (lane == 0) {
      ws[0] = kNone;
      ws[1] = INT_MAX;
    }
    __syncwarp();
  };
  reset_state();
  // warp groups: group g scans bands g, g + G, ... (G = a.groups), its
  // NWg warps splitting each band's columns
  const int G = a.groups, NWg = NW / G;
  const int lgw = G == 2 ? 3 : 4;  // log2 NWg
  const int grp = warp >> lgw, wl = warp - (grp << lgw);
  int band = 0, pl = 0, cb = 0, s = 0, use = 0, cuse = 0;
  auto step = [&]() {  // to the next band of the sequence
    if (++s == nst) {
      s = 0;
      ++use;
    }
    if (++band == nb) {
      band = 0;
      ++pl;
      if (++cb == ncb) {
        cb = 0;
        ++cuse;
      }
    }
  };
  for (int k = 0; k < grp; ++k) step();
  // shared-memory addresses computed once (not per band)
  const uint32_t full_a = smem_u32(full), empty_a = smem_u32(empty);
  const uint32_t colfull_a = smem_u32(colfull);
  const uint32_t R0 = smem_u32(rowbuf) + (uint32_t)lane * (S + 4u);
  for (int t = grp; t < total; t += G) {
    const int pq = (int)blockIdx.x + pl * (int)gridDim.x;
    const int pp = a.plist ? a.plist[pq] : pq;
    const int i0 = band * kRows;
    // the particle's column arrays (its first band for this warp), rows
    if (band < G) mbar_wait_sleep_u32(colfull_a + 8u * cb, (uint32_t)(cuse & 1));
    mbar_wait_sleep_u32(full_a + 8u * s, (uint32_t)(use & 1));
    const int* O = cols + cb * 2 * a.cw;
    const int* D = O + a.cw;
    const int i = i0 + lane;
    const bool live = (RPL == 2 || lane < kBandRows) && i <= n - 2;
    const int Di = live ? D[i] : 0;
    const uint32_t R = R0 + (uint32_t)s * stage_bytes;
    int L = lane_limit<MODE>(live, Di, i, ws[0], ws[1]);
    const int i2 = i0 + 32 + lane;
    const bool live2 = RPL == 2 && lane < 31 && i2 <= n - 2;
    const int Di2 = live2 ? D[i2] : 0;
    int L2 = RPL == 2 ? lane_limit<MODE>(live2, Di2, i2, ws[0], ws[1])
                      : INT_MIN;
    {  // capped by the CTA-wide minimum (other warps' finds)
      const int cm = *(volatile int*)&s_cmin[cb];
      if (live) L = min(L, cm + (MODE == 2 ? a.win : 0) + Di);
      if (live2) L2 = min(L2, cm + (MODE == 2 ? a.win : 0) + Di2);
    }
    const int cs = (i0 + 2) & ~7;
    const int per = ((((n - cs) + NWg - 1) >> lgw) + 7) & ~7;
    const int cA = cs + wl * per, cB = min(n, cA + per);
    if (cA < cB && a.probe != 1) {
      int prev = lds_el<ES>(R + (uint32_t)O[3 + cA]);
      int c0 = cA;
      if (RPL == 1) {
        for (; c0 < cB && c0 < i0 + 32; c0 += 8)
          band_group<MODE, true, ES>(O, D, c0, R, prev, L, i, Di, live,
                                     a.win, st, ws, &s_cmin[cb], S + 4u);
        for (; c0 < cB; c0 += 8)
          band_group<MODE, false, ES>(O, D, c0, R, prev, L, i, Di, live,
                                      a.win, st, ws, &s_cmin[cb], S + 4u);
      } else {
        const uint32_t s32 = 32u * (S + 4u), s33 = s32 + S + 4u;
        int prev2 = lds_s16(R + s32 + (uint32_t)O[3 + cA]);
        for (; c0 < cB && c0 < i0 + 32; c0 += 8)
          band_group2<MODE, true, true>(O, D, c0, R, prev, prev2, L, L2, i,
                                        i2, Di, Di2, live, live2, a.win, st,
                                        st2, ws, &s_cmin[cb], S + 4u, s32,
                                        s33);
        for (; c0 < cB && c0 < i0 + 64; c0 += 8)
          band_group2<MODE, false, true>(O, D, c0, R, prev, prev2, L, L2, i,
                                         i2, Di, Di2, live, live2, a.win, st,
                                         st2, ws, &s_cmin[cb], S + 4u, s32,
                                         s33);
        for (; c0 < cB; c0 += 8)
          band_group2<MODE, false, false>(O, D, c0, R, prev, prev2, L, L2, i,
                                          i2, Di, Di2, live, live2, a.win,
                                          st, st2, ws, &s_cmin[cb], S + 4u,
                                          s32, s33);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_u32(empty_a + 8u * s);  // stage reads done
    // this warp's last band of the particle: the next band of its group is
    // in a later particle (nb >= G, so every group has a band in each)
    if (band + G >= nb || t + G >= total) {
      // ---- particle done: this warp's result, then the CTA's (last warp)
      double bd = kInf;
      int bi = INT_MAX, bj = INT_MAX;
      const uint16_t* tour = a.tours + (size_t)pp * a.np;
      const double* dg = a.dcache + (size_t)pp * a.np;
      if (MODE == 1) {
        if (st[0] < kNone) {
          bd = (double)st[0];
          bi = st[32];
          bj = st[64];
        }
        if (RPL == 2 && st2[0] < kNone &&
            lex_lt((double)st2[0], st2[32], st2[64], bd, bi, bj)) {
          bd = (double)st2[0];
          bi = st2[32];
          bj = st2[64];
        }
      } else if (__any_sync(0xffffffffu,
                            st[64] || (RPL == 2 && st2[64]))) {
        if (lane == 0) atomicOr(&s_of[cb], 1);
      } else {
        int wm = RPL == 2 ? min(st[0], st2[0]) : st[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
          wm = min(wm, __shfl_xor_sync(0xffffffffu, wm, o));
        const int keep = wm + a.win;
        for (int set = 0; set < RPL; ++set) {
          const int* sts = set ? st2 : st;
          const int nc = sts[32];
          const int* cd = sts + 96;
          const int* cij = cd + 32 * kBandCand;
          for (int k = 0; k < nc; ++k) {
            if (cd[32 * k] <= keep) {
              const int ci = cij[32 * k] >> 16, cj = cij[32 * k] & 0xFFFF;
              const int ai = tour[ci], aj = tour[cj];
              const int si = tour[ci + 1],
                        sj = tour[cj + 1 == n ? 0 : cj + 1];
              double v = __dadd_rn(a.cost[(size_t)ai * a.ld + aj],
                                   a.cost[(size_t)si * a.ld + sj]);
              v = __dsub_rn(v, dg[ci]);
              v = __dsub_rn(v, dg[cj]);
              if (lex_lt(v, ci, cj, bd, bi, bj)) {
                bd = v;
                bi = ci;
                bj = cj;
              }
            }
          }
        }
        // structural pairs, exactly from d (this warp's share of rows)
        for (int ii = warp * 32 + lane; ii < n - 1; ii += NW * 32) {
          const double d0 = dg[ii], d1 = dg[ii + 1];
          double v = __dadd_rn(d0, d1);
          v = __dsub_rn(v, d0);
          v = __dsub_rn(v, d1);
          if (lex_lt(v, ii, ii + 1, bd, bi, bj)) {
            bd = v;
            bi = ii;
            bj = ii + 1;
          }
        }
        if (warp == 0 && lane == 0 && n - 1 > 1) {  // (0, n-1): s = a_0
          const int j = n - 1;
          double v = __dadd_rn(a.cost[(size_t)tour[0] * a.ld + tour[j]],
                               a.cost[(size_t)tour[1] * a.ld + tour[0]]);
          v = __dsub_rn(v, dg[0]);
          v = __dsub_rn(v, dg[j]);
          if (lex_lt(v, 0, j, bd, bi, bj)) {
            bd = v;
            bi = 0;
            bj = j;
          }
        }
      }
      warp_lexmin(bd, bi, bj);
      int last = 0;
      if (lane == 0) {
        s_rd[cb][warp] = bd;
        s_ri[cb][warp] = bi;
        s_rj[cb][warp] = bj;
        __threadfence_block();
        last = atomicAdd(&s_fin[cb], 1) == NW - 1;
        __threadfence_block();
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        double d = lane < NW ? s_rd[cb][lane] : kInf;
        int ri = lane < NW ? s_ri[cb][lane] : INT_MAX;
        int rj = lane < NW ? s_rj[cb][lane] : INT_MAX;
        warp_lexmin(d, ri, rj);
        TwoOptRes* out = a.res + (size_t)pp * a.chunks;
        const int of = MODE == 2 ? s_of[cb] : 0;
        int base = 0;
        if (of && lane == 0) base = atomicAdd(&a.ovf[0], a.chunks);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int c = lane; c < a.chunks; c += 32) {
          if (of) {
            out[c] = {kInf, kOvfTag, kOvfTag};
            a.ovf[1 + base + c] = pp * a.chunks + c;
          } else {
            out[c] = c == 0 ? TwoOptRes{d, ri, rj}
                            : TwoOptRes{kInf, INT_MAX, INT_MAX};
          }
        }
        __syncwarp();
        if (lane == 0) {
          s_fin[cb] = 0;
          s_cmin[cb] = kNone;
          s_of[cb] = 0;
        }
      }
      reset_state();
    }
    for (int k = 0; k < G; ++k) step();
  }
}

// 4 rotated int16 (or int8) versions of round(C * scale): version q, row r
// is the line at byte (q n + r) line; element c at byte 4q + es c of it.
template <typename T>
__global__ void k_cost_band(const double* cost, int64_t ld, int n, T* out,
                            int line, double scale, double vfrom,
                            double vto) {
  constexpr int es = (int)sizeof(T);
  const int per = line / es;
  const int64_t total = 4 * (int64_t)n * per;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / per;
    const int c = (int)(e % per);
    const int qv = (int)(row / n), r = (int)(row % n);
    const int cc = c - 4 / es * qv;
    T v = 0;
    if (cc >= 0 && cc < n) {
      double x = cost[(int64_t)r * ld + cc];
      if (vfrom > 0.0 && x == vfrom) x = vto;
      v = (T)__double2int_rn(x * scale);
    }
    out[e] = v;
  }
}

// slot l of a stage starts at l S + 16 (l div 4): S >= line keeps slots
// apart (the stagger never decreases); a stage spans 32 S + 128 bytes.
// gather4 staging: a slot is one box of S bytes, the line shifted by up to
// 112 bytes (16 g for group g), S a multiple of 32 (4 S: group starts
// 128-byte aligned), at most 256 8-byte columns per box.
uint32_t band_slot(int line, bool g4) {
  return g4 ? (uint32_t)round_up(line + 112, 32) : (uint32_t)round_up(line, 128);
}
constexpr int kG4MaxBox = 2048;

// bands of 32 rpl - 1 pair rows (rpl rows per lane)
int band_nb(int n, int rpl) {
  const int rows = 32 * rpl - 1;
  return (n + rows - 2) / rows;
}

// column buffers / result slots for nst stages: no warp runs more than nst
// bands ahead of another, so (ncb - 1) nb >= nst keeps a particle's buffers
// until every warp is past it
int band_ncb(int n, int nst, int rpl) {
  const int nb = band_nb(n, rpl);
  return std::min(kMaxNcb, std::max(2, (nst + nb - 1) / nb + 1));
}

// warp groups: two groups scan alternate bands when two stages can be
// scanned while the others load (nst == 4) and every group has a band in
// every particle (one row per lane only)
int band_groups(int n, int nst, int rpl) {
  if (rpl == 2) return 1;
  if (const char* e = getenv("DPSO_BAND_GROUPS")) {
    const int g = atoi(e);
    if (g == 1 || (g == 2 && nst % 2 == 0 && band_nb(n, 1) >= 2)) return g;
  }
  return nst == 4 && band_nb(n, 1) >= 2 ? 2 : 1;
}

int band_line_es(int n, int es) {
  return (int)round_up((int64_t)es * n + 12, 16);
}

size_t band_smem_l(int line, int n, int nst, bool g4, int rpl) {
  return (size_t)nst * (32 * rpl * band_slot(line, g4) + 128 * rpl) +
         (size_t)band_ncb(n, nst, rpl) * 2 * band_cw(n) * 4 +
         (size_t)kBandWarps * kLaneState * 32 * 4 * rpl;
}

constexpr size_t kBandSmemMax = 225 * 1024;

// row element size: int16 wherever two 32-slot stages of int16 rows fit
// (n <= ~1400), else int8 (n <= ~2500); 0: no band scan.  DPSO_BAND_ES=1
// forces int8 rows (testing at small n).
int band_es(int n) {
  if (n < 4 || n > kBandMaxN) return 0;
  const bool fit2 =
      band_smem_l(band_line_es(n, 2), n, 2, false, 1) <= kBandSmemMax;
  const bool fit1 =
      band_smem_l(band_line_es(n, 1), n, 2, false, 1) <= kBandSmemMax;
  if (const char* e = getenv("DPSO_BAND_ES"))
    if (atoi(e) == 1 && fit1) return 1;
  return fit2 ? 2 : fit1 ? 1 : 0;
}

size_t band_smem(int n, int nst, bool g4, int rpl) {
  return band_smem_l(band_line_es(n, std::max(1, band_es(n))), n, nst, g4,
                     rpl);
}

bool band_g4_fits(int n) {
  return (int)band_slot(band_line_es(n, std::max(1, band_es(n))), true) <=
         kG4MaxBox;
}

// stages: as many as fit, up to kMaxStages
int band_stages(int n, bool g4, int rpl) {
  int nst = kMaxStages;
  while (nst > 2 && band_smem(n, nst, g4, rpl) > kBandSmemMax) --nst;
  if (const char* e = getenv("DPSO_BAND_STAGES")) {
    const int x = atoi(e);
    if (x >= 2 && x <= kMaxStages &&
        band_smem(n, x, g4, rpl) <= kBandSmemMax)
      nst = x;
  }
  return nst;
}

// two rows per lane (64-slot bands) wherever two such stages fit;
// DPSO_BAND_RPL=1 keeps one
int band_rpl(int n, bool g4) {
  if (const char* e = getenv("DPSO_BAND_RPL"))
    if (atoi(e) == 1) return 1;
  return n >= 64 && band_es(n) == 2 && band_smem(n, 2, g4, 2) <= kBandSmemMax
             ? 2
             : 1;
}

// The tensor map of the row versions for gather4: a 2-D tensor of 4n lines
// (line bytes each) of 8-byte columns, one box = S / 8 columns x 1 line.
// False when the driver entry point is missing or the encode fails (the
// bulk-copy staging is used then).
bool band_encode_g4(const unsigned char* rows, int n, int line,
                    unsigned char* out) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static bool looked = false;
  if (!looked) {
    looked = true;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode,
                                cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      encode = nullptr;
    cudaGetLastError();
  }
  if (!encode) return false;
  alignas(64) CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)(line / 8), (cuuint64_t)(4 * (int64_t)n)};
  cuuint64_t gstride[1] = {(cuuint64_t)line};
  cuuint32_t box[2] = {band_slot(line, true) / 8, 1};
  cuuint32_t estr[2] = {1, 1};
  if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_INT64, 2, (void*)rows, gdim,
             gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap size");
  memcpy(out, &tm, sizeof tm);
  return true;
}

}  // namespace

int band_line(int n) { return band_line_es(n, std::max(1, band_es(n))); }

int band_cw(int n) { return (int)round_up(n + 16, 8); }

int64_t band_rows_bytes(int n) {
  if (band_es(n) == 0) return 0;
  return 4 * (int64_t)n * band_line(n);
}

int64_t band_cols_bytes(int n, int64_t count) {
  return band_rows_bytes(n) ? 8 * (int64_t)band_cw(n) * count : 0;
}

cudaError_t band_prepare(const double* cost, int64_t ld, int32_t n,
                         unsigned char* buf, double mx, bool integral,
                         double vfrom, double vto, cudaStream_t s,
                         TwoOptPlan* pl) {
  pl->band = nullptr;
  pl->band_mode = 0;
  pl->band_g4 = 0;
  if (!buf || band_rows_bytes(n) == 0) return cudaSuccess;
  if (const char* e = getenv("DPSO_SCAN_BAND"))
    if (atoi(e) == 0) return cudaSuccess;
  // the knobs that select variants of the column-per-lane scan
  // (k_two_opt.cu) select that scan
  if (getenv("DPSO_SCAN_MODE") || getenv("DPSO_SCAN16") ||
      getenv("DPSO_SCAN_NOPERSIST") || getenv("DPSO_SCAN_STREAM_ONLY") ||
      getenv("DPSO_SCAN_NPL"))
    return cudaSuccess;
  if (!(mx > 1e-30 && mx < 1e30)) return cudaSuccess;
  const int es = band_es(n);
  const double emax = es == 2 ? 32767.0 : 127.0;
  int mode;
  double scale = 1.0;
  if (integral && mx <= emax) {
    mode = 1;
  } else {
    mode = 2;
    scale = ldexp(1.0, (es == 2 ? 14 : 6) - ilogb(mx));
    while (mx * scale > emax) scale *= 0.5;
  }
  // testing: FILTER on an EXACT-eligible matrix (same rows, scale 1)
  if (const char* e = getenv("DPSO_BAND_MODE")) mode = atoi(e) == 2 ? 2 : mode;
  const int line = band_line(n);
  const int64_t total = 4 * (int64_t)n * (line / es);
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (es == 2)
    k_cost_band<int16_t><<<std::max(blocks, 1), 256, 0, s>>>(
        cost, ld, n, (int16_t*)buf, line, scale, vfrom, vto);
  else
    k_cost_band<int8_t><<<std::max(blocks, 1), 256, 0, s>>>(
        cost, ld, n, (int8_t*)buf, line, scale, vfrom, vto);
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  pl->band = buf;
  pl->band_line = line;
  pl->band_es = es;
  pl->band_mode = mode;
  pl->band_scale = scale;
  pl->band_win = mode == 2 ? 4 : 0;
  pl->band_vfrom = vfrom;
  pl->band_vto = vto;
  bool g4 = band_g4_fits(n);
  if (const char* e = getenv("DPSO_BAND_G4")) g4 = g4 && atoi(e) != 0;
  pl->band_g4 = g4 && band_encode_g4(buf, n, line, pl->band_tm) ? 1 : 0;
  pl->band_rpl = band_rpl(n, pl->band_g4 != 0);
  return cudaSuccess;
}

cudaError_t launch_two_opt_band(const TwoOptPlan& pl, int32_t n, int32_t np,
                                const uint16_t* tours, const double* dcache,
                                int32_t count, TwoOptRes* res, int32_t chunks,
                                int32_t* ovf, const DevCtl* ctl,
                                cudaStream_t s, int reserve_sms,
                                const int32_t* plist, const int32_t* pcnt,
                                int32_t* runs, bool cols_ready) {
  if (!pl.band_cols || count > pl.band_cols_cap) return cudaErrorInvalidValue;
  BandArgs a;
  memset(&a, 0, sizeof a);
  a.cost = pl.cost;
  a.ld = pl.ld;
  a.rows = pl.band;
  a.line = pl.band_line;
  a.g4 = pl.band_g4;
  a.slot = band_slot(pl.band_line, a.g4 != 0);
  a.n = n;
  a.np = np;
  a.count = count;
  a.chunks = chunks;
  a.tours = tours;
  a.dcache = dcache;
  a.res = res;
  a.ctl = ctl;
  a.ovf = ovf;
  a.scale = pl.band_scale;
  a.vfrom = pl.band_vfrom;
  a.vto = pl.band_vto;
  a.win = pl.band_win;
  a.cw = band_cw(n);
  a.cols = pl.band_cols;
  a.plist = plist;
  a.pcnt = pcnt;
  // (the bounded scan writes the records of the particles it lists)
  if (!cols_ready)
    k_band_cols<<<count, 256, 0, s>>>(tours, np, dcache, n, a.cw, count,
                                       a.scale, a.vfrom, a.vto, pl.band_cols,
                                       ctl, pl.band_es, plist, pcnt, runs);
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  const int rpl = pl.band_rpl;
  a.nst = band_stages(n, a.g4 != 0, rpl);
  a.ncb = band_ncb(n, a.nst, rpl);
  a.groups = band_groups(n, a.nst, rpl);
  if (const char* e = getenv("DPSO_BAND_PROBE")) a.probe = atoi(e);
  const size_t smem = band_smem(n, a.nst, a.g4 != 0, rpl);
  alignas(64) CUtensorMap tm;
  memcpy(&tm, pl.band_tm, sizeof tm);  // unused (zero) without gather4
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = std::max(1, std::min(count, sms - reserve_sms));
  auto go = [&](auto kern) {
    cudaError_t err = set_dyn_smem((const void*)kern, smem);
    if (err) return err;
    kern<<<blocks, (kBandWarps + kProdWarps) * 32, smem, s>>>(a, tm);
    return cudaGetLastError();
  };
  if (pl.band_es == 1)
    return pl.band_mode == 1 ? go(k_two_opt_band<1, 1, 1>)
                             : go(k_two_opt_band<2, 1, 1>);
  if (pl.band_mode == 1)
    return rpl == 2 ? go(k_two_opt_band<1, 2, 2>)
                    : go(k_two_opt_band<1, 1, 2>);
  return rpl == 2 ? go(k_two_opt_band<2, 2, 2>) : go(k_two_opt_band<2, 1, 2>);
}

}  // namespace dpso
