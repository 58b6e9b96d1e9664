// Best-improvement 2-opt (solver.py:88-106, applied at solver.py:309-317).
//
// delta(i,j) = ((C[a_i,a_j] + C[s_i,s_j]) - d_i) - d_j for 0 <= i < j < n,
// s = roll(a, -1), d_i = C[a_i, s_i]; the move is the first (row-major)
// argmin; it is applied when delta < -1e-12 and fitness += delta.
//
// Work decomposition: one warp owns a task = (particle, band of pair rows
// [r0, r1)); bands are cut so every task has ~equal pair count and there are
// ~4 tasks per resident warp slot.  The cost rows a_r0 .. a_r1 are streamed
// in tour order from L2 into a 3-deep per-warp ring in shared memory by
// cp.async.bulk (TMA bulk copy, mbarrier completion): each row is read once
// per task and used twice (A row of pair-row i, B row of pair-row i-1).
// Lane l owns columns j = l + 32m; a_j, s_j (packed u16) and d_j stay in
// registers for the whole task; a row costs two shared-memory gathers per
// pair.  Columns are processed in groups of 4 blocks of 32 with a
// warp-uniform skip of dead groups (j <= i), predicated masking inside, so
// gathers of a group are in flight together.
//
// Three scan modes, chosen once per cost matrix (k_cost_prep):
//   EXACT32  integer matrices with |C| < 2^22 (scene matrices): every fp32
//            delta equals the fp64 delta exactly, so the fp32 scan IS the
//            reference computation (half the L2 bytes and gathers of fp64).
//   FILTER32 everything else: fp32 deltas with a rigorous bound
//            |delta32 - delta64| <= eps (eps = 2^-18 max|C| >= 4x the
//            worst-case rounding), each lane keeps the pairs within 2 eps of
//            its running fp32 minimum; at the end the warp's candidates within
//            2 eps of the warp minimum are re-evaluated in fp64 (exact
//            reference arithmetic).  The true argmin and all its fp64 ties are
//            provably among the candidates.  The structural pairs (i, i+1)
//            and (0, n-1) - arithmetic no-ops whose fp64 residue the
//            reference can still pick - are evaluated exactly from d.  A
//            candidate-list overflow re-scans that task in fp64 (FP64 mode).
//   FP64     the reference expression on fp64 rows (fallback and for
//            matrices fp32 cannot represent).
// Each lane keeps its first strict minimum in (i, j) order; warp shuffles
// reduce (delta, i, j); the apply kernel merges bands in row order.
#include <float.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "dpso_internal.cuh"
#include "tma.cuh"

namespace dpso {

namespace {

constexpr int kMaxWarps = 4;  // warps (tasks) per CTA, upper bound
constexpr int kBufs = 3;      // row ring depth per warp
constexpr int kGroup = 4;     // column blocks (of 32) per uniform skip test
constexpr int kCand = 4;      // fp32 candidates kept per lane (FILTER32)
constexpr int kOverflowTag = -2;

struct ScanArgs {
  const double* cost;
  int64_t ld;
  const float* cost32;
  int64_t ld32;
  int32_t n, np, count, chunks;
  const uint16_t* tours;   // count x np
  const double* dcache;    // count x np
  const int32_t* chunk_row;
  TwoOptRes* res;          // count x chunks
  const DevCtl* ctl;       // nullable: skip when done or improved
  uint32_t row_bytes;      // bytes streamed per cost row (multiple of 16)
  uint32_t buf_stride;     // bytes between ring buffers
  uint32_t buf_stride2;    // bytes of one warp's smem (ring + d_j)
  float thr;               // FILTER32: 2 * eps
  int only_flagged;        // FP64 fallback: only tasks tagged kOverflowTag
  int stream_only;         // debug: stream the rows, skip the pair compute
};

__device__ __forceinline__ bool res_less(double d1, int i1, int j1, double d2,
                                         int i2, int j2) {
  if (d1 < d2) return true;
  if (d2 < d1) return false;
  return (i1 < i2) || (i1 == i2 && j1 < j2);
}

__device__ __forceinline__ void warp_argmin(double& best, int& bi, int& bj) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double d2 = __shfl_xor_sync(0xffffffffu, best, o);
    int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    int j2 = __shfl_xor_sync(0xffffffffu, bj, o);
    if (res_less(d2, i2, j2, best, bi, bj)) {
      best = d2;
      bi = i2;
      bj = j2;
    }
  }
}

// Row ring: lane 0 issues bulk copies; all lanes wait on the mbarriers.
template <typename T>
struct RowRing {
  unsigned char* base;
  uint64_t* bars;
  uint32_t row_bytes, stride;
  const T* mat;
  int64_t ld;
  const uint16_t* tour;
  int r0, nrows;

  __device__ void start() {
    if ((threadIdx.x & 31) == 0) {
      for (int b = 0; b < kBufs; ++b) mbar_init(&bars[b], 1);
      fence_barrier_init();
      for (int q = 0; q < 2 && q < nrows; ++q) issue(q);
    }
    __syncwarp();
  }
  __device__ void issue(int q) {
    const int b = q % kBufs;
    const int node = tour[r0 + q];
    mbar_expect_tx(&bars[b], row_bytes);
    bulk_g2s(base + (size_t)b * stride, mat + (size_t)node * ld, row_bytes,
             &bars[b]);
  }
  // rows q (A) and q+1 (B) ready; row q+2 requested
  __device__ void advance(int q, const T** A, const T** B) {
    if ((threadIdx.x & 31) == 0 && q + 2 < nrows) {
      fence_proxy_async();
      issue(q + 2);
    }
    const int ba = q % kBufs, bb = (q + 1) % kBufs;
    mbar_wait(&bars[ba], (uint32_t)((q / kBufs) & 1));
    mbar_wait(&bars[bb], (uint32_t)(((q + 1) / kBufs) & 1));
    *A = (const T*)(base + (size_t)ba * stride);
    *B = (const T*)(base + (size_t)bb * stride);
  }
};

// ---- FP64 scan (reference arithmetic on fp64 rows) -------------------------
// NPL > 0: lane-owned columns in registers (n <= 32*NPL); NPL == 0: columns
// read from global/L1 per row.  STAGE: rows in the smem ring (false = read
// the rows straight from global/L2, for n too large for the ring).
template <int NPL, bool STAGE>
__global__ void __launch_bounds__(kMaxWarps * 32)
    k_two_opt_scan64(ScanArgs a) {
  if (a.ctl && (a.ctl->done || a.ctl->improved)) return;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[kMaxWarps][kBufs];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int task = blockIdx.x * (blockDim.x >> 5) + warp;
  const int p = task / a.chunks, c = task % a.chunks;
  if (p >= a.count) return;
  const int n = a.n;
  const int r0 = a.chunk_row[c], r1 = a.chunk_row[c + 1];
  TwoOptRes* out = a.res + (size_t)p * a.chunks + c;
  if (a.only_flagged && out->i != kOverflowTag) return;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  if (r0 >= r1) {
    if (lane == 0) *out = {kInf, 0x7fffffff, 0x7fffffff};
    return;
  }
  const uint16_t* tour = a.tours + (size_t)p * a.np;
  const double* dg = a.dcache + (size_t)p * a.np;

  constexpr int NR = NPL > 0 ? NPL : 1;
  uint32_t pk[NR];
  double dj[NR];
  if (NPL > 0) {
#pragma unroll
    for (int m = 0; m < NR; ++m) {
      int j = lane + 32 * m;
      if (j < n) {
        uint32_t aj = tour[j], sj = tour[j + 1 == n ? 0 : j + 1];
        pk[m] = aj | (sj << 16);
        dj[m] = dg[j];
      } else {
        pk[m] = 0;
        dj[m] = 0.0;
      }
    }
  }
  RowRing<double> ring{smem + (size_t)warp * kBufs * a.buf_stride,
                       bars[warp], a.row_bytes, a.buf_stride, a.cost, a.ld,
                       tour, r0, r1 - r0 + 1};
  if (STAGE) ring.start();

  double best = kInf;
  int bi = 0x7fffffff, bj = 0x7fffffff;
  for (int i = r0; i < r1; ++i) {
    const double* A;
    const double* B;
    if (STAGE) {
      ring.advance(i - r0, &A, &B);
    } else {
      A = a.cost + (size_t)tour[i] * a.ld;
      B = a.cost + (size_t)tour[i + 1] * a.ld;
    }
    const double di = dg[i];
    double rbest = kInf;
    int rj = 0x7fffffff;
    if (NPL > 0) {
#pragma unroll
      for (int m0 = 0; m0 < NR; m0 += kGroup) {
        if (32 * (m0 + kGroup) - 1 > i) {  // warp-uniform: group not dead
          double av[kGroup], bv[kGroup];
#pragma unroll
          for (int g = 0; g < kGroup; ++g) {
            if (m0 + g < NR) {
              av[g] = A[pk[m0 + g] & 0xFFFFu];
              bv[g] = B[pk[m0 + g] >> 16];
            }
          }
#pragma unroll
          for (int g = 0; g < kGroup; ++g) {
            if (m0 + g < NR) {
              const int j = lane + 32 * (m0 + g);
              double t = __dadd_rn(av[g], bv[g]);
              t = __dsub_rn(t, di);
              t = __dsub_rn(t, dj[m0 + g]);
              t = (j > i && j < n) ? t : kInf;
              const bool lt = t < rbest;
              rbest = lt ? t : rbest;
              rj = lt ? j : rj;
            }
          }
        }
      }
    } else {
      for (int j = i + 1 + lane; j < n; j += 32) {
        const int aj = tour[j], sj = tour[j + 1 == n ? 0 : j + 1];
        double t = __dadd_rn(A[aj], B[sj]);
        t = __dsub_rn(t, di);
        t = __dsub_rn(t, dg[j]);
        const bool lt = t < rbest;
        rbest = lt ? t : rbest;
        rj = lt ? j : rj;
      }
    }
    if (rbest < best) {
      best = rbest;
      bi = i;
      bj = rj;
    }
    __syncwarp();
  }
  warp_argmin(best, bi, bj);
  if (lane == 0) *out = {best, bi, bj};
}

// ---- FP32 scan: EXACT32 (MODE 1) and FILTER32 (MODE 2) ---------------------
// FILTER32 candidate bookkeeping, out of line (rarely taken; keeping it out
// of the unrolled column loop keeps the kernel inside the instruction cache).
// Per lane state lives in shared memory (stride 32 between words): st[0] =
// running fp32 minimum, st[32] = candidate count, st[64] = overflow flag; cd/cij are this lane's
// candidate slots (stride 32).  Returns the new window limit.
__device__ __noinline__ float cand_group(float t0, float t1, float t2,
                                         float t3, int i, int j0, int jstep,
                                         float lim, float thr, float* cd,
                                         uint32_t* cij, float* st) {
  float best = st[0];
  int ncand = __float_as_int(st[32]);
  int overflow = __float_as_int(st[64]);
  const float tv[4] = {t0, t1, t2, t3};
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const float t = tv[g];
    if (t <= lim) {
      if (t < best) {
        best = t;
        lim = __fadd_ru(t, thr);
        int w = 0;
        for (int k = 0; k < ncand; ++k) {
          const float d = cd[32 * k];
          if (d <= lim) {
            cd[32 * w] = d;
            cij[32 * w] = cij[32 * k];
            ++w;
          }
        }
        ncand = w;
      }
      if (ncand < kCand) {
        cd[32 * ncand] = t;
        cij[32 * ncand] = ((uint32_t)i << 16) | (uint32_t)(j0 + jstep * g);
        ++ncand;
      } else {
        overflow = 1;
      }
    }
  }
  st[0] = best;
  st[32] = __int_as_float(ncand);
  st[64] = __int_as_float(overflow);
  return lim;
}

// One warp per task; lane l owns the columns j = l + 32m (m < NPL).
// Shift-reuse: the A term of pair (i+1, j) is C[a_{i+1}][a_j], which is the
// B term lane l-1 gathered for pair (i, j-1) (lane 0: lane 31 of block m-1),
// so it arrives by ONE warp rotate and each row costs ONE random
// shared-memory gather per pair; the first row of a task is primed by a
// B-gather of row a_r0.  Per lane in registers: the gathered B values and
// the gather indices s_j (two u16 per register); d_j sits in shared memory
// (lane-contiguous, conflict free).  Rows a_r0..a_r1 stream through a
// per-warp 3-slot ring, two rows ahead.  In fp32 modes the order of the
// three adds is free (EXACT32 sums are exact; FILTER32 is bounded).
constexpr int kBufs32 = 2;  // fp32 per-warp ring depth (one row ahead)
constexpr int kG32 = 8;     // column blocks per uniform group (fp32 scan)

template <int NPL, int MODE>
__global__ void __launch_bounds__(kMaxWarps * 32, 4)
    k_two_opt_scan32(ScanArgs a) {
  if (a.ctl && (a.ctl->done || a.ctl->improved)) return;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[kMaxWarps][kBufs32];
  __shared__ uint32_t s_cij[kMaxWarps][kCand][32];
  __shared__ float s_cd[kMaxWarps][kCand][32];
  __shared__ float s_st[kMaxWarps][3][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int task = blockIdx.x * (blockDim.x >> 5) + warp;
  const int p = task / a.chunks, c = task % a.chunks;
  if (p >= a.count) return;
  const int n = a.n;
  const int r0 = a.chunk_row[c], r1 = a.chunk_row[c + 1];
  TwoOptRes* out = a.res + (size_t)p * a.chunks + c;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const float kInfF = __int_as_float(0x7f800000);
  if (MODE == 2) {
    s_st[warp][0][lane] = kInfF;
    s_st[warp][1][lane] = __int_as_float(0);
    s_st[warp][2][lane] = __int_as_float(0);
  }
  if (r0 >= r1) {
    if (lane == 0) *out = {kInf, 0x7fffffff, 0x7fffffff};
    return;
  }
  const uint16_t* tour = a.tours + (size_t)p * a.np;
  const double* dg = a.dcache + (size_t)p * a.np;
  // FILTER32 excludes the structural pairs (i, i+1) (and (0, n-1) below)
  constexpr int kGap = MODE == 2 ? 1 : 0;
  unsigned char* wbase = smem + (size_t)warp * a.buf_stride2;
  float* sdj = (float*)(wbase + kBufs32 * a.buf_stride);  // d_j, fp32

  constexpr int NH = (NPL + 1) / 2;
  uint32_t sjp[NH];  // s_j = a_{j+1} for blocks 2h (lo) and 2h+1 (hi)
#pragma unroll
  for (int h = 0; h < NH; ++h) sjp[h] = 0;
#pragma unroll
  for (int m = 0; m < NPL; ++m) {
    const int j = lane + 32 * m;
    if (j < n) {
      const uint32_t s_ = tour[j + 1 == n ? 0 : j + 1];
      sjp[m / 2] |= (m & 1) ? (s_ << 16) : s_;
    }
  }
  for (int j = lane; j < 32 * NPL; j += 32)
    sdj[j] = j < n ? (float)dg[j] : 0.f;
  auto sj = [&](int m) -> uint32_t {
    return (m & 1) ? (sjp[m / 2] >> 16) : (sjp[m / 2] & 0xFFFFu);
  };
  const int nrows = r1 - r0 + 1;  // cost rows a_r0 .. a_r1
  uint64_t* wb = bars[warp];
  auto issue = [&](int q) {
    const int s_ = q % kBufs32;
    mbar_expect_tx(&wb[s_], a.row_bytes);
    bulk_g2s(wbase + (size_t)s_ * a.buf_stride,
             a.cost32 + (size_t)tour[r0 + q] * a.ld32, a.row_bytes, &wb[s_]);
  };
  if (lane == 0) {
    for (int s_ = 0; s_ < kBufs32; ++s_) mbar_init(&wb[s_], 1);
    fence_barrier_init();
    for (int q = 0; q < kBufs32 && q < nrows; ++q) issue(q);
  }
  __syncwarp();
  auto row = [&](int q) -> const float* {
    const int s_ = q % kBufs32;
    mbar_wait(&wb[s_], (uint32_t)((q / kBufs32) & 1));
    return (const float*)(wbase + (size_t)s_ * a.buf_stride);
  };
  // prime: Bv = row a_r0 gathered at s_j (the "B term of row r0 - 1")
  float Bv[NPL];
  {
    const float* R = row(0);
#pragma unroll
    for (int m = 0; m < NPL; ++m) Bv[m] = R[sj(m)];
  }

  float best = kInfF;
  int bi = 0x7fffffff, bj = 0x7fffffff;
  float lim = FLT_MAX;  // FILTER32: best + thr (finite: masked +inf never enters)
  for (int i = r0; i < r1; ++i) {
    const int q = i - r0 + 1;  // ring index of the B row a_{i+1}
    __syncwarp();
    if (lane == 0 && q + kBufs32 - 1 < nrows) {
      fence_proxy_async();
      issue(q + kBufs32 - 1);  // the slot of row q-1, consumed last iteration
    }
    const float* B = row(q);
    if (a.stream_only) {
      if (lane == 0 && B[0] == -1.f) bi = i;  // keep the load
      continue;
    }
    const float di = (float)dg[i];
    const int jlim = (MODE == 2 && i == 0) ? n - 1 : n;
    float rbest = kInfF;
    int rj = 0x7fffffff;
    float rprev = 0.f;  // rotate of the previous block (lane 0's A term)
#pragma unroll
    for (int m0 = 0; m0 < NPL; m0 += kG32) {
      if (32 * (m0 + kG32) - 1 > i + kGap) {  // warp-uniform: group not dead
        if (m0 > 0 && !(32 * m0 - 1 > i + kGap))  // previous group was dead
          rprev = __shfl_sync(0xffffffffu, Bv[m0 - 1], (lane + 31) & 31);
        // fully live group: every column j > i + gap and < jlim (only the
        // last block can reach n; row 0 also excludes (0, n-1) in FILTER32)
        const bool full = (32 * m0 > i + kGap) && (m0 + kG32 < NPL) &&
                          !(MODE == 2 && i == 0);
        float tv[kG32];
#pragma unroll
        for (int g = 0; g < kG32; ++g) {
          tv[g] = kInfF;
          if (m0 + g < NPL) {
            const int m = m0 + g;
            const float r = __shfl_sync(0xffffffffu, Bv[m], (lane + 31) & 31);
            const float av = lane == 0 ? rprev : r;
            rprev = r;
            const float bv = B[sj(m)];
            Bv[m] = bv;
            const int j = lane + 32 * m;
            float t = __fadd_rn(__fsub_rn(av, di), __fsub_rn(bv, sdj[j]));
            if (!full) t = (j > i + kGap && j < jlim) ? t : kInfF;
            tv[g] = t;
          }
        }
        if (MODE == 1) {
#pragma unroll
          for (int g = 0; g < kG32; ++g) {
            const bool lt = tv[g] < rbest;
            rbest = lt ? tv[g] : rbest;
            rj = lt ? lane + 32 * (m0 + g) : rj;
          }
        } else {
#pragma unroll
          for (int g4 = 0; g4 < kG32; g4 += 4) {
            bool hit = false;
#pragma unroll
            for (int g = 0; g < 4; ++g) hit |= tv[g4 + g] <= lim;
            if (hit)
              lim = cand_group(tv[g4], tv[g4 + 1], tv[g4 + 2], tv[g4 + 3], i,
                               lane + 32 * (m0 + g4), 32, lim, a.thr,
                               &s_cd[warp][0][lane], &s_cij[warp][0][lane],
                               &s_st[warp][0][lane]);
          }
        }
      }
    }
    if (MODE == 1 && rbest < best) {
      best = rbest;
      bi = i;
      bj = rj;
    }
  }
  __syncwarp();
  if (MODE == 1) {
    double bd = best == kInfF ? kInf : (double)best;
    warp_argmin(bd, bi, bj);
    if (lane == 0) *out = {bd, bi, bj};
    return;
  }
  // FILTER32: warp minimum, candidate re-evaluation in fp64
  best = s_st[warp][0][lane];
  const int ncand = __float_as_int(s_st[warp][1][lane]);
  if (__any_sync(0xffffffffu, __float_as_int(s_st[warp][2][lane]))) {
    if (lane == 0) *out = {kInf, kOverflowTag, kOverflowTag};
    return;
  }
  float m = best;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float keep = __fadd_ru(m, a.thr);
  double bd = kInf;
  int ei = 0x7fffffff, ej = 0x7fffffff;
  for (int k = 0; k < ncand; ++k) {
    if (s_cd[warp][k][lane] <= keep) {
      const uint32_t ij = s_cij[warp][k][lane];
      const int i = (int)(ij >> 16), j = (int)(ij & 0xFFFFu);
      const int ai = tour[i], aj = tour[j];
      const int si = tour[i + 1], sjj = tour[j + 1 == n ? 0 : j + 1];
      double t = __dadd_rn(a.cost[(size_t)ai * a.ld + aj],
                           a.cost[(size_t)si * a.ld + sjj]);
      t = __dsub_rn(t, dg[i]);
      t = __dsub_rn(t, dg[j]);
      if (res_less(t, i, j, bd, ei, ej)) {
        bd = t;
        ei = i;
        ej = j;
      }
    }
  }
  // structural pairs, exact from d: (i, i+1) has A = d_i, B = d_{i+1}
  for (int i = r0 + lane; i < r1; i += 32) {
    if (i + 1 < n) {
      const double d0 = dg[i], d1 = dg[i + 1];
      double t = __dadd_rn(d0, d1);
      t = __dsub_rn(t, d0);
      t = __dsub_rn(t, d1);
      if (res_less(t, i, i + 1, bd, ei, ej)) {
        bd = t;
        ei = i;
        ej = i + 1;
      }
    }
  }
  if (r0 == 0 && lane == 0 && n - 1 > 1) {  // (0, n-1): s_{n-1} = a_0
    const int j = n - 1;
    const int a0 = tour[0], aj = tour[j], s0 = tour[1], sjj = tour[0];
    double t = __dadd_rn(a.cost[(size_t)a0 * a.ld + aj],
                         a.cost[(size_t)s0 * a.ld + sjj]);
    t = __dsub_rn(t, dg[0]);
    t = __dsub_rn(t, dg[j]);
    if (res_less(t, 0, j, bd, ei, ej)) {
      bd = t;
      ei = 0;
      ej = j;
    }
  }
  warp_argmin(bd, ei, ej);
  if (lane == 0) *out = {bd, ei, ej};
}

struct ApplyArgs {
  int32_t n, np, count, chunks;
  uint16_t* tours;
  const TwoOptRes* res;
  double* fit;      // nullable
  double* pfit;     // nullable
  uint16_t* pbest;  // nullable
  double* delta_out;  // nullable
  const DevCtl* ctl;  // nullable
  const double* cost;  // non-null: refresh dcache after the move
  int64_t ld;
  double* dcache;
};

__global__ void __launch_bounds__(128) k_two_opt_apply(ApplyArgs a) {
  if (a.ctl && (a.ctl->done || a.ctl->improved)) return;
  const int p = blockIdx.x;
  if (p >= a.count) return;
  __shared__ int s_move[3];
  __shared__ double s_delta;
  __shared__ int s_better;
  const int tid = threadIdx.x;
  if (tid == 0) {
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int bi = 0x7fffffff, bj = 0x7fffffff;
    const TwoOptRes* r = a.res + (size_t)p * a.chunks;
    for (int c = 0; c < a.chunks; ++c)
      if (res_less(r[c].delta, r[c].i, r[c].j, best, bi, bj)) {
        best = r[c].delta;
        bi = r[c].i;
        bj = r[c].j;
      }
    int move = (a.n >= 4) && (best < -1e-12);
    s_move[0] = move;
    s_move[1] = bi;
    s_move[2] = bj;
    s_delta = move ? best : 0.0;
    if (a.delta_out) a.delta_out[p] = s_delta;
  }
  __syncthreads();
  if (!s_move[0]) return;
  const int i = s_move[1], j = s_move[2];
  uint16_t* t = a.tours + (size_t)p * a.np;
  const int len = j - i;  // reverse t[i+1 .. j]
  for (int u = tid; u < len / 2; u += blockDim.x) {
    uint16_t x = t[i + 1 + u];
    t[i + 1 + u] = t[j - u];
    t[j - u] = x;
  }
  __syncthreads();
  if (a.cost) {
    for (int k = i + tid; k <= j && k < a.n; k += blockDim.x) {
      int u = t[k], w = t[k + 1 == a.n ? 0 : k + 1];
      a.dcache[(size_t)p * a.np + k] = a.cost[(size_t)u * a.ld + w];
    }
  }
  if (a.fit) {
    if (tid == 0) {
      double f = __dadd_rn(a.fit[p], s_delta);
      a.fit[p] = f;
      s_better = f < a.pfit[p];
      if (s_better) a.pfit[p] = f;
    }
    __syncthreads();
    if (s_better) {
      uint16_t* pb = a.pbest + (size_t)p * a.np;
      for (int u = tid; u < a.n; u += blockDim.x) pb[u] = t[u];
    }
  }
}

// ---- cost-matrix preparation ------------------------------------------------
// fp32 copy + statistics: max |C| (as the bits of a non-negative double,
// which order like the values) and whether every entry is an integer.
__global__ void k_cost_prep(const double* cost, int64_t ld, int n,
                            float* cost32, int64_t ld32, CostStats* st) {
  unsigned long long mx = 0;
  int nonint = 0;
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n, c = e % n;
    const double v = cost[r * ld + c];
    cost32[r * ld32 + c] = (float)v;
    const unsigned long long b =
        (unsigned long long)__double_as_longlong(fabs(v));
    mx = b > mx ? b : mx;
    nonint |= (v != rint(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long m2 = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = m2 > mx ? m2 : mx;
    nonint |= __shfl_xor_sync(0xffffffffu, nonint, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&st->maxabs_bits, mx);
    if (nonint) atomicOr(&st->nonintegral, 1);
  }
}

template <int NPL, bool STAGE>
cudaError_t launch_scan64_t(const ScanArgs& a, int warps, int blocks,
                            size_t smem, cudaStream_t s) {
  auto k = k_two_opt_scan64<NPL, STAGE>;
  cudaError_t e = set_dyn_smem((const void*)k, smem);
  if (e != cudaSuccess) return e;
  k<<<blocks, warps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <int NPL, int MODE>
cudaError_t launch_scan32_t(const ScanArgs& a, int warps, int blocks,
                            size_t smem, cudaStream_t s) {
  auto k = k_two_opt_scan32<NPL, MODE>;
  cudaError_t e = set_dyn_smem((const void*)k, smem);
  if (e != cudaSuccess) return e;
  k<<<blocks, warps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

// bytes of one warp's row ring for element size `es`
size_t ring_bytes(int n, int es) {
  return (size_t)kBufs * round_up((int64_t)round_up(n, 16 / es) * es, 128);
}

constexpr size_t kSmemBudget = 200 * 1024;

int npl_for(int n) {
  if (n <= 32) return 1;
  if (n <= 64) return 2;
  if (n <= 128) return 4;
  if (n <= 256) return 8;
  if (n <= 512) return 16;
  if (n <= 1024) return 32;
  if (n <= 2048) return 64;
  return 0;
}

}  // namespace

int two_opt_mode(const CostStats& st, int n, float* thr) {
  double mx;
  memcpy(&mx, &st.maxabs_bits, sizeof mx);
  *thr = 0.f;
  if (npl_for(n) == 0) return kScanFP64;  // register layout needs n <= 2048
  if (!(mx < 1e30)) return kScanFP64;     // fp32 range
  if (!st.nonintegral && mx < 4194304.0) return kScanExact32;  // 2^22
  if (mx < 1e-30) return kScanFP64;       // fp32 subnormal range
  // eps = 2^-18 max|C| (>= 4x the worst-case fp32 rounding of a delta);
  // candidates within 2 eps of the fp32 minimum are re-evaluated in fp64.
  *thr = (float)(mx * (2.0 / 262144.0));
  return kScanFilter32;
}

cudaError_t launch_cost_prep(const double* cost, int64_t ld, int32_t n,
                             float* cost32, int64_t ld32, CostStats* st,
                             cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(st, 0, sizeof(CostStats), s);
  if (e) return e;
  const int64_t total = (int64_t)n * n;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (blocks < 1) blocks = 1;
  k_cost_prep<<<blocks, 256, 0, s>>>(cost, ld, n, cost32, ld32, st);
  return cudaGetLastError();
}

int two_opt_pick_chunks(int32_t n, int32_t P) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // fp32 scan: one warp per task (row ring + d_j in shared memory)
  size_t per_warp = (size_t)kBufs32 * round_up((int64_t)round_up(n, 4) * 4, 128) +
                    4 * (size_t)round_up(n, 32);
  int warps_per_sm = (int)(kSmemBudget / per_warp);
  if (warps_per_sm < 1) warps_per_sm = 1;
  if (warps_per_sm > 16) warps_per_sm = 16;
  int64_t slots = (int64_t)sms * warps_per_sm;
  int chunks = (int)((4 * slots + P - 1) / P);
  if (chunks < 1) chunks = 1;
  if (chunks > 32) chunks = 32;
  if (chunks > n / 8 + 1) chunks = n / 8 + 1;
  return chunks;
}

// Split pair rows 0..n-2 into `chunks` bands of roughly equal pair count.
int two_opt_chunk_rows(int32_t n, int32_t chunks, int32_t* rows) {
  const int last = n - 1;  // pair rows are 0 .. n-2
  const double total = 0.5 * (double)(n - 1) * n;
  rows[0] = 0;
  int r = 0;
  double acc = 0.0;
  for (int c = 1; c < chunks; ++c) {
    const double target = total * c / chunks;
    while (r < last && acc + (n - 1 - r) <= target) {
      acc += n - 1 - r;
      ++r;
    }
    rows[c] = r;
  }
  rows[chunks] = last > 0 ? last : 0;
  for (int c = 1; c <= chunks; ++c)
    if (rows[c] < rows[c - 1]) rows[c] = rows[c - 1];
  return 0;
}

cudaError_t launch_two_opt_core(const TwoOptPlan& pl, int32_t n, int32_t np,
                                uint16_t* tours, const double* dcache,
                                int32_t count, TwoOptRes* res, int32_t chunks,
                                const int32_t* chunk_row, const DevCtl* ctl,
                                double* fit, double* pfit, uint16_t* pbest,
                                double* delta_out, double* dcache_rw,
                                cudaStream_t s, int parts) {
  ScanArgs a;
  memset(&a, 0, sizeof a);
  a.cost = pl.cost;
  a.ld = pl.ld;
  a.cost32 = pl.cost32;
  a.ld32 = pl.ld32;
  a.n = n;
  a.np = np;
  a.count = count;
  a.chunks = chunks;
  a.tours = tours;
  a.dcache = dcache;
  a.chunk_row = chunk_row;
  a.res = res;
  a.ctl = ctl;
  a.thr = pl.thr;
  a.stream_only = getenv("DPSO_SCAN_STREAM_ONLY") ? 1 : 0;
  const int64_t tasks = (int64_t)count * chunks;
  cudaError_t e = cudaSuccess;
  const int npl = npl_for(n);
  auto fp64_scan = [&](int only_flagged) -> cudaError_t {
    a.only_flagged = only_flagged;
    a.row_bytes = (uint32_t)(round_up(n, 2) * 8);
    a.buf_stride = (uint32_t)round_up(a.row_bytes, 128);
    const size_t per_warp = ring_bytes(n, 8);
    const bool stage = per_warp <= kSmemBudget;
    const int warps =
        stage ? (int)std::min<size_t>(kMaxWarps, kSmemBudget / per_warp)
              : kMaxWarps;
    const size_t smem = stage ? (size_t)warps * per_warp : 0;
    const int blocks = (int)((tasks + warps - 1) / warps);
#define SCAN64(NPL)                                                 \
  (stage ? launch_scan64_t<NPL, true>(a, warps, blocks, smem, s)    \
         : launch_scan64_t<NPL, false>(a, warps, blocks, smem, s))
    switch (npl) {
      case 1: return SCAN64(1);
      case 2: return SCAN64(2);
      case 4: return SCAN64(4);
      case 8: return SCAN64(8);
      case 16: return SCAN64(16);
      case 32: return SCAN64(32);
      case 64: return SCAN64(64);
      default: return SCAN64(0);
    }
#undef SCAN64
  };
  if ((parts & 1) && n >= 4 && tasks > 0) {
    if (pl.mode == kScanFP64 || !pl.cost32) {
      e = fp64_scan(0);
    } else {
      a.row_bytes = (uint32_t)(round_up(n, 4) * 4);
      a.buf_stride = (uint32_t)round_up(a.row_bytes, 128);
      // per warp: 2-slot row ring + d_j (fp32, 32 * NPL entries)
      a.buf_stride2 = (uint32_t)(kBufs32 * a.buf_stride +
                                 round_up((int64_t)32 * std::max(npl, 1) * 4,
                                          128));
      const int warps = kMaxWarps;
      const size_t smem = (size_t)warps * a.buf_stride2;
      const int blocks = (int)((tasks + warps - 1) / warps);
#define SCAN32(NPL)                                                        \
  (pl.mode == kScanExact32                                                 \
       ? launch_scan32_t<NPL, 1>(a, warps, blocks, smem, s)                \
       : launch_scan32_t<NPL, 2>(a, warps, blocks, smem, s))
      switch (npl) {
        case 1: e = SCAN32(1); break;
        case 2: e = SCAN32(2); break;
        case 4: e = SCAN32(4); break;
        case 8: e = SCAN32(8); break;
        case 16: e = SCAN32(16); break;
        case 32: e = SCAN32(32); break;
        default: e = SCAN32(64); break;
      }
#undef SCAN32
      // FILTER32 candidate-list overflow: exact fp64 re-scan of those tasks
      if (!e && pl.mode == kScanFilter32) e = fp64_scan(1);
    }
    if (e != cudaSuccess) return e;
  }
  if (!(parts & 2)) return cudaSuccess;
  ApplyArgs b;
  b.n = n;
  b.np = np;
  b.count = count;
  b.chunks = chunks;
  b.tours = tours;
  b.res = res;
  b.fit = fit;
  b.pfit = pfit;
  b.pbest = pbest;
  b.delta_out = delta_out;
  b.ctl = ctl;
  b.cost = dcache_rw ? pl.cost : nullptr;
  b.ld = pl.ld;
  b.dcache = dcache_rw;
  if (n < 4) {
    // _best_exchange returns (body, 0.0) for n < 4 (solver.py:91-93)
    if (delta_out) cudaMemsetAsync(delta_out, 0, sizeof(double) * count, s);
    return cudaGetLastError();
  }
  if (count > 0) k_two_opt_apply<<<count, 128, 0, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_two_opt(const SwarmView& v, cudaStream_t s, int parts) {
  return launch_two_opt_core(v.plan, v.n, v.np, v.x, v.dcache, v.P, v.tores,
                             v.chunks, v.chunk_row, v.ctl, v.fit, v.pfit,
                             v.pbest, nullptr, nullptr, s, parts);
}

cudaError_t launch_two_opt_batch(const TwoOptPlan& pl, int32_t n, int32_t np,
                                 uint16_t* tours, const double* dcache,
                                 int32_t count, TwoOptRes* res, int32_t chunks,
                                 const int32_t* chunk_row, double* delta_out,
                                 cudaStream_t s) {
  return launch_two_opt_core(pl, n, np, tours, dcache, count, res, chunks,
                             chunk_row, nullptr, nullptr, nullptr, nullptr,
                             delta_out, const_cast<double*>(dcache), s, 3);
}

}  // namespace dpso
