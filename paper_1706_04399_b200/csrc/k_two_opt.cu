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

#include <stdio.h>

#include <algorithm>
#include <vector>

#include <cuda_fp16.h>
#include <math.h>

#include "dpso_internal.cuh"
#include "tma.cuh"

namespace dpso {

namespace {

constexpr int kMaxWarps = 4;  // warps (tasks) per CTA, upper bound
constexpr int kBufs = 3;      // row ring depth per warp
constexpr int kGroup = 4;     // column blocks (of 32) per uniform skip test
constexpr int kCand = 4;      // fp32 candidates kept per lane (FILTER32)
constexpr int kOverflowTag = -2;
constexpr int kAppliedTag = -3;  // the bounded scan applied the move itself

struct ScanArgs {
  const double* cost;
  int64_t ld;
  const float* cost32;
  int64_t ld32;
  int32_t n, np, count, chunks;
  const uint16_t* tours;   // count x np
  const double* dcache;    // count x np
  const int32_t* chunk_tab;  // chunks x (r0, r1, jlo, jhi)
  TwoOptRes* res;          // count x chunks
  const DevCtl* ctl;       // nullable: skip when done or improved
  uint32_t row_bytes;      // bytes streamed per cost row (multiple of 16)
  uint32_t buf_stride;     // bytes between ring buffers
  uint32_t buf_stride2;    // bytes of one warp's smem (ring + d_j)
  float thr;               // FILTER32: 2 * eps (row units)
  const void* rows;        // staged rows of the fp32 scan: cost32 or cost16
  int64_t row_pitch;       // bytes between staged rows
  float dscale;            // d values -> row units (power of two)
  double vfrom, vto;       // capped virtual level (TwoOptPlan), 0: none
  int32_t* ovf;            // FILTER32 overflow list: [0] count, [1..] tasks
  int32_t* task_ctr;       // fp32 scan: next task (persistent warps)
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
  const int4 tb = reinterpret_cast<const int4*>(a.chunk_tab)[c];
  const int r0 = tb.x, r1 = tb.y, jlo = tb.z, jhi = tb.w;
  TwoOptRes* out = a.res + (size_t)p * a.chunks + c;
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
        if (32 * (m0 + kGroup) - 1 > i && 32 * m0 < jhi &&
            32 * (m0 + kGroup) > jlo) {  // warp-uniform: group not dead
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
              t = (j > i && j >= jlo && j < jhi) ? t : kInf;
              const bool lt = t < rbest;
              rbest = lt ? t : rbest;
              rj = lt ? j : rj;
            }
          }
        }
      }
    } else {
      for (int j = max(i + 1, jlo) + lane; j < jhi; j += 32) {
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

// FILTER32 candidate-list overflow: the listed tasks re-scanned exactly in
// fp64 with the reference expression, rows straight from L2, one warp per
// listed task (grid-stride; a no-op when the list is empty).
__global__ void __launch_bounds__(128) k_two_opt_rescan64(ScanArgs a) {
  if (a.ctl && (a.ctl->done || a.ctl->improved)) return;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int cnt = a.ovf[0];
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const int n = a.n;
  for (int t = gw; t < cnt; t += nw) {
    const int task = a.ovf[1 + t];
    const int p = task / a.chunks, c = task % a.chunks;
    const int4 tb = reinterpret_cast<const int4*>(a.chunk_tab)[c];
    const int r0 = tb.x, r1 = tb.y, jlo = tb.z, jhi = tb.w;
    const uint16_t* tour = a.tours + (size_t)p * a.np;
    const double* dg = a.dcache + (size_t)p * a.np;
    double best = kInf;
    int bi = 0x7fffffff, bj = 0x7fffffff;
    for (int i = r0; i < r1; ++i) {
      const double* A = a.cost + (size_t)tour[i] * a.ld;
      const double* B = a.cost + (size_t)tour[i + 1] * a.ld;
      const double di = dg[i];
      for (int j = max(i + 1, jlo) + lane; j < jhi; j += 32) {
        const int aj = tour[j], sj = tour[j + 1 == n ? 0 : j + 1];
        double v = __dadd_rn(A[aj], B[sj]);
        v = __dsub_rn(v, di);
        v = __dsub_rn(v, dg[j]);
        if (v < best) {  // lane order: (i, j) increasing, first strict min
          best = v;
          bi = i;
          bj = j;
        }
      }
    }
    warp_argmin(best, bi, bj);
    if (lane == 0) a.res[(size_t)p * a.chunks + c] = {best, bi, bj};
  }
}

// ---- FP32 scan: EXACT32 (MODE 1) and FILTER32 (MODE 2) ---------------------
// Two pair rows (i, i+1) per pass.  Per pair a lane computes
// u = A + (B - d_j); d_i is folded into a per-row threshold Lrow, and one
// warp-uniform pre-test per group of column blocks (min of the group's
// u per row against Lrow) is the only per-pair branch.  Hits (rare once the
// running minimum has settled) go to an out-of-line handler, which keeps
// the kernel inside the instruction cache and maintains a warp-wide
// running minimum:
//   EXACT32  Lrow = best + d_i (exact: |u|, |best + d_i| < 2^24).  The
//            handler keeps the lane's first minimum in (t, i, j) order
//            (lexicographic, since the pass interleaves the two rows); the
//            pre-test is non-strict for row i and strict for row i+1.  The
//            reference argmin, bit for bit.
//   FILTER32 Lrow = fl_ru(best + thr + d_i) (capped at FLT_MAX).  The
//            handler records every pair with u <= Lrow as a candidate and
//            tightens the window to the warp minimum + thr, ~10x inside the
//            rounding bound, so the fp64 argmin and its ties are candidates.
// The structural pairs (i, i+1) and (0, n-1) are exact no-ops: 0 in
// EXACT32 (they can only be the argmin when no move is applied), and
// evaluated exactly in fp64 at the end in FILTER32 - so the fp32 pass may
// skip or repeat them freely.
// Per-lane state in shared memory (stride 32 between words): st[0] = the
// running minimum t; EXACT32: st[32], st[64] = its i, j; FILTER32: st[32] =
// candidate count, st[64] = overflow flag, cd/cij = candidate slots.
constexpr int kBufs32 = 4;     // fp32 per-warp row ring (one pass ahead)
// column blocks per skip test and pre-test: 8 for full-width tasks (more
// independent work per pre-test), 4 for narrow ones (finer dead-group skip)
template <int NPL>
constexpr int group_blocks() { return NPL >= 32 ? 8 : 4; }
// column blocks per fp32 task: 32 (1024 columns) or, by DPSO_SCAN_NPL, 16
// or 8 (narrower tasks: fewer registers per thread, more warps per SM, each
// row streamed once per column range)
static int npl_max32() {
  static const int v = [] {
    const char* e = getenv("DPSO_SCAN_NPL");
    const int x = e ? atoi(e) : 32;
    return (x == 8 || x == 16) ? x : 32;
  }();
  return v;
}
constexpr int kW32 = 2;        // warps (tasks) per CTA, fp32 scan

__device__ __forceinline__ bool lex_less(float t, int i, int j, float bt,
                                         int bi, int bj) {
  return t < bt || (t == bt && (i < bi || (i == bi && j < bj)));
}

template <int MODE>
__device__ __noinline__ float scan_hit(float u0, float u1, float u2, float u3,
                                       float w0, float w1, float w2, float w3,
                                       float da, float db, float la, float lb,
                                       int i, int j0, int jstep, float thr,
                                       float* cd, uint32_t* cij, float* st) {
  // entered by the whole warp (the pre-test is warp-uniform): u = row i,
  // w = row i+1 of the same 4 column blocks; returns the warp-wide
  // threshold base (EXACT32: warp minimum; FILTER32: warp minimum + thr)
  const float uv[8] = {u0, u1, u2, u3, w0, w1, w2, w3};
  float best = st[0];
  if (MODE == 1) {
    int bi = __float_as_int(st[32]), bj = __float_as_int(st[64]);
    // lb == -inf: the pass has no row i+1 (its values are not pairs)
    const int gend = lb == -__int_as_float(0x7f800000) ? 4 : 8;
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      if (g >= gend) break;
      const int ii = i + (g >> 2), jj = j0 + jstep * (g & 3);
      const float t = __fsub_rn(uv[g], g < 4 ? da : db);  // exact
      if (lex_less(t, ii, jj, best, bi, bj)) {
        best = t;
        bi = ii;
        bj = jj;
      }
    }
    st[0] = best;
    st[32] = __int_as_float(bi);
    st[64] = __int_as_float(bj);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      best = fminf(best, __shfl_xor_sync(0xffffffffu, best, o));
    return best;
  }
  int ncand = __float_as_int(st[32]);
  int overflow = __float_as_int(st[64]);
  // the new values in the window, then the new warp minimum, then the list
  // against the tightened window (so transient entries never overflow it)
  float tv[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const bool in = uv[g] <= (g < 4 ? la : lb);
    tv[g] = in ? __fsub_rn(uv[g], g < 4 ? da : db)
               : __int_as_float(0x7f800000);
    best = fminf(best, tv[g]);
  }
  float wbest = best;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    wbest = fminf(wbest, __shfl_xor_sync(0xffffffffu, wbest, o));
  const float lim = wbest < FLT_MAX ? __fadd_ru(wbest, thr) : FLT_MAX;
  int w = 0;
  for (int k = 0; k < ncand; ++k) {
    const float dv = cd[32 * k];
    if (dv <= lim) {
      cd[32 * w] = dv;
      cij[32 * w] = cij[32 * k];
      ++w;
    }
  }
  ncand = w;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    if (tv[g] <= lim) {
      if (ncand < kCand) {
        cd[32 * ncand] = tv[g];
        cij[32 * ncand] = ((uint32_t)(i + (g >> 2)) << 16) |
                          (uint32_t)(j0 + jstep * (g & 3));
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

// One warp per task (particle, rows [r0, r1), columns [jlo, jhi)); lane l
// owns the columns j = jlo + l + 32m (m < NPL).
// Shift-reuse: the A term of pair (i+1, j) is C[a_{i+1}][a_j], which is the
// B term lane l-1 gathered for pair (i, j-1) (lane 0: lane 31 of block m-1;
// block 0 of a range with jlo > 0 gathers it once per row), so it arrives by
// ONE warp rotate.  A pass over rows (i, i+1) gathers both B rows at the
// same offsets 4 s_j (unpacked once) and subtracts the same d_j (loaded
// once): two gathers, two rotates, one d_j load per column block.  The
// offsets stay in registers (two u16 per register).  d_j sits in shared
// memory (lane-owned, conflict free) as fp32; a column that is dead for the
// rest of the task (j <= i, or past the range) holds -inf there, so its u
// is +inf with no per-pair mask: before the pass the owning lanes retire
// columns i and i+1.  Groups of 4-8 blocks with no live column are skipped
// (warp-uniform test).  Rows a_r0..a_r1 stream through a 4-slot per-warp
// ring, one pass (two rows) ahead.
#ifndef DPSO_SCAN_MINB
#define DPSO_SCAN_MINB 5
#endif
template <int NPL, int MODE, int ES, bool PERSIST>
__global__ void __launch_bounds__(kW32 * 32, DPSO_SCAN_MINB)
    k_two_opt_scan32(ScanArgs a) {
  if (a.ctl && (a.ctl->done || a.ctl->improved)) return;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[kW32][2];
  __shared__ uint32_t s_cij[kW32][kCand][32];
  __shared__ float s_cd[kW32][kCand][32];
  __shared__ float s_st[kW32][3][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* wb = bars[warp];
  if (lane == 0) {
    mbar_init(&wb[0], 1);
    mbar_init(&wb[1], 1);
    fence_barrier_init();
  }
  __syncwarp();
  uint32_t ph = 0;  // phase bit per pair (bit 0: pair 0, bit 1: pair 1)
  // Persistent warps: tasks are taken from a counter until none is left, so
  // the grid is one resident wave and the tail is at most one task per warp.
  // Every row a task issues is waited by the task itself, so the ring and
  // the barrier phases carry over cleanly.
  // (PERSIST false: one task per warp, task = global warp index - the
  // launch has a warp for every task; measured faster when each particle is
  // one task, C3)
  const int ntasks = a.count * a.chunks;
  for (int it = 0;; ++it) {
  __syncwarp();
  int task = 0;
  if (PERSIST) {
    if (lane == 0) task = atomicAdd(a.task_ctr, 1);
    task = __shfl_sync(0xffffffffu, task, 0);
  } else {
    if (it > 0) break;
    task = blockIdx.x * (blockDim.x >> 5) + warp;
  }
  if (task >= ntasks) break;
  const int p = task / a.chunks, c = task % a.chunks;
  const int n = a.n;
  const int4 tb = reinterpret_cast<const int4*>(a.chunk_tab)[c];
  const int r0 = tb.x, r1 = tb.y, jlo = tb.z, jhi = tb.w;
  TwoOptRes* out = a.res + (size_t)p * a.chunks + c;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const float kInfF = __int_as_float(0x7f800000);
  float* st = &s_st[warp][0][lane];
  st[0] = kInfF;
  st[32] = __int_as_float(MODE == 1 ? 0x7fffffff : 0);
  st[64] = __int_as_float(MODE == 1 ? 0x7fffffff : 0);
  if (r0 >= r1) {
    if (lane == 0) *out = {kInf, 0x7fffffff, 0x7fffffff};
    continue;
  }
  const uint16_t* tour = a.tours + (size_t)p * a.np;
  const double* dg = a.dcache + (size_t)p * a.np;
  unsigned char* wbase = smem + (size_t)warp * a.buf_stride2;
  float* sdj = (float*)(wbase + kBufs32 * a.buf_stride);  // local column

  // Column layout: groups of GL blocks (32 GL columns); inside a group lane l
  // owns the GL consecutive columns jlo + 32 GL g + GL l + (0 .. GL-1), so
  // the shift-reuse neighbour j - 1 of a column is the same lane's previous
  // block except at a group's first block (one rotate per group and row).
  constexpr int GL = group_blocks<NPL>() < NPL ? group_blocks<NPL>() : NPL;
  auto col_of = [&](int m) -> int {
    return jlo + 32 * GL * (m / GL) + GL * lane + (m % GL);
  };
  constexpr int NH = (NPL + 1) / 2;
  uint32_t sjp[NH];  // 4 s_j for blocks 2h (lo) and 2h+1 (hi)
#pragma unroll
  for (int h = 0; h < NH; ++h) sjp[h] = 0;
#pragma unroll
  for (int m = 0; m < NPL; ++m) {
    const int j = col_of(m);
    if (j < jhi) {
      const uint32_t s4 = (uint32_t)ES * tour[j + 1 == n ? 0 : j + 1];
      sjp[m / 2] |= (m & 1) ? (s4 << 16) : s4;
    }
  }
  // d_j of block m at sdj[lane + 32 m] (lane-interleaved: conflict free)
#pragma unroll
  for (int m = 0; m < NPL; ++m) {
    const int j = col_of(m);
    sdj[lane + 32 * m] =
        (j >= r0 && j < jhi)
            ? (float)((dg[j] == a.vfrom ? a.vto : dg[j]) * a.dscale)
            : -kInfF;
  }
  auto sdj_index = [&](int c) -> int {  // c = j - jlo
    const int grp = c / (32 * GL), within = c % (32 * GL);
    return (within / GL) + 32 * (GL * grp + within % GL);
  };
  auto sj = [&](int m) -> uint32_t {
    return (m & 1) ? (sjp[m / 2] >> 16) : (sjp[m / 2] & 0xFFFFu);
  };
  const int nrows = r1 - r0 + 1;  // cost rows a_r0 .. a_r1 (ring index q)
  // The ring is two slot pairs with one mbarrier each: a pass's two B rows
  // sit in one pair (B2 one slot after B1) and arrive on one barrier; the
  // next pass's rows fill the other pair.  The prime row a_r0 uses pair 1
  // before pass 1 refills it.
  auto issue2 = [&](int pair, int ca, int cb2, int nr) {  // nr rows: 1 or 2
    mbar_expect_tx(&wb[pair], (uint32_t)nr * a.row_bytes);
    unsigned char* dst = wbase + (size_t)(2 * pair) * a.buf_stride;
    const unsigned char* rows = (const unsigned char*)a.rows;
    bulk_g2s(dst, rows + (size_t)ca * a.row_pitch, a.row_bytes, &wb[pair]);
    if (nr > 1)
      bulk_g2s(dst + a.buf_stride, rows + (size_t)cb2 * a.row_pitch,
               a.row_bytes, &wb[pair]);
  };
  if (lane == 0) {
    issue2(1, tour[r0], 0, 1);                                 // prime row
    issue2(0, tour[r0 + 1], nrows > 2 ? tour[r0 + 2] : 0,      // pass 0
           nrows > 2 ? 2 : 1);
  }
  // Per-pass scalars from lane-parallel loads of 32 rows at a time, one
  // block ahead: cb = the cities of ring rows 3 + k (+1), db = d_{r0 + k}.
  auto city_at = [&](int q) -> int {
    return q < nrows ? (int)tour[r0 + q] : 0;
  };
  auto d_at = [&](int k) -> float {
    if (r0 + k >= r1) return 0.f;
    const double d = dg[r0 + k];
    return (float)((d == a.vfrom ? a.vto : d) * a.dscale);
  };
  int cb = city_at(3 + lane), cb_next = city_at(3 + 32 + lane);
  float db = d_at(lane), db_next = d_at(32 + lane);
  __syncwarp();
  // rows as 32-bit shared-window addresses: gathers are plain LDS [R]
  const uint32_t wbase_s = smem_u32(wbase);
  auto pair_rows = [&](int pair) -> uint32_t {  // waits; the pair's base
    mbar_wait(&wb[pair], (ph >> pair) & 1u);
    ph ^= 1u << pair;
    return wbase_s + (uint32_t)(2 * pair) * a.buf_stride;
  };
  auto at4 = [](uint32_t R, uint32_t off4) -> float {
    float v;
    if (ES == 4) {
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(R + off4));
    } else {  // fp16 row entry, widened exactly
      asm volatile(
          "{\n\t.reg .b16 h;\n\tld.shared.b16 h, [%1];\n\t"
          "cvt.f32.f16 %0, h;\n\t}"
          : "=f"(v)
          : "r"(R + off4));
    }
    return v;
  };
  // prime: Bv = row a_r0 gathered at s_j (the "B term of row r0 - 1"); for
  // jlo > 0 lane 0's A term of block 0 is C[a_i][a_jlo], gathered per row
  const uint32_t s4lo = jlo > 0 ? (uint32_t)ES * tour[jlo] : 0u;
  float Bv[NPL];
  float a0;
  {
    const uint32_t R = pair_rows(1);
#pragma unroll
    for (int m = 0; m < NPL; ++m) Bv[m] = at4(R, sj(m));
    a0 = at4(R, s4lo);
  }
  float lim = MODE == 1 ? kInfF : FLT_MAX;
  for (int i = r0; i < r1; i += 2) {
    const int k = i - r0;  // even
    const bool two = i + 1 < r1;
    if (k > 0 && (k & 31) == 0) {  // next block of per-pass scalars
      cb = cb_next;
      db = db_next;
      cb_next = city_at(3 + k + 32 + lane);
      db_next = d_at(k + 32 + lane);
    }
    const int pass = k >> 1;
    {  // rows k + 3, k + 4 into the other pair (read by the previous pass,
       // or the prime row; those shared loads have completed)
      const int c3 = __shfl_sync(0xffffffffu, cb, k & 31);
      const int c4 = __shfl_sync(0xffffffffu, cb, (k + 1) & 31);
      if (lane == 0 && k + 3 < nrows)
        issue2((pass + 1) & 1, c3, c4, k + 4 < nrows ? 2 : 1);
    }
    const float di = __shfl_sync(0xffffffffu, db, k & 31);
    const float di2 = __shfl_sync(0xffffffffu, db, (k + 1) & 31);
    {  // retire columns i and i + 1 (lane 0 writes both slots)
      const int c0 = i - jlo, c1 = i + 1 - jlo;
      if (lane == 0) {
        if (c0 >= 0 && c0 < 32 * NPL) sdj[sdj_index(c0)] = -kInfF;
        if (two && c1 >= 0 && c1 < 32 * NPL) sdj[sdj_index(c1)] = -kInfF;
      }
      __syncwarp();
    }
    const uint32_t B1 = pair_rows(pass & 1);
    const uint32_t B2 = two ? B1 + a.buf_stride : B1;
    if (a.stream_only == 1) {  // probe: the row stream alone
      if (lane == 0 && at4(B2, 0) == -1.f) lim = 0.f;  // keep the loads
      continue;
    }
    if (a.stream_only == 2) {  // probe: stream + the live groups' gathers
      constexpr int kGp = group_blocks<NPL>();
      float acc = kInfF;
#pragma unroll
      for (int m0 = 0; m0 < NPL; m0 += kGp) {
        if (jlo + 32 * (m0 + kGp) - 1 > i + 1) {
#pragma unroll
          for (int g = 0; g < kGp; ++g)
            if (m0 + g < NPL)
              acc = fminf(acc, at4(B1, sj(m0 + g)) + at4(B2, sj(m0 + g)));
        }
      }
      if (acc == -1.f) lim = 0.f;  // keep the loads
      continue;
    }
    auto lrow_of = [&](float d) -> float {
      return MODE == 1 ? __fadd_rn(lim, d) : fminf(__fadd_ru(lim, d), FLT_MAX);
    };
    float la = lrow_of(di);
    float lb = two ? lrow_of(di2) : -kInfF;
    float rp1 = a0;             // lane 0's A term of the next block, row i
    float rp2 = at4(B1, s4lo);  // ... row i + 1
    a0 = at4(B2, s4lo);         // row i + 2 (next pass)
    constexpr int kG32 = group_blocks<NPL>();
#pragma unroll
    for (int m0 = 0; m0 < NPL; m0 += kG32) {
      if (jlo + 32 * (m0 + kG32) - 1 > i + 1) {  // warp-uniform: live
        if (m0 > 0 && !(jlo + 32 * m0 - 1 > i + 1)) {  // previous skipped
          // lane 0's A terms: column c - 1 of the previous pass's B row
          // (still in Bv) and of B1, c = the group's first column
          rp1 = __shfl_sync(0xffffffffu, Bv[m0 - 1], 31);
          rp2 = at4(B1, __shfl_sync(0xffffffffu, sj(m0 - 1), 31));
        }
        float u[kG32], w[kG32], b1v[kG32], b2v[kG32];
#pragma unroll
        for (int g = 0; g < kG32; ++g) {
          const int m = m0 + g;
          if (m < NPL) {
            const uint32_t o = sj(m);
            b1v[g] = at4(B1, o);
            b2v[g] = at4(B2, o);
          }
        }
#pragma unroll
        for (int g = 0; g < kG32; ++g) {
          const int m = m0 + g;
          if (m < NPL) {
            const float dj = sdj[lane + 32 * m];
            float av1, av2;
            if (m % GL == 0) {
              // first block of a layout group: column j - 1 is lane l-1's
              // last block (lane 0: the previous group's lane 31, carried
              // in rp by the same rotate)
              const int last = m + GL - 1;
              const float r1v =
                  __shfl_sync(0xffffffffu, Bv[last], (lane + 31) & 31);
              av1 = lane == 0 ? rp1 : r1v;
              rp1 = r1v;
              const float r2v = __shfl_sync(
                  0xffffffffu, b1v[last - m0], (lane + 31) & 31);
              av2 = lane == 0 ? rp2 : r2v;
              rp2 = r2v;
            } else {
              av1 = Bv[m - 1];  // previous pass's B row, column j - 1
              av2 = b1v[g - 1];
            }
            u[g] = __fadd_rn(av1, __fsub_rn(b1v[g], dj));
            w[g] = __fadd_rn(av2, __fsub_rn(b2v[g], dj));
          } else {
            u[g] = kInfF;
            w[g] = kInfF;
          }
        }
        // Bv of the group is rewritten only now: the shifts above read the
        // previous pass's values
#pragma unroll
        for (int g = 0; g < kG32; ++g)
          if (m0 + g < NPL) Bv[m0 + g] = b2v[g];
        float mu = u[0], mw = w[0];
#pragma unroll
        for (int g = 1; g < kG32; ++g) {
          mu = fminf(mu, u[g]);
          mw = fminf(mw, w[g]);
        }
        const bool hit = MODE == 1 ? (mu <= la || mw < lb)
                                   : (mu <= la || mw <= lb);
        if (__any_sync(0xffffffffu, hit)) {
#pragma unroll
          for (int h = 0; h < kG32; h += 4) {
            // columns of blocks m0 + h .. + 3: consecutive within a layout
            // group (GL >= 2); GL == 1 is the interleaved layout (step 32);
            // blocks past NPL hold +inf
            lim = scan_hit<MODE>(u[h], u[h + 1], u[h + 2], u[h + 3], w[h],
                                 w[h + 1], w[h + 2], w[h + 3], di, di2, la, lb,
                                 i, col_of(m0 + h), GL == 1 ? 32 : 1, a.thr,
                                 &s_cd[warp][0][lane], &s_cij[warp][0][lane],
                                 st);
            la = lrow_of(di);
            lb = two ? lrow_of(di2) : -kInfF;
          }
        }
      }
    }
  }
  __syncwarp();
  if (MODE == 1) {
    const float best = st[0];
    double bd = best == kInfF ? kInf : (double)best;
    int bi = __float_as_int(st[32]), bj = __float_as_int(st[64]);
    warp_argmin(bd, bi, bj);
    if (lane == 0) *out = {bd, bi, bj};
    continue;
  }
  // FILTER32: warp minimum, candidate re-evaluation in fp64
  const float best = st[0];
  const int ncand = __float_as_int(st[32]);
  if (__any_sync(0xffffffffu, __float_as_int(st[64]))) {
    if (lane == 0) {  // listed for the exact fp64 re-scan
      *out = {kInf, kOverflowTag, kOverflowTag};
      a.ovf[1 + atomicAdd(&a.ovf[0], 1)] = task;
    }
    continue;
  }
  float m = best;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float keep = __fadd_ru(m, a.thr);
  double bd = kInf;
  int ei = 0x7fffffff, ej = 0x7fffffff;
  for (int kc = 0; kc < ncand; ++kc) {
    if (s_cd[warp][kc][lane] <= keep) {
      const uint32_t ij = s_cij[warp][kc][lane];
      const int ci = (int)(ij >> 16), cj = (int)(ij & 0xFFFFu);
      const int ai = tour[ci], aj = tour[cj];
      const int si = tour[ci + 1], sjj = tour[cj + 1 == n ? 0 : cj + 1];
      double t = __dadd_rn(a.cost[(size_t)ai * a.ld + aj],
                           a.cost[(size_t)si * a.ld + sjj]);
      t = __dsub_rn(t, dg[ci]);
      t = __dsub_rn(t, dg[cj]);
      if (res_less(t, ci, cj, bd, ei, ej)) {
        bd = t;
        ei = ci;
        ej = cj;
      }
    }
  }
  // structural pairs of this task, exact from d: (i, i+1) has A = d_i,
  // B = d_{i+1}; (0, n-1) from the matrix
  for (int ii = r0 + lane; ii < r1; ii += 32) {
    if (ii + 1 < n && ii + 1 >= jlo && ii + 1 < jhi) {
      const double d0 = dg[ii], d1 = dg[ii + 1];
      double t = __dadd_rn(d0, d1);
      t = __dsub_rn(t, d0);
      t = __dsub_rn(t, d1);
      if (res_less(t, ii, ii + 1, bd, ei, ej)) {
        bd = t;
        ei = ii;
        ej = ii + 1;
      }
    }
  }
  if (r0 == 0 && n - 1 >= jlo && n - 1 < jhi && lane == 0 && n - 1 > 1) {
    const int j = n - 1;  // s_{n-1} = a_0
    const int a0c = tour[0], aj = tour[j], s0 = tour[1], sjj = tour[0];
    double t = __dadd_rn(a.cost[(size_t)a0c * a.ld + aj],
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
  }  // task loop
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
  const double* cost64;  // capped plan: re-evaluate the chosen pair in fp64
  const double* cost64r;  // the fp64 matrix (in-apply re-scan)
  const double* dcache_in;  // (with the tour's d values)
  int sym;  // symmetric matrix: reversed edges keep their costs
  // bounded-scan mode: no separate fp64 re-scan kernel runs; a particle
  // whose band-scan candidate list overflowed (tagged result, rare) is
  // re-scanned in fp64 here, by its CTA
  int ovf_scan;
  const int32_t* plist;  // nullable: only these particles (count in *pcnt)
  const int32_t* pcnt;
};

__device__ void apply_one(const ApplyArgs& a, int p) {
  __shared__ int s_move[3];
  __shared__ double s_delta;
  __shared__ int s_better;
  __shared__ double s_wd[4];
  __shared__ int s_wi[4], s_wj[4];
  const int tid = threadIdx.x;
  if (a.res[(size_t)p * a.chunks].i == kAppliedTag) return;
  const bool rescan = a.ovf_scan && a.n >= 4 &&
                      a.res[(size_t)p * a.chunks].i == kOverflowTag;
  if (rescan) {
    // every pair in fp64 with the reference expression (solver.py:94-100)
    const uint16_t* t = a.tours + (size_t)p * a.np;
    const double* dg = a.dcache_in + (size_t)p * a.np;
    const int n = a.n, lane = tid & 31, warp = tid >> 5;
    double bd = __longlong_as_double(0x7ff0000000000000ll);
    int ei = 0x7fffffff, ej = 0x7fffffff;
    for (int i = warp; i < n - 1; i += 4) {
      const int ai = t[i], si = t[i + 1];
      const double di = dg[i];
      for (int j = i + 1 + lane; j < n; j += 32) {
        const int aj = t[j], sj = t[j + 1 == n ? 0 : j + 1];
        double v = __dadd_rn(ld_cost(a.cost64r + (size_t)ai * a.ld + aj),
                             ld_cost(a.cost64r + (size_t)si * a.ld + sj));
        v = __dsub_rn(v, di);
        v = __dsub_rn(v, dg[j]);
        if (res_less(v, i, j, bd, ei, ej)) {
          bd = v;
          ei = i;
          ej = j;
        }
      }
    }
    warp_argmin(bd, ei, ej);
    if (lane == 0) {
      s_wd[warp] = bd;
      s_wi[warp] = ei;
      s_wj[warp] = ej;
    }
    __syncthreads();
  }
  if (tid == 0) {
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int bi = 0x7fffffff, bj = 0x7fffffff;
    const TwoOptRes* r = a.res + (size_t)p * a.chunks;
    if (rescan) {
      for (int w = 0; w < 4; ++w)
        if (res_less(s_wd[w], s_wi[w], s_wj[w], best, bi, bj)) {
          best = s_wd[w];
          bi = s_wi[w];
          bj = s_wj[w];
        }
    } else {
      for (int c = 0; c < a.chunks; ++c)
        if (res_less(r[c].delta, r[c].i, r[c].j, best, bi, bj)) {
          best = r[c].delta;
          bi = r[c].i;
          bj = r[c].j;
        }
    }
    if (a.cost64 && bi != 0x7fffffff && bj != 0x7fffffff &&
        best != __longlong_as_double(0x7ff0000000000000ll)) {
      // the scan compared capped values: the reference's fp64 delta of the
      // chosen pair (solver.py:94-101)
      const uint16_t* t = a.tours + (size_t)p * a.np;
      const double* dg = a.dcache_in + (size_t)p * a.np;
      const int ai = t[bi], aj = t[bj], si = t[bi + 1],
                sj = t[bj + 1 == a.n ? 0 : bj + 1];
      double v = __dadd_rn(a.cost64[(size_t)ai * a.ld + aj],
                           a.cost64[(size_t)si * a.ld + sj]);
      v = __dsub_rn(v, dg[bi]);
      best = __dsub_rn(v, dg[bj]);
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
  if (a.cost && a.sym) {
    // symmetric matrix: edge k in (i, j) of the new tour is old edge
    // i + j - k reversed, same cost bits: reverse d[i+1 .. j-1] along with
    // the tour; only the two new edges i and j are gathered
    double* dg = a.dcache + (size_t)p * a.np;
    const int m = len - 1;  // d[i+1 .. j-1]
    for (int u = tid; u < len / 2 || u < m / 2; u += blockDim.x) {
      if (u < len / 2) {
        uint16_t x = t[i + 1 + u];
        t[i + 1 + u] = t[j - u];
        t[j - u] = x;
      }
      if (u < m / 2) {
        const double y = dg[i + 1 + u];
        dg[i + 1 + u] = dg[j - 1 - u];
        dg[j - 1 - u] = y;
      }
    }
    __syncthreads();
    if (tid < 2) {
      const int k = tid == 0 ? i : j;
      const int u = t[k], w = t[k + 1 == a.n ? 0 : k + 1];
      dg[k] = ld_cost(a.cost + (size_t)u * a.ld + w);
    }
  } else {
    for (int u = tid; u < len / 2; u += blockDim.x) {
      uint16_t x = t[i + 1 + u];
      t[i + 1 + u] = t[j - u];
      t[j - u] = x;
    }
    __syncthreads();
    if (a.cost) {
      for (int k = i + tid; k <= j && k < a.n; k += blockDim.x) {
        int u = t[k], w = t[k + 1 == a.n ? 0 : k + 1];
        a.dcache[(size_t)p * a.np + k] = ld_cost(a.cost + (size_t)u * a.ld + w);
      }
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


// One CTA per particle; with a particle list (bounded-scan mode: the band
// scan's fallbacks, the others were applied by the bounded scan) a small
// grid strides over the list.
__global__ void __launch_bounds__(128) k_two_opt_apply(ApplyArgs a) {
  if (a.ctl && (a.ctl->done || a.ctl->improved)) return;
  if (a.plist) {
    const int cnt = *a.pcnt;
    for (int q = blockIdx.x; q < cnt; q += gridDim.x) {
      apply_one(a, a.plist[q]);
      __syncthreads();
    }
    return;
  }
  const int p = blockIdx.x;
  if (p >= a.count) return;
  apply_one(a, p);
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

// fp16 rows: round(C * scale) (scale a power of two, so only the final
// rounding to fp16 is inexact; integers <= 2048 are exact); entries equal to
// vfrom (vfrom > 0) read as vto
__global__ void k_cost_to16(const double* cost, int64_t ld, int n,
                            uint16_t* c16, int64_t ld16, double scale,
                            double vfrom, double vto) {
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n, c = e % n;
    double v = cost[r * ld + c];
    if (vfrom > 0.0 && v == vfrom) v = vto;
    const __half h = __double2half(v * scale);
    c16[r * ld16 + c] = __half_as_ushort(h);
  }
}

// second statistics pass: max |C| over |C| < max (the finite level under a
// virtual one) and whether -max occurs
__global__ void k_cost_second(const double* cost, int64_t ld, int n,
                              CostStats* st) {
  const double mx = __longlong_as_double((long long)st->maxabs_bits);
  unsigned long long m2 = 0;
  int neg = 0, asym = 0;
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n, c = e % n;
    const double v = cost[r * ld + c];
    if (c > r)
      asym |= __double_as_longlong(v) != __double_as_longlong(cost[c * ld + r]);
    const double a = fabs(v);
    if (a < mx) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(a);
      m2 = b > m2 ? b : m2;
    } else if (v < 0.0) {
      neg = 1;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, m2, o);
    m2 = x > m2 ? x : m2;
    neg |= __shfl_xor_sync(0xffffffffu, neg, o);
    asym |= __shfl_xor_sync(0xffffffffu, asym, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&st->second_bits, m2);
    if (neg) atomicOr(&st->negmax, 1);
    if (asym) atomicOr(&st->asym, 1);
  }
}

// fp32 rows: entries equal to (float)vfrom read as vto
__global__ void k_cost_cap32(float* c32, int64_t ld32, int n, float from,
                             float to) {
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    float* q = c32 + (e / n) * ld32 + e % n;
    if (*q == from) *q = to;
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

template <int NPL, int MODE, int ES>
cudaError_t launch_scan32_t(const ScanArgs& a, int warps, int blocks,
                            size_t smem, cudaStream_t s) {
  if (a.chunks == 1 || getenv("DPSO_SCAN_NOPERSIST")) {
    auto k = k_two_opt_scan32<NPL, MODE, ES, false>;
    cudaError_t e = set_dyn_smem((const void*)k, smem);
    if (e != cudaSuccess) return e;
    k<<<blocks, warps * 32, smem, s>>>(a);
    return cudaGetLastError();
  }
  auto k = k_two_opt_scan32<NPL, MODE, ES, true>;
  cudaError_t e = set_dyn_smem((const void*)k, smem);
  if (e != cudaSuccess) return e;
  // one resident wave of persistent warps
  int per_sm = 0, dev = 0, sms = 148;
  static const int mult = [] {  // resident waves launched (testing knob)
    const char* e = getenv("DPSO_SCAN_WAVES");
    return e ? std::max(1, atoi(e)) : 1;
  }();
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, warps * 32,
                                                    smem) == cudaSuccess &&
      per_sm > 0 && cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) ==
          cudaSuccess)
    blocks = std::min(blocks, per_sm * sms * mult);
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

cudaError_t two_opt_prepare(const double* cost, int64_t ld, int32_t n,
                            int64_t np, float* c32, uint16_t* c16,
                            unsigned char* band, CostStats* st,
                            cudaStream_t s, TwoOptPlan* pl, void* bound_buf) {
  memset(pl, 0, sizeof *pl);
  pl->cost = cost;
  pl->ld = ld;
  pl->cost32 = c32;
  pl->ld32 = np;
  pl->es = 4;
  pl->dscale = 1.f;
  cudaError_t e = launch_cost_prep(cost, ld, n, c32, np, st, s);
  if (e) return e;
  const int64_t total = (int64_t)n * n;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (blocks < 1) blocks = 1;
  k_cost_second<<<blocks, 256, 0, s>>>(cost, ld, n, st);
  CostStats h;
  e = cudaGetLastError();
  if (!e) e = cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (e) return e;
  double maxabs_raw;
  memcpy(&maxabs_raw, &h.maxabs_bits, sizeof maxabs_raw);
  pl->symmetric = !h.asym && !getenv("DPSO_NO_SYM");
  {
    // a virtual level (entries equal to max|C|, > 64 x every other |C|):
    // cap it at 5 x the finite maximum in the fp32/fp16 rows (> the spread
    // 4 max_finite of the finite parts of two deltas)
    double mx, m2;
    memcpy(&mx, &h.maxabs_bits, sizeof mx);
    memcpy(&m2, &h.second_bits, sizeof m2);
    if (!h.negmax && m2 > 0.0 && mx > 64.0 * m2 && mx < 1e300 &&
        !getenv("DPSO_NO_VCAP")) {
      pl->vfrom = mx;
      pl->vto = 5.0 * m2;
      k_cost_cap32<<<blocks, 256, 0, s>>>(c32, np, n, (float)mx,
                                           (float)pl->vto);
      e = cudaGetLastError();
      if (e) return e;
      const double capped = pl->vto;
      memcpy(&h.maxabs_bits, &capped, sizeof capped);
    }
  }
  {
    double mxc;
    memcpy(&mxc, &h.maxabs_bits, sizeof mxc);
    e = band_prepare(cost, ld, n, band, mxc, !h.nonintegral, pl->vfrom,
                     pl->vto, s, pl);
    if (e) return e;
    e = bound_prepare(cost, ld, n, bound_buf, maxabs_raw, s, pl);
    if (e) return e;
  }
  pl->mode = two_opt_mode(h, n, &pl->thr);
  if (getenv("DPSO_SCAN_MODE")) pl->mode = atoi(getenv("DPSO_SCAN_MODE"));
  if (pl->mode == kScanFilter32 && pl->thr == 0.f) pl->mode = kScanFP64;
  if (pl->mode == kScanFP64) pl->vfrom = pl->vto = 0.0;  // fp64 rows: exact
  const char* e16 = getenv("DPSO_SCAN16");
  if (!c16 || (e16 && atoi(e16) == 0) || pl->mode == kScanFP64) return e;
  double mx;
  memcpy(&mx, &h.maxabs_bits, sizeof mx);
  double scale = 1.0;
  if (pl->mode == kScanExact32) {
    if (!(mx <= 2048.0)) return e;  // fp16 integers are exact up to 2^11
  } else {
    if (!(mx > 1e-30 && mx < 1e30)) return e;
    // max |C| scale in (2^14, 2^15]: every scaled entry is an fp16 normal
    // or a subnormal with absolute error <= 2^-25
    scale = ldexp(1.0, 15 - ilogb(mx) - 1);
    while (mx * scale > 32768.0) scale *= 0.5;
    while (mx * scale * 2.0 <= 32768.0) scale *= 2.0;
    // |t - delta| <= e_max = 2^-11 (|A| + |B|) + fp32 terms
    //               <= 1.002 * 2^-10 max|C| (row units); window = 4 e_max
    // (a true tie of the argmin is within 2 e_max of its computed value,
    // which is within 2 e_max of the computed minimum), with margin
    pl->thr = (float)(mx * scale * 0.00403);
  }
  pl->dscale = (float)scale;
  k_cost_to16<<<blocks, 256, 0, s>>>(cost, ld, n, c16, np, scale, pl->vfrom,
                                     pl->vto);
  e = cudaGetLastError();
  if (e) return e;
  pl->cost16 = c16;
  pl->es = 2;
  return cudaSuccess;
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

// Column ranges of the fp32 scan (npl_max32() blocks of 32 columns each).
static int column_ranges(int32_t n) {
  const int w = 32 * npl_max32();
  return n <= w ? 1 : (n + w - 1) / w;
}

int two_opt_pick_chunks(int32_t n, int32_t P) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // fp32 scan: one warp per task (row ring + d_j in shared memory)
  const int npl = std::min(std::max(npl_for(n), 1), npl_max32());
  size_t per_warp =
      (size_t)kBufs32 * round_up((int64_t)round_up(n, 4) * 4, 128) +
      4 * (size_t)32 * npl;
  int warps_per_sm = (int)(kSmemBudget / per_warp);
  if (warps_per_sm < 1) warps_per_sm = 1;
  if (warps_per_sm > 16) warps_per_sm = 16;
  const int64_t slots = (int64_t)sms * warps_per_sm;
  const int R = column_ranges(n);
  // tasks per resident warp slot: balances the tail against per-task setup
  int per_slot = 6;
  if (const char* e = getenv("DPSO_TASKS_PER_SLOT")) per_slot = std::max(1, atoi(e));
  int chunks = (int)((per_slot * slots + P - 1) / P);
  chunks = std::max(chunks, R);
  chunks = std::min(chunks, 32 * R);
  chunks = std::min(chunks, std::max(R, n / 8 + 1));
  return chunks;
}

// Task table: chunks x (r0, r1, jlo, jhi).  Columns are split into ranges
// of 32 * npl_max32(); each range's pairs (i < j, j in the range) are cut into
// row bands of roughly equal pair count, with bands given to the ranges in
// proportion to their pairs.  Every pair i < j is in exactly one task.
int two_opt_chunk_table(int32_t n, int32_t chunks, int32_t* tab) {
  const int R = column_ranges(n);
  const int w = 32 * npl_max32();
  std::vector<double> pairs(R);
  double total = 0.0;
  for (int k = 0; k < R; ++k) {
    const double lo = (double)k * w, hi = std::min<double>(n, (k + 1.0) * w);
    pairs[k] = 0.5 * (lo + hi - 1.0) * (hi - lo);  // column c has c pairs
    total += pairs[k];
  }
  std::vector<int> bands(R, 1);
  int given = R;
  for (int k = 0; k < R && total > 0; ++k) {
    const int extra = (int)((chunks - R) * pairs[k] / total);
    bands[k] += extra;
    given += extra;
  }
  for (int k = R - 1; given < chunks; k = (k + R - 1) % R) {
    ++bands[k];
    ++given;
  }
  int c = 0;
  for (int k = 0; k < R; ++k) {
    const int jlo = k * w, jhi = std::min(n, (k + 1) * w);
    const int last = std::max(jhi - 1, 0);  // rows 0 .. jhi - 2
    auto cnt = [&](int i) { return (double)(jhi - std::max(jlo, i + 1)); };
    double acc = 0.0;
    int r = 0;
    for (int b = 0; b < bands[k]; ++b, ++c) {
      const int r0 = r;
      const double target = pairs[k] * (b + 1) / bands[k];
      if (b + 1 == bands[k]) {
        r = last;
      } else {
        while (r < last && acc + cnt(r) <= target) {
          acc += cnt(r);
          ++r;
        }
      }
      tab[4 * c + 0] = r0;
      tab[4 * c + 1] = std::max(r, r0);
      tab[4 * c + 2] = jlo;
      tab[4 * c + 3] = jhi;
    }
  }
  return 0;
}

cudaError_t launch_two_opt_core(const TwoOptPlan& pl, int32_t n, int32_t np,
                                uint16_t* tours, const double* dcache,
                                int32_t count, TwoOptRes* res, int32_t chunks,
                                const int32_t* chunk_tab, const DevCtl* ctl,
                                double* fit, double* pfit, uint16_t* pbest,
                                double* delta_out, double* dcache_rw,
                                cudaStream_t s, int parts, int reserve_sms) {
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
  a.chunk_tab = chunk_tab;
  a.res = res;
  a.ctl = ctl;
  a.thr = pl.thr;
  a.stream_only = getenv("DPSO_SCAN_STREAM_ONLY")
                      ? atoi(getenv("DPSO_SCAN_STREAM_ONLY"))
                      : 0;  // probes: 1 = row stream, 2 = stream + gathers
  const int64_t tasks = (int64_t)count * chunks;
  cudaError_t e = cudaSuccess;
  const int npl = npl_for(n);
  a.ovf = reinterpret_cast<int32_t*>(res + (size_t)count * chunks);
  auto fp64_scan = [&]() -> cudaError_t {
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
    if (pl.band_mode) {
      // row-per-lane band scan (k_two_opt_band.cu), then the FILTER
      // overflow re-scan over the listed chunk tasks
      if (getenv("DPSO_BAND_DEBUG"))  // unwritten results read as NaN
        e = cudaMemsetAsync(res, 0xFF, sizeof(TwoOptRes) * count * chunks, s);
      // bounded scan first; the band scan takes the particles it lists (a
      // launch that exits at once when the list is empty: measured as fast
      // as a conditional graph node around it, which ncu cannot profile)
      const bool bound = pl.bound != 0;
      int32_t* runs =
          ctl ? &const_cast<DevCtl*>(ctl)->band_runs : nullptr;
      // with the apply in this call, the bounded scan applies the moves it
      // resolves itself (k_two_opt_apply skips them)
      BoundApply ap{tours, dcache_rw, fit, pfit, pbest, delta_out};
      const bool ap_here = (parts & 2) && dcache_rw && !getenv("DPSO_BOUND_NOAPPLY");
      if (!e && bound)
        e = launch_two_opt_bound(pl, n, np, tours, dcache, count, res, chunks,
                                 ctl, s, runs, ap_here ? &ap : nullptr);
      if (!e && pl.band_mode == 2) e = cudaMemsetAsync(a.ovf, 0, 4, s);
      if (!e)
        e = launch_two_opt_band(pl, n, np, tours, dcache, count, res, chunks,
                                a.ovf, ctl, s, reserve_sms,
                                bound ? pl.bound_fb + 1 : nullptr,
                                bound ? pl.bound_fb : nullptr, runs, bound);
      // (bounded-scan mode: the apply re-scans a tagged particle itself)
      if (!e && pl.band_mode == 2 && !bound) {
        k_two_opt_rescan64<<<2 * 148, 128, 0, s>>>(a);
        e = cudaGetLastError();
      }
    } else if (pl.mode == kScanFP64 || !pl.cost32) {
      e = fp64_scan();
    } else {
      const int es = (pl.es == 2 && pl.cost16) ? 2 : 4;
      a.rows = es == 2 ? (const void*)pl.cost16 : (const void*)pl.cost32;
      a.row_pitch = (int64_t)es * pl.ld32;
      a.dscale = es == 2 ? pl.dscale : 1.f;
      a.vfrom = pl.vfrom;
      a.vto = pl.vto;
      a.row_bytes = (uint32_t)(round_up(n, 16 / es) * es);
      a.buf_stride = (uint32_t)round_up(a.row_bytes, 128);
      // per warp: 2-slot row ring + d_j (fp32, 32 * NPL entries)
      const int npl32 = std::min(std::max(npl, 1), npl_max32());
      a.buf_stride2 = (uint32_t)(kBufs32 * a.buf_stride +
                                 round_up((int64_t)32 * npl32 * 4, 128));
      const int warps = kW32;
      const size_t smem = (size_t)warps * a.buf_stride2;
      a.task_ctr = a.ovf + 1 + tasks;
      e = cudaMemsetAsync(a.task_ctr, 0, 4, s);
      if (!e && pl.mode == kScanFilter32) e = cudaMemsetAsync(a.ovf, 0, 4, s);
      if (e != cudaSuccess) return e;
      const int blocks = (int)((tasks + warps - 1) / warps);
#define SCAN32(NPL)                                                      \
  (es == 2 ? (pl.mode == kScanExact32                                    \
                  ? launch_scan32_t<NPL, 1, 2>(a, warps, blocks, smem, s) \
                  : launch_scan32_t<NPL, 2, 2>(a, warps, blocks, smem, s)) \
           : (pl.mode == kScanExact32                                    \
                  ? launch_scan32_t<NPL, 1, 4>(a, warps, blocks, smem, s) \
                  : launch_scan32_t<NPL, 2, 4>(a, warps, blocks, smem, s)))
      switch (npl32) {
        case 1: e = SCAN32(1); break;
        case 2: e = SCAN32(2); break;
        case 4: e = SCAN32(4); break;
        case 8: e = SCAN32(8); break;
        case 16: e = SCAN32(16); break;
        default: e = SCAN32(32); break;
      }
#undef SCAN32
      // FILTER32 candidate-list overflow: exact fp64 re-scan of those tasks
      if (!e && pl.mode == kScanFilter32) {
        k_two_opt_rescan64<<<2 * 148, 128, 0, s>>>(a);
        e = cudaGetLastError();
      }
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
  const bool capped = pl.band_mode ? pl.band_vfrom > 0.0
                                   : pl.vfrom > 0.0 && pl.mode != kScanFP64;
  b.cost64 = capped ? pl.cost : nullptr;
  b.dcache_in = dcache;
  b.sym = pl.symmetric;
  b.cost64r = pl.cost;
  b.ovf_scan = pl.band_mode == 2 && pl.bound;
  if (n < 4) {
    // _best_exchange returns (body, 0.0) for n < 4 (solver.py:91-93)
    if (delta_out) cudaMemsetAsync(delta_out, 0, sizeof(double) * count, s);
    return cudaGetLastError();
  }
  b.plist = nullptr;
  b.pcnt = nullptr;
  int grid = count;
  if (pl.bound && (parts & 1) && dcache_rw && !getenv("DPSO_BOUND_NOAPPLY")) {
    // the bounded scan applied every move it resolved: only its fallbacks
    b.plist = pl.bound_fb + 1;
    b.pcnt = pl.bound_fb;
    grid = std::min(count, 148);
  }
  if (count > 0) k_two_opt_apply<<<grid, 128, 0, s>>>(b);
  return cudaGetLastError();
}

// The swarm keeps dcache equal to the edge costs of x at all times (the
// update re-gathers only the edges it moved), so the apply refreshes the
// edges i..j of a move.
cudaError_t launch_two_opt(const SwarmView& v, cudaStream_t s, int parts) {
  // the numpy mutation-stream walk (one CTA, launch_mutation_walk) runs on
  // a forked stream concurrently with the scan: the band scan, one CTA per
  // SM, leaves it an SM
  const int reserve =
      v.use_mutation && v.rng_mode == DPSO_RNG_NUMPY ? 1 : 0;
  return launch_two_opt_core(v.plan, v.n, v.np, v.x, v.dcache, v.P, v.tores,
                             v.chunks, v.chunk_tab, v.ctl, v.fit, v.pfit,
                             v.pbest, nullptr, v.dcache, s, parts, reserve);
}

cudaError_t launch_two_opt_batch(const TwoOptPlan& pl, int32_t n, int32_t np,
                                 uint16_t* tours, const double* dcache,
                                 int32_t count, TwoOptRes* res, int32_t chunks,
                                 const int32_t* chunk_tab, double* delta_out,
                                 cudaStream_t s) {
  return launch_two_opt_core(pl, n, np, tours, dcache, count, res, chunks,
                             chunk_tab, nullptr, nullptr, nullptr, nullptr,
                             delta_out, const_cast<double*>(dcache), s, 3, 0);
}

}  // namespace dpso
