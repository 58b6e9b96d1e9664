// Best-improvement 2-opt (solver.py:88-106, applied at solver.py:309-317).
//
// delta(i,j) = ((C[a_i,a_j] + C[s_i,s_j]) - d_i) - d_j for 0 <= i < j < n,
// s = roll(a, -1), d_i = C[a_i, s_i]; the move is the first (row-major)
// argmin; it is applied when delta < -1e-12 and fitness += delta.
//
// Layout on the device: one warp owns a task = (particle, band of pair rows
// [r0, r1)).  The cost rows a_r0 .. a_r1 are streamed in order from L2 into a
// 3-deep per-warp ring in shared memory with cp.async.bulk (TMA bulk copy,
// mbarrier completion), so each cost row is read from L2 once per task and
// used twice: as the A row of pair-row i and the B row of pair-row i-1.
// Lane l owns the columns j = l + 32m; a_j, s_j (packed u16 pair) and d_j
// live in registers for the whole task.  Row i then costs two shared-memory
// gathers A[a_j], B[s_j] and three fp64 adds per pair in the reference's
// exact expression order (no FMA contraction possible for add/sub).  Each lane
// keeps its first strict minimum in (i, j) order; a warp shuffle reduction
// on (delta, i, j) gives the band's first-index argmin, and the apply kernel
// merges bands in row order (earlier band wins ties), reproducing numpy's
// argmin tie-break bit for bit.
#include <float.h>

#include <algorithm>

#include "dpso_internal.cuh"

namespace dpso {

namespace {

constexpr int kMaxWarps = 4;  // warps (tasks) per CTA, upper bound
constexpr int kBufs = 3;   // row ring depth per warp

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src,
                                         uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

struct ScanArgs {
  const double* cost;
  int64_t ld;
  int32_t n, np, count, chunks;
  const uint16_t* tours;   // count x np
  const double* dcache;    // count x np
  const int32_t* chunk_row;
  TwoOptRes* res;          // count x chunks
  const DevCtl* ctl;       // nullable: skip when done or improved
  uint32_t row_bytes;      // bytes streamed per cost row (multiple of 16)
  uint32_t buf_stride;     // bytes between ring buffers
};

__device__ __forceinline__ bool res_less(double d1, int i1, int j1, double d2,
                                         int i2, int j2) {
  if (d1 < d2) return true;
  if (d2 < d1) return false;
  return (i1 < i2) || (i1 == i2 && j1 < j2);
}

// NPL > 0: lane-owned columns in registers (n <= 32*NPL).
// NPL == 0: generic path, columns streamed from global/L1 per row.
// STAGE: cost rows staged in shared memory by bulk copies (false = read the
// rows straight from global/L2, for n too large for a 3-row ring).
constexpr int kGroup = 4;  // column blocks (of 32) per uniform skip test

template <int NPL, bool STAGE>
__global__ void __launch_bounds__(kMaxWarps * 32)
    k_two_opt_scan(ScanArgs a) {
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
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  if (r0 >= r1) {
    if (lane == 0) *out = {kInf, 0x7fffffff, 0x7fffffff};
    return;
  }
  const uint16_t* tour = a.tours + (size_t)p * a.np;
  const double* dg = a.dcache + (size_t)p * a.np;
  unsigned char* wbase = smem + (size_t)warp * kBufs * a.buf_stride;
  uint64_t* wb = bars[warp];

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

  const int nrows = r1 - r0 + 1;  // cost rows a_r0 .. a_r1
  if (STAGE && lane == 0) {
    for (int b = 0; b < kBufs; ++b) mbar_init(&wb[b], 1);
    fence_barrier_init();
    for (int q = 0; q < 2 && q < nrows; ++q) {
      int node = tour[r0 + q];
      mbar_expect_tx(&wb[q], a.row_bytes);
      bulk_g2s(wbase + (size_t)q * a.buf_stride,
               a.cost + (size_t)node * a.ld, a.row_bytes, &wb[q]);
    }
  }
  __syncwarp();

  double best = kInf;
  int bi = 0x7fffffff, bj = 0x7fffffff;

  for (int i = r0; i < r1; ++i) {
    const int q = i - r0;
    const double* A;
    const double* B;
    if (STAGE) {
      if (lane == 0 && q + 2 < nrows) {
        const int b = (q + 2) % kBufs;
        const int node = tour[r0 + q + 2];
        fence_proxy_async();
        mbar_expect_tx(&wb[b], a.row_bytes);
        bulk_g2s(wbase + (size_t)b * a.buf_stride,
                 a.cost + (size_t)node * a.ld, a.row_bytes, &wb[b]);
      }
      const int ba = q % kBufs, bb = (q + 1) % kBufs;
      mbar_wait(&wb[ba], (uint32_t)((q / kBufs) & 1));
      mbar_wait(&wb[bb], (uint32_t)(((q + 1) / kBufs) & 1));
      A = (const double*)(wbase + (size_t)ba * a.buf_stride);
      B = (const double*)(wbase + (size_t)bb * a.buf_stride);
    } else {
      A = a.cost + (size_t)tour[i] * a.ld;
      B = a.cost + (size_t)tour[i + 1] * a.ld;
    }
    const double di = dg[i];
    // row-local first minimum over this lane's columns (ascending j)
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
  if (lane == 0) *out = {best, bi, bj};
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
    for (int k = max(i, 0) + tid; k <= j && k < a.n; k += blockDim.x) {
      int u = t[k], w = t[k + 1 == a.n ? 0 : k + 1];
      a.dcache[(size_t)p * a.np + k] = a.cost[(size_t)u * a.ld + w];
    }
  }
  if (a.fit) {
    __shared__ int s_better;
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

template <int NPL, bool STAGE>
cudaError_t launch_scan_t(const ScanArgs& a, int warps, int blocks,
                          size_t smem, cudaStream_t s) {
  auto k = k_two_opt_scan<NPL, STAGE>;
  static size_t configured = 48 * 1024;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(
        k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  k<<<blocks, warps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

// bytes of the per-warp row ring
size_t ring_bytes(int n) {
  return (size_t)kBufs * round_up((int64_t)round_up(n, 2) * 8, 128);
}

constexpr size_t kSmemBudget = 220 * 1024;

}  // namespace

int two_opt_pick_chunks(int32_t n, int32_t P) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  size_t per_warp = ring_bytes(n);
  int warps_per_sm = (int)(kSmemBudget / per_warp);
  if (warps_per_sm < 1) warps_per_sm = 1;
  if (warps_per_sm > 32) warps_per_sm = 32;
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

cudaError_t launch_two_opt_core(const double* cost, int64_t ld, int32_t n,
                                int32_t np, uint16_t* tours,
                                const double* dcache, int32_t count,
                                TwoOptRes* res, int32_t chunks,
                                const int32_t* chunk_row, const DevCtl* ctl,
                                double* fit, double* pfit, uint16_t* pbest,
                                double* delta_out, double* dcache_rw,
                                cudaStream_t s, int parts = 3) {
  ScanArgs a;
  a.cost = cost;
  a.ld = ld;
  a.n = n;
  a.np = np;
  a.count = count;
  a.chunks = chunks;
  a.tours = tours;
  a.dcache = dcache;
  a.chunk_row = chunk_row;
  a.res = res;
  a.ctl = ctl;
  a.row_bytes = (uint32_t)(round_up(n, 2) * 8);
  a.buf_stride = (uint32_t)round_up(a.row_bytes, 128);
  const size_t per_warp = ring_bytes(n);
  const bool stage = per_warp <= kSmemBudget;
  int warps = stage ? (int)std::min<size_t>(kMaxWarps, kSmemBudget / per_warp)
                    : kMaxWarps;
  const size_t smem = stage ? (size_t)warps * per_warp : 0;
  const int64_t tasks = (int64_t)count * chunks;
  const int blocks = (int)((tasks + warps - 1) / warps);
  cudaError_t e = cudaSuccess;
  if ((parts & 1) && n >= 4 && blocks > 0) {
#define SCAN(NPL)                                                    \
  (stage ? launch_scan_t<NPL, true>(a, warps, blocks, smem, s)       \
         : launch_scan_t<NPL, false>(a, warps, blocks, smem, s))
    if (n <= 32)
      e = SCAN(1);
    else if (n <= 64)
      e = SCAN(2);
    else if (n <= 128)
      e = SCAN(4);
    else if (n <= 256)
      e = SCAN(8);
    else if (n <= 512)
      e = SCAN(16);
    else if (n <= 1024)
      e = SCAN(32);
    else if (n <= 2048)
      e = SCAN(64);
    else
      e = SCAN(0);
#undef SCAN
    if (e != cudaSuccess) return e;
  }
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
  b.cost = dcache_rw ? cost : nullptr;
  b.ld = ld;
  b.dcache = dcache_rw;
  if (!(parts & 2)) return cudaSuccess;
  if (n < 4) {
    // _best_exchange returns (body, 0.0) for n < 4 (solver.py:91-93)
    if (delta_out) cudaMemsetAsync(delta_out, 0, sizeof(double) * count, s);
    return cudaGetLastError();
  }
  if (count > 0) k_two_opt_apply<<<count, 128, 0, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_two_opt(const SwarmView& v, cudaStream_t s, int parts) {
  return launch_two_opt_core(v.cost, v.ld, v.n, v.np, v.x, v.dcache, v.P,
                             v.tores, v.chunks, v.chunk_row, v.ctl, v.fit,
                             v.pfit, v.pbest, nullptr, nullptr, s, parts);
}

cudaError_t launch_two_opt_batch(const double* cost, int64_t ld, int32_t n,
                                 int32_t np, uint16_t* tours,
                                 const double* dcache, int32_t count,
                                 TwoOptRes* res, int32_t chunks,
                                 const int32_t* chunk_row, double* delta_out,
                                 cudaStream_t s) {
  return launch_two_opt_core(cost, ld, n, np, tours, dcache, count, res,
                             chunks, chunk_row, nullptr, nullptr, nullptr,
                             nullptr, delta_out, const_cast<double*>(dcache),
                             s);
}

}  // namespace dpso
