// Gather-bandwidth microbenchmarks for the 2-opt scan's roofline (SURVEY
// §8(d); the op is the gather at solver.py:96-99, C[a_i, a_j] + C[s_i, s_j]).
//
//   l2_gather     random 8-byte loads from an fp64 table of 8..32 MB (L2
//                 resident) and 1 GB (HBM), 8 independent chains per thread
//   smem_gather   random 2-byte / 8-byte lane gathers from rows staged in
//                 shared memory (each lane's offsets fixed in registers, as
//                 the column-per-lane scan does) and the conflict-free
//                 pattern (lane l always in bank l, as the row-per-lane band
//                 scan does)
//   bulk_rows     cp.async.bulk of random 2-KB rows of an L2-resident matrix
//                 into shared memory, 32 rows per stage, 2 stages per CTA
//                 (the band scan's row stream)
//
// Output: one JSON object on stdout.  Build + run: tools/gather_peaks.py.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                          \
  do {                                                                 \
    cudaError_t e_ = (x);                                              \
    if (e_ != cudaSuccess) {                                           \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__,                \
              cudaGetErrorString(e_));                                 \
      exit(1);                                                         \
    }                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// ---- L2 / HBM random gathers ----------------------------------------------
__global__ void __launch_bounds__(256) k_l2_gather(const double* tbl,
                                                   uint32_t mask, int iters,
                                                   double* sink) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = hash32(t * 8 + k);
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x[k] = x[k] * 1664525u + 1013904223u;
      v[k] = __ldcg(tbl + ((x[k] >> 3) & mask));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k];
  }
  if (acc == 1.2345) sink[t] = acc;
}

// ---- shared-memory gathers ------------------------------------------------
// ES = element bytes (2: fp16 rows, 8: fp64 rows); PAT 0 = random offsets
// per lane (fixed in registers), 1 = conflict-free (lane l -> bank l).
// 4 staged rows of 2000 elements; every iteration gathers NOFF offsets from
// each row.
template <int ES, int PAT>
__global__ void __launch_bounds__(256) k_smem_gather(int iters, float* sink) {
  constexpr int kRow = 2000;
  constexpr int kRowBytes = ((kRow * ES + 127) / 128) * 128;
  constexpr int NOFF = 16;
  extern __shared__ __align__(128) unsigned char sm[];
  for (int i = threadIdx.x; i < 4 * kRowBytes / 4; i += blockDim.x)
    ((uint32_t*)sm)[i] = hash32(i) & 0x3c003c00u;  // small fp16 / junk fp64
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t off[NOFF];
#pragma unroll
  for (int m = 0; m < NOFF; ++m) {
    uint32_t e = PAT == 0 ? hash32(blockIdx.x * 4096 + threadIdx.x * 64 + m) %
                                (uint32_t)kRow
                          : (uint32_t)(ES == 2 ? 2 * lane + 64 * m
                                               : (lane % 16) + 32 * m);
    off[m] = e * ES;
  }
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const uint32_t R = base + (uint32_t)(it & 3) * kRowBytes;
#pragma unroll
    for (int m = 0; m < NOFF; ++m) {
      float v;
      if (ES == 2) {
        asm volatile(
            "{\n\t.reg .b16 h;\n\tld.shared.b16 h, [%1];\n\t"
            "cvt.f32.f16 %0, h;\n\t}"
            : "=f"(v)
            : "r"(R + off[m]));
      } else {
        double d;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(d) : "r"(R + off[m]));
        v = (float)d;
      }
      acc += v;
    }
  }
  if (acc == 1.2345f) sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// ---- bulk row copies L2 -> shared memory ----------------------------------
__device__ __forceinline__ uint32_t s32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__global__ void __launch_bounds__(256) k_bulk_rows(const unsigned char* mat,
                                                   int nrows, int row_bytes,
                                                   int rps, int nst,
                                                   int stages, float* sink) {
  // ring of nst stages of rps rows, issued by every warp of the CTA (warp w
  // copies rows w, w + nwarps, ...; one expect-tx arrival per warp), the
  // stage consumed at once: the band scan's producer pattern
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const uint32_t stride = (uint32_t)((row_bytes + 127) / 128 * 128);
  if (threadIdx.x == 0) {
    for (int b = 0; b < nst; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                       s32(&bar[b])),
                   "r"(nw));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int st) {
    const int b = st % nst;
    int mine = 0;
    for (int r = warp; r < rps; r += nw) ++mine;
    if (lane == 0)
      asm volatile(
          "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
              s32(&bar[b])),
          "r"((uint32_t)(mine * row_bytes))
          : "memory");
    __syncwarp();
    const int r = warp + nw * lane;
    if (lane < mine) {
      const uint32_t row =
          hash32(blockIdx.x * 100003u + st * 32 + r) % nrows;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
          "[%0], [%1], %2, [%3];" ::"r"(s32(sm + (size_t)b * rps * stride +
                                           (size_t)r * stride)),
          "l"(mat + (size_t)row * row_bytes), "r"((uint32_t)row_bytes),
          "r"(s32(&bar[b]))
          : "memory");
    }
  };
  float acc = 0.f;
  for (int st = 0; st < nst - 1 && st < stages; ++st) issue(st);
  for (int st = 0; st < stages; ++st) {
    if (st + nst - 1 < stages) issue(st + nst - 1);
    const int b = st % nst;
    const uint32_t par = (uint32_t)((st / nst) & 1);
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(s32(&bar[b])),
        "r"(par)
        : "memory");
    acc += ((const float*)(sm + (size_t)b * rps * stride))[threadIdx.x];
    __syncthreads();  // stage b consumed before it is reissued
  }
  if (acc == 1.2345f) sink[threadIdx.x] = acc;
}

// sequential 16-byte loads over an L2-resident buffer (each CTA sweeps a
// contiguous slice, the whole buffer read `reps` times)
__global__ void __launch_bounds__(256) k_l2_seq(const int4* buf, size_t n16,
                                                int reps, int* sink) {
  int acc = 0;
  const size_t per = n16 / gridDim.x;
  const int4* b = buf + per * blockIdx.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = threadIdx.x; i < per; i += blockDim.x) {
      const int4 v = __ldcg(b + i);
      acc += v.x ^ v.w;
    }
  if (acc == 12345) sink[threadIdx.x] = acc;
}

template <typename F>
float time_ms(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();  // warm-up
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, l2 = 0, clk = 0, smem_optin = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  CK(cudaDeviceGetAttribute(&smem_optin,
                            cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"clock_khz_attr\": %d, "
         "\"smem_per_block_optin\": %d",
         sms, l2, clk, smem_optin);
  float* sink;
  CK(cudaMalloc(&sink, 1 << 24));

  // L2 / HBM gathers
  const size_t sizes_mb[] = {8, 16, 32, 1024};
  for (size_t mb : sizes_mb) {
    const size_t elems = mb * (1u << 20) / 8;
    double* tbl;
    CK(cudaMalloc(&tbl, elems * 8));
    CK(cudaMemset(tbl, 0, elems * 8));
    const int blocks = sms * 8, iters = 64;
    const float ms = time_ms(
        [&] {
          k_l2_gather<<<blocks, 256>>>(tbl, (uint32_t)(elems - 1), iters,
                                       (double*)sink);
        },
        10);
    const double loads = (double)blocks * 256 * iters * 8;
    printf(", \"gather_f64_%zuMB\": {\"ms\": %.4f, \"gloads_per_s\": %.2f, "
           "\"useful_gbs\": %.1f, \"sector_gbs\": %.1f}",
           mb, ms, loads / ms / 1e6, loads * 8 / ms / 1e6,
           loads * 32 / ms / 1e6);
    CK(cudaFree(tbl));
  }

  // shared-memory gathers
  auto smem_run = [&](auto kern, int es, const char* name) {
    const int row_bytes = ((2000 * es + 127) / 128) * 128;
    const int smem = 4 * row_bytes;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
    const int blocks = sms * per_sm, iters = 2048;
    const float ms =
        time_ms([&] { kern<<<blocks, 256, smem>>>(iters, sink); }, 10);
    const double el = (double)blocks * 256 * iters * 16;
    printf(", \"%s\": {\"ms\": %.4f, \"warps_per_sm\": %d, "
           "\"gelem_per_s\": %.1f, \"elem_per_sm_clk_at_1965\": %.2f}",
           name, ms, per_sm * 8, el / ms / 1e6,
           el / ms / 1e-3 / sms / 1.965e9);
  };
  smem_run(k_smem_gather<2, 0>, 2, "smem_gather_f16_random");
  smem_run(k_smem_gather<2, 1>, 2, "smem_gather_f16_conflict_free");
  smem_run(k_smem_gather<8, 0>, 8, "smem_gather_f64_random");
  smem_run(k_smem_gather<8, 1>, 8, "smem_gather_f64_conflict_free");

  // sequential L2 reads (8 MB and 32 MB buffers)
  for (size_t mb : {8, 32}) {
    const size_t bytes = mb << 20;
    int4* buf;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 0, bytes));
    const int blocks = sms * 8, reps = 64;
    const float ms = time_ms(
        [&] { k_l2_seq<<<blocks, 256>>>(buf, bytes / 16, reps, (int*)sink); },
        10);
    printf(", \"l2_seq_read_%zuMB\": {\"ms\": %.4f, \"gbs\": %.1f}", mb, ms,
           (double)bytes * reps / ms / 1e6);
    CK(cudaFree(buf));
  }

  // bulk row stream L2 -> shared memory: 2 KB rows (n = 1000 int16), 1 KB
  // (n = 500); stages of 32 rows; ring of nst stages (nst - 1 in flight);
  // 1 or 4 issuing warps
  for (int row_bytes : {2016, 1008}) {
    const int nrows = (int)((8u << 20) / row_bytes);  // 8 MB of rows
    unsigned char* mat;
    CK(cudaMalloc(&mat, (size_t)nrows * row_bytes));
    CK(cudaMemset(mat, 0, (size_t)nrows * row_bytes));
    auto k = k_bulk_rows;
    const int stride = (row_bytes + 127) / 128 * 128;
    for (int nw : {1, 4, 8}) {
      for (int nst = 2; nst <= 4; ++nst) {
        const int rps = 32;
        const int smem = nst * rps * stride;
        if (smem > 200 * 1024) break;
        CK(cudaFuncSetAttribute(
            k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        const int blocks = sms, stages = 512;
        const float ms = time_ms(
            [&] {
              k<<<blocks, 32 * nw, smem>>>(mat, nrows, row_bytes, rps, nst,
                                           stages, sink);
            },
            5);
        const double bytes = (double)blocks * stages * rps * row_bytes;
        printf(", \"bulk_rows%d_x32_warps%d_stages%d\": {\"inflight_kb\": "
               "%.0f, \"ms\": %.4f, \"gbs\": %.1f}",
               row_bytes, nw, nst, (nst - 1) * rps * row_bytes / 1024.0, ms,
               bytes / ms / 1e6);
      }
    }
    CK(cudaFree(mat));
  }
  printf("}\n");
  return 0;
}
