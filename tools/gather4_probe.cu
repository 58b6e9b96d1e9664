// Row-stream probe for the band scan's producer side: 32 random rows of an
// L2-resident matrix per stage into shared memory, as
//   bulk     one cp.async.bulk per row (the band scan today)
//   gather4  one cp.async.bulk.tensor.2d.tile::gather4 per 4 rows (sm_100:
//            a 2-D tensor map, one column start and four row indices)
// at 1-KB and 2-KB rows, 1/2/4/8 issuing warps.  The question is whether a
// gather4 costs the TMA unit one row's issue time or four (answer,
// profiles/r02/gather4_probe.json: about 2.5 rows' time: 1-KB rows 7.8 TB/s
// bulk vs 12.3 TB/s gather4, 2-KB rows 14.4 vs 20.2 TB/s).
//
// Output: one JSON object on stdout (tools/gather4_probe.py builds + runs).
#include <cuda.h>
#include <cudaTypedefs.h>
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
__device__ __forceinline__ uint32_t s32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// MODE 0 bulk, 1 gather4.  Ring of nst stages of 32 rows; every warp issues
// its share of each stage (one expect-tx arrival per warp); the stage is
// consumed at once (one word read, CTA barrier) before it is reissued.
template <int MODE>
__global__ void k_rows(const __grid_constant__ CUtensorMap tm,
                       const unsigned char* mat, int nrows, int row_bytes,
                       int box_bytes, int nst, int stages, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const uint32_t stride = (uint32_t)box_bytes;  // bytes per staged row
  constexpr int rps = 32;
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
    unsigned char* stage = sm + (size_t)b * rps * stride;
    if (MODE == 0) {
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
            "[%0], [%1], %2, [%3];" ::"r"(s32(stage + (size_t)r * stride)),
            "l"(mat + (size_t)row * row_bytes), "r"((uint32_t)row_bytes),
            "r"(s32(&bar[b]))
            : "memory");
      }
    } else {
      // 8 groups of 4 rows; warp w issues groups w, w + nw, ...
      int mine = 0;
      for (int g = warp; g < rps / 4; g += nw) ++mine;
      if (lane == 0)
        asm volatile(
            "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                s32(&bar[b])),
            "r"((uint32_t)(mine * 4 * box_bytes))
            : "memory");
      __syncwarp();
      const int g = warp + nw * lane;
      if (lane < mine) {
        int rw[4];
        for (int k = 0; k < 4; ++k)
          rw[k] = (int)(hash32(blockIdx.x * 100003u + st * 32 + 4 * g + k) %
                        nrows);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4."
            "mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
            "[%7];" ::"r"(s32(stage + (size_t)4 * g * stride)),
            "l"(&tm), "r"(0), "r"(rw[0]), "r"(rw[1]), "r"(rw[2]), "r"(rw[3]),
            "r"(s32(&bar[b]))
            : "memory");
      }
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
    __syncthreads();
  }
  if (acc == 1.2345f) sink[threadIdx.x] = acc;
}

// check: gather4 rows land where expected (row k of a group at k * box)
__global__ void k_check(const __grid_constant__ CUtensorMap tm,
                        const unsigned char* mat, int row_bytes,
                        int box_bytes, int dst_off, int* bad) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  const int rows[4] = {7, 3, 1000, 42};
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile(
        "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
            s32(&bar)),
        "r"((uint32_t)(4 * box_bytes))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4."
        "mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
        "[%7];" ::"r"(s32(sm + dst_off)),
        "l"(&tm), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]),
        "r"(rows[3]), "r"(s32(&bar))
        : "memory");
  }
  __syncthreads();
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(s32(&bar)),
      "r"(0u)
      : "memory");
  for (int e = threadIdx.x; e < 4 * row_bytes; e += blockDim.x) {
    const int k = e / row_bytes, c = e % row_bytes;
    if (sm[dst_off + (size_t)k * box_bytes + c] !=
        mat[(size_t)rows[k] * row_bytes + c])
      atomicAdd(bad, 1);
  }
}

template <typename F>
float time_ms(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
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
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode,
                             cudaEnableDefault, &q));
  if (!encode) {
    printf("{\"error\": \"no cuTensorMapEncodeTiled\"}\n");
    return 1;
  }
  float* sink;
  CK(cudaMalloc(&sink, 1 << 20));
  int* bad;
  CK(cudaMalloc(&bad, 4));
  printf("{\"sms\": %d", sms);
  const int nrows = 4 * 2000;  // 4 rotated versions of a 2000-row matrix
  for (int row_bytes : {1008, 2016}) {
    // element type: 4-byte words for 1-KB rows, 8-byte for 2-KB rows, so a
    // 256-element box covers the row
    const int es = row_bytes <= 1024 ? 4 : 8;
    const int box_el = (row_bytes + es - 1) / es;
    const int box_bytes = ((box_el * es + 127) / 128) * 128;
    const int pitch = ((row_bytes + 15) / 16) * 16;
    unsigned char* mat;
    CK(cudaMalloc(&mat, (size_t)nrows * pitch));
    {
      unsigned char* h = (unsigned char*)malloc((size_t)nrows * pitch);
      for (size_t i = 0; i < (size_t)nrows * pitch; ++i)
        h[i] = (unsigned char)(i * 2654435761u >> 13);
      CK(cudaMemcpy(mat, h, (size_t)nrows * pitch, cudaMemcpyHostToDevice));
      free(h);
    }
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)(pitch / es), (cuuint64_t)nrows};
    cuuint64_t gstride[1] = {(cuuint64_t)pitch};
    cuuint32_t box[2] = {(cuuint32_t)(box_bytes / es), 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tm,
                        es == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                : CU_TENSOR_MAP_DATA_TYPE_INT64,
                        2, mat, gdim, gstride, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf(", \"encode_%d\": %d", row_bytes, (int)r);
    if (r != CUDA_SUCCESS) continue;
    const int check_smem = 4 * box_bytes + 128;
    CK(cudaFuncSetAttribute(k_check,
                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                            check_smem));
    // destinations must be 128-byte aligned: a 16-byte-aligned one faults
    // with "misaligned address" (measured; the fault is sticky, so only
    // aligned offsets are checked here)
    for (int dst_off : {0, 128}) {
      CK(cudaMemset(bad, 0, 4));
      k_check<<<1, 128, check_smem>>>(tm, mat,
                                      row_bytes < pitch ? row_bytes : pitch,
                                      box_bytes, dst_off, bad);
      cudaError_t e = cudaDeviceSynchronize();
      int hbad = -1;
      if (e == cudaSuccess)
        CK(cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost));
      printf(", \"gather4_check_%d_dst%d\": \"%s\"", row_bytes, dst_off,
             e != cudaSuccess ? cudaGetErrorString(e)
                              : (hbad == 0 ? "ok" : "mismatch"));
      if (e != cudaSuccess) {
        printf("}\n");
        return 1;
      }
    }
    const int nst = 3, stages = 2000;
    const int smem = nst * 32 * box_bytes;
    for (int mode = 0; mode < 2; ++mode) {
      for (int nw : {1, 2, 4, 8}) {
        auto kern = mode == 0 ? k_rows<0> : k_rows<1>;
        CK(cudaFuncSetAttribute(
            kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        const float ms = time_ms(
            [&] {
              kern<<<sms, 32 * nw, smem>>>(tm, mat, nrows, row_bytes,
                                           box_bytes, nst, stages, sink);
            },
            5);
        const double bytes = (double)sms * stages * 32 * row_bytes;
        const double copies = (double)sms * stages * (mode ? 8 : 32);
        printf(", \"%s_%dB_w%d\": {\"ms\": %.4f, \"tbs\": %.2f, "
               "\"sm_clk_per_copy_at_1965\": %.1f}",
               mode ? "gather4" : "bulk", row_bytes, nw, ms,
               bytes / ms / 1e9, ms * 1e-3 * 1.965e9 / (copies / sms));
      }
    }
    CK(cudaFree(mat));
  }
  printf("}\n");
  return 0;
}
