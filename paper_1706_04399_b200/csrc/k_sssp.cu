// Cost-matrix build (graph.py:41-78 + voxel.py:112-172): all-pairs
// obstacle-aware motion costs between viewpoint voxels.
//
// The reference runs one heap A* per pair i < j (N(N-1)/2 sequential
// searches).  Admissible A* returns the Dijkstra distance, so the device
// computes single-source shortest paths from every viewpoint instead, a
// batch of sources at a time: per source a fp64 distance array over the
// voxel grid and two frontier worklists.  Each round relaxes the 26
// neighbours of every frontier voxel with a 64-bit atomicMin on the distance
// bits (non-negative doubles order like their bit patterns) and appends
// improved voxels to the next worklist (a flag array dedupes).  Rounds repeat
// until every worklist is empty.  Because fl(d + w) is monotone in d, the
// fixed point is the minimum over paths of the left-to-right fp path sums,
// which is what Dijkstra returns.  The reference's A* returns the same bits
// for integer weights (all its scenes); otherwise it may be 1 ulp above.
//
// Then cost[i][j] = dist_min(i,j)(vox[max(i,j)]) (the reference computes
// each pair from its lower index), blocked pairs get
// VIRTUAL_SCALE * n * max_finite (1e6 when no finite edge).
#include <cstdlib>
#include <math.h>

#include <algorithm>
#include <vector>

#include "dpso_internal.cuh"

namespace dpso {

namespace {

struct SsspArgs {
  const uint8_t* occ;  // nx*ny*nz, C order (x, y, z), 1 = occupied
  int nx, ny, nz;
  int64_t V;
  double sc[26];       // step costs in NEIGHBOR_STEPS order
  int batch;
  const int64_t* src;  // batch: linear voxel of each source
  unsigned long long* dist;  // batch x V
  int32_t* q[2];       // batch x V worklists
  int32_t* qlen[2];    // batch lengths
  uint32_t* inq;       // batch x V: already in the next worklist
  int* next_total;     // voxels appended this round (all sources)
};

constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;

__global__ void k_sssp_init(SsspArgs a) {
  const int64_t total = (int64_t)a.batch * a.V;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    a.dist[e] = kInfBits;
    a.inq[e] = 0u;
  }
}

__global__ void k_sssp_seed(SsspArgs a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.batch) return;
  const int64_t v = a.src[s];
  a.dist[(size_t)s * a.V + v] = 0ull;  // bits of +0.0
  a.q[0][(size_t)s * a.V] = (int32_t)v;
  a.qlen[0][s] = 1;
  a.qlen[1][s] = 0;
}

__global__ void k_sssp_clear(int32_t* len, int batch, int* next_total) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < batch) len[s] = 0;
  if (s == 0) *next_total = 0;
}

// Before a round: reset the flags of the worklist about to be processed, so
// during the round flags only go 0 -> 1 (a voxel improved again while in the
// current worklist re-enters the next one and is re-relaxed then).
__global__ void k_sssp_unflag(SsspArgs a, int par) {
  const int s = blockIdx.y;
  const int len = a.qlen[par][s];
  const int32_t* cur = a.q[par] + (size_t)s * a.V;
  uint32_t* inq = a.inq + (size_t)s * a.V;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < len;
       k += gridDim.x * blockDim.x)
    inq[cur[k]] = 0u;
}

// grid: (blocks per source, batch); reads worklist `par`, writes par ^ 1
__global__ void __launch_bounds__(256) k_sssp_round(SsspArgs a, int par) {
  const int s = blockIdx.y;
  const int len = a.qlen[par][s];
  const int32_t* cur = a.q[par] + (size_t)s * a.V;
  int32_t* nxt = a.q[par ^ 1] + (size_t)s * a.V;
  unsigned long long* dist = a.dist + (size_t)s * a.V;
  uint32_t* inq = a.inq + (size_t)s * a.V;
  const int nyz = a.ny * a.nz;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < len;
       k += gridDim.x * blockDim.x) {
    const int v = cur[k];
    const double dv = __longlong_as_double((long long)dist[v]);
    const int x = v / nyz, y = (v / a.nz) % a.ny, z = v % a.nz;
    int d = 0;
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx)
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dz = -1; dz <= 1; ++dz) {
          if (dx == 0 && dy == 0 && dz == 0) continue;
          const int c = d++;
          const int X = x + dx, Y = y + dy, Z = z + dz;
          if (X < 0 || X >= a.nx || Y < 0 || Y >= a.ny || Z < 0 || Z >= a.nz)
            continue;
          const int u = (X * a.ny + Y) * a.nz + Z;
          if (a.occ[u]) continue;
          const double nd = __dadd_rn(dv, a.sc[c]);
          const unsigned long long nb =
              (unsigned long long)__double_as_longlong(nd);
          if (nb < dist[u]) {
            const unsigned long long old = atomicMin(&dist[u], nb);
            if (nb < old && atomicExch(&inq[u], 1u) == 0u) {
              const int pos = atomicAdd(&a.qlen[par ^ 1][s], 1);
              nxt[pos] = u;
              atomicAdd(a.next_total, 1);
            }
          }
        }
  }
}

// row i of the pairwise matrix: rowd[i * n + j] = dist_i(vox[j])
__global__ void k_sssp_gather(SsspArgs a, int first, int n,
                              const int64_t* vox, double* rowd) {
  const int s = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  rowd[(size_t)(first + s) * n + j] =
      __longlong_as_double((long long)a.dist[(size_t)s * a.V + vox[j]]);
}

// graph.py:58-78: cost[i][j] = cost[j][i] = A*(i -> j) for i < j; blocked
// pairs get the virtual cost.  max |finite| reduction first.
__global__ void k_cost_maxfinite(const double* rowd, int n,
                                 unsigned long long* mx) {
  unsigned long long m = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       e < (int64_t)n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    if (j <= i) continue;
    const double c = rowd[e];
    if (c < INFINITY) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(c);
      m = b > m ? b : m;
    }
  }
  atomicMax(mx, m);
}

__global__ void k_cost_fill(const double* rowd, int n,
                            const unsigned long long* mx, double* cost,
                            int64_t ld, uint8_t* virt, double* vcost_out) {
  const double maxf = __longlong_as_double((long long)*mx);
  // VIRTUAL_SCALE * n * max_finite, Python evaluation order
  const double vc =
      maxf > 0 ? __dmul_rn(__dmul_rn(1e3, (double)n), maxf) : 1e6;
  if (blockIdx.x == 0 && threadIdx.x == 0) *vcost_out = vc;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       e < (int64_t)n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    double c = 0.0;
    bool blocked = false;
    if (i != j) {
      const int lo = min(i, j), hi = max(i, j);
      c = rowd[(size_t)lo * n + hi];
      blocked = !(c < INFINITY);
      if (blocked) c = vc;
    }
    cost[(size_t)i * ld + j] = c;
    if (virt) virt[e] = blocked ? 1 : 0;
  }
}

__global__ void k_check_free(const uint8_t* occ, const int64_t* vox, int n,
                             int* bad) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n && occ[vox[j]]) atomicMin(bad, j);
}

// The build's workspace comes from the device's default stream-ordered
// pool; by default the pool returns freed memory to the driver at every
// synchronisation, so each build (and each batch's host poll) re-maps
// hundreds of MB.  Keep up to 1 GB cached (process-wide, once per device).
void keep_pool_memory() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 ||
      done[dev])
    return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = 1ull << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done[dev] = true;
}

}  // namespace

// Rows [src_begin, src_end) of the pairwise distance table:
// rows[(i - src_begin) * n + j] = dist_i(vox[j]) (+inf when unreachable).
// Every viewpoint is checked for occupancy first (all ranks of a sharded
// build fail the same way).
cudaError_t sssp_rows(const uint8_t* dev_occ, int nx, int ny, int nz,
                      const double* w, const int64_t* host_vox, int n,
                      int src_begin, int src_end, double* rows,
                      int* bad_viewpoint, cudaStream_t s) {
  *bad_viewpoint = -1;
  const int64_t V = (int64_t)nx * ny * nz;
  const int ns = src_end - src_begin;
  // concurrent sources: their distance arrays (8 B/voxel) capped at
  // ~256 MB (about twice the L2: a batch's hot frontier stays L2-resident)
  // (tools/sssp_batch_probe.py, profiles/r02/sssp_batch_probe.jsonl: ~220
  // sources build the office scene in 38 ms, all 816 at once in 58 ms),
  // under a 4 GB cap on dist + worklists + flags
  const int64_t per_src = 20 * V;
  const int64_t budget = 4ll << 30;
  int B = (int)std::max<int64_t>(
      1, std::min<int64_t>({(int64_t)std::max(ns, 1), budget / per_src,
                            (256ll << 20) / (8 * V)}));
  B = std::min(B, 1024);
  if (const char* ev = getenv("DPSO_SSSP_BATCH")) B = std::max(1, atoi(ev));
  keep_pool_memory();
  unsigned char* buf = nullptr;
  auto rnd = [](int64_t b) { return round_up(b, 256); };
  const size_t bytes = rnd(8 * B * V) + 2 * rnd(4 * B * V) + rnd(4 * B * V) +
                       2 * rnd(4 * B) + rnd(8 * (int64_t)n) + rnd(64);
  cudaError_t e = cudaMallocAsync(&buf, bytes, s);
  if (e) return e;
  size_t o = 0;
  auto take = [&](int64_t b) {
    unsigned char* p = buf + o;
    o += rnd(b);
    return p;
  };
  SsspArgs a;
  a.occ = dev_occ;
  a.nx = nx;
  a.ny = ny;
  a.nz = nz;
  a.V = V;
  {
    int c = 0;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          if (dx == 0 && dy == 0 && dz == 0) continue;
          // voxel.py:38: a1*alpha*alpha + a2*beta*beta + a3*gamma*gamma
          a.sc[c++] = w[0] * dx * dx + w[1] * dy * dy + w[2] * dz * dz;
        }
  }
  a.dist = (unsigned long long*)take(8 * B * V);
  a.q[0] = (int32_t*)take(4 * B * V);
  a.q[1] = (int32_t*)take(4 * B * V);
  a.inq = (uint32_t*)take(4 * B * V);
  a.qlen[0] = (int32_t*)take(4 * B);
  a.qlen[1] = (int32_t*)take(4 * B);
  int64_t* dvox = (int64_t*)take(8 * (int64_t)n);
  unsigned char* misc = take(64);
  int* next_total = (int*)misc;
  int* dbad = (int*)(misc + 16);
  a.next_total = next_total;
  if (!e) e = cudaMemcpyAsync(dvox, host_vox, 8 * (int64_t)n,
                              cudaMemcpyHostToDevice, s);
  int hbad = 0x7fffffff;
  if (!e) e = cudaMemcpyAsync(dbad, &hbad, 4, cudaMemcpyHostToDevice, s);
  if (!e) k_check_free<<<(n + 255) / 256, 256, 0, s>>>(dev_occ, dvox, n, dbad);
  if (!e) e = cudaMemcpyAsync(&hbad, dbad, 4, cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  if (!e && hbad != 0x7fffffff) {
    *bad_viewpoint = hbad;
    cudaFreeAsync(buf, s);
    return cudaSuccess;
  }
  const int blocks_per_src =
      (int)std::max<int64_t>(1, std::min<int64_t>(64, (V + 255) / 256));
  for (int first = src_begin; first < src_end && !e; first += B) {
    const int bs = std::min(B, src_end - first);
    a.batch = bs;
    a.src = dvox + first;
    const int64_t tot = (int64_t)bs * V;
    k_sssp_init<<<(int)std::min<int64_t>((tot + 255) / 256, 65535), 256, 0,
                  s>>>(a);
    k_sssp_seed<<<(bs + 255) / 256, 256, 0, s>>>(a);
    int par = 0;
    for (int round = 0;; ++round) {
      k_sssp_clear<<<(bs + 255) / 256, 256, 0, s>>>(a.qlen[par ^ 1], bs,
                                                    next_total);
      k_sssp_unflag<<<dim3(blocks_per_src, bs), 256, 0, s>>>(a, par);
      k_sssp_round<<<dim3(blocks_per_src, bs), 256, 0, s>>>(a, par);
      par ^= 1;
      if ((round & 7) == 7) {
        int h = 0;
        e = cudaMemcpyAsync(&h, next_total, 4, cudaMemcpyDeviceToHost, s);
        if (!e) e = cudaStreamSynchronize(s);
        if (e || h == 0) break;
      }
    }
    if (!e)
      k_sssp_gather<<<dim3((n + 255) / 256, bs), 256, 0, s>>>(
          a, first - src_begin, n, dvox, rows);
  }
  if (!e) e = cudaStreamSynchronize(s);
  cudaFreeAsync(buf, s);
  if (!e) e = cudaGetLastError();
  return e;
}

// graph.py:63-78 over a complete n x n distance table (upper triangle used)
cudaError_t cost_assemble(const double* rows, int n, double* dev_cost,
                          int64_t ld, uint8_t* dev_virtual,
                          double* host_vcost, cudaStream_t s) {
  unsigned char* misc = nullptr;
  cudaError_t e = cudaMallocAsync(&misc, 64, s);
  if (e) return e;
  unsigned long long* mx = (unsigned long long*)misc;
  double* dvc = (double*)(misc + 8);
  e = cudaMemsetAsync(mx, 0, 8, s);
  if (!e) {
    const int blocks = (int)std::min<int64_t>(((int64_t)n * n + 255) / 256,
                                              4096);
    k_cost_maxfinite<<<std::max(blocks, 1), 256, 0, s>>>(rows, n, mx);
    k_cost_fill<<<std::max(blocks, 1), 256, 0, s>>>(rows, n, mx, dev_cost, ld,
                                                    dev_virtual, dvc);
    e = cudaMemcpyAsync(host_vcost, dvc, 8, cudaMemcpyDeviceToHost, s);
  }
  if (!e) e = cudaStreamSynchronize(s);
  cudaFreeAsync(misc, s);
  if (!e) e = cudaGetLastError();
  return e;
}

cudaError_t build_cost_sssp(const uint8_t* dev_occ, int nx, int ny, int nz,
                            const double* w, const int64_t* host_vox, int n,
                            double* dev_cost, int64_t ld, uint8_t* dev_virtual,
                            double* host_vcost, int* bad_viewpoint,
                            cudaStream_t s) {
  double* rows = nullptr;
  cudaError_t e = cudaMallocAsync(&rows, 8 * (size_t)n * n, s);
  if (e) return e;
  e = sssp_rows(dev_occ, nx, ny, nz, w, host_vox, n, 0, n, rows,
                bad_viewpoint, s);
  if (!e && *bad_viewpoint < 0)
    e = cost_assemble(rows, n, dev_cost, ld, dev_virtual, host_vcost, s);
  cudaFreeAsync(rows, s);
  if (!e) e = cudaStreamSynchronize(s);
  return e;
}

}  // namespace dpso
