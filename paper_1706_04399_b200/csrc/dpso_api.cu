// C ABI (include/dpso.h): context lifecycle, workspace layout, the
// device-resident generation loop and the kernel-level entry points.
//
// One generation (solver.py:292-328) is a fixed sequence of launches that all
// read their control flags from device memory (DevCtl), so it is captured
// once into a CUDA graph and replayed; data-dependent branches (mutation
// period, 2-opt trigger, stall break) are flags checked at kernel entry.  The
// host polls `done` once per batch of generations.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "dpso_internal.cuh"
#include <nvtx3/nvToolsExt.h>
#include "philox.cuh"

using namespace dpso;

namespace dpso {
cudaError_t set_dyn_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> done;
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find(kernel);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(
      kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done[kernel] = bytes;
  return e;
}
}  // namespace dpso

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  std::string m = std::string(where) + ": " + cudaGetErrorString(e);
  return fail(DPSO_ECUDA, m);
}
}  // namespace

namespace dpso {
// the thread-local last error for the other translation units
int api_fail(int code, const char* msg) { return fail(code, msg); }
}  // namespace dpso

namespace {

#define CK(call)                                        \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

struct Layout {
  size_t off_ctl, off_streams, off_mut_start, off_init_start, off_x, off_pbest, off_vmap, off_vinv,
      off_vel, off_vel_len, off_fit, off_pfit, off_dcache, off_gbest,
      off_conv, off_tores, off_chunk_tab, off_rank, off_hash, off_flag, off_pbflag,
      off_sidx, off_order, off_surv, off_keep, off_ev_slot, off_ev_k,
      off_ev_cursor, off_ev_end, off_ev_idx, off_mstream, off_init_buf,
      off_init_state, off_init_cursor, off_init_aux, off_init_anchor, off_seed, off_cost32,
      off_stats, off_band_cols, off_bound, total;
  int64_t vel_cap;
  int chunks;
};

// Initial velocity-list capacity for w < 1 (entries per particle).  A list
// grows by at most 2(n - 1) per generation (k1, k2 <= n - 1) and shrinks to
// round(w len) first, so it stays below ~(2n)/(1 - w); the workspace holds
// up to 64n + 64 and ensure_velocity() moves the lists to a larger owned
// buffer before any batch of generations could outgrow it (solver.py:
// 213-216 has no bound).
int64_t vel_capacity(const dpso_params* p, int n) {
  if (p->inertia >= 1.0) return 0;
  double cap = (2.0 * n + 1.0) / (1.0 - p->inertia) + 8.0;
  if (cap > 64.0 * n + 64) cap = 64.0 * n + 64;
  return (int64_t)cap;
}

Layout make_layout(const dpso_params* prm, int n) {
  Layout L;
  const int64_t P = prm->n_particles;
  const int64_t np = round_up(n, 8);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = round_up(o + bytes, 256);
    return at;
  };
  L.chunks = two_opt_pick_chunks(n, (int32_t)P);
  L.vel_cap = vel_capacity(prm, n);
  L.off_ctl = take(sizeof(DevCtl));
  L.off_streams = take(sizeof(PcgState) * (P + 2));
  L.off_mut_start = take(2 * sizeof(PcgState));
  L.off_init_start = take(sizeof(PcgState));
  L.off_x = take(2 * P * np);
  L.off_pbest = take(2 * P * np);
  // vmap: w == 1 the composed velocity (solver.py:197-209); w < 1 the value
  // map of the whole transposition list, with its inverse (k_update_wl)
  L.off_vmap = take(2 * P * np);
  L.off_vinv = take(prm->inertia < 1.0 ? 2 * P * np : 0);
  L.off_vel = take(L.vel_cap ? 4 * P * (L.vel_cap + 2 * (int64_t)n) : 0);
  L.off_vel_len = take(4 * P);
  L.off_fit = take(8 * P);
  L.off_pfit = take(8 * P);
  L.off_dcache = take(8 * P * np);
  L.off_gbest = take(2 * np);
  L.off_conv = take(8 * ((int64_t)prm->max_generations + 1));
  // partial argmins, the FILTER32 overflow list (count + tasks), the scan's
  // task counter
  L.off_tores = take(sizeof(TwoOptRes) * P * L.chunks + 4 * (2 + P * L.chunks));
  L.off_chunk_tab = take(16 * L.chunks);
  L.off_rank = take(4 * P);
  L.off_hash = take(8 * P);
  L.off_flag = take(4 * P);
  L.off_pbflag = take(4 * P);
  L.off_sidx = take(4 * P);
  L.off_order = take(4 * P);
  L.off_surv = take(4 * P);
  L.off_keep = take(4 * P);
  L.off_ev_slot = take(4 * P);
  L.off_ev_k = take(2 * 4 * P);
  L.off_ev_cursor = take(2 * 8 * P);
  L.off_ev_end = take(2 * 8 * P);
  L.off_ev_idx = take(2 * P * np);
  L.off_mstream = take(prm->use_mutation && prm->rng_mode == DPSO_RNG_NUMPY
                           ? 2 * 6 * mstream_words(n, P)  // u32 + u16 skip
                           : 0);
  L.off_init_cursor = take(8 * P);
  L.off_init_buf = take(prm->rng_mode == DPSO_RNG_NUMPY ? 4 * init_buf_words(n, P) : 0);
  L.off_init_state = take(64);
  {
    const bool par = prm->rng_mode == DPSO_RNG_NUMPY && init_parallel_ok(n, (int)P);
    L.off_init_aux = take(par ? 3 * 4 * init_buf_words(n, P) : 0);
    L.off_init_anchor = take(par ? 8 * (P + 2) : 0);
  }
  L.off_seed = take(2 * np);
  // fp32 + fp16 rows, then the band scan's int16 row versions
  L.off_cost32 = take(prm->use_edge_exchange
                          ? round_up(6 * (int64_t)n * np, 256) +
                                band_rows_bytes(n)
                          : 0);
  L.off_stats = take(sizeof(CostStats));
  L.off_band_cols =
      take(prm->use_edge_exchange ? band_cols_bytes(n, P) : 0);
  L.off_bound = take(prm->use_edge_exchange ? bound_bytes(n, P) : 0);
  L.total = o;
  return L;
}

int check_params(const dpso_params* p, int n) {
  // messages follow solver.py:139-153
  if (!p) return fail(DPSO_EINVAL, "params is NULL");
  if (p->n_particles < 3) return fail(DPSO_EINVAL, "n_particles must be >= 3");
  const char* names[3] = {"inertia", "cognitive", "social"};
  double vals[3] = {p->inertia, p->cognitive, p->social};
  for (int i = 0; i < 3; ++i)
    if (!(vals[i] >= 0.0 && vals[i] <= 1.0)) {
      char buf[128];
      snprintf(buf, sizeof buf, "%s must be in [0, 1], got %g", names[i],
               vals[i]);
      return fail(DPSO_EINVAL, buf);
    }
  if (p->max_generations < 1)
    return fail(DPSO_EINVAL, "max_generations must be >= 1");
  if (p->stall_generations < 1)
    return fail(DPSO_EINVAL, "stall_generations must be >= 1");
  if (p->mutation_period < 1)
    return fail(DPSO_EINVAL, "mutation_period must be >= 1");
  if (!(p->seed_fraction >= 0.0 && p->seed_fraction <= 1.0))
    return fail(DPSO_EINVAL, "seed_fraction must be in [0, 1]");
  if (n < 2 || n > kMaxN)
    return fail(DPSO_EINVAL, "n must be in [2, 65535] for the device path");
  {
    // the update kernel keeps a particle's arrays in shared memory: 16
    // bytes per node (w < 1, or n <= 14000), 10 beyond (k_update_w1_lowmem)
    const int bpn = (p->inertia < 1.0 || n <= 14000) ? 16 : 10;
    int dev = 0, smax = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                               dev) == cudaSuccess &&
        smax > 0 && (int64_t)bpn * round_up(n, 8) > smax - 1024) {
      char buf[160];
      snprintf(buf, sizeof buf,
               "n = %d exceeds the device update kernel's shared memory "
               "(max n = %d on this device)",
               n, (int)((smax - 1024) / bpn / 8 * 8));
      return fail(DPSO_EINVAL, buf);
    }
  }
  if (p->rng_mode != DPSO_RNG_NUMPY && p->rng_mode != DPSO_RNG_PHILOX)
    return fail(DPSO_EINVAL, "unknown rng_mode");
  return DPSO_OK;
}

}  // namespace

struct dpso_ctx {
  dpso_params prm;
  int n;
  int dev = -1;  // the device of the workspace (every entry runs on it)
  Layout L;
  unsigned char* ws;
  cudaStream_t user;
  cudaStream_t stream;
  cudaStream_t stream2;  // fork for the mutation-stream walk
  cudaEvent_t ev, ev_fork, ev_join;
  cudaEvent_t ev_fix;  // the mutating graph's stream state is final
  cudaGraphExec_t graph;        // a generation with the mutation call
  cudaGraphExec_t graph_plain;  // a generation without it (gen % period)
  int64_t gen_next = 1;         // generation the next launch runs
  bool have_cost, have_streams, initialized;
  SwarmView v;
  DevCtl* host_ctl;  // pinned
  int init_path = -1;
  uint32_t* vel_owned = nullptr;  // grown velocity lists (w < 1)
};

// NVTX ranges around the host entry points (nsys / ncu --nvtx show the
// solve's phases: cost preparation, init, generation batches, exchanges)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Every entry that takes a context runs on the context's device (the device
// of its workspace) whatever device is current in the calling thread, and
// gives the caller its current device back on return.
struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev)
      cudaSetDevice(dev);
    else
      prev = -1;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// the device a device pointer lives on, -1 if it is not a device pointer
static int ptr_device(const void* p) {
  cudaPointerAttributes at;
  int d = -1;
  if (p && cudaPointerGetAttributes(&at, p) == cudaSuccess &&
      at.type == cudaMemoryTypeDevice)
    d = at.device;
  cudaGetLastError();
  return d;
}

static int sync_in(dpso_ctx* c) {
  CK(cudaEventRecord(c->ev, c->user));
  CK(cudaStreamWaitEvent(c->stream, c->ev, 0));
  return DPSO_OK;
}
// entries that rewrite what the mutation-stream walk reads (the streams,
// the swarm state) first wait for a walk still running on stream2
static int join_walk(dpso_ctx* c) {
  CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  return DPSO_OK;
}
static int sync_out(dpso_ctx* c) {
  CK(cudaEventRecord(c->ev, c->stream));
  CK(cudaStreamWaitEvent(c->user, c->ev, 0));
  return DPSO_OK;
}

static const char* g_stage = "";

// One generation.  With mutation on, the mutation-stream walk runs on a
// forked stream (s2) concurrently with the update and the dedupe pipeline.
// walk: whether the graph runs the next mutation call's stream walk
// (launch_mutation_walk) on the forked stream s2 after this generation's
// mutation call, overlapping its swap, select and 2-opt (mutation every
// generation, or one graph for all generations: kWalkAfterMutation), or
// leaves it to launch_generation (kWalkNone)
enum { kWalkAfterMutation, kWalkNone };

static cudaError_t enqueue_generation(const SwarmView& v, cudaStream_t s,
                                      cudaStream_t s2, cudaEvent_t fork,
                                      cudaEvent_t join,
                                      bool with_mutation = true,
                                      int walk = kWalkAfterMutation,
                                      cudaEvent_t fix = nullptr) {
  cudaError_t e;
#define STAGE(name, call)      \
  do {                         \
    g_stage = name;            \
    if ((e = (call))) return e; \
  } while (0)
  const bool mut = v.use_mutation && with_mutation;
  bool forked = false;
  STAGE("gen_begin", launch_gen_begin(v, s));
  STAGE("update", launch_update(v, s));
  if (mut) {
    STAGE("mutation_pre", launch_mutation_pre(v, s));
    STAGE("mutation_post", launch_mutation_post(v, s));
    // kWalkNone: the next call's walk (launched by the host after this
    // graph) may start as soon as the stream state is final - an external
    // event record node it waits on
    if (walk == kWalkNone && fix)
      STAGE("fix_event",
            cudaEventRecordWithFlags(fix, s, cudaEventRecordExternal));
    if (walk == kWalkAfterMutation) {
      // the next call's stream walk overlaps the rest of this generation
      STAGE("fork", cudaEventRecord(fork, s));
      STAGE("fork", cudaStreamWaitEvent(s2, fork, 0));
      STAGE("mutation_walk", launch_mutation_walk(v, s2));
      STAGE("join", cudaEventRecord(join, s2));
      forked = true;
    }
    STAGE("mutation_swap", launch_mutation_swap(v, s));
  }
  if (v.use_edge_exchange) {
    STAGE("select", launch_select(v, false, s));
    STAGE("two_opt", launch_two_opt(v, s));
    STAGE("finalize", launch_finalize(v, s));
  } else {
    STAGE("select+finalize", launch_select(v, true, s));
  }
  if (forked) STAGE("join", cudaStreamWaitEvent(s, join, 0));
#undef STAGE
  g_stage = "";
  return cudaSuccess;
}

extern "C" {

const char* dpso_last_error(void) { return g_err.c_str(); }

namespace {
// shared argument checks of the cost-build entry points; fills lin
int check_build_args(const uint8_t* dev_occ, int32_t nx, int32_t ny,
                     int32_t nz, const double* host_weights,
                     const int32_t* host_vox, int32_t n,
                     std::vector<int64_t>& lin) {
  if (!dev_occ || !host_weights || !host_vox || n < 1 || nx < 1 || ny < 1 ||
      nz < 1)
    return fail(DPSO_EINVAL, "bad arguments");
  if ((int64_t)nx * ny * nz >= (1ll << 31))
    return fail(DPSO_EINVAL, "grid too large for 32-bit voxel indices");
  for (int i = 0; i < 3; ++i)
    if (!(host_weights[i] >= 0.0))
      return fail(DPSO_EINVAL, "axis weights must be non-negative");
  lin.resize(n);
  for (int j = 0; j < n; ++j) {
    const int x = host_vox[3 * j], y = host_vox[3 * j + 1],
              z = host_vox[3 * j + 2];
    if (x < 0 || x >= nx || y < 0 || y >= ny || z < 0 || z >= nz)
      return fail(DPSO_EINVAL, "viewpoint voxel outside the grid");
    lin[j] = ((int64_t)x * ny + y) * nz + z;
  }
  return DPSO_OK;
}

int occupied_fail(const int32_t* host_vox, int bad) {
  char buf[160];
  snprintf(buf, sizeof buf, "viewpoint %d maps to occupied voxel (%d, %d, %d)",
           bad, host_vox[3 * bad], host_vox[3 * bad + 1],
           host_vox[3 * bad + 2]);
  return fail(DPSO_EINVAL, buf);
}
}  // namespace

int dpso_build_cost(const uint8_t* dev_occ, int32_t nx, int32_t ny,
                    int32_t nz, const double* host_weights,
                    const int32_t* host_vox, int32_t n, double* dev_cost,
                    int64_t ld, uint8_t* dev_virtual, double* host_vcost,
                    void* cuda_stream) {
  std::vector<int64_t> lin;
  if (int r = check_build_args(dev_occ, nx, ny, nz, host_weights, host_vox, n,
                               lin))
    return r;
  if (!dev_cost || !host_vcost || ld < n)
    return fail(DPSO_EINVAL, "bad arguments");
  DevGuard g(ptr_device(dev_occ));
  NvtxRange nv("dpso_build_cost");
  int bad = -1;
  cudaError_t e = build_cost_sssp(dev_occ, nx, ny, nz, host_weights,
                                  lin.data(), n, dev_cost, ld, dev_virtual,
                                  host_vcost, &bad, (cudaStream_t)cuda_stream);
  if (e) return cuda_fail(e, "build_cost_sssp");
  if (bad >= 0) return occupied_fail(host_vox, bad);
  return DPSO_OK;
}

int dpso_build_cost_rows(const uint8_t* dev_occ, int32_t nx, int32_t ny,
                         int32_t nz, const double* host_weights,
                         const int32_t* host_vox, int32_t n,
                         int32_t src_begin, int32_t src_end, double* dev_rows,
                         void* cuda_stream) {
  std::vector<int64_t> lin;
  if (int r = check_build_args(dev_occ, nx, ny, nz, host_weights, host_vox, n,
                               lin))
    return r;
  if (src_begin < 0 || src_end < src_begin || src_end > n ||
      (src_end > src_begin && !dev_rows))
    return fail(DPSO_EINVAL, "bad source range");
  DevGuard g(ptr_device(dev_occ));
  NvtxRange nv("dpso_build_cost_rows");
  int bad = -1;
  cudaError_t e = sssp_rows(dev_occ, nx, ny, nz, host_weights, lin.data(), n,
                            src_begin, src_end, dev_rows, &bad,
                            (cudaStream_t)cuda_stream);
  if (e) return cuda_fail(e, "sssp_rows");
  if (bad >= 0) return occupied_fail(host_vox, bad);
  return DPSO_OK;
}

int dpso_build_cost_assemble(const double* dev_rows, int32_t n,
                             double* dev_cost, int64_t ld,
                             uint8_t* dev_virtual, double* host_vcost,
                             void* cuda_stream) {
  if (!dev_rows || !dev_cost || !host_vcost || n < 1 || ld < n)
    return fail(DPSO_EINVAL, "bad arguments");
  DevGuard g(ptr_device(dev_rows));
  NvtxRange nv("dpso_build_cost_assemble");
  cudaError_t e = cost_assemble(dev_rows, n, dev_cost, ld, dev_virtual,
                                host_vcost, (cudaStream_t)cuda_stream);
  if (e) return cuda_fail(e, "cost_assemble");
  return DPSO_OK;
}

int dpso_philox4x32_10(const uint32_t* ctr, uint64_t key, uint32_t* out) {
  if (!ctr || !out) return fail(DPSO_EINVAL, "null argument");
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  philox4x32_10(c, key);
  for (int i = 0; i < 4; ++i) out[i] = c[i];
  return DPSO_OK;
}

const char* dpso_version(void) {
  return "paper_1706_04399_b200 dpso 0.1.0 (sm_100a)";
}

int dpso_workspace_size(const dpso_params* prm, int32_t n, size_t* bytes) {
  int rc = check_params(prm, n);
  if (rc) return rc;
  *bytes = make_layout(prm, n).total;
  return DPSO_OK;
}

// Pinned control blocks are recycled process-wide: cudaMallocHost /
// cudaFreeHost pin and unpin pages and can take milliseconds each, which a
// short fit() would pay on every call.
static std::mutex g_pinned_mu;
static std::vector<DevCtl*> g_pinned_free;

static DevCtl* pinned_ctl_get() {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (!g_pinned_free.empty()) {
      DevCtl* p = g_pinned_free.back();
      g_pinned_free.pop_back();
      return p;
    }
  }
  DevCtl* p = nullptr;
  if (cudaMallocHost(&p, sizeof(DevCtl)) != cudaSuccess) return nullptr;
  return p;
}

static void pinned_ctl_put(DevCtl* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_pinned_free.push_back(p);
}

int dpso_create(const dpso_params* prm, int32_t n, void* dev_workspace,
                size_t workspace_bytes, void* cuda_stream, dpso_ctx** out) {
  int wdev = -1;
  if (dev_workspace) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, dev_workspace) == cudaSuccess &&
        at.type == cudaMemoryTypeDevice)
      wdev = at.device;
    cudaGetLastError();
  }
  DevGuard g_(wdev);
  int rc = check_params(prm, n);
  if (rc) return rc;
  Layout L = make_layout(prm, n);
  if (!dev_workspace || workspace_bytes < L.total)
    return fail(DPSO_EINVAL, "workspace too small");
  dpso_ctx* c = new dpso_ctx();
  c->prm = *prm;
  c->n = n;
  c->dev = wdev;
  c->L = L;
  c->ws = (unsigned char*)dev_workspace;
  c->user = (cudaStream_t)cuda_stream;
  c->graph = nullptr;
  c->graph_plain = nullptr;
  c->have_cost = c->have_streams = c->initialized = false;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e) {
    delete c;
    return cuda_fail(e, "cudaStreamCreate");
  }
  cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_fix, cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking);
  c->host_ctl = pinned_ctl_get();
  SwarmView& v = c->v;
  memset(&v, 0, sizeof v);
  v.n = n;
  v.np = (int32_t)round_up(n, 8);
  v.P = prm->n_particles;
  v.max_generations = prm->max_generations;
  v.stall_generations = prm->stall_generations;
  v.mutation_period = prm->mutation_period;
  v.use_mutation = prm->use_mutation ? 1 : 0;
  v.use_edge_exchange = prm->use_edge_exchange ? 1 : 0;
  v.rng_mode = prm->rng_mode;
  v.philox_seed = prm->philox_seed;
  v.inertia = prm->inertia;
  v.cognitive = prm->cognitive;
  v.social = prm->social;
  unsigned char* w = c->ws;
  v.ctl = (DevCtl*)(w + L.off_ctl);
  v.streams = (PcgState*)(w + L.off_streams);
  v.mut_start = (PcgState*)(w + L.off_mut_start);
  v.init_start = (PcgState*)(w + L.off_init_start);
  v.x = (uint16_t*)(w + L.off_x);
  v.pbest = (uint16_t*)(w + L.off_pbest);
  v.vmap = (uint16_t*)(w + L.off_vmap);
  v.vinv = prm->inertia < 1.0 ? (uint16_t*)(w + L.off_vinv) : nullptr;
  v.vel = L.vel_cap ? (uint32_t*)(w + L.off_vel) : nullptr;
  v.vel_len = (int32_t*)(w + L.off_vel_len);
  v.vel_cap = L.vel_cap;
  v.fit = (double*)(w + L.off_fit);
  v.pfit = (double*)(w + L.off_pfit);
  v.dcache = (double*)(w + L.off_dcache);
  v.gbest = (uint16_t*)(w + L.off_gbest);
  v.conv = (double*)(w + L.off_conv);
  v.tores = (TwoOptRes*)(w + L.off_tores);
  v.chunks = L.chunks;
  v.chunk_tab = (int32_t*)(w + L.off_chunk_tab);
  v.rank = (int32_t*)(w + L.off_rank);
  v.hash = (uint64_t*)(w + L.off_hash);
  v.flag = (int32_t*)(w + L.off_flag);
  v.pbflag = (int32_t*)(w + L.off_pbflag);
  v.sidx = (int32_t*)(w + L.off_sidx);
  v.order = (int32_t*)(w + L.off_order);
  v.surv_list = (int32_t*)(w + L.off_surv);
  v.keep = (int32_t*)(w + L.off_keep);
  v.ev_slot = (int32_t*)(w + L.off_ev_slot);
  v.ev_k = (int32_t*)(w + L.off_ev_k);
  v.ev_cursor = (uint64_t*)(w + L.off_ev_cursor);
  v.ev_end = (uint64_t*)(w + L.off_ev_end);
  v.ev_idx = (uint16_t*)(w + L.off_ev_idx);
  v.mstream = (uint32_t*)(w + L.off_mstream);
  v.mstream_cap = prm->use_mutation && prm->rng_mode == DPSO_RNG_NUMPY
                      ? mstream_words(n, v.P)
                      : 0;
  v.init_cursor = (uint64_t*)(w + L.off_init_cursor);
  v.init_buf = (uint32_t*)(w + L.off_init_buf);
  v.init_buf_cap = prm->rng_mode == DPSO_RNG_NUMPY ? init_buf_words(n, v.P) : 0;
  v.init_state = (void*)(w + L.off_init_state);
  v.init_parallel = prm->rng_mode == DPSO_RNG_NUMPY && init_parallel_ok(n, v.P);
  v.init_aux = (int32_t*)(w + L.off_init_aux);
  v.init_anchor = (int64_t*)(w + L.off_init_anchor);
  std::vector<int32_t> tab(4 * L.chunks);
  two_opt_chunk_table(n, L.chunks, tab.data());
  if ((rc = sync_in(c))) {
    dpso_destroy(c);
    return rc;
  }
  e = cudaMemcpyAsync(v.chunk_tab, tab.data(), 4 * tab.size(),
                      cudaMemcpyHostToDevice, c->stream);
  if (!e) e = cudaMemsetAsync(v.ctl, 0, sizeof(DevCtl), c->stream);
  if (!e) e = cudaStreamSynchronize(c->stream);
  if (e) {
    dpso_destroy(c);
    return cuda_fail(e, "dpso_create");
  }
  *out = c;
  return DPSO_OK;
}

int dpso_set_cost(dpso_ctx* c, const double* dev_cost, int64_t ld) {
  DevGuard g_(c ? c->dev : -1);
  NvtxRange nv_("dpso_set_cost (2-opt plan: cost prep, row versions)");
  if (!c || !dev_cost) return fail(DPSO_EINVAL, "null argument");
  if (ld < round_up(c->n, 2) || (ld & 1) || ((uintptr_t)dev_cost & 15))
    return fail(DPSO_EINVAL,
                "cost matrix needs an even ld >= n (padded) and 16-B "
                "alignment");
  c->v.cost = dev_cost;
  c->v.ld = ld;
  TwoOptPlan& pl = c->v.plan;
  memset(&pl, 0, sizeof pl);
  pl.cost = dev_cost;
  pl.ld = ld;
  pl.ld32 = c->v.np;
  pl.mode = kScanFP64;
  pl.es = 4;
  pl.dscale = 1.f;
  if (c->prm.use_edge_exchange) {
    float* c32 = (float*)(c->ws + c->L.off_cost32);
    uint16_t* c16 = (uint16_t*)(c32 + (size_t)c->n * c->v.np);
    CostStats* st = (CostStats*)(c->ws + c->L.off_stats);
    int rc = sync_in(c);
    if (rc) return rc;
    unsigned char* band = band_rows_bytes(c->n)
                              ? (unsigned char*)c32 +
                                    round_up(6 * (int64_t)c->n * c->v.np, 256)
                              : nullptr;
    void* bbuf = bound_bytes(c->n, c->prm.n_particles)
                     ? (void*)(c->ws + c->L.off_bound)
                     : nullptr;
    CK(two_opt_prepare(dev_cost, ld, c->n, c->v.np, c32, c16, band, st,
                       c->stream, &pl, bbuf));
    pl.band_cols = (int32_t*)(c->ws + c->L.off_band_cols);
    pl.band_cols_cap = c->prm.n_particles;
  }
  c->have_cost = true;
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  if (c->graph_plain) {
    cudaGraphExecDestroy(c->graph_plain);
    c->graph_plain = nullptr;
  }
  return DPSO_OK;
}

int dpso_scan_mode(dpso_ctx* c) { return c ? c->v.plan.mode : -1; }

int dpso_scan_band(dpso_ctx* c) { return c ? c->v.plan.band_mode : -1; }

int dpso_scan_bound(dpso_ctx* c) { return c ? c->v.plan.bound : -1; }

int dpso_band_runs(dpso_ctx* c) {
  if (!c) return -1;
  DevGuard g_(c->dev);
  if (cudaMemcpyAsync(c->host_ctl, c->v.ctl, sizeof(DevCtl),
                      cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return -1;
  return c->host_ctl->band_runs;
}

int dpso_bound_pairs(dpso_ctx* c, unsigned long long* out) {
  if (!c || !out) return fail(DPSO_EINVAL, "bad arguments");
  *out = 0;
  if (!c->v.plan.bound) return DPSO_OK;
  DevGuard g_(c->dev);
  CK(cudaMemcpyAsync(out, c->v.plan.bound_pairs, 8, cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return DPSO_OK;
}

int dpso_bound_fallbacks(dpso_ctx* c) {
  if (!c || !c->v.plan.bound) return -1;
  DevGuard g_(c->dev);
  int32_t v = 0;
  if (cudaMemcpyAsync(&v, c->v.plan.bound_fb, 4, cudaMemcpyDeviceToHost,
                      c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return -1;
  return v;
}

int dpso_band_line(dpso_ctx* c) {
  if (!c) return -1;
  return c->v.plan.band_mode ? c->v.plan.band_line : 0;
}

int dpso_band_rows(dpso_ctx* c) {
  if (!c) return -1;
  return c->v.plan.band_mode ? 32 * c->v.plan.band_rpl - 1 : 0;
}

int dpso_band_staging(dpso_ctx* c) {
  if (!c) return -1;
  if (!c->v.plan.band_mode) return 0;
  return c->v.plan.band_g4 ? 2 : 1;
}

int dpso_init_path(dpso_ctx* c) { return c ? c->init_path : -1; }

int dpso_scan_rows_bytes(dpso_ctx* c) {
  if (!c) return -1;
  if (c->v.plan.mode == kScanFP64) return 8;
  return c->v.plan.es == 2 && c->v.plan.cost16 ? 2 : 4;
}

int dpso_set_streams(dpso_ctx* c, const uint64_t* host_states) {
  DevGuard g_(c ? c->dev : -1);
  if (!c || !host_states) return fail(DPSO_EINVAL, "null argument");
  const int64_t P = c->prm.n_particles;
  int rc = sync_in(c);
  if (rc) return rc;
  if ((rc = join_walk(c))) return rc;
  CK(cudaMemcpyAsync(c->v.streams, host_states, sizeof(PcgState) * (P + 2),
                     cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->have_streams = true;
  return DPSO_OK;
}

int dpso_init(dpso_ctx* c, const int32_t* seed_body, int32_t n_seed) {
  DevGuard g_(c ? c->dev : -1);
  NvtxRange nv_("dpso_init (swarm init)");
  if (!c) return fail(DPSO_EINVAL, "null context");
  if (!c->have_cost) return fail(DPSO_EINVAL, "cost matrix not set");
  if (!c->have_streams && c->prm.rng_mode == DPSO_RNG_NUMPY)
    return fail(DPSO_EINVAL, "rng streams not set");
  const int n = c->n;
  if (n_seed < 0 || n_seed > c->prm.n_particles)
    return fail(DPSO_EINVAL, "n_seed out of range");
  if (n_seed > 0 && !seed_body)
    return fail(DPSO_EINVAL, "seed_tour is not a tour over the matrix");
  uint16_t* dseed = (uint16_t*)(c->ws + c->L.off_seed);
  if (n_seed > 0) {
    std::vector<uint16_t> s(n);
    std::vector<char> seen(n, 0);
    for (int i = 0; i < n; ++i) {
      int32_t val = seed_body[i];
      if (val < 0 || val >= n || seen[val])
        return fail(DPSO_EINVAL, "seed_tour is not a tour over the matrix");
      seen[val] = 1;
      s[i] = (uint16_t)val;
    }
    int rc = sync_in(c);
    if (rc) return rc;
    CK(cudaMemcpyAsync(dseed, s.data(), 2 * n, cudaMemcpyHostToDevice,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  int rc = sync_in(c);
  if (rc) return rc;
  if ((rc = join_walk(c))) return rc;
  CK(launch_init(c->v, dseed, n_seed, c->stream, &c->init_path));
  CK(launch_init_best(c->v, c->stream));
  // stream walk of the first mutation call
  if (c->v.use_mutation) CK(launch_mutation_walk(c->v, c->stream));
  c->gen_next = 1;  // init leaves the device at generation 0
  c->initialized = true;
  return sync_out(c);
}

// Two graphs: a generation that runs the mutation call and one that does
// not (gen % mutation_period != 0: the mutation kernels would only exit at
// entry).  The host knows which generation each launch runs (gen_next; a
// generation after the stall break is a no-op either way).
static bool walk_early(const dpso_ctx* c);

static int capture_generation(dpso_ctx* c, bool with_mutation, int walk,
                              cudaGraphExec_t* out) {
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  cudaError_t e = enqueue_generation(
      c->v, c->stream, c->stream2, c->ev_fork, c->ev_join, with_mutation,
      walk, with_mutation && walk == kWalkNone && walk_early(c)
                ? c->ev_fix
                : nullptr);
  cudaError_t e2 = cudaStreamEndCapture(c->stream, &g);
  if (e) {
    std::string where = std::string("capture generation (") + g_stage + ")";
    return cuda_fail(e, where.c_str());
  }
  if (e2) return cuda_fail(e2, "cudaStreamEndCapture");
  e = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  if (e) return cuda_fail(e, "cudaGraphInstantiate");
  return DPSO_OK;
}

// The next call's walk starts at the mutating graph's event node right
// after the call's stream update (large swarms: C3 14.5 -> 14.9 M, C4 5.1
// -> 5.4 M particle-iter/s) or after the whole mutating generation (small
// swarms, where the one-SM walk then competes with the 2-opt scan: C2 0.148
// vs 0.150 ms per step).  DPSO_WALK_LATE=0/1 overrides.
static bool walk_early(const dpso_ctx* c) {
  if (const char* e = getenv("DPSO_WALK_LATE")) return atoi(e) == 0;
  return c->prm.n_particles >= 4096;
}

static bool walk_eager(const dpso_ctx* c) {
  return c->v.use_mutation && c->v.rng_mode == DPSO_RNG_NUMPY &&
         c->v.mutation_period > 1 && !getenv("DPSO_ONE_GRAPH") &&
         !getenv("DPSO_WALK_AFTER_MUTATION");
}

static int ensure_graph(dpso_ctx* c) {
  if (c->graph) return DPSO_OK;
  // mutation_period > 1: the walk is launched outside the graphs, right
  // after each mutating generation, on the forked stream, and the next
  // mutating generation waits for it (launch_generation): it hides behind
  // every generation in between
  int rc = capture_generation(c, true,
                              walk_eager(c) ? kWalkNone : kWalkAfterMutation,
                              &c->graph);
  if (rc) return rc;
  if (c->v.use_mutation && c->v.mutation_period > 1 &&
      !getenv("DPSO_ONE_GRAPH")) {
    rc = capture_generation(c, false, kWalkNone, &c->graph_plain);
    if (rc) return rc;
  }
  return DPSO_OK;
}

// w < 1: make room for `gens` more generations of velocity growth (each
// adds at most 2n - 2 entries to a list) before launching them: read the
// longest list, and if it could outgrow the capacity, move every list to a
// larger owned buffer (rows keep their entries; the graphs, which hold the
// old pointer, are re-captured).
static int ensure_velocity(dpso_ctx* c, int gens) {
  if (!c->v.vel) return DPSO_OK;
  CK(cudaMemcpyAsync(c->host_ctl, c->v.ctl, sizeof(DevCtl),
                     cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->host_ctl->vel_overflow)
    return fail(DPSO_ECUDA, "velocity list capacity exceeded");
  const int64_t n = c->n, P = c->prm.n_particles;
  // len' = round(w len) + k1 + k2 <= max(len, L*), L* = (2n - 1.5)/(1 - w):
  // a capacity of max(len, L*) is never outgrown
  const double lstar = (2.0 * n + 1.0) / (1.0 - c->prm.inertia) + 8.0;
  const int64_t need = std::min<int64_t>(
      (int64_t)c->host_ctl->vel_max + 2 * n * (int64_t)gens,
      std::max<int64_t>(c->host_ctl->vel_max, (int64_t)lstar));
  if (need <= c->v.vel_cap) return DPSO_OK;
  const int64_t cap = std::max<int64_t>(2 * c->v.vel_cap, need);
  const int64_t old_stride = c->v.vel_cap + 2 * n, stride = cap + 2 * n;
  uint32_t* nb = nullptr;
  CK(cudaMallocAsync(&nb, 4 * (size_t)P * stride, c->stream));
  CK(cudaMemcpy2DAsync(nb, 4 * stride, c->v.vel, 4 * old_stride,
                       4 * c->v.vel_cap, P, cudaMemcpyDeviceToDevice,
                       c->stream));
  if (c->vel_owned) CK(cudaFreeAsync(c->vel_owned, c->stream));
  c->vel_owned = nb;
  c->v.vel = nb;
  c->v.vel_cap = cap;
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  if (c->graph_plain) {
    cudaGraphExecDestroy(c->graph_plain);
    c->graph_plain = nullptr;
  }
  return DPSO_OK;
}

static cudaError_t launch_generation(dpso_ctx* c) {
  const int64_t g = c->gen_next++;
  const bool mut = !c->graph_plain || (g % c->v.mutation_period == 0);
  const bool eager = mut && walk_eager(c);
  cudaError_t e;
  // this call's walk (launched after the previous mutating generation)
  if (eager && (e = cudaStreamWaitEvent(c->stream, c->ev_join, 0))) return e;
  if ((e = cudaGraphLaunch(mut ? c->graph : c->graph_plain, c->stream)))
    return e;
  if (!eager) return cudaSuccess;
  // the next call's walk, concurrent with the generations until then: it
  // starts at the mutating graph's event node right after the call's
  // stream update (k_mut_fix), overlapping the rest of this generation
  const bool early = walk_early(c);
  if (!early && (e = cudaEventRecord(c->ev_fork, c->stream))) return e;
  if ((e = cudaStreamWaitEvent(c->stream2, early ? c->ev_fix : c->ev_fork,
                               0)))
    return e;
  if ((e = launch_mutation_walk(c->v, c->stream2))) return e;
  return cudaEventRecord(c->ev_join, c->stream2);
}

int dpso_step(dpso_ctx* c, int32_t gens) {
  DevGuard g_(c ? c->dev : -1);
  NvtxRange nv_("dpso_step");
  if (!c || !c->initialized) return fail(DPSO_EINVAL, "context not initialized");
  int rc = sync_in(c);
  if (rc) return rc;
  for (int done = 0; done < gens;) {
    // w < 1: batches of at most 64 generations, each with room for its
    // velocity growth
    const int b = c->v.vel ? std::min(64, gens - done) : gens - done;
    if ((rc = ensure_velocity(c, b))) return rc;
    if ((rc = ensure_graph(c))) return rc;
    for (int g = 0; g < b; ++g) CK(launch_generation(c));
    done += b;
  }
  if (c->v.vel) {
    CK(cudaMemcpyAsync(c->host_ctl, c->v.ctl, sizeof(DevCtl),
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->host_ctl->vel_overflow)
      return fail(DPSO_ECUDA, "velocity list capacity exceeded");
  }
  return sync_out(c);
}

int dpso_step_timed(dpso_ctx* c, int32_t gens, double* phase_ms,
                    int32_t* two_opt_count) {
  DevGuard g_(c ? c->dev : -1);
  NvtxRange nv_("dpso_step_timed");
  // Same launches as one graph replay, issued directly with CUDA events
  // between phases: [0] begin+update [1] mutation [2] select
  // [3] 2-opt scan [4] 2-opt apply [5] finalize.
  if (!c || !c->initialized) return fail(DPSO_EINVAL, "context not initialized");
  int rc = sync_in(c);
  if (rc) return rc;
  if ((rc = ensure_velocity(c, gens))) return rc;
  const SwarmView& v = c->v;
  cudaEvent_t ev[7];
  for (int i = 0; i < 7; ++i) CK(cudaEventCreate(&ev[i]));
  double acc[6] = {0, 0, 0, 0, 0, 0};
  // the walk's place as in dpso_step (launch_generation)
  const bool late = walk_eager(c);
  for (int g = 0; g < gens; ++g) {
    cudaStream_t s = c->stream;
    const bool mut_gen =
        v.use_mutation && (c->gen_next + g) % v.mutation_period == 0;
    if (late && mut_gen) CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    CK(cudaEventRecord(ev[0], s));
    CK(launch_gen_begin(v, s));
    CK(launch_update(v, s));
    CK(cudaEventRecord(ev[1], s));
    if (v.use_mutation) {
      CK(launch_mutation_pre(v, s));
      CK(launch_mutation_post(v, s));
      if (!late) {
        CK(cudaEventRecord(c->ev_fork, s));
        CK(cudaStreamWaitEvent(c->stream2, c->ev_fork, 0));
        CK(launch_mutation_walk(v, c->stream2));
        CK(cudaEventRecord(c->ev_join, c->stream2));
      }
      CK(launch_mutation_swap(v, s));
    }
    CK(cudaEventRecord(ev[2], s));
    CK(launch_select(v, !v.use_edge_exchange, s));
    CK(cudaEventRecord(ev[3], s));
    if (v.use_edge_exchange) CK(launch_two_opt(v, s, 1));
    CK(cudaEventRecord(ev[4], s));
    if (v.use_edge_exchange) CK(launch_two_opt(v, s, 2));
    CK(cudaEventRecord(ev[5], s));
    if (v.use_edge_exchange) CK(launch_finalize(v, s));
    if (v.use_mutation && !late) CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    CK(cudaEventRecord(ev[6], s));
    if (late && mut_gen) {
      CK(cudaEventRecord(c->ev_fork, s));
      CK(cudaStreamWaitEvent(c->stream2, c->ev_fork, 0));
      CK(launch_mutation_walk(v, c->stream2));
      CK(cudaEventRecord(c->ev_join, c->stream2));
    }
    CK(cudaEventSynchronize(ev[6]));
    for (int i = 0; i < 6; ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      acc[i] += ms;
    }
  }
  for (int i = 0; i < 7; ++i) cudaEventDestroy(ev[i]);
  c->gen_next += gens;
  if (phase_ms)
    for (int i = 0; i < 6; ++i) phase_ms[i] = acc[i];
  if (two_opt_count) {
    DevCtl h;
    CK(cudaMemcpy(&h, c->v.ctl, sizeof h, cudaMemcpyDeviceToHost));
    *two_opt_count = h.two_opt_count;
  }
  return sync_out(c);
}

int dpso_ctl(dpso_ctx* c, int32_t* out /* gen, stall, done, gens_run,
                                           two_opt_count, n_events */,
             double* gbest_fit) {
  DevGuard g_(c ? c->dev : -1);
  if (!c) return fail(DPSO_EINVAL, "null context");
  int rc = sync_in(c);
  if (rc) return rc;
  CK(cudaStreamSynchronize(c->stream));
  DevCtl h;
  CK(cudaMemcpy(&h, c->v.ctl, sizeof h, cudaMemcpyDeviceToHost));
  if (out) {
    out[0] = h.gen;
    out[1] = h.stall;
    out[2] = h.done;
    out[3] = h.gens_run;
    out[4] = h.two_opt_count;
    out[5] = h.n_events;
  }
  if (gbest_fit) *gbest_fit = h.gbest_fit;
  return DPSO_OK;
}

int dpso_run(dpso_ctx* c, int32_t* gens_run) {
  DevGuard g_(c ? c->dev : -1);
  NvtxRange nv_("dpso_run");
  if (!c || !c->initialized) return fail(DPSO_EINVAL, "context not initialized");
  int rc = sync_in(c);
  if (rc) return rc;
  int launched = 0;
  const int G = c->prm.max_generations;
  int batch = 4;
  while (launched < G) {
    const int b = std::min(batch, G - launched);
    if ((rc = ensure_velocity(c, b))) return rc;
    if ((rc = ensure_graph(c))) return rc;
    {
      NvtxRange nv_b("generation batch");
      for (int g = 0; g < b; ++g) CK(launch_generation(c));
    }
    launched += b;
    CK(cudaMemcpyAsync(c->host_ctl, c->v.ctl, sizeof(DevCtl),
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->host_ctl->done) break;
    if (batch < 64) batch *= 2;
  }
  CK(cudaMemcpyAsync(c->host_ctl, c->v.ctl, sizeof(DevCtl),
                     cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->host_ctl->vel_overflow)
    return fail(DPSO_ECUDA, "velocity list capacity exceeded (inertia too "
                            "close to 1 for the device list bound)");
  if (gens_run) *gens_run = c->host_ctl->gens_run;
  return sync_out(c);
}

int dpso_result(dpso_ctx* c, int32_t* tour, double* fitness, double* conv,
                int32_t* n_conv) {
  DevGuard g_(c ? c->dev : -1);
  if (!c || !c->initialized) return fail(DPSO_EINVAL, "context not initialized");
  const int n = c->n;
  int rc = sync_in(c);
  if (rc) return rc;
  std::vector<uint16_t> g(n);
  CK(cudaMemcpyAsync(c->host_ctl, c->v.ctl, sizeof(DevCtl),
                     cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(g.data(), c->v.gbest, 2 * n, cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const int gens = c->host_ctl->gens_run;
  if (conv)
    CK(cudaMemcpy(conv, c->v.conv, sizeof(double) * (gens + 1),
                  cudaMemcpyDeviceToHost));
  if (n_conv) *n_conv = gens + 1;
  if (tour) {
    for (int i = 0; i < n; ++i) tour[i] = g[i];
    tour[n] = g[0];
  }
  if (fitness) *fitness = c->host_ctl->gbest_fit;
  return DPSO_OK;
}

int dpso_get_state(dpso_ctx* c, int32_t* x, int32_t* pbest, double* fit,
                   double* pfit, int32_t* vmap, int32_t* gbest,
                   double* gbest_fit) {
  DevGuard g_(c ? c->dev : -1);
  if (!c) return fail(DPSO_EINVAL, "null context");
  const int64_t P = c->prm.n_particles, n = c->n, np = c->v.np;
  int rc = sync_in(c);
  if (rc) return rc;
  CK(cudaStreamSynchronize(c->stream));
  std::vector<uint16_t> buf(P * np);
  auto rows = [&](const uint16_t* src, int32_t* dst) -> int {
    if (!dst) return DPSO_OK;
    if (!src) {
      for (int64_t p = 0; p < P; ++p)
        for (int64_t i = 0; i < n; ++i) dst[p * n + i] = (int32_t)i;
      return DPSO_OK;
    }
    CK(cudaMemcpy(buf.data(), src, 2 * P * np, cudaMemcpyDeviceToHost));
    for (int64_t p = 0; p < P; ++p)
      for (int64_t i = 0; i < n; ++i) dst[p * n + i] = buf[p * np + i];
    return DPSO_OK;
  };
  if ((rc = rows(c->v.x, x))) return rc;
  if ((rc = rows(c->v.pbest, pbest))) return rc;
  if ((rc = rows(c->v.vmap, vmap))) return rc;
  if (fit) CK(cudaMemcpy(fit, c->v.fit, 8 * P, cudaMemcpyDeviceToHost));
  if (pfit) CK(cudaMemcpy(pfit, c->v.pfit, 8 * P, cudaMemcpyDeviceToHost));
  if (gbest) {
    std::vector<uint16_t> g(n);
    CK(cudaMemcpy(g.data(), c->v.gbest, 2 * n, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) gbest[i] = g[i];
  }
  if (gbest_fit) {
    DevCtl h;
    CK(cudaMemcpy(&h, c->v.ctl, sizeof h, cudaMemcpyDeviceToHost));
    *gbest_fit = h.gbest_fit;
  }
  return DPSO_OK;
}

int dpso_set_state(dpso_ctx* c, const int32_t* x, const int32_t* pbest,
                   const double* fit, const double* pfit, const int32_t* vmap,
                   const int32_t* gbest, double gbest_fit) {
  DevGuard g_(c ? c->dev : -1);
  if (!c) return fail(DPSO_EINVAL, "null context");
  const int64_t P = c->prm.n_particles, n = c->n, np = c->v.np;
  int rc = sync_in(c);
  if (rc) return rc;
  if ((rc = join_walk(c))) return rc;
  // every copy is stream-ordered on c->stream (pageable host sources are
  // staged by the driver; the stream sync below keeps them alive)
  std::vector<uint16_t> bx, bp, bv;
  auto put = [&](uint16_t* dst, const int32_t* src,
                 std::vector<uint16_t>& buf) -> int {
    if (!dst || !src) return DPSO_OK;
    buf.assign(P * np, 0);
    for (int64_t p = 0; p < P; ++p)
      for (int64_t i = 0; i < n; ++i) buf[p * np + i] = (uint16_t)src[p * n + i];
    CK(cudaMemcpyAsync(dst, buf.data(), 2 * P * np, cudaMemcpyHostToDevice,
                       c->stream));
    return DPSO_OK;
  };
  if ((rc = put(c->v.x, x, bx))) return rc;
  if ((rc = put(c->v.pbest, pbest, bp))) return rc;
  if ((rc = put(c->v.vmap, vmap, bv))) return rc;
  if (pfit)
    CK(cudaMemcpyAsync(c->v.pfit, pfit, 8 * P, cudaMemcpyHostToDevice,
                       c->stream));
  std::vector<uint16_t> g;
  if (gbest) {
    g.resize(n);
    for (int i = 0; i < n; ++i) g[i] = (uint16_t)gbest[i];
    CK(cudaMemcpyAsync(c->v.gbest, g.data(), 2 * n, cudaMemcpyHostToDevice,
                       c->stream));
    c->host_ctl->gbest_fit = gbest_fit;
    CK(cudaMemcpyAsync(&c->v.ctl->gbest_fit, &c->host_ctl->gbest_fit,
                       sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }
  // refresh the edge-cost cache (and fitness) for the new positions, then
  // let explicit fitness values override the recomputed ones
  CK(launch_tour_cost_rows(c->v.cost, c->v.ld, c->n, c->v.x, np,
                           c->prm.n_particles, c->v.fit, c->v.dcache,
                           c->stream));
  if (fit)
    CK(cudaMemcpyAsync(c->v.fit, fit, 8 * P, cudaMemcpyHostToDevice,
                       c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->initialized = true;
  return sync_out(c);
}

int dpso_mutate_step(dpso_ctx* c) {
  DevGuard g_(c ? c->dev : -1);
  if (!c || !c->initialized) return fail(DPSO_EINVAL, "context not initialized");
  if (!c->prm.use_mutation || c->prm.mutation_period != 1)
    return fail(DPSO_EINVAL,
                "dpso_mutate_step needs use_mutation and mutation_period == 1");
  int rc = sync_in(c);
  if (rc) return rc;
  if ((rc = join_walk(c))) return rc;
  const SwarmView& v = c->v;
  // one generation reduced to its mutation call: gen_begin (marks it
  // mutating, selects the buffers the last walk prepared), the dedupe /
  // sampling pipeline, the next call's stream walk, swap + fitness + pbest
  CK(launch_gen_begin(v, c->stream));
  CK(launch_mutation_pre(v, c->stream));
  CK(launch_mutation_post(v, c->stream));
  CK(launch_mutation_walk(v, c->stream));
  CK(launch_mutation_swap(v, c->stream));
  c->gen_next += 1;
  return sync_out(c);
}

int dpso_offer_gbest(dpso_ctx* c, const int32_t* tour, double fitness) {
  DevGuard g_(c ? c->dev : -1);
  NvtxRange nv_("dpso_offer_gbest");
  if (!c || !tour) return fail(DPSO_EINVAL, "null argument");
  const int n = c->n;
  int rc = sync_in(c);
  if (rc) return rc;
  CK(cudaMemcpyAsync(c->host_ctl, c->v.ctl, sizeof(DevCtl),
                     cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (!(fitness < c->host_ctl->gbest_fit)) return DPSO_OK;
  std::vector<uint16_t> g(n);
  for (int i = 0; i < n; ++i) g[i] = (uint16_t)tour[i];
  // tour and fitness in the same stream, ordered before the next generation
  c->host_ctl->gbest_fit = fitness;
  CK(cudaMemcpyAsync(c->v.gbest, g.data(), 2 * n, cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(&c->v.ctl->gbest_fit, &c->host_ctl->gbest_fit,
                     sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return sync_out(c);
}

int64_t dpso_island_record_bytes(int32_t n) {
  return island_rec_bytes((int)round_up(n, 8));
}

int dpso_island_pack(dpso_ctx* c, void* dev_record, int32_t rank) {
  DevGuard g_(c ? c->dev : -1);
  NvtxRange nv_("dpso_island_pack");
  if (!c || !dev_record) return fail(DPSO_EINVAL, "null argument");
  if (!c->initialized) return fail(DPSO_EINVAL, "context not initialized");
  int rc = sync_in(c);
  if (rc) return rc;
  CK(launch_island_pack(c->v, dev_record, rank, c->stream));
  return sync_out(c);
}

int dpso_island_adopt(dpso_ctx* c, const void* dev_records, int32_t world,
                      int32_t rank) {
  DevGuard g_(c ? c->dev : -1);
  NvtxRange nv_("dpso_island_adopt");
  if (!c || !dev_records || world < 1 || rank < 0 || rank >= world)
    return fail(DPSO_EINVAL, "bad arguments");
  if (!c->initialized) return fail(DPSO_EINVAL, "context not initialized");
  int rc = sync_in(c);
  if (rc) return rc;
  CK(launch_island_adopt(c->v, dev_records, world, rank, c->stream));
  return sync_out(c);
}

void dpso_destroy(dpso_ctx* c) {
  if (!c) return;
  DevGuard g_(c->dev);
  if (c->stream2) cudaStreamSynchronize(c->stream2);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->graph_plain) cudaGraphExecDestroy(c->graph_plain);
  if (c->ev) cudaEventDestroy(c->ev);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_fix) cudaEventDestroy(c->ev_fix);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->vel_owned) cudaFree(c->vel_owned);
  pinned_ctl_put(c->host_ctl);
  delete c;
}

// ---- kernel-level entry points -------------------------------------------

static int to_u16_tours(const int32_t* dev_tours, int32_t n, int32_t count,
                        uint16_t* dst, int64_t np, cudaStream_t s);

int dpso_tour_cost_batch(const double* dev_cost, int64_t ld, int32_t n,
                         const int32_t* dev_tours, int32_t count,
                         double* dev_out, void* cuda_stream) {
  if (!dev_cost || !dev_tours || !dev_out || n < 1 || n > kMaxN || count < 0)
    return fail(DPSO_EINVAL, "bad arguments");
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const int64_t np = round_up(n, 8);
  uint16_t* t16 = nullptr;
  CK(cudaMallocAsync(&t16, 2 * np * (int64_t)std::max(count, 1), s));
  int rc = to_u16_tours(dev_tours, n, count, t16, np, s);
  if (rc) return rc;
  CK(launch_tour_cost_rows(dev_cost, ld, n, t16, np, count, dev_out, nullptr,
                           s));
  CK(cudaFreeAsync(t16, s));
  return DPSO_OK;
}

__global__ void k_i32_to_u16(const int32_t* src, int n, int count,
                             uint16_t* dst, int64_t np) {
  const int64_t t = blockIdx.x;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    dst[t * np + i] = (uint16_t)src[t * n + i];
}
__global__ void k_u16_to_i32(const uint16_t* src, int n, int count,
                             int32_t* dst, int64_t np) {
  const int64_t t = blockIdx.x;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    dst[t * n + i] = (int32_t)src[t * np + i];
}

static int to_u16_tours(const int32_t* dev_tours, int32_t n, int32_t count,
                        uint16_t* dst, int64_t np, cudaStream_t s) {
  if (count > 0) k_i32_to_u16<<<count, 256, 0, s>>>(dev_tours, n, count, dst, np);
  CK(cudaGetLastError());
  return DPSO_OK;
}

int dpso_scan_chunks(int32_t n, int32_t count) {
  if (n < 1 || count < 0) {
    fail(DPSO_EINVAL, "bad arguments");
    return -1;
  }
  return two_opt_pick_chunks(n, std::max(count, 1));
}

int dpso_best_exchange_batch(const double* dev_cost, int64_t ld, int32_t n,
                             int32_t* dev_tours, int32_t count,
                             double* dev_delta, void* cuda_stream) {
  if (!dev_cost || !dev_tours || !dev_delta || n < 1 || n > kMaxN ||
      count < 0)
    return fail(DPSO_EINVAL, "bad arguments");
  if (ld < round_up(n, 2) || (ld & 1) || ((uintptr_t)dev_cost & 15))
    return fail(DPSO_EINVAL, "cost matrix needs an even ld >= n and 16-B "
                             "alignment");
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const int64_t np = round_up(n, 8);
  const int chunks = two_opt_pick_chunks(n, std::max(count, 1));
  std::vector<int32_t> tab(4 * chunks);
  two_opt_chunk_table(n, chunks, tab.data());
  const int64_t cnt = std::max(count, 1);
  size_t bytes = round_up(2 * np * cnt, 256) + round_up(8 * np * cnt, 256) +
                 round_up(sizeof(TwoOptRes) * chunks * cnt + 4 * (2 + chunks * cnt), 256) +
                 round_up(16 * chunks, 256) + round_up(8 * cnt, 256) +
                 // fp32 + fp16 rows, band rows, stats, band column arrays
                 round_up(round_up(6 * (int64_t)n * np, 256) +
                              band_rows_bytes(n), 256) +
                 256 + round_up(band_cols_bytes(n, cnt), 256) +
                 round_up(bound_bytes(n, cnt), 256);
  unsigned char* tmp = nullptr;
  CK(cudaMallocAsync(&tmp, bytes, s));
  size_t o = 0;
  auto take = [&](size_t b) {
    unsigned char* p = tmp + o;
    o += round_up(b, 256);
    return p;
  };
  uint16_t* t16 = (uint16_t*)take(2 * np * cnt);
  double* dc = (double*)take(8 * np * cnt);
  TwoOptRes* res = (TwoOptRes*)take(sizeof(TwoOptRes) * chunks * cnt +
                                    4 * (2 + chunks * cnt));
  int32_t* ctab = (int32_t*)take(16 * chunks);
  double* fsum = (double*)take(8 * cnt);
  float* c32 = (float*)take(round_up(6 * (int64_t)n * np, 256) +
                            band_rows_bytes(n));
  CostStats* st = (CostStats*)take(sizeof(CostStats));
  int32_t* bcols = (int32_t*)take(band_cols_bytes(n, cnt));
  void* bbuf = bound_bytes(n, cnt) ? take(bound_bytes(n, cnt)) : nullptr;
  CK(cudaMemcpyAsync(ctab, tab.data(), 16 * chunks,
                     cudaMemcpyHostToDevice, s));
  int rc = to_u16_tours(dev_tours, n, count, t16, np, s);
  if (rc) return rc;
  CK(launch_tour_cost_rows(dev_cost, ld, n, t16, np, count, fsum, dc, s));
  TwoOptPlan pl;
  unsigned char* band =
      band_rows_bytes(n)
          ? (unsigned char*)c32 + round_up(6 * (int64_t)n * np, 256)
          : nullptr;
  CK(two_opt_prepare(dev_cost, ld, n, np, c32,
                     (uint16_t*)(c32 + (size_t)n * np), band, st, s, &pl,
                     bbuf));
  pl.band_cols = bcols;
  pl.band_cols_cap = cnt;
  CK(launch_two_opt_batch(pl, n, (int32_t)np, t16, dc, count, res, chunks,
                          ctab, dev_delta, s));
  if (count > 0) k_u16_to_i32<<<count, 256, 0, s>>>(t16, n, count, dev_tours, np);
  CK(cudaGetLastError());
  CK(cudaFreeAsync(tmp, s));
  return DPSO_OK;
}

int dpso_nn_tour(const double* dev_cost, int64_t ld, int32_t n, int32_t start,
                 int32_t* host_tour, void* cuda_stream) {
  if (!dev_cost || !host_tour || n < 1 || start < 0 || start >= n)
    return fail(DPSO_EINVAL, "bad arguments");
  cudaStream_t s = (cudaStream_t)cuda_stream;
  int32_t* d = nullptr;
  CK(cudaMallocAsync(&d, 4 * n, s));
  CK(launch_nn(dev_cost, ld, n, start, d, s));
  CK(cudaMemcpyAsync(host_tour, d, 4 * n, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(d, s));
  CK(cudaStreamSynchronize(s));
  return DPSO_OK;
}

int dpso_nn_two_opt(const double* dev_cost, int64_t ld, int32_t n,
                    int32_t* host_tour, double* host_cost, void* cuda_stream) {
  // baselines.py:103-123: NN from 0, total = sum of edges in order, then
  // best-improvement 2-opt until delta == 0.0, total += delta each move.
  if (!dev_cost || !host_tour || !host_cost || n < 1)
    return fail(DPSO_EINVAL, "bad arguments");
  if (n == 1) {
    host_tour[0] = 0;
    host_tour[1] = 0;
    *host_cost = 0.0;
    return DPSO_OK;
  }
  cudaStream_t s = (cudaStream_t)cuda_stream;
  int32_t* d = nullptr;
  double* dd = nullptr;
  CK(cudaMallocAsync(&d, 4 * n, s));
  CK(cudaMallocAsync(&dd, 8, s));
  CK(launch_nn(dev_cost, ld, n, 0, d, s));
  // total = sum(rows[a][b] for a, b in zip(body, body[1:] + body[:1]))
  double total = 0.0;
  CK(launch_pysum_tour(dev_cost, ld, n, d, dd, s));
  CK(cudaMemcpyAsync(&total, dd, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (;;) {
    int rc = dpso_best_exchange_batch(dev_cost, ld, n, d, 1, dd, s);
    if (rc) return rc;
    double delta;
    CK(cudaMemcpyAsync(&delta, dd, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (delta == 0.0) break;
    total += delta;
  }
  CK(cudaMemcpyAsync(host_tour, d, 4 * n, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(d, s));
  CK(cudaFreeAsync(dd, s));
  CK(cudaStreamSynchronize(s));
  host_tour[n] = host_tour[0];
  *host_cost = total;
  return DPSO_OK;
}

}  // extern "C"
