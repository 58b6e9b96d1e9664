// Internal declarations of the B200 DPSO solve path (not part of the ABI).
//
// HBM layout of one swarm (all in the caller-owned workspace, 256-B aligned
// sections; NP = n rounded up to 8 so every u16 row is 16-B aligned):
//   ctl      DevCtl                      generation/stall/flags (one record)
//   streams  (P+2) x PcgState            numpy streams: init, mutation, particles
//   x        P x NP  u16                 current open tour per particle
//   pbest    P x NP  u16                 personal best tour
//   vmap     P x NP  u16                 composed velocity permutation (w == 1)
//   vel      P x (cap+2n) u32            transposition lists (w < 1 only)
//   fit,pfit P f64                       fitness / personal-best fitness
//   dcache   P x NP  f64                 edge costs d_i = C[x_i][x_{i+1}]
//   gbest    NP u16, conv (G+1) f64      global best tour, convergence trace
//   tores    P x chunks x TwoOptRes      2-opt partial argmins
//   mutation scratch (ranks, hashes, lists, events) and init cursors.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dpso.h"
#include "pcg64.cuh"

namespace dpso {

constexpr int kMaxN = 65535;  // u16 node ids

__host__ __device__ inline int64_t round_up(int64_t v, int64_t m) {
  return (v + m - 1) / m * m;
}

struct DevCtl {
  double gbest_fit;
  int32_t gen;        // generation currently running (1-based), 0 after init
  int32_t stall;
  int32_t done;       // stall break or max_generations reached
  int32_t gens_run;
  int32_t improved;   // cand.fitness < gbest_fit after update(+mutation)
  int32_t cand;
  int32_t mutating;   // this generation mutates
  int32_t two_opt_ran;
  int32_t n_surv;
  int32_t n_drop;
  int32_t n_events;
  int32_t collision;  // canonical-hash collision seen (diagnostic)
  int32_t vel_overflow;
  int32_t vel_max;        // longest velocity list after the last update
  int32_t two_opt_count;  // generations in which the 2-opt pass ran
  int32_t mut_bad;        // first event whose sample needed a redraw
  int32_t mut_round;      // last stream-walk round run this call
  int32_t mut_from;       // first event of that round
  int32_t mut_overflow;   // stream buffer too short (exact fallback)
  int32_t mut_cur;        // parity of the event buffers of the current call
  int32_t mut_pending;    // the next call's stream walk is still to run
  int32_t band_runs;      // 2-opt passes that handed the band scan work
  uint64_t mut_q;     // u32 draws consumed by the current mutation call
};

// 2-opt scan modes (k_two_opt.cu)
constexpr int kScanFP64 = 0;
constexpr int kScanExact32 = 1;
constexpr int kScanFilter32 = 2;

struct CostStats {
  unsigned long long maxabs_bits;  // bits of max |C| (non-negative double)
  int nonintegral;
  int negmax;                      // some entry equals -max|C|
  unsigned long long second_bits;  // bits of max |C| over |C| < max|C|
  int asym;                        // some C[a][b] differs bitwise from C[b][a]
};

struct TwoOptPlan {
  const double* cost;
  int64_t ld;
  const float* cost32;  // fp32 copy (EXACT32 / FILTER32), may be null
  int64_t ld32;
  int mode;
  float thr;  // FILTER32 candidate window (2 eps), in row units
  // 16-bit rows (es == 2): fp16 copy of C * dscale streamed by the fp32 scan
  // instead of cost32 (half the L2 -> shared-memory bytes).  EXACT32 with
  // integer |C| <= 2048 (exact in fp16, dscale 1); FILTER32 with the window
  // widened to the fp16 rounding bound (dscale = 2^k, max |C| dscale <= 2^15)
  const uint16_t* cost16;
  int es;        // 4 (cost32 rows) or 2 (cost16 rows)
  float dscale;  // power of two applied to d values (rows are pre-scaled)
  // Capped virtual level: every entry equal to vfrom (max|C|, far above all
  // other entries - the reference's blocked pairs, graph.py:63-78) reads as
  // vto (5 x the next largest |C|) in the fp32/fp16 rows and d values.
  // Deltas are F + g V with g = (#virtual added - #virtual removed) and
  // |F| spread <= 4 max_finite, so both V and V' order the pairs alike;
  // the apply re-evaluates the chosen pair in fp64.  vfrom == 0: none.
  double vfrom, vto;
  // Row-per-lane band scan (k_two_opt_band.cu): 4 rotated int16 versions
  // of round(C * band_scale); band_mode 1 EXACT, 2 FILTER (window
  // band_win), 0 not used.  band_vfrom/vto: the virtual cap of those rows.
  const unsigned char* band;
  int band_line;
  int band_es;             // row element bytes: 2 (int16) or 1 (int8)
  int band_rpl;            // pair rows per lane: 1 (32-slot) or 2 (64)
  int band_mode;
  double band_scale;
  int band_win;
  double band_vfrom, band_vto;
  int32_t* band_cols;      // scratch: band_cols_cap x 2 x band_cw(n) ints
  int64_t band_cols_cap;
  // TMA gather4 row staging (n <= ~960): the CUtensorMap of the row
  // versions (a 2-D tensor of 4n lines), 0 = one bulk copy per row
  int band_g4;
  unsigned char band_tm[128];
  // Bounded scan (k_two_opt_bound.cu): per-city off-diagonal row / column
  // minima, the fallback particle list ([0] count, [1..] particles) and the
  // rounding slack of the pair bound.  bound == 0: not used.
  int bound;
  const float2* bound_cmn;
  int32_t* bound_fb;
  unsigned long long* bound_pairs;  // pairs evaluated (cumulative)
  double bound_slack;
  // the matrix equals its transpose bit for bit: a reversed tour segment
  // keeps its edge costs (the 2-opt apply moves them instead of gathering)
  int symmetric;
};

struct TwoOptRes {
  double delta;
  int32_t i, j;
};

// Everything a kernel needs, passed by value.
struct SwarmView {
  int32_t n, np, P;
  int32_t max_generations, stall_generations, mutation_period;
  int32_t use_mutation, use_edge_exchange;
  int32_t rng_mode;
  uint64_t philox_seed;
  double inertia, cognitive, social;
  const double* cost;
  int64_t ld;
  DevCtl* ctl;
  PcgState* streams;   // [0] init, [1] mutation, [2+p] particle p
  PcgState* mut_start; // [2] mutation stream at call start, per parity
  PcgState* init_start; // init stream at init start
  uint16_t* x;
  uint16_t* pbest;
  uint16_t* vmap;
  uint16_t* vinv;      // w < 1: inverse of vmap (the list's value map)
  uint32_t* vel;
  int32_t* vel_len;
  int64_t vel_cap;     // entries per particle list (excl. 2n scratch)
  double* fit;
  double* pfit;
  double* dcache;
  uint16_t* gbest;
  double* conv;
  TwoOptPlan plan;     // cost matrix views + 2-opt scan mode
  TwoOptRes* tores;
  int32_t chunks;      // 2-opt tasks per particle
  int32_t* chunk_tab;  // chunks x (r0, r1, jlo, jhi): pairs i < j with
                       // r0 <= i < r1, jlo <= j < jhi
  // mutation scratch
  int32_t* rank;
  uint64_t* hash;
  int32_t* flag;       // 1 = dropped duplicate
  int32_t* pbflag;     // P: the last fitness pass improved pbest
  int32_t* sidx;       // survivor / dropped index in rank order
  int32_t* order;      // slot at each rank
  int32_t* surv_list;
  int32_t* keep;
  int32_t* ev_slot;
  // per mutation call, double-buffered by call parity ([2][P]): the walk
  // for the next call runs while the current generation finishes
  int32_t* ev_k;
  uint64_t* ev_cursor;
  uint64_t* ev_end;     // stream position after each event's draws
  uint16_t* ev_idx;    // P x np sampled positions per mutation event
  uint32_t* mstream;   // [2] generated mutation-stream span (u32), then
                       // [2] per-word event skips (u16, k_mut_gen)
  int64_t mstream_cap; // u32 capacity of one mstream buffer
  uint64_t* init_cursor;
  uint32_t* init_buf;  // generated init-stream window (u32)
  int64_t init_buf_cap;
  void* init_state;    // InitScanState
  // parallel init walk (init_parallel): the buffer holds the whole expected
  // span; init_aux = 3 x init_buf_cap i32 (walk lengths + two doubling
  // levels), init_anchor = P + 2 i64
  int32_t init_parallel;
  int32_t* init_aux;
  int64_t* init_anchor;
};

// sets dpso_last_error() (thread-local) and returns code
int api_fail(int code, const char* msg);

// ---- kernel launchers (each .cu owns its kernels) -------------------------
cudaError_t launch_gen_begin(const SwarmView& v, cudaStream_t s);
cudaError_t launch_update(const SwarmView& v, cudaStream_t s);
cudaError_t launch_mutation(const SwarmView& v, cudaStream_t s);
// The parts of one mutation call: launch_mutation_pre (dedupe, lists) and
// launch_mutation_post (event sampling, stream update) then
// launch_mutation_swap.  launch_mutation_walk prepares the NEXT call (it
// depends only on the mutation stream after launch_mutation_post, or after
// init) and may run on a forked stream concurrently with everything else.
cudaError_t launch_mutation_walk(const SwarmView& v, cudaStream_t s);
cudaError_t launch_fitness(const SwarmView& v, int use_list, cudaStream_t s);
cudaError_t launch_mutation_swap(const SwarmView& v, cudaStream_t s);
int64_t mstream_words(int n, int P);
int64_t init_buf_words(int n, int P);
bool init_parallel_ok(int n, int P);
cudaError_t launch_mutation_pre(const SwarmView& v, cudaStream_t s);
cudaError_t launch_mutation_post(const SwarmView& v, cudaStream_t s);
cudaError_t launch_select(const SwarmView& v, bool finalize, cudaStream_t s);
cudaError_t launch_two_opt(const SwarmView& v, cudaStream_t s, int parts = 3);
cudaError_t launch_finalize(const SwarmView& v, cudaStream_t s);
cudaError_t launch_init(const SwarmView& v, const uint16_t* dev_seed,
                        int32_t n_seed, cudaStream_t s, int* path);
cudaError_t launch_init_best(const SwarmView& v, cudaStream_t s);
int64_t island_rec_bytes(int np);
cudaError_t launch_island_pack(const SwarmView& v, void* rec, int rank,
                               cudaStream_t s);
cudaError_t launch_island_adopt(const SwarmView& v, const void* recs,
                                int world, int rank, cudaStream_t s);

// generic batch kernels (kernel-level ABI and internal reuse)
cudaError_t launch_tour_cost_rows(const double* cost, int64_t ld, int32_t n,
                                  const uint16_t* tours, int64_t stride,
                                  int32_t count, double* out, double* dcache,
                                  cudaStream_t s);
cudaError_t launch_two_opt_batch(const TwoOptPlan& pl, int32_t n, int32_t np,
                                 uint16_t* tours, const double* dcache,
                                 int32_t count, TwoOptRes* res, int32_t chunks,
                                 const int32_t* chunk_tab, double* delta_out,
                                 cudaStream_t s);
cudaError_t launch_cost_prep(const double* cost, int64_t ld, int32_t n,
                             float* cost32, int64_t ld32, CostStats* st,
                             cudaStream_t s);
int two_opt_mode(const CostStats& st, int n, float* thr);
// cost_prep + mode choice + optional fp16 rows; c16 may be null (no 16-bit
// rows).  Synchronizes the stream once (reads the matrix statistics).
// band: the band scan's row versions (band_rows_bytes(n)), may be null.
cudaError_t two_opt_prepare(const double* cost, int64_t ld, int32_t n,
                            int64_t np, float* c32, uint16_t* c16,
                            unsigned char* band, CostStats* st,
                            cudaStream_t s, TwoOptPlan* pl,
                            void* bound_buf = nullptr);
cudaError_t launch_nn(const double* cost, int64_t ld, int32_t n, int32_t start,
                      int32_t* out, cudaStream_t s);
cudaError_t launch_pysum_tour(const double* cost, int64_t ld, int32_t n,
                              const int32_t* body, double* out,
                              cudaStream_t s);
// Opt a kernel in to `bytes` of dynamic shared memory (cached per kernel;
// static shared memory counts against the same limit, so always opt in).
cudaError_t set_dyn_smem(const void* kernel, size_t bytes);
cudaError_t build_cost_sssp(const uint8_t* dev_occ, int nx, int ny, int nz,
                            const double* w, const int64_t* host_vox, int n,
                            double* dev_cost, int64_t ld, uint8_t* dev_virtual,
                            double* host_vcost, int* bad_viewpoint,
                            cudaStream_t s);
cudaError_t sssp_rows(const uint8_t* dev_occ, int nx, int ny, int nz,
                      const double* w, const int64_t* host_vox, int n,
                      int src_begin, int src_end, double* rows,
                      int* bad_viewpoint, cudaStream_t s);
cudaError_t cost_assemble(const double* rows, int n, double* dev_cost,
                          int64_t ld, uint8_t* dev_virtual,
                          double* host_vcost, cudaStream_t s);
int two_opt_chunk_table(int32_t n, int32_t chunks, int32_t* tab);
// band scan (k_two_opt_band.cu): two stages of 32 rows must fit shared
// memory (n <= ~1330)
constexpr int kBandMaxN = 2900;
int band_line(int n);
int band_cw(int n);
int64_t band_rows_bytes(int n);  // 0 when the band scan cannot run
int64_t band_cols_bytes(int n, int64_t count);
cudaError_t band_prepare(const double* cost, int64_t ld, int32_t n,
                         unsigned char* buf, double mx, bool integral,
                         double vfrom, double vto, cudaStream_t s,
                         TwoOptPlan* pl);
cudaError_t launch_two_opt_band(const TwoOptPlan& pl, int32_t n, int32_t np,
                                const uint16_t* tours, const double* dcache,
                                int32_t count, TwoOptRes* res, int32_t chunks,
                                int32_t* ovf, const DevCtl* ctl,
                                cudaStream_t s, int reserve_sms = 0,
                                const int32_t* plist = nullptr,
                                const int32_t* pcnt = nullptr,
                                int32_t* runs = nullptr,
                                bool cols_ready = false);
// bounded scan (k_two_opt_bound.cu): workspace bytes for count particles
// (0: not available at this n), preparation (needs the band plan), launch
constexpr int kBoundMaxN = kBandMaxN;
int64_t bound_bytes(int n, int64_t count);
cudaError_t bound_prepare(const double* cost, int64_t ld, int32_t n,
                          void* buf, double maxabs, cudaStream_t s,
                          TwoOptPlan* pl);
// the move applied by the bounded scan itself (nullable pointers as in
// k_two_opt_apply)
struct BoundApply {
  uint16_t* tours;
  double* dcache;
  double* fit;
  double* pfit;
  uint16_t* pbest;
  double* delta_out;
};
cudaError_t launch_two_opt_bound(const TwoOptPlan& pl, int32_t n, int32_t np,
                                 const uint16_t* tours, const double* dcache,
                                 int32_t count, TwoOptRes* res, int32_t chunks,
                                 const DevCtl* ctl, cudaStream_t s,
                                 int32_t* runs = nullptr,
                                 const BoundApply* ap = nullptr);
int two_opt_pick_chunks(int32_t n, int32_t P);

// A random fp64 gather from the cost matrix (edge costs C[a][b]).  sm_100
// fills 4 sectors (128 B) of L2 per random 8-B load by default; the
// L2::64B prefetch-size hint halves that (measured: 117 -> 61 DRAM bytes
// per load over a 1 GB table, tools/data/gran_probe), which matters when
// the matrix is far beyond L2 (N = 10000: 800 MB).
__device__ __forceinline__ double ld_cost(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::64B.f64 %0, [%1];"
               : "=d"(v)
               : "l"(p));
  return v;
}

// Fitness in the reference's order (solver.py:48-54):
// total = 0; total += d[n-1]; total += d[0]; ... total += d[n-2].
__device__ __forceinline__ double seq_tour_sum(const double* d, int n) {
  double total = 0.0;
  total = __dadd_rn(total, d[n - 1]);
  for (int i = 0; i < n - 1; ++i) total = __dadd_rn(total, d[i]);
  return total;
}

// _prefix_len (solver.py:82-85) without FMA contraction.
__device__ __forceinline__ int prefix_len(double c, int length) {
  if (!(c > 0.0)) return 0;
  double v = __dadd_rn(__dmul_rn(c, (double)length), 0.5);
  int k = (int)v;  // truncation == Python int() for v >= 0
  return k < length ? k : length;
}

}  // namespace dpso
