/*
 * dpso.h — C ABI of the B200-native enhanced discrete PSO solve path.
 *
 * This is the drop-in boundary for the reference's DPSO solve call
 * (`DiscreteSwarmSolver.fit`, /root/reference/pkg/src/inspectour/solver.py:262-335,
 * and `solve_matrix`, solver.py:352-356).  The reference is pure Python, so
 * its "FFI" is the estimator API; the Python host layer
 * (paper_1706_04399_b200/solver.py) binds these symbols with ctypes, and
 * INTEGRATION.md shows that binding.  Plain pointers and sizes only.
 *
 * Memory ownership: the caller allocates one device workspace of
 * dpso_workspace_size() bytes (e.g. a torch uint8 tensor) and the device
 * cost matrix; the library never allocates large device memory itself
 * (only a private stream, events and a CUDA graph).  Host arrays are
 * ordinary pageable or pinned buffers.
 *
 * Return codes: 0 ok, 1 invalid argument (Python: ValueError, same messages
 * as solver.py:139-172 where tests match them), 2 CUDA error (RuntimeError),
 * 3 NCCL/island error (RuntimeError).  dpso_last_error() is thread-local.
 */
#ifndef DPSO_H_
#define DPSO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPSO_OK 0
#define DPSO_EINVAL 1
#define DPSO_ECUDA 2
#define DPSO_ECOMM 3

#define DPSO_RNG_NUMPY 0  /* PCG64 streams exactly as numpy: bit-exact runs  */
#define DPSO_RNG_PHILOX 1 /* counter-based Philox4x32-10: fully parallel     */

/* Constructor parameters of DiscreteSwarmSolver (solver.py:118-135). */
typedef struct dpso_params {
  int32_t n_particles;       /* >= 3 */
  double inertia;            /* w in [0, 1] */
  double cognitive;          /* phi1 in [0, 1] */
  double social;             /* phi2 in [0, 1] */
  int32_t max_generations;   /* >= 1 */
  int32_t stall_generations; /* >= 1 */
  int32_t mutation_period;   /* >= 1 */
  double seed_fraction;      /* [0, 1] */
  int32_t use_mutation;
  int32_t use_edge_exchange;
  int32_t parallel; /* accepted for API parity; results are identical */
  int32_t rng_mode; /* DPSO_RNG_NUMPY | DPSO_RNG_PHILOX */
  uint64_t philox_seed;
} dpso_params;

typedef struct dpso_ctx dpso_ctx;

/* --- swarm solve (replaces DiscreteSwarmSolver.fit, solver.py:262-335) --- */

/* Bytes of device workspace needed for n nodes. */
int dpso_workspace_size(const dpso_params* prm, int32_t n, size_t* bytes);

/* Bind a context to a caller-owned workspace and CUDA stream (may be NULL =
 * legacy default stream; the library orders its private stream after it). */
int dpso_create(const dpso_params* prm, int32_t n, void* dev_workspace,
                size_t workspace_bytes, void* cuda_stream, dpso_ctx** out);

/* Device cost matrix, row-major fp64, leading dimension ld >= n (elements).
 * The caller owns it and must keep it alive while the context runs. */
int dpso_set_cost(dpso_ctx* ctx, const double* dev_cost, int64_t ld);

/* RNG streams for DPSO_RNG_NUMPY: (n_particles + 2) records of 6 uint64
 * {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger}, in the order
 * of SeedSequence(random_state).spawn(P + 2) (solver.py:278-282):
 * [0] = init stream, [1] = mutation stream, [2..] = particle streams. */
int dpso_set_streams(dpso_ctx* ctx, const uint64_t* host_states);

/* _init_swarm (solver.py:166-188).  seed_body: NULL or n node ids (the open
 * seed tour, already validated by the caller); n_seed as in solver.py:173. */
int dpso_init(dpso_ctx* ctx, const int32_t* host_seed_body, int32_t n_seed);

/* 2-opt scan mode chosen by dpso_set_cost from the matrix: 0 = fp64
 * rows, 1 = exact fp32 (integer |C| < 2^22), 2 = fp32 filter + exact fp64
 * re-evaluation of candidates (see k_two_opt.cu).  The environment variable
 * DPSO_SCAN_MODE overrides it (testing). */
int dpso_scan_mode(dpso_ctx* ctx);

/* Bytes per matrix entry the fp32 scan streams: 2 = fp16 rows (EXACT32
 * with integer |C| <= 2048; FILTER32 with the window widened to the fp16
 * rounding bound), 4 = fp32 rows, 8 = fp64 (FP64 mode).  DPSO_SCAN16=0
 * forces fp32 rows (testing). */
int dpso_scan_rows_bytes(dpso_ctx* ctx);

/* Which 2-opt scan runs: 0 = the column-per-lane scan of dpso_scan_mode,
 * 1 = the row-per-lane band scan, exact (integer |C| <= 32767), 2 = the
 * band scan with int16 fixed-point rows and exact fp64 re-evaluation of
 * the candidates (k_two_opt_band.cu).  DPSO_SCAN_BAND=0, or any of the
 * column scan's knobs, selects 0 (testing). */
int dpso_scan_band(dpso_ctx* ctx);

/* 1 when the bounded 2-opt scan runs first (a finite matrix with the band
 * scan available): every particle's pairs are pruned by an exact lower
 * bound, the band scan takes only the particles whose bound is weak.
 * Diagnostic; DPSO_BOUND=0 turns it off. */
int dpso_scan_bound(dpso_ctx* ctx);

/* Particles the bounded scan handed to the band scan in the last 2-opt
 * pass (-1: no bounded scan).  Synchronizes the context's stream. */
int dpso_bound_fallbacks(dpso_ctx* ctx);

/* 2-opt passes in which the bounded scan handed the band scan at least one
 * particle, since the context was created.  Synchronizes the context's
 * stream.  Diagnostic. */
int dpso_band_runs(dpso_ctx* ctx);

/* Pairs the bounded scan evaluated in fp64 since the context was created
 * (0 without a bounded scan).  Synchronizes the context's stream.
 * Diagnostic (the bench's gathered-byte count). */
int dpso_bound_pairs(dpso_ctx* ctx, unsigned long long* out);

/* How the band scan stages its rows: 2 = TMA gather4 (four rows per copy,
 * n <= ~960), 1 = one bulk copy per row, 0 = no band scan.  Diagnostic. */
int dpso_band_staging(dpso_ctx* ctx);

/* Bytes per staged row line of the band scan (int16 rows: round_up(2n + 12,
 * 16); int8 rows for n > ~1400: round_up(n + 12, 16)), 0 = no band scan.
 * Diagnostic (the bench's staged-byte count). */
int dpso_band_line(dpso_ctx* ctx);

/* Pair rows per band of the band scan: 31 (one row per lane) or 63 (two
 * rows per lane, n <= ~600), 0 = no band scan.  Diagnostic. */
int dpso_band_rows(dpso_ctx* ctx);

/* How the last dpso_init located each particle's draws in the shared numpy
 * init stream: 1 = parallel walk (every start's walk length, then pointer
 * doubling), 0 = serial scan (too large a span, a walk ran off the span, or
 * DPSO_INIT_SERIAL set), -1 = no numpy-mode init yet.  Diagnostic only:
 * both give the same cursors. */
int dpso_init_path(dpso_ctx* ctx);

/* Run generations until max_generations or the stall break.  Blocks the
 * calling thread; returns the number of generations run. */
int dpso_run(dpso_ctx* ctx, int32_t* gens_run);

/* Run exactly `gens` more generations (or fewer if the stall break fires);
 * no host synchronisation.  Used by the benchmark to time single steps. */
int dpso_step(dpso_ctx* ctx, int32_t gens);

/* Like dpso_step, but launches each phase directly with CUDA events between
 * phases and accumulates their device time (ms) into phase_ms[6]:
 * begin+update, mutation, select, 2-opt scan, 2-opt apply, finalize.
 * *two_opt_count = generations so far in which the 2-opt pass ran. */
int dpso_step_timed(dpso_ctx* ctx, int32_t gens, double* phase_ms,
                    int32_t* two_opt_count);

/* Control record: out[6] = {gen, stall, done, gens_run, two_opt_count,
 * n_mutation_events}; *gbest_fit = current global best fitness. */
int dpso_ctl(dpso_ctx* ctx, int32_t* out, double* gbest_fit);

/* Results: closed best tour (n + 1 ints), best fitness, convergence trace
 * (capacity max_generations + 1; *n_conv = generations_run + 1). */
int dpso_result(dpso_ctx* ctx, int32_t* host_tour, double* host_fitness,
                double* host_convergence, int32_t* n_conv);

/* Copy the full swarm state to host (parity tests): x, pbest as P*n int32;
 * fit, pfit as P doubles; vmap as P*n int32 (identity when inertia < 1). */
int dpso_get_state(dpso_ctx* ctx, int32_t* x, int32_t* pbest, double* fit,
                   double* pfit, int32_t* vmap, int32_t* gbest,
                   double* gbest_fit);
int dpso_set_state(dpso_ctx* ctx, const int32_t* x, const int32_t* pbest,
                   const double* fit, const double* pfit, const int32_t* vmap,
                   const int32_t* gbest, double gbest_fit);

/* Test hook: one mutation call (_mutate, solver.py:222-258) on the current
 * state - dedupe by canonical form, reseed the dropped, mutate the non-kept
 * in slot order from the mutation stream (stream 1 of dpso_set_streams),
 * re-cost, pbest - without the velocity update.  Needs use_mutation and
 * mutation_period == 1.  Pairs with dpso_set_state to replay the
 * reference's golden _mutate swarms on the device. */
int dpso_mutate_step(dpso_ctx* ctx);

/* Island exchange (multi-GPU): overwrite gbest when `fitness` is strictly
 * better; the host layer moves the 16-byte records and tours with NCCL. */
int dpso_offer_gbest(dpso_ctx* ctx, const int32_t* host_tour, double fitness);

/* Island exchange on the device, stream-ordered, no host synchronisation
 * (SURVEY §8(e)).  A record is (gbest fitness f64, rank i64, gbest tour
 * u16[round_up(n, 8)]) = dpso_island_record_bytes(n) bytes.
 * dpso_island_pack writes this island's record into dev_record;
 * after an all_gather of the records of all `world` ranks (NCCL on the
 * same stream), dpso_island_adopt picks the winner - smallest fitness,
 * lowest rank on ties - and adopts its tour iff it is another rank's and
 * strictly better than this island's gbest (as dpso_offer_gbest). */
int64_t dpso_island_record_bytes(int32_t n);
int dpso_island_pack(dpso_ctx* ctx, void* dev_record, int32_t rank);
int dpso_island_adopt(dpso_ctx* ctx, const void* dev_records, int32_t world,
                      int32_t rank);

void dpso_destroy(dpso_ctx* ctx);
const char* dpso_last_error(void);

/* --- kernel-level entry points (the reference's private helpers) ------- */

/* _tour_cost (solver.py:48-54) for `count` open tours of n nodes (device
 * int32, row-major), written to dev_out.  Sequential reference order. */
int dpso_tour_cost_batch(const double* dev_cost, int64_t ld, int32_t n,
                         const int32_t* dev_tours, int32_t count,
                         double* dev_out, void* cuda_stream);

/* Tasks per particle the 2-opt scan cuts a batch of `count` tours of n
 * nodes into (row bands x column ranges).  1 selects the one-warp-per-task
 * launch, more than 1 the persistent-warp launch (k_two_opt.cu); -1 on bad
 * arguments. */
int dpso_scan_chunks(int32_t n, int32_t count);

/* _best_exchange (solver.py:88-106) for `count` tours: best 2-opt move with
 * first-index tie break; tours are rewritten in place when the move is
 * strictly improving (< -1e-12), dev_delta gets the delta or 0.0. */
int dpso_best_exchange_batch(const double* dev_cost, int64_t ld, int32_t n,
                             int32_t* dev_tours, int32_t count,
                             double* dev_delta, void* cuda_stream);

/* Nearest-neighbour construction of baselines.py:110-116 (from `start`,
 * ties to the smallest index); host_tour gets n ids. */
int dpso_nn_tour(const double* dev_cost, int64_t ld, int32_t n, int32_t start,
                 int32_t* host_tour, void* cuda_stream);

/* nearest_neighbor_two_opt (baselines.py:103-123): NN tour then
 * best-improvement 2-opt to a fixed point, all on the device. */
int dpso_nn_two_opt(const double* dev_cost, int64_t ld, int32_t n,
                    int32_t* host_tour, double* host_cost, void* cuda_stream);

/* Cost-matrix build: replaces build_graph's pairwise A* loop (graph.py:41-78,
 * voxel.py:112-172).  dev_occ: nx*ny*nz occupancy (C order, 1 = occupied);
 * host_vox: n viewpoint voxels (x, y, z); dev_cost: n x ld fp64 output
 * (symmetric, zero diagonal, blocked pairs = 1e3 * n * max_finite or 1e6);
 * dev_virtual: optional n*n uint8 mask; *host_vcost: the virtual cost.
 * Costs are the admissible-A* / Dijkstra costs (exact fp path sums). */
int dpso_build_cost(const uint8_t* dev_occ, int32_t nx, int32_t ny,
                    int32_t nz, const double* host_weights,
                    const int32_t* host_vox, int32_t n, double* dev_cost,
                    int64_t ld, uint8_t* dev_virtual, double* host_vcost,
                    void* cuda_stream);

/* The same build in two steps, for a build sharded over GPUs (SURVEY
 * §8(e): shard the SSSP sources, all-gather the row blocks).
 * dpso_build_cost_rows: rows [src_begin, src_end) of the n x n distance
 * table, dev_rows[(i - src_begin) * n + j] = cost of the i -> j motion
 * (+inf when blocked), i.e. graph.py:58-66's pair loop for those sources.
 * Every viewpoint is checked (occupied -> DPSO_EINVAL on every rank).
 * dpso_build_cost_assemble: graph.py:63-78 over the complete table (its
 * upper triangle): symmetric cost, virtual mask and virtual cost exactly as
 * dpso_build_cost writes them. */
int dpso_build_cost_rows(const uint8_t* dev_occ, int32_t nx, int32_t ny,
                         int32_t nz, const double* host_weights,
                         const int32_t* host_vox, int32_t n,
                         int32_t src_begin, int32_t src_end, double* dev_rows,
                         void* cuda_stream);
int dpso_build_cost_assemble(const double* dev_rows, int32_t n,
                             double* dev_cost, int64_t ld,
                             uint8_t* dev_virtual, double* host_vcost,
                             void* cuda_stream);

/* Plain-text cost-matrix files (replaces graph.py:123-130
 * save_cost_matrix and graph.py:133-143 load_cost_matrix, host code).
 * Write: a header line "n", then n lines of n entries, each Python's
 * repr(float(x)), single-space separated: byte-identical to the reference.
 * Read: tokens split on whitespace, parsed like Python int()/float();
 * with host_out == NULL only the header is read (*n_out = n, to size the
 * buffer), else all n*n entries go to host_out (row-major, leading
 * dimension ld >= n, capacity cap_n rows).  Errors (DPSO_EINVAL) carry the
 * reference's messages: "empty cost matrix file <path>", "cost matrix
 * <path>: expected <n*n> entries, got <k>", Python's int()/float()
 * conversion messages. */
/* Host -> device upload of a row-major fp64 matrix (rows x cols, host
 * leading dimension host_ld, device leading dimension dev_ld >= cols; the
 * device padding columns are not written).  Replaces the reference's
 * in-memory hand-off of the matrix to the solver (solver.py:155-162 takes a
 * host array): large matrices go through a ring of two pinned chunks
 * filled by several host threads while the other chunk's DMA runs on
 * cuda_stream; returns after the copy completed. */
int dpso_upload_matrix(const double* host, int64_t host_ld, int32_t rows,
                       int32_t cols, double* dev, int64_t dev_ld,
                       void* cuda_stream);

int dpso_write_matrix_text(const char* path, const double* host, int64_t ld,
                           int32_t n);
int dpso_read_matrix_text(const char* path, double* host_out, int64_t ld,
                          int32_t cap_n, int32_t* n_out);
/* repr(float(x)) of one value into out (cap bytes incl. the NUL): the
 * writer's formatter, exposed for tests. */
int dpso_py_repr(double x, char* out, int32_t cap);

/* Voxel A* paths (replaces voxel.py:112-172 shortest_path for the legs
 * graph.py:58-66 stores, host code, all cores): host_occ = nx*ny*nz uint8
 * (C order, 1 = occupied), weights = axis weights (a1, a2, a3), mode 0 =
 * admissible, 1 = paper heuristic; pairs = k x (start xyz, goal xyz).
 * Path i goes to out_xyz + 3*cap_per*i as lens[i] (x, y, z) waypoints with
 * motion cost costs[i]; a blocked pair gives lens[i] = 0, costs[i] = inf.
 * The same path as the reference (heap order (f, g, voxel), neighbour
 * order, fp64 step costs).  An occupied endpoint fails with the
 * reference's message. */
int dpso_voxel_paths(const uint8_t* host_occ, int32_t nx, int32_t ny,
                     int32_t nz, const double* weights, int32_t mode,
                     const int32_t* pairs, int32_t k, int32_t* out_xyz,
                     int64_t cap_per, int64_t* lens, double* costs);

/* numpy's SeedSequence(entropy).spawn(count) + PCG64(child) (the reference's
 * stream setup, solver.py:278-282), host code: entropy as little-endian
 * uint32 words (numpy's _int_to_uint32_array), out = count x 6 uint64
 * records in dpso_set_streams' layout. */
int dpso_spawn_pcg64_states(const uint32_t* entropy_words, int32_t n_words,
                            int64_t count, uint64_t* out);

/* Philox4x32-10 block (host evaluation of the device RNG's code path, for
 * known-answer tests): out = philox(ctr[4], key = k0 | k1 << 32). */
int dpso_philox4x32_10(const uint32_t* ctr, uint64_t key, uint32_t* out);

/* Build/version string. */
const char* dpso_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DPSO_H_ */
