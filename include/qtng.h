/* qtng.h -- C ABI of the B200 bucket-elimination contraction engine.
 *
 * This is the drop-in boundary for the reference's contraction hot path
 * (/root/reference/proj, "qtnsim").  Plain pointers and sizes only; no C++
 * or torch types.  Each entry point names the reference interface it
 * replaces.  A C++ adaptor implementing qtnsim::ContractionBackend on top of
 * qtng_contract_bucket ships as include/qtng_backend.hpp; INTEGRATION.md
 * shows how a maintainer wires it into the reference's CLI/backend registry.
 *
 * Conventions (identical to the reference):
 *   - complex numbers are complex128, interleaved (re, im) doubles
 *     (proj/include/qtnsim/tensor.hpp:11,19);
 *   - a tensor over binary variables is row-major in its var order, first
 *     axis = most significant bit (tensor.hpp:13-15);
 *   - bucket results have their axes in ascending variable id
 *     (proj/include/qtnsim/engine.hpp:28-29); an empty result is a 1-element
 *     scalar;
 *   - graphs are edge lists of (u, v) int pairs; angles are p gammas and p
 *     betas (proj/include/qtnsim/circuit.hpp:14-20).
 *
 * Every function returns a qtng_status; on failure qtng_last_error() holds
 * the message, worded exactly like the reference's exception for the same
 * condition.  Status codes map 1:1 onto the reference's exception types
 * (proj/include/qtnsim/errors.hpp:8-36).
 *
 * Threading: a context serialises its device work internally, so one
 * context may be shared by the reference's `jobs` worker threads
 * (proj/src/engine.cpp:531-541).  Contexts on different devices are
 * independent.
 */
#ifndef QTNG_H
#define QTNG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum qtng_status {
  QTNG_OK = 0,
  QTNG_ERR_INVALID_INPUT = 1, /* qtnsim::InvalidInputError */
  QTNG_ERR_RESOURCE = 2,      /* qtnsim::ResourceError     */
  QTNG_ERR_SCHEDULE = 3,      /* qtnsim::ScheduleError     */
  QTNG_ERR_NUMERICAL = 4,     /* qtnsim::NumericalError    */
  QTNG_ERR_CUDA = 5,          /* device failure (no reference counterpart) */
  QTNG_ERR_GENERATION = 6     /* qtnsim::GenerationError   */
} qtng_status;

typedef struct qtng_ctx qtng_ctx;
typedef struct qtng_plan qtng_plan;

/* One record per non-empty bucket, as TimingRecord (proj/include/qtnsim/engine.hpp:71-80).
 * elapsed_s is the bucket's share (by algorithmic bytes) of its level's
 * device time; backend is always "b200". */
typedef struct qtng_record {
  int32_t edge_u, edge_v;
  int32_t bucket_seq;
  int32_t width;
  double elapsed_s;
  uint64_t ops;     /* 2^width */
  double flops_est; /* 8 * ops / elapsed_s */
} qtng_record;

typedef struct qtng_plan_info {
  int32_t n_lightcones;
  int32_t n_levels;          /* dependency levels = level_kernel launches */
  uint64_t n_buckets;        /* non-empty buckets (= records) */
  uint64_t n_device_ops;     /* bucket ops incl. pre-folds of >8-member buckets */
  int32_t max_width;
  int32_t max_result_rank;   /* peak_tensor_bytes = 16 << max_result_rank */
  double alg_bytes;          /* sum over ops of 16*(sum_in 2^rank + 2^r) */
  double sum_ops;            /* sum over buckets of 2^width */
  uint64_t arena_bytes;      /* peak HBM arena footprint */
  uint64_t desc_bytes;       /* descriptor bytes uploaded per plan */
  int32_t kernels_per_run;   /* kernel launches per execution */
  uint64_t n_segments;       /* fused-chain segments (seg_kernel units) */
  uint64_t n_fused_ops;      /* bucket ops evaluated inside segments */
  double dev_bytes;          /* HBM bytes the fused program must move: per
                                unit, its materialised inputs + its output */
  double fp64_ops;           /* FP64 multiplies + adds of the reference's
                                NaiveBackend loop over all buckets */
  double seg_fp64_ops;       /* ... of the buckets evaluated by seg_kernel */
  double single_alg_bytes;   /* B_alg of the buckets run by level/outer kernels */
} qtng_plan_info;

/* The report of a one-shot energy: ContractionReport's aggregate fields as
 * energy_expectation fills them (proj/include/qtnsim/engine.hpp:82-88,136-139;
 * engine.cpp:548-556).  `records`/`rec_cap` are inputs (records may be NULL);
 * one TimingRecord per contracted bucket, selection order, edge_u/edge_v set.
 * elapsed_s is the bucket's share (by algorithmic bytes) of its program's
 * measured device time: the level-batched kernels run hundreds of buckets at
 * once, so a per-bucket device time does not exist. */
typedef struct qtng_energy_report {
  qtng_record* records;       /* in: caller buffer (may be NULL) */
  int64_t rec_cap;            /* in: its capacity in records */
  int64_t n_records;          /* out: records of the contracted buckets */
  uint64_t peak_tensor_bytes; /* out: max over lightcones of 16 * 2^(largest result rank) */
  int32_t merges_applied;     /* out: summed over lightcones (merge_buckets) */
  int32_t merges_skipped;
  float device_ms;            /* out: device time of the program(s) */
} qtng_energy_report;

/* ---------------------------------------------------------------- context */

/* Create a context on CUDA `device`.  arena_bytes = initial HBM reservation
 * (0 = grow on demand). */
qtng_status qtng_create(int device, uint64_t arena_bytes, qtng_ctx** out);
void qtng_destroy(qtng_ctx* ctx);
/* Default arithmetic of the QAOA plans and energies created on ctx with
 * precision 0 (calls that pass 128 or 64 choose it themselves):
 * 128 (default) = complex128, bit-identical to the reference's naive backend;
 * 64 = complex64 arena and kernels (the north_star's optional mode, results
 * within 1e-5; complex128 per-lightcone products).  Explicit schedules and
 * single buckets always run in complex128. */
qtng_status qtng_set_precision(qtng_ctx* ctx, int bits);
/* Message of the calling thread's last failure ("" after success). */
const char* qtng_last_error(void);
/* Library build string (arch, version). */
const char* qtng_version(void);

/* Kernel launches the library has issued since it was loaded (eager launches
 * when enqueued; graph replays as kernels per graph x replays). */
uint64_t qtng_kernel_launches(void);

/* ---------------------------------------------------------------- host side */

/* random_regular (proj/src/graph.cpp:45-76): edges written to edges[2*m];
 * *m_out = edge count.  cap = capacity in edges. */
qtng_status qtng_random_regular(int n, int d, uint64_t seed, int* edges, int cap, int* m_out);

/* edge_schedule (proj/src/engine.cpp:493-501) for edge `edge_index` of the
 * sorted edge list, flattened as: per bucket n_sum, sum_vars, n_tensors,
 * per tensor rank, vars; data = every tensor's entries (re, im) in the same
 * order (the format of oracle/qtn_oracle.h).  *n_ints / *n_data receive the
 * required sizes; nothing is written when a capacity is too small.  merges
 * (may be NULL): the schedule's merges_applied, merges_skipped (ordering.hpp,
 * counted like merge_buckets, engine.cpp:306-358; 0, 0 unmerged). */
qtng_status qtng_edge_schedule(int n, int m, const int* edges, int p, const double* gammas,
                               const double* betas, int edge_index, int merged, int* ints,
                               int64_t int_cap, double* data, int64_t data_cap,
                               int64_t* n_ints, int64_t* n_data, int* n_buckets, int* merges);

/* merge_buckets (proj/src/engine.cpp:306-358) of an explicit schedule (format
 * of qtng_edge_schedule; tensor data is not needed).  Output per merged
 * bucket: n_sum, sum vars, n_tensors, then each member's index among the
 * input schedule's tensors (flattened order), so the caller moves its own
 * tensors.  *n_out / *out_buckets: sizes (nothing written when cap is
 * short); merges (may be NULL): merges_applied, merges_skipped.  Host only. */
qtng_status qtng_merge_schedule(int n_buckets, const int* ints, int64_t n_ints, int* out,
                                int64_t cap, int64_t* n_out, int* out_buckets, int* merges);

/* simulate_widths (proj/src/engine.cpp:235-240) of one edge's schedule. */
qtng_status qtng_simulate_widths(int n, int m, const int* edges, int p, int edge_index,
                                 int merged, int* widths, int cap, int* n_out);

/* Predicted algorithmic bytes (SURVEY.md §8(a) B_alg) of every edge's
 * lightcone: the load-balancing key for multi-GPU sharding. */
qtng_status qtng_edge_costs(int n, int m, const int* edges, int p, int merged,
                            double* bytes_out);

/* Predicted device work per edge lightcone (the sharding key of the
 * multi-GPU driver): per bucket 2^width * max(1, members-1) complex products
 * plus the summation adds -- the fused program is bound by arithmetic and
 * issue, not by bytes.  m doubles. */
qtng_status qtng_edge_work(int n, int m, const int* edges, int p, int merged, double* work_out);

/* Host-only pre-flight of energy_expectation: builds every edge's schedule and
 * runs the data-free contract_network walk (liveness / result-width cap /
 * routing checks, engine.cpp:160-169,246-304) and reports the first refusal
 * in edge order exactly as qtng_energy (and the reference) would raise it:
 * QTNG_ERR_SCHEDULE with "edge (u, v): <reason>".  No device is touched. */
qtng_status qtng_validate_energy(int n, int m, const int* edges, int p, int merged,
                                 int max_result_width);

/* Host-only dump of the device program for the selected edges (sel = NULL:
 * all), for analysis and tests.  Per device op (level-sorted), 8 ints:
 *   level, r (result rank), ns (summed bits), nt (inputs), cb (log2 outputs
 *   per work item), recorded (0 for a pre-fold helper), width, outer (1 when
 *   the op runs in the outer-join kernel)
 * then per input 34 ints: rank, initial (1 = gate/input-region tensor),
 *   src[32] (kMaxRank axis sources; <64 output bit, >=64 summed bit 64+j).
 * *n_ints receives the size needed; nothing is written if cap is short. */
qtng_status qtng_plan_dump(int n, int m, const int* edges, int p, int merged,
                           int max_result_width, int n_sel, const int* sel, int* ints,
                           int64_t cap, int64_t* n_ints, int* n_ops);

/* ---------------------------------------------------------------- device side */

/* ContractionBackend::contract (proj/include/qtnsim/engine.hpp:30;
 * NaiveBackend::contract proj/src/engine.cpp:68-108): sum `sum_vars` out of
 * the tensors.  ranks[t]; vars = concatenated var lists; data = concatenated
 * tensors.  Host buffers in and out.  Result axes ascending. */
qtng_status qtng_contract_bucket(qtng_ctx* ctx, int n_tensors, const int* ranks,
                                 const int* vars, const double* data, int n_sum,
                                 const int* sum_vars, int* out_rank, int* out_vars,
                                 double* out_data, int64_t out_cap);

/* contract_network (proj/src/engine.cpp:246-304) of one flattened schedule
 * (format of qtng_edge_schedule), with contract_bucket's result-width cap
 * (engine.cpp:160-169).  Records: up to rec_cap written, *n_records = count. */
qtng_status qtng_contract_schedule(qtng_ctx* ctx, int n_buckets, const int* ints, int64_t n_ints,
                                   const double* data, int max_result_width,
                                   double* scalar_re_im, qtng_record* records, int rec_cap,
                                   int* n_records, uint64_t* peak_tensor_bytes);

/* energy_expectation (proj/src/engine.cpp:503-563): <C> = m/2 - 1/2 sum Re e_jk,
 * all lightcones of the selected edges on this device in one level-batched
 * program.  precision: 0 (context default), 128 or 64.  sel = NULL selects
 * every edge; terms (may be NULL) receives 2*n_sel doubles (e_jk re, im) in
 * selection order.  *energy is NaN unless the selection is every edge in
 * edge order (a partial selection has terms, not an energy).  report (may be
 * NULL): peak bytes, merge counts, records. */
qtng_status qtng_energy(qtng_ctx* ctx, int n, int m, const int* edges, int p,
                        const double* gammas, const double* betas, int merged,
                        int max_result_width, int precision, int n_sel, const int* sel,
                        double* energy, double* terms, qtng_energy_report* report);

/* energy_expectation over several GPUs of one node: the edge pool of
 * engine.cpp:531-541 becomes the devices.  The lightcones are placed by LPT
 * on the predicted work (qtng_edge_work; qtng_shard_edges shows the
 * placement), one host thread per context plans and contracts its shard
 * (pipelined like qtng_energy), the final kernel writes each term into a
 * 2m-double device vector (zero elsewhere), and ONE ncclReduce (sum, fp64)
 * brings the vectors to ctxs[0]'s device.  The energy is summed there in edge
 * order (engine.cpp:549-551), so it is bit-identical to the 1-GPU energy.
 * Contexts must be on distinct devices.  terms (may be NULL): 2m doubles,
 * edge order.  shard_ms (may be NULL): n_ctx device times. */
qtng_status qtng_energy_multi(qtng_ctx* const* ctxs, int n_ctx, int n, int m, const int* edges,
                              int p, const double* gammas, const double* betas, int merged,
                              int max_result_width, int precision, double* energy, double* terms,
                              float* shard_ms);
/* Host-only: the shard (0..n_shards-1) qtng_energy_multi places each edge's
 * lightcone on.  owner: m ints. */
qtng_status qtng_shard_edges(int n, int m, const int* edges, int p, int merged, int n_shards,
                             int* owner);

/* ---------------------------------------------------------------- plans */

/* Angle-independent plan of the selected edges' lightcones, uploaded to the
 * device once; executions then take only the 2p angles.  precision: 0
 * (context default), 128 or 64. */
qtng_status qtng_plan_create(qtng_ctx* ctx, int n, int m, const int* edges, int p, int merged,
                             int max_result_width, int precision, int n_sel, const int* sel,
                             qtng_plan** out);
/* Device-resident plan of ONE explicit schedule (format of qtng_edge_schedule),
 * e.g. a single wide bucket for the C3 microbenchmark.  Its initial tensor
 * data is uploaded once; qtng_plan_execute then ignores the angles and
 * returns the schedule's scalar as terms[0..1].  A schedule of exactly one
 * bucket is planned as one ContractionBackend::contract (result kept in
 * place, not routed). */
qtng_status qtng_plan_create_schedule(qtng_ctx* ctx, int n_buckets, const int* ints,
                                      int64_t n_ints, const double* data, int max_result_width,
                                      qtng_plan** out);
/* Run the plan for one angle set: ONE CUDA-graph launch holding the
 * gate-table upload (memcpy node from the plan's pinned staging), every
 * level's kernels and the terms download.  terms (host, may be NULL)
 * receives 2*n_sel doubles.  device_ms (may be NULL) = device time of the
 * graph (CUDA events on the plan's stream). */
qtng_status qtng_plan_execute(qtng_plan* plan, const double* gammas, const double* betas,
                              double* terms, float* device_ms);
/* qtng_plan_execute enqueued eagerly with CUDA events around every level and
 * every kernel (the measurement behind qtng_plan_level_ms / _kernel_ms and
 * the per-level record times); same results. */
qtng_status qtng_plan_profile(qtng_plan* plan, const double* gammas, const double* betas,
                              double* terms, float* device_ms);
/* Device-only re-execution with the current angles (no host copies), for
 * throughput measurement: the plan captured once as a CUDA graph, n_runs
 * back-to-back replays, total device time. */
qtng_status qtng_plan_run_device(qtng_plan* plan, int n_runs, float* device_ms);
/* FP64 pipe rates of `device` at its current clocks (peak.cu): DMUL+DADD
 * operations per second (the instruction mix of the bucket kernels, which
 * round every product and never fuse) and DFMA flops per second (2 per FMA).
 * The roofline denominator of seg_kernel; MEASURED_PEAKS.json has no FP64 figure. */
qtng_status qtng_fp64_peak(int device, double* mul_add_ops_per_s, double* fma_flops_per_s);
/* The terms (2*n_sel doubles) the plan's last run left on the device --
 * qtng_plan_execute or a qtng_plan_run_device graph replay. */
qtng_status qtng_plan_terms(qtng_plan* plan, double* terms);
qtng_status qtng_plan_info_get(const qtng_plan* plan, qtng_plan_info* info);
/* State-vector oracle on the device: run_ansatz + expectation_cost
 * (proj/src/statevector.cpp:55-90) for n <= cap qubits (the reference's
 * default cap is 24; the device holds up to 33: 2^33 complex128 = 128 GiB).
 * The amplitudes are bit-identical to run_ansatz's; the sums over basis
 * states are reassociated.  zz (optional, m entries): <Z_u Z_v> per edge in
 * edge order.  Refusals: ResourceError "state vector of N qubits exceeds cap C". */
qtng_status qtng_statevector_energy(qtng_ctx* ctx, int n, int m, const int* edges, int p,
                                    const double* gammas, const double* betas, int cap,
                                    double* energy, double* zz);

/* Host-only analysis of the fused-chain segments of the plan for all m
 * edges.  Per segment (level-sorted): level, L (stages), rY, cY, nops, rb
 * (paired rows: the tile bit of the second row, 255 = unpaired), rb2 (quad
 * tiles: B's row bit, rb = A's; 255 = not quad); then
 * per stage: nt, ns, main (-1 for stage 1), and per member: rank,
 * initial (1 = gate / input-region tensor; a main placeholder has rank 0),
 * then its rank axis codes (device_plan.hpp: lane / digit / tile / summed bit).
 * *n_ints receives the size needed; nothing is written if cap is short. */
qtng_status qtng_plan_segments(int n, int m, const int* edges, int p, int merged,
                               int max_result_width, int* ints, int64_t cap, int64_t* n_ints);
/* Host-only: the plan qtng_plan_create would build for all m edges (fuse=1:
 * fused-chain segments, fuse=0: one device op per bucket), without a device. */
qtng_status qtng_plan_stats(int n, int m, const int* edges, int p, int merged,
                            int max_result_width, int fuse, qtng_plan_info* info);
/* Records of the last execution (edge_u/edge_v filled from the selection);
 * elapsed_s = the bucket's byte share of its level's time after
 * qtng_plan_profile, else of the last run's total device time. */
qtng_status qtng_plan_records(const qtng_plan* plan, qtng_record* records, int64_t cap,
                              int64_t* n_out);
/* Device time of the last qtng_plan_profile summed per kernel kind (ms):
 * ms4[0] level_kernel, ms4[1] outer_kernel, ms4[2] seg_kernel, ms4[3]
 * seg4_kernel (quad tiles) -- CUDA events on the stream each kernel runs on.
 * per_level (optional, cap entries): the same four times for each level,
 * level-major. */
qtng_status qtng_plan_kernel_ms(const qtng_plan* plan, float* ms4, float* per_level, int cap);
/* Per-level device time of the last qtng_plan_profile (ms), n_levels entries. */
qtng_status qtng_plan_level_ms(const qtng_plan* plan, float* ms, int cap);
void qtng_plan_destroy(qtng_plan* plan);

/* Largest-bucket microbenchmark support: time one level of the plan in
 * isolation (the level containing the plan's widest bucket when level < 0).
 * Returns the level index, its algorithmic bytes and the mean device ms over
 * n_runs launches. */
qtng_status qtng_plan_time_level(qtng_plan* plan, int level, int n_runs, int* level_out,
                                 double* level_bytes, float* mean_ms);

#ifdef __cplusplus
}
#endif
#endif /* QTNG_H */
