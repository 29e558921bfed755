// Host-side schedule construction for the B200 bucket-elimination path.
//
// Everything here is data-free (angle-independent) integer work: graph ->
// lightcone -> expectation network -> greedy elimination order -> buckets ->
// symbolic contraction walk.  It reproduces the reference's schedule
// bit-for-bit (elimination order, bucket membership and member order, result
// routing), which is what makes the device results comparable element by
// element with the reference's NaiveBackend.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace qtng {

// Status codes of the C ABI (include/qtng.h) and the reference exception
// each stands for (proj/include/qtnsim/errors.hpp:8-36).
enum Status : int {
  kOk = 0,
  kInvalidInput = 1,  // InvalidInputError
  kResource = 2,      // ResourceError
  kSchedule = 3,      // ScheduleError
  kNumerical = 4,     // NumericalError
  kCuda = 5,          // device failure (no reference counterpart)
  kGeneration = 6,    // GenerationError
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct Edge {
  int u = 0, v = 0;
};

struct Graph {
  int n = 0;
  std::vector<Edge> edges;  // sorted lexicographically, u < v, no duplicates
};

// make_graph (proj/src/graph.cpp:30-43): normalise, sort, reject duplicates.
Graph make_graph(int n, std::vector<Edge> edges);
// random_regular (proj/src/graph.cpp:45-76): pairing model on the libstdc++
// mt19937_64 / std::shuffle stream, restarting on loops or multi-edges.
Graph random_regular(int n, int d, uint64_t seed);

struct Lightcone {
  Graph sub;                 // relabelled to 0..k-1 in ascending old id
  std::vector<int> new_to_old;
  Edge target;               // the observable edge, relabelled
};
// lightcone (proj/src/graph.cpp:87-136): every edge with an endpoint within
// graph distance p-1 of {u, v}.
Lightcone lightcone(const Graph& g, Edge e, int p);

// ---------------------------------------------------------------- gates
// Every initial tensor of an expectation network is one of 2 + 4p distinct
// gate tensors (proj/src/circuit.cpp:38-74), so the device keeps one "gate
// table" per angle set and initial tensors point into it.
enum GateSlot : int { kSlotPlus = 0, kSlotZZ = 1 };
inline int slot_phase(int k) { return 2 + 4 * k; }
inline int slot_conj_phase(int k) { return 3 + 4 * k; }
inline int slot_mixer(int k) { return 4 + 4 * k; }
inline int slot_conj_mixer(int k) { return 5 + 4 * k; }
inline int n_gate_slots(int p) { return 2 + 4 * p; }
constexpr int kSlotElems = 4;  // complex entries reserved per slot
// Gate values exactly as gate_matrix builds them (std::exp / cos / sin on
// the host), interleaved (re, im), kSlotElems entries per slot.
void fill_gate_table(int p, const double* gammas, const double* betas, double* out);

// ---------------------------------------------------------------- network
struct InitTensor {
  int rank = 0;        // 1 or 2 for gates; arbitrary for explicit schedules
  int vars[2] = {0, 0};
  int slot = 0;        // gate slot (QAOA networks)
};

struct Network {
  int n_vars = 0;
  std::vector<InitTensor> tensors;  // network order (= gate order)
};

// circuit_to_network(build_edge_expectation_circuit(g, e, a))
// (proj/src/network.cpp:18-60, proj/src/circuit.cpp:76-118).
Network expectation_network(const Lightcone& lc, int p);

// greedy_order(line_graph(net)) (proj/src/ordering.cpp:16-42,
// proj/src/network.cpp:62-74): minimum degree, ties to the smallest id,
// neighbourhood cliqued.  Bitset adjacency, O(V^2/64) per lightcone.
std::vector<int> greedy_order(const Network& net);

// ---------------------------------------------------------------- schedule
// A schedule in the reference's shape (proj/include/qtnsim/ordering.hpp:22-31)
// but with tensor payloads held by reference: tensor t of bucket i is
// either an initial tensor (index into `init`) or -- during the walk -- the
// result of an earlier bucket.
struct SchedTensor {
  std::vector<int> vars;   // axis order (MSB first)
  int64_t data = 0;        // initial: element offset of its data in the input region
};

struct SchedBucket {
  std::vector<int> sum_vars;
  std::vector<int> tensors;  // indices into Schedule::init
};

struct Schedule {
  std::vector<SchedTensor> init;
  std::vector<SchedBucket> buckets;
  // merge_buckets bookkeeping (ContractionSchedule::merges_applied/_skipped,
  // proj/include/qtnsim/ordering.hpp; counted as engine.cpp:343-353 does)
  int merges_applied = 0;
  int merges_skipped = 0;
};

// assign_buckets (proj/src/ordering.cpp:44-68) for a QAOA network; initial
// tensor data offsets are gate-slot offsets (slot * kSlotElems).
Schedule assign_buckets(const Network& net, const std::vector<int>& order);

// edge_schedule (proj/src/engine.cpp:493-501) without merging.
Schedule edge_schedule(const Graph& g, Edge e, int p);

// merge_buckets (proj/src/engine.cpp:306-358).
Schedule merge_buckets(const Schedule& s);

// ---------------------------------------------------------------- symbolic walk
// One non-empty bucket of a lightcone, contracted.  Inputs are listed in the
// bucket's member order: initial tensors in network order, then results in
// production order (the routing of contract_network, engine.cpp:286-301).
// Flat storage: every var list lives in WalkResult::vars as DENSE ids
// (0..n_vars-1, ascending order preserved); WalkResult::ids maps them back.
struct OpIn {
  int64_t ref;       // initial: element offset in the input region; else producer op index
  int32_t var_off;   // axis vars (MSB first) at vars[var_off .. var_off+rank)
  int16_t rank;
  uint8_t initial;
  uint8_t pad;
};

struct Op {
  int32_t bucket_seq;  // schedule index of the bucket (TimingRecord.bucket_seq)
  int32_t width;       // |union of vars| (TimingRecord.width)
  int32_t level;       // dependency depth (0 = only initial inputs)
  int32_t consumer;    // op consuming the result, -1 => scalar (or kept in place)
  int32_t sum_off;     // sorted summed vars at vars[sum_off .. sum_off+ns)
  int32_t out_off;     // ascending result vars at vars[out_off .. out_off+r)
  int32_t in_off;      // inputs at ins[in_off .. in_off+nin)
  int16_t ns, r;
  int32_t nin;
};

struct WalkResult {
  std::vector<Op> ops;         // in schedule (execution) order
  std::vector<OpIn> ins;
  std::vector<int32_t> vars;   // dense var ids
  std::vector<int32_t> ids;    // dense -> schedule var id
  int n_vars = 0;
  std::vector<int> scalars;    // ops with empty results, in production order
  int max_result_rank = 0;     // peak_tensor_bytes = 16 << max_result_rank
  // contract_network failure, if any (code, message); ops before it are valid
  int fail_code = 0;
  std::string fail_msg;

  const int32_t* out_vars(const Op& o) const { return vars.data() + o.out_off; }
  const int32_t* sum_vars(const Op& o) const { return vars.data() + o.sum_off; }
  const OpIn* inputs(const Op& o) const { return ins.data() + o.in_off; }
  const int32_t* in_vars(const OpIn& i) const { return vars.data() + i.var_off; }
};

// Replace every op with more than kMaxInputs members by a chain of pre-fold
// helper ops (the product of the first kMaxInputs members over their joint
// vars, no summation).  prod = (1*P)*T8*... rounds exactly like the
// reference's left fold ((1*T0)*T1)*...*T8*...  Helper ops get bucket_seq -1.
void fold_wide_ops(WalkResult& w, int max_inputs);

// The data-free contract_network walk (engine.cpp:246-304, including the
// liveness check :261-266 and contract_bucket's cap check :160-169).
// route=false keeps every result in place (single-bucket contraction).
WalkResult walk_schedule(const Schedule& s, int max_result_width, bool route = true);

// simulate_widths (engine.cpp:235-240): widths of the non-empty buckets.
std::vector<int> simulate_widths(const Schedule& s);

// Flatten a schedule to the shared int/data format used by the oracle and the
// reference wrapper (see oracle/qtn_oracle.h).  `gate_table` resolves initial
// tensor data (may be null: data left empty).
void flatten_schedule(const Schedule& s, const double* input_region, std::vector<int>& ints,
                      std::vector<double>& data);
// Inverse: parse the shared format.  Initial tensor data offsets index `data`
// in complex elements.
Schedule parse_schedule(int n_buckets, const int* ints, long n_ints);

}  // namespace qtng
