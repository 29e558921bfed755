// Offline planning of a batch of lightcone eliminations for one device:
// level assignment across all lightcones, HBM arena placement, and the flat
// descriptor arrays the kernels consume.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "device_plan.hpp"
#include "host.hpp"

namespace qtng {

struct HostPlan {
  std::vector<DevOp> ops;              // level-sorted
  std::vector<uint32_t> ibeg;          // ops[i].item_begin, contiguous (kernel lookup table)
  std::vector<int32_t> op_width;       // bucket width per device op, 0 for pre-fold helpers
  std::vector<DevTensor> trefs;
  std::vector<DevSeg> segs;            // fused-chain segments, level-sorted
  std::vector<uint32_t> seg_ibeg;      // segs[i].item_begin, contiguous
  std::vector<DevStage> stages;
  std::vector<LevelLaunch> levels;
  // HBM bytes the device program must move (fused intermediates excluded):
  // per unit sum of its materialised inputs + its output
  double dev_bytes = 0;
  uint64_t n_fused_ops = 0;            // ops evaluated inside segments
  bool c64 = false;                    // complex64 arena/kernels (set by the caller)
  // dataflow program (flow=true): every unit in one persistent kernel
  bool flow = false;
  std::vector<FlowUnit> flow_units;    // indexed by unit id
  std::vector<uint64_t> flow_init;     // queue entries ready at start (longest remaining chain first)
  uint64_t flow_chunks = 0;            // total queue entries of one execution
  double fp64_ops = 0;                 // the reference's FP64 mul/add count (all ops)
  double seg_fp64_ops = 0;             // ... of the ops inside segments
  double single_alg_bytes = 0;         // B_alg of the single (level/outer kernel) ops
  std::vector<uint64_t> scalar_off;    // per lightcone: its scalar results, production order
  std::vector<uint32_t> lc_begin;      // n_lightcones + 1 prefix into scalar_off
  // per lightcone: its slot in the multi-GPU reduce vector (the edge index;
  // build_plan sets 0..n-1, callers overwrite before the upload)
  std::vector<int32_t> lc_edge;
  uint64_t input_elems = 0;
  uint64_t arena_elems = 0;            // peak arena size (elements)
  // accounting: B_alg = sum_in 16*2^rank + 16*2^r; ops = 2^width
  double alg_bytes = 0;
  double sum_ops = 0;
  std::vector<double> level_bytes;     // B_alg per level
  uint64_t n_buckets = 0;              // non-empty buckets (= TimingRecords)
  int max_width = 0;
  int max_result_rank = 0;
  // per lightcone record data (one per non-empty bucket, schedule order)
  std::vector<uint32_t> rec_begin;     // n_lightcones + 1
  std::vector<int32_t> rec_seq, rec_width, rec_level;
  std::vector<double> rec_bytes;
  std::vector<uint64_t> rec_out;       // arena offset of each recorded op's result
};

// Default for build_plan's `fuse`: on unless QTNG_FUSE=0.
bool fuse_default();
// Default for build_plan's `flow`: QTNG_FLOW=1.
bool flow_default();

// Plans `cones` (each the walk of one lightcone's schedule) onto one arena
// whose first `input_elems` elements hold the inputs.  Chains of buckets whose
// intermediate spans the consumer's whole width become fused segments;
// fuse=false keeps every op a separate level-kernel op (no chain fusion).
// qaoa_gates: the input region is the QAOA gate table (fill_gate_table), so
// initial operands are classified by gate slot (DevTensor::kind).
// flow: build a dataflow program (no arena reuse: every unit's output gets its
// own region, so no warp can hold a stale L1 line of it).
// stats = false skips the statistics pass (PlanInfo bytes / FP64 work /
// level bytes stay 0); records = false leaves the per-bucket records empty
// (the one-shot energy without a report needs neither)
HostPlan build_plan(const std::vector<const WalkResult*>& cones, uint64_t input_elems,
                    bool fuse = fuse_default(), bool qaoa_gates = false,
                    bool flow = flow_default(), bool stats = true, bool records = true);

}  // namespace qtng
