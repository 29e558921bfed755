// Device-side descriptors of a planned elimination, shared by the host planner
// (plan.cpp) and the sm_100a kernels (kernels.cu).
//
// HBM layout (one arena per context, complex128 = double2 elements):
//   [0, input_elems)          input region: the gate table of the current angle
//                             set (QAOA plans) or the uploaded initial tensors
//                             (explicit schedules / single buckets)
//   [input_elems, arena_elems) bucket results, placed by an offline best-fit
//                             allocator over their level lifetimes (a result
//                             lives from its producing level to its consuming
//                             level), 512-byte aligned
// Descriptors live in a separate device buffer owned by the plan.
#pragma once

#include <cstdint>

namespace qtng {

constexpr int kMaxInputs = 8;     // tensors per op (wider buckets are pre-folded)
constexpr int kMaxRank = 32;      // axes per input tensor (offsets are 32-bit)
constexpr int kMaxSumBits = 10;   // summed vars per op (merged buckets: <= 9 seen)
constexpr int kItemBits = 10;     // max outputs per warp work item = 2^kItemBits
constexpr uint8_t kSumSrc = 64;   // DevTensor::src >= kSumSrc: a summed bit

// One bucket contraction: out[k] = sum_s prod_t in_t[gather_t(k, s)].
// k runs MSB-first over the ascending kept vars, s MSB-first over the
// ascending summed vars (so s ascending == the reference's accumulation order).
struct alignas(16) DevOp {
  uint64_t out;         // arena element offset of the result
  uint32_t item_begin;  // first work item of this op inside its level
  uint32_t tref;        // index of the op's first DevTensor
  uint8_t r;            // result rank
  uint8_t ns;           // summed bits
  uint8_t nt;           // inputs (1..kMaxInputs), in bucket member order
  uint8_t cb;           // log2(outputs per work item), <= kItemBits
  // 1 when member 0 is row-invariant inside a work item (it has no output bit
  // in [5, cb), e.g. the gate on the summed variable): the kernel then loads
  // it once per item instead of once per row.  Only set for ns == 1, nt >= 2.
  uint8_t inv0;
  // Outer-join ops (run by outer_kernel): members [0, lead) are row-invariant
  // gates, member lead = "A", member lead+1 = "B" (nt == lead + 2); rb[0] is a
  // row bit of A that B lacks, rb[1] a row bit of B that A lacks.  A lane
  // computes the 4 rows over (rb[0], rb[1]) with 2 loads of A and 2 of B per
  // summed value instead of 4 + 4.
  uint8_t lead;
  uint8_t rb[2];
};
static_assert(sizeof(DevOp) == 32, "DevOp layout");

// An input operand: its arena offset and, per axis (MSB first), where the
// axis bit comes from -- output bit j (LSB-indexed) or summed bit kSumSrc+j.
struct alignas(16) DevTensor {
  uint64_t off;
  uint8_t rank;
  // kTensorRealScalar: every element is the same real number r (the QAOA |+>
  // state, gate slot 0).  A complex product with (r, 0) equals (r*x, r*y)
  // up to the sign of an exact zero, so the segment kernel scales instead of
  // multiplying (4 fewer FP64 ops, no gather).
  uint8_t kind;
  uint8_t src[kMaxRank + 6];
};
constexpr uint8_t kTensorGeneric = 0;
constexpr uint8_t kTensorRealScalar = 1;
static_assert(sizeof(DevTensor) == 48, "DevTensor layout");

// ---------------------------------------------------------------- fused chains
// A segment is a chain of L >= 2 bucket contractions op_1 -> ... -> op_L in
// which op_i (i >= 2) consumes op_{i-1}'s result as its LAST member (the
// "main") and that result spans op_i's whole width (every var of op_i), so
// each element of the intermediate X_{i-1} is used exactly once.  Only
// Y = X_L reaches HBM; the seg_kernel keeps X_1 .. X_{L-1} in registers.
//
// Index space.  A warp tile fixes Y's high rY-cY bits (the tile number) and
// its lanes cover Y's low cY = min(rY, 5) bits.  Each lane walks the
// J = L-1 digits j: bit i-2 of j is s_i, the var summed by stage i >= 2.
// DevTensor::src codes of a segment operand:
//   0..4     lane bit (Y bit b < cY)
//   8..15    digit bit (code - 8 = i - 2 for s_i)
//   32..63   tile-number bit (code - 32 = Y bit - cY)
//   64       stage 1's own summed bit (stage 1 sums at most one var)
constexpr int kSegYBits = 5;         // cY = min(rY, kSegYBits)
#ifndef QTNG_SEG_MAXJ
#define QTNG_SEG_MAXJ 4
#endif
// digits per segment (dlo/dhi tables: 4 + 1 bits).  4: the per-warp climb
// state shrinks by 1 KB, which leaves the L1 data cache 32 KB more per SM
constexpr int kSegMaxJ = QTNG_SEG_MAXJ;
constexpr int kSegMaxStages = kSegMaxJ + 1;
constexpr int kSegMaxOps = 16;       // operands per segment (all stages)
constexpr int kSegMaxNt1 = 6;        // members of stage 1
constexpr int kSegMaxNt = 4;         // members of a fused stage (incl. the main)
#ifndef QTNG_SEG_PAIR_MAXNT
#define QTNG_SEG_PAIR_MAXNT 4
#endif
constexpr int kSegPairMaxNt = QTNG_SEG_PAIR_MAXNT;  // paired rows only for stage-1 member counts up to this
constexpr int kSegQuadMaxNt = 4;    // quad tiles: stage-1 member counts 2..4
constexpr uint8_t kSegMain = 0xff;   // DevStage::main of stage 1 (no main)
constexpr uint8_t kLaneSrcEnd = 5;
constexpr uint8_t kJSrc = 8;
constexpr uint8_t kTileSrc = 32;
constexpr uint8_t kNoVar = 0xff;  // DevSeg::rb / rb2, DevStage::u: none

struct alignas(16) DevSeg {
  uint64_t out;         // arena element offset of Y
  uint32_t item_begin;  // first tile of this segment inside its level's segment group
  uint32_t tref;        // first DevTensor (stage 1's members, then stage 2's, ...)
  uint32_t stage;       // first DevStage
  uint8_t nst;          // L
  uint8_t ry;           // rank of Y
  uint8_t cy;           // in-tile Y bits
  uint8_t nops;         // DevTensors of the segment (mains included as placeholders)
  // Paired rows (cY = 5 only): a lane computes two Y rows, the tile number's
  // bit rb = 0 and = 1, sharing the digit walk, the side products and the
  // climb's control; rb is a tile bit that no side member (stage >= 2) reads,
  // so the side products are the same for both rows.  kNoVar: unpaired.  A
  // paired segment has half as many work items (tiles with bit rb removed).
  uint8_t rb;
  // Quad tiles (seg4_kernel; cY = 5, stage 1 = [prefix..., A, B]): a lane
  // computes four Y rows, tile bits rb (read by A, not by B or the prefix)
  // and rb2 (read by B only) = 0/1, the outer product of two A rows and two
  // B rows: 2 + 2 operand loads per summed value for 4 terms.  Side members
  // may read rb / rb2 (their products are then formed per row).  kNoVar:
  // not a quad segment.  A quad segment has a quarter as many work items.
  uint8_t rb2;
  uint8_t pad[6];
};
static_assert(sizeof(DevSeg) == 32, "DevSeg layout");

// Per-operand tables of a segment, built on the device once per plan upload
// (seg_prep_kernel) from the DevTensor bit maps and read by seg_kernel through
// the read-only path.  Indexed like the DevTensor array.
// log2 of a segment's work items: its tiles, halved for paired rows and
// quartered for quad tiles.
inline int seg_item_bits(const DevSeg& sg) {
  return sg.ry - sg.cy - (sg.rb2 != kNoVar ? 2 : (sg.rb != kNoVar ? 1 : 0));
}

struct alignas(16) SegOpTab {
  uint64_t off;                // arena element offset
  uint32_t sd;                 // stage 1: offset of its own summed bit
  uint32_t kind;               // DevTensor::kind
  uint32_t dj[kSegMaxJ];       // offset per digit bit
  uint32_t inc[kSegMaxJ];      // offset step from j-1 to j when bit b is the lowest set bit of j
  uint32_t dlo[16];            // subset sums of digit bits 0..3
  uint32_t dhi[16];            // subset sums of digit bits 4..7
  uint32_t dtile[32];          // offset per tile-number bit
  uint32_t llane[32];          // lane part of the offset, per lane
};
static_assert(sizeof(SegOpTab) % 16 == 0, "SegOpTab layout");

struct DevStage {
  uint8_t nt;    // members (bucket member order)
  uint8_t main;  // position of the main member (kSegMain for stage 1)
  uint8_t ns;    // summed bits of the stage (0 or 1)
  uint8_t op0;   // index of member 0 among the segment's DevTensors
  // Fused stage whose side members are all input-region tensors of rank <= 2
  // over s_i and at most two more vars u[0], u[1] (codes as DevTensor::src,
  // kNoVar if absent): the side product P_i depends only on (s_i, u) and is
  // tabulated once per tile instead of gathered per term.
  uint8_t ptab;  // 1 = tabulated
  uint8_t u[2];
  uint8_t pad;
};
static_assert(sizeof(DevStage) == 8, "DevStage layout");

// One level of the level-synchronous schedule: generic ops
// [op_begin, op_begin+op_count) of the level-sorted op array (`items` warp
// work items), then its outer-join ops [op_begin+op_count, +outer_count)
// (`outer_items` items, item_begin counted from 0 within that group).  The two
// groups run as concurrent kernels.
struct LevelLaunch {
  uint32_t op_begin;
  uint32_t op_count;
  uint32_t items;
  uint32_t max_nt;  // widest member list of the generic ops (selects the kernel instance)
  uint32_t outer_count;
  uint32_t outer_items;
  uint32_t seg_begin;  // fused-chain segments [seg_begin, seg_begin+seg_count)
  uint32_t seg_count;
  uint32_t seg_items;  // tiles
  // quad-tile segments (seg4_kernel): [seg_begin+seg_count, +seg4_count),
  // item_begin counted from 0 within that group
  uint32_t seg4_count;
  uint32_t seg4_items;
};

// ---------------------------------------------------------------- dataflow
// A "flow" program runs every unit (single op or segment) of a plan in ONE
// persistent kernel: a unit becomes ready when the units producing its
// materialised inputs have completed (each unit feeds at most one consumer),
// and warps take work items from the ready units in readiness order -- no
// level barriers, so small units overlap big ones.
struct FlowUnit {
  uint32_t idx;      // into the DevOp array (kind 0) or the DevSeg array (kind 1)
  uint32_t n_items;  // warp items (ops) or tiles (segments)
  int32_t succ;      // consuming unit, -1: none (scalar / kept result)
  uint16_t deps;     // materialised inputs produced by other units
  uint8_t kind;
  uint8_t chunk_log;  // items per queue entry = 2^chunk_log
};
static_assert(sizeof(FlowUnit) == 16, "FlowUnit layout");
// queue entry: unit << 32 | chunk index; kFlowEmpty = not yet published
constexpr uint64_t kFlowEmpty = ~uint64_t{0};
constexpr uint32_t kFlowMaxChunks = 8192;  // per unit: enough to spread over every warp

// Per-execution state of a flow program (device-only, reset by flow_reset):
// per unit: items finished and inputs still missing.  Two queues of chunks:
// "cold" = the chunks ready at start (longest remaining chain first), "hot" =
// chunks of units that became ready during the run (chain continuations,
// preferred so the critical path never waits behind bulk work).
struct FlowState {
  uint32_t head;   // cold queue (the initially ready chunks): next claim
  uint32_t tail;   // hot queue (chunks published during the run): publish counter
  uint32_t hot;    // hot queue: next claim (advanced by CAS, never past `tail`)
  uint32_t done;   // chunks finished (termination)
};

// Planner target for warp items per level: enough to cover every SM several
// times over, so small levels use 1-row items and big levels 32-row items.
constexpr uint64_t kTargetItems = 16384;

}  // namespace qtng
