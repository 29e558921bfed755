// Offline planner: turns per-lightcone symbolic walks into one level-
// synchronous device program (see plan.hpp / device_plan.hpp).  Linear-time
// passes over flat arrays: counting sorts by level, O(1) size-class arena
// allocation, stamp-array bit maps.
#include "plan.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>

#include "pool.hpp"

namespace qtng {

namespace {
// QTNG_TIMING=2: phase times of build_plan on stderr (host tuning aid)
struct PlanTimer {
  bool on;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  PlanTimer() {
    static const bool e = [] {
      const char* v = std::getenv("QTNG_TIMING");
      return v && v[0] == '2';
    }();
    on = e;
  }
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "build_plan %s %.3f ms\n", what,
                 std::chrono::duration<double>(now - t).count() * 1e3);
    t = now;
  }
};
}  // namespace


namespace {

constexpr uint64_t kAlign = 32;  // elements (512 B)
constexpr int kMinClass = 5;     // results are allocated in 2^max(r,5) blocks

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Member 0 row-invariant inside an item (no output bit in [5, cb)): the
// kernel hoists its loads out of the row loop (DevOp::inv0).
void mark_invariant_lead(DevOp& d, const DevTensor* ts) {
  d.inv0 = 0;
  if (d.ns != 1 || d.nt < 2) return;
  for (int ax = 0; ax < ts[0].rank; ++ax) {
    const int src = ts[0].src[ax];
    if (src >= 5 && src < d.cb) return;
  }
  d.inv0 = 1;
}

// Tuning switch: QTNG_OUTER=0 routes outer-join ops through the generic kernel.
bool outer_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("QTNG_OUTER");
    return !(v && v[0] == '0');
  }();
  return on;
}

// Power-of-two size classes; a class's freed blocks are reused first-in
// last-out, fresh blocks come from the top.  Result lifetimes are level
// intervals, so reuse is dense and the peak stays near the live maximum.
class ClassArena {
 public:
  explicit ClassArena(uint64_t base) : top_(base) {}
  uint64_t alloc(int cls) {
    if (cls < static_cast<int>(free_.size()) && !free_[cls].empty()) {
      const uint64_t off = free_[cls].back();
      free_[cls].pop_back();
      return off;
    }
    const uint64_t off = top_;
    top_ += uint64_t{1} << cls;
    return off;
  }
  void release(int cls, uint64_t off) {
    if (cls >= static_cast<int>(free_.size())) free_.resize(cls + 1);
    free_[cls].push_back(off);
  }
  uint64_t peak() const { return top_; }

 private:
  uint64_t top_;
  std::vector<std::vector<uint64_t>> free_;
};

}  // namespace

// Digits per segment (L - 1): QTNG_SEG_J, default 5 (tuned on C2: shorter
// segments give more, cheaper tiles; longer ones cut HBM traffic further).
int seg_max_j() {
  static const int j = [] {
    // 4 (measured, with quad tiles): C2 2.24 ms vs 2.28 ms at J = 5; 8-way
    // shard floor 0.53 vs 0.59 ms
    const char* v = std::getenv("QTNG_SEG_J");
    const int x = v ? std::atoi(v) : 4;
    return std::max(1, std::min(x, kSegMaxJ));
  }();
  return j;
}

// Level assignment of the units (QTNG_LEVELS): 0 = as soon as possible
// (1 + the deepest producer); 1 = each lightcone's ASAP levels shifted so all
// lightcones end on the last level; 2 = as late as possible (a unit runs on
// the level before its consumer; roots on the last level; default).
// Measured (graph replay, 1x B200): C2 2.10 / 2.05 / 1.87 ms, C4 seed 9
// 1.18 / 1.13 / 1.04 ms for modes 0 / 1 / 2 -- a late unit shares its level
// with the other lightcones' late units instead of idling the SMs early.
int level_mode() {
  static const int m = [] {
    const char* v = std::getenv("QTNG_LEVELS");
    return v ? std::atoi(v) : 2;
  }();
  return m;
}

// Levels whose segments have fewer tiles than this put digits on lanes
// (QTNG_SEG_STARVED; default 0 = never: with ALAP levels, 0 vs 1024
// measured C2 1.853 vs 1.871 ms, 8-way shard 0.491 vs 0.505 ms).
// Segments of levels with at least this many tiles pair their rows
// (DevSeg::rb; QTNG_SEG_PAIR, default 8192; 0 disables pairing).
uint64_t seg_pair_min_tiles() {
  static const uint64_t t = [] {
    const char* v = std::getenv("QTNG_SEG_PAIR");
    return static_cast<uint64_t>(v ? std::atoll(v) : 8192);
  }();
  return t;
}

// Stage-1 member counts paired (QTNG_SEG_PAIR_NT, at most kSegPairMaxNt).
int seg_pair_max_nt() {
  static const int t = [] {
    const char* v = std::getenv("QTNG_SEG_PAIR_NT");
    return std::min(v ? std::atoi(v) : kSegPairMaxNt, kSegPairMaxNt);
  }();
  return t;
}

// Segments of levels with at least this many tiles may use quad tiles when
// their head is an outer join (DevSeg::rb2; QTNG_SEG_QUAD, default 32768 --
// a quad tile is a quarter of the work items, so smaller levels starve; 0
// disables).  Measured on C2 (graph replay, J = 5): 8192 / 16384 / 32768 /
// 65536 -> 2.32 / 2.30 / 2.29 / 2.27 ms vs 2.32 ms without quad tiles; with
// J = 4: 32768 -> 2.234, 65536 -> 2.243 ms.
uint64_t seg_quad_min_tiles() {
  static const uint64_t t = [] {
    const char* v = std::getenv("QTNG_SEG_QUAD");
    return static_cast<uint64_t>(v ? std::atoll(v) : 32768);
  }();
  return t;
}

// Quad-tile segments run in their own kernel (seg4_kernel: its own register
// budget and tile queue, concurrent with seg_kernel).
bool seg4_split() { return true; }

// Quad tiles are used when their row score is below this multiple of the
// paired / single-row score (QTNG_SEG_QUAD_MARGIN, default 1.2: the score
// counts loads only, and a quad row also saves FP64 work and side lookups).
double seg_quad_margin() {
  static const double m = [] {
    const char* v = std::getenv("QTNG_SEG_QUAD_MARGIN");
    return v ? std::atof(v) : 1.2;
  }();
  return m;
}

// Tile-number bits (Y bits above the lanes) an operand of a segment reads.
uint32_t seg_tile_bits(const DevTensor& x) {
  uint32_t b = 0;
  for (int ax = 0; ax < x.rank; ++ax)
    if (x.src[ax] >= kTileSrc && x.src[ax] < kSumSrc) b |= 1u << (x.src[ax] - kTileSrc);
  return b;
}

// Operand loads per output row and tile pass of a segment whose lanes each
// compute the rows spanned by the tile bits `rows` (see the row-tiling
// choice in build_plan).  tr: the segment's DevTensors.
double seg_row_score(const DevSeg& sg, const DevStage* sts, const DevTensor* tr, uint32_t rows) {
  const int J = sg.nst - 1;
  double loads = 0.0;
  for (int t = 0; t < sts[0].nt; ++t) {
    const DevTensor& x = tr[sts[0].op0 + t];
    if (x.kind == kTensorRealScalar) continue;
    loads += std::ldexp(1.0, J + sts[0].ns + __builtin_popcount(seg_tile_bits(x) & rows));
  }
  for (int i = 1; i < sg.nst; ++i) {
    const double terms = std::ldexp(1.0, J - i + 1);
    if (sts[i].ptab) {
      int nr = 0;
      for (int w = 0; w < 2; ++w)
        if (sts[i].u[w] >= kTileSrc && sts[i].u[w] < kSumSrc && ((rows >> (sts[i].u[w] - kTileSrc)) & 1u)) ++nr;
      loads += 0.5 * terms * std::ldexp(1.0, nr);
      continue;
    }
    for (int t = 0; t < sts[i].nt; ++t) {
      if (t == sts[i].main) continue;
      const DevTensor& x = tr[sts[i].op0 + t];
      if (x.kind == kTensorRealScalar) continue;
      loads += terms * std::ldexp(1.0, __builtin_popcount(seg_tile_bits(x) & rows));
    }
  }
  return loads / std::ldexp(1.0, __builtin_popcount(rows));
}

uint64_t seg_starved_tiles() {
  static const uint64_t t = [] {
    const char* v = std::getenv("QTNG_SEG_STARVED");
    return static_cast<uint64_t>(v ? std::atoll(v) : 0);
  }();
  return t;
}

bool flow_default() {
  static const bool on = [] {
    const char* v = std::getenv("QTNG_FLOW");
    return v && v[0] == '1';
  }();
  return on;
}

bool fuse_default() {
  static const bool on = [] {
    const char* v = std::getenv("QTNG_FUSE");
    return !(v && v[0] == '0');
  }();
  return on;
}

HostPlan build_plan(const std::vector<const WalkResult*>& cones, uint64_t input_elems, bool fuse,
                    bool qaoa_gates, bool flow, bool stats, bool records) {
  HostPlan hp;
  hp.input_elems = input_elems;
  const int C = static_cast<int>(cones.size());
  std::vector<uint32_t> base(C + 1, 0);
  int max_vars = 0;
  for (int c = 0; c < C; ++c) {
    base[c + 1] = base[c] + static_cast<uint32_t>(cones[c]->ops.size());
    max_vars = std::max(max_vars, cones[c]->n_vars);
    hp.max_result_rank = std::max(hp.max_result_rank, cones[c]->max_result_rank);
  }
  const uint32_t N = base[C];
  std::vector<uint32_t> lc_of(N);
  for (int c = 0; c < C; ++c)
    for (uint32_t k = 0; k < cones[c]->ops.size(); ++k) {
      const Op& o = cones[c]->ops[k];
      if (o.nin > kMaxInputs) throw Error(kSchedule, "internal: op not pre-folded");
      if (o.ns > kMaxSumBits)
        throw Error(kInvalidInput, "bucket sums " + std::to_string(o.ns) +
                                       " variables; the device path supports at most " +
                                       std::to_string(kMaxSumBits));
      lc_of[base[c] + k] = c;
    }
  auto op_at = [&](uint32_t g) -> const Op& { return cones[lc_of[g]]->ops[g - base[lc_of[g]]]; };

  PlanTimer ptm;
  // ---- units: single ops, or fused chains (segments, see device_plan.hpp)
  // main_pos[g]: position of op g's fused main member, -1 when g heads its unit
  std::vector<int8_t> main_pos(N, -1);
  std::vector<uint32_t> unit_of(N);
  std::vector<uint32_t> next_in_unit(N, ~0u);
  // per cone in parallel (units never span lightcones), cone-local unit ids
  struct ConeUnits {
    std::vector<uint32_t> first, last, len, nops;
    int max_level = -1;
  };
  std::vector<ConeUnits> cus(C);
  Pool::get().parallel_for(C, [&](int c) {
    const WalkResult& w = *cones[c];
    ConeUnits& cu = cus[c];
    for (uint32_t k = 0; k < w.ops.size(); ++k) {
      const uint32_t g = base[c] + k;
      const Op& o = w.ops[k];
      // the main must be the LAST member: the stage term is then
      // P_i(s) * X_{i-1}(s) with P_i the left fold of the other members
      int t_main = -1;
      if (fuse && o.ns == 1 && o.nin <= kSegMaxNt) {
        const OpIn& in = w.inputs(o)[o.nin - 1];
        if (!in.initial && w.ops[in.ref].r == o.width) t_main = o.nin - 1;
      }
      if (t_main >= 0) {
        const uint32_t pg = base[c] + static_cast<uint32_t>(w.inputs(o)[t_main].ref);
        const Op& p = w.ops[pg - base[c]];
        const uint32_t u = unit_of[pg];
        const bool head_ok = cu.len[u] > 1 || (p.ns <= 1 && p.nin <= kSegMaxNt1);
        const int L = static_cast<int>(cu.len[u]) + 1;
        if (head_ok && cu.last[u] == pg && L - 1 <= seg_max_j() &&
            cu.nops[u] + static_cast<uint32_t>(o.nin) <= static_cast<uint32_t>(kSegMaxOps)) {
          main_pos[g] = static_cast<int8_t>(t_main);
          unit_of[g] = u;
          next_in_unit[pg] = g;
          cu.last[u] = g;
          ++cu.len[u];
          cu.nops[u] += static_cast<uint32_t>(o.nin);
          continue;
        }
      }
      unit_of[g] = static_cast<uint32_t>(cu.first.size());
      cu.first.push_back(g);
      cu.last.push_back(g);
      cu.len.push_back(1);
      cu.nops.push_back(static_cast<uint32_t>(o.nin));
    }
  });
  std::vector<uint32_t> ubase(C + 1, 0);
  for (int c = 0; c < C; ++c) ubase[c + 1] = ubase[c] + static_cast<uint32_t>(cus[c].first.size());
  const uint32_t U = ubase[C];
  std::vector<uint32_t> unit_first(U), unit_last(U), unit_len(U), unit_nops(U);
  ptm.mark("units");
  // unit levels: 1 + the deepest unit producing a materialised input; units
  // are visited in the order of their last op (producers come first)
  std::vector<int32_t> unit_level(U, 0);
  Pool::get().parallel_for(C, [&](int c) {
    ConeUnits& cu = cus[c];
    const uint32_t ub = ubase[c];
    std::copy(cu.first.begin(), cu.first.end(), unit_first.begin() + ub);
    std::copy(cu.last.begin(), cu.last.end(), unit_last.begin() + ub);
    std::copy(cu.len.begin(), cu.len.end(), unit_len.begin() + ub);
    std::copy(cu.nops.begin(), cu.nops.end(), unit_nops.begin() + ub);
    const WalkResult& w = *cones[c];
    for (uint32_t k = 0; k < w.ops.size(); ++k) unit_of[base[c] + k] += ub;
    for (uint32_t k = 0; k < w.ops.size(); ++k) {
      const uint32_t g = base[c] + k;
      const uint32_t u = unit_of[g];
      if (unit_last[u] != g) continue;
      int lvl = 0;
      for (uint32_t s = unit_first[u]; s != ~0u; s = next_in_unit[s]) {
        const Op& o = w.ops[s - base[c]];
        const OpIn* ins = w.inputs(o);
        for (int t = 0; t < o.nin; ++t) {
          if (ins[t].initial || t == main_pos[s]) continue;
          lvl = std::max(lvl, unit_level[unit_of[base[c] + static_cast<uint32_t>(ins[t].ref)]] + 1);
        }
      }
      unit_level[u] = lvl;
      cu.max_level = std::max(cu.max_level, lvl);
    }
  });
  int max_level = -1;
  for (const ConeUnits& cu : cus) max_level = std::max(max_level, cu.max_level);
  const int n_levels = max_level + 1;
  auto level_of = [&](uint32_t g) { return unit_level[unit_of[g]]; };
  auto consumer_unit = [&](uint32_t u) -> int64_t {
    const Op& o = op_at(unit_last[u]);
    return o.consumer >= 0 ? static_cast<int64_t>(unit_of[base[lc_of[unit_last[u]]] + o.consumer]) : -1;
  };
  if (level_mode() == 1) {
    Pool::get().parallel_for(C, [&](int c) {
      const int shift = max_level - cus[c].max_level;
      for (uint32_t u = ubase[c]; u < ubase[c + 1]; ++u) unit_level[u] += shift;
    });
  } else if (level_mode() == 2) {
    // a consumer's last op follows its producers' last ops: visiting units
    // in descending order of their last op sees every consumer first
    Pool::get().parallel_for(C, [&](int c) {
      for (uint32_t k = static_cast<uint32_t>(cones[c]->ops.size()); k-- > 0;) {
        const uint32_t g = base[c] + k, u = unit_of[g];
        if (unit_last[u] != g) continue;
        const int64_t cu = consumer_unit(u);
        unit_level[u] = cu >= 0 ? unit_level[cu] - 1 : max_level;
      }
    });
  }

  // stable counting sort of units by level; release lists by consumer level
  std::vector<uint32_t> lstart(n_levels + 1, 0), order(U);
  std::vector<uint32_t> rstart(n_levels + 1, 0), rel;
  std::vector<uint64_t> level_rows(n_levels, 0), level_tiles(n_levels, 0);
  for (uint32_t u = 0; u < U; ++u) {
    ++lstart[unit_level[u] + 1];
    const Op& o = op_at(unit_last[u]);
    if (unit_len[u] == 1) level_rows[unit_level[u]] += o.r > 5 ? uint64_t{1} << (o.r - 5) : 1;
    else level_tiles[unit_level[u]] += o.r > kSegYBits ? uint64_t{1} << (o.r - kSegYBits) : 1;
    const int64_t cu = consumer_unit(u);
    if (cu >= 0) ++rstart[unit_level[cu] + 1];
  }
  for (int L = 0; L < n_levels; ++L) {
    lstart[L + 1] += lstart[L];
    rstart[L + 1] += rstart[L];
  }
  rel.resize(rstart[n_levels]);
  {
    std::vector<uint32_t> lf(lstart.begin(), lstart.end() - 1), rf(rstart.begin(), rstart.end() - 1);
    for (uint32_t u = 0; u < U; ++u) {
      order[lf[unit_level[u]]++] = u;
      const int64_t cu = consumer_unit(u);
      if (cu >= 0) rel[rf[unit_level[cu]]++] = u;
    }
  }

  ptm.mark("levels");
  // arena placement of unit outputs over level lifetimes; scalars / kept
  // results live to the end; fused intermediates get no storage
  constexpr uint64_t kNoOut = ~uint64_t{0};
  std::vector<uint64_t> out(N, kNoOut);
  ClassArena arena(round_up(input_elems, kAlign));
  auto cls_of = [&](uint32_t u) { return std::max<int>(op_at(unit_last[u]).r, kMinClass); };
  for (int L = 0; L < n_levels; ++L) {
    if (L > 0 && !flow)  // flow programs never reuse a region
      for (uint32_t i = rstart[L - 1]; i < rstart[L]; ++i)
        arena.release(cls_of(rel[i]), out[unit_last[rel[i]]]);
    for (uint32_t i = lstart[L]; i < lstart[L + 1]; ++i)
      out[unit_last[order[i]]] = arena.alloc(cls_of(order[i]));
  }
  hp.arena_elems = arena.peak();

  // item size per level: 32-output rows per warp item, fewer for small levels
  // so the level still spreads over the whole GPU
  std::vector<int> level_cb(n_levels);
  for (int L = 0; L < n_levels; ++L) {
    int row_bits = 0;
    while (row_bits < kItemBits - 5 && (level_rows[L] >> (row_bits + 1)) >= kTargetItems) ++row_bits;
    level_cb[L] = 5 + row_bits;
  }
  // Y bits on the lanes of a segment tile: 5, unless the level's segments
  // have too few tiles to occupy the GPU (small plans, one GPU's shard of a
  // few lightcones) -- then fewer Y bits and the lowest digits move onto the
  // freed lanes (shorter serial digit walks per tile)
  std::vector<int> level_cy(n_levels, kSegYBits);
  for (int L = 0; L < n_levels; ++L) {
    int h = 0;
    while (h < kSegYBits && level_tiles[L] && (level_tiles[L] << h) < seg_starved_tiles()) ++h;
    level_cy[L] = kSegYBits - h;
  }
  auto seg_cy = [&](uint32_t u) {
    return std::min<int>(op_at(unit_last[u]).r, level_cy[unit_level[u]]);
  };
  ptm.mark("arena");
  // outer-join classification of single-op units (DevOp::lead/rb), in parallel
  std::vector<uint32_t> outer_sig(N, 0);  // 0 = generic; else 1 | lead<<8 | rb0<<16 | rb1<<24
  {
    const int chunks = static_cast<int>(std::min<uint32_t>(N, 256));
    Pool::get().parallel_for(chunks, [&](int ch) {
      std::vector<uint8_t> pm(max_vars);
      std::vector<uint32_t> pm_stamp(max_vars, ~0u);
      for (uint32_t g = static_cast<uint32_t>(uint64_t{N} * ch / chunks);
           g < static_cast<uint32_t>(uint64_t{N} * (ch + 1) / chunks); ++g) {
        if (unit_len[unit_of[g]] != 1) continue;
        const Op& o = op_at(g);
        const int cb = std::min<int>(o.r, level_cb[level_of(g)]);
        if (!outer_enabled() || o.ns != 1 || o.nin < 2 || o.nin > 4 || cb < 7) continue;
        const WalkResult& w = *cones[lc_of[g]];
        const int32_t* ov = w.out_vars(o);
        for (int k = 0; k < o.r; ++k) { pm[ov[k]] = static_cast<uint8_t>(o.r - 1 - k); pm_stamp[ov[k]] = g; }
        const uint64_t rowmask = ((uint64_t{1} << cb) - 1) & ~uint64_t{31};
        uint64_t mask[kMaxInputs] = {};
        const OpIn* ins = w.inputs(o);
        for (int t = 0; t < o.nin; ++t)
          for (int ax = 0; ax < ins[t].rank; ++ax) {
            const int v = w.in_vars(ins[t])[ax];
            if (pm_stamp[v] == g) mask[t] |= uint64_t{1} << pm[v];
          }
        int lead = 0;
        while (lead < o.nin && (mask[lead] & rowmask) == 0) ++lead;
        if (lead != o.nin - 2) continue;
        const uint64_t a_only = mask[lead] & ~mask[lead + 1] & rowmask;
        const uint64_t b_only = mask[lead + 1] & ~mask[lead] & rowmask;
        if (!a_only || !b_only) continue;
        const int rb0 = __builtin_ctzll(a_only), rb1 = __builtin_ctzll(b_only);
        outer_sig[g] = 1u | (static_cast<uint32_t>(lead) << 8) | (static_cast<uint32_t>(rb0) << 16) |
                       (static_cast<uint32_t>(rb1) << 24);
      }
    });
  }
  // per level: generic single ops, outer-join single ops, segments (stable)
  auto group_of = [&](uint32_t u) {
    return unit_len[u] > 1 ? 2 : (outer_sig[unit_last[u]] != 0 ? 1 : 0);
  };
  // segments: most expensive tile first (the seg_kernel's dynamic queue then
  // schedules longest-processing-time first)
  auto seg_cost = [&](uint32_t u) {
    return (uint64_t{1} << (unit_len[u] - 1)) * (unit_nops[u] + op_at(unit_first[u]).nin);
  };
  Pool::get().parallel_for(n_levels, [&](int L) {
    // sort keys first: the comparator would chase op pointers O(n log n) times
    const uint32_t n = lstart[L + 1] - lstart[L];
    std::vector<std::pair<uint64_t, uint32_t>> key(n);
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t u = order[lstart[L] + i];
      const int gr = group_of(u);
      // group ascending, then (segments) cost descending, then stable
      const uint64_t cost = gr == 2 ? seg_cost(u) : 0;
      key[i] = {(static_cast<uint64_t>(gr) << 56) | ((~cost) & ((uint64_t{1} << 56) - 1)), i};
    }
    std::sort(key.begin(), key.end());
    std::vector<uint32_t> tmp(n);
    for (uint32_t i = 0; i < n; ++i) tmp[i] = order[lstart[L] + key[i].second];
    std::copy(tmp.begin(), tmp.end(), order.begin() + lstart[L]);
  });

  ptm.mark("outer+order");
  // descriptors, level by level: item/tref prefix sums sequentially ...
  std::vector<uint32_t> unit_slot(U);   // index into hp.ops or hp.segs
  std::vector<uint32_t> unit_tref(U);
  uint32_t n_trefs = 0, n_ops_dev = 0, n_segs = 0, n_stages = 0;
  for (uint32_t u = 0; u < U; ++u) {
    if (unit_len[u] == 1) ++n_ops_dev; else { ++n_segs; n_stages += unit_len[u]; }
  }
  hp.ops.resize(n_ops_dev);
  hp.ibeg.resize(n_ops_dev);
  hp.op_width.resize(n_ops_dev);
  hp.segs.resize(n_segs);
  hp.seg_ibeg.resize(n_segs);
  hp.stages.resize(n_stages);
  hp.level_bytes.assign(n_levels, 0.0);
  std::vector<uint32_t> unit_stage(U, 0);
  {
    uint32_t io = 0, is = 0, ist = 0;
    for (int L = 0; L < n_levels; ++L) {
      LevelLaunch ll{io, 0, 0, 0, 0, 0, is, 0, 0, 0, 0};
      for (uint32_t i = lstart[L]; i < lstart[L + 1]; ++i) {
        const uint32_t u = order[i];
        unit_tref[u] = n_trefs;
        n_trefs += unit_nops[u];
        if (unit_len[u] > 1) {
          const uint32_t g = unit_last[u];
          const Op& o = op_at(g);
          DevSeg& sg = hp.segs[is];
          unit_slot[u] = is++;
          sg.out = out[g];
          sg.tref = unit_tref[u];
          sg.stage = ist;
          unit_stage[u] = ist;
          ist += unit_len[u];
          sg.nst = static_cast<uint8_t>(unit_len[u]);
          sg.ry = static_cast<uint8_t>(o.r);
          sg.cy = static_cast<uint8_t>(seg_cy(u));
          sg.nops = static_cast<uint8_t>(unit_nops[u]);
          sg.rb = kNoVar;  // chosen with the operand maps below
          sg.rb2 = kNoVar;
          sg.item_begin = ll.seg_items;
          hp.seg_ibeg[is - 1] = ll.seg_items;
          const uint64_t tiles = uint64_t{1} << (o.r - sg.cy);
          if (ll.seg_items + tiles > 0xffffffffull) throw Error(kResource, "level has too many tiles");
          ll.seg_items += static_cast<uint32_t>(tiles);
          ++ll.seg_count;
          continue;
        }
        const uint32_t g = unit_last[u];
        const Op& o = op_at(g);
        const bool outer = outer_sig[g] != 0;
        DevOp& d = hp.ops[io];
        unit_slot[u] = io;
        d.out = out[g];
        d.tref = unit_tref[u];
        d.r = static_cast<uint8_t>(o.r);
        d.ns = static_cast<uint8_t>(o.ns);
        d.nt = static_cast<uint8_t>(o.nin);
        d.cb = static_cast<uint8_t>(std::min<int>(o.r, level_cb[L]));
        d.lead = outer ? static_cast<uint8_t>((outer_sig[g] >> 8) & 0xff) : 0;
        d.rb[0] = outer ? static_cast<uint8_t>((outer_sig[g] >> 16) & 0xff) : 0;
        d.rb[1] = outer ? static_cast<uint8_t>(outer_sig[g] >> 24) : 0;
        uint32_t& items_acc = outer ? ll.outer_items : ll.items;
        d.item_begin = items_acc;
        const uint64_t items = uint64_t{1} << (o.r - d.cb);
        if (items_acc + items > 0xffffffffull) throw Error(kResource, "level has too many work items");
        items_acc += static_cast<uint32_t>(items);
        if (outer) {
          ++ll.outer_count;
        } else {
          ++ll.op_count;
          ll.max_nt = std::max<uint32_t>(ll.max_nt, d.nt);
        }
        hp.ibeg[io] = d.item_begin;
        hp.op_width[io] = o.bucket_seq >= 0 ? o.width : 0;
        ++io;
      }
      hp.levels.push_back(ll);
    }
  }
  ptm.mark("prefix");
  // ... then every operand's bit map in parallel chunks
  hp.trefs.resize(n_trefs);
  std::vector<double> op_bytes(N, 0.0), unit_dev_bytes(U, 0.0);
  const int chunks = static_cast<int>(std::min<uint32_t>(U, 256));
  std::vector<int> chunk_err(chunks, 0);
  Pool::get().parallel_for(chunks, [&](int ch) {
    const uint32_t u0 = static_cast<uint32_t>(uint64_t{U} * ch / chunks);
    const uint32_t u1 = static_cast<uint32_t>(uint64_t{U} * (ch + 1) / chunks);
    std::vector<uint8_t> pm(max_vars);
    std::vector<uint32_t> pm_stamp(max_vars, ~0u);
    uint32_t stamp = 0;
    for (uint32_t u = u0; u < u1; ++u) {
      const uint32_t c = lc_of[unit_first[u]];
      const WalkResult& w = *cones[c];
      const uint32_t cb0 = base[c];
      const Op& last = op_at(unit_last[u]);
      const bool seg = unit_len[u] > 1;
      ++stamp;
      // var -> code.  Single op: output bit (LSB-indexed) / kSumSrc + j.
      // Segment: Y bit -> in-tile or tile-number bit; digit s_k -> in-tile bit
      const int ry = last.r, cy = seg ? seg_cy(u) : 0;
      const int32_t* ov = w.out_vars(last);
      for (int k = 0; k < ry; ++k) {
        const int b = ry - 1 - k;
        pm[ov[k]] = static_cast<uint8_t>(!seg ? b : (b < cy ? b : kTileSrc + (b - cy)));
        pm_stamp[ov[k]] = stamp;
      }
      double dev_bytes = 16.0 * static_cast<double>(uint64_t{1} << ry);
      uint32_t tix = unit_tref[u];
      int stage = 0;
      for (uint32_t g = unit_first[u]; g != ~0u; g = next_in_unit[g], ++stage) {
        const Op& o = op_at(g);
        const int32_t* sv = w.sum_vars(o);
        // own summed vars; in a segment, stage i >= 2 sums digit s_i = j bit i-2
        for (int k = 0; k < o.ns; ++k) {
          pm[sv[k]] = static_cast<uint8_t>(seg && stage > 0 ? kJSrc + (stage - 1) : kSumSrc + o.ns - 1 - k);
          pm_stamp[sv[k]] = stamp;
        }
        if (seg) {
          // digits of the later stages: s_k (1-based k = stage + 2 .. L) = j bit k-2
          uint32_t h = next_in_unit[g];
          for (int k = stage + 2; h != ~0u; h = next_in_unit[h], ++k) {
            const Op& oh = op_at(h);
            const int32_t v = w.sum_vars(oh)[0];
            pm[v] = static_cast<uint8_t>(kJSrc + (k - 2));
            pm_stamp[v] = stamp;
          }
          DevStage& st = hp.stages[unit_stage[u] + stage];
          st = DevStage{};
          st.nt = static_cast<uint8_t>(o.nin);
          st.main = stage == 0 ? kSegMain : static_cast<uint8_t>(main_pos[g]);
          st.ns = static_cast<uint8_t>(o.ns);
          st.op0 = static_cast<uint8_t>(tix - unit_tref[u]);
          st.u[0] = st.u[1] = kNoVar;
        }
        double bytes = 16.0 * static_cast<double>(uint64_t{1} << o.r);
        const OpIn* ins = w.inputs(o);
        for (int t = 0; t < o.nin; ++t, ++tix) {
          const OpIn& in = ins[t];
          bytes += 16.0 * static_cast<double>(uint64_t{1} << in.rank);
          DevTensor& x = hp.trefs[tix];
          x = DevTensor{};
          if (seg && t == main_pos[g]) continue;  // placeholder: read from shared memory
          dev_bytes += 16.0 * static_cast<double>(uint64_t{1} << in.rank);
          if (in.rank > kMaxRank) { chunk_err[ch] = 1; return; }
          x.off = in.initial ? static_cast<uint64_t>(in.ref) : out[cb0 + in.ref];
          if (x.off == kNoOut) { chunk_err[ch] = 3; return; }
          x.rank = static_cast<uint8_t>(in.rank);
          if (qaoa_gates && in.initial && in.rank == 1 && in.ref == kSlotPlus * kSlotElems)
            x.kind = kTensorRealScalar;
          const int32_t* iv = w.in_vars(in);
          for (int ax = 0; ax < in.rank; ++ax) {
            if (pm_stamp[iv[ax]] != stamp) { chunk_err[ch] = 2; return; }
            x.src[ax] = pm[iv[ax]];
          }
        }
        op_bytes[g] = bytes;
        if (seg && stage > 0) {  // tabulate P_i when its members are small input tensors
          DevStage& st = hp.stages[unit_stage[u] + stage];
          const uint8_t own = static_cast<uint8_t>(kJSrc + (stage - 1));
          bool ok = st.main == o.nin - 1 && o.nin > 1;
          int nu = 0;
          for (int t = 0; ok && t < st.main; ++t) {
            const OpIn& in = ins[t];
            const DevTensor& x = hp.trefs[tix - o.nin + t];
            if (!in.initial || in.rank > 2) { ok = false; break; }
            for (int ax = 0; ax < x.rank; ++ax) {
              const uint8_t c = x.src[ax];
              if (c == own || (nu > 0 && st.u[0] == c) || (nu > 1 && st.u[1] == c)) continue;
              if (nu == 2) { ok = false; break; }
              st.u[nu++] = c;
            }
          }
          st.ptab = ok ? 1 : 0;
          if (!ok) st.u[0] = st.u[1] = kNoVar;
        }
        // the summed vars of this stage never reappear
        if (seg) for (int k = 0; k < o.ns; ++k) pm_stamp[sv[k]] = 0;
      }
      // Row tiling of the segment's lanes (DevSeg::rb / rb2).  Score = operand
      // loads per output row and tile pass (the L1 data path that a load's
      // register write-back occupies is seg_kernel's bound): stage-1 members
      // load per digit assignment and summed value once per distinct row they
      // read; a stage-i side member once per term (2^(J-i+1) terms) and
      // distinct row, a tabulated side product at half a load.
      bool quad = false;
      double quad_score = 0.0;
      if (seg && !flow && cy == kSegYBits && ry >= cy + 2 && seg_quad_min_tiles() &&
          level_tiles[unit_level[u]] >= seg_quad_min_tiles()) {
        // quad tiles: stage 1 = [prefix..., A, B] with a tile bit A reads
        // alone (rb) and one B reads alone (rb2)
        DevSeg& sg = hp.segs[unit_slot[u]];
        const DevStage* sts = hp.stages.data() + unit_stage[u];
        const int nt = sts[0].nt;
        if (nt >= 2 && nt <= kSegQuadMaxNt && sts[0].ns <= 1) {
          const DevTensor* m1 = hp.trefs.data() + unit_tref[u] + sts[0].op0;
          const DevTensor& A = m1[nt - 2];
          const DevTensor& B = m1[nt - 1];
          uint32_t pre = 0;
          for (int t = 0; t < nt - 2; ++t) pre |= seg_tile_bits(m1[t]);
          const uint32_t ta = seg_tile_bits(A), tb = seg_tile_bits(B);
          const uint32_t aonly = ta & ~tb & ~pre, bonly = tb & ~ta & ~pre;
          if (aonly && bonly && A.kind != kTensorRealScalar && B.kind != kTensorRealScalar) {
            // row bits no gathered side member reads (its product is shared
            // by the four rows; tabulated ones are looked up per row)
            uint32_t gside = 0;
            const DevTensor* tr = hp.trefs.data() + unit_tref[u];
            for (int i = 1; i < sg.nst; ++i) {
              if (sts[i].ptab) continue;
              for (int t = 0; t < sts[i].nt; ++t)
                if (t != sts[i].main) gside |= seg_tile_bits(tr[sts[i].op0 + t]);
            }
            int ba = -1, bb = -1;
            double best = 0.0;
            for (int a = 0; a < ry - cy; ++a) {
              if (!((aonly >> a) & 1u) || ((gside >> a) & 1u)) continue;
              for (int b = 0; b < ry - cy; ++b) {
                if (!((bonly >> b) & 1u) || ((gside >> b) & 1u)) continue;
                const double sc = seg_row_score(sg, sts, hp.trefs.data() + unit_tref[u],
                                                (1u << a) | (1u << b));
                if (ba < 0 || sc < best) {
                  best = sc;
                  ba = a;
                  bb = b;
                }
              }
            }
            if (ba >= 0) {
              sg.rb = static_cast<uint8_t>(ba);
              sg.rb2 = static_cast<uint8_t>(bb);
              quad = true;
              quad_score = best;
            }
          }
        }
      }
      if (!seg) {
        DevOp& d = hp.ops[unit_slot[u]];
        mark_invariant_lead(d, hp.trefs.data() + d.tref);
      } else if (!quad && cy == kSegYBits && ry > cy && seg_pair_min_tiles() &&
                 hp.stages[unit_stage[u]].nt <= seg_pair_max_nt() &&
                 level_tiles[unit_level[u]] >= seg_pair_min_tiles()) {
        // paired rows: a tile bit no side member reads, preferring one that
        // few stage-1 members read (their second-row loads differ)
        DevSeg& sg = hp.segs[unit_slot[u]];
        const DevStage* sts = hp.stages.data() + unit_stage[u];
        uint32_t side = 0, n1[32] = {};
        for (int i = 0; i < sg.nst; ++i)
          for (int t = 0; t < sts[i].nt; ++t) {
            if (i > 0 && t == sts[i].main) continue;
            const DevTensor& x = hp.trefs[unit_tref[u] + sts[i].op0 + t];
            for (int ax = 0; ax < x.rank; ++ax) {
              const uint8_t c = x.src[ax];
              if (c < kTileSrc || c >= kSumSrc) continue;
              if (i > 0) side |= 1u << (c - kTileSrc);
              else ++n1[c - kTileSrc];
            }
          }
        int best = -1;
        for (int b = 0; b < ry - cy; ++b)
          if (!((side >> b) & 1u) && (best < 0 || n1[b] < n1[best])) best = b;
        if (best >= 0) sg.rb = static_cast<uint8_t>(best);
      }
      if (quad) {  // quad tiles only where they beat paired rows (or one row) clearly
        DevSeg& sg = hp.segs[unit_slot[u]];
        const DevStage* sts = hp.stages.data() + unit_stage[u];
        const DevTensor* tr = hp.trefs.data() + unit_tref[u];
        double alt = seg_row_score(sg, sts, tr, 0u);
        if (cy == kSegYBits && ry > cy && seg_pair_min_tiles() &&
            hp.stages[unit_stage[u]].nt <= seg_pair_max_nt() &&
            level_tiles[unit_level[u]] >= seg_pair_min_tiles()) {
          uint32_t side = 0;
          for (int i = 1; i < sg.nst; ++i)
            for (int t = 0; t < sts[i].nt; ++t)
              if (t != sts[i].main) side |= seg_tile_bits(tr[sts[i].op0 + t]);
          for (int b = 0; b < ry - cy; ++b)
            if (!((side >> b) & 1u)) alt = std::min(alt, seg_row_score(sg, sts, tr, 1u << b));
        }
        if (!(quad_score < seg_quad_margin() * alt)) {
          // undo: fall back to the paired / single choice
          sg.rb = kNoVar;
          sg.rb2 = kNoVar;
          quad = false;
          uint32_t side = 0, n1[32] = {};
          for (int i = 0; i < sg.nst; ++i)
            for (int t = 0; t < sts[i].nt; ++t) {
              if (i > 0 && t == sts[i].main) continue;
              const uint32_t b = seg_tile_bits(tr[sts[i].op0 + t]);
              for (int k = 0; k < 32; ++k)
                if ((b >> k) & 1u) {
                  if (i > 0) side |= 1u << k; else ++n1[k];
                }
            }
          if (cy == kSegYBits && ry > cy && seg_pair_min_tiles() &&
              sts[0].nt <= seg_pair_max_nt() && level_tiles[unit_level[u]] >= seg_pair_min_tiles()) {
            int best = -1;
            for (int b = 0; b < ry - cy; ++b)
              if (!((side >> b) & 1u) && (best < 0 || n1[b] < n1[best])) best = b;
            if (best >= 0) sg.rb = static_cast<uint8_t>(best);
          }
        }
      }
      unit_dev_bytes[u] = dev_bytes;
    }
  });
  ptm.mark("fill");
  // segment work items (tiles; half as many for paired segments), per level;
  // a paired tile costs about two, so re-sort each level's segments by tile
  // cost (LPT order of the dynamic tile queue) and remap unit_slot
  {
    std::vector<uint32_t> perm, slot_of(hp.segs.size());
    std::vector<DevSeg> tmp;
    auto tile_cost = [&](const DevSeg& sg) {
      return (uint64_t{1} << (sg.nst - 1)) * (sg.nops + hp.stages[sg.stage].nt) *
             (sg.rb2 != kNoVar ? 3u : sg.rb != kNoVar ? 2u : 1u);  // a quad tile costs ~3
    };
    // quad segments go last (their own kernel and tile queue), each group in
    // decreasing tile cost
    for (LevelLaunch& ll : hp.levels) {
      perm.resize(ll.seg_count);
      for (uint32_t k = 0; k < ll.seg_count; ++k) perm[k] = ll.seg_begin + k;
      std::stable_sort(perm.begin(), perm.end(), [&](uint32_t a, uint32_t b) {
        const bool qa = seg4_split() && hp.segs[a].rb2 != kNoVar;
        const bool qb = seg4_split() && hp.segs[b].rb2 != kNoVar;
        if (qa != qb) return qb;
        return tile_cost(hp.segs[a]) > tile_cost(hp.segs[b]);
      });
      uint32_t nq = 0;  // QTNG_SEG4_SPLIT=1: quad segments in their own kernel
      for (uint32_t k = 0; k < ll.seg_count && seg4_split(); ++k) nq += hp.segs[perm[k]].rb2 != kNoVar;
      ll.seg4_count = nq;
      tmp.resize(ll.seg_count);
      for (uint32_t k = 0; k < ll.seg_count; ++k) {
        tmp[k] = hp.segs[perm[k]];
        slot_of[perm[k]] = ll.seg_begin + k;
      }
      std::copy(tmp.begin(), tmp.end(), hp.segs.begin() + ll.seg_begin);
      ll.seg_count -= nq;
    }
    for (uint32_t u = 0; u < U; ++u)
      if (unit_len[u] > 1) unit_slot[u] = slot_of[unit_slot[u]];
  }
  ptm.mark("seg re-sort");
  for (LevelLaunch& ll : hp.levels) {
    ll.seg_items = 0;
    ll.seg4_items = 0;
    for (uint32_t k = ll.seg_begin; k < ll.seg_begin + ll.seg_count + ll.seg4_count; ++k) {
      DevSeg& sg = hp.segs[k];
      const uint64_t tiles = uint64_t{1} << seg_item_bits(sg);
      uint32_t& acc = k < ll.seg_begin + ll.seg_count ? ll.seg_items : ll.seg4_items;
      sg.item_begin = acc;
      hp.seg_ibeg[k] = acc;
      acc += static_cast<uint32_t>(tiles);
    }
  }
  for (int e : chunk_err) {
    if (e == 1) throw Error(kResource, "tensor rank exceeds the device limit " + std::to_string(kMaxRank));
    if (e == 2) throw Error(kSchedule, "internal: operand var outside its bucket");
    if (e == 3) throw Error(kSchedule, "internal: operand reads a fused intermediate");
  }
  ptm.mark("items");
  // accounting (statistics only), in parallel over unit chunks
  if (stats) {
    struct Acc {
      double dev = 0, alg = 0, fp = 0, segfp = 0, single = 0, sum_ops = 0;
      uint64_t fused = 0, buckets = 0;
      int max_width = 0;
      std::vector<double> level_bytes;
    };
    const int nch = std::max(1, std::min<int>(Pool::get().size() * 2, static_cast<int>(U / 256) + 1));
    std::vector<Acc> acc(nch);
    Pool::get().parallel_for(nch, [&](int ch) {
      Acc& a = acc[ch];
      a.level_bytes.assign(n_levels, 0.0);
      const uint32_t u0 = static_cast<uint32_t>(uint64_t{U} * ch / nch);
      const uint32_t u1 = static_cast<uint32_t>(uint64_t{U} * (ch + 1) / nch);
      for (uint32_t u = u0; u < u1; ++u) {
        const int L = unit_level[u];
        a.dev += unit_dev_bytes[u];
        if (unit_len[u] > 1) a.fused += unit_len[u];
        for (uint32_t g = unit_first[u]; g != ~0u; g = next_in_unit[g]) {
          const Op& o = op_at(g);
          a.level_bytes[L] += op_bytes[g];
          a.alg += op_bytes[g];
          // the reference's FP64 operations (NaiveBackend::contract): per summed
          // assignment nt-1 complex products (4 mul + 2 add/sub), per output
          // 2^ns - 1 complex additions
          const double fl = 6.0 * std::ldexp(1.0, o.width) * (o.nin - 1) +
                            2.0 * std::ldexp(1.0, o.r) * (std::ldexp(1.0, o.ns) - 1.0);
          a.fp += fl;
          if (unit_len[u] > 1) a.segfp += fl; else a.single += op_bytes[g];
          if (o.bucket_seq >= 0) {
            a.sum_ops += static_cast<double>(uint64_t{1} << o.width);
            ++a.buckets;
            a.max_width = std::max(a.max_width, static_cast<int>(o.width));
          }
        }
      }
    });
    for (const Acc& a : acc) {
      hp.dev_bytes += a.dev;
      hp.n_fused_ops += a.fused;
      hp.alg_bytes += a.alg;
      hp.fp64_ops += a.fp;
      hp.seg_fp64_ops += a.segfp;
      hp.single_alg_bytes += a.single;
      hp.sum_ops += a.sum_ops;
      hp.n_buckets += a.buckets;
      hp.max_width = std::max(hp.max_width, a.max_width);
      for (int L = 0; L < n_levels; ++L) hp.level_bytes[L] += a.level_bytes[L];
    }
  }

  if (flow) {
    hp.flow = true;
    hp.flow_units.resize(U);
    std::vector<int32_t> height(U, 0);  // units on the longest path to a sink
    for (int64_t i = static_cast<int64_t>(U) - 1; i >= 0; --i) {  // descending level
      const uint32_t u = order[static_cast<size_t>(i)];
      const int64_t cu = consumer_unit(u);
      height[u] = cu >= 0 ? height[cu] + 1 : 0;
    }
    for (uint32_t u = 0; u < U; ++u) {
      FlowUnit& f = hp.flow_units[u];
      f = FlowUnit{};
      f.kind = unit_len[u] > 1 ? 1 : 0;
      f.idx = unit_slot[u];
      if (f.kind) {
        const DevSeg& sg = hp.segs[f.idx];
        f.n_items = 1u << seg_item_bits(sg);
      } else {
        const DevOp& d = hp.ops[f.idx];
        f.n_items = 1u << (d.r - d.cb);
      }
      f.succ = static_cast<int32_t>(consumer_unit(u));
      const uint32_t c = lc_of[unit_first[u]];
      const WalkResult& w = *cones[c];
      int deps = 0;
      for (uint32_t g = unit_first[u]; g != ~0u; g = next_in_unit[g]) {
        const Op& o = op_at(g);
        const OpIn* ins = w.inputs(o);
        for (int t = 0; t < o.nin; ++t)
          if (!ins[t].initial && t != main_pos[g]) ++deps;
      }
      f.deps = static_cast<uint16_t>(deps);
      int cl = 0;
      while ((f.n_items >> cl) > kFlowMaxChunks) ++cl;
      f.chunk_log = static_cast<uint8_t>(cl);
      hp.flow_chunks += (f.n_items + (1u << cl) - 1) >> cl;
    }
    std::vector<uint32_t> init;
    for (uint32_t u = 0; u < U; ++u)
      if (hp.flow_units[u].deps == 0) init.push_back(u);
    std::stable_sort(init.begin(), init.end(),
                     [&](uint32_t a, uint32_t b) { return height[a] > height[b]; });
    for (uint32_t u : init) {
      const FlowUnit& f = hp.flow_units[u];
      const uint32_t nc = (f.n_items + (1u << f.chunk_log) - 1) >> f.chunk_log;
      for (uint32_t c = 0; c < nc; ++c) hp.flow_init.push_back((uint64_t{u} << 32) | c);
    }
  }

  ptm.mark("accounting");
  // records (one per non-empty bucket, walk order) and per-lightcone scalars:
  // offsets first, then every lightcone fills its own range in parallel
  hp.rec_begin.assign(C + 1, 0);
  hp.lc_begin.assign(C + 1, 0);
  for (int c = 0; c < C; ++c) {
    const WalkResult& w = *cones[c];
    uint32_t nrec = 0;
    if (records)
      for (const Op& o : w.ops) nrec += o.bucket_seq >= 0;
    hp.rec_begin[c + 1] = hp.rec_begin[c] + nrec;
    hp.lc_begin[c + 1] = hp.lc_begin[c] + static_cast<uint32_t>(w.scalars.size());
    hp.lc_edge.push_back(c);
  }
  const uint32_t R = hp.rec_begin[C];
  hp.rec_seq.resize(R);
  hp.rec_width.resize(R);
  hp.rec_level.resize(R);
  hp.rec_bytes.resize(R);
  hp.rec_out.resize(R);
  hp.scalar_off.resize(hp.lc_begin[C]);
  Pool::get().parallel_for(C, [&](int c) {
    const WalkResult& w = *cones[c];
    uint32_t r = hp.rec_begin[c];
    for (uint32_t k = 0; records && k < w.ops.size(); ++k) {
      const Op& o = w.ops[k];
      if (o.bucket_seq < 0) continue;
      hp.rec_seq[r] = o.bucket_seq;
      hp.rec_width[r] = o.width;
      hp.rec_level[r] = level_of(base[c] + k);
      hp.rec_bytes[r] = op_bytes[base[c] + k];
      hp.rec_out[r] = out[base[c] + k];
      ++r;
    }
    uint32_t q = hp.lc_begin[c];
    for (int sc : w.scalars) hp.scalar_off[q++] = out[base[c] + sc];
  });
  ptm.mark("records");
  return hp;
}

}  // namespace qtng
