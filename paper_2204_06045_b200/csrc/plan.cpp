// Offline planner: turns per-lightcone symbolic walks into one level-
// synchronous device program (see plan.hpp / device_plan.hpp).  Linear-time
// passes over flat arrays: counting sorts by level, O(1) size-class arena
// allocation, stamp-array bit maps.
#include "plan.hpp"

#include <algorithm>
#include <cstdlib>

#include "pool.hpp"

namespace qtng {

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

HostPlan build_plan(const std::vector<const WalkResult*>& cones, uint64_t input_elems) {
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
  int max_level = -1;
  for (int c = 0; c < C; ++c)
    for (uint32_t k = 0; k < cones[c]->ops.size(); ++k) {
      const Op& o = cones[c]->ops[k];
      if (o.nin > kMaxInputs) throw Error(kSchedule, "internal: op not pre-folded");
      if (o.ns > kMaxSumBits)
        throw Error(kInvalidInput, "bucket sums " + std::to_string(o.ns) +
                                       " variables; the device path supports at most " +
                                       std::to_string(kMaxSumBits));
      lc_of[base[c] + k] = c;
      max_level = std::max(max_level, static_cast<int>(o.level));
    }
  const int n_levels = max_level + 1;
  auto op_at = [&](uint32_t g) -> const Op& { return cones[lc_of[g]]->ops[g - base[lc_of[g]]]; };

  // stable counting sort by level; release lists by consumer level
  std::vector<uint32_t> lstart(n_levels + 1, 0), order(N);
  std::vector<uint32_t> rstart(n_levels + 1, 0), rel;
  std::vector<uint64_t> level_rows(n_levels, 0);
  for (uint32_t g = 0; g < N; ++g) {
    const Op& o = op_at(g);
    ++lstart[o.level + 1];
    level_rows[o.level] += o.r > 5 ? uint64_t{1} << (o.r - 5) : 1;
    if (o.consumer >= 0) ++rstart[cones[lc_of[g]]->ops[o.consumer].level + 1];
  }
  for (int L = 0; L < n_levels; ++L) {
    lstart[L + 1] += lstart[L];
    rstart[L + 1] += rstart[L];
  }
  rel.resize(rstart[n_levels]);
  {
    std::vector<uint32_t> lf(lstart.begin(), lstart.end() - 1), rf(rstart.begin(), rstart.end() - 1);
    for (uint32_t g = 0; g < N; ++g) {
      const Op& o = op_at(g);
      order[lf[o.level]++] = g;
      if (o.consumer >= 0) rel[rf[cones[lc_of[g]]->ops[o.consumer].level]++] = g;
    }
  }

  // arena placement over level lifetimes; scalars / kept results live to the end
  std::vector<uint64_t> out(N);
  ClassArena arena(round_up(input_elems, kAlign));
  auto cls_of = [&](uint32_t g) { return std::max<int>(op_at(g).r, kMinClass); };
  for (int L = 0; L < n_levels; ++L) {
    if (L > 0)
      for (uint32_t i = rstart[L - 1]; i < rstart[L]; ++i) arena.release(cls_of(rel[i]), out[rel[i]]);
    for (uint32_t i = lstart[L]; i < lstart[L + 1]; ++i) out[order[i]] = arena.alloc(cls_of(order[i]));
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
  // outer-join classification (DevOp::lead/rb), in parallel
  std::vector<uint32_t> outer_sig(N, 0);  // 0 = generic; else 1 | lead<<8 | rb0<<16 | rb1<<24
  {
    const int chunks = static_cast<int>(std::min<uint32_t>(N, 256));
    Pool::get().parallel_for(chunks, [&](int ch) {
      std::vector<uint8_t> pm(max_vars);
      std::vector<uint32_t> pm_stamp(max_vars, ~0u);
      for (uint32_t g = static_cast<uint32_t>(uint64_t{N} * ch / chunks);
           g < static_cast<uint32_t>(uint64_t{N} * (ch + 1) / chunks); ++g) {
        const Op& o = op_at(g);
        const int cb = std::min<int>(o.r, level_cb[o.level]);
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
  // generic ops first, outer-join ops last within each level (stable)
  for (int L = 0; L < n_levels; ++L)
    std::stable_partition(order.begin() + lstart[L], order.begin() + lstart[L + 1],
                          [&](uint32_t g) { return outer_sig[g] == 0; });

  // descriptors, level by level: the item/tref prefix sums sequentially ...
  hp.ops.resize(N);
  hp.ibeg.resize(N);
  hp.op_width.resize(N);
  hp.level_bytes.assign(n_levels, 0.0);
  std::vector<double> op_bytes(N);
  uint32_t n_trefs = 0;
  for (int L = 0; L < n_levels; ++L) {
    LevelLaunch ll{lstart[L], 0, 0, 0, 0, 0};
    for (uint32_t i = lstart[L]; i < lstart[L + 1]; ++i) {
      const uint32_t g = order[i];
      const Op& o = op_at(g);
      const bool outer = outer_sig[g] != 0;
      DevOp& d = hp.ops[i];
      d.out = out[g];
      d.tref = n_trefs;
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
      hp.ibeg[i] = d.item_begin;
      hp.op_width[i] = o.bucket_seq >= 0 ? o.width : 0;
      n_trefs += static_cast<uint32_t>(o.nin);
    }
    hp.levels.push_back(ll);
  }
  // ... then every operand's bit map in parallel chunks
  hp.trefs.resize(n_trefs);
  const int chunks = static_cast<int>(std::min<uint32_t>(N, 256));
  std::vector<int> chunk_err(chunks, 0);
  Pool::get().parallel_for(chunks, [&](int ch) {
    const uint32_t i0 = static_cast<uint32_t>(uint64_t{N} * ch / chunks);
    const uint32_t i1 = static_cast<uint32_t>(uint64_t{N} * (ch + 1) / chunks);
    std::vector<uint8_t> pm(max_vars);
    std::vector<uint32_t> pm_stamp(max_vars, ~0u);
    for (uint32_t i = i0; i < i1; ++i) {
      const uint32_t g = order[i];
      const WalkResult& w = *cones[lc_of[g]];
      const Op& o = op_at(g);
      const uint32_t cb0 = base[lc_of[g]];
      DevOp& d = hp.ops[i];
      const int r = o.r, ns = o.ns;
      // output var -> bit (LSB-indexed), summed var -> kSumSrc + j
      const int32_t* ov = w.out_vars(o);
      const int32_t* sv = w.sum_vars(o);
      for (int k = 0; k < r; ++k) { pm[ov[k]] = static_cast<uint8_t>(r - 1 - k); pm_stamp[ov[k]] = g; }
      for (int k = 0; k < ns; ++k) { pm[sv[k]] = static_cast<uint8_t>(kSumSrc + ns - 1 - k); pm_stamp[sv[k]] = g; }
      double bytes = 16.0 * static_cast<double>(uint64_t{1} << r);
      const OpIn* ins = w.inputs(o);
      for (int t = 0; t < o.nin; ++t) {
        const OpIn& in = ins[t];
        if (in.rank > kMaxRank) { chunk_err[ch] = 1; return; }
        DevTensor& x = hp.trefs[d.tref + t];
        x = DevTensor{};
        x.off = in.initial ? static_cast<uint64_t>(in.ref) : out[cb0 + in.ref];
        x.rank = static_cast<uint8_t>(in.rank);
        const int32_t* iv = w.in_vars(in);
        for (int ax = 0; ax < in.rank; ++ax) {
          if (pm_stamp[iv[ax]] != g) { chunk_err[ch] = 2; return; }
          x.src[ax] = pm[iv[ax]];
        }
        bytes += 16.0 * static_cast<double>(uint64_t{1} << in.rank);
      }
      mark_invariant_lead(d, hp.trefs.data() + d.tref);
      op_bytes[g] = bytes;
    }
  });
  for (int e : chunk_err) {
    if (e == 1) throw Error(kResource, "tensor rank exceeds the device limit " + std::to_string(kMaxRank));
    if (e == 2) throw Error(kSchedule, "internal: operand var outside its bucket");
  }
  for (int L = 0; L < n_levels; ++L)
    for (uint32_t i = lstart[L]; i < lstart[L + 1]; ++i) {
      const uint32_t g = order[i];
      const Op& o = op_at(g);
      hp.level_bytes[L] += op_bytes[g];
      hp.alg_bytes += op_bytes[g];
      if (o.bucket_seq >= 0) {
        hp.sum_ops += static_cast<double>(uint64_t{1} << o.width);
        ++hp.n_buckets;
        hp.max_width = std::max(hp.max_width, static_cast<int>(o.width));
      }
    }

  // records (one per non-empty bucket, walk order) and per-lightcone scalars
  hp.rec_begin.reserve(C + 1);
  hp.rec_begin.push_back(0);
  hp.lc_begin.reserve(C + 1);
  hp.lc_begin.push_back(0);
  for (int c = 0; c < C; ++c) {
    const WalkResult& w = *cones[c];
    for (uint32_t k = 0; k < w.ops.size(); ++k) {
      const Op& o = w.ops[k];
      if (o.bucket_seq < 0) continue;
      hp.rec_seq.push_back(o.bucket_seq);
      hp.rec_width.push_back(o.width);
      hp.rec_level.push_back(o.level);
      hp.rec_bytes.push_back(op_bytes[base[c] + k]);
      hp.rec_out.push_back(out[base[c] + k]);
    }
    hp.rec_begin.push_back(static_cast<uint32_t>(hp.rec_seq.size()));
    for (int s : w.scalars) hp.scalar_off.push_back(out[base[c] + s]);
    hp.lc_begin.push_back(static_cast<uint32_t>(hp.scalar_off.size()));
  }
  return hp;
}

}  // namespace qtng
