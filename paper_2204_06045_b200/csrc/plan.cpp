// Offline planner: turns per-lightcone symbolic walks into one level-
// synchronous device program (see plan.hpp / device_plan.hpp).
#include "plan.hpp"

#include <algorithm>
#include <map>
#include <set>

namespace qtng {

namespace {

constexpr uint64_t kAlign = 32;  // elements (512 B)

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Best-fit allocator with coalescing over arena element offsets.
class Arena {
 public:
  explicit Arena(uint64_t base) : top_(base), peak_(base) {}
  uint64_t alloc(uint64_t n) {
    auto it = by_size_.lower_bound({n, 0});
    if (it != by_size_.end()) {
      const auto [size, off] = *it;
      by_size_.erase(it);
      by_off_.erase(off);
      if (size > n) insert_free(off + n, size - n);
      return off;
    }
    // grow: absorb a free block that ends at the top
    if (!by_off_.empty()) {
      auto last = std::prev(by_off_.end());
      if (last->first + last->second == top_) {
        const uint64_t off = last->first;
        by_size_.erase({last->second, off});
        by_off_.erase(last);
        top_ = off + n;
        peak_ = std::max(peak_, top_);
        return off;
      }
    }
    const uint64_t off = top_;
    top_ += n;
    peak_ = std::max(peak_, top_);
    return off;
  }
  void release(uint64_t off, uint64_t n) {
    auto next = by_off_.lower_bound(off);
    if (next != by_off_.end() && off + n == next->first) {
      by_size_.erase({next->second, next->first});
      n += next->second;
      next = by_off_.erase(next);
    }
    if (next != by_off_.begin()) {
      auto prev = std::prev(next);
      if (prev->first + prev->second == off) {
        by_size_.erase({prev->second, prev->first});
        off = prev->first;
        n += prev->second;
        by_off_.erase(prev);
      }
    }
    insert_free(off, n);
  }
  uint64_t peak() const { return peak_; }

 private:
  void insert_free(uint64_t off, uint64_t n) {
    by_off_[off] = n;
    by_size_.insert({n, off});
  }
  uint64_t top_, peak_;
  std::map<uint64_t, uint64_t> by_off_;
  std::set<std::pair<uint64_t, uint64_t>> by_size_;
};

struct GIn {
  bool initial;
  int64_t ref;  // initial: input-region offset; else global op index
  std::vector<int> vars;
};

struct GOp {
  int lc = 0;
  bool record = true;  // false for pre-fold helpers
  int width = 0;
  std::vector<int> sum_vars, out_vars;
  std::vector<GIn> ins;
  int level = 0;
  int consumer = -1;   // global op index, -1 scalar
  uint64_t out = 0;
};

uint64_t out_alloc_size(int r) { return round_up(uint64_t{1} << r, kAlign); }

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

}  // namespace

HostPlan build_plan(const std::vector<const WalkResult*>& cones, uint64_t input_elems) {
  HostPlan hp;
  hp.input_elems = input_elems;
  std::vector<GOp> g;
  std::vector<std::vector<int>> cone_scalars(cones.size());
  hp.rec_begin.push_back(0);
  size_t total = 0;
  for (const WalkResult* w : cones) total += w->ops.size();
  g.reserve(total + total / 8);

  for (size_t c = 0; c < cones.size(); ++c) {
    const WalkResult& w = *cones[c];
    std::vector<int> gid(w.ops.size());
    for (size_t k = 0; k < w.ops.size(); ++k) {
      const Op& op = w.ops[k];
      std::vector<GIn> ins;
      ins.reserve(op.inputs.size());
      for (const OpInput& in : op.inputs)
        ins.push_back(GIn{in.initial, in.initial ? in.ref : gid[in.ref], in.vars});
      // Pre-fold wide member lists: the product of the first kMaxInputs members
      // over their joint vars, no summation.  prod = (1*P)*T8*... rounds
      // exactly like the reference's left fold ((1*T0)*T1)*...*T8*...
      while (ins.size() > static_cast<size_t>(kMaxInputs)) {
        GOp f;
        f.lc = static_cast<int>(c);
        f.record = false;
        for (int t = 0; t < kMaxInputs; ++t)
          f.out_vars.insert(f.out_vars.end(), ins[t].vars.begin(), ins[t].vars.end());
        std::sort(f.out_vars.begin(), f.out_vars.end());
        f.out_vars.erase(std::unique(f.out_vars.begin(), f.out_vars.end()), f.out_vars.end());
        f.width = static_cast<int>(f.out_vars.size());
        f.ins.assign(ins.begin(), ins.begin() + kMaxInputs);
        const int fid = static_cast<int>(g.size());
        GIn folded{false, fid, f.out_vars};
        g.push_back(std::move(f));
        ins.erase(ins.begin(), ins.begin() + kMaxInputs);
        ins.insert(ins.begin(), std::move(folded));
      }
      GOp o;
      o.lc = static_cast<int>(c);
      o.width = op.width;
      o.sum_vars = op.sum_vars;
      o.out_vars = op.out_vars;
      o.ins = std::move(ins);
      gid[k] = static_cast<int>(g.size());
      g.push_back(std::move(o));
      // records (one per non-empty bucket, schedule order)
      hp.rec_seq.push_back(op.bucket_seq);
      hp.rec_width.push_back(op.width);
    }
    for (int s : w.scalars) cone_scalars[c].push_back(gid[s]);
    hp.rec_begin.push_back(static_cast<uint32_t>(hp.rec_seq.size()));
    hp.max_result_rank = std::max(hp.max_result_rank, w.max_result_rank);
  }

  // levels + consumers
  int max_level = 0;
  for (size_t i = 0; i < g.size(); ++i) {
    int lv = 0;
    for (const GIn& in : g[i].ins)
      if (!in.initial) {
        lv = std::max(lv, g[in.ref].level + 1);
        g[in.ref].consumer = static_cast<int>(i);
      }
    g[i].level = lv;
    max_level = std::max(max_level, lv);
  }
  const int n_levels = g.empty() ? 0 : max_level + 1;

  // stable level sort
  std::vector<std::vector<int>> by_level(n_levels);
  for (size_t i = 0; i < g.size(); ++i) by_level[g[i].level].push_back(static_cast<int>(i));

  // arena placement over level lifetimes; scalars live to the end
  Arena arena(round_up(input_elems, kAlign));
  std::vector<std::vector<int>> release(n_levels + 1);
  for (int L = 0; L < n_levels; ++L) {
    if (L > 0)
      for (int i : release[L - 1]) arena.release(g[i].out, out_alloc_size(static_cast<int>(g[i].out_vars.size())));
    for (int i : by_level[L]) {
      g[i].out = arena.alloc(out_alloc_size(static_cast<int>(g[i].out_vars.size())));
      if (g[i].consumer >= 0) release[g[g[i].consumer].level].push_back(i);
    }
  }
  hp.arena_elems = arena.peak();

  // descriptors
  hp.ops.reserve(g.size());
  hp.level_bytes.assign(n_levels, 0.0);
  for (int L = 0; L < n_levels; ++L) {
    LevelLaunch ll{static_cast<uint32_t>(hp.ops.size()), 0, 0, 0};
    // item size: 32-output rows per warp item, fewer for small levels so the
    // level still spreads over the whole GPU
    uint64_t level_rows = 0;
    for (int i : by_level[L]) {
      const int r = static_cast<int>(g[i].out_vars.size());
      level_rows += r > 5 ? uint64_t{1} << (r - 5) : 1;
    }
    int row_bits = 0;
    while (row_bits < kItemBits - 5 && (level_rows >> (row_bits + 1)) >= kTargetItems) ++row_bits;
    for (int i : by_level[L]) {
      const GOp& o = g[i];
      const int r = static_cast<int>(o.out_vars.size());
      const int ns = static_cast<int>(o.sum_vars.size());
      if (ns > kMaxSumBits)
        throw Error(kInvalidInput, "bucket sums " + std::to_string(ns) +
                                       " variables; the device path supports at most " +
                                       std::to_string(kMaxSumBits));
      DevOp d{};
      d.out = o.out;
      d.item_begin = ll.items;
      d.tref = static_cast<uint32_t>(hp.trefs.size());
      d.r = static_cast<uint8_t>(r);
      d.ns = static_cast<uint8_t>(ns);
      d.nt = static_cast<uint8_t>(o.ins.size());
      d.cb = static_cast<uint8_t>(std::min(r, 5 + row_bits));
      ll.max_nt = std::max<uint32_t>(ll.max_nt, d.nt);
      const uint64_t items = uint64_t{1} << (r - d.cb);
      if (ll.items + items > 0xffffffffull) throw Error(kResource, "level has too many work items");
      ll.items += static_cast<uint32_t>(items);
      double bytes = 16.0 * static_cast<double>(uint64_t{1} << r);
      for (const GIn& in : o.ins) {
        const int rank = static_cast<int>(in.vars.size());
        if (rank > kMaxRank)
          throw Error(kResource, "tensor rank " + std::to_string(rank) +
                                     " exceeds the device limit " + std::to_string(kMaxRank));
        DevTensor t{};
        t.off = in.initial ? static_cast<uint64_t>(in.ref) : g[in.ref].out;
        t.rank = static_cast<uint8_t>(rank);
        for (int ax = 0; ax < rank; ++ax) {
          const int v = in.vars[ax];
          auto ko = std::lower_bound(o.out_vars.begin(), o.out_vars.end(), v);
          if (ko != o.out_vars.end() && *ko == v) {
            t.src[ax] = static_cast<uint8_t>(r - 1 - (ko - o.out_vars.begin()));
          } else {
            auto ks = std::lower_bound(o.sum_vars.begin(), o.sum_vars.end(), v);
            if (ks == o.sum_vars.end() || *ks != v)
              throw Error(kSchedule, "internal: operand var outside its bucket");
            t.src[ax] = static_cast<uint8_t>(kSumSrc + (ns - 1 - (ks - o.sum_vars.begin())));
          }
        }
        hp.trefs.push_back(t);
        bytes += 16.0 * static_cast<double>(uint64_t{1} << rank);
      }
      mark_invariant_lead(d, hp.trefs.data() + d.tref);
      hp.ops.push_back(d);
      hp.ibeg.push_back(d.item_begin);
      hp.op_width.push_back(o.record ? o.width : 0);
      ++ll.op_count;
      hp.level_bytes[L] += bytes;
      hp.alg_bytes += bytes;
      if (o.record) {
        hp.sum_ops += static_cast<double>(uint64_t{1} << o.width);
        ++hp.n_buckets;
        hp.max_width = std::max(hp.max_width, o.width);
      }
    }
    hp.levels.push_back(ll);
  }
  // record levels / bytes (records follow the walk order of each cone)
  hp.rec_level.reserve(hp.rec_seq.size());
  for (const GOp& o : g)
    if (o.record) {
      double bytes = 16.0 * static_cast<double>(uint64_t{1} << o.out_vars.size());
      for (const GIn& in : o.ins) bytes += 16.0 * static_cast<double>(uint64_t{1} << in.vars.size());
      hp.rec_level.push_back(o.level);
      hp.rec_bytes.push_back(bytes);
      hp.rec_out.push_back(o.out);
    }
  hp.lc_begin.push_back(0);
  for (const auto& sc : cone_scalars) {
    for (int i : sc) hp.scalar_off.push_back(g[i].out);
    hp.lc_begin.push_back(static_cast<uint32_t>(hp.scalar_off.size()));
  }
  return hp;
}

}  // namespace qtng
