// The data-free contract_network walk (see host.hpp), on flat arrays.
//
// Reproduces proj/src/engine.cpp:246-304 symbolically: the liveness check
// (:261-266), contract_bucket's result-width cap (:160-169), the
// present-sum-var check (:28-36), and the routing of every result to the
// bucket of its earliest remaining variable (:292-301); scalars multiply in
// production order (:288-290).  Var ids are re-indexed densely once; all
// per-bucket work then uses stamp arrays and pooled var lists, so a whole
// lightcone walks in tens of microseconds.
#include <algorithm>
#include <limits>

#include "host.hpp"

namespace qtng {

namespace {

// Dense, order-preserving re-indexing of a schedule's var ids.
struct Dense {
  bool direct = true;       // ids already in [0, n)
  int n = 0;
  std::vector<int32_t> ids;  // dense -> original (empty when direct)
  int map(int v) const {
    if (direct) return v;
    return static_cast<int>(std::lower_bound(ids.begin(), ids.end(), v) - ids.begin());
  }
};

Dense densify(const Schedule& s) {
  Dense d;
  int lo = std::numeric_limits<int>::max(), hi = -1;
  auto see = [&](int v) { lo = std::min(lo, v); hi = std::max(hi, v); };
  for (const SchedBucket& b : s.buckets)
    for (int v : b.sum_vars) see(v);
  for (const SchedTensor& t : s.init)
    for (int v : t.vars) see(v);
  if (hi < 0) return d;
  if (lo >= 0 && hi < (1 << 22)) {
    d.n = hi + 1;
    return d;
  }
  d.direct = false;
  for (const SchedBucket& b : s.buckets) d.ids.insert(d.ids.end(), b.sum_vars.begin(), b.sum_vars.end());
  for (const SchedTensor& t : s.init) d.ids.insert(d.ids.end(), t.vars.begin(), t.vars.end());
  std::sort(d.ids.begin(), d.ids.end());
  d.ids.erase(std::unique(d.ids.begin(), d.ids.end()), d.ids.end());
  d.n = static_cast<int>(d.ids.size());
  return d;
}

}  // namespace

WalkResult walk_schedule(const Schedule& s, int max_result_width, bool route) {
  WalkResult w;
  const Dense dn = densify(s);
  const int V = dn.n;
  w.n_vars = V;
  if (dn.direct) {
    w.ids.resize(V);
    for (int v = 0; v < V; ++v) w.ids[v] = v;
  } else {
    w.ids = dn.ids;
  }
  const int B = static_cast<int>(s.buckets.size());
  std::vector<int32_t> pos(V, -1);  // sum_var_positions: later buckets overwrite
  for (int i = 0; i < B; ++i)
    for (int v : s.buckets[i].sum_vars) pos[dn.map(v)] = i;

  // members: per-bucket singly linked lists in insertion order
  struct Mem {
    int64_t ref;
    int32_t var_off;
    int16_t rank;
    uint8_t initial;
    int32_t next;
  };
  std::vector<Mem> mem;
  std::vector<int32_t> head(B, -1), tail(B, -1);
  mem.reserve(s.init.size() + B);
  w.vars.reserve(s.init.size() * 2 + 64 * static_cast<size_t>(B));
  std::vector<int32_t> live(V, 0);  // uncontracted members holding each var
  auto push = [&](int b, const Mem& m) {
    const int id = static_cast<int>(mem.size());
    mem.push_back(m);
    if (tail[b] < 0) head[b] = id; else mem[tail[b]].next = id;
    tail[b] = id;
  };
  for (int i = 0; i < B; ++i)
    for (int t : s.buckets[i].tensors) {
      const SchedTensor& st = s.init[t];
      Mem m{st.data, static_cast<int32_t>(w.vars.size()), static_cast<int16_t>(st.vars.size()), 1, -1};
      for (int v : st.vars) {
        const int d = dn.map(v);
        w.vars.push_back(d);
        ++live[d];
      }
      push(i, m);
    }

  w.ops.reserve(B);
  w.ins.reserve(mem.size());
  std::vector<int32_t> stamp(V, -1), sstamp(V, -1), uni;
  uni.reserve(64);
  std::vector<int32_t> op_of_bucket(B, -1), target_of_op;
  target_of_op.reserve(B);
  for (int i = 0; i < B; ++i) {
    if (head[i] < 0) continue;
    for (int m = head[i]; m >= 0; m = mem[m].next)
      for (int a = 0; a < mem[m].rank; ++a) --live[w.vars[mem[m].var_off + a]];
    for (int v : s.buckets[i].sum_vars)
      if (live[dn.map(v)] > 0) {
        w.fail_code = kSchedule;
        w.fail_msg = "sum variable " + std::to_string(v) + " still live outside its bucket";
        return w;
      }
    uni.clear();
    for (int m = head[i]; m >= 0; m = mem[m].next)
      for (int a = 0; a < mem[m].rank; ++a) {
        const int v = w.vars[mem[m].var_off + a];
        if (stamp[v] != i) { stamp[v] = i; uni.push_back(v); }
      }
    std::sort(uni.begin(), uni.end());
    const int width = static_cast<int>(uni.size());
    const int n_sum_raw = static_cast<int>(s.buckets[i].sum_vars.size());
    if (width - n_sum_raw > max_result_width) {
      w.fail_code = kResource;
      w.fail_msg = "contraction refused: result width " + std::to_string(width - n_sum_raw) +
                   " exceeds cap " + std::to_string(max_result_width);
      return w;
    }
    Op op{};
    op.bucket_seq = i;
    op.width = width;
    op.consumer = -1;
    op.sum_off = static_cast<int32_t>(w.vars.size());
    for (int v : s.buckets[i].sum_vars) {
      const int d = dn.map(v);
      if (stamp[d] != i) {
        w.fail_code = kSchedule;
        w.fail_msg = "bucket sums a variable absent from its tensors";
        return w;
      }
      if (sstamp[d] != i) { sstamp[d] = i; w.vars.push_back(d); }
    }
    std::sort(w.vars.begin() + op.sum_off, w.vars.end());
    op.ns = static_cast<int16_t>(w.vars.size() - op.sum_off);
    op.out_off = static_cast<int32_t>(w.vars.size());
    for (int v : uni)
      if (sstamp[v] != i) w.vars.push_back(v);
    op.r = static_cast<int16_t>(w.vars.size() - op.out_off);
    op.in_off = static_cast<int32_t>(w.ins.size());
    int level = 0;
    for (int m = head[i]; m >= 0; m = mem[m].next) {
      const Mem& mm = mem[m];
      if (!mm.initial) level = std::max(level, w.ops[mm.ref].level + 1);
      w.ins.push_back(OpIn{mm.ref, mm.var_off, mm.rank, mm.initial, 0});
    }
    op.nin = static_cast<int32_t>(w.ins.size() - op.in_off);
    op.level = level;
    head[i] = -1;
    const int me = static_cast<int>(w.ops.size());
    op_of_bucket[i] = me;
    w.max_result_rank = std::max(w.max_result_rank, static_cast<int>(op.r));
    int target = -1;
    if (op.r == 0) {
      w.scalars.push_back(me);
    } else if (route) {
      target = std::numeric_limits<int>::max();
      for (int k = 0; k < op.r; ++k) {
        const int p = pos[w.vars[op.out_off + k]];
        if (p < 0) {
          w.fail_code = kSchedule;
          w.fail_msg = "result variable not covered by the schedule";
          return w;
        }
        target = std::min(target, p);
      }
      if (target <= i) {
        w.fail_code = kSchedule;
        w.fail_msg = "result tensor flows backwards in the schedule";
        return w;
      }
      for (int k = 0; k < op.r; ++k) ++live[w.vars[op.out_off + k]];
      push(target, Mem{me, op.out_off, op.r, 0, -1});
    }
    w.ops.push_back(op);
    target_of_op.push_back(target);
  }
  for (size_t k = 0; k < w.ops.size(); ++k)
    if (target_of_op[k] >= 0) w.ops[k].consumer = op_of_bucket[target_of_op[k]];
  return w;
}

void fold_wide_ops(WalkResult& w, int max_inputs) {
  bool any = false;
  for (const Op& o : w.ops) any |= o.nin > max_inputs;
  if (!any) return;
  WalkResult out;
  out.vars = w.vars;
  out.ids = w.ids;
  out.n_vars = w.n_vars;
  out.max_result_rank = w.max_result_rank;
  out.fail_code = w.fail_code;
  out.fail_msg = w.fail_msg;
  std::vector<int32_t> remap(w.ops.size(), -1);
  std::vector<int32_t> stamp(w.n_vars, -1);
  for (size_t k = 0; k < w.ops.size(); ++k) {
    const Op& o = w.ops[k];
    std::vector<OpIn> ins(w.ins.begin() + o.in_off, w.ins.begin() + o.in_off + o.nin);
    for (OpIn& in : ins)
      if (!in.initial) in.ref = remap[in.ref];
    int level = 0;
    for (const OpIn& in : ins)
      if (!in.initial) level = std::max(level, out.ops[in.ref].level + 1);
    while (static_cast<int>(ins.size()) > max_inputs) {
      Op f{};
      f.bucket_seq = -1;
      f.consumer = -1;
      f.sum_off = static_cast<int32_t>(out.vars.size());
      f.ns = 0;
      f.out_off = static_cast<int32_t>(out.vars.size());
      const int fid = static_cast<int>(out.ops.size());
      for (int t = 0; t < max_inputs; ++t)
        for (int a = 0; a < ins[t].rank; ++a) {
          const int v = out.vars[ins[t].var_off + a];
          if (stamp[v] != fid) { stamp[v] = fid; out.vars.push_back(v); }
        }
      std::sort(out.vars.begin() + f.out_off, out.vars.end());
      f.r = static_cast<int16_t>(out.vars.size() - f.out_off);
      f.width = f.r;
      f.in_off = static_cast<int32_t>(out.ins.size());
      f.nin = max_inputs;
      int flevel = 0;
      for (int t = 0; t < max_inputs; ++t) {
        if (!ins[t].initial) {
          flevel = std::max(flevel, out.ops[ins[t].ref].level + 1);
          out.ops[ins[t].ref].consumer = fid;
        }
        out.ins.push_back(ins[t]);
      }
      f.level = flevel;
      out.ops.push_back(f);
      ins.erase(ins.begin(), ins.begin() + max_inputs);
      ins.insert(ins.begin(), OpIn{fid, f.out_off, f.r, 0, 0});
      level = 0;
      for (const OpIn& in : ins)
        if (!in.initial) level = std::max(level, out.ops[in.ref].level + 1);
    }
    Op m = o;
    m.in_off = static_cast<int32_t>(out.ins.size());
    m.nin = static_cast<int32_t>(ins.size());
    m.level = level;
    m.consumer = -1;
    const int me = static_cast<int>(out.ops.size());
    for (const OpIn& in : ins) {
      if (!in.initial) out.ops[in.ref].consumer = me;
      out.ins.push_back(in);
    }
    remap[k] = me;
    out.ops.push_back(m);
  }
  for (int& s : w.scalars) s = remap[s];
  out.scalars = w.scalars;
  w = std::move(out);
}

}  // namespace qtng
