// Host-side schedule construction (see host.hpp).  Written for the B200
// path's needs: flat arrays and bitsets instead of node-based maps/sets, so
// a whole N=30 p=4 energy (45 lightcones, ~7.9k buckets) plans in
// milliseconds, while the produced schedule is identical to the reference's.
#include "host.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <complex>
#include <deque>
#include <limits>
#include <numeric>
#include <random>
#include <unordered_set>

namespace qtng {

using cd = std::complex<double>;

// ---------------------------------------------------------------- graph

Graph make_graph(int n, std::vector<Edge> edges) {
  if (n < 0) throw Error(kInvalidInput, "vertex count must be non-negative");
  for (Edge& e : edges) {
    if (e.u > e.v) std::swap(e.u, e.v);
    if (e.u == e.v) throw Error(kInvalidInput, "self-loop at vertex " + std::to_string(e.u));
    if (e.u < 0 || e.v >= n)
      throw Error(kInvalidInput, "edge endpoint out of range: (" + std::to_string(e.u) + ", " +
                                     std::to_string(e.v) + ")");
  }
  std::sort(edges.begin(), edges.end(),
            [](const Edge& a, const Edge& b) { return a.u != b.u ? a.u < b.u : a.v < b.v; });
  for (size_t i = 1; i < edges.size(); ++i)
    if (edges[i].u == edges[i - 1].u && edges[i].v == edges[i - 1].v)
      throw Error(kInvalidInput, "duplicate edge");
  return Graph{n, std::move(edges)};
}

Graph random_regular(int n, int d, uint64_t seed) {
  if (d >= n) throw Error(kInvalidInput, "degree must be smaller than vertex count");
  if (d < 0 || n <= 0) throw Error(kInvalidInput, "n and d must be positive");
  if ((static_cast<long long>(n) * d) % 2 != 0)
    throw Error(kInvalidInput, "n*d must be even for a d-regular graph");
  // The graph is a function of the exact mt19937_64 -> std::shuffle stream,
  // and the stub array is re-shuffled in place on every restart.
  std::mt19937_64 rng(seed);
  std::vector<int> stubs(static_cast<size_t>(n) * d);
  for (int v = 0; v < n; ++v)
    for (int k = 0; k < d; ++k) stubs[static_cast<size_t>(v) * d + k] = v;
  const bool dense = n <= 4096;
  std::vector<uint8_t> seen_dense;
  std::unordered_set<uint64_t> seen_sparse;
  for (int attempt = 0; attempt < 10000; ++attempt) {
    std::shuffle(stubs.begin(), stubs.end(), rng);
    std::vector<Edge> edges;
    edges.reserve(stubs.size() / 2);
    if (dense) seen_dense.assign(static_cast<size_t>(n) * n, 0);
    else seen_sparse.clear();
    bool ok = true;
    for (size_t i = 0; i + 1 < stubs.size(); i += 2) {
      int u = stubs[i], v = stubs[i + 1];
      if (u == v) { ok = false; break; }
      if (u > v) std::swap(u, v);
      const uint64_t key = static_cast<uint64_t>(u) * n + v;
      bool fresh;
      if (dense) {
        fresh = !seen_dense[key];
        seen_dense[key] = 1;
      } else {
        fresh = seen_sparse.insert(key).second;
      }
      if (!fresh) { ok = false; break; }
      edges.push_back(Edge{u, v});
    }
    if (ok) return make_graph(n, std::move(edges));
  }
  throw Error(kGeneration, "random_regular: no simple pairing found in 10000 restarts");
}

static bool has_edge(const Graph& g, Edge e) {
  return std::binary_search(g.edges.begin(), g.edges.end(), e, [](const Edge& a, const Edge& b) {
    return a.u != b.u ? a.u < b.u : a.v < b.v;
  });
}

Lightcone lightcone(const Graph& g, Edge e, int p) {
  if (e.u > e.v) std::swap(e.u, e.v);
  if (!has_edge(g, e)) throw Error(kInvalidInput, "lightcone: edge not in graph");
  if (p < 1) throw Error(kInvalidInput, "lightcone: depth must be >= 1");
  // CSR adjacency + BFS ball of radius p-1 around the edge endpoints.
  std::vector<int> deg(g.n + 1, 0);
  for (const Edge& x : g.edges) { ++deg[x.u + 1]; ++deg[x.v + 1]; }
  for (int i = 0; i < g.n; ++i) deg[i + 1] += deg[i];
  std::vector<int> nb(deg[g.n]);
  std::vector<int> fill(deg.begin(), deg.end() - 1);
  for (const Edge& x : g.edges) { nb[fill[x.u]++] = x.v; nb[fill[x.v]++] = x.u; }
  std::vector<int> dist(g.n, -1);
  std::vector<int> queue{e.u, e.v};
  dist[e.u] = dist[e.v] = 0;
  for (size_t h = 0; h < queue.size(); ++h) {
    const int v = queue[h];
    if (dist[v] == p - 1) continue;
    for (int k = deg[v]; k < deg[v + 1]; ++k)
      if (dist[nb[k]] < 0) { dist[nb[k]] = dist[v] + 1; queue.push_back(nb[k]); }
  }
  std::vector<char> keep(g.n, 0);
  std::vector<Edge> kept;
  for (const Edge& x : g.edges)
    if (dist[x.u] >= 0 || dist[x.v] >= 0) { kept.push_back(x); keep[x.u] = keep[x.v] = 1; }
  Lightcone lc;
  std::vector<int> old_to_new(g.n, -1);
  for (int v = 0; v < g.n; ++v)
    if (keep[v]) { old_to_new[v] = static_cast<int>(lc.new_to_old.size()); lc.new_to_old.push_back(v); }
  for (Edge& x : kept) x = Edge{old_to_new[x.u], old_to_new[x.v]};
  lc.sub = make_graph(static_cast<int>(lc.new_to_old.size()), std::move(kept));
  lc.target = Edge{old_to_new[e.u], old_to_new[e.v]};
  if (lc.target.u > lc.target.v) std::swap(lc.target.u, lc.target.v);
  return lc;
}

// ---------------------------------------------------------------- gates

void fill_gate_table(int p, const double* gammas, const double* betas, double* out) {
  std::fill(out, out + 2 * kSlotElems * n_gate_slots(p), 0.0);
  auto put = [out](int slot, std::initializer_list<cd> vals) {
    int i = 0;
    for (const cd& v : vals) {
      out[2 * (slot * kSlotElems + i)] = v.real();
      out[2 * (slot * kSlotElems + i) + 1] = v.imag();
      ++i;
    }
  };
  const double r = 1.0 / std::sqrt(2.0);
  put(kSlotPlus, {cd{r, 0.0}, cd{r, 0.0}});
  put(kSlotZZ, {cd{1.0, 0.0}, cd{-1.0, 0.0}, cd{-1.0, 0.0}, cd{1.0, 0.0}});
  for (int k = 0; k < p; ++k) {
    const cd w = std::exp(cd{0.0, -gammas[k]});
    put(slot_phase(k), {cd{1.0, 0.0}, w, w, cd{1.0, 0.0}});
    put(slot_conj_phase(k), {std::conj(cd{1.0, 0.0}), std::conj(w), std::conj(w),
                             std::conj(cd{1.0, 0.0})});
    const double c = std::cos(betas[k]), s = std::sin(betas[k]);
    const cd m0{c, 0.0}, m1{0.0, -s};
    put(slot_mixer(k), {m0, m1, m1, m0});
    put(slot_conj_mixer(k), {std::conj(m0), std::conj(m1), std::conj(m1), std::conj(m0)});
  }
}

// ---------------------------------------------------------------- network

Network expectation_network(const Lightcone& lc, int p) {
  const Graph& g = lc.sub;
  Network net;
  std::vector<int> wire(g.n, -1);
  auto add = [&net](int slot, int rank, int a, int b) {
    InitTensor t;
    t.slot = slot;
    t.rank = rank;
    t.vars[0] = a;
    t.vars[1] = b;
    net.tensors.push_back(t);
  };
  // forward ansatz (build_ansatz, circuit.cpp:76-89)
  for (int q = 0; q < g.n; ++q) { wire[q] = net.n_vars++; add(kSlotPlus, 1, wire[q], 0); }
  for (int k = 0; k < p; ++k) {
    for (const Edge& e : g.edges) add(slot_phase(k), 2, wire[e.u], wire[e.v]);
    for (int q = 0; q < g.n; ++q) {
      const int out = net.n_vars++;
      add(slot_mixer(k), 2, out, wire[q]);  // axis order (out, in)
      wire[q] = out;
    }
  }
  add(kSlotZZ, 2, wire[lc.target.u], wire[lc.target.v]);
  // the forward gates in reverse order, conjugated (circuit.cpp:106-117)
  for (int k = p - 1; k >= 0; --k) {
    for (int q = g.n - 1; q >= 0; --q) {
      const int out = net.n_vars++;
      add(slot_conj_mixer(k), 2, out, wire[q]);
      wire[q] = out;
    }
    for (int i = static_cast<int>(g.edges.size()) - 1; i >= 0; --i)
      add(slot_conj_phase(k), 2, wire[g.edges[i].u], wire[g.edges[i].v]);
  }
  for (int q = g.n - 1; q >= 0; --q) add(kSlotPlus, 1, wire[q], 0);  // BraPlus
  return net;
}

// ---------------------------------------------------------------- ordering

std::vector<int> greedy_order(const Network& net) {
  const int V = net.n_vars;
  const int W = (V + 63) / 64;
  std::vector<uint64_t> adj(static_cast<size_t>(V) * W, 0);
  auto row = [&](int v) { return adj.data() + static_cast<size_t>(v) * W; };
  auto set = [&](int a, int b) { row(a)[b >> 6] |= uint64_t{1} << (b & 63); };
  for (const InitTensor& t : net.tensors)
    for (int i = 0; i < t.rank; ++i)
      for (int j = i + 1; j < t.rank; ++j) { set(t.vars[i], t.vars[j]); set(t.vars[j], t.vars[i]); }
  // Alive vertices bucketed by degree, one bitset per degree: the next
  // vertex is the lowest set bit of the lowest non-empty degree bucket, i.e.
  // minimum degree with ties to the smallest id, as the reference's std::map
  // scan picks it.
  std::vector<int> deg(V);
  std::vector<uint64_t> by_deg(static_cast<size_t>(V + 1) * W, 0);
  auto bucket = [&](int d) { return by_deg.data() + static_cast<size_t>(d) * W; };
  auto flip = [&](int d, int v) { bucket(d)[v >> 6] ^= uint64_t{1} << (v & 63); };
  for (int v = 0; v < V; ++v) {
    int c = 0;
    for (int w = 0; w < W; ++w) c += std::popcount(row(v)[w]);
    deg[v] = c;
    flip(c, v);
  }
  std::vector<uint64_t> nbrs(W);
  std::vector<int> order;
  order.reserve(V);
  for (int step = 0; step < V; ++step) {
    int best = -1;
    for (int d = 0; d <= V && best < 0; ++d) {
      const uint64_t* b = bucket(d);
      for (int w = 0; w < W; ++w)
        if (b[w]) { best = w * 64 + std::countr_zero(b[w]); break; }
    }
    order.push_back(best);
    flip(deg[best], best);
    std::copy(row(best), row(best) + W, nbrs.begin());
    for (int w = 0; w < W; ++w)
      for (uint64_t bits = nbrs[w]; bits; bits &= bits - 1) {
        const int a = w * 64 + std::countr_zero(bits);
        uint64_t* ra = row(a);
        int c = 0;
        for (int x = 0; x < W; ++x) ra[x] |= nbrs[x];
        ra[a >> 6] &= ~(uint64_t{1} << (a & 63));
        ra[best >> 6] &= ~(uint64_t{1} << (best & 63));
        for (int x = 0; x < W; ++x) c += std::popcount(ra[x]);
        if (c != deg[a]) {
          flip(deg[a], a);
          flip(c, a);
          deg[a] = c;
        }
      }
  }
  return order;
}

// ---------------------------------------------------------------- schedule

Schedule assign_buckets(const Network& net, const std::vector<int>& order) {
  std::vector<int> pos(net.n_vars, -1);
  for (size_t i = 0; i < order.size(); ++i) pos[order[i]] = static_cast<int>(i);
  Schedule s;
  s.buckets.resize(order.size());
  for (size_t i = 0; i < order.size(); ++i) s.buckets[i].sum_vars = {order[i]};
  s.init.reserve(net.tensors.size());
  for (const InitTensor& t : net.tensors) {
    if (t.rank == 0) continue;
    int earliest = std::numeric_limits<int>::max();
    for (int a = 0; a < t.rank; ++a) {
      const int p = (t.vars[a] >= 0 && t.vars[a] < net.n_vars) ? pos[t.vars[a]] : -1;
      if (p < 0)
        throw Error(kInvalidInput, "assign_buckets: variable " + std::to_string(t.vars[a]) +
                                       " missing from elimination order");
      earliest = std::min(earliest, p);
    }
    SchedTensor st;
    st.vars.assign(t.vars, t.vars + t.rank);
    st.data = static_cast<int64_t>(t.slot) * kSlotElems;
    s.buckets[earliest].tensors.push_back(static_cast<int>(s.init.size()));
    s.init.push_back(std::move(st));
  }
  return s;
}

Schedule edge_schedule(const Graph& g, Edge e, int p) {
  const Lightcone lc = lightcone(g, e, p);
  const Network net = expectation_network(lc, p);
  return assign_buckets(net, greedy_order(net));
}

// ---------------------------------------------------------------- symbolic walk
// walk_schedule / fold_wide_ops: walk.cpp

std::vector<int> simulate_widths(const Schedule& s) {
  const WalkResult w = walk_schedule(s, std::numeric_limits<int>::max());
  if (w.fail_code) throw Error(kSchedule, "invalid schedule in width simulation");
  std::vector<int> out;
  out.reserve(w.ops.size());
  for (const Op& op : w.ops) out.push_back(op.width);
  return out;
}

// ---------------------------------------------------------------- merge

namespace {

std::vector<int> bucket_vars(const Schedule& s, const SchedBucket& b) {
  std::vector<int> u;
  for (int t : b.tensors) u.insert(u.end(), s.init[t].vars.begin(), s.init[t].vars.end());
  std::sort(u.begin(), u.end());
  u.erase(std::unique(u.begin(), u.end()), u.end());
  return u;
}

int max_width_or_invalid(const Schedule& s) {
  const WalkResult w = walk_schedule(s, std::numeric_limits<int>::max());
  if (w.fail_code) return -1;
  int m = 0;
  for (const Op& op : w.ops) m = std::max(m, op.width);
  return m;
}

}  // namespace

Schedule merge_buckets(const Schedule& schedule) {
  Schedule sched = schedule;
  const int budget = max_width_or_invalid(sched);
  if (budget < 0) throw Error(kSchedule, "invalid schedule in width simulation");
  size_t i = 0;
  while (i < sched.buckets.size()) {
    const SchedBucket& a = sched.buckets[i];
    if (a.tensors.empty()) { ++i; continue; }
    const std::vector<int> uniq_a = bucket_vars(sched, a);
    std::vector<int> sum_a = a.sum_vars;
    std::sort(sum_a.begin(), sum_a.end());
    std::vector<int> need_a;
    std::set_difference(uniq_a.begin(), uniq_a.end(), sum_a.begin(), sum_a.end(),
                        std::back_inserter(need_a));
    bool merged = false;
    for (size_t j = i + 1; j < sched.buckets.size(); ++j) {
      const SchedBucket& b = sched.buckets[j];
      if (b.tensors.empty()) continue;
      const std::vector<int> uniq_b = bucket_vars(sched, b);
      if (!std::includes(uniq_b.begin(), uniq_b.end(), need_a.begin(), need_a.end())) continue;
      Schedule trial = sched;
      SchedBucket& tb = trial.buckets[j];
      tb.tensors.insert(tb.tensors.end(), sched.buckets[i].tensors.begin(),
                        sched.buckets[i].tensors.end());
      tb.sum_vars.insert(tb.sum_vars.end(), sched.buckets[i].sum_vars.begin(),
                         sched.buckets[i].sum_vars.end());
      std::sort(tb.sum_vars.begin(), tb.sum_vars.end());
      trial.buckets.erase(trial.buckets.begin() + static_cast<long>(i));
      const int mw = max_width_or_invalid(trial);
      if (mw >= 0 && mw <= budget) {
        trial.merges_applied = sched.merges_applied + 1;
        trial.merges_skipped = sched.merges_skipped;
        sched = std::move(trial);
        merged = true;
        break;
      }
      ++sched.merges_skipped;
    }
    if (!merged) ++i;
  }
  return sched;
}

// ---------------------------------------------------------------- flat format

void flatten_schedule(const Schedule& s, const double* input_region, std::vector<int>& ints,
                      std::vector<double>& data) {
  ints.clear();
  data.clear();
  for (const SchedBucket& b : s.buckets) {
    ints.push_back(static_cast<int>(b.sum_vars.size()));
    ints.insert(ints.end(), b.sum_vars.begin(), b.sum_vars.end());
    ints.push_back(static_cast<int>(b.tensors.size()));
    for (int t : b.tensors) {
      const SchedTensor& st = s.init[t];
      ints.push_back(static_cast<int>(st.vars.size()));
      ints.insert(ints.end(), st.vars.begin(), st.vars.end());
      if (input_region) {
        const int64_t n = int64_t{1} << st.vars.size();
        data.insert(data.end(), input_region + 2 * st.data, input_region + 2 * (st.data + n));
      }
    }
  }
}

Schedule parse_schedule(int n_buckets, const int* ints, long n_ints) {
  Schedule s;
  long ip = 0;
  int64_t dof = 0;
  auto next = [&]() {
    if (ip >= n_ints) throw Error(kInvalidInput, "schedule: truncated description");
    return ints[ip++];
  };
  s.buckets.resize(n_buckets < 0 ? 0 : n_buckets);
  for (int i = 0; i < n_buckets; ++i) {
    const int ns = next();
    if (ns < 0) throw Error(kInvalidInput, "schedule: negative sum count");
    for (int k = 0; k < ns; ++k) s.buckets[i].sum_vars.push_back(next());
    const int nt = next();
    if (nt < 0) throw Error(kInvalidInput, "schedule: negative tensor count");
    for (int t = 0; t < nt; ++t) {
      const int r = next();
      if (r < 0 || r > 40) throw Error(kInvalidInput, "schedule: tensor rank out of range");
      SchedTensor st;
      for (int a = 0; a < r; ++a) st.vars.push_back(next());
      st.data = dof;
      dof += int64_t{1} << r;
      s.buckets[i].tensors.push_back(static_cast<int>(s.init.size()));
      s.init.push_back(std::move(st));
    }
  }
  return s;
}

}  // namespace qtng
