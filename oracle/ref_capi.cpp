// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (never part of the product).
//
// A thin extern "C" wrapper around the UNMODIFIED reference library
// (/root/reference/proj, compiled by oracle/Makefile into
// oracle/_ref/libqtnsim_ref.so).  It lets the Python test-suite, the golden
// generator (oracle/gen_golden.py) and bench.py's reference / cpu_baseline arm
// drive the reference's own public API:
//
//   random_regular          proj/src/graph.cpp:45-76
//   edge_schedule           proj/src/engine.cpp:493-501
//   contract_network        proj/src/engine.cpp:246-304
//   energy_expectation      proj/src/engine.cpp:503-563
//   NaiveBackend/Matmul/Mixed::contract   proj/src/engine.cpp:68-156
//   simulate_widths         proj/src/engine.cpp:235-240
//   run_ansatz/expectation_cost           proj/src/statevector.cpp:55-84
//   read_timing_csv         proj/src/engine.cpp:575-601
//
// Nothing here re-implements reference behaviour; it only marshals arrays.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <sstream>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "qtnsim/engine.hpp"
#include "qtnsim/errors.hpp"
#include "qtnsim/graph.hpp"
#include "qtnsim/statevector.hpp"

using namespace qtnsim;

namespace {

thread_local std::string g_err;

int fail(const std::exception& ex) {
  g_err = ex.what();
  if (dynamic_cast<const InvalidInputError*>(&ex)) return 1;
  if (dynamic_cast<const ResourceError*>(&ex)) return 2;
  if (dynamic_cast<const ScheduleError*>(&ex)) return 3;
  if (dynamic_cast<const NumericalError*>(&ex)) return 4;
  if (dynamic_cast<const GenerationError*>(&ex)) return 6;
  return 99;
}

Graph graph_from(int n, int m, const int* edges) {
  std::vector<Edge> es(m);
  for (int i = 0; i < m; ++i) es[i] = Edge{edges[2 * i], edges[2 * i + 1]};
  return make_graph(n, std::move(es));
}

Angles angles_from(int p, const double* g, const double* b) {
  Angles a;
  a.gammas.assign(g, g + p);
  a.betas.assign(b, b + p);
  return a;
}

// backend kind: 0 naive, 1 matmul, 2 mixed(threshold, naive, matmul),
// 3 the acceptance scale backend Mixed(26, Mixed(15, naive, matmul), naive)
// (proj/tests/acceptance.cpp:174-175).
struct BackendBox {
  NaiveBackend naive;
  MatmulBackend matmul;
  std::unique_ptr<MixedBackend> inner, outer;
  const ContractionBackend* sel = nullptr;
  BackendBox(int kind, int threshold) {
    switch (kind) {
      case 0: sel = &naive; break;
      case 1: sel = &matmul; break;
      case 2:
        inner = std::make_unique<MixedBackend>(threshold, naive, matmul);
        sel = inner.get();
        break;
      default:
        inner = std::make_unique<MixedBackend>(15, naive, matmul);
        outer = std::make_unique<MixedBackend>(26, *inner, naive);
        sel = outer.get();
        break;
    }
  }
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Edges of random_regular(n, d, seed); returns the edge count or <0.
int ref_random_regular(int n, int d, uint64_t seed, int* edges_out, int cap) {
  try {
    const Graph g = random_regular(n, d, seed);
    const int m = static_cast<int>(g.edges.size());
    if (m > cap) return -1000;
    for (int i = 0; i < m; ++i) {
      edges_out[2 * i] = g.edges[i].u;
      edges_out[2 * i + 1] = g.edges[i].v;
    }
    return m;
  } catch (const std::exception& ex) {
    return -fail(ex);
  }
}

// energy_expectation through the reference's public API. wall_s receives the
// wall-clock of that single call.
int ref_energy(int n, int m, const int* edges, int p, const double* gammas,
               const double* betas, int backend_kind, int threshold, int merged,
               int max_width, int jobs, double* energy, double* wall_s,
               uint64_t* n_records, uint64_t* peak_bytes) {
  try {
    const Graph g = graph_from(n, m, edges);
    const Angles a = angles_from(p, gammas, betas);
    BackendBox box(backend_kind, threshold);
    EngineConfig cfg;
    cfg.max_result_width = max_width;
    const auto t0 = std::chrono::steady_clock::now();
    const EnergyResult r = energy_expectation(g, a, *box.sel, merged != 0, cfg, jobs);
    *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *energy = r.energy;
    if (n_records) *n_records = r.report.records.size();
    if (peak_bytes) *peak_bytes = r.report.peak_tensor_bytes;
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// Per-edge scalar e_jk for a subset of edges (indices into the sorted edge
// list), each computed exactly like energy_expectation's run_edge
// (edge_schedule + contract_network, engine.cpp:512-529), on `jobs` threads.
int ref_edge_terms(int n, int m, const int* edges, int p, const double* gammas,
                   const double* betas, int backend_kind, int threshold, int merged,
                   int max_width, int jobs, int n_sel, const int* sel,
                   double* terms_re_im, double* wall_s) {
  try {
    const Graph g = graph_from(n, m, edges);
    const Angles a = angles_from(p, gammas, betas);
    BackendBox box(backend_kind, threshold);
    EngineConfig cfg;
    cfg.max_result_width = max_width;
    std::vector<std::string> failures(n_sel);
    auto run = [&](int i) {
      try {
        const Edge e = g.edges.at(sel[i]);
        const ContractionReport rep =
            contract_network(edge_schedule(g, e, a, merged != 0), *box.sel, cfg);
        terms_re_im[2 * i] = rep.scalar.real();
        terms_re_im[2 * i + 1] = rep.scalar.imag();
      } catch (const std::exception& ex) {
        failures[i] = ex.what();
      }
    };
    const auto t0 = std::chrono::steady_clock::now();
    if (jobs <= 1) {
      for (int i = 0; i < n_sel; ++i) run(i);
    } else {
      std::atomic<int> next{0};
      std::vector<std::thread> pool;
      for (int t = 0; t < jobs; ++t)
        pool.emplace_back([&] {
          for (int i = next.fetch_add(1); i < n_sel; i = next.fetch_add(1)) run(i);
        });
      for (auto& t : pool) t.join();
    }
    if (wall_s)
      *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int i = 0; i < n_sel; ++i)
      if (!failures[i].empty()) throw ScheduleError(failures[i]);
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// State-vector oracle energy (statevector.cpp:55-84).
int ref_statevector_energy(int n, int m, const int* edges, int p, const double* gammas,
                           const double* betas, double* energy) {
  try {
    const Graph g = graph_from(n, m, edges);
    const Angles a = angles_from(p, gammas, betas);
    *energy = expectation_cost(run_ansatz(g, a, 26), g);
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// Flattened schedule of one edge (edge_schedule, engine.cpp:493-501):
//   ints: for each bucket: n_sum, sum vars..., n_tensors, per tensor: rank, vars...
//   data: every tensor's data (re, im) in the same order.
// Returns the number of ints written (or -needed if the buffer is too small).
long ref_edge_schedule(int n, int m, const int* edges, int p, const double* gammas,
                       const double* betas, int edge_index, int merged, int* ints,
                       long int_cap, double* data, long data_cap, long* data_len,
                       int* n_buckets) {
  try {
    const Graph g = graph_from(n, m, edges);
    const Angles a = angles_from(p, gammas, betas);
    const ContractionSchedule s = edge_schedule(g, g.edges.at(edge_index), a, merged != 0);
    std::vector<int> out;
    std::vector<double> dat;
    for (const Bucket& b : s.buckets) {
      out.push_back(static_cast<int>(b.sum_vars.size()));
      out.insert(out.end(), b.sum_vars.begin(), b.sum_vars.end());
      out.push_back(static_cast<int>(b.tensors.size()));
      for (const Tensor& t : b.tensors) {
        out.push_back(t.rank());
        out.insert(out.end(), t.vars.begin(), t.vars.end());
        for (const cd& x : t.data) {
          dat.push_back(x.real());
          dat.push_back(x.imag());
        }
      }
    }
    *n_buckets = static_cast<int>(s.buckets.size());
    *data_len = static_cast<long>(dat.size());
    if (static_cast<long>(out.size()) > int_cap || static_cast<long>(dat.size()) > data_cap)
      return -static_cast<long>(std::max(out.size(), dat.size()));
    std::copy(out.begin(), out.end(), ints);
    std::copy(dat.begin(), dat.end(), data);
    return static_cast<long>(out.size());
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// merge_buckets' counters of one edge's merged schedule (engine.cpp:306-358).
int ref_merge_counts(int n, int m, const int* edges, int p, const double* gammas,
                     const double* betas, int edge_index, int* applied, int* skipped) {
  try {
    const Graph g = graph_from(n, m, edges);
    const Angles a = angles_from(p, gammas, betas);
    const ContractionSchedule s = edge_schedule(g, g.edges.at(edge_index), a, true);
    *applied = s.merges_applied;
    *skipped = s.merges_skipped;
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// simulate_widths for one edge (engine.cpp:235-240).
int ref_simulate_widths(int n, int m, const int* edges, int p, const double* gammas,
                        const double* betas, int edge_index, int merged, int* widths,
                        int cap) {
  try {
    const Graph g = graph_from(n, m, edges);
    const Angles a = angles_from(p, gammas, betas);
    const std::vector<int> w =
        simulate_widths(edge_schedule(g, g.edges.at(edge_index), a, merged != 0));
    if (static_cast<int>(w.size()) > cap) return -1000;
    std::copy(w.begin(), w.end(), widths);
    return static_cast<int>(w.size());
  } catch (const std::exception& ex) {
    return -fail(ex);
  }
}

// One bucket through a reference backend's contract() (engine.hpp:22-31).
// vars: concatenated per-tensor var lists; data: concatenated (re,im) pairs.
// Returns the result rank, writing vars/data, or <0 on error.
int ref_contract_bucket(int backend_kind, int threshold, int n_tensors, const int* ranks,
                        const int* vars, const double* data, int n_sum,
                        const int* sum_vars, int* out_vars, double* out_data,
                        long out_cap) {
  try {
    Bucket b;
    long vo = 0, dof = 0;
    for (int t = 0; t < n_tensors; ++t) {
      Tensor x;
      x.label = "in";
      x.vars.assign(vars + vo, vars + vo + ranks[t]);
      vo += ranks[t];
      const long sz = 1L << ranks[t];
      x.data.resize(sz);
      for (long i = 0; i < sz; ++i) x.data[i] = cd{data[2 * (dof + i)], data[2 * (dof + i) + 1]};
      dof += sz;
      b.tensors.push_back(std::move(x));
    }
    b.sum_vars.assign(sum_vars, sum_vars + n_sum);
    BackendBox box(backend_kind, threshold);
    const Tensor r = box.sel->contract(b);
    if (static_cast<long>(r.data.size()) > out_cap) return -1000;
    std::copy(r.vars.begin(), r.vars.end(), out_vars);
    for (std::size_t i = 0; i < r.data.size(); ++i) {
      out_data[2 * i] = r.data[i].real();
      out_data[2 * i + 1] = r.data[i].imag();
    }
    return r.rank();
  } catch (const std::exception& ex) {
    return -fail(ex);
  }
}

// contract_bucket with a width cap (engine.cpp:160-169): the refusal path.
int ref_contract_bucket_capped(int n_tensors, const int* ranks, const int* vars,
                               int n_sum, const int* sum_vars, int max_width) {
  try {
    Bucket b;
    long vo = 0;
    for (int t = 0; t < n_tensors; ++t) {
      Tensor x;
      x.vars.assign(vars + vo, vars + vo + ranks[t]);
      vo += ranks[t];
      x.data.assign(1L << ranks[t], cd{1.0, 0.0});
      b.tensors.push_back(std::move(x));
    }
    b.sum_vars.assign(sum_vars, sum_vars + n_sum);
    EngineConfig cfg;
    cfg.max_result_width = max_width;
    contract_bucket(b, NaiveBackend{}, cfg);
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// The 20 seeded (graph, angles) instances of the reference's acceptance
// criteria 1-3 (proj/tests/acceptance.cpp:42-66), regenerated with the same
// standard-library engine and distributions so their angles are bit-identical.
// Writes n, seed, p and 2p angles (gammas then betas) per instance; returns 20.
int ref_acceptance_instances(int* ns, uint64_t* seeds, int* ps, double* angles /*20*2*3*/) {
  std::vector<std::pair<int, int>> shapes;
  for (int n : {6, 8, 10, 12, 14, 16}) {
    shapes.push_back({n, 1});
    shapes.push_back({n, 2});
  }
  for (int n : {6, 8, 10, 12}) shapes.push_back({n, 3});
  for (int n : {8, 10, 12, 14}) shapes.push_back({n, 2});
  std::mt19937_64 rng(0xacce97);
  std::uniform_real_distribution<double> gamma_dist(0.0, 6.283185307179586);
  std::uniform_real_distribution<double> beta_dist(0.0, 3.141592653589793);
  std::uint64_t seed = 1000;
  int i = 0;
  for (auto [n, p] : shapes) {
    ns[i] = n;
    seeds[i] = seed++;
    ps[i] = p;
    for (int layer = 0; layer < p; ++layer) {
      angles[i * 6 + layer] = gamma_dist(rng);
      angles[i * 6 + 3 + layer] = beta_dist(rng);
    }
    ++i;
  }
  return i;
}

// read_timing_csv (proj/src/engine.cpp:575-601) on a CSV text: the number of
// records and the sums of their widths and ops, or the reference's error.
int ref_read_timing_csv(const char* text, long* n_records, long* width_sum, double* ops_sum) {
  try {
    std::istringstream in(text);
    const std::vector<TimingRecord> recs = read_timing_csv(in);
    *n_records = static_cast<long>(recs.size());
    *width_sum = 0;
    *ops_sum = 0;
    for (const TimingRecord& r : recs) {
      *width_sum += r.width;
      *ops_sum += static_cast<double>(r.ops);
    }
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

}  // extern "C"
