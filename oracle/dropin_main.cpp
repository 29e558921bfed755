// oracle/dropin_main.cpp -- TEST INFRASTRUCTURE: the drop-in proof.
//
// Runs the UNMODIFIED reference's energy_expectation / contract_network with
// the B200 backend (include/qtng_backend.hpp) plugged into its
// ContractionBackend interface, next to the reference's own NaiveBackend,
// and prints one JSON line.  Built by `make -C oracle dropin` into
// oracle/_ref/dropin_energy (needs the reference headers + objects and the
// product library); run on the GPU box by tests/test_gpu_dropin.py.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "qtng_backend.hpp"
#include "qtnsim/engine.hpp"
#include "qtnsim/errors.hpp"
#include "qtnsim/graph.hpp"

using namespace qtnsim;

// "time" mode: the reference's energy_expectation through the per-bucket
// drop-in (GpuBackend::contract -> qtng_contract_bucket, one host round trip
// per bucket), serial and with `jobs` worker threads, wall-clock each.
int time_mode(int n, unsigned long long seed, int p, int jobs) {
  Angles a;
  const double g4[] = {0.30, 0.25, 0.20, 0.15}, b4[] = {0.35, 0.30, 0.25, 0.20};
  for (int k = 0; k < p; ++k) {  // the acceptance-scale angles (acceptance.cpp:70-71)
    a.gammas.push_back(g4[k % 4]);
    a.betas.push_back(b4[k % 4]);
  }
  const Graph g = random_regular(n, 3, seed);
  qtng::GpuBackend gpu(0);
  energy_expectation(g, a, gpu, false);  // warm-up (context, arena)
  auto wall = [&](int j, double* e, size_t* nrec) {
    const auto t0 = std::chrono::steady_clock::now();
    const EnergyResult r = energy_expectation(g, a, gpu, false, {}, j);
    *e = r.energy;
    *nrec = r.report.records.size();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  double e1 = 0, ej = 0;
  size_t r1 = 0, rj = 0;
  const double t1 = wall(1, &e1, &r1), tj = wall(jobs, &ej, &rj);
  std::printf("{\"mode\": \"time\", \"n\": %d, \"seed\": %llu, \"p\": %d, \"buckets\": %zu, "
              "\"energy_jobs1\": %.17g, \"wall_s_jobs1\": %.6f, \"jobs\": %d, "
              "\"energy_jobsN\": %.17g, \"wall_s_jobsN\": %.6f}\n",
              n, seed, p, r1, e1, t1, jobs, ej, tj);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "time")
    return time_mode(argc > 2 ? std::atoi(argv[2]) : 30,
                     argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 104478ull,
                     argc > 4 ? std::atoi(argv[4]) : 4, argc > 5 ? std::atoi(argv[5]) : 16);
  const int n = argc > 1 ? std::atoi(argv[1]) : 10;
  const unsigned long long seed = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 7;
  const int p = argc > 3 ? std::atoi(argv[3]) : 1;
  Angles a;
  for (int k = 0; k < p; ++k) {
    a.gammas.push_back(0.4 - 0.05 * k);
    a.betas.push_back(0.3 - 0.03 * k);
  }
  const Graph g = random_regular(n, 3, seed);
  qtng::GpuBackend gpu(0);
  const NaiveBackend naive;
  const MixedBackend mixed(3, naive, gpu);  // width <= 3 on the CPU, wider on the B200
  const EnergyResult r_naive = energy_expectation(g, a, naive, false);
  const EnergyResult r_gpu = energy_expectation(g, a, gpu, false);
  const EnergyResult r_gpu4 = energy_expectation(g, a, gpu, false, {}, 4);
  const EnergyResult r_mixed = energy_expectation(g, a, mixed, false);
  int gpu_recs = 0, low_recs = 0, bad_dispatch = 0;
  for (const TimingRecord& rec : r_mixed.report.records) {
    const bool hi = rec.backend == "b200";
    (hi ? gpu_recs : low_recs)++;
    if (hi != (rec.width > 3)) ++bad_dispatch;
  }
  bool all_b200 = true;
  for (const TimingRecord& rec : r_gpu.report.records) all_b200 &= rec.backend == "b200";
  // cap refusal through the reference driver (engine.cpp:160-169, 543-546)
  std::string refusal;
  try {
    EngineConfig cfg;
    cfg.max_result_width = 3;
    energy_expectation(g, a, gpu, false, cfg);
  } catch (const ScheduleError& ex) {
    refusal = ex.what();
  }
  std::printf(
      "{\"n\": %d, \"seed\": %llu, \"p\": %d, \"energy_naive\": %.17g, \"energy_b200\": %.17g, "
      "\"energy_b200_jobs4\": %.17g, \"energy_mixed\": %.17g, \"records_naive\": %zu, "
      "\"records_b200\": %zu, \"all_records_b200\": %s, \"mixed_gpu_records\": %d, "
      "\"mixed_low_records\": %d, \"mixed_bad_dispatch\": %d, \"peak_naive\": %llu, "
      "\"peak_b200\": %llu, \"refusal\": \"%s\"}\n",
      n, seed, p, r_naive.energy, r_gpu.energy, r_gpu4.energy, r_mixed.energy,
      r_naive.report.records.size(), r_gpu.report.records.size(), all_b200 ? "true" : "false",
      gpu_recs, low_recs, bad_dispatch,
      static_cast<unsigned long long>(r_naive.report.peak_tensor_bytes),
      static_cast<unsigned long long>(r_gpu.report.peak_tensor_bytes), refusal.c_str());
  return 0;
}
