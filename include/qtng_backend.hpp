// qtng_backend.hpp -- drop-in qtnsim::ContractionBackend on the B200.
//
// Header-only adaptor a maintainer of the reference (/root/reference/proj)
// compiles together with its headers: it implements the virtual interface of
// proj/include/qtnsim/engine.hpp:22-31 on top of the C ABI in qtng.h, so the
// reference's own contract_bucket / contract_network / energy_expectation /
// MixedBackend / calibrate run unchanged with the contraction on the GPU.
//
//   #include "qtnsim/engine.hpp"
//   #include "qtng_backend.hpp"
//   qtng::GpuBackend gpu(/*device=*/0);
//   auto r = qtnsim::energy_expectation(g, angles, gpu, false, cfg, jobs);
//
// Semantics kept from the interface contract:
//   * name() is "b200" and appears in every TimingRecord of buckets it ran
//     (engine.cpp:269,278);
//   * contract() returns the result with ascending var ids, MSB-first layout,
//     bit-identical to NaiveBackend::contract (engine.cpp:68-108);
//   * a sum var absent from the bucket throws qtnsim::ScheduleError with the
//     reference's message (engine.cpp:28-36); other failures map onto the
//     reference's exception types;
//   * const and thread-safe: every calling thread gets its own device context
//     (stream, arena, staging) from a pool owned by the backend, so the
//     reference's `jobs` worker threads contract their buckets concurrently
//     (engine.cpp:531-541; "usable from multiple workers").
#pragma once

#include <algorithm>
#include <atomic>
#include <complex>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "qtng.h"
#include "qtnsim/engine.hpp"
#include "qtnsim/errors.hpp"

namespace qtng {

class GpuBackend final : public qtnsim::ContractionBackend {
 public:
  explicit GpuBackend(int device = 0, uint64_t arena_bytes = 0)
      : device_(device), arena_bytes_(arena_bytes), id_(next_id()) {
    ctx_for_thread();  // fail at construction if the device is unusable
  }
  ~GpuBackend() override {
    for (qtng_ctx* c : pool_) qtng_destroy(c);
  }
  GpuBackend(const GpuBackend&) = delete;
  GpuBackend& operator=(const GpuBackend&) = delete;

  std::string name() const override { return "b200"; }

  qtnsim::Tensor contract(const qtnsim::Bucket& b) const override {
    std::vector<int> ranks, vars;
    std::vector<double> data;
    std::vector<int> uniq;
    for (const qtnsim::Tensor& t : b.tensors) {
      ranks.push_back(t.rank());
      vars.insert(vars.end(), t.vars.begin(), t.vars.end());
      const double* p = reinterpret_cast<const double*>(t.data.data());
      data.insert(data.end(), p, p + 2 * t.data.size());
    }
    uniq = vars;
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    const int64_t cap = int64_t{1} << uniq.size();
    qtnsim::Tensor out;
    out.label = "bucket_result";
    out.vars.resize(uniq.size());
    out.data.resize(static_cast<size_t>(cap));
    int rank = 0;
    const qtng_status st = qtng_contract_bucket(
        ctx_for_thread(), static_cast<int>(b.tensors.size()), ranks.data(), vars.data(), data.data(),
        static_cast<int>(b.sum_vars.size()), b.sum_vars.data(), &rank, out.vars.data(),
        reinterpret_cast<double*>(out.data.data()), cap);
    if (st != QTNG_OK) raise(st);
    out.vars.resize(rank);
    out.data.resize(size_t{1} << rank);
    return out;
  }

 private:
  [[noreturn]] static void raise(qtng_status st) {
    const std::string msg = qtng_last_error();
    switch (st) {
      case QTNG_ERR_INVALID_INPUT: throw qtnsim::InvalidInputError(msg);
      case QTNG_ERR_RESOURCE: throw qtnsim::ResourceError(msg);
      case QTNG_ERR_SCHEDULE: throw qtnsim::ScheduleError(msg);
      case QTNG_ERR_NUMERICAL: throw qtnsim::NumericalError(msg);
      case QTNG_ERR_GENERATION: throw qtnsim::GenerationError(msg);
      default: throw std::runtime_error(msg);
    }
  }
  static uint64_t next_id() {
    static std::atomic<uint64_t> n{0};
    return ++n;
  }
  // The calling thread's context (created on its first bucket).  Keyed by a
  // per-backend id, not the address, so a later backend at the same address
  // never sees a stale entry.
  qtng_ctx* ctx_for_thread() const {
    thread_local std::unordered_map<uint64_t, qtng_ctx*> mine;
    const auto it = mine.find(id_);
    if (it != mine.end()) return it->second;
    qtng_ctx* c = nullptr;
    if (qtng_create(device_, arena_bytes_, &c) != QTNG_OK)
      throw std::runtime_error(std::string("qtng_create: ") + qtng_last_error());
    {
      std::lock_guard<std::mutex> lk(pool_mu_);
      pool_.push_back(c);
    }
    mine[id_] = c;
    return c;
  }
  int device_;
  uint64_t arena_bytes_;
  uint64_t id_;
  mutable std::mutex pool_mu_;
  mutable std::vector<qtng_ctx*> pool_;
};

}  // namespace qtng
