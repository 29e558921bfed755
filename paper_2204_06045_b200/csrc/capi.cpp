// C ABI (include/qtng.h): contexts, plans, and the orchestration of the
// level-batched device program.
#include "qtng.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <complex>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "host.hpp"
#include "kernels.cuh"
#include "plan.hpp"
#include "pool.hpp"
#include "sv.cuh"

namespace qtng {
cudaError_t fp64_peak(int device, double* mul_add_ops_per_s, double* fma_flops_per_s);  // peak.cu
}

using namespace qtng;

namespace {

thread_local std::string g_err;

#define QTNG_CUDA(call)                                                                  \
  do {                                                                                   \
    const cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                               \
      throw Error(kCuda, std::string(#call) + ": " + cudaGetErrorString(e_));            \
  } while (0)

// Kernel launches issued by the library (eager launches as they are
// enqueued, graph replays as kernels-per-graph x replays): the evidence
// behind bench.py's gpu_launches.
std::atomic<uint64_t> g_launches{0};

// QTNG_TIMING=1: host phase times of the one-shot calls on stderr (tuning aid).
struct PhaseTimer {
  const char* name;
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit PhaseTimer(const char* n) : name(n) {
    static const bool enabled = [] {
      const char* v = std::getenv("QTNG_TIMING");
      return v && v[0] == '1';
    }();
    on = enabled;
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* phase) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "%s %s %.3f ms\n", name, phase,
                 std::chrono::duration<double>(now - t).count() * 1e3);
    t = now;
  }
};

template <class F>
qtng_status guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return QTNG_OK;
  } catch (const Error& ex) {
    g_err = ex.what();
    return static_cast<qtng_status>(ex.code);
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return QTNG_ERR_RESOURCE;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return QTNG_ERR_INVALID_INPUT;
  }
}

// Growable device / pinned-host buffers.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void ensure(size_t n) {
    if (n <= cap) return;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    QTNG_CUDA(cudaMalloc(&p, n));
    cap = n;
  }
  ~DevBuf() { if (p) cudaFree(p); }
};

struct PinBuf {
  void* p = nullptr;
  size_t cap = 0;
  void ensure(size_t n) {
    if (n <= cap) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    QTNG_CUDA(cudaHostAlloc(&p, n, cudaHostAllocDefault));
    cap = n;
  }
  ~PinBuf() { if (p) cudaFreeHost(p); }
};

Graph graph_from(int n, int m, const int* edges) {
  if (m < 0 || (m > 0 && !edges)) throw Error(kInvalidInput, "edge list missing");
  std::vector<Edge> es(m);
  for (int i = 0; i < m; ++i) es[i] = Edge{edges[2 * i], edges[2 * i + 1]};
  return make_graph(n, std::move(es));
}

void validate_angles(int p, const double* g, const double* b) {
  // Angles::validate (proj/src/circuit.cpp:9-16)
  if (p < 1 || !g || !b)
    throw Error(kInvalidInput, "angles: gammas and betas must have equal length p >= 1");
  for (int k = 0; k < p; ++k)
    if (!std::isfinite(g[k])) throw Error(kInvalidInput, "angles: non-finite gamma");
  for (int k = 0; k < p; ++k)
    if (!std::isfinite(b[k])) throw Error(kInvalidInput, "angles: non-finite beta");
}

std::vector<int> selection(int m, int n_sel, const int* sel) {
  std::vector<int> s;
  if (!sel) {
    s.resize(m);
    for (int i = 0; i < m; ++i) s[i] = i;
    return s;
  }
  s.assign(sel, sel + n_sel);
  for (int i : s)
    if (i < 0 || i >= m) throw Error(kInvalidInput, "edge index out of range");
  return s;
}

// The walk the device program is built from: contract_network's symbolic
// walk with >kMaxInputs-member buckets pre-folded.
WalkResult device_walk(const Schedule& s, int max_width, bool route = true) {
  WalkResult w = walk_schedule(s, max_width, route);
  if (!w.fail_code) fold_wide_ops(w, kMaxInputs);
  return w;
}

// Schedules + symbolic walks of the selected edges, built on host threads
// (every lightcone is independent, like the reference's edge pool).
struct ConeSet {
  std::vector<WalkResult> walks;
  std::vector<Edge> edges;
  std::vector<int> merges_applied, merges_skipped;  // per lightcone (merge_buckets)
};

ConeSet plan_cones(const Graph& g, int p, bool merged, int max_width, const std::vector<int>& sel) {
  ConeSet cs;
  const int k = static_cast<int>(sel.size());
  cs.walks.resize(k);
  cs.edges.resize(k);
  cs.merges_applied.assign(k, 0);
  cs.merges_skipped.assign(k, 0);
  std::vector<std::string> errs(k);
  std::vector<int> codes(k, 0);
  auto work = [&](int i) {
    try {
      const Edge e = g.edges[sel[i]];
      cs.edges[i] = e;
      Schedule s = edge_schedule(g, e, p);
      if (merged) s = merge_buckets(s);
      cs.merges_applied[i] = s.merges_applied;
      cs.merges_skipped[i] = s.merges_skipped;
      cs.walks[i] = device_walk(s, max_width);
    } catch (const Error& ex) {
      codes[i] = ex.code;
      errs[i] = ex.what();
    } catch (const std::bad_alloc&) {  // a worker thread must not terminate the process
      codes[i] = kResource;
      errs[i] = "host allocation failed";
    } catch (const std::exception& ex) {
      codes[i] = kInvalidInput;
      errs[i] = ex.what();
    }
  };
  Pool::get().parallel_for(k, work);
  for (int i = 0; i < k; ++i)
    if (codes[i]) throw Error(codes[i], errs[i]);
  return cs;
}

// Descriptor image of a HostPlan: one contiguous blob, 256-byte aligned sections.
struct DescLayout {
  size_t ops = 0, ibeg = 0, trefs = 0, segs = 0, seg_ibeg = 0, stages = 0, ctr = 0, scal = 0,
         lcb = 0, lce = 0, terms = 0, funits = 0, finit = 0, upload = 0, segtab = 0, fdone = 0, fdeps = 0,
         fqueue = 0, fstate = 0, total = 0;
};

size_t align256(size_t x) { return (x + 255) & ~size_t{255}; }

DescLayout layout_of(const HostPlan& hp) {
  DescLayout L;
  size_t o = 0;
  L.ops = o; o = align256(o + hp.ops.size() * sizeof(DevOp));
  L.ibeg = o; o = align256(o + hp.ibeg.size() * sizeof(uint32_t));
  L.trefs = o; o = align256(o + hp.trefs.size() * sizeof(DevTensor));
  L.segs = o; o = align256(o + hp.segs.size() * sizeof(DevSeg));
  L.seg_ibeg = o; o = align256(o + hp.seg_ibeg.size() * sizeof(uint32_t));
  L.stages = o; o = align256(o + hp.stages.size() * sizeof(DevStage));
  L.ctr = o; o = align256(o + hp.levels.size() * 4 * sizeof(uint32_t));
  L.scal = o; o = align256(o + hp.scalar_off.size() * sizeof(uint64_t));
  L.lcb = o; o = align256(o + hp.lc_begin.size() * sizeof(uint32_t));
  L.lce = o; o = align256(o + hp.lc_edge.size() * sizeof(int32_t));
  L.terms = o; o = align256(o + (hp.lc_begin.size()) * sizeof(double2));
  L.funits = o; o = align256(o + hp.flow_units.size() * sizeof(FlowUnit));
  L.finit = o; o = align256(o + hp.flow_init.size() * sizeof(uint64_t));
  L.upload = o;  // device-only sections follow
  L.segtab = o; o = align256(o + (hp.segs.empty() ? 0 : hp.trefs.size() * sizeof(SegOpTab)));
  const size_t nu = hp.flow_units.size();
  L.fdone = o; o = align256(o + nu * sizeof(uint32_t));
  L.fdeps = o; o = align256(o + nu * sizeof(int32_t));
  L.fqueue = o; o = align256(o + hp.flow_chunks * sizeof(uint64_t));
  L.fstate = o; o = align256(o + sizeof(FlowState));
  L.total = o;
  return L;
}

void pack_desc(const HostPlan& hp, const DescLayout& L, char* dst) {
  std::memcpy(dst + L.ops, hp.ops.data(), hp.ops.size() * sizeof(DevOp));
  std::memcpy(dst + L.ibeg, hp.ibeg.data(), hp.ibeg.size() * sizeof(uint32_t));
  std::memcpy(dst + L.trefs, hp.trefs.data(), hp.trefs.size() * sizeof(DevTensor));
  std::memcpy(dst + L.segs, hp.segs.data(), hp.segs.size() * sizeof(DevSeg));
  std::memcpy(dst + L.seg_ibeg, hp.seg_ibeg.data(), hp.seg_ibeg.size() * sizeof(uint32_t));
  std::memcpy(dst + L.stages, hp.stages.data(), hp.stages.size() * sizeof(DevStage));
  std::memset(dst + L.ctr, 0, hp.levels.size() * 4 * sizeof(uint32_t));  // seg(4)_kernel work counters
  std::memcpy(dst + L.funits, hp.flow_units.data(), hp.flow_units.size() * sizeof(FlowUnit));
  std::memcpy(dst + L.finit, hp.flow_init.data(), hp.flow_init.size() * sizeof(uint64_t));
  std::memcpy(dst + L.scal, hp.scalar_off.data(), hp.scalar_off.size() * sizeof(uint64_t));
  std::memcpy(dst + L.lcb, hp.lc_begin.data(), hp.lc_begin.size() * sizeof(uint32_t));
  std::memcpy(dst + L.lce, hp.lc_edge.data(), hp.lc_edge.size() * sizeof(int32_t));
}

}  // namespace

// ---------------------------------------------------------------- context

// An independent stream set + buffers: the one-shot energy pipelines two
// halves of the lightcones through two lanes (host planning of the second
// half overlaps the device work of the first).
struct Lane {
  cudaStream_t s = nullptr, s2 = nullptr, s3 = nullptr;
  cudaEvent_t fork = nullptr, join2 = nullptr, join3 = nullptr;
  cudaStream_t s4 = nullptr;      // quad-tile segment kernels, forked per level
  cudaEvent_t join4 = nullptr;
  DevBuf* arena = nullptr;
  DevBuf* desc = nullptr;
  PinBuf *pin_desc = nullptr, *pin_in = nullptr, *pin_out = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;  // device time of the lane's program (one-shot energy)
};

struct qtng_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  DevBuf arena;          // double2 elements
  uint64_t arena_gen = 0;
  DevBuf desc;           // scratch descriptors (one-shot calls)
  PinBuf pin_desc, pin_in, pin_out;
  cudaStream_t stream2 = nullptr;  // outer-join kernels, forked per level
  cudaStream_t stream3 = nullptr;  // fused-chain segment kernels, forked per level
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr, join3_ev = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  DevBuf sv_scratch;     // state-vector oracle: edge bits, per-edge sums, partials
  DevBuf multi_full;     // qtng_energy_multi: the 2m-double term vector NCCL reduces
  PinBuf stg[2];         // chunked staging of large pageable host buffers (bucket drop-in)
  cudaEvent_t stg_ev[2] = {nullptr, nullptr};
  static constexpr int kLanes = 4;
  Lane lane[kLanes];     // lane 0 aliases the fields above; lanes 1.. own theirs
  DevBuf arena_x[kLanes], desc_x[kLanes];
  PinBuf pin_desc_x[kLanes], pin_in_x[kLanes], pin_out_x[kLanes];
  // default arithmetic of QAOA plans / energies whose call passes precision 0:
  // 128 = complex128, 64 = complex64.  Read once per call (atomic).
  std::atomic<int> prec{128};
  std::atomic<int> refs{1};  // the owner + one per live plan (ctx_release)
  std::unique_ptr<qtng::Worker> enq;  // one-shot energy: chunk enqueue thread (under mu)

  // arena of `elems` elements of `elem_bytes` (16: double2, 8: float2)
  void ensure_arena(uint64_t elems, size_t elem_bytes = sizeof(double2)) {
    const size_t bytes = std::max<uint64_t>(elems, 32) * elem_bytes;
    if (bytes > arena.cap) {
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      if (bytes > free_b + arena.cap)
        throw Error(kResource, "device arena of " + std::to_string(bytes) +
                                   " bytes exceeds free HBM (" + std::to_string(free_b) + ")");
      arena.ensure(bytes);
      ++arena_gen;
    }
  }
  double2* A() { return static_cast<double2*>(arena.p); }
};

namespace {

struct DevProgram {
  char* base = nullptr;
  DescLayout L;
  bool c64 = false;  // complex64 arena (float2) and kernels
  const DevOp* ops() const { return reinterpret_cast<const DevOp*>(base + L.ops); }
  const uint32_t* ibeg() const { return reinterpret_cast<const uint32_t*>(base + L.ibeg); }
  const DevTensor* trefs() const { return reinterpret_cast<const DevTensor*>(base + L.trefs); }
  const DevSeg* segs() const { return reinterpret_cast<const DevSeg*>(base + L.segs); }
  const uint32_t* seg_ibeg() const { return reinterpret_cast<const uint32_t*>(base + L.seg_ibeg); }
  const DevStage* stages() const { return reinterpret_cast<const DevStage*>(base + L.stages); }
  SegOpTab* segtab() const { return reinterpret_cast<SegOpTab*>(base + L.segtab); }
  template <class T>
  T* at(size_t off) const { return reinterpret_cast<T*>(base + off); }
  // per level: seg_kernel's tile queue (2 counters), then seg4_kernel's
  uint32_t* ctr(size_t level) const { return reinterpret_cast<uint32_t*>(base + L.ctr) + 4 * level; }
  const uint64_t* scal() const { return reinterpret_cast<const uint64_t*>(base + L.scal); }
  const uint32_t* lcb() const { return reinterpret_cast<const uint32_t*>(base + L.lcb); }
  const int32_t* lce() const { return reinterpret_cast<const int32_t*>(base + L.lce); }
  double2* terms() const { return reinterpret_cast<double2*>(base + L.terms); }
};

// One level: the outer-join and segment kernels forked onto side streams, the
// generic kernel on the main stream, joined before the next level.
// kev (optional): 8 events bracketing this level's level / outer / segment /
// quad-segment kernels on the streams they run on (per-kernel device time).
void enqueue_level(qtng_ctx* ctx, const LevelLaunch& lv, size_t level, const DevProgram& pr,
                   void* arena, cudaEvent_t* kev = nullptr, const Lane* ln = nullptr) {
  const Lane& la = ln ? *ln : ctx->lane[0];
  const bool c64 = pr.c64;
  const bool fork2 = lv.outer_items > 0;
  const bool fork3 = lv.seg_items > 0 && (lv.items > 0 || fork2 || lv.seg4_items > 0);
  const bool fork4 = lv.seg4_items > 0;
  auto rec = [&](int k, cudaStream_t st) {
    if (kev) QTNG_CUDA(cudaEventRecord(kev[k], st));
  };
  if (fork2 || fork3 || fork4) QTNG_CUDA(cudaEventRecord(la.fork, la.s));
  static const bool seg4_first = [] {  // QTNG_SEG4_FIRST=0: quad kernel after seg_kernel
    const char* v = std::getenv("QTNG_SEG4_FIRST");
    return !(v && v[0] == '0');
  }();
  auto launch4 = [&] {
    QTNG_CUDA(cudaStreamWaitEvent(la.s4, la.fork, 0));
    rec(6, la.s4);
    QTNG_CUDA(c64 ? c64::launch_segs4(la.s4, pr.segs(), pr.seg_ibeg(), pr.stages(), pr.trefs(),
                                      pr.segtab(), arena, pr.ctr(level) + 2, lv)
                  : c128::launch_segs4(la.s4, pr.segs(), pr.seg_ibeg(), pr.stages(), pr.trefs(),
                                       pr.segtab(), arena, pr.ctr(level) + 2, lv));
    rec(7, la.s4);
    QTNG_CUDA(cudaEventRecord(la.join4, la.s4));
  };
  if (fork4 && seg4_first) launch4();
  if (fork2) {
    QTNG_CUDA(cudaStreamWaitEvent(la.s2, la.fork, 0));
    rec(2, la.s2);
    QTNG_CUDA(c64 ? c64::launch_outer(la.s2, pr.ops(), pr.ibeg(), pr.trefs(), arena, lv)
                  : c128::launch_outer(la.s2, pr.ops(), pr.ibeg(), pr.trefs(), arena, lv));
    rec(3, la.s2);
    QTNG_CUDA(cudaEventRecord(la.join2, la.s2));
  }
  cudaStream_t s3 = fork3 ? la.s3 : la.s;
  if (fork3) QTNG_CUDA(cudaStreamWaitEvent(la.s3, la.fork, 0));
  rec(4, s3);
  QTNG_CUDA(c64 ? c64::launch_segs(s3, pr.segs(), pr.seg_ibeg(), pr.stages(), pr.trefs(),
                                    pr.segtab(), arena, pr.ctr(level), lv)
                : c128::launch_segs(s3, pr.segs(), pr.seg_ibeg(), pr.stages(), pr.trefs(),
                                    pr.segtab(), arena, pr.ctr(level), lv));
  rec(5, s3);
  if (fork3) QTNG_CUDA(cudaEventRecord(la.join3, la.s3));
  if (fork4 && !seg4_first) launch4();
  rec(0, la.s);
  QTNG_CUDA(c64 ? c64::launch_level(la.s, pr.ops(), pr.ibeg(), pr.trefs(), arena, lv)
                : c128::launch_level(la.s, pr.ops(), pr.ibeg(), pr.trefs(), arena, lv));
  rec(1, la.s);
  if (fork2) QTNG_CUDA(cudaStreamWaitEvent(la.s, la.join2, 0));
  if (fork3) QTNG_CUDA(cudaStreamWaitEvent(la.s, la.join3, 0));
  if (fork4) QTNG_CUDA(cudaStreamWaitEvent(la.s, la.join4, 0));
}

size_t elem_bytes(const HostPlan& hp) { return hp.c64 ? sizeof(float2) : sizeof(double2); }

// Copy `elems` complex128 inputs (interleaved re, im) into a pinned staging
// buffer in the plan's element type.
void stage_input(const HostPlan& hp, const double* in, uint64_t elems, void* dst) {
  if (!hp.c64) {
    std::memcpy(dst, in, elems * sizeof(double2));
    return;
  }
  float* f = static_cast<float*>(dst);
  for (uint64_t i = 0; i < 2 * elems; ++i) f[i] = static_cast<float>(in[i]);
}

// Upload a HostPlan's descriptor image to `dev` (layout L) on the context
// stream and build its device-only segment tables.
void upload_desc(qtng_ctx* ctx, const HostPlan& hp, const DescLayout& L, char* dev,
                 const Lane* ln = nullptr) {
  const Lane& la = ln ? *ln : ctx->lane[0];
  la.pin_desc->ensure(L.upload);
  pack_desc(hp, L, static_cast<char*>(la.pin_desc->p));
  QTNG_CUDA(cudaMemcpyAsync(dev, la.pin_desc->p, L.upload, cudaMemcpyHostToDevice, la.s));
  const DevProgram pr{dev, L, hp.c64};
  if (!hp.segs.empty()) g_launches.fetch_add(1, std::memory_order_relaxed);
  QTNG_CUDA(c128::launch_seg_prep(la.s, pr.segs(), static_cast<uint32_t>(hp.segs.size()), pr.trefs(),
                            pr.segtab()));
}

// Enqueue the whole program on the context's stream: every level, then the
// per-lightcone products.
int launches_per_run(const HostPlan& hp);

// full (optional, device, 2 doubles per edge of the graph): every lightcone's
// term is also written to its edge slot (the multi-GPU reduce vector).
void enqueue_program(qtng_ctx* ctx, const HostPlan& hp, const DevProgram& pr, void* arena,
                     std::vector<cudaEvent_t>* level_events,
                     std::vector<cudaEvent_t>* kernel_events = nullptr, const Lane* ln = nullptr,
                     double2* full = nullptr) {
  const Lane& la = ln ? *ln : ctx->lane[0];
  cudaStream_t s = la.s;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  QTNG_CUDA(cudaStreamIsCapturing(s, &cap));
  if (cap == cudaStreamCaptureStatusNone)
    g_launches.fetch_add(static_cast<uint64_t>(launches_per_run(hp)), std::memory_order_relaxed);
  if (hp.flow) {  // one persistent dataflow kernel instead of the level sequence
    if (level_events) QTNG_CUDA(cudaEventRecord((*level_events)[0], s));
    const DescLayout& L = pr.L;
    const auto n = static_cast<uint32_t>(hp.flow_units.size());
    const auto ni = static_cast<uint32_t>(hp.flow_init.size());
    QTNG_CUDA((pr.c64 ? c64::launch_flow : c128::launch_flow)(
        s, pr.at<FlowUnit>(L.funits), n, pr.at<uint64_t>(L.finit), ni,
        static_cast<uint32_t>(hp.flow_chunks), pr.ops(), pr.segs(), pr.stages(), pr.trefs(),
        pr.segtab(), arena, pr.at<uint32_t>(L.fdone), pr.at<int32_t>(L.fdeps),
        pr.at<uint64_t>(L.fqueue), pr.at<FlowState>(L.fstate)));
    for (size_t k = 1; level_events && k <= hp.levels.size(); ++k)
      QTNG_CUDA(cudaEventRecord((*level_events)[k], s));
  }
  for (size_t L = 0; L < hp.levels.size() && !hp.flow; ++L) {
    if (level_events) QTNG_CUDA(cudaEventRecord((*level_events)[L], s));
    enqueue_level(ctx, hp.levels[L], L, pr, arena,
                  kernel_events ? kernel_events->data() + 8 * L : nullptr, &la);
  }
  if (level_events) QTNG_CUDA(cudaEventRecord((*level_events)[hp.levels.size()], s));
  QTNG_CUDA((pr.c64 ? c64::launch_final : c128::launch_final)(
      s, pr.scal(), pr.lcb(), static_cast<int>(hp.lc_begin.size()) - 1, arena, pr.terms(),
      pr.lce(), full));
}

int launches_per_run(const HostPlan& hp) {
  if (hp.flow) return 3;  // flow_reset, flow_kernel, final_kernel
  int lv = 0, outer = 0, seg = 0, seg4 = 0;
  for (const LevelLaunch& l : hp.levels) {
    lv += l.items > 0;
    outer += l.outer_items > 0;
    seg += l.seg_items > 0;
    seg4 += l.seg4_items > 0;
  }
  return kernels_per_plan(lv, outer, seg, seg4);
}

// Ops of the reference's run_edge post-processing (engine.cpp:517-519, 543-546).
// |imag e_jk| bound: the reference's 1e-8 (engine.cpp:517-519); complex64
// plans use the north_star's 1e-5.
double imag_tol(bool c64) { return c64 ? 1e-5 : 1e-8; }

// The arithmetic of a QAOA plan / energy call: `precision` 0 = the context's
// default (qtng_set_precision), read once.
int resolve_prec(const qtng_ctx* ctx, int precision) {
  if (precision == 0) return ctx->prec.load();
  if (precision != 128 && precision != 64)
    throw Error(kInvalidInput, "precision must be 128 or 64 bits");
  return precision;
}


void check_terms(const std::vector<Edge>& edges, const double* terms, double tol = 1e-8) {
  for (size_t i = 0; i < edges.size(); ++i)
    if (std::abs(terms[2 * i + 1]) > tol)
      throw Error(kSchedule, "edge (" + std::to_string(edges[i].u) + ", " +
                                 std::to_string(edges[i].v) +
                                 "): edge term has non-real value: imag = " +
                                 std::to_string(terms[2 * i + 1]));
}

}  // namespace

struct qtng_plan {
  qtng_ctx* ctx = nullptr;
  HostPlan hp;
  std::vector<Edge> edges;
  int p = 0;
  bool explicit_sched = false;  // qtng_plan_create_schedule: input region = pin_gate as given
  DevBuf desc;
  DevProgram prog;
  PinBuf pin_gate, pin_terms;
  std::vector<cudaEvent_t> lev_ev;
  std::vector<float> level_ms;
  std::vector<cudaEvent_t> ker_ev;  // 8 per level (enqueue_level)
  float kernel_ms[4] = {0.f, 0.f, 0.f, 0.f};  // level / outer / seg / seg4 kernels, last profile
  std::vector<float> level_kernel_ms;    // 4 per level, last profile
  cudaGraphExec_t graph = nullptr;       // kernels only (qtng_plan_run_device)
  uint64_t graph_gen = ~uint64_t{0};
  cudaGraphExec_t graph_io = nullptr;    // gate-table H2D + kernels + terms D2H (qtng_plan_execute)
  uint64_t graph_io_gen = ~uint64_t{0};
  float last_ms = 0.f;                   // device time of the last execute / run
  bool profiled = false;                 // level_ms holds a qtng_plan_profile measurement
  ~qtng_plan() {
    for (cudaEvent_t e : lev_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : ker_ev) cudaEventDestroy(e);
    if (graph) cudaGraphExecDestroy(graph);
    if (graph_io) cudaGraphExecDestroy(graph_io);
  }
};

extern "C" {

const char* qtng_last_error(void) { return g_err.c_str(); }

uint64_t qtng_kernel_launches(void) { return g_launches.load(); }

const char* qtng_version(void) {
  return "qtng 0.1 (sm_100a level-batched bucket elimination, complex128, bit-exact naive order)";
}

qtng_status qtng_create(int device, uint64_t arena_bytes, qtng_ctx** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalidInput, "null output pointer");
    auto ctx = std::make_unique<qtng_ctx>();
    ctx->device = device;
    QTNG_CUDA(cudaSetDevice(device));
    QTNG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    QTNG_CUDA(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
    QTNG_CUDA(cudaStreamCreateWithFlags(&ctx->stream3, cudaStreamNonBlocking));
    QTNG_CUDA(cudaEventCreate(&ctx->ev0));
    QTNG_CUDA(cudaEventCreate(&ctx->ev1));
    QTNG_CUDA(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
    QTNG_CUDA(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
    QTNG_CUDA(cudaEventCreateWithFlags(&ctx->join3_ev, cudaEventDisableTiming));
    Lane& l0 = ctx->lane[0];
    l0 = Lane{};
    l0.s = ctx->stream;
    l0.s2 = ctx->stream2;
    l0.s3 = ctx->stream3;
    l0.fork = ctx->fork_ev;
    l0.join2 = ctx->join_ev;
    l0.join3 = ctx->join3_ev;
    l0.arena = &ctx->arena;
    l0.desc = &ctx->desc;
    l0.pin_desc = &ctx->pin_desc;
    l0.pin_in = &ctx->pin_in;
    l0.pin_out = &ctx->pin_out;
    for (cudaEvent_t* ev : {&ctx->stg_ev[0], &ctx->stg_ev[1]})
      QTNG_CUDA(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    for (int i = 0; i < qtng_ctx::kLanes; ++i) {
      for (cudaEvent_t* ev : {&ctx->lane[i].t0, &ctx->lane[i].t1}) QTNG_CUDA(cudaEventCreate(ev));
      QTNG_CUDA(cudaStreamCreateWithFlags(&ctx->lane[i].s4, cudaStreamNonBlocking));
      QTNG_CUDA(cudaEventCreateWithFlags(&ctx->lane[i].join4, cudaEventDisableTiming));
    }
    for (int i = 1; i < qtng_ctx::kLanes; ++i) {
      Lane& l1 = ctx->lane[i];
      l1.arena = &ctx->arena_x[i];
      l1.desc = &ctx->desc_x[i];
      l1.pin_desc = &ctx->pin_desc_x[i];
      l1.pin_in = &ctx->pin_in_x[i];
      l1.pin_out = &ctx->pin_out_x[i];
      for (cudaStream_t* st : {&l1.s, &l1.s2, &l1.s3})
        QTNG_CUDA(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
      for (cudaEvent_t* ev : {&l1.fork, &l1.join2, &l1.join3})
        QTNG_CUDA(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    }
    if (arena_bytes) ctx->ensure_arena(arena_bytes / sizeof(double2));
    *out = ctx.release();
  });
}

}  // extern "C"

namespace {

// Frees a context once neither its owner (qtng_destroy) nor any plan created
// on it (qtng_plan_destroy) holds it: plans may outlive the qtng_destroy call
// (garbage-collected bindings destroy in any order).
void ctx_release(qtng_ctx* ctx) {
  if (ctx->refs.fetch_sub(1) != 1) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamSynchronize(ctx->stream2);
  cudaStreamSynchronize(ctx->stream3);
  std::vector<cudaStream_t> streams = {ctx->stream, ctx->stream2, ctx->stream3};
  for (int i = 1; i < qtng_ctx::kLanes; ++i) {
    const Lane& l1 = ctx->lane[i];
    for (cudaStream_t st : {l1.s, l1.s2, l1.s3})
      if (st) {
        cudaStreamSynchronize(st);
        streams.push_back(st);
      }
    for (cudaEvent_t e : {l1.fork, l1.join2, l1.join3})
      if (e) cudaEventDestroy(e);
  }
  for (int i = 0; i < qtng_ctx::kLanes; ++i) {
    if (ctx->lane[i].s4) {
      cudaStreamSynchronize(ctx->lane[i].s4);
      streams.push_back(ctx->lane[i].s4);
    }
    for (cudaEvent_t e : {ctx->lane[i].t0, ctx->lane[i].t1, ctx->lane[i].join4})
      if (e) cudaEventDestroy(e);
  }
  for (cudaEvent_t e : {ctx->ev0, ctx->ev1, ctx->fork_ev, ctx->join_ev, ctx->join3_ev,
                        ctx->stg_ev[0], ctx->stg_ev[1]})
    if (e) cudaEventDestroy(e);
  delete ctx;  // frees the arenas and staging buffers
  for (cudaStream_t st : streams)
    if (st) cudaStreamDestroy(st);
}

}  // namespace

extern "C" {

void qtng_destroy(qtng_ctx* ctx) {
  if (ctx) ctx_release(ctx);
}

qtng_status qtng_set_precision(qtng_ctx* ctx, int bits) {
  return guarded([&] {
    if (!ctx) throw Error(kInvalidInput, "null context");
    if (bits != 128 && bits != 64) throw Error(kInvalidInput, "precision must be 128 or 64 bits");
    ctx->prec.store(bits);
  });
}

qtng_status qtng_random_regular(int n, int d, uint64_t seed, int* edges, int cap, int* m_out) {
  return guarded([&] {
    const Graph g = random_regular(n, d, seed);
    const int m = static_cast<int>(g.edges.size());
    if (m_out) *m_out = m;
    if (m > cap) throw Error(kInvalidInput, "edge buffer too small");
    for (int i = 0; i < m; ++i) {
      edges[2 * i] = g.edges[i].u;
      edges[2 * i + 1] = g.edges[i].v;
    }
  });
}

qtng_status qtng_edge_schedule(int n, int m, const int* edges, int p, const double* gammas,
                               const double* betas, int edge_index, int merged, int* ints,
                               int64_t int_cap, double* data, int64_t data_cap,
                               int64_t* n_ints, int64_t* n_data, int* n_buckets, int* merges) {
  return guarded([&] {
    validate_angles(p, gammas, betas);
    const Graph g = graph_from(n, m, edges);
    if (edge_index < 0 || edge_index >= m) throw Error(kInvalidInput, "edge index out of range");
    Schedule s = edge_schedule(g, g.edges[edge_index], p);
    if (merged) s = merge_buckets(s);
    std::vector<double> table(2 * kSlotElems * n_gate_slots(p));
    fill_gate_table(p, gammas, betas, table.data());
    std::vector<int> iv;
    std::vector<double> dv;
    flatten_schedule(s, table.data(), iv, dv);
    *n_ints = static_cast<int64_t>(iv.size());
    *n_data = static_cast<int64_t>(dv.size());
    *n_buckets = static_cast<int>(s.buckets.size());
    if (merges) {
      merges[0] = s.merges_applied;
      merges[1] = s.merges_skipped;
    }
    if (static_cast<int64_t>(iv.size()) <= int_cap && static_cast<int64_t>(dv.size()) <= data_cap) {
      std::copy(iv.begin(), iv.end(), ints);
      std::copy(dv.begin(), dv.end(), data);
    }
  });
}

qtng_status qtng_merge_schedule(int n_buckets, const int* ints, int64_t n_ints, int* out,
                                int64_t cap, int64_t* n_out, int* out_buckets, int* merges) {
  return guarded([&] {
    if (!n_out || !out_buckets) throw Error(kInvalidInput, "null argument");
    const Schedule s = merge_buckets(parse_schedule(n_buckets, ints, static_cast<long>(n_ints)));
    std::vector<int> v;
    for (const SchedBucket& b : s.buckets) {
      v.push_back(static_cast<int>(b.sum_vars.size()));
      v.insert(v.end(), b.sum_vars.begin(), b.sum_vars.end());
      v.push_back(static_cast<int>(b.tensors.size()));
      v.insert(v.end(), b.tensors.begin(), b.tensors.end());  // input tensor indices
    }
    *n_out = static_cast<int64_t>(v.size());
    *out_buckets = static_cast<int>(s.buckets.size());
    if (merges) {
      merges[0] = s.merges_applied;
      merges[1] = s.merges_skipped;
    }
    if (out && static_cast<int64_t>(v.size()) <= cap) std::copy(v.begin(), v.end(), out);
  });
}

qtng_status qtng_simulate_widths(int n, int m, const int* edges, int p, int edge_index,
                                 int merged, int* widths, int cap, int* n_out) {
  return guarded([&] {
    const Graph g = graph_from(n, m, edges);
    if (edge_index < 0 || edge_index >= m) throw Error(kInvalidInput, "edge index out of range");
    Schedule s = edge_schedule(g, g.edges[edge_index], p);
    if (merged) s = merge_buckets(s);
    const std::vector<int> w = simulate_widths(s);
    *n_out = static_cast<int>(w.size());
    if (static_cast<int>(w.size()) > cap) throw Error(kInvalidInput, "width buffer too small");
    std::copy(w.begin(), w.end(), widths);
  });
}

qtng_status qtng_edge_costs(int n, int m, const int* edges, int p, int merged, double* bytes_out) {
  return guarded([&] {
    const Graph g = graph_from(n, m, edges);
    const ConeSet cs = plan_cones(g, p, merged != 0, 1 << 20, selection(m, m, nullptr));
    for (int i = 0; i < m; ++i) {
      double b = 0;
      const WalkResult& w = cs.walks[i];
      for (const Op& op : w.ops) {
        b += 16.0 * static_cast<double>(uint64_t{1} << op.r);
        for (int t = 0; t < op.nin; ++t)
          b += 16.0 * static_cast<double>(uint64_t{1} << w.inputs(op)[t].rank);
      }
      bytes_out[i] = b;
    }
  });
}

qtng_status qtng_edge_work(int n, int m, const int* edges, int p, int merged, double* work_out) {
  return guarded([&] {
    const Graph g = graph_from(n, m, edges);
    const ConeSet cs = plan_cones(g, p, merged != 0, 1 << 20, selection(m, m, nullptr));
    for (int i = 0; i < m; ++i) {
      double fl = 0;  // the reference loop's complex products + additions per lightcone
      for (const Op& op : cs.walks[i].ops)
        fl += std::ldexp(1.0, op.width) * std::max(1, op.nin - 1) +
              std::ldexp(1.0, op.r) * (std::ldexp(1.0, op.ns) - 1.0);
      work_out[i] = fl;
    }
  });
}

qtng_status qtng_validate_energy(int n, int m, const int* edges, int p, int merged,
                                 int max_result_width) {
  return guarded([&] {
    if (p < 1) throw Error(kInvalidInput, "angles: gammas and betas must have equal length p >= 1");
    const Graph g = graph_from(n, m, edges);
    const ConeSet cs = plan_cones(g, p, merged != 0, max_result_width, selection(m, m, nullptr));
    for (size_t i = 0; i < cs.walks.size(); ++i)
      if (cs.walks[i].fail_code)
        throw Error(kSchedule, "edge (" + std::to_string(cs.edges[i].u) + ", " +
                                   std::to_string(cs.edges[i].v) + "): " + cs.walks[i].fail_msg);
  });
}

qtng_status qtng_plan_dump(int n, int m, const int* edges, int p, int merged,
                           int max_result_width, int n_sel, const int* sel, int* ints,
                           int64_t cap, int64_t* n_ints, int* n_ops) {
  return guarded([&] {
    if (p < 1) throw Error(kInvalidInput, "angles: gammas and betas must have equal length p >= 1");
    const Graph g = graph_from(n, m, edges);
    const ConeSet cs = plan_cones(g, p, merged != 0, max_result_width, selection(m, n_sel, sel));
    std::vector<const WalkResult*> ptrs;
    for (const WalkResult& w : cs.walks) {
      if (w.fail_code) throw Error(w.fail_code, w.fail_msg);
      ptrs.push_back(&w);
    }
    // every op as its own device op (no chain fusion): the op-class view;
    // QTNG_DUMP_FUSED=1: the level ops of the fused program instead
    const char* fz = std::getenv("QTNG_DUMP_FUSED");
    const bool fuse = fz && fz[0] == '1';
    const HostPlan hp = build_plan(ptrs, static_cast<uint64_t>(n_gate_slots(p)) * kSlotElems, fuse, true);
    std::vector<int> out;
    for (size_t L = 0; L < hp.levels.size(); ++L)
      for (uint32_t k = 0; k < hp.levels[L].op_count + hp.levels[L].outer_count; ++k) {
        const uint32_t i = hp.levels[L].op_begin + k;
        const DevOp& d = hp.ops[i];
        const int outer = k >= hp.levels[L].op_count ? 1 : 0;
        out.insert(out.end(), {static_cast<int>(L), d.r, d.ns, d.nt, d.cb,
                               hp.op_width[i] > 0 ? 1 : 0, hp.op_width[i], outer});
        for (int t = 0; t < d.nt; ++t) {
          const DevTensor& x = hp.trefs[d.tref + t];
          out.push_back(x.rank);
          out.push_back(x.off < hp.input_elems ? 1 : 0);
          for (int a = 0; a < kMaxRank; ++a) out.push_back(a < x.rank ? x.src[a] : -1);
        }
      }
    *n_ints = static_cast<int64_t>(out.size());
    *n_ops = static_cast<int>(hp.ops.size());
    if (static_cast<int64_t>(out.size()) <= cap) std::copy(out.begin(), out.end(), ints);
  });
}

// ---------------------------------------------------------------- one-shot device calls

namespace {

// Run a single-"lightcone" program whose inputs are `input` (complex count
// input_elems) and return the HostPlan (for record / output offsets).
// Large pageable host <-> device copies on the context stream through two
// pinned 8 MiB chunks: the host memcpy of one chunk overlaps the DMA of the
// other (a pageable cudaMemcpy runs at a few GB/s; the per-bucket drop-in
// moves every bucket's operands and result across PCIe).  d2h returns with
// the data in dst (synchronous).
constexpr size_t kStageChunk = size_t{8} << 20;

void h2d_staged(qtng_ctx* ctx, void* dst, const void* src, size_t bytes) {
  for (int b = 0; b < 2; ++b) ctx->stg[b].ensure(kStageChunk);
  size_t i = 0;
  for (size_t off = 0; off < bytes; off += kStageChunk, ++i) {
    const int b = static_cast<int>(i & 1);
    if (i >= 2) QTNG_CUDA(cudaEventSynchronize(ctx->stg_ev[b]));  // chunk i-2's DMA is done
    const size_t n = std::min(kStageChunk, bytes - off);
    std::memcpy(ctx->stg[b].p, static_cast<const char*>(src) + off, n);
    QTNG_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, ctx->stg[b].p, n,
                              cudaMemcpyHostToDevice, ctx->stream));
    QTNG_CUDA(cudaEventRecord(ctx->stg_ev[b], ctx->stream));
  }
}

void d2h_staged(qtng_ctx* ctx, void* dst, const void* src, size_t bytes) {
  for (int b = 0; b < 2; ++b) ctx->stg[b].ensure(kStageChunk);
  const size_t nch = (bytes + kStageChunk - 1) / kStageChunk;
  auto issue = [&](size_t i) {
    const int b = static_cast<int>(i & 1);
    const size_t off = i * kStageChunk, n = std::min(kStageChunk, bytes - off);
    QTNG_CUDA(cudaMemcpyAsync(ctx->stg[b].p, static_cast<const char*>(src) + off, n,
                              cudaMemcpyDeviceToHost, ctx->stream));
    QTNG_CUDA(cudaEventRecord(ctx->stg_ev[b], ctx->stream));
  };
  for (size_t i = 0; i < nch && i < 2; ++i) issue(i);
  for (size_t i = 0; i < nch; ++i) {
    const int b = static_cast<int>(i & 1);
    QTNG_CUDA(cudaEventSynchronize(ctx->stg_ev[b]));
    const size_t off = i * kStageChunk, n = std::min(kStageChunk, bytes - off);
    std::memcpy(static_cast<char*>(dst) + off, ctx->stg[b].p, n);
    if (i + 2 < nch) issue(i + 2);
  }
}

void run_program_once(qtng_ctx* ctx, const HostPlan& hp, const double* input,
                      uint64_t input_elems, double2* terms_host) {
  const DescLayout L = layout_of(hp);
  const size_t eb = elem_bytes(hp);
  ctx->ensure_arena(std::max(hp.arena_elems, input_elems), eb);
  ctx->desc.ensure(L.total);
  if (!hp.c64 && input_elems * eb > kStageChunk) {  // large inputs: chunked, overlapped staging
    h2d_staged(ctx, ctx->arena.p, input, input_elems * eb);
  } else {
    ctx->pin_in.ensure(std::max<uint64_t>(input_elems, 1) * eb);
    stage_input(hp, input, input_elems, ctx->pin_in.p);
    QTNG_CUDA(cudaMemcpyAsync(ctx->arena.p, ctx->pin_in.p, input_elems * eb, cudaMemcpyHostToDevice,
                              ctx->stream));
  }
  upload_desc(ctx, hp, L, static_cast<char*>(ctx->desc.p));
  DevProgram pr{static_cast<char*>(ctx->desc.p), L, hp.c64};
  enqueue_program(ctx, hp, pr, ctx->arena.p, nullptr);
  if (terms_host) {
    const size_t nb = (hp.lc_begin.size() - 1) * sizeof(double2);
    QTNG_CUDA(cudaMemcpyAsync(terms_host, pr.terms(), nb, cudaMemcpyDeviceToHost, ctx->stream));
  }
}

}  // namespace

qtng_status qtng_contract_bucket(qtng_ctx* ctx, int n_tensors, const int* ranks, const int* vars,
                                 const double* data, int n_sum, const int* sum_vars,
                                 int* out_rank, int* out_vars, double* out_data,
                                 int64_t out_cap) {
  return guarded([&] {
    if (!ctx) throw Error(kInvalidInput, "null context");
    if (n_tensors < 0 || n_sum < 0) throw Error(kInvalidInput, "negative count");
    Schedule s;
    s.buckets.resize(1);
    s.buckets[0].sum_vars.assign(sum_vars, sum_vars + n_sum);
    int64_t dof = 0;
    long vo = 0;
    for (int t = 0; t < n_tensors; ++t) {
      if (ranks[t] < 0 || ranks[t] > kMaxRank)
        throw Error(kInvalidInput, "tensor rank out of range");
      SchedTensor st;
      st.vars.assign(vars + vo, vars + vo + ranks[t]);
      vo += ranks[t];
      st.data = dof;
      dof += int64_t{1} << ranks[t];
      s.buckets[0].tensors.push_back(t);
      s.init.push_back(std::move(st));
    }
    if (n_tensors == 0) {  // empty product: NaiveBackend yields the scalar 1
      if (n_sum > 0) throw Error(kSchedule, "bucket sums a variable absent from its tensors");
      *out_rank = 0;
      if (out_cap < 1) throw Error(kInvalidInput, "output buffer too small");
      out_data[0] = 1.0;
      out_data[1] = 0.0;
      return;
    }
    const WalkResult w = device_walk(s, 1 << 20, /*route=*/false);
    if (w.fail_code) throw Error(w.fail_code, w.fail_msg);
    const Op& op = w.ops.back();  // the bucket itself (pre-fold helpers come first)
    const int r = op.r;
    if ((int64_t{1} << r) > out_cap) throw Error(kInvalidInput, "output buffer too small");
    const HostPlan hp = build_plan({&w}, static_cast<uint64_t>(dof));
    std::lock_guard<std::mutex> lk(ctx->mu);
    QTNG_CUDA(cudaSetDevice(ctx->device));
    run_program_once(ctx, hp, data, static_cast<uint64_t>(dof), nullptr);
    d2h_staged(ctx, out_data, ctx->A() + hp.rec_out[0], (size_t{1} << r) * sizeof(double2));
    *out_rank = r;
    for (int k = 0; k < r; ++k) out_vars[k] = w.ids[w.out_vars(op)[k]];
  });
}

qtng_status qtng_contract_schedule(qtng_ctx* ctx, int n_buckets, const int* ints, int64_t n_ints,
                                   const double* data, int max_result_width,
                                   double* scalar_re_im, qtng_record* records, int rec_cap,
                                   int* n_records, uint64_t* peak_tensor_bytes) {
  return guarded([&] {
    if (!ctx) throw Error(kInvalidInput, "null context");
    const Schedule s = parse_schedule(n_buckets, ints, static_cast<long>(n_ints));
    const WalkResult w = device_walk(s, max_result_width);
    if (w.fail_code) throw Error(w.fail_code, w.fail_msg);
    uint64_t input_elems = 0;
    for (const SchedTensor& t : s.init) input_elems += uint64_t{1} << t.vars.size();
    double2 scalar = make_double2(1.0, 0.0);
    float ms = 0.f;
    HostPlan hp;
    if (!w.ops.empty()) {
      hp = build_plan({&w}, input_elems);
      std::lock_guard<std::mutex> lk(ctx->mu);
      QTNG_CUDA(cudaSetDevice(ctx->device));
      QTNG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
      run_program_once(ctx, hp, data, input_elems, &scalar);
      QTNG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
      QTNG_CUDA(cudaStreamSynchronize(ctx->stream));
      QTNG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    }
    scalar_re_im[0] = scalar.x;
    scalar_re_im[1] = scalar.y;
    const int n = static_cast<int>(hp.rec_seq.size());
    if (n_records) *n_records = n;
    double total_bytes = 0;
    for (double b : hp.rec_bytes) total_bytes += b;
    for (int i = 0; i < n && i < rec_cap && records; ++i) {
      qtng_record& r = records[i];
      r.edge_u = r.edge_v = -1;
      r.bucket_seq = hp.rec_seq[i];
      r.width = hp.rec_width[i];
      r.ops = uint64_t{1} << r.width;
      r.elapsed_s = std::max(1e-9, 1e-3 * ms * (total_bytes > 0 ? hp.rec_bytes[i] / total_bytes : 0));
      r.flops_est = 8.0 * static_cast<double>(r.ops) / r.elapsed_s;
    }
    if (peak_tensor_bytes) *peak_tensor_bytes = w.ops.empty() ? 0 : (uint64_t{16} << w.max_result_rank);
  });
}

// ---------------------------------------------------------------- plans

qtng_status qtng_plan_create(qtng_ctx* ctx, int n, int m, const int* edges, int p, int merged,
                             int max_result_width, int precision, int n_sel, const int* sel,
                             qtng_plan** out) {
  return guarded([&] {
    if (!ctx || !out) throw Error(kInvalidInput, "null argument");
    if (p < 1) throw Error(kInvalidInput, "angles: gammas and betas must have equal length p >= 1");
    const int prec = resolve_prec(ctx, precision);
    const Graph g = graph_from(n, m, edges);
    const std::vector<int> s = selection(m, n_sel, sel);
    ConeSet cs = plan_cones(g, p, merged != 0, max_result_width, s);
    for (size_t i = 0; i < cs.walks.size(); ++i)
      if (cs.walks[i].fail_code)
        throw Error(kSchedule, "edge (" + std::to_string(cs.edges[i].u) + ", " +
                                   std::to_string(cs.edges[i].v) + "): " + cs.walks[i].fail_msg);
    auto plan = std::make_unique<qtng_plan>();
    plan->ctx = ctx;
    plan->p = p;
    plan->edges = cs.edges;
    std::vector<const WalkResult*> ptrs;
    for (const WalkResult& w : cs.walks) ptrs.push_back(&w);
    plan->hp = build_plan(ptrs, static_cast<uint64_t>(n_gate_slots(p)) * kSlotElems, fuse_default(), true);
    plan->hp.c64 = prec == 64;
    const HostPlan& hp = plan->hp;
    const DescLayout L = layout_of(hp);
    std::lock_guard<std::mutex> lk(ctx->mu);
    QTNG_CUDA(cudaSetDevice(ctx->device));
    plan->desc.ensure(L.total);
    plan->prog = DevProgram{static_cast<char*>(plan->desc.p), L, hp.c64};
    upload_desc(ctx, hp, L, static_cast<char*>(plan->desc.p));
    QTNG_CUDA(cudaStreamSynchronize(ctx->stream));
    plan->pin_gate.ensure(hp.input_elems * elem_bytes(hp));
    plan->pin_terms.ensure(std::max<size_t>(1, cs.walks.size()) * sizeof(double2));
    plan->lev_ev.resize(hp.levels.size() + 1);
    for (cudaEvent_t& e : plan->lev_ev) QTNG_CUDA(cudaEventCreate(&e));
    plan->ker_ev.resize(8 * hp.levels.size());
    for (cudaEvent_t& e : plan->ker_ev) QTNG_CUDA(cudaEventCreate(&e));
    plan->level_ms.assign(hp.levels.size(), 0.f);
    ctx->refs.fetch_add(1);  // released by qtng_plan_destroy
    *out = plan.release();
  });
}

qtng_status qtng_plan_create_schedule(qtng_ctx* ctx, int n_buckets, const int* ints,
                                      int64_t n_ints, const double* data, int max_result_width,
                                      qtng_plan** out) {
  return guarded([&] {
    if (!ctx || !out) throw Error(kInvalidInput, "null argument");
    const Schedule s = parse_schedule(n_buckets, ints, static_cast<long>(n_ints));
    // a one-bucket schedule is a single ContractionBackend::contract: its
    // result stays in place instead of being routed
    const WalkResult w = device_walk(s, max_result_width, /*route=*/n_buckets != 1);
    if (w.fail_code) throw Error(w.fail_code, w.fail_msg);
    if (w.ops.empty()) throw Error(kInvalidInput, "schedule has no non-empty bucket");
    uint64_t input_elems = 0;
    for (const SchedTensor& t : s.init) input_elems += uint64_t{1} << t.vars.size();
    auto plan = std::make_unique<qtng_plan>();
    plan->ctx = ctx;
    plan->explicit_sched = true;
    plan->edges = {Edge{-1, -1}};
    plan->hp = build_plan({&w}, input_elems);
    const HostPlan& hp = plan->hp;
    const DescLayout L = layout_of(hp);
    std::lock_guard<std::mutex> lk(ctx->mu);
    QTNG_CUDA(cudaSetDevice(ctx->device));
    plan->desc.ensure(L.total);
    plan->prog = DevProgram{static_cast<char*>(plan->desc.p), L, false};
    upload_desc(ctx, hp, L, static_cast<char*>(plan->desc.p));
    QTNG_CUDA(cudaStreamSynchronize(ctx->stream));
    plan->pin_gate.ensure(std::max<uint64_t>(input_elems, 1) * sizeof(double2));
    std::memcpy(plan->pin_gate.p, data, input_elems * sizeof(double2));
    plan->pin_terms.ensure(sizeof(double2));
    plan->lev_ev.resize(hp.levels.size() + 1);
    for (cudaEvent_t& e : plan->lev_ev) QTNG_CUDA(cudaEventCreate(&e));
    plan->ker_ev.resize(8 * hp.levels.size());
    for (cudaEvent_t& e : plan->ker_ev) QTNG_CUDA(cudaEventCreate(&e));
    plan->level_ms.assign(hp.levels.size(), 0.f);
    ctx->refs.fetch_add(1);  // released by qtng_plan_destroy
    *out = plan.release();
  });
}

}  // extern "C"

namespace {

// Fill the plan's pinned input staging for one angle set (QAOA plans: the
// gate table; explicit schedules keep the data given at creation).
void stage_plan_inputs(qtng_plan* plan, const double* gammas, const double* betas) {
  const HostPlan& hp = plan->hp;
  if (plan->explicit_sched) return;
  std::vector<double> table(2 * hp.input_elems);
  fill_gate_table(plan->p, gammas, betas, table.data());
  stage_input(hp, table.data(), hp.input_elems, plan->pin_gate.p);
}

// Capture `body` on the context stream into an executable graph.
template <class F>
cudaGraphExec_t capture(qtng_ctx* ctx, F&& body) {
  cudaGraph_t gr = nullptr;
  QTNG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  try {
    body();
  } catch (...) {
    cudaStreamEndCapture(ctx->stream, &gr);
    if (gr) cudaGraphDestroy(gr);
    throw;
  }
  QTNG_CUDA(cudaStreamEndCapture(ctx->stream, &gr));
  cudaGraphExec_t ex = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&ex, gr, 0);
  cudaGraphDestroy(gr);
  QTNG_CUDA(e);
  return ex;
}

}  // namespace

extern "C" {

qtng_status qtng_plan_execute(qtng_plan* plan, const double* gammas, const double* betas,
                              double* terms, float* device_ms) {
  return guarded([&] {
    if (!plan) throw Error(kInvalidInput, "null plan");
    if (!plan->explicit_sched) validate_angles(plan->p, gammas, betas);
    qtng_ctx* ctx = plan->ctx;
    const HostPlan& hp = plan->hp;
    std::lock_guard<std::mutex> lk(ctx->mu);
    QTNG_CUDA(cudaSetDevice(ctx->device));
    ctx->ensure_arena(hp.arena_elems, elem_bytes(hp));
    stage_plan_inputs(plan, gammas, betas);
    const size_t nb = plan->edges.size() * sizeof(double2);
    // one graph: the gate-table upload (memcpy node from the plan's pinned
    // staging), every level's kernels, the terms download -- re-captured only
    // when the context's arena moves
    if (!plan->graph_io || plan->graph_io_gen != ctx->arena_gen) {
      if (plan->graph_io) cudaGraphExecDestroy(plan->graph_io);
      plan->graph_io = nullptr;
      plan->graph_io = capture(ctx, [&] {
        QTNG_CUDA(cudaMemcpyAsync(ctx->arena.p, plan->pin_gate.p, hp.input_elems * elem_bytes(hp),
                                  cudaMemcpyHostToDevice, ctx->stream));
        enqueue_program(ctx, hp, plan->prog, ctx->arena.p, nullptr);
        QTNG_CUDA(cudaMemcpyAsync(plan->pin_terms.p, plan->prog.terms(), nb,
                                  cudaMemcpyDeviceToHost, ctx->stream));
      });
      plan->graph_io_gen = ctx->arena_gen;
    }
    QTNG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    QTNG_CUDA(cudaGraphLaunch(plan->graph_io, ctx->stream));
    QTNG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    g_launches.fetch_add(static_cast<uint64_t>(launches_per_run(hp)), std::memory_order_relaxed);
    QTNG_CUDA(cudaStreamSynchronize(ctx->stream));
    float ms = 0.f;
    QTNG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    plan->last_ms = ms;
    if (device_ms) *device_ms = ms;
    const double* t = static_cast<const double*>(plan->pin_terms.p);
    if (terms) std::memcpy(terms, t, nb);
    if (!plan->explicit_sched) check_terms(plan->edges, t, imag_tol(hp.c64));
  });
}

qtng_status qtng_plan_profile(qtng_plan* plan, const double* gammas, const double* betas,
                              double* terms, float* device_ms) {
  return guarded([&] {
    if (!plan) throw Error(kInvalidInput, "null plan");
    if (!plan->explicit_sched) validate_angles(plan->p, gammas, betas);
    qtng_ctx* ctx = plan->ctx;
    const HostPlan& hp = plan->hp;
    std::lock_guard<std::mutex> lk(ctx->mu);
    QTNG_CUDA(cudaSetDevice(ctx->device));
    ctx->ensure_arena(hp.arena_elems, elem_bytes(hp));
    stage_plan_inputs(plan, gammas, betas);
    QTNG_CUDA(cudaMemcpyAsync(ctx->arena.p, plan->pin_gate.p, hp.input_elems * elem_bytes(hp),
                              cudaMemcpyHostToDevice, ctx->stream));
    QTNG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    enqueue_program(ctx, hp, plan->prog, ctx->arena.p, &plan->lev_ev, &plan->ker_ev);
    QTNG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    const size_t nb = plan->edges.size() * sizeof(double2);
    QTNG_CUDA(cudaMemcpyAsync(plan->pin_terms.p, plan->prog.terms(), nb, cudaMemcpyDeviceToHost,
                              ctx->stream));
    QTNG_CUDA(cudaStreamSynchronize(ctx->stream));
    float ms = 0.f;
    QTNG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    for (size_t L = 0; L < hp.levels.size(); ++L)
      QTNG_CUDA(cudaEventElapsedTime(&plan->level_ms[L], plan->lev_ev[L], plan->lev_ev[L + 1]));
    for (float& k : plan->kernel_ms) k = 0.f;
    plan->level_kernel_ms.assign(4 * hp.levels.size(), 0.f);
    if (hp.flow) plan->kernel_ms[2] = plan->level_ms.empty() ? 0.f : plan->level_ms[0];
    for (size_t L = 0; L < hp.levels.size() && !hp.flow; ++L) {
      const LevelLaunch& lv = hp.levels[L];
      const uint32_t present[4] = {lv.items, lv.outer_items, lv.seg_items, lv.seg4_items};
      for (int k = 0; k < 4; ++k) {
        if (!present[k]) continue;
        float kms = 0.f;
        QTNG_CUDA(cudaEventElapsedTime(&kms, plan->ker_ev[8 * L + 2 * k], plan->ker_ev[8 * L + 2 * k + 1]));
        plan->kernel_ms[k] += kms;
        plan->level_kernel_ms[4 * L + k] = kms;
      }
    }
    plan->last_ms = ms;
    plan->profiled = true;
    if (device_ms) *device_ms = ms;
    const double* t = static_cast<const double*>(plan->pin_terms.p);
    if (terms) std::memcpy(terms, t, nb);
    if (!plan->explicit_sched) check_terms(plan->edges, t, imag_tol(hp.c64));
  });
}

qtng_status qtng_plan_run_device(qtng_plan* plan, int n_runs, float* device_ms) {
  return guarded([&] {
    if (!plan) throw Error(kInvalidInput, "null plan");
    qtng_ctx* ctx = plan->ctx;
    const HostPlan& hp = plan->hp;
    std::lock_guard<std::mutex> lk(ctx->mu);
    QTNG_CUDA(cudaSetDevice(ctx->device));
    ctx->ensure_arena(hp.arena_elems, elem_bytes(hp));
    if (!plan->graph || plan->graph_gen != ctx->arena_gen) {
      if (plan->graph) cudaGraphExecDestroy(plan->graph);
      plan->graph = nullptr;
      plan->graph = capture(ctx, [&] { enqueue_program(ctx, hp, plan->prog, ctx->arena.p, nullptr); });
      plan->graph_gen = ctx->arena_gen;
    }
    QTNG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    for (int i = 0; i < n_runs; ++i) QTNG_CUDA(cudaGraphLaunch(plan->graph, ctx->stream));
    g_launches.fetch_add(static_cast<uint64_t>(launches_per_run(hp)) * static_cast<uint64_t>(n_runs),
                         std::memory_order_relaxed);
    QTNG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    QTNG_CUDA(cudaStreamSynchronize(ctx->stream));
    float ms = 0.f;
    QTNG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    plan->last_ms = ms / std::max(1, n_runs);
    if (device_ms) *device_ms = ms;
  });
}

namespace {
void fill_info(const HostPlan& hp, int n_lightcones, qtng_plan_info* info) {
    info->n_lightcones = n_lightcones;
    info->n_levels = static_cast<int32_t>(hp.levels.size());
    info->n_buckets = hp.n_buckets;
    info->n_device_ops = hp.ops.size();
    info->max_width = hp.max_width;
    info->max_result_rank = hp.max_result_rank;
    info->alg_bytes = hp.alg_bytes;
    info->sum_ops = hp.sum_ops;
    info->arena_bytes = hp.arena_elems * sizeof(double2);
    info->desc_bytes = layout_of(hp).upload;
    info->kernels_per_run = launches_per_run(hp);
    info->n_segments = hp.segs.size();
    info->n_fused_ops = hp.n_fused_ops;
    info->dev_bytes = hp.dev_bytes;
    info->fp64_ops = hp.fp64_ops;
    info->seg_fp64_ops = hp.seg_fp64_ops;
    info->single_alg_bytes = hp.single_alg_bytes;
}
}  // namespace

qtng_status qtng_plan_info_get(const qtng_plan* plan, qtng_plan_info* info) {
  return guarded([&] {
    if (!plan || !info) throw Error(kInvalidInput, "null argument");
    fill_info(plan->hp, static_cast<int>(plan->edges.size()), info);
  });
}

qtng_status qtng_plan_segments(int n, int m, const int* edges, int p, int merged,
                               int max_result_width, int* ints, int64_t cap, int64_t* n_ints) {
  return guarded([&] {
    if (p < 1) throw Error(kInvalidInput, "angles: gammas and betas must have equal length p >= 1");
    const Graph g = graph_from(n, m, edges);
    const ConeSet cs = plan_cones(g, p, merged != 0, max_result_width, selection(m, m, nullptr));
    std::vector<const WalkResult*> ptrs;
    for (const WalkResult& w : cs.walks) {
      if (w.fail_code) throw Error(w.fail_code, w.fail_msg);
      ptrs.push_back(&w);
    }
    const HostPlan hp = build_plan(ptrs, static_cast<uint64_t>(n_gate_slots(p)) * kSlotElems, true, true);
    std::vector<int> out;
    for (size_t L = 0; L < hp.levels.size(); ++L)
      for (uint32_t k = 0; k < hp.levels[L].seg_count + hp.levels[L].seg4_count; ++k) {
        const DevSeg& sg = hp.segs[hp.levels[L].seg_begin + k];
        out.insert(out.end(), {static_cast<int>(L), sg.nst, sg.ry, sg.cy, sg.nops, sg.rb, sg.rb2});
        for (int i = 0; i < sg.nst; ++i) {
          const DevStage& st = hp.stages[sg.stage + i];
          out.insert(out.end(), {st.nt, st.ns, st.main == kSegMain ? -1 : st.main});
          for (int t = 0; t < st.nt; ++t) {
            const DevTensor& x = hp.trefs[sg.tref + st.op0 + t];
            out.push_back(x.rank);
            out.push_back(x.rank && x.off < hp.input_elems ? 1 : 0);
            for (int ax = 0; ax < x.rank; ++ax) out.push_back(x.src[ax]);
          }
        }
      }
    *n_ints = static_cast<int64_t>(out.size());
    if (static_cast<int64_t>(out.size()) <= cap) std::copy(out.begin(), out.end(), ints);
  });
}

qtng_status qtng_plan_stats(int n, int m, const int* edges, int p, int merged,
                            int max_result_width, int fuse, qtng_plan_info* info) {
  return guarded([&] {
    if (!info) throw Error(kInvalidInput, "null argument");
    if (p < 1) throw Error(kInvalidInput, "angles: gammas and betas must have equal length p >= 1");
    const Graph g = graph_from(n, m, edges);
    const ConeSet cs = plan_cones(g, p, merged != 0, max_result_width, selection(m, m, nullptr));
    std::vector<const WalkResult*> ptrs;
    for (size_t i = 0; i < cs.walks.size(); ++i) {
      if (cs.walks[i].fail_code)
        throw Error(kSchedule, "edge (" + std::to_string(cs.edges[i].u) + ", " +
                                   std::to_string(cs.edges[i].v) + "): " + cs.walks[i].fail_msg);
      ptrs.push_back(&cs.walks[i]);
    }
    const HostPlan hp =
        build_plan(ptrs, static_cast<uint64_t>(n_gate_slots(p)) * kSlotElems, fuse != 0, true);
    fill_info(hp, static_cast<int>(ptrs.size()), info);
  });
}

qtng_status qtng_statevector_energy(qtng_ctx* ctx, int n, int m, const int* edges, int p,
                                    const double* gammas, const double* betas, int cap,
                                    double* energy, double* zz_out) {
  return guarded([&] {
    if (!ctx || !energy) throw Error(kInvalidInput, "null argument");
    if (p < 1) throw Error(kInvalidInput, "angles: gammas and betas must have equal length p >= 1");
    const Graph g = graph_from(n, m, edges);
    // StateVector::plus_state (proj/src/statevector.cpp:9-17)
    if (n < 1) throw Error(kInvalidInput, "state vector needs at least one qubit");
    if (n > cap)
      throw Error(kResource, "state vector of " + std::to_string(n) + " qubits exceeds cap " +
                                 std::to_string(cap));
    if (n > 33) throw Error(kResource, "state vector of " + std::to_string(n) +
                                           " qubits exceeds the device limit 33");
    const int me = static_cast<int>(g.edges.size());
    std::vector<int2> bits(me);
    for (int e = 0; e < me; ++e) bits[e] = int2{n - 1 - g.edges[e].u, n - 1 - g.edges[e].v};
    std::vector<double2> w(p), c(p), ms(p);
    for (int k = 0; k < p; ++k) {  // the reference's gate values (statevector.cpp:29,37-38)
      const std::complex<double> wk = std::exp(std::complex<double>{0.0, -gammas[k]});
      w[k] = double2{wk.real(), wk.imag()};
      c[k] = double2{std::cos(betas[k]), 0.0};
      ms[k] = double2{0.0, -std::sin(betas[k])};
    }
    const double amp0 = 1.0 / std::sqrt(static_cast<double>(uint64_t{1} << n));
    std::lock_guard<std::mutex> lk(ctx->mu);
    QTNG_CUDA(cudaSetDevice(ctx->device));
    ctx->ensure_arena(uint64_t{1} << n);
    ctx->sv_scratch.ensure(sv_scratch_bytes(std::max(me, 1)));
    char* scr = static_cast<char*>(ctx->sv_scratch.p);
    if (me)
      QTNG_CUDA(cudaMemcpyAsync(scr, bits.data(), sizeof(int2) * me, cudaMemcpyHostToDevice,
                                ctx->stream));
    double* zz_dev = reinterpret_cast<double*>(scr + sizeof(int2) * me);
    QTNG_CUDA(sv_run(ctx->stream, ctx->A(), n, me, reinterpret_cast<const int2*>(scr), p, w.data(),
                     c.data(), ms.data(), amp0, scr, zz_dev));
    std::vector<double> zz(me);
    if (me)
      QTNG_CUDA(cudaMemcpyAsync(zz.data(), zz_dev, sizeof(double) * me, cudaMemcpyDeviceToHost,
                                ctx->stream));
    QTNG_CUDA(cudaStreamSynchronize(ctx->stream));
    // expectation_cost (statevector.cpp:86-90): m/2 - 1/2 sum, edge order
    double sum = 0.0;
    for (double x : zz) sum += x;
    *energy = 0.5 * static_cast<double>(me) - 0.5 * sum;
    if (zz_out) std::copy(zz.begin(), zz.end(), zz_out);
  });
}

qtng_status qtng_plan_records(const qtng_plan* plan, qtng_record* records, int64_t cap,
                              int64_t* n_out) {
  return guarded([&] {
    if (!plan) throw Error(kInvalidInput, "null plan");
    const HostPlan& hp = plan->hp;
    const int64_t n = static_cast<int64_t>(hp.rec_seq.size());
    if (n_out) *n_out = n;
    for (size_t c = 0; c + 1 < hp.rec_begin.size(); ++c)
      for (uint32_t i = hp.rec_begin[c]; i < hp.rec_begin[c + 1] && i < cap; ++i) {
        qtng_record& r = records[i];
        r.edge_u = plan->edges[c].u;
        r.edge_v = plan->edges[c].v;
        r.bucket_seq = hp.rec_seq[i];
        r.width = hp.rec_width[i];
        r.ops = uint64_t{1} << r.width;
        const int L = hp.rec_level[i];
        double share, ms;
        if (plan->profiled) {  // the bucket's byte share of its level's measured time
          share = hp.level_bytes[L] > 0 ? hp.rec_bytes[i] / hp.level_bytes[L] : 0;
          ms = plan->level_ms[L];
        } else {  // ... of the whole program's (graph replay)
          share = hp.alg_bytes > 0 ? hp.rec_bytes[i] / hp.alg_bytes : 0;
          ms = plan->last_ms;
        }
        r.elapsed_s = std::max(1e-9, 1e-3 * ms * share);
        r.flops_est = 8.0 * static_cast<double>(r.ops) / r.elapsed_s;
      }
  });
}

qtng_status qtng_plan_kernel_ms(const qtng_plan* plan, float* ms4, float* per_level, int cap) {
  return guarded([&] {
    if (!plan || !ms4) throw Error(kInvalidInput, "null argument");
    for (int k = 0; k < 4; ++k) ms4[k] = plan->kernel_ms[k];
    if (per_level)
      for (int i = 0; i < cap && i < static_cast<int>(plan->level_kernel_ms.size()); ++i)
        per_level[i] = plan->level_kernel_ms[i];
  });
}

qtng_status qtng_plan_level_ms(const qtng_plan* plan, float* ms, int cap) {
  return guarded([&] {
    if (!plan) throw Error(kInvalidInput, "null plan");
    for (int i = 0; i < cap && i < static_cast<int>(plan->level_ms.size()); ++i) ms[i] = plan->level_ms[i];
  });
}

void qtng_plan_destroy(qtng_plan* plan) {
  if (!plan) return;
  qtng_ctx* ctx = plan->ctx;
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    cudaSetDevice(ctx->device);
    delete plan;
  }
  ctx_release(ctx);  // the plan's reference
}

qtng_status qtng_plan_time_level(qtng_plan* plan, int level, int n_runs, int* level_out,
                                 double* level_bytes, float* mean_ms) {
  return guarded([&] {
    if (!plan) throw Error(kInvalidInput, "null plan");
    const HostPlan& hp = plan->hp;
    if (hp.levels.empty()) throw Error(kInvalidInput, "empty plan");
    if (level < 0) {  // the level holding the widest bucket
      int best = 0;
      for (size_t i = 0; i < hp.rec_width.size(); ++i)
        if (hp.rec_width[i] > hp.rec_width[best]) best = static_cast<int>(i);
      level = hp.rec_level[best];
    }
    if (level >= static_cast<int>(hp.levels.size())) throw Error(kInvalidInput, "level out of range");
    qtng_ctx* ctx = plan->ctx;
    std::lock_guard<std::mutex> lk(ctx->mu);
    QTNG_CUDA(cudaSetDevice(ctx->device));
    ctx->ensure_arena(hp.arena_elems, elem_bytes(hp));
    enqueue_level(ctx, hp.levels[level], level, plan->prog, ctx->arena.p);  // warm-up
    QTNG_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    for (int i = 0; i < n_runs; ++i) enqueue_level(ctx, hp.levels[level], level, plan->prog, ctx->arena.p);
    QTNG_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    QTNG_CUDA(cudaStreamSynchronize(ctx->stream));
    float ms = 0.f;
    QTNG_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    *level_out = level;
    *level_bytes = hp.level_bytes[level];
    *mean_ms = ms / std::max(1, n_runs);
  });
}

// ---------------------------------------------------------------- energy (end to end)

}  // extern "C"

namespace {

// One device's share of energy_expectation (engine.cpp:503-563): the terms,
// refusals and report data of the selected lightcones.
struct EnergyRun {
  std::vector<double> t;          // (re, im) per selected edge, selection order
  std::vector<std::string> fail;  // per selected edge: refusal message ("" = contracted)
  std::vector<Edge> edge_at;
  uint64_t peak = 0;              // max over lightcones of 16 << largest result rank
  int merges_applied = 0, merges_skipped = 0;
  float device_ms = 0.f;          // device span: first lane's program start to the last end
  std::vector<qtng_record> recs;  // want_records: one per contracted bucket, selection order
};

// On an error path, every lane already enqueued is synchronised before the
// context lock is released: its copies and kernels still use the lane buffers.
struct LaneGuard {
  qtng_ctx* ctx;
  int n = 0;
  ~LaneGuard() {
    for (int c = 0; c < n; ++c) cudaStreamSynchronize(ctx->lane[c].s);
  }
};

// Upload + run + copy back one lightcone chunk on lane `la` (all asynchronous).
void enqueue_energy_chunk_timed(qtng_ctx* ctx, Lane& la, bool lane0, const HostPlan& hp,
                                const double* table, double2* full) {
  const DescLayout L = layout_of(hp);
  const size_t eb = elem_bytes(hp);
  const uint64_t elems = std::max(hp.arena_elems, hp.input_elems);
  if (lane0) {
    ctx->ensure_arena(elems, eb);
  } else if (std::max<uint64_t>(elems, 32) * eb > la.arena->cap) {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    if (std::max<uint64_t>(elems, 32) * eb > free_b + la.arena->cap)
      throw Error(kResource, "device arena of " + std::to_string(elems * eb) +
                                 " bytes exceeds free HBM (" + std::to_string(free_b) + ")");
    QTNG_CUDA(cudaStreamSynchronize(la.s));
    la.arena->ensure(std::max<uint64_t>(elems, 32) * eb);
  }
  la.desc->ensure(L.total);
  la.pin_in->ensure(std::max<uint64_t>(hp.input_elems, 1) * eb);
  stage_input(hp, table, hp.input_elems, la.pin_in->p);
  QTNG_CUDA(cudaMemcpyAsync(la.arena->p, la.pin_in->p, hp.input_elems * eb, cudaMemcpyHostToDevice,
                            la.s));
  upload_desc(ctx, hp, L, static_cast<char*>(la.desc->p), &la);
  const DevProgram pr{static_cast<char*>(la.desc->p), L, hp.c64};
  QTNG_CUDA(cudaEventRecord(la.t0, la.s));
  enqueue_program(ctx, hp, pr, la.arena->p, nullptr, nullptr, &la, full);
  QTNG_CUDA(cudaEventRecord(la.t1, la.s));
  const size_t nb = (hp.lc_begin.size() - 1) * sizeof(double2);
  la.pin_out->ensure(std::max<size_t>(nb, 16));
  QTNG_CUDA(cudaMemcpyAsync(la.pin_out->p, pr.terms(), nb, cudaMemcpyDeviceToHost, la.s));
}

// The selected lightcones `s` on ctx: host planning of chunk c+1 overlaps the
// device work of chunks <= c (K lanes, QTNG_PIPELINE).  full (optional,
// device, 2 doubles per graph edge, zeroed here): every contracted term is also
// written to its edge slot (the multi-GPU reduce vector).  Refusals are
// returned in `out.fail`, not thrown.
void energy_run(qtng_ctx* ctx, const Graph& g, int p, const double* gammas, const double* betas,
                bool merged, int max_result_width, int prec, const std::vector<int>& s,
                bool want_records, double2* full, EnergyRun& out) {
  PhaseTimer tm("qtng_energy");
  static const int lanes = [] {
    const char* v = std::getenv("QTNG_PIPELINE");  // lanes (1 = no pipelining)
    const int x = v ? std::atoi(v) : 3;
    return std::max(1, std::min(x, qtng_ctx::kLanes));
  }();
  const int K = std::max(1, std::min<int>(lanes, static_cast<int>(s.size()) / 4));
  // QTNG_PIPELINE_ORDER=0 (default): chunk c = every K-th lightcone, each
  // chunk's schedules built just before it is planned.  1: every schedule and
  // walk first (host threads), then chunks by decreasing predicted work (the
  // heaviest lightcones enqueued first).  Measured on C2: 3.64 vs 3.57 ms --
  // the device is throughput-bound once started, so starting it early wins.
  static const int order_mode = [] {
    const char* v = std::getenv("QTNG_PIPELINE_ORDER");
    return v ? std::atoi(v) : 0;
  }();
  std::vector<std::vector<int>> pos(K), part(K);  // positions in s, edge indices
  ConeSet all;
  if (order_mode == 1 && K > 1) {
    all = plan_cones(g, p, merged, max_result_width, s);
    tm.mark("schedules+walks (all)");
    std::vector<double> work(s.size(), 0.0);
    double total = 0.0;
    for (size_t i = 0; i < s.size(); ++i) {
      for (const Op& op : all.walks[i].ops)
        work[i] += std::ldexp(1.0, op.width) * std::max(1, op.nin - 1);
      total += work[i];
    }
    std::vector<int> ord(s.size());
    for (size_t i = 0; i < s.size(); ++i) ord[i] = static_cast<int>(i);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return work[a] > work[b]; });
    // chunk c closes when the cumulative work reaches 1 - 2^-(c+1) of the total
    double acc = 0.0;
    int c = 0;
    for (int i : ord) {
      pos[c].push_back(i);
      part[c].push_back(s[i]);
      acc += work[i];
      while (c + 1 < K && acc >= total * (1.0 - std::ldexp(1.0, -(c + 1))) &&
             static_cast<int>(pos[c].size()) >= 1)
        ++c;
    }
  } else {
    // QTNG_PIPELINE_SPLIT="f0,f1,...": chunk c takes a fraction f_c of the
    // lightcones (default 1/K each), chunks interleaving the selection: the
    // device starts once chunk 0 is planned, and the last chunk's own
    // latency chain runs after the host has planned it.
    static const std::vector<double> split = [] {
      std::vector<double> f;
      if (const char* v = std::getenv("QTNG_PIPELINE_SPLIT"))
        for (const char* q = v; *q;) {
          char* e = nullptr;
          const double x = std::strtod(q, &e);
          if (e == q) break;
          f.push_back(x);
          q = *e == ',' ? e + 1 : e;
        }
      return f;
    }();
    const size_t n = s.size();
    std::vector<double> want(K, 1.0 / K);
    if (static_cast<int>(split.size()) == K) {
      double t = 0.0;
      for (double x : split) t += std::max(x, 0.0);
      if (t > 0.0)
        for (int c = 0; c < K; ++c) want[c] = std::max(split[c], 0.0) / t;
    }
    // largest-deficit assignment in selection order: chunk c receives about
    // want[c] * n lightcones, spread evenly over the selection
    std::vector<double> got(K, 0.0);
    for (size_t i = 0; i < n; ++i) {
      int c = 0;
      double best = -1e300;
      for (int k = 0; k < K; ++k) {
        const double d = want[k] * static_cast<double>(i + 1) - got[k];
        if (d > best + 1e-12) best = d, c = k;
      }
      got[c] += 1.0;
      pos[c].push_back(static_cast<int>(i));
      part[c].push_back(s[i]);
    }
  }
  std::vector<ConeSet> cs(K);
  std::vector<HostPlan> hps(K);
  std::vector<std::vector<int>> okpos(K);  // positions (in s) of the contracted lightcones
  out.t.assign(2 * s.size(), 0.0);
  out.fail.assign(s.size(), std::string());
  out.edge_at.assign(s.size(), Edge{});
  std::vector<double> table;
  std::unique_lock<std::mutex> lk(ctx->mu, std::defer_lock);
  LaneGuard guard{ctx, 0};
  // chunk c's upload + launches run on the context's enqueue thread while
  // this thread plans chunk c + 1; every exit waits for it before the lane
  // guard synchronises (declared after the guard: destroyed first)
  struct EnqDrain {
    qtng::Worker* w = nullptr;
    ~EnqDrain() {
      if (w) try { w->wait(); } catch (...) {}
    }
  } drain;
  for (int c = 0; c < K; ++c) {
    if (pos[c].empty()) continue;
    const bool pre = order_mode == 1 && K > 1;
    if (!pre) cs[c] = plan_cones(g, p, merged, max_result_width, part[c]);
    std::vector<const WalkResult*> ok;
    for (size_t k = 0; k < pos[c].size(); ++k) {
      const int at = pos[c][k];
      const WalkResult& w = pre ? all.walks[at] : cs[c].walks[k];
      out.edge_at[at] = pre ? all.edges[at] : cs[c].edges[k];
      out.merges_applied += pre ? all.merges_applied[at] : cs[c].merges_applied[k];
      out.merges_skipped += pre ? all.merges_skipped[at] : cs[c].merges_skipped[k];
      if (w.fail_code) {
        out.fail[at] = w.fail_msg.empty() ? std::string("refused") : w.fail_msg;
      } else {
        ok.push_back(&w);
        okpos[c].push_back(at);
        if (!w.ops.empty()) out.peak = std::max(out.peak, uint64_t{16} << w.max_result_rank);
      }
    }
    tm.mark("schedules+walks");
    if (ok.empty()) continue;
    hps[c] = build_plan(ok, static_cast<uint64_t>(n_gate_slots(p)) * kSlotElems, fuse_default(), true,
                        flow_default(), /*stats=*/false, /*records=*/want_records);
    hps[c].c64 = prec == 64;
    for (size_t k = 0; k < okpos[c].size(); ++k) hps[c].lc_edge[k] = s[okpos[c][k]];
    tm.mark("build_plan");
    if (table.empty()) {
      table.resize(2 * hps[c].input_elems);
      fill_gate_table(p, gammas, betas, table.data());
    }
    if (!lk.owns_lock()) {
      lk.lock();
      QTNG_CUDA(cudaSetDevice(ctx->device));
      if (full) {  // before any lane's final kernel can write its slots
        QTNG_CUDA(cudaMemsetAsync(full, 0, static_cast<size_t>(g.edges.size()) * sizeof(double2),
                                  ctx->lane[0].s));
        QTNG_CUDA(cudaStreamSynchronize(ctx->lane[0].s));
      }
    }
    guard.n = c + 1;
    if (K > 1) {
      if (!ctx->enq) ctx->enq = std::make_unique<qtng::Worker>();
      drain.w = ctx->enq.get();
      const HostPlan* hp = &hps[c];
      const double* tb = table.data();
      drain.w->submit([ctx, c, hp, tb, full] {
        QTNG_CUDA(cudaSetDevice(ctx->device));
        enqueue_energy_chunk_timed(ctx, ctx->lane[c], c == 0, *hp, tb, full);
      });
    } else {
      enqueue_energy_chunk_timed(ctx, ctx->lane[c], c == 0, hps[c], table.data(), full);
    }
    tm.mark("upload+enqueue");
  }
  if (drain.w) drain.w->wait();  // rethrows an enqueue failure
  tm.mark("enqueue wait");
  std::vector<float> lane_ms(K, 0.f);
  int first = -1;
  for (int c = 0; c < K; ++c) {
    if (okpos[c].empty()) continue;
    if (first < 0) first = c;
    QTNG_CUDA(cudaStreamSynchronize(ctx->lane[c].s));
    QTNG_CUDA(cudaEventElapsedTime(&lane_ms[c], ctx->lane[c].t0, ctx->lane[c].t1));
    float span = 0.f;  // the lanes overlap: the span from the first start
    QTNG_CUDA(cudaEventElapsedTime(&span, ctx->lane[first].t0, ctx->lane[c].t1));
    out.device_ms = std::max(out.device_ms, span);
    const double* o = static_cast<const double*>(ctx->lane[c].pin_out->p);
    for (size_t k = 0; k < okpos[c].size(); ++k) {
      out.t[2 * okpos[c][k]] = o[2 * k];
      out.t[2 * okpos[c][k] + 1] = o[2 * k + 1];
    }
  }
  guard.n = 0;
  tm.mark("device+d2h");
  if (!want_records) return;
  // TimingRecords (engine.cpp:275-282), selection order: elapsed_s is the
  // bucket's share (by algorithmic bytes) of its lane's measured device time
  // -- a fused level kernel runs hundreds of buckets at once, so per-bucket
  // device times do not exist.
  std::vector<std::pair<int, int>> at_of(s.size(), {-1, -1});  // position -> (chunk, lightcone)
  for (int c = 0; c < K; ++c)
    for (size_t k = 0; k < okpos[c].size(); ++k) at_of[okpos[c][k]] = {c, static_cast<int>(k)};
  std::vector<double> chunk_bytes(K, 0.0);
  for (int c = 0; c < K; ++c)
    for (double b : hps[c].rec_bytes) chunk_bytes[c] += b;
  for (size_t i = 0; i < s.size(); ++i) {
    const auto [c, k] = at_of[i];
    if (c < 0) continue;
    const HostPlan& hp = hps[c];
    for (uint32_t r = hp.rec_begin[k]; r < hp.rec_begin[k + 1]; ++r) {
      qtng_record q{};
      q.edge_u = out.edge_at[i].u;
      q.edge_v = out.edge_at[i].v;
      q.bucket_seq = hp.rec_seq[r];
      q.width = hp.rec_width[r];
      q.ops = uint64_t{1} << q.width;
      const double share = chunk_bytes[c] > 0 ? hp.rec_bytes[r] / chunk_bytes[c] : 0.0;
      q.elapsed_s = std::max(1e-9, 1e-3 * lane_ms[c] * share);
      q.flops_est = 8.0 * static_cast<double>(q.ops) / q.elapsed_s;
      out.recs.push_back(q);
    }
  }
}

// energy_expectation's failure rule (engine.cpp:517-519, 543-546): the first
// refused or non-real lightcone in order raises ScheduleError("edge (u, v): ...").
void raise_first_failure(const std::vector<std::string>& fail, const std::vector<Edge>& edge_at,
                         const std::vector<double>& t, double tol) {
  for (size_t i = 0; i < fail.size(); ++i) {
    const bool refused = !fail[i].empty();
    const bool complex_term = !refused && std::abs(t[2 * i + 1]) > tol;
    if (refused || complex_term) {
      const std::string what = refused ? fail[i]
                                       : "edge term has non-real value: imag = " +
                                             std::to_string(t[2 * i + 1]);
      throw Error(kSchedule, "edge (" + std::to_string(edge_at[i].u) + ", " +
                                 std::to_string(edge_at[i].v) + "): " + what);
    }
  }
}

bool selects_all_in_order(const std::vector<int>& s, int m) {
  if (static_cast<int>(s.size()) != m) return false;
  for (int i = 0; i < m; ++i)
    if (s[i] != i) return false;
  return true;
}

void fill_report(const EnergyRun& r, qtng_energy_report* rep) {
  if (!rep) return;
  rep->n_records = static_cast<int64_t>(r.recs.size());
  rep->peak_tensor_bytes = r.peak;
  rep->merges_applied = r.merges_applied;
  rep->merges_skipped = r.merges_skipped;
  rep->device_ms = r.device_ms;
  if (rep->records)
    for (int64_t i = 0; i < rep->rec_cap && i < rep->n_records; ++i) rep->records[i] = r.recs[i];
}

}  // namespace

extern "C" {

qtng_status qtng_energy(qtng_ctx* ctx, int n, int m, const int* edges, int p,
                        const double* gammas, const double* betas, int merged,
                        int max_result_width, int precision, int n_sel, const int* sel,
                        double* energy, double* terms, qtng_energy_report* report) {
  return guarded([&] {
    if (!ctx) throw Error(kInvalidInput, "null context");
    validate_angles(p, gammas, betas);
    const int prec = resolve_prec(ctx, precision);
    const Graph g = graph_from(n, m, edges);
    const std::vector<int> s = selection(m, n_sel, sel);
    EnergyRun r;
    energy_run(ctx, g, p, gammas, betas, merged != 0, max_result_width, prec, s,
               report && report->records, nullptr, r);
    raise_first_failure(r.fail, r.edge_at, r.t, imag_tol(prec == 64));
    double sum = 0.0;  // edge order, like engine.cpp:549-551
    for (size_t i = 0; i < s.size(); ++i) sum += r.t[2 * i];
    // a partial selection has no energy (its terms are the result)
    if (energy)
      *energy = selects_all_in_order(s, m) ? 0.5 * static_cast<double>(m) - 0.5 * sum
                                           : std::numeric_limits<double>::quiet_NaN();
    if (terms) std::copy(r.t.begin(), r.t.end(), terms);
    fill_report(r, report);
  });
}

}  // extern "C"

// ---------------------------------------------------------------- multi-GPU driver

namespace {

// NCCL, resolved at first use (the library is loaded by soname, so a process
// that already holds torch's NCCL shares it; nothing links against it).
struct NcclApi {
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclReduce) reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string missing;

  static const NcclApi& get() {
    static const NcclApi api = [] {
      NcclApi a;
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) {
        a.missing = std::string("NCCL unavailable: ") + dlerror();
        return a;
      }
      a.init_all = reinterpret_cast<decltype(a.init_all)>(dlsym(h, "ncclCommInitAll"));
      a.reduce = reinterpret_cast<decltype(a.reduce)>(dlsym(h, "ncclReduce"));
      a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
      a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
      a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
      if (!a.init_all || !a.reduce || !a.group_start || !a.group_end || !a.error_string)
        a.missing = "NCCL unavailable: missing symbols in libnccl.so.2";
      return a;
    }();
    if (!api.missing.empty()) throw Error(kCuda, api.missing);
    return api;
  }
};

#define QTNG_NCCL(api, call)                                                        \
  do {                                                                              \
    const ncclResult_t r_ = (call);                                                 \
    if (r_ != ncclSuccess) throw Error(kCuda, std::string(#call) + ": " + (api).error_string(r_)); \
  } while (0)

// One communicator set per device list, created on first use and kept for
// the life of the process (ncclCommInitAll costs far more than an energy).
std::vector<ncclComm_t> comms_for(const std::vector<int>& devs) {
  static std::mutex mu;
  static std::map<std::vector<int>, std::vector<ncclComm_t>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(devs);
  if (it != cache.end()) return it->second;
  const NcclApi& nc = NcclApi::get();
  std::vector<ncclComm_t> c(devs.size());
  QTNG_NCCL(nc, nc.init_all(c.data(), static_cast<int>(devs.size()), devs.data()));
  cache[devs] = c;
  return c;
}

// LPT (longest processing time first) placement of the lightcones on
// n_shards devices by predicted work (qtng_edge_work): edges by decreasing
// work (ties: lower index) onto the least-loaded shard (ties: lower shard).
std::vector<int> lpt_owner(const std::vector<double>& work, int n_shards) {
  const int m = static_cast<int>(work.size());
  std::vector<int> order(m);
  for (int i = 0; i < m; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return work[a] > work[b]; });
  std::vector<double> load(n_shards, 0.0);
  std::vector<int> owner(m, 0);
  for (int i : order) {
    const int r = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
    owner[i] = r;
    load[r] += work[i];
  }
  return owner;
}

std::vector<double> predicted_work(const Graph& g, int p, bool merged) {
  const int m = static_cast<int>(g.edges.size());
  const ConeSet cs = plan_cones(g, p, merged, 1 << 20, selection(m, m, nullptr));
  std::vector<double> work(m, 0.0);
  for (int i = 0; i < m; ++i)
    for (const Op& op : cs.walks[i].ops)  // the reference loop's complex products + additions
      work[i] += std::ldexp(1.0, op.width) * std::max(1, op.nin - 1) +
                 std::ldexp(1.0, op.r) * (std::ldexp(1.0, op.ns) - 1.0);
  return work;
}

// The placement of a graph's lightcones on n_shards devices, cached per
// (edges, p, merged, n_shards): an optimiser calls the energy of one graph
// again and again with new angles, and the prediction costs a host planning
// pass.  One device needs no prediction.
std::vector<int> placement(const Graph& g, int p, bool merged, int n_shards) {
  const int m = static_cast<int>(g.edges.size());
  if (n_shards == 1) return std::vector<int>(m, 0);
  static std::mutex mu;
  static std::map<std::vector<int>, std::vector<int>> cache;
  std::vector<int> key = {g.n, p, merged ? 1 : 0, n_shards};
  for (const Edge& e : g.edges) {
    key.push_back(e.u);
    key.push_back(e.v);
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  std::vector<int> o = lpt_owner(predicted_work(g, p, merged), n_shards);
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() > 64) cache.clear();
  cache[key] = o;
  return o;
}

}  // namespace

extern "C" {

qtng_status qtng_shard_edges(int n, int m, const int* edges, int p, int merged, int n_shards,
                             int* owner) {
  return guarded([&] {
    if (n_shards < 1 || !owner) throw Error(kInvalidInput, "invalid shard count");
    const Graph g = graph_from(n, m, edges);
    const std::vector<int> o = lpt_owner(predicted_work(g, p, merged != 0), n_shards);
    std::copy(o.begin(), o.end(), owner);
  });
}

qtng_status qtng_energy_multi(qtng_ctx* const* ctxs, int n_ctx, int n, int m, const int* edges,
                              int p, const double* gammas, const double* betas, int merged,
                              int max_result_width, int precision, double* energy, double* terms,
                              float* shard_ms) {
  return guarded([&] {
    if (!ctxs || n_ctx < 1) throw Error(kInvalidInput, "no contexts");
    std::vector<int> devs(n_ctx);
    for (int i = 0; i < n_ctx; ++i) {
      if (!ctxs[i]) throw Error(kInvalidInput, "null context");
      devs[i] = ctxs[i]->device;
      for (int j = 0; j < i; ++j)
        if (devs[j] == devs[i]) throw Error(kInvalidInput, "contexts must be on distinct devices");
    }
    validate_angles(p, gammas, betas);
    const int prec = resolve_prec(ctxs[0], precision);
    const Graph g = graph_from(n, m, edges);
    const std::vector<int> owner = placement(g, p, merged != 0, n_ctx);
    std::vector<std::vector<int>> shard(n_ctx);
    for (int i = 0; i < m; ++i) shard[owner[i]].push_back(i);  // ascending edge order
    for (int r = 0; r < n_ctx; ++r) {
      std::lock_guard<std::mutex> lk(ctxs[r]->mu);
      QTNG_CUDA(cudaSetDevice(ctxs[r]->device));
      ctxs[r]->multi_full.ensure(std::max<size_t>(1, m) * sizeof(double2));
    }
    // one host thread per device: plan + contract the shard, terms scattered
    // into the device's reduce vector by the final kernel
    std::vector<EnergyRun> runs(n_ctx);
    std::vector<std::exception_ptr> errs(n_ctx);
    auto work = [&](int r) {
      try {
        if (shard[r].empty()) {  // nothing to contract: a zero vector joins the reduce
          std::lock_guard<std::mutex> lk(ctxs[r]->mu);
          QTNG_CUDA(cudaSetDevice(ctxs[r]->device));
          QTNG_CUDA(cudaMemset(ctxs[r]->multi_full.p, 0, std::max<size_t>(1, m) * sizeof(double2)));
          return;
        }
        energy_run(ctxs[r], g, p, gammas, betas, merged != 0, max_result_width, prec, shard[r],
                   false, static_cast<double2*>(ctxs[r]->multi_full.p), runs[r]);
      } catch (...) {
        errs[r] = std::current_exception();
      }
    };
    std::vector<std::thread> th;
    for (int r = 1; r < n_ctx; ++r) th.emplace_back(work, r);
    work(0);
    for (std::thread& t : th) t.join();
    for (const std::exception_ptr& e : errs)
      if (e) std::rethrow_exception(e);
    // the single collective: sum-reduce the 2m-double vectors onto ctxs[0]
    const std::vector<ncclComm_t> comms = comms_for(devs);
    const NcclApi& nc = NcclApi::get();
    std::vector<std::unique_lock<std::mutex>> locks;
    std::vector<int> by_addr(n_ctx);
    for (int r = 0; r < n_ctx; ++r) by_addr[r] = r;
    std::sort(by_addr.begin(), by_addr.end(), [&](int a, int b) { return ctxs[a] < ctxs[b]; });
    for (int r : by_addr) locks.emplace_back(ctxs[r]->mu);  // fixed order: no deadlock
    QTNG_NCCL(nc, nc.group_start());
    for (int r = 0; r < n_ctx; ++r) {
      QTNG_CUDA(cudaSetDevice(ctxs[r]->device));
      void* buf = ctxs[r]->multi_full.p;
      QTNG_NCCL(nc, nc.reduce(buf, buf, 2 * static_cast<size_t>(m), ncclFloat64, ncclSum, 0,
                              comms[r], ctxs[r]->stream));
    }
    QTNG_NCCL(nc, nc.group_end());
    std::vector<double> full(2 * static_cast<size_t>(m), 0.0);
    QTNG_CUDA(cudaSetDevice(ctxs[0]->device));
    if (m > 0)
      QTNG_CUDA(cudaMemcpyAsync(full.data(), ctxs[0]->multi_full.p, full.size() * sizeof(double),
                                cudaMemcpyDeviceToHost, ctxs[0]->stream));
    for (int r = 0; r < n_ctx; ++r) {
      QTNG_CUDA(cudaSetDevice(ctxs[r]->device));
      QTNG_CUDA(cudaStreamSynchronize(ctxs[r]->stream));
    }
    locks.clear();
    // failures and terms in edge order (engine.cpp:543-551)
    std::vector<std::string> fail(m);
    std::vector<Edge> edge_at(g.edges.begin(), g.edges.end());
    for (int r = 0; r < n_ctx; ++r)
      for (size_t k = 0; k < runs[r].fail.size(); ++k) fail[shard[r][k]] = runs[r].fail[k];
    raise_first_failure(fail, edge_at, full, imag_tol(prec == 64));
    double sum = 0.0;
    for (int i = 0; i < m; ++i) sum += full[2 * i];
    if (energy) *energy = 0.5 * static_cast<double>(m) - 0.5 * sum;
    if (terms) std::copy(full.begin(), full.end(), terms);
    if (shard_ms)
      for (int r = 0; r < n_ctx; ++r) shard_ms[r] = runs[r].device_ms;
  });
}

qtng_status qtng_fp64_peak(int device, double* mul_add_ops_per_s, double* fma_flops_per_s) {
  return guarded([&] {
    if (!mul_add_ops_per_s || !fma_flops_per_s) throw Error(kInvalidInput, "null argument");
    QTNG_CUDA(fp64_peak(device, mul_add_ops_per_s, fma_flops_per_s));
  });
}

qtng_status qtng_plan_terms(qtng_plan* plan, double* terms) {
  return guarded([&] {
    if (!plan || !terms) throw Error(kInvalidInput, "null argument");
    qtng_ctx* ctx = plan->ctx;
    std::lock_guard<std::mutex> lk(ctx->mu);
    QTNG_CUDA(cudaSetDevice(ctx->device));
    const size_t nb = plan->edges.size() * sizeof(double2);
    QTNG_CUDA(cudaMemcpyAsync(plan->pin_terms.p, plan->prog.terms(), nb, cudaMemcpyDeviceToHost,
                              ctx->stream));
    QTNG_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(terms, plan->pin_terms.p, nb);
  });
}

}  // extern "C"
