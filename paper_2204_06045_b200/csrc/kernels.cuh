// Launch interface of the sm_100a bucket kernels (kernels.cu).  kernels.cu is
// compiled twice: namespace qtng::c128 (complex128, bit-exact to the
// reference) and qtng::c64 (complex64 mode, -DQTNG_C64=1).  `arena` points at
// the context arena holding double2 (c128) or float2 (c64) elements.
#pragma once

#include <cuda_runtime.h>

#include "device_plan.hpp"

#if defined(QTNG_C64) && QTNG_C64
#define QTNG_PREC_NS c64
#else
#define QTNG_PREC_NS c128
#endif

namespace qtng {

#define QTNG_KERNEL_API                                                                        \
  /* CTAs (256 threads) a level launch with `items` warp work items uses */                   \
  int level_grid(uint32_t items);                                                              \
  /* one level: every single-op bucket of the level, all lightcones at once */                \
  cudaError_t launch_level(cudaStream_t s, const DevOp* ops, const uint32_t* ibeg,             \
                           const DevTensor* trefs, void* arena, const LevelLaunch& lv);        \
  /* the level's outer-join ops, concurrent with launch_level on a second stream */            \
  cudaError_t launch_outer(cudaStream_t s, const DevOp* ops, const uint32_t* ibeg,             \
                           const DevTensor* trefs, void* arena, const LevelLaunch& lv);        \
  /* the level's fused-chain segments (seg_kernel), concurrent with the others */              \
  cudaError_t launch_segs(cudaStream_t s, const DevSeg* segs, const uint32_t* seg_ibeg,        \
                          const DevStage* stages, const DevTensor* trefs,                     \
                          const SegOpTab* segtab, void* arena, uint32_t* ctr,                  \
                          const LevelLaunch& lv);                                              \
  /* the level's quad-tile segments (seg4_kernel), concurrent with the others; */            \
  /* ctr: its own queue counters */                                                            \
  cudaError_t launch_segs4(cudaStream_t s, const DevSeg* segs, const uint32_t* seg_ibeg,       \
                           const DevStage* stages, const DevTensor* trefs,                    \
                           const SegOpTab* segtab, void* arena, uint32_t* ctr,                 \
                           const LevelLaunch& lv);                                             \
  /* the segments' SegOpTab entries (once per descriptor upload) */                           \
  cudaError_t launch_seg_prep(cudaStream_t s, const DevSeg* segs, uint32_t n_segs,             \
                              const DevTensor* trefs, SegOpTab* segtab);                       \
  /* a whole dataflow program in one persistent kernel (after its state reset) */             \
  cudaError_t launch_flow(cudaStream_t s, const FlowUnit* units, uint32_t n_units,             \
                          const uint64_t* init, uint32_t n_init, uint32_t n_chunks,           \
                          const DevOp* ops, const DevSeg* segs, const DevStage* stages,       \
                          const DevTensor* trefs, const SegOpTab* segtab, void* arena,        \
                          uint32_t* done, int32_t* deps, uint64_t* queue, FlowState* st);      \
  /* resident warps of the level kernel on the current device */                              \
  int resident_warps();                                                                        \
  /* per lightcone: e_jk = prod of its scalar results in production order (complex128); */   \
  /* full (optional): also written to full[lc_edge[i]] (the multi-GPU reduce vector) */       \
  cudaError_t launch_final(cudaStream_t s, const uint64_t* scalar_off, const uint32_t* lc_begin, \
                           int n_lc, const void* arena, double2* terms,                       \
                           const int32_t* lc_edge, double2* full);

namespace c128 {
QTNG_KERNEL_API
}  // namespace c128
namespace c64 {
QTNG_KERNEL_API
}  // namespace c64

// Number of kernels launched per plan execution (level kernels, outer-join
// kernels, segment kernels, quad segment kernels, final).
inline int kernels_per_plan(int n_level_launches, int n_outer_launches, int n_seg_launches,
                            int n_seg4_launches = 0) {
  return n_level_launches + n_outer_launches + n_seg_launches + n_seg4_launches + 1;
}

}  // namespace qtng
