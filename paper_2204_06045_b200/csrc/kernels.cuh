// Launch interface of the sm_100a bucket kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "device_plan.hpp"

namespace qtng {

// Number of CTAs (256 threads) a level launch with `items` warp work items
// uses: enough for one item per warp, capped at the resident CTA count.
int level_grid(uint32_t items);

// One level: every op of the level, all lightcones at once.
cudaError_t launch_level(cudaStream_t s, const DevOp* ops, const uint32_t* ibeg,
                         const DevTensor* trefs, double2* arena, const LevelLaunch& lv);

// The level's outer-join ops (DevOp::lead/rb), meant to run concurrently with
// launch_level on a second stream.
cudaError_t launch_outer(cudaStream_t s, const DevOp* ops, const uint32_t* ibeg,
                         const DevTensor* trefs, double2* arena, const LevelLaunch& lv);

// The level's fused-chain segments (seg_kernel), concurrent with the others.
cudaError_t launch_segs(cudaStream_t s, const DevSeg* segs, const uint32_t* seg_ibeg,
                        const DevStage* stages, const DevTensor* trefs, const SegOpTab* segtab,
                        double2* arena, uint32_t* ctr, const LevelLaunch& lv);

// Build the segments' SegOpTab entries (once per descriptor upload).
cudaError_t launch_seg_prep(cudaStream_t s, const DevSeg* segs, uint32_t n_segs,
                            const DevTensor* trefs, SegOpTab* segtab);

// Resident warps of the level kernel on the current device.
int resident_warps();

// Per lightcone: e_jk = prod of its scalar results in production order.
cudaError_t launch_final(cudaStream_t s, const uint64_t* scalar_off, const uint32_t* lc_begin,
                         int n_lc, const double2* arena, double2* terms);

// Number of kernels launched per plan execution (level kernels, outer-join
// kernels, segment kernels, final).
inline int kernels_per_plan(int n_level_launches, int n_outer_launches, int n_seg_launches) {
  return n_level_launches + n_outer_launches + n_seg_launches + 1;
}

}  // namespace qtng
