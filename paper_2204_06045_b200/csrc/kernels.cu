// sm_100a kernels of the bucket-elimination path.
//
// level_kernel -- the generic fused bucket kernel.  One launch runs every
// bucket of one dependency level of ALL planned lightcones (tiny buckets cost
// no launch of their own).  The unit of work is a warp "item": 2^cb
// consecutive outputs of one bucket (cb <= 10, chosen per level by the
// planner so that small levels still spread over every SM).  Per item each lane
//   * decodes, once, every operand's bit-gather map into two 32-bit partial
//     offsets: `lo` for its own output bits 0..4 and `hi` for output bits >= 5
//     of the item row it will later broadcast (offsets are additive over bits
//     because every output/sum bit maps to a distinct operand bit),
//   * then walks the item's 2^(cb-5) rows, two at a time: operand offset =
//     lo + shfl(hi, row), 128-bit read-only loads of complex128, the product
//     over operands in bucket member order, accumulation over the summed
//     assignments in ascending order, one 128-bit store per output.  A
//     leading member without row bits (typically the gate on the summed
//     variable) is loaded once per item.
// Operands that are sorted (every intermediate result) map their low bits to
// the bucket's low output bits, so lanes read contiguous 16-byte elements;
// the rank<=2 gate operands are L1-resident.
//
// Rounding: every complex product is (ac-bd, ad+bc) with each product rounded
// (no FMA contraction) and the summed assignments accumulate in ascending
// order -- the exact operation sequence of the reference's
// std::complex<double> loop (NaiveBackend::contract, proj/src/engine.cpp:94-106)
// minus its multiplications by the initial 1 and additions to the initial 0,
// which are exact.  Results therefore equal the reference's as IEEE values
// (only the sign of an exact zero could differ).
#include "kernels.cuh"

#include <cstdint>
#include <cstdio>

#ifndef QTNG_C64
#define QTNG_C64 0  // 1: the complex64 build of this file (namespace qtng::c64)
#endif

namespace qtng {
namespace QTNG_PREC_NS {

#if QTNG_C64
using V = float2;  // complex64 mode: results within the north_star's 1e-5
using R = float;
#else
using V = double2;  // complex128: bit-identical to the reference's naive backend
using R = double;
#endif

namespace {

constexpr int kThreads = 256;
constexpr int kWarpsPerCta = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
#ifndef QTNG_SMEM_OPS
#define QTNG_SMEM_OPS 4096
#endif
constexpr int kSmemOps = QTNG_SMEM_OPS;  // item_begin entries staged in shared memory
#ifndef QTNG_LEVEL_CACHE_MIN
#define QTNG_LEVEL_CACHE_MIN 0u  // items per warp from which a CTA caches the item table (tuned)
#endif

__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ V mkv(R x, R y) { V v; v.x = x; v.y = y; return v; }

__device__ __forceinline__ V cmul(V a, V b) {
  // (a.x*b.x - a.y*b.y, a.x*b.y + a.y*b.x), every product rounded.
  return mkv(rsub(rmul(a.x, b.x), rmul(a.y, b.y)), radd(rmul(a.x, b.y), rmul(a.y, b.x)));
}

__device__ __forceinline__ V cadd(V a, V b) { return mkv(radd(a.x, b.x), radd(a.y, b.y)); }

__device__ __forceinline__ V ld(const V* p) { return __ldg(p); }

// ---- bulk async copy (cp.async.bulk + mbarrier; SASS UBLKCP / SYNCS)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Stage `count` consecutive uint32 of global memory into shared memory with
// ONE bulk copy issued by thread 0, completion tracked by the mbarrier `bar`
// (initialised here; single use).  The copy is widened to 16-byte alignment
// on both ends: the returned skew is where src[0] landed (dst[skew + i] ==
// src[i]); dst must hold count + 7 words; the up to 12 bytes read past the
// end must be readable (the descriptor blob's 256-byte padding).  Every
// thread of the CTA must call this (it contains __syncthreads).
__device__ __forceinline__ uint32_t bulk_stage_u32(uint32_t* dst, const uint32_t* src,
                                                   uint32_t count, uint64_t* bar) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src);
  const uint32_t skew = static_cast<uint32_t>((a & 15u) >> 2);
  const uint32_t nbytes = ((count + skew + 3u) & ~3u) * 4u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(nbytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(a & ~uintptr_t{15}), "r"(nbytes), "r"(smem_u32(bar))
        : "memory");
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar))
        : "memory");
  return skew;
}

// Product over the T operands of one summed assignment (left fold, member order).
template <int T>
__device__ __forceinline__ V chain(const V* const* base, const uint32_t* off,
                                         uint32_t add) {
  V p = ld(base[0] + off[0] + add);
#pragma unroll
  for (int t = 1; t < T; ++t) p = cmul(p, ld(base[t] + off[t] + add));
  return p;
}

// NSM: 0 => no summed bit, 1 => one summed bit, 2 => 2..kMaxSumBits.
// K: 1 => member 0 is row-invariant (DevOp::inv0), hoisted out of the row loop.
template <int T, int NSM, int K>
__device__ __forceinline__ void run_item(const DevOp& op, uint32_t chunk,
                                         const DevTensor* __restrict__ trefs,
                                         V* __restrict__ arena, int lane,
                                         DevTensor* slot) {
  const int cb = op.cb;
  const uint64_t kbase = static_cast<uint64_t>(chunk) << cb;
  const bool active = cb >= 5 || lane < (1 << cb);
  const uint32_t my = active ? lane : 0;
  const uint64_t khi = kbase | (static_cast<uint64_t>(lane) << 5);  // lane = row for `hi`
  // Stage the op's operand descriptors in this warp's shared slot; the
  // per-axis decode below then reads its source bits with broadcast LDS.
  {
    const uint4* src4 = reinterpret_cast<const uint4*>(trefs + op.tref);
    uint4* dst4 = reinterpret_cast<uint4*>(slot);
    if (lane < 3 * T) dst4[lane] = __ldg(src4 + lane);
    __syncwarp();
  }
  const V* base[T];
  uint32_t lo[T], hi[T], sa[T], sb[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const DevTensor& d = slot[t];
    base[t] = arena + d.off;
    const int rank = d.rank;
    uint32_t l = 0, h = 0, a = 0, b = 0;
#pragma unroll 1
    for (int ax = 0; ax < rank; ++ax) {
      const uint32_t src = d.src[ax];
      const uint32_t bit = 1u << (rank - 1 - ax);
      if (src < 5) {
        l |= ((my >> src) & 1u) ? bit : 0u;
      } else if (src < kSumSrc) {
        h |= ((khi >> src) & 1u) ? bit : 0u;
      } else {
        const uint32_t j = src - kSumSrc;
        if (NSM == 1) {
          a |= bit;
        } else if (j < 5) {
          a |= ((static_cast<uint32_t>(lane) >> j) & 1u) ? bit : 0u;
        } else {
          b |= ((static_cast<uint32_t>(lane) >> (j - 5)) & 1u) ? bit : 0u;
        }
      }
    }
    lo[t] = l;
    hi[t] = h;
    sa[t] = a;
    sb[t] = b;
  }
  __syncwarp();  // the slot is rewritten by the warp's next item
  const int rows = cb > 5 ? 1 << (cb - 5) : 1;
  V* out = arena + op.out + kbase + my;
  if (NSM != 2) {
    V g0 = mkv(0.0, 0.0), g1 = g0;
    if (K == 1) {  // member 0 has no row bit: one load per item, both summed values
      const uint32_t o = lo[0] + __shfl_sync(kFull, hi[0], 0);
      g0 = ld(base[0] + o);
      g1 = ld(base[0] + o + sa[0]);
    }
    // two rows in flight per iteration (rows is 1 or even)
    for (int e = 0; e < rows; e += 2) {
      const bool two = e + 1 < rows;
      uint32_t o0[T], o1[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        o0[t] = lo[t] + __shfl_sync(kFull, hi[t], e);
        o1[t] = lo[t] + __shfl_sync(kFull, hi[t], two ? e + 1 : e);
      }
      V r0, r1;
      if (NSM == 0) {
        r0 = chain<T>(base, o0, 0);
        r1 = chain<T>(base, o1, 0);
      } else {
        // s = 0 and s = 1 of both rows; a row-invariant member 0 (K == 1) was
        // loaded once for the whole item
        V a0, b0, a1, b1;
        if (K == 1) {
          a0 = a1 = g0;
          b0 = b1 = g1;
        } else {
          a0 = ld(base[0] + o0[0]);
          b0 = ld(base[0] + o0[0] + sa[0]);
          a1 = ld(base[0] + o1[0]);
          b1 = ld(base[0] + o1[0] + sa[0]);
        }
#pragma unroll
        for (int t = 1; t < T; ++t) {
          const V xa0 = ld(base[t] + o0[t]), xb0 = ld(base[t] + o0[t] + sa[t]);
          const V xa1 = ld(base[t] + o1[t]), xb1 = ld(base[t] + o1[t] + sa[t]);
          a0 = cmul(a0, xa0);
          b0 = cmul(b0, xb0);
          a1 = cmul(a1, xa1);
          b1 = cmul(b1, xb1);
        }
        r0 = cadd(a0, b0);
        r1 = cadd(a1, b1);
      }
      if (active) {
        out[static_cast<uint64_t>(e) << 5] = r0;
        if (two) out[static_cast<uint64_t>(e + 1) << 5] = r1;
      }
    }
  } else {
    const int ns = op.ns;
    const int n_hi = ns > 5 ? 1 << (ns - 5) : 1;
    const int n_lo = ns > 5 ? 32 : 1 << ns;
    for (int e = 0; e < rows; ++e) {
      uint32_t off[T];
#pragma unroll
      for (int t = 0; t < T; ++t) off[t] = lo[t] + __shfl_sync(kFull, hi[t], e);
      V acc = mkv(0.0, 0.0);
      bool first = true;
      for (int sh = 0; sh < n_hi; ++sh) {
        uint32_t offh[T];
#pragma unroll
        for (int t = 0; t < T; ++t) offh[t] = off[t] + __shfl_sync(kFull, sb[t], sh);
        for (int sl = 0; sl < n_lo; ++sl) {
          uint32_t o[T];
#pragma unroll
          for (int t = 0; t < T; ++t) o[t] = offh[t] + __shfl_sync(kFull, sa[t], sl);
          const V p = chain<T>(base, o, 0);
          acc = first ? p : cadd(acc, p);
          first = false;
        }
      }
      if (active) out[static_cast<uint64_t>(e) << 5] = acc;
    }
  }
}

template <int T>
__device__ __forceinline__ void dispatch_ns(const DevOp& op, uint32_t chunk,
                                            const DevTensor* __restrict__ trefs,
                                            V* __restrict__ arena, int lane,
                                            DevTensor* slot) {
  if (op.ns == 1) {
    if (T >= 2 && op.inv0) run_item<T, 1, 1>(op, chunk, trefs, arena, lane, slot);
    else run_item<T, 1, 0>(op, chunk, trefs, arena, lane, slot);
  } else if (op.ns == 0) {
    run_item<T, 0, 0>(op, chunk, trefs, arena, lane, slot);
  } else {
    run_item<T, 2, 0>(op, chunk, trefs, arena, lane, slot);
  }
}

// MAXT: the widest member list among the level's ops; smaller instantiations
// need fewer registers and run at higher occupancy.
template <int MAXT>
#ifndef QTNG_MINB_T2
#define QTNG_MINB_T2 4  // CTAs/SM the register budget must allow (tuned: tools/tune.py)
#endif
#ifndef QTNG_MINB_T4
#define QTNG_MINB_T4 3
#endif
#ifndef QTNG_MINB_T6
#define QTNG_MINB_T6 4
#endif
__global__ void __launch_bounds__(kThreads, MAXT <= 2 ? QTNG_MINB_T2
                                            : (MAXT <= 4 ? QTNG_MINB_T4
                                                         : (MAXT <= 6 ? QTNG_MINB_T6 : 2)))
level_kernel(const DevOp* __restrict__ ops, const uint32_t* __restrict__ ibeg,
             const DevTensor* __restrict__ trefs, V* __restrict__ arena,
             uint32_t op_count, uint32_t items) {
#ifdef QTNG_NOOP_LEVEL  // launch-floor experiments only (tools/tune.py)
  return;
#endif
  __shared__ DevTensor slots[kWarpsPerCta][MAXT];
  __shared__ alignas(16) uint32_t sbeg_raw[kSmemOps + 8];
  __shared__ alignas(8) uint64_t sbar;
  // stage the item table in shared memory with one bulk async copy (one
  // round trip; a binary search in global memory costs ~12 dependent ones)
  const bool cached = op_count <= kSmemOps && items >= QTNG_LEVEL_CACHE_MIN * gridDim.x * kWarpsPerCta;
  const uint32_t* sbeg = sbeg_raw;
  if (cached) sbeg = sbeg_raw + bulk_stage_u32(sbeg_raw, ibeg, op_count, &sbar);
  else __syncthreads();
  const int lane = threadIdx.x & 31;
  DevTensor* slot = slots[threadIdx.x >> 5];
  const uint32_t warp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * kThreads) >> 5;
  uint32_t cur = 0, cur_begin = 1, cur_end = 0;  // cached op lookup
  for (uint32_t item = warp; item < items; item += nwarps) {
    if (item < cur_begin || item >= cur_end) {
      uint32_t lo = 0, hi = op_count;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t b = cached ? sbeg[mid] : __ldg(ibeg + mid);
        if (b <= item) lo = mid; else hi = mid;
      }
      cur = lo;
      cur_begin = cached ? sbeg[lo] : __ldg(ibeg + lo);
      cur_end = lo + 1 < op_count ? (cached ? sbeg[lo + 1] : __ldg(ibeg + lo + 1)) : items;
    }
    const DevOp op = ops[cur];
    const uint32_t chunk = item - cur_begin;
    switch (op.nt) {
      case 1: dispatch_ns<1>(op, chunk, trefs, arena, lane, slot); break;
      case 2: dispatch_ns<2>(op, chunk, trefs, arena, lane, slot); break;
      case 3: if constexpr (MAXT >= 3) dispatch_ns<3>(op, chunk, trefs, arena, lane, slot); break;
      case 4: if constexpr (MAXT >= 4) dispatch_ns<4>(op, chunk, trefs, arena, lane, slot); break;
      case 5: if constexpr (MAXT >= 5) dispatch_ns<5>(op, chunk, trefs, arena, lane, slot); break;
      case 6: if constexpr (MAXT >= 6) dispatch_ns<6>(op, chunk, trefs, arena, lane, slot); break;
      case 7: if constexpr (MAXT >= 7) dispatch_ns<7>(op, chunk, trefs, arena, lane, slot); break;
      default: if constexpr (MAXT >= 8) dispatch_ns<8>(op, chunk, trefs, arena, lane, slot); break;
    }
  }
}

// Insert a zero bit at position q of x.
__device__ __forceinline__ uint32_t insert_zero(uint32_t x, uint32_t q) {
  return ((x >> q) << (q + 1)) | (x & ((1u << q) - 1u));
}

// Outer-join bucket (DevOp::lead/rb): out = sum_s  P_s * A_s * B_s with
// P = the product of the `lead` row-invariant leading members.  The lane
// computes the 4 rows over register bits (rb0: A-only, rb1: B-only) from 2+2
// operand loads per summed value -- half the loads of the generic path --
// while keeping the reference's left-fold order ((P*A)*B).
template <int LEAD>
__device__ __forceinline__ void run_outer(const DevOp& op, uint32_t chunk,
                                          const DevTensor* __restrict__ trefs,
                                          V* __restrict__ arena, int lane, DevTensor* slot) {
  constexpr int T = LEAD + 2;
  const int cb = op.cb;  // >= 7 by construction
  const uint64_t kbase = static_cast<uint64_t>(chunk) << cb;
  const uint64_t khi = kbase | (static_cast<uint64_t>(lane) << 5);
  const uint32_t r0 = op.rb[0], r1 = op.rb[1];
  {
    const uint4* src4 = reinterpret_cast<const uint4*>(trefs + op.tref);
    uint4* dst4 = reinterpret_cast<uint4*>(slot);
    if (lane < 3 * T) dst4[lane] = __ldg(src4 + lane);
    __syncwarp();
  }
  const V* base[T];
  uint32_t lo[T], hi[T], sa[T], d0[T], d1[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const DevTensor& d = slot[t];
    base[t] = arena + d.off;
    const int rank = d.rank;
    uint32_t l = 0, h = 0, a = 0, x0 = 0, x1 = 0;
#pragma unroll 1
    for (int ax = 0; ax < rank; ++ax) {
      const uint32_t src = d.src[ax];
      const uint32_t bit = 1u << (rank - 1 - ax);
      if (src < 5) l |= ((static_cast<uint32_t>(lane) >> src) & 1u) ? bit : 0u;
      else if (src == r0) x0 |= bit;
      else if (src == r1) x1 |= bit;
      else if (src < kSumSrc) h |= ((khi >> src) & 1u) ? bit : 0u;
      else a |= bit;
    }
    lo[t] = l;
    hi[t] = h;
    sa[t] = a;
    d0[t] = x0;
    d1[t] = x1;
  }
  __syncwarp();
  // prefix of the row-invariant leading members, both summed values
  V pre0 = mkv(1.0, 0.0), pre1 = pre0;
#pragma unroll
  for (int t = 0; t < LEAD; ++t) {
    const V* p = base[t] + lo[t] + __shfl_sync(kFull, hi[t], 0);
    const V x = ld(p), y = ld(p + sa[t]);
    pre0 = t == 0 ? x : cmul(pre0, x);
    pre1 = t == 0 ? y : cmul(pre1, y);
  }
  const uint32_t q0 = r0 - 5u, q1 = r1 - 5u;
  const uint32_t qa = q0 < q1 ? q0 : q1, qb = q0 < q1 ? q1 : q0;
  const int steps = 1 << (cb - 7);
  V* out = arena + op.out + kbase + lane;
  constexpr int A = LEAD, B = LEAD + 1;
  for (int it = 0; it < steps; ++it) {
    const uint32_t e = insert_zero(insert_zero(static_cast<uint32_t>(it), qa), qb);
    const V* pa = base[A] + lo[A] + __shfl_sync(kFull, hi[A], e);
    const V* pb = base[B] + lo[B] + __shfl_sync(kFull, hi[B], e);
    const V a00 = ld(pa), a01 = ld(pa + sa[A]);                   // rb0 = 0
    const V a10 = ld(pa + d0[A]), a11 = ld(pa + d0[A] + sa[A]);   // rb0 = 1
    const V b00 = ld(pb), b01 = ld(pb + sa[B]);                   // rb1 = 0
    const V b10 = ld(pb + d1[B]), b11 = ld(pb + d1[B] + sa[B]);   // rb1 = 1
    const V p00 = LEAD ? cmul(pre0, a00) : a00, p01 = LEAD ? cmul(pre1, a01) : a01;
    const V p10 = LEAD ? cmul(pre0, a10) : a10, p11 = LEAD ? cmul(pre1, a11) : a11;
    const uint64_t r00 = static_cast<uint64_t>(e) << 5;
    const uint64_t ra = static_cast<uint64_t>(1u << q0) << 5, rb = static_cast<uint64_t>(1u << q1) << 5;
    out[r00] = cadd(cmul(p00, b00), cmul(p01, b01));
    out[r00 + rb] = cadd(cmul(p00, b10), cmul(p01, b11));
    out[r00 + ra] = cadd(cmul(p10, b00), cmul(p11, b01));
    out[r00 + ra + rb] = cadd(cmul(p10, b10), cmul(p11, b11));
  }
}

__global__ void __launch_bounds__(kThreads, 2)
outer_kernel(const DevOp* __restrict__ ops, const uint32_t* __restrict__ ibeg,
             const DevTensor* __restrict__ trefs, V* __restrict__ arena,
             uint32_t op_count, uint32_t items) {
#ifdef QTNG_NOOP_LEVEL  // launch-floor experiments only (tools/tune.py)
  return;
#endif
  __shared__ DevTensor slots[kWarpsPerCta][4];
  __shared__ alignas(16) uint32_t sbeg_raw[kSmemOps + 8];
  __shared__ alignas(8) uint64_t sbar;
  // the item table staged in shared memory by one bulk async copy
  const bool cached = op_count <= kSmemOps && items >= QTNG_LEVEL_CACHE_MIN * gridDim.x * kWarpsPerCta;
  const uint32_t* sbeg = sbeg_raw;
  if (cached) sbeg = sbeg_raw + bulk_stage_u32(sbeg_raw, ibeg, op_count, &sbar);
  else __syncthreads();
  const int lane = threadIdx.x & 31;
  DevTensor* slot = slots[threadIdx.x >> 5];
  const uint32_t warp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * kThreads) >> 5;
  uint32_t cur = 0, cur_begin = 1, cur_end = 0;
  for (uint32_t item = warp; item < items; item += nwarps) {
    if (item < cur_begin || item >= cur_end) {
      uint32_t lo = 0, hi = op_count;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t b = cached ? sbeg[mid] : __ldg(ibeg + mid);
        if (b <= item) lo = mid; else hi = mid;
      }
      cur = lo;
      cur_begin = cached ? sbeg[lo] : __ldg(ibeg + lo);
      cur_end = lo + 1 < op_count ? (cached ? sbeg[lo + 1] : __ldg(ibeg + lo + 1)) : items;
    }
    const DevOp op = ops[cur];
    const uint32_t chunk = item - cur_begin;
    switch (op.lead) {
      case 0: run_outer<0>(op, chunk, trefs, arena, lane, slot); break;
      case 1: run_outer<1>(op, chunk, trefs, arena, lane, slot); break;
      default: run_outer<2>(op, chunk, trefs, arena, lane, slot); break;
    }
  }
}

// ---------------------------------------------------------------- fused chains
// seg_kernel: one warp evaluates one tile of a segment (device_plan.hpp):
// lane l owns Y output (tile << cY) + l and walks the 2^J digit assignments j
// (digit s_2 fastest) in post order.  For every j it evaluates stage 1 from
// HBM/L1 into a register, then climbs the chain: stage i's term
// P_i(s_i) * X_{i-1}(s_i) (P_i = left fold of its side members, s_i = bit
// i-2 of j) is parked in acc[i] when s_i = 0 and completes X_i = acc[i] +
// term when s_i = 1, which then feeds stage i+1.  No intermediate leaves the
// register file, no barrier is needed, and every X_i element is produced by
// the unfused bucket's exact operation sequence (left-fold product in member
// order, ascending summed values), so results are bit-identical.
// seg_prep_kernel: one warp per segment fills the SegOpTab of each operand.
__global__ void seg_prep_kernel(const DevSeg* __restrict__ segs, uint32_t n_segs,
                                const DevTensor* __restrict__ trefs, SegOpTab* __restrict__ tab) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n_segs) return;
  const DevSeg sg = segs[w];
  for (int op = 0; op < sg.nops; ++op) {
    const DevTensor* d = trefs + sg.tref + op;
    SegOpTab& t = tab[sg.tref + op];
    const int rank = d->rank;
    uint32_t lv = 0, dt = 0, s = 0, dj = 0;  // lane: own part; lane b: tile bit b / digit bit b
    for (int ax = 0; ax < rank; ++ax) {
      const uint32_t code = d->src[ax];
      const uint32_t bit = 1u << (rank - 1 - ax);
      if (code < kLaneSrcEnd) lv |= ((lane >> code) & 1u) ? bit : 0u;
      else if (code < kTileSrc) dj |= (code - kJSrc == static_cast<uint32_t>(lane)) ? bit : 0u;
      else if (code < kSumSrc) dt |= (code - kTileSrc == static_cast<uint32_t>(lane)) ? bit : 0u;
      else s = bit;
    }
    t.llane[lane] = lv;
    t.dtile[lane] = dt;
    if (lane < kSegMaxJ) t.dj[lane] = dj;
    uint32_t below = 0;
    for (int b = 0; b < kSegMaxJ; ++b) {
      const uint32_t djb = __shfl_sync(kFull, dj, b);
      if (lane == b) t.inc[b] = djb - below;
      below += djb;
    }
    uint32_t lo = 0, hi = 0;
    for (int b = 0; b < 4; ++b) {
      const uint32_t xl = __shfl_sync(kFull, dj, b), xh = __shfl_sync(kFull, dj, b + 4);
      lo += ((lane >> b) & 1) ? xl : 0u;
      hi += ((lane >> b) & 1) ? xh : 0u;
    }
    if (lane < 16) {
      t.dlo[lane] = lo;
      t.dhi[lane] = hi;
    }
    if (lane == 0) {
      t.sd = s;
      t.kind = d->kind;
      t.off = d->off;
    }
  }
}

// Per-warp state of seg_kernel: the current tile's offsets and the parked terms.
struct ChainWarp {
  uint32_t toff[kSegMaxOps];             // tile part of each operand's offset
  DevStage st[kSegMaxStages];
  V ptab[kSegMaxStages - 1][8];    // [i - 1]: tabulated side products P_i(s_i, u0, u1) of this tile
  // per stage: bits 0-1 mode (0 no side member, 1 table, 2 real table, 3
  // gathered), bits 8-12 / 13 and 16-20 / 21: source position / valid of the
  // table index bits 1 and 2, a position in x = j | lane << 16 (a digit bit
  // of j, or 16 + a lane bit); no per-lane table, so the climb state stays
  // small enough for the SM's 132 KB carveout (more L1)
  uint32_t sdesc[kSegMaxStages];
  V acc[kSegMaxStages - 2][32];    // per lane: parked s_i = 0 terms of stage k + 2 (k >= 1)
  V acc1[kSegMaxStages - 2][32];   // ... of the second row (paired segments)
  uint32_t drow[kSegMaxNt1];       // paired: stage-1 member offset of the second row
};

// (r, 0) * y and p * (r, 0): equal to cmul up to the sign of an exact zero.
__device__ __forceinline__ V rscale(R r, V y) {
  return mkv(rmul(r, y.x), rmul(r, y.y));
}

// One left-fold step p * y where either factor may be a real scalar (r, 0).
__device__ __forceinline__ V fmul(V p, bool p_real, V y, bool y_real) {
  if (y_real) return rscale(y.x, p);
  if (p_real) return rscale(p.x, y);
  return cmul(p, y);
}

// Side-member product P_i (left fold of members [op0, op0+m)) at digit
// assignment j; m >= 1.  *real: P is a real scalar (r, 0).
__device__ __forceinline__ V chain_side(const ChainWarp& cw, const SegOpTab* __restrict__ tab,
                                              const V* __restrict__ arena, int op0, int m,
                                              uint32_t j, int lane, bool* real) {
  const uint32_t jl = j & 15u, jh = j >> 4;
  V p = mkv(0.0, 0.0);
  bool pr = false;
#pragma unroll
  for (int t = 0; t < kSegMaxNt - 1; ++t) {  // unrolled: loads of independent terms overlap
    if (t >= m) break;
    const int op = op0 + t;
    const SegOpTab* tb = tab + op;
    const bool xr = __ldg(&tb->kind) == kTensorRealScalar;
    const V x = xr ? mkv(__ldg(&(arena + __ldg(&tb->off))->x), 0.0)
                         : ld(arena + __ldg(&tb->off) +
                              (cw.toff[op] + __ldg(&tb->llane[lane]) + __ldg(&tb->dlo[jl]) +
                               __ldg(&tb->dhi[jh])));
    if (t == 0) {
      p = x;
      pr = xr;
    } else {
      p = fmul(p, pr, x, xr);
      pr = false;
    }
  }
  *real = pr;
  return p;
}

#ifndef QTNG_SEG_U2_MAXNT
#define QTNG_SEG_U2_MAXNT 0  // heads with <= this many members walk digits in fours
#endif
#ifndef QTNG_SEG_PTAB
#define QTNG_SEG_PTAB 1  // tabulated side products in the climb
#endif

// term of stage i = k + 2 (DevStage st) at digit assignment j: P_i(j) * v, or v.
__device__ __forceinline__ V chain_term(const ChainWarp& cw, const SegOpTab* __restrict__ tab,
                                              const V* __restrict__ arena, const DevStage st,
                                              int k, uint32_t j, V v, int lane) {
  const uint32_t d = cw.sdesc[k + 1];
  const uint32_t mode = d & 3u;
  if (mode == 0) return v;
  if (mode != 3) {
    const uint32_t x = j | (static_cast<uint32_t>(lane) << 16);
    const uint32_t idx = ((j >> k) & 1u) | (((x >> ((d >> 8) & 31u)) & (d >> 13) & 1u) << 1) |
                         (((x >> ((d >> 16) & 31u)) & (d >> 21) & 1u) << 2);
    const V p = cw.ptab[k][idx];
    return mode == 2 ? rscale(p.x, v) : cmul(p, v);
  }
  const int m = st.nt - 1;
  bool real;
  const V p = chain_side(cw, tab, arena, st.op0, m, j, lane, &real);
  return real ? rscale(p.x, v) : cmul(p, v);
}

// chain_term for both rows of a paired tile: the side product P_i does not
// depend on the row bit, so it is looked up or gathered once.
__device__ __forceinline__ void chain_term2(const ChainWarp& cw, const SegOpTab* __restrict__ tab,
                                            const V* __restrict__ arena, const DevStage st,
                                            int k, uint32_t j, V& v0, V& v1, int lane) {
  const uint32_t d = cw.sdesc[k + 1];
  const uint32_t mode = d & 3u;
  if (mode == 0) return;
  V p;
  bool real;
  if (mode != 3) {
    const uint32_t x = j | (static_cast<uint32_t>(lane) << 16);
    const uint32_t idx = ((j >> k) & 1u) | (((x >> ((d >> 8) & 31u)) & (d >> 13) & 1u) << 1) |
                         (((x >> ((d >> 16) & 31u)) & (d >> 21) & 1u) << 2);
    p = cw.ptab[k][idx];
    real = mode == 2;
  } else {
    p = chain_side(cw, tab, arena, st.op0, st.nt - 1, j, lane, &real);
  }
  if (real) {
    v0 = rscale(p.x, v0);
    v1 = rscale(p.x, v1);
  } else {
    v0 = cmul(p, v0);
    v1 = cmul(p, v1);
  }
}

// One paired tile (DevSeg::rb): chain_tile's walk with U = 1 for two Y rows
// at once.  Row 1's stage-1 operands sit drow[t] further; everything else
// (digit offsets, side products, climb control) is shared.  Each row sees
// exactly the operation sequence of the unpaired walk.  RM: bit t set if
// stage-1 member t reads the row bit (drow[t] != 0); DM: bit t set if it
// does not read digit bit 0 (dj[0] == 0).  Specialised for the common masks;
// otherwise RM = all members, DM = none.
template <int NT, int NS, int K0, int RM, int DM>
__device__ __forceinline__ void chain_tile2(ChainWarp& cw, const SegOpTab* __restrict__ tab,
                                            const DevSeg& sg, V* __restrict__ arena,
                                            uint32_t tile, int lane) {
  const int L = sg.nst;
  const uint32_t nj = 1u << (L - 1);
  const V* B[NT];
  uint32_t o[NT], sdl[NT], d0[NT], dr[NT];
  const R r0 = K0 ? __ldg(&(arena + __ldg(&tab[0].off))->x) : 0.0;
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    B[t] = arena + __ldg(&tab[t].off);
    o[t] = cw.toff[t] + __ldg(&tab[t].llane[lane]);
    sdl[t] = __ldg(&tab[t].sd);
    d0[t] = __ldg(&tab[t].dj[0]);
    dr[t] = cw.drow[t];
  }
  const DevStage st2 = cw.st[1];
  V* y = arena + sg.out + (static_cast<uint64_t>(tile) << kSegYBits) + lane;
  const uint64_t y1 = uint64_t{1} << (sg.rb + kSegYBits);
  for (uint32_t j = 0; j < nj; j += 2) {
    if (j) {
      const int b = __ffs(j) - 1;
#pragma unroll
      for (int t = 0; t < NT; ++t) o[t] += __ldg(&tab[t].inc[b]) + d0[t];
    }
    // [row][member] at s = 0 (m) and s = 1 (n).  Row 1 reloads only the
    // members that read the row bit (RM), q = 1 only those that read digit
    // bit 0 (not in DM); the rest -- and the products of an invariant
    // leading run -- are shared
    V km[2][NT], kn[2][NT];  // q = 0 values of the DM members
    V v[2][2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      V m[2][NT], n[2][NT];
#pragma unroll
      for (int t = K0 ? 1 : 0; t < NT; ++t) {
        if (q == 1 && ((DM >> t) & 1)) {
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            m[r][t] = km[r][t];
            n[r][t] = kn[r][t];
          }
          continue;
        }
        const uint32_t oq = o[t] + (q ? d0[t] : 0u);
        m[0][t] = ld(B[t] + oq);
        m[1][t] = ((RM >> t) & 1) ? ld(B[t] + oq + dr[t]) : m[0][t];
        if (NS) {
          n[0][t] = ld(B[t] + oq + sdl[t]);
          n[1][t] = ((RM >> t) & 1) ? ld(B[t] + oq + sdl[t] + dr[t]) : n[0][t];
        }
        if (q == 0 && ((DM >> t) & 1)) {
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            km[r][t] = m[r][t];
            kn[r][t] = n[r][t];
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        V x = K0 ? rscale(r0, m[r][1]) : m[r][0];
#pragma unroll
        for (int t = K0 ? 2 : 1; t < NT; ++t) x = cmul(x, m[r][t]);
        if (NS) {
          V p = K0 ? rscale(r0, n[r][1]) : n[r][0];
#pragma unroll
          for (int t = K0 ? 2 : 1; t < NT; ++t) p = cmul(p, n[r][t]);
          x = cadd(x, p);
        }
        v[q][r] = x;
      }
    }
    chain_term2(cw, tab, arena, st2, 0, j, v[0][0], v[0][1], lane);
    chain_term2(cw, tab, arena, st2, 0, j | 1u, v[1][0], v[1][1], lane);
    V x0 = cadd(v[0][0], v[1][0]), x1 = cadd(v[0][1], v[1][1]);
    const uint32_t jj = j | 1u;
    bool carry = true;
    for (int k = 1; k + 2 <= L; ++k) {
      chain_term2(cw, tab, arena, cw.st[k + 1], k, jj, x0, x1, lane);
      if (!((jj >> k) & 1u)) {
        cw.acc[k - 1][lane] = x0;
        cw.acc1[k - 1][lane] = x1;
        carry = false;
        break;
      }
      x0 = cadd(cw.acc[k - 1][lane], x0);
      x1 = cadd(cw.acc1[k - 1][lane], x1);
    }
    if (carry) {
      y[0] = x0;
      y[y1] = x1;
    }
  }
}

// chain_tile2 specialised for the member masks key = RM | DM << 8 if it is
// one of Keys.
template <int NT, int NS, int K0, int... Keys>
__device__ __forceinline__ bool chain_tile2_masks(int key, ChainWarp& cw,
                                                  const SegOpTab* __restrict__ tab,
                                                  const DevSeg& sg, V* __restrict__ arena,
                                                  uint32_t tile, int lane) {
  return ((key == Keys ? (chain_tile2<NT, NS, K0, (Keys & 0xff), (Keys >> 8)>(cw, tab, sg, arena,
                                                                          tile, lane), true)
                       : false) || ...);
}

// One tile: 2^J stage-1 evaluations (NT members, NS summed bits), in groups
// of 2^U consecutive j (stages 2..U+1 resolved in registers, four independent
// stage-1 products in flight), then the climb above each group.
// DM: bit t set if member t does not read digit bit 0 (loaded once per pair).
template <int NT, int NS, int U, int K0, int DM = 0>
__device__ __forceinline__ void chain_tile(ChainWarp& cw, const SegOpTab* __restrict__ tab,
                                           const DevSeg& sg, V* __restrict__ arena,
                                           uint32_t tile, int lane) {
  constexpr int G = 1 << U;
  const int L = sg.nst;
  const uint32_t nj = 1u << (L - 1);
  const V* B[NT];
  uint32_t o[NT], sdl[NT], d0[NT], d1[NT];
  // K0: member 0 is a real scalar r (the |+> state on the summed var): the
  // first product (r, 0) * M1 becomes a scale, and member 0 is not gathered
  const R r0 = K0 ? __ldg(&(arena + __ldg(&tab[0].off))->x) : 0.0;
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    B[t] = arena + __ldg(&tab[t].off);
    o[t] = cw.toff[t] + __ldg(&tab[t].llane[lane]);
    sdl[t] = __ldg(&tab[t].sd);
    d0[t] = __ldg(&tab[t].dj[0]);
    d1[t] = U > 1 ? __ldg(&tab[t].dj[1]) : 0u;
  }
  const DevStage st2 = cw.st[1];
  const DevStage st3 = U > 1 ? cw.st[2] : st2;
  for (uint32_t j = 0; j < nj; j += G) {
    if (j) {  // from j - G (low U bits clear) to j: inc[b] assumes bits < b were set
      const int b = __ffs(j) - 1;
#pragma unroll
      for (int t = 0; t < NT; ++t) o[t] += __ldg(&tab[t].inc[b]) + d0[t] + d1[t];
    }
    V v[G];
    V km[NT], kn[NT];  // even-q values of the DM members
#pragma unroll
    for (int q = 0; q < G; ++q) {
      V m[NT], n[NT];  // member values at s = 0 / s = 1
#pragma unroll
      for (int t = K0 ? 1 : 0; t < NT; ++t) {
        if ((q & 1) && ((DM >> t) & 1)) {
          m[t] = km[t];
          n[t] = kn[t];
          continue;
        }
        const uint32_t oq = o[t] + ((q & 1) ? d0[t] : 0u) + ((q & 2) ? d1[t] : 0u);
        m[t] = ld(B[t] + oq);
        if (NS) n[t] = ld(B[t] + oq + sdl[t]);
        if (!(q & 1) && ((DM >> t) & 1)) {
          km[t] = m[t];
          kn[t] = n[t];
        }
      }
      V x = K0 ? rscale(r0, m[1]) : m[0];
#pragma unroll
      for (int t = K0 ? 2 : 1; t < NT; ++t) x = cmul(x, m[t]);
      if (NS) {
        V p = K0 ? rscale(r0, n[1]) : n[0];
#pragma unroll
        for (int t = K0 ? 2 : 1; t < NT; ++t) p = cmul(p, n[t]);
        x = cadd(x, p);
      }
      v[q] = x;
    }
    // stage 2 over bit 0, stage 3 over bit 1 (U == 2)
    V x = cadd(chain_term(cw, tab, arena, st2, 0, j, v[0], lane),
                     chain_term(cw, tab, arena, st2, 0, j | 1u, v[1], lane));
    if (U > 1) {
      const V y = cadd(chain_term(cw, tab, arena, st2, 0, j | 2u, v[2], lane),
                             chain_term(cw, tab, arena, st2, 0, j | 3u, v[3], lane));
      x = cadd(chain_term(cw, tab, arena, st3, 1, j, x, lane),
               chain_term(cw, tab, arena, st3, 1, j | 2u, y, lane));
    }
    // climb: stage i = k + 2 >= U + 2 while the carry propagates
    const uint32_t jj = j | (G - 1);
    bool carry = true;
    for (int k = U; k + 2 <= L; ++k) {
      const V term = chain_term(cw, tab, arena, cw.st[k + 1], k, jj, x, lane);
      if (!((jj >> k) & 1u)) {
        cw.acc[k - 1][lane] = term;
        carry = false;
        break;
      }
      x = cadd(cw.acc[k - 1][lane], term);
    }
    if (carry && lane < (1 << sg.cy)) arena[sg.out + (static_cast<uint64_t>(tile) << sg.cy) + lane] = x;
  }
}

// Tiles of segments whose Y has fewer than 32 outputs (cY < 5; the chain
// tails): 2^J stage-1 evaluations (NT members, NS summed bits) where the ld = min(5 - cY, J) lowest digits
// ride on the otherwise idle lanes: lane = (lane digits << cY) | Y bits, and
// stages 2 .. ld+1 combine sibling lanes with shfl_xor (t0 + t1 == t1 + t0
// exactly, so every sibling holds the unfused value).  The remaining digits
// are walked by the loop in pairs (the pair's stage resolved in registers),
// then the climb parks s_i = 0 terms in shared memory.
template <int NT, int NS, int K0>
__device__ __noinline__ void chain_tile_lanes(ChainWarp& cw, const SegOpTab* __restrict__ tab,
                                           const DevSeg& sg, V* __restrict__ arena,
                                           uint32_t tile, int lane) {
  const int L = sg.nst, J = L - 1, cy = sg.cy;
  const int nld = min(kSegYBits - cy, J);
  const uint32_t ldig = (static_cast<uint32_t>(lane) >> cy) & ((1u << nld) - 1u);
  const uint32_t nloop = 1u << (J - nld);
  const int G = nloop > 1 ? 2 : 1;
  const V* B[NT];
  uint32_t o[NT], sdl[NT], d0[NT], sld[NT];
  // K0: member 0 is a real scalar r (the |+> state on the summed var): the
  // first product (r, 0) * M1 becomes a scale, and member 0 is not gathered
  const R r0 = K0 ? __ldg(&(arena + __ldg(&tab[0].off))->x) : 0.0;
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const SegOpTab* tb = tab + t;
    B[t] = arena + __ldg(&tb->off);
    uint32_t lo = 0, sum = 0;  // lane digits: this lane's part and the sum of their deltas
    for (int b = 0; b < nld; ++b) {
      const uint32_t d = __ldg(&tb->dj[b]);
      lo += ((ldig >> b) & 1u) ? d : 0u;
      sum += d;
    }
    o[t] = cw.toff[t] + __ldg(&tb->llane[lane]) + lo;
    sld[t] = sum;
    sdl[t] = __ldg(&tb->sd);
    d0[t] = G > 1 ? __ldg(&tb->dj[nld]) : 0u;
  }
  for (uint32_t j = 0; j < nloop; j += G) {
    if (j) {  // from j - 2 (low loop bit clear) to j; inc[] assumes every lower digit was set
      const int b = nld + __ffs(j) - 1;
#pragma unroll
      for (int t = 0; t < NT; ++t) o[t] += __ldg(&tab[t].inc[b]) + sld[t] + d0[t];
    }
    V v[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (q >= G) break;
      uint32_t oq[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) oq[t] = o[t] + (q ? d0[t] : 0u);
      V x = K0 ? rscale(r0, ld(B[1] + oq[1])) : ld(B[0] + oq[0]);
#pragma unroll
      for (int t = K0 ? 2 : 1; t < NT; ++t) x = cmul(x, ld(B[t] + oq[t]));
      if (NS) {
        V p = K0 ? rscale(r0, ld(B[1] + oq[1] + sdl[1])) : ld(B[0] + oq[0] + sdl[0]);
#pragma unroll
        for (int t = K0 ? 2 : 1; t < NT; ++t) p = cmul(p, ld(B[t] + oq[t] + sdl[t]));
        x = cadd(x, p);
      }
      // lane-digit stages: combine with the sibling lane
      const uint32_t fj = ((j + q) << nld) | ldig;
      for (int k = 0; k < nld; ++k) {
        const V t = chain_term(cw, tab, arena, cw.st[k + 1], k, fj, x, lane);
        const V u = mkv(__shfl_xor_sync(kFull, t.x, 1 << (cy + k)),
                                       __shfl_xor_sync(kFull, t.y, 1 << (cy + k)));
        x = cadd(t, u);
      }
      v[q] = x;
    }
    V x = v[0];
    if (G > 1) {  // the pair's stage (digit nld) in registers
      const uint32_t f0 = (j << nld) | ldig;
      x = cadd(chain_term(cw, tab, arena, cw.st[nld + 1], nld, f0, v[0], lane),
               chain_term(cw, tab, arena, cw.st[nld + 1], nld, f0 | (1u << nld), v[1], lane));
    }
    // climb: stage i = k + 2 >= nld + 3 while the carry propagates
    const uint32_t jj = ((j | (G - 1)) << nld) | ldig;
    bool carry = true;
    for (int k = nld + 1; k + 2 <= L; ++k) {
      const V term = chain_term(cw, tab, arena, cw.st[k + 1], k, jj, x, lane);
      if (!((jj >> k) & 1u)) {
        cw.acc[k - 1][lane] = term;
        carry = false;
        break;
      }
      x = cadd(cw.acc[k - 1][lane], term);
    }
    if (carry && ldig == 0 && lane < (1 << cy))
      arena[sg.out + (static_cast<uint64_t>(tile) << cy) + lane] = x;
  }
}

template <int NT, int NS>
__device__ __forceinline__ void chain_tile_u(ChainWarp& cw, const SegOpTab* __restrict__ tab,
                                             const DevSeg& sg, V* __restrict__ arena,
                                             uint32_t tile, int lane) {
  const bool k0 = NT >= 2 && __ldg(&tab[0].kind) == kTensorRealScalar;
  if (sg.cy < kSegYBits) {  // chain tails: digits on the idle lanes
    if (k0) chain_tile_lanes<NT, NS, (NT >= 2 ? 1 : 0)>(cw, tab, sg, arena, tile, lane);
    else chain_tile_lanes<NT, NS, 0>(cw, tab, sg, arena, tile, lane);
    return;
  }
  if constexpr (NT <= kSegPairMaxNt) {
    if (sg.rb != kNoVar) {  // paired rows
      constexpr int kAll = (1 << NT) - 1;
      int key = 0;
#pragma unroll
      for (int t = 0; t < NT; ++t)
        key |= (cw.drow[t] ? 1 << t : 0) | (__ldg(&tab[t].dj[0]) ? 0 : 256 << t);
      if (k0) {
        constexpr int K = NT >= 2 ? 1 : 0;
        key &= ~0x101;
        if constexpr (NS == 1 && NT == 3) {
          if (chain_tile2_masks<3, 1, K, 2, 4, 6 | 4 << 8>(key, cw, tab, sg, arena, tile, lane))
            return;
        }
        if constexpr (NS == 1 && NT == 4) {
          if (chain_tile2_masks<4, 1, K, 4, 8, 12, 12 | 2 << 8, 4 | 2 << 8, 8 | 2 << 8>(
                  key, cw, tab, sg, arena, tile, lane))
            return;
        }
        chain_tile2<NT, NS, K, kAll, 0>(cw, tab, sg, arena, tile, lane);
      } else {
        if constexpr (NS == 1 && NT == 2) {
          if (chain_tile2_masks<2, 1, 0, 1, 2>(key, cw, tab, sg, arena, tile, lane)) return;
        }
        if constexpr (NS == 1 && NT == 3) {
          if (chain_tile2_masks<3, 1, 0, 2, 4, 4 | 1 << 8, 2 | 1 << 8>(key, cw, tab, sg, arena,
                                                                      tile, lane))
            return;
        }
        chain_tile2<NT, NS, 0, kAll, 0>(cw, tab, sg, arena, tile, lane);
      }
      return;
    }
  }
  constexpr int U = NT <= QTNG_SEG_U2_MAXNT ? 2 : 1;  // groups of 2^U digit values
  if (U == 2 && sg.nst >= 3) {
    if (k0) chain_tile<NT, NS, U, (NT >= 2 ? 1 : 0)>(cw, tab, sg, arena, tile, lane);
    else chain_tile<NT, NS, U, 0>(cw, tab, sg, arena, tile, lane);
    return;
  }
  if constexpr (NS == 1 && NT == 5) {  // the unpaired 5-member C2 head: members 1, 3 lack digit 0
    if (k0 && !__ldg(&tab[1].dj[0]) && __ldg(&tab[2].dj[0]) && !__ldg(&tab[3].dj[0]) &&
        __ldg(&tab[4].dj[0])) {
      chain_tile<5, 1, 1, 1, 10>(cw, tab, sg, arena, tile, lane);
      return;
    }
  }
  if (k0) chain_tile<NT, NS, 1, (NT >= 2 ? 1 : 0)>(cw, tab, sg, arena, tile, lane);
  else chain_tile<NT, NS, 1, 0>(cw, tab, sg, arena, tile, lane);
}

// Tabulate the side products of the fused stages for this tile: lane
// (stage, entry) folds the stage's side members at (s_i, u0, u1) = entry bits
// (a tile-bit u takes this tile's value) exactly like chain_side.  Cold path:
// kept out of line so the hot loop's registers are not spilled for it.
// fa / fb (quad tiles): tile-bit codes that stay table index bits (the rows'
// bits) instead of taking the tile's value; kNoVar otherwise.
__device__ __noinline__ void chain_ptab_build(ChainWarp& cw, const DevSeg& sg,
                                              const DevTensor* __restrict__ trefs,
                                              const V* __restrict__ arena, uint32_t tile,
                                              int lane, uint8_t fa = kNoVar,
                                              uint8_t fb = kNoVar) {
  for (int base = 8; base < 8 * sg.nst; base += 32) {
    const int i = (base + lane) >> 3, e = (base + lane) & 7;
    if (i < sg.nst && cw.st[i].ptab) {
      const DevStage st = cw.st[i];
      const uint8_t own = static_cast<uint8_t>(kJSrc + (i - 1));
      auto val = [&](uint8_t c) -> uint32_t {
        if (c == own) return e & 1;
        const int w = c == st.u[0] ? 0 : 1;
        if (c >= kTileSrc && c < kSumSrc && c != fa && c != fb) return (tile >> (c - kTileSrc)) & 1u;
        return (e >> (1 + w)) & 1;
      };
      V p = mkv(0.0, 0.0);
      bool pr = false;
      for (int t = 0; t < st.nt - 1; ++t) {
        const DevTensor* d = trefs + sg.tref + st.op0 + t;
        const int rank = d->rank;
        uint32_t o = 0;
        for (int ax = 0; ax < rank; ++ax) o |= val(d->src[ax]) << (rank - 1 - ax);
        const bool xr = d->kind == kTensorRealScalar;
        const V x = xr ? mkv(__ldg(&(arena + d->off)->x), 0.0) : ld(arena + d->off + o);
        if (t == 0) {
          p = x;
          pr = xr;
        } else {
          p = fmul(p, pr, x, xr);
          pr = false;
        }
      }
      cw.ptab[i - 1][e] = p;
    }
  }
}

// Per-warp state of the segment currently being evaluated.
struct SegCursor {
  int cur = -1;            // segment index whose tables are loaded
  bool ptab_fresh = false;  // side-product tables built for this segment
  bool ptab_tile = false;   // ... and they depend on the tile number
  DevSeg sg{};
};

// Load segment `si` into the warp state: stages, climb descriptors, per-lane
// table-index bits.
__device__ __forceinline__ void seg_switch(ChainWarp& cw, SegCursor& sc, const DevSeg* __restrict__ segs,
                                           int si, const DevStage* __restrict__ stages,
                                           const SegOpTab* __restrict__ segtab, int lane) {
  sc.cur = si;
  sc.sg = segs[si];
  const DevSeg& sg = sc.sg;
  const bool quad = sg.rb2 != kNoVar;
  __syncwarp();
  bool tile_dep = false;
  if (lane < sg.nst) {
    const DevStage st = stages[sg.stage + lane];
    cw.st[lane] = st;
    bool real = lane > 0 && st.nt > 1;  // every side member a real scalar
    for (int t = 0; real && t < st.nt - 1; ++t)
      real = __ldg(&segtab[sg.tref + st.op0 + t].kind) == kTensorRealScalar;
    for (int w = 0; w < 2; ++w)  // quad rows' bits are table index bits, not tile values
      tile_dep |= st.ptab && st.u[w] >= kTileSrc && st.u[w] < kSumSrc &&
                  !(quad && (st.u[w] == kTileSrc + sg.rb || st.u[w] == kTileSrc + sg.rb2));
    const uint32_t mode = st.nt <= 1 ? 0u : (QTNG_SEG_PTAB && st.ptab ? (real ? 2u : 1u) : 3u);
    uint32_t d = mode;
    for (int w = 0; w < 2; ++w)
      if (mode == 1u || mode == 2u) {
        const uint32_t c = st.u[w];
        if (c >= kJSrc && c < kTileSrc) d |= ((c - kJSrc) | 32u) << (8 + 8 * w);   // digit bit of j
        else if (c < kLaneSrcEnd) d |= ((16u + c) | 32u) << (8 + 8 * w);        // lane bit
      }
    cw.sdesc[lane] = d;
  }
  __syncwarp();
  // the side-product tables depend on the tile only through tile-bit u's
  sc.ptab_tile = __any_sync(kFull, tile_dep);
  sc.ptab_fresh = false;
}

// One tile of the loaded segment.
__device__ __forceinline__ void seg_tile(ChainWarp& cw, SegCursor& sc, uint32_t item,
                                         const DevTensor* __restrict__ trefs,
                                         const SegOpTab* __restrict__ segtab,
                                         V* __restrict__ arena, int lane) {
  const DevSeg& sg = sc.sg;
  const SegOpTab* tab = segtab + sg.tref;
  // paired: the work item is the tile number without bit rb (row 0 = bit clear)
  const bool paired = sg.rb != kNoVar;
  const uint32_t tile = paired ? insert_zero(item, sg.rb) : item;
  if (paired && lane < kSegMaxNt1 && lane < sg.nops) cw.drow[lane] = __ldg(&tab[lane].dtile[sg.rb]);
  for (int op = 0; op < sg.nops; ++op) {
    const uint32_t v = ((tile >> lane) & 1u) ? __ldg(&tab[op].dtile[lane]) : 0u;
    const uint32_t sum = __reduce_add_sync(kFull, v);
    if (lane == 0) cw.toff[op] = sum;
  }
  if (!sc.ptab_fresh || sc.ptab_tile) {
    chain_ptab_build(cw, sg, trefs, arena, tile, lane);
    sc.ptab_fresh = true;
  }
  __syncwarp();
  const DevStage s1 = cw.st[0];
#ifdef QTNG_SASS_ONE_SHAPE  // SASS inspection build: only the dominant head shape
  chain_tile_u<3, 1>(cw, tab, sg, arena, tile, lane);
  return;
#endif
  switch (s1.nt * 2 + s1.ns) {
    case 2: chain_tile_u<1, 0>(cw, tab, sg, arena, tile, lane); break;
    case 3: chain_tile_u<1, 1>(cw, tab, sg, arena, tile, lane); break;
    case 4: chain_tile_u<2, 0>(cw, tab, sg, arena, tile, lane); break;
    case 5: chain_tile_u<2, 1>(cw, tab, sg, arena, tile, lane); break;
    case 6: chain_tile_u<3, 0>(cw, tab, sg, arena, tile, lane); break;
    case 7: chain_tile_u<3, 1>(cw, tab, sg, arena, tile, lane); break;
    case 8: chain_tile_u<4, 0>(cw, tab, sg, arena, tile, lane); break;
    case 9: chain_tile_u<4, 1>(cw, tab, sg, arena, tile, lane); break;
    case 10: chain_tile_u<5, 0>(cw, tab, sg, arena, tile, lane); break;
    case 11: chain_tile_u<5, 1>(cw, tab, sg, arena, tile, lane); break;
    case 12: chain_tile_u<6, 0>(cw, tab, sg, arena, tile, lane); break;
    default: chain_tile_u<6, 1>(cw, tab, sg, arena, tile, lane); break;
  }
  __syncwarp();
}

// ---------------------------------------------------------------- quad tiles
// seg4_kernel: segments whose head (stage 1) is an outer join
// [prefix..., A, B] -- A reads tile bit rb and B does not, B reads rb2 and A
// does not, the prefix (the |+> scale, small gates) reads neither.  A lane
// evaluates four Y rows at once, r = (rb, rb2) in {0,1}^2: per digit
// assignment and summed value it loads A at rb = 0/1 and B at rb2 = 0/1 and
// forms the 2 x 2 outer product PA[rb] * B[rb2] with PA = prefix * A -- four
// terms from four operand loads, where a lane of seg_kernel loads two (paired)
// or one (unpaired) operand per term.  Register reuse is the lever: every
// operand value reaching the register file costs the SM's 128 B/clk L1 data
// path, which bounds seg_kernel before its FP64 pipe does (ncu:
// l1tex__data_pipe_lsu_wavefronts 59% vs FP64 30%).
// Each row sees exactly the unfused operation sequence: left fold in member
// order ((prefix * A) * B), summed values ascending, the climb as in
// chain_tile2; a tabulated side product that depends on rb / rb2 is looked
// up per row (build_plan never picks row bits a gathered side member reads).
struct ChainWarp4 {
  ChainWarp b;                          // rows 0 / 1 park in b.acc / b.acc1
  V acc2[kSegMaxStages - 2][32];        // ... rows 2 / 3
  V acc3[kSegMaxStages - 2][32];
  uint32_t da[kSegMaxOps], db[kSegMaxOps];  // per operand: offset of tile bit rb / rb2
  // per stage: bits 0-7 = ptab index bit fed by rb, 8-15 = by rb2 (a tabulated
  // side product may depend on the row; gathered side members never do)
  uint32_t rdesc[kSegMaxStages];
};

// Quad extras of the segment just loaded by seg_switch.
__device__ __forceinline__ void seg_switch4(ChainWarp4& cw, const DevSeg& sg,
                                            const SegOpTab* __restrict__ tab, int lane) {
  if (lane < sg.nops) {
    cw.da[lane] = __ldg(&tab[lane].dtile[sg.rb]);
    cw.db[lane] = __ldg(&tab[lane].dtile[sg.rb2]);
  }
  __syncwarp();
  if (lane >= 1 && lane < sg.nst) {
    const DevStage st = cw.b.st[lane];
    const uint32_t mode = cw.b.sdesc[lane] & 3u;
    const uint8_t ca = static_cast<uint8_t>(kTileSrc + sg.rb), cb = static_cast<uint8_t>(kTileSrc + sg.rb2);
    uint32_t d = 0;
    if (mode == 1u || mode == 2u) {
      for (int w = 0; w < 2; ++w) {
        if (st.u[w] == ca) d |= 2u << w;
        if (st.u[w] == cb) d |= (2u << w) << 8;
      }
    }
    cw.rdesc[lane] = d;
  }
  __syncwarp();
}

// Stage k + 2's term for the four rows: x[r] = P(j, row r) * x[r].
__device__ __forceinline__ void chain_term4(const ChainWarp4& cw, const SegOpTab* __restrict__ tab,
                                            const V* __restrict__ arena, const DevStage st, int k,
                                            uint32_t j, V (&x)[4], int lane) {
  const uint32_t d = cw.b.sdesc[k + 1];
  const uint32_t mode = d & 3u;
  if (mode == 0) return;
  const uint32_t rd = cw.rdesc[k + 1];
  if (mode != 3) {
    const uint32_t jx = j | (static_cast<uint32_t>(lane) << 16);
    const uint32_t idx = ((j >> k) & 1u) | (((jx >> ((d >> 8) & 31u)) & (d >> 13) & 1u) << 1) |
                         (((jx >> ((d >> 16) & 31u)) & (d >> 21) & 1u) << 2);
    const uint32_t ma = rd & 0xffu, mb = (rd >> 8) & 0xffu;
    if (!(ma | mb)) {
      const V p = cw.b.ptab[k][idx];
#pragma unroll
      for (int r = 0; r < 4; ++r) x[r] = mode == 2 ? rscale(p.x, x[r]) : cmul(p, x[r]);
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const V p = cw.b.ptab[k][idx | ((r & 1) ? ma : 0u) | ((r & 2) ? mb : 0u)];
        x[r] = mode == 2 ? rscale(p.x, x[r]) : cmul(p, x[r]);
      }
    }
    return;
  }
  // gathered side members never read rb / rb2 (build_plan): one product for all rows
  bool real;
  const V p = chain_side(cw.b, tab, arena, st.op0, st.nt - 1, j, lane, &real);
#pragma unroll
  for (int r = 0; r < 4; ++r) x[r] = real ? rscale(p.x, x[r]) : cmul(p, x[r]);
}

// One quad tile: NT stage-1 members (A = NT-2, B = NT-1), NS summed bits,
// K0: member 0 is the real |+> scale.
template <int NT, int NS, int K0>
__device__ __forceinline__ void chain_tile4(ChainWarp4& cw, const SegOpTab* __restrict__ tab,
                                            const DevSeg& sg, V* __restrict__ arena,
                                            uint32_t tile, int lane) {
  constexpr int IA = NT - 2, IB = NT - 1;
  constexpr int P0 = K0 ? 1 : 0;  // first gathered prefix member
  const int L = sg.nst;
  const uint32_t nj = 1u << (L - 1);
  const V* Bp[NT];
  uint32_t o[NT], sdl[NT], d0[NT];
  const R r0 = K0 ? __ldg(&(arena + __ldg(&tab[0].off))->x) : R(0);
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    Bp[t] = arena + __ldg(&tab[t].off);
    o[t] = cw.b.toff[t] + __ldg(&tab[t].llane[lane]);
    sdl[t] = __ldg(&tab[t].sd);
    d0[t] = __ldg(&tab[t].dj[0]);
  }
  const uint32_t da = cw.da[IA], db = cw.db[IB];
  const DevStage st2 = cw.b.st[1];
  V* y = arena + sg.out + (static_cast<uint64_t>(tile) << kSegYBits) + lane;
  const uint64_t ya = uint64_t{1} << (sg.rb + kSegYBits), yb = uint64_t{1} << (sg.rb2 + kSegYBits);
  for (uint32_t j = 0; j < nj; j += 2) {
    if (j) {
      const int b = __ffs(j) - 1;
#pragma unroll
      for (int t = 0; t < NT; ++t) o[t] += __ldg(&tab[t].inc[b]) + d0[t];
    }
    V x[4];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      V h[4];
#pragma unroll
      for (int s = 0; s <= NS; ++s) {
        const uint32_t oa = o[IA] + (q ? d0[IA] : 0u) + (s ? sdl[IA] : 0u);
        const uint32_t ob = o[IB] + (q ? d0[IB] : 0u) + (s ? sdl[IB] : 0u);
        const V a0 = ld(Bp[IA] + oa), a1 = ld(Bp[IA] + oa + da);
        const V b0 = ld(Bp[IB] + ob), b1 = ld(Bp[IB] + ob + db);
        V pa0, pa1;
        if constexpr (IA == P0) {  // no gathered prefix
          pa0 = K0 ? rscale(r0, a0) : a0;
          pa1 = K0 ? rscale(r0, a1) : a1;
        } else {
          V pf = ld(Bp[P0] + o[P0] + (q ? d0[P0] : 0u) + (s ? sdl[P0] : 0u));
          if (K0) pf = rscale(r0, pf);
#pragma unroll
          for (int t = P0 + 1; t < IA; ++t)
            pf = cmul(pf, ld(Bp[t] + o[t] + (q ? d0[t] : 0u) + (s ? sdl[t] : 0u)));
          pa0 = cmul(pf, a0);
          pa1 = cmul(pf, a1);
        }
        const V t0 = cmul(pa0, b0), t1 = cmul(pa1, b0), t2 = cmul(pa0, b1), t3 = cmul(pa1, b1);
        if (s == 0) {
          h[0] = t0;
          h[1] = t1;
          h[2] = t2;
          h[3] = t3;
        } else {
          h[0] = cadd(h[0], t0);
          h[1] = cadd(h[1], t1);
          h[2] = cadd(h[2], t2);
          h[3] = cadd(h[3], t3);
        }
      }
      chain_term4(cw, tab, arena, st2, 0, j | static_cast<uint32_t>(q), h, lane);
#pragma unroll
      for (int r = 0; r < 4; ++r) x[r] = q ? cadd(x[r], h[r]) : h[r];
    }
    const uint32_t jj = j | 1u;
    bool carry = true;
    for (int k = 1; k + 2 <= L; ++k) {
      chain_term4(cw, tab, arena, cw.b.st[k + 1], k, jj, x, lane);
      if (!((jj >> k) & 1u)) {
        cw.b.acc[k - 1][lane] = x[0];
        cw.b.acc1[k - 1][lane] = x[1];
        cw.acc2[k - 1][lane] = x[2];
        cw.acc3[k - 1][lane] = x[3];
        carry = false;
        break;
      }
      x[0] = cadd(cw.b.acc[k - 1][lane], x[0]);
      x[1] = cadd(cw.b.acc1[k - 1][lane], x[1]);
      x[2] = cadd(cw.acc2[k - 1][lane], x[2]);
      x[3] = cadd(cw.acc3[k - 1][lane], x[3]);
    }
    if (carry) {
      y[0] = x[0];
      y[ya] = x[1];
      y[yb] = x[2];
      y[ya + yb] = x[3];
    }
  }
}

// One work item of the loaded quad segment (the tile number without bits rb, rb2).
__device__ __forceinline__ void seg_tile4(ChainWarp4& cw, SegCursor& sc, uint32_t item,
                                          const DevTensor* __restrict__ trefs,
                                          const SegOpTab* __restrict__ segtab,
                                          V* __restrict__ arena, int lane) {
  const DevSeg& sg = sc.sg;
  const SegOpTab* tab = segtab + sg.tref;
  const uint32_t lo = min(sg.rb, sg.rb2), hi = max(sg.rb, sg.rb2);
  const uint32_t tile = insert_zero(insert_zero(item, lo), hi);
  for (int op = 0; op < sg.nops; ++op) {
    const uint32_t v = ((tile >> lane) & 1u) ? __ldg(&tab[op].dtile[lane]) : 0u;
    const uint32_t sum = __reduce_add_sync(kFull, v);
    if (lane == 0) cw.b.toff[op] = sum;
  }
  if (!sc.ptab_fresh || sc.ptab_tile) {
    chain_ptab_build(cw.b, sg, trefs, arena, tile, lane, static_cast<uint8_t>(kTileSrc + sg.rb),
                     static_cast<uint8_t>(kTileSrc + sg.rb2));
    sc.ptab_fresh = true;
  }
  __syncwarp();
  const DevStage s1 = cw.b.st[0];
  const bool k0 = s1.nt >= 3 && __ldg(&tab[0].kind) == kTensorRealScalar;
#ifdef QTNG_SASS_ONE_SHAPE
  chain_tile4<3, 1, 1>(cw, tab, sg, arena, tile, lane);
  return;
#endif
  switch (s1.nt * 4 + s1.ns * 2 + (k0 ? 1 : 0)) {
    case 8: chain_tile4<2, 0, 0>(cw, tab, sg, arena, tile, lane); break;
    case 10: chain_tile4<2, 1, 0>(cw, tab, sg, arena, tile, lane); break;
    case 12: chain_tile4<3, 0, 0>(cw, tab, sg, arena, tile, lane); break;
    case 13: chain_tile4<3, 0, 1>(cw, tab, sg, arena, tile, lane); break;
    case 14: chain_tile4<3, 1, 0>(cw, tab, sg, arena, tile, lane); break;
    case 15: chain_tile4<3, 1, 1>(cw, tab, sg, arena, tile, lane); break;
    case 16: chain_tile4<4, 0, 0>(cw, tab, sg, arena, tile, lane); break;
    case 17: chain_tile4<4, 0, 1>(cw, tab, sg, arena, tile, lane); break;
    case 18: chain_tile4<4, 1, 0>(cw, tab, sg, arena, tile, lane); break;
    default: chain_tile4<4, 1, 1>(cw, tab, sg, arena, tile, lane); break;
  }
  __syncwarp();
}

#ifndef QTNG_SEG_MINB
#define QTNG_SEG_MINB 28  // resident seg_kernel warps per SM the register budget must allow (72 regs)
#endif
#ifndef QTNG_SEG_WARPS
#define QTNG_SEG_WARPS 1  // warps per CTA (independent; fewer CTAs = less reserved shared memory)
#endif
#ifndef QTNG_SEG_GROUP
#define QTNG_SEG_GROUP (QTNG_SEG_WARPS > 1)  // CTAs take consecutive items (L1 sharing)
#endif
constexpr int kSegWarps = QTNG_SEG_WARPS;
__global__ void __launch_bounds__(32 * kSegWarps, QTNG_SEG_MINB / kSegWarps)
seg_kernel(const DevSeg* __restrict__ segs, const uint32_t* __restrict__ ibeg,
           const DevStage* __restrict__ stages, const DevTensor* __restrict__ trefs,
           const SegOpTab* __restrict__ segtab, V* __restrict__ arena, uint32_t seg_count,
           uint32_t items, uint32_t* ctr) {
#ifdef QTNG_NOOP_SEG  // launch-floor experiments only (tools/tune.py)
  return;
#endif
  __shared__ ChainWarp cws[kSegWarps];
  ChainWarp& cw = cws[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  // dynamic tile queue (segments are sorted by per-tile cost, largest first);
  // ctr[0] = next tile, ctr[1] = finished warps (CTAs); the last one resets both
  SegCursor sc;
  uint32_t cur_begin = 0, cur_end = 0;
#if QTNG_SEG_GROUP
  // the CTA's warps take kSegWarps CONSECUTIVE items per round: neighbouring
  // tiles share operand rows, so co-resident warps hit each other's L1 lines
  __shared__ uint32_t blk[2];
  const uint32_t wid = threadIdx.x >> 5;
  int ph = 0;
  if (threadIdx.x == 0) blk[0] = atomicAdd(ctr, static_cast<uint32_t>(kSegWarps));
  __syncthreads();
  for (;;) {
    const uint32_t base = blk[ph];
    if (base >= items) break;
    if (threadIdx.x == 0) blk[ph ^ 1] = atomicAdd(ctr, static_cast<uint32_t>(kSegWarps));
    const uint32_t item = base + wid;
    if (item < items) {
      if (sc.cur < 0 || item < cur_begin || item >= cur_end) {
        uint32_t lo = 0, hi = seg_count;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (__ldg(ibeg + mid) <= item) lo = mid; else hi = mid;
        }
        if (static_cast<int>(lo) != sc.cur) seg_switch(cw, sc, segs, static_cast<int>(lo), stages, segtab, lane);
        cur_begin = __ldg(ibeg + lo);
        cur_end = lo + 1 < seg_count ? __ldg(ibeg + lo + 1) : items;
      }
      seg_tile(cw, sc, item - cur_begin, trefs, segtab, arena, lane);
    }
    __syncthreads();
    ph ^= 1;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
  return;
#endif
  uint32_t nxt = 0;  // the next tile is fetched while the current one runs
  if (lane == 0) nxt = atomicAdd(ctr, 1u);
  for (;;) {
    const uint32_t item = __shfl_sync(kFull, nxt, 0);
    if (item >= items) break;
    if (lane == 0) nxt = atomicAdd(ctr, 1u);
    if (sc.cur < 0 || item < cur_begin || item >= cur_end) {
      uint32_t lo = 0, hi = seg_count;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(ibeg + mid) <= item) lo = mid; else hi = mid;
      }
      if (static_cast<int>(lo) != sc.cur) seg_switch(cw, sc, segs, static_cast<int>(lo), stages, segtab, lane);
      cur_begin = __ldg(ibeg + lo);
      cur_end = lo + 1 < seg_count ? __ldg(ibeg + lo + 1) : items;
    }
    seg_tile(cw, sc, item - cur_begin, trefs, segtab, arena, lane);
  }
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1u) == gridDim.x * kSegWarps - 1) {  // every warp has left the queue
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
}

#ifndef QTNG_SEG4_MINB
// resident seg4_kernel warps per SM the register budget must allow.  ASAP
// levels: 16 -> 2.206, 20 (96 regs) -> 2.151, 24 -> 2.149 ms; ALAP levels
// (bigger quad levels): 16 -> 1.897, 20 -> 1.873, 24 (80 regs) -> 1.862,
// 28 -> 1.934 ms (two interleaved passes each)
#define QTNG_SEG4_MINB 24
#endif
__global__ void __launch_bounds__(32, QTNG_SEG4_MINB)
seg4_kernel(const DevSeg* __restrict__ segs, const uint32_t* __restrict__ ibeg,
            const DevStage* __restrict__ stages, const DevTensor* __restrict__ trefs,
            const SegOpTab* __restrict__ segtab, V* __restrict__ arena, uint32_t seg_count,
            uint32_t items, uint32_t* ctr) {
#ifdef QTNG_NOOP_SEG  // launch-floor experiments only
  return;
#endif
  __shared__ ChainWarp4 cw;
  const int lane = threadIdx.x & 31;
  SegCursor sc;
  uint32_t cur_begin = 0, cur_end = 0;
  uint32_t nxt = 0;
  if (lane == 0) nxt = atomicAdd(ctr, 1u);
  for (;;) {
    const uint32_t item = __shfl_sync(kFull, nxt, 0);
    if (item >= items) break;
    if (lane == 0) nxt = atomicAdd(ctr, 1u);
    if (sc.cur < 0 || item < cur_begin || item >= cur_end) {
      uint32_t lo = 0, hi = seg_count;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(ibeg + mid) <= item) lo = mid; else hi = mid;
      }
      if (static_cast<int>(lo) != sc.cur) {
        seg_switch(cw.b, sc, segs, static_cast<int>(lo), stages, segtab, lane);
        seg_switch4(cw, sc.sg, segtab + sc.sg.tref, lane);
      }
      cur_begin = __ldg(ibeg + lo);
      cur_end = lo + 1 < seg_count ? __ldg(ibeg + lo + 1) : items;
    }
    seg_tile4(cw, sc, item - cur_begin, trefs, segtab, arena, lane);
  }
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {  // every warp has left the queue
      ctr[0] = 0;
      ctr[1] = 0;
    }
  }
}

// ---------------------------------------------------------------- dataflow
// flow_reset: the per-execution state of a flow program.
__global__ void flow_reset(const FlowUnit* __restrict__ units, uint32_t n_units,
                           const uint64_t* __restrict__ init, uint32_t n_init, uint32_t n_chunks,
                           uint32_t* __restrict__ done, int32_t* __restrict__ deps,
                           uint64_t* __restrict__ queue, FlowState* __restrict__ st) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_units) {
    done[i] = 0;
    deps[i] = units[i].deps;
  }
  if (i < n_chunks) queue[i] = i < n_init ? init[i] : kFlowEmpty;  // hot queue: [n_init, n_chunks)
  if (i == 0) {
    st->head = 0;
    st->tail = n_init;
    st->hot = n_init;
    st->done = 0;
  }
}

// Run one work item of a single-op unit (the level kernel's item code).
__device__ __forceinline__ void flow_op_item(const DevOp& op, uint32_t item,
                                             const DevTensor* __restrict__ trefs, V* __restrict__ arena,
                                             int lane, DevTensor* slot) {
  switch (op.nt) {
    case 1: dispatch_ns<1>(op, item, trefs, arena, lane, slot); break;
    case 2: dispatch_ns<2>(op, item, trefs, arena, lane, slot); break;
    case 3: dispatch_ns<3>(op, item, trefs, arena, lane, slot); break;
    case 4: dispatch_ns<4>(op, item, trefs, arena, lane, slot); break;
    case 5: dispatch_ns<5>(op, item, trefs, arena, lane, slot); break;
    case 6: dispatch_ns<6>(op, item, trefs, arena, lane, slot); break;
    case 7: dispatch_ns<7>(op, item, trefs, arena, lane, slot); break;
    default: dispatch_ns<8>(op, item, trefs, arena, lane, slot); break;
  }
}

// flow_kernel: a persistent warp claims the next queue position (one atomic),
// waits until that position is published, runs the chunk's items with the
// level-kernel or segment-kernel code, and counts them done; the warp that
// finishes a unit decrements its consumer's missing inputs and, at zero,
// appends all of the consumer's chunks to the queue.  Producers fence before
// counting, consumers fence after reading a published entry; outputs never
// share an arena region (no L1 line can be stale).
__global__ void __launch_bounds__(32, QTNG_SEG_MINB)
flow_kernel(const FlowUnit* __restrict__ units, uint32_t n_init, uint32_t n_chunks,
            const DevOp* __restrict__ ops,
            const DevSeg* __restrict__ segs, const DevStage* __restrict__ stages,
            const DevTensor* __restrict__ trefs, const SegOpTab* __restrict__ segtab,
            V* __restrict__ arena, uint32_t* __restrict__ done, int32_t* __restrict__ deps,
            volatile uint64_t* queue, FlowState* st) {
  __shared__ ChainWarp cw;
  __shared__ DevTensor slot[kMaxInputs];
  const int lane = threadIdx.x;
  SegCursor sc;
  for (;;) {
    uint64_t e = kFlowEmpty;
    bool quit = false;
    if (lane == 0) {
      // hot first (chain continuations) when some are published; else cold;
      // with cold exhausted, claim a hot position and wait for it -- every hot
      // position [n_init, n_chunks) is published exactly once
      const uint32_t h = *reinterpret_cast<volatile uint32_t*>(&st->hot);
      const uint32_t t = *reinterpret_cast<volatile uint32_t*>(&st->tail);
      uint32_t c = n_init;
      if (!(h < t) && *reinterpret_cast<volatile uint32_t*>(&st->head) < n_init)
        c = atomicAdd(&st->head, 1u);
      if (c < n_init) {
        e = queue[c];
      } else {
        const uint32_t p = atomicAdd(&st->hot, 1u);
        if (p >= n_chunks) {
          quit = true;
        } else {
          while ((e = queue[p]) == kFlowEmpty) __nanosleep(128);
        }
      }
      __threadfence();  // acquire: the producers' results are visible
    }
    if (__shfl_sync(kFull, quit ? 1 : 0, 0)) break;
    e = __shfl_sync(kFull, e, 0);
    const uint32_t u = static_cast<uint32_t>(e >> 32), c = static_cast<uint32_t>(e);
    const FlowUnit f = units[u];
    const uint32_t i0 = c << f.chunk_log, i1 = min(f.n_items, (c + 1) << f.chunk_log);
    if (f.kind) {
      if (sc.cur != static_cast<int>(f.idx)) seg_switch(cw, sc, segs, static_cast<int>(f.idx), stages, segtab, lane);
      for (uint32_t item = i0; item < i1; ++item) seg_tile(cw, sc, item, trefs, segtab, arena, lane);
    } else {
      const DevOp op = ops[f.idx];
      for (uint32_t item = i0; item < i1; ++item) flow_op_item(op, item, trefs, arena, lane, slot);
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();  // this chunk's results before its count
      if (atomicAdd(done + u, i1 - i0) + (i1 - i0) == f.n_items && f.succ >= 0) {
        __threadfence();
        if (atomicSub(deps + f.succ, 1) == 1) {  // the consumer is ready: publish its chunks
          const FlowUnit g = units[f.succ];
          const uint32_t nc = (g.n_items + (1u << g.chunk_log) - 1) >> g.chunk_log;
          const uint32_t base = atomicAdd(&st->tail, nc);
          for (uint32_t k = 0; k < nc; ++k)
            queue[base + k] = (static_cast<uint64_t>(f.succ) << 32) | k;
        }
      }
    }
  }
}

int seg_grid(uint32_t items) {
  static int cap = 0;
  if (cap == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#ifdef QTNG_SEG_CARVEOUT  // tuning: preferred shared-memory carveout (percent)
    cudaFuncSetAttribute(seg_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, QTNG_SEG_CARVEOUT);
#endif
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, seg_kernel, 32 * kSegWarps, 0);
    cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const uint32_t ctas = (items + kSegWarps - 1) / kSegWarps;
  return static_cast<int>(ctas < static_cast<uint32_t>(cap) ? (ctas > 0 ? ctas : 1) : cap);
}

// Per lightcone: e_jk = prod of its scalar results in production order
// (complex128 arithmetic also for complex64 plans).
__global__ void final_kernel(const uint64_t* __restrict__ scalar_off,
                             const uint32_t* __restrict__ lc_begin, int n_lc,
                             const V* __restrict__ arena, double2* __restrict__ terms,
                             const int32_t* __restrict__ lc_edge, double2* __restrict__ full) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_lc) return;
  double2 s = make_double2(1.0, 0.0);  // report.scalar = 1 (engine.cpp:253)
  for (uint32_t k = lc_begin[i]; k < lc_begin[i + 1]; ++k) {
    const V a = arena[scalar_off[k]];
    const double2 b = make_double2(static_cast<double>(a.x), static_cast<double>(a.y));
    s = make_double2(__dsub_rn(__dmul_rn(s.x, b.x), __dmul_rn(s.y, b.y)),
                     __dadd_rn(__dmul_rn(s.x, b.y), __dmul_rn(s.y, b.x)));
  }
  terms[i] = s;
  if (full) full[lc_edge[i]] = s;
}

template <int MAXT>
int resident_ctas() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, level_kernel<MAXT>, kThreads, 0);
    cached = sms * (per_sm > 0 ? per_sm : 1);
  }
  return cached;
}

template <int MAXT>
int grid_for(uint32_t items) {
  const uint32_t want = (items + kWarpsPerCta - 1) / kWarpsPerCta;
  const uint32_t cap = static_cast<uint32_t>(resident_ctas<MAXT>());
  return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
}

int outer_grid(uint32_t items) {
  static int cap = 0;
  if (cap == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, outer_kernel, kThreads, 0);
    cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const uint32_t want = (items + kWarpsPerCta - 1) / kWarpsPerCta;
  return static_cast<int>(want < static_cast<uint32_t>(cap) ? (want > 0 ? want : 1) : cap);
}

}  // namespace

cudaError_t launch_outer(cudaStream_t s, const DevOp* ops, const uint32_t* ibeg,
                         const DevTensor* trefs, void* arena_v, const LevelLaunch& lv) {
  if (lv.outer_items == 0) return cudaSuccess;
  V* arena = static_cast<V*>(arena_v);
  const uint32_t first = lv.op_begin + lv.op_count;
  outer_kernel<<<outer_grid(lv.outer_items), kThreads, 0, s>>>(ops + first, ibeg + first, trefs,
                                                               arena, lv.outer_count,
                                                               lv.outer_items);
  return cudaGetLastError();
}

cudaError_t launch_flow(cudaStream_t s, const FlowUnit* units, uint32_t n_units,
                        const uint64_t* init, uint32_t n_init, uint32_t n_chunks, const DevOp* ops,
                        const DevSeg* segs, const DevStage* stages, const DevTensor* trefs,
                        const SegOpTab* segtab, void* arena_v, uint32_t* done, int32_t* deps,
                        uint64_t* queue, FlowState* st) {
  if (n_units == 0) return cudaSuccess;
  const uint32_t n = n_units > n_chunks ? n_units : n_chunks;
  flow_reset<<<(n + 255) / 256, 256, 0, s>>>(units, n_units, init, n_init, n_chunks, done, deps,
                                             queue, st);
  static int cap = 0;
  if (cap == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, flow_kernel, 32, 0);
    cap = sms * (per_sm > 0 ? per_sm : 1);  // persistent: every CTA resident
  }
  flow_kernel<<<cap, 32, 0, s>>>(units, n_init, n_chunks, ops, segs, stages, trefs, segtab,
                                 static_cast<V*>(arena_v), done, deps, queue, st);
  return cudaGetLastError();
}

cudaError_t launch_seg_prep(cudaStream_t s, const DevSeg* segs, uint32_t n_segs,
                            const DevTensor* trefs, SegOpTab* segtab) {
  if (n_segs == 0) return cudaSuccess;
  seg_prep_kernel<<<(n_segs + 3) / 4, 128, 0, s>>>(segs, n_segs, trefs, segtab);
  return cudaGetLastError();
}

cudaError_t launch_segs(cudaStream_t s, const DevSeg* segs, const uint32_t* seg_ibeg,
                        const DevStage* stages, const DevTensor* trefs, const SegOpTab* segtab,
                        void* arena_v, uint32_t* ctr, const LevelLaunch& lv) {
  if (lv.seg_items == 0) return cudaSuccess;
  V* arena = static_cast<V*>(arena_v);
  seg_kernel<<<seg_grid(lv.seg_items), 32 * kSegWarps, 0, s>>>(
      segs + lv.seg_begin, seg_ibeg + lv.seg_begin, stages, trefs, segtab, arena, lv.seg_count,
      lv.seg_items, ctr);
  return cudaGetLastError();
}

int seg4_grid(uint32_t items) {
  static int cap = 0;
  if (cap == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, seg4_kernel, 32, 0);
    cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  return static_cast<int>(items < static_cast<uint32_t>(cap) ? (items > 0 ? items : 1) : cap);
}

cudaError_t launch_segs4(cudaStream_t s, const DevSeg* segs, const uint32_t* seg_ibeg,
                         const DevStage* stages, const DevTensor* trefs, const SegOpTab* segtab,
                         void* arena_v, uint32_t* ctr, const LevelLaunch& lv) {
  if (lv.seg4_items == 0) return cudaSuccess;
  V* arena = static_cast<V*>(arena_v);
  const uint32_t first = lv.seg_begin + lv.seg_count;
  seg4_kernel<<<seg4_grid(lv.seg4_items), 32, 0, s>>>(segs + first, seg_ibeg + first, stages, trefs,
                                                      segtab, arena, lv.seg4_count, lv.seg4_items,
                                                      ctr);
  return cudaGetLastError();
}

int level_grid(uint32_t items) { return grid_for<8>(items); }

int resident_warps() { return resident_ctas<4>() * kWarpsPerCta; }

cudaError_t launch_level(cudaStream_t s, const DevOp* ops, const uint32_t* ibeg,
                         const DevTensor* trefs, void* arena_v, const LevelLaunch& lv) {
  if (lv.items == 0) return cudaSuccess;
  V* arena = static_cast<V*>(arena_v);
  const DevOp* o = ops + lv.op_begin;
  const uint32_t* b = ibeg + lv.op_begin;
  if (lv.max_nt <= 2)
    level_kernel<2><<<grid_for<2>(lv.items), kThreads, 0, s>>>(o, b, trefs, arena, lv.op_count, lv.items);
  else if (lv.max_nt <= 4)
    level_kernel<4><<<grid_for<4>(lv.items), kThreads, 0, s>>>(o, b, trefs, arena, lv.op_count, lv.items);
  else if (lv.max_nt <= 6)
    level_kernel<6><<<grid_for<6>(lv.items), kThreads, 0, s>>>(o, b, trefs, arena, lv.op_count, lv.items);
  else
    level_kernel<8><<<grid_for<8>(lv.items), kThreads, 0, s>>>(o, b, trefs, arena, lv.op_count, lv.items);
  return cudaGetLastError();
}

cudaError_t launch_final(cudaStream_t s, const uint64_t* scalar_off, const uint32_t* lc_begin,
                         int n_lc, const void* arena_v, double2* terms, const int32_t* lc_edge,
                         double2* full) {
  if (n_lc <= 0) return cudaSuccess;
  const V* arena = static_cast<const V*>(arena_v);
  final_kernel<<<(n_lc + 127) / 128, 128, 0, s>>>(scalar_off, lc_begin, n_lc, arena, terms,
                                                  lc_edge, full);
  return cudaGetLastError();
}

}  // namespace QTNG_PREC_NS
}  // namespace qtng
