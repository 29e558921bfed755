// sm_100a kernels of the bucket-elimination path.
//
// level_kernel -- the generic fused bucket kernel.  One launch runs every
// bucket of one dependency level of ALL planned lightcones (tiny buckets cost
// no launch of their own).  The unit of work is a warp "item": 2^cb
// consecutive outputs of one bucket (cb <= 10, chosen per level by the
// planner so that small levels still spread over every SM).  An item is a
// set of 32-output "rows" (lanes = output bits 0..4).  Per item each lane
//   * decodes, once, every operand's bit-gather map into 32-bit partial
//     offsets: `lo` for its own output bits 0..4, `hi` for output bits >= 5 of
//     the row it will later broadcast, and d0/d1 = the operand strides of the
//     two register-tiling bits (offsets are additive over bits because every
//     output/summed bit maps to a distinct operand bit),
//   * then walks the item's rows 2^NR at a time (the rows differing in the
//     planner-chosen register bits): operand offset = lo + shfl(hi, row) +
//     {0, d0, d1, d0+d1}; an operand that lacks a register bit is loaded once
//     for both rows (warp-uniform branch), so outer-join buckets -- two large
//     operands over disjoint bits -- issue ~half the loads per output.
//     128-bit read-only loads of complex128, the product over operands in
//     bucket member order, accumulation over the summed assignments in
//     ascending order, one 128-bit store per output.
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

namespace qtng {

namespace {

constexpr int kThreads = 256;
constexpr int kWarpsPerCta = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kSmemOps = 4096;  // item_begin entries cached in shared memory

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  // (a.x*b.x - a.y*b.y, a.x*b.y + a.y*b.x), every product rounded.
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

__device__ __forceinline__ double2 ld(const double2* p) { return __ldg(p); }

// Product over the T operands of one summed assignment (left fold, member order).
template <int T>
__device__ __forceinline__ double2 chain(const double2* const* base, const uint32_t* off) {
  double2 p = ld(base[0] + off[0]);
#pragma unroll
  for (int t = 1; t < T; ++t) p = cmul(p, ld(base[t] + off[t]));
  return p;
}

// Insert a zero bit at position q of x (q < 32).
__device__ __forceinline__ uint32_t insert_zero(uint32_t x, uint32_t q) {
  const uint32_t low = x & ((1u << q) - 1u);
  return ((x >> q) << (q + 1)) | low;
}

// Per-lane decode of the op's operands (see the file comment).
template <int T, int NSM>
struct Decoded {
  const double2* base[T];
  uint32_t lo[T], hi[T], sa[T], sb[T], d0[T], d1[T];
};

template <int T, int NSM>
__device__ __forceinline__ void decode(const DevOp& op, uint64_t kbase, uint32_t my, int lane,
                                       const DevTensor* __restrict__ trefs,
                                       double2* __restrict__ arena, DevTensor* slot,
                                       Decoded<T, NSM>& D) {
  const uint64_t khi = kbase | (static_cast<uint64_t>(lane) << 5);  // lane = row for `hi`
  const uint32_t r0 = op.rb[0], r1 = op.rb[1];
  // Stage the op's operand descriptors in this warp's shared slot; the
  // per-axis decode then reads its source bits with broadcast LDS.
  {
    const uint4* src4 = reinterpret_cast<const uint4*>(trefs + op.tref);
    uint4* dst4 = reinterpret_cast<uint4*>(slot);
    if (lane < 3 * T) dst4[lane] = __ldg(src4 + lane);
    __syncwarp();
  }
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const DevTensor& d = slot[t];
    D.base[t] = arena + d.off;
    const int rank = d.rank;
    uint32_t l = 0, h = 0, a = 0, b = 0, x0 = 0, x1 = 0;
#pragma unroll 1
    for (int ax = 0; ax < rank; ++ax) {
      const uint32_t src = d.src[ax];
      const uint32_t bit = 1u << (rank - 1 - ax);
      if (src < 5) {
        l |= ((my >> src) & 1u) ? bit : 0u;
      } else if (src == r0) {
        x0 |= bit;
      } else if (src == r1) {
        x1 |= bit;
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
    D.lo[t] = l;
    D.hi[t] = h;
    D.sa[t] = a;
    D.sb[t] = b;
    D.d0[t] = x0;
    D.d1[t] = x1;
  }
  __syncwarp();  // the slot is rewritten by the warp's next item
}

// Loads of operand t for the (up to) four register-tile rows, deduplicated
// when the operand lacks a register bit (d == 0, warp-uniform).
template <int NR>
__device__ __forceinline__ void load_tile(const double2* p, uint32_t d0, uint32_t d1,
                                          double2 (&x)[1 << NR]) {
  x[0] = ld(p);
  if (NR >= 1) x[1] = d0 ? ld(p + d0) : x[0];
  if (NR >= 2) {
    if (d1) {
      x[2] = ld(p + d1);
      x[3] = d0 ? ld(p + d0 + d1) : x[2];
    } else {
      x[2] = x[0];
      x[3] = x[1];
    }
  }
}

// NSM: 0 => no summed bit, 1 => one summed bit.  NR: log2 rows per step.
template <int T, int NSM, int NR>
__device__ __forceinline__ void run_rows(const DevOp& op, uint32_t chunk,
                                         const DevTensor* __restrict__ trefs,
                                         double2* __restrict__ arena, int lane, DevTensor* slot) {
  const int cb = op.cb;
  const uint64_t kbase = static_cast<uint64_t>(chunk) << cb;
  const bool active = cb >= 5 || lane < (1 << cb);
  const uint32_t my = active ? lane : 0;
  Decoded<T, NSM> D;
  decode<T, NSM>(op, kbase, my, lane, trefs, arena, slot, D);
  // register bits relative to the row index (output bit 5 = row bit 0)
  const bool v0 = NR >= 1 && op.rb[0] != kNoBit;
  const bool v1 = NR >= 2 && op.rb[1] != kNoBit;
  const uint32_t q0 = v0 ? op.rb[0] - 5u : 0u, q1 = v1 ? op.rb[1] - 5u : 0u;
  const int rows = cb > 5 ? 1 << (cb - 5) : 1;
  const int steps = rows >> ((v0 ? 1 : 0) + (v1 ? 1 : 0));
  double2* out = arena + op.out + kbase + my;
  constexpr int J = 1 << NR;
  for (int it = 0; it < steps; ++it) {
    uint32_t e = it;
    if (v0) e = insert_zero(e, q0);
    if (v1) e = insert_zero(e, q1);
    const double2* p[T];
#pragma unroll
    for (int t = 0; t < T; ++t) p[t] = D.base[t] + D.lo[t] + __shfl_sync(kFull, D.hi[t], e);
    double2 acc[J];
#pragma unroll
    for (int s = 0; s < (NSM == 1 ? 2 : 1); ++s) {
      double2 prod[J];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        double2 x[J];
        load_tile<NR>(p[t] + (s ? D.sa[t] : 0u), D.d0[t], D.d1[t], x);
#pragma unroll
        for (int j = 0; j < J; ++j) prod[j] = t == 0 ? x[j] : cmul(prod[j], x[j]);
      }
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] = s == 0 ? prod[j] : cadd(acc[j], prod[j]);
    }
    if (active) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        if ((j & 1) && !v0) continue;
        if ((j & 2) && !v1) continue;
        const uint32_t row = e | ((j & 1) ? 1u << q0 : 0u) | ((j & 2) ? 1u << q1 : 0u);
        out[static_cast<uint64_t>(row) << 5] = acc[j];
      }
    }
  }
}

// Two or more summed bits (merged buckets): one row at a time, the summed
// assignments enumerated in ascending order through two shuffle tables.
template <int T>
__device__ __forceinline__ void run_multisum(const DevOp& op, uint32_t chunk,
                                             const DevTensor* __restrict__ trefs,
                                             double2* __restrict__ arena, int lane,
                                             DevTensor* slot) {
  const int cb = op.cb;
  const uint64_t kbase = static_cast<uint64_t>(chunk) << cb;
  const bool active = cb >= 5 || lane < (1 << cb);
  const uint32_t my = active ? lane : 0;
  Decoded<T, 2> D;
  decode<T, 2>(op, kbase, my, lane, trefs, arena, slot, D);
  const int rows = cb > 5 ? 1 << (cb - 5) : 1;
  double2* out = arena + op.out + kbase + my;
  const int ns = op.ns;
  const int n_hi = ns > 5 ? 1 << (ns - 5) : 1;
  const int n_lo = ns > 5 ? 32 : 1 << ns;
  for (int e = 0; e < rows; ++e) {
    uint32_t off[T];
#pragma unroll
    for (int t = 0; t < T; ++t) off[t] = D.lo[t] + __shfl_sync(kFull, D.hi[t], e);
    double2 acc = make_double2(0.0, 0.0);
    bool first = true;
    for (int sh = 0; sh < n_hi; ++sh) {
      uint32_t offh[T];
#pragma unroll
      for (int t = 0; t < T; ++t) offh[t] = off[t] + __shfl_sync(kFull, D.sb[t], sh);
      for (int sl = 0; sl < n_lo; ++sl) {
        uint32_t o[T];
#pragma unroll
        for (int t = 0; t < T; ++t) o[t] = offh[t] + __shfl_sync(kFull, D.sa[t], sl);
        const double2 p = chain<T>(D.base, o);
        acc = first ? p : cadd(acc, p);
        first = false;
      }
    }
    if (active) out[static_cast<uint64_t>(e) << 5] = acc;
  }
}

template <int T>
__device__ __forceinline__ void dispatch_ns(const DevOp& op, uint32_t chunk,
                                            const DevTensor* __restrict__ trefs,
                                            double2* __restrict__ arena, int lane,
                                            DevTensor* slot) {
  if (op.ns == 1) {
    if (T <= 4 && op.rb[1] != kNoBit) run_rows<T, 1, (T <= 4 ? 2 : 1)>(op, chunk, trefs, arena, lane, slot);
    else run_rows<T, 1, 1>(op, chunk, trefs, arena, lane, slot);
  } else if (op.ns == 0) {
    run_rows<T, 0, 1>(op, chunk, trefs, arena, lane, slot);
  } else {
    run_multisum<T>(op, chunk, trefs, arena, lane, slot);
  }
}

// MAXT: the widest member list among the level's ops; smaller instantiations
// need fewer registers and run at higher occupancy.
template <int MAXT>
__global__ void __launch_bounds__(kThreads, MAXT <= 2 ? 3 : 2)
level_kernel(const DevOp* __restrict__ ops, const uint32_t* __restrict__ ibeg,
             const DevTensor* __restrict__ trefs, double2* __restrict__ arena,
             uint32_t op_count, uint32_t items) {
  __shared__ DevTensor slots[kWarpsPerCta][MAXT];
  __shared__ uint32_t sbeg[kSmemOps];
  const bool cached = op_count <= kSmemOps;
  if (cached)
    for (uint32_t i = threadIdx.x; i < op_count; i += kThreads) sbeg[i] = __ldg(ibeg + i);
  __syncthreads();
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

__global__ void final_kernel(const uint64_t* __restrict__ scalar_off,
                             const uint32_t* __restrict__ lc_begin, int n_lc,
                             const double2* __restrict__ arena, double2* __restrict__ terms) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_lc) return;
  double2 s = make_double2(1.0, 0.0);  // report.scalar = 1 (engine.cpp:253)
  for (uint32_t k = lc_begin[i]; k < lc_begin[i + 1]; ++k) s = cmul(s, arena[scalar_off[k]]);
  terms[i] = s;
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

}  // namespace

int level_grid(uint32_t items) { return grid_for<8>(items); }

int resident_warps() { return resident_ctas<4>() * kWarpsPerCta; }

cudaError_t launch_level(cudaStream_t s, const DevOp* ops, const uint32_t* ibeg,
                         const DevTensor* trefs, double2* arena, const LevelLaunch& lv) {
  if (lv.items == 0) return cudaSuccess;
  const DevOp* o = ops + lv.op_begin;
  const uint32_t* b = ibeg + lv.op_begin;
  if (lv.max_nt <= 2)
    level_kernel<2><<<grid_for<2>(lv.items), kThreads, 0, s>>>(o, b, trefs, arena, lv.op_count, lv.items);
  else if (lv.max_nt <= 4)
    level_kernel<4><<<grid_for<4>(lv.items), kThreads, 0, s>>>(o, b, trefs, arena, lv.op_count, lv.items);
  else
    level_kernel<8><<<grid_for<8>(lv.items), kThreads, 0, s>>>(o, b, trefs, arena, lv.op_count, lv.items);
  return cudaGetLastError();
}

cudaError_t launch_final(cudaStream_t s, const uint64_t* scalar_off, const uint32_t* lc_begin,
                         int n_lc, const double2* arena, double2* terms) {
  if (n_lc <= 0) return cudaSuccess;
  final_kernel<<<(n_lc + 127) / 128, 128, 0, s>>>(scalar_off, lc_begin, n_lc, arena, terms);
  return cudaGetLastError();
}

}  // namespace qtng
