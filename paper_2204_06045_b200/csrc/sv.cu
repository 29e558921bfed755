// sm_100a QAOA state-vector oracle: the reference's
// run_ansatz + expectation_cost (proj/src/statevector.cpp:9-84) for up to 33
// qubits in HBM (2^33 complex128 = 128 GiB), an independent check of the
// tensor-network energies at sizes the CPU oracle cannot reach (its cap is 24).
//
// Layout: amps[z], z's bit n-1-q = qubit q (qubit 0 is the MSB), in the
// context arena.  One layer = the phase of every edge fused into the first
// mixer pass, then the mixers of qubits 0..n-1 applied group by group: a CTA
// loads a tile spanning a group of <= kGroupBits qubit bits (plus the lowest
// kCoalBits bits, carried along so that global accesses stay 128-byte
// coalesced) into shared memory, applies that group's butterflies in qubit
// order and writes the tile back.  Every amplitude therefore sees exactly the
// reference's operation sequence -- phases in edge order, then the mixers in
// qubit order, each a std::complex product/sum with every product rounded --
// so the state is bit-identical to run_ansatz's.  Only the final sums over
// 2^n basis states are reassociated (a fixed-shape tree instead of one
// running sum), so energies agree to ~1e-15 relative.
//
// Roofline: HBM.  Each group pass reads and writes the state once (the
// phase rides along with the first), the expectation reads it once per 16
// edges: bytes per layer = groups * 2 * 16 * 2^n.
#include "sv.cuh"

#include <cstdint>

namespace qtng {

namespace {

constexpr int kSvThreads = 256;
constexpr int kCoalBits = 3;     // 8 consecutive amplitudes = 128 B per row
constexpr int kTileBits = 12;    // 4096 amplitudes = 64 KiB of shared memory
constexpr int kGroupBits = kTileBits - kCoalBits;
constexpr int kEdgeChunk = 16;   // edges per expectation pass

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

__global__ void sv_init(double2* __restrict__ amps, uint64_t dim, double amp) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t z = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; z < dim; z += stride)
    amps[z] = make_double2(amp, 0.0);
}

// One tile pass.  Tile bits: `gbits` group bits starting at bit `glo`, plus
// (when glo >= kCoalBits) the lowest kCoalBits bits; the tile index t packs
// [low bits | group bits].  The remaining bits enumerate the tiles.
// If phase_m > 0, every amplitude is first multiplied by w once per edge whose
// endpoints' bits differ (edge order), before the mixers.
__global__ void __launch_bounds__(kSvThreads)
sv_pass(double2* __restrict__ amps, int n, int glo, int gbits, int phase_m,
        const int2* __restrict__ phase_bits, double2 w, double2 c, double2 ms) {
  extern __shared__ double2 tile[];
  const bool carry = glo >= kCoalBits;
  const int lbits = carry ? kCoalBits : 0;
  const int tbits = gbits + lbits;
  const uint32_t tsize = 1u << tbits;
  // bits outside the tile, in ascending order, enumerate the tiles
  const int rest = n - tbits;
  const uint64_t n_tiles = uint64_t{1} << rest;
  for (uint64_t tile_id = blockIdx.x; tile_id < n_tiles; tile_id += gridDim.x) {
    // scatter tile_id's bits around the tile's bit ranges
    auto zof = [&](uint32_t t) -> uint64_t {
      uint64_t z = 0, r = tile_id;
      // low carried bits
      z |= carry ? (t & ((1u << kCoalBits) - 1u)) : 0;
      const uint32_t tg = carry ? (t >> kCoalBits) : t;
      z |= static_cast<uint64_t>(tg) << glo;
      // rest bits: [lbits, glo) then [glo + gbits, n)
      const int a0 = lbits, a1 = glo;  // range A
      const int na = a1 - a0;
      z |= (r & ((uint64_t{1} << na) - 1)) << a0;
      r >>= na;
      z |= r << (glo + gbits);
      return z;
    };
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < tsize; t += kSvThreads) {
      const uint64_t z = zof(t);
      double2 a = amps[z];
      for (int e = 0; e < phase_m; ++e) {
        const int2 b = phase_bits[e];
        if (((z >> b.x) ^ (z >> b.y)) & 1) a = cmul(a, w);
      }
      tile[t] = a;
    }
    __syncthreads();
    // mixers in qubit order = group bits from the highest down
    for (int gb = gbits - 1; gb >= 0; --gb) {
      const uint32_t mask = 1u << (gb + lbits);
      for (uint32_t h = threadIdx.x; h < tsize / 2; h += kSvThreads) {
        const uint32_t lo = h & (mask - 1u), t0 = ((h ^ lo) << 1) | lo, t1 = t0 | mask;
        const double2 a = tile[t0], b = tile[t1];
        tile[t0] = cadd(cmul(c, a), cmul(ms, b));
        tile[t1] = cadd(cmul(ms, a), cmul(c, b));
      }
      __syncthreads();
    }
    for (uint32_t t = threadIdx.x; t < tsize; t += kSvThreads) amps[zof(t)] = tile[t];
  }
}

// Per-CTA partial sums of sign_e(z) * |amp(z)|^2 for edges [e0, e0+ne).
__global__ void __launch_bounds__(kSvThreads)
sv_zz(const double2* __restrict__ amps, uint64_t dim, const int2* __restrict__ ebits, int e0,
      int ne, double* __restrict__ partial) {
  double acc[kEdgeChunk];
#pragma unroll
  for (int k = 0; k < kEdgeChunk; ++k) acc[k] = 0.0;
  int2 eb[kEdgeChunk];
#pragma unroll
  for (int k = 0; k < kEdgeChunk; ++k) eb[k] = k < ne ? ebits[e0 + k] : make_int2(0, 0);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kSvThreads;
  for (uint64_t z = blockIdx.x * static_cast<uint64_t>(kSvThreads) + threadIdx.x; z < dim; z += stride) {
    const double2 a = amps[z];
    const double p = __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));  // std::norm
#pragma unroll
    for (int k = 0; k < kEdgeChunk; ++k)
      if (k < ne) acc[k] += (((z >> eb[k].x) ^ (z >> eb[k].y)) & 1) ? -p : p;
  }
  // fixed-shape reduction: warp butterfly, then the CTA's warps in order
  __shared__ double red[kSvThreads / 32][kEdgeChunk];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kEdgeChunk; ++k) {
    double v = acc[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < ne) {
    double s = 0.0;
    for (int w = 0; w < kSvThreads / 32; ++w) s += red[w][threadIdx.x];
    partial[static_cast<uint64_t>(blockIdx.x) * kEdgeChunk + threadIdx.x] = s;
  }
}

__global__ void sv_zz_final(const double* __restrict__ partial, int blocks, int ne,
                            double* __restrict__ zz) {
  const int k = threadIdx.x;
  if (k >= ne) return;
  double s = 0.0;
  for (int b = 0; b < blocks; ++b) s += partial[static_cast<uint64_t>(b) * kEdgeChunk + k];
  zz[k] = s;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace

size_t sv_scratch_bytes(int m) {
  return sizeof(int2) * static_cast<size_t>(m) + sizeof(double) * static_cast<size_t>(m) +
         sizeof(double) * static_cast<size_t>(sm_count()) * 4 * kEdgeChunk;
}

cudaError_t sv_run(cudaStream_t s, double2* amps, int n, int m, const int2* phase_bits_dev,
                   int p, const double2* w, const double2* c, const double2* ms, double amp0,
                   void* scratch, double* zz_dev) {
  const uint64_t dim = uint64_t{1} << n;
  const int sms = sm_count();
  const int tile_smem = (1 << kTileBits) * static_cast<int>(sizeof(double2));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sv_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem);
    attr = true;
  }
  sv_init<<<sms * 8, kSvThreads, 0, s>>>(amps, dim, amp0);
  for (int k = 0; k < p; ++k) {
    // groups of qubit bits from the top: [hi - g, hi)
    int hi = n;
    bool first = true;
    while (hi > 0) {
      int glo = hi - kGroupBits;
      if (glo <= kCoalBits) glo = 0;           // the lowest group: contiguous tile
      const int gbits = hi - glo;
      const int tbits = gbits + (glo >= kCoalBits ? kCoalBits : 0);
      const uint64_t tiles = uint64_t{1} << (n - tbits);
      const int grid = static_cast<int>(tiles < static_cast<uint64_t>(sms) * 4 ? tiles : sms * 4);
      sv_pass<<<grid, kSvThreads, (1u << tbits) * sizeof(double2), s>>>(
          amps, n, glo, gbits, first ? m : 0, phase_bits_dev, w[k], c[k], ms[k]);
      first = false;
      hi = glo;
    }
  }
  const int blocks = sms * 4;
  double* partial = reinterpret_cast<double*>(static_cast<char*>(scratch) + sizeof(int2) * m +
                                              sizeof(double) * m);
  for (int e0 = 0; e0 < m; e0 += kEdgeChunk) {
    const int ne = m - e0 < kEdgeChunk ? m - e0 : kEdgeChunk;
    sv_zz<<<blocks, kSvThreads, 0, s>>>(amps, dim, phase_bits_dev, e0, ne, partial);
    sv_zz_final<<<1, kEdgeChunk, 0, s>>>(partial, blocks, ne, zz_dev + e0);
  }
  return cudaGetLastError();
}

}  // namespace qtng
