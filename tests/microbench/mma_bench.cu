// tcgen05 issue-rate microbenchmark (experiment, not product).
// One CTA per SM; the issuing warp runs n_groups groups of 8 MMAs (one K=128 / 128-key
// pass) with descriptors precomputed outside the loop, optionally committing after each
// group; cycles per MMA are written per CTA.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../../paper_2505_09326_b200/csrc/sm100.cuh"

using namespace fs::ptx;

// MODE 0: SS  M128 N128 (A,B K-major)          -- QK^T
// MODE 1: SS  M128 N256
// MODE 2: TS  M128 N128 (A tmem, B MN-major)   -- PV
// MODE 3: alternating groups MODE0 / MODE2     -- QK, PV interleaved, like FlashSign
// MODE 4: d=64 pattern: 4 SS M128N128 (QK, K=64) then 8 TS M128N64 (PV, 128 keys) per group
// MODE 5: 8 TS M128N64 only
template <int MODE, bool WARP, bool COMMIT, int NACC>
__global__ void __launch_bounds__(128, 1) mma_bench(int n_groups, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  // random bf16 operands (sign, exponent near 1, random mantissa): realistic multiplier toggling
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    const uint32_t lo = 0x3f00u | (x & 0x807fu), hi = 0x3f00u | ((x >> 16) & 0x807fu);
    reinterpret_cast<uint32_t*>(smem)[i] = lo | (hi << 16);
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_barrier_init(); }
  if (warp == 1) tmem_alloc(&tbase, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const bool active = WARP ? (warp == 0) : (threadIdx.x == 0);
  if (active) {
    const uint32_t a = smem_u32(smem), b = a + 32768, v = a + 65536;
    const uint64_t da = sdesc_sw128(a, 16, 1024), db = sdesc_sw128(b, 16, 1024), dv = sdesc_sw128(v, 32768, 1024);
    constexpr uint32_t id_qk = idesc_make(1, 1, 0, 0, 128, MODE == 1 ? 256 : 128);
    constexpr uint32_t id_pv = idesc_make(1, 1, 0, 1, 128, 128);
    const long long t0 = clock64();
    for (int g = 0; g < n_groups; ++g) {
      const bool leader = WARP ? elect_one() : true;
      const uint32_t acc = (NACC == 1) ? 0u : (uint32_t)(g & 1) * 128u;
      const bool do_pv = (MODE == 2) || (MODE == 3 && (g & 1));
      if (MODE >= 4) {
        if (leader) {
          constexpr uint32_t id_qk64 = idesc_make(1, 1, 0, 0, 128, 128);
          constexpr uint32_t id_pv64 = idesc_make(1, 1, 0, 1, 128, 64);
          if (MODE == 4) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) mma_f16_ss(tmem + acc, da + ks * 2, db + ks * 2, id_qk64, ks > 0);
          }
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            mma_f16_ts(tmem + 256 + (acc % 256) / 2, tmem + 448 + ks * 8, dv + ((ks * 2048) >> 4), id_pv64, ks > 0);
          if (COMMIT) tc_commit(&bar2);
        }
        if (WARP) __syncwarp();
        continue;
      }
      if (leader) {
        if (!do_pv) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint32_t off = ((ks >> 2) * 16384 + (ks & 3) * 32) >> 4;
            mma_f16_ss(tmem + acc, da + off, db + off, id_qk, ks > 0);
          }
        } else {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            mma_f16_ts(tmem + 256 + acc % 256, tmem + 448 + ks * 8, dv + ((ks * 2048) >> 4), id_pv, ks > 0);
        }
        if (COMMIT) tc_commit(&bar2);
      }
      if (WARP) __syncwarp();
    }
    if (!WARP || elect_one()) tc_commit(&bar);
    if (WARP) __syncwarp();
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE, bool WARP, bool COMMIT, int NACC>
static int run(int n_groups, int grid, unsigned long long* out_dev, float* ms) {
  auto k = mma_bench<MODE, WARP, COMMIT, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<grid, 128, 140 * 1024>>>(n_groups, out_dev);
  cudaEventRecord(e0);
  k<<<grid, 128, 140 * 1024>>>(n_groups, out_dev);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  return (err != cudaSuccess || cudaGetLastError() != cudaSuccess) ? 1 : 0;
}

#define CASE(M, W, C, N) \
  if (mode == M && warp_issue == W && commit == C && nacc == N) return run<M, W, C, N>(n_groups, grid, out_dev, ms);

extern "C" int run_mma_bench(int mode, int warp_issue, int commit, int nacc, int n_groups, int grid,
                             unsigned long long* out_dev, float* ms) {
  CASE(0, 0, 0, 1) CASE(0, 1, 0, 1) CASE(0, 1, 1, 1) CASE(0, 1, 1, 2) CASE(0, 0, 1, 2)
  CASE(1, 1, 0, 1) CASE(1, 1, 1, 1)
  CASE(2, 0, 0, 1) CASE(2, 1, 0, 1) CASE(2, 1, 1, 1) CASE(2, 1, 1, 2)
  CASE(3, 1, 0, 2) CASE(3, 1, 1, 2) CASE(3, 0, 1, 2)
  CASE(4, 1, 0, 2) CASE(4, 1, 1, 2) CASE(5, 1, 0, 1) CASE(5, 1, 1, 2)
  return 2;
}
