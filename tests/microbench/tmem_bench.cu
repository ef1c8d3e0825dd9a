// TMEM load/store throughput microbenchmark (experiment, not product).
// One CTA per SM, NW "reader" warps stream tcgen05.ld (various shapes) over TMEM,
// optionally writing packed halves back with tcgen05.st (the FlashSign norm pattern),
// optionally with one extra warp keeping the tensor core busy with SS MMAs into
// other TMEM columns.  Reports cycles per warp-iteration (4 KiB read per iteration).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../../paper_2505_09326_b200/csrc/sm100.cuh"

using namespace fs::ptx;

#define R8(i) "=r"(r[i + 0]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3]), "=r"(r[i + 4]), "=r"(r[i + 5]), \
              "=r"(r[i + 6]), "=r"(r[i + 7])
#define REGS32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}"

template <int SHAPE>
__device__ __forceinline__ void ld4k(uint32_t taddr, uint32_t* r) {
  if constexpr (SHAPE == 0)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " REGS32 ", [%32];"
                 : R8(0), R8(8), R8(16), R8(24) : "r"(taddr) : "memory");
  else if constexpr (SHAPE == 1)
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 " REGS32 ", [%32];"
                 : R8(0), R8(8), R8(16), R8(24) : "r"(taddr) : "memory");
  else if constexpr (SHAPE == 2)
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 " REGS32 ", [%32];"
                 : R8(0), R8(8), R8(16), R8(24) : "r"(taddr) : "memory");
  else
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 " REGS32 ", [%32];"
                 : R8(0), R8(8), R8(16), R8(24) : "r"(taddr) : "memory");
}

// columns covered by one 4 KiB warp load of each shape
template <int SHAPE>
__host__ __device__ constexpr int cols4k() { return SHAPE == 0 ? 32 : SHAPE == 1 ? 64 : SHAPE == 2 ? 64 : 64; }

// MODE 0: ld only; MODE 1: ld + st16 (packed half back, the norm pattern); MODE 2: ld + st32
template <int SHAPE, int MODE, bool MMA>
__global__ void __launch_bounds__(512, 1) tmem_bench(int iters, int nw, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ unsigned long long cyc[16];
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&tbase, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  __shared__ int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (warp < nw) {
    const int quarter = warp & 3;
    // readers use columns [256, 512) when an MMA warp writes [0, 256)
    const uint32_t base = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + (MMA ? 256u : 0u);
    const int span = MMA ? 256 : 512;
    uint32_t acc = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t col = (it * cols4k<SHAPE>() * (MODE == 3 ? 2 : MODE == 4 ? 4 : 1)) % span;
      constexpr int LPW = MODE == 3 ? 2 : MODE == 4 ? 4 : 1;  // loads in flight per wait
      uint32_t r[32 * LPW];
#pragma unroll
      for (int l = 0; l < LPW; ++l) ld4k<SHAPE>(base + (col + l * cols4k<SHAPE>()) % span, r + 32 * l);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32 * LPW; ++i) acc ^= r[i];
      if constexpr (MODE == 1) {
        tmem_st16(base + col, r);
        tmem_wait_st();
      } else if constexpr (MODE == 2) {
        tmem_st32(base + col, r);
        tmem_wait_st();
      }
    }
    const long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) {
      cyc[warp] = (unsigned long long)(t1 - t0) + (acc == 0x12345678u ? 1 : 0);
      atomicAdd(&done, 1);
    }
  } else if (MMA && warp == nw) {
    const uint32_t a = smem_u32(smem), b = a + 32768;
    const uint64_t da = sdesc_sw128(a, 16, 1024), db = sdesc_sw128(b, 16, 1024);
    constexpr uint32_t id_qk = idesc_make(1, 1, 0, 0, 128, 128);
    int g = 0;
    while (*(volatile int*)&done < nw) {
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t off = ((ks >> 2) * 16384 + (ks & 3) * 32) >> 4;
          mma_f16_ss(tmem + (g & 1) * 128, da + off, db + off, id_qk, ks > 0);
        }
        tc_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, g & 1);
      ++g;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long mx = 0;
    for (int w = 0; w < nw; ++w) mx = cyc[w] > mx ? cyc[w] : mx;
    out[blockIdx.x] = mx;
  }
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int SHAPE, int MODE, bool MMA>
static int run(int iters, int nw, int grid, unsigned long long* out_dev, float* ms) {
  auto k = tmem_bench<SHAPE, MODE, MMA>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 32 * (nw + (MMA ? 1 : 0));
  k<<<grid, threads < 64 ? 64 : threads, 80 * 1024>>>(iters, nw, out_dev);
  cudaEventRecord(e0);
  k<<<grid, threads < 64 ? 64 : threads, 80 * 1024>>>(iters, nw, out_dev);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  if (err != cudaSuccess) printf("err %s\n", cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}

extern "C" int run_tmem_bench(int shape, int mode, int mma, int iters, int nw, int grid, unsigned long long* out,
                              float* ms) {
#define CASE(S, M, X) \
  if (shape == S && mode == M && mma == X) return run<S, M, X>(iters, nw, grid, out, ms);
  CASE(0, 0, 0) CASE(1, 0, 0) CASE(2, 0, 0) CASE(3, 0, 0)
  CASE(0, 1, 0) CASE(0, 2, 0) CASE(1, 1, 0)
  CASE(0, 0, 1) CASE(0, 1, 1) CASE(1, 0, 1)
  CASE(0, 3, 0) CASE(0, 4, 0) CASE(1, 3, 0) CASE(0, 3, 1)
#undef CASE
  return 2;
}
