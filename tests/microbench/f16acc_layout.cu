// TMEM layout of a tcgen05 kind::f16 MMA with an f16 accumulator (experiment, not product):
// A[m][k] = (k == 0), B[n][k] = (k == 0) * n  =>  D[m][n] = n.  Reads TMEM back with
// tcgen05.ld 32x32b and prints what columns 0..7 of lane 5 hold, for D formats F32 and F16.
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2505_09326_b200/csrc/sm100.cuh"
using namespace fs::ptx;

template <int DFMT>  // 1 = F32, 0 = F16
__global__ void k(uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int N = 64;
  uint8_t* A = sm;            // 128 rows x 128 B
  uint8_t* B = sm + 128 * 128;  // 64 rows x 128 B
  for (int i = threadIdx.x; i < (128 + 64) * 128 / 2; i += blockDim.x) reinterpret_cast<__half*>(sm)[i] = __float2half(0.f);
  __syncthreads();
  if (threadIdx.x < 128) {  // element (r, 0): chunk 0 ^ (r % 8)
    const int r = threadIdx.x;
    *reinterpret_cast<__half*>(A + r * 128 + ((0 ^ (r & 7)) << 4)) = __float2half(1.f);
    if (r < N) *reinterpret_cast<__half*>(B + r * 128 + ((0 ^ (r & 7)) << 4)) = __float2half(float(r));
  }
  fence_proxy_async();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (threadIdx.x < 32) {
    const uint32_t lp = elect_one() ? 1u : 0u;
    const uint32_t idesc = (uint32_t(DFMT) << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24);
    mma_f16_ss_p(tm, sdesc_sw128(smem_u32(A), 16, 1024), sdesc_sw128(smem_u32(B), 16, 1024), idesc, 0u, lp);
    tc_commit_p(&bar, lp);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (threadIdx.x < 32) {
    uint32_t r[32];
    tmem_ld32(tm + (0u << 16), r);
    tmem_wait_ld();
    if (threadIdx.x == 5) for (int i = 0; i < 32; ++i) out[i] = r[i];
    uint32_t q[16];  // the same 32 columns, two 16-bit elements per register (pack::16b)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
                   "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
                 : "r"(tm) : "memory");
    tmem_wait_ld();
    if (threadIdx.x == 5) for (int i = 0; i < 16; ++i) out[32 + i] = q[i];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 64); }
}

int main() {
  uint32_t* d; cudaMalloc(&d, 256);
  uint32_t h[48];
  for (int f = 0; f < 2; ++f) {
    if (f == 0) { cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000); k<1><<<1, 128, 60000>>>(d); }
    else { cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000); k<0><<<1, 128, 60000>>>(d); }
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 192, cudaMemcpyDeviceToHost);
    printf("%s (%s): ", f == 0 ? "F32 acc" : "F16 acc", cudaGetErrorString(e));
    for (int i = 0; i < 8; ++i) {
      if (f == 0) printf("%g ", *reinterpret_cast<float*>(&h[i]));
      else { __half lo = *reinterpret_cast<__half*>(&h[i]); __half hi = *(reinterpret_cast<__half*>(&h[i]) + 1);
             printf("[%g|%g] ", __half2float(lo), __half2float(hi)); }
    }
    printf("\n   pack::16b: ");
    for (int i = 32; i < 36; ++i) { __half lo = *reinterpret_cast<__half*>(&h[i]); __half hi = *(reinterpret_cast<__half*>(&h[i]) + 1);
                                     printf("[%g|%g] ", __half2float(lo), __half2float(hi)); }
    printf("\n");
  }
  return 0;
}
