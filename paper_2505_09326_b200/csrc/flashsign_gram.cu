// flashsign_gram.cu -- the Gram form of spherical attention.
//
// With s_ij = c q_i . k_j, the spherical normaliser (normalizers.py:94-100) needs only two d x d
// moments of the key stream:
//     num_i = sum_j s_ij v_j = c q_i^T W,           W = sum_j k_j v_j^T
//     z_i   = sum_j s_ij^2   = c^2 q_i^T G q_i,     G = sum_j k_j k_j^T
//     O_i   = num_i / sqrt(z_i + eps)
// -- the same function as the reference's streamed loop (attention.py:146-200), exact in real
// arithmetic, at 8 N d^2 instead of 4 N^2 d flops per (b, h).  Three launches, all on the tensor
// cores (tcgen05, operands staged by TMA / bulk copies, accumulators in TMEM):
//
//   1. gram_kv_kernel     per (b, h_kv, key chunk): [G | W] partial = K^T [K | V] (d = 128) or
//                         [K | V]^T K = [G ; W^T] (d = 64), kind::f16 with both operands MN-major
//                         straight from the TMA tiles, fp32 in TMEM -> fp32 partials in global.
//   2. gram_reduce_kernel per (b, h_kv, 16 rows): sum the chunks, split W^T and G into 16-bit hi + lo terms
//                         (x = hi + lo to ~2^-16 relative) under one power-of-two scale each, and
//                         write them as the SW128 K-major shared-memory image of the B operand.
//   3. gram_apply_kernel  persistent over (b, h, 128-row query tile): T = Q [W^T ; G]^T with both
//                         terms accumulated into TMEM (M = 128, N = 2d, K = d), then per row
//                         z = c^2 sum_a T^G_a q_a, O = c T^W / sqrt(z + eps), the bad-row key of
//                         fs_fwd (first degenerate row in (batch, head, row) order) and the store.
//
// HBM-bound end to end: K and V are read once (launch 1), Q read and O written once (launch 3).
// Not the FlashSign loop -- a different algorithm for the same contract, kept beside it: it needs
// 16-bit inputs and the spherical normaliser (signed L1's |s| has no moment form).

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/flashsign.h"
#include "sm100.cuh"

namespace fs {

bool encode_bshd_shared(CUtensorMap* map, int in_dtype, const void* ptr, int head_dim, int seqlen, int heads,
                        int batch, const int64_t* stride, int box_w, int box_rows, std::string* err);
void set_last_error(const char* msg);

namespace gram {

constexpr int BK = 128;             // keys per K/V tile (launch 1) = query rows per tile (launch 3)
constexpr int kGramPrefetch = 0;    // apply kernel: L2 prefetch distance of Q tiles (FLASHSIGN_GRAM_PF)
#ifndef FS_GRAM_PROF
#define FS_GRAM_PROF 0  // diagnostic build: per-role wait counters of the apply kernel (fs_gram_prof_read)
#endif
#if FS_GRAM_PROF
__device__ unsigned long long g_gprof[8];
#define GPROF_ADD(i, v) atomicAdd(&g_gprof[i], (unsigned long long)(v))
#define GPROF_T() clock64()
#else
#define GPROF_ADD(i, v)
#define GPROF_T() 0ll
#endif
#ifndef FS_GRAM_NQB128
#define FS_GRAM_NQB128 3  // apply kernel, d = 128: Q tile buffers (227 KB of shared memory)
#endif
constexpr int BLK = BK * 128;       // one SW128 column block: 128 rows x 64 16-bit elements

template <int D>
struct KvCfg {
  static constexpr int NB = D / 64;                 // column blocks per operand tile
  static constexpr int STAGE = 2 * NB * BLK;        // K blocks, then V blocks (contiguous)
  static constexpr int STAGES = D == 128 ? 3 : 6;
  static constexpr int N = D == 128 ? 256 : 64;     // accumulator columns
  static constexpr int TCOLS = D == 128 ? 256 : 64;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 1024;
};

struct KvArgs {
  float* partial;   // [items][128][N] fp32
  float* amax;      // [B*H_kv][2] max |partial| of G, W over the chunks (zeroed before the launch)
  int n_chunks, chunk_tiles, n_kv_tiles, heads_kv;
};

template <int IN>
__host__ __device__ constexpr uint32_t fmt() { return IN == FS_BF16 ? 1u : 0u; }

// Launch 1: one CTA per (b, h_kv, chunk).  Warp 0 streams K / V tiles, warp 1 issues the MMAs,
// all four warps drain the accumulator.
template <int IN, int D>
__global__ void __launch_bounds__(128, 1)
    gram_kv_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v, KvArgs a) {
  using C = KvCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* done = empty + C::STAGES;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x;
  const int bh = item / a.n_chunks, chunk = item % a.n_chunks;
  const int b = bh / a.heads_kv, g = bh % a.heads_kv;
  const int t0 = chunk * a.chunk_tiles, t1 = min(a.n_kv_tiles, t0 + a.chunk_tiles);
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc(tbase, C::TCOLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tbase;
  if (warp == 0 && lane == 0) {
    const uint64_t pol = ptx::policy_evict_first();
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int s = i % C::STAGES;
      ptx::mbar_wait(&empty[s], ((i / C::STAGES) & 1u) ^ 1u);
      ptx::mbar_arrive_expect_tx(&full[s], C::STAGE);
      uint8_t* st = smem + s * C::STAGE;
#pragma unroll
      for (int nb = 0; nb < C::NB; ++nb) {
        ptx::tma_load_4d(st + nb * BLK, &tm_k, &full[s], nb * 64, t * BK, g, b, pol);
        ptx::tma_load_4d(st + (C::NB + nb) * BLK, &tm_v, &full[s], nb * 64, t * BK, g, b, pol);
      }
    }
  } else if (warp == 1) {
    const uint32_t lp = ptx::elect_one() ? 1u : 0u;
    // both operands MN-major (feature index contiguous within a 128-byte row, keys along K):
    // LBO = column-block stride, SBO = 8-row group stride; one K step = 16 keys = 2048 bytes
    constexpr uint32_t idesc = ptx::idesc_make(fmt<IN>(), fmt<IN>(), 1, 1, 128, C::N);
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int s = i % C::STAGES;
      ptx::mbar_wait(&full[s], (i / C::STAGES) & 1u);
      ptx::tc_fence_after();
      const uint32_t base = ptx::smem_u32(smem + s * C::STAGE);
#pragma unroll
      for (int ks = 0; ks < BK / 16; ++ks) {
        // d = 128: A = K^T (M = 128 features), B = [K | V]^T (N = 256);
        // d = 64:  A = [K | V]^T (M = 128: K's 64 features, then V's), B = K^T (N = 64)
        const uint64_t da = ptx::sdesc_sw128(base + ks * 2048, BLK, 1024);
        ptx::mma_f16_ss_p(tmem, da, da, idesc, (i > 0 || ks > 0) ? 1u : 0u, lp);
      }
      ptx::tc_commit_p(&empty[s], lp);
    }
    ptx::tc_commit_p(done, lp);
  }
  __syncwarp();
  const int row = warp * 32 + lane;
  float* dst = a.partial + static_cast<int64_t>(item) * 128 * C::N + row * C::N;
  if (t1 > t0) {
    ptx::mbar_wait(done, 0);
    ptx::tc_fence_after();
    float mx[2] = {0.f, 0.f};  // G, W parts of this row
#pragma unroll 1
    for (int c = 0; c < C::N / 32; ++c) {
      uint32_t r[32];
      ptx::tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c * 32, r);
      ptx::tmem_wait_ld();
      float cm = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 f = make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]),
                                     __uint_as_float(r[4 * k + 2]), __uint_as_float(r[4 * k + 3]));
        reinterpret_cast<float4*>(dst + c * 32)[k] = f;
        cm = fmaxf(cm, fmaxf(fmaxf(fabsf(f.x), fabsf(f.y)), fmaxf(fabsf(f.z), fabsf(f.w))));
      }
      if (D == 128 ? (c * 32 >= 128) : (row >= 64))
        mx[1] = fmaxf(mx[1], cm);
      else
        mx[0] = fmaxf(mx[0], cm);
    }
#pragma unroll
    for (int m = 0; m < 2; ++m) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx[m] = fmaxf(mx[m], __shfl_xor_sync(0xffffffffu, mx[m], o));
      // non-negative floats order like their bit patterns
      if (lane == 0) atomicMax(reinterpret_cast<int*>(a.amax) + 2 * bh + m, __float_as_int(mx[m]));
    }
  } else {
    for (int c = 0; c < C::N; c += 4) *reinterpret_cast<float4*>(dst + c) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, C::TCOLS);
  }
}

// B-operand image of launch 3 for one (b, h_kv): rows n < d hold W^T (row n = column n of W),
// rows d..2d-1 hold G; K = d columns; two terms (hi, lo), each SW128 K-major: column block kb of
// 64 elements = [2d rows][128 B], 16-byte chunk j of row n at chunk position j ^ (n & 7).
template <int D>
struct ImgCfg {
  static constexpr int ROWS = 2 * D;
  static constexpr int TERM = ROWS * D * 2;  // bytes per term
  static constexpr int BYTES = 2 * TERM;
};

template <int D>
__device__ __forceinline__ int img_offset(int n, int k) {  // element offset within one term
  const int kb = k >> 6, kk = k & 63;
  return kb * (ImgCfg<D>::ROWS * 64) + n * 64 + ((((kk >> 3) ^ (n & 7))) << 3) + (kk & 7);
}

template <int IN>
__device__ __forceinline__ uint16_t to16(float x) {
  if constexpr (IN == FS_BF16) return __bfloat16_as_ushort(__float2bfloat16_rn(x));
  else return __half_as_ushort(__float2half_rn(x));
}
template <int IN>
__device__ __forceinline__ float from16(uint16_t x) {
  if constexpr (IN == FS_BF16) return __bfloat162float(__ushort_as_bfloat16(x));
  else return __half2float(__ushort_as_half(x));
}

// Launch 2: grid (b*h_kv, 2d/16): each CTA writes 16 image rows.  A thread forms one 16-byte chunk
// (8 elements) of a row: the chunk sums of the moments, one power-of-two scale per moment and
// (b, h_kv) from launch 1's max |partial| (times the chunk count: a bound on max |sum|, keeping
// |x 2^-e| < 2^14, fp16-safe), then hi = rn(x), lo = rn(x - hi).
constexpr int RED_ROWS = 16;

template <int IN, int D>
__global__ void __launch_bounds__(128) gram_reduce_kernel(const float* __restrict__ partial, int n_chunks,
                                                          const float* __restrict__ amax, uint16_t* __restrict__ img,
                                                          float* __restrict__ scl) {
  constexpr int N = KvCfg<D>::N;
  constexpr int CPR = D / 8;  // 16-byte chunks per image row
  const int bh = blockIdx.x;
  int ex[2];
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const float am = amax[2 * bh + m] * static_cast<float>(n_chunks);
    ex[m] = (am > 0.f && isfinite(am)) ? ilogbf(am) - 13 : 0;
  }
  if (blockIdx.y == 0 && threadIdx.x == 0) {
    scl[2 * bh + 0] = exp2f(static_cast<float>(ex[1]));  // W
    scl[2 * bh + 1] = exp2f(static_cast<float>(ex[0]));  // G
  }
  const float* src = partial + static_cast<int64_t>(bh) * n_chunks * 128 * N;
  uint16_t* out = img + static_cast<int64_t>(bh) * (ImgCfg<D>::BYTES / 2);
  for (int e = threadIdx.x; e < RED_ROWS * CPR; e += blockDim.x) {
    const int n = blockIdx.y * RED_ROWS + e / CPR, k0 = (e % CPR) * 8;
    const int m = n < D ? 1 : 0;  // image rows: W^T first, then G
    float x[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int c = 0; c < n_chunks; ++c) {
      const float* pc = src + static_cast<int64_t>(c) * 128 * N;
      if (m == 0 || D == 64) {  // a contiguous run of one accumulator row
        const float* r = m == 0 ? pc + (n - D) * N + k0 : pc + (64 + n) * N + k0;
        const float4 u = *reinterpret_cast<const float4*>(r), w = *reinterpret_cast<const float4*>(r + 4);
        x[0] += u.x; x[1] += u.y; x[2] += u.z; x[3] += u.w;
        x[4] += w.x; x[5] += w.y; x[6] += w.z; x[7] += w.w;
      } else {  // d = 128: W^T[n][k] = W[k][n], a column of the accumulator
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] += pc[(k0 + u) * N + 128 + n];
      }
    }
    uint4 hi4, lo4;
    uint16_t* hp = reinterpret_cast<uint16_t*>(&hi4);
    uint16_t* lp = reinterpret_cast<uint16_t*>(&lo4);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float v = ldexpf(x[u], -ex[m]);
      hp[u] = to16<IN>(v);
      lp[u] = to16<IN>(v - from16<IN>(hp[u]));
    }
    const int off = img_offset<D>(n, k0);  // k0 % 8 == 0: the chunk's first element
    *reinterpret_cast<uint4*>(out + off) = hi4;
    *reinterpret_cast<uint4*>(out + ImgCfg<D>::TERM / 2 + off) = lo4;
  }
}

// NT: B-image terms applied -- 2 (hi + lo, ~2^-16: float32 outputs) or 1 (hi only, one rounding of
// the moments to the operand dtype, below a 16-bit output's own rounding); the smem the lo term
// would take holds four Q buffers instead of two (HBM latency x bandwidth needs ~3 in flight)
template <int D, int NT>
struct ApplyCfg {
  static constexpr int Q_BYTES = BK * D * 2;
  // Q buffers: as many as fit beside the B image (d = 128: 3 x 32 KB + 128 KB, with the barrier
  // block trimmed to 3 KB and no alignment slack -- the kernel checks the base is 1024-aligned);
  // the third buffer pays once the MMA issue loop is no longer the limit (C3 -5 %)
  static constexpr int NQB = NT == 1 ? 4 : (D == 128 ? FS_GRAM_NQB128 : 4);
  static constexpr int IMG_OFF = NQB * Q_BYTES;
  static constexpr int IMG_BYTES = NT * ImgCfg<D>::TERM;
  static constexpr int BAR_OFF = IMG_OFF + IMG_BYTES;
  static constexpr int BAR_BYTES = 3072;  // barriers (128 B) + the epilogue's z exchange (2 KB)
  static constexpr int SLACK = BAR_OFF + BAR_BYTES + 1024 <= 232448 ? 1024 : 0;
  static constexpr int SMEM = BAR_OFF + BAR_BYTES + SLACK;
  static_assert(SMEM <= 232448, "gram apply: shared memory");
  static_assert(NQB <= 4, "q_full / q_empty hold 4 barriers each");
  static constexpr int TN = 2 * D;  // accumulator columns per buffer
  static constexpr int TCOLS = 2 * TN;
};

struct ApplyArgs {
  void* o;
  int64_t o_sb, o_sn, o_sh;
  const uint16_t* img;
  const float* scl;
  uint64_t* bad_key;
  int heads_q, heads_kv, seqlen_q, head_dim, n_qt, n_tiles;
  float scale, eps;
  int pf;  // L2 prefetch distance for Q tiles (0: off)
};

template <int OUT>
__device__ __forceinline__ void store8(void* dst, const float* v) {
  if constexpr (OUT == FS_F32) {
    reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
  } else {
    uint4 w;
    uint32_t* wi = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (OUT == FS_BF16) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        wi[i] = *reinterpret_cast<uint32_t*>(&h);
      } else {
        __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
        wi[i] = *reinterpret_cast<uint32_t*>(&h);
      }
    }
    *reinterpret_cast<uint4*>(dst) = w;
  }
}

// Launch 3: persistent; CTA i takes a contiguous range of (b, h, query tile) so the B image of a
// (b, h_kv) is loaded once per run of tiles.  Warp 0: bulk / TMA loads; warp 1: MMAs; warps 2-9:
// epilogue (warp w reads TMEM lane quarter w % 4, column half (w - 2) / 4).
template <int IN, int D, int OUT>
__global__ void __launch_bounds__(320, 1) gram_apply_kernel(const __grid_constant__ CUtensorMap tm_q, ApplyArgs a) {
  constexpr int NT = 2;  // (1 -- hi only, four Q buffers -- measured no faster and outside bf16 tolerance)
  using C = ApplyCfg<D, NT>;
  constexpr int NB = D / 64;
  extern __shared__ uint8_t smem_raw[];
  if (C::SLACK == 0 && (ptx::smem_u32(smem_raw) & 1023u) != 0) __trap();  // layout needs an aligned base
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t *q_full = bars, *q_empty = bars + 4, *t_full = bars + 8, *t_empty = bars + 10;
  uint64_t *img_full = bars + 12, *img_empty = bars + 13;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(bars + 14);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = (a.n_tiles + gridDim.x - 1) / gridDim.x;
  const int tb0 = blockIdx.x * per, tb1 = min(a.n_tiles, tb0 + per);
  auto bhkv_of = [&](int tile) {
    const int bh = tile / a.n_qt;
    const int h = bh % a.heads_q, b = bh / a.heads_q;
    return b * a.heads_kv + static_cast<int>((static_cast<int64_t>(h) * a.heads_kv) / a.heads_q);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NQB; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 1 + 8);  // the MMAs' commit + the eight epilogue warps (they read q)
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&t_full[i], 1);
      ptx::mbar_init(&t_empty[i], 8);
    }
    ptx::mbar_init(img_full, 1);
    ptx::mbar_init(img_empty, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc(tbase, C::TCOLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tbase;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = ptx::policy_evict_first();
      int cur = -1, n_img = 0;
      for (int tile = tb0, it = 0; tile < tb1; ++tile, ++it) {
        const int kv = bhkv_of(tile);
        if (kv != cur) {
          if (n_img > 0) ptx::mbar_wait(img_empty, (n_img - 1) & 1u);
          ptx::mbar_arrive_expect_tx(img_full, C::IMG_BYTES);
          const uint8_t* src = reinterpret_cast<const uint8_t*>(a.img) + static_cast<int64_t>(kv) * ImgCfg<D>::BYTES;
          for (int off = 0; off < C::IMG_BYTES; off += 32768)
            ptx::bulk_load(smem + C::IMG_OFF + off, src + off, min(32768, C::IMG_BYTES - off), img_full);
          cur = kv;
          ++n_img;
        }
        const int qb = it % C::NQB;
        if (a.pf > 0) {
          // two Q buffers hold ~64 KB in flight per SM; the HBM latency x bandwidth product needs
          // ~160 KB: the tile `pf` ahead is pulled into L2 (each tile once), so its TMA load hits L2
          const int tp = tile + a.pf;
          if (tp < tb1) {
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
              ptx::tma_prefetch_l2_4d(&tm_q, nb * 64, (tp % a.n_qt) * BK, (tp / a.n_qt) % a.heads_q,
                                      (tp / a.n_qt) / a.heads_q);
          }
        }
        [[maybe_unused]] const long long tp0 = GPROF_T();
        ptx::mbar_wait(&q_empty[qb], ((it / C::NQB) & 1u) ^ 1u);
        GPROF_ADD(4, GPROF_T() - tp0);
        ptx::mbar_arrive_expect_tx(&q_full[qb], C::Q_BYTES);
        const int bh = tile / a.n_qt, qt = tile % a.n_qt;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
          ptx::tma_load_4d(smem + qb * C::Q_BYTES + nb * BLK, &tm_q, &q_full[qb], nb * 64, qt * BK, bh % a.heads_q,
                           bh / a.heads_q, pol);
      }
    }
  } else if (warp == 1) {
    const uint32_t lp = ptx::elect_one() ? 1u : 0u;
    constexpr uint32_t idesc = ptx::idesc_make(fmt<IN>(), fmt<IN>(), 0, 0, 128, C::TN);
    const uint64_t q_desc0 = ptx::sdesc_sw128(ptx::smem_u32(smem), 16, 1024);
    const uint64_t img_desc0 = ptx::sdesc_sw128(ptx::smem_u32(smem + C::IMG_OFF), 16, 1024);
    int cur = -1, n_img = 0;
    [[maybe_unused]] const long long tm0 = GPROF_T();
    for (int tile = tb0, it = 0; tile < tb1; ++tile, ++it) {
      const int kv = bhkv_of(tile);
      if (kv != cur) {
        ptx::mbar_wait(img_full, n_img & 1u);
        cur = kv;
        ++n_img;
      }
      const int qb = it % C::NQB, tb = it & 1;
      [[maybe_unused]] const long long tq0 = GPROF_T();
      ptx::mbar_wait(&q_full[qb], (it / C::NQB) & 1u);
      [[maybe_unused]] const long long tq1 = GPROF_T();
      ptx::mbar_wait(&t_empty[tb], ((it >> 1) & 1u) ^ 1u);
      if (lp) {
        GPROF_ADD(0, tq1 - tq0);
        GPROF_ADD(1, GPROF_T() - tq1);
        GPROF_ADD(3, 1);
      }
      ptx::tc_fence_after();
      // descriptors: one base per operand, per-step offsets are constants (address field in 16 B
      // units) -- rebuilding both descriptors per MMA held the issue loop at ~1.6x the MMA time
      const uint64_t a0 = q_desc0 + static_cast<uint32_t>((qb * C::Q_BYTES) >> 4);
#pragma unroll
      for (int term = 0; term < NT; ++term)
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off_a = ((ks * 32 / 128) * BLK + (ks * 32) % 128) >> 4;
          const uint32_t off_b =
              (term * ImgCfg<D>::TERM + (ks * 32 / 128) * (ImgCfg<D>::ROWS * 128) + (ks * 32) % 128) >> 4;
          ptx::mma_f16_ss_p(tmem + tb * C::TN, a0 + off_a, img_desc0 + off_b, idesc, (term > 0 || ks > 0) ? 1u : 0u, lp);
        }
      ptx::tc_commit_p(&t_full[tb], lp);
      ptx::tc_commit_p(&q_empty[qb], lp);
      if (tile + 1 >= tb1 || bhkv_of(tile + 1) != kv) ptx::tc_commit_p(img_empty, lp);
    }
    if (lp) GPROF_ADD(2, GPROF_T() - tm0);
  } else {
    // epilogue, 8 warps: warp w reads TMEM lane quarter w % 4 (rows r) and column half hf of both
    // moments -- partial z over its half of G's columns, exchanged with its partner warp (same
    // quarter, other half) through shared memory and a 64-thread named barrier, then its half of O
    constexpr int HD = D / 2;     // columns per half
    constexpr int NL = HD / 32;   // 32-column TMEM loads per half
    const int quarter = warp & 3, hf = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    float* zx = reinterpret_cast<float*>(bars + 16);  // [2 tiles][2 halves][128 rows]
    int cur_kv = -1;
    float sW = 0.f, sG = 0.f;  // the moments' scales, loaded once per run of tiles of a (b, h_kv)
    for (int tile = tb0, it = 0; tile < tb1; ++tile, ++it) {
      const int qb = it % C::NQB, tb = it & 1;
      const int bh = tile / a.n_qt, qt = tile % a.n_qt;
      const int kv = bhkv_of(tile);
      if (kv != cur_kv) {  // (issued before the accumulator wait: the load latency hides behind it)
        sW = a.scl[2 * kv];
        sG = a.scl[2 * kv + 1];
        cur_kv = kv;
      }
      // this row's half of q, straight from the swizzled Q tile as soon as it lands (the buffer is
      // released once the partial z below has consumed it)
      ptx::mbar_wait(&q_full[qb], (it / C::NQB) & 1u);
      const uint8_t* qrow = smem + qb * C::Q_BYTES + r * 128;
      uint4 qv[HD / 8];
#pragma unroll
      for (int j = 0; j < HD / 8; ++j) {  // 16-byte chunk of the row: 8 elements
        const int chunk = hf * (HD / 8) + j, kb = chunk >> 3, cj = chunk & 7;
        qv[j] = *reinterpret_cast<const uint4*>(qrow + kb * BLK + ((cj ^ (r & 7)) << 4));
      }
      [[maybe_unused]] const long long te0 = GPROF_T();
      ptx::mbar_wait(&t_full[tb], (it >> 1) & 1u);
      if (warp == 2 && lane == 0) GPROF_ADD(5, GPROF_T() - te0);
      ptx::tc_fence_after();
      // partial z = sum over this half's columns a of T^G_a q_a
      uint32_t t[NL][32];
#pragma unroll
      for (int l = 0; l < NL; ++l) ptx::tmem_ld32(tmem + lane_off + tb * C::TN + D + hf * HD + l * 32, t[l]);
      ptx::tmem_wait_ld();
      float zs0 = 0.f, zs1 = 0.f;
#pragma unroll
      for (int l = 0; l < NL; ++l)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint16_t* e = reinterpret_cast<const uint16_t*>(&qv[l * 4 + j]);
#pragma unroll
          for (int u = 0; u < 8; u += 2) {
            zs0 = fmaf(__uint_as_float(t[l][j * 8 + u]), from16<IN>(e[u]), zs0);
            zs1 = fmaf(__uint_as_float(t[l][j * 8 + u + 1]), from16<IN>(e[u + 1]), zs1);
          }
        }
      // T^W half in flight while the partial z is exchanged
#pragma unroll
      for (int l = 0; l < NL; ++l) ptx::tmem_ld32(tmem + lane_off + tb * C::TN + hf * HD + l * 32, t[l]);
      float* zt = zx + (it & 1) * 256;
      zt[hf * 128 + r] = zs0 + zs1;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
      const float zsum = zt[r] + zt[128 + r];
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&t_empty[tb]);
        // Q buffer released only now that q has been consumed (the partial z above): an arrive
        // right after the shared loads let the next TMA load overwrite the tile before those
        // loads had returned (bad rows at C3 size, many tiles per CTA; tests/test_gpu_gram.py)
        ptx::mbar_arrive(&q_empty[qb]);
      }
      const int row = qt * BK + r;
      const bool live = row < a.seqlen_q;
      // the reference's z and denominator (normalizers.py:83-91); Gram rounding can leave a tiny
      // negative z where the exact one is 0
      const float z = a.scale * a.scale * fmaxf(zsum, 0.f) * sG;
      const float den = sqrtf(z + a.eps);
      const bool bad = !(den > 0.f) || isinf(den);
      if (hf == 0 && live && bad && a.bad_key != nullptr) {
        const uint64_t lin = static_cast<uint64_t>(bh) * a.seqlen_q + row;
        atomicMin(reinterpret_cast<unsigned long long*>(a.bad_key),
                  static_cast<unsigned long long>((lin << 32) | __float_as_uint(z)));
      }
      const float mul = a.scale * sW / den;
      const int h = bh % a.heads_q, b = bh / a.heads_q;
      using OT = typename std::conditional<OUT == FS_F32, float,
                                           typename std::conditional<OUT == FS_BF16, __nv_bfloat16, __half>::type>::type;
      OT* dst = reinterpret_cast<OT*>(a.o) + b * a.o_sb + static_cast<int64_t>(row) * a.o_sn + h * a.o_sh + hf * HD;
      if (live) {
#pragma unroll
        for (int l = 0; l < NL; ++l)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (hf * HD + l * 32 + j * 8 < a.head_dim) {
              float v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) v[u] = bad ? 0.f : __uint_as_float(t[l][j * 8 + u]) * mul;
              store8<OUT>(dst + l * 32 + j * 8, v);
            }
          }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, C::TCOLS);
  }
}

// ---------------------------------------------------------------------------------- host
struct Plan {
  int d, n_kv_tiles, n_chunks, chunk_tiles, items;
  int64_t partial_floats, img_bytes, scl_floats;
};

static int num_sms_now() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

static Plan plan_of(const fs_fwd_params* p) {
  Plan pl{};
  pl.d = p->head_dim > 64 ? 128 : 64;
  pl.n_kv_tiles = (p->seqlen_kv + BK - 1) / BK;
  const int64_t bhkv = static_cast<int64_t>(p->batch) * p->heads_kv;
  // enough (b, h_kv, chunk) items for two waves of CTAs, chunks of >= 4 tiles
  const int64_t want = bhkv > 0 ? (2LL * num_sms_now() + bhkv - 1) / bhkv : 1;
  pl.n_chunks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, std::max(1, pl.n_kv_tiles / 4))));
  pl.chunk_tiles = std::max(1, (pl.n_kv_tiles + pl.n_chunks - 1) / pl.n_chunks);
  pl.n_chunks = std::max(1, (pl.n_kv_tiles + pl.chunk_tiles - 1) / pl.chunk_tiles);
  pl.items = static_cast<int>(bhkv * pl.n_chunks);
  pl.partial_floats = static_cast<int64_t>(pl.items) * 128 * (pl.d == 128 ? 256 : 64);
  pl.img_bytes = bhkv * (pl.d == 128 ? ImgCfg<128>::BYTES : ImgCfg<64>::BYTES);
  pl.scl_floats = 4 * bhkv;  // scales, then the moments' max |partial|
  return pl;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t workspace_bytes(const Plan& pl) {
  return align256(pl.partial_floats * 4) + align256(pl.img_bytes) + align256(pl.scl_floats * 4);
}

template <int IN, int D>
static fs_status run(const fs_fwd_params* p, const Plan& pl, uint8_t* ws, cudaStream_t stream, std::string* err) {
  float* partial = reinterpret_cast<float*>(ws);
  uint16_t* img = reinterpret_cast<uint16_t*>(ws + align256(pl.partial_floats * 4));
  float* scl = reinterpret_cast<float*>(ws + align256(pl.partial_floats * 4) + align256(pl.img_bytes));
  float* amax = scl + pl.scl_floats / 2;
  if (cudaMemsetAsync(amax, 0, sizeof(float) * pl.scl_floats / 2, stream) != cudaSuccess) {
    *err = "cudaMemsetAsync failed";
    return FS_ERR_CUDA;
  }
  CUtensorMap tk, tv, tq;
  if (!encode_bshd_shared(&tk, IN, p->k, p->head_dim, p->seqlen_kv, p->heads_kv, p->batch, p->k_stride, 64, BK,
                          err) ||
      !encode_bshd_shared(&tv, IN, p->v, p->head_dim, p->seqlen_kv, p->heads_kv, p->batch, p->v_stride, 64, BK,
                          err) ||
      !encode_bshd_shared(&tq, IN, p->q, p->head_dim, p->seqlen_q, p->heads_q, p->batch, p->q_stride, 64, BK, err))
    return FS_ERR_UNSUPPORTED;
  // 1. moments per (b, h_kv, chunk)
  {
    auto kern = gram_kv_kernel<IN, D>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, KvCfg<D>::SMEM);
    KvArgs a{partial, amax, pl.n_chunks, pl.chunk_tiles, pl.n_kv_tiles, p->heads_kv};
    kern<<<pl.items, 128, KvCfg<D>::SMEM, stream>>>(tk, tv, a);
  }
  // 2. reduce + image
  {
    gram_reduce_kernel<IN, D><<<dim3(p->batch * p->heads_kv, 2 * D / RED_ROWS), 128, 0, stream>>>(
        partial, pl.n_chunks, amax, img, scl);
  }
  // 3. apply
  {
    ApplyArgs a;
    a.o = p->o;
    a.o_sb = p->o_stride[0];
    a.o_sn = p->o_stride[1];
    a.o_sh = p->o_stride[2];
    a.img = img;
    a.scl = scl;
    a.bad_key = p->bad_key;
    a.heads_q = p->heads_q;
    a.heads_kv = p->heads_kv;
    a.seqlen_q = p->seqlen_q;
    a.head_dim = p->head_dim;
    a.n_qt = (p->seqlen_q + BK - 1) / BK;
    const int64_t tiles = static_cast<int64_t>(a.n_qt) * p->heads_q * p->batch;
    if (tiles > INT32_MAX) return FS_ERR_UNSUPPORTED;
    a.n_tiles = static_cast<int>(tiles);
    a.scale = p->scale;
    a.eps = p->eps;
    {
      static const int pf_env = [] {
        const char* e = getenv("FLASHSIGN_GRAM_PF");
        return e ? atoi(e) : -1;
      }();
      a.pf = pf_env >= 0 ? pf_env : kGramPrefetch;
    }
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(tiles, num_sms_now())));
    auto go = [&](auto kern) {
      const int sm = ApplyCfg<D, 2>::SMEM;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      kern<<<grid, 320, sm, stream>>>(tq, a);
    };
    switch (p->out_dtype) {
      case FS_F32: go(gram_apply_kernel<IN, D, FS_F32>); break;
      case FS_BF16: go(gram_apply_kernel<IN, D, FS_BF16>); break;
      default: go(gram_apply_kernel<IN, D, FS_F16>); break;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("gram launch: ") + cudaGetErrorString(e);
    return FS_ERR_CUDA;
  }
  return FS_OK;
}

}  // namespace gram
}  // namespace fs

#if FS_GRAM_PROF
extern "C" int fs_gram_prof_read(unsigned long long* out8) {
  if (cudaMemcpyFromSymbol(out8, fs::gram::g_gprof, sizeof(unsigned long long) * 8) != cudaSuccess) return 1;
  unsigned long long z[8] = {0};
  return cudaMemcpyToSymbol(fs::gram::g_gprof, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" {

int64_t fs_gram_workspace_bytes(const fs_fwd_params* p) {
  if (!p || p->head_dim < 1 || p->head_dim > 128 || p->batch < 0 || p->heads_kv < 1) return 0;
  return static_cast<int64_t>(fs::gram::workspace_bytes(fs::gram::plan_of(p)));
}

fs_status fs_gram_fwd(const fs_fwd_params* p, void* workspace, int64_t workspace_bytes, fs_stream_t stream_) {
  using namespace fs::gram;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  auto fail = [](fs_status st, const std::string& m) {
    fs::set_last_error(m.c_str());
    return st;
  };
  if (!p) return fail(FS_ERR_CONFIG, "null params");
  if (p->batch < 0 || p->heads_q < 1 || p->heads_kv < 1 || p->seqlen_q < 0 || p->seqlen_kv < 0)
    return fail(FS_ERR_SHAPE, "negative or zero extents (batch>=0, heads>=1, seqlen>=0)");
  if (p->heads_q % p->heads_kv != 0) return fail(FS_ERR_CONFIG, "query heads must be a multiple of kv heads");
  if (p->in_dtype != FS_BF16 && p->in_dtype != FS_F16)
    return fail(FS_ERR_DTYPE, "fs_gram_fwd: in_dtype must be FS_F16 or FS_BF16");
  if (p->out_dtype != FS_F32 && p->out_dtype != FS_BF16 && p->out_dtype != FS_F16)
    return fail(FS_ERR_DTYPE, "out_dtype must be FS_F32, FS_BF16 or FS_F16");
  if (p->normalizer != FS_NORM_SPHERICAL)
    return fail(FS_ERR_UNSUPPORTED, "fs_gram_fwd: the moment form exists for the spherical normaliser only");
  if (p->key_scale) return fail(FS_ERR_UNSUPPORTED, "fs_gram_fwd: form K' = m K first (fs_scale_keys)");
  if (p->dev_scales || p->partial_only || p->kv_splits > 1)
    return fail(FS_ERR_UNSUPPORTED, "fs_gram_fwd: dev_scales / partials / splits are not supported");
  if (!std::isfinite(p->scale)) return fail(FS_ERR_CONFIG, "score_scale must be finite");
  if (!(p->eps >= 0.0f) || !std::isfinite(p->eps)) return fail(FS_ERR_CONFIG, "denom_epsilon must be finite and >= 0");
  if (p->head_dim < 1 || p->head_dim > 128 || p->head_dim % 8 != 0)
    return fail(FS_ERR_UNSUPPORTED, "head_dim must be a multiple of 8 in [8, 128]");
  if (static_cast<int64_t>(p->batch) * p->heads_q * p->seqlen_q > static_cast<int64_t>(UINT32_MAX))
    return fail(FS_ERR_UNSUPPORTED, "batch * heads_q * seqlen_q must be < 2^32");
  const int ob = p->out_dtype == FS_F32 ? 4 : 2;
  auto al16 = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15u) == 0; };
  if (!al16(p->q) || !al16(p->k) || !al16(p->v) || !al16(p->o)) return fail(FS_ERR_UNSUPPORTED, "16-byte alignment");
  for (int i = 0; i < 3; ++i)
    if ((p->q_stride[i] * 2) % 16 || (p->k_stride[i] * 2) % 16 || (p->v_stride[i] * 2) % 16 ||
        (p->o_stride[i] * ob) % 16)
      return fail(FS_ERR_UNSUPPORTED, "batch/token/head strides must be multiples of 16 bytes");
  if (p->bad_key) {
    cudaError_t e = cudaMemsetAsync(p->bad_key, 0xFF, sizeof(uint64_t), stream);
    if (e != cudaSuccess) return fail(FS_ERR_CUDA, cudaGetErrorString(e));
  }
  if (p->batch == 0 || p->seqlen_q == 0) return FS_OK;
  const Plan pl = plan_of(p);
  if (!workspace || workspace_bytes < static_cast<int64_t>(fs::gram::workspace_bytes(pl)) ||
      (reinterpret_cast<uintptr_t>(workspace) & 255u))
    return fail(FS_ERR_CONFIG, "fs_gram_fwd: a 256-byte aligned workspace of fs_gram_workspace_bytes(p) is required");
  std::string err;
  fs_status st;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  if (p->seqlen_kv == 0) {  // every row has z = 0: moments are zero (the kv kernel writes zeros)
    fs_fwd_params p2 = *p;
    p2.k = p2.v = p->q;
    for (int i = 0; i < 3; ++i) p2.k_stride[i] = p2.v_stride[i] = p->q_stride[i];
    p2.heads_kv = p->heads_kv;
    p2.seqlen_kv = 1;  // one (zero-multiplied) tile keeps the maps valid; chunk ranges are empty
    Plan pz = pl;
    pz.n_kv_tiles = 0;
    pz.chunk_tiles = 1;
    if (p->in_dtype == FS_BF16)
      st = pl.d == 128 ? run<FS_BF16, 128>(&p2, pz, ws, stream, &err) : run<FS_BF16, 64>(&p2, pz, ws, stream, &err);
    else
      st = pl.d == 128 ? run<FS_F16, 128>(&p2, pz, ws, stream, &err) : run<FS_F16, 64>(&p2, pz, ws, stream, &err);
  } else if (p->in_dtype == FS_BF16) {
    st = pl.d == 128 ? run<FS_BF16, 128>(p, pl, ws, stream, &err) : run<FS_BF16, 64>(p, pl, ws, stream, &err);
  } else {
    st = pl.d == 128 ? run<FS_F16, 128>(p, pl, ws, stream, &err) : run<FS_F16, 64>(p, pl, ws, stream, &err);
  }
  if (st != FS_OK) return fail(st, err);
  return FS_OK;
}

}  // extern "C"
