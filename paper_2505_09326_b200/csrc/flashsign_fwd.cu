// flashsign_fwd.cu -- FlashSign (spherical attention) forward for sm_100a.
//
// Replaces the reference hot loop `_streamed_tiles` (pkg/src/ncstream/attention.py:146-200)
// behind `streamed_attention_array` / `multi_head_attention_array`
// (attention.py:252-279, 318-361).  Contract (normalizers.py:94-100):
//     O_i = c * sum_j s_ij v_j / sqrt(c^2 * sum_j s_ij^2 + eps),   s_ij = q_i . k_j
//
// One CTA owns NQT=2 query tiles of BM=128 rows of one (batch, head) and streams
// the K/V tiles of that head's kv-group through a TMA-fed shared-memory ring:
//
//   warp 0      TMA producer   Q tiles once, then K_j, V_j into a STAGES-deep ring
//   warp 1      MMA issuer     S_t = Q_t K_j^T  (tcgen05 SS, S in TMEM, fp32)
//                              O_t += P_t V_j   (tcgen05 TS: P read from TMEM, V MN-major)
//   warp 2      TMEM allocator (512 columns: O_0, O_1, S_0, S_1)
//   warps 4-7   norm WG 0      row r of tile 0: z += sum s^2 (registers), P = cvt(s) -> TMEM
//   warps 8-11  norm WG 1      same for tile 1, ping-ponging with WG 0
//
// Spherical normalisation has no exp and no running max, so O never needs
// rescaling: it stays in TMEM for the whole K/V stream and is scaled exactly
// once in the epilogue by c / sqrt(c^2 z + eps).  Zero padding is exact
// (a1(0)=a2(0)=0), so ragged N uses TMA out-of-bounds zero fill, no masking.
//
// MMA issue order per K/V tile j (keeps each norm WG a full two-MMA window):
//     QK0(j)  PV1(j-1)  QK1(j)  PV0(j)
// tcgen05 MMAs from one thread execute in issue order, so QK_t(j+1) may be
// issued right after PV_t(j) although both touch S_t's columns (P aliases S).

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/flashsign.h"
#include "sm100.cuh"

#ifndef FS_VARIANT
#define FS_VARIANT 0  // experiment knob (0 = production path)
#endif
#ifndef FS_TMA_ONCE
#define FS_TMA_ONCE 0  // experiment: load the ring once, then reuse stale tiles
#endif
#ifndef FS_PURE_MMA
#define FS_PURE_MMA 0  // experiment: MMA thread never waits on the norm warpgroups
#endif
#ifndef FS_SKIP_QK
#define FS_SKIP_QK 0
#endif
#ifndef FS_SKIP_PV
#define FS_SKIP_PV 0
#endif

namespace fs {

constexpr int BM = 128;  // query rows per Q tile (= TMEM lanes)
constexpr int BN = 128;  // keys per K/V tile
constexpr int NQT = 2;   // Q tiles per CTA
constexpr int NUM_THREADS = 384;
constexpr int TMEM_COLS = 512;

struct KParams {
  void* o;
  int64_t o_sb, o_sn, o_sh;
  int32_t heads_q, heads_kv, seqlen_q, seqlen_kv, head_dim;
  float g2;       // (scale * q_descale * k_descale)^2
  float out_mul;  // scale * q_descale * k_descale * v_descale / p_scale
  float eps;
  float p_scale;
  uint64_t* bad_key;
};

template <int IN>
struct InTraits;
template <>
struct InTraits<FS_BF16> {
  static constexpr int EB = 2, KSTEP = 16;
  static constexpr uint32_t FMT = 1;
  static constexpr bool F8 = false, CHECK_OVF = false;
  static constexpr float PMAX = 3.0e38f;
};
template <>
struct InTraits<FS_F16> {
  static constexpr int EB = 2, KSTEP = 16;
  static constexpr uint32_t FMT = 0;
  static constexpr bool F8 = false, CHECK_OVF = true;
  static constexpr float PMAX = 65504.0f;
};
template <>
struct InTraits<FS_E4M3> {
  static constexpr int EB = 1, KSTEP = 32;
  static constexpr uint32_t FMT = 0;
  static constexpr bool F8 = true, CHECK_OVF = true;
  static constexpr float PMAX = 448.0f;
};

template <int IN, int D>
struct Cfg {
  using TR = InTraits<IN>;
  static constexpr int EB = TR::EB;
  static constexpr int ROW_BYTES = D * EB;
  static_assert(ROW_BYTES % 128 == 0, "head_dim * elem_bytes must be a multiple of 128 B (SW128)");
  static constexpr int NDB = ROW_BYTES / 128;  // 128-byte column blocks per row
  static constexpr int BOXW = 128 / EB;        // elements per TMA box row
  static constexpr int Q_TILE_BYTES = BM * ROW_BYTES;
  static constexpr int SLOT_BYTES = BN * ROW_BYTES;
  static constexpr int STAGES = (SLOT_BYTES >= 32768) ? 4 : 6;
  static constexpr int RING_OFF = NQT * Q_TILE_BYTES;
  static constexpr int BAR_OFF = RING_OFF + STAGES * SLOT_BYTES;
  static constexpr int SMEM_BYTES = BAR_OFF + 256 + 1024;  // + barriers + alignment slack
  static constexpr int QK_STEPS = ROW_BYTES / 32;          // 32 B of K-dim per MMA
  static constexpr int PV_STEPS = BN / TR::KSTEP;
  static constexpr int P_COLS = BN * EB / 4;  // packed P columns per tile
  static constexpr uint32_t COL_O0 = 0;
  static constexpr uint32_t COL_S0 = NQT * D;
  static_assert(NQT * D + NQT * BN <= TMEM_COLS, "TMEM budget");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static constexpr uint32_t IDESC_QK = ptx::idesc_make(TR::FMT, TR::FMT, 0, 0, BM, BN);
  static constexpr uint32_t IDESC_PV = ptx::idesc_make(TR::FMT, TR::FMT, 0, 1, BM, D);
};

struct Bars {
  uint64_t q_full[NQT];
  uint64_t kv_full[8];
  uint64_t kv_empty[8];
  uint64_t s_full[NQT];
  uint64_t p_full[NQT];
  uint64_t o_full[NQT];
  uint32_t tmem_base;
};

template <int IN>
__device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <>
__device__ __forceinline__ uint32_t pack2<FS_BF16>(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
template <>
__device__ __forceinline__ uint32_t pack2<FS_F16>(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t pack4_e4m3(float a, float b, float c, float d) {
  const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
  const uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2(c, d), __NV_SATFINITE, __NV_E4M3);
  return lo | (hi << 16);
}

template <int OUT>
struct OutT;
template <>
struct OutT<FS_F32> {
  using T = float;
};
template <>
struct OutT<FS_BF16> {
  using T = __nv_bfloat16;
};
template <>
struct OutT<FS_F16> {
  using T = __half;
};

// Store 32 consecutive output columns [c0, c0+32) of one row, clipped to head_dim.
template <int OUT>
__device__ __forceinline__ void store32(typename OutT<OUT>::T* dst, const float* v, int c0, int head_dim) {
  if constexpr (OUT == FS_F32) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (c0 + 4 * k < head_dim)
        *reinterpret_cast<float4*>(dst + 4 * k) = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (c0 + 8 * k < head_dim) {
        uint4 w;
        w.x = pack2<OUT>(v[8 * k + 0], v[8 * k + 1]);
        w.y = pack2<OUT>(v[8 * k + 2], v[8 * k + 3]);
        w.z = pack2<OUT>(v[8 * k + 4], v[8 * k + 5]);
        w.w = pack2<OUT>(v[8 * k + 6], v[8 * k + 7]);
        *reinterpret_cast<uint4*>(dst + 8 * k) = w;
      }
    }
  }
}

template <int IN, int D, int OUT>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    flashsign_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const KParams p) {
  using C = Cfg<IN, D>;
  using TR = InTraits<IN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = ptx::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_s & 1023u)) & 1023u);
  const uint32_t smem_s = ptx::smem_u32(smem);
  Bars* bars = reinterpret_cast<Bars*>(smem + C::BAR_OFF);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int qblk = blockIdx.x;
  const int head = blockIdx.y;
  const int batch = blockIdx.z;
  const int head_kv = static_cast<int>((static_cast<int64_t>(head) * p.heads_kv) / p.heads_q);
  const int n_kv_tiles = (p.seqlen_kv + BN - 1) / BN;
  const int q_row0 = qblk * (NQT * BM);

  if (threadIdx.x == 32) {
#pragma unroll
    for (int t = 0; t < NQT; ++t) {
      ptx::mbar_init(&bars->q_full[t], 1);
      ptx::mbar_init(&bars->s_full[t], 1);
      ptx::mbar_init(&bars->p_full[t], 4);
      ptx::mbar_init(&bars->o_full[t], 1);
    }
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&bars->kv_full[s], 1);
      ptx::mbar_init(&bars->kv_empty[s], 1);
    }
    ptx::fence_barrier_init();
    ptx::fence_proxy_async();
  }
  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 2) ptx::tmem_alloc(&bars->tmem_base, TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol_q = ptx::policy_evict_first();
      const uint64_t pol_kv = ptx::policy_evict_last();
#pragma unroll
      for (int t = 0; t < NQT; ++t) {
        ptx::mbar_arrive_expect_tx(&bars->q_full[t], C::Q_TILE_BYTES);
#pragma unroll
        for (int db = 0; db < C::NDB; ++db)
          ptx::tma_load_4d(smem + t * C::Q_TILE_BYTES + db * (BM * 128), &tm_q, &bars->q_full[t], db * C::BOXW,
                           q_row0 + t * BM, head, batch, pol_q);
      }
      for (int i = 0; i < 2 * n_kv_tiles; ++i) {
        const int slot = i % C::STAGES;
        const int round = i / C::STAGES;
        if (FS_TMA_ONCE && round > 0) break;
        if (round > 0) ptx::mbar_wait(&bars->kv_empty[slot], (round - 1) & 1);
        ptx::mbar_arrive_expect_tx(&bars->kv_full[slot], C::SLOT_BYTES);
        const CUtensorMap* tm = (i & 1) ? &tm_v : &tm_k;
        const int key0 = (i >> 1) * BN;
#pragma unroll
        for (int db = 0; db < C::NDB; ++db)
          ptx::tma_load_4d(smem + C::RING_OFF + slot * C::SLOT_BYTES + db * (BN * 128), tm, &bars->kv_full[slot],
                           db * C::BOXW, key0, head_kv, batch, pol_kv);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the (warp-uniform) control flow and waits; one elected
    // lane issues.  Descriptors are built once; per-step offsets are constants, so
    // every MMA is a couple of uniform-register adds (~64 cycles of tensor work each).
    if (n_kv_tiles > 0) {
      const bool leader = ptx::elect_one();
      const uint64_t q_desc = ptx::sdesc_sw128(smem_s, 16, 1024);
      const uint64_t k_desc = ptx::sdesc_sw128(smem_s + C::RING_OFF, 16, 1024);
      const uint64_t v_desc = ptx::sdesc_sw128(smem_s + C::RING_OFF, BN * 128, 1024);
      auto qk = [&](int t, int slot) {
        if (FS_SKIP_QK) return;
        const uint64_t a0 = q_desc + static_cast<uint32_t>((t * C::Q_TILE_BYTES) >> 4);
        const uint64_t b0 = k_desc + static_cast<uint32_t>((slot * C::SLOT_BYTES) >> 4);
        const uint32_t d_tmem = tmem + C::COL_S0 + t * BN;
#pragma unroll
        for (int ks = 0; ks < C::QK_STEPS; ++ks) {
          const uint32_t off_a = ((ks * 32 / 128) * (BM * 128) + (ks * 32) % 128) >> 4;
          const uint32_t off_b = ((ks * 32 / 128) * (BN * 128) + (ks * 32) % 128) >> 4;
          if constexpr (TR::F8)
            ptx::mma_f8_ss(d_tmem, a0 + off_a, b0 + off_b, C::IDESC_QK, ks > 0);
          else
            ptx::mma_f16_ss(d_tmem, a0 + off_a, b0 + off_b, C::IDESC_QK, ks > 0);
        }
      };
      auto pv = [&](int t, int slot, bool acc) {
        if (FS_SKIP_PV) return;
        const uint64_t b0 = v_desc + static_cast<uint32_t>((slot * C::SLOT_BYTES) >> 4);
        const uint32_t a_tmem = tmem + C::COL_S0 + t * BN;
        const uint32_t d_tmem = tmem + C::COL_O0 + t * D;
#pragma unroll
        for (int ks = 0; ks < C::PV_STEPS; ++ks) {
          const uint32_t off_b = (ks * TR::KSTEP * 128) >> 4;
          const uint32_t at = a_tmem + ks * (TR::KSTEP * C::EB / 4);
          if constexpr (TR::F8)
            ptx::mma_f8_ts(d_tmem, at, b0 + off_b, C::IDESC_PV, (acc || ks > 0) ? 1u : 0u);
          else
            ptx::mma_f16_ts(d_tmem, at, b0 + off_b, C::IDESC_PV, (acc || ks > 0) ? 1u : 0u);
        }
      };
#pragma unroll
      for (int t = 0; t < NQT; ++t) ptx::mbar_wait(&bars->q_full[t], 0);
      ptx::tc_fence_after();
      // ring position of K_j (even loads) and V_j (odd loads)
      int k_slot = 0, k_phase = 0;
      int v_slot = 1 % C::STAGES, v_phase = (1 >= C::STAGES) ? 1 : 0;
      int prev_v_slot = 0;
      for (int j = 0; j < n_kv_tiles; ++j) {
        if (!FS_TMA_ONCE || 2 * j < C::STAGES) ptx::mbar_wait(&bars->kv_full[k_slot], k_phase);
        ptx::tc_fence_after();
        if (leader) {
          qk(0, k_slot);
          ptx::tc_commit(&bars->s_full[0]);
        }
        __syncwarp();
        if (j > 0) {
          if (!FS_PURE_MMA) ptx::mbar_wait(&bars->p_full[1], (j - 1) & 1);
          ptx::tc_fence_after();
          if (leader) {
            pv(1, prev_v_slot, j - 1 > 0);
            ptx::tc_commit(&bars->kv_empty[prev_v_slot]);
          }
          __syncwarp();
        }
        if (leader) {
          qk(1, k_slot);
          ptx::tc_commit(&bars->s_full[1]);
          ptx::tc_commit(&bars->kv_empty[k_slot]);
        }
        __syncwarp();
        if (!FS_TMA_ONCE || 2 * j + 1 < C::STAGES) ptx::mbar_wait(&bars->kv_full[v_slot], v_phase);
        if (!FS_PURE_MMA) ptx::mbar_wait(&bars->p_full[0], j & 1);
        ptx::tc_fence_after();
        if (leader) {
          pv(0, v_slot, j > 0);
          if (j == n_kv_tiles - 1) ptx::tc_commit(&bars->o_full[0]);
        }
        __syncwarp();
        prev_v_slot = v_slot;
        // advance both ring cursors by two loads
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          if (++k_slot == C::STAGES) { k_slot = 0; k_phase ^= 1; }
          if (++v_slot == C::STAGES) { v_slot = 0; v_phase ^= 1; }
        }
      }
      if (!FS_PURE_MMA) ptx::mbar_wait(&bars->p_full[1], (n_kv_tiles - 1) & 1);
      ptx::tc_fence_after();
      if (leader) {
        pv(1, prev_v_slot, n_kv_tiles - 1 > 0);
        ptx::tc_commit(&bars->kv_empty[prev_v_slot]);
        ptx::tc_commit(&bars->o_full[1]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ norm warpgroups
    const int t = (warp - 4) >> 2;  // Q tile owned by this warpgroup
    const int quarter = warp & 3;   // TMEM lane quarter this warp may access
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t s_addr = tmem + lane_off + C::COL_S0 + t * BN;
    const uint32_t o_addr = tmem + lane_off + C::COL_O0 + t * D;
    const float ps = p.p_scale;
    float z0 = 0.f, z1 = 0.f, z2 = 0.f, z3 = 0.f;
    float amax = 0.f;
    for (int j = 0; j < (FS_PURE_MMA ? 0 : n_kv_tiles); ++j) {
      ptx::mbar_wait(&bars->s_full[t], j & 1);
      ptx::tc_fence_after();
#if FS_VARIANT == 3
      // experiment: no TMEM traffic at all
#elif FS_VARIANT == 5
      {
        uint32_t s[128];
        ptx::tmem_ld32(s_addr + 0, s);
        ptx::tmem_ld32(s_addr + 32, s + 32);
        ptx::tmem_ld32(s_addr + 64, s + 64);
        ptx::tmem_ld32(s_addr + 96, s + 96);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 128; i += 4) {
          const float a = __uint_as_float(s[i]), b = __uint_as_float(s[i + 1]);
          const float c = __uint_as_float(s[i + 2]), d = __uint_as_float(s[i + 3]);
          z0 = fmaf(a, a, z0);
          z1 = fmaf(b, b, z1);
          z2 = fmaf(c, c, z2);
          z3 = fmaf(d, d, z3);
        }
        if constexpr (!TR::F8) {
#pragma unroll
          for (int i = 0; i < 64; ++i) s[i] = pack2<IN>(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1]));
          ptx::tmem_st32(s_addr, s);
          ptx::tmem_st32(s_addr + 32, s + 32);
        }
      }
#else
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t s[64];
#if FS_VARIANT == 1
#pragma unroll
        for (int i = 0; i < 64; ++i) s[i] = __float_as_uint((float)(lane + i));
#else
        ptx::tmem_ld32(s_addr + half * 64, s);
        ptx::tmem_ld32(s_addr + half * 64 + 32, s + 32);
        ptx::tmem_wait_ld();
#endif
#if FS_VARIANT != 2
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
          const float a = __uint_as_float(s[i]), b = __uint_as_float(s[i + 1]);
          const float c = __uint_as_float(s[i + 2]), d = __uint_as_float(s[i + 3]);
          z0 = fmaf(a, a, z0);
          z1 = fmaf(b, b, z1);
          z2 = fmaf(c, c, z2);
          z3 = fmaf(d, d, z3);
          if constexpr (TR::CHECK_OVF) amax = fmaxf(amax, fmaxf(fmaxf(fabsf(a), fabsf(b)), fmaxf(fabsf(c), fabsf(d))));
        }
        if constexpr (TR::F8) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            pk[i] = pack4_e4m3(ps * __uint_as_float(s[4 * i]), ps * __uint_as_float(s[4 * i + 1]),
                               ps * __uint_as_float(s[4 * i + 2]), ps * __uint_as_float(s[4 * i + 3]));
          ptx::tmem_st16(s_addr + half * 16, pk);
        } else {
          uint32_t pk[32];
          if (ps == 1.0f) {
#pragma unroll
            for (int i = 0; i < 32; ++i) pk[i] = pack2<IN>(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1]));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              pk[i] = pack2<IN>(ps * __uint_as_float(s[2 * i]), ps * __uint_as_float(s[2 * i + 1]));
          }
          ptx::tmem_st32(s_addr + half * 32, pk);
        }
#else
        z0 += __uint_as_float(s[half]);
#endif
      }
#endif
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&bars->p_full[t]);
    }
    // ------------------------------------------------------------ epilogue
    const float z = (z0 + z1) + (z2 + z3);
    const float zr = p.g2 * z;  // = sum_j (c s_ij)^2, what the reference calls z
    const float den = sqrtf(zr + p.eps);
    bool bad = !(den > 0.f) || isinf(den);
    float z_report = zr;
    if constexpr (TR::CHECK_OVF) {
      if (amax * fabsf(ps) > TR::PMAX) {
        bad = true;
        z_report = __int_as_float(0x7f800000);
      }
    }
    const int row = q_row0 + t * BM + r;
    if (n_kv_tiles > 0) {
      ptx::mbar_wait(&bars->o_full[t], 0);
      ptx::tc_fence_after();
    }
    using OT = typename OutT<OUT>::T;
    OT* dst = reinterpret_cast<OT*>(p.o) + batch * p.o_sb + static_cast<int64_t>(row) * p.o_sn + head * p.o_sh;
    const bool live = row < p.seqlen_q;
    if (live && bad && p.bad_key != nullptr) {
      const uint64_t lin = (static_cast<uint64_t>(batch) * p.heads_q + head) * p.seqlen_q + row;
      atomicMin(reinterpret_cast<unsigned long long*>(p.bad_key),
                static_cast<unsigned long long>((lin << 32) | __float_as_uint(z_report)));
    }
    const float mul = p.out_mul;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t acc[32];
      float v[32];
      ptx::tmem_ld32(o_addr + c * 32, acc);  // warp-collective: every lane participates
      ptx::tmem_wait_ld();
      if (n_kv_tiles == 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = 0u;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __fdiv_rn(mul * __uint_as_float(acc[i]), den);
      if (live && c * 32 < p.head_dim) store32<OUT>(dst + c * 32, v, c * 32, p.head_dim);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, TMEM_COLS);
  }
}

// ====================================================================== host

static thread_local std::string g_last_error;

static fs_status fail(fs_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

static bool encode_bshd(CUtensorMap* map, CUtensorMapDataType dt, int eb, const void* ptr, int head_dim, int seqlen,
                        int heads, int batch, const int64_t* stride, int box_w, std::string* err) {
  auto enc = get_encode_fn();
  if (!enc) {
    *err = "cuTensorMapEncodeTiled unavailable (driver too old?)";
    return false;
  }
  cuuint64_t dims[4] = {(cuuint64_t)head_dim, (cuuint64_t)(seqlen > 0 ? seqlen : 1), (cuuint64_t)heads,
                        (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)(stride[1] * eb), (cuuint64_t)(stride[2] * eb),
                           (cuuint64_t)(stride[0] * eb)};
  cuuint32_t box[4] = {(cuuint32_t)box_w, (cuuint32_t)BM, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, dt, 4, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r);
    return false;
  }
  return true;
}

template <int IN, int D, int OUT>
static fs_status launch(const fs_fwd_params* p, cudaStream_t stream) {
  using C = Cfg<IN, D>;
  auto kern = flashsign_fwd_kernel<IN, D, OUT>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  });
  if (attr_err != cudaSuccess)
    return fail(FS_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));

  const CUtensorMapDataType dt = (IN == FS_BF16)  ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                 : (IN == FS_F16) ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                  : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  CUtensorMap tq, tk, tv;
  std::string err;
  if (!encode_bshd(&tq, dt, C::EB, p->q, p->head_dim, p->seqlen_q, p->heads_q, p->batch, p->q_stride, C::BOXW, &err) ||
      !encode_bshd(&tk, dt, C::EB, p->k, p->head_dim, p->seqlen_kv, p->heads_kv, p->batch, p->k_stride, C::BOXW,
                   &err) ||
      !encode_bshd(&tv, dt, C::EB, p->v, p->head_dim, p->seqlen_kv, p->heads_kv, p->batch, p->v_stride, C::BOXW,
                   &err))
    return fail(FS_ERR_UNSUPPORTED, err);

  KParams kp;
  kp.o = p->o;
  kp.o_sb = p->o_stride[0];
  kp.o_sn = p->o_stride[1];
  kp.o_sh = p->o_stride[2];
  kp.heads_q = p->heads_q;
  kp.heads_kv = p->heads_kv;
  kp.seqlen_q = p->seqlen_q;
  kp.seqlen_kv = p->seqlen_kv;
  kp.head_dim = p->head_dim;
  const double g = (double)p->scale * p->q_descale * p->k_descale;
  kp.g2 = (float)(g * g);
  kp.out_mul = (float)(g * p->v_descale / p->p_scale);
  kp.eps = p->eps;
  kp.p_scale = p->p_scale;
  kp.bad_key = p->bad_key;

  dim3 grid((p->seqlen_q + NQT * BM - 1) / (NQT * BM), p->heads_q, p->batch);
  kern<<<grid, NUM_THREADS, C::SMEM_BYTES, stream>>>(tq, tk, tv, kp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return FS_OK;
}

template <int IN, int D>
static fs_status dispatch_out(const fs_fwd_params* p, cudaStream_t s) {
  switch (p->out_dtype) {
    case FS_F32:
      return launch<IN, D, FS_F32>(p, s);
    case FS_BF16:
      return launch<IN, D, FS_BF16>(p, s);
    case FS_F16:
      return launch<IN, D, FS_F16>(p, s);
    default:
      return fail(FS_ERR_DTYPE, "out_dtype must be FS_F32, FS_BF16 or FS_F16");
  }
}

}  // namespace fs

static fs_status fs_fwd_dispatch(const fs_fwd_params* p, cudaStream_t stream) {
  using namespace fs;

  if (p->in_dtype == FS_E4M3) {
    // 1-byte rows: the SW128 layout needs 128-byte rows -> D = 128 (TMA zero-fills d >= head_dim).
    return dispatch_out<FS_E4M3, 128>(p, stream);
  }
  const bool d64 = p->head_dim <= 64;
  if (p->in_dtype == FS_BF16) return d64 ? dispatch_out<FS_BF16, 64>(p, stream) : dispatch_out<FS_BF16, 128>(p, stream);
  return d64 ? dispatch_out<FS_F16, 64>(p, stream) : dispatch_out<FS_F16, 128>(p, stream);
}


extern "C" {

const char* fs_last_error(void) { return fs::g_last_error.c_str(); }

int fs_version(void) { return 100; }

int fs_query_tile(int head_dim, fs_dtype dt, int* bm, int* bn) {
  if (!bm || !bn || head_dim < 1 || head_dim > 128) return 1;
  if (dt != FS_F16 && dt != FS_BF16 && dt != FS_E4M3) return 1;
  *bm = fs::BM;
  *bn = fs::BN;
  return 0;
}

fs_status fs_fwd(const fs_fwd_params* p, fs_stream_t stream_) {
  using namespace fs;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (!p) return fail(FS_ERR_CONFIG, "null params");
  if (p->batch < 0 || p->heads_q < 1 || p->heads_kv < 1 || p->seqlen_q < 0 || p->seqlen_kv < 0)
    return fail(FS_ERR_SHAPE, "negative or zero extents (batch>=0, heads>=1, seqlen>=0)");
  if (p->heads_q % p->heads_kv != 0)
    return fail(FS_ERR_CONFIG, "query heads must be a multiple of kv heads, got h=" + std::to_string(p->heads_q) +
                                   ", h_kv=" + std::to_string(p->heads_kv));
  if (!(std::isfinite(p->scale)))  // 0 is allowed: every row is then degenerate unless eps > 0
    return fail(FS_ERR_CONFIG, "score_scale must be finite");
  if (!(p->eps >= 0.0f) || !std::isfinite(p->eps)) return fail(FS_ERR_CONFIG, "denom_epsilon must be finite and >= 0");
  if (!(std::isfinite(p->p_scale)) || p->p_scale <= 0.0f || !(p->q_descale > 0.0f) || !(p->k_descale > 0.0f) ||
      !(p->v_descale > 0.0f))
    return fail(FS_ERR_CONFIG, "p_scale and descales must be finite and positive");
  if (p->in_dtype != FS_BF16 && p->in_dtype != FS_F16 && p->in_dtype != FS_E4M3)
    return fail(FS_ERR_DTYPE, "in_dtype must be FS_F16, FS_BF16 or FS_E4M3");
  const int eb = p->in_dtype == FS_E4M3 ? 1 : 2;
  const int ob = p->out_dtype == FS_F32 ? 4 : 2;
  if (p->head_dim < 1 || p->head_dim > 128)
    return fail(FS_ERR_UNSUPPORTED, "head_dim must be in [1, 128], got " + std::to_string(p->head_dim));
  if ((p->head_dim * eb) % 16 != 0)
    return fail(FS_ERR_UNSUPPORTED, "head_dim * elem_bytes must be a multiple of 16 (pad the head dim)");
  if (p->heads_q > 65535 || p->batch > 65535) return fail(FS_ERR_UNSUPPORTED, "heads/batch must be <= 65535");
  auto aligned16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; };
  if (!aligned16(p->q) || !aligned16(p->k) || !aligned16(p->v) || !aligned16(p->o))  // NULL is aligned
    return fail(FS_ERR_UNSUPPORTED, "q/k/v/o must be 16-byte aligned");
  for (int i = 0; i < 3; ++i) {
    if ((p->q_stride[i] * eb) % 16 || (p->k_stride[i] * eb) % 16 || (p->v_stride[i] * eb) % 16 ||
        (p->o_stride[i] * ob) % 16)
      return fail(FS_ERR_UNSUPPORTED, "batch/token/head strides must be multiples of 16 bytes");
  }
  if (p->bad_key) {
    cudaError_t e = cudaMemsetAsync(p->bad_key, 0xFF, sizeof(uint64_t), stream);
    if (e != cudaSuccess) return fail(FS_ERR_CUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
  }
  if (p->batch == 0 || p->seqlen_q == 0) return FS_OK;
  if (!p->q || !p->o || (p->seqlen_kv > 0 && (!p->k || !p->v))) return fail(FS_ERR_CONFIG, "null tensor pointer");
  if (p->seqlen_kv == 0) {
    // Empty K/V stream: nothing is loaded, every row has z = 0.  The TMA maps still need a
    // valid global address, so describe K/V over q's storage (never dereferenced).
    fs_fwd_params p2 = *p;
    p2.k = p2.v = p->q;
    for (int i = 0; i < 3; ++i) p2.k_stride[i] = p2.v_stride[i] = p->q_stride[i];
    p2.heads_kv = p->heads_q;
    p2.seqlen_kv = 0;
    return fs_fwd_dispatch(&p2, stream);
  }
  return fs_fwd_dispatch(p, stream);
}

}  // extern "C"
