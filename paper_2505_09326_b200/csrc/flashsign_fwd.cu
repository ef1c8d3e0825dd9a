// flashsign_fwd.cu -- FlashSign (spherical attention) forward for sm_100a.
//
// Replaces the reference hot loop `_streamed_tiles` (pkg/src/ncstream/attention.py:146-200)
// behind `streamed_attention_array` / `multi_head_attention_array`
// (attention.py:252-279, 318-361).  Contract (normalizers.py:94-100):
//     O_i = c * sum_j s_ij v_j / sqrt(c^2 * sum_j s_ij^2 + eps),   s_ij = q_i . k_j
//
// Persistent kernel: one CTA per SM walks work tiles (batch, head, K/V range, 256 query
// rows = NQT=2 query tiles of BM=128) with a static stride.  Roles (768 threads):
//
//   warp 0       TMA producer   Q tiles of the next work tile as soon as their buffer frees,
//                               K_j / V_j into a STAGES-deep ring that runs across work tiles
//   warp 1       MMA issuer     S_t = Q_t K_j^T  (tcgen05 SS, S in TMEM, fp32)
//                               O_t += P_t V_j   (tcgen05 TS: P read from TMEM, V MN-major),
//                               issued once all of P_t is in TMEM; every lane runs the
//                               issue code, the elected lane's predicate makes it the issuer
//   warp 2       TMEM allocator (512 columns: S_0, S_1, O_0, O_1 [, second O set when d=64])
//   warps 4-11   norm, tile 0   warp (column half h, lane quarter) owns 32 rows x BN/2 scores of
//                               S_0: z += a2(s) (packed FFMA2/FADD2, registers), P = cvt(s) ->
//                               TMEM in place (first columns of its own half of S)
//   warps 12-19  norm, tile 1   same for S_1, ping-ponging with tile 0
//   warps 20-23  epilogue WG    O_t -> registers (frees TMEM for the next work tile),
//                               O = acc * c / b(z + eps) -> global, or fp32 partials (split K/V;
//                               peer mode: straight into the owning rank's workspace)
//
// CTAs run in clusters of two on adjacent query blocks of the same (batch, head, K/V range).
// d=128 16-bit (Cfg::P2): the pair is one tcgen05 CTA pair -- the rank-0 CTA issues M=256
// cta_group::2 MMAs over both CTAs' Q tiles; each CTA's ring holds half of every K/V tile (K: its
// 64 keys; V: its 64 columns), its TMA loads complete on the leader's barriers, and the peer's
// norm / epilogue warps arrive on the leader's p_full / o_empty remotely.  Otherwise each CTA
// issues its own MMAs and every K/V tile is TMA-multicast into both CTAs (each loads half).
//
// Normalisers (compile-time NORM): spherical (a2 = s^2, b = sqrt) and signed L1 (a2 = |s|,
// b = id), normalizers.py:94-117.  KS: per-key multiplicities m_j scale the scores in fp32.
//
// Spherical normalisation has no exp and no running max, so O never needs
// rescaling: it stays in TMEM for the whole K/V stream and is scaled exactly
// once by the epilogue warpgroup, which overlaps the next work tile's MMAs.
// Zero padding is exact (a1(0)=a2(0)=0), so ragged N uses TMA out-of-bounds
// zero fill, no masking.
//
// MMA issue order per K/V tile j (keeps each tile's norm warps a full two-MMA window):
//     QK0(j)  PV1(j-1)  QK1(j)  PV0(j)
// tcgen05 MMAs from one thread execute in issue order, so QK_t(j+1) may be
// issued right after PV_t(j) although both touch S_t's columns (P aliases S).

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/flashsign.h"
#include "sm100.cuh"

#ifndef FS_PROF
#define FS_PROF 0  // diagnostic build: clock64 latency counters (fs_prof_read)
#endif

namespace fs {

#if FS_PROF
__device__ unsigned long long g_prof[16];
__device__ unsigned long long g_cta_t[1024][6];  // per CTA: entry, set-up done, work done, exit (globaltimer), smid, work tiles
#define FS_PROF_ADD(i, v) atomicAdd(&g_prof[i], (unsigned long long)(v))
#else
#define FS_PROF_ADD(i, v)
#endif

constexpr int BM = 128;  // query rows per Q tile (= TMEM lanes)
#ifndef FS_BN192
#define FS_BN192 1  // d=64 16-bit: 192-key K/V tiles (1.5x the work per ring / barrier round trip)
#endif
// keys per K/V tile: 192 for d=64 16-bit (S 2 x 192 + O 2 x 64 = 512 TMEM columns), else 128
__host__ __device__ constexpr int bn_for(int in, int d) { return (FS_BN192 && in != FS_E4M3 && d == 64) ? 192 : 128; }
constexpr int BN = 128;  // the default K/V tile (kernels use Cfg::BN)
constexpr int NQT = 2;   // Q tiles per work tile
#ifndef FS_NWT
#define FS_NWT 8  // norm warps per Q tile: 8 (one per lane quarter x column half) or 4
#endif
#ifndef FS_KV1
#define FS_KV1 1  // K_j and V_j share one ring barrier when the ring has >= FS_KV1_MIN slots (Cfg::KV1)
#endif
#ifndef FS_NO_OVF
#define FS_NO_OVF 0  // experiment knob: skip the FP16 / FP8 P-range checks
#endif
#ifndef FS_STAGES32
#define FS_STAGES32 4  // K/V ring depth for 32 KB slots (d=128 16-bit); 5 fits without multiplicities but measured equal
#endif
#ifndef FS_KV1_MIN
#define FS_KV1_MIN 6  // smallest ring (slots) that pairs K_j and V_j on one barrier
#endif
#ifndef FS_TMA_ONCE
#define FS_TMA_ONCE 0  // experiment (wrong results): stream K/V once, then reuse the stale ring
#endif
#ifndef FS_MC
#define FS_MC 1  // CTA pairs (clusters of 2) on adjacent query blocks: K/V tiles multicast, L2 reads halved
#endif
#ifndef FS_STAGES16
#define FS_STAGES16 8  // K/V ring depth for 16 KB slots (d=128 e4m3)
#endif
#ifndef FS_2SM
// CTA pairs run M=256 tcgen05.mma.cta_group::2, each CTA holding half of every K/V tile:
// 0 off, 1 for d=128 16-bit inputs (C3 +2.4 %: half the shared-memory fill and operand reads per
// SM, one issuer per pair), 2 for every configuration (d=64 / e4m3: -1 to -2 % per GHz, measured)
#define FS_2SM 1
#endif
#ifndef FS_PV_TRIM
#define FS_PV_TRIM 1  // skip the PV K-steps past the end of the sequence on a ragged last K/V tile
#endif
#ifndef FS_CARRY
#define FS_CARRY 1  // double-buffered Q: a work tile's last PV_1 is issued after the next tile's first QK_0
#endif
#ifndef FS_P2_NQB2
#define FS_P2_NQB2 0  // CTA pairs at d=128: double-buffer Q (fewer ring slots)
#endif
#ifndef FS_KS_SMEM
#define FS_KS_SMEM 0  // experiment: 16-bit multiplicities scaled in the K slot in shared memory (Cfg::KSM)
#endif
#ifndef FS_EXP_NOZ
#define FS_EXP_NOZ 0  // experiment (wrong results): skip the norm warps' a2(s) accumulation
#endif
#ifndef FS_F16ACC
#define FS_F16ACC 0  // experiment (measured slower): fp16 QK accumulation, S is P (Cfg HA)
#endif
#ifndef FS_ZP
// 16-bit inputs: z = sum a2(p) over the packed P the PV MMA reads, accumulated after P is handed
// over (mixed-precision FHFMA straight from the packed halves, re-read from TMEM), so the norm
// step's critical path is only the conversion; the issuer waits for that re-read (s_free) before
// the next QK overwrites the columns
#define FS_ZP 0  // measured slower: experiment knob
#endif
#ifndef FS_DEFER_Z
#define FS_DEFER_Z 1  // 16-bit inputs: the norm warps' last-chunk a2(s) accumulation after the P hand-off
#endif
#ifndef FS_NORM_DB
// 16-bit inputs: the norm warps read S in 16-column chunks into two register buffers, the next
// chunk's TMEM load in flight while this chunk is converted (instead of 32-column chunks, one buffer)
#define FS_NORM_DB 0  // measured slower: experiment knob
#endif

#ifndef FS_P2_STAGES
#define FS_P2_STAGES 0  // CTA-pair ring depth override (0: as many half-tile slots as fit)
#endif
constexpr int NWT = FS_NWT;
#ifndef FS_CL
#define FS_CL 2  // cluster size when FS_MC (2 or 4)
#endif
constexpr int CL = FS_MC ? FS_CL : 1;  // CTAs per cluster (sharing every K/V tile)
static_assert(NWT == 4 || NWT == 8, "norm warps per Q tile");
constexpr int NUM_THREADS = 32 * (4 + 2 * NWT + 4);
constexpr int TMEM_COLS = 512;
constexpr int WARP_NORM0 = 4;              // norm warps for Q tile t = warps 4+NWT*t ..
constexpr int WARP_EPI = 4 + 2 * NWT;      // epilogue WG = the last four warps

struct KParams {
  void* o;
  int64_t o_sb, o_sn, o_sh;
  int32_t heads_q, heads_kv, seqlen_q, seqlen_kv, head_dim;
  int32_t n_qblk;   // work tiles per (batch, head, K/V range) = ceil(seqlen_q / (NQT*BM*CL))
  int32_t n_tiles;  // n_qblk * heads_q * batch
  float scale, eps;                                // score scale c, denom_epsilon
  float q_descale, k_descale, v_descale, p_scale;  // host values (fs_fwd_params)
  const float* dev_scales;  // non-NULL: {q, k, v descale, p_scale} read on the device instead
  uint64_t* bad_key;
  // split K/V stream (streaming.py:122-128 merge): work tile = (batch, head, split, query block)
  int32_t n_batch;
  int32_t kv_splits;       // >= 1 (uniform mode: every work tile's K/V stream cut into this many ranges)
  int32_t split_tiles;     // K/V tiles per split (the last split may be shorter)
  int32_t n_kv_tiles;      // ceil(seqlen_kv / BN)
  // tail mode (tail_splits > 0, kv_splits == 1): the work tiles [0, n_whole) fill whole waves of the
  // persistent grid and run unsplit; the last partial wave's tail_T tiles are each cut into
  // tail_splits K/V ranges (items n_whole + w * tail_splits + s), so the last wave keeps every
  // cluster busy.  Their partials go to part_num / part_z, rows (s * tail_T + w) * TROWS + local.
  int32_t tail_splits, n_whole, tail_T;
  float* part_num;         // non-NULL: write fp32 partial numerators [S][B][H][Nq][D] here instead of O
  float* part_z;           //           and partial z [S][B][H][Nq] (no normalisation, no bad-row check)
  // context parallelism over peer memory (fs_fwd_peer): partials go straight to the owner of
  // the query position, n / peer_rows, into its workspace slot peer_rank
  float* const* peer;      // device array [peer_world] of the ranks' workspaces (NULL: off)
  int32_t peer_world, peer_rank, peer_rows;
};

// Epilogue constants, derived once per thread from (c, eps, descales, p_scale) in double.
// With g = c * q_descale * k_descale and raw = sum_j a2(q'_i . k'_j) (the kernel's operands):
//   spherical  O = c sum s v / sqrt(c^2 sum s^2 + eps) = sign(g) vd/p * acc / sqrt(raw + eps/g^2)
//   signed L1  O = ...                                = sign(g) vd/p * acc / (raw + eps/|g|)
// -- the row norm is taken in the operands' own units, so neither g^2 nor the original-unit z
// has to fit fp32 (the drop-in path scales its operands by powers of two, attention.py).
struct Fold {
  float eps_f;    // eps / g^2 (spherical) or eps / |g| (signed L1)
  float zrep;     // raw -> the reference's z (g^2 or |g|), reported for bad rows / partials
  float out_sgn;  // sign(g) * v_descale / p_scale: normalised output multiplier
  float out_mul;  // g * v_descale / p_scale: unnormalised numerator (split / partial mode)
  float ps;       // p_scale
  bool zero_g;    // c == 0: every score is 0 (raw forced to 0)
};
template <int NORM>
__device__ __forceinline__ Fold make_fold(const KParams& p) {
  double qd = p.q_descale, kd = p.k_descale, vd = p.v_descale, ps = p.p_scale;
  if (p.dev_scales != nullptr) {
    qd = p.dev_scales[0];
    kd = p.dev_scales[1];
    vd = p.dev_scales[2];
    ps = p.dev_scales[3];
  }
  const double g = static_cast<double>(p.scale) * qd * kd;
  const double ag = fabs(g);
  Fold f;
  f.zero_g = (g == 0.0);
  const double zrep = NORM == FS_NORM_SIGNED_L1 ? ag : g * g;
  f.zrep = static_cast<float>(zrep);
  f.eps_f = f.zero_g ? p.eps : static_cast<float>(fmin(static_cast<double>(p.eps) / zrep, 3.0e38));
  f.out_sgn = f.zero_g ? 0.f : static_cast<float>((g < 0.0 ? -vd : vd) / ps);
  f.out_mul = static_cast<float>(g * vd / ps);
  f.ps = static_cast<float>(ps);
  return f;
}

template <int IN>
struct InTraits;
template <>
struct InTraits<FS_BF16> {
  static constexpr int EB = 2, KSTEP = 16;
  static constexpr uint32_t FMT = 1;
  static constexpr bool F8 = false, SAT_CHECK = false, INF_CHECK = false;
  static constexpr float PMAX = 3.0e38f;
};
template <>
struct InTraits<FS_F16> {
  static constexpr int EB = 2, KSTEP = 16;
  static constexpr uint32_t FMT = 0;
  // P overflow rounds to inf, which makes every element of the row's O non-finite: the
  // epilogue checks O (free) instead of the norm warps checking every score
  static constexpr bool F8 = false, SAT_CHECK = false, INF_CHECK = !FS_NO_OVF;
  static constexpr float PMAX = 65504.0f;
};
template <>
struct InTraits<FS_E4M3> {
  static constexpr int EB = 1, KSTEP = 32;
  static constexpr uint32_t FMT = 0;
  // e4m3 conversion saturates (satfinite) instead of producing inf: the norm warps look for
  // saturated codes (|p| rounded to 448, i.e. |p_scale s| >= 432) in chunks whose sum of a2(s)
  // could reach that range
  static constexpr bool F8 = true, SAT_CHECK = !FS_NO_OVF, INF_CHECK = false;
  static constexpr float PMAX = 432.0f;
};

template <int IN, int D, bool KS = false, bool HA = false>
struct Cfg {
  using TR = InTraits<IN>;
  static constexpr int EB = TR::EB;
  static constexpr int ROW_BYTES = D * EB;
  static_assert(ROW_BYTES % 128 == 0, "head_dim * elem_bytes must be a multiple of 128 B (SW128)");
  static constexpr int NDB = ROW_BYTES / 128;  // 128-byte column blocks per row
  static constexpr int BOXW = 128 / EB;        // elements per TMA box row
  static constexpr int BN = bn_for(IN, D);
  static constexpr int Q_TILE_BYTES = BM * ROW_BYTES;
  // CTA-pair MMA (cta_group::2, M = 256): the pair leader issues every MMA for both CTAs; a CTA's
  // ring slot holds half of a K/V tile -- K: its BN/2 keys, all columns; V: all BN keys, its half
  // of the columns (the MMA's B operand is split along N between the pair).  The multiplicity
  // variant (KS) keeps one MMA per CTA with multicast K/V.
  static constexpr bool P2 = FS_2SM && CL == 2 && !KS && (FS_2SM == 2 || (!TR::F8 && D == 128));
  // Experiment (FS_KS_SMEM=1, 16-bit inputs with multiplicities): K_j' = m_j K_j formed in the K ring
  // slot by the otherwise idle warps 2-3 (packed HMUL2, one rounding -- the numerics of pre-scaling
  // K), once per CTA and K/V tile, instead of m_j s_ij per score in the norm step.  Measured equal at
  // d=64 and -10 % at d=128: the slot's extra read + write (~32 B/clk) pushes the SM past its
  // shared-memory bandwidth, which the SS MMAs already use at 83-128 B/clk.  The torch entry instead
  // forms K' in one HBM pass (fs_scale_keys); FP8 keeps the per-score multiply (its norm step is
  // bound by the e4m3 conversion pipe, where the FMUL2s hide).
  static constexpr bool KSM = KS && !TR::F8 && FS_KS_SMEM;
  static constexpr bool ZP = FS_ZP && !TR::F8;  // z from the packed P (see FS_ZP)
  static constexpr int KROWS = P2 ? BN / 2 : BN;                   // K rows in a CTA's slot
  static constexpr int VROW_BYTES = P2 ? ROW_BYTES / 2 : ROW_BYTES;  // bytes per key in a CTA's V slot
  static constexpr int V_SW = (VROW_BYTES % 128 == 0) ? 128 : 64;  // V slot swizzle span (B)
  static_assert(!P2 || VROW_BYTES == 128 || VROW_BYTES == 64, "pair V slot: 64 or 128 B per key");
  static constexpr int SLOT_BYTES = P2 ? BN * ROW_BYTES / 2 : BN * ROW_BYTES;
  // O accumulators double-buffered in TMEM when they still fit: the epilogue never gates the MMAs.
  static constexpr int NOB_ = (2 * BN + 2 * NQT * D <= TMEM_COLS) ? 2 : 1;
  // 32 KB slots (d=128, 16-bit): one Q buffer per tile, 4 ring slots.  16 KB slots (d=128 e4m3):
  // Q double-buffered (the next work tile's Q lands during this one), 8 ring slots.  24 KB slots
  // (d=64 16-bit, 192 keys): double-buffered Q, 6 ring slots.  CTA pairs: half-size slots, as
  // many as fit (even, <= 16).
  static constexpr int NQB = P2 ? (Q_TILE_BYTES >= 32768 && !FS_P2_NQB2 ? 1 : 2) : (SLOT_BYTES >= 32768) ? 1 : 2;
  static constexpr int P2_STAGES =
      std::min(16, ((232448 - 1024 - 1024 - NQT * NOB_ * 2 * BM * 4 - NQT * NQB * Q_TILE_BYTES) / SLOT_BYTES) & ~1);
  // (32 KB slots: a fifth slot fits when no per-key multiplicity ring is needed and the dynamic
  //  shared-memory base is 1024-aligned -- checked on the device, see SLACK)
  static constexpr int STAGES = P2 ? (FS_P2_STAGES ? std::min(FS_P2_STAGES, P2_STAGES) : P2_STAGES)
                                : (SLOT_BYTES >= 32768) ? (KS ? 4 : FS_STAGES32)
                                : (SLOT_BYTES > 16384 ? 6 : FS_STAGES16);
  static_assert(STAGES <= 16, "ring barriers");
  // K_j and V_j share one ring barrier when the ring is deep (8 slots): one wait per K/V tile on
  // the MMA issuer.  With 4 slots the pair would halve the prefetch distance (measured -10 % at C3).
  static constexpr bool KV1 = FS_KV1 && STAGES >= FS_KV1_MIN;
  __device__ static uint32_t kv_bar(uint32_t slot) { return KV1 ? (slot & ~1u) : slot; }
  static constexpr int RING_OFF = NQT * NQB * Q_TILE_BYTES;
  static constexpr int BAR_OFF = RING_OFF + STAGES * SLOT_BYTES;
  static constexpr int ZBUF_OFF = BAR_OFF + 1024;
  // S buffers in TMEM: one per Q tile (P aliases its S).  (A third rotating buffer at d=64, for
  // a four-MMA norm window, measured slower with a generic issuer; see profiles/r1/SUMMARY.md.)
  static constexpr int NSB = 2;
  static constexpr int NOB = NOB_;
  static_assert(NSB == 2, "NOB_ assumes two S buffers");
  // per-key multiplicities m_j of each V slot's keys (fused K' = m K, grn.py:150)
  static constexpr int MS_OFF = ZBUF_OFF + NQT * NOB * 2 * BM * 4;
  static constexpr int MS_SLOT_BYTES = BN * 4;
  static constexpr int LAYOUT_BYTES = MS_OFF + (KS ? STAGES * MS_SLOT_BYTES : 0);
  // 1024-byte alignment slack for the SW128 buffers when it fits; else the base must be aligned
  static constexpr int SLACK = (LAYOUT_BYTES + 1024 <= 232448) ? 1024 : 0;
  static constexpr int SMEM_BYTES = LAYOUT_BYTES + SLACK;
  static constexpr int QK_STEPS = ROW_BYTES / 32;                          // 32 B of K-dim per MMA
  static constexpr int MMA_M = P2 ? 2 * BM : BM;
  // With the next work tile's Q already resident (NQB = 2), the issue order runs on across the
  // tile boundary: ... QK1(L-1) PV0(L-1) | QK0'(0) PV1(L-1) QK1'(0) PV0'(0) ..., so the last and
  // first norm steps of a tile keep their two-MMA window too.
  static constexpr bool CARRY = FS_CARRY && NQB == 2 && !P2;
  static constexpr int PV_STEPS = BN / TR::KSTEP;
  static constexpr uint32_t COL_S0 = 0;
  static constexpr uint32_t COL_O0 = NSB * BN;
  static_assert(NSB * BN + NOB * NQT * D <= TMEM_COLS, "TMEM budget");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(PV_STEPS % 2 == 0, "P is produced in two column halves");
  // HA (fp16 inputs): QK accumulates in fp16, so S is already P's type; tcgen05 writes a 16-bit D
  // one element per 32-bit column, and tcgen05.ld .pack::16b hands two adjacent ones over packed
  static constexpr uint32_t IDESC_QK =
      ptx::idesc_make(TR::FMT, TR::FMT, 0, 0, MMA_M, BN) & ~(HA ? (3u << 4) : 0u);
  static constexpr uint32_t IDESC_PV = ptx::idesc_make(TR::FMT, TR::FMT, 0, 1, MMA_M, D);
};

struct Bars {
  uint64_t q_full[NQT][2], q_empty[NQT][2];
  uint64_t kv_full[16], kv_empty[16];
  uint64_t ks_full[16];     // Cfg::KSM: the K slot holds m_j K_j (warps 2 and 3 arrived)
  uint64_t s_full[2];       // per S buffer (= Q tile)
  uint64_t p_full[2];       // per S buffer: all norm warps of the tile (both CTAs of a pair) wrote P
  uint64_t s_free[2];       // per S buffer (FS_ZP): the norm warps re-read their P; the next QK may write
  uint64_t o_full[NQT][2], o_empty[NQT][2];
  uint64_t z_full[NQT][2], z_empty[NQT][2];
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 1024, "barrier block");

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
// four e4m3 codes, a in the lowest byte (cvt puts its first source in the upper byte of a pair)
__device__ __forceinline__ uint32_t pack4_e4m3(float a, float b, float c, float d) {
  uint32_t r;
  asm("{\n\t.reg .b16 lo, hi;\n\t"
      "cvt.rn.satfinite.e4m3x2.f32 lo, %2, %1;\n\t"
      "cvt.rn.satfinite.e4m3x2.f32 hi, %4, %3;\n\t"
      "mov.b32 %0, {lo, hi};\n\t}"
      : "=r"(r)
      : "f"(a), "f"(b), "f"(c), "f"(d));
  return r;
}

// z += lo^2 + hi^2 of a packed 16-bit pair, in fp32 (FHFMA: mixed-precision, no unpacking)
template <int IN>
__device__ __forceinline__ float fma_sq_hi_lo(uint32_t w, float z) {
  if constexpr (IN == FS_BF16)
    asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\t"
        "fma.rn.f32.bf16 %0, lo, lo, %0;\n\tfma.rn.f32.bf16 %0, hi, hi, %0;\n\t}"
        : "+f"(z) : "r"(w));
  else
    asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\t"
        "fma.rn.f32.f16 %0, lo, lo, %0;\n\tfma.rn.f32.f16 %0, hi, hi, %0;\n\t}"
        : "+f"(z) : "r"(w));
  return z;
}
// z += |lo| + |hi| (the sign bits already cleared) as lo*1 + hi*1
template <int IN>
__device__ __forceinline__ float fma_abs_hi_lo(uint32_t w, float z) {
  if constexpr (IN == FS_BF16)
    asm("{\n\t.reg .b16 lo, hi, one;\n\tmov.b32 {lo, hi}, %1;\n\tmov.b16 one, 0x3F80;\n\t"
        "fma.rn.f32.bf16 %0, lo, one, %0;\n\tfma.rn.f32.bf16 %0, hi, one, %0;\n\t}"
        : "+f"(z) : "r"(w));
  else
    asm("{\n\t.reg .b16 lo, hi, one;\n\tmov.b32 {lo, hi}, %1;\n\tmov.b16 one, 0x3C00;\n\t"
        "fma.rn.f32.f16 %0, lo, one, %0;\n\tfma.rn.f32.f16 %0, hi, one, %0;\n\t}"
        : "+f"(z) : "r"(w));
  return z;
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

constexpr int TROWS = NQT * BM * CL;  // query rows of one cluster work tile

struct TileCoord {
  int qblk, head, batch, split, kb0, L;  // K/V tiles [kb0, kb0 + L) of this work tile
  bool part;                             // write fp32 partials (numerator, z) instead of O
  int64_t pbase;                         // partial row of query position n = pbase + n
};
__device__ __forceinline__ TileCoord decode_tile(int tile, const KParams& p, int rank) {
  TileCoord c;
  const bool tail = p.tail_splits > 0 && tile >= p.n_whole;
  int u = tile, w = 0, s = 0;  // u: the work tile in the unsplit order (tail mode)
  if (tail) {
    const int x = tile - p.n_whole;
    w = x / p.tail_splits;
    s = x - w * p.tail_splits;
    u = p.n_whole + w;
  }
  const int qc = u % p.n_qblk;
  c.qblk = qc * CL + rank;  // the CTAs of a cluster take adjacent query blocks
  const int rest = u / p.n_qblk;
  c.split = tail ? s : rest % p.kv_splits;
  const int bh = tail ? rest : rest / p.kv_splits;
  c.head = bh % p.heads_q;
  c.batch = bh / p.heads_q;
  const int span = (p.tail_splits > 0 && !tail) ? p.n_kv_tiles : p.split_tiles;
  c.kb0 = c.split * p.split_tiles;
  c.L = min(span, p.n_kv_tiles - c.kb0);
  c.part = tail || (p.tail_splits == 0 && p.part_num != nullptr);
  c.pbase = tail ? (static_cast<int64_t>(s) * p.tail_T + w) * TROWS - static_cast<int64_t>(qc) * TROWS
                 : ((static_cast<int64_t>(c.split) * p.n_batch + c.batch) * p.heads_q + c.head) * p.seqlen_q;
  return c;
}

// NORM: FS_NORM_SPHERICAL (a2 = s^2, b = sqrt) | FS_NORM_SIGNED_L1 (a2 = |s|, b = id), normalizers.py:94-117.
// KS: per-key multiplicity scale m_j fused into the score (s_ij -> m_j s_ij), attention.py:381-388.
// PEER: partials stored into the owning rank's workspace over peer memory (fs_fwd_peer).
template <int IN, int D, int OUT, int NORM, bool KS, bool PEER, bool HA = false>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    flashsign_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_m,
                         const KParams p) {
  using C = Cfg<IN, D, KS, HA>;
  static_assert(!HA || (IN == FS_F16 && !KS), "fp16 accumulation: fp16 inputs, no per-score multiplicities");
  using TR = InTraits<IN>;
  constexpr int BN = C::BN;  // keys per K/V tile for this configuration
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_s = ptx::smem_u32(smem_raw);
  if (C::SLACK == 0 && (raw_s & 1023u) != 0) __trap();  // layout needs an aligned base (see Cfg::SLACK)
  uint8_t* smem = smem_raw + ((1024u - (raw_s & 1023u)) & 1023u);
  const uint32_t smem_s = ptx::smem_u32(smem);
  Bars* bars = reinterpret_cast<Bars*>(smem + C::BAR_OFF);
  float* zbuf = reinterpret_cast<float*>(smem + C::ZBUF_OFF);  // [NQT][NOB][2 halves][BM]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_kv_tiles = (p.seqlen_kv + BN - 1) / BN;
  // clusters of CL CTAs walk the work tiles together (same K/V stream, adjacent query blocks)
  const int rank = CL > 1 ? static_cast<int>(ptx::cluster_ctarank()) : 0;
  const int tile0 = static_cast<int>(blockIdx.x) / CL, tstride = static_cast<int>(gridDim.x) / CL;
#if FS_PROF
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_t[blockIdx.x][0] = ptx::globaltimer();
#endif

  if (threadIdx.x == 32) {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&bars->s_full[b], 1);
      ptx::mbar_init(&bars->p_full[b], C::P2 ? 16 : 8);  // 2 column halves x 4 lane quarters (x 2 CTAs)
      ptx::mbar_init(&bars->s_free[b], C::P2 ? 16 : 8);
    }
#pragma unroll
    for (int t = 0; t < NQT; ++t) {
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        ptx::mbar_init(&bars->q_full[t][b], 1);
        ptx::mbar_init(&bars->q_empty[t][b], 1);
        ptx::mbar_init(&bars->o_full[t][b], 1);
        ptx::mbar_init(&bars->o_empty[t][b], C::P2 ? 8 : 4);
        ptx::mbar_init(&bars->z_full[t][b], NWT);
        ptx::mbar_init(&bars->z_empty[t][b], 4);
      }
    }
    for (int s = 0; s < C::STAGES; ++s) {
      if (C::KSM) ptx::mbar_init(&bars->ks_full[s], 2);
      ptx::mbar_init(&bars->kv_full[s], 1);
      ptx::mbar_init(&bars->kv_empty[s], C::P2 ? 1 : CL);  // both CTAs' MMAs (multicast) / the pair MMA
    }
    ptx::fence_barrier_init();
    ptx::fence_proxy_async();
  }
  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
    if (KS) ptx::tma_prefetch_desc(&tm_m);
  }
  if (warp == 2) {
    if constexpr (C::P2)
      ptx::tmem_alloc2(&bars->tmem_base, TMEM_COLS);
    else
      ptx::tmem_alloc(&bars->tmem_base, TMEM_COLS);
  }
  ptx::tc_fence_before();
  if (CL > 1)
    ptx::cluster_sync();  // the peer's barriers exist before anything is multicast into them
  else
    __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
#if FS_PROF
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_t[blockIdx.x][1] = ptx::globaltimer();
#endif
  // CTA pair: the leader (rank 0) owns the barriers the MMAs wait on (q_full, kv_full, p_full,
  // o_empty); the peer's TMA loads complete on them and its norm / epilogue warps arrive remotely
  auto lead = [&](uint64_t* bar) { return ptx::mapa(ptx::smem_u32(bar), 0u); };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && n_kv_tiles > 0) {
      const uint64_t pol_q = ptx::policy_evict_first();
      const uint64_t pol_kv = ptx::policy_evict_last();
      uint32_t kv_i = 0;  // loads issued into the ring so far (K and V alternate)
      // Q tiles of work tile `tile_` (the it_-th of this CTA) into buffer it_ % NQB once it is free
      auto load_q = [&](int tile_, int it_) {
        const TileCoord qc = decode_tile(tile_, p, rank);
        const int qb = it_ % C::NQB;
        const uint32_t q_use = static_cast<uint32_t>(it_ / C::NQB);
#pragma unroll
        for (int t = 0; t < NQT; ++t) {
          ptx::mbar_wait(&bars->q_empty[t][qb], (q_use & 1u) ^ 1u);
          if (!C::P2 || rank == 0) ptx::mbar_arrive_expect_tx(&bars->q_full[t][qb], (C::P2 ? 2 : 1) * C::Q_TILE_BYTES);
#pragma unroll
          for (int db = 0; db < C::NDB; ++db) {
            uint8_t* dst = smem + (t * C::NQB + qb) * C::Q_TILE_BYTES + db * (BM * 128);
            const int row0 = qc.qblk * (NQT * BM) + t * BM;
            if constexpr (C::P2)
              ptx::tma_load_4d_2sm(dst, &tm_q, lead(&bars->q_full[t][qb]), db * C::BOXW, row0, qc.head, qc.batch,
                                   pol_q);
            else
              ptx::tma_load_4d(dst, &tm_q, &bars->q_full[t][qb], db * C::BOXW, row0, qc.head, qc.batch, pol_q);
          }
        }
      };
      load_q(tile0, 0);
      int it = 0;
      for (int tile = tile0; tile < p.n_tiles; tile += tstride, ++it) {
        const TileCoord tc = decode_tile(tile, p, rank);
        const int head_kv = static_cast<int>((static_cast<int64_t>(tc.head) * p.heads_kv) / p.heads_q);
        const int next = tile + tstride;
        if (C::NQB == 1 && next < p.n_tiles) {
          // single Q buffer: pull the next work tile's Q into L2 now so its reload is an L2 hit
          const TileCoord nx = decode_tile(next, p, rank);
#pragma unroll
          for (int t = 0; t < NQT; ++t)
#pragma unroll
            for (int db = 0; db < C::NDB; ++db)
              ptx::tma_prefetch_l2_4d(&tm_q, db * C::BOXW, nx.qblk * (NQT * BM) + t * BM, nx.head, nx.batch);
        }
        // double-buffered Q: the next work tile's Q goes out right after this tile's first two
        // K/V tiles, a whole work tile ahead of its first QK
        const int L = tc.L;
        const int q_next_at = C::NQB == 2 ? std::min(3, 2 * L - 1) : 2 * L - 1;
        for (int i = 0; i < 2 * L; ++i, ++kv_i) {
          const uint32_t slot = kv_i % C::STAGES;
          const uint32_t round = kv_i / C::STAGES;
          // the tile's key multiplicities ride in the K slot (KSM: scaled into K) or the V slot (FP8:
          // read by the norm warps)
          const bool with_m = KS && (C::KSM ? !(i & 1) : (i & 1));
          uint64_t* full = &bars->kv_full[C::kv_bar(slot)];
          if (FS_TMA_ONCE && !C::P2 && kv_i >= C::STAGES) {  // experiment: no K/V traffic after the first ring
            if (!C::KV1 || !(i & 1)) {
              ptx::mbar_wait(&bars->kv_empty[C::kv_bar(slot)], (round & 1u) ^ 1u);
              ptx::mbar_arrive(full);
            }
            if (i == q_next_at && next < p.n_tiles) load_q(next, it + 1);
            continue;
          }
          if (!C::KV1 || !(i & 1)) {
            ptx::mbar_wait(&bars->kv_empty[C::kv_bar(slot)], (round & 1u) ^ 1u);
            // with KV1 the K load announces both tiles' bytes (V follows right after); a pair's
            // leader announces both CTAs' halves
            if (!C::P2 || rank == 0)
              ptx::mbar_arrive_expect_tx(full, (C::P2 ? 2 : 1) * (C::KV1 ? 2 : 1) * C::SLOT_BYTES +
                                                   (KS ? C::MS_SLOT_BYTES : 0) * (C::KV1 || with_m ? 1 : 0));
          }
          const CUtensorMap* tm = (i & 1) ? &tm_v : &tm_k;
          const int key0 = (tc.kb0 + (i >> 1)) * BN;
          if (with_m)
            ptx::tma_load_2d(smem + C::MS_OFF + slot * C::MS_SLOT_BYTES, &tm_m, full, key0, tc.batch, pol_kv);
          if constexpr (C::P2) {
            uint8_t* dst = smem + C::RING_OFF + slot * C::SLOT_BYTES;
            const uint32_t fl = lead(full);
            if (!(i & 1)) {  // K: this CTA's BN/2 keys, every column block
#pragma unroll
              for (int db = 0; db < C::NDB; ++db)
                ptx::tma_load_4d_2sm(dst + db * (C::KROWS * 128), &tm_k, fl, db * C::BOXW, key0 + rank * C::KROWS,
                                     head_kv, tc.batch, pol_kv);
            } else {  // V: every key of the tile, this CTA's half of the columns
              ptx::tma_load_4d_2sm(dst, &tm_v, fl, rank * (C::VROW_BYTES / C::EB), key0, head_kv, tc.batch, pol_kv);
            }
          } else
#pragma unroll
          for (int db = 0; db < C::NDB; ++db) {
            uint8_t* dst = smem + C::RING_OFF + slot * C::SLOT_BYTES + db * (BN * 128);
            if constexpr (CL > 1)  // this CTA's rows of the tile, into both CTAs of the pair
              ptx::tma_load_4d_mc(dst + rank * (BN / CL) * 128, tm, full, db * C::BOXW, key0 + rank * (BN / CL),
                                  head_kv, tc.batch, static_cast<uint16_t>((1u << CL) - 1u), pol_kv);
            else
              ptx::tma_load_4d(dst, tm, full, db * C::BOXW, key0, head_kv, tc.batch, pol_kv);
          }
          if (i == q_next_at && next < p.n_tiles) load_q(next, it + 1);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the (warp-uniform) control flow and waits; one elected
    // lane issues.  Descriptors are built once; per-step offsets are constants.
    // (CTA pair: the leader issues the M=256 MMAs of both CTAs; the peer's warp 1 idles)
    if (n_kv_tiles > 0 && (!C::P2 || rank == 0)) {
      const bool leader = ptx::elect_one();
      // every lane runs the issue code; the elected lane's predicate makes it the only issuer
      const uint32_t lp = leader ? 1u : 0u;
      constexpr uint16_t ALL = static_cast<uint16_t>((1u << CL) - 1u);
      // a ring slot is free once every CTA of the cluster has consumed it
      auto kv_release = [&](uint64_t* bar) {
        if constexpr (C::P2)
          ptx::tc2_commit_mc_p(bar, ALL, lp);
        else if constexpr (CL > 1)
          ptx::tc_commit_mc_p(bar, ALL, lp);
        else
          ptx::tc_commit_p(bar, lp);
      };
      // MMA-completion signals every CTA waits on (S ready, Q buffer free, O ready)
      auto signal = [&](uint64_t* bar) {
        if constexpr (C::P2)
          ptx::tc2_commit_mc_p(bar, ALL, lp);
        else
          ptx::tc_commit_p(bar, lp);
      };
      const uint64_t q_desc = ptx::sdesc_sw128(smem_s, 16, 1024);
      const uint64_t k_desc = ptx::sdesc_sw128(smem_s + C::RING_OFF, 16, 1024);
      const uint64_t v_desc = C::V_SW == 128 ? ptx::sdesc_sw128(smem_s + C::RING_OFF, BN * 128, 1024)
                                             : ptx::sdesc_sw64(smem_s + C::RING_OFF, BN * 64, 512);
#if FS_PROF
      long long pr_pw = 0, pr_pn = 0, pr_kw = 0, pr_kn = 0;
      const long long pr_t0 = clock64();
#endif
      {
      uint32_t kv_i = 0;                 // ring position of this work tile's K_0
      uint32_t p_use[NQT] = {0u, 0u};    // completed phases of p_full[t]
      uint32_t qk_use[NQT] = {0u, 0u};   // QKs issued into S_t (ZP: each after the previous P's re-read)
      // the previous work tile's last PV_1, carried over the tile boundary (Cfg::CARRY)
      bool pend = false;
      uint32_t pend_slot = 0, pend_o_use = 0;
      int pend_j = 0, pend_ob = 0, pend_kb0 = 0;
      int it = 0;
      for (int tile = tile0; tile < p.n_tiles; tile += tstride, ++it) {
        const int qb = it % C::NQB;
        const uint32_t q_use = static_cast<uint32_t>(it / C::NQB);
        const int ob = it % C::NOB;
        const uint32_t o_use = static_cast<uint32_t>(it / C::NOB);
        const TileCoord tcm = decode_tile(tile, p, rank);
        const int L = tcm.L;
        // S_t = Q_t K^T over the BN keys of the slot
        auto qk = [&](int t, uint32_t slot) {
          constexpr uint32_t idesc = C::IDESC_QK;
          if constexpr (C::ZP) {
            if (qk_use[t] > 0) {
              if constexpr (C::P2)
                ptx::mbar_wait_cluster(&bars->s_free[t], (qk_use[t] - 1) & 1u);
              else
                ptx::mbar_wait(&bars->s_free[t], (qk_use[t] - 1) & 1u);
              ptx::tc_fence_after();
            }
            ++qk_use[t];
          }
          const uint64_t a0 = q_desc + static_cast<uint32_t>(((t * C::NQB + qb) * C::Q_TILE_BYTES) >> 4);
          const uint64_t b0 = k_desc + static_cast<uint32_t>((slot * C::SLOT_BYTES) >> 4);
          const uint32_t d_tmem = tmem + C::COL_S0 + t * BN;
#pragma unroll
          for (int ks = 0; ks < C::QK_STEPS; ++ks) {
            const uint32_t off_a = ((ks * 32 / 128) * (BM * 128) + (ks * 32) % 128) >> 4;
            const uint32_t off_b = ((ks * 32 / 128) * (C::KROWS * 128) + (ks * 32) % 128) >> 4;
            if constexpr (C::P2 && TR::F8)
              ptx::mma2_f8_ss_p(d_tmem, a0 + off_a, b0 + off_b, idesc, ks > 0, lp);
            else if constexpr (C::P2)
              ptx::mma2_f16_ss_p(d_tmem, a0 + off_a, b0 + off_b, idesc, ks > 0, lp);
            else if constexpr (TR::F8)
              ptx::mma_f8_ss_p(d_tmem, a0 + off_a, b0 + off_b, idesc, ks > 0, lp);
            else
              ptx::mma_f16_ss_p(d_tmem, a0 + off_a, b0 + off_b, idesc, ks > 0, lp);
          }
        };
        // O_t += P_t V_j once all of P_t is in TMEM (one hand-off per tile: every extra
        // barrier round trip on the issuing warp costs more than it overlaps, measured)
        // (ob_, o_use_, kb0_: the work tile the PV belongs to -- the previous one for a carried PV_1)
        auto pv = [&](int t, uint32_t slot, int j, int ob_, uint32_t o_use_, int kb0_) {
          if (j == 0) {
            if constexpr (C::P2)
              ptx::mbar_wait_cluster(&bars->o_empty[t][ob_], (o_use_ & 1u) ^ 1u);
            else
              ptx::mbar_wait(&bars->o_empty[t][ob_], (o_use_ & 1u) ^ 1u);
          }
          const uint64_t b0 = v_desc + static_cast<uint32_t>((slot * C::SLOT_BYTES) >> 4);
          const uint32_t a_tmem = tmem + C::COL_S0 + t * BN;
          const uint32_t d_tmem = tmem + C::COL_O0 + (ob_ * NQT + t) * D;
          auto wait_p = [&]() {
#if FS_PROF
            const long long tw0 = clock64();
#endif
            if constexpr (C::P2)
              ptx::mbar_wait_cluster(&bars->p_full[t], p_use[t] & 1u);
            else
              ptx::mbar_wait(&bars->p_full[t], p_use[t] & 1u);
#if FS_PROF
            pr_pw += clock64() - tw0;
            ++pr_pn;
#endif
            ptx::tc_fence_after();
          };
          wait_p();
          auto issue = [&](int ks, uint32_t pred) {
            const int h = ks / (C::PV_STEPS / 2), k2 = ks % (C::PV_STEPS / 2);
            // (V rows are 128 B per column block; a pair's V slot has VROW_BYTES per key)
            const uint32_t off_b = (ks * TR::KSTEP * (C::P2 ? C::VROW_BYTES : 128)) >> 4;
            // P of column half h is packed into the first columns of S_t's half h
            const uint32_t at = a_tmem + h * (BN / 2) + k2 * (TR::KSTEP * C::EB / 4);
            const uint32_t acc = (j > 0 || ks > 0) ? 1u : 0u;
            if constexpr (C::P2 && TR::F8)
              ptx::mma2_f8_ts_p(d_tmem, at, b0 + off_b, C::IDESC_PV, acc, pred);
            else if constexpr (C::P2)
              ptx::mma2_f16_ts_p(d_tmem, at, b0 + off_b, C::IDESC_PV, acc, pred);
            else if constexpr (TR::F8)
              ptx::mma_f8_ts_p(d_tmem, at, b0 + off_b, C::IDESC_PV, acc, pred);
            else
              ptx::mma_f16_ts_p(d_tmem, at, b0 + off_b, C::IDESC_PV, acc, pred);
          };
          // keys of this K/V tile inside the sequence: on a ragged last tile the K-steps past them
          // would multiply P = 0 (zero-filled K rows) with zero-filled V rows -- not issued
          const int keys_left = p.seqlen_kv - (kb0_ + j) * BN;
          if (FS_PV_TRIM && keys_left < BN) {
            const int n_steps = (keys_left + TR::KSTEP - 1) / TR::KSTEP;
#pragma unroll 1
            for (int ks = 0; ks < n_steps; ++ks) issue(ks, lp);
          } else {
#pragma unroll
            for (int ks = 0; ks < C::PV_STEPS; ++ks) issue(ks, lp);
          }
          ++p_use[t];
        };
#pragma unroll
        for (int t = 0; t < NQT; ++t) ptx::mbar_wait(&bars->q_full[t][qb], q_use & 1u);
        ptx::tc_fence_after();
        uint32_t prev_v_slot = 0;
        for (int j = 0; j < L; ++j) {
          const uint32_t k_idx = kv_i + 2 * j, v_idx = k_idx + 1;
          const uint32_t k_slot = k_idx % C::STAGES, v_slot = v_idx % C::STAGES;
#if FS_PROF
          const long long tk0 = clock64();
#endif
          ptx::mbar_wait(&bars->kv_full[C::kv_bar(k_slot)], (k_idx / C::STAGES) & 1u);
          if constexpr (C::KSM) ptx::mbar_wait(&bars->ks_full[k_slot], (k_idx / C::STAGES) & 1u);
#if FS_PROF
          pr_kw += clock64() - tk0;
          ++pr_kn;
#endif
          ptx::tc_fence_after();
          auto qk_signal = [&](int t) {
            qk(t, k_slot);
            signal(&bars->s_full[t]);
          };
          qk_signal(0);
          if (j == L - 1) signal(&bars->q_empty[0][qb]);
          if (j > 0) {
            pv(1, prev_v_slot, j - 1, ob, o_use, tcm.kb0);
            kv_release(&bars->kv_empty[C::kv_bar(prev_v_slot)]);
          } else if (C::CARRY && pend) {
            pv(1, pend_slot, pend_j, pend_ob, pend_o_use, pend_kb0);
            kv_release(&bars->kv_empty[C::kv_bar(pend_slot)]);
            signal(&bars->o_full[1][pend_ob]);
            pend = false;
          }
          qk_signal(1);
          if (!C::KV1) kv_release(&bars->kv_empty[k_slot]);  // KV1: freed with V after PV1
          if (j == L - 1) signal(&bars->q_empty[1][qb]);
          if (!C::KV1) ptx::mbar_wait(&bars->kv_full[v_slot], (v_idx / C::STAGES) & 1u);
          pv(0, v_slot, j, ob, o_use, tcm.kb0);
          if (j == L - 1) signal(&bars->o_full[0][ob]);
          prev_v_slot = v_slot;
        }
        if (C::CARRY && tile + tstride < p.n_tiles) {
          pend = true;
          pend_slot = prev_v_slot;
          pend_j = L - 1;
          pend_ob = ob;
          pend_o_use = o_use;
          pend_kb0 = tcm.kb0;
        } else {
          pv(1, prev_v_slot, L - 1, ob, o_use, tcm.kb0);
          kv_release(&bars->kv_empty[C::kv_bar(prev_v_slot)]);
          signal(&bars->o_full[1][ob]);
        }
        kv_i += 2 * L;
      }
      }
#if FS_PROF
      if (leader) { FS_PROF_ADD(2, pr_pw); FS_PROF_ADD(3, pr_pn); FS_PROF_ADD(4, pr_kw); FS_PROF_ADD(5, pr_kn);
                    FS_PROF_ADD(7, clock64() - pr_t0); }
#endif
    }
  } else if (C::KSM && (warp == 2 || warp == 3)) {
    // ------------------------------------------------------------ K scaling (Cfg::KSM)
    // K_j' = m_j K_j in the K ring slot, in place: a 16-byte chunk holds 8 elements of one key row
    // (the 128B swizzle permutes chunks within a row), so chunk x scales by m of row
    // (x mod BN*8) / 8.  Integer (any 16-bit-representable) m: packed HMUL2, one rounding, exactly
    // what pre-scaling K in float64 and casting gives; other m: fp32 multiply, then RNE.
    using E2 = typename std::conditional<IN == FS_BF16, __nv_bfloat162, __half2>::type;
    uint32_t kv_i = 0;
    for (int tile = tile0; tile < p.n_tiles && n_kv_tiles > 0; tile += tstride) {
      const int L = decode_tile(tile, p, rank).L;
      for (int j = 0; j < L; ++j, kv_i += 2) {
        const uint32_t slot = kv_i % C::STAGES;
        ptx::mbar_wait(&bars->kv_full[C::kv_bar(slot)], (kv_i / C::STAGES) & 1u);
        const float* ms = reinterpret_cast<const float*>(smem + C::MS_OFF + slot * C::MS_SLOT_BYTES);
        uint4* base = reinterpret_cast<uint4*>(smem + C::RING_OFF + slot * C::SLOT_BYTES);
        // 8 chunks per thread in flight: loads first, then the multiplies, then the stores (one
        // chunk at a time would serialise on the shared-memory latency)
        constexpr int CPT = C::SLOT_BYTES / 16 / 64, NBT = 8;
        static_assert(!C::KSM || CPT % NBT == 0, "K slot chunks per scaler thread");
#pragma unroll 1
        for (int b0 = 0; b0 < CPT; b0 += NBT) {
          uint4 w[NBT];
          float m[NBT];
          bool exact = true;
#pragma unroll
          for (int u = 0; u < NBT; ++u) {
            const int x = (b0 + u) * 64 + (warp - 2) * 32 + lane;
            w[u] = base[x];
            m[u] = ms[(x % (BN * 8)) / 8];
          }
#pragma unroll
          for (int u = 0; u < NBT; ++u) {
            E2 m2;
            if constexpr (IN == FS_BF16) m2 = __float2bfloat162_rn(m[u]);
            else m2 = __float2half2_rn(m[u]);
            exact = exact && (__low2float(m2) == m[u]);
          }
          if (__all_sync(0xffffffffu, exact)) {
#pragma unroll
            for (int u = 0; u < NBT; ++u) {
              E2 m2;
              if constexpr (IN == FS_BF16) m2 = __float2bfloat162_rn(m[u]);
              else m2 = __float2half2_rn(m[u]);
              E2* e = reinterpret_cast<E2*>(&w[u]);
#pragma unroll
              for (int k = 0; k < 4; ++k) e[k] = __hmul2(e[k], m2);
            }
          } else {  // fp32 product then RNE (bitwise the same as HMUL2 when m is representable)
#pragma unroll
            for (int u = 0; u < NBT; ++u) {
              E2* e = reinterpret_cast<E2*>(&w[u]);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                float2 f2;
                if constexpr (IN == FS_BF16) f2 = __bfloat1622float2(e[k]);
                else f2 = __half22float2(e[k]);
                reinterpret_cast<uint32_t*>(&w[u])[k] = pack2<IN>(f2.x * m[u], f2.y * m[u]);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < NBT; ++u) base[(b0 + u) * 64 + (warp - 2) * 32 + lane] = w[u];
        }
        ptx::fence_proxy_async();  // generic-proxy stores -> visible to the tensor core's reads
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&bars->ks_full[slot]);
      }
    }
  } else if (warp >= WARP_NORM0 && warp < WARP_EPI) {
    // ------------------------------------------------------------ norm warps
    // Eight warps per Q tile: warp (t, h, quarter) owns TMEM lanes 32*quarter.. and the
    // score columns [64h, 64h+64) of S_t, so both halves of P are produced in parallel.
    // P half h is packed into the first columns of its own S half (never over unread S).
    // (With NWT=4 a warp owns all 128 columns and produces the two halves in turn.)
    const int t = (warp - WARP_NORM0) / NWT;                             // Q tile
    const int hh0 = NWT == 8 ? ((warp - WARP_NORM0) >> 2) & 1 : 0;      // first column half
    constexpr int NH = NWT == 8 ? 1 : 2;                                 // halves per warp
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int r = quarter * 32 + lane;
    const uint32_t s_lane = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + C::COL_S0;
    const float ps = p.dev_scales != nullptr ? p.dev_scales[3] : p.p_scale;
    // a half whose sum of a2(s) stays below this cannot hold an out-of-range P: (PMAX/|p_scale|)^{2|1}
    const float ovf_z = NORM == FS_NORM_SIGNED_L1 ? TR::PMAX / fabsf(ps) : (TR::PMAX / fabsf(ps)) * (TR::PMAX / fabsf(ps));
    // ZP: z over P = p_scale * s is in P units; back to the operands' units (raw)
    const float inv_pz = NORM == FS_NORM_SIGNED_L1 ? 1.f / ps : 1.f / (ps * ps);
    uint32_t s_use = 0;
#if FS_PROF
    long long pr_sw = 0, pr_nc = 0, pr_nn = 0;
#endif
    int it = 0;
    for (int tile = tile0; tile < p.n_tiles && n_kv_tiles > 0; tile += tstride, ++it) {
      const int ob = it % C::NOB;
      float2 za = make_float2(0.f, 0.f), zb = za;
      bool ovf = false;
      const int L = decode_tile(tile, p, rank).L;
      for (int j = 0; j < L; ++j) {
#if FS_PROF
        const long long tn0 = clock64();
#endif
        const uint32_t sb = t;  // S_t's TMEM buffer; one phase per K/V tile
        ptx::mbar_wait(&bars->s_full[sb], s_use & 1u);
        const uint32_t s_base = s_lane + sb * BN;
        // key multiplicities of this K/V tile ride in V_j's ring slot; that slot is released only
        // after PV_1(j), which needs this warp's P, so they stay valid while they are read here
        const uint32_t v_idx = 2u * s_use + 1u, v_slot = v_idx % C::STAGES;
        if constexpr (KS && !C::KSM) ptx::mbar_wait(&bars->kv_full[C::kv_bar(v_slot)], (v_idx / C::STAGES) & 1u);
        ++s_use;
#if FS_PROF
        const long long tn1 = clock64();
        pr_sw += tn1 - tn0;
#endif
        ptx::tc_fence_after();
#pragma unroll
        for (int hi = 0; hi < NH; ++hi) {
        const int hh = hh0 + hi;
        const uint32_t s_addr = s_base + hh * (BN / 2);
        if constexpr (HA) {
          // fp16 S straight from the MMA: packed pairs by the TMEM load path (no conversion),
          // stored as P over the half's first columns once every chunk is in registers; z from
          // the same packed values after P is handed over (FHFMA), off the critical path
          constexpr int NCH = BN / 64;
          uint32_t pk[NCH][16];
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) ptx::tmem_ld16_pack(s_addr + 32 * ch, pk[ch]);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) ptx::tmem_st16(s_addr + 16 * ch, pk[ch]);
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (C::P2 && rank != 0)
              ptx::mbar_arrive_cluster(lead(&bars->p_full[sb]));
            else
              ptx::mbar_arrive(&bars->p_full[sb]);
          }
          float zc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if constexpr (NORM == FS_NORM_SIGNED_L1)
                zc[i & 3] = fma_abs_hi_lo<IN>(pk[ch][i] & 0x7FFF7FFFu, zc[i & 3]);
              else
                zc[i & 3] = fma_sq_hi_lo<IN>(pk[ch][i], zc[i & 3]);
            }
          za.x += zc[0] + zc[1];
          za.y += zc[2] + zc[3];
#if FS_PROF
          pr_nc += clock64() - tn1;
          ++pr_nn;
#endif
          continue;
        }
        // BN/2 columns in 32-column chunks (80 registers/thread at 768 threads): the next chunk's
        // TMEM load is issued once this chunk is packed, and overlaps this chunk's P store.
        // FS_NORM_DB (16-bit): 16-column chunks, two buffers, the next load issued before this
        // chunk's conversion so that it overlaps the ALU work.
        // (Two 32-column buffers do not fit: with setmaxnreg moving the producer / MMA warpgroup to
        // 24-32 and the epilogue to 40-64 registers, the norm warps get at most 96 and ptxas needs
        // more -- 768 threads share 80 x 768 registers.)
        constexpr bool DB = FS_NORM_DB && !TR::F8;
        constexpr int CW = DB ? 16 : 32;  // columns per chunk
        constexpr int NCH = (BN / 2) / CW;
        // 16-bit P, 192-key tiles: accumulate the last 32 columns' a2(s) after the P hand-off (FP8: the e4m3 conversion
        // runs on its own pipe and hides the FFMA2s; its saturation check needs the sums first)
        constexpr bool DEFER_Z = FS_DEFER_Z && !TR::F8 && BN / 2 >= 96 && !C::ZP;
        constexpr int NDEF = DEFER_Z ? 32 / CW : 0;  // deferred chunks (the last ones, still in registers)
        uint32_t sbuf[DB ? 2 : 1][CW];
        auto ld_chunk = [&](uint32_t addr, uint32_t* dst) {
          if constexpr (CW == 16)
            ptx::tmem_ld16(addr, dst);
          else
            ptx::tmem_ld32(addr, dst);
        };
        ld_chunk(s_addr, sbuf[0]);
        ptx::tmem_wait_ld();
        // FP8: every chunk's packed codes and the half's sum of a2(s), for one saturation check per
        // half after its last store (off the chunk-to-chunk path)
        uint32_t pk8[TR::SAT_CHECK ? NCH * 8 : 1];
        // sum of a2(s) over this half: packed FP32 FMAs / adds, two independent chains
        float2 h0 = make_float2(0.f, 0.f), h1 = h0;
        auto accum_a2 = [&](float2 a, float2 b) {
          if constexpr (FS_EXP_NOZ) return;  // experiment (wrong z): what the a2(s) sums cost
          if constexpr (NORM == FS_NORM_SIGNED_L1) {
            h0 = __fadd2_rn(h0, make_float2(fabsf(a.x), fabsf(a.y)));
            h1 = __fadd2_rn(h1, make_float2(fabsf(b.x), fabsf(b.y)));
          } else {
            h0 = __ffma2_rn(a, a, h0);
            h1 = __ffma2_rn(b, b, h1);
          }
        };
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          uint32_t* s = sbuf[DB ? (ch & 1) : 0];
          if constexpr (DB) {
            if (ch + 1 < NCH) ld_chunk(s_addr + CW * (ch + 1), sbuf[(ch + 1) & 1]);  // the other buffer
          }
          // (a2(s) accumulates into the half's h0 / h1 chains)  With KS the scores are
          // first scaled by the key multiplicities, s_ij <- m_j s_ij (fp32; exact for integer m).
          const float4* mp = reinterpret_cast<const float4*>(smem + C::MS_OFF + v_slot * C::MS_SLOT_BYTES) +
                             (hh * (BN / 2) + ch * CW) / 4;
#pragma unroll
          for (int i = 0; i < CW; i += 4) {
            float2 a = make_float2(__uint_as_float(s[i + 0]), __uint_as_float(s[i + 1]));
            float2 b = make_float2(__uint_as_float(s[i + 2]), __uint_as_float(s[i + 3]));
            if constexpr (KS && !C::KSM) {
              const float4 m4 = mp[i / 4];
              a = __fmul2_rn(a, make_float2(m4.x, m4.y));
              b = __fmul2_rn(b, make_float2(m4.z, m4.w));
              s[i + 0] = __float_as_uint(a.x);
              s[i + 1] = __float_as_uint(a.y);
              s[i + 2] = __float_as_uint(b.x);
              s[i + 3] = __float_as_uint(b.y);
            }
            if (!C::ZP && !(DEFER_Z && ch >= NCH - NDEF)) accum_a2(a, b);
          }
          // pack P (s[i] is written only after s[2i], s[2i+1] / s[4i..4i+3] are read)
          uint32_t pk_local[CW / 2];
          uint32_t* pk = TR::SAT_CHECK ? pk8 + (TR::SAT_CHECK ? ch * 8 : 0) : pk_local;
          if constexpr (TR::F8) {
            if (ps == 1.0f) {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                pk[i] = pack4_e4m3(__uint_as_float(s[4 * i]), __uint_as_float(s[4 * i + 1]),
                                   __uint_as_float(s[4 * i + 2]), __uint_as_float(s[4 * i + 3]));
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                pk[i] = pack4_e4m3(ps * __uint_as_float(s[4 * i]), ps * __uint_as_float(s[4 * i + 1]),
                                   ps * __uint_as_float(s[4 * i + 2]), ps * __uint_as_float(s[4 * i + 3]));
            }
          } else if (ps == 1.0f) {
#pragma unroll
            for (int i = 0; i < CW / 2; ++i) pk[i] = pack2<IN>(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1]));
          } else {
#pragma unroll
            for (int i = 0; i < CW / 2; ++i)
              pk[i] = pack2<IN>(ps * __uint_as_float(s[2 * i]), ps * __uint_as_float(s[2 * i + 1]));
          }
          if constexpr (!DB) {
            if (ch + 1 < NCH) ptx::tmem_ld32(s_addr + 32 * (ch + 1), s);  // next chunk (s is consumed)
          }
          if constexpr (TR::F8 || CW == 16)
            ptx::tmem_st8(s_addr + ch * 8, pk);
          else
            ptx::tmem_st16(s_addr + ch * 16, pk);
          if (ch + 1 < NCH) {
            if constexpr (CW == 16)
              ptx::tmem_wait_ld16(sbuf[(ch + 1) & 1]);
            else
              ptx::tmem_wait_ld();
          }
        }
        if constexpr (!DEFER_Z && !C::ZP) {
          za = __fadd2_rn(za, h0);
          zb = __fadd2_rn(zb, h1);
        }
        if constexpr (TR::SAT_CHECK) {
          // max|s| <= sqrt(sum s^2) (<= sum |s|): only a half whose sum reaches ovf_z can hold a
          // saturated code; then look for 0x7e / 0xfe (+-448) in its packed P
          if ((h0.x + h0.y) + (h1.x + h1.y) >= ovf_z) {
            uint32_t sat = 0;
#pragma unroll
            for (int i = 0; i < NCH * 8; ++i) {
              const uint32_t tt = (pk8[i] & 0x7f7f7f7fu) ^ 0x7e7e7e7eu;  // zero byte <=> saturated
              sat |= (tt - 0x01010101u) & ~tt & 0x80808080u;
            }
            if (sat) ovf = true;
          }
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (C::P2 && rank != 0)
            ptx::mbar_arrive_cluster(lead(&bars->p_full[sb]));  // the pair leader issues PV
          else
            ptx::mbar_arrive(&bars->p_full[sb]);
        }
        if constexpr (C::ZP) {
          // z from the packed P this warp just handed to the MMA (the values the PV products use):
          // re-read its BN/4 columns, release S_t for the next QK, then a2(p) in fp32 with
          // mixed-precision FMAs straight from the 16-bit halves (two pairs of chains)
          constexpr int PC = BN / 4;  // 32-bit P columns of this warp's half
          uint32_t pw[PC];
          ptx::tmem_ld32(s_addr, pw);
          if constexpr (PC > 32) ptx::tmem_ld16(s_addr + 32, pw + 32);
          ptx::tmem_wait_ld();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (C::P2 && rank != 0)
              ptx::mbar_arrive_cluster(lead(&bars->s_free[sb]));
            else
              ptx::mbar_arrive(&bars->s_free[sb]);
          }
          float zc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int i = 0; i < PC; ++i) {
            if constexpr (NORM == FS_NORM_SIGNED_L1)
              zc[i & 3] = fma_abs_hi_lo<IN>(pw[i] & 0x7FFF7FFFu, zc[i & 3]);
            else
              zc[i & 3] = fma_sq_hi_lo<IN>(pw[i], zc[i & 3]);
          }
          za.x += (zc[0] + zc[1]) * inv_pz;
          za.y += (zc[2] + zc[3]) * inv_pz;
        }
        if constexpr (DEFER_Z) {
          // the last 32 columns' a2(s) after P is handed over: off the P critical path (16-bit P:
          // the FFMA2s share the conversion's pipe); the buffers still hold those chunks
#pragma unroll
          for (int c = NCH - NDEF; c < NCH; ++c) {
            const uint32_t* s = sbuf[DB ? (c & 1) : 0];
#pragma unroll
            for (int i = 0; i < CW; i += 4)
              accum_a2(make_float2(__uint_as_float(s[i + 0]), __uint_as_float(s[i + 1])),
                       make_float2(__uint_as_float(s[i + 2]), __uint_as_float(s[i + 3])));
          }
          za = __fadd2_rn(za, h0);
          zb = __fadd2_rn(zb, h1);
        }
#if FS_PROF
        pr_nc += clock64() - tn1;
        ++pr_nn;
#endif
        }
      }
      // hand this half's z to the epilogue warpgroup and move on to the next work tile
      const float z = (za.x + za.y) + (zb.x + zb.y) + (FS_EXP_NOZ ? 1.f : 0.f);
      ptx::mbar_wait(&bars->z_empty[t][ob], (static_cast<uint32_t>(it / C::NOB) & 1u) ^ 1u);
      zbuf[((t * C::NOB + ob) * 2 + hh0) * BM + r] = ovf ? __int_as_float(0x7f800000) : z;
      if (NWT == 4) zbuf[((t * C::NOB + ob) * 2 + 1) * BM + r] = 0.f;
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&bars->z_full[t][ob]);
    }
#if FS_PROF
    if (lane == 0) { FS_PROF_ADD(0, pr_nc); FS_PROF_ADD(1, pr_nn); FS_PROF_ADD(6, pr_sw); }
#endif
  } else if (warp >= WARP_EPI) {
    // ------------------------------------------------------------ epilogue warpgroup
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    using OT = typename OutT<OUT>::T;
    const Fold fd = make_fold<NORM>(p);
    // FP16 P overflow needs some |p s| >= 65520, hence raw z >= (65504 / p)^2 (or 65504 / p for L1)
    // (device scales come from fs_prepare, whose p_scale bounds |p s| below 2^15 for every score:
    //  no overflow is possible and the check is off)
    const float ovf_raw = p.dev_scales != nullptr ? __int_as_float(0x7f800000)
                          : NORM == FS_NORM_SIGNED_L1 ? TR::PMAX / fd.ps
                                                      : (TR::PMAX / fd.ps) * (TR::PMAX / fd.ps);
    int it = 0;
    for (int tile = tile0; tile < p.n_tiles; tile += tstride, ++it) {
      const TileCoord tc = decode_tile(tile, p, rank);
      const int ob = it % C::NOB;
      const uint32_t o_use = static_cast<uint32_t>(it / C::NOB);
#pragma unroll 1
      for (int t = 0; t < NQT; ++t) {
        // raw = sum_j a2(q'_i . k'_j) in the operands' units (+inf for a saturated FP8 P);
        // the reference's z is raw * zrep
        float raw = 0.f;
        if (tc.L > 0) {
          ptx::mbar_wait(&bars->z_full[t][ob], o_use & 1u);
          const float* zt = zbuf + (t * C::NOB + ob) * 2 * BM + r;
          raw = fd.zero_g ? 0.f : zt[0] + zt[BM];  // the two column halves of the row
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&bars->z_empty[t][ob]);
        }
        const int row = tc.qblk * (NQT * BM) + t * BM + r;
        const bool live = row < p.seqlen_q;
        const bool partial = PEER || tc.part;
        const float zr = raw * fd.zrep;  // z in the reference's units (bad-row report, partials)
        const float den = NORM == FS_NORM_SIGNED_L1 ? raw + fd.eps_f : sqrtf(raw + fd.eps_f);
        // partial mode: the unnormalised numerator (the combine step divides by b(sum z + eps))
        float mul = partial ? fd.out_mul : __fdiv_rn(fd.out_sgn, den);
        // partial row index: ((split * B + batch) * H + head) * Nq + row (tail mode: see KParams)
        const int64_t prow = tc.pbase + row;
        // where this row's partial goes: the local workspace, or (peer mode) slot peer_rank of the
        // owner's workspace -- numerators [world][B][H][Rn][D] then z [world][B][H][Rn]
        float* num_dst = p.part_num + prow * D;
        float* z_dst = p.part_z + prow;
        if (PEER && live) {
          const int owner = row / p.peer_rows;
          const int64_t rows_slot = static_cast<int64_t>(p.n_batch) * p.heads_q * p.peer_rows;
          const int64_t loc = p.peer_rank * rows_slot +
                              (static_cast<int64_t>(tc.batch) * p.heads_q + tc.head) * p.peer_rows +
                              (row - owner * p.peer_rows);
          float* base = p.peer[owner];
          num_dst = base + loc * D;
          z_dst = base + static_cast<int64_t>(p.peer_world) * rows_slot * D + loc;
        }
        // row status once O's first columns are in: FP16 P overflow (inf) makes every O element
        // non-finite, so one column tells -- but only a row whose raw z reaches the overflow range
        // can have overflowed (a NaN / inf in V alone leaves z below it and is passed through, as
        // the reference does); it is reported as z = +inf like a saturated FP8 P
        auto finish_row = [&](bool ovf_o) {
          const float z_report = ovf_o ? __int_as_float(0x7f800000) : zr;
          const bool bad = !partial && (ovf_o || !(den > 0.f) || isinf(den));
          if (partial && live) *z_dst = z_report;
          if (live && bad && p.bad_key != nullptr) {
            const uint64_t lin = (static_cast<uint64_t>(tc.batch) * p.heads_q + tc.head) * p.seqlen_q + row;
            atomicMin(reinterpret_cast<unsigned long long*>(p.bad_key),
                      static_cast<unsigned long long>((lin << 32) | __float_as_uint(z_report)));
          }
          if (ovf_o) mul = 0.f;  // flagged row: zeros rather than inf/NaN
        };
        OT* dst = reinterpret_cast<OT*>(p.o) + tc.batch * p.o_sb + static_cast<int64_t>(row) * p.o_sn +
                  tc.head * p.o_sh;
        const uint32_t o_addr = tmem + lane_off + C::COL_O0 + (ob * NQT + t) * D;
        if (tc.L > 0) {
          ptx::mbar_wait(&bars->o_full[t][ob], o_use & 1u);
          ptx::tc_fence_after();
        }
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          if (c == 0) {
            // FP16 P overflow: an inf P_ij makes EVERY column of O_i non-finite (inf * v, or
            // inf * 0 = NaN) and needs raw z >= (65504/p)^2.  Only rows past that z bound are
            // scanned, before the first accumulator chunk is loaded (so no register set is live
            // besides the scan's): no finite column = overflow.  A NaN / inf in V alone (some
            // columns) is passed through unflagged, as the reference does.
            bool ovf_row = false;
            if constexpr (TR::INF_CHECK) {
              const bool cand = tc.L > 0 && isfinite(raw) && raw >= ovf_raw;
              if (__any_sync(0xffffffffu, cand)) {  // warp-uniform: tcgen05.ld is warp-collective
                bool fin = false;
#pragma unroll 1
                for (int c2 = 0; c2 < D / 32; ++c2) {
                  uint32_t w[32];
                  ptx::tmem_ld32(o_addr + c2 * 32, w);
                  ptx::tmem_wait_ld();
#pragma unroll
                  for (int i = 0; i < 32; ++i)
                    if (c2 * 32 + i < p.head_dim && isfinite(__uint_as_float(w[i]))) fin = true;
                }
                ovf_row = cand && !fin;
              }
            }
            finish_row(ovf_row);
          }
          uint32_t acc[32];
          float v[32];
          if (tc.L > 0) {
            ptx::tmem_ld32(o_addr + c * 32, acc);  // warp-collective: every lane participates
            ptx::tmem_wait_ld();
            if (c == D / 32 - 1) {  // all of O_t is in registers: release the accumulator
              ptx::tc_fence_before();
              __syncwarp();
              if (lane == 0) {
                if (C::P2 && rank != 0)
                  ptx::mbar_arrive_cluster(lead(&bars->o_empty[t][ob]));
                else
                  ptx::mbar_arrive(&bars->o_empty[t][ob]);
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = 0u;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = (mul == 0.f) ? 0.f : __uint_as_float(acc[i]) * mul;
          if (partial) {
            if (live) store32<FS_F32>(num_dst + c * 32, v, c * 32, D);
          } else if (live && c * 32 < p.head_dim) {
            store32<OUT>(dst + c * 32, v, c * 32, p.head_dim);
          }
        }
      }
    }
  }

  // peer mode: the partials went to other GPUs' memory; make them visible system-wide before exit
  if (PEER && warp >= WARP_EPI) __threadfence_system();
#if FS_PROF
  if (warp == WARP_EPI && lane == 0 && blockIdx.x < 1024) {
    g_cta_t[blockIdx.x][2] = ptx::globaltimer();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_cta_t[blockIdx.x][4] = smid;
    g_cta_t[blockIdx.x][5] = tile0 < p.n_tiles ? (p.n_tiles - 1 - tile0) / tstride + 1 : 0;
  }
#endif
  ptx::tc_fence_before();
  if constexpr (C::P2) {
    ptx::cluster_sync();  // both CTAs are done with the pair's TMEM and with each other's barriers
    if (warp == 2) {
      ptx::tc_fence_after();
      ptx::tmem_dealloc2(tmem, TMEM_COLS);
    }
  } else {
    __syncthreads();
    if (warp == 2) {
      ptx::tc_fence_after();
      ptx::tmem_dealloc(tmem, TMEM_COLS);
    }
  }
  if (CL > 1) ptx::cluster_sync();  // no CTA leaves while its peer may still signal it
#if FS_PROF
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_t[blockIdx.x][3] = ptx::globaltimer();
#endif
}

// ====================================================================== host

static thread_local std::string g_last_error;
// set by fs_fwd_peer around its fs_fwd call: route the partials to the owners' workspaces
static thread_local const fs_peer_params* g_peer = nullptr;

static fs_status fail(fs_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

void set_last_error(const char* msg) { g_last_error = msg; }

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

constexpr int kMaxDevices = 64;

// Encoded TMA descriptors, cached per thread: repeated calls on the same buffers (a layer loop,
// a benchmark, a GRN forward) skip cuTensorMapEncodeTiled.  Key = everything the encode reads.
struct TmaKey {
  const void* ptr;
  int64_t dims[4], strides[3];
  int32_t box_w, box_rows, dt, swizzle, dev;
  bool operator==(const TmaKey& o) const { return std::memcmp(this, &o, sizeof(TmaKey)) == 0; }
};
struct TmaCache {
  static constexpr int N = 32;
  TmaKey key[N];
  CUtensorMap map[N];
  uint64_t stamp[N] = {0};
  uint64_t clock = 0;
  const CUtensorMap* find(const TmaKey& k) {
    for (int i = 0; i < N; ++i)
      if (stamp[i] != 0 && key[i] == k) {
        stamp[i] = ++clock;
        return &map[i];
      }
    return nullptr;
  }
  void put(const TmaKey& k, const CUtensorMap& m) {
    int v = 0;
    for (int i = 1; i < N; ++i)
      if (stamp[i] < stamp[v]) v = i;
    key[v] = k;
    map[v] = m;
    stamp[v] = ++clock;
  }
};
static thread_local TmaCache g_tma_cache;

static bool encode_bshd_uncached(CUtensorMap* map, CUtensorMapDataType dt, int eb, const void* ptr, int head_dim,
                                 int seqlen, int heads, int batch, const int64_t* stride, int box_w, int box_rows,
                                 std::string* err, int swizzle);

static bool encode_bshd(CUtensorMap* map, CUtensorMapDataType dt, int eb, const void* ptr, int head_dim, int seqlen,
                        int heads, int batch, const int64_t* stride, int box_w, int box_rows, std::string* err,
                        int swizzle = 128) {
  TmaKey k;
  std::memset(&k, 0, sizeof(k));  // padding bytes take part in the comparison
  k.ptr = ptr;
  k.dims[0] = head_dim;
  k.dims[1] = seqlen;
  k.dims[2] = heads;
  k.dims[3] = batch;
  k.strides[0] = stride[0] * eb;
  k.strides[1] = stride[1] * eb;
  k.strides[2] = stride[2] * eb;
  k.box_w = box_w;
  k.box_rows = box_rows;
  k.dt = static_cast<int32_t>(dt);
  k.swizzle = swizzle;
  cudaGetDevice(&k.dev);
  if (const CUtensorMap* hit = g_tma_cache.find(k)) {
    *map = *hit;
    return true;
  }
  if (!encode_bshd_uncached(map, dt, eb, ptr, head_dim, seqlen, heads, batch, stride, box_w, box_rows, err, swizzle))
    return false;
  g_tma_cache.put(k, *map);
  return true;
}

static bool encode_bshd_uncached(CUtensorMap* map, CUtensorMapDataType dt, int eb, const void* ptr, int head_dim,
                                 int seqlen, int heads, int batch, const int64_t* stride, int box_w, int box_rows,
                                 std::string* err, int swizzle) {
  auto enc = get_encode_fn();
  if (!enc) {
    *err = "cuTensorMapEncodeTiled unavailable (driver too old?)";
    return false;
  }
  cuuint64_t dims[4] = {(cuuint64_t)head_dim, (cuuint64_t)(seqlen > 0 ? seqlen : 1), (cuuint64_t)heads,
                        (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)(stride[1] * eb), (cuuint64_t)(stride[2] * eb),
                           (cuuint64_t)(stride[0] * eb)};
  cuuint32_t box[4] = {(cuuint32_t)box_w, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, dt, 4, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r);
    return false;
  }
  return true;
}

// for flashsign_gram.cu: the same (cached) BSHD tensor-map encoding
bool encode_bshd_shared(CUtensorMap* map, int in_dtype, const void* ptr, int head_dim, int seqlen, int heads,
                        int batch, const int64_t* stride, int box_w, int box_rows, std::string* err) {
  const CUtensorMapDataType dt = in_dtype == FS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                 : in_dtype == FS_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                      : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  return encode_bshd(map, dt, in_dtype == FS_E4M3 ? 1 : 2, ptr, head_dim, seqlen, heads, batch, stride, box_w,
                     box_rows, err);
}

static int kernel_d(const fs_fwd_params* p) { return (p->in_dtype == FS_E4M3 || p->head_dim > 64) ? 128 : 64; }
static int kernel_bn(const fs_fwd_params* p) { return bn_for(p->in_dtype, kernel_d(p)); }

// Key multiplicities m [batch, seqlen_kv] fp32 (token stride 1): 128-key boxes, zero-filled past
// seqlen_kv so padded keys stay exactly zero.
static bool encode_key_scale(CUtensorMap* map, const fs_fwd_params* p, std::string* err) {
  auto enc = get_encode_fn();
  if (!enc) {
    *err = "cuTensorMapEncodeTiled unavailable (driver too old?)";
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)(p->seqlen_kv > 0 ? p->seqlen_kv : 1), (cuuint64_t)p->batch};
  const int64_t sb = p->batch > 1 ? p->key_scale_stride : ((p->seqlen_kv + 3) / 4) * 4;
  cuuint64_t strides[1] = {(cuuint64_t)(sb * 4)};
  cuuint32_t box[2] = {(cuuint32_t)kernel_bn(p), 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(p->key_scale), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled (key_scale) failed with CUresult " + std::to_string((int)r);
    return false;
  }
  return true;
}

// SM count of the current device (persistent grid size), cached per device.
static int num_sms() {
  static std::atomic<int> cache[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (dev < 0 || dev >= kMaxDevices) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }
  if (cache[dev].load(std::memory_order_relaxed) == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) cache[dev].store(n);
  }
  return cache[dev].load(std::memory_order_relaxed);
}

// Co-resident clusters of the persistent grid on the current device.  Every instantiation runs
// one 768-thread CTA per SM with > 113 KB of dynamic shared memory in clusters of CL, so one
// representative kernel answers for all (a GPC with an odd SM count holds one pair fewer).
static int resident_clusters() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return std::max(1, num_sms() / CL);
  static std::atomic<int> cache[kMaxDevices];
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n > 0) return n;
  n = std::max(1, num_sms() / CL);
  if constexpr (CL > 1) {
    using C = Cfg<FS_BF16, 128, false>;
    auto kern = flashsign_fwd_kernel<FS_BF16, 128, FS_BF16, FS_NORM_SPHERICAL, false, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(n * CL);
      cfg.blockDim = dim3(NUM_THREADS);
      cfg.dynamicSmemBytes = C::SMEM_BYTES;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = CL;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int m = 0;
      if (cudaOccupancyMaxActiveClusters(&m, kern, &cfg) == cudaSuccess && m > 0) n = std::min(n, m);
    }
    cudaGetLastError();  // a failed query leaves no sticky error
  }
  cache[dev].store(n);
  return n;
}

// K/V split plan.  Work tiles are (batch, head, 512-row query block) per cluster, walked by the G
// co-resident clusters with a static stride.  Uniform mode cuts every work tile's K/V stream into
// `splits` ranges (small B*H, long N); tail mode cuts only the tiles of the last, partial wave
// (tiles = W*G + T, 0 < T < G), so that wave has T*splits items instead of T (e.g. 8-GPU shards
// of C2 / C4: 256 tiles on 74 clusters = 3.46 waves -> 3 + 68/74).  Requested splits are clamped
// to [1, K/V tiles] with every range non-empty.
struct SplitPlan {
  int32_t splits, split_tiles, n_kv_tiles;
  int32_t tail, n_whole, tail_T, clusters;
  int64_t n_qblk, n_tiles0, n_items, part_rows;
};
constexpr int kPlanOverhead = 2;  // per-item prologue + epilogue, in K/V-tile steps (wave model)

// Wave-model choice of (splits, tail) for FS_SPLITS_AUTO.  Cost unit: one K/V-tile step of one
// cluster work tile; each item pays kPlanOverhead; a split pays the combine pass (its partial
// rows of Dk+1 fp32 read at ~5 TB/s, plus ~4 us of launch) converted into steps.
static void auto_plan(const fs_fwd_params* p, const SplitPlan& sp, int G, int* s_out, bool* tail_out) {
  *s_out = 1;
  *tail_out = false;
  const int64_t L = sp.n_kv_tiles, tiles = sp.n_tiles0;
  if (tiles == 0 || L < 8) return;
  const int dk = kernel_d(p);
  const double step_s = 4.0 * (NQT * BM) * kernel_bn(p) * dk / 10.8e12;  // one CTA of the pair
  const double rows = static_cast<double>(p->batch) * p->heads_q * p->seqlen_q;
  auto comb = [&](double prow) { return (prow * (dk + 1) * 4.0 / 5.0e12 + 4.0e-6) / step_s; };
  // costs of s = 1..smax; the smallest s within 0.5 % of the minimum wins (fewer Q reloads and
  // partial rows than the model charges for)
  const int64_t smax = std::min<int64_t>(16, L / 4);
  double cost_of[17];
  bool tail_of[17] = {};
  std::fill(cost_of, cost_of + 17, 1e300);
  cost_of[1] = static_cast<double>((tiles + G - 1) / G) * (L + kPlanOverhead);
  tail_of[1] = false;
  double best = cost_of[1];
  const int64_t W = tiles / G, T = tiles % G;
  for (int64_t s = 2; s <= smax; ++s) {
    const int64_t st = (L + s - 1) / s, se = (L + st - 1) / st;
    double cost;
    bool tail;
    if (tiles < G) {
      cost = static_cast<double>((tiles * se + G - 1) / G) * (st + kPlanOverhead) + comb(se * rows);
      tail = false;
    } else {
      if (T == 0) break;
      cost = static_cast<double>(W) * (L + kPlanOverhead) +
             static_cast<double>((T * se + G - 1) / G) * (st + kPlanOverhead) + comb(static_cast<double>(se * T * TROWS));
      tail = true;
    }
    cost_of[s] = cost;
    tail_of[s] = tail;
    best = std::min(best, cost);
  }
  for (int64_t s = 1; s <= std::max<int64_t>(1, smax); ++s)
    if (cost_of[s] <= best * 1.005) {
      *s_out = static_cast<int>(s);
      *tail_out = tail_of[s];
      return;
    }
}

// clusters: the co-resident cluster count to plan for (<= 0: query the current device)
static SplitPlan split_plan(const fs_fwd_params* p, int clusters = 0) {
  SplitPlan sp{};
  const int bn = kernel_bn(p);
  sp.n_kv_tiles = (p->seqlen_kv + bn - 1) / bn;
  sp.n_qblk = (static_cast<int64_t>(p->seqlen_q) + TROWS - 1) / TROWS;
  sp.n_tiles0 = sp.n_qblk * p->heads_q * p->batch;
  // context parallelism wants every row's partial: uniform mode only
  const bool every_row = p->partial_only || g_peer != nullptr;
  int s = p->kv_splits;
  bool tail = p->split_tail != 0 && !every_row;
  auto G = [&]() {
    if (clusters <= 0) clusters = resident_clusters();
    return clusters;
  };
  if (s == FS_SPLITS_AUTO) {
    s = 1;
    tail = false;
    if (!every_row) auto_plan(p, sp, G(), &s, &tail);
  }
  s = std::max(1, std::min(std::max(1, s), sp.n_kv_tiles));
  sp.split_tiles = sp.n_kv_tiles > 0 ? (sp.n_kv_tiles + s - 1) / s : 0;
  sp.splits = sp.split_tiles > 0 ? (sp.n_kv_tiles + sp.split_tiles - 1) / sp.split_tiles : 1;
  sp.clusters = clusters;
  const int64_t rows = static_cast<int64_t>(p->batch) * p->heads_q * p->seqlen_q;
  if (tail && sp.splits > 1) {
    const int64_t g = G();
    sp.clusters = clusters;
    const int64_t T = sp.n_tiles0 % g;
    if (T == 0) {  // whole waves: nothing to balance
      sp.splits = 1;
      sp.split_tiles = sp.n_kv_tiles;
    } else {
      sp.tail = 1;
      sp.n_whole = static_cast<int32_t>(sp.n_tiles0 - T);
      sp.tail_T = static_cast<int32_t>(T);
    }
  }
  if (sp.tail) {
    sp.n_items = sp.n_whole + static_cast<int64_t>(sp.tail_T) * sp.splits;
    sp.part_rows = static_cast<int64_t>(sp.splits) * sp.tail_T * TROWS;
  } else {
    sp.n_items = sp.n_tiles0 * sp.splits;
    sp.part_rows = sp.splits * rows;
  }
  return sp;
}

// Merge of K/V-range partials (streaming.py:122-128, Lemma 1: (o, z) add, no
// rescale): O = sum_s num_s / b(sum_s z_s + eps), plus the bad-row key.  One thread per 4 columns.
// `rows` partial rows per part.  Uniform splits: partial row = (b*H + h)*Nq + n.  Tail splits
// (TAIL): partial row = w*TROWS + local for tail work tile w, i.e. work tile u = n_whole + w of the
// unsplit order, query position n = (u % n_qblk)*TROWS + local of (b, h) = u / n_qblk.
template <int OUT, int NORM, int DK, bool TAIL>
__global__ void __launch_bounds__(256) flashsign_combine_kernel(const float* __restrict__ num,
                                                                const float* __restrict__ zp, int n_parts,
                                                                int64_t rows, int heads, int seqlen_q, void* o,
                                                                int64_t o_sb, int64_t o_sn, int64_t o_sh,
                                                                int head_dim, float eps, uint64_t* bad_key,
                                                                int n_whole, int n_qblk) {
  constexpr int TPR = DK / 4;
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t row = gid / TPR;
  const int c4 = static_cast<int>(gid % TPR) * 4;
  if (row >= rows) return;
  int n;
  int64_t bh;
  if constexpr (TAIL) {
    const int64_t u = n_whole + row / TROWS;
    n = static_cast<int>((u % n_qblk) * TROWS + row % TROWS);
    bh = u / n_qblk;
    if (n >= seqlen_q) return;  // past the sequence end: never written by the forward kernel
  } else {
    n = static_cast<int>(row % seqlen_q);
    bh = row / seqlen_q;
  }
  float z = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = 0; s < n_parts; ++s) {
    z += zp[s * rows + row];
    const float4 a = *reinterpret_cast<const float4*>(num + (s * rows + row) * DK + c4);
    acc.x += a.x;
    acc.y += a.y;
    acc.z += a.z;
    acc.w += a.w;
  }
  const float den = NORM == FS_NORM_SIGNED_L1 ? z + eps : sqrtf(z + eps);
  if ((!(den > 0.f) || isinf(den)) && c4 == 0 && bad_key != nullptr) {
    const uint64_t lin = static_cast<uint64_t>(bh) * seqlen_q + n;
    atomicMin(reinterpret_cast<unsigned long long*>(bad_key),
              static_cast<unsigned long long>((lin << 32) | __float_as_uint(z)));
  }
  if (c4 >= head_dim) return;
  const float inv = __fdiv_rn(1.0f, den);
  const int h = static_cast<int>(bh % heads);
  const int64_t b = bh / heads;
  using OT = typename OutT<OUT>::T;
  OT* dst = reinterpret_cast<OT*>(o) + b * o_sb + static_cast<int64_t>(n) * o_sn + h * o_sh + c4;
  const float v0 = acc.x * inv, v1 = acc.y * inv, v2 = acc.z * inv, v3 = acc.w * inv;
  if constexpr (OUT == FS_F32) {
    *reinterpret_cast<float4*>(dst) = make_float4(v0, v1, v2, v3);
  } else {
    uint2 w;
    w.x = pack2<OUT>(v0, v1);
    w.y = pack2<OUT>(v2, v3);
    *reinterpret_cast<uint2*>(dst) = w;
  }
}

// rows / n_whole / n_qblk: see flashsign_combine_kernel (tail = 0: uniform splits, every row)
template <int DK>
static fs_status combine(const fs_fwd_params* p, int n_parts, cudaStream_t stream, int64_t tail_rows = 0,
                         int n_whole = 0, int n_qblk = 1) {
  const bool tail = tail_rows > 0;
  const int64_t rows = tail ? tail_rows : (int64_t)p->batch * p->heads_q * p->seqlen_q;
  if (rows == 0) return FS_OK;
  const float* num = p->partial;
  const float* zp = p->partial + (int64_t)n_parts * rows * DK;
  const int64_t threads = rows * (DK / 4);
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  auto go = [&](auto kern) {
    kern<<<blocks, 256, 0, stream>>>(num, zp, n_parts, rows, p->heads_q, p->seqlen_q, p->o, p->o_stride[0],
                                     p->o_stride[1], p->o_stride[2], p->head_dim, p->eps, p->bad_key, n_whole,
                                     n_qblk);
  };
  const bool l1 = p->normalizer == FS_NORM_SIGNED_L1;
#define FS_COMBINE_GO(OUT)                                                                           \
  (tail ? (l1 ? go(flashsign_combine_kernel<OUT, FS_NORM_SIGNED_L1, DK, true>)                        \
              : go(flashsign_combine_kernel<OUT, FS_NORM_SPHERICAL, DK, true>))                       \
        : (l1 ? go(flashsign_combine_kernel<OUT, FS_NORM_SIGNED_L1, DK, false>)                       \
              : go(flashsign_combine_kernel<OUT, FS_NORM_SPHERICAL, DK, false>)))
  switch (p->out_dtype) {
    case FS_F32:
      FS_COMBINE_GO(FS_F32);
      break;
    case FS_BF16:
      FS_COMBINE_GO(FS_BF16);
      break;
    case FS_F16:
      FS_COMBINE_GO(FS_F16);
      break;
    default:
      return fail(FS_ERR_DTYPE, "out_dtype must be FS_F32, FS_BF16 or FS_F16");
  }
#undef FS_COMBINE_GO
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FS_ERR_CUDA, std::string("combine launch: ") + cudaGetErrorString(e));
  return FS_OK;
}

// Peer-mode merge (context parallelism over peer memory): this rank owns query positions
// [n0, n0 + nr) of every (b, h); its workspace holds the world ranks' partials of them,
// numerators [world][B][H][Rn][DK] then z [world][B][H][Rn].  O = sum num / b(sum z + eps)
// into O[b, n, h, :], plus the bad-row key (linear row (b*H + h)*Nq + n).  One thread per 4 columns.
template <int OUT, int NORM, int DK>
__global__ void __launch_bounds__(256) flashsign_combine_peer_kernel(const float* __restrict__ ws, int world,
                                                                     int batch, int heads, int seqlen_q, int rn,
                                                                     int n0, int nr, void* o, int64_t o_sb,
                                                                     int64_t o_sn, int64_t o_sh, int head_dim,
                                                                     float eps, uint64_t* bad_key) {
  constexpr int TPR = DK / 4;
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t r = gid / TPR;  // (b*H + h)*nr + i
  const int c4 = static_cast<int>(gid % TPR) * 4;
  if (r >= static_cast<int64_t>(batch) * heads * nr) return;
  const int i = static_cast<int>(r % nr);
  const int64_t bh = r / nr;
  const int64_t slot_rows = static_cast<int64_t>(batch) * heads * rn;
  const int64_t loc = bh * rn + i;
  float z = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = 0; s < world; ++s) {
    z += ws[static_cast<int64_t>(world) * slot_rows * DK + s * slot_rows + loc];
    const float4 a = *reinterpret_cast<const float4*>(ws + (s * slot_rows + loc) * DK + c4);
    acc.x += a.x;
    acc.y += a.y;
    acc.z += a.z;
    acc.w += a.w;
  }
  const int n = n0 + i;
  const float den = NORM == FS_NORM_SIGNED_L1 ? z + eps : sqrtf(z + eps);
  if ((!(den > 0.f) || isinf(den)) && c4 == 0 && bad_key != nullptr) {
    const uint64_t lin = static_cast<uint64_t>(bh) * seqlen_q + n;
    atomicMin(reinterpret_cast<unsigned long long*>(bad_key),
              static_cast<unsigned long long>((lin << 32) | __float_as_uint(z)));
  }
  if (c4 >= head_dim) return;
  const float inv = __fdiv_rn(1.0f, den);
  const int h = static_cast<int>(bh % heads);
  const int64_t b = bh / heads;
  using OT = typename OutT<OUT>::T;
  OT* dst = reinterpret_cast<OT*>(o) + b * o_sb + static_cast<int64_t>(n) * o_sn + h * o_sh + c4;
  const float v0 = acc.x * inv, v1 = acc.y * inv, v2 = acc.z * inv, v3 = acc.w * inv;
  if constexpr (OUT == FS_F32) {
    *reinterpret_cast<float4*>(dst) = make_float4(v0, v1, v2, v3);
  } else {
    uint2 w;
    w.x = pack2<OUT>(v0, v1);
    w.y = pack2<OUT>(v2, v3);
    *reinterpret_cast<uint2*>(dst) = w;
  }
}

template <int DK>
static fs_status combine_peer(const fs_fwd_params* p, const fs_peer_params* pp, cudaStream_t stream) {
  const int n0 = pp->rank * pp->rows_per_rank;
  const int nr = std::max(0, std::min(pp->rows_per_rank, p->seqlen_q - n0));
  const int64_t rows = (int64_t)p->batch * p->heads_q * nr;
  if (rows == 0) return FS_OK;
  const int64_t threads = rows * (DK / 4);
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  auto go = [&](auto kern) {
    kern<<<blocks, 256, 0, stream>>>(pp->local_partial, pp->world, p->batch, p->heads_q, p->seqlen_q,
                                     pp->rows_per_rank, n0, nr, p->o, p->o_stride[0], p->o_stride[1],
                                     p->o_stride[2], p->head_dim, p->eps, p->bad_key);
  };
  const bool l1 = p->normalizer == FS_NORM_SIGNED_L1;
  switch (p->out_dtype) {
    case FS_F32:
      l1 ? go(flashsign_combine_peer_kernel<FS_F32, FS_NORM_SIGNED_L1, DK>)
         : go(flashsign_combine_peer_kernel<FS_F32, FS_NORM_SPHERICAL, DK>);
      break;
    case FS_BF16:
      l1 ? go(flashsign_combine_peer_kernel<FS_BF16, FS_NORM_SIGNED_L1, DK>)
         : go(flashsign_combine_peer_kernel<FS_BF16, FS_NORM_SPHERICAL, DK>);
      break;
    case FS_F16:
      l1 ? go(flashsign_combine_peer_kernel<FS_F16, FS_NORM_SIGNED_L1, DK>)
         : go(flashsign_combine_peer_kernel<FS_F16, FS_NORM_SPHERICAL, DK>);
      break;
    default:
      return fail(FS_ERR_DTYPE, "out_dtype must be FS_F32, FS_BF16 or FS_F16");
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FS_ERR_CUDA, std::string("combine_peer launch: ") + cudaGetErrorString(e));
  return FS_OK;
}

template <int IN, int D, int OUT, int NORM, bool KS, bool PEER = false, bool HA = false>
static fs_status launch(const fs_fwd_params* p, cudaStream_t stream) {
  using C = Cfg<IN, D, KS, HA>;
  auto kern = flashsign_fwd_kernel<IN, D, OUT, NORM, KS, PEER, HA>;
  // the >48 KB dynamic shared-memory opt-in is per device (context): set it once per device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    return fail(FS_ERR_CUDA, "cudaGetDevice failed or device index out of range");
  static std::atomic<bool> attr_set[kMaxDevices];
  if (!attr_set[dev].load(std::memory_order_acquire)) {
    cudaError_t attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (attr_err != cudaSuccess)
      return fail(FS_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
    attr_set[dev].store(true, std::memory_order_release);
  }

  const CUtensorMapDataType dt = (IN == FS_BF16)  ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                 : (IN == FS_F16) ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                  : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  CUtensorMap tq, tk, tv;
  std::string err;
  if (!encode_bshd(&tq, dt, C::EB, p->q, p->head_dim, p->seqlen_q, p->heads_q, p->batch, p->q_stride, C::BOXW, BM,
                   &err) ||
      !encode_bshd(&tk, dt, C::EB, p->k, p->head_dim, p->seqlen_kv, p->heads_kv, p->batch, p->k_stride, C::BOXW,
                   C::BN / CL, &err) ||
      // V: multicast halves of the key rows, or (CTA pair) this CTA's half of the columns, all keys
      !encode_bshd(&tv, dt, C::EB, p->v, p->head_dim, p->seqlen_kv, p->heads_kv, p->batch, p->v_stride,
                   C::P2 ? C::VROW_BYTES / C::EB : C::BOXW, C::P2 ? C::BN : C::BN / CL, &err, C::V_SW))
    return fail(FS_ERR_UNSUPPORTED, err);
  CUtensorMap tm = tq;  // unused unless KS
  if (KS && !encode_key_scale(&tm, p, &err)) return fail(FS_ERR_UNSUPPORTED, err);

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
  kp.scale = p->scale;
  kp.eps = p->eps;
  kp.q_descale = p->q_descale;
  kp.k_descale = p->k_descale;
  kp.v_descale = p->v_descale;
  kp.p_scale = p->p_scale;
  kp.dev_scales = p->dev_scales;
  kp.bad_key = p->bad_key;
  const SplitPlan sp = split_plan(p);
  const int64_t n_tiles = sp.n_items;
  if (n_tiles > INT32_MAX) return fail(FS_ERR_UNSUPPORTED, "too many work tiles for one launch");
  kp.n_qblk = (int32_t)sp.n_qblk;
  kp.n_tiles = (int32_t)n_tiles;
  kp.n_batch = p->batch;
  kp.kv_splits = sp.tail ? 1 : sp.splits;
  kp.split_tiles = sp.split_tiles;
  kp.n_kv_tiles = sp.n_kv_tiles;
  kp.tail_splits = sp.tail ? sp.splits : 0;
  kp.n_whole = sp.n_whole;
  kp.tail_T = sp.tail_T;
  const bool partial = sp.splits > 1 || p->partial_only;
  kp.part_num = partial ? p->partial : nullptr;
  kp.part_z = partial ? p->partial + sp.part_rows * D : nullptr;
  kp.peer = nullptr;
  kp.peer_world = kp.peer_rank = kp.peer_rows = 0;
  if (g_peer != nullptr) {
    kp.part_num = kp.part_z = nullptr;
    kp.peer = g_peer->peer_partial;
    kp.peer_world = g_peer->world;
    kp.peer_rank = g_peer->rank;
    kp.peer_rows = g_peer->rows_per_rank;
  }
  int grid = (int)std::min<int64_t>(n_tiles * CL, (num_sms() / CL) * CL);
  if (grid <= 0) return fail(FS_ERR_CUDA, "no SMs reported for the current device");
  cudaError_t e;
  if constexpr (CL > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = C::SMEM_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // persistent grid: never more clusters than can be co-resident (a GPC with an odd SM count
    // holds one pair fewer), or the surplus clusters would run as a second wave
    static std::atomic<int> max_clusters[kMaxDevices];
    if (max_clusters[dev].load(std::memory_order_relaxed) == 0) {
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) max_clusters[dev].store(n);
    }
    const int mc = max_clusters[dev].load(std::memory_order_relaxed);
    if (mc > 0) grid = std::min(grid, mc * CL);
    cfg.gridDim = dim3(grid);
    e = cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, tm, kp);
  } else {
    kern<<<grid, NUM_THREADS, C::SMEM_BYTES, stream>>>(tq, tk, tv, tm, kp);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  if (sp.splits > 1 && !p->partial_only)
    return sp.tail ? combine<D>(p, sp.splits, stream, static_cast<int64_t>(sp.tail_T) * TROWS, sp.n_whole,
                                static_cast<int>(sp.n_qblk))
                   : combine<D>(p, sp.splits, stream);
  return FS_OK;
}

template <int IN, int D, int NORM, bool KS>
static fs_status dispatch_out(const fs_fwd_params* p, cudaStream_t s) {
  // fp16 inputs at p_scale 1 (no device scales, no per-score multiplicities): fp16 QK accumulation
  // (Cfg HA; `FS_F16ACC`), S is P without a conversion pass
  constexpr bool HA_OK = FS_F16ACC && IN == FS_F16 && !KS;
  if constexpr (HA_OK) {
    if (p->p_scale == 1.0f && p->dev_scales == nullptr) {
      switch (p->out_dtype) {
        case FS_F32:
          return launch<IN, D, FS_F32, NORM, KS, false, true>(p, s);
        case FS_BF16:
          return launch<IN, D, FS_BF16, NORM, KS, false, true>(p, s);
        case FS_F16:
          return launch<IN, D, FS_F16, NORM, KS, false, true>(p, s);
        default:
          return fail(FS_ERR_DTYPE, "out_dtype must be FS_F32, FS_BF16 or FS_F16");
      }
    }
  }
  switch (p->out_dtype) {
    case FS_F32:
      return launch<IN, D, FS_F32, NORM, KS>(p, s);
    case FS_BF16:
      return launch<IN, D, FS_BF16, NORM, KS>(p, s);
    case FS_F16:
      return launch<IN, D, FS_F16, NORM, KS>(p, s);
    default:
      return fail(FS_ERR_DTYPE, "out_dtype must be FS_F32, FS_BF16 or FS_F16");
  }
}

template <int IN, int D>
static fs_status dispatch_norm(const fs_fwd_params* p, cudaStream_t s) {
  const bool ks = p->key_scale != nullptr;
  if (g_peer != nullptr) {  // peer mode: partials only (no O, so one output type), no multiplicities
    if (ks) return fail(FS_ERR_UNSUPPORTED, "fs_fwd_peer: key_scale is not supported");
    return p->normalizer == FS_NORM_SIGNED_L1 ? launch<IN, D, FS_F32, FS_NORM_SIGNED_L1, false, true>(p, s)
                                              : launch<IN, D, FS_F32, FS_NORM_SPHERICAL, false, true>(p, s);
  }
  if (p->normalizer == FS_NORM_SIGNED_L1)
    return ks ? dispatch_out<IN, D, FS_NORM_SIGNED_L1, true>(p, s) : dispatch_out<IN, D, FS_NORM_SIGNED_L1, false>(p, s);
  return ks ? dispatch_out<IN, D, FS_NORM_SPHERICAL, true>(p, s) : dispatch_out<IN, D, FS_NORM_SPHERICAL, false>(p, s);
}

}  // namespace fs

static fs_status fs_fwd_dispatch(const fs_fwd_params* p, cudaStream_t stream) {
  using namespace fs;

  if (p->in_dtype == FS_E4M3) {
    // 1-byte rows: the SW128 layout needs 128-byte rows -> D = 128 (TMA zero-fills d >= head_dim).
    return dispatch_norm<FS_E4M3, 128>(p, stream);
  }
  const bool d64 = p->head_dim <= 64;
  if (p->in_dtype == FS_BF16) return d64 ? dispatch_norm<FS_BF16, 64>(p, stream) : dispatch_norm<FS_BF16, 128>(p, stream);
  return d64 ? dispatch_norm<FS_F16, 64>(p, stream) : dispatch_norm<FS_F16, 128>(p, stream);
}


extern "C" {

#if FS_PROF
// diagnostic builds only: read and reset the latency counters
int fs_prof_read(unsigned long long* out8) {
  if (cudaMemcpyFromSymbol(out8, fs::g_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
  unsigned long long z[16] = {0};
  return cudaMemcpyToSymbol(fs::g_prof, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
// per-CTA timeline of the last launch: [1024][6] (entry, set-up done, work done, exit: globaltimer
// ns; SM id; work tiles)
int fs_prof_timeline(unsigned long long* out6144) {
  return cudaMemcpyFromSymbol(out6144, fs::g_cta_t, sizeof(unsigned long long) * 6144) == cudaSuccess ? 0 : 1;
}
#endif

const char* fs_last_error(void) { return fs::g_last_error.c_str(); }

int fs_version(void) { return 300; }

int32_t fs_kv_splits(const fs_fwd_params* p) { return p ? fs::split_plan(p).splits : 0; }

int64_t fs_partial_floats(const fs_fwd_params* p) {
  if (!p) return 0;
  return fs::split_plan(p).part_rows * (fs::kernel_d(p) + 1);
}

fs_status fs_plan(const fs_fwd_params* p, int32_t clusters, fs_plan_info* out) {
  using namespace fs;
  if (!p || !out) return fail(FS_ERR_CONFIG, "fs_plan: null argument");
  if (p->kv_splits < FS_SPLITS_AUTO) return fail(FS_ERR_CONFIG, "kv_splits must be >= 0 or FS_SPLITS_AUTO");
  if (p->batch < 0 || p->heads_q < 1 || p->seqlen_q < 0 || p->seqlen_kv < 0 || p->head_dim < 1)
    return fail(FS_ERR_SHAPE, "fs_plan: bad extents");
  if (clusters <= 0) clusters = resident_clusters();
  const SplitPlan sp = split_plan(p, clusters);
  std::memset(out, 0, sizeof(*out));
  out->splits = sp.splits;
  out->split_tail = sp.tail;
  out->clusters = clusters;
  out->n_whole = sp.n_whole;
  out->tail_tiles = sp.tail_T;
  out->n_kv_tiles = sp.n_kv_tiles;
  out->work_tiles = sp.n_tiles0;
  out->items = sp.n_items;
  out->partial_floats = sp.part_rows * (kernel_d(p) + 1);
  // static-stride assignment of the items to G clusters: K/V steps on the busiest cluster and
  // the busy fraction (total steps / (G * busiest)).  Item i goes to cluster i % G.
  const int64_t G = out->clusters > 0 ? out->clusters : 1;
  auto item_len = [&](int64_t i) -> int64_t {
    int64_t split = 0;
    if (sp.tail) {
      if (i < sp.n_whole) return sp.n_kv_tiles;
      split = (i - sp.n_whole) % sp.splits;
    } else {
      split = (i / sp.n_qblk) % sp.splits;
    }
    return std::max<int64_t>(0, std::min<int64_t>(sp.split_tiles, sp.n_kv_tiles - split * sp.split_tiles));
  };
  const int64_t g_used = std::min<int64_t>(G, std::max<int64_t>(1, sp.n_items));
  int64_t busiest = 0, total = 0;
  if (sp.n_items <= (int64_t{1} << 22)) {
    std::vector<int64_t> load(static_cast<size_t>(g_used), 0);
    for (int64_t i = 0; i < sp.n_items; ++i) load[static_cast<size_t>(i % g_used)] += item_len(i);
    for (int64_t v : load) {
      busiest = std::max(busiest, v);
      total += v;
    }
  } else {  // closed form for huge launches (uniform length items)
    total = sp.n_items * item_len(0);
    busiest = ((sp.n_items + g_used - 1) / g_used) * item_len(0);
  }
  out->busiest_steps = static_cast<double>(busiest);
  out->efficiency = busiest > 0 ? static_cast<double>(total) / (static_cast<double>(G) * busiest) : 1.0;
  return FS_OK;
}

fs_status fs_combine(const fs_fwd_params* p, int32_t n_parts, fs_stream_t stream_) {
  using namespace fs;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (!p || !p->partial || n_parts < 1) return fail(FS_ERR_CONFIG, "fs_combine needs `partial` and n_parts >= 1");
  if (p->normalizer != FS_NORM_SPHERICAL && p->normalizer != FS_NORM_SIGNED_L1)
    return fail(FS_ERR_CONFIG, "normalizer must be FS_NORM_SPHERICAL or FS_NORM_SIGNED_L1");
  if (!(p->eps >= 0.0f) || !std::isfinite(p->eps)) return fail(FS_ERR_CONFIG, "denom_epsilon must be finite and >= 0");
  if (p->bad_key) {
    cudaError_t e = cudaMemsetAsync(p->bad_key, 0xFF, sizeof(uint64_t), stream);
    if (e != cudaSuccess) return fail(FS_ERR_CUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
  }
  return kernel_d(p) == 128 ? combine<128>(p, n_parts, stream) : combine<64>(p, n_parts, stream);
}

static fs_status check_peer(const fs_fwd_params* p, const fs_peer_params* pp) {
  using namespace fs;
  if (!p || !pp) return fail(FS_ERR_CONFIG, "null params");
  if (pp->world < 1 || pp->rank < 0 || pp->rank >= pp->world)
    return fail(FS_ERR_CONFIG, "peer: need 0 <= rank < world");
  if (pp->rows_per_rank < 1 || (int64_t)pp->rows_per_rank * pp->world < p->seqlen_q)
    return fail(FS_ERR_CONFIG, "peer: rows_per_rank * world must cover seqlen_q");
  if (!pp->peer_partial || !pp->local_partial || (reinterpret_cast<uintptr_t>(pp->local_partial) & 15u))
    return fail(FS_ERR_CONFIG, "peer: peer_partial (device array) and a 16-byte aligned local_partial are required");
  return FS_OK;
}

int64_t fs_peer_floats(const fs_fwd_params* p, const fs_peer_params* pp) {
  if (!p || !pp || pp->world < 1 || pp->rows_per_rank < 1) return 0;
  return (int64_t)pp->world * p->batch * p->heads_q * pp->rows_per_rank * (fs::kernel_d(p) + 1);
}

fs_status fs_fwd_peer(const fs_fwd_params* p, const fs_peer_params* pp, fs_stream_t stream) {
  fs_status st = check_peer(p, pp);
  if (st != FS_OK) return st;
  fs_fwd_params q = *p;
  q.kv_splits = 1;
  q.partial_only = 1;
  q.partial = nullptr;
  q.bad_key = nullptr;  // partials carry z; the owner's combine flags bad rows
  fs::g_peer = pp;
  st = fs_fwd(&q, stream);
  fs::g_peer = nullptr;
  return st;
}

fs_status fs_combine_peer(const fs_fwd_params* p, const fs_peer_params* pp, fs_stream_t stream_) {
  using namespace fs;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  fs_status st = check_peer(p, pp);
  if (st != FS_OK) return st;
  if (p->normalizer != FS_NORM_SPHERICAL && p->normalizer != FS_NORM_SIGNED_L1)
    return fail(FS_ERR_CONFIG, "normalizer must be FS_NORM_SPHERICAL or FS_NORM_SIGNED_L1");
  if (!(p->eps >= 0.0f) || !std::isfinite(p->eps)) return fail(FS_ERR_CONFIG, "denom_epsilon must be finite and >= 0");
  if (p->bad_key) {
    cudaError_t e = cudaMemsetAsync(p->bad_key, 0xFF, sizeof(uint64_t), stream);
    if (e != cudaSuccess) return fail(FS_ERR_CUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
  }
  return kernel_d(p) == 128 ? combine_peer<128>(p, pp, stream) : combine_peer<64>(p, pp, stream);
}

fs_status fs_ipc_malloc(int64_t bytes, void** ptr, void* handle64) {
  using namespace fs;
  if (!ptr || !handle64 || bytes <= 0) return fail(FS_ERR_CONFIG, "fs_ipc_malloc: bad arguments");
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle64), *ptr);
  if (e != cudaSuccess) return fail(FS_ERR_CUDA, std::string("fs_ipc_malloc: ") + cudaGetErrorString(e));
  return FS_OK;
}

fs_status fs_ipc_open(const void* handle64, void** ptr) {
  using namespace fs;
  if (!ptr || !handle64) return fail(FS_ERR_CONFIG, "fs_ipc_open: bad arguments");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(FS_ERR_CUDA, std::string("fs_ipc_open: ") + cudaGetErrorString(e));
  return FS_OK;
}

fs_status fs_ipc_close(void* ptr) {
  using namespace fs;
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  if (e != cudaSuccess) return fail(FS_ERR_CUDA, std::string("fs_ipc_close: ") + cudaGetErrorString(e));
  return FS_OK;
}

fs_status fs_ipc_free(void* ptr) {
  using namespace fs;
  cudaError_t e = cudaFree(ptr);
  if (e != cudaSuccess) return fail(FS_ERR_CUDA, std::string("fs_ipc_free: ") + cudaGetErrorString(e));
  return FS_OK;
}

int fs_query_tile(int head_dim, fs_dtype dt, int* bm, int* bn) {
  if (!bm || !bn || head_dim < 1 || head_dim > 128) return 1;
  if (dt != FS_F16 && dt != FS_BF16 && dt != FS_E4M3) return 1;
  *bm = fs::BM;
  *bn = fs::bn_for(dt, (dt == FS_E4M3 || head_dim > 64) ? 128 : 64);
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
  // the bad-row key carries the linear query row (b*H + h)*N + n in its upper 32 bits
  if (static_cast<int64_t>(p->batch) * p->heads_q * p->seqlen_q > static_cast<int64_t>(UINT32_MAX))
    return fail(FS_ERR_UNSUPPORTED, "batch * heads_q * seqlen_q must be < 2^32 (split the call)");
  auto aligned16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; };
  if (!aligned16(p->q) || !aligned16(p->k) || !aligned16(p->v) || !aligned16(p->o))  // NULL is aligned
    return fail(FS_ERR_UNSUPPORTED, "q/k/v/o must be 16-byte aligned");
  for (int i = 0; i < 3; ++i) {
    if ((p->q_stride[i] * eb) % 16 || (p->k_stride[i] * eb) % 16 || (p->v_stride[i] * eb) % 16 ||
        (p->o_stride[i] * ob) % 16)
      return fail(FS_ERR_UNSUPPORTED, "batch/token/head strides must be multiples of 16 bytes");
  }
  if (p->normalizer != FS_NORM_SPHERICAL && p->normalizer != FS_NORM_SIGNED_L1)
    return fail(FS_ERR_CONFIG, "normalizer must be FS_NORM_SPHERICAL or FS_NORM_SIGNED_L1");
  if (p->key_scale) {
    if (!aligned16(p->key_scale)) return fail(FS_ERR_UNSUPPORTED, "key_scale must be 16-byte aligned");
    if (p->batch > 1 && (p->key_scale_stride < p->seqlen_kv || (p->key_scale_stride * 4) % 16 != 0))
      return fail(FS_ERR_UNSUPPORTED, "key_scale_stride must be >= seqlen_kv and a multiple of 4 elements");
  }
  if (p->kv_splits < FS_SPLITS_AUTO) return fail(FS_ERR_CONFIG, "kv_splits must be >= 0 or FS_SPLITS_AUTO");
  if (p->split_tail != 0 && p->split_tail != 1) return fail(FS_ERR_CONFIG, "split_tail must be 0 or 1");
  if (g_peer == nullptr && (split_plan(p).splits > 1 || p->partial_only) &&
      (p->partial == nullptr || !aligned16(p->partial)))
    return fail(FS_ERR_CONFIG, "kv_splits > 1 / partial_only need a 16-byte aligned `partial` workspace of "
                               "fs_partial_floats(p) floats");
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
    p2.key_scale = nullptr;  // nothing is streamed: multiplicities are irrelevant
    p2.k = p2.v = p->q;
    for (int i = 0; i < 3; ++i) p2.k_stride[i] = p2.v_stride[i] = p->q_stride[i];
    p2.heads_kv = p->heads_q;
    p2.seqlen_kv = 0;
    return fs_fwd_dispatch(&p2, stream);
  }
  return fs_fwd_dispatch(p, stream);
}

}  // extern "C"
