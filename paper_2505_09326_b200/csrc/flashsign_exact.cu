// flashsign_exact.cu -- float64 streamed FlashSign for the drop-in path's float32 / float64 callers.
//
// The reference's streamed loop (attention.py:146-200) computes in float64: scores s = q_i . k_j
// (rounded to float32 when the caller's arrays are float32, attention.py:163-166, then scaled in
// float32), a2(s) summed into a float64 z (attention.py:188; for float32 grids the squares are
// float32), o += a1(s) v_j in float64 (attention.py:183-187), O = o / b(z + eps).  The tensor-core
// kernel cannot reach the float64 tolerances the reference's own tests use (rtol 1e-12), so the
// drop-in API's `f64` compute mode runs this kernel instead: the same algorithm and rounding
// points on the SM's FP64 units, keys accumulated strictly in order for every row (so appending
// or deleting a zero-score key leaves the output bit-identical, as in the reference).
//
// CTA = (b, h, 64 query rows), 256 threads; K / V stream through shared memory in 32-key tiles:
//   phase 1: S = Q K^T (thread: 2 rows x 4 keys, float64 dot products), reference rounding
//   phase 2: o += s v_j for every key in order (thread: 2 rows x d/8 columns), z likewise
// Epilogue: b(z + eps), the first-bad-row key of fs_fwd (packed (linear row << 32) | float bits),
// per-row z in float64 for the exception text, O in float64.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "../../include/flashsign.h"

namespace fs {
void set_last_error(const char* msg);

namespace exact {

constexpr int BR = 64;       // query rows per CTA
constexpr int BC = 32;       // keys per tile
constexpr int THREADS = 256;

template <int D, int NORM, bool F32>
__global__ void __launch_bounds__(THREADS) exact_kernel(fs_exact_params p) {
  // Register-blocked: thread t owns rows {t/8, t/8 + 32} of the CTA's 64 and, in phase 1, keys
  // {t%8 + 8u} of the tile (2 x 4 scores), in phase 2 columns {2 (t%8) + 16 w, + 1} (2 x D/8
  // accumulators).  Rows are padded to D + 2 doubles so 16-byte loads of eight different keys
  // (or columns) land in different banks.
  constexpr int DP = D + 2;
  constexpr int SP = BC + 1;
  constexpr int NW = D / 16;  // column pairs per thread
  extern __shared__ double sm[];
  double* qs = sm;                 // [BR][DP]
  double* ks = qs + BR * DP;       // [BC][DP]
  double* vs = ks + BC * DP;       // [BC][DP]
  double* ss = vs + BC * DP;       // [BR][SP] scores after the reference's rounding
  const int tid = threadIdx.x;
  const int n_rb = (p.seqlen_q + BR - 1) / BR;
  const int rb = blockIdx.x % n_rb;
  const int bh = blockIdx.x / n_rb;
  const int h = bh % p.heads_q, b = bh / p.heads_q;
  const int g = static_cast<int>((static_cast<int64_t>(h) * p.heads_kv) / p.heads_q);
  const int r0 = rb * BR;
  const int d = p.head_dim;
  for (int e = tid; e < BR * D; e += THREADS) {
    const int r = e / D, a = e % D;
    const int n = r0 + r;
    qs[r * DP + a] = (n < p.seqlen_q && a < d) ? p.q[b * p.q_stride[0] + n * p.q_stride[1] + h * p.q_stride[2] + a] : 0.0;
  }
  const int rg = tid >> 3, kg = tid & 7;
  double o[2][2 * NW];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int w = 0; w < 2 * NW; ++w) o[i][w] = 0.0;
  double z[2] = {0.0, 0.0};
  const double scale = p.scale;
  const float scale_f = static_cast<float>(p.scale);
  for (int c0 = 0; c0 < p.seqlen_kv; c0 += BC) {
    const int nc = min(BC, p.seqlen_kv - c0);
    __syncthreads();  // previous tile fully consumed
    for (int e = tid; e < BC * D; e += THREADS) {
      const int c = e / D, a = e % D;
      const bool ok = c < nc && a < d;
      const int64_t off = b * p.k_stride[0] + static_cast<int64_t>(c0 + c) * p.k_stride[1] + g * p.k_stride[2] + a;
      const int64_t offv = b * p.v_stride[0] + static_cast<int64_t>(c0 + c) * p.v_stride[1] + g * p.v_stride[2] + a;
      ks[c * DP + a] = ok ? p.k[off] : 0.0;
      vs[c * DP + a] = ok ? p.v[offv] : 0.0;
    }
    __syncthreads();
    // phase 1: the 2 x 4 score block
    {
      double acc[2][4] = {};
#pragma unroll 4
      for (int a = 0; a < D; a += 2) {
        const double2 q0 = *reinterpret_cast<const double2*>(qs + rg * DP + a);
        const double2 q1 = *reinterpret_cast<const double2*>(qs + (rg + 32) * DP + a);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 kv = *reinterpret_cast<const double2*>(ks + (kg + 8 * u) * DP + a);
          acc[0][u] = fma(q0.y, kv.y, fma(q0.x, kv.x, acc[0][u]));
          acc[1][u] = fma(q1.y, kv.y, fma(q1.x, kv.x, acc[1][u]));
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          double sv = acc[i][u];
          if constexpr (F32) {
            float sf = static_cast<float>(sv);
            if (scale != 1.0) sf *= scale_f;
            sv = static_cast<double>(sf);
          } else if (scale != 1.0) {
            sv *= scale;
          }
          ss[(rg + 32 * i) * SP + kg + 8 * u] = sv;
        }
    }
    __syncthreads();
    // phase 2: every key of the tile in order
    for (int c = 0; c < nc; ++c) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double sv = ss[(rg + 32 * i) * SP + c];
        double a2;
        if constexpr (NORM == FS_NORM_SIGNED_L1) {
          a2 = fabs(sv);
        } else if constexpr (F32) {
          const float sf = static_cast<float>(sv);
          a2 = static_cast<double>(sf * sf);  // the float32 grid squares in float32
        } else {
          a2 = sv * sv;
        }
        z[i] += a2;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const double2 vv = *reinterpret_cast<const double2*>(vs + c * DP + 2 * kg + 16 * w);
          o[i][2 * w] = fma(sv, vv.x, o[i][2 * w]);
          o[i][2 * w + 1] = fma(sv, vv.y, o[i][2 * w + 1]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int n = r0 + rg + 32 * i;
    if (n >= p.seqlen_q) continue;
    const double zz = p.eps != 0.0 ? z[i] + p.eps : z[i];
    const double den = NORM == FS_NORM_SIGNED_L1 ? zz : sqrt(zz);
    const bool bad = !(den != 0.0) || !isfinite(den);
    const uint64_t lin = static_cast<uint64_t>(bh) * p.seqlen_q + n;
    if (kg == 0) {
      if (p.z_out) p.z_out[lin] = z[i];
      if (bad && p.bad_key)
        atomicMin(reinterpret_cast<unsigned long long*>(p.bad_key),
                  static_cast<unsigned long long>((lin << 32) | __float_as_uint(static_cast<float>(z[i]))));
    }
    double* dst = p.o + b * p.o_stride[0] + static_cast<int64_t>(n) * p.o_stride[1] + h * p.o_stride[2];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int a = 2 * kg + 16 * w;
      if (a < d) dst[a] = o[i][2 * w] / den;
      if (a + 1 < d) dst[a + 1] = o[i][2 * w + 1] / den;
    }
  }
}

}  // namespace exact
}  // namespace fs

extern "C" fs_status fs_exact_fwd(const fs_exact_params* p, fs_stream_t stream_) {
  using namespace fs::exact;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  auto fail = [](fs_status st, const char* m) {
    fs::set_last_error(m);
    return st;
  };
  if (!p) return fail(FS_ERR_CONFIG, "null params");
  if (p->batch < 0 || p->heads_q < 1 || p->heads_kv < 1 || p->seqlen_q < 0 || p->seqlen_kv < 0)
    return fail(FS_ERR_SHAPE, "negative or zero extents (batch>=0, heads>=1, seqlen>=0)");
  if (p->heads_q % p->heads_kv != 0) return fail(FS_ERR_CONFIG, "query heads must be a multiple of kv heads");
  if (p->head_dim < 1 || p->head_dim > 128) return fail(FS_ERR_UNSUPPORTED, "head_dim must be in [1, 128]");
  if (p->normalizer != FS_NORM_SPHERICAL && p->normalizer != FS_NORM_SIGNED_L1)
    return fail(FS_ERR_CONFIG, "normalizer must be FS_NORM_SPHERICAL or FS_NORM_SIGNED_L1");
  if (!std::isfinite(p->scale)) return fail(FS_ERR_CONFIG, "score_scale must be finite");
  if (!(p->eps >= 0.0) || !std::isfinite(p->eps)) return fail(FS_ERR_CONFIG, "denom_epsilon must be finite and >= 0");
  if (p->bad_key) {
    cudaError_t e = cudaMemsetAsync(p->bad_key, 0xFF, sizeof(uint64_t), stream);
    if (e != cudaSuccess) return fail(FS_ERR_CUDA, cudaGetErrorString(e));
  }
  if (p->batch == 0 || p->seqlen_q == 0) return FS_OK;
  if (!p->q || !p->o || (p->seqlen_kv > 0 && (!p->k || !p->v))) return fail(FS_ERR_CONFIG, "null tensor pointer");
  const int64_t blocks = static_cast<int64_t>((p->seqlen_q + BR - 1) / BR) * p->heads_q * p->batch;
  if (blocks > INT32_MAX) return fail(FS_ERR_UNSUPPORTED, "too many query blocks");
  auto go = [&](auto kern, int d) {
    const size_t smem = sizeof(double) * (static_cast<size_t>(BR + 2 * BC) * (d + 2) + BR * (BC + 1));
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<static_cast<unsigned>(blocks), THREADS, smem, stream>>>(*p);
  };
  const bool l1 = p->normalizer == FS_NORM_SIGNED_L1;
  const bool f32 = p->f32_grid != 0;
#define FS_EXACT_GO(D)                                                                                         \
  (l1 ? (f32 ? go(exact_kernel<D, FS_NORM_SIGNED_L1, true>, D) : go(exact_kernel<D, FS_NORM_SIGNED_L1, false>, D)) \
      : (f32 ? go(exact_kernel<D, FS_NORM_SPHERICAL, true>, D) : go(exact_kernel<D, FS_NORM_SPHERICAL, false>, D)))
  if (p->head_dim <= 32)
    FS_EXACT_GO(32);
  else if (p->head_dim <= 64)
    FS_EXACT_GO(64);
  else
    FS_EXACT_GO(128);
#undef FS_EXACT_GO
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FS_ERR_CUDA, cudaGetErrorString(e));
  return FS_OK;
}
