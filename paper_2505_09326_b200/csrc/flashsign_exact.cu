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
//   phase 1: S = Q K^T (thread: one row x 8 keys, float64 dot products), reference rounding
//   phase 2: o += s v_j for every key in order (thread: one row x d/4 columns), z likewise
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
  constexpr int DP = D + 1;  // padded row stride (doubles): rows land in different banks
  extern __shared__ double sm[];
  double* qs = sm;                 // [BR][DP]
  double* ks = qs + BR * DP;       // [BC][DP]
  double* vs = ks + BC * DP;       // [BC][DP]
  double* ss = vs + BC * DP;       // [BR][BC + 1] scores after the reference's rounding
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
  const int row = tid >> 2, sub = tid & 3;  // phase 1 / 2 ownership: 4 threads per row
  constexpr int NW = D / 4;
  double o[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) o[w] = 0.0;
  double z = 0.0;
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
    // phase 1: keys sub, sub + 4, ... of this tile for `row`
#pragma unroll
    for (int u = 0; u < BC / 4; ++u) {
      const int c = sub + 4 * u;
      double s = 0.0;
#pragma unroll 8
      for (int a = 0; a < D; ++a) s = fma(qs[row * DP + a], ks[c * DP + a], s);
      if constexpr (F32) {
        float sf = static_cast<float>(s);
        if (scale != 1.0) sf *= scale_f;
        s = static_cast<double>(sf);
      } else if (scale != 1.0) {
        s *= scale;
      }
      ss[row * (BC + 1) + c] = s;
    }
    __syncthreads();
    // phase 2: every key of the tile in order
    for (int c = 0; c < nc; ++c) {
      const double s = ss[row * (BC + 1) + c];
      double a2;
      if constexpr (NORM == FS_NORM_SIGNED_L1) {
        a2 = fabs(s);
      } else if constexpr (F32) {
        const float sf = static_cast<float>(s);
        a2 = static_cast<double>(sf * sf);  // the float32 grid squares in float32
      } else {
        a2 = s * s;
      }
      z += a2;
#pragma unroll
      for (int w = 0; w < NW; ++w) o[w] = fma(s, vs[c * DP + sub + 4 * w], o[w]);
    }
  }
  const int n = r0 + row;
  if (n >= p.seqlen_q) return;
  const double zz = p.eps != 0.0 ? z + p.eps : z;
  const double den = NORM == FS_NORM_SIGNED_L1 ? zz : sqrt(zz);
  const bool bad = !(den != 0.0) || !isfinite(den);
  const uint64_t lin = static_cast<uint64_t>(bh) * p.seqlen_q + n;
  if (sub == 0) {
    if (p.z_out) p.z_out[lin] = z;
    if (bad && p.bad_key)
      atomicMin(reinterpret_cast<unsigned long long*>(p.bad_key),
                static_cast<unsigned long long>((lin << 32) | __float_as_uint(static_cast<float>(z))));
  }
  double* dst = p.o + b * p.o_stride[0] + static_cast<int64_t>(n) * p.o_stride[1] + h * p.o_stride[2];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int a = sub + 4 * w;
    if (a < d) dst[a] = o[w] / den;
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
    const size_t smem = sizeof(double) * (static_cast<size_t>(BR + 2 * BC) * (d + 1) + BR * (BC + 1));
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
