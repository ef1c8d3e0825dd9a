// flashsign_prep.cu -- operand preparation for the drop-in (host-array) path.
//
// The reference accepts any float32 / float64 array (attention.py:252-279: q, k, v are upcast to
// float64 and every row is normalised in float64).  The tensor cores take 16-bit (or 8-bit)
// operands, so the caller's Q / K / V are converted here -- on the device, with no host round
// trip -- to the kernel's input dtype with one power-of-two scale per tensor:
//
//   x' = x * 2^e_x,  e_x chosen so that amax|x'| lies in [2^(T-1), 2^T)   (T = 14 fp16/bf16, 8 e4m3)
//
// and a power-of-two P scale chosen from the Cauchy-Schwarz bound |q'.k'| <= max||q'|| max||k'||,
// so that p * |s'| < 2^15 (fp16) / 2^8 (e4m3): the PV operand P = p s' can never overflow, for
// any finite input the reference accepts.  Spherical and signed-L1 normalisation are invariant
// to these factors (normalizers.py:94-117; the kernel folds them out exactly, Fold in
// flashsign_fwd.cu), so the result is the reference's up to the operands' rounding.
//
// fs_prepare = one memset + two kernels on the caller's stream:
//   1. stats:    amax and max row L2 norm of each present tensor (double, atomicMax on the bits)
//   2. quantise: every block derives the scales from the stats (same pure function), converts its
//                rows (zero-padded to d_pad) and block (0, 0) publishes {q, k, v descale, p_scale}
//                for fs_fwd_params.dev_scales.
// HBM-bound, one read of the source per kernel and one write of the operand.

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "../../include/flashsign.h"

namespace fsprep {

constexpr int kThreads = 256;

// ------------------------------------------------------------------ scale selection (device)
// e such that a * 2^e lies in [2^(target-1), 2^target); 0 for a = 0 / non-finite (inf and NaN pass
// through unscaled, so the reference's degenerate rows stay degenerate).
__device__ __forceinline__ int pow2_exp(double a, int target) {
  if (!(a > 0.0) || isinf(a)) return 0;
  int e = target - 1 - ilogb(a);
  return max(-120, min(120, e));
}

struct Scales {
  int eq, ek, ev, ep;  // operand exponents and the P exponent
};

__device__ __forceinline__ int target_exp(int dst) { return dst == FS_E4M3 ? 8 : 14; }
__device__ __forceinline__ int p_target_exp(int dst) { return dst == FS_E4M3 ? 8 : 15; }

// stats: {amax_q, rn_q, amax_k, rn_k, amax_v, rn_v}.  Each operand exponent depends on its own
// tensor only (K / V converted once stay valid for every later query chunk); only p_scale, which
// is applied inside fs_fwd and never baked into an operand, combines q and k.
__device__ Scales choose_scales(const double* st, int dst, int exact, int norm, float scale, float eps) {
  Scales s;
  const int T = target_exp(dst);
  // eps is folded as eps / g^2 (eps / |g|) with g = c 2^-(eq+ek): cap each of eq, ek so that even
  // both at the cap keep it below 2^100 (bites only when tiny q, k meet eps > 0)
  int cap = 120;
  if (eps > 0.f && scale != 0.f && !exact) {
    const double r = log2(fabs(static_cast<double>(scale))) * (norm == FS_NORM_SIGNED_L1 ? 1.0 : 2.0) -
                     log2(static_cast<double>(eps));  // log2(c^2 / eps) or log2(|c| / eps)
    cap = static_cast<int>(floor((100.0 + r) / (norm == FS_NORM_SIGNED_L1 ? 2.0 : 4.0)));
  }
  s.eq = exact ? 0 : min(pow2_exp(st[0], T), cap);
  s.ek = exact ? 0 : min(pow2_exp(st[2], T), cap);
  s.ev = exact ? 0 : pow2_exp(st[4], T);
  s.ep = 0;
  if (dst != FS_BF16) {  // bf16 has the fp32 range: P needs no scale
    const double bound = st[1] * exp2(static_cast<double>(s.eq)) * st[3] * exp2(static_cast<double>(s.ek));
    s.ep = pow2_exp(bound, p_target_exp(dst));
  }
  return s;
}

// ------------------------------------------------------------------ element access
template <typename T>
__device__ __forceinline__ double load_d(const T* p);
template <>
__device__ __forceinline__ double load_d<float>(const float* p) { return static_cast<double>(*p); }
template <>
__device__ __forceinline__ double load_d<double>(const double* p) { return *p; }
template <>
__device__ __forceinline__ double load_d<__half>(const __half* p) { return static_cast<double>(__half2float(*p)); }
template <>
__device__ __forceinline__ double load_d<__nv_bfloat16>(const __nv_bfloat16* p) {
  return static_cast<double>(__bfloat162float(*p));
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // non-negative doubles (and NaN, whose bits exceed +inf's) order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr), static_cast<unsigned long long>(__double_as_longlong(v)));
}

struct TensorArgs {
  const void* src;
  int64_t rows, src_stride, dst_stride;
  void* dst;
  int32_t d, src_dtype;
};
struct PrepArgs {
  TensorArgs t[3];
  int32_t dst_dtype, d_pad, exact, normalizer;
  float scale, eps;
  double* stats;
  float* scales;
};

// One warp per row (d <= 128: four elements per lane), grid-stride; per-block maxima in shared
// memory, one global atomic per block and tensor.
template <typename T>
__device__ void stats_rows(const TensorArgs& a, double* out) {
  __shared__ unsigned long long s_amax, s_rn;
  if (threadIdx.x == 0) s_amax = s_rn = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  double amax = 0.0, rn2 = 0.0;
  const T* src = static_cast<const T*>(a.src);
  for (int64_t r = warp0; r < a.rows; r += nwarps) {
    const T* row = src + r * a.src_stride;
    double ss = 0.0;
    for (int c = lane; c < a.d; c += 32) {
      const double x = load_d(row + c);
      const double ax = fabs(x);
      amax = (ax > amax || isnan(ax)) ? ax : amax;
      ss = fma(x, x, ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    rn2 = (ss > rn2 || isnan(ss)) ? ss : rn2;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oa = __shfl_xor_sync(0xffffffffu, amax, o);
    amax = (oa > amax || isnan(oa)) ? oa : amax;
  }
  if (lane == 0) {
    atomicMax(&s_amax, static_cast<unsigned long long>(__double_as_longlong(amax)));
    atomicMax(&s_rn, static_cast<unsigned long long>(__double_as_longlong(sqrt(rn2))));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomic_max_nonneg(out, __longlong_as_double(static_cast<long long>(s_amax)));
    atomic_max_nonneg(out + 1, __longlong_as_double(static_cast<long long>(s_rn)));
  }
}

__global__ void __launch_bounds__(kThreads) stats_kernel(PrepArgs p) {
  const TensorArgs& a = p.t[blockIdx.y];
  if (a.src == nullptr || a.rows == 0) return;
  double* out = p.stats + 2 * blockIdx.y;
  switch (a.src_dtype) {
    case FS_F32: stats_rows<float>(a, out); break;
    case FS_F64: stats_rows<double>(a, out); break;
    case FS_F16: stats_rows<__half>(a, out); break;
    default: stats_rows<__nv_bfloat16>(a, out); break;
  }
}

template <int DST>
__device__ __forceinline__ void store_dst(void* dst, int64_t i, double x);
template <>
__device__ __forceinline__ void store_dst<FS_F16>(void* dst, int64_t i, double x) {
  static_cast<__half*>(dst)[i] = __double2half(x);
}
template <>
__device__ __forceinline__ void store_dst<FS_BF16>(void* dst, int64_t i, double x) {
  static_cast<__nv_bfloat16*>(dst)[i] = __double2bfloat16(x);
}
template <>
__device__ __forceinline__ void store_dst<FS_E4M3>(void* dst, int64_t i, double x) {
  static_cast<__nv_fp8_storage_t*>(dst)[i] = __nv_cvt_double_to_fp8(x, __NV_SATFINITE, __NV_E4M3);
}

// One thread per output element of [rows, d_pad] (columns >= d written as 0).  The conversion
// rounds once, from the exact double product x * 2^e, to the operand dtype (RNE).
template <typename T, int DST>
__device__ void quant_rows(const TensorArgs& a, int d_pad, int e) {
  const double mul = exp2(static_cast<double>(e));
  const T* src = static_cast<const T*>(a.src);
  const int64_t n = a.rows * d_pad;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / d_pad;
    const int c = static_cast<int>(i - r * d_pad);
    const double x = c < a.d ? load_d(src + r * a.src_stride + c) * mul : 0.0;
    store_dst<DST>(a.dst, r * a.dst_stride + c, x);
  }
}

template <int DST>
__device__ void quant_tensor(const TensorArgs& a, int d_pad, int e) {
  switch (a.src_dtype) {
    case FS_F32: quant_rows<float, DST>(a, d_pad, e); break;
    case FS_F64: quant_rows<double, DST>(a, d_pad, e); break;
    case FS_F16: quant_rows<__half, DST>(a, d_pad, e); break;
    default: quant_rows<__nv_bfloat16, DST>(a, d_pad, e); break;
  }
}

__global__ void __launch_bounds__(kThreads) quant_kernel(PrepArgs p) {
  const Scales s = choose_scales(p.stats, p.dst_dtype, p.exact, p.normalizer, p.scale, p.eps);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    p.scales[0] = static_cast<float>(exp2(-static_cast<double>(s.eq)));
    p.scales[1] = static_cast<float>(exp2(-static_cast<double>(s.ek)));
    p.scales[2] = static_cast<float>(exp2(-static_cast<double>(s.ev)));
    p.scales[3] = static_cast<float>(exp2(static_cast<double>(s.ep)));
  }
  const TensorArgs& a = p.t[blockIdx.y];
  if (a.src == nullptr || a.rows == 0) return;
  const int e = blockIdx.y == 0 ? s.eq : (blockIdx.y == 1 ? s.ek : s.ev);
  switch (p.dst_dtype) {
    case FS_F16: quant_tensor<FS_F16>(a, p.d_pad, e); break;
    case FS_BF16: quant_tensor<FS_BF16>(a, p.d_pad, e); break;
    default: quant_tensor<FS_E4M3>(a, p.d_pad, e); break;
  }
}

// ------------------------------------------------------------------ K' = m K (fs_scale_keys)
// One 16-byte chunk (8 elements of one key row) per thread and step: read, multiply in fp32 (exact
// for integer m and 16-bit K), round to nearest even, write.  HBM-bound streaming pass.
template <typename T>
__global__ void __launch_bounds__(kThreads) scale_keys_kernel(const T* __restrict__ k, T* __restrict__ out,
                                                              const float* __restrict__ m, int64_t m_sb,
                                                              int64_t k_sb, int64_t k_sn, int64_t k_sh,
                                                              int64_t o_sb, int64_t o_sn, int64_t o_sh, int n,
                                                              int h, int cpr, int64_t chunks) {
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; c < chunks;
       c += static_cast<int64_t>(gridDim.x) * kThreads) {
    const int col = static_cast<int>(c % cpr) * 8;
    const int64_t row = c / cpr;  // (b * n + j) * h + g
    const int g = static_cast<int>(row % h);
    const int64_t bj = row / h;
    const int j = static_cast<int>(bj % n);
    const int64_t b = bj / n;
    const float mj = m[b * m_sb + j];
    const uint4 w = *reinterpret_cast<const uint4*>(k + b * k_sb + j * k_sn + g * k_sh + col);
    uint4 r;
    const uint32_t* wi = reinterpret_cast<const uint32_t*>(&w);
    uint32_t* ri = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (std::is_same<T, __half>::value) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&wi[i]));
        const __half2 o = __floats2half2_rn(f.x * mj, f.y * mj);
        ri[i] = *reinterpret_cast<const uint32_t*>(&o);
      } else {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wi[i]));
        const __nv_bfloat162 o = __floats2bfloat162_rn(f.x * mj, f.y * mj);
        ri[i] = *reinterpret_cast<const uint32_t*>(&o);
      }
    }
    *reinterpret_cast<uint4*>(out + b * o_sb + j * o_sn + g * o_sh + col) = r;
  }
}

}  // namespace fsprep

namespace fs {
void set_last_error(const char* msg);  // flashsign_fwd.cu: the text fs_last_error returns
}

extern "C" {

fs_status fs_prepare(const fs_prep_params* p, fs_stream_t stream_) {
  using namespace fsprep;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  auto fail = [](fs_status st, const char* m) {
    fs::set_last_error(m);
    return st;
  };
  if (!p || !p->stats || !p->scales) return fail(FS_ERR_CONFIG, "fs_prepare: stats and scales are required");
  if (p->dst_dtype != FS_F16 && p->dst_dtype != FS_BF16 && p->dst_dtype != FS_E4M3)
    return fail(FS_ERR_DTYPE, "fs_prepare: dst_dtype must be FS_F16, FS_BF16 or FS_E4M3");
  if (p->mode != FS_PREP_SCALE && p->mode != FS_PREP_EXACT) return fail(FS_ERR_CONFIG, "fs_prepare: bad mode");
  if (!(p->eps >= 0.f) || !std::isfinite(p->eps) || !std::isfinite(p->scale))
    return fail(FS_ERR_CONFIG, "fs_prepare: scale must be finite and eps finite and >= 0");
  PrepArgs a;
  int64_t most = 0;
  for (int i = 0; i < 3; ++i) {
    const fs_prep_tensor& t = p->t[i];
    TensorArgs& x = a.t[i];
    x.src = t.src;
    x.rows = t.src ? t.rows : 0;
    x.src_stride = t.src_row_stride;
    x.dst_stride = t.dst_row_stride;
    x.dst = t.dst;
    x.d = t.d;
    x.src_dtype = t.src_dtype;
    if (!t.src) continue;
    if (t.src_dtype != FS_F32 && t.src_dtype != FS_F64 && t.src_dtype != FS_F16 && t.src_dtype != FS_BF16)
      return fail(FS_ERR_DTYPE, "fs_prepare: src_dtype must be FS_F32, FS_F64, FS_F16 or FS_BF16");
    if (t.rows < 0 || t.d < 1 || t.d > p->d_pad || t.src_row_stride < t.d || t.dst_row_stride < p->d_pad ||
        (t.rows > 0 && !t.dst))
      return fail(FS_ERR_SHAPE, "fs_prepare: need rows >= 0, 1 <= d <= d_pad <= row strides, dst");
    most = std::max<int64_t>(most, t.rows * p->d_pad);
    // reset this tensor's stats (the others are reused: the K / V of a chunked query stream)
    cudaError_t e = cudaMemsetAsync(p->stats + 2 * i, 0, 2 * sizeof(double), stream);
    if (e != cudaSuccess) return fail(FS_ERR_CUDA, cudaGetErrorString(e));
  }
  a.dst_dtype = p->dst_dtype;
  a.d_pad = p->d_pad;
  a.exact = p->mode == FS_PREP_EXACT;
  a.normalizer = p->normalizer;
  a.scale = p->scale;
  a.eps = p->eps;
  a.stats = p->stats;
  a.scales = p->scales;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (most + kThreads - 1) / kThreads;
  const unsigned gx = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, 8LL * sms)));
  stats_kernel<<<dim3(gx, 3), kThreads, 0, stream>>>(a);
  quant_kernel<<<dim3(gx, 3), kThreads, 0, stream>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FS_ERR_CUDA, cudaGetErrorString(e));
  return FS_OK;
}

fs_status fs_scale_keys(const fs_fwd_params* p, void* k_out, const int64_t* k_out_stride, fs_stream_t stream_) {
  using namespace fsprep;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  auto fail = [](fs_status st, const char* m) {
    fs::set_last_error(m);
    return st;
  };
  if (!p || !k_out || !k_out_stride || !p->key_scale)
    return fail(FS_ERR_CONFIG, "fs_scale_keys: params, key_scale, k_out and its strides are required");
  if (p->in_dtype != FS_F16 && p->in_dtype != FS_BF16)
    return fail(FS_ERR_DTYPE, "fs_scale_keys: in_dtype must be FS_F16 or FS_BF16");
  if (p->batch < 0 || p->seqlen_kv < 0 || p->heads_kv < 1 || p->head_dim < 1 || p->head_dim % 8 != 0)
    return fail(FS_ERR_SHAPE, "fs_scale_keys: bad extents (head_dim a multiple of 8)");
  auto al16 = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15u) == 0; };
  for (int i = 0; i < 3; ++i)
    if ((p->k_stride[i] * 2) % 16 || (k_out_stride[i] * 2) % 16)
      return fail(FS_ERR_UNSUPPORTED, "fs_scale_keys: strides must be multiples of 16 bytes");
  if (!al16(p->k) || !al16(k_out)) return fail(FS_ERR_UNSUPPORTED, "fs_scale_keys: 16-byte aligned k / k_out");
  const int cpr = p->head_dim / 8;
  const int64_t chunks = static_cast<int64_t>(p->batch) * p->seqlen_kv * p->heads_kv * cpr;
  if (chunks == 0) return FS_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid =
      static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((chunks + kThreads - 1) / kThreads, 16LL * sms)));
  const int64_t m_sb = p->batch > 1 ? p->key_scale_stride : 0;
  if (p->in_dtype == FS_F16)
    scale_keys_kernel<__half><<<grid, kThreads, 0, stream>>>(
        static_cast<const __half*>(p->k), static_cast<__half*>(k_out), p->key_scale, m_sb, p->k_stride[0],
        p->k_stride[1], p->k_stride[2], k_out_stride[0], k_out_stride[1], k_out_stride[2], p->seqlen_kv,
        p->heads_kv, cpr, chunks);
  else
    scale_keys_kernel<__nv_bfloat16><<<grid, kThreads, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(p->k), static_cast<__nv_bfloat16*>(k_out), p->key_scale, m_sb,
        p->k_stride[0], p->k_stride[1], p->k_stride[2], k_out_stride[0], k_out_stride[1], k_out_stride[2],
        p->seqlen_kv, p->heads_kv, cpr, chunks);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(FS_ERR_CUDA, cudaGetErrorString(e));
  return FS_OK;
}

}  // extern "C"
