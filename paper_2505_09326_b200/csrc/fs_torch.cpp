// fs_torch.cpp -- PyTorch C++ extension over the FlashSign C-ABI (include/flashsign.h).
//
// The torch-native entry `flashsign.fwd_async` (the batched, device-resident form of the
// reference's multi_head_attention_array, attention.py:318-361) lands here: tensor checks,
// output / bad-row-key / split-workspace allocation, the automatic K/V split choice and the
// fs_fwd call all happen in C++ on the caller's current CUDA stream, so a call costs a few
// microseconds of host time (the TMA descriptors are cached inside libflashsign.so).
// The extension holds no kernels: it links libflashsign.so ($ORIGIN rpath) and calls the C-ABI,
// exactly what an external binding would do.

#include <ATen/cuda/CUDAContext.h>
#include <c10/cuda/CUDAGuard.h>
#include <torch/extension.h>

#include <algorithm>
#include <cmath>
#include <mutex>

#include "../../include/flashsign.h"

namespace {

int in_code(at::ScalarType t) {
  switch (t) {
    case at::kHalf: return FS_F16;
    case at::kBFloat16: return FS_BF16;
    case at::kFloat8_e4m3fn: return FS_E4M3;
    default: return -1;
  }
}
int out_code(at::ScalarType t) {
  switch (t) {
    case at::kHalf: return FS_F16;
    case at::kBFloat16: return FS_BF16;
    case at::kFloat: return FS_F32;
    default: return -1;
  }
}

// Python raises the mapped exception (ShapeMismatchError / ConfigError / RuntimeError) from the
// status; validation failures detected here use the same codes.
struct Fail {
  int status;
  std::string msg;
};

void check_bshd(const at::Tensor& t, const char* name) {
  if (!t.is_cuda()) throw Fail{FS_ERR_CUDA, std::string("flashsign: ") + name + " must be a CUDA tensor (no CPU fallback)"};
  if (t.dim() != 4) throw Fail{FS_ERR_SHAPE, std::string("flashsign: ") + name + " must be BSHD rank-4"};
  if (t.stride(3) != 1) throw Fail{FS_ERR_SHAPE, std::string("flashsign: ") + name + " head dim must be contiguous"};
}

// Returns (status, message, out, bad_key, partial, n_parts).
py::tuple fwd(const at::Tensor& q, const at::Tensor& k, const at::Tensor& v, c10::optional<at::Tensor> out,
              c10::optional<at::ScalarType> out_dtype, c10::optional<at::Tensor> bad_key, double scale, double eps,
              double p_scale, double q_descale, double k_descale, double v_descale, int64_t normalizer,
              c10::optional<at::Tensor> key_scale, int64_t kv_splits, c10::optional<at::Tensor> partial,
              bool partial_only, c10::optional<at::Tensor> dev_scales, int64_t tile_m, int64_t tile_n,
              bool split_tail) {
  try {
    check_bshd(q, "q");
    check_bshd(k, "k");
    check_bshd(v, "v");
    if (q.scalar_type() != k.scalar_type() || q.scalar_type() != v.scalar_type())
      throw Fail{FS_ERR_SHAPE, "dtype mismatch: q, k, v must share a dtype"};
    const int ic = in_code(q.scalar_type());
    if (ic < 0) throw Fail{FS_ERR_SHAPE, "flashsign: unsupported input dtype (bf16, fp16, float8_e4m3fn)"};
    if (q.device() != k.device() || q.device() != v.device())
      throw Fail{FS_ERR_CUDA, "flashsign: q, k, v must be on the same device"};
    const int64_t b = q.size(0), nq = q.size(1), h = q.size(2), d = q.size(3);
    const int64_t nkv = k.size(1), hkv = k.size(2);
    if (k.size(0) != b || v.size(0) != b) throw Fail{FS_ERR_SHAPE, "batch mismatch between q, k, v"};
    if (k.size(3) != d) throw Fail{FS_ERR_SHAPE, "Q and K feature dims differ"};
    if (v.size(1) != nkv || v.size(2) != hkv) throw Fail{FS_ERR_SHAPE, "K and V shapes differ"};
    if (v.size(3) != d) throw Fail{FS_ERR_SHAPE, "flashsign: value dim must equal head dim"};
    if (h < 1 || hkv < 1 || h % hkv != 0)
      throw Fail{FS_ERR_CONFIG, "query heads must be a multiple of kv heads, got h=" + std::to_string(h) +
                                    ", h_kv=" + std::to_string(hkv)};
    if (!std::isfinite(scale)) throw Fail{FS_ERR_CONFIG, "score_scale must be finite"};
    const c10::cuda::CUDAGuard guard(q.device());
    const auto dev = q.device();
    at::ScalarType odt;
    if (out_dtype.has_value())
      odt = *out_dtype;
    else if (out.has_value())
      odt = out->scalar_type();
    else
      odt = (q.scalar_type() == at::kHalf || q.scalar_type() == at::kBFloat16) ? q.scalar_type() : at::kBFloat16;
    const int oc = out_code(odt);
    if (oc < 0) throw Fail{FS_ERR_SHAPE, "flashsign: unsupported output dtype"};
    at::Tensor o;
    if (out.has_value()) {
      o = *out;
      if (o.dim() != 4 || o.size(0) != b || o.size(1) != nq || o.size(2) != h || o.size(3) != d ||
          o.scalar_type() != odt || o.stride(3) != 1 || o.device() != dev)
        throw Fail{FS_ERR_SHAPE, "flashsign: bad out tensor"};
    } else {
      o = at::empty({b, nq, h, d}, q.options().dtype(odt));
    }
    at::Tensor bad = bad_key.has_value() ? *bad_key : at::empty({1}, q.options().dtype(at::kLong));

    fs_fwd_params p;
    std::memset(&p, 0, sizeof(p));
    p.q = q.data_ptr();
    p.k = k.data_ptr();
    p.v = v.data_ptr();
    p.o = o.data_ptr();
    for (int i = 0; i < 3; ++i) {
      p.q_stride[i] = q.stride(i);
      p.k_stride[i] = k.stride(i);
      p.v_stride[i] = v.stride(i);
      p.o_stride[i] = o.stride(i);
    }
    p.batch = static_cast<int32_t>(b);
    p.heads_q = static_cast<int32_t>(h);
    p.heads_kv = static_cast<int32_t>(hkv);
    p.seqlen_q = static_cast<int32_t>(nq);
    p.seqlen_kv = static_cast<int32_t>(nkv);
    p.head_dim = static_cast<int32_t>(d);
    p.in_dtype = static_cast<fs_dtype>(ic);
    p.out_dtype = static_cast<fs_dtype>(oc);
    p.scale = static_cast<float>(scale);
    p.eps = static_cast<float>(eps);
    p.p_scale = static_cast<float>(p_scale);
    p.q_descale = static_cast<float>(q_descale);
    p.k_descale = static_cast<float>(k_descale);
    p.v_descale = static_cast<float>(v_descale);
    p.bad_key = reinterpret_cast<uint64_t*>(bad.data_ptr());
    p.tile_m_hint = static_cast<int32_t>(tile_m);
    p.tile_n_hint = static_cast<int32_t>(tile_n);
    p.normalizer = static_cast<int32_t>(normalizer);
    auto stream = at::cuda::getCurrentCUDAStream(dev.index());
    at::Tensor ks, k_scaled;  // (kept alive until the launch is queued)
    if (key_scale.has_value()) {
      ks = key_scale->dim() == 2 ? *key_scale : key_scale->reshape({1, -1});
      if (!ks.is_cuda() || ks.scalar_type() != at::kFloat || ks.device() != dev || ks.size(0) != b ||
          ks.size(1) != nkv || (nkv > 0 && ks.stride(1) != 1))
        throw Fail{FS_ERR_SHAPE, "flashsign: key_scale must be float32 [B, Nkv] on q's device with unit key stride"};
      const bool aligned = (reinterpret_cast<uintptr_t>(ks.data_ptr()) % 16) == 0 &&
                           (b == 1 || ((ks.stride(0) * 4) % 16 == 0 && ks.stride(0) >= nkv));
      if (!aligned) {  // TMA needs 16-byte rows: aligned copy on this (the launch) stream
        at::Tensor buf = at::zeros({b, std::max<int64_t>(4, (nkv + 3) / 4 * 4)}, ks.options());
        buf.narrow(1, 0, nkv).copy_(ks);
        ks = buf.narrow(1, 0, nkv);
      }
      p.key_scale = ks.data_ptr<float>();
      p.key_scale_stride = ks.stride(0);
      if ((ic == FS_F16 || ic == FS_BF16) && d % 8 == 0 && nkv > 0) {
        // 16-bit inputs: K' = m K in one HBM pass (fs_scale_keys), then the plain kernel -- cheaper
        // than the in-kernel per-score multiply (include/flashsign.h)
        at::Tensor kp = at::empty({b, nkv, hkv, d}, k.options());
        const int64_t kst[3] = {kp.stride(0), kp.stride(1), kp.stride(2)};
        const fs_status s2 = fs_scale_keys(&p, kp.data_ptr(), kst, reinterpret_cast<fs_stream_t>(stream.stream()));
        if (s2 != FS_OK) throw Fail{static_cast<int>(s2), std::string(fs_last_error())};
        p.k = kp.data_ptr();
        for (int i = 0; i < 3; ++i) p.k_stride[i] = kst[i];
        p.key_scale = nullptr;
        p.key_scale_stride = 0;
        k_scaled = kp;
      }
    }
    // kv_splits < 0: the library's wave model picks the split (FS_SPLITS_AUTO, tail-only or uniform)
    p.kv_splits = static_cast<int32_t>(kv_splits >= 0 ? kv_splits : FS_SPLITS_AUTO);
    p.split_tail = split_tail ? 1 : 0;
    p.partial_only = partial_only ? 1 : 0;
    if (dev_scales.has_value()) {
      const at::Tensor& ds = *dev_scales;
      if (!ds.is_cuda() || ds.scalar_type() != at::kFloat || ds.numel() < 4 || !ds.is_contiguous() || ds.device() != dev)
        throw Fail{FS_ERR_SHAPE, "flashsign: dev_scales must be a contiguous float32 CUDA tensor of 4 elements"};
      p.dev_scales = ds.data_ptr<float>();
    }
    at::Tensor part;
    int32_t n_parts = fs_kv_splits(&p);
    if (partial_only || n_parts > 1) {
      const int64_t need = fs_partial_floats(&p);
      if (partial.has_value()) {
        part = *partial;
        if (part.scalar_type() != at::kFloat || part.numel() < need || !part.is_contiguous() || part.device() != dev)
          throw Fail{FS_ERR_SHAPE, "flashsign: partial workspace needs " + std::to_string(need) +
                                       " contiguous float32 elements"};
      } else {
        part = at::empty({need}, q.options().dtype(at::kFloat));
      }
      p.partial = part.data_ptr<float>();
    }
    const fs_status st = fs_fwd(&p, reinterpret_cast<fs_stream_t>(stream.stream()));
    if (st != FS_OK) return py::make_tuple(static_cast<int>(st), std::string(fs_last_error()), py::none(),
                                           py::none(), py::none(), 0);
    return py::make_tuple(0, std::string(), o, bad, part.defined() ? py::cast(part) : py::none(), n_parts);
  } catch (const Fail& f) {
    return py::make_tuple(f.status, f.msg, py::none(), py::none(), py::none(), 0);
  }
}

int src_code(at::ScalarType t) {
  switch (t) {
    case at::kHalf: return FS_F16;
    case at::kFloat: return FS_F32;
    case at::kDouble: return FS_F64;
    default: return -1;
  }
}

// The numpy drop-in's small-call path (hostpath._run_small: multi_head_attention_array,
// attention.py:318-361, on a few MB of host arrays) in one call, so that per-call host time is
// the copies and launches, not Python: Q|K|V (the caller's C-contiguous numpy buffers, [n, h, d] /
// [x, h_kv, d], one dtype, passed as addresses) packed into the pinned `host_in`, one H2D copy into `dev_in`,
// fs_prepare of all three (device-chosen scales into `scales`), fs_fwd with dev_scales (automatic
// split, as flashsign.fwd_async), the result converted to `host_out_t` on the device and read back
// into a fresh pinned tensor with the bad-row key, one stream synchronisation.
// Returns (status, message, host_out [n, h, d_pad], bad_key).
py::tuple small_call(int64_t q_ptr, int64_t k_ptr, int64_t v_ptr, at::ScalarType src_t, int64_t n, int64_t h,
                     int64_t x, int64_t hkv, int64_t d, const at::Tensor& host_in, const at::Tensor& dev_in,
                     const at::Tensor& stats, const at::Tensor& scales, const at::Tensor& bad_host,
                     at::ScalarType compute, int64_t d_pad, at::ScalarType kout, at::ScalarType host_out_t,
                     double scale, double eps, int64_t normalizer, bool exact) {
  try {
    const int sc = src_code(src_t);
    const int cc = in_code(compute);
    const int oc = out_code(kout);
    if (sc < 0 || cc < 0 || oc < 0) throw Fail{FS_ERR_SHAPE, "flashsign: small_call dtypes"};
    if (n < 1 || h < 1 || x < 1 || hkv < 1 || d < 1 || d_pad < d || !q_ptr || !k_ptr || !v_ptr)
      throw Fail{FS_ERR_SHAPE, "flashsign: small_call shapes"};
    const int64_t isz = c10::elementSize(src_t);
    auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
    const int64_t nb[3] = {n * h * d * isz, x * hkv * d * isz, x * hkv * d * isz};
    const int64_t off[3] = {0, al(nb[0]), al(nb[0]) + al(nb[1])};
    const int64_t tot = off[2] + nb[2];
    if (!host_in.is_pinned() || host_in.numel() < tot || !dev_in.is_cuda() || dev_in.numel() < tot)
      throw Fail{FS_ERR_SHAPE, "flashsign: small_call staging buffers too small"};
    const c10::cuda::CUDAGuard guard(dev_in.device());
    const auto dopt = dev_in.options();
    auto stream = at::cuda::getCurrentCUDAStream(dev_in.device().index());
    const auto cst = stream.stream();
    auto* hb = static_cast<uint8_t*>(host_in.data_ptr());
    const int64_t src[3] = {q_ptr, k_ptr, v_ptr};  // the caller's C-contiguous numpy buffers
    for (int i = 0; i < 3; ++i) {  // streaming stores past a few hundred KB (no read-for-ownership)
      if (nb[i] >= (256 << 10))
        fs_host_copy(hb + off[i], reinterpret_cast<const void*>(src[i]), static_cast<size_t>(nb[i]));
      else
        std::memcpy(hb + off[i], reinterpret_cast<const void*>(src[i]), nb[i]);
    }
    auto* db = static_cast<uint8_t*>(dev_in.data_ptr());
    cudaError_t ce = cudaMemcpyAsync(db, hb, tot, cudaMemcpyHostToDevice, cst);
    if (ce != cudaSuccess) throw Fail{FS_ERR_CUDA, cudaGetErrorString(ce)};

    at::Tensor qq = at::empty({1, n, h, d_pad}, dopt.dtype(compute));
    at::Tensor kq = at::empty({1, x, hkv, d_pad}, dopt.dtype(compute));
    at::Tensor vq = at::empty({1, x, hkv, d_pad}, dopt.dtype(compute));
    fs_prep_params pp;
    std::memset(&pp, 0, sizeof(pp));
    const at::Tensor* dst[3] = {&qq, &kq, &vq};
    const int64_t rows[3] = {n * h, x * hkv, x * hkv};
    for (int i = 0; i < 3; ++i) {
      pp.t[i].src = db + off[i];
      pp.t[i].src_dtype = sc;
      pp.t[i].d = static_cast<int32_t>(d);
      pp.t[i].rows = rows[i];
      pp.t[i].src_row_stride = d;
      pp.t[i].dst = dst[i]->data_ptr();
      pp.t[i].dst_row_stride = d_pad;
    }
    pp.dst_dtype = cc;
    pp.d_pad = static_cast<int32_t>(d_pad);
    pp.mode = exact ? FS_PREP_EXACT : FS_PREP_SCALE;
    pp.normalizer = static_cast<int32_t>(normalizer);
    pp.scale = static_cast<float>(scale);
    pp.eps = static_cast<float>(eps);
    pp.stats = stats.data_ptr<double>();
    pp.scales = scales.data_ptr<float>();
    fs_status st = fs_prepare(&pp, reinterpret_cast<fs_stream_t>(cst));
    if (st != FS_OK) throw Fail{static_cast<int>(st), std::string(fs_last_error())};

    at::Tensor o = at::empty({1, n, h, d_pad}, dopt.dtype(kout));
    at::Tensor bad = at::empty({1}, dopt.dtype(at::kLong));
    fs_fwd_params p;
    std::memset(&p, 0, sizeof(p));
    p.q = qq.data_ptr();
    p.k = kq.data_ptr();
    p.v = vq.data_ptr();
    p.o = o.data_ptr();
    for (int i = 0; i < 3; ++i) {
      p.q_stride[i] = qq.stride(i);
      p.k_stride[i] = kq.stride(i);
      p.v_stride[i] = vq.stride(i);
      p.o_stride[i] = o.stride(i);
    }
    p.batch = 1;
    p.heads_q = static_cast<int32_t>(h);
    p.heads_kv = static_cast<int32_t>(hkv);
    p.seqlen_q = static_cast<int32_t>(n);
    p.seqlen_kv = static_cast<int32_t>(x);
    p.head_dim = static_cast<int32_t>(d_pad);
    p.in_dtype = static_cast<fs_dtype>(cc);
    p.out_dtype = static_cast<fs_dtype>(oc);
    p.scale = static_cast<float>(scale);
    p.eps = static_cast<float>(eps);
    p.p_scale = p.q_descale = p.k_descale = p.v_descale = 1.f;
    p.bad_key = reinterpret_cast<uint64_t*>(bad.data_ptr());
    p.normalizer = static_cast<int32_t>(normalizer);
    p.kv_splits = FS_SPLITS_AUTO;
    p.dev_scales = scales.data_ptr<float>();
    at::Tensor part;
    if (fs_kv_splits(&p) > 1) {
      part = at::empty({fs_partial_floats(&p)}, dopt.dtype(at::kFloat));
      p.partial = part.data_ptr<float>();
    }
    st = fs_fwd(&p, reinterpret_cast<fs_stream_t>(cst));
    if (st != FS_OK) throw Fail{static_cast<int>(st), std::string(fs_last_error())};
    at::Tensor res = o[0];
    if (host_out_t != kout) res = res.to(host_out_t);
    at::Tensor host_out = at::empty({n, h, d_pad}, at::TensorOptions().dtype(host_out_t).pinned_memory(true));
    ce = cudaMemcpyAsync(host_out.data_ptr(), res.data_ptr(), host_out.nbytes(), cudaMemcpyDeviceToHost, cst);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(bad_host.data_ptr(), bad.data_ptr(), 8, cudaMemcpyDeviceToHost, cst);
    if (ce != cudaSuccess) throw Fail{FS_ERR_CUDA, cudaGetErrorString(ce)};
    {
      py::gil_scoped_release nogil;
      ce = cudaStreamSynchronize(cst);
    }
    if (ce != cudaSuccess) throw Fail{FS_ERR_CUDA, cudaGetErrorString(ce)};
    return py::make_tuple(0, std::string(), host_out, *static_cast<int64_t*>(bad_host.data_ptr()));
  } catch (const Fail& f) {
    return py::make_tuple(f.status, f.msg, py::none(), 0);
  }
}

}  // namespace

PYBIND11_MODULE(TORCH_EXTENSION_NAME, m) {
  m.def("small_call", &small_call, "the numpy drop-in's small-call path (hostpath._run_small) in one call");
  m.doc() = "FlashSign torch binding over the C-ABI (include/flashsign.h)";
  m.def("fwd", &fwd, "FlashSign forward on BSHD CUDA tensors (current stream)", py::arg("q"), py::arg("k"),
        py::arg("v"), py::arg("out"), py::arg("out_dtype"), py::arg("bad_key"), py::arg("scale"), py::arg("eps"),
        py::arg("p_scale"), py::arg("q_descale"), py::arg("k_descale"), py::arg("v_descale"),
        py::arg("normalizer"), py::arg("key_scale"), py::arg("kv_splits"), py::arg("partial"),
        py::arg("partial_only"), py::arg("dev_scales"), py::arg("tile_m"), py::arg("tile_n"),
        py::arg("split_tail"));
  m.def("version", []() { return fs_version(); });
}
