// fs_host.cpp -- host-side copy for the drop-in path's pinned staging ring (hostpath.py).
//
// The numpy callers of the reference API (attention.py:252-279, 318-361) hand over pageable
// arrays; the drop-in copies them into pinned slots that the DMA engine then reads.  With plain
// memcpy each staged byte costs four bytes of host-memory traffic (read, read-for-ownership of
// the destination line, write, DMA read) while the DMA engine competes for the same memory; the
// copy here writes with non-temporal stores (no read-for-ownership, no cache pollution), three
// bytes per staged byte.  Called from the staging threads through ctypes (the GIL is released).

#include <immintrin.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstring>

namespace {

__attribute__((target("avx512f"))) void copy_nt512(uint8_t* d, const uint8_t* s, size_t n) {
  size_t i = 0;
  for (; i + 256 <= n; i += 256) {
    const __m512i a = _mm512_loadu_si512(s + i);
    const __m512i b = _mm512_loadu_si512(s + i + 64);
    const __m512i c = _mm512_loadu_si512(s + i + 128);
    const __m512i e = _mm512_loadu_si512(s + i + 192);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i), a);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i + 64), b);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i + 128), c);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i + 192), e);
  }
  for (; i + 64 <= n; i += 64) _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i), _mm512_loadu_si512(s + i));
  if (i < n) std::memcpy(d + i, s + i, n - i);
  _mm_sfence();
}

__attribute__((target("avx2"))) void copy_nt256(uint8_t* d, const uint8_t* s, size_t n) {
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
    const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
  }
  if (i < n) std::memcpy(d + i, s + i, n - i);
  _mm_sfence();
}

}  // namespace

extern "C" {

// Copy `bytes` from `src` to `dst` with non-temporal stores.  `dst` is aligned up to 64 bytes by a
// short memcpy head; any `src` alignment.  Returns 512 / 256 (vector width used) or 0 (memcpy).
int fs_host_copy(void* dst, const void* src, size_t bytes) {
  auto* d = static_cast<uint8_t*>(dst);
  const auto* s = static_cast<const uint8_t*>(src);
  const size_t head = std::min<size_t>(bytes, (64 - (reinterpret_cast<uintptr_t>(d) & 63)) & 63);
  if (head) std::memcpy(d, s, head);
  d += head;
  s += head;
  bytes -= head;
  if (__builtin_cpu_supports("avx512f")) {
    copy_nt512(d, s, bytes);
    return 512;
  }
  if (__builtin_cpu_supports("avx2")) {
    copy_nt256(d, s, bytes);
    return 256;
  }
  std::memcpy(d, s, bytes);
  return 0;
}

}  // extern "C"
