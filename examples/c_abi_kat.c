/* Standalone C caller of the FlashSign C-ABI (no Python, no torch): the reference's
 * known-answer test (tests/test_attention.py:46-52: q = [1], K = [[3], [4]], V = [[10], [20]]
 * -> O = (3*10 + 4*20) / sqrt(3^2 + 4^2) = 22) on the GPU, head dim padded to 8 with zeros.
 *   gcc -std=c99 c_abi_kat.c -I../include -I$CUDA/include -L../paper_2505_09326_b200/_lib \
 *       -lflashsign -L$CUDA/lib64 -lcudart -o kat && ./kat                                   */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "flashsign.h"

static uint16_t f16(float x) { /* exact for the small integers used here */
  uint32_t b;
  memcpy(&b, &x, 4);
  if (x == 0.0f) return 0;
  int e = (int)((b >> 23) & 0xff) - 127 + 15;
  return (uint16_t)(((b >> 16) & 0x8000) | (e << 10) | ((b >> 13) & 0x3ff));
}

int main(void) {
  enum { D = 8 };
  uint16_t q[D] = {0}, k[2 * D] = {0}, v[2 * D] = {0};
  q[0] = f16(1.0f);
  k[0] = f16(3.0f);
  k[D] = f16(4.0f);
  v[0] = f16(10.0f);
  v[D] = f16(20.0f);
  void *dq, *dk, *dv, *dout;
  uint64_t *dbad, bad = 0;
  float out[D];
  if (cudaMalloc(&dq, sizeof q) || cudaMalloc(&dk, sizeof k) || cudaMalloc(&dv, sizeof v) ||
      cudaMalloc(&dout, sizeof out) || cudaMalloc((void **)&dbad, 8))
    return 2;
  cudaMemcpy(dq, q, sizeof q, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, k, sizeof k, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, v, sizeof v, cudaMemcpyHostToDevice);

  fs_fwd_params p;
  memset(&p, 0, sizeof p);
  p.q = dq; p.k = dk; p.v = dv; p.o = dout;
  /* BSHD strides in elements (batch, token, head): one head, d contiguous */
  p.q_stride[0] = D; p.q_stride[1] = D; p.q_stride[2] = D;
  p.k_stride[0] = 2 * D; p.k_stride[1] = D; p.k_stride[2] = D;
  p.v_stride[0] = 2 * D; p.v_stride[1] = D; p.v_stride[2] = D;
  p.o_stride[0] = D; p.o_stride[1] = D; p.o_stride[2] = D;
  p.batch = 1; p.heads_q = 1; p.heads_kv = 1; p.seqlen_q = 1; p.seqlen_kv = 2; p.head_dim = D;
  p.in_dtype = FS_F16; p.out_dtype = FS_F32;
  p.scale = 1.0f; p.eps = 0.0f;
  p.p_scale = p.q_descale = p.k_descale = p.v_descale = 1.0f;
  p.bad_key = dbad;
  p.normalizer = FS_NORM_SPHERICAL;
  if (fs_fwd(&p, NULL) != FS_OK) {
    fprintf(stderr, "fs_fwd: %s\n", fs_last_error());
    return 1;
  }
  cudaMemcpy(out, dout, sizeof out, cudaMemcpyDeviceToHost);
  cudaMemcpy(&bad, dbad, 8, cudaMemcpyDeviceToHost);
  printf("O[0] = %.6f, bad_key = %s\n", out[0], bad == FS_BAD_NONE ? "none" : "set");
  return (out[0] == 22.0f && bad == FS_BAD_NONE) ? 0 : 1;
}
