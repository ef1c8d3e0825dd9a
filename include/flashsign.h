/*
 * flashsign.h -- C-ABI of the B200-native FlashSign (spherical attention) forward.
 *
 * This is the drop-in boundary for the reference hot path.  The reference
 * (arxiv 2505.09326, package `ncstream`, pure Python) has no FFI of its own;
 * each entry point below replaces one reference interface:
 *
 *   fs_fwd          <- ncstream.attention.streamed_attention_array
 *                      (pkg/src/ncstream/attention.py:252-279) and its batched
 *                      caller multi_head_attention_array (attention.py:318-361):
 *                      one launch covers every (batch, head, query tile); query
 *                      head h reads kv head (h*heads_kv)/heads_q (attention.py:352).
 *                      Errors mirror ShapeMismatchError (tensor.py:32-33,
 *                      attention.py:104-111, 339-344), ConfigError
 *                      (attention.py:36-37, 54-56, 77-80, 337-338) and
 *                      DegenerateDenominatorError (normalizers.py:29-35,
 *                      attention.py:196-199) -- the latter reported on the device
 *                      through `bad_key` (below) because the launch is async.
 *   fs_query_tile   <- the transient score tile recorded by ScoreBufferMeter
 *                      (attention.py:86-97, 169-171).
 *   fs_last_error   <- the exception message text.
 *
 * Math (eps = denom_epsilon, normalizers.py:69; m_j = optional key multiplicity,
 * attention.py:381-388 / grn.py:150, 1 when key_scale is NULL):
 *     s_ij = scale * q_descale * k_descale * m_j * (q_i . k_j)
 *     SPHERICAL (normalizers.py:94-100):  O_i = v_descale * sum_j s_ij v_j / sqrt(sum_j s_ij^2 + eps)
 *     SIGNED_L1 (normalizers.py:111-117): O_i = v_descale * sum_j s_ij v_j / (sum_j |s_ij| + eps)
 *
 * No torch types cross this boundary: plain device pointers, element strides,
 * sizes and a cudaStream_t.  All calls are asynchronous on `stream`.
 */
#ifndef FLASHSIGN_H
#define FLASHSIGN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *fs_stream_t; /* == cudaStream_t */

typedef enum {
  FS_OK = 0,
  FS_ERR_SHAPE = 1,       /* -> ShapeMismatchError  */
  FS_ERR_CONFIG = 2,      /* -> ConfigError         */
  FS_ERR_DTYPE = 3,       /* -> ShapeMismatchError (dtype) */
  FS_ERR_UNSUPPORTED = 4, /* -> ConfigError (outside the kernel envelope) */
  FS_ERR_CUDA = 5         /* -> RuntimeError        */
} fs_status;

typedef enum {
  FS_F16 = 0,
  FS_BF16 = 1,
  FS_E4M3 = 2,
  FS_F32 = 3, /* output (fs_fwd) / source (fs_prepare) */
  FS_F64 = 4  /* source only (fs_prepare) */
} fs_dtype;

typedef enum {
  FS_NORM_SPHERICAL = 0, /* a1(u) = u, a2(u) = u^2, b = sqrt  (normalizers.py:94-100)  */
  FS_NORM_SIGNED_L1 = 1  /* a1(u) = u, a2(u) = |u|, b = id    (normalizers.py:111-117) */
} fs_normalizer;

/* Sentinel value of *bad_key when no row was degenerate. */
#define FS_BAD_NONE 0xFFFFFFFFFFFFFFFFull

typedef struct {
  /* Device pointers (caller-owned).  Layout BSHD: element (b, n, h, d) lives at
     ptr[b*stride[0] + n*stride[1] + h*stride[2] + d]; the d stride is 1. */
  const void *q, *k, *v;
  void *o;
  int64_t q_stride[3], k_stride[3], v_stride[3], o_stride[3];
  int32_t batch, heads_q, heads_kv, seqlen_q, seqlen_kv, head_dim;
  fs_dtype in_dtype;  /* FS_F16 | FS_BF16 | FS_E4M3 (q, k, v share it)        */
  fs_dtype out_dtype; /* FS_F16 | FS_BF16 | FS_F32                              */
  float scale;        /* score_scale c: finite, may be negative (0: all rows degenerate unless eps>0) */
  float eps;          /* denom_epsilon >= 0                                    */
  float p_scale;      /* P = p_scale * s before the PV MMA (FP8: fit e4m3); 1.0 */
  float q_descale, k_descale, v_descale; /* per-tensor dequant (FP8); 1.0      */
  /* Optional device scalar (may be NULL).  fs_fwd resets it to FS_BAD_NONE on
     `stream`, then the kernel atomically keeps the minimum of
       (linear_row << 32) | float_bits(z),  linear_row = (b*heads_q + h)*seqlen_q + n
     over rows whose denominator b(z + eps) is 0 or non-finite, i.e. the
     first bad row in the reference's loop order (batch, head, row) and its z
     = sum_j a2(s_ij).  A P that does not fit the MMA dtype is reported as z = +inf
     (and the row's O is zeroed): FP16 P overflowing to inf (|p_scale s| >= 65520), FP8 P
     saturating the e4m3 range (|p_scale s| >= 432, i.e. rounded to +-448). */
  uint64_t *bad_key;
  int32_t tile_m_hint, tile_n_hint; /* TileConfig (g_y, s_x); advisory only    */
  int32_t normalizer;               /* fs_normalizer; 0 = SPHERICAL            */
  /* Split K/V stream (streaming.py:122-128 merge; Lemma 1): 0 or 1 = one pass.
     S > 1 cuts every (b, h) K/V stream into S contiguous ranges computed by independent work
     tiles (for small B*H with long N); partial numerators and z go to `partial` and fs_fwd then
     runs the combine kernel (O = sum_s num_s / b(sum_s z_s + eps)) on the same stream.
     fs_kv_splits(p) returns the effective S (clamped so that every range is non-empty).
     FS_SPLITS_AUTO (-1): the library picks S and split_tail from its wave model of the persistent
     grid on the current device (fs_plan); size `partial` with fs_partial_floats(p). */
  int32_t kv_splits;
  /* Optional per-key multiplicity m (NULL: none): fp32 device array [batch, seqlen_kv],
     element (b, n) at key_scale[b*key_scale_stride + n], shared by all kv heads -- the
     reference's apply_multiplicity_array(K, m) (attention.py:381-388) fused into the
     score.  m must be finite and >= 0 (the caller validates; the reference raises
     ValueError).  16-byte aligned; key_scale_stride*4 a multiple of 16 when batch > 1. */
  const float *key_scale;
  int64_t key_scale_stride;
  /* fp32 workspace of fs_partial_floats(p) floats, 16-byte aligned (needed when the effective
     kv_splits > 1 or partial_only): numerators [S][B][H][Nq][Dk] then z [S][B][H][Nq],
     Dk = 128 for e4m3 or head_dim > 64, else 64.  Caller-owned; fs_fwd never allocates. */
  float *partial;
  /* 1: stop after writing the partials (no O, no bad-row key).  Context parallelism: every rank
     runs its K/V shard with partial_only = 1, the ranks all-reduce(sum) `partial`, then each
     calls fs_combine(p, 1, stream) to normalise. */
  int32_t partial_only;
  /* 0: every work tile is split into kv_splits K/V ranges (uniform).  1: only the work tiles of
     the persistent grid's last, partial wave are split (tiles = W*G + T over G co-resident
     clusters of 2 CTAs, each 512 query rows of one (b, h); the T tail tiles become T*S items), so
     the last wave keeps every SM busy; `partial` then holds S*T*512 rows.  Ignored with
     partial_only.  (Was reserved1, required 0.) */
  int32_t split_tail;
  /* Optional device array of 4 floats {q_descale, k_descale, v_descale, p_scale} (NULL: the host
     fields above).  Read by the kernel at launch time, so per-tensor scales chosen on the device
     (fs_prepare, below) need no host round trip.  Same constraints as the host fields. */
  const float *dev_scales;
} fs_fwd_params;

#define FS_SPLITS_AUTO (-1)

/* Validate, encode TMA descriptors (cached per call), launch.  Async. */
fs_status fs_fwd(const fs_fwd_params *p, fs_stream_t stream);

/* Effective number of K/V ranges for p (>= 1) and the partial workspace size in floats. */
int32_t fs_kv_splits(const fs_fwd_params *p);
int64_t fs_partial_floats(const fs_fwd_params *p);

/* The split plan fs_fwd would use for p (host only when clusters > 0: plan for that many
   co-resident 2-CTA clusters, e.g. 74 on a 148-SM B200; 0 = query the current device), and the
   wave model's result: items are walked by the clusters with a static stride (item i on cluster
   i % G), busiest_steps = K/V-tile steps on the most loaded cluster, efficiency = all steps /
   (G * busiest_steps). */
typedef struct {
  int32_t splits, split_tail, clusters, n_whole, tail_tiles, n_kv_tiles;
  int64_t work_tiles, items, partial_floats;
  double busiest_steps, efficiency;
} fs_plan_info;
fs_status fs_plan(const fs_fwd_params *p, int32_t clusters, fs_plan_info *out);

/* O = sum_s num_s / b(sum_s z_s + eps) over the first n_parts partials in p->partial, written to
   p->o with p->o_stride / out_dtype, and the bad-row key (reset first) -- the merge step of the
   split / context-parallel path.  Async on `stream`. */
fs_status fs_combine(const fs_fwd_params *p, int32_t n_parts, fs_stream_t stream);

/* Context parallelism over peer memory (NVLink P2P / CUDA IPC) instead of an all-reduce
   (streaming.py:122-128 merge; Lemma 1).  `world` ranks hold disjoint K/V
   shards of the same (b, h) streams and all of Q; query positions are owned in ranges of
   rows_per_rank (owner of position n = n / rows_per_rank).  fs_fwd_peer runs this rank's K/V
   shard and its epilogue stores every row's partial (numerator, z) straight into the OWNER's
   workspace, slot `rank`: workspace = numerators [world][B][H][rows_per_rank][Dk] then
   z [world][B][H][rows_per_rank] (fs_peer_floats floats; Dk as for `partial`).  Once every
   rank's fs_fwd_peer has completed (the caller synchronises its stream and barriers),
   fs_combine_peer normalises this rank's positions [rank*R, rank*R + R) into p->o and sets the
   bad-row key.  No collective library call on the data path. */
typedef struct fs_peer_params {
  int32_t world;              /* ranks */
  int32_t rank;               /* this rank: its slot in every owner's workspace */
  int32_t rows_per_rank;      /* query positions owned per rank; world * R >= seqlen_q */
  int32_t reserved0;          /* must be 0 */
  float *const *peer_partial; /* device array [world] of the ranks' workspaces (peer-mapped) */
  float *local_partial;       /* this rank's workspace (== peer_partial[rank] on the device) */
} fs_peer_params;

int64_t fs_peer_floats(const fs_fwd_params *p, const fs_peer_params *peer);
fs_status fs_fwd_peer(const fs_fwd_params *p, const fs_peer_params *peer, fs_stream_t stream);
fs_status fs_combine_peer(const fs_fwd_params *p, const fs_peer_params *peer, fs_stream_t stream);

/* Peer workspaces: cudaMalloc + cudaIpcGetMemHandle (64-byte handle out), open / close a peer's
   handle (lazy peer access), free. */
fs_status fs_ipc_malloc(int64_t bytes, void **ptr, void *handle64);
fs_status fs_ipc_open(const void *handle64, void **ptr);
fs_status fs_ipc_close(void *ptr);
fs_status fs_ipc_free(void *ptr);

/* Operand preparation for host-array callers (the drop-in path; attention.py:252-279 accepts any
   float32 / float64 array and computes in float64).  Converts up to three caller tensors -- rows of
   d elements, row-major, on the device -- to the kernel's input dtype, each with one power-of-two
   scale chosen ON THE DEVICE: amax|x 2^e| in [2^(T-1), 2^T) (T = 14 for FS_F16 / FS_BF16, 8 for
   FS_E4M3), plus a power-of-two p_scale from the Cauchy-Schwarz bound max||q'|| max||k'|| so
   that the PV operand P = p s can never overflow (fp16 / e4m3) for any finite input.  Spherical and
   signed-L1 outputs are invariant to these factors; fs_fwd folds them out exactly when given
   `scales` as fs_fwd_params.dev_scales.  FS_PREP_EXACT keeps the values (no operand scaling; the
   f16 emulation's binary16-rounded inputs, tensor.py:132-139, attention.py:265-270) and still
   chooses p_scale.  A tensor with src == NULL is not converted and its stats from an earlier call
   (same `stats` workspace) are reused: the K / V of a query stream processed in chunks.
   One memset + two kernels, async on `stream`. */
typedef enum { FS_PREP_SCALE = 0, FS_PREP_EXACT = 1 } fs_prep_mode;

typedef struct {
  const void *src;        /* device, [rows, d] with src_row_stride; NULL = reuse this slot's stats  */
  int32_t src_dtype;      /* FS_F32 | FS_F64 | FS_F16 | FS_BF16                                      */
  int32_t d;              /* valid columns, 1 <= d <= d_pad                                           */
  int64_t rows;           /* rows (token x head) of d elements                                       */
  int64_t src_row_stride; /* elements, >= d                                                          */
  void *dst;              /* device, [rows, d_pad] in dst_dtype, columns >= d zero-filled            */
  int64_t dst_row_stride; /* elements, >= d_pad                                                      */
} fs_prep_tensor;

typedef struct {
  fs_prep_tensor t[3];  /* q, k, v */
  int32_t dst_dtype;    /* FS_F16 | FS_BF16 | FS_E4M3                                        */
  int32_t d_pad;        /* columns written per operand row                                   */
  int32_t mode;         /* fs_prep_mode                                                      */
  int32_t normalizer;   /* fs_normalizer of the call (bounds eps / g)                        */
  float scale, eps;     /* the call's score scale c and denom_epsilon                        */
  double *stats;        /* device workspace, 6 doubles: {amax, max row L2 norm} of q, k, v   */
  float *scales;        /* device out, 4 floats -> fs_fwd_params.dev_scales                  */
} fs_prep_params;

fs_status fs_prepare(const fs_prep_params *p, fs_stream_t stream);

/* K' = m K for 16-bit inputs: k_out[b, n, h, :] = RNE(key_scale[b*key_scale_stride + n] * k[b, n, h, :])
   (fp32 product: exact for integer m), the reference's apply_multiplicity_array (attention.py:381-388,
   grn.py:150) as one HBM-bound pass.  Uses p->k, k_stride, batch, seqlen_kv, heads_kv, head_dim (a
   multiple of 8), in_dtype (FS_F16 | FS_BF16), key_scale, key_scale_stride; k_out strides in
   elements, 16-byte multiples.  Then fs_fwd with k = k_out and key_scale = NULL computes the
   multiplicity attention with the tensor cores' operand traffic unchanged: for 16-bit inputs this
   is cheaper than fs_fwd's in-kernel key_scale (one extra multiply per score on the norm step's
   critical path, measured -20 % at d = 64; scaling the K slot in shared memory instead exceeds the
   SM's shared-memory bandwidth, FS_KS_SMEM).  Async on `stream`. */
fs_status fs_scale_keys(const fs_fwd_params *p, void *k_out, const int64_t *k_out_stride, fs_stream_t stream);

/* The Gram (moment) form of the spherical contract (the identity behind
   attention.py:146-200 for a2(u) = u^2): with G = sum_j k_j k_j^T and W = sum_j k_j v_j^T per (b, h_kv),
       O_i = c q_i^T W / sqrt(c^2 q_i^T G q_i + eps)
   -- the same function at 8 N d^2 instead of 4 N^2 d flops, HBM-bound.  Three tensor-core launches
   (moments per key chunk; reduce into 16-bit hi + lo B-operand images; apply per 128-row query tile).
   Same fs_fwd_params as fs_fwd (q, k, v, o, strides, extents, scale, eps, bad_key with fs_fwd's
   first-bad-row key); FS_F16 / FS_BF16 inputs, head_dim a multiple of 8 (<= 128), the spherical
   normaliser only, no key_scale (form K' first with fs_scale_keys), no splits / partials /
   dev_scales.  `workspace`: device memory of fs_gram_workspace_bytes(p) bytes, 256-byte aligned.
   Async on `stream`. */
int64_t fs_gram_workspace_bytes(const fs_fwd_params *p);
fs_status fs_gram_fwd(const fs_fwd_params *p, void *workspace, int64_t workspace_bytes, fs_stream_t stream);

/* Float64 streamed FlashSign for float32 / float64 callers of the drop-in API: the reference's
   own loop (attention.py:146-200) with its rounding points -- float64 scores, or for a float32
   grid (f32_grid = 1) scores rounded to float32 and scaled in float32 (attention.py:163-166) and
   float32 squares summed in float64 (attention.py:188) -- on the SM's FP64 units, keys
   accumulated in order for every row.  Reaches the reference's float64 tolerances (the tensor-core
   fs_fwd cannot); a precision mode, not the hot path.  Layout as fs_fwd (BSHD, element strides,
   head_dim <= 128); output float64; optional per-row z (float64, [B][H][Nq]) for the exception
   text; bad_key as in fs_fwd.  Async on `stream`. */
typedef struct {
  const double *q, *k, *v;
  double *o;
  int64_t q_stride[3], k_stride[3], v_stride[3], o_stride[3];
  int32_t batch, heads_q, heads_kv, seqlen_q, seqlen_kv, head_dim;
  double scale, eps;   /* score scale c (finite), denom_epsilon >= 0 */
  int32_t normalizer;  /* fs_normalizer */
  int32_t f32_grid;    /* 1: the caller's arrays are float32 (the reference's float32 rounding points) */
  uint64_t *bad_key;   /* optional device scalar, as fs_fwd */
  double *z_out;       /* optional device [B*H*Nq]: each row's z */
} fs_exact_params;

fs_status fs_exact_fwd(const fs_exact_params *p, fs_stream_t stream);

/* ------------------------------------------------------------------ host staging copy
   Host memory to host memory with non-temporal stores: the drop-in path's fill of its pinned
   staging slots from the caller's pageable numpy arrays (hostpath.py; the reference's callers
   pass numpy arrays, attention.py:252-279, 318-361).  No device work.  Returns the vector width
   used (512, 256) or 0 (plain memcpy). */
int fs_host_copy(void *dst, const void *src, size_t bytes);

/* Thread-local text of the last non-FS_OK status. */
const char *fs_last_error(void);

/* Score tile (query rows x keys) held on chip per Q tile for (head_dim, dtype):
   what ScoreBufferMeter records.  Returns 0 on success. */
int fs_query_tile(int head_dim, fs_dtype dt, int *bm, int *bn);

/* Library version (major*10000 + minor*100 + patch). */
int fs_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FLASHSIGN_H */
