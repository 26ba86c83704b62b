/*
 * kvrot_b200.h -- C ABI of the B200-native Hadamard-INT4 KV hot path.
 *
 * One shared library (libkvrot_b200.so, sm_100a) exports these symbols.  All
 * buffers are DEVICE pointers unless a parameter says "host"; every entry
 * point is asynchronous on `stream` (a cudaStream_t passed as void*), never
 * allocates, never throws, and returns a kvr_status.  Global state: a
 * thread-local last-error string (kvr_last_error), per-device caches of kernel
 * attributes, and a mutex-protected note of which streams last wrote pool cells
 * (see kvr_note_pool_write).
 *
 * The entry points replace, one for one, the reference's operator boundary
 * `kvrot._kernels` (pkg/src/kvrot/_kernels/__init__.py:35-39) and the
 * serving-path callers above it:
 *
 *   kvr_fwht_rows_f64        <- _kernels.fwht_rows        (_ref.py:22-40, _core.pyx:22-47)
 *   kvr_pack_rows            <- _kernels.pack_rows        (_ref.py:43-45, _core.pyx:50-60)
 *   kvr_unpack_rows          <- _kernels.unpack_rows      (_ref.py:48-54, _core.pyx:63-73)
 *   kvr_quantize_rows_f64    <- _kernels.quantize_rows    (_ref.py:57-80, _core.pyx:76-130)
 *   kvr_dequantize_rows_f64  <- _kernels.dequantize_rows  (_ref.py:83-95, _core.pyx:133-158)
 *   kvr_block_rotate         <- rotation.apply_block_rotation / apply_inverse_rotation
 *                               (rotation.py:118-159), hadamard.fwht_blocks (hadamard.py:70-89)
 *   kvr_rotate_quantize_store<- cache.PageTable.append_token / append_tokens_two_pass
 *                               (cache.py:235-317) incl. _rotate_token (cache.py:453-462)
 *   kvr_dequantize_pages     <- cache.PageTable.read_token / read_sequence (cache.py:319-362)
 *   kvr_paged_decode         <- attention.decode_step (attention.py:50-87)
 *   kvr_decode_step          <- PageTable.append_token + decode_step fused: one serving
 *                               decode step (cache.py:235-270 then attention.py:50-87)
 *   kvr_decode_flat_f64      <- attention.decode_step_fp (attention.py:90-115), the flat
 *                               full-precision decode (paged-vs-flat exactness oracle)
 *   kvr_rows_matmul_f64      <- the learned factor's `out @ spec.learned` / `@ spec.learned.T`
 *                               (rotation.py:140-141, 154-155) and compose_transform's T
 *                               (rotation.py:171-184) applied to queries / outputs
 *   kvr_rotate_quantize_store_learned <- append with a learned spec (rotation.py:118-168 then
 *                               cache.py:235-270), R fused into the write kernel
 *   kvr_paged_decode_learned <- attention.decode_step on a learned spec (attention.py:50-87,
 *                               rotation.py:162-184), q T and the value branch's inverse fused
 */
#ifndef KVROT_B200_H
#define KVROT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVR_ABI_VERSION 2
#define KVR_MAX_HEAD_DIM 256

typedef enum {
  KVR_OK = 0,
  KVR_ERR_SHAPE = 1,        /* maps to kvrot.errors.ShapeError            */
  KVR_ERR_ORDER = 2,        /* maps to kvrot.errors.InvalidOrderError     */
  KVR_ERR_UNSUPPORTED = 3,  /* configuration not built into this library  */
  KVR_ERR_CUDA = 4,         /* CUDA runtime failure (see kvr_last_error)  */
  KVR_ERR_ARG = 5,          /* null pointer / negative size / bad enum    */
  KVR_ERR_NONFINITE = 6     /* a host input holds NaN/Inf (maps to NonFiniteInputError); nothing launched */
} kvr_status;

typedef enum { KVR_F64 = 0, KVR_F32 = 1, KVR_BF16 = 2, KVR_F16 = 3 } kvr_dtype;

/* rotation.Targets (rotation.py:32-36) */
typedef enum { KVR_KEYS_ONLY = 0, KVR_KEYS_AND_VALUES = 1 } kvr_targets;

/* Device-side status bits written by the write kernel (never cleared by it). */
#define KVR_FLAG_NONFINITE 1u   /* a K/V row held NaN/Inf -> NonFiniteInputError */
#define KVR_FLAG_LEN_OVERFLOW 2u /* a decode seq_lens[b] exceeded max_seq_len (tokens past it ignored) */

/*
 * The paged pool: `num_pages` page blobs of `page_bytes` each.  A page holds
 * P tokens x H kv heads; inside it, every head owns P / T "cells" of T tokens
 * (T = cell_tokens = 16 when P is a multiple of 16, else P), and a cell keeps
 * everything one decode tile of that head needs contiguous:
 *
 *     cell = k_scale f32[T] | v_scale f32[T] | k_codes u8[T][d/2] |
 *            v_codes u8[T][d/2] | k_zp u8[T] | v_zp u8[T]   (padded to 16 B)
 *     page = cell[h = 0][0 .. P/T) | cell[h = 1][...] | ...
 *
 * so a (page, head) tile is ONE bulk copy (2208 B at d = 128, T = 16).  This is
 * a B200-first re-layout of the reference KvPage (cache.py:103-114); the
 * `.kvpg` record order (cache.py:387-397) is produced on export (PageTable.dump).
 */
typedef struct {
  void* base;           /* device pointer, 16-byte aligned                 */
  int64_t num_pages;
  int32_t page_tokens;  /* P  */
  int32_t num_kv_heads; /* H  */
  int32_t head_dim;     /* d  */
  int32_t page_bytes;   /* H * (P / T) * cell_bytes                        */
  int32_t cell_tokens;  /* T                                                */
  int32_t cell_bytes;   /* INT4: roundup16(T * (d + 10)); BF16: 4 * T * d   */
  int32_t precision;    /* KVR_PREC_INT4 | KVR_PREC_BF16                    */
} kvr_pool;

/* Page precision (cache.py:36-37).  A BF16 pool (cache.py:115-118) stores the raw
 * K / V vectors as bf16 bits, rounded f32 -> bf16 to nearest even (cache.py:43-47);
 * its cell is  k_bits u16[T][d] | v_bits u16[T][d]  and it ignores rotations
 * (append_token, cache.py:243-246; decode_step uses the query as-is, attention.py:67-71). */
#define KVR_PREC_INT4 0
#define KVR_PREC_BF16 1

/* Fill a kvr_pool for (P, H, d); the page size is returned in pool->page_bytes. */
int kvr_pool_init(kvr_pool* pool, void* base, int64_t num_pages, int32_t page_tokens,
                  int32_t num_kv_heads, int32_t head_dim);

/* Same for a BF16 pool (precision KVR_PREC_BF16). */
int kvr_pool_init_bf16(kvr_pool* pool, void* base, int64_t num_pages, int32_t page_tokens,
                       int32_t num_kv_heads, int32_t head_dim);
const char* kvr_last_error(void);
/* Profiling aid: when non-NULL, decode launches record a per-CTA timeline into
 * `trace` (device buffer of (batch * splits * num_kv_heads + batch * num_q_heads)
 * * 16 u64): decode CTA rows first, [0] the globaltimer (ns) and [1] clock64 at
 * CTA entry, [k >= 2] clock64 at stamp k (2 loop start, 3 loop end, 4/5 CTA
 * merge, 6 partial stored / cluster barrier, 9 merged, 10 exit; 0 = not
 * reached); then one row per split-merge CTA (splits > 8): globaltimer at [0]
 * entry, [1] past the grid-dependency wait, [2] exit.  NULL disables. */
void kvr_debug_decode_trace(void* trace);
/* A/B aid: the kernel behind the fast bf16/fp16 path of kvr_rotate_quantize_store --
 * 0 the default (the tcgen05/TMEM kernel from ~4 tiles of 128 rows per SM on, the mma.sync
 * kernel below), 1 the mma.sync kernel at every size, 2 the tcgen05 kernel at every size.
 * Process-wide; call between launches, not concurrently with them. */
void kvr_debug_set_k1_impl(int32_t impl);
int kvr_abi_version(void);
/* The caller wrote pool bytes on `stream` outside this library (e.g. a checkpoint
 * load): the next decode launched on that stream issues no pool reads before its
 * grid-dependency wait. */
void kvr_note_pool_write(void* stream);
/* Host validation helper: 1 when the n values (dtype F64/F32/BF16/F16) at HOST
 * pointer p are all finite, 0 when one is NaN/Inf, -1 on a bad argument. */
int kvr_host_all_finite(const void* p, int32_t dtype, int64_t n);
/* Per-step host helpers of a graph-replayed serving step (DecodePlan.step; host code only).
 * kvr_step_stage: waits for `ring_event` (the last launch that read this staging slot), then
 * -- when `check` -- scans the HOST inputs q / k / v (any may be NULL) for NaN/Inf and copies
 * them into the pinned `staging` buffer at their offsets.  Returns 1 (staged), 0 (a non-finite
 * value: nothing was copied), < 0 on an error.
 * kvr_step_launch: enqueues on `stream` the staging -> `dev_buf` copy of `bytes` (slot ids,
 * lengths and the staged inputs), a launch of the instantiated CUDA graph `graph_exec`
 * (cudaGraphExec_t; NULL = none) and a record of `ring_event`. */
int kvr_step_stage(void* ring_event, void* staging, const void* q, int64_t q_off, int64_t q_bytes, int32_t q_dtype,
                   const void* k, int64_t k_off, const void* v, int64_t v_off, int64_t kv_bytes, int32_t kv_dtype,
                   int32_t check);
int kvr_step_launch(void* dev_buf, const void* staging, int64_t bytes, void* graph_exec, void* ring_event,
                    void* stream);
/* A staging ring bound to fixed host inputs q / k / v (any may be NULL: not staged) and, per slot,
 * a pinned staging buffer, its device twin, an instantiated CUDA graph and an event: then
 * kvr_step_ring_run(ring, slot, meta) is the whole per-step host work of a graph-replayed serving
 * step -- kvr_step_stage (wait for the slot's event, NaN/Inf scan when `check`, copy-in), the
 * `meta_bytes` of step metadata (slot ids, lengths) copied to the front of the staging buffer,
 * then kvr_step_launch.  Returns KVR_ERR_NONFINITE (nothing launched) on a NaN/Inf input. */
typedef struct kvr_step_ring kvr_step_ring;
kvr_step_ring* kvr_step_ring_create(int32_t n_slots, const void* q, int64_t q_off, int64_t q_bytes, int32_t q_dtype,
                                    const void* k, int64_t k_off, const void* v, int64_t v_off, int64_t kv_bytes,
                                    int32_t kv_dtype, int64_t meta_bytes, int64_t bytes, int32_t check, void* stream);
int kvr_step_ring_set_slot(kvr_step_ring* ring, int32_t slot, void* staging, void* dev, void* graph_exec, void* event);
int kvr_step_ring_run(kvr_step_ring* ring, int32_t slot, const void* meta);
void kvr_step_ring_destroy(kvr_step_ring* ring);
/* Direct modes: each kvr_step_ring_run launches kvr_decode_step itself (no graph), consecutive
 * steps chained by programmatic dependent launch; new_slot / seq_lens point into the pinned slot.
 *   mode 1: q / new_k / new_v are read by the kernel in place from the pinned slot (over the bus;
 *           the query before the grid-dependency wait: a staged query is immutable for that launch);
 *   mode 2: a one-CTA copy kernel chained in front of the decode moves the slot to its device twin
 *           (overlapping the previous step) and the decode reads q / k / v there.
 * The other arguments are kvr_decode_step's, fixed for the ring. */
int kvr_step_ring_set_decode(kvr_step_ring* ring, int32_t q_dtype, int32_t kv_dtype, const kvr_pool* pool,
                             const int32_t* block_table, int32_t bt_stride, int32_t batch, int32_t num_q_heads,
                             int32_t max_seq_len, int32_t rot_order, int32_t rotate, int32_t targets,
                             const uint32_t* sign_words, float* out, void* workspace, size_t workspace_bytes,
                             int32_t num_splits, uint32_t* flags, int32_t mode);
/* Profiling aid: mean host ns per kvr_step_ring_run since load -- stage (slot wait, scan, copy-in),
 * metadata copy, decode launch, event record. */
void kvr_debug_step_ring_times(double* out4);
/* Optional: stage-in copies go on `copy_stream` (the step stream waits for each); NULL = same stream. */
int kvr_step_ring_set_copy_stream(kvr_step_ring* ring, void* copy_stream);
/* Number of SMs of the current device (0 if no device). */
int kvr_device_sms(void);

/* ---- operator layer: kvrot._kernels on device buffers, bit-exact f64 ------- */
int kvr_fwht_rows_f64(double* x, int64_t n, int32_t d, int32_t order, void* stream);
int kvr_pack_rows(const uint8_t* nibbles, uint8_t* out, int64_t n, int32_t d, void* stream);
int kvr_unpack_rows(const uint8_t* packed, uint8_t* out, int64_t n, int32_t logical_len,
                    void* stream);
int kvr_quantize_rows_f64(const double* x, int64_t n, int32_t d, uint8_t* packed, float* scale,
                          uint8_t* zp, void* stream);
int kvr_dequantize_rows_f64(const uint8_t* packed, const float* scale, const uint8_t* zp,
                            int64_t n, int32_t logical_len, double* out, void* stream);

/*
 * Block rotation of rows (n, d): forward  y = x diag(s) H_blk   (inverse=0)
 *                                inverse  y = x H_blk diag(s)   (inverse=1)
 * in_dtype in {F64, F32, BF16, F16}; out_dtype in {F64, F32}.  F64->F64 is
 * bit-identical to the reference.  sign_words (host): d/32 little-endian
 * words, bit i set <=> signs[i] == -1; NULL means no sign flips.
 */
int kvr_block_rotate(const void* x, int32_t in_dtype, void* out, int32_t out_dtype, int64_t n,
                     int32_t d, int32_t order, const uint32_t* sign_words, int32_t inverse,
                     void* stream);

/*
 * Dense factor of a rotation spec (row f3): y = x M for rows (n, d), M a device f64
 * [d][d] row-major matrix, f64 arithmetic (k ascending).  Replaces the learned R's
 * `out @ spec.learned` / `out @ spec.learned.T` (rotation.py:140-141, 154-155) and applies
 * the composed T = diag(s) H_blk R (compose_transform, rotation.py:171-184) to decode
 * queries and T^T to outputs in one launch.  in_dtype {F64, F32, BF16, F16}, out_dtype
 * {F64, F32}; x and y must not alias; d <= 768.
 */
int kvr_rows_matmul_f64(const void* x, int32_t in_dtype, const double* m, void* y, int32_t out_dtype, int64_t n,
                        int32_t d, void* stream);

/*
 * K1: fused rotate -> token-wise INT4 quantize -> paged store.
 *   k, v         : (n_tok, H, d) rows of in_dtype (F64/F32/BF16/F16), contiguous
 *   slot_mapping : int64[n_tok] device, page_id * P + slot; negative = skip
 *   rotate       : 0 = plain INT4 twin (no rotation anywhere)
 *   targets      : KVR_KEYS_ONLY rotates K only; KVR_KEYS_AND_VALUES both
 *   exact        : 1 = f64 arithmetic (bit-identical to the reference for any
 *                  input); 0 = fast path (fp32 butterfly)
 *   flags        : device uint32, KVR_FLAG_* bits OR-ed in (may be NULL)
 */
int kvr_rotate_quantize_store(const void* k, const void* v, int32_t in_dtype, int64_t n_tok,
                              const int64_t* slot_mapping, const kvr_pool* pool,
                              int32_t rot_order, int32_t rotate, int32_t targets,
                              const uint32_t* sign_words, int32_t exact, uint32_t* flags,
                              void* stream);

/*
 * Row f3, K1 with a learned R fused: y = x diag(s) H_blk R (rotation.py:118-142) for the K
 * rows and for V per value_branch_spec (rotation.py:162-168: learned_values=1 the same T,
 * 0 the Hadamard part only; targets KVR_KEYS_ONLY leaves V plain).  One tcgen05 kernel: T as
 * three bf16 parts in shared memory (24 mantissa bits), fp32 accumulation in TMEM.  A row with
 * a code within the margin of a rounding boundary (or a zero point near a tie) is redone whole
 * in f64 (FWHT then R) under the reference's own scale and zero point, so codes and zero points
 * equal the reference composition's.  KVR_K1L_FAST=1 (environment, read per call) recomputes only
 * the flagged 8-code words under this kernel's scale: ~6x faster, ~1.5e-6 of codes one step off.
 *   t_img : device image of T, 98,304 bytes (kvr_learned_pack_image)
 *   r_t   : device R^T, f64 [d][d] row-major (r_t[n * d + k] = R[k][n])
 * Only bf16 rows, d = 128, T = 16, power-of-two pages: KVR_ERR_UNSUPPORTED otherwise (the
 * caller rotates in f64 and stores through kvr_rotate_quantize_store(exact=1)).
 */
int kvr_rotate_quantize_store_learned(const void* k, const void* v, int32_t in_dtype, int64_t n_tok,
                                      const int64_t* slot_mapping, const kvr_pool* pool, int32_t rot_order,
                                      int32_t targets, int32_t learned_values, const uint32_t* sign_words,
                                      const void* t_img, const double* r_t, uint32_t* flags, void* stream);
/* Host helper: the kernel's shared-memory image of T (host f64 [128][128] row-major, the dense
 * compose_transform, rotation.py:171-184) into `img` (host, 49,152 uint16: three bf16 parts). */
void kvr_learned_pack_image(const double* t, uint16_t* img);

/*
 * K4: flatten-dequant of sequences into dense stored-space rows.
 *   block_table : int32[batch][bt_stride] page ids; seq_lens: int32[batch]
 *   k_out/v_out : (batch, max_len, H, d) of out_dtype (F64/F32/BF16); rows past a
 *                 sequence's length are left untouched.
 */
int kvr_dequantize_pages(const kvr_pool* pool, const int32_t* block_table, int32_t bt_stride,
                         const int32_t* seq_lens, int32_t batch, int32_t max_len, void* k_out,
                         void* v_out, int32_t out_dtype, void* stream);

/*
 * K2+K3: paged INT4 decode attention, split-K over pages, rotated-frame query,
 * inverse-rotated output for V (when rotate && targets == KEYS_AND_VALUES).
 *   q        : (batch, num_q_heads, d) of q_dtype (F32/BF16/F16)
 *   out      : (batch, num_q_heads, d) f32
 *   seq_lens[b] <= max_seq_len <= bt_stride * page_tokens: the split ranges are
 *   cut from max_seq_len so the page-id loads do not wait on seq_lens; tokens
 *   past max_seq_len are ignored (kvr_decode_step sets KVR_FLAG_LEN_OVERFLOW).
 *   num_splits <= 0 picks a split count for the device.  Workspace must be at
 *   least kvr_decode_workspace_bytes(...) bytes and zero-filled once before
 *   first use (the kernels leave the split counters at zero afterwards).
 */
/*
 * Both decode entry points launch with programmatic dependent launch: before their
 * dependency wait they read block_table, seq_lens and new_slot, and -- unless the
 * stream's last pool access was a write -- pool cells older than the last two
 * tokens of each sequence.  Every store entry point of this library notes its
 * stream; a caller that writes pool bytes by other means (a copy, its own kernel)
 * calls kvr_note_pool_write(stream) before the next decode on that stream.  Splits merge inside the decode
 * kernel up to 32 splits (a thread-block cluster up to 8, the last CTA of each
 * (sequence, kv head) above that); with more, a second split-merge kernel follows
 * the decode kernel on the stream.
 */
size_t kvr_decode_workspace_bytes(int32_t batch, int32_t num_kv_heads, int32_t num_q_heads,
                                  int32_t head_dim, int32_t num_splits);
int kvr_decode_pick_splits(int32_t batch, int32_t num_kv_heads, int32_t max_seq_len,
                           int32_t page_tokens);
int kvr_paged_decode(const void* q, int32_t q_dtype, const kvr_pool* pool,
                     const int32_t* block_table, int32_t bt_stride, const int32_t* seq_lens,
                     int32_t batch, int32_t num_q_heads, int32_t max_seq_len, int32_t rot_order,
                     int32_t rotate, int32_t targets, const uint32_t* sign_words, float* out,
                     void* workspace, size_t workspace_bytes, int32_t num_splits, void* stream);

/*
 * Row f3: paged INT4 decode with a learned rotation fused into the kernel (attention.py:50-87 on
 * a learned spec, rotation.py:118-168): the query is multiplied by the composed key transform
 * T = diag(s) H_blk R (compose_transform, rotation.py:171-184) in the kernel's prologue, and the
 * output goes back through the value branch (value_branch_spec, rotation.py:162-168) before the
 * store.  Same arguments as kvr_paged_decode, plus
 *   t_pad    : device f32 [128][129] = T with a row stride of 129 floats (16-B aligned)
 *   out_mode : 0 keys only (no output transform), 1 values rotated by the Hadamard part only
 *              (learned_values = False: block Hadamard inverse of rot_order, then sign_words),
 *              2 values through T as well (learned_values = True: o T^T)
 * At most 32 splits (the merge runs inside the grid).  d = 128, T = 16, power-of-two pages,
 * G in {1, 2, 4, 8}: KVR_ERR_UNSUPPORTED otherwise (the caller then rotates the query and the
 * output itself around kvr_paged_decode, e.g. with kvr_rows_matmul_f64).
 */
int kvr_paged_decode_learned(const void* q, int32_t q_dtype, const kvr_pool* pool,
                             const int32_t* block_table, int32_t bt_stride, const int32_t* seq_lens,
                             int32_t batch, int32_t num_q_heads, int32_t max_seq_len, const float* t_pad,
                             int32_t out_mode, int32_t rot_order, const uint32_t* sign_words, float* out,
                             void* workspace, size_t workspace_bytes, int32_t num_splits, void* stream);

/*
 * Flat full-precision decode (attention.decode_step_fp): q (num_q_heads, d), k / v
 * (t, num_kv_heads, d) f64 device arrays, out (num_q_heads, d) f64; f64 arithmetic,
 * max-subtracted softmax; head_dim <= 256.
 */
int kvr_decode_flat_f64(const double* q, const double* k, const double* v, int64_t t, int32_t num_q_heads,
                        int32_t num_kv_heads, int32_t head_dim, double* out, void* stream);

/*
 * One serving decode step, fused into a single launch: for every sequence b the
 * new token's K/V rows (new_k/new_v: (batch, H, d) of kv_dtype) are rotated and
 * INT4-quantized reference-exactly (f64) into slot new_slot[b], and the decode
 * attends over seq_lens[b] tokens -- which must already count that token (the
 * host allocator's slot).  new_slot[b] < 0 skips the write for sequence b (its
 * decode then covers seq_lens[b] stored tokens).  A row with NaN/Inf is not
 * written and sets KVR_FLAG_NONFINITE in *flags.  Slots past a sequence's length
 * are never read (their bytes may be anything).  Same output/workspace contract
 * as kvr_paged_decode.
 */
int kvr_decode_step(const void* q, int32_t q_dtype, const void* new_k, const void* new_v, int32_t kv_dtype,
                    const int64_t* new_slot, const kvr_pool* pool, const int32_t* block_table, int32_t bt_stride,
                    const int32_t* seq_lens, int32_t batch, int32_t num_q_heads, int32_t max_seq_len,
                    int32_t rot_order, int32_t rotate, int32_t targets, const uint32_t* sign_words, float* out,
                    void* workspace, size_t workspace_bytes, int32_t num_splits, uint32_t* flags, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KVROT_B200_H */
