// Host-side launcher declarations shared between the .cu translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/kvrot_b200.h"

namespace kvr {
struct Signs;
struct Pool;
}  // namespace kvr

int kvr_launch_fwht_f64(double* x, int64_t n, int d, int order, cudaStream_t st);
int kvr_launch_quantize_f64(const double* x, int64_t n, int d, uint8_t* p, float* s, uint8_t* z, cudaStream_t st);
int kvr_launch_dequantize_f64(const uint8_t* p, const float* s, const uint8_t* z, int64_t n, int len, double* out,
                              cudaStream_t st);
int kvr_launch_pack(const uint8_t* nib, uint8_t* out, int64_t n, int d, cudaStream_t st);
int kvr_launch_unpack(const uint8_t* p, uint8_t* out, int64_t n, int len, cudaStream_t st);
int kvr_launch_block_rotate(const void* x, int in_dtype, void* out, int out_dtype, int64_t n, int d, int order,
                            const kvr::Signs& s, int has, int inv, cudaStream_t st);
int kvr_launch_store_exact(const void* k, const void* v, int in_dtype, int64_t n_tok, const int64_t* slots,
                           const kvr::Pool& pool, int order, int rot_k, int rot_v, const kvr::Signs& s, int has,
                           uint32_t* flags, cudaStream_t st);
int kvr_launch_store_bf16(const void* k, const void* v, int in_dtype, int64_t n_tok, const int64_t* slots,
                          const kvr::Pool& pool, uint32_t* flags, cudaStream_t st);
int kvr_launch_dequant_pages(const kvr::Pool& pool, const int32_t* bt, int bt_stride, const int32_t* lens, int batch,
                             int max_len, void* k_out, void* v_out, int out_dtype, cudaStream_t st);
int kvr_launch_decode_flat_f64(const double* q, const double* k, const double* v, int64_t t, int nq, int H, int d,
                               double* out, cudaStream_t st);

int kvr_launch_rows_matmul(const void* x, int in_dtype, const double* m, void* y, int out_dtype, int64_t n, int d,
                           cudaStream_t st);

// Fast serving-path write (bf16/fp16 rows, head_dim 128): returns KVR_ERR_UNSUPPORTED
// when the configuration has no specialised kernel (caller falls back to the exact path).
int kvr_launch_store_fast(const void* k, const void* v, int in_dtype, int64_t n_tok, const int64_t* slots,
                          const kvr::Pool& pool, int order, int rot_k, int rot_v, const kvr::Signs& s, int has,
                          uint32_t* flags, cudaStream_t st);
// Row f3: the tcgen05 K1 with the learned R fused (bf16 rows, head_dim 128); K tiles through T,
// V tiles in mode_v (0 plain, 1 block Hadamard, 2 T).  KVR_ERR_UNSUPPORTED otherwise.
int kvr_launch_store_learned(const void* k, const void* v, int in_dtype, int64_t n_tok, const int64_t* slots,
                             const kvr::Pool& pool, int order, int mode_v, const kvr::Signs& s, int has,
                             const void* t_img, const double* rt, uint32_t* flags, cudaStream_t st);
void kvr_pack_learned_image(const double* t, uint16_t* img);

// Decode (kvr_decode.cu)
size_t kvr_decode_ws_bytes(int batch, int H, int nq, int d, int splits);
int kvr_pick_splits(int batch, int H, int max_len, int P);
int kvr_launch_decode(const void* q, int q_dtype, const kvr::Pool& pool, const int32_t* bt, int bt_stride,
                      const int32_t* lens, int batch, int nq, int max_len, int order, int rotate, int rot_v,
                      const kvr::Signs& s, int has, float* out, void* ws, size_t ws_bytes, int splits,
                      cudaStream_t st, const void* new_k = nullptr, const void* new_v = nullptr, int new_dtype = 0,
                      const int64_t* new_slot = nullptr, uint32_t* flags = nullptr, int q_host_staged = 0,
                      const float* lq = nullptr, int lq_out = 0, int lq_order = 0);
// lq (row f3): the composed learned transform T as f32 [128][129] (decode_tma_kernel<., 0, .>), the
// query multiplied by it in the prologue; lq_out: 0 no output transform, 1 block Hadamard inverse of
// order lq_order with the signs, 2 T^T
// q_host_staged: 0 plain; 1 the query is host-staged (read before the wait); 2 lengths / slot ids
// are written by the preceding grid (read after the wait; no pre-wait cell requests)

void kvr_set_decode_trace(void* trace);
int kvr_launch_stage_copy(void* dst, const void* src, int64_t bytes, cudaStream_t st);
void kvr_set_k1_impl(int impl);

// Tensor-map encoder resolved through the runtime (no -lcuda link dependency).
CUresult kvr_encode_tensor_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows,
                                  uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_rows,
                                  CUtensorMapSwizzle swz);
// Per-device launch state: function attributes and occupancy answers are cached per
// CUDA device (index = kvr_current_device()), so one process may drive several GPUs.
constexpr int KVR_MAX_DEVICES = 64;
int kvr_current_device();
int kvr_num_sms();

// Pool-write notes per stream (host side, mutex-protected): every launch that writes
// pool cells marks its stream; the next decode launch on that stream takes the mark
// and then issues no pool reads before its grid-dependency wait (griddepcontrol.wait
// is the only point where a preceding grid's writes are guaranteed visible).
void kvr_mark_pool_written(cudaStream_t st);
bool kvr_take_pool_written(cudaStream_t st);
