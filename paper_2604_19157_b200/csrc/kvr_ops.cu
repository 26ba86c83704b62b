// Operator-layer kernels (kvrot._kernels on the GPU) and the generic f64
// ("exact") variants of the rotation, the fused write and the flatten-dequant.
//
// Everything here computes in IEEE f64 with the reference's operation order,
// so results are bit-identical to kvrot's numpy/Cython backends:
//   fwht_rows        _ref.py:22-40  / _core.pyx:22-47
//   quantize_rows    _ref.py:57-80  / _core.pyx:76-130
//   dequantize_rows  _ref.py:83-95  / _core.pyx:133-158
//   pack/unpack      _ref.py:43-54  / _core.pyx:50-73
// These kernels are warp-per-row and latency-oriented; the bandwidth-bound
// serving path (bf16/fp16 rows, head_dim 128) lives in kvr_store_fast.cu and
// kvr_decode.cu.
#include "kvr_common.cuh"
#include "kvr_exact.cuh"
#include "kvr_internal.h"

namespace kvr {

__global__ void fwht_rows_f64_kernel(double* x, int64_t n, int d, int order) {
  extern __shared__ double sm_f64[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* s = sm_f64 + (size_t)wib * d;
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; row < n;
       row += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    double* xr = x + row * d;
    for (int i = lane; i < d; i += 32) s[i] = xr[i];
    __syncwarp();
    warp_fwht_f64(s, d, order, lane);
    for (int i = lane; i < d; i += 32) xr[i] = s[i];
    __syncwarp();
  }
}

__global__ void quantize_rows_f64_kernel(const double* x, int64_t n, int d, uint8_t* packed, float* scale,
                                         uint8_t* zp) {
  extern __shared__ double sm_f64[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* s = sm_f64 + (size_t)wib * d;
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; row < n;
       row += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    for (int i = lane; i < d; i += 32) s[i] = x[row * d + i];
    __syncwarp();
    warp_quantize_f64(s, d, lane, packed + row * (d >> 1), scale + row, zp + row);
    __syncwarp();
  }
}

__global__ void dequantize_rows_f64_kernel(const uint8_t* packed, const float* scale, const uint8_t* zp, int64_t n,
                                           int len, double* out) {
  const int half = len >> 1;
  const int64_t total = n * half;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / half;
    const int m = (int)(idx % half);
    const double s64 = (double)scale[row];
    const uint8_t z = zp[row];
    double* o = out + row * len + 2 * m;
    if (z == 0xFF) {
      o[0] = s64;
      o[1] = s64;
    } else {
      const uint8_t b = packed[row * half + m];
      const double zf = (double)z;
      o[0] = s64 * ((double)(b & 0x0F) - zf);
      o[1] = s64 * ((double)(b >> 4) - zf);
    }
  }
}

__global__ void pack_rows_kernel(const uint8_t* nib, uint8_t* out, int64_t n, int d) {
  const int64_t total = n * (d >> 1);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / (d >> 1);
    const int m = (int)(idx % (d >> 1));
    out[idx] = (uint8_t)(nib[row * d + 2 * m] | (nib[row * d + 2 * m + 1] << 4));
  }
}

__global__ void unpack_rows_kernel(const uint8_t* packed, uint8_t* out, int64_t n, int len) {
  const int half = len >> 1;
  const int64_t total = n * half;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / half;
    const int m = (int)(idx % half);
    const uint8_t b = packed[row * half + m];
    out[row * len + 2 * m] = b & 0x0F;
    out[row * len + 2 * m + 1] = b >> 4;
  }
}

// Rotation of rows in f64 (exact for f64 input), any input dtype, f64/f32 out.
template <typename TIn, typename TOut>
__global__ void block_rotate_kernel(const TIn* x, TOut* out, int64_t n, int d, int order, Signs signs, int has_signs,
                                    int inverse) {
  extern __shared__ double sm_f64[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* s = sm_f64 + (size_t)wib * d;
  for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; row < n;
       row += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    for (int i = lane; i < d; i += 32) {
      double v = load_as_f64<TIn>(x, row * d + i);
      if (has_signs && !inverse && sign_bit(signs, i)) v = v * -1.0;
      s[i] = v;
    }
    __syncwarp();
    warp_fwht_f64(s, d, order, lane);
    for (int i = lane; i < d; i += 32) {
      double v = s[i];
      if (has_signs && inverse && sign_bit(signs, i)) v = v * -1.0;
      out[row * d + i] = (TOut)v;
    }
    __syncwarp();
  }
}

// Row f3's dense factor: y = x M in f64 (M [d][d] row-major), the learned R of
// rotation.py:140-141 / 154-155 (M = R or R^T) and the composed transforms of the query
// prep and the output's value branch (M = T = diag(s) H_blk R, or T^T).  Latency-shaped
// for the few rows of a decode step: a CTA owns 8 rows (staged in shared memory as f64)
// and 32 output columns; its 16 warps split k (warp = k group, lane = column: every M
// read is a coalesced 256-B row segment), the first 8 M values per thread are loaded
// before the grid-dependency wait (M is constant, x may be the previous kernel's output),
// and the 16 partial sums are added in k-group order through shared memory.
constexpr int RM_ROWS = 8, RM_COLS = 32, RM_KG = 16;
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(RM_COLS * RM_KG) rows_matmul_kernel(const TIn* x, const double* __restrict__ m,
                                                                       TOut* y, int64_t n, int d) {
  extern __shared__ double rm_sm[];  // xs [RM_ROWS][d] | part [RM_KG][RM_ROWS][RM_COLS]
  double* xs = rm_sm;
  double* part = rm_sm + RM_ROWS * d;
  const int c = threadIdx.x & (RM_COLS - 1), kg = threadIdx.x / RM_COLS;
  const int col = blockIdx.y * RM_COLS + c;
  const int kq = (d + RM_KG - 1) / RM_KG, k0 = kg * kq, k1 = min(d, k0 + kq);
  const bool live = col < d;
  double mk[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) mk[u] = (live && k0 + u < k1) ? __ldg(m + (size_t)(k0 + u) * d + col) : 0.0;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t r0 = (int64_t)blockIdx.x * RM_ROWS;
  const int nr = (int)((n - r0) < RM_ROWS ? (n - r0) : RM_ROWS);
  for (int i = threadIdx.x; i < RM_ROWS * d; i += blockDim.x) {
    const int r = i / d, k = i - r * d;
    xs[i] = r < nr ? load_as_f64<TIn>(x, (r0 + r) * d + k) : 0.0;
  }
  __syncthreads();
  double acc[RM_ROWS];
#pragma unroll
  for (int r = 0; r < RM_ROWS; ++r) acc[r] = 0.0;
  if (live) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < k1)
#pragma unroll
        for (int r = 0; r < RM_ROWS; ++r) acc[r] = fma(xs[r * d + k0 + u], mk[u], acc[r]);
    for (int k = k0 + 8; k < k1; ++k) {
      const double mv = __ldg(m + (size_t)k * d + col);
#pragma unroll
      for (int r = 0; r < RM_ROWS; ++r) acc[r] = fma(xs[r * d + k], mv, acc[r]);
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll
  for (int r = 0; r < RM_ROWS; ++r) part[(kg * RM_ROWS + r) * RM_COLS + c] = acc[r];
  __syncthreads();
  if (threadIdx.x < RM_ROWS * RM_COLS) {
    const int r = threadIdx.x / RM_COLS, cc = threadIdx.x & (RM_COLS - 1);
    const int oc = blockIdx.y * RM_COLS + cc;
    if (r < nr && oc < d) {
      double v = part[r * RM_COLS + cc];
#pragma unroll
      for (int g = 1; g < RM_KG; ++g) v += part[(g * RM_ROWS + r) * RM_COLS + cc];
      y[(r0 + r) * d + oc] = (TOut)v;
    }
  }
}

template <typename TIn>
static int rows_matmul_out(const void* x, const double* m, void* y, int out_dtype, int64_t n, int d, cudaStream_t st) {
  const size_t sm = (size_t)RM_ROWS * d * 8 + (size_t)RM_KG * RM_ROWS * RM_COLS * 8;
  auto kd = rows_matmul_kernel<TIn, double>;
  auto kf = rows_matmul_kernel<TIn, float>;
  static bool attr_set[KVR_MAX_DEVICES];
  const int dev = kvr_current_device();
  if (!attr_set[dev]) {  // up to d = 768: 48 KB + 32 KB
    cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((n + RM_ROWS - 1) / RM_ROWS), (unsigned)((d + RM_COLS - 1) / RM_COLS));
  cfg.blockDim = dim3(RM_COLS * RM_KG);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (out_dtype == KVR_F64)
    e = cudaLaunchKernelEx(&cfg, kd, (const TIn*)x, m, (double*)y, n, d);
  else if (out_dtype == KVR_F32)
    e = cudaLaunchKernelEx(&cfg, kf, (const TIn*)x, m, (float*)y, n, d);
  else
    return KVR_ERR_UNSUPPORTED;
  return e == cudaSuccess ? 0 : KVR_ERR_CUDA;
}

// Generic exact fused write: warp per (token, head, side) row, f64 arithmetic.
// Row order: all K rows (token-major, head-minor) then all V rows.
template <typename TIn>
__global__ void store_exact_kernel(const TIn* k, const TIn* v, int64_t n_tok, const int64_t* slots, Pool pool,
                                   int order, int rot_k, int rot_v, Signs signs, int has_signs, uint32_t* flags) {
  extern __shared__ double sm_f64[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int d = pool.d, H = pool.H;
  double* s = sm_f64 + (size_t)wib * d;
  const int64_t rows = n_tok * H;
  for (int64_t r2 = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; r2 < 2 * rows;
       r2 += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int side = r2 >= rows;  // 0 = K, 1 = V
    const int64_t row = side ? r2 - rows : r2;
    const int64_t tok = row / H;
    const int head = (int)(row % H);
    const int64_t slot = slots[tok];
    if (slot < 0) continue;
    const TIn* src = side ? v : k;
    const int rot = side ? rot_v : rot_k;
    bool finite = true;
    for (int i = lane; i < d; i += 32) {
      double val = load_as_f64<TIn>(src, row * d + i);
      finite &= isfinite(val);
      if (rot && has_signs && sign_bit(signs, i)) val = val * -1.0;
      s[i] = val;
    }
    finite = __all_sync(0xffffffffu, finite);
    __syncwarp();
    if (!finite) {
      if (lane == 0 && flags) atomicOr(flags, (uint32_t)KVR_FLAG_NONFINITE);
      continue;
    }
    if (rot) warp_fwht_f64(s, d, order, lane);
    const int64_t page = slot / pool.P;
    int ci;
    uint8_t* cell = cell_of(pool, page, head, (int)(slot % pool.P), ci);
    uint8_t* payload = cell + (side ? cell_vcode(pool, ci) : cell_kcode(pool, ci));
    float* sc = reinterpret_cast<float*>(cell + (side ? cell_vscale(pool, ci) : cell_kscale(pool, ci)));
    uint8_t* zp = cell + (side ? cell_vzp(pool, ci) : cell_kzp(pool, ci));
    warp_quantize_f64(s, d, lane, payload, sc, zp);
    __syncwarp();
  }
}

// Flatten-dequant (cache.py:337-362): thread per (row, byte) -> two outputs.
template <typename TOut>
__global__ void dequant_pages_kernel(Pool pool, const int32_t* bt, int bt_stride, const int32_t* lens, int batch,
                                     int max_len, TOut* k_out, TOut* v_out) {
  const int d = pool.d, H = pool.H, half = d >> 1;
  const int64_t per_side = (int64_t)batch * max_len * H * half;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * per_side;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int side = idx >= per_side;
    int64_t r = side ? idx - per_side : idx;
    const int m = (int)(r % half);
    r /= half;
    const int head = (int)(r % H);
    r /= H;
    const int t = (int)(r % max_len);
    const int b = (int)(r / max_len);
    if (t >= lens[b]) continue;
    const int page = bt[(int64_t)b * bt_stride + t / pool.P];
    int ci;
    const uint8_t* cell = cell_of(pool, page, head, t % pool.P, ci);
    const uint8_t byte = cell[(side ? cell_vcode(pool, ci) : cell_kcode(pool, ci)) + m];
    const float sc = *reinterpret_cast<const float*>(cell + (side ? cell_vscale(pool, ci) : cell_kscale(pool, ci)));
    const uint8_t z = cell[side ? cell_vzp(pool, ci) : cell_kzp(pool, ci)];
    TOut* o = (side ? v_out : k_out) + ((((int64_t)b * max_len + t) * H + head) * d) + 2 * m;
    if (z == 0xFF) {
      o[0] = (TOut)sc;
      o[1] = (TOut)sc;
    } else {
      if constexpr (sizeof(TOut) == 8) {
        const double s64 = (double)sc, zf = (double)z;
        o[0] = (TOut)(s64 * ((double)(byte & 0x0F) - zf));
        o[1] = (TOut)(s64 * ((double)(byte >> 4) - zf));
      } else {
        const float zf = (float)z;
        o[0] = (TOut)(sc * ((float)(byte & 0x0F) - zf));
        o[1] = (TOut)(sc * ((float)(byte >> 4) - zf));
      }
    }
  }
}

// Fast flatten-dequant for the serving geometry (d = 128, 16-token cells): four warps
// per cell (16 tokens of one head), four tokens each; a lane owns 32 dims of one token's
// K or V row (a token's 128 outputs are one contiguous 256-B (bf16) / 512-B (f32) run,
// written by 4 adjacent lanes as whole 64-B groups per store instruction).
// Arithmetic: f32 s * (q - z) (q - z exact, one rounding), then the output cast.
template <typename TOut>
__global__ void __launch_bounds__(256) dequant_cells_kernel(Pool pool, const int32_t* bt, int bt_stride,
                                                            const int32_t* lens, int max_len, int cps_log2,
                                                            int h_log2, TOut* k_out, TOut* v_out) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = blockIdx.x * 8u + (threadIdx.x >> 5);  // grid (cells of one sequence / 2, sequence)
  const int H = pool.H, ntiles = (max_len + 15) >> 4, b = blockIdx.y;
  const uint32_t cell_id = wid >> 2;  // four warps per cell, four tokens each
  if (cell_id >= (uint32_t)(ntiles * H)) return;
  int head, tile;
  if (h_log2 >= 0) {  // the usual power-of-two head count: no integer division
    head = (int)(cell_id & (uint32_t)(H - 1));
    tile = (int)(cell_id >> h_log2);
  } else {
    tile = (int)(cell_id / (uint32_t)H);
    head = (int)cell_id - tile * H;
  }
  // lane: token r of the cell, side (K | V), 32-dim quarter qt of the row
  const int r = 4 * (int)(wid & 3) + (lane >> 3), side = (lane >> 2) & 1, qt = lane & 3, t = tile * 16 + r;
  // programmatic dependent launch: the index math above overlaps the previous grid's tail; the
  // lengths, the block table and the pool may be its output.  This kernel writes no pool cell, so
  // its dependents may be scheduled at once (they wait for its completion before reading)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (t >= max_len) return;
  const int len_b = __ldg(&lens[b]);  // the length and the page id load side by side
  const int page = __ldg(&bt[(int64_t)b * bt_stride + (t >> (4 + cps_log2))]);
  if (t >= len_b) return;
  const uint8_t* cell = pool.base + (int64_t)page * pool.page_bytes +
                        (int64_t)((head << cps_log2) + (tile & ((1 << cps_log2) - 1))) * pool.cell_bytes;
  // lane qt takes code bytes 16 i + 4 qt .. + 3 of the row (dims 32 i + 8 qt .. + 7), i = 0..3: its
  // outputs then sit at 16-B chunk qt of every 64-B group, so each store instruction of the row's four
  // lanes writes 64 contiguous bytes (whole sectors)
  const uint32_t* crow = reinterpret_cast<const uint32_t*>(cell + (side ? 1152 : 128) + r * 64) + qt;
  uint32_t w[4] = {__ldg(crow), __ldg(crow + 4), __ldg(crow + 8), __ldg(crow + 12)};
  const float sc = __ldg(reinterpret_cast<const float*>(cell + side * 64 + r * 4));
  const uint32_t zp = __ldg(cell + 2176 + side * 16 + r);
  // a code c as the float 2^23 + c (one PRMT puts the nibble under the exponent byte 0x4B), minus
  // 2^23 + z: the exact c - z, then one f32 product by the scale (FADD2 / FMUL2 on the element pair of
  // one code byte).  A sentinel row (zp 0xFF) outputs its offset, held in the scale slot: its codes
  // are taken as 0 and its zero point as -1, so every element is (0 + 1) * offset.
  const bool sent = zp == 0xFFu;
  const float zf = sent ? 8388607.0f : 8388608.0f + (float)zp;
  const unsigned long long z2 = pk(zf, zf), s2 = pk(sc, sc);
  TOut* dst = (side ? v_out : k_out) + (((int64_t)b * max_len + t) * H + head) * 128 + qt * 8;
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // word i: dims 32 i + 8 qt + 2 j (low nibble of byte j), + 2 j + 1 (high)
    const uint32_t wi = sent ? 0u : w[i];
    const uint32_t lo = wi & 0x0F0F0F0Fu, hi = (wi >> 4) & 0x0F0F0F0Fu;
    float f[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned long long x = pk(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7440u | j)),
                                      __uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7440u | j)));
      upk(mul2(sub2(x, z2), s2), f[2 * j], f[2 * j + 1]);
    }
    if constexpr (sizeof(TOut) == 2) {
      uint32_t u[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
        u[j] = *reinterpret_cast<const uint32_t*>(&h2);
      }
      *reinterpret_cast<uint4*>(dst + 32 * i) = make_uint4(u[0], u[1], u[2], u[3]);
    } else {
      float4* d4 = reinterpret_cast<float4*>(dst + 32 * i);
      d4[0] = make_float4(f[0], f[1], f[2], f[3]);
      d4[1] = make_float4(f[4], f[5], f[6], f[7]);
    }
  }
}

// BF16 pool write (cache.py:264-266): one warp per (token, head, side) row; raw
// values rounded f64 -> f32 (RN) -> bf16 (RNE, cache.py:43-47).  A non-finite row
// is not written and raises the flag (the reference rejects it, cache.py:453-462).
KVR_DEV uint16_t f32_to_bf16_rne(float x) {
  const uint32_t u = __float_as_uint(x);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
template <typename T>
__global__ void store_bf16_kernel(const T* k, const T* v, int64_t n_tok, const int64_t* slots, Pool pool,
                                  uint32_t* flags) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // (token, head, side)
  const int H = pool.H, d = pool.d;
  if (row >= 2 * n_tok * H) return;
  const int side = (int)(row & 1);
  const int64_t th = row >> 1, tok = th / H;
  const int head = (int)(th % H);
  const int64_t slot = slots[tok];
  const T* src = (side ? v : k) + th * d;
  float x[8];
  bool fin = true;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int i = lane + 32 * e;
    x[e] = i < d ? (float)load_as_f64<T>(src, i) : 0.f;
    fin &= (bool)isfinite(x[e]);
  }
  fin = __all_sync(0xffffffffu, fin);
  if (!fin) {
    if (lane == 0 && flags) atomicOr(flags, (uint32_t)KVR_FLAG_NONFINITE);
    return;
  }
  if (slot < 0) return;
  int ci;
  uint8_t* cell = cell_of(pool, slot / pool.P, head, (int)(slot % pool.P), ci);
  uint16_t* dst = reinterpret_cast<uint16_t*>(cell + cell_bf16(pool, side, ci));
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int i = lane + 32 * e;
    if (i < d) dst[i] = f32_to_bf16_rne(x[e]);
  }
}

// BF16 pool flatten-read (cache.py:355-361): bf16 bits -> out dtype, exact.
template <typename TOut>
__global__ void dequant_bf16_kernel(Pool pool, const int32_t* bt, int bt_stride, const int32_t* lens, int batch,
                                    int max_len, TOut* k_out, TOut* v_out) {
  const int d = pool.d, H = pool.H;
  const int64_t per_side = (int64_t)batch * max_len * H * d;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * per_side;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int side = idx >= per_side;
    int64_t r = side ? idx - per_side : idx;
    const int e = (int)(r % d);
    r /= d;
    const int head = (int)(r % H);
    r /= H;
    const int t = (int)(r % max_len);
    const int b = (int)(r / max_len);
    if (t >= lens[b]) continue;
    const int page = bt[(int64_t)b * bt_stride + t / pool.P];
    int ci;
    const uint8_t* cell = cell_of(pool, page, head, t % pool.P, ci);
    const uint16_t bits = reinterpret_cast<const uint16_t*>(cell + cell_bf16(pool, side, ci))[e];
    const float f = __uint_as_float((uint32_t)bits << 16);
    (side ? v_out : k_out)[(((int64_t)b * max_len + t) * H + head) * d + e] = (TOut)f;
  }
}

// Flat full-precision decode (attention.decode_step_fp, attention.py:90-115): per q
// head, softmax(K[:, kv] q / sqrt(d)) V[:, kv] over flat (t, H, d) f64 arrays, all in
// f64.  One CTA per q head; warp w takes tokens w, w + nw, ... with lanes over the
// dims (warp-reduced dot), an online max-subtracted softmax per warp, then the warps
// merge through shared memory.
__global__ void decode_flat_f64_kernel(const double* q, const double* k, const double* v, int64_t t, int H, int G,
                                       int d, double* out) {
  extern __shared__ double fsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int qh = blockIdx.x, kv = qh / G;
  double* so = fsm;                // [nw][d]
  double* sml = fsm + nw * d;      // [nw][2]
  const double scale = 1.0 / sqrt((double)d);
  double qr[8], o[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int x = lane + 32 * e;
    qr[e] = x < d ? q[(int64_t)qh * d + x] : 0.0;
    o[e] = 0.0;
  }
  double m = -INFINITY, l = 0.0;
  for (int64_t tok = warp; tok < t; tok += nw) {
    const double* kr = k + (tok * H + kv) * d;
    const double* vr = v + (tok * H + kv) * d;
    double dot = 0.0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int x = lane + 32 * e;
      if (x < d) dot = fma(kr[x], qr[e], dot);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
    dot *= scale;
    const double mn = fmax(m, dot);
    const double a = exp(m - mn), pw = exp(dot - mn);
    l = l * a + pw;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int x = lane + 32 * e;
      if (x < d) o[e] = fma(pw, vr[x], o[e] * a);
    }
    m = mn;
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int x = lane + 32 * e;
    if (x < d) so[warp * d + x] = o[e];
  }
  if (lane == 0) {
    sml[2 * warp] = m;
    sml[2 * warp + 1] = l;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < d; x += blockDim.x) {
    double mm = -INFINITY;
    for (int w = 0; w < nw; ++w) mm = fmax(mm, sml[2 * w]);
    double lt = 0.0, ot = 0.0;
    for (int w = 0; w < nw; ++w) {
      if (sml[2 * w] == -INFINITY) continue;
      const double f = exp(sml[2 * w] - mm);
      lt += f * sml[2 * w + 1];
      ot += f * so[w * d + x];
    }
    out[(int64_t)qh * d + x] = ot / lt;
  }
}

}  // namespace kvr

// ============================ host launchers ================================
using namespace kvr;

static int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  const int cap = 148 * 32;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

static int warps_per_block_for(int d) {
  // smem per warp = d doubles; keep <= 48 KB per block (no opt-in needed)
  int w = 8;
  while (w > 1 && (size_t)w * d * 8 > 48 * 1024) w >>= 1;
  return w;
}

int kvr_launch_fwht_f64(double* x, int64_t n, int d, int order, cudaStream_t st) {
  const int w = warps_per_block_for(d);
  fwht_rows_f64_kernel<<<grid_for(n, w), 32 * w, (size_t)w * d * 8, st>>>(x, n, d, order);
  return 0;
}

int kvr_launch_quantize_f64(const double* x, int64_t n, int d, uint8_t* p, float* s, uint8_t* z, cudaStream_t st) {
  const int w = warps_per_block_for(d);
  quantize_rows_f64_kernel<<<grid_for(n, w), 32 * w, (size_t)w * d * 8, st>>>(x, n, d, p, s, z);
  return 0;
}

int kvr_launch_dequantize_f64(const uint8_t* p, const float* s, const uint8_t* z, int64_t n, int len, double* out,
                              cudaStream_t st) {
  dequantize_rows_f64_kernel<<<grid_for(n * (len / 2), 256), 256, 0, st>>>(p, s, z, n, len, out);
  return 0;
}

int kvr_launch_pack(const uint8_t* nib, uint8_t* out, int64_t n, int d, cudaStream_t st) {
  pack_rows_kernel<<<grid_for(n * (d / 2), 256), 256, 0, st>>>(nib, out, n, d);
  return 0;
}

int kvr_launch_unpack(const uint8_t* p, uint8_t* out, int64_t n, int len, cudaStream_t st) {
  unpack_rows_kernel<<<grid_for(n * (len / 2), 256), 256, 0, st>>>(p, out, n, len);
  return 0;
}

template <typename TIn>
static int rotate_dispatch_out(const void* x, void* out, int out_dtype, int64_t n, int d, int order, const Signs& s,
                               int has, int inv, cudaStream_t st) {
  const int w = warps_per_block_for(d);
  const size_t sm = (size_t)w * d * 8;
  if (out_dtype == KVR_F64)
    block_rotate_kernel<TIn, double><<<grid_for(n, w), 32 * w, sm, st>>>((const TIn*)x, (double*)out, n, d, order, s,
                                                                         has, inv);
  else if (out_dtype == KVR_F32)
    block_rotate_kernel<TIn, float><<<grid_for(n, w), 32 * w, sm, st>>>((const TIn*)x, (float*)out, n, d, order, s,
                                                                        has, inv);
  else
    return KVR_ERR_UNSUPPORTED;
  return 0;
}

int kvr_launch_block_rotate(const void* x, int in_dtype, void* out, int out_dtype, int64_t n, int d, int order,
                            const Signs& s, int has, int inv, cudaStream_t st) {
  switch (in_dtype) {
    case KVR_F64: return rotate_dispatch_out<double>(x, out, out_dtype, n, d, order, s, has, inv, st);
    case KVR_F32: return rotate_dispatch_out<float>(x, out, out_dtype, n, d, order, s, has, inv, st);
    case KVR_BF16: return rotate_dispatch_out<__nv_bfloat16>(x, out, out_dtype, n, d, order, s, has, inv, st);
    case KVR_F16: return rotate_dispatch_out<__half>(x, out, out_dtype, n, d, order, s, has, inv, st);
  }
  return KVR_ERR_ARG;
}

int kvr_launch_rows_matmul(const void* x, int in_dtype, const double* m, void* y, int out_dtype, int64_t n, int d,
                           cudaStream_t st) {
  switch (in_dtype) {
    case KVR_F64: return rows_matmul_out<double>(x, m, y, out_dtype, n, d, st);
    case KVR_F32: return rows_matmul_out<float>(x, m, y, out_dtype, n, d, st);
    case KVR_BF16: return rows_matmul_out<__nv_bfloat16>(x, m, y, out_dtype, n, d, st);
    case KVR_F16: return rows_matmul_out<__half>(x, m, y, out_dtype, n, d, st);
  }
  return KVR_ERR_ARG;
}

int kvr_launch_store_exact(const void* k, const void* v, int in_dtype, int64_t n_tok, const int64_t* slots,
                           const Pool& pool, int order, int rot_k, int rot_v, const Signs& s, int has,
                           uint32_t* flags, cudaStream_t st) {
  const int w = warps_per_block_for(pool.d);
  const size_t sm = (size_t)w * pool.d * 8;
  const int g = grid_for(2 * n_tok * pool.H, w);
  switch (in_dtype) {
    case KVR_F64:
      store_exact_kernel<double><<<g, 32 * w, sm, st>>>((const double*)k, (const double*)v, n_tok, slots, pool, order,
                                                        rot_k, rot_v, s, has, flags);
      break;
    case KVR_F32:
      store_exact_kernel<float><<<g, 32 * w, sm, st>>>((const float*)k, (const float*)v, n_tok, slots, pool, order,
                                                       rot_k, rot_v, s, has, flags);
      break;
    case KVR_BF16:
      store_exact_kernel<__nv_bfloat16><<<g, 32 * w, sm, st>>>((const __nv_bfloat16*)k, (const __nv_bfloat16*)v,
                                                               n_tok, slots, pool, order, rot_k, rot_v, s, has, flags);
      break;
    case KVR_F16:
      store_exact_kernel<__half><<<g, 32 * w, sm, st>>>((const __half*)k, (const __half*)v, n_tok, slots, pool, order,
                                                        rot_k, rot_v, s, has, flags);
      break;
    default: return KVR_ERR_ARG;
  }
  return 0;
}

int kvr_launch_store_bf16(const void* k, const void* v, int in_dtype, int64_t n_tok, const int64_t* slots,
                          const Pool& pool, uint32_t* flags, cudaStream_t st) {
  if (pool.d > 256) return KVR_ERR_UNSUPPORTED;
  const int64_t rows = 2 * n_tok * pool.H;
  const int g = (int)((rows * 32 + 255) / 256);
  switch (in_dtype) {
    case KVR_F64: store_bf16_kernel<double><<<g, 256, 0, st>>>((const double*)k, (const double*)v, n_tok, slots, pool, flags); break;
    case KVR_F32: store_bf16_kernel<float><<<g, 256, 0, st>>>((const float*)k, (const float*)v, n_tok, slots, pool, flags); break;
    case KVR_BF16:
      store_bf16_kernel<__nv_bfloat16><<<g, 256, 0, st>>>((const __nv_bfloat16*)k, (const __nv_bfloat16*)v, n_tok, slots,
                                                          pool, flags);
      break;
    case KVR_F16:
      store_bf16_kernel<__half><<<g, 256, 0, st>>>((const __half*)k, (const __half*)v, n_tok, slots, pool, flags);
      break;
    default: return KVR_ERR_ARG;
  }
  return 0;
}

int kvr_launch_dequant_pages(const Pool& pool, const int32_t* bt, int bt_stride, const int32_t* lens, int batch,
                             int max_len, void* k_out, void* v_out, int out_dtype, cudaStream_t st) {
  if (pool.prec == KVR_PREC_BF16) {
    const int g = grid_for(2LL * batch * max_len * pool.H * pool.d, 256);
    switch (out_dtype) {
      case KVR_F64: dequant_bf16_kernel<double><<<g, 256, 0, st>>>(pool, bt, bt_stride, lens, batch, max_len, (double*)k_out, (double*)v_out); break;
      case KVR_F32: dequant_bf16_kernel<float><<<g, 256, 0, st>>>(pool, bt, bt_stride, lens, batch, max_len, (float*)k_out, (float*)v_out); break;
      case KVR_BF16:
        dequant_bf16_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(pool, bt, bt_stride, lens, batch, max_len,
                                                               (__nv_bfloat16*)k_out, (__nv_bfloat16*)v_out);
        break;
      default: return KVR_ERR_ARG;
    }
    return 0;
  }
  int cl = 0;
  while ((16 << cl) < pool.P) ++cl;
  const bool fast = pool.d == 128 && pool.T == 16 && (16 << cl) == pool.P && (pool.cell_bytes & 15) == 0 && batch <= 65535 &&
                    ((reinterpret_cast<uintptr_t>(k_out) | reinterpret_cast<uintptr_t>(v_out)) & 15) == 0;
  if (fast && (out_dtype == KVR_BF16 || out_dtype == KVR_F32)) {
    const int64_t cells = (int64_t)((max_len + 15) / 16) * pool.H;  // per sequence
    const int g = (int)((cells * 4 + 7) / 8);  // four warps per cell, eight warps per block
    int hl = 0;
    while ((1 << hl) < pool.H) ++hl;
    if ((1 << hl) != pool.H) hl = -1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g, batch);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (out_dtype == KVR_BF16)
      e = cudaLaunchKernelEx(&cfg, dequant_cells_kernel<__nv_bfloat16>, pool, bt, bt_stride, lens, max_len, cl, hl,
                             (__nv_bfloat16*)k_out, (__nv_bfloat16*)v_out);
    else
      e = cudaLaunchKernelEx(&cfg, dequant_cells_kernel<float>, pool, bt, bt_stride, lens, max_len, cl, hl,
                             (float*)k_out, (float*)v_out);
    return e == cudaSuccess ? 0 : KVR_ERR_CUDA;
  }
  const int64_t work = 2LL * batch * max_len * pool.H * (pool.d / 2);
  const int g = grid_for(work, 256);
  switch (out_dtype) {
    case KVR_F64:
      dequant_pages_kernel<double><<<g, 256, 0, st>>>(pool, bt, bt_stride, lens, batch, max_len, (double*)k_out,
                                                      (double*)v_out);
      break;
    case KVR_F32:
      dequant_pages_kernel<float><<<g, 256, 0, st>>>(pool, bt, bt_stride, lens, batch, max_len, (float*)k_out,
                                                     (float*)v_out);
      break;
    case KVR_BF16:
      dequant_pages_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(pool, bt, bt_stride, lens, batch, max_len,
                                                             (__nv_bfloat16*)k_out, (__nv_bfloat16*)v_out);
      break;
    default: return KVR_ERR_ARG;
  }
  return 0;
}

int kvr_launch_decode_flat_f64(const double* q, const double* k, const double* v, int64_t t, int nq, int H, int d,
                               double* out, cudaStream_t st) {
  if (d > 256 || nq % H) return KVR_ERR_UNSUPPORTED;
  const int warps = 8;
  const size_t smem = (size_t)(warps * d + 2 * warps) * sizeof(double);
  decode_flat_f64_kernel<<<nq, warps * 32, smem, st>>>(q, k, v, t, H, nq / H, d, out);
  return 0;
}
