// K1 -- fused block-Hadamard rotate -> token-wise INT4 quantize -> paged store,
// the serving-path write for bf16/fp16 rows with head_dim 128.
//
// Reference semantics: cache.PageTable.append_token (cache.py:235-270) ->
// _rotate_token (cache.py:453-462) -> apply_block_rotation (rotation.py:118-142)
// -> _kernels.fwht_rows + quantize_rows (_ref.py:22-40, 57-80).
//
// Design (B200, sm_100a):
//  * persistent CTAs of 4 warps; each warp streams 32-row tiles (8 KB) through a
//    private double buffer filled by TMA (cp.async.bulk.tensor.2d, SWIZZLE_128B:
//    conflict-free row-per-thread shared-memory reads);
//  * one thread owns one 128-element row in registers: sign flip + unpack in 2
//    ops per bf16 pair, the 7-stage butterfly as f32x2 (FADD2) except the one
//    lane-crossing stage, NaN-propagating 3-input min/max (FMNMX3.NAN);
//  * the row scale / zero point are formed in f64 exactly as the reference does,
//    from the fp32 butterfly's extreme values;
//  * codes: one FFMA2.RM per element pair evaluates floor((t + z + 1/2) * 2^16)
//    as a fixed-point integer (magic 2^23), twice (+-delta) -- if both agree on
//    the integer part the nibble is provably the reference's round-half-away
//    code for this y; otherwise (|t| within delta of a half step) the element
//    is recomputed in f64 from the bf16 inputs with the reference's own
//    butterfly tree (bit-exact), see exact_code();
//  * 8 nibbles are packed with 3 PRMT + 1 IMAD.HI per 4 codes.
#include "kvr_common.cuh"
#include "kvr_internal.h"

namespace kvr {

constexpr int FS_WARPS = 4;
constexpr int FS_TILE_ROWS = 32;
constexpr int FS_TILE_BYTES = FS_TILE_ROWS * 256;  // 128 bf16 per row
constexpr float FS_MAGIC = 8388608.0f;            // 2^23
constexpr float FS_FIX = 65536.0f;                // 16 fraction bits
constexpr float FS_D = 2.0f;                      // +-delta in units of 2^-16 (delta ~ 3.1e-5)

struct FastStoreParams {
  Pool pool;
  const int64_t* slots;
  uint32_t* flags;
  int64_t n_rows;          // n_tok * H
  int32_t tiles_per_side;  // ceil(n_rows / 32)
  int32_t rot_k, rot_v;
  uint32_t sgn_hi[64];  // word j: bit 31 <=> element 2j+1 negated
  uint32_t sgn_lo[64];  // word j: 0x80000000 <=> element 2j negated (added to w << 16)
};

template <bool F16>
KVR_DEV void unpack_pair(uint32_t w, uint32_t s_hi, uint32_t s_lo, bool rot, float& e, float& o) {
  if constexpr (!F16) {
    // bf16 pair -> two f32 (exact); the sign flip is folded into the same ops
    const uint32_t lo = rot ? (w << 16) + s_lo : (w << 16);
    const uint32_t hi = rot ? ((w ^ s_hi) & 0xFFFF0000u) : (w & 0xFFFF0000u);
    e = __uint_as_float(lo);
    o = __uint_as_float(hi);
  } else {
    const uint32_t ws = rot ? (w ^ ((s_lo >> 16) | s_hi)) : w;
    const __half2 h = *reinterpret_cast<const __half2*>(&ws);
    const float2 f = __half22float2(h);
    e = f.x;
    o = f.y;
  }
}

// Element `e` (0..127) of the row staged in the swizzled TMA tile, as f64.
template <bool F16>
KVR_DEV double tile_elem(const uint8_t* buf, int lane, int e) {
  const int h = e >> 6, c = (e >> 3) & 7, within = e & 7;
  const uint8_t* p = buf + h * 4096 + lane * 128 + ((c ^ (lane & 7)) << 4) + within * 2;
  const uint16_t bits = *reinterpret_cast<const uint16_t*>(p);
  if constexpr (F16) return (double)__half2float(__ushort_as_half(bits));
  return (double)__uint_as_float((uint32_t)bits << 16);
}

// Reference-exact code for element e: the f64 butterfly tree that produces
// output e in _ref.fwht_rows (pairs combined lowest-index-first, stage by
// stage, sign by the bits of e), then * inv, / s64, round-half-away, + z, clip.
template <int ORDER, bool F16>
__device__ __noinline__ uint32_t exact_code(const uint8_t* buf, int lane, int e, bool rot, const Signs* sg,
                                            double inv, double s64, double z) {
  double y;
  if (rot) {
    double acc[ORDER];
    const int base = (e / ORDER) * ORDER, j = e % ORDER;
#pragma unroll 1
    for (int i = 0; i < ORDER; ++i) {
      double x = tile_elem<F16>(buf, lane, base + i);
      if (sign_bit(*sg, base + i)) x = x * -1.0;
      acc[i] = x;
    }
    int n = ORDER;
#pragma unroll 1
    for (int lvl = 0; (1 << lvl) < ORDER; ++lvl) {
      const bool minus = (j >> lvl) & 1;
#pragma unroll 1
      for (int m = 0; m < (n >> 1); ++m) acc[m] = minus ? acc[2 * m] - acc[2 * m + 1] : acc[2 * m] + acc[2 * m + 1];
      n >>= 1;
    }
    y = acc[0] * inv;
  } else {
    y = tile_elem<F16>(buf, lane, e);
  }
  double q = round_half_away(y / s64) + z;
  q = q < 0.0 ? 0.0 : (q > 15.0 ? 15.0 : q);
  return (uint32_t)q;
}

KVR_DEV uint32_t pack4(uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
  // codes sit in byte 2 of each magic-floored value
  const uint32_t c = prmt(prmt(m0, m1, 0x0062u), prmt(m2, m3, 0x0062u), 0x5410u);  // [k0,k1,k2,k3]
  return __umulhi(c, 1u << 28) + c;  // c | c >> 4: bytes 0 and 2 hold k0|k1<<4, k2|k3<<4
}

template <int ORDER, bool F16>
__global__ void __launch_bounds__(FS_WARPS * 32, 3)
    store_fast_kernel(const __grid_constant__ FastStoreParams p, const __grid_constant__ CUtensorMap map_k,
                      const __grid_constant__ CUtensorMap map_v, const __grid_constant__ Signs signs) {
  extern __shared__ uint8_t fs_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fs_smem_raw) + 1023) & ~uintptr_t(1023));
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t* bufs = smem + wib * 2 * FS_TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + FS_WARPS * 2 * FS_TILE_BYTES) + wib * 2;

  const int total_tiles = 2 * p.tiles_per_side;
  const int warp_global = blockIdx.x * FS_WARPS + wib;
  const int warp_stride = gridDim.x * FS_WARPS;

  if (lane == 0) {
    prefetch_tensormap(&map_k);
    prefetch_tensormap(&map_v);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncwarp();

  auto issue = [&](int tile, int b) {
    const int side = tile >= p.tiles_per_side;
    const int row0 = (side ? tile - p.tiles_per_side : tile) * FS_TILE_ROWS;
    const CUtensorMap* m = side ? &map_v : &map_k;
    uint8_t* dst = bufs + b * FS_TILE_BYTES;
    fence_proxy_async();
    mbar_expect_tx(&bars[b], FS_TILE_BYTES);
    tma_load_2d(dst, m, &bars[b], 0, row0);
    tma_load_2d(dst + 4096, m, &bars[b], 64, row0);
  };

  int tile = warp_global;
  if (tile < total_tiles && lane == 0) issue(tile, 0);
  uint32_t phase[2] = {0u, 0u};
  const double inv64 = 1.0 / sqrt((double)ORDER);

  for (int it = 0; tile < total_tiles; ++it, tile += warp_stride) {
    const int b = it & 1;
    const int next = tile + warp_stride;
    if (next < total_tiles && lane == 0) issue(next, b ^ 1);
    mbar_wait(&bars[b], phase[b]);
    phase[b] ^= 1u;
    const uint8_t* buf = bufs + b * FS_TILE_BYTES;

    const int side = tile >= p.tiles_per_side;
    const int64_t row = (int64_t)(side ? tile - p.tiles_per_side : tile) * FS_TILE_ROWS + lane;
    const bool rot = side ? p.rot_v : p.rot_k;
    bool valid = row < p.n_rows;
    int64_t slot = -1;
    if (valid) {
      slot = p.slots[row / p.pool.H];
      valid = slot >= 0;
    }

    // ---- stage the row: 16 x 16 B swizzled reads -> 64 packed words --------
    uint32_t w[64];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 q = *reinterpret_cast<const uint4*>(buf + h * 4096 + lane * 128 + ((c ^ (lane & 7)) << 4));
        w[h * 32 + c * 4 + 0] = q.x;
        w[h * 32 + c * 4 + 1] = q.y;
        w[h * 32 + c * 4 + 2] = q.z;
        w[h * 32 + c * 4 + 3] = q.w;
      }

    // ---- unpack (+ signs) and butterfly: v[j] = (y_{2j}, y_{2j+1}) -----------
    unsigned long long v[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      float e, o;
      unpack_pair<F16>(w[j], p.sgn_hi[j], p.sgn_lo[j], rot, e, o);
      v[j] = pk(e, o);
    }
    if (rot) {
      // stages half = 2 .. ORDER/2 act on (E_j, O_j) pairs vertically
#pragma unroll
      for (int hh = 1; hh < ORDER / 2; hh <<= 1) {
#pragma unroll
        for (int j = 0; j < 64; ++j) {
          if ((j & hh) == 0) {
            const unsigned long long a = v[j], c = v[j + hh];
            v[j] = add2(a, c);
            v[j + hh] = sub2(a, c);
          }
        }
      }
      // stage half = 1 pairs the two lanes of each f32x2
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        float e, o;
        upk(v[j], e, o);
        v[j] = pk(e + o, e - o);
      }
    }

    // ---- row extremes (NaN-propagating) --------------------------------------
    float mx0, mn0, mx1, mn1;
    {
      float a0, a1, b0, b1;
      upk(v[0], a0, a1);
      upk(v[1], b0, b1);
      mx0 = fmaxf(a0, a1);
      mn0 = fminf(a0, a1);
      mx1 = fmaxf(b0, b1);
      mn1 = fminf(b0, b1);
#pragma unroll
      for (int j = 2; j < 64; j += 2) {
        float x0, x1, y0, y1;
        upk(v[j], x0, x1);
        upk(v[j + 1], y0, y1);
        mx0 = max3_nan(mx0, x0, x1);
        mn0 = min3_nan(mn0, x0, x1);
        mx1 = max3_nan(mx1, y0, y1);
        mn1 = min3_nan(mn1, y0, y1);
      }
    }
    const float mxf = max3_nan(mx0, mx1, mx1), mnf = min3_nan(mn0, mn1, mn1);

    uint32_t packed[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) packed[i] = 0u;
    float scale_out = 0.f;
    uint32_t zp_out = 0;
    bool write = valid;
    if (valid && !(isfinite(mxf) && isfinite(mnf))) {
      if (p.flags) atomicOr(p.flags, (uint32_t)KVR_FLAG_NONFINITE);
      write = false;
    }
    // ---- row scale / zero point in f64, exactly as _ref.quantize_rows --------
    bool do_codes = false, clamp_row = false;
    double s64 = 1.0, z = 0.0, cst = 0.0;
    if (write) {
      const double scl = rot ? inv64 : 1.0;
      const double mx = (double)mxf * scl, mn = (double)mnf * scl;  // == fl64(S * inv) of the reference
      const float s32 = (float)((mx - mn) / 15.0);
      if (s32 == 0.0f) {
        scale_out = (float)mn;  // sentinel row: offset in the scale slot, zp 0xFF, codes 0
        zp_out = 0xFFu;
      } else {
        s64 = (double)s32;
        z = round_half_away(-mn / s64);
        z = z < 0.0 ? 0.0 : (z > 15.0 ? 15.0 : z);
        scale_out = s32;
        zp_out = (uint32_t)z;
        cst = scl / s64;
        const double ulo = mn * (1.0 / s64) + z + 0.5, uhi = mx * (1.0 / s64) + z + 0.5;
        // rows whose codes may leave [0, 15] (z clipped / boundary ties) clamp u first;
        // clamping is exact at both ends because floor-then-clip agrees on either side
        clamp_row = !((ulo > 1e-3) && (uhi < 16.0 - 1e-3));
        do_codes = true;
      }
    }
    const bool clamp = __any_sync(0xffffffffu, do_codes && clamp_row);
    if (do_codes) {
      // fixed-point code evaluation: U = floor((y*c + z + 1/2 (+-delta)) * 2^16) + 2^23
      if (!clamp) {
        const float cf = (float)(cst * (double)FS_FIX);
        const float bias = (float)((z + 0.5) * (double)FS_FIX) + FS_MAGIC;
        const unsigned long long c2 = pk(cf, cf);
        const unsigned long long bp = pk(bias + FS_D, bias + FS_D), bm = pk(bias - FS_D, bias - FS_D);
        uint32_t diff = 0u;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          uint32_t mp[8];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const unsigned long long up = fma2_rm(v[q * 4 + r], c2, bp);
            const unsigned long long um = fma2_rm(v[q * 4 + r], c2, bm);
            const uint32_t p0 = (uint32_t)up, p1 = (uint32_t)(up >> 32);
            diff |= (p0 ^ (uint32_t)um) | (p1 ^ (uint32_t)(um >> 32));
            mp[2 * r] = p0;
            mp[2 * r + 1] = p1;
          }
          packed[q] = prmt(pack4(mp[0], mp[1], mp[2], mp[3]), pack4(mp[4], mp[5], mp[6], mp[7]), 0x6420u);
        }
        if (diff & 0xFFFF0000u) {
          // rare: an element within delta of a rounding boundary -> reference-exact recomputation
#pragma unroll
          for (int j = 0; j < 64; ++j) {
            const unsigned long long up = fma2_rm(v[j], c2, bp);
            const unsigned long long um = fma2_rm(v[j], c2, bm);
            if (((uint32_t)up ^ (uint32_t)um) & 0xFFFF0000u) {
              const uint32_t code = exact_code<ORDER, F16>(buf, lane, 2 * j, rot, &signs, inv64, s64, z);
              const int sh = 4 * ((2 * j) & 7);
              packed[j >> 2] = (packed[j >> 2] & ~(0xFu << sh)) | (code << sh);
            }
            if (((uint32_t)(up >> 32) ^ (uint32_t)(um >> 32)) & 0xFFFF0000u) {
              const uint32_t code = exact_code<ORDER, F16>(buf, lane, 2 * j + 1, rot, &signs, inv64, s64, z);
              const int sh = 4 * ((2 * j + 1) & 7);
              packed[j >> 2] = (packed[j >> 2] & ~(0xFu << sh)) | (code << sh);
            }
          }
        }
      } else {
        // clamped variant: u in f32 (error <= 2^-20), clamp to [2^-13, 15.99] (both ends are
        // exact: floor-then-clip agrees on either side of 0 and 16), then the magic floor
        const float zb = (float)(z + 0.5), cu = (float)cst;
        const unsigned long long fix2 = pk(FS_FIX, FS_FIX);
        const unsigned long long mgp = pk(FS_MAGIC + FS_D, FS_MAGIC + FS_D), mgm = pk(FS_MAGIC - FS_D, FS_MAGIC - FS_D);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          uint32_t mp[8], mm[8];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            float a0, a1;
            upk(v[q * 4 + r], a0, a1);
            const float u0 = fminf(fmaxf(fmaf(a0, cu, zb), 1.0f / 8192.0f), 15.99f);
            const float u1 = fminf(fmaxf(fmaf(a1, cu, zb), 1.0f / 8192.0f), 15.99f);
            const unsigned long long uu = pk(u0, u1);
            const unsigned long long up = fma2_rm(uu, fix2, mgp);
            const unsigned long long um = fma2_rm(uu, fix2, mgm);
            mp[2 * r] = (uint32_t)up;
            mp[2 * r + 1] = (uint32_t)(up >> 32);
            mm[2 * r] = (uint32_t)um;
            mm[2 * r + 1] = (uint32_t)(um >> 32);
          }
          packed[q] = prmt(pack4(mp[0], mp[1], mp[2], mp[3]), pack4(mp[4], mp[5], mp[6], mp[7]), 0x6420u);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            if ((mp[e] ^ mm[e]) & 0xFFFF0000u) {
              const uint32_t code = exact_code<ORDER, F16>(buf, lane, 8 * q + e, rot, &signs, inv64, s64, z);
              packed[q] = (packed[q] & ~(0xFu << (4 * e))) | (code << (4 * e));
            }
          }
        }
      }
    }
    __syncwarp();  // every lane done with the staged tile -> buffer may be refilled

    if (write) {
      const Pool& pl = p.pool;
      const int head = (int)(row % pl.H);
      const int64_t page = slot / pl.P;
      const int sl = (int)(slot % pl.P);
      uint8_t* blob = pl.base + page * (int64_t)pl.page_bytes;
      const int idx = sl * pl.H + head;
      uint4* dst = reinterpret_cast<uint4*>(blob + (side ? pl.off_vp : pl.off_kp) + (int64_t)idx * 64);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
      reinterpret_cast<float*>(blob + (side ? pl.off_vs : pl.off_ks))[idx] = scale_out;
      blob[(side ? pl.off_vz : pl.off_kz) + idx] = (uint8_t)zp_out;
    }
  }
}

}  // namespace kvr

using namespace kvr;

template <int ORDER, bool F16>
static int launch_fast_impl(const void* k, const void* v, int64_t n_tok, const int64_t* slots, const Pool& pool,
                            int rot_k, int rot_v, const Signs& s, int has, uint32_t* flags, cudaStream_t st) {
  FastStoreParams prm{};
  prm.pool = pool;
  prm.slots = slots;
  prm.flags = flags;
  prm.n_rows = n_tok * pool.H;
  prm.tiles_per_side = (int)((prm.n_rows + FS_TILE_ROWS - 1) / FS_TILE_ROWS);
  prm.rot_k = rot_k;
  prm.rot_v = rot_v;
  for (int j = 0; j < 64; ++j) {
    const bool ne = has && ((s.w[(2 * j) >> 5] >> ((2 * j) & 31)) & 1u);
    const bool no = has && ((s.w[(2 * j + 1) >> 5] >> ((2 * j + 1) & 31)) & 1u);
    prm.sgn_lo[j] = ne ? 0x80000000u : 0u;
    prm.sgn_hi[j] = no ? 0x80000000u : 0u;
  }
  Signs sg = s;
  if (!has) for (auto& x : sg.w) x = 0u;
  CUtensorMap mk, mv;
  if (kvr_encode_tensor_map_2d(&mk, k, 128, (uint64_t)prm.n_rows, 256, 64, FS_TILE_ROWS,
                               CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return KVR_ERR_CUDA;
  if (kvr_encode_tensor_map_2d(&mv, v, 128, (uint64_t)prm.n_rows, 256, 64, FS_TILE_ROWS,
                               CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return KVR_ERR_CUDA;
  const size_t smem = FS_WARPS * 2 * FS_TILE_BYTES + FS_WARPS * 2 * sizeof(uint64_t) + 1024;
  auto kern = store_fast_kernel<ORDER, F16>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  const int total_tiles = 2 * prm.tiles_per_side;
  int grid = (total_tiles + FS_WARPS - 1) / FS_WARPS;
  const int cap = kvr_num_sms() * 3;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  kern<<<grid, FS_WARPS * 32, smem, st>>>(prm, mk, mv, sg);
  return 0;
}

int kvr_launch_store_fast(const void* k, const void* v, int in_dtype, int64_t n_tok, const int64_t* slots,
                          const Pool& pool, int order, int rot_k, int rot_v, const Signs& s, int has,
                          uint32_t* flags, cudaStream_t st) {
  if (pool.d != 128) return KVR_ERR_UNSUPPORTED;
  if (in_dtype != KVR_BF16 && in_dtype != KVR_F16) return KVR_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15) return KVR_ERR_UNSUPPORTED;
  if (!(rot_k || rot_v)) order = 128;  // plain twin: order is irrelevant
  const bool f16 = in_dtype == KVR_F16;
  switch (order) {
    case 128: return f16 ? launch_fast_impl<128, true>(k, v, n_tok, slots, pool, rot_k, rot_v, s, has, flags, st)
                         : launch_fast_impl<128, false>(k, v, n_tok, slots, pool, rot_k, rot_v, s, has, flags, st);
    case 64: return f16 ? launch_fast_impl<64, true>(k, v, n_tok, slots, pool, rot_k, rot_v, s, has, flags, st)
                        : launch_fast_impl<64, false>(k, v, n_tok, slots, pool, rot_k, rot_v, s, has, flags, st);
    case 32: return f16 ? launch_fast_impl<32, true>(k, v, n_tok, slots, pool, rot_k, rot_v, s, has, flags, st)
                        : launch_fast_impl<32, false>(k, v, n_tok, slots, pool, rot_k, rot_v, s, has, flags, st);
    case 16: return f16 ? launch_fast_impl<16, true>(k, v, n_tok, slots, pool, rot_k, rot_v, s, has, flags, st)
                        : launch_fast_impl<16, false>(k, v, n_tok, slots, pool, rot_k, rot_v, s, has, flags, st);
  }
  return KVR_ERR_UNSUPPORTED;
}
