// K1 -- fused block-Hadamard rotate -> token-wise INT4 quantize -> paged store,
// the serving-path bulk write for bf16/fp16 rows with head_dim 128.
//
// Reference semantics: cache.PageTable.append_token (cache.py:235-270) ->
// _rotate_token (cache.py:453-462) -> apply_block_rotation (rotation.py:118-142)
// -> _kernels.fwht_rows + quantize_rows (_ref.py:22-40, 57-80).
//
// Design (B200, sm_100a):
//  * persistent CTAs of 4 warps, 4 CTAs per SM; each warp streams 16-row tiles
//    (4 KB) through a private double buffer filled by TMA (cp.async.bulk.tensor.2d,
//    SWIZZLE_128B: conflict-free half-row-per-thread shared-memory reads);
//  * a lane pair owns one 128-element row, 64 elements each in registers: sign
//    flip + bf16 unpack fused with the first butterfly stage, stages up to half 32
//    as f32x2 (FADD2), the half-64 stage across the pair (64 shuffles), NaN-
//    propagating 3-input min/max (FMNMX3.NAN) combined across the pair;
//  * the row scale / zero point are formed in f64 exactly as the reference does,
//    from the fp32 butterfly's extreme values;
//  * codes: one FFMA2.RM per element pair evaluates floor((t + z + 1/2) * 2^16)
//    as a fixed-point integer (magic 2^23), twice (+-delta) -- if both agree on
//    the integer part the nibble is the reference's round-half-away code for this
//    y; a row with an element within delta of a half step is recomputed in f64
//    from the bf16 inputs with the reference's butterfly order, warp-cooperatively
//    (warp_exact_row), and its flagged 8-code groups are replaced.  Unrotated
//    (plain) rows hold y exactly, so their flagged groups are fixed in-thread by
//    exact FMA sign tests against the rounding boundaries instead;
//  * 8 nibbles are packed with 3 PRMT + 1 IMAD.HI per 4 codes.
#include "kvr_common.cuh"
#include "kvr_internal.h"

namespace kvr {

constexpr int FS_WARPS = 4;
#ifndef KVR_FS_MINB
#define KVR_FS_MINB 4
#endif
constexpr int FS_TILE_ROWS = 16;
constexpr int FS_SUB_BYTES = FS_TILE_ROWS * 128;    // one 64-element half of the tile's rows
constexpr int FS_TILE_BYTES = FS_TILE_ROWS * 256;  // 128 x 16-bit per row
constexpr float FS_MAGIC = 8388608.0f;            // 2^23
constexpr float FS_FIX = 65536.0f;                // 16 fraction bits
// +-delta of the boundary test in units of 2^-16 of u = y c + z + 1/2: the
// magic-number floor works at 2^23 <= U < 2^24, where one unit is the f32 ulp.
constexpr float FS_D = 1.0f;
constexpr float FS_D_CLAMP = 1.0f;

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

template <bool F16, bool ROT>
KVR_DEV void unpack_pair(uint32_t w, uint32_t s_hi, uint32_t s_lo, float& e, float& o) {
  if constexpr (!F16) {
    // bf16 pair -> two f32 (exact); the sign flip is folded into the same ops
    e = __uint_as_float(ROT ? (w << 16) + s_lo : (w << 16));
    o = __uint_as_float(ROT ? ((w ^ s_hi) & 0xFFFF0000u) : (w & 0xFFFF0000u));
  } else {
    const uint32_t ws = ROT ? (w ^ ((s_lo >> 16) | s_hi)) : w;
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&ws));
    e = f.x;
    o = f.y;
  }
}

// Elements 4l..4l+3 of the row staged for lane `src` in the swizzled tile, as f64.
template <bool F16>
KVR_DEV void tile_quad(const uint8_t* buf, int src, int l, double (&x)[4]) {
  const int e = 4 * l;
  const int h = e >> 6, c = (e >> 3) & 7, within = e & 7;
  const uint2 q = *reinterpret_cast<const uint2*>(buf + h * FS_SUB_BYTES + src * 128 + ((c ^ (src & 7)) << 4) + within * 2);
  const uint32_t w[2] = {q.x, q.y};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t bits = (u & 1) ? (w[u >> 1] >> 16) : (w[u >> 1] & 0xFFFFu);
    if constexpr (F16) x[u] = (double)__half2float(__ushort_as_half((unsigned short)bits));
    else x[u] = (double)__uint_as_float(bits << 16);
  }
}

// Reference-exact codes of the row staged for lane `src`, computed by the whole
// warp: lane l owns elements 4l..4l+3; f64 butterfly in _ref.fwht_rows order
// (stages half = 1, 2 in registers, 4..ORDER/2 by shuffles, lowest index first),
// * 1/sqrt(ORDER), then round-half-away(y / s64) + z, clip (_ref.py:22-40, 57-80).
// Returns the 4 codes of lane l as a 16-bit group (element 4l in the low nibble).
template <int ORDER, bool F16, bool ROT>
__device__ __noinline__ uint32_t warp_exact_row(const uint8_t* buf, int src, const Signs& sg, double s64, double z) {
  const int lane = threadIdx.x & 31;
  double x[4];
  tile_quad<F16>(buf, src, lane, x);
  if constexpr (ROT) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (sign_bit(sg, 4 * lane + u)) x[u] = x[u] * -1.0;
    const double a0 = x[0] + x[1], a1 = x[0] - x[1], a2 = x[2] + x[3], a3 = x[2] - x[3];  // half = 1
    x[0] = a0 + a2;                                                                     // half = 2
    x[1] = a1 + a3;
    x[2] = a0 - a2;
    x[3] = a1 - a3;
#pragma unroll
    for (int k = 0; (4 << k) < ORDER; ++k) {
      const bool upper = (lane >> k) & 1;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double o = __shfl_xor_sync(0xffffffffu, x[u], 1 << k);
        x[u] = upper ? o - x[u] : x[u] + o;
      }
    }
    const double inv = 1.0 / sqrt((double)ORDER);
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = x[u] * inv;
  }
  uint32_t g = 0u;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    double q = round_half_away(x[u] / s64) + z;
    q = q < 0.0 ? 0.0 : (q > 15.0 ? 15.0 : q);
    g |= (uint32_t)q << (4 * u);
  }
  return g;
}

KVR_DEV uint32_t pack4(uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
  // codes sit in byte 2 of each magic-floored value
  const uint32_t c = prmt(prmt(m0, m1, 0x0062u), prmt(m2, m3, 0x0062u), 0x5410u);  // [k0,k1,k2,k3]
  return __umulhi(c, 1u << 28) + c;  // c | c >> 4: bytes 0 and 2 hold k0|k1<<4, k2|k3<<4
}

// Exact reference code of a plain (unrotated) element: y is x itself (exact in
// f32) and s = f32 scale, so round_half_away(x / s64) is decided by the signs of
// x - (m -+ 1/2) s, each evaluated with one rounding (FMA) and hence exact.
KVR_DEV uint32_t plain_code_exact(float x, float s, float inv, float z) {
  const float ax = fabsf(x);
  float m = floorf(fmaf(ax, inv, 0.5f));
  if (fmaf(-(m - 0.5f), s, ax) < 0.f) m -= 1.f;
  else if (fmaf(-(m + 0.5f), s, ax) >= 0.f) m += 1.f;
  const float q = fminf(fmaxf(copysignf(m, x) + z, 0.f), 15.f);
  return (uint32_t)q;
}

// Quantize the half row (64 elements, half `hf`) this lane shares with lane ^ 1:
// its 32 packed code bytes, the row scale and zero point; returns the write flag.
template <int ORDER, bool F16, bool ROT>
KVR_DEV bool half_row_codes(const uint8_t* buf, int row, int hf, const FastStoreParams& p, const Signs& signs,
                            bool valid, uint32_t (&packed)[8], float& scale_out, uint32_t& zp_out) {
  const int lane = threadIdx.x & 31;
  // ---- stage the half row: 8 x 16 B swizzled reads; unpack fused with stage half = 1
  unsigned long long v[32];  // v[j] = (y_{2j}, y_{2j+1}) of this half
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 q = *reinterpret_cast<const uint4*>(buf + hf * FS_SUB_BYTES + row * 128 + ((c ^ (row & 7)) << 4));
    const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = c * 4 + u;
      float e, o;
      unpack_pair<F16, ROT>(w4[u], p.sgn_hi[32 * hf + j], p.sgn_lo[32 * hf + j], e, o);
      v[j] = ROT ? pk(e + o, e - o) : pk(e, o);
    }
  }
  if constexpr (ROT) {
    // stages half = 2 .. min(ORDER/2, 32) inside the half: pairs (j, j + hh) of (y_{2j}, y_{2j+1})
#pragma unroll
    for (int hh = 1; hh < ORDER / 2 && hh < 32; hh <<= 1) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if ((j & hh) == 0) {
          const unsigned long long a = v[j], c = v[j + hh];
          v[j] = add2(a, c);
          v[j + hh] = sub2(a, c);
        }
      }
    }
    if constexpr (ORDER == 128) {
      // stage half = 64 across the lane pair: y_j = a_j + b_j (half 0), a_j - b_j (half 1)
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float x0, x1;
        upk(v[j], x0, x1);
        const float o0 = __shfl_xor_sync(0xffffffffu, x0, 1), o1 = __shfl_xor_sync(0xffffffffu, x1, 1);
        v[j] = hf ? sub2(pk(o0, o1), v[j]) : add2(v[j], pk(o0, o1));
      }
    }
  }
  // ---- row extremes (NaN-propagating), combined across the pair
  float mxf, mnf;
  {
    float mx0, mn0, mx1, mn1, a0, a1, b0, b1;
    upk(v[0], a0, a1);
    upk(v[1], b0, b1);
    mx0 = max3_nan(a0, a1, a1);
    mn0 = min3_nan(a0, a1, a1);
    mx1 = max3_nan(b0, b1, b1);
    mn1 = min3_nan(b0, b1, b1);
#pragma unroll
    for (int j = 2; j < 32; j += 2) {
      float x0, x1, y0, y1;
      upk(v[j], x0, x1);
      upk(v[j + 1], y0, y1);
      mx0 = max3_nan(mx0, x0, x1);
      mn0 = min3_nan(mn0, x0, x1);
      mx1 = max3_nan(mx1, y0, y1);
      mn1 = min3_nan(mn1, y0, y1);
    }
    const float mxh = max3_nan(mx0, mx1, mx1), mnh = min3_nan(mn0, mn1, mn1);
    mxf = max3_nan(mxh, __shfl_xor_sync(0xffffffffu, mxh, 1), mxh);
    mnf = min3_nan(mnh, __shfl_xor_sync(0xffffffffu, mnh, 1), mnh);
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) packed[i] = 0u;
  scale_out = 0.f;
  zp_out = 0u;
  bool write = valid;
  if (valid && !(isfinite(mxf) && isfinite(mnf))) {
    if (p.flags && hf == 0) atomicOr(p.flags, (uint32_t)KVR_FLAG_NONFINITE);
    write = false;
  }
  // ---- row scale / zero point in f64, exactly as _ref.quantize_rows
  const double inv64 = 1.0 / sqrt((double)ORDER);
  bool do_codes = false, clamp_row = false;
  double s64 = 1.0, z = 0.0, cst = 0.0;
  float s32 = 0.f;
  if (write) {
    const double scl = ROT ? inv64 : 1.0;
    const double mx = (double)mxf * scl, mn = (double)mnf * scl;  // == fl64(S * inv) of the reference
    s32 = (float)((mx - mn) / 15.0);
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
  uint32_t gflags = 0u;  // bit q: an element of 8q..8q+7 (of this half) is within delta of a boundary
  if (do_codes) {
    if (!clamp) {
      // U = floor((y*c + z + 1/2 (+-delta)) * 2^16) + 2^23, one FFMA2.RM per pair and sign
      const float cf = (float)(cst * (double)FS_FIX);
      const float bias = (float)((z + 0.5) * (double)FS_FIX) + FS_MAGIC;
      const unsigned long long c2 = pk(cf, cf);
      const unsigned long long bp = pk(bias + FS_D, bias + FS_D), bm = pk(bias - FS_D, bias - FS_D);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t mp[8], dq = 0u;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const unsigned long long up = fma2_rm(v[q * 4 + r], c2, bp);
          const unsigned long long um = fma2_rm(v[q * 4 + r], c2, bm);
          const uint32_t p0 = (uint32_t)up, p1 = (uint32_t)(up >> 32);
          dq |= (p0 ^ (uint32_t)um) | (p1 ^ (uint32_t)(um >> 32));
          mp[2 * r] = p0;
          mp[2 * r + 1] = p1;
        }
        packed[q] = prmt(pack4(mp[0], mp[1], mp[2], mp[3]), pack4(mp[4], mp[5], mp[6], mp[7]), 0x6420u);
        gflags |= (dq >= 0x10000u ? 1u : 0u) << q;
      }
    } else {
      // clamped variant: u in f32 (error <= 2^-20), clamped to [2^-13, 15.99], then the magic floor
      const float zb = (float)(z + 0.5), cu = (float)cst;
      const unsigned long long fix2 = pk(FS_FIX, FS_FIX);
      const unsigned long long mgp = pk(FS_MAGIC + FS_D_CLAMP, FS_MAGIC + FS_D_CLAMP),
                               mgm = pk(FS_MAGIC - FS_D_CLAMP, FS_MAGIC - FS_D_CLAMP);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t mp[8], dq = 0u;
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
          dq |= ((uint32_t)up ^ (uint32_t)um) | ((uint32_t)(up >> 32) ^ (uint32_t)(um >> 32));
        }
        packed[q] = prmt(pack4(mp[0], mp[1], mp[2], mp[3]), pack4(mp[4], mp[5], mp[6], mp[7]), 0x6420u);
        gflags |= (dq >= 0x10000u ? 1u : 0u) << q;
      }
    }
  }
  if constexpr (!ROT) {
    // plain rows: exact in-thread fix of the flagged groups
    if (gflags) {
      const float inv = 1.0f / s32, zf = (float)z;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if ((gflags >> q) & 1u) {
          uint32_t w = 0u;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            float a0, a1;
            upk(v[q * 4 + r], a0, a1);
            w |= plain_code_exact(a0, s32, inv, zf) << (8 * r);
            w |= plain_code_exact(a1, s32, inv, zf) << (8 * r + 4);
          }
          packed[q] = w;
        }
      }
    }
  } else {
    // ---- rare: reference-exact recomputation of flagged rows, warp-cooperative
    uint32_t todo = __ballot_sync(0xffffffffu, gflags != 0u);
    while (todo) {
      const int src = __ffs(todo) - 1;  // lane src: half (src & 1) of tile row 16 pass + src / 2
      todo &= todo - 1;
      const uint32_t gf = __shfl_sync(0xffffffffu, gflags, src);
      const double sb = __shfl_sync(0xffffffffu, s64, src), zb = __shfl_sync(0xffffffffu, z, src);
      const int srow = __shfl_sync(0xffffffffu, row, src);
      const uint32_t g16 = warp_exact_row<ORDER, F16, ROT>(buf, srow, signs, sb, zb);
      const int hb = (src & 1) * 8;  // the half's groups are row groups hb .. hb + 7
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if ((gf >> q) & 1u) {  // warp-uniform
          const uint32_t lo = __shfl_sync(0xffffffffu, g16, 2 * (hb + q)),
                         hi = __shfl_sync(0xffffffffu, g16, 2 * (hb + q) + 1);
          if (lane == src) packed[q] = lo | (hi << 16);
        }
      }
    }
  }
  return write;
}

template <int ORDER, bool F16>
__global__ void __launch_bounds__(FS_WARPS * 32, KVR_FS_MINB)
    store_fast_kernel(const __grid_constant__ FastStoreParams p, const __grid_constant__ CUtensorMap map_k,
                      const __grid_constant__ CUtensorMap map_v, const __grid_constant__ Signs signs) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t* bufs = smem + wib * 2 * FS_TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + FS_WARPS * 2 * FS_TILE_BYTES) + wib * 2;

  const int total_tiles = 2 * p.tiles_per_side;
  const int warp_stride = gridDim.x * FS_WARPS;
  const int H = p.pool.H;
  const int trow = lane >> 1, hf = lane & 1;  // this lane: half hf of tile row trow

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
    tma_load_2d(dst + FS_SUB_BYTES, m, &bars[b], 64, row0);
  };
  auto row_of = [&](int tile) -> int64_t {
    const int side = tile >= p.tiles_per_side;
    return (int64_t)(side ? tile - p.tiles_per_side : tile) * FS_TILE_ROWS + trow;
  };
  auto slot_of = [&](int tile) -> int64_t {  // slot id of this lane's row (or -1)
    if (tile >= total_tiles) return -1;
    const int64_t row = row_of(tile);
    return row < p.n_rows ? __ldg(&p.slots[row / H]) : -1;
  };

  int tile = blockIdx.x * FS_WARPS + wib;
  if (tile < total_tiles && lane == 0) issue(tile, 0);
  uint32_t phase[2] = {0u, 0u};
  int64_t slot_cur = slot_of(tile);

  for (int it = 0; tile < total_tiles; ++it, tile += warp_stride) {
    const int b = it & 1;
    const int next = tile + warp_stride;
    if (next < total_tiles && lane == 0) issue(next, b ^ 1);
    const int64_t slot = slot_cur;
    slot_cur = slot_of(next);  // prefetch: consumed one tile later
    mbar_wait(&bars[b], phase[b]);
    phase[b] ^= 1u;
    const uint8_t* buf = bufs + b * FS_TILE_BYTES;
    const int side = tile >= p.tiles_per_side;
    const int64_t row = row_of(tile);
    const bool valid = row < p.n_rows;  // codes are computed whatever the slot; the store is predicated

    uint32_t packed[8];
    float scale_out;
    uint32_t zp_out;
    bool write;
    if (side ? p.rot_v : p.rot_k)  // warp-uniform
      write = half_row_codes<ORDER, F16, true>(buf, trow, hf, p, signs, valid, packed, scale_out, zp_out);
    else
      write = half_row_codes<128, F16, false>(buf, trow, hf, p, signs, valid, packed, scale_out, zp_out);
    __syncwarp();  // every lane done with the staged tile -> buffer may be refilled

    if (write && slot >= 0) {
      const Pool& pl = p.pool;
      const int head = (int)(row % H);
      int ci;
      uint8_t* cell = cell_of(pl, slot / pl.P, head, (int)(slot % pl.P), ci);
      uint4* dst = reinterpret_cast<uint4*>(cell + (side ? cell_vcode(pl, ci) : cell_kcode(pl, ci)) + 32 * hf);
      dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
      if (hf == 0) {
        *reinterpret_cast<float*>(cell + (side ? cell_vscale(pl, ci) : cell_kscale(pl, ci))) = scale_out;
        cell[side ? cell_vzp(pl, ci) : cell_kzp(pl, ci)] = (uint8_t)zp_out;
      }
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
  const int cap = kvr_num_sms() * KVR_FS_MINB;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  kern<<<grid, FS_WARPS * 32, smem, st>>>(prm, mk, mv, sg);
  return 0;
}

int kvr_launch_store_fast(const void* k, const void* v, int in_dtype, int64_t n_tok, const int64_t* slots,
                          const Pool& pool, int order, int rot_k, int rot_v, const Signs& s, int has,
                          uint32_t* flags, cudaStream_t st) {
  if (pool.d != 128 || (pool.T & 1)) return KVR_ERR_UNSUPPORTED;  // 16-B aligned code rows
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
