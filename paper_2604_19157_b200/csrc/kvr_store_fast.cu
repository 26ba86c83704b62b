// K1 -- fused block-Hadamard rotate -> token-wise INT4 quantize -> paged store,
// the serving-path bulk write for bf16/fp16 rows with head_dim 128.
//
// Reference semantics: cache.PageTable.append_token (cache.py:235-270) ->
// _rotate_token (cache.py:453-462) -> apply_block_rotation (rotation.py:118-142)
// -> _kernels.fwht_rows + quantize_rows (_ref.py:22-40, 57-80).
//
// Design (B200, sm_100a): see store_mma_kernel below -- H_128 = H_8 (x) H_16 with
// H_16 on the tensor cores (bf16/fp16 HMMA, +-1 weights), H_8 as lane-local FADD2
// stages, the reference's f64 row scale / zero point, codes by FFMA2.RM with a
// +-delta boundary test and an exact recomputation of flagged rows.
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
  int32_t log2P;        // page_tokens = 2^log2P (tensor-core path)
};

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
      const double sgn = ((lane >> k) & 1) ? -1.0 : 1.0;  // upper half of the pair: o - x
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double o = __shfl_xor_sync(0xffffffffu, x[u], 1 << k);
        x[u] = fma(sgn, x[u], o);  // o -+ x, one rounding
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

// ---------------------------------------------------------------------------
// K1 on the tensor cores.  H_ORDER = H_{ORDER/16} (x) H_16 (Sylvester order): a
// warp-tile of 16 rows is multiplied by H_16 per 16-column block with
// mma.sync m16n8k16 (bf16/fp16 inputs, +-1 weights: exact products, fp32
// accumulation), the sign flip is an XOR on the A fragments, and the remaining
// stages across blocks are lane-local FADD2s (every lane holds the same
// (row, column-in-block) positions of all 8 blocks).  Lane (g, t) then owns rows
// g and g + 8, columns 16 b + 8 nn + 2 t (+ 1): code byte t + 4 (2 b + nn).
// Bytes go to a padded shared-memory staging row and leave as 16-B stores.
constexpr int MS_ROW = 80;                        // staging pitch: 16-B aligned, STS.U8 conflict-free
constexpr int MS_STAGE = FS_TILE_ROWS * MS_ROW;   // per warp

KVR_DEV void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
template <bool F16>
KVR_DEV void mma_h16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (F16)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  else
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <bool F16>
KVR_DEV float2 b16x2_to_f2(uint32_t w) {
  if constexpr (F16) return __half22float2(*reinterpret_cast<const __half2*>(&w));
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}

// Row scale / zero point (f64, _ref.quantize_rows) and the fast-code constants.
struct RowQ {
  double s64, z;
  float s32, cf, bias, zb, cu;  // bias / zb, cu: plain and clamped code constants
  bool codes, clamp;            // codes: a regular (non-sentinel, finite, valid) row
  float scale_out;
  uint32_t zp_out;
};
KVR_DEV RowQ row_quant(float mxf, float mnf, double scl, bool valid) {
  RowQ q{};
  q.s64 = 1.0;
  if (!valid) return q;
  const double mx = (double)mxf * scl, mn = (double)mnf * scl;
  const float s32 = (float)((mx - mn) / 15.0);
  q.s32 = s32;
  if (s32 == 0.0f) {
    q.scale_out = (float)mn;  // sentinel row: offset in the scale slot, zp 0xFF, codes 0
    q.zp_out = 0xFFu;
    return q;
  }
  q.s64 = (double)s32;
  double z = round_half_away(-mn / q.s64);
  z = z < 0.0 ? 0.0 : (z > 15.0 ? 15.0 : z);
  q.z = z;
  q.scale_out = s32;
  q.zp_out = (uint32_t)z;
  // fast-code constants in f32: c = scl / s to 2^-23 relative (|u| <= 16 -> 2^-19 of a
  // code step, inside the +-2^-16 boundary test)
  const float cst = (float)scl / s32;
  q.cf = cst * FS_FIX;
  q.bias = (float)((z + 0.5) * (double)FS_FIX) + FS_MAGIC;
  q.zb = (float)(z + 0.5);
  q.cu = cst;
  const float ulo = (float)mn / s32 + q.zb, uhi = (float)mx / s32 + q.zb;
  q.clamp = !((ulo > 2e-3f) && (uhi < 16.0f - 2e-3f));
  q.codes = true;
  return q;
}

// One 16-row tile (rows row0 .. row0 + 15 of one side) through the tensor-core K1.
template <int ORDER, bool F16, bool ROT>
KVR_DEV void mma_tile(const uint8_t* buf, uint8_t* stage, const uint2* smask, const FastStoreParams& p,
                      const Signs& signs, const uint32_t (&bh)[2][2], int64_t row0, int side,
                      const int64_t (&slot)[2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int lrow = (lane & 7) + 8 * ((lane >> 3) & 1), lcol = lane >> 4;
  const uint32_t abase = smem_u32(buf) + lrow * 128;
  // ---- y = x diag(s) H per 16-column block on the tensor cores (x itself for plain rows)
  unsigned long long v[8][2][2];  // [block][n-tile][row g | g + 8] = (col 2t, 2t + 1)
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const int c = (2 * (b & 3) + lcol) ^ (lrow & 7);
    uint32_t a[4];
    ldsm_x4(abase + (b >> 2) * FS_SUB_BYTES + (c << 4), a);
    if constexpr (ROT) {
      // sign flips of this lane's elements (cols 16 b + 2 t (+1), and + 8): one XOR each
      const uint2 m = smask[b * 4 + t];
      a[0] ^= m.x;
      a[1] ^= m.x;
      a[2] ^= m.y;
      a[3] ^= m.y;
      float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
      mma_h16<F16>(d0, a, bh[0][0], bh[0][1]);
      mma_h16<F16>(d1, a, bh[1][0], bh[1][1]);
      v[b][0][0] = pk(d0[0], d0[1]);
      v[b][0][1] = pk(d0[2], d0[3]);
      v[b][1][0] = pk(d1[0], d1[1]);
      v[b][1][1] = pk(d1[2], d1[3]);
    } else {
      const float2 x0 = b16x2_to_f2<F16>(a[0]), x1 = b16x2_to_f2<F16>(a[1]);
      const float2 x2 = b16x2_to_f2<F16>(a[2]), x3 = b16x2_to_f2<F16>(a[3]);
      v[b][0][0] = pk(x0.x, x0.y);
      v[b][0][1] = pk(x1.x, x1.y);
      v[b][1][0] = pk(x2.x, x2.y);
      v[b][1][1] = pk(x3.x, x3.y);
    }
  }
  if constexpr (ROT) {  // stages half = 16, 32, 64 (< ORDER) across blocks
#pragma unroll
    for (int h = 1; h < 8 && 16 * h < ORDER; h <<= 1)
#pragma unroll
      for (int b = 0; b < 8; ++b)
        if ((b & h) == 0)
#pragma unroll
          for (int nn = 0; nn < 2; ++nn)
#pragma unroll
            for (int rh = 0; rh < 2; ++rh) {
              const unsigned long long x = v[b][nn][rh], y = v[b + h][nn][rh];
              v[b][nn][rh] = add2(x, y);
              v[b + h][nn][rh] = sub2(x, y);
            }
  }

  // ---- row extremes (NaN-propagating), across the 4 lanes of a row
  bool wr[2];
  float rmx[2], rmn[2];
#pragma unroll
  for (int rh = 0; rh < 2; ++rh) {
    float mx, mn, a0, a1;
    upk(v[0][0][rh], a0, a1);
    mx = max3_nan(a0, a1, a1);
    mn = min3_nan(a0, a1, a1);
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      upk(v[k >> 1][k & 1][rh], a0, a1);
      mx = max3_nan(mx, a0, a1);
      mn = min3_nan(mn, a0, a1);
    }
    mx = max3_nan(mx, __shfl_xor_sync(0xffffffffu, mx, 1), __shfl_xor_sync(0xffffffffu, mx, 2));
    mn = min3_nan(mn, __shfl_xor_sync(0xffffffffu, mn, 1), __shfl_xor_sync(0xffffffffu, mn, 2));
    mx = max3_nan(mx, __shfl_xor_sync(0xffffffffu, mx, 1), mx);
    mn = min3_nan(mn, __shfl_xor_sync(0xffffffffu, mn, 1), mn);
    const bool valid = row0 + g + 8 * rh < p.n_rows;
    const bool fin = isfinite(mx) && isfinite(mn);
    if (valid && !fin && t == 0 && p.flags) atomicOr(p.flags, (uint32_t)KVR_FLAG_NONFINITE);
    wr[rh] = valid && fin;
    rmx[rh] = mx;
    rmn[rh] = mn;
  }
  // the row parameters (two f64 divisions) once per row: lane t < 2 of a row group
  // computes row g + 8 t, the group takes both rows by shuffles
  const double scl = ROT ? 1.0 / sqrt((double)ORDER) : 1.0;
  RowQ rq[2];
  {
    const int mine = t & 1;
    const RowQ own = row_quant(rmx[mine], rmn[mine], scl, wr[mine]);
#pragma unroll
    for (int rh = 0; rh < 2; ++rh) {
      const int src = 4 * g + rh;
      RowQ& q = rq[rh];
      q.s64 = __shfl_sync(0xffffffffu, own.s64, src);
      q.z = __shfl_sync(0xffffffffu, own.z, src);
      q.s32 = __shfl_sync(0xffffffffu, own.s32, src);
      q.cf = __shfl_sync(0xffffffffu, own.cf, src);
      q.bias = __shfl_sync(0xffffffffu, own.bias, src);
      q.zb = __shfl_sync(0xffffffffu, own.zb, src);
      q.cu = __shfl_sync(0xffffffffu, own.cu, src);
      q.scale_out = __shfl_sync(0xffffffffu, own.scale_out, src);
      const uint32_t bits =
          __shfl_sync(0xffffffffu, own.zp_out | (own.codes ? 0x100u : 0u) | (own.clamp ? 0x200u : 0u), src);
      q.zp_out = bits & 0xFFu;
      q.codes = (bits >> 8) & 1u;
      q.clamp = (bits >> 9) & 1u;
    }
  }
  const bool clamp = __any_sync(0xffffffffu, (rq[0].codes && rq[0].clamp) || (rq[1].codes && rq[1].clamp));

  // ---- codes into the staging rows (branch-free per byte; rows without codes get
  // c = 0, bias = 2^23 -> code 0, no flags); flagged bytes are fixed below
  uint32_t fl[2] = {0u, 0u};
#pragma unroll
  for (int rh = 0; rh < 2; ++rh) {
    uint8_t* srow = stage + (g + 8 * rh) * MS_ROW + t;
    const bool cd = rq[rh].codes;
    if (!clamp) {  // warp-uniform
      // rows without codes: u = 1/2 (mid-step, never near a boundary), code 0
      const float cfv = cd ? rq[rh].cf : 0.f, bias = cd ? rq[rh].bias : FS_MAGIC + 0.5f * FS_FIX;
      const unsigned long long c2 = pk(cfv, cfv);
      const unsigned long long bp = pk(bias + FS_D, bias + FS_D), bm = pk(bias - FS_D, bias - FS_D);
#pragma unroll
      for (int k = 0; k < 16; k += 2) {
        const unsigned long long upa = fma2_rm(v[k >> 1][0][rh], c2, bp), uma = fma2_rm(v[k >> 1][0][rh], c2, bm);
        const unsigned long long upb = fma2_rm(v[k >> 1][1][rh], c2, bp), umb = fma2_rm(v[k >> 1][1][rh], c2, bm);
        const uint32_t m0 = (uint32_t)upa, m1 = (uint32_t)(upa >> 32), m2 = (uint32_t)upb, m3 = (uint32_t)(upb >> 32);
        const uint32_t da = (m0 ^ (uint32_t)uma) | (m1 ^ (uint32_t)(uma >> 32));
        const uint32_t db = (m2 ^ (uint32_t)umb) | (m3 ^ (uint32_t)(umb >> 32));
        if constexpr (ROT) {
          fl[rh] |= da | db;  // row-level: bits >= 16 set <=> a code is within delta of a boundary
        } else {
          fl[rh] |= ((da >= 0x10000u ? 1u : 0u) | (db >= 0x10000u ? 2u : 0u)) << k;
        }
        const uint32_t two = pack4(m0, m1, m2, m3);  // byte 0: code byte k, byte 2: k + 1
        srow[4 * k] = (uint8_t)two;
        srow[4 * k + 4] = (uint8_t)(two >> 16);
      }
    } else {  // clamped variant: u in f32 clamped to [2^-13, 15.99], then the magic floor
      const float cu = cd ? rq[rh].cu : 0.f, zb = cd ? rq[rh].zb : 1.0f / 8192.0f;
      const unsigned long long fix2 = pk(FS_FIX, FS_FIX);
      const unsigned long long mgp = pk(FS_MAGIC + FS_D_CLAMP, FS_MAGIC + FS_D_CLAMP);
      const unsigned long long mgm = pk(FS_MAGIC - FS_D_CLAMP, FS_MAGIC - FS_D_CLAMP);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        float a0, a1;
        upk(v[k >> 1][k & 1][rh], a0, a1);
        const float u0 = fminf(fmaxf(fmaf(a0, cu, zb), 1.0f / 8192.0f), 15.99f);
        const float u1 = fminf(fmaxf(fmaf(a1, cu, zb), 1.0f / 8192.0f), 15.99f);
        const unsigned long long uu = pk(u0, u1);
        const unsigned long long up = fma2_rm(uu, fix2, mgp), um = fma2_rm(uu, fix2, mgm);
        const uint32_t m0 = (uint32_t)up, m1 = (uint32_t)(up >> 32);
        const uint32_t d = (m0 ^ (uint32_t)um) | (m1 ^ (uint32_t)(um >> 32));
        if constexpr (ROT) {
          fl[rh] |= cd ? d : 0u;
        } else {
          fl[rh] |= (cd && d >= 0x10000u ? 1u : 0u) << k;
        }
        srow[4 * k] = (uint8_t)(((m0 >> 16) & 15u) | ((m1 >> 12) & 0xF0u));
      }
    }
  }
  if constexpr (!ROT) {
    if (__any_sync(0xffffffffu, (fl[0] | fl[1]) != 0u)) {
      // plain rows: y = x exactly -> the flagged bytes by exact FMA sign tests, in-thread
#pragma unroll
      for (int rh = 0; rh < 2; ++rh) {
        uint8_t* srow = stage + (g + 8 * rh) * MS_ROW + t;
        const float inv = 1.0f / rq[rh].s32, zf = (float)rq[rh].z;
#pragma unroll
        for (int k = 0; k < 16; ++k) {  // static indices keep v[] in registers
          if (!((fl[rh] >> k) & 1u)) continue;
          float a0, a1;
          upk(v[k >> 1][k & 1][rh], a0, a1);
          srow[4 * k] = (uint8_t)(plain_code_exact(a0, rq[rh].s32, inv, zf) |
                                  (plain_code_exact(a1, rq[rh].s32, inv, zf) << 4));
        }
      }
    }
  } else {
    // ---- rare (rotated rows): reference-exact recomputation of flagged rows, warp-cooperative
#pragma unroll
    for (int rh = 0; rh < 2; ++rh) {
      fl[rh] = fl[rh] >= 0x10000u ? 0xFFFFu : 0u;  // the whole row is rewritten
      fl[rh] |= __shfl_xor_sync(0xffffffffu, fl[rh], 1);
      fl[rh] |= __shfl_xor_sync(0xffffffffu, fl[rh], 2);
    }
    uint32_t todo = __ballot_sync(0xffffffffu, t == 0 && (fl[0] | fl[1]) != 0u);
    while (todo) {
      const int src = __ffs(todo) - 1;  // lane 4 g' of row pair (g', g' + 8)
      todo &= todo - 1;
#pragma unroll
      for (int rh = 0; rh < 2; ++rh) {
        const uint32_t gf = __shfl_sync(0xffffffffu, fl[rh], src);
        if (gf == 0u) continue;  // warp-uniform
        const double sb = __shfl_sync(0xffffffffu, rq[rh].s64, src), zb = __shfl_sync(0xffffffffu, rq[rh].z, src);
        const int r = (src >> 2) + 8 * rh;
        const uint32_t g16 = warp_exact_row<ORDER, F16, true>(buf, r, signs, sb, zb);
        // lane l holds the codes of elements 4l..4l+3 = bytes 2l, 2l+1 = half of group l / 2
        if ((gf >> (lane >> 1)) & 1u) *reinterpret_cast<uint16_t*>(stage + r * MS_ROW + 2 * lane) = (uint16_t)g16;
      }
    }
  }
  __syncwarp();

  // ---- write-out: lane (g, t) stores 16-B part t of rows g and g + 8, lane t == 0 the sidecars
  const Pool& pl = p.pool;
#pragma unroll
  for (int rh = 0; rh < 2; ++rh) {
    if (!(wr[rh] && slot[rh] >= 0)) continue;
    const int row = (int)(row0 + g + 8 * rh);
    const int head = row % pl.H;
    const int64_t page = slot[rh] >> p.log2P;
    const int ci = (int)(slot[rh] & (pl.P - 1)) & 15;
    uint8_t* cell = pl.base + page * pl.page_bytes +
                    (int64_t)(head * (pl.P >> 4) + ((int)(slot[rh] & (pl.P - 1)) >> 4)) * pl.cell_bytes;
    const uint4 w = *reinterpret_cast<const uint4*>(stage + (g + 8 * rh) * MS_ROW + 16 * t);
    *reinterpret_cast<uint4*>(cell + (side ? 1152 : 128) + ci * 64 + 16 * t) = w;
    if (t == 0) {
      *reinterpret_cast<float*>(cell + side * 64 + ci * 4) = rq[rh].scale_out;
      cell[2176 + side * 16 + ci] = (uint8_t)rq[rh].zp_out;
    }
  }
  __syncwarp();  // staging reads done before the next tile overwrites it
}

template <int ORDER, bool F16>
__global__ void __launch_bounds__(FS_WARPS * 32, KVR_FS_MINB)
    store_mma_kernel(const __grid_constant__ FastStoreParams p, const __grid_constant__ CUtensorMap map_k,
                     const __grid_constant__ CUtensorMap map_v, const __grid_constant__ Signs signs) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  uint8_t* bufs = smem + wib * 2 * FS_TILE_BYTES;
  uint8_t* stage = smem + FS_WARPS * 2 * FS_TILE_BYTES + wib * MS_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + FS_WARPS * (2 * FS_TILE_BYTES + MS_STAGE)) + wib * 2;
  uint2* smask = reinterpret_cast<uint2*>(smem + FS_WARPS * (2 * FS_TILE_BYTES + MS_STAGE) + 64);  // [8 blocks][4 t]

  const int total_tiles = 2 * p.tiles_per_side;
  const int warp_stride = gridDim.x * FS_WARPS;
  const int H = p.pool.H;

  // sign-flip masks of A-fragment words: block b, lane column group t -> cols 16 b + 2 t (+1) | + 8
  if (threadIdx.x < 32) {
    const int b = threadIdx.x >> 2, tt = threadIdx.x & 3, c0 = 16 * b + 2 * tt;
    const uint32_t w = signs.w[c0 >> 5] >> (c0 & 31);
    smask[threadIdx.x] = make_uint2(((w & 1u) ? 0x8000u : 0u) | ((w & 2u) ? 0x80000000u : 0u),
                                    ((w & 0x100u) ? 0x8000u : 0u) | ((w & 0x200u) ? 0x80000000u : 0u));
  }
  __syncthreads();

  // H_16 as B fragments (k = 2t, 2t + 1 | 8 + 2t, 9 + 2t; column g + 8 nn), +-1 exact
  uint32_t bh[2][2];
  {
    const uint32_t one = F16 ? 0x3C00u : 0x3F80u;
#pragma unroll
    for (int nn = 0; nn < 2; ++nn)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int c = g + 8 * nn, k0 = 2 * t + 8 * r;
        const uint32_t lo = one | ((__popc(k0 & c) & 1) ? 0x8000u : 0u);
        const uint32_t hi = one | ((__popc((k0 + 1) & c) & 1) ? 0x8000u : 0u);
        bh[nn][r] = lo | (hi << 16);
      }
  }

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
  auto slot_pair = [&](int tile, int64_t (&sl)[2]) {
#pragma unroll
    for (int rh = 0; rh < 2; ++rh) {
      sl[rh] = -1;
      if (tile < total_tiles) {
        const int side = tile >= p.tiles_per_side;
        const int row = (side ? tile - p.tiles_per_side : tile) * FS_TILE_ROWS + g + 8 * rh;
        if (row < p.n_rows) sl[rh] = __ldg(&p.slots[row / H]);
      }
    }
  };

  // programmatic dependent launch: the setup above overlaps the previous kernel;
  // the inputs, slot ids and the pool may come from it
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int tile = blockIdx.x * FS_WARPS + wib;
  if (tile < total_tiles && elect_one()) issue(tile, 0);
  uint32_t phases = 0u;  // bit b: parity of buffer b
  int64_t slot_cur[2];
  slot_pair(tile, slot_cur);

  for (int it = 0; tile < total_tiles; ++it, tile += warp_stride) {
    const int bsel = it & 1;
    const int next = tile + warp_stride;
    if (next < total_tiles && elect_one()) issue(next, bsel ^ 1);
    const int64_t slot[2] = {slot_cur[0], slot_cur[1]};
    slot_pair(next, slot_cur);  // prefetch: consumed one tile later
    mbar_wait(&bars[bsel], (phases >> bsel) & 1u);
    phases ^= 1u << bsel;
    const uint8_t* buf = bufs + bsel * FS_TILE_BYTES;
    const int side = tile >= p.tiles_per_side;
    const int64_t row0 = (int64_t)(side ? tile - p.tiles_per_side : tile) * FS_TILE_ROWS;
    if (side ? p.rot_v : p.rot_k)  // warp-uniform
      mma_tile<ORDER, F16, true>(buf, stage, smask, p, signs, bh, row0, side, slot);
    else
      mma_tile<ORDER, F16, false>(buf, stage, smask, p, signs, bh, row0, side, slot);
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
  prm.log2P = 0;
  while ((1 << prm.log2P) < pool.P) ++prm.log2P;
  Signs sg = s;
  if (!has) for (auto& x : sg.w) x = 0u;
  CUtensorMap mk, mv;
  if (kvr_encode_tensor_map_2d(&mk, k, 128, (uint64_t)prm.n_rows, 256, 64, FS_TILE_ROWS,
                               CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return KVR_ERR_CUDA;
  if (kvr_encode_tensor_map_2d(&mv, v, 128, (uint64_t)prm.n_rows, 256, 64, FS_TILE_ROWS,
                               CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
    return KVR_ERR_CUDA;
  const size_t smem = FS_WARPS * (2 * FS_TILE_BYTES + MS_STAGE) + 64 + 256 + 1024;
  auto kern = store_mma_kernel<ORDER, F16>;
  static bool attr_set[KVR_MAX_DEVICES];  // per device (cudaFuncSetAttribute is per device)
  const int dev = kvr_current_device();
  if (!attr_set[dev]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set[dev] = true;
  }
  const int total_tiles = 2 * prm.tiles_per_side;
  int grid = (total_tiles + FS_WARPS - 1) / FS_WARPS;
  const int cap = kvr_num_sms() * KVR_FS_MINB;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(FS_WARPS * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, prm, mk, mv, sg) == cudaSuccess ? 0 : KVR_ERR_CUDA;
}

int kvr_launch_store_fast(const void* k, const void* v, int in_dtype, int64_t n_tok, const int64_t* slots,
                          const Pool& pool, int order, int rot_k, int rot_v, const Signs& s, int has,
                          uint32_t* flags, cudaStream_t st) {
  // tensor-core K1: d = 128, 16-token cells, power-of-two pages (others take the exact kernel)
  if (pool.d != 128 || pool.T != 16 || (pool.P & (pool.P - 1)) || (pool.cell_bytes & 15)) return KVR_ERR_UNSUPPORTED;
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
