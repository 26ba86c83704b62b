// K2 + K3 -- paged INT4 decode attention with a Hadamard-rotated query,
// split-K over the sequence and an inverse-rotated output for V.
//
// Reference semantics: attention.decode_step (attention.py:50-87):
//   q_frame = apply_block_rotation(q)            (rotation.py:118-142)
//   k_hat, v_hat = read_sequence(seq)            (cache.py:337-362, _ref.py:83-95)
//   out[qh] = softmax(k_hat[:, kv] q_frame[qh] / sqrt(d)) v_hat[:, kv]
//   out = out @ compose_transform(value_branch_spec(spec)).T  when V is rotated
//
// Design (B200, sm_100a, head_dim 128, GQA group G in {1,2,4,8}):
//  * grid = (split, kv head, sequence); 4 warps per CTA stride over 16-token
//    tiles of the split; a warp owns one (kv head, tile) at a time;
//  * INT4 codes never become floats in memory: a nibble masked into the low
//    mantissa bits of an fp16 IS the fp16 subnormal c * 2^-24 (exact), so one
//    LOP3 turns a code word into two MMA operands; the 2^-24 (and the x16 of
//    high nibbles) are folded into the query / the epilogue;
//  * dequantisation is factored out of the inner products:
//        logit = s_k * (q.c - z * sum(q)) / sqrt(d),  out = sum_t w_t (c_t - z_t)
//    with w_t = p_t s_t, so the tensor cores (mma.sync m16n8k16, fp16 in /
//    fp32 accumulate) only ever see exact codes;
//  * the query and the softmax weights are split hi + lo fp16 (22-bit
//    significand) and packed as column pairs of the same 8-wide MMA tile, so
//    one MMA per (16 tokens x 16 dims) yields both halves;
//  * the QK accumulator layout (tokens x q-cols) is turned into the PV B
//    operand with movmatrix.trans (no shared memory round trip);
//  * per-split (lse, o) partials go to a workspace; the last CTA of a
//    (sequence, kv head) merges them and applies the inverse rotation.
#include "kvr_common.cuh"
#include "kvr_internal.h"

namespace kvr {

constexpr float LOG2E = 1.4426950408889634f;

struct DecodeParams {
  Pool pool;
  const void* q;
  int q_dtype;
  const int32_t* bt;
  int bt_stride;
  const int32_t* lens;
  int batch, nq, G, splits, order, rotate, rot_v, has_signs, log2P, max_len;
  float* out;
  float* ws_o;       // [B][H][S][8][128]
  float* ws_lse;     // [B][H][S][8]
  uint32_t* ws_cnt;  // [B][H]
  // fused decode-step append (kvr_decode_step): one token per sequence
  const void* new_k;
  const void* new_v;
  int new_dtype;
  const int64_t* new_slot;  // [B] slot id of the appended token (it is the last of seq_lens[b])
  uint32_t* flags;
  unsigned long long* trace;  // optional: per CTA 8 globaltimer stamps (ns), see kvr_debug_decode_trace
};

KVR_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

KVR_DEV uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

KVR_DEV void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

KVR_DEV float ex2f(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

KVR_DEV uint32_t movtrans(uint32_t x) {
  uint32_t r;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}

KVR_DEV float load_q(const void* q, int dtype, int64_t i) {
  if (dtype == KVR_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(q)[i]);
  if (dtype == KVR_F16) return __half2float(reinterpret_cast<const __half*>(q)[i]);
  return reinterpret_cast<const float*>(q)[i];
}

// Cell of (sequence b, token t, head h) and the token's index inside it.
KVR_DEV const uint8_t* token_cell(const DecodeParams& p, int b, int t, int h, int& ci) {
  const int page = p.bt[(int64_t)b * p.bt_stride + (t >> p.log2P)];
  return cell_of(p.pool, page, h, t & ((1 << p.log2P) - 1), ci);
}

// dims held by A-operand register (k-step s, lane group i, slot R0/R2, half e)
KVR_DEV int qk_dim(int s, int i, int slot2, int e) { return 32 * i + 8 * (s >> 1) + 2 * (s & 1) + slot2 + 4 * e; }

// fp32 block FWHT of `rows` rows of 128 in shared memory, whole CTA, then * 1/sqrt(ORDER).
template <int ORDER>
KVR_DEV void cta_fwht_rows(float* s, int rows) {
#pragma unroll
  for (int half = 1; half < ORDER; half <<= 1) {
    for (int p = threadIdx.x; p < rows * 64; p += blockDim.x) {
      const int r = p >> 6, q = p & 63;
      const int i = r * 128 + ((q / half) * 2 * half) + (q % half);  // half is a power-of-two constant
      const float a = s[i], b = s[i + half];
      s[i] = a + b;
      s[i + half] = a - b;
    }
    __syncthreads();
  }
  const float inv = (float)(1.0 / sqrt((double)ORDER));
  for (int i = threadIdx.x; i < rows * 128; i += blockDim.x) s[i] *= inv;
  __syncthreads();
}

// ---- the fused decode-step append: one token's K or V row of head h, computed
// reference-exactly in f64 by one warp (lane l owns elements 4l..4l+3): sign
// flip, butterfly stages half = 1, 2 in registers and 4..ORDER/2 via shuffles
// (pairs combined lowest index first, exactly _ref.fwht_rows), * 1/sqrt(ORDER),
// then _ref.quantize_rows (_ref.py:22-40, 57-80) and the paged store.
template <int ORDER>
KVR_DEV void append_row_exact(const DecodeParams& p, const Signs& sg, int b, int h, int side) {
  const int lane = threadIdx.x & 31;
  const int64_t slot = p.new_slot[b];
  const int64_t base = ((int64_t)b * p.pool.H + h) * 128 + 4 * lane;
  const void* src = side ? p.new_v : p.new_k;
  double x[4];
  bool fin = true;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (p.new_dtype == KVR_BF16) x[u] = (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(src)[base + u]);
    else if (p.new_dtype == KVR_F16) x[u] = (double)__half2float(reinterpret_cast<const __half*>(src)[base + u]);
    else if (p.new_dtype == KVR_F32) x[u] = (double)reinterpret_cast<const float*>(src)[base + u];
    else x[u] = reinterpret_cast<const double*>(src)[base + u];
    fin &= (bool)isfinite(x[u]);
  }
  fin = __all_sync(0xffffffffu, fin);
  if (!fin) {
    if (lane == 0 && p.flags) atomicOr(p.flags, (uint32_t)KVR_FLAG_NONFINITE);
    return;
  }
  const bool rot = side ? (p.rotate && p.rot_v) : p.rotate;
  if (rot) {
    if (p.has_signs) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (sign_bit(sg, 4 * lane + u)) x[u] = x[u] * -1.0;
    }
    double a0 = x[0] + x[1], a1 = x[0] - x[1], a2 = x[2] + x[3], a3 = x[2] - x[3];  // half = 1
    x[0] = a0 + a2;                                                               // half = 2
    x[1] = a1 + a3;
    x[2] = a0 - a2;
    x[3] = a1 - a3;
#pragma unroll
    for (int k = 0; (4 << k) < ORDER; ++k) {  // half = 4 << k: partner lane = lane ^ (1 << k)
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
  double mn = x[0], mx = x[0];
#pragma unroll
  for (int u = 1; u < 4; ++u) {
    mn = x[u] < mn ? x[u] : mn;
    mx = x[u] > mx ? x[u] : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double a = __shfl_xor_sync(0xffffffffu, mn, o), c = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = c > mx ? c : mx;
  }
  int ci;
  uint8_t* cell = cell_of(p.pool, slot >> p.log2P, h, (int)(slot & ((1 << p.log2P) - 1)), ci);
  const float s32 = (float)((mx - mn) / 15.0);
  uint32_t bytes2 = 0u, zpv = 0xFFu;
  float scv = (float)mn;
  if (s32 != 0.0f) {
    const double s64 = (double)s32;
    double z = round_half_away(-mn / s64);
    z = z < 0.0 ? 0.0 : (z > 15.0 ? 15.0 : z);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double q = round_half_away(x[u] / s64) + z;
      q = q < 0.0 ? 0.0 : (q > 15.0 ? 15.0 : q);
      bytes2 |= (uint32_t)q << (4 * u);
    }
    scv = s32;
    zpv = (uint32_t)z;
  }
  *reinterpret_cast<uint16_t*>(cell + (side ? cell_vcode(p.pool, ci) : cell_kcode(p.pool, ci)) + 2 * lane) =
      (uint16_t)bytes2;
  if (lane == 0) {
    *reinterpret_cast<float*>(cell + (side ? cell_vscale(p.pool, ci) : cell_kscale(p.pool, ci))) = scv;
    cell[side ? cell_vzp(p.pool, ci) : cell_kzp(p.pool, ci)] = (uint8_t)zpv;
  }
}

KVR_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
KVR_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

constexpr int DW = 15;  // tile warps per CTA (one CTA per SM) + 1 writer warp for the fused append;
                       // 16 warps in all: 4 per SM sub-partition keeps the 128-register budget
constexpr int NSTG = 4;          // TMA pipeline depth per warp
constexpr int STG = 2560;        // stage: K codes 1 KB | V codes 1 KB | sidecars 256 B | pad
constexpr int MAX_CTA_TILES = 8192;

size_t decode_smem_bytes() { return 1024 + DW * NSTG * STG + (DW * NSTG + 1) * 8 + 2 * 1024 * 4 + 16; }

template <int NT, int ORDER>
__global__ void __launch_bounds__((DW + 1) * 32, 1)
    decode_tma_kernel(const __grid_constant__ DecodeParams p, const __grid_constant__ Signs signs) {
  // dynamic smem starts 1024-aligned (no static smem in this kernel); indexing the
  // __shared__ array directly keeps every access in the shared window (LDS/STS)
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint8_t* ring = sm;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + DW * NSTG * STG);
  uint64_t* app_bar = bars + DW * NSTG;
  float* sq = reinterpret_cast<float*>(app_bar + 1);
  float* sqlo = sq + 1024;
  uint32_t* s_last = reinterpret_cast<uint32_t*>(sqlo + 1024);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, i = lane & 3;
  const int h = blockIdx.x, split = blockIdx.y, b = blockIdx.z;
  const int G = p.G, H = p.pool.H;
  // split ranges come from max_len, so the page-id loads below do not wait on lens[b]
  const int len_raw = p.lens[b];
  const int n_tiles_max = (p.max_len + 15) >> 4;
  const int per = (n_tiles_max + p.splits - 1) / p.splits;
  const int lo = min(n_tiles_max, split * per);
  const int hi_max = min(n_tiles_max, lo + per);
  const int len = min(len_raw, p.max_len);
  const int n_tiles = (len + 15) >> 4;
  const int hi = min(n_tiles, hi_max);
  const int t_new = (len - 1) >> 4;
  const bool has_app = p.new_slot != nullptr && len > 0 && p.new_slot[b] >= 0 && t_new >= lo && t_new < hi;
  const int64_t cta_id = ((int64_t)b * p.splits + split) * H + h;
  if (threadIdx.x == 0) {
    if (p.trace) p.trace[cta_id * 8 + 0] = gtimer();
    if (len_raw > p.max_len && p.flags && h == 0 && split == 0) atomicOr(p.flags, KVR_FLAG_LEN_OVERFLOW);
  }

  // ---- setup (latency-ordered): q loads and the page-id windows go out first, the
  // first NSTG bulk copies right after the one CTA-wide barrier; the query is
  // prepared while they are in flight.
  const bool tile_warp = warp < DW;  // warp DW is the append writer
  const int my_tiles = (tile_warp && hi - lo - warp > 0) ? (hi - lo - warp + DW - 1) / DW : 0;
  float qx[4] = {0.f, 0.f, 0.f, 0.f};
  if (warp < 4 * NT && warp < G) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      qx[u] = load_q(p.q, p.q_dtype, ((int64_t)b * p.nq + (int64_t)h * G + warp) * 128 + 4 * lane + u);
  }
  if (tile_warp && lane < NSTG) mbar_init(&bars[warp * NSTG + lane], 1);
  if (warp == DW && lane == 0) mbar_init(app_bar, 1);
  fence_mbar_init();
  __syncwarp();

  const int pmask = (1 << p.log2P) - 1;
  const int32_t* btrow = p.bt + (int64_t)b * p.bt_stride;
  // one bulk copy per (page, head) tile: the cell holds codes and sidecars of 16 tokens
  auto issue = [&](int k, int page) {
    const int t = lo + warp + DW * k;
    uint8_t* st = ring + (warp * NSTG + (k % NSTG)) * STG;
    uint64_t* bar = &bars[warp * NSTG + (k % NSTG)];
    if (lane == 0) {
      int ci;
      const uint8_t* cell = cell_of(p.pool, page, h, (t << 4) & pmask, ci);
      fence_proxy_async();
      mbar_expect_tx(bar, (uint32_t)p.pool.cell_bytes);
      bulk_g2s(st, cell, (uint32_t)p.pool.cell_bytes, bar);
    }
  };
  // page ids of this warp's tiles live in registers, 32 tiles per window: lane l
  // of window w holds the page of tile k = 32 w + l; windows load one ahead
  auto page_window = [&](int w) -> int {
    const int t = lo + warp + DW * (32 * w + lane);
    return (tile_warp && t < hi_max) ? __ldg(&btrow[(t << 4) >> p.log2P]) : 0;
  };
  int win_idx = 0;
  int win0 = page_window(0), win1 = page_window(1);
  auto page_of = [&](int k) -> int {  // warp-uniform k
    while ((k >> 5) > win_idx) {
      win0 = win1;
      ++win_idx;
      win1 = page_window(win_idx + 1);
    }
    return __shfl_sync(0xffffffffu, win0, k & 31);
  };
  __syncthreads();  // barrier inits visible CTA-wide
  int deferred = -1;  // the tile holding the token appended by this launch waits for the append
#pragma unroll 1
  for (int k = 0; k < NSTG && k < my_tiles; ++k) {
    const int t = lo + warp + DW * k;
    if (has_app && t == t_new) {
      deferred = k;
      continue;
    }
    issue(k, page_of(k));
  }

  // ---- the fused append: the writer warp produces the new token's K and V rows
  // while the tile warps stream; only the tile holding that token waits for it
  if (has_app && warp == DW) {
    append_row_exact<ORDER>(p, signs, b, h, 0);
    append_row_exact<ORDER>(p, signs, b, h, 1);
    fence_proxy_async_global();
    __threadfence();
    __syncwarp();
    if (lane == 0) mbar_arrive(app_bar);
  }
  if (deferred >= 0) {
    mbar_wait(app_bar, 0);
    issue(deferred, page_of(deferred));
  }

  // ---- query prep (overlaps the TMA fill): warp j < 4*NT owns q head j of this kv
  // head: sign flip + fp32 butterfly in registers/shuffles, per-head power-of-two
  // normalisation, fp16 hi/lo split, scattered straight into MMA-fragment order
  uint16_t* sfrag = reinterpret_cast<uint16_t*>(sq);        // [NT][8 k-steps][2 regs][32 lanes][2 halves]
  float* s_sumq = sqlo;                                     // [8]
  float* s_ksc = sqlo + 8;                                  // [8]
  if (warp < 4 * NT) {
    const int j = warp;
    float x[4] = {0.f, 0.f, 0.f, 0.f};
    if (j < G) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u] = qx[u];
        if (p.rotate && p.has_signs && sign_bit(signs, 4 * lane + u)) x[u] = -x[u];
      }
      if (p.rotate) {
        const float a0 = x[0] + x[1], a1 = x[0] - x[1], a2 = x[2] + x[3], a3 = x[2] - x[3];
        x[0] = a0 + a2;
        x[1] = a1 + a3;
        x[2] = a0 - a2;
        x[3] = a1 - a3;
#pragma unroll
        for (int k = 0; (4 << k) < ORDER; ++k) {
          const bool upper = (lane >> k) & 1;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float o = __shfl_xor_sync(0xffffffffu, x[u], 1 << k);
            x[u] = upper ? o - x[u] : x[u] + o;
          }
        }
        const float inv = (float)(1.0 / sqrt((double)ORDER));
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] *= inv;
      }
    }
    float amax = fmaxf(fmaxf(fabsf(x[0]), fabsf(x[1])), fmaxf(fabsf(x[2]), fabsf(x[3])));
    amax = warp_max(amax);
    const int e2 = amax > 0.f ? ilogbf(amax) - 13 : 0;  // q' = q 2^-e2, max|q'| in [2^13, 2^14)
    const float qs = ldexpf(1.0f, -e2);
    float hs = 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int d = 4 * lane + u, rem = d & 31;
      const int ii = d >> 5, s = 2 * (rem >> 3) + ((rem & 3) >> 1), slot2 = rem & 1, e = (rem >> 2) & 1;
      const float v = x[u] * qs;
      const float hi = __half2float(__float2half_rn(v));
      const float lo = __half2float(__float2half_rn(v - hi));
      hs += hi + lo;
      const float f = slot2 ? (1.0f / 16.0f) : 1.0f;  // x16 nibble slots
      const int nt = j >> 2, col = 2 * (j & 3);
      const int base = (((nt * 8 + s) * 2 + slot2) * 32) * 2 + e;
      sfrag[base + ((col + 0) * 4 + ii) * 2] = __half_as_ushort(__float2half_rn(hi * f));
      sfrag[base + ((col + 1) * 4 + ii) * 2] = __half_as_ushort(__float2half_rn(lo * f));
    }
    hs = warp_sum(hs);
    if (lane == 0) {
      s_sumq[j] = hs * 5.9604644775390625e-08f;  // x 2^-24 (MMA units)
      s_ksc[j] = ldexpf(1.0f, e2 + 24) * LOG2E * (float)(1.0 / sqrt(128.0));
    }
  }
  __syncthreads();
  uint32_t bq[NT][8][2];
  float sumq[NT], kscale[NT];
  {
    const uint32_t* f32 = reinterpret_cast<const uint32_t*>(sfrag);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        bq[nt][s][0] = f32[((nt * 8 + s) * 2 + 0) * 32 + lane];
        bq[nt][s][1] = f32[((nt * 8 + s) * 2 + 1) * 32 + lane];
      }
      sumq[nt] = s_sumq[4 * nt + i];
      kscale[nt] = s_ksc[4 * nt + i];
    }
  }

  float M[NT], lsum[NT], Zs[NT];
  float acc[NT][8][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    M[nt] = -INFINITY;
    lsum[nt] = 0.f;
    Zs[nt] = 0.f;
#pragma unroll
    for (int m = 0; m < 8; ++m)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[nt][m][c] = 0.f;
  }

  // ---- main loop over this warp's tiles ---------------------------------------------
  if (p.trace && threadIdx.x == 0) p.trace[cta_id * 8 + 1] = gtimer();
#pragma unroll 1
  for (int k = 0; k < my_tiles; ++k) {
    const int t = lo + warp + DW * k;
    const int stg = k % NSTG;
    const uint8_t* st = ring + (warp * NSTG + stg) * STG;
    mbar_wait(&bars[warp * NSTG + stg], (uint32_t)((k / NSTG) & 1));
    // fragments out of the staged cell: k_scale[16] | v_scale[16] | K codes [16][64] |
    // V codes [16][64] | k_zp[16] | v_zp[16]
    const uint4 ka = *reinterpret_cast<const uint4*>(st + 128 + r * 64 + 16 * i);
    const uint4 kb = *reinterpret_cast<const uint4*>(st + 128 + (r + 8) * 64 + 16 * i);
    uint2 vw[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int tok = 2 * i + (u & 1) + 8 * (u >> 1);
      vw[u] = *reinterpret_cast<const uint2*>(st + 1152 + tok * 64 + 8 * r);
    }
    const float* sc = reinterpret_cast<const float*>(st);
    float sk0 = sc[r], sk1 = sc[r + 8], sv0 = sc[16 + r], sv1 = sc[16 + r + 8];
    const uint32_t kz0 = st[2176 + r], kz1 = st[2176 + r + 8], vz0 = st[2192 + r], vz1 = st[2192 + r + 8];
    __syncwarp();
    if (k + NSTG < my_tiles) {
      const int tn = t + DW * NSTG;
      if (has_app && tn == t_new) mbar_wait(app_bar, 0);
      issue(k + NSTG, page_of(k + NSTG));
    }

    // ---- S = C_k q : 8 k-steps of m16n8k16 per 8-column tile
    float scv[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) scv[nt][0] = scv[nt][1] = scv[nt][2] = scv[nt][3] = 0.f;
    const uint32_t kw0[4] = {ka.x, ka.y, ka.z, ka.w};
    const uint32_t kw1[4] = {kb.x, kb.y, kb.z, kb.w};
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const uint32_t wa = kw0[s >> 1], wb = kw1[s >> 1];
      const uint32_t xa = (s & 1) ? (wa >> 8) : wa, xb = (s & 1) ? (wb >> 8) : wb;
      const uint32_t a0 = xa & 0x000F000Fu, a2 = xa & 0x00F000F0u;
      const uint32_t a1 = xb & 0x000F000Fu, a3 = xb & 0x00F000F0u;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) mma16816(scv[nt], a0, a1, a2, a3, bq[nt][s][0], bq[nt][s][1]);
    }

    // ---- sidecars (sentinel rows: the scale slot holds the offset, codes are 0)
    float zk0 = (float)kz0, zk1 = (float)kz1, zv0 = (float)vz0, zv1 = (float)vz1;
    if (kz0 == 0xFFu) { zk0 = -sk0; sk0 = 1.f; }
    if (kz1 == 0xFFu) { zk1 = -sk1; sk1 = 1.f; }
    if (vz0 == 0xFFu) { zv0 = -sv0; sv0 = 1.f; }
    if (vz1 == 0xFFu) { zv1 = -sv1; sv1 = 1.f; }
    const int t0 = (t << 4) + r, t1 = t0 + 8;
    const bool ok0 = t0 < len, ok1 = t1 < len;
    const float lgv0 = ok0 ? __log2f(sv0) : 0.f, lgv1 = ok1 ? __log2f(sv1) : 0.f;

    uint32_t wlo[NT], whi[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const float l0 = ok0 ? (scv[nt][0] + scv[nt][1] - zk0 * sumq[nt]) * (sk0 * kscale[nt]) : -INFINITY;
      const float l1 = ok1 ? (scv[nt][2] + scv[nt][3] - zk1 * sumq[nt]) * (sk1 * kscale[nt]) : -INFINITY;
      const float b0 = l0 + lgv0, b1 = l1 + lgv1;  // log2(p * s_v)
      float tm = fmaxf(b0, b1);
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 4));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 8));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 16));
      // lazy rescaling: the reference point M only moves when a logit exceeds it by
      // > 2^7, so w = 2^(b - M) <= 128 and w * 2^8 stays inside fp16 range
      if (__any_sync(0xffffffffu, tm > M[nt] + 7.0f)) {
        const float mnew = fmaxf(M[nt], tm);
        const float alpha = (M[nt] == -INFINITY) ? 0.f : ex2f(M[nt] - mnew);
        if (mnew != -INFINITY) {
          lsum[nt] *= alpha;
          Zs[nt] *= alpha;
#pragma unroll
          for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[nt][m][c] *= alpha;
          M[nt] = mnew;
        }
      }
      const float ms = (M[nt] == -INFINITY) ? 0.f : M[nt];
      const float w0 = ex2f(b0 - ms), w1 = ex2f(b1 - ms);  // = p_t * s_v * 2^(.)
      const float p0 = ex2f(l0 - ms), p1 = ex2f(l1 - ms);  // = p_t * 2^(.)
      lsum[nt] += p0 + p1;
      Zs[nt] += w0 * zv0 + w1 * zv1;
      // fp16 hi/lo of w * 2^8 (w <= 2^7): 22-bit weights, the lo half out of fp16
      // subnormals for weights down to ~2^-21 of the reference point
      const float w0s = w0 * 256.0f, w1s = w1 * 256.0f;
      const float w0h = __half2float(__float2half_rn(w0s)), w1h = __half2float(__float2half_rn(w1s));
      wlo[nt] = movtrans(pack_h2(w0h, w0s - w0h));  // tokens 0..7  -> b0,b1
      whi[nt] = movtrans(pack_h2(w1h, w1s - w1h));  // tokens 8..15 -> b2,b3
    }

    // ---- O^T += C_v^T W : 8 m-tiles (16 dims each) of m16n8k16
    uint32_t xr[2][2][8];  // [token pair (2i,2i+1)|(2i+8,2i+9)][word][dim e]
#pragma unroll
    for (int tp = 0; tp < 2; ++tp)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t wa = q ? vw[2 * tp].y : vw[2 * tp].x;
        const uint32_t wb = q ? vw[2 * tp + 1].y : vw[2 * tp + 1].x;
        const uint32_t t0w = prmt(wa, wb, 0x5410u), t1w = prmt(wa, wb, 0x7632u);
        const uint32_t t0s = t0w >> 8, t1s = t1w >> 8;
        xr[tp][q][0] = t0w & 0x000F000Fu;
        xr[tp][q][1] = t0w & 0x00F000F0u;
        xr[tp][q][2] = t0s & 0x000F000Fu;
        xr[tp][q][3] = t0s & 0x00F000F0u;
        xr[tp][q][4] = t1w & 0x000F000Fu;
        xr[tp][q][5] = t1w & 0x00F000F0u;
        xr[tp][q][6] = t1s & 0x000F000Fu;
        xr[tp][q][7] = t1s & 0x00F000F0u;
      }
#pragma unroll
    for (int m = 0; m < 8; ++m)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        mma16816(acc[nt][m], xr[0][0][m], xr[0][1][m], xr[1][0][m], xr[1][1][m], wlo[nt], whi[nt]);
  }

  // ---- per-warp finalisation into shared memory (the ring is free now)
  __syncthreads();
  if (p.trace && threadIdx.x == 0) p.trace[cta_id * 8 + 2] = gtimer();
  float* sred = reinterpret_cast<float*>(ring);  // [DW][8][130]
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      lsum[nt] += __shfl_xor_sync(0xffffffffu, lsum[nt], o);
      Zs[nt] += __shfl_xor_sync(0xffffffffu, Zs[nt], o);
    }
    const int j = 4 * nt + i;
    if (tile_warp && j < G) {
      float* row = sred + (warp * 8 + j) * 130;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const float f = (m & 1) ? 65536.0f / 16.0f : 65536.0f;  // undo 2^-24 (codes), 2^8 (w), x16 nibble
        row[16 * r + m] = (acc[nt][m][0] + acc[nt][m][1]) * f - Zs[nt];
        row[16 * r + 8 + m] = (acc[nt][m][2] + acc[nt][m][3]) * f - Zs[nt];
      }
      if (r == 0) {
        row[128] = M[nt];
        row[129] = lsum[nt];
      }
    }
  }
  __syncthreads();

  // ---- CTA merge over warps -> (o, lse) of this split
  float* obuf = sq;
  const int64_t hbase = (((int64_t)b * H + h) * p.splits) * 8;
  for (int x = threadIdx.x; x < G * 128; x += blockDim.x) {
    const int j = x >> 7, dd = x & 127;
    float mmax = -INFINITY;
#pragma unroll
    for (int w = 0; w < DW; ++w) mmax = fmaxf(mmax, sred[(w * 8 + j) * 130 + 128]);
    float lt = 0.f, ot = 0.f;
    if (mmax != -INFINITY) {
#pragma unroll
      for (int w = 0; w < DW; ++w) {
        const float mw = sred[(w * 8 + j) * 130 + 128];
        const float f = (mw == -INFINITY) ? 0.f : ex2f(mw - mmax);
        lt += f * sred[(w * 8 + j) * 130 + 129];
        ot += f * sred[(w * 8 + j) * 130 + dd];
      }
    }
    const float o = (lt > 0.f) ? ot / lt : 0.f;
    const float lse = (lt > 0.f) ? mmax + __log2f(lt) : -INFINITY;
    if (p.splits == 1) {
      obuf[x] = o;
    } else {
      p.ws_o[(hbase + (int64_t)split * 8 + j) * 128 + dd] = o;
      if (dd == 0) p.ws_lse[hbase + (int64_t)split * 8 + j] = lse;
    }
  }
  if (p.splits > 1) {
    // release the partial: CTA barrier, then one gpu-scope acq_rel atomic by thread 0
    // (cumulative over the CTA's writes ordered before it by the barrier)
    __syncthreads();
    if (threadIdx.x == 0) {
      if (p.trace) p.trace[cta_id * 8 + 3] = gtimer();
      uint32_t prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                   : "=r"(prev)
                   : "l"(&p.ws_cnt[(int64_t)b * H + h])
                   : "memory");
      *s_last = (prev == (uint32_t)p.splits - 1) ? 1u : 0u;
      if (p.trace) p.trace[cta_id * 8 + 4] = gtimer();
    }
    __syncthreads();
    if (!*s_last) {
      if (p.trace && threadIdx.x == 0) p.trace[cta_id * 8 + 6] = gtimer();
      return;
    }
    // last CTA of (b, h): LSE-merge all splits.  Every thread re-derives the split
    // weights of its q head from the lse values (same address across the warp), so
    // the lse and o loads of a 32-split chunk go out together: one L2 round trip.
    for (int x = threadIdx.x; x < G * 128; x += blockDim.x) {
      const int j = x >> 7, dd = x & 127;
      const float* lsrc = p.ws_lse + hbase + j;
      const float* osrc = p.ws_o + (hbase + j) * 128 + dd;
      float lmax = -INFINITY, tot = 0.f, ot = 0.f;
      for (int s0 = 0; s0 < p.splits; s0 += 32) {
        float lv[32], ov[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const bool in = s0 + u < p.splits;
          lv[u] = in ? __ldcg(lsrc + (int64_t)(s0 + u) * 8) : -INFINITY;
          ov[u] = in ? __ldcg(osrc + (int64_t)(s0 + u) * 8 * 128) : 0.f;
        }
        float cm = lmax;
#pragma unroll
        for (int u = 0; u < 32; ++u) cm = fmaxf(cm, lv[u]);
        if (cm == -INFINITY) continue;
        const float a = (lmax == -INFINITY) ? 0.f : exp2f(lmax - cm);
        tot *= a;
        ot *= a;
        lmax = cm;
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const float f = (lv[u] == -INFINITY) ? 0.f : exp2f(lv[u] - cm);
          tot += f;
          ot += f * ov[u];
        }
      }
      obuf[x] = tot > 0.f ? ot / tot : 0.f;
    }
    if (threadIdx.x == 0) {
      p.ws_cnt[(int64_t)b * H + h] = 0u;  // re-arm for the next launch
      if (p.trace) p.trace[cta_id * 8 + 5] = gtimer();
    }
  }
  __syncthreads();
  // ---- output: inverse rotation of the value branch (o @ H_blk @ diag(signs)),
  // one warp per q head, fp32 butterfly in registers / shuffles
  if (warp < G) {
    float x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = obuf[warp * 128 + 4 * lane + u];
    if (p.rotate && p.rot_v) {
      const float a0 = x[0] + x[1], a1 = x[0] - x[1], a2 = x[2] + x[3], a3 = x[2] - x[3];
      x[0] = a0 + a2;
      x[1] = a1 + a3;
      x[2] = a0 - a2;
      x[3] = a1 - a3;
#pragma unroll
      for (int k = 0; (4 << k) < ORDER; ++k) {
        const bool upper = (lane >> k) & 1;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float o = __shfl_xor_sync(0xffffffffu, x[u], 1 << k);
          x[u] = upper ? o - x[u] : x[u] + o;
        }
      }
      const float inv = (float)(1.0 / sqrt((double)ORDER));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u] *= inv;
        if (p.has_signs && sign_bit(signs, 4 * lane + u)) x[u] = -x[u];
      }
    }
    float4* dst = reinterpret_cast<float4*>(p.out + ((int64_t)b * p.nq + (int64_t)h * G + warp) * 128) + lane;
    *dst = make_float4(x[0], x[1], x[2], x[3]);
  }
  if (p.trace && threadIdx.x == 0) p.trace[cta_id * 8 + 6] = gtimer();
}

// Generic (any head_dim <= 256, any group) CUDA-core decode: one CTA per
// (sequence, q head), warps stride over tokens with an online softmax.
__global__ void decode_generic_kernel(const __grid_constant__ DecodeParams p, const __grid_constant__ Signs signs,
                                      int d) {
  extern __shared__ float gsm[];
  float* sq = gsm;                          // d
  float* so = gsm + d;                      // [warps][d]
  float* sml = gsm + d + (blockDim.x >> 5) * d;  // [warps][2]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int qh = blockIdx.x, b = blockIdx.y;
  const int G = p.G, h = qh / G;
  const int len = min(p.lens[b], p.max_len);
  for (int x = threadIdx.x; x < d; x += blockDim.x) {
    float v = load_q(p.q, p.q_dtype, ((int64_t)b * p.nq + qh) * d + x);
    if (p.rotate && p.has_signs && sign_bit(signs, x)) v = -v;
    sq[x] = v;
  }
  __syncthreads();
  if (p.rotate) {
    for (int half = 1; half < p.order; half <<= 1) {
      for (int pp = threadIdx.x; pp < d / 2; pp += blockDim.x) {
        const int blk = pp / (p.order >> 1), w = pp % (p.order >> 1);
        const int ii = blk * p.order + (w / half) * 2 * half + (w % half);
        const float a = sq[ii], c = sq[ii + half];
        sq[ii] = a + c;
        sq[ii + half] = a - c;
      }
      __syncthreads();
    }
    const float inv = (float)(1.0 / sqrt((double)p.order));
    for (int x = threadIdx.x; x < d; x += blockDim.x) sq[x] *= inv;
    __syncthreads();
  }
  const float scale = (float)(1.0 / sqrt((double)d));
  float m = -INFINITY, l = 0.f;
  float o[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) o[k] = 0.f;
  for (int t = warp; t < len; t += nw) {
    int ci;
    const uint8_t* cell = token_cell(p, b, t, h, ci);
    const float ks = *reinterpret_cast<const float*>(cell + cell_kscale(p.pool, ci));
    const uint8_t kz = cell[cell_kzp(p.pool, ci)];
    const float vs = *reinterpret_cast<const float*>(cell + cell_vscale(p.pool, ci));
    const uint8_t vz = cell[cell_vzp(p.pool, ci)];
    const uint8_t* kc = cell + cell_kcode(p.pool, ci);
    const uint8_t* vc = cell + cell_vcode(p.pool, ci);
    float dot = 0.f;
    for (int k = 0, x = lane; x < d; x += 32, ++k) {
      const uint8_t byte = kc[x >> 1];
      const float c = (float)((x & 1) ? (byte >> 4) : (byte & 15));
      const float kh = (kz == 0xFF) ? ks : ks * (c - (float)kz);
      dot += kh * sq[x];
    }
    dot = warp_sum(dot) * scale;
    const float mn = fmaxf(m, dot);
    const float a = exp2f((m - mn) * LOG2E), pw = exp2f((dot - mn) * LOG2E);
    l = l * a + pw;
    for (int k = 0, x = lane; x < d; x += 32, ++k) {
      const uint8_t byte = vc[x >> 1];
      const float c = (float)((x & 1) ? (byte >> 4) : (byte & 15));
      const float vh = (vz == 0xFF) ? vs : vs * (c - (float)vz);
      o[k] = o[k] * a + pw * vh;
    }
    m = mn;
  }
  for (int k = 0, x = lane; x < d; x += 32, ++k) so[warp * d + x] = o[k];
  if (lane == 0) {
    sml[2 * warp] = m;
    sml[2 * warp + 1] = l;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < d; x += blockDim.x) {
    float mm = -INFINITY;
    for (int w = 0; w < nw; ++w) mm = fmaxf(mm, sml[2 * w]);
    float lt = 0.f, ot = 0.f;
    for (int w = 0; w < nw; ++w) {
      if (sml[2 * w] == -INFINITY) continue;
      const float f = exp2f((sml[2 * w] - mm) * LOG2E);
      lt += f * sml[2 * w + 1];
      ot += f * so[w * d + x];
    }
    sq[x] = lt > 0.f ? ot / lt : 0.f;
  }
  __syncthreads();
  if (p.rotate && p.rot_v) {
    for (int half = 1; half < p.order; half <<= 1) {
      for (int pp = threadIdx.x; pp < d / 2; pp += blockDim.x) {
        const int blk = pp / (p.order >> 1), w = pp % (p.order >> 1);
        const int ii = blk * p.order + (w / half) * 2 * half + (w % half);
        const float a = sq[ii], c = sq[ii + half];
        sq[ii] = a + c;
        sq[ii + half] = a - c;
      }
      __syncthreads();
    }
    const float inv = (float)(1.0 / sqrt((double)p.order));
    for (int x = threadIdx.x; x < d; x += blockDim.x) {
      float v = sq[x] * inv;
      if (p.has_signs && sign_bit(signs, x)) v = -v;
      sq[x] = v;
    }
    __syncthreads();
  }
  for (int x = threadIdx.x; x < d; x += blockDim.x) p.out[((int64_t)b * p.nq + qh) * d + x] = sq[x];
}

}  // namespace kvr

using namespace kvr;

size_t kvr_decode_ws_bytes(int batch, int H, int nq, int d, int splits) {
  (void)nq;
  (void)d;
  if (splits < 1) splits = 1;
  const size_t units = (size_t)batch * H * splits * 8;
  size_t bytes = units * 128 * sizeof(float) + units * sizeof(float) + (size_t)batch * H * sizeof(uint32_t);
  return (bytes + 255) & ~size_t(255);
}

int kvr_pick_splits(int batch, int H, int max_len, int P) {
  (void)P;
  const int sms = kvr_num_sms() > 0 ? kvr_num_sms() : 148;
  const int tiles = (max_len + 15) / 16;
  const int units = batch * H;
  int s = sms / units;  // one CTA per SM, a single wave
  const int min_tiles_per_cta = 2 * DW;
  const int max_s = tiles / min_tiles_per_cta;
  if (s > max_s) s = max_s;
  if (s > 128) s = 128;
  if (s < 1) s = 1;
  while ((tiles + s - 1) / s > MAX_CTA_TILES && s < 128) ++s;
  return s;
}

template <int NT>
static int launch_tma(const DecodeParams& p, const Signs& sg, dim3 grid, size_t smem, int order, cudaStream_t st) {
#define KVR_DEC_CASE(ORD)                                                                               \
  case ORD: {                                                                                           \
    auto kern = decode_tma_kernel<NT, ORD>;                                                             \
    static bool set = false;                                                                            \
    if (!set) {                                                                                         \
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);               \
      set = true;                                                                                       \
    }                                                                                                   \
    kern<<<grid, (DW + 1) * 32, smem, st>>>(p, sg);                                                     \
    return 0;                                                                                           \
  }
  switch (order) {
    KVR_DEC_CASE(128)
    KVR_DEC_CASE(64)
    KVR_DEC_CASE(32)
    KVR_DEC_CASE(16)
  }
#undef KVR_DEC_CASE
  return KVR_ERR_UNSUPPORTED;
}

static unsigned long long* g_trace = nullptr;
void kvr_set_decode_trace(void* trace) { g_trace = reinterpret_cast<unsigned long long*>(trace); }

int kvr_launch_decode(const void* q, int q_dtype, const Pool& pool, const int32_t* bt, int bt_stride,
                      const int32_t* lens, int batch, int nq, int max_len, int order, int rotate, int rot_v,
                      const Signs& s, int has, float* out, void* ws, size_t ws_bytes, int splits, cudaStream_t st,
                      const void* new_k, const void* new_v, int new_dtype, const int64_t* new_slot,
                      uint32_t* flags) {
  DecodeParams p{};
  p.pool = pool;
  p.q = q;
  p.q_dtype = q_dtype;
  p.bt = bt;
  p.bt_stride = bt_stride;
  p.lens = lens;
  p.batch = batch;
  p.nq = nq;
  p.G = nq / pool.H;
  p.order = order;
  p.rotate = rotate;
  p.rot_v = rot_v;
  p.has_signs = has;
  p.out = out;
  p.new_k = new_k;
  p.new_v = new_v;
  p.new_dtype = new_dtype;
  p.new_slot = new_slot;
  p.flags = flags;
  p.trace = g_trace;
  p.max_len = max_len;
  int l2 = 0;
  while ((1 << l2) < pool.P) ++l2;
  const bool pow2 = (1 << l2) == pool.P;
  p.log2P = l2;
  Signs sg = s;
  if (!has) for (auto& x : sg.w) x = 0u;
  if (!pow2) return KVR_ERR_UNSUPPORTED;
  const bool tma_ok = pool.d == 128 && pool.T == 16 && (p.G == 1 || p.G == 2 || p.G == 4 || p.G == 8) &&
                      (reinterpret_cast<uintptr_t>(pool.base) & 15) == 0 && (pool.cell_bytes & 15) == 0;
  if (tma_ok) {
    if (splits <= 0) splits = kvr_pick_splits(batch, pool.H, max_len, pool.P);
    if (splits > 128) splits = 128;
    if ((max_len + 15) / 16 > (int64_t)splits * MAX_CTA_TILES) return KVR_ERR_UNSUPPORTED;
    if (splits > 1 && kvr_decode_ws_bytes(batch, pool.H, nq, 128, splits) > ws_bytes) return KVR_ERR_ARG;
    p.splits = splits;
    const size_t units = (size_t)batch * pool.H * splits * 8;
    p.ws_o = reinterpret_cast<float*>(ws);
    p.ws_lse = p.ws_o + units * 128;
    p.ws_cnt = reinterpret_cast<uint32_t*>(p.ws_lse + units);
    dim3 grid(pool.H, splits, batch);
    const int ord = rotate ? order : 128;
    const size_t smem = decode_smem_bytes();
    return p.G == 8 ? launch_tma<2>(p, sg, grid, smem, ord, st) : launch_tma<1>(p, sg, grid, smem, ord, st);
  }
  if (new_slot) return KVR_ERR_UNSUPPORTED;  // the fused append lives in the TMA kernel only
  if (pool.d > 256 || (pool.d & 31)) return KVR_ERR_UNSUPPORTED;
  p.splits = 1;
  const int warps = 4;
  const size_t smem = (size_t)(pool.d + warps * pool.d + warps * 2) * sizeof(float);
  decode_generic_kernel<<<dim3(nq, batch), warps * 32, smem, st>>>(p, sg, pool.d);
  return 0;
}
