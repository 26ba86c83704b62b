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
//  * INT4 codes never become floats in memory: for QK a nibble masked into the
//    low mantissa bits of an fp16 IS the fp16 subnormal c * 2^-24 (exact), so one
//    LOP3 turns a code word into two MMA operands (or the code bytes feed the int8
//    MMA directly); for PV a nibble masked into the mantissa of 1024.0 minus
//    1024 + z gives the exact signed c - z (LOP3 + HSUB2 per two operands);
//  * dequantisation is factored out of the inner products:
//        logit = s_k * (q.c - z * sum(q)) / sqrt(d),  out = sum_t w_t (c_t - z_t)
//    with w_t = p_t s_t, so the tensor cores (mma.sync, fp16 / int8 in, fp32 /
//    int32 accumulate) only ever see exact integers; PV products carry both signs
//    (c - z), so the tensor core's truncating accumulation does not drift;
//  * the query and the softmax weights are split hi + lo fp16 (22-bit
//    significand) and packed as column pairs of the same 8-wide MMA tile, so
//    one MMA per (16 tokens x 16 dims) yields both halves;
//  * the QK accumulator layout (tokens x q-cols) is turned into the PV B
//    operand with movmatrix.trans (no shared memory round trip);
//  * per-split (lse, o) partials go to a workspace; the last CTA of a
//    (sequence, kv head) merges them and applies the inverse rotation.
#include <cstdlib>

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
  int cps_log2;       // log2(cells of one head per page) = log2(P / 16) on the TMA path
  int split_tiles;    // ceil(ceil(max_len / 16) / splits): the tiles of one split (host-computed: no division in-kernel)
  int use_cluster;    // 2..16 splits: merge them in a thread-block cluster
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
  int pre_groups;    // ring groups per warp requested before griddepcontrol.wait
  int evict_first;   // KV cells are streamed with an L2 evict-first policy
  int merge_inline;  // splits > 1 without a cluster: the last CTA merges (ws_cnt counters)
  // flag-in-data split merge (the grid is one wave): every split stores its (o, lse) as 64-bit
  // words (value bits | epoch + 1) with relaxed stores; CTA j < G polls the words of q head j
  int merge_ll;
  uint32_t* ws_epoch;             // [B][H][8] epochs, bumped by each head's merger
  unsigned long long* ll_lse;     // [B][H][8][32]
  unsigned long long* ll_o;       // [B][H][8][32][128]
  int q_pre_wait;       // the query is host-staged for this launch (immutable): load it before the wait
  int meta_post_wait;   // lengths / slot ids come from the previous grid: read them after the wait
  uint32_t f16x2_1024;  // 0x64006400 (fp16x2 1024.0) from the parameter bank: an opaque operand lets
                        // ptxas fuse (x & mask) | 1024 into one LOP3 (two immediates need two)
  // row f3, learned rotation fused into the decode (the ORDER = 0 instantiation): the composed
  // T = diag(s) H_blk R as f32 [128][LT_STRIDE] (bulk-copied into shared memory before the wait);
  // the query is multiplied by T in the prologue, the output mapped back by lq_out: 0 none
  // (KEYS_ONLY), 1 the value branch's block Hadamard inverse (order lq_order, the signs), 2 T^T
  const float* lq;
  int lq_out, lq_order;
};

KVR_DEV unsigned long long clk64() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
  return t;
}
// Debug timeline (kvr_debug_decode_trace): per CTA 16 u64, [0] globaltimer and
// [1] clock64 at entry, [k >= 2] clock64 at stamp k (written by thread 0).
#define KVR_STAMP(k)                                                   \
  do {                                                                 \
    if (p.trace && threadIdx.x == 0) p.trace[cta_id * 16 + (k)] = clk64(); \
  } while (0)

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

KVR_DEV void imma16832(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

KVR_DEV float ex2f(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

KVR_DEV uint32_t hsub2_u32(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// (a & MASK) | c in one LOP3 (c in a register or the constant bank)
template <uint32_t MASK>
KVR_DEV uint32_t and_or(uint32_t a, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "n"(MASK), "r"(c));
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

// floor(log2 a) of a finite a > 0 (ilogbf) from the exponent bits; 2^e (ldexpf(1, e))
// as bits -- the library forms only for subnormals / out-of-range exponents
KVR_DEV int ilog2_pos(float a) {
  const int ex = (__float_as_int(a) >> 23) & 0xFF;
  return ex ? ex - 127 : ilogbf(a);
}
KVR_DEV float exp2i(int e) { return (e >= -126 && e <= 127) ? __int_as_float((e + 127) << 23) : ldexpf(1.0f, e); }

// Elements i..i+3 (i % 4 == 0) of the query as one 8-B (bf16/f16) or 16-B (f32) load
// (element loads when the query is not aligned for that).
KVR_DEV void load_q4(const void* q, int dtype, int64_t i, float (&x)[4]) {
  if (reinterpret_cast<uintptr_t>(q) & (dtype == KVR_F32 ? 15 : 7)) {
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = load_q(q, dtype, i + u);
    return;
  }
  if (dtype == KVR_F32) {
    const float4 v = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(q) + i);
    x[0] = v.x;
    x[1] = v.y;
    x[2] = v.z;
    x[3] = v.w;
    return;
  }
  const uint2 w = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(q) + i);
  const uint32_t h[4] = {w.x & 0xFFFFu, w.x >> 16, w.y & 0xFFFFu, w.y >> 16};
#pragma unroll
  for (int u = 0; u < 4; ++u)
    x[u] = dtype == KVR_BF16 ? __uint_as_float(h[u] << 16) : __half2float(__ushort_as_half((unsigned short)h[u]));
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

// ---- the fused decode-step append: one token's K and V rows of head h, computed
// reference-exactly in f64 by one warp (lane l owns elements 4l..4l+3 of both
// rows; the two rows are interleaved for instruction-level parallelism): sign
// flip, butterfly stages half = 1, 2 in registers and 4..ORDER/2 via shuffles
// (pairs combined lowest index first, exactly _ref.fwht_rows), * 1/sqrt(ORDER),
// then _ref.quantize_rows (_ref.py:22-40, 57-80) and the paged store.
// Returns the stored-space (rotated) dequantised elements of lane l in deq[side]
// (dims 4l..4l+3); a non-finite row is flagged, not written, and reads as 0.
KVR_DEV double load_any(const void* src, int dtype, int64_t i) {
  if (dtype == KVR_BF16) return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(src)[i]);
  if (dtype == KVR_F16) return (double)__half2float(reinterpret_cast<const __half*>(src)[i]);
  if (dtype == KVR_F32) return (double)reinterpret_cast<const float*>(src)[i];
  return reinterpret_cast<const double*>(src)[i];
}

template <int ORDER>
KVR_DEV bool append_rows_exact(const DecodeParams& p, const Signs& sg, int b, int h, float (&deq)[2][4],
                               unsigned long long* tr = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t slot = p.new_slot[b];
  const int64_t base = ((int64_t)b * p.pool.H + h) * 128 + 4 * lane;
  double x[2][4];
  int ci;
  uint8_t* cell = cell_of(p.pool, slot >> p.log2P, h, (int)(slot & ((1 << p.log2P) - 1)), ci);
  // the token is all-or-nothing (the reference validates the whole (H, d) K and V
  // before any write, cache.py:225-233): a NaN/Inf in any head's row leaves every
  // head's rows unwritten -- so this writer also scans the other heads' rows
  bool all_fin = true;
  if ((p.new_dtype == KVR_BF16 || p.new_dtype == KVR_F16) &&
      !((reinterpret_cast<uintptr_t>(p.new_k) | reinterpret_cast<uintptr_t>(p.new_v)) & 7)) {
    // every head's K and V quad of this lane as one batch of independent 8-byte loads (the
    // rows may come over the bus from a pinned staging buffer: one round trip, not one per head)
    const bool bf = p.new_dtype == KVR_BF16;
    const uint32_t em = bf ? 0x7F80u : 0x7C00u;  // exponent all ones <=> NaN / Inf
    const uint16_t* kq = reinterpret_cast<const uint16_t*>(p.new_k) + (int64_t)b * p.pool.H * 128 + 4 * lane;
    const uint16_t* vq = reinterpret_cast<const uint16_t*>(p.new_v) + (int64_t)b * p.pool.H * 128 + 4 * lane;
    for (int h0 = 0; h0 < p.pool.H; h0 += 8) {
      uint2 wk[8], wv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (h0 + j < p.pool.H) {
          wk[j] = *reinterpret_cast<const uint2*>(kq + (h0 + j) * 128);
          wv[j] = *reinterpret_cast<const uint2*>(vq + (h0 + j) * 128);
        }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (h0 + j < p.pool.H) {
          const uint32_t w4[4] = {wk[j].x, wk[j].y, wv[j].x, wv[j].y};
#pragma unroll
          for (int u = 0; u < 4; ++u)
            all_fin &= ((w4[u] & em) != em) && (((w4[u] >> 16) & em) != em);
          if (h0 + j == h) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint32_t hk = (u & 1) ? (w4[u >> 1] >> 16) : (w4[u >> 1] & 0xFFFFu);
              const uint32_t hv = (u & 1) ? (w4[2 + (u >> 1)] >> 16) : (w4[2 + (u >> 1)] & 0xFFFFu);
              x[0][u] = bf ? (double)__uint_as_float(hk << 16) : (double)__half2float(__ushort_as_half((unsigned short)hk));
              x[1][u] = bf ? (double)__uint_as_float(hv << 16) : (double)__half2float(__ushort_as_half((unsigned short)hv));
            }
          }
        }
    }
  } else {
#pragma unroll
    for (int sd = 0; sd < 2; ++sd) {
      const void* src = sd ? p.new_v : p.new_k;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[sd][u] = load_any(src, p.new_dtype, base + u);
        all_fin &= (bool)isfinite(x[sd][u]);
      }
    }
    for (int hh = 0; hh < p.pool.H; ++hh) {
      if (hh == h) continue;
      const int64_t ob = ((int64_t)b * p.pool.H + hh) * 128 + 4 * lane;
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) {
        const void* src = sd ? p.new_v : p.new_k;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          all_fin &= (bool)isfinite(load_any(src, p.new_dtype, ob + u));
        }
      }
    }
  }
  const bool ok = __all_sync(0xffffffffu, all_fin);
  if (tr) tr[14] = clk64();  // rows landed
  if (!ok && lane == 0 && p.flags) atomicOr(p.flags, (uint32_t)KVR_FLAG_NONFINITE);
  const bool rot[2] = {p.rotate != 0, p.rotate && p.rot_v};
#pragma unroll
  for (int sd = 0; sd < 2; ++sd)
    if (rot[sd] && p.has_signs) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (sign_bit(sg, 4 * lane + u)) x[sd][u] = x[sd][u] * -1.0;
    }
#pragma unroll
  for (int sd = 0; sd < 2; ++sd)
    if (rot[sd]) {
      const double a0 = x[sd][0] + x[sd][1], a1 = x[sd][0] - x[sd][1];  // half = 1
      const double a2 = x[sd][2] + x[sd][3], a3 = x[sd][2] - x[sd][3];
      x[sd][0] = a0 + a2;                                                  // half = 2
      x[sd][1] = a1 + a3;
      x[sd][2] = a0 - a2;
      x[sd][3] = a1 - a3;
    }
#pragma unroll
  for (int k = 0; (4 << k) < ORDER; ++k) {  // half = 4 << k: partner lane = lane ^ (1 << k)
    const double sgn = ((lane >> k) & 1) ? -1.0 : 1.0;  // upper half of the pair: o - x
#pragma unroll
    for (int sd = 0; sd < 2; ++sd)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double o = __shfl_xor_sync(0xffffffffu, x[sd][u], 1 << k);
        if (rot[sd]) x[sd][u] = fma(sgn, x[sd][u], o);  // o -+ x, one rounding
      }
  }
  if (tr) tr[15] = clk64();  // rotated
  const double inv = 1.0 / sqrt((double)ORDER);
  double mn[2], mx[2];
#pragma unroll
  for (int sd = 0; sd < 2; ++sd) {
    if (rot[sd]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) x[sd][u] = x[sd][u] * inv;
    }
    mn[sd] = x[sd][0];
    mx[sd] = x[sd][0];
#pragma unroll
    for (int u = 1; u < 4; ++u) {
      mn[sd] = x[sd][u] < mn[sd] ? x[sd][u] : mn[sd];
      mx[sd] = x[sd][u] > mx[sd] ? x[sd][u] : mx[sd];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int sd = 0; sd < 2; ++sd) {
      const double a = __shfl_xor_sync(0xffffffffu, mn[sd], o), c = __shfl_xor_sync(0xffffffffu, mx[sd], o);
      mn[sd] = a < mn[sd] ? a : mn[sd];
      mx[sd] = c > mx[sd] ? c : mx[sd];
    }
#pragma unroll
  for (int sd = 0; sd < 2; ++sd) {
    // the reference's f64 divisions, each correctly rounded (div_rn_recip): one
    // reciprocal per row instead of six divisions
    const float s32 = (float)div_rn_recip(mx[sd] - mn[sd], 15.0, 1.0 / 15.0);
    uint32_t bytes2 = 0u, zpv = 0xFFu;
    float scv = (float)mn[sd];
    if (s32 != 0.0f) {
      const double s64 = (double)s32;
      const double rs = 1.0 / s64;
      double z = round_half_away(div_rn_recip(-mn[sd], s64, rs));
      z = z < 0.0 ? 0.0 : (z > 15.0 ? 15.0 : z);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double q = round_half_away(div_rn_recip(x[sd][u], s64, rs)) + z;
        q = q < 0.0 ? 0.0 : (q > 15.0 ? 15.0 : q);
        bytes2 |= (uint32_t)q << (4 * u);
      }
      scv = s32;
      zpv = (uint32_t)z;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        deq[sd][u] = (float)((double)s32 * (double)((int)((bytes2 >> (4 * u)) & 15u) - (int)zpv));
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) deq[sd][u] = scv;  // sentinel row: the offset
    }
    if (!ok) {
#pragma unroll
      for (int u = 0; u < 4; ++u) deq[sd][u] = 0.f;
      continue;
    }
    *reinterpret_cast<uint16_t*>(cell + (sd ? cell_vcode(p.pool, ci) : cell_kcode(p.pool, ci)) + 2 * lane) =
        (uint16_t)bytes2;
    if (lane == 0) {
      *reinterpret_cast<float*>(cell + (sd ? cell_vscale(p.pool, ci) : cell_kscale(p.pool, ci))) = scv;
      cell[sd ? cell_vzp(p.pool, ci) : cell_kzp(p.pool, ci)] = (uint8_t)zpv;
    }
  }
  return ok;
}

KVR_DEV void st_relaxed_u64(unsigned long long* a, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
KVR_DEV unsigned long long ld_relaxed_u64(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}

// named barriers (id 0 is __syncthreads): 1 = the tile warps after query prep,
// 2 = query-prep warps -> writer warp (rotated q in smem for scoring the new token)
KVR_DEV void named_bar_sync(int id, int threads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory"); }
KVR_DEV void named_bar_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

KVR_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
KVR_DEV bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0u;
}
KVR_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// Programmatic dependent launch: wait for the previous grid in the stream / let
// the next one start its prologue (griddepcontrol, sm_90+).
KVR_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
KVR_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- thread-block cluster helpers (split merge through distributed shared memory)
KVR_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// final barrier: only says "my remote reads are done" (their values were consumed)
KVR_DEV void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
KVR_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// generic address of `local` in the shared memory of cluster CTA `rank`: plain
// loads through it are independent and pipeline (ordering comes from the barrier)
KVR_DEV const float* dsmem_ptr(const float* local, uint32_t rank) {
  const float* r;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(local), "r"(rank));
  return r;
}

constexpr int NWARPS = 16;       // one CTA per SM, 4 warps per SM sub-partition (128-register budget)
constexpr int CELL = 2208;       // one cell: T = 16 tokens of one head, d = 128
constexpr int RING_CELLS = 4;    // cells in flight per warp (NSTG stages of C cells)
#ifndef KVR_NT2_CELLS
#define KVR_NT2_CELLS 2  // cells per ring group of the G = 8 kernel (2: -2 % on C4 despite a small spill)
#endif
#ifndef KVR_PREWAIT_GROUPS
#define KVR_PREWAIT_GROUPS 1
#endif
#ifndef KVR_PREWAIT_GROUPS_LL
#define KVR_PREWAIT_GROUPS_LL 2
#endif
#ifndef KVR_EVICT_FIRST
#define KVR_EVICT_FIRST 1
#endif
#ifndef KVR_MERGE_INLINE
#define KVR_MERGE_INLINE 1
#endif
#ifndef KVR_CLUSTER_MAX
#define KVR_CLUSTER_MAX 8
#endif
#ifndef KVR_MERGE_LL
#define KVR_MERGE_LL 1
#endif
#ifndef KVR_PRMT_SENT
#define KVR_PRMT_SENT 1  // sentinel zero points cleared by a sign-replicating PRMT (no predicated compare)
#endif
constexpr int MAX_SPLITS = 256;
constexpr int MERGE_INLINE_MAX = 32;  // up to this many splits the last CTA merges them inline

// smem: ring [NWARPS][RING_CELLS][CELL] | bars [NWARPS*RING_CELLS + 1] | q fragments 4 KB | out 4 KB | misc
constexpr int SM_BARS = NWARPS * RING_CELLS * CELL;
constexpr int SM_FRAG = SM_BARS + (NWARPS * RING_CELLS + 1) * 8 + 8;  // 16-B aligned
constexpr int SM_OBUF = SM_FRAG + 4096;
constexpr int SM_QROT = SM_OBUF + 4096;                               // fp32 rotated q [8][128] (APPEND)
constexpr int SM_VNEW = SM_QROT + 4096;                               // new token's V row [128] (APPEND)
constexpr int SM_MISC = SM_VNEW + 512;                               // sumq[8] ksc[8] tot[8] flag lse[8]
constexpr int SM_TOTAL = SM_MISC + 256;
// learned instantiation only: T [128][129] f32 (row stride 129 floats: both the q T column walk and
// the o T^T row walk hit 32 distinct banks) and its mbarrier
constexpr int LT_STRIDE = 129;
constexpr int LT_BYTES = 128 * LT_STRIDE * 4;  // 66,048 (a multiple of 16: one bulk copy)
constexpr int SM_LT = SM_TOTAL;
constexpr int SM_LTBAR = SM_LT + LT_BYTES;
constexpr int SM_TOTAL_LQ = SM_LTBAR + 16;
static_assert(SM_LT % 16 == 0, "bulk-copy destination");
static_assert(1024 + SM_TOTAL_LQ <= 232448, "learned decode shared memory");
size_t decode_smem_bytes() { return 1024 + SM_TOTAL; }
size_t decode_smem_bytes_lq() { return 1024 + SM_TOTAL_LQ; }

// Fragments of one staged cell: k_scale[16] | v_scale[16] | K codes [16][64] |
// V codes [16][64] | k_zp[16] | v_zp[16]
struct CellFrag {
  uint4 ka, kb;
  uint2 vw[4];
  float sk0, sk1, sv0, sv1;
  uint32_t kz0, kz1, vz0, vz1;
  uint32_t vzp0, vzp1;  // V zero points of tokens (2i, 2i + 1) and (2i + 8, 2i + 9): the PV operand pairs
};
KVR_DEV void load_cell_k(CellFrag& f, const uint8_t* st, int r, int i) {
  f.ka = *reinterpret_cast<const uint4*>(st + 128 + r * 64 + 16 * i);
  f.kb = *reinterpret_cast<const uint4*>(st + 128 + (r + 8) * 64 + 16 * i);
}
KVR_DEV void load_cell_rest(CellFrag& f, const uint8_t* st, int r, int i) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int tok = 2 * i + (u & 1) + 8 * (u >> 1);
    f.vw[u] = *reinterpret_cast<const uint2*>(st + 1152 + tok * 64 + 8 * r);
  }
  const float* sc = reinterpret_cast<const float*>(st);
  f.sk0 = sc[r];
  f.sk1 = sc[r + 8];
  f.sv0 = sc[16 + r];
  f.sv1 = sc[16 + r + 8];
  f.kz0 = st[2176 + r];
  f.kz1 = st[2176 + r + 8];
  f.vz0 = st[2192 + r];
  f.vz1 = st[2192 + r + 8];
  f.vzp0 = *reinterpret_cast<const uint16_t*>(st + 2192 + 2 * i);
  f.vzp1 = *reinterpret_cast<const uint16_t*>(st + 2192 + 8 + 2 * i);
}

// One q head's final output (warp-wide, lane owns dims 4l..4l+3): the inverse
// rotation of the value branch (o @ H_blk @ diag(signs)) as an fp32 butterfly in
// registers / shuffles, then a 16-B store per lane.  `row` is o in natural order.
template <int ORDER>
KVR_DEV void emit_head(const DecodeParams& p, uint32_t sgw, int b, int h, int j, const float* row, int lane,
                       const float* s_t = nullptr) {
  float* orow = p.out + ((int64_t)b * p.nq + (int64_t)h * p.G + j) * 128;
  float x[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) x[u] = row[4 * lane + u];
  if constexpr (ORDER == 0) {  // row f3 (learned R fused): the output transform of the value branch
    if (p.lq_out == 2) {
      // o T^T: lane owns outputs n = lane + 32 m, y_n = sum_k o_k T[n][k] (T rows in shared memory)
      float ya[4] = {0.f, 0.f, 0.f, 0.f}, yb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
      for (int k = 0; k < 128; k += 2) {
        const float o0 = row[k], o1 = row[k + 1];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          ya[m] = fmaf(o0, s_t[(lane + 32 * m) * LT_STRIDE + k], ya[m]);
          yb[m] = fmaf(o1, s_t[(lane + 32 * m) * LT_STRIDE + k + 1], yb[m]);
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) orow[lane + 32 * m] = ya[m] + yb[m];
      return;
    }
    if (p.lq_out == 1) {  // the block Hadamard inverse at the runtime order, then the signs
      const float a0 = x[0] + x[1], a1 = x[0] - x[1], a2 = x[2] + x[3], a3 = x[2] - x[3];
      x[0] = a0 + a2;
      x[1] = a1 + a3;
      x[2] = a0 - a2;
      x[3] = a1 - a3;
#pragma unroll 1
      for (int k = 0; (4 << k) < p.lq_order; ++k) {
        const float sgn = ((lane >> k) & 1) ? -1.f : 1.f;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float o = __shfl_xor_sync(0xffffffffu, x[u], 1 << k);
          x[u] = fmaf(sgn, x[u], o);
        }
      }
      const float inv = rsqrtf((float)p.lq_order);  // a power of two: exact
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u] *= inv;
        if ((sgw >> (4 * (lane & 7) + u)) & 1u) x[u] = -x[u];
      }
    }
  } else if (p.rotate && p.rot_v) {
    const float a0 = x[0] + x[1], a1 = x[0] - x[1], a2 = x[2] + x[3], a3 = x[2] - x[3];
    x[0] = a0 + a2;
    x[1] = a1 + a3;
    x[2] = a0 - a2;
    x[3] = a1 - a3;
#pragma unroll
    for (int k = 0; (4 << k) < ORDER; ++k) {
      const float sgn = ((lane >> k) & 1) ? -1.f : 1.f;  // upper half of the pair: o - x
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float o = __shfl_xor_sync(0xffffffffu, x[u], 1 << k);
        x[u] = fmaf(sgn, x[u], o);  // o -+ x, one rounding
      }
    }
    const float inv = (float)(1.0 / sqrt((double)ORDER));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[u] *= inv;
      if ((sgw >> (4 * (lane & 7) + u)) & 1u) x[u] = -x[u];
    }
  }
  reinterpret_cast<float4*>(orow)[lane] = make_float4(x[0], x[1], x[2], x[3]);
}

// K2+K3.  grid (kv head, split, sequence); NWARPS warps, one CTA per SM.  With
// APPEND the last warp writes the step's new K/V token (bit-exact f64) while the
// other DW warps stream their tiles through private rings of NSTG stages of C
// cells (one mbarrier per stage, one bulk copy per cell).
template <int NT, int ORDER, bool APPEND, int C, bool CL>
__global__ void __launch_bounds__(NWARPS * 32, 1)
    decode_tma_kernel(const __grid_constant__ DecodeParams p, const __grid_constant__ Signs signs) {
  constexpr int DW = APPEND ? NWARPS - 1 : NWARPS;
  constexpr int NSTG = RING_CELLS / C;
  // QK on the int8 tensor path (u8 codes x s8 query digits) for one column tile of
  // q heads; two (G = 8) keep the fp16 hi/lo HMMA path, which needs fewer B registers
  constexpr bool QK_INT8 = NT == 1;
  constexpr int STG = C * CELL;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + SM_BARS);
  uint16_t* sfrag = reinterpret_cast<uint16_t*>(sm + SM_FRAG);  // [NT][8 k-steps][32 lanes][2 regs][2 halves]
  float* obuf = reinterpret_cast<float*>(sm + SM_OBUF);         // [G][128]
  float* s_sumq = reinterpret_cast<float*>(sm + SM_MISC);       // [8]
  float* s_ksc = s_sumq + 8;                                    // [8]
  float* s_lse = s_sumq + 25;                                   // [8] (cluster merge)
  float* s_mstar = s_sumq + 40;                                 // [8] CTA reference point per q head
  float* s_lnew = s_sumq + 48;                                  // [8] new token's logits (APPEND)
  float* s_qrot = reinterpret_cast<float*>(sm + SM_QROT);
  float* s_vnew = reinterpret_cast<float*>(sm + SM_VNEW);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, i = lane & 3;
  const int h = blockIdx.x, split = blockIdx.y, b = blockIdx.z;
  const uint32_t k1024 = p.f16x2_1024;
  const int G = p.G, H = p.pool.H;
  const int64_t cta_id = ((int64_t)b * p.splits + split) * H + h;
  if (p.trace && threadIdx.x == 0) {
    p.trace[cta_id * 16 + 0] = gtimer();
    p.trace[cta_id * 16 + 1] = clk64();
    for (int k = 2; k < 16; ++k) p.trace[cta_id * 16 + k] = 0ull;
  }

  // a host-staged query (kvr_step_ring) cannot change during this launch: its read (over the bus
  // from pinned memory) goes out first, beside the length's, and overlaps the previous grid's tail
  float qx[4] = {0.f, 0.f, 0.f, 0.f};
  if (p.q_pre_wait && warp < G) load_q4(p.q, p.q_dtype, ((int64_t)b * p.nq + (int64_t)h * G + warp) * 128 + 4 * lane, qx);

  // ---- prologue (independent of the previous grid): split range from max_len,
  // the cell addresses of this warp's first 64 tiles, barrier init.
  // Warp w owns the groups g = w, w + DW, ... of C consecutive tiles of the split;
  // its j-th tile is t = lo + C (w + DW (j / C)) + j % C.
  const int n_tiles_max = (p.max_len + 15) >> 4;
  const int per = p.split_tiles;
  const int lo = min(n_tiles_max, split * per);
  const int hi_max = min(n_tiles_max, lo + per);
  const bool tile_warp = warp < DW;
  const int32_t* btrow = p.bt + (int64_t)b * p.bt_stride;
  const int cps = p.cps_log2;  // log2(cells of one head per page)
  auto tile_of = [&](int j) { return lo + C * (warp + DW * (j / C)) + j % C; };
  // lane l of window w holds the address of this warp's tile j = 32 w + l
  auto page_window = [&](int w) -> int {
    const int t = tile_of(32 * w + lane);
    return (tile_warp && t < hi_max) ? __ldg(&btrow[t >> cps]) : 0;
  };
  const uint8_t* head_base = p.pool.base + (int64_t)(h << cps) * p.pool.cell_bytes;
  const int cmask = (1 << cps) - 1;
  auto window_addr = [&](int w, int page) -> const uint8_t* {
    const int t = tile_of(32 * w + lane);
    return head_base + (int64_t)page * p.pool.page_bytes + (t & cmask) * p.pool.cell_bytes;
  };
  int wnext = page_window(1), win_idx = 0;
  const uint8_t* wcur = window_addr(0, page_window(0));
  // the length and the new token's slot (host-written, read before the wait): one
  // load per CTA, broadcast through shared memory (they may live in mapped host memory)
  int* s_len = reinterpret_cast<int*>(s_sumq + 58);
  long long* s_slot = reinterpret_cast<long long*>(s_sumq + 60);
  // ... unless the previous grid writes them (meta_post_wait: the step ring's stage-copy kernel):
  // then everything waits here, and no cell is requested before the wait either (pre_groups = 0)
  if (p.meta_post_wait) pdl_wait();
  if (threadIdx.x == 0) {
    if (p.meta_post_wait) {
      // coherent loads, not the read-only (.nc) path: the lengths / slot ids were written by the
      // stage-copy kernel, a grid this one may have been launched beside (PDL); the .nc path returned
      // a previous step's values there (tools/soak_step.py: a step every few hundred decoded an older
      // length).  (Host-written metadata -- pinned or copied in before the launch -- keeps __ldg.)
      *s_len = *reinterpret_cast<const volatile int32_t*>(&p.lens[b]);
      if (APPEND) *s_slot = *reinterpret_cast<const volatile long long*>(&p.new_slot[b]);
    } else {
      *s_len = __ldg(&p.lens[b]);
      if (APPEND) *s_slot = __ldg(&p.new_slot[b]);
    }
  }
  // this lane's word of the sign vector (dims 4l..4l+3), read from the parameter
  // bank before the dependency wait (0 = no flips)
  const uint32_t sgw = p.has_signs ? signs.w[lane >> 3] : 0u;
  if (threadIdx.x < NWARPS * RING_CELLS) mbar_init(&bars[threadIdx.x], 1);
  // row f3 (learned instantiation): T is a parameter of the rotation (immutable), so its bulk copy
  // goes out before the dependency wait
  float* s_t = reinterpret_cast<float*>(sm + SM_LT);
  uint64_t* ltbar = reinterpret_cast<uint64_t*>(sm + SM_LTBAR);
  if constexpr (ORDER == 0)
    if (threadIdx.x == NWARPS * RING_CELLS) mbar_init(ltbar, 1);
  reinterpret_cast<uint2*>(sfrag)[threadIdx.x] = make_uint2(0u, 0u);  // 4 KB of query digits (padding = 0)
  fence_mbar_init();
  __syncthreads();
  if constexpr (ORDER == 0) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(ltbar, (uint32_t)LT_BYTES);
      bulk_g2s(s_t, p.lq, (uint32_t)LT_BYTES, ltbar);
    }
  }
  const int len_raw = *s_len;
  const int64_t new_slot = APPEND ? *s_slot : -1;

  const int len = min(len_raw, p.max_len);
  // APPEND: the step's token (position len - 1) is written and scored by the writer
  // warp straight from registers; the tiles cover the len_kv older tokens, so no
  // tile load waits for the write
  const bool app = APPEND && len > 0 && new_slot >= 0;
  const int len_kv = app ? len - 1 : len;
  const int t_new = (len - 1) >> 4;
  const bool app_owner = app && t_new >= lo && t_new < hi_max;  // this CTA writes + scores it
  const int n_tiles = (len_kv + 15) >> 4;
  const int hi = min(n_tiles, hi_max);
  // tiles from `guard` on may hold tokens written by the previous grid (the last
  // step's append): they are requested only after griddepcontrol.wait
  const int guard = max(len - 2, 0) >> 4;
  const int my_groups = (tile_warp && hi - lo - C * warp > 0) ? (hi - lo - C * warp + C * DW - 1) / (C * DW) : 0;

  uint8_t* ring_w = sm + warp * RING_CELLS * CELL;
  uint64_t* bar_w = bars + warp * RING_CELLS;
  auto advance_to = [&](int j) {  // warp-uniform, non-decreasing j
    if ((j >> 5) != win_idx) {
      wcur = window_addr(win_idx + 1, wnext);
      ++win_idx;
      wnext = page_window(win_idx + 1);
    }
  };
  const uint64_t pol = policy_evict_first();
  // group k -> stage k % NSTG: one expect_tx, one bulk copy per valid cell
  auto issue = [&](int k) {
    advance_to(C * k);
    const uint8_t* src[C];
#pragma unroll
    for (int c = 0; c < C; ++c)
      src[c] = reinterpret_cast<const uint8_t*>(
          __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(wcur), (C * k + c) & 31));
    if (elect_one()) {
      const int t0 = tile_of(C * k);
      const int nc = min(C, hi - t0);
      const int s = k % NSTG;
      fence_proxy_async();
      mbar_expect_tx(&bar_w[s], (uint32_t)(nc * CELL));
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (c < nc) {
          if (p.evict_first)
            bulk_g2s_hint(ring_w + s * STG + c * CELL, src[c], (uint32_t)CELL, &bar_w[s], pol);
          else
            bulk_g2s(ring_w + s * STG + c * CELL, src[c], (uint32_t)CELL, &bar_w[s]);
        }
    }
  };
  auto group_last = [&](int k) { return min(tile_of(C * k) + C, hi) - 1; };
  // the first pre_groups groups of this warp: immutable ones go out before the wait
  // on the previous grid (programmatic dependent launch overlaps them with its tail)
  int k0 = 0;
#pragma unroll 1
  for (; k0 < NSTG && k0 < p.pre_groups && k0 < my_groups && group_last(k0) < guard; ++k0) issue(k0);

  pdl_wait();  // q, the new token, the workspace and recent pages may come from the previous grid
  pdl_launch_dependents();
  uint32_t* s_ep = reinterpret_cast<uint32_t*>(s_sumq + 16);  // [8] merge epochs of this (sequence, kv head)
  if (p.merge_ll && threadIdx.x < 8) s_ep[threadIdx.x] = p.ws_epoch[((int64_t)b * H + h) * 8 + threadIdx.x];
  KVR_STAMP(11);  // past the grid-dependency wait
  // ---- the writer warp (no tiles of its own) quantizes + stores the new token's K
  // and V rows bit-exactly (f64, reference arithmetic) right away, overlapping the
  // query prep and the main loop of the others; scored once the rotated q is in smem
  float newd[2][4];
  bool new_ok = true;
  if (APPEND && warp == DW && app_owner) {
    new_ok = append_rows_exact<ORDER>(p, signs, b, h, newd, p.trace && lane == 0 ? p.trace + cta_id * 16 : nullptr);
    *reinterpret_cast<float4*>(s_vnew + 4 * lane) = make_float4(newd[1][0], newd[1][1], newd[1][2], newd[1][3]);
  }
  if (threadIdx.x == 0 && len_raw > p.max_len && p.flags && h == 0 && split == 0)
    atomicOr(p.flags, KVR_FLAG_LEN_OVERFLOW);

  if (!p.q_pre_wait && warp < G) load_q4(p.q, p.q_dtype, ((int64_t)b * p.nq + (int64_t)h * G + warp) * 128 + 4 * lane, qx);
  if (p.trace) {  // q landed
    asm volatile("" ::"f"(qx[0]), "f"(qx[1]), "f"(qx[2]), "f"(qx[3]));
    KVR_STAMP(13);
  }
#pragma unroll 1
  for (int k = k0; k < NSTG && k < my_groups; ++k) issue(k);

  // ---- query prep: warp j < 4 NT owns q head j of this kv head (sign flip + fp32
  // butterfly, power-of-two normalisation, fp16 hi/lo split in MMA-fragment order);
  // columns j >= G are zero padding (qx = 0)
  if (warp < 4 * NT) {
    const int j = warp;
    float x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[u] = qx[u];
      if (ORDER != 0 && p.rotate && ((sgw >> (4 * (lane & 7) + u)) & 1u)) x[u] = -x[u];
    }
    if constexpr (ORDER == 0) {
      // row f3: q' = q T (T = diag(s) H_blk R composed, rotation.py:171-184) in fp32 from shared
      // memory: lane owns n = lane + 32 m while it sums over k (row stride 129: conflict-free), then
      // the lanes trade back to dims 4 l .. 4 l + 3 through the head's row of s_qrot
      float* s_x = s_qrot + j * 128;
      *reinterpret_cast<float4*>(s_x + 4 * lane) = make_float4(x[0], x[1], x[2], x[3]);
      __syncwarp();
      mbar_wait(ltbar, 0);
      float ya[4] = {0.f, 0.f, 0.f, 0.f}, yb[4] = {0.f, 0.f, 0.f, 0.f};
      if (j < G) {
#pragma unroll 4
        for (int k = 0; k < 128; k += 2) {
          const float x0 = s_x[k], x1 = s_x[k + 1];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            ya[m] = fmaf(x0, s_t[k * LT_STRIDE + lane + 32 * m], ya[m]);
            yb[m] = fmaf(x1, s_t[(k + 1) * LT_STRIDE + lane + 32 * m], yb[m]);
          }
        }
      }
      __syncwarp();
#pragma unroll
      for (int m = 0; m < 4; ++m) s_x[lane + 32 * m] = ya[m] + yb[m];
      __syncwarp();
      const float4 y4 = *reinterpret_cast<const float4*>(s_x + 4 * lane);
      x[0] = y4.x;
      x[1] = y4.y;
      x[2] = y4.z;
      x[3] = y4.w;
    } else if (p.rotate) {
      const float a0 = x[0] + x[1], a1 = x[0] - x[1], a2 = x[2] + x[3], a3 = x[2] - x[3];
      x[0] = a0 + a2;
      x[1] = a1 + a3;
      x[2] = a0 - a2;
      x[3] = a1 - a3;
#pragma unroll
      for (int k = 0; (4 << k) < ORDER; ++k) {
        const float sgn = ((lane >> k) & 1) ? -1.f : 1.f;  // upper half of the pair: o - x
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float o = __shfl_xor_sync(0xffffffffu, x[u], 1 << k);
          x[u] = fmaf(sgn, x[u], o);  // o -+ x, one rounding
        }
      }
      const float inv = (float)(1.0 / sqrt((double)ORDER));
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] *= inv;
    }
    if (APPEND && app_owner) {  // hand the rotated q to the writer warp
      *reinterpret_cast<float4*>(s_qrot + j * 128 + 4 * lane) = make_float4(x[0], x[1], x[2], x[3]);
      named_bar_arrive(2, (4 * NT + 1) * 32);
    }
    if constexpr (QK_INT8) {
      float amax = fmaxf(fmaxf(fabsf(x[0]), fabsf(x[1])), fmaxf(fabsf(x[2]), fabsf(x[3])));
      amax = warp_max(amax);
      // q' = rint(q 2^(19 - e2)), |q'| < 2^20, as three balanced base-128 digits
      // q' = p0 + 128 p1 + 16384 p2 (p0, p1 in [-64, 63], |p2| <= 64): the int8 IMMA
      // columns.  Lane l owns dims 4l..4l+3; dim d sits in IMMA m = ((d >> 4) & 1) +
      // 2 (d & 1) (odd dims are the high nibbles), B register (d >> 3) & 1, byte
      // (d >> 1) & 3 of lane (column * 4 + d / 32).
      const int e2 = amax > 0.f ? ilog2_pos(amax) : 0;
      const float qs = exp2i(19 - e2);
      int qsum = 0;
      uint8_t* s8 = reinterpret_cast<uint8_t*>(sfrag);  // [tile][m][lane][2 regs][4 bytes]
  #pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int d = 4 * lane + u, rem = d & 31;
        const int qi = __float2int_rn(x[u] * qs);
        qsum += qi;
        const int p0 = ((qi + 64) & 127) - 64;
        const int t1 = (qi - p0) >> 7;
        const int p1 = ((t1 + 64) & 127) - 64;
        const int p2 = (t1 - p1) >> 7;
        const int m = ((rem >> 4) & 1) + 2 * (rem & 1), reg = (rem >> 3) & 1, e = (rem >> 1) & 3, ii = d >> 5;
        const int pl[3] = {p0, p1, p2};
  #pragma unroll
        for (int pp = 0; pp < 3; ++pp) {
          int t, c;
          if (NT == 1) {  // tile 0: (head, plane 0|1) pairs; tile 1: (head, plane 2) on even columns
            t = pp < 2 ? 0 : 1;
            c = pp < 2 ? 2 * j + pp : 2 * j;
          } else {  // tiles 0/1: heads 0-3 / 4-7 planes 0|1; tile 2: plane 2 of heads (c/2, 4 + c/2)
            t = pp < 2 ? (j >> 2) : 2;
            c = pp < 2 ? 2 * (j & 3) + pp : 2 * (j & 3) + (j >> 2);
          }
          s8[(((t * 4 + m) * 32 + c * 4 + ii) * 2 + reg) * 4 + e] = (uint8_t)(int8_t)pl[pp];
        }
      }
      qsum = __reduce_add_sync(0xffffffffu, qsum);
      if (lane == 0) {
        s_sumq[j] = (float)qsum;
        s_ksc[j] = exp2i(e2 - 19) * LOG2E * (float)(1.0 / sqrt(128.0));
      }
  
    } else {
      float amax = fmaxf(fmaxf(fabsf(x[0]), fabsf(x[1])), fmaxf(fabsf(x[2]), fabsf(x[3])));
      amax = warp_max(amax);
      const int e2 = amax > 0.f ? ilog2_pos(amax) - 13 : 0;  // q' = q 2^-e2, max|q'| in [2^13, 2^14)
      const float qs = exp2i(-e2);
      float hs = 0.f;
  #pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int d = 4 * lane + u, rem = d & 31;
        const int ii = d >> 5, s = 2 * (rem >> 3) + ((rem & 3) >> 1), slot2 = rem & 1, e = (rem >> 2) & 1;
        const float v = x[u] * qs;
        const float hi_ = __half2float(__float2half_rn(v));
        const float lo_ = __half2float(__float2half_rn(v - hi_));
        hs += hi_ + lo_;
        const float f = slot2 ? (1.0f / 16.0f) : 1.0f;  // x16 nibble slots
        const int nt = j >> 2, col = 2 * (j & 3);
        // sfrag[nt][s][lane'][slot2][e]: lane' = col * 4 + ii owns B-fragment word slot2
        const int base = (nt * 8 + s) * 128 + slot2 * 2 + e;
        sfrag[base + ((col + 0) * 4 + ii) * 4] = __half_as_ushort(__float2half_rn(hi_ * f));
        sfrag[base + ((col + 1) * 4 + ii) * 4] = __half_as_ushort(__float2half_rn(lo_ * f));
      }
      hs = warp_sum(hs);
      if (lane == 0) {
        s_sumq[j] = hs * 5.9604644775390625e-08f;  // x 2^-24 (MMA units)
        s_ksc[j] = exp2i(e2 + 24) * LOG2E * (float)(1.0 / sqrt(128.0));
      }
  
    }
  }
  KVR_STAMP(12);  // warp 0's query prep done
  if (APPEND) {  // the tile warps only: the writer warp joins again after the loop
    if (tile_warp) named_bar_sync(1, DW * 32);
  } else {
    __syncthreads();
  }
  // query B fragments: registers for one 8-column tile; with two (G = 8) they stay
  // in shared memory (one LDS.64 per k-step) to keep the loop inside 128 registers
  constexpr bool BQ_REG = NT == 1;
  constexpr int NTL = NT + 1;  // int8 column tiles: 3 digit planes x 4 NT heads (+ padding)
  const uint2* sfrag2 = reinterpret_cast<const uint2*>(sfrag);
  uint2 bq[BQ_REG ? (QK_INT8 ? NTL * 4 : 8 * NT) : 1];
  float sumq[NT], kscale[NT];
  // (tile warps only: the writer warp is not ordered after the query prep by barrier 1)
  if (BQ_REG && tile_warp) {
#pragma unroll
    for (int s = 0; s < (QK_INT8 ? NTL * 4 : 8 * NT); ++s) bq[BQ_REG ? s : 0] = sfrag2[s * 32 + lane];
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    // the int8 QK yields 16 S (integer combination of the nibble planes): fold the
    // 1/16 into the query sum and the scale (powers of two: the same roundings)
    sumq[nt] = tile_warp ? s_sumq[4 * nt + i] * (QK_INT8 ? 16.0f : 1.0f) : 0.f;
    kscale[nt] = tile_warp ? s_ksc[4 * nt + i] * (QK_INT8 ? 0.0625f : 1.0f) : 0.f;
  }

  // ---- the writer warp scores the new token (logits in log2 units)
  if (APPEND && warp == DW && app_owner) {
    if (p.trace && lane == 0) p.trace[cta_id * 16 + 8] = clk64();  // append done
    named_bar_sync(2, (4 * NT + 1) * 32);  // rotated q of every head in smem
    for (int j = 0; j < G; ++j) {
      const float4 qv = *reinterpret_cast<const float4*>(s_qrot + j * 128 + 4 * lane);
      const float dot =
          warp_sum(qv.x * newd[0][0] + qv.y * newd[0][1] + qv.z * newd[0][2] + qv.w * newd[0][3]);
      // a rejected (non-finite) token is not attended: no phantom zero key / value
      if (lane == 0) s_lnew[j] = new_ok ? dot * (LOG2E * (float)(1.0 / sqrt(128.0))) : -INFINITY;
    }
    __syncwarp();
  }

  float M[NT], lsum[NT];
  float acc[NT][8][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    M[nt] = -INFINITY;
    lsum[nt] = 0.f;
#pragma unroll
    for (int m = 0; m < 8; ++m)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[nt][m][c] = 0.f;
  }

  // ---- main loop over this warp's groups of C tiles ----------------------------------
  KVR_STAMP(2);  // main loop start
  int stg = 0;
  uint32_t phase = 0;
#pragma unroll 1
  for (int k = 0; k < my_groups; ++k) {
    const int tg = tile_of(C * k);  // first tile of the group
    const uint8_t* st = ring_w + stg * STG;
    mbar_wait(&bar_w[stg], phase);
    CellFrag f[C];
#pragma unroll
    for (int c = 0; c < C; ++c) load_cell_k(f[c], st + c * CELL, r, i);

    // ---- S = C_k q : 8 k-steps of m16n8k16 per 8-column tile and cell
    float scv[C][NT][4];  // S per (token r -> [0] | r + 8 -> [2]) and head of this lane
    if constexpr (QK_INT8) {
      // ---- S = C_k q' on the int8 tensor path: per cell and column tile, two IMMA
      // m16n8k32 on the low nibbles (mask 0x0F0F0F0F) into D_lo and two on the high
      // nibbles kept in place (mask 0xF0F0F0F0, = 16 c) into D_hi; S = D_lo + D_hi / 16
      // is exact.  Column tiles hold the query's three digit planes.
  #pragma unroll
      for (int c = 0; c < C; ++c) {
        const uint32_t kw0[4] = {f[c].ka.x, f[c].ka.y, f[c].ka.z, f[c].ka.w};
        const uint32_t kw1[4] = {f[c].kb.x, f[c].kb.y, f[c].kb.z, f[c].kb.w};
        float sp[NTL][4];
  #pragma unroll
        for (int t = 0; t < NTL; ++t) {
          int dlo[4] = {0, 0, 0, 0}, dhi[4] = {0, 0, 0, 0};
  #pragma unroll
          for (int m = 0; m < 4; ++m) {
            const uint32_t mask = m < 2 ? 0x0F0F0F0Fu : 0xF0F0F0F0u;
            const int w = 2 * (m & 1);
            const uint2 b0 = BQ_REG ? bq[BQ_REG ? t * 4 + m : 0] : sfrag2[(t * 4 + m) * 32 + lane];
            imma16832(m < 2 ? dlo : dhi, kw0[w] & mask, kw1[w] & mask, kw0[w + 1] & mask, kw1[w + 1] & mask, b0.x, b0.y);
          }
  #pragma unroll
          for (int q = 0; q < 4; ++q) sp[t][q] = (float)(dlo[q] * 16 + dhi[q]);  // 16 S, exact (< 2^24)
        }
  #pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          // planes of this lane's head(s): tile nt holds (p0, p1) in (c0, c1) / (c2, c3);
          // the plane-2 tile holds p2 in c0 / c2 (NT == 1) or c(nt) / c(2 + nt) (NT == 2)
          const int t2 = NTL - 1, q0 = NT == 1 ? 0 : nt, q1 = NT == 1 ? 2 : 2 + nt;
          scv[c][nt][0] = fmaf(16384.0f, sp[t2][q0], fmaf(128.0f, sp[nt][1], sp[nt][0]));
          scv[c][nt][2] = fmaf(16384.0f, sp[t2][q1], fmaf(128.0f, sp[nt][3], sp[nt][2]));
        }
      }
    } else {
      // C * NT independent accumulator chains of 8 HMMAs
  #pragma unroll
      for (int c = 0; c < C; ++c) {
  #pragma unroll
        for (int nt = 0; nt < NT; ++nt)
  #pragma unroll
          for (int q = 0; q < 4; ++q) scv[c][nt][q] = 0.f;
        const uint32_t kw0[4] = {f[c].ka.x, f[c].ka.y, f[c].ka.z, f[c].ka.w};
        const uint32_t kw1[4] = {f[c].kb.x, f[c].kb.y, f[c].kb.z, f[c].kb.w};
  #pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint32_t wa = kw0[s >> 1], wb = kw1[s >> 1];
          const uint32_t xa = (s & 1) ? (wa >> 8) : wa, xb = (s & 1) ? (wb >> 8) : wb;
          const uint32_t a0 = xa & 0x000F000Fu, a2 = xa & 0x00F000F0u;
          const uint32_t a1 = xb & 0x000F000Fu, a3 = xb & 0x00F000F0u;
  #pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const uint2 bb = BQ_REG ? bq[BQ_REG ? s : 0] : sfrag2[(nt * 8 + s) * 32 + lane];
            mma16816(scv[c][nt], a0, a1, a2, a3, bb.x, bb.y);
          }
        }
  #pragma unroll
        for (int nt = 0; nt < NT; ++nt) {  // hi + lo query halves
          scv[c][nt][0] += scv[c][nt][1];
          scv[c][nt][2] += scv[c][nt][3];
        }
      }
    }

    // V words and sidecars after the QK MMAs (keeps the register peak down), then
    // refill this stage with group k + NSTG
#pragma unroll
    for (int c = 0; c < C; ++c) load_cell_rest(f[c], st + c * CELL, r, i);
    if (k + NSTG < my_groups) {
      __syncwarp();
      issue(k + NSTG);
    }

    // ---- logits from the sidecars (sentinel rows: the scale slot holds the
    // offset and the codes are 0)
    float l0[C][NT], l1[C][NT], svc0[C], svc1[C], zv0[C], zv1[C];
    bool sentinel = false;
#pragma unroll
    for (int c = 0; c < C; ++c) sentinel |= (f[c].kz0 | f[c].kz1 | f[c].vz0 | f[c].vz1) > 15u;
    const bool rare = __any_sync(0xffffffffu, sentinel);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      float sk0 = f[c].sk0, sk1 = f[c].sk1, sv0 = f[c].sv0, sv1 = f[c].sv1;
      float zk0 = (float)f[c].kz0, zk1 = (float)f[c].kz1;
      // zv: a sentinel V token's offset (its codes are 0 and enter the PV product as
      // 0 - 0); every other token's zero point is inside its PV operand (c - z)
      zv0[c] = 0.f;
      zv1[c] = 0.f;
      if (rare) {
        if (f[c].kz0 == 0xFFu) { zk0 = -sk0; sk0 = 1.f; }
        if (f[c].kz1 == 0xFFu) { zk1 = -sk1; sk1 = 1.f; }
        if (f[c].vz0 == 0xFFu) { zv0[c] = sv0; sv0 = 1.f; }
        if (f[c].vz1 == 0xFFu) { zv1[c] = sv1; sv1 = 1.f; }
      }
      svc0[c] = sv0;
      svc1[c] = sv1;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        l0[c][nt] = (scv[c][nt][0] - zk0 * sumq[nt]) * (sk0 * kscale[nt]);
        l1[c][nt] = (scv[c][nt][2] - zk1 * sumq[nt]) * (sk1 * kscale[nt]);
      }
    }
    if (tg + C > hi || tg + C >= n_tiles) {  // a missing or partial tile in this group
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int t0 = ((tg + c) << 4) + r;
        const bool in = tg + c < hi;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          if (!in || t0 >= len_kv) l0[c][nt] = -INFINITY;
          if (!in || t0 + 8 >= len_kv) l1[c][nt] = -INFINITY;
        }
        // a masked token's weight p * s_v and offset term must be 0 whatever its slot
        // holds (a stale or never-written scale / sentinel may be Inf/NaN: 0 * NaN)
        if (!in || t0 >= len_kv) svc0[c] = zv0[c] = 0.f;
        if (!in || t0 + 8 >= len_kv) svc1[c] = zv1[c] = 0.f;
      }
    }
    // probabilities at the current reference point, p = 2^(l - M), and the PV
    // weights w = p s_v.  Lazy rescaling: M only moves when a weight exceeds 2^7
    // (log2(p s_v) > M + 7, so w * 2^8 stays inside fp16 range) or on the first logits
    float pr0[C][NT], pr1[C][NT];
    bool over = false;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const float ms = (M[nt] == -INFINITY) ? 0.f : M[nt];
      float lmax = -INFINITY;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        pr0[c][nt] = ex2f(l0[c][nt] - ms);
        pr1[c][nt] = ex2f(l1[c][nt] - ms);
        over |= fmaxf(pr0[c][nt] * svc0[c], pr1[c][nt] * svc1[c]) > 128.0f;
        lmax = fmaxf(lmax, fmaxf(l0[c][nt], l1[c][nt]));
      }
      over |= M[nt] == -INFINITY && lmax > -INFINITY;
    }
    if (__any_sync(0xffffffffu, over)) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        float tm = -INFINITY;  // max of log2(p s_v) over the group
#pragma unroll
        for (int c = 0; c < C; ++c)
          tm = fmaxf(tm, fmaxf(l0[c][nt] + __log2f(svc0[c]), l1[c][nt] + __log2f(svc1[c])));
        tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 4));
        tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 8));
        tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 16));
        if (tm > M[nt] + 7.0f) {
          const float alpha = (M[nt] == -INFINITY) ? 0.f : ex2f(M[nt] - tm);
          lsum[nt] *= alpha;
#pragma unroll
          for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[nt][m][q] *= alpha;
          M[nt] = tm;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            pr0[c][nt] = ex2f(l0[c][nt] - tm);
            pr1[c][nt] = ex2f(l1[c][nt] - tm);
          }
        }
      }
    }

    // sentinel V tokens' offsets, sum_t w_t offset_t per q head (rare groups only)
    float zt[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) zt[nt] = 0.f;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      uint32_t wlo[NT], whi[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const float p0 = pr0[c][nt], p1 = pr1[c][nt];  // = p_t * 2^(.)
        const float w0 = p0 * svc0[c], w1 = p1 * svc1[c];  // = p_t * s_v * 2^(.)
        lsum[nt] += p0 + p1;
        zt[nt] = fmaf(w0, zv0[c], fmaf(w1, zv1[c], zt[nt]));
        // fp16 hi/lo of w * 2^8 (w <= 2^7): 22-bit weights, the lo half out of fp16
        // subnormals for weights down to ~2^-21 of the reference point
        const float w0s = w0 * 256.0f, w1s = w1 * 256.0f;
        const float w0h = __half2float(__float2half_rn(w0s)), w1h = __half2float(__float2half_rn(w1s));
        wlo[nt] = movtrans(pack_h2(w0h, w0s - w0h));  // tokens 0..7  -> b0,b1
        whi[nt] = movtrans(pack_h2(w1h, w1s - w1h));  // tokens 8..15 -> b2,b3
      }

      // ---- O^T += (C_v - z)^T W : 8 m-tiles (16 dims each) of m16n8k16.  The A operand
      // is the exact signed integer c - z of each token as an fp16 (a nibble masked into
      // the mantissa of 1024.0, minus 1024 + z): the products then carry both signs, so
      // the tensor core's truncating fp32 accumulation has no systematic drift (raw
      // codes 0..15 against positive weights bias every output dim the same way).
      uint32_t off[2][2];  // [token pair][low | high nibble]: fp16x2 (1024 + z, 1024 + 16 z)
#pragma unroll
      for (int tp = 0; tp < 2; ++tp) {
        const uint32_t zz = tp ? f[c].vzp1 : f[c].vzp0;  // z of the pair's two tokens (bytes 0, 1)
        // [z_a, 0, z_b, 0]; a sentinel's 0xFF (its codes are 0, its offset is handled apart) -> 0: the
        // second PRMT replicates each byte's bit 7, set only by 0xFF (valid z <= 15)
#if KVR_PRMT_SENT
        const uint32_t x = prmt(zz, 0u, 0x4140u) & ~prmt(zz, 0u, 0x4948u);
#else
        const uint32_t x = prmt(rare ? (zz & ~__vcmpeq4(zz, 0x0000FFFFu)) : zz, 0u, 0x4140u);
#endif
        off[tp][0] = x + k1024;
        off[tp][1] = x * 16u + k1024;
      }
      uint32_t xr[2][2][8];  // [token pair (2i,2i+1)|(2i+8,2i+9)][word][dim e]
#pragma unroll
      for (int tp = 0; tp < 2; ++tp)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const uint32_t wa = q ? f[c].vw[2 * tp].y : f[c].vw[2 * tp].x;
          const uint32_t wb = q ? f[c].vw[2 * tp + 1].y : f[c].vw[2 * tp + 1].x;
          const uint32_t t0w = prmt(wa, wb, 0x5410u), t1w = prmt(wa, wb, 0x7632u);
          const uint32_t t0s = t0w >> 8, t1s = t1w >> 8;
          xr[tp][q][0] = hsub2_u32(and_or<0x000F000Fu>(t0w, k1024), off[tp][0]);
          xr[tp][q][1] = hsub2_u32(and_or<0x00F000F0u>(t0w, k1024), off[tp][1]);
          xr[tp][q][2] = hsub2_u32(and_or<0x000F000Fu>(t0s, k1024), off[tp][0]);
          xr[tp][q][3] = hsub2_u32(and_or<0x00F000F0u>(t0s, k1024), off[tp][1]);
          xr[tp][q][4] = hsub2_u32(and_or<0x000F000Fu>(t1w, k1024), off[tp][0]);
          xr[tp][q][5] = hsub2_u32(and_or<0x00F000F0u>(t1w, k1024), off[tp][1]);
          xr[tp][q][6] = hsub2_u32(and_or<0x000F000Fu>(t1s, k1024), off[tp][0]);
          xr[tp][q][7] = hsub2_u32(and_or<0x00F000F0u>(t1s, k1024), off[tp][1]);
        }
#pragma unroll
      for (int m = 0; m < 8; ++m)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          mma16816(acc[nt][m], xr[0][0][m], xr[0][1][m], xr[1][0][m], xr[1][1][m], wlo[nt], whi[nt]);
    }
    if (rare) {
      // sentinel V tokens: p * offset, the same for every dim -- summed over the 8 lanes
      // of the q head's column (lanes i, i + 4, ...) and added to the hi column of every
      // output row in accumulator units (x 2^8 weights; x 16 on the high-nibble tiles)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        float z = zt[nt];
        z += __shfl_xor_sync(0xffffffffu, z, 4);
        z += __shfl_xor_sync(0xffffffffu, z, 8);
        z += __shfl_xor_sync(0xffffffffu, z, 16);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const float u = (m & 1) ? 4096.0f : 256.0f;
          acc[nt][m][0] = fmaf(z, u, acc[nt][m][0]);
          acc[nt][m][2] = fmaf(z, u, acc[nt][m][2]);
        }
      }
    }
    if (++stg == NSTG) {
      stg = 0;
      phase ^= 1u;
    }
  }

  // ---- CTA merge: every warp publishes its reference points M and takes the CTA
  // maximum M*, stores its partial rescaled to M*, and one pass sums the warps.
  // Dims are stored permuted, p = (d % 16) * 8 + d / 16, with a 136-float head
  // stride, so both the stores (lane = (r, i)) and the summing reads hit 32 banks.
  __syncthreads();  // all warps are out of the loop: the rings are free
  KVR_STAMP(3);  // all warps out of the loop
  float* s_m = reinterpret_cast<float*>(sm);  // [NWARPS][8] reference points
  float* s_lw = s_m + NWARPS * 8;             // [NWARPS][8] rescaled softmax sums
  float* sred = s_lw + NWARPS * 8;            // [NWARPS][8][136] rescaled partials
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) lsum[nt] += __shfl_xor_sync(0xffffffffu, lsum[nt], o);
    if (r == 0) s_m[warp * 8 + 4 * nt + i] = tile_warp ? M[nt] : -INFINITY;
  }
  if (APPEND && warp == DW && lane < 8)  // the writer warp's partial: the new token alone
    s_m[DW * 8 + lane] = (app_owner && lane < G) ? s_lnew[lane] : -INFINITY;
  __syncthreads();
  KVR_STAMP(4);  // reference points published
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int j = 4 * nt + i;
    if (j < G && tile_warp) {
      float mstar = -INFINITY;
#pragma unroll
      for (int w = 0; w < NWARPS; ++w) mstar = fmaxf(mstar, s_m[w * 8 + j]);
      if (warp == 0 && r == 0) s_mstar[j] = mstar;
      const float sc = (M[nt] == -INFINITY) ? 0.f : ex2f(M[nt] - mstar);
      float* dst = sred + (warp * 8 + j) * 136 + r;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const float f = ((m & 1) ? 0x1p-12f : 0x1p-8f) * sc;  // undo the x 2^8 weights (x 16 high nibbles)
        dst[m * 8] = (acc[nt][m][0] + acc[nt][m][1]) * f;
        dst[(m + 8) * 8] = (acc[nt][m][2] + acc[nt][m][3]) * f;
      }
      if (r == 0) s_lw[warp * 8 + j] = lsum[nt] * sc;
    }
  }
  if (APPEND && warp == DW) {  // p = 1 at its own reference point, o = its V row
    const float4 vv = *reinterpret_cast<const float4*>(s_vnew + 4 * lane);
    const float vr[4] = {vv.x, vv.y, vv.z, vv.w};
    for (int j = 0; j < G; ++j) {
      const float mj = s_m[DW * 8 + j];
      float mstar = -INFINITY;
#pragma unroll
      for (int w = 0; w < NWARPS; ++w) mstar = fmaxf(mstar, s_m[w * 8 + j]);
      const float sc = (mj == -INFINITY) ? 0.f : ex2f(mj - mstar);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int dd = 4 * lane + u;
        sred[(DW * 8 + j) * 136 + (dd & 15) * 8 + (dd >> 4)] = (sc != 0.f) ? sc * vr[u] : 0.f;
      }
      if (lane == 0) s_lw[DW * 8 + j] = sc;
    }
  }
  __syncthreads();
  KVR_STAMP(5);  // rescaled warp partials in smem

  // ---- normalised (o, lse) of this split: thread x sums permuted slot pp of head j
  const int64_t hbase = (((int64_t)b * H + h) * p.splits) * 8;
  for (int x = threadIdx.x; x < G * 128; x += blockDim.x) {
    const int j = x >> 7, pp = x & 127, dd = (pp & 7) * 16 + (pp >> 3);
    float lt = 0.f, ot = 0.f;
#pragma unroll
    for (int w = 0; w < NWARPS; ++w) {  // tile warps (+ the writer warp's new token)
      lt += s_lw[w * 8 + j];
      ot += sred[(w * 8 + j) * 136 + pp];
    }
    const float o = (lt > 0.f) ? ot / lt : 0.f;
    const float lse = (lt > 0.f) ? s_mstar[j] + __log2f(lt) : -INFINITY;
    if (p.splits == 1 || CL) {
      obuf[j * 128 + dd] = o;
      if (CL && pp == 0) s_lse[j] = lse;
    } else if (p.merge_ll) {
      const int64_t hj = (((int64_t)b * H + h) * 8 + j) * 32 + split;
      const unsigned long long tag = (unsigned long long)(s_ep[j] + 1u) << 32;
      st_relaxed_u64(p.ll_o + hj * 128 + dd, tag | __float_as_uint(o));
      if (pp == 0) st_relaxed_u64(p.ll_lse + hj, tag | __float_as_uint(lse));
    } else {
      __stcg(&p.ws_o[(hbase + (int64_t)split * 8 + j) * 128 + dd], o);
      if (pp == 0) __stcg(&p.ws_lse[hbase + (int64_t)split * 8 + j], lse);
    }
  }
  if (CL) {
    // ---- split merge inside the thread-block cluster (grid.y = splits = cluster
    // size): CTA r merges the q heads j = r, r + S, ... from every CTA's shared
    // memory and applies the inverse rotation
    cluster_sync_all();
    KVR_STAMP(6);  // cluster barrier passed
    const int S = p.splits;
    const int rank = (int)cluster_rank();
    float* omerge = reinterpret_cast<float*>(sm);  // [8][128] in the (free) rings
    for (int j = rank; j < G; j += S) {
      if (threadIdx.x < 128) {
        const int dd = threadIdx.x;
        float lv[16], ov[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          lv[u] = u < S ? *dsmem_ptr(s_lse + j, (uint32_t)u) : -INFINITY;
          ov[u] = u < S ? *dsmem_ptr(obuf + j * 128 + dd, (uint32_t)u) : 0.f;
        }
        float mx = -INFINITY;
#pragma unroll
        for (int u = 0; u < 16; ++u) mx = fmaxf(mx, lv[u]);
        float tot = 0.f, ot = 0.f;
        if (mx != -INFINITY) {
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const float w = (lv[u] == -INFINITY) ? 0.f : ex2f(lv[u] - mx);
            tot += w;
            ot += w * ov[u];
          }
        }
        omerge[j * 128 + dd] = tot > 0.f ? ot / tot : 0.f;
      }
    }
    __syncthreads();
    if (warp < G && warp % S == rank) emit_head<ORDER>(p, sgw, b, h, warp, omerge + warp * 128, lane, s_t);
    KVR_STAMP(9);  // merged + stored
    cluster_sync_relaxed();  // every CTA's partial stays readable until all merges are done
    KVR_STAMP(10);
    return;
  }
  if (p.splits > 1 && !p.merge_inline) {  // the partial is final: decode_merge_kernel (next in the stream) merges
    KVR_STAMP(6);
    return;
  }
  if (p.merge_ll) {
    // ---- flag-in-data split merge: CTA j < G merges q head j.  No fence, no counter: each
    // 64-bit word carries its split's epoch tag, and the merger's threads poll (split, 4 dims)
    // words until every tag is this launch's (the whole grid is resident: one wave).
    const int S = p.splits, j = split;
    if (j >= G) return;
    __syncthreads();  // the rings / reduction space are free; this CTA's own words are out
    const uint32_t want = s_ep[j] + 1u;
    const int64_t hj = (((int64_t)b * H + h) * 8 + j) * 32;
    float* so = reinterpret_cast<float*>(sm);  // [S][128]
    float* sl = so + 32 * 128;                 // [S]

#pragma unroll 1
    for (int k = threadIdx.x; k < S * 33; k += blockDim.x) {
      if (k < S * 32) {
        const int sp = k >> 5, l = k & 31;
        const unsigned long long* a = p.ll_o + (hj + sp) * 128 + 4 * l;
        unsigned long long v0, v1, v2, v3;
        do {
          v0 = ld_relaxed_u64(a);
          v1 = ld_relaxed_u64(a + 1);
          v2 = ld_relaxed_u64(a + 2);
          v3 = ld_relaxed_u64(a + 3);
        } while ((uint32_t)(v0 >> 32) != want || (uint32_t)(v1 >> 32) != want || (uint32_t)(v2 >> 32) != want ||
                 (uint32_t)(v3 >> 32) != want);
        *reinterpret_cast<float4*>(so + sp * 128 + 4 * l) =
            make_float4(__uint_as_float((uint32_t)v0), __uint_as_float((uint32_t)v1), __uint_as_float((uint32_t)v2),
                        __uint_as_float((uint32_t)v3));
      } else {
        const int sp = k - S * 32;
        unsigned long long v;
        do {
          v = ld_relaxed_u64(p.ll_lse + hj + sp);
        } while ((uint32_t)(v >> 32) != want);
        sl[sp] = __uint_as_float((uint32_t)v);
      }
    }
    __syncthreads();
    KVR_STAMP(7);  // merge inputs landed
    {
      // all 16 warps: warp w owns dims 8 w .. 8 w + 7, lane = (split group sg = lane >> 3, dim); lane l
      // also holds split l's LSE (S <= 32), so the max and the weight sum are warp reductions and
      // each split's weight a shuffle.  Runs once per launch with no other warps to hide latency:
      // short per-warp instruction streams, every load independent.
      const float lv = lane < S ? sl[lane] : -INFINITY;
      float mx = lv;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float wl = (lv == -INFINITY) ? 0.f : ex2f(lv - mx);
      float tot = wl;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      const int sg = lane >> 3, dd = 8 * warp + (lane & 7);
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int sp = sg + 4 * k;
        const float w = __shfl_sync(0xffffffffu, wl, sp & 31);
        if (sp < S) acc = fmaf(w, so[sp * 128 + dd], acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 8);
      acc += __shfl_xor_sync(0xffffffffu, acc, 16);
      if (sg == 0) obuf[dd] = tot > 0.f ? acc / tot : 0.f;
    }
    __syncthreads();  // the merged row is in obuf
    if (warp == 0) emit_head<ORDER>(p, sgw, b, h, j, obuf, lane, s_t);
    if (threadIdx.x == 0) p.ws_epoch[((int64_t)b * H + h) * 8 + j] = want;  // read again only by the next launch
    KVR_STAMP(9);  // merged + stored
    return;
  }
  if (p.splits > 1) {
    // ---- inline split merge: the last CTA of (sequence, kv head) to publish its
    // partial merges all of them.  Its thread 0 pulls the S contiguous partials
    // ([S][8][128] o, [S][8] lse) into the free rings with two bulk copies (one
    // round trip), then every thread merges its (q head, dim) in compact loops --
    // once-per-launch code is kept short, it runs from a cold instruction cache.
    __syncthreads();  // every thread's partial stores precede thread 0's release
    int* s_last = reinterpret_cast<int*>(s_sumq + 56);
    const int S = p.splits;
    float* so = reinterpret_cast<float*>(sm);  // [S][8][128]
    float* sl = so + S * 1024;                 // [S][8]
    uint64_t* mbar = bars + NWARPS * RING_CELLS;
    if (threadIdx.x == 0) {
      // release the CTA's partial (ordered before by the barrier), acquire the others'
      uint32_t prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                   : "=r"(prev)
                   : "l"(p.ws_cnt + (int64_t)b * H + h)
                   : "memory");
      const int last = prev == (uint32_t)(S - 1);
      *s_last = last;
      if (last) {
        fence_proxy_async_global();  // the others' generic-proxy stores -> the bulk reads
        fence_proxy_async();         // this CTA's generic smem accesses -> the bulk writes
        mbar_init(mbar, 1);
        fence_mbar_init();
        mbar_expect_tx(mbar, (uint32_t)(S * 4096 + S * 32));
        bulk_g2s(so, p.ws_o + hbase * 128, (uint32_t)(S * 4096), mbar);
        bulk_g2s(sl, p.ws_lse + hbase, (uint32_t)(S * 32), mbar);
      }
    }
    __syncthreads();
    KVR_STAMP(6);  // partial stored, counter back
    if (!*s_last) return;
    mbar_wait(mbar, 0);
    KVR_STAMP(7);  // merge inputs landed
    // split weights once per q head (warp j, lane = split): w_s = 2^(lse_s - max),
    // normalised by their sum; then every (head, dim) thread is S FMAs
    float* sw = s_qrot;  // [8][32] normalised split weights (the query copy is dead)
    if (warp < G) {
      const float l = lane < S ? sl[lane * 8 + warp] : -INFINITY;
      const float mx = warp_max(l);
      const float w = (l == -INFINITY) ? 0.f : ex2f(l - mx);
      const float tot = warp_sum(w);
      sw[warp * 32 + lane] = tot > 0.f ? w / tot : 0.f;
    }
    __syncthreads();
#pragma unroll 1
    for (int x = threadIdx.x; x < G * 128; x += blockDim.x) {
      const int j = x >> 7, dd = x & 127;
      const float* wj = sw + j * 32;
      float ot = 0.f;
#pragma unroll 4
      for (int sp = 0; sp < S; ++sp) ot += wj[sp] * so[(sp * 8 + j) * 128 + dd];
      obuf[j * 128 + dd] = ot;
    }
    __syncthreads();
    if (warp < G) emit_head<ORDER>(p, sgw, b, h, warp, obuf + warp * 128, lane, s_t);
    if (threadIdx.x == 0) p.ws_cnt[(int64_t)b * H + h] = 0u;  // read again only after this grid completes
    KVR_STAMP(9);  // merged + stored
    return;
  }
  __syncthreads();
  // ---- output: one warp per q head
  if (warp < G) emit_head<ORDER>(p, sgw, b, h, warp, obuf + warp * 128, lane, s_t);
  KVR_STAMP(10);
}

// ---------------------------------------------------------------------------
// BF16-pool decode (the reference's BF16 baseline pool: raw bf16 K / V rows, no rotation,
// cache.py:115-118, attention.py:67-71) -- the comparison point for the INT4 kernel.
// A 16-token cell of one head is 32 rows of 256 B (16 K | 16 V).  Grid (kv head, split,
// sequence), 8 warps; each warp streams its cells as two SW128 TMA boxes (the pool viewed
// as a 2-D tensor of 256-B rows) through a 2-stage ring, and per cell runs
//   S = K q on mma.sync m16n8k16 bf16 (K fragments by ldmatrix from the swizzled tile,
//       q split hi + lo bf16 in the columns of an 8-wide tile),
//   an online softmax in log2 units,
//   O^T += V^T P (V^T fragments by ldmatrix.trans, P hi + lo bf16 via movmatrix),
// then the CTA merge and, with splits, decode_merge_kernel (no inverse rotation).
namespace bfd {
constexpr int NW = 8;
constexpr int TILE = 8192;
constexpr int NSTG = 2;
constexpr int OFF_BARS = NW * NSTG * TILE;  // 128 KB of rings
constexpr int SM_M = OFF_BARS + 256;        // [NW][8] reference points
constexpr int SM_L = SM_M + NW * 8 * 4;    // [NW][8] softmax sums
constexpr int SM_RED = SM_L + NW * 8 * 4;  // [NW][8][128] partials
constexpr int SM_MSTAR = SM_RED + NW * 8 * 128 * 4;
constexpr int SM_TOTAL = SM_MSTAR + 64 + 1024;
}  // namespace bfd

KVR_DEV void ldsm_x4_u(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
KVR_DEV void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
KVR_DEV void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
KVR_DEV uint32_t pack_bf2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
// hi + lo bf16 split of x: (bf16(x), bf16(x - bf16(x)))
KVR_DEV void split_bf(float x, float& hi, float& lo) {
  hi = __bfloat162float(__float2bfloat16_rn(x));
  lo = x - hi;
}

template <int NT>
__global__ void __launch_bounds__(bfd::NW * 32, 1)
    decode_bf16_kernel(const __grid_constant__ DecodeParams p, const __grid_constant__ CUtensorMap map) {
  using namespace bfd;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BARS);
  float* s_m = reinterpret_cast<float*>(sm + SM_M);
  float* s_lw = reinterpret_cast<float*>(sm + SM_L);
  float* sred = reinterpret_cast<float*>(sm + SM_RED);
  float* s_mstar = reinterpret_cast<float*>(sm + SM_MSTAR);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, i = lane & 3;
  const int h = blockIdx.x, split = blockIdx.y, b = blockIdx.z;
  const int G = p.G, H = p.pool.H;
  if (threadIdx.x < NW * NSTG) mbar_init(&bars[threadIdx.x], 1);
  fence_mbar_init();
  if (threadIdx.x == 0) prefetch_tensormap(&map);
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();

  const int len = min(__ldg(&p.lens[b]), p.max_len);
  const int n_tiles = (len + 15) >> 4;
  const int per = (((p.max_len + 15) >> 4) + p.splits - 1) / p.splits;
  const int lo = min(n_tiles, split * per), hi = min(n_tiles, lo + per);
  const int my = hi - lo - warp > 0 ? (hi - lo - warp + NW - 1) / NW : 0;
  const int32_t* btrow = p.bt + (int64_t)b * p.bt_stride;
  const int cpp = p.pool.P >> 4;  // cells of a head per page
  uint8_t* ring = sm + warp * NSTG * TILE;
  uint64_t* bw = bars + warp * NSTG;
  auto issue = [&](int k) {
    if (elect_one()) {
      const int t = lo + warp + k * NW;
      const int page = __ldg(&btrow[t / cpp]);
      const int64_t row = ((int64_t)page * p.pool.page_bytes + (int64_t)(h * cpp + t % cpp) * p.pool.cell_bytes) >> 8;
      uint8_t* dst = ring + (k % NSTG) * TILE;
      mbar_expect_tx(&bw[k % NSTG], TILE);
      tma_load_2d(dst, &map, &bw[k % NSTG], 0, (int32_t)row);
      tma_load_2d(dst + TILE / 2, &map, &bw[k % NSTG], 64, (int32_t)row);
    }
    __syncwarp();
  };
  for (int k = 0; k < NSTG && k < my; ++k) issue(k);

  // q as the B operand: column n = lane >> 2 of tile nt is (head 4 nt + n / 2, hi | lo); the
  // 1/sqrt(d) and log2(e) are applied to S
  uint32_t qb[NT][8][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int head = 4 * nt + (r >> 1);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        float v[2] = {0.f, 0.f};
        if (head < G) {
#pragma unroll
          for (int u = 0; u < 2; ++u)
            v[u] = load_q(p.q, p.q_dtype, ((int64_t)b * p.nq + (int64_t)h * G + head) * 128 + 16 * ks + 8 * hf + 2 * i + u);
        }
        float h0, l0, h1, l1;
        split_bf(v[0], h0, l0);
        split_bf(v[1], h1, l1);
        qb[nt][ks][hf] = (r & 1) ? pack_bf2(l0, l1) : pack_bf2(h0, h1);
      }
  }
  const float qk = LOG2E * (float)(1.0 / sqrt(128.0));
  float M[NT], lsum[NT], acc[NT][8][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    M[nt] = -INFINITY;
    lsum[nt] = 0.f;
#pragma unroll
    for (int m = 0; m < 8; ++m)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[nt][m][c] = 0.f;
  }
  const int arow = (lane & 7) + 8 * ((lane >> 3) & 1), acol = lane >> 4;  // K: ldmatrix.x4 lane -> (token, chunk)
  const int vrow = (lane & 7) + 8 * (lane >> 4), vcol = (lane >> 3) & 1;  // V: ldmatrix.x4.trans
#pragma unroll 1
  for (int k = 0; k < my; ++k) {
    const int st = k % NSTG;
    mbar_wait(&bw[st], (k / NSTG) & 1);
    const uint8_t* tile = ring + st * TILE;
    const uint32_t tb = smem_u32(tile);
    const int t0 = (lo + warp + k * NW) * 16;
    if (t0 + 16 > len) {  // the last, partial cell: zero the V rows past the length (stale slots)
      for (int x = lane; x < 16 * 16; x += 32) {
        const int tok = x >> 4, c = x & 15;
        if (t0 + tok >= len)
          *reinterpret_cast<uint4*>(const_cast<uint8_t*>(tile) + (c >> 3) * (TILE / 2) + (16 + tok) * 128 +
                                    (((c & 7) ^ ((16 + tok) & 7)) << 4)) = make_uint4(0u, 0u, 0u, 0u);
      }
      __syncwarp();
    }
    // ---- S = K q
    float sa[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int c = 0; c < 4; ++c) sa[nt][c] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int ch = 2 * ks + acol;
      uint32_t a[4];
      ldsm_x4_u(tb + (ch >> 3) * (TILE / 2) + arow * 128 + (((ch & 7) ^ (arow & 7)) << 4), a);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) mma_bf16(sa[nt], a, qb[nt][ks][0], qb[nt][ks][1]);
    }
    // ---- online softmax (lane: tokens r, r + 8 of head 4 nt + i)
    float p0[NT], p1[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float l0 = (sa[nt][0] + sa[nt][1]) * qk, l1 = (sa[nt][2] + sa[nt][3]) * qk;
      if (t0 + r >= len) l0 = -INFINITY;
      if (t0 + r + 8 >= len) l1 = -INFINITY;
      float mx = fmaxf(l0, l1);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      if (mx > M[nt]) {
        const float alpha = (M[nt] == -INFINITY) ? 0.f : ex2f(M[nt] - mx);
        lsum[nt] *= alpha;
#pragma unroll
        for (int m = 0; m < 8; ++m)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[nt][m][c] *= alpha;
        M[nt] = mx;
      }
      p0[nt] = (l0 == -INFINITY) ? 0.f : ex2f(l0 - M[nt]);
      p1[nt] = (l1 == -INFINITY) ? 0.f : ex2f(l1 - M[nt]);
      lsum[nt] += p0[nt] + p1[nt];
    }
    // ---- O^T += V^T P
    uint32_t wlo[NT], whi[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float h0, l0, h1, l1;
      split_bf(p0[nt], h0, l0);
      split_bf(p1[nt], h1, l1);
      wlo[nt] = movtrans(pack_bf2(h0, l0));  // tokens 0..7
      whi[nt] = movtrans(pack_bf2(h1, l1));  // tokens 8..15
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int ch = 2 * m + vcol, row = 16 + vrow;
      uint32_t a[4];
      ldsm_x4_t(tb + (ch >> 3) * (TILE / 2) + row * 128 + (((ch & 7) ^ (row & 7)) << 4), a);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) mma_bf16(acc[nt][m], a, wlo[nt], whi[nt]);
    }
    __syncwarp();
    if (k + NSTG < my) issue(k + NSTG);
  }

  // ---- CTA merge (reference points, rescaled partials, one summing pass)
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) lsum[nt] += __shfl_xor_sync(0xffffffffu, lsum[nt], o);
    if (r == 0) s_m[warp * 8 + 4 * nt + i] = M[nt];
  }
  __syncthreads();
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int j = 4 * nt + i;
    float mstar = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) mstar = fmaxf(mstar, s_m[w * 8 + j]);
    if (warp == 0 && r == 0) s_mstar[j] = mstar;
    const float sc = (M[nt] == -INFINITY) ? 0.f : ex2f(M[nt] - mstar);
    float* dst = sred + (warp * 8 + j) * 128;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      dst[16 * m + r] = (acc[nt][m][0] + acc[nt][m][1]) * sc;
      dst[16 * m + r + 8] = (acc[nt][m][2] + acc[nt][m][3]) * sc;
    }
    if (r == 0) s_lw[warp * 8 + j] = lsum[nt] * sc;
  }
  __syncthreads();
  const int64_t hbase = (((int64_t)b * H + h) * p.splits) * 8;
  for (int x = threadIdx.x; x < G * 128; x += blockDim.x) {
    const int j = x >> 7, dd = x & 127;
    float lt = 0.f, ot = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      lt += s_lw[w * 8 + j];
      ot += sred[(w * 8 + j) * 128 + dd];
    }
    const float o = lt > 0.f ? ot / lt : 0.f;
    if (p.splits == 1) {
      p.out[((int64_t)b * p.nq + (int64_t)h * G + j) * 128 + dd] = o;
    } else {
      __stcg(&p.ws_o[(hbase + (int64_t)split * 8 + j) * 128 + dd], o);
      if (dd == 0) __stcg(&p.ws_lse[hbase + (int64_t)split * 8 + j], lt > 0.f ? s_mstar[j] + __log2f(lt) : -INFINITY);
    }
  }
}

// Stage-in of one serving step's host inputs (kvr_step_ring): pinned staging -> its device twin,
// 16 B per thread.  Launched with programmatic dependent launch right after the previous step's
// decode: the copy (the slot's last reader finished long ago) overlaps that decode, then the grid
// waits for it, so the next decode -- chained to this grid -- still starts after the previous one.
__global__ void __launch_bounds__(1024) stage_copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, int n16) {
  // all of a thread's loads before its stores: one round trip over the bus for up to 64 KB
  uint4 v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = threadIdx.x + u * 1024;
    if (i < n16) v[u] = src[i];
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = threadIdx.x + u * 1024;
    if (i < n16) dst[i] = v[u];
  }
  pdl_launch_dependents();
  pdl_wait();
}

// Split merge (K3), launched right after a split decode with programmatic
// dependent launch: one CTA per (q head j, kv head, sequence), 512 threads =
// 128 dims x 4 split slices.  LSE-weighted sum of the splits' (o, lse)
// partials, then the inverse rotation of the value branch.
constexpr int MERGE_THREADS = 512;
template <int ORDER>
__global__ void __launch_bounds__(MERGE_THREADS)
    decode_merge_kernel(const __grid_constant__ DecodeParams p, const __grid_constant__ Signs signs) {
  __shared__ float s_w[MAX_SPLITS];
  __shared__ float s_red[16];
  __shared__ float s_o[4][128];
  const int j = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = p.splits, H = p.pool.H;
  const int dd = tid & 127, sl = tid >> 7;
  const int64_t hbase = (((int64_t)b * H + h) * S) * 8;
  // trace rows after the decode grid's: [0] entry, [1] past the wait, [2] exit (globaltimer)
  unsigned long long* tr = nullptr;
  if (p.trace && tid == 0)
    tr = p.trace + ((int64_t)gridDim.z * S * H + ((int64_t)b * H + h) * gridDim.x + j) * 16;
  if (tr) tr[0] = gtimer();
  pdl_wait();
  pdl_launch_dependents();
  if (tr) tr[1] = gtimer();
  // o-values of this thread's splits s = sl, sl + 4, ... (first 16 preloaded with the lse)
  float ov[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int s = sl + 4 * u;
    ov[u] = s < S ? __ldcg(p.ws_o + (hbase + (int64_t)s * 8 + j) * 128 + dd) : 0.f;
  }
  float l = -INFINITY;
  if (tid < S) l = __ldcg(p.ws_lse + hbase + (int64_t)tid * 8 + j);
  float m = warp_max(l);
  if (lane == 0) s_red[warp] = m;
  __syncthreads();
  if (tr) tr[3] = gtimer();
  m = s_red[lane & 15];
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float w = (tid < S && l != -INFINITY) ? ex2f(l - m) : 0.f;
  if (tid < S) s_w[tid] = w;
  float tw = warp_sum(w);
  __syncthreads();  // s_red reads done before reuse
  if (lane == 0) s_red[warp] = tw;
  __syncthreads();
  tw = 0.f;
#pragma unroll
  for (int q = 0; q < MERGE_THREADS / 32; ++q) tw += s_red[q];
  float acc = 0.f;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int s = sl + 4 * u;
    if (s < S) acc += s_w[s] * ov[u];
  }
#pragma unroll 8
  for (int s = sl + 64; s < S; s += 4) acc += s_w[s] * __ldcg(p.ws_o + (hbase + (int64_t)s * 8 + j) * 128 + dd);
  s_o[sl][dd] = acc;
  __syncthreads();
  if (warp == 0) {
    float x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int d = 4 * lane + u;
      const float v = s_o[0][d] + s_o[1][d] + s_o[2][d] + s_o[3][d];
      x[u] = tw > 0.f ? v / tw : 0.f;
    }
    if (p.rotate && p.rot_v) {
      const float a0 = x[0] + x[1], a1 = x[0] - x[1], a2 = x[2] + x[3], a3 = x[2] - x[3];
      x[0] = a0 + a2;
      x[1] = a1 + a3;
      x[2] = a0 - a2;
      x[3] = a1 - a3;
#pragma unroll
      for (int k = 0; (4 << k) < ORDER; ++k) {
        const float sgn = ((lane >> k) & 1) ? -1.f : 1.f;  // upper half of the pair: o - x
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float o = __shfl_xor_sync(0xffffffffu, x[u], 1 << k);
          x[u] = fmaf(sgn, x[u], o);  // o -+ x, one rounding
        }
      }
      const float inv = (float)(1.0 / sqrt((double)ORDER));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u] *= inv;
        if (p.has_signs && sign_bit(signs, 4 * lane + u)) x[u] = -x[u];
      }
    }
    float4* dst = reinterpret_cast<float4*>(p.out + ((int64_t)b * p.nq + (int64_t)h * p.G + j) * 128) + lane;
    *dst = make_float4(x[0], x[1], x[2], x[3]);
  }
  if (tr) tr[2] = gtimer();
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
    const uint8_t* cell = cell_of(p.pool, p.bt[(int64_t)b * p.bt_stride + t / p.pool.P], h, t % p.pool.P, ci);
    const bool bf = p.pool.prec == KVR_PREC_BF16;  // raw bf16 rows (cache.py:115-118)
    const uint16_t* kb = reinterpret_cast<const uint16_t*>(cell + cell_bf16(p.pool, 0, ci));
    const uint16_t* vb = reinterpret_cast<const uint16_t*>(cell + cell_bf16(p.pool, 1, ci));
    const float ks = bf ? 0.f : *reinterpret_cast<const float*>(cell + cell_kscale(p.pool, ci));
    const uint8_t kz = bf ? 0 : cell[cell_kzp(p.pool, ci)];
    const float vs = bf ? 0.f : *reinterpret_cast<const float*>(cell + cell_vscale(p.pool, ci));
    const uint8_t vz = bf ? 0 : cell[cell_vzp(p.pool, ci)];
    const uint8_t* kc = cell + cell_kcode(p.pool, ci);
    const uint8_t* vc = cell + cell_vcode(p.pool, ci);
    float dot = 0.f;
    for (int k = 0, x = lane; x < d; x += 32, ++k) {
      float kh;
      if (bf) {
        kh = __uint_as_float((uint32_t)kb[x] << 16);
      } else {
        const uint8_t byte = kc[x >> 1];
        const float c = (float)((x & 1) ? (byte >> 4) : (byte & 15));
        kh = (kz == 0xFF) ? ks : ks * (c - (float)kz);
      }
      dot += kh * sq[x];
    }
    dot = warp_sum(dot) * scale;
    const float mn = fmaxf(m, dot);
    const float a = exp2f((m - mn) * LOG2E), pw = exp2f((dot - mn) * LOG2E);
    l = l * a + pw;
    for (int k = 0, x = lane; x < d; x += 32, ++k) {
      float vh;
      if (bf) {
        vh = __uint_as_float((uint32_t)vb[x] << 16);
      } else {
        const uint8_t byte = vc[x >> 1];
        const float c = (float)((x & 1) ? (byte >> 4) : (byte & 15));
        vh = (vz == 0xFF) ? vs : vs * (c - (float)vz);
      }
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

// Workspace: split counters u32[B][H] first (padded to 256 B, so a workspace reused
// with another split count still finds them at zero), then lse f32[B][H][S][8],
// then o f32[B][H][S][8][128].
// (counters u32[B][H] | merge epochs u32[B][H][8]) -- zeroed once by the owner, left consistent by
// every launch -- padded to 256 B
static size_t ws_cnt_bytes(int batch, int H) { return ((size_t)batch * H * 9 * sizeof(uint32_t) + 255) & ~size_t(255); }
// the flag-in-data merge's words: split-count independent slots [B][H][8][32] lse and [.][128] o
static bool ws_has_ll(int batch, int H, int splits) {
  return splits > 8 && splits <= MERGE_INLINE_MAX && (long)batch * H * splits <= 256;
}
static size_t ws_ll_bytes(int batch, int H) { return (size_t)batch * H * 8 * 32 * 129 * sizeof(unsigned long long); }
size_t kvr_decode_ws_bytes(int batch, int H, int nq, int d, int splits) {
  (void)nq;
  (void)d;
  if (splits < 1) splits = 1;
  const size_t units = (size_t)batch * H * splits * 8;
  size_t bytes = ws_cnt_bytes(batch, H) + units * sizeof(float) + units * 128 * sizeof(float);
  bytes = (bytes + 255) & ~size_t(255);
  if (ws_has_ll(batch, H, splits)) bytes += ws_ll_bytes(batch, H);
  return (bytes + 255) & ~size_t(255);
}

// Split count: minimise (waves of one-CTA-per-SM) x (tiles per CTA) + a merge cost,
// keeping >= 2 tiles per warp; ties go to fewer splits.
int kvr_pick_splits(int batch, int H, int max_len, int P) {
  (void)P;
  const int sms = kvr_num_sms() > 0 ? kvr_num_sms() : 148;
  const int tiles = (max_len + 15) / 16;
  const long units = (long)batch * H;
  if (units <= 0 || tiles <= 0) return 1;
  int best = 1;
  double best_cost = 1e300;
  const long fill = sms / units;  // splits that fill the SMs in one wave
  for (int s = 1; s <= MAX_SPLITS; ++s) {
    const int per = (tiles + s - 1) / s;
    if (s > 1 && per < 2 * NWARPS) break;
    // above the inline-merge range only multiples of 16 and the one-wave fill are
    // tried (measured on C5 128k: other counts run 5-15 % slower)
    if (s > MERGE_INLINE_MAX && (s % 16) && s != fill) continue;
    const long ctas = units * s;
    const long waves = (ctas + sms - 1) / sms;
    // in tile-times (one tile ~ 1/15 of a warp's 0.9 us per cell): a CTA's fixed
    // prologue + epilogue ~ 80, its partial write (+ read in the merge) ~ 2, and the
    // latency of the split merge once (inline up to 32 splits; the merge kernel's
    // grows faster with the split count)
    const double merge = s <= MERGE_INLINE_MAX ? 24.0 + 0.25 * s : 32.0 + 0.5 * (s - MERGE_INLINE_MAX);
    const double cost = (double)waves * (80.0 + per + (s > 1 ? 2.0 : 0.0)) + (s > 1 ? merge : 0.0);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

// One launch of decode_tma_kernel with programmatic stream serialization (PDL: the
// prologue may overlap the previous grid) and, for 2..16 splits, a thread-block
// cluster spanning the splits of one (sequence, kv head) so they merge in DSMEM.
template <int NT, int ORDER, bool APP, bool CL>
static int launch_one(dim3 grid, size_t smem, cudaStream_t st, const DecodeParams& p, const Signs& sg) {
  auto kern = decode_tma_kernel<NT, ORDER, APP, NT == 1 ? 2 : KVR_NT2_CELLS, CL>;
  static bool set[KVR_MAX_DEVICES];  // per instantiation and device
  const int dev = kvr_current_device();
  if (!set[dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return KVR_ERR_CUDA;
    if (CL && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      return KVR_ERR_CUDA;
    set[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(NWARPS * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = grid.y;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CL ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, p, sg) == cudaSuccess ? 0 : KVR_ERR_CUDA;
}

// Can clusters of `splits` CTAs of this kernel be co-scheduled? (cached per size)
template <int NT, int ORDER, bool APP>
static bool cluster_ok(int splits, size_t smem) {
  static int cache_all[KVR_MAX_DEVICES][17];  // per device: 0 unknown, 1 yes, 2 no
  if (splits < 2 || splits > 16) return false;
  int* cache = cache_all[kvr_current_device()];
  if (!cache[splits]) {
    auto kern = decode_tma_kernel<NT, ORDER, APP, NT == 1 ? 2 : KVR_NT2_CELLS, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, splits, 1);
    cfg.blockDim = dim3(NWARPS * 32);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = splits;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    cache[splits] = (e == cudaSuccess && n >= 1) ? 1 : 2;
    if (e != cudaSuccess) (void)cudaGetLastError();
  }
  return cache[splits] == 1;
}

template <int ORDER>
static int launch_merge(const DecodeParams& p, const Signs& sg, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.G, p.pool.H, p.batch);
  cfg.blockDim = dim3(MERGE_THREADS);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_merge_kernel<ORDER>, p, sg) == cudaSuccess ? 0 : KVR_ERR_CUDA;
}

template <int NT, int ORDER, bool APP>
static int launch_sel(dim3 grid, size_t smem, cudaStream_t st, const DecodeParams& p, const Signs& sg) {
  if (p.use_cluster && cluster_ok<NT, ORDER, APP>((int)grid.y, smem))
    return launch_one<NT, ORDER, APP, true>(grid, smem, st, p, sg);
  if (int rc = launch_one<NT, ORDER, APP, false>(grid, smem, st, p, sg)) return rc;
  return (p.splits > 1 && !p.merge_inline) ? launch_merge<ORDER>(p, sg, st) : 0;
}

template <int NT, bool APP>
static int launch_tma(const DecodeParams& p, const Signs& sg, dim3 grid, size_t smem, int order, cudaStream_t st) {
  switch (order) {
    case 128: return launch_sel<NT, 128, APP>(grid, smem, st, p, sg);
    case 64: return launch_sel<NT, 64, APP>(grid, smem, st, p, sg);
    case 32: return launch_sel<NT, 32, APP>(grid, smem, st, p, sg);
    case 16: return launch_sel<NT, 16, APP>(grid, smem, st, p, sg);
  }
  return KVR_ERR_UNSUPPORTED;
}

int kvr_launch_stage_copy(void* dst, const void* src, int64_t bytes, cudaStream_t st) {
  if ((bytes & 15) || bytes > 65536 || ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15))
    return KVR_ERR_ARG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(1024);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, stage_copy_kernel, reinterpret_cast<uint4*>(dst), reinterpret_cast<const uint4*>(src),
                            (int)(bytes >> 4)) == cudaSuccess
             ? 0
             : KVR_ERR_CUDA;
}

static unsigned long long* g_trace = nullptr;
void kvr_set_decode_trace(void* trace) { g_trace = reinterpret_cast<unsigned long long*>(trace); }

int kvr_launch_decode(const void* q, int q_dtype, const Pool& pool, const int32_t* bt, int bt_stride,
                      const int32_t* lens, int batch, int nq, int max_len, int order, int rotate, int rot_v,
                      const Signs& s, int has, float* out, void* ws, size_t ws_bytes, int splits, cudaStream_t st,
                      const void* new_k, const void* new_v, int new_dtype, const int64_t* new_slot,
                      uint32_t* flags, int q_host_staged, const float* lq, int lq_out, int lq_order) {
  DecodeParams p{};
  p.q_pre_wait = q_host_staged == 1;
  p.meta_post_wait = q_host_staged == 2;
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
  // tuning switches (compile-time, for A/B builds with tools/build_variants.py; the
  // defaults are the measured best): one ring group per warp before the wait (a
  // full-ring burst queues the query load behind it), evict-first KV streaming,
  // inline split merge for 9..32 splits
  // (pool cells read before griddepcontrol.wait are only those no preceding grid on
  // the stream writes: after a store kernel on this stream the prefetch waits)
  p.pre_groups = (kvr_take_pool_written(st) || p.meta_post_wait) ? 0 : KVR_PREWAIT_GROUPS;
  p.evict_first = KVR_EVICT_FIRST;
  p.f16x2_1024 = 0x64006400u;
  int l2 = 0;
  while ((1 << l2) < pool.P) ++l2;
  const bool pow2 = (1 << l2) == pool.P;
  p.log2P = l2;
  Signs sg = s;
  if (!has) for (auto& x : sg.w) x = 0u;
  const bool tma_ok = pow2 && pool.prec == KVR_PREC_INT4 && pool.d == 128 && pool.T == 16 &&
                      (p.G == 1 || p.G == 2 || p.G == 4 || p.G == 8) &&
                      (reinterpret_cast<uintptr_t>(pool.base) & 15) == 0 && (pool.cell_bytes & 15) == 0;
  if (lq && !tma_ok) return KVR_ERR_UNSUPPORTED;  // row f3 fused only in the TMA kernel
  if (tma_ok) {
    if (splits <= 0) splits = kvr_pick_splits(batch, pool.H, max_len, pool.P);
    if (splits > MAX_SPLITS) splits = MAX_SPLITS;
    if (lq && splits > MERGE_INLINE_MAX) splits = MERGE_INLINE_MAX;  // row f3: merged in-grid (the merge kernel has no T)
    // the partials' space is required; the flag-in-data merge's words only where the caller sized
    // the workspace for them (merge_ll below checks that they fit)
    if (splits > 1 && ws_cnt_bytes(batch, pool.H) + (size_t)batch * pool.H * splits * 8 * 129 * sizeof(float) > ws_bytes)
      return KVR_ERR_ARG;
    p.splits = splits;
    p.split_tiles = (((max_len + 15) >> 4) + splits - 1) / splits;
    const size_t units = (size_t)batch * pool.H * splits * 8;
    p.ws_cnt = reinterpret_cast<uint32_t*>(ws);
    p.ws_epoch = p.ws_cnt + (size_t)batch * pool.H;
    p.ws_lse = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + ws_cnt_bytes(batch, pool.H));
    p.ws_o = p.ws_lse + units;
    size_t ll_end;
    {
      const size_t base = (ws_cnt_bytes(batch, pool.H) + units * sizeof(float) * 129 + 255) & ~size_t(255);
      p.ll_lse = reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(ws) + base);
      p.ll_o = p.ll_lse + (size_t)batch * pool.H * 8 * 32;
      ll_end = base + ws_ll_bytes(batch, pool.H);
    }
    if (lq) {  // row f3 fused: a merge inside the decode grid (the merge kernel has no T)
      if (new_slot) return KVR_ERR_UNSUPPORTED;
      p.lq = lq;
      p.lq_out = lq_out;
      p.lq_order = lq_order;
      p.rotate = 0;
      p.rot_v = 0;
    }
    dim3 grid(pool.H, splits, batch);
    const int ord = rotate ? order : 128;
    const size_t smem = lq ? decode_smem_bytes_lq() : decode_smem_bytes();
    int cl = 0;
    while ((16 << cl) < pool.P) ++cl;
    p.cps_log2 = cl;
#ifndef KVR_NO_CLUSTER
    // portable cluster sizes only: 16-CTA clusters of one-CTA-per-SM kernels do not
    // all co-schedule on B200 (a second wave appears), measured slower
    p.use_cluster = splits >= 2 && splits <= KVR_CLUSTER_MAX;
#else
    p.use_cluster = 0;
#endif
    p.merge_inline = KVR_MERGE_INLINE && !p.use_cluster && splits > 1 && splits <= MERGE_INLINE_MAX;
    // flag-in-data merge when the grid is one wave (the merger CTAs spin on the others' words)
    p.merge_ll = KVR_MERGE_LL && p.merge_inline && ws_has_ll(batch, pool.H, splits) && ll_end <= ws_bytes &&
                 (long)batch * pool.H * splits <= (kvr_num_sms() > 0 ? kvr_num_sms() : 148) && p.G <= 8;
    // the one-wave flag-in-data grids (C2-like: a short stream per CTA, the step a latency chain) take
    // their whole ring before the wait (C2 step 14.1 -> 13.9 us); the long streams keep one group
    // (a full-ring burst there queues the query load behind it: C5 1M +2 %)
    if (p.pre_groups > 0 && p.merge_ll) p.pre_groups = KVR_PREWAIT_GROUPS_LL;
    if (lq) return p.G == 8 ? launch_sel<2, 0, false>(grid, smem, st, p, sg) : launch_sel<1, 0, false>(grid, smem, st, p, sg);
    if (new_slot)
      return p.G == 8 ? launch_tma<2, true>(p, sg, grid, smem, ord, st) : launch_tma<1, true>(p, sg, grid, smem, ord, st);
    return p.G == 8 ? launch_tma<2, false>(p, sg, grid, smem, ord, st) : launch_tma<1, false>(p, sg, grid, smem, ord, st);
  }
  if (new_slot) return KVR_ERR_UNSUPPORTED;  // the fused append lives in the TMA kernel only
  if (pool.prec == KVR_PREC_BF16 && pool.d == 128 && pool.T == 16 && pool.P % 16 == 0 && p.G >= 1 && p.G <= 8 &&
      (reinterpret_cast<uintptr_t>(pool.base) & 255) == 0 && (pool.page_bytes & 255) == 0 && pool.cell_bytes == 8192 &&
      !getenv("KVR_BF16_DECODE_GENERIC")) {
    if (splits <= 0) splits = kvr_pick_splits(batch, pool.H, max_len, pool.P);
    if (splits > MAX_SPLITS) splits = MAX_SPLITS;
    if (splits > 1 && kvr_decode_ws_bytes(batch, pool.H, nq, 128, splits) > ws_bytes) return KVR_ERR_ARG;
    p.splits = splits;
    const size_t units = (size_t)batch * pool.H * splits * 8;
    p.ws_cnt = reinterpret_cast<uint32_t*>(ws);
    p.ws_lse = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + ws_cnt_bytes(batch, pool.H));
    p.ws_o = p.ws_lse + units;
    p.rotate = 0;
    p.rot_v = 0;
    CUtensorMap map;
    const uint64_t rows = (uint64_t)pool.num_pages * (uint64_t)pool.page_bytes / 256;
    if (kvr_encode_tensor_map_2d(&map, pool.base, 128, rows, 256, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B) != CUDA_SUCCESS)
      return KVR_ERR_CUDA;
    const size_t smem = bfd::SM_TOTAL;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pool.H, splits, batch);
    cfg.blockDim = dim3(bfd::NW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static bool attr_set[KVR_MAX_DEVICES][2];
    const int dev = kvr_current_device();
    cudaError_t e;
    if (p.G > 4) {
      if (!attr_set[dev][1]) {
        cudaFuncSetAttribute(decode_bf16_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set[dev][1] = true;
      }
      e = cudaLaunchKernelEx(&cfg, decode_bf16_kernel<2>, p, map);
    } else {
      if (!attr_set[dev][0]) {
        cudaFuncSetAttribute(decode_bf16_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set[dev][0] = true;
      }
      e = cudaLaunchKernelEx(&cfg, decode_bf16_kernel<1>, p, map);
    }
    if (e != cudaSuccess) return KVR_ERR_CUDA;
    return splits > 1 ? launch_merge<128>(p, sg, st) : 0;
  }
  if (pool.d > 256) return KVR_ERR_UNSUPPORTED;
  p.splits = 1;
  const int warps = 4;
  const size_t smem = (size_t)(pool.d + warps * pool.d + warps * 2) * sizeof(float);
  decode_generic_kernel<<<dim3(nq, batch), warps * 32, smem, st>>>(p, sg, pool.d);
  return 0;
}
