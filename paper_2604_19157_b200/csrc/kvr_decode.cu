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

constexpr int DEC_WARPS = 4;
constexpr float LOG2E = 1.4426950408889634f;

struct DecodeParams {
  Pool pool;
  const void* q;
  int q_dtype;
  const int32_t* bt;
  int bt_stride;
  const int32_t* lens;
  int batch, nq, G, splits, order, rotate, rot_v, has_signs, log2P;
  float* out;
  float* ws_o;    // [B][H][S][G][128]
  float* ws_lse;  // [B][H][S][G]
  uint32_t* ws_cnt;  // [B][H]
};

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

// fp32 block FWHT on rows of 128 held in shared memory, whole CTA cooperating.
// rows*64 butterflies per stage; inv = 1/sqrt(order).
KVR_DEV void cta_fwht128(float* s, int rows, int order) {
  for (int half = 1; half < order; half <<= 1) {
    for (int p = threadIdx.x; p < rows * 64; p += blockDim.x) {
      const int r = p >> 6, q = p & 63;
      const int blk = q / (order >> 1), w = q % (order >> 1);
      const int i = r * 128 + blk * order + (w / half) * 2 * half + (w % half);
      const float a = s[i], b = s[i + half];
      s[i] = a + b;
      s[i + half] = a - b;
    }
    __syncthreads();
  }
  const float inv = (float)(1.0 / sqrt((double)order));
  for (int i = threadIdx.x; i < rows * 128; i += blockDim.x) s[i] *= inv;
  __syncthreads();
}

struct TileRegs {
  uint4 k0, k1;          // K codes, tokens r and r+8 (16 B each: dims 32i..32i+31)
  uint2 v[4];            // V codes, tokens 2i, 2i+1, 2i+8, 2i+9 (8 B each: dims 16r..16r+15)
  float ks0, ks1, vs0, vs1;
  uint32_t kz0, kz1, vz0, vz1;
};

KVR_DEV const uint8_t* token_blob(const DecodeParams& p, int b, int t, int& slot) {
  const int page = p.bt[(int64_t)b * p.bt_stride + (t >> p.log2P)];
  slot = t & ((1 << p.log2P) - 1);
  return p.pool.base + (int64_t)page * p.pool.page_bytes;
}

KVR_DEV void load_tile(const DecodeParams& p, int b, int h, int t0, int len, int lane, TileRegs& R) {
  const int r = lane >> 2, i = lane & 3;
  const int H = p.pool.H;
  const int ta = t0 + r, tb = t0 + r + 8;
  R.k0 = make_uint4(0, 0, 0, 0);
  R.k1 = make_uint4(0, 0, 0, 0);
  R.ks0 = R.ks1 = R.vs0 = R.vs1 = 0.f;
  R.kz0 = R.kz1 = R.vz0 = R.vz1 = 0u;
  if (ta < len) {
    int sl;
    const uint8_t* blob = token_blob(p, b, ta, sl);
    const int idx = sl * H + h;
    R.k0 = __ldg(reinterpret_cast<const uint4*>(blob + p.pool.off_kp + (int64_t)idx * 64 + 16 * i));
    R.ks0 = __ldg(reinterpret_cast<const float*>(blob + p.pool.off_ks) + idx);
    R.kz0 = __ldg(blob + p.pool.off_kz + idx);
    R.vs0 = __ldg(reinterpret_cast<const float*>(blob + p.pool.off_vs) + idx);
    R.vz0 = __ldg(blob + p.pool.off_vz + idx);
  }
  if (tb < len) {
    int sl;
    const uint8_t* blob = token_blob(p, b, tb, sl);
    const int idx = sl * H + h;
    R.k1 = __ldg(reinterpret_cast<const uint4*>(blob + p.pool.off_kp + (int64_t)idx * 64 + 16 * i));
    R.ks1 = __ldg(reinterpret_cast<const float*>(blob + p.pool.off_ks) + idx);
    R.kz1 = __ldg(blob + p.pool.off_kz + idx);
    R.vs1 = __ldg(reinterpret_cast<const float*>(blob + p.pool.off_vs) + idx);
    R.vz1 = __ldg(blob + p.pool.off_vz + idx);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int t = t0 + 2 * i + (u & 1) + 8 * (u >> 1);
    R.v[u] = make_uint2(0, 0);
    if (t < len) {
      int sl;
      const uint8_t* blob = token_blob(p, b, t, sl);
      R.v[u] = __ldg(reinterpret_cast<const uint2*>(blob + p.pool.off_vp + (int64_t)(sl * H + h) * 64 + 8 * r));
    }
  }
}

// dims held by A-operand register (k-step s, lane group i, slot R0/R2, half e)
KVR_DEV int qk_dim(int s, int i, int slot2, int e) { return 32 * i + 8 * (s >> 1) + 2 * (s & 1) + slot2 + 4 * e; }

template <int NT>  // number of 8-column MMA tiles: G <= 4 -> 1, G == 8 -> 2
__global__ void __launch_bounds__(DEC_WARPS * 32, 3) decode_mma_kernel(const __grid_constant__ DecodeParams p,
                                                                        const __grid_constant__ Signs signs) {
  __shared__ float sq[8 * 128];                  // rotated query of this kv head's group
  __shared__ float sred[DEC_WARPS][8][128 + 2];  // per-warp (o_unnorm, M, l) for the CTA merge
  __shared__ uint32_t s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, i = lane & 3;
  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int G = p.G, H = p.pool.H;
  const int len = p.lens[b];

  // ---- query: load, rotate into the stored-key frame, normalise, split hi/lo
  for (int x = threadIdx.x; x < 8 * 128; x += blockDim.x) {
    const int j = x >> 7, dd = x & 127;
    float v = 0.f;
    if (j < G) {
      v = load_q(p.q, p.q_dtype, ((int64_t)b * p.nq + (int64_t)h * G + j) * 128 + dd);
      if (p.rotate && p.has_signs && sign_bit(signs, dd)) v = -v;
    }
    sq[x] = v;
  }
  __syncthreads();
  if (p.rotate) cta_fwht128(sq, G, p.order);
  float amax = 0.f;
  for (int x = lane; x < G * 128; x += 32) amax = fmaxf(amax, fabsf(sq[x]));
  amax = warp_max(amax);
  // q' = q * 2^-e with max|q'| in [2^13, 2^14): fp16 hi/lo keep ~22 bits
  int e2 = 0;
  if (amax > 0.f) e2 = ilogbf(amax) - 13;
  const float qscale = ldexpf(1.0f, -e2);
  __syncthreads();  // every warp has read sq for amax
  // hi/lo split in place: sq[x] <- hi, sred used as scratch for lo
  float* sqlo = &sred[0][0][0];
  for (int x = threadIdx.x; x < G * 128; x += blockDim.x) {
    const float v = sq[x] * qscale;
    const float hi = __half2float(__float2half_rn(v));
    sq[x] = hi;
    sqlo[x] = __half2float(__float2half_rn(v - hi));
  }
  __syncthreads();

  uint32_t bq[NT][8][2];
  float sumq[2] = {0.f, 0.f};  // per head owned by this lane: j = 4*nt + i
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int col = r;  // B-fragment column = lane / 4
    const int j = 4 * nt + (col >> 1), part = col & 1;
    const float* src = part ? sqlo : sq;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      float v4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int slot2 = k >> 1, e = k & 1;
        const float v = (j < G) ? src[j * 128 + qk_dim(s, i, slot2, e)] : 0.f;
        v4[k] = slot2 ? v * (1.0f / 16.0f) : v;
      }
      bq[nt][s][0] = pack_h2(v4[0], v4[1]);
      bq[nt][s][1] = pack_h2(v4[2], v4[3]);
    }
  }
  // sum over d of (hi + lo) per head, in MMA units (x 2^-24)
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    for (int jj = 4 * nt; jj < min(G, 4 * nt + 4); ++jj) {
      float a = 0.f;
      for (int dd = lane; dd < 128; dd += 32) a += sq[jj * 128 + dd] + sqlo[jj * 128 + dd];
      a = warp_sum(a);
      if (jj == 4 * nt + i) sumq[nt] = a * 5.9604644775390625e-08f;  // 2^-24
    }
  }
  __syncthreads();  // sred scratch is reused by the merge below
  // logit (log2 units) = (D - z * sumq) * s_k * kscale
  const float kscale = ldexpf(1.0f, e2 + 24) * LOG2E * (float)(1.0 / sqrt(128.0));

  // ---- split range in 16-token tiles
  const int n_tiles = (len + 15) >> 4;
  const int per = (n_tiles + p.splits - 1) / p.splits;
  const int tile_lo = split * per;
  const int tile_hi = min(n_tiles, tile_lo + per);

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

  TileRegs cur, nxt;
  int tile = tile_lo + warp;
  if (tile < tile_hi) load_tile(p, b, h, tile * 16, len, lane, cur);
  for (; tile < tile_hi; tile += DEC_WARPS) {
    const int tnext = tile + DEC_WARPS;
    if (tnext < tile_hi) load_tile(p, b, h, tnext * 16, len, lane, nxt);

    // ---- S = C_k q : 8 k-steps of m16n8k16 per 8-column tile
    float sc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
    const uint32_t kw0[4] = {cur.k0.x, cur.k0.y, cur.k0.z, cur.k0.w};
    const uint32_t kw1[4] = {cur.k1.x, cur.k1.y, cur.k1.z, cur.k1.w};
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const uint32_t wa = kw0[s >> 1], wb = kw1[s >> 1];
      const uint32_t xa = (s & 1) ? (wa >> 8) : wa, xb = (s & 1) ? (wb >> 8) : wb;
      const uint32_t a0 = xa & 0x000F000Fu, a2 = xa & 0x00F000F0u;
      const uint32_t a1 = xb & 0x000F000Fu, a3 = xb & 0x00F000F0u;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) mma16816(sc[nt], a0, a1, a2, a3, bq[nt][s][0], bq[nt][s][1]);
    }

    // ---- sidecars (sentinel rows: scale slot holds the offset, codes are 0)
    float sk0 = cur.ks0, sk1 = cur.ks1, zk0 = (float)cur.kz0, zk1 = (float)cur.kz1;
    if (cur.kz0 == 0xFFu) { zk0 = -sk0; sk0 = 1.f; }
    if (cur.kz1 == 0xFFu) { zk1 = -sk1; sk1 = 1.f; }
    float sv0 = cur.vs0, sv1 = cur.vs1, zv0 = (float)cur.vz0, zv1 = (float)cur.vz1;
    if (cur.vz0 == 0xFFu) { zv0 = -sv0; sv0 = 1.f; }
    if (cur.vz1 == 0xFFu) { zv1 = -sv1; sv1 = 1.f; }
    const int t0 = tile * 16 + r, t1 = t0 + 8;
    const bool ok0 = t0 < len, ok1 = t1 < len;
    const float lgv0 = ok0 ? __log2f(sv0) : 0.f, lgv1 = ok1 ? __log2f(sv1) : 0.f;

    uint32_t wb_lo[NT], wb_hi[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const float l0 = ok0 ? (sc[nt][0] + sc[nt][1] - zk0 * sumq[nt]) * (sk0 * kscale) : -INFINITY;
      const float l1 = ok1 ? (sc[nt][2] + sc[nt][3] - zk1 * sumq[nt]) * (sk1 * kscale) : -INFINITY;
      const float b0 = l0 + lgv0, b1 = l1 + lgv1;  // log2(p * s_v) up to the running max
      float tm = fmaxf(b0, b1);
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 4));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 8));
      tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, 16));
      const float mnew = fmaxf(M[nt], tm);
      const float alpha = (mnew == -INFINITY) ? 1.f : exp2f(M[nt] - mnew);
      M[nt] = mnew;
      const float ms = (mnew == -INFINITY) ? 0.f : mnew;
      const float w0 = exp2f(b0 - ms), w1 = exp2f(b1 - ms);   // = p_t * s_v <= 1
      const float p0 = exp2f(l0 - ms), p1 = exp2f(l1 - ms);   // = p_t
      lsum[nt] = lsum[nt] * alpha + p0 + p1;
      Zs[nt] = Zs[nt] * alpha + w0 * zv0 + w1 * zv1;
      if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
        for (int m = 0; m < 8; ++m)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[nt][m][c] *= alpha;
      }
      // fp16 hi/lo of w * 2^15 (w <= 1): keeps the lo half out of fp16 subnormals
      // for weights down to ~2^-28 of the running max
      const float w0s = w0 * 32768.0f, w1s = w1 * 32768.0f;
      const float w0h = __half2float(__float2half_rn(w0s)), w1h = __half2float(__float2half_rn(w1s));
      wb_lo[nt] = movtrans(pack_h2(w0h, w0s - w0h));  // tokens 0..7  -> b0,b1
      wb_hi[nt] = movtrans(pack_h2(w1h, w1s - w1h));  // tokens 8..15 -> b2,b3
    }

    // ---- O^T += C_v^T W : 8 m-tiles (16 dims each) of m16n8k16
    uint32_t xr[2][2][8];  // [token pair (2i,2i+1)|(2i+8,2i+9)][word q][dim e]
#pragma unroll
    for (int tp = 0; tp < 2; ++tp)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t wa = q ? cur.v[2 * tp].y : cur.v[2 * tp].x;
        const uint32_t wb = q ? cur.v[2 * tp + 1].y : cur.v[2 * tp + 1].x;
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
        mma16816(acc[nt][m], xr[0][0][m], xr[0][1][m], xr[1][0][m], xr[1][1][m], wb_lo[nt], wb_hi[nt]);
    cur = nxt;
  }

  // ---- per-warp finalisation: reduce l and Z over the 8 lanes of a head
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      lsum[nt] += __shfl_xor_sync(0xffffffffu, lsum[nt], o);
      Zs[nt] += __shfl_xor_sync(0xffffffffu, Zs[nt], o);
    }
    const int j = 4 * nt + i;
    if (j < G) {
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const float f = (m & 1) ? 512.0f / 16.0f : 512.0f;  // undo 2^-24 (codes), 2^15 (w) and the x16 nibble
        sred[warp][j][16 * r + m] = (acc[nt][m][0] + acc[nt][m][1]) * f - Zs[nt];
        sred[warp][j][16 * r + 8 + m] = (acc[nt][m][2] + acc[nt][m][3]) * f - Zs[nt];
      }
      if (r == 0) {
        sred[warp][j][128] = M[nt];
        sred[warp][j][129] = lsum[nt];
      }
    }
  }
  __syncthreads();

  // ---- CTA merge over warps -> (o, lse) for this split
  float* obuf = sq;  // reuse: [G][128] merged normalised output
  for (int x = threadIdx.x; x < G * 128; x += blockDim.x) {
    const int j = x >> 7, dd = x & 127;
    float mmax = -INFINITY;
#pragma unroll
    for (int w = 0; w < DEC_WARPS; ++w) mmax = fmaxf(mmax, sred[w][j][128]);
    float lt = 0.f, ot = 0.f;
    if (mmax != -INFINITY) {
#pragma unroll
      for (int w = 0; w < DEC_WARPS; ++w) {
        const float mw = sred[w][j][128];
        if (mw == -INFINITY) continue;
        const float f = exp2f(mw - mmax);
        lt += f * sred[w][j][129];
        ot += f * sred[w][j][dd];
      }
    }
    const float o = (lt > 0.f) ? ot / lt : 0.f;
    const float lse = (lt > 0.f) ? mmax + __log2f(lt) : -INFINITY;
    if (p.splits == 1) {
      obuf[x] = o;
    } else {
      const int64_t base = (((int64_t)b * H + h) * p.splits + split) * 8 + j;
      p.ws_o[base * 128 + dd] = o;
      if (dd == 0) p.ws_lse[base] = lse;
    }
  }
  if (p.splits > 1) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t prev = atomicAdd(&p.ws_cnt[(int64_t)b * H + h], 1u);
      s_last = (prev == (uint32_t)p.splits - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // last CTA of (b, h): LSE-merge all splits
    for (int x = threadIdx.x; x < G * 128; x += blockDim.x) {
      const int j = x >> 7, dd = x & 127;
      const int64_t base0 = (((int64_t)b * H + h) * p.splits) * 8 + j;
      float lmax = -INFINITY;
      for (int s = 0; s < p.splits; ++s) lmax = fmaxf(lmax, __ldcg(&p.ws_lse[base0 + (int64_t)s * 8]));
      float wt = 0.f, ot = 0.f;
      for (int s = 0; s < p.splits; ++s) {
        const float ls = __ldcg(&p.ws_lse[base0 + (int64_t)s * 8]);
        if (ls == -INFINITY) continue;
        const float f = exp2f(ls - lmax);
        wt += f;
        ot += f * __ldcg(&p.ws_o[(base0 + (int64_t)s * 8) * 128 + dd]);
      }
      obuf[x] = wt > 0.f ? ot / wt : 0.f;
    }
    if (threadIdx.x == 0) p.ws_cnt[(int64_t)b * H + h] = 0u;  // re-arm for the next launch
  }
  __syncthreads();
  // ---- inverse rotation of the value branch: o @ H_blk @ diag(signs)
  if (p.rotate && p.rot_v) {
    cta_fwht128(obuf, G, p.order);
    if (p.has_signs)
      for (int x = threadIdx.x; x < G * 128; x += blockDim.x)
        if (sign_bit(signs, x & 127)) obuf[x] = -obuf[x];
    __syncthreads();
  }
  for (int x = threadIdx.x; x < G * 128; x += blockDim.x) {
    const int j = x >> 7, dd = x & 127;
    p.out[((int64_t)b * p.nq + (int64_t)h * G + j) * 128 + dd] = obuf[x];
  }
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
  const int G = p.G, H = p.pool.H, h = qh / G;
  const int len = p.lens[b];
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
    int sl;
    const uint8_t* blob = token_blob(p, b, t, sl);
    const int idx = sl * H + h;
    const float ks = reinterpret_cast<const float*>(blob + p.pool.off_ks)[idx];
    const uint8_t kz = blob[p.pool.off_kz + idx];
    const float vs = reinterpret_cast<const float*>(blob + p.pool.off_vs)[idx];
    const uint8_t vz = blob[p.pool.off_vz + idx];
    float dot = 0.f;
    for (int k = 0, x = lane; x < d; x += 32, ++k) {
      const uint8_t byte = blob[p.pool.off_kp + (int64_t)idx * (d / 2) + (x >> 1)];
      const float c = (float)((x & 1) ? (byte >> 4) : (byte & 15));
      const float kh = (kz == 0xFF) ? ks : ks * (c - (float)kz);
      dot += kh * sq[x];
    }
    dot = warp_sum(dot) * scale;
    const float mn = fmaxf(m, dot);
    const float a = exp2f((m - mn) * LOG2E), pw = exp2f((dot - mn) * LOG2E);
    l = l * a + pw;
    for (int k = 0, x = lane; x < d; x += 32, ++k) {
      const uint8_t byte = blob[p.pool.off_vp + (int64_t)idx * (d / 2) + (x >> 1)];
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
  const int target = sms * 3;  // resident CTAs
  const int units = batch * H;
  int s = (target + units - 1) / units;
  const int max_s = (tiles + 2 * DEC_WARPS - 1) / (2 * DEC_WARPS);  // >= 2 tiles per warp
  if (s > max_s) s = max_s;
  if (s < 1) s = 1;
  return s;
}

int kvr_launch_decode(const void* q, int q_dtype, const Pool& pool, const int32_t* bt, int bt_stride,
                      const int32_t* lens, int batch, int nq, int max_len, int order, int rotate, int rot_v,
                      const Signs& s, int has, float* out, void* ws, size_t ws_bytes, int splits, cudaStream_t st) {
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
  int l2 = 0;
  while ((1 << l2) < pool.P) ++l2;
  const bool pow2 = (1 << l2) == pool.P;
  p.log2P = l2;
  Signs sg = s;
  if (!has) for (auto& x : sg.w) x = 0u;
  const bool mma_ok = pool.d == 128 && pow2 && (p.G == 1 || p.G == 2 || p.G == 4 || p.G == 8);
  if (!pow2) return KVR_ERR_UNSUPPORTED;
  if (mma_ok) {
    if (splits <= 0) splits = kvr_pick_splits(batch, pool.H, max_len, pool.P);
    if (splits > 1 && kvr_decode_ws_bytes(batch, pool.H, nq, 128, splits) > ws_bytes) return KVR_ERR_ARG;
    p.splits = splits;
    const size_t units = (size_t)batch * pool.H * splits * 8;
    p.ws_o = reinterpret_cast<float*>(ws);
    p.ws_lse = p.ws_o + units * 128;
    p.ws_cnt = reinterpret_cast<uint32_t*>(p.ws_lse + units);
    dim3 grid(splits, pool.H, batch);
    if (p.G == 8)
      decode_mma_kernel<2><<<grid, DEC_WARPS * 32, 0, st>>>(p, sg);
    else
      decode_mma_kernel<1><<<grid, DEC_WARPS * 32, 0, st>>>(p, sg);
    return 0;
  }
  if (pool.d > 256 || (pool.d & 31)) return KVR_ERR_UNSUPPORTED;
  p.splits = 1;
  const int warps = 4;
  const size_t smem = (size_t)(pool.d + warps * pool.d + warps * 2) * sizeof(float);
  decode_generic_kernel<<<dim3(nq, batch), warps * 32, smem, st>>>(p, sg, pool.d);
  return 0;
}
