// Reference-exact (IEEE f64, reference operation order) warp-level row
// primitives shared by the operator kernels and the fused decode-step append.
//   warp_fwht_f64      _ref.fwht_rows      (_ref.py:22-40, _core.pyx:22-47)
//   warp_quantize_f64  _ref.quantize_rows  (_ref.py:57-80, _core.pyx:76-130)
#pragma once
#include "kvr_common.cuh"

namespace kvr {

// In-place f64 block butterfly over a row held in shared memory by one warp.
// Pair (i, i+half) -> (a+b, a-b) for half = 1, 2, ..., order/2, then * inv.
KVR_DEV void warp_fwht_f64(double* s, int d, int order, int lane) {
  if (order == 1) return;
  const int npairs = d >> 1;
  for (int half = 1; half < order; half <<= 1) {
    for (int p = lane; p < npairs; p += 32) {
      const int blk = p / (order >> 1), q = p % (order >> 1);
      const int i = blk * order + (q / half) * 2 * half + (q % half);
      const double a = s[i], b = s[i + half];
      s[i] = a + b;
      s[i + half] = a - b;
    }
    __syncwarp();
  }
  const double inv = 1.0 / sqrt((double)order);
  for (int i = lane; i < d; i += 32) s[i] = s[i] * inv;
  __syncwarp();
}

// Quantize one f64 row held in smem (one warp) -> packed bytes / scale / zp.
// Writes packed[0 .. d/2), *scale, *zp.  Bit-exact with _ref.quantize_rows.
KVR_DEV void warp_quantize_f64(const double* s, int d, int lane, uint8_t* packed, float* scale, uint8_t* zp) {
  double mn = s[0], mx = s[0];
  for (int i = lane; i < d; i += 32) {
    const double v = s[i];
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double a = __shfl_xor_sync(0xffffffffu, mn, o);
    const double b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  const float s32 = (float)((mx - mn) / 15.0);
  if (s32 == 0.0f) {
    for (int m = lane; m < (d >> 1); m += 32) packed[m] = 0;
    if (lane == 0) {
      *scale = (float)mn;
      *zp = 0xFF;
    }
    return;
  }
  const double s64 = (double)s32;
  double z = round_half_away(-mn / s64);
  z = z < 0.0 ? 0.0 : (z > 15.0 ? 15.0 : z);
  for (int m = lane; m < (d >> 1); m += 32) {
    double lo = round_half_away(s[2 * m] / s64) + z;
    double hi = round_half_away(s[2 * m + 1] / s64) + z;
    lo = lo < 0.0 ? 0.0 : (lo > 15.0 ? 15.0 : lo);
    hi = hi < 0.0 ? 0.0 : (hi > 15.0 ? 15.0 : hi);
    packed[m] = (uint8_t)((uint32_t)lo | ((uint32_t)hi << 4));
  }
  if (lane == 0) {
    *scale = s32;
    *zp = (uint8_t)z;
  }
}

}  // namespace kvr
