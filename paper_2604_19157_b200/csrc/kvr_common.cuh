// Shared device helpers for the sm_100a Hadamard-INT4 KV kernels.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/kvrot_b200.h"

#define KVR_DEV __device__ __forceinline__

namespace kvr {

// Rotation signs: bit i of w[i/32] set <=> signs[i] == -1 (rotation.py:81-101).
struct Signs {
  uint32_t w[KVR_MAX_HEAD_DIM / 32];
};

// Pool geometry passed by value to kernels (mirror of kvr_pool; see the cell
// layout in include/kvrot_b200.h).
struct Pool {
  uint8_t* base;
  int64_t num_pages;
  int32_t P, H, d, page_bytes, T, cell_bytes;
  int32_t prec;  // KVR_PREC_INT4 | KVR_PREC_BF16
};

// Address of the cell holding (page, head, slot) and the slot's index in it.
KVR_DEV uint8_t* cell_of(const Pool& p, int64_t page, int h, int slot, int& i) {
  const int u = slot / p.T;
  i = slot - u * p.T;
  return p.base + page * (int64_t)p.page_bytes + (int64_t)(h * (p.P / p.T) + u) * p.cell_bytes;
}
// field offsets inside a cell of T tokens
KVR_DEV int cell_kscale(const Pool& p, int i) { return 4 * i; }
KVR_DEV int cell_vscale(const Pool& p, int i) { return 4 * p.T + 4 * i; }
KVR_DEV int cell_kcode(const Pool& p, int i) { return 8 * p.T + i * (p.d >> 1); }
KVR_DEV int cell_vcode(const Pool& p, int i) { return 8 * p.T + p.T * (p.d >> 1) + i * (p.d >> 1); }
KVR_DEV int cell_kzp(const Pool& p, int i) { return 8 * p.T + p.T * p.d + i; }
KVR_DEV int cell_vzp(const Pool& p, int i) { return 9 * p.T + p.T * p.d + i; }

// BF16 cells: k_bits u16[T][d] | v_bits u16[T][d]
KVR_DEV int cell_bf16(const Pool& p, int side, int i) { return 2 * p.d * (side * p.T + i); }

KVR_DEV bool sign_bit(const Signs& s, int i) { return (s.w[i >> 5] >> (i & 31)) & 1u; }

// ---- f64 reference arithmetic (_ref.py:16-19) ------------------------------
KVR_DEV double round_half_away(double t) { return copysign(floor(fabs(t) + 0.5), t); }

// a / b correctly rounded (IEEE double, round to nearest) from rb = RN(1 / b):
// q0 = RN(a rb) is within an ulp of a / b, the fma residual a - b q0 is exact and
// RN(q0 + r rb) is RN(a / b) (Markstein) while nothing over/underflows.  b is an
// f32 value or 15 here, so its significand is never all ones.  Results that
// leave the safe range (or NaN from an infinite b) take the IEEE division.
static __device__ __noinline__ double div_ieee_slow(double a, double b) { return a / b; }
KVR_DEV double div_rn_recip(double a, double b, double rb) {
  const double q0 = a * rb;
  const double q = fma(fma(-q0, b, a), rb, q0);
  if (__builtin_expect(fabs(q) < 0x1p1000, 1)) return q;  // a branch: the IEEE division stays out of line
  return div_ieee_slow(a, b);
}

// ---- f32x2 packed arithmetic (FADD2 / FFMA2 on sm_100a) --------------------
KVR_DEV unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
KVR_DEV void upk(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
KVR_DEV unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
KVR_DEV unsigned long long sub2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
KVR_DEV unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// fl_RM(a*b + c) elementwise: the magic-number floor (exact product-sum, one rounding)
KVR_DEV unsigned long long fma2_rm(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
KVR_DEV float max3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
KVR_DEV float min3_nan(float a, float b, float c) {
  float r;
  asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
KVR_DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// ---- mbarrier + TMA (cp.async.bulk.tensor) ---------------------------------
KVR_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

KVR_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
KVR_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
KVR_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
KVR_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
KVR_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
KVR_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t x, int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// 1-D bulk copy global -> shared completing on an mbarrier (16-B aligned, size % 16 == 0)
KVR_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// same with an L2 cache policy (createpolicy): streamed KV cells go in as
// evict-first so they do not push code, queries and tables out of L2
KVR_DEV void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
KVR_DEV uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// One lane of the (converged) warp, chosen by the hardware: elect.sync keeps the
// issuing region warp-uniform for the compiler, so the bulk-copy operands move to
// uniform registers without a per-lane loop.
KVR_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(pred));
  return pred != 0;
}
KVR_DEV void prefetch_tensormap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// ---- warp helpers ----------------------------------------------------------
KVR_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
KVR_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
KVR_DEV double load_as_f64(const T* p, int64_t i);
template <>
KVR_DEV double load_as_f64<double>(const double* p, int64_t i) { return p[i]; }
template <>
KVR_DEV double load_as_f64<float>(const float* p, int64_t i) { return (double)p[i]; }
template <>
KVR_DEV double load_as_f64<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return (double)__bfloat162float(p[i]);
}
template <>
KVR_DEV double load_as_f64<__half>(const __half* p, int64_t i) { return (double)__half2float(p[i]); }

}  // namespace kvr
