// Precision probe: fp16 MMA with codes encoded as subnormals (c*2^-24) vs as
// integers (c as fp16 normal), fp32 accumulate, vs an f64 reference.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_fp16.h>
__device__ uint32_t packh(float a, float b){ __half2 h=__floats2half2_rn(a,b); return *reinterpret_cast<uint32_t*>(&h);}
__global__ void probe(const uint8_t* codes, const float* qv, float* out_sub, float* out_int) {
  // one warp: 16 tokens x 128 dims codes (row-major, c in [0,15]), q 128 (hi/lo in cols 0/1)
  int lane = threadIdx.x, r = lane >> 2, i = lane & 3;
  float ds[4] = {0,0,0,0}, di[4] = {0,0,0,0};
  for (int s = 0; s < 8; ++s) {
    int k0 = 16*s + 2*i, k1 = k0 + 8;
    auto A = [&](int row, int k, bool sub) { float c = codes[row*128+k]; return sub ? c * 5.9604644775390625e-08f : c; };
    uint32_t a_s[4], a_i[4];
    a_s[0] = packh(A(r,k0,1), A(r,k0+1,1)); a_s[1] = packh(A(r+8,k0,1), A(r+8,k0+1,1));
    a_s[2] = packh(A(r,k1,1), A(r,k1+1,1)); a_s[3] = packh(A(r+8,k1,1), A(r+8,k1+1,1));
    a_i[0] = packh(A(r,k0,0), A(r,k0+1,0)); a_i[1] = packh(A(r+8,k0,0), A(r+8,k0+1,0));
    a_i[2] = packh(A(r,k1,0), A(r,k1+1,0)); a_i[3] = packh(A(r+8,k1,0), A(r+8,k1+1,0));
    // B col n = r: n=0 hi, n=1 lo, others 0
    auto Bv = [&](int k) { float x = qv[k]; float hi = __half2float(__float2half_rn(x)); float lo = x - hi;
                           return r == 0 ? hi : (r == 1 ? lo : 0.f); };
    uint32_t b0 = packh(Bv(k0), Bv(k0+1)), b1 = packh(Bv(k1), Bv(k1+1));
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(ds[0]), "+f"(ds[1]), "+f"(ds[2]), "+f"(ds[3]) : "r"(a_s[0]), "r"(a_s[1]), "r"(a_s[2]), "r"(a_s[3]), "r"(b0), "r"(b1));
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(di[0]), "+f"(di[1]), "+f"(di[2]), "+f"(di[3]) : "r"(a_i[0]), "r"(a_i[1]), "r"(a_i[2]), "r"(a_i[3]), "r"(b0), "r"(b1));
  }
  if (i == 0) {  // cols 0 (hi) and 1 (lo) of rows r, r+8
    out_sub[r] = (ds[0] + ds[1]) * 16777216.0f; out_sub[r+8] = (ds[2] + ds[3]) * 16777216.0f;
    out_int[r] = di[0] + di[1]; out_int[r+8] = di[2] + di[3];
  }
}
int main() {
  uint8_t hc[16*128]; float hq[128];
  unsigned s = 12345; auto rnd = [&]{ s = s*1664525u + 1013904223u; return s; };
  double worst_s = 0, worst_i = 0;
  uint8_t* dc; float *dq, *ds, *di; cudaMalloc(&dc, sizeof hc); cudaMalloc(&dq, sizeof hq); cudaMalloc(&ds, 64); cudaMalloc(&di, 64);
  for (int trial = 0; trial < 200; ++trial) {
    for (int j = 0; j < 16*128; ++j) hc[j] = rnd() % 16;
    for (int j = 0; j < 128; ++j) hq[j] = ((int)(rnd() % 20001) - 10000) * (8192.0f / 10000.0f) + (rnd()%1000)*1e-3f;
    cudaMemcpy(dc, hc, sizeof hc, cudaMemcpyHostToDevice); cudaMemcpy(dq, hq, sizeof hq, cudaMemcpyHostToDevice);
    probe<<<1,32>>>(dc, dq, ds, di);
    float os[16], oi[16]; cudaMemcpy(os, ds, 64, cudaMemcpyDeviceToHost); cudaMemcpy(oi, di, 64, cudaMemcpyDeviceToHost);
    for (int t = 0; t < 16; ++t) {
      double ref = 0, mag = 0; for (int k = 0; k < 128; ++k) { ref += (double)hc[t*128+k] * hq[k]; mag += fabs((double)hc[t*128+k]*hq[k]); }
      worst_s = fmax(worst_s, fabs(os[t] - ref) / mag); worst_i = fmax(worst_i, fabs(oi[t] - ref) / mag);
    }
  }
  printf("max |err|/sum|terms|: subnormal-coded %.3e   integer-coded %.3e\n", worst_s, worst_i);
  return 0;
}
