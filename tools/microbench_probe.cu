// Microbenchmarks for design decisions (scratch; not product code).
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

__global__ void hmma_subnormal(float* out) {
  // A = subnormal fp16 values c*2^-24, B = 1.0 ; check D = sum
  int lane = threadIdx.x;
  uint32_t a[4], b[2];
  // a element values: nibble value (lane%4)+1 as subnormal
  uint32_t v = (uint32_t)((lane % 4) + 1);
  for (int i = 0; i < 4; i++) a[i] = v | (v << 16);
  uint32_t one = 0x3C00u; b[0] = one | (one << 16); b[1] = b[0];
  float d[4] = {0,0,0,0};
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
    : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  for (int i = 0; i < 4; i++) out[lane * 4 + i] = d[i] * 16777216.0f;
}

__global__ void fadd2_tput(float* x, int iters) {
  float a0 = x[threadIdx.x], a1 = a0 + 1, b0 = a0 * 2, b1 = a0 * 3;
  unsigned long long A[8], B;
  asm("mov.b64 %0, {%1,%2};" : "=l"(B) : "f"(b0), "f"(b1));
  for (int j = 0; j < 8; j++) asm("mov.b64 %0, {%1,%2};" : "=l"(A[j]) : "f"(a0 + j), "f"(a1));
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(A[j]) : "l"(B));
  }
  unsigned long long s = 0; for (int j = 0; j < 8; j++) s ^= A[j];
  if (s == 12345) x[0] = 1;
}
__global__ void fadd_tput(float* x, int iters) {
  float a[8]; float b = x[threadIdx.x] * 2;
  for (int j = 0; j < 8; j++) a[j] = x[threadIdx.x] + j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[j]) : "f"(b));
  }
  float s = 0; for (int j = 0; j < 8; j++) s += a[j];
  if (s == 12345) x[0] = 1;
}
__global__ void dadd_tput(double* x, int iters) {
  double a[8]; double b = x[threadIdx.x] * 2;
  for (int j = 0; j < 8; j++) a[j] = x[threadIdx.x] + j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a[j]) : "d"(b));
  }
  double s = 0; for (int j = 0; j < 8; j++) s += a[j];
  if (s == 12345) x[0] = 1;
}
__global__ void lop_tput(uint32_t* x, int iters) {
  uint32_t a[8]; uint32_t b = x[threadIdx.x] * 2;
  for (int j = 0; j < 8; j++) a[j] = x[threadIdx.x] + j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) asm volatile("lop3.b32 %0, %0, %1, 0x0F0F0F0F, 0x6a;" : "+r"(a[j]) : "r"(b));
  }
  uint32_t s = 0; for (int j = 0; j < 8; j++) s += a[j];
  if (s == 12345) x[0] = 1;
}
__global__ void hmma_tput(float* x, int iters) {
  uint32_t a0 = __float_as_uint(x[threadIdx.x]);
  float d[8][4] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%4,%4}, {%0,%1,%2,%3};"
        : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3]) : "r"(a0));
  }
  float s = 0; for (int j = 0; j < 8; j++) s += d[j][0] + d[j][3];
  if (s == 12345) x[0] = 1;
}
__global__ void imma_tput(float* x, int iters) {
  uint32_t a0 = __float_as_uint(x[threadIdx.x]);
  int d[8][4] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%4,%4}, {%0,%1,%2,%3};"
        : "+r"(d[j][0]), "+r"(d[j][1]), "+r"(d[j][2]), "+r"(d[j][3]) : "r"(a0));
  }
  int s = 0; for (int j = 0; j < 8; j++) s += d[j][0] + d[j][3];
  if (s == 12345) x[0] = 1;
}
__global__ void shf_tput(uint32_t* x, int iters) {
  uint32_t a[8];
  for (int j = 0; j < 8; j++) a[j] = x[threadIdx.x] + j;
  uint32_t sh = x[1] & 7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = (a[j] >> sh) ^ (a[j] << 3);
  }
  uint32_t s = 0; for (int j = 0; j < 8; j++) s += a[j];
  if (s == 12345) x[0] = 1;
}
__global__ void prmt_tput(uint32_t* x, int iters) {
  uint32_t a[8];
  for (int j = 0; j < 8; j++) a[j] = x[threadIdx.x] + j;
  uint32_t b = x[2];
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(a[j]) : "r"(b));
  }
  uint32_t s = 0; for (int j = 0; j < 8; j++) s += a[j];
  if (s == 12345) x[0] = 1;
}
__global__ void i2f_tput(float* x, int iters) {
  int a[8]; float f[8];
  for (int j = 0; j < 8; j++) { a[j] = (int)(x[threadIdx.x] * 100.f) + j; f[j] = 0.f; }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) { float t; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(t) : "r"(a[j])); f[j] += t; }
  }
  float s = 0; for (int j = 0; j < 8; j++) s += f[j];
  if (s == 12345) x[0] = 1;
}
__global__ void mufu_tput(float* x, int iters) {
  float a[8];
  for (int j = 0; j < 8; j++) a[j] = x[threadIdx.x] * 0.001f + j * 0.0001f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
  }
  float s = 0; for (int j = 0; j < 8; j++) s += a[j];
  if (s == 12345) x[0] = 1;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  float* dx; CK(cudaMalloc(&dx, 1 << 20)); CK(cudaMemset(dx, 0, 1 << 20));
  float h[128];
  hmma_subnormal<<<1, 32>>>(dx); CK(cudaMemcpy(h, dx, 512, cudaMemcpyDeviceToHost));
  printf("hmma subnormal D lane0: %g %g %g %g (expect 16*(1+2+3+4)/... per row)\n", h[0], h[1], h[2], h[3]);
  printf("lane5: %g %g %g %g\n", h[20], h[21], h[22], h[23]);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SMs %d clock %d kHz L2 %d\n", p.multiProcessorCount, clk, p.l2CacheSize);
  int iters = 4096, blocks = p.multiProcessorCount * 8, threads = 256;
  double lanes = (double)blocks * threads * iters * 8;
  float ms;
  ms = timeit([&]{ fadd2_tput<<<blocks, threads>>>(dx, iters); });
  printf("FADD2: %.1f G instr-lanes/s -> %.2f flop-lanes/clk/SM (at 1.9GHz)\n", lanes / ms / 1e6, 2 * lanes / ms / 1e6 / p.multiProcessorCount / 1.9e3 * 1e3 / 1e3);
  ms = timeit([&]{ fadd_tput<<<blocks, threads>>>(dx, iters); });
  printf("FADD: %.1f G lanes/s -> %.2f lanes/clk/SM\n", lanes / ms / 1e6, lanes / ms / 1e6 / p.multiProcessorCount / 1.9);
  ms = timeit([&]{ dadd_tput<<<blocks, threads>>>((double*)dx, iters); });
  printf("DADD: %.1f G lanes/s -> %.2f lanes/clk/SM\n", lanes / ms / 1e6, lanes / ms / 1e6 / p.multiProcessorCount / 1.9);
  ms = timeit([&]{ lop_tput<<<blocks, threads>>>((uint32_t*)dx, iters); });
  printf("LOP3: %.1f G lanes/s -> %.2f lanes/clk/SM\n", lanes / ms / 1e6, lanes / ms / 1e6 / p.multiProcessorCount / 1.9);
  ms = timeit([&]{ mufu_tput<<<blocks, threads>>>(dx, iters); });
  printf("EX2: %.1f G lanes/s -> %.2f lanes/clk/SM\n", lanes / ms / 1e6, lanes / ms / 1e6 / p.multiProcessorCount / 1.9);
  ms = timeit([&]{ hmma_tput<<<blocks, threads>>>(dx, iters / 4); });
  double mmas = (double)blocks * (threads / 32) * (iters / 4) * 8;
  printf("HMMA m16n8k16: %.3f G warp-mma/s -> %.3f mma/clk/SM ; %.1f TFLOPS\n", mmas / ms / 1e6, mmas / ms / 1e6 / p.multiProcessorCount / 1.9, mmas * 4096 / ms / 1e9);
  ms = timeit([&]{ imma_tput<<<blocks, threads>>>(dx, iters / 4); });
  printf("IMMA m16n8k32 u8.s8: %.3f G warp-mma/s -> %.3f mma/clk/SM ; %.1f TOPS\n", mmas / ms / 1e6, mmas / ms / 1e6 / p.multiProcessorCount / 1.9, mmas * 8192 / ms / 1e9);
  ms = timeit([&]{ shf_tput<<<blocks, threads>>>((uint32_t*)dx, iters); });
  printf("SHF+LOP pair: %.1f G pair-lanes/s -> %.2f pairs/clk/SM\n", lanes / ms / 1e6, lanes / ms / 1e6 / p.multiProcessorCount / 1.9);
  ms = timeit([&]{ prmt_tput<<<blocks, threads>>>((uint32_t*)dx, iters); });
  printf("PRMT: %.1f G lanes/s -> %.2f lanes/clk/SM\n", lanes / ms / 1e6, lanes / ms / 1e6 / p.multiProcessorCount / 1.9);
  ms = timeit([&]{ i2f_tput<<<blocks, threads>>>(dx, iters); });
  printf("I2F+FADD: %.1f G lanes/s -> %.2f lanes/clk/SM\n", lanes / ms / 1e6, lanes / ms / 1e6 / p.multiProcessorCount / 1.9);
  return 0;
}
