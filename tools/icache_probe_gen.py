# generates icache_probe.cu: straight-line code of N FADD-ish instructions, run cold then warm
N = 2048
body = "\n".join(f"    x{i%8} = __fadd_rn(x{i%8}, y{i%4});" for i in range(N))
src = f'''
#include <cstdio>
#include <cuda_runtime.h>
__device__ __noinline__ float straight(float a, float b) {{
  float x0=a,x1=a+1,x2=a+2,x3=a+3,x4=a+4,x5=a+5,x6=a+6,x7=a+7;
  float y0=b,y1=b*2,y2=b*3,y3=b*4;
{body}
  return x0+x1+x2+x3+x4+x5+x6+x7;
}}
__global__ void probe(float* out, long long* t, float a, float b) {{
  if (threadIdx.x >= 32) return;
  long long t0 = clock64();
  float r = straight(a, b);
  __syncwarp();
  long long t1 = clock64();
  float r2 = straight(r, b);
  __syncwarp();
  long long t2 = clock64();
  if (threadIdx.x == 0) {{ t[blockIdx.x*2] = t1 - t0; t[blockIdx.x*2+1] = t2 - t1; }}
  out[blockIdx.x*32+threadIdx.x] = r + r2;
}}
int main() {{
  float* o; long long* t; cudaMalloc(&o, 148*32*4); cudaMalloc(&t, 148*16);
  for (int rep = 0; rep < 3; ++rep) {{
    probe<<<148, 32>>>(o, t, 1.f, 2.f);
    cudaDeviceSynchronize();
    long long h[296]; cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    double c=0,w=0; for (int i=0;i<148;++i){{c+=h[2*i];w+=h[2*i+1];}}
    printf("rep %d: %d instrs (~%d B): cold %.0f cycles (%.1f per 128-B line), warm %.0f cycles\\n", rep, {N}, {N}*16, c/148, c/148/({N}*16/128.0), w/148);
  }}
  return 0;
}}
'''
open("/tmp/icp/icache_probe.cu","w").write(src)
