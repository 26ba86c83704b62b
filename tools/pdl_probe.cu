// Floor of a kernel-to-kernel boundary on this GPU: per-launch time of a CUDA
// graph of back-to-back small grids, with and without programmatic dependent
// launch, and with one dependent global load / an atomic arrival per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_probe tools/pdl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_go() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// mode 0: store only; 1: one dependent load then store; 2: + last-arriver atomic
__global__ void __launch_bounds__(512) k_step(float* buf, unsigned* cnt, int mode) {
  pdl_wait();
  pdl_go();
  float v = 1.f;
  if (mode >= 1) v = __ldcg(buf + blockIdx.x * 128 + (threadIdx.x & 127));
  __syncthreads();
  if (mode >= 2) {
    __shared__ int last;
    if (threadIdx.x == 0) {
      unsigned prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(cnt) : "memory");
      last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      v += __ldcg(buf + ((blockIdx.x + 1) % gridDim.x) * 128 + (threadIdx.x & 127));
      if (threadIdx.x == 0) *cnt = 0;
    }
  }
  if (threadIdx.x < 128) buf[blockIdx.x * 128 + threadIdx.x] = v * 0.5f + 0.25f;
}

// straight-line code (UNROLL = 2048 FMAs = 32 KB of SASS) vs the same work as a loop
template <bool STRAIGHT>
__global__ void __launch_bounds__(512) k_code(float* buf, float a, float c) {
  pdl_wait();
  pdl_go();
  float x = buf[threadIdx.x];
  if (STRAIGHT) {
#pragma unroll
    for (int i = 0; i < 2048; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(a), "f"(c));
  } else {
#pragma unroll 1
    for (int i = 0; i < 2048; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(a), "f"(c));
  }
  if (x == 1234.5f) buf[threadIdx.x] = x;
}

template <typename K, typename... A>
static float run_k(K kern, int grid, A... args) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  const int N = 64;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < N; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(512);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
  cudaEventRecord(e0, s);
  for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / (20 * N);
}

static float run(int grid, int threads, int mode, bool pdl, float* buf, unsigned* cnt, int smem = 0) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  const int N = 64;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < N; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.stream = s;
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_step, buf, cnt, mode);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
  cudaEventRecord(e0, s);
  const int R = 20;
  for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return ms * 1000.f / (R * N);
}

int main() {
  float* buf;
  unsigned* cnt;
  cudaMalloc(&buf, 1 << 20);
  cudaMemset(buf, 0, 1 << 20);
  cudaMalloc(&cnt, 4);
  cudaMemset(cnt, 0, 4);
  const char* names[3] = {"store", "load+store", "load+atomic last-arriver+load"};
  for (int mode = 0; mode < 3; ++mode)
    for (int grid : {8, 144})
      for (int pdl = 0; pdl < 2; ++pdl)
        printf("%-32s grid %3d x 512  pdl %d : %6.2f us/launch\n", names[mode], grid, pdl,
               run(grid, 512, mode, pdl, buf, cnt));
  cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 0; mode < 3; ++mode)
    printf("%-32s grid 144 x 512  pdl 1, 200 KB smem : %6.2f us/launch\n", names[mode],
           run(144, 512, mode, true, buf, cnt, 200 * 1024));
  for (int grid : {8, 144}) {
    printf("2048 dependent FMAs, loop          grid %3d: %6.2f us/launch\n", grid, run_k(k_code<false>, grid, buf, 1.0001f, 0.5f));
    printf("2048 dependent FMAs, straight-line grid %3d: %6.2f us/launch\n", grid, run_k(k_code<true>, grid, buf, 1.0001f, 0.5f));
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
