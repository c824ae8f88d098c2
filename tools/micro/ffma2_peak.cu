// FP32 FMA-pipe throughput on this GPU: scalar FFMA, FFMA2 with pair operands,
// FFMA2 with a broadcast scalar operand (the LUD far update's form), each with
// 16 independent accumulators per thread over many warps.  Test infrastructure.
#include <cstdio>
__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
template <int MODE>
__global__ void __launch_bounds__(256) peak(float *out, int iters, float s) {
  float a = threadIdx.x * 1e-3f, b = 1.0001f;
  if (MODE == 0) {
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = fmaf(a, b, acc[j]);
      a += s;
    }
    float r = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) r += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  } else {
    unsigned long long acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = pk(j, j + 1);
    unsigned long long bb = pk(b, b + 1e-4f);
    for (int it = 0; it < iters; ++it) {
      if (MODE == 1) {
        unsigned long long aa = pk(a, a + 1e-3f);
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[j]) : "l"(aa), "l"(bb));
      } else {
        unsigned long long aa = pk(a, a);
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[j]) : "l"(aa), "l"(bb));
      }
      a += s;
    }
    float r = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float x, y;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(acc[j]));
      r += x + y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  }
}
int main() {
  float *o;
  cudaMalloc(&o, 1 << 26);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int occ : {1, 2, 4, 8}) {
    const int grid = sms * occ;
    for (int mode = 0; mode < 3; ++mode) {
      auto run = [&] {
        if (mode == 0) peak<0><<<grid, 256>>>(o, iters, 1e-7f);
        else if (mode == 1) peak<1><<<grid, 256>>>(o, iters, 1e-7f);
        else peak<2><<<grid, 256>>>(o, iters, 1e-7f);
      };
      run();
      cudaEventRecord(e0);
      run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flop = 2.0 * 32 * double(iters) * grid * 256;
      printf("warps/SM %2d mode %s  %.1f TFLOP/s\n", occ * 8, mode == 0 ? "FFMA     " : mode == 1 ? "FFMA2    " : "FFMA2 bc ",
             flop / ms / 1e9);
    }
  }
}
