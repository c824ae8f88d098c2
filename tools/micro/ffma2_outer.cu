// FFMA2 throughput for the LUD far update's operand pattern: an 8 x 8 outer
// product per thread, acc[i][j] += l[i] (scalar broadcast) * u[j] (register
// pairs), all operands in registers (no shared memory), at 8 and 16 warps per
// SM.  Separates the FMA-pipe / register-file ceiling of the pattern from the
// kernel's memory and scheduling overheads.  Test infrastructure.
#include <cstdio>
__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
template <int NI, int NJ, bool JOUTER>
__global__ void __launch_bounds__(256) outer(float *out, int iters, float s) {
  float l[NI];
  unsigned long long u[NJ], acc[NI][NJ];
#pragma unroll
  for (int i = 0; i < NI; ++i) l[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int j = 0; j < NJ; ++j) u[j] = pk(1.0001f + j + threadIdx.x * 1e-6f, 0.9999f - j - threadIdx.x * 1e-6f);
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j] = pk(i, j);
  for (int it = 0; it < iters; ++it) {
    if (JOUTER) {
      // U pair fixed across consecutive FFMA2 (operand reuse on the pair), L scalar varying
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int i = 0; i < NI; ++i)
          asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i][j]) : "l"(pk(l[i], l[i])), "l"(u[j]));
    } else {
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const unsigned long long ll = pk(l[i], l[i]);
#pragma unroll
        for (int j = 0; j < NJ; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i][j]) : "l"(ll), "l"(u[j]));
      }
    }
#pragma unroll
    for (int i = 0; i < NI; ++i) l[i] += s;       // new operands every round (not hoistable)
#pragma unroll
    for (int j = 0; j < NJ; ++j) u[j] ^= 1ull;
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      float x, y;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(acc[i][j]));
      r += x + y;
    }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  float *o;
  if (cudaMalloc(&o, 1 << 26) != cudaSuccess) {
    fprintf(stderr, "no CUDA device\n");
    return 1;
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  for (int occ : {1, 2}) {
    const int grid = sms * occ;
    for (int jo = 0; jo < 2; ++jo) {
      auto run = [&] {
        if (jo) outer<8, 4, true><<<grid, 256>>>(o, iters, 1e-7f);
        else outer<8, 4, false><<<grid, 256>>>(o, iters, 1e-7f);
      };
      run();
      cudaEventRecord(e0);
      run();
      cudaEventRecord(e1);
      if (cudaEventSynchronize(e1) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        fprintf(stderr, "kernel failed\n");
        return 1;
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flop = 2.0 * 2 * 8 * 4 * double(iters) * grid * 256;
      printf("8x8 outer product (8 x 4 FFMA2, %s), warps/SM %2d: %.1f TFLOP/s\n",
             jo ? "U pair reused, L varying" : "L reused, U varying", occ * 8, flop / ms / 1e9);
    }
  }
}
