// Does an outer product whose column operand is warp-uniform (U[k][cols of the
// warp], read from shared memory at a warp-uniform address) get FFMA2 with
// uniform-register operands, and what rate does it reach?  Lane = row (per-
// thread L scalar), warp = column group (uniform U pairs).  Test infrastructure.
#include <cstdio>
__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = pk(a.x, a.y), rb = pk(b.x, b.y), rc = pk(c.x, c.y), rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  float2 d;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
  return d;
}
constexpr int K = 32;
__global__ void __launch_bounds__(256) uu(float *out, int iters) {
  __shared__ __align__(16) float Ls[256][36];        // rows x k (padded; k wraps at 32)
  __shared__ __align__(16) float Us[K][64];        // k x cols
  for (int i = threadIdx.x; i < 256 * 36; i += 256) (&Ls[0][0])[i] = i * 1e-4f;
  for (int i = threadIdx.x; i < K * 64; i += 256) (&Us[0][0])[i] = 1.0f + i * 1e-5f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);   // uniform
  float2 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int k4 = 0; k4 < K / 4; ++k4) {
      float4 l[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) l[i] = *reinterpret_cast<const float4 *>(&Ls[lane + 32 * i][(4 * k4) & 31]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 u0 = *reinterpret_cast<const float4 *>(&Us[4 * k4 + q][8 * warp]);
        const float4 u1 = *reinterpret_cast<const float4 *>(&Us[4 * k4 + q][8 * warp + 4]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float li = q == 0 ? l[i].x : q == 1 ? l[i].y : q == 2 ? l[i].z : l[i].w;
          const float2 ll = make_float2(li, li);
          acc[i][0] = fma2(ll, make_float2(u0.x, u0.y), acc[i][0]);
          acc[i][1] = fma2(ll, make_float2(u0.z, u0.w), acc[i][1]);
          acc[i][2] = fma2(ll, make_float2(u1.x, u1.y), acc[i][2]);
          acc[i][3] = fma2(ll, make_float2(u1.z, u1.w), acc[i][3]);
        }
      }
    }
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) r += acc[i][j].x + acc[i][j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  float *o;
  cudaMalloc(&o, 1 << 26);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 400;
  for (int occ : {1, 2}) {
    const int grid = sms * occ;
    uu<<<grid, 256>>>(o, iters);
    cudaEventRecord(e0);
    uu<<<grid, 256>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 2.0 * 64.0 * K * double(iters) * grid * 256;
    printf("uniform-U outer product, warps/SM %2d: %.1f TFLOP/s\n", occ * 8, flop / ms / 1e9);
  }
}
