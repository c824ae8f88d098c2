// Shared-load wavefronts per warp instruction for the access patterns the LUD
// far-update kernel can use (ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum
// / smsp__sass_inst_executed_op_shared_ld.sum per kernel).  Test infrastructure.
#include <cstdio>
template <int P>
__global__ void lds128(float4 *out, int iters) {
  __shared__ float4 s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_float4(i, i, i, i);
  __syncthreads();
  const int l = threadIdx.x & 31;
  int idx;
  if (P == 0) idx = 0;                          // one address for the warp
  else if (P == 1) idx = l & 7;                 // quarters identical, 128 B each
  else if (P == 2) idx = l;                     // 512 B contiguous
  else if (P == 3) idx = (l >> 3) * 8;          // quarter-uniform, 4 addresses on distinct banks
  else if (P == 4) idx = l & 15;                // halves identical, 256 B
  else if (P == 5) idx = (l >> 4) * 8;          // half-uniform, 2 addresses distinct banks
  else if (P == 6) idx = (l >> 3) * 32;         // quarter-uniform, 4 addresses same banks
  else idx = (l & 7) + 8 * ((l >> 3) & 1);      // quarters 0,2 identical / 1,3 identical (256 B)
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    float4 v = s[(idx + it * 0) & 1023];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    asm volatile("" ::: "memory");
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int P>
__global__ void lds32(float *out, int iters) {
  __shared__ float s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int l = threadIdx.x & 31;
  const int idx = P == 0 ? 0 : P == 1 ? l : (l >> 3) * 33;
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
    acc += s[idx];
    asm volatile("" ::: "memory");
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  float4 *o;
  cudaMalloc(&o, 1 << 24);
  lds128<0><<<148, 256>>>(o, 1000);
  lds128<1><<<148, 256>>>(o, 1000);
  lds128<2><<<148, 256>>>(o, 1000);
  lds128<3><<<148, 256>>>(o, 1000);
  lds128<4><<<148, 256>>>(o, 1000);
  lds128<5><<<148, 256>>>(o, 1000);
  lds128<6><<<148, 256>>>(o, 1000);
  lds128<7><<<148, 256>>>(o, 1000);
  lds32<0><<<148, 256>>>((float *)o, 1000);
  lds32<1><<<148, 256>>>((float *)o, 1000);
  lds32<2><<<148, 256>>>((float *)o, 1000);
  cudaDeviceSynchronize();
  printf("ok\n");
}
