// Throughput microbenchmark: cycles per warp-instruction per SMSP for packed fp32 ops.
#include <cstdio>
#include <cuda_runtime.h>
#define N 256
template <int MODE>
__global__ void kern(float* out, long long* cyc, float a, float b) {
  float2 x[8];
  for (int i = 0; i < 8; ++i) x[i] = make_float2(a + i + threadIdx.x, b - i);
  const float2 av = make_float2(a, b), cv = make_float2(b, a);
  unsigned u[8];
  for (int i = 0; i < 8; ++i) u[i] = __float_as_uint(a) + i * 7 + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int k = 0; k < N; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) x[i] = __ffma2_rn(x[i], av, cv);                                   // FFMA2 reg
      if (MODE == 1) x[i] = __fadd2_rn(x[i], make_float2(12582912.0f, 12582912.0f));     // FADD2 imm
      if (MODE == 2) x[i].x = __fmaf_rn(x[i].x, a, b);                                   // FFMA scalar reg
      if (MODE == 3) x[i].x = __fmaf_rn(x[i].x, 1.0001f, 0.5f);                          // FFMA imm
      if (MODE == 4) u[i] = u[i] * 0x800000u + u[(i + 1) & 7];                           // IMAD
      if (MODE == 5) u[i] = __byte_perm(u[i], u[(i + 3) & 7], 0x5140);                   // PRMT
      if (MODE == 6) x[i] = __ffma2_rn(x[i], x[(i + 1) & 7], make_float2(0.5f, 0.25f));  // FFMA2 reg x reg + imm
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8 * 1024);
  const char* names[] = {"FFMA2 r,s,s", "FADD2 imm", "FFMA reg", "FFMA imm", "IMAD", "PRMT", "FFMA2 r,r,imm"};
  for (int warps = 4; warps <= 32; warps *= 2)
    for (int m = 0; m < 7; ++m) {
      auto launch = [&](void) {
        switch (m) {
          case 0: kern<0><<<148, warps * 32>>>(out, cyc, 1.f, 2.f); break;
          case 1: kern<1><<<148, warps * 32>>>(out, cyc, 1.f, 2.f); break;
          case 2: kern<2><<<148, warps * 32>>>(out, cyc, 1.f, 2.f); break;
          case 3: kern<3><<<148, warps * 32>>>(out, cyc, 1.f, 2.f); break;
          case 4: kern<4><<<148, warps * 32>>>(out, cyc, 1.f, 2.f); break;
          case 5: kern<5><<<148, warps * 32>>>(out, cyc, 1.f, 2.f); break;
          case 6: kern<6><<<148, warps * 32>>>(out, cyc, 1.f, 2.f); break;
        }
      };
      launch(); cudaDeviceSynchronize(); launch();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      // per SMSP: warps/4 warps each issuing N*8 instrs
      double per = double(c) / (double(N) * 8 * (warps / 4));
      printf("warps/SM %2d  %-14s cycles per warp-instr per SMSP: %.2f\n", warps, names[m], per);
    }
  return 0;
}
