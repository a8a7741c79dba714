// Throughput microbenchmark, part 2: cycles per warp-instruction per SMSP for
// the fp16x2 / integer ops a half-precision snapkv epilogue would use.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 profiles/pipebench2.cu -o pipebench2 && ./pipebench2
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#define N 256
template <int MODE>
__global__ void kern(float* out, long long* cyc, float a, float b) {
  __half2 h[8];
  float2 x[8];
  unsigned u[8];
  for (int i = 0; i < 8; ++i) {
    h[i] = __floats2half2_rn(a * 0.01f * i, b * 0.01f + threadIdx.x * 1e-4f);
    x[i] = make_float2(a + i + threadIdx.x, b - i);
    u[i] = __float_as_uint(a) + i * 7 + threadIdx.x;
  }
  const __half2 hc = __floats2half2_rn(0.999f, 1.001f), hd = __floats2half2_rn(0.5f, 0.25f);
  __syncthreads();
  long long t0 = clock64();
  for (int k = 0; k < N; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) h[i] = __hfma2(h[i], hc, hd);                                 // HFMA2 reg, reg, reg
      if (MODE == 1) h[i] = __hadd2(h[i], __floats2half2_rn(1536.f, 1536.f));     // HADD2 imm
      if (MODE == 2) h[i] = __hmax2(h[i], h[(i + 1) & 7]);                        // HMNMX2
      if (MODE == 3) {                                                            // F2FP.F16.F32.PACK_AB
        const __half2 c = __float22half2_rn(x[i]);
        x[i] = make_float2(__uint_as_float(*reinterpret_cast<const unsigned*>(&c)), x[i].y);
      }
      if (MODE == 4) u[i] = (u[i] & 0x003f003fu) ^ u[(i + 1) & 7];                // LOP3
      if (MODE == 5) x[i].x = fmaxf(x[i].x, x[(i + 1) & 7].x);                    // FMNMX
      if (MODE == 6) u[i] = __dp4a(u[i], 0x01010101u, u[(i + 1) & 7]);            // IDP.4A
      if (MODE == 7) u[i] = max(u[i], u[(i + 1) & 7]);                            // VIMNMX
      if (MODE == 8) u[i] = u[i] + (u[(i + 1) & 7] << 10);                        // LEA / IMAD.SHL + IADD
      if (MODE == 9) h[i] = __hfma2(h[i], h[(i + 1) & 7], hd);                     // HFMA2 r, r, r (dep)
      if (MODE == 10) {                                                           // FHFMA.BF16: bf16 x bf16 + f32
        float r;
        asm("{.reg .b16 l, h; mov.b32 {l, h}, %1; fma.rn.f32.bf16 %0, h, l, %2;}" : "=f"(r) : "r"(u[i]), "f"(x[i].x));
        x[i].x = r;
        u[i] ^= __float_as_uint(r);
      }
      if (MODE == 11) u[i] = __vimin_s16x2_relu(u[i], u[(i + 3) & 7]);            // VIMNMX.S16x2 relu
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += __low2float(h[i]) + __high2float(h[i]) + x[i].x + x[i].y + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int M>
void run(float* out, long long* cyc, int warps) { kern<M><<<148, warps * 32>>>(out, cyc, 1.f, 2.f); }
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8 * 1024);
  const char* names[] = {"HFMA2", "HADD2 imm", "HMNMX2", "F2FP f32x2->f16x2", "LOP3", "FMNMX", "IDP.4A", "VIMNMX",
                         "shift+add", "HFMA2 r,r,r", "FHFMA.BF16 (+LOP3)", "VIMNMX.S16x2.RELU"};
  void (*fn[])(float*, long long*, int) = {run<0>, run<1>, run<2>, run<3>, run<4>, run<5>, run<6>, run<7>, run<8>, run<9>, run<10>, run<11>};
  for (int warps = 8; warps <= 32; warps *= 2)
    for (int m = 0; m < 12; ++m) {
      fn[m](out, cyc, warps); cudaDeviceSynchronize(); fn[m](out, cyc, warps);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double per = double(c) / (double(N) * 8 * (warps / 4));
      printf("warps/SM %2d  %-18s cycles per warp-instr per SMSP: %.2f\n", warps, names[m], per);
    }
  return 0;
}
