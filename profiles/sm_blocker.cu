// Occupies n SMs (one CTA per SM via max dynamic smem) until *flag != 0.
#include <cuda_runtime.h>
__global__ void k_block(volatile int* flag) {
  extern __shared__ int s[];
  if (threadIdx.x == 0) { s[0] = 0; while (*flag == 0) { __nanosleep(1000); } }
  __syncthreads();
}
extern "C" int blocker_launch(void* stream, int n, int* flag) {
  cudaFuncSetAttribute(k_block, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_block<<<n, 32, 200 * 1024, (cudaStream_t)stream>>>(flag);
  return (int)cudaGetLastError();
}
