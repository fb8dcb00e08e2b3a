#include <cstdio>
#include <cuda_runtime.h>
// 32M floats y; each warp adds a 8-column x 32-row block repeatedly: scalar red (lane=row),
// or v4 red (lane holds 4 consecutive rows of one column).
__global__ void k_scalar(float* y, int n, int reps) {
  int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int r = 0; r < reps; ++r) {
    long base = ((long)(w * reps + r) * 256) % (32L << 20);
    for (int j = 0; j < 8; ++j) atomicAdd(y + base + j * 32 + lane, 1.0f);
  }
}
__global__ void k_v4(float* y, int n, int reps) {
  int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int r = 0; r < reps; ++r) {
    long base = ((long)(w * reps + r) * 256) % (32L << 20);
    for (int j = 0; j < 2; ++j) {
      float* p = y + base + j * 128 + lane * 4;
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
    }
  }
}
__global__ void k_st(float* y, int n, int reps) {
  int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int r = 0; r < reps; ++r) {
    long base = ((long)(w * reps + r) * 256) % (32L << 20);
    for (int j = 0; j < 2; ++j) reinterpret_cast<float4*>(y + base + j * 128)[lane] = make_float4(1, 1, 1, 1);
  }
}
int main() {
  float* y; cudaMalloc(&y, (32L << 20) * 4); cudaMemset(y, 0, (32L << 20) * 4);
  int blocks = 148 * 4, threads = 128, reps = 256;
  double floats = (double)blocks * threads / 32 * reps * 256;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int kind = 0; kind < 3; ++kind) {
    for (int it = 0; it < 2; ++it) {
      cudaEventRecord(a);
      if (kind == 0) k_scalar<<<blocks, threads>>>(y, 0, reps);
      else if (kind == 1) k_v4<<<blocks, threads>>>(y, 0, reps);
      else k_st<<<blocks, threads>>>(y, 0, reps);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (it) printf("%s: %.3f ms, %.1f G floats/s\n", kind == 0 ? "scalar red" : kind == 1 ? "v4 red" : "st.v4", ms, floats / ms / 1e6);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
