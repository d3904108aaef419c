// Pipe-rate microbenchmark (dev tool): FFMA (immediate and 3-register),
// FFMA2, FMNMX and DFMA issue rates per SMSP cycle on the box's GPU, and
// whether DFMA (fp64 pipe) overlaps FFMA2 (fma pipe) in one instruction
// stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mb tools/mb_pipes.cu && /tmp/mb
#include <cstdio>
#include "../paper_2605_10433_b200/csrc/qsg_math2.cuh"
using namespace qsg;
// throughput: 8 independent chains per thread, imm-form coefficient
__global__ void k1(float* o, int n) {  // scalar FFMA imm
  float a[8]; for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], 0.999f, 0.5f);
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j]; o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k2(float* o, int n) {  // paired FFMA2 imm
  F2 a[8]; for (int j = 0; j < 8; ++j) a[j] = pk(threadIdx.x * 1e-3f + j, j * 0.5f);
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma2(a[j], bc(0.999f), bc(0.5f));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += lo(a[j]) + hi(a[j]); o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k3(float* o, int n) {  // scalar FFMA 3-reg
  float a[8], b = threadIdx.x * 1e-6f + 0.999f, c = 0.5f + threadIdx.x * 1e-7f; for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b, c);
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j]; o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k4(float* o, int n) {  // FMNMX (ALU)
  float a[8], b = threadIdx.x * 1e-6f + 0.999f; for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fminf(fmaxf(a[j], b), 100.f + j);
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j]; o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k5(double* o, int n) {  // DFMA
  double a[8], b = threadIdx.x * 1e-6 + 0.999, c = 0.5 + threadIdx.x * 1e-7; for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += a[j]; o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k6(float* o, int n) {  // 8 FFMA2 + 4 DFMA per iteration (independent chains)
  F2 a[8]; for (int j = 0; j < 8; ++j) a[j] = pk(threadIdx.x * 1e-3f + j, j * 0.5f);
  double d[4], b = threadIdx.x * 1e-6 + 0.999, c = 0.5 + threadIdx.x * 1e-7; for (int j = 0; j < 4; ++j) d[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a[j] = fma2(a[j], bc(0.999f), bc(0.5f));
      if (j & 1) d[j >> 1] = fma(d[j >> 1], b, c);
    }
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += lo(a[j]) + hi(a[j]);
  for (int j = 0; j < 4; ++j) s += (float)d[j];
  o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k7(float* o, int n) {  // MUFU.EX2
  float a[8]; for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j * 0.1f;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[j])); a[j] = y * -0.5f; }
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j]; o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int n = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int w = 1; w <= 7; ++w) {
      cudaEventRecord(e0);
      if (w == 1) k1<<<148 * 2, 512>>>(o, n);
      if (w == 2) k2<<<148 * 2, 512>>>(o, n);
      if (w == 3) k3<<<148 * 2, 512>>>(o, n);
      if (w == 4) k4<<<148 * 2, 512>>>(o, n);
      if (w == 5) k5<<<148 * 2, 512>>>((double*)o, n);
      if (w == 6) k6<<<148 * 2, 512>>>(o, n);
      if (w == 7) k7<<<148 * 2, 512>>>(o, n);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warp_instr = 148.0 * 2 * 512 / 32 * n * 8 * (w == 4 || w == 7 ? 2 : (w == 6 ? 1.5 : 1));
      double cyc = ms * 1e-3 * 1.965e9 * 148 * 4;  // SMSP-cycles
      const char* nm[] = {"", "FFMA imm", "FFMA2 imm", "FFMA 3reg", "FMNMX x2", "DFMA", "FFMA2 x8 + DFMA x4", "MUFU.EX2 + FMUL"};
      printf("%s: %.3f ms, warp-instr per SMSP-cycle %.3f\n", nm[w], ms, warp_instr / cyc);
    }
  }
}
