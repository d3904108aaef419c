// Microbenchmark (dev tool): mixed-branch BP4 phi on edge pairs, all-fp32
// (phi2: both sides on FFMA2) against a split that evaluates the x < ln 2
// side in double on the fp64 pipe (DFMA), which runs beside the fp32 pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -o /tmp/mbphi tools/mb_phi.cu && /tmp/mbphi
#include <cstdio>
#include "../paper_2605_10433_b200/csrc/qsg_math2.cuh"
using namespace qsg;

// phi_lo in double: ln2 - log x + v H(v), log x = e ln2 + log1p(m - 1)
__device__ __forceinline__ float phi_lo_d(float x)
{
    const uint32_t xb = f2u(x);
    const double fe = (double)(int)((xb >> 23) - 127u);
    const double f = (double)(u2f((xb & 0x007fffffu) | 0x3f800000u) - 1.0f);
    double p = -0.003227271;
    p = fma(p, f, 0.019791102);
    p = fma(p, f, -0.05688295);
    p = fma(p, f, 0.106008776);
    p = fma(p, f, -0.15308061);
    p = fma(p, f, 0.19678909);
    p = fma(p, f, -0.24955378);
    p = fma(p, f, 0.33330205);
    p = fma(p, f, -0.49999923);
    p = fma(p, f, 1.0);
    const double lg = fma(fe, 0.6931471805599453, f * p);
    const double xd = (double)x;
    const double v = xd * xd;
    double H = -2.4306313e-05;
    H = fma(H, v, 0.0003411371);
    H = fma(H, v, -0.0048610563);
    H = fma(H, v, 0.083333336);
    return (float)fma(v, H, 0.6931471805599453 - lg);
}

template <int MODE>
__global__ void kphi(float *o, int n)
{
    float x[8];
    for (int j = 0; j < 8; ++j) x[j] = 0.05f + 0.3f * j + threadIdx.x * 1e-4f;
    float acc = 0.0f;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
            F2 y;
            if (MODE == 0) {
                y = phi2(pk(x[j], x[j + 1]));
            } else if (MODE == 1) {
                const F2 a = phi_hi2(pk(x[j], x[j + 1]));
                const float b0 = phi_lo_d(x[j]), b1 = phi_lo_d(x[j + 1]);
                y = pk(x[j] < kLn2f ? b0 : lo(a), x[j + 1] < kLn2f ? b1 : hi(a));
            } else {
                y = phi_hi2(pk(x[j], x[j + 1]));
            }
            x[j] = fminf(fmaxf(lo(y), 1e-6f), 30.0f);
            x[j + 1] = fminf(fmaxf(hi(y), 1e-6f), 30.0f);
        }
    }
    for (int j = 0; j < 8; ++j) acc += x[j];
    o[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main()
{
    float *o;
    cudaMalloc(&o, 148 * 1024 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int n = 2000;
    const char *nm[] = {"phi2 (both sides FFMA2)", "phi_hi2 FFMA2 + phi_lo double", "phi_hi2 only"};
    for (int rep = 0; rep < 2; ++rep)
        for (int w = 0; w < 3; ++w)
            for (int blk = 128; blk <= 512; blk *= 4) {
                cudaEventRecord(e0);
                if (w == 0) kphi<0><<<148 * (1024 / blk), blk>>>(o, n);
                if (w == 1) kphi<1><<<148 * (1024 / blk), blk>>>(o, n);
                if (w == 2) kphi<2><<<148 * (1024 / blk), blk>>>(o, n);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double phis = 148.0 * 1024 * n * 8;
                printf("%-32s block %3d: %.3f ms, %.3g phi/s\n", nm[w], blk, ms, phis / (ms * 1e-3));
            }
}
