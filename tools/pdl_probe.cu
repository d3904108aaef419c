// Does programmatic dependent launch overlap a draining grid with the next
// one on this box?  (dev tool)  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void drain_kernel(long long slow_ns, long long fast_ns, int trigger)
{
    if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const long long ns = blockIdx.x == 0 ? slow_ns : fast_ns;
    const unsigned long long t0 = gtime();
    while ((long long)(gtime() - t0) < ns) {
    }
}

int main()
{
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int pdl = 0; pdl < 2; ++pdl) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a, s);
            for (int k = 0; k < 4; ++k) {
                cudaLaunchConfig_t c = {};
                c.gridDim = dim3(sms * 4);
                c.blockDim = dim3(160);
                c.dynamicSmemBytes = 0;
                c.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                c.attrs = at;
                c.numAttrs = pdl;
                // block 0 runs 2 ms, the rest 0.5 ms: without overlap 4 x 2 ms
                cudaLaunchKernelEx(&c, drain_kernel, 2000000LL, 500000LL, pdl);
            }
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("pdl=%d rep=%d: 4 launches in %.3f ms (%s)\n", pdl, rep, ms, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
