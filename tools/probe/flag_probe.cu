// Device-flag hand-off probe: stream B polls a flag that stream A sets after a
// delay kernel.  Prints whether B observed it (and how long it took).  Under
// lazy module loading (the CUDA 12 default) round 1 times out: A's kernels are
// loaded on first launch, which waits for the device while B's poller spins;
// with CUDA_MODULE_LOADING=EAGER every round sees the flag after the delay.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o flag_probe flag_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void delay(long long ns) {
    long long t0 = clock64();
    while (clock64() - t0 < ns) {}
}
__global__ void set_ready(uint32_t* f, uint32_t v) {
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__global__ void wait_ready(const uint32_t* f, uint32_t want, int* timed_out) {
    if (threadIdx.x != 0) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (static_cast<int32_t>(v - want) >= 0) return;
        __nanosleep(256);
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 5000000000ull) { *timed_out = 1; return; }
    }
}
int main() {
    uint32_t* f; int* to;
    cudaMalloc(&f, 4); cudaMalloc(&to, 4);
    cudaMemset(f, 0, 4); cudaMemset(to, 0, 4);
    cudaStream_t a, b;
    int lo, hi;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, hi);
    cudaStreamCreateWithPriority(&b, cudaStreamNonBlocking, lo);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (uint32_t k = 1; k <= 5; ++k) {
        cudaMemset(to, 0, 4);
        cudaEventRecord(e0, b);
        wait_ready<<<1, 32, 0, b>>>(f, k, to);
        cudaEventRecord(e1, b);
        delay<<<1, 1, 0, a>>>(2000000);
        set_ready<<<1, 32, 0, a>>>(f, k);
        cudaDeviceSynchronize();
        int h = 0; cudaMemcpy(&h, to, 4, cudaMemcpyDeviceToHost);
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
        printf("round %u: timed_out=%d wait %.3f ms err=%s\n", k, h, ms, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
