// Block -> SM placement of a one-CTA-per-SM launch (148 blocks, 200 KB smem).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
    extern __shared__ char sm[];
    unsigned s, n;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(n));
    sm[threadIdx.x] = 1;
    if (threadIdx.x == 0) { out[2 * blockIdx.x] = s; out[2 * blockIdx.x + 1] = n; }
}
int main() {
    int *d, h[2 * 148];
    cudaMalloc(&d, sizeof(h));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int rep = 0; rep < 2; ++rep) {
        k<<<148, 512, 200 * 1024>>>(d);
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("nsmid %d\nblock->smid:", h[1]);
        for (int b = 0; b < 148; ++b) printf(" %d", h[2 * b]);
        printf("\n");
    }
    return 0;
}
