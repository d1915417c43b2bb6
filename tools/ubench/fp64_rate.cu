// FP64 pipe throughput/latency probe: independent DFMA/DADD chains at several
// warps-per-SM and ILP settings.  Prints warp-instructions per cycle per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, int OP>
__global__ void k(double* out, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < ILP; ++i) {
                if (OP == 0) x[i] = fma(x[i], a, b);
                else if (OP == 1) x[i] = x[i] + b;
                else if (OP == 2) x[i] = x[i] * a;
                else if (OP == 3) x[i] = x[i] + x[(i + 1) % ILP];           // two vector operands
                else if (OP == 4) x[i] = fma(x[i], x[(i + 1) % ILP], x[(i + 2) % ILP]);  // three
                else x[i] = fma(x[i], a, x[(i + 1) % ILP]);                // two + uniform (the kernel's form)
            }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

template <int ILP, int OP>
void run(const char* name, int warps_per_sm, int nsm, int clk_mhz) {
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 2000;
    dim3 grid(nsm), block(32 * warps_per_sm);
    k<ILP, OP><<<grid, block>>>(out, 10, 0.999, 1e-3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<ILP, OP><<<grid, block>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double winstr = (double)warps_per_sm * iters * 16 * ILP;  // per SM
    const double cycles = ms * 1e-3 * clk_mhz * 1e6;
    printf("%-5s ILP=%d warps/SM=%2d : %.3f warp-instr/clk/SM  (%.2f TFLOP/s-equiv)\n", name, ILP, warps_per_sm,
           winstr / cycles, winstr * 32 * nsm * (OP == 0 || OP >= 4 ? 2 : 1) / (ms * 1e-3) / 1e12);
    cudaFree(out);
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int clk = 1965;
    for (int w : {4, 8, 16, 32}) {
        run<1, 0>("dfma", w, nsm, clk);
        run<2, 0>("dfma", w, nsm, clk);
        run<4, 0>("dfma", w, nsm, clk);
        run<8, 0>("dfma", w, nsm, clk);
    }
    for (int w : {8, 16}) {
        run<4, 3>("dadd2", w, nsm, clk);
        run<8, 3>("dadd2", w, nsm, clk);
        run<4, 4>("dfma3", w, nsm, clk);
        run<8, 4>("dfma3", w, nsm, clk);
        run<4, 5>("dfma2u", w, nsm, clk);
        run<8, 5>("dfma2u", w, nsm, clk);
    }
    for (int w : {8, 16}) {
        run<1, 1>("dadd", w, nsm, clk);
        run<4, 1>("dadd", w, nsm, clk);
        run<8, 1>("dadd", w, nsm, clk);
        run<4, 2>("dmul", w, nsm, clk);
    }
    return 0;
}
