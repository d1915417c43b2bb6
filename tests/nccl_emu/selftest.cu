// selftest.cu -- TEST INFRASTRUCTURE: the NCCL emulator alone, 2 ranks as threads.
#include <cuda_runtime.h>
#include <nccl.h>
#include <cstdio>
#include <thread>
#include <vector>

static ncclUniqueId id;
static int fails = 0;

static void rank_main(int r) {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    double *a, *b, *s;
    cudaMalloc(&a, 8 * 16);
    cudaMalloc(&b, 8 * 16);
    cudaMalloc(&s, 8);
    std::vector<double> h(16, r + 1.0);
    cudaMemcpy(a, h.data(), 8 * 16, cudaMemcpyHostToDevice);
    ncclComm_t c;
    if (ncclCommInitRank(&c, 2, id, r) != ncclSuccess) { std::printf("init failed\n"); ++fails; return; }
    std::printf("rank %d init\n", r); std::fflush(stdout);
    for (int it = 0; it < 3; ++it) {
        ncclGroupStart();
        ncclSend(a, 16, ncclDouble, 1 - r, c, st);
        ncclRecv(b, 16, ncclDouble, 1 - r, c, st);
        ncclGroupEnd();
    }
    double v = r + 1.0;
    cudaMemcpyAsync(s, &v, 8, cudaMemcpyHostToDevice, st);
    ncclAllReduce(s, s, 1, ncclDouble, ncclSum, c, st);
    std::printf("rank %d posted, syncing\n", r); std::fflush(stdout);
    cudaError_t e = cudaStreamSynchronize(st);
    double hb[16], hs;
    cudaMemcpy(hb, b, 8 * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hs, s, 8, cudaMemcpyDeviceToHost);
    std::printf("rank %d sync=%s b[0]=%g sum=%g\n", r, cudaGetErrorString(e), hb[0], hs);
    if (hb[0] != 2.0 - r || hs != 3.0) ++fails;
}

int main() {
    ncclGetUniqueId(&id);
    std::thread t0(rank_main, 0), t1(rank_main, 1);
    t0.join();
    t1.join();
    std::printf(fails ? "SELFTEST FAILED\n" : "SELFTEST OK\n");
    return fails != 0;
}
