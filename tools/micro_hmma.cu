// micro_hmma.cu -- legacy mma.sync.m16n8k16 bf16 on B200: cycles per MMA for
// C independent accumulator chains per warp and W warps per SM (latency vs
// issue throughput of the tensor path the fused step's small GEMMs use).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_02570_b200/csrc micro_hmma.cu -o micro_hmma
#include <cstdio>
#include "common.cuh"
using namespace wsvd_dev;

template <int C>
__global__ void chains(int iters, float* out, long long* cyc) {
    float d[C][4];
    for (int c = 0; c < C; ++c)
        for (int i = 0; i < 4; ++i) d[c][i] = 0.f;
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 9, b1 = a0 ^ 11;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < C; ++c) mma_bf16_16816(d[c], a0, a1, a2, a3, b0, b1);
    }
    const long long t1 = clock64();
    float s = 0.f;
    for (int c = 0; c < C; ++c)
        for (int i = 0; i < 4; ++i) s += d[c][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
void run(int warps) {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 8);
    const int iters = 4096;
    chains<C><<<148, 32 * warps>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("chains %d warps/SM %2d: %.2f cycles per MMA per warp, %.2f cycles per MMA per SM\n", C, warps,
           double(h) / (iters * C), double(h) / (iters * C * warps));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {1, 2, 4, 8, 16}) {
        run<1>(w);
        run<2>(w);
        run<4>(w);
        run<8>(w);
    }
    return 0;
}
