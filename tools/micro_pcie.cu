// micro_pcie.cu -- how fast can kernels move a decode token's x / y (256 KB)
// across PCIe through mapped (zero-copy) pinned host memory?  Probes the
// request shapes the fused step could use (per-thread loads with different
// cache operators, TMA bulk copies from host memory, coalesced vs fragment
// stores) against the copy engine.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_02570_b200/csrc micro_pcie.cu -o micro_pcie
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

using namespace wsvd_dev;

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

// mode 0: __ldcv float4; 1: plain float4; 2: __ldg float4; 3: __ldcg float4
__global__ void read_thread(const float4* __restrict__ src, float4* __restrict__ dst, int n4, int mode) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
        float4 v;
        if (mode == 0) v = __ldcv(src + i);
        else if (mode == 1) v = src[i];
        else if (mode == 2) v = __ldg(src + i);
        else v = __ldcg(src + i);
        dst[i] = v;
    }
}

// each CTA: one TMA bulk copy of its contiguous piece into shared memory, then out to dst
__global__ void read_tma(const uint8_t* src, uint8_t* dst, int bytes) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t bar;
    const int per = ((bytes / gridDim.x) + 15) & ~15;
    const int off = blockIdx.x * per;
    const int n = min(per, bytes - off);
    if (n <= 0) return;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, n);
        tma_bulk_g2s(sm, src + off, n, &bar);
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x * 16; i < n; i += blockDim.x * 16)
        *reinterpret_cast<uint4*>(dst + off + i) = *reinterpret_cast<const uint4*>(sm + i);
}

// stores: mode 0 = coalesced float4 per thread; 1 = MMA-fragment-like 8-byte
// stores (4 lanes cover 32 contiguous bytes of a row, 8 rows per warp)
__global__ void write_thread(float* __restrict__ dst, int rows, int cols, int mode) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nthr = gridDim.x * blockDim.x;
    if (mode == 0) {
        const int n4 = rows * cols / 4;
        for (int i = tid; i < n4; i += nthr)
            reinterpret_cast<float4*>(dst)[i] = make_float4(1.f, 2.f, 3.f, static_cast<float>(i));
    } else {
        // a 16-column tile per warp: lane (g8, t4) writes columns 2t4.. of rows g8, g8+8 (x 2 column halves)
        const int warp = tid >> 5, lane = tid & 31, nwarp = nthr >> 5;
        const int tiles = cols / 16;
        for (int t = warp; t < tiles; t += nwarp)
            for (int r0 = 0; r0 < rows; r0 += 16)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int r = r0 + (lane >> 2) + ((i & 1) ? 8 : 0);
                    const int c = t * 16 + 2 * (lane & 3) + ((i & 2) ? 8 : 0);
                    if (r < rows) *reinterpret_cast<float2*>(dst + static_cast<size_t>(r) * cols + c) = make_float2(1.f, 2.f);
                }
    }
}

__global__ void write_tma(uint8_t* dst, int bytes) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int per = ((bytes / gridDim.x) + 15) & ~15;
    const int off = blockIdx.x * per;
    const int n = min(per, bytes - off);
    if (n <= 0) return;
    for (int i = threadIdx.x * 16; i < n; i += blockDim.x * 16) *reinterpret_cast<uint4*>(sm + i) = make_uint4(1, 2, 3, i);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                     "r"(smem_u32(sm)), "r"(n) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// a persistent kernel (one 200 KB CTA per SM, like the fused step) that
// waits for a flag a copy-engine stream writes behind an x copy
__global__ void wait_flag(const unsigned* flag, unsigned target, unsigned long long* t) {
    extern __shared__ uint8_t sm[];
    if (threadIdx.x == 0) {
        unsigned long long t0;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
        unsigned v;
        do {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        } while (v < target);
        unsigned long long t1;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
        if (blockIdx.x == 0) {
            t[0] = t0;
            t[1] = t1;
        }
        sm[0] = 1;
    }
}

using WV = int (*)(cudaStream_t, unsigned long long, unsigned, unsigned);

int main() {
    const int B = 16, E = 4096;
    const int bytes = B * E * 4;
    float *xh, *xd, *yh;
    CK(cudaHostAlloc(&xh, bytes, cudaHostAllocMapped));
    CK(cudaHostAlloc(&yh, bytes, cudaHostAllocMapped));
    CK(cudaMalloc(&xd, bytes));
    for (int i = 0; i < B * E; ++i) xh[i] = static_cast<float>(i);
    float *xhd, *yhd;
    CK(cudaHostGetDevicePointer(&xhd, xh, 0));
    CK(cudaHostGetDevicePointer(&yhd, yh, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int reps = 50;
    auto timeit = [&](const char* name, auto fn) {
        for (int i = 0; i < 5; ++i) fn();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int i = 0; i < reps; ++i) fn();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double us = ms * 1e3 / reps;
        printf("%-44s %8.2f us  %7.1f GB/s\n", name, us, bytes / us * 1e-3);
        CK(cudaGetLastError());
    };
    timeit("copy engine H2D 256 KB", [&] { CK(cudaMemcpyAsync(xd, xh, bytes, cudaMemcpyHostToDevice)); });
    timeit("copy engine D2H 256 KB", [&] { CK(cudaMemcpyAsync(yh, xd, bytes, cudaMemcpyDeviceToHost)); });
    const char* rn[4] = {"ldcv", "ld", "ldg", "ldcg"};
    for (int mode = 0; mode < 4; ++mode)
        for (int grid : {148, 296, 592}) {
            char name[96];
            snprintf(name, sizeof name, "zero-copy read %s float4, grid %d x 256", rn[mode], grid);
            timeit(name, [&] { read_thread<<<grid, 256>>>(reinterpret_cast<const float4*>(xhd), reinterpret_cast<float4*>(xd), bytes / 16, mode); });
        }
    for (int grid : {32, 64, 128, 148}) {
        const int smem = ((bytes / grid) + 15) & ~15;
        CK(cudaFuncSetAttribute(read_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        char name[96];
        snprintf(name, sizeof name, "zero-copy read TMA bulk, %d CTAs x %d KB", grid, smem / 1024);
        timeit(name, [&] { read_tma<<<grid, 256, smem>>>(reinterpret_cast<const uint8_t*>(xhd), reinterpret_cast<uint8_t*>(xd), bytes); });
    }
    for (int grid : {148, 296}) {
        char name[96];
        snprintf(name, sizeof name, "zero-copy write float4 coalesced, grid %d", grid);
        timeit(name, [&] { write_thread<<<grid, 256>>>(yhd, B, E, 0); });
        snprintf(name, sizeof name, "zero-copy write 8-byte fragments, grid %d", grid);
        timeit(name, [&] { write_thread<<<grid, 256>>>(yhd, B, E, 1); });
    }
    for (int grid : {32, 64, 148}) {
        const int smem = ((bytes / grid) + 15) & ~15;
        CK(cudaFuncSetAttribute(write_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        char name[96];
        snprintf(name, sizeof name, "zero-copy write TMA bulk, %d CTAs", grid);
        timeit(name, [&] { write_tma<<<grid, 256, smem>>>(reinterpret_cast<uint8_t*>(yhd), bytes); });
    }
    {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        CK(cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q));
        WV wv = reinterpret_cast<WV>(fn);
        unsigned* flag;
        unsigned long long* tt;
        CK(cudaMalloc(&flag, 4));
        CK(cudaMemset(flag, 0, 4));
        CK(cudaHostAlloc(&tt, 16, cudaHostAllocMapped));
        unsigned long long* ttd;
        CK(cudaHostGetDevicePointer(&ttd, tt, 0));
        cudaStream_t ks, xs;
        CK(cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking));
        CK(cudaFuncSetAttribute(wait_flag, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        for (int order = 0; order < 2; ++order) {
            double sum = 0, wall = 0;
            const int n = 20;
            for (int it = 0; it < n + 3; ++it) {
                const unsigned target = order * 1000 + it + 1;
                cudaEvent_t a0, a1;
                CK(cudaEventCreate(&a0));
                CK(cudaEventCreate(&a1));
                CK(cudaEventRecord(a0, ks));
                if (order == 0) {
                    CK(cudaMemcpyAsync(xd, xh, bytes, cudaMemcpyHostToDevice, xs));
                    if (wv(xs, reinterpret_cast<unsigned long long>(flag), target, 0) != 0) { printf("wv failed\n"); return 1; }
                    wait_flag<<<148, 320, 200 * 1024, ks>>>(flag, target, ttd);
                } else {
                    wait_flag<<<148, 320, 200 * 1024, ks>>>(flag, target, ttd);
                    CK(cudaMemcpyAsync(xd, xh, bytes, cudaMemcpyHostToDevice, xs));
                    if (wv(xs, reinterpret_cast<unsigned long long>(flag), target, 0) != 0) { printf("wv failed\n"); return 1; }
                }
                CK(cudaEventRecord(a1, ks));
                CK(cudaStreamSynchronize(ks));
                CK(cudaStreamSynchronize(xs));
                float ms;
                CK(cudaEventElapsedTime(&ms, a0, a1));
                if (it >= 3) {
                    sum += (tt[1] - tt[0]) * 1e-3;
                    wall += ms * 1e3;
                }
            }
            printf("CE x copy + flag, %s: kernel waits %.2f us, stream span %.2f us\n",
                   order == 0 ? "copy issued first" : "kernel issued first", sum / n, wall / n);
        }
    }
    // link bandwidth with a large copy
    float *bh, *bd;
    const size_t big = 64ull << 20;
    CK(cudaHostAlloc(&bh, big, 0));
    CK(cudaMalloc(&bd, big));
    CK(cudaEventRecord(e0));
    for (int i = 0; i < 5; ++i) CK(cudaMemcpyAsync(bd, bh, big, cudaMemcpyHostToDevice));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("copy engine H2D 64 MB: %.1f GB/s\n", 5 * big / (ms * 1e-3) * 1e-9);
    CK(cudaEventRecord(e0));
    for (int i = 0; i < 5; ++i) CK(cudaMemcpyAsync(bh, bd, big, cudaMemcpyDeviceToHost));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("copy engine D2H 64 MB: %.1f GB/s\n", 5 * big / (ms * 1e-3) * 1e-9);
    return 0;
}
