// micro_tma.cu -- streaming-bandwidth probe for the attention kernel's
// pipeline structure (producer warp + TMA bulk ring + consumer warps).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2604_02570_b200/csrc micro_tma.cu -o micro_tma
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace wsvd_dev;

template <int NCW>
__global__ void __launch_bounds__(32 * (NCW + 1), 1)
    stream_kernel(const uint8_t* __restrict__ src, size_t total, int stage_bytes, int stages, int mode,
                  float* sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
    uint64_t* empty = full + stages;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int i = 0; i < stages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const size_t nstage = total / stage_bytes;
    if (warp == NCW) {
        if (lane == 0) {
            int slot = 0;
            uint32_t ph = 0;
            const size_t per = (nstage + gridDim.x - 1) / gridDim.x;
            const size_t s0 = (mode & 2) ? blockIdx.x * per : blockIdx.x, s1 = (mode & 2) ? min(nstage, s0 + per) : nstage;
            const size_t ds = (mode & 2) ? 1 : gridDim.x;
            for (size_t s = s0; s < s1; s += ds) {
                mbar_wait(&empty[slot], ph ^ 1u);
                mbar_arrive_expect_tx(&full[slot], stage_bytes);
                tma_bulk_g2s(smem + slot * stage_bytes, src + s * stage_bytes, stage_bytes, &full[slot]);
                if (++slot == stages) { slot = 0; ph ^= 1u; }
            }
        }
        return;
    }
    int slot = 0;
    uint32_t ph = 0;
    float acc = 0.f;
    const int rowb = stage_bytes / (32 * NCW);
    const size_t per = (nstage + gridDim.x - 1) / gridDim.x;
    const size_t s0 = (mode & 2) ? blockIdx.x * per : blockIdx.x, s1 = (mode & 2) ? min(nstage, s0 + per) : nstage;
    const size_t ds = (mode & 2) ? 1 : gridDim.x;
    for (size_t s = s0; s < s1; s += ds) {
        mbar_wait(&full[slot], ph);
        if (mode & 1) {
            const uint32_t row = smem_u32(smem + slot * stage_bytes) + tid * rowb;
            for (int c = 0; c < rowb; c += 16) {
                uint4 v = lds128(row + ((c + lane * 16) % rowb));
                acc += __uint_as_float(v.x) + __uint_as_float(v.w);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == stages) { slot = 0; ph ^= 1u; }
    }
    if (acc == 123.f) sink[0] = acc;
}

// plain vectorised loads, many CTAs (reference point)
__global__ void ldg_kernel(const uint4* __restrict__ src, size_t n, float* sink) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = ldg_nc128(src + i);
        acc += __uint_as_float(v.x);
    }
    if (acc == 123.f) sink[0] = acc;
}

int main() {
    const size_t total = 1024ull << 20;
    uint8_t* buf;
    float* sink;
    cudaMalloc(&buf, total);
    cudaMalloc(&sink, 64);
    cudaMemset(buf, 0, total);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto timeit = [&](auto fn) {
        fn();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        return total / (ms / 10 / 1e3) / 1e9;
    };
    printf("ldg 148x8x256: %.0f GB/s\n", timeit([&] { ldg_kernel<<<sms * 8, 256>>>((const uint4*)buf, total / 16, sink); }));
    for (int mode = 0; mode < 4; ++mode)
        for (int sb : {8192, 16384, 32768})
            for (int st : {4, 6, 8, 12}) {
                const int smem = sb * st + 256;
                if (smem > 220 * 1024) continue;
                auto k = stream_kernel<8>;
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                for (int g : {sms / 2, sms, 2 * sms}) {
                    if (g == 2 * sms && smem > 110 * 1024) continue;
                    double gbs = timeit([&] { k<<<g, 288, smem>>>(buf, total, sb, st, mode, sink); });
                    cudaError_t err = cudaGetLastError();
                    printf("mode %d stage %6d x %2d grid %3d: %6.0f GB/s %s\n", mode, sb, st, g, gbs,
                           err == cudaSuccess ? "" : cudaGetErrorString(err));
                }
            }
    return 0;
}
