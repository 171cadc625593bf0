// micro_barrier.cu -- latency of grid-wide barriers among 148 persistent CTAs
// (one per SM), as used by the fused step (step.cu):
//   A: one counter + generation (atom.add.acq_rel, last arriver releases)
//   B: per-CTA flags (st.release) polled by CTA 0, then one release word
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_barrier micro_barrier.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(320, 1) bar_a(unsigned* bar, int iters, unsigned long long* out) {
    extern __shared__ char pad[];
    (void)pad;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned g0 = ld_acq(bar + 1);
            unsigned old;
            asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
            if (old == gridDim.x - 1) {
                asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
            } else {
                while (ld_acq(bar + 1) == g0) {
                }
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

__global__ void __launch_bounds__(320, 1) bar_b(unsigned* flags, unsigned* go, int iters, unsigned base,
                                                unsigned long long* out) {
    extern __shared__ char pad[];
    (void)pad;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const unsigned epoch = base + it + 1;
        __syncthreads();
        if (threadIdx.x == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * 32), "r"(epoch) : "memory");
        if (blockIdx.x == 0) {
            for (int i = threadIdx.x; i < gridDim.x; i += blockDim.x)
                while (ld_acq(flags + i * 32) < epoch) {
                }
            __syncthreads();
            if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(go), "r"(epoch) : "memory");
        } else if (threadIdx.x == 0) {
            while (ld_acq(go) < epoch) {
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

// C: every CTA polls every flag (thread i <-> CTA i): one hop
__global__ void __launch_bounds__(320, 1) bar_c(unsigned* flags, int iters, unsigned base, unsigned long long* out) {
    extern __shared__ char pad[];
    (void)pad;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const unsigned epoch = base + it + 1;
        __syncthreads();
        if (threadIdx.x == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * 32), "r"(epoch) : "memory");
        for (int i = threadIdx.x; i < gridDim.x; i += blockDim.x)
            while (ld_acq(flags + i * 32) < epoch) {
            }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

// D: monotone counter, fire-and-forget arrival, everyone polls for epoch * G
__global__ void __launch_bounds__(320, 1) bar_d(unsigned* cnt, int iters, unsigned base, unsigned long long* out) {
    extern __shared__ char pad[];
    (void)pad;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const unsigned target = (base + it + 1) * gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
            while (ld_acq(cnt) < target) {
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *bar, *flags, *go;
    unsigned long long* out;
    cudaMalloc(&bar, 64);
    cudaMalloc(&flags, sms * 128);
    cudaMalloc(&go, 64);
    cudaMalloc(&out, 64);
    cudaMemset(bar, 0, 64);
    cudaMemset(flags, 0, sms * 128);
    cudaMemset(go, 0, 64);
    const int smem = 200 * 1024, iters = 1000;
    cudaFuncSetAttribute(bar_a, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bar_b, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    bar_a<<<sms, 320, smem>>>(bar, 10, out);
    cudaEventRecord(e0);
    bar_a<<<sms, 320, smem>>>(bar, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("A counter+generation: %.3f us per barrier (%s)\n", ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    unsigned base = 0;
    bar_b<<<sms, 320, smem>>>(flags, go, 10, base, out);
    base += 10;
    cudaEventRecord(e0);
    bar_b<<<sms, 320, smem>>>(flags, go, iters, base, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("B flags+master: %.3f us per barrier (%s)\n", ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    cudaFuncSetAttribute(bar_c, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bar_d, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(flags, 0, sms * 128);
    bar_c<<<sms, 320, smem>>>(flags, 10, 0, out);
    cudaEventRecord(e0);
    bar_c<<<sms, 320, smem>>>(flags, iters, 10, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("C all-poll flags: %.3f us per barrier (%s)\n", ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    cudaMemset(bar, 0, 64);
    bar_d<<<sms, 320, smem>>>(bar, 10, 0, out);
    cudaEventRecord(e0);
    bar_d<<<sms, 320, smem>>>(bar, iters, 10, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("D monotone counter: %.3f us per barrier (%s)\n", ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
