// Is %globaltimer consistent across SMs?  CTA 0 releases a flag after ~20 us;
// every CTA records the globaltimer when it observes it (the observations
// spread by the flag's propagation only if the timers agree).
// nvcc -gencode arch=compute_100a,code=sm_100a -o micro_gtimer tools/micro_gtimer.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
__device__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(unsigned* flag, uint64_t* out, unsigned gen) {
    if (threadIdx.x) return;
    unsigned smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (blockIdx.x == 0) {
        const uint64_t t0 = gt();
        while (gt() - t0 < 20000) {}
        out[3 * gridDim.x] = gt();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(gen) : "memory");
    }
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); } while (v != gen);
    out[3 * blockIdx.x] = gt();
    out[3 * blockIdx.x + 1] = smid;
    // a second observation: the clock64-based elapsed since the first (no timer skew)
    out[3 * blockIdx.x + 2] = clock64();
}
int main() {
    unsigned* flag; uint64_t* out; cudaMalloc(&flag, 4); cudaMemset(flag, 0, 4);
    int G = 148; cudaMalloc(&out, (3 * G + 1) * 8);
    std::vector<uint64_t> h(3 * G + 1);
    for (int it = 1; it <= 5; ++it) {
        k<<<G, 32>>>(flag, out, it);
        cudaDeviceSynchronize();
        cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
        uint64_t mn = ~0ull, mx = 0;
        for (int c = 0; c < G; ++c) { mn = std::min(mn, h[3 * c]); mx = std::max(mx, h[3 * c]); }
        printf("iter %d: observe spread %.2f us (release at %+.2f us from the first observation)\n", it,
               (mx - mn) / 1e3, ((double)h[3 * G] - (double)mn) / 1e3);
        if (it == 5) {
            std::vector<std::pair<uint64_t,int>> v;
            for (int c = 0; c < G; ++c) v.push_back({h[3 * c], (int)h[3 * c + 1]});
            std::sort(v.begin(), v.end());
            printf("earliest smids:"); for (int i = 0; i < 6; ++i) printf(" %d(%.2f)", v[i].second, (v[i].first - mn) / 1e3);
            printf("\nlatest smids:"); for (int i = G - 6; i < G; ++i) printf(" %d(%.2f)", v[i].second, (v[i].first - mn) / 1e3);
            printf("\n");
        }
    }
    return 0;
}
