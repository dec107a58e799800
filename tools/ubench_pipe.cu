// The tc3 row pipeline in isolation: 12 producer warps cp.async 96 random 512-byte rows per
// group into a ring of NS stages (48 KB, 128B-swizzled), completion by
// cp.async.mbarrier.arrive.noinc (or wait_group + arrive), one consumer warp releasing each
// stage as soon as it is full.  Reports GB/s of row data.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

constexpr int NGROUPS = 200000;  // x 96 rows = 19.2M rows = 9.8 GB
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(su32(bar)), "r"(parity) : "memory");
}

__device__ int g_delay;
template <int NS, int NP, bool NOINC>
__global__ void k_pipe(const float *__restrict__ data, const int *__restrict__ ids, float *out) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char *base = raw + ((1024 - (su32(raw) & 1023)) & 1023);
    __shared__ uint64_t full[NS], empty[NS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(NOINC ? NP * 32 : NP));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int nmine = (NGROUPS - blockIdx.x + gridDim.x - 1) / gridDim.x;
    if (warp == 0) {  // consumer
        float acc = 0;
        for (int g = 0; g < nmine; ++g) {
            const int s = g % NS;
            mbar_wait(&full[s], (g / NS) & 1);
            acc += *(float *)(base + s * 49152 + lane * 4);
            { const long long t0 = clock64(); while (clock64() - t0 < g_delay) { } }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        }
        if (acc == 12345.f) out[0] = acc;
    } else if (warp <= NP) {
        const int pi = warp - 1;
        const uint32_t lo = (uint32_t)((lane >> 3) * 12288), lx = lane & 7;
        for (int g = 0; g < nmine; ++g) {
            const int s = g % NS;
            mbar_wait(&empty[s], ((g / NS) & 1) ^ 1);
            const int gg = blockIdx.x + g * gridDim.x;
            const uint32_t stg = su32(base + s * 49152);
            for (int q = 0; q < 96 / NP; ++q) {
                const int r = pi + NP * q;
                const int id = ids[(int64_t)gg * 96 + r];
                const float *src = data + (int64_t)id * 128 + lane * 4;
                const uint32_t dst = stg + lo + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128) + ((lx ^ (uint32_t)(r & 7)) << 4);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(16));
            }
            if (NOINC) {
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
            } else {
                asm volatile("cp.async.commit_group;\n" ::);
                asm volatile("cp.async.wait_group 0;\n" ::);
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
            }
        }
    }
}

int main() {
    const int64_t N = 1000000;
    std::vector<float> h(N * 128, 1.0f);
    std::vector<int> hid((size_t)NGROUPS * 96);
    std::mt19937 rng(1);
    for (auto &x : hid) x = rng() % N;
    float *d; int *did; float *out;
    cudaMalloc(&d, N * 512); cudaMalloc(&did, hid.size() * 4); cudaMalloc(&out, 4);
    cudaMemcpy(d, h.data(), N * 512, cudaMemcpyHostToDevice);
    cudaMemcpy(did, hid.data(), hid.size() * 4, cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char *name, auto kern, int nthreads, int smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kern<<<sms, nthreads, smem>>>(d, did, out); cudaDeviceSynchronize();
        cudaEventRecord(e0);
        kern<<<sms, nthreads, smem>>>(d, did, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s %8.3f ms  %7.1f GB/s  %s\n", name, ms, NGROUPS * 96.0 * 512 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    for (int dly : {0, 1000, 2000, 4000, 8000}) {
        cudaMemcpyToSymbol(g_delay, &dly, 4);
        char nm[64]; snprintf(nm, 64, "NS=4 NP=9 noinc consumer delay %d", dly);
        run(nm, k_pipe<4, 9, true>, 10 * 32, 4 * 49152 + 2048);
    }
    int z = 0; cudaMemcpyToSymbol(g_delay, &z, 4);
    run("NS=4 NP=12 noinc", k_pipe<4, 12, true>, 13 * 32, 4 * 49152 + 2048);
    run("NS=4 NP=12 waitgroup", k_pipe<4, 12, false>, 13 * 32, 4 * 49152 + 2048);
    run("NS=4 NP=16 noinc", k_pipe<4, 16, true>, 17 * 32, 4 * 49152 + 2048);
    run("NS=4 NP=24 noinc", k_pipe<4, 24, true>, 25 * 32, 4 * 49152 + 2048);
    run("NS=2 NP=12 noinc", k_pipe<2, 12, true>, 13 * 32, 2 * 49152 + 2048);
    run("NS=3 NP=12 noinc", k_pipe<3, 12, true>, 13 * 32, 3 * 49152 + 2048);
    return 0;
}
