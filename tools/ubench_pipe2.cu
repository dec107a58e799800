// The tc3 row pipeline in isolation with a stage HOLD: NP producer warps cp.async 96 random
// 512-byte rows per group into NS 48-KB stages (noinc arrivals); NS consumer warps (one per
// stage) keep each landed stage for HOLD cycles before releasing it.  Reports GB/s and the
// mean issue -> landed latency, to separate memory latency from consumer hold time.
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

__device__ int g_hold, g_mode;
__device__ float *g_meta_src; __device__ float *g_store_dst;
__device__ unsigned long long g_lat, g_cnt;
template <int NS, int NP>
__global__ void k_pipe(const float *__restrict__ data, const int *__restrict__ ids, float *out) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char *base = raw + ((1024 - (su32(raw) & 1023)) & 1023);
    __shared__ uint64_t full[NS], empty[NS];
    __shared__ long long issued[NS];
    __shared__ __align__(128) float meta[NS][352];
    __shared__ uint64_t mfull[NS];
    const int mode = g_mode;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(NP * 32));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mfull[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int nmine = (NGROUPS - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int hold = g_hold;
    if (warp < NS) {  // consumer of stage `warp`
        float acc = 0;
        unsigned long long lat = 0, cnt = 0;
        for (int g = warp; g < nmine; g += NS) {
            const int s = warp;
            mbar_wait(&full[s], (g / NS) & 1);
            const long long t = clock64();
            lat += t - issued[s];
            ++cnt;
            acc += *(float *)(base + s * 49152 + lane * 4);
            if (mode & 1) {  // tensor-core-like smem read volume: 112 KB per group
                const float4 *p = (const float4 *)(base + s * 49152);
                float4 a4 = make_float4(0, 0, 0, 0);
#pragma unroll 8
                for (int i = lane; i < 7168; i += 32) { const float4 v = p[i % 3072]; a4.x += v.x; a4.y += v.w; }
                acc += a4.x + a4.y;
            }
            if ((mode & 4) && lane == 0) {  // bulk store of 272 B to a random vertex record
                const long long v = ((long long)(blockIdx.x + g * gridDim.x) * 2654435761ll) % 1000000;
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g_store_dst + v * 132), "r"(su32(&meta[s][0])), "r"(272) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            while (clock64() - t < hold) { }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        }
        if (lane == 0) { atomicAdd(&g_lat, lat); atomicAdd(&g_cnt, cnt); }
        if (acc == 12345.f) out[0] = acc;
    } else if (warp < NS + NP) {
        const int pi = warp - NS;
        const uint32_t lo = (uint32_t)((lane >> 3) * 12288), lx = lane & 7;
        for (int g = 0; g < nmine; ++g) {
            const int s = g % NS;
            mbar_wait(&empty[s], ((g / NS) & 1) ^ 1);
            if (mode & 2) {  // metadata bulk copy (1.3 KB) per group, waited on by every producer
                if (pi == 0 && lane == 0) {
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mfull[s])), "r"(1408) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(&meta[s][0])),
                                 "l"(g_meta_src + (int64_t)(blockIdx.x + g * gridDim.x) * 352), "r"(1408), "r"(su32(&mfull[s])) : "memory");
                }
                mbar_wait(&mfull[s], (g / NS) & 1);
            }
            if (pi == 0 && lane == 0) issued[s] = clock64();
            const int gg = blockIdx.x + g * gridDim.x;
            const uint32_t stg = su32(base + s * 49152);
            for (int r = pi; r < 96; r += NP) {
                const int id = ids[(int64_t)gg * 96 + r];
                const float *src = data + (int64_t)id * 128 + lane * 4;
                const uint32_t dst = stg + lo + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128) + ((lx ^ (uint32_t)(r & 7)) << 4);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(16));
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
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
    auto run = [&](const char *name, auto kern, int nthreads, int smem, int grid) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kern<<<grid, nthreads, smem>>>(d, did, out); cudaDeviceSynchronize();
        unsigned long long z = 0;
        cudaMemcpyToSymbol(g_lat, &z, 8); cudaMemcpyToSymbol(g_cnt, &z, 8);
        cudaEventRecord(e0);
        kern<<<grid, nthreads, smem>>>(d, did, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long lat, cnt; cudaMemcpyFromSymbol(&lat, g_lat, 8); cudaMemcpyFromSymbol(&cnt, g_cnt, 8);
        printf("%-44s %8.3f ms  %7.1f GB/s  mean issue->landed %6.0f cycles  %s\n", name, ms, NGROUPS * 96.0 * 512 / ms / 1e6,
               (double)lat / (cnt ? cnt : 1), cudaGetErrorString(cudaGetLastError()));
    };
    float *ms_, *st_;
    cudaMalloc(&ms_, (size_t)NGROUPS * 352 * 4); cudaMalloc(&st_, (size_t)1000000 * 132 * 4);
    cudaMemcpyToSymbol(g_meta_src, &ms_, 8); cudaMemcpyToSymbol(g_store_dst, &st_, 8);
    for (int mode : {0, 1, 2, 4, 7}) {
        for (int hold : {0, 4000}) {
            cudaMemcpyToSymbol(g_hold, &hold, 4);
            cudaMemcpyToSymbol(g_mode, &mode, 4);
            char nm[80];
            snprintf(nm, 80, "NS=4 NP=9 mode %d hold %d", mode, hold);
            run(nm, k_pipe<4, 9>, 13 * 32, 4 * 49152 + 2048, sms);
        }
    }
    return 0;
}
