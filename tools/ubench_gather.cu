// Random-row gather bandwidth on B200 (the pair phase's memory access pattern):
// rows of 512 B (128 fp32) at random ids.  Variants: LDG.128 to registers, cp.async 16 B to
// shared memory (per-warp row copies), with varying CTAs/threads.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__global__ void gather_ldg(const float4 *__restrict__ data, const int *__restrict__ ids, int nrows, float *out) {
    // warp per row: lane = 16-byte chunk
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * blockDim.x / 32;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) / 32; r < nrows; r += warps) {
        const float4 v = __ldg(&data[(int64_t)ids[r] * 32 + lane]);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (acc.x == 12345.f) out[0] = acc.y + acc.z + acc.w;
}

template <int ROWS_PER_WARP>
__global__ void gather_cpasync(const float4 *__restrict__ data, const int *__restrict__ ids, int nrows, float *out) {
    extern __shared__ float4 buf[];
    const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
    float4 *mybuf = buf + w * ROWS_PER_WARP * 32;
    const int warps = gridDim.x * blockDim.x / 32;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    for (int r0 = gw * ROWS_PER_WARP; r0 < nrows; r0 += warps * ROWS_PER_WARP) {
        for (int i = 0; i < ROWS_PER_WARP && r0 + i < nrows; ++i) {
            const float4 *src = &data[(int64_t)ids[r0 + i] * 32 + lane];
            unsigned s = (unsigned)__cvta_generic_to_shared(&mybuf[i * 32 + lane]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 0;\n" ::);
    }
    if (mybuf[lane].x == 12345.f) out[0] = 1;
}

int main() {
    const int64_t N = 1000000;
    const int nrows = 20000000;  // 20M rows = 10.24 GB (a C2 round's gather)
    std::vector<float> h(N * 128);
    for (auto &x : h) x = 1.0f;
    std::vector<int> hid(nrows);
    std::mt19937 rng(1);
    for (auto &x : hid) x = rng() % N;
    float4 *d; int *did; float *out;
    cudaMalloc(&d, N * 512); cudaMalloc(&did, nrows * 4); cudaMalloc(&out, 4);
    cudaMemcpy(d, h.data(), N * 512, cudaMemcpyHostToDevice);
    cudaMemcpy(did, hid.data(), nrows * 4, cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char *name, auto launch) {
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
        printf("%-40s %8.3f ms  %7.1f GB/s  err=%s\n", name, ms, nrows * 512.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    for (int tpb : {128, 256, 512, 1024}) for (int per : {4, 8, 16}) {
        char nm[64]; snprintf(nm, 64, "ldg  tpb=%d ctas/sm=%d", tpb, per);
        run(nm, [&] { gather_ldg<<<sms * per, tpb>>>(d, did, nrows, out); });
    }
    for (int tpb : {32, 64, 128, 256}) for (int per : {1, 2, 4, 8}) {
        const int smem = tpb / 32 * 8 * 512;
        if (smem * per > 200 * 1024) continue;
        cudaFuncSetAttribute(gather_cpasync<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        char nm[64]; snprintf(nm, 64, "cpasync8 tpb=%d ctas/sm=%d", tpb, per);
        run(nm, [&] { gather_cpasync<8><<<sms * per, tpb, smem>>>(d, did, nrows, out); });
    }
    for (int tpb : {32, 128}) for (int per : {1, 2}) {
        const int smem = tpb / 32 * 96 * 512;
        if (smem * per > 200 * 1024) continue;
        cudaFuncSetAttribute(gather_cpasync<96>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        char nm[64]; snprintf(nm, 64, "cpasync96 tpb=%d ctas/sm=%d", tpb, per);
        run(nm, [&] { gather_cpasync<96><<<sms * per, tpb, smem>>>(d, did, nrows, out); });
    }
    // sequential copy for reference
    run("memcpy d2d 5 GB", [&] { static float *x = nullptr; if (!x) cudaMalloc(&x, 5120000000ll / 2); cudaMemcpyAsync(x, d, N * 512 / 2, cudaMemcpyDeviceToDevice); });
    return 0;
}
