// Per-warp random-row gather throughput on B200 (512 B rows): how many producer warps per SM
// does each mechanism need?  cp.async (LDGSTS) pipelined, LDG.128 to registers, TMA tensor
// 1-row boxes (128 B) with 128B swizzle, and 1-D bulk copies (cp.async.bulk, 512 B).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

constexpr int NROWS = 8000000;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// each producer warp streams rows r = w, w+W, ... into a 16-row smem ring, keeping DEPTH batches in flight
template <int DEPTH>
__global__ void k_cpasync(const float4 *__restrict__ data, const int *__restrict__ ids, float *out) {
    extern __shared__ float4 buf[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    float4 *ring = buf + w * 16 * 32;
    const int gw = blockIdx.x * nw + w, W = gridDim.x * nw;
    int b = 0;
    for (int r0 = gw * 4; r0 < NROWS; r0 += W * 4, ++b) {
        for (int i = 0; i < 4; ++i) {
            const float4 *src = &data[(int64_t)ids[r0 + i] * 32 + lane];
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(&ring[((b * 4 + i) & 15) * 32 + lane])), "l"(src));
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(DEPTH));
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    if (ring[lane].x == 12345.f) out[0] = 1;
}

template <int U>
__global__ void k_ldg(const float4 *__restrict__ data, const int *__restrict__ ids, float *out) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int gw = blockIdx.x * nw + w, W = gridDim.x * nw;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int r0 = gw * U; r0 < NROWS; r0 += W * U) {
        float4 v[U];
#pragma unroll
        for (int i = 0; i < U; ++i) v[i] = __ldg(&data[(int64_t)ids[r0 + i] * 32 + lane]);
#pragma unroll
        for (int i = 0; i < U; ++i) { acc.x += v[i].x; acc.y += v[i].y; }
    }
    if (acc.x == 12345.f) out[0] = acc.y;
}

// one thread per CTA issues TMA 1-row boxes (4 per row: 4 k-blocks), ring of 32 rows, mbarrier per 8 rows
__global__ void k_tma(const __grid_constant__ CUtensorMap tmap, const int *__restrict__ ids, float *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
    __shared__ uint64_t bar[4];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        int it = 0;
        for (int r0 = blockIdx.x * 8; r0 < NROWS; r0 += gridDim.x * 8, ++it) {
            const int slot = it & 3;
            if (it >= 4) {  // wait for this slot's previous batch
                uint32_t done = 0, par = ((it >> 2) - 1) & 1;
                while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(su32(&bar[slot])), "r"(par));
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[slot])), "r"(8 * 512));
            for (int i = 0; i < 8; ++i) {
                const int row = slot * 8 + i;
                for (int kb = 0; kb < 4; ++kb) {
                    const uint32_t dst = su32(base + kb * 32 * 128 + (row >> 3) * 1024 + (row & 7) * 128);
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                                 ::"r"(dst), "l"((uint64_t)&tmap), "r"(kb * 32), "r"(ids[r0 + i]), "r"(su32(&bar[slot])) : "memory");
                }
            }
        }
        for (int s = 0; s < 4; ++s) {
            uint32_t done = 0;
            while (!done) asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(su32(&bar[s])), "r"(0));
            break;
        }
    }
    __syncthreads();
    if (base[threadIdx.x] == 123) out[0] = 1;
}

// one warp per CTA: each lane issues a 1-D bulk copy of one 512 B row
__global__ void k_bulk(const float *__restrict__ data, const int *__restrict__ ids, float *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar[4];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    if (lane == 0) {
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    int it = 0;
    for (int r0 = blockIdx.x * 32; r0 < NROWS; r0 += gridDim.x * 32, ++it) {
        const int slot = it & 3;
        if (it >= 4) {
            uint32_t done = 0, par = ((it >> 2) - 1) & 1;
            while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(su32(&bar[slot])), "r"(par));
        }
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[slot])), "r"(32 * 512));
        __syncwarp();
        const uint32_t dst = su32(sm + (slot * 32 + lane) * 512);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];"
                     ::"r"(dst), "l"(data + (int64_t)ids[r0 + lane] * 128), "r"(su32(&bar[slot])) : "memory");
    }
    if (sm[lane] == 123) out[0] = 1;
}

int main() {
    const int64_t N = 1000000;
    std::vector<float> h(N * 128, 1.0f);
    std::vector<int> hid(NROWS);
    std::mt19937 rng(1);
    for (auto &x : hid) x = rng() % N;
    float *d; int *did; float *out;
    cudaMalloc(&d, N * 512); cudaMalloc(&did, NROWS * 4); cudaMalloc(&out, 4);
    cudaMemcpy(d, h.data(), N * 512, cudaMemcpyHostToDevice);
    cudaMemcpy(did, hid.data(), NROWS * 4, cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char *name, auto launch) {
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
        printf("%-44s %8.3f ms  %7.1f GB/s  %s\n", name, ms, NROWS * 512.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    for (int nw : {1, 2, 4, 8, 16}) {
        char nm[80];
        cudaFuncSetAttribute(k_cpasync<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 16 * 512);
        cudaFuncSetAttribute(k_cpasync<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 16 * 512);
        snprintf(nm, 80, "cp.async depth3x4rows warps/SM=%d", nw);
        run(nm, [&] { k_cpasync<2><<<sms, 32 * nw, nw * 16 * 512>>>((float4 *)d, did, out); });
        snprintf(nm, 80, "cp.async depth7x4rows warps/SM=%d", nw);
        run(nm, [&] { k_cpasync<6><<<sms, 32 * nw, nw * 16 * 512>>>((float4 *)d, did, out); });
        snprintf(nm, 80, "ldg unroll8 warps/SM=%d", nw);
        run(nm, [&] { k_ldg<8><<<sms, 32 * nw>>>((float4 *)d, did, out); });
        snprintf(nm, 80, "ldg unroll16 warps/SM=%d", nw);
        run(nm, [&] { k_ldg<16><<<sms, 32 * nw>>>((float4 *)d, did, out); });
    }
    PFN_cuTensorMapEncodeTiled_v12000 encode; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, (cuuint64_t)N}; cuuint64_t str[1] = {512}; cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    for (int per : {1, 2, 4}) {
        cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 128 * 4 + 2048);
        char nm[80]; snprintf(nm, 80, "tma 1-row boxes, 1 thread/CTA, CTAs/SM=%d", per);
        run(nm, [&] { k_tma<<<sms * per, 32, 4 * 32 * 128 * 4 + 2048>>>(tm, did, out); });
        cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 512);
        snprintf(nm, 80, "bulk 512B 1 warp/CTA, CTAs/SM=%d", per);
        run(nm, [&] { k_bulk<<<sms * per, 32, 4 * 32 * 512>>>(d, did, out); });
    }
    return 0;
}
