// common.cuh -- shared device helpers for the sm_100a GRNND kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "grnnd_b200.h"

namespace grnnd {

constexpr int32_t TOMB = -1;
constexpr uint64_t STREAM_INIT = 0ull;       // rng.py:16
constexpr uint64_t ATTEMPT_STRIDE = 1ull << 22;  // rng.py:20
constexpr int WARP = 32;
constexpr unsigned FULL = 0xffffffffu;

// ---- counter-based RNG: splitmix64 finalizer, rng.py:25-41 / _numba_kernels.py:28-41 ----
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
// hash4 = mix(mix(mix(mix(seed) ^ stream) ^ v) ^ i); the first three mixes depend only on
// (seed, stream, v) so kernels hoist them: hash4 = mix64(vertex_prefix(seed,stream,v) ^ i).
__host__ __device__ __forceinline__ uint64_t vertex_prefix(uint64_t seed, uint64_t stream,
                                                           uint64_t v) {
    return mix64(mix64(mix64(seed) ^ stream) ^ v);
}
__host__ __device__ __forceinline__ uint64_t hash4(uint64_t seed, uint64_t stream, uint64_t v,
                                                   uint64_t i) {
    return mix64(vertex_prefix(seed, stream, v) ^ i);
}

// ---- exact squared L2: _numba_kernels.py:50-56 --------------------------------------
// s += (a-b)*(a-b) strictly in index order, each op rounded to nearest (no FMA):
// __fsub_rn/__fmul_rn/__fadd_rn are never contracted by nvcc/ptxas.
__device__ __forceinline__ float exact_step(float s, float a, float b) {
    float d = __fsub_rn(a, b);
    return __fadd_rn(s, __fmul_rn(d, d));
}

// Four consecutive exact_steps (dims x, y, z, w in order).  The differences and squares go
// through the packed f32x2 pipes (FADD2 / FMUL2: each lane rounded like __fsub_rn / __fmul_rn;
// a - b == a + (-b) exactly in IEEE arithmetic); the running sum stays scalar and sequential,
// so nothing can be contracted into an FMA and the bits equal four exact_steps.
__device__ __forceinline__ float2 sq2(float a0, float a1, float b0, float b1) {
    const float2 d = __fadd2_rn(make_float2(a0, a1), make_float2(-b0, -b1));
    return __fmul2_rn(d, d);
}
__device__ __forceinline__ float exact_step4(float s, const float4 &a, const float4 &b) {
    const float2 p0 = sq2(a.x, a.y, b.x, b.y), p1 = sq2(a.z, a.w, b.z, b.w);
    s = __fadd_rn(s, p0.x);
    s = __fadd_rn(s, p0.y);
    s = __fadd_rn(s, p1.x);
    return __fadd_rn(s, p1.y);
}
// the four squared differences alone (exact_step(0, a, b) == (a - b)^2: adding +0 is exact)
__device__ __forceinline__ float4 sq4(const float4 &a, const float4 &b) {
    const float2 p0 = sq2(a.x, a.y, b.x, b.y), p1 = sq2(a.z, a.w, b.z, b.w);
    return make_float4(p0.x, p0.y, p1.x, p1.y);
}

// Sequential exact distance between two global rows (used off the hot loop).
__device__ __forceinline__ float exact_sqdist_global(const float* __restrict__ a,
                                                     const float* __restrict__ b, int32_t dim) {
    float s = 0.0f;
    int32_t d = 0;
    if ((((uintptr_t)a | (uintptr_t)b) & 15) == 0) {
        for (; d + 4 <= dim; d += 4) {
            float4 x = __ldg(reinterpret_cast<const float4*>(a + d));
            float4 y = __ldg(reinterpret_cast<const float4*>(b + d));
            s = exact_step4(s, x, y);
        }
    }
    for (; d < dim; ++d) s = exact_step(s, __ldg(a + d), __ldg(b + d));
    return s;
}

// ceil(rho*k) with the reference's 1e-9 float guard (_numba_kernels.py:207-212)
__host__ __device__ __forceinline__ int32_t reverse_count(double rho, int32_t k) {
    double f = rho * (double)k;
    int64_t m = (int64_t)f;
    if (f - (double)m > 1e-9) m += 1;
    if (m > k) m = k;
    return (int32_t)m;
}

// (dist, id) lexicographic "less" used by reverse selection and finalize (builder.py:350)
__device__ __forceinline__ bool key_less(float da, int32_t ia, float db, int32_t ib) {
    return da < db || (da == db && ia < ib);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

}  // namespace grnnd

// ---- host-side error plumbing and per-device launch state (capi.cu) ----
namespace grnnd {
void set_error(const char* fmt, ...);
int check_launch(const char* what, int nkernels = 1);
unsigned long long launch_count();
int instrumentation();  // grnnd_set_instrumentation
constexpr int MAX_DEVICES = 64;
// SM count of the CUDA runtime's current device (cached per device)
int device_sm_count();
int current_device();
// Dynamic shared memory opt-in of one kernel, remembered per device: the attribute is set
// on the first launch on each device (and again if a launch needs more).
struct SmemOptIn {
    int bytes[MAX_DEVICES] = {0};
    template <class K>
    cudaError_t ensure(K kern, size_t smem) {
        const int d = current_device();
        if (d < 0 || d >= MAX_DEVICES) return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if ((int)smem <= bytes[d]) return cudaSuccess;
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) bytes[d] = (int)smem;
        return e;
    }
};
}  // namespace grnnd

#define GRNND_TRY(expr)                        \
    do {                                       \
        int _rc = (expr);                      \
        if (_rc != GRNND_OK) return _rc;       \
    } while (0)

#define GRNND_CUDA(expr)                                                              \
    do {                                                                              \
        cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess) {                                                      \
            ::grnnd::set_error("%s failed: %s", #expr, cudaGetErrorString(_e));        \
            return GRNND_ECUDA;                                                       \
        }                                                                             \
    } while (0)
