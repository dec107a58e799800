// tc_pairs.cuh -- tensor-core pre-screen of the pair phase for D <= 128 (included by
// propagate.cu inside namespace grnnd, after cp_async16 / cp_async4 / the mask helpers).
//
// Per group of up to 128 pool rows (one pool of k <= 128, or 128/SZ pools of k <= SZ
// packed block-diagonally) the Gram matrix G = R R^T is one chain of 16
// tcgen05.mma.kind::tf32 (M = 128, K = 8 each) from the rows staged in shared memory
// (K-major, 128-byte swizzle, gathered by cp.async) into a TMEM accumulator.  The
// epilogue reads G back (tcgen05.ld, one thread per row), forms d~ = |a|^2 + |b|^2 - 2 G
// and settles every pair whose d~ is outside a rigorous error band around the redirect
// threshold hi = max(dv_a, dv_b); the rest (~1-3%) are re-evaluated with the reference's
// exact sequential fp32 arithmetic on the CUDA cores, so every redirect decision and
// every emitted distance is bit-identical to the reference.
//
// Error band: TF32 keeps 10 explicit mantissa bits (|a - tf32(a)| <= 2^-10 |a|), products
// of two TF32 values are exact in fp32 and accumulation is fp32, so
// |G~ - a.b| <= (2^-9 + O(K 2^-23)) sum |a_i b_i| <= 2^-10 (|a|^2 + |b|^2) (+ small); the band
// uses eps_tc = 2^-7, a 4x margin over the input-rounding term that also absorbs the
// accumulation order / alignment of the tensor-core adder.
//
// Pipeline (persistent CTA, 128 threads = 4 warps, thread i <-> group row i <-> TMEM
// lane i): rows of group j+2 and metadata of group j+3 are in flight (cp.async) while the
// tensor core computes group j and the CUDA cores run the epilogue of group j-1; three
// row stages of 64 KB, two TMEM accumulators of 128 columns.
#pragma once

namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (true) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) break;
#ifdef GRNND_MBAR_BACKOFF
        __nanosleep(GRNND_MBAR_BACKOFF);
#endif
    }
}
__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t ncols) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// 32 consecutive TMEM columns of this warp's 32 lanes: r[c] = column col + c of lane (32 w + lane)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 consecutive TMEM columns of this warp's 32 lanes, without the wait (tmem_wait_ld)
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t *r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 16 consecutive TMEM columns of this warp's 32 lanes
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// K-major, 128-byte-swizzle shared-memory matrix descriptor (sm_100 UMMA layout):
// start >> 4 in [0,14), LBO = 16 B (unused when swizzled), SBO = 1024 B between 8-row
// groups, version 1, layout type 2 = SWIZZLE_128B
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
// byte offset of float4 chunk c (dims 4c..4c+3) of row r in a 128-row stage: four 16 KB
// k-blocks of 32 dims, 8-row x 128 B swizzle atoms (chunk index XOR row % 8)
__device__ __forceinline__ uint32_t stage_off(int r, int c) {
    return (uint32_t)((c >> 3) * 16384 + (r >> 3) * 1024 + (r & 7) * 128 + (((c & 7) ^ (r & 7)) << 4));
}

}  // namespace tc

constexpr int TC_STAGE_BYTES = 128 * 512;  // 128 rows x 128 fp32
constexpr int TC_NSTAGE = 3;
constexpr int TC_TMEM_COLS = 256;          // two 128-column accumulators
constexpr int TC_THREADS = 256;            // 8 warps: warp w reads TMEM lanes 32 (w % 4).., column half w / 4
// Filter band coefficient on |a|^2 + |b|^2 (see the header comment): 2^-8 = 2x the
// worst-case TF32 input rounding of d~ = |a|^2 + |b|^2 - 2 G (truncation: 2^-9), plus 8u
// for the rounding of the rearranged test below.
constexpr float TC_EPS = 0.00390625f + 4.8e-7f;

template <int SZ>
struct TcSmem {
    static constexpr int GP = 128 / SZ;  // pools per group
    static constexpr int NM = 4;         // metadata slots
    static constexpr int CL = 64;  // redirect-capable pairs handed to decide (<= PAIR_LIST, workspace.cuh)
    static constexpr int QC = 1024;      // filter candidates per group (overflow: exact sweep)
    int32_t ids[NM][128];
    float dv[NM][128];
    uint8_t pos[NM][128];
    int32_t k[NM][GP];
    int32_t v[NM][GP];
    float nrm[TC_NSTAGE][128];
    // per-row filter terms of the group computed at (a): A = |r|^2 (1 - eps_tc),
    // B = dv (1 + eps_h) + tiny (B = -1: not a live pool row)
    float2 ab[2][128];
    uint64_t cond[128][2];  // row = p * SZ + anchor position; bit = partner position
    uint64_t afar[128][2];
    uint32_t cl_key[GP][CL];
    float cl_d[GP][CL];
    int cl_n[2][GP];
    int qn[2];
    int big[2];             // a live row's norm is too large for the rearranged test
    uint32_t q[QC];         // (row i << 8) | row j, group rows
    uint64_t mbar[2];
    uint32_t tmem_base;
};

template <int SZ>
__global__ void __launch_bounds__(TC_THREADS, 1) tc_pairs_kernel(PropArgs a, int bin) {
    using S = TcSmem<SZ>;
    constexpr int GP = S::GP;
    constexpr int NT = TC_THREADS;
    extern __shared__ __align__(1024) unsigned char tc_raw[];
    unsigned char *base = tc_raw + ((1024 - (tc::smem_u32(tc_raw) & 1023)) & 1023);
    S &sm = *reinterpret_cast<S *>(base + TC_NSTAGE * TC_STAGE_BYTES);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nbin = (int64_t)a.w.ctr[C_BIN0 + bin];
    const int64_t ngroups = (nbin + GP - 1) / GP;
    const int64_t G = gridDim.x;
    if ((int64_t)blockIdx.x >= ngroups) return;
    const int64_t nmine = (ngroups - blockIdx.x + G - 1) / G;
    const int2 *blist = a.w.bins + (int64_t)bin * a.w.n;
    const int nq = (a.dim + 3) >> 2;  // float4 chunks per row (<= 32)
    const int cap = a.cap, pcap = a.w.pcap, mw = a.w.mw;
    const float eps_h = a.eps_h + 4.8e-7f;
    unsigned long long pairs_local = 0, cand_local = 0, ovf_local = 0, red_local = 0;

    // ---- setup: TMEM, barriers, masks ----
    if (warp == 0) tc::tmem_alloc(&sm.tmem_base, TC_TMEM_COLS);
    if (tid == 0) {
        tc::mbar_init(&sm.mbar[0], 1);
        tc::mbar_init(&sm.mbar[1], 1);
        tc::fence_mbar_init();
    }
    for (int i = tid; i < 128 * 2; i += NT) {
        (&sm.cond[0][0])[i] = 0ull;
        (&sm.afar[0][0])[i] = 0ull;
    }
    if (tid < 2) sm.qn[tid] = 0;
    if (tid < 2 * GP) (&sm.cl_n[0][0])[tid] = 0;
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = sm.tmem_base;

    // thread t < 128 owns group row t = pool t / SZ, slot t % SZ
    const int my_p = (tid & 127) / SZ, my_s = (tid & 127) - my_p * SZ;
    auto load_vk = [&](int64_t j) -> int2 {  // (vertex row, k) of this thread's pool in group j
        int2 r = make_int2(-1, 0);
        if (tid < 128 && j < nmine) {
            const int64_t e = (blockIdx.x + j * G) * GP + my_p;
            if (e < nbin) r = blist[e];
        }
        return r;
    };
    auto issue_meta = [&](int64_t j, int2 vk) {
        const int sl = (int)(j & 3);
        if (tid < 128) {
            if (my_s == 0) {
                sm.v[sl][my_p] = vk.x;
                sm.k[sl][my_p] = vk.y;
            }
            if (my_s < vk.y) {
                const int64_t off = (int64_t)vk.x * cap + my_s;
                cp_async4(&sm.ids[sl][tid], a.read_ids + off, true);
                cp_async4(&sm.dv[sl][tid], a.read_dists + off, true);
                if ((my_s & 3) == 0) cp_async4(&sm.pos[sl][tid], a.w.pos8 + (int64_t)vk.x * pcap + my_s, true);
            }
        }
    };
    // rows of group j: warp w stages group rows w, w+8, ..; lane = 16-byte chunk (a whole
    // 512 B row per warp instruction, swizzled into the K-major SW128 layout)
    auto issue_rows = [&](int64_t j) {
        const int sl = (int)(j & 3), st = (int)(j % TC_NSTAGE);
        const uint32_t stg = tc::smem_u32(base + st * TC_STAGE_BYTES);
        const bool cv = lane < nq;
        const uint32_t lo = (uint32_t)((lane >> 3) * 16384), lx = (uint32_t)(lane & 7);
#pragma unroll 4
        for (int r = warp; r < 128; r += NT / 32) {
            const int p = r / SZ;
            if (r - p * SZ >= sm.k[sl][p]) continue;  // warp-uniform
            const int32_t id = sm.ids[sl][r];
            const float *src = a.data + (int64_t)(id < 0 ? 0 : id) * a.ld + (cv ? lane * 4 : 0);
            const uint32_t dst = stg + lo + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128) + ((lx ^ (uint32_t)(r & 7)) << 4);
            const int sz = (id >= 0 && cv) ? 16 : 0;  // dims >= D: zero
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
        }
        if (tid < 128 && my_s < sm.k[sl][my_p]) {
            const int32_t id = sm.ids[sl][tid];
            cp_async4(&sm.nrm[st][tid], a.norms + (id < 0 ? 0 : id), id >= 0);
        }
    };
    // exact sequential distance (the reference's _sqdist) of group rows i, j of a stage
    auto exact_rows = [&](const unsigned char *stg, int i, int j) -> float {
        float s = 0.0f;
#pragma unroll 4
        for (int c = 0; c < nq; ++c) {
            const float4 x = *reinterpret_cast<const float4 *>(stg + tc::stage_off(i, c));
            const float4 y = *reinterpret_cast<const float4 *>(stg + tc::stage_off(j, c));
            s = exact_step4(s, x, y);
        }
        return s;
    };
    // two independent exact distances in lockstep (their dependent add chains interleave)
    auto exact_rows2 = [&](const unsigned char *stg, int i1, int j1, int i2, int j2, float &d1, float &d2) {
        float s1 = 0.0f, s2 = 0.0f;
#pragma unroll 4
        for (int c = 0; c < nq; ++c) {
            const float4 x1 = *reinterpret_cast<const float4 *>(stg + tc::stage_off(i1, c));
            const float4 y1 = *reinterpret_cast<const float4 *>(stg + tc::stage_off(j1, c));
            const float4 x2 = *reinterpret_cast<const float4 *>(stg + tc::stage_off(i2, c));
            const float4 y2 = *reinterpret_cast<const float4 *>(stg + tc::stage_off(j2, c));
            s1 = exact_step4(s1, x1, y1);
            s2 = exact_step4(s2, x2, y2);
        }
        d1 = s1;
        d2 = s2;
    };
    auto record = [&](int ms, int qs, int i, int j, float d) {  // pair of group rows i < j, same pool
        const int p = i / SZ;
        const int x1 = sm.pos[ms][i], x2 = sm.pos[ms][j];
        const float d1 = sm.dv[ms][i], d2 = sm.dv[ms][j];
        const int xa = x1 < x2 ? x1 : x2, xb = x1 < x2 ? x2 : x1;
        const float dva = x1 < x2 ? d1 : d2, dvb = x1 < x2 ? d2 : d1;
        const unsigned long long bit = 1ull << (xb & 63);
        const bool far = !(dvb >= dva);
        atomicOr((unsigned long long *)&sm.cond[p * SZ + xa][xb >> 6], bit);
        if (far) atomicOr((unsigned long long *)&sm.afar[p * SZ + xa][xb >> 6], bit);
        const int c = atomicAdd(&sm.cl_n[qs][p], 1);
        if (c < S::CL) {
            sm.cl_key[p][c] = (uint32_t)((far ? 1u << 16 : 0u) | (xa << 8) | xb);
            sm.cl_d[p][c] = d;
        }
    };

    auto epilogue = [&](int64_t g) {
        const int ms = (int)(g & 3), st = (int)(g % TC_NSTAGE), acc = (int)(g & 1), qs = (int)(g & 1);
        const unsigned char *stg = base + st * TC_STAGE_BYTES;
        tc::mbar_wait(&sm.mbar[acc], (uint32_t)((g >> 1) & 1));
        tc::fence_after();
        // ---- filter: warp (rb, h) = TMEM lanes 32 rb.., its pools' column half h ----
        const int rb = warp & 3, h = warp >> 2;
        const int i = rb * 32 + lane;  // group row
        const float2 abi = sm.ab[qs][i];
        const bool big = sm.big[qs] != 0;
        unsigned np = 0;
        auto scan = [&](const uint32_t *r, int cb, int nc) {
            uint32_t cm = 0u;  // candidate columns (branch free: the 32 columns interleave)
#pragma unroll
            for (int c = 0; c < nc; ++c) {
                const int jr = cb + c;
                const float2 abj = sm.ab[qs][jr];
                // same pool, upper triangle, both live (B >= 0 marks a live row)
                const bool valid = jr > i && (jr / SZ) == (i / SZ) && abi.y >= 0.0f && abj.y >= 0.0f;
                np += valid ? 1u : 0u;
                // settled iff (|a|^2+|b|^2)(1-eps) - 2G >= max(dv)(1+eps_h) + tiny, which implies
                // d~ >= hi + E with E the band of the header comment
                const float lhs = fmaf(-2.0f, __uint_as_float(r[c]), abi.x + abj.x);
                const float rhs = abi.y >= abj.y ? abi.y : abj.y;
                cm |= (valid && (big || !(lhs >= rhs))) ? (1u << c) : 0u;
#ifdef GRNND_TC_VALIDATE
                // bound check (validation builds): |d~ - d_exact| <= eps_tc (|a|^2 + |b|^2)
                if (valid && a.stats) {
                    const float nn = sm.nrm[st][i] + sm.nrm[st][jr];
                    const float dx = exact_rows(stg, i, jr);
                    const float err = fabsf(fmaf(-2.0f, __uint_as_float(r[c]), nn) - dx);
                    const float ratio = err / fmaf(TC_EPS, nn, 1e-30f);
                    atomicMax((int *)&a.stats[GRNND_ST_TCV_MAX_RATIO], __float_as_int(ratio));  // ratio >= 0: int order = float order
                    if (ratio > 1.0f) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_TCV_VIOLATIONS], 1ull);
                    atomicAdd((unsigned long long *)&a.stats[GRNND_ST_TCV_CHECKED], 1ull);
                }
#endif
            }
            if (__any_sync(FULL, cm != 0u)) {
                const int n = __popc(cm);
                int qi = n ? atomicAdd(&sm.qn[qs], n) : 0;
                while (cm) {
                    const int c = __ffs(cm) - 1;
                    cm &= cm - 1u;
                    if (qi < S::QC) sm.q[qi] = (uint32_t)((i << 8) | (cb + c));
                    ++qi;
                }
            }
        };
        const uint32_t trow = tmem + ((uint32_t)(rb * 32) << 16) + (uint32_t)(acc * 128);
        if (SZ <= 32) {
            // 16 columns: SZ = 32: this warp's pool rb, half h; SZ = 16: pool 2 rb + h
            const int cb = rb * 32 + h * 16;
            uint32_t r[16];
            tc::tmem_ld16(trow + (uint32_t)cb, r);
            scan(r, cb, 16);
        } else {
            // SZ = 64: pool rb / 2, columns [64 (rb/2) + 32 h, +32); SZ = 128: [64 h, +64)
            const int cb0 = SZ == 64 ? (rb >> 1) * 64 + h * 32 : h * 64;
            constexpr int NCH = SZ == 64 ? 1 : 2;
            const int kcols = SZ == 64 ? 128 : sm.k[ms][0];
#pragma unroll 1
            for (int ch = 0; ch < NCH; ++ch) {
                const int cb = cb0 + ch * 32;
                if (cb >= kcols) break;  // warp-uniform
                uint32_t r[32];
                tc::tmem_ld32(trow + (uint32_t)cb, r);
                scan(r, cb, 32);
            }
        }
        pairs_local += np;
        tc::fence_before();
        __syncthreads();  // candidate queue complete; TMEM reads done
        // ---- exact re-evaluation of the candidates (CUDA cores, reference arithmetic) ----
        const int qn = sm.qn[qs];
        if (tid == 0) {
            cand_local += (unsigned long long)qn;
            ovf_local += qn > S::QC ? 1ull : 0ull;
        }
        if (qn <= S::QC) {
            for (int e = tid; e < qn; e += 2 * NT) {
                const bool two = e + NT < qn;
                const uint32_t k1 = sm.q[e], k2 = two ? sm.q[e + NT] : k1;
                const int i1 = (int)(k1 >> 8), j1 = (int)(k1 & 255u), i2 = (int)(k2 >> 8), j2 = (int)(k2 & 255u);
                float x1, x2;
                exact_rows2(stg, i1, j1, i2, j2, x1, x2);
                const float a1 = sm.dv[ms][i1], b1 = sm.dv[ms][j1];
                if (x1 < (a1 >= b1 ? a1 : b1)) record(ms, qs, i1, j1, x1);
                const float a2 = sm.dv[ms][i2], b2 = sm.dv[ms][j2];
                if (two && x2 < (a2 >= b2 ? a2 : b2)) record(ms, qs, i2, j2, x2);
            }
        } else {
            // queue overflow (degenerate data: many near-ties): exact sweep of every pair
#pragma unroll
            for (int pp = 0; pp < GP; ++pp) {
                const int k = sm.k[ms][pp];
                const int npairs = k * (k - 1) / 2;
                for (int t = tid; t < npairs; t += NT) {
                    int s1, u1;
                    tile_decode(t, s1, u1);
                    u1 += 1;
                    const int ii = pp * SZ + s1, jj = pp * SZ + u1;
                    if (sm.ids[ms][ii] == TOMB || sm.ids[ms][jj] == TOMB) continue;
                    const float d = exact_rows(stg, ii, jj);
                    const float d1 = sm.dv[ms][ii], d2 = sm.dv[ms][jj];
                    if (d < (d1 >= d2 ? d1 : d2)) record(ms, qs, ii, jj, d);
                }
            }
        }
        __syncthreads();  // masks + kept distances complete
        // ---- kept pairs -> global (decide_kernel); masks only for incomplete lists; re-zero ----
        for (int e = tid; e < 128 * mw; e += NT) {
            const int r = mw == 2 ? e >> 1 : e, wd = mw == 2 ? e & 1 : 0;  // group row = p * SZ + anchor pos
            const int pp = r / SZ, x = r - pp * SZ;
            const int64_t v = sm.v[ms][pp];
            if (v < 0 || x >= sm.k[ms][pp] - 1) continue;
            uint64_t cv = 0ull, fv = 0ull;
            if (wd < 2) {
                cv = sm.cond[r][wd];
                fv = sm.afar[r][wd];
                sm.cond[r][wd] = 0ull;
                sm.afar[r][wd] = 0ull;
            }
            if (sm.cl_n[qs][pp] > S::CL) {
                a.w.cond[(v * cap + x) * mw + wd] = cv;
                a.w.afar[(v * cap + x) * mw + wd] = fv;
            }
        }
        for (int e = tid; e < GP * S::CL; e += NT) {
            const int pp = e / S::CL, c = e - pp * S::CL;
            const int64_t v = sm.v[ms][pp];
            if (v < 0) continue;
            const int ncl = sm.cl_n[qs][pp];
            const int nw = ncl < S::CL ? ncl : S::CL;
            int32_t *rec = a.w.clrec + v * (int64_t)CLREC;
            if (c == 0) {
                if (ncl > 0) a.w.clcnt[v] = nw | (ncl > S::CL ? CL_TRUNC : 0);
                red_local += (unsigned long long)ncl;
            }
            if (c < nw) {
                rec[4 + 2 * c] = (int32_t)sm.cl_key[pp][c];
                rec[5 + 2 * c] = __float_as_int(sm.cl_d[pp][c]);
            }
        }
    };

    // ---- prologue ----
    issue_meta(0, load_vk(0));
    cp_async_commit();
    issue_meta(1, load_vk(1));
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    issue_rows(0);
    cp_async_commit();
    issue_meta(2, load_vk(2));
    cp_async_commit();
    if (nmine > 1) issue_rows(1);
    cp_async_commit();
    int2 vkr = load_vk(3);

    for (int64_t j = 0; j < nmine; ++j) {
        const int ms = (int)(j & 3), st = (int)(j % TC_NSTAGE), qs = (int)(j & 1);
        // (a) rows of j and metadata of j+2 landed (rows of j+1 may still be in flight)
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        tc::fence_proxy_async();  // cp.async writes -> visible to the tensor core (async proxy)
        if (tid == 0) sm.big[qs] = 0;
        __syncthreads();
        // (b) one thread issues the Gram of group j into accumulator j & 1
        if (tid == 0) {
            // counters of group j (epilogue at iteration j+1); last used by group j-2
            sm.qn[qs] = 0;
#pragma unroll
            for (int p = 0; p < GP; ++p) sm.cl_n[qs][p] = 0;
            tc::fence_after();
            const int n = GP == 1 ? ((sm.k[ms][0] + 15) / 16 * 16) : 128;
            const uint32_t idesc = tc::idesc_tf32(n < 16 ? 16 : n);
            const uint32_t sa = tc::smem_u32(base + st * TC_STAGE_BYTES);
            const uint32_t d = tmem + (uint32_t)(qs * 128);
#pragma unroll
            for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t desc = tc::sw128_desc(sa + kb * 16384 + kk * 32);
                    tc::mma_tf32(d, desc, desc, idesc, (kb | kk) != 0);
                }
            tc::mma_commit(&sm.mbar[qs]);
        }
        // per-row filter terms of group j (read by its epilogue at iteration j+1)
        if (tid < 128) {
            const int p = tid / SZ, s = tid - p * SZ;
            const bool live = s < sm.k[ms][p] && sm.ids[ms][tid] != TOMB;
            const float nr = sm.nrm[st][tid];
            sm.ab[qs][tid] = live ? make_float2(nr * (1.0f - TC_EPS), fmaf(sm.dv[ms][tid], 1.0f + eps_h, 1e-30f))
                                  : make_float2(0.0f, -1.0f);
            if (live && !(nr <= 1.0e37f)) sm.big[qs] = 1;  // rearranged test could overflow
        }
        // (c) epilogue of group j-1 overlaps the tensor core working on group j
        if (j >= 1) epilogue(j - 1);
        // (d) refill: metadata of j+3 (its slot held group j-1), rows of j+2 (stage of j-1)
        if (j + 3 < nmine) issue_meta(j + 3, vkr);
        cp_async_commit();
        if (j + 2 < nmine) issue_rows(j + 2);
        cp_async_commit();
        vkr = load_vk(j + 4);
    }
    __syncthreads();
    epilogue(nmine - 1);
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, TC_TMEM_COLS);
    if (a.stats) {
        pairs_local = warp_sum(pairs_local);
        if (lane == 0 && pairs_local) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_PAIRS], pairs_local);
        if (tid == 0 && cand_local) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_CANDIDATES], cand_local);
        if (tid == 0 && ovf_local) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_OVERFLOWS], ovf_local);
        red_local = warp_sum(red_local);
        if (lane == 0 && red_local) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_REDIRECTABLE], red_local);
    }
}
