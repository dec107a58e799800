// tc3_pairs.cuh -- warp-specialised tensor-core pair phase for D <= 128, R <= 96 (the
// benchmark shape).  Included by propagate.cu inside namespace grnnd after tc_pairs.cuh.
//
// Same contract and filter as tc_pairs.cuh: the Gram of a group of pool rows on
// tcgen05.mma.kind::tf32, a rigorous error band around the redirect threshold, and the
// reference's exact sequential fp32 arithmetic for the pairs inside the band -- so every
// decision and emitted distance is bit-identical to the reference.  The schedule has no
// CTA-wide barrier per group and no dependent global load on its critical path:
//   * tc_stage_kernel (propagate.cu) lays every group's metadata out contiguously (pool
//     ids, stored distances, permutation positions, row norms, (vertex, k) header);
//   warp 0       metadata: one thread streams group g's metadata into meta slot g % 8 with
//                1-D bulk copies (TMA), completing on mfull[m];
//   warps 11-19  row producers: cp.async of the 96 vector rows into stage g % 4 (K-major,
//                128-byte swizzle); completion arrives on full[s] in hardware
//                (cp.async.mbarrier.arrive.noinc).  Random 512-byte row gathers need ~16
//                issuing warps per SM to approach HBM bandwidth (a warp's cp.async stream is
//                capped near 4-5 GB/s, TMA boxes near 1-3.6 TB/s chip-wide for this access
//                size: tools/ubench_gather*.cu);
//   warp 1       MMA: one thread fences the async proxy and issues the 16 MMAs of group g
//                into TMEM accumulator g % 2;
//   warps 4-6    filter (TMEM lanes 0..95): Gram -> band candidates -> queue g % 2; warps
//                20-22 (FSPLIT, default) scan the other half of the Gram's column blocks;
//   warps 2,3,7 / 8,9,10  two exact sets (even / odd groups): exact chains of the queue ->
//                redirect records -> global (bulk stores); release the stage and meta slot.
// Groups: 96 rows = one pool of k <= 96, or 96/SZ pools of k <= SZ (SZ = 8, 16, 24, 32, 48).
#pragma once

constexpr int T3_ROWS = 96;
constexpr int T3_KB = T3_ROWS * 128;  // one 32-dim k-block of a stage (12 KB)
constexpr int T3_STAGE = 4 * T3_KB;   // 96 rows x 128 fp32 (48 KB)
constexpr int T3_NS = 4;              // row stages
// SPLIT (data far from the origin): the Gram as hi*hi + hi*lo + lo*hi with hi = the row
// truncated to TF32 and lo = row - hi (both exact in fp32, converted per k-block into a
// 2-slot ring by the MMA warp); 3 row stages make room for the ring
constexpr int T3_NS_SPLIT = 3;
constexpr int T3_RING = 2 * 2 * T3_KB;  // 2 slots x (hi, lo) k-blocks
constexpr float TC_EPS_SPLIT = 3.0517578125e-05f;  // 2^-15 (~3x the split bound)
#ifndef GRNND_T3_NM
#define GRNND_T3_NM 6
#endif
#ifndef GRNND_T3_PAD
#define GRNND_T3_PAD 0
#endif
#ifndef GRNND_T3_WCOOP
#define GRNND_T3_WCOOP 8
#endif
constexpr int T3_WCOOP = GRNND_T3_WCOOP;  // queues up to this length: warp-cooperative chains (<= 32)
constexpr int T3_NM = GRNND_T3_NM;    // metadata slots
// the M = 128 MMA reads 32 rows (4 KB) past the last k-block of the last stage: with no pad
// those are bytes of T3Smem (> 4 KB), read into accumulator rows 96..127 that nothing uses
constexpr int T3_PAD = GRNND_T3_PAD;
#ifndef GRNND_T3_WARPS
#define GRNND_T3_WARPS 23
#endif
#ifndef GRNND_T3_EXACT1
#define GRNND_T3_EXACT1 1  // a thread with one queued pair runs one chain (not the pair twice)
#endif
#ifndef GRNND_T3_PREF
#define GRNND_T3_PREF 0  // 1: the filter issues two 32-column TMEM loads before scanning either
#endif
#ifndef GRNND_T3_FSPLIT
#define GRNND_T3_FSPLIT 1  // 1: warps 20..22 take half of the filter's Gram columns (23 warps)
#endif
// warp layout per pipeline: D <= 128 runs the split filter (23 warps); MULTI (D > 128) keeps
// one filter set and 20 warps (its register budget: measured 1.45 vs 1.53 s at C3)
template <bool MULTI>
struct T3Cfg {
    static constexpr int WARPS = MULTI ? 20 : GRNND_T3_WARPS;
    static constexpr int FSPLIT = MULTI ? 0 : GRNND_T3_FSPLIT;
    static constexpr int NT = 32 * WARPS;
    static constexpr int NP = WARPS - 11 - 3 * FSPLIT;  // row producers (warps 11..)
    static constexpr int NF = 96 * (1 + FSPLIT);         // filter threads
    static_assert(!FSPLIT || (11 + NP) % 4 == 0, "filter warps must map to TMEM lane quarters 0..2");
};

struct alignas(16) T3Meta {  // one group's metadata (staged by tc_stage_kernel, one bulk copy)
    int32_t ids[T3_ROWS];
    float dv[T3_ROWS];
    float nrm[T3_ROWS];
    uint8_t pos[T3_ROWS];
    int2 hdr[12];  // (vertex row, k) of pool p < GP
};
constexpr uint32_t T3_META_BYTES = 3 * 4 * T3_ROWS + T3_ROWS + 96;
static_assert(sizeof(T3Meta) == T3_META_BYTES && T3_META_BYTES == T3_META_REC, "metadata record layout");


template <int SZ, bool MULTI>
struct T3Smem {
    static constexpr int GP = T3_ROWS / SZ;
    // redirect-capable pairs handed to decide (workspace.cuh); a pool of k <= SZ has at most
    // SZ (SZ - 1) / 2 pairs, so small slots never truncate a list
    static constexpr int CL = PAIR_LIST < SZ * (SZ - 1) / 2 ? PAIR_LIST : SZ * (SZ - 1) / 2;
    static constexpr int RS = 4 + 2 * CL;  // record stride (int32), a multiple of 4
    // filter candidates per group in shared memory (overflow: an exact sweep; MULTI: the rest
    // spill to the CTA's global list, so a smaller queue leaves room for wider exact batches)
    static constexpr int QC = MULTI ? 256 : 512;
    static constexpr int CN = MULTI && SZ >= 32 ? 4 : 2;  // MULTI: pairs per warp-cooperative batch
    T3Meta meta[T3_NM];
    float2 ab[2][T3_ROWS];        // filter terms (A = -inf: always a candidate; B = -1: dead row)
    uint32_t livec[2][4];         // bit r: row r's B >= 0 (a column that can pair)
    uint64_t cond[2][T3_ROWS][2];  // per exact set: row = p * SZ + anchor position; bit = partner
    uint64_t afar[2][T3_ROWS][2];
    alignas(16) int32_t rec[2][GP][RS];  // per exact set, per pool: pair records (workspace.cuh layout)
    int cl_n[2][GP];
    int qn[2];
    uint32_t q[2][QC];            // (row i << 8) | row j
    // per exact warp: the squared differences of two pairs (MULTI: one 128-dim chunk; the
    // second pair's row starts 132 floats in, so the two summing lanes read distinct banks)
    static constexpr int PSQW = MULTI ? CN * 132 : 2 * 128;
    alignas(16) float psq[6 * PSQW];
    uint64_t mfull[T3_NM], mempty[T3_NM], full[T3_NS], empty[T3_NS], accf[2], acce[2], qrdy[2], qemp[2], rfree[2];
    uint32_t tmem_base;
};

namespace tc {
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// one arrival per warp, after every lane's prior shared-memory accesses (barrier counts = warps)
__device__ __forceinline__ void warp_arrive(uint64_t *bar) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
}  // namespace tc

__device__ __forceinline__ uint32_t t3_off(int r, int c) {
    return (uint32_t)((c >> 3) * T3_KB + (r >> 3) * 1024 + (r & 7) * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// TC bins 1..6 (slot sizes 8, 16, 24, 32, 48, 96): groups of bin b start at staging group
// tc_group_base(b) (all bins' groups back to back)
__host__ __device__ __forceinline__ int tc_bin_gp(int b) { return b == 1 ? 12 : b == 2 ? 6 : b == 3 ? 4 : b == 4 ? 3 : b == 5 ? 2 : 1; }
__host__ __device__ __forceinline__ int tc_bin_sz(int b) { return 96 / tc_bin_gp(b); }
constexpr int T3_NBINS = 6;  // TC bins 1..6: slot sizes 8, 16, 24, 32, 48, 96
__device__ __forceinline__ int64_t tc_group_base(const unsigned long long *ctr, int b) {
    int64_t base = 0;
    for (int x = 1; x < b; ++x) {
        const int gp = tc_bin_gp(x);
        base += ((int64_t)ctr[C_BIN0 + x] + gp - 1) / gp;
    }
    return base;
}

#ifdef GRNND_T3_PROF
__device__ unsigned long long g_t3prof[8][32];  // per TC bin
__device__ long long g_t3trace[64][10];  // CTA 0: per group event times (profiling builds)
#define T3P_BEGIN() const long long _t3p0 = clock64()
#define T3P_EV(g, ev) do { if (blockIdx.x == 0 && (g) < 64) g_t3trace[(g)][(ev)] = clock64(); } while (0)
#ifdef GRNND_T3_TRACE_ONLY  // events of CTA 0 only: no per-wait accounting (near-production timing)
#define T3P_ADD(slot, since)
#define T3P_WAIT(slot, stmt) stmt
#else
#define T3P_ADD(slot, since) atomicAdd(&t3p_sm[slot], (unsigned long long)(clock64() - (since)))  // per-CTA
#define T3P_WAIT(slot, stmt) do { const long long _w = clock64(); stmt; if (lane == 0) T3P_ADD(slot, _w); } while (0)
#endif
#else
#define T3P_BEGIN()
#define T3P_ADD(slot, since)
#define T3P_EV(g, ev)
#define T3P_WAIT(slot, stmt) stmt
#endif
#ifndef GRNND_T3_NOFILTER
#define GRNND_T3_NOFILTER 0  // timing experiment only (results invalid): the filter queues nothing
#endif

// MULTI (D > 128): each group's rows stream through the stage ring as ceil(D / 128) chunks of
// 128 dims; the MMA accumulates the chunks' Grams in the same TMEM accumulator and releases
// each stage with tcgen05.commit (the exact sets never hold a stage); the exact chains read
// the candidate pairs' rows from global memory (L2: the group's rows were just streamed).
template <int SZ, bool MULTI, bool SPLIT>
__global__ void __launch_bounds__(T3Cfg<MULTI>::NT, 1) tc3_pairs_kernel(PropArgs a, int bin) {
    using CF = T3Cfg<MULTI>;
    constexpr int T3_NT = CF::NT, T3_NP = CF::NP, T3_NF = CF::NF;
    using S = T3Smem<SZ, MULTI>;
    constexpr int GP = S::GP;
    constexpr int R = T3_ROWS;
    constexpr int NS = SPLIT ? T3_NS_SPLIT : T3_NS;
    constexpr float EPS_TC = SPLIT ? TC_EPS_SPLIT : TC_EPS;
    constexpr int NM = T3_NM;
    extern __shared__ __align__(1024) unsigned char t3_raw[];
    unsigned char *base = t3_raw + ((1024 - (tc::smem_u32(t3_raw) & 1023)) & 1023);
    unsigned char *ring = base + NS * T3_STAGE;  // SPLIT only
    S &sm = *reinterpret_cast<S *>(base + NS * T3_STAGE + (SPLIT ? T3_RING : 0) + T3_PAD);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef GRNND_T3_PROF
    __shared__ unsigned long long t3p_sm[32];
    if (tid < 32) t3p_sm[tid] = 0ull;
    __syncthreads();
#endif
    const int64_t nbin = (int64_t)a.w.ctr[C_BIN0 + bin];
    const int64_t ngroups = (nbin + GP - 1) / GP;
    const int64_t G = gridDim.x;
    if ((int64_t)blockIdx.x >= ngroups) return;
    const int64_t nmine = (ngroups - blockIdx.x + G - 1) / G;
    const int64_t gbase = tc_group_base(a.w.ctr, bin);
    const int nq = (a.dim + 3) >> 2;
    const int nch = MULTI ? (nq + 31) >> 5 : 1;  // 128-dim chunks per group
    const int cap = a.cap, mw = a.w.mw;
    unsigned long long st_pairs = 0, st_cand = 0, st_ovf = 0, st_red = 0;

    // ---- setup ----
    if (warp == 1) tc::tmem_alloc(&sm.tmem_base, TC_TMEM_COLS);
    if (tid == 0) {
        for (int m = 0; m < NM; ++m) {
            tc::mbar_init(&sm.mfull[m], 1);
            tc::mbar_init(&sm.mempty[m], 3);  // arrivals: one per warp
        }
        for (int s = 0; s < NS; ++s) {
#ifdef GRNND_T3_WAITGROUP
            tc::mbar_init(&sm.full[s], T3_NP);
#else
            tc::mbar_init(&sm.full[s], T3_NP * 32);
#endif
            tc::mbar_init(&sm.empty[s], MULTI ? 1 : 3);  // MULTI: the MMA's commit frees a stage
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&sm.rfree[b], 1);
            tc::mbar_init(&sm.accf[b], 1);
            tc::mbar_init(&sm.acce[b], T3_NF / 32);
            tc::mbar_init(&sm.qrdy[b], T3_NF / 32);
            tc::mbar_init(&sm.qemp[b], 3);
        }
        tc::fence_mbar_init();
    }
    for (int i = tid; i < 2 * R * 2; i += T3_NT) {
        (&sm.cond[0][0][0])[i] = 0ull;
        (&sm.afar[0][0][0])[i] = 0ull;
    }
    if (tid < 2) sm.qn[tid] = 0;
    if (tid < 2 * GP) (&sm.cl_n[0][0])[tid] = 0;
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = sm.tmem_base;

    T3P_BEGIN();
    if (warp == 0) {
        // ================= metadata (bulk copies of the staged group) =================
        for (int64_t g = 0; g < nmine; ++g) {
            const int m = (int)(g % NM);
            const int64_t e0 = (gbase + blockIdx.x + g * G) * R;  // first staging slot of the group
            if (lane == 0) {
                T3P_WAIT(0, tc::mbar_wait(&sm.mempty[m], (uint32_t)(((g / NM) & 1) ^ 1)));
                T3Meta &mt = sm.meta[m];
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(&sm.mfull[m])),
                             "r"(T3_META_BYTES)
                             : "memory");
                tc::bulk_g2s(&mt, a.w.s_meta + (e0 / R) * (int64_t)T3_META_BYTES, T3_META_BYTES, &sm.mfull[m]);
                T3P_EV(g, 0);
            }
            __syncwarp();
        }
    } else if (warp >= 11 && warp < 11 + T3_NP) {
        // ================= row producers (9 warps) =================
        // warp pi stages group rows pi, pi + 9, ..: one 512-byte row per instruction (lane =
        // 16-byte chunk, 128-byte swizzle)
        const int pi = warp - 11;
        const uint32_t lo = (uint32_t)((lane >> 3) * T3_KB), lx = (uint32_t)(lane & 7);
        for (int64_t g = 0; g < nmine; ++g) {
            const int m = (int)(g % NM);
            T3P_WAIT(15, tc::mbar_wait(&sm.mfull[m], (uint32_t)((g / NM) & 1)));
            for (int c = 0; c < nch; ++c) {
                const int64_t u = g * nch + c;  // stage use index
                const int s = (int)(u % NS);
                const bool cv = c * 32 + lane < nq;
                T3P_WAIT(16, tc::mbar_wait(&sm.empty[s], (uint32_t)(((u / NS) & 1) ^ 1)));
                const uint32_t stg = tc::smem_u32(base + s * T3_STAGE);
#pragma unroll
                for (int q = 0; q < (R + T3_NP - 1) / T3_NP; ++q) {
                    const int r = pi + T3_NP * q;
                    if (r >= R) break;
                    const int32_t id = sm.meta[m].ids[r];
                    if (id == TOMB) continue;  // empty slot (warp-uniform)
                    const float *src = a.data + (int64_t)id * a.ld + (cv ? (c * 32 + lane) * 4 : 0);
                    const uint32_t dst = stg + lo + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128) + ((lx ^ (uint32_t)(r & 7)) << 4);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(cv ? 16 : 0));
                }
                if (pi == 0 && lane == 0 && c == 0) T3P_EV(g, 1);
#ifdef GRNND_T3_PROF
                if (lane == 0 && blockIdx.x == 0 && g < 64 && c == 0) atomicMax((unsigned long long *)&g_t3trace[g][2], (unsigned long long)clock64());
#endif
                // one arrive per lane, performed by the hardware when the lane's copies have landed;
                // the MMA thread fences the async proxy before the tensor core reads the stage
#ifdef GRNND_T3_WAITGROUP
                cp_async_commit();
                asm volatile("cp.async.wait_group 0;\n" ::: "memory");
                tc::fence_proxy_async();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&sm.full[s]);
#else
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&sm.full[s])) : "memory");
#endif
            }
        }
    } else if (warp == 1 && SPLIT) {
        // ================= split-TF32 MMA (the whole warp converts, lane 0 issues) =================
        for (int64_t g = 0; g < nmine; ++g) {
            const int s = (int)(g % NS), m = (int)(g % NM), ac = (int)(g & 1);
            tc::mbar_wait(&sm.full[s], (uint32_t)((g / NS) & 1));
            tc::mbar_wait(&sm.mfull[m], (uint32_t)((g / NM) & 1));
            tc::mbar_wait(&sm.acce[ac], (uint32_t)(((g >> 1) & 1) ^ 1));
            tc::fence_after();
            const int n = GP == 1 ? ((sm.meta[m].hdr[0].y + 15) / 16 * 16) : R;
            const uint32_t idesc = tc::idesc_tf32(n < 16 ? 16 : n);
            const uint32_t d = tmem + (uint32_t)(ac * 128);
#pragma unroll 1
            for (int kb = 0; kb < 4; ++kb) {
                const int64_t u = g * 4 + kb;
                const int slot = (int)(u & 1);
                tc::mbar_wait(&sm.rfree[slot], (uint32_t)(((u >> 1) & 1) ^ 1));  // MMAs of u - 2 done
                const float4 *src = reinterpret_cast<const float4 *>(base + s * T3_STAGE + kb * T3_KB);
                float4 *hi = reinterpret_cast<float4 *>(ring + slot * 2 * T3_KB);
                float4 *lo = hi + T3_KB / 16;
                for (int e = lane; e < T3_KB / 16; e += 32) {  // same (swizzled) layout as the stage
                    const float4 v = src[e];
                    float4 h;
                    h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                    h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                    h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                    h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                    hi[e] = h;
                    lo[e] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);  // exact
                }
                tc::fence_proxy_async();  // generic writes -> tensor-core reads
                __syncwarp();
                if (lane == 0) {
                    tc::fence_after();
                    const uint32_t ha = tc::smem_u32(hi), la = tc::smem_u32(lo);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t dh = tc::sw128_desc(ha + kk * 32), dl = tc::sw128_desc(la + kk * 32);
                        tc::mma_tf32(d, dh, dh, idesc, (kb | kk) != 0);
                        tc::mma_tf32(d, dh, dl, idesc, 1u);
                        tc::mma_tf32(d, dl, dh, idesc, 1u);
                    }
                    tc::mma_commit(&sm.rfree[slot]);
                }
                __syncwarp();
            }
            if (lane == 0) tc::mma_commit(&sm.accf[ac]);
            __syncwarp();
        }
    } else if (warp == 1) {
        // ================= MMA issuer =================
        if (lane == 0) {
            for (int64_t g = 0; g < nmine; ++g) {
                const int m = (int)(g % NM), ac = (int)(g & 1);
                const uint32_t d = tmem + (uint32_t)(ac * 128);
                for (int c = 0; c < nch; ++c) {
                    const int64_t u = g * nch + c;
                    const int s = (int)(u % NS);
                    T3P_WAIT(2, tc::mbar_wait(&sm.full[s], (uint32_t)((u / NS) & 1)));
                    if (c == 0) {
                        T3P_EV(g, 0);  // (overrides "meta issued"): rows landed, as seen by the MMA thread
                        tc::mbar_wait(&sm.mfull[m], (uint32_t)((g / NM) & 1));
                        T3P_WAIT(3, tc::mbar_wait(&sm.acce[ac], (uint32_t)(((g >> 1) & 1) ^ 1)));
                    }
                    T3P_WAIT(20, tc::fence_after(); tc::fence_proxy_async());  // cp.async (generic proxy) writes -> tensor core reads
                    const int n = GP == 1 ? ((sm.meta[m].hdr[0].y + 15) / 16 * 16) : R;
                    const uint32_t idesc = tc::idesc_tf32(n < 16 ? 16 : n);
                    const uint32_t sa = tc::smem_u32(base + s * T3_STAGE);
                    // k-blocks of 32 dims holding data (a short last chunk: fewer; the rest is 0)
                    const int kbn = MULTI ? min(4, (nq - c * 32 + 7) >> 3) : 4;
#pragma unroll
                    for (int kb = 0; kb < 4; ++kb) {
                        if (kb >= kbn) break;
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint64_t desc = tc::sw128_desc(sa + kb * T3_KB + kk * 32);
#ifndef GRNND_T3_NOMMA
                            tc::mma_tf32(d, desc, desc, idesc, (c | kb | kk) != 0);
#endif
                        }
                    }
                    if (MULTI) tc::mma_commit(&sm.empty[s]);  // the stage is free once these MMAs have read it
                }
                T3P_EV(g, 3);
                T3P_WAIT(21, tc::mma_commit(&sm.accf[ac]));
            }
        }
        __syncwarp();
    } else if ((warp >= 4 && warp <= 6) || (warp >= 11 + T3_NP && warp < 11 + T3_NP + 3 * CF::FSPLIT)) {
        // ================= filter (TMEM lanes 0..95) =================
        // warps 4..6 (and with FSPLIT 20..22: the same TMEM lanes, the other column blocks)
        const bool fb = warp >= 11 + T3_NP;
        const int fw = fb ? warp - 11 - T3_NP : warp - 4, i = fw * 32 + lane;
        const float eps_h = a.eps_h + 4.8e-7f;
        for (int64_t g = 0; g < nmine; ++g) {
            const int m = (int)(g % NM), b = (int)(g & 1);
            T3P_WAIT(4, tc::mbar_wait(&sm.mfull[m], (uint32_t)((g / NM) & 1)));
            const T3Meta &mt = sm.meta[m];
#ifdef GRNND_T3_PROF
            const long long _tf0 = clock64();
#endif
            if (!fb) {  // this row's filter terms
                const int p = i / SZ, sl = i - p * SZ;
                const bool live = sl < mt.hdr[p].y && mt.ids[i] != TOMB;
                const float nr = mt.nrm[i];
                float A = nr * (1.0f - EPS_TC);
                if (!(nr <= 1.0e37f)) A = -INFINITY;  // rearranged test could overflow: always a candidate
                const float2 t = live ? make_float2(A, fmaf(mt.dv[i], 1.0f + eps_h, 1e-30f)) : make_float2(0.0f, -1.0f);
                sm.ab[b][i] = t;
                const unsigned ok = __ballot_sync(FULL, t.y >= 0.0f);
                if (lane == 0) sm.livec[b][fw] = ok;
            }
#ifdef GRNND_T3_PROF
            if (lane == 0) T3P_ADD(22, _tf0);
#endif
            // queue b free (the exact set of group g - 2 has read it): reset its count
            if (!fb) T3P_WAIT(6, tc::mbar_wait(&sm.qemp[b], (uint32_t)(((g >> 1) & 1) ^ 1)));
            if (tid == 128) sm.qn[b] = 0;
            T3P_WAIT(5, tc::named_bar(1, T3_NF));
            T3P_WAIT(7, tc::mbar_wait(&sm.accf[b], (uint32_t)((g >> 1) & 1)));
            if (tid == 128) T3P_EV(g, 4);
            tc::fence_after();
#ifdef GRNND_T3_PROF
            const long long _tf1 = clock64();
#endif
#ifdef GRNND_T3_PROF
            {  // shared-memory load latency as seen by the filter
                const long long _l0 = clock64();
                const float v = *(volatile float *)&sm.ab[b][i].x;
                if (__float_as_uint(v) == 0x7fc00001u) sm.qn[b] = 0;  // never: consumes v
                if (lane == 0) T3P_ADD(24, _l0);
            }
#endif
            const float2 abi = sm.ab[b][i];
            uint32_t *gq = a.w.t3q + ((int64_t)blockIdx.x * 2 + b) * T3Q_GROUP;  // MULTI: queue overflow
            const int kcols = GP == 1 ? mt.hdr[0].y : R;
            const uint32_t trow = tmem + ((uint32_t)(fw * 32) << 16) + (uint32_t)(b * 128);
            unsigned np = 0;
            // 16 Gram columns [cb, cb+16) of this warp's rows; tr: the columns are the smaller
            // member of each pair (a block below the diagonal read in place of its transpose)
            auto scan16 = [&](const uint32_t *r, int cb, bool tr) {
                float4 ab4[8];  // column terms, two columns per 16-byte load
#pragma unroll
                for (int c = 0; c < 8; ++c) ab4[c] = *reinterpret_cast<const float4 *>(&sm.ab[b][cb + 2 * c]);
                // pairs of this row with columns cb..cb+15 that can be tested: live column, the
                // right side of the diagonal, the same pool, live row (bit masks, not per column)
                uint32_t vm = (sm.livec[b][cb >> 5] >> (cb & 16)) & 0xFFFFu;
                {
                    const int d = i - cb;
                    vm &= tr ? (d <= 0 ? 0u : d >= 16 ? 0xFFFFu : (1u << d) - 1u)
                             : (d < 0 ? 0xFFFFu : d >= 15 ? 0u : (0xFFFFu << (d + 1)) & 0xFFFFu);
                    if (GP > 1) {
                        const int lo = (i / SZ) * SZ - cb, hi = lo + SZ;  // columns [lo, hi) of this pool
                        vm &= (lo <= 0 ? 0xFFFFu : lo >= 16 ? 0u : (0xFFFFu << lo) & 0xFFFFu) &
                              (hi >= 16 ? 0xFFFFu : hi <= 0 ? 0u : (1u << hi) - 1u);
                    }
                    if (!(abi.y >= 0.0f)) vm = 0u;
                }
                np += (unsigned)__popc(vm);
                uint32_t cm = 0u;
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const float ax = (c & 1) ? ab4[c >> 1].z : ab4[c >> 1].x;
                    const float ay = (c & 1) ? ab4[c >> 1].w : ab4[c >> 1].y;
                    // settled iff (|a|^2+|b|^2)(1-eps) - 2G >= max(dv)(1+eps_h) + tiny (tc_pairs.cuh)
                    const float lhs = fmaf(-2.0f, __uint_as_float(r[c]), abi.x + ax);
                    const float rhs = abi.y >= ay ? abi.y : ay;
                    cm |= !(lhs >= rhs) ? (1u << c) : 0u;
                }
                cm &= vm;
#ifdef GRNND_TC_VALIDATE
                // validation builds: every screened pair's |d~ - d_exact| against the bound
                // TC_EPS (|a|^2 + |b|^2) the filter relies on (the stage is still resident)
                if (a.stats) {
                    const unsigned char *stg = base + (int)(g % NS) * T3_STAGE;
                    uint32_t vv = vm;
                    unsigned long long chk = 0, bad = 0;
                    float worst = 0.0f;
                    while (vv) {
                        const int c = __ffs(vv) - 1;
                        vv &= vv - 1u;
                        const int jr = cb + c, ii = tr ? jr : i, jj = tr ? i : jr;
                        float dx = 0.0f;
                        for (int q = 0; q < nq; ++q) {
                            // (MULTI: the group's rows are no longer staged: from global memory)
                            const float4 x = MULTI ? __ldg(reinterpret_cast<const float4 *>(a.data + (int64_t)mt.ids[ii] * a.ld) + q)
                                                   : *reinterpret_cast<const float4 *>(stg + t3_off(ii, q));
                            const float4 y = MULTI ? __ldg(reinterpret_cast<const float4 *>(a.data + (int64_t)mt.ids[jj] * a.ld) + q)
                                                   : *reinterpret_cast<const float4 *>(stg + t3_off(jj, q));
                            dx = exact_step4(dx, x, y);
                        }
                        const float nn = mt.nrm[i] + mt.nrm[jr];
                        const float err = fabsf(fmaf(-2.0f, __uint_as_float(r[c]), nn) - dx);
                        const float ratio = err / fmaf(EPS_TC, nn, 1e-30f);
                        worst = ratio > worst ? ratio : worst;
                        bad += ratio > 1.0f ? 1ull : 0ull;
                        ++chk;
                    }
                    if (chk) {
                        atomicMax((int *)&a.stats[GRNND_ST_TCV_MAX_RATIO], __float_as_int(worst));
                        atomicAdd((unsigned long long *)&a.stats[GRNND_ST_TCV_CHECKED], chk);
                        if (bad) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_TCV_VIOLATIONS], bad);
                    }
                }
#endif
                if (__any_sync(FULL, cm != 0u)) {
                    const int n = __popc(cm);
                    int qi = n ? atomicAdd(&sm.qn[b], n) : 0;
                    while (cm) {
                        const int c = __ffs(cm) - 1;
                        cm &= cm - 1u;
                        const int jr = cb + c;
                        const uint32_t key = tr ? (uint32_t)((jr << 8) | i) : (uint32_t)((i << 8) | jr);
                        if (qi < S::QC) sm.q[b][qi] = key;
                        else if (MULTI) gq[qi - S::QC] = key;  // (< T3Q_GROUP - QC beyond: all pairs fit)
                        ++qi;
                    }
                }
            };
            // Gram columns in 32-column TMEM loads
            auto scan32 = [&](int cb, int hi, bool tr) {  // columns [cb, min(cb + 32, hi))
                uint32_t r[32];
                tc::tmem_ld32_nw(trow + (uint32_t)cb, r);
                tc::tmem_wait_ld();
                scan16(r, cb, tr);
                if (cb + 16 < hi) scan16(r + 16, cb + 16, tr);
            };
            // both 32-column TMEM loads of a warp in flight before either is scanned
            auto scan64 = [&](int ca, bool ta, int cb2, bool tb, int hi) {  // columns [ca, ca+32), [cb2, cb2+32)
                uint32_t r0[32], r1[32];
                const bool h0 = ca < hi, h1 = cb2 >= 0 && cb2 < hi;
                if (h0) tc::tmem_ld32_nw(trow + (uint32_t)ca, r0);
                if (h1) tc::tmem_ld32_nw(trow + (uint32_t)cb2, r1);
                tc::tmem_wait_ld();
                if (h0) {
                    scan16(r0, ca, ta);
                    if (ca + 16 < hi) scan16(r0 + 16, ca + 16, ta);
                }
                if (h1) {
                    scan16(r1, cb2, tb);
                    if (cb2 + 16 < hi) scan16(r1 + 16, cb2 + 16, tb);
                }
            };
            if (GRNND_T3_NOFILTER) {
            } else if (GRNND_T3_PREF && !CF::FSPLIT) {
                if (GP == 1) {
                    scan64(fw * 32, false, fw < 2 ? fw * 32 + 32 : 0, fw == 2, kcols);
                } else {
                    const int c_lo = ((fw * 32) / SZ) * SZ, c_hi = ((fw * 32 + 31) / SZ + 1) * SZ;
                    const int start = ((c_lo >> 4) << 4) > fw * 32 ? ((c_lo >> 4) << 4) : fw * 32;
#pragma unroll 1
                    for (int cb = start; cb < c_hi; cb += 64) scan64(cb, false, cb + 32, false, c_hi);  // warp-uniform
                }
            } else if (GP == 1) {
                // upper-triangle 32x32 blocks (a, b'), a <= b' < 3, two per warp: (fw, fw) and
                // (fw, fw+1); warp 2 takes (0, 2) as its transpose (rows 64.., columns 0..31)
                const int c0 = fw * 32, c1 = fw < 2 ? fw * 32 + 32 : 0;
                const bool t1 = fw == 2;
                if constexpr (CF::FSPLIT) {
                    const int cb = fb ? c1 : c0;
                    if (cb < kcols) scan32(cb, kcols, fb && t1);
                } else {
#pragma unroll 1
                    for (int h = 0; h < 2; ++h) {  // warp-uniform
                        const int cb = h ? c1 : c0;
                        if (cb < kcols) scan32(cb, kcols, h && t1);
                    }
                }
            } else {
                const int c_lo = ((fw * 32) / SZ) * SZ, c_hi = ((fw * 32 + 31) / SZ + 1) * SZ;
                const int start = ((c_lo >> 4) << 4) > fw * 32 ? ((c_lo >> 4) << 4) : fw * 32;
                constexpr int CSTEP = 32 * (1 + CF::FSPLIT);
#pragma unroll 1
                for (int cb = start + (fb ? 32 : 0); cb < c_hi; cb += CSTEP) scan32(cb, c_hi, false);  // warp-uniform
            }
            st_pairs += np;
#ifdef GRNND_T3_PROF
            if (lane == 0) T3P_ADD(23, _tf1);
#endif
            tc::fence_before();
            if (tid == 128) T3P_EV(g, 5);
            tc::warp_arrive(&sm.acce[b]);
            tc::warp_arrive(&sm.qrdy[b]);
        }
    } else {
        // ================= exact chains + write-out: two sets of 3 warps =================
        // set E (warps 2, 3, 7 / 8, 9, 10) takes the groups g = E mod 2, so the chains (~600+
        // cycles of dependent adds) and write-out of one group overlap the next group's
        const int E = warp >= 8 ? 1 : 0;
        const int et = E ? (warp - 8) * 32 + lane : (warp == 7 ? 64 + lane : (warp - 2) * 32 + lane);  // 0..95
        const int bar_id = 2 + E;
        constexpr int NE = 96;
        // two chains per thread, the next chunk's four 16-byte loads issued before this chunk's
        // sums (the shared-memory latency is otherwise exposed once per chunk)
        // one chain (a thread without a second pair: the chains are shared-memory bound --
        // random rows hit the same 16-byte bank groups -- so a duplicated second chain is not free)
        auto exact1 = [&](const unsigned char *stg, int i1, int j1) -> float {
            const uint32_t r0 = (uint32_t)((i1 >> 3) * 1024 + (i1 & 7) * 128), q0 = (uint32_t)(i1 & 7);
            const uint32_t r1 = (uint32_t)((j1 >> 3) * 1024 + (j1 & 7) * 128), q1 = (uint32_t)(j1 & 7);
            auto ld = [&](uint32_t rb, uint32_t rq, int c) {
                return *reinterpret_cast<const float4 *>(stg + (uint32_t)(c >> 3) * T3_KB + rb +
                                                         ((((uint32_t)c & 7u) ^ rq) << 4));
            };
            float s1 = 0.0f;
            float4 x1 = ld(r0, q0, 0), y1 = ld(r1, q1, 0);
#pragma unroll 4
            for (int c = 0; c < nq; ++c) {
                const int cn = c + 1 < nq ? c + 1 : c;
                const float4 nx1 = ld(r0, q0, cn), ny1 = ld(r1, q1, cn);
                s1 = exact_step4(s1, x1, y1);
                x1 = nx1;
                y1 = ny1;
            }
            return s1;
        };
        auto exact2 = [&](const unsigned char *stg, int i1, int j1, int i2, int j2, float &d1, float &d2) {
            const uint32_t r0 = (uint32_t)((i1 >> 3) * 1024 + (i1 & 7) * 128), q0 = (uint32_t)(i1 & 7);
            const uint32_t r1 = (uint32_t)((j1 >> 3) * 1024 + (j1 & 7) * 128), q1 = (uint32_t)(j1 & 7);
            const uint32_t r2 = (uint32_t)((i2 >> 3) * 1024 + (i2 & 7) * 128), q2 = (uint32_t)(i2 & 7);
            const uint32_t r3 = (uint32_t)((j2 >> 3) * 1024 + (j2 & 7) * 128), q3 = (uint32_t)(j2 & 7);
            auto ld = [&](uint32_t rb, uint32_t rq, int c) {
                return *reinterpret_cast<const float4 *>(stg + (uint32_t)(c >> 3) * T3_KB + rb +
                                                         ((((uint32_t)c & 7u) ^ rq) << 4));
            };
            float s1 = 0.0f, s2 = 0.0f;
            float4 x1 = ld(r0, q0, 0), y1 = ld(r1, q1, 0), x2 = ld(r2, q2, 0), y2 = ld(r3, q3, 0);
#pragma unroll 2
            for (int c = 0; c < nq; ++c) {
                const int cn = c + 1 < nq ? c + 1 : c;
                const float4 nx1 = ld(r0, q0, cn), ny1 = ld(r1, q1, cn), nx2 = ld(r2, q2, cn), ny2 = ld(r3, q3, cn);
                s1 = exact_step4(s1, x1, y1);
                s2 = exact_step4(s2, x2, y2);
                x1 = nx1;
                y1 = ny1;
                x2 = nx2;
                y2 = ny2;
            }
            d1 = s1;
            d2 = s2;
        };
        for (int64_t g = E; g < nmine; g += 2) {
            const int s = (int)(g % NS), m = (int)(g % NM), b = (int)(g & 1);
            const unsigned char *stg = base + s * T3_STAGE;
            const T3Meta &mt = sm.meta[m];
            if (g >= 2) {  // group g - 2: record bulk stores have read the records (counts and
                           // mask rows were cleared at the end of its epilogue)
                if (et == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                tc::named_bar(bar_id, 96);
            }
            T3P_WAIT(9, tc::mbar_wait(&sm.qrdy[b], (uint32_t)((g >> 1) & 1)));
            auto record = [&](int i, int j, float d) {  // pair of group rows i < j, same pool
                const int p = i / SZ;
                const int x1 = mt.pos[i], x2 = mt.pos[j];
                const float d1 = mt.dv[i], d2 = mt.dv[j];
                const int xa = x1 < x2 ? x1 : x2, xb = x1 < x2 ? x2 : x1;
                const float dva = x1 < x2 ? d1 : d2, dvb = x1 < x2 ? d2 : d1;
                const unsigned long long bit = 1ull << (xb & 63);
                const bool far = !(dvb >= dva);
                atomicOr((unsigned long long *)&sm.cond[b][p * SZ + xa][xb >> 6], bit);
                if (far) atomicOr((unsigned long long *)&sm.afar[b][p * SZ + xa][xb >> 6], bit);
                const int c = atomicAdd(&sm.cl_n[b][p], 1);
                if (c < S::CL) {
                    sm.rec[b][p][4 + 2 * c] = (int32_t)((far ? 1u << 16 : 0u) | (xa << 8) | xb);
                    sm.rec[b][p][5 + 2 * c] = __float_as_int(d);
                }
            };
            const int qn = sm.qn[b];
#ifdef GRNND_T3_PROF
            const long long _tx0 = clock64();
#endif
            if constexpr (MULTI) {
                // D > 128: the exact chains read the rows from global memory.  Two pairs per
                // warp: the lanes square 16-byte chunks of the four rows, 128 dims at a time (the
                // next chunk's loads issued before this chunk's sums), lanes 0 / 1 add the
                // squares in the reference's order.  The queue is read in place and handed back
                // to the filter afterwards (the filter is not this path's bottleneck).
                if (et == 0) {
                    st_cand += (unsigned long long)qn;
                    st_ovf += qn > S::QC ? 1ull : 0ull;
                }
                const int ew = et >> 5;
                float *ps = sm.psq + (E * 3 + ew) * S::PSQW;
                // two pairs per warp (keys k1, k2: group rows (i << 8) | j): the lanes square
                // 16-byte chunks of the four rows, 128 dims at a time (the next chunk's loads
                // issued before this chunk's sums), lanes 0 / 1 add the squares in order
                // S::CN pairs per warp (key of pair p in lane p): every lane squares its 16-byte
                // chunk of all pairs' rows (the next 128-dim chunk's loads issued before this
                // chunk's sums); lane p adds pair p's squares in the reference's order
                constexpr int CN = S::CN;
                auto coopN = [&](uint32_t mykey, int np) -> float {
                    int32_t ia[CN], ib[CN];
#pragma unroll
                    for (int p = 0; p < CN; ++p) {
                        const uint32_t kk = __shfl_sync(FULL, mykey, p);
                        const int32_t x = mt.ids[kk >> 8], y = mt.ids[kk & 255u];
                        ia[p] = p < np && x >= 0 ? x : 0;
                        ib[p] = p < np && y >= 0 ? y : 0;
                    }
                    float4 pv[CN];
                    auto sq = [&](int c) {
                        const int q = c * 32 + lane;
#pragma unroll
                        for (int p = 0; p < CN; ++p) {
                            pv[p] = make_float4(0.f, 0.f, 0.f, 0.f);
                            if (p < np && q < nq)
                                pv[p] = sq4(__ldg(reinterpret_cast<const float4 *>(a.data + (int64_t)ia[p] * a.ld) + q),
                                            __ldg(reinterpret_cast<const float4 *>(a.data + (int64_t)ib[p] * a.ld) + q));
                        }
                    };
                    sq(0);
                    float acc = 0.0f;
                    for (int c = 0; c < nch; ++c) {
#pragma unroll
                        for (int p = 0; p < CN; ++p) reinterpret_cast<float4 *>(ps + 132 * p)[lane] = pv[p];
                        __syncwarp();
                        if (c + 1 < nch) sq(c + 1);
                        if (lane < np) {
                            const float4 *pr = reinterpret_cast<const float4 *>(ps + 132 * lane);
                            const int nc = nq - c * 32 < 32 ? nq - c * 32 : 32;
#pragma unroll 8
                            for (int cc = 0; cc < nc; ++cc) {
                                const float4 v = pr[cc];
                                acc = __fadd_rn(acc, v.x);
                                acc = __fadd_rn(acc, v.y);
                                acc = __fadd_rn(acc, v.z);
                                acc = __fadd_rn(acc, v.w);
                            }
                        }
                        __syncwarp();
                    }
                    return acc;
                };
                auto keep = [&](uint32_t kk, float x) {
                    const int i = (int)(kk >> 8), j = (int)(kk & 255u);
                    const float av = mt.dv[i], bv = mt.dv[j];
                    if (mt.ids[i] != TOMB && mt.ids[j] != TOMB && x < (av >= bv ? av : bv)) record(i, j, x);
                };
                // the queue: its first QC entries in shared memory, the rest in the CTA's global
                // overflow buffer (written by the filter before its qrdy arrival)
                const uint32_t *gqb = a.w.t3q + ((int64_t)blockIdx.x * 2 + b) * T3Q_GROUP;
                auto qkey = [&](int e) { return e < S::QC ? sm.q[b][e] : gqb[e - S::QC]; };
                for (int e0 = ew * CN; e0 < qn; e0 += 3 * CN) {  // warp-uniform
                    const int np = qn - e0 < CN ? qn - e0 : CN;
                    const uint32_t mykey = lane < np ? qkey(e0 + lane) : 0u;
                    const float x = coopN(mykey, np);
                    if (lane < np) keep(mykey, x);
                }
                tc::warp_arrive(&sm.qemp[b]);
                if (et == 0) T3P_EV(g, 6);
            } else {
            // this thread's queue entries to registers, then hand the queue back to the filter
            const uint32_t qw = (qn <= 32 && lane < qn) ? sm.q[b][lane] : 0u;  // short queues: per warp
            constexpr int QT = (S::QC + NE - 1) / NE;
            uint32_t qk[QT + (QT & 1)];
#pragma unroll
            for (int t = 0; t < QT + (QT & 1); ++t) {
                const int e = et + NE * t;
                qk[t] = (qn <= S::QC && e < qn) ? sm.q[b][e] : 0u;
            }
            tc::warp_arrive(&sm.qemp[b]);
            if (et == 0) T3P_EV(g, 6);
            if (et == 0) {
                st_cand += (unsigned long long)qn;
                st_ovf += qn > S::QC ? 1ull : 0ull;
            }
            if (qn <= T3_WCOOP) {
                // short queue: a warp per two pairs: the lanes square 16-byte chunks of the rows in
                // parallel (one shared-memory latency instead of one per chunk) into a scratch
                // row, then lanes 0 / 1 sum the squares in the reference's order
                const int ew = et >> 5;
                for (int e = ew; e < qn; e += 6) {  // warp-uniform
                    const bool two = e + 3 < qn;
                    const uint32_t k1 = __shfl_sync(FULL, qw, e), k2 = __shfl_sync(FULL, qw, two ? e + 3 : e);
                    const int i1 = (int)(k1 >> 8), j1 = (int)(k1 & 255u), i2 = (int)(k2 >> 8), j2 = (int)(k2 & 255u);
                    float4 p1 = make_float4(0.f, 0.f, 0.f, 0.f), p2 = p1;
                    if (lane < nq) {
                        const float4 x1 = *reinterpret_cast<const float4 *>(stg + t3_off(i1, lane));
                        const float4 y1 = *reinterpret_cast<const float4 *>(stg + t3_off(j1, lane));
                        p1 = sq4(x1, y1);
                        if (two) {  // (warp-uniform; no second pair: no second pair of row reads)
                            const float4 x2 = *reinterpret_cast<const float4 *>(stg + t3_off(i2, lane));
                            const float4 y2 = *reinterpret_cast<const float4 *>(stg + t3_off(j2, lane));
                            p2 = sq4(x2, y2);
                        }
                    }
                    {
                        float *ps = sm.psq + (E * 3 + ew) * S::PSQW;
                        reinterpret_cast<float4 *>(ps)[lane] = p1;
                        if (two) reinterpret_cast<float4 *>(ps + 128)[lane] = p2;
                        __syncwarp();
                        if (lane < (two ? 2 : 1)) {  // lane 0: pair 1, lane 1: pair 2; the reference's order
                            const float4 *pv = reinterpret_cast<const float4 *>(ps + 128 * lane);
                            float sx = 0.0f;
#pragma unroll 8
                            for (int c = 0; c < nq; ++c) {
                                const float4 v = pv[c];
                                sx = __fadd_rn(sx, v.x);
                                sx = __fadd_rn(sx, v.y);
                                sx = __fadd_rn(sx, v.z);
                                sx = __fadd_rn(sx, v.w);
                            }
                            const int ii = lane ? i2 : i1, jj = lane ? j2 : j1;
                            const float av = mt.dv[ii], bv = mt.dv[jj];
                            if ((lane == 0 || two) && sx < (av >= bv ? av : bv)) record(ii, jj, sx);
                        }
                        __syncwarp();
                    }
                }
            } else if (qn <= S::QC) {
#pragma unroll
                for (int t = 0; t < QT; t += 2) {
                    const int e = et + NE * t;
                    if (e >= qn) break;
                    const bool two = e + NE < qn;
                    const uint32_t k1 = qk[t], k2 = two ? qk[t + 1] : k1;
                    const int i1 = (int)(k1 >> 8), j1 = (int)(k1 & 255u), i2 = (int)(k2 >> 8), j2 = (int)(k2 & 255u);
                    float x1, x2 = 0.0f;
                    if (GRNND_T3_EXACT1 && !two) x1 = exact1(stg, i1, j1);
                    else exact2(stg, i1, j1, i2, j2, x1, x2);
                    const float a1 = mt.dv[i1], b1 = mt.dv[j1];
                    if (x1 < (a1 >= b1 ? a1 : b1)) record(i1, j1, x1);
                    const float a2 = mt.dv[i2], b2 = mt.dv[j2];
                    if (two && x2 < (a2 >= b2 ? a2 : b2)) record(i2, j2, x2);
                }
            } else {
                // queue overflow (degenerate data or the first rounds): exact sweep of every pair
#pragma unroll 1
                for (int pp = 0; pp < GP; ++pp) {
                    const int k = mt.hdr[pp].y;
                    const int npairs = k * (k - 1) / 2;
                    for (int t = et; t < npairs; t += 2 * NE) {
                        const bool two = t + NE < npairs;
                        int s1, u1, s2 = 0, u2 = 0;
                        tile_decode(t, s1, u1);
                        if (two) tile_decode(t + NE, s2, u2);
                        const int i1 = pp * SZ + s1, j1 = pp * SZ + u1 + 1;
                        const int i2 = two ? pp * SZ + s2 : i1, j2 = two ? pp * SZ + u2 + 1 : j1;
                        float x1, x2 = 0.0f;
                        if (GRNND_T3_EXACT1 && !two) x1 = exact1(stg, i1, j1);
                        else exact2(stg, i1, j1, i2, j2, x1, x2);
                        const float a1 = mt.dv[i1], b1 = mt.dv[j1];
                        if (mt.ids[i1] != TOMB && mt.ids[j1] != TOMB && x1 < (a1 >= b1 ? a1 : b1)) record(i1, j1, x1);
                        const float a2 = mt.dv[i2], b2 = mt.dv[j2];
                        if (two && mt.ids[i2] != TOMB && mt.ids[j2] != TOMB && x2 < (a2 >= b2 ? a2 : b2))
                            record(i2, j2, x2);
                    }
                }
            }
            }  // !MULTI
#ifdef GRNND_T3_PROF
            if (lane == 0) T3P_ADD(18, _tx0);
#endif
            // every thread that wrote pair records makes them visible to the async proxy (the
            // bulk stores below read them) before the set's barrier
            tc::fence_proxy_async();
            T3P_WAIT(10, tc::named_bar(bar_id, 96));  // masks + kept distances of group g complete
            if (et == 0) T3P_EV(g, 8);
#ifdef GRNND_T3_PROF
            const long long _tx1 = clock64();
#endif
            // the stage's rows are no longer read: let the producers refill it (MULTI: the MMA
            // released the group's stages)
            if (!MULTI) tc::warp_arrive(&sm.empty[s]);
            // pair records -> global (decide_kernel); masks only for incomplete
            // lists (rare; regular stores); every mask row re-zeroed for the next group
            if (et < GP && mt.hdr[et].x >= 0) {
                const int c = sm.cl_n[b][et];
                sm.rec[b][et][0] = c;
                tc::fence_proxy_async();  // the header, for the bulk store issued by et == 0
                if (c > 0) {  // the counts were zeroed for the round
                    a.w.clcnt[mt.hdr[et].x] = (c < S::CL ? c : S::CL) | (c > S::CL ? CL_TRUNC : 0);
                    st_red += (unsigned long long)c;
                }
            }
            for (int e = et; e < R * 2; e += NE) {
                const int r = e >> 1, wd = e & 1;
                const int pp = r / SZ, x = r - pp * SZ;
                if (sm.cl_n[b][pp] == 0) continue;  // no record: the pool's mask rows are still zero
                const int64_t v = mt.hdr[pp].x;
                const uint64_t cv = sm.cond[b][r][wd], fv = sm.afar[b][r][wd];
                sm.cond[b][r][wd] = 0ull;
                sm.afar[b][r][wd] = 0ull;
                if (v >= 0 && wd < mw && x < mt.hdr[pp].y - 1 && sm.cl_n[b][pp] > S::CL) {
                    a.w.cond[(v * cap + x) * mw + wd] = cv;
                    a.w.afar[(v * cap + x) * mw + wd] = fv;
                }
            }
            if (et < 32) __syncwarp();  // record headers (written by this warp) -> bulk stores
            if (et == 0) T3P_EV(g, 7);
            // pair records -> global by bulk stores (decide_kernel); their shared-memory reads
            // are waited for before this set writes records again (next group's start)
            if (et == 0) {
#pragma unroll
                for (int pp = 0; pp < GP; ++pp) {
                    const int64_t v = mt.hdr[pp].x;
                    if (v < 0 || sm.cl_n[b][pp] == 0) continue;  // no records: nothing to store
                    const int nw = sm.cl_n[b][pp] < S::CL ? sm.cl_n[b][pp] : S::CL;
                    const uint32_t bytes = (uint32_t)((16 + 8 * nw + 15) & ~15);
                    tc::fence_proxy_async();
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                     a.w.clrec + v * (int64_t)CLREC),
                                 "r"(tc::smem_u32(&sm.rec[b][pp][0])), "r"(bytes)
                                 : "memory");
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
#ifdef GRNND_T3_PROF
            if (lane == 0) T3P_ADD(19, _tx1);
#endif
            if (et == 0) T3P_EV(g, 9);
            // every thread of the set is past its reads of the pair counts (the mask-row loop
            // and the bulk-store sizes above): only now may they be reset for group g + 2.
            // (Resetting them at the next group's start, after a wait only by et == 0, let a
            // slow warp of the set still in this loop read a zeroed count and skip clearing --
            // and exporting -- that pool's mask rows: a rare, timing-dependent wrong graph.)
            tc::named_bar(bar_id, 96);
            if (et < GP) sm.cl_n[b][et] = 0;
            tc::warp_arrive(&sm.mempty[m]);
        }
    }
    if ((warp == 2 || warp == 8) && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#ifdef GRNND_T3_PROF
    if (lane == 0) T3P_ADD(warp == 0 ? 1 : warp == 1 ? 17 : (warp >= 4 && warp <= 6) ? 8 : (warp >= 11 && warp < 11 + T3_NP) ? 14 : warp >= 11 ? 25 : 11, _t3p0);
    if (tid == 0) atomicAdd(&t3p_sm[12], (unsigned long long)nmine);
#endif
    tc::fence_before();
    __syncthreads();
#ifdef GRNND_T3_PROF
    if (tid < 32 && t3p_sm[tid]) atomicAdd(&g_t3prof[bin][tid], t3p_sm[tid]);
#endif
    if (warp == 1) tc::tmem_dealloc(tmem, TC_TMEM_COLS);
    if (a.stats) {
        st_pairs = warp_sum(st_pairs);
        st_red = warp_sum(st_red);
        if (lane == 0 && st_pairs) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_PAIRS], st_pairs);
        if (lane == 0 && st_red) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_REDIRECTABLE], st_red);
        if (st_cand) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_CANDIDATES], st_cand);
        if (st_ovf) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_OVERFLOWS], st_ovf);
    }
}

// Lays out the metadata of every TC group contiguously (staging slot e = group * 96 + row):
// pool id, stored distance, permutation position, row norm; plus per group the (vertex, k)
// of its pools.  Thread per staging slot: reads of a pool's row are coalesced.
__global__ void tc_stage_kernel(PropArgs a) {
    const unsigned long long *ctr = a.w.ctr;
    int64_t gb[T3_NBINS + 2];
    gb[1] = 0;
    for (int b = 1; b <= T3_NBINS; ++b) gb[b + 1] = gb[b] + ((int64_t)ctr[C_BIN0 + b] + tc_bin_gp(b) - 1) / tc_bin_gp(b);
    const int64_t total = gb[T3_NBINS + 1] * T3_ROWS;
    const int cap = a.cap, pcap = a.w.pcap;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t grp = e / T3_ROWS;
        const int r = (int)(e - grp * T3_ROWS);
        int b = 1;
        while (b < T3_NBINS && grp >= gb[b + 1]) ++b;
        const int sz = tc_bin_sz(b), gp = tc_bin_gp(b);
        const int p = r / sz, s = r - p * sz;
        const int64_t posn = (grp - gb[b]) * gp + p;  // position in bin b's list
        int2 vk = make_int2(-1, 0);
        if (posn < (int64_t)ctr[C_BIN0 + b]) vk = a.w.bins[(int64_t)b * a.w.n + posn];
        int32_t id = TOMB;
        float dv = 0.0f, nr = 0.0f;
        uint8_t ps = 0;
        if (s < vk.y) {
            const int64_t off = (int64_t)vk.x * cap + s;
            id = a.read_ids[off];
            dv = a.read_dists[off];
            ps = a.w.pos8[(int64_t)vk.x * pcap + s];
            nr = a.norms[id];
        }
        T3Meta &mt = reinterpret_cast<T3Meta *>(a.w.s_meta)[grp];
        mt.ids[r] = id;
        mt.dv[r] = dv;
        mt.nrm[r] = nr;
        mt.pos[r] = ps;
        if (s == 0) mt.hdr[p] = vk;
    }
}
