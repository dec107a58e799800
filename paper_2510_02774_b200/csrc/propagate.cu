// propagate.cu -- the pair phase of one GRNND update round (the hot kernels).
//
// Reference: gen_update_messages, /root/reference/pkg/src/grnnd/_numba_kernels.py:125-192
// (with _fill_perm :64-88, _hash4 :36-41, _sqdist :50-56).  Per vertex v with k live
// pool entries: visit all pairs in a hash-driven Fisher-Yates order; a pair whose
// mutual distance is strictly below the larger stored distance redirects the farther
// member toward the closer one (tombstoning it); survivors stay.
//
// B200 design -- three kernels per round:
//  1. bin_kernel (thread per vertex): bins vertices by k and computes each vertex's
//     Fisher-Yates permutation (positions stored as bytes).
//  2. pairs_kernel<bin> (the FP32 hot loop, order free): CTA per vertex, persistent over
//     its bin, k vector rows gathered HBM -> smem by cp.async (16 B, L2-only) into a
//     double buffer so the next vertex's rows land while this one computes; ALL
//     upper-triangle pair distances in TxT register tiles with the reference's exact
//     arithmetic (sequential fp32 sub/mul/add, no FMA -> bit-identical distances); the
//     redirect condition of every pair becomes two bit masks in permutation space:
//     cond[x] (pair redirects) and afar[x] (the anchor x is the farther member).  No
//     order-dependent work and no serial phase: every warp does tiles.
//  3. decide_kernel (warp per vertex): the anchor-serial rule (SURVEY 7 hard part 1) as
//     a scan over the masks -- __ballot finds the next anchor that still has a live
//     redirect partner, anchors without one cost nothing -- then emission (distance
//     re-evaluated exactly from L2-resident rows; ~10% of entries), tombstones, stats.
#include <cstdio>

#include "common.cuh"
#include "propagate.cuh"

namespace grnnd {

__device__ __forceinline__ int bin_of(int k, int tc_bins) {
    if (tc_bins)  // tensor-core groups of 96 rows: slot sizes 8, 16, 24, 32, 48, 96 (tc3_pairs.cuh)
        return k <= 1 ? 0 : k <= 8 ? 1 : k <= 16 ? 2 : k <= 24 ? 3 : k <= 32 ? 4 : k <= 48 ? 5 : 6;
    return k <= 1 ? 0 : k <= 16 ? 1 : k <= 32 ? 2 : k <= 64 ? 3 : k <= 128 ? 4 : 5;
}

constexpr int DC4 = 32;  // float4 per row chunk (128 dims)
#ifndef GRNND_B1_BATCH
#define GRNND_B1_BATCH 4  // pools per CTA batch, k <= 16
#endif
#ifndef GRNND_B2_BATCH
#define GRNND_B2_BATCH 2  // pools per CTA batch, k <= 32
#endif

// ---------------------------------------------------------------------------------
// 1. binning + per-vertex Fisher-Yates permutation (_fill_perm :64-74)
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t mod_small(uint64_t h, uint32_t m) {
    // h % m for m < 2^16 with 32-bit remainders only: h = hi * 2^32 + lo
    const uint32_t hi = (uint32_t)(h >> 32), lo = (uint32_t)h;
    const uint32_t r32 = (0xFFFFFFFFu % m + 1u) % m;  // 2^32 mod m in 32-bit arithmetic
    return (uint32_t)(((uint64_t)(hi % m) * r32 + (lo % m)) % m);
}

__global__ void bin_kernel(const int32_t *__restrict__ read_count, int64_t n, int32_t cap, Workspace w,
                           int64_t *__restrict__ stats, int slice_mode, const int32_t *__restrict__ read_ids,
                           const float *__restrict__ read_dists, int64_t lo, uint64_t seed, uint64_t stream_id,
                           int order_code, int32_t *__restrict__ msg_tgt, int32_t *__restrict__ msg_id,
                           float *__restrict__ msg_dist, int32_t *__restrict__ msg_cnt, int tc_bins) {
    // thread = vertex for the binning; the Fisher-Yates hashes (the costly part, ~k x 100
    // instructions per vertex) are computed warp-cooperatively for the warp's 32 vertices,
    // so a warp costs sum(ceil(k / 32)) hash rounds instead of max(k); each lane then runs
    // its own vertex's (cheap) swap chain from the staged swap targets.
    __shared__ unsigned long long s_sum, s_act;
    extern __shared__ uint8_t fy_scratch[];  // [blockDim.x][cap] perm + [blockDim.x][cap] swap targets
    if (threadIdx.x == 0) s_sum = s_act = 0;
    __syncthreads();
    const int lane = lane_id();
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int k = 0, b = 0;
    unsigned long long ak = 0;
    if (v < n) {
        k = read_count[v];
        b = bin_of(k, tc_bins);
        // Round API: a pool unchanged since a round in which it had no redirect-capable pair
        // still has none -- the condition d(a, b) < max(dv_a, dv_b) does not depend on the
        // visiting order -- so its pair phase would emit nothing and tombstone nothing: skip
        if (!slice_mode && w.idle[v]) b = 0;
        if (b > 0) ak = (unsigned long long)k;
        if (b > 0) {
            const unsigned peers = __match_any_sync(__activemask(), b);
            const int leader = __ffs(peers) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(&w.ctr[C_BIN0 + b], (unsigned long long)__popc(peers));
            base = __shfl_sync(peers, base, leader);
            const int rank = __popc(peers & ((1u << lane) - 1));
            w.bins[(int64_t)b * w.n + (int64_t)base + rank] = make_int2((int)v, k);
        } else if (slice_mode) {
            // k <= 1: no pairs; the lone live entry (if any) survives (:186-192)
            int c = 0;
            if (k == 1 && read_ids[v * cap] != TOMB) {
                msg_tgt[v * cap] = (int32_t)(lo + v);
                msg_id[v * cap] = read_ids[v * cap];
                msg_dist[v * cap] = read_dists[v * cap];
                c = 1;
            }
            msg_cnt[v] = c;
        }
    }
    if (order_code == 0) {
        // perm = identity; for i = k-1..1: swap(perm[i], perm[hash4(seed,stream,v,i) % (i+1)])
        uint8_t *perm = fy_scratch + threadIdx.x * cap;
        uint8_t *warp_j = fy_scratch + (size_t)blockDim.x * cap + (threadIdx.x - lane) * cap;
        const int kk = b > 0 ? k : 0;
        const uint64_t pre = vertex_prefix(seed, stream_id, (uint64_t)(lo + v));
        unsigned todo = __ballot_sync(FULL, kk > 1);
        while (todo) {
            const int u = __ffs(todo) - 1;
            todo &= todo - 1;
            const int ku = __shfl_sync(FULL, kk, u);
            const uint64_t pu = ((uint64_t)__shfl_sync(FULL, (unsigned)(pre >> 32), u) << 32) |
                                (uint64_t)__shfl_sync(FULL, (unsigned)pre, u);
            uint8_t *ju = warp_j + u * cap;
            for (int i = lane + 1; i < ku; i += 32) ju[i] = (uint8_t)mod_small(mix64(pu ^ (uint64_t)i), (uint32_t)(i + 1));
        }
        __syncwarp();
        if (kk > 1) {
            const uint8_t *jv = warp_j + lane * cap;
            for (int i = 0; i < kk; ++i) perm[i] = (uint8_t)i;
            for (int i = kk - 1; i > 0; --i) {
                const int j = jv[i];
                const uint8_t t = perm[i];
                perm[i] = perm[j];
                perm[j] = t;
            }
            uint8_t *pos = w.pos8 + v * w.pcap;
            for (int x = 0; x < kk; ++x) pos[perm[x]] = (uint8_t)x;
        }
    }
    unsigned long long ks = (unsigned long long)k;
    ks = warp_sum(ks);
    ak = warp_sum(ak);
    if (lane == 0 && ks) atomicAdd(&s_sum, ks);
    if (lane == 0 && ak) atomicAdd(&s_act, ak);
    __syncthreads();
    if (threadIdx.x == 0 && s_sum && stats) atomicAdd((unsigned long long *)&stats[GRNND_ST_MESSAGES], s_sum);
    if (threadIdx.x == 0 && s_act && stats) atomicAdd((unsigned long long *)&stats[GRNND_ST_ACTIVE_K], s_act);
}

// ---------------------------------------------------------------------------------
// 2. pairs kernel
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// Row staging: row r's float4 column q at r * rs4 + q with an ODD row stride rs4 (in
// 16-byte units), and strided tiles (tile (bI, bJ) = rows bI + nb*i x bJ + nb*j), so the
// 8 lanes of an LDS.128 phase -- consecutive bI -- read 8 consecutive rows: every 16-byte
// bank group once, conflict free without any swizzle arithmetic in the inner loop.
__host__ __device__ __forceinline__ int row_stride16(int nq_total) {
    const int c = nq_total < 32 ? nq_total : 32;
    return c | 1;
}

// upper-triangle tile index t (bJ-major) -> (bI, bJ), bI <= bJ
__device__ __forceinline__ void tile_decode(int t, int &bI, int &bJ) {
    int j = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
    while ((j + 1) * (j + 2) / 2 <= t) ++j;
    while (j * (j + 1) / 2 > t) --j;
    bJ = j;
    bI = t - j * (j + 1) / 2;
}

// T*T exact accumulators of tile (rows rA + nb*i) x (rows rB + nb*j) over float4 columns
// [0, nq); NQ > 0 fixes the trip count at compile time (D = 128: 32 columns)
template <int T, int NQ>
__device__ __forceinline__ void tile_accumulate(float (&acc)[T * T], const float4 *__restrict__ rows, int rA, int rB,
                                                int nb, int nq, int rs4) {
    const float4 *pa[T], *pb[T];
#pragma unroll
    for (int i = 0; i < T; ++i) {
        pa[i] = rows + (rA + nb * i) * rs4;
        pb[i] = rows + (rB + nb * i) * rs4;
    }
    const int n = NQ > 0 ? NQ : nq;
#pragma unroll 4
    for (int q = 0; q < n; ++q) {
        float4 A[T], B[T];
#pragma unroll
        for (int i = 0; i < T; ++i) A[i] = pa[i][q];
#pragma unroll
        for (int j = 0; j < T; ++j) B[j] = pb[j][q];
#pragma unroll
        for (int i = 0; i < T; ++i)
#pragma unroll
            for (int j = 0; j < T; ++j) {
                float s = acc[i * T + j];
                s = exact_step4(s, A[i], B[j]);
                acc[i * T + j] = s;
            }
    }
}

// T*T FFMA dot products (filtered mode): one FP32 op per pair-dim instead of three; the
// result only pre-screens pairs (tile_epilogue), so its summation order is free
template <int T, int NQ>
__device__ __forceinline__ void tile_dot(float (&acc)[T * T], const float4 *__restrict__ rows, int rA, int rB, int nb,
                                         int nq, int rs4) {
    const float4 *pa[T], *pb[T];
#pragma unroll
    for (int i = 0; i < T; ++i) {
        pa[i] = rows + (rA + nb * i) * rs4;
        pb[i] = rows + (rB + nb * i) * rs4;
    }
    const int n = NQ > 0 ? NQ : nq;
    // operands of column q+1 are loaded before the FFMAs of column q (register double
    // buffer): the LDS latency overlaps 4*T*T FFMAs instead of stalling each use
    float4 A[T], B[T];
#pragma unroll
    for (int i = 0; i < T; ++i) {
        A[i] = pa[i][0];
        B[i] = pb[i][0];
    }
#pragma unroll 2
    for (int q = 0; q < n; ++q) {
        float4 An[T], Bn[T];
        const int qn = q + 1 < n ? q + 1 : q;
#pragma unroll
        for (int i = 0; i < T; ++i) {
            An[i] = pa[i][qn];
            Bn[i] = pb[i][qn];
        }
#pragma unroll
        for (int i = 0; i < T; ++i)
#pragma unroll
            for (int j = 0; j < T; ++j) {
                float s = acc[i * T + j];
                s = fmaf(A[i].x, B[j].x, s);
                s = fmaf(A[i].y, B[j].y, s);
                s = fmaf(A[i].z, B[j].z, s);
                s = fmaf(A[i].w, B[j].w, s);
                acc[i * T + j] = s;
            }
#pragma unroll
        for (int i = 0; i < T; ++i) {
            A[i] = An[i];
            B[i] = Bn[i];
        }
    }
}

#include "pairs.cuh"
#include "lazy.cuh"

// ---------------------------------------------------------------------------------
// 3. decide kernel: anchor-serial rule over the masks, emission, tombstones
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t bits_above(int x, int w) {  // bits of word w at positions > x
    const int b = x - w * 64;
    if (b < 0) return ~0ull;
    if (b >= 63) return 0ull;
    return ~0ull << (b + 1);
}
__device__ __forceinline__ uint64_t bits_below(int f, int w) {  // bits of word w at positions < f
    const int b = f - w * 64;
    if (b <= 0) return 0ull;
    if (b >= 64) return ~0ull;
    return (1ull << b) - 1ull;
}

// bit x of a multi-word mask without a runtime index into the array (which would put it in
// local memory): every word is compared against x's word
template <int MW>
__device__ __forceinline__ bool mask_bit(const uint64_t (&m)[MW], int x) {
    // (an unconditional AND-OR per word: a conditional select is turned back into an
    // indexed -- local-memory -- load by the compiler)
    uint64_t w = 0ull;
#pragma unroll
    for (int i = 0; i < MW; ++i) w |= m[i] & (0ull - (uint64_t)((x >> 6) == i));
    return (w >> (x & 63)) & 1ull;
}

// warps per decide CTA: 8 (R <= 128), 4 for the wider rows (static shared memory <= 48 KB)
template <int MW>
constexpr int dec_warps() { return MW <= 2 ? 8 : 4; }

template <int MW>
struct DecideSmem {
    static constexpr int DEC_WARPS = dec_warps<MW>();
    static constexpr int CAPM = MW * 64;
    int32_t ids[DEC_WARPS][CAPM];
    int16_t perm[DEC_WARPS][CAPM];
    uint8_t pos[DEC_WARPS][CAPM];
    int16_t e_tgt[DEC_WARPS][CAPM];
    int16_t e_id[DEC_WARPS][CAPM];
    uint16_t e_key[DEC_WARPS][CAPM];  // (anchor pos << 8) | partner pos of message j
    float e_d[DEC_WARPS][CAPM];       // kept exact distance of message j (NaN bits: not kept)
    int2 rec[DEC_WARPS][PAIR_LIST];   // the pool's kept records (key, distance bits)
    uint64_t bm[DEC_WARPS][32][MW];   // cond / afar words of the current 32-anchor block
    uint64_t bf[DEC_WARPS][32][MW];
};

// The anchor-serial rule of one pool (SURVEY 7 hard part 1), warp-collective: anchors are
// visited in permutation-position order; an anchor with a live redirect partner emits its
// partner-far messages in position order up to the first anchor-far partner (which
// redirects the anchor and ends its row).  masks(x, c, am) gives anchor x's cond / afar
// words; dist_of(key, j, nm, found) looks message j's exact distance up (warp-collective);
// missing ones are re-evaluated from global rows.  Emits to the message list (or the
// reference's slices), tombstones read_ids, counts redirects and reference-semantics pairs.
template <int MW, bool REFP, class MaskFn, class DistFn>
__device__ __forceinline__ void decide_pool(const PropArgs &a, int k, int64_t v, const int32_t *ids,
                                            const uint8_t *pos, int16_t *perm, int16_t *e_tgt, int16_t *e_id,
                                            uint16_t *e_key, MaskFn masks, DistFn dist_of,
                                            unsigned long long &red_total, unsigned long long &refp_total) {
    const int lane = lane_id();
    const int cap = a.cap;
    const int64_t vg = a.lo + v;
    for (int s = lane; s < k; s += 32) perm[pos[s]] = (int16_t)s;
    __syncwarp();
    uint64_t live[MW];
#pragma unroll
    for (int i = 0; i < MW; ++i) {
        const int x0 = i * 64;
        const bool l0 = x0 + lane < k && ids[perm[x0 + lane]] != TOMB;
        const bool l1 = x0 + 32 + lane < k && ids[perm[x0 + 32 + lane]] != TOMB;
        live[i] = (uint64_t)__ballot_sync(FULL, l0) | ((uint64_t)__ballot_sync(FULL, l1) << 32);
    }
    int nm = 0;
    unsigned long long refp = 0;
    for (int x0 = 0; x0 < k - 1; x0 += 32) {
        const int x = x0 + lane;
        uint64_t c[MW], am[MW];
        masks(x, c, am);
        int cur = x0;
        while (true) {
            const bool mylive = x < k - 1 && mask_bit<MW>(live, x);
            bool hit = false;
#pragma unroll
            for (int i = 0; i < MW; ++i) hit |= (c[i] & live[i]) != 0ull;
            const unsigned act = __ballot_sync(FULL, x >= cur && mylive && hit);
            const int xa = act ? x0 + __ffs(act) - 1 : x0 + 32;
            // live anchors in [cur, xa) have no live redirect partner: they visit every
            // live partner after them (reference-semantics pair count)
            if (REFP && x >= cur && x < xa && mylive) {
#pragma unroll
                for (int i = 0; i < MW; ++i) refp += __popcll(live[i] & bits_above(x, i));
            }
            if (!act) break;
            const int src = xa - x0;
            int f = k;
            uint64_t em[MW];
            if (lane == src) {
#pragma unroll
                for (int i = 0; i < MW; ++i) {
                    const uint64_t m = am[i] & live[i];
                    if (m && f == k) f = i * 64 + __ffsll((long long)m) - 1;
                }
#pragma unroll
                for (int i = 0; i < MW; ++i) {
                    em[i] = c[i] & live[i] & ~am[i] & bits_below(f, i);
                    if (REFP) {  // partners visited: live, position in (xa, f] (or (xa, k) without a break)
                        const uint64_t vis = live[i] & bits_above(xa, i) & (f < k ? bits_below(f + 1, i) : ~0ull);
                        refp += __popcll(vis);
                    }
                }
            }
            f = __shfl_sync(FULL, f, src);
#pragma unroll
            for (int i = 0; i < MW; ++i) em[i] = __shfl_sync(FULL, em[i], src);
            // emission records: partner-far messages in position order, then anchor-far
            const int sa = perm[xa];
            int base = nm;
#pragma unroll
            for (int i = 0; i < MW; ++i) {
                const uint64_t m = em[i];
                if (!m) continue;
                const uint32_t lo_ = (uint32_t)m, hi_ = (uint32_t)(m >> 32);
                if ((lo_ >> lane) & 1u) {
                    const int j = base + __popc(lo_ & ((1u << lane) - 1u));
                    e_tgt[j] = (int16_t)sa;
                    e_id[j] = perm[i * 64 + lane];
                    e_key[j] = (uint16_t)((xa << 8) | (i * 64 + lane));
                }
                if ((hi_ >> lane) & 1u) {
                    const int j = base + __popc(lo_) + __popc(hi_ & ((1u << lane) - 1u));
                    e_tgt[j] = (int16_t)sa;
                    e_id[j] = perm[i * 64 + 32 + lane];
                    e_key[j] = (uint16_t)((xa << 8) | (i * 64 + 32 + lane));
                }
                base += __popcll(m);
                live[i] &= ~m;
            }
            if (f < k) {
                if (lane == 0) {
                    e_tgt[base] = perm[f];
                    e_id[base] = (int16_t)sa;
                    e_key[base] = (uint16_t)((xa << 8) | f);
                }
                ++base;
#pragma unroll
                for (int i = 0; i < MW; ++i)  // (unconditional per word: keeps live[] in registers)
                    live[i] &= ~((1ull << (xa & 63)) & (0ull - (uint64_t)((xa >> 6) == i)));
            }
            nm = base;
            cur = xa + 1;
        }
    }
    __syncwarp();
    refp_total += refp;
    red_total += (unsigned long long)nm;
    if (!a.slice_mode && nm > 0 && lane == 0) a.w.dirty[v] = 1;  // tombstoned: the apply must compact it
    unsigned long long base = 0;
    if (!a.slice_mode && nm > 0) {
        if (lane == 0) base = atomicAdd(&a.w.ctr[C_LIST], (unsigned long long)nm);
        base = __shfl_sync(FULL, base, 0);
    }
    for (int jb = 0; jb < nm; jb += 32) {
        const int j = jb + lane;
        const uint32_t mykey = j < nm ? (uint32_t)e_key[j] : 0xFFFFFFFFu;
        bool found = false;
        float d = dist_of(mykey, j, nm, found);
        if (j >= nm) continue;
        const int32_t tgt = ids[e_tgt[j]];
        const int32_t id = ids[e_id[j]];
#ifndef GRNND_DEC_NOREEVAL
        if (!found)  // list truncated (pathological pools): exact re-evaluation from global rows
#else
        if (false)   // timing experiment only (results invalid)
#endif
            d = exact_sqdist_global(a.data + (int64_t)tgt * a.ld, a.data + (int64_t)id * a.ld, a.dim);
        if (a.slice_mode) {
            a.msg_tgt[v * cap + j] = tgt;
            a.msg_id[v * cap + j] = id;
            a.msg_dist[v * cap + j] = d;
        } else {
            const unsigned long long p = base + (unsigned long long)j;
            if (p < (unsigned long long)a.w.msg_capacity) {
                a.w.e_key[p] = vg * cap + j;
                a.w.e_tgt[p] = tgt;
                a.w.e_id[p] = id;
                a.w.e_dist[p] = d;
            } else {
                a.w.ctr[C_OVERFLOW] = 1ull;
            }
        }
    }
    // tombstones (read_ids mutated in place, as the reference does) + survivors
    int sbase = nm;
    for (int s0 = 0; s0 < k; s0 += 32) {
        const int s = s0 + lane;
        bool alive = false;
        if (s < k) {
            const int x = pos[s];
            alive = mask_bit<MW>(live, x);
            if (!alive && ids[s] != TOMB) a.read_ids[v * cap + s] = TOMB;
            alive = alive && ids[s] != TOMB;
        }
        if (a.slice_mode) {  // survivors in slot order after the redirects (:186-191)
            const unsigned bal = __ballot_sync(FULL, alive);
            if (alive) {
                const int o = sbase + __popc(bal & ((1u << lane) - 1));
                a.msg_tgt[v * cap + o] = (int32_t)vg;
                a.msg_id[v * cap + o] = ids[s];
                a.msg_dist[v * cap + o] = a.read_dists[v * cap + s];
            }
            sbase += __popc(bal);
        }
    }
    if (a.slice_mode && lane == 0) a.msg_cnt[v] = sbase;
    __syncwarp();
}

// REFP: count the reference-semantics pairs (GRNND_ST_PAIRS_REF, instrumentation only:
// ~20% of the kernel's instructions; grnnd_set_instrumentation)
template <int MW, bool REFP>
__global__ void __launch_bounds__(dec_warps<MW>() * 32, 4) decide_kernel(PropArgs a) {
    __shared__ DecideSmem<MW> sm;
    const int lane = lane_id(), wib = threadIdx.x >> 5;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t n = a.hi - a.lo;
    const int cap = a.cap;
    int32_t *ids = sm.ids[wib];
    uint8_t *pos = sm.pos[wib];
    unsigned long long red_total = 0, refp_total = 0, recpools = 0;

    // Round API: the lanes screen 32 vertices at a time; only pools with a redirect-capable
    // pair have anything to decide (the others emit and tombstone nothing -- their survivors
    // stay in the row -- and the reference visits every one of their pairs)
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t step = a.slice_mode ? warps : warps * 32;
    for (int64_t v0 = a.slice_mode ? wid : wid * 32; v0 < n; v0 += step) {
        unsigned todo = 1u;  // slice mode: this warp's one vertex v0
        if (!a.slice_mode) {
            const int64_t vl = v0 + lane;
            int kl = 0;
            int32_t cl = 0;
            if (vl < n) {
                kl = a.read_count[vl];
                cl = kl >= 2 ? a.w.clcnt[vl] : 0;
            }
            if (REFP) {
                unsigned long long rp = (kl >= 2 && cl == 0) ? (unsigned long long)kl * (unsigned long long)(kl - 1) / 2ull : 0ull;
                refp_total += warp_sum(rp) * (lane == 0 ? 1ull : 0ull);
            }
            todo = __ballot_sync(FULL, cl != 0 && cl != CL_DONE);
        }
        while (todo) {
        const int64_t v = v0 + (__ffs(todo) - 1);
        todo &= todo - 1u;
        const int k = a.read_count[v];
        if (k < 2) continue;  // no pairs (slice-mode survivors of k <= 1 come from bin_kernel)
        const int32_t clc = a.w.clcnt[v];
        recpools += clc != 0 ? 1ull : 0ull;
        for (int s = lane; s < k; s += 32) {
            ids[s] = a.read_ids[v * cap + s];
            pos[s] = a.w.pos8[v * a.w.pcap + s];
        }
        const uint64_t *gc = a.w.cond + v * (int64_t)cap * MW;
        const uint64_t *ga = a.w.afar + v * (int64_t)cap * MW;
        // redirect-capable pairs (workspace.cuh PAIR_LIST): a complete list replaces the masks
        const bool from_list = (clc & CL_TRUNC) == 0;
        const int ncl = clc & (CL_TRUNC - 1);
        const int32_t *rec = a.w.clrec + v * (int64_t)CLREC;
        int2 *srec = sm.rec[wib];  // staged in shared memory (registers would spill)
        for (int t = lane; t < ncl; t += 32) srec[t] = *reinterpret_cast<const int2 *>(rec + 4 + 2 * t);
        __syncwarp();
        uint64_t(*bm)[MW] = sm.bm[wib];
        uint64_t(*bf)[MW] = sm.bf[wib];
        // a complete list: each lane ORs its (<= 2) records of the current anchor block into
        // the block's mask rows (instead of every lane scanning the whole list)
        auto masks = [&](int x, uint64_t (&c)[MW], uint64_t (&am)[MW]) {
            if (from_list) {
                const int x0 = x - lane;
#pragma unroll
                for (int i = 0; i < MW; ++i) bm[lane][i] = bf[lane][i] = 0ull;
                __syncwarp();
                for (int t = lane; t < ncl; t += 32) {
                    const uint32_t kk = (uint32_t)srec[t].x;
                    {
                        const int xr = (int)((kk >> 8) & 255u) - x0, xb = (int)(kk & 255u);
                        if (xr >= 0 && xr < 32) {
                            const uint64_t bit = 1ull << (xb & 63);
                            atomicOr((unsigned long long *)&bm[xr][xb >> 6], bit);
                            if (kk >> 16) atomicOr((unsigned long long *)&bf[xr][xb >> 6], bit);
                        }
                    }
                }
                __syncwarp();
#pragma unroll
                for (int i = 0; i < MW; ++i) {
                    c[i] = bm[lane][i];
                    am[i] = bf[lane][i];
                }
            } else {
#pragma unroll
                for (int i = 0; i < MW; ++i) {
                    c[i] = x < k - 1 ? gc[x * MW + i] : 0ull;
                    am[i] = x < k - 1 ? ga[x * MW + i] : 0ull;
                }
            }
        };
        // kept distances scattered to their messages once (the records held by each lane
        // against the nm emitted keys), then read by message index
        float *e_d = sm.e_d[wib];
        const uint16_t *ek = sm.e_key[wib];
        auto dist_of = [&](uint32_t mykey, int j, int nm, bool &found) -> float {
            if (j < 32) {  // first batch: scatter
                for (int t = lane; t < nm; t += 32) e_d[t] = __int_as_float(0x7FFFFFFF);
                __syncwarp();
                // the emitted keys ek[0, nm) ascend ((anchor pos, partner pos): anchors in
                // position order, each anchor's messages in partner order, its anchor-far
                // message last and beyond them): each record finds its message by bisection
#pragma unroll 1
                for (int h = lane; h < ncl; h += 32) {
                    const uint32_t kk = (uint32_t)srec[h].x & 0xFFFFu;
                    int lo = 0, n = nm;
#pragma unroll 1
                    while (n > 0) {
                        const int half = n >> 1;
                        if ((uint32_t)ek[lo + half] < kk) {
                            lo += half + 1;
                            n -= half + 1;
                        } else {
                            n = half;
                        }
                    }
                    if (lo < nm && (uint32_t)ek[lo] == kk) e_d[lo] = __int_as_float(srec[h].y);
                }
                __syncwarp();
            }
            if (j >= nm) return 0.0f;
            const float d = e_d[j];
            found = __float_as_int(d) != 0x7FFFFFFF;
            return d;
        };
        decide_pool<MW, REFP>(a, k, v, ids, pos, sm.perm[wib], sm.e_tgt[wib], sm.e_id[wib], sm.e_key[wib], masks, dist_of,
                        red_total, refp_total);
        }
    }
    refp_total = warp_sum(refp_total);
    if (lane == 0 && a.stats) {
        if (red_total) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_REDIRECTS], red_total);
        if (refp_total) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_PAIRS_REF], refp_total);
        if (recpools) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_RECPOOLS], recpools);
    }
}

#include "tc_pairs.cuh"
#include "tc3_pairs.cuh"


// ---------------------------------------------------------------------------------
// squared row norms for the filtered pair phase (warp per row, any summation order:
// the filter's error bound covers every order)
// ---------------------------------------------------------------------------------
__global__ void row_norms_kernel(const float *__restrict__ data, int64_t n, int32_t dim, int32_t ld,
                                 float *__restrict__ out) {
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = lane_id();
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        const float *row = data + r * ld;
        float s = 0.0f;
        for (int d = lane; d < dim; d += 32) s = fmaf(row[d], row[d], s);
        s = warp_sum(s);
        if (lane == 0) out[r] = s;
    }
}

// ---------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------
void filter_eps(int32_t dim, float *eps_n, float *eps_h) {
    // |d~ - d_seq| <= (2 gamma_D + u)(|a|^2 + |b|^2) + (D + 4) u hi near the boundary
    // (u = 2^-24, gamma_D = D u / (1 - D u)); a 2x margin covers the rounding of the
    // bound's own evaluation.  DESIGN.md 4 has the derivation.
    const double u = 1.0 / 16777216.0;
    const double D = (double)dim;
    const double g = D * u / (1.0 - D * u);
    *eps_n = (float)(2.02 * (2.0 * g + u));
    *eps_h = (float)(2.02 * (D + 5.0) * u);
}

int launch_row_norms(const float *data, int64_t n, int32_t dim, int32_t ld, float *out, cudaStream_t st) {
    if (n <= 0) return GRNND_OK;
    const int64_t blocks = std::min<int64_t>((n + 7) / 8, (int64_t)device_sm_count() * 32);
    row_norms_kernel<<<(unsigned)blocks, 256, 0, st>>>(data, n, dim, ld, out);
    return check_launch("row_norms_kernel");
}


template <int MAXK, int B, int THREADS, int TPT, int T, bool MULTI, int NQ, bool DOT>
static int launch_pairs_impl(const PropArgs &a, int bin, cudaStream_t st) {
    auto kern = pairs_kernel<MAXK, B, THREADS, TPT, T, MULTI, NQ, DOT>;
    // TxT tiles read rows up to round_up(k, T) - 1: size each member's slab for that
    const int kmax = ((MAXK < a.cap ? MAXK : a.cap) + T - 1) / T * T;
    const int nq_total = (a.dim + 3) >> 2;
    const int rs4 = row_stride16(nq_total);
    const size_t smem = align_up(sizeof(PairSmem<MAXK, B>), 128) + (size_t)B * kmax * rs4 * 16;
    static SmemOptIn optin;
    GRNND_CUDA(optin.ensure(kern, smem));
    int per_sm = 0;
    GRNND_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
    if (per_sm < 1) {
        set_error("pairs bin %d: no CTA fits (smem %zu B)", bin, smem);
        return GRNND_EUNSUPPORTED;
    }
    kern<<<device_sm_count() * per_sm, THREADS, smem, st>>>(a, bin, kmax);
    return check_launch("pairs_kernel");
}

// (MAXK, batch B, threads, tiles/thread kept across 128-dim chunks when D > 128, tile edge T)
template <int MAXK, int B, int THREADS, int TPT, int T, bool DOT>
static int launch_pairs_mode(const PropArgs &a, int bin, cudaStream_t st) {
    const int nq_total = (a.dim + 3) >> 2;
    if (nq_total == DC4) return launch_pairs_impl<MAXK, B, THREADS, TPT, T, false, DC4, DOT>(a, bin, st);
    if (a.dim <= DC4 * 4) return launch_pairs_impl<MAXK, B, THREADS, TPT, T, false, 0, DOT>(a, bin, st);
    return launch_pairs_impl<MAXK, 1, THREADS, TPT, T, true, 0, DOT>(a, bin, st);
}
// filtered mode when the caller supplied row norms (the round API), exact mode otherwise
template <int MAXK, int B, int THREADS, int TPT, int T>
static int launch_pairs(const PropArgs &a, int bin, cudaStream_t st) {
    if (a.norms) return launch_pairs_mode<MAXK, B, THREADS, TPT, T, true>(a, bin, st);
    return launch_pairs_mode<MAXK, B, THREADS, TPT, T, false>(a, bin, st);
}


template <int SZ>
static int launch_tc_pairs(const PropArgs &a, int bin, cudaStream_t st) {
    auto kern = tc_pairs_kernel<SZ>;
    const size_t smem = (size_t)TC_NSTAGE * TC_STAGE_BYTES + sizeof(TcSmem<SZ>) + 1024;
    static SmemOptIn optin;
    GRNND_CUDA(optin.ensure(kern, smem));
    kern<<<device_sm_count(), TC_THREADS, smem, st>>>(a, bin);
    return check_launch("tc_pairs_kernel");
}

#ifndef GRNND_T3_FORCE_MULTI
#define GRNND_T3_FORCE_MULTI 0  // 1: D <= 128 runs the MULTI pipeline too (stage freed by the MMA)
#endif
template <int SZ>
static int launch_tc3_pairs(const PropArgs &a, int bin, cudaStream_t st) {
    const bool multi = a.dim > 128 || GRNND_T3_FORCE_MULTI;
    const bool split = !multi && a.split;
    if (multi && device_sm_count() > T3Q_CTAS) {
        set_error("tc3: %d SMs > %d overflow-queue slots", device_sm_count(), T3Q_CTAS);
        return GRNND_EUNSUPPORTED;
    }
    auto kern = multi ? tc3_pairs_kernel<SZ, true, false>
                      : split ? tc3_pairs_kernel<SZ, false, true> : tc3_pairs_kernel<SZ, false, false>;
    const size_t smem = split ? (size_t)T3_NS_SPLIT * T3_STAGE + T3_RING + T3_PAD + sizeof(T3Smem<SZ, false>) + 1024
                              : (size_t)T3_NS * T3_STAGE + T3_PAD +
                                    (multi ? sizeof(T3Smem<SZ, true>) : sizeof(T3Smem<SZ, false>)) + 1024;
    static SmemOptIn optin[3];  // one per kernel
    GRNND_CUDA(optin[multi ? 1 : split ? 2 : 0].ensure(kern, smem));
    kern<<<device_sm_count(), multi ? T3Cfg<true>::NT : T3Cfg<false>::NT, smem, st>>>(a, bin);
    return check_launch("tc3_pairs_kernel");
}

#ifndef GRNND_TC
#define GRNND_TC 1  // tensor-core Gram pre-screen (tc_pairs.cuh) for D <= 128, R <= 128
#endif
#ifndef GRNND_LAZY_ROUNDS
#define GRNND_LAZY_ROUNDS 2  // update rounds (stream ids 1..) whose k <= 32 pools run lazy_pairs_kernel
#endif
#ifndef GRNND_TC_MULTI
#define GRNND_TC_MULTI 1  // ... and for D > 128 with R <= 96 (tc3 MULTI)
#endif


int launch_propagate(const PropArgs &a, cudaStream_t st) {
    const int64_t n = a.hi - a.lo;
    if (n <= 0) return GRNND_OK;
    GRNND_CUDA(cudaMemsetAsync(a.w.ctr + C_BIN0, 0, sizeof(unsigned long long) * NBINS, st));
    GRNND_CUDA(cudaMemsetAsync(a.w.clcnt, 0, sizeof(int32_t) * (size_t)n, st));
    // tensor-core pair phase: D <= 128 stages whole rows; D > 128 streams 128-dim chunks
    // through the same pipeline (tc3_pairs.cuh, MULTI)
    const bool tc3 = GRNND_TC && a.norms && (a.dim <= 128 || GRNND_TC_MULTI) && a.cap <= T3_ROWS && a.order_code == 0;
    const int tb = 128;
    {
        static SmemOptIn optin;
        GRNND_CUDA(optin.ensure(bin_kernel, (size_t)tb * a.cap * 2));
    }
    bin_kernel<<<(unsigned)((n + tb - 1) / tb), tb, (size_t)tb * a.cap * 2, st>>>(a.read_count, n, a.cap, a.w, a.stats, a.slice_mode,
                                                            a.read_ids, a.read_dists, a.lo, a.seed, a.stream_id,
                                                            a.order_code, a.msg_tgt, a.msg_id, a.msg_dist,
                                                            a.msg_cnt, tc3 ? 1 : 0);
    GRNND_TRY(check_launch("bin_kernel"));
    // largest k first so long CTAs start early
    if (a.cap > 128) GRNND_TRY((launch_pairs<256, 1, 256, 3, 4>(a, 5, st)));
    if (tc3) {
        tc_stage_kernel<<<device_sm_count() * 8, 256, 0, st>>>(a);
        GRNND_TRY(check_launch("tc_stage_kernel"));
        if (a.cap > 48) GRNND_TRY(launch_tc3_pairs<96>(a, 6, st));
        if (a.cap > 32) GRNND_TRY(launch_tc3_pairs<48>(a, 5, st));
        if (a.cap > 24) GRNND_TRY(launch_tc3_pairs<32>(a, 4, st));
        if (a.cap > 16) GRNND_TRY(launch_tc3_pairs<24>(a, 3, st));
        if (a.cap > 8) GRNND_TRY(launch_tc3_pairs<16>(a, 2, st));
        if (a.cap > 1) GRNND_TRY(launch_tc3_pairs<8>(a, 1, st));
    } else if (GRNND_TC && a.norms && a.dim <= 128 && a.cap <= 128 && a.order_code == 0) {
        if (a.cap > 64) GRNND_TRY(launch_tc_pairs<128>(a, 4, st));
        if (a.cap > 32) GRNND_TRY(launch_tc_pairs<64>(a, 3, st));
        if (a.cap > 16) GRNND_TRY(launch_tc_pairs<32>(a, 2, st));
        if (a.cap > 1) GRNND_TRY(launch_tc_pairs<16>(a, 1, st));
    } else {
    // k <= 32, D <= 128, round API: the anchor-serial lazy kernel evaluates only the pairs the
    // reference evaluates (first rounds of a build) and decides the pools itself
    // (rounds 1-2: redirect-dense random pools, 17-19% of the pairs evaluated; by round 3 the
    // all-pairs tile kernel plus decide is as fast)
    const bool lazy = !a.slice_mode && a.order_code == 0 && a.dim <= 128 && a.stream_id <= GRNND_LAZY_ROUNDS;
    if (lazy) {
        const size_t smem = sizeof(LazyWarp) * LZ_WARPS;
        static SmemOptIn optin;
        GRNND_CUDA(optin.ensure(lazy_pairs_kernel, smem));
        int per_sm = 0;
        GRNND_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lazy_pairs_kernel, LZ_WARPS * 32, smem));
        lazy_pairs_kernel<<<device_sm_count() * (per_sm > 0 ? per_sm : 1), LZ_WARPS * 32, smem, st>>>(a);
        GRNND_TRY(check_launch("lazy_pairs_kernel"));
    }
    // k in (64, 96] with R <= 96 (the benchmark shape): a slab sized for 96 rows fits four
    // CTAs per SM where the 128-row one fits three
    if (a.cap > 64 && a.cap <= 96) GRNND_TRY((launch_pairs<96, 1, 128, 3, 4>(a, 4, st)));
    if (a.cap > 96) GRNND_TRY((launch_pairs<128, 1, 128, 3, 4>(a, 4, st)));
    if (a.cap > 32) GRNND_TRY((launch_pairs<64, 1, 128, 3, 2>(a, 3, st)));
    if (a.cap > 16 && !lazy) GRNND_TRY((launch_pairs<32, GRNND_B2_BATCH, 128, 3, 2>(a, 2, st)));
    if (a.cap > 1 && !lazy) GRNND_TRY((launch_pairs<16, GRNND_B1_BATCH, 128, 2, 2>(a, 1, st)));
    }
    auto dec = [&](auto kern, int warps) {
        const int64_t blocks = std::min<int64_t>((n + warps - 1) / warps, (int64_t)device_sm_count() * 16);
        kern<<<(unsigned)std::max<int64_t>(1, blocks), warps * 32, 0, st>>>(a);
    };
    const bool refp = instrumentation() != 0;
    switch (a.w.mw * 2 + (refp ? 1 : 0)) {
        case 2: dec(decide_kernel<1, false>, dec_warps<1>()); break;
        case 3: dec(decide_kernel<1, true>, dec_warps<1>()); break;
        case 4: dec(decide_kernel<2, false>, dec_warps<2>()); break;
        case 5: dec(decide_kernel<2, true>, dec_warps<2>()); break;
        case 6: dec(decide_kernel<3, false>, dec_warps<3>()); break;
        case 7: dec(decide_kernel<3, true>, dec_warps<3>()); break;
        case 8: dec(decide_kernel<4, false>, dec_warps<4>()); break;
        case 9: dec(decide_kernel<4, true>, dec_warps<4>()); break;
        default: set_error("cap %d > %d unsupported", a.cap, GRNND_MAX_CAP); return GRNND_EUNSUPPORTED;
    }
    return check_launch("decide_kernel");
}

}  // namespace grnnd

#ifdef GRNND_T3_PROF
// profiling builds only: role timers of tc3_pairs_kernel (read and reset)
extern "C" int grnnd_debug_counters(unsigned long long *out, int n) {  // [8 bins][32]
    unsigned long long buf[256] = {0};
    if (cudaMemcpyFromSymbol(buf, grnnd::g_t3prof, sizeof(buf)) != cudaSuccess) return GRNND_ECUDA;
    for (int i = 0; i < n && i < 256; ++i) out[i] = buf[i];
    unsigned long long z[256] = {0};
    if (cudaMemcpyToSymbol(grnnd::g_t3prof, z, sizeof(z)) != cudaSuccess) return GRNND_ECUDA;
    return GRNND_OK;
}
extern "C" int grnnd_debug_trace(long long *out) {  // 64 x 10 event clocks of CTA 0 (read + reset)
    if (cudaMemcpyFromSymbol(out, grnnd::g_t3trace, sizeof(long long) * 640) != cudaSuccess) return GRNND_ECUDA;
    static long long z[640] = {0};
    if (cudaMemcpyToSymbol(grnnd::g_t3trace, z, sizeof(z)) != cudaSuccess) return GRNND_ECUDA;
    return GRNND_OK;
}
#endif
