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

__device__ __forceinline__ int bin_of(int k) {
    return k <= 1 ? 0 : k <= 16 ? 1 : k <= 32 ? 2 : k <= 64 ? 3 : k <= 128 ? 4 : 5;
}

constexpr int DC4 = 32;  // float4 per row chunk (128 dims)
#ifndef GRNND_NBUF
#define GRNND_NBUF 1  // row buffers per pairs CTA (2 = cross-vertex prefetch, half the CTAs/SM)
#endif
#ifndef GRNND_BIN3_T
#define GRNND_BIN3_T 2
#define GRNND_BIN3_THREADS 128
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
                           float *__restrict__ msg_dist, int32_t *__restrict__ msg_cnt) {
    __shared__ unsigned long long s_sum;
    if (threadIdx.x == 0) s_sum = 0;
    __syncthreads();
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int k = 0;
    if (v < n) {
        k = read_count[v];
        const int b = bin_of(k);
        if (b > 0) {
            const unsigned peers = __match_any_sync(__activemask(), b);
            const int leader = __ffs(peers) - 1;
            unsigned long long base = 0;
            if (lane_id() == leader) base = atomicAdd(&w.ctr[C_BIN0 + b], (unsigned long long)__popc(peers));
            base = __shfl_sync(peers, base, leader);
            const int rank = __popc(peers & ((1u << lane_id()) - 1));
            w.bins[(int64_t)b * w.n + (int64_t)base + rank] = (int32_t)v;
            if (order_code == 0) {
                // perm = identity; for i = k-1..1: swap(perm[i], perm[hash4(seed,stream,v,i) % (i+1)])
                uint8_t perm[GRNND_MAX_CAP];
                for (int i = 0; i < k; ++i) perm[i] = (uint8_t)i;
                const uint64_t pre = vertex_prefix(seed, stream_id, (uint64_t)(lo + v));
                for (int i = k - 1; i > 0; --i) {
                    const int j = (int)mod_small(mix64(pre ^ (uint64_t)i), (uint32_t)(i + 1));
                    const uint8_t t = perm[i];
                    perm[i] = perm[j];
                    perm[j] = t;
                }
                uint8_t *pos = w.pos8 + v * cap;
                for (int x = 0; x < k; ++x) pos[perm[x]] = (uint8_t)x;
            }
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
    unsigned long long ks = (unsigned long long)k;
    ks = warp_sum(ks);
    if (lane_id() == 0 && ks) atomicAdd(&s_sum, ks);
    __syncthreads();
    if (threadIdx.x == 0 && s_sum && stats) atomicAdd((unsigned long long *)&stats[GRNND_ST_MESSAGES], s_sum);
}

// ---------------------------------------------------------------------------------
// 2. pairs kernel
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// row r, float4 column q -> swizzled float4 index: lanes reading the same q of rows
// T*b + i for consecutive b hit distinct 16-byte bank groups
template <int T>
__device__ __forceinline__ int swz(int r, int q, int rs4) {
    return r * rs4 + (q ^ ((r / T) & 7));
}

// upper-triangle tile index t (bJ-major) -> (bI, bJ), bI <= bJ
__device__ __forceinline__ void tile_decode(int t, int &bI, int &bJ) {
    int j = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
    while ((j + 1) * (j + 2) / 2 <= t) ++j;
    while (j * (j + 1) / 2 > t) --j;
    bJ = j;
    bI = t - j * (j + 1) / 2;
}

template <int MAXK>
struct PairSmem {
    static constexpr int W = (MAXK + 63) / 64;  // 64-bit words per mask row
    uint64_t cond[MAXK * W];
    uint64_t afar[MAXK * W];
    int32_t ids[2][MAXK];  // pool rows of the current / next vertex
    float dv[2][MAXK];
    int32_t pos[2][MAXK];  // slot -> permutation position
    static constexpr int CL = 4 * MAXK;  // redirect-capable pairs whose distance is kept
    uint32_t cl_key[CL];   // (anchor pos << 8) | partner pos
    float cl_d[CL];
    int cl_n;
};

// T*T exact accumulators of a TxT tile over float4 columns [q0, q1)
template <int T>
__device__ __forceinline__ void tile_accumulate(float (&acc)[T * T], const float4 *__restrict__ rows, int rA, int rB,
                                                int q0, int q1, int rs4) {
#pragma unroll 2
    for (int q = q0; q < q1; ++q) {
        float4 A[T], B[T];
#pragma unroll
        for (int i = 0; i < T; ++i) A[i] = rows[swz<T>(rA + i, q, rs4)];
#pragma unroll
        for (int j = 0; j < T; ++j) B[j] = rows[swz<T>(rB + j, q, rs4)];
#pragma unroll
        for (int i = 0; i < T; ++i)
#pragma unroll
            for (int j = 0; j < T; ++j) {
                float s = acc[i * T + j];
                s = exact_step(s, A[i].x, B[j].x);
                s = exact_step(s, A[i].y, B[j].y);
                s = exact_step(s, A[i].z, B[j].z);
                s = exact_step(s, A[i].w, B[j].w);
                acc[i * T + j] = s;
            }
    }
}

// redirect condition of the T*T pairs of tile (bI, bJ), as bits in permutation space
template <int MAXK, int T>
__device__ __forceinline__ unsigned tile_epilogue(PairSmem<MAXK> &sm, int cur, const float (&acc)[T * T], int bI,
                                                  int bJ, int k) {
    constexpr int W = PairSmem<MAXK>::W;
    unsigned npairs = 0;
#pragma unroll
    for (int i = 0; i < T; ++i)
#pragma unroll
        for (int j = 0; j < T; ++j) {
            const int s = bI * T + i, u = bJ * T + j;
            if (s < u && u < k && sm.ids[cur][s] != TOMB && sm.ids[cur][u] != TOMB) {
                ++npairs;
                const float d1 = sm.dv[cur][s], d2 = sm.dv[cur][u];
                const float hi = d1 >= d2 ? d1 : d2;
                if (acc[i * T + j] < hi) {
                    const int x1 = sm.pos[cur][s], x2 = sm.pos[cur][u];
                    // anchor = the member visited first (smaller position)
                    const int xa = x1 < x2 ? x1 : x2, xb = x1 < x2 ? x2 : x1;
                    const float dva = x1 < x2 ? d1 : d2, dvb = x1 < x2 ? d2 : d1;
                    const unsigned long long bit = 1ull << (xb & 63);
                    atomicOr((unsigned long long *)&sm.cond[xa * W + (xb >> 6)], bit);
                    if (!(dvb >= dva)) atomicOr((unsigned long long *)&sm.afar[xa * W + (xb >> 6)], bit);
                    const int c = atomicAdd(&sm.cl_n, 1);
                    if (c < PairSmem<MAXK>::CL) {
                        sm.cl_key[c] = (uint32_t)((xa << 8) | xb);
                        sm.cl_d[c] = acc[i * T + j];
                    }
                }
            }
        }
    return npairs;
}

// MULTI: D > 128, rows staged 128 dims at a time with accumulators held across chunks.
// NBUF: 2 = the next vertex's rows are gathered while this vertex computes.
template <int MAXK, int THREADS, int TPT, int T, bool MULTI, int NBUF>
__global__ void __launch_bounds__(THREADS) pairs_kernel(PropArgs a, int bin, int kmax) {
    using S = PairSmem<MAXK>;
    constexpr int W = S::W;
    constexpr int PER = (MAXK + THREADS - 1) / THREADS;  // pool slots per thread
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S &sm = *reinterpret_cast<S *>(smem_raw);
    float4 *rows0 = reinterpret_cast<float4 *>(smem_raw + align_up(sizeof(S), 128));

    const int tid = threadIdx.x;
    const int64_t nbin = (int64_t)a.w.ctr[C_BIN0 + bin];
    const int32_t *blist = a.w.bins + (int64_t)bin * a.w.n;
    const int nq_total = (a.dim + 3) >> 2;  // float4 per row (ld % 4 == 0, pad cols are 0)
    const int rs4 = nq_total >= DC4 ? DC4 : ((nq_total + 7) & ~7);
    const int nchunks = (nq_total + DC4 - 1) / DC4;
    const int cap = a.cap;
    const int mw = a.w.mw;
    const int buf_elems = kmax * rs4;
    unsigned long long pairs_local = 0;

    int32_t nid[PER];
    float ndv[PER];
    int32_t npos[PER];
    auto fetch_meta = [&](int64_t it) {  // next vertex's pool row -> registers
        const int64_t v = blist[it];
        const int k = a.read_count[v];
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int s = r * THREADS + tid;
            if (s < k) {
                nid[r] = a.read_ids[v * cap + s];
                ndv[r] = a.read_dists[v * cap + s];
                npos[r] = a.order_code == 0 ? (int32_t)a.w.pos8[v * cap + s] : 0;
            }
        }
        return k;
    };
    auto store_meta = [&](int slot, int k) {
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int s = r * THREADS + tid;
            if (s < k) {
                sm.ids[slot][s] = nid[r];
                sm.dv[slot][s] = ndv[r];
                sm.pos[slot][s] = npos[r];
            }
        }
    };
    auto load_rows = [&](float4 *rows, int slot, int k, int c) {
        const int q0 = c * DC4;
        const int nq = min(DC4, nq_total - q0);
        const int total = k * nq;
        for (int e = tid; e < total; e += THREADS) {
            const int r = e / nq;
            const int q = e - r * nq;
            const int32_t id = sm.ids[slot][r];
            const float *src = a.data + (int64_t)(id < 0 ? 0 : id) * a.ld + (int64_t)(q0 + q) * 4;
            cp_async16(&rows[swz<T>(r, q, rs4)], src, id >= 0);
        }
        cp_async_commit();
    };

    int64_t it = blockIdx.x;
    if (it >= nbin) return;
    int kn = fetch_meta(it);
    store_meta(0, kn);
    __syncthreads();
    if (!MULTI) load_rows(rows0, 0, kn, 0);
    int cur = 0;

    for (; it < nbin; it += gridDim.x) {
        const int64_t v = blist[it];
        const int k = kn;
        const int64_t it_next = it + gridDim.x;
        const bool has_next = it_next < nbin;
        float4 *rows = rows0 + (NBUF == 2 ? cur * buf_elems : 0);
        float4 *rows_next = rows0 + (NBUF == 2 ? (cur ^ 1) * buf_elems : 0);

        if (a.order_code != 0) {
            // ascending debug order (:75-87): stable rank by (dist, id); published for decide
            for (int s = tid; s < k; s += THREADS) {
                const float ds = sm.dv[cur][s];
                const int32_t is = sm.ids[cur][s];
                int r = 0;
                for (int t = 0; t < k; ++t) {
                    const float dt = sm.dv[cur][t];
                    const int32_t it2 = sm.ids[cur][t];
                    r += (dt < ds || (dt == ds && (it2 < is || (it2 == is && t < s)))) ? 1 : 0;
                }
                sm.pos[cur][s] = r;
                a.w.pos8[v * cap + s] = (uint8_t)r;
            }
        }
        for (int i = tid; i < k * W; i += THREADS) {
            sm.cond[i] = 0ull;
            sm.afar[i] = 0ull;
        }
        if (tid == 0) sm.cl_n = 0;
        if (has_next) kn = fetch_meta(it_next);
        const int nb = (k + T - 1) / T;
        const int ntiles = nb * (nb + 1) / 2;
        if (!MULTI) {
            cp_async_wait_all();
            if (NBUF == 2 && has_next) store_meta(cur ^ 1, kn);
            __syncthreads();  // rows(v) landed; masks zeroed; next pool row visible
            if (NBUF == 2 && has_next) load_rows(rows_next, cur ^ 1, kn, 0);
            for (int t = tid; t < ntiles; t += THREADS) {
                int bI, bJ;
                tile_decode(t, bI, bJ);
                float acc[T * T];
#pragma unroll
                for (int p = 0; p < T * T; ++p) acc[p] = 0.0f;
                tile_accumulate<T>(acc, rows, bI * T, bJ * T, 0, nq_total, rs4);
                pairs_local += tile_epilogue<MAXK, T>(sm, cur, acc, bI, bJ, k);
            }
            if (NBUF == 1 && has_next) store_meta(cur ^ 1, kn);
            __syncthreads();  // masks complete; single buffer free
            if (NBUF == 1 && has_next) load_rows(rows0, cur ^ 1, kn, 0);
        } else {
            __syncthreads();
            for (int g0 = 0; g0 < ntiles; g0 += THREADS * TPT) {
                float acc[TPT][T * T];
#pragma unroll
                for (int tt = 0; tt < TPT; ++tt)
#pragma unroll
                    for (int p = 0; p < T * T; ++p) acc[tt][p] = 0.0f;
                for (int c = 0; c < nchunks; ++c) {
                    __syncthreads();  // everyone done with the previous chunk
                    load_rows(rows0, cur, k, c);
                    cp_async_wait_all();
                    __syncthreads();
                    const int nq = min(DC4, nq_total - c * DC4);
#pragma unroll
                    for (int tt = 0; tt < TPT; ++tt) {
                        const int t = g0 + tt * THREADS + tid;
                        if (t < ntiles) {
                            int bI, bJ;
                            tile_decode(t, bI, bJ);
                            tile_accumulate<T>(acc[tt], rows0, bI * T, bJ * T, 0, nq, rs4);
                        }
                    }
                }
#pragma unroll
                for (int tt = 0; tt < TPT; ++tt) {
                    const int t = g0 + tt * THREADS + tid;
                    if (t < ntiles) {
                        int bI, bJ;
                        tile_decode(t, bI, bJ);
                        pairs_local += tile_epilogue<MAXK, T>(sm, cur, acc[tt], bI, bJ, k);
                    }
                }
            }
            if (has_next) store_meta(cur ^ 1, kn);
            __syncthreads();
        }
        // masks -> global, rows of anchor positions 0..k-2 (coalesced words)
        uint64_t *gc = a.w.cond + v * (int64_t)cap * mw;
        uint64_t *ga = a.w.afar + v * (int64_t)cap * mw;
        for (int e = tid; e < (k - 1) * mw; e += THREADS) {
            const int x = e / mw, wd = e - x * mw;
            gc[e] = wd < W ? sm.cond[x * W + wd] : 0ull;
            ga[e] = wd < W ? sm.afar[x * W + wd] : 0ull;
        }
        {  // distances of the redirect-capable pairs (looked up by decide_kernel)
            const int lcap = 4 * (MAXK < cap ? MAXK : cap);
            const int ncl = sm.cl_n;
            const int nw = ncl < lcap ? ncl : lcap;
            if (tid == 0) a.w.cl_n[v] = nw;  // truncated lists: decide re-evaluates misses
            for (int e = tid; e < nw; e += THREADS) {
                a.w.cl[v * 4 * (int64_t)cap + e] = sm.cl_key[e];
                a.w.cl_d[v * 4 * (int64_t)cap + e] = sm.cl_d[e];
            }
        }
        __syncthreads();  // masks / pool row of this vertex are reused next iteration
        cur ^= 1;
    }
    if (a.stats) {
        pairs_local = warp_sum(pairs_local);
        if (lane_id() == 0 && pairs_local) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_PAIRS], pairs_local);
    }
}

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

constexpr int DEC_WARPS = 8;

template <int MW>
struct DecideSmem {
    static constexpr int CAPM = MW * 64;
    int32_t ids[DEC_WARPS][CAPM];
    int16_t perm[DEC_WARPS][CAPM];
    uint8_t pos[DEC_WARPS][CAPM];
    int16_t e_tgt[DEC_WARPS][CAPM];
    int16_t e_id[DEC_WARPS][CAPM];
    uint16_t e_key[DEC_WARPS][CAPM];  // (anchor pos << 8) | partner pos of message j
};

template <int MW>
__global__ void __launch_bounds__(DEC_WARPS * 32) decide_kernel(PropArgs a) {
    __shared__ DecideSmem<MW> sm;
    const int lane = lane_id(), wib = threadIdx.x >> 5;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t n = a.hi - a.lo;
    const int cap = a.cap;
    int32_t *ids = sm.ids[wib];
    int16_t *perm = sm.perm[wib];
    uint8_t *pos = sm.pos[wib];
    unsigned long long red_total = 0, refp_total = 0;

    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
        const int k = a.read_count[v];
        if (k < 2) continue;  // no pairs (slice-mode survivors of k <= 1 come from bin_kernel)
        const int64_t vg = a.lo + v;
        for (int s = lane; s < k; s += 32) {
            ids[s] = a.read_ids[v * cap + s];
            const uint8_t x = a.w.pos8[v * cap + s];
            pos[s] = x;
            perm[x] = (int16_t)s;
        }
        __syncwarp();
        uint64_t live[MW];
#pragma unroll
        for (int i = 0; i < MW; ++i) {
            const int x0 = i * 64;
            const bool l0 = x0 + lane < k && ids[perm[x0 + lane]] != TOMB;
            const bool l1 = x0 + 32 + lane < k && ids[perm[x0 + 32 + lane]] != TOMB;
            live[i] = (uint64_t)__ballot_sync(FULL, l0) | ((uint64_t)__ballot_sync(FULL, l1) << 32);
        }
        const uint64_t *gc = a.w.cond + v * (int64_t)cap * MW;
        const uint64_t *ga = a.w.afar + v * (int64_t)cap * MW;
        int nm = 0;
        unsigned long long refp = 0;
        for (int x0 = 0; x0 < k - 1; x0 += 32) {
            const int x = x0 + lane;
            uint64_t c[MW], am[MW];
#pragma unroll
            for (int i = 0; i < MW; ++i) {
                c[i] = x < k - 1 ? gc[x * MW + i] : 0ull;
                am[i] = x < k - 1 ? ga[x * MW + i] : 0ull;
            }
            int cur = x0;
            while (true) {
                const bool mylive = x < k - 1 && ((live[x >> 6] >> (x & 63)) & 1ull);
                bool hit = false;
#pragma unroll
                for (int i = 0; i < MW; ++i) hit |= (c[i] & live[i]) != 0ull;
                const unsigned act = __ballot_sync(FULL, x >= cur && mylive && hit);
                const int xa = act ? x0 + __ffs(act) - 1 : x0 + 32;
                // live anchors in [cur, xa) have no live redirect partner: they visit every
                // live partner after them (reference-semantics pair count)
                if (x >= cur && x < xa && mylive) {
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
                        // partners visited: live, position in (xa, f] (or (xa, k) without a break)
                        const uint64_t vis = live[i] & bits_above(xa, i) & (f < k ? bits_below(f + 1, i) : ~0ull);
                        refp += __popcll(vis);
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
                        sm.e_tgt[wib][j] = (int16_t)sa;
                        sm.e_id[wib][j] = perm[i * 64 + lane];
                        sm.e_key[wib][j] = (uint16_t)((xa << 8) | (i * 64 + lane));
                    }
                    if ((hi_ >> lane) & 1u) {
                        const int j = base + __popc(lo_) + __popc(hi_ & ((1u << lane) - 1u));
                        sm.e_tgt[wib][j] = (int16_t)sa;
                        sm.e_id[wib][j] = perm[i * 64 + 32 + lane];
                        sm.e_key[wib][j] = (uint16_t)((xa << 8) | (i * 64 + 32 + lane));
                    }
                    base += __popcll(m);
                    live[i] &= ~m;
                }
                if (f < k) {
                    if (lane == 0) {
                        sm.e_tgt[wib][base] = perm[f];
                        sm.e_id[wib][base] = (int16_t)sa;
                        sm.e_key[wib][base] = (uint16_t)((xa << 8) | f);
                    }
                    ++base;
                    live[xa >> 6] &= ~(1ull << (xa & 63));
                }
                nm = base;
                cur = xa + 1;
            }
        }
        __syncwarp();
        refp_total += refp;
        red_total += (unsigned long long)nm;
        // emit: exact distance re-evaluated from L2-resident rows (same arithmetic as the tiles)
        unsigned long long base = 0;
        if (!a.slice_mode && nm > 0) {
            if (lane == 0) base = atomicAdd(&a.w.ctr[C_LIST], (unsigned long long)nm);
            base = __shfl_sync(FULL, base, 0);
        }
        const int lcap = 4 * cap;
        const int ncl_raw = nm > 0 ? a.w.cl_n[v] : 0;
        const int ncl = ncl_raw < lcap ? ncl_raw : lcap;
        const uint32_t *clk = a.w.cl + v * (int64_t)lcap;
        const float *cld = a.w.cl_d + v * (int64_t)lcap;
        for (int jb = 0; jb < nm; jb += 32) {
            const int j = jb + lane;
            const uint32_t mykey = j < nm ? (uint32_t)sm.e_key[wib][j] : 0xFFFFFFFFu;
            // the pairs kernel kept every redirect-capable pair's exact distance: warp search
            float d = 0.0f;
            bool found = false;
            for (int c0 = 0; c0 < ncl; c0 += 32) {
                const uint32_t ck = c0 + lane < ncl ? clk[c0 + lane] : 0xFFFFFFFEu;
                const float cd = c0 + lane < ncl ? cld[c0 + lane] : 0.0f;
                const int nc = ncl - c0 < 32 ? ncl - c0 : 32;
                for (int t = 0; t < nc; ++t) {
                    const uint32_t kk = __shfl_sync(FULL, ck, t);
                    const float dd = __shfl_sync(FULL, cd, t);
                    if (kk == mykey) {
                        d = dd;
                        found = true;
                    }
                }
            }
            if (j >= nm) continue;
            const int32_t tgt = ids[sm.e_tgt[wib][j]];
            const int32_t id = ids[sm.e_id[wib][j]];
            if (!found)  // list truncated (pathological pools): exact re-evaluation from L2
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
                alive = (live[x >> 6] >> (x & 63)) & 1ull;
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
    refp_total = warp_sum(refp_total);
    if (lane == 0 && a.stats) {
        if (red_total) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_REDIRECTS], red_total);
        if (refp_total) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_PAIRS_REF], refp_total);
    }
}

// ---------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------
static int sm_count() {
    static int s = 0;
    if (!s) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
        if (s <= 0) s = 148;
    }
    return s;
}

template <int MAXK, int THREADS, int TPT, int T, bool MULTI, int NBUF>
static int launch_pairs_impl(const PropArgs &a, int bin, cudaStream_t st) {
    auto kern = pairs_kernel<MAXK, THREADS, TPT, T, MULTI, NBUF>;
    // TxT tiles read rows up to round_up(k, T) - 1: size each slab for that
    const int kmax = ((MAXK < a.cap ? MAXK : a.cap) + T - 1) / T * T;
    const int nq_total = (a.dim + 3) >> 2;
    const int rs4 = nq_total >= DC4 ? DC4 : ((nq_total + 7) & ~7);
    const size_t smem = align_up(sizeof(PairSmem<MAXK>), 128) + (size_t)NBUF * kmax * rs4 * 16;
    static int configured_smem = 0;
    if ((int)smem > configured_smem) {
        GRNND_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured_smem = (int)smem;
    }
    int per_sm = 0;
    GRNND_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
    if (per_sm < 1) {
        set_error("pairs bin %d: no CTA fits (smem %zu B)", bin, smem);
        return GRNND_EUNSUPPORTED;
    }
    kern<<<sm_count() * per_sm, THREADS, smem, st>>>(a, bin, kmax);
    return check_launch("pairs_kernel");
}

template <int MAXK, int THREADS, int TPT, int T>
static int launch_pairs(const PropArgs &a, int bin, cudaStream_t st) {
    if (a.dim <= DC4 * 4) return launch_pairs_impl<MAXK, THREADS, TPT, T, false, GRNND_NBUF>(a, bin, st);
    return launch_pairs_impl<MAXK, THREADS, TPT, T, true, 1>(a, bin, st);
}

int launch_propagate(const PropArgs &a, cudaStream_t st) {
    const int64_t n = a.hi - a.lo;
    if (n <= 0) return GRNND_OK;
    GRNND_CUDA(cudaMemsetAsync(a.w.ctr + C_BIN0, 0, sizeof(unsigned long long) * NBINS, st));
    const int tb = 128;
    bin_kernel<<<(unsigned)((n + tb - 1) / tb), tb, 0, st>>>(a.read_count, n, a.cap, a.w, a.stats, a.slice_mode,
                                                            a.read_ids, a.read_dists, a.lo, a.seed, a.stream_id,
                                                            a.order_code, a.msg_tgt, a.msg_id, a.msg_dist,
                                                            a.msg_cnt);
    GRNND_TRY(check_launch("bin_kernel"));
    // largest k first so long CTAs start early
    if (a.cap > 128) GRNND_TRY((launch_pairs<256, 256, 3, 4>(a, 5, st)));
    if (a.cap > 64) GRNND_TRY((launch_pairs<128, 128, 3, 4>(a, 4, st)));
    if (a.cap > 32) GRNND_TRY((launch_pairs<64, GRNND_BIN3_THREADS, 3, GRNND_BIN3_T>(a, 3, st)));
    if (a.cap > 16) GRNND_TRY((launch_pairs<32, 64, 3, 2>(a, 2, st)));
    if (a.cap > 1) GRNND_TRY((launch_pairs<16, 32, 2, 2>(a, 1, st)));
    const int64_t blocks = std::min<int64_t>((n + DEC_WARPS - 1) / DEC_WARPS, (int64_t)sm_count() * 16);
    const unsigned g = (unsigned)std::max<int64_t>(1, blocks);
    switch (a.w.mw) {
        case 1: decide_kernel<1><<<g, DEC_WARPS * 32, 0, st>>>(a); break;
        case 2: decide_kernel<2><<<g, DEC_WARPS * 32, 0, st>>>(a); break;
        case 3: decide_kernel<3><<<g, DEC_WARPS * 32, 0, st>>>(a); break;
        case 4: decide_kernel<4><<<g, DEC_WARPS * 32, 0, st>>>(a); break;
        default: set_error("cap %d > %d unsupported", a.cap, GRNND_MAX_CAP); return GRNND_EUNSUPPORTED;
    }
    return check_launch("decide_kernel");
}

}  // namespace grnnd
