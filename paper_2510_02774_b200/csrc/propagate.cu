// propagate.cu -- the pair phase of one GRNND update round (the hot kernel).
//
// Reference: gen_update_messages, /root/reference/pkg/src/grnnd/_numba_kernels.py:125-192
// (with _fill_perm :64-88, _hash4 :36-41, _sqdist :50-56).  Per vertex v with k live
// pool entries: visit all pairs in a hash-driven Fisher-Yates order; a pair whose
// mutual distance is strictly below the larger stored distance redirects the farther
// member toward the closer one (tombstoning it); survivors stay.
//
// B200 design:
//  * bin_kernel (thread per vertex) bins vertices by k and computes each vertex's
//    Fisher-Yates permutation off the critical path (positions stored as bytes);
//  * each bin runs a persistent kernel whose CTA processes one vertex at a time with a
//    CTA size / shared-memory slab matched to the bin;
//  * the k pool rows are gathered HBM -> smem with cp.async (16 B, L2-only), row-major
//    with a 16-byte XOR swizzle so the register-tiled reads below are conflict free;
//  * ALL pair distances of the pool (upper triangle, slot order) are computed with
//    4x4 register tiles in the reference's exact arithmetic (sequential fp32
//    sub/mul/add, no FMA) -> bit-identical distances to the numba oracle;
//  * the order-dependent part (anchor-serial rule, SURVEY 7 hard part 1) is a
//    warp-parallel scan over 64-bit masks: cond[x] (pair redirects) and afar[x] (anchor
//    is the farther member), indexed by permutation position; __ballot finds the next
//    anchor that still has a live redirect partner, so anchors without one cost nothing;
//  * emitted redirects get their distance re-evaluated exactly from the smem rows
//    (or L2 for D > 128), keeping the k x k distance matrix out of shared memory.
#include <cstdio>

#include "common.cuh"
#include "propagate.cuh"

namespace grnnd {

__device__ __forceinline__ int bin_of(int k) {
    return k <= 1 ? 0 : k <= 16 ? 1 : k <= 32 ? 2 : k <= 64 ? 3 : k <= 128 ? 4 : 5;
}

constexpr int DC4 = 32;  // float4 per row chunk (128 dims)

// ---------------------------------------------------------------------------------
// binning + per-vertex Fisher-Yates permutation (_fill_perm :64-74), thread per vertex
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
// the pair kernel
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// row r, float4 column q -> swizzled float4 index (conflict-free 4x4 tile reads)
// (T = tile edge: lanes reading the same q of rows T*b + i, b consecutive, hit distinct banks)
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
struct PropSmem {
    static constexpr int W = (MAXK + 63) / 64;  // 64-bit words per bitset row
    uint64_t cond[MAXK * W];
    uint64_t afar[MAXK * W];
    uint64_t live[W];
    int32_t ids[MAXK];
    float dv[MAXK];
    int32_t perm[MAXK];  // position -> slot
    int32_t pos[MAXK];   // slot -> position
    int16_t e_tgt[MAXK];  // emitted message j: target slot
    int16_t e_id[MAXK];   // emitted message j: id slot
    int nmsg;
    unsigned long long list_base;
    unsigned long long ref_pairs;
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
__device__ __forceinline__ unsigned tile_epilogue(PropSmem<MAXK> &sm, const float (&acc)[T * T], int bI, int bJ,
                                                  int k) {
    constexpr int W = PropSmem<MAXK>::W;
    unsigned npairs = 0;
#pragma unroll
    for (int i = 0; i < T; ++i)
#pragma unroll
        for (int j = 0; j < T; ++j) {
            const int s = bI * T + i, u = bJ * T + j;
            if (s < u && u < k && sm.ids[s] != TOMB && sm.ids[u] != TOMB) {
                ++npairs;
                const float d1 = sm.dv[s], d2 = sm.dv[u];
                const float hi = d1 >= d2 ? d1 : d2;
                if (acc[i * T + j] < hi) {
                    const int x1 = sm.pos[s], x2 = sm.pos[u];
                    // anchor = the member visited first (smaller position)
                    const int xa = x1 < x2 ? x1 : x2, xb = x1 < x2 ? x2 : x1;
                    const float dva = x1 < x2 ? d1 : d2, dvb = x1 < x2 ? d2 : d1;
                    const unsigned long long bit = 1ull << (xb & 63);
                    atomicOr((unsigned long long *)&sm.cond[xa * W + (xb >> 6)], bit);
                    if (!(dvb >= dva)) atomicOr((unsigned long long *)&sm.afar[xa * W + (xb >> 6)], bit);
                }
            }
        }
    return npairs;
}

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

// Anchor-serial decision (_numba_kernels.py:158-185) by warp 0, over the masks.
template <int MAXK>
__device__ __forceinline__ void decide(PropSmem<MAXK> &sm, int k) {
    constexpr int W = PropSmem<MAXK>::W;
    const int lane = lane_id();
    uint64_t live[W];
#pragma unroll
    for (int i = 0; i < W; ++i) live[i] = sm.live[i];
    int nm = 0;
    unsigned long long refp = 0;
    for (int x0 = 0; x0 < k - 1; x0 += 32) {
        const int x = x0 + lane;
        uint64_t c[W], a[W];
#pragma unroll
        for (int i = 0; i < W; ++i) {
            c[i] = x < k - 1 ? sm.cond[x * W + i] : 0ull;
            a[i] = x < k - 1 ? sm.afar[x * W + i] : 0ull;
        }
        int cur = x0;
        while (true) {
            const bool mylive = x < k - 1 && ((live[x >> 6] >> (x & 63)) & 1ull);
            bool hit = false;
#pragma unroll
            for (int i = 0; i < W; ++i) hit |= (c[i] & live[i]) != 0ull;
            const unsigned act = __ballot_sync(FULL, x >= cur && mylive && hit);
            const int xa = act ? x0 + __ffs(act) - 1 : x0 + 32;
            // live anchors in [cur, xa) have no live redirect partner: they visit every
            // live partner after them (reference-semantics pair count)
            if (x >= cur && x < xa && mylive) {
                unsigned long long cnt = 0;
#pragma unroll
                for (int i = 0; i < W; ++i) cnt += __popcll(live[i] & bits_above(x, i));
                refp += cnt;
            }
            if (!act) break;
            // the active anchor's lane resolves its row
            const int src = xa - x0;
            int f = k;
            uint64_t em[W];
            unsigned long long visited = 0;
            if (lane == src) {
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    const uint64_t m = a[i] & live[i];
                    if (m && f == k) f = i * 64 + __ffsll((long long)m) - 1;
                }
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    em[i] = c[i] & live[i] & ~a[i] & bits_below(f, i);
                    // partners visited: live, position in (xa, f] (or (xa, k) without a break)
                    const uint64_t vis = live[i] & bits_above(xa, i) & (f < k ? bits_below(f + 1, i) : ~0ull);
                    visited += __popcll(vis);
                }
                refp += visited;
            }
            f = __shfl_sync(FULL, f, src);
#pragma unroll
            for (int i = 0; i < W; ++i) em[i] = __shfl_sync(FULL, em[i], src);
            // emission records, partner-far messages in position order, then anchor-far
            const int sa = sm.perm[xa];
            int base = nm;
#pragma unroll
            for (int i = 0; i < W; ++i) {
                const uint64_t m = em[i];
                if (!m) continue;
                const uint32_t lo_ = (uint32_t)m, hi_ = (uint32_t)(m >> 32);
                if ((lo_ >> lane) & 1u) {
                    const int j = base + __popc(lo_ & ((1u << lane) - 1u));
                    sm.e_tgt[j] = (int16_t)sa;
                    sm.e_id[j] = (int16_t)sm.perm[i * 64 + lane];
                }
                if ((hi_ >> lane) & 1u) {
                    const int j = base + __popc(lo_) + __popc(hi_ & ((1u << lane) - 1u));
                    sm.e_tgt[j] = (int16_t)sa;
                    sm.e_id[j] = (int16_t)sm.perm[i * 64 + 32 + lane];
                }
                base += __popcll(m);
                live[i] &= ~m;
            }
            if (f < k) {
                if (lane == 0) {
                    sm.e_tgt[base] = (int16_t)sm.perm[f];
                    sm.e_id[base] = (int16_t)sa;
                }
                ++base;
                live[xa >> 6] &= ~(1ull << (xa & 63));
            }
            nm = base;
            cur = xa + 1;
        }
    }
    refp = warp_sum(refp);
    if (lane == 0) {
        sm.nmsg = nm;
        sm.ref_pairs = refp;
#pragma unroll
        for (int i = 0; i < W; ++i) sm.live[i] = live[i];
    }
}

// MULTI: D > 128, rows staged 128 dims at a time with accumulators held across chunks
// (a separate instantiation keeps the common D <= 128 kernel's register count low)
template <int MAXK, int THREADS, int TPT, int T, bool MULTI>
__global__ void __launch_bounds__(THREADS) propagate_kernel(PropArgs a, int bin) {
    using S = PropSmem<MAXK>;
    constexpr int W = S::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S &sm = *reinterpret_cast<S *>(smem_raw);
    float4 *rows = reinterpret_cast<float4 *>(smem_raw + align_up(sizeof(S), 128));

    const int tid = threadIdx.x;
    const int64_t nbin = (int64_t)a.w.ctr[C_BIN0 + bin];
    const int32_t *blist = a.w.bins + (int64_t)bin * a.w.n;
    const int nq_total = (a.dim + 3) >> 2;  // float4 per row (ld % 4 == 0, pad cols are 0)
    const int rs4 = nq_total >= DC4 ? DC4 : ((nq_total + 7) & ~7);
    const int nchunks = (nq_total + DC4 - 1) / DC4;
    const int cap = a.cap;
    unsigned long long pairs_local = 0;

    for (int64_t it = blockIdx.x; it < nbin; it += gridDim.x) {
        const int64_t v = blist[it];  // local row
        const int64_t vg = a.lo + v;  // global vertex id
        const int k = a.read_count[v];
        const int32_t *rid = a.read_ids + v * cap;
        const float *rdv = a.read_dists + v * cap;

        // ---- 1. pool row + permutation positions, bitset reset ----
        for (int s = tid; s < k; s += THREADS) {
            sm.ids[s] = rid[s];
            sm.dv[s] = rdv[s];
            if (a.order_code == 0) sm.pos[s] = a.w.pos8[v * cap + s];
        }
        for (int i = tid; i < k * W; i += THREADS) {
            sm.cond[i] = 0ull;
            sm.afar[i] = 0ull;
        }
        __syncthreads();

        // ---- 2. gather the pool rows (first 128-dim chunk) ----
        auto load_chunk = [&](int c) {
            const int q0 = c * DC4;
            const int nq = min(DC4, nq_total - q0);
            const int total = k * nq;
            for (int e = tid; e < total; e += THREADS) {
                const int r = e / nq;
                const int q = e - r * nq;
                const int32_t id = sm.ids[r];
                const float *src = a.data + (int64_t)(id < 0 ? 0 : id) * a.ld + (int64_t)(q0 + q) * 4;
                cp_async16(&rows[swz<T>(r, q, rs4)], src, id >= 0);
            }
            cp_async_commit();
        };
        load_chunk(0);

        if (a.order_code != 0) {
            // ascending debug order (:75-87): stable rank by (dist, id)
            for (int s = tid; s < k; s += THREADS) {
                const float ds = sm.dv[s];
                const int32_t is = sm.ids[s];
                int r = 0;
                for (int t = 0; t < k; ++t) {
                    const float dt = sm.dv[t];
                    const int32_t it2 = sm.ids[t];
                    r += (dt < ds || (dt == ds && (it2 < is || (it2 == is && t < s)))) ? 1 : 0;
                }
                sm.pos[s] = r;
            }
            __syncthreads();
        }
        for (int s = tid; s < k; s += THREADS) sm.perm[sm.pos[s]] = s;
        __syncthreads();
        if (tid < 32) {
            // live mask by permutation position (one ballot per 32 positions)
            for (int x0 = 0; x0 < W * 64; x0 += 32) {
                const int x = x0 + tid;
                const bool lv = x < k && sm.ids[sm.perm[x]] != TOMB;
                const unsigned b = __ballot_sync(FULL, lv);
                if (tid == 0) {
                    if ((x0 & 63) == 0) sm.live[x0 >> 6] = (uint64_t)b;
                    else sm.live[x0 >> 6] |= (uint64_t)b << 32;
                }
            }
        }

        // ---- 3. all-pairs exact distances, TxT register tiles, upper triangle ----
        const int nb = (k + T - 1) / T;
        const int ntiles = nb * (nb + 1) / 2;
        if (!MULTI) {
            cp_async_wait_all();
            __syncthreads();
            for (int t = tid; t < ntiles; t += THREADS) {
                int bI, bJ;
                tile_decode(t, bI, bJ);
                float acc[T * T];
#pragma unroll
                for (int p = 0; p < T * T; ++p) acc[p] = 0.0f;
                tile_accumulate<T>(acc, rows, bI * T, bJ * T, 0, nq_total, rs4);
                pairs_local += tile_epilogue<MAXK, T>(sm, acc, bI, bJ, k);
            }
        } else {
            for (int g0 = 0; g0 < ntiles; g0 += THREADS * TPT) {
                float acc[TPT][T * T];
#pragma unroll
                for (int tt = 0; tt < TPT; ++tt)
#pragma unroll
                    for (int p = 0; p < T * T; ++p) acc[tt][p] = 0.0f;
                for (int c = 0; c < nchunks; ++c) {
                    if (c > 0 || g0 > 0) {
                        __syncthreads();  // everyone done with the previous chunk
                        load_chunk(c);
                    }
                    cp_async_wait_all();
                    __syncthreads();
                    const int nq = min(DC4, nq_total - c * DC4);
#pragma unroll
                    for (int tt = 0; tt < TPT; ++tt) {
                        const int t = g0 + tt * THREADS + tid;
                        if (t < ntiles) {
                            int bI, bJ;
                            tile_decode(t, bI, bJ);
                            tile_accumulate<T>(acc[tt], rows, bI * T, bJ * T, 0, nq, rs4);
                        }
                    }
                }
#pragma unroll
                for (int tt = 0; tt < TPT; ++tt) {
                    const int t = g0 + tt * THREADS + tid;
                    if (t < ntiles) {
                        int bI, bJ;
                        tile_decode(t, bI, bJ);
                        pairs_local += tile_epilogue<MAXK, T>(sm, acc[tt], bI, bJ, k);
                    }
                }
            }
        }
        __syncthreads();

        // ---- 4. anchor-serial decision over the masks (warp 0) ----
        if (tid < 32) {
            decide<MAXK>(sm, k);
            if (tid == 0 && !a.slice_mode && sm.nmsg > 0)
                sm.list_base = atomicAdd(&a.w.ctr[C_LIST], (unsigned long long)sm.nmsg);
        }
        __syncthreads();

        // ---- 5. emit redirects: exact distance re-evaluated from the staged rows ----
        const int nm = sm.nmsg;
        for (int j = tid; j < nm; j += THREADS) {
            const int st = sm.e_tgt[j], si = sm.e_id[j];
            const int32_t tgt = sm.ids[st];
            const int32_t id = sm.ids[si];
            float d;
            if (!MULTI) {
                d = 0.0f;
                for (int q = 0; q < nq_total; ++q) {
                    const float4 x = rows[swz<T>(st, q, rs4)];
                    const float4 y = rows[swz<T>(si, q, rs4)];
                    d = exact_step(d, x.x, y.x);
                    d = exact_step(d, x.y, y.y);
                    d = exact_step(d, x.z, y.z);
                    d = exact_step(d, x.w, y.w);
                }
            } else {
                d = exact_sqdist_global(a.data + (int64_t)tgt * a.ld, a.data + (int64_t)id * a.ld, a.dim);
            }
            if (a.slice_mode) {
                a.msg_tgt[v * cap + j] = tgt;
                a.msg_id[v * cap + j] = id;
                a.msg_dist[v * cap + j] = d;
            } else {
                const unsigned long long p = sm.list_base + (unsigned long long)j;
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
        for (int s = tid; s < k; s += THREADS) {
            const int x = sm.pos[s];
            const bool alive = (sm.live[x >> 6] >> (x & 63)) & 1ull;
            if (!alive && sm.ids[s] != TOMB) a.read_ids[v * cap + s] = TOMB;
        }
        if (a.slice_mode && tid < 32) {
            // survivors in slot order after the redirects (:186-191)
            int base = nm;
            for (int s0 = 0; s0 < k; s0 += 32) {
                const int s = s0 + tid;
                bool alive = false;
                if (s < k) {
                    const int x = sm.pos[s];
                    alive = ((sm.live[x >> 6] >> (x & 63)) & 1ull) && sm.ids[s] != TOMB;
                }
                const unsigned bal = __ballot_sync(FULL, alive);
                if (alive) {
                    const int o = base + __popc(bal & ((1u << tid) - 1));
                    a.msg_tgt[v * cap + o] = (int32_t)vg;
                    a.msg_id[v * cap + o] = sm.ids[s];
                    a.msg_dist[v * cap + o] = sm.dv[s];
                }
                base += __popc(bal);
            }
            if (tid == 0) a.msg_cnt[v] = base;
        }
        if (tid == 0 && a.stats) {
            if (nm) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_REDIRECTS], (unsigned long long)nm);
            atomicAdd((unsigned long long *)&a.stats[GRNND_ST_PAIRS_REF], sm.ref_pairs);
        }
        __syncthreads();  // smem reuse by the next vertex
    }
    if (a.stats) {
        pairs_local = warp_sum(pairs_local);
        if (lane_id() == 0 && pairs_local) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_PAIRS], pairs_local);
    }
}

// ---------------------------------------------------------------------------------
// host launcher
// ---------------------------------------------------------------------------------
template <int MAXK, int THREADS, int TPT, int T, bool MULTI>
static int launch_bin_impl(const PropArgs &a, int bin, int num_sms, cudaStream_t st) {
    auto kern = propagate_kernel<MAXK, THREADS, TPT, T, MULTI>;
    // TxT tiles read rows up to round_up(k, T) - 1: size the slab for that
    const int kmax = ((MAXK < a.cap ? MAXK : a.cap) + T - 1) / T * T;
    const int nq_total = (a.dim + 3) >> 2;
    const int rs4 = nq_total >= DC4 ? DC4 : ((nq_total + 7) & ~7);
    const size_t smem = align_up(sizeof(PropSmem<MAXK>), 128) + (size_t)kmax * rs4 * 16;
    static int configured_smem = 0;
    if ((int)smem > configured_smem) {
        GRNND_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured_smem = (int)smem;
    }
    int per_sm = 0;
    GRNND_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
    if (per_sm < 1) {
        set_error("propagate bin %d: no CTA fits (smem %zu B)", bin, smem);
        return GRNND_EUNSUPPORTED;
    }
    kern<<<num_sms * per_sm, THREADS, smem, st>>>(a, bin);
    return check_launch("propagate_kernel");
}

template <int MAXK, int THREADS, int TPT, int T>
static int launch_bin(const PropArgs &a, int bin, int num_sms, cudaStream_t st) {
    if (a.dim <= DC4 * 4) return launch_bin_impl<MAXK, THREADS, TPT, T, false>(a, bin, num_sms, st);
    return launch_bin_impl<MAXK, THREADS, TPT, T, true>(a, bin, num_sms, st);
}

int launch_propagate(const PropArgs &a, cudaStream_t st) {
    int dev = 0, num_sms = 0;
    GRNND_CUDA(cudaGetDevice(&dev));
    GRNND_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
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
    if (a.cap > 128) GRNND_TRY((launch_bin<256, 256, 3, 4>(a, 5, num_sms, st)));
    if (a.cap > 64) GRNND_TRY((launch_bin<128, 128, 3, 4>(a, 4, num_sms, st)));
    if (a.cap > 32) GRNND_TRY((launch_bin<64, 64, 3, 4>(a, 3, num_sms, st)));
    if (a.cap > 16) GRNND_TRY((launch_bin<32, 64, 3, 2>(a, 2, num_sms, st)));
    if (a.cap > 1) GRNND_TRY((launch_bin<16, 32, 2, 2>(a, 1, num_sms, st)));
    return GRNND_OK;
}

}  // namespace grnnd
