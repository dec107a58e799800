// propagate.cu -- the pair phase of one GRNND update round (the hot kernel).
//
// Reference: gen_update_messages, /root/reference/pkg/src/grnnd/_numba_kernels.py:125-192
// (with _fill_perm :64-88, _hash4 :36-41, _sqdist :50-56).  Per vertex v with k live
// pool entries: visit all pairs in a hash-driven Fisher-Yates order; a pair whose
// mutual distance is strictly below the larger stored distance redirects the farther
// member toward the closer one (tombstoning it); survivors stay.
//
// B200 design:
//  * vertices are binned by k; each bin runs a persistent kernel whose CTA processes
//    one vertex at a time with a CTA size / shared-memory slab matched to the bin;
//  * the k pool rows are gathered HBM -> smem with cp.async (16 B, L2-only), row-major
//    with a 16-byte XOR swizzle so the register-tiled reads below are conflict free;
//  * ALL pair distances of the pool (upper triangle, slot order) are computed with
//    4x4 register tiles in the reference's exact arithmetic (sequential fp32
//    sub/mul/add, no FMA) -> bit-identical distances to the numba oracle;
//  * the order-dependent part (anchor-serial rule, SURVEY 7 hard part 1) is then a
//    cheap pass over 64-bit masks: cond[x] (pair redirects) and afar[x] (anchor is the
//    farther one), both indexed by permutation position;
//  * emitted messages get their distance re-evaluated exactly from L2-resident rows
//    (only ~10% of entries are redirected), keeping the big distance matrix out of smem.
#include <cstdio>

#include "common.cuh"
#include "propagate.cuh"

namespace grnnd {

// bin b covers k in (BIN_HI[b-1], BIN_HI[b]]; bin 0 = k <= 1 (no pairs)
__host__ __device__ constexpr int bin_hi(int b) {
    return b == 0 ? 1 : b == 1 ? 16 : b == 2 ? 32 : b == 3 ? 64 : b == 4 ? 128 : 256;
}
__device__ __forceinline__ int bin_of(int k) {
    return k <= 1 ? 0 : k <= 16 ? 1 : k <= 32 ? 2 : k <= 64 ? 3 : k <= 128 ? 4 : 5;
}

constexpr int DC4 = 32;  // float4 per row chunk (128 dims)

// ---------------------------------------------------------------------------------
// binning: one pass over read_count; bin lists + sum(k) into stats
// ---------------------------------------------------------------------------------
__global__ void bin_kernel(const int32_t *__restrict__ read_count, int64_t n, int32_t cap,
                           Workspace w, int64_t *__restrict__ stats, int slice_mode,
                           const int32_t *__restrict__ read_ids,
                           const float *__restrict__ read_dists, int64_t lo,
                           int32_t *__restrict__ msg_tgt, int32_t *__restrict__ msg_id,
                           float *__restrict__ msg_dist, int32_t *__restrict__ msg_cnt) {
    __shared__ unsigned long long s_sum;
    if (threadIdx.x == 0) s_sum = 0;
    __syncthreads();
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int k = 0;
    if (v < n) {
        k = read_count[v];
        int b = bin_of(k);
        if (b > 0) {
            unsigned peers = __match_any_sync(__activemask(), b);
            int leader = __ffs(peers) - 1;
            unsigned long long base = 0;
            if (lane_id() == leader) base = atomicAdd(&w.ctr[C_BIN0 + b], (unsigned long long)__popc(peers));
            base = __shfl_sync(peers, base, leader);
            int rank = __popc(peers & ((1u << lane_id()) - 1));
            w.bins[(int64_t)b * w.n + (int64_t)base + rank] = (int32_t)v;
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
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::);
}

// row r, float4 column q -> swizzled float4 index (conflict-free 4x4 tile reads)
__device__ __forceinline__ int swz(int r, int q, int rs4) { return r * rs4 + (q ^ ((r >> 2) & 7)); }

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
    uint32_t fyj[MAXK];  // Fisher-Yates partner for position i
    int16_t e_tgt[MAXK];  // emitted message j: target slot
    int16_t e_id[MAXK];   // emitted message j: id slot
    int nmsg;
    int vertex;
    unsigned long long list_base;
    unsigned long long ref_pairs;
};

template <int MAXK, int THREADS, int TPT>
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
    const int cap = a.cap;
    unsigned long long pairs_local = 0;

    for (int64_t it = blockIdx.x; it < nbin; it += gridDim.x) {
        const int64_t v = blist[it];  // local row
        const int64_t vg = a.lo + v;  // global vertex id
        const int k = a.read_count[v];
        const int32_t *rid = a.read_ids + v * cap;
        const float *rdv = a.read_dists + v * cap;

        // ---- 1. pool row, permutation partners, bitset reset ----
        const uint64_t pre = vertex_prefix(a.seed, a.stream_id, (uint64_t)vg);
        for (int s = tid; s < k; s += THREADS) {
            sm.ids[s] = rid[s];
            sm.dv[s] = rdv[s];
            sm.perm[s] = s;
            if (a.order_code == 0 && s > 0) sm.fyj[s] = (uint32_t)(mix64(pre ^ (uint64_t)s) % (uint64_t)(s + 1));
        }
        for (int i = tid; i < k * W; i += THREADS) {
            sm.cond[i] = 0ull;
            sm.afar[i] = 0ull;
        }
        __syncthreads();

        // ---- 2. gather the first row chunk (overlaps the serial permutation below) ----
        const int nchunks = (nq_total + DC4 - 1) / DC4;
        auto load_chunk = [&](int c) {
            const int q0 = c * DC4;
            const int nq = min(DC4, nq_total - q0);
            const int total = k * nq;
            for (int e = tid; e < total; e += THREADS) {
                const int r = e / nq;
                const int q = e - r * nq;
                const int32_t id = sm.ids[r];
                const float *src = a.data + (int64_t)(id < 0 ? 0 : id) * a.ld + (int64_t)(q0 + q) * 4;
                cp_async16(&rows[swz(r, q, rs4)], src, id >= 0);
            }
            asm volatile("cp.async.commit_group;\n" ::);
        };
        load_chunk(0);

        if (a.order_code == 0) {
            // hash-driven Fisher-Yates (_numba_kernels.py:70-74): serial, one thread
            if (tid == 0) {
                for (int i = k - 1; i > 0; --i) {
                    int j = (int)sm.fyj[i];
                    int t = sm.perm[i];
                    sm.perm[i] = sm.perm[j];
                    sm.perm[j] = t;
                }
            }
        } else {
            // ascending debug order (:75-87): stable rank by (dist, id)
            for (int s = tid; s < k; s += THREADS) {
                float ds = sm.dv[s];
                int32_t is = sm.ids[s];
                int r = 0;
                for (int t = 0; t < k; ++t) {
                    float dt = sm.dv[t];
                    int32_t it2 = sm.ids[t];
                    r += (dt < ds || (dt == ds && (it2 < is || (it2 == is && t < s)))) ? 1 : 0;
                }
                sm.pos[s] = r;
            }
            __syncthreads();
            for (int s = tid; s < k; s += THREADS) sm.perm[sm.pos[s]] = s;
        }
        __syncthreads();
        for (int x = tid; x < k; x += THREADS) sm.pos[sm.perm[x]] = x;
        if (tid < W) {
            uint64_t m = 0;
            for (int b = 0; b < 64; ++b) {
                int x = tid * 64 + b;
                if (x < k && sm.ids[sm.perm[x]] != TOMB) m |= 1ull << b;
            }
            sm.live[tid] = m;
        }

        // ---- 3. all-pairs exact distances, 4x4 register tiles, upper triangle ----
        const int nb = (k + 3) >> 2;
        const int ntiles = nb * (nb + 1) / 2;
        for (int g0 = 0; g0 < ntiles; g0 += THREADS * TPT) {
            float acc[TPT][16];
#pragma unroll
            for (int tt = 0; tt < TPT; ++tt)
#pragma unroll
                for (int p = 0; p < 16; ++p) acc[tt][p] = 0.0f;
            for (int c = 0; c < nchunks; ++c) {
                if (nchunks > 1 && (c > 0 || g0 > 0)) {
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
                        const int rA = bI * 4, rB = bJ * 4;
#pragma unroll 2
                        for (int q = 0; q < nq; ++q) {
                            float4 A[4], B[4];
#pragma unroll
                            for (int i = 0; i < 4; ++i) A[i] = rows[swz(rA + i, q, rs4)];
#pragma unroll
                            for (int j = 0; j < 4; ++j) B[j] = rows[swz(rB + j, q, rs4)];
#pragma unroll
                            for (int i = 0; i < 4; ++i)
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    float s = acc[tt][i * 4 + j];
                                    s = exact_step(s, A[i].x, B[j].x);
                                    s = exact_step(s, A[i].y, B[j].y);
                                    s = exact_step(s, A[i].z, B[j].z);
                                    s = exact_step(s, A[i].w, B[j].w);
                                    acc[tt][i * 4 + j] = s;
                                }
                        }
                    }
                }
            }
            // epilogue: redirect condition per pair, as bits in permutation-position space
#pragma unroll
            for (int tt = 0; tt < TPT; ++tt) {
                const int t = g0 + tt * THREADS + tid;
                if (t < ntiles) {
                    int bI, bJ;
                    tile_decode(t, bI, bJ);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int s = bI * 4 + i, u = bJ * 4 + j;
                            if (s < u && u < k && sm.ids[s] != TOMB && sm.ids[u] != TOMB) {
                                ++pairs_local;
                                const float d1 = sm.dv[s], d2 = sm.dv[u];
                                const float hi = d1 >= d2 ? d1 : d2;
                                if (acc[tt][i * 4 + j] < hi) {
                                    const int x1 = sm.pos[s], x2 = sm.pos[u];
                                    // anchor = the member visited first (smaller position)
                                    const int xa = x1 < x2 ? x1 : x2, xb = x1 < x2 ? x2 : x1;
                                    const float dva = x1 < x2 ? d1 : d2, dvb = x1 < x2 ? d2 : d1;
                                    const uint64_t bit = 1ull << (xb & 63);
                                    atomicOr((unsigned long long *)&sm.cond[xa * W + (xb >> 6)], bit);
                                    if (!(dvb >= dva)) atomicOr((unsigned long long *)&sm.afar[xa * W + (xb >> 6)], bit);
                                }
                            }
                        }
                }
            }
        }
        __syncthreads();

        // ---- 4. anchor-serial decision over the masks (one thread) ----
        if (tid == 0) {
            uint64_t live[W];
#pragma unroll
            for (int i = 0; i < W; ++i) live[i] = sm.live[i];
            int nm = 0;
            unsigned long long refp = 0;
            for (int x = 0; x < k - 1; ++x) {
                if (!((live[x >> 6] >> (x & 63)) & 1ull)) continue;
                // first partner that makes the anchor the farther one
                int f = k;
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    uint64_t m = sm.afar[x * W + i] & live[i];
                    if (m && f == k) f = i * 64 + __ffsll((long long)m) - 1;
                }
                // visited partners: live, position in (x, f]  (reference-semantics pair count)
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    uint64_t m = live[i];
                    int lo_b = x + 1 - i * 64, hi_b = (f < k ? f : k - 1) - i * 64;
                    if (hi_b < 0 || lo_b > 63) continue;
                    if (lo_b > 0) m &= ~0ull << lo_b;
                    if (hi_b < 63) m &= (2ull << hi_b) - 1ull;
                    refp += __popcll(m);
                }
                const int sa = sm.perm[x];
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    uint64_t m = sm.cond[x * W + i] & live[i];
                    int hb = f - i * 64;  // keep bits < f
                    if (hb <= 0) m = 0;
                    else if (hb < 64) m &= (1ull << hb) - 1ull;
                    uint64_t em = m & ~sm.afar[x * W + i];
                    while (em) {
                        int b = __ffsll((long long)em) - 1;
                        em &= em - 1;
                        int y = i * 64 + b;
                        sm.e_tgt[nm] = (int16_t)sa;
                        sm.e_id[nm] = (int16_t)sm.perm[y];
                        ++nm;
                        live[i] &= ~(1ull << b);
                    }
                }
                if (f < k) {
                    sm.e_tgt[nm] = (int16_t)sm.perm[f];
                    sm.e_id[nm] = (int16_t)sa;
                    ++nm;
                    live[x >> 6] &= ~(1ull << (x & 63));
                }
            }
            sm.nmsg = nm;
            sm.ref_pairs = refp;
#pragma unroll
            for (int i = 0; i < W; ++i) sm.live[i] = live[i];
            if (!a.slice_mode && nm > 0) sm.list_base = atomicAdd(&a.w.ctr[C_LIST], (unsigned long long)nm);
        }
        __syncthreads();

        // ---- 5. emit redirects (exact distance re-evaluated from L2-resident rows) ----
        const int nm = sm.nmsg;
        for (int j = tid; j < nm; j += THREADS) {
            const int32_t tgt = sm.ids[sm.e_tgt[j]];
            const int32_t id = sm.ids[sm.e_id[j]];
            const float d = exact_sqdist_global(a.data + (int64_t)tgt * a.ld, a.data + (int64_t)id * a.ld, a.dim);
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
        if (a.slice_mode) {
            // survivors in slot order after the redirects (:186-191)
            if (tid < 32) {
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
template <int MAXK, int THREADS, int TPT>
static int launch_bin(const PropArgs &a, int bin, int num_sms, cudaStream_t st) {
    auto kern = propagate_kernel<MAXK, THREADS, TPT>;
    const int kmax = MAXK < a.cap ? MAXK : a.cap;
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

int launch_propagate(const PropArgs &a, cudaStream_t st) {
    int dev = 0, num_sms = 0;
    GRNND_CUDA(cudaGetDevice(&dev));
    GRNND_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t n = a.hi - a.lo;
    if (n <= 0) return GRNND_OK;
    // counters: bins
    GRNND_CUDA(cudaMemsetAsync(a.w.ctr + C_BIN0, 0, sizeof(unsigned long long) * NBINS, st));
    const int tb = 256;
    bin_kernel<<<(unsigned)((n + tb - 1) / tb), tb, 0, st>>>(
        a.read_count, n, a.cap, a.w, a.stats, a.slice_mode, a.read_ids, a.read_dists, a.lo,
        a.msg_tgt, a.msg_id, a.msg_dist, a.msg_cnt);
    GRNND_TRY(check_launch("bin_kernel"));
    // largest k first so long CTAs start early
    if (a.cap > 128) GRNND_TRY((launch_bin<256, 256, 3>(a, 5, num_sms, st)));
    if (a.cap > 64) GRNND_TRY((launch_bin<128, 256, 3>(a, 4, num_sms, st)));
    if (a.cap > 32) GRNND_TRY((launch_bin<64, 128, 2>(a, 3, num_sms, st)));
    if (a.cap > 16) GRNND_TRY((launch_bin<32, 64, 1>(a, 2, num_sms, st)));
    if (a.cap > 1) GRNND_TRY((launch_bin<16, 32, 1>(a, 1, num_sms, st)));
    return GRNND_OK;
}

}  // namespace grnnd
