// apply.cu -- the pool insert (apply phase of a round).
//
// Reference: apply_grouped_messages (_numba_kernels.py:303-351) with the scalar spec
// cooperative_insert (builder.py:66-99): per target pool, messages in grouped order;
// (1) duplicate id -> skip, (2) free slot -> append at count, (3) full -> replace the
// farthest entry (first slot among equal maxima) if strictly closer, else reject.
//
// B200 design: one warp owns one target pool for the whole round, the pool row lives in
// registers (slot s -> lane s % 32, register s / 32), dedupe is one __ballot, the
// farthest-slot search a 5-step shuffle arg-max that is cached until the next replace.
// No global atomics touch pool data: a pool is written by exactly one warp.  The
// reference's global vertex-major message order per pool is reproduced exactly:
// incoming redirects are pre-sorted by (source, emission index) (group.cu) and the
// pool's own survivors are spliced in at source == target (update round) or after all
// incoming messages (reverse round: builder.py:325-336 applies reverse messages before
// the merge), without ever materialising survivor messages.
#include <climits>

#include "common.cuh"
#include "propagate.cuh"

namespace grnnd {

struct Outcome {
    unsigned long long ins = 0, dup = 0, rep = 0, rej = 0;
};

template <int RPL>
struct WarpPool {
    int32_t id[RPL];
    float d[RPL];
    int cnt;
    int cap;
    float mx;
    int mi;
    bool mxv;

    __device__ __forceinline__ void argmax() {
        const int lane = lane_id();
        float bd = -1.0f;  // reference starts at mx = -1.0 with strict '>' (:339-344)
        int bs = INT_MAX;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            const int s = r * 32 + lane;
            if (s < cap && d[r] > bd) {
                bd = d[r];
                bs = s;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float od = __shfl_xor_sync(FULL, bd, o);
            const int os = __shfl_xor_sync(FULL, bs, o);
            if (od > bd || (od == bd && os < bs)) {
                bd = od;
                bs = os;
            }
        }
        mx = bd;
        mi = bs;
        mxv = true;
    }

    __device__ __forceinline__ void insert(int32_t cid, float cd, Outcome &oc) {
        const int lane = lane_id();
        bool hit = false;
#pragma unroll
        for (int r = 0; r < RPL; ++r) hit |= (r * 32 + lane < cnt) && id[r] == cid;
        if (__any_sync(FULL, hit)) {
            ++oc.dup;
            return;
        }
        if (cnt < cap) {
#pragma unroll
            for (int r = 0; r < RPL; ++r)
                if (r * 32 + lane == cnt) {
                    id[r] = cid;
                    d[r] = cd;
                }
            ++cnt;
            ++oc.ins;
            mxv = false;
            return;
        }
        if (!mxv) argmax();
        if (cd < mx) {
#pragma unroll
            for (int r = 0; r < RPL; ++r)
                if (r * 32 + lane == mi) {
                    id[r] = cid;
                    d[r] = cd;
                }
            ++oc.rep;
            mxv = false;
        } else {
            ++oc.rej;
        }
    }

    __device__ __forceinline__ void store(int32_t *wi, float *wd) const {
        const int lane = lane_id();
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            const int s = r * 32 + lane;
            if (s < cnt) {
                wi[s] = id[r];
                wd[s] = d[r];
            }
        }
    }
};

// messages [b, e) of a sorted inbox, processed in order
template <int RPL>
__device__ __forceinline__ void apply_range(WarpPool<RPL> &P, const int32_t *__restrict__ iid,
                                            const float *__restrict__ idist, int64_t b, int64_t e, Outcome &oc) {
    const int lane = lane_id();
    for (int64_t c = b; c < e; c += 32) {
        const int nch = (int)(e - c < 32 ? e - c : 32);
        int32_t mid = 0;
        float md = 0.0f;
        if (lane < nch) {
            mid = iid[c + lane];
            md = idist[c + lane];
        }
        for (int j = 0; j < nch; ++j) {
            const int32_t cid = __shfl_sync(FULL, mid, j);
            const float cd = __shfl_sync(FULL, md, j);
            P.insert(cid, cd, oc);
        }
    }
}

// messages [b, e) of a sorted inbox, settled a chunk of 32 at a time while the pool has room:
// a message is a duplicate of the pool (one shuffle scan) or of an earlier message of its chunk
// (__match_any), else it is appended -- in order, as the sequential loop would; from the
// message that would overflow the pool on, the ordered insert() (replacement order matters)
template <int RPL>
__device__ __forceinline__ void apply_range_bulk(WarpPool<RPL> &P, const int32_t *__restrict__ iid,
                                                 const float *__restrict__ idist, int64_t b, int64_t e, Outcome &oc,
                                                 int32_t *s_id, float *s_d) {
    const int lane = lane_id();
    int64_t c = b;
    bool serial = false;
    for (; c < e && !serial; c += 32) {
        const int nch = (int)(e - c < 32 ? e - c : 32);
        const bool live = lane < nch;
        const int32_t x = live ? iid[c + lane] : -2 - lane;  // dead lanes: distinct non-ids
        const float xd = live ? idist[c + lane] : 0.0f;
        bool dup = false;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            const int lim = min(32, P.cnt - r * 32);  // warp-uniform
            for (int jj = 0; jj < lim; ++jj) dup |= __shfl_sync(FULL, P.id[r], jj) == x;
        }
        const unsigned peers = __match_any_sync(FULL, x);
        dup = live && (dup || (peers & ((1u << lane) - 1u)) != 0u);
        const unsigned addm = __ballot_sync(FULL, live && !dup), dupm = __ballot_sync(FULL, dup);
        const int room = P.cap - P.cnt;
        int nbulk = nch;
        if (__popc(addm) > room) {  // the (room+1)-th append overflows: bulk stops before it
            unsigned mm = addm;
            for (int t = 0; t < room; ++t) mm &= mm - 1u;
            nbulk = __ffs(mm) - 1;
            serial = true;
        }
        const unsigned pre = nbulk >= 32 ? 0xFFFFFFFFu : ((1u << nbulk) - 1u);
        const int nadd = __popc(addm & pre);
        if (lane < nbulk && live && !dup) {
            const int p = P.cnt + __popc(addm & ((1u << lane) - 1u));
            s_id[p] = x;
            s_d[p] = xd;
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            const int q = r * 32 + lane;
            if (q >= P.cnt && q < P.cnt + nadd) {
                P.id[r] = s_id[q];
                P.d[r] = s_d[q];
            }
        }
        __syncwarp();
        if (nadd) P.mxv = false;
        P.cnt += nadd;
        oc.ins += (unsigned long long)nadd;
        oc.dup += (unsigned long long)__popc(dupm & pre);
        for (int j = nbulk; j < nch; ++j)  // only after an overflow
            P.insert(__shfl_sync(FULL, x, j), __shfl_sync(FULL, xd, j), oc);
    }
    apply_range<RPL>(P, iid, idist, c, e, oc);  // the pool is full: the ordered insert
}

template <int RPL>
__global__ void __launch_bounds__(256) apply_round_kernel(ApplyArgs a) {
    __shared__ int32_t s_id[8][RPL * 32];
    __shared__ float s_d[8][RPL * 32];
    const int lane = lane_id(), wib = threadIdx.x >> 5;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int cap = a.cap;
    Outcome oc;
    unsigned long long own_total = 0;
    auto pool = [&](const int64_t t) {
        const int64_t tg = a.lo + t;
        const int64_t b = a.w.starts[t], e = a.w.starts[t + 1];
        // split point: messages from sources < tg come first (key = src * cap + j)
        int64_t split = e;
        if (!a.own_after_all) {
            // segment is sorted by key; first index with key >= tg * cap: 32 keys per coalesced
            // load and a ballot (a binary search was a chain of dependent global loads)
            const int64_t lim = tg * (int64_t)cap;
            split = e;
            for (int64_t c0 = b; c0 < e; c0 += 32) {
                const bool below = c0 + lane < e && a.w.i_key[c0 + lane] < lim;
                const unsigned bl = __ballot_sync(FULL, below);
                if (bl != FULL) {
                    split = c0 + __popc(bl);
                    break;
                }
            }
        }
        WarpPool<RPL> P;
        P.cnt = 0;
        P.cap = cap;
        P.mxv = false;
        apply_range_bulk<RPL>(P, a.w.i_id, a.w.i_dist, b, split, oc, s_id[wib], s_d[wib]);
        // own entries (survivors / merge) in slot order
        const int k = a.read_count[t];
        const int32_t *rid = a.read_ids + t * cap;
        const float *rd = a.read_dists + t * cap;
        if (P.cnt == 0) {
            // empty pool: own entries are distinct (pool invariant) -> plain ordered append
            int base = 0;
            for (int s0 = 0; s0 < k; s0 += 32) {
                const int s = s0 + lane;
                int32_t x = s < k ? rid[s] : TOMB;
                const bool live = x != TOMB;
                const unsigned bal = __ballot_sync(FULL, live);
                if (live) {
                    const int p = base + __popc(bal & ((1u << lane) - 1));
                    s_id[wib][p] = x;
                    s_d[wib][p] = rd[s];
                }
                base += __popc(bal);
            }
            __syncwarp();
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
                const int s = r * 32 + lane;
                if (s < base) {
                    P.id[r] = s_id[wib][s];
                    P.d[r] = s_d[wib][s];
                }
            }
            __syncwarp();
            P.cnt = base;
            oc.ins += (unsigned long long)base;
            own_total += (unsigned long long)base;
        } else {
            // Own entries after cnt0 messages from smaller sources.  Until the pool fills, an
            // own entry is either a duplicate of one of those messages (own entries are
            // distinct) or appended: a whole chunk is settled with ballots.  From the entry
            // that would overflow the pool on, the ordered insert() (replacement order).
            const int cnt0 = P.cnt;
            int s0 = 0;
            bool serial = false;
            for (; s0 < k && !serial; s0 += 32) {
                const int s = s0 + lane;
                const int32_t x = s < k ? rid[s] : TOMB;
                const float xd = s < k ? rd[s] : 0.0f;
                const int nch = min(32, k - s0);
                const bool live = x != TOMB;
                bool dup = false;
#pragma unroll
                for (int r = 0; r < RPL; ++r) {
                    const int lim = min(32, cnt0 - r * 32);  // warp-uniform
                    for (int jj = 0; jj < lim; ++jj) dup |= __shfl_sync(FULL, P.id[r], jj) == x;
                }
                dup = dup && live;
                const unsigned addm = __ballot_sync(FULL, live && !dup), dupm = __ballot_sync(FULL, dup),
                               livem = __ballot_sync(FULL, live);
                const int room = cap - P.cnt;
                int nbulk = nch;
                if (__popc(addm) > room) {  // the (room+1)-th append overflows: bulk stops before it
                    unsigned mm = addm;
                    for (int t = 0; t < room; ++t) mm &= mm - 1u;
                    nbulk = __ffs(mm) - 1;
                    serial = true;
                }
                const unsigned pre = nbulk >= 32 ? 0xFFFFFFFFu : ((1u << nbulk) - 1u);
                const int nadd = __popc(addm & pre);
                if (lane < nbulk && live && !dup) {
                    const int p = P.cnt + __popc(addm & ((1u << lane) - 1u));
                    s_id[wib][p] = x;
                    s_d[wib][p] = xd;
                }
                __syncwarp();
#pragma unroll
                for (int r = 0; r < RPL; ++r) {
                    const int q = r * 32 + lane;
                    if (q >= P.cnt && q < P.cnt + nadd) {
                        P.id[r] = s_id[wib][q];
                        P.d[r] = s_d[wib][q];
                    }
                }
                __syncwarp();
                if (nadd) P.mxv = false;
                P.cnt += nadd;
                oc.ins += (unsigned long long)nadd;
                oc.dup += (unsigned long long)__popc(dupm & pre);
                own_total += (unsigned long long)__popc(livem & pre);
                for (int j = nbulk; j < nch; ++j) {  // only after an overflow
                    const int32_t cid = __shfl_sync(FULL, x, j);
                    const float cd = __shfl_sync(FULL, xd, j);
                    if (cid != TOMB) {
                        P.insert(cid, cd, oc);
                        ++own_total;
                    }
                }
            }
            for (; s0 < k; s0 += 32) {
                const int s = s0 + lane;
                const int32_t x = s < k ? rid[s] : TOMB;
                const float xd = s < k ? rd[s] : 0.0f;
                const int nch = min(32, k - s0);
                for (int j = 0; j < nch; ++j) {
                    const int32_t cid = __shfl_sync(FULL, x, j);
                    const float cd = __shfl_sync(FULL, xd, j);
                    if (cid != TOMB) {
                        P.insert(cid, cd, oc);
                        ++own_total;
                    }
                }
            }
        }
        apply_range_bulk<RPL>(P, a.w.i_id, a.w.i_dist, split, e, oc, s_id[wib], s_d[wib]);
        __syncwarp();  // in place: every lane's reads of the row precede the stores
        P.store(a.write_ids + t * cap, a.write_dists + t * cap);
        if (lane == 0) {
            a.write_count[t] = P.cnt;
            if (a.in_place) a.w.dirty[t] = 0;
        }
    };
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (a.in_place) {
        // one pool buffer: a pool without incoming messages and without tombstones is its
        // own result (its entries re-inserted in slot order into an empty pool), so only the
        // others are rewritten; the lanes screen 32 pools at a time and the clean pools'
        // entries are counted as inserted survivors, as the reference counts them
        for (int64_t t0 = wid * 32; t0 < a.n; t0 += warps * 32) {
            const int64_t t = t0 + lane;
            bool work = false;
            unsigned long long kc = 0;
            if (t < a.n) {
                work = a.w.starts[t + 1] != a.w.starts[t] || a.w.dirty[t] != 0;
                if (!work) kc = (unsigned long long)a.read_count[t];
                // next update round's pair phase: only pools that changed, or whose pair phase
                // found a redirect-capable pair (dirty).  After an update round an unchanged,
                // clean pool ran a pair phase that found none (or was idle already); a reverse
                // round runs no pair phase, so it can only wake pools up
                if (work) a.w.idle[t] = 0;
                else if (!a.own_after_all) a.w.idle[t] = 1;
            }
            kc = warp_sum(kc);
            oc.ins += kc;
            own_total += kc;
            unsigned m = __ballot_sync(FULL, work);
            while (m) {
                const int l = __ffs(m) - 1;
                m &= m - 1u;
                pool(t0 + l);
            }
        }
    } else {
        for (int64_t t = wid; t < a.n; t += warps) {
            pool(t);
            if (lane == 0) a.w.idle[t] = 0;  // (two buffers: every pool rewritten)
        }
    }
    if (lane == 0 && a.stats) {
        unsigned long long *st = (unsigned long long *)a.stats;
        if (oc.ins) atomicAdd(&st[GRNND_ST_INSERTED], oc.ins);
        if (oc.dup) atomicAdd(&st[GRNND_ST_DUPLICATE], oc.dup);
        if (oc.rep) atomicAdd(&st[GRNND_ST_REPLACED], oc.rep);
        if (oc.rej) atomicAdd(&st[GRNND_ST_REJECTED], oc.rej);
        if (own_total) {
            atomicAdd(&st[GRNND_ST_SURVIVORS], own_total);
            if (a.own_after_all) atomicAdd(&st[GRNND_ST_MESSAGES], own_total);
        }
    }
}

// kernel-module apply_grouped_messages: messages through an explicit order, onto existing rows
template <int RPL>
__global__ void __launch_bounds__(256) apply_grouped_kernel(int32_t *__restrict__ write_ids, float *__restrict__ write_dists,
                                                            int32_t *__restrict__ write_count, int64_t n, int32_t cap,
                                                            const int32_t *__restrict__ flat_id,
                                                            const float *__restrict__ flat_dist,
                                                            const int64_t *__restrict__ order,
                                                            const int64_t *__restrict__ starts,
                                                            unsigned long long *__restrict__ outcomes) {
    const int lane = lane_id();
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    Outcome oc;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += warps) {
        const int64_t b = starts[t], e = starts[t + 1];
        if (b == e) continue;
        WarpPool<RPL> P;
        P.cap = cap;
        P.mxv = false;
        P.cnt = write_count[t];
        int32_t *wi = write_ids + t * cap;
        float *wd = write_dists + t * cap;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            const int s = r * 32 + lane;
            P.id[r] = s < cap ? wi[s] : TOMB;
            P.d[r] = s < cap ? wd[s] : 0.0f;
        }
        for (int64_t c = b; c < e; c += 32) {
            const int nch = (int)(e - c < 32 ? e - c : 32);
            int32_t mid = 0;
            float md = 0.0f;
            if (lane < nch) {
                const int64_t m = order[c + lane];
                mid = flat_id[m];
                md = flat_dist[m];
            }
            for (int j = 0; j < nch; ++j) P.insert(__shfl_sync(FULL, mid, j), __shfl_sync(FULL, md, j), oc);
        }
        P.store(wi, wd);
        if (lane == 0) write_count[t] = P.cnt;
    }
    if (lane == 0) {
        if (oc.ins) atomicAdd(&outcomes[0], oc.ins);
        if (oc.dup) atomicAdd(&outcomes[1], oc.dup);
        if (oc.rep) atomicAdd(&outcomes[2], oc.rep);
        if (oc.rej) atomicAdd(&outcomes[3], oc.rej);
    }
}



int launch_apply_round(const ApplyArgs &a, cudaStream_t st) {
    if (a.n <= 0) return GRNND_OK;
    const int64_t blocks = std::min<int64_t>((a.n + 7) / 8, (int64_t)device_sm_count() * 8);
    const unsigned g = (unsigned)std::max<int64_t>(1, blocks);
    switch ((a.cap + 31) / 32) {
        case 1: apply_round_kernel<1><<<g, 256, 0, st>>>(a); break;
        case 2: apply_round_kernel<2><<<g, 256, 0, st>>>(a); break;
        case 3: apply_round_kernel<3><<<g, 256, 0, st>>>(a); break;
        case 4: apply_round_kernel<4><<<g, 256, 0, st>>>(a); break;
        case 5: apply_round_kernel<5><<<g, 256, 0, st>>>(a); break;
        case 6: apply_round_kernel<6><<<g, 256, 0, st>>>(a); break;
        case 7: apply_round_kernel<7><<<g, 256, 0, st>>>(a); break;
        case 8: apply_round_kernel<8><<<g, 256, 0, st>>>(a); break;
        default: set_error("cap %d > %d unsupported", a.cap, GRNND_MAX_CAP); return GRNND_EUNSUPPORTED;
    }
    return check_launch("apply_round_kernel");
}

int launch_apply_grouped(int32_t *write_ids, float *write_dists, int32_t *write_count, int64_t n, int32_t cap,
                         const int32_t *flat_id, const float *flat_dist, const int64_t *order, const int64_t *starts,
                         int64_t *outcomes, cudaStream_t st) {
    if (n <= 0) return GRNND_OK;
    const int64_t blocks = std::min<int64_t>((n + 7) / 8, (int64_t)device_sm_count() * 8);
    const unsigned g = (unsigned)std::max<int64_t>(1, blocks);
    unsigned long long *oc = (unsigned long long *)outcomes;
    switch ((cap + 31) / 32) {
        case 1: apply_grouped_kernel<1><<<g, 256, 0, st>>>(write_ids, write_dists, write_count, n, cap, flat_id, flat_dist, order, starts, oc); break;
        case 2: apply_grouped_kernel<2><<<g, 256, 0, st>>>(write_ids, write_dists, write_count, n, cap, flat_id, flat_dist, order, starts, oc); break;
        case 3: apply_grouped_kernel<3><<<g, 256, 0, st>>>(write_ids, write_dists, write_count, n, cap, flat_id, flat_dist, order, starts, oc); break;
        case 4: apply_grouped_kernel<4><<<g, 256, 0, st>>>(write_ids, write_dists, write_count, n, cap, flat_id, flat_dist, order, starts, oc); break;
        case 5: apply_grouped_kernel<5><<<g, 256, 0, st>>>(write_ids, write_dists, write_count, n, cap, flat_id, flat_dist, order, starts, oc); break;
        case 6: apply_grouped_kernel<6><<<g, 256, 0, st>>>(write_ids, write_dists, write_count, n, cap, flat_id, flat_dist, order, starts, oc); break;
        case 7: apply_grouped_kernel<7><<<g, 256, 0, st>>>(write_ids, write_dists, write_count, n, cap, flat_id, flat_dist, order, starts, oc); break;
        case 8: apply_grouped_kernel<8><<<g, 256, 0, st>>>(write_ids, write_dists, write_count, n, cap, flat_id, flat_dist, order, starts, oc); break;
        default: set_error("cap %d > %d unsupported", cap, GRNND_MAX_CAP); return GRNND_EUNSUPPORTED;
    }
    return check_launch("apply_grouped_kernel");
}

}  // namespace grnnd
