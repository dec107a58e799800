// group.cu -- grouping of a round's messages by target pool.
//
// Reference: build_flat + group_by_target (_numba_kernels.py:253-300): a stable counting
// sort of the vertex-major message stream by target.  The B200 path reaches the same
// per-pool order without a serial pass: messages carry a global order key
// (source * cap + emission index), are counted and scattered per target with atomics
// (arbitrary order), and each target's segment is then sorted by key -- a warp register
// sort for the common short segments, a CTA shared-memory bitonic sort for hubs.
#include <climits>

#include "common.cuh"
#include "propagate.cuh"

namespace grnnd {

// ---------------------------------------------------------------------------------
// exclusive scan int32 counts[n] -> int64 out[n+1] (reduce-then-scan, 3 launches)
// ---------------------------------------------------------------------------------
constexpr int SCAN_T = 256;
constexpr int SCAN_V = SCAN_ITEMS / SCAN_T;  // 8 items per thread

__device__ __forceinline__ int64_t block_excl_scan(int64_t x, int64_t *s_warp, int64_t &total) {
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    int64_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int64_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
        int64_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(FULL, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < (int)(blockDim.x >> 5)) s_warp[lane] = wi - w;
        if (lane == 31) s_warp[32] = wi;
    }
    __syncthreads();
    total = s_warp[32];
    int64_t r = s_warp[wid] + inc - x;
    __syncthreads();
    return r;
}

__global__ void scan_reduce_kernel(const int32_t *__restrict__ in, int64_t n, int64_t *__restrict__ tmp) {
    __shared__ int64_t s_warp[33];
    const int64_t base = (int64_t)blockIdx.x * SCAN_ITEMS + (int64_t)threadIdx.x * SCAN_V;
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_V; ++i)
        if (base + i < n) s += in[base + i];
    int64_t total;
    block_excl_scan(s, s_warp, total);
    if (threadIdx.x == 0) tmp[blockIdx.x] = total;
}

__global__ void scan_top_kernel(int64_t *__restrict__ tmp, int64_t nb) {
    __shared__ int64_t s_warp[33];
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += blockDim.x) {
        const int64_t i = b0 + threadIdx.x;
        int64_t x = i < nb ? tmp[i] : 0;
        int64_t total;
        int64_t e = block_excl_scan(x, s_warp, total);
        if (i < nb) tmp[i] = carry + e;
        carry += total;
    }
    if (threadIdx.x == 0) tmp[nb] = carry;
}

__global__ void scan_down_kernel(const int32_t *__restrict__ in, int64_t n, const int64_t *__restrict__ tmp,
                                 int64_t *__restrict__ out, int64_t nb, unsigned long long *heavy_ctr,
                                 int32_t *heavy_list) {
    __shared__ int64_t s_warp[33];
    const int64_t base = (int64_t)blockIdx.x * SCAN_ITEMS + (int64_t)threadIdx.x * SCAN_V;
    int32_t v[SCAN_V];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_V; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        s += v[i];
    }
    int64_t total;
    int64_t e = block_excl_scan(s, s_warp, total) + tmp[blockIdx.x];
#pragma unroll
    for (int i = 0; i < SCAN_V; ++i) {
        if (base + i < n) {
            out[base + i] = e;
            if (heavy_list && v[i] > HEAVY_SEG) {
                unsigned long long p = atomicAdd(heavy_ctr, 1ull);
                heavy_list[p] = (int32_t)(base + i);
            }
        }
        e += v[i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = tmp[nb];
}

static int scan_impl(const int32_t *counts, int64_t n, int64_t *out, int64_t *tmp,
                     unsigned long long *heavy_ctr, int32_t *heavy_list, cudaStream_t st) {
    const int64_t nb = scan_blocks(n);
    if (n <= 0) {
        GRNND_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
        return GRNND_OK;
    }
    scan_reduce_kernel<<<(unsigned)nb, SCAN_T, 0, st>>>(counts, n, tmp);
    scan_top_kernel<<<1, 1024, 0, st>>>(tmp, nb);
    scan_down_kernel<<<(unsigned)nb, SCAN_T, 0, st>>>(counts, n, tmp, out, nb, heavy_ctr, heavy_list);
    return check_launch("scan", 3);
}

int launch_scan_counts(const int32_t *counts, int64_t n, int64_t *out, int64_t *tmp, cudaStream_t st) {
    return scan_impl(counts, n, out, tmp, nullptr, nullptr, st);
}

// ---------------------------------------------------------------------------------
// count + scatter into target segments
// ---------------------------------------------------------------------------------
__device__ __forceinline__ int64_t msg_count(const unsigned long long *m_dev, int64_t m_host, int64_t cap) {
    if (!m_dev) return m_host;
    const unsigned long long m = *m_dev;
    return m < (unsigned long long)cap ? (int64_t)m : cap;
}

__global__ void count_targets_kernel(const int32_t *__restrict__ tgt, const unsigned long long *m_dev, int64_t m_host,
                                     int64_t lo, int32_t *__restrict__ cnt) {
    const int64_t m = msg_count(m_dev, m_host, m_host);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[tgt[i] - lo], 1);
}

__global__ void scatter_kernel(const int64_t *__restrict__ key, const int32_t *__restrict__ tgt,
                               const int32_t *__restrict__ id, const float *__restrict__ dist,
                               const unsigned long long *m_dev, int64_t m_host, int64_t lo, int32_t *__restrict__ cnt, const int64_t *__restrict__ starts,
                               int64_t *__restrict__ okey, int32_t *__restrict__ oid, float *__restrict__ odist) {
    const int64_t m = msg_count(m_dev, m_host, m_host);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = tgt[i] - lo;
        const int p = atomicSub(&cnt[t], 1) - 1;  // leaves cnt at 0 for the next round
        const int64_t o = starts[t] + p;
        okey[o] = key ? key[i] : (int64_t)i;
        oid[o] = id ? id[i] : 0;
        odist[o] = dist ? dist[i] : 0.0f;
    }
}

// ---------------------------------------------------------------------------------
// per-segment sort by key
// ---------------------------------------------------------------------------------
// light: a warp scans 32 consecutive targets, sorts each 2..32 segment in registers
__global__ void segsort_light_kernel(const int64_t *__restrict__ starts, int64_t n, int64_t *__restrict__ key,
                                     int32_t *__restrict__ id, float *__restrict__ dist) {
    const int lane = lane_id();
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; t0 < n; t0 += warps * 32) {
        const int64_t t = t0 + lane;
        int64_t b = 0, len = 0;
        if (t < n) {
            b = starts[t];
            len = starts[t + 1] - b;
        }
        unsigned todo = __ballot_sync(FULL, len >= 2 && len <= HEAVY_SEG);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const int64_t sb = __shfl_sync(FULL, b, src);
            const int sl = (int)__shfl_sync(FULL, len, src);
            int64_t kk = LLONG_MAX;
            int32_t ii = 0;
            float dd = 0.0f;
            if (lane < sl) {
                kk = key[sb + lane];
                ii = id[sb + lane];
                dd = dist[sb + lane];
            }
            int r = 0;
            for (int j = 0; j < sl; ++j) {
                const int64_t kj = __shfl_sync(FULL, kk, j);
                r += kj < kk ? 1 : 0;
            }
            if (lane < sl) {
                key[sb + r] = kk;
                id[sb + r] = ii;
                dist[sb + r] = dd;
            }
            __syncwarp();
        }
    }
}

constexpr int HEAVY_CAP = 8192;
constexpr int HEAVY_T = 512;
constexpr int MEDIUM_CAP = 256;  // segments of 33..256 messages: one warp each (rank sort)
constexpr int MEDIUM_WARPS = 8;

// medium: warp per segment of HEAVY_SEG < len <= MEDIUM_CAP; keys are unique, so each
// message's rank is the number of smaller keys (keys staged in shared memory)
__global__ void __launch_bounds__(MEDIUM_WARPS * 32) segsort_medium_kernel(const int64_t *__restrict__ starts,
                                                                         const int32_t *__restrict__ heavy,
                                                                         const unsigned long long *__restrict__ heavy_ctr,
                                                                         int64_t *__restrict__ key, int32_t *__restrict__ id,
                                                                         float *__restrict__ dist) {
    __shared__ int64_t sk[MEDIUM_WARPS][MEDIUM_CAP];
    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int64_t nh = (int64_t)*heavy_ctr;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t h = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; h < nh; h += warps) {
        const int64_t t = heavy[h];
        const int64_t b = starts[t];
        const int len = (int)(starts[t + 1] - b);
        if (len > MEDIUM_CAP) continue;  // the CTA kernel takes it
        constexpr int PER = MEDIUM_CAP / 32;
        int64_t k[PER];
        int32_t ii[PER];
        float dd[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = lane + 32 * j;
            if (i < len) {
                k[j] = key[b + i];
                ii[j] = id[b + i];
                dd[j] = dist[b + i];
                sk[w][i] = k[j];
            }
        }
        __syncwarp();
        int r[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) r[j] = 0;
        for (int t2 = 0; t2 < len; ++t2) {
            const int64_t kt = sk[w][t2];
#pragma unroll
            for (int j = 0; j < PER; ++j) r[j] += kt < k[j] ? 1 : 0;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = lane + 32 * j;
            if (i < len) {
                key[b + r[j]] = k[j];
                id[b + r[j]] = ii[j];
                dist[b + r[j]] = dd[j];
            }
        }
        __syncwarp();
    }
}

// heavy: one CTA per long segment; bitonic sort of (key, index) in smem
__global__ void __launch_bounds__(HEAVY_T) segsort_heavy_kernel(const int64_t *__restrict__ starts,
                                                                const int32_t *__restrict__ heavy,
                                                                const unsigned long long *__restrict__ heavy_ctr,
                                                                int64_t *__restrict__ key, int32_t *__restrict__ id,
                                                                float *__restrict__ dist, int64_t *__restrict__ tkey,
                                                                int32_t *__restrict__ tid_, float *__restrict__ tdist) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int64_t *sk = reinterpret_cast<int64_t *>(smem_raw);
    int32_t *sid = reinterpret_cast<int32_t *>(sk + HEAVY_CAP);
    float *sd = reinterpret_cast<float *>(sid + HEAVY_CAP);
    uint16_t *sx = reinterpret_cast<uint16_t *>(sd + HEAVY_CAP);
    const int64_t nh = (int64_t)*heavy_ctr;
    for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const int64_t t = heavy[h];
        const int64_t b = starts[t];
        const int64_t len = starts[t + 1] - b;
        if (len <= MEDIUM_CAP) continue;  // sorted by segsort_medium_kernel
        if (len <= HEAVY_CAP) {
            int P = 1;
            while (P < len) P <<= 1;
            for (int i = threadIdx.x; i < P; i += HEAVY_T) {
                if (i < len) {
                    sk[i] = key[b + i];
                    sid[i] = id[b + i];
                    sd[i] = dist[b + i];
                } else {
                    sk[i] = LLONG_MAX;
                }
                sx[i] = (uint16_t)i;
            }
            __syncthreads();
            for (int size = 2; size <= P; size <<= 1) {
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    for (int i = threadIdx.x; i < P / 2; i += HEAVY_T) {
                        const int lo = 2 * i - (i & (stride - 1));
                        const int hi = lo + stride;
                        const bool up = (lo & size) == 0;
                        const int64_t a = sk[lo], c = sk[hi];
                        if ((a > c) == up) {
                            sk[lo] = c;
                            sk[hi] = a;
                            const uint16_t x = sx[lo];
                            sx[lo] = sx[hi];
                            sx[hi] = x;
                        }
                    }
                    __syncthreads();
                }
            }
            for (int i = threadIdx.x; i < len; i += HEAVY_T) {
                key[b + i] = sk[i];
                id[b + i] = sid[sx[i]];
                dist[b + i] = sd[sx[i]];
            }
            __syncthreads();
        } else {
            // rare fallback: rank by counting (keys are unique), via the scratch lists
            for (int64_t i = threadIdx.x; i < len; i += HEAVY_T) {
                const int64_t ki = key[b + i];
                int64_t r = 0;
                for (int64_t j = 0; j < len; ++j) r += key[b + j] < ki ? 1 : 0;
                tkey[b + r] = ki;
                tid_[b + r] = id[b + i];
                tdist[b + r] = dist[b + i];
            }
            __syncthreads();
            for (int64_t i = threadIdx.x; i < len; i += HEAVY_T) {
                key[b + i] = tkey[b + i];
                id[b + i] = tid_[b + i];
                dist[b + i] = tdist[b + i];
            }
            __syncthreads();
        }
    }
}


int launch_segsort(const Workspace &w, int64_t n, int64_t *key, int32_t *id, float *dist, cudaStream_t st) {
    const int sms = device_sm_count();
    const int64_t warps_needed = (n + 31) / 32;
    const int64_t blocks = std::min<int64_t>((warps_needed + 7) / 8, (int64_t)sms * 16);
    segsort_light_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, st>>>(w.starts, n, key, id, dist);
    GRNND_TRY(check_launch("segsort_light"));
    const size_t smem = (size_t)HEAVY_CAP * (8 + 4 + 4 + 2);
    static SmemOptIn optin;
    GRNND_CUDA(optin.ensure(segsort_heavy_kernel, smem));
    segsort_medium_kernel<<<sms * 8, MEDIUM_WARPS * 32, 0, st>>>(w.starts, w.heavy, w.ctr + C_HEAVY, key, id, dist);
    GRNND_TRY(check_launch("segsort_medium"));
    segsort_heavy_kernel<<<sms, HEAVY_T, smem, st>>>(w.starts, w.heavy, w.ctr + C_HEAVY, key, id, dist, w.h_key,
                                                     w.h_id, w.h_dist);
    return check_launch("segsort_heavy");
}

// emitted list (key, tgt, id, dist)[m] -> inbox segments sorted by key
// m_dev (device counter, clamped to m_host) or m_host when m_dev is null
int launch_group_inbox(const Workspace &w, const int64_t *key, const int32_t *tgt, const int32_t *id,
                       const float *dist, const unsigned long long *m_dev, int64_t m_host, int64_t lo, int64_t n,
                       cudaStream_t st) {
    const int64_t m = m_host;
    const int sms = device_sm_count();
    GRNND_CUDA(cudaMemsetAsync(w.in_count, 0, sizeof(int32_t) * (size_t)(n + 1), st));
    GRNND_CUDA(cudaMemsetAsync(w.ctr + C_HEAVY, 0, sizeof(unsigned long long), st));
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, (int64_t)sms * 8));
    if (m > 0) {
        count_targets_kernel<<<g, 256, 0, st>>>(tgt, m_dev, m, lo, w.in_count);
        GRNND_TRY(check_launch("count_targets"));
    }
    GRNND_TRY(scan_impl(w.in_count, n, w.starts, w.scan_tmp, w.ctr + C_HEAVY, w.heavy, st));
    if (m > 0) {
        scatter_kernel<<<g, 256, 0, st>>>(key, tgt, id, dist, m_dev, m, lo, w.in_count, w.starts, w.i_key, w.i_id, w.i_dist);
        GRNND_TRY(check_launch("scatter"));
    }
    return launch_segsort(w, n, w.i_key, w.i_id, w.i_dist, st);
}

// ---------------------------------------------------------------------------------
// kernel-module build_flat/_compact (:253-262): slices -> flat arrays, vertex-major
// ---------------------------------------------------------------------------------
__global__ void compact_kernel(const int32_t *__restrict__ mt, const int32_t *__restrict__ mi,
                               const float *__restrict__ md, const int32_t *__restrict__ mc, int64_t n,
                               int32_t cap, const int64_t *__restrict__ offs, int32_t *__restrict__ ft,
                               int32_t *__restrict__ fi, float *__restrict__ fd, int32_t *__restrict__ fs) {
    const int lane = lane_id();
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
        const int c = mc[v];
        const int64_t o = offs[v];
        for (int i = lane; i < c; i += 32) {
            ft[o + i] = mt[v * cap + i];
            fi[o + i] = mi[v * cap + i];
            fd[o + i] = md[v * cap + i];
            if (fs) fs[o + i] = (int32_t)v;
        }
    }
}

int launch_compact(const int32_t *msg_tgt, const int32_t *msg_id, const float *msg_dist, const int32_t *msg_cnt,
                   int64_t n, int32_t cap, const int64_t *offs, int32_t *flat_tgt, int32_t *flat_id,
                   float *flat_dist, int32_t *flat_src, cudaStream_t st) {
    if (n <= 0) return GRNND_OK;
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, (int64_t)device_sm_count() * 16));
    compact_kernel<<<g, 256, 0, st>>>(msg_tgt, msg_id, msg_dist, msg_cnt, n, cap, offs, flat_tgt, flat_id,
                                      flat_dist, flat_src);
    return check_launch("compact_kernel");
}

// ---------------------------------------------------------------------------------
// multi-GPU: bucket the emitted list by owner rank (contiguous id ranges)
// ---------------------------------------------------------------------------------
constexpr int MAX_RANKS = 64;

__device__ __forceinline__ int owner_of(int64_t t, const int64_t *rb, int nranks) {
    int r = 0;
    while (r + 1 < nranks && t >= rb[r + 1]) ++r;
    return r;
}

__global__ void rank_count_kernel(const Workspace w, const int64_t *__restrict__ rb, int nranks,
                                  unsigned long long *__restrict__ rc) {
    __shared__ unsigned long long s_c[MAX_RANKS];
    for (int i = threadIdx.x; i < nranks; i += blockDim.x) s_c[i] = 0;
    __syncthreads();
    const unsigned long long mm = *(w.ctr + C_LIST);
    const int64_t m = mm < (unsigned long long)w.msg_capacity ? (int64_t)mm : w.msg_capacity;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&s_c[owner_of(w.e_tgt[i], rb, nranks)], 1ull);
    __syncthreads();
    for (int i = threadIdx.x; i < nranks; i += blockDim.x)
        if (s_c[i]) atomicAdd(&rc[i], s_c[i]);
}

__global__ void rank_offsets_kernel(const unsigned long long *__restrict__ rc, int nranks,
                                    unsigned long long *__restrict__ cursor, int64_t *__restrict__ send_counts) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        unsigned long long o = 0;
        for (int r = 0; r < nranks; ++r) {
            cursor[r] = o;
            send_counts[r] = (int64_t)rc[r];
            o += rc[r];
        }
    }
}

__global__ void rank_scatter_kernel(const Workspace w, const int64_t *__restrict__ rb, int nranks,
                                    unsigned long long *__restrict__ cursor) {
    const unsigned long long mm = *(w.ctr + C_LIST);
    const int64_t m = mm < (unsigned long long)w.msg_capacity ? (int64_t)mm : w.msg_capacity;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = owner_of(w.e_tgt[i], rb, nranks);
        const unsigned long long p = atomicAdd(&cursor[r], 1ull);
        const int64_t key = w.e_key[i];
        int32_t *o = w.o_pack + p * MSG_WORDS;
        o[0] = (int32_t)(uint32_t)(uint64_t)key;
        o[1] = (int32_t)(uint32_t)((uint64_t)key >> 32);
        o[2] = w.e_tgt[i];
        o[3] = w.e_id[i];
        o[4] = __float_as_int(w.e_dist[i]);
    }
}

// received packed messages (source-rank order) -> the SoA emit list the grouping reads;
// a target outside the owned range [lo, lo + n) is a protocol error (flagged, dropped)
__global__ void unpack_kernel(Workspace w, int64_t m, int64_t lo, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t *r = w.r_pack + i * MSG_WORDS;
        const int64_t key = (int64_t)(((uint64_t)(uint32_t)r[1] << 32) | (uint64_t)(uint32_t)r[0]);
        int32_t t = r[2];
        if (t < lo || t >= lo + n) {
            w.ctr[C_BADTGT] = 1ull;
            t = (int32_t)lo;  // kept in range; the host raises on the flag
        }
        w.e_key[i] = key;
        w.e_tgt[i] = t;
        w.e_id[i] = r[3];
        w.e_dist[i] = __int_as_float(r[4]);
    }
}

int launch_unpack(const Workspace &w, int64_t m, int64_t lo, int64_t n, cudaStream_t st) {
    if (m <= 0) return GRNND_OK;
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, (int64_t)device_sm_count() * 8));
    unpack_kernel<<<g, 256, 0, st>>>(w, m, lo, n);
    return check_launch("unpack_kernel");
}

int launch_bucket_by_rank(const Workspace &w, const int64_t *rank_bounds, int32_t nranks, int64_t *send_counts,
                          cudaStream_t st) {
    if (nranks < 1 || nranks > MAX_RANKS) {
        set_error("nranks %d outside [1, %d]", nranks, MAX_RANKS);
        return GRNND_EINVAL;
    }
    // per-rank counters live in the scan scratch (free at this point of the round)
    unsigned long long *rc = (unsigned long long *)w.scan_tmp;
    unsigned long long *cursor = rc + MAX_RANKS;
    GRNND_CUDA(cudaMemsetAsync(rc, 0, sizeof(unsigned long long) * MAX_RANKS, st));
    const unsigned g = (unsigned)device_sm_count() * 4;
    rank_count_kernel<<<g, 256, 0, st>>>(w, rank_bounds, nranks, rc);
    rank_offsets_kernel<<<1, 32, 0, st>>>(rc, nranks, cursor, send_counts);
    rank_scatter_kernel<<<g, 256, 0, st>>>(w, rank_bounds, nranks, cursor);
    return check_launch("bucket_by_rank", 3);
}

}  // namespace grnnd
