#include <algorithm>
// reverse.cu -- reverse-edge sampling and the self merge, plus init and finalize kernels.
//
// References:
//   gen_reverse_messages   _numba_kernels.py:195-233  (ceil(rho*k) closest by (dist, id))
//   gen_merge_messages     _numba_kernels.py:236-250  (own entries, slot order)
//   sample_initial         _numba_kernels.py:91-115   (hash rejection sampling)
//   init_dists             _numba_kernels.py:118-122
//   finalize_graph         builder.py:342-362         (rows sorted by (dist, id) -> CSR)
//
// All are one-warp-per-vertex kernels: a pool row (<= 256 slots) sits in registers,
// ranks by (dist, id) come from one broadcast sweep (O(k^2/32) per warp, no sort
// network needed at these sizes).
#include "common.cuh"
#include "propagate.cuh"

namespace grnnd {

template <int RPL>
__device__ __forceinline__ void row_ranks(const int32_t (&id)[RPL], const float (&d)[RPL], int k, int (&rank)[RPL],
                                          bool *dup = nullptr) {
    const int lane = lane_id();
#pragma unroll
    for (int r = 0; r < RPL; ++r) rank[r] = 0;
#pragma unroll
    for (int rr = 0; rr < RPL; ++rr) {
        if (rr * 32 >= k) break;
        for (int l = 0; l < 32; ++l) {
            const int t = rr * 32 + l;
            if (t >= k) break;
            const float dt = __shfl_sync(FULL, d[rr], l);
            const int32_t it = __shfl_sync(FULL, id[rr], l);
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
                const int s = r * 32 + lane;
                // strict (dist, id) order; equal keys keep slot order (stable insertion sort)
                const bool less = dt < d[r] || (dt == d[r] && (it < id[r] || (it == id[r] && t < s)));
                rank[r] += less ? 1 : 0;
                if (dup && s < k && t != s && it == id[r]) *dup = true;
            }
        }
    }
}

template <int RPL>
__global__ void __launch_bounds__(256) reverse_select_kernel(ReverseArgs a) {
    // warp per vertex, 32 consecutive vertices per warp step: their message counts are known
    // from the pool sizes alone, so one list reservation (atomicAdd) covers all 32
    const int lane = lane_id();
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long attempts = 0;
    for (int64_t v0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; v0 < a.n; v0 += warps * 32) {
        const int kl = v0 + lane < a.n ? a.read_count[v0 + lane] : 0;
        const int ml = kl > 0 ? reverse_count(a.rho, kl) : 0;
        int incl = ml;  // inclusive warp scan of the counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        unsigned long long wbase = 0;
        if (!a.slice_mode) {
            if (lane == 31 && incl > 0) wbase = atomicAdd(&a.w.ctr[C_LIST], (unsigned long long)incl);
            wbase = __shfl_sync(FULL, wbase, 31);
        }
        const int excl = incl - ml;
        const int tot = __shfl_sync(FULL, incl, 31);  // (every lane: a full-mask shuffle)
        attempts += lane == 0 ? (unsigned long long)tot : 0ull;
        const int nv = a.n - v0 < 32 ? (int)(a.n - v0) : 32;
        for (int j = 0; j < nv; ++j) {
            const int64_t v = v0 + j;
            const int k = __shfl_sync(FULL, kl, j);
            const int m = __shfl_sync(FULL, ml, j);
            const unsigned long long base = wbase + (unsigned long long)__shfl_sync(FULL, excl, j);
            const int64_t vg = a.lo + v;
            if (k == 0) {
                if (a.slice_mode && lane == 0) a.msg_cnt[v] = 0;
                continue;
            }
            int32_t id[RPL];
            float d[RPL];
            int rank[RPL];
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
                const int s = r * 32 + lane;
                id[r] = s < k ? a.read_ids[v * a.cap + s] : TOMB;
                d[r] = s < k ? a.read_dists[v * a.cap + s] : 0.0f;
            }
            row_ranks<RPL>(id, d, k, rank);
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
                const int s = r * 32 + lane;
                if (s < k && rank[r] < m) {
                    if (a.slice_mode) {
                        a.msg_tgt[v * a.cap + rank[r]] = id[r];
                        a.msg_id[v * a.cap + rank[r]] = (int32_t)vg;
                        a.msg_dist[v * a.cap + rank[r]] = d[r];
                    } else {
                        const unsigned long long p = base + (unsigned long long)rank[r];
                        if (p < (unsigned long long)a.w.msg_capacity) {
                            a.w.e_key[p] = vg * a.cap + rank[r];
                            a.w.e_tgt[p] = id[r];
                            a.w.e_id[p] = (int32_t)vg;
                            a.w.e_dist[p] = d[r];
                        } else {
                            a.w.ctr[C_OVERFLOW] = 1ull;
                        }
                    }
                }
            }
            if (a.slice_mode && lane == 0) a.msg_cnt[v] = m;
        }
    }
    if (lane == 0 && a.stats && attempts) {
        atomicAdd((unsigned long long *)&a.stats[GRNND_ST_REVERSE_ATTEMPTS], attempts);
        atomicAdd((unsigned long long *)&a.stats[GRNND_ST_MESSAGES], attempts);
    }
}

__global__ void merge_slices_kernel(ReverseArgs a) {
    const int lane = lane_id();
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < a.n; v += warps) {
        const int k = a.read_count[v];
        int base = 0;
        for (int s0 = 0; s0 < k; s0 += 32) {
            const int s = s0 + lane;
            const int32_t x = s < k ? a.read_ids[v * a.cap + s] : TOMB;
            const bool live = x != TOMB;
            const unsigned bal = __ballot_sync(FULL, live);
            if (live) {
                const int o = base + __popc(bal & ((1u << lane) - 1));
                a.msg_tgt[v * a.cap + o] = (int32_t)(a.lo + v);
                a.msg_id[v * a.cap + o] = x;
                a.msg_dist[v * a.cap + o] = a.read_dists[v * a.cap + s];
            }
            base += __popc(bal);
        }
        if (lane == 0) a.msg_cnt[v] = base;
    }
}


static unsigned warp_grid(int64_t n) {
    const int64_t blocks = std::min<int64_t>((n + 7) / 8, (int64_t)device_sm_count() * 16);
    return (unsigned)std::max<int64_t>(1, blocks);
}

int launch_reverse_select(const ReverseArgs &a, cudaStream_t st) {
    if (a.n <= 0) return GRNND_OK;
    const unsigned g = warp_grid((a.n + 31) / 32);  // a warp step covers 32 vertices
    switch ((a.cap + 31) / 32) {
        case 1: reverse_select_kernel<1><<<g, 256, 0, st>>>(a); break;
        case 2: reverse_select_kernel<2><<<g, 256, 0, st>>>(a); break;
        case 3: reverse_select_kernel<3><<<g, 256, 0, st>>>(a); break;
        case 4: reverse_select_kernel<4><<<g, 256, 0, st>>>(a); break;
        case 5: reverse_select_kernel<5><<<g, 256, 0, st>>>(a); break;
        case 6: reverse_select_kernel<6><<<g, 256, 0, st>>>(a); break;
        case 7: reverse_select_kernel<7><<<g, 256, 0, st>>>(a); break;
        case 8: reverse_select_kernel<8><<<g, 256, 0, st>>>(a); break;
        default: set_error("cap %d > %d unsupported", a.cap, GRNND_MAX_CAP); return GRNND_EUNSUPPORTED;
    }
    return check_launch("reverse_select_kernel");
}

int launch_merge_slices(const ReverseArgs &a, cudaStream_t st) {
    if (a.n <= 0) return GRNND_OK;
    merge_slices_kernel<<<warp_grid(a.n), 256, 0, st>>>(a);
    return check_launch("merge_slices_kernel");
}

// ---------------------------------------------------------------------------------
// init: sample_initial (thread per vertex, the reference's exact attempt sequence)
// ---------------------------------------------------------------------------------
__global__ void sample_initial_kernel(int64_t n_total, int64_t lo, int64_t rows, int32_t count, uint64_t seed,
                                      int32_t *__restrict__ out, int32_t ld_out, unsigned long long *fail) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int64_t v = lo + r;
    uint64_t limit = (uint64_t)(64 * n_total + 64);
    if (limit > ATTEMPT_STRIDE) limit = ATTEMPT_STRIDE;
    const uint64_t pre = vertex_prefix(seed, STREAM_INIT, (uint64_t)v);
    int32_t *row = out + r * ld_out;
    for (int s = 0; s < count; ++s) {
        bool placed = false;
        for (uint64_t at = 0; at < limit; ++at) {
            const uint64_t idx = (uint64_t)s * ATTEMPT_STRIDE + at;
            const int64_t c = (int64_t)(mix64(pre ^ idx) % (uint64_t)n_total);
            if (c == v) continue;
            bool dup = false;
            for (int t = 0; t < s; ++t)
                if (row[t] == c) {
                    dup = true;
                    break;
                }
            if (dup) continue;
            row[s] = (int32_t)c;
            placed = true;
            break;
        }
        if (!placed) *fail = 1ull;
    }
}

int launch_sample_initial(int64_t n_total, int64_t lo, int64_t rows, int32_t count, uint64_t seed, int32_t *out,
                          int32_t ld_out, int64_t *fail_flag, cudaStream_t st) {
    if (rows <= 0) return GRNND_OK;
    sample_initial_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(
        n_total, lo, rows, count, seed, out, ld_out, (unsigned long long *)fail_flag);
    return check_launch("sample_initial_kernel");
}

// init_dists: one thread per (vertex, slot); exact sequential distance
__global__ void init_dists_pair_kernel(const float *__restrict__ data, int32_t dim, int32_t ld, int64_t lo,
                                       int64_t rows, const int32_t *__restrict__ ids, int32_t ld_ids, int32_t count,
                                       float *__restrict__ out, int32_t ld_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * count) return;
    const int64_t r = i / count;
    const int s = (int)(i - r * count);
    const int32_t j = ids[r * ld_ids + s];
    out[r * ld_out + s] = exact_sqdist_global(data + (lo + r) * (int64_t)ld, data + (int64_t)j * ld, dim);
}

// warp per vertex row: the row is staged once in shared memory; lane s < count walks
// neighbour s's row (16-byte loads, independent addresses) in the reference's sequential
// order against it
constexpr int ID_WARPS = 8;
__global__ void __launch_bounds__(ID_WARPS * 32) init_dists_kernel(const float *__restrict__ data, int32_t dim,
                                                                  int32_t ld, int64_t lo, int64_t rows,
                                                                  const int32_t *__restrict__ ids, int32_t ld_ids,
                                                                  int32_t count, float *__restrict__ out,
                                                                  int32_t ld_out) {
    extern __shared__ float4 id_rows[];  // [ID_WARPS][ld / 4]
    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int nq = ld >> 2;
    float4 *mine = id_rows + w * nq;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
        const float4 *a = reinterpret_cast<const float4 *>(data + (lo + r) * (int64_t)ld);
        for (int q = lane; q < nq; q += 32) mine[q] = a[q];
        __syncwarp();
        for (int s0 = 0; s0 < count; s0 += 32) {
            const int s = s0 + lane;
            if (s < count) {
                const int32_t j = ids[r * ld_ids + s];
                const float4 *b = reinterpret_cast<const float4 *>(data + (int64_t)j * ld);
                float acc = 0.0f;
                const int nfull = dim >> 2;
#pragma unroll 8
                for (int q = 0; q < nfull; ++q) {
                    const float4 x = mine[q], y = __ldg(b + q);
                    acc = exact_step4(acc, x, y);
                }
                if (dim & 3) {  // the first dim % 4 columns of the last chunk (padding ignored)
                    const float4 x = mine[nfull], y = __ldg(b + nfull);
                    acc = exact_step(acc, x.x, y.x);
                    if ((dim & 3) > 1) acc = exact_step(acc, x.y, y.y);
                    if ((dim & 3) > 2) acc = exact_step(acc, x.z, y.z);
                }
                out[r * ld_out + s] = acc;
            }
        }
        __syncwarp();
    }
}

int launch_init_dists(const float *data, int32_t dim, int32_t ld, int64_t lo, int64_t rows, const int32_t *ids,
                      int32_t ld_ids, int32_t count, float *out, int32_t ld_out, cudaStream_t st) {
    if (rows <= 0 || count <= 0) return GRNND_OK;
    if (ld & 3) {  // rows not float4-addressable: thread per pair
        const int64_t total = rows * count;
        init_dists_pair_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(data, dim, ld, lo, rows, ids, ld_ids,
                                                                                count, out, ld_out);
        return check_launch("init_dists_pair_kernel");
    }
    const size_t smem = (size_t)ID_WARPS * ld * 4;
    if (smem > 48 * 1024) GRNND_CUDA(cudaFuncSetAttribute(init_dists_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = std::min<int64_t>((rows + ID_WARPS - 1) / ID_WARPS, 148 * 64);
    init_dists_kernel<<<(unsigned)blocks, ID_WARPS * 32, smem, st>>>(data, dim, ld, lo, rows, ids, ld_ids, count, out,
                                                                      ld_out);
    return check_launch("init_dists_kernel");
}

// ---------------------------------------------------------------------------------
// finalize: rows sorted by (dist, id) into CSR (and optionally the fixed-degree view)
// ---------------------------------------------------------------------------------
template <int RPL>
__global__ void __launch_bounds__(256) finalize_kernel(const int32_t *__restrict__ ids, const float *__restrict__ dists,
                                                       const int32_t *__restrict__ counts, int64_t n, int32_t cap,
                                                       int64_t lo, int64_t n_total,
                                                       const int64_t *__restrict__ offsets, int32_t *__restrict__ nbrs,
                                                       int32_t *__restrict__ fixed_out,
                                                       unsigned long long *__restrict__ bad) {
    const int lane = lane_id();
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
        const int k = counts[v];
        int32_t id[RPL];
        float d[RPL];
        int rank[RPL];
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            const int s = r * 32 + lane;
            id[r] = s < k ? ids[v * cap + s] : TOMB;
            d[r] = s < k ? dists[v * cap + s] : 0.0f;
        }
        bool dup = false;
        row_ranks<RPL>(id, d, k, rank, bad ? &dup : nullptr);
        unsigned long long flags = dup ? 4ull : 0ull;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            const int s = r * 32 + lane;
            if (s < k) {
                if (id[r] < 0 || id[r] >= n_total) flags |= 1ull;
                if (id[r] == lo + v) flags |= 2ull;
                if (nbrs) nbrs[offsets[v] + rank[r]] = id[r];
                if (fixed_out) fixed_out[v * cap + rank[r]] = id[r];
            } else if (s < cap && fixed_out) {
                fixed_out[v * cap + s] = TOMB;
            }
        }
        if (bad && flags) atomicOr(bad, flags);
    }
}

int launch_finalize(const int32_t *ids, const float *dists, const int32_t *counts, int64_t n, int32_t cap,
                    int64_t lo, int64_t n_total, const int64_t *offsets, int32_t *nbrs, int32_t *fixed_out,
                    int64_t *bad_flag, cudaStream_t st) {
    unsigned long long *bad = (unsigned long long *)bad_flag;
    if (n <= 0) return GRNND_OK;
    const unsigned g = warp_grid(n);
#define GRNND_FIN(R) finalize_kernel<R><<<g, 256, 0, st>>>(ids, dists, counts, n, cap, lo, n_total, offsets, nbrs, fixed_out, bad)
    switch ((cap + 31) / 32) {
        case 1: GRNND_FIN(1); break;
        case 2: GRNND_FIN(2); break;
        case 3: GRNND_FIN(3); break;
        case 4: GRNND_FIN(4); break;
        case 5: GRNND_FIN(5); break;
        case 6: GRNND_FIN(6); break;
        case 7: GRNND_FIN(7); break;
        case 8: GRNND_FIN(8); break;
#undef GRNND_FIN
        default: set_error("cap %d > %d unsupported", cap, GRNND_MAX_CAP); return GRNND_EUNSUPPORTED;
    }
    return check_launch("finalize_kernel");
}

}  // namespace grnnd
