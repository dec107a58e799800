// search.cu -- the evaluation kernels on the device: exact brute-force k-NN ground truth,
// greedy beam search over the built graph, and the row normalisation of the IP metric.
//
// Reference: brute_force (/root/reference/pkg/src/grnnd/_numba_kernels.py:384-413),
// _greedy_single / greedy_search_batch (:416-513), search.py:72-142.  Both are
// bit-identical to the reference: every distance is the reference's sequential fp32
// _sqdist (:50-56, exact_step), and both results are defined by the (dist, id) order.
//
// brute force: the reference keeps, per query, the k smallest (dist, id) keys over all
//   points (a new point that ties the k-th key loses to the smaller id).  That is the
//   lexicographic top-k of the set, so it can be assembled from disjoint chunks in any
//   order.  bf_partial_kernel: CTA = 16 queries x one chunk of points; 256-point tiles are
//   staged in shared memory 32 dims at a time (coalesced 128-byte row segments), every
//   thread owns one point and accumulates its 16 query distances in index order; keys at or
//   below a query's running k-th key go to a per-query shared buffer, which a warp merges
//   into the query's top-k list after each tile.  bf_merge_kernel: warp per query, top-k of
//   the chunk lists.  The distance arithmetic is FP32-issue bound (3 ops per query-point-
//   dim): ~11 ms for 1000 queries over 1M x 128.
//
// greedy search: the reference's list update (insert at the first key greater than the
//   candidate, drop the tail beyond L, skip a candidate that cannot enter) makes the list
//   after any batch of insertions the top-L keys of (old list U batch), with the expanded
//   flags travelling with their entries.  Neighbours of one expanded vertex are distinct, so
//   their visited tests do not interact either.  greedy_kernel: warp per query; a node's
//   neighbours are taken 32 at a time (lane per neighbour: visited test-and-set, exact
//   distance), sorted by a warp bitonic network, and merged into the list by ranks (each new
//   key's position = its rank among the new keys + its rank in the list, and vice versa),
//   into the other half of a ping-pong list.  The next node is the first unexpanded entry
//   (ballot), as in the reference.
#include <cfloat>
#include <climits>

#include "common.cuh"
#include "workspace.cuh"

namespace grnnd {

constexpr int BF_QB = 16;     // queries per CTA
constexpr int BF_TILE = 256;  // points per tile (= threads per CTA)
constexpr int BF_DC = 8;      // float4 columns per staged chunk (32 dims)
constexpr int BF_TS = BF_DC + 1;  // tile row stride in float4 (odd: conflict-free LDS.128)
constexpr int BF_BUF = BF_TILE;   // candidates one tile can add per query
constexpr int BF_KMAX = 64;

__device__ __forceinline__ bool klt(float da, int ia, float db, int ib) { return da < db || (da == db && ia < ib); }

// warp argmin of (d, i) keys
__device__ __forceinline__ void warp_argmin(float &d, int &i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float od = __shfl_xor_sync(FULL, d, o);
        const int oi = __shfl_xor_sync(FULL, i, o);
        if (klt(od, oi, d, i)) {
            d = od;
            i = oi;
        }
    }
}

// Top-k selection (warp-collective) over keys a[0..na) followed by b[0..nb) (dist / id arrays
// in shared memory, consumed: selected entries are overwritten with +inf); the r-th smallest
// key lands in (od[r], oi[r]) for r < min(k, na + nb).  Returns that count.
__device__ int warp_select(float *ad, int *ai, int na, float *bd, int *bi, int nb, int k, float *od, int *oi) {
    const int lane = lane_id();
    const int tot = na + nb;
    const int rounds = k < tot ? k : tot;
    // winners kept in registers until all rounds are done (k <= 64: two per lane)
    float rd0 = INFINITY, rd1 = INFINITY;
    int ri0 = INT_MAX, ri1 = INT_MAX;
    for (int r = 0; r < rounds; ++r) {
        float bdv = INFINITY;
        int biv = INT_MAX, bpos = -1;
        for (int t = lane; t < tot; t += 32) {
            const float d = t < na ? ad[t] : bd[t - na];
            const int i = t < na ? ai[t] : bi[t - na];
            if (klt(d, i, bdv, biv)) {
                bdv = d;
                biv = i;
                bpos = t;
            }
        }
        float wd = bdv;
        int wi = biv;
        warp_argmin(wd, wi);
        // the owner of the winning key retires it
        if (bpos >= 0 && biv == wi && bdv == wd) {
            if (bpos < na) {
                ad[bpos] = INFINITY;
                ai[bpos] = INT_MAX;
            } else {
                bd[bpos - na] = INFINITY;
                bi[bpos - na] = INT_MAX;
            }
        }
        if (r == lane) {
            rd0 = wd;
            ri0 = wi;
        } else if (r == lane + 32) {
            rd1 = wd;
            ri1 = wi;
        }
        __syncwarp();
    }
    if (lane < rounds) {
        od[lane] = rd0;
        oi[lane] = ri0;
    }
    if (lane + 32 < rounds) {
        od[lane + 32] = rd1;
        oi[lane + 32] = ri1;
    }
    __syncwarp();
    return rounds;
}

struct BfSmemSizes {
    size_t q, tile, list, buf, total;
};
__host__ __device__ inline BfSmemSizes bf_smem(int ld) {
    BfSmemSizes s;
    s.q = (size_t)BF_QB * ld * 4;
    s.tile = (size_t)BF_TILE * BF_TS * 16;
    s.list = (size_t)BF_QB * BF_KMAX * 8;
    s.buf = (size_t)BF_QB * BF_BUF * 8;
    s.total = s.q + s.tile + s.list + s.buf + 3 * BF_QB * 4 + 64;
    return s;
}

__global__ void __launch_bounds__(BF_TILE) bf_partial_kernel(const float *__restrict__ data, int64_t n, int32_t ld,
                                                             const float *__restrict__ queries, int64_t nq, int32_t k,
                                                             int64_t chunk_pts, float *__restrict__ part_d,
                                                             int32_t *__restrict__ part_i) {
    extern __shared__ __align__(16) unsigned char bf_raw[];
    const BfSmemSizes z = bf_smem(ld);
    float4 *qv = reinterpret_cast<float4 *>(bf_raw);
    float4 *tile = reinterpret_cast<float4 *>(bf_raw + z.q);
    float *ld_d = reinterpret_cast<float *>(bf_raw + z.q + z.tile);
    int *ld_i = reinterpret_cast<int *>(ld_d + BF_QB * BF_KMAX);
    float *bdd = reinterpret_cast<float *>(bf_raw + z.q + z.tile + z.list);
    int *bii = reinterpret_cast<int *>(bdd + BF_QB * BF_BUF);
    int *bcnt = bii + BF_QB * BF_BUF;
    int *lsize = bcnt + BF_QB;
    float *thr = reinterpret_cast<float *>(lsize + BF_QB);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nq4 = ld >> 2;
    const int64_t q0 = (int64_t)blockIdx.x * BF_QB;
    const int nqb = (int)(nq - q0 < BF_QB ? nq - q0 : BF_QB);
    const int64_t c_lo = (int64_t)blockIdx.y * chunk_pts;
    const int64_t c_hi = c_lo + chunk_pts < n ? c_lo + chunk_pts : n;

    for (int x = tid; x < BF_QB * nq4; x += BF_TILE) {
        const int q = x / nq4, c = x - q * nq4;
        qv[x] = q < nqb ? reinterpret_cast<const float4 *>(queries + (q0 + q) * ld)[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (tid < BF_QB) {
        bcnt[tid] = 0;
        lsize[tid] = 0;
        thr[tid] = INFINITY;
    }
    __syncthreads();

    for (int64_t t0 = c_lo; t0 < c_hi; t0 += BF_TILE) {
        const int64_t p = t0 + tid;
        const bool valid = p < c_hi;
        float acc[BF_QB];
#pragma unroll
        for (int q = 0; q < BF_QB; ++q) acc[q] = 0.0f;
        for (int dc = 0; dc < nq4; dc += BF_DC) {
            const int ncol = nq4 - dc < BF_DC ? nq4 - dc : BF_DC;
            __syncthreads();  // the previous chunk is consumed
#pragma unroll
            for (int it = 0; it < BF_DC; ++it) {
                const int x = it * BF_TILE + tid;
                const int r = x >> 3, c = x & 7;
                const int64_t pr = t0 + r;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (pr < c_hi && c < ncol) v = __ldg(reinterpret_cast<const float4 *>(data + pr * ld) + dc + c);
                tile[r * BF_TS + c] = v;
            }
            __syncthreads();
            for (int c = 0; c < ncol; ++c) {
                const float4 x = tile[tid * BF_TS + c];
#pragma unroll
                for (int q = 0; q < BF_QB; ++q) {
                    const float4 y = qv[q * nq4 + dc + c];
                    float s = acc[q];
                    s = exact_step4(s, y, x);
                    acc[q] = s;
                }
            }
        }
        if (valid) {
#pragma unroll
            for (int q = 0; q < BF_QB; ++q) {
                if (q < nqb && acc[q] <= thr[q]) {
                    const int slot = atomicAdd(&bcnt[q], 1);
                    bdd[q * BF_BUF + slot] = acc[q];
                    bii[q * BF_BUF + slot] = (int)p;
                }
            }
        }
        __syncthreads();
        for (int q = warp; q < nqb; q += BF_TILE / 32) {
            const int nb = bcnt[q];
            if (nb == 0) continue;
            const int ls = lsize[q];
            float *od = ld_d + q * BF_KMAX;
            int *oi = ld_i + q * BF_KMAX;
            float *sd = bdd + q * BF_BUF;
            int *si = bii + q * BF_BUF;
            // the old list (<= k <= 64 keys) and the buffer (<= 256 keys) are selected together;
            // the winners are written back into the list after all rounds (warp_select)
            const int cnt = warp_select(od, oi, ls, sd, si, nb, k, od, oi);
            if (lane == 0) {
                lsize[q] = cnt;
                bcnt[q] = 0;
                thr[q] = cnt == k ? od[k - 1] : INFINITY;
            }
            __syncwarp();
        }
        __syncthreads();
    }
    const int64_t nchunk = gridDim.y;
    for (int q = warp; q < nqb; q += BF_TILE / 32) {
        const int ls = lsize[q];
        for (int r = lane; r < k; r += 32) {
            const int64_t o = ((q0 + q) * nchunk + blockIdx.y) * k + r;
            part_d[o] = r < ls ? ld_d[q * BF_KMAX + r] : INFINITY;
            part_i[o] = r < ls ? ld_i[q * BF_KMAX + r] : INT_MAX;
        }
    }
}

__global__ void bf_merge_kernel(float *__restrict__ part_d, int32_t *__restrict__ part_i, int64_t nq, int32_t nchunk,
                                int32_t k, int32_t *__restrict__ out_ids, float *__restrict__ out_d) {
    __shared__ float od[4][BF_KMAX];
    __shared__ int oi[4][BF_KMAX];
    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * 4 + w;
    if (q >= nq) return;
    float *pd = part_d + q * (int64_t)nchunk * k;
    int *pi = part_i + q * (int64_t)nchunk * k;
    const int cnt = warp_select(pd, pi, nchunk * k, pd, pi, 0, k, od[w], oi[w]);
    for (int r = lane; r < k; r += 32) {
        const bool ok = r < cnt && oi[w][r] != INT_MAX;
        out_ids[q * k + r] = ok ? oi[w][r] : -1;
        if (out_d) out_d[q * k + r] = ok ? od[w][r] : INFINITY;
    }
}

// ---------------------------------------------------------------------------------
// greedy beam search (warp per query)
// ---------------------------------------------------------------------------------
constexpr int GS_WARPS = 4;
constexpr int GS_LMAX = 1024;

__host__ __device__ inline size_t gs_warp_bytes(int ld, int L) {
    // query row, 2 x (ids, dists, expanded) list halves, 32 new keys
    return align_up(align_up((size_t)ld * 4, 16) + 2 * align_up((size_t)L * 9, 16) + 32 * 8 + 64, 16);
}

// keys < (d, i) in the sorted (dist, id) array [0, n)
__device__ __forceinline__ int lower_rank(const float *sd, const int *si, int n, float d, int i) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (klt(sd[mid], si[mid], d, i)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(GS_WARPS * 32) greedy_kernel(const int64_t *__restrict__ offsets,
                                                               const int32_t *__restrict__ nbrs, const float *__restrict__ data,
                                                               int32_t ld, const float *__restrict__ queries, int64_t nq,
                                                               int32_t L, int32_t k, const int64_t *__restrict__ entries,
                                                               uint32_t *__restrict__ visited, int64_t vwords,
                                                               int32_t *__restrict__ out_ids, float *__restrict__ out_d,
                                                               int64_t *__restrict__ out_cnt) {
    extern __shared__ __align__(16) unsigned char gs_raw[];
    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int64_t qi = (int64_t)blockIdx.x * GS_WARPS + w;
    if (qi >= nq) return;
    unsigned char *my = gs_raw + (size_t)w * gs_warp_bytes(ld, L);
    float *qrow = reinterpret_cast<float *>(my);
    unsigned char *lb = my + align_up((size_t)ld * 4, 16);
    const size_t hb = align_up((size_t)L * 9, 16);  // bytes of one list half: ids, dists, expanded flags
    auto hid = [&](int hh) { return reinterpret_cast<int *>(lb + hh * hb); };
    auto hds = [&](int hh) { return reinterpret_cast<float *>(lb + hh * hb + (size_t)L * 4); };
    auto hex = [&](int hh) { return lb + hh * hb + (size_t)L * 8; };
    float *nd = reinterpret_cast<float *>(lb + 2 * hb);
    int *ni = reinterpret_cast<int *>(nd + 32);
    const int nq4 = ld >> 2;
    for (int c = lane; c < nq4; c += 32)
        reinterpret_cast<float4 *>(qrow)[c] = reinterpret_cast<const float4 *>(queries + qi * ld)[c];
    __syncwarp();
    uint32_t *vis = visited + qi * vwords;
    auto dist_to = [&](int64_t v) {  // exact sequential distance (query row in shared memory)
        const float4 *x = reinterpret_cast<const float4 *>(data + v * ld);
        const float4 *y = reinterpret_cast<const float4 *>(qrow);
        float s = 0.0f;
#pragma unroll 4
        for (int c = 0; c < nq4; ++c) {
            const float4 a = __ldg(x + c), b = y[c];
            s = exact_step4(s, b, a);
        }
        return s;
    };
    const int64_t entry = entries[qi];
    int h = 0, size = 1;
    if (lane == 0) {
        hid(0)[0] = (int)entry;
        hds(0)[0] = dist_to(entry);
        hex(0)[0] = 0;
        vis[entry >> 5] |= 1u << (entry & 31);
    }
    __syncwarp();
    while (true) {
        int cur = -1;
        for (int b0 = 0; b0 < size; b0 += 32) {
            const unsigned m = __ballot_sync(FULL, b0 + lane < size && !hex(h)[b0 + lane]);
            if (m) {
                cur = b0 + __ffs(m) - 1;
                break;
            }
        }
        if (cur < 0) break;
        __syncwarp();
        if (lane == 0) hex(h)[cur] = 1;
        const int node = hid(h)[cur];
        __syncwarp();
        const int64_t beg = offsets[node], end = offsets[node + 1];
        for (int64_t e0 = beg; e0 < end; e0 += 32) {
            const int64_t e = e0 + lane;
            int nb = INT_MAX;
            bool isnew = false;
            if (e < end) {
                nb = nbrs[e];
                const uint32_t bit = 1u << (nb & 31);
                isnew = (atomicOr(&vis[nb >> 5], bit) & bit) == 0u;
            }
            const unsigned newm = __ballot_sync(FULL, isnew);
            if (!newm) continue;
            float d = isnew ? dist_to(nb) : INFINITY;
            int id = isnew ? nb : INT_MAX;
            // bitonic sort of the 32 keys, ascending by (dist, id)
#pragma unroll
            for (int k2 = 2; k2 <= 32; k2 <<= 1) {
#pragma unroll
                for (int j = k2 >> 1; j > 0; j >>= 1) {
                    const float od = __shfl_xor_sync(FULL, d, j);
                    const int oi = __shfl_xor_sync(FULL, id, j);
                    const bool up = (lane & k2) == 0 || k2 == 32;
                    const bool lower = (lane & j) == 0;
                    const bool other_less = klt(od, oi, d, id);
                    if ((lower == up) ? other_less : !other_less) {
                        d = od;
                        id = oi;
                    }
                }
            }
            const int nn = __popc(newm);
            nd[lane] = d;
            ni[lane] = id;
            __syncwarp();
            const int o = h ^ 1;
            // new keys: position = own rank + rank in the list
            if (lane < nn) {
                const int pos = lane + lower_rank(hds(h), hid(h), size, d, id);
                if (pos < L) {
                    hid(o)[pos] = id;
                    hds(o)[pos] = d;
                    hex(o)[pos] = 0;
                }
            }
            // list keys: position = own index + rank among the new keys
            for (int i = lane; i < size; i += 32) {
                const float dd = hds(h)[i];
                const int ii = hid(h)[i];
                const int pos = i + lower_rank(nd, ni, nn, dd, ii);
                if (pos < L) {
                    hid(o)[pos] = ii;
                    hds(o)[pos] = dd;
                    hex(o)[pos] = hex(h)[i];
                }
            }
            size = size + nn < L ? size + nn : L;
            h = o;
            __syncwarp();
        }
    }
    const int cnt = k < size ? k : size;
    for (int r = lane; r < k; r += 32) {
        out_ids[qi * k + r] = r < cnt ? hid(h)[r] : -1;
        if (out_d) out_d[qi * k + r] = r < cnt ? hds(h)[r] : INFINITY;
    }
    if (lane == 0 && out_cnt) out_cnt[qi] = cnt;
}

// ---------------------------------------------------------------------------------
// IP metric: rows scaled to unit L2 norm (norm = sqrt of the sequential fp32 sum of
// squares, correctly rounded sqrt and division), so squared L2 = 2 - 2 <a, b>.
// Thread per row: the order of the sum is the oracle's.
// ---------------------------------------------------------------------------------
__global__ void normalize_rows_kernel(float *__restrict__ data, int64_t n, int32_t dim, int32_t ld) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    float *row = data + r * ld;
    float s = 0.0f;
    for (int d = 0; d < dim; ++d) s = __fadd_rn(s, __fmul_rn(row[d], row[d]));
    if (!(s > 0.0f)) return;  // zero row: left as is
    const float nr = __fsqrt_rn(s);
    for (int d = 0; d < dim; ++d) row[d] = __fdiv_rn(row[d], nr);
}


int64_t bf_chunks(int64_t n, int64_t nq) {
    const int64_t qblocks = (nq + BF_QB - 1) / BF_QB;
    int64_t want = ((int64_t)device_sm_count() * 4 + qblocks - 1) / qblocks;
    const int64_t maxc = (n + BF_TILE - 1) / BF_TILE;
    if (want > maxc) want = maxc;
    if (want > 65535) want = 65535;
    return want < 1 ? 1 : want;
}

}  // namespace grnnd

using namespace grnnd;

extern "C" {

size_t grnnd_brute_force_workspace_bytes(int64_t n, int64_t nq, int32_t k) {
    if (n <= 0 || nq <= 0 || k <= 0) return 0;
    const int64_t nc = bf_chunks(n, nq);
    return (size_t)nq * (size_t)nc * (size_t)k * 8 + 256;
}

int grnnd_brute_force(const float *data, int64_t n, int32_t dim, int32_t ld, const float *queries, int64_t nq,
                      int32_t k, int32_t *out_ids, float *out_dists, void *workspace, size_t workspace_bytes,
                      grnnd_stream_t s) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    if (n < 1 || dim < 1 || ld < dim || (ld & 3) || nq < 0) {
        set_error("brute_force: bad shape n=%lld dim=%d ld=%d", (long long)n, dim, ld);
        return GRNND_EINVAL;
    }
    if (k < 1 || k > n) {
        set_error("k must satisfy 1 <= k <= N");
        return GRNND_EINVAL;
    }
    if (k > BF_KMAX) {
        set_error("brute_force: k=%d above the device limit %d", k, BF_KMAX);
        return GRNND_EUNSUPPORTED;
    }
    if (nq == 0) return GRNND_OK;
    const BfSmemSizes z = bf_smem(ld);
    if (z.total > 227 * 1024) {
        set_error("brute_force: row stride %d too large for the staged query block", ld);
        return GRNND_EUNSUPPORTED;
    }
    const int64_t nc = bf_chunks(n, nq);
    if (!workspace || workspace_bytes < grnnd_brute_force_workspace_bytes(n, nq, k)) {
        set_error("brute_force: workspace too small");
        return GRNND_EWORKSPACE;
    }
    float *pd = reinterpret_cast<float *>(workspace);
    int32_t *pi = reinterpret_cast<int32_t *>(pd + (size_t)nq * nc * k);
    const int64_t chunk = ((n + nc - 1) / nc + BF_TILE - 1) / BF_TILE * BF_TILE;
    const int64_t nc_eff = (n + chunk - 1) / chunk;
    static SmemOptIn optin;
    GRNND_CUDA(optin.ensure(bf_partial_kernel, z.total));
    dim3 grid((unsigned)((nq + BF_QB - 1) / BF_QB), (unsigned)nc_eff);
    bf_partial_kernel<<<grid, BF_TILE, z.total, st>>>(data, n, ld, queries, nq, k, chunk, pd, pi);
    GRNND_TRY(check_launch("bf_partial_kernel"));
    bf_merge_kernel<<<(unsigned)((nq + 3) / 4), 128, 0, st>>>(pd, pi, nq, (int32_t)nc_eff, k, out_ids, out_dists);
    return check_launch("bf_merge_kernel");
}

size_t grnnd_search_visited_bytes(int64_t n, int64_t nq) { return (size_t)nq * (size_t)((n + 31) / 32) * 4; }

int grnnd_greedy_search(const int64_t *offsets, const int32_t *nbrs, int64_t n, const float *data, int32_t dim,
                        int32_t ld, const float *queries, int64_t nq, int32_t L, int32_t k, const int64_t *entries,
                        int32_t *out_ids, float *out_dists, int64_t *out_cnt, void *visited, size_t visited_bytes,
                        grnnd_stream_t s) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    if (n < 1 || dim < 1 || ld < dim || (ld & 3) || nq < 0) {
        set_error("greedy_search: bad shape n=%lld dim=%d ld=%d", (long long)n, dim, ld);
        return GRNND_EINVAL;
    }
    if (k < 1 || L < k) {
        set_error(k < 1 ? "k >= 1" : "L >= k");
        return GRNND_EINVAL;
    }
    if (L > GS_LMAX) {
        set_error("greedy_search: L=%d above the device limit %d", L, GS_LMAX);
        return GRNND_EUNSUPPORTED;
    }
    if (nq == 0) return GRNND_OK;
    const size_t need = grnnd_search_visited_bytes(n, nq);
    if (!visited || visited_bytes < need) {
        set_error("greedy_search: visited bitmap needs %zu bytes", need);
        return GRNND_EWORKSPACE;
    }
    const size_t smem = (size_t)GS_WARPS * gs_warp_bytes(ld, L);
    if (smem > 227 * 1024) {
        set_error("greedy_search: L=%d with row stride %d exceeds shared memory", L, ld);
        return GRNND_EUNSUPPORTED;
    }
    GRNND_CUDA(cudaMemsetAsync(visited, 0, need, st));
    static SmemOptIn optin;
    GRNND_CUDA(optin.ensure(greedy_kernel, smem));
    greedy_kernel<<<(unsigned)((nq + GS_WARPS - 1) / GS_WARPS), GS_WARPS * 32, smem, st>>>(
        offsets, nbrs, data, ld, queries, nq, L, k, entries, reinterpret_cast<uint32_t *>(visited), (n + 31) / 32,
        out_ids, out_dists, out_cnt);
    return check_launch("greedy_kernel");
}

// refine_accept_loop (_numba_kernels.py:354-381), the sequential oracle's accept loop for one
// vertex: candidates in (dist, id) order; a candidate is kept unless an already-kept
// neighbour lies at or within its distance to the owner (then it is redirected to the FIRST
// such neighbour with their exact mutual distance).  One warp: the lanes evaluate the kept
// neighbours 32 at a time, a ballot finds the first hit -- the reference's break.
__global__ void refine_accept_kernel(const float *__restrict__ data, int32_t ld, int32_t dim,
                                     const int32_t *__restrict__ ids, const float *__restrict__ dists, int32_t k,
                                     int32_t *__restrict__ acc_ids, float *__restrict__ acc_dists,
                                     int32_t *__restrict__ red_tgt, int32_t *__restrict__ red_id,
                                     float *__restrict__ red_dist, int64_t *__restrict__ counts) {
    const int lane = lane_id();
    int na = 0, nr = 0;
    for (int i = 0; i < k; ++i) {
        const int32_t cand = ids[i];
        const float dvn = dists[i];
        int first = -1;
        float fd = 0.0f;
        for (int j0 = 0; j0 < na && first < 0; j0 += 32) {
            const int j = j0 + lane;
            float d = 0.0f;
            if (j < na) d = exact_sqdist_global(data + (int64_t)cand * ld, data + (int64_t)acc_ids[j] * ld, dim);
            const unsigned hit = __ballot_sync(FULL, j < na && d <= dvn);
            if (hit) {
                const int l = __ffs(hit) - 1;
                first = j0 + l;
                fd = __shfl_sync(FULL, d, l);
            }
        }
        if (lane == 0) {
            if (first >= 0) {
                red_tgt[nr] = acc_ids[first];
                red_id[nr] = cand;
                red_dist[nr] = fd;
            } else {
                acc_ids[na] = cand;
                acc_dists[na] = dvn;
            }
        }
        if (first >= 0) ++nr;
        else ++na;
        __syncwarp();
    }
    if (lane == 0) {
        counts[0] = na;
        counts[1] = nr;
    }
}

int grnnd_refine_accept_loop(const float *data, int32_t dim, int32_t ld, const int32_t *ids, const float *dists,
                             int32_t k, int32_t *acc_ids, float *acc_dists, int32_t *red_tgt, int32_t *red_id,
                             float *red_dist, int64_t *counts, grnnd_stream_t s) {
    if (dim < 1 || ld < dim || k < 0) {
        set_error("refine_accept_loop: bad dim/ld/k");
        return GRNND_EINVAL;
    }
    refine_accept_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(s)>>>(data, ld, dim, ids, dists, k, acc_ids,
                                                                           acc_dists, red_tgt, red_id, red_dist, counts);
    return check_launch("refine_accept_kernel");
}

int grnnd_normalize_rows(float *data, int64_t n, int32_t dim, int32_t ld, grnnd_stream_t s) {
    if (n < 0 || dim < 1 || ld < dim) {
        set_error("normalize_rows: bad shape");
        return GRNND_EINVAL;
    }
    if (n == 0) return GRNND_OK;
    normalize_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(data, n, dim, ld);
    return check_launch("normalize_rows_kernel");
}

}  // extern "C"
