// pairs.cuh -- the order-free FP32 hot loop of the pair phase (included by propagate.cu,
// inside namespace grnnd, after row_stride16 / tile_decode / tile_accumulate).
//
// A CTA processes a BATCH of B pools at a time (B = 4 for k <= 16, 2 for k <= 32, else 1):
// the pools' rows share one shared-memory slab and their TxT tiles share one thread
// loop, so small pools (most of them: the median k is ~13) still keep every lane busy
// and amortise the gather latency and barriers over B vertices.  The next batch's rows
// are gathered (cp.async) while this batch's masks are written out.
#pragma once

template <int MAXK, int B>
struct PairSmem {
    static constexpr int W = (MAXK + 63) / 64;  // 64-bit words per mask row
    static constexpr int CL = PAIR_LIST;  // redirect-capable pairs handed to decide (workspace.cuh)
    uint64_t cond[B][MAXK * W];
    uint64_t afar[B][MAXK * W];
    int32_t ids[2][B][MAXK];  // pool rows of the current / next batch
    float dv[2][B][MAXK];
    uint8_t pos[2][B][MAXK];  // slot -> permutation position
    float nrm[2][B][MAXK];    // squared norms of the pool members' rows (filtered mode)
    int32_t k[2][B];
    int64_t v[2][B];          // local row of each batch member (-1: none)
    uint32_t cl_key[B][CL];   // (afar << 16) | (anchor pos << 8) | partner pos
    float cl_d[B][CL];
    int cl_n[B];
    int tp[B + 1];            // tile prefix over the batch members
    static constexpr int QC = 256;  // filter candidates per batch (overflow: exact sweep)
    uint32_t q[QC];           // (member << 16) | (slot s << 8) | slot u
    int qn;
};

// A redirect-capable pair (s, u) of member g with its exact distance d < max(dv[s], dv[u]):
// set its bits in permutation space and keep the distance for the decide kernel.
template <int MAXK, int B>
__device__ __forceinline__ void record_redirect(PairSmem<MAXK, B> &sm, int cur, int g, int s, int u, float d) {
    using S = PairSmem<MAXK, B>;
    constexpr int W = S::W;
    const int x1 = sm.pos[cur][g][s], x2 = sm.pos[cur][g][u];
    const float d1 = sm.dv[cur][g][s], d2 = sm.dv[cur][g][u];
    // anchor = the member visited first (smaller position)
    const int xa = x1 < x2 ? x1 : x2, xb = x1 < x2 ? x2 : x1;
    const float dva = x1 < x2 ? d1 : d2, dvb = x1 < x2 ? d2 : d1;
    const unsigned long long bit = 1ull << (xb & 63);
    const bool far = !(dvb >= dva);
    atomicOr((unsigned long long *)&sm.cond[g][xa * W + (xb >> 6)], bit);
    if (far) atomicOr((unsigned long long *)&sm.afar[g][xa * W + (xb >> 6)], bit);
    const int c = atomicAdd(&sm.cl_n[g], 1);
    if (c < S::CL) {
        sm.cl_key[g][c] = (uint32_t)((far ? 1u << 16 : 0u) | (xa << 8) | xb);
        sm.cl_d[g][c] = d;
    }
}

// Epilogue of tile (bI, bJ) of member g.
//  exact (DOT = false): acc holds the reference's sequential distances; decide directly.
//  filtered (DOT = true): acc holds FFMA dot products; d~ = |a|^2 + |b|^2 - 2 a.b is within
//  E = eps_n (|a|^2 + |b|^2) + eps_h hi of the exact sequential distance (forward error
//  bound of both summations, 2x margin), so a pair with d~ >= hi + E can not
//  redirect and is settled here; the rest (~1% of pairs) are queued for an exact
//  re-evaluation.  NaN/inf compare false and are queued too.
template <int MAXK, int B, int T, bool DOT>
__device__ __forceinline__ unsigned tile_epilogue(PairSmem<MAXK, B> &sm, int cur, int g, const float (&acc)[T * T],
                                                  int bI, int bJ, int nb, int k, float eps_n, float eps_h) {
    float dA[T], dB[T], nA[T], nB[T];
    bool vA[T], vB[T];
#pragma unroll
    for (int i = 0; i < T; ++i) {
        const int s = bI + nb * i, u = bJ + nb * i;
        vA[i] = s < k && sm.ids[cur][g][s] != TOMB;
        vB[i] = u < k && sm.ids[cur][g][u] != TOMB;
        dA[i] = vA[i] ? sm.dv[cur][g][s] : 0.0f;
        dB[i] = vB[i] ? sm.dv[cur][g][u] : 0.0f;
        if (DOT) {
            nA[i] = vA[i] ? sm.nrm[cur][g][s] : 0.0f;
            nB[i] = vB[i] ? sm.nrm[cur][g][u] : 0.0f;
        }
    }
    unsigned npairs = 0;
#pragma unroll
    for (int i = 0; i < T; ++i)
#pragma unroll
        for (int j = 0; j < T; ++j) {
            const int s = bI + nb * i, u = bJ + nb * j;
            // off-diagonal tiles hold each unordered pair once; diagonal ones twice
            const bool valid = vA[i] && vB[j] && (bI != bJ || i < j);
            npairs += valid ? 1u : 0u;
            const float d1 = dA[i], d2 = dB[j];
            const float hi = d1 >= d2 ? d1 : d2;
            if (DOT) {
                const float nn = nA[i] + nB[j];
                const float dap = fmaf(-2.0f, acc[i * T + j], nn);
                const float e = fmaf(eps_n, nn, fmaf(eps_h, hi, 1e-30f));
                // settled iff d~ >= hi + E with finite norms; NaN / overflow fall through
                if (valid && !(dap >= hi + e && nn <= 3.0e38f)) {
                    const int c = atomicAdd(&sm.qn, 1);
                    if (c < PairSmem<MAXK, B>::QC) sm.q[c] = (uint32_t)((g << 16) | (s << 8) | u);
                }
            } else if (valid && acc[i * T + j] < hi) {
                record_redirect<MAXK, B>(sm, cur, g, s, u, acc[i * T + j]);
            }
        }
    return npairs;
}

// Exact sequential distance of two staged rows (the reference's _sqdist arithmetic).
__device__ __forceinline__ float exact_sqdist_smem(const float4 *__restrict__ a, const float4 *__restrict__ b,
                                                   int nq) {
    float s = 0.0f;
    for (int q = 0; q < nq; ++q) {
        const float4 x = a[q], y = b[q];
        s = exact_step4(s, x, y);
    }
    return s;
}

// MULTI: D > 128, rows staged 128 dims at a time with accumulators held across chunks
// (always B = 1).  DOT: filtered mode (tile_epilogue); the kernel then needs a.norms.
template <int MAXK, int B, int THREADS, int TPT, int T, bool MULTI, int NQ, bool DOT>
__global__ void __launch_bounds__(THREADS) pairs_kernel(PropArgs a, int bin, int kmax) {
    using S = PairSmem<MAXK, B>;
    constexpr int W = S::W;
    constexpr int PER = (B * MAXK + THREADS - 1) / THREADS;  // pool slots per thread
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S &sm = *reinterpret_cast<S *>(smem_raw);
    float4 *rows = reinterpret_cast<float4 *>(smem_raw + align_up(sizeof(S), 128));

    const int tid = threadIdx.x;
    const int64_t nbin = (int64_t)a.w.ctr[C_BIN0 + bin];
    const int64_t nbatch = (nbin + B - 1) / B;
    const int2 *blist = a.w.bins + (int64_t)bin * a.w.n;
    const int nq_total = (a.dim + 3) >> 2;  // float4 per row (ld % 4 == 0, pad cols are 0)
    const int rs4 = row_stride16(nq_total);
    const int nchunks = (nq_total + DC4 - 1) / DC4;
    const int cap = a.cap;
    const int mw = a.w.mw;
    const float eps_n = a.eps_n, eps_h = a.eps_h;
    unsigned long long pairs_local = 0;

    int32_t nid[PER];
    float ndv[PER];
    float nnr[PER];
    int32_t npos[PER];
    int nk[PER];
    int64_t nv[PER];
    auto fetch_meta = [&](int64_t bi) {  // next batch's pool rows -> registers
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int e = r * THREADS + tid;
            const int g = e / MAXK, s = e - g * MAXK;
            nk[r] = 0;
            nv[r] = -1;
            if (g < B && bi * B + g < nbin) {
                const int2 vk = blist[bi * B + g];
                const int64_t v = vk.x;
                const int k = vk.y;
                nv[r] = v;
                nk[r] = k;
                if (s < k) {
                    nid[r] = a.read_ids[v * cap + s];
                    ndv[r] = a.read_dists[v * cap + s];
                    npos[r] = a.order_code == 0 ? (int32_t)a.w.pos8[v * a.w.pcap + s] : 0;
                    if (DOT) nnr[r] = nid[r] >= 0 ? a.norms[nid[r]] : 0.0f;
                }
            }
        }
    };
    auto store_meta = [&](int slot) {
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int e = r * THREADS + tid;
            const int g = e / MAXK, s = e - g * MAXK;
            if (g < B) {
                if (s < nk[r]) {
                    sm.ids[slot][g][s] = nid[r];
                    sm.dv[slot][g][s] = ndv[r];
                    sm.pos[slot][g][s] = (uint8_t)npos[r];
                    if (DOT) sm.nrm[slot][g][s] = nnr[r];
                }
                if (s == 0) {
                    sm.k[slot][g] = nk[r];
                    sm.v[slot][g] = nv[r];
                }
            }
        }
    };
    auto load_rows = [&](int slot, int c) {  // chunk c of every member's rows (cp.async)
        const int q0 = c * DC4;
        const int nq = min(DC4, nq_total - q0);
#pragma unroll
        for (int g = 0; g < B; ++g) {
            const int k = sm.k[slot][g];
            const int total = k * nq;
            for (int e = tid; e < total; e += THREADS) {
                const int r = e / nq;
                const int q = e - r * nq;
                const int32_t id = sm.ids[slot][g][r];
                const float *src = a.data + (int64_t)(id < 0 ? 0 : id) * a.ld + (int64_t)(q0 + q) * 4;
                cp_async16(&rows[(g * kmax + r) * rs4 + q], src, id >= 0);
            }
        }
        cp_async_commit();
    };

    int64_t bi = blockIdx.x;
    if (bi >= nbatch) return;
    fetch_meta(bi);
    store_meta(0);
    __syncthreads();
    if (!MULTI) load_rows(0, 0);
    int cur = 0;

    for (; bi < nbatch; bi += gridDim.x) {
        const int64_t bi_next = bi + gridDim.x;
        const bool has_next = bi_next < nbatch;

        if (a.order_code != 0) {
            // ascending debug order (:75-87): stable rank by (dist, id); published for decide
#pragma unroll
            for (int g = 0; g < B; ++g) {
                const int k = sm.k[cur][g];
                for (int s = tid; s < k; s += THREADS) {
                    const float ds = sm.dv[cur][g][s];
                    const int32_t is = sm.ids[cur][g][s];
                    int r = 0;
                    for (int t = 0; t < k; ++t) {
                        const float dt = sm.dv[cur][g][t];
                        const int32_t it2 = sm.ids[cur][g][t];
                        r += (dt < ds || (dt == ds && (it2 < is || (it2 == is && t < s)))) ? 1 : 0;
                    }
                    sm.pos[cur][g][s] = (uint8_t)r;
                    a.w.pos8[sm.v[cur][g] * a.w.pcap + s] = (uint8_t)r;
                }
            }
        }
#pragma unroll
        for (int g = 0; g < B; ++g) {
            const int k = sm.k[cur][g];
            for (int i = tid; i < k * W; i += THREADS) {
                sm.cond[g][i] = 0ull;
                sm.afar[g][i] = 0ull;
            }
        }
        if (tid == 0) {
            int t = 0;
#pragma unroll
            for (int g = 0; g < B; ++g) {
                sm.cl_n[g] = 0;
                sm.tp[g] = t;
                const int nb = (sm.k[cur][g] + T - 1) / T;
                t += nb * (nb + 1) / 2;
            }
            sm.tp[B] = t;
            sm.qn = 0;
        }
        if (has_next) fetch_meta(bi_next);

        if (!MULTI) {
            cp_async_wait_all();
            __syncthreads();  // rows landed; masks zeroed; tile prefix visible
            const int ntiles = sm.tp[B];
            for (int t = tid; t < ntiles; t += THREADS) {
                int g = 0;
#pragma unroll
                for (int h = 1; h < B; ++h) g += t >= sm.tp[h] ? 1 : 0;
                int bI, bJ;
                tile_decode(t - sm.tp[g], bI, bJ);
                float acc[T * T];
#pragma unroll
                for (int p = 0; p < T * T; ++p) acc[p] = 0.0f;
                const int r0 = g * kmax;
                const int kg = sm.k[cur][g];
                const int nb = (kg + T - 1) / T;
                if (DOT) tile_dot<T, NQ>(acc, rows, r0 + bI, r0 + bJ, nb, nq_total, rs4);
                else tile_accumulate<T, NQ>(acc, rows, r0 + bI, r0 + bJ, nb, nq_total, rs4);
                pairs_local += tile_epilogue<MAXK, B, T, DOT>(sm, cur, g, acc, bI, bJ, nb, kg, eps_n, eps_h);
            }
        } else {
            const int k = sm.k[cur][0];
            const int nb = (k + T - 1) / T;
            const int ntiles = nb * (nb + 1) / 2;
            __syncthreads();
            for (int g0 = 0; g0 < ntiles; g0 += THREADS * TPT) {
                float acc[TPT][T * T];
#pragma unroll
                for (int tt = 0; tt < TPT; ++tt)
#pragma unroll
                    for (int p = 0; p < T * T; ++p) acc[tt][p] = 0.0f;
                for (int c = 0; c < nchunks; ++c) {
                    __syncthreads();  // everyone done with the previous chunk
                    load_rows(cur, c);
                    cp_async_wait_all();
                    __syncthreads();
                    const int nq = min(DC4, nq_total - c * DC4);
#pragma unroll
                    for (int tt = 0; tt < TPT; ++tt) {
                        const int t = g0 + tt * THREADS + tid;
                        if (t < ntiles) {
                            int bI, bJ;
                            tile_decode(t, bI, bJ);
                            if (DOT) tile_dot<T, 0>(acc[tt], rows, bI, bJ, nb, nq, rs4);
                            else tile_accumulate<T, 0>(acc[tt], rows, bI, bJ, nb, nq, rs4);
                        }
                    }
                }
#pragma unroll
                for (int tt = 0; tt < TPT; ++tt) {
                    const int t = g0 + tt * THREADS + tid;
                    if (t < ntiles) {
                        int bI, bJ;
                        tile_decode(t, bI, bJ);
                        pairs_local += tile_epilogue<MAXK, B, T, DOT>(sm, cur, 0, acc[tt], bI, bJ, nb, k, eps_n, eps_h);
                    }
                }
            }
        }
        if (DOT) {
            // exact re-evaluation of the filter's candidates (rows still staged unless MULTI)
            __syncthreads();
            const int qn = sm.qn;
            if (qn <= S::QC) {
                for (int e = tid; e < qn; e += THREADS) {
                    const uint32_t key = sm.q[e];
                    const int g = (int)(key >> 16), s = (int)((key >> 8) & 255u), u = (int)(key & 255u);
                    const float d = MULTI ? exact_sqdist_global(a.data + (int64_t)sm.ids[cur][g][s] * a.ld,
                                                                a.data + (int64_t)sm.ids[cur][g][u] * a.ld, a.dim)
                                          : exact_sqdist_smem(rows + (g * kmax + s) * rs4,
                                                              rows + (g * kmax + u) * rs4, nq_total);
                    const float d1 = sm.dv[cur][g][s], d2 = sm.dv[cur][g][u];
                    if (d < (d1 >= d2 ? d1 : d2)) record_redirect<MAXK, B>(sm, cur, g, s, u, d);
                }
            } else {
                // queue overflow (degenerate data: many near-ties): exact sweep of every pair
#pragma unroll
                for (int g = 0; g < B; ++g) {
                    const int k = sm.k[cur][g];
                    const int np = k * (k - 1) / 2;
                    for (int p = tid; p < np; p += THREADS) {
                        int s, u;
                        tile_decode(p, s, u);  // s <= u over the triangle incl. diagonal
                        u += 1;                // strict upper triangle: (s, u) with s < u
                        if (sm.ids[cur][g][s] == TOMB || sm.ids[cur][g][u] == TOMB) continue;
                        const float d = MULTI ? exact_sqdist_global(a.data + (int64_t)sm.ids[cur][g][s] * a.ld,
                                                                    a.data + (int64_t)sm.ids[cur][g][u] * a.ld, a.dim)
                                              : exact_sqdist_smem(rows + (g * kmax + s) * rs4,
                                                                  rows + (g * kmax + u) * rs4, nq_total);
                        const float d1 = sm.dv[cur][g][s], d2 = sm.dv[cur][g][u];
                        if (d < (d1 >= d2 ? d1 : d2)) record_redirect<MAXK, B>(sm, cur, g, s, u, d);
                    }
                }
            }
        }
        if (!MULTI) {
            if (has_next) store_meta(cur ^ 1);
            __syncthreads();  // masks complete; row slab free; next pool rows visible
            if (has_next) load_rows(cur ^ 1, 0);  // lands while the masks are written out
        } else {
            if (has_next) store_meta(cur ^ 1);
            __syncthreads();
        }
        // masks + kept distances -> global (decide_kernel)
#pragma unroll
        for (int g = 0; g < B; ++g) {
            const int64_t v = sm.v[cur][g];
            if (v < 0) continue;
            const int k = sm.k[cur][g];
            const int ncl = sm.cl_n[g];
            if (ncl > S::CL) {  // incomplete list: the masks go to global too
                uint64_t *gc = a.w.cond + v * (int64_t)cap * mw;
                uint64_t *ga = a.w.afar + v * (int64_t)cap * mw;
                for (int e = tid; e < (k - 1) * mw; e += THREADS) {
                    const int x = e / mw, wd = e - x * mw;
                    gc[e] = wd < W ? sm.cond[g][x * W + wd] : 0ull;
                    ga[e] = wd < W ? sm.afar[g][x * W + wd] : 0ull;
                }
            }
            const int nw = ncl < S::CL ? ncl : S::CL;
            int32_t *rec = a.w.clrec + v * (int64_t)CLREC;
            if (tid == 0) a.w.clcnt[v] = nw | (ncl > S::CL ? CL_TRUNC : 0);
            for (int e = tid; e < nw; e += THREADS) {
                rec[4 + 2 * e] = (int32_t)sm.cl_key[g][e];
                rec[5 + 2 * e] = __float_as_int(sm.cl_d[g][e]);
            }
        }
        __syncthreads();  // per-batch shared state is reused next iteration
        cur ^= 1;
    }
    if (a.stats) {
        pairs_local = warp_sum(pairs_local);
        if (lane_id() == 0 && pairs_local) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_PAIRS], pairs_local);
    }
}
