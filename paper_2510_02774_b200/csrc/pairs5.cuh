// pairs5.cuh -- the pipelined filtered pair phase for D <= 128 (included by propagate.cu
// inside namespace grnnd after tile_dot / record_redirect / exact_sqdist_smem).
//
// Same contract as pairs_kernel<..., DOT = true> (masks + kept distances for decide_kernel,
// bit-identical to the reference), restructured for the B200 memory system:
//  * three-deep software pipeline per persistent CTA: while batch j is computed, the
//    vector rows (+ norms) of batch j+1 and the pool metadata of batch j+2 are in flight
//    (cp.async, no register staging), and the (vertex, k) list entries of batch j+3 are
//    in registers -- no dependent global load sits on the critical path;
//  * rows double-buffered in shared memory (odd float4 stride: conflict free);
//  * large pools (BLOCKED): a warp computes a 4 x 8 block of T x T tiles, so a column
//    of A rows is read by 8 lanes and a column of B rows by 4 lanes (shared-memory
//    broadcast): 2T wavefronts per 4T^2 FFMA per lane instead of ~5T;
//  * small pools (linear): consecutive tiles of up to B pools share the warps.
// The exact re-evaluation of the filter's candidates (C3) and the mask write-out (C5)
// run between two CTA barriers, as before.
#pragma once

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

constexpr int P5_RS4 = 33;  // staged row stride in float4 (128 dims + 1: odd, conflict free)

template <int MAXK, int B>
struct P5Smem {
    static constexpr int W = (MAXK + 63) / 64;
    static constexpr int CL = 64;   // kept redirect distances per pool (overflow: decide re-evaluates)
    static constexpr int QC = 256;  // filter candidates per batch (overflow: exact sweep)
    static constexpr int NBLK = 128;
    // pool metadata, three slots: batch j (in use), j+1 (landed), j+2 (landing)
    int32_t ids[3][B][MAXK];
    float dv[3][B][MAXK];
    uint8_t pos[3][B][MAXK];
    int32_t k[3][B];
    int32_t v[3][B];
    float nrm[2][B][MAXK];  // with the rows: two slots
    uint64_t cond[B][MAXK * W];
    uint64_t afar[B][MAXK * W];
    uint32_t cl_key[B][CL];
    float cl_d[B][CL];
    int cl_n[2][B];
    int qn[2];
    uint32_t q[QC];
    int tp[B + 1];           // linear mode: tile prefix over the batch members
    uint8_t blk[NBLK][2];    // blocked mode: (p, q) of each 4x8 tile block
    int nblk;
};

// p5 counterpart of record_redirect (meta slot ms, counter slot qs)
template <int MAXK, int B>
__device__ __forceinline__ void p5_record(P5Smem<MAXK, B> &sm, int ms, int qs, int g, int s, int u, float d) {
    using S = P5Smem<MAXK, B>;
    constexpr int W = S::W;
    const int x1 = sm.pos[ms][g][s], x2 = sm.pos[ms][g][u];
    const float d1 = sm.dv[ms][g][s], d2 = sm.dv[ms][g][u];
    // anchor = the member visited first (smaller position)
    const int xa = x1 < x2 ? x1 : x2, xb = x1 < x2 ? x2 : x1;
    const float dva = x1 < x2 ? d1 : d2, dvb = x1 < x2 ? d2 : d1;
    const unsigned long long bit = 1ull << (xb & 63);
    atomicOr((unsigned long long *)&sm.cond[g][xa * W + (xb >> 6)], bit);
    if (!(dvb >= dva)) atomicOr((unsigned long long *)&sm.afar[g][xa * W + (xb >> 6)], bit);
    const int c = atomicAdd(&sm.cl_n[qs][g], 1);
    if (c < S::CL) {
        sm.cl_key[g][c] = (uint32_t)((xa << 8) | xb);
        sm.cl_d[g][c] = d;
    }
}

template <int MAXK, int B, int NW, int T, bool BLOCKED, int NQ>
__global__ void __launch_bounds__(NW * 32) pairs5_kernel(PropArgs a, int bin, int kmax) {
    using S = P5Smem<MAXK, B>;
    constexpr int THREADS = NW * 32;
    constexpr int W = S::W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S &sm = *reinterpret_cast<S *>(smem_raw);
    float4 *slabs = reinterpret_cast<float4 *>(smem_raw + align_up(sizeof(S), 128));
    const int slab_f4 = B * kmax * P5_RS4;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nbin = (int64_t)a.w.ctr[C_BIN0 + bin];
    const int64_t nbatch = (nbin + B - 1) / B;
    const int2 *blist = a.w.bins + (int64_t)bin * a.w.n;
    const int nq = NQ > 0 ? NQ : (a.dim + 3) >> 2;
    const int cap = a.cap, pcap = a.w.pcap, mw = a.w.mw;
    const float eps_n = a.eps_n, eps_h = a.eps_h;
    const int64_t G = gridDim.x;
    if ((int64_t)blockIdx.x >= nbatch) return;
    const int64_t nmine = (nbatch - blockIdx.x + G - 1) / G;  // batches j = 0.. of this CTA
    unsigned long long pairs_local = 0;

    auto load_vk = [&](int64_t j, int2 (&vk)[B]) {
#pragma unroll
        for (int g = 0; g < B; ++g) {
            vk[g] = make_int2(-1, 0);
            if (j < nmine) {
                const int64_t e = (blockIdx.x + j * G) * B + g;
                if (e < nbin) vk[g] = blist[e];
            }
        }
    };
    // publish (v, k) of batch j into meta slot j % 3 and start its id / dist / pos copies
    auto issue_meta = [&](int64_t j, const int2 (&vk)[B]) {
        const int sl = (int)(j % 3);
#pragma unroll
        for (int g = 0; g < B; ++g) {
            if (tid == 0) {
                sm.v[sl][g] = vk[g].x;
                sm.k[sl][g] = vk[g].y;
            }
            const int kg = vk[g].y;
            const int64_t v = vk[g].x;
            for (int s = tid; s < kg; s += THREADS) {
                cp_async4(&sm.ids[sl][g][s], a.read_ids + v * cap + s, true);
                cp_async4(&sm.dv[sl][g][s], a.read_dists + v * cap + s, true);
            }
            if (a.order_code == 0)
                for (int c = tid; c < (kg + 3) >> 2; c += THREADS)
                    cp_async4(&sm.pos[sl][g][c * 4], a.w.pos8 + v * pcap + c * 4, true);
        }
    };
    // start the vector-row and norm copies of batch j (its metadata has landed)
    auto issue_rows = [&](int64_t j) {
        const int sl = (int)(j % 3), rs = (int)(j & 1);
        float4 *slab = slabs + rs * slab_f4;
#pragma unroll
        for (int g = 0; g < B; ++g) {
            const int kg = sm.k[sl][g];
            const int total = kg * nq;
            for (int e = tid; e < total; e += THREADS) {
                const int r = e / nq;
                const int c = e - r * nq;
                const int32_t id = sm.ids[sl][g][r];
                cp_async16(&slab[(g * kmax + r) * P5_RS4 + c],
                           a.data + (int64_t)(id < 0 ? 0 : id) * a.ld + (int64_t)c * 4, id >= 0);
            }
            for (int s = tid; s < kg; s += THREADS) {
                const int32_t id = sm.ids[sl][g][s];
                cp_async4(&sm.nrm[rs][g][s], a.norms + (id < 0 ? 0 : id), id >= 0);
            }
        }
    };

    // ---- prologue: metadata of batches 0 and 1, rows of batch 0, (v, k) of batch 2 ----
    int2 vkr[B];
    load_vk(0, vkr);
    issue_meta(0, vkr);
    load_vk(1, vkr);
    issue_meta(1, vkr);
    cp_async_commit();
    for (int i = tid; i < B * MAXK * W; i += THREADS) {
        (&sm.cond[0][0])[i] = 0ull;
        (&sm.afar[0][0])[i] = 0ull;
    }
    if (tid < 2) sm.qn[tid] = 0;
    if (tid < 2 * B) (&sm.cl_n[0][0])[tid] = 0;
    cp_async_wait_all();
    __syncthreads();
    issue_rows(0);
    cp_async_commit();
    load_vk(2, vkr);

    for (int64_t j = 0; j < nmine; ++j) {
        const int ms = (int)(j % 3), rs = (int)(j & 1), qs = (int)(j & 1);
        const float4 *slab = slabs + rs * slab_f4;
        // ---- A: schedule of batch j (its k landed two iterations ago) ----
        if (tid == 0) {
            if (!BLOCKED) {
                int t = 0;
#pragma unroll
                for (int g = 0; g < B; ++g) {
                    sm.tp[g] = t;
                    const int nb = (sm.k[ms][g] + T - 1) / T;
                    t += nb * (nb + 1) / 2;
                }
                sm.tp[B] = t;
            } else {
                const int nb = (sm.k[ms][0] + T - 1) / T;
                int c = 0;
                for (int qq = 0; qq * 8 < nb; ++qq)
                    for (int p = 0; p * 4 < nb && p * 4 <= qq * 8 + 7; ++p)
                        if (c < S::NBLK) {
                            sm.blk[c][0] = (uint8_t)p;
                            sm.blk[c][1] = (uint8_t)qq;
                            ++c;
                        }
                sm.nblk = c;
            }
        }
        cp_async_wait_all();
        __syncthreads();  // rows + norms of j, metadata of j+1 landed; schedule visible
        // ---- B: keep the pipeline full ----
        if (j + 1 < nmine) issue_rows(j + 1);
        if (j + 2 < nmine) issue_meta(j + 2, vkr);
        cp_async_commit();
        load_vk(j + 3, vkr);
        if (tid == 0) {
            sm.qn[qs ^ 1] = 0;
#pragma unroll
            for (int g = 0; g < B; ++g) sm.cl_n[qs ^ 1][g] = 0;
        }
        // ---- C0: ascending debug order (:75-87): rank by (dist, id), published for decide ----
        if (a.order_code != 0) {
#pragma unroll
            for (int g = 0; g < B; ++g) {
                const int k = sm.k[ms][g];
                for (int s = tid; s < k; s += THREADS) {
                    const float ds = sm.dv[ms][g][s];
                    const int32_t is = sm.ids[ms][g][s];
                    int r = 0;
                    for (int t = 0; t < k; ++t) {
                        const float dt = sm.dv[ms][g][t];
                        const int32_t it2 = sm.ids[ms][g][t];
                        r += (dt < ds || (dt == ds && (it2 < is || (it2 == is && t < s)))) ? 1 : 0;
                    }
                    sm.pos[ms][g][s] = (uint8_t)r;
                    a.w.pos8[(int64_t)sm.v[ms][g] * pcap + s] = (uint8_t)r;
                }
            }
        }
        // ---- C1: filtered tiles -> candidate queue ----
        auto epilogue = [&](int g, const float(&acc)[T * T], int bI, int bJ, int nb, int k) {
            float dA[T], dB[T], nA[T], nB[T];
            bool vA[T], vB[T];
#pragma unroll
            for (int i = 0; i < T; ++i) {
                const int s = bI + nb * i, u = bJ + nb * i;
                vA[i] = bI < nb && s < k && sm.ids[ms][g][s] != TOMB;
                vB[i] = bJ < nb && u < k && sm.ids[ms][g][u] != TOMB;
                dA[i] = vA[i] ? sm.dv[ms][g][s] : 0.0f;
                dB[i] = vB[i] ? sm.dv[ms][g][u] : 0.0f;
                nA[i] = vA[i] ? sm.nrm[rs][g][s] : 0.0f;
                nB[i] = vB[i] ? sm.nrm[rs][g][u] : 0.0f;
            }
            unsigned np = 0;
#pragma unroll
            for (int i = 0; i < T; ++i)
#pragma unroll
                for (int jj = 0; jj < T; ++jj) {
                    const bool valid = vA[i] && vB[jj] && (bI < bJ || (bI == bJ && i < jj));
                    np += valid ? 1u : 0u;
                    const float hi = dA[i] >= dB[jj] ? dA[i] : dB[jj];
                    const float nn = nA[i] + nB[jj];
                    const float dap = fmaf(-2.0f, acc[i * T + jj], nn);
                    const float e = fmaf(eps_n, nn, fmaf(eps_h, hi, 1e-30f));
                    // settled iff d~ >= hi + E with finite norms; NaN / overflow fall through
                    if (valid && !(dap >= hi + e && nn <= 3.0e38f)) {
                        const int c = atomicAdd(&sm.qn[qs], 1);
                        if (c < S::QC)
                            sm.q[c] = (uint32_t)((g << 16) | ((bI + nb * i) << 8) | (bJ + nb * jj));
                    }
                }
            return np;
        };
        if (!BLOCKED) {
            const int ntiles = sm.tp[B];
            for (int t = tid; t < ntiles; t += THREADS) {
                int g = 0;
#pragma unroll
                for (int h = 1; h < B; ++h) g += t >= sm.tp[h] ? 1 : 0;
                int bI, bJ;
                tile_decode(t - sm.tp[g], bI, bJ);
                const int kg = sm.k[ms][g];
                const int nb = (kg + T - 1) / T;
                float acc[T * T];
#pragma unroll
                for (int p = 0; p < T * T; ++p) acc[p] = 0.0f;
                tile_dot<T, NQ>(acc, slab, g * kmax + bI, g * kmax + bJ, nb, nq, P5_RS4);
                pairs_local += epilogue(g, acc, bI, bJ, nb, kg);
            }
        } else {
            const int kg = sm.k[ms][0];
            const int nb = (kg + T - 1) / T;
            const int nblk = sm.nblk;
            const int li = lane >> 3, lj = lane & 7;
            for (int b = warp; b < nblk; b += NW) {
                const int bI = sm.blk[b][0] * 4 + li, bJ = sm.blk[b][1] * 8 + lj;
                // lanes outside the triangle compute a clamped (in-bounds) tile and discard it
                const int cI = bI < nb ? bI : nb - 1, cJ = bJ < nb ? bJ : nb - 1;
                float acc[T * T];
#pragma unroll
                for (int p = 0; p < T * T; ++p) acc[p] = 0.0f;
                tile_dot<T, NQ>(acc, slab, cI, cJ, nb, nq, P5_RS4);
                pairs_local += epilogue(0, acc, bI, bJ, nb, kg);
            }
        }
        __syncthreads();  // C2: candidate queue complete
        // ---- C3: exact re-evaluation of the candidates ----
        {
            const int qn = sm.qn[qs];
            if (qn <= S::QC) {
                for (int e = tid; e < qn; e += THREADS) {
                    const uint32_t key = sm.q[e];
                    const int g = (int)(key >> 16), s = (int)((key >> 8) & 255u), u = (int)(key & 255u);
                    const float d = exact_sqdist_smem(slab + (g * kmax + s) * P5_RS4,
                                                      slab + (g * kmax + u) * P5_RS4, nq);
                    const float d1 = sm.dv[ms][g][s], d2 = sm.dv[ms][g][u];
                    if (d < (d1 >= d2 ? d1 : d2)) p5_record(sm, ms, qs, g, s, u, d);
                }
            } else {
                // queue overflow (degenerate data: many near-ties): exact sweep of every pair
#pragma unroll
                for (int g = 0; g < B; ++g) {
                    const int k = sm.k[ms][g];
                    const int np = k * (k - 1) / 2;
                    for (int p = tid; p < np; p += THREADS) {
                        int s, u;
                        tile_decode(p, s, u);
                        u += 1;
                        if (sm.ids[ms][g][s] == TOMB || sm.ids[ms][g][u] == TOMB) continue;
                        const float d = exact_sqdist_smem(slab + (g * kmax + s) * P5_RS4,
                                                          slab + (g * kmax + u) * P5_RS4, nq);
                        const float d1 = sm.dv[ms][g][s], d2 = sm.dv[ms][g][u];
                        if (d < (d1 >= d2 ? d1 : d2)) p5_record(sm, ms, qs, g, s, u, d);
                    }
                }
            }
        }
        __syncthreads();  // C4: masks + kept distances complete
        // ---- C5: masks + kept distances -> global (decide_kernel); masks re-zeroed ----
#pragma unroll
        for (int g = 0; g < B; ++g) {
            const int64_t v = sm.v[ms][g];
            if (v < 0) continue;
            const int k = sm.k[ms][g];
            uint64_t *gc = a.w.cond + v * (int64_t)cap * mw;
            uint64_t *ga = a.w.afar + v * (int64_t)cap * mw;
            for (int e = tid; e < (k - 1) * mw; e += THREADS) {
                const int x = e / mw, wd = e - x * mw;
                uint64_t c = 0ull, f = 0ull;
                if (wd < W) {
                    c = sm.cond[g][x * W + wd];
                    f = sm.afar[g][x * W + wd];
                    sm.cond[g][x * W + wd] = 0ull;
                    sm.afar[g][x * W + wd] = 0ull;
                }
                gc[e] = c;
                ga[e] = f;
            }
            const int lcap = S::CL < 4 * cap ? S::CL : 4 * cap;
            const int ncl = sm.cl_n[qs][g];
            const int nw = ncl < lcap ? ncl : lcap;
            if (tid == 0) a.w.cl_n[v] = nw;  // truncated lists: decide re-evaluates misses
            for (int e = tid; e < nw; e += THREADS) {
                a.w.cl[v * 4 * (int64_t)cap + e] = sm.cl_key[g][e];
                a.w.cl_d[v * 4 * (int64_t)cap + e] = sm.cl_d[g][e];
            }
        }
    }
    if (a.stats) {
        pairs_local = warp_sum(pairs_local);
        if (lane == 0 && pairs_local) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_PAIRS], pairs_local);
    }
}
