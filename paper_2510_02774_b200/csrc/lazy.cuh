// lazy.cuh -- anchor-serial, partner-parallel pair phase for small pools (k <= 32, D <= 128)
// of the round API.  Included by propagate.cu inside namespace grnnd after decide_pool.
//
// The reference's loop (_numba_kernels.py:151-185) evaluates a pair only when both members
// are still live when the pair's anchor is visited; in the first rounds of a build (random
// pools, most pairs redirect) that is 17-29% of all pairs (C2 rounds 1-3).  The exact
// CUDA-core kernel (pairs.cuh) computes every pair and decide_kernel replays the rule; this
// kernel IS the rule: a warp owns a pool, stages its rows in shared memory, and visits the
// anchors in permutation order -- lane y holds the row of the member at position y in
// registers, so at each live anchor the lanes after it compute the reference's exact
// sequential distance to the anchor (a shared-memory broadcast) in parallel, and the
// anchor's messages and tombstones follow from one ballot (the anchor-serial,
// partner-parallel formulation is bit-identical).  It emits straight into the message list
// (keys = source * R + emission index, the reference's order) and marks the pool decided.
#pragma once

constexpr int LZ_WARPS = 4;        // warps per CTA
constexpr int LZ_RS4 = 33;         // staged row stride in float4 (odd: lanes on distinct banks)

struct LazyWarp {
    float4 rows[32 * LZ_RS4];      // the pool's rows, slot order
    int32_t ids[32];
    float dv[32];
    int8_t perm[32];               // position -> slot
    int32_t e_tgt[32], e_id[32];   // this pool's messages, emission order
    float e_d[32];
};

__global__ void __launch_bounds__(LZ_WARPS * 32, 3) lazy_pairs_kernel(PropArgs a) {
    extern __shared__ __align__(16) unsigned char lz_raw[];
    const int lane = lane_id(), wib = threadIdx.x >> 5;
    LazyWarp &sm = reinterpret_cast<LazyWarp *>(lz_raw)[wib];
    const int cap = a.cap;
    const int nq = (a.dim + 3) >> 2;
    const int64_t n1 = (int64_t)a.w.ctr[C_BIN0 + 1], n2 = (int64_t)a.w.ctr[C_BIN0 + 2];
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long red = 0, refp = 0, pools = 0;

    for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n1 + n2; e += warps) {
        const int2 vk = e < n1 ? a.w.bins[(int64_t)1 * a.w.n + e] : a.w.bins[(int64_t)2 * a.w.n + (e - n1)];
        const int64_t v = vk.x;
        const int k = vk.y;  // 2 <= k <= 32
        // pool row, positions, staged vectors
        int32_t myid = TOMB;
        if (lane < k) {
            myid = a.read_ids[v * cap + lane];
            sm.ids[lane] = myid;
            sm.dv[lane] = a.read_dists[v * cap + lane];
            sm.perm[a.w.pos8[v * a.w.pcap + lane]] = (int8_t)lane;
        }
        __syncwarp();
        for (int s = 0; s < k; ++s) {  // row s: lane = 16-byte chunk (coalesced 512-byte row)
            const int32_t id = sm.ids[s];
            if (lane < nq) cp_async16(&sm.rows[s * LZ_RS4 + lane], a.data + (int64_t)(id < 0 ? 0 : id) * a.ld + lane * 4, id >= 0);
        }
        cp_async_commit();
        cp_async_wait_all();
        __syncwarp();

        // lane y owns the pool member at permutation position y: its row moves to registers
        // once, so a step reads only the anchor's row from shared memory (a broadcast)
        const int myslot = lane < k ? sm.perm[lane] : 0;
        float4 mine[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) mine[q] = q < nq ? sm.rows[myslot * LZ_RS4 + q] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float mydv = lane < k ? sm.dv[myslot] : 0.0f;
        // live[x] over positions (entries are live at the start of the round; TOMB slots dead)
        unsigned live = __ballot_sync(FULL, lane < k && sm.ids[myslot] != TOMB);
        int nm = 0;
        for (int x = 0; x < k - 1; ++x) {
            if (!((live >> x) & 1u)) continue;  // warp-uniform
            const int sa = sm.perm[x];
            const bool py = lane > x && lane < k && ((live >> lane) & 1u);  // partner = position `lane`
            float d = 0.0f;
            if (py) {
                const float4 *ra = &sm.rows[sa * LZ_RS4];
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    if (q < nq) {
                        const float4 u = ra[q], w = mine[q];
                        d = exact_step4(d, u, w);
                    }
                }
            }
            const float dva = sm.dv[sa], dvb = mydv;
            const bool cond = py && d < (dva >= dvb ? dva : dvb);
            const bool far = cond && !(dvb >= dva);  // the anchor is the farther member
            const unsigned fm = __ballot_sync(FULL, far);
            const int fl = fm ? __ffs(fm) - 1 : 32;  // position of the first anchor-far partner
            const unsigned vis = __ballot_sync(FULL, py) & (fl < 32 ? (fl == 31 ? FULL : ((2u << fl) - 1u)) : FULL);
            refp += (unsigned long long)__popc(vis);
            const unsigned em = __ballot_sync(FULL, cond && !far) & (fl < 32 ? ((1u << fl) - 1u) : FULL);
            // partner-far messages in position order: (tgt = anchor, id = partner); partners die
            if ((em >> lane) & 1u) {
                const int j = nm + __popc(em & ((1u << lane) - 1u));
                sm.e_tgt[j] = sm.ids[sa];
                sm.e_id[j] = sm.ids[myslot];
                sm.e_d[j] = d;
            }
            nm += __popc(em);
            live &= ~em;
            if (fl < 32) {  // the anchor is redirected to its first anchor-far partner and dies
                if (lane == fl) {
                    sm.e_tgt[nm] = sm.ids[myslot];
                    sm.e_id[nm] = sm.ids[sa];
                    sm.e_d[nm] = d;
                }
                ++nm;
                live &= ~(1u << x);
            }
            __syncwarp();
        }
        // live anchors never visited as partners: the last position has no later partner
        red += (unsigned long long)nm;
        if (nm > 0) {
            ++pools;
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(&a.w.ctr[C_LIST], (unsigned long long)nm);
            base = __shfl_sync(FULL, base, 0);
            if (lane < nm) {
                const unsigned long long p = base + (unsigned long long)lane;
                if (p < (unsigned long long)a.w.msg_capacity) {
                    a.w.e_key[p] = (a.lo + v) * cap + lane;
                    a.w.e_tgt[p] = sm.e_tgt[lane];
                    a.w.e_id[p] = sm.e_id[lane];
                    a.w.e_dist[p] = sm.e_d[lane];
                } else {
                    a.w.ctr[C_OVERFLOW] = 1ull;
                }
            }
            // tombstones (read_ids mutated in place, as the reference does)
            if (lane < k && myid != TOMB) {
                const int x = a.w.pos8[v * a.w.pcap + lane];
                if (!((live >> x) & 1u)) a.read_ids[v * cap + lane] = TOMB;
            }
            if (lane == 0) a.w.dirty[v] = 1;
        }
        if (lane == 0) a.w.clcnt[v] = CL_DONE;  // decide_kernel: nothing left for this pool
        __syncwarp();
    }
    if (a.stats) {  // (red, refp, pools: warp-uniform; lane 0 adds them)
        if (lane == 0) {
            if (red) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_REDIRECTS], red);
            if (refp) {
                atomicAdd((unsigned long long *)&a.stats[GRNND_ST_PAIRS_REF], refp);
                atomicAdd((unsigned long long *)&a.stats[GRNND_ST_PAIRS], refp);
            }
            if (pools) atomicAdd((unsigned long long *)&a.stats[GRNND_ST_RECPOOLS], pools);
        }
    }
}
