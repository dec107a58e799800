// workspace.cuh -- carving of the caller-provided workspace (device bytes) into the
// per-round scratch the kernels use.  The library never allocates device memory.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace grnnd {

constexpr int NBINS = 8;  // propagate bins by live count k: see propagate.cu
constexpr int HEAVY_SEG = 32;  // segments longer than this are sorted by a CTA
// Redirect-capable pairs of a pool, as the pair phase hands them to decide_kernel: one
// record of CLREC int32 per vertex: [4 + 2c] = (afar << 16) | (anchor pos << 8) | partner
// pos and [5 + 2c] = the pair's exact distance (fp32 bits) for the c < stored count kept;
// clcnt[v] = stored count | CL_TRUNC when the pair kernel found more pairs than its list
// holds (its shared-memory list: <= PAIR_LIST).  A complete list is all decide needs; for an
// incomplete one the full cond / afar masks are written too and decide re-evaluates the
// distances the list lacks.  (16-byte aligned records: bulk-stored by tc3.)
constexpr int PAIR_LIST = 64;
constexpr int32_t CL_TRUNC = 1 << 30;
constexpr int32_t CL_DONE = 1 << 29;  // clcnt: the pool was decided by its pair kernel (lazy.cuh)
constexpr int T3_META_REC = 1344;  // sizeof(T3Meta): 96 x (id, dv, norm: 4 B; pos: 1 B) + 12 x int2
constexpr int CLREC = 4 + 2 * PAIR_LIST;
constexpr int T3Q_CTAS = 256;    // tc3 global candidate overflow: CTAs (>= SMs) x 2 buffers
constexpr int T3Q_GROUP = 4608;  // x entries (>= 96 * 95 / 2 pairs of a group)

// small counters block (unsigned long long so atomicAdd works on it)
enum Counter : int {
    C_LIST = 0,          // messages appended to the emit list this round
    C_BIN0 = 1,          // C_BIN0 + b: vertices in propagate bin b
    C_HEAVY = C_BIN0 + NBINS,  // segments with > HEAVY_SEG entries
    C_OVERFLOW,          // set when the emit list would exceed msg_capacity
    C_BADTGT,            // set when a received message targets a row this rank does not own
    C_NCOUNTERS = 16
};

struct Workspace {
    unsigned long long *ctr;  // [C_NCOUNTERS]
    // emit list (message order irrelevant: the key carries the global order)
    int64_t *e_key;
    int32_t *e_tgt;
    int32_t *e_id;
    float *e_dist;
    // multi-GPU send buffer: the emit list bucketed by owner rank, packed as MSG_WORDS int32
    // per message (key lo, key hi, tgt, id, dist bits) so one all-to-all moves it.  Outside
    // the exchange it is scratch for huge segment sorts (h_key / h_id / h_dist alias it).
    int32_t *o_pack;
    int64_t *h_key;
    int32_t *h_id;
    float *h_dist;
    // inbox grouped by target row; before grouping the same bytes receive the packed
    // messages of the exchange (r_pack)
    int64_t *i_key;
    int32_t *i_id;
    float *i_dist;
    int32_t *r_pack;
    int32_t *in_count;   // [n+1] per-target counts (self-resetting)
    int64_t *starts;     // [n+1]
    int64_t *scan_tmp;   // [scan blocks + 1]
    int2 *bins;          // [NBINS, n] (vertex row, k) lists per propagate bin
    int32_t *heavy;      // [n] heavy segment ids
    uint8_t *pos8;       // [n, pcap] permutation position of each pool slot (this round)
    int32_t pcap;        // pos8 row stride = round_up(cap, 4) (4-byte cp.async rows)
    int32_t cap;
    int32_t mw;          // 64-bit words per mask row = ceil(cap / 64)
    uint64_t *cond;      // [n, cap, mw] redirect-condition bits, row = anchor position
    uint64_t *afar;      // [n, cap, mw] "anchor is the farther member" bits
    int32_t *clrec;      // [n, CLREC] redirect-capable pair records (see PAIR_LIST)
    int32_t *clcnt;      // [n] stored count | CL_TRUNC (zeroed per round; written for pools with records only)
    // tensor-core pair phase (tc3_pairs.cuh): one T3_META_REC-byte metadata record per
    // group of 96 slots -- pool ids, stored distances, row norms, positions, (vertex, k) per
    // pool -- fetched by ONE bulk copy (only carved when cap <= 96)
    unsigned char *s_meta;
    // tc3 MULTI (D > 128): per CTA and queue buffer, the filter candidates beyond the
    // shared-memory queue (a group has <= 96 * 95 / 2 pairs), so no group falls back to an
    // exact sweep of all its pairs from global rows
    uint32_t *t3q;
    uint8_t *dirty;      // [n] pool tombstoned this round (decide sets, the in-place apply clears)
    uint8_t *idle;       // [n] 1: the pool's pair phase is a no-op this round (unchanged since a
                         // round in which it had no redirect-capable pair); set by the apply,
                         // zero (all run) in a fresh workspace and after init
    int64_t n;
    int64_t msg_capacity;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

constexpr int SCAN_ITEMS = 2048;  // elements per scan block
constexpr int MSG_WORDS = 5;       // packed message: int64 key, int32 tgt, int32 id, fp32 dist

inline int64_t scan_blocks(int64_t n) { return (n + SCAN_ITEMS - 1) / SCAN_ITEMS; }

// Layout: computes offsets; with base == nullptr returns the byte size only.
inline size_t carve(Workspace *w, void *base, int64_t n, int32_t cap, int64_t msg_capacity) {
    size_t off = 0;
    auto take = [&](size_t bytes) -> void * {
        off = align_up(off, 256);
        void *p = base ? (void *)((char *)base + off) : nullptr;
        off += bytes;
        return p;
    };
    const size_t C = (size_t)(msg_capacity > 0 ? msg_capacity : 1);
    const size_t N = (size_t)(n > 0 ? n : 1);
    Workspace t;
    t.ctr = (unsigned long long *)take(sizeof(unsigned long long) * C_NCOUNTERS);
    t.e_key = (int64_t *)take(8 * C);
    t.e_tgt = (int32_t *)take(4 * C);
    t.e_id = (int32_t *)take(4 * C);
    t.e_dist = (float *)take(4 * C);
    t.o_pack = (int32_t *)take(4 * MSG_WORDS * C);
    t.h_key = (int64_t *)t.o_pack;
    t.h_id = t.o_pack ? (int32_t *)((char *)t.o_pack + 8 * C) : nullptr;
    t.h_dist = t.o_pack ? (float *)((char *)t.o_pack + 12 * C) : nullptr;
    {
        char *ib = (char *)take(4 * MSG_WORDS * C);  // >= the 16 C bytes of the inbox
        t.r_pack = (int32_t *)ib;
        t.i_key = (int64_t *)ib;
        t.i_id = ib ? (int32_t *)(ib + 8 * C) : nullptr;
        t.i_dist = ib ? (float *)(ib + 12 * C) : nullptr;
    }
    t.in_count = (int32_t *)take(4 * (N + 1));
    t.starts = (int64_t *)take(8 * (N + 1));
    t.scan_tmp = (int64_t *)take(8 * (size_t)(scan_blocks((int64_t)N) + 2 + 128));
    t.bins = (int2 *)take(8 * N * NBINS);
    t.heavy = (int32_t *)take(4 * N);
    t.pcap = (cap > 0 ? cap + 3 : 4) / 4 * 4;
    t.pos8 = (uint8_t *)take(N * (size_t)t.pcap);
    t.cap = cap;
    t.mw = (cap + 63) / 64 > 0 ? (cap + 63) / 64 : 1;
    t.cond = (uint64_t *)take(8 * N * (size_t)(cap > 0 ? cap : 1) * (size_t)t.mw);
    t.afar = (uint64_t *)take(8 * N * (size_t)(cap > 0 ? cap : 1) * (size_t)t.mw);
    t.clrec = (int32_t *)take(4 * N * (size_t)CLREC);
    t.clcnt = (int32_t *)take(4 * N);
    const size_t SG = (cap > 0 && cap <= 96) ? N + 8 : 1;  // staging groups (<= one per pool + bins)
    t.s_meta = (unsigned char *)take((size_t)T3_META_REC * SG);
    t.t3q = (uint32_t *)take((cap > 0 && cap <= 96) ? (size_t)4 * T3Q_CTAS * 2 * T3Q_GROUP : 4);
    t.dirty = (uint8_t *)take(N);
    t.idle = (uint8_t *)take(N);
    t.n = n;
    t.msg_capacity = msg_capacity;
    if (w) *w = t;
    return align_up(off, 256);
}

}  // namespace grnnd
