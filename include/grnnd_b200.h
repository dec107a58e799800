/*
 * grnnd_b200.h -- C ABI of libgrnnd_b200.so, the B200 (sm_100a) GRNND graph builder.
 *
 * Two layers, both plain pointers + sizes, no torch types:
 *
 *  (1) Kernel-module entry points.  One per function of the reference's
 *      operator layer, the kernel module returned by grnnd.backend.get_kernels()
 *      (/root/reference/pkg/src/grnnd/backend.py:58-64), with the same argument
 *      meaning, the same in-place mutation of caller-owned arrays and the same
 *      "no exceptions, status via flag" convention.  The
 *      arrays are DEVICE pointers; paper_2510_02774_b200/kernels.py wraps them
 *      in a numpy-in/numpy-out module with the reference's exact signatures.
 *
 *  (2) The fused round API used by paper_2510_02774_b200.build(): whole update /
 *      reverse rounds as one asynchronous call each, on device-resident pools
 *      (replaces builder.update_round / reverse_edge_sampling / finalize_graph,
 *      /root/reference/pkg/src/grnnd/builder.py:283-362).
 *
 * Conventions: every function returns GRNND_OK (0) or an error code and never
 * aborts; grnnd_last_error() describes the last failure on the calling thread.
 * Calls are asynchronous on the given CUDA stream (NULL = legacy default
 * stream); only functions documented as synchronising wait on the device.
 * Device buffers belong to the caller (PyTorch tensors in the Python layer);
 * the library never frees caller memory and keeps no device allocations of
 * its own.  Ids are int32 with TOMBSTONE = -1 (core.py:22); distances are
 * squared L2 in fp32, accumulated sequentially with separately rounded
 * sub/mul/add exactly as the reference's _sqdist (_numba_kernels.py:50-56).
 */
#ifndef GRNND_B200_H
#define GRNND_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GRNND_OK 0
#define GRNND_EINVAL 1       /* bad argument (maps to ParamError in Python)        */
#define GRNND_ECUDA 2        /* CUDA runtime / launch failure                        */
#define GRNND_EUNSUPPORTED 3 /* shape outside what the kernels were built for        */
#define GRNND_EWORKSPACE 4   /* workspace too small                                  */

#define GRNND_TOMBSTONE (-1)
#define GRNND_MAX_CAP 256 /* largest pool capacity R the kernels are compiled for */

/* RoundStats fields (builder.py:102-114), device int64 counters */
enum {
    GRNND_ST_MESSAGES = 0,
    GRNND_ST_REDIRECTS = 1,
    GRNND_ST_SURVIVORS = 2,
    GRNND_ST_REVERSE_ATTEMPTS = 3,
    GRNND_ST_INSERTED = 4,
    GRNND_ST_DUPLICATE = 5,
    GRNND_ST_REPLACED = 6,
    GRNND_ST_REJECTED = 7,
    GRNND_ST_PAIRS = 8,     /* pair distances computed (all live pairs; instrumentation) */
    GRNND_ST_PAIRS_REF = 9, /* pairs the reference loop would evaluate (instrumentation) */
    GRNND_ST_CANDIDATES = 10, /* pairs the filtered pair phase re-evaluated exactly (instrumentation) */
    GRNND_ST_OVERFLOWS = 11,  /* groups whose candidate queue overflowed into an exact sweep */
    GRNND_ST_REDIRECTABLE = 12, /* pairs meeting the redirect condition (instrumentation)      */
    GRNND_ST_RECPOOLS = 14,   /* pools with at least one redirect-capable pair (instrumentation) */
    GRNND_ST_ACTIVE_K = 15,   /* pool entries whose pair phase ran (the rest: pools unchanged since a
                                 round in which they had no redirect-capable pair -- a no-op) */
    GRNND_ST_LOST = 13,       /* messages a round could not hold (emit list beyond msg_capacity)
                                 or that reached the wrong rank: non-zero = the round is invalid,
                                 the Python layer raises DeviceError (GRNND_EWORKSPACE meaning) */
    /* validation builds only (-DGRNND_TC_VALIDATE, libgrnnd_b200_tcv.so): the tensor-core
       pre-screen's error against its rigorous bound, checked on every screened pair */
    GRNND_ST_TCV_CHECKED = 16,    /* pairs whose screened distance was compared with the exact one */
    GRNND_ST_TCV_MAX_RATIO = 17,  /* max |d~ - d| / bound, fp32 bits (ratio >= 0)                  */
    GRNND_ST_TCV_VIOLATIONS = 18, /* pairs with |d~ - d| > bound (must stay 0)                     */
    GRNND_NSTATS = 20
};

typedef void *grnnd_stream_t; /* a cudaStream_t */

const char *grnnd_last_error(void);
int grnnd_abi_version(void);
/* kernels launched by this library since load (host-side counter; for launch accounting) */
unsigned long long grnnd_launch_count(void);
/* costly instrumentation counters (GRNND_ST_PAIRS_REF: the reference-semantics pair count,
   ~20% of the decide kernel's instructions) on / off for later launches; off by default
   (the counter then stays 0).  Returns the previous setting. */
int grnnd_set_instrumentation(int on);

/* ------------------------------------------------------------------------ */
/* (1) kernel-module entry points (device pointers)                          */
/* ------------------------------------------------------------------------ */

/* rng.hash4 / _numba_kernels.hash4_u64 (rng.py:34-41), elementwise over m (v, i) pairs */
int grnnd_hash4_batch(uint64_t seed, uint64_t stream, const uint64_t *v, const uint64_t *i,
                      int64_t m, uint64_t *out, grnnd_stream_t s);

/* _numba_kernels.sqdist (:59-61): out[r] = sqdist(a[r,:], b[r,:]) for m row pairs */
int grnnd_sqdist_batch(const float *a, const float *b, int64_t m, int32_t dim, float *out,
                       grnnd_stream_t s);

/* _numba_kernels.sample_initial (:91-115): out int32[n,count]; *fail_flag set to 1 on failure */
int grnnd_sample_initial(int64_t n, int32_t count, uint64_t seed, int32_t *out,
                         int64_t *fail_flag, grnnd_stream_t s);

/* _numba_kernels.init_dists (:118-122): data fp32[n, ld] (first dim columns used) */
int grnnd_init_dists(const float *data, int64_t n, int32_t dim, int32_t ld, const int32_t *ids,
                     int32_t count, float *out, grnnd_stream_t s);

/* Workspace the message-generating / grouping entry points need (bytes). */
size_t grnnd_workspace_bytes(int64_t n, int32_t cap, int64_t msg_capacity);

/* _numba_kernels.gen_update_messages (:125-192).  Writes per-vertex message
 * slices (redirects in discovery order, then survivors in slot order) and
 * tombstones redirected slots of read_ids in place. */
int grnnd_gen_update_messages(const float *data, int64_t n, int32_t dim, int32_t ld,
                              int32_t *read_ids, const float *read_dists,
                              const int32_t *read_count, int32_t cap, uint64_t seed,
                              uint64_t stream_id, int32_t order_code, int32_t *msg_tgt,
                              int32_t *msg_id, float *msg_dist, int32_t *msg_cnt,
                              void *workspace, size_t workspace_bytes, grnnd_stream_t s);

/* _numba_kernels.gen_reverse_messages (:195-233) */
int grnnd_gen_reverse_messages(const int32_t *read_ids, const float *read_dists,
                               const int32_t *read_count, int64_t n, int32_t cap, double rho,
                               int32_t *msg_tgt, int32_t *msg_id, float *msg_dist,
                               int32_t *msg_cnt, grnnd_stream_t s);

/* _numba_kernels.gen_merge_messages (:236-250) */
int grnnd_gen_merge_messages(const int32_t *read_ids, const float *read_dists,
                             const int32_t *read_count, int64_t n, int32_t cap, int32_t *msg_tgt,
                             int32_t *msg_id, float *msg_dist, int32_t *msg_cnt,
                             grnnd_stream_t s);

/* build_flat step 1 (:265-270): offs int64[n+1] = exclusive prefix of msg_cnt (device). */
int grnnd_message_offsets(const int32_t *msg_cnt, int64_t n, int64_t *offs, void *workspace,
                          size_t workspace_bytes, grnnd_stream_t s);

/* build_flat step 2 / _compact (:253-262): pack slices vertex-major using offs. */
int grnnd_compact_messages(const int32_t *msg_tgt, const int32_t *msg_id, const float *msg_dist,
                           const int32_t *msg_cnt, int64_t n, int32_t cap, const int64_t *offs,
                           int32_t *flat_tgt, int32_t *flat_id, float *flat_dist,
                           int32_t *flat_src, grnnd_stream_t s);

/* group_by_target (:279-300): stable grouping; order int64[m], starts int64[n+1]. */
int grnnd_group_by_target(const int32_t *flat_tgt, int64_t m, int64_t n, int64_t *order,
                          int64_t *starts, void *workspace, size_t workspace_bytes,
                          grnnd_stream_t s);

/* apply_grouped_messages (:303-351).  outcomes: device int64[4] (ins, dup, rep, rej),
 * accumulated (caller zeroes). */
int grnnd_apply_grouped_messages(int32_t *write_ids, float *write_dists, int32_t *write_count,
                                 int64_t n, int32_t cap, const int32_t *flat_id,
                                 const float *flat_dist, const int64_t *order,
                                 const int64_t *starts, int64_t *outcomes, grnnd_stream_t s);

/* ------------------------------------------------------------------------ */
/* (2) fused round API on device-resident double-buffered pools              */
/* ------------------------------------------------------------------------ */

typedef struct {
    const float *data; /* fp32 [n_total, ld], replicated on every rank                     */
    int64_t n_total;   /* global vertex count                                              */
    int64_t lo, hi;    /* owned vertex range [lo, hi) (0, n_total on one GPU)              */
    int32_t dim, ld, cap;
    int32_t *read_ids; /* int32 [hi-lo, cap]   row r = vertex lo + r                       */
    float *read_dists; /* fp32  [hi-lo, cap]                                               */
    int32_t *read_count;
    int32_t *write_ids;
    float *write_dists;
    int32_t *write_count;
    void *workspace;   /* >= grnnd_workspace_bytes(hi-lo, cap, msg_capacity)               */
    size_t workspace_bytes;
    int64_t msg_capacity; /* messages one round may emit / receive on this rank             */
    int64_t *stats;    /* device int64 [GRNND_NSTATS], accumulated by the round calls      */
    const float *norms; /* fp32 [n_total] squared row norms (grnnd_row_norms) enabling the
                           filtered pair phase, or NULL for the exact-only pair phase; the
                           built graph is the same either way                              */
    int32_t filter_split; /* 1: the tensor-core Gram as hi*hi + hi*lo + lo*hi (split TF32,
                           ~fp32 accurate: a band 2^7 narrower) for data far from the origin
                           relative to its neighbour distances; 0: plain TF32            */
} grnnd_pools;

/* Squared L2 norm of every row of data[n, ld] (first dim columns) into out[n] (device).
 * Feeds grnnd_pools.norms: the pair phase then pre-screens pairs with FFMA dot products
 * and re-evaluates only the pairs within a rigorous error bound of the redirect
 * threshold exactly, so every decision and distance stays bit-identical. */
int grnnd_row_norms(const float *data, int64_t n, int32_t dim, int32_t ld, float *out,
                    grnnd_stream_t s);

/* Width of the tensor-core filter's error band relative to the pools' distances: out
 * (device double[2]) = (sum over every read entry of |member|^2 / its stored distance,
 * number of entries).
 * The band is 2^-8 (|a|^2 + |b|^2) wide, so data far from the origin relative to its
 * neighbour distances (clustered, all-positive descriptors) makes most pairs candidates; the
 * host then keeps the exact pair phase (the graph is the same either way). */
int grnnd_band_terms(const grnnd_pools *p, double *out, grnnd_stream_t s);

/* builder.init_neighbors (:221-257): sample S ids, their distances, count = S.
 * fail_flag: device int64[1]. */
int grnnd_init_pools(const grnnd_pools *p, int32_t S, uint64_t seed, int64_t *fail_flag,
                     grnnd_stream_t s);

/* builder.update_round (:283-312) minus the buffer swap (the caller swaps pointers).
 * One GPU: everything on device, asynchronous. */
int grnnd_update_round(const grnnd_pools *p, uint64_t seed, uint64_t stream_id,
                       int32_t order_code, grnnd_stream_t s);

/* builder.reverse_edge_sampling (:315-339) minus the swap. */
int grnnd_reverse_round(const grnnd_pools *p, double rho, grnnd_stream_t s);

/* The two halves of a round, for per-phase timing: emit (pair phase / reverse selection
 * into the message list) then apply (group by target + pool insert).  update_round ==
 * update_emit + apply_emitted(kind 0); reverse_round == reverse_emit + apply_emitted(1). */
int grnnd_update_emit(const grnnd_pools *p, uint64_t seed, uint64_t stream_id,
                      int32_t order_code, grnnd_stream_t s);
int grnnd_reverse_emit(const grnnd_pools *p, double rho, grnnd_stream_t s);
int grnnd_apply_emitted(const grnnd_pools *p, int32_t kind, grnnd_stream_t s);

/* Multi-GPU split of a round.  emit: pair phase (or reverse selection) of owned
 * vertices into the outgoing message list, bucketed by owner rank.  The host then
 * exchanges the buckets (NCCL all-to-all) into the incoming list and calls
 * grnnd_round_apply. See paper_2510_02774_b200/sharded.py. */
int grnnd_round_emit(const grnnd_pools *p, int32_t kind /*0 update, 1 reverse*/, uint64_t seed,
                     uint64_t stream_id, int32_t order_code, double rho,
                     const int64_t *rank_bounds /*device int64[nranks+1]*/, int32_t nranks,
                     int64_t *send_counts /*device int64[nranks]*/, grnnd_stream_t s);
/* Device pointers to the packed outgoing (bucketed by rank, send_counts[r] messages for
 * rank r in rank order) and incoming message buffers inside the workspace; each message is
 * GRNND_MSG_WORDS int32 (key low, key high, tgt, id, dist bits), so one all-to-all moves a
 * round's payload.  Capacity: msg_capacity messages each. */
#define GRNND_MSG_WORDS 5
int grnnd_round_buffers(const grnnd_pools *p, int32_t **out_pack, int32_t **in_pack);
/* Apply the n_incoming packed messages received (in source-rank order) in in_pack. */
int grnnd_round_apply(const grnnd_pools *p, int32_t kind, int64_t n_incoming, grnnd_stream_t s);

/* builder.finalize_graph (:342-362): rows sorted by (dist, id) into CSR.
 * offsets int64[n+1] (device), nbrs int32[sum(counts)] (device).  The Graph.validate
 * checks of core.py:171-201 run in the same pass: *bad_flag (device int64, nullable)
 * gets bit 0 = id out of range, bit 1 = self loop, bit 2 = duplicate within a row. */
int grnnd_finalize(const int32_t *ids, const float *dists, const int32_t *counts, int64_t n,
                   int32_t cap, int64_t *offsets, int32_t *nbrs, int64_t *bad_flag,
                   void *workspace, size_t workspace_bytes, grnnd_stream_t s);

/* grnnd_finalize on the read side of a (possibly sharded) pool set: rows lo..hi-1, ids
 * validated against [0, n_total) and the global owner id. */
int grnnd_finalize_pools(const grnnd_pools *p, int64_t *offsets, int32_t *nbrs, int64_t *bad_flag,
                         grnnd_stream_t s);

/* Dataset.validate finiteness scan (core.py:70-71) on device: *bad_flag = 1 if any of the
 * first dim columns of data[n, ld] is NaN/inf. */
int grnnd_check_finite(const float *data, int64_t n, int32_t dim, int32_t ld, int64_t *bad_flag,
                       grnnd_stream_t s);

/* Row-sorted fixed-degree view (the fixed-degree int32 [n, cap] adjacency, -1 padded). */
int grnnd_sorted_rows(const int32_t *ids, const float *dists, const int32_t *counts, int64_t n,
                      int32_t cap, int32_t *out_ids, grnnd_stream_t s);

/* ------------------------------------------------------------------------ */
/* (3) evaluation kernels (csrc/search.cu)                                   */
/* ------------------------------------------------------------------------ */

/* _numba_kernels.brute_force (:384-413) / search.brute_force_knn_batch (search.py:130-142):
 * exact k nearest ids of queries[nq, ld] among data[n, ld] (first dim columns, zero padded),
 * ties broken by ascending id; out_ids int32[nq, k], out_dists fp32[nq, k] (nullable).
 * 1 <= k <= min(n, 64). */
size_t grnnd_brute_force_workspace_bytes(int64_t n, int64_t nq, int32_t k);
int grnnd_brute_force(const float *data, int64_t n, int32_t dim, int32_t ld, const float *queries, int64_t nq,
                      int32_t k, int32_t *out_ids, float *out_dists, void *workspace, size_t workspace_bytes,
                      grnnd_stream_t s);

/* _numba_kernels.greedy_search_batch / _greedy_single (:416-513), search.search_batch
 * (search.py:90-115): best-first search with a candidate list of L keys ordered by
 * (dist, id) from entries[q] over the CSR graph (offsets int64[n+1], nbrs int32).
 * out_ids int32[nq, k] / out_dists fp32[nq, k] (nullable) are written for the first
 * out_cnt[q] = min(k, list size) ranks, -1 / inf after.  visited: >= grnnd_search_visited_bytes
 * (zeroed by the call).  L <= 1024. */
size_t grnnd_search_visited_bytes(int64_t n, int64_t nq);
int grnnd_greedy_search(const int64_t *offsets, const int32_t *nbrs, int64_t n, const float *data, int32_t dim,
                        int32_t ld, const float *queries, int64_t nq, int32_t L, int32_t k, const int64_t *entries,
                        int32_t *out_ids, float *out_dists, int64_t *out_cnt, void *visited, size_t visited_bytes,
                        grnnd_stream_t s);

/* refine_accept_loop (_numba_kernels.py:354-381): the sequential oracle's (build_seq,
 * sequential.py:85-113) accept loop for one vertex on device arrays; ids / dists sorted by
 * (dist, id), duplicate-free; counts (device int64[2]) = (accepted, redirected). */
int grnnd_refine_accept_loop(const float *data, int32_t dim, int32_t ld, const int32_t *ids, const float *dists,
                             int32_t k, int32_t *acc_ids, float *acc_dists, int32_t *red_tgt, int32_t *red_id,
                             float *red_dist, int64_t *counts, grnnd_stream_t s);

/* Inner-product metric (not in the reference, SURVEY 7 hard part 6): scale each row of
 * data[n, ld] in place to unit L2 norm (sequential fp32 sum of squares, correctly rounded
 * sqrt and division; zero rows unchanged), so squared L2 = 2 - 2<a, b> and the L2 build is
 * the IP build. */
int grnnd_normalize_rows(float *data, int64_t n, int32_t dim, int32_t ld, grnnd_stream_t s);

#ifdef __cplusplus
}
#endif
#endif /* GRNND_B200_H */
