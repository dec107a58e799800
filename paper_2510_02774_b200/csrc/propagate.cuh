// propagate.cuh -- argument blocks and launchers shared by the .cu files.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "workspace.cuh"

namespace grnnd {

struct PropArgs {
    const float *data;
    int64_t n_total;  // rows of data (the TMA tensor map's extent)
    int64_t lo, hi;  // owned rows [lo, hi) ; row r of the pool arrays = vertex lo + r
    int32_t dim, ld, cap;
    int32_t *read_ids;
    const float *read_dists;
    const int32_t *read_count;
    uint64_t seed, stream_id;
    int32_t order_code;
    int32_t slice_mode;  // 1: reference message-slice layout (kernel-module API)
    int32_t *msg_tgt;
    int32_t *msg_id;
    float *msg_dist;
    int32_t *msg_cnt;
    Workspace w;
    int64_t *stats;
    // filtered pair phase (pairs.cuh): squared row norms of all rows, or nullptr for the
    // exact-only pair phase; eps_n / eps_h are the filter's error-bound coefficients
    const float *norms;
    float eps_n, eps_h;
    int32_t split;  // tensor-core Gram in split TF32 (tc3_pairs.cuh SPLIT)
};

// error-bound coefficients of the filtered pair phase for dimension dim
void filter_eps(int32_t dim, float *eps_n, float *eps_h);
int launch_row_norms(const float *data, int64_t n, int32_t dim, int32_t ld, float *out, cudaStream_t st);

int launch_propagate(const PropArgs &a, cudaStream_t st);

// reverse selection (gen_reverse_messages :195-233) / merge (gen_merge_messages :236-250)
struct ReverseArgs {
    const int32_t *read_ids;
    const float *read_dists;
    const int32_t *read_count;
    int64_t lo, n;  // rows
    int32_t cap;
    double rho;
    int32_t slice_mode;
    int32_t *msg_tgt;
    int32_t *msg_id;
    float *msg_dist;
    int32_t *msg_cnt;
    Workspace w;
    int64_t *stats;
};
int launch_reverse_select(const ReverseArgs &a, cudaStream_t st);
int launch_merge_slices(const ReverseArgs &a, cudaStream_t st);

// grouping: emitted list -> inbox grouped by target row and sorted by key
int launch_group_inbox(const Workspace &w, const int64_t *key, const int32_t *tgt,
                       const int32_t *id, const float *dist, const unsigned long long *m_dev,
                       int64_t m_host, int64_t lo, int64_t n, cudaStream_t st);
int launch_compact(const int32_t *msg_tgt, const int32_t *msg_id, const float *msg_dist,
                   const int32_t *msg_cnt, int64_t n, int32_t cap, const int64_t *offs,
                   int32_t *flat_tgt, int32_t *flat_id, float *flat_dist, int32_t *flat_src,
                   cudaStream_t st);
int launch_bucket_by_rank(const Workspace &w, const int64_t *rank_bounds, int32_t nranks,
                          int64_t *send_counts, cudaStream_t st);
int launch_unpack(const Workspace &w, int64_t m, int64_t lo, int64_t n, cudaStream_t st);
int launch_scan_counts(const int32_t *counts, int64_t n, int64_t *out, int64_t *tmp,
                       cudaStream_t st);
int launch_segsort(const Workspace &w, int64_t n, int64_t *key, int32_t *id, float *dist,
                   cudaStream_t st);

// apply
struct ApplyArgs {
    int32_t *write_ids;
    float *write_dists;
    int32_t *write_count;
    const int32_t *read_ids;  // own entries (survivors / merge), slot order, TOMB = skip
    const int32_t *read_count;
    const float *read_dists;
    int64_t lo, n;
    int32_t cap;
    int32_t own_after_all;  // 0: own entries spliced at source == target (update round)
                            // 1: own entries after every inbox message (reverse round)
    int32_t in_place;       // write_* == read_*: only pools with incoming messages or
                            // tombstones (w.dirty) are rewritten; the rest are their own result
    Workspace w;
    int64_t *stats;
};
int launch_apply_round(const ApplyArgs &a, cudaStream_t st);
int launch_apply_grouped(int32_t *write_ids, float *write_dists, int32_t *write_count, int64_t n,
                         int32_t cap, const int32_t *flat_id, const float *flat_dist,
                         const int64_t *order, const int64_t *starts, int64_t *outcomes,
                         cudaStream_t st);

// init / finalize
int launch_sample_initial(int64_t n_total, int64_t lo, int64_t rows, int32_t count, uint64_t seed,
                          int32_t *out, int32_t ld_out, int64_t *fail_flag, cudaStream_t st);
int launch_init_dists(const float *data, int32_t dim, int32_t ld, int64_t lo, int64_t rows,
                      const int32_t *ids, int32_t ld_ids, int32_t count, float *out,
                      int32_t ld_out, cudaStream_t st);
int launch_finalize(const int32_t *ids, const float *dists, const int32_t *counts, int64_t n,
                    int32_t cap, int64_t lo, int64_t n_total, const int64_t *offsets, int32_t *nbrs,
                    int32_t *fixed_out, int64_t *bad_flag, cudaStream_t st);

}  // namespace grnnd
