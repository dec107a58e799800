// capi.cu -- extern "C" boundary of libgrnnd_b200.so (declared in include/grnnd_b200.h).
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a profiler injects itself

#include "common.cuh"
#include "propagate.cuh"

namespace grnnd {

// NVTX range over one C-ABI call (per-stage ranges for nsys / ncu --nvtx)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define GRNND_RANGE(name) ::grnnd::NvtxRange grnnd_nvtx_range_(name)

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

static unsigned long long g_launches = 0;  // kernels this library launched (host-side count)

unsigned long long launch_count() { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

static int g_instr = 0;  // costly instrumentation counters on (GRNND_ST_PAIRS_REF)
int instrumentation() { return __atomic_load_n(&g_instr, __ATOMIC_RELAXED); }

int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) return 0;
    return d;
}

int device_sm_count() {
    static int cache[MAX_DEVICES] = {0};
    const int d = current_device();
    const int slot = d >= 0 && d < MAX_DEVICES ? d : 0;
    int s = __atomic_load_n(&cache[slot], __ATOMIC_RELAXED);
    if (!s) {
        if (cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || s <= 0) s = 148;
        __atomic_store_n(&cache[slot], s, __ATOMIC_RELAXED);
    }
    return s;
}

int check_launch(const char *what, int nkernels) {
    __atomic_fetch_add(&g_launches, (unsigned long long)nkernels, __ATOMIC_RELAXED);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return GRNND_ECUDA;
    }
    return GRNND_OK;
}

static inline cudaStream_t S(grnnd_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

static int check_ws(void *ws, size_t bytes, int64_t n, int32_t cap, int64_t mcap, Workspace *w) {
    const size_t need = carve(nullptr, nullptr, n, cap, mcap);
    if (!ws || bytes < need) {
        set_error("workspace too small: %zu < %zu bytes", bytes, need);
        return GRNND_EWORKSPACE;
    }
    carve(w, ws, n, cap, mcap);
    return GRNND_OK;
}

static int check_pool_shape(int64_t n, int32_t dim, int32_t ld, int32_t cap) {
    if (n < 0 || dim < 1 || cap < 1) {
        set_error("bad shape n=%lld dim=%d cap=%d", (long long)n, dim, cap);
        return GRNND_EINVAL;
    }
    if (cap > GRNND_MAX_CAP) {
        set_error("pool capacity R=%d exceeds the compiled maximum %d", cap, GRNND_MAX_CAP);
        return GRNND_EUNSUPPORTED;
    }
    if (ld < dim || (ld & 3)) {
        set_error("row stride ld=%d must be >= dim=%d and a multiple of 4 (zero padded)", ld, dim);
        return GRNND_EINVAL;
    }
    return GRNND_OK;
}

// ---- small elementwise kernels for the kernel-module API ----
__global__ void hash4_kernel(uint64_t seed, uint64_t stream, const uint64_t *v, const uint64_t *i, int64_t m,
                             uint64_t *out) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < m) out[x] = hash4(seed, stream, v[x], i[x]);
}

__global__ void sqdist_kernel(const float *a, const float *b, int64_t m, int32_t dim, float *out) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < m) {
        const float *pa = a + x * dim, *pb = b + x * dim;
        float s = 0.0f;
        for (int d = 0; d < dim; ++d) s = exact_step(s, pa[d], pb[d]);
        out[x] = s;
    }
}

__global__ void check_finite_kernel(const float *__restrict__ data, int64_t n, int32_t dim, int32_t ld,
                                    unsigned long long *bad) {
    const int64_t total = n * (int64_t)dim;
    bool b = false;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = x / dim;
        const float f = data[r * ld + (x - r * dim)];
        b |= !isfinite(f);
    }
    if (__any_sync(FULL, b) && lane_id() == 0) *bad = 1ull;
}

// end of a round's apply: messages the round could not hold (emit list beyond capacity,
// or a received message for a row this rank does not own) -> stats[GRNND_ST_LOST]; resets
// the flags.  The counters are read back with the round's stats (no extra host sync).
__global__ void lost_kernel(unsigned long long *ctr, int64_t capacity, int64_t *stats) {
    const unsigned long long m = ctr[C_LIST];
    unsigned long long lost = m > (unsigned long long)capacity ? m - (unsigned long long)capacity : 0ull;
    if (ctr[C_OVERFLOW] && !lost) lost = 1ull;
    if (ctr[C_BADTGT]) lost += 1ull;
    if (lost && stats) atomicAdd((unsigned long long *)&stats[GRNND_ST_LOST], lost);
    ctr[C_OVERFLOW] = 0ull;
    ctr[C_BADTGT] = 0ull;
}

__global__ void fill_i32_kernel(int32_t *p, int64_t n, int32_t v) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < n) p[x] = v;
}

}  // namespace grnnd

using namespace grnnd;

extern "C" {

const char *grnnd_last_error(void) { return g_err; }
int grnnd_abi_version(void) { return 1; }
unsigned long long grnnd_launch_count(void) { return launch_count(); }
int grnnd_set_instrumentation(int on) {
    const int old = instrumentation();
    __atomic_store_n(&g_instr, on ? 1 : 0, __ATOMIC_RELAXED);
    return old;
}

int grnnd_hash4_batch(uint64_t seed, uint64_t stream, const uint64_t *v, const uint64_t *i, int64_t m, uint64_t *out,
                      grnnd_stream_t s) {
    if (m <= 0) return GRNND_OK;
    hash4_kernel<<<(unsigned)((m + 255) / 256), 256, 0, S(s)>>>(seed, stream, v, i, m, out);
    return check_launch("hash4_kernel");
}

int grnnd_sqdist_batch(const float *a, const float *b, int64_t m, int32_t dim, float *out, grnnd_stream_t s) {
    if (m <= 0) return GRNND_OK;
    if (dim < 1) {
        set_error("dim must be >= 1");
        return GRNND_EINVAL;
    }
    sqdist_kernel<<<(unsigned)((m + 127) / 128), 128, 0, S(s)>>>(a, b, m, dim, out);
    return check_launch("sqdist_kernel");
}

int grnnd_sample_initial(int64_t n, int32_t count, uint64_t seed, int32_t *out, int64_t *fail_flag,
                         grnnd_stream_t s) {
    if (n < 1 || count < 0) {
        set_error("sample_initial: bad n=%lld count=%d", (long long)n, count);
        return GRNND_EINVAL;
    }
    return launch_sample_initial(n, 0, n, count, seed, out, count, fail_flag, S(s));
}

int grnnd_init_dists(const float *data, int64_t n, int32_t dim, int32_t ld, const int32_t *ids, int32_t count,
                     float *out, grnnd_stream_t s) {
    if (ld < dim || dim < 1) {
        set_error("init_dists: bad dim/ld");
        return GRNND_EINVAL;
    }
    return launch_init_dists(data, dim, ld, 0, n, ids, count, count, out, count, S(s));
}

size_t grnnd_workspace_bytes(int64_t n, int32_t cap, int64_t msg_capacity) {
    return carve(nullptr, nullptr, n, cap, msg_capacity);
}

int grnnd_gen_update_messages(const float *data, int64_t n, int32_t dim, int32_t ld, int32_t *read_ids,
                              const float *read_dists, const int32_t *read_count, int32_t cap, uint64_t seed,
                              uint64_t stream_id, int32_t order_code, int32_t *msg_tgt, int32_t *msg_id,
                              float *msg_dist, int32_t *msg_cnt, void *workspace, size_t workspace_bytes,
                              grnnd_stream_t s) {
    GRNND_TRY(check_pool_shape(n, dim, ld, cap));
    if (order_code != 0 && order_code != 1) {
        set_error("order_code must be 0 (disordered) or 1 (ascending)");
        return GRNND_EINVAL;
    }
    Workspace w;
    GRNND_TRY(check_ws(workspace, workspace_bytes, n, cap, 0, &w));
    PropArgs a{};
    a.data = data;
    a.n_total = n;
    a.lo = 0;
    a.hi = n;
    a.dim = dim;
    a.ld = ld;
    a.cap = cap;
    a.read_ids = read_ids;
    a.read_dists = read_dists;
    a.read_count = read_count;
    a.seed = seed;
    a.stream_id = stream_id;
    a.order_code = order_code;
    a.slice_mode = 1;
    a.msg_tgt = msg_tgt;
    a.msg_id = msg_id;
    a.msg_dist = msg_dist;
    a.msg_cnt = msg_cnt;
    a.w = w;
    a.stats = nullptr;
    return launch_propagate(a, S(s));
}

int grnnd_gen_reverse_messages(const int32_t *read_ids, const float *read_dists, const int32_t *read_count,
                               int64_t n, int32_t cap, double rho, int32_t *msg_tgt, int32_t *msg_id,
                               float *msg_dist, int32_t *msg_cnt, grnnd_stream_t s) {
    if (cap > GRNND_MAX_CAP || cap < 1) {
        set_error("cap %d unsupported", cap);
        return GRNND_EUNSUPPORTED;
    }
    ReverseArgs a{};
    a.read_ids = read_ids;
    a.read_dists = read_dists;
    a.read_count = read_count;
    a.lo = 0;
    a.n = n;
    a.cap = cap;
    a.rho = rho;
    a.slice_mode = 1;
    a.msg_tgt = msg_tgt;
    a.msg_id = msg_id;
    a.msg_dist = msg_dist;
    a.msg_cnt = msg_cnt;
    return launch_reverse_select(a, S(s));
}

int grnnd_gen_merge_messages(const int32_t *read_ids, const float *read_dists, const int32_t *read_count, int64_t n,
                             int32_t cap, int32_t *msg_tgt, int32_t *msg_id, float *msg_dist, int32_t *msg_cnt,
                             grnnd_stream_t s) {
    ReverseArgs a{};
    a.read_ids = read_ids;
    a.read_dists = read_dists;
    a.read_count = read_count;
    a.lo = 0;
    a.n = n;
    a.cap = cap;
    a.slice_mode = 1;
    a.msg_tgt = msg_tgt;
    a.msg_id = msg_id;
    a.msg_dist = msg_dist;
    a.msg_cnt = msg_cnt;
    return launch_merge_slices(a, S(s));
}

int grnnd_message_offsets(const int32_t *msg_cnt, int64_t n, int64_t *offs, void *workspace, size_t workspace_bytes,
                          grnnd_stream_t s) {
    Workspace w;
    GRNND_TRY(check_ws(workspace, workspace_bytes, n, 1, 0, &w));
    return launch_scan_counts(msg_cnt, n, offs, w.scan_tmp, S(s));
}

int grnnd_compact_messages(const int32_t *msg_tgt, const int32_t *msg_id, const float *msg_dist,
                           const int32_t *msg_cnt, int64_t n, int32_t cap, const int64_t *offs, int32_t *flat_tgt,
                           int32_t *flat_id, float *flat_dist, int32_t *flat_src, grnnd_stream_t s) {
    return launch_compact(msg_tgt, msg_id, msg_dist, msg_cnt, n, cap, offs, flat_tgt, flat_id, flat_dist, flat_src,
                          S(s));
}

int grnnd_group_by_target(const int32_t *flat_tgt, int64_t m, int64_t n, int64_t *order, int64_t *starts,
                          void *workspace, size_t workspace_bytes, grnnd_stream_t s) {
    Workspace w;
    GRNND_TRY(check_ws(workspace, workspace_bytes, n, 1, m, &w));
    // key = message index: sorting each target's segment by it = the stable counting sort
    GRNND_TRY(launch_group_inbox(w, nullptr, flat_tgt, nullptr, nullptr, nullptr, m, 0, n, S(s)));
    if (m > 0) GRNND_CUDA(cudaMemcpyAsync(order, w.i_key, sizeof(int64_t) * (size_t)m, cudaMemcpyDeviceToDevice, S(s)));
    GRNND_CUDA(cudaMemcpyAsync(starts, w.starts, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyDeviceToDevice, S(s)));
    return GRNND_OK;
}

int grnnd_apply_grouped_messages(int32_t *write_ids, float *write_dists, int32_t *write_count, int64_t n, int32_t cap,
                                 const int32_t *flat_id, const float *flat_dist, const int64_t *order,
                                 const int64_t *starts, int64_t *outcomes, grnnd_stream_t s) {
    if (cap > GRNND_MAX_CAP || cap < 1) {
        set_error("cap %d unsupported", cap);
        return GRNND_EUNSUPPORTED;
    }
    return launch_apply_grouped(write_ids, write_dists, write_count, n, cap, flat_id, flat_dist, order, starts,
                                outcomes, S(s));
}

// ------------------------------------------------------------------------------------
// fused round API
// ------------------------------------------------------------------------------------
static int pools_workspace(const grnnd_pools *p, Workspace *w) {
    if (!p) {
        set_error("null pools");
        return GRNND_EINVAL;
    }
    const int64_t n = p->hi - p->lo;
    GRNND_TRY(check_pool_shape(n, p->dim, p->ld, p->cap));
    if (p->lo < 0 || p->hi > p->n_total || p->lo > p->hi) {
        set_error("owned range [%lld, %lld) outside [0, %lld)", (long long)p->lo, (long long)p->hi,
                  (long long)p->n_total);
        return GRNND_EINVAL;
    }
    return check_ws(p->workspace, p->workspace_bytes, n, p->cap, p->msg_capacity, w);
}

int grnnd_init_pools(const grnnd_pools *p, int32_t S_, uint64_t seed, int64_t *fail_flag, grnnd_stream_t s) {
    GRNND_RANGE("grnnd_init_pools");
    Workspace w;
    GRNND_TRY(pools_workspace(p, &w));
    const int64_t n = p->hi - p->lo;
    if (S_ < 1 || S_ > p->cap || S_ > p->n_total - 1) {
        set_error("S=%d outside [1, min(R, N-1)]", S_);
        return GRNND_EINVAL;
    }
    GRNND_TRY(launch_sample_initial(p->n_total, p->lo, n, S_, seed, p->read_ids, p->cap, fail_flag, S(s)));
    GRNND_TRY(launch_init_dists(p->data, p->dim, p->ld, p->lo, n, p->read_ids, p->cap, S_, p->read_dists, p->cap,
                                S(s)));
    if (n > 0) {
        fill_i32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, S(s)>>>(p->read_count, n, S_);
        if (p->write_count != p->read_count)  // (in-place pools: one buffer)
            fill_i32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, S(s)>>>(p->write_count, n, 0);
        GRNND_TRY(check_launch("fill_counts", 2));
        GRNND_CUDA(cudaMemsetAsync(w.dirty, 0, (size_t)n, S(s)));
        GRNND_CUDA(cudaMemsetAsync(w.idle, 0, (size_t)n, S(s)));
    }
    GRNND_CUDA(cudaMemsetAsync(w.ctr, 0, sizeof(unsigned long long) * C_NCOUNTERS, S(s)));
    return GRNND_OK;
}

static int emit_update(const grnnd_pools *p, const Workspace &w, uint64_t seed, uint64_t stream_id,
                       int32_t order_code, cudaStream_t st) {
    PropArgs a{};
    a.data = p->data;
    a.n_total = p->n_total;
    a.lo = p->lo;
    a.hi = p->hi;
    a.dim = p->dim;
    a.ld = p->ld;
    a.cap = p->cap;
    a.read_ids = p->read_ids;
    a.read_dists = p->read_dists;
    a.read_count = p->read_count;
    a.seed = seed;
    a.stream_id = stream_id;
    a.order_code = order_code;
    a.slice_mode = 0;
    a.w = w;
    a.stats = p->stats;
    a.norms = p->norms;
    a.split = p->filter_split;
    filter_eps(p->dim, &a.eps_n, &a.eps_h);
    return launch_propagate(a, st);
}

static int emit_reverse(const grnnd_pools *p, const Workspace &w, double rho, cudaStream_t st) {
    ReverseArgs a{};
    a.read_ids = p->read_ids;
    a.read_dists = p->read_dists;
    a.read_count = p->read_count;
    a.lo = p->lo;
    a.n = p->hi - p->lo;
    a.cap = p->cap;
    a.rho = rho;
    a.slice_mode = 0;
    a.w = w;
    a.stats = p->stats;
    return launch_reverse_select(a, st);
}

static int apply_phase(const grnnd_pools *p, const Workspace &w, int32_t kind, const unsigned long long *m_dev,
                       int64_t m_host, cudaStream_t st) {
    const int64_t n = p->hi - p->lo;
    GRNND_TRY(launch_group_inbox(w, w.e_key, w.e_tgt, w.e_id, w.e_dist, m_dev, m_host, p->lo, n, st));
    ApplyArgs a{};
    a.write_ids = p->write_ids;
    a.write_dists = p->write_dists;
    a.write_count = p->write_count;
    a.read_ids = p->read_ids;
    a.read_count = p->read_count;
    a.read_dists = p->read_dists;
    a.lo = p->lo;
    a.n = n;
    a.cap = p->cap;
    a.own_after_all = kind == 1 ? 1 : 0;
    a.in_place = p->write_ids == p->read_ids ? 1 : 0;
    if (a.in_place != (p->write_dists == p->read_dists ? 1 : 0) ||
        a.in_place != (p->write_count == p->read_count ? 1 : 0)) {
        set_error("write_ids / write_dists / write_count must all alias the read side or none of them");
        return GRNND_EINVAL;
    }
    a.w = w;
    a.stats = p->stats;
    GRNND_TRY(launch_apply_round(a, st));
    lost_kernel<<<1, 1, 0, st>>>(w.ctr, m_dev ? p->msg_capacity : (int64_t)0x7fffffffffffffffLL, p->stats);
    return check_launch("lost_kernel");
}

int grnnd_update_round(const grnnd_pools *p, uint64_t seed, uint64_t stream_id, int32_t order_code,
                       grnnd_stream_t s) {
    GRNND_RANGE("grnnd_update_round");
    Workspace w;
    GRNND_TRY(pools_workspace(p, &w));
    if (order_code != 0 && order_code != 1) {
        set_error("order_code must be 0 or 1");
        return GRNND_EINVAL;
    }
    GRNND_CUDA(cudaMemsetAsync(w.ctr + C_LIST, 0, sizeof(unsigned long long), S(s)));
    GRNND_TRY(emit_update(p, w, seed, stream_id, order_code, S(s)));
    return apply_phase(p, w, 0, w.ctr + C_LIST, p->msg_capacity, S(s));
}

int grnnd_reverse_round(const grnnd_pools *p, double rho, grnnd_stream_t s) {
    GRNND_RANGE("grnnd_reverse_round");
    Workspace w;
    GRNND_TRY(pools_workspace(p, &w));
    if (!(rho > 0.0 && rho <= 1.0)) {
        set_error("rho must be in (0, 1]");
        return GRNND_EINVAL;
    }
    GRNND_CUDA(cudaMemsetAsync(w.ctr + C_LIST, 0, sizeof(unsigned long long), S(s)));
    GRNND_TRY(emit_reverse(p, w, rho, S(s)));
    return apply_phase(p, w, 1, w.ctr + C_LIST, p->msg_capacity, S(s));
}

int grnnd_update_emit(const grnnd_pools *p, uint64_t seed, uint64_t stream_id, int32_t order_code,
                      grnnd_stream_t s) {
    GRNND_RANGE("grnnd_update_emit");
    Workspace w;
    GRNND_TRY(pools_workspace(p, &w));
    if (order_code != 0 && order_code != 1) {
        set_error("order_code must be 0 or 1");
        return GRNND_EINVAL;
    }
    GRNND_CUDA(cudaMemsetAsync(w.ctr + C_LIST, 0, sizeof(unsigned long long), S(s)));
    return emit_update(p, w, seed, stream_id, order_code, S(s));
}

int grnnd_reverse_emit(const grnnd_pools *p, double rho, grnnd_stream_t s) {
    GRNND_RANGE("grnnd_reverse_emit");
    Workspace w;
    GRNND_TRY(pools_workspace(p, &w));
    if (!(rho > 0.0 && rho <= 1.0)) {
        set_error("rho must be in (0, 1]");
        return GRNND_EINVAL;
    }
    GRNND_CUDA(cudaMemsetAsync(w.ctr + C_LIST, 0, sizeof(unsigned long long), S(s)));
    return emit_reverse(p, w, rho, S(s));
}

int grnnd_apply_emitted(const grnnd_pools *p, int32_t kind, grnnd_stream_t s) {
    GRNND_RANGE("grnnd_apply_emitted");
    Workspace w;
    GRNND_TRY(pools_workspace(p, &w));
    return apply_phase(p, w, kind, w.ctr + C_LIST, p->msg_capacity, S(s));
}

int grnnd_round_emit(const grnnd_pools *p, int32_t kind, uint64_t seed, uint64_t stream_id, int32_t order_code,
                     double rho, const int64_t *rank_bounds, int32_t nranks, int64_t *send_counts,
                     grnnd_stream_t s) {
    GRNND_RANGE("grnnd_round_emit");
    Workspace w;
    GRNND_TRY(pools_workspace(p, &w));
    GRNND_CUDA(cudaMemsetAsync(w.ctr + C_LIST, 0, sizeof(unsigned long long), S(s)));
    if (kind == 0) GRNND_TRY(emit_update(p, w, seed, stream_id, order_code, S(s)));
    else GRNND_TRY(emit_reverse(p, w, rho, S(s)));
    return launch_bucket_by_rank(w, rank_bounds, nranks, send_counts, S(s));
}

int grnnd_round_buffers(const grnnd_pools *p, int32_t **out_pack, int32_t **in_pack) {
    Workspace w;
    GRNND_TRY(pools_workspace(p, &w));
    if (out_pack) *out_pack = w.o_pack;
    if (in_pack) *in_pack = w.r_pack;
    return GRNND_OK;
}

int grnnd_round_apply(const grnnd_pools *p, int32_t kind, int64_t n_incoming, grnnd_stream_t s) {
    GRNND_RANGE("grnnd_round_apply");
    Workspace w;
    GRNND_TRY(pools_workspace(p, &w));
    if (n_incoming < 0 || n_incoming > p->msg_capacity) {
        set_error("incoming message count %lld exceeds capacity %lld", (long long)n_incoming,
                  (long long)p->msg_capacity);
        return GRNND_EWORKSPACE;
    }
    GRNND_TRY(launch_unpack(w, n_incoming, p->lo, p->hi - p->lo, S(s)));
    return apply_phase(p, w, kind, nullptr, n_incoming, S(s));
}

int grnnd_finalize(const int32_t *ids, const float *dists, const int32_t *counts, int64_t n, int32_t cap,
                   int64_t *offsets, int32_t *nbrs, int64_t *bad_flag, void *workspace, size_t workspace_bytes,
                   grnnd_stream_t s) {
    if (cap > GRNND_MAX_CAP || cap < 1) {
        set_error("cap %d unsupported", cap);
        return GRNND_EUNSUPPORTED;
    }
    Workspace w;
    GRNND_TRY(check_ws(workspace, workspace_bytes, n, cap, 0, &w));
    GRNND_TRY(launch_scan_counts(counts, n, offsets, w.scan_tmp, S(s)));
    return launch_finalize(ids, dists, counts, n, cap, 0, n, offsets, nbrs, nullptr, bad_flag, S(s));
}

int grnnd_finalize_pools(const grnnd_pools *p, int64_t *offsets, int32_t *nbrs, int64_t *bad_flag,
                         grnnd_stream_t s) {
    GRNND_RANGE("grnnd_finalize_pools");
    Workspace w;
    GRNND_TRY(pools_workspace(p, &w));
    const int64_t n = p->hi - p->lo;
    GRNND_TRY(launch_scan_counts(p->read_count, n, offsets, w.scan_tmp, S(s)));
    return launch_finalize(p->read_ids, p->read_dists, p->read_count, n, p->cap, p->lo, p->n_total, offsets,
                           nbrs, nullptr, bad_flag, S(s));
}

int grnnd_sorted_rows(const int32_t *ids, const float *dists, const int32_t *counts, int64_t n, int32_t cap,
                      int32_t *out_ids, grnnd_stream_t s) {
    if (cap > GRNND_MAX_CAP || cap < 1) {
        set_error("cap %d unsupported", cap);
        return GRNND_EUNSUPPORTED;
    }
    return launch_finalize(ids, dists, counts, n, cap, 0, n, nullptr, nullptr, out_ids, nullptr, S(s));
}


__global__ void band_terms_kernel(const int32_t *__restrict__ ids, const float *__restrict__ dists,
                                  const int32_t *__restrict__ counts, const float *__restrict__ norms, int64_t n,
                                  int32_t cap, double *out) {
    double sn = 0.0, sd = 0.0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * cap; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = e / cap;
        const int s = (int)(e - v * cap);
        if (s < counts[v]) {
            const int32_t id = ids[e];
            if (id >= 0) {  // |member|^2 / its stored distance, averaged over the entries
                const double dv = (double)dists[e];
                sn += (double)norms[id] / (dv > 1e-30 ? dv : 1e-30);
                sd += 1.0;
            }
        }
    }
    sn = warp_sum(sn);
    sd = warp_sum(sd);
    if (lane_id() == 0) {
        atomicAdd(&out[0], sn);
        atomicAdd(&out[1], sd);
    }
}

int grnnd_band_terms(const grnnd_pools *p, double *out, grnnd_stream_t s) {
    if (!p || !out || !p->norms) {
        set_error("band_terms: pools with norms and an output buffer required");
        return GRNND_EINVAL;
    }
    const int64_t n = p->hi - p->lo;
    GRNND_CUDA(cudaMemsetAsync(out, 0, 2 * sizeof(double), S(s)));
    if (n <= 0) return GRNND_OK;
    band_terms_kernel<<<(unsigned)(device_sm_count() * 8), 256, 0, S(s)>>>(p->read_ids, p->read_dists, p->read_count,
                                                                          p->norms, n, p->cap, out);
    return check_launch("band_terms_kernel");
}

int grnnd_row_norms(const float *data, int64_t n, int32_t dim, int32_t ld, float *out, grnnd_stream_t s) {
    if (dim < 1 || ld < dim || n < 0) {
        set_error("row_norms: bad n/dim/ld");
        return GRNND_EINVAL;
    }
    return launch_row_norms(data, n, dim, ld, out, S(s));
}

int grnnd_check_finite(const float *data, int64_t n, int32_t dim, int32_t ld, int64_t *bad_flag, grnnd_stream_t s) {
    if (dim < 1 || ld < dim) {
        set_error("check_finite: bad dim/ld");
        return GRNND_EINVAL;
    }
    const int64_t total = n * (int64_t)dim;
    if (total <= 0) return GRNND_OK;
    const int64_t blocks = total / 256 + 1 < 148 * 32 ? total / 256 + 1 : 148 * 32;
    check_finite_kernel<<<(unsigned)blocks, 256, 0, S(s)>>>(data, n, dim, ld, (unsigned long long *)bad_flag);
    return check_launch("check_finite_kernel");
}

}  // extern "C"
