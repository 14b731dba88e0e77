// colgraph.cu -- host side of the B200 column-graph max-flow library (include/colgraph.h).
//
// Hot path of arXiv 2601.17026 (§3.2), redesigned for one GPU per process:
// the paper's per-thread FIFO queues, per-vertex locks and level barriers (§3.2.1-3.2.4)
// become device worklists of 32-vertex chunks, single-decrementer atomics and
// level-synchronous frontier kernels launched back to back on one stream.  The host
// only reads a few counters every `check_every` sweeps.
//
// Solve loop:
//   a2  exact global relabel (frontier BFS from t) -> rebuild the active-chunk list
//   a3  sweeps over the active-chunk list (batch of check_every launches, no host sync)
//   a5  re-run the global relabel when the work since the last one reaches gr_factor*n
//        or the sweep time since the last one exceeds its cost
//   a4  when a sweep finds no active vertex: exact global relabel; stop if no vertex
//       with excess has a finite height (the preflow is then maximum)
//   a6  |f| = sum(T0) - sum(T)
#include "colgraph.h"
#include "kernels.cuh"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

using namespace cg;

namespace {
constexpr int RING = 256;
constexpr int BFS_BATCH = 32;
constexpr int EXT_BATCH = 16;
}  // namespace

struct cg_graph {
    cg_dims dims{};
    cg_dist dist{};
    Geo geo{};
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    // one stream-ordered workspace allocation
    char *ws = nullptr;
    size_t ws_bytes = 0;
    Soa s{};
    int *blist[2] = {nullptr, nullptr};  // BFS frontiers (vertices)
    int *clist[2] = {nullptr, nullptr};  // sweep worklists (chunks)
    int *cstamp = nullptr;               // per-chunk list tag
    int *vstamp = nullptr;               // per-vertex list tag
    bool vertex_lists = true;            // sweep worklist granularity (CG_CHUNK_LISTS=1: chunks)
    int32_t *top = nullptr, *proc = nullptr;
    int *colstamp = nullptr;
    int *collist[2] = {nullptr, nullptr};
    unsigned *hist = nullptr;
    BfsState *bst = nullptr, *h_bst = nullptr;  // device BFS state + pinned mirror
    unsigned *cnt = nullptr;              // [0..2] sweep lists, [4..6] bfs, [8..10] extraction
    unsigned long long *work = nullptr;   // [RING] active visits per sweep
    unsigned long long *u64 = nullptr;    // [0]=N [1]=sumT0 [2]=sumT [3]=active [4]=gap lifted
    int *flags = nullptr;                 // [0]=overflow [1]=maxh [2]=gap [3]=empty
    // pinned host mirrors
    unsigned *h_cnt = nullptr;
    unsigned long long *h_work = nullptr, *h_u64 = nullptr;
    int *h_flags = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int64_t N = 0, sumT0 = 0;
    int tag = 0;        // monotone worklist tag
    int sweep_par = 0;  // sweeps since the last list rebuild (selects list/counter buffers)
    bool solved = false;
    cg_solve_stats st{};
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

#define CG_CUDA(call)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            if (getenv("CG_DEBUG"))                                                            \
                fprintf(stderr, "colgraph: %s -> %s (%s:%d)\n", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                   \
            return e_ == cudaErrorMemoryAllocation ? CG_E_NOMEM : CG_E_CUDA;                   \
        }                                                                                      \
    } while (0)

inline int grid_for(int64_t n, int block, int cap) {
    int64_t b = (n + block - 1) / block;
    if (b < 1) b = 1;
    return (int)std::min<int64_t>(b, cap);
}

inline double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

inline bool tracing() { return getenv("CG_TRACE") != nullptr; }

// Grid for worklist kernels: enough warps to fill every SM (8 x 256 threads per SM).
inline int list_grid(const cg_graph *g, int64_t items) { return grid_for(items * 32, 256, g->num_sms * 8); }

// a2/a5: exact global relabel + rebuild of the sweep worklist; h_u64[3] = active count.
cg_status global_relabel(cg_graph *g) {
    const Geo &geo = g->geo;
    cudaStream_t st = g->stream;
    // device-driven levels: state {L = 1, counters 0}; seeds = level 1
    CG_CUDA(cudaMemsetAsync(g->bst, 0, sizeof(BfsState), st));
    g->h_bst->L = 1;
    CG_CUDA(cudaMemcpyAsync(&g->bst->L, &g->h_bst->L, sizeof(int), cudaMemcpyHostToDevice, st));
    k_bfs_init<<<grid_for(geo.n, 256, g->num_sms * 16), 256, 0, st>>>(geo, g->s, g->blist[0], &g->bst->cnt[0]);
    g->st.kernel_launches++;
    int L = 1;
    for (int batch = 0;; batch++) {
        const int nb = batch == 0 ? 8 : BFS_BATCH;
        for (int b = 0; b < nb; b++)
            k_bfs_step<<<g->num_sms * 2, 512, 0, st>>>(geo, g->s, g->blist[0], g->blist[1], g->bst);
        g->st.kernel_launches += nb;
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaMemcpyAsync(g->h_bst, g->bst, sizeof(BfsState), cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaStreamSynchronize(st));
        L = g->h_bst->L;
        if (g->h_bst->cnt[(L - 1) % 3] == 0) break;
        if ((int64_t)L > (int64_t)geo.INF + 2) return CG_E_CUDA;  // every level claims >= 1 vertex
    }
    g->st.gr_passes += L - 1;
    // rebuild the active-chunk worklist into clist[0] / cnt[0]
    CG_CUDA(cudaMemsetAsync(g->cnt, 0, 3 * sizeof(unsigned), st));
    CG_CUDA(cudaMemsetAsync(g->u64 + 3, 0, sizeof(unsigned long long), st));
    const int tag = ++g->tag;
    if (g->vertex_lists)
        k_rebuild_vertices<<<grid_for(geo.n, 256, g->num_sms * 16), 256, 0, st>>>(geo, g->s, g->blist[0], g->cnt,
                                                                                  g->vstamp, tag, g->u64 + 3);
    else
        k_rebuild_chunks<<<grid_for(geo.nchunks, 256, g->num_sms * 16), 256, 0, st>>>(
            geo, g->s, g->clist[0], g->cnt, g->cstamp, tag, g->u64 + 3);
    g->st.kernel_launches++;
    g->sweep_par = 0;
    CG_CUDA(cudaMemcpyAsync(g->h_u64 + 3, g->u64 + 3, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    CG_CUDA(cudaGetLastError());
    g->st.global_relabels++;
    return CG_OK;
}

cg_status run_gap(cg_graph *g) {
    const Geo &geo = g->geo;
    cudaStream_t st = g->stream;
    CG_CUDA(cudaMemsetAsync(g->hist, 0, sizeof(unsigned) * GAP_BINS, st));
    CG_CUDA(cudaMemsetAsync(g->flags + 1, 0, sizeof(int), st));
    k_gap_hist<<<g->num_sms * 8, 256, 0, st>>>(geo, g->s.H, g->hist, g->flags + 1);
    k_gap_find<<<1, 1024, 0, st>>>(g->hist, g->flags + 1, g->flags + 2);
    k_gap_lift<<<g->num_sms * 8, 256, 0, st>>>(geo, g->s.H, g->flags + 2, g->u64 + 4);
    CG_CUDA(cudaGetLastError());
    g->st.kernel_launches += 3;
    g->st.gap_runs++;
    return CG_OK;
}

template <typename T>
T *carve(char *&p, int64_t count) {
    T *r = reinterpret_cast<T *>(p);
    p += ((size_t)count * sizeof(T) + 255) & ~(size_t)255;
    return r;
}

size_t workspace_bytes(const Geo &geo) {
    const int64_t ncol = (int64_t)geo.X * geo.Y;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    size_t b = 0;
    b += al(sizeof(int32_t) * 8 * geo.n);
    b += 2 * al(sizeof(int) * geo.n);
    b += 3 * al(sizeof(int) * geo.nchunks);
    b += al(sizeof(int) * geo.n);
    b += 5 * al(sizeof(int) * ncol);
    b += al(sizeof(unsigned) * GAP_BINS);
    b += al(sizeof(BfsState));
    b += al(sizeof(unsigned) * 16) + al(sizeof(unsigned long long) * RING) + al(sizeof(unsigned long long) * 16) +
         al(sizeof(int) * 16);
    return b;
}

}  // namespace

extern "C" {

const char *cg_status_str(cg_status s) {
    switch (s) {
        case CG_OK: return "CG_OK";
        case CG_E_INVAL: return "CG_E_INVAL";
        case CG_E_OVERFLOW: return "CG_E_OVERFLOW";
        case CG_E_NOMEM: return "CG_E_NOMEM";
        case CG_E_CUDA: return "CG_E_CUDA";
        case CG_E_NCCL: return "CG_E_NCCL";
        case CG_E_EMPTY_COLUMN: return "CG_E_EMPTY_COLUMN";
        case CG_E_STATE: return "CG_E_STATE";
        case CG_E_NOT_CONVERGED: return "CG_E_NOT_CONVERGED";
    }
    return "CG_E_UNKNOWN";
}

const char *cg_version(void) {
    return "colgraph 0.2 sm_100a (chunk-worklist lock-free push-relabel, frontier-BFS global relabel, "
           "worklist extraction)";
}

cg_status cg_slab_range(const cg_dims *dims, int32_t rank, int32_t nranks, int32_t *x0, int32_t *x1) {
    if (!dims || !x0 || !x1 || nranks < 1 || rank < 0 || rank >= nranks || dims->X < nranks) return CG_E_INVAL;
    const int32_t q = dims->X / nranks, r = dims->X % nranks;
    *x0 = rank * q + std::min(rank, r);
    *x1 = *x0 + q + (rank < r ? 1 : 0);
    return CG_OK;
}

void colgraph_free(cg_graph *g) {
    if (!g) return;
    {
        DeviceGuard dg(g->dist.device);
        if (g->ws) cudaFreeAsync(g->ws, g->stream);
        if (g->ev0) cudaEventDestroy(g->ev0);
        if (g->ev1) cudaEventDestroy(g->ev1);
        cudaFreeHost(g->h_cnt);
        cudaFreeHost(g->h_work);
        cudaFreeHost(g->h_u64);
        cudaFreeHost(g->h_flags);
        cudaFreeHost(g->h_bst);
    }
    delete g;
}

cg_status colgraph_build(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight, const cg_dist *dist,
                         cg_graph **out) {
    if (!dims || !cost_dev || !out) return CG_E_INVAL;
    *out = nullptr;
    if (dims->X < 1 || dims->Y < 1 || dims->Z < 1 || dims->delta < 0) return CG_E_INVAL;
    const int64_t n = (int64_t)dims->X * dims->Y * dims->Z;
    if (n + dims->Z + 64 >= (int64_t)INT_MAX) return CG_E_INVAL;
    cg_dist dd{0, 1, nullptr, 0, nullptr};
    if (dist) dd = *dist;
    if (dd.nranks != 1 || dd.rank != 0) return CG_E_INVAL;  // multi-GPU x-slabs: not in this build
    DeviceGuard dg(dd.device);
    const double t0 = now_ms();
    cg_graph *g = new cg_graph();
    g->dims = *dims;
    g->dist = dd;
    g->stream = (cudaStream_t)dd.stream;
    cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, dd.device);
    Geo &geo = g->geo;
    geo.X = dims->X;
    geo.Y = dims->Y;
    geo.Z = dims->Z;
    geo.delta = dims->delta;
    geo.CPC = (dims->Z + 31) / 32;
    geo.n = n;
    geo.YZ = (int64_t)dims->Y * dims->Z;
    geo.nchunks = (int64_t)dims->X * dims->Y * geo.CPC;
    geo.INF = (int32_t)(n + 1);
    auto fail = [&](cg_status st) {
        colgraph_free(g);
        return st;
    };
    cudaStream_t st = g->stream;
    {  // keep freed workspaces cached in the stream-ordered pool (repeated solves allocate for free)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dd.device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    g->ws_bytes = workspace_bytes(geo);
    if (cudaMallocAsync(&g->ws, g->ws_bytes, st) != cudaSuccess) {
        g->ws = nullptr;
        return fail(CG_E_NOMEM);
    }
    if (cudaHostAlloc(&g->h_cnt, sizeof(unsigned) * 16, cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc(&g->h_work, sizeof(unsigned long long) * RING, cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc(&g->h_u64, sizeof(unsigned long long) * 16, cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc(&g->h_flags, sizeof(int) * 16, cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc(&g->h_bst, sizeof(BfsState), cudaHostAllocDefault) != cudaSuccess)
        return fail(CG_E_NOMEM);
    if (cudaEventCreate(&g->ev0) != cudaSuccess || cudaEventCreate(&g->ev1) != cudaSuccess) return fail(CG_E_CUDA);
    const int64_t ncol = (int64_t)geo.X * geo.Y;
    char *p = g->ws;
    int32_t *soa = carve<int32_t>(p, 8 * n);
    g->s.E = soa;
    g->s.H = soa + n;
    g->s.T = soa + 2 * n;
    g->s.D = soa + 3 * n;
    g->s.L = soa + 4 * n;
    g->blist[0] = carve<int>(p, n);
    g->blist[1] = carve<int>(p, n);
    g->clist[0] = carve<int>(p, geo.nchunks);
    g->clist[1] = carve<int>(p, geo.nchunks);
    g->cstamp = carve<int>(p, geo.nchunks);
    g->vstamp = carve<int>(p, n);
    g->vertex_lists = getenv("CG_CHUNK_LISTS") == nullptr;
    g->top = carve<int32_t>(p, ncol);
    g->proc = carve<int32_t>(p, ncol);
    g->colstamp = carve<int>(p, ncol);
    g->collist[0] = carve<int>(p, ncol);
    g->collist[1] = carve<int>(p, ncol);
    g->hist = carve<unsigned>(p, GAP_BINS);
    g->bst = carve<BfsState>(p, 1);
    g->cnt = carve<unsigned>(p, 16);
    g->work = carve<unsigned long long>(p, RING);
    g->u64 = carve<unsigned long long>(p, 16);
    g->flags = carve<int>(p, 16);
    if (cudaMemsetAsync(g->s.H, 0, sizeof(int32_t) * n, st) != cudaSuccess ||
        cudaMemsetAsync(g->s.D, 0, sizeof(int32_t) * 5 * n, st) != cudaSuccess ||
        cudaMemsetAsync(g->cstamp, 0, sizeof(int) * geo.nchunks, st) != cudaSuccess ||
        cudaMemsetAsync(g->vstamp, 0, sizeof(int) * n, st) != cudaSuccess ||
        cudaMemsetAsync(g->colstamp, 0, sizeof(int) * ncol, st) != cudaSuccess ||
        cudaMemsetAsync(g->cnt, 0, sizeof(unsigned) * 16, st) != cudaSuccess ||
        cudaMemsetAsync(g->u64, 0, sizeof(unsigned long long) * 16, st) != cudaSuccess ||
        cudaMemsetAsync(g->flags, 0, sizeof(int) * 16, st) != cudaSuccess)
        return fail(CG_E_CUDA);
    k_build<<<grid_for(ncol * 32, 256, g->num_sms * 16), 256, 0, st>>>(geo, cost_dev, input_is_weight ? 1 : 0, g->s,
                                                                       g->u64, g->flags);
    if (cudaGetLastError() != cudaSuccess) return fail(CG_E_CUDA);
    cudaMemcpyAsync(g->h_u64, g->u64, sizeof(unsigned long long) * 2, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(g->h_flags, g->flags, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(CG_E_CUDA);
    if (g->h_flags[0] & FLAG_OVERFLOW) return fail(CG_E_OVERFLOW);
    g->N = (int64_t)g->h_u64[0];
    g->sumT0 = (int64_t)g->h_u64[1];
    g->st.source_capacity = g->N;
    g->st.bytes_per_sweep_alg = 32.0 * (double)n;
    g->st.kernel_launches = 1;
    g->st.ms_build = now_ms() - t0;
    *out = g;
    return CG_OK;
}

cg_status maxflow_solve(cg_graph *g, const cg_solve_opts *opts, int64_t *flow_value, cg_solve_stats *stats) {
    if (!g || !flow_value) return CG_E_INVAL;
    if (g->solved) return CG_E_STATE;
    DeviceGuard dg(g->dist.device);
    cg_solve_opts o{1.0f, 0, 16, (int64_t)1 << 30, 1, 0};
    if (opts) o = *opts;
    if (o.walk_len == 0) o.walk_len = getenv("CG_WALK") ? atoi(getenv("CG_WALK")) : 64;  // library default
    o.check_every = std::max(1, std::min(o.check_every, RING));
    o.ops_per_sweep = std::max(1, o.ops_per_sweep);
    if (!(o.gr_factor > 0.f)) o.gr_factor = 1.0f;
    const Geo &geo = g->geo;
    cudaStream_t st = g->stream;
    const bool trace = tracing();
    const double t0 = now_ms();
    double ms_gr = 0.0, last_gr_ms = 0.0;
    auto timed_gr = [&]() {
        const double a = now_ms();
        const int64_t p0 = g->st.gr_passes;
        const cg_status s = global_relabel(g);
        last_gr_ms = now_ms() - a;
        ms_gr += last_gr_ms;
        if (trace) {
            // diagnostics only: current flow into t and total excess on active vertices
            cudaMemsetAsync(g->u64 + 2, 0, sizeof(unsigned long long), st);
            k_sum_T<<<g->num_sms * 8, 256, 0, st>>>(geo, g->s.T, g->u64 + 2);
            cudaMemcpyAsync(g->h_u64 + 2, g->u64 + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            fprintf(stderr, "[cg] GR#%lld levels=%lld active=%llu ms=%.3f (sweeps %lld) flow=%lld\n",
                    (long long)g->st.global_relabels, (long long)(g->st.gr_passes - p0), g->h_u64[3], last_gr_ms,
                    (long long)g->st.sweeps, (long long)(g->sumT0 - (int64_t)g->h_u64[2]));
        }
        return s;
    };
    // a1': exact per-column pre-cancellation (valid initial preflow)
    const size_t pc_smem = (size_t)8 * (geo.Z + 1) * sizeof(long long);
    if (getenv("CG_PRECANCEL") && pc_smem <= 200 * 1024) {  // opt-in: measured slower on C4/C5
        if (pc_smem > 48 * 1024)
            CG_CUDA(cudaFuncSetAttribute(k_precancel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pc_smem));
        k_precancel<<<grid_for((int64_t)geo.X * geo.Y * 32, 256, g->num_sms * 16), 256, pc_smem, st>>>(geo, g->s,
                                                                                                        g->flags);
        g->st.kernel_launches++;
        CG_CUDA(cudaGetLastError());
    }
    cg_status rs = timed_gr();
    if (rs) return rs;
    int64_t active = (int64_t)g->h_u64[3];
    const double gr_budget = (double)o.gr_factor * (double)geo.n;
    double work_since_gr = 0.0, sweep_ms_since_gr = 0.0;
    int64_t sweeps = 0, since_gap = 0;
    const int grid = list_grid(g, geo.nchunks);
    const int gridv = list_grid(g, (geo.n + 31) / 32);
    const double walk_min = getenv("CG_WALK_MIN") ? atof(getenv("CG_WALK_MIN")) : 1e-3;
    int64_t last_active = active;
    cg_status result = CG_OK;
    while (active > 0) {
        if (sweeps >= o.max_sweeps) { result = CG_E_NOT_CONVERGED; break; }
        const int batch = (int)std::min<int64_t>(o.check_every, o.max_sweeps - sweeps);
        CG_CUDA(cudaMemsetAsync(g->work, 0, sizeof(unsigned long long) * batch, st));
        CG_CUDA(cudaEventRecord(g->ev0, st));
        // multi-hop walks while many vertices are active; single hops in the sparse tail
        const bool walk = o.walk_len > 0 && (double)last_active >= walk_min * (double)geo.n;
        // size the grid for the current worklist (the kernels stride, so growth is safe)
        const int gv = std::max(g->num_sms, std::min(gridv, grid_for(2 * last_active, 256, gridv)));
        for (int i = 0; i < batch; i++) {
            const int k = g->sweep_par++;
            if (walk)
                k_walk<<<gv, 256, 0, st>>>(geo, g->s, o.walk_len, g->blist[k & 1], g->cnt + k % 3,
                                           g->blist[(k + 1) & 1], g->cnt + (k + 1) % 3, g->cnt + (k + 2) % 3,
                                           g->vstamp, ++g->tag, g->work + i, g->flags);
            else if (g->vertex_lists)
                k_sweep_v<<<gv, 256, 0, st>>>(geo, g->s, o.ops_per_sweep, g->blist[k & 1], g->cnt + k % 3,
                                              g->blist[(k + 1) & 1], g->cnt + (k + 1) % 3, g->cnt + (k + 2) % 3,
                                              g->vstamp, ++g->tag, g->work + i, g->flags);
            else
                k_sweep<<<grid, 256, 0, st>>>(geo, g->s, o.ops_per_sweep, g->clist[k & 1], g->cnt + k % 3,
                                              g->clist[(k + 1) & 1], g->cnt + (k + 1) % 3, g->cnt + (k + 2) % 3,
                                              g->cstamp, ++g->tag, g->work + i, g->flags);
        }
        CG_CUDA(cudaEventRecord(g->ev1, st));
        g->st.kernel_launches += batch;
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaMemcpyAsync(g->h_work, g->work, sizeof(unsigned long long) * batch, cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaMemcpyAsync(g->h_flags, g->flags, sizeof(int), cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaStreamSynchronize(st));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g->ev0, g->ev1);
        g->st.ms_sweep_kernels += ms;
        sweep_ms_since_gr += ms;
        if (g->h_flags[0] & FLAG_OVERFLOW) { result = CG_E_OVERFLOW; break; }
        if (trace) {
            fprintf(stderr, "[cg] sweeps %lld..%lld active:", (long long)sweeps, (long long)(sweeps + batch - 1));
            for (int i = 0; i < batch; i += std::max(1, batch / 8)) fprintf(stderr, " %llu", g->h_work[i]);
            fprintf(stderr, " | %.3f ms\n", ms);
        }
        bool quiescent = false;
        last_active = (int64_t)g->h_work[batch - 1];
        for (int i = 0; i < batch; i++) {
            const unsigned long long c = g->h_work[i];
            g->st.sweep_bytes_alg += 44.0 * (double)c;  // 32 B state read + 12 B push writes
            if (c == 0) { quiescent = true; break; }
            work_since_gr += (double)c;
            g->st.work += (int64_t)c;
        }
        sweeps += batch;
        since_gap += batch;
        g->st.sweeps = sweeps;
        if (quiescent || work_since_gr >= gr_budget || sweep_ms_since_gr >= std::max(last_gr_ms, 0.05)) {
            // a4: termination is decided only after an exact global relabel
            rs = timed_gr();
            if (rs) { result = rs; break; }
            active = (int64_t)g->h_u64[3];
            last_active = active;
            work_since_gr = 0.0;
            sweep_ms_since_gr = 0.0;
            since_gap = 0;
        } else if (o.gap_every > 0 && since_gap >= o.gap_every) {
            rs = run_gap(g);
            if (rs) { result = rs; break; }
            since_gap = 0;
        }
    }
    if (result != CG_OK && result != CG_E_NOT_CONVERGED) return result;
    // a6: |f| = sum(T0) - sum(T)
    CG_CUDA(cudaMemsetAsync(g->u64 + 2, 0, sizeof(unsigned long long), st));
    k_sum_T<<<g->num_sms * 8, 256, 0, st>>>(geo, g->s.T, g->u64 + 2);
    g->st.kernel_launches++;
    CG_CUDA(cudaMemcpyAsync(g->h_u64 + 2, g->u64 + 2, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    CG_CUDA(cudaGetLastError());
    *flow_value = g->sumT0 - (int64_t)g->h_u64[2];
    g->st.gap_lifted = (int64_t)g->h_u64[4];
    g->st.ms_global_relabel = ms_gr;
    g->st.ms_solve = now_ms() - t0;
    g->st.ms_sweeps = g->st.ms_solve - ms_gr;
    g->solved = true;
    if (stats) *stats = g->st;
    return result;
}

cg_status mincut_extract_surface(cg_graph *g, int32_t *surface_dev, uint8_t *mask_dev) {
    if (!g || !surface_dev) return CG_E_INVAL;
    if (!g->solved) return CG_E_STATE;
    DeviceGuard dg(g->dist.device);
    const Geo &geo = g->geo;
    cudaStream_t st = g->stream;
    const double t0 = now_ms();
    const int64_t ncol = (int64_t)geo.X * geo.Y;
    CG_CUDA(cudaMemsetAsync(g->cnt + 8, 0, 3 * sizeof(unsigned), st));
    const int tag = ++g->tag;
    k_ext_seed<<<grid_for(ncol, 256, g->num_sms * 16), 256, 0, st>>>(geo, g->s, g->top, g->proc, g->collist[0],
                                                                      g->cnt + 8, g->colstamp, tag);
    g->st.kernel_launches++;
    const int grid = list_grid(g, ncol);
    int r = 0;
    for (;;) {
        for (int b = 0; b < EXT_BATCH; b++, r++) {
            k_ext_round<<<grid, 256, 0, st>>>(geo, g->s, g->collist[r & 1], g->cnt + 8 + r % 3,
                                               g->collist[(r + 1) & 1], g->cnt + 8 + (r + 1) % 3,
                                               g->cnt + 8 + (r + 2) % 3, g->top, g->proc, g->colstamp, ++g->tag);
        }
        g->st.kernel_launches += EXT_BATCH;
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaMemcpyAsync(g->h_cnt + 8, g->cnt + 8 + r % 3, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaStreamSynchronize(st));
        if (g->h_cnt[8] == 0) break;
    }
    g->st.extract_passes += r;
    CG_CUDA(cudaMemsetAsync(g->flags + 3, 0, sizeof(int), st));
    k_ext_out<<<g->num_sms * 8, 256, 0, st>>>(geo, g->top, surface_dev, mask_dev, g->flags + 3);
    g->st.kernel_launches++;
    CG_CUDA(cudaMemcpyAsync(g->h_flags + 3, g->flags + 3, sizeof(int), cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    CG_CUDA(cudaGetLastError());
    g->st.ms_extract = now_ms() - t0;
    return g->h_flags[3] ? CG_E_EMPTY_COLUMN : CG_OK;
}

cg_status colgraph_stats(const cg_graph *g, cg_solve_stats *stats) {
    if (!g || !stats) return CG_E_INVAL;
    *stats = g->st;
    return CG_OK;
}

cg_status colgraph_export_state(cg_graph *g, int32_t *out_dev) {
    if (!g || !out_dev) return CG_E_INVAL;
    DeviceGuard dg(g->dist.device);
    CG_CUDA(cudaMemcpyAsync(out_dev, g->s.E, sizeof(int32_t) * 8 * g->geo.n, cudaMemcpyDeviceToDevice, g->stream));
    CG_CUDA(cudaStreamSynchronize(g->stream));
    return CG_OK;
}

cg_status colgraph_solve_host(const cg_dims *dims, const int32_t *cost_host, int32_t input_is_weight,
                              const cg_dist *dist, const cg_solve_opts *opts, int64_t *flow_value,
                              int32_t *surface_host, uint8_t *mask_host, cg_solve_stats *stats) {
    if (!dims || !cost_host || !flow_value || !surface_host) return CG_E_INVAL;
    if (dims->X < 1 || dims->Y < 1 || dims->Z < 1) return CG_E_INVAL;
    cg_dist dd{0, 1, nullptr, 0, nullptr};
    if (dist) dd = *dist;
    if (dd.nranks != 1) return CG_E_INVAL;
    DeviceGuard dg(dd.device);
    cudaStream_t st = (cudaStream_t)dd.stream;
    const int64_t n = (int64_t)dims->X * dims->Y * dims->Z, ncol = (int64_t)dims->X * dims->Y;
    int32_t *d_in = nullptr, *d_surf = nullptr;
    uint8_t *d_mask = nullptr;
    CG_CUDA(cudaMallocAsync(&d_in, sizeof(int32_t) * n, st));
    CG_CUDA(cudaMallocAsync(&d_surf, sizeof(int32_t) * ncol, st));
    if (mask_host) CG_CUDA(cudaMallocAsync(&d_mask, n, st));
    CG_CUDA(cudaMemcpyAsync(d_in, cost_host, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    cg_graph *g = nullptr;
    cg_status s = colgraph_build(dims, d_in, input_is_weight, &dd, &g);
    cudaFreeAsync(d_in, st);
    if (s == CG_OK) s = maxflow_solve(g, opts, flow_value, stats);
    cg_status se = CG_OK;
    if (s == CG_OK) {
        se = mincut_extract_surface(g, d_surf, d_mask);
        if (se == CG_OK || se == CG_E_EMPTY_COLUMN) {
            cudaMemcpyAsync(surface_host, d_surf, sizeof(int32_t) * ncol, cudaMemcpyDeviceToHost, st);
            if (mask_host) cudaMemcpyAsync(mask_host, d_mask, n, cudaMemcpyDeviceToHost, st);
            if (cudaStreamSynchronize(st) != cudaSuccess) se = CG_E_CUDA;
        }
        if (stats) *stats = g->st;
    }
    colgraph_free(g);
    cudaFreeAsync(d_surf, st);
    if (d_mask) cudaFreeAsync(d_mask, st);
    cudaStreamSynchronize(st);
    return s != CG_OK ? s : se;
}

}  // extern "C"
