// colgraph.cu -- host side of the B200 column-graph max-flow library (include/colgraph.h).
//
// Hot path of arXiv 2601.17026 (§3.2), redesigned for one GPU per process:
// the paper's per-thread FIFO queues, per-vertex locks and level barriers (§3.2.1-3.2.4)
// become device worklists, single-decrementer atomics and level kernels launched back to
// back on one stream; the host reads a few counters every `check_every` sweeps.
//
// Solve loop:
//   a2  exact global relabel (frontier BFS from t) -> rebuild the active-vertex list
//   a3  sweeps over the active list (a batch of check_every launches without host sync)
//   a5  re-run the global relabel when the work since the last one reaches gr_factor*n
//        or the sweep time since the last one exceeds its cost
//   a4  when a sweep finds no active vertex: exact global relabel; stop if no vertex with
//       excess has a finite height (the preflow is then maximum)
//   a6  |f| = sum(T0) - sum(T)
//
// x-slabs (§8(e), §3.2.1 column segmentation): the volume is cut into
// contiguous x-ranges ("slabs"), each with a ghost plane of its neighbours.  After every
// sweep the slabs exchange one halo message per side (k_halo_pack/unpack); the global
// relabel becomes label-correcting waves + ghost-height exchanges until no label changes;
// the extraction exchanges column tops.  Two transports share this driver:
//   NCCL    one slab per process/GPU (colgraph_build with nranks > 1): ncclSend/Recv to
//           the x-neighbours, ncclAllReduce for counts;
//   LOCAL   several slabs in one process (colgraph_build_slabs): the same messages moved
//           with device-to-device copies -- used to test the multi-slab algorithm on one GPU.
#include "colgraph.h"
#include "kernels.cuh"
#include "relabel.cuh"
#include "nccl_shim.h"
#include "nccl_loopback.h"
#include "tile.cuh"
#include "bk.cuh"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

using namespace cg;

namespace {
constexpr int RING = 256;
constexpr int BFS_BATCH = 32;
constexpr int EXT_BATCH = 16;
constexpr int LC_BATCH = 16;

struct Slab {
    Geo geo{};
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    int x0 = 0, x1 = 0;  // owned global x-range
    char *ws = nullptr;
    Soa s{};
    int *blist[2] = {nullptr, nullptr};  // BFS frontiers / sweep worklists (vertices)
    int *vstamp = nullptr;               // per-vertex list tag
    int32_t *top = nullptr, *proc = nullptr;  // per column (top has ghost columns)
    int *colstamp = nullptr;
    int *collist[2] = {nullptr, nullptr};
    unsigned *hist = nullptr;
    BfsState *bst = nullptr;
    unsigned *cnt = nullptr;             // [0..2] sweep lists, [4..6] lc waves, [8..10] extraction, [12] changes
    unsigned long long *work = nullptr;  // [2*RING] per sweep: operations, relabels
    unsigned long long *visits = nullptr;  // [RING] tile visits per phase
    unsigned *heads = nullptr;             // [RING] work-fetch cursors of k_walk_ws
    unsigned *visited = nullptr;           // [n/32 + 1] BFS visited bitmap (persistent BFS)
    unsigned *dbits = nullptr;             // [7][n/32 + 1] dense BFS levels: Dm, Lm0..3, F0, F1 bit planes
    int32_t *lab = nullptr;                // column-fixpoint relabel: labels, planes [-YZ, n + YZ)
    uint8_t *gflags = nullptr;             // column-fixpoint relabel: residual-arc flags, same range
    ColGrState *cst = nullptr, *h_cst = nullptr;
    int colgr_grid = 0;                    // > 0: cooperative grid of k_colgr_run
    int32_t *band = nullptr;               // narrow band (lo, hi) per column (NEXT-3), device copy; null = none
    unsigned long long *u64 = nullptr;   // [0]=N [1]=sumT0 [2]=sumT [3]=active [4]=gap lifted [5]=scratch
    int *flags = nullptr;                // [0]=overflow [1]=maxh [2]=gap [3]=empty
    int32_t *snap[2] = {nullptr, nullptr};   // ghost lateral residual at the last refresh
    int32_t *ssnap[2] = {nullptr, nullptr};  // ghost soft-arc flows at the last refresh (soft graphs)
    int32_t *hold[2] = {nullptr, nullptr};   // ghost heights before the last relabel exchange
    int32_t *hsend[2] = {nullptr, nullptr};  // halo messages (4 planes)
    int32_t *hrecv[2] = {nullptr, nullptr};
    // pinned host mirrors
    unsigned *h_cnt = nullptr;
    unsigned long long *h_work = nullptr, *h_u64 = nullptr, *h_visits = nullptr;
    int *h_flags = nullptr;
    BfsState *h_bst = nullptr;
    char *h_block = nullptr;  // pinned scratch the h_* mirrors are carved from (pinned_acquire)
    int64_t N = 0, sumT0 = 0;
    int tag = 0;       // monotone list tag
    int sweep_k = 0;   // sweeps since the last list rebuild (list/counter parity)
    int out_tag = 0;   // tag of the list the last sweep wrote (halo appends must reuse it)
    int wave_k = 0;    // label-correcting waves since the relabel started
    int ext_k = 0;     // extraction rounds
    // tile discharge (tile.cuh)
    int bfs_coop_grid = 0;      // > 0: persistent cooperative BFS (k_bfs_run) with this grid
    bool tiles = false;
    TileGeo tg{};
    int tS = 0;                 // lane segment length (template instance)
    int tgrid = 0;              // persistent grid of k_tile_phase
    size_t tsmem = 0;           // dynamic shared memory per CTA
    TileLists tl{};
    int tphase = 0;             // next phase number (colour = phase & 1)
};
}  // namespace

struct cg_graph {
    cg_dims dims{};
    cg_dist dist{};
    int nranks = 1, rank = 0;   // global slab count / this process's first slab
    bool local = true;          // LOCAL transport (all slabs in this process)
    std::vector<Slab *> slabs;  // slabs owned by this process
    ncclComm_t comm = nullptr;
    int64_t *d_red = nullptr;   // NCCL allreduce buffer
    // in-process slabs: descriptors + state of the all-slab BFS launch (k_bfs_run_slabs)
    SlabBfsDesc *d_sdesc = nullptr;
    MultiBfsState *d_mst = nullptr, *h_mst = nullptr;
    std::vector<SlabBfsDesc> h_sdesc;
    int mslab_grid = 0;
    int64_t *h_red = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int64_t n_global = 0;
    bool solved = false;
    bool exported = false;      // phase 2 ran (maxflow_export_flow): the preflow is now a flow
    bool top_ready = false;     // the solve ended on a source-side termination check: top[] is S
    unsigned trunc_small = 0, trunc_levels = 0;  // truncated relabels (CG_BFS_TRUNC), 0 = off
    bool trunc_until_quiescent = true;           // truncation ends with the first quiescent batch of a solve
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

#define CG_NCCL(call)                                                                   \
    do {                                                                                \
        ncclResult_t r_ = (call);                                                       \
        if (r_ != ncclSuccess) {                                                        \
            if (getenv("CG_DEBUG")) fprintf(stderr, "colgraph: %s -> nccl %d\n", #call, (int)r_); \
            return CG_E_NCCL;                                                           \
        }                                                                               \
    } while (0)

#define CG_TRY(expr)                 \
    do {                             \
        cg_status s_ = (expr);       \
        if (s_ != CG_OK) return s_;  \
    } while (0)

// CG_DEBUG_BOUNDS builds: CG_E_CUDA if any kernel indexed state out of range
inline cg_status debug_check(cg_status s) {
#ifdef CG_DEBUG_BOUNDS
    unsigned long long oob = 0;
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(&oob, g_oob, sizeof(oob)) != cudaSuccess) return CG_E_CUDA;
    if (oob) {
        fprintf(stderr, "colgraph: %llu out-of-range state accesses\n", oob);
        return CG_E_CUDA;
    }
#endif
    return s;
}

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
inline int list_grid(const Slab *sl, int64_t items) { return grid_for(items * 32, 256, sl->num_sms * 8); }

// NCCL communicators, cached by (unique id, rank, nranks, device): ncclCommInitRank costs tens
// to hundreds of milliseconds, and a job that builds one handle per solve with the same id
// (bench.py --gpus N) would otherwise pay it inside every solve.  A communicator is in use by
// at most one handle at a time; colgraph_free returns it to the cache.
struct CommEntry {
    unsigned char id[sizeof(ncclUniqueId)];
    int rank, nranks, device;
    ncclComm_t comm;
    bool in_use;
};
std::mutex g_comm_mu;
std::vector<CommEntry> g_comms;

cg_status comm_acquire(const void *id, int rank, int nranks, int device, ncclComm_t *out) {
    {
        std::lock_guard<std::mutex> lk(g_comm_mu);
        for (CommEntry &e : g_comms)
            if (!e.in_use && e.rank == rank && e.nranks == nranks && e.device == device &&
                memcmp(e.id, id, sizeof(e.id)) == 0) {
                e.in_use = true;
                *out = e.comm;
                return CG_OK;
            }
    }
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm = nullptr;
    if (nccl().commInitRank(&comm, nranks, uid, rank) != ncclSuccess) return CG_E_NCCL;
    std::lock_guard<std::mutex> lk(g_comm_mu);
    CommEntry e{};
    memcpy(e.id, id, sizeof(e.id));
    e.rank = rank;
    e.nranks = nranks;
    e.device = device;
    e.comm = comm;
    e.in_use = true;
    g_comms.push_back(e);
    *out = comm;
    return CG_OK;
}

void comm_release(ncclComm_t comm) {
    std::lock_guard<std::mutex> lk(g_comm_mu);
    for (CommEntry &e : g_comms)
        if (e.comm == comm) {
            e.in_use = false;
            return;
        }
    nccl().commDestroy(comm);  // not from the cache
}

// Pinned host scratch blocks, recycled across handles: cudaHostAlloc / cudaFreeHost pin pages
// and synchronise the device, which made repeated build/free cycles occasionally cost
// tens of milliseconds.
constexpr size_t PINNED_BLOCK = 16384;
std::mutex g_pinned_mu;
std::vector<char *> g_pinned_free;

char *pinned_acquire() {
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        if (!g_pinned_free.empty()) {
            char *b = g_pinned_free.back();
            g_pinned_free.pop_back();
            return b;
        }
    }
    void *b = nullptr;
    if (cudaHostAlloc(&b, PINNED_BLOCK, cudaHostAllocPortable) != cudaSuccess) return nullptr;
    return (char *)b;
}

void pinned_release(char *b) {
    if (!b) return;
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.push_back(b);
}

template <typename T>
T *carve(char *&p, int64_t count) {
    T *r = reinterpret_cast<T *>(p);
    p += ((size_t)count * sizeof(T) + 255) & ~(size_t)255;
    return r;
}

// halo message per side: 4 planes (dE, dL, H, L) + for soft graphs 2 K planes (dF, F)
int64_t halo_msg_ints(const Geo &geo) {
    return std::max<int64_t>((4 + 2 * (int64_t)geo.soft_k) * geo.YZ, 8 * (int64_t)geo.Y);
}

size_t workspace_bytes(const Geo &geo) {
    const int64_t ncol = (int64_t)geo.X * geo.Y, plane = (int64_t)(geo.X + 2) * geo.YZ;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    size_t b = (8 + (CG_LAYOUT_AOS && CG_H_PLANE)) * al(sizeof(int32_t) * plane);
    // soft flows over the owned and the two ghost planes; per side a snapshot of the ghost copy
    if (geo.soft_k) b += al(sizeof(int32_t) * plane * 4 * geo.soft_k) + 2 * al(sizeof(int32_t) * geo.YZ * geo.soft_k);
    b += 3 * al(sizeof(int) * geo.n);
    b += 3 * al(sizeof(int32_t) * (ncol + 2 * geo.Y)) + 2 * al(sizeof(int) * ncol);
    b += al(sizeof(unsigned) * GAP_BINS) + al(sizeof(BfsState));
    b += al(sizeof(unsigned) * 16) + al(sizeof(unsigned long long) * 2 * RING) + al(sizeof(unsigned long long) * 16) +
         al(sizeof(int) * 16);
    b += 4 * al(sizeof(int32_t) * geo.YZ) + 4 * al(sizeof(int32_t) * halo_msg_ints(geo));
    b += 5 * al(sizeof(int) * ncol) + al(sizeof(unsigned) * 4) + al(sizeof(unsigned long long) * RING) +
         al(sizeof(unsigned long long) * 16) + al(sizeof(unsigned) * RING) + al(sizeof(unsigned) * (geo.n / 32 + 1)) +
         al(sizeof(unsigned) * 7 * (geo.n / 32 + 1));
    b += al(sizeof(int32_t) * plane) + al(plane) + al(sizeof(ColGrState)) + al(sizeof(int32_t) * 2 * ncol);
    return b;
}

void slab_free(Slab *sl) {
    if (!sl) return;
    if (sl->ws) cudaFreeAsync(sl->ws, sl->stream);
    pinned_release(sl->h_block);
    delete sl;
}

// Allocate and initialise a slab, then run a1 (k_build) on its x-range of cost_dev.
cg_status slab_build(Slab *sl, const int32_t *cost_dev, int weight_mode, const int32_t *band_dev) {
    const Geo &geo = sl->geo;
    cudaStream_t st = sl->stream;
    const int64_t n = geo.n, ncol = (int64_t)geo.X * geo.Y, plane = (int64_t)(geo.X + 2) * geo.YZ;
    {  // keep freed workspaces cached in the stream-ordered pool (repeated solves allocate for free)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, sl->device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    const size_t bytes = workspace_bytes(geo);
    if (cudaMallocAsync(&sl->ws, bytes, st) != cudaSuccess) {
        sl->ws = nullptr;
        return CG_E_NOMEM;
    }
    sl->h_block = pinned_acquire();
    if (!sl->h_block) return CG_E_NOMEM;
    {
        char *hp = sl->h_block;
        sl->h_cnt = carve<unsigned>(hp, 16);
        sl->h_work = carve<unsigned long long>(hp, 2 * RING);
        sl->h_u64 = carve<unsigned long long>(hp, 16);
        sl->h_flags = carve<int>(hp, 16);
        sl->h_bst = carve<BfsState>(hp, 1);
        sl->h_visits = carve<unsigned long long>(hp, RING);
        sl->h_cst = carve<ColGrState>(hp, 1);
        if (hp > sl->h_block + PINNED_BLOCK) return CG_E_NOMEM;
    }
    char *p = sl->ws;
#if CG_LAYOUT_AOS
    int32_t *rec = carve<int32_t>(p, 8 * plane) + 8 * geo.YZ;  // owned plane x = 0
    Field fl[8];
    for (int i = 0; i < 8; i++) fl[i] = Field{rec + i, -geo.YZ, geo.n + geo.YZ};
#else
    Field fl[8];
    for (int i = 0; i < 8; i++) fl[i] = Field{carve<int32_t>(p, plane) + geo.YZ, -geo.YZ, geo.n + geo.YZ};
#endif
    // soft flows: vertex index v in [-YZ, n + YZ) (ghost planes included), 4 K ints each
    sl->s.SF = geo.soft_k ? carve<int32_t>(p, plane * 4 * geo.soft_k) + geo.YZ * 4 * geo.soft_k : nullptr;
    for (int side = 0; side < 2; side++) sl->ssnap[side] = geo.soft_k ? carve<int32_t>(p, geo.YZ * geo.soft_k) : nullptr;
    sl->s.E = fl[0];
#if CG_LAYOUT_AOS && CG_H_PLANE
    sl->s.H = FieldH{carve<int32_t>(p, plane) + geo.YZ, -geo.YZ, geo.n + geo.YZ};
#else
    sl->s.H = FieldH{fl[1].p, fl[1].lo, fl[1].hi};
#endif
    sl->s.T = fl[2];
    sl->s.D = fl[3];
    for (int d = 0; d < 4; d++) sl->s.L[d] = fl[4 + d];
    sl->blist[0] = carve<int>(p, n);
    sl->blist[1] = carve<int>(p, n);
    sl->vstamp = carve<int>(p, n);
    sl->top = carve<int32_t>(p, ncol + 2 * geo.Y) + geo.Y;
    sl->proc = carve<int32_t>(p, ncol + 2 * geo.Y) + geo.Y;
    sl->colstamp = carve<int>(p, ncol + 2 * geo.Y) + geo.Y;
    sl->collist[0] = carve<int>(p, ncol);
    sl->collist[1] = carve<int>(p, ncol);
    sl->hist = carve<unsigned>(p, GAP_BINS);
    sl->bst = carve<BfsState>(p, 1);
    sl->cnt = carve<unsigned>(p, 16);
    sl->work = carve<unsigned long long>(p, 2 * RING);
    sl->u64 = carve<unsigned long long>(p, 16);
    sl->flags = carve<int>(p, 16);
    const int64_t msg = halo_msg_ints(geo);
    for (int k = 0; k < 4; k++) sl->tl.list[k] = carve<int>(p, ncol);
    sl->tl.stamp = carve<int>(p, ncol);
    sl->tl.cnt = carve<unsigned>(p, 4);
    sl->tl.prof = carve<unsigned long long>(p, 16);
    sl->visits = carve<unsigned long long>(p, RING);
    sl->heads = carve<unsigned>(p, RING);
    sl->visited = carve<unsigned>(p, n / 32 + 1);
    sl->dbits = carve<unsigned>(p, 7 * (n / 32 + 1));
    sl->lab = carve<int32_t>(p, plane) + geo.YZ;
    sl->gflags = carve<uint8_t>(p, plane) + geo.YZ;
    sl->cst = carve<ColGrState>(p, 1);
    {
        int32_t *bnd = carve<int32_t>(p, 2 * ncol);
        sl->band = band_dev ? bnd : nullptr;
    }
    for (int side = 0; side < 2; side++) {
        sl->snap[side] = carve<int32_t>(p, geo.YZ);
        sl->hold[side] = carve<int32_t>(p, geo.YZ);
        sl->hsend[side] = carve<int32_t>(p, msg);
        sl->hrecv[side] = carve<int32_t>(p, msg);
    }
    // everything starts at zero (E, T written by k_build; heights set by the first relabel)
    CG_CUDA(cudaMemsetAsync(sl->ws, 0, bytes, st));
    if (sl->band) CG_CUDA(cudaMemcpyAsync(sl->band, band_dev, sizeof(int32_t) * 2 * ncol, cudaMemcpyDeviceToDevice, st));
    k_build<<<grid_for(ncol * 32, 256, sl->num_sms * 16), 256, 0, st>>>(geo, cost_dev, weight_mode, sl->band, sl->s, sl->u64,
                                                                        sl->flags);
    CG_CUDA(cudaGetLastError());
    CG_CUDA(cudaMemcpyAsync(sl->h_u64, sl->u64, sizeof(unsigned long long) * 2, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaMemcpyAsync(sl->h_flags, sl->flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    if (sl->h_flags[0] & FLAG_BAD_BAND) return CG_E_INVAL;
    if (sl->h_flags[0] & FLAG_OVERFLOW) return CG_E_OVERFLOW;
    sl->N = (int64_t)sl->h_u64[0];
    sl->sumT0 = (int64_t)sl->h_u64[1];
    return CG_OK;
}

// ---------------------------------------------------------------- transport

// Sum of per-slab int64 vectors over every slab of the job (in place on `v`, which holds
// this process's sum on entry).
cg_status gsum(cg_graph *g, int64_t *v, int count) {
    if (g->local || g->nranks == 1) return CG_OK;
    if (count > RING + 8) return CG_E_INVAL;
    Slab *sl = g->slabs[0];
    memcpy(g->h_red, v, sizeof(int64_t) * count);
    CG_CUDA(cudaMemcpyAsync(g->d_red, g->h_red, sizeof(int64_t) * count, cudaMemcpyHostToDevice, sl->stream));
    CG_NCCL(nccl().allReduce(g->d_red, g->d_red, count, ncclInt64, ncclSum, g->comm, sl->stream));
    CG_CUDA(cudaMemcpyAsync(g->h_red, g->d_red, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, sl->stream));
    CG_CUDA(cudaStreamSynchronize(sl->stream));
    memcpy(v, g->h_red, sizeof(int64_t) * count);
    return CG_OK;
}

cg_status gmax(cg_graph *g, int64_t *v) {
    if (g->local || g->nranks == 1) return CG_OK;
    Slab *sl = g->slabs[0];
    g->h_red[0] = *v;
    CG_CUDA(cudaMemcpyAsync(g->d_red, g->h_red, sizeof(int64_t), cudaMemcpyHostToDevice, sl->stream));
    CG_NCCL(nccl().allReduce(g->d_red, g->d_red, 1, ncclInt64, ncclMax, g->comm, sl->stream));
    CG_CUDA(cudaMemcpyAsync(g->h_red, g->d_red, sizeof(int64_t), cudaMemcpyDeviceToHost, sl->stream));
    CG_CUDA(cudaStreamSynchronize(sl->stream));
    *v = g->h_red[0];
    return CG_OK;
}

// Move `count` int32 of every slab's hsend[side] to the x-neighbour's hrecv[1-side].
cg_status transfer(cg_graph *g, int64_t count) {
    if (g->local) {
        const int R = (int)g->slabs.size();
        for (int r = 0; r + 1 < R; r++) {
            Slab *a = g->slabs[r], *b = g->slabs[r + 1];
            CG_CUDA(cudaMemcpyAsync(b->hrecv[0], a->hsend[1], sizeof(int32_t) * count, cudaMemcpyDeviceToDevice,
                                    a->stream));
            CG_CUDA(cudaMemcpyAsync(a->hrecv[1], b->hsend[0], sizeof(int32_t) * count, cudaMemcpyDeviceToDevice,
                                    a->stream));
        }
        return CG_OK;
    }
    Slab *sl = g->slabs[0];
    CG_NCCL(nccl().groupStart());
    if (sl->geo.gl) {
        CG_NCCL(nccl().send(sl->hsend[0], count, ncclInt32, g->rank - 1, g->comm, sl->stream));
        CG_NCCL(nccl().recv(sl->hrecv[0], count, ncclInt32, g->rank - 1, g->comm, sl->stream));
    }
    if (sl->geo.gh) {
        CG_NCCL(nccl().send(sl->hsend[1], count, ncclInt32, g->rank + 1, g->comm, sl->stream));
        CG_NCCL(nccl().recv(sl->hrecv[1], count, ncclInt32, g->rank + 1, g->comm, sl->stream));
    }
    CG_NCCL(nccl().groupEnd());
    return CG_OK;
}

bool multi(const cg_graph *g) { return g->nranks > 1; }

// a8: sweep halo (excess/residual deltas out, heights/residual refresh in); the receiving
// slab lists boundary vertices that got excess for its next sweep.
cg_status halo_sweep(cg_graph *g) {
    for (Slab *sl : g->slabs) {
        const Geo &geo = sl->geo;
        const int grid = grid_for(geo.YZ, 256, sl->num_sms * 4);
        if (geo.gl) k_halo_pack<<<grid, 256, 0, sl->stream>>>(geo, sl->s, 0, sl->snap[0], sl->ssnap[0], sl->hsend[0]);
        if (geo.gh) k_halo_pack<<<grid, 256, 0, sl->stream>>>(geo, sl->s, 1, sl->snap[1], sl->ssnap[1], sl->hsend[1]);
    }
    CG_TRY(transfer(g, (4 + 2 * (int64_t)g->slabs[0]->geo.soft_k) * g->slabs[0]->geo.YZ));
    for (Slab *sl : g->slabs) {
        const Geo &geo = sl->geo;
        const int grid = grid_for(geo.YZ, 256, sl->num_sms * 4);
        const int k = sl->sweep_k;  // the next sweep reads list[k&1] / cnt[k%3]
        const int tag = sl->out_tag;  // same tag as the sweep that wrote that list: no duplicates
        for (int side = 0; side < 2; side++)
            if (side ? geo.gh : geo.gl)
                k_halo_unpack<<<grid, 256, 0, sl->stream>>>(geo, sl->s, side, sl->hrecv[side], sl->hsend[side],
                                                            sl->snap[side], sl->ssnap[side], sl->blist[k & 1], sl->cnt + k % 3,
                                                            sl->vstamp, tag, sl->flags);
        g->st.kernel_launches += geo.gl + geo.gh;
    }
    CG_CUDA(cudaGetLastError());
    return CG_OK;
}

// ---------------------------------------------------------------- a2/a5 global relabel

// ghost planes' heights start at INF (unknown) for the label-correcting relabel
void k_fill_ghost_h(Slab *sl) {
    const Geo &geo = sl->geo;
    const int grid = grid_for(geo.YZ, 256, sl->num_sms * 4);
    if (geo.gl) k_fill<<<grid, 256, 0, sl->stream>>>(sl->s.H, -geo.YZ, geo.YZ, geo.INF);
    if (geo.gh) k_fill<<<grid, 256, 0, sl->stream>>>(sl->s.H, geo.n, geo.YZ, geo.INF);
}

// Strict level-synchronous BFS of one slab without neighbours (the single-GPU path).  flag_plane:
// the flag-plane BFS (k_bfs2_init + k_bfs_run<true>, labels in sl->lab; the default for hard
// graphs), else the record BFS (k_bfs_init + k_bfs_run<false> / k_bfs_step, labels in the records).
cg_status bfs_strict(cg_graph *g, Slab *sl, bool allow_coop = true, bool flag_plane = false, bool exhaustive = true) {
    const Geo &geo = sl->geo;
    cudaStream_t st = sl->stream;
    CG_CUDA(cudaMemsetAsync(sl->bst, 0, sizeof(BfsState), st));
    sl->h_bst->L = 1;
    sl->h_bst->small = getenv("CG_BFS_SMALL") ? (unsigned)atoi(getenv("CG_BFS_SMALL")) : BFS_RUN_SMALL;
    CG_CUDA(cudaMemcpyAsync(&sl->bst->L, &sl->h_bst->L, sizeof(int), cudaMemcpyHostToDevice, st));
    CG_CUDA(cudaMemcpyAsync(&sl->bst->small, &sl->h_bst->small, sizeof(unsigned), cudaMemcpyHostToDevice, st));
    sl->h_bst->bar[2] = getenv("CG_BAR_NS") ? (unsigned)atoi(getenv("CG_BAR_NS")) : 0;  // 0: 1024 ns
    CG_CUDA(cudaMemcpyAsync(&sl->bst->bar[2], &sl->h_bst->bar[2], sizeof(unsigned), cudaMemcpyHostToDevice, st));
    // truncated relabel (flag-plane BFS, not exhaustive): CG_BFS_TRUNC="small,levels" stops after
    // `levels` consecutive frontiers of <= `small` vertices
    sl->h_bst->trunc_small = sl->h_bst->trunc_levels = 0;
    if (flag_plane && !exhaustive && g->trunc_levels > 0) {
        sl->h_bst->trunc_small = g->trunc_small;
        sl->h_bst->trunc_levels = g->trunc_levels;
    }
    CG_CUDA(cudaMemcpyAsync(&sl->bst->trunc_small, &sl->h_bst->trunc_small, 2 * sizeof(unsigned),
                            cudaMemcpyHostToDevice, st));
    // bottom-up levels (flag-plane BFS): CG_BFS_BU="div,min"
    sl->h_bst->bu_div = sl->h_bst->bu_min = 0;
    if (flag_plane)
        if (const char *e = getenv("CG_BFS_BU")) {
            unsigned a = 0, b = 0;
            if (sscanf(e, "%u,%u", &a, &b) == 2) {
                sl->h_bst->bu_div = a;
                sl->h_bst->bu_min = b;
            }
        }
    CG_CUDA(cudaMemcpyAsync(&sl->bst->bu_div, &sl->h_bst->bu_div, 2 * sizeof(unsigned), cudaMemcpyHostToDevice, st));
    const bool coop = allow_coop && sl->bfs_coop_grid > 0;
    if (flag_plane && !coop) return CG_E_INVAL;
    // dense bit-plane levels for the large frontiers (one slab without ghost planes, Z % 32 == 0 so a
    // bitmap word is 32 z of one column, intervals < 32): CG_BFS_DENSE = frontier threshold in
    // vertices (0: off; default n / 256)
    unsigned dense_min = 0;
    if (flag_plane && !geo.gl && !geo.gh && geo.Z % 32 == 0 && geo.dl[0] < 32 && geo.dl[1] < 32 && geo.dl[2] < 32 &&
        geo.dl[3] < 32) {
        const char *e = getenv("CG_BFS_DENSE");
        const long long dm = e ? atoll(e) : std::max<long long>(1, geo.n / 256);
        dense_min = (unsigned)std::max<long long>(0, std::min<long long>(dm, 0xffffffffll));
    }
    unsigned *dbits = dense_min ? sl->dbits : nullptr;
    if (flag_plane)
        k_bfs2_init<<<grid_for(geo.n, 256, sl->num_sms * 16), 256, 0, st>>>(geo, sl->s, sl->gflags, sl->lab,
                                                                             sl->visited, sl->blist[0], &sl->bst->cnt[0],
                                                                             dbits);
    else
        k_bfs_init<<<grid_for(geo.n, 256, sl->num_sms * 16), 256, 0, st>>>(geo, sl->s, sl->blist[0], &sl->bst->cnt[0],
                                                                            coop ? sl->visited : nullptr);
    k_bfs_seeded<<<1, 1, 0, st>>>(sl->bst);
    g->st.kernel_launches += 2;
    int L = 1;
    if (coop) {  // every level in one cooperative launch (k_bfs_run)
        const uint8_t *fl = flag_plane ? sl->gflags : nullptr;
        int32_t *lb = flag_plane ? sl->lab : nullptr;
        void *args[] = {(void *)&sl->geo, (void *)&sl->s,       (void *)&sl->blist[0], (void *)&sl->blist[1],
                        (void *)&sl->bst, (void *)&sl->visited, (void *)&fl,          (void *)&lb,
                        (void *)&dbits,   (void *)&dense_min};
        CG_CUDA(cudaLaunchCooperativeKernel(flag_plane ? (const void *)k_bfs_run<true> : (const void *)k_bfs_run<false>,
                                            sl->bfs_coop_grid, 512, args, 0, st));
        g->st.kernel_launches++;
        CG_CUDA(cudaMemcpyAsync(sl->h_bst, sl->bst, sizeof(BfsState), cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaStreamSynchronize(st));
        L = sl->h_bst->L;
        if (sl->h_bst->cnt[(L - 1) % 3] != 0 && !sl->h_bst->truncated) return CG_E_CUDA;
        g->st.gr_passes += L - 1;
        return CG_OK;
    }
    for (int batch = 0;; batch++) {
        const int nb = batch == 0 ? 8 : BFS_BATCH;
        for (int b = 0; b < nb; b++)
            k_bfs_step<<<sl->num_sms * 2, 512, 0, st>>>(geo, sl->s, sl->blist[0], sl->blist[1], sl->bst);
        g->st.kernel_launches += nb;
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaMemcpyAsync(sl->h_bst, sl->bst, sizeof(BfsState), cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaStreamSynchronize(st));
        L = sl->h_bst->L;
        if (sl->h_bst->cnt[(L - 1) % 3] == 0) break;
        if ((int64_t)L > (int64_t)geo.INF + 2) return CG_E_CUDA;  // every level claims >= 1 vertex
    }
    g->st.gr_passes += L - 1;
    return CG_OK;
}

// ---- column-scan fixpoint relabel (relabel.cuh; default for hard graphs with Z <= 256)
const void *colgr_kernel(int Z) {
    if (Z <= 32) return (const void *)k_colgr_run<1>;
    if (Z <= 64) return (const void *)k_colgr_run<2>;
    if (Z <= 96) return (const void *)k_colgr_run<3>;
    if (Z <= 128) return (const void *)k_colgr_run<4>;
    if (Z <= 32 * COLGR_MAX_CPC) return (const void *)k_colgr_run<COLGR_MAX_CPC>;
    return nullptr;
}

// the column fixpoint serves hard graphs with Z <= 256 on a device with cooperative launch;
// CG_RELABEL=bfs selects the vertex-frontier BFS (measured alternative)
// Relabel flavour: FLAGS = the flag-plane vertex BFS (default for hard graphs on
// one slab), COLGR = the column fixpoint (default on x-slabs: its exchanges count slab-boundary
// crossings, not BFS levels), RECORD = the record BFS (soft graphs, tiles, Z > 256 for the
// fixpoint, no cooperative launch).  CG_RELABEL = flags | colgr | bfs overrides where applicable.
// On x-slabs, BFS_COLGR = in-slab flag-plane BFS + the column fixpoint across slab boundaries.
enum RelabelKind { RELABEL_RECORD, RELABEL_FLAGS, RELABEL_COLGR, RELABEL_BFS_COLGR };
RelabelKind relabel_kind(const cg_graph *g) {
    const Slab *sl = g->slabs[0];
    if (sl->geo.soft_k || sl->tiles) return RELABEL_RECORD;
    const char *e = getenv("CG_RELABEL");
    if (e && !strcmp(e, "bfs")) return RELABEL_RECORD;
    const bool colgr_ok = sl->colgr_grid > 0;
    const bool flags_ok = sl->bfs_coop_grid > 0;
    if (e && !strcmp(e, "colgr") && colgr_ok) return RELABEL_COLGR;
    if (multi(g)) {
        if (e && !strcmp(e, "levels")) return RELABEL_RECORD;
        return colgr_ok && flags_ok ? RELABEL_BFS_COLGR : colgr_ok ? RELABEL_COLGR : RELABEL_RECORD;
    }
    return flags_ok ? RELABEL_FLAGS : RELABEL_RECORD;
}

cg_status colgr_launch(Slab *sl, int dense) {
    void *args[] = {(void *)&sl->geo, (void *)&sl->gflags, (void *)&sl->lab, (void *)&sl->collist[0],
                    (void *)&sl->collist[1], (void *)&sl->cst, (void *)&sl->colstamp, (void *)&dense};
    CG_CUDA(cudaLaunchCooperativeKernel(colgr_kernel(sl->geo.Z), sl->colgr_grid, 512, args, 0, sl->stream));
    return CG_OK;
}

// flags of the residual arcs + labels reset to INF over the ghost planes and (owned = true) the
// owned planes, fixpoint state
cg_status colgr_begin(cg_graph *g, Slab *sl, bool owned = true) {
    const Geo &geo = sl->geo;
    CG_CUDA(cudaMemsetAsync(sl->cst, 0, sizeof(ColGrState), sl->stream));
    sl->h_cst->small = getenv("CG_COLGR_SMALL") ? (unsigned)atoi(getenv("CG_COLGR_SMALL")) : 16;
    sl->h_cst->tag0 = sl->tag + 1;
    CG_CUDA(cudaMemcpyAsync(&sl->cst->small, &sl->h_cst->small, 2 * sizeof(int), cudaMemcpyHostToDevice, sl->stream));
    auto flags = [&](int64_t lo, int64_t hi) {
        k_colgr_flags<<<grid_for(hi - lo, 256, sl->num_sms * 16), 256, 0, sl->stream>>>(geo, sl->s, sl->gflags, sl->lab,
                                                                                         lo, hi);
        g->st.kernel_launches++;
    };
    if (owned) {
        flags(geo.gl ? -geo.YZ : 0, geo.n + (geo.gh ? geo.YZ : 0));
    } else {
        if (geo.gl) flags(-geo.YZ, 0);
        if (geo.gh) flags(geo.n, geo.n + geo.YZ);
    }
    CG_CUDA(cudaGetLastError());
    return CG_OK;
}

// after the fixpoint: round count, tags consumed
cg_status colgr_end(cg_graph *g, Slab *sl) {
    CG_CUDA(cudaMemcpyAsync(sl->h_cst, sl->cst, sizeof(ColGrState), cudaMemcpyDeviceToHost, sl->stream));
    CG_CUDA(cudaStreamSynchronize(sl->stream));
    sl->tag = sl->h_cst->tag0 + sl->h_cst->round + 1;
    g->st.gr_passes += sl->h_cst->round;
    return CG_OK;
}

// one slab without neighbours: flags, one cooperative launch for every round
cg_status colgr_strict(cg_graph *g, Slab *sl) {
    CG_TRY(colgr_begin(g, sl));
    CG_TRY(colgr_launch(sl, 1));
    g->st.kernel_launches++;
    return colgr_end(g, sl);
}

// x-slabs: every slab runs its fixpoint to local convergence, then the boundary planes' labels go
// to the neighbours' ghost planes; a boundary column facing a ghost column whose labels dropped
// restarts the fixpoint.  Stop when no slab listed anything (one global sum per exchange): the
// number of exchanges is the number of slab-boundary crossings of the shortest paths (+1), not the
// BFS depth (§3.2.2 L274-289 synchronises every level).
// In-process slabs: every slab's in-slab flag-plane BFS in ONE cooperative launch (k_bfs_run_slabs).
cg_status bfs_slabs_flags(cg_graph *g) {
    const int S = (int)g->slabs.size();
    Slab *s0 = g->slabs[0];
    cudaStream_t st = s0->stream;  // in-process slabs share the stream
    if (!g->d_sdesc) {
        CG_CUDA(cudaMalloc(&g->d_sdesc, sizeof(SlabBfsDesc) * S));
        CG_CUDA(cudaMalloc(&g->d_mst, sizeof(MultiBfsState)));
        CG_CUDA(cudaHostAlloc(&g->h_mst, sizeof(MultiBfsState), cudaHostAllocDefault));
        g->h_sdesc.resize(S);
        for (int k = 0; k < S; k++) {
            Slab *sl = g->slabs[k];
            g->h_sdesc[k] = SlabBfsDesc{sl->geo, sl->s, {sl->blist[0], sl->blist[1]}, sl->bst->cnt, sl->visited,
                                        sl->gflags, sl->lab};
        }
        CG_CUDA(cudaMemcpy(g->d_sdesc, g->h_sdesc.data(), sizeof(SlabBfsDesc) * S, cudaMemcpyHostToDevice));
    }
    for (Slab *sl : g->slabs) {
        const Geo &geo = sl->geo;
        CG_CUDA(cudaMemsetAsync(sl->bst, 0, sizeof(BfsState), st));
        k_bfs2_init<<<grid_for(geo.n, 256, sl->num_sms * 16), 256, 0, st>>>(geo, sl->s, sl->gflags, sl->lab,
                                                                             sl->visited, sl->blist[0], &sl->bst->cnt[0]);
        g->st.kernel_launches++;
    }
    CG_CUDA(cudaMemsetAsync(g->d_mst, 0, sizeof(MultiBfsState), st));
    g->h_mst->L = 1;
    CG_CUDA(cudaMemcpyAsync(&g->d_mst->L, &g->h_mst->L, sizeof(int), cudaMemcpyHostToDevice, st));
    int Sarg = S;
    void *args[] = {(void *)&g->d_sdesc, (void *)&Sarg, (void *)&g->d_mst};
    CG_CUDA(cudaLaunchCooperativeKernel((const void *)k_bfs_run_slabs, g->mslab_grid, 512, args, 0, st));
    g->st.kernel_launches++;
    CG_CUDA(cudaMemcpyAsync(g->h_mst, g->d_mst, sizeof(MultiBfsState), cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    g->st.gr_passes += g->h_mst->L - 1;
    return CG_OK;
}

//   bfs_init: each slab first computes its in-slab distances with the flag-plane BFS (paths that
//   stay inside the slab: upper bounds of the true distances, work-efficient); the fixpoint then
//   only corrects the labels that cross-slab paths lower.  Otherwise the fixpoint starts from INF.
cg_status colgr_slabs(cg_graph *g, bool bfs_init) {
    const bool all_slabs = bfs_init && g->local && g->mslab_grid > 0 && (int)g->slabs.size() <= MSLAB_MAX &&
                           !(getenv("CG_SLAB_BFS_EACH") && atoi(getenv("CG_SLAB_BFS_EACH")));
    if (all_slabs) CG_TRY(bfs_slabs_flags(g));
    for (Slab *sl : g->slabs) {
        if (bfs_init) {
            if (!all_slabs) CG_TRY(bfs_strict(g, sl, true, true));
            CG_TRY(colgr_begin(g, sl, false));
        } else {
            CG_TRY(colgr_begin(g, sl));
            CG_TRY(colgr_launch(sl, 1));
            g->st.kernel_launches++;
        }
    }
    const int64_t YZ = g->slabs[0]->geo.YZ;
    for (int iter = 0;; iter++) {
        for (Slab *sl : g->slabs) {
            k_colgr_pack<<<grid_for(2 * YZ, 256, sl->num_sms * 4), 256, 0, sl->stream>>>(sl->geo, sl->lab, sl->hsend[0],
                                                                                        sl->hsend[1]);
            g->st.kernel_launches++;
        }
        CG_TRY(transfer(g, YZ));
        int64_t listed = 0;
        for (Slab *sl : g->slabs) {
            const Geo &geo = sl->geo;
            k_colgr_unpack<<<grid_for((int64_t)(geo.gl + geo.gh) * geo.Y * 32, 256, sl->num_sms * 4), 256, 0,
                             sl->stream>>>(geo, sl->lab, sl->hrecv[0], sl->hrecv[1], sl->colstamp, sl->collist[0],
                                           sl->collist[1], sl->cst);
            g->st.kernel_launches++;
            CG_CUDA(cudaGetLastError());
            CG_CUDA(cudaMemcpyAsync(sl->h_cst, sl->cst, sizeof(ColGrState), cudaMemcpyDeviceToHost, sl->stream));
        }
        for (Slab *sl : g->slabs) {
            CG_CUDA(cudaStreamSynchronize(sl->stream));
            listed += sl->h_cst->cnt[sl->h_cst->round % 3];
        }
        CG_TRY(gsum(g, &listed, 1));
        if (listed == 0) {
            if (tracing()) fprintf(stderr, "[cg]   x-slab column fixpoint: %d boundary exchanges\n", iter + 1);
            break;
        }
        if (iter > 4 * (int64_t)g->dims.X + 64) return CG_E_CUDA;  // every exchange lowers some label
        for (Slab *sl : g->slabs)
            if (sl->h_cst->cnt[sl->h_cst->round % 3]) {
                CG_TRY(colgr_launch(sl, 0));
                g->st.kernel_launches++;
            }
    }
    for (Slab *sl : g->slabs) {
        const Geo &geo = sl->geo;
        k_colgr_ghost_h<<<grid_for(2 * YZ, 256, sl->num_sms * 4), 256, 0, sl->stream>>>(geo, sl->s, sl->lab);
        g->st.kernel_launches++;
        CG_TRY(colgr_end(g, sl));
    }
    return CG_OK;
}

// Level-synchronous relabel across slabs (default): every level, each slab expands its own
// frontier (claiming ghost predecessors in its ghost planes), the ghost planes go to their
// owners, and each owner claims the boundary vertices its neighbour reached -- exact BFS
// labels, one exchange per level (~#levels exchanges instead of the label-correcting
// variant's waves x outer rounds).  Termination is checked every SLAB_BATCH
// levels with one global sum.
constexpr int SLAB_BATCH = 8;
cg_status bfs_slabs_levels(cg_graph *g) {
    for (Slab *sl : g->slabs) {
        const Geo &geo = sl->geo;
        CG_CUDA(cudaMemsetAsync(sl->cnt + 4, 0, 3 * sizeof(unsigned), sl->stream));
        k_bfs_init<<<grid_for(geo.n, 256, sl->num_sms * 16), 256, 0, sl->stream>>>(geo, sl->s, sl->blist[0],
                                                                                     sl->cnt + 4);
        k_fill_ghost_h(sl);
        g->st.kernel_launches += 1 + geo.gl + geo.gh;
    }
    const int64_t YZ = g->slabs[0]->geo.YZ;
    int i = 0;  // level index: frontier of label i+1 in list[i&1] / cnt[4 + i%3]
    for (;;) {
        for (int b = 0; b < SLAB_BATCH; b++, i++) {
            const int nl = i + 2;
            for (Slab *sl : g->slabs) {
                const Geo &geo = sl->geo;
                k_slab_level<<<list_grid(sl, geo.n), 256, 0, sl->stream>>>(
                    geo, sl->s, nl, sl->blist[i & 1], sl->cnt + 4 + i % 3, sl->blist[(i + 1) & 1],
                    sl->cnt + 4 + (i + 1) % 3, sl->cnt + 4 + (i + 2) % 3);
                k_ghost_pack_h<<<grid_for(2 * YZ, 256, sl->num_sms * 4), 256, 0, sl->stream>>>(
                    geo, sl->s, sl->hsend[0], sl->hsend[1]);
                g->st.kernel_launches += 2;
            }
            CG_TRY(transfer(g, YZ));
            for (Slab *sl : g->slabs) {
                const Geo &geo = sl->geo;
                k_slab_ghost_claim<<<grid_for(2 * YZ * 32, 256, sl->num_sms * 4), 256, 0, sl->stream>>>(
                    geo, sl->s, sl->hrecv[0], sl->hrecv[1], nl, sl->blist[(i + 1) & 1], sl->cnt + 4 + (i + 1) % 3);
                g->st.kernel_launches++;
            }
            CG_CUDA(cudaGetLastError());
        }
        int64_t pending = 0;
        for (Slab *sl : g->slabs)
            CG_CUDA(cudaMemcpyAsync(sl->h_cnt + 4, sl->cnt + 4, 3 * sizeof(unsigned), cudaMemcpyDeviceToHost,
                                    sl->stream));
        for (Slab *sl : g->slabs) {
            CG_CUDA(cudaStreamSynchronize(sl->stream));
            pending += sl->h_cnt[4 + i % 3];
        }
        CG_TRY(gsum(g, &pending, 1));
        if (pending == 0) break;
        if ((int64_t)i > (int64_t)g->slabs[0]->geo.INF + SLAB_BATCH) return CG_E_CUDA;
    }
    g->st.gr_passes += i;
    // exact ghost labels for the sweeps: boundary heights -> neighbours' ghost planes
    for (Slab *sl : g->slabs) {
        const Geo &geo = sl->geo;
        const int grid = grid_for(YZ, 256, sl->num_sms * 4);
        if (geo.gl) k_halo_pack_h<<<grid, 256, 0, sl->stream>>>(geo, sl->s, 0, sl->hsend[0]);
        if (geo.gh) k_halo_pack_h<<<grid, 256, 0, sl->stream>>>(geo, sl->s, 1, sl->hsend[1]);
    }
    CG_TRY(transfer(g, YZ));
    for (Slab *sl : g->slabs) {
        const Geo &geo = sl->geo;
        const int grid = grid_for(YZ, 256, sl->num_sms * 4);
        for (int side = 0; side < 2; side++)
            if (side ? geo.gh : geo.gl)
                k_halo_unpack_h<<<grid, 256, 0, sl->stream>>>(geo, sl->s, side, sl->hrecv[side], sl->hold[side]);
    }
    CG_CUDA(cudaGetLastError());
    return CG_OK;
}

// a2/a5: global relabel + rebuild of every slab's active list; returns the global active count.
// exhaustive = false allows the truncated flag-plane BFS (g->trunc_levels > 0); a truncated relabel
// that leaves no active vertex is redone exhaustively (termination is decided only on an exact one)
cg_status global_relabel(cg_graph *g, int64_t *active, bool exhaustive = true) {
    const RelabelKind kind = relabel_kind(g);
    const bool colgr = kind != RELABEL_RECORD;  // labels are in sl->lab: the rebuild writes the records' H
    bool truncated = false;
    if (kind == RELABEL_COLGR || kind == RELABEL_BFS_COLGR) {
        CG_TRY(multi(g) ? colgr_slabs(g, kind == RELABEL_BFS_COLGR) : colgr_strict(g, g->slabs[0]));
    } else if (kind == RELABEL_FLAGS) {
        CG_TRY(bfs_strict(g, g->slabs[0], true, true, exhaustive));
        truncated = g->slabs[0]->h_bst->truncated != 0;
        g->st.gr_truncated += truncated;
    } else if (!multi(g)) {
        CG_TRY(bfs_strict(g, g->slabs[0]));
    } else {
        CG_TRY(bfs_slabs_levels(g));
    }
    int64_t act = 0;
    for (Slab *sl : g->slabs) {
        const Geo &geo = sl->geo;
        CG_CUDA(cudaMemsetAsync(sl->u64 + 3, 0, sizeof(unsigned long long), sl->stream));
        if (sl->tiles) {  // tile worklists: colour 0 tiles for the next even phase, colour 1 for the one after
            sl->tphase += sl->tphase & 1;
            CG_CUDA(cudaMemsetAsync(sl->tl.cnt, 0, 4 * sizeof(unsigned), sl->stream));
            k_tile_rebuild<<<sl->num_sms * 8, 256, 0, sl->stream>>>(geo, sl->tg, sl->s, sl->tl, sl->tphase,
                                                                    sl->u64 + 3);
        } else {
            CG_CUDA(cudaMemsetAsync(sl->cnt, 0, 3 * sizeof(unsigned), sl->stream));
            if (colgr)  // records' H = the relabel's labels, fused with the active list
                k_colgr_rebuild<<<grid_for(geo.n, 256, sl->num_sms * 16), 256, 0, sl->stream>>>(
                    geo, sl->s, sl->lab, sl->blist[0], sl->cnt, sl->vstamp, ++sl->tag, sl->u64 + 3);
            else
                k_rebuild_vertices<<<grid_for(geo.n, 256, sl->num_sms * 16), 256, 0, sl->stream>>>(
                    geo, sl->s, sl->blist[0], sl->cnt, sl->vstamp, ++sl->tag, sl->u64 + 3);
        }
        g->st.kernel_launches++;
        sl->sweep_k = 0;
        CG_CUDA(cudaMemcpyAsync(sl->h_u64 + 3, sl->u64 + 3, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                sl->stream));
    }
    for (Slab *sl : g->slabs) {
        CG_CUDA(cudaStreamSynchronize(sl->stream));
        act += (int64_t)sl->h_u64[3];
    }
    CG_CUDA(cudaGetLastError());
    CG_TRY(gsum(g, &act, 1));
    *active = act;
    g->st.global_relabels++;
    if (truncated && act == 0) {
        if (g->trunc_until_quiescent) g->trunc_levels = 0;
        return global_relabel(g, active, true);
    }
    return CG_OK;
}

// a5 gap heuristic (§2.1) over every slab of the job: the label histogram is
// summed over all slabs (LOCAL: added into slab 0's on the shared stream; NCCL: an int32
// allreduce of the histogram up to the global maximum label), so every slab finds the same
// smallest empty label g and lifts its own vertices above g to INF.  Ghost copies of lifted
// vertices are refreshed by the next halo exchange; a push into a stale ghost copy only moves
// excess onto a vertex that then waits at INF for the next exact relabel (a4 stays the safety net).
cg_status run_gap(cg_graph *g) {
    for (Slab *sl : g->slabs) {
        CG_CUDA(cudaMemsetAsync(sl->hist, 0, sizeof(unsigned) * GAP_BINS, sl->stream));
        CG_CUDA(cudaMemsetAsync(sl->flags + 1, 0, sizeof(int), sl->stream));
        k_gap_hist<<<sl->num_sms * 2, 512, 0, sl->stream>>>(sl->geo, sl->s.H, sl->hist, sl->flags + 1);
        g->st.kernel_launches++;
    }
    Slab *s0 = g->slabs[0];
    if (g->local) {  // in-process slabs share one stream: fold every histogram and maximum into slab 0's
        for (size_t i = 1; i < g->slabs.size(); i++) {
            Slab *sl = g->slabs[i];
            k_hist_fold<<<s0->num_sms * 4, 256, 0, s0->stream>>>(sl->hist, sl->flags + 1, s0->hist, s0->flags + 1);
            g->st.kernel_launches++;
        }
    } else if (multi(g)) {  // NCCL ranks: global maximum label, then the histogram up to it
        CG_CUDA(cudaMemcpyAsync(s0->h_flags + 1, s0->flags + 1, sizeof(int), cudaMemcpyDeviceToHost, s0->stream));
        CG_CUDA(cudaStreamSynchronize(s0->stream));
        int64_t mh = s0->h_flags[1];
        CG_TRY(gmax(g, &mh));
        const int32_t m32 = (int32_t)mh;
        CG_CUDA(cudaMemcpyAsync(s0->flags + 1, &m32, sizeof(int), cudaMemcpyHostToDevice, s0->stream));
        const size_t bins = (size_t)std::min<int64_t>(mh + 1, GAP_BINS);
        CG_NCCL(nccl().allReduce(s0->hist, s0->hist, bins, ncclInt32, ncclSum, g->comm, s0->stream));
        CG_CUDA(cudaStreamSynchronize(s0->stream));  // m32 is a host stack value
    }
    k_gap_find<<<1, 1024, 0, s0->stream>>>(s0->hist, s0->flags + 1, s0->flags + 2);
    g->st.kernel_launches++;
    for (Slab *sl : g->slabs) {
        if (sl != s0) CG_CUDA(cudaMemcpyAsync(sl->flags + 2, s0->flags + 2, sizeof(int), cudaMemcpyDeviceToDevice,
                                              s0->stream));
        k_gap_lift<<<sl->num_sms * 8, 256, 0, sl->stream>>>(sl->geo, sl->s.H, sl->flags + 2, sl->u64 + 4);
        g->st.kernel_launches++;
    }
    CG_CUDA(cudaGetLastError());
    g->st.gap_runs++;
    return CG_OK;
}

// ---------------------------------------------------------------- a3 on column tiles (tile.cuh)

typedef void (*TileKernel)(Geo, TileGeo, Soa, TileLists, int, unsigned long long *, unsigned long long *, int *);

TileKernel tile_kernel(int S) {
    switch (S) {
        case 1: return k_tile_phase<1>;
        case 2: return k_tile_phase<2>;
        case 3: return k_tile_phase<3>;
        case 4: return k_tile_phase<4>;
        case 6: return k_tile_phase<6>;
        case 8: return k_tile_phase<8>;
        default: return nullptr;
    }
}

int tile_max_threads_rt(int) { return 512; }

// Choose the lane segment S (>= ceil(Z/32)) and the largest tile shape that fits shared
// memory; false if Z is too tall for the instantiated sizes (the vertex-worklist sweep is
// used then).  CG_TILE=TXxTY overrides the shape.
bool tile_setup(Slab *sl, int steps, int relabel_every) {
    const Geo &geo = sl->geo;
    if (geo.soft_k) return false;  // tiles hold hard arcs only
    const int need = (geo.Z + 31) / 32;
    static const int sizes[] = {1, 2, 3, 4, 6, 8};
    int S = 0;
    for (int c : sizes)
        if (c >= need) { S = c; break; }
    if (!S) return false;
    int smem_max = 0;
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, sl->device);
    TileGeo t{};
    t.P = S | 1;
    t.CS = 32 * t.P;
    t.steps = steps;
    t.relabel_every = relabel_every;
    static const int shapes[][2] = {{4, 8}, {4, 4}, {2, 4}, {2, 2}, {1, 2}, {1, 1}};
    bool ok = false;
    int ox = 0, oy = 0;
    if (const char *e = getenv("CG_TILE")) sscanf(e, "%dx%d", &ox, &oy);
    for (auto &sh : shapes) {
        t.TX = ox > 0 ? ox : sh[0];
        t.TY = oy > 0 ? oy : sh[1];
        t.NC = t.TX * t.TY;
        t.NH = 2 * (t.TX + t.TY);
        if (t.NC * 32 <= tile_max_threads_rt(S) && tile_smem_bytes(t) <= (size_t)smem_max) { ok = true; break; }
        if (ox > 0) break;
    }
    if (!ok) return false;
    t.NTX = (geo.X + t.TX - 1) / t.TX;
    t.NTY = (geo.Y + t.TY - 1) / t.TY;
    TileKernel k = tile_kernel(S);
    const size_t bytes = tile_smem_bytes(t);
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) return false;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, t.NC * 32, bytes) != cudaSuccess || per_sm < 1)
        return false;
    sl->tg = t;
    sl->tS = S;
    sl->tsmem = bytes;
    sl->tgrid = sl->num_sms * per_sm;
    sl->tiles = true;
    if (!getenv("CG_TILE_PROF")) sl->tl.prof = nullptr;
    return true;
}

Geo make_geo(const cg_dims *dims, const int32_t *dl4, int x0, int x1, int nranks_total, bool gl, bool gh,
             int64_t n_global) {
    Geo geo{};
    geo.X = x1 - x0;
    geo.Y = dims->Y;
    geo.Z = dims->Z;
    for (int d = 0; d < 4; d++) geo.dl[d] = dl4[d];
    geo.CPC = (dims->Z + 31) / 32;
    geo.gl = gl;
    geo.gh = gh;
    geo.n = (int64_t)geo.X * geo.Y * geo.Z;
    geo.YZ = (int64_t)dims->Y * dims->Z;
    geo.nchunks = (int64_t)geo.X * geo.Y * geo.CPC;
    geo.INF = (int32_t)(n_global + 1);
    fastdiv_params((uint32_t)geo.Z, geo.mZ, geo.shZ);
    fastdiv_params((uint32_t)geo.Y, geo.mY, geo.shY);
    (void)nranks_total;
    return geo;
}

cg_status validate_dims(const cg_dims *dims) {
    if (!dims || dims->X < 1 || dims->Y < 1 || dims->Z < 1 || dims->delta < 0 || dims->delta_y < -1) return CG_E_INVAL;
    const int64_t n = (int64_t)dims->X * dims->Y * dims->Z;
    if (n + dims->Z + 64 >= (int64_t)INT_MAX) return CG_E_INVAL;
    return CG_OK;
}

}  // namespace

// Solver options with library defaults (NULL = defaults; 0 fields = defaults); use_tiles = the
// tile sweep was requested and set up.
cg_status normalize_opts(cg_graph *g, const cg_solve_opts *opts, cg_solve_opts &o, bool &use_tiles) {
    // check_every 8: the relabel triggers are checked every 8 sweeps (measured against 4 / 16:
    // C4 -5 %, C5 -13 %)
    o = cg_solve_opts{1.0f, 0, 8, (int64_t)1 << 30, 1, 0, 0, 0, 0};
    if (opts) o = *opts;
    if (o.check_every <= 0) o.check_every = 8;
    if (o.max_sweeps <= 0) o.max_sweeps = (int64_t)1 << 30;
    if (o.sweep_kind == CG_SWEEP_AUTO && getenv("CG_SWEEP")) o.sweep_kind = atoi(getenv("CG_SWEEP"));
    if (o.tile_steps <= 0) o.tile_steps = getenv("CG_TILE_STEPS") ? atoi(getenv("CG_TILE_STEPS")) : 64;
    if (o.tile_relabel_every == 0)
        o.tile_relabel_every = getenv("CG_TILE_RELABEL") ? atoi(getenv("CG_TILE_RELABEL")) : 16;
    if (o.sweep_kind < CG_SWEEP_AUTO || o.sweep_kind > CG_SWEEP_VERTEX) return CG_E_INVAL;
    // a3 flavour: the vertex-worklist sweep (AUTO: measured fastest) or
    // shared-memory column tiles (single slab, Z within the instantiated sizes)
    use_tiles = false;
    if (o.sweep_kind == CG_SWEEP_TILES && !multi(g)) use_tiles = tile_setup(g->slabs[0], o.tile_steps, o.tile_relabel_every);
    if (o.sweep_kind == CG_SWEEP_TILES && !use_tiles) return CG_E_INVAL;
    if (o.walk_len == 0) o.walk_len = getenv("CG_WALK") ? atoi(getenv("CG_WALK")) : 64;  // library default
    o.check_every = std::max(1, std::min(o.check_every, RING));
    if (getenv("CG_OPS")) o.ops_per_sweep = atoi(getenv("CG_OPS"));  // experiments
    o.ops_per_sweep = std::max(1, o.ops_per_sweep);
    if (!(o.gr_factor > 0.f)) o.gr_factor = 1.0f;
    for (Slab *sl : g->slabs) sl->tiles = sl->tiles && use_tiles;
    return CG_OK;
}

// a2-a5: exact global relabel, then sweeps until a global relabel finds no active vertex
// (a maximum preflow).  Shared by maxflow_solve (phase 1) and maxflow_export_flow (phase 2).
// Forward residual closure of {E > 0} as column tops (the extraction's rounds, one slab), at most
// max_passes rounds; *converged = the worklist emptied.
cg_status closure_tops(cg_graph *g, Slab *sl, int max_passes, bool *converged) {
    const Geo &geo = sl->geo;
    const int64_t ncol = (int64_t)geo.X * geo.Y;
    CG_CUDA(cudaMemsetAsync(sl->cnt + 8, 0, 3 * sizeof(unsigned), sl->stream));
    CG_CUDA(cudaMemsetAsync(sl->top - geo.Y, 0xff, sizeof(int32_t) * (ncol + 2 * geo.Y), sl->stream));
    sl->ext_k = 0;
    k_ext_seed<<<grid_for(ncol, 256, sl->num_sms * 16), 256, 0, sl->stream>>>(geo, sl->s, sl->top, sl->proc,
                                                                             sl->collist[0], sl->cnt + 8,
                                                                             sl->colstamp, ++sl->tag);
    g->st.kernel_launches++;
    *converged = false;
    const int grid = list_grid(sl, ncol);
    while (sl->ext_k < max_passes) {
        for (int b = 0; b < EXT_BATCH; b++) {
            const int r = sl->ext_k++;
            k_ext_round<<<grid, 256, 0, sl->stream>>>(geo, sl->s, sl->collist[r & 1], sl->cnt + 8 + r % 3,
                                                       sl->collist[(r + 1) & 1], sl->cnt + 8 + (r + 1) % 3,
                                                       sl->cnt + 8 + (r + 2) % 3, sl->top, sl->proc, sl->colstamp,
                                                       ++sl->tag);
        }
        g->st.kernel_launches += EXT_BATCH;
        g->st.extract_passes += EXT_BATCH;
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaMemcpyAsync(sl->h_cnt + 8, sl->cnt + 8, 5 * sizeof(unsigned), cudaMemcpyDeviceToHost, sl->stream));
        CG_CUDA(cudaStreamSynchronize(sl->stream));
        if (sl->h_cnt[8 + sl->ext_k % 3] == 0) {
            *converged = true;
            break;
        }
    }
    return CG_OK;
}

// a4 by the source side (one slab): when a batch went quiescent, the preflow is maximum iff the
// residual closure of the vertices with excess holds no vertex with a residual arc into t.  If that
// closure converges within a few rounds and reaches no such vertex, the solve ends without the
// exhaustive global relabel (and mincut_extract_surface reuses the tops); otherwise the relabel runs
// as before.  CG_SRC_TERM=0 disables it; CG_SRC_TERM=k caps the rounds (default 48).
cg_status source_side_done(cg_graph *g, bool *done) {
    *done = false;
    const int cap = getenv("CG_SRC_TERM") ? atoi(getenv("CG_SRC_TERM")) : 48;
    if (cap <= 0 || g->slabs.size() != 1 || multi(g)) return CG_OK;
    Slab *sl = g->slabs[0];
    bool conv = false;
    CG_TRY(closure_tops(g, sl, cap, &conv));
    if (!conv) return CG_OK;
    CG_CUDA(cudaMemsetAsync(sl->flags + 4, 0, sizeof(int), sl->stream));
    k_ext_check_t<<<list_grid(sl, (int64_t)sl->geo.X * sl->geo.Y), 256, 0, sl->stream>>>(sl->geo, sl->s, sl->top,
                                                                                      sl->flags + 4);
    g->st.kernel_launches++;
    CG_CUDA(cudaMemcpyAsync(sl->h_flags + 4, sl->flags + 4, sizeof(int), cudaMemcpyDeviceToHost, sl->stream));
    CG_CUDA(cudaStreamSynchronize(sl->stream));
    *done = sl->h_flags[4] == 0;
    g->top_ready = *done;
    g->st.src_terminated = *done;
    return CG_OK;
}

cg_status pr_loop(cg_graph *g, const cg_solve_opts &o, bool use_tiles, double &ms_gr) {
    const bool trace = tracing();
    Slab *s0 = g->slabs[0];
    // truncated relabels (default 65536,32 since round 2): a relabel that is not forced to be
    // exhaustive stops after trunc_levels consecutive frontiers of <= trunc_small vertices and leaves the
    // deferred deep tail at INF -- parked, i.e. inactive -- so the sweeps stop moving excess that is hundreds
    // of arcs from t while nearer excess still drains.  Truncation ends with the first quiescent batch: from
    // then on the flow still to deliver sits in that tail and a truncated relabel would park it again
    // (measured on C3).  CG_BFS_TRUNC="small,levels[,0]": 0,0 = off; a third field 0 keeps truncating.
    g->trunc_small = 65536;
    g->trunc_levels = 32;
    g->trunc_until_quiescent = true;
    if (const char *e = getenv("CG_BFS_TRUNC")) {
        unsigned a = 0, b = 0, c = 1;
        if (sscanf(e, "%u,%u,%u", &a, &b, &c) >= 2) {
            g->trunc_small = a;
            g->trunc_levels = b;
            g->trunc_until_quiescent = c != 0;
        }
    }
    cudaStream_t st0 = s0->stream;
    double last_gr_ms = 0.0;
    int64_t active = 0;
    auto timed_gr = [&](bool exhaustive) -> cg_status {
        const double a = now_ms();
        const int64_t p0 = g->st.gr_passes;
        const cg_status s = global_relabel(g, &active, exhaustive);
        last_gr_ms = now_ms() - a;
        ms_gr += last_gr_ms;
        if (trace) {
            int64_t sumT = 0;
            for (Slab *sl : g->slabs) {
                cudaMemsetAsync(sl->u64 + 2, 0, sizeof(unsigned long long), sl->stream);
                k_sum_T<<<sl->num_sms * 8, 256, 0, sl->stream>>>(sl->geo, sl->s.T, sl->u64 + 2);
                cudaMemcpyAsync(sl->h_u64 + 2, sl->u64 + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                sl->stream);
                cudaStreamSynchronize(sl->stream);
                sumT += (int64_t)sl->h_u64[2] - sl->sumT0;
            }
            gsum(g, &sumT, 1);
            fprintf(stderr, "[cg] GR#%lld levels=%lld active=%lld ms=%.3f (sweeps %lld) flow=%lld\n",
                    (long long)g->st.global_relabels, (long long)(g->st.gr_passes - p0), (long long)active, last_gr_ms,
                    (long long)g->st.sweeps, (long long)-sumT);
            if (s0->h_bst->bu_levels) fprintf(stderr, "[cg]   bottom-up levels %u\n", s0->h_bst->bu_levels);
            if (s0->h_bst->dense_levels) fprintf(stderr, "[cg]   dense levels %u\n", s0->h_bst->dense_levels);
            const unsigned *h = s0->h_bst->hist;
            fprintf(stderr, "[cg]   levels by frontier: <=32 %u <=256 %u <=2K %u <=16K %u <=128K %u <=1M %u more %u "
                    "(bottom-up %u)\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
            const unsigned long long *cy = s0->h_bst->cyc;
            fprintf(stderr, "[cg]   ms by bucket: small %.2f <=16K %.2f <=128K %.2f <=1M %.2f more %.2f bottom-up %.2f"
                    " | small-level vertices %llu\n",
                    (cy[0] + cy[1] + cy[2]) / 1.965e6, cy[3] / 1.965e6, cy[4] / 1.965e6, cy[5] / 1.965e6,
                    cy[6] / 1.965e6, cy[7] / 1.965e6, (unsigned long long)s0->h_bst->svert);
        }
        return s;
    };
    CG_TRY(timed_gr(true));
    const double gr_budget = (double)o.gr_factor * (double)g->n_global;
    const double walk_min = getenv("CG_WALK_MIN") ? atof(getenv("CG_WALK_MIN")) : 1e-3;
    // tail batches of 8 x check_every single-hop sweeps (measured C3 -5 %, C5 =)
    const int tail_mult = std::max(1, getenv("CG_TAIL_BATCH") ? atoi(getenv("CG_TAIL_BATCH")) : 8);
    const double gr_beta = getenv("CG_GR_BETA") ? atof(getenv("CG_GR_BETA")) : 1.0;
    double work_since_gr = 0.0, sweep_ms_since_gr = 0.0;
    int64_t sweeps = g->st.sweeps, since_gap = 0, last_active = active;
    std::vector<int64_t> wv(RING + 3);  // batch <= RING op counters, the overflow flag, the time trigger, relabels
    // Profiling aid (vertex loop): CG_GR_LOG=file appends the sweep counts at which this solve's
    // triggers fired; CG_GR_SCHEDULE="s1,s2,..." replays such a schedule instead of the work /
    // time triggers, so a run under ncu (whose replay-slowed kernels distort the time trigger)
    // follows the relabel schedule of an unprofiled run; once the schedule is used up the
    // work / time triggers apply again.
    std::vector<int64_t> sched, fired;
    if (const char *e = getenv("CG_GR_SCHEDULE"))
        for (const char *q = e; *q;) {
            char *end = nullptr;
            const long long v = strtoll(q, &end, 10);
            if (end == q) break;
            sched.push_back(v);
            q = *end ? end + 1 : end;
        }
    size_t sched_i = 0;
    cg_status result = CG_OK;
    while (use_tiles && active > 0) {
        // a3 on tiles: batches of checkerboard phases, no host sync inside a batch
        if (sweeps >= o.max_sweeps) { result = CG_E_NOT_CONVERGED; break; }
        const int batch = (int)std::min<int64_t>(o.check_every, o.max_sweeps - sweeps);
        Slab *sl = s0;
        const TileKernel tk = tile_kernel(sl->tS);
        CG_CUDA(cudaMemsetAsync(sl->work, 0, sizeof(unsigned long long) * 2 * batch, st0));
        CG_CUDA(cudaEventRecord(g->ev0, st0));
        for (int i = 0; i < batch; i++) {
            tk<<<sl->tgrid, sl->tg.NC * 32, sl->tsmem, st0>>>(sl->geo, sl->tg, sl->s, sl->tl, sl->tphase++,
                                                               sl->work + 2 * i, sl->visits + i, sl->flags);
            g->st.kernel_launches++;
        }
        CG_CUDA(cudaEventRecord(g->ev1, st0));
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaMemcpyAsync(sl->h_work, sl->work, sizeof(unsigned long long) * 2 * batch, cudaMemcpyDeviceToHost, st0));
        CG_CUDA(cudaMemcpyAsync(sl->h_visits, sl->visits, sizeof(unsigned long long) * batch, cudaMemcpyDeviceToHost,
                                st0));
        CG_CUDA(cudaMemcpyAsync(sl->h_cnt, sl->tl.cnt, 4 * sizeof(unsigned), cudaMemcpyDeviceToHost, st0));
        CG_CUDA(cudaMemcpyAsync(sl->h_flags, sl->flags, sizeof(int), cudaMemcpyDeviceToHost, st0));
        CG_CUDA(cudaStreamSynchronize(st0));
        if (sl->h_flags[0] & FLAG_OVERFLOW) { result = CG_E_OVERFLOW; break; }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g->ev0, g->ev1);
        g->st.ms_sweep_kernels += ms;
        sweep_ms_since_gr += ms;
        // algorithmic bytes of a tile visit: its state read and written once (2 x 32 B per
        // vertex) + the halo's height and lateral residual (8 B per halo vertex)
        const double visit_bytes = (64.0 * sl->tg.NC + 8.0 * sl->tg.NH) * (double)sl->geo.Z;
        int64_t wsum = 0;
        for (int i = 0; i < batch; i++) {
            wsum += (int64_t)sl->h_work[2 * i];
            g->st.sweep_bytes_alg += visit_bytes * (double)sl->h_visits[i];
            g->st.tile_visits += (int64_t)sl->h_visits[i];
        }
        work_since_gr += (double)wsum;
        g->st.work += wsum;
        sweeps += batch;
        g->st.sweeps = sweeps;
        const bool quiescent = sl->h_cnt[sl->tphase & 3] == 0 && sl->h_cnt[(sl->tphase + 1) & 3] == 0;
        if (trace)
            fprintf(stderr, "[cg] tile phases ..%d ops=%lld visits0=%llu next=%u/%u | %.3f ms\n", sl->tphase,
                    (long long)wsum, (unsigned long long)sl->h_visits[0], sl->h_cnt[sl->tphase & 3],
                    sl->h_cnt[(sl->tphase + 1) & 3], ms);
        if (sl->tl.prof) {
            unsigned long long pf[16];
            CG_CUDA(cudaMemcpy(pf, sl->tl.prof, sizeof(pf), cudaMemcpyDeviceToHost));
            const double v = (double)std::max(1ull, pf[PF_VISITS]);
            fprintf(stderr, "[cg]   per visit: load %.0f relabel %.0f steps %.0f store %.0f cyc | relabels %.2f lat_it %.1f "
                    "vert_it %.1f steps %.1f\n", pf[PF_LOAD] / v, pf[PF_RELABEL] / v, pf[PF_STEPS] / v,
                    pf[PF_STORE] / v, pf[PF_N_RELABEL] / v, pf[PF_LAT_IT] / std::max(1.0, (double)pf[PF_N_RELABEL]),
                    pf[PF_VERT_IT] / std::max(1.0, (double)pf[PF_LAT_IT]), pf[PF_N_STEPS] / v);
            CG_CUDA(cudaMemset(sl->tl.prof, 0, sizeof(pf)));
        }
        if (quiescent || work_since_gr >= gr_budget || sweep_ms_since_gr >= gr_beta * std::max(last_gr_ms, 0.05)) {
            CG_TRY(timed_gr(true));
            work_since_gr = 0.0;
            sweep_ms_since_gr = 0.0;
        }
    }
    double walk_sweep_ms = 0.0;  // average sweep time of the last walk batch
    const int adapt_min = getenv("CG_ADAPT_BATCH") ? atoi(getenv("CG_ADAPT_BATCH")) : 2;
    while (!use_tiles && active > 0) {
        if (sweeps >= o.max_sweeps) { result = CG_E_NOT_CONVERGED; break; }
        // multi-hop walks while many vertices are active; single hops in the sparse tail, where a
        // sweep is ~15 us of GPU time and the host round trip after every batch would otherwise
        // idle the GPU for a comparable time: tail batches are tail_mult x longer (CG_TAIL_BATCH)
        const bool walk = o.walk_len > 0 && (double)last_active >= walk_min * (double)g->n_global;
        int64_t per_batch = walk ? o.check_every : std::min<int64_t>(RING, (int64_t)o.check_every * tail_mult);
        // a walk batch ends when the cost-balance trigger is due: with sweeps of ~1 ms and relabels of
        // 2-3 ms (C4) a fixed batch of check_every = 8 sweeps overshoots the trigger by 3x; sized from the
        // previous batch's average sweep time, at least adapt_min sweeps (CG_ADAPT_BATCH).
        // One process only: the batch length sizes a collective, and this estimate is a local clock
        if (walk && adapt_min > 0 && g->nranks == 1 && walk_sweep_ms > 0.0) {
            const double due = gr_beta * std::max(last_gr_ms, 0.05) - sweep_ms_since_gr;
            per_batch = std::max<int64_t>(adapt_min, std::min<int64_t>(o.check_every, (int64_t)std::ceil(due / walk_sweep_ms)));
        }
        if (walk && sched_i < sched.size() && sched[sched_i] > sweeps)  // replayed schedule: end the batch where it fired
            per_batch = std::min<int64_t>(per_batch > 0 ? o.check_every : 1, sched[sched_i] - sweeps);
        const int batch = (int)std::min<int64_t>(per_batch, o.max_sweeps - sweeps);
        for (Slab *sl : g->slabs) {
            CG_CUDA(cudaMemsetAsync(sl->work, 0, sizeof(unsigned long long) * 2 * batch, sl->stream));
            if (walk) CG_CUDA(cudaMemsetAsync(sl->heads, 0, sizeof(unsigned) * batch, sl->stream));
        }
        CG_CUDA(cudaEventRecord(g->ev0, st0));
        for (int i = 0; i < batch; i++) {
            for (Slab *sl : g->slabs) {
                const Geo &geo = sl->geo;
                const int gridv = list_grid(sl, (geo.n + 31) / 32);
                const int64_t la = std::max<int64_t>(1, last_active / (int64_t)g->nranks);
                const int gv = std::max(sl->num_sms, std::min(gridv, grid_for(2 * la, 256, gridv)));
                const int k = sl->sweep_k++;
                sl->out_tag = ++sl->tag;
                const bool soft = geo.soft_k > 0;
                if (walk) {  // multi-hop work-fetching walks
                    (soft ? k_walk_ws<true> : k_walk_ws<false>)<<<gv, 256, 0, sl->stream>>>(
                        geo, sl->s, o.walk_len, sl->blist[k & 1], sl->cnt + k % 3, sl->blist[(k + 1) & 1],
                        sl->cnt + (k + 1) % 3, sl->cnt + (k + 2) % 3, sl->vstamp, sl->out_tag, sl->work + 2 * i,
                        sl->flags, sl->heads + i);
                }
                else
                    (soft ? k_sweep_v<true> : k_sweep_v<false>)<<<gv, 256, 0, sl->stream>>>(geo, sl->s, o.ops_per_sweep, sl->blist[k & 1],
                                                          sl->cnt + k % 3, sl->blist[(k + 1) & 1],
                                                          sl->cnt + (k + 1) % 3, sl->cnt + (k + 2) % 3, sl->vstamp,
                                                          sl->out_tag, sl->work + 2 * i, sl->flags);
                g->st.kernel_launches++;
            }
            if (multi(g)) CG_TRY(halo_sweep(g));
        }
        CG_CUDA(cudaEventRecord(g->ev1, st0));
        CG_CUDA(cudaGetLastError());
        for (Slab *sl : g->slabs) {
            CG_CUDA(cudaMemcpyAsync(sl->h_work, sl->work, sizeof(unsigned long long) * 2 * batch, cudaMemcpyDeviceToHost,
                                    sl->stream));
            CG_CUDA(cudaMemcpyAsync(sl->h_flags, sl->flags, sizeof(int), cudaMemcpyDeviceToHost, sl->stream));
        }
        int64_t overflow = 0;
        std::fill(wv.begin(), wv.begin() + batch + 3, 0);
        for (Slab *sl : g->slabs) {
            CG_CUDA(cudaStreamSynchronize(sl->stream));
            overflow |= sl->h_flags[0] & FLAG_OVERFLOW;
            for (int i = 0; i < batch; i++) {
                wv[i] += (int64_t)sl->h_work[2 * i];
                wv[batch + 2] += (int64_t)sl->h_work[2 * i + 1];
            }
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, g->ev0, g->ev1);
        g->st.ms_sweep_kernels += ms;
        sweep_ms_since_gr += ms;
        if (walk) walk_sweep_ms = ms / batch;
        wv[batch] = overflow;
        // the time-based relabel trigger is a local measurement: ranks agree on it through the
        // same allreduce as the sweep counters (one collective per batch)
        wv[batch + 1] = sweep_ms_since_gr >= gr_beta * std::max(last_gr_ms, 0.05);
        CG_TRY(gsum(g, wv.data(), batch + 3));
        if (wv[batch]) { result = CG_E_OVERFLOW; break; }
        if (trace) {
            fprintf(stderr, "[cg] sweeps %lld..%lld ops:", (long long)sweeps, (long long)(sweeps + batch - 1));
            for (int i = 0; i < batch; i += std::max(1, batch / 8)) fprintf(stderr, " %lld", (long long)wv[i]);
            fprintf(stderr, " | %.3f ms%s\n", ms, walk ? " (walk)" : "");
        }
        bool quiescent = false;
        last_active = wv[batch - 1];
        // algorithmic bytes: 32 B per vertex visit (its state read once), +12 B per
        // push (own E, target E, residual), +4 B per relabel (H)
        const int64_t rel = wv[batch + 2];
        int64_t ops = 0;
        for (int i = 0; i < batch; i++) {
            if (wv[i] == 0) { quiescent = true; break; }
            ops += wv[i];
            work_since_gr += (double)wv[i];
            g->st.work += wv[i];
        }
        g->st.relabel_ops += rel;
        g->st.sweep_bytes_alg += 32.0 * (double)ops + 12.0 * (double)(ops - rel) + 4.0 * (double)rel;
        sweeps += batch;
        since_gap += batch;
        g->st.sweeps = sweeps;
        bool trigger = quiescent || work_since_gr >= gr_budget || wv[batch + 1] > 0;
        if (sched_i < sched.size()) trigger = quiescent || sweeps >= sched[sched_i];  // then the usual triggers
        if (trigger) {
            fired.push_back(sweeps);
            while (sched_i < sched.size() && sched[sched_i] <= sweeps) sched_i++;
            // a4: termination is decided only after an exact global relabel (a quiescent batch asks
            // for an exhaustive one; a truncated one that leaves nothing active is redone exhaustively)
            bool done = false;
            if (quiescent) {
                const double a = now_ms();
                CG_TRY(source_side_done(g, &done));
                if (trace) fprintf(stderr, "[cg] source-side termination check: %s (%.3f ms)\n", done ? "max" : "no",
                                   now_ms() - a);
            }
            if (done) {
                active = 0;
                break;
            }
            if (quiescent && g->trunc_until_quiescent) g->trunc_levels = 0;
            CG_TRY(timed_gr(quiescent));
            last_active = active;
            work_since_gr = 0.0;
            sweep_ms_since_gr = 0.0;
            since_gap = 0;
        } else if (o.gap_every > 0 && since_gap >= o.gap_every) {
            CG_TRY(run_gap(g));
            since_gap = 0;
        }
    }
    if (const char *path = getenv("CG_GR_LOG")) {
        if (FILE *f = fopen(path, "a")) {
            for (size_t i = 0; i < fired.size(); i++) fprintf(f, i ? ",%lld" : "%lld", (long long)fired[i]);
            fprintf(f, "\n");
            fclose(f);
        }
    }
    return result;
}

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
    return "colgraph 0.4 sm_100a (lock-free push-relabel: multi-hop walks + single-hop sweeps over vertex worklists, "
           "device-driven frontier BFS relabel, worklist extraction, x-slab halos over NCCL)"
#ifdef CG_DEBUG_BOUNDS
           " [debug-bounds build]"
#endif
        ;
}

cg_status cg_slab_range(const cg_dims *dims, int32_t rank, int32_t nranks, int32_t *x0, int32_t *x1) {
    if (!dims || !x0 || !x1 || nranks < 1 || rank < 0 || rank >= nranks || dims->X < nranks) return CG_E_INVAL;
    const int32_t q = dims->X / nranks, r = dims->X % nranks;
    *x0 = rank * q + std::min(rank, r);
    *x1 = *x0 + q + (rank < r ? 1 : 0);
    return CG_OK;
}

cg_status cg_nccl_loopback(int32_t enable) {
    static const NcclApi lb = loopback::api();
    nccl_active() = enable ? &lb : nullptr;
    return CG_OK;
}

cg_status cg_nccl_unique_id(void *id_out) {
    if (!id_out) return CG_E_INVAL;
    if (!nccl().ok) return CG_E_NCCL;
    ncclUniqueId id;
    if (nccl().getUniqueId(&id) != ncclSuccess) return CG_E_NCCL;
    memcpy(id_out, &id, sizeof(id));
    return CG_OK;
}

void colgraph_free(cg_graph *g) {
    if (!g) return;
    {
        DeviceGuard dg(g->dist.device);
        for (Slab *sl : g->slabs) slab_free(sl);
        if (g->comm) comm_release(g->comm);
        if (g->d_red) cudaFree(g->d_red);
        if (g->d_sdesc) cudaFree(g->d_sdesc);
        if (g->d_mst) cudaFree(g->d_mst);
        if (g->h_mst) cudaFreeHost(g->h_mst);
        if (g->h_red) cudaFreeHost(g->h_red);
        if (g->ev0) cudaEventDestroy(g->ev0);
        if (g->ev1) cudaEventDestroy(g->ev1);
    }
    delete g;
}

// Common constructor: `nslabs_local` slabs in this process starting at global slab `rank`.
static cg_status build_common(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight,
                              const cg_dist *dist, int nranks, int rank, int nslabs_local, bool local,
                              cg_graph **out, const int32_t *penalty = nullptr, int32_t npenalty = 0,
                              const int32_t *dl4_in = nullptr, const int32_t *band_dev = nullptr) {
    CG_TRY(validate_dims(dims));
    // edge intervals toward +x, -x, +y, -y (NEXT-3): from dims unless given
    int32_t dl4[4];
    {
        const int32_t dy = dims->delta_y < 0 ? dims->delta : dims->delta_y;
        const int32_t def[4] = {dims->delta, dims->delta, dy, dy};
        for (int d = 0; d < 4; d++) {
            dl4[d] = dl4_in ? dl4_in[d] : def[d];
            if (dl4[d] < 0) return CG_E_INVAL;
        }
    }
    if (band_dev && input_is_weight) return CG_E_INVAL;  // bands apply to the cost rule
    // soft smoothness (NEXT-1): capacities c_0 = f(1), c_k = f(k+1) - 2 f(k) + f(k-1) >= 0
    int32_t soft_k = 0, soft_cap[SOFT_KMAX] = {0};
    if (penalty) {
        soft_k = std::max(std::max(dl4[0], dl4[1]), std::max(dl4[2], dl4[3]));
        if (npenalty < soft_k || soft_k > SOFT_KMAX) return CG_E_INVAL;
        for (int k = 0; k < soft_k; k++) {
            const int64_t f1 = penalty[k], f0 = k >= 1 ? penalty[k - 1] : 0, fm = k >= 2 ? penalty[k - 2] : 0;
            const int64_t c = k == 0 ? f1 : f1 - 2 * f0 + fm;
            if (c < 0 || c > INT_MAX) return CG_E_INVAL;
            soft_cap[k] = (int32_t)c;
        }
    }
    if (!cost_dev || !out) return CG_E_INVAL;
    *out = nullptr;
    if (nranks < 1 || nranks > dims->X) return CG_E_INVAL;
    cg_dist dd{0, 1, nullptr, 0, nullptr};
    if (dist) dd = *dist;
    DeviceGuard dg(dd.device);
    const double t0 = now_ms();
    cg_graph *g = new cg_graph();
    g->dims = *dims;
    g->dist = dd;
    g->nranks = nranks;
    g->rank = rank;
    g->local = local;
    g->n_global = (int64_t)dims->X * dims->Y * dims->Z;
    auto fail = [&](cg_status st) {
        colgraph_free(g);
        return st;
    };
    int num_sms = 148;
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dd.device);
    if (cudaEventCreate(&g->ev0) != cudaSuccess || cudaEventCreate(&g->ev1) != cudaSuccess) return fail(CG_E_CUDA);
    if (!local && nranks > 1) {
        if (!dd.nccl_id || !nccl().ok) return fail(CG_E_NCCL);
        if (comm_acquire(dd.nccl_id, rank, nranks, dd.device, &g->comm) != CG_OK) return fail(CG_E_NCCL);
        // allreduce buffers: one counter per sweep of a batch (<= RING) + the overflow flag
        if (cudaMalloc(&g->d_red, (RING + 8) * sizeof(int64_t)) != cudaSuccess ||
            cudaHostAlloc(&g->h_red, (RING + 8) * sizeof(int64_t), cudaHostAllocDefault) != cudaSuccess)
            return fail(CG_E_NOMEM);
    }
    for (int i = 0; i < nslabs_local; i++) {
        const int r = rank + i;
        int32_t x0, x1;
        if (cg_slab_range(dims, r, nranks, &x0, &x1) != CG_OK) return fail(CG_E_INVAL);
        Slab *sl = new Slab();
        sl->device = dd.device;
        sl->stream = (cudaStream_t)dd.stream;
        sl->num_sms = num_sms;
        {  // persistent BFS: as many 512-thread blocks as are co-resident (cooperative launch)
            int per_sm = 0, coop = 0;
            cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dd.device);
            if (coop && !getenv("CG_BFS_LEVEL_LAUNCHES") &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bfs_run<true>, 512, 0) == cudaSuccess && per_sm > 0)
                sl->bfs_coop_grid = num_sms * std::min(per_sm, CG_BFS_RUN_MINB);
            const void *kc = colgr_kernel(dims->Z);
            per_sm = 0;
            if (coop && kc && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kc, 512, 0) == cudaSuccess &&
                per_sm > 0)
                sl->colgr_grid = num_sms * std::min(per_sm, 2);
        }
        sl->x0 = x0;
        sl->x1 = x1;
        sl->geo = make_geo(dims, dl4, x0, x1, nranks, r > 0, r + 1 < nranks, g->n_global);
        sl->geo.soft_k = soft_k;
        for (int k = 0; k < SOFT_KMAX; k++) sl->geo.soft_cap[k] = soft_cap[k];
        g->slabs.push_back(sl);
        // LOCAL: cost_dev is the whole volume; NCCL / single: this rank's slab
        const int32_t *src = local ? cost_dev + (int64_t)x0 * sl->geo.YZ : cost_dev;
        // band: whole-volume array in LOCAL mode, this rank's slab otherwise (2 ints per column)
        const int32_t *bsrc = band_dev ? (local ? band_dev + (int64_t)x0 * dims->Y * 2 : band_dev) : nullptr;
        const cg_status s = slab_build(sl, src, input_is_weight ? 1 : 0, bsrc);
        if (s != CG_OK) return fail(s);
    }
    if (local && nslabs_local > 1) {  // all-slab BFS launch (k_bfs_run_slabs)
        int per_sm = 0, coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dd.device);
        if (coop && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bfs_run_slabs, 512, 0) == cudaSuccess &&
            per_sm > 0)
            g->mslab_grid = num_sms;
    }
    int64_t fl = 0;
    for (Slab *sl : g->slabs) fl |= sl->h_flags[0];
    g->st.source_capacity = 0;
    for (Slab *sl : g->slabs) g->st.source_capacity += sl->N;
    CG_TRY(gsum(g, &g->st.source_capacity, 1));
    g->st.bytes_per_sweep_alg = 32.0 * (double)g->n_global;
    g->st.kernel_launches = nslabs_local;
    g->st.ms_build = now_ms() - t0;
    *out = g;
    return CG_OK;
}

static cg_status colgraph_build_impl(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight, const cg_dist *dist,
                         cg_graph **out) {
    cg_dist dd{0, 1, nullptr, 0, nullptr};
    if (dist) dd = *dist;
    if (dd.nranks < 1 || dd.rank < 0 || dd.rank >= dd.nranks) return CG_E_INVAL;
    return build_common(dims, cost_dev, input_is_weight, &dd, dd.nranks, dd.rank, 1, false, out);
}

cg_status colgraph_build(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight, const cg_dist *dist,
                         cg_graph **out) {
    return debug_check(colgraph_build_impl(dims, cost_dev, input_is_weight, dist, out));
}

static cg_status colgraph_build_slabs_impl(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight, int32_t nslabs,
                               const cg_dist *dist, cg_graph **out) {
    if (nslabs < 1) return CG_E_INVAL;
    return build_common(dims, cost_dev, input_is_weight, dist, nslabs, 0, nslabs, true, out);
}

cg_status colgraph_build_slabs(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight, int32_t nslabs,
                               const cg_dist *dist, cg_graph **out) {
    return debug_check(colgraph_build_slabs_impl(dims, cost_dev, input_is_weight, nslabs, dist, out));
}

static cg_status maxflow_solve_impl(cg_graph *g, const cg_solve_opts *opts, int64_t *flow_value, cg_solve_stats *stats) {
    if (!g || !flow_value) return CG_E_INVAL;
    if (g->solved) return CG_E_STATE;
    DeviceGuard dg(g->dist.device);
    cg_solve_opts o{};
    bool use_tiles = false;
    CG_TRY(normalize_opts(g, opts, o, use_tiles));
    const bool trace = tracing();
    const double t0 = now_ms();
    Slab *s0 = g->slabs[0];
    // a1': optional exact per-column pre-cancellation (a valid initial preflow)
    const size_t pc_smem = (size_t)8 * (g->dims.Z + 1) * sizeof(long long);
    if (getenv("CG_PRECANCEL") && atoi(getenv("CG_PRECANCEL")) && pc_smem <= 200 * 1024 && !g->slabs[0]->geo.soft_k) {
        if (pc_smem > 48 * 1024)
            CG_CUDA(cudaFuncSetAttribute(k_precancel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pc_smem));
        for (Slab *sl : g->slabs) {
            k_precancel<<<grid_for((int64_t)sl->geo.X * sl->geo.Y * 32, 256, sl->num_sms * 16), 256, pc_smem,
                          sl->stream>>>(sl->geo, sl->s, sl->flags);
            g->st.kernel_launches++;
        }
        CG_CUDA(cudaGetLastError());
    }
    double ms_gr = 0.0;
    const cg_status result = pr_loop(g, o, use_tiles, ms_gr);
    if (result != CG_OK && result != CG_E_NOT_CONVERGED) return result;
    // a6: |f| = sum(T0) - sum(T)
    int64_t red[3] = {0, 0, 0};
    for (Slab *sl : g->slabs) {
        CG_CUDA(cudaMemsetAsync(sl->u64 + 2, 0, sizeof(unsigned long long), sl->stream));
        k_sum_T<<<sl->num_sms * 8, 256, 0, sl->stream>>>(sl->geo, sl->s.T, sl->u64 + 2);
        g->st.kernel_launches++;
        CG_CUDA(cudaMemcpyAsync(sl->h_u64 + 2, sl->u64 + 2, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                sl->stream));
    }
    for (Slab *sl : g->slabs) {
        CG_CUDA(cudaStreamSynchronize(sl->stream));
        red[0] += sl->sumT0;
        red[1] += (int64_t)sl->h_u64[2];
        red[2] += (int64_t)sl->h_u64[4];
    }
    CG_CUDA(cudaGetLastError());
    CG_TRY(gsum(g, red, 3));
    *flow_value = red[0] - red[1];
    g->st.gap_lifted = red[2];
    g->st.ms_global_relabel = ms_gr;
    g->st.ms_solve = now_ms() - t0;
    g->st.ms_sweeps = g->st.ms_solve - ms_gr;
    g->solved = true;
    if (stats) *stats = g->st;
    return result;
}

cg_status colgraph_build_soft(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight,
                              const int32_t *penalty, int32_t npenalty, const cg_dist *dist, cg_graph **out) {
    if (!penalty || npenalty < 1) return CG_E_INVAL;
    cg_dist dd{0, 1, nullptr, 0, nullptr};
    if (dist) dd = *dist;
    if (dd.nranks < 1 || dd.rank < 0 || dd.rank >= dd.nranks) return CG_E_INVAL;
    return debug_check(build_common(dims, cost_dev, input_is_weight, &dd, dd.nranks, dd.rank, 1, false, out, penalty,
                                    npenalty));
}

cg_status colgraph_build_slabs_soft(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight,
                                    const int32_t *penalty, int32_t npenalty, int32_t nslabs, const cg_dist *dist,
                                    cg_graph **out) {
    if (!penalty || npenalty < 1 || nslabs < 1) return CG_E_INVAL;
    return debug_check(build_common(dims, cost_dev, input_is_weight, dist, nslabs, 0, nslabs, true, out, penalty,
                                    npenalty));
}

cg_status colgraph_build_general(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight,
                                 const int32_t *dl4, const int32_t *band_dev, const int32_t *penalty, int32_t npenalty,
                                 int32_t nslabs, const cg_dist *dist, cg_graph **out) {
    if (nslabs < 0 || (penalty && npenalty < 1)) return CG_E_INVAL;
    if (nslabs >= 1)
        return debug_check(build_common(dims, cost_dev, input_is_weight, dist, nslabs, 0, nslabs, true, out, penalty,
                                        npenalty, dl4, band_dev));
    cg_dist dd{0, 1, nullptr, 0, nullptr};
    if (dist) dd = *dist;
    if (dd.nranks < 1 || dd.rank < 0 || dd.rank >= dd.nranks) return CG_E_INVAL;
    return debug_check(build_common(dims, cost_dev, input_is_weight, &dd, dd.nranks, dd.rank, 1, false, out, penalty,
                                    npenalty, dl4, band_dev));
}

cg_status maxflow_solve(cg_graph *g, const cg_solve_opts *opts, int64_t *flow_value, cg_solve_stats *stats) {
#if CG_SCAN_PROF
    {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_scanprof, z, sizeof(z));
        const cg_status st = maxflow_solve_impl(g, opts, flow_value, stats);
        cudaDeviceSynchronize();
        cudaMemcpyFromSymbol(z, g_scanprof, sizeof(z));
        fprintf(stderr, "scanprof");
        for (int i = 0; i < 16; i++) fprintf(stderr, " %llu", z[i]);
        fprintf(stderr, "\n");
        return debug_check(st);
    }
#endif
    return debug_check(maxflow_solve_impl(g, opts, flow_value, stats));
}

// NEXT-4: parallel BK with hierarchical merging (bk.cuh; §3.1).  The segment
// schedule: first-stage segments of bx x by columns, then pairwise merges alternating x and y (an
// axis stops merging once its segments span the volume) until one segment remains.
static cg_status maxflow_solve_bk_impl(cg_graph *g, const cg_bk_opts *opts, int64_t *flow_value, cg_solve_stats *stats) {
    if (!g || !flow_value) return CG_E_INVAL;
    if (g->solved) return CG_E_STATE;
    if (g->slabs.size() != 1 || multi(g) || g->slabs[0]->geo.soft_k) return CG_E_INVAL;
    const int bx = opts && opts->seg_x > 0 ? opts->seg_x : 1, by = opts && opts->seg_y > 0 ? opts->seg_y : 1;
    const int limit_ms = opts && opts->time_limit_ms > 0 ? opts->time_limit_ms : 600000;
    DeviceGuard dg(g->dist.device);
    Slab *sl = g->slabs[0];
    const Geo &geo = sl->geo;
    cudaStream_t st = sl->stream;
    const double t0 = now_ms();
    BkArrays a{sl->blist[0], sl->blist[1], sl->vstamp, sl->lab, sl->u64 + 8, sl->flags + 8, sl->flags};
    CG_CUDA(cudaMemsetAsync(a.ctr, 0, 4 * sizeof(unsigned long long), st));
    CG_CUDA(cudaMemsetAsync(sl->flags, 0, 16 * sizeof(int), st));
    k_bk_init<<<grid_for(geo.n, 256, sl->num_sms * 16), 256, 0, st>>>(geo, sl->s, a);
    g->st.kernel_launches++;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    CG_CUDA(cudaEventCreate(&e0));
    CG_CUDA(cudaEventCreate(&e1));
    bool tail_started = false;
    int sx = std::min(bx, geo.X), sy = std::min(by, geo.Y), axis = -1, half = 0;
    bool prefer_x = true;
    int64_t stages = 0;
    cg_status result = CG_OK;
    for (;;) {
        const int nsx = (geo.X + sx - 1) / sx, nsy = (geo.Y + sy - 1) / sy;
        if (nsx * nsy <= 4 && !tail_started) {
            tail_started = true;
            CG_CUDA(cudaEventRecord(e0, st));
        }
        k_bk_stage<<<nsx * nsy, 32, 0, st>>>(geo, sl->s, a, sx, sy, axis, half, (unsigned long long)limit_ms * 1000000ull);
        k_bk_time_fold<<<1, 1, 0, st>>>(a);
        g->st.kernel_launches += 2;
        stages++;
        CG_CUDA(cudaGetLastError());
        if (nsx == 1 && nsy == 1) break;
        // next merge: x and y alternate while both still have more than one segment
        const bool can_x = nsx > 1, can_y = nsy > 1;
        if (can_x && (prefer_x || !can_y)) {
            half = sx, sx *= 2, axis = 0;
        } else {
            half = sy, sy *= 2, axis = 1;
        }
        prefer_x = !prefer_x;
    }
    if (!tail_started) CG_CUDA(cudaEventRecord(e0, st));
    CG_CUDA(cudaEventRecord(e1, st));
    // a6: |f| = sum(T0) - sum(T)
    CG_CUDA(cudaMemsetAsync(sl->u64 + 2, 0, sizeof(unsigned long long), st));
    k_sum_T<<<sl->num_sms * 8, 256, 0, st>>>(geo, sl->s.T, sl->u64 + 2);
    g->st.kernel_launches++;
    CG_CUDA(cudaMemcpyAsync(sl->h_u64, sl->u64, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaMemcpyAsync(sl->h_flags, sl->flags, 16 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    float ms_tail = 0.f;
    cudaEventElapsedTime(&ms_tail, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CG_CUDA(cudaGetLastError());
    const int err = sl->h_flags[10];
    if (err & 8) result = CG_E_NOT_CONVERGED;
    else if (err) result = CG_E_CUDA;
    else if (sl->h_flags[0] & FLAG_OVERFLOW) result = CG_E_OVERFLOW;
    if (err && getenv("CG_DEBUG")) fprintf(stderr, "colgraph: maxflow_solve_bk error flags %d\n", err);
    *flow_value = sl->sumT0 - (int64_t)sl->h_u64[2];
    g->st.bk_stages = stages;
    g->st.sweeps = stages;
    g->st.bk_growths = (int64_t)sl->h_u64[8];
    g->st.work = g->st.bk_growths;
    g->st.bk_augmentations = (int64_t)sl->h_u64[9];
    g->st.bk_orphans = (int64_t)sl->h_u64[10];
    g->st.bk_freed = (int64_t)sl->h_u64[11];
    g->st.ms_bk_last_stages = ms_tail;
    g->st.ms_solve = now_ms() - t0;
    g->st.ms_sweeps = g->st.ms_solve;
    g->solved = result == CG_OK;
    if (stats) *stats = g->st;
    return result;
}

cg_status maxflow_solve_bk(cg_graph *g, const cg_bk_opts *opts, int64_t *flow_value, cg_solve_stats *stats) {
    return debug_check(maxflow_solve_bk_impl(g, opts, flow_value, stats));
}

static cg_status mincut_extract_surface_impl(cg_graph *g, int32_t *surface_dev, uint8_t *mask_dev) {
    if (!g || !surface_dev) return CG_E_INVAL;
    if (!g->solved || g->exported) return CG_E_STATE;
    DeviceGuard dg(g->dist.device);
    const double t0 = now_ms();
    for (Slab *sl : g->slabs) {
        if (g->top_ready) break;  // the solve's termination check left the tops of S
        const Geo &geo = sl->geo;
        const int64_t ncol = (int64_t)geo.X * geo.Y;
        CG_CUDA(cudaMemsetAsync(sl->cnt + 8, 0, 3 * sizeof(unsigned), sl->stream));
        CG_CUDA(cudaMemsetAsync(sl->top - geo.Y, 0xff, sizeof(int32_t) * (ncol + 2 * geo.Y), sl->stream));
        sl->ext_k = 0;
        k_ext_seed<<<grid_for(ncol, 256, sl->num_sms * 16), 256, 0, sl->stream>>>(
            geo, sl->s, sl->top, sl->proc, sl->collist[0], sl->cnt + 8, sl->colstamp, ++sl->tag);
        g->st.kernel_launches++;
    }
    for (int outer = 0; !g->top_ready; outer++) {
        if (multi(g)) {  // exchange column tops (proposals for ghosts, boundary tops)
            for (Slab *sl : g->slabs) {
                const Geo &geo = sl->geo;
                CG_CUDA(cudaMemsetAsync(sl->cnt + 12, 0, sizeof(unsigned), sl->stream));
                if (geo.gl) k_top_halo_pack<<<1, 256, 0, sl->stream>>>(geo, sl->top, 0, sl->hsend[0]);
                if (geo.gh) k_top_halo_pack<<<1, 256, 0, sl->stream>>>(geo, sl->top, 1, sl->hsend[1]);
            }
            CG_TRY(transfer(g, 2 * g->dims.Y));
            for (Slab *sl : g->slabs) {
                const Geo &geo = sl->geo;
                const int r = sl->ext_k;
                const int tag = ++sl->tag;
                for (int side = 0; side < 2; side++)
                    if (side ? geo.gh : geo.gl)
                        k_top_halo_unpack<<<grid_for(geo.Y, 256, sl->num_sms), 256, 0, sl->stream>>>(
                            geo, sl->top, side, sl->hrecv[side], sl->hsend[side], sl->collist[r & 1],
                            sl->cnt + 8 + r % 3, sl->colstamp, tag, sl->cnt + 12);
            }
        }
        // local rounds until every column list is empty
        for (;;) {
            int64_t pending = 0;
            for (Slab *sl : g->slabs) {
                const Geo &geo = sl->geo;
                const int grid = list_grid(sl, (int64_t)geo.X * geo.Y);
                for (int b = 0; b < EXT_BATCH; b++) {
                    const int r = sl->ext_k++;
                    k_ext_round<<<grid, 256, 0, sl->stream>>>(geo, sl->s, sl->collist[r & 1], sl->cnt + 8 + r % 3,
                                                               sl->collist[(r + 1) & 1], sl->cnt + 8 + (r + 1) % 3,
                                                               sl->cnt + 8 + (r + 2) % 3, sl->top, sl->proc,
                                                               sl->colstamp, ++sl->tag);
                }
                g->st.kernel_launches += EXT_BATCH;
                g->st.extract_passes += EXT_BATCH;
                CG_CUDA(cudaGetLastError());
                CG_CUDA(cudaMemcpyAsync(sl->h_cnt + 8, sl->cnt + 8, 5 * sizeof(unsigned), cudaMemcpyDeviceToHost,
                                        sl->stream));
            }
            for (Slab *sl : g->slabs) {
                CG_CUDA(cudaStreamSynchronize(sl->stream));
                pending += sl->h_cnt[8 + sl->ext_k % 3];
            }
            if (pending == 0) break;
        }
        if (!multi(g)) break;
        // another exchange is needed iff some ghost proposal or boundary top changed: run one
        // more exchange and stop when it changed nothing anywhere
        int64_t changed = 0;
        if (outer > 0)
            for (Slab *sl : g->slabs) changed += sl->h_cnt[12];
        else
            changed = 1;
        CG_TRY(gsum(g, &changed, 1));
        if (changed == 0) break;
    }
    int empty = 0;
    for (Slab *sl : g->slabs) {
        const Geo &geo = sl->geo;
        CG_CUDA(cudaMemsetAsync(sl->flags + 3, 0, sizeof(int), sl->stream));
        const int64_t soff = g->local ? (int64_t)sl->x0 * geo.Y : 0, moff = g->local ? (int64_t)sl->x0 * geo.YZ : 0;
        k_ext_out<<<sl->num_sms * 8, 256, 0, sl->stream>>>(geo, sl->top, surface_dev + soff,
                                                            mask_dev ? mask_dev + moff : nullptr, sl->flags + 3);
        g->st.kernel_launches++;
        CG_CUDA(cudaMemcpyAsync(sl->h_flags + 3, sl->flags + 3, sizeof(int), cudaMemcpyDeviceToHost, sl->stream));
    }
    for (Slab *sl : g->slabs) {
        CG_CUDA(cudaStreamSynchronize(sl->stream));
        empty |= sl->h_flags[3];
    }
    CG_CUDA(cudaGetLastError());
    int64_t e64 = empty;
    CG_TRY(gmax(g, &e64));
    g->st.ms_extract = now_ms() - t0;
    return e64 ? CG_E_EMPTY_COLUMN : CG_OK;
}

cg_status mincut_extract_surface(cg_graph *g, int32_t *surface_dev, uint8_t *mask_dev) {
    return debug_check(mincut_extract_surface_impl(g, surface_dev, mask_dev));
}

static cg_status maxflow_export_flow_impl(cg_graph *g, const int32_t *cost_dev, int32_t input_is_weight, const cg_solve_opts *opts,
                              int32_t *flow_dev) {
    if (!g || !cost_dev || !flow_dev) return CG_E_INVAL;
    if (!g->solved || g->exported) return CG_E_STATE;
    DeviceGuard dg(g->dist.device);
    cg_solve_opts o{};
    bool use_tiles = false;
    cg_solve_opts oo = opts ? *opts : cg_solve_opts{};
    oo.sweep_kind = CG_SWEEP_VERTEX;  // phase 2 runs on the vertex worklists
    CG_TRY(normalize_opts(g, &oo, o, use_tiles));
    const int ns = (int)g->slabs.size();
    // LOCAL slabs: cost_dev / flow_dev are whole-volume arrays; NCCL / single: this slab's
    const int64_t plane_stride = g->local ? g->n_global : g->slabs[0]->geo.n;
    std::vector<int32_t *> tmp(ns, nullptr);
    for (int i = 0; i < ns; i++) {
        Slab *sl = g->slabs[i];
        const Geo &geo = sl->geo;
        const int64_t ncol = (int64_t)geo.X * geo.Y;
        const int32_t *src = g->local ? cost_dev + (int64_t)sl->x0 * geo.YZ : cost_dev;
        CG_CUDA(cudaMallocAsync(&tmp[i], sizeof(int32_t) * std::max<int64_t>(1, geo.n), sl->stream));
        // phase 2 (NEXT-2): the terminal becomes s -- T(v) := flow on s->v, the phase-1 sink
        // residuals are parked in tmp.  Vertices with excess cannot reach t (maximum preflow),
        // so no flow into t changes.
        k_phase2_setup<<<grid_for(ncol * 32, 256, sl->num_sms * 16), 256, 0, sl->stream>>>(
            geo, src, input_is_weight ? 1 : 0, sl->band, sl->s, tmp[i]);
        g->st.kernel_launches++;
    }
    CG_CUDA(cudaGetLastError());
    cg_status r = CG_OK;
    const bool pr_only = getenv("CG_PHASE2_PR") != nullptr;  // the generic alternative (slow tail)
    const Geo &g0 = g->slabs[0]->geo;
    if (!pr_only) {
        // level-ordered cancellation (k_return_level): one pass per level; levels whose lateral
        // arcs stay on the level (z = 0, Delta_d = 0, k = 0 soft arcs) first net antiparallel
        // flows, then repeat until a pass sees no excess there (at most SAME_LEVEL_PASSES).
        // x-slabs: a halo exchange after every pass delivers the excess cancelled into ghost
        // vertices (and the consumed ghost residuals) before the owner reaches that level.
        constexpr int SAME_LEVEL_PASSES = 64;
        const bool flat = g0.dl[0] == 0 || g0.dl[1] == 0 || g0.dl[2] == 0 || g0.dl[3] == 0 ||
                          (g0.soft_k > 0 && g0.soft_cap[0] > 0);
        for (int z = 0; z < g0.Z && r == CG_OK; z++) {
            const bool same_level = z == 0 || flat;
            for (Slab *sl : g->slabs)
                if (same_level) {
                    k_net_level<<<grid_for((int64_t)sl->geo.X * sl->geo.Y, 256, sl->num_sms * 8), 256, 0,
                                  sl->stream>>>(sl->geo, sl->s, z);
                    g->st.kernel_launches++;
                }
            for (int it = 0; it < (same_level ? SAME_LEVEL_PASSES : 1); it++) {
                for (Slab *sl : g->slabs) {
                    if (same_level) CG_CUDA(cudaMemsetAsync(sl->cnt + 13, 0, sizeof(unsigned), sl->stream));
                    k_return_level<<<grid_for((int64_t)sl->geo.X * sl->geo.Y, 256, sl->num_sms * 8), 256, 0,
                                     sl->stream>>>(sl->geo, sl->s, z, sl->cnt + 13);
                    g->st.kernel_launches++;
                }
                if (multi(g)) CG_TRY(halo_sweep(g));
                if (!same_level) break;
                int64_t seen = 0;
                for (Slab *sl : g->slabs)
                    CG_CUDA(cudaMemcpyAsync(sl->h_cnt + 13, sl->cnt + 13, sizeof(unsigned), cudaMemcpyDeviceToHost,
                                            sl->stream));
                for (Slab *sl : g->slabs) {
                    CG_CUDA(cudaStreamSynchronize(sl->stream));
                    seen += sl->h_cnt[13];
                }
                CG_TRY(gsum(g, &seen, 1));
                if (seen == 0) break;
            }
        }
        CG_CUDA(cudaGetLastError());
    }
    {
        // whatever a capped same-level level left (cycles longer than 2) goes back to s by the
        // generic phase-2 push-relabel (exact; rarely needed)
        int64_t left = 0;
        for (Slab *sl : g->slabs) {
            CG_CUDA(cudaMemsetAsync(sl->cnt + 14, 0, sizeof(unsigned), sl->stream));
            k_count_excess<<<grid_for(sl->geo.n, 256, sl->num_sms * 8), 256, 0, sl->stream>>>(sl->geo, sl->s,
                                                                                               sl->cnt + 14);
            CG_CUDA(cudaMemcpyAsync(sl->h_cnt + 14, sl->cnt + 14, sizeof(unsigned), cudaMemcpyDeviceToHost,
                                    sl->stream));
        }
        for (Slab *sl : g->slabs) {
            CG_CUDA(cudaStreamSynchronize(sl->stream));
            left += sl->h_cnt[14];
        }
        CG_TRY(gsum(g, &left, 1));
        if (pr_only || left) {
            double ms_gr = 0.0;
            r = pr_loop(g, o, false, ms_gr);
        }
    }
    if (r == CG_OK) {
        int64_t bad = 0;
        for (int i = 0; i < ns; i++) {
            Slab *sl = g->slabs[i];
            const Geo &geo = sl->geo;
            const int64_t ncol = (int64_t)geo.X * geo.Y;
            const int32_t *src = g->local ? cost_dev + (int64_t)sl->x0 * geo.YZ : cost_dev;
            int32_t *dst = g->local ? flow_dev + (int64_t)sl->x0 * geo.YZ : flow_dev;
            CG_CUDA(cudaMemsetAsync(sl->flags + 3, 0, sizeof(int), sl->stream));
            k_flow_export<<<grid_for(ncol * 32, 256, sl->num_sms * 16), 256, 0, sl->stream>>>(
                geo, src, input_is_weight ? 1 : 0, sl->band, sl->s, tmp[i], dst, plane_stride, sl->flags + 3);
            g->st.kernel_launches++;
            CG_CUDA(cudaMemcpyAsync(sl->h_flags + 3, sl->flags + 3, sizeof(int), cudaMemcpyDeviceToHost, sl->stream));
        }
        for (Slab *sl : g->slabs) {
            CG_CUDA(cudaStreamSynchronize(sl->stream));
            bad |= sl->h_flags[3];
        }
        CG_TRY(gmax(g, &bad));
        if (bad) r = CG_E_NOT_CONVERGED;  // some vertex kept excess: not a flow
    }
    for (int i = 0; i < ns; i++) cudaFreeAsync(tmp[i], g->slabs[i]->stream);
    for (Slab *sl : g->slabs) CG_CUDA(cudaStreamSynchronize(sl->stream));
    g->exported = true;
    return r;
}

cg_status maxflow_export_flow(cg_graph *g, const int32_t *cost_dev, int32_t input_is_weight, const cg_solve_opts *opts,
                              int32_t *flow_dev) {
    return debug_check(maxflow_export_flow_impl(g, cost_dev, input_is_weight, opts, flow_dev));
}

cg_status colgraph_stats(const cg_graph *g, cg_solve_stats *stats) {
    if (!g || !stats) return CG_E_INVAL;
    *stats = g->st;
    return CG_OK;
}

cg_status colgraph_export_state(cg_graph *g, int32_t *out_dev) {
    if (!g || !out_dev) return CG_E_INVAL;
    DeviceGuard dg(g->dist.device);
    const int64_t ntot = g->local ? g->n_global : g->slabs[0]->geo.n;
    for (Slab *sl : g->slabs) {
        const int64_t off = g->local ? (int64_t)sl->x0 * sl->geo.YZ : 0;
        const Field planes[8] = {sl->s.E, sl->s.E, sl->s.T, sl->s.D, sl->s.L[0], sl->s.L[1], sl->s.L[2], sl->s.L[3]};
        const int grid = grid_for(sl->geo.n, 256, sl->num_sms * 8);
        for (int f = 0; f < 8; f++) {
            if (f == 1)
                k_export<<<grid, 256, 0, sl->stream>>>(sl->s.H, sl->geo.n, out_dev + f * ntot + off);
            else
                k_export<<<grid, 256, 0, sl->stream>>>(planes[f], sl->geo.n, out_dev + f * ntot + off);
        }
        CG_CUDA(cudaGetLastError());
    }
    for (Slab *sl : g->slabs) CG_CUDA(cudaStreamSynchronize(sl->stream));
    return CG_OK;
}

cg_status colgraph_solve_host(const cg_dims *dims, const int32_t *cost_host, int32_t input_is_weight,
                              const cg_dist *dist, const cg_solve_opts *opts, int64_t *flow_value,
                              int32_t *surface_host, uint8_t *mask_host, cg_solve_stats *stats) {
    if (!cost_host || !flow_value || !surface_host) return CG_E_INVAL;
    CG_TRY(validate_dims(dims));
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

