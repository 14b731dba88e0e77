/*
 * colgraph.h -- C ABI of the B200-native column-graph max-flow / min-cut library
 * (hot path of arXiv 2601.17026, "Parallel maxflow for proper-ordered graphs").
 *
 * The problem (§1.2, §1.3):
 *   A proper-ordered multi-column graph of X*Y columns, each of Z vertices
 *   (x, y, z), z = 0 the bottom ("base").  Vertex weights w(v) are converted to
 *   terminal arcs ("converted to the costs associated with the
 *   edges connecting the node v to the source or the sink"):
 *       w < 0 : arc s -> v of capacity -w        w > 0 : arc v -> t of capacity w
 *   Intra-column arcs (x,y,z) -> (x,y,z-1) have infinite capacity; inter-column
 *   arcs to the 4 neighbour columns realise the hard smoothness interval Delta
 *   ("edge interval").  The library computes the maximum flow value
 *   |f| (Eq. 5), the minimal minimum-cut source set (Eq. 6-7, Theorem 1
 *   L86-90) and the optimal net surface S(x,y) = max{z : (x,y,z) in S}
 *   (SPEC.md:151).
 *
 * Vertex weights from a cost volume c[x][y][z] (reading R1):
 *       w(x,y,0) = c(x,y,0) - (sum_z c(x,y,z) + 1),   w(x,y,z) = c(x,y,z) - c(x,y,z-1)
 *
 * Addressing is implicit (§3.2.3): vertex (x,y,z) has index
 * i = (x*Y + y)*Z + z (z fastest); no adjacency list is stored.
 *
 * Environment (diagnostics and measured alternatives only; defaults are the measured
 * best; results never depend on them -- the max-flow value and the minimal
 * cut are unique):
 *   CG_TRACE=1            per-batch / per-relabel trace on stderr
 *   CG_DEBUG=1            print the failing CUDA / NCCL call on stderr
 *   CG_WALK=K             hop budget of multi-hop walks (default 64)
 *   CG_WALK_MIN=f         walks while >= f*n vertices are active (default 1e-3), single hops below
 *   CG_GR_LOG=file        append the sweep counts at which the relabel triggers fired
 *   CG_GR_SCHEDULE=s1,..  replay such a schedule (profiling under ncu); afterwards the
 *                         usual triggers
 *   CG_OPS=k              push/relabel operations per vertex per single-hop sweep
 *   CG_GR_BETA=b          time trigger: relabel when sweep time since the last one >= b * its cost
 *   CG_BFS_SMALL=k        persistent BFS: frontiers <= k run in block 0 alone (default 64)
 *   CG_BFS_LEVEL_LAUNCHES one kernel launch per BFS level instead of the persistent BFS
 *   CG_SWEEP=1            tile sweeps (as sweep_kind = CG_SWEEP_TILES); CG_TILE=TXxTY,
 *                         CG_TILE_STEPS, CG_TILE_RELABEL, CG_TILE_PROF=1 (clock counters)
 *   CG_PHASE2_PR=1        maxflow_export_flow: generic push-relabel phase 2 only
 *   CG_RELABEL=bfs|colgr|levels  global relabel flavour: default one slab: BFS
 *                         over the residual-flag plane; x-slabs: in-slab flag BFS + column fixpoint
 *                         across boundaries; bfs: BFS over the records (also soft graphs, tiles);
 *                         colgr: column fixpoint from INF; levels (x-slabs): level-synchronous BFS
 *   CG_COLGR_SMALL=k      column fixpoint: worklists <= k columns run in block 0 alone
 *   CG_BFS_TRUNC=s,k[,0]  truncated relabels (default 65536,32; 0,0 = off): a flag-plane BFS relabel that
 *                         is not forced to be exhaustive stops after k consecutive frontiers of <= s
 *                         vertices; unreached vertices stay at INF (inactive) until the next exhaustive
 *                         relabel.  A quiescent batch always gets an exhaustive relabel (the one that
 *                         decides termination) and ends truncation for the rest of the solve; a third
 *                         field 0 keeps truncating after it
 *   CG_ADAPT_BATCH=m      walk batches end when the cost-balance relabel trigger is due (sized from the
 *                         previous batch's average sweep time), at least m sweeps, at most check_every
 *                         (default 2; 0 = fixed batches of check_every sweeps; single-process jobs only)
 *   CG_BAR_NS=ns          back-off cap of the persistent kernels' grid barrier (default 1024)
 *   CG_BFS_BU=div,min     flag-plane BFS: bottom-up levels when the frontier >= unvisited / div
 *                         and >= min (measured alternative; off)
 *   CG_BFS_DENSE=k        flag-plane BFS on one slab with Z % 32 == 0 (intervals < 32): levels
 *                         whose frontier has >= k vertices run as dense bit-plane shifts over
 *                         32-z words (from level 1 on, until the first smaller frontier); default
 *                         n / 256, 0 = off
 *   CG_TAIL_BATCH=k       single-hop tail: k x check_every sweeps between host reads (default 8)
 *   CG_SRC_TERM=k         a4 source-side check: closure rounds cap (default 48; 0 = always end
 *                         on an exhaustive relabel)
 *   CG_PRECANCEL=1        exact per-column pre-cancellation before the first relabel (measured
 *                         alternative; off)
 *   CG_SLAB_BFS_EACH=1    in-process x-slabs: one in-slab BFS launch per slab instead of one for all
 * Conventions for every entry point:
 *   - Errors are returned as cg_status, never thrown; no C++ exception crosses
 *     this ABI.
 *   - "_dev" pointers are CUDA device pointers on cg_dist.device; "_host"
 *     pointers are host memory (pinned or pageable).
 *   - All device work is enqueued on cg_dist.stream (NULL = legacy default
 *     stream).  Calls return after their results are defined (maxflow_solve
 *     returns with |f| on the host; mincut_extract_surface returns after its
 *     outputs are written).
 *   - One handle per thread; a handle is single-solve: build -> solve ->
 *     extract -> free.
 *   - Multi-GPU: every rank of a job calls every function collectively with
 *     its own x-slab (cg_slab_range); results are global on every rank.
 */
#ifndef COLGRAPH_H
#define COLGRAPH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cg_graph cg_graph; /* opaque, library-owned */

typedef enum {
    CG_OK = 0,
    CG_E_INVAL = 1,          /* bad dims (X,Y,Z < 1, n >= 2^31-2), Delta < 0, NULL argument,
                                nranks > X, unsupported option */
    CG_E_OVERFLOW = 2,       /* a weight or an excess would exceed INT32_MAX */
    CG_E_NOMEM = 3,          /* device allocation failed */
    CG_E_CUDA = 4,           /* a CUDA call or kernel failed */
    CG_E_NCCL = 5,           /* an NCCL call failed (multi-GPU) */
    CG_E_EMPTY_COLUMN = 6,   /* some column has no source-side vertex;
                                outputs are still written, that column's surface is -1 */
    CG_E_STATE = 7,          /* call out of order (e.g. extract before solve) */
    CG_E_NOT_CONVERGED = 8   /* max_sweeps reached before termination */
} cg_status;

/* Full-volume dimensions; Delta >= 0 is the smoothness interval
 * (Delta >= Z-1: unconstrained columns; Delta = 0: flat surface).
 *   delta   : edge interval toward the x-neighbour columns (Delta_x)
 *   delta_y : edge interval toward the y-neighbour columns (Delta_y); -1 = same as delta.
 *             Anisotropic smoothness is SURVEY.md §8(f) NEXT-3 (the paper defines the edge
 *             interval per adjacent column).  Callers must set it (-1 for the
 *             isotropic case); values < -1 are CG_E_INVAL. */
typedef struct {
    int32_t X, Y, Z, delta;
    int32_t delta_y;
} cg_dims;

/* Process / device placement.
 *   rank, nranks : this process's rank and the job size (nranks = 1: single GPU)
 *   nccl_id      : 128-byte ncclUniqueId shared by all ranks (NULL if nranks == 1)
 *   device       : CUDA device ordinal the handle lives on
 *   stream       : cudaStream_t for all work (NULL = legacy default stream) */
typedef struct {
    int32_t rank, nranks;
    const void *nccl_id;
    int32_t device;
    void *stream;
} cg_dist;

/* Solver options (NULL = defaults).
 *   gr_factor   : global relabel after gr_factor * n units of push/relabel work
 *                 (factor 1..2); default 1.0
 *   gap_every   : run the gap heuristic every gap_every sweeps
 *                 (0 = never); default 0
 *   check_every : sweeps between host reads of the active-vertex count (and relabel-trigger
 *                 checks); 1..256, default 8
 *   max_sweeps  : give up with CG_E_NOT_CONVERGED after this many sweeps; default 1<<30
 *   ops_per_sweep : push/relabel operations a vertex may perform per sweep; default 1
 *   walk_len    : > 0 selects multi-hop sweeps: a vertex's excess follows admissible arcs
 *                 for up to walk_len hops per launch; 0 = library default, -1 = single hop
 *                 (vertex-worklist sweep only)
 *   sweep_kind  : CG_SWEEP_AUTO (0, default) = CG_SWEEP_VERTEX (2): vertex worklists with
 *                 multi-hop walks; CG_SWEEP_TILES (1): shared-memory column tiles (single
 *                 slab and Z <= 256, else CG_E_INVAL).
 *                 A "sweep" of the tile kind is one checkerboard phase (one tile colour).
 *   tile_steps  : synchronous push steps per tile visit (0 = default 64)
 *   tile_relabel_every : exact local relabel at the start of a tile visit and every k push
 *                 steps (0 = default 16, < 0 = never) */
typedef struct {
    float gr_factor;
    int32_t gap_every;
    int32_t check_every;
    int64_t max_sweeps;
    int32_t ops_per_sweep;
    int32_t walk_len;
    int32_t sweep_kind;
    int32_t tile_steps;
    int32_t tile_relabel_every;
} cg_solve_opts;

enum { CG_SWEEP_AUTO = 0, CG_SWEEP_TILES = 1, CG_SWEEP_VERTEX = 2 };

typedef struct {
    int64_t sweeps;            /* push-relabel sweep launches */
    int64_t global_relabels;   /* exact global relabels (incl. initial and final) */
    int64_t gr_passes;         /* column-scan passes summed over all global relabels */
    int64_t work;              /* push/relabel operations (active vertex visits) */
    int64_t gap_runs;          /* gap heuristic invocations */
    int64_t gap_lifted;        /* vertices lifted to INF by the gap heuristic */
    int64_t extract_passes;    /* fixpoint passes of the surface extraction */
    double ms_build, ms_solve, ms_extract, ms_global_relabel, ms_sweeps;
    double bytes_per_sweep_alg; /* algorithmic bytes of a dense sweep (32 B / vertex) */
    int64_t source_capacity;   /* N = sum of source-arc capacities (int64) */
    int64_t kernel_launches;   /* library kernel launches during solve + extract */
    double ms_sweep_kernels;   /* CUDA-event time of all sweep launches (on the library stream) */
    double sweep_bytes_alg;    /* algorithmic bytes moved by all sweeps: vertex
                                  worklists 32 B per vertex visit + 12 B per push + 4 B per relabel;
                                  tiles (64 B per tile vertex + 8 B per halo vertex) per tile visit */
    int64_t tile_visits;       /* tile visits summed over all phases (tile sweeps only) */
    int64_t relabel_ops;       /* sweep operations that were relabels (vertex worklists) */
    int64_t gr_truncated;      /* global relabels that deferred a thin BFS tail (CG_BFS_TRUNC) */
    /* maxflow_solve_bk only (NEXT-4); zero after maxflow_solve */
    int64_t bk_stages;         /* merge stages run (one launch each) */
    int64_t bk_growths;        /* growth steps (an active vertex's arcs scanned once) */
    int64_t bk_augmentations;  /* augmenting paths */
    int64_t bk_orphans;        /* orphans processed by the adoption stage */
    int64_t bk_freed;          /* orphans that found no parent and became free */
    double ms_bk_last_stages;  /* CUDA-event time of the stages with <= 4 segments (the serial tail) */
    int64_t src_terminated;    /* 1: maxflow_solve ended on the source-side check (a4: the residual
                                  closure of the vertices with excess reaches no arc into t) instead
                                  of an exhaustive global relabel */
} cg_solve_stats;

/* Options of maxflow_solve_bk (NULL = defaults).
 *   seg_x, seg_y : columns per first-stage segment along x and y (0 = default 1: measured fastest,
 *                  larger first segments grow deep trees whose orphans cascade); every segment
 *                  spans all of Z (§3.1: the volume is split "along the columns and
 *                  slices", the two dominant dimensions)
 *   time_limit_ms: give up with CG_E_NOT_CONVERGED when a stage runs longer (0 = 600000) */
typedef struct {
    int32_t seg_x, seg_y;
    int32_t time_limit_ms;
} cg_bk_opts;

/* a1 -- build the int32 structure-of-arrays residual graph.
 *   cost_dev : device int32[X_r*Y*Z], this rank's x-slab [x][y][z], z fastest;
 *              costs c (input_is_weight = 0) or vertex weights w (input_is_weight = 1).
 *              Read during the call only; owned by the caller.
 *   out      : receives the library-owned handle (free with colgraph_free).
 * Excess is initialised to the saturated source arcs (Goldberg-Tarjan init,
 * PAPER.md:134), sink residuals to the sink capacities, all flows to 0.
 * Multi-GPU (cg_dist.nranks > 1): one process per GPU, each passing its own x-slab
 * (cg_slab_range) and the shared cg_dist.nccl_id; the ranks exchange one halo message
 * per x-neighbour per sweep with ncclSend/ncclRecv and agree on termination with
 * ncclAllReduce.
 * Errors: CG_E_INVAL, CG_E_OVERFLOW (a weight outside int32), CG_E_NOMEM,
 *         CG_E_CUDA, CG_E_NCCL. */
cg_status colgraph_build(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight,
                         const cg_dist *dist, cg_graph **out);

/* a8 -- the same graph cut into `nslabs` x-slabs held by THIS process (cg_slab_range
 * partition), each with its own residual state and ghost planes, exchanging exactly the
 * halo messages the NCCL ranks of colgraph_build(nranks > 1) exchange -- moved with
 * device-to-device copies instead of ncclSend/ncclRecv (§3.2.1 L254 column
 * segmentation).  Used to validate the multi-GPU algorithm on one GPU.
 *   cost_dev : device int32[X*Y*Z], the WHOLE volume; outputs of the other calls are
 *              whole-volume arrays as well.
 * Errors: as colgraph_build; CG_E_INVAL if nslabs < 1 or nslabs > X. */
cg_status colgraph_build_slabs(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight,
                               int32_t nslabs, const cg_dist *dist, cg_graph **out);

/* NEXT-1 -- soft smoothness: the VCE-weight net surface problem of PAPER.md:42-43 (edge
 * costs convex over the edge interval), SURVEY.md §8(f).  As colgraph_build (single GPU,
 * nranks = 1), plus a convex penalty f(d) on |S(p) - S(q)| = d for 4-neighbour columns
 * (|dS| <= Delta_d stays hard):
 *   penalty : HOST int32[npenalty], penalty[i] = f(i+1) (f(0) = 0); npenalty >= max(Delta_x,
 *             Delta_y) <= 16; f convex: f(k+1) - 2 f(k) + f(k-1) >= 0, f(1) >= 0.  Copied.
 * Each column pair gets finite arcs (x,y,z) -> (nbr, z-k), k < Delta_d, of capacity
 * f(k+1) - 2 f(k) + f(k-1) (f(1) for k = 0): an arc is cut for (d - k)_+ values of z, so a
 * pair costs f(d).  maxflow_solve / mincut_extract_surface then minimise
 * sum c(x,y,S) + sum_pairs f(|dS|).  With cg_dist.nranks > 1 it is the NCCL x-slab path of
 * colgraph_build (the halo message grows by 2 K planes of soft-arc flows).  Tiles
 * (CG_SWEEP_TILES) are not available for soft graphs (CG_E_INVAL).
 * Errors: as colgraph_build; CG_E_INVAL for a non-convex / too short / NULL penalty. */
cg_status colgraph_build_soft(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight,
                              const int32_t *penalty, int32_t npenalty, const cg_dist *dist, cg_graph **out);

/* colgraph_build_slabs with the soft penalty of colgraph_build_soft (in-process x-slabs). */
cg_status colgraph_build_slabs_soft(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight,
                                    const int32_t *penalty, int32_t npenalty, int32_t nslabs, const cg_dist *dist,
                                    cg_graph **out);

/* NEXT-3 -- general proper-ordered edge intervals and narrow bands; the most
 * general builder (also soft smoothness and in-process slabs).
 *   dl4      : HOST int32[4] (nullable = from dims): the edge interval toward +x, -x, +y, -y.  The
 *              lateral arc of (x,y,z) toward direction d lands at z - dl4[d], i.e. S(p) - S(q) <=
 *              dl4[d] for the neighbour q of p in direction d, so the pair (p, q = p + x) has
 *              S(q) - S(p) in [-dl4[0], dl4[1]] (and y likewise): the edge interval of PAPER.md:42
 *              per adjacent column, possibly asymmetric.  {D, D, D, D} is colgraph_build's
 *              isotropic case, {Dx, Dx, Dy, Dy} its anisotropic one.  Each >= 0.
 *   band_dev : DEVICE int32[2 * X_r * Y] (nullable): (lo, hi) per column of this rank's slab (the
 *              whole volume with nslabs >= 1), 0 <= lo < hi <= Z: the narrow band the surface of
 *              that column is confined to (PAPER.md:456, 475 -- the paper's graphs are narrow bands
 *              around landmarks; reading R15).  The base rule applies inside the band
 *              (w(lo) = c(lo) - (sum_{lo<=z<hi} c + 1), w(z) = c(z) - c(z-1)); vertices outside get
 *              no terminal arc, so the infinite down arcs keep the ones below the band in S and
 *              nothing pulls the ones above it in: S(x,y) lies in [lo, hi) when the bands move by no
 *              more than the intervals between neighbours.  Storage stays X*Y*Z (no compaction).
 *              Costs only (input_is_weight = 1 with a band: CG_E_INVAL).  Copied into the handle.
 *   penalty, npenalty : as colgraph_build_soft (NULL / 0 = hard only; npenalty >= max dl4).
 *   nslabs   : >= 1 -- in-process x-slabs as colgraph_build_slabs (cost_dev / band_dev whole-volume);
 *              0 -- one slab per process as colgraph_build (dist.nranks > 1: NCCL ranks).
 * Errors: as colgraph_build; CG_E_INVAL for a negative interval or an invalid band. */
cg_status colgraph_build_general(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight,
                                 const int32_t *dl4, const int32_t *band_dev, const int32_t *penalty, int32_t npenalty,
                                 int32_t nslabs, const cg_dist *dist, cg_graph **out);

/* Fill id_out (128 bytes) with a fresh ncclUniqueId for colgraph_build's cg_dist.nccl_id
 * (rank 0 calls it and broadcasts the bytes, e.g. with torch.distributed).
 * Errors: CG_E_INVAL (NULL), CG_E_NCCL (libnccl.so.2 not loadable). */
cg_status cg_nccl_unique_id(void *id_out);

/* TEST HOOK -- enable != 0 replaces NCCL with an in-process loopback transport
 * (csrc/nccl_loopback.h) for every later NCCL call of this process: all ranks of a job live in
 * this process on one device, one host thread per rank, each passing its own stream and a
 * cg_nccl_unique_id() obtained AFTER enabling.  The x-slab driver then runs its NCCL code path
 * (communicator cache, grouped send/recv halos, allreduce counters) unchanged, which lets a
 * one-GPU test suite execute it (§3.2.1-3.2.2: segment boundary exchange and
 * per-level synchronisation).  enable = 0 restores libnccl.  Not for production use.
 * Errors: none (CG_OK). */
cg_status cg_nccl_loopback(int32_t enable);

/* a2-a6 -- lock-free push-relabel to a maximum preflow (§2.1,
 * Alg. 2) with exact global relabels from the sink (Alg. 3,
 * §3.2.2), optional gap relabeling (L170-184) and termination decided after an
 * exact global relabel (§3.2.4).
 *   flow_value : host int64, receives |f| (Eq. 5) -- global over all ranks.
 *   stats      : nullable.
 * Errors: CG_E_STATE (already solved), CG_E_OVERFLOW, CG_E_CUDA, CG_E_NCCL,
 *         CG_E_NOT_CONVERGED. */
cg_status maxflow_solve(cg_graph *g, const cg_solve_opts *opts, int64_t *flow_value, cg_solve_stats *stats);

/* NEXT-4 -- the paper's first parallelisation, parallel Boykov-Kolmogorov with hierarchical
 * merging (§3.1; BK's growth / augmentation / adoption stages, §2.2),
 * as a second solver on the same handle: the volume is cut into segments of seg_x x seg_y columns,
 * BK exhausts the augmenting paths inside every segment in parallel (one warp per segment), then
 * adjacent segments merge pairwise (alternating x and y) and the search trees grow across the old
 * boundaries, until one segment covers the volume.  The result is a maximum FLOW whose residual
 * state the other calls read like maxflow_solve's: mincut_extract_surface gives the same minimal
 * source set and surface, maxflow_export_flow the flow on every arc.
 *   flow_value : host int64, receives |f| (Eq. 5).
 *   opts, stats: nullable.
 * One slab, hard smoothness only (general intervals and narrow bands included): handles from
 * colgraph_build_slabs*, NCCL ranks or soft penalties return CG_E_INVAL.
 * Errors: CG_E_INVAL, CG_E_STATE (already solved), CG_E_OVERFLOW (an arc flow above INT32_MAX),
 *         CG_E_NOT_CONVERGED (time_limit_ms passed), CG_E_CUDA (incl. an internal tree check). */
cg_status maxflow_solve_bk(cg_graph *g, const cg_bk_opts *opts, int64_t *flow_value, cg_solve_stats *stats);

/* a7 -- minimal min-cut source set and surface (Theorem 1).
 *   surface_dev : device int32[X_r*Y], S(x,y) = max{z : (x,y,z) in S}, -1 if none.
 *   mask_dev    : nullable device uint8[X_r*Y*Z], 1 iff the vertex is in S.
 * Errors: CG_E_STATE (not solved), CG_E_EMPTY_COLUMN (outputs still written),
 *         CG_E_CUDA, CG_E_NCCL. */
cg_status mincut_extract_surface(cg_graph *g, int32_t *surface_dev, uint8_t *mask_dev);

/* NEXT-2 -- phase 2 and flow export: turn the maximum preflow left by
 * maxflow_solve into a maximum FLOW by returning every unit of stranded excess to s (the
 * paper's Alg. 2 runs until excess returns to s; §2.1, Eq. 2-4),
 * and write the flow on every arc.  The same push-relabel runs with s as its terminal
 * (terminal residual = flow on s->v); flows into t do not change, so |f| is unchanged.
 *   cost_dev : the SAME device input and mode passed to colgraph_build (the source / sink
 *              capacities are recomputed from it; the handle does not keep them).
 *   opts     : solver options for phase 2 (nullable; sweep_kind is forced to the vertex kind).
 *   flow_dev : device int32[(7 + 4 K) * n] (K = 0, or max(Delta_x, Delta_y) for soft graphs),
 *              planes of n = X*Y*Z in index order (x*Y + y)*Z + z:
 *              [0] s->v   [1] v->t   [2] down arc v -> (x,y,z-1)
 *              [3..6] lateral arc of v in direction +x, -x, +y, -y, i.e. v -> (nbr, zo(z))
 *              with zo(0) = 0, zo(z) = z - Delta for z > Delta (reading R2)
 *              [7 + d K + k] soft graphs: the soft arc v -> (nbr_d, z - k).
 * x-slabs: with colgraph_build_slabs* the input and flow_dev are whole-volume arrays (planes of
 * n = X*Y*Z); with NCCL ranks each rank passes its own slab (planes of n = X_r*Y*Z).  Collective.
 * Call mincut_extract_surface BEFORE this (afterwards it returns CG_E_STATE: the handle then
 * holds a flow, not a preflow).
 * Errors: CG_E_INVAL (NULL), CG_E_STATE (not solved / already exported),
 *         CG_E_NOT_CONVERGED (max_sweeps hit, or excess left), CG_E_CUDA. */
cg_status maxflow_export_flow(cg_graph *g, const int32_t *cost_dev, int32_t input_is_weight, const cg_solve_opts *opts,
                              int32_t *flow_dev);

/* Convenience end-to-end call on HOST buffers (single GPU): copies cost_host to
 * the device, builds, solves, extracts and copies surface/mask back.
 *   surface_host : int32[X*Y];  mask_host : nullable uint8[X*Y*Z].
 * Same errors as the three calls above. */
cg_status colgraph_solve_host(const cg_dims *dims, const int32_t *cost_host, int32_t input_is_weight,
                              const cg_dist *dist, const cg_solve_opts *opts, int64_t *flow_value,
                              int32_t *surface_host, uint8_t *mask_host, cg_solve_stats *stats);

/* Copy the residual state (8 int32 planes of n_r each: E, H, T, D, L+x, L-x, L+y, L-y)
 * to device memory out_dev (int32[8*n_r]) -- for certificates and tests. */
cg_status colgraph_export_state(cg_graph *g, int32_t *out_dev);

/* Copy the handle's accumulated statistics (solve + extract) to *stats (host). */
cg_status colgraph_stats(const cg_graph *g, cg_solve_stats *stats);

void colgraph_free(cg_graph *g);
const char *cg_status_str(cg_status s);

/* x-slab of a rank: ceil(X/nranks) planes to the first X mod nranks ranks,
 * floor to the rest ("larger first"); [x0, x1).
 * Errors: CG_E_INVAL if nranks < 1, rank out of range or nranks > X. */
cg_status cg_slab_range(const cg_dims *dims, int32_t rank, int32_t nranks, int32_t *x0, int32_t *x1);

/* Library version string and build flags (for bench provenance). */
const char *cg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* COLGRAPH_H */
