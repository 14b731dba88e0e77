// bk.cuh -- NEXT-4: parallel Boykov-Kolmogorov with hierarchical merging.
//
// PAPER.md §3.1 (L225-228): "we extended Liu and Sun's parallel BK algorithm to 3D by first
// segmenting the structured graph into smaller segments of uniform size ... splitting across the
// two most dominant dimensions ... In the first stage of the algorithm, the source and the sink
// search trees are expanded to exhaust all the paths within the small segments.  When no further
// paths are found in the small segments, they are hierarchically merged into larger segments by
// combining adjacent segments into larger segments containing twice the number of nodes ... any
// new capacity carrying path has to include the nodes along the segment boundaries."  The BK stages
// themselves (growth, augmentation, adoption of orphans, §2.2) follow Boykov &
// Kolmogorov as the paper summarises them.
//
// B200 mapping: one warp per segment (segments are disjoint, so a warp owns every vertex and every
// arc it touches during a stage: no atomics, no locks -- "since the segments are logically separated
// and the paths are restricted to these segments, we do not use any kind of locking", L228).  A
// growth step scans the (at most 10) neighbours of the current active vertex with one lane per arc;
// an adoption scans the orphan's neighbours the same way and walks every candidate's origin in its
// own lane; augmentation walks the two tree paths serially (lane 0).  One launch per merge stage;
// segments are bx x by columns (full Z) and merge pairwise, alternating x and y, until one segment
// covers the volume.  The last stages run on few warps: the serial tail the paper measured ("capped
// at a meager 3x", L216) is inherent to the scheme and is what the measurement shows.
//
// State: the residual record of the push-relabel path (E = residual of the source arc -- the
// build pre-saturates source arcs, so the excess IS that residual --, T = residual of the sink
// arc, D / L = flows of the implicit arcs, SURVEY.md §8 notation); BK's per-vertex tree state is
// packed into the record's H field (unused by BK), so a growth step reads one sector per vertex.
#pragma once

#include "common.cuh"

namespace cg {

// H field under BK: bits 0-1 tree (0 free, 1 source tree S, 2 sink tree T), bit 2 "in the active
// list", bits 4-7 parent: an arc code (below), BK_TERM (child of its terminal), BK_ORPHAN, BK_NOPAR.
constexpr int BK_FREE = 0, BK_S = 1, BK_T = 2;
constexpr int BK_INQ = 4;
constexpr int BK_TERM = 10, BK_ORPHAN = 11, BK_NOPAR = 15;
constexpr int BK_INFCAP = INT_MAX;  // residual of an infinite arc

__device__ __forceinline__ int bk_tree(int h) { return h & 3; }
__device__ __forceinline__ int bk_par(int h) { return (h >> 4) & 15; }
__device__ __forceinline__ int bk_pack(int tree, int inq, int par) { return tree | inq | (par << 4); }
__device__ __forceinline__ int bk_with_par(int h, int par) { return (h & ~(15 << 4)) | (par << 4); }

struct BkSeg {
    int x0, x1, y0, y1;  // columns [x0, x1) x [y0, y1), all z
};

struct BkArrays {
    int *next;                // active-list links (-1 = end)
    int *onext;               // orphan-list links
    int *ts;                  // BK's TS mark: origin verified at this TIME
    int *dist;                // BK's DIST: tree distance to the terminal when ts was set
    unsigned long long *ctr;  // [0] growth scans [1] augmentations [2] orphans [3] freed orphans
    int *time;                // [0] first TIME of this stage, [1] largest TIME used so far
    int *flags;               // [0] FLAG_OVERFLOW; [10] errors: 1 TIME overflow, 2/4 a tree walk longer
                              // than the segment (a broken tree), 8 deadline passed
};

__device__ __forceinline__ void bk_xyz(const Geo &g, int64_t v, int &x, int &y, int &z) {
    const int64_t col = v / g.Z;
    z = (int)(v - col * g.Z);
    x = (int)(col / g.Y);
    y = (int)(col - (int64_t)x * g.Y);
}

// Neighbour of v through arc code k, -1 if none or outside the segment.  Codes (the GPU's minimal
// arc set, SURVEY.md §8 notation): 0 down (v-1, infinite), 1 up (v+1: residual D[v+1]), 2+d v's own
// lateral arc toward d (infinite; lands at zo(z)), 6+d the lateral arc INTO v from direction d
// (leaves (nbr_d, zi(z)); v -> that vertex is its reverse, residual L[d^1] of the tail).
__device__ __forceinline__ int64_t bk_nbr(const Geo &g, const BkSeg &sg, int64_t v, int x, int y, int z, int k) {
    if (k == 0) return z >= 1 ? v - 1 : -1;
    if (k == 1) return z + 1 < g.Z ? v + 1 : -1;
    const int d = (k - 2) & 3;
    const int nx = x + (d == 0) - (d == 1), ny = y + (d == 2) - (d == 3);
    if (nx < sg.x0 || nx >= sg.x1 || ny < sg.y0 || ny >= sg.y1) return -1;
    const int zz = k < 6 ? zo_of(z, dl_out(g, d)) : zi_of(z, dl_in(g, d), g.Z);
    if (zz < 0) return -1;
    return ((int64_t)nx * g.Y + ny) * g.Z + zz;
}
__device__ __forceinline__ int64_t bk_step(const Geo &g, int64_t v, int k) {  // along a tree arc (always present)
    int x, y, z;
    bk_xyz(g, v, x, y, z);
    const BkSeg all{0, g.X, 0, g.Y};
    return bk_nbr(g, all, v, x, y, z, k);
}
// the code of the same neighbour pair seen from the other end
__device__ __forceinline__ int bk_rev_code(int k) {
    return k == 0 ? 1 : k == 1 ? 0 : k < 6 ? 6 + ((k - 2) ^ 1) : 2 + ((k - 6) ^ 1);
}
// residual of v -> u (fwd) and u -> v (rev) for u = bk_nbr(v, k)
__device__ __forceinline__ int bk_res_fwd(const Soa &s, int64_t v, int k, int64_t u) {
    if (k == 1) return s.D[u];
    if (k >= 6) return s.L[(k - 6) ^ 1][u];
    return BK_INFCAP;
}
__device__ __forceinline__ int bk_res_rev(const Soa &s, int64_t v, int k, int64_t u) {
    if (k == 0) return s.D[v];
    if (k >= 2 && k < 6) return s.L[k - 2][v];
    return BK_INFCAP;
}
// send f units v -> u (fwd) or u -> v (!fwd): the flow of the stored arc rises or falls
__device__ __forceinline__ void bk_push(const Soa &s, int64_t v, int k, int64_t u, int f, bool fwd, int *flags) {
    int32_t *p;
    int sg;
    if (k == 0) p = &s.D[v], sg = fwd ? 1 : -1;
    else if (k == 1) p = &s.D[u], sg = fwd ? -1 : 1;
    else if (k < 6) p = &s.L[k - 2][v], sg = fwd ? 1 : -1;
    else p = &s.L[(k - 6) ^ 1][u], sg = fwd ? -1 : 1;
    const long long nv = (long long)*p + (long long)sg * f;
    if (nv > INT_MAX) atomicOr(flags, FLAG_OVERFLOW);
    *p = (int32_t)nv;
}

// a1 -> BK trees: vertices with source residual are S roots, with sink residual T roots (a vertex
// with both sends min(E, T) straight through s -> v -> t first)
__global__ void k_bk_init(Geo g, Soa s, BkArrays a) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += (int64_t)gridDim.x * blockDim.x) {
        int e = s.E[v], t = s.T[v];
        if (e > 0 && t > 0) {
            const int m = min(e, t);
            e -= m, t -= m;
            s.E[v] = e, s.T[v] = t;
        }
        s.H[v] = e > 0 ? bk_pack(BK_S, 0, BK_TERM) : t > 0 ? bk_pack(BK_T, 0, BK_TERM) : bk_pack(BK_FREE, 0, BK_NOPAR);
        a.ts[v] = 0;
        a.dist[v] = 1;
        a.next[v] = -1;
        a.onext[v] = -1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.time[0] = a.time[1] = 1;
}

__global__ void k_bk_time_fold(BkArrays a) {
    a.time[0] = a.time[1] + 1;
    if (a.time[0] > (1 << 30)) atomicOr(&a.flags[10], 1);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct BkQ {
    int head, tail;
};

// Append the vertices of the lanes in m (lane order) to a per-warp list (warp-collective).
__device__ __forceinline__ void bk_qpush(BkQ *q, unsigned m, int64_t v, int *next) {
    const int lane = lane_id();
    const bool has = (m >> lane) & 1u;
    const unsigned later = lane == 31 ? 0u : (m & (~0u << (lane + 1)));
    const int succ = later ? __ffs(later) - 1 : 0;
    const int vs = __shfl_sync(FULL, (int)v, succ);
    if (has) next[v] = later ? vs : -1;
    const int first = __shfl_sync(FULL, (int)v, __ffs(m) - 1);
    const int last = __shfl_sync(FULL, (int)v, 31 - __clz(m));
    __syncwarp();
    if (lane == 0) {
        if (q->tail >= 0) next[q->tail] = first;
        else q->head = first;
        q->tail = last;
    }
    __syncwarp();
}

// lane 0 only: j becomes an orphan (parent link saturated)
__device__ __forceinline__ void bk_orphan(const Soa &s, const BkArrays &a, BkQ *oq, int64_t j) {
    s.H[j] = bk_with_par(s.H[j], BK_ORPHAN);
    a.onext[j] = -1;
    if (oq->tail >= 0) a.onext[oq->tail] = (int)j;
    else oq->head = (int)j;
    oq->tail = (int)j;
}

// Augmentation (lane 0): the path s -> ... -> sa -> tb -> ... -> t through the bridge arc found by
// the growth of vertex i (tree X) along code k to u; saturated tree links make orphans.
__device__ bool bk_augment(const Geo &g, const Soa &s, const BkArrays &a, BkQ *oq, int64_t i, int k, int64_t u,
                           int X, int64_t wcap) {
    int64_t sa, tb;
    int f;
    int64_t steps = 0;
    if (X == BK_S) sa = i, tb = u, f = bk_res_fwd(s, i, k, u);
    else sa = u, tb = i, f = bk_res_rev(s, i, k, u);
    for (int64_t j = sa;;) {
        const int pc = bk_par(s.H[j]);
        if (pc == BK_TERM) {
            f = min(f, (int)s.E[j]);
            break;
        }
        if (++steps > wcap || pc >= BK_ORPHAN) return false;
        const int64_t q = bk_step(g, j, pc);
        f = min(f, bk_res_rev(s, j, pc, q));
        j = q;
    }
    for (int64_t j = tb;;) {
        const int pc = bk_par(s.H[j]);
        if (pc == BK_TERM) {
            f = min(f, (int)s.T[j]);
            break;
        }
        if (++steps > wcap || pc >= BK_ORPHAN) return false;
        const int64_t q = bk_step(g, j, pc);
        f = min(f, bk_res_fwd(s, j, pc, q));
        j = q;
    }
    bk_push(s, i, k, u, f, X == BK_S, a.flags);
    for (int64_t j = sa;;) {
        const int pc = bk_par(s.H[j]);
        if (pc == BK_TERM) {
            const int e = s.E[j] - f;
            s.E[j] = e;
            if (e == 0) bk_orphan(s, a, oq, j);
            break;
        }
        const int64_t q = bk_step(g, j, pc);
        bk_push(s, j, pc, q, f, false, a.flags);
        if (bk_res_rev(s, j, pc, q) == 0) bk_orphan(s, a, oq, j);
        j = q;
    }
    for (int64_t j = tb;;) {
        const int pc = bk_par(s.H[j]);
        if (pc == BK_TERM) {
            const int t = s.T[j] - f;
            s.T[j] = t;
            if (t == 0) bk_orphan(s, a, oq, j);
            break;
        }
        const int64_t q = bk_step(g, j, pc);
        bk_push(s, j, pc, q, f, true, a.flags);
        if (bk_res_fwd(s, j, pc, q) == 0) bk_orphan(s, a, oq, j);
        j = q;
    }
    return true;
}

// One merge stage: block = one warp = one segment of sx x sy columns.  axis < 0: first stage (every
// tree vertex of the segment is active); axis 0 / 1: the segment was merged from two halves split at
// x0 + half (y0 + half) -- only the tree vertices of the two columns along that line gain arcs.
__global__ void __launch_bounds__(32) k_bk_stage(Geo g, Soa s, BkArrays a, int sx, int sy, int axis, int half,
                                                      unsigned long long limit_ns) {
    __shared__ BkQ q[2];  // [0] active list, [1] orphan list
    const int lane = lane_id();
    const int nsx = (g.X + sx - 1) / sx;
    BkSeg sg;
    sg.x0 = (int)(blockIdx.x % nsx) * sx;
    sg.x1 = min(g.X, sg.x0 + sx);
    sg.y0 = (int)(blockIdx.x / nsx) * sy;
    sg.y1 = min(g.Y, sg.y0 + sy);
    if (lane == 0) q[0] = q[1] = BkQ{-1, -1};
    __syncwarp();
    int TIME = a.time[0];
    const unsigned long long deadline_ns = globaltimer_ns() + limit_ns;  // this block's time budget
    const int64_t wcap = (int64_t)(sg.x1 - sg.x0) * (sg.y1 - sg.y0) * g.Z + 1;

    // seed the active list
    {
        int cx0 = sg.x0, cx1 = sg.x1, cy0 = sg.y0, cy1 = sg.y1;
        if (axis == 0) {
            if (sg.x0 + half >= sg.x1) cx1 = cx0;  // no partner half (volume edge)
            else cx0 = sg.x0 + half - 1, cx1 = sg.x0 + half + 1;
        } else if (axis == 1) {
            if (sg.y0 + half >= sg.y1) cy1 = cy0;
            else cy0 = sg.y0 + half - 1, cy1 = sg.y0 + half + 1;
        }
        for (int x = cx0; x < cx1; x++)
            for (int y = cy0; y < cy1; y++) {
                const int64_t v0 = ((int64_t)x * g.Y + y) * g.Z;
                for (int zb = 0; zb < g.Z; zb += 32) {
                    const int z = zb + lane;
                    bool has = false;
                    if (z < g.Z) {
                        const int h = s.H[v0 + z];
                        has = bk_tree(h) != BK_FREE && !(h & BK_INQ);
                        if (has) s.H[v0 + z] = h | BK_INQ;
                    }
                    const unsigned m = __ballot_sync(FULL, has);
                    if (m) bk_qpush(&q[0], m, v0 + z, a.next);
                }
            }
    }

    unsigned long long n_grow = 0, n_aug = 0, n_orph = 0, n_free = 0;
    int64_t cur = -1;
    for (;;) {
        // the current active vertex: kept after an augmentation (it may have more paths), else the
        // next listed vertex that is still in a tree
        if (lane == 0) {
            if (cur >= 0 && bk_tree(s.H[cur]) == BK_FREE) cur = -1;
            for (int64_t pops = 0; cur < 0; pops++) {
                const int v = q[0].head;
                if (v < 0) break;
                if (pops > wcap) {  // a list longer than the segment: a bug, never a wrong answer
                    atomicOr(&a.flags[10], 16);
                    q[0].head = -1;
                    break;
                }
                q[0].head = a.next[v];
                if (q[0].head < 0) q[0].tail = -1;
                const int h = s.H[v] & ~BK_INQ;
                s.H[v] = h;
                if (bk_tree(h) != BK_FREE) cur = v;
            }
        }
        __syncwarp();
        cur = __shfl_sync(FULL, cur, 0);
        if (cur < 0) break;
        if ((++n_grow & 1023) == 0 && globaltimer_ns() > deadline_ns) {  // bounded run time (tests, hangs)
            if (lane == 0) atomicOr(&a.flags[10], 8);
            break;
        }
        // growth: one lane per arc of cur
        const int X = bk_tree(s.H[cur]);
        int x, y, z;
        bk_xyz(g, cur, x, y, z);
        int64_t u = -1;
        int cap = 0, hu = 0;
        if (lane < 10) {
            u = bk_nbr(g, sg, cur, x, y, z, lane);
            if (u >= 0) {
                cap = X == BK_S ? bk_res_fwd(s, cur, lane, u) : bk_res_rev(s, cur, lane, u);
                if (cap > 0) hu = s.H[u];
            }
        }
        const bool can = u >= 0 && cap > 0;
        const int tu = bk_tree(hu);
        bool claim = can && tu == BK_FREE;
        const unsigned peers = __match_any_sync(FULL, claim ? (int)u : -1);
        if (claim && (__ffs(peers) - 1) != lane) claim = false;  // one lane per distinct vertex
        if (claim) {
            s.H[u] = bk_pack(X, BK_INQ, bk_rev_code(lane));
            a.ts[u] = a.ts[cur];
            a.dist[u] = a.dist[cur] + 1;
        }
        // a freed vertex may still sit in the active list (its INQ bit is set): list it only once
        const unsigned mc = __ballot_sync(FULL, claim && !(hu & BK_INQ));
        if (mc) bk_qpush(&q[0], mc, u, a.next);
        const unsigned meet = __ballot_sync(FULL, can && tu != BK_FREE && tu != X);
        if (!meet) {
            cur = -1;  // no path from cur: passive
            continue;
        }
        const int k = __ffs(meet) - 1;
        const int64_t um = __shfl_sync(FULL, u, k);
        __syncwarp();
        int ok = 1;
        if (lane == 0) ok = bk_augment(g, s, a, &q[1], cur, k, um, X, wcap);
        ok = __shfl_sync(FULL, ok, 0);
        if (!ok) {  // a tree path that does not end at its terminal: a bug, never a wrong answer
            if (lane == 0) atomicOr(&a.flags[10], 4);
            break;
        }
        n_aug++;
        TIME++;
        // adoption: every orphan looks for a new parent in its own tree whose origin is a terminal
        for (;;) {
            int p = -1;
            if (lane == 0) {
                p = q[1].head;
                if (p >= 0) {
                    q[1].head = a.onext[p];
                    if (q[1].head < 0) q[1].tail = -1;
                }
            }
            __syncwarp();
            p = __shfl_sync(FULL, p, 0);
            if (p < 0) break;
            if ((++n_orph & 1023) == 0 && globaltimer_ns() > deadline_ns) {
                if (lane == 0) atomicOr(&a.flags[10], 8);
                cur = -2;
                break;
            }
            const int hp = s.H[p], Xp = bk_tree(hp);
            bk_xyz(g, p, x, y, z);
            int64_t w = -1;
            int hw = 0, capa = 0;
            if (lane < 10) {
                w = bk_nbr(g, sg, p, x, y, z, lane);
                if (w >= 0) {
                    hw = s.H[w];
                    if (bk_tree(hw) == Xp) capa = Xp == BK_S ? bk_res_rev(s, p, lane, w) : bk_res_fwd(s, p, lane, w);
                }
            }
            int dd = INT_MAX;
            if (capa > 0 && bk_par(hw) != BK_ORPHAN) {  // origin check: walk to the terminal
                int64_t j = w;
                for (int steps = 0;;) {
                    if (a.ts[j] == TIME) {
                        dd = steps + a.dist[j];
                        break;
                    }
                    const int pj = bk_par(s.H[j]);
                    steps++;
                    if (pj == BK_TERM) {
                        dd = steps;
                        break;
                    }
                    if (pj >= BK_ORPHAN) break;
                    if (steps > wcap) {
                        atomicOr(&a.flags[10], 2);
                        break;
                    }
                    j = bk_step(g, j, pj);
                }
            }
            int best = dd;
#pragma unroll
            for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(FULL, best, o));
            if (best != INT_MAX) {
                const int win = __ffs(__ballot_sync(FULL, dd == best)) - 1;
                if (lane == win) {
                    s.H[p] = bk_with_par(hp, win);
                    a.ts[p] = TIME;
                    a.dist[p] = best + 1;
                    a.ts[w] = TIME;
                    a.dist[w] = best;
                }
                __syncwarp();
                continue;
            }
            // no valid parent: p becomes free; same-tree neighbours with residual toward p become
            // active, its children orphans
            n_free++;
            const bool same = lane < 10 && w >= 0 && bk_tree(hw) == Xp;
            const bool act = same && capa > 0 && !(hw & BK_INQ);
            const bool orp = same && bk_par(hw) == bk_rev_code(lane);
            const unsigned grp = __match_any_sync(FULL, same ? (int)w : -1);
            const unsigned mact = __ballot_sync(FULL, act), morp = __ballot_sync(FULL, orp);
            const bool lead = same && (__ffs(grp) - 1) == lane;
            const bool gact = lead && (mact & grp), gorp = lead && (morp & grp);
            if (gact || gorp) {
                int h = hw;
                if (gact) h |= BK_INQ;
                if (gorp) h = bk_with_par(h, BK_ORPHAN);
                s.H[w] = h;
            }
            const unsigned ma = __ballot_sync(FULL, gact);
            if (ma) bk_qpush(&q[0], ma, w, a.next);
            const unsigned mo = __ballot_sync(FULL, gorp);
            if (mo) bk_qpush(&q[1], mo, w, a.onext);
            if (lane == 0) s.H[p] = bk_pack(BK_FREE, hp & BK_INQ, BK_NOPAR);
            __syncwarp();
        }
        if (cur == -2) break;
    }
    if (lane == 0) {
        atomicAdd(&a.ctr[0], n_grow);
        atomicAdd(&a.ctr[1], n_aug);
        atomicAdd(&a.ctr[2], n_orph);
        atomicAdd(&a.ctr[3], n_free);
        atomicMax(&a.time[1], TIME);
    }
}

}  // namespace cg
