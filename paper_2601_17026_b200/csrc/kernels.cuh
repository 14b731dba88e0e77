// kernels.cuh -- the sm_100a kernels of the column-graph max-flow hot path.
//
//   a1 build            k_build               PAPER.md §1.2; §2.1 L134 (init)
//   a2/a5 global relabel k_bfs_init/k_bfs_level PAPER.md §2.1; Alg. 3; §3.2.2
//   a3 sweep            k_sweep               PAPER.md §2.1; Alg. 2
//   a4 termination      k_rebuild_chunks (+ host loop)  PAPER.md §3.2.4; Alg. 1
//   a5 gap              k_gap_*               PAPER.md §2.1
//   a6 flow value       k_sum_T               PAPER.md Eq. 5
//   a7 extraction       k_ext_*               PAPER.md Theorem 1
#pragma once

#include "common.cuh"

namespace cg {

// ------------------------------------------------------------------ a1: build
// One warp per column: w(0) = c(0) - (sum_z c + 1), w(z) = c(z) - c(z-1) (R1).
// E = max(0,-w): source arcs pre-saturated (Goldberg-Tarjan init);
// T = max(0, w): sink-arc residual.  Totals N = sum E and sum T0 in int64.
__global__ void k_build(Geo g, const int32_t *__restrict__ in, int weight_mode, Soa s,
                        unsigned long long *sums /* [0]=N [1]=sum T0 */, int *flags) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    long long accN = 0, accT = 0;
    bool bad = false;
    for (int64_t col = gwarp(); col < ncol; col += nwarps()) {
        const int32_t *cc = in + col * g.Z;
        long long colsum = 0;
        if (!weight_mode) {
            for (int z = lane_id(); z < g.Z; z += 32) colsum += cc[z];
            colsum = warp_sum_ll(colsum);
        }
        for (int z = lane_id(); z < g.Z; z += 32) {
            long long w;
            if (weight_mode) w = cc[z];
            else w = z == 0 ? (long long)cc[0] - (colsum + 1) : (long long)cc[z] - (long long)cc[z - 1];
            const bool ok = w <= INT_MAX && w >= -(long long)INT_MAX;
            bad |= !ok;
            const int32_t e = (ok && w < 0) ? (int32_t)(-w) : 0, t = (ok && w > 0) ? (int32_t)w : 0;
            s.E[col * g.Z + z] = e;
            s.T[col * g.Z + z] = t;
            accN += e;
            accT += t;
        }
    }
    accN = warp_sum_ll(accN);
    accT = warp_sum_ll(accT);
    if (lane_id() == 0) {
        if (accN) atomicAdd(&sums[0], (unsigned long long)accN);
        if (accT) atomicAdd(&sums[1], (unsigned long long)accT);
    }
    if (bad) atomicOr(flags, FLAG_OVERFLOW);
}

__global__ void k_fill(int32_t *p, int64_t n, int32_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// ------------------------------------------------------------------ a3: push-relabel sweep
// One warp per listed chunk (32 consecutive z of a column; all state loads coalesced).
// Each active lane (E > 0, H < INF) performs up to `ops` operations of Alg. 2:
//   scan the residual out-arcs in the fixed order t, down, lateral-out(+x,-x,+y,-y),
//   up, lateral-in-reverse(+x,-x,+y,-y); h_min = lowest neighbour height (first wins);
//   relabel H = h_min + 1 if H <= h_min ("newd = min label(w)+1 ... only if newd >
//   label(v)"); push delta = min(E, r) along that arc (r = INF on infinite arcs).
// Lock-free: every residual has one decrementer, so each
// stale read is a lower bound of what the reader may subtract.
// Worklist: chunks that received a push or still hold active excess are appended to
// the next list (de-duplicated by stamp == tag).
struct OpCtx {
    int64_t v, v0, col;
    int z, zo, zi;
    int64_t off[4];  // vertex offset of the neighbour column (0 = none)
    int coff[4];     // column-index offset of the neighbour column
};

// One push/relabel operation; returns the chunk id that received flow (or -1).
__device__ __forceinline__ int pr_op(const Geo &g, const Soa &s, const OpCtx &c, int &e, int &h, int &sent,
                                     int *flags) {
    int best = g.INF, arc = -1, res = 0, tz = 0, tco = 0;
    int64_t tgt = -1;
    const int tres = s.T[c.v];
    if (tres > 0) {
        best = 0;
        arc = 0;
    } else {
        if (c.z >= 1) {
            const int hh = s.H[c.v - 1];
            if (hh < best) { best = hh; arc = 1; tgt = c.v - 1; tz = c.z - 1; tco = 0; }
        }
        if (c.zo >= 0) {
#pragma unroll
            for (int d = 0; d < 4; d++) {
                if (!c.off[d]) continue;
                const int64_t t = c.v0 + c.off[d] + c.zo;
                const int hh = s.H[t];
                if (hh < best) { best = hh; arc = 2 + d; tgt = t; tz = c.zo; tco = c.coff[d]; }
            }
        }
        if (c.z + 1 < g.Z) {
            const int r = s.D[c.v + 1];
            if (r > 0) {
                const int hh = s.H[c.v + 1];
                if (hh < best) { best = hh; arc = 6; tgt = c.v + 1; res = r; tz = c.z + 1; tco = 0; }
            }
        }
        if (c.zi >= 0) {
#pragma unroll
            for (int d = 0; d < 4; d++) {
                if (!c.off[d]) continue;
                const int64_t u = c.v0 + c.off[d] + c.zi;
                const int r = s.L[(int64_t)(d ^ 1) * g.n + u];
                if (r > 0) {
                    const int hh = s.H[u];
                    if (hh < best) { best = hh; arc = 7 + d; tgt = u; res = r; tz = c.zi; tco = c.coff[d]; }
                }
            }
        }
    }
    if (best >= g.INF) {  // no residual path known: dead until the next global relabel
        h = g.INF;
        s.H[c.v] = h;
        return -1;
    }
    if (h <= best) {  // relabel (Alg. 2 Relabel)
        h = best + 1;
        s.H[c.v] = h;
        if (h >= g.INF) return -1;
    }
    int df;  // push (Alg. 2 Push)
    switch (arc) {
        case 0:
            df = min(e, tres);
            s.T[c.v] = tres - df;
            break;
        case 1:
            df = e;
            atomicAdd(&s.D[c.v], df);
            break;
        case 2: case 3: case 4: case 5:
            df = e;
            atomicAdd(&s.L[(int64_t)(arc - 2) * g.n + c.v], df);
            break;
        case 6:
            df = min(e, res);
            atomicSub(&s.D[c.v + 1], df);
            break;
        default:
            df = min(e, res);
            atomicSub(&s.L[(int64_t)((arc - 7) ^ 1) * g.n + tgt], df);
            break;
    }
    e -= df;
    sent += df;
    if (tgt < 0) return -1;
    const int old = atomicAdd(&s.E[tgt], df);
    if (old > INT_MAX - df) atomicOr(flags, FLAG_OVERFLOW);
    return (int)((c.col + tco) * g.CPC + (tz >> 5));
}

__global__ void __launch_bounds__(256) k_sweep(Geo g, Soa s, int ops, const int *__restrict__ lin,
                                               const unsigned *cin, int *lout, unsigned *cout, unsigned *czero,
                                               int *stamp, int tag, unsigned long long *work, int *flags) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *czero = 0;
    const int64_t count = *cin;
    unsigned long long mywork = 0;
    for (int64_t i = gwarp(); i < count; i += nwarps()) {
        const int chunk = lin[i];
        OpCtx c;
        c.col = chunk / g.CPC;
        c.z = (int)(chunk - c.col * g.CPC) * 32 + lane_id();
        const bool valid = c.z < g.Z;
        c.v0 = c.col * g.Z;
        c.v = c.v0 + c.z;
        int e = valid ? s.E[c.v] : 0;
        int h = valid ? s.H[c.v] : g.INF;
        bool act = e > 0 && h < g.INF;
        const unsigned am = __ballot_sync(FULL, act);
        if (!am) continue;
        mywork += __popc(am);
        const int x = (int)(c.col / g.Y), y = (int)(c.col - (int64_t)x * g.Y);
        c.zo = zo_of(c.z, g.delta);
        c.zi = zi_of(c.z, g.delta, g.Z);
#pragma unroll
        for (int d = 0; d < 4; d++) c.off[d] = nbr_off(g, x, y, d);
        c.coff[0] = g.Y; c.coff[1] = -g.Y; c.coff[2] = 1; c.coff[3] = -1;
        int sent = 0;
        for (int it = 0; it < ops; ++it) {
            int tchunk = -1;
            if (act) {
                tchunk = pr_op(g, s, c, e, h, sent, flags);
                act = e > 0 && h < g.INF;
            }
            warp_mark(tchunk, stamp, tag, lout, cout);
            if (!__any_sync(FULL, act)) break;
        }
        if (sent) atomicSub(&s.E[c.v], sent);
        warp_mark(__any_sync(FULL, act) ? chunk : -1, stamp, tag, lout, cout);
    }
    if (lane_id() == 0 && mywork) atomicAdd(work, mywork);
}

// Vertex-granular worklist variant (default): one thread per listed vertex.  Sparse
// activity (1-2% of the vertices, scattered) would leave 31 of 32 lanes idle in the
// chunk variant; here every lane carries an active vertex.
__device__ __forceinline__ void mark_vertex(int64_t id, int *vstamp, int tag, int *list, unsigned *count) {
    bool add = id >= 0 && vstamp[id] != tag;
    if (add) add = atomicExch(&vstamp[id], tag) != tag;
    warp_append(add, (int)id, list, count);
}

struct ArcPick {
    int best, arc, res;
    int64_t tgt;
};

// Arc scan in the fixed order t, down, lateral-out(+x,-x,+y,-y), up, lateral-in-reverse.
// Returns the FIRST admissible arc (neighbour label < hx: Alg. 2 pushes on any admissible
// arc, and with exact labels every admissible neighbour sits at hx-1); if none is
// admissible, the lowest residual neighbour (for the relabel "newd = min label(w)+1").
// Early exit saves most of the scattered loads in the common case.
__device__ __forceinline__ ArcPick scan_arcs(const Geo &g, const Soa &s, const OpCtx &c, int hx) {
    ArcPick p{g.INF, -1, 0, -1};
    const int tres = s.T[c.v];
    if (tres > 0) {
        p.best = 0; p.arc = 0; p.res = tres;
        return p;
    }
    if (c.z >= 1) {
        const int hh = s.H[c.v - 1];
        if (hh < p.best) { p.best = hh; p.arc = 1; p.tgt = c.v - 1; }
        if (p.best < hx) return p;
    }
    if (c.zo >= 0) {
#pragma unroll
        for (int d = 0; d < 4; d++) {
            if (!c.off[d]) continue;
            const int64_t t = c.v0 + c.off[d] + c.zo;
            const int hh = s.H[t];
            if (hh < p.best) { p.best = hh; p.arc = 2 + d; p.tgt = t; }
            if (p.best < hx) return p;
        }
    }
    if (c.z + 1 < g.Z) {
        const int r = s.D[c.v + 1];
        if (r > 0) {
            const int hh = s.H[c.v + 1];
            if (hh < p.best) { p.best = hh; p.arc = 6; p.tgt = c.v + 1; p.res = r; }
            if (p.best < hx) return p;
        }
    }
    if (c.zi >= 0) {
#pragma unroll
        for (int d = 0; d < 4; d++) {
            if (!c.off[d]) continue;
            const int64_t u = c.v0 + c.off[d] + c.zi;
            const int r = s.L[(int64_t)(d ^ 1) * g.n + u];
            if (r > 0) {
                const int hh = s.H[u];
                if (hh < p.best) { p.best = hh; p.arc = 7 + d; p.tgt = u; p.res = r; }
                if (p.best < hx) return p;
            }
        }
    }
    return p;
}

__device__ __forceinline__ int64_t pr_op_v(const Geo &g, const Soa &s, const OpCtx &c, int &e, int &h, int &sent,
                                           int *flags) {
    const ArcPick p = scan_arcs(g, s, c, h);
    const int best = p.best, arc = p.arc, res = p.res, tres = p.res;
    const int64_t tgt = p.tgt;
    if (best >= g.INF) {
        h = g.INF;
        s.H[c.v] = h;
        return -1;
    }
    if (h <= best) {
        h = best + 1;
        s.H[c.v] = h;
        if (h >= g.INF) return -1;
    }
    int df;
    switch (arc) {
        case 0:
            df = min(e, tres);
            s.T[c.v] = tres - df;
            break;
        case 1:
            df = e;
            atomicAdd(&s.D[c.v], df);
            break;
        case 2: case 3: case 4: case 5:
            df = e;
            atomicAdd(&s.L[(int64_t)(arc - 2) * g.n + c.v], df);
            break;
        case 6:
            df = min(e, res);
            atomicSub(&s.D[c.v + 1], df);
            break;
        default:
            df = min(e, res);
            atomicSub(&s.L[(int64_t)((arc - 7) ^ 1) * g.n + tgt], df);
            break;
    }
    e -= df;
    sent += df;
    if (tgt < 0) return -1;
    const int old = atomicAdd(&s.E[tgt], df);
    if (old > INT_MAX - df) atomicOr(flags, FLAG_OVERFLOW);
    return tgt;
}

__global__ void __launch_bounds__(256) k_sweep_v(Geo g, Soa s, int ops, const int *__restrict__ lin,
                                                 const unsigned *cin, int *lout, unsigned *cout, unsigned *czero,
                                                 int *vstamp, int tag, unsigned long long *work, int *flags) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *czero = 0;
    const int64_t count = *cin;
    unsigned long long mywork = 0;
    for (int64_t base = gwarp() * 32; base < count; base += nwarps() * 32) {
        const int64_t i = base + lane_id();
        OpCtx c;
        c.v = i < count ? lin[i] : -1;
        int e = 0, h = g.INF;
        if (c.v >= 0) {
            e = s.E[c.v];
            h = s.H[c.v];
        }
        bool act = e > 0 && h < g.INF;
        if (!__any_sync(FULL, act)) continue;
        int sent = 0;
        if (act) {
            mywork++;
            c.col = c.v / g.Z;
            c.z = (int)(c.v - c.col * g.Z);
            c.v0 = c.col * g.Z;
            const int x = (int)(c.col / g.Y), y = (int)(c.col - (int64_t)x * g.Y);
            c.zo = zo_of(c.z, g.delta);
            c.zi = zi_of(c.z, g.delta, g.Z);
#pragma unroll
            for (int d = 0; d < 4; d++) c.off[d] = nbr_off(g, x, y, d);
        }
        for (int it = 0; it < ops; ++it) {
            int64_t tgt = -1;
            if (act) {
                tgt = pr_op_v(g, s, c, e, h, sent, flags);
                act = e > 0 && h < g.INF;
            }
            mark_vertex(tgt, vstamp, tag, lout, cout);
            if (!__any_sync(FULL, act)) break;
        }
        if (sent) atomicSub(&s.E[c.v], sent);
        mark_vertex(act ? c.v : -1, vstamp, tag, lout, cout);
    }
    mywork = warp_sum_ll((long long)mywork);
    if (lane_id() == 0 && mywork) atomicAdd(work, mywork);
}

// ------------------------------------------------------------------ a3': multi-hop sweep ("walk")
// Alg. 2's discharge applied along a path: the owner of an active vertex v takes all
// of E(v) and carries it down admissible arcs (strictly decreasing labels) for up to K
// hops, pushing delta = min(carry, r) on each arc.  Finite residuals (T, up, lateral-in
// reverse) may now be decremented by several walkers, so they are RESERVED with a CAS
// loop (never negative); infinite arcs only increase the reverse flow (atomicAdd).  A
// carry that cannot go further is deposited (atomicAdd) on the vertex where it stops,
// which is listed for the next launch; a stuck vertex is relabelled monotonically
// (atomicMax, labels never decrease between global relabels).  Excess is decremented
// only by its owner (the walk start), so conservation is exact.
__device__ __forceinline__ void set_ctx(const Geo &g, OpCtx &c, int64_t v) {
    c.v = v;
    c.col = v / g.Z;
    c.z = (int)(v - c.col * g.Z);
    c.v0 = c.col * g.Z;
    const int x = (int)(c.col / g.Y), y = (int)(c.col - (int64_t)x * g.Y);
    c.zo = zo_of(c.z, g.delta);
    c.zi = zi_of(c.z, g.delta, g.Z);
#pragma unroll
    for (int d = 0; d < 4; d++) c.off[d] = nbr_off(g, x, y, d);
}

// take up to `want` from a residual that several threads may decrement
__device__ __forceinline__ int reserve(int32_t *p, int want) {
    int cur = *(volatile int32_t *)p;
    while (cur > 0) {
        const int take = min(cur, want);
        const int old = atomicCAS(p, cur, cur - take);
        if (old == cur) return take;
        cur = old;
    }
    return 0;
}

struct BlockQueue {  // block-local append buffer, flushed with one global atomic per block
    static constexpr int CAP = 2048;
    int buf[CAP];
    unsigned n;
};

__device__ __forceinline__ void deposit(const Geo &g, const Soa &s, int64_t x, int c, int *vstamp, int tag,
                                        BlockQueue &q, int *lout, unsigned *cout, int *flags) {
    const int old = atomicAdd(&s.E[x], c);
    if (old > INT_MAX - c) atomicOr(flags, FLAG_OVERFLOW);
    if (vstamp[x] != tag && atomicExch(&vstamp[x], tag) != tag) {
        const unsigned pos = atomicAdd(&q.n, 1u);
        if (pos < BlockQueue::CAP) q.buf[pos] = (int)x;
        else lout[atomicAdd(cout, 1u)] = (int)x;
    }
}

__global__ void __launch_bounds__(256) k_walk(Geo g, Soa s, int K, const int *__restrict__ lin, const unsigned *cin,
                                              int *lout, unsigned *cout, unsigned *czero, int *vstamp, int tag,
                                              unsigned long long *work, int *flags) {
    __shared__ BlockQueue q;
    __shared__ unsigned qbase;
    if (threadIdx.x == 0) q.n = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *czero = 0;
    __syncthreads();
    const int64_t count = *cin;
    unsigned long long mywork = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = lin[i];
        int c = s.E[v];
        int hx = s.H[v];
        if (!(c > 0 && hx < g.INF)) continue;
        atomicSub(&s.E[v], c);  // the owner takes its whole excess
        OpCtx ctx;
        set_ctx(g, ctx, v);
        for (int step = 0; c > 0; ++step) {
            const ArcPick p = scan_arcs(g, s, ctx, hx);
            mywork++;  // one push or relabel operation per hop
            if (p.best >= hx || step >= K) {  // stuck (or hop budget spent): deposit the carry here
                if (p.best >= hx) atomicMax(&s.H[ctx.v], p.best >= g.INF ? g.INF : p.best + 1);
                deposit(g, s, ctx.v, c, vstamp, tag, q, lout, cout, flags);
                break;
            }
            int df;
            switch (p.arc) {
                case 0: df = reserve(&s.T[ctx.v], c); break;
                case 1: df = c; atomicAdd(&s.D[ctx.v], df); break;
                case 2: case 3: case 4: case 5:
                    df = c;
                    atomicAdd(&s.L[(int64_t)(p.arc - 2) * g.n + ctx.v], df);
                    break;
                case 6: df = reserve(&s.D[ctx.v + 1], c); break;
                default: df = reserve(&s.L[(int64_t)((p.arc - 7) ^ 1) * g.n + p.tgt], c); break;
            }
            if (df == 0) continue;  // lost a reservation race: rescan this vertex
            if (p.arc == 0) {       // absorbed by t
                c -= df;
                continue;
            }
            if (df < c) deposit(g, s, ctx.v, c - df, vstamp, tag, q, lout, cout, flags);
            c = df;
            hx = p.best;
            set_ctx(g, ctx, p.tgt);
        }
    }
    __syncthreads();
    const unsigned nq = min(q.n, (unsigned)BlockQueue::CAP);
    if (threadIdx.x == 0 && nq) qbase = atomicAdd(cout, nq);
    __syncthreads();
    for (unsigned j = threadIdx.x; j < nq; j += blockDim.x) lout[qbase + j] = q.buf[j];
    mywork = warp_sum_ll((long long)mywork);
    if (lane_id() == 0 && mywork) atomicAdd(work, mywork);
}

// After an exact global relabel: list every active vertex (E > 0, H < INF) in index order.
__global__ void k_rebuild_vertices(Geo g, const Soa s, int *lout, unsigned *cout, int *vstamp, int tag,
                                   unsigned long long *active) {
    unsigned long long myact = 0;
    for (int64_t base = gwarp() * 32; base < g.n; base += nwarps() * 32) {
        const int64_t v = base + lane_id();
        bool a = false;
        if (v < g.n) a = s.E[v] > 0 && s.H[v] < g.INF;
        if (a) vstamp[v] = tag;
        myact += a;
        warp_append(a, (int)v, lout, cout);
    }
    myact = warp_sum_ll((long long)myact);
    if (lane_id() == 0 && myact) atomicAdd(active, myact);
}

// ------------------------------------------------------------------ a2/a5: exact global relabel
// H(v) = BFS distance from v to t in the residual graph (Alg. 3: level 1 = vertices
// with a residual arc into t -- the "{v,s}" of L414 read as t, R6 -- then
// level L+1 = unlabelled residual predecessors of level L).  Level-synchronous,
// frontier-based: each vertex is claimed exactly once by atomicCAS(H, INF, L+1).
// Residual in-arcs u -> v of v = (x,y,z):
//   u = (x,y,z+1)             down arc, infinite
//   u = (x,y,z-1)             up arc, residual D(v)
//   u = (nbr, zi(z))          lateral arc of u into v, infinite
//   u = (nbr_d, zo(z))        reverse of v's lateral arc in direction d, residual L_d(v)
__global__ void k_bfs_init(Geo g, Soa s, int *lout, unsigned *cout) {
    for (int64_t base = gwarp() * 32; base < g.n; base += nwarps() * 32) {
        const int64_t v = base + lane_id();
        bool seed = false;
        if (v < g.n) {
            seed = s.T[v] > 0;
            s.H[v] = seed ? 1 : g.INF;
        }
        warp_append(seed, (int)v, lout, cout);
    }
}

// Expand one frontier vertex per lane (v < 0: none): claim every unlabelled residual
// predecessor with label nl and append the claims with one atomic per warp.
__device__ __forceinline__ void bfs_expand_warp(const Geo &g, const Soa &s, int nl, int64_t v, int *lout,
                                                unsigned *cout) {
    const int INF = g.INF;
    int u[10];
    unsigned got = 0;
    if (v >= 0) {
        const int64_t col = v / g.Z;
        const int z = (int)(v - col * g.Z);
        const int x = (int)(col / g.Y), y = (int)(col - (int64_t)x * g.Y);
        const int64_t v0 = col * g.Z;
        const int zo = zo_of(z, g.delta), zi = zi_of(z, g.delta, g.Z);
        auto claim = [&](int slot, int64_t w) {
            if (s.H[w] >= INF && atomicCAS(&s.H[w], INF, nl) == INF) {
                u[slot] = (int)w;
                got |= 1u << slot;
            }
        };
        if (z + 1 < g.Z) claim(0, v + 1);
        if (z >= 1 && s.D[v] > 0) claim(1, v - 1);
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const int64_t o = nbr_off(g, x, y, d);
            if (!o) continue;
            if (zi >= 0) claim(2 + d, v0 + o + zi);
            if (zo >= 0 && s.L[(int64_t)d * g.n + v] > 0) claim(6 + d, v0 + o + zo);
        }
    }
    const int k = __popc(got);
    const int incl = warp_incl_scan(k);
    const int total = __shfl_sync(FULL, incl, 31);
    if (total == 0) return;
    unsigned b = 0;
    if (lane_id() == 31) b = atomicAdd(cout, (unsigned)total);
    b = __shfl_sync(FULL, b, 31);
    unsigned pos = b + incl - k;
#pragma unroll
    for (int j = 0; j < 10; j++)
        if (got >> j & 1u) lout[pos++] = u[j];
}

__global__ void __launch_bounds__(256) k_bfs_level(Geo g, Soa s, int L, const int *__restrict__ lin,
                                                   const unsigned *cin, int *lout, unsigned *cout,
                                                   unsigned *czero) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *czero = 0;
    const int64_t count = *cin;
    for (int64_t base = gwarp() * 32; base < count; base += nwarps() * 32) {
        const int64_t i = base + lane_id();
        bfs_expand_warp(g, s, L + 1, i < count ? (int64_t)lin[i] : -1, lout, cout);
    }
}

// Device-driven BFS step (the level counter lives on the device, so identical launches
// can be queued back to back).  Step i = level L = i+1 reads list[i&1] / cnt[i%3],
// writes list[(i+1)&1] / cnt[(i+1)%3] and zeroes cnt[(i+2)%3].
//   large frontier: every block expands one level; the last block to finish advances L;
//   small frontier (<= BFS_SMALL): block 0 alone runs levels back to back separated by
//   __syncthreads (a level costs ~1-2 us instead of a launch), until the frontier grows
//   or empties.
constexpr unsigned BFS_SMALL = 2048;
struct BfsState {
    int L;              // current level (1-based)
    unsigned cnt[3];    // frontier counters
    unsigned finished;  // blocks done with the current large level
};

__global__ void __launch_bounds__(512) k_bfs_step(Geo g, Soa s, int *list0, int *list1, BfsState *st) {
    __shared__ int sL;
    if (threadIdx.x == 0) sL = *(volatile int *)&st->L;
    __syncthreads();
    int L = sL;
    unsigned count = *(volatile unsigned *)&st->cnt[(L - 1) % 3];
    if (count == 0) return;
    if (count <= BFS_SMALL) {
        if (blockIdx.x != 0) return;
        for (;;) {
            const int i = L - 1;
            int *lin = (i & 1) ? list1 : list0;
            int *lout = (i & 1) ? list0 : list1;
            if (threadIdx.x == 0) st->cnt[(i + 2) % 3] = 0;
            for (unsigned base = (threadIdx.x >> 5) * 32; base < count; base += (blockDim.x >> 5) * 32) {
                const unsigned j = base + lane_id();
                bfs_expand_warp(g, s, L + 1, j < count ? (int64_t)lin[j] : -1, lout, &st->cnt[(i + 1) % 3]);
            }
            __syncthreads();
            ++L;
            count = *(volatile unsigned *)&st->cnt[(L - 1) % 3];
            __syncthreads();
            if (count == 0 || count > BFS_SMALL) break;
        }
        if (threadIdx.x == 0) st->L = L;
        return;
    }
    const int i = L - 1;
    const int *lin = (i & 1) ? list1 : list0;
    int *lout = (i & 1) ? list0 : list1;
    if (blockIdx.x == 0 && threadIdx.x == 0) st->cnt[(i + 2) % 3] = 0;
    for (int64_t base = gwarp() * 32; base < count; base += nwarps() * 32) {
        const int64_t j = base + lane_id();
        bfs_expand_warp(g, s, L + 1, j < count ? (int64_t)lin[j] : -1, lout, &st->cnt[(i + 1) % 3]);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned f = atomicAdd(&st->finished, 1u);
        if (f == gridDim.x - 1) {
            st->finished = 0;
            st->L = L + 1;
        }
    }
}

// ------------------------------------------------------------------ a1': column pre-cancellation
// Exact max-flow of every column in isolation (ignoring lateral arcs), applied as the
// initial preflow: source excess may only move DOWN a column (infinite down arcs) into
// sink arcs below it, and the top-down greedy is optimal because the set of sinks a
// source can feed is nested.  With a(z) = E(z) - T(z) and S(z) = sum_{j>=z} a(j):
//   carry leaving z downward    c(z) = S(z) - min_{m in [z, Z]} S(m)       (S(Z) = 0)
//   absorbed at a sink          ab(z) = min(T(z), c(z+1))
//   flow on the down arc z->z-1 f(z) = min(c(z), sum_{z'<z} ab(z'))  (only what is absorbed below)
//   new state  T -= ab,  D = f,  E = f(z+1) + E(z) - ab(z) - f(z) >= 0.
// Not in the paper: an accelerator whose result is a valid preflow, so the maximum flow
// and the minimal cut are unchanged.  One warp per column, z in chunks of 32.
__device__ __forceinline__ long long warp_suffix_sum_ll(long long v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_down_sync(FULL, v, o);
        if (lane_id() + o < 32) v += t;
    }
    return v;
}
__device__ __forceinline__ long long warp_suffix_min_ll(long long v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_down_sync(FULL, v, o);
        if (lane_id() + o < 32) v = min(v, t);
    }
    return v;
}
__device__ __forceinline__ long long warp_excl_prefix_sum_ll(long long v) {
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(FULL, x, o);
        if (lane_id() >= o) x += t;
    }
    return x - v;
}

__global__ void __launch_bounds__(256) k_precancel(Geo g, Soa s, int *flags) {
    extern __shared__ long long sh_c[];  // per warp: Z+1 carries c(z)
    long long *cz = sh_c + (int64_t)(threadIdx.x >> 5) * (g.Z + 1);
    const int64_t ncol = (int64_t)g.X * g.Y;
    const int last_c0 = ((g.Z - 1) >> 5) << 5;
    bool bad = false;
    for (int64_t col = gwarp(); col < ncol; col += nwarps()) {
        const int64_t v0 = col * g.Z;
        // pass 1, top-down: suffix sums S(z) and carries c(z)
        long long sum_above = 0, min_above = 0;  // S over chunks above; min over m above incl. S(Z) = 0
        if (lane_id() == 0) cz[g.Z] = 0;
        for (int c0 = last_c0; c0 >= 0; c0 -= 32) {
            const int z = c0 + lane_id();
            long long a = 0;
            if (z < g.Z) a = (long long)s.E[v0 + z] - (long long)s.T[v0 + z];
            const long long S = warp_suffix_sum_ll(a) + sum_above;
            const long long m = min(warp_suffix_min_ll(z < g.Z ? S : LLONG_MAX), min_above);
            if (z < g.Z) cz[z] = S - m;
            sum_above = __shfl_sync(FULL, S, 0);
            min_above = __shfl_sync(FULL, m, 0);
        }
        __syncwarp();
        // pass 2, bottom-up: absorption, flows, new state
        long long ab_below = 0;  // sum of ab(z') for z' below the chunk
        for (int c0 = 0; c0 < g.Z; c0 += 32) {
            const int z = c0 + lane_id();
            const bool ok = z < g.Z;
            int e = 0, t = 0;
            long long ab = 0, f = 0;
            if (ok) {
                e = s.E[v0 + z];
                t = s.T[v0 + z];
                ab = t > 0 ? min((long long)t, cz[z + 1]) : 0;
            }
            const long long AB = warp_excl_prefix_sum_ll(ab) + ab_below;
            if (ok && z >= 1) f = min(cz[z], AB);
            long long f_up = __shfl_down_sync(FULL, f, 1);
            const long long ab_total = __shfl_sync(FULL, AB + ab, 31);
            if (lane_id() == 31) f_up = (z + 1 < g.Z) ? min(cz[z + 1], ab_total) : 0;
            if (ok) {
                const long long ne = f_up + (long long)e - ab - f;
                if (ne < 0 || ne > INT_MAX || f > INT_MAX) bad = true;
                s.E[v0 + z] = (int32_t)ne;
                s.T[v0 + z] = t - (int32_t)ab;
                s.D[v0 + z] = (int32_t)f;
            }
            ab_below = ab_total;
        }
        __syncwarp();
    }
    if (bad) atomicOr(flags, FLAG_OVERFLOW);
}

// After an exact global relabel: list every chunk holding an active vertex (E > 0,
// H < INF) and count active vertices.  A warp handles 32 consecutive chunks and
// appends them with one atomic.
__global__ void k_rebuild_chunks(Geo g, const Soa s, int *lout, unsigned *cout, int *stamp, int tag,
                                 unsigned long long *active) {
    unsigned long long myact = 0;
    for (int64_t gb = gwarp() * 32; gb < g.nchunks; gb += nwarps() * 32) {
        unsigned mask = 0;
        for (int k = 0; k < 32; k++) {
            const int64_t ch = gb + k;
            if (ch >= g.nchunks) break;
            const int64_t col = ch / g.CPC;
            const int z = (int)(ch - col * g.CPC) * 32 + lane_id();
            bool a = false;
            if (z < g.Z) {
                const int64_t v = col * g.Z + z;
                a = s.E[v] > 0 && s.H[v] < g.INF;
            }
            const unsigned m = __ballot_sync(FULL, a);
            if (m) {
                mask |= 1u << k;
                myact += __popc(m);
            }
        }
        const bool has = (mask >> lane_id()) & 1u;
        if (has) stamp[gb + lane_id()] = tag;
        warp_append(has, (int)(gb + lane_id()), lout, cout);
    }
    if (lane_id() == 0 && myact) atomicAdd(active, myact);
}

// ------------------------------------------------------------------ a5: gap heuristic
// Cherkassky-Goldberg gap: if no vertex has label g (0 < g < max
// finite label), every vertex labelled above g cannot reach t: lift it to INF.
constexpr int GAP_BINS = 1 << 20;
__global__ void k_gap_hist(Geo g, const int32_t *__restrict__ H, unsigned *hist, int *maxh) {
    int mymax = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int h = H[i];
        if (h < g.INF) {
            mymax = max(mymax, h);
            if (h < GAP_BINS) atomicAdd(&hist[h], 1u);
        }
    }
    mymax = warp_max_i(mymax);
    if (lane_id() == 0) atomicMax(maxh, mymax);
}
__global__ void k_gap_find(const unsigned *hist, const int *maxh, int *gap) {
    const int lim = min(*maxh, GAP_BINS - 1);
    int best = INT_MAX;
    for (int h = 1 + (int)threadIdx.x; h < lim; h += blockDim.x)
        if (hist[h] == 0) { best = h; break; }
#pragma unroll
    for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(FULL, best, o));
    __shared__ int sb[32];
    if (lane_id() == 0) sb[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        int b = INT_MAX;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) b = min(b, sb[i]);
        *gap = b;
    }
}
__global__ void k_gap_lift(Geo g, int32_t *H, const int *gap, unsigned long long *lifted) {
    const int gp = *gap;
    int c = 0;
    if (gp != INT_MAX) {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int h = H[i];
            if (h > gp && h < g.INF) { H[i] = g.INF; c++; }
        }
    }
    c = warp_sum_i(c);
    if (lane_id() == 0 && c) atomicAdd(lifted, (unsigned long long)c);
}

// ------------------------------------------------------------------ a6: flow value
__global__ void k_sum_T(Geo g, const int32_t *__restrict__ T, unsigned long long *out) {
    long long acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (int64_t)gridDim.x * blockDim.x)
        acc += T[i];
    acc = warp_sum_ll(acc);
    if (lane_id() == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

// ------------------------------------------------------------------ a7: extraction
// Minimal source set S = forward residual closure of {v : E(v) > 0} (R5,
// SURVEY.md V3).  Infinite down arcs make S downward closed per column, so S is
// top(x,y) = max{z : (x,y,z) in S}.  Worklist closure over columns: proc(col) is the
// highest z whose out-arcs were already scanned; a listed column scans (proc, top]:
//   up arcs        climb while D(top+1) > 0
//   lateral-out    top(nbr) >= zo_eff(top) = max(0, top - Delta)
//   lateral-in rev top(nbr_d) >= zi(z) for z in (proc, top] with L_{d^1}(nbr_d, zi(z)) > 0
// A neighbour whose top rises is listed for the next round.
__device__ __forceinline__ int warp_climb(const Geo &g, const int32_t *__restrict__ D, int64_t v0, int t) {
    for (int base = t + 1; base < g.Z; base += 32) {
        const int z = base + lane_id();
        const bool stop = (z >= g.Z) || D[v0 + z] <= 0;
        const unsigned m = __ballot_sync(FULL, stop);
        if (m) return base + __ffs(m) - 2;
    }
    return g.Z - 1;
}

__global__ void k_ext_seed(Geo g, Soa s, int32_t *top, int32_t *proc, int *lout, unsigned *cout, int *stamp,
                           int tag) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    for (int64_t gb = gwarp() * 32; gb < ncol; gb += nwarps() * 32) {
        int mine = -1;
        for (int k = 0; k < 32; k++) {
            const int64_t col = gb + k;
            if (col >= ncol) break;
            const int64_t v0 = col * g.Z;
            int t = -1;
            for (int c0 = ((g.Z - 1) >> 5) << 5; c0 >= 0 && t < 0; c0 -= 32) {
                const int z = c0 + lane_id();
                const unsigned m = __ballot_sync(FULL, z < g.Z && s.E[v0 + z] > 0);
                if (m) t = c0 + 31 - __clz(m);
            }
            if (lane_id() == k) mine = t;
        }
        const int64_t col = gb + lane_id();
        const bool ok = col < ncol;
        if (ok) {
            top[col] = mine;
            proc[col] = -1;
        }
        const bool has = ok && mine >= 0;
        if (has) stamp[col] = tag;
        warp_append(has, (int)col, lout, cout);
    }
}

__global__ void __launch_bounds__(256) k_ext_round(Geo g, Soa s, const int *__restrict__ lin, const unsigned *cin,
                                                   int *lout, unsigned *cout, unsigned *czero, int32_t *top,
                                                   int32_t *proc, int *stamp, int tag) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *czero = 0;
    const int64_t count = *cin;
    for (int64_t i = gwarp(); i < count; i += nwarps()) {
        const int64_t col = lin[i];
        const int p = proc[col];
        int t = *(volatile int32_t *)&top[col];
        if (t <= p) continue;
        const int64_t v0 = col * g.Z;
        const int x = (int)(col / g.Y), y = (int)(col - (int64_t)x * g.Y);
        t = warp_climb(g, s.D, v0, t);
        if (lane_id() == 0) atomicMax(&top[col], t);
        int64_t ncol[4];
        ncol[0] = x + 1 < g.X ? col + g.Y : -1;
        ncol[1] = x >= 1 ? col - g.Y : -1;
        ncol[2] = y + 1 < g.Y ? col + 1 : -1;
        ncol[3] = y >= 1 ? col - 1 : -1;
        int cd[4] = {-1, -1, -1, -1};
        for (int zb = p + 1; zb <= t; zb += 32) {
            const int z = zb + lane_id();
            const int zi = z <= t ? zi_of(z, g.delta, g.Z) : -1;
#pragma unroll
            for (int d = 0; d < 4; d++)
                if (zi >= 0 && ncol[d] >= 0 && s.L[(int64_t)(d ^ 1) * g.n + ncol[d] * g.Z + zi] > 0)
                    cd[d] = max(cd[d], zi);
        }
        const int zout = t > g.delta ? t - g.delta : 0;
        int mark = -1;
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const int cand = max(warp_max_i(cd[d]), zout);
            if (lane_id() == d && ncol[d] >= 0) {
                const int old = atomicMax(&top[ncol[d]], cand);
                if (old < cand) mark = (int)ncol[d];
            }
        }
        warp_mark(mark, stamp, tag, lout, cout);
        if (lane_id() == 0) proc[col] = t;
    }
}

__global__ void k_ext_out(Geo g, const int32_t *__restrict__ top, int32_t *surface, uint8_t *mask, int *empty) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ncol; i += (int64_t)gridDim.x * blockDim.x) {
        surface[i] = top[i];
        if (top[i] < 0) atomicOr(empty, 1);
    }
    if (mask) {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n;
             i += (int64_t)gridDim.x * blockDim.x)
            mask[i] = (uint8_t)((int)(i % g.Z) <= top[i / g.Z]);
    }
}

}  // namespace cg
