// relabel.cuh -- a2/a5 global relabel as a column-scan fixpoint (default since round 2).
//
// What it computes is unchanged: H(v) = the exact BFS distance from v to t in the residual graph
// (§2.1, Alg. 3; reading R6/R8), INF if t is unreachable.  How:
// distances satisfy d(v) = 1 + min over residual out-arcs v -> u of d(u) (d(t) = 0), and inside a
// column the arcs are only the infinite down arcs z -> z-1 and the up arcs z -> z+1 whose residual
// D(z+1) > 0.  So, given the labels of the four neighbour columns, a column's exact labels follow
// from two warp scans over z ("reachability is upward-closed per column"):
//     ext(z) = min( 1 if T(z) > 0,  1 + d(nbr_d, zo(z)),  1 + d(nbr_d, zi(z)) if L_{d^1}(nbr_d, zi(z)) > 0 )
//     A(z)   = min_{z' <= z} ext(z') + (z - z')                       (prefix-min: down arcs)
//     d(z)   = min_{z' >= z, up-chain z..z' residual} A(z') + (z' - z)   (segmented suffix-min: up arcs)
// A column whose labels drop lists its four neighbours for the next round; rounds repeat until no
// label changes (Bellman-Ford from INF over columns: every value is the length of a real path, so
// it is an upper bound that only decreases, and the fixpoint is the exact distance).  One
// cooperative launch runs every round with a grid barrier between rounds (the paper's per-level
// barrier, L281); small worklists are run by block 0 alone with block barriers.
//
// Compared with the vertex-frontier BFS (k_bfs_run): a round's work is coalesced 32-z chunks of
// listed columns (flags 1 B + labels 4 B per vertex, neighbour spans shifted by Delta) instead of
// scattered 32-B records per frontier vertex, and the labels live in their own int32 plane; the
// records' H is written once, by the rebuild pass that lists the active vertices.
#pragma once

#include "kernels.cuh"

#ifndef CG_INIT_PRELOAD
#define CG_INIT_PRELOAD 1
#endif
#define CG_REBUILD_PRELOAD (CG_INIT_PRELOAD && CG_LAYOUT_AOS && !CG_H_PLANE)
namespace cg {

// flags[v]: bit 0 T(v) > 0 (arc to t), bit 1 D(v) > 0 (residual of the up arc (v-1) -> v),
// bits 2+d: L_d(v) > 0 (residual of the reverse of v's lateral arc in direction d, i.e. an arc from
// v's lateral target back to v).  Over owned and ghost planes; labels start at INF.
__global__ void k_colgr_flags(Geo g, Soa s, uint8_t *flags, int32_t *lab, int64_t lo, int64_t hi) {
    for (int64_t v = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < hi;
         v += (int64_t)gridDim.x * blockDim.x) {
#if CG_LAYOUT_AOS
        const int4 *rec = reinterpret_cast<const int4 *>(&s.E[v]);  // E H T D | L0 L1 L2 L3
        const int4 a = rec[0], b = rec[1];
        const int T = a.z, D = a.w, L0 = b.x, L1 = b.y, L2 = b.z, L3 = b.w;
#else
        const int T = s.T[v], D = s.D[v], L0 = s.L[0][v], L1 = s.L[1][v], L2 = s.L[2][v], L3 = s.L[3][v];
#endif
        flags[v] = (uint8_t)((T > 0) | (D > 0) << 1 | (L0 > 0) << 2 | (L1 > 0) << 3 | (L2 > 0) << 4 | (L3 > 0) << 5);
        lab[v] = g.INF;
    }
}

// Flag-plane BFS init (hard graphs, the default relabel): one dense pass over the records writes the
// flags, the labels (1 for the seeds T > 0 -- Alg. 3's first level, reading R6 -- else INF), the
// visited bitmap and the seed list; k_bfs_run<true> then expands from the flags and writes `lab`.
__global__ void k_bfs2_init(Geo g, Soa s, uint8_t *flags, int32_t *lab, unsigned *visited, int *lout,
                            unsigned *cout, unsigned *dbits = nullptr) {
    // dbits (dense bit-plane levels, k_bfs_run): the residual bits as 32-vertex words -- Dm (D > 0),
    // Lm[d] (L_d > 0) -- and the seed frontier F0, NW words per plane
    const int64_t NW = g.n / 32 + 1;
    // (measured: loading a span's records ahead of the flag writes with streaming loads made this
    // pass slower, 0.80 -> 1.22 ms at C4 under ncu; CG_INIT_PRELOAD loads the span's records with
    // plain loads before any store -- the stores to flags / lab / visited otherwise keep each
    // record load waiting for the previous iteration's, one DRAM round trip per 32 vertices)
    constexpr int SPAN = 8;
    SpanAppender<SPAN> ap;
    for (int64_t base = gwarp() * 32 * SPAN; base < g.n; base += nwarps() * 32 * SPAN) {
#if CG_LAYOUT_AOS && CG_INIT_PRELOAD
        int4 ra[SPAN], rb[SPAN];
#pragma unroll
        for (int j = 0; j < SPAN; j++) {
            const int64_t v = base + 32 * j + lane_id();
            if (v < g.n) {
                const int4 *rec = reinterpret_cast<const int4 *>(&s.E[v]);
                ra[j] = rec[0];
                rb[j] = rec[1];
            }
        }
#endif
#pragma unroll
        for (int j = 0; j < SPAN; j++) {
            const int64_t b0 = base + 32 * j;
            const int64_t v = b0 + lane_id();
            bool seed = false;
            unsigned bits = 0;  // bit 1: D > 0, bits 2+d: L_d > 0
            if (v < g.n) {
#if CG_LAYOUT_AOS && CG_INIT_PRELOAD
                const int4 a = ra[j], b = rb[j];
                const int T = a.z, D = a.w, L0 = b.x, L1 = b.y, L2 = b.z, L3 = b.w;
#elif CG_LAYOUT_AOS
                const int4 *rec = reinterpret_cast<const int4 *>(&s.E[v]);  // E H T D | L0 L1 L2 L3
                const int4 a = rec[0], b = rec[1];
                const int T = a.z, D = a.w, L0 = b.x, L1 = b.y, L2 = b.z, L3 = b.w;
#else
                const int T = s.T[v], D = s.D[v], L0 = s.L[0][v], L1 = s.L[1][v], L2 = s.L[2][v], L3 = s.L[3][v];
#endif
                seed = T > 0;
                bits = (D > 0) << 1 | (L0 > 0) << 2 | (L1 > 0) << 3 | (L2 > 0) << 4 | (L3 > 0) << 5;
                flags[v] = (uint8_t)(seed | bits);
                lab[v] = seed ? 1 : g.INF;
            }
            const unsigned m = __ballot_sync(FULL, seed);
            if (lane_id() == 0 && b0 < g.n) visited[b0 >> 5] = m;
            if (dbits) {
                const unsigned md = __ballot_sync(FULL, bits & 2u), m0 = __ballot_sync(FULL, bits & 4u),
                               m1 = __ballot_sync(FULL, bits & 8u), m2 = __ballot_sync(FULL, bits & 16u),
                               m3 = __ballot_sync(FULL, bits & 32u);
                if (lane_id() == 0 && b0 < g.n) {
                    const int64_t w = b0 >> 5;
                    dbits[w] = md;
                    dbits[NW + w] = m0;
                    dbits[2 * NW + w] = m1;
                    dbits[3 * NW + w] = m2;
                    dbits[4 * NW + w] = m3;
                    dbits[5 * NW + w] = m;
                }
            }
            ap.add(m, b0);
        }
        ap.flush(lout, cout);
    }
}

// In-process x-slabs (colgraph_build_slabs): the in-slab flag-plane BFS of EVERY slab in one
// cooperative launch.  The slabs' BFSes are independent (each claims owned vertices only); running
// them level by level in the same grid shares the grid barrier and the latency of the small levels
// instead of paying them once per slab.  With one slab per GPU (NCCL) each rank runs k_bfs_run.
constexpr int MSLAB_MAX = 32;
struct SlabBfsDesc {
    Geo g;
    Soa s;
    int *list[2];
    unsigned *cnt;  // 3 frontier counters (the slab's BfsState.cnt)
    unsigned *visited;
    const uint8_t *flags;
    int32_t *lab;
};
struct MultiBfsState {
    int L;
    unsigned bar[3];
};
__global__ void __launch_bounds__(512, 1) k_bfs_run_slabs(const SlabBfsDesc *__restrict__ sd, int S, MultiBfsState *st) {
    __shared__ unsigned pre[MSLAB_MAX + 1], cnt[MSLAB_MAX];
    int L = *(volatile int *)&st->L;
    for (int guard = 0;; guard++) {
        const int i = L - 1;
        if (threadIdx.x == 0) {  // chunks of 32 * BFS_R frontier vertices per slab, prefix over the slabs
            unsigned acc = 0;
            for (int k = 0; k < S; k++) {
                const unsigned c = *(volatile unsigned *)&sd[k].cnt[i % 3];
                cnt[k] = c;
                pre[k] = acc;
                acc += (c + 32 * BFS_R - 1) / (32 * BFS_R);
            }
            pre[S] = acc;
        }
        __syncthreads();
        const unsigned total = pre[S];
        if (total == 0 || guard > sd[0].g.INF + 2) break;
        if (blockIdx.x == 0 && threadIdx.x < S) sd[threadIdx.x].cnt[(i + 2) % 3] = 0;
        for (int64_t ch = gwarp(); ch < total; ch += nwarps()) {
            int k = 0;
            while (k + 1 < S && pre[k + 1] <= ch) k++;
            const SlabBfsDesc &d = sd[k];
            const int *lin = d.list[i & 1];
            int *lout = d.list[(i + 1) & 1];
            const unsigned c = cnt[k];
            const int64_t base = (ch - pre[k]) * 32 * BFS_R;
            int vv[BFS_R];
#pragma unroll
            for (int r = 0; r < BFS_R; r++) {
                const int64_t j = base + r * 32 + lane_id();
                vv[r] = j < c ? __ldcg(&lin[j]) : -1;
            }
            bfs_expand_multi<BFS_R, true>(d.g, d.s, L + 1, vv, lout, &d.cnt[(i + 1) % 3], d.visited, d.flags, d.lab);
        }
        grid_barrier(st->bar, gridDim.x);
        ++L;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) st->L = L;
}

struct ColGrState {
    int round;                  // current round (0: every column)
    unsigned cnt[3];            // worklist counters (round r reads cnt[r % 3])
    unsigned bar[3];            // grid barrier (arrivals, generation, back-off cap in ns)
    unsigned small;             // worklists <= small run in block 0 alone
    int tag0;                   // colstamp tag of round r's output list = tag0 + r
    unsigned long long updates; // column updates
    unsigned long long changed; // column updates that lowered a label
    unsigned rounds_small;      // rounds run by block 0
};

constexpr int COLGR_MAX_CPC = 8;  // Z <= 256 (larger Z: the vertex BFS)

// Exact labels of one column (warp-collective) from its neighbours' current labels; returns true
// (warp-uniform) if any label of the column dropped.  Every load of the column (own flags and
// labels, the neighbours' labels at zo / zi and their flags at zi, all chunks) is issued before the
// scans, so an update costs one memory round trip instead of one per chunk and direction.
template <int CPC>
__device__ __forceinline__ bool colgr_update(const Geo &g, const uint8_t *__restrict__ flags, int32_t *lab,
                                             int64_t col) {
    const int lane = lane_id();
    const int Z = g.Z, INF = g.INF;
    const int64_t v0 = col * Z;
    const int x = (int)(col / g.Y), y = (int)(col - (int64_t)x * g.Y);
    int64_t off[4];
#pragma unroll
    for (int d = 0; d < 4; d++) off[d] = nbr_off(g, x, y, d);
    int e[CPC], old[CPC];
    unsigned fl[CPC];
#pragma unroll
    for (int k = 0; k < CPC; k++) {
        const int z = 32 * k + lane;
        e[k] = INF;
        old[k] = INF;
        fl[k] = 0;
        if (z < Z) {
            fl[k] = flags[v0 + z];
            old[k] = __ldcg(&lab[v0 + z]);  // L1 may hold this column from an earlier round
            int lo[4], li[4];
            unsigned fi[4];
#pragma unroll
            for (int d = 0; d < 4; d++) {
                const int zo = zo_of(z, dl_out(g, d)), zi = zi_of(z, dl_in(g, d), Z);
                const int64_t u0 = v0 + off[d];
                lo[d] = off[d] && zo >= 0 ? __ldcg(&lab[u0 + zo]) : INF;
                li[d] = off[d] && zi >= 0 ? __ldcg(&lab[u0 + zi]) : INF;
                fi[d] = off[d] && zi >= 0 ? flags[u0 + zi] : 0u;
            }
            int m = (fl[k] & 1) ? 0 : INF;
#pragma unroll
            for (int d = 0; d < 4; d++) {
                m = min(m, lo[d]);
                if (fi[d] >> (2 + (d ^ 1)) & 1) m = min(m, li[d]);
            }
            e[k] = m >= INF ? INF : m + 1;
        }
    }
    // prefix-min of ext(z') - z' over the column (infinite down arcs)
    int carry = INT_MAX;
#pragma unroll
    for (int k = 0; k < CPC; k++) {
        const int z = 32 * k + lane;
        int a = z < Z ? e[k] - z : INT_MAX;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL, a, o);
            if (lane >= o) a = min(a, t);
        }
        a = min(a, carry);
        carry = __shfl_sync(FULL, a, 31);
        e[k] = z < Z ? min(a + z, INF) : INF;  // A(z)
    }
    // segmented suffix-min of A(z') + z' along residual up-chains, top chunk first
    bool changed = false;
    int carry2 = INT_MAX;
#pragma unroll
    for (int k = CPC - 1; k >= 0; k--) {
        const int z = 32 * k + lane;
        // residual up arc z -> z+1: bit 1 of the flags of z+1 (next lane, or lane 0 of the chunk above)
        unsigned fnext = __shfl_down_sync(FULL, fl[k], 1);
        const unsigned fabove = k + 1 < CPC ? __shfl_sync(FULL, fl[k + 1 < CPC ? k + 1 : k], 0) : 0u;
        if (lane == 31) fnext = fabove;
        const bool up = z + 1 < Z && (fnext & 2);
        const unsigned brk = __ballot_sync(FULL, !up);  // chain ends at these lanes
        const unsigned m = brk >> lane;
        const int hi = m ? lane + __ffs(m) - 1 : 32;    // last lane of this lane's chain in the chunk
        int s = z < Z ? e[k] + z : INT_MAX;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_down_sync(FULL, s, o);
            if (lane + o <= min(hi, 31)) s = min(s, t);
        }
        if (hi == 32) s = min(s, carry2);  // the chain continues into the chunk above
        carry2 = __shfl_sync(FULL, s, 0);
        if (z < Z) {
            const int dz = min(e[k], s == INT_MAX ? INF : s - z);
            if (dz < old[k]) {
                lab[v0 + z] = dz;
                changed = true;
            }
        }
    }
    return __any_sync(FULL, changed);
}

// the (up to four) neighbour columns of a changed column join the next round's worklist (owned
// columns only; a ghost column's owner learns about the change through the slab exchange)
__device__ __forceinline__ void colgr_mark_nbrs(const Geo &g, int64_t col, bool changed, int *stamp, int tag,
                                                int *lout, unsigned *cout) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    int64_t nc = -1;
    if (changed && lane_id() < 4) {
        const int x = (int)(col / g.Y), y = (int)(col - (int64_t)x * g.Y);
        switch (lane_id()) {
            case 0: nc = x + 1 < g.X ? col + g.Y : -1; break;
            case 1: nc = x >= 1 ? col - g.Y : -1; break;
            case 2: nc = y + 1 < g.Y ? col + 1 : -1; break;
            default: nc = y >= 1 ? col - 1 : -1; break;
        }
    }
    warp_mark(nc >= 0 && nc < ncol ? (int)nc : -1, stamp, tag, lout, cout);
}

// Persistent fixpoint: rounds until a worklist is empty.  Round r's input is the list
// list[r & 1] with count st->cnt[r % 3], or (dense = 1, first round) every column.  A round whose
// list holds more than a quarter of the columns walks all columns in index order instead (forward
// on even rounds, backward on odd ones) and updates those stamped for this round or later: labels
// written earlier in the same round are read by later columns (Gauss-Seidel), so one round carries
// paths across many columns in the walking direction.  Lists of <= st->small columns are run by
// block 0 alone, rounds separated by block barriers.  Launch cooperatively.
template <int CPC>
__global__ void __launch_bounds__(512, (CPC > 4 ? 1 : 2)) k_colgr_run(Geo g, const uint8_t *__restrict__ flags, int32_t *lab,
                                                     int *list0, int *list1, ColGrState *st, int *stamp, int dense) {
    unsigned *bar = st->bar;
    const int64_t ncol = (int64_t)g.X * g.Y;
    const int tag0 = st->tag0;
    int r = *(volatile int *)&st->round;
    unsigned long long upd = 0, chg = 0;
    for (int guard = 0; guard <= g.INF + 2; guard++) {
        const bool first = dense && guard == 0;
        const unsigned count = first ? (unsigned)ncol : *(volatile unsigned *)&st->cnt[r % 3];
        if (count == 0) break;
        const int *lin = (r & 1) ? list1 : list0;
        int *lout = (r & 1) ? list0 : list1;
        const bool walk_all = first || (int64_t)count * 4 > ncol;
        if (!walk_all && count <= st->small) {
            // small worklists: block 0 alone, rounds separated by block barriers
            grid_barrier(bar, gridDim.x);
            if (blockIdx.x == 0) {
                unsigned c = count;
                for (;;) {
                    const int *li = (r & 1) ? list1 : list0;
                    int *lo = (r & 1) ? list0 : list1;
                    if (threadIdx.x == 0) {
                        st->cnt[(r + 2) % 3] = 0;
                        st->rounds_small++;
                    }
                    for (unsigned i = threadIdx.x >> 5; i < c; i += blockDim.x >> 5) {
                        const int64_t col = __ldcg(&li[i]);
                        const bool ch = colgr_update<CPC>(g, flags, lab, col);
                        upd++;
                        chg += ch;
                        colgr_mark_nbrs(g, col, ch, stamp, tag0 + r + 1, lo, &st->cnt[(r + 1) % 3]);
                    }
                    __syncthreads();
                    ++r;
                    c = *(volatile unsigned *)&st->cnt[r % 3];
                    __syncthreads();
                    if (c == 0 || c > st->small) break;
                }
                if (threadIdx.x == 0) st->round = r;
            }
            grid_barrier(bar, gridDim.x);
            r = *(volatile int *)&st->round;
            continue;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) st->cnt[(r + 2) % 3] = 0;
        if (walk_all) {
            for (int64_t i = gwarp(); i < ncol; i += nwarps()) {
                const int64_t col = (r & 1) ? ncol - 1 - i : i;
                if (!first && __ldcg(&stamp[col]) < tag0 + r) continue;  // not listed for this round (yet)
                const bool ch = colgr_update<CPC>(g, flags, lab, col);
                upd++;
                chg += ch;
                colgr_mark_nbrs(g, col, ch, stamp, tag0 + r + 1, lout, &st->cnt[(r + 1) % 3]);
            }
        } else {
            for (int64_t i = gwarp(); i < count; i += nwarps()) {
                const int64_t col = __ldcg(&lin[i]);
                const bool ch = colgr_update<CPC>(g, flags, lab, col);
                upd++;
                chg += ch;
                colgr_mark_nbrs(g, col, ch, stamp, tag0 + r + 1, lout, &st->cnt[(r + 1) % 3]);
            }
        }
        grid_barrier(bar, gridDim.x);
        ++r;
    }
    if (lane_id() == 0) {
        atomicAdd(&st->updates, upd);
        atomicAdd(&st->changed, chg);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) st->round = r;
}

// After the fixpoint: the records' H = the labels, and every active vertex (E > 0, H < INF) is
// listed for the sweeps in index order (replaces k_rebuild_vertices for this relabel).
__global__ void k_colgr_rebuild(Geo g, Soa s, const int32_t *__restrict__ lab, int *lout, unsigned *cout, int *vstamp,
                                int tag, unsigned long long *active) {
    constexpr int SPAN = 8;
    SpanAppender<SPAN> ap;
    unsigned long long myact = 0;
    for (int64_t base = gwarp() * 32 * SPAN; base < g.n; base += nwarps() * 32 * SPAN) {
#if CG_REBUILD_PRELOAD
        int hl[SPAN], hh[SPAN], he[SPAN];  // every load of the span before any store (see k_bfs2_init)
#pragma unroll
        for (int j = 0; j < SPAN; j++) {
            const int64_t v = base + 32 * j + lane_id();
            if (v < g.n) {
                hl[j] = lab[v];
                const int2 eh = *reinterpret_cast<const int2 *>(&s.E[v]);  // E, H (adjacent in the record)
                he[j] = eh.x;
                hh[j] = eh.y;
            }
        }
#endif
#pragma unroll
        for (int j = 0; j < SPAN; j++) {
            const int64_t b0 = base + 32 * j;
            const int64_t v = b0 + lane_id();
            bool a = false;
            if (v < g.n) {
#if CG_REBUILD_PRELOAD
                const int h = hl[j];
                if (hh[j] != h) s.H[v] = h;  // same sector as E: an unchanged label leaves it clean
                a = he[j] > 0 && h < g.INF;
#else
                const int h = lab[v];
                if (s.H[v] != h) s.H[v] = h;  // same sector as E: an unchanged label leaves it clean
                a = s.E[v] > 0 && h < g.INF;
#endif
            }
            if (a) vstamp[v] = tag;
            myact += a;
            ap.add(__ballot_sync(FULL, a), b0);
        }
        ap.flush(lout, cout);
    }
    myact = warp_sum_ll((long long)myact);
    if (lane_id() == 0 && myact) atomicAdd(active, myact);
}

// x-slabs: labels of this slab's boundary planes -> send buffers (both sides, one launch)
__global__ void k_colgr_pack(Geo g, const int32_t *__restrict__ lab, int32_t *send0, int32_t *send1) {
    const int64_t m = (int64_t)(g.gl + g.gh) * g.YZ;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const bool hi = !g.gl || t >= g.YZ;
        const int64_t i = t - (g.gl && hi ? g.YZ : 0);
        (hi ? send1 : send0)[i] = lab[(hi ? g.n - g.YZ : 0) + i];
    }
}

// x-slabs: a neighbour's boundary labels land in this slab's ghost plane; every boundary column
// facing a ghost column whose labels dropped is listed for the next fixpoint (warp per column).
// The list and tag are those of the round the fixpoint stopped at (read from st on the device).
__global__ void k_colgr_unpack(Geo g, int32_t *lab, const int32_t *__restrict__ recv0,
                               const int32_t *__restrict__ recv1, int *stamp, int *list0, int *list1, ColGrState *st) {
    const int r = st->round;
    int *lout = (r & 1) ? list1 : list0;
    unsigned *cout = &st->cnt[r % 3];
    const int tag = st->tag0 + r;
    const int64_t m = (int64_t)(g.gl + g.gh) * g.Y;  // ghost columns of both sides
    for (int64_t t = gwarp(); t < m; t += nwarps()) {
        const bool hi = !g.gl || t >= g.Y;
        const int64_t y = t - (g.gl && hi ? g.Y : 0);
        const int32_t *rc = (hi ? recv1 : recv0) + y * g.Z;
        int32_t *gl = lab + (hi ? g.n : -g.YZ) + y * g.Z;
        bool ch = false;
        for (int z = lane_id(); z < g.Z; z += 32) {
            const int nv = rc[z];
            if (nv < gl[z]) {
                gl[z] = nv;
                ch = true;
            }
        }
        ch = __any_sync(FULL, ch);
        const int64_t col = (hi ? (int64_t)(g.X - 1) * g.Y : 0) + y;  // the facing boundary column
        warp_mark(ch && lane_id() == 0 ? (int)col : -1, stamp, tag, lout, cout);
    }
}

// x-slabs: ghost records' H = the owner's exact labels (for the sweeps)
__global__ void k_colgr_ghost_h(Geo g, Soa s, const int32_t *__restrict__ lab) {
    const int64_t m = (int64_t)(g.gl + g.gh) * g.YZ;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const bool hi = !g.gl || t >= g.YZ;
        const int64_t i = (hi ? g.n : -g.YZ) + t - (g.gl && hi ? g.YZ : 0);
        s.H[i] = lab[i];
    }
}

}  // namespace cg
