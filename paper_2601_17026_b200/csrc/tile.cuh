// tile.cuh -- a3 on shared-memory column tiles ("tile discharge").
//
// The paper discharges vertices of a column segment from per-thread queues and locks the
// vertices it shares with other segments (§3.2.1, §3.3).  On B200 the
// unit of work is a TILE of TX x TY whole columns (all Z vertices) held in shared memory by
// one CTA, with a read-only halo of the 2(TX+TY) neighbour columns (their heights and the
// residual of their lateral arc into the tile).  Tiles are 2-coloured like a checkerboard
// and a launch ("phase") processes tiles of ONE colour, so no two tiles of a phase are
// lateral neighbours: the halo is an exact snapshot, and the only shared writes are
// excess and reverse residuals pushed into halo vertices (global atomics at the end).
//
// Inside a tile (Alg. 2 L355-404 applied to a region, with Alg. 3's labels made local):
//   A  exact LOCAL relabel: d(v) = BFS distance to t inside the tile, where an arc into a
//      halo vertex u ends the path with cost H(u)+1.  Vertical moves use warp scans
//      (infinite down arcs: d(z) <= d(z-1)+1 is a prefix-min; residual up arcs: a
//      segmented suffix-min), lateral moves use Bellman-Ford rounds over the tile; labels
//      only rise: H = max(H, d) (valid labels are lower bounds of d).
//   B  synchronous push steps: every vertex picks its first admissible arc in the fixed
//      order t, down, lateral-out, up, lateral-in (label of the head < own label).  Runs of
//      vertices whose choice is "down" form chains of infinite arcs: a segmented warp scan
//      moves all excess of a chain to its bottom in one step.  The other arcs push
//      min(E, r); a vertex with excess and no admissible arc relabels to min(H(w))+1.
// Every residual field keeps one decrementer, and within one step the two
// directions of an arc pair are never both admissible (strict label order), so the step
// is race-free with shared-memory atomics on excess.
//
// Thread mapping: warp c owns tile column c; lane l owns the S consecutive vertices
// z = l*S .. l*S+S-1 (S = ceil(Z/32) rounded to an instantiated size).  Shared arrays are
// stored with a lane stride P = S|1 (odd), so the lane-segment accesses are bank-conflict
// free.
#pragma once

#include "kernels.cuh"

namespace cg {

struct TileGeo {
    int32_t TX, TY;      // columns per tile in x and y
    int32_t NTX, NTY;    // tiles in x and y
    int32_t P, CS;       // lane stride (S|1) and column stride (32*P) in shared memory
    int32_t NC, NH;      // TX*TY tile columns, 2*(TX+TY) halo slots
    int32_t steps;       // push steps per tile visit
    int32_t relabel_every;  // exact local relabel every k push steps (and at the visit start)
};

enum : int { CH_NONE = 0, CH_T = 1, CH_DOWN = 2, CH_LOUT = 3, CH_UP = 7, CH_LIN = 8 };
constexpr int LINF = 0x3fffffff;
enum { PF_LOAD = 0, PF_RELABEL, PF_STEPS, PF_STORE, PF_N_RELABEL, PF_LAT_IT, PF_VERT_IT, PF_N_STEPS, PF_VISITS };
constexpr int NB_NONE = INT_MIN;

// shared-memory image of one tile: offsets (in ints) into the dynamic shared array tsm, so
// every access compiles to LDS/STS/ATOMS (pointers kept in a struct would be generic)
extern __shared__ int tsm[];
struct TileSmem {
    int E, H, T, D, L0;  // [NC][CS] each; L[d] at L0 + d*ncs
    int hH, hL, hE;      // [NH][CS]: halo heights, lateral residual toward the tile, pushed excess
    int hflag;           // [NH]: 1 = something was pushed into this slot
    int ncs;             // NC*CS
};

__host__ __device__ inline size_t tile_smem_bytes(const TileGeo &t) {
    return sizeof(int) * ((size_t)8 * t.NC * t.CS + (size_t)3 * t.NH * t.CS + t.NH + 8);
}

__device__ __forceinline__ TileSmem carve_tile(const TileGeo &t) {
    TileSmem m;
    const int ncs = t.NC * t.CS, nhs = t.NH * t.CS;
    m.ncs = ncs;
    m.E = 0;
    m.H = ncs;
    m.T = 2 * ncs;
    m.D = 3 * ncs;
    m.L0 = 4 * ncs;
    m.hH = 8 * ncs;
    m.hL = 8 * ncs + nhs;
    m.hE = 8 * ncs + 2 * nhs;
    m.hflag = 8 * ncs + 3 * nhs;
    return m;
}

template <int S>
__device__ __forceinline__ int tpos(int z, int P) { return (z / S) * P + (z % S); }

// Neighbour column in direction d of tile column (cx, cy) at global (x, y):
//   >= 0     : tile column index
//   < 0      : -1 - halo slot
//   NB_NONE  : no neighbour (volume boundary)
__device__ __forceinline__ int tile_nb(const Geo &g, const TileGeo &t, int cx, int cy, int x, int y, int d) {
    const int dx = d == 0 ? 1 : (d == 1 ? -1 : 0), dy = d == 2 ? 1 : (d == 3 ? -1 : 0);
    const int nx = x + dx, ny = y + dy;
    if (ny < 0 || ny >= g.Y) return NB_NONE;
    const bool in_vol = nx >= 0 && nx < g.X;
    const bool ghost = (nx == -1 && g.gl) || (nx == g.X && g.gh);
    if (!in_vol && !ghost) return NB_NONE;
    const int ncx = cx + dx, ncy = cy + dy;
    if (in_vol && ncx >= 0 && ncx < t.TX && ncy >= 0 && ncy < t.TY) return ncx * t.TY + ncy;
    // halo slot, unique per (side, row): the last present column of a row owns its +x slot
    int slot;
    switch (d) {
        case 0: slot = cy; break;
        case 1: slot = t.TY + cy; break;
        case 2: slot = 2 * t.TY + cx; break;
        default: slot = 2 * t.TY + t.TX + cx; break;
    }
    return -1 - slot;
}

// Per-warp view of its column.
struct ColCtx {
    int c;            // tile column (== warp id)
    int x, y;         // slab-local coordinates
    bool present;
    int64_t v0;       // vertex index of (x, y, 0)
    int nb[4];
};

template <int S>
struct TileOps {
    const Geo &g;
    const TileGeo &t;
    const TileSmem &m;
    const ColCtx &cc;
    __device__ __forceinline__ int at(int zz) const { return cc.c * t.CS + tpos<S>(zz, t.P); }
    __device__ __forceinline__ int nH(int nb, int zz) const {
        return nb >= 0 ? tsm[m.H + (nb * t.CS + tpos<S>(zz, t.P))] : tsm[m.hH + ((-1 - nb) * t.CS + tpos<S>(zz, t.P))];
    }
    // residual of the lateral arc of (nb, zz) pointing back at this column (direction d^1)
    __device__ __forceinline__ int nLres(int nb, int d, int zz) const {
        return nb >= 0 ? tsm[m.L0 + (d ^ 1) * m.ncs + (nb * t.CS + tpos<S>(zz, t.P))] : tsm[m.hL + ((-1 - nb) * t.CS + tpos<S>(zz, t.P))];
    }
};

// ---------------------------------------------------------------- A: exact local relabel
// Column-scan helpers on per-lane register segments d[0..S) (z = lane*S + k).
template <int S>
__device__ __forceinline__ bool vertical_relax(int (&d)[S], unsigned uplink, unsigned frozen, int lane, int Z) {
    // (1) infinite down arcs: d(z) <= d(z-1) + 1  ->  d(z) = z + prefix-min(d(z') - z')
    bool changed = false;
    int m = LINF;
#pragma unroll
    for (int k = 0; k < S; k++) m = min(m, d[k] - (lane * S + k));
    int carry = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, carry, o);
        if (lane >= o) carry = min(carry, t);
    }
    int ex = __shfl_up_sync(FULL, carry, 1);
    if (lane == 0) ex = LINF;
#pragma unroll
    for (int k = 0; k < S; k++) {
        const int z = lane * S + k;
        ex = min(ex, d[k] - z);
        const int nv = ex + z;
        if (nv < d[k] && z < Z && !((frozen >> k) & 1u)) { d[k] = nv; changed = true; }
    }
    // (2) residual up arcs z -> z+1 (uplink bit k: D(z+1) > 0): d(z) <= d(z+1) + 1,
    //     segmented suffix-min of d(z') + z' over linked runs.
    int A = LINF;        // lane transfer: out(in) = min(A, all ? in : LINF)
    bool all = true;
#pragma unroll
    for (int k = S - 1; k >= 0; k--) {
        const int z = lane * S + k;
        const bool lk = (uplink >> k) & 1u;
        A = min(d[k] + z, lk ? A : LINF);
        all = all && lk;
    }
    // suffix scan over lanes (upper lanes are applied first)
    int sA = A;
    bool sall = all;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int uA = __shfl_down_sync(FULL, sA, o);
        const bool uall = __shfl_down_sync(FULL, (int)sall, o);
        if (lane + o < 32) {
            sA = min(sA, sall ? uA : LINF);
            sall = sall && uall;
        }
    }
    int in = __shfl_down_sync(FULL, sA, 1);  // best(z) entering this lane from above
    if (lane == 31) in = LINF;
#pragma unroll
    for (int k = S - 1; k >= 0; k--) {
        const int z = lane * S + k;
        const bool lk = (uplink >> k) & 1u;
        in = min(d[k] + z, lk ? in : LINF);
        const int nv = in - z;
        if (nv < d[k] && z < Z && !((frozen >> k) & 1u)) { d[k] = nv; changed = true; }
    }
    return changed;
}

template <int S>
__device__ __forceinline__ void local_relabel(const Geo &g, const TileGeo &t, const TileSmem &m, const ColCtx &cc, int lane,
                              unsigned long long *prof) {
    int n_lat = 0, n_vert = 0;
    TileOps<S> op{g, t, m, cc};
    const int Z = g.Z;
    int d[S], hold[S];
    unsigned uplink = 0, frozen = 0;
#pragma unroll
    for (int k = 0; k < S; k++) {
        const int z = lane * S + k;
        d[k] = LINF;
        hold[k] = g.INF;
        if (cc.present && z < Z) {
            const int a = op.at(z);
            hold[k] = tsm[m.H + (a)];
            if (z + 1 < Z && tsm[m.D + (op.at(z + 1))] > 0) uplink |= 1u << k;
            if (hold[k] >= g.INF) frozen |= 1u << k;
            if (hold[k] < g.INF) {
                int b = tsm[m.T + (a)] > 0 ? 1 : LINF;
#pragma unroll
                for (int dd = 0; dd < 4; dd++) {
                    const int nb = cc.nb[dd];
                    if (nb == NB_NONE || nb >= 0) continue;  // halo exits only
                    const int zo = zo_of(z, dl_out(g, dd)), zi = zi_of(z, dl_in(g, dd), Z);
                    if (zo >= 0) {
                        const int hh = op.nH(nb, zo);
                        if (hh < g.INF) b = min(b, hh + 1);
                    }
                    if (zi >= 0 && op.nLres(nb, dd, zi) > 0) {
                        const int hh = op.nH(nb, zi);
                        if (hh < g.INF) b = min(b, hh + 1);
                    }
                }
                d[k] = b;
            }
        }
    }
    // vertices at INF stay there (frozen: they cannot have gained out-arcs).  Both loops
    // only lower finite values, so they terminate; the caps are a safety net.
    for (int it = 0; it < 4096; it++) {
        n_lat++;
        for (int vi = 0; vi < 64; vi++) {
            const bool ch = vertical_relax<S>(d, uplink, frozen, lane, Z);
            n_vert++;
            if (!__any_sync(FULL, ch)) break;
        }
        if (cc.present) {
#pragma unroll
            for (int k = 0; k < S; k++) {
                const int z = lane * S + k;
                if (z < Z) tsm[m.H + (op.at(z))] = d[k];
            }
        }
        __syncthreads();
        bool lat = false;
        if (cc.present) {
#pragma unroll
            for (int k = 0; k < S; k++) {
                const int z = lane * S + k;
                if (z >= Z || hold[k] >= g.INF) continue;
                int b = d[k];
#pragma unroll
                for (int dd = 0; dd < 4; dd++) {
                    const int nb = cc.nb[dd];
                    if (nb < 0) continue;  // tile neighbours only (halo exits are in base)
                    const int zo = zo_of(z, dl_out(g, dd)), zi = zi_of(z, dl_in(g, dd), Z);
                    if (zo >= 0) b = min(b, tsm[m.H + (nb * t.CS + tpos<S>(zo, t.P))] + 1);
                    if (zi >= 0 && tsm[m.L0 + (dd ^ 1) * m.ncs + (nb * t.CS + tpos<S>(zi, t.P))] > 0)
                        b = min(b, tsm[m.H + (nb * t.CS + tpos<S>(zi, t.P))] + 1);
                }
                if (b < d[k]) { d[k] = b; lat = true; }
            }
        }
        if (!__syncthreads_or(lat)) break;
    }
    // labels only rise: H = max(H_old, d); d beyond INF means no exit
    if (cc.present) {
#pragma unroll
        for (int k = 0; k < S; k++) {
            const int z = lane * S + k;
            if (z >= Z) continue;
            const int nl = d[k] >= g.INF ? g.INF : d[k];
            tsm[m.H + (op.at(z))] = max(hold[k], nl);
        }
    }
    if (prof && threadIdx.x == 0) {
        atomicAdd(&prof[PF_N_RELABEL], 1ull);
        atomicAdd(&prof[PF_LAT_IT], (unsigned long long)n_lat);
        atomicAdd(&prof[PF_VERT_IT], (unsigned long long)n_vert);
    }
    __syncthreads();
}

// ---------------------------------------------------------------- B: synchronous push steps
template <int S>
__device__ __forceinline__ int min_nbr_label(const Geo &g, const TileOps<S> &op, const ColCtx &cc, int z) {
    const TileSmem &m = op.m;
    const int a = op.at(z);
    if (tsm[m.T + (a)] > 0) return 0;
    int b = g.INF;
    if (z >= 1) b = min(b, tsm[m.H + (op.at(z - 1))]);
#pragma unroll
    for (int d = 0; d < 4; d++) {
        const int nb = cc.nb[d];
        if (nb == NB_NONE) continue;
        const int zo = zo_of(z, dl_out(g, d)), zi = zi_of(z, dl_in(g, d), g.Z);
        if (zo >= 0) b = min(b, op.nH(nb, zo));
        if (zi >= 0 && op.nLres(nb, d, zi) > 0) b = min(b, op.nH(nb, zi));
    }
    if (z + 1 < g.Z && tsm[m.D + (op.at(z + 1))] > 0) b = min(b, tsm[m.H + (op.at(z + 1))]);
    return b;
}

// One synchronous push step.  Returns false (doing nothing) when no vertex of the tile is
// active (E > 0, H < INF).  ops += pushes + relabels of this thread.
//   B1  own segment state in registers; "down" bit = first admissible arc is the down arc
//       (T = 0 and H(z-1) < H(z)) -- needs no neighbour loads (H(z-1) of k = 0 by shuffle)
//   B2  chains of down bits carry their excess to the chain bottom (segmented suffix sum)
//   B3  vertices with excess that are not "down": full arc scan, push on the first
//       admissible arc (t, lateral-out, up, lateral-in); none -> relabel candidate
//   B4  relabel candidates that still hold excess: H = min(H(w)) + 1
template <int S>
__device__ __forceinline__ bool push_step(const Geo &g, const TileGeo &t, const TileSmem &m, const ColCtx &cc, int lane,
                                          unsigned long long &ops, int *flags, bool check_only) {
    TileOps<S> op{g, t, m, cc};
    const int Z = g.Z;
    int e[S], h[S];
    unsigned down = 0, tmask = 0;
    bool act = false;
#pragma unroll
    for (int k = 0; k < S; k++) {
        const int z = lane * S + k;
        e[k] = 0;
        h[k] = g.INF;
        if (cc.present && z < Z) {
            const int a = op.at(z);
            e[k] = tsm[m.E + a];
            h[k] = tsm[m.H + a];
            if (tsm[m.T + a] > 0) tmask |= 1u << k;
            act |= e[k] > 0 && h[k] < g.INF;
        }
    }
    if (!__syncthreads_or(act)) return false;
    if (check_only) return true;
    int hprev = __shfl_up_sync(FULL, h[S - 1], 1);
    if (lane == 0) hprev = g.INF;  // z = 0 has no down arc
#pragma unroll
    for (int k = 0; k < S; k++) {
        const int hb = k == 0 ? hprev : h[k - 1];
        if (h[k] < g.INF && !((tmask >> k) & 1u) && hb < h[k]) down |= 1u << k;
    }
    // B2: lane transfer out(in) = alld ? in + add : add (carry leaving the lane's bottom vertex)
    long long add = 0;
    bool alld = true;
#pragma unroll
    for (int k = S - 1; k >= 0; k--) {
        if ((down >> k) & 1u) add += e[k];
        else { add = 0; alld = false; }
    }
    long long sadd = add;
    bool sall = alld;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long ua = __shfl_down_sync(FULL, sadd, o);
        const bool uall = __shfl_down_sync(FULL, (int)sall, o);
        if (lane + o < 32) {
            sadd = sall ? ua + sadd : sadd;
            sall = sall && uall;
        }
    }
    long long in = __shfl_down_sync(FULL, sadd, 1);
    if (lane == 31) in = 0;
#pragma unroll
    for (int k = S - 1; k >= 0; k--) {
        const int z = lane * S + k;
        if (!cc.present || z >= Z) { in = 0; continue; }
        const int a = op.at(z);
        if ((down >> k) & 1u) {
            const long long f = in + e[k];
            if (f > 0) {
                const long long nd = (long long)tsm[m.D + a] + f;
                if (nd > INT_MAX) atomicOr(flags, FLAG_OVERFLOW);
                tsm[m.D + a] = (int)nd;
                ops++;
            }
            if (e[k]) tsm[m.E + a] = 0;
            e[k] = 0;
            in = f;
        } else {
            if (in > 0) {
                const long long ne = (long long)e[k] + in;
                if (ne > INT_MAX) atomicOr(flags, FLAG_OVERFLOW);
                e[k] = (int)ne;
                tsm[m.E + a] = e[k];
            }
            in = 0;
        }
    }
    __syncthreads();
    // B3: pushes of the vertices holding excess.  Residuals are read here: the pusher is their
    // only decrementer and the reverse pusher is excluded by the label order (strict <).
    unsigned need = 0;
#pragma unroll
    for (int k = 0; k < S; k++) {
        const int z = lane * S + k;
        if (e[k] <= 0 || h[k] >= g.INF) continue;
        const int a = op.at(z);
        const int hk = h[k];
        int df = 0;
        if ((tmask >> k) & 1u) {  // t
            df = min(e[k], tsm[m.T + a]);
            tsm[m.T + a] -= df;
        } else {
            bool done = false;
            {
#pragma unroll
                for (int d = 0; d < 4; d++) {
                    const int nb = cc.nb[d];
                    const int zo = zo_of(z, dl_out(g, d));
                    if (done || nb == NB_NONE || zo < 0) continue;
                    if (op.nH(nb, zo) < hk) {  // lateral-out (infinite)
                        df = e[k];
                        atomicAdd(&tsm[m.L0 + d * m.ncs + a], df);
                        if (nb >= 0) atomicAdd(&tsm[m.E + nb * t.CS + tpos<S>(zo, t.P)], df);
                        else {
                            atomicAdd(&tsm[m.hE + (-1 - nb) * t.CS + tpos<S>(zo, t.P)], df);
                            tsm[m.hflag + (-1 - nb)] = 1;
                        }
                        done = true;
                    }
                }
            }
            if (!done && z + 1 < Z) {
                const int u = op.at(z + 1);
                const int r = tsm[m.D + u];
                const int hu = (k + 1 < S) ? h[(k + 1) % S] : tsm[m.H + u];
                if (r > 0 && hu < hk) {  // up
                    df = min(e[k], r);
                    atomicSub(&tsm[m.D + u], df);
                    atomicAdd(&tsm[m.E + u], df);
                    done = true;
                }
            }
            if (!done) {
#pragma unroll
                for (int d = 0; d < 4; d++) {
                    const int nb = cc.nb[d];
                    const int zi = zi_of(z, dl_in(g, d), Z);
                    if (done || nb == NB_NONE || zi < 0) continue;
                    const int r = op.nLres(nb, d, zi);
                    if (r > 0 && op.nH(nb, zi) < hk) {  // lateral-in reverse
                        df = min(e[k], r);
                        if (nb >= 0) {
                            const int u = nb * t.CS + tpos<S>(zi, t.P);
                            atomicSub(&tsm[m.L0 + (d ^ 1) * m.ncs + u], df);
                            atomicAdd(&tsm[m.E + u], df);
                        } else {
                            const int u = (-1 - nb) * t.CS + tpos<S>(zi, t.P);
                            atomicSub(&tsm[m.hL + u], df);
                            atomicAdd(&tsm[m.hE + u], df);
                            tsm[m.hflag + (-1 - nb)] = 1;
                        }
                        done = true;
                    }
                }
            }
            if (!done) need |= 1u << k;
        }
        if (df > 0) {
            atomicSub(&tsm[m.E + a], df);
            ops++;
        }
    }
    __syncthreads();
    // B4: relabel (labels of neighbours may be changing concurrently: any value read is a
    // valid label of this step, so min + 1 stays a valid label)
#pragma unroll
    for (int k = 0; k < S; k++) {
        if (!((need >> k) & 1u)) continue;
        const int z = lane * S + k;
        const int a = op.at(z);
        if (tsm[m.E + a] <= 0) continue;
        const int b = min_nbr_label<S>(g, op, cc, z);
        const int nh = b >= g.INF ? g.INF : b + 1;
        if (nh > h[k]) {
            tsm[m.H + a] = nh;
            ops++;
        }
    }
    return true;
}

// ---------------------------------------------------------------- the phase kernel
struct TileLists {
    int *list[4];        // ring of tile worklists (phase p reads list[p & 3])
    unsigned *cnt;       // [4]
    int *stamp;          // [ntiles]: phase a tile is listed for
    unsigned long long *prof;  // nullable [16]: cycle / iteration counters (CG_TILE_PROF)
};

__device__ __forceinline__ void tile_list_push(const TileLists &tl, int tile, int phase) {
    if (atomicExch(&tl.stamp[tile], phase) != phase) {
        const unsigned pos = atomicAdd(&tl.cnt[phase & 3], 1u);
        tl.list[phase & 3][pos] = tile;
    }
}

template <int S>
constexpr int tile_max_threads() { return 512; }

template <int S>
__global__ void __launch_bounds__(tile_max_threads<S>(), 1)
    k_tile_phase(Geo g, TileGeo t, Soa s, TileLists tl, int phase, unsigned long long *work,
                 unsigned long long *visits, int *flags) {
    const TileSmem m = carve_tile(t);
    const int lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (blockIdx.x == 0 && threadIdx.x == 0) tl.cnt[(phase + 3) & 3] = 0;
    const unsigned count = *(volatile unsigned *)&tl.cnt[phase & 3];
    if (blockIdx.x == 0 && threadIdx.x == 0) *visits = count;
    const int *lin = tl.list[phase & 3];
    unsigned long long ops = 0;
    for (unsigned li = blockIdx.x; li < count; li += gridDim.x) {
        const long long c0 = clock64();
        const int tile = lin[li];
        const int ttx = tile / t.NTY, tty = tile - ttx * t.NTY;
        const int x0 = ttx * t.TX, y0 = tty * t.TY;
        // ---- column context (warp c = tile column c)
        ColCtx cc;
        cc.c = warp;
        const int cx = warp / t.TY, cy = warp - cx * t.TY;
        cc.x = x0 + cx;
        cc.y = y0 + cy;
        cc.present = warp < t.NC && cc.x < g.X && cc.y < g.Y;
        cc.v0 = ((int64_t)cc.x * g.Y + cc.y) * g.Z;
#pragma unroll
        for (int d = 0; d < 4; d++) cc.nb[d] = cc.present ? tile_nb(g, t, cx, cy, cc.x, cc.y, d) : NB_NONE;
        // ---- load the tile (coalesced along z) and the halo
        if (warp < t.NC) {
            const int cs = warp * t.CS;
            for (int z = lane; z < 32 * S; z += 32) {
                const int a = cs + tpos<S>(z, t.P);
                if (cc.present && z < g.Z) {
                    const int64_t v = cc.v0 + z;
                    tsm[m.E + (a)] = s.E[v]; tsm[m.H + (a)] = s.H[v]; tsm[m.T + (a)] = s.T[v]; tsm[m.D + (a)] = s.D[v];
                    tsm[m.L0 + (0) * m.ncs + (a)] = s.L[0][v]; tsm[m.L0 + (1) * m.ncs + (a)] = s.L[1][v]; tsm[m.L0 + (2) * m.ncs + (a)] = s.L[2][v]; tsm[m.L0 + (3) * m.ncs + (a)] = s.L[3][v];
                } else {
                    tsm[m.E + (a)] = 0; tsm[m.H + (a)] = g.INF; tsm[m.T + (a)] = 0; tsm[m.D + (a)] = 0;
                    tsm[m.L0 + (0) * m.ncs + (a)] = 0; tsm[m.L0 + (1) * m.ncs + (a)] = 0; tsm[m.L0 + (2) * m.ncs + (a)] = 0; tsm[m.L0 + (3) * m.ncs + (a)] = 0;
                }
            }
#pragma unroll
            for (int d = 0; d < 4; d++) {
                const int nb = cc.nb[d];
                if (nb == NB_NONE || nb >= 0) continue;
                const int slot = -1 - nb;
                const int64_t off = d == 0 ? g.YZ : (d == 1 ? -g.YZ : (d == 2 ? (int64_t)g.Z : -(int64_t)g.Z));
                const int64_t u0 = cc.v0 + off;
                const int hs = slot * t.CS;
                for (int z = lane; z < 32 * S; z += 32) {
                    const int a = hs + tpos<S>(z, t.P);
                    if (z < g.Z) {
                        tsm[m.hH + (a)] = s.H[u0 + z];
                        tsm[m.hL + (a)] = s.L[d ^ 1][u0 + z];
                    } else {
                        tsm[m.hH + (a)] = g.INF;
                        tsm[m.hL + (a)] = 0;
                    }
                    tsm[m.hE + (a)] = 0;
                }
                if (lane == 0) tsm[m.hflag + (slot)] = 0;
            }
        }
        __syncthreads();
        long long c1 = clock64();
        // ---- discharge
        bool active = true;
        if (t.relabel_every > 0) local_relabel<S>(g, t, m, cc, lane, tl.prof);
        long long c2 = clock64();
        long long crl = 0;
        int nst = 0;
        for (int st = 0; st <= t.steps; st++) {
            active = push_step<S>(g, t, m, cc, lane, ops, flags, st == t.steps);
            if (!active || st == t.steps) break;
            nst++;
            if (t.relabel_every > 0 && (st + 1) % t.relabel_every == 0) {
                const long long a = clock64();
                local_relabel<S>(g, t, m, cc, lane, tl.prof);
                crl += clock64() - a;
            }
        }
        long long c3 = clock64();
        // ---- write back
        if (cc.present) {
            const int cs = warp * t.CS;
            for (int z = lane; z < g.Z; z += 32) {
                const int a = cs + tpos<S>(z, t.P);
                const int64_t v = cc.v0 + z;
                s.E[v] = tsm[m.E + (a)]; s.H[v] = tsm[m.H + (a)]; s.T[v] = tsm[m.T + (a)]; s.D[v] = tsm[m.D + (a)];
                s.L[0][v] = tsm[m.L0 + (0) * m.ncs + (a)]; s.L[1][v] = tsm[m.L0 + (1) * m.ncs + (a)]; s.L[2][v] = tsm[m.L0 + (2) * m.ncs + (a)]; s.L[3][v] = tsm[m.L0 + (3) * m.ncs + (a)];
            }
#pragma unroll
            for (int d = 0; d < 4; d++) {
                const int nb = cc.nb[d];
                if (nb == NB_NONE || nb >= 0) continue;
                const int slot = -1 - nb;
                if (!tsm[m.hflag + (slot)]) continue;
                const int64_t off = d == 0 ? g.YZ : (d == 1 ? -g.YZ : (d == 2 ? (int64_t)g.Z : -(int64_t)g.Z));
                const int64_t u0 = cc.v0 + off;
                const int hs = slot * t.CS;
                bool got = false;
                for (int z = lane; z < g.Z; z += 32) {
                    const int a = hs + tpos<S>(z, t.P);
                    const int de = tsm[m.hE + (a)];
                    if (de > 0) {
                        const int old = atomicAdd(&s.E[u0 + z], de);
                        if (old > INT_MAX - de) atomicOr(flags, FLAG_OVERFLOW);
                        got = true;
                    }
                    s.L[d ^ 1][u0 + z] = tsm[m.hL + (a)];
                }
                // list the neighbour tile (owned columns only; ghosts go through the halo exchange)
                const int nx = cc.x + (d == 0 ? 1 : (d == 1 ? -1 : 0));
                const int ny = cc.y + (d == 2 ? 1 : (d == 3 ? -1 : 0));
                if (__any_sync(FULL, got) && lane == 0 && nx >= 0 && nx < g.X)
                    tile_list_push(tl, (nx / t.TX) * t.NTY + ny / t.TY, phase + 1);
            }
        }
        if (threadIdx.x == 0 && active) tile_list_push(tl, tile, phase + 2);
        __syncthreads();
        if (tl.prof && threadIdx.x == 0) {
            const long long c4 = clock64();
            atomicAdd(&tl.prof[PF_LOAD], (unsigned long long)(c1 - c0));
            atomicAdd(&tl.prof[PF_RELABEL], (unsigned long long)(c2 - c1 + crl));
            atomicAdd(&tl.prof[PF_STEPS], (unsigned long long)(c3 - c2 - crl));
            atomicAdd(&tl.prof[PF_STORE], (unsigned long long)(c4 - c3));
            atomicAdd(&tl.prof[PF_N_STEPS], (unsigned long long)nst);
            atomicAdd(&tl.prof[PF_VISITS], 1ull);
        }
    }
    // ops of the phase
    ops = warp_sum_ll((long long)ops);
    if (lane == 0 && ops) atomicAdd(work, ops);
    (void)nw;
}

// After a global relabel: list every tile holding an active vertex (E > 0, H < INF) for
// phase p0 (colour 0) or p0 + 1 (colour 1); count active vertices.
__global__ void k_tile_rebuild(Geo g, TileGeo t, Soa s, TileLists tl, int p0, unsigned long long *active) {
    const int ntiles = t.NTX * t.NTY;
    unsigned long long myact = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int ttx = tile / t.NTY, tty = tile - ttx * t.NTY;
        const int x0 = ttx * t.TX, y0 = tty * t.TY;
        int a = 0;
        for (int c = threadIdx.x >> 5; c < t.NC; c += blockDim.x >> 5) {
            const int x = x0 + c / t.TY, y = y0 + c % t.TY;
            if (x >= g.X || y >= g.Y) continue;
            const int64_t v0 = ((int64_t)x * g.Y + y) * g.Z;
            for (int z = lane_id(); z < g.Z; z += 32) a += (s.E[v0 + z] > 0 && s.H[v0 + z] < g.INF);
        }
        a = warp_sum_i(a);
        if (lane_id() == 0) myact += a;
        if (__syncthreads_or(a > 0) && threadIdx.x == 0) {
            const int ph = p0 + ((ttx + tty) & 1);
            tl.stamp[tile] = ph;
            const unsigned pos = atomicAdd(&tl.cnt[ph & 3], 1u);
            tl.list[ph & 3][pos] = tile;
        }
    }
    if (lane_id() == 0 && myact) atomicAdd(active, myact);
}

}  // namespace cg
