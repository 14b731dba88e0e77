// kernels.cuh -- the sm_100a kernels of the column-graph max-flow hot path.
//
//   a1  build             k_build                      PAPER.md §1.2; §2.1 L134 (init)
//   a2/a5 global relabel  column fixpoint: relabel.cuh; vertex-frontier BFS (soft graphs, Z > 256,
//                         CG_RELABEL=bfs): k_bfs_init + k_bfs_run / k_bfs_step, x-slab levels
//                         k_slab_level   PAPER.md §2.1; Alg. 3; §3.2.2
//   a3  sweep             k_walk_ws (multi-hop), k_sweep_v PAPER.md §2.1; Alg. 2
//   a4  termination       k_rebuild_vertices + host    PAPER.md §3.2.4; Alg. 1
//   a5  gap               k_gap_*                      PAPER.md §2.1
//   a6  flow value        k_sum_T                      PAPER.md Eq. 5
//   a7  extraction        k_ext_*                      PAPER.md Theorem 1
//   a8  halo exchange     k_halo_*, k_ghost_*          PAPER.md §3.2.1 L254 (shared vertices)
#pragma once

#include "common.cuh"

namespace cg {

// Occupancy targets of the latency-bound worklist kernels (blocks per SM).
#ifndef CG_SWEEP_MINB
#define CG_SWEEP_MINB 3
#endif
#ifndef CG_BFS_MINB
#define CG_BFS_MINB 2
#endif

// ------------------------------------------------------------------ a1: build
// Vertex weights of one column (warp-collective): w(0) = c(0) - (sum_z c + 1), w(z) = c(z) - c(z-1)
// (R1); with a narrow band [lo, hi) (NEXT-3, reading R15) the rule applies to the band
// (w(lo) = c(lo) - (sum_{lo<=z<hi} c + 1)) and vertices outside it get w = 0; weight mode takes w as
// given.  k_build, the phase-2 setup and the flow export all recompute w with these two functions.
struct ColW {
    int lo, hi;
    long long colsum;
    bool bad;  // invalid band (lo < 0, lo >= hi or hi > Z)
};
__device__ __forceinline__ ColW col_w_setup(const int32_t *cc, int Z, const int32_t *band, int64_t col, int weight_mode) {
    ColW w{0, Z, 0, false};
    if (band) {
        w.lo = band[2 * col];
        w.hi = band[2 * col + 1];
        w.bad = w.lo < 0 || w.lo >= w.hi || w.hi > Z;
        if (w.bad) w.lo = 0, w.hi = Z;
    }
    if (!weight_mode) {
        long long cs = 0;
        for (int z = w.lo + lane_id(); z < w.hi; z += 32) cs += cc[z];
        w.colsum = warp_sum_ll(cs);
    }
    return w;
}
__device__ __forceinline__ long long col_w(const int32_t *cc, int z, const ColW &w, int weight_mode) {
    if (weight_mode) return cc[z];
    if (z < w.lo || z >= w.hi) return 0;
    return z == w.lo ? (long long)cc[z] - (w.colsum + 1) : (long long)cc[z] - (long long)cc[z - 1];
}

// One warp per column.  E = max(0,-w): source arcs pre-saturated (Goldberg-Tarjan init,
// PAPER.md:134); T = max(0, w): sink-arc residual.  Totals N = sum E and sum T0 in int64.
__global__ void k_build(Geo g, const int32_t *__restrict__ in, int weight_mode, const int32_t *__restrict__ band,
                        Soa s, unsigned long long *sums /* [0]=N [1]=sum T0 */, int *flags) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    long long accN = 0, accT = 0;
    bool bad = false, badband = false;
    for (int64_t col = gwarp(); col < ncol; col += nwarps()) {
        const int32_t *cc = in + col * g.Z;
        const ColW cw = col_w_setup(cc, g.Z, band, col, weight_mode);
        badband |= cw.bad;
        for (int z = lane_id(); z < g.Z; z += 32) {
            const long long w = col_w(cc, z, cw, weight_mode);
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
    if (badband) atomicOr(flags, FLAG_BAD_BAND);
}

// ------------------------------------------------------------------ NEXT-2: phase 2 + flow export
// Vertex weights are recomputed from the caller's input exactly as k_build does (one warp per
// column) to recover the source / sink capacities E0 = max(0,-w), T0 = max(0,w).
// tmp = phase-1 sink residual T; T := E0 (flow on the saturated source arc s->v)
__global__ void k_phase2_setup(Geo g, const int32_t *__restrict__ in, int weight_mode, const int32_t *__restrict__ band,
                               Soa s, int32_t *tmp) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    for (int64_t col = gwarp(); col < ncol; col += nwarps()) {
        const int32_t *cc = in + col * g.Z;
        const ColW cw = col_w_setup(cc, g.Z, band, col, weight_mode);
        for (int z = lane_id(); z < g.Z; z += 32) {
            const int64_t v = col * g.Z + z;
            const long long w = col_w(cc, z, cw, weight_mode);
            tmp[v] = s.T[v];
            s.T[v] = w < 0 ? (int32_t)(-w) : 0;
        }
    }
}

// Phase 2 by level-ordered flow cancellation.  Every arc that carries flow goes down in z
// (down arcs, lateral arcs to z - Delta) except the lateral arcs on the same level (z = 0, or
// Delta_d = 0), so the excess of a vertex at level z is returned by cancelling its inflows:
// first its source arc (T holds the source-arc flow in phase 2), then the flow from above
// (D(z+1), moving the excess up to z+1), then the lateral inflows from (nbr, zi(z)) (moving it
// to level zi(z) >= z).  E(v) = fs(v) + inflow - outflow <= fs(v) + inflow, so the
// cancellation never runs out.  One launch per level processes every column; levels with
// same-level arcs repeat until a pass sees no excess there (*left counts vertices with excess).
__global__ void k_return_level(Geo g, Soa s, int z, unsigned *left) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    unsigned myleft = 0;
    for (int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; col < ncol;
         col += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = col * g.Z + z;
        int e = __ldcg(&s.E[v]);
        if (e <= 0) continue;
        myleft++;  // excess seen on this level in this pass (same-level passes repeat until none)
        const int x = (int)(col / g.Y), y = (int)(col - (int64_t)x * g.Y);
        int taken = 0;
        auto cancel = [&](int32_t *res, int32_t *eto) {
            const int r = min(e, *(volatile int32_t *)res);
            if (r > 0) {
                atomicSub(res, r);
                if (eto) atomicAdd(eto, r);
                e -= r;
                taken += r;
            }
        };
        cancel(&s.T[v], nullptr);  // back to s
        if (e > 0 && z + 1 < g.Z) cancel(&s.D[v + 1], &s.E[v + 1]);
#pragma unroll
        for (int d = 0; d < 4 && e > 0; d++) {
            const int64_t o = nbr_off(g, x, y, d);
            const int zi = zi_of(z, dl_in(g, d), g.Z);
            if (!o || zi < 0) continue;
            const int64_t u = col * g.Z + o + zi;  // may be a ghost vertex: the halo delivers E(u)
            cancel(&s.L[d ^ 1][u], &s.E[u]);
        }
        for (int d = 0; d < 4 && e > 0 && g.soft_k; d++) {  // soft inflows from (nbr, z + k), level >= z
            const int64_t o = nbr_off(g, x, y, d);
            if (!o) continue;
            const int kmax = min(g.soft_k, dl_in(g, d));  // the neighbour's soft arcs toward d^1
            for (int k = 0; k < kmax && e > 0; k++) {
                if (z + k >= g.Z) break;
                const int64_t u = col * g.Z + o + z + k;
                cancel(soft_flow(g, s, u, d ^ 1, k), &s.E[u]);
            }
        }
        if (taken) atomicSub(&s.E[v], taken);
    }
    myleft = warp_sum_i((int)myleft);
    if (lane_id() == 0 && myleft) atomicAdd(left, myleft);
}

// Same-level flow circulations: where the lateral arcs of level z stay on level z (z = 0,
// or Delta_d = 0), the two antiparallel arcs v -> u and u -> v may both carry flow; netting
// them removes a 2-cycle without changing any excess (each pair is owned by the vertex on
// its +x / +y side... i.e. by v for directions d = 0, 2).
__global__ void k_net_level(Geo g, Soa s, int z) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    for (int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; col < ncol;
         col += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = col * g.Z + z;
        const int x = (int)(col / g.Y), y = (int)(col - (int64_t)x * g.Y);
#pragma unroll
        for (int d = 0; d < 4; d += 2) {
            // both antiparallel arcs must stay on the level (z = 0, or a zero interval each way)
            if (zo_of(z, dl_out(g, d)) != z || zo_of(z, dl_in(g, d)) != z) continue;
            const int64_t o = nbr_off(g, x, y, d);
            if (!o || !owned(g, v + o)) continue;
            const int a = s.L[d][v], b = s.L[d ^ 1][v + o];
            const int m = min(a, b);
            if (m > 0) {
                s.L[d][v] = a - m;
                s.L[d ^ 1][v + o] = b - m;
            }
        }
#pragma unroll
        for (int d = 0; d < 4; d += 2) {  // soft arcs with k = 0 stay on the level
            if (!g.soft_k || g.soft_cap[0] <= 0 || dl_out(g, d) < 1 || dl_in(g, d) < 1) continue;
            const int64_t o = nbr_off(g, x, y, d);
            if (!o || !owned(g, v + o)) continue;
            int32_t *fa = soft_flow(g, s, v, d, 0), *fb = soft_flow(g, s, v + o, d ^ 1, 0);
            const int m = min(*fa, *fb);
            if (m > 0) {
                *fa -= m;
                *fb -= m;
            }
        }
    }
}

// vertices still holding excess -> *count
__global__ void k_count_excess(Geo g, const Soa s, unsigned *count) {
    unsigned c = 0;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += (int64_t)gridDim.x * blockDim.x)
        c += s.E[v] != 0;
    c = warp_sum_i((int)c);
    if (lane_id() == 0 && c) atomicAdd(count, c);
}

// out planes (int32[7][n]): s->v, v->t, down v->v-1, lateral +x, -x, +y, -y.  Any vertex left
// with excess sets *bad (the result would not be a flow).
__global__ void k_flow_export(Geo g, const int32_t *__restrict__ in, int weight_mode, const int32_t *__restrict__ band,
                              Soa s, const int32_t *__restrict__ tmp, int32_t *out, int64_t n, int *bad) {
    const int64_t ncol = (int64_t)g.X * g.Y;  // n: plane stride of out (whole volume for in-process slabs)
    bool b = false;
    for (int64_t col = gwarp(); col < ncol; col += nwarps()) {
        const int32_t *cc = in + col * g.Z;
        const ColW cw = col_w_setup(cc, g.Z, band, col, weight_mode);
        for (int z = lane_id(); z < g.Z; z += 32) {
            const int64_t v = col * g.Z + z;
            const long long w = col_w(cc, z, cw, weight_mode);
            const int32_t t0 = w > 0 ? (int32_t)w : 0;
            out[v] = s.T[v];
            out[n + v] = t0 - tmp[v];
            out[2 * n + v] = s.D[v];
#pragma unroll
            for (int d = 0; d < 4; d++) out[(3 + d) * n + v] = s.L[d][v];
            for (int d = 0; d < 4 && g.soft_k; d++)  // soft graphs: planes 7 + d K + k
                for (int k = 0; k < g.soft_k; k++) out[(7 + d * g.soft_k + k) * n + v] = *soft_flow(g, s, v, d, k);
            b |= s.E[v] != 0;
        }
    }
    if (b) atomicOr(bad, 1);
}

// f[lo .. lo+n) = v
template <class F>
__global__ void k_fill(F f, int64_t lo, int64_t n, int32_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        f[lo + i] = v;
}

// out[0 .. n) = f[0 .. n)  (state export to plain planes)
template <class F>
__global__ void k_export(F f, int64_t n, int32_t *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = f[i];
}

// ------------------------------------------------------------------ a3: push-relabel sweep
// An active vertex (E > 0, H < INF) runs Alg. 2: it scans its residual out-arcs and pushes
// delta = min(E, r) (r = INF on infinite arcs) on an admissible arc (neighbour label < own label),
// or relabels to min label(w)+1 ("newd = min label(w)+1 ... only if newd > label(v)").  Default
// scan (CG_SCAN_COL_GATHER, CG_SCAN_UP_EARLY, CG_SCAN_LAT_GATHER) in three rounds
// of independent loads: (1) the own column -- t if T > 0, else down, else up (first admissible in
// that order); (2) the four lateral-out targets, taking the LOWEST-height admissible one; (3) the
// four lateral-in reverse arcs with residual, again the lowest.  Any admissible arc keeps the
// algorithm correct; the order only decides which one is used.
// Lock-free rule: every residual field has one decrementer, so each stale
// read is a lower bound of what the reader may subtract.
struct OpCtx {
    int64_t v, v0, col;
    int z, zo[4], zi[4];  // per direction d: target level of v's lateral arc (dl_out) and source
                          // level of the lateral in-arc (dl_in); -1 = none
    int64_t off[4];  // vertex offset of the neighbour column (0 = none)
};

struct ArcPick {
    int best, arc, res;
    int64_t tgt;
};

// An admissible arc (label < hx) -- in the default build the own-column arcs first (t, down, up),
// then the lowest of the lateral-out targets, then the lowest of the lateral-in reverse arcs (see
// above); if none, the lowest residual neighbour (for the relabel).  CG_SCAN_SERIAL = 0 at compile
// time selects a two-stage gather instead (t, down and lateral-out in one batch of independent
// loads, the reverse arcs in a second; measured within noise).
#ifndef CG_SCAN_SERIAL
#define CG_SCAN_SERIAL 1
#endif
// Soft arcs (NEXT-1) are scanned after every hard arc: arc codes 11 + 16 d + k (forward, v ->
// (nbr_d, z-k), residual cap_k - F) and 75 + 16 d + k (reverse of (nbr_d, z+k)'s arc in direction
// d^1, residual its flow).  Only when no hard arc is admissible, so the hard path is unchanged.
constexpr int ARC_SOFT_FWD = 11, ARC_SOFT_REV = 75;
#ifndef CG_SOFT_GATHER
#define CG_SOFT_GATHER 1
#endif
__device__ __noinline__ void scan_soft(const Geo &g, const Soa &s, const OpCtx &c, int hx, ArcPick &p) {
    for (int d = 0; d < 4; d++) {
        if (!c.off[d]) continue;
        // forward soft arcs of v toward d: k < dl_out(d); reverse of the neighbour's arcs toward d^1: k < dl_in(d)
        const int kf = min(g.soft_k, dl_out(g, d)), kr = min(g.soft_k, dl_in(g, d)), kmax = max(kf, kr);
#if CG_SOFT_GATHER
        // four offsets k at a time: their soft-flow values in one round of loads, then the
        // heights of the targets with residual in another (instead of one dependent chain per arc)
        for (int k0 = 0; k0 < kmax; k0 += 4) {
            int rf[4], rr[4], hf[4], hr[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int k = k0 + j;
                const int cap = k < kmax ? g.soft_cap[k] : 0;
                rf[j] = (cap > 0 && k < kf && c.z - k >= 0) ? cap - *soft_flow(g, s, c.v, d, k) : 0;
                rr[j] = (cap > 0 && k < kr && c.z + k < g.Z) ? *soft_flow(g, s, c.v0 + c.off[d] + c.z + k, d ^ 1, k) : 0;
            }
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int k = k0 + j;
                hf[j] = rf[j] > 0 ? s.H[c.v0 + c.off[d] + c.z - k] : g.INF;
                hr[j] = rr[j] > 0 ? s.H[c.v0 + c.off[d] + c.z + k] : g.INF;
            }
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int k = k0 + j;
                if (hf[j] < p.best) {
                    p.best = hf[j]; p.arc = ARC_SOFT_FWD + 16 * d + k; p.tgt = c.v0 + c.off[d] + c.z - k; p.res = rf[j];
                }
                if (p.best < hx) return;
                if (hr[j] < p.best) {
                    p.best = hr[j]; p.arc = ARC_SOFT_REV + 16 * d + k; p.tgt = c.v0 + c.off[d] + c.z + k; p.res = rr[j];
                }
                if (p.best < hx) return;
            }
        }
#else
        for (int k = 0; k < kmax; k++) {
            const int cap = g.soft_cap[k];
            if (cap <= 0) continue;
            if (k < kf && c.z - k >= 0) {  // forward
                const int r = cap - *soft_flow(g, s, c.v, d, k);
                if (r > 0) {
                    const int64_t t = c.v0 + c.off[d] + c.z - k;
                    const int hh = s.H[t];
                    if (hh < p.best) { p.best = hh; p.arc = ARC_SOFT_FWD + 16 * d + k; p.tgt = t; p.res = r; }
                    if (p.best < hx) return;
                }
            }
            if (k < kr && c.z + k < g.Z) {  // reverse of the arc of u = (nbr_d, z+k) toward this column
                const int64_t u = c.v0 + c.off[d] + c.z + k;
                const int r = *soft_flow(g, s, u, d ^ 1, k);
                if (r > 0) {
                    const int hh = s.H[u];
                    if (hh < p.best) { p.best = hh; p.arc = ARC_SOFT_REV + 16 * d + k; p.tgt = u; p.res = r; }
                    if (p.best < hx) return;
                }
            }
        }
#endif
    }
}

__device__ __forceinline__ ArcPick scan_arcs_hard(const Geo &g, const Soa &s, const OpCtx &c, int hx);
// serial arc-scan order: t, down, up, lateral-out, lateral-in (CG_SCAN_UP_EARLY = 1, measured
// -8 % C4 / -18 % C5) or the up arc after the lateral-out arcs (0)
#ifndef CG_SCAN_UP_EARLY
#define CG_SCAN_UP_EARLY 1
#endif
// lateral records gathered per group (CG_SCAN_LAT_GATHER, measured -1..-8 %);
// own-column checks gathered in one round (CG_SCAN_COL_GATHER)
#ifndef CG_SCAN_LAT_GATHER
#define CG_SCAN_LAT_GATHER 1
#endif
#ifndef CG_SCAN_COL_GATHER
#define CG_SCAN_COL_GATHER 1
#endif
#ifndef CG_SCAN_LAT_ONE
#define CG_SCAN_LAT_ONE 0
#endif
#if CG_SCAN_PROF
// profiling build (`build --scan-prof`): which arc each scan picks (15 = none admissible:
// a relabel), printed to stderr by maxflow_solve
__device__ unsigned long long g_scanprof[16];
#endif
template <bool SOFT>
__device__ __forceinline__ ArcPick scan_arcs(const Geo &g, const Soa &s, const OpCtx &c, int hx) {
    ArcPick p = scan_arcs_hard(g, s, c, hx);
    if (SOFT && p.arc != 0 && p.best >= hx) scan_soft(g, s, c, hx, p);
#if CG_SCAN_PROF
    atomicAdd(&g_scanprof[p.best < hx ? (p.arc < 11 ? p.arc : 11) : 15], 1ull);
#endif
    return p;
}

__device__ __forceinline__ ArcPick scan_arcs_hard(const Geo &g, const Soa &s, const OpCtx &c, int hx) {
    ArcPick p{g.INF, -1, 0, NONE};
#if !CG_SCAN_SERIAL
    const int INF = g.INF;
    const bool dn = c.z >= 1, up = c.z + 1 < g.Z;
    int64_t to[4], ti[4];
    bool oko[4], oki[4];
#pragma unroll
    for (int d = 0; d < 4; d++) {
        oko[d] = c.off[d] && c.zo[d] >= 0;
        oki[d] = c.off[d] && c.zi[d] >= 0;
        to[d] = c.v0 + c.off[d] + c.zo[d];
        ti[d] = c.v0 + c.off[d] + c.zi[d];
    }
    // stage 1: the arcs that are usually admissible (t, down, lateral-out), loaded together
    const int tres = s.T[c.v];
    const int hdn = dn ? s.H[c.v - 1] : INF;
    int hlo[4];
#pragma unroll
    for (int d = 0; d < 4; d++) hlo[d] = oko[d] ? s.H[to[d]] : INF;
    if (tres > 0) {
        p.best = 0; p.arc = 0; p.res = tres;
        return p;
    }
    if (hdn < p.best) { p.best = hdn; p.arc = 1; p.tgt = c.v - 1; }
    if (p.best < hx) return p;
#pragma unroll
    for (int d = 0; d < 4; d++) {
        if (hlo[d] < p.best) { p.best = hlo[d]; p.arc = 2 + d; p.tgt = to[d]; }
        if (p.best < hx) return p;
    }
    // stage 2: reverse residual arcs (up, lateral-in), loaded together
    const int dres = up ? s.D[c.v + 1] : 0;
    const int hup = up ? s.H[c.v + 1] : INF;
    int lres[4], hli[4];
#pragma unroll
    for (int d = 0; d < 4; d++) {
        lres[d] = oki[d] ? s.L[d ^ 1][ti[d]] : 0;
        hli[d] = oki[d] ? s.H[ti[d]] : INF;
    }
    if (dres > 0 && hup < p.best) { p.best = hup; p.arc = 6; p.tgt = c.v + 1; p.res = dres; }
    if (p.best < hx) return p;
#pragma unroll
    for (int d = 0; d < 4; d++) {
        if (lres[d] > 0 && hli[d] < p.best) { p.best = hli[d]; p.arc = 7 + d; p.tgt = ti[d]; p.res = lres[d]; }
        if (p.best < hx) return p;
    }
    return p;
#else
#if CG_SCAN_COL_GATHER && CG_SCAN_UP_EARLY
    {  // own column in one round: t residual, H(v-1), D(v+1) and H(v+1) (adjacent records)
        const int tres = s.T[c.v];
        const int hdn = c.z >= 1 ? s.H[c.v - 1] : g.INF;
        const bool up = c.z + 1 < g.Z;
        const int rup = up ? s.D[c.v + 1] : 0;
        const int hup = up ? s.H[c.v + 1] : g.INF;
        if (tres > 0) {
            p.best = 0; p.arc = 0; p.res = tres;
            return p;
        }
        if (hdn < p.best) { p.best = hdn; p.arc = 1; p.tgt = c.v - 1; }
        if (p.best < hx) return p;
        if (rup > 0 && hup < p.best) { p.best = hup; p.arc = 6; p.tgt = c.v + 1; p.res = rup; }
        if (p.best < hx) return p;
    }
#else
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
#endif
#if CG_SCAN_UP_EARLY && !CG_SCAN_COL_GATHER
    // the up arc's record (v+1) is adjacent to v's own: checked before the lateral records
    if (c.z + 1 < g.Z) {
        const int r = s.D[c.v + 1];
        if (r > 0) {
            const int hh = s.H[c.v + 1];
            if (hh < p.best) { p.best = hh; p.arc = 6; p.tgt = c.v + 1; p.res = r; }
            if (p.best < hx) return p;
        }
    }
#endif
#if CG_SCAN_LAT_GATHER && CG_SCAN_UP_EARLY
    // lateral records: the four lateral-out heights in one round of independent loads, then
    // the four lateral-in (residual, height) pairs in another -- two latency steps instead of
    // up to eight dependent ones for the scans that reach them (relabels: a third of all ops)
    {
        int64_t t4[4];
        int h4[4];
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const bool ok = c.off[d] && c.zo[d] >= 0;
            t4[d] = c.v0 + c.off[d] + c.zo[d];
            h4[d] = ok ? s.H[t4[d]] : g.INF;
        }
#if CG_SCAN_LAT_ONE  // all eight lateral records in one round
        int64_t ti4[4];
        int r4[4], hi4[4];
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const bool ok = c.off[d] && c.zi[d] >= 0;
            ti4[d] = c.v0 + c.off[d] + c.zi[d];
            r4[d] = ok ? s.L[d ^ 1][ti4[d]] : 0;
            hi4[d] = ok ? s.H[ti4[d]] : g.INF;
        }
#endif
#pragma unroll
        for (int d = 0; d < 4; d++)
            if (h4[d] < p.best) { p.best = h4[d]; p.arc = 2 + d; p.tgt = t4[d]; }
        if (p.best < hx) return p;
#if !CG_SCAN_LAT_ONE
        int64_t ti4[4];
        int r4[4], hi4[4];
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const bool ok = c.off[d] && c.zi[d] >= 0;
            ti4[d] = c.v0 + c.off[d] + c.zi[d];
            r4[d] = ok ? s.L[d ^ 1][ti4[d]] : 0;
            hi4[d] = ok ? s.H[ti4[d]] : g.INF;
        }
#endif
#pragma unroll
        for (int d = 0; d < 4; d++)
            if (r4[d] > 0 && hi4[d] < p.best) { p.best = hi4[d]; p.arc = 7 + d; p.tgt = ti4[d]; p.res = r4[d]; }
        return p;
    }
#endif
    if (c.zo[0] >= 0 || c.zo[1] >= 0 || c.zo[2] >= 0 || c.zo[3] >= 0) {
#pragma unroll
        for (int d = 0; d < 4; d++) {
            if (!c.off[d] || c.zo[d] < 0) continue;
            const int64_t t = c.v0 + c.off[d] + c.zo[d];
            const int hh = s.H[t];
            if (hh < p.best) { p.best = hh; p.arc = 2 + d; p.tgt = t; }
            if (p.best < hx) return p;
        }
    }
#if !CG_SCAN_UP_EARLY
    if (c.z + 1 < g.Z) {
        const int r = s.D[c.v + 1];
        if (r > 0) {
            const int hh = s.H[c.v + 1];
            if (hh < p.best) { p.best = hh; p.arc = 6; p.tgt = c.v + 1; p.res = r; }
            if (p.best < hx) return p;
        }
    }
#endif
    if (c.zi[0] >= 0 || c.zi[1] >= 0 || c.zi[2] >= 0 || c.zi[3] >= 0) {
#pragma unroll
        for (int d = 0; d < 4; d++) {
            if (!c.off[d] || c.zi[d] < 0) continue;
            const int64_t u = c.v0 + c.off[d] + c.zi[d];
            const int r = s.L[d ^ 1][u];
            if (r > 0) {
                const int hh = s.H[u];
                if (hh < p.best) { p.best = hh; p.arc = 7 + d; p.tgt = u; p.res = r; }
                if (p.best < hx) return p;
            }
        }
    }
    return p;
#endif
}

__device__ __forceinline__ void set_ctx(const Geo &g, OpCtx &c, int64_t v) {  // v owned (>= 0)
    c.v = v;
    const uint32_t col = CG_DIVZ(g, v);
    c.col = col;
    c.z = (int)((uint32_t)v - col * (uint32_t)g.Z);
    c.v0 = c.col * g.Z;
    const int x = (int)CG_DIVY(g, col), y = (int)(col - (uint32_t)x * (uint32_t)g.Y);
#pragma unroll
    for (int d = 0; d < 4; d++) {
        c.zo[d] = zo_of(c.z, dl_out(g, d));
        c.zi[d] = zi_of(c.z, dl_in(g, d), g.Z);
    }
#pragma unroll
    for (int d = 0; d < 4; d++) c.off[d] = nbr_off(g, x, y, d);
}

// Single push/relabel operation of the owner of c.v; returns the vertex that received
// flow (NONE: none or t; ghost vertices have negative indices).  Decrements follow the
// single-decrementer rule.
template <bool SOFT>
__device__ __forceinline__ int64_t pr_op(const Geo &g, const Soa &s, const OpCtx &c, int &e, int &h, int &sent,
                                         int *flags, unsigned long long &nrel) {
    const ArcPick p = scan_arcs<SOFT>(g, s, c, h);
    if (p.best >= g.INF) {  // no residual path known: dead until the next global relabel
        h = g.INF;
        s.H[c.v] = h;
        nrel++;
        return NONE;
    }
    if (h <= p.best) {  // relabel
        nrel++;
        h = p.best + 1;
        s.H[c.v] = h;
        if (h >= g.INF) return NONE;
    }
    int df;  // push
    switch (p.arc) {
        case 0:
            df = min(e, p.res);
            s.T[c.v] = p.res - df;
            break;
        case 1:
            df = e;
            atomicAdd(&s.D[c.v], df);
            break;
        case 2: case 3: case 4: case 5:
            df = e;
            atomicAdd(&s.L[p.arc - 2][c.v], df);
            break;
        case 6:
            df = min(e, p.res);
            atomicSub(&s.D[c.v + 1], df);
            break;
        case 7: case 8: case 9: case 10:
            df = min(e, p.res);
            atomicSub(&s.L[(p.arc - 7) ^ 1][p.tgt], df);
            break;
        default: {  // soft arcs: this vertex is the only incrementer (forward) / decrementer (reverse)
            df = min(e, p.res);
            if (!SOFT) break;
            if (p.arc < ARC_SOFT_REV) {
                const int a = p.arc - ARC_SOFT_FWD;
                atomicAdd(soft_flow(g, s, c.v, a >> 4, a & 15), df);
            } else {
                const int a = p.arc - ARC_SOFT_REV;
                atomicSub(soft_flow(g, s, p.tgt, (a >> 4) ^ 1, a & 15), df);
            }
            break;
        }
    }
    e -= df;
    sent += df;
    if (p.arc == 0) return NONE;
    const int old = atomicAdd(&s.E[p.tgt], df);
    if (old > INT_MAX - df) atomicOr(flags, FLAG_OVERFLOW);
    return p.tgt;
}

// List an owned vertex for the next sweep (stamp == tag: already listed).  Ghost
// vertices are listed by their owner when the halo delta arrives.
__device__ __forceinline__ void mark_vertex(const Geo &g, int64_t id, int *vstamp, int tag, int *list,
                                            unsigned *count) {
    bool add = owned(g, id) && vstamp[id] != tag;
    if (add) add = atomicExch(&vstamp[id], tag) != tag;
    warp_append(add, (int)id, list, count);
}

// per-sweep counters: work[0] += push/relabel operations (vertex visits), work[1] += relabels
__device__ __forceinline__ void flush_work(unsigned long long *work, unsigned long long ops, unsigned long long rel) {
    ops = warp_sum_ll((long long)ops);
    rel = warp_sum_ll((long long)rel);
    if (lane_id() == 0) {
        if (ops) atomicAdd(work, ops);
        if (rel) atomicAdd(work + 1, rel);
    }
}

template <bool SOFT>
__global__ void __launch_bounds__(256, CG_SWEEP_MINB) k_sweep_v(Geo g, Soa s, int ops, const int *__restrict__ lin,
                                                 const unsigned *cin, int *lout, unsigned *cout, unsigned *czero,
                                                 int *vstamp, int tag, unsigned long long *work, int *flags) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *czero = 0;
    const int64_t count = *cin;
    unsigned long long mywork = 0, myrel = 0;
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
        if (act) set_ctx(g, c, c.v);
        for (int it = 0; it < ops; ++it) {
            int64_t tgt = NONE;
            if (act) {
                mywork++;
                tgt = pr_op<SOFT>(g, s, c, e, h, sent, flags, myrel);
                act = e > 0 && h < g.INF;
            }
            mark_vertex(g, tgt, vstamp, tag, lout, cout);
            if (!__any_sync(FULL, act)) break;
        }
        if (sent) atomicSub(&s.E[c.v], sent);
        mark_vertex(g, act ? c.v : NONE, vstamp, tag, lout, cout);
    }
    flush_work(work, mywork, myrel);
}

// ------------------------------------------------------------------ a3': multi-hop sweep ("walk")
// Alg. 2's discharge applied along a path: the owner of an active vertex v takes all of
// E(v) and carries it down admissible arcs (strictly decreasing labels) for up to K hops,
// pushing delta = min(carry, r) on each arc.  Finite residuals (T, up, lateral-in
// reverse) may now be decremented by several walkers, so they are RESERVED with a CAS
// loop (never negative); infinite arcs only increase the reverse flow (atomicAdd).  A
// carry that cannot go further is deposited (atomicAdd) on the vertex where it stops,
// which is listed for the next launch; a stuck vertex is relabelled monotonically
// (atomicMax).  Excess is decremented only by its owner (the walk start), so
// conservation is exact.  A walk that enters a ghost vertex (neighbour slab) deposits
// there: the halo exchange delivers it to the owner.
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

// raise *p by up to `want` without exceeding cap (several walkers may use the same soft arc)
__device__ __forceinline__ int reserve_up(int32_t *p, int cap, int want) {
    int cur = *(volatile int32_t *)p;
    while (cur < cap) {
        const int take = min(cap - cur, want);
        const int old = atomicCAS(p, cur, cur + take);
        if (old == cur) return take;
        cur = old;
    }
    return 0;
}

__device__ __forceinline__ int walk_push_soft(const Geo &g, const Soa &s, const OpCtx &ctx, const ArcPick &p, int c) {
    if (p.arc < ARC_SOFT_REV) {
        const int a = p.arc - ARC_SOFT_FWD;
        return reserve_up(soft_flow(g, s, ctx.v, a >> 4, a & 15), g.soft_cap[a & 15], c);
    }
    const int a = p.arc - ARC_SOFT_REV;
    return reserve(soft_flow(g, s, p.tgt, (a >> 4) ^ 1, a & 15), c);
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
    if (owned(g, x) && vstamp[x] != tag && atomicExch(&vstamp[x], tag) != tag) {
        const unsigned pos = atomicAdd(&q.n, 1u);
        if (pos < BlockQueue::CAP) q.buf[pos] = (int)x;
        else lout[atomicAdd(cout, 1u)] = (int)x;
    }
}

// Work-fetching walk: a lane whose walk has ended takes the next worklist item itself
// (warp-aggregated atomicAdd on *head), so every iteration of the loop advances 32 independent
// walks by one hop (a warp-per-item walk lasts as long as its longest walk while the lanes whose
// walks ended idle: measured -25 % sweep time per batch).
template <bool SOFT>
__global__ void __launch_bounds__(256, CG_SWEEP_MINB) k_walk_ws(Geo g, Soa s, int K, const int *__restrict__ lin,
                                                     const unsigned *cin, int *lout, unsigned *cout, unsigned *czero,
                                                     int *vstamp, int tag, unsigned long long *work, int *flags,
                                                     unsigned *head) {
    __shared__ BlockQueue q;
    __shared__ unsigned qbase;
    if (threadIdx.x == 0) q.n = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *czero = 0;
    __syncthreads();
    const unsigned count = *cin;
    unsigned long long mywork = 0, myrel = 0;
    bool exhausted = false, walking = false;
    int c = 0, hx = 0, step = 0;
    OpCtx ctx;
    ctx.v = NONE;
    for (;;) {
        // lanes without a walk fetch the next items (one atomic per warp)
        const bool need = !walking && !exhausted;
        const unsigned m = __ballot_sync(FULL, need);
        if (m) {
            unsigned base = 0;
            if (lane_id() == (__ffs(m) - 1)) base = atomicAdd(head, (unsigned)__popc(m));
            base = __shfl_sync(FULL, base, __ffs(m) - 1);
            if (need) {
                const unsigned idx = base + __popc(m & lanemask_lt());
                if (idx >= count) {
                    exhausted = true;
                } else {
                    const int64_t v = lin[idx];
                    c = s.E[v];
                    hx = s.H[v];
                    if (c > 0 && hx < g.INF) {
                        atomicSub(&s.E[v], c);  // the owner takes its whole excess
                        set_ctx(g, ctx, v);
                        step = 0;
                        walking = true;
                    }
                }
            }
        }
        if (!__any_sync(FULL, walking || !exhausted)) break;
        if (!walking) continue;
        // one hop of this lane's walk
        const ArcPick p = scan_arcs<SOFT>(g, s, ctx, hx);
        mywork++;
        if (p.best >= hx || step >= K) {  // stuck (or hop budget spent): deposit the carry here
            if (p.best >= hx) {
                myrel++;
                atomicMax(&s.H[ctx.v], p.best >= g.INF ? g.INF : p.best + 1);
            }
            deposit(g, s, ctx.v, c, vstamp, tag, q, lout, cout, flags);
            walking = false;
            continue;
        }
        ++step;
        int df;
        switch (p.arc) {
            case 0: df = reserve(&s.T[ctx.v], c); break;
            case 1: df = c; atomicAdd(&s.D[ctx.v], df); break;
            case 2: case 3: case 4: case 5: df = c; atomicAdd(&s.L[p.arc - 2][ctx.v], df); break;
            case 6: df = reserve(&s.D[ctx.v + 1], c); break;
            case 7: case 8: case 9: case 10: df = reserve(&s.L[(p.arc - 7) ^ 1][p.tgt], c); break;
            default: df = SOFT ? walk_push_soft(g, s, ctx, p, c) : 0; break;
        }
        if (df == 0) continue;  // lost a reservation race: rescan this vertex
        if (p.arc == 0) {       // absorbed by t
            c -= df;
            if (c == 0) walking = false;
            continue;
        }
        if (df < c) deposit(g, s, ctx.v, c - df, vstamp, tag, q, lout, cout, flags);
        c = df;
        if (!owned(g, p.tgt)) {  // crossed into a neighbour slab: hand the carry over
            deposit(g, s, p.tgt, c, vstamp, tag, q, lout, cout, flags);
            walking = false;
            continue;
        }
        hx = p.best;
        set_ctx(g, ctx, p.tgt);
    }
    __syncthreads();
    const unsigned nq = min(q.n, (unsigned)BlockQueue::CAP);
    if (threadIdx.x == 0 && nq) qbase = atomicAdd(cout, nq);
    __syncthreads();
    for (unsigned j = threadIdx.x; j < nq; j += blockDim.x) lout[qbase + j] = q.buf[j];
    flush_work(work, mywork, myrel);
}

// After a global relabel: list every active vertex (E > 0, H < INF) in index order.
__global__ void k_rebuild_vertices(Geo g, const Soa s, int *lout, unsigned *cout, int *vstamp, int tag,
                                   unsigned long long *active) {
    constexpr int SPAN = 8;
    SpanAppender<SPAN> ap;
    unsigned long long myact = 0;
    for (int64_t base = gwarp() * 32 * SPAN; base < g.n; base += nwarps() * 32 * SPAN) {
#pragma unroll
        for (int j = 0; j < SPAN; j++) {
            const int64_t b0 = base + 32 * j;
            const int64_t v = b0 + lane_id();
            bool a = false;
            if (v < g.n) a = s.E[v] > 0 && s.H[v] < g.INF;
            if (a) vstamp[v] = tag;
            myact += a;
            ap.add(__ballot_sync(FULL, a), b0);
        }
        ap.flush(lout, cout);
    }
    myact = warp_sum_ll((long long)myact);
    if (lane_id() == 0 && myact) atomicAdd(active, myact);
}

// ------------------------------------------------------------------ a2/a5: global relabel
// H(v) = BFS distance from v to t in the residual graph (Alg. 3: level 1 = vertices with a
// residual arc into t -- the "{v,s}" of L414 read as t, R6 -- then level L+1 =
// unlabelled residual predecessors of level L).  Residual in-arcs u -> v of v = (x,y,z):
//   u = (x,y,z+1)             down arc, infinite
//   u = (x,y,z-1)             up arc, residual D(v)
//   u = (nbr, zi(z))          lateral arc of u into v, infinite
//   u = (nbr_d, zo(z))        reverse of v's lateral arc in direction d, residual L_d(v)
// visited: nullable bitmap (1 bit per owned vertex, word = 32 consecutive vertices) written
// whole here -- the persistent BFS claims through it (bfs_expand_multi) so that testing a
// candidate hits an L2-resident word instead of the candidate's DRAM record.
__global__ void k_bfs_init(Geo g, Soa s, int *lout, unsigned *cout, unsigned *visited = nullptr) {
    constexpr int SPAN = 8;
    SpanAppender<SPAN> ap;
    for (int64_t base = gwarp() * 32 * SPAN; base < g.n; base += nwarps() * 32 * SPAN) {
#pragma unroll
        for (int j = 0; j < SPAN; j++) {
            const int64_t b0 = base + 32 * j;
            const int64_t v = b0 + lane_id();
            bool seed = false;
            if (v < g.n) {
                seed = s.T[v] > 0;
                s.H[v] = seed ? 1 : g.INF;
            }
            const unsigned m = __ballot_sync(FULL, seed);
            if (visited && lane_id() == 0 && b0 < g.n) visited[b0 >> 5] = m;
            ap.add(m, b0);
        }
        ap.flush(lout, cout);
    }
}

// Expand one frontier vertex per lane (v < 0: none) and append the new frontier with one
// atomic per warp: claim unlabelled predecessors with atomicCAS(H, INF, L+1) -- each vertex
// exactly once.
// Soft-arc predecessors of v (NEXT-1): w = (nbr_d, z+k) whose forward arc (d^1, k) into v has
// residual, and w = (nbr_d, z-k) through the reverse of v's forward arc (d, k) when it carries
// flow.  WARP-COLLECTIVE: every lane of the warp calls it (v < 0: no vertex); the loop over
// (d, k) is warp-uniform and claims are appended with one atomic per warp (warp_append).
// MODE 0: claim through the visited bitmap (k_bfs_run); 1: CAS on INF labels (k_bfs_step,
// x-slab levels).
template <int MODE>
__device__ __noinline__ void bfs_soft_preds(const Geo &g, const Soa &s, int64_t v, int nl, int *lout, unsigned *cout,
                                            unsigned *visited) {
    const bool has = v >= 0 && nl < g.INF;  // lists hold owned vertices only; -1 = no vertex
    const int64_t col = has ? v / g.Z : 0;
    const int z = has ? (int)(v - col * g.Z) : 0;
    const int x = (int)(col / g.Y), y = (int)(col - (int64_t)x * g.Y);
    const int64_t v0 = col * g.Z;
    auto claim = [&](int64_t w) -> bool {
        if (MODE == 0) {
            const unsigned bit = 1u << (w & 31);
            if ((__ldcg(&visited[w >> 5]) & bit) || (atomicOr(&visited[w >> 5], bit) & bit)) return false;
            s.H[w] = nl;
            return true;
        }
        return __ldcg(&s.H[w]) >= g.INF && atomicCAS(&s.H[w], g.INF, nl) == g.INF;
    };
    for (int d = 0; d < 4; d++) {
        const int64_t o = has ? nbr_off(g, x, y, d) : 0;
        // wu's forward arc (d^1, k) into v exists for k < dl_in(d); v's own arc (d, k) for k < dl_out(d)
        const int kin = min(g.soft_k, dl_in(g, d)), kout = min(g.soft_k, dl_out(g, d));
        const int kmax = max(kin, kout);
        for (int k = 0; k < kmax; k++) {
            const int cap = g.soft_cap[k];
            bool up = false, dn = false;
            const int64_t wu = v0 + o + z + k, wd = v0 + o + z - k;
            if (o && cap > 0) {
                // MODE 1 (strict) also claims ghost vertices: the owner learns the label through
                // the ghost plane; ghosts are never listed here
                up = k < kin && z + k < g.Z && (MODE == 1 || owned(g, wu)) &&
                     cap - *soft_flow(g, s, wu, d ^ 1, k) > 0 && claim(wu) && owned(g, wu);
                dn = k < kout && z - k >= 0 && (MODE == 1 || owned(g, wd)) && *soft_flow(g, s, v, d, k) > 0 &&
                     claim(wd) && owned(g, wd);
            }
            warp_append(up, (int)wu, lout, cout);
            warp_append(dn, (int)wd, lout, cout);
        }
    }
}

__device__ __forceinline__ void bfs_expand_warp(const Geo &g, const Soa &s, int nl, int64_t v, int *lout,
                                                unsigned *cout) {
    const int INF = g.INF;
    int u[10];
    unsigned got = 0;
    if (v >= 0 && nl < INF) {
        const int64_t col = v / g.Z;
        const int z = (int)(v - col * g.Z);
        const int x = (int)(col / g.Y), y = (int)(col - (int64_t)x * g.Y);
        const int64_t v0 = col * g.Z;
        // all candidate predecessors and their labels first (independent loads in flight
        // together), then CAS only the unlabelled ones: one latency chain per vertex
        int w[10];  // vertex indices fit int32 (validate_dims: n + ghosts < 2^31)
        unsigned cand = 0;
        if (z + 1 < g.Z) { w[0] = (int)(v + 1); cand |= 1u; }
        if (z >= 1 && s.D[v] > 0) { w[1] = (int)(v - 1); cand |= 2u; }
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const int64_t o = nbr_off(g, x, y, d);
            if (!o) continue;
            const int zi = zi_of(z, dl_in(g, d), g.Z), zo = zo_of(z, dl_out(g, d));
            if (zi >= 0) { w[2 + d] = (int)(v0 + o + zi); cand |= 1u << (2 + d); }
            if (zo >= 0 && s.L[d][v] > 0) {
                w[6 + d] = (int)(v0 + o + zo);
                cand |= 1u << (6 + d);
            }
        }
        int hw[10];
#pragma unroll
        for (int j = 0; j < 10; j++) hw[j] = (cand >> j & 1u) ? __ldcg(&s.H[w[j]]) : 0;
#pragma unroll
        for (int j = 0; j < 10; j++)
            if ((cand >> j & 1u) && hw[j] >= INF && atomicCAS(&s.H[w[j]], INF, nl) == INF && owned(g, w[j])) {
                // a claimed ghost vertex is not expanded here: its label reaches the owner
                // through the ghost plane (k_slab_ghost_claim) and the owner expands it
                u[j] = w[j];
                got |= 1u << j;
            }
    }
    if (g.soft_k)  // warp-uniform: every lane calls it
        bfs_soft_preds<1>(g, s, v, v >= 0 ? nl : INF, lout, cout, nullptr);
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

// Strict BFS expansion of R frontier vertices per lane at once (vv[r] < 0: none): the R
// vertex records, then all candidate predecessors' labels are loaded before any CAS, so a
// lane pays one dependent-load chain per call instead of R; one append atomic per warp.
__device__ __forceinline__ void load_DL(const Soa &s, int v, int &D, int (&L)[4]) {
#if CG_LAYOUT_AOS
    const int4 *rec = reinterpret_cast<const int4 *>(&s.E[v]);  // E H T D | L0 L1 L2 L3
    const int4 a = rec[0], b = rec[1];
    D = a.w;
    L[0] = b.x; L[1] = b.y; L[2] = b.z; L[3] = b.w;
#else
    D = s.D[v];
#pragma unroll
    for (int d = 0; d < 4; d++) L[d] = s.L[d][v];
#endif
}

// FL (flag-plane BFS, hard graphs): a frontier vertex's in-arc residuals come from its flag byte
// (bit 1: D(v) > 0, bits 2+d: L_d(v) > 0; relabel.cuh k_bfs2_init) instead of its 32-B record, and
// claimed labels go to the label plane `lab` (the records' H is written once by the rebuild): the
// flag plane (1 B / vertex) and the visited bitmap stay L2-resident, so a level touches DRAM only
// for the label stores and the frontier lists.
template <int R, bool FL = false>
__device__ __forceinline__ void bfs_expand_multi(const Geo &g, const Soa &s, int nl, const int (&vv)[R], int *lout,
                                                 unsigned *cout, unsigned *visited, const uint8_t *flags = nullptr,
                                                 int32_t *lab = nullptr) {
    const int INF = g.INF;
    int w[R][10], hw[R][10];
    unsigned cand[R], got[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
        cand[r] = 0;
        got[r] = 0;
        const int v = vv[r];
        if (v < 0 || nl >= INF) continue;
        const int col = (int)CG_DIVZ(g, v);
        const int z = v - col * g.Z;
        const int x = (int)CG_DIVY(g, col), y = col - x * g.Y;
        const int v0 = col * g.Z;
        int D, L[4];
        if (FL) {
            const unsigned f = __ldg(&flags[v]);
            D = f & 2;
#pragma unroll
            for (int d = 0; d < 4; d++) L[d] = f & (4u << d);
        } else {
            load_DL(s, v, D, L);
        }
        if (z + 1 < g.Z) { w[r][0] = v + 1; cand[r] |= 1u; }
        if (z >= 1 && D > 0) { w[r][1] = v - 1; cand[r] |= 2u; }
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const int o = (int)nbr_off(g, x, y, d);
            if (!o) continue;
            const int zi = zi_of(z, dl_in(g, d), g.Z), zo = zo_of(z, dl_out(g, d));
            if (zi >= 0 && owned(g, v0 + o + zi)) { w[r][2 + d] = v0 + o + zi; cand[r] |= 1u << (2 + d); }
            if (zo >= 0 && L[d] > 0 && owned(g, v0 + o + zo)) { w[r][6 + d] = v0 + o + zo; cand[r] |= 1u << (6 + d); }
        }
    }
    // visited words (L2-resident bitmap): hw = 1 if the candidate is already labelled.
    // CG_BFS_PRECHECK = 0 skips this round of loads and lets the atomicOr decide (one L2 round trip
    // less per level, more atomics).
#ifndef CG_BFS_PRECHECK
#define CG_BFS_PRECHECK 1
#endif
#ifndef CG_BFS_ATOM_BATCH
#define CG_BFS_ATOM_BATCH 1
#endif
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int j = 0; j < 10; j++)
            hw[r][j] = (cand[r] >> j & 1u)
                           ? (CG_BFS_PRECHECK ? (int)((__ldcg(&visited[w[r][j] >> 5]) >> (w[r][j] & 31)) & 1u) : 0)
                           : 1;
    if (!FL && g.soft_k && nl < INF)  // warp-uniform: every lane calls it
        for (int r = 0; r < R; r++) bfs_soft_preds<0>(g, s, vv[r], nl, lout, cout, visited);
    int k = 0;
#if CG_BFS_ATOM_BATCH
    // every claim's atomicOr is issued before any label store: a store between two atomics (possibly
    // aliasing in the compiler's view) would make each atomic wait for the previous one's round trip
    unsigned old[R][10];
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int j = 0; j < 10; j++)
            old[r][j] = hw[r][j] ? 0xffffffffu : atomicOr(&visited[w[r][j] >> 5], 1u << (w[r][j] & 31));
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int j = 0; j < 10; j++)
            if (!((old[r][j] >> (w[r][j] & 31)) & 1u)) {  // claimed: this lane owns w's label
                if (FL) lab[w[r][j]] = nl;
                else s.H[w[r][j]] = nl;
                got[r] |= 1u << j;
                k++;
            }
#else
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int j = 0; j < 10; j++)
            if (!hw[r][j]) {
                const unsigned bit = 1u << (w[r][j] & 31);
                if (!(atomicOr(&visited[w[r][j] >> 5], bit) & bit)) {  // claimed: this lane owns w's label
                    if (FL) lab[w[r][j]] = nl;
                    else s.H[w[r][j]] = nl;
                    got[r] |= 1u << j;
                    k++;
                }
            }
#endif
    const int incl = warp_incl_scan(k);
    const int total = __shfl_sync(FULL, incl, 31);
    if (total == 0) return;
    unsigned b = 0;
    if (lane_id() == 31) b = atomicAdd(cout, (unsigned)total);
    b = __shfl_sync(FULL, b, 31);
    unsigned pos = b + incl - k;
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int j = 0; j < 10; j++)
            if (got[r] >> j & 1u) lout[pos++] = w[r][j];
}

// Device-driven strict BFS step (the level counter lives on the device, so identical
// launches are queued back to back).  Step i = level L = i+1 reads list[i&1] / cnt[i%3],
// writes list[(i+1)&1] / cnt[(i+1)%3] and zeroes cnt[(i+2)%3].
//   large frontier: every block expands one level; the last block to finish advances L;
//   small frontier (<= BFS_SMALL): block 0 alone runs levels back to back separated by
//   __syncthreads (a level costs ~1-2 us instead of a launch), until the frontier grows
//   or empties.
constexpr unsigned BFS_SMALL = 2048;       // k_bfs_step (level-per-launch fallback)
constexpr unsigned BFS_RUN_SMALL = 64;    // k_bfs_run default (measured)
struct BfsState {
    int L;                 // current level (1-based)
    unsigned cnt[3];       // frontier counters
    unsigned finished;     // blocks done with the current large level
    unsigned long long claimed;  // vertices labelled so far (direction-optimising switch)
    unsigned bar[3];       // grid barrier of k_bfs_run (arrivals, generation, back-off cap in ns)
    unsigned hist[8];      // levels by frontier size: <=32, <=256, <=2048, <=16K, <=128K, <=1M, more; [7] bottom-up
    unsigned long long cyc[8];  // block-0 clock cycles spent in levels of each bucket ([7]: bottom-up levels)
    unsigned small;             // k_bfs_run: frontiers <= small are run by block 0 alone
    unsigned long long svert;   // vertices expanded in block-0 (small) levels
    // truncated relabel (flag-plane BFS, trunc_levels > 0): after trunc_levels consecutive levels
    // with frontiers <= trunc_small the BFS stops; the vertices it did not reach keep INF ("parked"
    // until the next exhaustive relabel); truncated = 1 when it stopped early
    unsigned trunc_small, trunc_levels, truncated;
    unsigned thin;              // consecutive thin levels, handed from block 0's small-level loop to the grid
    // bottom-up levels of the flag-plane BFS (CG_BFS_BU=div,min): when the frontier exceeds both
    // (vertices not yet labelled) / bu_div and bu_min; 0 = top-down only
    unsigned bu_div, bu_min, bu_levels;
    unsigned conv, dense_levels;  // dense bit-plane levels: list-conversion cursor, levels run dense
};
__device__ __forceinline__ int bfs_bucket(unsigned c) {
    return c <= 32 ? 0 : c <= 256 ? 1 : c <= 2048 ? 2 : c <= 16384 ? 3 : c <= 131072 ? 4 : c <= 1048576 ? 5 : 6;
}

__global__ void k_bfs_seeded(BfsState *st) { st->claimed = st->cnt[0]; }

__global__ void __launch_bounds__(512, CG_BFS_MINB) k_bfs_step(Geo g, Soa s, int *list0, int *list1, BfsState *st) {
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
            if (threadIdx.x == 0) st->claimed += count;
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
            st->claimed += *(volatile unsigned *)&st->cnt[(i + 1) % 3];
            st->L = L + 1;
        }
    }
}

// Persistent strict BFS: ONE cooperative launch runs every level, levels separated by a grid
// barrier instead of a kernel boundary (a level with a small frontier costs a barrier, ~1-2 us,
// instead of a launch and a host round trip every BFS batch).  Same level logic as
// k_bfs_step: small frontiers are run by block 0 alone with block barriers, large ones by
// the whole grid, top-down or bottom-up.  Must be launched with cudaLaunchCooperativeKernel
// (all blocks co-resident).
// bar[2] (nullable 0) caps the pollers' exponential back-off in ns (CG_BAR_NS, default 1024): every
// poller re-reads the generation at most that often after the release.
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned nblocks) {
    // sense-free counting barrier: bar[0] = arrivals, bar[1] = generation
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g0 = *gen;
        const unsigned cap = bar[2] ? bar[2] : 1024u;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            unsigned ns = 32;
            while (*gen == g0) {  // back off: ~300 pollers on one line slow the working blocks
                __nanosleep(ns);
                ns = min(ns * 2, cap);
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// Bottom-up level of the flag-plane BFS (Beamer's direction optimisation) for very large frontiers:
// each word of the visited bitmap (32 consecutive vertices) that still has unvisited vertices is
// taken by one warp, and an unvisited vertex u joins level L+1 if one of its residual out-arcs
// leads to a vertex labelled L -- down (u-1), up (u+1, residual D(u+1) > 0: flag bit 1 of u+1),
// lateral-out (nbr, zo(z)), lateral-in reverse (nbr, zi(z), flag bit 2+(d^1) of that vertex).  The
// labels come from the label plane in coalesced 32-vertex spans (one column per word when Z is a
// multiple of 32), the warp owns its bitmap word (plain store), and a vertex written L+1 here is
// never read as L by another lane.  Neighbour columns in ghost planes are skipped (in-slab BFS).
__device__ void bfs2_bottom_up_level(const Geo &g, const uint8_t *__restrict__ flags, int32_t *lab, unsigned *visited,
                                     int L, int *lout, unsigned *cout) {
    const int64_t nw = (g.n + 31) >> 5;
    for (int64_t w = gwarp(); w < nw; w += nwarps()) {
        const unsigned word = __ldcg(&visited[w]);  // warp-uniform
        if (word == 0xffffffffu) continue;
        const int64_t u = w * 32 + lane_id();
        bool hit = false;
        if (u < g.n && !((word >> lane_id()) & 1u)) {
            const int64_t col = u / g.Z;
            const int z = (int)(u - col * g.Z);
            const int x = (int)(col / g.Y), y = (int)(col - (int64_t)x * g.Y);
            const int64_t v0 = col * g.Z;
            // every candidate's label (and flag) in one round of independent loads
            int ld = -1, lu = -1, lo[4], li[4];
            unsigned fu = 0, fi[4];
            if (z >= 1) ld = __ldcg(&lab[u - 1]);
            if (z + 1 < g.Z) {
                fu = flags[u + 1];
                lu = __ldcg(&lab[u + 1]);
            }
#pragma unroll
            for (int d = 0; d < 4; d++) {
                lo[d] = li[d] = -1;
                fi[d] = 0;
                const int64_t o = nbr_off(g, x, y, d);
                // paths inside this slab only: a ghost column's labels are not this BFS's (on x-slabs
                // the boundary fixpoint brings the cross-slab paths in afterwards)
                if (!o || !owned(g, v0 + o)) continue;
                const int zo = zo_of(z, dl_out(g, d)), zi = zi_of(z, dl_in(g, d), g.Z);
                if (zo >= 0) lo[d] = __ldcg(&lab[v0 + o + zo]);
                if (zi >= 0) {
                    fi[d] = flags[v0 + o + zi];
                    li[d] = __ldcg(&lab[v0 + o + zi]);
                }
            }
            hit = ld == L || ((fu & 2u) && lu == L);
#pragma unroll
            for (int d = 0; d < 4; d++) hit |= lo[d] == L || (((fi[d] >> (2 + (d ^ 1))) & 1u) && li[d] == L);
        }
        const unsigned m = __ballot_sync(FULL, hit);
        if (hit) lab[u] = L + 1;
        if (m && lane_id() == 0) visited[w] = word | m;
        warp_append(hit, (int)u, lout, cout);
    }
}

// Dense bit-plane level of the flag-plane BFS (the large early levels of a relabel; hard graphs on one
// slab with Z % 32 == 0, so a 32-bit word is 32 consecutive z of ONE column).  The same predecessor
// sets as bfs_expand_multi, written as shifts of the frontier's bit words instead of per-vertex
// neighbour lists (the columns' z order makes every arc family a shift):
//   down arc (v+1) -> v, infinite           : u = v + 1                      -> F << 1
//   up arc (v-1) -> v, residual iff D(v) > 0 : u = v - 1                      -> (F & Dm) >> 1
//   lateral arc of u = (nbr_d(v), zi(z)) -> v, infinite: u.z = z + dl_in(d) (z >= 1), 0 (z = 0)
//   reverse of v's lateral arc, residual iff L_d(v) > 0: u = (nbr_d(v), zo(z)): u.z = z - dl_out(d)
//                                            (z > dl_out(d)), 0 (z = 0)
// Seen from u's column, v's column is nbr_{d^1}(u's column).  N = preds(F) & ~visited; each lane owns
// one word of the visited bitmap and of the next frontier bitmap (plain stores, no atomics), and the
// warp writes the labels of its 32 words in coalesced 128-B rows.  The frontier bitmaps are
// double-buffered (Fn is fully rewritten, zeros included).  dl < 32 (checked on the host).
__device__ __forceinline__ unsigned shl_w(unsigned a, unsigned am1, int s) { return s ? (a << s) | (am1 >> (32 - s)) : a; }
__device__ __forceinline__ unsigned shr_w(unsigned a, unsigned ap1, int s) { return s ? (a >> s) | (ap1 << (32 - s)) : a; }

#ifndef CG_DENSE_R
#define CG_DENSE_R 1
#endif
#ifndef CG_DENSE_ROWS_ALL  // words with new vertices from which the label rows are written unrolled
#define CG_DENSE_ROWS_ALL 12
#endif
__device__ void bfs_dense_level(const Geo &g, const unsigned *__restrict__ Dm, const unsigned *__restrict__ Lm,
                                int64_t NW, const unsigned *F, unsigned *Fn, unsigned *visited, int32_t *lab, int nl,
                                unsigned *cout) {
    constexpr int R = CG_DENSE_R;  // words per lane, every load of the R words issued before any use
                                   // (measured: R = 1 / 2 / 3 equal or worse)
    const int WPC = g.Z >> 5;
    const int64_t nw = g.n >> 5;
    unsigned tot = 0;
    for (int64_t base = gwarp() * 32 * R; base < nw; base += nwarps() * 32 * R) {
        unsigned vis[R], f0[R], fm[R], fp[R], d0[R], dp[R], a0[R][4], am[R][4], ap[R][4], l0[R][4], lp[R][4];
        int kk[R];
        unsigned on[R];  // bit d: the neighbour column toward d^1 exists
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int64_t w = base + r * 32 + lane_id();
            on[r] = 0;
            kk[r] = 0;
            vis[r] = 0xffffffffu;
            f0[r] = fm[r] = fp[r] = d0[r] = dp[r] = 0;
#pragma unroll
            for (int d = 0; d < 4; d++) a0[r][d] = am[r][d] = ap[r][d] = l0[r][d] = lp[r][d] = 0;
            if (w >= nw) continue;
            const uint32_t col = CG_DIVZ(g, (uint32_t)w * 32u);  // 32-bit indices, as in bfs_expand_multi
            const int k = (int)((uint32_t)w - col * (uint32_t)WPC);
            kk[r] = k;
            const int x = (int)CG_DIVY(g, col), y = (int)(col - (uint32_t)x * (uint32_t)g.Y);
            const bool hasm = k > 0, hasp = k + 1 < WPC;
            vis[r] = __ldcg(&visited[w]);
            f0[r] = __ldcg(&F[w]);
            if (hasm) fm[r] = __ldcg(&F[w - 1]);
            if (hasp) fp[r] = __ldcg(&F[w + 1]);
            d0[r] = __ldg(&Dm[w]);
            if (hasp) dp[r] = __ldg(&Dm[w + 1]);
#pragma unroll
            for (int d = 0; d < 4; d++) {
                const int64_t o = nbr_off(g, x, y, d ^ 1);  // v's column, seen from u's
                if (!o) continue;
                on[r] |= 1u << d;
                const int64_t wv = w + o / 32;
                a0[r][d] = __ldcg(&F[wv]);
                if (hasm) am[r][d] = __ldcg(&F[wv - 1]);
                if (hasp) ap[r][d] = __ldcg(&F[wv + 1]);
                l0[r][d] = __ldg(&Lm[d * NW + wv]);
                if (hasp) lp[r][d] = __ldg(&Lm[d * NW + wv + 1]);
            }
        }
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int64_t w = base + r * 32 + lane_id();
            unsigned N = shl_w(f0[r], fm[r], 1) | shr_w(f0[r] & d0[r], fp[r] & dp[r], 1);
            const bool first = kk[r] == 0;
#pragma unroll
            for (int d = 0; d < 4; d++) {
                if (!((on[r] >> d) & 1u)) continue;
                const int si = dl_in(g, d), so = dl_out(g, d);
                // infinite lateral arcs into v: from v.z >= 1 shifted up by si; v.z = 0 -> u.z = 0
                unsigned t = shl_w(a0[r][d], am[r][d], si);
                if (first) t = (t & ~(1u << si)) | (a0[r][d] & 1u);
                N |= t;
                // reverse lateral arcs (L_d(v) > 0): v.z > so shifted down by so; v.z = 0 -> u.z = 0
                unsigned g0 = a0[r][d] & l0[r][d];
                if (first) {
                    N |= g0 & 1u;
                    g0 &= so >= 31 ? 0u : ~((2u << so) - 1u);
                }
                N |= shr_w(g0, ap[r][d] & lp[r][d], so);
            }
            N &= ~vis[r];
            if (w < nw) {
                if (N) visited[w] = vis[r] | N;
                Fn[w] = N;
            }
            tot += __popc(N);
            unsigned m = __ballot_sync(FULL, N != 0);
            // labels of the new vertices, one coalesced row per word; streaming stores (evict-first in
            // L2: the label plane is 4 B/vertex and must not push the bit planes out of L2)
            int32_t *row = lab + (base + r * 32) * 32 + lane_id();
            if (__popc(m) >= CG_DENSE_ROWS_ALL) {
#pragma unroll
                for (int j = 0; j < 32; j++) {
                    const unsigned Nj = __shfl_sync(FULL, N, j);
                    if ((Nj >> lane_id()) & 1u) __stcs(row + j * 32, nl);
                }
            } else {
                while (m) {
                    const int j = __ffs(m) - 1;
                    m &= m - 1;
                    const unsigned Nj = __shfl_sync(FULL, N, j);
                    if ((Nj >> lane_id()) & 1u) __stcs(row + j * 32, nl);
                }
            }
        }
    }
    tot = (unsigned)warp_sum_ll((long long)tot);
    if (lane_id() == 0 && tot) atomicAdd(cout, tot);
}

// List the vertices of a frontier bitmap (the switch from dense to list levels), 32 words per warp.
__device__ void bfs_dense_list(const Geo &g, const unsigned *F, int *lout, unsigned *cout) {
    const int64_t nw = g.n >> 5;
    for (int64_t base = gwarp() * 32; base < nw; base += nwarps() * 32) {
        const int64_t w = base + lane_id();
        const unsigned N = w < nw ? __ldcg(&F[w]) : 0u;
        const int c = __popc(N);
        const int incl = warp_incl_scan(c);
        const int total = __shfl_sync(FULL, incl, 31);
        if (!total) continue;
        unsigned b = 0;
        if (lane_id() == 31) b = atomicAdd(cout, (unsigned)total);
        b = __shfl_sync(FULL, b, 31);
        unsigned pos = b;
        unsigned m = __ballot_sync(FULL, N != 0);
        while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            const unsigned Nj = __shfl_sync(FULL, N, j);
            if ((Nj >> lane_id()) & 1u) lout[pos + __popc(Nj & lanemask_lt())] = (int)((base + j) * 32 + lane_id());
            pos += __popc(Nj);
        }
    }
}

#ifndef BFS_R
#define BFS_R 2
#endif
#ifndef CG_BFS_RUN_MINB
#define CG_BFS_RUN_MINB 1
#endif
template <bool FL>
__global__ void __launch_bounds__(512, CG_BFS_RUN_MINB) k_bfs_run(Geo g, Soa s, int *list0, int *list1, BfsState *st,
                                                                  unsigned *visited, const uint8_t *flags,
                                                                  int32_t *lab, unsigned *dbits, unsigned dense_min) {
    unsigned *bar = st->bar;
    int L = *(volatile int *)&st->L;
    unsigned long long claimed = *(volatile unsigned long long *)&st->claimed;
    const unsigned tr_small = st->trunc_small, tr_levels = FL ? st->trunc_levels : 0;
    unsigned thin = 0;  // consecutive levels with a frontier <= tr_small
    // dense bit-plane levels (bfs_dense_level) while the frontier has >= dense_min vertices, from level 1
    // on: dbits = [Dm | Lm0..3 | F0 | F1], NW words each (k_bfs2_init wrote Dm, Lm and F0 = the seeds)
    bool dense = FL && dbits && dense_min && L == 1;
    bool dense_ran = false;
    int fcur = 0;
    const int64_t NW = g.n / 32 + 1;
    for (int guard = 0; guard <= g.INF + 2; guard++) {
        const unsigned count = *(volatile unsigned *)&st->cnt[(L - 1) % 3];
        if (count == 0) break;
        thin = count <= tr_small ? thin + 1 : 0;
        if (tr_levels && thin > tr_levels) {  // the thin tail is deferred (every block sees the same counts)
            if (blockIdx.x == 0 && threadIdx.x == 0) st->truncated = 1;
            break;
        }
        const int i = L - 1;
        if (dense) {
            unsigned *F = dbits + (5 + fcur) * NW;
            if (count >= dense_min) {
                if (blockIdx.x == 0 && threadIdx.x == 0) {
                    st->cnt[(i + 2) % 3] = 0;
                    st->hist[bfs_bucket(count)]++;
                    st->dense_levels++;
                }
                const long long t0 = clock64();
                bfs_dense_level(g, dbits, dbits + NW, NW, F, dbits + (6 - fcur) * NW, visited, lab, L + 1,
                                &st->cnt[(i + 1) % 3]);
                grid_barrier(bar, gridDim.x);
                if (blockIdx.x == 0 && threadIdx.x == 0) st->cyc[bfs_bucket(count)] += clock64() - t0;
                fcur ^= 1;
                dense_ran = true;
                ++L;
                claimed += *(volatile unsigned *)&st->cnt[(L - 1) % 3];
                continue;
            }
            dense = false;
            if (dense_ran) {  // this level's frontier exists only as the bitmap F: list it
                bfs_dense_list(g, F, (i & 1) ? list1 : list0, &st->conv);
                grid_barrier(bar, gridDim.x);
            }
        }
        if (count <= st->small) {
            // everyone has read this level's counter before block 0 starts recycling counters
            grid_barrier(bar, gridDim.x);
            if (blockIdx.x == 0) {
                if (threadIdx.x == 0) st->claimed = claimed;
                unsigned c = count;
                const long long t0 = clock64();
                for (;;) {
                    const int j = L - 1;
                    int *lin = (j & 1) ? list1 : list0;
                    int *lout = (j & 1) ? list0 : list1;
                    if (threadIdx.x == 0) {
                        st->cnt[(j + 2) % 3] = 0;
                        st->hist[bfs_bucket(c)]++;
                        st->svert += c;
                    }
                    for (unsigned base = (threadIdx.x >> 5) * 32 * BFS_R; base < c;
                         base += (blockDim.x >> 5) * 32 * BFS_R) {
                        int vv[BFS_R];
#pragma unroll
                        for (int r = 0; r < BFS_R; r++) {
                            const unsigned jj = base + r * 32 + lane_id();
                            vv[r] = jj < c ? __ldcg(&lin[jj]) : -1;
                        }
                        bfs_expand_multi<BFS_R, FL>(g, s, L + 1, vv, lout, &st->cnt[(j + 1) % 3], visited, flags, lab);
                    }
                    __syncthreads();
                    ++L;
                    c = *(volatile unsigned *)&st->cnt[(L - 1) % 3];
                    if (threadIdx.x == 0) st->claimed += c;
                    __syncthreads();
                    if (c == 0 || c > st->small) break;
                    if (tr_levels && c <= tr_small && thin + 1 > tr_levels) break;  // the grid loop stops
                    thin = c <= tr_small ? thin + 1 : 0;
                }
                if (threadIdx.x == 0) {
                    st->L = L;
                    st->thin = thin;
                    st->cyc[2] += clock64() - t0;  // small levels, accounted to the <=2K bucket
                }
            }
            grid_barrier(bar, gridDim.x);
            L = *(volatile int *)&st->L;
            thin = *(volatile unsigned *)&st->thin;  // every block continues from block 0's count
            claimed = *(volatile unsigned long long *)&st->claimed;
            continue;
        }
        const int *lin = (i & 1) ? list1 : list0;
        int *lout = (i & 1) ? list0 : list1;
        // the counter of level L+1 was read by everyone before the previous barrier
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->cnt[(i + 2) % 3] = 0;
            st->hist[bfs_bucket(count)]++;
        }
        const long long t0 = clock64();
        const unsigned long long unvisited = (unsigned long long)g.n - claimed;
        if (FL && st->bu_div && count >= st->bu_min && (unsigned long long)count * st->bu_div >= unvisited) {
            if (blockIdx.x == 0 && threadIdx.x == 0) st->bu_levels++;
            bfs2_bottom_up_level(g, flags, lab, visited, L, lout, &st->cnt[(i + 1) % 3]);
        } else {
            // few vertices per warp: spread them (R = 1); many: R per lane for load-level parallelism
            if ((int64_t)count < nwarps() * 32 * BFS_R) {
                for (int64_t base = gwarp() * 32; base < count; base += nwarps() * 32) {
                    const int64_t j = base + lane_id();
                    int vv[1] = {j < count ? __ldcg(&lin[j]) : -1};
                    bfs_expand_multi<1, FL>(g, s, L + 1, vv, lout, &st->cnt[(i + 1) % 3], visited, flags, lab);
                }
            } else {
                for (int64_t base = gwarp() * 32 * BFS_R; base < count; base += nwarps() * 32 * BFS_R) {
                    int vv[BFS_R];
#pragma unroll
                    for (int r = 0; r < BFS_R; r++) {
                        const int64_t j = base + r * 32 + lane_id();
                        vv[r] = j < count ? __ldcg(&lin[j]) : -1;
                    }
                    bfs_expand_multi<BFS_R, FL>(g, s, L + 1, vv, lout, &st->cnt[(i + 1) % 3], visited, flags, lab);
                }
            }
        }
        grid_barrier(bar, gridDim.x);
        if (blockIdx.x == 0 && threadIdx.x == 0) st->cyc[bfs_bucket(count)] += clock64() - t0;
        ++L;
        claimed += *(volatile unsigned *)&st->cnt[(L - 1) % 3];  // every block: same value
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->L = L;
        st->claimed = claimed;
    }
}

// Level-synchronous x-slab BFS (a5 across slabs): expand level L's frontier (labels nl = L+1
// for unlabelled predecessors, ghost predecessors included -- their CAS marks the ghost plane,
// which k_slab_ghost_claim delivers to the owner before level L+1 starts).
__global__ void __launch_bounds__(256) k_slab_level(Geo g, Soa s, int nl, const int *__restrict__ lin,
                                                    const unsigned *cin, int *lout, unsigned *cout, unsigned *czero) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *czero = 0;
    const int64_t count = *cin;
    for (int64_t base = gwarp() * 32; base < count; base += nwarps() * 32) {
        const int64_t j = base + lane_id();
        bfs_expand_warp(g, s, nl, j < count ? (int64_t)lin[j] : -1, lout, cout);
    }
}
// ghost-plane labels of this slab (both sides, one launch) -> the owners of those vertices
__global__ void k_ghost_pack_h(Geo g, Soa s, int32_t *send0, int32_t *send1) {
    const int64_t m = (int64_t)(g.gl + g.gh) * g.YZ;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const bool hi = !g.gl || t >= g.YZ;
        const int64_t i = t - (g.gl && hi ? g.YZ : 0);
        (hi ? send1 : send0)[i] = s.H[(hi ? g.n : -g.YZ) + i];
    }
}
// owner side: a boundary vertex a neighbour claimed at label nl this level joins the next
// frontier unless this slab already labelled it (then its own label is <= nl)
__global__ void k_slab_ghost_claim(Geo g, Soa s, const int32_t *__restrict__ recv0, const int32_t *__restrict__ recv1,
                                   int nl, int *lout, unsigned *cout) {
    const int64_t m = (int64_t)(g.gl + g.gh) * g.YZ;
    for (int64_t b0 = gwarp() * 32; b0 < m; b0 += nwarps() * 32) {
        const int64_t t = b0 + lane_id();
        const bool hi = !g.gl || t >= g.YZ;
        const int64_t i = t - (g.gl && hi ? g.YZ : 0);
        const int64_t v = (hi ? g.n - g.YZ : 0) + i;
        bool add = false;
        if (t < m && (hi ? recv1 : recv0)[i] == nl)
            add = s.H[v] >= g.INF && atomicCAS(&s.H[v], g.INF, nl) == g.INF;
        warp_append(add, (int)v, lout, cout);
    }
}

// ------------------------------------------------------------------ a8: halo exchange (x-slabs)
// Per side (0: x = -1 ghost / x = 0 boundary; 1: x = X ghost / x = X-1 boundary) one
// message of 4 planes of Y*Z int32:
//   [0] dE : excess pushed into the ghost plane since the last exchange
//   [1] dL : decrements of the ghost's lateral residual toward this slab (snapshot - now)
//   [2] H  : heights of the boundary plane
//   [3] L  : the boundary plane's lateral flow toward the neighbour (its ghost residual)
// The receiver adds dE, subtracts dL (it is the single decrementer's delta), lists the
// vertices that received excess, and refreshes its ghost plane with H and L - (its own dL).
// Soft graphs add 2 K planes: [4 YZ + i K + k] the consumed part of the ghost copy of the
// neighbour's soft flows toward us (its reverse arcs were used here), [4 YZ + YZ K + i K + k]
// this slab's boundary soft flows toward the neighbour (refreshes its ghost copy).  Same rule
// as L: a flow lives at its tail, the other side only decrements a lower-bound copy.
__global__ void k_halo_pack(Geo g, Soa s, int side, const int32_t *__restrict__ snap, const int32_t *__restrict__ ssnap,
                            int32_t *send) {
    const int64_t gbase = side ? g.n : -g.YZ, bbase = side ? g.n - g.YZ : 0;
    const int gdir = side ? 1 : 0, bdir = side ? 0 : 1;
    const int K = g.soft_k;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.YZ; i += (int64_t)gridDim.x * blockDim.x) {
        send[i] = s.E[gbase + i];
        send[g.YZ + i] = snap[i] - s.L[gdir][gbase + i];
        send[2 * g.YZ + i] = s.H[bbase + i];
        send[3 * g.YZ + i] = s.L[bdir][bbase + i];
        for (int k = 0; k < K; k++) {
            send[4 * g.YZ + i * K + k] = ssnap[i * K + k] - *soft_flow(g, s, gbase + i, gdir, k);
            send[4 * g.YZ + g.YZ * K + i * K + k] = *soft_flow(g, s, bbase + i, bdir, k);
        }
    }
}

__global__ void k_halo_unpack(Geo g, Soa s, int side, const int32_t *__restrict__ recv,
                              const int32_t *__restrict__ sent, int32_t *snap, int32_t *ssnap, int *lout,
                              unsigned *cout, int *vstamp, int tag, int *flags) {
    const int64_t gbase = side ? g.n : -g.YZ, bbase = side ? g.n - g.YZ : 0;
    const int gdir = side ? 1 : 0, bdir = side ? 0 : 1;
    for (int64_t b0 = gwarp() * 32; b0 < g.YZ; b0 += nwarps() * 32) {
        const int64_t i = b0 + lane_id();
        bool add = false;
        if (i < g.YZ) {
            const int64_t bv = bbase + i, gv = gbase + i;
            const int de = recv[i];
            if (de) {
                const long long ne = (long long)s.E[bv] + de;
                if (ne > INT_MAX) atomicOr(flags, FLAG_OVERFLOW);
                s.E[bv] = (int32_t)ne;
                add = vstamp[bv] != tag;
                if (add) vstamp[bv] = tag;
            }
            s.L[bdir][bv] -= recv[g.YZ + i];
            s.H[gv] = recv[2 * g.YZ + i];
            const int lg = recv[3 * g.YZ + i] - sent[g.YZ + i];
            s.L[gdir][gv] = lg;
            snap[i] = lg;
            s.E[gv] = 0;
            const int K = g.soft_k;
            for (int k = 0; k < K; k++) {
                *soft_flow(g, s, bv, bdir, k) -= recv[4 * g.YZ + i * K + k];
                const int fg = recv[4 * g.YZ + g.YZ * K + i * K + k] - sent[4 * g.YZ + i * K + k];
                *soft_flow(g, s, gv, gdir, k) = fg;
                ssnap[i * K + k] = fg;
            }
        }
        warp_append(add, (int)(bbase + i), lout, cout);
    }
}

// Global-relabel halo: heights of the boundary plane -> the neighbour's ghost plane
// (the previous ghost heights are kept in old[] to detect improvements).
__global__ void k_halo_pack_h(Geo g, Soa s, int side, int32_t *send) {
    const int64_t bbase = side ? g.n - g.YZ : 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.YZ; i += (int64_t)gridDim.x * blockDim.x)
        send[i] = s.H[bbase + i];
}
__global__ void k_halo_unpack_h(Geo g, Soa s, int side, const int32_t *__restrict__ recv, int32_t *old) {
    const int64_t gbase = side ? g.n : -g.YZ;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.YZ; i += (int64_t)gridDim.x * blockDim.x) {
        old[i] = s.H[gbase + i];
        s.H[gbase + i] = recv[i];
    }
}

// ------------------------------------------------------------------ a5: gap heuristic
// Cherkassky-Goldberg gap: if no vertex has label g (0 < g < max
// finite label), every vertex labelled above g cannot reach t: lift it to INF.
constexpr int GAP_BINS = 1 << 20;
// Label histogram: a block-private shared-memory histogram of the labels < GAP_SMEM (one global
// atomic per non-empty bin per block afterwards); larger labels go straight to global memory.  A
// global atomic per vertex serialised on the few hundred busy bins (measured: ~10 ms per C4 pass).
constexpr int GAP_SMEM = 8192;
__global__ void __launch_bounds__(512) k_gap_hist(Geo g, const FieldH H, unsigned *hist, int *maxh) {
    __shared__ unsigned sh[GAP_SMEM];
    for (int i = threadIdx.x; i < GAP_SMEM; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    int mymax = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int h = H[i];
        if (h < g.INF) {
            mymax = max(mymax, h);
            if (h < GAP_SMEM) atomicAdd(&sh[h], 1u);
            else if (h < GAP_BINS) atomicAdd(&hist[h], 1u);
        }
    }
    mymax = warp_max_i(mymax);
    if (lane_id() == 0) atomicMax(maxh, mymax);
    __syncthreads();
    for (int i = threadIdx.x; i < GAP_SMEM; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}
// in-process slabs: dst histogram += src histogram, dst max = max(dst, src)
__global__ void k_hist_fold(const unsigned *src, const int *src_max, unsigned *dst, int *dst_max) {
    const int lim = min(*src_max + 1, GAP_BINS);
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < lim; h += gridDim.x * blockDim.x)
        if (src[h]) dst[h] += src[h];
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicMax(dst_max, *src_max);
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
__global__ void k_gap_lift(Geo g, FieldH H, const int *gap, unsigned long long *lifted) {
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
__global__ void k_sum_T(Geo g, const Field T, unsigned long long *out) {
    long long acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (int64_t)gridDim.x * blockDim.x)
        acc += T[i];
    acc = warp_sum_ll(acc);
    if (lane_id() == 0 && acc) atomicAdd(out, (unsigned long long)acc);
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
        long long ab_below = 0;
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

// ------------------------------------------------------------------ a7: extraction
// Minimal source set S = forward residual closure of {v : E(v) > 0} (R5,
// SURVEY.md V3).  Infinite down arcs make S downward closed per column, so S is
// top(x,y) = max{z : (x,y,z) in S}.  Worklist closure over columns: proc(col) is the
// highest z whose out-arcs were already scanned; a listed column scans (proc, top]:
//   up arcs        climb while D(top+1) > 0
//   lateral-out    top(nbr) >= zo_eff(top) = max(0, top - Delta)
//   lateral-in rev top(nbr_d) >= zi(z) for z in (proc, top] with L_{d^1}(nbr_d, zi(z)) > 0
// A neighbour whose top rises is listed for the next round; a ghost column's rise is
// delivered to its owner by the top halo (k_top_halo_*).  top[] is indexed by column with
// the ghost columns at [-Y, 0) and [ncol, ncol + Y).
__device__ __forceinline__ int warp_climb(const Geo &g, const Field D, int64_t v0, int t) {
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
    const int64_t ncols = (int64_t)g.X * g.Y;
    for (int64_t i = gwarp(); i < count; i += nwarps()) {
        const int64_t col = lin[i];
        const int p = proc[col];
        int t = *(volatile int32_t *)&top[col];
        if (t <= p) continue;
        const int64_t v0 = col * g.Z;
        const int x = (int)(col / g.Y), y = (int)(col - (int64_t)x * g.Y);
        t = warp_climb(g, s.D, v0, t);
        if (lane_id() == 0) atomicMax(&top[col], t);
        int64_t nc[4];
        nc[0] = (x + 1 < g.X || g.gh) ? col + g.Y : INT64_MIN;
        nc[1] = (x >= 1 || g.gl) ? col - g.Y : INT64_MIN;
        nc[2] = y + 1 < g.Y ? col + 1 : INT64_MIN;
        nc[3] = y >= 1 ? col - 1 : INT64_MIN;
        int cd[4] = {-1, -1, -1, -1};
        for (int zb = p + 1; zb <= t; zb += 32) {
            const int z = zb + lane_id();
#pragma unroll
            for (int d = 0; d < 4; d++) {
                const int zi = z <= t ? zi_of(z, dl_in(g, d), g.Z) : -1;
                if (zi >= 0 && nc[d] != INT64_MIN && s.L[d ^ 1][nc[d] * g.Z + zi] > 0) cd[d] = max(cd[d], zi);
            }
            if (g.soft_k && z <= t)  // soft arcs with residual (NEXT-1)
                for (int d = 0; d < 4; d++) {
                    if (nc[d] == INT64_MIN) continue;
                    const int kout = min(g.soft_k, dl_out(g, d)), kin = min(g.soft_k, dl_in(g, d));
                    for (int k = 0; k < max(kout, kin); k++) {
                        const int cap = g.soft_cap[k];
                        if (cap <= 0) continue;
                        if (k < kout && z - k >= 0 && cap - *soft_flow(g, s, v0 + z, d, k) > 0) cd[d] = max(cd[d], z - k);
                        if (k < kin && z + k < g.Z && *soft_flow(g, s, nc[d] * g.Z + z + k, d ^ 1, k) > 0)
                            cd[d] = max(cd[d], z + k);
                    }
                }
        }
        int mark = -1;
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const int zout = t > dl_out(g, d) ? t - dl_out(g, d) : 0;
            const int cand = max(warp_max_i(cd[d]), zout);
            if (lane_id() == d && nc[d] != INT64_MIN) {
                const int old = atomicMax(&top[nc[d]], cand);
                if (old < cand && nc[d] >= 0 && nc[d] < ncols) mark = (int)nc[d];
            }
        }
        warp_mark(mark, stamp, tag, lout, cout);
        if (lane_id() == 0) proc[col] = t;
    }
}

// a4 by the source side: after the closure rounds, is there a vertex in S = {z <= top(x,y)} with a
// residual arc into t (T > 0)?  None <=> no vertex with excess can reach t <=> the preflow is
// maximum (Theorem 1).  Warp per column.
__global__ void k_ext_check_t(Geo g, const Soa s, const int32_t *__restrict__ top, int *hit) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    for (int64_t col = gwarp(); col < ncol; col += nwarps()) {
        const int t = top[col];
        bool h = false;
        for (int z = lane_id(); z <= t; z += 32) h |= s.T[col * g.Z + z] > 0;
        if (__any_sync(FULL, h)) {
            if (lane_id() == 0) atomicOr(hit, 1);
            return;
        }
    }
}

// Top halo: [0] this slab's proposals for the ghost columns, [1] its boundary tops.
__global__ void k_top_halo_pack(Geo g, const int32_t *top, int side, int32_t *send) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    const int64_t gbase = side ? ncol : -g.Y, bbase = side ? ncol - g.Y : 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.Y; i += gridDim.x * blockDim.x) {
        send[i] = top[gbase + i];
        send[g.Y + i] = top[bbase + i];
    }
}
__global__ void k_top_halo_unpack(Geo g, int32_t *top, int side, const int32_t *__restrict__ recv,
                                  const int32_t *__restrict__ sent, int *lout, unsigned *cout, int *stamp, int tag,
                                  unsigned *changed) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    const int64_t gbase = side ? ncol : -g.Y, bbase = side ? ncol - g.Y : 0;
    for (int64_t b0 = gwarp() * 32; b0 < g.Y; b0 += nwarps() * 32) {
        const int64_t i = b0 + lane_id();
        bool add = false;
        if (i < g.Y) {
            const int prop = recv[i];
            if (prop > top[bbase + i]) {
                top[bbase + i] = prop;
                add = stamp[bbase + i] != tag;
                if (add) stamp[bbase + i] = tag;
                atomicAdd(changed, 1u);
            }
            top[gbase + i] = max(recv[g.Y + i], sent[i]);
        }
        warp_append(add, (int)(bbase + i), lout, cout);
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
