// chunk.cuh -- column-chunk sweep (measured alternative to the vertex-worklist walks; SURVEY.md §8(a)
// a3: "a warp owns 32 consecutive z of one column"; round-1 verdict item 3).
//
// One warp per listed chunk (32 consecutive z of one column, lane = z offset).  The chunk's 32
// records are loaded coalesced (two int4 per lane = one 1-KB span), the neighbour data once per
// visit as coalesced spans (the four lateral-out targets (nbr, zo(z)) and the four lateral-in
// sources (nbr, zi(z)) are 32 consecutive records of the neighbour column each), z +- 1 comes from
// shuffles.  The warp then runs up to `rounds` synchronous push/relabel rounds on the registers
// (Alg. 2's operation per active vertex per round, same arc order as the vertex sweeps: t, down, up,
// lowest lateral-out, lowest lateral-in), so excess moves along the column inside one visit;
// lateral pushes and pushes across the chunk ends go out with atomics and list the target chunk.
// Write-back is by deltas (atomicAdd) for the fields other warps also change (E, D, L), plain
// stores for T and H (single writer).  Single-decrementer rule as in DESIGN.md §7: the residuals
// this warp consumes (T, D of the chunk above's lowest vertex, L of the lateral-in sources) have no
// other decrementer, so the values loaded at the start are lower bounds.
#pragma once

#include "kernels.cuh"

namespace cg {

// After a global relabel: list every chunk holding an active vertex (E > 0, H < INF).
__global__ void k_chunk_rebuild(Geo g, const Soa s, int *lout, unsigned *cout, int *cstamp, int tag) {
    for (int64_t base = gwarp() * 32; base < g.nchunks; base += nwarps() * 32) {
        unsigned mine = 0;  // bit k: chunk base + k is active
        for (int k = 0; k < 32; k++) {
            const int64_t ch = base + k;
            if (ch >= g.nchunks) break;
            const int64_t col = ch / g.CPC;
            const int z = (int)(ch - col * g.CPC) * 32 + lane_id();
            bool a = false;
            if (z < g.Z) {
                const int64_t v = col * g.Z + z;
                a = s.E[v] > 0 && s.H[v] < g.INF;
            }
            if (__any_sync(FULL, a)) mine |= 1u << k;
        }
        const bool has = (mine >> lane_id()) & 1u;
        if (has) cstamp[base + lane_id()] = tag;
        warp_append(has, (int)(base + lane_id()), lout, cout);
    }
}

__global__ void __launch_bounds__(256) k_chunk_sweep(Geo g, Soa s, int rounds, const int *__restrict__ lin,
                                                     const unsigned *cin, int *lout, unsigned *cout, unsigned *czero,
                                                     int *cstamp, int tag, unsigned long long *work,
                                                     unsigned long long *visits, int *flags) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *czero = 0;
    const int64_t count = *cin;
    const int lane = lane_id();
    const int INF = g.INF;
    unsigned long long mywork = 0, myrel = 0, myvis = 0;
    for (int64_t i = gwarp(); i < count; i += nwarps()) {
        const int64_t ch = lin[i];
        const int64_t col = ch / g.CPC;
        const int z = (int)(ch - col * g.CPC) * 32 + lane;
        const bool valid = z < g.Z;
        const int64_t v0 = col * g.Z, v = v0 + z;
        const int x = (int)(col / g.Y), y = (int)(col - (int64_t)x * g.Y);
        int E = 0, H = INF, T = 0, D = 0, L[4] = {0, 0, 0, 0};
        if (valid) {
            const int4 *rec = reinterpret_cast<const int4 *>(&s.E[v]);  // E H T D | L0 L1 L2 L3
            const int4 a = rec[0], b = rec[1];
            E = a.x, H = a.y, T = a.z, D = a.w;
            L[0] = b.x, L[1] = b.y, L[2] = b.z, L[3] = b.w;
        }
        const int E0 = E, H0 = H, T0 = T, D0 = D, L00 = L[0], L01 = L[1], L02 = L[2], L03 = L[3];
        if (!__any_sync(FULL, valid && E > 0 && H < INF)) continue;
        if (lane == 0) myvis++;
        // neighbour data, one round of independent loads
        const bool dn = valid && z >= 1, upv = valid && z + 1 < g.Z;
        const int hdn_ext = (lane == 0 && dn) ? (int)s.H[v - 1] : INF;
        int hup_ext = INF, dup_ext = 0;
        if (lane == 31 && upv) {
            hup_ext = s.H[v + 1];
            dup_ext = s.D[v + 1];
        }
        int ho[4], hi[4], ri[4];
        int64_t to[4], ti[4];
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const int64_t off = nbr_off(g, x, y, d);
            const int zo = zo_of(z, dl_out(g, d)), zi = zi_of(z, dl_in(g, d), g.Z);
            const bool oko = valid && off && zo >= 0, oki = valid && off && zi >= 0;
            to[d] = v0 + off + zo;
            ti[d] = v0 + off + zi;
            ho[d] = oko ? (int)s.H[to[d]] : INF;
            ri[d] = oki ? (int)s.L[d ^ 1][ti[d]] : 0;
            hi[d] = oki ? (int)s.H[ti[d]] : INF;
        }
        for (int r = 0; r < rounds; r++) {
            bool act = valid && E > 0 && H < INF;
            if (!__any_sync(FULL, act)) break;
            int hd = __shfl_up_sync(FULL, H, 1), hu = __shfl_down_sync(FULL, H, 1), du = __shfl_down_sync(FULL, D, 1);
            if (lane == 0) hd = hdn_ext;
            if (lane == 31) hu = hup_ext, du = dup_ext;
            if (!dn) hd = INF;
            if (!upv) hu = INF, du = 0;
            int arc = -1, best = INF, res = 0;
            int give_dn = 0, give_up = 0;
            int64_t ext = NONE;
            if (act) {
                mywork++;
                if (T > 0) {
                    arc = 0, best = 0, res = T;
                } else {
                    if (hd < best) best = hd, arc = 1;
                    if (best >= H && du > 0 && hu < best) best = hu, arc = 6, res = du;
                    if (best >= H) {
#pragma unroll
                        for (int d = 0; d < 4; d++)
                            if (ho[d] < best) best = ho[d], arc = 2 + d;
                    }
                    if (best >= H) {
#pragma unroll
                        for (int d = 0; d < 4; d++)
                            if (ri[d] > 0 && hi[d] < best) best = hi[d], arc = 7 + d, res = ri[d];
                    }
                }
                if (best >= INF) {  // no residual path known: dead until the next global relabel
                    H = INF;
                    myrel++;
                    act = false;
                } else if (H <= best) {  // relabel, then push in the same operation
                    myrel++;
                    H = best + 1;
                    if (H >= INF) H = INF, act = false;
                }
            }
            if (act) {
                int df = 0;
                switch (arc) {
                    case 0: df = min(E, res); T -= df; break;
                    case 1:
                        df = E;
                        D += df;
                        if (lane > 0) give_dn = df;
                        else ext = v - 1;
                        break;
                    case 6:
                        df = min(E, du);
                        if (lane < 31) {
                            give_up = df;
                        } else {
                            atomicSub(&s.D[v + 1], df);
                            dup_ext -= df;
                            ext = v + 1;
                        }
                        break;
                    default:  // lateral (unrolled: no dynamically indexed register arrays)
#pragma unroll
                        for (int d = 0; d < 4; d++) {
                            if (arc == 2 + d) {
                                df = E;
                                L[d] += df;
                                ext = to[d];
                            } else if (arc == 7 + d) {
                                df = min(E, ri[d]);
                                ri[d] -= df;
                                atomicSub(&s.L[d ^ 1][ti[d]], df);
                                ext = ti[d];
                            }
                        }
                        break;
                }
                E -= df;
                if (ext != NONE) {
                    const int old = atomicAdd(&s.E[ext], df);
                    if (old > INT_MAX - df) atomicOr(flags, FLAG_OVERFLOW);
                }
            }
            // in-chunk transfers: lane i+1's down push and lane i-1's up push arrive at lane i
            int from_up = __shfl_down_sync(FULL, give_dn, 1), from_dn = __shfl_up_sync(FULL, give_up, 1);
            if (lane == 31) from_up = 0;
            if (lane == 0) from_dn = 0;
            if ((long long)E + from_up + from_dn > INT_MAX) atomicOr(flags, FLAG_OVERFLOW);
            E += from_up + from_dn;
            D -= from_dn;
            // list the chunk that received an external push
            int mark = -1;
            if (ext != NONE) {
                const int64_t tc = ext / g.Z;
                mark = (int)(tc * g.CPC + (ext - tc * g.Z) / 32);
            }
            warp_mark(mark, cstamp, tag, lout, cout);
        }
        if (valid) {
            if (H != H0) s.H[v] = H;
            if (T != T0) s.T[v] = T;
            if (E != E0) atomicAdd(&s.E[v], E - E0);
            if (D != D0) atomicAdd(&s.D[v], D - D0);
            if (L[0] != L00) atomicAdd(&s.L[0][v], L[0] - L00);
            if (L[1] != L01) atomicAdd(&s.L[1][v], L[1] - L01);
            if (L[2] != L02) atomicAdd(&s.L[2][v], L[2] - L02);
            if (L[3] != L03) atomicAdd(&s.L[3][v], L[3] - L03);
        }
        const bool still = __any_sync(FULL, valid && E > 0 && H < INF);
        warp_mark(still && lane == 0 ? (int)ch : -1, cstamp, tag, lout, cout);
    }
    flush_work(work, mywork, myrel);
    const unsigned long long vs = warp_sum_ll((long long)myvis);
    if (lane == 0 && vs) atomicAdd(visits, vs);
}

}  // namespace cg
