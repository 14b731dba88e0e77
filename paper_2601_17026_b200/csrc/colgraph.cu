// colgraph.cu -- B200 (sm_100a) implementation of include/colgraph.h.
//
// Hot path of arXiv 2601.17026 (§3.2): push-relabel max-flow on
// Wu-Chen proper-ordered column graphs with implicit (x,y,z) addressing,
// redesigned for one GPU per process:
//   a1 build            k_build                    (§1.2, §2.1)
//   a2/a5 global relabel k_gr_pass (column scans)  (§2.1, Alg. 3)
//   a3 sweep            k_sweep (lock-free)        (§2.1, Alg. 2)
//   a4 termination      host loop + exact relabel  (§3.2.4, Alg. 1)
//   a5 gap              k_gap_*                    (§2.1)
//   a6 flow value       k_sum_T                    (Eq. 5)
//   a7 extraction       k_ext_*                    (Theorem 1)
//
// Residual layout: 8 int32 planes of n each,
//   E  excess            H  height (INF = n_global + 1 = cannot reach t)
//   T  sink-arc residual D  flow on the down arc (x,y,z)->(x,y,z-1) = residual of the up arc
//   L0..L3 flow on the lateral arc in direction d (+x,-x,+y,-y) = residual of its reverse.
// Arc set ("minimal" form, reading R2): down arcs z->z-1 (INF);
// lateral arcs (x,y,z)->(nbr, zo(z)) with zo(0)=0, zo(z)=z-Delta for z>Delta,
// none for 1<=z<=Delta.  Each vertex then has at most one lateral in-arc per
// direction, from (nbr, zi(z)), zi(0)=0, zi(z)=z+Delta.
//
// Lock-free rule: every residual field has exactly one decrementer, so every
// value a thread reads (possibly stale) is a lower bound of what it may
// subtract; termination is certified by an exact global relabel.
#include "colgraph.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {

constexpr unsigned FULL = 0xffffffffu;

struct Geo {
    int32_t X, Y, Z, delta;  // X = planes owned by this rank
    int64_t n;               // vertices owned by this rank
    int64_t YZ;              // vertices per x-plane
    int32_t INF;             // n_global + 1
};

struct Soa {
    int32_t *E, *H, *T, *D, *L;  // L: 4 planes at L + d*n
};

enum { FLAG_OVERFLOW = 1 };

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ int zo_of(int z, int delta) { return z == 0 ? 0 : (z > delta ? z - delta : -1); }
__device__ __forceinline__ int zi_of(int z, int delta, int Z) { return z == 0 ? 0 : (z + delta < Z ? z + delta : -1); }

// neighbour column in direction d (0:+x 1:-x 2:+y 3:-y): offset in vertices, or 0 if absent
__device__ __forceinline__ int64_t nbr_off(const Geo &g, int x, int y, int d) {
    switch (d) {
        case 0: return x + 1 < g.X ? g.YZ : 0;
        case 1: return x >= 1 ? -g.YZ : 0;
        case 2: return y + 1 < g.Y ? (int64_t)g.Z : 0;
        default: return y >= 1 ? -(int64_t)g.Z : 0;
    }
}

__device__ __forceinline__ int warp_sum_i(int v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// ------------------------------------------------------------------ a1: build
// One warp per column: w(0) = c(0) - (sum_z c + 1), w(z) = c(z) - c(z-1)
// (R1); E = max(0,-w) (source arcs saturated), T = max(0,w).
__global__ void k_build(Geo g, const int32_t *__restrict__ in, int weight_mode, Soa s,
                        unsigned long long *sums /* [0]=N, [1]=sum T0 */, int *flags) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    long long accN = 0, accT = 0;
    bool bad = false;
    for (int64_t col = (int64_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); col < ncol; col += warps) {
        const int32_t *cc = in + col * g.Z;
        long long colsum = 0;
        if (!weight_mode) {
            for (int z = lane_id(); z < g.Z; z += 32) colsum += cc[z];
            colsum = warp_sum_ll(colsum);
        }
        for (int z = lane_id(); z < g.Z; z += 32) {
            long long w;
            if (weight_mode) {
                w = cc[z];
            } else {
                w = z == 0 ? (long long)cc[0] - (colsum + 1) : (long long)cc[z] - (long long)cc[z - 1];
            }
            if (w > INT_MAX || w < -(long long)INT_MAX) bad = true;
            int32_t e = w < 0 ? (int32_t)(-w) : 0, t = w > 0 ? (int32_t)w : 0;
            s.E[col * g.Z + z] = bad ? 0 : e;
            s.T[col * g.Z + z] = bad ? 0 : t;
            accN += e;
            accT += t;
        }
    }
    accN = warp_sum_ll(accN);
    accT = warp_sum_ll(accT);
    if (lane_id() == 0) {
        atomicAdd(&sums[0], (unsigned long long)accN);
        atomicAdd(&sums[1], (unsigned long long)accT);
    }
    if (bad) atomicOr(flags, FLAG_OVERFLOW);
}

__global__ void k_fill(int32_t *p, int64_t n, int32_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// ------------------------------------------------------------------ a3: push-relabel sweep
// One thread per vertex.  An active vertex (E > 0, H < INF) scans its residual
// out-arcs in the fixed order t, down, lateral-out(+x,-x,+y,-y), up,
// lateral-in-reverse(+x,-x,+y,-y), takes the lowest neighbour height h_min
// (first wins ties), relabels to h_min+1 if H <= h_min (Alg. 2 Relabel,
// "newd = min label(w)+1", only if larger) and pushes delta = min(E, r) along
// that arc (Alg. 2 Push).  Up to `ops` push/relabel operations per sweep.
// Fused: warp-aggregated count of vertices active at the start of the sweep.
__global__ void __launch_bounds__(256) k_sweep(Geo g, Soa s, int ops, unsigned long long *cnt, int *flags) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool act = false;
    if (v < g.n) {
        int e = s.E[v];
        int h = s.H[v];
        if (e > 0 && h < g.INF) {
            act = true;
            const int z = (int)(v % g.Z);
            const int64_t col = v / g.Z;
            const int x = (int)(col / g.Y), y = (int)(col % g.Y);
            const int64_t v0 = v - z;  // column base
            const int zo = zo_of(z, g.delta), zi = zi_of(z, g.delta, g.Z);
            int64_t off[4];
#pragma unroll
            for (int d = 0; d < 4; d++) off[d] = nbr_off(g, x, y, d);
            int sent = 0;
            for (int it = 0; it < ops && e > 0; ++it) {
                int best = g.INF, arc = -1, res = 0;
                int64_t tgt = -1;
                const int tres = s.T[v];
                if (tres > 0) {
                    best = 0;
                    arc = 0;
                } else {
                    if (z >= 1) {
                        int hh = s.H[v - 1];
                        if (hh < best) { best = hh; arc = 1; tgt = v - 1; }
                    }
                    if (zo >= 0) {
#pragma unroll
                        for (int d = 0; d < 4; d++) {
                            if (!off[d]) continue;
                            int64_t t = v0 + off[d] + zo;
                            int hh = s.H[t];
                            if (hh < best) { best = hh; arc = 2 + d; tgt = t; }
                        }
                    }
                    if (z + 1 < g.Z) {
                        int r = s.D[v + 1];
                        if (r > 0) {
                            int hh = s.H[v + 1];
                            if (hh < best) { best = hh; arc = 6; tgt = v + 1; res = r; }
                        }
                    }
                    if (zi >= 0) {
#pragma unroll
                        for (int d = 0; d < 4; d++) {
                            if (!off[d]) continue;
                            int64_t u = v0 + off[d] + zi;
                            int r = s.L[(int64_t)(d ^ 1) * g.n + u];
                            if (r > 0) {
                                int hh = s.H[u];
                                if (hh < best) { best = hh; arc = 7 + d; tgt = u; res = r; }
                            }
                        }
                    }
                }
                if (best >= g.INF) {  // no residual path known: dead until the next global relabel
                    s.H[v] = g.INF;
                    break;
                }
                if (h <= best) {  // relabel
                    h = best + 1;
                    s.H[v] = h;
                    if (h >= g.INF) break;
                }
                int df;
                switch (arc) {
                    case 0:
                        df = min(e, tres);
                        s.T[v] = tres - df;
                        break;
                    case 1:
                        df = e;
                        atomicAdd(&s.D[v], df);
                        break;
                    case 2: case 3: case 4: case 5:
                        df = e;
                        atomicAdd(&s.L[(int64_t)(arc - 2) * g.n + v], df);
                        break;
                    case 6:
                        df = min(e, res);
                        atomicSub(&s.D[v + 1], df);
                        break;
                    default:
                        df = min(e, res);
                        atomicSub(&s.L[(int64_t)((arc - 7) ^ 1) * g.n + tgt], df);
                        break;
                }
                if (tgt >= 0) {
                    int old = atomicAdd(&s.E[tgt], df);
                    if (old > INT_MAX - df) atomicOr(flags, FLAG_OVERFLOW);
                }
                e -= df;
                sent += df;
            }
            if (sent) atomicSub(&s.E[v], sent);
        }
    }
    unsigned b = __ballot_sync(FULL, act);
    if (lane_id() == 0 && b) atomicAdd(cnt, (unsigned long long)__popc(b));
}

// ------------------------------------------------------------------ a2/a5: exact global relabel
// H(v) = residual BFS distance from v to t (Alg. 3; PAPER.md:134 footnote).
// Column structure: down arcs are infinite, so d(z) <= d(z-1)+1; up arcs exist
// where D(z+1) > 0, so d(z) <= d(z+1)+1 there.  Given the lateral/terminal
// "external" distances ext(z), a column's distances are two scans:
//   forward  a(z) = z + prefix_min_{s<=z}(ext(s) - s)
//   backward d(z) = -z + segmented suffix_min_{s>=z, up-linked}(a(s) + s)
// Passes repeat (monotone Bellman-Ford relaxation, in place) until a pass
// changes nothing: the fixpoint is the exact BFS distance.
__device__ __forceinline__ int warp_prefix_min(int v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(FULL, v, o);
        if (lane_id() >= o) v = min(v, t);
    }
    return v;
}
// v_l = min over j >= l reachable through consecutive links (link_l: l -> l+1), within the warp
__device__ __forceinline__ int warp_seg_suffix_min(int v, bool link) {
    int f = link;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v2 = __shfl_down_sync(FULL, v, o);
        int f2 = __shfl_down_sync(FULL, f, o);
        if (lane_id() + o < 32) {
            if (f) v = min(v, v2);
            f = f && f2;
        } else {
            f = 0;
        }
    }
    return v;
}

__global__ void __launch_bounds__(256) k_gr_pass(Geo g, Soa s, int *changed) {
    extern __shared__ int32_t sh_a[];  // per warp: Z ints
    const int wib = threadIdx.x >> 5;
    int32_t *a = sh_a + (int64_t)wib * g.Z;
    const int64_t ncol = (int64_t)g.X * g.Y;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int INF = g.INF;
    bool any = false;
    for (int64_t col = (int64_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); col < ncol; col += warps) {
        const int x = (int)(col / g.Y), y = (int)(col % g.Y);
        const int64_t v0 = col * g.Z;
        int64_t off[4];
#pragma unroll
        for (int d = 0; d < 4; d++) off[d] = nbr_off(g, x, y, d);
        // forward: ext and prefix-min
        int carry = INF;  // min over earlier chunks of (ext(s) - s)
        for (int c0 = 0; c0 < g.Z; c0 += 32) {
            const int z = c0 + lane_id();
            int ext = INF;
            if (z < g.Z) {
                const int64_t v = v0 + z;
                if (s.T[v] > 0) ext = 1;
                const int zo = zo_of(z, g.delta);
                if (zo >= 0) {
#pragma unroll
                    for (int d = 0; d < 4; d++) {
                        if (!off[d]) continue;
                        int hh = s.H[v0 + off[d] + zo];
                        if (hh < INF) ext = min(ext, hh + 1);
                    }
                }
                const int zi = zi_of(z, g.delta, g.Z);
                if (zi >= 0) {
#pragma unroll
                    for (int d = 0; d < 4; d++) {
                        if (!off[d]) continue;
                        int64_t u = v0 + off[d] + zi;
                        if (s.L[(int64_t)(d ^ 1) * g.n + u] > 0) {
                            int hh = s.H[u];
                            if (hh < INF) ext = min(ext, hh + 1);
                        }
                    }
                }
            }
            int val = min(warp_prefix_min(ext - (z < g.Z ? z : 0)), carry);
            carry = __shfl_sync(FULL, val, 31);
            if (z < g.Z) a[z] = min(INF, val + z);
        }
        __syncwarp();
        // backward: segmented suffix min along residual up arcs
        int carry_b = INF;  // min reachable value (a(s)+s) from the element just above this chunk
        const int last_c0 = ((g.Z - 1) / 32) * 32;
        for (int c0 = last_c0; c0 >= 0; c0 -= 32) {
            const int z = c0 + lane_id();
            int val = INF;
            bool link = false;
            if (z < g.Z) {
                val = a[z] + z;
                link = (z + 1 < g.Z) && s.D[v0 + z + 1] > 0;
            }
            val = warp_seg_suffix_min(val, link);
            const unsigned m = __ballot_sync(FULL, link);
            const unsigned need = FULL << lane_id();
            if ((m & need) == need) val = min(val, carry_b);
            carry_b = __shfl_sync(FULL, val, 0);
            if (z < g.Z) {
                int d = min(INF, val - z);
                const int64_t v = v0 + z;
                int old = s.H[v];
                if (d < old) {
                    s.H[v] = d;
                    any = true;
                }
            }
        }
        __syncwarp();
    }
    if (__any_sync(FULL, any) && lane_id() == 0) atomicOr(changed, 1);
}

__global__ void k_count_active(Geo g, const int32_t *__restrict__ E, const int32_t *__restrict__ H,
                               unsigned long long *cnt) {
    int c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (int64_t)gridDim.x * blockDim.x)
        c += (E[i] > 0 && H[i] < g.INF);
    c = warp_sum_i(c);
    if (lane_id() == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}

// ------------------------------------------------------------------ a5: gap heuristic
constexpr int GAP_BINS = 1 << 20;
__global__ void k_gap_hist(Geo g, const int32_t *__restrict__ H, unsigned *hist, int *maxh) {
    int mymax = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (int64_t)gridDim.x * blockDim.x) {
        int h = H[i];
        if (h < g.INF) {
            mymax = max(mymax, h);
            if (h < GAP_BINS) atomicAdd(&hist[h], 1u);
        }
    }
    for (int o = 16; o; o >>= 1) mymax = max(mymax, __shfl_xor_sync(FULL, mymax, o));
    if (lane_id() == 0) atomicMax(maxh, mymax);
}
// smallest g in [1, min(maxh, GAP_BINS)) with hist[g] == 0
__global__ void k_gap_find(const unsigned *hist, const int *maxh, int *gap) {
    const int lim = min(*maxh, GAP_BINS - 1);
    int best = INT_MAX;
    for (int h = 1 + (int)threadIdx.x; h < lim; h += blockDim.x)
        if (hist[h] == 0) { best = h; break; }
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
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (int64_t)gridDim.x * blockDim.x) {
            int h = H[i];
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
// Minimal source set S = forward residual closure of {v : E(v) > 0} (SURVEY.md
// §8(a) a7, reading R5).  S is downward closed in every column (infinite down
// arcs), so it is top(x,y); pull-style fixpoint per column:
//   seed   top >= max{z : E(z) > 0}
//   lat-out from nbr   top >= max(0, top(nbr) - Delta)             (nbr's arcs (nbr,z)->(C,zo(z)))
//   lat-in  from nbr   top >= max{z' : L_dir(C->nbr)(C,z') > 0, z' = zi(z), z <= top(nbr)}
//   up     climb while D(top+1) > 0
__device__ int warp_climb(const Geo &g, const int32_t *__restrict__ D, int64_t v0, int t) {
    if (t < 0) return t;
    for (int base = t + 1; base < g.Z; base += 32) {
        const int z = base + lane_id();
        const bool stop = (z >= g.Z) || D[v0 + z] <= 0;
        const unsigned m = __ballot_sync(FULL, stop);
        if (m) return base + __ffs(m) - 1 - 1;
    }
    return g.Z - 1;
}

__global__ void k_ext_seed(Geo g, Soa s, int32_t *top) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int64_t col = (int64_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); col < ncol; col += warps) {
        const int64_t v0 = col * g.Z;
        int t = -1;
        for (int c0 = 0; c0 < g.Z; c0 += 32) {
            const int z = c0 + lane_id();
            const unsigned m = __ballot_sync(FULL, z < g.Z && s.E[v0 + z] > 0);
            if (m) t = c0 + 31 - __clz(m);
        }
        t = warp_climb(g, s.D, v0, t);
        if (lane_id() == 0) top[col] = t;
    }
}

__global__ void k_ext_pass(Geo g, Soa s, int32_t *top, int *changed) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    bool any = false;
    for (int64_t col = (int64_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); col < ncol; col += warps) {
        const int x = (int)(col / g.Y), y = (int)(col % g.Y);
        const int64_t v0 = col * g.Z;
        const int t0 = top[col];
        int t = t0;
        int tn[4];
#pragma unroll
        for (int d = 0; d < 4; d++) {
            int64_t o = nbr_off(g, x, y, d);
            tn[d] = o ? top[col + o / g.Z] : -1;
            if (tn[d] >= 0) t = max(t, max(0, tn[d] - g.delta));
        }
#pragma unroll
        for (int d = 0; d < 4; d++) {
            if (tn[d] < 0) continue;
            // C's own lateral arc in direction d points at nbr_d; its flow L_d(C,z') > 0 is a
            // residual arc (nbr, zo(z')) -> (C, z').  Allowed z' in {0} U [Delta+1, tn+Delta].
            const int lim = min(g.Z - 1, tn[d] + g.delta);
            const int32_t *Ld = s.L + (int64_t)d * g.n + v0;
            for (int hi = lim; hi > t && hi >= g.delta + 1; hi -= 32) {
                const int z = hi - lane_id();
                const bool ok = z > t && z >= g.delta + 1 && Ld[z] > 0;
                const unsigned m = __ballot_sync(FULL, ok);
                if (m) { t = hi - (__ffs(m) - 1); break; }
            }
            if (t < 0 && Ld[0] > 0) t = 0;
        }
        if (t > t0 || (t0 < 0 && t >= 0)) t = warp_climb(g, s.D, v0, t);
        if (t != t0) {
            any = true;
            if (lane_id() == 0) top[col] = t;
        }
    }
    if (__any_sync(FULL, any) && lane_id() == 0) atomicOr(changed, 1);
}

__global__ void k_ext_out(Geo g, const int32_t *__restrict__ top, int32_t *surface, uint8_t *mask, int *empty) {
    const int64_t ncol = (int64_t)g.X * g.Y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ncol; i += (int64_t)gridDim.x * blockDim.x) {
        surface[i] = top[i];
        if (top[i] < 0) atomicOr(empty, 1);
    }
    if (mask) {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += (int64_t)gridDim.x * blockDim.x)
            mask[i] = (uint8_t)((int)(i % g.Z) <= top[i / g.Z]);
    }
}

}  // namespace

// ====================================================================== host side

struct cg_graph {
    cg_dims dims{};
    cg_dist dist{};
    Geo geo{};
    cudaStream_t stream = nullptr;
    int32_t *soa = nullptr;  // 8 planes
    Soa s{};
    // device scratch
    unsigned long long *d_u64 = nullptr;  // [0]=N [1]=sumT0 [2]=sumT [3]=active [4]=lifted [8..8+RING) sweep counts
    int *d_i32 = nullptr;                 // [0]=flags [1]=changed [2]=maxh [3]=gap [4]=empty
    unsigned *d_hist = nullptr;
    int32_t *d_top = nullptr;
    // pinned host mirrors
    unsigned long long *h_u64 = nullptr;
    int *h_i32 = nullptr;
    int64_t N = 0, sumT0 = 0;
    bool solved = false;
    int num_sms = 148;
    cg_solve_stats st{};
};

namespace {

constexpr int RING = 256;
constexpr int U64_SLOTS = 8 + RING;

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

#define CG_CUDA(call)                                                   \
    do {                                                                \
        cudaError_t e_ = (call);                                        \
        if (e_ != cudaSuccess) {                                        \
            if (getenv("CG_DEBUG"))                                     \
                fprintf(stderr, "colgraph: %s -> %s (%s:%d)\n", #call,  \
                        cudaGetErrorString(e_), __FILE__, __LINE__);    \
            return e_ == cudaErrorMemoryAllocation ? CG_E_NOMEM : CG_E_CUDA; \
        }                                                               \
    } while (0)

int grid_for(int64_t n, int block, int cap) {
    int64_t b = (n + block - 1) / block;
    if (b < 1) b = 1;
    return (int)std::min<int64_t>(b, cap);
}

cg_status sync_read(cg_graph *g) {
    CG_CUDA(cudaStreamSynchronize(g->stream));
    return CG_OK;
}

// exact global relabel; leaves the active count in h_u64[3]
cg_status global_relabel(cg_graph *g) {
    const Geo &geo = g->geo;
    const int block = 256;
    const int wpb = block / 32;
    const size_t shmem = (size_t)wpb * geo.Z * sizeof(int32_t);
    if (shmem > 200 * 1024) return CG_E_INVAL;
    const int64_t ncol = (int64_t)geo.X * geo.Y;
    const int grid_cols = grid_for(ncol * 32, block, g->num_sms * 16);
    static bool attr_set = false;
    if (!attr_set && shmem > 48 * 1024) {
        CG_CUDA(cudaFuncSetAttribute(k_gr_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_set = true;
    }
    k_fill<<<g->num_sms * 8, 256, 0, g->stream>>>(g->s.H, geo.n, geo.INF);
    for (int pass = 0;; pass++) {
        CG_CUDA(cudaMemsetAsync(g->d_i32 + 1, 0, sizeof(int), g->stream));
        k_gr_pass<<<grid_cols, block, shmem, g->stream>>>(geo, g->s, g->d_i32 + 1);
        g->st.kernel_launches++;
        CG_CUDA(cudaMemcpyAsync(g->h_i32 + 1, g->d_i32 + 1, sizeof(int), cudaMemcpyDeviceToHost, g->stream));
        cg_status st = sync_read(g);
        if (st) return st;
        g->st.gr_passes++;
        if (!g->h_i32[1]) break;
    }
    CG_CUDA(cudaMemsetAsync(g->d_u64 + 3, 0, sizeof(unsigned long long), g->stream));
    k_count_active<<<g->num_sms * 8, 256, 0, g->stream>>>(geo, g->s.E, g->s.H, g->d_u64 + 3);
    g->st.kernel_launches += 2;  // fill + count
    CG_CUDA(cudaMemcpyAsync(g->h_u64 + 3, g->d_u64 + 3, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            g->stream));
    cg_status st = sync_read(g);
    if (st) return st;
    CG_CUDA(cudaGetLastError());
    g->st.global_relabels++;
    return CG_OK;
}

cg_status run_gap(cg_graph *g) {
    const Geo &geo = g->geo;
    CG_CUDA(cudaMemsetAsync(g->d_hist, 0, sizeof(unsigned) * GAP_BINS, g->stream));
    CG_CUDA(cudaMemsetAsync(g->d_i32 + 2, 0, sizeof(int), g->stream));
    k_gap_hist<<<g->num_sms * 8, 256, 0, g->stream>>>(geo, g->s.H, g->d_hist, g->d_i32 + 2);
    k_gap_find<<<1, 1024, 0, g->stream>>>(g->d_hist, g->d_i32 + 2, g->d_i32 + 3);
    k_gap_lift<<<g->num_sms * 8, 256, 0, g->stream>>>(geo, g->s.H, g->d_i32 + 3, g->d_u64 + 4);
    CG_CUDA(cudaGetLastError());
    g->st.kernel_launches += 3;
    g->st.gap_runs++;
    return CG_OK;
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

const char *cg_version(void) { return "colgraph 0.1 sm_100a (lock-free push-relabel, column-scan global relabel)"; }

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
        cudaFree(g->soa);
        cudaFree(g->d_u64);
        cudaFree(g->d_i32);
        cudaFree(g->d_hist);
        cudaFree(g->d_top);
        cudaFreeHost(g->h_u64);
        cudaFreeHost(g->h_i32);
    }
    delete g;
}

cg_status colgraph_build(const cg_dims *dims, const int32_t *cost_dev, int32_t input_is_weight, const cg_dist *dist,
                         cg_graph **out) {
    if (!dims || !cost_dev || !out) return CG_E_INVAL;
    *out = nullptr;
    if (dims->X < 1 || dims->Y < 1 || dims->Z < 1 || dims->delta < 0) return CG_E_INVAL;
    const int64_t n = (int64_t)dims->X * dims->Y * dims->Z;
    if (n + dims->Z + 2 >= (int64_t)INT_MAX) return CG_E_INVAL;
    cg_dist dd{0, 1, nullptr, 0, nullptr};
    if (dist) dd = *dist;
    if (dd.nranks != 1 || dd.rank != 0) return CG_E_INVAL;  // multi-GPU: see colgraph_mgpu (not in this build)
    DeviceGuard dg(dd.device);
    auto t0 = std::chrono::steady_clock::now();
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
    geo.n = n;
    geo.YZ = (int64_t)dims->Y * dims->Z;
    geo.INF = (int32_t)(n + 1);
    auto fail = [&](cg_status st) {
        colgraph_free(g);
        return st;
    };
    if (cudaMalloc(&g->soa, sizeof(int32_t) * 8 * n) != cudaSuccess) return fail(CG_E_NOMEM);
    if (cudaMalloc(&g->d_u64, sizeof(unsigned long long) * U64_SLOTS) != cudaSuccess) return fail(CG_E_NOMEM);
    if (cudaMalloc(&g->d_i32, sizeof(int) * 16) != cudaSuccess) return fail(CG_E_NOMEM);
    if (cudaMalloc(&g->d_hist, sizeof(unsigned) * GAP_BINS) != cudaSuccess) return fail(CG_E_NOMEM);
    if (cudaMalloc(&g->d_top, sizeof(int32_t) * dims->X * dims->Y) != cudaSuccess) return fail(CG_E_NOMEM);
    if (cudaHostAlloc(&g->h_u64, sizeof(unsigned long long) * U64_SLOTS, cudaHostAllocDefault) != cudaSuccess)
        return fail(CG_E_NOMEM);
    if (cudaHostAlloc(&g->h_i32, sizeof(int) * 16, cudaHostAllocDefault) != cudaSuccess) return fail(CG_E_NOMEM);
    g->s.E = g->soa;
    g->s.H = g->soa + n;
    g->s.T = g->soa + 2 * n;
    g->s.D = g->soa + 3 * n;
    g->s.L = g->soa + 4 * n;
    cudaStream_t st = g->stream;
    if (cudaMemsetAsync(g->d_u64, 0, sizeof(unsigned long long) * U64_SLOTS, st) != cudaSuccess ||
        cudaMemsetAsync(g->d_i32, 0, sizeof(int) * 16, st) != cudaSuccess ||
        cudaMemsetAsync(g->s.H, 0, sizeof(int32_t) * n, st) != cudaSuccess ||
        cudaMemsetAsync(g->s.D, 0, sizeof(int32_t) * 5 * n, st) != cudaSuccess)
        return fail(CG_E_CUDA);
    const int64_t ncol = (int64_t)dims->X * dims->Y;
    k_build<<<grid_for(ncol * 32, 256, g->num_sms * 16), 256, 0, st>>>(geo, cost_dev, input_is_weight ? 1 : 0, g->s,
                                                                       g->d_u64, g->d_i32);
    if (cudaGetLastError() != cudaSuccess) return fail(CG_E_CUDA);
    cudaMemcpyAsync(g->h_u64, g->d_u64, sizeof(unsigned long long) * 2, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(g->h_i32, g->d_i32, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(CG_E_CUDA);
    if (g->h_i32[0] & FLAG_OVERFLOW) return fail(CG_E_OVERFLOW);
    g->N = (int64_t)g->h_u64[0];
    g->sumT0 = (int64_t)g->h_u64[1];
    g->st.source_capacity = g->N;
    g->st.bytes_per_sweep_alg = 32.0 * (double)n;
    g->st.ms_build = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    *out = g;
    return CG_OK;
}

cg_status maxflow_solve(cg_graph *g, const cg_solve_opts *opts, int64_t *flow_value, cg_solve_stats *stats) {
    if (!g || !flow_value) return CG_E_INVAL;
    if (g->solved) return CG_E_STATE;
    DeviceGuard dg(g->dist.device);
    cg_solve_opts o{1.0f, 0, 16, (int64_t)1 << 30, 1};
    if (opts) o = *opts;
    if (o.check_every < 1) o.check_every = 1;
    if (o.check_every > RING) o.check_every = RING;
    if (o.ops_per_sweep < 1) o.ops_per_sweep = 1;
    if (o.gr_factor <= 0.f) o.gr_factor = 1.0f;
    const Geo &geo = g->geo;
    cudaStream_t st = g->stream;
    auto t0 = std::chrono::steady_clock::now();
    double ms_gr = 0.0;
    auto timed_gr = [&]() {
        auto a = std::chrono::steady_clock::now();
        cg_status s = global_relabel(g);
        ms_gr += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
        return s;
    };
    cg_status rs = timed_gr();
    if (rs) return rs;
    int64_t active = (int64_t)g->h_u64[3];
    const double gr_budget = (double)o.gr_factor * (double)geo.n;
    double work_since_gr = 0.0;
    const int block = 256;
    const int grid = grid_for(geo.n, block, INT_MAX);
    int64_t sweeps = 0, since_gap = 0;
    cg_status result = CG_OK;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    CG_CUDA(cudaEventCreate(&ev0));
    CG_CUDA(cudaEventCreate(&ev1));
    while (active > 0) {
        if (sweeps >= o.max_sweeps) { result = CG_E_NOT_CONVERGED; break; }
        const int batch = (int)std::min<int64_t>(o.check_every, o.max_sweeps - sweeps);
        CG_CUDA(cudaMemsetAsync(g->d_u64 + 8, 0, sizeof(unsigned long long) * batch, st));
        CG_CUDA(cudaEventRecord(ev0, st));
        for (int i = 0; i < batch; i++)
            k_sweep<<<grid, block, 0, st>>>(geo, g->s, o.ops_per_sweep, g->d_u64 + 8 + i, g->d_i32);
        CG_CUDA(cudaEventRecord(ev1, st));
        g->st.kernel_launches += batch;
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaMemcpyAsync(g->h_u64 + 8, g->d_u64 + 8, sizeof(unsigned long long) * batch,
                                cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaMemcpyAsync(g->h_i32, g->d_i32, sizeof(int), cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaStreamSynchronize(st));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev0, ev1);
        g->st.ms_sweep_kernels += ms;
        if (g->h_i32[0] & FLAG_OVERFLOW) { result = CG_E_OVERFLOW; break; }
        bool quiescent = false;
        int done = 0;
        for (int i = 0; i < batch; i++) {
            const unsigned long long c = g->h_u64[8 + i];
            g->st.sweep_bytes_alg += 4.0 * (double)geo.n + 40.0 * (double)c;
            if (c == 0) { quiescent = true; break; }
            work_since_gr += (double)c;
            g->st.work += (int64_t)c;
            done++;
        }
        // sweeps after the first idle one in a batch are no-ops (nothing is active)
        for (int i = done + 1; i < batch && quiescent; i++) g->st.sweep_bytes_alg += 4.0 * (double)geo.n;
        sweeps += batch;
        since_gap += batch;
        if (quiescent || work_since_gr >= gr_budget) {
            // a4: termination is decided only after an exact global relabel
            rs = timed_gr();
            if (rs) { result = rs; break; }
            active = (int64_t)g->h_u64[3];
            work_since_gr = 0.0;
            since_gap = 0;
        } else if (o.gap_every > 0 && since_gap >= o.gap_every) {
            rs = run_gap(g);
            if (rs) { result = rs; break; }
            since_gap = 0;
        }
    }
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    if (result != CG_OK && result != CG_E_NOT_CONVERGED) return result;
    // a6: |f| = sum(T0) - sum(T)
    CG_CUDA(cudaMemsetAsync(g->d_u64 + 2, 0, sizeof(unsigned long long), st));
    k_sum_T<<<g->num_sms * 8, 256, 0, st>>>(geo, g->s.T, g->d_u64 + 2);
    g->st.kernel_launches++;
    CG_CUDA(cudaMemcpyAsync(g->h_u64 + 2, g->d_u64 + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaMemcpyAsync(g->h_u64 + 4, g->d_u64 + 4, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    CG_CUDA(cudaGetLastError());
    *flow_value = g->sumT0 - (int64_t)g->h_u64[2];
    g->st.sweeps = sweeps;
    g->st.gap_lifted = (int64_t)g->h_u64[4];
    g->st.ms_global_relabel = ms_gr;
    g->st.ms_solve = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
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
    auto t0 = std::chrono::steady_clock::now();
    const int64_t ncol = (int64_t)geo.X * geo.Y;
    const int grid_cols = grid_for(ncol * 32, 256, g->num_sms * 16);
    k_ext_seed<<<grid_cols, 256, 0, st>>>(geo, g->s, g->d_top);
    for (;;) {
        CG_CUDA(cudaMemsetAsync(g->d_i32 + 1, 0, sizeof(int), st));
        k_ext_pass<<<grid_cols, 256, 0, st>>>(geo, g->s, g->d_top, g->d_i32 + 1);
        g->st.kernel_launches++;
        CG_CUDA(cudaMemcpyAsync(g->h_i32 + 1, g->d_i32 + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaStreamSynchronize(st));
        g->st.extract_passes++;
        if (!g->h_i32[1]) break;
    }
    CG_CUDA(cudaMemsetAsync(g->d_i32 + 4, 0, sizeof(int), st));
    k_ext_out<<<g->num_sms * 8, 256, 0, st>>>(geo, g->d_top, surface_dev, mask_dev, g->d_i32 + 4);
    g->st.kernel_launches += 2;  // seed + out
    CG_CUDA(cudaMemcpyAsync(g->h_i32 + 4, g->d_i32 + 4, sizeof(int), cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    CG_CUDA(cudaGetLastError());
    g->st.ms_extract = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return g->h_i32[4] ? CG_E_EMPTY_COLUMN : CG_OK;
}

cg_status colgraph_stats(const cg_graph *g, cg_solve_stats *stats) {
    if (!g || !stats) return CG_E_INVAL;
    *stats = g->st;
    return CG_OK;
}

cg_status colgraph_export_state(cg_graph *g, int32_t *out_dev) {
    if (!g || !out_dev) return CG_E_INVAL;
    DeviceGuard dg(g->dist.device);
    CG_CUDA(cudaMemcpyAsync(out_dev, g->soa, sizeof(int32_t) * 8 * g->geo.n, cudaMemcpyDeviceToDevice, g->stream));
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
