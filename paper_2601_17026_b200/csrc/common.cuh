// common.cuh -- geometry, SoA layout and warp utilities shared by the colgraph kernels.
//
// Implicit addressing (§3.2.3): vertex (x,y,z) of this rank's
// slab has index v = (x*Y + y)*Z + z, z fastest.  A "chunk" is 32 consecutive z
// of one column -- the unit a warp processes (lane = z offset), so every state
// load of a chunk is one coalesced 128-byte line.
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

namespace cg {

constexpr unsigned FULL = 0xffffffffu;

struct Geo {
    int32_t X, Y, Z;         // X = x-planes owned by this slab
    int32_t dl[4];           // edge interval toward +x, -x, +y, -y: v's lateral arc in direction d lands
                             // at z - dl[d] (S(v) - S(nbr_d(v)) <= dl[d], NEXT-3); the
                             // isotropic case has all four equal
    int32_t CPC;             // chunks per column = ceil(Z / 32)
    int32_t gl, gh;          // a ghost plane exists at x = -1 (gl) / x = X (gh): neighbour slab
    int64_t n;               // vertices owned by this slab
    int64_t YZ;              // vertices per x-plane
    int64_t nchunks;         // X*Y*CPC
    int32_t INF;             // n_global + 1: "cannot reach t"
    // soft smoothness (NEXT-1): soft_k = K > 0 finite arcs per direction, (x,y,z) -> (nbr, z-k),
    // k < Delta_d, capacity soft_cap[k] = f(k+1) - 2 f(k) + f(k-1); 0 = hard constraint only
    int32_t soft_k;
    int32_t soft_cap[16];
    // division by Z and by Y without the division routine (set_fastdiv): q = n * m >> sh for
    // 0 <= n < 2^31 (Granlund-Montgomery: m = ceil(2^(31+l) / d), l = ceil(log2 d), sh = 31 + l)
    uint64_t mZ, mY;
    int32_t shZ, shY;
};
inline void fastdiv_params(uint32_t d, uint64_t &m, int32_t &sh) {
    int l = 0;
    while ((1ull << l) < d) l++;
    m = ((1ull << (31 + l)) + d - 1) / d;
    sh = 31 + l;
}
#ifndef CG_FASTDIV
#define CG_FASTDIV 1
#endif
#if CG_FASTDIV
#define CG_DIVZ(g, n) fdiv((uint32_t)(n), (g).mZ, (g).shZ)
#define CG_DIVY(g, n) fdiv((uint32_t)(n), (g).mY, (g).shY)
#else
#define CG_DIVZ(g, n) ((uint32_t)(n) / (uint32_t)(g).Z)
#define CG_DIVY(g, n) ((uint32_t)(n) / (uint32_t)(g).Y)
#endif
__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint64_t m, int sh) { return (uint32_t)(((uint64_t)n * m) >> sh); }
constexpr int SOFT_KMAX = 16;

// Residual state: 8 int32 fields per vertex -- E excess, H height, T sink residual, D flow
// on the down arc (= residual of the up arc into this vertex from below), L[d] flow on the
// lateral arc in direction d (= residual of its reverse arc); directions 0:+x 1:-x 2:+y 3:-y.
// Layout: CG_LAYOUT_AOS = 1 (default) stores the 8 fields of a vertex as one
// 32-byte record (one DRAM sector): the sweep and relabel kernels touch scattered vertices,
// and one sector then carries all of a vertex's fields.  CG_LAYOUT_AOS = 0 stores 8 planes.
// Either way z is fastest and each field spans X+2 x-planes: Field::p addresses owned plane
// x = 0, so the ghost planes of the neighbour slabs sit at vertex indices [-YZ, 0) and
// [n, n+YZ).
#ifndef CG_LAYOUT_AOS
#define CG_LAYOUT_AOS 1
#endif
constexpr int FIELD_STRIDE = CG_LAYOUT_AOS ? 8 : 1;

// CG_DEBUG_BOUNDS (debug build, `build --debug-bounds`): every state access checks its vertex
// index against the slab's range including the ghost planes, [-YZ, n + YZ); a violation
// increments g_oob and is clamped (no fault), and every API call then returns CG_E_CUDA.
// compute-sanitizer is closed on this pool: this is the bad-access check.
#ifdef CG_DEBUG_BOUNDS
__device__ unsigned long long g_oob;
template <int S>
struct FieldT {
    int32_t *p;
    int64_t lo, hi;
    __device__ __forceinline__ int32_t &operator[](int64_t i) const {
        if (i < lo || i >= hi) {
            atomicAdd(&g_oob, 1ull);
            i = lo;
        }
        return p[i * S];
    }
};
#else
template <int S>
struct FieldT {
    int32_t *p;
    int64_t lo, hi;  // valid vertex range (checked only in CG_DEBUG_BOUNDS builds)
    __device__ __forceinline__ int32_t &operator[](int64_t i) const { return p[i * S]; }
};
#endif
// CG_H_PLANE = 1 (AoS variant, `build --hplane`): the heights live in their own int32 plane
// (the record's H slot is unused), so the neighbour-height reads of the arc scans and the
// relabel hit 8 heights per sector instead of one record per height.
#ifndef CG_H_PLANE
#define CG_H_PLANE 0
#endif
using Field = FieldT<FIELD_STRIDE>;
using FieldH = FieldT<(CG_LAYOUT_AOS && CG_H_PLANE) ? 1 : FIELD_STRIDE>;

struct Soa {
    Field E;
    FieldH H;
    Field T, D;
    Field L[4];
    int32_t *SF;  // soft-arc flows, [v][d][k] (4 * soft_k ints per owned vertex); null if hard only
};

// flow on the soft arc (v, d, k): v -> (nbr_d, z - k)
__device__ __forceinline__ int32_t *soft_flow(const Geo &g, const Soa &s, int64_t v, int d, int k) {
    return s.SF + (v * 4 + d) * g.soft_k + k;
}

constexpr int64_t NONE = INT64_MIN;  // "no vertex" (ghost vertices of the x = -1 plane are negative)

__device__ __forceinline__ bool owned(const Geo &g, int64_t v) { return v >= 0 && v < g.n; }

enum { FLAG_OVERFLOW = 1, FLAG_BAD_BAND = 2 };

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() { return (1u << lane_id()) - 1u; }
__device__ __forceinline__ int64_t gwarp() { return ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; }
__device__ __forceinline__ int64_t nwarps() { return ((int64_t)gridDim.x * blockDim.x) >> 5; }

// "Minimal" arc set (R2): lateral arc (x,y,z) -> (nbr, zo(z)); the unique
// lateral in-arc of (x,y,z) per direction comes from (nbr, zi(z)).
__device__ __forceinline__ int zo_of(int z, int delta) { return z == 0 ? 0 : (z > delta ? z - delta : -1); }
__device__ __forceinline__ int zi_of(int z, int delta, int Z) { return z == 0 ? 0 : (z + delta < Z ? z + delta : -1); }
// edge intervals (NEXT-3): dl_out(d) is that of v's own lateral arc toward direction d (0:+x 1:-x
// 2:+y 3:-y); dl_in(d) that of the arc INTO v from its neighbour in direction d, i.e. the
// neighbour's arc toward d^1 -- the in-arc of (x,y,z) from direction d leaves (nbr_d, zi(z)) with
// zi computed from dl_in(d)
__device__ __forceinline__ int dl_out(const Geo &g, int d) { return g.dl[d]; }
__device__ __forceinline__ int dl_in(const Geo &g, int d) { return g.dl[d ^ 1]; }

// neighbour column offset (in vertices) in direction d, 0 if the neighbour is outside the slab
__device__ __forceinline__ int64_t nbr_off(const Geo &g, int x, int y, int d) {
    switch (d) {
        case 0: return (x + 1 < g.X || g.gh) ? g.YZ : 0;
        case 1: return (x >= 1 || g.gl) ? -g.YZ : 0;
        case 2: return y + 1 < g.Y ? (int64_t)g.Z : 0;
        default: return y >= 1 ? -(int64_t)g.Z : 0;
    }
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ int warp_max_i(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
    return v;
}
__device__ __forceinline__ int warp_incl_scan(int v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(FULL, v, o);
        if (lane_id() >= o) v += t;
    }
    return v;
}

// Warp-aggregated append of one optional item per lane: one atomic per warp.
__device__ __forceinline__ void warp_append(bool has, int item, int *list, unsigned *count) {
    const unsigned m = __ballot_sync(FULL, has);
    if (!m) return;
    unsigned base = 0;
    if (lane_id() == 0) base = atomicAdd(count, (unsigned)__popc(m));
    base = __shfl_sync(FULL, base, 0);
    if (has) list[base + __popc(m & lanemask_lt())] = item;
}

// Span append: a warp collects up to SPAN lane masks (item j of lane l = base_j + l) and
// appends all selected items with ONE atomic (dense list builders would otherwise put one
// atomic per 32 items on a single counter).
template <int SPAN>
struct SpanAppender {
    unsigned m[SPAN];
    int64_t b[SPAN];
    int k = 0;
    __device__ __forceinline__ void add(unsigned mask, int64_t base) {
        m[k] = mask;
        b[k] = base;
        ++k;
    }
    __device__ __forceinline__ void flush(int *list, unsigned *count) {
        int tot = 0;
#pragma unroll
        for (int j = 0; j < SPAN; j++)
            if (j < k) tot += __popc(m[j]);
        if (tot) {
            unsigned base = 0;
            if (lane_id() == 0) base = atomicAdd(count, (unsigned)tot);
            base = __shfl_sync(FULL, base, 0);
#pragma unroll
            for (int j = 0; j < SPAN; j++) {
                if (j >= k) break;
                if ((m[j] >> lane_id()) & 1u) list[base + __popc(m[j] & lanemask_lt())] = (int)(b[j] + lane_id());
                base += __popc(m[j]);
            }
        }
        k = 0;
    }
};

// Mark a chunk / column id (or -1) for the next worklist, de-duplicated inside the warp
// (__match_any_sync) and across warps (stamp[id] == tag means "already listed").
__device__ __forceinline__ void warp_mark(int id, int *stamp, int tag, int *list, unsigned *count) {
    const unsigned peers = __match_any_sync(FULL, id);
    bool add = id >= 0 && (__ffs(peers) - 1) == lane_id();
    if (add) add = (stamp[id] != tag) && (atomicExch(&stamp[id], tag) != tag);
    warp_append(add, id, list, count);
}

}  // namespace cg
