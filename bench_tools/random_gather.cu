// random_gather.cu -- the access-pattern roofline of the push-relabel walk:
// throughput of scattered 32-byte record reads (one AoS vertex record per read, the walk's
// unit access) over a buffer far larger than L2, with independent reads in flight (a bound
// for latency-bound traversals), compared with the streaming copy peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o random_gather random_gather.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// each thread reads `per` random 32-byte records (2 x int4) and folds them into one value
__global__ void gather(const int4 *__restrict__ rec, uint64_t nrec, int per, uint64_t seed, int *out) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int acc = 0;
#pragma unroll 4
    for (int i = 0; i < per; i++) {
        const uint64_t r = mix(seed ^ (tid * 0x100000001b3ull + i)) % nrec;
        const int4 a = __ldcg(&rec[2 * r]), b = __ldcg(&rec[2 * r + 1]);
        acc += a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
    }
    if (acc == 0x7fffffff) out[0] = acc;  // keep the loads alive
}

__global__ void copyk(const int4 *__restrict__ a, int4 *__restrict__ b, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

int main() {
    const uint64_t bytes = 2ull << 30, nrec = bytes / 32;
    int4 *buf, *buf2;
    int *out;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&buf2, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(buf, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best_copy = 1e9;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        copyk<<<sms * 8, 256>>>(buf, buf2, bytes / 16);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best_copy) best_copy = ms;
    }
    printf("{\"copy_gbs\": %.1f", 2.0 * bytes / best_copy / 1e6);
    const int per = 64;
    for (int blocks_per_sm : {4, 8, 16, 32}) {
        const uint64_t threads = (uint64_t)sms * blocks_per_sm * 256;
        float best = 1e9;
        for (int rep = 0; rep < 5; rep++) {
            cudaEventRecord(e0);
            gather<<<sms * blocks_per_sm, 256>>>(buf, nrec, per, 1234 + rep, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double recs = (double)threads * per;
        printf(", \"gather_%dblk_gbs\": %.1f, \"gather_%dblk_grecs_per_s\": %.2f", blocks_per_sm,
               recs * 32 / best / 1e6, blocks_per_sm, recs / best / 1e6);
    }
    printf(", \"buffer_gib\": 2, \"record_bytes\": 32}\n");
    return cudaGetLastError() != cudaSuccess;
}
