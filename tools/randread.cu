// tools/randread.cu -- random-access read rate on B200: the ceiling of the
// general path's random-shift view gather (one 16-B complex128 sample per
// d-block per random shift).
//
// Every group of G adjacent lanes reads G adjacent 16-B elements (16·G bytes)
// at a random 16·G-aligned position of a 16-GiB buffer (>> 126 MB L2, so
// every access misses).  Reports accesses/s (one access = one group's
// contiguous run) and useful GB/s, for the default load and for the
// L2::64B prefetch-size hint (SFDT_GATHER_HINT=1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o randread randread.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int G, int HINT, int UNROLL>
__global__ void __launch_bounds__(256) rr(const double2 *__restrict__ x, int64_t nmask_groups, int rounds,
                                          double *__restrict__ out) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t grp = tid / G;
    const int lane = (int)(tid % G);
    double acc = 0.0;
    for (int r = 0; r < rounds; r += UNROLL) {
        double2 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const int64_t gi = (int64_t)(mix((uint64_t)grp * 1000003ull + r + u) & (uint64_t)nmask_groups);
            const double2 *p = x + gi * G + lane;
            if (HINT == 1)
                asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.f64 {%0,%1}, [%2];"
                             : "=d"(v[u].x), "=d"(v[u].y) : "l"(p));
            else
                v[u] = __ldg(p);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++) acc += v[u].x + v[u].y;
    }
    if (acc == 1.2345) out[0] = acc;
}

// Blocked variant: groups of BL lanes read BL random 16-B samples inside the
// same random 4-KiB block (one random shift per lane, like the random-shift
// views of one d-block at d = 256): does DRAM page locality lift the rate?
template <int BL, int UNROLL>
__global__ void __launch_bounds__(256) rrb(const double2 *__restrict__ x, int64_t nmask_blocks, int rounds,
                                           double *__restrict__ out) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t grp = tid / BL;
    double acc = 0.0;
    for (int r = 0; r < rounds; r += UNROLL) {
        double2 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const uint64_t h = mix((uint64_t)grp * 1000003ull + r + u);
            const int64_t blk = (int64_t)(h & (uint64_t)nmask_blocks);
            const int64_t off = (int64_t)(mix(h + threadIdx.x) & 255);   // sample within the 4-KiB block
            v[u] = __ldg(x + blk * 256 + off);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++) acc += v[u].x + v[u].y;
    }
    if (acc == 1.2345) out[0] = acc;
}

template <int BL>
void runb(const double2 *x, int64_t n, double *out) {
    const int blocks = 148 * 8, rounds = 64;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; rep++) rrb<BL, 8><<<blocks, 256>>>(x, n / 256 - 1, rounds, out);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(a);
        rrb<BL, 8><<<blocks, 256>>>(x, n / 256 - 1, rounds, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double acc = double(blocks) * 256 * rounds;
    printf("blocked: %2d random 16-B samples per random 4-KiB block: %.3f ms, %.1f G accesses/s\n", BL, best,
           acc / (best * 1e-3) / 1e9);
}

template <int G, int HINT>
void run(const double2 *x, int64_t n, double *out) {
    const int blocks = 148 * 8, rounds = 64;
    const int64_t groups = n / G;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; rep++) rr<G, HINT, 8><<<blocks, 256>>>(x, groups - 1, rounds, out);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(a);
        rr<G, HINT, 8><<<blocks, 256>>>(x, groups - 1, rounds, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double acc = double(blocks) * 256 / G * rounds;
    printf("G=%d (%3d B contiguous) hint=%d: %.3f ms, %.1f G accesses/s, %.0f GB/s useful\n", G, 16 * G, HINT,
           best, acc / (best * 1e-3) / 1e9, acc * 16 * G / (best * 1e-3) / 1e9);
}

int main() {
    const int64_t n = int64_t(1) << 30;   // 1 Gi complex128 = 16 GiB
    double2 *x;
    double *out;
    if (cudaMalloc(&x, n * sizeof(double2)) != cudaSuccess) return 1;
    cudaMalloc(&out, 8);
    cudaMemset(x, 0, n * sizeof(double2));
    run<1, 0>(x, n, out);
    run<1, 1>(x, n, out);
    run<2, 0>(x, n, out);
    run<2, 1>(x, n, out);
    run<4, 0>(x, n, out);
    run<8, 0>(x, n, out);
    run<16, 0>(x, n, out);
    runb<1>(x, n, out);
    runb<9>(x, n, out);
    runb<16>(x, n, out);
    runb<32>(x, n, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
