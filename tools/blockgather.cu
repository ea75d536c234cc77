// tools/blockgather.cu -- the general path's view gather as a separate
// "window" pass: lanes over a signal's views, one warp
// instruction per pair of d-blocks, W[b][m][v] rows of 256 B written
// coalesced.  Config-4 shape: B = 1024 signals of N = 2^20 complex128,
// d = 256 (L = 4096 d-blocks of 4 KiB), 15 views = shifts 0..5 (one 128-B
// line) + 9 random shifts in [0, 256).
//
// Measures the gather alone (the FFT would then read W), for the default
// load, the L2::64B prefetch-size hint and L2::evict_first, and with W either
// the whole batch (1 GiB, spills to DRAM) or a ring of RING signals (stays in
// L2 when the chunks are consumed right away).  Lines/s = distinct 128-B
// lines touched per second (1 + distinct random lines per d-block).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o blockgather blockgather.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <set>
#include <cuda_runtime.h>

constexpr int NVP = 16;   // padded views per d-block row

template <int MODE>
__device__ __forceinline__ double2 ld(const double2 *p) {
    double2 v;
    if (MODE == 1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    else if (MODE == 2)
    {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                     : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    }
    else if (MODE == 3)
        asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    else
        v = __ldg(p);
    return v;
}

// CTA = 256 threads = 16 half-warps; half-warp h, step u handles d-block
// m = tile*TILE + u*16 + h of signal b; lane (0..15) = view.
template <int MODE, int U>
__global__ void __launch_bounds__(256) k_window(const double2 *__restrict__ x, int64_t n, int d, int L,
                                                const int *__restrict__ shifts /* B x NVP */, int nv,
                                                double2 *__restrict__ W, int64_t ring /* signals */) {
    const int tiles = L / (16 * U);
    const int64_t b = blockIdx.x / tiles;
    const int tile = blockIdx.x % tiles;
    const int v = threadIdx.x & 15, h = threadIdx.x >> 4;
    if (v >= nv) return;
    const int sh = shifts[b * NVP + v];
    const double2 *xs = x + b * n + sh;
    double2 *wr = W + ((b % ring) * L) * NVP + v;
    double2 val[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int m = tile * (16 * U) + u * 16 + h;
        val[u] = ld<MODE>(xs + (int64_t)m * d);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int m = tile * (16 * U) + u * 16 + h;
        wr[(int64_t)m * NVP] = val[u];
    }
}

// the fused kernel's pattern for comparison: CTA = one view, lanes walk the
// d-blocks (each lane's sample is in a different 4-KiB block)
template <int MODE, int U>
__global__ void __launch_bounds__(256) k_perview(const double2 *__restrict__ x, int64_t n, int d, int L,
                                                 const int *__restrict__ shifts, int nv,
                                                 double2 *__restrict__ W, int64_t ring) {
    const int64_t b = blockIdx.x / nv;
    const int v = blockIdx.x % nv;
    const int sh = shifts[b * NVP + v];
    const double2 *xs = x + b * n + sh;
    double2 *wr = W + (((b % ring) * nv + v) * (int64_t)L);
    for (int m0 = threadIdx.x; m0 < L; m0 += 256 * U) {
        double2 val[U];
#pragma unroll
        for (int u = 0; u < U; u++) val[u] = ld<MODE>(xs + (int64_t)(m0 + u * 256) * d);
#pragma unroll
        for (int u = 0; u < U; u++) wr[m0 + u * 256] = val[u];
    }
}

template <typename F>
float timeit(F &&launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    launch();
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    const int64_t B = 1024, n = int64_t(1) << 20;
    const int d = 256, L = 4096, nv = 15;
    double2 *x, *W;
    int *shifts;
    if (cudaMalloc(&x, B * n * sizeof(double2)) != cudaSuccess) return 1;
    if (cudaMalloc(&W, B * L * NVP * sizeof(double2)) != cudaSuccess) return 1;
    cudaMalloc(&shifts, B * NVP * 4);
    cudaMemset(x, 0, B * n * sizeof(double2));
    std::vector<int> hs(B * NVP, 0);
    srand(12345);
    double lines = 0;
    for (int64_t b = 0; b < B; b++) {
        std::set<int> used, ls;
        for (int v = 0; v < 6; v++) { hs[b * NVP + v] = v; used.insert(v); }
        ls.insert(0);
        for (int v = 6; v < nv; v++) {
            int s;
            do s = rand() % d; while (used.count(s));
            used.insert(s);
            hs[b * NVP + v] = s;
            ls.insert(s / 8);
        }
        lines += double(ls.size()) * L;
    }
    cudaMemcpy(shifts, hs.data(), B * NVP * 4, cudaMemcpyHostToDevice);
    printf("B=%lld signals, %d views, %.1fM samples, %.1fM distinct 128-B lines (%.2f GB)\n", (long long)B, nv,
           double(B) * L * nv / 1e6, lines / 1e6, lines * 128 / 1e9);
    auto report = [&](const char *name, int mode, int64_t ring, float ms) {
        printf("%-10s mode=%d ring=%4lld: %.3f ms  %.1f G lines/s  %.1f G samples/s\n", name, mode,
               (long long)ring, ms, lines / (ms * 1e-3) / 1e9, double(B) * L * nv / (ms * 1e-3) / 1e9);
    };
    for (int64_t ring : {B, int64_t(32)}) {
        constexpr int U = 8;
        const unsigned grid = (unsigned)(B * (L / (16 * U)));
        report("window", 0, ring, timeit([&] { k_window<0, U><<<grid, 256>>>(x, n, d, L, shifts, nv, W, ring); }));
        report("window", 1, ring, timeit([&] { k_window<1, U><<<grid, 256>>>(x, n, d, L, shifts, nv, W, ring); }));
        report("window", 2, ring, timeit([&] { k_window<2, U><<<grid, 256>>>(x, n, d, L, shifts, nv, W, ring); }));
        report("window", 3, ring, timeit([&] { k_window<3, U><<<grid, 256>>>(x, n, d, L, shifts, nv, W, ring); }));
        const unsigned g2 = (unsigned)(B * nv);
        report("perview", 0, ring, timeit([&] { k_perview<0, 8><<<g2, 256>>>(x, n, d, L, shifts, nv, W, ring); }));
        report("perview", 1, ring, timeit([&] { k_perview<1, 8><<<g2, 256>>>(x, n, d, L, shifts, nv, W, ring); }));
    }
    {
        constexpr int U = 16;
        const unsigned grid = (unsigned)(B * (L / (16 * U)));
        report("window16", 0, 32, timeit([&] { k_window<0, U><<<grid, 256>>>(x, n, d, L, shifts, nv, W, 32); }));
        report("window16", 1, 32, timeit([&] { k_window<1, U><<<grid, 256>>>(x, n, d, L, shifts, nv, W, 32); }));
    }
    {
        constexpr int U = 4;
        const unsigned grid = (unsigned)(B * (L / (16 * U)));
        report("window4", 0, 32, timeit([&] { k_window<0, U><<<grid, 256>>>(x, n, d, L, shifts, nv, W, 32); }));
        report("window4", 1, 32, timeit([&] { k_window<1, U><<<grid, 256>>>(x, n, d, L, shifts, nv, W, 32); }));
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
