// tools/membw.cu -- read-bandwidth microbenchmark for the k_stream design
// space on B200 (sum of squares over a large complex128 buffer).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membw membw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int THREADS, int UNROLL, int MODE>
__global__ void __launch_bounds__(THREADS) rd(const double2 *__restrict__ x, int64_t n, int64_t CH,
                                              double *__restrict__ out) {
    const int64_t base = int64_t(blockIdx.x) * CH;
    double acc = 0.0;
    for (int64_t off = 0; off < CH; off += int64_t(THREADS) * UNROLL) {
        double2 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const double2 *p = x + base + off + int64_t(u) * THREADS + threadIdx.x;
            if (MODE == 0) v[u] = __ldcs(p);
            else if (MODE == 1) v[u] = __ldg(p);
            else {
                double2 r;
                asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                             : "=d"(r.x), "=d"(r.y) : "l"(p));
                v[u] = r;
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++) acc = fma(v[u].x, v[u].x, fma(v[u].y, v[u].y, acc));
    }
    if (acc == 1.2345) out[blockIdx.x] = acc;
}

// 32-byte-per-thread variant: each thread loads two adjacent complex values
template <int THREADS, int UNROLL, int EF>
__global__ void __launch_bounds__(THREADS) rd32(const double4 *__restrict__ x, int64_t n4, int64_t CH4,
                                                double *__restrict__ out) {
    const int64_t base = int64_t(blockIdx.x) * CH4;
    double acc = 0.0;
    for (int64_t off = 0; off < CH4; off += int64_t(THREADS) * UNROLL) {
        double4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const double4 *p = x + base + off + int64_t(u) * THREADS + threadIdx.x;
            if (EF)
                asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                             : "=d"(v[u].x), "=d"(v[u].y), "=d"(v[u].z), "=d"(v[u].w) : "l"(p));
            else
                asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                             : "=d"(v[u].x), "=d"(v[u].y), "=d"(v[u].z), "=d"(v[u].w) : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++)
            acc = fma(v[u].x, v[u].x, fma(v[u].y, v[u].y, fma(v[u].z, v[u].z, fma(v[u].w, v[u].w, acc))));
    }
    if (acc == 1.2345) out[blockIdx.x] = acc;
}

template <int THREADS, int UNROLL>
__global__ void __launch_bounds__(THREADS) rd32s(const double4 *__restrict__ x, int64_t n4, int64_t CH4,
                                                 double *__restrict__ out) {
    extern __shared__ double dummy[];
    const int64_t base = int64_t(blockIdx.x) * CH4;
    double acc = 0.0;
    for (int64_t off = 0; off < CH4; off += int64_t(THREADS) * UNROLL) {
        double4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const double4 *p = x + base + off + int64_t(u) * THREADS + threadIdx.x;
            asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(v[u].x), "=d"(v[u].y), "=d"(v[u].z), "=d"(v[u].w) : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++)
            acc = fma(v[u].x, v[u].x, fma(v[u].y, v[u].y, fma(v[u].z, v[u].z, fma(v[u].w, v[u].w, acc))));
    }
    if (acc == 1.2345) { dummy[0] = acc; out[blockIdx.x] = dummy[threadIdx.x & 7]; }
}

template <typename F>
float timeit(F f, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    for (int i = 0; i < reps; i++) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    const int64_t n = int64_t(1) << 32;   // 4G complex128 = 64 GiB
    double2 *x;
    if (cudaMalloc(&x, n * 16) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(x, 0, n * 16);
    double *out;
    cudaMalloc(&out, 1 << 24);
    const double gb = n * 16 / 1e9;
#define RUN(T, U, M, CH)                                                                       \
    {                                                                                          \
        float ms = timeit([&] { rd<T, U, M><<<(unsigned)(n / CH), T>>>(x, n, CH, out); }, 5); \
        printf("rd T=%d U=%d mode=%d CH=%d : %.3f ms  %.1f GB/s\n", T, U, M, (int)CH, ms, gb / ms * 1e3); \
    }
    RUN(256, 8, 0, 16384);
    RUN(256, 16, 0, 16384);
    RUN(512, 8, 0, 16384);
    RUN(256, 8, 2, 16384);
    RUN(256, 16, 2, 16384);
    RUN(256, 8, 0, 65536);
    RUN(128, 16, 0, 16384);
    RUN(1024, 4, 0, 16384);
#define RUN32(T, U, CH4, EF)                                                                          \
    {                                                                                             \
        float ms = timeit([&] { rd32<T, U, EF><<<(unsigned)(n / 2 / CH4), T>>>((const double4 *)x, n / 2, CH4, out); }, 5); \
        printf("rd32 T=%d U=%d CH4=%d ef=%d : %.3f ms  %.1f GB/s\n", T, U, (int)CH4, EF, ms, gb / ms * 1e3); \
    }
    RUN32(256, 4, 8192, 0);
    RUN32(256, 8, 8192, 0);
    RUN32(512, 4, 8192, 0);
    RUN32(256, 4, 8192, 1);
    RUN32(256, 8, 8192, 1);
    RUN32(256, 8, 32768, 1);
#define RUNS(T, U, CH4, SMEM)                                                                      \
    {                                                                                             \
        cudaFuncSetAttribute(rd32s<T, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);     \
        float ms = timeit([&] { rd32s<T, U><<<(unsigned)(n / 2 / CH4), T, SMEM>>>((const double4 *)x, n / 2, CH4, out); }, 5); \
        printf("rd32s T=%d U=%d CH4=%d smem=%d : %.3f ms  %.1f GB/s\n", T, U, (int)CH4, SMEM, ms, gb / ms * 1e3); \
    }
    RUNS(512, 4, 8192, 0);
    RUNS(512, 4, 8192, 60000);
    RUNS(512, 4, 8192, 80000);
    RUNS(512, 8, 8192, 80000);
    RUNS(1024, 4, 8192, 120000);
    RUNS(1024, 8, 8192, 120000);
    RUNS(256, 8, 8192, 60000);
    RUNS(256, 16, 8192, 60000);
    return 0;
}
