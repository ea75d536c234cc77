// tools/h2d_gather.cu -- moving the general path's view samples from pinned
// host memory to the GPU, config-4 shape (N = 2^20 complex128, d = 256,
// L = 4096, 9 random shifts + a 6-sample consecutive window per d-block):
//   (a) zero-copy: a kernel reads the 16-B samples through UVA (what
//       solve_host_batch does now);
//   (b) the copy engine: one cudaMemcpy2DAsync per view (width 16 B, pitch
//       d*16 B, height L) into a device window buffer;
//   (c) the whole signal by one H2D copy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o h2d_gather h2d_gather.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int64_t N = 1 << 20, D = 256, L = N / D;
constexpr int NV = 15;

__global__ void zc_gather(const double2 *__restrict__ x, const int *__restrict__ shifts, int nsig,
                          double2 *__restrict__ out) {
    const int64_t total = (int64_t)nsig * NV * L;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = i % L, v = (i / L) % NV, b = i / (L * NV);
        out[i] = x[b * N + j * D + shifts[v]];
    }
}

int main() {
    const int nsig = 16;
    double2 *h, *dwin, *dsig;
    int *dsh;
    if (cudaHostAlloc(&h, size_t(nsig) * N * 16, cudaHostAllocMapped) != cudaSuccess) return 1;
    for (int64_t i = 0; i < int64_t(nsig) * N; i++) h[i] = make_double2(double(i & 1023), 1.0);
    cudaMalloc(&dwin, size_t(nsig) * NV * L * 16);
    cudaMalloc(&dsig, size_t(N) * 16);
    int sh[NV] = {0, 1, 2, 3, 4, 5, 17, 45, 77, 101, 133, 160, 199, 222, 250};
    cudaMalloc(&dsh, sizeof(sh));
    cudaMemcpy(dsh, sh, sizeof(sh), cudaMemcpyHostToDevice);
    double2 *hd;
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        zc_gather<<<148 * 8, 256>>>(hd, dsh, nsig, dwin);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("(a) zero-copy gather: %.3f ms per signal (%.0f signals/s)\n", ms / nsig, nsig / (ms * 1e-3));
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        for (int s = 0; s < nsig; s++)
            for (int v = 0; v < NV; v++)
                cudaMemcpy2DAsync(dwin + (int64_t(s) * NV + v) * L, 16, h + int64_t(s) * N + sh[v], D * 16, 16, L,
                                  cudaMemcpyHostToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("(b) copy-engine 2D per view: %.3f ms per signal (%.0f signals/s)\n", ms / nsig, nsig / (ms * 1e-3));
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        for (int s = 0; s < nsig; s++) cudaMemcpyAsync(dsig, h + int64_t(s) * N, N * 16, cudaMemcpyHostToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("(c) whole-signal H2D: %.3f ms per signal (%.0f signals/s)\n", ms / nsig, nsig / (ms * 1e-3));
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
