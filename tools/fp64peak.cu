// tools/fp64peak.cu -- FP64 FMA throughput microbenchmark (the
// FP64 peak is not in MEASURED_PEAKS.json; the general-path kernels report
// their FP64 pipe fraction against this number).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64peak fp64peak.cu
// Each thread runs ACC independent DFMA chains (enough to cover the pipe
// latency); the grid is a multiple of the SM count.  2 flop per DFMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int ACC>
__global__ void __launch_bounds__(256) fma_chain(double *out, int iters, double a, double b) {
    double acc[ACC];
#pragma unroll
    for (int i = 0; i < ACC; i++) acc[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < ACC; i++) acc[i] = fma(acc[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < ACC; i++) s += acc[i];
    if (s == 1.2345) out[blockIdx.x] = s;
}

template <int ACC>
static void run(int sms, int ctas_per_sm) {
    double *out;
    cudaMalloc(&out, sizeof(double) * sms * ctas_per_sm);
    const int iters = 1 << 14;
    const dim3 grid(sms * ctas_per_sm), block(256);
    fma_chain<ACC><<<grid, block>>>(out, iters, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        fma_chain<ACC><<<grid, block>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * ACC * double(iters) * grid.x * block.x;
    printf("{\"acc\": %d, \"ctas_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", ACC, ctas_per_sm, best,
           flops / (best * 1e-3) / 1e12);
    cudaFree(out);
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    run<4>(sms, 4);
    run<8>(sms, 4);
    run<8>(sms, 8);
    run<16>(sms, 4);
    run<16>(sms, 8);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
        printf("error: %s\n", cudaGetErrorString(err));
        return 1;
    }
    return 0;
}
