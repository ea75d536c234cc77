// Where does one multi-collision decode trial spend its cycles?  Runs the
// cooperative trial (decode_coop.cuh) and the one-thread trial (decode.cuh)
// of one synthetic a-collision bin, `reps` times in a row in one warp, with
// clock64 stamps between the phases: the first repetition fetches its
// instructions cold, the later ones show the dependent-issue chain alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 \
//        -o tools/decode_phases tools/decode_phases.cu && tools/decode_phases
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ long long g_clk[16];
#define SFDT_COOP_CLK(i) do { if (threadIdx.x == 0) g_clk[i] = clock64(); } while (0)
#include "../paper_1407_8315_b200/csrc/decode_coop.cuh"

using namespace sfdt;

template <int A>
__global__ void k_phases(const cx *syn_in, int64_t n, int64_t m, int64_t bin, int reps, long long *out,
                         int *acc) {
    const int g = threadIdx.x & 7;
    cx syn[8];
    for (int s = 0; s < 8; s++) syn[s] = syn_in[s];
    for (int r = 0; r < reps; r++) {
        __syncwarp();
        const long long t0 = clock64();
        DecodedCoop o;
        decode_try_coop<A, 8>(syn, n, m, bin, g, o);
        if (threadIdx.x == 0) {
            out[r * 16 + 0] = t0;
            for (int i = 1; i <= 7; i++) out[r * 16 + i] = g_clk[i];
            acc[r] = o.accept;
        }
        // perturb so the compiler cannot hoist the repetition
        syn[0].re += (double)(o.loc[0] & 1) * 1e-300;
    }
}

template <int A>
__global__ void k_thread(const cx *syn_in, int64_t n, int64_t m, int64_t bin, int reps, long long *out,
                         int *acc) {
    cx syn[8];
    for (int s = 0; s < 8; s++) syn[s] = syn_in[s];
    for (int r = 0; r < reps; r++) {
        const long long t0 = clock64();
        Decoded o;
        decode_try_t<A, 8>(syn, n, m, bin, o);
        const long long t1 = clock64();
        out[r * 16] = t1 - t0;
        acc[r] = o.accept;
        syn[0].re += (double)(o.loc[0] & 1) * 1e-300;
    }
}

template <int A>
static void run(int reps) {
    const int64_t n = 1 << 20, m = 1024, bin = 37;
    std::vector<double> syn(16, 0.0);
    for (int j = 0; j < A; j++) {
        const int64_t loc = bin + m * (int64_t)(17 + 211 * j);
        const double mag = 1.0 + 2.0 * j, ph = 0.3 + j;
        for (int l = 0; l < 8; l++) {
            const double th = 2 * M_PI * (double)((loc * l) % n) / (double)n;
            syn[2 * l] += mag * cos(th + ph);
            syn[2 * l + 1] += mag * sin(th + ph);
        }
    }
    cx *d_syn; long long *d_out; int *d_acc;
    cudaMalloc(&d_syn, 128); cudaMalloc(&d_out, reps * 16 * 8); cudaMalloc(&d_acc, reps * 4);
    cudaMemcpy(d_syn, syn.data(), 128, cudaMemcpyHostToDevice);
    std::vector<long long> out(reps * 16); std::vector<int> acc(reps);
    k_phases<A><<<1, 32>>>(d_syn, n, m, bin, reps, d_out, d_acc);
    cudaMemcpy(out.data(), d_out, reps * 16 * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(acc.data(), d_acc, reps * 4, cudaMemcpyDeviceToHost);
    for (int r = 0; r < reps; r++) {
        printf("coop a=%d rep %d accept=%d total %6lld | scale %5lld hankel %5lld roots %5lld resid %5lld vand %5lld snap %5lld cons %5lld\n",
               A, r, acc[r], out[r * 16 + 7] - out[r * 16], out[r * 16 + 1] - out[r * 16],
               out[r * 16 + 2] - out[r * 16 + 1], out[r * 16 + 3] - out[r * 16 + 2], out[r * 16 + 4] - out[r * 16 + 3],
               out[r * 16 + 5] - out[r * 16 + 4], out[r * 16 + 6] - out[r * 16 + 5], out[r * 16 + 7] - out[r * 16 + 6]);
    }
    k_thread<A><<<1, 32>>>(d_syn, n, m, bin, reps, d_out, d_acc);
    cudaMemcpy(out.data(), d_out, reps * 16 * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(acc.data(), d_acc, reps * 4, cudaMemcpyDeviceToHost);
    for (int r = 0; r < reps; r++) printf("thread a=%d rep %d accept=%d total %6lld\n", A, r, acc[r], out[r * 16]);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}

int main() {
    run<2>(3);
    run<3>(3);
    run<4>(3);
    return 0;
}
